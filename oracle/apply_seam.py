"""Apply INTEGRATION.md's B200-lane stub to a scratch copy of the reference
package -- TEST INFRASTRUCTURE ONLY (tests/test_reference_seam.py).

The pristine copy is oracle/_ref/txfem_pkg (staged by oracle/build_ref.sh from
/root/reference/pkg; git-ignored, travels to the GPU box).  The two python
blocks marked ``<!-- seam:backend -->`` and ``<!-- seam:executor -->`` in
INTEGRATION.md are appended verbatim to txfem/backend.py and
txfem/executor.py of the copy -- the edit a maintainer of the reference makes.

    python oracle/apply_seam.py DEST     # -> DEST/src/txfem (patched), DEST/tests
"""

from __future__ import annotations

import re
import shutil
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
REPO = HERE.parent
PRISTINE = HERE / "_ref" / "txfem_pkg"


def seam_blocks(doc: Path = REPO / "INTEGRATION.md") -> dict:
    text = doc.read_text()
    out = {}
    for name in ("backend", "executor"):
        m = re.search(r"<!-- seam:%s -->\s*```python\n(.*?)```" % name, text, re.S)
        if not m:
            raise ValueError(f"INTEGRATION.md has no seam:{name} block")
        out[name] = m.group(1)
    return out


def apply(dest: Path) -> Path:
    if not (PRISTINE / "src" / "txfem").exists():
        raise FileNotFoundError(f"{PRISTINE} missing: run oracle/build_ref.sh where /root/reference exists")
    dest = Path(dest)
    if dest.exists():
        shutil.rmtree(dest)
    shutil.copytree(PRISTINE, dest, ignore=shutil.ignore_patterns("__pycache__"))
    blocks = seam_blocks()
    for name in ("backend", "executor"):
        f = dest / "src" / "txfem" / f"{name}.py"
        f.write_text(f.read_text().rstrip("\n") + "\n\n\n" + blocks[name])
    return dest


if __name__ == "__main__":
    print(apply(Path(sys.argv[1])))
