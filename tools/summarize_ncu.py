"""Summarise ncu outputs from gpurun_out/ into profiles/ (committed evidence).

python tools/summarize_ncu.py TAG
  reads  gpurun_out/TAG_launches.csv          (ncu --metrics gpu__time_duration.sum)
         gpurun_out/TAG_prof_*.ncu-rep         (ncu --set full, one launch each)
  writes profiles/TAG_ncu.md                   (launch shares + key metrics + top stalls)
  (profiles/ncu_traffic.json -- the write-back-inclusive traffic bench.py reads -- is tools/traffic.py's)
"""
import collections
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
OUT = REPO / "gpurun_out"
PROF = REPO / "profiles"

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__cycles_elapsed.avg", "sm__cycles_active.avg", "smsp__cycles_active.avg",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "launch__shared_mem_per_block_dynamic", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__average_warp_latency_issue_stalled_barrier", "gpc__cycles_elapsed.max", "dram__cycles_active.avg",
]
TO_NS = {"nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}
TO_B = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def launch_shares(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, data = rows[0], rows[1:]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in data:
        v = float(r[iv].replace(",", "")) * TO_NS.get(r[iu], 1.0)
        name = r[ik].split("(")[0][:80]
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    lines = ["| kernel | launches | total us | mean us | share |", "|---|---:|---:|---:|---:|"]
    for n in sorted(tot, key=lambda n: -tot[n]):
        lines.append(f"| `{n}` | {cnt[n]} | {tot[n] / 1e3:.1f} | {tot[n] / cnt[n] / 1e3:.2f} | {100 * tot[n] / T:.1f}% |")
    return "\n".join(lines)


def raw_metrics(rep):
    txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {}
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            out[k] = (vals[i], units[i])
    return out, vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"


def top_stalls(rep, n=12):
    txt = subprocess.run(["ncu", "-i", str(rep), "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        return ""
    hdr, data = rows[1], rows[2:]
    i_src, i_ex = hdr.index("Source"), hdr.index("Instructions Executed")
    i_st = hdr.index("Warp Stall Sampling (All Samples)")
    tot = sum(int(r[i_st] or 0) for r in data) or 1
    lines = ["| SASS | executed | stall samples |", "|---|---:|---:|"]
    for r in sorted(data, key=lambda r: -int(r[i_st] or 0))[:n]:
        lines.append(f"| `{r[i_src].strip()[:70]}` | {r[i_ex]} | {100 * int(r[i_st] or 0) / tot:.1f}% |")
    ops = collections.Counter()
    for r in data:
        op = r[i_src].split()
        if not op:
            continue
        op = op[1] if op[0].startswith("@") else op[0]
        ops[op.split(".")[0]] += int(r[i_ex] or 0)
    lines.append("")
    lines.append("Executed warp instructions by opcode: " +
                 ", ".join(f"{k} {v}" for k, v in ops.most_common(14)))
    return "\n".join(lines)


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
    md = [f"# ncu summary `{tag}` (B200, `--clock-control none`)", ""]
    lpath = OUT / f"{tag}_launches.csv"
    if lpath.exists():
        md += ["## Launch list of `python bench.py --steps 20 --warmup 5 --no-variants --no-cpu --no-e2e`",
               "(cold-cache, serialised per-launch times: compare shares, not absolutes; the stream probe",
               "and torch fills are bench.py's measurement scaffolding, outside the timed region)", "",
               launch_shares(lpath), ""]
    for rep in sorted(OUT.glob(f"{tag}_prof_*.ncu-rep")):
        cfg = rep.stem.replace(f"{tag}_prof_", "")
        m, name = raw_metrics(rep)
        md += [f"## `{cfg}`: `{name[:110]}`", "", "| metric | value | unit |", "|---|---:|---|"]
        md += [f"| {k} | {v} | {u} |" for k, (v, u) in m.items()]
        rd = float(m["dram__bytes_read.sum"][0].replace(",", "")) * TO_B.get(m["dram__bytes_read.sum"][1], 1)
        wr = float(m["dram__bytes_write.sum"][0].replace(",", "")) * TO_B.get(m["dram__bytes_write.sum"][1], 1)
        md += ["", f"DRAM traffic inside the profiled launch (cold L2, write-back still pending at its end is "
                   f"not counted here; see *_traffic.md): read {rd / 1e6:.2f} MB + write {wr / 1e6:.2f} MB", "",
               "Top stall sites:", "", top_stalls(rep), ""]
    (PROF / f"{tag}_ncu.md").write_text("\n".join(md) + "\n")
    print("wrote", PROF / f"{tag}_ncu.md")


if __name__ == "__main__":
    main()
