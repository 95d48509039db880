// txb_jit_kernel.cuh — the thread-transposed integration kernel for a
// user-supplied physics form, compiled at run time by NVRTC (txb_jit.cu).
//
// Same schedule as the ahead-of-time kernel (txb_integrate.cu): persistent
// warp-specialised CTAs, one producer lane bulk-copying batches into a ring
// of shared-memory stages, consumer warps running the quadrature phase
// (lane <-> (cell, q)), a warp-scope transposition and the basis phase
// (lane <-> element entry (cell, b, c)).  What is generic here:
//   * the pointwise f1 and optional f0 are the user's source strings
//     (TXB_F1 / TXB_F0, the reference's f1_<name> / f0_<name> convention,
//     txfem/codegen.py:215-221), inlined;
//   * any number of auxiliary fields (TXB_NAUX), P0 or P1, with the P1
//     gradient when the form asks for it (txfem/_kernels_py.py:93-110);
//   * any tabulation: every chain starts at +0 and runs in the numpy lane's
//     order (txfem/_kernels_py.py:20-90), so the element vectors are
//     bit-identical to the reference's python lane for sources that evaluate
//     like their f1_many / f0_many.  Two entry points share the source:
//     txb_jit_integrate (any D table) and txb_jit_integrate_std (the standard
//     P1 table, chosen by the host when D is bitwise that table): there the
//     pulled-back gradients are T[0] = -invJ[0] - invJ[1] (- invJ[2]) and
//     T[b>=1] = invJ row b-1 -- the same values as the full chain up to the
//     sign of zero, which the +0-started consumer chains (grad u, grad a and
//     the basis-phase sums) absorb -- and only T[0] goes through the exchange
//     area (the basis phase reads the invJ rows from the stage).
//
// The including unit defines: real, TXB_DIM, TXB_NQ, TXB_NCOMP, TXB_NAUX,
// TXB_AUX_MODE (0 none, 1 P0, 2 P1), TXB_HAS_F0, TXB_GRAD_A, TXB_F1 and, with
// an f0, TXB_F0.
#pragma once

#include "txb_pipeline.cuh"

namespace txb {
namespace jit {

constexpr int D = TXB_DIM, NB = D + 1, NQ = TXB_NQ, NCOMP = TXB_NCOMP;
constexpr int NAUX = TXB_NAUX, AUXM = TXB_AUX_MODE, NAS = NAUX > 0 ? NAUX : 1;
constexpr bool HAS_F0 = TXB_HAS_F0 != 0, GRAD_A = TXB_GRAD_A != 0;
constexpr int DD = D * D, NBC = NB * NCOMP;
constexpr int AUXW = AUXM == 1 ? NAUX : (AUXM == 2 ? NB * NAUX : 0);
constexpr int CW = 32 / NQ;  // cells per warp slice
constexpr int S = (int)sizeof(real);
// warp-private exchange area, component-major: row r of T (r = (q*NB+b)*D+k),
// of f1s (r = (q*NCOMP+c)*D+k) and of f0s (r = q*NCOMP+c) holds the CW cells of
// the slice at pitch P = CW + 4.  The quadrature-phase stores (lane = cell) hit
// consecutive words; the basis-phase loads (lanes = (cell, b, c)) spread over
// the banks (the cell-major odd stride left 4-way conflicts on the T loads).
constexpr int P = CW + 4;
constexpr int NF1 = NQ * NCOMP * D, NF0 = HAS_F0 ? NQ * NCOMP : 0;
// STAGE_T: only T[0] goes through the exchange area, the basis phase reads
// the invJ rows from the stage (standard tables, cell-array entry points);
// the mesh entry points compute invJ in-kernel and keep every T row there.
template <bool STAGE_T>
struct Area {
  static constexpr int NTR = STAGE_T ? D : NQ * NB * D;  // rows of T in the exchange area
  static constexpr int BYTES = round_up(P * (NTR + NF1 + NF0) * S, 16);
};

// Mesh inputs of one batch: connectivity rows (stage or global), coordinates,
// global coefficients, the orientation flag and the batch's first cell.
struct MeshIn {
  const int64_t* ids;
  const double* X;
  const real* glob;
  unsigned long long* bad;
  int64_t c0_batch;
  // tiled entry points: the stage's local indices and its vertex table (structure of arrays)
  const unsigned char* s_local;
  const double* sx;
  const real* su;
  int vpitch, upitch, lb;
  // tiled with the caller's geometry: the batch's inv_j / det_j rows (stage or global)
  const real* g_inv;
  const real* g_det;
};

// Where a slice's per-cell inputs come from.
enum { SRC_CELLS = 0, SRC_MESH = 1, SRC_TILED = 2, SRC_TILED_GEOM = 3 };

__device__ __forceinline__ int inv_bytes(int n) { return round_up(n * DD * S, 16); }
__device__ __forceinline__ int det_bytes(int n) { return round_up(n * S, 16); }
__device__ __forceinline__ int coef_bytes(int n) { return round_up(n * NBC * S, 16); }
__device__ __forceinline__ int aux_bytes(int n) { return round_up(n * AUXW * S, 16); }

template <bool STD, bool VEC, int SRC>
__device__ __forceinline__ void warp_slice(const Tabulation<real>& tab, const real* __restrict__ s_inv,
                                           const real* __restrict__ s_det, const real* __restrict__ s_coef,
                                           const real* __restrict__ s_aux, real* __restrict__ scratch, int c0,
                                           int ncell, real* __restrict__ out, int lane, const MeshIn& mi) {
  constexpr bool MESH = SRC != SRC_CELLS;
  constexpr bool STAGE_T = STD && !MESH;
  real* s_tr = scratch;
  real* s_f1 = s_tr + P * Area<STAGE_T>::NTR;
  real* s_f0 = s_f1 + P * NF1;
  const int nc = min(CW, ncell - c0);

  // ---------------- quadrature phase: lane <-> (cell, q) ----------------
  const int lc = lane / NQ;
  const int q = lane - lc * NQ;
  if (lc < nc) {
    const int cell = c0 + lc;
    real J[DD];
    real cf[NBC];
    real det;
    if constexpr (SRC == SRC_TILED_GEOM) {
      // coefficients from the tile's table, the caller's geometry as given (run precision)
      int ids[NB];
      if (mi.lb == 1) {
        const uint32_t w = reinterpret_cast<const uint32_t*>(mi.s_local)[cell];
#pragma unroll
        for (int b = 0; b < NB; ++b) ids[b] = (w >> (8 * b)) & 0xffu;
      } else {
        const uint2 w = reinterpret_cast<const uint2*>(mi.s_local)[cell];
#pragma unroll
        for (int b = 0; b < NB; ++b) ids[b] = ((b < 2 ? w.x : w.y) >> (16 * (b & 1))) & 0xffffu;
      }
#pragma unroll
      for (int b = 0; b < NB; ++b)
#pragma unroll
        for (int c = 0; c < NCOMP; ++c) cf[b * NCOMP + c] = mi.su[c * mi.upitch + ids[b]];
#pragma unroll
      for (int i = 0; i < DD; ++i) J[i] = mi.g_inv[cell * DD + i];
      det = mi.g_det[cell];
    } else if constexpr (MESH) {
      // gather (mesh.py:202-217) and float64 geometry (mesh.py:150-190), cast once to the run
      // precision (executor.py:77-90): the reference's host steps, in-kernel
      double X[NB][D];
      if constexpr (SRC == SRC_TILED) {
        // the tile's vertex table in shared memory, through the cell's local indices
        int ids[NB];
        if (mi.lb == 1) {
          const uint32_t w = reinterpret_cast<const uint32_t*>(mi.s_local)[cell];
#pragma unroll
          for (int b = 0; b < NB; ++b) ids[b] = (w >> (8 * b)) & 0xffu;
        } else {
          const uint2 w = reinterpret_cast<const uint2*>(mi.s_local)[cell];
#pragma unroll
          for (int b = 0; b < NB; ++b) ids[b] = ((b < 2 ? w.x : w.y) >> (16 * (b & 1))) & 0xffffu;
        }
#pragma unroll
        for (int b = 0; b < NB; ++b)
#pragma unroll
          for (int c = 0; c < NCOMP; ++c) cf[b * NCOMP + c] = mi.su[c * mi.upitch + ids[b]];
#pragma unroll
        for (int b = 0; b < NB; ++b)
#pragma unroll
          for (int i = 0; i < D; ++i) X[b][i] = mi.sx[i * mi.vpitch + ids[b]];
      } else {
        int64_t ids[NB];
        load_row<int64_t, NB, VEC>(mi.ids + cell * NB, ids);
#pragma unroll
        for (int b = 0; b < NB; ++b)
#pragma unroll
          for (int c = 0; c < NCOMP; ++c) cf[b * NCOMP + c] = __ldg(mi.glob + ids[b] * NCOMP + c);
#pragma unroll
        for (int b = 0; b < NB; ++b)
#pragma unroll
          for (int i = 0; i < D; ++i) X[b][i] = __ldg(mi.X + ids[b] * D + i);
      }
      double detd;
      // branch-free quotients, signed zeros kept (user forms may see them);
      // exact division for the rare rejected cell
      cell_geometry<real, D, true>(X, J, det, detd);
      if (q == 0 && mi.bad && detd <= 0.0) atomicMin(mi.bad, (unsigned long long)(mi.c0_batch + cell));
    } else {
      load_row<real, DD, VEC>(s_inv + cell * DD, J);
      load_row_rot<real, NBC, VEC>(s_coef + cell * NBC, cf, lane);
      det = s_det[cell];
    }

    // pulled-back gradients T[b][k] = sum_j D[q][b][j] invJ[j][k]  (_kernels_py.py:78-90)
    real tr[NB][D];
    if constexpr (STD) {
#pragma unroll
      for (int k = 0; k < D; ++k) {
        real acc = -J[k];
#pragma unroll
        for (int j = 1; j < D; ++j) acc = add(acc, -J[j * D + k]);
        tr[0][k] = acc;
        if (STAGE_T && q == 0) s_tr[k * P + lc] = acc;
      }
#pragma unroll
      for (int b = 1; b < NB; ++b)
#pragma unroll
        for (int k = 0; k < D; ++k) tr[b][k] = J[(b - 1) * D + k];
      if constexpr (!STAGE_T) {
#pragma unroll
        for (int b = 0; b < NB; ++b)
#pragma unroll
          for (int k = 0; k < D; ++k) s_tr[((q * NB + b) * D + k) * P + lc] = tr[b][k];
      }
    } else {
#pragma unroll
      for (int b = 0; b < NB; ++b)
#pragma unroll
        for (int k = 0; k < D; ++k) {
          real acc = real(0);
#pragma unroll
          for (int j = 0; j < D; ++j) acc = add(acc, mul(tab.D[(q * NB + b) * D + j], J[j * D + k]));
          tr[b][k] = acc;
          s_tr[((q * NB + b) * D + k) * P + lc] = acc;
        }
    }

    // u and grad u at the point (_kernels_py.py:44-51)
    real u[NCOMP];
    realv gradU[NCOMP];
#pragma unroll
    for (int c = 0; c < NCOMP; ++c) {
      u[c] = real(0);
      gradU[c] = realv(real(0));
    }
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
      for (int c = 0; c < NCOMP; ++c) {
        u[c] = add(u[c], mul(cf[b * NCOMP + c], tab.B[q * NB + b]));
#pragma unroll
        for (int k = 0; k < D; ++k) gradU[c][k] = add(gradU[c][k], mul(cf[b * NCOMP + c], tr[b][k]));
      }

    // auxiliary fields (_kernels_py.py:93-110)
    real a[NAS];
    realv gradA[NAS];
#pragma unroll
    for (int j = 0; j < NAS; ++j) {
      a[j] = real(0);
      gradA[j] = realv(real(0));
    }
    if constexpr (AUXM == 1) {
#pragma unroll
      for (int j = 0; j < NAUX; ++j) a[j] = s_aux[cell * NAUX + j];
    } else if constexpr (AUXM == 2) {
      // the cell's nodal row once, vectorised (conflict-free for 32/96-byte rows)
      real av[NB * NAS];
      load_row_rot<real, NB * NAS, VEC>(s_aux + cell * AUXW, av, lane);
#pragma unroll
      for (int b = 0; b < NB; ++b)
#pragma unroll
        for (int j = 0; j < NAUX; ++j) a[j] = add(a[j], mul(av[b * NAUX + j], tab.B[q * NB + b]));
      if constexpr (GRAD_A) {
#pragma unroll
        for (int b = 0; b < NB; ++b)
#pragma unroll
          for (int j = 0; j < NAUX; ++j)
#pragma unroll
            for (int k = 0; k < D; ++k) gradA[j][k] = add(gradA[j][k], mul(av[b * NAUX + j], tr[b][k]));
      }
    }

    // pointwise physics, scaled by detJ then w_q (_kernels_py.py:53-65)
    const real w = tab.W[q];
#pragma unroll
    for (int c = 0; c < NCOMP; ++c) {
      const realv f1 = TXB_F1(u, gradU, a, gradA, c);
#pragma unroll
      for (int k = 0; k < D; ++k) s_f1[((q * NCOMP + c) * D + k) * P + lc] = mul(mul(f1[k], det), w);
#if TXB_HAS_F0
      const real f0 = TXB_F0(u, gradU, a, gradA, c);
      s_f0[(q * NCOMP + c) * P + lc] = mul(mul(f0, det), w);
#endif
    }
  }

  __syncwarp();  // ==== transpose threads (warp scope) ====

  // ------------- basis phase: lane <-> element entry (cell, b, c) -------------
  real* o_base = out + (int64_t)c0 * NBC;
  auto entry = [&](int o) {
    const int ec = o / NBC;
    const int r = o - ec * NBC;
    const int b = r / NCOMP;
    const int c = r - b * NCOMP;
    real e = real(0);  // _kernels_py.py:67-75: q-major, f0 term then the k terms
    if constexpr (STAGE_T) {
      // T[0] from the exchange area, T[b>=1] = invJ row b-1 (stage, or global on the direct path)
      real t[D];
      const real* tp = b == 0 ? s_tr + ec : s_inv + (c0 + ec) * DD + (b - 1) * D;
      const int step = b == 0 ? P : 1;
#pragma unroll
      for (int k = 0; k < D; ++k) t[k] = tp[k * step];
#pragma unroll
      for (int qq = 0; qq < NQ; ++qq) {
        if constexpr (HAS_F0) e = add(e, mul(tab.B[qq * NB + b], s_f0[(qq * NCOMP + c) * P + ec]));
#pragma unroll
        for (int k = 0; k < D; ++k) e = add(e, mul(t[k], s_f1[((qq * NCOMP + c) * D + k) * P + ec]));
      }
    } else {
#pragma unroll
      for (int qq = 0; qq < NQ; ++qq) {
        if constexpr (HAS_F0) e = add(e, mul(tab.B[qq * NB + b], s_f0[(qq * NCOMP + c) * P + ec]));
#pragma unroll
        for (int k = 0; k < D; ++k)
          e = add(e, mul(s_tr[((qq * NB + b) * D + k) * P + ec], s_f1[((qq * NCOMP + c) * D + k) * P + ec]));
      }
    }
    o_base[o] = e;
  };
  constexpr int FULL = CW * NBC;
  if (nc == CW && FULL % 32 == 0) {
#pragma unroll
    for (int i = 0; i < FULL / 32; ++i) entry(i * 32 + lane);  // consecutive lanes, consecutive entries
  } else {
    for (int o = lane; o < nc * NBC; o += 32) entry(o);
  }
  __syncwarp();  // scratch is reused by the next slice
}

template <bool STD, bool MESH>
__device__ __forceinline__ void integrate_body(const IntegrateArgs<real>& a, const MeshLaunchArgs<real>* m) {
  constexpr int SRC = MESH ? SRC_MESH : SRC_CELLS;
  constexpr int SCRATCH_BYTES = Area<STD && !MESH>::BYTES;
  extern __shared__ __align__(128) unsigned char smem[];
  const int nbc = a.n_bc;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int W = a.warps;
  // stage: inv_j | det_j | coeffs | aux  (cell arrays)   or   cells (int64) | aux  (mesh)
  const int o_det = MESH ? 0 : inv_bytes(nbc);
  const int o_coef = MESH ? 0 : o_det + det_bytes(nbc);
  const int o_aux = MESH ? round_up(nbc * NB * 8, 16) : o_coef + coef_bytes(nbc);
  const int stage_bytes = o_aux + aux_bytes(nbc);
  unsigned char* scratch_base = smem + a.stages * stage_bytes;
  const PipelineSmem p = carve_pipeline(scratch_base + W * SCRATCH_BYTES);
  pipeline_init(a, p);
  if (warp == W && lane == 0 && a.bulk) {
    pipeline_first_batches(a, a.prefetch, [&](int64_t c0, int ncell) {
      const uint32_t ab = ncell * AUXW * S;
      if constexpr (MESH) {
        const uint32_t kb = ncell * NB * 8;
        if ((kb | ab) & 15u) return;
        bulk_prefetch_l2(m->cells + c0 * NB, kb);
      } else {
        const uint32_t ib = ncell * DD * S, db = ncell * S, cb = ncell * NBC * S;
        if ((ib | db | cb | ab) & 15u) return;
        bulk_prefetch_l2(a.inv_j + c0 * DD, ib);
        bulk_prefetch_l2(a.det_j + c0, db);
        bulk_prefetch_l2(a.coeffs + c0 * NBC, cb);
      }
      if (AUXW) bulk_prefetch_l2(a.aux + c0 * AUXW, ab);
    });
  }
  pipeline_wait_prior_grid();

  if (warp == W) {
    // ============================ producer warp ============================
    if (lane != 0) return;
    const uint64_t policy = l2_evict_first_policy();
    pipeline_produce(a, p, smem, stage_bytes, [&](unsigned char* st, int64_t c0, int ncell, uint64_t* bar) {
      const uint32_t ab = ncell * AUXW * S;
      if constexpr (MESH) {
        const uint32_t kb = ncell * NB * 8;
        if (!a.bulk || ((kb | ab) & 15u)) return false;
        mbar_arrive_expect_tx(bar, kb + ab);
        bulk_g2s(st, m->cells + c0 * NB, kb, bar, policy);
      } else {
        const uint32_t ib = ncell * DD * S, db = ncell * S, cb = ncell * NBC * S;
        if (!a.bulk || ((ib | db | cb | ab) & 15u)) return false;
        mbar_arrive_expect_tx(bar, ib + db + cb + ab);
        bulk_g2s(st, a.inv_j + c0 * DD, ib, bar, policy);
        bulk_g2s(st + o_det, a.det_j + c0, db, bar, policy);
        bulk_g2s(st + o_coef, a.coeffs + c0 * NBC, cb, bar, policy);
      }
      if (AUXW) bulk_g2s(st + o_aux, a.aux + c0 * AUXW, ab, bar, policy);
      return true;
    });
    return;
  }

  // ============================ consumer warps ============================
  real* scratch = reinterpret_cast<real*>(scratch_base + warp * SCRATCH_BYTES);
  pipeline_consume(a, p, smem, stage_bytes, [&](const unsigned char* st, int64_t c0, int ncell) {
    real* out = a.out + c0 * NBC;
    MeshIn mi{nullptr, nullptr, nullptr, nullptr, c0, nullptr, nullptr, nullptr, 0, 0, 0, nullptr, nullptr};
    if constexpr (MESH) {
      mi.ids = st ? reinterpret_cast<const int64_t*>(st) : m->cells + c0 * NB;
      mi.X = m->vertices;
      mi.glob = m->coeffs_global;
      mi.bad = m->bad;
    }
    if (st) {
      const real* s_inv = reinterpret_cast<const real*>(st);
      const real* s_det = reinterpret_cast<const real*>(st + o_det);
      const real* s_coef = reinterpret_cast<const real*>(st + o_coef);
      const real* s_aux = reinterpret_cast<const real*>(st + o_aux);
      for (int c = warp * CW; c < ncell; c += W * CW)
        warp_slice<STD, true, SRC>(a.tab, s_inv, s_det, s_coef, s_aux, scratch, c, ncell, out, lane, mi);
    } else {
      // unaligned caller buffers or an odd-sized partial batch: straight from global memory
      const real* g_aux = AUXW ? a.aux + c0 * AUXW : nullptr;
      for (int c = warp * CW; c < ncell; c += W * CW)
        warp_slice<STD, false, SRC>(a.tab, a.inv_j + c0 * DD, a.det_j + c0, a.coeffs + c0 * NBC, g_aux, scratch, c,
                                    ncell, out, lane, mi);
    }
  });
}

// ---------------------------------------------------------------------------
// Tiled mesh entry points (csrc/txb_integrate_tiled.cu's design): a batch is a
// tile; the producer lane bulk-copies the tile's local indices, aux slice and
// distinct-vertex record; the gatherer warp copies each distinct vertex's
// coordinates and coefficients once into the stage's structure-of-arrays table
// (cp.async, completion on `ready`); the consumers run the slices above with
// their rows read from that table.
// Stage: [local indices][aux][record][x | y (| z) float64][coefficient components]
// ---------------------------------------------------------------------------
__device__ __forceinline__ int t_local_bytes(int n, int lb) { return round_up(n * 4 * lb, 16); }
__device__ __forceinline__ int t_xyz_pitch(int vrec) { return round_up(vrec * 8, 16) / 8; }
__device__ __forceinline__ int t_u_pitch(int vrec) { return round_up(vrec * S, 16) / S; }

template <bool STD, bool GEOM>
__device__ __forceinline__ void integrate_tiled_body(const TiledLaunchArgs<real>& t) {
  const IntegrateArgs<real>& a = t.a;
  constexpr int SCRATCH_BYTES = Area<false>::BYTES;
  extern __shared__ __align__(128) unsigned char smem[];
  const int nbc = a.n_bc, vrec = t.vrec, lb = t.lb;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int W = a.warps;
  const int o_aux = t_local_bytes(nbc, lb);
  const int o_inv = o_aux + aux_bytes(nbc);
  const int o_det = o_inv + (GEOM ? inv_bytes(nbc) : 0);
  const int o_rec = o_det + (GEOM ? det_bytes(nbc) : 0);
  const int o_xyz = o_rec + vrec * 4;
  const int vpitch = t_xyz_pitch(vrec), upitch = t_u_pitch(vrec);
  const int o_u = o_xyz + (GEOM ? 0 : D * vpitch * 8);
  const int stage_bytes = o_u + NCOMP * upitch * S;
  unsigned char* scratch_base = smem + a.stages * stage_bytes;
  const PipelineSmem p = carve_pipeline(scratch_base + W * SCRATCH_BYTES);
  uint64_t* ready = reinterpret_cast<uint64_t*>(scratch_base + W * SCRATCH_BYTES + PIPELINE_SMEM_BYTES);
  if (threadIdx.x == 0)
    for (int s = 0; s < a.stages; ++s) mbar_init(&ready[s], 32);
  pipeline_init(a, p);
  if (warp == W && lane == 0) {
    pipeline_first_batches(a, a.prefetch, [&](int64_t c0, int ncell) {
      bulk_prefetch_l2(t.local + c0 * 4 * lb, (uint32_t)t_local_bytes(nbc, lb));
      bulk_prefetch_l2(t.records + (c0 / nbc) * vrec, (uint32_t)(vrec * 4));
    });
  }
  pipeline_wait_prior_grid();

  if (warp == W) {
    // ============================ producer lane ============================
    if (lane != 0) return;
    const uint64_t policy = l2_evict_first_policy();
    pipeline_produce(a, p, smem, stage_bytes, [&](unsigned char* st, int64_t c0, int ncell, uint64_t* bar) {
      const uint32_t lbytes = t_local_bytes(nbc, lb), rb = vrec * 4;
      const uint32_t ab = ncell * AUXW * S;
      const bool auxb = AUXW != 0 && t.aux_bulk && (ab & 15u) == 0;
      const uint32_t ib = GEOM ? ncell * DD * S : 0, db = GEOM ? ncell * S : 0;
      const bool geob = GEOM && t.geom_bulk && ((ib | db) & 15u) == 0;
      mbar_arrive_expect_tx(bar, lbytes + rb + (auxb ? ab : 0) + (geob ? ib + db : 0));
      bulk_g2s(st, t.local + c0 * 4 * lb, lbytes, bar, policy);
      if (auxb) bulk_g2s(st + o_aux, a.aux + c0 * AUXW, ab, bar, policy);
      if (geob) {
        bulk_g2s(st + o_inv, a.inv_j + c0 * DD, ib, bar, policy);
        bulk_g2s(st + o_det, a.det_j + c0, db, bar, policy);
      }
      bulk_g2s(st + o_rec, t.records + (c0 / nbc) * vrec, rb, bar, policy);
      return true;
    });
    return;
  }

  if (warp == W + 1) {
    // ============================ gatherer warp ============================
    int stage = 0;
    uint32_t phase = 0;
    for (;;) {
      mbar_wait(&p.full[stage], phase);
      const int n = p.info_n[stage];
      if (n != 0) {
        unsigned char* st = smem + stage * stage_bytes;
        const int32_t* rec = reinterpret_cast<const int32_t*>(st + o_rec);
        const int cnt = rec[0];
        double* sx = reinterpret_cast<double*>(st + o_xyz);
        real* su = reinterpret_cast<real*>(st + o_u);
        for (int j = lane; j < cnt; j += 32) {
          const int64_t v = rec[4 + j];
          if constexpr (!GEOM) {
#pragma unroll
            for (int i = 0; i < D; ++i) cp_async<8>(sx + i * vpitch + j, t.vertices + v * D + i);
          }
#pragma unroll
          for (int c = 0; c < NCOMP; ++c) cp_async<S>(su + c * upitch + j, t.coeffs_global + v * NCOMP + c);
        }
      }
      cp_async_arrive_noinc(&ready[stage]);
      if (n == 0) break;
      if (++stage == a.stages) {
        stage = 0;
        phase ^= 1;
      }
    }
    return;
  }

  // ============================ consumer warps ============================
  real* scratch = reinterpret_cast<real*>(scratch_base + warp * SCRATCH_BYTES);
  int stage = 0;
  uint32_t phase = 0;
  for (;;) {
    mbar_wait(&ready[stage], phase);
    mbar_wait(&p.full[stage], phase);
    const int64_t c0 = p.info_c0[stage];
    const int ncell = p.info_n[stage];
    if (ncell == 0) break;
    const unsigned char* st = smem + stage * stage_bytes;
    const uint32_t ab = ncell * AUXW * S;
    const real* aux_src = (AUXW != 0 && t.aux_bulk && (ab & 15u) == 0) ? reinterpret_cast<const real*>(st + o_aux)
                                                                        : a.aux + c0 * AUXW;
    MeshIn mi{nullptr, nullptr, nullptr, t.bad, c0, st, reinterpret_cast<const double*>(st + o_xyz),
              reinterpret_cast<const real*>(st + o_u), vpitch, upitch, lb, nullptr, nullptr};
    if constexpr (GEOM) {
      const uint32_t ib = ncell * DD * S, db = ncell * S;
      const bool geob = t.geom_bulk && ((ib | db) & 15u) == 0;
      mi.g_inv = geob ? reinterpret_cast<const real*>(st + o_inv) : a.inv_j + c0 * DD;
      mi.g_det = geob ? reinterpret_cast<const real*>(st + o_det) : a.det_j + c0;
    }
    real* out = a.out + c0 * NBC;
    for (int c = warp * CW; c < ncell; c += W * CW)
      warp_slice<STD, true, GEOM ? SRC_TILED_GEOM : SRC_TILED>(a.tab, nullptr, nullptr, nullptr, aux_src, scratch, c,
                                                                ncell, out, lane, mi);
    mbar_arrive(&p.empty[stage]);
    if (++stage == a.stages) {
      stage = 0;
      phase ^= 1;
    }
  }
}

}  // namespace jit
}  // namespace txb

// CTA bound of the cell-array and per-cell mesh entry points (the host's
// jit_cta_threads): multi-component float64 forms get 256 threads and 2 CTAs
// per SM (128 registers, as the ahead-of-time kernels' CtaBound), the rest the
// wide bound -- measured on the shipped 3D elasticity form through NVRTC:
// f64 44.7 -> 43.9 us, while f32 went 24.8 -> 27.8 us with the narrow bound.
#ifdef TXB_JIT_WIDE  // TXB_JIT_WIDE=1 in the environment: the wide bound for every form (tuning)
#define TXB_JIT_NARROW 0
#else
#define TXB_JIT_NARROW (TXB_NCOMP > 1 && sizeof(real) == 8)
#endif
#define TXB_JIT_BOUNDS __launch_bounds__(TXB_JIT_NARROW ? 256 : txb::MAX_CTA_THREADS, TXB_JIT_NARROW ? 2 : 1)

#ifndef TXB_JIT_MESH
extern "C" __global__ void TXB_JIT_BOUNDS
txb_jit_integrate(const __grid_constant__ txb::IntegrateArgs<real> a) {
  txb::jit::integrate_body<false, false>(a, nullptr);
}

extern "C" __global__ void TXB_JIT_BOUNDS
txb_jit_integrate_std(const __grid_constant__ txb::IntegrateArgs<real> a) {
  txb::jit::integrate_body<true, false>(a, nullptr);
}

#else
// mesh-fused: connectivity in, geometry + gather in-kernel (the reference's
// compute_geometry -> gather_coefficients -> cast -> integrate, executor.py:194-212).
// A second program (TXB_JIT_MESH), compiled on first use by txb_jit_integrate_mesh.
extern "C" __global__ void TXB_JIT_BOUNDS
txb_jit_integrate_mesh(const __grid_constant__ txb::MeshLaunchArgs<real> m) {
  txb::jit::integrate_body<false, true>(m.a, &m);
}

extern "C" __global__ void TXB_JIT_BOUNDS
txb_jit_integrate_mesh_std(const __grid_constant__ txb::MeshLaunchArgs<real> m) {
  txb::jit::integrate_body<true, true>(m.a, &m);
}

// tiled mesh entry points (geometry + gather from per-tile vertex tables)
extern "C" __global__ void __launch_bounds__(txb::MAX_CTA_THREADS, 1)
txb_jit_integrate_tiled(const __grid_constant__ txb::TiledLaunchArgs<real> t) {
  txb::jit::integrate_tiled_body<false, false>(t);
}

extern "C" __global__ void __launch_bounds__(txb::MAX_CTA_THREADS, 1)
txb_jit_integrate_tiled_std(const __grid_constant__ txb::TiledLaunchArgs<real> t) {
  txb::jit::integrate_tiled_body<true, false>(t);
}

// the caller's geometry streamed with the batch, coefficients from the tile tables
extern "C" __global__ void __launch_bounds__(txb::MAX_CTA_THREADS, 1)
txb_jit_integrate_tiled_geom(const __grid_constant__ txb::TiledLaunchArgs<real> t) {
  txb::jit::integrate_tiled_body<false, true>(t);
}

extern "C" __global__ void __launch_bounds__(txb::MAX_CTA_THREADS, 1)
txb_jit_integrate_tiled_geom_std(const __grid_constant__ txb::TiledLaunchArgs<real> t) {
  txb::jit::integrate_tiled_body<true, true>(t);
}
#endif
