// txb_integrate.cu — thread-transposed P1 element integration for sm_100a.
//
// B200-native restatement of the paper's kernel (Knepley, Rupp, Terrel,
// arXiv:1607.04245, §3 and the appendix pseudocode) behind the reference's
// compiled-lane interface (txfem/_kernels_cy.pyx:37-123).
//
// Decomposition (paper §3; txfem/schedule.py:82-113):
//   block  = N_bs = N_b * N_q cells
//   batch  = N_bc = N_bl * N_bs cells        -> one shared-memory ring stage
//   chunk  = N_cb consecutive batches         -> one CTA work item
// A CTA is persistent and warp-specialised:
//   producer warp   one elected lane streams batches into a ring of `stages`
//                   shared-memory stages with cp.async.bulk (SASS UBLKCP):
//                   the batch's contiguous inv_j / det_j / coeffs / aux byte
//                   ranges, completion counted on a `full` mbarrier
//                   (expect_tx); it refills a stage once every consumer lane
//                   has arrived on the stage's `empty` mbarrier.
//   consumer warps  each owns warp slices of CW = 32 / N_q cells of a batch:
//     quadrature phase  lane <-> (cell, q): pulled-back gradients, grad u,
//                       aux value, inlined f1, scaled by detJ * w_q
//                       (txfem/device.py:267-330, _kernels_cy.pyx:70-111)
//     transpose         through a warp-private scratch area + __syncwarp (the
//                       paper's "TRANSPOSE THREADS" barrier, no CTA barrier)
//     basis phase       lane <-> element-vector entry (cell, b, c): the
//                       reduction-free sum over (q, k) of T[q][b][k] * f1s[q][c][k];
//                       consecutive lanes own consecutive output entries, so
//                       the stores coalesce (device.py:335-361, pyx:113-123)
// CTAs walk chunks blockIdx.x, blockIdx.x + gridDim.x, ... so the whole grid
// streams through the cell arrays together.
//
// Numerics: products and sums round one at a time in the reference's pinned
// order (txfem/reference.py:10-19) -> bit-identical to the reference lanes.
// When the tabulated reference gradients are exactly the P1 ones
// (-1 / unit vectors, element.py:55-77) the kernel uses the exact IEEE
// identities 1*x = x, (-1)*x = -x, 0*x = +-0, x + (+-0) = x (x != 0) to
// evaluate the pull-back T[b][k] = sum_j D[b][j] invJ[j][k] with the same
// rounded results and far fewer instructions (bit-identical for finite inputs).
#include "txb_kernels.cuh"

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <thread>
#include <tuple>
#include <vector>

namespace txb {


// One warp slice: CW cells starting at batch-local cell `c0` of a batch with
// `ncell` cells whose per-cell arrays start at the given pointers (shared
// stage or global memory); element vectors go to `out` (batch base, global).
// FULLS: the slice is known to be full (CW cells) -- no bounds checks, no
// divergent regions (the common case: full batches, one slice per warp).
template <typename T, int D, int NQ, int NCOMP, int FORM, int AUX, bool STD, bool VEC, bool FULLS = false>
__device__ __forceinline__ void warp_slice(const Tabulation<T>& tab, const T* __restrict__ s_inv,
                                           const T* __restrict__ s_det, const T* __restrict__ s_coef,
                                           const T* __restrict__ s_aux, unsigned char* __restrict__ scratch,
                                           int c0, int ncell, T* __restrict__ out, int lane) {
  constexpr int NB = D + 1, DD = D * D, NBC = NB * NCOMP;
  using S = Scratch<T, D, NQ, NCOMP, STD>;
  constexpr int AUXW = AUX == 1 ? 1 : (AUX == 2 ? NB : 0);
  T* s_tr = reinterpret_cast<T*>(scratch);
  T* s_f1 = reinterpret_cast<T*>(scratch + S::TR_BYTES);
  const int nc = FULLS ? S::CW : min(S::CW, ncell - c0);

  // ---------------- quadrature phase: lane <-> (cell, q) ----------------
  {
    const int lc = NQ == 1 ? lane : lane / NQ;
    const int q = NQ == 1 ? 0 : lane - lc * NQ;
    if (lc < nc) {  // with FULLS, nc == CW: folds away when N_q divides 32
      const int cell = c0 + lc;
      T J[DD];
      load_row<T, DD, VEC>(s_inv + cell * DD, J);
      T cf[NBC];
      load_row_rot<T, NBC, VEC>(s_coef + cell * NBC, cf, lane);
      const T det = s_det[cell];

      T tr[NB][D];
      if constexpr (STD) {
        // T[0][k] = ((0 + (-1)J0k) + (-1)J1k) + (-1)J2k  ==  (-J0k - J1k) - J2k  (up to the sign of 0)
        // T[b][k] = ((0 + 0 J0k) + 1 J1k) + 0 J2k ...     ==  J[b-1][k]          (up to the sign of 0)
#pragma unroll
        for (int k = 0; k < D; ++k) {
          T acc = -J[k];
#pragma unroll
          for (int j = 1; j < D; ++j) acc = add(acc, -J[j * D + k]);
          tr[0][k] = acc;
        }
#pragma unroll
        for (int bb = 1; bb < NB; ++bb)
#pragma unroll
          for (int k = 0; k < D; ++k) tr[bb][k] = J[(bb - 1) * D + k];
        if (q == 0) {
          if constexpr (S::SJ) {
#pragma unroll
            for (int i = 0; i < DD; ++i) s_tr[S::tr(lc, i)] = J[i];
#pragma unroll
            for (int k = 0; k < D; ++k) s_tr[S::tr(lc, DD + k)] = tr[0][k];
          } else {
#pragma unroll
            for (int k = 0; k < D; ++k) s_tr[S::tr(lc, k)] = tr[0][k];
          }
        }
      } else {
        const T* Dq = tab.D + q * NB * D;
#pragma unroll
        for (int bb = 0; bb < NB; ++bb)
#pragma unroll
          for (int k = 0; k < D; ++k) {
            T acc = mul(Dq[bb * D], J[k]);
#pragma unroll
            for (int j = 1; j < D; ++j) acc = add(acc, mul(Dq[bb * D + j], J[j * D + k]));
            tr[bb][k] = acc;
            s_tr[S::tr(lc, (q * NB + bb) * D + k)] = acc;
          }
      }

      T g[NCOMP][D];
#pragma unroll
      for (int c = 0; c < NCOMP; ++c)
#pragma unroll
        for (int k = 0; k < D; ++k) {
          T acc = mul(cf[c], tr[0][k]);
#pragma unroll
          for (int bb = 1; bb < NB; ++bb) acc = add(acc, mul(cf[bb * NCOMP + c], tr[bb][k]));
          g[c][k] = acc;
        }

      T a0 = T(0);
      if constexpr (AUX == 1) {
        a0 = s_aux[cell];
      } else if constexpr (AUX == 2) {
        T av[NB];
        load_row_rot<T, NB, VEC>(s_aux + cell * AUXW, av, lane);
        const T* Bq = tab.B + q * NB;
        a0 = mul(av[0], Bq[0]);
#pragma unroll
        for (int bb = 1; bb < NB; ++bb) a0 = add(a0, mul(av[bb], Bq[bb]));
      }
      (void)a0;

      const T wq = tab.W[q];

#pragma unroll
      for (int c = 0; c < NCOMP; ++c)
#pragma unroll
        for (int k = 0; k < D; ++k) {
          T fv;
          if constexpr (FORM == 0) {
            fv = g[c][k];
          } else if constexpr (FORM == 1) {
            fv = mul(a0, g[c][k]);
          } else {
            fv = mul(T(0.5), add(g[c][k], g[k][c]));
          }
          s_f1[S::f1(lc, (q * NCOMP + c) * D + k)] = mul(mul(fv, det), wq);
        }
    }
  }

  __syncwarp();  // ==== transpose threads (warp scope) ====

  // ------------- basis phase: lane <-> element entry (cell, b, c) -------------
  T* o_base = out + (int64_t)c0 * NBC;
  auto entry = [&](int o) {
    const int lc = o / NBC;
    const int r = o - lc * NBC;
    const int b = r / NCOMP;
    const int c = r - b * NCOMP;
    // f1s rows of this entry's component
    T f1[NQ * D];
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
      for (int k = 0; k < D; ++k) f1[q * D + k] = s_f1[S::f1(lc, (q * NCOMP + c) * D + k)];
    T e = T(0);  // the output chain starts at +0 exactly as the reference's
    if constexpr (STD) {
      T t[D];
      if constexpr (S::SJ) {  // all rows from the exchange area
        const int r0 = b == 0 ? DD : (b - 1) * D;
#pragma unroll
        for (int k = 0; k < D; ++k) t[k] = s_tr[S::tr(lc, r0 + k)];
      } else {  // T[0] from the exchange area, T[b>=1] = invJ row b-1 of the stage
        const T* tp = b == 0 ? s_tr + S::tr(lc, 0) : s_inv + (c0 + lc) * DD + (b - 1) * D;
        const int step = b == 0 ? S::tr(0, 1) - S::tr(0, 0) : 1;
#pragma unroll
        for (int k = 0; k < D; ++k) t[k] = tp[k * step];
      }
#pragma unroll
      for (int q = 0; q < NQ; ++q)
#pragma unroll
        for (int k = 0; k < D; ++k) e = add(e, mul(t[k], f1[q * D + k]));
    } else {
#pragma unroll
      for (int q = 0; q < NQ; ++q)
#pragma unroll
        for (int k = 0; k < D; ++k) e = add(e, mul(s_tr[S::tr(lc, (q * NB + b) * D + k)], f1[q * D + k]));
    }
    o_base[o] = e;
  };
  constexpr int FULL = S::CW * NBC;
  if (FULL % 32 == 0 && (FULLS || nc == S::CW)) {
#pragma unroll
    for (int s = 0; s < FULL / 32; ++s) entry(s * 32 + lane);
  } else {
    for (int o = lane; o < nc * NBC; o += 32) entry(o);
  }
  __syncwarp();  // scratch is reused by the next slice
}

// Register budget per instantiation.  The elasticity kernels need ~130-190
// registers without spills (3D, standard tables); under the 544-thread bound
// ptxas held them to 96 with spills.  A 256-thread CTA bound (<= 7 consumer
// warps, 128 registers, 2 CTAs/SM guaranteed) is faster for every elasticity
// configuration but 2D f32, whose small rows favour wide CTAs
// (profiles/r2bd_bounds.md: 3D f32 24.2 -> 22.7 us, 3D f64 45.5 -> 43.3,
// 2D f64 23.0 -> 22.4; 2D f32 11.9 -> 13.5 with it).  TXB_ELAST_THREADS /
// TXB_ELAST_MINB override it in tuning builds.
template <typename T, int D, int NCOMP>
struct CtaBound {
#ifdef TXB_ELAST_THREADS
  static constexpr bool NARROW = NCOMP > 1;
  static constexpr int THREADS = NARROW ? TXB_ELAST_THREADS : MAX_CTA_THREADS;
  static constexpr int MIN_BLOCKS = NARROW ? TXB_ELAST_MINB : 1;
#else
  static constexpr bool NARROW = NCOMP > 1 && !(D == 2 && sizeof(T) == 4);
  static constexpr int THREADS = NARROW ? 256 : MAX_CTA_THREADS;
  static constexpr int MIN_BLOCKS = NARROW ? 2 : 1;
#endif
};

template <typename T, int D, int NQ, int NCOMP, int FORM, int AUX, bool STD>
__global__ void __launch_bounds__(CtaBound<T, D, NCOMP>::THREADS, CtaBound<T, D, NCOMP>::MIN_BLOCKS)
integrate_kernel(const __grid_constant__ IntegrateArgs<T> a) {
  constexpr int DD = D * D, NBC = (D + 1) * NCOMP;
  using L = StageLayout<T, D, NCOMP, AUX>;
  using S = Scratch<T, D, NQ, NCOMP, STD>;

  extern __shared__ __align__(128) unsigned char smem[];
  const int nbc = a.n_bc;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int W = a.warps;
  if (threadIdx.x == 0) trace_stamp(a.trace, 0);
  const int stage_bytes = L::stage_bytes(nbc);
  unsigned char* scratch_base = smem + a.stages * stage_bytes;
  const PipelineSmem p = carve_pipeline(scratch_base + W * S::BYTES);
  pipeline_init(a, p);
  if (warp == W && lane == 0 && a.bulk) {
    // warm L2 with this CTA's first batches while the previous grid drains
    pipeline_first_batches(a, a.prefetch, [&](int64_t c0, int ncell) {
      const uint32_t ib = ncell * DD * sizeof(T), db = ncell * sizeof(T), cb = ncell * NBC * sizeof(T),
                     ab = ncell * L::AUXW * sizeof(T);
      if ((ib | db | cb | ab) & 15u) return;
      bulk_prefetch_l2(a.inv_j + c0 * DD, ib);
      bulk_prefetch_l2(a.det_j + c0, db);
      bulk_prefetch_l2(a.coeffs + c0 * NBC, cb);
      if constexpr (AUX != 0) bulk_prefetch_l2(a.aux + c0 * L::AUXW, ab);
    });
  }
  pipeline_wait_prior_grid();
  if (threadIdx.x == 0) trace_stamp(a.trace, 1);

  if (warp == W) {
    // ============================ producer warp ============================
    if (lane != 0) return;
    const uint64_t policy = l2_evict_first_policy();
    // A batch may arrive by bulk copy when its four slices are 16-byte aligned
    // and sized (base pointers and N_bc*s*k % 16 are checked on the host; only
    // a partial batch can fail the size test).
    pipeline_produce(a, p, smem, stage_bytes, [&](unsigned char* st, int64_t c0, int ncell, uint64_t* bar) {
      const uint32_t ib = ncell * DD * sizeof(T), db = ncell * sizeof(T), cb = ncell * NBC * sizeof(T),
                     ab = ncell * L::AUXW * sizeof(T);
      if (!a.bulk || ((ib | db | cb | ab) & 15u)) return false;
      mbar_arrive_expect_tx(bar, ib + db + cb + ab);
      bulk_g2s(st, a.inv_j + c0 * DD, ib, bar, policy);
      bulk_g2s(st + L::inv_bytes(nbc), a.det_j + c0, db, bar, policy);
      bulk_g2s(st + L::inv_bytes(nbc) + L::det_bytes(nbc), a.coeffs + c0 * NBC, cb, bar, policy);
      if constexpr (AUX != 0)
        bulk_g2s(st + L::inv_bytes(nbc) + L::det_bytes(nbc) + L::coef_bytes(nbc), a.aux + c0 * L::AUXW, ab, bar,
                 policy);
      return true;
    });
    return;
  }

  // ============================ consumer warps ============================
  unsigned char* scratch = scratch_base + warp * S::BYTES;
#ifdef TXB_TRACE_FIRST_BATCH  // costs registers in the consumer loop: tuning builds only
  bool first = true;
#endif
  pipeline_consume(a, p, smem, stage_bytes, [&](const unsigned char* st, int64_t c0, int ncell) {
#ifdef TXB_TRACE_FIRST_BATCH
    if (first && threadIdx.x == 0) trace_stamp(a.trace, 2);
    first = false;
#endif
    T* out = a.out + c0 * NBC;
    if (st) {
      const T* s_inv = reinterpret_cast<const T*>(st);
      const T* s_det = reinterpret_cast<const T*>(st + L::inv_bytes(nbc));
      const T* s_coef = reinterpret_cast<const T*>(st + L::inv_bytes(nbc) + L::det_bytes(nbc));
      const T* s_aux = reinterpret_cast<const T*>(st + L::inv_bytes(nbc) + L::det_bytes(nbc) + L::coef_bytes(nbc));
      // full batch, one slice per warp: the check-free slice (scalar forms; for
      // elasticity the second instantiation costs registers and a stack frame)
      if (NCOMP == 1 && ncell == nbc && nbc == W * S::CW)
        warp_slice<T, D, NQ, NCOMP, FORM, AUX, STD, true, NCOMP == 1>(a.tab, s_inv, s_det, s_coef, s_aux,
                                                                     scratch, warp * S::CW, ncell, out, lane);
      else
        for (int c = warp * S::CW; c < ncell; c += W * S::CW)
          warp_slice<T, D, NQ, NCOMP, FORM, AUX, STD, true>(a.tab, s_inv, s_det, s_coef, s_aux, scratch, c, ncell,
                                                           out, lane);
    } else {
      // unaligned caller buffers or an odd-sized partial batch: straight from global memory
      const T* g_aux = AUX != 0 ? a.aux + c0 * L::AUXW : nullptr;
      for (int c = warp * S::CW; c < ncell; c += W * S::CW)
        warp_slice<T, D, NQ, NCOMP, FORM, AUX, STD, false>(a.tab, a.inv_j + c0 * DD, a.det_j + c0,
                                                          a.coeffs + c0 * NBC, g_aux, scratch, c, ncell, out,
                                                          lane);
    }
  });
  if (threadIdx.x == 0) trace_stamp(a.trace, 3);
}

// ---------------------------------------------------------------------------
// Host side: dispatch and launch.
// ---------------------------------------------------------------------------

template <typename T, int D, int NQ, int NCOMP, int FORM, int AUX, bool STD>
struct Kernel {
  using L = StageLayout<T, D, NCOMP, AUX>;
  static void* fn() { return (void*)integrate_kernel<T, D, NQ, NCOMP, FORM, AUX, STD>; }
  static int stage_bytes(int n_bc) { return L::stage_bytes(n_bc); }
  static int scratch(int) { return Scratch<T, D, NQ, NCOMP, STD>::BYTES; }
  static constexpr int CW = 32 / NQ;
};

template <typename T, int D, int NQ, bool STD>
static bool pick_form(const Config& c, KernelInfo& k) {
  if (c.form == 0) {
    using K = Kernel<T, D, NQ, 1, 0, 0, STD>;
    k = {K::fn(), K::stage_bytes, K::scratch, K::CW};
  } else if (c.form == 1 && c.aux == 1) {
    using K = Kernel<T, D, NQ, 1, 1, 1, STD>;
    k = {K::fn(), K::stage_bytes, K::scratch, K::CW};
  } else if (c.form == 1 && c.aux == 2) {
    using K = Kernel<T, D, NQ, 1, 1, 2, STD>;
    k = {K::fn(), K::stage_bytes, K::scratch, K::CW};
  } else if (c.form == 2) {
    using K = Kernel<T, D, NQ, D, 2, 0, STD>;
    k = {K::fn(), K::stage_bytes, K::scratch, K::CW};
    k.max_warps = CtaBound<T, D, D>::THREADS / 32 - 1;
  } else {
    return false;
  }
  return true;
}

template <typename T, int D>
static bool pick_nq(const Config& c, bool std_tab, KernelInfo& k) {
  if (std_tab) {  // standard P1 tables: midpoint and two-point rules
    if (c.n_q == 1) return pick_form<T, D, 1, true>(c, k);
    if (c.n_q == 2) return pick_form<T, D, 2, true>(c, k);
  }
  switch (c.n_q) {
    case 1: return pick_form<T, D, 1, false>(c, k);
    case 2: return pick_form<T, D, 2, false>(c, k);
    case 3: return pick_form<T, D, 3, false>(c, k);
    case 4: return pick_form<T, D, 4, false>(c, k);
    case 5: return pick_form<T, D, 5, false>(c, k);
    case 6: return pick_form<T, D, 6, false>(c, k);
    case 7: return pick_form<T, D, 7, false>(c, k);
    case 8: return pick_form<T, D, 8, false>(c, k);
  }
  return false;
}

// 2D f32 elasticity, launch-sized problems: 4 consumer warps looping over the
// 9 slices of a 288-cell batch beat 9 warps (2^20 cells 11.9 -> 11.7 us; at
// 2^22 cells and above the wide CTA stays faster; profiles/r2bd_bounds.md).
static void size_tuning(const Config& c, int64_t n_cells, KernelInfo& k) {
  if (c.form == 2 && c.dim == 2 && c.dtype == 4 && n_cells < ((int64_t)1 << 22)) k.max_warps = 4;
}

static bool pick_kernel(const Config& c, bool std_tab, KernelInfo& k) {
  if (env_int("TXB_DISABLE_STD", 0)) std_tab = false;
  if (c.dtype == 4) return c.dim == 2 ? pick_nq<float, 2>(c, std_tab, k) : pick_nq<float, 3>(c, std_tab, k);
  return c.dim == 2 ? pick_nq<double, 2>(c, std_tab, k) : pick_nq<double, 3>(c, std_tab, k);
}

template <typename T>
static int launch_t(bool zero_copy, const Config& c, const KernelInfo& k, const Geometry& g, int64_t n_cells,
                    const void* basis,
                    const void* basis_der, const void* weights, const void* inv_j, const void* det_j,
                    const void* coeffs, const void* aux, void* out, cudaStream_t stream) {
  IntegrateArgs<T> a;
  a.inv_j = (const T*)inv_j;
  a.det_j = (const T*)det_j;
  a.coeffs = (const T*)coeffs;
  a.aux = (const T*)aux;
  a.out = (T*)out;
  a.n_cells = n_cells;
  a.n_chunks = g.n_chunks;
  a.chunk_cells = g.chunk_cells;
  a.n_bc = g.n_bc;
  a.stages = g.stages;
  a.warps = g.warps;
  a.dynamic = g.dynamic;
  a.resident = g.resident;
  a.static_batches = g.static_batches;
  // Bulk copies need 16-byte aligned, 16-byte sized slices for EVERY batch:
  // aligned base pointers and N_bc * (per-cell scalars) * sizeof(T) % 16 == 0
  // for each of the four arrays.  Otherwise every batch is read from global.
  auto al16 = [](const void* p) { return ((uintptr_t)p & 15u) == 0; };
  const int nb = c.dim + 1, auxw = c.aux == 1 ? 1 : (c.aux == 2 ? nb : 0);
  auto sized16 = [&](int per_cell) { return ((int64_t)g.n_bc * per_cell * (int64_t)sizeof(T)) % 16 == 0; };
  // (zero_copy: the arrays are mapped pinned HOST memory; the bulk copies read
  // them over PCIe -- measured as fast as staged copies, while per-lane loads
  // from host memory were 1.3x slower -- and the L2 prefetch is skipped)
  a.bulk = al16(inv_j) && al16(det_j) && al16(coeffs) && (c.aux == 0 || al16(aux)) &&
           sized16(c.dim * c.dim) && sized16(1) && sized16(nb * c.n_comp) && (c.aux == 0 || sized16(auxw)) &&
           env_int("TXB_DISABLE_BULK", 0) == 0;
  a.prefetch = zero_copy ? 0 : prefetch_batches(g);
  a.trace = next_trace_slot(g.grid);
  fill_tab(a.tab, c.n_q, c.dim + 1, c.dim, basis, basis_der, weights);
  void* params[] = {&a};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(g.grid);
  cfg.blockDim = dim3(g.threads);
  cfg.dynamicSmemBytes = (size_t)g.smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = env_int("TXB_PDL", 1) ? 1 : 0;
  TXB_CUDA_TRY(cudaLaunchKernelExC(&cfg, k.fn, params));
  return TXB_OK;
}

int integrate_device(const Config& c, int n_b, int64_t n_cells, const void* basis, const void* basis_der,
                     const void* weights, const void* inv_j, const void* det_j, const void* coeffs,
                     const void* aux, void* out, int n_bl, int n_cb, cudaStream_t stream, bool zero_copy = false) {
  int rc = validate(c);
  if (rc) return rc;
  if (n_b != c.dim + 1) {
    set_error("P1 element needs n_b = dim + 1 = %d, got %d", c.dim + 1, n_b);
    return TXB_E_SHAPE;
  }
  if (n_cells < 0) {
    set_error("n_cells must be >= 0, got %lld", (long long)n_cells);
    return TXB_E_SHAPE;
  }
  if (!basis || !basis_der || !weights) {
    set_error("basis, basis_der and weights are required (host pointers)");
    return TXB_E_ARG;
  }
  KernelInfo k;
  if (!pick_kernel(c, standard_tables(c, basis_der), k)) {
    set_error("no kernel instantiation for this configuration");
    return TXB_E_UNSUPPORTED;
  }
  size_tuning(c, n_cells, k);
  Geometry g;
  rc = compute_geometry(c, k, n_cells, n_bl, n_cb, true, g);
  if (rc) return rc;
  if (n_cells == 0) return TXB_OK;
  if (!inv_j || !det_j || !coeffs || !out || (c.aux != 0 && !aux)) {
    set_error("NULL device pointer for a per-cell array");
    return TXB_E_ARG;
  }
  if (c.dtype == 4)
    return launch_t<float>(zero_copy, c, k, g, n_cells, basis, basis_der, weights, inv_j, det_j, coeffs, aux, out,
                           stream);
  return launch_t<double>(zero_copy, c, k, g, n_cells, basis, basis_der, weights, inv_j, det_j, coeffs, aux, out,
                          stream);
}

// ---------------------------------------------------------------------------
// Host-buffer path: pieces of cells pipelined over NS streams (slots); the
// H2D of piece p+1.. overlaps the kernel and the D2H of earlier pieces, so the
// H2D copy engine (the PCIe-bound resource: inputs are 3.7x the output bytes)
// stays busy.  Small pieces shorten the pipeline fill and drain.
// ---------------------------------------------------------------------------
constexpr int HOST_MAX_SLOTS = 4;

struct HostPathState {
  int device = -1;
  size_t cap = 0;
  unsigned char* buf[HOST_MAX_SLOTS] = {};
  cudaStream_t streams[HOST_MAX_SLOTS] = {};
  // bounce path (pageable caller buffers): pinned staging per slot, and completion events
  size_t pin_cap = 0;
  unsigned char* pin[2] = {};
  cudaEvent_t h2d_done[2] = {}, d2h_done[2] = {};
};

// ---------------------------------------------------------------------------
// Parallel host memcpy (the bounce path's pageable <-> pinned copies): a
// persistent pool of worker threads pulls 1 MiB chunks of a job list; the
// caller works too and returns when every chunk is copied.  One DMA engine
// moves ~55 GB/s over PCIe, one CPU thread copies ~10 GB/s: pageable buffers
// handed straight to cudaMemcpyAsync are staged by the driver on one thread.
// ---------------------------------------------------------------------------
class CopyPool {
 public:
  struct Job {
    unsigned char* dst;
    const unsigned char* src;
    size_t bytes;
  };
  static CopyPool& get() {
    static CopyPool pool;
    return pool;
  }
  void copy(const std::vector<Job>& jobs) {
    std::vector<Job> chunks;
    const size_t CH = (size_t)1 << 20;
    for (const Job& j : jobs)
      for (size_t o = 0; o < j.bytes; o += CH) chunks.push_back({j.dst + o, j.src + o, std::min(CH, j.bytes - o)});
    if (chunks.empty()) return;
    std::unique_lock<std::mutex> lk(mu_);
    work_ = &chunks;
    next_.store(0);
    pending_.store((int64_t)chunks.size());
    ++gen_;
    cv_.notify_all();
    lk.unlock();
    drain(&chunks);
    lk.lock();
    // every chunk copied AND no worker still inside drain() with this job list
    done_cv_.wait(lk, [&] { return pending_.load() == 0 && active_ == 0; });
    work_ = nullptr;
  }

 private:
  CopyPool() {
    const int hw = (int)std::thread::hardware_concurrency();
    // 8 copy threads (measured best on a 16-core host: more contend with the DMA for host memory)
    const int n = std::max(0, std::min(env_int("TXB_HOST_THREADS", std::min(8, std::max(1, hw / 2))), 64) - 1);
    for (int i = 0; i < n; ++i) threads_.emplace_back([this] { loop(); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : threads_) t.join();
  }
  void drain(std::vector<Job>* w) {
    for (;;) {
      const int64_t i = next_.fetch_add(1);
      if (i >= (int64_t)w->size()) return;
      const Job& j = (*w)[i];
      memcpy(j.dst, j.src, j.bytes);
      if (pending_.fetch_sub(1) == 1) {
        std::lock_guard<std::mutex> lk(mu_);
        done_cv_.notify_all();
      }
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
      if (stop_) return;
      seen = gen_;
      std::vector<Job>* w = work_;  // read under the lock: this generation's list (or none)
      if (!w) continue;
      ++active_;
      lk.unlock();
      drain(w);
      lk.lock();
      if (--active_ == 0) done_cv_.notify_all();
    }
  }
  std::vector<std::thread> threads_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  std::vector<Job>* work_ = nullptr;
  std::atomic<int64_t> next_{0}, pending_{0};
  int active_ = 0;  // workers inside drain() (guarded by mu_)
  uint64_t gen_ = 0;
  bool stop_ = false;
};

static std::mutex g_host_mu;
static std::vector<HostPathState> g_host_state;

static int host_state(int dev, size_t need, HostPathState*& out) {
  if ((int)g_host_state.size() <= dev) g_host_state.resize(dev + 1);
  HostPathState& s = g_host_state[dev];
  if (!s.streams[0]) {
    for (int i = 0; i < HOST_MAX_SLOTS; ++i)
      TXB_CUDA_TRY(cudaStreamCreateWithFlags(&s.streams[i], cudaStreamNonBlocking));
  }
  if (s.cap < need) {
    for (int i = 0; i < HOST_MAX_SLOTS; ++i) {
      if (s.buf[i]) cudaFree(s.buf[i]);
      s.buf[i] = nullptr;
    }
    s.cap = 0;
    for (int i = 0; i < HOST_MAX_SLOTS; ++i) TXB_CUDA_TRY(cudaMalloc(&s.buf[i], need));
    s.cap = need;
  }
  s.device = dev;
  out = &s;
  return TXB_OK;
}

int integrate_host(const Config& c, int n_b, int64_t n_cells, const void* basis,
                   const void* basis_der, const void* weights, const void* inv_j,
                   const void* det_j, const void* coeffs, const void* aux, void* out, int n_bl,
                   int n_cb) {
  int rc = validate(c);
  if (rc) return rc;
  if (n_cells == 0) return TXB_OK;
  if (!inv_j || !det_j || !coeffs || !out || (c.aux != 0 && !aux)) {
    set_error("NULL host pointer for a per-cell array");
    return TXB_E_ARG;
  }
  const int s = c.dtype;
  const int nb = c.dim + 1;
  const int auxw = c.aux == 1 ? 1 : (c.aux == 2 ? nb : 0);
  const int64_t per_cell[5] = {(int64_t)c.dim * c.dim * s, s, (int64_t)nb * c.n_comp * s,
                               (int64_t)auxw * s, (int64_t)nb * c.n_comp * s};

  // Zero copy: when every buffer is pinned host memory mapped into the device
  // address space (cudaHostAlloc / torch pin_memory under UVA), the kernel's
  // bulk copies read the inputs and its stores write the element vectors over
  // PCIe directly: one launch, no device staging buffers, the H2D and D2H
  // streams overlapping each other and the arithmetic.  Same PCIe-bound speed
  // as the staged path (profiles/r1s_e2e.md).  Pageable buffers take the
  // staged, pipelined path below.
  if (env_int("TXB_HOST_ZERO_COPY", 1)) {
    const void* hp[5] = {inv_j, det_j, coeffs, aux, out};
    void* dp[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    bool mapped = true;
    for (int r = 0; r < 5 && mapped; ++r) {
      if (r == 3 && !auxw) continue;
      cudaPointerAttributes at;
      if (cudaPointerGetAttributes(&at, hp[r]) != cudaSuccess || at.type != cudaMemoryTypeHost ||
          !at.devicePointer) {
        cudaGetLastError();
        mapped = false;
        break;
      }
      dp[r] = at.devicePointer;
    }
    if (mapped) {
      int dev = 0;
      TXB_CUDA_TRY(cudaGetDevice(&dev));
      std::lock_guard<std::mutex> lk(g_host_mu);
      HostPathState* st = nullptr;
      int rc0 = host_state(dev, 0, st);
      if (rc0) return rc0;
      rc0 = integrate_device(c, n_b, n_cells, basis, basis_der, weights, dp[0], dp[1], dp[2], auxw ? dp[3] : nullptr,
                             dp[4], n_bl, n_cb, st->streams[0], true);
      if (rc0) return rc0;
      TXB_CUDA_TRY(cudaStreamSynchronize(st->streams[0]));
      return TXB_OK;
    }
  }
  int64_t cell_bytes = 0;
  for (int64_t v : per_cell) cell_bytes += v;
  // Pageable caller buffers (plain numpy arrays: the reference's own calling
  // convention): bounce through pinned staging, the host copies in parallel
  // (CopyPool) and overlapped with the DMA / kernel / DMA of the neighbouring
  // piece.  (Handing pageable memory to cudaMemcpyAsync makes the driver stage
  // it on one thread: 14.4 ms per 2^20-cell f64 call; profiles/r1s_e2e.md.)
  {
    const void* hp[5] = {inv_j, det_j, coeffs, aux, out};
    bool pageable = false;
    for (int r = 0; r < 5; ++r) {
      if (r == 3 && !auxw) continue;
      cudaPointerAttributes at;
      if (cudaPointerGetAttributes(&at, hp[r]) != cudaSuccess) {
        cudaGetLastError();
        pageable = true;
      } else if (at.type == cudaMemoryTypeUnregistered) {
        pageable = true;
      }
    }
    if (pageable && env_int("TXB_HOST_BOUNCE", 1)) {
      const int64_t pb = (int64_t)std::max(1, env_int("TXB_HOST_BOUNCE_MB", 32)) << 20;
      int64_t piece = std::max<int64_t>(64, pb / cell_bytes);
      piece = (piece + 63) / 64 * 64;
      piece = std::min<int64_t>(piece, (n_cells + 63) / 64 * 64);
      size_t reg[5], need = 0;
      for (int r = 0; r < 5; ++r) {
        reg[r] = need;
        need += (size_t)((per_cell[r] * piece + 255) / 256 * 256);
      }
      int dev = 0;
      TXB_CUDA_TRY(cudaGetDevice(&dev));
      std::lock_guard<std::mutex> lk(g_host_mu);
      HostPathState* st = nullptr;
      int rc0 = host_state(dev, need, st);
      if (rc0) return rc0;
      if (st->pin_cap < need) {
        for (int i = 0; i < 2; ++i) {
          if (st->pin[i]) cudaFreeHost(st->pin[i]);
          st->pin[i] = nullptr;
        }
        st->pin_cap = 0;
        for (int i = 0; i < 2; ++i) TXB_CUDA_TRY(cudaHostAlloc((void**)&st->pin[i], need, cudaHostAllocDefault));
        st->pin_cap = need;
      }
      for (int i = 0; i < 2; ++i) {
        if (!st->h2d_done[i]) TXB_CUDA_TRY(cudaEventCreateWithFlags(&st->h2d_done[i], cudaEventDisableTiming));
        if (!st->d2h_done[i]) TXB_CUDA_TRY(cudaEventCreateWithFlags(&st->d2h_done[i], cudaEventDisableTiming));
      }
      const unsigned char* src[4] = {(const unsigned char*)inv_j, (const unsigned char*)det_j,
                                     (const unsigned char*)coeffs, (const unsigned char*)aux};
      CopyPool& pool = CopyPool::get();
      const int64_t n_pieces = (n_cells + piece - 1) / piece;
      auto copy_out = [&](int64_t q) {
        const int sl = (int)(q % 2);
        const int64_t c0 = q * piece, n = std::min(piece, n_cells - c0);
        cudaError_t e = cudaEventSynchronize(st->d2h_done[sl]);
        if (e != cudaSuccess) return cuda_fail(e, "cudaEventSynchronize(d2h)");
        pool.copy({{(unsigned char*)out + c0 * per_cell[4], st->pin[sl] + reg[4], (size_t)(n * per_cell[4])}});
        return (int)TXB_OK;
      };
      for (int64_t q = 0; q < n_pieces; ++q) {
        const int sl = (int)(q % 2);
        cudaStream_t sm = st->streams[sl];
        const int64_t c0 = q * piece, n = std::min(piece, n_cells - c0);
        if (q >= 2) TXB_CUDA_TRY(cudaEventSynchronize(st->h2d_done[sl]));  // staging slot free again
        std::vector<CopyPool::Job> in;
        for (int r = 0; r < 4; ++r)
          if (per_cell[r]) in.push_back({st->pin[sl] + reg[r], src[r] + c0 * per_cell[r], (size_t)(n * per_cell[r])});
        pool.copy(in);
        unsigned char* dptr[5];
        for (int r = 0; r < 5; ++r) dptr[r] = st->buf[sl] + reg[r];
        for (int r = 0; r < 4; ++r)
          if (per_cell[r])
            TXB_CUDA_TRY(cudaMemcpyAsync(dptr[r], st->pin[sl] + reg[r], n * per_cell[r], cudaMemcpyHostToDevice, sm));
        TXB_CUDA_TRY(cudaEventRecord(st->h2d_done[sl], sm));
        rc0 = integrate_device(c, n_b, n, basis, basis_der, weights, dptr[0], dptr[1], dptr[2],
                               auxw ? dptr[3] : nullptr, dptr[4], n_bl, n_cb, sm);
        if (rc0) return rc0;
        TXB_CUDA_TRY(cudaMemcpyAsync(st->pin[sl] + reg[4], dptr[4], n * per_cell[4], cudaMemcpyDeviceToHost, sm));
        TXB_CUDA_TRY(cudaEventRecord(st->d2h_done[sl], sm));
        if (q >= 1) {  // the previous piece's element vectors, while this piece runs
          rc0 = copy_out(q - 1);
          if (rc0) return rc0;
        }
      }
      rc0 = copy_out(n_pieces - 1);
      if (rc0) return rc0;
      return TXB_OK;
    }
  }
  // Pieces of ~TXB_HOST_PIECE_MB MiB (multiple of 64 cells, keeps every slice 16B aligned).
  const int64_t piece_bytes = (int64_t)std::max(1, env_int("TXB_HOST_PIECE_MB", 32)) << 20;
  const int slots = std::min(HOST_MAX_SLOTS, std::max(2, env_int("TXB_HOST_SLOTS", 2)));
  int64_t piece = std::max<int64_t>(64, piece_bytes / cell_bytes);
  piece = (piece + 63) / 64 * 64;
  piece = std::min<int64_t>(piece, (n_cells + 63) / 64 * 64);
  size_t need = 0;
  for (int64_t v : per_cell) need += (size_t)((v * piece + 255) / 256 * 256);

  int dev = 0;
  TXB_CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_host_mu);
  HostPathState* st = nullptr;
  rc = host_state(dev, need, st);
  if (rc) return rc;

  const unsigned char* src[4] = {(const unsigned char*)inv_j, (const unsigned char*)det_j,
                                 (const unsigned char*)coeffs, (const unsigned char*)aux};
  int64_t p = 0;
  for (int64_t c0 = 0; c0 < n_cells; c0 += piece, ++p) {
    const int slot = (int)(p % slots);
    cudaStream_t sm = st->streams[slot];
    const int64_t n = std::min(piece, n_cells - c0);
    unsigned char* base = st->buf[slot];
    unsigned char* dptr[5];
    size_t off = 0;
    for (int r = 0; r < 5; ++r) {
      dptr[r] = base + off;
      off += (size_t)((per_cell[r] * piece + 255) / 256 * 256);
    }
    for (int r = 0; r < 4; ++r)
      if (per_cell[r])
        TXB_CUDA_TRY(cudaMemcpyAsync(dptr[r], src[r] + c0 * per_cell[r], n * per_cell[r],
                                     cudaMemcpyHostToDevice, sm));
    rc = integrate_device(c, n_b, n, basis, basis_der, weights, dptr[0], dptr[1], dptr[2],
                          auxw ? dptr[3] : nullptr, dptr[4], n_bl, n_cb, sm);
    if (rc) return rc;
    TXB_CUDA_TRY(cudaMemcpyAsync((unsigned char*)out + c0 * per_cell[4], dptr[4], n * per_cell[4],
                                 cudaMemcpyDeviceToHost, sm));
  }
  for (int i = 0; i < slots; ++i) TXB_CUDA_TRY(cudaStreamSynchronize(st->streams[i]));
  return TXB_OK;
}

// STREAM-like probe: read R bytes, write W bytes with 16-byte accesses,
// grid-stride; the write value depends on the reads so nothing is elided.
__global__ void stream_probe_kernel(const uint4* __restrict__ src, int64_t n_read,
                                    uint4* __restrict__ dst, int64_t n_write) {
  constexpr int U = 8;  // independent 16-byte loads in flight per thread
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = n_read > n_write ? n_read : n_write;
  for (int64_t base = t0; base < n; base += stride * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * stride;
      v[u] = i < n_read ? __ldcs(src + i) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * stride;
      if (i < n_write) __stcs(dst + i, v[u]);
    }
  }
}

}  // namespace txb

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
using namespace txb;

extern "C" int txb_abi_version(void) { return 1; }

extern "C" int txb_query(int form_code, int aux_mode, int dtype_bytes, int dim, int n_q,
                         int n_comp) {
  Config c{form_code, aux_mode, dtype_bytes, dim, n_q, n_comp};
  return validate(c);
}

extern "C" int txb_launch_config(int form_code, int aux_mode, int dtype_bytes, int dim, int n_q,
                                 int n_comp, int64_t n_cells, int n_bl, int n_cb, int* n_bc,
                                 int* n_t, int* stages, int* smem_bytes, int* grid, int* n_bl_used,
                                 int* n_cb_used) {
  Config c{form_code, aux_mode, dtype_bytes, dim, n_q, n_comp};
  int rc = validate(c);
  if (rc) return rc;
  KernelInfo k;  // reports the standard-P1-table kernel's geometry
  if (!pick_kernel(c, true, k)) return TXB_E_UNSUPPORTED;
  size_tuning(c, n_cells, k);
  int ndev = 0;
  const bool have_dev = cudaGetDeviceCount(&ndev) == cudaSuccess && ndev > 0;
  if (!have_dev) cudaGetLastError();
  Geometry g;
  rc = compute_geometry(c, k, n_cells, n_bl, n_cb, have_dev, g);
  if (rc) return rc;
  if (n_bc) *n_bc = g.n_bc;
  if (n_t) *n_t = g.n_t;
  if (stages) *stages = g.stages;
  if (smem_bytes) *smem_bytes = g.smem;
  if (grid) *grid = g.grid;
  if (n_bl_used) *n_bl_used = g.n_bl;
  if (n_cb_used) *n_cb_used = g.n_cb;
  return TXB_OK;
}

extern "C" int txb_integrate_cells(int form_code, int aux_mode, int dtype_bytes, int dim, int n_b,
                                   int n_q, int n_comp, int64_t n_cells, const void* basis,
                                   const void* basis_der, const void* weights, const void* inv_j,
                                   const void* det_j, const void* coeffs, const void* aux,
                                   void* out, int n_bl, int n_cb, void* stream) {
  Config c{form_code, aux_mode, dtype_bytes, dim, n_q, n_comp};
  return integrate_device(c, n_b, n_cells, basis, basis_der, weights, inv_j, det_j, coeffs, aux,
                          out, n_bl, n_cb, (cudaStream_t)stream);
}

extern "C" int txb_integrate_cells_host(int form_code, int aux_mode, int dtype_bytes, int dim,
                                        int n_b, int n_q, int n_comp, int64_t n_cells,
                                        const void* basis, const void* basis_der,
                                        const void* weights, const void* inv_j, const void* det_j,
                                        const void* coeffs, const void* aux, void* out, int n_bl,
                                        int n_cb) {
  Config c{form_code, aux_mode, dtype_bytes, dim, n_q, n_comp};
  return integrate_host(c, n_b, n_cells, basis, basis_der, weights, inv_j, det_j, coeffs, aux, out,
                        n_bl, n_cb);
}

extern "C" int txb_debug_trace(void* device_buf, int64_t capacity_u64) {
  set_trace_buffer((unsigned long long*)device_buf, capacity_u64);
  return TXB_OK;
}

extern "C" int txb_stream_probe(const void* src, int64_t read_bytes, void* dst,
                                int64_t write_bytes, void* stream) {
  if ((read_bytes && !src) || (write_bytes && !dst) || (read_bytes % 16) || (write_bytes % 16)) {
    set_error("stream probe needs non-NULL buffers and 16-byte multiples");
    return TXB_E_ARG;
  }
  int dev = 0;
  TXB_CUDA_TRY(cudaGetDevice(&dev));
  const DeviceProps p = device_props(dev);
  const int grid = std::max(1, p.sms) * 4;
  // 4 x 512-thread CTAs per SM, 8 loads each in flight

  stream_probe_kernel<<<grid, 512, 0, (cudaStream_t)stream>>>(
      (const uint4*)src, read_bytes / 16, (uint4*)dst, write_bytes / 16);
  TXB_CUDA_TRY(cudaGetLastError());
  return TXB_OK;
}
