// txb_integrate.cu — thread-transposed P1 element integration for sm_100a.
//
// B200-native restatement of the paper's kernel (Knepley, Rupp, Terrel,
// arXiv:1607.04245, §3 and the appendix pseudocode) behind the reference's
// compiled-lane interface (txfem/_kernels_cy.pyx:37-123).
//
// Decomposition (paper §3; txfem/schedule.py:82-113):
//   block  = N_bs = N_b * N_q cells
//   batch  = N_bc = N_bl * N_bs cells            -> one shared-memory stage
//   chunk  = N_cb consecutive batches             -> one CTA work item
//   N_t    = N_bc * N_comp threads per CTA (capped at 512 physical threads;
//            a CTA then walks the same work items in more steps)
// Each CTA is persistent: it walks chunks blockIdx.x, blockIdx.x + gridDim.x,
// ... and their batches in order, so every CTA streams through the cell arrays
// in lock-step with the others.
//
// Per batch:
//   loader      one elected thread issues cp.async.bulk copies (UBLKCP) of the
//               batch's contiguous inv_j / det_j / coeffs / aux byte ranges
//               into a ring of `stages` shared-memory stages, completion on an
//               mbarrier (expect_tx); the ring runs `stages-1` batches ahead.
//   quadrature  one thread per (cell, q): pulled-back gradients T[q][b][k],
//   phase       grad u, aux value, inlined f1, scale by detJ*w -> smem
//               (txfem/device.py:267-330, _kernels_cy.pyx:70-111)
//   barrier     one __syncthreads (the paper's "TRANSPOSE THREADS")
//   basis       one thread per element-vector entry (cell, b, c): the
//   phase       reduction-free sum over (q, k) of T[q][b][k] * f1s[q][c][k];
//               thread index == flat output index, so the stores coalesce
//               (txfem/device.py:335-361, _kernels_cy.pyx:113-123)
//
// Numerics: products and sums round one at a time in the reference's pinned
// order (txfem/reference.py:10-19) -> bit-identical to the reference lanes.
#include "txb_common.cuh"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

namespace txb {

constexpr int MAX_D = TXB_MAX_DIM, MAX_B = TXB_MAX_BASIS, MAX_C = TXB_MAX_COMP,
              MAX_Q = TXB_MAX_QUAD;
constexpr int MAX_CTA_THREADS = 512;

template <typename T>
struct Tabulation {
  T B[MAX_Q * MAX_B];          // basis[q][b]
  T D[MAX_Q * MAX_B * MAX_D];  // basis_der[q][b][j]
  T W[MAX_Q];                  // weights[q]
};

template <typename T>
struct IntegrateArgs {
  const T* inv_j;
  const T* det_j;
  const T* coeffs;
  const T* aux;
  T* out;
  int64_t n_cells;
  int64_t n_batches;
  int64_t n_chunks;
  int n_bc;     // cells per batch
  int n_cb;     // batches per chunk
  int stages;   // ring depth
  int bulk;     // 1: full batches arrive by bulk copy; 0: cooperative loads
  Tabulation<T> tab;
};

// Per-cell shared-memory strides of the phase-1 -> phase-2 exchange; odd
// element strides keep both 32- and 64-bit accesses bank-conflict free.
template <int D, int NQ, int NCOMP>
struct Strides {
  static constexpr int NB = D + 1;
  static constexpr int TRANS = make_odd(NQ * NB * D);
  static constexpr int F1S = make_odd(NQ * NCOMP * D);
};

// Byte layout of one ring stage: four 16-byte aligned regions holding the
// batch's contiguous slices of inv_j, det_j, coeffs and aux.
template <typename T, int D, int NCOMP, int AUX>
struct StageLayout {
  static constexpr int NB = D + 1;
  static constexpr int AUXW = AUX == 1 ? 1 : (AUX == 2 ? NB : 0);
  __host__ __device__ static int inv_bytes(int n) { return round_up(n * D * D * (int)sizeof(T), 16); }
  __host__ __device__ static int det_bytes(int n) { return round_up(n * (int)sizeof(T), 16); }
  __host__ __device__ static int coef_bytes(int n) { return round_up(n * NB * NCOMP * (int)sizeof(T), 16); }
  __host__ __device__ static int aux_bytes(int n) { return round_up(n * AUXW * (int)sizeof(T), 16); }
  __host__ __device__ static int stage_bytes(int n) {
    return inv_bytes(n) + det_bytes(n) + coef_bytes(n) + aux_bytes(n);
  }
};

template <typename T, int D, int NQ, int NCOMP>
__host__ __device__ inline int scratch_bytes(int n_bc) {
  using S = Strides<D, NQ, NCOMP>;
  return round_up(n_bc * (S::TRANS + S::F1S) * (int)sizeof(T), 16);
}

// Vectorised shared-memory row load: N consecutive T starting at p; uses the
// widest access the row alignment allows (row starts are multiples of N*sizeof(T)).
template <typename T, int N>
__device__ __forceinline__ void load_row(const T* __restrict__ p, T (&r)[N]) {
  constexpr int BYTES = N * (int)sizeof(T);
  if constexpr (BYTES % 16 == 0) {
    constexpr int V = 16 / sizeof(T);
#pragma unroll
    for (int i = 0; i < N; i += V) {
      const uint4 v = *reinterpret_cast<const uint4*>(p + i);
      memcpy(&r[i], &v, 16);
    }
  } else if constexpr (BYTES % 8 == 0) {
    constexpr int V = 8 / sizeof(T);
#pragma unroll
    for (int i = 0; i < N; i += V) {
      const uint2 v = *reinterpret_cast<const uint2*>(p + i);
      memcpy(&r[i], &v, 8);
    }
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) r[i] = p[i];
  }
}

template <typename T, int D, int NQ, int NCOMP, int FORM, int AUX>
__global__ void __launch_bounds__(MAX_CTA_THREADS)
integrate_kernel(const __grid_constant__ IntegrateArgs<T> a) {
  constexpr int NB = D + 1;
  constexpr int DD = D * D;
  constexpr int NBC = NB * NCOMP;  // element-vector entries per cell
  using L = StageLayout<T, D, NCOMP, AUX>;
  using S = Strides<D, NQ, NCOMP>;

  extern __shared__ __align__(128) unsigned char smem[];
  const int nbc = a.n_bc;
  const int tid = threadIdx.x;
  const int nt = blockDim.x;
  const int stage_bytes = L::stage_bytes(nbc);
  T* s_trans = reinterpret_cast<T*>(smem + a.stages * stage_bytes);
  T* s_f1s = s_trans + nbc * S::TRANS;
  uint64_t* bars =
      reinterpret_cast<uint64_t*>(smem + a.stages * stage_bytes + scratch_bytes<T, D, NQ, NCOMP>(nbc));

  // Batch sequence of this CTA: chunks blockIdx.x + k*gridDim.x, N_cb batches each.
  auto batch_of = [&](int64_t i) -> int64_t {
    const int64_t k = i / a.n_cb;
    const int64_t ci = blockIdx.x + k * gridDim.x;
    if (ci >= a.n_chunks) return -1;
    const int64_t b = ci * a.n_cb + (i - k * a.n_cb);
    return b < a.n_batches ? b : -1;
  };
  auto full_batch = [&](int64_t b) { return (b + 1) * (int64_t)nbc <= a.n_cells; };

  const uint64_t policy = l2_evict_first_policy();
  // Loader: one thread posts the byte count and the four bulk copies.
  auto issue = [&](int64_t i) {
    const int64_t b = batch_of(i);
    if (b < 0 || !a.bulk || !full_batch(b)) return;
    unsigned char* st = smem + (int)(i % a.stages) * stage_bytes;
    uint64_t* bar = bars + (i % a.stages);
    const int64_t c0 = b * nbc;
    const uint32_t ib = nbc * DD * sizeof(T), db = nbc * sizeof(T), cb = nbc * NBC * sizeof(T),
                   ab = nbc * L::AUXW * sizeof(T);
    mbar_arrive_expect_tx(bar, ib + db + cb + ab);
    bulk_g2s(st, a.inv_j + c0 * DD, ib, bar, policy);
    bulk_g2s(st + L::inv_bytes(nbc), a.det_j + c0, db, bar, policy);
    bulk_g2s(st + L::inv_bytes(nbc) + L::det_bytes(nbc), a.coeffs + c0 * NBC, cb, bar, policy);
    if constexpr (AUX != 0)
      bulk_g2s(st + L::inv_bytes(nbc) + L::det_bytes(nbc) + L::coef_bytes(nbc),
               a.aux + c0 * L::AUXW, ab, bar, policy);
  };

  if (tid == 0) {
    for (int s = 0; s < a.stages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < a.stages; ++s) issue(s);

  // Basis-phase ownership is fixed per thread because N_t is a multiple of
  // N_b*N_comp: entry r = (b, c) of every cell this thread visits.
  const int r = tid % NBC;
  const int my_b = r / NCOMP, my_c = r % NCOMP;

  for (int64_t i = 0;; ++i) {
    const int64_t b = batch_of(i);
    if (b < 0) break;
    const int stage = (int)(i % a.stages);
    unsigned char* st = smem + stage * stage_bytes;
    const T* s_inv = reinterpret_cast<const T*>(st);
    const T* s_det = reinterpret_cast<const T*>(st + L::inv_bytes(nbc));
    const T* s_coef = reinterpret_cast<const T*>(st + L::inv_bytes(nbc) + L::det_bytes(nbc));
    const T* s_aux =
        reinterpret_cast<const T*>(st + L::inv_bytes(nbc) + L::det_bytes(nbc) + L::coef_bytes(nbc));
    const int64_t c0 = b * nbc;
    const int64_t rem = a.n_cells - c0;
    const int ncell = rem < nbc ? (int)rem : nbc;

    if (a.bulk && ncell == nbc) {
      mbar_wait(&bars[stage], (uint32_t)((i / a.stages) & 1));
    } else {
      // Cooperative load: partial tail batch or unaligned caller buffers.
      T* w_inv = const_cast<T*>(s_inv);
      T* w_det = const_cast<T*>(s_det);
      T* w_coef = const_cast<T*>(s_coef);
      T* w_aux = const_cast<T*>(s_aux);
      for (int e = tid; e < ncell * DD; e += nt) w_inv[e] = a.inv_j[c0 * DD + e];
      for (int e = tid; e < ncell; e += nt) w_det[e] = a.det_j[c0 + e];
      for (int e = tid; e < ncell * NBC; e += nt) w_coef[e] = a.coeffs[c0 * NBC + e];
      if constexpr (AUX != 0)
        for (int e = tid; e < ncell * L::AUXW; e += nt) w_aux[e] = a.aux[c0 * L::AUXW + e];
      __syncthreads();
    }

    // ---------------- quadrature phase: thread <-> (cell, q) ----------------
    for (int it = tid; it < ncell * NQ; it += nt) {
      const int cell = NQ == 1 ? it : it / NQ;
      const int q = NQ == 1 ? 0 : it - cell * NQ;
      T J[DD];
      load_row<T, DD>(s_inv + cell * DD, J);
      T cf[NBC];
      load_row<T, NBC>(s_coef + cell * NBC, cf);
      const T det = s_det[cell];
      const T* Dq = a.tab.D + q * NB * D;
      const T* Bq = a.tab.B + q * NB;

      T tr[NB][D];
      T* trans_out = s_trans + cell * S::TRANS + q * NB * D;
#pragma unroll
      for (int bb = 0; bb < NB; ++bb)
#pragma unroll
        for (int k = 0; k < D; ++k) {
          T acc = T(0);
#pragma unroll
          for (int j = 0; j < D; ++j) acc = add(acc, mul(Dq[bb * D + j], J[j * D + k]));
          tr[bb][k] = acc;
          trans_out[bb * D + k] = acc;
        }

      T g[NCOMP][D];
#pragma unroll
      for (int c = 0; c < NCOMP; ++c)
#pragma unroll
        for (int k = 0; k < D; ++k) g[c][k] = T(0);
#pragma unroll
      for (int bb = 0; bb < NB; ++bb)
#pragma unroll
        for (int c = 0; c < NCOMP; ++c)
#pragma unroll
          for (int k = 0; k < D; ++k) g[c][k] = add(g[c][k], mul(cf[bb * NCOMP + c], tr[bb][k]));

      T a0 = T(0);
      if constexpr (AUX == 1) {
        a0 = s_aux[cell];
      } else if constexpr (AUX == 2) {
#pragma unroll
        for (int bb = 0; bb < NB; ++bb) a0 = add(a0, mul(s_aux[cell * NB + bb], Bq[bb]));
      }
      (void)Bq;
      (void)a0;

      const T wq = a.tab.W[q];
      T* f1_out = s_f1s + cell * S::F1S + q * NCOMP * D;
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
          f1_out[c * D + k] = mul(mul(fv, det), wq);
        }
    }

    __syncthreads();  // ==== transpose threads ====

    // ------------- basis phase: thread <-> element entry (cell, b, c) -------------
    T* out = a.out + c0 * NBC;
    for (int o = tid; o < ncell * NBC; o += nt) {
      const int cell = o / NBC;
      const T* tr = s_trans + cell * S::TRANS + my_b * D;
      const T* f1 = s_f1s + cell * S::F1S + my_c * D;
      T e = T(0);
#pragma unroll
      for (int q = 0; q < NQ; ++q)
#pragma unroll
        for (int k = 0; k < D; ++k) e = add(e, mul(tr[q * NB * D + k], f1[q * NCOMP * D + k]));
      out[o] = e;
    }

    __syncthreads();  // stage and scratch free again
    if (tid == 0) issue(i + a.stages);
  }
}

// ---------------------------------------------------------------------------
// Host side: launch geometry, dispatch, C ABI.
// ---------------------------------------------------------------------------

struct Config {
  int form, aux, dtype, dim, n_q, n_comp;
};

struct Geometry {
  int n_bl, n_cb, n_bc, n_t, threads, stages, smem, grid;
  int64_t n_batches, n_chunks;
};

static int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return (v && *v) ? std::atoi(v) : dflt;
}

int validate(const Config& c) {
  if (c.dtype != 4 && c.dtype != 8) {
    set_error("dtype_bytes must be 4 or 8, got %d", c.dtype);
    return TXB_E_UNSUPPORTED;
  }
  if (c.dim < 2 || c.dim > 3) {
    set_error("dim must be 2 or 3, got %d", c.dim);
    return TXB_E_UNSUPPORTED;
  }
  if (c.n_q < 1 || c.n_q > MAX_Q) {
    set_error("n_q must be in [1, %d], got %d", MAX_Q, c.n_q);
    return TXB_E_UNSUPPORTED;
  }
  const bool ok = (c.form == 0 && c.aux == 0 && c.n_comp == 1) ||
                  (c.form == 1 && (c.aux == 1 || c.aux == 2) && c.n_comp == 1) ||
                  (c.form == 2 && c.aux == 0 && c.n_comp == c.dim);
  if (!ok) {
    set_error("cuda lane does not cover form_code=%d aux_mode=%d n_comp=%d dim=%d", c.form,
              c.aux, c.n_comp, c.dim);
    return TXB_E_UNSUPPORTED;
  }
  return TXB_OK;
}

// Tuned defaults (B200): N_bc*N_comp = N_t near 256-384 threads.
static void default_decomposition(const Config& c, int& n_bl, int& n_cb) {
  const int nb = c.dim + 1;
  if (n_bl <= 0) {
    const int target = env_int("TXB_TARGET_THREADS", 256);
    n_bl = std::max(1, target / (nb * c.n_q * c.n_comp));
    // keep N_bc a multiple of 4 cells so every batch slice is 16-byte sized
    while ((n_bl * nb * c.n_q) % 4 != 0) ++n_bl;
  }
  if (n_cb <= 0) n_cb = env_int("TXB_DEFAULT_NCB", 1);
}

template <typename T, int D, int NQ, int NCOMP, int FORM, int AUX>
struct Kernel {
  using L = StageLayout<T, D, NCOMP, AUX>;
  static void* fn() { return (void*)integrate_kernel<T, D, NQ, NCOMP, FORM, AUX>; }
  static int stage_bytes(int n_bc) { return L::stage_bytes(n_bc); }
  static int scratch(int n_bc) { return scratch_bytes<T, D, NQ, NCOMP>(n_bc); }
};

struct KernelInfo {
  void* fn;
  int (*stage_bytes)(int);
  int (*scratch)(int);
};

template <typename T, int D, int NQ>
static bool pick_form(const Config& c, KernelInfo& k) {
  if (c.form == 0) {
    using K = Kernel<T, D, NQ, 1, 0, 0>;
    k = {K::fn(), K::stage_bytes, K::scratch};
  } else if (c.form == 1 && c.aux == 1) {
    using K = Kernel<T, D, NQ, 1, 1, 1>;
    k = {K::fn(), K::stage_bytes, K::scratch};
  } else if (c.form == 1 && c.aux == 2) {
    using K = Kernel<T, D, NQ, 1, 1, 2>;
    k = {K::fn(), K::stage_bytes, K::scratch};
  } else if (c.form == 2) {
    using K = Kernel<T, D, NQ, D, 2, 0>;
    k = {K::fn(), K::stage_bytes, K::scratch};
  } else {
    return false;
  }
  return true;
}

template <typename T, int D>
static bool pick_nq(const Config& c, KernelInfo& k) {
  switch (c.n_q) {
    case 1: return pick_form<T, D, 1>(c, k);
    case 2: return pick_form<T, D, 2>(c, k);
    case 3: return pick_form<T, D, 3>(c, k);
    case 4: return pick_form<T, D, 4>(c, k);
    case 5: return pick_form<T, D, 5>(c, k);
    case 6: return pick_form<T, D, 6>(c, k);
    case 7: return pick_form<T, D, 7>(c, k);
    case 8: return pick_form<T, D, 8>(c, k);
  }
  return false;
}

static bool pick_kernel(const Config& c, KernelInfo& k) {
  if (c.dtype == 4) return c.dim == 2 ? pick_nq<float, 2>(c, k) : pick_nq<float, 3>(c, k);
  return c.dim == 2 ? pick_nq<double, 2>(c, k) : pick_nq<double, 3>(c, k);
}

struct DeviceProps {
  int sms = 0, smem_optin = 0;
};

static DeviceProps device_props(int dev) {
  static std::mutex mu;
  static std::vector<DeviceProps> cache;
  std::lock_guard<std::mutex> g(mu);
  if ((int)cache.size() <= dev) cache.resize(dev + 1);
  if (cache[dev].sms == 0) {
    cudaDeviceGetAttribute(&cache[dev].sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&cache[dev].smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  }
  return cache[dev];
}

static int compute_geometry(const Config& c, const KernelInfo& k, int64_t n_cells, int n_bl,
                            int n_cb, bool query_device, Geometry& g) {
  default_decomposition(c, n_bl, n_cb);
  const int nb = c.dim + 1;
  const int64_t n_bc64 = (int64_t)n_bl * nb * c.n_q;
  const int64_t n_t64 = n_bc64 * c.n_comp;
  if (n_bl < 1 || n_cb < 1) {
    set_error("n_bl and n_cb must be >= 1 (got %d, %d)", n_bl, n_cb);
    return TXB_E_CONFIG;
  }
  if (n_t64 > TXB_THREAD_LIMIT) {
    // txfem/schedule.py:86-90: the thread block may not exceed the device limit.
    set_error("thread block needs %lld threads, device limit is %d (n_bs=%d * n_comp=%d * n_bl=%d)",
              (long long)n_t64, TXB_THREAD_LIMIT, nb * c.n_q, c.n_comp, n_bl);
    return TXB_E_CONFIG;
  }
  g.n_bl = n_bl;
  g.n_cb = n_cb;
  g.n_bc = (int)n_bc64;
  g.n_t = (int)n_t64;
  // Physical CTA size: N_t, or the largest multiple of N_b*N_comp dividing it
  // that fits MAX_CTA_THREADS (same work items, walked in more steps).
  const int unit = nb * c.n_comp;
  int threads = g.n_t;
  if (threads > MAX_CTA_THREADS) {
    int best = unit;
    for (int m = unit; m <= MAX_CTA_THREADS; m += unit)
      if (g.n_t % m == 0) best = m;
    threads = best;
  }
  g.threads = threads;
  g.n_batches = (n_cells + g.n_bc - 1) / g.n_bc;
  g.n_chunks = (g.n_batches + n_cb - 1) / n_cb;

  const int stage = k.stage_bytes(g.n_bc);
  const int fixed = k.scratch(g.n_bc) + 8 * 8;  // scratch + up to 8 mbarriers
  int smem_cap = 227 * 1024;
  int dev = 0, sms = 148;
  if (query_device && cudaGetDevice(&dev) == cudaSuccess) {
    DeviceProps p = device_props(dev);
    if (p.smem_optin > 0) smem_cap = p.smem_optin;
    if (p.sms > 0) sms = p.sms;
  }
  const int target = env_int("TXB_SMEM_TARGET", 100 * 1024);
  int stages = env_int("TXB_STAGES", 0);
  if (stages <= 0) stages = std::min(8, std::max(2, (target - fixed) / std::max(stage, 1)));
  stages = std::min(stages, 8);
  while (stages > 2 && fixed + stages * stage > smem_cap) --stages;
  if (fixed + stages * stage > smem_cap) {
    set_error("shared-memory image needs %d bytes, budget is %d (n_bl=%d, scalar width %d)",
              fixed + 2 * stage, smem_cap, n_bl, c.dtype);
    return TXB_E_CAPACITY;
  }
  g.stages = stages;
  g.smem = fixed + stages * stage;

  int occ = 1;
  if (query_device) {
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    cudaFuncSetAttribute(k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, g.smem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k.fn, g.threads, g.smem) != cudaSuccess ||
        occ < 1)
      occ = 1;
  } else {
    occ = std::max(1, std::min(2048 / g.threads, smem_cap / std::max(g.smem, 1)));
  }
  const int64_t resident = (int64_t)occ * sms;
  g.grid = (int)std::max<int64_t>(1, std::min<int64_t>(g.n_chunks, resident));
  return TXB_OK;
}

template <typename T>
static void fill_tab(Tabulation<T>& t, int n_q, int n_b, int d, const void* basis,
                     const void* basis_der, const void* weights) {
  memset(&t, 0, sizeof(t));
  memcpy(t.B, basis, sizeof(T) * n_q * n_b);
  memcpy(t.D, basis_der, sizeof(T) * n_q * n_b * d);
  memcpy(t.W, weights, sizeof(T) * n_q);
}

template <typename T>
static int launch_t(const Config& c, const KernelInfo& k, const Geometry& g, int64_t n_cells,
                    const void* basis, const void* basis_der, const void* weights,
                    const void* inv_j, const void* det_j, const void* coeffs, const void* aux,
                    void* out, cudaStream_t stream) {
  IntegrateArgs<T> a;
  a.inv_j = (const T*)inv_j;
  a.det_j = (const T*)det_j;
  a.coeffs = (const T*)coeffs;
  a.aux = (const T*)aux;
  a.out = (T*)out;
  a.n_cells = n_cells;
  a.n_batches = g.n_batches;
  a.n_chunks = g.n_chunks;
  a.n_bc = g.n_bc;
  a.n_cb = g.n_cb;
  a.stages = g.stages;
  auto al16 = [](const void* p) { return ((uintptr_t)p & 15u) == 0; };
  a.bulk = al16(inv_j) && al16(det_j) && al16(coeffs) && (c.aux == 0 || al16(aux)) &&
           env_int("TXB_DISABLE_BULK", 0) == 0;
  fill_tab(a.tab, c.n_q, c.dim + 1, c.dim, basis, basis_der, weights);
  void* params[] = {&a};
  TXB_CUDA_TRY(cudaLaunchKernel(k.fn, dim3(g.grid), dim3(g.threads), params, (size_t)g.smem, stream));
  return TXB_OK;
}

int integrate_device(const Config& c, int n_b, int64_t n_cells, const void* basis,
                     const void* basis_der, const void* weights, const void* inv_j,
                     const void* det_j, const void* coeffs, const void* aux, void* out, int n_bl,
                     int n_cb, cudaStream_t stream) {
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
  if (!pick_kernel(c, k)) {
    set_error("no kernel instantiation for this configuration");
    return TXB_E_UNSUPPORTED;
  }
  Geometry g;
  rc = compute_geometry(c, k, n_cells, n_bl, n_cb, true, g);
  if (rc) return rc;
  if (n_cells == 0) return TXB_OK;
  if (!inv_j || !det_j || !coeffs || !out || (c.aux != 0 && !aux)) {
    set_error("NULL device pointer for a per-cell array");
    return TXB_E_ARG;
  }
  if (c.dtype == 4)
    return launch_t<float>(c, k, g, n_cells, basis, basis_der, weights, inv_j, det_j, coeffs, aux,
                           out, stream);
  return launch_t<double>(c, k, g, n_cells, basis, basis_der, weights, inv_j, det_j, coeffs, aux,
                          out, stream);
}

// ---------------------------------------------------------------------------
// Host-buffer path: pieces of cells pipelined over two streams
// (H2D of piece p+1 overlaps the kernel of p and the D2H of p-1).
// ---------------------------------------------------------------------------
struct HostPathState {
  int device = -1;
  size_t cap = 0;
  unsigned char* buf[2] = {nullptr, nullptr};
  cudaStream_t streams[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
};

static std::mutex g_host_mu;
static std::vector<HostPathState> g_host_state;

static int host_state(int dev, size_t need, HostPathState*& out) {
  if ((int)g_host_state.size() <= dev) g_host_state.resize(dev + 1);
  HostPathState& s = g_host_state[dev];
  if (!s.streams[0]) {
    for (int i = 0; i < 2; ++i) {
      TXB_CUDA_TRY(cudaStreamCreateWithFlags(&s.streams[i], cudaStreamNonBlocking));
      TXB_CUDA_TRY(cudaEventCreateWithFlags(&s.done[i], cudaEventDisableTiming));
    }
  }
  if (s.cap < need) {
    for (int i = 0; i < 2; ++i) {
      if (s.buf[i]) cudaFree(s.buf[i]);
      s.buf[i] = nullptr;
    }
    s.cap = 0;
    for (int i = 0; i < 2; ++i) TXB_CUDA_TRY(cudaMalloc(&s.buf[i], need));
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
  int64_t cell_bytes = 0;
  for (int64_t v : per_cell) cell_bytes += v;
  // Pieces of ~32 MiB (multiple of 64 cells, keeps every slice 16B aligned).
  int64_t piece = std::max<int64_t>(64, ((int64_t)32 << 20) / cell_bytes);
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
    const int slot = (int)(p & 1);
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
  for (int i = 0; i < 2; ++i) TXB_CUDA_TRY(cudaStreamSynchronize(st->streams[i]));
  return TXB_OK;
}

// STREAM-like probe: read R bytes, write W bytes with 16-byte accesses,
// grid-stride; the write value depends on the reads so nothing is elided.
__global__ void stream_probe_kernel(const uint4* __restrict__ src, int64_t n_read,
                                    uint4* __restrict__ dst, int64_t n_write) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = n_read > n_write ? n_read : n_write;
  uint32_t acc = 0;
  for (int64_t i = t0; i < n; i += stride) {
    uint4 v = make_uint4(0, 0, 0, 0);
    if (i < n_read) v = __ldcs(src + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
    if (i < n_write) __stcs(dst + i, make_uint4(v.x, v.y, v.z, acc));
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
  KernelInfo k;
  if (!pick_kernel(c, k)) return TXB_E_UNSUPPORTED;
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

extern "C" int txb_stream_probe(const void* src, int64_t read_bytes, void* dst,
                                int64_t write_bytes, void* stream) {
  if ((read_bytes && !src) || (write_bytes && !dst) || (read_bytes % 16) || (write_bytes % 16)) {
    set_error("stream probe needs non-NULL buffers and 16-byte multiples");
    return TXB_E_ARG;
  }
  int dev = 0;
  TXB_CUDA_TRY(cudaGetDevice(&dev));
  const DeviceProps p = device_props(dev);
  const int grid = std::max(1, p.sms) * 8;
  stream_probe_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
      (const uint4*)src, read_bytes / 16, (uint4*)dst, write_bytes / 16);
  TXB_CUDA_TRY(cudaGetLastError());
  return TXB_OK;
}
