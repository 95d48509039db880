// txb_kernels.cuh — device and host building blocks shared by the streaming
// kernels (cell-array integration, mesh-fused integration): tabulation in the
// parameter space, ring-stage layouts, the warp-specialised bulk-copy batch
// pipeline, launch-geometry selection.  See txb_integrate.cu for the design.
#pragma once

#include "txb_common.cuh"
#include "txb_pipeline.cuh"

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

namespace txb {

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

// Warp-private exchange area between the two phases: T and f1s.  Scalar forms
// use a component-major layout: row r holds the slice's CW cells at pitch
// P = CW + 4 (T: with the standard tables T[0] at r = k -- or, for SJ, the
// invJ rows = T[b>=1] at r = 0..D*D-1 and T[0] at r = D*D + k -- otherwise
// T[q][b][k] at r = (q*N_b+b)*D+k; f1s: r = (q*N_comp+c)*D+k), so the
// quadrature-phase stores (lane = cell) hit consecutive words and the
// basis-phase loads (lanes = (cell, b)) spread over the banks.  Vector forms keep a
// cell-major layout with odd strides (T[0] only; invJ rows from the stage),
// which measured faster for them.
template <typename T, int D, int NQ, int NCOMP, bool STD>
struct Scratch {
  static constexpr int NB = D + 1;
  static constexpr int CW = 32 / NQ;  // cells per warp slice
  static constexpr bool CM = NCOMP == 1;
  static constexpr int P = CW + 4;
  // STD: SJ keeps the invJ rows (T[b>=1]) and T[0] in the exchange area
  // (measured faster for 2D f32 only: 9.74 -> 9.15 us; 3D f32 and 2D f64 lose
  // to the larger area), otherwise T[0] only, the invJ rows read from the stage
  static constexpr bool SJ = CM && STD && D == 2 && sizeof(T) == 4;
  static constexpr int TR = STD ? (SJ ? D * D + D : D) : NQ * NB * D;
  static constexpr int F1 = NQ * NCOMP * D;
  static constexpr int TRS = make_odd(TR);
  static constexpr int F1S = make_odd(F1);
  __device__ static int tr(int lc, int r) { return CM ? r * P + lc : lc * TRS + r; }
  __device__ static int f1(int lc, int r) { return CM ? r * P + lc : lc * F1S + r; }
  static constexpr int TR_BYTES = round_up((CM ? P * TR : CW * TRS) * (int)sizeof(T), 16);
  static constexpr int BYTES = TR_BYTES + round_up((CM ? P * F1 : CW * F1S) * (int)sizeof(T), 16);
};

// Warp-private exchange area of the mesh-fused kernels: per cell the (cast) invJ rows = T[b>=1], T[0], and
// f1s, component-major (row = one component, the slice's cells at pitch
// CW + 4): conflict-free stores and loads (3D elasticity f64 given geometry
// 56.1 -> 48.6 us; the cell-major stride had 4-way conflicts).
template <typename T, int D, int NQ, int NCOMP>
struct MeshScratch {
  static constexpr int CW = 32 / NQ;
  static constexpr bool CM = true;  // component-major (measured faster for every form here)
  static constexpr int P = CW + 4;
  static constexpr int TR = D * D + D;  // invJ (D*D) then T[0] (D)
  static constexpr int TRS = make_odd(TR);
  static constexpr int F1 = NQ * NCOMP * D;
  static constexpr int F1S = make_odd(F1);
  __device__ static int tr(int lc, int r) { return CM ? r * P + lc : lc * TRS + r; }
  __device__ static int f1(int lc, int r) { return CM ? r * P + lc : lc * F1S + r; }
  static constexpr int TR_BYTES = round_up((CM ? P * TR : CW * TRS) * (int)sizeof(T), 16);
  static constexpr int BYTES = TR_BYTES + round_up((CM ? P * F1 : CW * F1S) * (int)sizeof(T), 16);
};

// Exactness note (why the chains below may skip the reference's "acc = 0;
// acc = acc + x" first step and its 0*x / 1*x products): in round-to-nearest
// a sum is -0 only if both operands are -0, so a chain started at +0 is never
// -0, and chains started at +0 vs at their first term differ at most in the
// SIGN OF A ZERO.  Every intermediate (T, grad u, f1s) only ever enters
// products that are summed into such a +0-started chain, where a zero term of
// either sign leaves the partial sum unchanged.  Hence only the final
// element-vector chain must start at +0 to reproduce the reference bit for
// bit; everything upstream may drop exact no-ops.  (Finite inputs.)

// ---------------------------------------------------------------------------
// Host-side launch geometry (shared)
// ---------------------------------------------------------------------------
struct Config {
  int form, aux, dtype, dim, n_q, n_comp;
};

struct Geometry {
  int n_bl, n_cb, n_bc, n_t, threads, warps, stages, smem, grid;
  int64_t n_chunks, chunk_cells;
  bool dynamic;
  // dynamic (cluster launch control): CTAs 0..resident-1 deal the first
  // static_batches batches round-robin, CTA resident + j owns batch
  // static_batches + j (txb_pipeline.cuh unit_batches)
  int resident;
  int64_t static_batches;
};

static int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return (v && *v) ? std::atoi(v) : dflt;
}

static int validate(const Config& c) {
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
    set_error("cuda lane does not cover form_code=%d aux_mode=%d n_comp=%d dim=%d", c.form, c.aux, c.n_comp,
              c.dim);
    return TXB_E_UNSUPPORTED;
  }
  return TXB_OK;
}

static int gcd(int a, int b) { return b ? gcd(b, a % b) : a; }

// Kernel families sharing the launch-geometry logic.
enum KernelFamily { FAMILY_CELLS = 0, FAMILY_MESH = 1, FAMILY_JIT = 2 };

// Cells per batch and in-flight bytes per SM (the ring-depth target),
// measured on B200 (profiles/r1v_batch_sweep.md).  Launch-sized problems
// (< 2^22 cells) favour smaller batches -- a shorter ramp and tail -- for the
// cell-array kernels: 128 cells except the 2D configurations whose N_bc steps
// are 96 cells, where 192 wins for scalar f32 and f64 elasticity (288 for f32
// elasticity once scheduling is dynamic, profiles/r2w_sweep.md); 96 KB in
// flight except 3D var-coef f64 (96 KB costs it an occupancy step: 26.0 ->
// 31.4 us) and 2D var-coef f32.  Streaming-sized problems keep the batches that
// amortise the per-batch overhead best (f32 256 cells: 3D var-coef f32 at 2^24
// 190 vs 208 us), as do the mesh-fused and run-time compiled kernels.
static int tuned_target_cells(const Config& c, int family, int64_t n_cells) {
  if (family != FAMILY_CELLS || n_cells >= ((int64_t)1 << 22)) return c.dtype == 8 ? 128 : 256;
  if (c.dim == 2 && c.n_q == 1 && c.n_comp == 2 && c.dtype == 4) return 288;  // r2w: 12.27 -> 11.92 us
  if (c.dim == 2 && c.n_q == 1 && ((c.n_comp == 1 && c.dtype == 4) || (c.n_comp == 2 && c.dtype == 8))) return 192;
  return 128;
}

static int tuned_inflight_kb(const Config& c, int family, int64_t n_cells) {
  if (family != FAMILY_CELLS || n_cells >= ((int64_t)1 << 22)) return 72;
  if (c.n_comp == 1 && ((c.dim == 3 && c.dtype == 8) || (c.dim == 2 && c.dtype == 4))) return 72;
  return 96;
}

// Default N_bl: batch near the tuned target (TXB_TARGET_CELLS overrides), N_bc
// a multiple of the warp slice CW = 32/N_q so no warp slice is partial.
static void default_decomposition(const Config& c, int family, int64_t n_cells, int& n_bl, int& n_cb) {
  const int nbs = (c.dim + 1) * c.n_q;
  if (n_bl <= 0) {
    const int cw = 32 / c.n_q;
    const int step = cw / gcd(cw, nbs);  // n_bl multiple of step -> N_bc multiple of cw
    const int target = env_int("TXB_TARGET_CELLS", tuned_target_cells(c, family, n_cells));
    int best = step, best_err = 1 << 30;
    for (int m = 1; m * step * nbs <= 1024; ++m) {
      const int err = std::abs(m * step * nbs - target);
      if (err < best_err) {
        best_err = err;
        best = m * step;
      }
    }
    n_bl = best;
  }
  if (n_cb <= 0) n_cb = env_int("TXB_DEFAULT_NCB", 0);  // 0: balanced contiguous chunks
}

struct KernelInfo {
  void* fn;
  int (*stage_bytes)(int);  // NULL: run-time layout below (JIT kernels)
  int (*scratch)(int);      // per consumer warp
  int cw;
  // run-time stage layout: scalars per cell of each of the four ring regions,
  // scalar width, scratch bytes per consumer warp (used when stage_bytes is NULL)
  int rt_region[4];
  int rt_s;
  int rt_scratch;
  int family;  // KernelFamily (0: the ahead-of-time cell-array kernels)
  int stage_extra;  // bytes per stage on top of stage_bytes(n_bc) (tiled kernels: the vertex table)
  int extra_warps;  // warps besides the consumers and the producer (tiled kernels: the gatherer)
  int fixed_extra;  // fixed shared-memory bytes besides scratch + pipeline (tiled kernels: `ready` barriers)
  int prefer_dynamic;  // dynamic batch scheduling whatever the stage size (tiled kernels: measured faster)
  int max_stages;      // ring-depth search limit (0: 8)
  int max_warps;       // consumer-warp cap (0: MAX_CONSUMER_WARPS); the warps loop over a batch's slices
  int stage(int n_bc) const {
    if (stage_bytes) return stage_bytes(n_bc) + stage_extra;
    int b = stage_extra;
    for (int r = 0; r < 4; ++r) b += round_up(n_bc * rt_region[r] * rt_s, 16);
    return b;
  }
  int scratch_bytes(int n_bc) const { return scratch ? scratch(n_bc) : rt_scratch; }
};

// True when every tabulated reference gradient is exactly the P1 one:
// D[q][0][j] = -1, D[q][b][j] = (b-1 == j) for b >= 1 (element.py:55-77).
template <typename T>
static bool is_standard_p1(const void* basis_der, int n_q, int d) {
  const T* D = (const T*)basis_der;
  const int nb = d + 1;
  for (int q = 0; q < n_q; ++q)
    for (int b = 0; b < nb; ++b)
      for (int j = 0; j < d; ++j) {
        const T want = b == 0 ? T(-1) : (b - 1 == j ? T(1) : T(0));
        const T got = D[(q * nb + b) * d + j];
        if (memcmp(&got, &want, sizeof(T)) != 0) return false;  // bitwise (no -0)
      }
  return true;
}

static bool standard_tables(const Config& c, const void* basis_der) {
  if (!basis_der) return false;
  return c.dtype == 4 ? is_standard_p1<float>(basis_der, c.n_q, c.dim)
                      : is_standard_p1<double>(basis_der, c.n_q, c.dim);
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

// The kernel's dynamic shared-memory limit is raised ONCE per (function,
// device) to the device's opt-in maximum and never lowered, so launches of
// the same kernel with different stage sizes from concurrent threads cannot
// race on the attribute (each launch passes its own size).
static bool allow_max_smem(void* fn, int dev, int smem_cap) {
  static std::mutex mu;
  static std::map<std::pair<void*, int>, bool> done;
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_pair(fn, dev);
  if (done.count(key)) return true;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_cap);
  if (e != cudaSuccess) {
    cuda_fail(e, "cudaFuncSetAttribute(MaxDynamicSharedMemorySize)");
    return false;
  }
  done[key] = true;
  return true;
}

static int compute_geometry(const Config& c, const KernelInfo& k, int64_t n_cells, int n_bl, int n_cb,
                            bool query_device, Geometry& g) {
  default_decomposition(c, k.family, n_cells, n_bl, n_cb);
  const int nb = c.dim + 1;
  const int64_t n_bc64 = (int64_t)n_bl * nb * c.n_q;
  const int64_t n_t64 = n_bc64 * c.n_comp;
  if (n_bl < 1 || n_cb < 0) {
    set_error("n_bl must be >= 1 and n_cb >= 1 (got %d, %d)", n_bl, n_cb);
    return TXB_E_CONFIG;
  }
  if (n_t64 > TXB_THREAD_LIMIT) {
    // txfem/schedule.py:86-90: the paper's thread block may not exceed the device limit.
    set_error("thread block needs %lld threads, device limit is %d (n_bs=%d * n_comp=%d * n_bl=%d)",
              (long long)n_t64, TXB_THREAD_LIMIT, nb * c.n_q, c.n_comp, n_bl);
    return TXB_E_CONFIG;
  }
  g.n_bl = n_bl;
  g.n_cb = n_cb;
  g.n_bc = (int)n_bc64;
  g.n_t = (int)n_t64;
  const int slices = (g.n_bc + k.cw - 1) / k.cw;
  const int wcap = std::max(1, std::min(k.max_warps > 0 ? k.max_warps : MAX_CONSUMER_WARPS,
                                        env_int("TXB_MAX_WARPS", MAX_CONSUMER_WARPS)));
  g.warps = std::min(wcap, slices);

  const int stage = k.stage(g.n_bc);
  int smem_cap = 227 * 1024;
  int dev = 0, sms = 148;
  if (query_device && cudaGetDevice(&dev) == cudaSuccess) {
    DeviceProps p = device_props(dev);
    if (p.smem_optin > 0) smem_cap = p.smem_optin;
    if (p.sms > 0) sms = p.sms;
  }
  // Large warp-private exchange areas (many quadrature points, big batches) may
  // not fit next to a 2-stage ring with one consumer warp per slice: fewer
  // consumer warps then loop over the batch's slices.
  const int scratch_w = k.scratch_bytes(g.n_bc);
  auto fixed_for = [&](int w) { return w * scratch_w + PIPELINE_SMEM_BYTES + 16 + k.fixed_extra; };
  while (g.warps > 1 && fixed_for(g.warps) + 2 * stage > smem_cap) --g.warps;
  g.threads = 32 * (g.warps + 1 + k.extra_warps);
  const int fixed = fixed_for(g.warps);
  // Ring depth: keep about TXB_INFLIGHT_KB (72 KB) of batch loads in flight
  // per SM -- (CTAs/SM) x (stages-1) x stage bytes ~ HBM bandwidth x latency
  // per SM.  Deeper rings only queue more requests and lengthen the launch
  // ramp (measured, profiles/r1_sweep.md).  TXB_STAGES forces a depth.
  const int forced = env_int("TXB_STAGES", 0);
  const int64_t inflight_target = (int64_t)env_int("TXB_INFLIGHT_KB", tuned_inflight_kb(c, k.family, n_cells)) * 1024;
  if (query_device && !allow_max_smem(k.fn, dev, smem_cap)) return TXB_E_CUDA;
  auto occupancy = [&](int smem) {
    int occ = 1;
    if (query_device) {
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k.fn, g.threads, smem) != cudaSuccess || occ < 1) {
        cudaGetLastError();
        occ = 1;
      }
    } else {
      occ = std::max(1, std::min(2048 / g.threads, smem_cap / std::max(smem, 1)));
    }
    return occ;
  };
  int best_s = -1, occ = 1;
  int64_t best_err = -1;
  // the choice depends only on the kernel shape: memoise it (the occupancy
  // queries cost microseconds of host time per launch otherwise)
  struct Key {
    void* fn;
    int threads, stage, fixed, forced, dev;
    int64_t target;
    bool operator<(const Key& o) const {
      return std::tie(fn, threads, stage, fixed, forced, dev, target) <
             std::tie(o.fn, o.threads, o.stage, o.fixed, o.forced, o.dev, o.target);
    }
  };
  static std::mutex memo_mu;
  static std::map<Key, std::pair<int, int>> memo;
  const Key key{k.fn, g.threads, stage, fixed, forced, query_device ? dev : -1, inflight_target};
  {
    std::lock_guard<std::mutex> lk(memo_mu);
    auto it = memo.find(key);
    if (it != memo.end()) {
      best_s = it->second.first;
      occ = it->second.second;
    }
  }
  const bool memoised = best_s >= 0;
  const int st_max = k.max_stages > 0 ? std::min(k.max_stages, MAX_STAGES) : 8;
  for (int st = 2; !memoised && st <= st_max; ++st) {
    if (forced > 0 && st != std::min(std::max(forced, 2), st_max)) continue;
    const int smem = fixed + st * stage;
    if (smem > smem_cap) break;
    const int o = occupancy(smem);
    const int64_t err = std::llabs((int64_t)o * (st - 1) * stage - inflight_target);
    if (best_s < 0 || err < best_err) {
      best_s = st;
      best_err = err;
      occ = o;
    }
  }
  if (best_s < 0) {
    set_error("shared-memory image needs %d bytes, budget is %d (n_bl=%d, scalar width %d)", fixed + 2 * stage,
              smem_cap, n_bl, c.dtype);
    return TXB_E_CAPACITY;
  }
  if (!memoised) {
    std::lock_guard<std::mutex> lk(memo_mu);
    memo[key] = {best_s, occ};
  }
  g.stages = best_s;
  g.smem = fixed + best_s * stage;
  const int64_t resident = (int64_t)occ * sms;
  if (n_cb > 0) {
    // paper mode: chunks of N_cb batches, round-robin over the CTAs
    g.chunk_cells = (int64_t)n_cb * g.n_bc;
  } else {
    // balanced mode: one contiguous chunk per resident CTA, 16-cell granular
    // (keeps every bulk-copy slice 16-byte aligned), so all CTAs finish together
    const int64_t per = (n_cells + resident - 1) / std::max<int64_t>(resident, 1);
    g.chunk_cells = std::max<int64_t>(16, (per + 15) / 16 * 16);
    g.n_cb = (int)((g.chunk_cells + g.n_bc - 1) / g.n_bc);
  }
  g.n_chunks = (n_cells + g.chunk_cells - 1) / g.chunk_cells;
  g.grid = (int)std::max<int64_t>(1, std::min<int64_t>(g.n_chunks, resident));
  // Default: dynamic batch scheduling so CTAs on SMs that get more bandwidth
  // take more batches and all finish together.  An explicit n_cb keeps the
  // paper's static chunk order.  Round 1 (an atomic-counter scheduler) found
  // it worth it only for >= 10 KB stages; with cluster launch control it wins
  // for every launch of >= 2^18 cells whatever the stage size (2^20 cells:
  // 2D var-coef f32 9.14 -> 8.45 us, 3D var-coef f32 13.49 -> 12.75, 2D
  // var-coef f64 16.70 -> 15.73; profiles/r2v_dyn.md) and loses ~1 % on the
  // 65,536-cell launch.
  const int dyn_env = env_int("TXB_DYNAMIC", -1);
  g.dynamic = n_cb <= 0 && (dyn_env < 0 ? (stage >= 10 * 1024 || k.prefer_dynamic || n_cells >= ((int64_t)1 << 18))
                                         : dyn_env != 0);
  g.resident = 0;
  g.static_batches = 0;
  if (g.dynamic) {
    // One CTA per scheduling unit; the resident CTAs cancel the grid's
    // not-yet-launched CTAs and run their units (cluster launch control), so
    // the grid stays persistent in effect.  ~TXB_STATIC_PCT % of the batches
    // (whole rounds of the resident grid) are dealt round-robin first.
    const int64_t n_batches = (n_cells + g.n_bc - 1) / g.n_bc;
    const int64_t r = std::max<int64_t>(1, std::min<int64_t>(n_batches, resident));
    // share of the batches dealt round-robin first (2D elasticity f32: 40 %, profiles/r2as_pct.md)
    const int pct_default = (c.dim == 2 && c.n_comp == 2 && c.dtype == 4 && k.family == FAMILY_CELLS) ? 40 : 60;
    const int pct = std::min(100, std::max(0, env_int("TXB_STATIC_PCT", pct_default)));
    g.static_batches = n_batches * pct / 100 / r * r;
    g.resident = g.static_batches > 0 ? (int)r : 0;
    const int64_t units = g.resident + (n_batches - g.static_batches);
    if (units > 0x7fffffff) {
      set_error("%lld batches exceed the grid limit", (long long)n_batches);
      return TXB_E_CONFIG;
    }
    g.grid = (int)std::max<int64_t>(1, units);
  }
  return TXB_OK;
}

// Debug timeline (txb_debug_trace): consecutive launches on this thread take
// consecutive slots of 4 stamps per CTA from the installed device buffer.
struct TraceState {
  unsigned long long* buf = nullptr;
  int64_t cap = 0, used = 0;
};
static thread_local TraceState g_trace;

static void set_trace_buffer(unsigned long long* buf, int64_t cap) {
  g_trace.buf = buf;
  g_trace.cap = buf ? cap : 0;
  g_trace.used = 0;
}

static unsigned long long* next_trace_slot(int grid) {
  if (!g_trace.buf || g_trace.used + 4 * (int64_t)grid > g_trace.cap) return nullptr;
  unsigned long long* p = g_trace.buf + g_trace.used;
  g_trace.used += 4 * (int64_t)grid;
  return p;
}

// Batches per CTA to warm into L2 before the programmatic-launch wait
// (TXB_PREFETCH_BATCHES; default: the ring depth).
static int prefetch_batches(const Geometry& g) {
  const int v = env_int("TXB_PREFETCH_BATCHES", -1);
  return v < 0 ? g.stages : v;
}

template <typename T>
static void fill_tab(Tabulation<T>& t, int n_q, int n_b, int d, const void* basis, const void* basis_der,
                     const void* weights) {
  memset(&t, 0, sizeof(t));
  memcpy(t.B, basis, sizeof(T) * n_q * n_b);
  memcpy(t.D, basis_der, sizeof(T) * n_q * n_b * d);
  memcpy(t.W, weights, sizeof(T) * n_q);
}


}  // namespace txb
