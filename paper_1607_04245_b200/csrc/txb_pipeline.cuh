// txb_pipeline.cuh — the warp-specialised bulk-copy batch pipeline shared by
// every streaming kernel of the library (cell-array integration, mesh-fused
// integration, run-time compiled user physics).  Device code only: NVRTC
// compiles this file from memory for the user-physics kernels (txb_jit.cu).
#pragma once

#include "txb_device.cuh"

namespace txb {

// Stage release: every consumer lane arrives on the stage's `empty` barrier
// (1), or lane 0 alone after __syncwarp (0).  Both are race-free by the PTX
// memory model; (1) does not rely on __syncwarp's memory ordering and is the
// form compute-sanitizer racecheck verifies clean (profiles/r1_sanitizer.md).
#ifndef TXB_EMPTY_ARRIVE_ALL
#define TXB_EMPTY_ARRIVE_ALL 1
#endif
constexpr int EMPTY_ARRIVALS_PER_WARP = TXB_EMPTY_ARRIVE_ALL ? 32 : 1;

constexpr int MAX_D = TXB_MAX_DIM, MAX_B = TXB_MAX_BASIS, MAX_Q = TXB_MAX_QUAD;
constexpr int MAX_CONSUMER_WARPS = 16;
constexpr int MAX_STAGES = 16;  // ring depth cap (the cell-array kernels search <= 8)
constexpr int MAX_CTA_THREADS = 32 * (MAX_CONSUMER_WARPS + 1);

template <typename T>
struct Tabulation {
  T B[MAX_Q * MAX_B];          // basis[q][b]
  T D[MAX_Q * MAX_B * MAX_D];  // basis_der[q][b][j]
  T W[MAX_Q];                  // weights[q]
};

// Kernel parameters of the cell-array integration kernels (ahead-of-time and
// run-time compiled): one __grid_constant__ struct, tabulation included.
template <typename T>
struct IntegrateArgs {
  const T* inv_j;
  const T* det_j;
  const T* coeffs;
  const T* aux;
  T* out;
  int64_t n_cells;
  int64_t n_chunks;     // chunks, round-robin over the CTAs
  int64_t chunk_cells;  // cells per chunk (a multiple of 16 or of N_bc)
  int n_bc;    // cells per batch
  int stages;  // ring depth
  int warps;   // consumer warps
  int bulk;    // 1: full batches arrive by bulk copy; 0: every batch read from global
  int dynamic;               // 1: cluster-launch-control scheduling (units below); 0: static chunks
  int resident;              // dynamic: CTAs 0..resident-1 own the round-robin share of the first
  int64_t static_batches;    //   static_batches batches; CTA resident + j owns batch static_batches + j
  int prefetch;              // batches per CTA warmed into L2 before the programmatic-launch wait
  unsigned long long* trace; // debug (txb_debug_trace): 4 %globaltimer stamps per CTA, NULL = off
  Tabulation<T> tab;
};

// Arguments of a mesh-fused kernel: the batch pipeline's (cells, batches,
// tables, aux, out) plus the mesh -- connectivity (streamed through the
// stage), vertex coordinates and the global coefficient vector (gathered).
template <typename T>
struct MeshLaunchArgs {
  IntegrateArgs<T> a;           // inv_j / det_j / coeffs unused
  const int64_t* cells;         // (n_cells, D+1)
  const double* vertices;       // (n_vertices, D)
  const T* coeffs_global;       // (n_vertices * n_comp), run precision
  unsigned long long* bad;      // lowered to the first cell with detJ <= 0 (NULL = no check)
};

// Arguments of a tiled mesh kernel (run-time compiled lane): the batch
// pipeline's (a batch = one tile of tile_cells cells), the per-tile distinct
// vertex records and local indices (txb_tile_build), vertex coordinates and the
// global coefficient vector (gathered once per tile by the gatherer warp).
template <typename T>
struct TiledLaunchArgs {
  IntegrateArgs<T> a;           // inv_j / det_j / coeffs unused
  const double* vertices;       // (n_vertices, D)
  const T* coeffs_global;       // (n_vertices * n_comp)
  unsigned long long* bad;      // lowered to the first cell with detJ <= 0 (NULL = no check)
  const int32_t* records;       // (n_tiles, vrec): [count, 0, 0, 0, ids...]
  const unsigned char* local;   // (n_tiles * tile, 4) uint8 | uint16
  int vrec;
  int lb;                       // local index bytes, 1 | 2
  int aux_bulk;                 // aux base 16-byte aligned
  int geom_bulk;                // given geometry (a.inv_j / a.det_j) bases 16-byte aligned
};

// 16- and 8-byte vector types per element type (type-preserving: the lanes of
// the vector ARE elements of the row, no conversion).
template <typename T> struct Vec16;
template <> struct Vec16<double> { using type = double2; static constexpr int N = 2; };
template <> struct Vec16<float> { using type = float4; static constexpr int N = 4; };
template <> struct Vec16<long> { using type = longlong2; static constexpr int N = 2; };
template <> struct Vec16<long long> { using type = longlong2; static constexpr int N = 2; };
template <> struct Vec16<int> { using type = int4; static constexpr int N = 4; };
template <typename T> struct Vec8;
template <> struct Vec8<float> { using type = float2; };
template <> struct Vec8<int> { using type = int2; };

// Vectorised row load: N consecutive T at p (row starts are multiples of
// N*sizeof(T) from a 16-byte aligned base); widest access the alignment allows.
template <typename T, int N, bool VEC = true>
__device__ __forceinline__ void load_row(const T* __restrict__ p, T (&r)[N]) {
  constexpr int BYTES = N * (int)sizeof(T);
  constexpr bool V16 = VEC && BYTES % 16 == 0;
  constexpr bool V8 = VEC && !V16 && sizeof(T) == 4 && BYTES % 8 == 0;
  if constexpr (V16) {
    using V = typename Vec16<T>::type;
    constexpr int E = 16 / (int)sizeof(T);
#pragma unroll
    for (int i = 0; i < N; i += E) {
      const V v = *reinterpret_cast<const V*>(p + i);
      r[i] = (T)v.x;
      r[i + 1] = (T)v.y;
      if constexpr (E == 4) {
        r[i + 2] = (T)v.z;
        r[i + 3] = (T)v.w;
      }
    }
  } else if constexpr (V8) {
    using V = typename Vec8<T>::type;
#pragma unroll
    for (int i = 0; i < N; i += 2) {
      const V v = *reinterpret_cast<const V*>(p + i);
      r[i] = (T)v.x;
      r[i + 1] = (T)v.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) r[i] = p[i];
  }
}

// Row load from a shared-memory stage where consecutive lanes read consecutive
// rows.  Rows of 32 or 96 bytes put the 8 lanes of a quarter warp on only the
// even 16-byte bank groups (a 2-way conflict on every LDS.128); lanes 4..7 of
// each quarter read the row's 16-byte chunks rotated by one -- the odd groups
// -- and rotate back in registers (3D elasticity f64: 47.0 -> 45.6 us).
template <typename T, int N, bool VEC = true>
__device__ __forceinline__ void load_row_rot(const T* __restrict__ p, T (&r)[N], int lane) {
  constexpr int BYTES = N * (int)sizeof(T);
  if constexpr (VEC && (BYTES == 32 || BYTES == 96)) {
    using V = typename Vec16<T>::type;
    constexpr int E = 16 / (int)sizeof(T), C = BYTES / 16;
    const bool rot = (lane >> 2) & 1;
    const V* row = reinterpret_cast<const V*>(p);
    V ch[C];
#pragma unroll
    for (int k = 0; k < C; ++k) ch[k] = row[rot ? (k == C - 1 ? 0 : k + 1) : k];
#pragma unroll
    for (int k = 0; k < C; ++k) {
      const V v = rot ? ch[k == 0 ? C - 1 : k - 1] : ch[k];
      r[k * E] = v.x;
      r[k * E + 1] = v.y;
      if constexpr (E == 4) {
        r[k * E + 2] = v.z;
        r[k * E + 3] = v.w;
      }
    }
  } else {
    load_row<T, N, VEC>(p, r);
  }
}

// ---------------------------------------------------------------------------
// The batch pipeline shared by every streaming kernel of the library.
//
// Args provides: n_cells, n_chunks, chunk_cells, n_bc, stages, warps,
// dynamic, resident, static_batches.  One producer lane (warp `warps`, lane 0)
// walks the batch sequence -- static contiguous chunks, or (dynamic) its own
// scheduling unit and then the units of the CTAs it cancels through cluster
// launch control -- and for each batch calls
//     issue(stage_ptr, c0, ncell, full_bar)  -> true if it posted expect_tx and
//                                              bulk copies, false if the batch
//                                              must be read from global memory
// Consumer warps wait on the stage's `full` barrier and call
//     consume(stage_ptr or nullptr, c0, ncell)
// then every consumer lane arrives on `empty`.  A count of 0 published in the
// stage info stops them.
// ---------------------------------------------------------------------------
struct PipelineSmem {
  uint64_t* full;
  uint64_t* empty;
  int64_t* info_c0;
  uint64_t* clc_bar;        // cluster-launch-control response barrier
  unsigned char* clc_resp;  // 16-byte response (16-byte aligned)
  int* info_n;
};

// mbarriers + stage info + the launch-control response, carved after `base`
// (16-byte aligned)
__device__ __forceinline__ PipelineSmem carve_pipeline(unsigned char* base) {
  PipelineSmem p;
  p.full = reinterpret_cast<uint64_t*>(base);
  p.empty = p.full + MAX_STAGES;
  p.info_c0 = reinterpret_cast<int64_t*>(p.empty + MAX_STAGES);
  p.clc_bar = reinterpret_cast<uint64_t*>(p.info_c0 + MAX_STAGES);
  p.clc_resp = reinterpret_cast<unsigned char*>(p.clc_bar + 2);
  p.info_n = reinterpret_cast<int*>(p.clc_resp + 16);
  return p;
}
constexpr int PIPELINE_SMEM_BYTES = 8 * (3 * MAX_STAGES) + 16 + 16 + 4 * MAX_STAGES;

template <class Args>
__device__ __forceinline__ void pipeline_init(const Args& a, const PipelineSmem& p) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(&p.full[s], 1);
      mbar_init(&p.empty[s], a.warps * EMPTY_ARRIVALS_PER_WARP);
    }
    mbar_init(p.clc_bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
}

// First cells of this CTA's first `count` batches (for L2 prefetch before the
// programmatic-launch wait): calls f(c0, ncell) for each.
// Dynamic mode, the batches of scheduling unit u (a CTA index of the grid):
// u < resident: batches u, u + resident, ... below static_batches (dealt
// round-robin, so the whole grid sweeps the arrays together); u >= resident:
// the single batch static_batches + (u - resident).  f(c0, ncell) per batch
// until f returns false.
template <class Args, class F>
__device__ __forceinline__ void unit_batches(const Args& a, int64_t u, F f) {
  const int nbc = a.n_bc;
  if (u < a.resident) {
    for (int64_t b = u; b < a.static_batches; b += a.resident) {
      const int64_t c0 = b * nbc;
      if (!f(c0, (int)min((int64_t)nbc, a.n_cells - c0))) return;
    }
  } else {
    const int64_t c0 = (a.static_batches + (u - a.resident)) * nbc;
    if (c0 < a.n_cells) f(c0, (int)min((int64_t)nbc, a.n_cells - c0));
  }
}

template <class Args, class F>
__device__ __forceinline__ void pipeline_first_batches(const Args& a, int count, F f) {
  if (a.dynamic) {
    unit_batches(a, blockIdx.x, [&](int64_t c0, int ncell) {
      f(c0, ncell);
      return --count > 0;
    });
  } else if ((int64_t)blockIdx.x < a.n_chunks) {
    const int nbc = a.n_bc;
    const int64_t lo = (int64_t)blockIdx.x * a.chunk_cells;
    const int64_t hi = min(a.n_cells, lo + a.chunk_cells);
    for (int64_t c0 = lo; count > 0 && c0 < hi; c0 += nbc, --count) f(c0, (int)min((int64_t)nbc, hi - c0));
  }
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Debug timeline (txb_debug_trace): per CTA [entry, after the grid-dependency
// wait, first batch ready in consumer warp 0, consumer warp 0 done].
__device__ __forceinline__ void trace_stamp(unsigned long long* trace, int k) {
  if (trace) trace[blockIdx.x * 4 + k] = global_ns();
}

// Programmatic dependent launch: everything before this overlapped the
// previous grid in the stream (barrier setup and L2 prefetches, which return
// no data and so cannot observe a value the previous grid is still writing);
// from here on we read and write global memory, so wait for it (a no-op when
// launched without the PDL attribute), then let the next grid start its own
// prologue as our CTAs retire.
__device__ __forceinline__ void pipeline_wait_prior_grid() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <class Args, class Issue>
__device__ __forceinline__ void pipeline_produce(const Args& a, const PipelineSmem& p, unsigned char* stages,
                                                 int stage_bytes, Issue issue) {
  const int nbc = a.n_bc;
  int stage = 0;
  uint32_t phase = 0;
  auto publish = [&](int64_t c0, int ncell) {
    mbar_wait(&p.empty[stage], phase ^ 1);
    p.info_c0[stage] = c0;
    p.info_n[stage] = ncell;  // 0 = stop
    if (ncell == 0 || !issue(stages + stage * stage_bytes, c0, ncell, &p.full[stage])) {
      if (ncell) p.info_n[stage] = -ncell;  // consumers read this batch from global memory
      mbar_arrive(&p.full[stage]);
    }
    if (++stage == a.stages) {
      stage = 0;
      phase ^= 1;
    }
  };
  if (a.dynamic) {
    // Cluster launch control: run this CTA's own unit, then keep cancelling
    // CTAs of the grid that have not launched yet and run their units, until
    // none is left.  One request is always in flight ahead of the unit being
    // published, hiding its latency; none is issued after a failed one.
    clc_try_cancel(p.clc_resp, p.clc_bar);
    uint32_t clc_phase = 0;
    unit_batches(a, blockIdx.x, [&](int64_t c0, int ncell) {
      publish(c0, ncell);
      return true;
    });
    for (;;) {
      mbar_wait(p.clc_bar, clc_phase);
      clc_phase ^= 1;
      const int64_t u = clc_cancelled_cta(p.clc_resp);
      if (u < 0) break;
      clc_try_cancel(p.clc_resp, p.clc_bar);
      unit_batches(a, u, [&](int64_t c0, int ncell) {
        publish(c0, ncell);
        return true;
      });
    }
  } else {
    // static: contiguous chunks, round-robin over the CTAs
    for (int64_t ci = blockIdx.x; ci < a.n_chunks; ci += gridDim.x) {
      const int64_t lo = ci * a.chunk_cells;
      const int64_t hi = min(a.n_cells, lo + a.chunk_cells);
      for (int64_t c0 = lo; c0 < hi; c0 += nbc) publish(c0, (int)min((int64_t)nbc, hi - c0));
    }
  }
  publish(0, 0);  // stop
}

template <class Args, class Consume>
__device__ __forceinline__ void pipeline_consume(const Args& a, const PipelineSmem& p, unsigned char* stages,
                                                 int stage_bytes, Consume consume) {
  const int lane = threadIdx.x & 31;
  int stage = 0;
  uint32_t phase = 0;
  for (;;) {
    mbar_wait(&p.full[stage], phase);
    const int64_t c0 = p.info_c0[stage];
    const int nsig = p.info_n[stage];
    if (nsig == 0) break;
    if (nsig > 0)
      consume(stages + stage * stage_bytes, c0, nsig);
    else
      consume(nullptr, c0, -nsig);
#if TXB_EMPTY_ARRIVE_ALL
    mbar_arrive(&p.empty[stage]);  // every lane releases its own reads of the stage
#else
    __syncwarp();  // orders the other lanes' reads of the stage before lane 0's release
    if (lane == 0) mbar_arrive(&p.empty[stage]);
#endif
    if (++stage == a.stages) {
      stage = 0;
      phase ^= 1;
    }
  }
  (void)lane;
}

}  // namespace txb
