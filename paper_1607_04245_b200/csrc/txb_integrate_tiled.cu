// txb_integrate_tiled.cu — the mesh-fused integration (geometry + gather in
// kernel) over CELL TILES with batch-local vertex
// tables.
//
// Why: the per-cell fused kernel (txb_integrate_mesh.cu) gathers every cell's
// N_b vertex rows (D float64 coordinates + N_comp coefficients each) with
// per-lane 8-byte loads through the connectivity.  A P1 vertex is shared by
// ~24 tetrahedra, so consecutive cells mostly re-gather the same rows; the
// kernel is bound by the L1 data pipe on those scattered loads (~4.3 global
// wavefronts per cell, profiles/r1_pipeline.md r1zw), not by HBM.
//
// Here a mesh is cut once into tiles of TILE consecutive cells (one batch of
// the pipeline each) and every tile carries
//   record[t] = [count, 0, 0, 0, v_0 .. v_{count-1}]   int32, its distinct
//               vertex ids ascending (fixed stride vrec per tile)
//   local[t]  = per cell 4 local indices into that list (uint8 when every tile
//               has <= 256 distinct vertices, else uint16; 2D pads the 4th)
// built on the device by txb_tile_counts / txb_tile_build (a block-wide bitonic
// sort per tile) and cached with the mesh.  On a Kuhn mesh a 128-cell 3D tile
// has ~91 distinct vertices (0.71 per cell instead of 4 references), and the
// local connectivity is 4 B/cell instead of 32 B of int64.
//
// Per batch, three warp roles (mbarrier-synchronised, no CTA barrier):
//   producer  (1 lane)  bulk-copies the tile's record, local indices and aux
//                       slice into a ring stage (cp.async.bulk, `full`);
//   gatherer  (1 warp)  after `full`, copies each distinct vertex's D
//                       coordinates and N_comp coefficients ONCE into the
//                       stage's structure-of-arrays table with cp.async
//                       (LDGSTS), completion tracked on `ready` (noinc arrive);
//   consumers (W warps) after `ready`, lane <-> (cell, q): coordinates and
//                       coefficients from the shared table through the local
//                       indices, float64 geometry (mesh.py:150-190 expression
//                       order, cast once), quadrature phase, then the basis
//                       phase: thread-transposed through the warp exchange
//                       area (lane <-> element entry, N_q > 1) or, for the
//                       midpoint rule, in-lane (lane <-> cell owns its whole
//                       element vector and stores it with vector stores; the
//                       same chains in the same order);
//                       release the stage on `empty`.
// Every chain rounds as the reference's (bit-identical to compute_geometry ->
// gather -> cast -> integrate_cells, like txb_integrate_mesh).
#include "txb_kernels.cuh"

namespace txb {

// ---------------------------------------------------------------------------
// Tile builder: one CTA per tile, P = next_pow2(TILE * NB) threads, one
// (vertex id, position) key each; bitonic sort in shared memory; the first
// occurrence of each id gets the next local index (block scan).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int block_inclusive_scan(int v, int* warp_tot) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  if (lane == 31) warp_tot[w] = v;
  __syncthreads();
  if (w == 0) {
    int t = lane < nw ? warp_tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < nw) warp_tot[lane] = t;
  }
  __syncthreads();
  return v + (w > 0 ? warp_tot[w - 1] : 0);
}

template <int NB>
__global__ void __launch_bounds__(1024) tile_build_kernel(const int64_t* __restrict__ cells, int64_t n_cells,
                                                          int tile, int vrec, int lb, int32_t* __restrict__ counts,
                                                          int32_t* __restrict__ records, unsigned char* __restrict__ local) {
  extern __shared__ unsigned long long keys[];  // blockDim.x keys
  __shared__ int warp_tot[32];
  const int P = blockDim.x, i = threadIdx.x;
  const int64_t t = blockIdx.x;
  const int64_t c0 = t * tile;
  const int ncell = (int)min((int64_t)tile, n_cells - c0);
  const int nent = ncell * NB;
  constexpr unsigned long long NONE = ~0ull;
  const long long id = i < nent ? (long long)cells[c0 * NB + i] : 0;
  keys[i] = i < nent ? ((unsigned long long)id << 11) | (unsigned long long)i : NONE;
  // vertex ids must lie in [0, 2^31): report a tile holding any other id with count -1
  if (__syncthreads_or(id < 0 || id >= (1LL << 31))) {
    if (i == 0 && counts) counts[t] = -1;
    return;
  }
  for (int k = 2; k <= P; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      const int x = i ^ j;
      if (x > i) {
        const unsigned long long a = keys[i], b = keys[x];
        if ((a > b) == ((i & k) == 0)) {
          keys[i] = b;
          keys[x] = a;
        }
      }
      __syncthreads();
    }
  const unsigned long long key = keys[i];
  const bool valid = key != NONE;
  const long long vid = (long long)(key >> 11);
  const bool first = valid && (i == 0 || (long long)(keys[i - 1] >> 11) != vid);
  const int incl = block_inclusive_scan(first ? 1 : 0, warp_tot);
  const int count = warp_tot[(P >> 5) - 1];
  if (!records) {
    if (i == 0) counts[t] = count;
    return;
  }
  int32_t* rec = records + t * vrec;
  if (i < 4) rec[i] = i == 0 ? count : 0;
  if (valid) {
    const int idx = incl - 1;
    if (first) rec[4 + idx] = (int32_t)vid;
    const int pos = (int)(key & 2047u);
    const int64_t slot = (c0 + pos / NB) * 4 + pos % NB;
    if (lb == 1)
      local[slot] = (unsigned char)idx;
    else
      reinterpret_cast<uint16_t*>(local)[slot] = (uint16_t)idx;
  }
}

static int tile_launch(int dim, int64_t n_cells, const int64_t* cells, int tile, int vrec, int lb, int32_t* counts,
                       int32_t* records, void* local, cudaStream_t s) {
  const int nb = dim + 1;
  if (dim < 2 || dim > 3 || n_cells < 0 || tile < 1 || tile * nb > 1024) {
    set_error("tiles: dim must be 2 or 3 and tile_cells * (dim + 1) <= 1024 (got dim %d, tile %d)", dim, tile);
    return TXB_E_SHAPE;
  }
  const int64_t n_tiles = (n_cells + tile - 1) / tile;
  if (n_tiles == 0) return TXB_OK;
  if (!cells || (!records && !counts) || (records && !local)) {
    set_error("tiles: NULL device pointer");
    return TXB_E_ARG;
  }
  int P = 32;
  while (P < tile * nb) P <<= 1;
  const size_t sm = (size_t)P * sizeof(unsigned long long);
  if (nb == 3)
    tile_build_kernel<3><<<(unsigned)n_tiles, P, sm, s>>>(cells, n_cells, tile, vrec, lb, counts, records,
                                                          (unsigned char*)local);
  else
    tile_build_kernel<4><<<(unsigned)n_tiles, P, sm, s>>>(cells, n_cells, tile, vrec, lb, counts, records,
                                                          (unsigned char*)local);
  TXB_CUDA_TRY(cudaGetLastError());
  return TXB_OK;
}

// ---------------------------------------------------------------------------
// The tiled integration kernel
// ---------------------------------------------------------------------------
template <typename T>
struct TiledArgs {
  // batch pipeline (txb_pipeline.cuh): a batch is one tile
  int64_t n_cells;
  int64_t n_chunks;
  int64_t chunk_cells;  // a multiple of the tile
  int n_bc;             // = tile
  int stages;
  int warps;
  int dynamic;
  int resident;
  int64_t static_batches;
  int prefetch;
  // mesh
  const double* vertices;      // (n_vertices, D) float64
  const int32_t* records;      // (n_tiles, vrec)
  const unsigned char* local;  // (n_tiles * tile, 4) uint8 | uint16
  const T* coeffs_global;      // (n_vertices * NCOMP)
  const T* aux;                // (n, 1) P0 | (n, D+1, 1) P1 | NULL
  const T* inv_j;              // GEOM == 1: the caller's geometry (n, D, D) and (n), run precision
  const T* det_j;
  T* out;                      // (n, D+1, NCOMP)
  unsigned long long* bad;     // lowered to the first cell with detJ <= 0 (NULL = no check)
  int vrec;                    // int32 per tile record (multiple of 4): 4 + the largest count, rounded
  int aux_bulk;                // aux base 16-byte aligned: full batches' aux slices arrive by bulk copy
  int geom_bulk;               // GEOM == 1: inv_j / det_j bases 16-byte aligned (bulk copies, else global loads)
  int out_vec;                 // out base 16-byte aligned: in-lane rows stored with vector stores
  uint32_t consumer_sleep_ns;  // consumer `ready` try_wait suspend hint (0: plain retry)
  Tabulation<T> tab;
};

// Stage: [local indices][aux][GEOM: inv_j | det_j][record][coordinates (GEOM 0)][coefficient components]
template <typename T, int D, int NCOMP, int AUX, int LB, int GEOM>
struct TiledStage {
  static constexpr int NB = D + 1;
  static constexpr int AUXW = AUX == 1 ? 1 : (AUX == 2 ? NB : 0);
  __host__ __device__ static int local_bytes(int n) { return round_up(n * 4 * LB, 16); }
  __host__ __device__ static int aux_bytes(int n) { return round_up(n * AUXW * (int)sizeof(T), 16); }
  __host__ __device__ static int inv_bytes(int n) { return GEOM ? round_up(n * D * D * (int)sizeof(T), 16) : 0; }
  __host__ __device__ static int det_bytes(int n) { return GEOM ? round_up(n * (int)sizeof(T), 16) : 0; }
  __host__ __device__ static int rec_bytes(int vrec) { return vrec * 4; }
  __host__ __device__ static int xyz_bytes(int vrec) { return GEOM ? 0 : D * round_up(vrec * 8, 16); }
  __host__ __device__ static int u_pitch(int vrec) { return round_up(vrec * (int)sizeof(T), 16) / (int)sizeof(T); }
  __host__ __device__ static int u_bytes(int vrec) { return NCOMP * u_pitch(vrec) * (int)sizeof(T); }
  __host__ __device__ static int aux_off(int n) { return local_bytes(n); }
  __host__ __device__ static int inv_off(int n) { return local_bytes(n) + aux_bytes(n); }
  __host__ __device__ static int det_off(int n) { return inv_off(n) + inv_bytes(n); }
  __host__ __device__ static int rec_off(int n) { return det_off(n) + det_bytes(n); }
  __host__ __device__ static int xyz_off(int n, int vrec) { return rec_off(n) + rec_bytes(vrec); }
  __host__ __device__ static int u_off(int n, int vrec) { return xyz_off(n, vrec) + xyz_bytes(vrec); }
  __host__ __device__ static int stage_bytes(int n, int vrec) { return u_off(n, vrec) + u_bytes(vrec); }
};

template <typename T, int N>
__device__ __forceinline__ void store_row(T* __restrict__ p, const T (&r)[N], bool vec) {
  constexpr int BYTES = N * (int)sizeof(T);
  if constexpr (BYTES % 16 == 0) {
    if (vec) {
      using V = typename Vec16<T>::type;
      constexpr int E = 16 / (int)sizeof(T);
#pragma unroll
      for (int i = 0; i < N; i += E) {
        V v;
        if constexpr (E == 2) {
          v.x = r[i];
          v.y = r[i + 1];
        } else {
          v.x = r[i];
          v.y = r[i + 1];
          v.z = r[i + 2];
          v.w = r[i + 3];
        }
        *reinterpret_cast<V*>(p + i) = v;
      }
      return;
    }
  } else if constexpr (sizeof(T) == 4 && BYTES % 8 == 0) {
    if (vec) {
#pragma unroll
      for (int i = 0; i < N; i += 2) *reinterpret_cast<float2*>(p + i) = make_float2(r[i], r[i + 1]);
      return;
    }
  }
#pragma unroll
  for (int i = 0; i < N; ++i) p[i] = r[i];
}

// One warp slice of CW cells: c0 = batch-local first cell.
template <typename T, int D, int NQ, int NCOMP, int FORM, int AUX, int LB, bool XP, int GEOM>
__device__ __forceinline__ void tiled_slice(const TiledArgs<T>& a, const unsigned char* __restrict__ s_local,
                                            const T* __restrict__ aux_src, const double* __restrict__ sx,
                                            const T* __restrict__ su, const T* __restrict__ g_inv,
                                            const T* __restrict__ g_det, int vpitch, int upitch,
                                            unsigned char* __restrict__ scratch, int64_t c0_batch, int c0,
                                            int ncell, int lane) {
  constexpr int NB = D + 1, DD = D * D, NBC = NB * NCOMP;
  constexpr int AUXW = AUX == 1 ? 1 : (AUX == 2 ? NB : 0);
  using S = MeshScratch<T, D, NQ, NCOMP>;
  constexpr int CW = 32 / NQ;
  const int nc = min(CW, ncell - c0);
  T* s_tr = reinterpret_cast<T*>(scratch);
  T* s_f1 = reinterpret_cast<T*>(scratch + S::TR_BYTES);

  const int lc = NQ == 1 ? lane : lane / NQ;
  const int q = NQ == 1 ? 0 : lane - lc * NQ;
  if (lc < nc) {
    const int cell = c0 + lc;
    int ids[NB];
    if constexpr (LB == 1) {
      const uint32_t w = reinterpret_cast<const uint32_t*>(s_local)[cell];
#pragma unroll
      for (int b = 0; b < NB; ++b) ids[b] = (w >> (8 * b)) & 0xffu;
    } else {
      const uint2 w = reinterpret_cast<const uint2*>(s_local)[cell];
#pragma unroll
      for (int b = 0; b < NB; ++b) ids[b] = ((b < 2 ? w.x : w.y) >> (16 * (b & 1))) & 0xffffu;
    }
    // gather (mesh.py:202-217) from the tile's table
    T cf[NBC];
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
      for (int c = 0; c < NCOMP; ++c) cf[b * NCOMP + c] = su[c * upitch + ids[b]];
    T J[DD];
    T det;
    if constexpr (GEOM) {
      // the caller's geometry in the run precision (stage or global)
#pragma unroll
      for (int i = 0; i < DD; ++i) J[i] = g_inv[cell * DD + i];
      det = g_det[cell];
      (void)sx;
      (void)vpitch;
    } else {
      double X[NB][D];
#pragma unroll
      for (int b = 0; b < NB; ++b)
#pragma unroll
        for (int i = 0; i < D; ++i) X[b][i] = sx[i * vpitch + ids[b]];
      double detd;
      cell_geometry<T, D>(X, J, det, detd);
      if (q == 0 && a.bad && detd <= 0.0) atomicMin(a.bad, (unsigned long long)(c0_batch + cell));
    }

    // standard P1 pull-back (exactness note in txb_kernels.cuh)
    T tr[NB][D];
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
      a0 = aux_src[cell];
    } else if constexpr (AUX == 2) {
      const T* Bq = a.tab.B + q * NB;
      a0 = mul(aux_src[cell * AUXW], Bq[0]);
#pragma unroll
      for (int bb = 1; bb < NB; ++bb) a0 = add(a0, mul(aux_src[cell * AUXW + bb], Bq[bb]));
    }
    (void)a0;
    const T wq = a.tab.W[q];
    T f1s[NCOMP][D];
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
        f1s[c][k] = mul(mul(fv, det), wq);
      }

    if constexpr (!XP) {
      // in-lane basis phase (N_q = 1): e[b][c] = sum_k T[b][k] f1s[c][k], +0-started chain
      T e[NBC];
#pragma unroll
      for (int b = 0; b < NB; ++b)
#pragma unroll
        for (int c = 0; c < NCOMP; ++c) {
          T acc = T(0);
#pragma unroll
          for (int k = 0; k < D; ++k) acc = add(acc, mul(tr[b][k], f1s[c][k]));
          e[b * NCOMP + c] = acc;
        }
      store_row<T, NBC>(a.out + (c0_batch + cell) * NBC, e, a.out_vec);
      return;
    } else {
      if (q == 0) {
#pragma unroll
        for (int i = 0; i < DD; ++i) s_tr[S::tr(lc, i)] = J[i];
#pragma unroll
        for (int k = 0; k < D; ++k) s_tr[S::tr(lc, DD + k)] = tr[0][k];
      }
#pragma unroll
      for (int c = 0; c < NCOMP; ++c)
#pragma unroll
        for (int k = 0; k < D; ++k) s_f1[S::f1(lc, (q * NCOMP + c) * D + k)] = f1s[c][k];
    }
  }
  if constexpr (XP) {
    __syncwarp();  // ==== transpose threads (warp scope) ====
    T* o_base = a.out + (c0_batch + c0) * NBC;
    auto entry = [&](int o) {
      const int lc2 = o / NBC;
      const int r = o - lc2 * NBC;
      const int b = r / NCOMP;
      const int c = r - b * NCOMP;
      T f1[NQ * D];
#pragma unroll
      for (int qq = 0; qq < NQ; ++qq)
#pragma unroll
        for (int k = 0; k < D; ++k) f1[qq * D + k] = s_f1[S::f1(lc2, (qq * NCOMP + c) * D + k)];
      const int r0 = b == 0 ? DD : (b - 1) * D;
      T t[D];
#pragma unroll
      for (int k = 0; k < D; ++k) t[k] = s_tr[S::tr(lc2, r0 + k)];
      T e = T(0);
#pragma unroll
      for (int qq = 0; qq < NQ; ++qq)
#pragma unroll
        for (int k = 0; k < D; ++k) e = add(e, mul(t[k], f1[qq * D + k]));
      o_base[o] = e;
    };
    constexpr int FULL = CW * NBC;
    if (nc == CW && FULL % 32 == 0) {
#pragma unroll
      for (int s = 0; s < FULL / 32; ++s) entry(s * 32 + lane);
    } else {
      for (int o = lane; o < nc * NBC; o += 32) entry(o);
    }
    __syncwarp();
  }
}

constexpr int TILED_MAX_CONSUMER_WARPS = 6;
constexpr int TILED_MAX_THREADS = 32 * (TILED_MAX_CONSUMER_WARPS + 2);
// Register budget: the consumers are latency-bound on the float64 geometry
// chains, so CTAs per SM (warps in flight) matter more than a few spilled
// registers -- 3 CTAs of <= 256 threads (<= 80 registers) for scalar forms.
#ifndef TXB_TILED_MIN_BLOCKS
#define TXB_TILED_MIN_BLOCKS(NCOMP) ((NCOMP) == 1 ? 3 : 2)
#endif

template <typename T, int D, int NQ, int NCOMP, int FORM, int AUX, int LB, bool XP, int GEOM>
__global__ void __launch_bounds__(TILED_MAX_THREADS, TXB_TILED_MIN_BLOCKS(NCOMP))
integrate_tiled_kernel(const __grid_constant__ TiledArgs<T> a) {
  using L = TiledStage<T, D, NCOMP, AUX, LB, GEOM>;
  using S = MeshScratch<T, D, NQ, NCOMP>;
  constexpr int NB = D + 1;
  constexpr int SCR = XP ? S::BYTES : 0;
  constexpr int CW = 32 / NQ;

  extern __shared__ __align__(128) unsigned char smem[];
  const int nbc = a.n_bc, vrec = a.vrec;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int W = a.warps;
  const int stage_bytes = L::stage_bytes(nbc, vrec);
  unsigned char* scratch_base = smem + a.stages * stage_bytes;
  const PipelineSmem p = carve_pipeline(scratch_base + W * SCR);
  uint64_t* ready = reinterpret_cast<uint64_t*>(scratch_base + W * SCR + PIPELINE_SMEM_BYTES);
  if (threadIdx.x == 0)
    for (int s = 0; s < a.stages; ++s) mbar_init(&ready[s], 32);
  pipeline_init(a, p);  // (its fence + __syncthreads also publish `ready`)

  const int vpitch = L::xyz_bytes(vrec) / D / 8;
  const int upitch = L::u_pitch(vrec);
  if (warp == W && lane == 0) {
    pipeline_first_batches(a, a.prefetch, [&](int64_t c0, int ncell) {
      bulk_prefetch_l2(a.local + c0 * 4 * LB, (uint32_t)L::local_bytes(nbc));
      bulk_prefetch_l2(a.records + (c0 / nbc) * vrec, (uint32_t)L::rec_bytes(vrec));
    });
  }
  pipeline_wait_prior_grid();

  if (warp == W) {
    // ============================ producer lane ============================
    if (lane != 0) return;
    const uint64_t policy = l2_evict_first_policy();
    pipeline_produce(a, p, smem, stage_bytes, [&](unsigned char* st, int64_t c0, int ncell, uint64_t* bar) {
      const uint32_t lbytes = L::local_bytes(nbc), rb = L::rec_bytes(vrec);
      const uint32_t ab = ncell * L::AUXW * (uint32_t)sizeof(T);
      const bool auxb = AUX != 0 && a.aux_bulk && (ab & 15u) == 0;
      const uint32_t ib = GEOM ? ncell * D * D * (uint32_t)sizeof(T) : 0, db = GEOM ? ncell * (uint32_t)sizeof(T) : 0;
      const bool geob = GEOM && a.geom_bulk && ((ib | db) & 15u) == 0;
      mbar_arrive_expect_tx(bar, lbytes + rb + (auxb ? ab : 0) + (geob ? ib + db : 0));
      bulk_g2s(st, a.local + c0 * 4 * LB, lbytes, bar, policy);
      if (auxb) bulk_g2s(st + L::aux_off(nbc), a.aux + c0 * L::AUXW, ab, bar, policy);
      if (geob) {
        bulk_g2s(st + L::inv_off(nbc), a.inv_j + c0 * D * D, ib, bar, policy);
        bulk_g2s(st + L::det_off(nbc), a.det_j + c0, db, bar, policy);
      }
      bulk_g2s(st + L::rec_off(nbc), a.records + (c0 / nbc) * vrec, rb, bar, policy);
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
        const int32_t* rec = reinterpret_cast<const int32_t*>(st + L::rec_off(nbc));
        const int cnt = rec[0];
        double* sx = reinterpret_cast<double*>(st + L::xyz_off(nbc, vrec));
        T* su = reinterpret_cast<T*>(st + L::u_off(nbc, vrec));
        for (int j = lane; j < cnt; j += 32) {
          const int64_t v = rec[4 + j];
          if constexpr (!GEOM) {
#pragma unroll
            for (int i = 0; i < D; ++i) cp_async<8>(sx + i * vpitch + j, a.vertices + v * D + i);
          }
#pragma unroll
          for (int c = 0; c < NCOMP; ++c)
            cp_async<(int)sizeof(T)>(su + c * upitch + j, a.coeffs_global + v * NCOMP + c);
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
  unsigned char* scratch = scratch_base + warp * SCR;
  int stage = 0;
  uint32_t phase = 0;
  for (;;) {
    if (a.consumer_sleep_ns)
      mbar_wait_sleep(&ready[stage], phase, a.consumer_sleep_ns);
    else
      mbar_wait(&ready[stage], phase);
    mbar_wait(&p.full[stage], phase);  // (complete: the bulk-copied bytes are visible to this thread too)
    const int64_t c0 = p.info_c0[stage];
    const int ncell = p.info_n[stage];
    if (ncell == 0) break;
    const unsigned char* st = smem + stage * stage_bytes;
    const T* aux_src = nullptr;
    if constexpr (AUX != 0) {
      const uint32_t ab = ncell * L::AUXW * (uint32_t)sizeof(T);
      aux_src = (a.aux_bulk && (ab & 15u) == 0) ? reinterpret_cast<const T*>(st + L::aux_off(nbc))
                                                : a.aux + c0 * L::AUXW;
    }
    const double* sx = reinterpret_cast<const double*>(st + L::xyz_off(nbc, vrec));
    const T* su = reinterpret_cast<const T*>(st + L::u_off(nbc, vrec));
    const T* g_inv = nullptr;
    const T* g_det = nullptr;
    if constexpr (GEOM) {
      const uint32_t ib = ncell * D * D * (uint32_t)sizeof(T), db = ncell * (uint32_t)sizeof(T);
      const bool geob = a.geom_bulk && ((ib | db) & 15u) == 0;
      g_inv = geob ? reinterpret_cast<const T*>(st + L::inv_off(nbc)) : a.inv_j + c0 * D * D;
      g_det = geob ? reinterpret_cast<const T*>(st + L::det_off(nbc)) : a.det_j + c0;
    }
    for (int c = warp * CW; c < ncell; c += W * CW)
      tiled_slice<T, D, NQ, NCOMP, FORM, AUX, LB, XP, GEOM>(a, st, aux_src, sx, su, g_inv, g_det, vpitch, upitch,
                                                            scratch, c0, c, ncell, lane);
    mbar_arrive(&p.empty[stage]);
    if (++stage == a.stages) {
      stage = 0;
      phase ^= 1;
    }
  }
  (void)NB;
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
template <typename T, int D, int NQ, int NCOMP, int FORM, int AUX, int LB, bool XP, int GEOM>
struct TiledKernel {
  using L = TiledStage<T, D, NCOMP, AUX, LB, GEOM>;
  static void* fn() { return (void*)integrate_tiled_kernel<T, D, NQ, NCOMP, FORM, AUX, LB, XP, GEOM>; }
  static int stage_bytes(int n_bc) {
    return L::local_bytes(n_bc) + L::aux_bytes(n_bc) + L::inv_bytes(n_bc) + L::det_bytes(n_bc);
  }
  static int scratch(int) { return XP ? MeshScratch<T, D, NQ, NCOMP>::BYTES : 0; }
  static int vrec_bytes(int vrec) { return L::rec_bytes(vrec) + L::xyz_bytes(vrec) + L::u_bytes(vrec); }
};

// In-lane basis phase for the midpoint rule (TXB_TILED_XPOSE=1 forces the
// exchange-area transposition there too, for measurement).
template <typename T, int D, int NQ, int LB, int GEOM>
static bool pick_tiled_form(const Config& c, int vrec, bool xpose, KernelInfo& k) {
#define TXB_TK(NCOMP, FORM, AUX, XP)                                        \
  {                                                                         \
    using K = TiledKernel<T, D, NQ, NCOMP, FORM, AUX, LB, XP, GEOM>;        \
    k = {K::fn(), K::stage_bytes, K::scratch, 32 / NQ};                     \
    k.family = FAMILY_MESH;                                                 \
    k.stage_extra = K::vrec_bytes(vrec);                                    \
    k.extra_warps = 1;                                                      \
    k.fixed_extra = 8 * MAX_STAGES;                                         \
    k.prefer_dynamic = 1;                                                   \
    k.max_stages = env_int("TXB_TILED_MAX_STAGES", 8);                      \
    k.max_warps = TILED_MAX_CONSUMER_WARPS;                                 \
    return true;                                                            \
  }
#define TXB_TK2(NCOMP, FORM, AUX)                                           \
  {                                                                         \
    if (NQ > 1 || xpose) TXB_TK(NCOMP, FORM, AUX, true) else TXB_TK(NCOMP, FORM, AUX, false) \
  }
  if (c.form == 0) TXB_TK2(1, 0, 0)
  if (c.form == 1 && c.aux == 1) TXB_TK2(1, 1, 1)
  if (c.form == 1 && c.aux == 2) TXB_TK2(1, 1, 2)
  if (c.form == 2) TXB_TK2(D, 2, 0)
#undef TXB_TK2
#undef TXB_TK
  return false;
}

template <typename T, int D, int GEOM>
static bool pick_tiled_nq(const Config& c, int lb, int vrec, bool xpose, KernelInfo& k) {
  if (c.n_q == 1) return lb == 1 ? pick_tiled_form<T, D, 1, 1, GEOM>(c, vrec, xpose, k)
                                 : pick_tiled_form<T, D, 1, 2, GEOM>(c, vrec, xpose, k);
  if (c.n_q == 2) return lb == 1 ? pick_tiled_form<T, D, 2, 1, GEOM>(c, vrec, true, k)
                                 : pick_tiled_form<T, D, 2, 2, GEOM>(c, vrec, true, k);
  return false;
}

template <int GEOM>
static bool pick_tiled_geom(const Config& c, int lb, int vrec, bool xpose, KernelInfo& k) {
  if (c.dtype == 4)
    return c.dim == 2 ? pick_tiled_nq<float, 2, GEOM>(c, lb, vrec, xpose, k)
                      : pick_tiled_nq<float, 3, GEOM>(c, lb, vrec, xpose, k);
  return c.dim == 2 ? pick_tiled_nq<double, 2, GEOM>(c, lb, vrec, xpose, k)
                    : pick_tiled_nq<double, 3, GEOM>(c, lb, vrec, xpose, k);
}

static bool pick_tiled_kernel(const Config& c, int lb, int vrec, bool geom, KernelInfo& k) {
  const bool xpose = env_int("TXB_TILED_XPOSE", 0) != 0;
  return geom ? pick_tiled_geom<1>(c, lb, vrec, xpose, k) : pick_tiled_geom<0>(c, lb, vrec, xpose, k);
}

template <typename T>
static int launch_tiled(const Config& c, const KernelInfo& k, Geometry g, int64_t n_cells, const void* basis,
                        const void* basis_der, const void* weights, const double* vertices, const int32_t* records,
                        const void* local, int vrec, const void* coeffs_global, const void* inv_j,
                        const void* det_j, const void* aux, void* out, int64_t* bad_cell, cudaStream_t stream) {
  TiledArgs<T> a;
  a.n_cells = n_cells;
  // static chunks must start on tile boundaries
  g.chunk_cells = (g.chunk_cells + g.n_bc - 1) / g.n_bc * g.n_bc;
  g.n_chunks = (n_cells + g.chunk_cells - 1) / g.chunk_cells;
  if (!g.dynamic) g.grid = (int)std::max<int64_t>(1, std::min<int64_t>(g.n_chunks, g.grid));
  a.n_chunks = g.n_chunks;
  a.chunk_cells = g.chunk_cells;
  a.n_bc = g.n_bc;
  a.stages = g.stages;
  a.warps = g.warps;
  a.dynamic = g.dynamic;
  a.resident = g.resident;
  a.static_batches = g.static_batches;
  a.prefetch = prefetch_batches(g);
  a.vertices = vertices;
  a.records = records;
  a.local = (const unsigned char*)local;
  a.coeffs_global = (const T*)coeffs_global;
  a.aux = (const T*)aux;
  a.out = (T*)out;
  a.bad = (unsigned long long*)bad_cell;
  a.vrec = vrec;
  auto al16 = [](const void* p) { return ((uintptr_t)p & 15u) == 0; };
  a.aux_bulk = c.aux != 0 && al16(aux) && env_int("TXB_DISABLE_BULK", 0) == 0;
  a.inv_j = (const T*)inv_j;
  a.det_j = (const T*)det_j;
  a.geom_bulk = inv_j && al16(inv_j) && al16(det_j) && env_int("TXB_DISABLE_BULK", 0) == 0;
  a.out_vec = al16(out);
  a.consumer_sleep_ns = (uint32_t)std::max(0, env_int("TXB_TILED_CONSUMER_SLEEP_NS", 20000));  // measured +2 %
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

// Test hook: the fused kernels' branch-free geometry (affine_inverse_fast) per
// cell, with its range predicate, for a direct comparison with numpy's
// correctly rounded quotients (tests/test_gpu_tiled.py).
template <int D>
__global__ void geometry_fast_kernel(const double* __restrict__ vertices, const int64_t* __restrict__ cells,
                                     int64_t n, double* __restrict__ inv_out, double* __restrict__ det_out,
                                     int32_t* __restrict__ ok_out, int exact_zero) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n) return;
  double X[D + 1][D];
#pragma unroll
  for (int b = 0; b <= D; ++b)
#pragma unroll
    for (int i = 0; i < D; ++i) X[b][i] = vertices[cells[c * (D + 1) + b] * D + i];
  double inv[D * D], det;
  ok_out[c] = (exact_zero ? affine_inverse_fast<D, true>(X, inv, det) : affine_inverse_fast<D>(X, inv, det)) ? 1 : 0;
#pragma unroll
  for (int i = 0; i < D * D; ++i) inv_out[c * D * D + i] = inv[i];
  det_out[c] = det;
}

template <int D>
__global__ void geometry_fast32_kernel(const double* __restrict__ vertices, const int64_t* __restrict__ cells,
                                       int64_t n, float* __restrict__ inv_out, float* __restrict__ det_out,
                                       int32_t* __restrict__ ok_out) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n) return;
  double X[D + 1][D];
#pragma unroll
  for (int b = 0; b <= D; ++b)
#pragma unroll
    for (int i = 0; i < D; ++i) X[b][i] = vertices[cells[c * (D + 1) + b] * D + i];
  float inv[D * D];
  double det;
  ok_out[c] = affine_inverse_fast32<D>(X, inv, det) ? 1 : 0;
#pragma unroll
  for (int i = 0; i < D * D; ++i) inv_out[c * D * D + i] = inv[i];
  det_out[c] = (float)det;
}

}  // namespace txb

using namespace txb;

extern "C" int txb_debug_geometry_fast32(int dim, int64_t n_cells, const double* vertices, const int64_t* cells,
                                         float* inv_j, float* det_j, int32_t* ok, void* stream) {
  if (n_cells <= 0) return TXB_OK;
  const unsigned blocks = (unsigned)((n_cells + 255) / 256);
  if (dim == 2)
    geometry_fast32_kernel<2><<<blocks, 256, 0, (cudaStream_t)stream>>>(vertices, cells, n_cells, inv_j, det_j, ok);
  else if (dim == 3)
    geometry_fast32_kernel<3><<<blocks, 256, 0, (cudaStream_t)stream>>>(vertices, cells, n_cells, inv_j, det_j, ok);
  else {
    set_error("dim must be 2 or 3");
    return TXB_E_UNSUPPORTED;
  }
  TXB_CUDA_TRY(cudaGetLastError());
  return TXB_OK;
}

extern "C" int txb_debug_geometry_fast(int dim, int64_t n_cells, const double* vertices, const int64_t* cells,
                                       double* inv_j, double* det_j, int32_t* ok, int exact_zero, void* stream) {
  if (n_cells <= 0) return TXB_OK;
  const unsigned blocks = (unsigned)((n_cells + 255) / 256);
  if (dim == 2)
    geometry_fast_kernel<2><<<blocks, 256, 0, (cudaStream_t)stream>>>(vertices, cells, n_cells, inv_j, det_j, ok, exact_zero);
  else if (dim == 3)
    geometry_fast_kernel<3><<<blocks, 256, 0, (cudaStream_t)stream>>>(vertices, cells, n_cells, inv_j, det_j, ok, exact_zero);
  else {
    set_error("dim must be 2 or 3");
    return TXB_E_UNSUPPORTED;
  }
  TXB_CUDA_TRY(cudaGetLastError());
  return TXB_OK;
}

extern "C" int txb_tile_counts(int dim, int64_t n_cells, const int64_t* cells, int tile_cells, int32_t* counts,
                               void* stream) {
  return tile_launch(dim, n_cells, cells, tile_cells, 0, 0, counts, nullptr, nullptr, (cudaStream_t)stream);
}

extern "C" int txb_tile_build(int dim, int64_t n_cells, const int64_t* cells, int tile_cells, int vrec,
                              int local_bytes, int32_t* records, void* local, void* stream) {
  if (local_bytes != 1 && local_bytes != 2) {
    set_error("tiles: local_bytes must be 1 or 2, got %d", local_bytes);
    return TXB_E_ARG;
  }
  if (vrec < 8 || vrec % 4) {
    set_error("tiles: vrec must be a multiple of 4 and >= 8, got %d", vrec);
    return TXB_E_ARG;
  }
  return tile_launch(dim, n_cells, cells, tile_cells, vrec, local_bytes, nullptr, records, local,
                     (cudaStream_t)stream);
}

extern "C" int txb_integrate_mesh_tiled(int form_code, int aux_mode, int dtype_bytes, int dim, int n_q, int n_comp,
                                        int64_t n_cells, int64_t n_vertices, const void* basis,
                                        const void* basis_der, const void* weights, const double* vertices,
                                        int tile_cells, const int32_t* records, int vrec, const void* local,
                                        int local_bytes, const void* coeffs_global, const void* inv_j,
                                        const void* det_j, const void* aux, void* out, int64_t* bad_cell,
                                        void* stream) {
  Config c{form_code, aux_mode, dtype_bytes, dim, n_q, n_comp};
  int rc = validate(c);
  if (rc) return rc;
  if (n_cells < 0 || n_vertices < 0 || n_vertices >= ((int64_t)1 << 31)) {
    set_error("tiled mesh integration needs n_cells >= 0 and 0 <= n_vertices < 2^31");
    return TXB_E_SHAPE;
  }
  if (!basis || !basis_der || !weights) {
    set_error("basis, basis_der and weights are required (host pointers)");
    return TXB_E_ARG;
  }
  if (!standard_tables(c, basis_der) || c.n_q > 2) {
    set_error("mesh-fused integration needs the standard P1 tabulation with n_q <= 2");
    return TXB_E_UNSUPPORTED;
  }
  const int nbs = (dim + 1) * n_q;
  if (tile_cells < 1 || tile_cells % nbs || tile_cells % (32 / n_q) || tile_cells * (dim + 1) > 1024) {
    set_error("tile_cells %d must be a multiple of n_b*n_q = %d and of 32/n_q, with tile_cells*(dim+1) <= 1024",
              tile_cells, nbs);
    return TXB_E_CONFIG;
  }
  if ((local_bytes != 1 && local_bytes != 2) || vrec < 8 || vrec % 4) {
    set_error("tiles: local_bytes 1|2 and vrec a multiple of 4 >= 8 (got %d, %d)", local_bytes, vrec);
    return TXB_E_ARG;
  }
  if ((inv_j == nullptr) != (det_j == nullptr)) {
    set_error("give both inv_j and det_j, or neither (computed from the vertices)");
    return TXB_E_ARG;
  }
  const bool geom = inv_j != nullptr;
  KernelInfo k;
  if (!pick_tiled_kernel(c, local_bytes, vrec, geom, k)) {
    set_error("no tiled kernel instantiation for this configuration");
    return TXB_E_UNSUPPORTED;
  }
  Geometry g;
  rc = compute_geometry(c, k, n_cells, tile_cells / nbs, 0, true, g);
  if (rc) return rc;
  if (n_cells == 0) return TXB_OK;
  auto al16 = [](const void* p) { return ((uintptr_t)p & 15u) == 0; };
  if ((!geom && !vertices) || !records || !local || !coeffs_global || !out || (c.aux != 0 && !aux)) {
    set_error("NULL device pointer");
    return TXB_E_ARG;
  }
  if (!al16(records) || !al16(local)) {
    set_error("tile records and local indices must be 16-byte aligned");
    return TXB_E_ARG;
  }
  if (dtype_bytes == 4)
    return launch_tiled<float>(c, k, g, n_cells, basis, basis_der, weights, vertices, records, local, vrec,
                               coeffs_global, inv_j, det_j, aux, out, bad_cell, (cudaStream_t)stream);
  return launch_tiled<double>(c, k, g, n_cells, basis, basis_der, weights, vertices, records, local, vrec,
                              coeffs_global, inv_j, det_j, aux, out, bad_cell, (cudaStream_t)stream);
}
