// txb_integrate_mesh.cu — element integration fused with the data movement
// the reference performs on the host before it:
//
//   reference (txfem/executor.py:194-212):  cell_geom = compute_geometry(mesh)
//                                           coeffs = gather_coefficients(mesh, layout, global)
//                                           cast to the run dtype, run the lane
//   here (one kernel):  per batch the producer bulk-copies the connectivity
//   slice (and the aux slice; with given geometry also inv_j/det_j); in the
//   quadrature phase each lane gathers its cell's vertex coordinates and
//   coefficients through the connectivity (L2-resident: a vertex is shared by
//   ~24 tetrahedra), computes invJ/detJ in float64 with the reference's
//   expressions, casts to the run precision, and integrates.  HBM traffic per
//   3D var-coef f64 cell drops from 152 B (+ the gather pass) to 72 B.
//
// Bit-identical to compute_geometry -> gather -> cast -> integrate_cells.
// Requires the standard P1 tables (every tabulation the reference builds:
// element.tabulate of the midpoint and two-point rules); other tables use the
// unfused kernels.
#include "txb_kernels.cuh"

namespace txb {

template <typename T>
struct MeshArgs {
  const double* vertices;     // (n_vertices, D) float64
  const int64_t* cells;       // (n_cells, D+1)
  const T* coeffs_global;     // (n_vertices * NCOMP)
  const T* inv_j;             // GEOM == 1: given geometry (n, D, D)
  const T* det_j;             //            and (n)
  const T* aux;               // (n, 1) P0 | (n, D+1, 1) P1 | NULL
  T* out;                     // (n, D+1, NCOMP)
  unsigned long long* bad;    // GEOM == 0: lowered to the first cell with detJ <= 0 (may be NULL)
  int64_t n_cells;
  int64_t n_chunks;
  int64_t chunk_cells;
  int n_bc;
  int stages;
  int warps;
  int bulk;
  int vec_coeffs;             // coeffs_global aligned to 2 scalars: paired loads for NCOMP 2 / 3
  int dynamic;
  int resident;
  int64_t static_batches;
  int prefetch;  // batches per CTA warmed into L2 before the programmatic-launch wait
  Tabulation<T> tab;
};

// Stage: connectivity (int64), aux, and for GEOM == 1 the given inv_j / det_j.
template <typename T, int D, int AUX, int GEOM>
struct MeshStage {
  static constexpr int NB = D + 1;
  static constexpr int AUXW = AUX == 1 ? 1 : (AUX == 2 ? NB : 0);
  __host__ __device__ static int cell_bytes(int n) { return round_up(n * NB * 8, 16); }
  __host__ __device__ static int aux_bytes(int n) { return round_up(n * AUXW * (int)sizeof(T), 16); }
  __host__ __device__ static int inv_bytes(int n) { return GEOM ? round_up(n * D * D * (int)sizeof(T), 16) : 0; }
  __host__ __device__ static int det_bytes(int n) { return GEOM ? round_up(n * (int)sizeof(T), 16) : 0; }
  __host__ __device__ static int stage_bytes(int n) { return cell_bytes(n) + aux_bytes(n) + inv_bytes(n) + det_bytes(n); }
};

template <typename T, int D, int NQ, int NCOMP, int FORM, int AUX, int GEOM, bool SMEM>
__device__ __forceinline__ void mesh_slice(const MeshArgs<T>& a, const int64_t* __restrict__ s_cells,
                                           const T* __restrict__ s_aux, const T* __restrict__ s_inv,
                                           const T* __restrict__ s_det, unsigned char* __restrict__ scratch,
                                           int64_t c0_batch, int c0, int ncell, int lane) {
  constexpr int NB = D + 1, DD = D * D, NBC = NB * NCOMP;
  constexpr int AUXW = AUX == 1 ? 1 : (AUX == 2 ? NB : 0);
  using S = MeshScratch<T, D, NQ, NCOMP>;
  T* s_tr = reinterpret_cast<T*>(scratch);
  T* s_f1 = reinterpret_cast<T*>(scratch + S::TR_BYTES);
  const int nc = min(S::CW, ncell - c0);

  // ---------------- quadrature phase: lane <-> (cell, q) ----------------
  {
    const int lc = NQ == 1 ? lane : lane / NQ;
    const int q = NQ == 1 ? 0 : lane - lc * NQ;
    if (lc < nc) {
      const int cell = c0 + lc;
      int64_t ids[NB];
      load_row<int64_t, NB, SMEM>(s_cells + cell * NB, ids);
      // gather (mesh.py:202-217): coefficient block of the cell's vertices --
      // issued before the geometry so its L2 latency overlaps the coordinates'
      T cf[NBC];
      using V2 = typename std::conditional<sizeof(T) == 8, double2, float2>::type;
      bool paired = false;
      // (given geometry only: with the in-kernel geometry the extra selects cost
      // more than the saved loads -- 3D elasticity f64 60.9 -> 62.8 us vs
      // 48.5 -> 46.7 us given)
      if constexpr (NCOMP == 2 && GEOM == 1) {
        if (a.vec_coeffs) {
          paired = true;
#pragma unroll
          for (int b = 0; b < NB; ++b) {
            const V2 v = __ldg(reinterpret_cast<const V2*>(a.coeffs_global + ids[b] * NCOMP));
            cf[b * NCOMP] = v.x;
            cf[b * NCOMP + 1] = v.y;
          }
        }
      } else if constexpr (NCOMP == 3 && GEOM == 1) {
        // a vertex's 3 components start on a pair boundary (even vertex: pair
        // then single) or one scalar past it (odd vertex: single then pair)
        if (a.vec_coeffs) {
          paired = true;
#pragma unroll
          for (int b = 0; b < NB; ++b) {
            const T* p = a.coeffs_global + ids[b] * NCOMP;
            const bool odd = ids[b] & 1;
            const T sgl = __ldg(p + (odd ? 0 : 2));
            const V2 v = __ldg(reinterpret_cast<const V2*>(p + (odd ? 1 : 0)));
            cf[b * NCOMP] = odd ? sgl : v.x;
            cf[b * NCOMP + 1] = odd ? v.x : v.y;
            cf[b * NCOMP + 2] = odd ? v.y : sgl;
          }
        }
      }
      if (!paired) {
#pragma unroll
        for (int b = 0; b < NB; ++b)
#pragma unroll
          for (int c = 0; c < NCOMP; ++c) cf[b * NCOMP + c] = __ldg(a.coeffs_global + ids[b] * NCOMP + c);
      }
      T J[DD];
      T det;
      if constexpr (GEOM == 0) {
        double X[NB][D];
#pragma unroll
        for (int b = 0; b < NB; ++b)
#pragma unroll
          for (int i = 0; i < D; ++i) X[b][i] = __ldg(a.vertices + ids[b] * D + i);
        double detd;
        cell_geometry<T, D>(X, J, det, detd);  // branch-free; exact fallback
        if (q == 0 && a.bad && detd <= 0.0) atomicMin(a.bad, (unsigned long long)(c0_batch + cell));
      } else {
        load_row<T, DD, SMEM>(s_inv + cell * DD, J);
        det = s_det[cell];
      }

      // standard P1 pull-back (see the exactness note in txb_kernels.cuh)
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
      if (q == 0) {
#pragma unroll
        for (int i = 0; i < DD; ++i) s_tr[S::tr(lc, i)] = J[i];
#pragma unroll
        for (int k = 0; k < D; ++k) s_tr[S::tr(lc, DD + k)] = tr[0][k];
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
        load_row<T, NB, SMEM>(s_aux + cell * AUXW, av);
        const T* Bq = a.tab.B + q * NB;
        a0 = mul(av[0], Bq[0]);
#pragma unroll
        for (int bb = 1; bb < NB; ++bb) a0 = add(a0, mul(av[bb], Bq[bb]));
      }
      (void)a0;

      const T wq = a.tab.W[q];

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
  T* o_base = a.out + (c0_batch + c0) * NBC;
  auto entry = [&](int o) {
    const int lc = o / NBC;
    const int r = o - lc * NBC;
    const int b = r / NCOMP;
    const int c = r - b * NCOMP;
    T f1[NQ * D];
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
      for (int k = 0; k < D; ++k) f1[q * D + k] = s_f1[S::f1(lc, (q * NCOMP + c) * D + k)];
    const int r0 = b == 0 ? DD : (b - 1) * D;  // T[0] after the invJ rows
    T t[D];
#pragma unroll
    for (int k = 0; k < D; ++k) t[k] = s_tr[S::tr(lc, r0 + k)];
    T e = T(0);  // the output chain starts at +0 exactly as the reference's
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
      for (int k = 0; k < D; ++k) e = add(e, mul(t[k], f1[q * D + k]));
    o_base[o] = e;
  };
  constexpr int FULL = S::CW * NBC;
  if (nc == S::CW && FULL % 32 == 0) {
#pragma unroll
    for (int s = 0; s < FULL / 32; ++s) entry(s * 32 + lane);
  } else {
    for (int o = lane; o < nc * NBC; o += 32) entry(o);
  }
  __syncwarp();
}

template <typename T, int D, int NQ, int NCOMP, int FORM, int AUX, int GEOM>
__global__ void __launch_bounds__(MAX_CTA_THREADS, 1)
integrate_mesh_kernel(const __grid_constant__ MeshArgs<T> a) {
  constexpr int NB = D + 1, DD = D * D;
  using L = MeshStage<T, D, AUX, GEOM>;
  using S = MeshScratch<T, D, NQ, NCOMP>;

  extern __shared__ __align__(128) unsigned char smem[];
  const int nbc = a.n_bc;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int W = a.warps;
  const int stage_bytes = L::stage_bytes(nbc);
  unsigned char* scratch_base = smem + a.stages * stage_bytes;
  const PipelineSmem p = carve_pipeline(scratch_base + W * S::BYTES);
  pipeline_init(a, p);
  if (warp == W && lane == 0 && a.bulk) {
    pipeline_first_batches(a, a.prefetch, [&](int64_t c0, int ncell) {
      const uint32_t kb = ncell * NB * 8, ab = ncell * L::AUXW * sizeof(T),
                     ib = GEOM ? ncell * DD * sizeof(T) : 0, db = GEOM ? ncell * sizeof(T) : 0;
      if ((kb | ab | ib | db) & 15u) return;
      bulk_prefetch_l2(a.cells + c0 * NB, kb);
      if constexpr (AUX != 0) bulk_prefetch_l2(a.aux + c0 * L::AUXW, ab);
      if constexpr (GEOM != 0) {
        bulk_prefetch_l2(a.inv_j + c0 * DD, ib);
        bulk_prefetch_l2(a.det_j + c0, db);
      }
    });
  }
  pipeline_wait_prior_grid();

  if (warp == W) {
    if (lane != 0) return;
    const uint64_t policy = l2_evict_first_policy();
    pipeline_produce(a, p, smem, stage_bytes, [&](unsigned char* st, int64_t c0, int ncell, uint64_t* bar) {
      const uint32_t kb = ncell * NB * 8, ab = ncell * L::AUXW * sizeof(T),
                     ib = GEOM ? ncell * DD * sizeof(T) : 0, db = GEOM ? ncell * sizeof(T) : 0;
      if (!a.bulk || ((kb | ab | ib | db) & 15u)) return false;
      mbar_arrive_expect_tx(bar, kb + ab + ib + db);
      bulk_g2s(st, a.cells + c0 * NB, kb, bar, policy);
      if constexpr (AUX != 0) bulk_g2s(st + L::cell_bytes(nbc), a.aux + c0 * L::AUXW, ab, bar, policy);
      if constexpr (GEOM != 0) {
        bulk_g2s(st + L::cell_bytes(nbc) + L::aux_bytes(nbc), a.inv_j + c0 * DD, ib, bar, policy);
        bulk_g2s(st + L::cell_bytes(nbc) + L::aux_bytes(nbc) + L::inv_bytes(nbc), a.det_j + c0, db, bar, policy);
      }
      return true;
    });
    return;
  }

  unsigned char* scratch = scratch_base + warp * S::BYTES;
  pipeline_consume(a, p, smem, stage_bytes, [&](const unsigned char* st, int64_t c0, int ncell) {
    if (st) {
      const int64_t* s_cells = reinterpret_cast<const int64_t*>(st);
      const T* s_aux = reinterpret_cast<const T*>(st + L::cell_bytes(nbc));
      const T* s_inv = reinterpret_cast<const T*>(st + L::cell_bytes(nbc) + L::aux_bytes(nbc));
      const T* s_det = reinterpret_cast<const T*>(st + L::cell_bytes(nbc) + L::aux_bytes(nbc) + L::inv_bytes(nbc));
      for (int c = warp * S::CW; c < ncell; c += W * S::CW)
        mesh_slice<T, D, NQ, NCOMP, FORM, AUX, GEOM, true>(a, s_cells, s_aux, s_inv, s_det, scratch, c0, c, ncell,
                                                           lane);
    } else {
      const T* g_aux = AUX != 0 ? a.aux + c0 * L::AUXW : nullptr;
      const T* g_inv = GEOM ? a.inv_j + c0 * DD : nullptr;
      const T* g_det = GEOM ? a.det_j + c0 : nullptr;
      for (int c = warp * S::CW; c < ncell; c += W * S::CW)
        mesh_slice<T, D, NQ, NCOMP, FORM, AUX, GEOM, false>(a, a.cells + c0 * NB, g_aux, g_inv, g_det, scratch, c0,
                                                            c, ncell, lane);
    }
  });
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
template <typename T, int D, int NQ, int NCOMP, int FORM, int AUX, int GEOM>
struct MeshKernel {
  static void* fn() { return (void*)integrate_mesh_kernel<T, D, NQ, NCOMP, FORM, AUX, GEOM>; }
  static int stage_bytes(int n_bc) { return MeshStage<T, D, AUX, GEOM>::stage_bytes(n_bc); }
  static int scratch(int) { return MeshScratch<T, D, NQ, NCOMP>::BYTES; }
  static constexpr int CW = 32 / NQ;
};

template <typename T, int D, int NQ, int GEOM>
static bool pick_mesh_form(const Config& c, KernelInfo& k) {
#define TXB_MK(NCOMP, FORM, AUX)                                            \
  {                                                                         \
    using K = MeshKernel<T, D, NQ, NCOMP, FORM, AUX, GEOM>;                 \
    k = {K::fn(), K::stage_bytes, K::scratch, K::CW};                       \
    k.family = FAMILY_MESH;                                                 \
    return true;                                                            \
  }
  if (c.form == 0) TXB_MK(1, 0, 0)
  if (c.form == 1 && c.aux == 1) TXB_MK(1, 1, 1)
  if (c.form == 1 && c.aux == 2) TXB_MK(1, 1, 2)
  if (c.form == 2) TXB_MK(D, 2, 0)
#undef TXB_MK
  return false;
}

template <typename T, int D>
static bool pick_mesh_nq(const Config& c, bool geom, KernelInfo& k) {
  if (c.n_q == 1) return geom ? pick_mesh_form<T, D, 1, 1>(c, k) : pick_mesh_form<T, D, 1, 0>(c, k);
  if (c.n_q == 2) return geom ? pick_mesh_form<T, D, 2, 1>(c, k) : pick_mesh_form<T, D, 2, 0>(c, k);
  return false;
}

static bool pick_mesh_kernel(const Config& c, bool geom, KernelInfo& k) {
  if (c.dtype == 4) return c.dim == 2 ? pick_mesh_nq<float, 2>(c, geom, k) : pick_mesh_nq<float, 3>(c, geom, k);
  return c.dim == 2 ? pick_mesh_nq<double, 2>(c, geom, k) : pick_mesh_nq<double, 3>(c, geom, k);
}

template <typename T>
static int launch_mesh(const Config& c, const KernelInfo& k, const Geometry& g, int64_t n_cells,
                       const void* basis, const void* basis_der, const void* weights, const double* vertices,
                       const int64_t* cells, const void* coeffs_global, const void* inv_j, const void* det_j,
                       const void* aux, void* out, int64_t* bad_cell, cudaStream_t stream) {
  MeshArgs<T> a;
  a.vertices = vertices;
  a.cells = cells;
  a.coeffs_global = (const T*)coeffs_global;
  a.inv_j = (const T*)inv_j;
  a.det_j = (const T*)det_j;
  a.aux = (const T*)aux;
  a.out = (T*)out;
  a.bad = (unsigned long long*)bad_cell;
  a.n_cells = n_cells;
  a.n_chunks = g.n_chunks;
  a.chunk_cells = g.chunk_cells;
  a.n_bc = g.n_bc;
  a.stages = g.stages;
  a.warps = g.warps;
  auto al16 = [](const void* p) { return ((uintptr_t)p & 15u) == 0; };
  const int nb = c.dim + 1, auxw = c.aux == 1 ? 1 : (c.aux == 2 ? nb : 0);
  auto sized16 = [&](int64_t per_cell_bytes) { return ((int64_t)g.n_bc * per_cell_bytes) % 16 == 0; };
  const bool geom = inv_j != nullptr;
  a.bulk = al16(cells) && sized16(nb * 8) && (c.aux == 0 || (al16(aux) && sized16(auxw * (int)sizeof(T)))) &&
           (!geom || (al16(inv_j) && al16(det_j) && sized16(c.dim * c.dim * (int)sizeof(T)) &&
                      sized16((int)sizeof(T)))) &&
           env_int("TXB_DISABLE_BULK", 0) == 0;
  a.vec_coeffs = ((uintptr_t)coeffs_global % (2 * sizeof(T))) == 0 && env_int("TXB_VEC_COEFFS", 1);
  a.dynamic = g.dynamic;
  a.resident = g.resident;
  a.static_batches = g.static_batches;
  a.prefetch = prefetch_batches(g);
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

}  // namespace txb

using namespace txb;

extern "C" int txb_integrate_mesh(int form_code, int aux_mode, int dtype_bytes, int dim, int n_q, int n_comp,
                                  int64_t n_cells, int64_t n_vertices, const void* basis, const void* basis_der,
                                  const void* weights, const double* vertices, const int64_t* cells,
                                  const void* coeffs_global, const void* inv_j, const void* det_j,
                                  const void* aux, void* out, int64_t* bad_cell, int n_bl, void* stream) {
  Config c{form_code, aux_mode, dtype_bytes, dim, n_q, n_comp};
  int rc = validate(c);
  if (rc) return rc;
  if (n_cells < 0 || n_vertices < 0) {
    set_error("n_cells and n_vertices must be >= 0");
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
  if ((inv_j == nullptr) != (det_j == nullptr)) {
    set_error("give both inv_j and det_j, or neither (computed from the vertices)");
    return TXB_E_ARG;
  }
  const bool geom = inv_j != nullptr;
  KernelInfo k;
  if (!pick_mesh_kernel(c, geom, k)) {
    set_error("no mesh kernel instantiation for this configuration");
    return TXB_E_UNSUPPORTED;
  }
  Geometry g;
  rc = compute_geometry(c, k, n_cells, n_bl, 0, true, g);
  if (rc) return rc;
  if (n_cells == 0) return TXB_OK;
  if (!cells || !coeffs_global || !out || (!geom && !vertices) || (c.aux != 0 && !aux)) {
    set_error("NULL device pointer");
    return TXB_E_ARG;
  }
  if (c.dtype == 4)
    return launch_mesh<float>(c, k, g, n_cells, basis, basis_der, weights, vertices, cells, coeffs_global, inv_j,
                              det_j, aux, out, bad_cell, (cudaStream_t)stream);
  return launch_mesh<double>(c, k, g, n_cells, basis, basis_der, weights, vertices, cells, coeffs_global, inv_j,
                             det_j, aux, out, bad_cell, (cudaStream_t)stream);
}
