// txb_mesh.cu — the data movement either side of the integration kernel
// (SURVEY.md §8f rows 1-3), on the device and bit-identical to the reference:
//
//   txb_gather_coefficients  <- txfem/mesh.py:202-217  (E: global -> per-cell blocks)
//   txb_build_incidence      vertex -> (cell, b) CSR in ascending cell order
//   txb_scatter_add          <- txfem/mesh.py:220-234  (E^T: np.add.at order, no atomics)
//   txb_build_scatter_order / txb_scatter_add_slots: the same sums visited in
//                            element-row order (locality past the L2 size)
//   txb_compute_geometry     <- txfem/mesh.py:150-190  (cofactor inverse, detJ > 0 check)
//
// Plus the library's error plumbing (txb_last_error).
#include "txb_common.cuh"

#include <algorithm>
#include <atomic>
#include <mutex>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

namespace txb {

static thread_local char g_err[512] = {0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_fail(cudaError_t e, const char* what) {
  set_error("CUDA error %d (%s) in %s", (int)e, cudaGetErrorString(e), what);
  return TXB_E_CUDA;
}

constexpr int TPB = 256;

static int blocks_for(int64_t n) { return (int)std::min<int64_t>((n + TPB - 1) / TPB, 1 << 20); }

// ---- gather: one thread per output scalar (coalesced stores, indirect loads)
template <typename T>
__global__ void gather_kernel(int64_t n_out, int n_b, int n_comp, const int64_t* __restrict__ cells,
                              const T* __restrict__ global, T* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < n_out; o += stride) {
    const int64_t cb = o / n_comp;  // flat (cell, b)
    const int k = (int)(o - cb * n_comp);
    out[o] = global[__ldg(cells + cb) * n_comp + k];
  }
}

// Fixed component count: one thread per (cell, b) entry -- one connectivity
// load, NCOMP adjacent coefficient loads, no 64-bit division per scalar.
template <typename T, int NCOMP>
__global__ void gather_entries_kernel(int64_t n_entries, const int64_t* __restrict__ cells,
                                      const T* __restrict__ global, T* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_entries; i += stride) {
    const int64_t v = __ldg(cells + i);
    T x[NCOMP];
#pragma unroll
    for (int k = 0; k < NCOMP; ++k) x[k] = __ldg(global + v * NCOMP + k);
#pragma unroll
    for (int k = 0; k < NCOMP; ++k) out[i * NCOMP + k] = x[k];
  }
}

// ---- scatter-add: one thread per (vertex, component), sums its incident
// element entries in ascending (cell, b) order starting from +0, exactly the
// sequence np.add.at applies (mesh.py:232-233).  The incidence list is read
// U entries at a time so U element loads are in flight per thread; the
// NCOMP threads of a vertex read the same element rows (shared sectors).
// (Measured alternatives -- one thread per vertex for all components, and a
// shared-memory staged CSR range per CTA -- were slower; profiles/r1_pipeline.md.)
constexpr int SCATTER_TPB = 256;

template <typename T, int NCOMP>
__global__ void __launch_bounds__(SCATTER_TPB)
scatter_kernel(int64_t n_vertices, const int64_t* __restrict__ offsets, const int32_t* __restrict__ incidence,
               const int32_t* __restrict__ slot_vertex, const T* __restrict__ elem, T* __restrict__ out) {
  constexpr int U = 8;
  const int64_t n = n_vertices * NCOMP;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < n; o += stride) {
    const int64_t v = NCOMP == 1 ? o : o / NCOMP;  // CSR row (vertex, or slot when slot_vertex)
    const int k = NCOMP == 1 ? 0 : (int)(o - v * NCOMP);
    int64_t e = offsets[v];
    const int64_t end = offsets[v + 1];
    T sum = T(0);
    for (; e < end; e += U) {
      int32_t idx[U];
#pragma unroll
      for (int u = 0; u < U; ++u) idx[u] = e + u < end ? __ldg(incidence + e + u) : -1;
      T val[U];
#pragma unroll
      for (int u = 0; u < U; ++u) val[u] = idx[u] >= 0 ? __ldg(elem + (int64_t)idx[u] * NCOMP + k) : T(0);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (idx[u] >= 0) sum = add(sum, val[u]);
    }
    if (slot_vertex) out[(int64_t)__ldg(slot_vertex + v) * NCOMP + k] = sum;
    else out[o] = sum;
  }
}

// ---- scatter order.  The element rows are laid out in cell order, the
// output in vertex order; when the two orders disagree (the reference's 3D
// unit mesh numbers vertices x-fastest and cubes z-fastest,
// txfem/mesh.py:113-127) the consecutive vertices of one warp read element
// rows megabytes apart and, past the L2 size, every row costs a scattered DRAM
// sector.  A SLOT order visits the vertices by their first incident element
// row instead, so neighbouring threads read neighbouring rows; the CSR is
// re-laid out in slot order (coalesced incidence reads) and slot_vertex[t]
// says which vertex slot t writes.  Every vertex keeps its own chain, so the
// sums are unchanged bit for bit.
__global__ void first_row_keys_kernel(int64_t n_vertices, const int64_t* __restrict__ offsets,
                                      const int32_t* __restrict__ incidence, int32_t sentinel, int32_t* keys,
                                      int32_t* vals) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n_vertices; v += stride) {
    const int64_t e = offsets[v];
    keys[v] = e < offsets[v + 1] ? incidence[e] : sentinel;
    vals[v] = (int32_t)v;
  }
}

__global__ void slot_counts_kernel(int64_t n_slots, const int64_t* __restrict__ offsets,
                                   const int32_t* __restrict__ slot_vertex, int64_t* counts) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n_slots; t += stride) {
    const int64_t v = slot_vertex[t];
    counts[t] = offsets[v + 1] - offsets[v];
  }
}

// One warp per 32 consecutive slots; the lanes copy each slot's list together
// (coalesced stores into the slot-ordered CSR).
__global__ void slot_copy_kernel(int64_t n_slots, const int64_t* __restrict__ offsets,
                                 const int32_t* __restrict__ incidence, const int32_t* __restrict__ slot_vertex,
                                 const int64_t* __restrict__ slot_offsets, int32_t* __restrict__ slot_incidence) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w * 32 < n_slots; w += warps) {
    const int64_t t_end = w * 32 + 32 < n_slots ? w * 32 + 32 : n_slots;
    for (int64_t t = w * 32; t < t_end; ++t) {
      const int64_t v = slot_vertex[t];
      const int64_t src = offsets[v], len = offsets[v + 1] - src, dst = slot_offsets[t];
      for (int64_t i = lane; i < len; i += 32) slot_incidence[dst + i] = incidence[src + i];
    }
  }
}

__global__ void iota_keys_kernel(int64_t n, const int64_t* __restrict__ cells, int32_t* keys, int32_t* vals,
                                 int64_t* counts) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int64_t v = cells[i];
    keys[i] = (int32_t)v;
    vals[i] = (int32_t)i;
    atomicAdd(reinterpret_cast<unsigned long long*>(counts + v), 1ull);
  }
}

// ---- geometry: one thread per cell, float64, the reference's expression
// order (numpy evaluates a*b - c*d as two rounded products and a rounded
// difference; the 3x3 determinant sums left to right).
// One thread per cell; the CTA stages its cells' inverse Jacobians in shared
// memory (odd stride D*D) and stores them as one contiguous coalesced run.
template <int D>
__global__ void __launch_bounds__(TPB) geometry_kernel(int64_t n, const double* __restrict__ X_,
                                                       const int64_t* __restrict__ cells,
                                                       double* __restrict__ inv_j, double* __restrict__ det_j,
                                                       unsigned long long* bad) {
  constexpr int DD = D * D;
  __shared__ double s_inv[TPB * DD];
  for (int64_t base = (int64_t)blockIdx.x * TPB; base < n; base += (int64_t)gridDim.x * TPB) {
    const int64_t c = base + threadIdx.x;
    if (c < n) {
      const int64_t* cv = cells + c * (D + 1);
      int64_t ids[D + 1];
#pragma unroll
      for (int b = 0; b <= D; ++b) ids[b] = __ldg(cv + b);
      double X[D + 1][D];
#pragma unroll
      for (int b = 0; b <= D; ++b)
#pragma unroll
        for (int i = 0; i < D; ++i) X[b][i] = __ldg(X_ + ids[b] * D + i);
      double inv[DD], det;
      affine_inverse<D>(X, inv, det);
#pragma unroll
      for (int i = 0; i < DD; ++i) s_inv[threadIdx.x * DD + i] = inv[i];
      det_j[c] = det;
      if (det <= 0.0) atomicMin(bad, (unsigned long long)c);
    }
    __syncthreads();
    const int cnt = (n - base < TPB ? (int)(n - base) : TPB) * DD;
    for (int i = threadIdx.x; i < cnt; i += TPB) inv_j[base * DD + i] = s_inv[i];
    __syncthreads();
  }
}

}  // namespace txb

using namespace txb;

extern "C" const char* txb_last_error(void) { return g_err; }

extern "C" int txb_gather_coefficients(int dtype_bytes, int64_t n_cells, int n_b, int n_comp,
                                       const int64_t* cells, const void* global, void* out,
                                       void* stream) {
  if (n_cells < 0 || n_b < 1 || n_comp < 1) {
    set_error("gather: bad sizes n_cells=%lld n_b=%d n_comp=%d", (long long)n_cells, n_b, n_comp);
    return TXB_E_SHAPE;
  }
  if (n_cells == 0) return TXB_OK;
  if (!cells || !global || !out) {
    set_error("gather: NULL device pointer");
    return TXB_E_ARG;
  }
  const int64_t n_out = n_cells * n_b * n_comp;
  cudaStream_t s = (cudaStream_t)stream;
  if ((dtype_bytes == 4 || dtype_bytes == 8) && n_comp <= 3) {
    const int64_t n_e = n_cells * n_b;
#define TXB_GATHER(T, NC) \
  gather_entries_kernel<T, NC><<<blocks_for(n_e), TPB, 0, s>>>(n_e, cells, (const T*)global, (T*)out)
    if (dtype_bytes == 8) {
      if (n_comp == 1) TXB_GATHER(double, 1);
      else if (n_comp == 2) TXB_GATHER(double, 2);
      else TXB_GATHER(double, 3);
    } else {
      if (n_comp == 1) TXB_GATHER(float, 1);
      else if (n_comp == 2) TXB_GATHER(float, 2);
      else TXB_GATHER(float, 3);
    }
#undef TXB_GATHER
  } else if (dtype_bytes == 8)
    gather_kernel<double><<<blocks_for(n_out), TPB, 0, s>>>(n_out, n_b, n_comp, cells,
                                                            (const double*)global, (double*)out);
  else if (dtype_bytes == 4)
    gather_kernel<float><<<blocks_for(n_out), TPB, 0, s>>>(n_out, n_b, n_comp, cells,
                                                           (const float*)global, (float*)out);
  else {
    set_error("dtype_bytes must be 4 or 8");
    return TXB_E_UNSUPPORTED;
  }
  TXB_CUDA_TRY(cudaGetLastError());
  return TXB_OK;
}

static int scatter_impl(int dtype_bytes, int64_t n_vertices, int n_comp, const int64_t* offsets,
                        const int32_t* incidence, const int32_t* slot_vertex, const void* elem, void* out,
                        void* stream) {
  if (n_vertices < 0 || n_comp < 1 || n_comp > TXB_MAX_COMP) {
    set_error("scatter: bad sizes (n_vertices=%lld, n_comp=%d)", (long long)n_vertices, n_comp);
    return TXB_E_SHAPE;
  }
  if (n_vertices == 0) return TXB_OK;
  if (!offsets || !incidence || !elem || !out) {
    set_error("scatter: NULL device pointer");
    return TXB_E_ARG;
  }
  if (dtype_bytes != 4 && dtype_bytes != 8) {
    set_error("dtype_bytes must be 4 or 8");
    return TXB_E_UNSUPPORTED;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int blocks = (int)std::min<int64_t>((n_vertices * n_comp + SCATTER_TPB - 1) / SCATTER_TPB, 1 << 20);
#define TXB_SCATTER(T, NC)                                                                                  \
  scatter_kernel<T, NC><<<blocks, SCATTER_TPB, 0, s>>>(n_vertices, offsets, incidence, slot_vertex, (const T*)elem, \
                                                        (T*)out)
  if (dtype_bytes == 8) {
    if (n_comp == 1) TXB_SCATTER(double, 1);
    else if (n_comp == 2) TXB_SCATTER(double, 2);
    else TXB_SCATTER(double, 3);
  } else {
    if (n_comp == 1) TXB_SCATTER(float, 1);
    else if (n_comp == 2) TXB_SCATTER(float, 2);
    else TXB_SCATTER(float, 3);
  }
#undef TXB_SCATTER
  TXB_CUDA_TRY(cudaGetLastError());
  return TXB_OK;
}

extern "C" int txb_scatter_add(int dtype_bytes, int64_t n_vertices, int n_comp, const int64_t* offsets,
                               const int32_t* incidence, const void* elem, void* out, void* stream) {
  return scatter_impl(dtype_bytes, n_vertices, n_comp, offsets, incidence, nullptr, elem, out, stream);
}

extern "C" int txb_scatter_add_slots(int dtype_bytes, int64_t n_vertices, int n_comp, const int64_t* slot_offsets,
                                     const int32_t* slot_incidence, const int32_t* slot_vertex, const void* elem,
                                     void* out, void* stream) {
  if (n_vertices > 0 && !slot_vertex) {
    set_error("scatter: NULL slot_vertex");
    return TXB_E_ARG;
  }
  return scatter_impl(dtype_bytes, n_vertices, n_comp, slot_offsets, slot_incidence, slot_vertex, elem, out,
                      stream);
}

// Scratch: keys_in, keys_out, vals_in (int32, n*n_b each), counts (int64,
// n_vertices+1), CUB temp storage for the radix sort and the scan.
static size_t cub_temp_bytes(int64_t n_entries, int64_t n_vertices) {
  size_t sort_b = 0, scan_b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sort_b, (const int32_t*)nullptr, (int32_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, (int64_t)n_entries);
  cub::DeviceScan::ExclusiveSum(nullptr, scan_b, (const int64_t*)nullptr, (int64_t*)nullptr,
                                (int64_t)(n_vertices + 1));
  return std::max(sort_b, scan_b);
}

static size_t a256(size_t x) { return (x + 255) / 256 * 256; }

extern "C" int64_t txb_incidence_scratch_bytes(int64_t n_cells, int n_b, int64_t n_vertices) {
  const int64_t n = n_cells * n_b;
  return (int64_t)(3 * a256(n * sizeof(int32_t)) + a256((n_vertices + 1) * sizeof(int64_t)) +
                   a256(cub_temp_bytes(n, n_vertices)));
}

extern "C" int txb_build_incidence(int64_t n_cells, int n_b, int64_t n_vertices, const int64_t* cells,
                                   int64_t* offsets, int32_t* incidence, void* scratch, void* stream) {
  if (n_cells < 0 || n_b < 1 || n_vertices < 0) {
    set_error("incidence: bad sizes");
    return TXB_E_SHAPE;
  }
  if (n_cells * n_b >= ((int64_t)1 << 31) || n_vertices >= ((int64_t)1 << 31)) {
    set_error("incidence: n_cells*n_b and n_vertices must be < 2^31 (int32 CSR)");
    return TXB_E_SHAPE;
  }
  if (!offsets || (n_cells > 0 && (!cells || !incidence || !scratch))) {
    set_error("incidence: NULL device pointer");
    return TXB_E_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = n_cells * n_b;
  unsigned char* p = (unsigned char*)scratch;
  int32_t* keys_in = (int32_t*)p;
  p += a256(n * sizeof(int32_t));
  int32_t* keys_out = (int32_t*)p;
  p += a256(n * sizeof(int32_t));
  int32_t* vals_in = (int32_t*)p;
  p += a256(n * sizeof(int32_t));
  int64_t* counts = (int64_t*)p;
  p += a256((n_vertices + 1) * sizeof(int64_t));
  void* temp = p;
  size_t temp_b = cub_temp_bytes(n, n_vertices);

  TXB_CUDA_TRY(cudaMemsetAsync(counts, 0, (n_vertices + 1) * sizeof(int64_t), s));
  if (n > 0) {
    iota_keys_kernel<<<blocks_for(n), TPB, 0, s>>>(n, cells, keys_in, vals_in, counts);
    TXB_CUDA_TRY(cudaGetLastError());
    // Stable LSD radix sort by vertex id: entries of one vertex keep their
    // ascending (cell, b) order.
    int end_bit = 1;
    while (end_bit < 31 && ((int64_t)1 << end_bit) < n_vertices) ++end_bit;
    TXB_CUDA_TRY(cub::DeviceRadixSort::SortPairs(temp, temp_b, keys_in, keys_out, vals_in, incidence,
                                                 (int64_t)n, 0, end_bit, s));
  }
  TXB_CUDA_TRY(cub::DeviceScan::ExclusiveSum(temp, temp_b, counts, offsets, (int64_t)(n_vertices + 1), s));
  return TXB_OK;
}

// Scratch: keys_in, keys_out, vals_in (int32, n_vertices each), counts
// (int64, n_vertices+1), CUB temp storage for the radix sort and the scan.
static size_t order_temp_bytes(int64_t n_vertices) {
  size_t sort_b = 0, scan_b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sort_b, (const int32_t*)nullptr, (int32_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, (int64_t)n_vertices);
  cub::DeviceScan::ExclusiveSum(nullptr, scan_b, (const int64_t*)nullptr, (int64_t*)nullptr,
                                (int64_t)(n_vertices + 1));
  return std::max(sort_b, scan_b);
}

extern "C" int64_t txb_scatter_order_scratch_bytes(int64_t n_vertices) {
  if (n_vertices < 0) return 0;
  return (int64_t)(3 * a256(n_vertices * sizeof(int32_t)) + a256((n_vertices + 1) * sizeof(int64_t)) +
                   a256(order_temp_bytes(n_vertices)));
}

extern "C" int txb_build_scatter_order(int64_t n_vertices, int64_t n_entries, const int64_t* offsets,
                                       const int32_t* incidence, int64_t* slot_offsets, int32_t* slot_incidence,
                                       int32_t* slot_vertex, void* scratch, void* stream) {
  if (n_vertices < 0 || n_entries < 0 || n_vertices >= ((int64_t)1 << 31) || n_entries >= ((int64_t)1 << 31)) {
    set_error("scatter order: n_vertices and n_entries must be in [0, 2^31)");
    return TXB_E_SHAPE;
  }
  if (!slot_offsets || (n_vertices > 0 && (!offsets || !slot_vertex || !scratch)) ||
      (n_entries > 0 && (!incidence || !slot_incidence))) {
    set_error("scatter order: NULL device pointer");
    return TXB_E_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  unsigned char* p = (unsigned char*)scratch;
  int32_t* keys_in = (int32_t*)p;
  p += a256(n_vertices * sizeof(int32_t));
  int32_t* keys_out = (int32_t*)p;
  p += a256(n_vertices * sizeof(int32_t));
  int32_t* vals_in = (int32_t*)p;
  p += a256(n_vertices * sizeof(int32_t));
  int64_t* counts = (int64_t*)p;
  p += a256((n_vertices + 1) * sizeof(int64_t));
  void* temp = p;
  size_t temp_b = order_temp_bytes(n_vertices);

  TXB_CUDA_TRY(cudaMemsetAsync(counts, 0, (n_vertices + 1) * sizeof(int64_t), s));
  if (n_vertices > 0) {
    // key = the vertex's first (smallest) element row; untouched vertices
    // (empty lists, output +0) go last.  The radix sort is stable.
    const int32_t sentinel = (int32_t)n_entries;
    first_row_keys_kernel<<<blocks_for(n_vertices), TPB, 0, s>>>(n_vertices, offsets, incidence, sentinel,
                                                                  keys_in, vals_in);
    TXB_CUDA_TRY(cudaGetLastError());
    int end_bit = 1;
    while (end_bit < 31 && ((int64_t)1 << end_bit) <= n_entries) ++end_bit;
    TXB_CUDA_TRY(cub::DeviceRadixSort::SortPairs(temp, temp_b, keys_in, keys_out, vals_in, slot_vertex,
                                                 (int64_t)n_vertices, 0, end_bit, s));
    slot_counts_kernel<<<blocks_for(n_vertices), TPB, 0, s>>>(n_vertices, offsets, slot_vertex, counts);
    TXB_CUDA_TRY(cudaGetLastError());
  }
  TXB_CUDA_TRY(cub::DeviceScan::ExclusiveSum(temp, temp_b, counts, slot_offsets, (int64_t)(n_vertices + 1), s));
  if (n_vertices > 0 && n_entries > 0) {
    slot_copy_kernel<<<blocks_for(n_vertices), TPB, 0, s>>>(n_vertices, offsets, incidence, slot_vertex,
                                                             slot_offsets, slot_incidence);
    TXB_CUDA_TRY(cudaGetLastError());
  }
  return TXB_OK;
}

// Orientation flags of txb_compute_geometry: a static device array (slots
// rotate, so concurrent calls on different streams do not share one) instead
// of an allocation per call.
constexpr int GEOM_FLAGS = 256;
__device__ unsigned long long g_geom_flags[GEOM_FLAGS];

static unsigned long long* geometry_flag() {
  static std::mutex mu;
  static std::vector<unsigned long long*> cache;
  static std::atomic<uint32_t> seq{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  unsigned long long* base;
  {
    std::lock_guard<std::mutex> lk(mu);
    if ((int)cache.size() <= dev) cache.resize(dev + 1, nullptr);
    if (!cache[dev]) {
      void* p = nullptr;
      if (cudaGetSymbolAddress(&p, g_geom_flags) != cudaSuccess) return nullptr;
      cache[dev] = (unsigned long long*)p;
    }
    base = cache[dev];
  }
  return base + seq.fetch_add(1) % GEOM_FLAGS;
}

extern "C" int txb_compute_geometry(int dim, int64_t n_cells, const double* vertices, const int64_t* cells,
                                    double* inv_j, double* det_j, int64_t* bad_cell, void* stream) {
  if (dim != 2 && dim != 3) {
    set_error("dim must be 2 or 3, got %d", dim);
    return TXB_E_UNSUPPORTED;
  }
  if (n_cells < 0) {
    set_error("n_cells must be >= 0");
    return TXB_E_SHAPE;
  }
  if (bad_cell) *bad_cell = -1;
  if (n_cells == 0) return TXB_OK;
  if (!vertices || !cells || !inv_j || !det_j) {
    set_error("geometry: NULL device pointer");
    return TXB_E_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  unsigned long long* flag = geometry_flag();
  if (!flag) return cuda_fail(cudaGetLastError(), "cudaGetSymbolAddress(g_geom_flags)");
  TXB_CUDA_TRY(cudaMemsetAsync(flag, 0xff, sizeof(unsigned long long), s));
  if (dim == 2)
    geometry_kernel<2><<<blocks_for(n_cells), TPB, 0, s>>>(n_cells, vertices, cells, inv_j, det_j, flag);
  else
    geometry_kernel<3><<<blocks_for(n_cells), TPB, 0, s>>>(n_cells, vertices, cells, inv_j, det_j, flag);
  TXB_CUDA_TRY(cudaGetLastError());
  unsigned long long h = ~0ull;
  TXB_CUDA_TRY(cudaMemcpyAsync(&h, flag, sizeof(h), cudaMemcpyDeviceToHost, s));
  TXB_CUDA_TRY(cudaStreamSynchronize(s));
  if (h != ~0ull) {
    if (bad_cell) *bad_cell = (int64_t)h;
    set_error("cell %lld is degenerate or negatively oriented", (long long)h);
    return TXB_E_ORIENTATION;
  }
  return TXB_OK;
}
