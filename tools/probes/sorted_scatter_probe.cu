// sorted_scatter_probe.cu -- would a two-pass scatter-add beat the gather
// walk?  Pass 1 (permute): element entry i = (cell, b) is stored at pos[i],
// its position in the slot-ordered CSR (the inverse of slot_incidence), so
// every vertex's entries become one contiguous run in ascending cell order.
// Pass 2 (runs): one thread per slot sums its run sequentially from +0 (the
// np.add.at chain) and writes out[slot_vertex[t]].  Pass 2s: the same with
// the CTA's contiguous range of the sorted array staged in shared memory by
// coalesced loads first.  Same chains, same bits as txb_scatter_add_slots.
// Scalar fields (n_comp = 1).  Build (tools/sorted_scatter_probe.py does it):
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -shared -o sorted_scatter_probe.so sorted_scatter_probe.cu
#include <cstdint>
#include <cuda_runtime.h>

template <typename T>
__global__ void __launch_bounds__(256) permute_kernel(int64_t n, const int32_t* __restrict__ pos,
                                                      const T* __restrict__ elem, T* __restrict__ sorted) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    sorted[__ldg(pos + i)] = __ldg(elem + i);
}

template <typename T>
__global__ void __launch_bounds__(256) runs_kernel(int64_t n_slots, const int64_t* __restrict__ so,
                                                   const int32_t* __restrict__ sv, const T* __restrict__ sorted,
                                                   T* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_slots; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = so[t], e = so[t + 1];
    T s = T(0);
    for (int64_t k = b; k < e; ++k) s += __ldg(sorted + k);
    out[__ldg(sv + t)] = s;
  }
}

// 256 slots per CTA; their runs are one contiguous range [so[t0], so[t0+256])
template <typename T>
__global__ void __launch_bounds__(256) runs_staged_kernel(int64_t n_slots, const int64_t* __restrict__ so,
                                                          const int32_t* __restrict__ sv,
                                                          const T* __restrict__ sorted, T* __restrict__ out,
                                                          int cap) {
  extern __shared__ __align__(16) unsigned char smem[];
  T* buf = reinterpret_cast<T*>(smem);
  const int64_t t0 = (int64_t)blockIdx.x * 256;
  const int64_t t1 = t0 + 256 < n_slots ? t0 + 256 : n_slots;
  const int64_t lo = so[t0], hi = so[t1];
  const int64_t t = t0 + threadIdx.x;
  if (hi - lo <= cap) {
    for (int64_t k = lo + threadIdx.x; k < hi; k += 256) buf[k - lo] = __ldg(sorted + k);
    __syncthreads();
    if (t < t1) {
      const int64_t b = so[t] - lo, e = so[t + 1] - lo;
      T s = T(0);
      for (int64_t k = b; k < e; ++k) s += buf[k];
      out[__ldg(sv + t)] = s;
    }
  } else if (t < t1) {
    T s = T(0);
    for (int64_t k = so[t]; k < so[t + 1]; ++k) s += __ldg(sorted + k);
    out[__ldg(sv + t)] = s;
  }
}

extern "C" int probe_permute(int dtype, int64_t n, const int32_t* pos, const void* elem, void* sorted, void* stream) {
  const int blocks = (int)((n + 255) / 256 < 148 * 16 ? (n + 255) / 256 : 148 * 16);
  if (dtype == 8)
    permute_kernel<double><<<blocks, 256, 0, (cudaStream_t)stream>>>(n, pos, (const double*)elem, (double*)sorted);
  else
    permute_kernel<float><<<blocks, 256, 0, (cudaStream_t)stream>>>(n, pos, (const float*)elem, (float*)sorted);
  return (int)cudaGetLastError();
}

extern "C" int probe_runs(int dtype, int staged, int64_t n_slots, const int64_t* so, const int32_t* sv,
                          const void* sorted, void* out, void* stream) {
  const int blocks = (int)((n_slots + 255) / 256);
  cudaStream_t s = (cudaStream_t)stream;
  if (!staged) {
    if (dtype == 8) runs_kernel<double><<<blocks, 256, 0, s>>>(n_slots, so, sv, (const double*)sorted, (double*)out);
    else runs_kernel<float><<<blocks, 256, 0, s>>>(n_slots, so, sv, (const float*)sorted, (float*)out);
  } else {
    const int bytes = 64 * 1024;
    if (dtype == 8) {
      cudaFuncSetAttribute(runs_staged_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
      runs_staged_kernel<double><<<blocks, 256, bytes, s>>>(n_slots, so, sv, (const double*)sorted, (double*)out,
                                                           bytes / 8);
    } else {
      cudaFuncSetAttribute(runs_staged_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
      runs_staged_kernel<float><<<blocks, 256, bytes, s>>>(n_slots, so, sv, (const float*)sorted, (float*)out,
                                                          bytes / 4);
    }
  }
  return (int)cudaGetLastError();
}
