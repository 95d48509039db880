// txb_halo.cu — the global-residual halo exchange over peer memory (one node,
// NVLink / NVSwitch): pack-and-put and flag-gated assembly, no NCCL.
//
// The exchange of halo.py: vertex v is owned by the
// lowest rank touching it; higher ranks send their RAW element rows for v to
// the owner, which chains them after its own rows in (rank, cell) order — the
// reference's np.add.at order (txfem/mesh.py:220-234), bit for bit.  Instead
// of pack -> NCCL all_to_all -> scatter, each rank exposes a WINDOW (device
// memory, shared by CUDA IPC handle between the processes of one node):
//
//   header  flags[s]  epoch of the last rows sender s delivered here (written by s)
//           acks[p]   epoch receiver p has finished reading this rank's rows (written by p)
//           counters  per-epoch-parity completion counters of the local kernels
//           error     first failure (spin timeout)
//   recv    two slots (epoch parity) of n_recv rows x n_comp scalars
//
//   txb_halo_put       reads this rank's owed rows from its element buffer and
//                      stores them straight into each owner's window (P2P
//                      stores over NVLink); the last CTA publishes
//                      flags[me] = epoch in every destination with a release
//                      store at system scope.  Before writing slot (epoch & 1)
//                      of a peer it waits for that peer's ack of epoch - 2.
//   txb_halo_assemble  waits (acquire, system scope) until every sender's flag
//                      reached the epoch, then runs the CSR chain over
//                      [local rows | received rows] (the txb_scatter_add chain);
//                      the last CTA acks the epoch to every sender.
//
// Spins are bounded (%globaltimer, TXB_HALO_TIMEOUT_MS, default 10 s): on
// timeout the kernel records an error in the window and finishes, so a lost
// peer never hangs the GPU; txb_halo_window_error reports it.
#include "txb_common.cuh"
#include "txb_halo.cuh"

#include <algorithm>
#include <cstdlib>
#include <cstring>

namespace txb {
namespace {

using namespace halo;  // window layout and spin/release primitives (txb_halo.cuh)
constexpr int TPB = 256;

template <typename T>
__global__ void __launch_bounds__(TPB)
put_kernel(int64_t n_send, int n_comp, int rank, const int64_t* __restrict__ send_rows,
           const int32_t* __restrict__ send_peer, const int64_t* __restrict__ send_dst, const T* __restrict__ elem,
           void* const* __restrict__ windows, const int64_t* __restrict__ slot_bytes,
           const int32_t* __restrict__ out_peers, int n_out_peers, unsigned long long epoch,
           unsigned long long timeout_ns) {
  WindowHeader* mine = header(windows[rank]);
  __shared__ int ok;
  if (threadIdx.x == 0) {
    ok = 1;
    // slot (epoch & 1) of each destination was last read at epoch - 2
    for (int i = 0; i < n_out_peers && epoch > 2; ++i)
      if (!wait_at_least(&mine->acks[out_peers[i]], epoch - 2, timeout_ns)) {
        atomicCAS(&mine->error, 0, 1);
        ok = 0;
        break;
      }
  }
  __syncthreads();
  if (ok) {
    const int64_t n = n_send * n_comp;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < n; o += stride) {
      const int64_t i = o / n_comp;
      const int c = (int)(o - i * n_comp);
      const int p = send_peer[i];
      T* slot = reinterpret_cast<T*>(static_cast<unsigned char*>(windows[p]) + HEADER_BYTES +
                                     (int64_t)(epoch & 1) * slot_bytes[p]);
      slot[send_dst[i] * n_comp + c] = elem[send_rows[i] * n_comp + c];  // P2P store into the owner's window
    }
  } else if (threadIdx.x == 0) {
    atomicExch(&mine->put_failed[epoch & 1], 1u);  // this CTA skipped its stores
  }
  __threadfence_system();  // this CTA's stores (or failure mark) before its completion count
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int* ctr = &mine->counters[epoch & 1];
    if (atomicAdd(ctr, 1u) == gridDim.x - 1) {
      __threadfence_system();
      atomicExch(ctr, 0u);  // reused at epoch + 2 (stream order)
      // a failed put still publishes the epoch (the receivers must not wait
      // out their own timeout), but poisoned: they report error 3 instead of
      // assembling rows that never arrived
      const unsigned long long flag = atomicExch(&mine->put_failed[epoch & 1], 0u) ? (epoch | POISON) : epoch;
      for (int i = 0; i < n_out_peers; ++i) store_release_sys(&header(windows[out_peers[i]])->flags[rank], flag);
    }
  }
}

template <typename T, int NC>
__global__ void __launch_bounds__(TPB)
assemble_kernel(int64_t n_owned, const int64_t* __restrict__ offsets, const int32_t* __restrict__ incidence,
                int64_t n_local_rows, const T* __restrict__ elem, int rank, void* const* __restrict__ windows,
                int64_t my_slot_bytes, const int32_t* __restrict__ in_peers, int n_in_peers,
                unsigned long long epoch, unsigned long long timeout_ns, T* __restrict__ out) {
  WindowHeader* mine = header(windows[rank]);
  const T* recv = reinterpret_cast<const T*>(static_cast<const unsigned char*>(windows[rank]) + HEADER_BYTES +
                                             (int64_t)(epoch & 1) * my_slot_bytes);
  __shared__ int bad;
  if (threadIdx.x == 0) {
    bad = 0;
    for (int i = 0; i < n_in_peers; ++i) {
      const unsigned long long f = wait_flag(&mine->flags[in_peers[i]], epoch, timeout_ns);
      if (f == 0 || (f & POISON)) {  // timed out, or the sender's put failed
        atomicCAS(&mine->error, 0, f == 0 ? 2 : 3);
        bad = 1;
        break;
      }
    }
  }
  __syncthreads();
  if (bad) {
    // never a silently wrong residual: the owned entries become NaN, the error
    // stays in the window (PeerHalo.check), and the epoch is NOT acked, so the
    // senders fail too instead of overwriting the slot
    const int64_t n = n_owned * NC;
    for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x)
      out[o] = T(__longlong_as_double(0x7ff8000000000000ll));
  } else {
    constexpr int U = 8;
    const int64_t n = n_owned * NC;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < n; o += stride) {
      const int64_t v = NC == 1 ? o : o / NC;
      const int k = NC == 1 ? 0 : (int)(o - v * NC);
      int64_t e = offsets[v];
      const int64_t end = offsets[v + 1];
      T sum = T(0);  // +0, then every row in (rank, cell) order: np.add.at's chain
      for (; e < end; e += U) {
        int32_t idx[U];
#pragma unroll
        for (int u = 0; u < U; ++u) idx[u] = e + u < end ? __ldg(incidence + e + u) : -1;
        T val[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (idx[u] < 0)
            val[u] = T(0);
          else if (idx[u] < n_local_rows)
            val[u] = __ldg(elem + (int64_t)idx[u] * NC + k);
          else  // peer-written: bypass L1 (the slot is rewritten every other epoch)
            val[u] = __ldcg(recv + ((int64_t)idx[u] - n_local_rows) * NC + k);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (idx[u] >= 0) sum = add(sum, val[u]);
      }
      out[o] = sum;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int* ctr = &mine->counters[2 + (epoch & 1)];
    if (atomicAdd(ctr, 1u) == gridDim.x - 1) {
      __threadfence_system();  // every CTA's reads of the slot are done
      atomicExch(ctr, 0u);
      // the error is sticky: a rank that failed once never acks again, so its
      // senders fail as well rather than reuse a slot it may not have read
      if (atomicAdd(&mine->error, 0) == 0)
        for (int i = 0; i < n_in_peers; ++i) store_release_sys(&header(windows[in_peers[i]])->acks[rank], epoch);
    }
  }
}



int grid_for(int64_t n, int sms_cap = 4 * 148) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + TPB - 1) / TPB, sms_cap));
}

}  // namespace
}  // namespace txb

using namespace txb;

extern "C" int64_t txb_halo_window_bytes(int64_t n_recv_rows, int n_comp, int dtype_bytes) {
  const int64_t slot = (std::max<int64_t>(n_recv_rows, 1) * n_comp * dtype_bytes + 255) / 256 * 256;
  return HEADER_BYTES + 2 * slot;
}

extern "C" int txb_halo_window_alloc(int64_t bytes, void** window, void* ipc_handle) {
  if (!window || bytes < HEADER_BYTES) {
    set_error("halo window: need a result pointer and at least %lld bytes", (long long)HEADER_BYTES);
    return TXB_E_ARG;
  }
  *window = nullptr;
  void* p = nullptr;
  TXB_CUDA_TRY(cudaMalloc(&p, (size_t)bytes));
  TXB_CUDA_TRY(cudaMemset(p, 0, (size_t)bytes));
  if (ipc_handle) {
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, p);
    if (e != cudaSuccess) {
      cudaFree(p);
      return cuda_fail(e, "cudaIpcGetMemHandle");
    }
    memcpy(ipc_handle, &h, sizeof h);
  }
  *window = p;
  return TXB_OK;
}

extern "C" int txb_halo_window_open(const void* ipc_handle, void** window) {
  if (!ipc_handle || !window) {
    set_error("halo window open: NULL argument");
    return TXB_E_ARG;
  }
  cudaIpcMemHandle_t h;
  memcpy(&h, ipc_handle, sizeof h);
  TXB_CUDA_TRY(cudaIpcOpenMemHandle(window, h, cudaIpcMemLazyEnablePeerAccess));
  return TXB_OK;
}

extern "C" int txb_halo_window_close(void* window) {
  if (window) TXB_CUDA_TRY(cudaIpcCloseMemHandle(window));
  return TXB_OK;
}

extern "C" int txb_halo_window_free(void* window) {
  if (window) TXB_CUDA_TRY(cudaFree(window));
  return TXB_OK;
}

extern "C" int txb_halo_window_error(void* window, int* error) {
  if (!window || !error) {
    set_error("halo window error: NULL argument");
    return TXB_E_ARG;
  }
  TXB_CUDA_TRY(cudaMemcpy(error, &header(window)->error, sizeof(int), cudaMemcpyDeviceToHost));
  return TXB_OK;
}

extern "C" int txb_halo_put(int dtype_bytes, int n_comp, int rank, int world, int64_t n_send,
                            const int64_t* send_rows, const int32_t* send_peer, const int64_t* send_dst,
                            const void* elem, void* const* windows, const int64_t* slot_bytes,
                            const int32_t* out_peers, int n_out_peers, uint64_t epoch, void* stream) {
  if (world < 1 || world > MAX_RANKS || rank < 0 || rank >= world || n_comp < 1 || n_comp > TXB_MAX_COMP ||
      n_send < 0 || n_out_peers < 0 || n_out_peers > world - 1 || epoch == 0) {
    set_error("halo put: bad arguments (rank %d of %d, n_comp %d, n_send %lld, epoch %llu)", rank, world, n_comp,
              (long long)n_send, (unsigned long long)epoch);
    return TXB_E_ARG;
  }
  if (!windows || !slot_bytes || (n_send && (!send_rows || !send_peer || !send_dst || !elem)) ||
      (n_out_peers && !out_peers)) {
    set_error("halo put: NULL device pointer");
    return TXB_E_ARG;
  }
  if (n_out_peers == 0) return TXB_OK;  // nothing owed to anyone
  cudaStream_t s = (cudaStream_t)stream;
  const int grid = grid_for(n_send * n_comp);
  if (dtype_bytes == 8)
    put_kernel<double><<<grid, TPB, 0, s>>>(n_send, n_comp, rank, send_rows, send_peer, send_dst,
                                            (const double*)elem, windows, slot_bytes, out_peers, n_out_peers,
                                            epoch, timeout_ns());
  else if (dtype_bytes == 4)
    put_kernel<float><<<grid, TPB, 0, s>>>(n_send, n_comp, rank, send_rows, send_peer, send_dst,
                                           (const float*)elem, windows, slot_bytes, out_peers, n_out_peers,
                                           epoch, timeout_ns());
  else {
    set_error("dtype_bytes must be 4 or 8");
    return TXB_E_UNSUPPORTED;
  }
  TXB_CUDA_TRY(cudaGetLastError());
  return TXB_OK;
}

extern "C" int txb_halo_assemble(int dtype_bytes, int n_comp, int rank, int world, int64_t n_owned,
                                 const int64_t* offsets, const int32_t* incidence, int64_t n_local_rows,
                                 const void* elem, void* const* windows, int64_t my_slot_bytes,
                                 const int32_t* in_peers, int n_in_peers, uint64_t epoch, void* out,
                                 void* stream) {
  if (world < 1 || world > MAX_RANKS || rank < 0 || rank >= world || n_comp < 1 || n_comp > TXB_MAX_COMP ||
      n_owned < 0 || n_local_rows < 0 || n_in_peers < 0 || epoch == 0) {
    set_error("halo assemble: bad arguments");
    return TXB_E_ARG;
  }
  if (!windows || (n_owned && (!offsets || !incidence || !out)) || (n_local_rows && !elem) ||
      (n_in_peers && !in_peers)) {
    set_error("halo assemble: NULL device pointer");
    return TXB_E_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int grid = grid_for(n_owned * n_comp, 1 << 20);
#define TXB_ASM(T, NC)                                                                                   \
  assemble_kernel<T, NC><<<grid, TPB, 0, s>>>(n_owned, offsets, incidence, n_local_rows, (const T*)elem, \
                                              rank, windows, my_slot_bytes, in_peers, n_in_peers, epoch,  \
                                              timeout_ns(), (T*)out)
  if (dtype_bytes == 8) {
    if (n_comp == 1) TXB_ASM(double, 1);
    else if (n_comp == 2) TXB_ASM(double, 2);
    else TXB_ASM(double, 3);
  } else if (dtype_bytes == 4) {
    if (n_comp == 1) TXB_ASM(float, 1);
    else if (n_comp == 2) TXB_ASM(float, 2);
    else TXB_ASM(float, 3);
  } else {
    set_error("dtype_bytes must be 4 or 8");
    return TXB_E_UNSUPPORTED;
  }
#undef TXB_ASM
  TXB_CUDA_TRY(cudaGetLastError());
  return TXB_OK;
}
