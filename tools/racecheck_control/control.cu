// Control experiment for compute-sanitizer racecheck (tuning/verification aid).
//
// The canonical single-stage pattern: one thread posts expect_tx and a
// cp.async.bulk global->shared copy completing on an mbarrier, and writes a
// plain shared-memory word before its (release) arrive; every other thread
// waits on the mbarrier (acquire) and then reads both.  This is race-free by
// the PTX memory model (mbarrier arrive = release, try_wait = acquire,
// complete_tx makes the bulk copy's writes visible to the waiting threads).
// If racecheck reports hazards here, it does not model mbarrier
// synchronisation and the same reports on the library's pipeline are not
// evidence of a race.  `mode 1` uses __syncthreads instead (expected clean).
//
// nvcc -gencode arch=compute_100a,code=sm_100a -I../../paper_1607_04245_b200/csrc control.cu -o control
// compute-sanitizer --tool racecheck ./control 0 ; compute-sanitizer --tool racecheck ./control 1
#include <cstdio>
#include <cstdlib>

#include "txb_device.cuh"

using namespace txb;

__global__ void control(const double* __restrict__ src, double* __restrict__ dst, int mode) {
  __shared__ __align__(128) double stage[256];
  __shared__ int info;
  __shared__ uint64_t full;
  if (threadIdx.x == 0) {
    mbar_init(&full, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (mode == 0) {
    if (threadIdx.x == 0) {
      info = 7;
      mbar_arrive_expect_tx(&full, 256 * sizeof(double));
      bulk_g2s(stage, src, 256 * sizeof(double), &full, l2_evict_first_policy());
    }
    mbar_wait(&full, 0);
  } else {
    if (threadIdx.x == 0) info = 7;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) stage[i] = src[i];
    __syncthreads();
  }
  dst[threadIdx.x] = stage[threadIdx.x] + info;
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  double *src, *dst;
  cudaMalloc(&src, 256 * sizeof(double));
  cudaMalloc(&dst, 256 * sizeof(double));
  cudaMemset(src, 0, 256 * sizeof(double));
  control<<<1, 256>>>(src, dst, mode);
  double h[256];
  cudaMemcpy(h, dst, sizeof h, cudaMemcpyDeviceToHost);
  printf("mode %d: dst[255] = %g (%s)\n", mode, h[255], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
