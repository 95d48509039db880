// gather_probe.cu -- micro-benchmark of the fused mesh kernel's vertex gathers
// (SURVEY.md §8f row 3): per tetrahedron, 4 vertex rows gathered through the
// connectivity of a 3D Kuhn mesh (generate_unit_simplex_mesh ordering: cubes
// z fastest, vertices x fastest), one thread per cell.
//   v0: coordinates (n_v, 3) f64 as three 8-byte loads + the coefficient (8 B)
//   v1: packed rows [x, y, z, u] f64 (32 B): one 256-bit load
//   v2: packed rows, two 128-bit loads
//   v3: padded coordinates [x, y, z, 0] one 256-bit load + the coefficient (8 B)
//   v4: v0 with int32 connectivity
//   v5: v1 with int32 connectivity
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gather_probe gather_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ void ld256(const double* p, double& a, double& b, double& c, double& d) {
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}

template <int V, typename I>
__global__ void __launch_bounds__(256) probe(const I* __restrict__ cells, const double* __restrict__ xyz,
                                             const double* __restrict__ u, const double* __restrict__ rows,
                                             double* __restrict__ out, int64_t n) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
    int64_t id[4];
    if constexpr (sizeof(I) == 8) {
      const longlong2 a = reinterpret_cast<const longlong2*>(cells)[2 * c];
      const longlong2 b = reinterpret_cast<const longlong2*>(cells)[2 * c + 1];
      id[0] = a.x; id[1] = a.y; id[2] = b.x; id[3] = b.y;
    } else {
      const int4 a = reinterpret_cast<const int4*>(cells)[c];
      id[0] = a.x; id[1] = a.y; id[2] = a.z; id[3] = a.w;
    }
    double X[4][3], f[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      if constexpr (V == 0) {
        X[b][0] = __ldg(xyz + id[b] * 3); X[b][1] = __ldg(xyz + id[b] * 3 + 1); X[b][2] = __ldg(xyz + id[b] * 3 + 2);
        f[b] = __ldg(u + id[b]);
      } else if constexpr (V == 1) {
        ld256(rows + id[b] * 4, X[b][0], X[b][1], X[b][2], f[b]);
      } else if constexpr (V == 2) {
        const double2 p = __ldg(reinterpret_cast<const double2*>(rows + id[b] * 4));
        const double2 q = __ldg(reinterpret_cast<const double2*>(rows + id[b] * 4) + 1);
        X[b][0] = p.x; X[b][1] = p.y; X[b][2] = q.x; f[b] = q.y;
      } else {
        double pad;
        ld256(rows + id[b] * 4, X[b][0], X[b][1], X[b][2], pad);
        f[b] = __ldg(u + id[b]) + pad;
      }
    }
    double s = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) s += (X[b][0] - X[0][0]) * (X[b][1] + X[b][2]) * f[b];
    out[c] = s;
  }
}

int main() {
  const int n = 56, m = n + 1;
  const int64_t nc = 6LL * n * n * n, nv = (int64_t)m * m * m;
  std::vector<int64_t> cells(nc * 4);
  const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  int64_t k = 0;
  for (int cx = 0; cx < n; ++cx)
    for (int cy = 0; cy < n; ++cy)
      for (int cz = 0; cz < n; ++cz)
        for (int t = 0; t < 6; ++t) {
          int p[3] = {cx, cy, cz};
          auto id = [&]() { return ((int64_t)p[2] * m + p[1]) * m + p[0]; };
          cells[k++] = id();
          for (int s = 0; s < 3; ++s) { p[perms[t][s]]++; cells[k++] = id(); }
        }
  std::vector<int> cells32(cells.begin(), cells.end());
  std::vector<double> xyz(nv * 3), u(nv), rows(nv * 4);
  for (int64_t v = 0; v < nv; ++v) {
    for (int i = 0; i < 3; ++i) xyz[v * 3 + i] = (double)((v / (i == 0 ? 1 : i == 1 ? m : m * m)) % m) / n;
    u[v] = 0.001 * (v % 997);
    for (int i = 0; i < 3; ++i) rows[v * 4 + i] = xyz[v * 3 + i];
    rows[v * 4 + 3] = u[v];
  }
  int64_t *d_cells; int *d_cells32; double *d_xyz, *d_u, *d_rows, *d_out;
  const int SETS = 4;  // rotating connectivity copies (> L2 together)
  CK(cudaMalloc(&d_cells, SETS * nc * 32)); CK(cudaMalloc(&d_cells32, SETS * nc * 16));
  CK(cudaMalloc(&d_xyz, nv * 24)); CK(cudaMalloc(&d_u, nv * 8)); CK(cudaMalloc(&d_rows, nv * 32));
  CK(cudaMalloc(&d_out, SETS * nc * 8));
  for (int s = 0; s < SETS; ++s) {
    CK(cudaMemcpy(d_cells + s * nc * 4, cells.data(), nc * 32, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_cells32 + s * nc * 4, cells32.data(), nc * 16, cudaMemcpyHostToDevice));
  }
  CK(cudaMemcpy(d_xyz, xyz.data(), nv * 24, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_u, u.data(), nv * 8, cudaMemcpyHostToDevice));
  // v3 reads rows' 4th entry as padding: zero it in a copy
  double* d_pad; CK(cudaMalloc(&d_pad, nv * 32));
  {
    std::vector<double> pad(rows); for (int64_t v = 0; v < nv; ++v) pad[v * 4 + 3] = 0; 
    CK(cudaMemcpy(d_pad, pad.data(), nv * 32, cudaMemcpyHostToDevice));
  }
  CK(cudaMemcpy(d_rows, rows.data(), nv * 32, cudaMemcpyHostToDevice));
  int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int grid = sms * 8, reps = 40;
  const char* names[6] = {"v0 3x8B coords + 8B coef, int64 conn", "v1 packed [x,y,z,u] 256-bit, int64 conn",
                          "v2 packed 2x128-bit, int64 conn", "v3 padded coords 256-bit + 8B coef, int64 conn",
                          "v0 with int32 conn", "v1 with int32 conn"};
  for (int v = 0; v < 6; ++v) {
    auto launch = [&](int s) {
      const int64_t* c64 = d_cells + (s % SETS) * nc * 4;
      const int* c32 = d_cells32 + (s % SETS) * nc * 4;
      double* o = d_out + (s % SETS) * nc;
      switch (v) {
        case 0: probe<0><<<grid, 256>>>(c64, d_xyz, d_u, d_rows, o, nc); break;
        case 1: probe<1><<<grid, 256>>>(c64, d_xyz, d_u, d_rows, o, nc); break;
        case 2: probe<2><<<grid, 256>>>(c64, d_xyz, d_u, d_rows, o, nc); break;
        case 3: probe<3><<<grid, 256>>>(c64, d_xyz, d_u, d_pad, o, nc); break;
        case 4: probe<0><<<grid, 256>>>(c32, d_xyz, d_u, d_rows, o, nc); break;
        case 5: probe<1><<<grid, 256>>>(c32, d_xyz, d_u, d_rows, o, nc); break;
      }
    };
    for (int s = 0; s < 8; ++s) launch(s);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int s = 0; s < reps; ++s) launch(s);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double us = ms * 1e3 / reps;
    const double bytes = nc * ((v >= 4 ? 16 : 32) + 8);
    printf("%-48s %8.2f us  (%6.0f GB/s on conn+out)\n", names[v], us, bytes / us / 1e3);
  }
  return 0;
}
