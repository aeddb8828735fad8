// Microbenchmark: latency of a dependent FP64 add chain on sm_100a, from registers and
// from shared memory (the serial in-group fold of the TTV kernels is bound by it).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench_dadd tools/ubench_dadd.cu
#include <cstdio>

__global__ void chain_reg(double* out, long long* cyc, int n) {
  double a = out[0], b = out[1];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    a = __dadd_rn(a, b);
    a = __dadd_rn(a, b);
    a = __dadd_rn(a, b);
    a = __dadd_rn(a, b);
  }
  long long t1 = clock64();
  out[2] = a;
  cyc[0] = t1 - t0;
}

__global__ void chain_smem(double* out, long long* cyc, int n, int unroll8) {
  __shared__ double s[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = out[0] * i;
  __syncthreads();
  if (threadIdx.x) return;
  double acc = 0.0;
  long long t0 = clock64();
  for (int rep = 0; rep < n; ++rep) {
    if (unroll8) {
      for (int j = 0; j < 2048; j += 8) {
        double v0 = s[j], v1 = s[j + 1], v2 = s[j + 2], v3 = s[j + 3], v4 = s[j + 4], v5 = s[j + 5], v6 = s[j + 6],
               v7 = s[j + 7];
        acc = __dadd_rn(acc, v0); acc = __dadd_rn(acc, v1); acc = __dadd_rn(acc, v2); acc = __dadd_rn(acc, v3);
        acc = __dadd_rn(acc, v4); acc = __dadd_rn(acc, v5); acc = __dadd_rn(acc, v6); acc = __dadd_rn(acc, v7);
      }
    } else {
      for (int j = 0; j < 2048; ++j) acc = __dadd_rn(acc, s[j]);
    }
  }
  long long t1 = clock64();
  out[3] = acc;
  cyc[1] = t1 - t0;
}

int main() {
  double* d;
  long long* c;
  cudaMalloc(&d, 64);
  cudaMalloc(&c, 64);
  double h[4] = {1.0, 1e-3, 0, 0};
  cudaMemcpy(d, h, 32, cudaMemcpyHostToDevice);
  const int n = 1 << 16;
  chain_reg<<<1, 1>>>(d, c, n);
  chain_smem<<<1, 64>>>(d, c, 64, 0);
  long long hc[2];
  cudaMemcpy(hc, c, 16, cudaMemcpyDeviceToHost);
  printf("dadd reg chain: %.2f cycles/add\n", (double)hc[0] / (4.0 * n));
  printf("smem fold (rolled): %.2f cycles/row\n", (double)hc[1] / (64.0 * 2048));
  chain_smem<<<1, 64>>>(d, c, 64, 1);
  cudaMemcpy(hc, c, 16, cudaMemcpyDeviceToHost);
  printf("smem fold (unroll 8): %.2f cycles/row\n", (double)hc[1] / (64.0 * 2048));
  return 0;
}
