// Standalone check of stitch_dev::tc::gemm_64x64_tf32x3 (tcgen05 3xTF32):
// batch of D[b] = A[b] @ B[b], 64x64x64, against an fp64 host reference.
// Built by scripts (nvcc -gencode arch=compute_100a,code=sm_100a); prints
// max abs error / bound and exits nonzero on failure.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../../paper_1911_11576_b200/csrc/device/stitch_device.cuh"

using namespace stitch_dev;

__global__ void __launch_bounds__(256) tc_test(const float* A, const float* B, float* D, int batch) {
  extern __shared__ __align__(1024) unsigned char sm[];
  float* sA = reinterpret_cast<float*>(sm);           // 16 KB
  float* sB = sA + 4096;                              // 16 KB
  float* sD = sB + 4096;                              // 17 KB (padded rows)
  unsigned char* scratch = sm + 4 * 16384;            // 64 KB, 1024-aligned
  u64* bar = reinterpret_cast<u64*>(sm + 4 * 16384 + 65536);
  u32* slot = reinterpret_cast<u32*>(sm + 4 * 16384 + 65536 + 16);
  if (threadIdx.x == 0) mbar_init(bar, 1);
  const u32 tmem = tc::alloc(slot, 64);
  u32 phase = 0;
  for (int b = blockIdx.x; b < batch; b += gridDim.x) {
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) {
      sA[i] = A[(long long)b * 4096 + i];
      sB[i] = B[(long long)b * 4096 + i];
    }
    __syncthreads();
    tc::gemm_64x64_tf32x3<64>(sA, sB, sD, scratch, tmem, bar, phase);
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) D[(long long)b * 4096 + i] = sD[(i / 64) * tc::kDStride + i % 64];
    __syncthreads();
  }
  tc::dealloc(tmem, 64);
}

int main() {
  const int batch = 300;
  std::vector<float> A(batch * 4096), B(batch * 4096), D(batch * 4096);
  srand(1);
  for (auto& x : A) x = (rand() / (float)RAND_MAX - 0.5f) * 2.f;
  for (auto& x : B) x = (rand() / (float)RAND_MAX - 0.5f) * 2.f;
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0xff, D.size() * 4);
  const int smem = 4 * 16384 + 65536 + 64;
  cudaFuncSetAttribute(tc_test, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  tc_test<<<148, 256, smem>>>(dA, dB, dD, batch);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 2; }
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double worst = 0, maxerr = 0;
  for (int b = 0; b < batch; ++b)
    for (int m = 0; m < 64; ++m)
      for (int n = 0; n < 64; ++n) {
        double ref = 0, mag = 0;
        for (int k = 0; k < 64; ++k) {
          double p = (double)A[b * 4096 + m * 64 + k] * B[b * 4096 + k * 64 + n];
          ref += p; mag += fabs(p);
        }
        double got = D[b * 4096 + m * 64 + n];
        double err = fabs(got - ref);
        double bound = 64 * 5.96e-8 * mag + 1e-6;
        maxerr = fmax(maxerr, err);
        worst = fmax(worst, err / bound);
      }
  printf("tc_gemm 3xTF32: max abs err %.3g, worst err/bound %.3g\n", maxerr, worst);
  // timing
  cudaEvent_t t0, t1; cudaEventCreate(&t0); cudaEventCreate(&t1);
  cudaEventRecord(t0);
  for (int r = 0; r < 10; ++r) tc_test<<<148, 256, smem>>>(dA, dB, dD, batch);
  cudaEventRecord(t1); cudaEventSynchronize(t1);
  float ms; cudaEventElapsedTime(&ms, t0, t1);
  printf("%.2f us per launch (%d samples)\n", ms * 100, batch);
  return worst <= 1.0 ? 0 : 1;
}
