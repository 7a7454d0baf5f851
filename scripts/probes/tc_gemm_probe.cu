// Layout probe for the tcgen05 gemm stage: A = I, B[k][n] = k*64+n (so D
// must equal B), and A[m][k] = m*64+k with B = I (D must equal A). Prints
// mismatches as (m,n): got -> decoded (row,col) of the value found.
#include <cstdio>
#include <vector>
#include "../../paper_1911_11576_b200/csrc/device/stitch_device.cuh"
using namespace stitch_dev;

__global__ void __launch_bounds__(256) probe(const float* A, const float* B, float* D, float* raw) {
  extern __shared__ __align__(1024) unsigned char sm[];
  float* sA = reinterpret_cast<float*>(sm);
  float* sB = sA + 4096;
  float* sD = sB + 4096;
  unsigned char* scratch = sm + 4 * 16384;
  u64* bar = reinterpret_cast<u64*>(sm + 4 * 16384 + 65536);
  u32* slot = reinterpret_cast<u32*>(sm + 4 * 16384 + 65536 + 16);
  if (threadIdx.x == 0) mbar_init(bar, 1);
  const u32 tmem = tc::alloc(slot, 64);
  u32 phase = 0;
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) { sA[i] = A[i]; sB[i] = B[i]; }
  __syncthreads();
  tc::gemm_64x64_tf32x3<64>(sA, sB, sD, scratch, tmem, bar, phase);
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) D[i] = sD[(i / 64) * tc::kDStride + i % 64];
  // raw TMEM dump: warps 0-3, lane quarter w, all 32 lanes, columns 0..63
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (w < 4) {
    for (int c0 = 0; c0 < 64; c0 += 32) {
      u32 r[32];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
            "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
            "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
            "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
          : "r"(tmem + ((u32)(32 * w) << 16) + c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int c = 0; c < 32; ++c) raw[(32 * w + lane) * 64 + c0 + c] = __uint_as_float(r[c]);
    }
  }
  if (threadIdx.x == 0) printf("tmem base 0x%08x phase %u\n", tmem, phase);
  tc::dealloc(tmem, 64);
}

int main() {
  std::vector<float> I(4096, 0.f), V(4096), D(4096);
  for (int i = 0; i < 64; ++i) I[i * 64 + i] = 1.f;
  for (int i = 0; i < 4096; ++i) V[i] = (float)i;
  float *dA, *dB, *dD, *dR;
  std::vector<float> R(128 * 64);
  cudaMalloc(&dA, 16384); cudaMalloc(&dB, 16384); cudaMalloc(&dD, 16384); cudaMalloc(&dR, 128 * 64 * 4);
  const int smem = 4 * 16384 + 65536 + 64;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int test = 0; test < 2; ++test) {
    cudaMemcpy(dA, test == 0 ? I.data() : V.data(), 16384, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, test == 0 ? V.data() : I.data(), 16384, cudaMemcpyHostToDevice);
    probe<<<1, 256, smem>>>(dA, dB, dD, dR);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 2; }
    cudaMemcpy(D.data(), dD, 16384, cudaMemcpyDeviceToHost);
    int bad = 0;
    printf("test %d (%s)\n", test, test == 0 ? "A=I: D should be B" : "B=I: D should be A");
    for (int m = 0; m < 64; ++m)
      for (int n = 0; n < 64; ++n) {
        float g = D[m * 64 + n];
        if (g != (float)(m * 64 + n)) {
          if (bad < 4) {
            int gi = (int)g;
            printf("  (%d,%d): got %.1f -> (%d,%d)\n", m, n, g, gi / 64, gi % 64);
          }
          ++bad;
        }
      }
    printf("  mismatches %d of 4096\n", bad);
    cudaMemcpy(R.data(), dR, R.size() * 4, cudaMemcpyDeviceToHost);
    int nz = 0;
    for (int l = 0; l < 128; ++l)
      for (int c = 0; c < 64; ++c)
        if (R[l * 64 + c] != 0.f) {
          if (nz < 24) printf("  tmem lane %d col %d = %.1f\n", l, c, R[l * 64 + c]);
          ++nz;
        }
    printf("  tmem nonzeros %d\n", nz);
  }
  return 0;
}
