// tcgen05 bring-up probes: TMEM st/ld round trip, and tf32 MMAs with
// A K-major and B either K-major or MN-major (SW128), on tiny known inputs.
#include <cstdio>
#include <vector>
#include "../../paper_1911_11576_b200/csrc/device/stitch_device.cuh"
using namespace stitch_dev;

__device__ void ld32(u32 taddr, u32* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__global__ void __launch_bounds__(128) probe(int mode, float* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  u64* bar = reinterpret_cast<u64*>(sm + 65536);
  u32* slot = reinterpret_cast<u32*>(sm + 65536 + 16);
  const int t = threadIdx.x, w = t >> 5, lane = t & 31;
  if (t == 0) mbar_init(bar, 1);
  const u32 tmem = tc::alloc(slot, 64);
  if (mode == 0) {
    // st/ld round trip: value = lane*1000 + col
    u32 v[32];
    for (int c = 0; c < 32; ++c) v[c] = __float_as_uint((float)((32 * w + lane) * 1000 + c));
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(tmem + ((u32)(32 * w) << 16)),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
        "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
        "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  } else {
    // A (K-major SW128, 64 rows x 32 tf32): A[m][k] = (k == m % 32) ? 1 : 0 -> D[m][n] = B[m%32][n]
    // B: mode 1 = K-major (N rows x K), mode 2 = MN-major (K rows x N), both encode B[k][n] = k*100 + n (n < 64)
    unsigned char* A = sm;            // 8 KB: 64 rows x 128 B
    unsigned char* B = sm + 16384;    // 8 KB
    for (int i = t; i < 64 * 8; i += blockDim.x) {  // A: 64 rows x 8 chunks
      const int m = i / 8, c = i % 8;
      float4 q;
      float* f = reinterpret_cast<float*>(&q);
      for (int e = 0; e < 4; ++e) f[e] = (c * 4 + e == m % 32) ? 1.f : 0.f;
      *reinterpret_cast<float4*>(A + (m >> 3) * 1024 + (m & 7) * 128 + (((c ^ (m & 7))) << 4)) = q;
    }
    if (mode == 1) {  // K-major B: row n (64 rows), 32 k per row
      for (int i = t; i < 64 * 8; i += blockDim.x) {
        const int n = i / 8, c = i % 8;
        float4 q;
        float* f = reinterpret_cast<float*>(&q);
        for (int e = 0; e < 4; ++e) f[e] = (float)((c * 4 + e) * 100 + n);
        *reinterpret_cast<float4*>(B + (n >> 3) * 1024 + (n & 7) * 128 + (((c ^ (n & 7))) << 4)) = q;
      }
    } else {  // MN-major B: k rows (32), 64 n in 2 panels of 32 (128 B)
      for (int i = t; i < 32 * 16; i += blockDim.x) {
        const int k = i / 16, c4 = i % 16, p = c4 >> 3, c = c4 & 7;
        float4 q;
        float* f = reinterpret_cast<float*>(&q);
        for (int e = 0; e < 4; ++e) f[e] = (float)(k * 100 + c4 * 4 + e);
        *reinterpret_cast<float4*>(B + p * (32 * 128) + (k >> 3) * 1024 + (k & 7) * 128 + (((c ^ (k & 7))) << 4)) = q;
      }
    }
    tc::fence_proxy_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (t == 0) {
      const u32 a0 = smem_addr(A), b0 = smem_addr(B);
      const u32 idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((mode >= 2 ? 1u : 0u) << 16) | ((64u >> 3) << 17) | ((64u >> 4) << 24);
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t ad = tc::sw128_desc(a0 + kk * 32u, 16u, 1024u);
        const uint64_t bd = mode == 1 ? tc::sw128_desc(b0 + kk * 32u, 16u, 1024u)
                            : mode == 2 ? tc::sw128_desc(b0 + kk * 1024u, 32u * 128u, 1024u)
                                        : tc::sw128_desc(b0 + kk * 1024u, 1024u, 32u * 128u);
        tc::mma_tf32(tmem, ad, bd, idesc, kk != 0);
      }
      tc::commit(bar);
    }
    mbar_wait(bar, 0);
    tc::fence_after();
  }
  // dump: out[lane 0..127][col 0..31]
  u32 r[32];
  ld32(tmem + ((u32)(32 * w) << 16), r);
  for (int c = 0; c < 32; ++c) out[(32 * w + lane) * 32 + c] = __uint_as_float(r[c]);
  tc::dealloc(tmem, 64);
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * 32 * 4);
  std::vector<float> h(128 * 32);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 64);
  for (int mode = 0; mode < 4; ++mode) {
    cudaMemset(d, 0, 128 * 32 * 4);
    probe<<<1, 128, 65536 + 64>>>(mode, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("mode %d CUDA error %s\n", mode, cudaGetErrorString(e)); return 2; }
    cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost);
    int nz = 0;
    for (float x : h) nz += x != 0.f;
    printf("mode %d nonzeros %d | lane0: %.0f %.0f %.0f | lane1: %.0f %.0f | lane16: %.0f %.0f | lane32: %.0f %.0f | lane33 %.0f\n",
           mode, nz, h[0], h[1], h[2], h[32], h[33], h[16 * 32], h[16 * 32 + 1], h[32 * 32], h[32 * 32 + 1], h[33 * 32]);
  }
  return 0;
}
