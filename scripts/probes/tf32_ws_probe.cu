// Bring-up probes for the warp-specialised tcgen05 gemm stage (GRU group):
//   mode 0: does kind::tf32 truncate or round raw fp32 operands?
//   mode 1: TMA (cp.async.bulk.tensor, SWIZZLE_128B) loads of row-major
//           [64][64] fp32 tiles straight into UMMA layouts -- A K-major,
//           B MN-major (LBO = 8 KB between the two 32-column boxes,
//           SBO = 1 KB between 8-row groups) -- and a 3xTF32 product
//           D = Ah.Bh + Ah.Bl + Al.Bh, lo parts computed in place of layout;
//   mode 2: the tcgen05.ld.16x256b fragment map (which TMEM lane / column
//           each thread's registers hold).
// nvcc -gencode arch=compute_100a,code=sm_100a -o tf32_ws_probe tf32_ws_probe.cu -lcuda
#include <cuda.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../../paper_1911_11576_b200/csrc/device/stitch_device.cuh"
using namespace stitch_dev;

struct alignas(64) TmaDesc {
  unsigned long long v[16];
};

__device__ __forceinline__ void tma_load_3d(void* dst, const TmaDesc* tm, int c0, int c1, int c2, u64* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_addr(dst)),
      "l"(reinterpret_cast<u64>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ u64 desc(u32 saddr, u32 lbo, u32 sbo, u32 layout = 2) {
  return static_cast<u64>((saddr >> 4) & 0x3FFFu) | (static_cast<u64>((lbo >> 4) & 0x3FFFu) << 16) |
         (static_cast<u64>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (static_cast<u64>(layout) << 61);
}
// kind::tf32, D f32, M = 64, N = 64; b_major: 0 K-major, 1 MN-major
__host__ __device__ constexpr u32 idesc(u32 b_major) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (b_major << 16) | ((64u >> 3) << 17) | ((64u >> 4) << 24);
}

__device__ void ld32x32(u32 taddr, u32* r) {
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

// D (M=64, 64 columns at tmem) -> out[64][64] (4 warps)
__device__ void store_d(u32 tmem, float* out) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (w >= 4) return;
  for (int half = 0; half < 2; ++half) {
    u32 r[32];
    ld32x32(tmem + ((u32)(32 * w) << 16) + 32 * half, r);
    if (lane < 16)
      for (int c = 0; c < 32; ++c) out[(16 * w + lane) * 64 + 32 * half + c] = __uint_as_float(r[c]);
  }
}

__global__ void __launch_bounds__(128) probe(int mode, const __grid_constant__ TmaDesc tmA,
                                             const __grid_constant__ TmaDesc tmB, float* out, u32* map,
                                             u32 blbo, u32 bsbo, u32 bmajor) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* A = sm;             // 16 KB raw (2 k-boxes of 8 KB)
  unsigned char* B = sm + 16384;     // 16 KB raw (2 n-boxes of 8 KB)
  unsigned char* Al = sm + 32768;    // 16 KB lo
  unsigned char* Bl = sm + 49152;    // 16 KB lo
  u64* bar = reinterpret_cast<u64*>(sm + 65536);
  u64* mbar = bar + 1;
  u32* slot = reinterpret_cast<u32*>(sm + 65536 + 64);
  const int t = threadIdx.x;
  if (t == 0) {
    mbar_init(bar, 1);
    mbar_init(mbar, 1);
  }
  const u32 tmem = tc::alloc(slot, 64);
  if (mode == 0) {
    // A[m][k] = k == 0 ? 1 + m 2^-13 : 0 (K-major SW128, box 0 only matters);
    // B[k][n] = k == 0 ? 1 : 0 (K-major: row n, element k)
    for (int i = t; i < 4096; i += blockDim.x) {
      reinterpret_cast<float*>(A)[i] = 0.f;
      reinterpret_cast<float*>(B)[i] = 0.f;
    }
    __syncthreads();
    for (int m = t; m < 64; m += blockDim.x) {
      // element k = 0 of row m: chunk 0 -> swizzled chunk (0 ^ (m & 7))
      reinterpret_cast<float*>(A + (m >> 3) * 1024 + (m & 7) * 128 + ((m & 7) << 4))[0] = 1.f + m * exp2f(-13.f);
      reinterpret_cast<float*>(B + (m >> 3) * 1024 + (m & 7) * 128 + ((m & 7) << 4))[0] = 1.f;
    }
    tc::publish_operands();
    if (t == 0) {
      for (int kk = 0; kk < 8; ++kk)
        tc::mma_tf32(tmem, desc(smem_addr(A) + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024),
                     desc(smem_addr(B) + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024), idesc(0), kk != 0);
      tc::commit(mbar);
    }
    mbar_wait(mbar, 0);
    tc::fence_after();
    store_d(tmem, out);
  } else if (mode == 1) {
    if (t == 0) {
      mbar_expect_tx(bar, 32768);
      tma_load_3d(A, &tmA, 0, 0, 0, bar);
      tma_load_3d(A + 8192, &tmA, 32, 0, 0, bar);
      tma_load_3d(B, &tmB, 0, 0, 0, bar);
      tma_load_3d(B + 8192, &tmB, 32, 0, 0, bar);
    }
    mbar_wait(bar, 0);
    // lo = x - tf32(x): same offsets, layout-agnostic
    for (int i = t; i < 4096; i += blockDim.x) {
      const float a = reinterpret_cast<const float*>(A)[i], b = reinterpret_cast<const float*>(B)[i];
      reinterpret_cast<float*>(Al)[i] = a - __uint_as_float(__float_as_uint(a) & 0xffffe000u);
      reinterpret_cast<float*>(Bl)[i] = b - __uint_as_float(__float_as_uint(b) & 0xffffe000u);
    }
    tc::publish_operands();
    if (t == 0) {
      const unsigned char* as[3] = {A, A, Al};
      const unsigned char* bs[3] = {B, Bl, B};
      for (int p = 0; p < 3; ++p)
        for (int kk = 0; kk < 8; ++kk)
          tc::mma_tf32(tmem, desc(smem_addr(as[p]) + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024),
                       bmajor == 2 ? desc(smem_addr(bs[p]) + kk * 1024, blbo, bsbo, 1)
                       : bmajor ? desc(smem_addr(bs[p]) + kk * 1024, blbo, bsbo)
                              : desc(smem_addr(bs[p]) + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024),
                       idesc(bmajor ? 1 : 0), (p | kk) != 0);
      tc::commit(mbar);
    }
    mbar_wait(mbar, 0);
    tc::fence_after();
    if (bmajor == 7) {  // dump raw smem A then B
      for (int i = t; i < 4096; i += blockDim.x) out[i] = reinterpret_cast<const float*>(A)[i];
      for (int i = t; i < 4096; i += blockDim.x) out[4096 + i] = reinterpret_cast<const float*>(B)[i];
    } else {
      store_d(tmem, out);
    }
  } else {
    // st 32x32b: TMEM lane L, column c holds L * 1000 + c; ld 16x256b.x1 at
    // lane base 32w, column 0: record what each thread got
    const int w = t >> 5, lane = t & 31;
    for (int c0 = 0; c0 < 64; c0 += 32) {
      u32 v[32];
      for (int c = 0; c < 32; ++c) v[c] = (32 * w + lane) * 1000 + c0 + c;
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
          "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(tmem + ((u32)(32 * w) << 16) + c0),
          "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
          "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
          "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
          "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    __syncthreads();
    u32 r[4];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(tmem + ((u32)(32 * w) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 4; ++j) map[t * 4 + j] = r[j];
  }
  tc::dealloc(tmem, 64);
}

static TmaDesc make_map(CUdeviceptr base, int batch, CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
  TmaDesc d;
  cuuint64_t dims[3] = {64, 64, (cuuint64_t)batch};
  cuuint64_t strides[2] = {256, 16384};
  cuuint32_t box[3] = {32, 64, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = cuTensorMapEncodeTiled(reinterpret_cast<CUtensorMap*>(&d), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                                      reinterpret_cast<void*>(base), dims, strides, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("tensor map encode failed %d\n", (int)r);
    exit(1);
  }
  return d;
}

int main() {
  float *dA, *dB, *dOut;
  u32* dMap;
  std::vector<float> A(4096), B(4096), out(4096);
  srand(3);
  for (auto& x : A) x = (float)(rand() / (double)RAND_MAX * 2 - 1);
  for (auto& x : B) x = (float)(rand() / (double)RAND_MAX * 2 - 1);
  cudaMalloc(&dA, 16384);
  cudaMalloc(&dB, 16384);
  cudaMalloc(&dOut, 16384);
  cudaMalloc(&dMap, 128 * 4 * 4);
  cudaMemcpy(dA, A.data(), 16384, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), 16384, cudaMemcpyHostToDevice);
  TmaDesc tA = make_map((CUdeviceptr)dA, 1), tB = make_map((CUdeviceptr)dB, 1);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  // mode 0
  probe<<<1, 128, 70000>>>(0, tA, tB, dOut, dMap, 0, 0, 0);
  if (cudaDeviceSynchronize() != cudaSuccess) { printf("mode0 failed: %s\n", cudaGetErrorString(cudaGetLastError())); return 1; }
  cudaMemcpy(out.data(), dOut, 16384, cudaMemcpyDeviceToHost);
  int trunc_ok = 0, rn_ok = 0;
  for (int m = 0; m < 64; ++m) {
    const double v = 1.0 + m * std::ldexp(1.0, -13);
    const double tr = std::floor(v * 1024) / 1024, rn = std::nearbyint(v * 1024) / 1024;
    trunc_ok += out[m * 64 + 5] == (float)tr;
    rn_ok += out[m * 64 + 5] == (float)rn;
  }
  printf("mode0 tf32 operand conversion: matches truncation %d/64, round-to-nearest %d/64  (D[7][5]=%.9g)\n", trunc_ok,
         rn_ok, out[7 * 64 + 5]);
  // mode 1 variants: (lbo, sbo, b_major); b_major 7 = dump smem after TMA
  std::vector<float> big(8192);
  cudaMalloc(&dOut, 32768);
  probe<<<1, 128, 70000>>>(1, tA, tB, dOut, dMap, 0, 0, 7);
  if (cudaDeviceSynchronize() != cudaSuccess) { printf("dump failed\n"); return 1; }
  cudaMemcpy(big.data(), dOut, 32768, cudaMemcpyDeviceToHost);
  {
    // expected SW128 placement of A[m][k] (box kb = k/32): kb*2048 + m*32 + ((k%32/4) ^ (m%8))*4 + k%4 (floats)
    int okA = 0, okB = 0;
    for (int m = 0; m < 64; ++m)
      for (int k = 0; k < 64; ++k) {
        const int kb = k / 32, kc = (k % 32) / 4;
        const int off = kb * 2048 + m * 32 + ((kc ^ (m % 8)) * 4) + k % 4;
        okA += big[off] == A[m * 64 + k];
        okB += big[4096 + off] == B[m * 64 + k];
      }
    printf("TMA dump: A matches SW128 placement %d/4096, B %d/4096; A[0]=%g smem[0]=%g\n", okA, okB, A[0], big[0]);
  }
  // B loaded with the 128B swizzle of 32-byte atoms: dump and decode
  TmaDesc tB32 = make_map((CUdeviceptr)dB, 1, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  probe<<<1, 128, 70000>>>(1, tA, tB32, dOut, dMap, 0, 0, 7);
  cudaDeviceSynchronize();
  cudaMemcpy(big.data(), dOut, 32768, cudaMemcpyDeviceToHost);
  printf("ATOM_32B dump, rows 0..8 (k), element position of B[k][n] for n = 0,4,8,...,28 (in floats within the row):\n");
  for (int k = 0; k < 9; ++k) {
    printf("  k=%d:", k);
    for (int n = 0; n < 32; n += 4) {
      int pos = -1;
      for (int q = 0; q < 32; ++q)
        if (big[4096 + k * 32 + q] == B[k * 64 + n]) pos = q;
      printf(" %2d", pos);
    }
    printf("\n");
  }
  tB = tB32;
  const unsigned variants[][3] = {{8192, 512, 2}, {8192, 1024, 2}, {512, 8192, 2}, {1024, 8192, 2}, {8192, 256, 2}};
  for (auto& v : variants) {
    probe<<<1, 128, 70000>>>(1, tA, tB, dOut, dMap, v[0], v[1], v[2]);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("mode1 failed: %s\n", cudaGetErrorString(cudaGetLastError())); return 1; }
    cudaMemcpy(out.data(), dOut, 16384, cudaMemcpyDeviceToHost);
    double worst = 0, maxerr = 0, worstT = 0;
    for (int m = 0; m < 64; ++m)
      for (int n = 0; n < 64; ++n) {
        double ref = 0, ab = 0, refT = 0;
        for (int k = 0; k < 64; ++k) {
          ref += (double)A[m * 64 + k] * B[k * 64 + n];
          refT += (double)A[m * 64 + k] * B[n * 64 + k];
          ab += std::fabs((double)A[m * 64 + k] * B[k * 64 + n]);
        }
        const double e = std::fabs(out[m * 64 + n] - ref);
        maxerr = std::max(maxerr, e);
        worst = std::max(worst, e / (64 * std::ldexp(1.0, -24) * ab));
        worstT = std::max(worstT, std::fabs(out[m * 64 + n] - refT));
      }
    printf("mode1 lbo=%u sbo=%u b_major=%u: max abs err %.3g (vs A.B^T %.3g), worst err/(K u sum|ab|) %.3g, D[0][0]=%.6f D[5][40]=%.6f\n",
           v[0], v[1], v[2], maxerr, worstT, worst, out[0], out[5 * 64 + 40]);
  }
  // mode 2
  probe<<<1, 128, 70000>>>(2, tA, tB, dOut, dMap, 0, 0, 0);
  if (cudaDeviceSynchronize() != cudaSuccess) { printf("mode2 failed: %s\n", cudaGetErrorString(cudaGetLastError())); return 1; }
  std::vector<u32> map(512);
  cudaMemcpy(map.data(), dMap, 512 * 4, cudaMemcpyDeviceToHost);
  printf("mode2 16x256b.x1 fragment (warp 0): thread: reg -> (lane, col)\n");
  for (int t = 0; t < 4; ++t) {
    printf("  t%02d:", t);
    for (int j = 0; j < 4; ++j) printf(" (%u,%u)", map[t * 4 + j] / 1000, map[t * 4 + j] % 1000);
    printf("\n");
  }
  return 0;
}
