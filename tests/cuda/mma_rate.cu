// tcgen05.mma kind::tf32 issue/execute rate on one SM per CTA (bring-up
// measurement for the gws stage): one thread issues R back-to-back MMAs of
// a shape, commit, wait; reports ns per MMA and effective TFLOP/s per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rate mma_rate.cu
#include <cstdio>
#include "../../paper_1911_11576_b200/csrc/device/stitch_device.cuh"
using namespace stitch_dev;

template <int M, int N, bool TS, bool BMN>
__global__ void __launch_bounds__(128, 1) rate(int R, unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<unsigned long long>(sm_raw) + 1023ull) & ~1023ull);
  u64* bar = reinterpret_cast<u64*>(sm + 131072);
  u32* slot = reinterpret_cast<u32*>(sm + 131072 + 64);
  for (int i = threadIdx.x; i < 131072 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  if (threadIdx.x == 0) mbar_init(bar, 1);
  const u32 tmem = tc::alloc(slot, 512);
  tc::publish_operands();
  constexpr u32 idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((BMN ? 1u : 0u) << 16) | ((N >> 3) << 17) | ((M >> 4) << 24);
  if (threadIdx.x == 0) {
    const u64 da = gws::desc(smem_addr(sm), 16, 1024, 2);
    const u64 db = BMN ? gws::desc(smem_addr(sm + 65536), 8192, 512, 1) : gws::desc(smem_addr(sm + 65536), 16, 1024, 2);
    unsigned long long t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int r = 0; r < R; ++r) {
      const int kk = r & 7;
      if (TS)
        gws::mma_tf32_ts(tmem, tmem + 256 + 8 * kk, db + static_cast<u64>(kk * 64), idesc);
      else
        tc::mma_tf32(tmem, da + static_cast<u64>(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4), db + static_cast<u64>(kk * 64), idesc, r != 0);
    }
    tc::commit(bar);
    mbar_wait(bar, 0);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (blockIdx.x == 0) *out = t1 - t0;
  }
  tc::dealloc(tmem, 512);
}

template <int M, int N, bool TS, bool BMN>
void go(const char* name, int grid) {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  const int smem = 131072 + 2048;
  cudaFuncSetAttribute(rate<M, N, TS, BMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int R = 4096;
  rate<M, N, TS, BMN><<<grid, 128, smem>>>(R, d);
  rate<M, N, TS, BMN><<<grid, 128, smem>>>(R, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long ns;
  cudaMemcpy(&ns, d, 8, cudaMemcpyDeviceToHost);
  const double per = (double)ns / R;
  printf("%-28s grid %3d: %.1f ns / MMA (%.0f clk at 1.965 GHz), %.1f TFLOP/s per SM  %s\n", name, grid, per, per * 1.965,
         2.0 * M * N * 8 / per / 1e3, cudaGetErrorString(e));
}

int main() {
  for (int grid : {1, 148}) {
    go<128, 128, false, true>("M128 N128 SS (B MN-major)", grid);
    go<128, 128, true, true>("M128 N128 TS (B MN-major)", grid);
    go<128, 128, false, false>("M128 N128 SS (B K-major)", grid);
    go<128, 256, false, false>("M128 N256 SS (B K-major)", grid);
    go<128, 64, false, false>("M128 N64 SS (B K-major)", grid);
    go<64, 64, false, false>("M64 N64 SS (B K-major)", grid);
  }
  return 0;
}
