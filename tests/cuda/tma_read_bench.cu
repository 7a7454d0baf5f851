// Read bandwidth of TMA tile streams (bring-up measurement for the gws
// stage): per CTA, one thread streams samples' four 64x64 fp32 tiles
// (box 32 x ROWS) into a NST-deep shared-memory ring and recycles a slot as
// soon as it lands. nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_read_bench tma_read_bench.cu -lcuda
#include <cuda.h>
#include <cstdio>
#include <vector>
#include "../../paper_1911_11576_b200/csrc/device/stitch_device.cuh"
using namespace stitch_dev;

template <int NST, int ROWS>
__global__ void __launch_bounds__(32, 1) tma_only(const __grid_constant__ gws::TmaDesc t0, const __grid_constant__ gws::TmaDesc t1,
                                                  const __grid_constant__ gws::TmaDesc t2, const __grid_constant__ gws::TmaDesc t3,
                                                  long long batch) {
  extern __shared__ unsigned char raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<unsigned long long>(raw) + 1023ull) & ~1023ull);
  u64* full = reinterpret_cast<u64*>(sm + NST * 65536);
  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; ++i) mbar_init(full + i, 1);
    const gws::TmaDesc* t[4] = {&t0, &t1, &t2, &t3};
    int i = 0;
    for (long long s = blockIdx.x; s < batch; s += gridDim.x, ++i) {
      const int st = i % NST;
      if (i >= NST) mbar_wait(full + st, ((i / NST) - 1) & 1);
      mbar_expect_tx(full + st, 65536);
      const u32 base = smem_addr(sm + st * 65536);
      for (int k = 0; k < 4; ++k)
        for (int c = 0; c < 2; ++c)
          for (int g = 0; g < 64 / ROWS; ++g)
            gws::tma_load_3d(base + k * 16384 + c * 8192 + g * ROWS * 128, t[k], 32 * c, ROWS * g, s, full + st);
    }
    for (int j = i - NST; j < i; ++j)
      if (j >= 0) mbar_wait(full + j % NST, (j / NST) & 1);
  }
}

// plain 128-bit loads: every thread streams float4s of the four arrays
__global__ void __launch_bounds__(512) ldg_only(const float4* a, const float4* b, const float4* c, const float4* d,
                                                long long n4, float* sink) {
  float acc = 0.f;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    const float4 x = ld4_stream(reinterpret_cast<const float*>(a + i)), y = ld4_stream(reinterpret_cast<const float*>(b + i));
    const float4 z = ld4_stream(reinterpret_cast<const float*>(c + i)), w = ld4_stream(reinterpret_cast<const float*>(d + i));
    acc += x.x + y.y + z.z + w.w;
  }
  if (acc == 1234.5f) *sink = acc;
}
__global__ void __launch_bounds__(512) copy_only(const float4* a, float4* b, long long n4) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x)
    b[i] = a[i];
}

static gws::TmaDesc make_map(const float* base, long long batch, int rows) {
  gws::TmaDesc d;
  cuuint64_t dims[3] = {64, 64, (cuuint64_t)batch};
  cuuint64_t strides[2] = {256, 16384};
  cuuint32_t box[3] = {32, (cuuint32_t)rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  cuTensorMapEncodeTiled(reinterpret_cast<CUtensorMap*>(&d), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)base, dims,
                         strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return d;
}

template <int NST, int ROWS>
void run(float** d, long long batch, int grid, float* flush) {
  gws::TmaDesc t[4];
  for (int k = 0; k < 4; ++k) t[k] = make_map(d[k], batch, ROWS);
  const int smem = NST * 65536 + 1024 + 64;
  cudaFuncSetAttribute(tma_only<NST, ROWS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9;
  for (int r = 0; r < 10; ++r) {
    cudaMemsetAsync(flush, r, 256 << 20);
    cudaEventRecord(e0);
    tma_only<NST, ROWS><<<grid, 32, smem>>>(t[0], t[1], t[2], t[3], batch);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  printf("stages %d box rows %2d grid %d: %.1f us, %.0f GB/s read  (%s)\n", NST, ROWS, grid, best * 1e3,
         4.0 * batch * 16384 / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const long long batch = 4096;
  float* d[4];
  for (auto& p : d) {
    cudaMalloc(&p, batch * 16384);
    cudaMemset(p, 0, batch * 16384);
  }
  float* flush;
  cudaMalloc(&flush, 256 << 20);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int bpsm : {2, 4, 8}) {
      float best = 1e9;
      for (int r = 0; r < 10; ++r) {
        cudaMemsetAsync(flush, r, 256 << 20);
        cudaEventRecord(e0);
        ldg_only<<<sms * bpsm, 512>>>((float4*)d[0], (float4*)d[1], (float4*)d[2], (float4*)d[3], batch * 1024, flush);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
      }
      printf("ldg.128 4 arrays, %d x 512 thr/SM: %.1f us, %.0f GB/s read\n", bpsm, best * 1e3, 4.0 * batch * 16384 / (best * 1e-3) / 1e9);
      best = 1e9;
      for (int r = 0; r < 10; ++r) {
        cudaMemsetAsync(flush, r, 256 << 20);
        cudaEventRecord(e0);
        copy_only<<<sms * bpsm, 512>>>((float4*)d[0], (float4*)d[1], batch * 1024);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
      }
      printf("copy 67 MB -> 67 MB, %d x 512 thr/SM: %.1f us, %.0f GB/s read+write\n", bpsm, best * 1e3, 2.0 * batch * 16384 / (best * 1e-3) / 1e9);
    }
  }
  run<1, 64>(d, batch, sms, flush);
  run<2, 64>(d, batch, sms, flush);
  run<3, 64>(d, batch, sms, flush);
  run<2, 16>(d, batch, sms, flush);
  run<3, 16>(d, batch, sms, flush);
  return 0;
}
