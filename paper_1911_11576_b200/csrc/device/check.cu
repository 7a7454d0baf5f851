// Build-time instantiation of the device templates for sm_100a (nvcc -cubin
// -Xptxas -v): catches template errors before the runtime ever sees them and
// records register / shared-memory use in build/device_check.ptxas.txt.
#include "stitch_device.cuh"

using namespace stitch_dev;

extern "C" __global__ void __launch_bounds__(256) check_row_warp(const float* __restrict__ x, float* __restrict__ y,
                                                                 int rows) {
  const int lane = threadIdx.x & 31;
  const long long g = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  for (long long r = g; r < rows; r += (long long)gridDim.x * (blockDim.x >> 5)) {
    float v[8];
    const float4 a = ld4_stream(x + r * 256 + lane * 4);
    const float4 b = ld4_stream(x + r * 256 + 128 + lane * 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    float m = MaxOp::init(), s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) m = fmaxf(m, v[i]);
    m = row_allreduce<32, MaxOp>(m, nullptr);
#pragma unroll
    for (int i = 0; i < 8; ++i) s += (v[i] = expf(v[i] - m));
    s = row_allreduce<32, SumOp>(s, nullptr);
    st4(y + r * 256 + lane * 4, v[0] / s, v[1] / s, v[2] / s, v[3] / s);
    st4(y + r * 256 + 128 + lane * 4, v[4] / s, v[5] / s, v[6] / s, v[7] / s);
  }
}

extern "C" __global__ void __launch_bounds__(256) check_row_cta(const float* __restrict__ x, float* __restrict__ y,
                                                                float* __restrict__ ws, unsigned* __restrict__ sync,
                                                                int rows) {
  extern __shared__ __align__(128) float smem[];
  u64* bar = reinterpret_cast<u64*>(smem + 4096);
  if (threadIdx.x == 0) mbar_init(bar, 1);
  __syncthreads();
  unsigned phase = 0;
  float part = 0.f;
  for (int r = blockIdx.x; r < rows; r += gridDim.x) {
    if (threadIdx.x == 0) {
      mbar_expect_tx(bar, 4096 * 4);
      bulk_g2s(smem, x + (long long)r * 4096, 4096 * 4, bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1u;
    float acc = 0.f;
    for (int i = threadIdx.x; i < 4096; i += 256) acc += smem[i];
    acc = row_allreduce<256, SumOp>(acc, smem + 4100);
    if (threadIdx.x == 0) y[r] = acc;
    part += acc;
    __syncthreads();
  }
  if (threadIdx.x == 0) ws[blockIdx.x] = part;
  grid_barrier(sync);
  if (blockIdx.x == 0 && threadIdx.x == 0) y[rows] = combine_parts<SumOp>(ws, gridDim.x, 1, 0);
}

extern "C" __global__ void __launch_bounds__(256) check_gemm(const float* __restrict__ a, const float* __restrict__ b,
                                                             float* __restrict__ c) {
  extern __shared__ __align__(128) float smem[];
  gemm::run<512, 512, 512, 1, 512, 1, 0, 512, 1, 0>(a, b, c, smem);
}

extern "C" __global__ void __launch_bounds__(256) check_gemm_ragged(const float* __restrict__ a,
                                                                    const float* __restrict__ b, float* __restrict__ c) {
  extern __shared__ __align__(128) float smem[];
  gemm::run<300, 130, 77, 3, 1, 300, 300 * 77, 1, 77, 77 * 130>(a, b, c, smem);
}
