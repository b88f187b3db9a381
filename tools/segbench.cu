// segbench.cu -- microbenchmark for the fused-pass memory pattern (design study,
// not product code): every CTA repeatedly gathers R random rows of T positions
// (T*4-byte segments) of a neuron-major Y[N][stride] (or position-blocked
// Y[B/T][N][T]) into a 64 KB shared tile with cp.async.bulk, then writes the
// tile to R other random rows.  Reports read+write GB/s per (layout, T, store
// path).  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o segbench segbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

constexpr int kTile = 16384;  // floats

template <int T>
__global__ void __launch_bounds__(128, 3) k_seg(const float *Yin, float *Yout, int64_t stride, int N,
                                                 int blocked, int64_t items, int bulk_store, uint32_t salt) {
  constexpr int R = kTile / T;
  extern __shared__ __align__(128) unsigned char smem[];
  float *tile = reinterpret_cast<float *>(smem);
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem + kTile * 4);
  const int tid = threadIdx.x;
  const int64_t tiles = stride / T;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto rowaddr = [&](int64_t it, int r, uint32_t s) -> int64_t {
    const int n = (int)(hash32((uint32_t)(it * R + r) ^ s) % (uint32_t)N);
    const int64_t tl = it % tiles;
    return blocked ? tl * (int64_t)N * T + (int64_t)n * T : (int64_t)n * stride + tl * T;
  };
  auto issue = [&](int64_t it) {
    if (tid == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                   "r"((uint32_t)(R * T * 4)) : "memory");
    __syncwarp();
    for (int r = tid; r < R; r += 128) {
      const float *src = Yin + rowaddr(it, r, salt);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(tile + r * T)), "l"(src), "r"((uint32_t)(T * 4)), "r"(smem_u32(bar)) : "memory");
    }
  };
  uint32_t ph = 0;
  if (blockIdx.x < items) issue(blockIdx.x);
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x, ph ^= 1u) {
    asm volatile("{\n .reg .pred P;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
                 " @!P bra W_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(ph) : "memory");
    if (bulk_store) {
      for (int r = tid; r < R; r += 128) {
        float *dst = Yout + rowaddr(it, r, salt ^ 0x9e3779b9u);
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                     "r"(smem_u32(tile + r * T)), "r"((uint32_t)(T * 4)) : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    } else {
      // warp w stores rows w, w+4, ...; lane covers 4 floats, T/128 vectors per row-lane
      const int warp = tid >> 5, lane = tid & 31;
      for (int r = warp; r < R; r += 4) {
        float *dst = Yout + rowaddr(it, r, salt ^ 0x9e3779b9u);
        for (int p = lane * 4; p < T; p += 128)
          *reinterpret_cast<float4 *>(dst + p) = *reinterpret_cast<const float4 *>(tile + r * T + p);
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (it + gridDim.x < items) issue(it + gridDim.x);
  }
}

// sub-warp store variant for T < 128 (lanes split over rows)
template <int T>
__global__ void __launch_bounds__(128, 3) k_seg_small(const float *Yin, float *Yout, int64_t stride, int N,
                                                       int blocked, int64_t items, uint32_t salt) {
  constexpr int R = kTile / T;
  constexpr int LPR = T / 4, RPW = 32 / LPR;
  extern __shared__ __align__(128) unsigned char smem[];
  float *tile = reinterpret_cast<float *>(smem);
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem + kTile * 4);
  const int tid = threadIdx.x;
  const int64_t tiles = stride / T;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto rowaddr = [&](int64_t it, int r, uint32_t s) -> int64_t {
    const int n = (int)(hash32((uint32_t)(it * R + r) ^ s) % (uint32_t)N);
    const int64_t tl = it % tiles;
    return blocked ? tl * (int64_t)N * T + (int64_t)n * T : (int64_t)n * stride + tl * T;
  };
  auto issue = [&](int64_t it) {
    if (tid == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                   "r"((uint32_t)(R * T * 4)) : "memory");
    __syncwarp();
    for (int r = tid; r < R; r += 128) {
      const float *src = Yin + rowaddr(it, r, salt);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(tile + r * T)), "l"(src), "r"((uint32_t)(T * 4)), "r"(smem_u32(bar)) : "memory");
    }
  };
  uint32_t ph = 0;
  if (blockIdx.x < items) issue(blockIdx.x);
  const int warp = tid >> 5, lane = tid & 31, sub = lane / LPR, l2 = lane % LPR;
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x, ph ^= 1u) {
    asm volatile("{\n .reg .pred P;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
                 " @!P bra W_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(ph) : "memory");
    for (int r = warp * RPW + sub; r < R; r += 4 * RPW) {
      float *dst = Yout + rowaddr(it, r, salt ^ 0x9e3779b9u);
      *reinterpret_cast<float4 *>(dst + l2 * 4) = *reinterpret_cast<const float4 *>(tile + r * T + l2 * 4);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (it + gridDim.x < items) issue(it + gridDim.x);
  }
}

template <int T>
void run(float *a, float *b, int64_t stride, int N, int sms) {
  const size_t smem = kTile * 4 + 16;
  cudaFuncSetAttribute(k_seg<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_seg_small<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t items = (int64_t)sms * 3 * 120;  // 120 items per CTA
  const double bytes = 2.0 * items * kTile * 4;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int blocked = 0; blocked < 2; ++blocked)
    for (int mode = 0; mode < 2; ++mode) {
      float best = 1e30f;
      for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0);
        if (mode == 1)
          k_seg<T><<<sms * 3, 128, smem>>>(a, b, stride, N, blocked, items, 1, 0x1234u + rep);
        else if (T >= 128)
          k_seg<T><<<sms * 3, 128, smem>>>(a, b, stride, N, blocked, items, 0, 0x1234u + rep);
        else
          k_seg_small<T><<<sms * 3, 128, smem>>>(a, b, stride, N, blocked, items, 0x1234u + rep);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      cudaError_t err = cudaGetLastError();
      printf("T=%4d seg=%5d B layout=%s store=%s : %7.1f GB/s  %s\n", T, T * 4, blocked ? "blocked" : "neuron ",
             mode ? "bulk" : "stg ", bytes / best / 1e6, err == cudaSuccess ? "" : cudaGetErrorString(err));
    }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int N = 65536;
  const int64_t stride = 61440 + 1024;  // product skew; divisible by every T
  float *a, *b;
  if (cudaMalloc(&a, (size_t)N * stride * 4) || cudaMalloc(&b, (size_t)N * stride * 4)) {
    printf("alloc failed\n");
    return 1;
  }
  cudaMemset(a, 0, (size_t)N * stride * 4);
  cudaMemset(b, 0, (size_t)N * stride * 4);
  run<32>(a, b, stride, N, sms);
  run<64>(a, b, stride, N, sms);
  run<128>(a, b, stride, N, sms);
  run<256>(a, b, stride, N, sms);
  run<512>(a, b, stride, N, sms);
  return 0;
}
