// kernels.cu -- sm_100a device kernels of the sparse-DNN inference hot path.
//
//   densify      Y0 CSR -> Yt[N][stride] (neuron-major, batch contiguous),
//                dropping empty input rows when compaction is exact  (row a2)
//   layer        Y_{l+1} = clamp(Y_l . W_l + b_l) over groups x batch tiles,
//                with per-row liveness bits                            (row a3)
//   scan/copy    popcount scan of the liveness bits, compaction of the live
//                batch columns (data-dependent, decided on device)      (row a4)
//   readout      ascending category ids / device bitmask / optional Y_L (a6)
//
// Arithmetic of every output (A5/A6, identical to oracle/):
//   acc = +0; for t ascending: acc = __fmaf_rn(Y[k_t], w_t, acc);
//   z = __fadd_rn(acc, b_j);  y = z > 0 ? fminf(z, ymax) : +0.
// The explicit _rn intrinsics forbid the compiler from contracting or
// reassociating; the chain order is the group's ascending source order.
#include <cstdio>

#include "sdnn_internal.h"

namespace sdnn {

#define FULL 0xffffffffu

__device__ __forceinline__ float clampy(float z, float ymax) {
  return z > 0.f ? fminf(z, ymax) : 0.f;
}

template <int VEC>
struct VecT;
template <>
struct VecT<1> {
  using T = float;
  __device__ static T ld(const float *p) { return __ldg(p); }
  __device__ static void st(float *p, const float (&v)[1]) { *p = v[0]; }
  __device__ static void unpack(const T &x, float (&v)[1]) { v[0] = x; }
};
template <>
struct VecT<2> {
  using T = float2;
  __device__ static T ld(const float *p) { return __ldg(reinterpret_cast<const float2 *>(p)); }
  __device__ static void st(float *p, const float (&v)[2]) {
    *reinterpret_cast<float2 *>(p) = make_float2(v[0], v[1]);
  }
  __device__ static void unpack(const T &x, float (&v)[2]) { v[0] = x.x; v[1] = x.y; }
};
template <>
struct VecT<4> {
  using T = float4;
  __device__ static T ld(const float *p) { return __ldg(reinterpret_cast<const float4 *>(p)); }
  __device__ static void st(float *p, const float (&v)[4]) {
    *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
  __device__ static void unpack(const T &x, float (&v)[4]) {
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
  }
};

// Combine per-lane liveness bits (lane covers positions lane*VEC + e of a
// 32*VEC-wide tile) into the tile's VEC 32-bit words and OR them into alive[].
template <int VEC>
__device__ __forceinline__ void publish_alive(uint32_t am, int lane, int64_t tile_pos, int width,
                                              uint32_t *alive) {
  uint32_t bal[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) bal[e] = __ballot_sync(FULL, (am >> e) & 1u);
  if (lane < VEC) {
    uint32_t word = 0;
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const int pos = lane * 32 + q;         // position inside the tile
      const int src_lane = pos / VEC, e = pos % VEC;
      uint32_t b = 0;
#pragma unroll
      for (int ee = 0; ee < VEC; ++ee)
        if (ee == e) b = (bal[ee] >> src_lane) & 1u;
      word |= b << q;
    }
    const int64_t base = tile_pos + lane * 32;
    if (base < width) {
      const int64_t rem = width - base;
      if (rem < 32) word &= (1u << rem) - 1u;
      if (word) atomicOr(&alive[base >> 5], word);
    }
  }
}

// ---------------------------------------------------------------------------
// Layer kernel, uniform weights (every stored value of W_l equals wu).
// One warp per (group, batch tile) item; lanes own VEC consecutive batch
// positions.  The group's chain is evaluated once per position and then
// finished per member column (bias add, clamp, store): members of a group share
// sources AND (uniform) weights, so their chains are the same operation
// sequence on the same operands.
// ---------------------------------------------------------------------------
template <int VEC, bool REG32>
__global__ void __launch_bounds__(256, 2) k_layer_uniform(DevLayer L, const LayerState *__restrict__ st,
                                                        int layer, float *Ya, float *Yb,
                                                        uint32_t *__restrict__ alive,
                                                        int64_t stride, float ymax) {
  using V = VecT<VEC>;
  const LayerState S = st[layer];
  const int width = S.width;
  if (width <= 0) return;
  const float *__restrict__ Yin = S.in ? Yb : Ya;
  float *__restrict__ Yout = S.in ? Ya : Yb;
  constexpr int TILE = 32 * VEC;
  const int tiles = (width + TILE - 1) / TILE;
  const int64_t items = (int64_t)L.ngroups * tiles;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const float w = L.wu;
  for (int64_t it = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < items;
       it += nwarps) {
    const int g = (int)(it / tiles);
    const int tile = (int)(it - (int64_t)g * tiles);
    const int64_t tpos = (int64_t)tile * TILE;
    const int64_t b0 = tpos + lane * VEC;
    const int K = REG32 ? 32 : L.gk[g];
    const int G = L.regular ? L.gmax : L.gg[g];
    float acc[VEC];
#pragma unroll
    for (int e = 0; e < VEC; ++e) acc[e] = 0.f;
    for (int t0 = 0; t0 < K; t0 += 32) {
      const int kk = min(32, K - t0);
      const int mysrc = lane < kk ? (int)L.src[(int64_t)g * L.kmax + t0 + lane] : 0;
      if (REG32) {
        // two batches of 16 independent loads in flight per lane (16 x 16 B)
#pragma unroll
        for (int h = 0; h < 32; h += 16) {
          typename V::T buf[16];
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            const int k = __shfl_sync(FULL, mysrc, h + t);
            buf[t] = V::ld(Yin + (int64_t)k * stride + b0);
          }
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            float v[VEC];
            V::unpack(buf[t], v);
#pragma unroll
            for (int e = 0; e < VEC; ++e) acc[e] = __fmaf_rn(v[e], w, acc[e]);
          }
        }
      } else {
#pragma unroll 4
        for (int t = 0; t < kk; ++t) {
          const int k = __shfl_sync(FULL, mysrc, t);
          float v[VEC];
          V::unpack(V::ld(Yin + (int64_t)k * stride + b0), v);
#pragma unroll
          for (int e = 0; e < VEC; ++e) acc[e] = __fmaf_rn(v[e], w, acc[e]);
        }
      }
    }
    const int mycol = lane < G ? L.col[(int64_t)g * L.gmax + lane] : 0;
    uint32_t am = 0;
    for (int m = 0; m < G; ++m) {
      const int j = __shfl_sync(FULL, mycol, m);
      const float b = __ldg(L.bias + j);
      float y[VEC];
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        y[e] = clampy(__fadd_rn(acc[e], b), ymax);
        am |= (y[e] > 0.f ? 1u : 0u) << e;
      }
      V::st(Yout + (int64_t)j * stride + b0, y);
    }
    publish_alive<VEC>(am, lane, tpos, width, alive);
  }
}

// ---------------------------------------------------------------------------
// Layer kernel, uniform weights, TMA bulk-copy pipeline (sm_90+/sm_100a).
// Persistent CTAs: warp 0 is the producer -- lane t issues one
// cp.async.bulk (global -> shared, completion on an mbarrier) for the group's
// t-th source row segment [tile*T, tile*T + T) -- and warps 1..4 consume: the
// canonical chain over the K_g staged rows (conflict-free LDS.128), then one
// bias-add + clamp + STG.128 per member column.  kStages stages of
// 32 rows x T floats keep ~3 x 64 KB of HBM reads in flight per SM without
// costing registers (the register-staged kernel above is latency bound).
// ---------------------------------------------------------------------------
constexpr int kBulkT = 512;                      // positions per item (2 KB per row)
constexpr int kBulkStages = 3;
constexpr int kBulkConsumers = 4;                // 4 warps x 32 lanes x 4 positions = 512
constexpr int kBulkThreads = 32 * (1 + kBulkConsumers);
constexpr size_t kBulkSmem = (size_t)kBulkStages * 32 * kBulkT * sizeof(float) + 2 * kBulkStages * 8;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_arrive(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      " @!P bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__global__ void __launch_bounds__(kBulkThreads, 1) k_layer_bulk(DevLayer L, const LayerState *__restrict__ st,
                                                               int layer, float *Ya, float *Yb,
                                                               uint32_t *__restrict__ alive,
                                                               int64_t stride, float ymax) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float *stage = reinterpret_cast<float *>(smem_raw);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem_raw + (size_t)kBulkStages * 32 * kBulkT * 4);
  uint64_t *empty = full + kBulkStages;
  const LayerState S = st[layer];
  const int width = S.width;
  if (width <= 0) return;
  const float *__restrict__ Yin = S.in ? Yb : Ya;
  float *__restrict__ Yout = S.in ? Ya : Yb;
  const int tiles = (width + kBulkT - 1) / kBulkT;
  const int64_t items = (int64_t)L.ngroups * tiles;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kBulkStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kBulkConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    // ---------------- producer ----------------
    int s = 0;
    uint32_t ph = 0;
    for (int64_t it = blockIdx.x, n = 0; it < items; it += gridDim.x, ++n) {
      const int g = (int)(it / tiles);
      const int tile = (int)(it - (int64_t)g * tiles);
      const int K = L.regular ? L.kmax : L.gk[g];
      if (n >= kBulkStages) mbar_wait(&empty[s], ph ^ 1);
      if (lane == 0) mbar_expect_tx_arrive(&full[s], (uint32_t)K * kBulkT * 4);
      __syncwarp();
      if (lane < K) {
        const int k = L.src[(int64_t)g * L.kmax + lane];
        bulk_g2s(stage + ((size_t)s * 32 + lane) * kBulkT, Yin + (int64_t)k * stride + (int64_t)tile * kBulkT,
                 kBulkT * 4, &full[s]);
      }
      if (++s == kBulkStages) { s = 0; ph ^= 1; }
    }
  } else {
    // ---------------- consumers ----------------
    const int cw = warp - 1;
    const float w = L.wu;
    int s = 0;
    uint32_t ph = 0;
    for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
      const int g = (int)(it / tiles);
      const int tile = (int)(it - (int64_t)g * tiles);
      const int K = L.regular ? L.kmax : L.gk[g];
      const int G = L.regular ? L.gmax : L.gg[g];
      const int mycol = lane < G ? L.col[(int64_t)g * L.gmax + lane] : 0;
      const float bmy = lane < G ? __ldg(L.bias + mycol) : 0.f;
      mbar_wait(&full[s], ph);
      const float *src = stage + (size_t)s * 32 * kBulkT + cw * 128 + lane * 4;
      float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
      if (K == 32) {
#pragma unroll
        for (int t = 0; t < 32; ++t) {
          const float4 v = *reinterpret_cast<const float4 *>(src + t * kBulkT);
          a0 = __fmaf_rn(v.x, w, a0);
          a1 = __fmaf_rn(v.y, w, a1);
          a2 = __fmaf_rn(v.z, w, a2);
          a3 = __fmaf_rn(v.w, w, a3);
        }
      } else {
        for (int t = 0; t < K; ++t) {
          const float4 v = *reinterpret_cast<const float4 *>(src + t * kBulkT);
          a0 = __fmaf_rn(v.x, w, a0);
          a1 = __fmaf_rn(v.y, w, a1);
          a2 = __fmaf_rn(v.z, w, a2);
          a3 = __fmaf_rn(v.w, w, a3);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == kBulkStages) { s = 0; ph ^= 1; }
      const int64_t tpos = (int64_t)tile * kBulkT + cw * 128;
      float *dst = Yout + tpos + lane * 4;
      uint32_t am = 0;
      for (int m = 0; m < G; ++m) {
        const int j = __shfl_sync(FULL, mycol, m);
        const float b = __shfl_sync(FULL, bmy, m);
        float4 y;
        y.x = clampy(__fadd_rn(a0, b), ymax);
        y.y = clampy(__fadd_rn(a1, b), ymax);
        y.z = clampy(__fadd_rn(a2, b), ymax);
        y.w = clampy(__fadd_rn(a3, b), ymax);
        am |= (y.x > 0.f ? 1u : 0u) | (y.y > 0.f ? 2u : 0u) | (y.z > 0.f ? 4u : 0u) | (y.w > 0.f ? 8u : 0u);
        *reinterpret_cast<float4 *>(dst + (int64_t)j * stride) = y;
      }
      publish_alive<4>(am, lane, tpos, width, alive);
    }
  }
}

// ---------------------------------------------------------------------------
// Layer kernel, per-slot weights.  Sources of the group are loaded once into
// registers (K_g <= 32) and every member runs its own chain with its own
// weights (warp-uniform loads, L1-resident).  K_g > 32 falls back to reloading
// the sources per member (L1 hits).
// ---------------------------------------------------------------------------
template <int VEC>
__global__ void __launch_bounds__(256) k_layer_general(DevLayer L, const LayerState *__restrict__ st,
                                                        int layer, float *Ya, float *Yb,
                                                        uint32_t *__restrict__ alive,
                                                        int64_t stride, float ymax) {
  using V = VecT<VEC>;
  const LayerState S = st[layer];
  const int width = S.width;
  if (width <= 0) return;
  const float *__restrict__ Yin = S.in ? Yb : Ya;
  float *__restrict__ Yout = S.in ? Ya : Yb;
  constexpr int TILE = 32 * VEC;
  const int tiles = (width + TILE - 1) / TILE;
  const int64_t items = (int64_t)L.ngroups * tiles;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t it = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < items;
       it += nwarps) {
    const int g = (int)(it / tiles);
    const int tile = (int)(it - (int64_t)g * tiles);
    const int64_t tpos = (int64_t)tile * TILE;
    const int64_t b0 = tpos + lane * VEC;
    const int K = L.gk[g];
    const int G = L.gg[g];
    const uint16_t *gsrc = L.src + (int64_t)g * L.kmax;
    const int mycol = lane < G ? L.col[(int64_t)g * L.gmax + lane] : 0;
    uint32_t am = 0;
    if (K <= 32) {
      const int mysrc = lane < K ? (int)gsrc[lane] : 0;
      float v[32][VEC];
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        const int k = __shfl_sync(FULL, mysrc, t);
        if (t < K) {
          V::unpack(V::ld(Yin + (int64_t)k * stride + b0), v[t]);
        } else {
#pragma unroll
          for (int e = 0; e < VEC; ++e) v[t][e] = 0.f;
        }
      }
      for (int m = 0; m < G; ++m) {
        const int j = __shfl_sync(FULL, mycol, m);
        const float *wv = L.val + ((int64_t)g * L.gmax + m) * L.kmax;
        float acc[VEC];
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc[e] = 0.f;
#pragma unroll
        for (int t = 0; t < 32; ++t) {
          if (t < K) {
            const float wt = __ldg(wv + t);
#pragma unroll
            for (int e = 0; e < VEC; ++e) acc[e] = __fmaf_rn(v[t][e], wt, acc[e]);
          }
        }
        const float b = __ldg(L.bias + j);
        float y[VEC];
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          y[e] = clampy(__fadd_rn(acc[e], b), ymax);
          am |= (y[e] > 0.f ? 1u : 0u) << e;
        }
        V::st(Yout + (int64_t)j * stride + b0, y);
      }
    } else {
      for (int m = 0; m < G; ++m) {
        const int j = __shfl_sync(FULL, mycol, m);
        const float *wv = L.val + ((int64_t)g * L.gmax + m) * L.kmax;
        float acc[VEC];
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc[e] = 0.f;
        for (int t = 0; t < K; ++t) {
          const int k = gsrc[t];
          float v[VEC];
          V::unpack(V::ld(Yin + (int64_t)k * stride + b0), v);
          const float wt = __ldg(wv + t);
#pragma unroll
          for (int e = 0; e < VEC; ++e) acc[e] = __fmaf_rn(v[e], wt, acc[e]);
        }
        const float b = __ldg(L.bias + j);
        float y[VEC];
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          y[e] = clampy(__fadd_rn(acc[e], b), ymax);
          am |= (y[e] > 0.f ? 1u : 0u) << e;
        }
        V::st(Yout + (int64_t)j * stride + b0, y);
      }
    }
    publish_alive<VEC>(am, lane, tpos, width, alive);
  }
}

// ---------------------------------------------------------------------------
// Block-wide exclusive scan helpers (1024 threads).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int64_t block_exclusive_scan(int64_t v, int64_t *total) {
  __shared__ int64_t warp_sums[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[wid] = x;
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    int64_t s = lane < nw ? warp_sums[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(FULL, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nw) warp_sums[lane] = s;      // inclusive
  }
  __syncthreads();
  const int64_t before = wid ? warp_sums[wid - 1] : 0;
  const int64_t incl = x + before;
  *total = warp_sums[(blockDim.x >> 5) - 1];
  __syncthreads();
  return incl - v;
}

// Scan over `words` bitmask words -> wpre (exclusive prefix), returns total.
__device__ int64_t scan_words(const uint32_t *__restrict__ bits, int64_t words, int32_t *wpre) {
  const int64_t per = (words + blockDim.x - 1) / blockDim.x;
  const int64_t w0 = min(words, (int64_t)threadIdx.x * per), w1 = min(words, w0 + per);
  int64_t s = 0;
  for (int64_t q = w0; q < w1; ++q) s += __popc(bits[q]);
  int64_t total;
  int64_t run = block_exclusive_scan(s, &total);
  for (int64_t q = w0; q < w1; ++q) {
    wpre[q] = (int32_t)run;
    run += __popc(bits[q]);
  }
  if (threadIdx.x == 0) wpre[words] = (int32_t)total;
  return total;
}

// ---------------------------------------------------------------------------
// Densify (row a2)
// ---------------------------------------------------------------------------
// keep(i): with compaction, rows without any nonzero stored value are dropped
// (an all-zero Y0 row gives clamp(0 + b) = 0 when every b <= 0 -- invariant I3).
__global__ void k_rowflags(int64_t batch, const int64_t *__restrict__ rowptr,
                           const float *__restrict__ val, int compact, uint32_t *inmask,
                           int64_t words) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < words * 32;
       i += (int64_t)gridDim.x * blockDim.x) {
    bool keep = false;
    if (i < batch) {
      if (!compact) {
        keep = true;
      } else if (val == nullptr) {
        keep = rowptr[i + 1] > rowptr[i];
      } else {
        for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e)
          if (val[e] != 0.f) { keep = true; break; }
      }
    }
    const uint32_t b = __ballot_sync(FULL, keep);
    if ((threadIdx.x & 31) == 0) inmask[i >> 5] = b;
  }
}

__global__ void __launch_bounds__(1024) k_scan_input(const uint32_t *inmask, int64_t words,
                                                     int32_t *wpre, LayerState *st,
                                                     uint32_t *alive0) {
  const int64_t total = scan_words(inmask, words, wpre);
  for (int64_t q = threadIdx.x; q < words; q += blockDim.x) alive0[q] = 0u;
  if (threadIdx.x == 0) {
    LayerState s0;
    s0.in = 0;
    s0.width = (int32_t)total;
    s0.rid = 0;
    s0.compacted = 0;
    st[0] = s0;
  }
}

// warp per input row: scatter its stored values into its (compacted) column
__global__ void k_scatter(int64_t batch, const int64_t *__restrict__ rowptr,
                          const int32_t *__restrict__ idx, const float *__restrict__ val,
                          const uint32_t *__restrict__ inmask, const int32_t *__restrict__ wpre,
                          float *Y0, int32_t *rid0, int64_t stride) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < batch; i += nw) {
    const uint32_t word = inmask[i >> 5];
    if (!((word >> (i & 31)) & 1u)) continue;
    const int64_t pos = wpre[i >> 5] + __popc(word & ((1u << (i & 31)) - 1u));
    if (lane == 0) rid0[pos] = (int32_t)i;
    for (int64_t e = rowptr[i] + lane; e < rowptr[i + 1]; e += 32)
      Y0[(int64_t)idx[e] * stride + pos] = val ? val[e] : 1.0f;
  }
}

// zero-layer networks: category = row with a positive stored value (reading A7)
__global__ void k_y0_positive(int64_t batch, const int64_t *__restrict__ rowptr,
                              const float *__restrict__ val, uint32_t *alive0, int64_t words) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < words * 32;
       i += (int64_t)gridDim.x * blockDim.x) {
    bool pos = false;
    if (i < batch) {
      if (val == nullptr) {
        pos = rowptr[i + 1] > rowptr[i];
      } else {
        for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e)
          if (val[e] > 0.f) { pos = true; break; }
      }
    }
    const uint32_t b = __ballot_sync(FULL, pos);
    if ((threadIdx.x & 31) == 0) alive0[i >> 5] = b;
  }
}

// ---------------------------------------------------------------------------
// Liveness scan + compaction decision (row a4).  Single CTA.
// ---------------------------------------------------------------------------
constexpr int kCompactMin = 128;

__global__ void __launch_bounds__(1024) k_scan_layer(LayerState *st, int layer,
                                                     const uint32_t *alive_cur,
                                                     uint32_t *alive_next, int32_t *wpre,
                                                     int32_t *live, int compact) {
  const LayerState S = st[layer];
  const int64_t words = ((int64_t)S.width + 31) >> 5;
  const int64_t count = scan_words(alive_cur, words, wpre);
  for (int64_t q = threadIdx.x; q < words; q += blockDim.x) alive_next[q] = 0u;
  if (threadIdx.x == 0) {
    live[layer] = (int32_t)count;
    const int64_t dead = S.width - count;
    LayerState n;
    if (compact && dead >= kCompactMin && dead * 16 >= S.width) {
      n.in = S.in;               // layer l's input buffer is free: compact into it
      n.width = (int32_t)count;
      n.rid = 1 - S.rid;
      n.compacted = 1;
    } else {
      n.in = 1 - S.in;
      n.width = S.width;
      n.rid = S.rid;
      n.compacted = 0;
    }
    st[layer + 1] = n;
  }
}

// Move the live batch columns of layer l's output into the free buffer.
__global__ void k_compact(const LayerState *__restrict__ st, int layer, float *Ya, float *Yb,
                          int32_t *ridA, int32_t *ridB, const uint32_t *__restrict__ alive,
                          const int32_t *__restrict__ wpre, int32_t n, int64_t stride) {
  const LayerState N1 = st[layer + 1];
  if (!N1.compacted) return;
  const LayerState S = st[layer];
  const float *__restrict__ src = S.in ? Ya : Yb;   // layer output = Y[1 - S.in]
  float *__restrict__ dst = S.in ? Yb : Ya;         // layer input buffer
  const int32_t *__restrict__ rsrc = S.rid ? ridB : ridA;
  int32_t *__restrict__ rdst = S.rid ? ridA : ridB;
  const int64_t words = ((int64_t)S.width + 31) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t items = (int64_t)(n + 1) * words;   // row n = the row-id vector
  for (int64_t it = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < items; it += nw) {
    const int64_t k = it / words, q = it - k * words;
    const uint32_t bits = alive[q];
    if (!((bits >> lane) & 1u)) continue;
    const int64_t to = wpre[q] + __popc(bits & ((1u << lane) - 1u));
    const int64_t from = q * 32 + lane;
    if (k < n)
      dst[k * stride + to] = src[k * stride + from];
    else
      rdst[to] = rsrc[from];
  }
}

// ---------------------------------------------------------------------------
// Readout (row a6).  Single CTA: ascending ids (positions are in ascending
// original-row order because densify and compaction are stable).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_readout(const LayerState *__restrict__ st, int sidx,
                                                  const uint32_t *__restrict__ alive,
                                                  const int32_t *ridA, const int32_t *ridB,
                                                  int32_t *wpre, int32_t *cats, int32_t *ncat,
                                                  uint32_t *d_alive_out, int32_t *live,
                                                  int live_idx) {
  const LayerState S = st[sidx];
  const int64_t words = ((int64_t)S.width + 31) >> 5;
  const int32_t *rid = S.rid ? ridB : ridA;
  const int64_t total = scan_words(alive, words, wpre);
  __syncthreads();
  for (int64_t q = threadIdx.x; q < words; q += blockDim.x) {
    uint32_t bits = alive[q];
    int64_t o = wpre[q];
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      const int32_t id = rid[q * 32 + b];
      cats[o++] = id;
      if (d_alive_out) atomicOr(&d_alive_out[id >> 5], 1u << (id & 31));
    }
  }
  if (threadIdx.x == 0) {
    *ncat = (int32_t)total;
    if (live_idx >= 0) live[live_idx] = (int32_t)total;
  }
}

// Y_L (neuron-major, positions) -> row-major [batch][n] (rows not present are 0)
__global__ void k_yout(const LayerState *__restrict__ st, int sidx, int final_out,
                       const float *Ya, const float *Yb, const int32_t *ridA,
                       const int32_t *ridB, int32_t n, int64_t stride, float *yout) {
  const LayerState S = st[sidx];
  const int bufsel = final_out ? 1 - S.in : S.in;
  const float *Y = bufsel ? Yb : Ya;
  const int32_t *rid = S.rid ? ridB : ridA;
  const int64_t total = (int64_t)n * S.width;
  for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < total;
       it += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = it / S.width, p = it - j * S.width;
    yout[(int64_t)rid[p] * n + j] = Y[j * stride + p];
  }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
int bulk_stride_quantum() { return kBulkT; }

void configure_kernels() {
  cudaFuncSetAttribute(k_layer_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBulkSmem);
}

void launch_densify(const LaunchCfg &c, const Workspace &w, int32_t n, int64_t batch,
                    const int64_t *rowptr, const int32_t *idx, const float *val, bool compact,
                    cudaStream_t s) {
  const int64_t words = (batch + 31) / 32;
  cudaMemsetAsync(w.Y[0], 0, sizeof(float) * (size_t)n * (size_t)w.stride, s);
  if (words > 0) {
    const int blocks = (int)std::min<int64_t>((words * 32 + 255) / 256, c.sms * 8);
    k_rowflags<<<blocks, 256, 0, s>>>(batch, rowptr, val, compact ? 1 : 0, w.inmask, words);
  }
  k_scan_input<<<1, 1024, 0, s>>>(w.inmask, words, w.wpre, w.st, w.alive[0]);
  if (batch > 0)
    k_scatter<<<c.sms * 8, 256, 0, s>>>(batch, rowptr, idx, val, w.inmask, w.wpre, w.Y[0],
                                        w.rid[0], w.stride);
}

void launch_zero_layers_alive(const Workspace &w, int64_t batch, const int64_t *rowptr,
                              const float *val, cudaStream_t s) {
  const int64_t words = (batch + 31) / 32;
  if (words > 0)
    k_y0_positive<<<(int)std::min<int64_t>((words * 32 + 255) / 256, 148 * 8), 256, 0, s>>>(
        batch, rowptr, val, w.alive[0], words);
}

void launch_layer(const LaunchCfg &c, const Workspace &w, const DevLayer &L, int32_t layer,
                  float ymax, int32_t n, cudaStream_t s) {
  (void)n;
  uint32_t *alive = w.alive[layer & 1];
  if (L.uniform && L.kmax <= 32 && c.bulk) {
    k_layer_bulk<<<c.sms, kBulkThreads, kBulkSmem, s>>>(L, w.st, layer, w.Y[0], w.Y[1], alive,
                                                       w.stride, ymax);
  } else if (L.uniform) {
    if (L.regular && L.kmax == 32)
      k_layer_uniform<4, true><<<c.layer_blocks, 256, 0, s>>>(L, w.st, layer, w.Y[0], w.Y[1],
                                                               alive, w.stride, ymax);
    else
      k_layer_uniform<4, false><<<c.layer_blocks, 256, 0, s>>>(L, w.st, layer, w.Y[0], w.Y[1],
                                                                alive, w.stride, ymax);
  } else {
    k_layer_general<2><<<c.layer_blocks, 256, 0, s>>>(L, w.st, layer, w.Y[0], w.Y[1], alive,
                                                      w.stride, ymax);
  }
}

void launch_scan(const Workspace &w, int32_t layer, bool compact, int32_t n, cudaStream_t s) {
  (void)n;
  k_scan_layer<<<1, 1024, 0, s>>>(w.st, layer, w.alive[layer & 1], w.alive[(layer + 1) & 1],
                                  w.wpre, w.live, compact ? 1 : 0);
}

void launch_compact_copy(const LaunchCfg &c, const Workspace &w, int32_t layer, int32_t n,
                         cudaStream_t s) {
  k_compact<<<c.copy_blocks, 256, 0, s>>>(w.st, layer, w.Y[0], w.Y[1], w.rid[0], w.rid[1],
                                          w.alive[layer & 1], w.wpre, n, w.stride);
}

void launch_readout(const Workspace &w, int32_t last_state, bool after_layer,
                    uint32_t *d_alive_out, int64_t batch, cudaStream_t s) {
  if (d_alive_out) cudaMemsetAsync(d_alive_out, 0, sizeof(uint32_t) * (size_t)((batch + 31) / 32), s);
  k_readout<<<1, 1024, 0, s>>>(w.st, last_state, w.alive[last_state & 1], w.rid[0], w.rid[1],
                               w.wpre, w.cats, w.ncat, d_alive_out, w.live,
                               after_layer ? last_state : -1);
}

void launch_yout(const Workspace &w, int32_t last_state, int32_t n, int64_t batch,
                 float *d_yout, cudaStream_t s) {
  cudaMemsetAsync(d_yout, 0, sizeof(float) * (size_t)n * (size_t)batch, s);
  (void)batch;
  k_yout<<<148 * 4, 256, 0, s>>>(w.st, last_state < 0 ? 0 : last_state, last_state < 0 ? 0 : 1,
                                 w.Y[0], w.Y[1], w.rid[0], w.rid[1], n, w.stride, d_yout);
}

}  // namespace sdnn
