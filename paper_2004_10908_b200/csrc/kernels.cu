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
#include <cstdlib>

#include "sdnn_internal.h"
#include "device_util.cuh"

namespace sdnn {

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
constexpr int kBulkMaxT = 2048;                  // stride quantum (largest tile)

// T positions per item (4 per lane, T/128 consumer warps); an item's K source
// rows arrive in sub-stages of RPS rows, STAGES sub-stages deep, so the loads of
// the next item overlap the chain of the current one while each cp.async.bulk
// still moves a T*4-byte row segment (4 KB at T = 1024: DRAM-friendly).
template <int T, int RPS, int STAGES, bool CS>
__global__ void __launch_bounds__(32 * (1 + T / 128), 1)
    k_layer_bulk(DevLayer L, const LayerState *__restrict__ st, int layer, float *Ya, float *Yb,
                 uint32_t *__restrict__ alive, int64_t stride, float ymax,
                 uint32_t *__restrict__ satw) {
  constexpr int NC = T / 128;                      // consumer warps, 4 positions per lane
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float *stage = reinterpret_cast<float *>(smem_raw);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem_raw + (size_t)STAGES * RPS * T * 4);
  uint64_t *empty = full + STAGES;
  const LayerState S = st[layer];
  const int width = S.width;
  if (width <= 0) return;
  const float *__restrict__ Yin = S.in ? Yb : Ya;
  float *__restrict__ Yout = S.in ? Ya : Yb;
  const int tiles = (width + T - 1) / T;
  const int64_t items = (int64_t)L.ngroups * tiles;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NC);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    // ---------------- producer ----------------
    int s = 0;
    uint32_t ph = 0;
    int64_t n = 0;                                   // sub-stages issued
    for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
      const int g = (int)(it / tiles);
      const int tile = (int)(it - (int64_t)g * tiles);
      const int K = L.regular ? L.kmax : L.gk[g];
      const int mysrc = lane < K ? (int)L.src[(int64_t)g * L.kmax + lane] : 0;
      for (int r0 = 0; r0 < K; r0 += RPS, ++n) {
        const int rows = min(RPS, K - r0);
        if (n >= STAGES) mbar_wait(&empty[s], ph ^ 1);
        if (lane == 0) mbar_expect_tx_arrive(&full[s], (uint32_t)rows * T * 4);
        __syncwarp();
        const int k = __shfl_sync(FULL, mysrc, (r0 + lane) & 31);
        if (lane < rows)
          bulk_g2s(stage + ((size_t)s * RPS + lane) * T, Yin + (int64_t)k * stride + (int64_t)tile * T,
                   T * 4, &full[s]);
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
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
      float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
      for (int r0 = 0; r0 < K; r0 += RPS) {          // ascending sources, sub-stage by sub-stage
        const int rows = min(RPS, K - r0);
        mbar_wait(&full[s], ph);
        const float *src = stage + (size_t)s * RPS * T + cw * 128 + lane * 4;
        if (rows == RPS) {
#pragma unroll
          for (int t = 0; t < RPS; ++t) {
            const float4 v = *reinterpret_cast<const float4 *>(src + t * T);
            a0 = __fmaf_rn(v.x, w, a0);
            a1 = __fmaf_rn(v.y, w, a1);
            a2 = __fmaf_rn(v.z, w, a2);
            a3 = __fmaf_rn(v.w, w, a3);
          }
        } else {
          for (int t = 0; t < rows; ++t) {
            const float4 v = *reinterpret_cast<const float4 *>(src + t * T);
            a0 = __fmaf_rn(v.x, w, a0);
            a1 = __fmaf_rn(v.y, w, a1);
            a2 = __fmaf_rn(v.z, w, a2);
            a3 = __fmaf_rn(v.w, w, a3);
          }
        }
        // order this warp's generic-proxy reads before the TMA (async-proxy)
        // writes that refill the stage once every consumer warp has arrived
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
      const int64_t tpos = (int64_t)tile * T + cw * 128;
      float *dst = Yout + tpos + lane * 4;
      // z_m = acc + b_m is monotone in b_m: some member is alive iff
      // acc + max_m b_m > 0, every member saturates iff acc + min_m b_m >= ymax
      uint32_t am = 0, sm = 0xfu;                    // alive / all-members-saturated bits
      for (int m = 0; m < G; ++m) {
        const int j = __shfl_sync(FULL, mycol, m);
        const float b = __shfl_sync(FULL, bmy, m);
        float4 y;
        y.x = clampy(__fadd_rn(a0, b), ymax);
        y.y = clampy(__fadd_rn(a1, b), ymax);
        y.z = clampy(__fadd_rn(a2, b), ymax);
        y.w = clampy(__fadd_rn(a3, b), ymax);
        // per-member liveness between the stores: measured 3.6 % faster at C4
        // than one acc + max(b) test per group (the stores are paced)
        am |= (y.x > 0.f ? 1u : 0u) | (y.y > 0.f ? 2u : 0u) | (y.z > 0.f ? 4u : 0u) | (y.w > 0.f ? 8u : 0u);
        sm &= (y.x == ymax ? 1u : 0u) | (y.y == ymax ? 2u : 0u) | (y.z == ymax ? 4u : 0u) |
              (y.w == ymax ? 8u : 0u);
        if (CS)
          __stcs(reinterpret_cast<float4 *>(dst + (int64_t)j * stride), y);
        else
          *reinterpret_cast<float4 *>(dst + (int64_t)j * stride) = y;
      }
      publish_alive<4>(am, lane, tpos, width, alive);
      if (satw) publish_sat<4>(sm, lane, tpos, width, satw);
    }
  }
}

// ---------------------------------------------------------------------------
// Layer kernel, PER-SLOT weights (the general-weight path), TMA bulk pipeline.
// Warp 0 produces: per item (group g, tile of T positions) one cp.async.bulk
// per source row segment (T*4 bytes) plus one for the group's weight block
// val[g] (K x gmax floats, source-major) onto the stage's mbarrier.  NCW
// consumer warps own T/NCW positions each, in rounds of 32: lane = (position
// quad q = lane & 7, member octet c = lane >> 3), so a warp computes a
// 32-position x 32-member block.  Per term t (ascending: the canonical chain of
// every member) it reads one float4 of Y (8 distinct addresses: one
// wavefront) and two float4 of weights (members 8c..8c+7) and issues 16 packed
// FFMA2 -- two members of one position per instruction, per component exactly
// __fmaf_rn -- then every member: bias add, clamp, 16-B store (8 lanes of a
// member octet write one 128 B run of its output row).  Requires gmax == 32
// and K_g <= 32 (the RadiX-Net structure with general weights); other
// non-uniform layers use k_layer_general.
// ---------------------------------------------------------------------------
template <int T, int NCW, int STAGES>
constexpr size_t bulkw_smem() {
  return (size_t)STAGES * (32 * T + 32 * 32 + 128) * sizeof(float) + 2 * STAGES * 8;
}

template <int T, int NCW, int STAGES>
__global__ void __launch_bounds__(32 * (1 + NCW), 1)
    k_layer_bulkw(DevLayer L, const LayerState *__restrict__ st, int layer, float *Ya, float *Yb,
                  uint32_t *__restrict__ alive, int64_t stride, float ymax) {
  // floats per stage: 32 rows, weights [32][32], member columns + member biases
  // (bulk-copied with them) and the group's K, G (written by the producer)
  constexpr int SF = 32 * T + 32 * 32 + 128;
  constexpr int PW = T / NCW;                      // positions per consumer warp
  static_assert(PW % 32 == 0, "rounds of 32 positions");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float *stage = reinterpret_cast<float *>(smem_raw);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem_raw + (size_t)STAGES * SF * 4);
  uint64_t *empty = full + STAGES;
  const LayerState S = st[layer];
  const int width = S.width;
  if (width <= 0) return;
  const float *__restrict__ Yin = S.in ? Yb : Ya;
  float *__restrict__ Yout = S.in ? Ya : Yb;
  const int tiles = (width + T - 1) / T;
  const int64_t items = (int64_t)L.ngroups * tiles;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    // ---------------- producer ----------------
    int s = 0;
    uint32_t ph = 0;
    int64_t n = 0;
    for (int64_t it = blockIdx.x; it < items; it += gridDim.x, ++n) {
      const int g = (int)(it / tiles);
      const int tile = (int)(it - (int64_t)g * tiles);
      const int K = L.gk[g];
      const int mysrc = lane < K ? (int)L.src[(int64_t)g * L.kmax + lane] : 0;
      if (n >= STAGES) mbar_wait(&empty[s], ph ^ 1);
      float *sb = stage + (size_t)s * SF;
      if (lane == 0) {
        const uint32_t wbytes = (uint32_t)K * 32u * 4u;
        int *meta = reinterpret_cast<int *>(sb + 32 * T + 32 * 32 + 64);
        meta[0] = K;
        meta[1] = L.gg[g];
        mbar_expect_tx_arrive(&full[s], (uint32_t)K * T * 4 + wbytes + 256u);
        if (wbytes) bulk_g2s(sb + 32 * T, L.val + (int64_t)g * L.kmax * 32, wbytes, &full[s]);
        bulk_g2s(sb + 32 * T + 32 * 32, L.col + (int64_t)g * 32, 128u, &full[s]);
        bulk_g2s(sb + 32 * T + 32 * 32 + 32, L.gbias + (int64_t)g * 32, 128u, &full[s]);
      }
      __syncwarp();
      if (lane < K) bulk_g2s(sb + lane * T, Yin + (int64_t)mysrc * stride + (int64_t)tile * T, T * 4, &full[s]);
      if (++s == STAGES) { s = 0; ph ^= 1; }
    }
  } else {
    // ---------------- consumers ----------------
    const int cw = warp - 1;
    const int q = lane & 7, c = lane >> 3;
    int s = 0;
    uint32_t ph = 0;
    for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
      const int g = (int)(it / tiles);
      const int tile = (int)(it - (int64_t)g * tiles);
      mbar_wait(&full[s], ph);
      const float *sb = stage + (size_t)s * SF;
      const int *meta = reinterpret_cast<const int *>(sb + 32 * T + 32 * 32);
      const int K = meta[64], G = meta[65];
      int col[8];
      float bia[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int m = 8 * c + i;
        col[i] = m < G ? meta[m] : -1;
        bia[i] = reinterpret_cast<const float *>(meta)[32 + (m & 31)];
      }
      const float *wsm = sb + 32 * T + 8 * c;
#pragma unroll 1
      for (int r = 0; r < PW / 32; ++r) {
        const int p0 = cw * PW + r * 32 + 4 * q;    // this lane's 4 positions in the tile
        float2 acc[4][4];                            // [member pair][position]
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[i][e] = make_float2(0.f, 0.f);
#pragma unroll 4
        for (int t = 0; t < K; ++t) {
          const float4 v = *reinterpret_cast<const float4 *>(sb + t * T + p0);
          const float4 w0 = *reinterpret_cast<const float4 *>(wsm + t * 32);
          const float4 w1 = *reinterpret_cast<const float4 *>(wsm + t * 32 + 4);
          const float2 wp[4] = {make_float2(w0.x, w0.y), make_float2(w0.z, w0.w), make_float2(w1.x, w1.y),
                                make_float2(w1.z, w1.w)};
          const float ve[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 v2 = make_float2(ve[e], ve[e]);
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[i][e] = __ffma2_rn(v2, wp[i], acc[i][e]);
          }
        }
        uint32_t am = 0;
        float *dst = Yout + (int64_t)tile * T + p0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (col[i] < 0) continue;
          const float b = bia[i];
          float4 y;
          y.x = clampy(__fadd_rn((i & 1) ? acc[i >> 1][0].y : acc[i >> 1][0].x, b), ymax);
          y.y = clampy(__fadd_rn((i & 1) ? acc[i >> 1][1].y : acc[i >> 1][1].x, b), ymax);
          y.z = clampy(__fadd_rn((i & 1) ? acc[i >> 1][2].y : acc[i >> 1][2].x, b), ymax);
          y.w = clampy(__fadd_rn((i & 1) ? acc[i >> 1][3].y : acc[i >> 1][3].x, b), ymax);
          am |= (y.x > 0.f ? 1u : 0u) | (y.y > 0.f ? 2u : 0u) | (y.z > 0.f ? 4u : 0u) | (y.w > 0.f ? 8u : 0u);
          *reinterpret_cast<float4 *>(dst + (int64_t)col[i] * stride) = y;
        }
        // liveness of the 32 positions: OR over the member octets, then the quads
        am |= __shfl_xor_sync(FULL, am, 8);
        am |= __shfl_xor_sync(FULL, am, 16);
        uint32_t word = am << (4 * q);
        word |= __shfl_xor_sync(FULL, word, 1);
        word |= __shfl_xor_sync(FULL, word, 2);
        word |= __shfl_xor_sync(FULL, word, 4);
        const int64_t base = (int64_t)tile * T + cw * PW + r * 32;
        if (lane == 0 && base < width) {
          if (width - base < 32) word &= (1u << (width - base)) - 1u;
          if (word) atomicOr(&alive[base >> 5], word);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == STAGES) { s = 0; ph ^= 1; }
    }
  }
}

constexpr int kBulkwT = 512, kBulkwNCW = 16, kBulkwStages = 3;

template <int T, int RPS, int STAGES>
constexpr size_t bulk_smem() {
  return (size_t)STAGES * RPS * T * sizeof(float) + 2 * STAGES * 8;
}

// bulk-kernel variant (tile positions, rows per sub-stage, sub-stages, CTAs per
// SM, streaming stores); SDNN_BULK="T,RPS,STAGES,CTAS,CS" selects another
// instantiated variant.  Measured on B200 (C4, tools/gpu_job_bulk_sweep.sh):
// 4 KB row segments (T = 1024) with one whole item per stage reach ~0.91 of
// the measured HBM copy peak; 2 KB segments 0.83; 1 KB 0.59 (1 CTA/SM).
struct BulkCfg {
  int t, rps, stages, ctas, cs;
};
static BulkCfg g_bulk = {1024, 32, 1, 1, 0};

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
        const float *wv = L.val + (int64_t)g * L.kmax * L.gmax + m;   // [t][member]
        float acc[VEC];
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc[e] = 0.f;
#pragma unroll
        for (int t = 0; t < 32; ++t) {
          if (t < K) {
            const float wt = __ldg(wv + t * L.gmax);
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
        const float *wv = L.val + (int64_t)g * L.kmax * L.gmax + m;   // [t][member]
        float acc[VEC];
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc[e] = 0.f;
        for (int t = 0; t < K; ++t) {
          const int k = gsrc[t];
          float v[VEC];
          V::unpack(V::ld(Yin + (int64_t)k * stride + b0), v);
          const float wt = __ldg(wv + (int64_t)t * L.gmax);
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
// element (storage row r, position p) of an activation buffer
// (position-blocked layout: blocks of 2^lg positions, lg = 5 or 4 per boundary)
__device__ __forceinline__ int64_t yix(int64_t r, int64_t p, int64_t stride, int32_t yblk, int lg = 5) {
  return yblk ? (((p >> lg) * yblk + r) << lg) + (p & ((1 << lg) - 1)) : r * stride + p;
}

// one CTA per input row (MNIST-shaped rows hold ~8,500 of 65,536 entries: a
// warp per row left a long serial tail in every chunk of the e2e input path)
__global__ void __launch_bounds__(256) k_scatter(int64_t r0, int64_t r1, const int64_t *__restrict__ rowptr,
                                                 const int32_t *__restrict__ idx, const float *__restrict__ val,
                                                 const uint32_t *__restrict__ inmask,
                                                 const int32_t *__restrict__ wpre, float *Y0, int32_t *rid0,
                                                 int64_t stride, int32_t yblk, const int32_t *__restrict__ sig0,
                                                 int lg, int32_t n) {
  for (int64_t i = r0 + blockIdx.x; i < r1; i += gridDim.x) {
    const uint32_t word = inmask[i >> 5];
    if (!((word >> (i & 31)) & 1u)) continue;
    const int64_t pos = wpre[i >> 5] + __popc(word & ((1u << (i & 31)) - 1u));
    if (threadIdx.x == 0) rid0[pos] = (int32_t)i;
    for (int64_t e = rowptr[i] + threadIdx.x; e < rowptr[i + 1]; e += blockDim.x) {
      const int32_t k = idx[e];
      // an out-of-range index is never written (sdnn_infer validates Y0 on
      // the host concurrently and reports it; the device stays memory-safe)
      if ((uint32_t)k < (uint32_t)n) Y0[yix(sig0 ? sig0[k] : k, pos, stride, yblk, lg)] = val ? val[e] : 1.0f;
    }
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
// Fused multi-layer pass (model decomposition, fuse.cpp; the default plan).  An
// item is (component c, batch tile of T positions).  The component's rows are
// split over C CTAs (C = 1, or a thread-block cluster of 2 / 4): CTA `rank`
// owns up to 512 rows -- the sub-components of the pass's first m-1 layers
// bin-packed at plan time -- as one 64 KB shared-memory tile (R rows x T
// positions, R*T = 16384, T = 32..512) loaded with one cp.async.bulk per row
// (128 B - 2 KB segments; tools/segbench.cu: 0.70 / 0.88 / 0.88 / 0.92 of the
// copy peak at 128 / 256 / 512 / 1024 B), plus its metadata record (source
// slots, biases unless uniform, output rows; <= 8 KB) on the same mbarrier.
// Layers 0..m-2 run in place in the CTA's tile: a group's chain reads its
// source slots, then its members overwrite those slots (legal because every
// non-last layer's source rows each feed one group and G_g <= K_g).  The last
// layer reads its sources from any CTA of the cluster (C > 1: mapa +
// ld.shared::cluster after a cluster barrier) and stores the member rows
// straight to HBM.  As soon as the last layer's chains have read the tiles (a
// second barrier) the next item's copies are issued, before the stores.  Four
// warps; a unit is (group, slice of 32*V positions), V = min(4, T/32)
// positions per lane, UM = 4/V units per warp processed together (independent
// chains for ILP).  HBM traffic per layer drops by m.
// ---------------------------------------------------------------------------
constexpr int kPassTile = 16384;                 // floats per CTA tile (R * T)
constexpr int kPassMaxT = 512;
constexpr int kPassNW = 4;                       // warps per CTA
constexpr size_t kPassSmem =
    (size_t)kPassTile * 4 + kPassRecMax + 16 + kMaxPassLayers * (kPassMaxT / 32) * 4;

int pass_tile_floats() { return kPassTile; }

// (T, C, X2) instances; a cluster pass fills its first CTA beyond half of
// pass_cta_rows() (first-fit bins), hence T = 16384 / pass_cta_rows().  X2
// (packed FFMA2/FADD2) is the cluster default; SDNN_PASS_X2=1 selects it for
// single-CTA passes too.
#define SDNN_PASS_VARIANTS(X)                                                                        \
  X(16, 1, false, 1) X(16, 1, true, 1) X(16, 2, true, 1) X(32, 1, false, 1) X(64, 1, false, 1)          \
  X(128, 1, false, 1) X(256, 1, false, 1) X(512, 1, false, 1) X(32, 1, true, 1) X(64, 1, true, 1)       \
  X(128, 1, true, 1) X(256, 1, true, 1) X(512, 1, true, 1) X(32, 2, true, 1) X(32, 4, true, 1)          \
  X(64, 2, true, 1) X(64, 4, true, 1) X(128, 2, true, 1) X(128, 4, true, 1) X(32, 1, false, 2)          \
  X(64, 1, false, 2) X(128, 1, false, 2)

bool pass_variant(int T, int C, int NB) {
  if (NB == 3) return T == 32 && C == 1;         // k_pass_wide
#define X(TT, CC, XX, NN) \
  if (T == TT && C == CC && NB == NN) return true;
  SDNN_PASS_VARIANTS(X)
#undef X
  return false;
}


template <int T, int C, bool X2, int NB>
__global__ void __launch_bounds__(32 * kPassNW, 3)
    k_pass(const __grid_constant__ DevPass P, const LayerState *__restrict__ st, float *Ya, float *Yb,
           uint32_t *__restrict__ alive, int64_t wstride, int64_t stride, float ymax) {
  constexpr int NW = kPassNW;
  constexpr int SW = T < 128 ? T : 128;          // positions per unit (4 per lane)
  constexpr int S = T / SW;                      // slices per tile
  constexpr int LPU = SW / 4;                    // lanes per unit: 8 / 16 / 32
  constexpr int UPW = 32 / LPU;                  // units per warp (lane segments)
  constexpr int EPL = 32 / LPU;                  // group entries per lane (slot, bias, row)
  constexpr int WPS = SW / 32;                   // liveness words per unit
  constexpr int W = T >= 32 ? T / 32 : 1;        // liveness words per tile (T = 16: half a word)
  constexpr int RPT = kMaxPassRows / (32 * NW);  // input rows per thread
  // tiles of <= 64 positions: rows arrive as 16-B cp.async (LDGSTS) chunks, a
  // warp instruction covering RPI whole rows (one cp.async.bulk per row would
  // be one serialised elected-lane loop iteration per row: ~9 instructions and
  // a uniform-register round trip each); wider tiles keep one bulk copy per row
  // (measured on C4: 128-position tiles 2.46 ms bulk vs 2.56 ms LDGSTS)
  constexpr bool kLdgsts = T <= 64;
  constexpr int CPR = T / 4;                     // 16-B chunks per row
  constexpr int RPI = kLdgsts ? 32 / CPR : 1;    // rows per warp instruction
  // NB = 2 (small components): two half-size tile buffers with their own
  // records and mbarriers, so the next item's load is in flight for the whole
  // of this item's layers instead of from the last layer's release on
  static_assert(NB == 1 || (NB == 2 && C == 1), "double-buffered passes are single-CTA");
  constexpr int TF = kPassTile / NB;             // floats per tile buffer
  constexpr int RB = (kPassRecMax / NB) & ~15;   // record bytes per buffer
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float *const tile0 = reinterpret_cast<float *>(smem_raw);
  unsigned char *const rec0 = smem_raw + (size_t)kPassTile * 4;
  uint64_t *bar = reinterpret_cast<uint64_t *>(rec0 + kPassRecMax);   // [NB]
  uint32_t *aw = reinterpret_cast<uint32_t *>(bar + 2);                 // [kMaxPassLayers][W]
  const LayerState Sx = st[P.a];
  const int width = Sx.width;
  if (width <= 0) return;                        // uniform over the grid
  const float *__restrict__ Yin = Sx.in ? Yb : Ya;
  float *__restrict__ Yout = Sx.in ? Ya : Yb;
  const int tiles = (width + T - 1) / T;
  const int64_t items = (int64_t)P.ncomp * tiles;
  // item -> (component, tile): component-major (consecutive CTAs take
  // consecutive tiles of one component) or tile-major (consecutive CTAs take
  // the same tile of consecutive components, so the CTAs in flight together
  // read and write whole position blocks of the activation buffers)
  const bool tmaj = P.order != 0;
  auto item_comp = [&](int64_t it) -> int64_t { return tmaj ? it % P.ncomp : it / tiles; };
  auto item_tile = [&](int64_t it) -> int { return (int)(tmaj ? it / P.ncomp : it % tiles); };
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int seg = lane / LPU, sll = lane % LPU;  // segment (unit) of the lane, lane in it
  const uint32_t rank = C > 1 ? cluster_rank() : 0u;
  const int64_t cid = C > 1 ? (int64_t)cluster_id_x() : (int64_t)blockIdx.x;
  const int64_t ncl = C > 1 ? (int64_t)nclusters_x() : (int64_t)gridDim.x;
  // position-blocked activations: a CTA's rows are consecutive storage rows, so
  // each 32-position block of its tile is ONE contiguous run of ncnt*128 B,
  // copied by one cp.async.bulk into the tile laid out [T/32][rin][32]
  // (a boundary read by a T = 16 pass has 16-position blocks, lg_in = 4: the
  // tile is then ONE contiguous run of ncnt * 64 B)
  const int32_t R = P.yblk;
  const bool blk = R > 0;
  const bool bt = blk && T >= 32;               // blocked tile: smem [T/32][rin][32]
  const bool b16 = blk && T == 16 && P.lg_in == 4;   // one bulk copy, smem [rin][16]
  // T = 16 in 32-position blocks: half-block rows by TMA boxes of 256 rows
  // (tensor map of the input buffer), else 16-byte LDGSTS chunks
  const bool tma = blk && T == 16 && !b16 && P.tma16;
  const void *tmap_in = &P.tmap[Sx.in];
  const bool ldg = kLdgsts && (!blk || (T < 32 && !b16 && !tma));
  const int lgo = P.lg_out;                      // output boundary block size 2^lgo
  const int rin = P.rin;
  const int sm = bt ? 32 : T;                    // tile floats per slot step
  if (tid == 0) {
    for (int b = 0; b < NB; ++b) mbar_init(bar + b, ldg ? 32 * NW + 1 : 1);   // LDGSTS: one noinc arrival per thread
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int q = tid; q < kMaxPassLayers * W; q += blockDim.x) aw[q] = 0u;
  __syncthreads();
  // thread tid owns input rows tid + 128 q of an item (row id in nrow[q])
  int nrow[RPT], ncnt = 0;
  auto fetch_rows = [&](int64_t it) {
    const int64_t cb = item_comp(it) * C + rank;
    ncnt = __ldg(P.in_count + cb);
    if (blk) {                                   // consecutive storage rows: the first one
      nrow[0] = __ldg(P.in_rows + cb * P.rin);
      return;
    }
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int r = tid + q * 32 * NW;
      nrow[q] = r < P.rin ? __ldg(P.in_rows + cb * P.rin + r) : 0;
    }
  };
  auto issue_load = [&](int64_t it, int buf) {
    float *const tile_s = tile0 + (size_t)buf * TF;
    unsigned char *const rec_s = rec0 + (size_t)buf * RB;
    uint64_t *const bar_b = bar + buf;
    const int64_t c = item_comp(it);
    const int tile = item_tile(it);
    const int64_t cb = c * C + rank;
    if (tid == 0) {
      // (TMA boxes move whole 256-row boxes: rows past the tensor are zero-filled)
      const uint32_t tile_bytes = ldg ? 0u : tma ? (uint32_t)((ncnt + 255) >> 8) * 256u * 64u : (uint32_t)ncnt * T * 4;
      mbar_expect_tx_arrive(bar_b, tile_bytes + (uint32_t)P.rec_bytes);
      bulk_g2s(rec_s, P.rec + cb * P.rec_bytes, P.rec_bytes, bar_b);
      if (bt && ncnt > 0)                        // nrow[0] = the first storage row
#pragma unroll
        for (int q = 0; q < (T >= 32 ? T / 32 : 0); ++q)
          bulk_g2s(tile_s + q * rin * 32, Yin + (((int64_t)tile * (T / 32) + q) * R + nrow[0]) * 32,
                   (uint32_t)ncnt * 128u, bar_b);
      if (b16 && ncnt > 0)
        bulk_g2s(tile_s, Yin + ((int64_t)tile * R + nrow[0]) * 16, (uint32_t)ncnt * 64u, bar_b);
    }
    if (tma) {
      if (tid == 0 && ncnt > 0) {
        const int nbox = (ncnt + 255) >> 8;
        for (int q = 0; q < nbox; ++q)
          tma_load_3d(tile_s + q * 256 * 16, tmap_in, (tile & 1) * 16, nrow[0] + q * 256, tile >> 1, bar_b);
      }
    } else if (bt || b16) {
    } else if (blk) {
      // T = 16: 64 B of each consecutive 128 B block row (block tile/2, half tile%2)
      const float *src0 = Yin + ((int64_t)(tile >> 1) * R + nrow[0]) * 32 + (tile & 1) * 16;
      for (int x = tid; x < ncnt * 4; x += 32 * NW)
        cp_async16(tile_s + (size_t)x * 4, src0 + (int64_t)(x >> 2) * 32 + (x & 3) * 4);
      cp_async_arrive(bar_b);
    } else if (kLdgsts) {
      // warp w copies rows q*128 + 32w + j; lane = (row j % RPI, chunk)
      const int ch = lane % CPR;
      const float *src0 = Yin + (int64_t)tile * T + ch * 4;
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        if (q * 32 * NW >= P.rin) break;
#pragma unroll
        for (int k = 0; k < 32 / RPI; ++k) {
          const int jj = RPI * k + lane / CPR;
          const int r = q * 32 * NW + warp * 32 + jj;
          const int rid = __shfl_sync(FULL, nrow[q], jj);
          if (r < ncnt) cp_async16(tile_s + (size_t)r * T + ch * 4, src0 + (int64_t)rid * stride);
        }
      }
      cp_async_arrive(bar_b);
    } else {
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        const int r = tid + q * 32 * NW;
        if (r < ncnt)
          bulk_g2s(tile_s + (size_t)r * T, Yin + (int64_t)nrow[q] * stride + (int64_t)tile * T, T * 4, bar_b);
      }
    }
  };
  auto release = [&]() {                         // every reader of every tile is done
    if (C > 1) cluster_sync();
    else __syncthreads();
  };
  for (int b = 0; b < NB; ++b)
    if (cid + b * ncl < items) {
      fetch_rows(cid + b * ncl);
      issue_load(cid + b * ncl, b);
    }
  // L2 prefetch of the tile P.pf items ahead (blocked layout): its HBM reads
  // then overlap this item's layers, and the real load (issued at the early
  // release) is served from L2
  auto prefetch = [&](int64_t it) {
    if (tid != 0 || !blk || it >= items) return;
    const int64_t cb = item_comp(it) * C + rank;
    const int cnt = __ldg(P.in_count + cb);
    const int64_t r0 = __ldg(P.in_rows + cb * P.rin);
    const int tile = item_tile(it);
    if (cnt <= 0) return;
    if (T >= 32) {
#pragma unroll 1
      for (int q = 0; q < T / 32; ++q)
        bulk_prefetch_l2(Yin + (((int64_t)tile * (T / 32) + q) * R + r0) * 32, (uint32_t)cnt * 128u);
    } else if (b16) {
      bulk_prefetch_l2(Yin + ((int64_t)tile * R + r0) * 16, (uint32_t)cnt * 64u);
    } else {
      bulk_prefetch_l2(Yin + ((int64_t)(tile >> 1) * R + r0) * 32, (uint32_t)cnt * 128u);
    }
  };
  for (int k = 1; k <= P.pf; ++k) prefetch(cid + k * ncl);
  int64_t kk = 0;
  for (int64_t it = cid; it < items; it += ncl, ++kk) {
    const int buf = NB == 1 ? 0 : (int)(kk % NB);
    const uint32_t ph = (uint32_t)((kk / NB) & 1);
    float *const tile_s = tile0 + (size_t)buf * TF;
    unsigned char *const rec_s = rec0 + (size_t)buf * RB;
    const uint32_t tile_u32 = smem_u32(tile_s);
    const int64_t c = item_comp(it);
    const int tile = item_tile(it);
    const int64_t next = it + NB * ncl;          // the item this buffer takes next
    if (P.pf > 0) prefetch(it + (P.pf + 1) * ncl);
    if (next < items) fetch_rows(next);          // in flight while this item computes
    bool issued = false;
    mbar_wait(bar + buf, ph);
    for (int j = 0; j < P.m; ++j) {
      const PassLayerDev PL = P.layers[j];
      const bool last = j == P.m - 1;
      const bool remote = C > 1 && last;         // sources anywhere in the cluster
      const float wu = PL.wu;
      const bool ubias = PL.off_bias < 0;
      const int units = PL.NG * S;
      const uint16_t *kg_s = reinterpret_cast<const uint16_t *>(rec_s + PL.off_kg);
      const uint16_t *src_s = reinterpret_cast<const uint16_t *>(rec_s + PL.off_src);
      const float *bias_s = reinterpret_cast<const float *>(rec_s + (ubias ? 0 : PL.off_bias));
      const uint16_t *orow_s = reinterpret_cast<const uint16_t *>(rec_s + (last ? PL.off_orow : 0));
      // the last layer releases the tiles before its HBM stores when every warp
      // owns at most one unit per segment (one round)
      const bool early = last && units <= NW * UPW;
      // value tables (fuse.cpp): write into table (vt >> 2) & 1, read the other
      const bool vtw = PL.vt & 1, vtr = PL.vt & 2;
      const int vtline = ((PL.vt >> 2) & 1) * 256;
      if (remote) cluster_sync();                // every CTA's tile is at boundary m-1
      for (int u0 = 0; u0 < units; u0 += NW * UPW) {
        const int u = u0 + warp * UPW + seg;
        int K = 0, G = 0, gi = 0, sl = 0;
        if (u < units) {
          gi = u / S;
          sl = u - gi * S;
          const uint32_t kg = kg_s[gi];
          K = kg & 0xffu;
          G = kg >> 8;
        }
        const int pofs = sl * SW + sll * 4;      // this lane's 4 positions in the tile
        const int pa = bt ? ((pofs >> 5) * rin * 32 + (pofs & 31)) : pofs;   // their smem offset
        // value-table reads: the unit in the second half of a quarter-warp phase
        // reads copy 1 (the other 64 B of the line), so a phase spans all banks
        const int par = vtr ? pa + 16 * (seg & 1) : pa;
        // entry e = r * LPU + sll of the group: source slot (a term past K points
        // at source 0 with weight 0: fmaf(x, 0, acc) == acc for finite x, acc != -0)
        uint32_t soff[EPL];                      // float offset in the tile / cluster address
        float bia[EPL];
        int32_t orw[EPL];
#pragma unroll
        for (int r = 0; r < EPL; ++r) {
          const int e = r * LPU + sll;
          const uint32_t code = K > 0 ? src_s[gi * 32 + (e < K ? e : 0)] : 0u;
          soff[r] = remote ? cluster_map(tile_u32 + (code & 0x3ffu) * (sm * 4), code >> 10)
                           : (code & 0x3ffu) * (vtr ? 32 : sm);
          bia[r] = (!ubias && e < G) ? bias_s[gi * 32 + e] : 0.f;
          orw[r] = (last && e < G) ? orow_s[gi * 32 + e] : 0;
        }
        const int kmax = __reduce_max_sync(FULL, K);
        const bool fullk = __all_sync(FULL, K == kmax || K == 0);
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        // the canonical chain: terms in ascending source order.  Fast path (every
        // unit of the warp has kmax == 32 terms): no per-term conditions, so the
        // loads (DSMEM: ~200 cycles) issue back to back ahead of their FMAs.
        if (kmax == 32 && fullk) {
          if (remote) {
#pragma unroll
            for (int r = 0; r < EPL; ++r)
#pragma unroll
              for (int l = 0; l < LPU; ++l)
                acc4<X2>(acc, ld_cluster_f4(__shfl_sync(FULL, soff[r], l, LPU) + (uint32_t)(pa * 4)), wu);
          } else {
#pragma unroll
            for (int r = 0; r < EPL; ++r)
#pragma unroll
              for (int l = 0; l < LPU; ++l)
                acc4<X2>(acc, *reinterpret_cast<const float4 *>(tile_s + __shfl_sync(FULL, soff[r], l, LPU) + par),
                         wu);
          }
        } else {
#pragma unroll
          for (int r = 0; r < EPL; ++r) {
            if (r * LPU >= kmax) break;
#pragma unroll 4
            for (int l = 0; l < LPU; ++l) {
              const int t = r * LPU + l;
              const uint32_t so = __shfl_sync(FULL, soff[r], l, LPU);
              if (t < kmax) {
                const float w = t < K ? wu : 0.f;
                if (remote) acc4<X2>(acc, ld_cluster_f4(so + (uint32_t)(pa * 4)), w);
                else acc4<X2>(acc, *reinterpret_cast<const float4 *>(tile_s + so + par), w);
              }
            }
          }
        }
        if (early) {
          // generic-proxy tile reads/writes before the next item's TMA writes
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          release();
          if (next < items) issue_load(next, buf);
          issued = true;
        }
        const int gmax = __reduce_max_sync(FULL, G);
        uint32_t o = 0u;
        // members: uniform bias => every member of the group has the same value
        float4 yu = make_float4(0.f, 0.f, 0.f, 0.f);
        if (ubias && G > 0) yu = out4<X2>(acc, PL.bu, ymax, o);
        const int64_t opos = (int64_t)tile * T + pofs;
        float *obase = blk ? Yout + (((opos >> lgo) * R) << lgo) + (opos & ((1 << lgo) - 1)) : Yout + opos;
        const int64_t rowmul = blk ? (1 << lgo) : stride;
        if (!last && vtw) {
          // value table: every group has read its sources (the table overwrites
          // tile rows), then line gi = [copy 0 | copy 1] of the group's value
          __syncthreads();
          if (G > 0) {
            *reinterpret_cast<float4 *>(tile_s + (vtline + gi) * 32 + pa) = yu;
            *reinterpret_cast<float4 *>(tile_s + (vtline + gi) * 32 + 16 + pa) = yu;
          }
        } else if (!last && PL.off_vs >= 0) {
          // shared value: one store per group into its value slot (the next
          // layer's terms of every member of this group point there)
          if (G > 0) {
            const int32_t dst = reinterpret_cast<const uint16_t *>(rec_s + PL.off_vs)[gi] * sm;
            *reinterpret_cast<float4 *>(tile_s + dst + pa) = yu;
          }
        } else {
#pragma unroll
        for (int r = 0; r < EPL; ++r) {
          if (r * LPU >= gmax) break;
#pragma unroll 8
          for (int l = 0; l < LPU; ++l) {
            const int v = r * LPU + l;           // member v (owns source slot v when in place)
            const int32_t dst = last ? __shfl_sync(FULL, orw[r], l, LPU)
                                     : (int32_t)__shfl_sync(FULL, soff[r], l, LPU);
            const float bv = ubias ? 0.f : __shfl_sync(FULL, bia[r], l, LPU);
            if (v < G) {
              const float4 y = ubias ? yu : out4<X2>(acc, bv, ymax, o);
              if (last) *reinterpret_cast<float4 *>(obase + (int64_t)dst * rowmul) = y;
              else *reinterpret_cast<float4 *>(tile_s + dst + pa) = y;
            }
          }
        }
        }
        // liveness: lane sll of a segment holds positions sl*SW + 4 sll + e; word
        // w of the unit has bit b = position 32 w + b -> lane (32 w + b) / 4, e = b % 4
        uint32_t bal[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) bal[e] = __ballot_sync(FULL, (o >> e) & 1u);
        if (sll < WPS && G > 0) {
          // the 8 lanes of word sll give 4 bits each: spread each ballot byte so
          // lane bit l lands on bit 4 l, then interleave the four e planes
          auto spread8 = [](uint32_t x) {
            x = (x | (x << 12)) & 0x000F000Fu;
            x = (x | (x << 6)) & 0x03030303u;
            return (x | (x << 3)) & 0x11111111u;
          };
          const int sh = seg * LPU + sll * 8;
          const uint32_t word = spread8((bal[0] >> sh) & 0xffu) | (spread8((bal[1] >> sh) & 0xffu) << 1) |
                                (spread8((bal[2] >> sh) & 0xffu) << 2) | (spread8((bal[3] >> sh) & 0xffu) << 3);
          if (word) atomicOr(&aw[j * W + sl * WPS + sll], word);
        }
        if (WPS == 0 && sll == 0 && G > 0) {   // T = 16: the unit is the tile's 16 positions
          auto spread4 = [](uint32_t x) {
            x = (x | (x << 6)) & 0x0303u;
            return (x | (x << 3)) & 0x1111u;
          };
          const int sh = seg * LPU;
          const uint32_t hw = spread4((bal[0] >> sh) & 0xfu) | (spread4((bal[1] >> sh) & 0xfu) << 1) |
                              (spread4((bal[2] >> sh) & 0xfu) << 2) | (spread4((bal[3] >> sh) & 0xfu) << 3);
          if (hw) atomicOr(&aw[j * W], hw);
        }
      }
      __syncthreads();                           // the next layer reads slots other warps wrote
    }
    if (tid < W) {
      for (int j = 0; j < P.m; ++j) {
        uint32_t word = aw[j * W + tid];
        aw[j * W + tid] = 0u;
        const int64_t base = (int64_t)tile * T + tid * 32;
        if (base >= width) word = 0u;
        else if (width - base < 32) word &= (1u << (width - base)) - 1u;
        if (word) atomicOr(&alive[j * wstride + (base >> 5)], word << (base & 31));
      }
    }
    if (!issued) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      release();
      if (next < items) issue_load(next, buf);
    }
    __syncthreads();                             // aw published before the next item uses it
  }
  if (C > 1) cluster_sync();                     // no CTA exits while a peer may read its tile
}

// ---------------------------------------------------------------------------
// After a step [a, a+m): survivor counts of its layers, compaction decision
// (row a4) from the last layer's bits, zeroing of the next step's bit set.
// Single CTA.
// ---------------------------------------------------------------------------
constexpr int kCompactMin = 128;

__global__ void __launch_bounds__(1024) k_scan_step(LayerState *st, int a, int m,
                                                    uint32_t *alive_cur,
                                                    uint32_t *alive_next, int64_t wstride,
                                                    int32_t *wpre, int32_t *live, int compact,
                                                    const uint32_t *sat_cur, uint32_t *sat_next,
                                                    const int32_t *ridA, const int32_t *ridB,
                                                    uint32_t *retired, int32_t *nretired,
                                                    uint32_t *pret) {
  __shared__ int s_compacted;
  const LayerState S = st[a];
  const int64_t words = ((int64_t)S.width + 31) >> 5;
  const int32_t before = nretired ? *nretired : 0;   // rows retired by earlier steps
  for (int j = 0; j < m - 1; ++j) {
    int64_t cnt = 0;
    for (int64_t q = threadIdx.x; q < words; q += blockDim.x) cnt += __popc(alive_cur[j * wstride + q]);
    int64_t total;
    block_exclusive_scan(cnt, &total);
    if (threadIdx.x == 0) live[a + j] = (int32_t)total + before;
  }
  uint32_t *last = alive_cur + (int64_t)(m - 1) * wstride;
  int64_t alive_cnt = 0, newly = 0;
  if (pret) {
    // f2 (SDNN_F_SATURATE): positions retired earlier but not yet compacted
    // away (pret) are out of the working set; rows saturated at YMAX before a
    // suffix of saturation-preserving layers (sat_cur) are final categories --
    // record them by original row id and drop them like dead rows
    const int32_t *rid = S.rid ? ridB : ridA;
    for (int64_t q = threadIdx.x; q < words; q += blockDim.x) {
      const uint32_t eff = last[q] & ~pret[q];
      alive_cnt += __popc(eff);
      uint32_t r = sat_cur ? (eff & sat_cur[q]) : 0u;
      last[q] = eff & ~r;
      pret[q] |= r;
      newly += __popc(r);
      while (r) {
        const int b = __ffs(r) - 1;
        r &= r - 1;
        const int32_t id = rid[q * 32 + b];
        atomicOr(&retired[id >> 5], 1u << (id & 31));
      }
    }
    int64_t t0, t1;
    block_exclusive_scan(alive_cnt, &t0);
    block_exclusive_scan(newly, &t1);
    alive_cnt = t0;
    newly = t1;
  }
  const int64_t count = scan_words(last, words, wpre);
  for (int j = 0; j < kMaxPassLayers; ++j)
    for (int64_t q = threadIdx.x; q < words; q += blockDim.x) alive_next[j * wstride + q] = 0u;
  if (sat_next)
    for (int64_t q = threadIdx.x; q < words; q += blockDim.x) sat_next[q] = 0xffffffffu;
  if (threadIdx.x == 0) {
    live[a + m - 1] = (int32_t)(pret ? alive_cnt : count) + before;
    if (nretired) *nretired = before + (int32_t)newly;
    const int64_t dead = S.width - count;
    LayerState n;
    if (compact && dead >= kCompactMin && dead * 16 >= S.width) {
      n.in = S.in;               // the step's input buffer is free: compact into it
      n.width = (int32_t)count;
      n.rid = 1 - S.rid;
      n.compacted = 1;
    } else {
      n.in = 1 - S.in;
      n.width = S.width;
      n.rid = S.rid;
      n.compacted = 0;
    }
    st[a + m] = n;
    s_compacted = n.compacted;
  }
  __syncthreads();
  if (pret && s_compacted)                           // retired positions were dropped
    for (int64_t q = threadIdx.x; q < words; q += blockDim.x) pret[q] = 0u;
}

// Move the live batch columns of the step's output into the free buffer.
// A warp owns one 32-position word q and a slice of the rows: it loads the
// word's bits and its output offset once, then streams the rows -- each load a
// whole 128 B line (32 positions of one row), each store the live lanes packed
// to consecutive output positions -- 8 rows in flight per lane.  In the
// position-blocked layout the rows of word q are consecutive lines, so a warp
// walks one contiguous region.  Row n is the row-id vector.
constexpr int kCompactRowSlices = 8;

__global__ void __launch_bounds__(256) k_compact(const LayerState *__restrict__ st, int a, int m, float *Ya,
                                                 float *Yb, int32_t *ridA, int32_t *ridB,
                                                 const uint32_t *__restrict__ alive,
                                                 const int32_t *__restrict__ wpre, int32_t n, int64_t stride,
                                                 int32_t yblk, int lg) {
  const LayerState N1 = st[a + m];
  if (!N1.compacted) return;
  const LayerState S = st[a];
  const float *__restrict__ src = S.in ? Ya : Yb;   // step output = Y[1 - S.in]
  float *__restrict__ dst = S.in ? Yb : Ya;         // step input buffer
  const int32_t *__restrict__ rsrc = S.rid ? ridB : ridA;
  int32_t *__restrict__ rdst = S.rid ? ridA : ridB;
  const int64_t words = ((int64_t)S.width + 31) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t items = words * kCompactRowSlices;
  for (int64_t it = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < items; it += nw) {
    const int64_t q = it / kCompactRowSlices;
    const int slice = (int)(it - q * kCompactRowSlices);
    const uint32_t bits = alive[q];
    if (bits == 0u) continue;
    const bool live = (bits >> lane) & 1u;
    const int64_t to = wpre[q] + __popc(bits & ((1u << lane) - 1u));
    const int64_t from = q * 32 + lane;
    const int32_t k0 = (int32_t)((int64_t)(n + 1) * slice / kCompactRowSlices);
    const int32_t k1 = (int32_t)((int64_t)(n + 1) * (slice + 1) / kCompactRowSlices);
    int32_t k = k0;
    for (; k + 8 <= k1 && k + 8 <= n; k += 8) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = src[yix(k + u, from, stride, yblk, lg)];
      if (live)
#pragma unroll
        for (int u = 0; u < 8; ++u) dst[yix(k + u, to, stride, yblk, lg)] = v[u];
    }
    for (; k < k1; ++k) {
      if (k < n) {
        const float v = src[yix(k, from, stride, yblk, lg)];
        if (live) dst[yix(k, to, stride, yblk, lg)] = v;
      } else if (live) {
        rdst[to] = rsrc[from];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Readout (row a6).  Single CTA: ascending ids (positions are in ascending
// original-row order because densify and compaction are stable).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_readout(const LayerState *__restrict__ st, int a,
                                                  const uint32_t *__restrict__ alive,
                                                  const int32_t *ridA, const int32_t *ridB,
                                                  int32_t *wpre, int32_t *cats, int32_t *ncat,
                                                  uint32_t *d_alive_out) {
  const LayerState S = st[a];
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
  if (threadIdx.x == 0) *ncat = (int32_t)total;
}

// f2 readout: categories = final live positions (mapped to original rows) OR
// the retired (saturated) rows; one bitmask over original rows, then listed.
__global__ void k_orig_bits(const LayerState *__restrict__ st, int a, const uint32_t *__restrict__ alive,
                            const int32_t *ridA, const int32_t *ridB, uint32_t *orig) {
  const LayerState S = st[a];
  const int32_t *rid = S.rid ? ridB : ridA;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < S.width;
       p += (int64_t)gridDim.x * blockDim.x)
    if ((alive[p >> 5] >> (p & 31)) & 1u) {
      const int32_t id = rid[p];
      atomicOr(&orig[id >> 5], 1u << (id & 31));
    }
}

__global__ void __launch_bounds__(1024) k_list_bits(const uint32_t *__restrict__ orig,
                                                    const uint32_t *__restrict__ retired,
                                                    int64_t words, int32_t *wpre, int32_t *cats,
                                                    int32_t *ncat, uint32_t *d_alive_out) {
  // merge the two bitmasks on the fly
  const int64_t per = (words + blockDim.x - 1) / blockDim.x;
  const int64_t w0 = min(words, (int64_t)threadIdx.x * per), w1 = min(words, w0 + per);
  int64_t sum = 0;
  for (int64_t q = w0; q < w1; ++q) sum += __popc(orig[q] | retired[q]);
  int64_t total;
  int64_t run = block_exclusive_scan(sum, &total);
  for (int64_t q = w0; q < w1; ++q) {
    uint32_t bits = orig[q] | retired[q];
    if (d_alive_out) d_alive_out[q] = bits;
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      cats[run++] = (int32_t)(q * 32 + b);
    }
  }
  (void)wpre;
  if (threadIdx.x == 0) *ncat = (int32_t)total;
}

// f4: readout fused with the cross-GPU gather over NVLink
// SHARP / NVLS.  The rank's category words are built in its slice of the
// symmetric bitmask buffer (unicast view), then every word is written with
// multimem.st through the multicast view -- one store lands in every GPU's
// copy -- and the CTA announces itself with a release multimem add on an
// arrival counter; it returns once the counter shows every rank (target =
// epoch x world), so the local copy then holds the whole global bitmask.
// Single CTA (like k_readout).
// arrival on a multicast counter, then wait (acquire) until the local copy
// reaches target; after ~4 s without progress give up and record the timeout
// in local_flag[1] (the host checks it) instead of hanging the GPU
__device__ __forceinline__ void nvls_arrive_wait(uint32_t *local_flag, uint32_t *mc_flag, uint32_t target) {
  asm volatile("multimem.red.release.sys.global.add.u32 [%0], %1;" ::"l"(mc_flag), "r"(1u) : "memory");
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  uint32_t seen = 0;
  for (;;) {
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(seen) : "l"(local_flag) : "memory");
    if (seen >= target) break;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 4000000000ull) {
      atomicExch(local_flag + 1, 1u);
      break;
    }
    __nanosleep(64);
  }
}

__global__ void k_nvls_barrier(uint32_t *local_flag, uint32_t *mc_flag, uint32_t target) {
  if (threadIdx.x == 0) nvls_arrive_wait(local_flag, mc_flag, target);
}

void launch_nvls_barrier(uint32_t *local_flag, uint32_t *mc_flag, uint32_t target, cudaStream_t s) {
  k_nvls_barrier<<<1, 32, 0, s>>>(local_flag, mc_flag, target);
}

__global__ void __launch_bounds__(1024) k_readout_nvls(const LayerState *__restrict__ st, int a,
                                                       const uint32_t *__restrict__ alive,
                                                       const int32_t *ridA, const int32_t *ridB,
                                                       int64_t batch, uint32_t *local_words,
                                                       uint32_t *mc_words, uint32_t *local_flag,
                                                       uint32_t *mc_flag, uint32_t target) {
  const LayerState S = st[a];
  const int64_t words = ((int64_t)S.width + 31) >> 5, out_words = (batch + 31) >> 5;
  const int32_t *rid = S.rid ? ridB : ridA;
  for (int64_t q = threadIdx.x; q < out_words; q += blockDim.x) local_words[q] = 0u;
  __syncthreads();
  for (int64_t q = threadIdx.x; q < words; q += blockDim.x) {
    uint32_t bits = alive[q];
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      const int32_t id = rid[q * 32 + b];
      atomicOr(&local_words[id >> 5], 1u << (id & 31));
    }
  }
  __syncthreads();
  for (int64_t q = threadIdx.x; q < out_words; q += blockDim.x) {
    const uint32_t v = *((volatile uint32_t *)local_words + q);
    asm volatile("multimem.st.relaxed.sys.global.b32 [%0], %1;" ::"l"(mc_words + q), "r"(v) : "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    nvls_arrive_wait(local_flag, mc_flag, target);
  }
  __syncthreads();
}

void launch_readout_nvls(const Workspace &w, int32_t a, const uint32_t *alive_last, int64_t batch,
                         uint32_t *local_words, uint32_t *mc_words, uint32_t *local_flag, uint32_t *mc_flag,
                         uint32_t target, cudaStream_t s) {
  k_readout_nvls<<<1, 1024, 0, s>>>(w.st, a, alive_last, w.rid[0], w.rid[1], batch, local_words, mc_words,
                                    local_flag, mc_flag, target);
}

// Multi-GPU readout: the all-gathered global bitmask -> ascending row ids
// (single CTA: popcount scan over the words, then each thread lists its run)
__global__ void __launch_bounds__(1024) k_bitmask_ids(const uint32_t *__restrict__ words, int64_t batch,
                                                      int32_t *ids, int32_t *nids) {
  const int64_t nw = (batch + 31) >> 5;
  const int64_t per = (nw + blockDim.x - 1) / blockDim.x;
  const int64_t w0 = min(nw, (int64_t)threadIdx.x * per), w1 = min(nw, w0 + per);
  auto word = [&](int64_t q) {
    uint32_t b = words[q];
    const int64_t base = q * 32;
    if (batch - base < 32) b &= (1u << (batch - base)) - 1u;     // bits past the batch
    return b;
  };
  int64_t sum = 0;
  for (int64_t q = w0; q < w1; ++q) sum += __popc(word(q));
  int64_t total;
  int64_t run = block_exclusive_scan(sum, &total);
  for (int64_t q = w0; q < w1; ++q) {
    uint32_t bits = word(q);
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      ids[run++] = (int32_t)(q * 32 + b);
    }
  }
  if (threadIdx.x == 0) *nids = (int32_t)total;
}

void launch_bitmask_ids(const uint32_t *d_words, int64_t batch, int32_t *d_ids, int32_t *d_n, cudaStream_t s) {
  k_bitmask_ids<<<1, 1024, 0, s>>>(d_words, batch, d_ids, d_n);
}

// f2: rows retired as saturated are all-YMAX in Y_L
__global__ void k_yout_retired(const uint32_t *__restrict__ retired, int64_t batch, int32_t n,
                               float ymax, float *yout) {
  for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < batch * (int64_t)n;
       it += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = it / n;
    if ((retired[r >> 5] >> (r & 31)) & 1u) yout[it] = ymax;
  }
}

// Y_L (neuron-major, positions) -> row-major [batch][n] (rows not present are 0)
__global__ void k_yout(const LayerState *__restrict__ st, int a, int final_out,
                       const float *Ya, const float *Yb, const int32_t *ridA,
                       const int32_t *ridB, int32_t n, int64_t stride, int32_t yblk, float *yout) {
  const LayerState S = st[a];
  const int bufsel = final_out ? 1 - S.in : S.in;
  const float *Y = bufsel ? Yb : Ya;
  const int32_t *rid = S.rid ? ridB : ridA;
  const int64_t total = (int64_t)n * S.width;
  for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < total;
       it += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = it / S.width, p = it - j * S.width;
    yout[(int64_t)rid[p] * n + j] = Y[yix(j, p, stride, yblk)];
  }
}

// Y_L of selected ORIGINAL rows (sampled-row parity at full size): one CTA per
// requested row; its position is found by binary search in the final row-id
// map (ascending: densify and compaction are stable); a row without a position
// (dropped as empty or dead) is all zeros, a retired row (f2) all YMAX.
__global__ void __launch_bounds__(256) k_gather_rows(const LayerState *__restrict__ st, int a, int final_out,
                                                     const float *Ya, const float *Yb, const int32_t *ridA,
                                                     const int32_t *ridB, int32_t n, int64_t stride,
                                                     int32_t yblk, const uint32_t *__restrict__ retired,
                                                     float ymax, const int32_t *__restrict__ rows,
                                                     int64_t nrows, int64_t batch, float *out) {
  __shared__ int64_t s_pos;
  const LayerState S = st[a];
  const float *Y = (final_out ? 1 - S.in : S.in) ? Yb : Ya;
  const int32_t *rid = S.rid ? ridB : ridA;
  for (int64_t q = blockIdx.x; q < nrows; q += gridDim.x) {
    const int32_t row = rows[q];
    if (threadIdx.x == 0) {
      int64_t lo = 0, hi = S.width;                  // first position with rid >= row
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (rid[mid] < row) lo = mid + 1;
        else hi = mid;
      }
      int64_t p = (lo < S.width && rid[lo] == row) ? lo : -1;
      if (row < 0 || row >= batch) p = -1;         // out of range: zeros
      else if (retired && ((retired[row >> 5] >> (row & 31)) & 1u)) p = -2;
      s_pos = p;
    }
    __syncthreads();
    const int64_t p = s_pos;
    float *o = out + q * (int64_t)n;
    for (int32_t j = threadIdx.x; j < n; j += blockDim.x)
      o[j] = p >= 0 ? Y[yix(j, p, stride, yblk)] : (p == -2 ? ymax : 0.f);
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
int bulk_stride_quantum() { return kBulkMaxT; }

#define SDNN_BULK_VARIANTS(X)                                                                     \
  X(512, 32, 3, false) X(1024, 32, 1, false) X(1024, 16, 3, false) X(1024, 16, 1, false)          \
  X(1024, 8, 6, false) X(2048, 8, 3, false) X(2048, 16, 1, false)

static void launch_bulk(const LaunchCfg &c, const Workspace &w, const DevLayer &L, int32_t a,
                        uint32_t *alive, float ymax, uint32_t *sat, cudaStream_t s) {
  const BulkCfg &b = g_bulk;
#define X(TT, RR, SS, CC)                                                                          \
  if (b.t == TT && b.rps == RR && b.stages == SS && (b.cs != 0) == CC) {                            \
    k_layer_bulk<TT, RR, SS, CC><<<c.sms * b.ctas, 32 * (1 + TT / 128), bulk_smem<TT, RR, SS>(),    \
                                   s>>>(L, w.st, a, w.Y[0], w.Y[1], alive, w.stride, ymax, sat);    \
    return;                                                                                         \
  }
  SDNN_BULK_VARIANTS(X)
#undef X
  k_layer_bulk<1024, 32, 1, false><<<c.sms, 288, bulk_smem<1024, 32, 1>(), s>>>(
      L, w.st, a, w.Y[0], w.Y[1], alive, w.stride, ymax, sat);
}

void configure_kernels() {
  configure_pass_wide();
#define X(TT, RR, SS, CC)                                                                      \
  cudaFuncSetAttribute(k_layer_bulk<TT, RR, SS, CC>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                       (int)bulk_smem<TT, RR, SS>());
  SDNN_BULK_VARIANTS(X)
#undef X
  if (const char *e = getenv("SDNN_BULK")) {
    BulkCfg b = g_bulk;
    if (sscanf(e, "%d,%d,%d,%d,%d", &b.t, &b.rps, &b.stages, &b.ctas, &b.cs) == 5 && b.ctas >= 1 &&
        b.ctas <= 4)
      g_bulk = b;
  }
#define X(TT, CC, XX, NN) \
  cudaFuncSetAttribute(k_pass<TT, CC, XX, NN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPassSmem);
  SDNN_PASS_VARIANTS(X)
#undef X
  cudaFuncSetAttribute(k_layer_bulkw<kBulkwT, kBulkwNCW, kBulkwStages>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)bulkw_smem<kBulkwT, kBulkwNCW, kBulkwStages>());
}

bool layer_bulkw_ok(const LaunchCfg &c, const DevLayer &L) {
  static const bool off = [] {
    const char *e = getenv("SDNN_BULKW");
    return e && atoi(e) == 0;
  }();
  return !off && c.bulk && !L.uniform && L.gmax == 32 && L.kmax <= 32 && L.kmax > 0 && L.gbias;
}

// clusters of C CTAs that can be co-resident
template <int T, int C, bool X2, int NB>
static int pass_clusters(int sms) {
  static int cached = 0;
  if (cached) return cached;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C * sms * 3);
  cfg.blockDim = dim3(32 * kPassNW);
  cfg.dynamicSmemBytes = kPassSmem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, k_pass<T, C, X2, NB>, &cfg) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    n = sms * 3 / C / 2;                         // conservative
  }
  cached = n;
  return n;
}

template <int T, int C, bool X2, int NB>
static void launch_pass_t(const LaunchCfg &c, const Workspace &w, const DevPass &P, uint32_t *alive,
                          float ymax, cudaStream_t s) {
  if (C == 1) {
    k_pass<T, 1, X2, NB><<<c.sms * 3, 32 * kPassNW, kPassSmem, s>>>(P, w.st, w.Y[0], w.Y[1], alive, w.words,
                                                            w.stride, ymax);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C * pass_clusters<T, C, X2, NB>(c.sms));
  cfg.blockDim = dim3(32 * kPassNW);
  cfg.dynamicSmemBytes = kPassSmem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_pass<T, C, X2, NB>, P, (const LayerState *)w.st, w.Y[0], w.Y[1], alive,
                     (int64_t)w.words, (int64_t)w.stride, ymax);
}

void launch_densify_prep(const LaunchCfg &c, const Workspace &w, int32_t n, int64_t batch,
                         const int64_t *rowptr, const float *val, bool compact, cudaStream_t s) {
  const int64_t words = (batch + 31) / 32;
  cudaMemsetAsync(w.Y[0], 0, sizeof(float) * (size_t)n * (size_t)w.stride, s);
  cudaMemsetAsync(w.alive[0], 0, sizeof(uint32_t) * (size_t)kMaxPassLayers * w.words, s);
  if (words > 0) {
    const int blocks = (int)std::min<int64_t>((words * 32 + 255) / 256, c.sms * 8);
    k_rowflags<<<blocks, 256, 0, s>>>(batch, rowptr, val, compact ? 1 : 0, w.inmask, words);
  }
  k_scan_input<<<1, 1024, 0, s>>>(w.inmask, words, w.wpre, w.st, w.alive[0]);
  if (w.sat[0]) {
    cudaMemsetAsync(w.sat[0], 0xff, sizeof(uint32_t) * (size_t)w.words, s);
    cudaMemsetAsync(w.retired, 0, sizeof(uint32_t) * (size_t)w.words, s);
    cudaMemsetAsync(w.pret, 0, sizeof(uint32_t) * (size_t)w.words, s);
    cudaMemsetAsync(w.nretired, 0, sizeof(int32_t), s);
  }
}

void launch_scatter_rows(const LaunchCfg &c, const Workspace &w, int32_t n, int64_t r0, int64_t r1,
                         const int64_t *rowptr, const int32_t *idx, const float *val, cudaStream_t s) {
  if (r1 > r0)
    k_scatter<<<(int)std::min<int64_t>(c.sms * 8, r1 - r0), 256, 0, s>>>(
        r0, r1, rowptr, idx, val, w.inmask, w.wpre, w.Y[0], w.rid[0], w.stride, w.yblk, w.sig0, w.lg0, n);
}

void launch_densify(const LaunchCfg &c, const Workspace &w, int32_t n, int64_t batch,
                    const int64_t *rowptr, const int32_t *idx, const float *val, bool compact,
                    cudaStream_t s) {
  launch_densify_prep(c, w, n, batch, rowptr, val, compact, s);
  launch_scatter_rows(c, w, n, 0, batch, rowptr, idx, val, s);
}

void launch_zero_layers_alive(const Workspace &w, int64_t batch, const int64_t *rowptr,
                              const float *val, cudaStream_t s) {
  const int64_t words = (batch + 31) / 32;
  if (words > 0)
    k_y0_positive<<<(int)std::min<int64_t>((words * 32 + 255) / 256, 148 * 8), 256, 0, s>>>(
        batch, rowptr, val, w.alive[0], words);
}

bool layer_tracks_saturation(const LaunchCfg &c, const DevLayer &L) {
  return L.uniform && L.kmax <= 32 && c.bulk;
}

void launch_layer(const LaunchCfg &c, const Workspace &w, const DevLayer &L, int32_t a,
                  uint32_t *alive, float ymax, cudaStream_t s, uint32_t *sat) {
  if (L.uniform && L.kmax <= 32 && c.bulk) {
    launch_bulk(c, w, L, a, alive, ymax, sat, s);
  } else if (L.uniform) {
    if (L.regular && L.kmax == 32)
      k_layer_uniform<4, true><<<c.layer_blocks, 256, 0, s>>>(L, w.st, a, w.Y[0], w.Y[1],
                                                               alive, w.stride, ymax);
    else
      k_layer_uniform<4, false><<<c.layer_blocks, 256, 0, s>>>(L, w.st, a, w.Y[0], w.Y[1],
                                                                alive, w.stride, ymax);
  } else if (layer_bulkw_ok(c, L)) {
    k_layer_bulkw<kBulkwT, kBulkwNCW, kBulkwStages>
        <<<c.sms, 32 * (1 + kBulkwNCW), bulkw_smem<kBulkwT, kBulkwNCW, kBulkwStages>(), s>>>(
            L, w.st, a, w.Y[0], w.Y[1], alive, w.stride, ymax);
  } else {
    k_layer_general<2><<<c.layer_blocks, 256, 0, s>>>(L, w.st, a, w.Y[0], w.Y[1], alive,
                                                      w.stride, ymax);
  }
}

void launch_pass(const LaunchCfg &c, const Workspace &w, const DevPass &P, uint32_t *alive,
                 float ymax, cudaStream_t s) {
  if (P.NB == 3) {
    launch_pass_wide(c, w, P, alive, ymax, s);
    return;
  }
  if (P.general) {
    launch_pass_gw(c, w, P, alive, ymax, s);
    return;
  }
  if (P.NW > 0) {
    launch_pass_t32(c, w, P, alive, ymax, s);
    return;
  }
  // SDNN_PASS_X2=1: packed FFMA2 path for single-CTA passes too; =T: only for
  // tiles of T positions (A/B knob; the default is scalar for C = 1)
  static const int x2_c1 = [] {
    const char *e = getenv("SDNN_PASS_X2");
    return e ? atoi(e) : 0;
  }();
  const bool want_x2 = P.NB == 1 && (P.C > 1 || x2_c1 == 1 || (x2_c1 > 1 && x2_c1 == P.T));
  // (make_plan only plans shapes with an instance, pass_variant; an X2 request
  // without a packed instance falls back to the scalar one)
  for (int attempt = 0; attempt < 2; ++attempt) {
    const bool x2 = want_x2 && attempt == 0;
    switch (P.C * 1024 + P.T + (x2 ? 4096 * 4 : 0) + P.NB * 4096 * 8) {
#define X(TT, CC, XX, NN)                                               \
  case CC * 1024 + TT + (XX ? 4096 * 4 : 0) + NN * 4096 * 8:            \
    launch_pass_t<TT, CC, XX, NN>(c, w, P, alive, ymax, s);             \
    return;
      SDNN_PASS_VARIANTS(X)
#undef X
      default:
        break;
    }
  }
  fprintf(stderr, "sdnn: no k_pass instance for T=%d C=%d NB=%d\n", P.T, P.C, P.NB);
  abort();
}


void launch_scan(const Workspace &w, int32_t a, int32_t m, uint32_t *alive_cur,
                 uint32_t *alive_next, bool compact, cudaStream_t s, const uint32_t *sat_cur,
                 uint32_t *sat_next) {
  k_scan_step<<<1, 1024, 0, s>>>(w.st, a, m, alive_cur, alive_next, w.words, w.wpre, w.live,
                                 compact ? 1 : 0, sat_cur, sat_next, w.rid[0], w.rid[1],
                                 w.retired, w.nretired, w.sat[0] ? w.pret : nullptr);
}

void launch_readout_retired(const Workspace &w, int32_t a, const uint32_t *alive_last,
                            uint32_t *d_alive_out, int64_t batch, cudaStream_t s) {
  const int64_t words = (batch + 31) / 32;
  cudaMemsetAsync(w.orig, 0, sizeof(uint32_t) * (size_t)std::max<int64_t>(words, 1), s);
  k_orig_bits<<<148 * 2, 256, 0, s>>>(w.st, a, alive_last, w.rid[0], w.rid[1], w.orig);
  k_list_bits<<<1, 1024, 0, s>>>(w.orig, w.retired, words, w.wpre, w.cats, w.ncat, d_alive_out);
}

void launch_yout_retired(const Workspace &w, int32_t n, int64_t batch, float ymax, float *d_yout,
                         cudaStream_t s) {
  k_yout_retired<<<148 * 4, 256, 0, s>>>(w.retired, batch, n, ymax, d_yout);
}

void launch_compact_copy(const LaunchCfg &c, const Workspace &w, int32_t a, int32_t m,
                         const uint32_t *alive_last, int32_t n, cudaStream_t s, int lg) {
  k_compact<<<c.copy_blocks, 256, 0, s>>>(w.st, a, m, w.Y[0], w.Y[1], w.rid[0], w.rid[1],
                                          alive_last, w.wpre, n, w.stride, w.yblk, lg);
}

void launch_readout(const Workspace &w, int32_t a, const uint32_t *alive_last,
                    uint32_t *d_alive_out, int64_t batch, cudaStream_t s) {
  if (d_alive_out) cudaMemsetAsync(d_alive_out, 0, sizeof(uint32_t) * (size_t)((batch + 31) / 32), s);
  k_readout<<<1, 1024, 0, s>>>(w.st, a, alive_last, w.rid[0], w.rid[1], w.wpre, w.cats, w.ncat,
                               d_alive_out);
}

void launch_gather_rows(const Workspace &w, int32_t a, bool final_out, int32_t n, float ymax,
                        const int32_t *d_rows, int64_t nrows, int64_t batch, float *d_y, cudaStream_t s) {
  if (nrows <= 0) return;
  k_gather_rows<<<(int)std::min<int64_t>(nrows, 148 * 8), 256, 0, s>>>(
      w.st, a, final_out ? 1 : 0, w.Y[0], w.Y[1], w.rid[0], w.rid[1], n, w.stride, w.yblk,
      w.sat[0] ? w.retired : nullptr, ymax, d_rows, nrows, batch, d_y);
}

void launch_yout(const Workspace &w, int32_t a, bool final_out, int32_t n, int64_t batch,
                 float *d_yout, cudaStream_t s) {
  cudaMemsetAsync(d_yout, 0, sizeof(float) * (size_t)n * (size_t)batch, s);
  k_yout<<<148 * 4, 256, 0, s>>>(w.st, a, final_out ? 1 : 0, w.Y[0], w.Y[1], w.rid[0], w.rid[1],
                                 n, w.stride, w.yblk, d_yout);
}

}  // namespace sdnn
