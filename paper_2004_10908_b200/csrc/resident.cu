// resident.cu -- SMEM-resident multi-layer kernel for narrow networks
// (N <= 4096): BASELINE.json north_star asks that batch tiles of Y stay
// "resident across consecutive layers where the width fits".
//
// A CTA owns P = 16384 / N batch positions (4 at N = 4096, 16 at N = 1024).
// Their activations, Y[N][P] fp32, live in shared memory (two ping-pong
// buffers) for every remaining layer [a, L); only the layer weights move, and
// they come from L2 (every CTA streams the same layer) through a cp.async
// double buffer that is filled while the previous layer computes.  Each of the
// 512 threads owns one (group g, position p) chain per layer -- the canonical
// ascending-source fmaf chain -- then the P lanes of a group split the group's
// member columns between them and write all P positions of each member with
// vector stores.  Rows still nonzero are counted per layer (survivor profile);
// with all biases <= 0 a CTA whose P rows are all dead stops early (their
// outputs stay 0, invariant I2).  Arithmetic is identical to every other
// kernel (A5/A6).
#include "sdnn_internal.h"
#include "device_util.cuh"

#include <algorithm>
#include <cstdlib>

namespace sdnn {

constexpr int kResThreads = 512;
constexpr int kResActFloats = 16384;              // N * P
constexpr int kResMaxBlob = 33 * 1024;            // weight bytes per layer in smem

int resident_positions(int n) {
  if (n > 4096 || n < 1) return 0;
  int p = kResActFloats / n;
  if (p > 32) p = 32;
  int q = 4;
  while (q * 2 <= p) q *= 2;                       // power of two in [4, 32]
  return q;
}
int resident_max_blob() { return kResMaxBlob; }

// same bits as z > 0 ? min(z, ymax) : +0 because z is never -0 (see clampy)
__device__ __forceinline__ float clamp_res(float z, float ymax) {
  return fminf(fmaxf(z, 0.f), ymax);
}

template <int P, int PAD>
__global__ void __launch_bounds__(kResThreads, 1)
    k_resident(const ResLayerDev *__restrict__ layers, int a, int L, int n, const LayerState *__restrict__ st,
               float *Ya, float *Yb, int64_t stride, uint32_t *alive_final, int32_t *live, int compact,
               float ymax) {
  constexpr int RS = P + PAD;                      // smem row stride (PAD = 1 spreads rows over banks)
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float *ys0 = reinterpret_cast<float *>(smem_raw);
  float *ys1 = ys0 + kResActFloats * RS / P;
  unsigned char *wb0 = reinterpret_cast<unsigned char *>(ys1 + kResActFloats * RS / P);
  unsigned char *wb1 = wb0 + kResMaxBlob;
  uint32_t *am = reinterpret_cast<uint32_t *>(wb1 + kResMaxBlob);   // [2]
  __shared__ int s_stop;
  const LayerState S = st[a];
  const int width = S.width;
  const int p0 = blockIdx.x * P;
  if (p0 >= width) return;
  const int nvalid = min(P, width - p0);
  const uint32_t validmask = nvalid >= 32 ? 0xffffffffu : ((1u << nvalid) - 1u);
  const float *__restrict__ Yin = S.in ? Yb : Ya;
  float *__restrict__ Yout = S.in ? Ya : Yb;
  const int tid = threadIdx.x, lane = tid & 31;

  // ---- activations of this CTA's P positions into shared memory ------------
  if (PAD == 0) {
    for (int q = tid; q < n * (P / 4); q += kResThreads) {
      const int k = q / (P / 4), c4 = q - k * (P / 4);
      cp_async16(ys0 + k * RS + c4 * 4, Yin + (int64_t)k * stride + p0 + c4 * 4);
    }
  } else {
    for (int q = tid; q < n * P; q += kResThreads) {
      const int k = q / P, c = q - k * P;
      ys0[k * RS + c] = Yin[(int64_t)k * stride + p0 + c];
    }
  }
  // ---- weights of layer a --------------------------------------------------
  {
    const ResLayerDev L0 = layers[a];
    for (int q = tid; q < L0.bytes / 16; q += kResThreads) cp_async16(wb0 + q * 16, L0.blob + q * 16);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  if (tid == 0) {
    am[0] = 0u;
    am[1] = 0u;
    s_stop = 0;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();

  float *yc = ys0, *yn = ys1;
  bool stopped = false;
  for (int l = a; l < L; ++l) {
    const int par = (l - a) & 1;
    unsigned char *wcur = par ? wb1 : wb0, *wnext = par ? wb0 : wb1;
    if (l + 1 < L) {                              // prefetch the next layer's weights
      const ResLayerDev Ln = layers[l + 1];
      for (int q = tid; q < Ln.bytes / 16; q += kResThreads) cp_async16(wnext + q * 16, Ln.blob + q * 16);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    const ResLayerDev Ld = layers[l];
    const int G = Ld.G;
    const float wu = Ld.wu;
    const uint16_t *src16 = reinterpret_cast<const uint16_t *>(wcur);          // [32][G]
    const uint16_t *col16 = reinterpret_cast<const uint16_t *>(wcur + Ld.off_col); // [G][gmax]
    const float *biasm = reinterpret_cast<const float *>(wcur + Ld.off_bias);     // [G][gmax]
    const uint8_t *k8 = wcur + Ld.off_counts;                                    // [G] K_g
    const uint8_t *g8 = k8 + G;                                                  // [G] G_g
    uint32_t bits = 0;
    for (int u = tid; u < G * P; u += kResThreads) {
      const int g = u / P, p = u & (P - 1);
      const int K = Ld.regular ? 32 : k8[g];
      const int Gg = Ld.regular ? 32 : g8[g];
      float acc = 0.f;
      if (K == 32) {
#pragma unroll 8
        for (int t = 0; t < 32; ++t) acc = __fmaf_rn(yc[src16[t * G + g] * RS + p], wu, acc);
      } else {
        for (int t = 0; t < K; ++t) acc = __fmaf_rn(yc[src16[t * G + g] * RS + p], wu, acc);
      }
      // the P lanes of group g hold its P chains; gather them, then lane p
      // writes the contiguous member block [p*MPL, p*MPL + MPL) for all P
      // positions (member arrays are group-major: one vector load per lane)
      float av[P];
#pragma unroll
      for (int q = 0; q < P; ++q) av[q] = __shfl_sync(FULL, acc, (lane & ~(P - 1)) | q);
      constexpr int MPL = 32 / P;                 // members per lane when G_g = 32
      const int GM = Ld.gmax;
      uint16_t cols[MPL];
      float bs[MPL];
      const int m0 = p * MPL;
      if (Ld.regular) {
        const uint16_t *cg = col16 + g * 32 + m0;
        if (MPL == 8) {
          const uint4 v = *reinterpret_cast<const uint4 *>(cg);
          const uint16_t *h = reinterpret_cast<const uint16_t *>(&v);
#pragma unroll
          for (int i = 0; i < MPL; ++i) cols[i] = h[i];
        } else {
#pragma unroll
          for (int i = 0; i < MPL; ++i) cols[i] = cg[i];
        }
      } else {
#pragma unroll
        for (int i = 0; i < MPL; ++i) cols[i] = (m0 + i < Gg) ? col16[g * GM + m0 + i] : 0;
      }
#pragma unroll
      for (int i = 0; i < MPL; ++i)
        bs[i] = Ld.bias_uniform ? Ld.bias0 : ((m0 + i < Gg) ? biasm[g * GM + m0 + i] : 0.f);
      // liveness: some member of this lane alive iff acc + max bias > 0 (monotone)
      float bhi = -INFINITY;
#pragma unroll
      for (int i = 0; i < MPL; ++i)
        if (m0 + i < Gg) bhi = fmaxf(bhi, bs[i]);
#pragma unroll
      for (int q = 0; q < P; ++q) bits |= (__fadd_rn(av[q], bhi) > 0.f ? 1u : 0u) << q;
#pragma unroll
      for (int i = 0; i < MPL; ++i) {
        if (m0 + i >= Gg) break;
        const float b = bs[i];
        float *dst = yn + cols[i] * RS;
#pragma unroll
        for (int q = 0; q < P; q += 4) {
          float4 y;
          y.x = clamp_res(__fadd_rn(av[q], b), ymax);
          y.y = clamp_res(__fadd_rn(av[q + 1], b), ymax);
          y.z = clamp_res(__fadd_rn(av[q + 2], b), ymax);
          y.w = clamp_res(__fadd_rn(av[q + 3], b), ymax);
          if (PAD == 0) {
            *reinterpret_cast<float4 *>(dst + q) = y;
          } else {
            dst[q] = y.x;
            dst[q + 1] = y.y;
            dst[q + 2] = y.z;
            dst[q + 3] = y.w;
          }
        }
      }
    }
    const uint32_t wbits = __reduce_or_sync(FULL, bits);
    if (lane == 0 && wbits) atomicOr(&am[par], wbits);
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();                              // outputs, liveness bits, next weights ready
    if (tid == 0) {
      const uint32_t alive_bits = am[par] & validmask;
      am[par ^ 1] = 0u;
      if (alive_bits) atomicAdd(&live[l], __popc(alive_bits));
      if (l == L - 1 && alive_bits) {
        const int pos = p0;                       // P divides 32: the word holds all P bits
        atomicOr(&alive_final[pos >> 5], alive_bits << (pos & 31));
      }
      s_stop = (compact && alive_bits == 0) ? 1 : 0;
    }
    float *t = yc;
    yc = yn;
    yn = t;
    __syncthreads();
    if (s_stop) {                                 // every row of this CTA is dead for good
      stopped = true;
      break;
    }
  }
  // ---- final activations back to HBM (the step's output buffer) -------------
  if (PAD == 0) {
    for (int q = tid; q < n * (P / 4); q += kResThreads) {
      const int k = q / (P / 4), c4 = q - k * (P / 4);
      const float4 v =
          stopped ? make_float4(0.f, 0.f, 0.f, 0.f) : *reinterpret_cast<const float4 *>(yc + k * RS + c4 * 4);
      *reinterpret_cast<float4 *>(Yout + (int64_t)k * stride + p0 + c4 * 4) = v;
    }
  } else {
    for (int q = tid; q < n * P; q += kResThreads) {
      const int k = q / P, c = q - k * P;
      Yout[(int64_t)k * stride + p0 + c] = stopped ? 0.f : yc[k * RS + c];
    }
  }
}

template <int P, int PAD>
static size_t res_smem() {
  return (size_t)2 * (kResActFloats / P) * (P + PAD) * 4 + 2 * kResMaxBlob + 16;
}
static int g_res_pad = 0;   // SDNN_RES_PAD=1: rows padded to P+1 floats (measured slower on C2)

void configure_resident() {
  if (const char *e = getenv("SDNN_RES_PAD")) g_res_pad = atoi(e) ? 1 : 0;
#define SDNN_RES_ATTR(PP, DD) \
  cudaFuncSetAttribute(k_resident<PP, DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)res_smem<PP, DD>())
  SDNN_RES_ATTR(4, 0); SDNN_RES_ATTR(8, 0); SDNN_RES_ATTR(16, 0); SDNN_RES_ATTR(32, 0);
  SDNN_RES_ATTR(4, 1); SDNN_RES_ATTR(8, 1); SDNN_RES_ATTR(16, 1); SDNN_RES_ATTR(32, 1);
#undef SDNN_RES_ATTR
}

void launch_resident(const Workspace &w, const ResLayerDev *layers, int a, int L, int n,
                     uint32_t *alive_final, bool compact, float ymax, cudaStream_t s) {
  const int P = resident_positions(n);
  cudaMemsetAsync(w.live + a, 0, sizeof(int32_t) * (size_t)(L - a), s);
  const int grid = (int)((w.stride + P - 1) / P);   // CTAs past the live width exit at once
#define SDNN_RES(PP, DD)                                                                         \
  k_resident<PP, DD><<<grid, kResThreads, res_smem<PP, DD>(), s>>>(                              \
      layers, a, L, n, w.st, w.Y[0], w.Y[1], w.stride, alive_final, w.live, compact ? 1 : 0, ymax)
  if (g_res_pad) {
    switch (P) {
      case 4: SDNN_RES(4, 1); break;
      case 8: SDNN_RES(8, 1); break;
      case 16: SDNN_RES(16, 1); break;
      default: SDNN_RES(32, 1); break;
    }
  } else {
    switch (P) {
      case 4: SDNN_RES(4, 0); break;
      case 8: SDNN_RES(8, 0); break;
      case 16: SDNN_RES(16, 0); break;
      default: SDNN_RES(32, 0); break;
    }
  }
#undef SDNN_RES
}

// Shared-memory weight image of one layer (host side):
//   src u16 [kmax][G] | col u16 [gmax][G] | bias f32 [gmax][G] (omitted when
//   every bias of the layer is equal) | K_g u8 [G] | G_g u8 [G],
//   sections 16-byte aligned; slot-major so a warp's consecutive groups hit
//   consecutive banks.
bool build_resident_blob(const PackedLayer &p, std::vector<unsigned char> &blob, ResLayerDev &d) {
  if (!p.uniform || p.kmax > 32 || p.gmax > 32) return false;
  const int G = p.ngroups, KM = std::max(p.kmax, 1), GM = std::max(p.gmax, 1);
  bool bu = true;
  for (int j = 1; j < p.n && bu; ++j) bu = p.bias[j] == p.bias[0];
  auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
  const size_t off_col = al((size_t)KM * G * 2);
  const size_t off_bias = al(off_col + (size_t)GM * G * 2);
  const size_t off_cnt = bu ? off_bias : al(off_bias + (size_t)GM * G * 4);
  const size_t bytes = al(off_cnt + 2 * (size_t)G);
  if (bytes > (size_t)kResMaxBlob) return false;
  blob.assign(bytes, 0);
  uint16_t *src = reinterpret_cast<uint16_t *>(blob.data());              // [KM][G] slot-major
  uint16_t *col = reinterpret_cast<uint16_t *>(blob.data() + off_col);    // [G][GM] group-major
  float *bias = reinterpret_cast<float *>(blob.data() + off_bias);        // [G][GM]
  uint8_t *cnt = blob.data() + off_cnt;
  for (int g = 0; g < G; ++g) {
    const int K = p.gk[g], Gg = p.gg[g];
    for (int t = 0; t < K; ++t) src[t * G + g] = p.src[(size_t)g * p.kmax + t];
    for (int m = 0; m < Gg; ++m) {
      const int j = p.col[(size_t)g * p.gmax + m];
      col[g * GM + m] = (uint16_t)j;
      if (!bu) bias[g * GM + m] = p.bias[j];
    }
    cnt[g] = (uint8_t)K;
    cnt[G + g] = (uint8_t)Gg;
  }
  d.blob = nullptr;
  d.G = G;
  d.gmax = GM;
  d.bytes = (int32_t)bytes;
  d.wu = p.wu;
  d.regular = p.regular && p.kmax == 32 && p.gmax == 32 ? 1 : 0;
  d.bias_uniform = bu ? 1 : 0;
  d.bias0 = p.bias.empty() ? 0.f : p.bias[0];
  d.off_col = (int32_t)off_col;
  d.off_bias = (int32_t)off_bias;
  d.off_counts = (int32_t)off_cnt;
  return true;
}

}  // namespace sdnn
