// pass_wide.cu -- fused multi-layer pass for components of 513-1024 rows with
// 32-position tiles, one CTA per SM (position-blocked activations only).
//
// k_pass holds a component's rows for one batch tile in a 64 KB shared-memory
// tile, 3 CTAs per SM.  A 1024-row component then gets 16-position tiles: 64 B
// half-block rows, loaded as 16-byte LDGSTS chunks, two rows per 128 B bank
// line (a quarter-warp phase of two units conflicts whenever their source rows
// have equal parity -- 31 % of the shared-load wavefronts on C4).  Here the
// tile keeps 32 positions (128 B rows, one bank line each: conflict-free) and
// is split into two 64 KB halves (rows 0-511 and 512-1023 of the component,
// each ONE contiguous run of the position-blocked buffer, one cp.async.bulk
// each) that rotate through three 64 KB buffers:
//
//   item k of the CTA: half 0 (+ the record) in buffer (2k) % 3, half 1 in
//   buffer (2k+1) % 3.  When item k's last layer has read its tile, its two
//   buffers take half 1 of item k+1 and half 0 of item k+2 -- so half 0 of
//   the next item streams in during this item's whole layer chain.
//
// 8 warps; a unit is (group, the 32 positions), 8 lanes x 4 positions, 4 units
// per warp: one round of units covers the 32 groups of a 1024-row layer.  The
// arithmetic is k_pass's (the canonical ascending-source fmaf chain per group,
// bias add, clamp; A5/A6) and the record format is the same
// (fuse.cpp build_pass, PassHost.NB = 3).  Slot s of the component lives at
// float offset hoff[s >= split] + s * 32 of the buffer space (split = 512).
//
// Measured on C4 (1024-row 3-layer passes): 3.27 ms vs 3.43-3.50 ms for the
// 16-position k_pass tiles.  Tried and slower: half-warp units of 2
// positions per lane with layers 0..m-2 of the half-0 sub-components run
// before half 1 is waited for (5.08 ms: a third of the chains per lane, twice
// the barriers; with one CTA per SM every barrier idles the SM); the
// sub-components packed into the halves and layers 0..m-2 of each half run by
// its own 4-warp group on a named barrier as soon as its half has landed
// (3.52 vs 3.35 ms).
#include <algorithm>
#include <cassert>
#include <array>
#include <atomic>
#include <cstdio>
#include <cstdlib>

#include "sdnn_internal.h"
#include "device_util.cuh"

namespace sdnn {

#ifndef SDNN_T32_FETCH
#define SDNN_T32_FETCH 0                                // k_pass_t32: next item's rows fetched an item ahead
#endif
#ifndef SDNN_REMOTE_FAST
#define SDNN_REMOTE_FAST 0                              // k_pass_t32 C = 2: unconditional 32-term DSMEM chain
#endif
// (both measured within run-to-run noise, 1754 vs 1762-1766 ms/step on one box: off)
#ifndef SDNN_SPLIT_RELEASE
#define SDNN_SPLIT_RELEASE 0                            // clusters: arrive before the stores, wait after
#endif
// (measured in alternating runs: 1772 / 1771 vs 1762 / 1760 ms/step on C4: off)
constexpr bool kSplitRelease = SDNN_SPLIT_RELEASE != 0;
// SDNN_DEBUG_CHECKS=1 (build time, tools/debug_checks.sh): device asserts on
// every slot, storage row and row count the pass kernels use (a stand-in for
// compute-sanitizer, which is closed on the GPU pool)
#ifndef SDNN_DEBUG_CHECKS
#define SDNN_DEBUG_CHECKS 0
#endif
#if SDNN_DEBUG_CHECKS
#define SDNN_CHECK(c) assert(c)
#else
#define SDNN_CHECK(c) ((void)0)
#endif
#ifndef SDNN_CHAIN_B
#define SDNN_CHAIN_B 0
#endif
constexpr int kChainB = SDNN_CHAIN_B;                   // loads in flight per lane (chain32)
#ifndef SDNN_CHAIN_REGS
#define SDNN_CHAIN_REGS 0
#endif
constexpr bool kChainRegs = SDNN_CHAIN_REGS != 0;       // k_pass_t32: shuffle-free addresses
constexpr int kWideNW = 8;                              // warps
constexpr int kWideHalf = 512;                          // rows per half buffer
constexpr int kWideHalfFloats = kWideHalf * 32;         // 64 KB
constexpr int kWideRec = (kPassRecMax + 15) & ~15;      // record buffer bytes
constexpr size_t kWideSmem = 3 * (size_t)kWideHalfFloats * 4 + 2 * (size_t)kWideRec + 3 * 8 + kMaxPassLayers * 4;

// The 32-term fast path of a unit (8 lanes x 4 positions, every unit of the
// warp with 32 terms): all 32 shared-memory addresses first (the shuffles are
// independent), then the loads in batches of B ahead of their FMAs, so a warp
// keeps B loads in flight (SDNN_CHAIN_B, default 0 = the plain interleaved
// loop; measured on C4: B = 8 / 16 / 32: 1849 / 1837 / 1817 vs 1816 ms/step)
template <bool X2, int B>
__device__ __forceinline__ void chain32(float (&acc)[4], const float *base, const uint32_t (&soff)[4], int pa,
                                        float wu) {
  if constexpr (B == 0) {
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int l = 0; l < 8; ++l)
        acc4<X2>(acc, *reinterpret_cast<const float4 *>(base + __shfl_sync(FULL, soff[r], l, 8) + pa), wu);
  } else {
  uint32_t ad[32];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int l = 0; l < 8; ++l) ad[r * 8 + l] = __shfl_sync(FULL, soff[r], l, 8) + (uint32_t)pa;
#pragma unroll
  for (int t0 = 0; t0 < 32; t0 += (B > 0 ? B : 32)) {
    float4 v[B > 0 ? B : 1];
#pragma unroll
    for (int q = 0; q < B; ++q) v[q] = *reinterpret_cast<const float4 *>(base + ad[t0 + q]);
#pragma unroll
    for (int q = 0; q < B; ++q) acc4<X2>(acc, v[q], wu);
  }
  }
}

// The 32-term fast path without shuffles: every lane of the unit reads the
// group's 32 u16 slot codes itself (four 16-byte shared loads, broadcast to
// the unit's 8 lanes) and forms each term's address with two integer ops, so
// no term waits on a shuffle (opt-in, SDNN_CHAIN_REGS=1 at build time:
// measured on C4 1797 vs 1760 ms/step for the shuffle version)
template <bool X2>
__device__ __forceinline__ void chain32_regs(float (&acc)[4], const float *base, const uint16_t *codes, int pa,
                                             float wu) {
  const uint4 *c4 = reinterpret_cast<const uint4 *>(codes);
  uint32_t w[16];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint4 v = c4[q];
    w[4 * q] = v.x;
    w[4 * q + 1] = v.y;
    w[4 * q + 2] = v.z;
    w[4 * q + 3] = v.w;
  }
#pragma unroll
  for (int t = 0; t < 32; ++t) {
    const uint32_t slot = ((t & 1) ? (w[t >> 1] >> 16) : w[t >> 1]) & 0x3ffu;
    acc4<X2>(acc, *reinterpret_cast<const float4 *>(base + slot * 32u + (uint32_t)pa), wu);
  }
}

template <bool X2>
__global__ void __launch_bounds__(32 * kWideNW, 1)
    k_pass_wide(const __grid_constant__ DevPass P, const LayerState *__restrict__ st, float *Ya, float *Yb,
                uint32_t *__restrict__ alive, int64_t wstride, float ymax) {
  constexpr int NW = kWideNW, T = 32, LPU = 8, UPW = 4, EPL = 4;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float *const smf = reinterpret_cast<float *>(smem_raw);                          // [3][512][32]
  unsigned char *const rec0 = smem_raw + 3 * (size_t)kWideHalfFloats * 4;          // [2][kWideRec]
  uint64_t *const bar = reinterpret_cast<uint64_t *>(rec0 + 2 * (size_t)kWideRec); // [3]
  uint32_t *const aw = reinterpret_cast<uint32_t *>(bar + 3);                       // [kMaxPassLayers]
  const LayerState Sx = st[P.a];
  const int width = Sx.width;
  if (width <= 0) return;                        // uniform over the grid
  const float *__restrict__ Yin = Sx.in ? Yb : Ya;
  float *__restrict__ Yout = Sx.in ? Ya : Yb;
  const int tiles = (width + T - 1) / T;
  const int64_t items = (int64_t)P.ncomp * tiles;
  const bool tmaj = P.order != 0;
  auto item_comp = [&](int64_t it) -> int64_t { return tmaj ? it % P.ncomp : it / tiles; };
  auto item_tile = [&](int64_t it) -> int { return (int)(tmaj ? it / P.ncomp : it % tiles); };
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int seg = lane / LPU, sll = lane % LPU;  // unit (lane octet) of the lane, lane in it
  const int pa = sll * 4;                        // this lane's 4 positions in the tile
  const int64_t R = P.yblk;                      // storage rows per position block
  const int lgo = P.lg_out;
  const int64_t cid = blockIdx.x, ncl = gridDim.x;
  if (tid == 0) {
    for (int b = 0; b < 3; ++b) mbar_init(bar + b, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int q = tid; q < kMaxPassLayers; q += blockDim.x) aw[q] = 0u;
  __syncthreads();
  // half h of item it into buffer j (half 0 also brings the record into rb):
  // rows [0, split) and [split, cnt) of the component, each one contiguous run
  auto issue_half = [&](int64_t it, int h, int j, int rb) {
    if (tid != 0 || it >= items) return;
    const int64_t c = item_comp(it);
    const int tile = item_tile(it);
    const int cnt = __ldg(P.in_count + c);
    const int s0 = __ldg(P.split + c);
    const int nh = h == 0 ? s0 : cnt - s0;
    mbar_expect_tx_arrive(bar + j, (uint32_t)nh * 128u + (h ? 0u : (uint32_t)P.rec_bytes));
    if (!h) bulk_g2s(rec0 + (size_t)rb * kWideRec, P.rec + c * P.rec_bytes, (uint32_t)P.rec_bytes, bar + j);
    if (nh > 0) {
      const int64_t row0 = __ldg(P.in_rows + c * P.rin) + (h ? s0 : 0);
      bulk_g2s(smf + (size_t)j * kWideHalfFloats, Yin + ((int64_t)tile * R + row0) * 32, (uint32_t)nh * 128u,
               bar + j);
    }
  };
  issue_half(cid, 0, 0, 0);
  issue_half(cid, 1, 1, 0);
  issue_half(cid + ncl, 0, 2, 1);
  uint32_t phase = 0u;                           // bit j: parity of buffer j's next completion
  int64_t kk = 0;
  for (int64_t it = cid; it < items; it += ncl, ++kk) {
    const int bA = (int)((2 * kk) % 3), bB = (int)((2 * kk + 1) % 3);
    const unsigned char *rec_s = rec0 + (size_t)(kk & 1) * kWideRec;
    const int tile = item_tile(it);
    const int s0 = __ldg(P.split + item_comp(it));
    // slot s -> float offset hoff[s >= s0] + s * 32 in the buffer space
    const int32_t hoff0 = bA * kWideHalfFloats, hoff1 = bB * kWideHalfFloats - s0 * 32;
    if (P.pf > 0 && tid == 0 && it + ncl < items) {
      // L2 prefetch of half 1 of the next item (its TMA load is issued at this
      // item's release): its HBM read overlaps this item's layers
      const int64_t nx = it + ncl;
      const int64_t c1 = item_comp(nx);
      const int cnt1 = __ldg(P.in_count + c1), s1 = __ldg(P.split + c1);
      if (cnt1 > s1)
        bulk_prefetch_l2(Yin + ((int64_t)item_tile(nx) * R + __ldg(P.in_rows + c1 * P.rin) + s1) * 32,
                         (uint32_t)(cnt1 - s1) * 128u);
    }
    mbar_wait(bar + bA, (phase >> bA) & 1u);     // half 0 and the record
    phase ^= 1u << bA;
    mbar_wait(bar + bB, (phase >> bB) & 1u);
    phase ^= 1u << bB;
    auto release_and_load = [&]() {
      // generic-proxy tile reads/writes before the next items' TMA writes
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      issue_half(it + ncl, 1, bA, 0);
      issue_half(it + 2 * ncl, 0, bB, (int)(kk & 1));
    };
    bool issued = false;
    // groups [g0, g1) of layer j on nwg warps starting at warp w0 (the last
    // layer: all groups, all warps, with the early release)
    auto run = [&](int j, int g0, int g1, int w0, int nwg) {
      const PassLayerDev PL = P.layers[j];
      const bool last = j == P.m - 1;
      const float wu = PL.wu;
      const bool ubias = PL.off_bias < 0;
      const int units = g1;
      const uint16_t *kg_s = reinterpret_cast<const uint16_t *>(rec_s + PL.off_kg);
      const uint16_t *src_s = reinterpret_cast<const uint16_t *>(rec_s + PL.off_src);
      const float *bias_s = reinterpret_cast<const float *>(rec_s + (ubias ? 0 : PL.off_bias));
      const uint16_t *orow_s = reinterpret_cast<const uint16_t *>(rec_s + (last ? PL.off_orow : 0));
      const bool early = last && g1 - g0 <= nwg * UPW;
      for (int u0 = g0; u0 < units; u0 += nwg * UPW) {
        const int u = u0 + (warp - w0) * UPW + seg;
        int K = 0, G = 0, gi = 0;
        if (u < units) {
          gi = u;
          const uint32_t kg = kg_s[gi];
          K = kg & 0xffu;
          G = kg >> 8;
        }
        uint32_t soff[EPL];                      // float offset of the entry's slot row
        float bia[EPL];
        int32_t orw[EPL];
#pragma unroll
        for (int r = 0; r < EPL; ++r) {
          const int e = r * LPU + sll;
          const int32_t slot = K > 0 ? (src_s[gi * 32 + (e < K ? e : 0)] & 0x3ff) : 0;
          soff[r] = (uint32_t)((slot < s0 ? hoff0 : hoff1) + slot * 32);
          bia[r] = (!ubias && e < G) ? bias_s[gi * 32 + e] : 0.f;
          orw[r] = (last && e < G) ? orow_s[gi * 32 + e] : 0;
        }
        const int kmax = __reduce_max_sync(FULL, K);
        const bool fullk = __all_sync(FULL, K == kmax || K == 0);
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        // the canonical chain: terms in ascending source order (a term past K
        // reads source 0 with weight 0: fmaf(x, 0, acc) == acc, acc != -0)
        if (kmax == 32 && fullk) {
          chain32<X2, kChainB>(acc, smf, soff, pa, wu);
        } else {
#pragma unroll
          for (int r = 0; r < EPL; ++r) {
            if (r * LPU >= kmax) break;
#pragma unroll 4
            for (int l = 0; l < LPU; ++l) {
              const int t = r * LPU + l;
              const uint32_t so = __shfl_sync(FULL, soff[r], l, LPU);
              if (t < kmax) acc4<X2>(acc, *reinterpret_cast<const float4 *>(smf + so + pa), t < K ? wu : 0.f);
            }
          }
        }
        if (early) {
          release_and_load();
          issued = true;
        }
        const int gmax = __reduce_max_sync(FULL, G);
        uint32_t o = 0u;
        float4 yu = make_float4(0.f, 0.f, 0.f, 0.f);   // uniform bias: one value per group
        if (ubias && G > 0) yu = out4<X2>(acc, PL.bu, ymax, o);
        const int64_t opos = (int64_t)tile * T + pa;
        float *obase = Yout + (((opos >> lgo) * R) << lgo) + (opos & ((1 << lgo) - 1));
        const int64_t rowmul = (int64_t)1 << lgo;
#pragma unroll
        for (int r = 0; r < EPL; ++r) {
          if (r * LPU >= gmax) break;
#pragma unroll 8
          for (int l = 0; l < LPU; ++l) {
            const int v = r * LPU + l;           // member v (owns source slot v when in place)
            const int32_t dst = last ? __shfl_sync(FULL, orw[r], l, LPU) : (int32_t)__shfl_sync(FULL, soff[r], l, LPU);
            const float bv = ubias ? 0.f : __shfl_sync(FULL, bia[r], l, LPU);
            if (v < G) {
              const float4 y = ubias ? yu : out4<X2>(acc, bv, ymax, o);
              if (last) *reinterpret_cast<float4 *>(obase + (int64_t)dst * rowmul) = y;
              else *reinterpret_cast<float4 *>(smf + dst + pa) = y;
            }
          }
        }
        // liveness: word bit b = position b -> lane b / 4 of the unit, e = b % 4
        uint32_t bal[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) bal[e] = __ballot_sync(FULL, (o >> e) & 1u);
        if (sll == 0 && G > 0) {
          auto spread8 = [](uint32_t x) {
            x = (x | (x << 12)) & 0x000F000Fu;
            x = (x | (x << 6)) & 0x03030303u;
            return (x | (x << 3)) & 0x11111111u;
          };
          const int sh = seg * LPU;
          const uint32_t word = spread8((bal[0] >> sh) & 0xffu) | (spread8((bal[1] >> sh) & 0xffu) << 1) |
                                (spread8((bal[2] >> sh) & 0xffu) << 2) | (spread8((bal[3] >> sh) & 0xffu) << 3);
          if (word) atomicOr(&aw[j], word);
        }
      }
    };
    for (int j = 0; j + 1 < P.m; ++j) {
      run(j, 0, P.layers[j].NG, 0, NW);
      __syncthreads();                           // the next layer reads slots other warps wrote
    }
    run(P.m - 1, 0, P.layers[P.m - 1].NG, 0, NW);
    __syncthreads();
    if (tid == 0) {
      const int64_t base = (int64_t)tile * T;
      for (int j = 0; j < P.m; ++j) {
        uint32_t word = aw[j];
        aw[j] = 0u;
        if (base >= width) word = 0u;
        else if (width - base < 32) word &= (1u << (width - base)) - 1u;
        if (word) atomicOr(&alive[j * wstride + (base >> 5)], word);
      }
    }
    if (!issued) release_and_load();
    __syncthreads();                             // aw published before the next item uses it
  }
}

// function attributes are per device: launches track the configured shared
// memory size per device ordinal
constexpr int kMaxDevices = 64;
static int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d < 0 || d >= kMaxDevices ? 0 : d;
}

static bool wide_x2() {                          // packed FFMA2 / FADD2 (SDNN_PASS_X2=0: scalar)
  // measured on one box, alternating runs: C4 1748.2 / 1748.6 vs 1756.1 / 1756.6
  // ms/step scalar, C3 329.1 vs 329.8 ms
  static const bool v = [] {
    const char *e = getenv("SDNN_PASS_X2");
    return !(e && atoi(e) == 0);
  }();
  return v;
}

void configure_pass_wide() {
  cudaFuncSetAttribute(k_pass_wide<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kWideSmem);
  cudaFuncSetAttribute(k_pass_wide<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kWideSmem);
}

void launch_pass_wide(const LaunchCfg &c, const Workspace &w, const DevPass &P, uint32_t *alive, float ymax,
                      cudaStream_t s) {
  if (wide_x2())
    k_pass_wide<true><<<c.sms, 32 * kWideNW, kWideSmem, s>>>(P, w.st, w.Y[0], w.Y[1], alive, w.words, ymax);
  else
    k_pass_wide<false><<<c.sms, 32 * kWideNW, kWideSmem, s>>>(P, w.st, w.Y[0], w.Y[1], alive, w.words, ymax);
}

// planner switch (fuse.cpp): 513-1024-row components in one CTA get this
// kernel (SDNN_PASS_WIDE=0: 16-position k_pass tiles instead)
bool pass_wide_enabled() { return pass_wide_mode() >= 1; }   // (mode 2: the 2-layer passes)



// ---------------------------------------------------------------------------
// k_pass_t32<NW, S>: fused pass over components of <= 128 * NW rows with
// 32-position tiles in CTAs of NW warps (position-blocked activations, one CTA
// per component tile).  A tile (R rows x 128 B) is ONE contiguous run of the
// blocked buffer: one cp.async.bulk plus the record on one mbarrier per
// buffer; S buffers per CTA (S = 2: the next item streams in during this
// item's layers).  The shared-memory footprint follows the pass (S x (R x
// 128 B + record)), so small components get many small CTAs per SM -- a
// 128-row pass runs one-warp CTAs, every warp busy -- where k_pass gives every
// CTA a 64 KB tile and 4 warps (128-row passes: 4 groups = 2 busy warps).  The
// arithmetic and the record are k_pass's (fuse.cpp, PassHost.NW > 0).
// ---------------------------------------------------------------------------
template <int NW, int S, bool X2, int C>
__global__ void __launch_bounds__(32 * NW)
    k_pass_t32(const __grid_constant__ DevPass P, const LayerState *__restrict__ st, float *Ya, float *Yb,
               uint32_t *__restrict__ alive, int64_t wstride, float ymax, uint32_t buf_bytes) {
  constexpr int T = 32, LPU = 8, UPW = 4, EPL = 4;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // per buffer: [tile R x 32 floats | record], buf_bytes each (128 B multiple)
  uint64_t *const bar = reinterpret_cast<uint64_t *>(smem_raw + (size_t)S * buf_bytes);   // [S]
  uint32_t *const aw = reinterpret_cast<uint32_t *>(bar + S);                              // [m]
  const LayerState Sx = st[P.a];
  const int width = Sx.width;
  if (width <= 0) return;
  const float *__restrict__ Yin = Sx.in ? Yb : Ya;
  float *__restrict__ Yout = Sx.in ? Ya : Yb;
  const int tiles = (width + T - 1) / T;
  const int64_t items = (int64_t)P.ncomp * tiles;
  const bool tmaj = P.order != 0;
  auto item_comp = [&](int64_t it) -> int64_t { return tmaj ? it % P.ncomp : it / tiles; };
  auto item_tile = [&](int64_t it) -> int { return (int)(tmaj ? it / P.ncomp : it % tiles); };
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int seg = lane / LPU, sll = lane % LPU;
  const int pa = sll * 4;
  const int64_t R = P.yblk;
  const int lgo = P.lg_out;
  const uint32_t rec_off = (uint32_t)P.R * 128u;  // record after the tile in each buffer
  // C = 2: a component of up to 1024 rows over a 2-CTA cluster (each CTA
  // holds its bin's rows); layers 0..m-2 stay in the CTA, the last reads its
  // sources from both CTAs' tiles (DSMEM) between two cluster barriers
  const uint32_t rank = C > 1 ? cluster_rank() : 0u;
  const int64_t cid = C > 1 ? (int64_t)cluster_id_x() : (int64_t)blockIdx.x;
  const int64_t ncl = C > 1 ? (int64_t)nclusters_x() : (int64_t)gridDim.x;
  if (tid == 0) {
    for (int b = 0; b < S; ++b) mbar_init(bar + b, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int q = tid; q < P.m; q += blockDim.x) aw[q] = 0u;
  __syncthreads();
  // the row count and first storage row of an item's (component, rank) come
  // from global memory: fetched (thread 0) an item ahead of the issue, so the
  // issue after the release does not wait on a dependent global load
  int nx_cnt = 0;
  int64_t nx_row = 0;
  auto fetch = [&](int64_t it) {
    if (tid != 0 || it >= items) return;
    const int64_t c = item_comp(it) * C + rank;
    nx_cnt = __ldg(P.in_count + c);
    nx_row = __ldg(P.in_rows + c * P.rin);
  };
  auto issue = [&](int64_t it, int b) {          // (after fetch(it))
    if (tid != 0 || it >= items) return;
    const int64_t c = item_comp(it) * C + rank;
    const int tile = item_tile(it);
    const int cnt = nx_cnt;
    SDNN_CHECK(cnt >= 0 && cnt <= P.R && (cnt == 0 || (nx_row >= 0 && nx_row + cnt <= P.yblk)));
    unsigned char *dst = smem_raw + (size_t)b * buf_bytes;
    mbar_expect_tx_arrive(bar + b, (uint32_t)cnt * 128u + (uint32_t)P.rec_bytes);
    bulk_g2s(dst + rec_off, P.rec + c * P.rec_bytes, (uint32_t)P.rec_bytes, bar + b);
    if (cnt > 0) bulk_g2s(dst, Yin + ((int64_t)tile * R + nx_row) * 32, (uint32_t)cnt * 128u, bar + b);
  };
  for (int b = 0; b < S; ++b) {
    fetch(cid + b * ncl);
    issue(cid + b * ncl, b);
  }
  int64_t kk = 0;
  for (int64_t it = cid; it < items; it += ncl, ++kk) {
    const int b = S == 1 ? 0 : (int)(kk % S);
    const uint32_t ph = (uint32_t)((kk / S) & 1);
    float *const tile_s = reinterpret_cast<float *>(smem_raw + (size_t)b * buf_bytes);
    const unsigned char *rec_s = smem_raw + (size_t)b * buf_bytes + rec_off;
    const int tile = item_tile(it);
#if SDNN_T32_FETCH
    fetch(it + S * ncl);                         // in flight while this item computes
#endif
    mbar_wait(bar + b, ph);
    auto release_and_load = [&]() {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (C > 1) cluster_sync();                 // the peer has read this tile too
      else __syncthreads();
#if !SDNN_T32_FETCH
      fetch(it + S * ncl);
#endif
      issue(it + S * ncl, b);
    };
    bool issued = false, split_pending = false;
    for (int j = 0; j < P.m; ++j) {
      const PassLayerDev PL = P.layers[j];
      const bool last = j == P.m - 1;
      const float wu = PL.wu;
      const bool ubias = PL.off_bias < 0;
      const int units = PL.NG;
      const uint16_t *kg_s = reinterpret_cast<const uint16_t *>(rec_s + PL.off_kg);
      const uint16_t *src_s = reinterpret_cast<const uint16_t *>(rec_s + PL.off_src);
      const float *bias_s = reinterpret_cast<const float *>(rec_s + (ubias ? 0 : PL.off_bias));
      const uint16_t *orow_s = reinterpret_cast<const uint16_t *>(rec_s + (last ? PL.off_orow : 0));
      const bool early = last && units <= NW * UPW;
      const bool remote = C > 1 && last;
      if (remote) cluster_sync();                // every CTA's tile is at boundary m-1
      for (int u0 = 0; u0 < units; u0 += NW * UPW) {
        const int u = u0 + warp * UPW + seg;
        int K = 0, G = 0, gi = 0;
        if (u < units) {
          gi = u;
          const uint32_t kg = kg_s[gi];
          K = kg & 0xffu;
          G = kg >> 8;
        }
        uint32_t soff[EPL];
        float bia[EPL];
        int32_t orw[EPL];
#pragma unroll
        for (int r = 0; r < EPL; ++r) {
          const int e = r * LPU + sll;
          const uint32_t code = K > 0 ? src_s[gi * 32 + (e < K ? e : 0)] : 0u;
          SDNN_CHECK((code & 0x3ffu) < (uint32_t)P.R && (code >> 10) < (uint32_t)C);
          soff[r] = remote ? cluster_map(smem_u32(tile_s) + (code & 0x3ffu) * 128u, code >> 10)
                           : (code & 0x3ffu) * 32u;
          bia[r] = (!ubias && e < G) ? bias_s[gi * 32 + e] : 0.f;
          orw[r] = (last && e < G) ? orow_s[gi * 32 + e] : 0;
        }
        const int kmax = __reduce_max_sync(FULL, K);
        const bool fullk = __all_sync(FULL, K == kmax || K == 0);
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        if (SDNN_REMOTE_FAST && remote && kmax == 32 && fullk) {   // DSMEM: cluster-window byte addresses
#pragma unroll
          for (int r = 0; r < EPL; ++r)
#pragma unroll
            for (int l = 0; l < LPU; ++l)
              acc4<X2>(acc, ld_cluster_f4(__shfl_sync(FULL, soff[r], l, LPU) + (uint32_t)(pa * 4)), wu);
        } else if (remote) {
#pragma unroll
          for (int r = 0; r < EPL; ++r) {
            if (r * LPU >= kmax) break;
#pragma unroll
            for (int l = 0; l < LPU; ++l) {
              const int t = r * LPU + l;
              const uint32_t a = __shfl_sync(FULL, soff[r], l, LPU);
              if (t < kmax) acc4<X2>(acc, ld_cluster_f4(a + (uint32_t)(pa * 4)), t < K ? wu : 0.f);
            }
          }
        } else if (kmax == 32 && fullk) {
          if (kChainRegs) chain32_regs<X2>(acc, tile_s, src_s + gi * 32, pa, wu);
          else chain32<X2, kChainB>(acc, tile_s, soff, pa, wu);
        } else {
#pragma unroll
          for (int r = 0; r < EPL; ++r) {
            if (r * LPU >= kmax) break;
#pragma unroll 4
            for (int l = 0; l < LPU; ++l) {
              const int t = r * LPU + l;
              const uint32_t so = __shfl_sync(FULL, soff[r], l, LPU);
              if (t < kmax) acc4<X2>(acc, *reinterpret_cast<const float4 *>(tile_s + so + pa), t < K ? wu : 0.f);
            }
          }
        }
        if (early) {
          if (C > 1 && kSplitRelease) {
            // arrive now (this CTA's reads of every tile are done), wait for the
            // peers only after the member stores below, then issue the load
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            cluster_arrive();
            split_pending = true;
          } else {
            release_and_load();
          }
          issued = true;
        }
        const int gmax = __reduce_max_sync(FULL, G);
        uint32_t o = 0u;
        float4 yu = make_float4(0.f, 0.f, 0.f, 0.f);
        if (ubias && G > 0) yu = out4<X2>(acc, PL.bu, ymax, o);
        const int64_t opos = (int64_t)tile * T + pa;
        float *obase = Yout + (((opos >> lgo) * R) << lgo) + (opos & ((1 << lgo) - 1));
        const int64_t rowmul = (int64_t)1 << lgo;
#pragma unroll
        for (int r = 0; r < EPL; ++r) {
          if (r * LPU >= gmax) break;
#pragma unroll 8
          for (int l = 0; l < LPU; ++l) {
            const int v = r * LPU + l;
            const int32_t dst = last ? __shfl_sync(FULL, orw[r], l, LPU) : (int32_t)__shfl_sync(FULL, soff[r], l, LPU);
            const float bv = ubias ? 0.f : __shfl_sync(FULL, bia[r], l, LPU);
            if (v < G) {
              const float4 y = ubias ? yu : out4<X2>(acc, bv, ymax, o);
              SDNN_CHECK(last ? (dst >= 0 && dst < P.yblk) : (uint32_t)dst < (uint32_t)P.R * 32u);
              if (last) *reinterpret_cast<float4 *>(obase + (int64_t)dst * rowmul) = y;
              else *reinterpret_cast<float4 *>(tile_s + dst + pa) = y;
            }
          }
        }
        uint32_t bal[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) bal[e] = __ballot_sync(FULL, (o >> e) & 1u);
        if (sll == 0 && G > 0) {
          auto spread8 = [](uint32_t x) {
            x = (x | (x << 12)) & 0x000F000Fu;
            x = (x | (x << 6)) & 0x03030303u;
            return (x | (x << 3)) & 0x11111111u;
          };
          const int sh = seg * LPU;
          const uint32_t word = spread8((bal[0] >> sh) & 0xffu) | (spread8((bal[1] >> sh) & 0xffu) << 1) |
                                (spread8((bal[2] >> sh) & 0xffu) << 2) | (spread8((bal[3] >> sh) & 0xffu) << 3);
          if (word) atomicOr(&aw[j], word);
        }
      }
      if (split_pending) {                       // (last layer, C > 1)
        cluster_wait();
        issue(it + S * ncl, b);
        split_pending = false;
      }
      __syncthreads();
    }
    if (tid == 0) {
      const int64_t base = (int64_t)tile * T;
      for (int j = 0; j < P.m; ++j) {
        uint32_t word = aw[j];
        aw[j] = 0u;
        if (base >= width) word = 0u;
        else if (width - base < 32) word &= (1u << (width - base)) - 1u;
        if (word) atomicOr(&alive[j * wstride + (base >> 5)], word);
      }
    }
    if (!issued) release_and_load();
    __syncthreads();
  }
  if (C > 1) cluster_sync();                     // no CTA exits while its peer may read its tile
}

// ---------------------------------------------------------------------------
// k_pass_gw<NW>: the fused pass for layers with per-slot weights (RW nets).
// Structure of k_pass_t32 (one 32-position tile of the component per CTA,
// one bulk copy + record, in-place slots, writer-ordered rows), but every
// member has its own chain: a warp takes one group per round and computes its
// 32 members x 32 positions as a register block -- lane = (member octet mo,
// position quad pq): 8 members x 4 positions, 32 accumulators -- per term one
// float4 of Y from shared memory and the 8 weights W_l[g][t][8mo..8mo+7] as
// two float4 from L2 (the layer's weight block stays L2-resident across the
// pass's tiles), 32 FMAs, each the canonical per-member chain (terms in
// ascending source order, fmaf from +0, then the bias add and clamp; DESIGN
// A5/A6).  Uniform layers of the same pass use the same loop with wu.
// ---------------------------------------------------------------------------
template <int NW>
__global__ void __launch_bounds__(32 * NW)
    k_pass_gw(const __grid_constant__ DevPass P, const LayerState *__restrict__ st, float *Ya, float *Yb,
              uint32_t *__restrict__ alive, int64_t wstride, float ymax, uint32_t buf_bytes) {
  constexpr int T = 32;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t *const bar = reinterpret_cast<uint64_t *>(smem_raw + (size_t)buf_bytes);
  uint32_t *const aw = reinterpret_cast<uint32_t *>(bar + 1);
  // per warp: the current group's weight block W_l[g] (<= 32 x 32 floats),
  // copied from L2 with 16-byte cp.async before its chain
  float *const wsm = reinterpret_cast<float *>(smem_raw + (size_t)buf_bytes + 128) + (threadIdx.x >> 5) * 1024;
  float *const tile_s = reinterpret_cast<float *>(smem_raw);
  const uint32_t rec_off = (uint32_t)P.R * 128u;
  const unsigned char *rec_s = smem_raw + rec_off;
  const LayerState Sx = st[P.a];
  const int width = Sx.width;
  if (width <= 0) return;
  const float *__restrict__ Yin = Sx.in ? Yb : Ya;
  float *__restrict__ Yout = Sx.in ? Ya : Yb;
  const int tiles = (width + T - 1) / T;
  const int64_t items = (int64_t)P.ncomp * tiles;
  const bool tmaj = P.order != 0;
  auto item_comp = [&](int64_t it) -> int64_t { return tmaj ? it % P.ncomp : it / tiles; };
  auto item_tile = [&](int64_t it) -> int { return (int)(tmaj ? it / P.ncomp : it % tiles); };
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int mo = lane >> 3, pq = lane & 7;       // members 8 mo .. 8 mo + 7, positions 4 pq .. 4 pq + 3
  const int pa = pq * 4;
  const int64_t R = P.yblk;
  const int lgo = P.lg_out;
  const int64_t cid = blockIdx.x, ncl = gridDim.x;
  if (tid == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int q = tid; q < P.m; q += blockDim.x) aw[q] = 0u;
  __syncthreads();
  auto issue = [&](int64_t it) {
    if (tid != 0 || it >= items) return;
    const int64_t c = item_comp(it);
    const int tile = item_tile(it);
    const int cnt = __ldg(P.in_count + c);
    mbar_expect_tx_arrive(bar, (uint32_t)cnt * 128u + (uint32_t)P.rec_bytes);
    bulk_g2s(smem_raw + rec_off, P.rec + c * P.rec_bytes, (uint32_t)P.rec_bytes, bar);
    if (cnt > 0)
      bulk_g2s(tile_s, Yin + ((int64_t)tile * R + __ldg(P.in_rows + c * P.rin)) * 32, (uint32_t)cnt * 128u, bar);
  };
  issue(cid);
  int64_t kk = 0;
  for (int64_t it = cid; it < items; it += ncl, ++kk) {
    const int tile = item_tile(it);
    mbar_wait(bar, (uint32_t)(kk & 1));
    for (int j = 0; j < P.m; ++j) {
      const PassLayerDev PL = P.layers[j];
      const bool last = j == P.m - 1;
      const bool ubias = PL.off_bias < 0;
      const uint16_t *kg_s = reinterpret_cast<const uint16_t *>(rec_s + PL.off_kg);
      const uint16_t *src_s = reinterpret_cast<const uint16_t *>(rec_s + PL.off_src);
      const float *bias_s = reinterpret_cast<const float *>(rec_s + (ubias ? 0 : PL.off_bias));
      const uint16_t *orow_s = reinterpret_cast<const uint16_t *>(rec_s + (last ? PL.off_orow : 0));
      const uint16_t *gid_s = reinterpret_cast<const uint16_t *>(rec_s + (PL.off_gid >= 0 ? PL.off_gid : 0));
      for (int u = warp; u < PL.NG; u += NW) {   // warp-uniform: one group per warp
        const uint32_t kg = kg_s[u];
        const int K = kg & 0xffu, G = kg >> 8;
        if (G == 0) continue;
        const uint32_t code = lane < K ? src_s[u * 32 + lane] : 0u;   // lane t: source t's slot
        float acc[4][8];
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[p][i] = 0.f;
        if (PL.off_gid >= 0) {
          const float *Wg = PL.wv + (size_t)gid_s[u] * PL.wk * PL.wg;   // [t][32 members], wg == 32
          for (int q = lane; q < K * 8; q += 32) cp_async16(wsm + q * 4, Wg + q * 4);
          asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
          __syncwarp();
          const float *W = wsm + mo * 8;
#pragma unroll 4
          for (int t = 0; t < K; ++t) {
            const uint32_t slot = __shfl_sync(FULL, code, t) & 0x3ffu;
            const float4 y = *reinterpret_cast<const float4 *>(tile_s + slot * 32u + pa);
            const float4 w0 = *reinterpret_cast<const float4 *>(W + t * 32);
            const float4 w1 = *reinterpret_cast<const float4 *>(W + t * 32 + 4);
            const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
            const float yv[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
            for (int p = 0; p < 4; ++p)
#pragma unroll
              for (int i = 0; i < 8; ++i) acc[p][i] = __fmaf_rn(yv[p], wv[i], acc[p][i]);
          }
        } else {                                 // a uniform layer inside a per-slot pass
#pragma unroll 4
          for (int t = 0; t < K; ++t) {
            const uint32_t slot = __shfl_sync(FULL, code, t) & 0x3ffu;
            const float4 y = *reinterpret_cast<const float4 *>(tile_s + slot * 32u + pa);
            const float yv[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
            for (int p = 0; p < 4; ++p)
#pragma unroll
              for (int i = 0; i < 8; ++i) acc[p][i] = __fmaf_rn(yv[p], PL.wu, acc[p][i]);
          }
        }
        __syncwarp();                            // every source (and weight) read before a member
                                                 // overwrites one / the next group's weights land
        const int64_t opos = (int64_t)tile * T + pa;
        float *obase = Yout + (((opos >> lgo) * R) << lgo) + (opos & ((1 << lgo) - 1));
        const int64_t rowmul = (int64_t)1 << lgo;
        uint32_t ob = 0u;                        // positions of this lane alive in some member
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int mm = mo * 8 + i;
          const uint32_t dslot = __shfl_sync(FULL, code, mm & 31) & 0x3ffu;   // in place: member mm -> slot of source mm
          const int32_t orw = (last && mm < G) ? orow_s[u * 32 + mm] : 0;
          if (mm < G) {
            const float b = ubias ? PL.bu : bias_s[u * 32 + mm];
            float4 y;
            y.x = clampy(__fadd_rn(acc[0][i], b), ymax);
            y.y = clampy(__fadd_rn(acc[1][i], b), ymax);
            y.z = clampy(__fadd_rn(acc[2][i], b), ymax);
            y.w = clampy(__fadd_rn(acc[3][i], b), ymax);
            ob |= (__float_as_uint(y.x) ? 1u : 0u) | (__float_as_uint(y.y) ? 2u : 0u) |
                  (__float_as_uint(y.z) ? 4u : 0u) | (__float_as_uint(y.w) ? 8u : 0u);
            if (last) *reinterpret_cast<float4 *>(obase + (int64_t)orw * rowmul) = y;
            else *reinterpret_cast<float4 *>(tile_s + dslot * 32u + pa) = y;
          }
        }
        // liveness word of the tile: bit 4 pq + p from any member octet
        uint32_t word = 0u;
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          uint32_t b = __ballot_sync(FULL, (ob >> p) & 1u);
          b = (b | (b >> 8) | (b >> 16) | (b >> 24)) & 0xffu;   // lane pq of any octet
          b = (b | (b << 12)) & 0x000F000Fu;                    // bit k -> bit 4 k
          b = (b | (b << 6)) & 0x03030303u;
          b = (b | (b << 3)) & 0x11111111u;
          word |= b << p;
        }
        if (lane == 0 && word) atomicOr(&aw[j], word);
      }
      if (last) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();                         // every read of the tile and record is done
        issue(it + ncl);
      } else {
        __syncthreads();                         // the next layer reads slots other warps wrote
      }
    }
    if (tid == 0) {
      const int64_t base = (int64_t)tile * T;
      for (int j = 0; j < P.m; ++j) {
        uint32_t word = aw[j];
        aw[j] = 0u;
        if (base >= width) word = 0u;
        else if (width - base < 32) word &= (1u << (width - base)) - 1u;
        if (word) atomicOr(&alive[j * wstride + (base >> 5)], word);
      }
    }
    __syncthreads();
  }
}

template <int NW>
static void launch_gw(const LaunchCfg &c, const Workspace &w, const DevPass &P, uint32_t *alive, float ymax,
                      cudaStream_t s) {
  const uint32_t bb = (uint32_t)(((size_t)P.R * 128 + P.rec_bytes + 127) / 128 * 128);
  const size_t smem = (size_t)bb + 128 + (size_t)NW * 4096;   // + barrier, liveness words, weight blocks
  static std::atomic<size_t> set_smem[kMaxDevices];   // per device: the largest size configured
  const int dev = current_device();
  if (smem > set_smem[dev].load()) {
    cudaFuncSetAttribute(k_pass_gw<NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    set_smem[dev] = smem;
  }
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_pass_gw<NW>, 32 * NW, smem) != cudaSuccess || occ <= 0) {
    cudaGetLastError();
    occ = 1;
  }
  k_pass_gw<NW><<<c.sms * occ, 32 * NW, smem, s>>>(P, w.st, w.Y[0], w.Y[1], alive, w.words, ymax, bb);
}

void launch_pass_gw(const LaunchCfg &c, const Workspace &w, const DevPass &P, uint32_t *alive, float ymax,
                    cudaStream_t s) {
  if (P.NW <= 4) launch_gw<4>(c, w, P, alive, ymax, s);
  else launch_gw<8>(c, w, P, alive, ymax, s);
}

// (NW, S) instances: NW = ceil(rows / 128) warps, S buffers
#define SDNN_T32_VARIANTS(X) X(1, 1) X(1, 2) X(1, 3) X(2, 1) X(2, 2) X(2, 3) X(4, 1) X(4, 2)
#define SDNN_T32C_VARIANTS(X) X(4, 1)           // clusters (2 or 4 CTAs)

static uint32_t t32_buf_bytes(const DevPass &P) {
  return (uint32_t)(((size_t)P.R * 128 + P.rec_bytes + 127) / 128 * 128);
}
static size_t t32_smem(const DevPass &P, int S) { return (size_t)S * t32_buf_bytes(P) + 8 * S + 4 * kMaxPassLayers; }

bool pass_t32_variant(int nw, int s, int c) {
#define X(NN, SS) if (c == 1 && nw == NN && s == SS) return true;
  SDNN_T32_VARIANTS(X)
#undef X
#define X(NN, SS) if ((c == 2 || c == 4) && nw == NN && s == SS) return true;
  SDNN_T32C_VARIANTS(X)
#undef X
  return false;
}
// 513-1024-row components (SDNN_PASS_WIDE): 2 = 2-CTA clusters of k_pass_t32
// for passes of >= 3 layers and k_pass_wide for 2-layer passes (default; C4
// 1024-row 3-layer passes 3.03 vs 3.35 ms; on the plain schedule, whose
// 1024-row passes have 2 layers, half the terms of a 2-layer pass are remote:
// C4-plain 2742 ms/step with clusters vs 2567 with k_pass_wide), 1 =
// k_pass_wide always, 0 = 16-position k_pass tiles (3.45 ms)
int pass_wide_mode() {
  static const int v = [] {
    const char *e = getenv("SDNN_PASS_WIDE");
    return e ? atoi(e) : 2;
  }();
  return v;
}
size_t pass_t32_smem_max() { return 227 * 1024; }

template <int NW, int S, bool X2, int C>
static void launch_t32(const LaunchCfg &c, const Workspace &w, const DevPass &P, uint32_t *alive, float ymax,
                       cudaStream_t s) {
  const size_t smem = t32_smem(P, S);
  static std::atomic<size_t> set_smem[kMaxDevices];   // per device: the largest size configured
  const int dev = current_device();
  if (smem > set_smem[dev].load()) {
    cudaFuncSetAttribute(k_pass_t32<NW, S, X2, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    set_smem[dev] = smem;
  }
  if (C == 1) {
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_pass_t32<NW, S, X2, C>, 32 * NW, smem) !=
            cudaSuccess ||
        occ <= 0) {
      cudaGetLastError();
      occ = 1;
    }
    k_pass_t32<NW, S, X2, C><<<c.sms * occ, 32 * NW, smem, s>>>(P, w.st, w.Y[0], w.Y[1], alive, w.words, ymax,
                                                               t32_buf_bytes(P));
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cfg.blockDim = dim3(32 * NW);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.gridDim = dim3(C * c.sms);
  int ncl = 0;
  if (cudaOccupancyMaxActiveClusters(&ncl, k_pass_t32<NW, S, X2, C>, &cfg) != cudaSuccess || ncl <= 0) {
    cudaGetLastError();
    ncl = c.sms / C;
  }
  cfg.gridDim = dim3(C * ncl);
  cudaLaunchKernelEx(&cfg, k_pass_t32<NW, S, X2, C>, P, (const LayerState *)w.st, w.Y[0], w.Y[1], alive,
                     (int64_t)w.words, ymax, t32_buf_bytes(P));
}

void launch_pass_t32(const LaunchCfg &c, const Workspace &w, const DevPass &P, uint32_t *alive, float ymax,
                     cudaStream_t s) {
  const bool x2 = wide_x2();
#define X(NN, SS)                                                      \
  if (P.C == 1 && P.NW == NN && P.S == SS) {                           \
    if (x2) launch_t32<NN, SS, true, 1>(c, w, P, alive, ymax, s);      \
    else launch_t32<NN, SS, false, 1>(c, w, P, alive, ymax, s);        \
    return;                                                            \
  }
  SDNN_T32_VARIANTS(X)
#undef X
#define X(NN, SS)                                                      \
  if (P.C == 2 && P.NW == NN && P.S == SS) {                           \
    if (x2) launch_t32<NN, SS, true, 2>(c, w, P, alive, ymax, s);      \
    else launch_t32<NN, SS, false, 2>(c, w, P, alive, ymax, s);        \
    return;                                                            \
  }                                                                    \
  if (P.C == 4 && P.NW == NN && P.S == SS) {                           \
    if (x2) launch_t32<NN, SS, true, 4>(c, w, P, alive, ymax, s);      \
    else launch_t32<NN, SS, false, 4>(c, w, P, alive, ymax, s);        \
    return;                                                            \
  }
  SDNN_T32C_VARIANTS(X)
#undef X
  fprintf(stderr, "sdnn: no k_pass_t32 instance for NW=%d S=%d C=%d\n", P.NW, P.S, P.C);
  abort();
}

// planner switch: components of <= 512 rows in the blocked layout get
// k_pass_t32 (SDNN_PASS_T32: 0 off, 1 up to 256 rows, 2 up to 512 rows);
// buffers per CTA by warps (SDNN_PASS_T32_S = "s1,s2,s4" for 1 / 2 / 4 warps).
// Measured on C4 (ms/step): k_pass everywhere 1906; t32 for <= 256 rows with
// S = 1: 1894, S = 2: 1870; t32 up to 512 rows: S = 1 1838, S = 2 2678 (two
// 64 KB tiles leave one CTA per SM)
int pass_t32_mode() {
  static const int v = [] {
    const char *e = getenv("SDNN_PASS_T32");
    return e ? atoi(e) : 2;
  }();
  return v;
}
int pass_t32_stages(int nw) {
  static const std::array<int, 3> v = [] {
    std::array<int, 3> r = {2, 2, 1};
    if (const char *e = getenv("SDNN_PASS_T32_S")) {
      int a = 0, b = 0, c = 0;
      const int k = sscanf(e, "%d,%d,%d", &a, &b, &c);
      if (k == 1) r = {a, a, a};
      else if (k == 3) r = {a, b, c};
      for (int &x : r) x = std::max(1, std::min(3, x));
    }
    return r;
  }();
  return v[nw <= 1 ? 0 : nw == 2 ? 1 : 2];
}

}  // namespace sdnn
