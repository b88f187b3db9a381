// device_util.cuh -- small device helpers shared by the product kernels
// (kernels.cu, chain.cu): canonical clamp, vector load/store, liveness-bit
// publication, mbarrier and cp.async.bulk (TMA bulk copy) wrappers.
#pragma once
#include <cstdint>

namespace sdnn {

#define FULL 0xffffffffu

// min(max(z, 0), ymax) with the canonical reading z > 0 ? min(z, ymax) : +0
// (A6).  The two agree bit for bit because z is never -0 here: every
// chain starts at acc = +0 and a round-to-nearest sum (fma or add) is -0 only
// when both addends are -0, so acc and z = acc + b are never -0; NaN -> +0 in
// both.  Two FMNMX instead of FSETP + FMNMX + FSEL.
__device__ __forceinline__ float clampy(float z, float ymax) {
  return fminf(fmaxf(z, 0.f), ymax);
}


// Lane arithmetic on 4 consecutive positions.  X2: packed fp32x2 FFMA2 / FADD2
// (sm_100; per component identical to __fmaf_rn / __fadd_rn).
template <bool X2>
__device__ __forceinline__ void acc4(float (&a)[4], const float4 &v, float w) {
  if (X2) {
    const float2 w2 = make_float2(w, w);
    const float2 lo = __ffma2_rn(make_float2(v.x, v.y), w2, make_float2(a[0], a[1]));
    const float2 hi = __ffma2_rn(make_float2(v.z, v.w), w2, make_float2(a[2], a[3]));
    a[0] = lo.x;
    a[1] = lo.y;
    a[2] = hi.x;
    a[3] = hi.y;
  } else {
    a[0] = __fmaf_rn(v.x, w, a[0]);
    a[1] = __fmaf_rn(v.y, w, a[1]);
    a[2] = __fmaf_rn(v.z, w, a[2]);
    a[3] = __fmaf_rn(v.w, w, a[3]);
  }
}
// y = clamp(acc + b); o |= bit pattern (y is +0 exactly when dead: z is never -0)
template <bool X2>
__device__ __forceinline__ float4 out4(const float (&a)[4], float b, float ymax, uint32_t &o) {
  float4 y;
  if (X2) {
    const float2 b2 = make_float2(b, b);
    const float2 lo = __fadd2_rn(make_float2(a[0], a[1]), b2);
    const float2 hi = __fadd2_rn(make_float2(a[2], a[3]), b2);
    y = make_float4(clampy(lo.x, ymax), clampy(lo.y, ymax), clampy(hi.x, ymax), clampy(hi.y, ymax));
  } else {
    y = make_float4(clampy(__fadd_rn(a[0], b), ymax), clampy(__fadd_rn(a[1], b), ymax),
                    clampy(__fadd_rn(a[2], b), ymax), clampy(__fadd_rn(a[3], b), ymax));
  }
  o |= (__float_as_uint(y.x) ? 1u : 0u) | (__float_as_uint(y.y) ? 2u : 0u) |
       (__float_as_uint(y.z) ? 4u : 0u) | (__float_as_uint(y.w) ? 8u : 0u);
  return y;
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

// AND per-lane "all outputs saturated" bits of a tile into sat[] (only words
// that lose a bit are touched)
template <int VEC>
__device__ __forceinline__ void publish_sat(uint32_t sm, int lane, int64_t tile_pos, int width,
                                            uint32_t *sat) {
  uint32_t bal[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) bal[e] = __ballot_sync(FULL, (sm >> e) & 1u);
  if (lane < VEC) {
    uint32_t word = 0;
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const int pos = lane * 32 + q;
      const int src_lane = pos / VEC, e = pos % VEC;
      uint32_t b = 0;
#pragma unroll
      for (int ee = 0; ee < VEC; ++ee)
        if (ee == e) b = (bal[ee] >> src_lane) & 1u;
      word |= b << q;
    }
    const int64_t base = tile_pos + lane * 32;
    if (base < width && word != 0xffffffffu) atomicAnd(&sat[base >> 5], word);
  }
}

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
// bulk prefetch of a global range into L2 (no completion tracking)
__device__ __forceinline__ void bulk_prefetch_l2(const void *src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// TMA tile load of a 3D box (tensor map in param/const/global space)
__device__ __forceinline__ void tma_load_3d(void *dst, const void *tmap, int c0, int c1, int c2, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(smem_u32(dst)), "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---- thread-block clusters / distributed shared memory ----
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t nclusters_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
// all threads of all CTAs of the cluster; release/acquire orders shared::cluster
// accesses across the barrier
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// the two halves of cluster_sync, for work between them
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cta address -> the same offset in CTA `rank`'s window (shared::cluster)
__device__ __forceinline__ uint32_t cluster_map(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// volatile (stays between the cluster barriers around it) but no memory
// clobber, so independent loads can be issued back to back
__device__ __forceinline__ float4 ld_cluster_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}

__device__ __forceinline__ float2 ld_cluster_f2(uint32_t addr) {
  float2 v;
  asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr) : "memory");
  return v;
}

// 16-byte cp.async (LDGSTS, L2 only) global -> shared
__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
// arrive on `bar` once all of this thread's prior cp.async have landed (the
// barrier's expected count must include one arrival per calling thread)
__device__ __forceinline__ void cp_async_arrive(uint64_t *bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

}  // namespace sdnn
