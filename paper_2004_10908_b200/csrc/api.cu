// api.cu -- the C ABI of include/sdnn.h: handle lifetime, streamed layer
// loading into resident HBM, workspace management, the whole-network launch
// (one captured CUDA Graph of the layer chain, "a cudaFlow maps
// to a CUDA graph that can be executed using a single CPU call"), and the
// host-buffer end-to-end call.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <cudaTypedefs.h>

#include "../../include/sdnn.h"
#include "sdnn_internal.h"

using namespace sdnn;

namespace {

thread_local std::string g_err = "";

sdnn_status fail(sdnn_status s, const std::string &m) {
  g_err = m;
  return s;
}

// bump allocator over large cudaMalloc chunks (layers are loaded once, freed
// together at destroy)
struct Arena {
  std::vector<void *> chunks;
  char *cur = nullptr;
  size_t left = 0;
  size_t total = 0;
  std::mutex mu;
  static constexpr size_t kChunk = size_t(256) << 20;
  cudaError_t alloc(size_t bytes, void **out) {
    std::lock_guard<std::mutex> g(mu);
    bytes = (bytes + 255) & ~size_t(255);
    if (bytes > left) {
      const size_t sz = std::max(bytes, kChunk);
      void *p = nullptr;
      cudaError_t e = cudaMalloc(&p, sz);
      if (e != cudaSuccess) return e;
      chunks.push_back(p);
      cur = (char *)p;
      left = sz;
    }
    *out = cur;
    cur += bytes;
    left -= bytes;
    total += bytes;
    return cudaSuccess;
  }
  void release() {
    for (void *p : chunks) cudaFree(p);
    chunks.clear();
    cur = nullptr;
    left = 0;
  }
};

}  // namespace

// one input slot of the host-buffer inference (api.cu host_enqueue)
struct HostSlot {
  int64_t *d_rowptr = nullptr;
  int32_t *d_idx = nullptr;
  float *d_val = nullptr;
  int64_t cap_rows = -1, cap_nnz = -1, cap_val = -1;
  int32_t *h_res = nullptr;            // pinned: [0] = category count, [1..] = ids
  int64_t h_res_cap = 0, batch = 0;
  cudaEvent_t done = nullptr;          // result copied back
  cudaEvent_t in_free = nullptr;       // the slot's device input buffers consumed
  std::thread validator;
  sdnn_status vst = SDNN_OK;
  std::string vmsg;
};

struct sdnn_net {
  int32_t n = 0, L = 0;
  sdnn_opts opts{-1, 0u, 32.f, nullptr, -1, -1, -1, 0};
  int device = 0;
  cudaStream_t own = nullptr;
  // a pageable cudaMemcpy may return before its DMA lands, and the streams are
  // non-blocking: the first inference after an upload synchronises the device
  std::atomic<bool> uploads_pending{false};
  Arena arena;
  std::vector<DevLayer> dl;
  std::vector<PackedLayer> host;   // host copy of every packed layer (pass planning)
  std::vector<uint8_t> set;        // layer loaded?
  std::vector<void *> lblock;      // per layer: its arena block (reused on re-set)
  std::vector<size_t> lbytes;
  std::vector<uint8_t> bias_nonpos;
  std::vector<int64_t> nnz;
  std::vector<int64_t> fma_l;      // FMAs per batch position of layer l (sum K_g if uniform, else nnz)
  std::atomic<int> nset{0};
  int32_t grouped_layers = 0, max_group = 0, max_k = 0;
  std::mutex stat_mu;
  bool sticky = false;
  LaunchCfg cfg;
  // workspace
  Workspace ws;
  int64_t ws_cap = -1;             // stride the workspace was sized for
  // execution plan: steps of one layer or one fused multi-layer pass
  std::vector<Step> steps;
  std::vector<int8_t> step_lg;         // per step: log2 positions per block of its input boundary
  std::vector<DevPass> passes;
  Arena pass_arena;
  bool plan_dirty = true;
  int64_t plan_gen = 0;                // bumped by every make_plan
  float *tmap_y[2] = {nullptr, nullptr};   // buffers the pass tensor maps were encoded for
  int64_t tmap_plan = -1;
  int32_t fused_layers = 0;
  int32_t resident_layers = 0;
  ResLayerDev *d_res = nullptr;        // device table for the resident step (pass_arena)
  int32_t yblk = 0;                    // plan: position-blocked activations (Workspace::yblk)
  const int32_t *d_sig0 = nullptr;     // plan: input storage order (pass_arena)
  std::vector<uint8_t> sat_suffix;     // f2: layers [l, L) all saturation-preserving
  // f3 weight streaming (opts.stream_slots > 0): every step's weight block in one
  // pinned host buffer, copied into a ring of device slots during the chain
  std::vector<DevLayer> step_dl;       // per step: layer view into its slot
  unsigned char *h_wblob = nullptr;
  std::vector<size_t> wb_off, wb_bytes;
  unsigned char *d_slots = nullptr;    // [stream_slots][slot_bytes] (pass_arena)
  size_t slot_bytes = 0;
  int64_t stream_bytes = 0;
  cudaStream_t copy_s = nullptr;
  std::vector<cudaEvent_t> ev_ready, ev_done;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // captured layer chain
  cudaGraphExec_t chain = nullptr;
  bool chain_compact = false;
  int64_t chain_launches = 0;
  // host-buffer inference: two input slots (sdnn_infer uses slot 0;
  // sdnn_infer_submit alternates) and the outstanding tickets
  HostSlot slots[2];
  int64_t pending[2] = {-1, -1};
  int64_t next_ticket = 0;
  // input stream of sdnn_infer, its events (staging slots, per-chunk arrival)
  cudaStream_t in_s = nullptr;
  cudaEvent_t ev_stage[2] = {nullptr, nullptr};
  cudaEvent_t ev_in = nullptr;
  std::vector<cudaEvent_t> ev_chunk;
  // pinned host staging
  void *h_stage = nullptr;
  size_t h_stage_cap = 0;
  int32_t *h_cats = nullptr;
  int64_t h_cats_cap = 0;
  // per-layer timing events (SDNN_F_PROFILE)
  std::vector<cudaEvent_t> ev_before, ev_after;
  bool profiled = false;
  // stats
  int64_t last_batch = 0, last_ncat = 0, launches = 0;
  std::vector<int32_t> last_live;
};

namespace {

#define CK(call)                                                                 \
  do {                                                                           \
    cudaError_t _e = (call);                                                     \
    if (_e != cudaSuccess) {                                                     \
      net->sticky = true;                                                        \
      return fail(SDNN_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
    }                                                                            \
  } while (0)

#define CKN(NET, call)                                                           \
  do {                                                                           \
    cudaError_t _e = (call);                                                     \
    if (_e != cudaSuccess) {                                                     \
      (NET)->sticky = true;                                                      \
      return fail(SDNN_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
    }                                                                            \
  } while (0)

bool compact_enabled(const sdnn_net *net) {
  if (net->opts.flags & SDNN_F_NO_COMPACT) return false;
  if (net->L < 1) return false;
  for (int l = 0; l < net->L; ++l)
    if (!net->bias_nonpos[l]) return false;     // a dead row could revive (reading A2/I2)
  return true;
}

sdnn_status check_opts(const sdnn_opts *o, sdnn_opts &out) {
  out = sdnn_opts{-1, 0u, 32.f, nullptr, -1, -1, -1, 0};
  if (o) out = *o;
  if (out.stream_slots < 0 || out.stream_slots > 64) return fail(SDNN_E_ARG, "stream_slots must be in [0, 64]");
  if (out.fuse_rows > kMaxPassRows * kMaxPassCluster) out.fuse_rows = kMaxPassRows * kMaxPassCluster;
  if (out.fuse_layers > kMaxPassLayers) return fail(SDNN_E_ARG, "fuse_layers > 16");
  if (!(out.ymax > 0.f) || !std::isfinite(out.ymax)) return fail(SDNN_E_ARG, "ymax must be finite and > 0");
  return SDNN_OK;
}

sdnn_status set_device(sdnn_net *net) {
  if (net->sticky) return fail(SDNN_E_CUDA, "handle is in a failed CUDA state; destroy it");
  CK(cudaSetDevice(net->device));
  return SDNN_OK;
}

void free_ws(sdnn_net *net) {
  Workspace &w = net->ws;
  for (int i = 0; i < 2; ++i) {
    cudaFree(w.Y[i]);
    cudaFree(w.rid[i]);
    cudaFree(w.alive[i]);
    w.Y[i] = nullptr;
    w.rid[i] = nullptr;
    w.alive[i] = nullptr;
  }
  cudaFree(w.inmask);
  cudaFree(w.wpre);
  cudaFree(w.st);
  cudaFree(w.live);
  cudaFree(w.cats);
  cudaFree(w.ncat);
  cudaFree(w.sat[0]);
  cudaFree(w.sat[1]);
  cudaFree(w.retired);
  cudaFree(w.pret);
  cudaFree(w.nretired);
  cudaFree(w.orig);
  w = Workspace();
  if (net->chain) cudaGraphExecDestroy(net->chain);
  net->chain = nullptr;
  net->ws_cap = -1;
}

sdnn_status ensure_ws(sdnn_net *net, int64_t batch) {
  // row stride: whole tiles plus a skew so that row starts are not aligned to a
  // large power of two (the 32 source segments of an item would otherwise share
  // their low address bits); one extra tile at the end keeps the last row's tail
  // tile inside the allocation
  const int64_t q = bulk_stride_quantum();
  static const int64_t skew = [] {
    const char *e = getenv("SDNN_SKEW");
    return e ? std::max<int64_t>(0, atoll(e)) / 32 * 32 : int64_t(1024);
  }();
  const int64_t stride = std::max<int64_t>(q, (batch + q - 1) / q * q) + skew;
  if (net->ws_cap >= stride) return SDNN_OK;
  free_ws(net);
  if ((int64_t)net->n * stride > (int64_t(1) << 36)) return fail(SDNN_E_UNSUPPORTED, "batch too large");
  Workspace &w = net->ws;
  w.stride = stride;
  w.words = stride / 32;
  const size_t ybytes = sizeof(float) * ((size_t)net->n * (size_t)stride + (size_t)q);
  for (int i = 0; i < 2; ++i) {
    if (cudaMalloc(&w.Y[i], ybytes) != cudaSuccess) {
      cudaGetLastError();
      free_ws(net);
      return fail(SDNN_E_NOMEM, "cannot allocate activation buffers (" + std::to_string(2 * ybytes) + " B)");
    }
    CK(cudaMalloc(&w.rid[i], sizeof(int32_t) * stride));
    CK(cudaMalloc(&w.alive[i], sizeof(uint32_t) * w.words * kMaxPassLayers));
  }
  CK(cudaMemset(w.Y[1], 0, ybytes));
  CK(cudaMalloc(&w.inmask, sizeof(uint32_t) * w.words));
  CK(cudaMalloc(&w.wpre, sizeof(int32_t) * (w.words + 1)));
  CK(cudaMalloc(&w.st, sizeof(LayerState) * (net->L + 1)));
  CK(cudaMalloc(&w.live, sizeof(int32_t) * std::max(1, net->L)));
  CK(cudaMalloc(&w.cats, sizeof(int32_t) * stride));
  CK(cudaMalloc(&w.ncat, sizeof(int32_t)));
  if (net->opts.flags & SDNN_F_SATURATE) {
    CK(cudaMalloc(&w.sat[0], sizeof(uint32_t) * w.words));
    CK(cudaMalloc(&w.sat[1], sizeof(uint32_t) * w.words));
    CK(cudaMalloc(&w.retired, sizeof(uint32_t) * w.words));
    CK(cudaMalloc(&w.pret, sizeof(uint32_t) * w.words));
    CK(cudaMalloc(&w.nretired, sizeof(int32_t)));
    CK(cudaMalloc(&w.orig, sizeof(uint32_t) * w.words));
  }
  net->ws_cap = stride;
  return SDNN_OK;
}

int nthreads_default() {
  unsigned h = std::thread::hardware_concurrency();
  return (int)std::max(1u, std::min(h, 32u));
}

bool weight_streaming(const sdnn_net *net) { return net->opts.stream_slots > 0; }

void free_stream(sdnn_net *net) {
  if (net->h_wblob) cudaFreeHost(net->h_wblob);
  net->h_wblob = nullptr;
  for (auto e : net->ev_ready) cudaEventDestroy(e);
  for (auto e : net->ev_done) cudaEventDestroy(e);
  net->ev_ready.clear();
  net->ev_done.clear();
  net->d_slots = nullptr;                          // lives in pass_arena
  net->slot_bytes = 0;
  net->stream_bytes = 0;
}

constexpr size_t kBlobAlign = 256;
size_t blob_align(size_t x) { return (x + kBlobAlign - 1) & ~(kBlobAlign - 1); }

// f3: lay out every step's weight block (a layer's packed arrays or a fused
// pass's row lists and records) in one pinned host buffer; point the per-step
// device views into ring slot (step mod S)
sdnn_status build_stream_blobs(sdnn_net *net, const std::vector<PassHost> &ph) {
  const int ns = (int)net->steps.size();
  const int S = net->opts.stream_slots;
  net->wb_off.assign(ns, 0);
  net->wb_bytes.assign(ns, 0);
  net->step_dl.assign(ns, DevLayer{});
  // per-step part sizes
  struct Part { const void *h; size_t bytes; };
  std::vector<std::vector<Part>> parts(ns);
  for (int i = 0; i < ns; ++i) {
    const Step &S_ = net->steps[i];
    if (S_.m == 1) {
      const PackedLayer &p = net->host[S_.a];
      parts[i] = {{p.src.data(), p.src.size() * 2}, {p.col.data(), p.col.size() * 4},
                  {p.gk.data(), p.gk.size() * 4}, {p.gg.data(), p.gg.size() * 4},
                  {p.val.data(), p.uniform ? 0 : p.val.size() * 4}, {p.bias.data(), p.bias.size() * 4},
                  {p.gbias.data(), p.gbias.size() * 4}};
    } else {
      const PassHost &H = ph[i];
      parts[i] = {{H.in_rows.data(), H.in_rows.size() * 4}, {H.in_count.data(), H.in_count.size() * 4},
                  {H.rec.data(), H.rec.size()}};
    }
  }
  size_t total = 0, smax = 0;
  for (int i = 0; i < ns; ++i) {
    size_t b = 0;
    for (auto &q : parts[i]) b += blob_align(q.bytes);
    net->wb_off[i] = total;
    net->wb_bytes[i] = b;
    total += b;
    smax = std::max(smax, b);
  }
  if (cudaHostAlloc((void **)&net->h_wblob, std::max<size_t>(total, 1), cudaHostAllocDefault) != cudaSuccess) {
    cudaGetLastError();
    net->h_wblob = nullptr;
    return fail(SDNN_E_NOMEM, "pinned host allocation for weight streaming failed");
  }
  void *d = nullptr;
  if (net->pass_arena.alloc(std::max<size_t>(smax, 1) * S, &d) != cudaSuccess) {
    cudaGetLastError();
    return fail(SDNN_E_NOMEM, "device allocation for the weight-streaming ring failed");
  }
  net->d_slots = (unsigned char *)d;
  net->slot_bytes = smax;
  net->stream_bytes = (int64_t)total;
  for (int i = 0; i < ns; ++i) {
    unsigned char *h = net->h_wblob + net->wb_off[i];
    unsigned char *dv = net->d_slots + (size_t)(i % S) * smax;
    std::vector<unsigned char *> at;
    size_t o = 0;
    for (auto &q : parts[i]) {
      if (q.bytes) std::memcpy(h + o, q.h, q.bytes);
      at.push_back(q.bytes ? dv + o : nullptr);
      o += blob_align(q.bytes);
    }
    const Step &S_ = net->steps[i];
    if (S_.m == 1) {
      DevLayer dl = net->dl[S_.a];                 // metadata (sizes, uniform value)
      dl.src = (const uint16_t *)at[0];
      dl.col = (const int32_t *)at[1];
      dl.gk = (const int32_t *)at[2];
      dl.gg = (const int32_t *)at[3];
      dl.val = net->host[S_.a].uniform ? nullptr : (const float *)at[4];
      dl.bias = (const float *)at[5];
      dl.gbias = (const float *)at[6];
      net->step_dl[i] = dl;
    } else {
      DevPass &D = net->passes[S_.pass];
      D.in_rows = (const int32_t *)at[0];
      D.in_count = (const int32_t *)at[1];
      D.rec = (const unsigned char *)at[2];
    }
  }
  net->ev_ready.resize(ns);
  net->ev_done.resize(ns);
  for (int i = 0; i < ns; ++i) {
    CK(cudaEventCreateWithFlags(&net->ev_ready[i], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&net->ev_done[i], cudaEventDisableTiming));
  }
  if (!net->copy_s) CK(cudaStreamCreateWithFlags(&net->copy_s, cudaStreamNonBlocking));
  if (!net->ev_fork) CK(cudaEventCreateWithFlags(&net->ev_fork, cudaEventDisableTiming));
  if (!net->ev_join) CK(cudaEventCreateWithFlags(&net->ev_join, cudaEventDisableTiming));
  return SDNN_OK;
}

// Plan the steps (fused passes where the component cap allows) and upload the
// pass descriptors.  Create-time work, redone only when layers change.
// position-blocked activations wanted (default on; SDNN_YBLOCK=0 disables)
bool yblock_wanted() {
  const char *e = getenv("SDNN_YBLOCK");
  return e ? atoi(e) != 0 : kYBlockDefault;
}

// fused-pass item order: -1 = by tile size (default: component-major for the
// 16-position tiles of 1024-row components, tile-major otherwise; measured on
// C4: k_pass<32> 2.52 vs 2.67 ms, <128> 2.75 vs 2.84, <64> 2.61 vs 2.72, but
// <16> 4.23 vs 3.40 ms tile-major vs component-major); SDNN_PASS_ORDER=comp|tile
int pass_order() {
  static const int v = [] {
    const char *e = getenv("SDNN_PASS_ORDER");
    if (e && std::strcmp(e, "tile") == 0) return 1;
    if (e && std::strcmp(e, "comp") == 0) return 0;
    return -1;
  }();
  return v;
}

sdnn_status make_plan(sdnn_net *net) {
  if (!net->plan_dirty) return SDNN_OK;
  const bool sat = net->opts.flags & SDNN_F_SATURATE;
  net->sat_suffix.assign(net->L + 1, 1);
  for (int l = net->L - 1; l >= 0; --l)
    net->sat_suffix[l] = net->sat_suffix[l + 1] && saturation_preserving(net->host[l], net->opts.ymax);
  const int maxm = net->opts.fuse_layers < 0 ? 8 : net->opts.fuse_layers;
  // the SMEM-resident tail (N <= 4096) starts at layer ar; fused passes never cross it
  int ar = net->L;
  std::vector<std::vector<unsigned char>> blobs;
  std::vector<ResLayerDev> rl;
  if (!(net->opts.flags & (SDNN_F_NO_RESIDENT | SDNN_F_SATURATE)) && !weight_streaming(net) &&
      resident_positions(net->n) > 0 && (net->opts.resident_from >= 0 || net->n <= kResidentDefaultMaxN)) {
    int a0 = net->opts.resident_from >= 0 ? net->opts.resident_from : (net->L > 32 ? 24 : net->L);
    a0 = std::min(a0, net->L);
    bool ok = a0 < net->L;
    blobs.resize(ok ? net->L - a0 : 0);
    rl.resize(blobs.size());
    for (int l = a0; ok && l < net->L; ++l) ok = build_resident_blob(net->host[l], blobs[l - a0], rl[l - a0]);
    if (ok) ar = a0;
  }
  std::vector<const PackedLayer *> lp(net->L);
  for (int l = 0; l < net->L; ++l) lp[l] = &net->host[l];
  std::vector<const PackedLayer *> head(lp.begin(), lp.begin() + ar);
  std::vector<PassHost> ph;
  const bool want_yblk = yblock_wanted() && !weight_streaming(net) && !sat && ar == net->L;
  // position-blocked plans put up to 1024 rows in a CTA (16-position tiles);
  // (merging small components into full 512-row CTAs for the blocked layout was
  // measured no faster on C4: 2080 vs 2069 ms/step)
  auto plan_for = [&](bool blocked) {
    const int cta = pass_cta_rows(blocked);
    const int cap = sat ? 0 : std::min(net->opts.fuse_rows < 0 ? kDefaultPassRows : net->opts.fuse_rows,
                                       cta * kMaxPassCluster);
    net->steps = plan_passes(head, net->n, cap, maxm, pass_tile_floats(), nthreads_default(), &ph, cta,
                             blocked, (net->opts.flags & SDNN_F_SHARE_VALUES) != 0);
  };
  plan_for(want_yblk);
  if (want_yblk) {
    // the blocked layout needs every step to be a fused pass; otherwise plan
    // again for row-major activations (<= 512 rows per CTA, no one-layer passes)
    bool all = net->L > 0 && !net->steps.empty();
    for (size_t q = 0; q < ph.size(); ++q) all = all && ph[q].m > 0;
    if (!all) {
      ph.clear();
      plan_for(false);
    }
  }
  net->pass_arena.release();
  free_stream(net);
  net->passes.clear();
  net->fused_layers = 0;
  const bool streaming = weight_streaming(net);
  auto up = [&](const void *h, size_t bytes, void **d) -> sdnn_status {
    cudaError_t e = net->pass_arena.alloc(std::max<size_t>(bytes, 4), d);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(SDNN_E_NOMEM, "device allocation for pass descriptors failed");
    }
    if (bytes) CK(cudaMemcpy(*d, h, bytes, cudaMemcpyHostToDevice));
    net->uploads_pending = true;
    return SDNN_OK;
  };
  // Position-blocked activations (SDNN_YBLOCK; only when every step is a fused
  // pass): at the input boundary of each pass the neurons get a storage order
  // in which every (component, CTA) row list is consecutive, so a tile's
  // 32-position blocks are single contiguous runs; the final boundary keeps
  // the identity order.  in_rows and the last layer's output rows are
  // rewritten to storage rows; the input scatter uses sig0.
  bool yblk = want_yblk && net->L > 0 && !net->steps.empty();
  for (size_t q = 0; q < ph.size(); ++q) yblk = yblk && ph[q].m > 0;   // every step a pass
  std::vector<int32_t> sig0;
  if (yblk) {
    const int n = net->n;
    const size_t ns = net->steps.size();
    std::vector<std::vector<int32_t>> sig(ns);
    for (size_t q = 0; q < ns; ++q) {
      const PassHost &H = ph[q];
      std::vector<int32_t> &sq = sig[q];
      sq.assign(n, -1);
      int32_t next = 0;
      for (int64_t cb = 0; cb < (int64_t)H.ncomp * H.C; ++cb)
        for (int i = 0; i < H.in_count[cb]; ++i) sq[H.in_rows[cb * H.rin + i]] = next++;
      for (int j = 0; j < n; ++j)
        if (sq[j] < 0) sq[j] = next++;
    }
    for (size_t q = 0; q < ns; ++q) {
      PassHost &H = ph[q];
      for (auto &r : H.in_rows)
        if (r >= 0) r = sig[q][r];
      if (q + 1 < ns) {
        const PassHostLayer &HL = H.layers[H.m - 1];
        for (int64_t cb = 0; cb < (int64_t)H.ncomp * H.C; ++cb) {
          uint16_t *orow = reinterpret_cast<uint16_t *>(H.rec.data() + cb * H.rec_bytes + HL.off_orow);
          for (int k = 0; k < HL.NG * 32; ++k) orow[k] = (uint16_t)sig[q + 1][orow[k]];
        }
      }
    }
    sig0 = std::move(sig[0]);
  }
  net->yblk = yblk ? net->n : 0;
  // block size per boundary: 16 positions where a T = 16 pass (1024-row
  // components) reads, so its tile is one contiguous run (SDNN_BLK16=0: 32)
  // (off by default: the passes writing 16-position blocks lose more than the
  // T = 16 passes gain -- C4 1998 vs 1964 ms/step; SDNN_BLK16=1 enables)
  static const bool blk16 = [] {
    const char *e = getenv("SDNN_BLK16");
    return e && atoi(e) != 0;
  }();
  static const int pf = [] {
    const char *e = getenv("SDNN_PASS_PF");
    return e ? std::max(0, std::min(4, atoi(e))) : 0;   // measured: PF=1 2586, PF=2 2653 vs 1978 ms on C4
  }();
  net->step_lg.assign(net->steps.size() + 1, 5);
  if (yblk && blk16)
    for (size_t q = 0; q < net->steps.size(); ++q)
      if (ph[q].m > 0 && ph[q].T == 16 && ph[q].C == 1) net->step_lg[q] = 4;
  net->d_sig0 = nullptr;
  if (yblk) {
    void *d;
    sdnn_status st2 = up(sig0.data(), sig0.size() * 4, &d);
    if (st2) return st2;
    net->d_sig0 = (const int32_t *)d;
  }
  for (size_t q = 0; q < net->steps.size(); ++q) {
    if (ph[q].m == 0) continue;                  // a plain layer step
    PassHost &H = ph[q];
    if (!pass_variant(H.T, H.C, H.NB))
      return fail(SDNN_E_UNSUPPORTED, "no fused-pass kernel for tile " + std::to_string(H.T) + " x cluster " +
                                          std::to_string(H.C));
    DevPass D{};
    D.a = H.a;
    D.m = H.m;
    D.ncomp = H.ncomp;
    D.rin = H.rin;
    D.R = H.R;
    D.T = H.T;
    D.C = H.C;
    D.NB = H.NB;
    D.NW = H.NW;
    D.S = H.S;
    D.general = H.general ? 1 : 0;
    D.rec_bytes = H.rec_bytes;
    if ((H.NB == 3 || H.NW > 0) && !net->yblk)
      return fail(SDNN_E_UNSUPPORTED, "a position-blocked pass kernel was planned for row-major activations");
    D.yblk = net->yblk;
    // tile-major pays when a pass has many components (C4: 128-512); with few
    // (C2: 8-32) component-major was measured faster (18.4 vs 18.8 ms)
    D.order = pass_order() >= 0 ? pass_order() : ((H.T == 16 || H.ncomp < 64) ? 0 : 1);
    D.lg_in = net->step_lg[q];
    D.lg_out = net->step_lg[q + 1];
    D.pf = net->yblk ? pf : 0;
    if (H.NB == 3) {                             // k_pass_wide: SDNN_WIDE_PF / SDNN_WIDE_ORDER knobs
      static const int wpf = [] {
        const char *e = getenv("SDNN_WIDE_PF");
        return e ? atoi(e) : 0;
      }();
      static const int word = [] {
        const char *e = getenv("SDNN_WIDE_ORDER");
        return e ? atoi(e) : -1;
      }();
      D.pf = wpf;
      if (word >= 0) D.order = word;
    }
    if (!streaming) {                            // else: pointers into the slot ring
      void *p1, *p2, *p3;
      sdnn_status st;
      if ((st = up(H.in_rows.data(), H.in_rows.size() * 4, &p1)) ||
          (st = up(H.in_count.data(), H.in_count.size() * 4, &p2)) ||
          (st = up(H.rec.data(), H.rec.size(), &p3)))
        return st;
      D.in_rows = (const int32_t *)p1;
      D.in_count = (const int32_t *)p2;
      D.rec = (const unsigned char *)p3;
      if (H.NB == 3) {
        void *p4;
        if ((st = up(H.split.data(), H.split.size() * 4, &p4))) return st;
        D.split = (const int32_t *)p4;
      }
    }
    for (int j = 0; j < H.m; ++j) {
      const PassHostLayer &HL = H.layers[j];
      const DevLayer &DL = net->dl[H.a + j];
      D.layers[j] = PassLayerDev{HL.off_kg, HL.off_src, HL.off_bias, HL.off_orow, HL.NG, HL.wu, HL.bu,
                                 HL.off_vs, HL.vt, HL.off_gid, HL.general ? DL.val : nullptr,
                                 DL.kmax, DL.gmax};
      if (HL.general && (!DL.val || (reinterpret_cast<uintptr_t>(DL.val) & 15)))
        return fail(SDNN_E_UNSUPPORTED, "per-slot weights of a fused layer are not 16-byte aligned");
    }
    net->steps[q].pass = (int32_t)net->passes.size();
    net->passes.push_back(D);
    net->fused_layers += H.m;
  }
  if (streaming) {
    sdnn_status st2 = build_stream_blobs(net, ph);
    if (st2) return st2;
  }
  // SMEM-resident tail: layers [ar, L) in one persistent kernel when the width fits
  net->resident_layers = 0;
  net->d_res = nullptr;
  if (ar < net->L) {
    for (size_t q = 0; q < rl.size(); ++q) {
      void *d;
      sdnn_status st2 = up(blobs[q].data(), blobs[q].size(), &d);
      if (st2) return st2;
      rl[q].blob = (const unsigned char *)d;
    }
    std::vector<ResLayerDev> full(net->L);      // indexed by absolute layer
    for (size_t q = 0; q < rl.size(); ++q) full[ar + q] = rl[q];
    void *d;
    sdnn_status st2 = up(full.data(), sizeof(ResLayerDev) * full.size(), &d);
    if (st2) return st2;
    net->d_res = (ResLayerDev *)d;
    Step r;
    r.a = ar;
    r.m = net->L - ar;
    r.pass = kResidentStep;
    net->steps.push_back(r);
    net->resident_layers = r.m;
  }
  net->plan_dirty = false;
  ++net->plan_gen;
  return SDNN_OK;
}

// The layer chain of one inference as a list of single-kernel operations in
// dependency order (each depends on the previous): per step its layer / pass
// kernel, the survivor scan and (between steps) the compaction.  Used by
// enqueue_chain and by the f1 task graphs (sdnn_flow_infer).  Not for weight
// streaming or per-layer profiling (they add events on a second stream).
using Op = std::function<void(cudaStream_t)>;
std::vector<Op> chain_ops(sdnn_net *net, bool compact) {
  std::vector<Op> ops;
  const float ymax = net->opts.ymax;
  const int ns = (int)net->steps.size();
  for (int si = 0; si < ns; ++si) {
    const Step S = net->steps[si];
    const bool last = si + 1 == ns;
    if (S.pass == kResidentStep) {            // always the last step
      ops.push_back([=](cudaStream_t s) {
        const Workspace &w = net->ws;
        launch_resident(w, net->d_res, S.a, net->L, net->n, w.alive_row(si, 0), compact, ymax, s);
      });
      continue;
    }
    const bool sat = (net->opts.flags & SDNN_F_SATURATE) && S.m == 1 &&
                     layer_tracks_saturation(net->cfg, net->dl[S.a]);
    ops.push_back([=](cudaStream_t s) {
      const Workspace &w = net->ws;
      if (S.pass < 0)
        launch_layer(net->cfg, w, net->dl[S.a], S.a, w.alive_row(si, 0), ymax, s, sat ? w.sat[si & 1] : nullptr);
      else
        launch_pass(net->cfg, w, net->passes[S.pass], w.alive_set(si), ymax, s);
    });
    const bool retire = sat && net->sat_suffix[S.a + 1];
    ops.push_back([=](cudaStream_t s) {
      const Workspace &w = net->ws;
      launch_scan(w, S.a, S.m, w.alive_set(si), w.alive_set(si + 1), compact && !last, s,
                  retire ? w.sat[si & 1] : nullptr,
                  (net->opts.flags & SDNN_F_SATURATE) ? w.sat[(si + 1) & 1] : nullptr);
    });
    if (!last)
      ops.push_back([=](cudaStream_t s) {
        const Workspace &w = net->ws;
        launch_compact_copy(net->cfg, w, S.a, S.m, w.alive_row(si, S.m - 1), net->n, s,
                            w.yblk ? net->step_lg[si + 1] : 5);
      });
  }
  return ops;
}

void enqueue_chain(sdnn_net *net, bool compact, cudaStream_t s, int64_t *launches) {
  if (!weight_streaming(net) && !(net->opts.flags & SDNN_F_PROFILE)) {
    const std::vector<Op> ops = chain_ops(net, compact);
    for (const Op &op : ops) op(s);
    int64_t c = (int64_t)ops.size();
    for (const Step &S : net->steps) c += S.pass == kResidentStep ? 1 : 0;   // the resident step launches 2 kernels
    if (launches) *launches = c;
    return;
  }
  const float ymax = net->opts.ymax;
  const bool prof = (net->opts.flags & SDNN_F_PROFILE) && (int)net->ev_before.size() == net->L;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cap);
  // inside a capture the record must be an explicit (external) event node
  const unsigned evflags = cap == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : 0u;
  const Workspace &w = net->ws;
  const int ns = (int)net->steps.size();
  int64_t c = 0;
  // f3: the copy stream forks from s; step j's block goes into slot j mod S once
  // step j - S has released it; step j waits for its own block
  const bool streaming = weight_streaming(net);
  const int nslot = net->opts.stream_slots;
  auto issue_copy = [&](int j) {
    if (j >= ns) return;
    if (j >= nslot) cudaStreamWaitEvent(net->copy_s, net->ev_done[j - nslot], 0);
    cudaMemcpyAsync(net->d_slots + (size_t)(j % nslot) * net->slot_bytes, net->h_wblob + net->wb_off[j],
                    net->wb_bytes[j], cudaMemcpyHostToDevice, net->copy_s);
    cudaEventRecord(net->ev_ready[j], net->copy_s);
  };
  if (streaming) {
    cudaEventRecord(net->ev_fork, s);
    cudaStreamWaitEvent(net->copy_s, net->ev_fork, 0);
    for (int j = 0; j < nslot; ++j) issue_copy(j);
  }
  for (int si = 0; si < ns; ++si) {
    const Step &S = net->steps[si];
    const bool last = si + 1 == ns;
    if (streaming) cudaStreamWaitEvent(s, net->ev_ready[si], 0);
    if (prof) cudaEventRecordWithFlags(net->ev_before[S.a], s, evflags);
    if (S.pass == kResidentStep) {            // always the last step
      launch_resident(w, net->d_res, S.a, net->L, net->n, w.alive_row(si, 0), compact, ymax, s);
      if (prof) cudaEventRecordWithFlags(net->ev_after[S.a], s, evflags);
      c += 2;
      continue;
    }
    const DevLayer &dl = streaming ? net->step_dl[si] : net->dl[S.a];
    const bool sat = (net->opts.flags & SDNN_F_SATURATE) && S.m == 1 &&
                     layer_tracks_saturation(net->cfg, dl);
    if (S.pass < 0)
      launch_layer(net->cfg, w, dl, S.a, w.alive_row(si, 0), ymax, s, sat ? w.sat[si & 1] : nullptr);
    else                                          // a fused pass (m >= 1)
      launch_pass(net->cfg, w, net->passes[S.pass], w.alive_set(si), ymax, s);
    if (prof) cudaEventRecordWithFlags(net->ev_after[S.a], s, evflags);
    if (streaming) {                              // slot si mod S is free again
      cudaEventRecord(net->ev_done[si], s);
      issue_copy(si + nslot);
    }
    // survivor counts for every layer of the step; compaction between steps;
    // f2: retire rows saturated before a saturation-preserving suffix
    const bool retire = sat && net->sat_suffix[S.a + 1];
    launch_scan(w, S.a, S.m, w.alive_set(si), w.alive_set(si + 1), compact && !last, s,
                retire ? w.sat[si & 1] : nullptr,
                (net->opts.flags & SDNN_F_SATURATE) ? w.sat[(si + 1) & 1] : nullptr);
    c += 2;
    if (!last) {
      launch_compact_copy(net->cfg, w, S.a, S.m, w.alive_row(si, S.m - 1), net->n, s,
                          w.yblk ? net->step_lg[si + 1] : 5);
      ++c;
    }
  }
  if (streaming) {                                // join the copy stream back
    cudaEventRecord(net->ev_join, net->copy_s);
    cudaStreamWaitEvent(s, net->ev_join, 0);      // (memcpy nodes are not kernel launches)
  }
  if (launches) *launches = c;
}

sdnn_status run_chain(sdnn_net *net, bool compact, cudaStream_t s) {
  if (net->L == 0) return SDNN_OK;
  sdnn_status st0 = make_plan(net);
  if (st0) return st0;
  if (net->opts.flags & SDNN_F_NO_GRAPH) {
    enqueue_chain(net, compact, s, &net->chain_launches);
    CK(cudaGetLastError());
    return SDNN_OK;
  }
  if (!net->chain || net->chain_compact != compact) {
    if (net->chain) cudaGraphExecDestroy(net->chain);
    net->chain = nullptr;
    cudaStream_t cs;
    CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaGraph_t graph;
    CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    enqueue_chain(net, compact, cs, &net->chain_launches);
    cudaError_t e = cudaStreamEndCapture(cs, &graph);
    cudaStreamDestroy(cs);
    CK(e);
    e = cudaGraphInstantiate(&net->chain, graph, 0);
    cudaGraphDestroy(graph);
    CK(e);
    net->chain_compact = compact;
  }
  CK(cudaGraphLaunch(net->chain, s));
  return SDNN_OK;
}

void launch_final_yout(sdnn_net *net, int64_t batch, float *d_yout, cudaStream_t s) {
  if (net->L == 0) {
    launch_yout(net->ws, 0, false, net->n, batch, d_yout, s);
  } else {
    launch_yout(net->ws, net->steps.back().a, true, net->n, batch, d_yout, s);
    if (net->opts.flags & SDNN_F_SATURATE)
      launch_yout_retired(net->ws, net->n, batch, net->opts.ymax, d_yout, s);
  }
}

// Everything of one inference after Y0 is on the device.
// workspace for `batch` rows and the execution plan (whose activation layout
// the workspace records)
// TMA tensor maps of the two activation buffers for the 16-position passes
// (position-blocked layout, 32-position blocks): dims {32, N, stride/32},
// box {16 positions, 256 rows, 1 block}.  Encoded whenever the buffers or the
// plan change.  Opt-in (SDNN_PASS_TMA16=1): measured on C4 the boxes of 64 B
// rows are slower than the 16-byte LDGSTS half-row loads (4.25 vs 3.43 ms per
// 16-position pass, 2027 vs 1939 ms/step).
sdnn_status encode_tmaps(sdnn_net *net) {
  static const bool on = [] {
    const char *e = getenv("SDNN_PASS_TMA16");
    return e && atoi(e) == 1;
  }();
  bool need = false;
  for (const DevPass &D : net->passes) need = need || (D.T == 16 && D.C == 1 && D.yblk && D.lg_in == 5);
  if (!on || !need) return SDNN_OK;
  if (net->tmap_y[0] == net->ws.Y[0] && net->tmap_y[1] == net->ws.Y[1] && net->tmap_plan == net->plan_gen)
    return SDNN_OK;
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    cudaGetLastError();
    return (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }();
  CUtensorMap maps[2];
  bool ok = encode != nullptr;
  for (int i = 0; i < 2 && ok; ++i) {
    const cuuint64_t dims[3] = {32, (cuuint64_t)net->n, (cuuint64_t)(net->ws.stride / 32)};
    const cuuint64_t strides[2] = {128, (cuuint64_t)net->n * 128};
    const cuuint32_t box[3] = {16, 256, 1}, es[3] = {1, 1, 1};
    ok = encode(&maps[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, net->ws.Y[i], dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  for (DevPass &D : net->passes)
    if (D.T == 16 && D.C == 1 && D.yblk && D.lg_in == 5) {
      D.tma16 = ok ? 1 : 0;
      if (ok) {
        D.tmap[0] = maps[0];
        D.tmap[1] = maps[1];
      }
    }
  net->tmap_y[0] = net->ws.Y[0];
  net->tmap_y[1] = net->ws.Y[1];
  net->tmap_plan = net->plan_gen;
  if (net->chain) {                              // pass parameters changed: recapture
    cudaGraphExecDestroy(net->chain);
    net->chain = nullptr;
  }
  return SDNN_OK;
}

sdnn_status prepare_infer(sdnn_net *net, int64_t batch) {
  if (net->nset.load() != net->L) return fail(SDNN_E_STATE, "not every layer has been set");
  sdnn_status st = ensure_ws(net, batch);
  if (st) return st;
  if (net->L > 0 && (st = make_plan(net))) return st;   // the layout of Y is a plan property
  net->ws.yblk = net->L > 0 ? net->yblk : 0;
  net->ws.sig0 = net->L > 0 ? net->d_sig0 : nullptr;
  net->ws.lg0 = (net->L > 0 && net->yblk && !net->step_lg.empty()) ? net->step_lg[0] : 5;
  if (net->L > 0 && (st = encode_tmaps(net))) return st;
  if (net->uploads_pending.exchange(false)) CK(cudaDeviceSynchronize());
  return SDNN_OK;
}

// feed (sdnn_infer): enqueues the chunked input copies and their scatters
// after the densify prep; NULL = Y0 is already on the device
using Feed = std::function<sdnn_status(cudaStream_t)>;
sdnn_status infer_device_impl(sdnn_net *net, const int64_t *d_rowptr, const int32_t *d_idx,
                              const float *d_val, int64_t batch, uint32_t *d_alive,
                              float *d_yout, cudaStream_t s, const Feed *feed = nullptr,
                              const sdnn_nvls *nv = nullptr) {
  sdnn_status st = prepare_infer(net, batch);
  if (st) return st;
  const bool compact = compact_enabled(net);
  int64_t launches = 4;
  if (feed) {
    launch_densify_prep(net->cfg, net->ws, net->n, batch, d_rowptr, d_val, compact, s);
    st = (*feed)(s);
    if (st) return st;
  } else {
    launch_densify(net->cfg, net->ws, net->n, batch, d_rowptr, d_idx, d_val, compact, s);
  }
  if (net->L == 0) {
    launch_zero_layers_alive(net->ws, batch, d_rowptr, d_val, s);
    launches += 1;
  } else {
    st = run_chain(net, compact, s);
    if (st) return st;
    launches += net->chain_launches;
  }
  if (nv) {                                      // f4: fused NVLS gather (L >= 1, checked by the caller)
    const int si = (int)net->steps.size() - 1;
    const Step &S = net->steps[si];
    const int row = S.pass == kResidentStep ? 0 : S.m - 1;
    launch_readout_nvls(net->ws, S.a, net->ws.alive_row(si, row), batch, nv->local_words + nv->word_offset,
                        nv->mc_words + nv->word_offset, nv->local_flag, nv->mc_flag, nv->target, s);
  } else if (net->L == 0) {
    launch_readout(net->ws, 0, net->ws.alive_row(0, 0), d_alive, batch, s);
  } else {
    const int si = (int)net->steps.size() - 1;
    const Step &S = net->steps[si];
    const int row = S.pass == kResidentStep ? 0 : S.m - 1;
    if (net->opts.flags & SDNN_F_SATURATE)
      launch_readout_retired(net->ws, S.a, net->ws.alive_row(si, row), d_alive, batch, s);
    else
      launch_readout(net->ws, S.a, net->ws.alive_row(si, row), d_alive, batch, s);
  }
  launches += 1 + (d_alive ? 1 : 0);
  if (d_yout) {
    launch_final_yout(net, batch, d_yout, s);
    launches += 2;
  }
  CK(cudaGetLastError());
  net->last_batch = batch;
  net->launches = launches;
  net->profiled = (net->opts.flags & SDNN_F_PROFILE) && net->L > 0;
  return SDNN_OK;
}


template <class F>
void parallel_for(int64_t n, int nt, F f) {
  if (nt <= 1 || n < 4096) {
    f(0, n);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t) {
    const int64_t a = n * t / nt, b = n * (t + 1) / nt;
    th.emplace_back([=] { f(a, b); });
  }
  for (auto &x : th) x.join();
}

// Host validation of Y0 (sdnn_infer only): monotone rowptr, index range,
// no duplicate per row, finite values.
sdnn_status validate_y0(int32_t n, const int64_t *rowptr, const int32_t *idx, const float *val,
                        int64_t batch) {
  if (rowptr[0] != 0) return fail(SDNN_E_FORMAT, "y0_rowptr[0] != 0");
  for (int64_t i = 0; i < batch; ++i)
    if (rowptr[i + 1] < rowptr[i]) return fail(SDNN_E_FORMAT, "y0_rowptr not non-decreasing");
  std::atomic<int64_t> bad{-1};
  std::atomic<int> kind{0};
  const int nt = nthreads_default();
  parallel_for(batch, nt, [&](int64_t a, int64_t b) {
    std::vector<int64_t> mark(n, -1);
    for (int64_t i = a; i < b && bad.load() < 0; ++i)
      for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
        const int32_t k = idx[e];
        if (k < 0 || k >= n) { bad = i; kind = 1; break; }
        if (mark[k] == i) { bad = i; kind = 2; break; }
        mark[k] = i;
        if (val && !std::isfinite(val[e])) { bad = i; kind = 3; break; }
      }
  });
  if (bad.load() >= 0) {
    const char *what[] = {"", "index out of range", "duplicate index", "non-finite value"};
    return fail(SDNN_E_FORMAT, std::string("Y0 row ") + std::to_string(bad.load()) + ": " + what[kind.load()]);
  }
  return SDNN_OK;
}

void *grow_pinned(sdnn_net *net, size_t bytes) {
  if (bytes <= net->h_stage_cap) return net->h_stage;
  if (net->h_stage) cudaFreeHost(net->h_stage);
  net->h_stage = nullptr;
  net->h_stage_cap = 0;
  const size_t cap = std::max(bytes, net->h_stage_cap * 3 / 2);
  if (cudaHostAlloc(&net->h_stage, cap, cudaHostAllocDefault) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  net->h_stage_cap = cap;
  return net->h_stage;
}


// ---------------------------------------------------------------------------
// f1: the inference of P batch partitions as ONE GPU task graph
// -- per partition: densify -> every kernel of its handle's layer chain ->
// readout into its word slice of a global category bitmask; then the device
// decode of that bitmask -- launched three ways (Sec. 4.6.2):
//   graph     explicit nodes and edges (the paper's cudaFlow): tasks are
//             captured one by one into a graph whose dependency set is set to
//             exactly the task's predecessors (cudaStreamUpdateCaptureDependencies)
//   capturer  Algorithm 1: levelize, stream = (id in level) mod max_streams,
//             events only on cross-stream edges, one stream capture -> graph
//   streams   the same stream assignment and events, launched directly
// ---------------------------------------------------------------------------
struct FlowTask {
  Op op;
  std::vector<int> pred, succ;
  int level = 0, id = 0;
};

// Alg. 1's levelize(C): topological levels (Kahn's algorithm, one level per
// round); id = the task's index in its level
std::vector<std::vector<int>> levelize(std::vector<FlowTask> &T) {
  std::vector<int> indeg(T.size());
  std::vector<int> cur;
  for (size_t t = 0; t < T.size(); ++t)
    if ((indeg[t] = (int)T[t].pred.size()) == 0) cur.push_back((int)t);
  std::vector<std::vector<int>> L;
  while (!cur.empty()) {
    std::vector<int> next;
    for (size_t i = 0; i < cur.size(); ++i) {
      T[cur[i]].level = (int)L.size();
      T[cur[i]].id = (int)i;
      for (int n : T[cur[i]].succ)
        if (--indeg[n] == 0) next.push_back(n);
    }
    L.push_back(cur);
    cur.swap(next);
  }
  return L;
}

struct FlowStreams {
  std::vector<cudaStream_t> S;
  std::vector<cudaEvent_t> ev;                   // per task (recorded on cross-stream edges)
  cudaEvent_t fork = nullptr;
  std::vector<cudaEvent_t> join;
  ~FlowStreams() {
    for (auto s : S) cudaStreamDestroy(s);
    for (auto e : ev) cudaEventDestroy(e);
    for (auto e : join) cudaEventDestroy(e);
    if (fork) cudaEventDestroy(fork);
  }
};

// Algorithm 1 (make_graph), its loop body shared by the capturer and the plain
// stream launch: stream_wait_event on every predecessor issued in another
// stream, the task, stream_record_event for successors in another stream (the
// listing records `p.event` in the successor loop; the task's own event is
// meant)
void alg1_issue(std::vector<FlowTask> &T, const std::vector<std::vector<int>> &L, FlowStreams &F, int k) {
  cudaEventRecord(F.fork, F.S[0]);
  for (int s = 1; s < k; ++s) cudaStreamWaitEvent(F.S[s], F.fork, 0);
  for (const auto &lev : L)
    for (int t : lev) {
      const int s = T[t].id % k;
      for (int p : T[t].pred)
        if (T[p].id % k != s) cudaStreamWaitEvent(F.S[s], F.ev[p], 0);
      T[t].op(F.S[s]);
      bool rec = false;
      for (int n : T[t].succ) rec = rec || (T[n].id % k != s);
      if (rec) cudaEventRecord(F.ev[t], F.S[s]);
    }
  for (int s = 1; s < k; ++s) {                  // end_capture_mode_streams: join into S[0]
    cudaEventRecord(F.join[s], F.S[s]);
    cudaStreamWaitEvent(F.S[0], F.join[s], 0);
  }
}

}  // namespace

extern "C" sdnn_status sdnn_flow_plan(int32_t ntasks, int32_t nedges, const int32_t *edges, int32_t max_streams,
                                      int32_t *level, int32_t *id, int32_t *stream, int32_t *nevents,
                                      int32_t *event_edges) {
  if (ntasks < 0 || nedges < 0 || max_streams < 1 || (nedges > 0 && !edges) || !nevents)
    return fail(SDNN_E_ARG, "bad argument");
  std::vector<FlowTask> T(ntasks);
  for (int e = 0; e < nedges; ++e) {
    const int u = edges[2 * e], v = edges[2 * e + 1];
    if (u < 0 || u >= ntasks || v < 0 || v >= ntasks || u == v) return fail(SDNN_E_ARG, "bad edge");
    T[u].succ.push_back(v);
    T[v].pred.push_back(u);
  }
  const std::vector<std::vector<int>> L = levelize(T);
  size_t placed = 0;
  for (const auto &lev : L) placed += lev.size();
  if ((int)placed != ntasks) return fail(SDNN_E_FORMAT, "the task graph has a cycle");
  int32_t ne = 0;
  for (int t = 0; t < ntasks; ++t) {
    if (level) level[t] = T[t].level;
    if (id) id[t] = T[t].id;
    if (stream) stream[t] = T[t].id % max_streams;
  }
  // Alg. 1's events: one per edge whose ends sit in different streams, in the
  // order the algorithm issues them (level by level, successors per task)
  for (const auto &lev : L)
    for (int t : lev)
      for (int n : T[t].succ)
        if (T[n].id % max_streams != T[t].id % max_streams) {
          if (event_edges) {
            event_edges[2 * ne] = t;
            event_edges[2 * ne + 1] = n;
          }
          ++ne;
        }
  *nevents = ne;
  return SDNN_OK;
}

extern "C" sdnn_status sdnn_flow_infer(sdnn_net *const *nets, int32_t parts, const sdnn_flow_part *pp,
                                       uint32_t *d_words, int64_t total_batch, int32_t *d_ids,
                                       int32_t *d_n, int32_t mode, int32_t max_streams, int32_t reps,
                                       float *ms, int32_t *ntasks) {
  if (!nets || !pp || parts < 1 || !d_words || !d_ids || !d_n || max_streams < 1 || reps < 1)
    return fail(SDNN_E_ARG, "bad argument");
  if (mode < SDNN_FLOW_GRAPH || mode > SDNN_FLOW_STREAMS) return fail(SDNN_E_ARG, "bad mode");
  for (int p = 0; p < parts; ++p) {
    sdnn_net *net = nets[p];
    if (!net) return fail(SDNN_E_ARG, "NULL handle");
    for (int q = 0; q < p; ++q)
      if (nets[q] == net) return fail(SDNN_E_ARG, "a handle may serve one partition only (own workspace)");
    if (net->L < 1) return fail(SDNN_E_UNSUPPORTED, "task graphs need >= 1 layer");
    if (weight_streaming(net) || (net->opts.flags & SDNN_F_PROFILE))
      return fail(SDNN_E_UNSUPPORTED, "weight streaming / profiling handles are not supported here");
    if (pp[p].batch < 0 || pp[p].word_offset < 0 || (pp[p].batch > 0 && !pp[p].d_rowptr))
      return fail(SDNN_E_ARG, "bad partition");
    sdnn_status st = set_device(net);
    if (st) return st;
    if ((st = prepare_infer(net, pp[p].batch))) return st;
  }
  sdnn_net *net0 = nets[0];
  // ---- the task graph ----
  std::vector<FlowTask> T;
  std::vector<int> tails;
  for (int p = 0; p < parts; ++p) {
    sdnn_net *net = nets[p];
    const sdnn_flow_part P = pp[p];
    const bool compact = compact_enabled(net);
    auto add = [&](Op op) {
      FlowTask t;
      t.op = std::move(op);
      if (!T.empty() && (int)T.size() > 0 && !tails.empty() && tails.back() >= 0) {
        t.pred.push_back(tails.back());
        T[tails.back()].succ.push_back((int)T.size());
      }
      T.push_back(std::move(t));
      tails.back() = (int)T.size() - 1;
    };
    tails.push_back(-1);
    add([=](cudaStream_t s) {
      launch_densify(net->cfg, net->ws, net->n, P.batch, P.d_rowptr, P.d_idx, P.d_val, compact, s);
    });
    for (Op &op : chain_ops(net, compact)) add(std::move(op));
    const int si = (int)net->steps.size() - 1;
    const Step S = net->steps[si];
    const int row = S.pass == kResidentStep ? 0 : S.m - 1;
    add([=](cudaStream_t s) {
      launch_readout(net->ws, S.a, net->ws.alive_row(si, row), d_words + P.word_offset, P.batch, s);
    });
  }
  {
    FlowTask j;
    j.op = [=](cudaStream_t s) { launch_bitmask_ids(d_words, total_batch, d_ids, d_n, s); };
    for (int t : tails) {
      j.pred.push_back(t);
      T[t].succ.push_back((int)T.size());
    }
    T.push_back(std::move(j));
  }
  if (ntasks) *ntasks = (int32_t)T.size();
  const std::vector<std::vector<int>> L = levelize(T);
  const int k = mode == SDNN_FLOW_GRAPH ? 1 : max_streams;
  FlowStreams F;
  F.S.resize(k);
  for (auto &s : F.S) CKN(net0, cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  F.ev.resize(T.size());
  for (auto &e : F.ev) CKN(net0, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  F.join.assign(k, nullptr);
  for (auto &e : F.join) CKN(net0, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  CKN(net0, cudaEventCreateWithFlags(&F.fork, cudaEventDisableTiming));
  cudaGraphExec_t exec = nullptr;
  if (mode == SDNN_FLOW_CAPTURER) {
    cudaGraph_t g;
    CKN(net0, cudaStreamBeginCapture(F.S[0], cudaStreamCaptureModeThreadLocal));
    alg1_issue(T, L, F, k);
    CKN(net0, cudaStreamEndCapture(F.S[0], &g));
    const cudaError_t e = cudaGraphInstantiate(&exec, g, 0);
    cudaGraphDestroy(g);
    CKN(net0, e);
  } else if (mode == SDNN_FLOW_GRAPH) {
    // explicit DAG: each task is captured with its dependency set replaced by
    // the graph nodes that end its predecessors
    cudaGraph_t g;
    CKN(net0, cudaGraphCreate(&g, 0));
    cudaStream_t s = F.S[0];
    CKN(net0, cudaStreamBeginCaptureToGraph(s, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    std::vector<std::vector<cudaGraphNode_t>> ends(T.size());
    for (const auto &lev : L)
      for (int t : lev) {
        std::vector<cudaGraphNode_t> deps;
        for (int p : T[t].pred) deps.insert(deps.end(), ends[p].begin(), ends[p].end());
        CKN(net0, cudaStreamUpdateCaptureDependencies(s, deps.empty() ? nullptr : deps.data(), deps.size(),
                                                      cudaStreamSetCaptureDependencies));
        T[t].op(s);
        cudaStreamCaptureStatus cs;
        const cudaGraphNode_t *dn = nullptr;
        size_t nd = 0;
        CKN(net0, cudaStreamGetCaptureInfo(s, &cs, nullptr, nullptr, &dn, &nd));
        ends[t].assign(dn, dn + nd);
      }
    cudaGraph_t g2;
    CKN(net0, cudaStreamEndCapture(s, &g2));
    const cudaError_t e = cudaGraphInstantiate(&exec, g2, 0);
    cudaGraphDestroy(g2);
    CKN(net0, e);
  }
  cudaEvent_t t0, t1;
  CKN(net0, cudaEventCreate(&t0));
  CKN(net0, cudaEventCreate(&t1));
  auto run = [&]() {
    if (exec) cudaGraphLaunch(exec, F.S[0]);
    else alg1_issue(T, L, F, k);
  };
  run();                                         // warm-up (and the result if reps == 1)
  cudaEventRecord(t0, F.S[0]);
  for (int r = 0; r < reps; ++r) run();
  cudaEventRecord(t1, F.S[0]);
  cudaError_t e = cudaEventSynchronize(t1);
  float tm = 0.f;
  if (e == cudaSuccess) e = cudaEventElapsedTime(&tm, t0, t1);
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  if (exec) cudaGraphExecDestroy(exec);
  CKN(net0, e);
  CKN(net0, cudaGetLastError());
  if (ms) *ms = tm / reps;
  return SDNN_OK;
}

namespace {
// The host-buffer inference, split so that it can be pipelined
// (sdnn_infer_submit / sdnn_infer_wait): host_enqueue validates rowptr, starts
// the full host validation on its own thread, enqueues the chunked input copy
// (input stream), the densify + layer chain + readout (compute stream) and the
// copy of the categories into the slot's pinned result buffer; host_finish
// joins the validation and waits for the result.  Two input slots: the copy of
// submission k+1 (slot (k+1) & 1) overlaps the layers of submission k, and
// waits (on the device) until the scatter of submission k-1 has consumed that
// slot's buffers.
sdnn_status host_enqueue(sdnn_net *net, int slot_i, const int64_t *y0_rowptr, const int32_t *y0_idx,
                         const float *y0_val, int64_t batch) {
  HostSlot &H = net->slots[slot_i];
  sdnn_status st = SDNN_OK;
  const int64_t nnz = y0_rowptr[batch];
  if (nnz > 0 && !y0_idx) return fail(SDNN_E_ARG, "y0_idx is NULL");
  // rowptr must be sane before its last entry sizes the copies below; the full
  // validation runs on the host while the (page-locked) input is in flight
  if (!(net->opts.flags & SDNN_F_TRUST_INPUT)) {
    if (y0_rowptr[0] != 0) return fail(SDNN_E_FORMAT, "y0_rowptr[0] != 0");
    for (int64_t i = 0; i < batch; ++i)
      if (y0_rowptr[i + 1] < y0_rowptr[i]) return fail(SDNN_E_FORMAT, "y0_rowptr not non-decreasing");
  }
  cudaStream_t s = net->opts.stream ? (cudaStream_t)net->opts.stream : net->own;
  if (!net->in_s) CK(cudaStreamCreateWithFlags(&net->in_s, cudaStreamNonBlocking));
  if (!H.done) CK(cudaEventCreateWithFlags(&H.done, cudaEventDisableTiming));
  if (!H.in_free) CK(cudaEventCreateWithFlags(&H.in_free, cudaEventDisableTiming));
  // device input buffers of the slot (grow-only; a growing slot first waits
  // for its previous use)
  if (batch + 1 > H.cap_rows || nnz > H.cap_nnz || (y0_val && nnz > H.cap_val)) CK(cudaEventSynchronize(H.in_free));
  if (batch + 1 > H.cap_rows) {
    cudaFree(H.d_rowptr);
    H.d_rowptr = nullptr;
    CK(cudaMalloc(&H.d_rowptr, sizeof(int64_t) * (batch + 1)));
    H.cap_rows = batch + 1;
  }
  if (nnz > H.cap_nnz) {
    cudaFree(H.d_idx);
    H.d_idx = nullptr;
    CK(cudaMalloc(&H.d_idx, sizeof(int32_t) * std::max<int64_t>(nnz, 1)));
    H.cap_nnz = nnz;
  }
  if (y0_val && nnz > H.cap_val) {
    cudaFree(H.d_val);
    H.d_val = nullptr;
    CK(cudaMalloc(&H.d_val, sizeof(float) * std::max<int64_t>(nnz, 1)));
    H.cap_val = nnz;
  }
  if (batch + 1 > H.h_res_cap) {
    CK(cudaEventSynchronize(H.done));
    if (H.h_res) cudaFreeHost(H.h_res);
    H.h_res = nullptr;
    H.h_res_cap = 0;
    CK(cudaHostAlloc((void **)&H.h_res, sizeof(int32_t) * (size_t)(batch + 1), cudaHostAllocDefault));
    H.h_res_cap = batch + 1;
  }
  H.batch = batch;
  // Input path (A14: the copies are inside the timed call).  rowptr first (the
  // device prep -- zero Y0, row flags, scan -- needs only it), then the column
  // indices in row chunks of ~64 MB on the input stream, each chunk scattered
  // on the compute stream as soon as it has landed, so the copy of chunk c+1
  // overlaps the scatter of chunk c; page-locked caller buffers are DMA'd
  // directly, pageable ones through a pinned double buffer.  Explicit values
  // (y0_val) are needed by the row flags, so they are copied up front.  The
  // full host validation (index range, duplicates, finite values) runs on a
  // separate host thread meanwhile and is joined in host_finish; the device
  // path is memory-safe on invalid input (out-of-range indices are skipped).
  static const size_t kChunk = [] {               // SDNN_IN_CHUNK_MB: A/B knob (default 64)
    const char *e = getenv("SDNN_IN_CHUNK_MB");
    const long v = e ? atol(e) : 64;
    return size_t(std::max(1L, std::min(v, 4096L))) << 20;
  }();
  char *stage = (char *)grow_pinned(net, 2 * kChunk);
  if (!stage) return fail(SDNN_E_NOMEM, "pinned staging allocation failed");
  auto is_pinned = [](const void *p) {
    cudaPointerAttributes pa;
    const bool r = cudaPointerGetAttributes(&pa, p) == cudaSuccess && pa.type == cudaMemoryTypeHost;
    cudaGetLastError();
    return r;
  };
  H.vst = SDNN_OK;
  H.vmsg.clear();
  if (!(net->opts.flags & SDNN_F_TRUST_INPUT) && batch > 0)
    H.validator = std::thread([net, &H, y0_rowptr, y0_idx, y0_val, batch] {
      H.vst = validate_y0(net->n, y0_rowptr, y0_idx, y0_val, batch);
      if (H.vst) H.vmsg = sdnn_last_error();
    });
  auto abort_enqueue = [&](sdnn_status e) -> sdnn_status {
    if (H.validator.joinable()) H.validator.join();
    cudaStreamSynchronize(s);                    // no DMA may still read the caller's buffers
    cudaStreamSynchronize(net->in_s);
    return e;
  };
  int sslot = 0;
  auto copy_h2d = [&](void *d, const void *h, size_t bytes, cudaStream_t cs, bool pinned) -> sdnn_status {
    if (bytes == 0) return SDNN_OK;
    if (pinned) {
      CK(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, cs));
      return SDNN_OK;
    }
    for (size_t off = 0; off < bytes; off += kChunk) {
      const size_t b = std::min(kChunk, bytes - off);
      // (also across calls: a pipelined submission may still be copying from
      // this staging slot; an event never recorded counts as complete)
      CK(cudaEventSynchronize(net->ev_stage[sslot]));
      char *dst = stage + sslot * kChunk;
      const char *src = (const char *)h + off;
      parallel_for((int64_t)b, std::min(nthreads_default(), 8),
                   [&](int64_t x, int64_t y) { std::memcpy(dst + x, src + x, (size_t)(y - x)); });
      CK(cudaMemcpyAsync((char *)d + off, dst, b, cudaMemcpyHostToDevice, cs));
      CK(cudaEventRecord(net->ev_stage[sslot], cs));
      sslot ^= 1;
    }
    return SDNN_OK;
  };
  for (int i = 0; i < 2; ++i)
    if (!net->ev_stage[i]) CK(cudaEventCreateWithFlags(&net->ev_stage[i], cudaEventDisableTiming));
  // this slot's buffers are free once the previous scatter from them is done
  CK(cudaStreamWaitEvent(net->in_s, H.in_free, 0));
  if ((st = copy_h2d(H.d_rowptr, y0_rowptr, sizeof(int64_t) * (size_t)(batch + 1), net->in_s,
                     is_pinned(y0_rowptr))) ||
      (y0_val && (st = copy_h2d(H.d_val, y0_val, sizeof(float) * (size_t)nnz, net->in_s, is_pinned(y0_val)))))
    return abort_enqueue(st);
  if (!net->ev_in) CK(cudaEventCreateWithFlags(&net->ev_in, cudaEventDisableTiming));
  CK(cudaEventRecord(net->ev_in, net->in_s));
  CK(cudaStreamWaitEvent(s, net->ev_in, 0));       // rowptr (and values) on the device
  const bool idx_pinned = nnz > 0 && is_pinned(y0_idx);
  // row chunks of ~kChunk bytes of indices
  std::vector<int64_t> cut{0};
  {
    const int64_t per = (int64_t)(kChunk / sizeof(int32_t));
    int64_t r = 0;
    while (r < batch) {
      const int64_t lim = y0_rowptr[r] + per;
      int64_t hi = std::upper_bound(y0_rowptr + r + 1, y0_rowptr + batch + 1, lim) - y0_rowptr - 1;
      if (hi <= r) hi = r + 1;                   // one row larger than a chunk
      r = std::min(hi, batch);
      cut.push_back(r);
    }
  }
  while (net->ev_chunk.size() + 1 < cut.size()) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    net->ev_chunk.push_back(e);
  }
  const Feed feed = [&](cudaStream_t cs) -> sdnn_status {
    for (size_t c = 0; c + 1 < cut.size(); ++c) {
      const int64_t r0 = cut[c], r1 = cut[c + 1];
      const int64_t e0 = y0_rowptr[r0], e1 = y0_rowptr[r1];
      sdnn_status s2 = copy_h2d(H.d_idx + e0, y0_idx + e0, sizeof(int32_t) * (size_t)(e1 - e0), net->in_s,
                                idx_pinned);
      if (s2) return s2;
      CK(cudaEventRecord(net->ev_chunk[c], net->in_s));
      CK(cudaStreamWaitEvent(cs, net->ev_chunk[c], 0));
      launch_scatter_rows(net->cfg, net->ws, net->n, r0, r1, H.d_rowptr, H.d_idx,
                          y0_val ? H.d_val : nullptr, cs);
    }
    CK(cudaEventRecord(H.in_free, cs));           // the slot's input buffers are consumed
    return SDNN_OK;
  };
  st = infer_device_impl(net, H.d_rowptr, H.d_idx, y0_val ? H.d_val : nullptr, batch, nullptr, nullptr, s,
                         &feed);
  if (st) return abort_enqueue(st);
  // result: [0] = count, [1..] = the ascending ids (the capacity of the batch)
  CK(cudaMemcpyAsync(H.h_res, net->ws.ncat, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  if (batch > 0)
    CK(cudaMemcpyAsync(H.h_res + 1, net->ws.cats, sizeof(int32_t) * (size_t)batch, cudaMemcpyDeviceToHost, s));
  CK(cudaEventRecord(H.done, s));
  return SDNN_OK;
}

sdnn_status host_finish(sdnn_net *net, int slot_i, int32_t *categories, int64_t *n_categories) {
  HostSlot &H = net->slots[slot_i];
  if (H.validator.joinable()) H.validator.join();
  CK(cudaEventSynchronize(H.done));
  if (H.vst) return fail(H.vst, H.vmsg);
  const int32_t ncat = H.h_res[0];
  if (ncat > 0) std::memcpy(categories, H.h_res + 1, sizeof(int32_t) * (size_t)ncat);
  *n_categories = ncat;
  net->last_ncat = ncat;
  return SDNN_OK;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

int32_t sdnn_abi_version(void) { return SDNN_ABI_VERSION; }

const char *sdnn_last_error(void) { return g_err.c_str(); }

sdnn_status sdnn_create_empty(int32_t neurons, int32_t layers, const sdnn_opts *opts,
                              sdnn_net **out) {
  if (!out) return fail(SDNN_E_ARG, "out is NULL");
  *out = nullptr;
  if (neurons < 1) return fail(SDNN_E_ARG, "neurons < 1");
  if (neurons > 65536) return fail(SDNN_E_UNSUPPORTED, "neurons > 65536 (u16 source indices)");
  if (layers < 0) return fail(SDNN_E_ARG, "layers < 0");
  sdnn_opts o;
  sdnn_status st = check_opts(opts, o);
  if (st) return st;
  int dev = o.device;
  if (dev < 0) {
    if (cudaGetDevice(&dev) != cudaSuccess) {
      cudaGetLastError();
      return fail(SDNN_E_CUDA, "no CUDA device");
    }
  }
  if (cudaSetDevice(dev) != cudaSuccess) {
    cudaGetLastError();
    return fail(SDNN_E_CUDA, "cannot select CUDA device " + std::to_string(dev));
  }
  sdnn_net *net = new (std::nothrow) sdnn_net();
  if (!net) return fail(SDNN_E_NOMEM, "host allocation failed");
  net->n = neurons;
  net->L = layers;
  net->opts = o;
  net->device = dev;
  net->dl.resize(layers);
  net->host.resize(layers);
  net->set.assign(layers, 0);
  net->lblock.assign(layers, nullptr);
  net->lbytes.assign(layers, 0);
  net->bias_nonpos.assign(layers, 1);
  net->nnz.assign(layers, 0);
  net->fma_l.assign(layers, 0);
  net->last_live.assign(std::max(layers, 1), 0);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  net->cfg.sms = sms;
  net->cfg.layer_blocks = sms * 2;   // 2 resident 256-thread CTAs per SM (128 regs)
  net->cfg.copy_blocks = sms * 4;
  net->cfg.bulk = !(o.flags & SDNN_F_NO_BULK);
  configure_kernels();
  configure_resident();
  if (cudaStreamCreateWithFlags(&net->own, cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    delete net;
    return fail(SDNN_E_CUDA, "cudaStreamCreate failed");
  }
  if (o.flags & SDNN_F_PROFILE) {
    net->ev_before.resize(layers);
    net->ev_after.resize(layers);
    for (int l = 0; l < layers; ++l)
      if (cudaEventCreate(&net->ev_before[l]) != cudaSuccess ||
          cudaEventCreate(&net->ev_after[l]) != cudaSuccess) {
        cudaGetLastError();
        sdnn_destroy(net);
        return fail(SDNN_E_CUDA, "cudaEventCreate failed");
      }
  }
  *out = net;
  return SDNN_OK;
}

sdnn_status sdnn_set_layer(sdnn_net *net, int32_t l, const sdnn_layer *W, const float *bias_l) {
  if (!net || !W || !bias_l) return fail(SDNN_E_ARG, "NULL argument");
  if (l < 0 || l >= net->L) return fail(SDNN_E_ARG, "layer index out of range");
  sdnn_status st = set_device(net);
  if (st) return st;
  LayerIn in{W->format, W->ell_k, W->rowptr, W->idx, W->val, W->uniform_value};
  PackedLayer p;
  std::string msg;
  const int rc = pack_layer(net->n, in, bias_l, !(net->opts.flags & SDNN_F_NO_GROUPS), p, msg);
  if (rc) return fail(rc, "layer " + std::to_string(l) + ": " + msg);
  // upload: one arena block per layer, reused when the layer is set again and
  // the new packing fits (a larger one takes a fresh block; the old one is
  // returned only at destroy)
  const size_t G = p.ngroups;
  const size_t b_src = sizeof(uint16_t) * p.src.size(), b_col = sizeof(int32_t) * p.col.size();
  const size_t b_gk = sizeof(int32_t) * G, b_val = sizeof(float) * p.val.size();
  const size_t b_bias = sizeof(float) * net->n, b_gbias = sizeof(float) * p.gbias.size();
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t total = al(b_src) + al(b_col) + 2 * al(b_gk) + al(b_val) + al(b_bias) + al(b_gbias);
  DevLayer d{};
  void *ps = nullptr, *pc = nullptr, *pk = nullptr, *pg = nullptr, *pv = nullptr, *pb = nullptr, *pgb = nullptr;
  if (!weight_streaming(net)) {                   // f3: the blocks stay on the host
    char *blk = nullptr;
    {
      std::lock_guard<std::mutex> g(net->stat_mu);
      if (net->set[l] && net->lbytes[l] >= total) {
        blk = (char *)net->lblock[l];
        CK(cudaDeviceSynchronize());              // no inference may still read the old layer
      }
    }
    if (!blk) {
      void *v = nullptr;
      if (net->arena.alloc(total, &v) != cudaSuccess) {
        cudaGetLastError();
        return fail(SDNN_E_NOMEM, "device allocation for layer " + std::to_string(l) + " failed");
      }
      blk = (char *)v;
    }
    size_t off = 0;
    auto up = [&](const void *h, size_t bytes, void **dp) -> sdnn_status {
      *dp = bytes ? blk + off : nullptr;
      if (bytes) CK(cudaMemcpy(*dp, h, bytes, cudaMemcpyHostToDevice));
      net->uploads_pending = true;
      off += al(bytes);
      return SDNN_OK;
    };
    if ((st = up(p.src.data(), b_src, &ps)) || (st = up(p.col.data(), b_col, &pc)) ||
        (st = up(p.gk.data(), b_gk, &pk)) || (st = up(p.gg.data(), b_gk, &pg)) ||
        (st = up(p.val.data(), b_val, &pv)) || (st = up(p.bias.data(), b_bias, &pb)) ||
        (st = up(p.gbias.data(), b_gbias, &pgb)))
      return st;
    std::lock_guard<std::mutex> g(net->stat_mu);
    if (!(net->set[l] && net->lblock[l] == blk)) {
      net->lblock[l] = blk;
      net->lbytes[l] = total;
    }
  }
  d.src = (const uint16_t *)ps;
  d.col = (const int32_t *)pc;
  d.gk = (const int32_t *)pk;
  d.gg = (const int32_t *)pg;
  d.val = p.uniform ? nullptr : (const float *)pv;
  d.bias = (const float *)pb;
  d.gbias = (const float *)pgb;
  d.ngroups = p.ngroups;
  d.kmax = p.kmax;
  d.gmax = p.gmax;
  d.wu = p.wu;
  d.uniform = p.uniform ? 1 : 0;
  d.regular = p.regular ? 1 : 0;
  d.nnz = p.nnz;
  {
    std::lock_guard<std::mutex> g(net->stat_mu);
    const bool was = net->set[l];
    net->dl[l] = d;
    net->host[l] = std::move(p);
    net->plan_dirty = true;
    net->bias_nonpos[l] = net->host[l].bias_nonpos ? 1 : 0;
    net->nnz[l] = net->host[l].nnz;
    {
      const PackedLayer &P = net->host[l];
      int64_t f = 0;
      if (P.uniform)
        for (int32_t g = 0; g < P.ngroups; ++g) f += P.gk[g];
      net->fma_l[l] = P.uniform ? f : P.nnz;
    }
    if (net->host[l].gmax > 1) net->grouped_layers += was ? 0 : 1;
    net->max_group = std::max(net->max_group, net->host[l].gmax);
    net->max_k = std::max(net->max_k, net->host[l].kmax);
    if (!was) {
      net->set[l] = 1;
      net->nset.fetch_add(1);
    }
    if (net->chain) {                     // layer pointers changed: recapture
      cudaGraphExecDestroy(net->chain);
      net->chain = nullptr;
    }
  }
  return SDNN_OK;
}

sdnn_status sdnn_create(int32_t neurons, int32_t layers, const sdnn_layer *W, const float *bias,
                        const sdnn_opts *opts, sdnn_net **out) {
  if (!out) return fail(SDNN_E_ARG, "out is NULL");
  *out = nullptr;
  if (layers > 0 && (!W || !bias)) return fail(SDNN_E_ARG, "W or bias is NULL");
  sdnn_net *net = nullptr;
  sdnn_status st = sdnn_create_empty(neurons, layers, opts, &net);
  if (st) return st;
  // pack layers in parallel (create-time, not in the timed region)
  const int nt = std::min(nthreads_default(), std::max(1, layers));
  std::vector<sdnn_status> rcs(nt, SDNN_OK);
  std::vector<std::string> errs(nt);
  std::vector<std::thread> th;
  std::atomic<int> next{0};
  for (int t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      cudaSetDevice(net->device);
      for (int l = next++; l < layers; l = next++) {
        const sdnn_status r = sdnn_set_layer(net, l, &W[l], bias + (int64_t)l * neurons);
        if (r && !rcs[t]) {
          rcs[t] = r;
          errs[t] = sdnn_last_error();
        }
      }
    });
  for (auto &x : th) x.join();
  for (int t = 0; t < nt; ++t)
    if (rcs[t]) {
      sdnn_destroy(net);
      return fail(rcs[t], errs[t]);
    }
  *out = net;
  return SDNN_OK;
}

sdnn_status sdnn_infer_device(sdnn_net *net, const int64_t *d_rowptr, const int32_t *d_idx,
                              const float *d_val, int64_t batch, uint32_t *d_alive,
                              float *d_y_out, void *stream) {
  if (!net) return fail(SDNN_E_ARG, "net is NULL");
  if (batch < 0) return fail(SDNN_E_ARG, "batch < 0");
  if (batch > (int64_t(1) << 30)) return fail(SDNN_E_UNSUPPORTED, "batch > 2^30");
  if (!d_rowptr) return fail(SDNN_E_ARG, "d_rowptr is NULL");
  sdnn_status st = set_device(net);
  if (st) return st;
  return infer_device_impl(net, d_rowptr, d_idx, d_val, batch, d_alive, d_y_out,
                           (cudaStream_t)stream);
}

sdnn_status sdnn_infer(sdnn_net *net, const int64_t *y0_rowptr, const int32_t *y0_idx,
                       const float *y0_val, int64_t batch, int32_t *categories,
                       int64_t *n_categories, float *y_out) {
  if (!net || !y0_rowptr || !n_categories) return fail(SDNN_E_ARG, "NULL argument");
  if (batch < 0) return fail(SDNN_E_ARG, "batch < 0");
  if (batch > (int64_t(1) << 30)) return fail(SDNN_E_UNSUPPORTED, "batch > 2^30");
  if (batch > 0 && !categories) return fail(SDNN_E_ARG, "categories is NULL");
  sdnn_status st = set_device(net);
  if (st) return st;
  if (net->pending[0] >= 0 || net->pending[1] >= 0)
    return fail(SDNN_E_STATE, "submitted inferences are outstanding (sdnn_infer_wait first)");
  if ((st = host_enqueue(net, 0, y0_rowptr, y0_idx, y0_val, batch))) return st;
  float *d_yout = nullptr;
  cudaStream_t s = net->opts.stream ? (cudaStream_t)net->opts.stream : net->own;
  if (y_out && batch > 0) {
    CK(cudaMalloc(&d_yout, sizeof(float) * (size_t)net->n * (size_t)batch));
    launch_final_yout(net, batch, d_yout, s);
  }
  if ((st = host_finish(net, 0, categories, n_categories))) {
    cudaFree(d_yout);
    return st;
  }
  if (d_yout) {
    // on the compute stream, after k_yout (H.done was recorded before it, and
    // a legacy-stream copy does not wait for a non-blocking stream)
    CK(cudaMemcpyAsync(y_out, d_yout, sizeof(float) * (size_t)net->n * (size_t)batch, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    cudaFree(d_yout);
  }
  return SDNN_OK;
}

sdnn_status sdnn_infer_submit(sdnn_net *net, const int64_t *y0_rowptr, const int32_t *y0_idx,
                              const float *y0_val, int64_t batch, int64_t *ticket) {
  if (!net || !y0_rowptr || !ticket) return fail(SDNN_E_ARG, "NULL argument");
  if (batch < 0) return fail(SDNN_E_ARG, "batch < 0");
  if (batch > (int64_t(1) << 30)) return fail(SDNN_E_UNSUPPORTED, "batch > 2^30");
  sdnn_status st = set_device(net);
  if (st) return st;
  const int64_t t = net->next_ticket;
  const int slot = (int)(t & 1);
  if (net->pending[slot] >= 0) return fail(SDNN_E_STATE, "two submissions outstanding: sdnn_infer_wait first");
  if ((st = host_enqueue(net, slot, y0_rowptr, y0_idx, y0_val, batch))) return st;
  net->pending[slot] = t;
  net->next_ticket = t + 1;
  *ticket = t;
  return SDNN_OK;
}

sdnn_status sdnn_infer_wait(sdnn_net *net, int64_t ticket, int32_t *categories, int64_t *n_categories) {
  if (!net || !n_categories) return fail(SDNN_E_ARG, "NULL argument");
  const int slot = (int)(ticket & 1);
  if (ticket < 0 || net->pending[slot] != ticket) return fail(SDNN_E_STATE, "unknown or finished ticket");
  if (net->slots[slot].batch > 0 && !categories) return fail(SDNN_E_ARG, "categories is NULL");
  sdnn_status st = set_device(net);
  if (st) return st;
  net->pending[slot] = -1;
  return host_finish(net, slot, categories, n_categories);
}

sdnn_status sdnn_infer_device_nvls(sdnn_net *net, const int64_t *d_rowptr, const int32_t *d_idx,
                                   const float *d_val, int64_t batch, const sdnn_nvls *nv, void *stream) {
  if (!net || !nv) return fail(SDNN_E_ARG, "NULL argument");
  if (batch < 0 || batch > (int64_t(1) << 30)) return fail(SDNN_E_ARG, "batch out of range");
  if (!d_rowptr || !nv->local_words || !nv->mc_words || !nv->local_flag || !nv->mc_flag || nv->word_offset < 0)
    return fail(SDNN_E_ARG, "NULL argument");
  if (net->L < 1) return fail(SDNN_E_UNSUPPORTED, "the NVLS readout needs >= 1 layer");
  if (net->opts.flags & SDNN_F_SATURATE) return fail(SDNN_E_UNSUPPORTED, "NVLS readout with SDNN_F_SATURATE");
  sdnn_status st = set_device(net);
  if (st) return st;
  return infer_device_impl(net, d_rowptr, d_idx, d_val, batch, nullptr, nullptr, (cudaStream_t)stream,
                           nullptr, nv);
}

sdnn_status sdnn_nvls_barrier(uint32_t *local_flag, uint32_t *mc_flag, uint32_t target, void *stream) {
  if (!local_flag || !mc_flag) return fail(SDNN_E_ARG, "NULL argument");
  launch_nvls_barrier(local_flag, mc_flag, target, (cudaStream_t)stream);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(SDNN_E_CUDA, std::string("k_nvls_barrier: ") + cudaGetErrorString(e));
  return SDNN_OK;
}

sdnn_status sdnn_bitmask_to_ids(const uint32_t *d_words, int64_t batch, int32_t *d_ids, int32_t *d_n,
                                void *stream) {
  if (batch < 0 || batch > (int64_t(1) << 30)) return fail(SDNN_E_ARG, "batch out of range");
  if (!d_n || (batch > 0 && (!d_words || !d_ids))) return fail(SDNN_E_ARG, "NULL argument");
  launch_bitmask_ids(d_words, batch, d_ids, d_n, (cudaStream_t)stream);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(SDNN_E_CUDA, std::string("k_bitmask_ids: ") + cudaGetErrorString(e));
  return SDNN_OK;
}

sdnn_status sdnn_gather_rows(sdnn_net *net, const int32_t *d_rows, int64_t nrows, float *d_y,
                             void *stream) {
  if (!net) return fail(SDNN_E_ARG, "net is NULL");
  if (nrows < 0) return fail(SDNN_E_ARG, "nrows < 0");
  if (nrows > 0 && (!d_rows || !d_y)) return fail(SDNN_E_ARG, "NULL argument");
  if (net->ws_cap < 0 || (net->L > 0 && net->plan_dirty)) return fail(SDNN_E_STATE, "no inference yet");
  sdnn_status st = set_device(net);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  if (net->L == 0)
    launch_gather_rows(net->ws, 0, false, net->n, net->opts.ymax, d_rows, nrows, net->last_batch, d_y, s);
  else
    launch_gather_rows(net->ws, net->steps.back().a, true, net->n, net->opts.ymax, d_rows, nrows,
                       net->last_batch, d_y, s);
  CK(cudaGetLastError());
  return SDNN_OK;
}

sdnn_status sdnn_validate_layer(int32_t neurons, const sdnn_layer *W, const float *bias_l,
                                uint32_t flags, sdnn_layer_info *info) {
  if (!W || !bias_l) return fail(SDNN_E_ARG, "NULL argument");
  if (neurons < 1) return fail(SDNN_E_ARG, "neurons < 1");
  if (neurons > 65536) return fail(SDNN_E_UNSUPPORTED, "neurons > 65536 (u16 source indices)");
  LayerIn in{W->format, W->ell_k, W->rowptr, W->idx, W->val, W->uniform_value};
  PackedLayer p;
  std::string msg;
  const int rc = pack_layer(neurons, in, bias_l, !(flags & SDNN_F_NO_GROUPS), p, msg);
  if (rc) return fail(rc, msg);
  if (info) {
    info->ngroups = p.ngroups;
    info->kmax = p.kmax;
    info->gmax = p.gmax;
    info->uniform = p.uniform ? 1 : 0;
    info->regular = p.regular ? 1 : 0;
    info->bias_nonpositive = p.bias_nonpos ? 1 : 0;
    info->nnz = p.nnz;
  }
  return SDNN_OK;
}

sdnn_status sdnn_layer_times(const sdnn_net *cnet, float *ms) {
  sdnn_net *net = const_cast<sdnn_net *>(cnet);
  if (!net || !ms) return fail(SDNN_E_ARG, "NULL argument");
  if (!(net->opts.flags & SDNN_F_PROFILE)) return fail(SDNN_E_STATE, "handle not created with SDNN_F_PROFILE");
  if (!net->profiled) return fail(SDNN_E_STATE, "no profiled inference yet");
  sdnn_status st = set_device(net);
  if (st) return st;
  for (const Step &S : net->steps) {            // a fused pass is one kernel: split evenly
    float t = 0.f;
    CK(cudaEventSynchronize(net->ev_after[S.a]));
    CK(cudaEventElapsedTime(&t, net->ev_before[S.a], net->ev_after[S.a]));
    for (int j = 0; j < S.m; ++j) ms[S.a + j] = t / S.m;
  }
  return SDNN_OK;
}

sdnn_status sdnn_step_plan(const sdnn_net *net, int32_t *step_len, int32_t *nsteps) {
  if (!net || !nsteps || !step_len) return fail(SDNN_E_ARG, "NULL argument");
  if (net->plan_dirty && net->L > 0) return fail(SDNN_E_STATE, "no plan yet (run an inference first)");
  for (size_t i = 0; i < net->steps.size(); ++i) step_len[i] = net->steps[i].m;
  *nsteps = (int32_t)net->steps.size();
  return SDNN_OK;
}

sdnn_status sdnn_plan_steps(int32_t neurons, int32_t layers, const sdnn_layer *W,
                            const float *bias, const sdnn_opts *opts, int32_t *step_len,
                            int32_t *nsteps) {
  if (!nsteps || (layers > 0 && (!W || !bias || !step_len))) return fail(SDNN_E_ARG, "NULL argument");
  if (neurons < 1 || layers < 0) return fail(SDNN_E_ARG, "bad sizes");
  if (neurons > 65536) return fail(SDNN_E_UNSUPPORTED, "neurons > 65536");
  sdnn_opts o;
  sdnn_status st = check_opts(opts, o);
  if (st) return st;
  std::vector<PackedLayer> host(layers);
  for (int l = 0; l < layers; ++l) {
    LayerIn in{W[l].format, W[l].ell_k, W[l].rowptr, W[l].idx, W[l].val, W[l].uniform_value};
    std::string msg;
    const int rc = pack_layer(neurons, in, bias + (int64_t)l * neurons,
                              !(o.flags & SDNN_F_NO_GROUPS), host[l], msg);
    if (rc) return fail(rc, "layer " + std::to_string(l) + ": " + msg);
  }
  std::vector<const PackedLayer *> lp(layers);
  for (int l = 0; l < layers; ++l) lp[l] = &host[l];
  // as make_plan, without the resident tail (a plan of fused passes and layers)
  const int cta = pass_cta_rows(yblock_wanted() && !(o.flags & SDNN_F_SATURATE) && o.stream_slots == 0);
  const int cap = (o.flags & SDNN_F_SATURATE)
                      ? 0
                      : std::min(o.fuse_rows < 0 ? kDefaultPassRows : o.fuse_rows, cta * kMaxPassCluster);
  const int maxm = o.fuse_layers < 0 ? 8 : o.fuse_layers;
  const std::vector<Step> steps = plan_passes(lp, neurons, cap, maxm, pass_tile_floats(), 1, nullptr, cta);
  for (size_t i = 0; i < steps.size(); ++i) step_len[i] = steps[i].m;
  *nsteps = (int32_t)steps.size();
  return SDNN_OK;
}

sdnn_status sdnn_stats_get(const sdnn_net *cnet, sdnn_stats *out, int64_t *live_rows) {
  sdnn_net *net = const_cast<sdnn_net *>(cnet);
  if (!net || !out) return fail(SDNN_E_ARG, "NULL argument");
  if (out->struct_size < (int32_t)sizeof(sdnn_stats)) return fail(SDNN_E_ARG, "struct_size too small");
  sdnn_stats s{};
  s.struct_size = sizeof(sdnn_stats);
  s.neurons = net->n;
  s.layers = net->L;
  s.path = (net->fused_layers > 0 ? 1 : 0) | (net->resident_layers > 0 ? 2 : 0) | (net->yblk > 0 ? 4 : 0);
  s.steps = (int32_t)net->steps.size();
  s.fused_layers = net->fused_layers;
  s.resident_layers = net->resident_layers;
  s.grouped_layers = net->grouped_layers;
  s.max_group = net->max_group;
  s.max_k = net->max_k;
  s.compaction = compact_enabled(net) ? 1 : 0;
  s.packed_weight_bytes = (int64_t)net->arena.total;
  s.stream_bytes = weight_streaming(net) ? net->stream_bytes : 0;
  s.stream_slot_bytes = weight_streaming(net) ? (int64_t)net->slot_bytes : 0;
  for (int l = 0; l < net->L; ++l) s.total_nnz += net->nnz[l];
  s.last_batch = net->last_batch;
  s.last_n_categories = net->last_ncat;
  s.launches_per_infer = net->launches;
  if (net->L > 0 && net->ws.live && net->last_batch > 0) {
    sdnn_status st = set_device(net);
    if (st) return st;
    std::vector<int32_t> live(net->L);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(live.data(), net->ws.live, sizeof(int32_t) * net->L, cudaMemcpyDeviceToHost));
    if (live_rows)
      for (int l = 0; l < net->L; ++l) live_rows[l] = live[l];
    // live edges: layer l processes the rows alive after layer l-1 (all kept rows for l = 0)
    int32_t kept0 = 0;
    LayerState s0;
    CK(cudaMemcpy(&s0, net->ws.st, sizeof(LayerState), cudaMemcpyDeviceToHost));
    kept0 = s0.width;
    s.kept_rows = kept0;
    if (net->ws.nretired) {
      int32_t r = 0;
      CK(cudaMemcpy(&r, net->ws.nretired, sizeof(int32_t), cudaMemcpyDeviceToHost));
      s.retired_rows = r;
    }
    for (int l = 0; l < net->L; ++l)
      s.live_edges += (int64_t)(l == 0 ? kept0 : live[l - 1]) * net->nnz[l];
    std::vector<LayerState> sts(net->L + 1);
    CK(cudaMemcpy(sts.data(), net->ws.st, sizeof(LayerState) * (net->L + 1), cudaMemcpyDeviceToHost));
    for (const Step &S : net->steps)
      for (int l = S.a; l < S.a + S.m; ++l) {
        s.executed_fma += (int64_t)sts[S.a].width * net->fma_l[l];
        s.computed_rows += sts[S.a].width;
      }
  }
  *out = s;
  return SDNN_OK;
}

void sdnn_destroy(sdnn_net *net) {
  if (!net) return;
  cudaSetDevice(net->device);
  cudaDeviceSynchronize();
  free_ws(net);
  net->arena.release();
  free_stream(net);
  net->pass_arena.release();
  if (net->copy_s) cudaStreamDestroy(net->copy_s);
  if (net->ev_fork) cudaEventDestroy(net->ev_fork);
  if (net->ev_join) cudaEventDestroy(net->ev_join);
  for (HostSlot &H : net->slots) {
    if (H.validator.joinable()) H.validator.join();
    cudaFree(H.d_rowptr);
    cudaFree(H.d_idx);
    cudaFree(H.d_val);
    if (H.h_res) cudaFreeHost(H.h_res);
    if (H.done) cudaEventDestroy(H.done);
    if (H.in_free) cudaEventDestroy(H.in_free);
  }
  if (net->h_stage) cudaFreeHost(net->h_stage);
  if (net->in_s) cudaStreamDestroy(net->in_s);
  for (auto e : net->ev_stage) if (e) cudaEventDestroy(e);
  if (net->ev_in) cudaEventDestroy(net->ev_in);
  for (auto e : net->ev_chunk) cudaEventDestroy(e);
  if (net->own) cudaStreamDestroy(net->own);
  for (auto e : net->ev_before) if (e) cudaEventDestroy(e);
  for (auto e : net->ev_after) if (e) cudaEventDestroy(e);
  cudaGetLastError();
  delete net;
}

}  // extern "C"
