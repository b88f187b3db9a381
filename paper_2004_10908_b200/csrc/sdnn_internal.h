// sdnn_internal.h -- shared declarations of the product library (host packer,
// launch layer, device kernels).  Not part of the public ABI (include/sdnn.h).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include <cuda.h>
#include <cuda_runtime.h>

namespace sdnn {

// ---------------------------------------------------------------------------
// Packed layer (host side, produced by pack.cpp)
//
// A layer is stored as GROUPS: a group is a set of up to kMaxGroup output
// columns whose (ascending) source lists are identical.  The RadiX-Net-shaped
// workload has N/32 groups of 32 per layer (every layer is a set of dense
// 32x32 blocks); a random-regular layer has N groups of 1.  A group carries
//   src[K_g]           its sources, ascending (u16 when N <= 65536),
//   col[G_g]           its member output columns, ascending,
//   val[K_g][G_g]      per-slot weights (source-major: the weights of term t
//                      for all members are contiguous), unless the layer is uniform,
// The chain of every member is evaluated over exactly its K_g sources in
// ascending order, so no padding term ever enters the arithmetic.
// ---------------------------------------------------------------------------
constexpr int kMaxGroup = 32;

struct PackedLayer {
  int32_t n = 0;
  int32_t ngroups = 0;
  int32_t kmax = 0;           // max K_g
  int32_t gmax = 0;           // max G_g
  int64_t nnz = 0;            // stored nonzeros (explicit zeros included)
  bool uniform = true;        // every stored value bit-identical
  float wu = 0.f;             // the uniform value
  bool bias_nonpos = true;    // all b_j <= 0
  // flattened group arrays, row stride kmax / gmax (padding never read)
  bool regular = true;        // every group has K_g == kmax and G_g == gmax
  std::vector<uint16_t> src;  // [ngroups][kmax]
  std::vector<int32_t> col;   // [ngroups][gmax] (-1 pad)
  std::vector<int32_t> gk;    // [ngroups] K_g
  std::vector<int32_t> gg;    // [ngroups] G_g
  std::vector<float> val;     // [ngroups][kmax][gmax] (empty if uniform)
  std::vector<float> bias;    // [n]
  std::vector<float> gbias;   // [ngroups][gmax] bias of each member (non-uniform layers only)
};

struct LayerIn {              // mirrors sdnn_layer
  int32_t format;
  int32_t ell_k;
  const int64_t *rowptr;
  const int32_t *idx;
  const float *val;
  float uniform_value;
};

// f2: does an all-ymax input row give an all-ymax output row (every column's
// canonical chain on ymax inputs plus its bias >= ymax)?
bool saturation_preserving(const PackedLayer &p, float ymax);

// Validate and pack one layer.  Returns 0 or a negative sdnn_status with msg.
int pack_layer(int32_t n, const LayerIn &in, const float *bias, bool allow_groups,
               PackedLayer &out, std::string &msg);

// ---------------------------------------------------------------------------
// Device-side views
// ---------------------------------------------------------------------------
struct DevLayer {
  const uint16_t *src;   // [ngroups][kmax]
  const int32_t *col;    // [ngroups][gmax]
  const int32_t *gk;     // [ngroups]
  const int32_t *gg;     // [ngroups]
  const float *val;      // [ngroups][kmax][gmax], nullptr if uniform
  const float *bias;     // [n]
  const float *gbias;    // [ngroups][gmax] member biases (non-uniform layers), else nullptr
  int32_t ngroups, kmax, gmax;
  float wu;
  int32_t uniform;
  int32_t regular;
  int64_t nnz;
};

// Per-layer device state written by the scan kernel of layer l-1 (or densify
// for l = 0) and read by every kernel of layer l.  Lets a captured CUDA Graph
// follow data-dependent compaction without host round trips.
struct LayerState {
  int32_t in;        // which Y buffer holds this layer's input (0/1)
  int32_t width;     // live positions (batch columns) in that buffer
  int32_t rid;       // which row-id buffer maps positions -> original rows
  int32_t compacted; // 1 if the scan before this layer compacted
};

// ---------------------------------------------------------------------------
// Multi-layer passes ("model decomposition").
// A step runs layers [a, a+m).  For m > 1 the union of the m layers' bipartite
// graphs splits into small connected components (for RadiX-Net butterflies:
// 2^(5+2(m-1)) neurons); every component is closed, so one CTA can load a
// component's input rows for a batch tile, run all m layers out of shared
// memory, and write only the last layer's rows back to HBM.  When every source
// row of a (non-last) layer feeds exactly one group and no group has more
// members than sources, each group overwrites its own source slots in place, so
// a component tile needs no second buffer.  Each output's chain is still the
// canonical ascending-source fmaf sequence.
// ---------------------------------------------------------------------------
constexpr int kMaxPassLayers = 16;
constexpr int kMaxPassRows = 1024;     // slots per CTA (one 64 KB tile of >= 16 positions)
constexpr int kDefaultPassRows = 1024; // default component cap (C4: 2324 ms vs 2435 at 512, 2652 at 2048)
constexpr int kDefaultCtaRows = 512;   // slots per CTA with row-major activations
constexpr bool kYBlockDefault = true;  // position-blocked activations (SDNN_YBLOCK=0 disables)
int pass_cta_rows(bool blocked);
constexpr int kMaxPassCluster = 4;     // CTAs per component (thread-block cluster, DSMEM)

struct Step {
  int32_t a = 0, m = 1;                // layers [a, a+m)
  int32_t pass = -1;                   // fused-pass table index; -1 single layer; kResidentStep
};
constexpr int32_t kResidentStep = -2;  // layers [a, L) in the SMEM-resident kernel

// plan greedy fused passes: extend while the layers are uniform with K <= 32,
// every layer but the last allows in-place slots (exclusive sources,
// G_g <= K_g), the sub-components of all layers but the last fit one CTA
// (kMaxPassRows slots) and every component's sub-components pack into
// cap / kMaxPassRows CTAs (cap <= kMaxPassRows * kMaxPassCluster); tile
// T = 16384 / (rows per CTA rounded up to a power of two), 32 <= T <= 512
std::vector<Step> plan_steps(const std::vector<const PackedLayer *> &layers, int32_t n, int cap,
                             int max_m, int cta_rows, int a_begin = 0, bool general = false);

struct PassHostLayer {
  int32_t NG = 0;                      // group slots per component (max over components)
  float wu = 0.f;
  bool bias_uniform = false;           // every member's bias is bu (no bias array in the record)
  bool dedup = false;                  // members share one value slot (uniform w, equal biases)
  std::vector<uint16_t> vs;            // dedup: [ncomp][NG] value slot of each group
  int32_t off_vs = -1;
  int32_t vt = 0;                      // value table (fuse.cpp): 1 = this layer writes it, 2 = reads it
  float bu = 0.f;
  int32_t off_kg = 0, off_src = 0, off_bias = 0, off_orow = -1;  // record byte offsets
  std::vector<uint16_t> src;           // [ncomp][NG][32] smem slots of the sources
  std::vector<float> bias;             // [ncomp][NG][32] bias of each member
  std::vector<uint16_t> orow;          // last layer only: [ncomp][NG][32] output rows (N <= 65536)
  std::vector<uint8_t> k, g;           // [ncomp][NG] sources / members (0 = empty slot)
  bool general = false;                // per-slot weights (k_pass_gw): gid[ncomp][NG] = the group's
  std::vector<uint16_t> gid;           // index in W_l (source-major [G][kmax][gmax])
  int32_t off_gid = -1;
};
struct PassHost {
  int32_t a = 0, m = 0, ncomp = 0, rin = 0, R = 0, T = 0;
  int32_t C = 1;                       // CTAs per component (cluster size; rows/records per [comp][bin])
  int32_t NB = 1;                      // tile buffers per CTA (2: T for a half tile, double-buffered;
                                       // 3: pass_wide.cu, 1024 rows x 32 positions in rotating halves)
  std::vector<int32_t> in_rows;        // [ncomp][rin]  global neuron ids at boundary a
  std::vector<int32_t> in_count;       // [ncomp]
  std::vector<int32_t> split;          // NB = 3: [ncomp] slots in half 0 (pass_wide.cu)
  int32_t NW = 0, S = 1;               // > 0: k_pass_t32 with NW warps and S tile buffers per CTA
  bool general = false;                // some layer has per-slot weights: k_pass_gw<NW>
  std::vector<PassHostLayer> layers;   // [m]
  // per-component metadata record (one bulk copy next to the tile):
  //   for each layer j: kg[NG_j] u16 (K | G << 8) padded to 16 B, src[NG_j][32] u16
  //   slot codes (bin << 10 | slot), bias[NG_j][32] f32 unless the layer's biases
  //   are uniform over the pass; last layer: orow[NG][32] u16
  int32_t rec_bytes = 0;
  std::vector<unsigned char> rec;      // [ncomp][rec_bytes]
};
constexpr int kPassRecMax = 10224;     // record bytes per component (3 CTAs per SM: 3 x 75 KB)
// blocked: the plan is for position-blocked activations (pass_wide.cu kernels allowed)
// prev: the step before s (its components order the rows of s's bins)
void build_pass(const std::vector<const PackedLayer *> &layers, int32_t n, const Step &s,
                int tile_floats, int cta_rows, PassHost &out, bool share_values = false, bool blocked = false,
                const Step *prev = nullptr);
// plan_steps, build every fused pass; a pass whose record exceeds kPassRecMax
// drops its last layer and the rest is planned again; `built[i]` is the
// PassHost of steps[i] (m > 1, or m == 1 with single_passes; else m == 0)
std::vector<Step> plan_passes(const std::vector<const PackedLayer *> &layers, int32_t n, int cap,
                              int max_m, int tile_floats, int threads,
                              std::vector<PassHost> *built, int cta_rows, bool single_passes = false,
                              bool share_values = false);

struct PassLayerDev {
  int32_t off_kg, off_src, off_bias, off_orow;   // byte offsets in the component record
  int32_t NG;                                    // off_bias < 0: every bias is bu
  float wu, bu;
  int32_t off_vs;                                // >= 0: non-last layer stores one value per group
                                                 // into the slot vs[group] (u16 array at this offset)
  int32_t vt;                                    // value table: 1 = write (two copies per group line),
                                                 // 2 = read (line = code, copy = phase half)
  int32_t off_gid;                               // >= 0: per-slot weights, u16 group ids at this offset
  const float *wv;                               // ... of W_l = wv[gid][t][member], strides wk, wg
  int32_t wk, wg;
};
struct alignas(64) DevPass {
  // T = 16 passes over position-blocked activations: one TMA tensor map per
  // activation buffer (dims {32 positions, N rows, stride/32 blocks}, box
  // {16, 256, 1}), so a tile's half-block rows arrive as <= 4 box copies
  // instead of 16-byte LDGSTS chunks; tma16 = 0 when not encoded
  CUtensorMap tmap[2];
  int32_t tma16;
  int32_t a, m, ncomp, rin, R, T, rec_bytes;
  int32_t C;                           // cluster size: in_rows/in_count/rec indexed [comp * C + rank]
  int32_t yblk;                        // 0: Y is [rows][stride]; R > 0: Y is [stride/32][R][32] and
                                       // every (comp, rank)'s rows are R-consecutive storage rows
  int32_t order;                       // item order: 0 component-major, 1 tile-major
  int32_t lg_in, lg_out;               // yblk: log2 positions per block at the input / output
                                       // boundary (5; 4 where a T = 16 pass reads)
  int32_t pf;                          // yblk: L2-prefetch the tiles of the next pf items
  int32_t NB;                          // tile buffers per CTA (2: half-size tiles, double-buffered)
  const int32_t *in_rows, *in_count;
  const int32_t *split;                // NB = 3: [ncomp] slots in half 0
  int32_t NW, S;                       // NW > 0: k_pass_t32<NW, S> (pass_wide.cu)
  int32_t general;                     // k_pass_gw<NW> (per-slot weights)
  const unsigned char *rec;            // [ncomp][rec_bytes]
  PassLayerDev layers[kMaxPassLayers]; // by value: the kernel parameter carries them
};

// SMEM-resident multi-layer kernel (resident.cu), N <= 4096
struct ResLayerDev {
  const unsigned char *blob;           // device weight image of the layer (see resident.cu)
  int32_t G, gmax, bytes;
  float wu;
  int32_t regular, bias_uniform;
  float bias0;
  int32_t off_col, off_bias, off_counts;
};
int resident_positions(int n);         // batch positions per CTA (0 = not eligible)
constexpr int kResidentDefaultMaxN = 1024;  // resident tail by default only up to this width
int resident_max_blob();
bool build_resident_blob(const PackedLayer &p, std::vector<unsigned char> &blob, ResLayerDev &d);
void configure_resident();

// ---------------------------------------------------------------------------
// Workspace
// ---------------------------------------------------------------------------
struct Workspace {
  float *Y[2] = {nullptr, nullptr};   // [n][stride] neuron-major activations
  int32_t *rid[2] = {nullptr, nullptr};
  uint32_t *alive[2] = {nullptr, nullptr};  // two sets of [kMaxPassLayers][words] bitmasks
  uint32_t *inmask = nullptr;         // densify: rows kept
  int32_t *wpre = nullptr;            // [words + 1] exclusive prefix of popcounts
  LayerState *st = nullptr;           // [L + 1]
  int32_t *live = nullptr;            // [L] live rows after each layer
  int32_t *cats = nullptr;            // [stride] category list
  int32_t *ncat = nullptr;            // [1]
  // f2 (SDNN_F_SATURATE): all-outputs-saturated bits per step parity, rows
  // retired as saturated (original-row bitmask), their count, readout scratch
  uint32_t *sat[2] = {nullptr, nullptr};
  uint32_t *retired = nullptr;         // original-row bitmask of retired rows
  uint32_t *pret = nullptr;            // positions retired but not yet compacted away
  int32_t *nretired = nullptr;
  uint32_t *orig = nullptr;
  int64_t stride = 0;                 // row stride (capacity in batch columns)
  // position-blocked activations (plan property, see make_plan): yblk = storage
  // rows R, element (row r, position p) at ((p / 32) * R + r) * 32 + p % 32;
  // sig0[neuron] = storage row of an input neuron (NULL: identity)
  int32_t yblk = 0;
  int32_t lg0 = 5;                    // log2 positions per block at boundary 0
  const int32_t *sig0 = nullptr;
  int64_t words = 0;                  // stride / 32
  uint32_t *alive_set(int s) const { return alive[s & 1]; }
  uint32_t *alive_row(int s, int j) const { return alive[s & 1] + (int64_t)j * words; }
};

// ---------------------------------------------------------------------------
// Kernel launchers (kernels.cu).  All enqueue on `s`, never synchronise.
// ---------------------------------------------------------------------------
struct LaunchCfg {
  int sms = 148;
  int layer_blocks = 148 * 8;
  int copy_blocks = 148 * 4;
  bool bulk = true;            // TMA bulk-copy pipeline for uniform layers with K <= 32
};

int bulk_stride_quantum();     // activation row stride must be a multiple of this
void configure_kernels();      // one-time function attributes (dynamic smem)

void launch_densify(const LaunchCfg &c, const Workspace &w, int32_t n, int64_t batch,
                    const int64_t *rowptr, const int32_t *idx, const float *val, bool compact,
                    cudaStream_t s);
// densify in two parts (sdnn_infer overlaps the input copy with the scatter):
// zero Y0 + row flags + scan (needs rowptr, and val when it is given), then
// the scatter of rows [r0, r1) once their indices are on the device
void launch_densify_prep(const LaunchCfg &c, const Workspace &w, int32_t n, int64_t batch,
                         const int64_t *rowptr, const float *val, bool compact, cudaStream_t s);
void launch_scatter_rows(const LaunchCfg &c, const Workspace &w, int32_t n, int64_t r0, int64_t r1,
                         const int64_t *rowptr, const int32_t *idx, const float *val, cudaStream_t s);
// one layer: reads state st[a], writes its liveness bits to `alive`
void launch_layer(const LaunchCfg &c, const Workspace &w, const DevLayer &L, int32_t a,
                  uint32_t *alive, float ymax, cudaStream_t s, uint32_t *sat = nullptr);
bool layer_tracks_saturation(const LaunchCfg &c, const DevLayer &L);
int pass_tile_floats();        // smem floats per component tile (tile T = this / R)
bool pass_variant(int T, int C, int NB = 1);   // a k_pass instance exists for tile T, cluster C, NB buffers
// 513-1024-row components, 32-position tiles, one CTA per SM (pass_wide.cu;
// PassHost.NB = 3); pass_wide_enabled(): SDNN_PASS_WIDE != 0
bool pass_wide_enabled();
// <= 512-row components, 32-position tiles, CTAs of NW = ceil(rows / 128)
// warps sized by the pass (pass_wide.cu; PassHost.NW > 0); pass_t32_mode():
// SDNN_PASS_T32 (0 off, 1 up to 256 rows, 2 up to 512 rows); buffers per CTA
// for NW warps: pass_t32_stages(NW) (SDNN_PASS_T32_S)
int pass_t32_mode();
int pass_t32_stages(int nw);
bool pass_t32_variant(int nw, int s, int c = 1);
int pass_wide_mode();
void launch_pass_t32(const LaunchCfg &c, const Workspace &w, const DevPass &P, uint32_t *alive, float ymax,
                     cudaStream_t s);
void configure_pass_wide();
void launch_pass_gw(const LaunchCfg &c, const Workspace &w, const DevPass &P, uint32_t *alive, float ymax,
                    cudaStream_t s);
void launch_pass_wide(const LaunchCfg &c, const Workspace &w, const DevPass &P, uint32_t *alive, float ymax,
                      cudaStream_t s);
// a fused pass: reads st[P.a], liveness of layer a+j to alive + j*words
void launch_pass(const LaunchCfg &c, const Workspace &w, const DevPass &P, uint32_t *alive,
                 float ymax, cudaStream_t s);
// after a step [a, a+m): live counts of its m layers, compaction decision -> st[a+m],
// zero the next step's bitmask set
void launch_scan(const Workspace &w, int32_t a, int32_t m, uint32_t *alive_cur,
                 uint32_t *alive_next, bool compact, cudaStream_t s,
                 const uint32_t *sat_cur = nullptr, uint32_t *sat_next = nullptr);
void launch_readout_retired(const Workspace &w, int32_t a, const uint32_t *alive_last,
                            uint32_t *d_alive_out, int64_t batch, cudaStream_t s);
void launch_yout_retired(const Workspace &w, int32_t n, int64_t batch, float ymax, float *d_yout,
                         cudaStream_t s);
void launch_compact_copy(const LaunchCfg &c, const Workspace &w, int32_t a, int32_t m,
                         const uint32_t *alive_last, int32_t n, cudaStream_t s, int lg = 5);
void launch_zero_layers_alive(const Workspace &w, int64_t batch, const int64_t *rowptr,
                              const float *val, cudaStream_t s);
// categories from the final liveness bits `alive_last` of the step entered with st[a]
void launch_readout(const Workspace &w, int32_t a, const uint32_t *alive_last,
                    uint32_t *d_alive_out, int64_t batch, cudaStream_t s);
// Y_L: final_out = the output buffer of the step entered with st[a] (L > 0), else Y_0
void launch_yout(const Workspace &w, int32_t a, bool final_out, int32_t n, int64_t batch,
                 float *d_yout, cudaStream_t s);
// f4: readout into the symmetric bitmask + multimem.st to every GPU + arrival wait
void launch_readout_nvls(const Workspace &w, int32_t a, const uint32_t *alive_last, int64_t batch,
                         uint32_t *local_words, uint32_t *mc_words, uint32_t *local_flag, uint32_t *mc_flag,
                         uint32_t target, cudaStream_t s);
void launch_nvls_barrier(uint32_t *local_flag, uint32_t *mc_flag, uint32_t target, cudaStream_t s);
// global category bitmask (batch bits) -> ascending ids, count in *d_n
void launch_bitmask_ids(const uint32_t *d_words, int64_t batch, int32_t *d_ids, int32_t *d_n, cudaStream_t s);
// Y_L rows of the given original row ids (same buffer selection as launch_yout)
void launch_gather_rows(const Workspace &w, int32_t a, bool final_out, int32_t n, float ymax,
                        const int32_t *d_rows, int64_t nrows, int64_t batch, float *d_y, cudaStream_t s);
void launch_resident(const Workspace &w, const ResLayerDev *layers, int a, int L, int n,
                     uint32_t *alive_final, bool compact, float ymax, cudaStream_t s);

}  // namespace sdnn
