// sdnn_internal.h -- shared declarations of the product library (host packer,
// launch layer, device kernels).  Not part of the public ABI (include/sdnn.h).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

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
//   val[G_g][K_g]      per-slot weights, unless the layer is uniform,
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
  std::vector<float> val;     // [ngroups][gmax][kmax] (empty if uniform)
  std::vector<float> bias;    // [n]
};

struct LayerIn {              // mirrors sdnn_layer
  int32_t format;
  int32_t ell_k;
  const int64_t *rowptr;
  const int32_t *idx;
  const float *val;
  float uniform_value;
};

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
  const float *val;      // nullptr if uniform
  const float *bias;     // [n]
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

struct Workspace {
  float *Y[2] = {nullptr, nullptr};   // [n][stride] neuron-major activations
  int32_t *rid[2] = {nullptr, nullptr};
  uint32_t *alive[2] = {nullptr, nullptr};  // [stride/32]
  uint32_t *inmask = nullptr;         // densify: rows kept
  int32_t *wpre = nullptr;            // [stride/32 + 1] exclusive prefix of popcounts
  LayerState *st = nullptr;           // [L + 1]
  int32_t *live = nullptr;            // [L] live rows after each layer
  int32_t *cats = nullptr;            // [stride] category list
  int32_t *ncat = nullptr;            // [1]
  int64_t stride = 0;                 // row stride (capacity in batch columns, mult of 128)
  int64_t words = 0;                  // stride / 32
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
void launch_layer(const LaunchCfg &c, const Workspace &w, const DevLayer &L, int32_t layer,
                  float ymax, int32_t n, cudaStream_t s);
void launch_scan(const Workspace &w, int32_t layer, bool compact, int32_t n, cudaStream_t s);
void launch_compact_copy(const LaunchCfg &c, const Workspace &w, int32_t layer, int32_t n,
                         cudaStream_t s);
void launch_zero_layers_alive(const Workspace &w, int64_t batch, const int64_t *rowptr,
                              const float *val, cudaStream_t s);
void launch_readout(const Workspace &w, int32_t last_state, bool after_layer,
                    uint32_t *d_alive_out, int64_t batch, cudaStream_t s);
void launch_yout(const Workspace &w, int32_t last_state, int32_t n, int64_t batch,
                 float *d_yout, cudaStream_t s);

}  // namespace sdnn
