/*
 * sdnn.h -- C ABI of the B200-native sparse-DNN inference hot path.
 *
 * The operation (one call of sdnn_infer / sdnn_infer_device):
 *
 *   Y_0          = the input matrix (B rows x N neurons), given as CSR
 *   Y_{l+1}      = min(max(Y_l . W_l + b_l, 0), YMAX)      l = 0 .. L-1
 *   categories   = { i : exists j, Y_L[i][j] > 0 }          ascending, 0-based
 *
 *   - layer formula, YMAX = 32, "which rows remain nonzero", the function names
 *     sdnn_create / sdnn_infer / sdnn_destroy: BASELINE.json north_star;
 *   - dataset parts (input matrix, L sparse layers, bias values, truth
 *     categories): PAPER.md:2557-2559 (Sec. 7.4, Large Sparse Neural Network
 *     Inference); the golden check of categories: PAPER.md:2570;
 *   - raw caller-owned pointers, no data abstraction: the design stance of
 *     PAPER.md:646-660 (Sec. 4.5).
 *
 * Arithmetic (readings A5/A6, identical to the oracle's): every
 * output is the fp32 chain  acc = +0; acc = fmaf(Y[i][k_t], w_t, acc)  over the
 * column's stored sources k_t in ASCENDING k, then z = acc + b_j (one fp32
 * add), then y = z > 0 ? fminf(z, YMAX) : +0.  Results are therefore
 * bit-identical to the CPU oracle (oracle/), not merely within tolerance.
 *
 * Conventions for every function:
 *   - return SDNN_OK (0) or a negative sdnn_status; on error the outputs are
 *     unspecified and sdnn_last_error() returns a thread-local message;
 *   - SDNN_E_CUDA is sticky: the handle must be destroyed;
 *   - a handle is not re-entrant: do not call two functions on the same handle
 *     concurrently (sdnn_set_layer on DIFFERENT layers is the one exception);
 *   - the caller owns every buffer it passes; the library keeps no caller
 *     pointer after a call returns (sdnn_infer_device: until the stream reaches
 *     the end of the enqueued work).
 */
#ifndef SDNN_H
#define SDNN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SDNN_ABI_VERSION 3

typedef struct sdnn_net sdnn_net;
typedef int32_t sdnn_status;

enum {
  SDNN_OK = 0,
  SDNN_E_ARG = -1,          /* NULL pointer, size out of range, bad option        */
  SDNN_E_FORMAT = -2,       /* malformed CSR/ELL, duplicate entry, non-finite     */
  SDNN_E_UNSUPPORTED = -3,  /* valid but outside this build (e.g. N > 2^30)      */
  SDNN_E_NOMEM = -4,        /* host or device allocation failed                  */
  SDNN_E_CUDA = -5,         /* CUDA runtime error (sticky)                       */
  SDNN_E_STATE = -6         /* call out of order (e.g. infer before all layers)  */
};

/* Weight formats of one layer W_l (an N x N sparse matrix; W_l[k][j] connects
 * input neuron k to output neuron j, i.e. Y_{l+1} = Y_l . W_l). */
enum {
  SDNN_W_CSR = 0,    /* rows = input neurons k: rowptr[N+1], idx[nnz] = output j */
  SDNN_W_ELLCOL = 1  /* per OUTPUT j, ell_k slots: idx[j*ell_k + t] = source k or -1
                        (padding, any position); slot order is irrelevant          */
};

typedef struct sdnn_layer {
  int32_t format;          /* SDNN_W_CSR or SDNN_W_ELLCOL                                 */
  int32_t ell_k;           /* ELLCOL: slots per output (>= 0); CSR: ignored               */
  const int64_t *rowptr;   /* CSR: [N+1], rowptr[0] = 0, non-decreasing; ELLCOL: NULL    */
  const int32_t *idx;      /* CSR: [rowptr[N]] output ids; ELLCOL: [N*ell_k] source ids  */
  const float *val;        /* same length as idx, or NULL: every stored value is
                              uniform_value (the challenge style, w = 1/16)              */
  float uniform_value;     /* used iff val == NULL                                        */
} sdnn_layer;

/* Option flags */
enum {
  SDNN_F_NO_COMPACT = 1u << 0,   /* never drop dead rows (always also implied when some
                                    bias > 0, because then a dead row can revive)        */
  SDNN_F_NO_GROUPS = 1u << 1,    /* do not merge columns with identical source lists
                                    (forces the one-column-per-group gather path)        */
  SDNN_F_NO_GRAPH = 1u << 2,     /* launch the layer chain as a plain stream loop
                                    instead of one captured CUDA Graph (f1 study)        */
  SDNN_F_NO_RESIDENT = 1u << 3,  /* disable the SMEM-resident multi-layer kernel        */
  SDNN_F_TRUST_INPUT = 1u << 4,  /* sdnn_infer: skip host validation of Y0              */
  SDNN_F_PROFILE = 1u << 5,      /* record a CUDA event pair around every layer kernel
                                    (read back with sdnn_layer_times)                    */
  SDNN_F_NO_BULK = 1u << 6,      /* uniform layers: use the register-staged gather kernel
                                    instead of the TMA bulk-copy pipeline                */
  SDNN_F_SHARE_VALUES = 1u << 9, /* fused passes: a layer with uniform weights and equal
                                    biases stores one value per column group in shared
                                    memory instead of one per member (exact; measured
                                    slower on C4, so opt-in)                             */
  SDNN_F_SATURATE = 1u << 8      /* f2 (reported separately): a row whose
                                    every output equals YMAX before a suffix of layers
                                    that map all-YMAX rows to all-YMAX rows (checked per
                                    layer with the canonical fmaf chain at create time)
                                    is a category with Y_L = YMAX: it is retired from
                                    the working set like a dead row.  Exact; it changes
                                    the work, so its numbers are not the headline.
                                    Streaming path only (no resident/fused steps)       */
};

typedef struct sdnn_opts {
  int32_t device;   /* CUDA device ordinal; -1 = the calling thread's current device  */
  uint32_t flags;   /* SDNN_F_*                                                        */
  float ymax;       /* clip value YMAX (> 0, finite); north_star: 32                   */
  void *stream;     /* cudaStream_t for sdnn_infer (NULL = a stream owned by the net) */
  int32_t fuse_rows;   /* multi-layer passes ("model decomposition"):
                          consecutive uniform layers run as one pass over the
                          connected components of their union, so a component
                          has <= fuse_rows neurons (0 = off; -1 = 1024).  All
                          layers but the last stay inside one CTA (sub-components
                          of <= R neurons updated in place in shared memory); the
                          last layer may read across a thread-block cluster
                          (distributed shared memory).  Position-blocked
                          activations (stats.path bit 2): R = 1024, 32-position
                          tiles of <= 512-row components in CTAs sized by the
                          component, 1024-row components over 2-CTA clusters
                          (passes of >= 3 layers) or one CTA per SM (2 layers);
                          row-major: R = 512, up to 4 R over clusters, larger
                          values are clamped                                      */
  int32_t fuse_layers; /* at most this many layers per pass (<= 16; -1 = 8)           */
  int32_t resident_from; /* N <= 4096: layers [resident_from, L) run in one kernel that
                          keeps each CTA's batch tile resident in shared memory
                          (earlier layers stream with dead-row compaction);
                          -1 = 24 when L > 32 and N <= 1024 (else off: from 2048
                          neurons the fused passes are faster, C2 4096x480: 19.2
                          vs 20.3 ms); >= L or SDNN_F_NO_RESIDENT = off           */
  int32_t stream_slots; /* weight streaming (the paper streams weight
                          partitions because "preloading ... is impossible",
                          PAPER.md:2560-2569).  0 = every packed layer and pass
                          descriptor resident in HBM.  S >= 1: they stay in pinned
                          host memory and each step's block is copied into a ring
                          of S device slots on a copy stream, step i+S's copy
                          issued as soon as step i's kernel has released its slot,
                          so the upload of later steps overlaps the compute of
                          earlier ones (inside the same captured graph).  Device
                          footprint: S x the largest step block.  The SMEM-resident
                          tail is not used in this mode.  Results are identical. */
} sdnn_opts;        /* opts = NULL means {-1, 0, 32.0f, NULL, -1, -1, -1, 0}           */

/* Create a network handle and load all L layers.
 *   neurons  N, 1 <= N <= 65536 on this build (u16 source indices); larger N
 *            returns SDNN_E_UNSUPPORTED;
 *   layers   L >= 0;
 *   W        [layers] layer descriptors (may be NULL iff layers == 0);
 *   bias     [layers * neurons] fp32, layer-major (b_l = bias + l*neurons);
 *   out      receives the handle (set to NULL on error).
 * Validates every layer (index range, monotone rowptr, no duplicate (k,j),
 * finite values), packs it into the device layout and
 * uploads it; weights stay resident in HBM for the life of the handle. */
sdnn_status sdnn_create(int32_t neurons, int32_t layers, const sdnn_layer *W,
                        const float *bias, const sdnn_opts *opts, sdnn_net **out);

/* Streamed creation for networks too large to stage on the host at once
 * (65536 x 1920 is 4.0e9 nonzeros): create the handle, then call
 * sdnn_set_layer for every l in [0, layers) (any order; distinct layers may be
 * set from different host threads concurrently).  sdnn_infer* returns
 * SDNN_E_STATE until every layer has been set. */
sdnn_status sdnn_create_empty(int32_t neurons, int32_t layers, const sdnn_opts *opts,
                              sdnn_net **out);
sdnn_status sdnn_set_layer(sdnn_net *net, int32_t l, const sdnn_layer *W_l,
                           const float *bias_l /* [neurons] */);

/* Synchronous inference from HOST buffers (the end-to-end call).
 *   y0_rowptr   [batch+1] int64, y0_rowptr[0] = 0, non-decreasing;
 *   y0_idx      [y0_rowptr[batch]] int32 neuron ids in [0, N), no duplicate per row;
 *   y0_val      same length, finite, or NULL meaning every stored value is 1.0f
 *               (binary challenge-style input);
 *   batch       B >= 0;
 *   categories  [batch] capacity; receives the ascending 0-based category ids;
 *   n_categories receives their count;
 *   y_out       NULL, or [batch * neurons] fp32 row-major: receives Y_L.
 * Host->device copy of Y0, the whole layer chain and the device->host copy of
 * the categories all happen inside this call; the device work runs on
 * opts->stream (or the handle's stream) and is complete on return. */
sdnn_status sdnn_infer(sdnn_net *net, const int64_t *y0_rowptr, const int32_t *y0_idx,
                       const float *y0_val, int64_t batch, int32_t *categories,
                       int64_t *n_categories, float *y_out);

/* Pipelined host-buffer inference (serving): sdnn_infer_submit does what
 * sdnn_infer does up to the device work -- host checks, input copy, densify,
 * layer chain, readout, the copy of the categories into a page-locked result
 * buffer -- and returns once it is enqueued; sdnn_infer_wait(ticket) blocks
 * until that inference is complete and returns its categories (and the status
 * of its host validation).  Up to two submissions may be outstanding on a
 * handle: the input copy of the next one then overlaps the layers of the
 * current one.  The caller's input buffers must stay valid and unchanged until
 * the matching wait returns.  y_out is not available on this path;
 * sdnn_infer returns SDNN_E_STATE while submissions are outstanding.
 *   ticket      receives an id for sdnn_infer_wait (waits in submission order
 *               are not required, but a third submit before a wait returns
 *               SDNN_E_STATE). */
sdnn_status sdnn_infer_submit(sdnn_net *net, const int64_t *y0_rowptr, const int32_t *y0_idx,
                              const float *y0_val, int64_t batch, int64_t *ticket);
sdnn_status sdnn_infer_wait(sdnn_net *net, int64_t ticket, int32_t *categories,
                            int64_t *n_categories);

/* Asynchronous inference from DEVICE buffers on `stream` (cudaStream_t; NULL =
 * legacy default stream).  Same Y0 layout as sdnn_infer, all pointers device
 * pointers; Y0 is NOT validated here.
 *   d_alive   [ceil(batch/32)] uint32 device bitmask: bit (i%32) of word i/32 is
 *             set iff row i is a category (all other bits are cleared);
 *   d_y_out   NULL or [batch * neurons] fp32 device, row-major Y_L.
 * This is the entry point of the torch / NCCL multi-GPU driver: pointers come
 * from tensor.data_ptr(), the stream from torch.cuda.current_stream(). */
sdnn_status sdnn_infer_device(sdnn_net *net, const int64_t *d_rowptr, const int32_t *d_idx,
                              const float *d_val, int64_t batch, uint32_t *d_alive,
                              float *d_y_out, void *stream);

/* Final activations Y_L of SELECTED input rows of the last inference, without
 * materialising the whole [batch x neurons] matrix (15.7 GB at 65536 neurons x
 * 60,000 inputs): the golden-reference check of PAPER.md:2570 on sampled rows.
 *   d_rows  [nrows] int32 DEVICE array of original (0-based) row ids, any
 *           order, repeats allowed; an id outside [0, last batch) yields zeros;
 *   d_y     [nrows * neurons] fp32 DEVICE, row-major: row q receives Y_L of
 *           input row d_rows[q] (all zeros for a row that died or was empty,
 *           all YMAX for a row retired as saturated under SDNN_F_SATURATE).
 * Asynchronous on `stream` (cudaStream_t; NULL = legacy default stream); it
 * must be ordered after the inference it reads (same stream, or after the
 * synchronous sdnn_infer returned) and before the next inference on the
 * handle.  Returns SDNN_E_STATE before the first inference. */
sdnn_status sdnn_gather_rows(sdnn_net *net, const int32_t *d_rows, int64_t nrows, float *d_y,
                             void *stream);

/* f4: sdnn_infer_device with the category readout fused with the
 * cross-GPU gather over NVLink SHARP (NVLS multicast), replacing the separate
 * NCCL all-gather: the readout kernel builds this rank's words in its slice of
 * a symmetric bitmask buffer, writes each word through the buffer's
 * MULTICAST mapping with multimem.st (one store reaches every GPU's copy),
 * adds 1 to a multicast arrival counter (release) and waits until the local
 * copy of the counter reaches `target`.  On return of the enqueued work every
 * GPU's local_words holds the whole global bitmask (decode it with
 * sdnn_bitmask_to_ids).  The buffers come from the caller (e.g. torch
 * symmetric memory with NVLS multicast, paper_2004_10908_b200/dist.py
 * NvlsGather); the ranks' slices are word-aligned (dist.partition).
 *   local_words  unicast VA of this GPU's copy of the global bitmask
 *   mc_words     multicast VA of the same buffer
 *   local_flag / mc_flag  unicast / multicast VA of a uint32 arrival counter that
 *                every rank increments once per call (never reset); local_flag[1]
 *                is set to 1 if a wait gave up after ~4 s (a rank missing: the
 *                result is then invalid, the GPU is not hung)
 *   word_offset  this rank's first word; target = (calls so far) x world size.
 * Reuse of a word buffer must alternate (two buffers by call parity): a rank
 * may start its next call while another still decodes this one.  Needs >= 1
 * layer; not with SDNN_F_SATURATE.  Asynchronous on `stream`. */
typedef struct sdnn_nvls {
  uint32_t *local_words;
  uint32_t *mc_words;
  uint32_t *local_flag;
  uint32_t *mc_flag;
  int64_t word_offset;
  uint32_t target;
} sdnn_nvls;
sdnn_status sdnn_infer_device_nvls(sdnn_net *net, const int64_t *d_rowptr, const int32_t *d_idx,
                                   const float *d_val, int64_t batch, const sdnn_nvls *nv,
                                   void *stream);

/* The arrival/wait of sdnn_infer_device_nvls alone (an NVLS barrier; used to
 * check a multicast mapping once before relying on it): adds 1 through mc_flag,
 * waits until local_flag reaches target (local_flag[1] = 1 on a ~4 s timeout). */
sdnn_status sdnn_nvls_barrier(uint32_t *local_flag, uint32_t *mc_flag, uint32_t target, void *stream);

/* Multi-GPU readout (no handle needed): decode a global category bitmask --
 * e.g. the NCCL all-gather of every rank's d_alive words, rows partitioned in
 * word-aligned contiguous slices (paper_2004_10908_b200/dist.py; the per-GPU
 * cudaFlows of PAPER.md:2566-2569 followed by one gather of the categories,
 * north_star) -- into the ascending 0-based category ids.
 *   d_words  [ceil(batch/32)] uint32 DEVICE: bit i%32 of word i/32 = row i
 *            (bits at and beyond `batch` are ignored);
 *   d_ids    [batch] int32 DEVICE capacity: receives the ascending ids;
 *   d_n      [1] int32 DEVICE: receives their count.
 * Asynchronous on `stream` (cudaStream_t; NULL = legacy default stream). */
sdnn_status sdnn_bitmask_to_ids(const uint32_t *d_words, int64_t batch, int32_t *d_ids,
                                int32_t *d_n, void *stream);

/* f1 launch study (Sec. 4.6.2 "Scheduling GPU
 * Tasks", Algorithm 1): ONE inference of `parts` batch partitions, partition p
 * on its own handle nets[p] (own workspace; weights loaded into each), as one
 * GPU task graph -- per partition: densify -> every kernel of the handle's
 * layer chain -> readout of its categories into the word slice
 * d_words + word_offset of a global bitmask -- joined by the device decode of
 * that bitmask into d_ids / d_n (sdnn_bitmask_to_ids).  Launched as
 *   SDNN_FLOW_GRAPH     an explicit graph of the task DAG (the paper's cudaFlow);
 *   SDNN_FLOW_CAPTURER  Algorithm 1: levelize, stream = (task id in its level) mod
 *                       max_streams, events only on cross-stream edges, captured
 *                       into one CUDA graph and replayed;
 *   SDNN_FLOW_STREAMS   the same stream assignment launched directly (no graph).
 * Runs one warm-up and `reps` timed repetitions; *ms = device time per
 * repetition (CUDA events); *ntasks = tasks in the graph.  Synchronous.
 * Partitions must be word-aligned (word_offset = first row / 32, every batch
 * but the last a multiple of 32).  Handles with stream_slots > 0 or
 * SDNN_F_PROFILE are not supported. */
enum { SDNN_FLOW_GRAPH = 0, SDNN_FLOW_CAPTURER = 1, SDNN_FLOW_STREAMS = 2 };
/* Host-only (no device): Algorithm 1's stream assignment for an arbitrary task
 * DAG -- the same code sdnn_flow_infer runs.  edges: [nedges] (from, to) pairs
 * (int32 x 2); level / id / stream: [ntasks] outputs (NULL allowed): level =
 * topological level (Kahn rounds), id = index inside the level, stream = id mod
 * max_streams; event_edges: [2 * nedges] capacity or NULL, receives the edges
 * that cross streams (the stream_record_event / stream_wait_event pairs) in
 * issue order, *nevents their count.  SDNN_E_FORMAT on a cycle. */
sdnn_status sdnn_flow_plan(int32_t ntasks, int32_t nedges, const int32_t *edges, int32_t max_streams,
                           int32_t *level, int32_t *id, int32_t *stream, int32_t *nevents,
                           int32_t *event_edges);
typedef struct sdnn_flow_part {
  const int64_t *d_rowptr;   /* device CSR of the partition's rows (as sdnn_infer_device) */
  const int32_t *d_idx;
  const float *d_val;        /* NULL => 1.0f */
  int64_t batch;
  int64_t word_offset;       /* first word of the partition in d_words */
} sdnn_flow_part;
sdnn_status sdnn_flow_infer(sdnn_net *const *nets, int32_t parts, const sdnn_flow_part *p,
                            uint32_t *d_words, int64_t total_batch, int32_t *d_ids, int32_t *d_n,
                            int32_t mode, int32_t max_streams, int32_t reps, float *ms,
                            int32_t *ntasks);

/* Statistics of the handle and of its last completed inference. */
typedef struct sdnn_stats {
  int32_t struct_size;        /* caller sets sizeof(sdnn_stats) (versioning)            */
  int32_t neurons, layers;
  int32_t path;               /* bit 0: fused multi-layer passes used; bit 1: the
                                 SMEM-resident kernel runs the last layers; bit 2:
                                 position-blocked activations (every step a fused
                                 pass; SDNN_YBLOCK=0 in the environment disables)     */
  int32_t grouped_layers;     /* layers packed with >1 column per source-list group    */
  int32_t max_group;          /* largest group size (columns sharing a source list)    */
  int32_t max_k;              /* largest column nnz over all layers                    */
  int32_t compaction;         /* 1 if dead-row compaction is enabled                   */
  int64_t packed_weight_bytes;/* device bytes of packed W and bias                     */
  int64_t total_nnz;          /* sum over layers of stored nonzeros                    */
  int64_t last_batch;
  int64_t last_n_categories;
  int64_t launches_per_infer; /* kernels (graph nodes) one inference launches          */
  int64_t live_edges;         /* sum_l (rows nonzero before layer l) * nnz_l, last call */
  int64_t kept_rows;          /* rows entering layer 0 (empty rows dropped when exact)   */
  int32_t steps;              /* kernel steps of the layer chain (fused passes count 1)  */
  int32_t fused_layers;       /* layers executed inside fused multi-layer passes         */
  int32_t resident_layers;    /* layers executed by the SMEM-resident kernel             */
  int64_t retired_rows;       /* SDNN_F_SATURATE: rows retired as saturated categories    */
  int64_t stream_bytes;       /* stream_slots > 0: host->device weight bytes per inference
                                 (0 when every layer is resident)                        */
  int64_t stream_slot_bytes;  /* stream_slots > 0: device bytes of one ring slot            */
  int64_t executed_fma;       /* fp32 FMAs the kernels executed in the last inference:
                                 sum over steps of (batch positions the step computed) x
                                 (per layer: sum_g K_g when the layer's weights are uniform
                                 -- the members of a group share one chain -- else nnz_l).
                                 Compare with the nominal edges inputs x sum_l nnz_l      */
  int64_t computed_rows;      /* sum over layers of the batch positions computed (dead rows
                                 are dropped only at the compactions between steps)      */
} sdnn_stats;

/* live_rows: NULL or [layers] receives the number of rows still nonzero after
 * each layer of the last inference (the survivor profile). */
sdnn_status sdnn_stats_get(const sdnn_net *net, sdnn_stats *out, int64_t *live_rows);

/* SDNN_F_PROFILE only: device duration (ms) of every layer kernel of the last
 * inference, from CUDA events recorded on the launching stream around it.
 * ms: [layers].  Synchronises the handle's work. */
sdnn_status sdnn_layer_times(const sdnn_net *net, float *ms);

/* Host-only validation + packing of one layer (no device needed): the same
 * checks and grouping sdnn_set_layer performs, reported in `info`. */
typedef struct sdnn_layer_info {
  int32_t ngroups;   /* groups of columns with identical ascending source lists */
  int32_t kmax;      /* largest column nnz                                      */
  int32_t gmax;      /* largest group                                           */
  int32_t uniform;   /* 1 if every stored value is bit-identical                */
  int32_t regular;   /* 1 if every group has kmax sources and gmax members      */
  int32_t bias_nonpositive;
  int64_t nnz;
} sdnn_layer_info;
sdnn_status sdnn_validate_layer(int32_t neurons, const sdnn_layer *W_l, const float *bias_l,
                                uint32_t flags, sdnn_layer_info *info);

/* The execution plan of a handle (valid after the first inference): step_len
 * [layers] capacity receives the number of layers of each kernel step. */
sdnn_status sdnn_step_plan(const sdnn_net *net, int32_t *step_len, int32_t *nsteps);

/* Host-only (no device): the fused-pass plan sdnn_create would use for these
 * layers, before the SMEM-resident tail (N <= 4096) replaces the last ones --
 * step_len[i] = number of layers of step i (1 = one kernel per layer, > 1 = a
 * fused multi-layer pass, see sdnn_opts.fuse_rows); *nsteps = number of
 * steps.  step_len: [layers] capacity. */
sdnn_status sdnn_plan_steps(int32_t neurons, int32_t layers, const sdnn_layer *W,
                            const float *bias, const sdnn_opts *opts, int32_t *step_len,
                            int32_t *nsteps);

void sdnn_destroy(sdnn_net *net);          /* NULL-safe; frees all device memory       */
const char *sdnn_last_error(void);         /* thread-local, never NULL                 */
int32_t sdnn_abi_version(void);            /* == SDNN_ABI_VERSION                      */

#ifdef __cplusplus
}
#endif
#endif /* SDNN_H */
