/*
 * ll.h -- C ABI of the B200-native label-looping greedy Transducer decoder.
 *
 * Method: batched label-looping greedy decoding for RNN-T and TDT models,
 * arXiv 2406.06220 (the paper's text is PAPER.md; citations are PAPER.md line
 * numbers).  The outer loop runs over labels, the inner loop over frames:
 * Alg. 3 "Label-looping Algorithm", TDT variant
 * (PAPER.md:211-213), precomputed projections, batched
 * hypotheses.  The problem statement follows Alg. 3 line 1
 * (PAPER.md:133): "acoustic input x_1..x_B, input_length".
 *
 * Conventions (all entry points):
 *  - Tensor pointers are DEVICE pointers unless marked HOST, row-major,
 *    contiguous, caller-owned (e.g. allocated with PyTorch).  The library
 *    allocates nothing on the decode path; all scratch lives in the caller's
 *    `workspace`.
 *  - Calls are stream-ordered and asynchronous: they enqueue work on `stream`
 *    and return.  Weights, inputs, outputs and workspace must stay valid until
 *    that work completes.  Calls on different streams with distinct
 *    workspaces are independent.
 *  - Host-side validation errors are returned synchronously and nothing is
 *    enqueued.  Errors found on the device (a length > T_max, a hypothesis
 *    overflowing `out_capacity`) are returned by ll_sync().
 *  - No C++ exception crosses this boundary.
 *  - There is no CPU fallback: every step of decoding runs in the library's
 *    CUDA kernels for sm_100a.
 */
#ifndef LL_H_
#define LL_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t ll_status;
enum {
  LL_OK = 0,
  LL_ERR_INVALID_ARGUMENT = 1, /* null pointer, negative size, bad id, inconsistent dims */
  LL_ERR_UNSUPPORTED = 2,      /* valid but not implemented (dims not multiple of 16, ...) */
  LL_ERR_WORKSPACE = 3,        /* workspace_bytes < ll_workspace_size(...) */
  LL_ERR_CUDA = 4,             /* a CUDA launch / runtime call failed */
  LL_ERR_CAPACITY = 5          /* (ll_sync) a hypothesis exceeded out_capacity */
};

/* Element type of `enc` and of every weight and bias tensor. */
typedef enum { LL_BF16 = 0, LL_F32 = 1 } ll_dtype;

/* LL_PREC_FAST: bf16 tensor-core contractions with fp32 accumulation; the
 * projected encoder rows f, the recurrent operand h and the joint operand z are
 * rounded to bf16.  (LL_F32 inputs are always computed in fp32.)
 * LL_PREC_EXACT with LL_BF16 inputs: the call computes the SAME model in fp32
 * (f, g, h, c, z never rounded to bf16; the fp32 tolerance class of north_star,
 * 1e-5 on the logits): fp32 copies of the bf16 values (exact: every bf16 value
 * is an fp32 value) are made behind the fp32 call's workspace and the fp32
 * kernels run on them; ll_workspace_size includes the copies (weights + the
 * encoder output); slower than FAST; model tables are rebuilt on every call
 * (ll_prepare records nothing).  LL_PREC_EXACT with LL_F32 inputs = LL_PREC_FAST.
 * Not combinable with ll_options.projections = 1 or the probe
 * (LL_ERR_UNSUPPORTED). */
typedef enum { LL_PREC_FAST = 0, LL_PREC_EXACT = 1 } ll_prec;

typedef enum { LL_PRED_LSTM = 0, LL_PRED_STATELESS = 1 } ll_pred_kind;

/* An opaque CUDA stream (binary-compatible with cudaStream_t; NULL = legacy default stream). */
typedef struct CUstream_st *ll_stream;

/*
 * Prediction network (Fig. 1; "stateful (LSTM) and stateless", :33).
 *  LSTM (PyTorch nn.LSTM convention, gate rows i,f,g,o; layer 1 shown, more below):
 *    x = embedding[y];  gates = w_ih x + b_ih + w_hh h + b_hh
 *    c' = sigmoid(f) c + sigmoid(i) tanh(g);  h' = sigmoid(o) tanh(c');  dec = h'
 *    embedding [num_tokens, hidden], w_ih/w_hh [4*hidden, hidden], b_ih/b_hh [4*hidden].
 *  Stateless: dec = concat_k embedding[k][y_{-1-k}], k < context,
 *    embedding [context][num_tokens][hidden/context]; w_ih..b_hh unused (may be NULL).
 *  Initial state: h = c = 0, context = [blank]*context.  The first predictor
 *  input (SOS / "BOS") is the blank id, i.e. embedding row blank_id.
 */
typedef struct {
  int32_t kind;        /* ll_pred_kind */
  int32_t num_tokens;  /* V+1 (blank included); must equal ll_joint.num_outputs */
  int32_t hidden;      /* P; must equal ll_joint.pred_dim */
  int32_t context;     /* stateless only: 1..4, hidden % context == 0 */
  const void *embedding;
  const void *w_ih, *w_hh, *b_ih, *b_hh;
  /* LSTM layers 2..num_layers ("more layers"; PyTorch nn.LSTM
   * stacking: layer l's input is the NEW h of layer l-1, dec = h of the last
   * layer).  num_layers 0 or 1: one layer, the fields below unused.  Stacked
   * [num_layers-1, 4*hidden, hidden] (w_*_rest) and [num_layers-1, 4*hidden]
   * (b_*_rest).  Computed by the fp32 generic kernel (every layer's weights
   * read through L2); LL_BF16 weights with num_layers > 1 are widened to fp32
   * as under LL_PREC_EXACT (the bf16 FC kernel keeps ONE layer's W_hh in TMEM). */
  int32_t num_layers;
  const void *w_ih_rest, *w_hh_rest, *b_ih_rest, *b_hh_rest;
} ll_predictor;

/*
 * Joint network with its two projections (§3.4):
 *   f[t] = w_enc enc[t] + b_enc           [H]   (precomputed once per call, Alg. 3 line 2)
 *   g    = w_pred dec + b_pred            [H]   (once per predictor call, Alg. 3 line 6)
 *   z    = ReLU(f[t] + g)
 *   logits     = w_out z + b_out          [V+1] (Alg. 3 lines 7, 13)
 *   dur_logits = w_dur z + b_dur          [|D|] (TDT only)
 * w_enc [H, D_e], b_enc [H], w_pred [H, P], b_pred [H], w_out [V+1, H], b_out [V+1],
 * w_dur [|D|, H], b_dur [|D|] (NULL for RNN-T).
 */
typedef struct {
  int32_t enc_dim, pred_dim, joint_dim, num_outputs; /* D_e, P, H, V+1 */
  const void *w_enc, *b_enc, *w_pred, *b_pred;
  const void *w_out, *b_out;
  const void *w_dur, *b_dur;
} ll_joint;

/* Bytes of device workspace needed by a decode (or ll_debug_joint) call with
 * these shapes.  num_durations = 0 for RNN-T.  Returns 0 if the arguments are
 * invalid. */
size_t ll_workspace_size(int32_t B, int32_t T_max, const ll_predictor *pred, const ll_joint *joint,
                         ll_dtype dtype, ll_prec prec, int32_t num_durations);

/*
 * Greedy RNN-T decoding of B utterances by label looping (Alg. 3).
 *  enc          [B, T_max, D_e] encoder outputs (frames t >= lengths[b] are never read)
 *  lengths      [B] int32, 0 <= lengths[b] <= T_max (checked on the device -> ll_sync)
 *  blank_id     in [0, V]; also the SOS input of the predictor
 *  max_symbols  >= 1: after max_symbols labels at one frame, decoding moves to the
 *               next frame without evaluating a blank (termination guard)
 *  out_tokens, out_timestamps  [B, out_capacity] int32: label ids and the frame index
 *               each label was emitted at; entries >= out_lengths[b] are untouched
 *  out_lengths  [B] int32: number of labels of each hypothesis (true count, even if it
 *               exceeded out_capacity -- then ll_sync returns LL_ERR_CAPACITY and only
 *               the first out_capacity labels are written).  out_capacity >=
 *               T_max*max_symbols can never overflow.
 *  workspace    >= ll_workspace_size(...) bytes, 256-byte aligned.
 * Results are identical to per-utterance greedy decoding (Alg. 1)
 * up to floating-point near-ties of the joint logits.
 */
ll_status ll_decode_rnnt(const void *enc, ll_dtype dtype, ll_prec prec, int32_t B, int32_t T_max,
                         const int32_t *lengths, const ll_predictor *pred, const ll_joint *joint,
                         int32_t blank_id, int32_t max_symbols,
                         int32_t *out_tokens, int32_t *out_timestamps, int32_t *out_lengths,
                         int32_t out_capacity, void *workspace, size_t workspace_bytes,
                         ll_stream stream);

/*
 * Greedy TDT decoding.  As ll_decode_rnnt, plus:
 *  durations      HOST int32 [num_durations], each >= 0, 1 <= num_durations <= 16: the
 *                 duration set D; dur_logits index i means "advance by durations[i]".
 *  out_durations  [B, out_capacity] int32 or NULL: predicted duration of each label.
 * Time rule: blank -> t += max(d, 1); label -> append (timestamp = t), then
 * d > 0 ? t += d : (count toward max_symbols at frame t).
 */
ll_status ll_decode_tdt(const void *enc, ll_dtype dtype, ll_prec prec, int32_t B, int32_t T_max,
                        const int32_t *lengths, const ll_predictor *pred, const ll_joint *joint,
                        int32_t blank_id, int32_t max_symbols,
                        const int32_t *durations, int32_t num_durations,
                        int32_t *out_tokens, int32_t *out_timestamps, int32_t *out_durations,
                        int32_t *out_lengths, int32_t out_capacity,
                        void *workspace, size_t workspace_bytes, ll_stream stream);

/*
 * Greedy decoding with scores (BatchedHyps keeps "tokens,
 * time-stamps, scores").  As ll_decode_rnnt / ll_decode_tdt, plus
 *  out_scores  [B] f32 (DEVICE, non-NULL when B > 0): the greedy score of each
 *              hypothesis = the sum over EVERY decision the method takes (blanks
 *              included, reading A19 after SPEC.md:239, :266) of the decision's
 *              log-probability log softmax(logits)[y]; for TDT plus the duration
 *              log-probability log softmax(dur_logits)[d] (the pair's joint
 *              log-probability, reading A26).
 * The log-sum-exp over the V+1 (and |D|) logits is fused into the joint
 * epilogue and combined across the cluster with the argmax keys; logits never
 * reach HBM.  Hypotheses are identical to the calls without scores.  Per-row
 * tick schedule only (ll_options.schedule = 0 returns LL_ERR_UNSUPPORTED).
 */
ll_status ll_decode_rnnt_scores(const void *enc, ll_dtype dtype, ll_prec prec, int32_t B, int32_t T_max,
                                const int32_t *lengths, const ll_predictor *pred, const ll_joint *joint,
                                int32_t blank_id, int32_t max_symbols,
                                int32_t *out_tokens, int32_t *out_timestamps, int32_t *out_lengths,
                                int32_t out_capacity, float *out_scores,
                                void *workspace, size_t workspace_bytes, ll_stream stream);
ll_status ll_decode_tdt_scores(const void *enc, ll_dtype dtype, ll_prec prec, int32_t B, int32_t T_max,
                               const int32_t *lengths, const ll_predictor *pred, const ll_joint *joint,
                               int32_t blank_id, int32_t max_symbols,
                               const int32_t *durations, int32_t num_durations,
                               int32_t *out_tokens, int32_t *out_timestamps, int32_t *out_durations,
                               int32_t *out_lengths, int32_t out_capacity, float *out_scores,
                               void *workspace, size_t workspace_bytes, ll_stream stream);

/*
 * Frame-looping BASELINE (Alg. 2, "Batched Inference of Transducer",
 * PAPER.md:84-115) on the same kernels, for the paper's label- vs frame-looping
 * comparison.  Same arguments, ownership, errors and
 * results as ll_decode_rnnt (the hypotheses are identical: both reach the
 * greedy result of Alg. 1).  Control flow: all rows advance through frames in
 * lockstep (line 22); at frame t the joint is evaluated for the rows not yet
 * done with t, rows that emit a label get a predictor update and are evaluated
 * again at t (lines 11-20) until they emit a blank or hit max_symbols.  Unlike
 * the paper's listing, the predictor output of rows whose state did not change is
 * reused, not recomputed (a stronger baseline).  RNN-T only.
 */
ll_status ll_decode_rnnt_frame_looping(const void *enc, ll_dtype dtype, ll_prec prec, int32_t B, int32_t T_max,
                                       const int32_t *lengths, const ll_predictor *pred, const ll_joint *joint,
                                       int32_t blank_id, int32_t max_symbols,
                                       int32_t *out_tokens, int32_t *out_timestamps, int32_t *out_lengths,
                                       int32_t out_capacity, void *workspace, size_t workspace_bytes,
                                       ll_stream stream);

/*
 * Weight-only preprocessing, once per model and workspace: builds the model
 * tables of a decode call (LSTM: E' = Emb W_ih^T + b_ih + b_hh and the packed
 * W_hh / W_pred tile stream; stateless: G_k = W_pred[:, k] Emb_k) into
 * `workspace` and records their fingerprint (weight pointers, shapes, dtype,
 * cluster layout, workspace size) for that workspace (the tables sit at batch-independent
 * offsets, so decodes of any B <= the workspace's B reuse them).  A later ll_decode_* on the
 * same workspace whose fingerprint matches skips rebuilding them; any other
 * decode on the workspace rebuilds them and drops the record.  Call it again
 * after modifying weights IN PLACE (the fingerprint holds pointers, not
 * contents), and ll_release() the workspace before freeing it or the weights.
 * Arguments as ll_decode_*: durations is HOST [num_durations] for
 * TDT, NULL for RNN-T; B / T_max are the batch shape the workspace was sized
 * for.  Stream-ordered; host validation errors return synchronously.
 */
ll_status ll_prepare(const ll_predictor *pred, const ll_joint *joint, ll_dtype dtype, ll_prec prec,
                     int32_t B, int32_t T_max, const int32_t *durations, int32_t num_durations,
                     void *workspace, size_t workspace_bytes, ll_stream stream);

/* Waits for the work enqueued on `stream` and returns the device-side status of
 * the last decode that used `workspace`: LL_OK, LL_ERR_INVALID_ARGUMENT (some
 * lengths[b] > T_max; that row decodes as empty), LL_ERR_CAPACITY, or
 * LL_ERR_CUDA. */
ll_status ll_sync(void *workspace, ll_stream stream);

/* Static description of a status code (never NULL). */
const char *ll_status_string(ll_status status);

/* Decode statistics of the last call that used `workspace`, copied to HOST
 * `out[13]` after synchronising `stream`: [0] outer steps (label-loop
 * iterations, summed over groups), [1] joint rounds (W-frame windows),
 * [2] joint evaluations whose decision was used (the algorithmic count of
 * Alg. 1), [3] batched predictor steps, [4] predictor row evaluations,
 * [5] labels emitted, [6] groups decoded, [7] cluster size, [8] joint rows
 * computed (including speculative window frames), [9] window W, [10] rows
 * per group R, [11] the longest per-cluster chain, packed (rounds + steps) << 40
 * | joint rounds << 20 | predictor steps of that cluster (each field saturates
 * at 2^20 - 1): the critical path of the launch (bench.py's chain floor),
 * [12] kernels the call launched (projection GEMM, model tables if rebuilt,
 * length ranking, widening, the decode kernel). */
ll_status ll_stats(const void *workspace, uint64_t *out, ll_stream stream);

/*
 * Test/debug: the joint of the decode kernel on n given rows, with the
 * encoder projection of Alg. 3 line 2 applied first:
 *   f_i = w_enc enc_rows[i] + b_enc;  logits_i = w_out ReLU(f_i + g_rows[i]) + b_out
 *  enc_rows        [n, D_e] (dtype);  g_rows [n, H] fp32 (predictor projection outputs)
 *  out_logits      [n, V+1+num_durations] fp32 or NULL (token logits then duration logits)
 *  out_argmax      [n] int32 (lowest index among ties)
 *  out_dur_argmax  [n] int32 or NULL (TDT)
 * Runs the generic cluster kernel's joint (register-resident weight slices,
 * mma.sync, fused argmax, cross-CTA reduction: the path of every shape other
 * than the FastConformer one).  The production FastConformer kernels (tcgen05
 * joint, background recurrent GEMM) are checked through ll_options.probe_*,
 * which makes the decode kernel itself write its logits and g.
 */
ll_status ll_debug_joint(const void *enc_rows, const float *g_rows, int32_t n, const ll_joint *joint,
                         ll_dtype dtype, ll_prec prec, int32_t num_durations,
                         float *out_logits, int32_t *out_argmax, int32_t *out_dur_argmax,
                         void *workspace, size_t workspace_bytes, ll_stream stream);

/* Test/debug: CUDA events (cudaEvent_t handles created by the caller) that the
 * following decode calls made from this host thread record on their stream
 * immediately before and after the persistent decode kernel, so a caller can
 * time that kernel alone with CUDA events.  Pass NULL, NULL to disable. */
ll_status ll_set_timing_events(void *ev_before_decode, void *ev_after_decode);

/* Library version string. */
const char *ll_version(void);

/*
 * Drops the record ll_prepare() keeps for `workspace` (its model tables are
 * rebuilt by the next decode on it).  Call it before freeing or reusing a
 * workspace's memory: the record is keyed by the workspace address and the
 * weight pointers, and a caching allocator can hand the same addresses to
 * other weights.  Unknown or NULL workspaces are a no-op.  Host-only, no
 * stream work.  (ll_debug_joint drops the record of the workspace it uses.)
 */
ll_status ll_release(void *workspace);

/*
 * Test / debug options of the decode calls made AFTERWARDS FROM THIS HOST
 * THREAD (thread-local; ll_set_options(NULL) restores the defaults).  The
 * production path reads no environment variable: every knob that changes the
 * kernel path is here, explicit.  Zero / -1 fields mean "library default".
 *
 *  cluster_size, group_rows, window   force the cluster size C (2..16), rows
 *                 per group R (1..32) and multi-frame window W (1..8; R*W <= 32)
 *                 instead of the occupancy-based choice.
 *  max_clusters   cap on concurrently resident clusters (0: all).
 *  schedule       -1 default (per-row ticks), 0 the batched outer loop of
 *                 Alg. 3 as listed, 1 per-row ticks.
 *  spec_prefetch  -1 default (on), 0 off, 1 on: speculative next-window copies.
 *  group_plan     -1 default (on), 0 off, 1 on: which utterances share a group
 *                 (hypotheses are the same either way).  On:
 *                 one-wave decodes of the FastConformer shape (B <= 32, RNN-T and
 *                 TDT, tick schedule, no scores / probe) use length-sorted
 *                 unequal groups (the groups with a spare slot hold the longest
 *                 utterances and take a wider window); every other decode with
 *                 more than one group ranks the utterances by length on the
 *                 device (one small kernel) and groups consecutive ranks, so a
 *                 group's rows have similar lengths and the longest groups run
 *                 first.  Off: groups of consecutive utterances.
 *  gemm_mma_sync  1: encoder projection on the mma.sync GEMM instead of tcgen05.
 *  timeline       DEVICE u64 buffer for the per-warp timeline (libll_timeline
 *                 builds only; ignored by libll.so).
 *  trace          host-mapped u32 progress markers (libll_trace builds only).
 *
 *  Probe (parity tests of the production FastConformer instantiations, H = P
 *  = 640 in 16-CTA clusters, per-row tick schedule; other shapes return
 *  LL_ERR_UNSUPPORTED while a probe is set).  The SAME decode kernel code is
 *  instantiated with a probe hook that also writes, per cluster region
 *  r < probe_regions (at most probe_regions clusters run):
 *    probe_logits  DEVICE f32 [probe_regions][probe_rows][V+1+|D|]: the logits
 *                  (token then duration) of every joint row the kernel evaluated
 *    probe_lmeta   DEVICE i32 [probe_regions][probe_rows][4]: (utterance b,
 *                  frame t, labels emitted by b before this evaluation, 0)
 *    probe_g       DEVICE f32 [probe_regions][probe_rows][H]: the predictor
 *                  output g = W_pred dec + b_pred after every predictor step
 *    probe_gmeta   DEVICE i32 [probe_regions][probe_rows][4]: (b, labels the
 *                  predictor has consumed = hypothesis length, 0, 0)
 *    probe_counts  DEVICE i32 [probe_regions][2]: logit rows, g rows written
 *                  (values > probe_rows mean the region was truncated)
 *    probe_stall   cycles that the odd ranks of every cluster spin before each
 *                  group's initialisation (test hook: skews the CTAs of a cluster
 *                  at group starts, to stress the cross-CTA exchanges); 0 = off
 *  Set probe_logits = NULL to disable the probe.
 *
 *  projections    0 (default): the joint's input projections are precomputed
 *                 (encoder: one GEMM over all frames before the decode, Alg. 3
 *                 line 2; predictor: once per predictor step, line 6 --
 *                 PAPER.md §3.4 :216-222).  1: ON THE FLY -- the ablation arm of
 *                 the paper's Table 3: the decode kernel reads
 *                 the encoder rows themselves and applies W_enc and W_pred (+ both
 *                 biases) at every joint evaluation; no f is stored.  Supported
 *                 for bf16, 1-layer LSTM predictors of the FastConformer shape
 *                 (H = P = 640), D_e a multiple of 32 and <= 1024, the per-row
 *                 tick schedule, no scores / probe, RNN-T and TDT (label-looping);
 *                 anything else returns LL_ERR_UNSUPPORTED.  Same hypotheses up
 *                 to near-ties (f is not rounded to bf16 on this path).
 */
typedef struct {
  int32_t cluster_size, group_rows, window, max_clusters;
  int32_t schedule, spec_prefetch, gemm_mma_sync;
  void *timeline;
  void *trace;
  float *probe_logits;
  int32_t *probe_lmeta;
  float *probe_g;
  int32_t *probe_gmeta;
  int32_t *probe_counts;
  int32_t probe_rows, probe_regions;
  int32_t projections;
  int32_t probe_stall;
  int32_t group_plan;
} ll_options;

ll_status ll_set_options(const ll_options *options);

/*
 * Multi-GPU: gathering the ragged hypotheses (SURVEY.md §8(b) ll_gather_ragged;
 * north_star "NCCL is used only to gather the ragged results").  Utterances are
 * independent (Alg. 1 decodes each on its own), so ranks decode
 * disjoint shards with no data-path collective; this is the one exchange.
 *
 * NCCL is resolved at run time (dlopen of libnccl.so.2, preferring the copy the
 * process already loaded, e.g. PyTorch's); without it these calls return
 * LL_ERR_UNSUPPORTED.  A communicator is an opaque handle (ncclComm_t).
 *
 * ll_nccl_unique_id: writes the 128-byte NCCL unique id to HOST `id_out`; call
 *   on one rank and share the bytes with all ranks (e.g. torch.distributed).
 * ll_nccl_comm_init: collective over `nranks` processes, one GPU each (the
 *   current CUDA device); *comm_out receives the handle.
 * ll_nccl_comm_destroy: frees a handle (NULL is a no-op).
 */
ll_status ll_nccl_unique_id(void *id_out);
ll_status ll_nccl_comm_init(void **comm_out, int32_t nranks, const void *id, int32_t rank);
ll_status ll_nccl_comm_destroy(void *comm);

/* Device workspace (bytes) ll_gather_ragged needs for B rows of out_capacity. */
size_t ll_gather_workspace_size(int32_t B, int32_t out_capacity, int32_t with_durations);

/*
 * ll_gather_ragged: collective over the communicator.  Each rank packs its B
 * decoded rows (the outputs of one or more ll_decode_* calls, concatenated by
 * the caller) into one int32 record on the device
 *     [n, ids[n], lens[n], tokens(ragged), timestamps(ragged)(, durations(ragged))]
 * with lens[i] = min(lengths[i], out_capacity) and the ragged fields the first
 * lens[i] entries of each row, in row order; the records of all ranks are then
 * concatenated in rank order into `root_buf` on rank `root` (ncclAllGather of
 * the record sizes, then ncclSend / ncclRecv of the records).
 *   utt_ids      DEVICE int32 [B]: global utterance id of each row
 *   lengths      DEVICE int32 [B]: the decoders' out_lengths
 *   tokens, timestamps  DEVICE int32 [B, out_capacity];  durations likewise or NULL
 *   root_buf     DEVICE int32 [root_capacity] on root (ignored elsewhere)
 *   root_capacity  elements of root_buf; every rank passes the same value
 *   root_used    HOST int64 out (every rank): elements written on root
 *   workspace    DEVICE, >= ll_gather_workspace_size(B, out_capacity, durations != NULL)
 * Synchronises `stream` once (the record sizes are needed on the host to post
 * the receives).  Returns LL_ERR_CAPACITY on every rank, with nothing
 * written and *root_used = the elements needed, when the records do not fit
 * root_capacity (so every rank can retry with a larger root buffer); LL_ERR_INVALID_ARGUMENT
 * for NULL pointers or B < 0; LL_ERR_CUDA for CUDA or NCCL failures.  B = 0
 * contributes the record [0].
 */
ll_status ll_gather_ragged(void *comm, int32_t root, int32_t B, const int32_t *utt_ids, const int32_t *lengths,
                           const int32_t *tokens, const int32_t *timestamps, const int32_t *durations,
                           int32_t out_capacity, int32_t *root_buf, int64_t root_capacity, int64_t *root_used,
                           void *workspace, size_t workspace_bytes, ll_stream stream);

#ifdef __cplusplus
}
#endif
#endif /* LL_H_ */
