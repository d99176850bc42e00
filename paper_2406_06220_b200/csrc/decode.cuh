// decode.cuh -- persistent thread-block-cluster kernel for batched label-looping
// greedy decoding of RNN-T and TDT (arXiv 2406.06220, Alg. 3 PAPER.md:129-159,
// TDT PAPER.md:211-213).
//
// One cluster of C CTAs decodes one GROUP of up to R utterances at a time
// (groups come from a device work counter; a batch is split into groups
// because utterances are independent -- batch composition does not change
// any hypothesis).  Inside a group the control loop of Alg. 3
// runs entirely on the device:
//
//   outer step (label loop, Alg. 3 line 5):
//     predictor phase (Alg. 3 line 6) for rows that found a label and are still
//       active.  FastConformer shape (TG, see TG_* below): gates = E'[y] + W_hh h
//       where W_hh h was computed in the BACKGROUND on tcgen05 (A = this CTA's
//       W_hh slice, resident in TMEM) as soon as h was known -- it does not
//       depend on the label; the cell update reads it back from TMEM.  h' and
//       g = W_pred h' + b_pred (W_pred in registers, mma.sync, K split over the
//       warps) slices are exchanged between the CTAs with st.async + mbarriers
//       (no global memory, no cluster barrier).  Other shapes: the gate GEMM on
//       mma.sync with W_hh read from TMEM (tcgen05.ld), or fp32 SIMT with the
//       weights read through L2 (any number of LSTM layers).  Stateless:
//       g = sum_k G_k[ctx_k] (precomputed tables).
//     scan (frame loop, Alg. 3 lines 7-19) in ROUNDS.  While a row scans, its
//       predictor output g is fixed, so the joint at frames t..t+W-1 does not
//       depend on the blank decisions between them: a round evaluates a W-frame
//       window of every scanning row at once and then applies the decisions in
//       frame order (first non-blank wins; TDT follows the duration chain).
//       This is an exact reordering of the inner loop.
//       Per round (FastConformer shape, TJ, see TJ_* below):
//         z = ReLU(f[b, t..t+W-1] + g_b)            (bf16, the swizzled B operand)
//         joint GEMM on tcgen05: this CTA's 64 vocabulary rows K-folded into an
//           M = 128 A operand (shared memory), z rows as N, D' in TMEM; the
//           extra rows (1024..): <= 2 held by every CTA and evaluated on CUDA
//           cores for its own joint rows during the MMAs, else spread over the
//           CTAs on mma.sync after them
//         argmax fused in the TMEM epilogue (packed 64-bit keys, butterfly),
//         per-CTA partial keys st.async'ed to every CTA of the cluster,
//         mbarrier completion, every CTA reduces the C partials and applies the
//         same rules -> replicated row state.
//       (Other shapes: the joint weight slice in registers, mma.sync.)
//       f windows arrive by tensor / bulk copies; the next window is prefetched
//       speculatively (assuming the row keeps scanning).
//     append + time rules + guard (BatchedHyps add_results):
//       masked append into the caller's preallocated [B, cap] buffers, one lane
//       per row (each row has one owner, no atomics).
//
// Warps: 10 consumer warps run the control loop; in the TJ instantiations an
// 11th "MMA warp" sleeps on an mbarrier and executes the commands consumer
// thread 0 posts (tcgen05 gate batches, the joint MMAs, the f window copies).
#pragma once
#include <cuda.h>
#include "common.cuh"

namespace ll {

constexpr int MAX_R = 32;        // rows per group (<= 32: one lane per row)
constexpr int MAX_JR = 32;       // joint rows per round R*W (<= 32: one lane per joint row)
constexpr int MAX_DUR = 16;
constexpr int MAX_CTX = 4;
constexpr int MAX_LAYERS = 8;    // LSTM predictor layers (fp32 generic kernel)
enum { SC_OUTER, SC_ROUNDS, SC_ALGEVALS, SC_PRED, SC_PREDROWS, SC_LABELS, SC_GROUPS, SC_ROWEVALS, SC_N };
constexpr int MAX_NW = 10;       // warps per CTA (320 threads; 168 registers per thread at most)
constexpr int MAX_C = 16;        // cluster size
constexpr int KREG = 20;         // 32-wide K blocks of the joint weight slice held in registers (H <= 656)
constexpr int KREG_SMALL = 4;    // small-H instantiation (H <= 144): no register budget lost to padding
constexpr int TL_N = 128;        // timeline: rounds / predictor steps recorded
constexpr int TL_PH = 16;        // timeline: phase slots per event

// mbarrier indices
enum {
  BAR_F = 0,        // [2] f-row bulk copies into fbuf[0/1]
  BAR_X = 2,        // [2] partial keys arriving (st.async) in part[0/1]
  BAR_GRP = 4,      // [2] group index broadcast
  BAR_ACK = 6,      // [2] (rank 0) acknowledgements of the group index
  BAR_H = 8,        // h' slices arriving
  BAR_G = 9,        // g slices arriving
  BAR_FULL = 10,    // W_pred tiles landed (generic bf16 LSTM, kernel start)
  BAR_E = 11,       // E' slices of the predictor rows landed
  BAR_GQ = 12,      // (TJ) MMA warp: a command was posted (consumer thread 0 arrives)
  BAR_GATE = 13,    // (TG) gate batch complete (tcgen05.commit)
  BAR_MACK = 14,    // (TJ) MMA warp: command read (the command word may be reused)
  BAR_JOINT = 15,   // (TJ) joint MMAs complete (tcgen05.commit)
  BAR_SPEC = 16,    // (TJ) MMA warp: speculative copies issued, fbase / fcnt written
  BAR_Z = 17,       // (OTF) z slices of the other CTAs arriving (st.async)
  NBARS = 18
};
enum { MCMD_GATES = 1, MCMD_JOINT = 2, MCMD_EXIT = 3, MCMD_FLOAD = 4 };

// ---------------------------------------------------------------------------
// TG: the FC LSTM instantiation (P = 640 in 16-CTA clusters: 40 units = 160
// gate rows per CTA) computes the recurrent pre-activations W_hh h on the
// 5th-generation tensor cores, in the BACKGROUND: W_hh h does not depend on
// the next label (only E'[y] does, Alg. 3 line 6), so as soon as a predictor
// step has produced h' a dedicated MMA warp issues tcgen05.mma (A = W_hh
// resident in TMEM, B = h' in shared memory) for every slot of the group, and
// the next predictor step only reads the result back.
//   TMEM columns [0, 320):   gate rows 0..127 (units 0..31, row = 4 unit + gate),
//                            lane = row, column j = K elements 2j, 2j+1
//   TMEM columns [320, 400): gate rows 128..159 (units 32..39) K-folded: lanes
//                            32j + r hold row 128 + r over K [160j, 160j + 160)
//   TMEM columns [400, 408): D main  (M=128, N=8 slots)
//   TMEM columns [408, 440): D fold  (M=128, N=32 = 4 K-quarters x 8 slots; the
//                            diagonal blocks are the 4 partial sums)
// h lives in shared memory as the MMA's B operand, K-major without swizzle:
// 8-row x 16-byte core matrices 144 bytes apart (128 + 16 of padding, so the
// mma.sync W_pred step's 16-byte loads of 4 consecutive chunks hit different
// banks), element (slot n, k) at (k / 8) * 144 + n * 16 + (k % 8) * 2:
// the main MMA reads it with LBO = 144 (next 8 K) and the fold MMA reads the
// same bytes as a 32-row operand (row 8j + n = slot n's K-quarter j, SBO = 2880).
// ---------------------------------------------------------------------------
constexpr int TG_P = 640, TG_C = 16, TG_UPC = TG_P / TG_C;   // 40 units per CTA
constexpr int TG_NH = 8;                                       // slots (B rows): R <= 8
constexpr int TG_CM = 144;                                     // h: core-matrix (8 rows x 16 B) stride, padded
constexpr int TG_QB = (TG_P / 4 / 8) * TG_CM;                  // bytes per K-quarter of h (2880)
constexpr int TG_HBYTES = 4 * TG_QB;                           // h buffer (11520)
constexpr uint32_t TG_COL_FOLD = TG_P / 2, TG_COL_DMAIN = TG_P / 2 + TG_P / 8, TG_COL_DFOLD = TG_COL_DMAIN + TG_NH;
__host__ __device__ inline bool tg_shape(bool bf, bool lstm, int H, int P, int C) {
  return bf && lstm && H == TG_P && P == TG_P && C == TG_C;
}

// ---------------------------------------------------------------------------
// TJ: the FC joint (H = 640 in 16-CTA clusters, LSTM or stateless) on tcgen05.
// Each CTA owns 64 vocabulary rows (8 n8 tiles) on the tensor core plus the
// extra rows (1024.. when V+1+|D| > 1024; see joint_keys_tj).  The
// 64 x 640 weight slice is the A operand in shared memory, K-folded into
// M = 128: A row r = 32 (v / 16) + 16 a + v % 16 holds vocabulary row v's
// K-half a (320 elements); the z rows are the B operand with both K-halves
// stacked along N (B row 32 a + k = joint row k's K-half a), so ONE 20-MMA
// chain (M = 128, N = 64, K = 320) replaces a 40-MMA one: tcgen05.mma is
// issue-bound at ~48 cycles per instruction for these small N
// (tools/tc_probe2.cu), so the fold halves the joint's tensor-core time.  The
// accumulator D'[r][32 a' + k] is useful where a' = a; TMEM lane quarter q
// holds both halves of vocabulary rows 16q .. 16q + 15.
//   A: K-major, no swizzle: row r, 16-byte chunk c (K' 8c .. 8c+7) at
//      (r / 8) * 5120 + c * 128 + (r % 8) * 16                      (80 KB)
//   z: K-major, 128-byte swizzle (1024-byte aligned): row k, 16-byte chunk c
//      of 80 (half a = c / 40, 64-element block kb = (c % 40) / 8, j = c % 8) at
//      kb * 8192 + a * 4096 + (k / 8) * 1024 + (k % 8) * 128 + ((j ^ (k % 8)) * 16)
//      so B row 32 a + k sits in 8-row group 4 a + k / 8 (SBO = 1024) and a
//      warp storing 32 consecutive chunks of one row is bank-conflict free (40 KB)
//   f rows in shared memory with a 1296-byte stride (bank-conflict-free
//   8-row x 16-byte reads in build_z), one bulk copy per frame.
//   TMEM columns [440, 504): D' (after the TG gate columns).
// ---------------------------------------------------------------------------
constexpr int TJ_H = 640, TJ_C = 16;
constexpr int TJ_FROW = TJ_H * 2 + 16;          // f row stride in shared memory (bytes)
constexpr int TJ_GRP = (TJ_H / 2 / 8) * 128;    // bytes per 8-row group of one K-half (5120)
constexpr int TJ_ZHALF = 4 * TJ_GRP;            // z: one K-half of 32 rows (20480)
constexpr int TJ_ZBYTES = 2 * TJ_ZHALF;         // 40960
constexpr int TJ_ABYTES = 16 * TJ_GRP;          // A: 128 rows (81920)
constexpr int TJ_XROW = TJ_H * 2 + 16;          // extra tile weights: 8 rows, padded stride
constexpr int TJ_NKW = 5;                       // per-CTA key partials: 4 lane quarters + the extra tile
constexpr uint32_t TJ_COL_D = 440;
__host__ __device__ inline bool tj_shape(bool bf, int H, int P, int C) {
  return bf && H == TJ_H && P == TJ_H && C == TJ_C;
}

// ---------------------------------------------------------------------------
// OTF: on-the-fly projections (the "w/o precomputation" arm of the paper's
// Table 3; §3.4 :216-222 is the precompute it ablates).  The
// FC LSTM tick kernel (LM = 4) reads ENCODER rows instead of precomputed f rows
// and applies both joint input projections at every joint evaluation:
//   z[k] = bf16(ReLU(W_enc e[b, t] + b_enc + W_pred h_s + b_pred))
// for the live joint rows k of a round, distributed by output dims: each CTA
// computes its 40 dims (mma.sync, K = D_e + P split over the 10 consumer warps;
// W_pred fragments in registers as in the precompute kernel, W_enc fragments
// read through L2 every round) and st.async's the 16-byte z chunks into the
// swizzled z operand of every CTA of the cluster (BAR_Z), so no f or g is
// stored.  The predictor step produces h' only.
//   encoder rows in shared memory: stride 2 D_e + 16 bytes (one bulk copy per
//   frame; conflict-free 8-row x 16-byte B-fragment loads)
//   K-split partials [10 warps][16 rows][44] f32 in the g region (OTF_PART)
// ---------------------------------------------------------------------------
constexpr int OTF_ROWS = 16;                                   // joint rows per projection pass
constexpr int OTF_PS = 44;                                     // partial row stride (floats, conflict-free)
constexpr int OTF_PART = MAX_NW * OTF_ROWS * OTF_PS * 4;       // 28160 bytes
constexpr int OTF_MAX_DE = 1024;
__host__ __device__ inline int otf_row(int De) { return 2 * De + 16; }

// Shared-memory layout (identical on host and device).
struct Layout {
  int zstride, hstride, tiles_max, UPC, DPC, NW, JR, JRp, ring, NS;
  int tg, tj, NTH;               // TG (tcgen05 gate pre-activations), TJ (tcgen05 joint + MMA warp), threads per CTA
  size_t off_wa, off_wx;         // TJ: joint weight slice (A operand), extra tile weights
  int fss;                       // TJ: f bytes per slot (WF padded rows, 128-byte aligned for the tensor copy)
  int otf;                       // on-the-fly projections (OTF_*): encoder rows of D_e = otf elements, else 0
  int wks, pks;                  // u64 words per per-warp key entry / per cluster partial (scores: 4)
  size_t off_b, off_z, off_f, off_g, off_c, off_part, off_wkey, off_hs, off_ring, off_es, total;
};

__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// ring: bf16 LSTM (producer warp + weight ring + shared-memory h); NS slots.
// sc: greedy scores (N2): per-warp entries carry log-sum-exp partials (4 words),
// TDT cluster partials too (token + duration partials: 4 words).
// allow_tj = false: a kernel without the TJ / TG paths (debug_joint_kernel).
__host__ __device__ inline Layout make_layout(bool bf, bool lstm, int H, int P, int V1, int nD, int R, int W,
                                              int WF, int C, int NS, int sc = 0, bool allow_tj = true,
                                              int layers = 1, int otf_de = 0, int jr_min = 0) {
  Layout L;
  L.otf = otf_de;
  L.wks = sc ? 4 : 2;
  L.pks = (sc && nD > 0) ? 4 : 2;
  if (allow_tj && tj_shape(bf, H, P, C) && !sc && nD == 0) L.pks = 1;   // TJ RNN-T: the token key alone
  const int NT = (V1 + nD + 7) / 8;
  L.tiles_max = (NT + C - 1) / C;
  L.UPC = lstm ? P / C : 0;
  L.DPC = H / C;
  L.NW = bf ? MAX_NW : 8;          // bf16: one vocab tile per warp (<= MAX_NW tiles per CTA)
  L.ring = (bf && lstm) ? 1 : 0;   // bf16 LSTM: W_hh in TMEM, W_pred tiles resident in smem
  L.tg = (allow_tj && tg_shape(bf, lstm, H, P, C)) ? 1 : 0;
  L.tj = (allow_tj && tj_shape(bf, H, P, C)) ? 1 : 0;
  L.NTH = L.NW * 32 + (L.tj ? 32 : 0);
  L.NS = (L.ring && !L.tj) ? L.DPC / 8 : 0;   // W_pred tiles of this CTA in smem (TJ: registers)
  (void)NS;
  L.JR = R * W > jr_min ? R * W : jr_min;   // jr_min: unequal groups (a smaller group's wider window)
  L.JRp = (L.JR + 15) / 16 * 16;
  if (L.JRp < R) L.JRp = (R + 15) / 16 * 16;
  const int K = H > P ? H : P;
  L.zstride = bf ? (int)(align_up((size_t)K * 2, 128) + 64) : K * 4;
  L.hstride = (int)(align_up((size_t)P * 2, 128) + 64);
  size_t o = 0;
  L.off_b = o;    o = align_up(o + (size_t)(L.tiles_max * 8 + 48) * 4, 128);   // joint bias slice (+ TG: b_pred slice at 72)
  if (L.tj) o = align_up(o, 1024);   // the swizzled z operand: 1024-byte aligned (dynamic smem base is)
  L.off_z = o;    // joint operand rows; in the bf16 LSTM predictor: W_pred partials [NW][3][2][32] float4
  {
    size_t zb = L.tj ? (size_t)TJ_ZBYTES : (size_t)L.JRp * L.zstride;
    const size_t wp = (size_t)L.NW * 3 * 2 * 32 * 16;
    if (L.ring && zb < wp) zb = wp;
    o = align_up(o + zb, 128);
  }
  L.fss = (int)align_up((size_t)WF * (otf_de ? otf_row(otf_de) : TJ_FROW), 128);
  L.off_f = o;    o = align_up(o + (L.tj ? (size_t)R * L.fss : (size_t)2 * R * WF * H * (bf ? 2 : 4)), 128);
  {   // OTF: g is not kept; the region holds the projection's K-split partials
    const size_t gb = (size_t)R * H * 4, pb = otf_de ? (size_t)OTF_PART : 0;
    L.off_g = o;  o = align_up(o + (gb > pb ? gb : pb), 128);
  }
  L.off_c = o;    o = align_up(o + (size_t)R * (lstm ? L.UPC : 0) * layers * 4, 128);   // c of every layer
  L.off_part = o; o = align_up(o + (size_t)2 * C * L.JR * 8 * L.pks, 128);
  {   // TJ: 3..8 extra rows -> 5 more per-warp-subset partials (xall, joint_keys_tj)
    const int ext = V1 + nD - 64 * TJ_C;
    const int nkw = L.tj ? (ext > 2 && ext <= 8 ? TJ_NKW + 4 : TJ_NKW) : L.NW;
    L.off_wkey = o; o = align_up(o + (size_t)nkw * L.JR * 8 * L.wks, 128);
  }
  L.off_hs = o;   o = align_up(o + (size_t)(L.tg ? TG_HBYTES : L.ring ? 2 * R * L.hstride : 0), 128);
  L.off_ring = o; o = align_up(o + (size_t)L.NS * 8 * P * 2, 128);
  // E' slices (bf16 LSTM); fp32 LSTM with layers > 1: the input-side gate partials of a layer
  L.off_es = o;   o = align_up(o + (size_t)((L.ring || (lstm && layers > 1)) ? R * 4 * L.UPC * 4 : 0), 128);
  L.off_wa = o;   o = align_up(o + (size_t)(L.tj ? TJ_ABYTES : 0), 128);
  L.off_wx = o;   o = align_up(o + (size_t)(L.tj ? 8 * TJ_XROW : 0), 128);
  L.total = o;
  return L;
}

struct DecodeParams {
  // TJ: f as a 3-D tensor {8 elements, 81 chunks, B*T_max frames} with chunk
  // stride 16 B and frame stride 2H: a box of WF frames lands in shared memory
  // as rows of 81 chunks = the 1296-byte padded f rows (the 81st chunk is the
  // next frame's first, never read); fmap_ok = 0: one bulk copy per frame
  alignas(64) CUtensorMap fmap;
  int fmap_ok;
  Layout L;                      // shared-memory layout of the launch (read from the constant bank)
  int B, T_max, H, P, V1, nD;
  int blank, max_sym, tdt;
  int durations[MAX_DUR];
  int context;
  int R, W, WF;                  // rows per group, window frames, buffered frames per row
  int NS;                        // weight-ring slots (bf16 LSTM), 0 otherwise
  int n_groups, cap;
  int spec_prefetch;             // speculative next-window prefetch
  int frame_looping;             // 1: Alg. 2 baseline control flow (RNN-T, W = 1)
  int sched;                     // label-looping schedule: 0 = Alg. 3 batched outer loop, 1 = per-row ticks
  const int *lengths;
  const int *perm;               // optional: group rows are perm[grp * R + slot] (length-ranked utterances)
  const void *f;                 // [B, T_max, H] bf16 (bf16 path) / f32
  const void *w_out, *b_out, *w_dur, *b_dur;
  const void *w_pred, *b_pred, *w_hh;
  int layers;                    // LSTM layers (> 1: fp32 generic kernel only)
  const void *w_ih_rest, *w_hh_rest, *b_ih_rest, *b_hh_rest;   // layers 2..L, stacked
  const float *tab;              // LSTM: E' [V1][4P]; stateless: G [ctx][V1][H] (b_pred in G_0)
  const bf16 *wst;               // bf16 LSTM: per-CTA tile stream [C][NG+NPT][8][P] (packed, swizzled)
  void *h;                       // f32 LSTM: [2][B][P]
  float *gglob;                  // f32 LSTM: [B][H]
  int *out_tokens, *out_timestamps, *out_durations, *out_lengths;
  float *out_scores;             // greedy scores [B] (SC instantiations), else NULL
  int *status;                   // bit0 bad length, bit1 capacity
  int *group_counter;
  unsigned long long *stats;     // see ll.h ll_stats
  unsigned long long *prof;      // optional per-warp timeline of block 0 (LL_TIMELINE_PTR)
  volatile unsigned *trace;      // debug: host-mapped progress markers [gridDim.x][8] (LL debug hook)
  // probe (parity tests, ll.h ll_options): DBG instantiations only
  float *probe_logits, *probe_g;
  int *probe_lmeta, *probe_gmeta, *probe_counts;
  int probe_rows, probe_regions;
  int probe_stall;               // probe kernels: cycles odd ranks spin before each group's init
  // ll_debug_joint mode
  const float *dbg_g;
  float *dbg_logits;
  int *dbg_argmax, *dbg_dargmax;
  int dbg_n;
  // length-sorted unequal groups (RNN-T FC tick kernels, one wave, B <= 32):
  // groups g < gp_small hold gp_rsmall utterances with a gp_wsmall-frame
  // window, the others R with W; utterances dealt by (length desc, index)
  int gp_small, gp_rsmall, gp_wsmall;
  int n_launch;                  // kernels launched by this call (host count; ll_stats [12])
  // OTF (LM = 4): p.f points at the ENCODER output [B, T_max, De] (bf16)
  int De;
  const void *w_enc, *b_enc;
};

struct RowState {
  int b[MAX_R], L[MAX_R], t[MAX_R], k[MAX_R], len[MAX_R], last[MAX_R], hpar[MAX_R], hzero[MAX_R];
  int ctx[MAX_CTX][MAX_R];
  int active[MAX_R], scanning[MAX_R], found[MAX_R], needp[MAX_R];
  int fy[MAX_R], ft[MAX_R], fd[MAX_R];
  float score[MAX_R];                    // greedy score of each slot (SC)
  float lp[MAX_JR];                      // log-probability of each logical joint row's decision (SC)
  int fbase[2][MAX_R], fcnt[2][MAX_R];   // frames held in fbuf[X] for each slot
  int slist[MAX_R], plist[MAX_R];
  int llist[MAX_R], nload;               // per-row schedule: slots whose window must be (re)loaded
  int zsrc[MAX_JR], zdst[MAX_JR];        // live joint rows k: f row offset (elements) / logical row s*W+j
  int dec[MAX_JR];                        // per joint row: token | dur_index << 24
  int zbeg[MAX_R], zcnt[MAX_R];          // per slot: first compact joint row of its window, live rows
  int nscan, npred, nactive, nz, ready;
  int wg;                                // window of the current group (p.W, or gp_wsmall)
  int grp[2];                            // group index broadcast (double-buffered)
  int ack[2];
  volatile int mcmd;                     // (TJ) command word for the MMA warp (MCMD_*)
};

// Consumer-only CTA barrier (named barrier 1): the producer warp never joins.
__device__ __forceinline__ void csync(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

// Per-CTA context of the cluster kernel.
// HC / PC / CC: compile-time joint dim H, predictor dim P and cluster size
// (0 = runtime).  The production shape (H = P = 640, 16-CTA clusters) is
// instantiated with all three fixed so that loops unroll and addressing folds.
// SC: 1 = greedy scores (N2): log-sum-exp partials ride along with the argmax keys.
// OTF: 1 = on-the-fly projections (OTF_* above; FC LSTM tick kernel only).
template <typename T, int KR, int HC = 0, int PC = 0, int CC = 0, int TM = 0, int SC = 0, int OTF = 0>
struct Ctx {
  static constexpr bool BF = sizeof(T) == 2;
  // the FC LSTM shape: tcgen05 gate pre-activations (see TG_* above); only the
  // LSTM member functions use it (the stateless FC kernel never issues a batch)
  static constexpr bool TG = BF && HC == TG_P && PC == TG_P && CC == TG_C;
  // the FC joint on tcgen05 (TJ_* above), LSTM and stateless FC kernels
  static constexpr bool TJ = BF && HC == TJ_H && PC == TJ_H && CC == TJ_C;
  const DecodeParams &p;
  const Layout &L;            // in the kernel parameters (constant bank; uniform, no registers)
  uint8_t *sm;
  RowState &rs;
  uint64_t *bars;
  uint32_t tmem;              // TMEM base address (bf16 LSTM: W_hh tiles)
  int C, rank, tid, warp, lane, NW, NCT, g, q;
  int tile0, ntiles;          // vocab n8 tiles owned by this CTA
  int vm0, nmain, vx0, nx;    // TJ: main rows [vm0, vm0 + nmain) (tensor core), extra rows [vx0, vx0 + nx) (CUDA cores)
  bool xrep;                  // TJ: <= 2 extra rows in all, held by EVERY CTA (joint rows dealt by rank)
  bool xall;                  // TJ: 3..8 extra rows, held by every CTA, dealt over all 10 warps during the MMAs
  int u0, d0;                 // LSTM units / W_pred output dims owned
  int iw;                     // issuing warp for bulk copies (a warp without a joint tile if any)
  // Barrier phase bookkeeping, replicated in every consumer thread and packed
  // into one register: bits 0-1 fph (BAR_F+X phase), 2-3 fpend (bulk copy into
  // fbuf[X] outstanding), 4-5 xph (BAR_X+par phase), 6 hph (BAR_H/G/E phase),
  // 7 par (partial-key buffer parity); TG: 8 gate batch pending, 9 BAR_GATE
  // phase, 10 the gate pre-activations in TMEM are valid for this group;
  // TJ: 11 BAR_JOINT phase, 12 BAR_SPEC phase, 13 speculative copies posted this round.
  uint32_t phs;
  uint32_t npost = 0;         // TJ, thread 0: commands posted to the MMA warp
  uint4 wpr[2][3][2];         // TJ LSTM: this warp's W_pred fragments (K blocks warp, warp + 10)
  __device__ __forceinline__ uint32_t fph(int X) const { return (phs >> X) & 1u; }
  __device__ __forceinline__ uint32_t fpend(int X) const { return (phs >> (2 + X)) & 1u; }
  __device__ __forceinline__ uint32_t xph(int X) const { return (phs >> (4 + X)) & 1u; }
  __device__ __forceinline__ uint32_t hph() const { return (phs >> 6) & 1u; }
  __device__ __forceinline__ int par() const { return (int)((phs >> 7) & 1u); }
  __device__ __forceinline__ void flip_par() {
    phs ^= 1u << 7;
    if (phs & (1u << 13)) phs ^= (1u << 12) | (1u << 13);   // BAR_SPEC consumed (warp 0) this round
  }
  unsigned long long ntile_c; // weight-ring tiles consumed so far (replicated)
  // optional timeline (debug builds with -DLL_TIMELINE, buffer from
  // LL_TIMELINE_PTR): clock64 of every warp at phase boundaries of the first
  // TL_N rounds / predictor steps of block 0.  Compiled out of libll.so.
#ifdef LL_TIMELINE
  unsigned long long *tl = nullptr;
  int tl_round = 0, tl_step = 0;
  __device__ void tl_stamp(int area, int idx, int ph) const {
    if (tl != nullptr && idx < TL_N && lane == 0) tl[(((size_t)area * TL_N + idx) * TL_PH + ph) * MAX_NW + warp] = clock64();
  }
  // after a (deferred-blocking) bar.sync: a dependent shared load first, so the
  // stamp is taken after the barrier has released this warp
  __device__ void tl_stamp_bar(int area, int idx, int ph) const {
    if (tl != nullptr) {
      const int v = *(volatile int *)&rs.nz;
      if (v >= -1) tl_stamp(area, idx, ph);
    }
  }
  // one [2][TL_N][TL_PH][MAX_NW] record per block (the buffer holds gridDim.x of them)
  __device__ void tl_init() {
    tl = p.prof != nullptr ? p.prof + (size_t)blockIdx.x * 2 * TL_N * TL_PH * MAX_NW : nullptr;
  }
  // warp 0's sub-phases of a round's finish (phase slot 14, "warp" column k)
  __device__ void tl_sub(int k) const {
    if (tl != nullptr && tl_round < TL_N && lane == 0) tl[((size_t)tl_round * TL_PH + 14) * MAX_NW + k] = clock64();
  }
  __device__ void tl_next_round() { ++tl_round; }
  __device__ void tl_next_step() { ++tl_step; }
#else
  __device__ __forceinline__ void tl_stamp(int, int, int) const {}
  __device__ __forceinline__ void tl_stamp_bar(int, int, int) const {}
  __device__ __forceinline__ void tl_init() {}
  __device__ __forceinline__ void tl_sub(int) const {}
  __device__ __forceinline__ void tl_next_round() {}
  __device__ __forceinline__ void tl_next_step() {}
  static constexpr int tl_round = 0, tl_step = 0;
#endif
  __device__ void tl_round_(int ph) const { tl_stamp(0, tl_round, ph); }
  __device__ void tl_round_bar(int ph) const { tl_stamp_bar(0, tl_round, ph); }
  __device__ void tl_pred(int ph) const { tl_stamp(1, tl_step, ph); }
  __device__ void tl_pred_bar(int ph) const { tl_stamp_bar(1, tl_step, ph); }
  uint4 wreg[KR];             // this warp's joint weight tile (bf16), K-permuted fragments
  uint2 wtail;
  __device__ Ctx(const DecodeParams &p_, uint8_t *sm_, RowState &rs_, bool lstm, uint64_t *bars_)
      : p(p_), L(p_.L), sm(sm_), rs(rs_), bars(bars_), phs(0), ntile_c(0) {
    (void)lstm;
    tl_init();
    C = CC ? CC : (int)cluster_size();
    rank = (int)cluster_rank();
    tid = threadIdx.x; warp = tid >> 5; lane = tid & 31;
    NW = BF ? MAX_NW : L.NW;  // consumer warps
    NCT = NW * 32;           // consumer threads
    g = lane >> 2; q = lane & 3;
    const int NT = (p.V1 + p.nD + 7) / 8;
    const int base = NT / C, rem = NT % C;
    ntiles = base + (rank < rem ? 1 : 0);
    tile0 = rank * base + (rank < rem ? rank : rem);
    if constexpr (TJ) {   // 64 rows per CTA on the tensor core; the rest (<= 8 per CTA) spread over the CTAs
      const int NV = p.V1 + p.nD, nxr = NV > 64 * TJ_C ? (NV - 64 * TJ_C + TJ_C - 1) / TJ_C : 0;
      vm0 = 64 * rank;
      nmain = min(max(NV - vm0, 0), 64);
      // <= 2 extra rows (the FC RNN-T: 1): warps 8-9; 3..8 (TDT: 6): all 10 warps
      xrep = NV > 64 * TJ_C && NV - 64 * TJ_C <= 2;
      xall = NV - 64 * TJ_C > 2 && NV - 64 * TJ_C <= 8;
      if (xrep || xall) {   // every CTA holds all extra rows; CTA r evaluates them for joint rows r, r + 16
        vx0 = 64 * TJ_C;
        nx = NV - 64 * TJ_C;
      } else {      // more extra rows: spread over the CTAs (<= 8 each), every joint row
        vx0 = 64 * TJ_C + nxr * rank;
        nx = min(max(NV - vx0, 0), nxr);
      }
    }
    u0 = rank * upc();
    d0 = rank * dpc();
    iw = (BF && L.tiles_max < NW) ? NW - 1 : 0;
  }
  __device__ __forceinline__ int Hd() const { return HC ? HC : p.H; }
  // shared-memory row strides (compile-time in the FC instantiation; must
  // match make_layout): bf16 z rows / h rows padded by 64 B against bank conflicts
  __device__ __forceinline__ int zstride() const {
    if constexpr (BF && HC && PC) return (int)align_up((size_t)(HC > PC ? HC : PC) * 2, 128) + 64;
    else return L.zstride;
  }
  __device__ __forceinline__ int hstride() const {
    if constexpr (PC != 0) return (int)align_up((size_t)PC * 2, 128) + 64;
    else return L.hstride;
  }
  // units / output dims per CTA (compile-time in the FC instantiation)
  __device__ __forceinline__ int upc() const { return (PC && CC) ? PC / CC : L.UPC; }
  __device__ __forceinline__ int dpc() const { return (HC && CC) ? HC / CC : L.DPC; }
  __device__ __forceinline__ bool is_tdt() const { return TM == 0 ? p.tdt != 0 : TM == 2; }
  // TJ RNN-T tick kernels without scores / probe / OTF: the decisions are read
  // from warp 0's registers (finish_round_rnnt) and z rows from (slot, frame),
  // so the compact-row tables (zsrc / zdst) and the per-row decision array are
  // not written
  __device__ __forceinline__ bool lean() const {
    return TJ && !is_tdt() && !SC && !OTF && p.sched == 1 && !p.frame_looping && p.probe_logits == nullptr;
  }
  __device__ __forceinline__ int Pd() const { return PC ? PC : p.P; }
  __device__ uint64_t *bar(int i) const { return bars + i; }
  __device__ float *bsl() const { return (float *)(sm + L.off_b); }
  __device__ uint8_t *zs() const { return sm + L.off_z; }
  // TJ: byte offset of row k's 16-byte chunk c in the swizzled z operand
  __device__ __forceinline__ static int zoff(int k, int c) {
    const int a = c >= 40 ? 1 : 0, cc = c - 40 * a;
    return (cc >> 3) * 8192 + a * 4096 + (k >> 3) * 1024 + (k & 7) * 128 + (((cc & 7) ^ (k & 7)) << 4);
  }
  // TJ window rows: bytes per source row (f, or the encoder row under OTF) and
  // the padded row stride in shared memory
  __device__ __forceinline__ int frow_src() const { return OTF ? p.De * 2 : TJ_H * 2; }
  __device__ __forceinline__ int frow_smem() const { return OTF ? otf_row(p.De) : TJ_FROW; }
  __device__ uint8_t *fbuf(int X) const {
    if constexpr (TJ) return sm + L.off_f;   // one buffer (the bookkeeping of both halves is kept)
    else return sm + L.off_f + (size_t)X * p.R * p.WF * Hd() * sizeof(T);
  }

  __device__ float *gs() const { return (float *)(sm + L.off_g); }
  // bf16 path: g rows are stored as two planes, so that build_z's per-lane
  // 8-dim chunk c is two CONSECUTIVE float4s across lanes (conflict-free):
  // dims 8c..8c+3 at float 4c, dims 8c+4..8c+7 at float H/2 + 4c.  f32 path: plain.
  __device__ __forceinline__ int goff(int d) const {   // d % 4 == 0: float offset of the float4 at dim d
    if constexpr (BF) return ((d >> 2) & 1) * (Hd() / 2) + (d >> 3) * 4;
    else return d;
  }
  __device__ float *cs() const { return (float *)(sm + L.off_c); }
  __device__ uint64_t *part(int pr) const { return (uint64_t *)(sm + L.off_part) + (size_t)pr * C * L.JR * pks(); }
  // words per per-warp key entry / per cluster partial (compile-time unless SC with a runtime family)
  __device__ __forceinline__ int wks() const { return SC ? 4 : 2; }
  __device__ __forceinline__ int pks() const { return (SC && is_tdt()) ? 4 : (TJ && !SC && !is_tdt()) ? 1 : 2; }
  __device__ uint64_t *wkey() const { return (uint64_t *)(sm + L.off_wkey); }
  __device__ uint8_t *hsrow(int hp, int s) const { return sm + L.off_hs + ((size_t)hp * p.R + s) * hstride(); }
  __device__ float *es() const { return (float *)(sm + L.off_es); }
  __device__ uint8_t *ringslot(int slot) const { return sm + L.off_ring + (size_t)slot * 8 * Pd() * 2; }
  __device__ void sync() const { csync(NCT); }

  // ---- TG: gate pre-activation batches (MMA warp) ---------------------------
  __device__ uint8_t *hbuf() const { return sm + L.off_hs; }
  // byte offset of 16-byte chunk c (K elements 8c .. 8c+7) of slot n's h row
  __device__ __forceinline__ static int hoff(int n, int c) { return c * TG_CM + n * 16; }
  // every consumer thread: wait for the outstanding gate batch, if any
  __device__ __forceinline__ void gate_wait() {
    if constexpr (TG) {
      if (phs & (1u << 8)) {
        mbar_wait(bar(BAR_GATE), (phs >> 9) & 1u);
        phs ^= 1u << 9;
        phs &= ~(1u << 8);
      }
    }
  }
  // consumer thread 0 (after a CTA barrier that follows every thread's
  // fence.proxy.async): request a gate batch over the current h buffer.
  // Every consumer thread calls it (replicated bookkeeping).
  __device__ __forceinline__ void gate_request() {
    if (tid == 0) post(MCMD_GATES);
    phs |= (1u << 8) | (1u << 10);
  }
  // thread 0: hand a command to the MMA warp (after the previous one was read)
  __device__ void post(int cmd) {
    if (npost > 0) mbar_wait(bar(BAR_MACK), (npost - 1) & 1u);
    rs.mcmd = cmd;
    mbar_arrive(bar(BAR_GQ));
    ++npost;
  }
  __device__ __forceinline__ uint32_t jph() const { return (phs >> 11) & 1u; }
  // The MMA warp (lane 0) executes the posted commands in order:
  //   MCMD_GATES: D_main = W_hh[rows 0..127] h, D_fold = the K-quarter partials
  //               of rows 128..159 (TS mode, A in TMEM) -> BAR_GATE
  //   MCMD_JOINT: D' = A(W_out slice, K-folded) . z^T (SS mode)  -> BAR_JOINT
  __device__ void mma_warp_loop() {
    if constexpr (TJ) {
      constexpr uint32_t ID_MAIN = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(TG_NH >> 3) << 17) | (8u << 24);
      constexpr uint32_t ID_FOLD = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(4 * TG_NH >> 3) << 17) | (8u << 24);
      constexpr uint32_t ID_J = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(64 >> 3) << 17) | (8u << 24);
      const uint32_t hb = smem_u32(hbuf()), za = smem_u32(zs()), wa = smem_u32(sm + L.off_wa);
      for (uint32_t ph = 0;; ph ^= 1u) {
        mbar_wait(bar(BAR_GQ), ph);
        const int word = rs.mcmd, cmd = word & 0xFF;
        __syncwarp();
        if (lane == 0) mbar_arrive(bar(BAR_MACK));
        if (cmd == MCMD_EXIT) break;
        tc_fence_after();
        if (lane == 0 && cmd == MCMD_GATES) {
#pragma unroll
          for (int kk = 0; kk < TG_P / 16; ++kk) {   // K = 16 per MMA: h chunks 2kk, 2kk + 1
            const int c = 2 * kk;
            const uint64_t db = umma_desc_ns(hb + (uint32_t)(c * TG_CM), TG_CM, 1024);
            umma_ts(tmem + TG_COL_DMAIN, tmem + (uint32_t)(8 * kk), db, ID_MAIN, kk > 0);
          }
#pragma unroll
          for (int kk = 0; kk < TG_P / 64; ++kk) {   // the 4 K-quarters side by side (32 B rows)
            const uint64_t db = umma_desc_ns(hb + (uint32_t)(kk * 2 * TG_CM), TG_CM, TG_QB);
            umma_ts(tmem + TG_COL_DFOLD, tmem + TG_COL_FOLD + (uint32_t)(8 * kk), db, ID_FOLD, kk > 0);
          }
          umma_commit(bar(BAR_GATE));
        } else if (lane == 0 && cmd == MCMD_JOINT) {
#pragma unroll
          for (int kk = 0; kk < TJ_H / 32; ++kk) {   // K' = 320: A / B chunks 2kk, 2kk + 1
            const uint64_t da = umma_desc_ns(wa + (uint32_t)(kk * 256), 128, TJ_GRP);
            const uint64_t db = umma_desc_sw128(za + (uint32_t)((kk >> 2) * 8192 + (kk & 3) * 32));
            umma_ss(tmem + TJ_COL_D, da, db, ID_J, kk > 0);
          }
          umma_commit(bar(BAR_JOINT));
        }
        __syncwarp();
        if (cmd == MCMD_FLOAD) spec_copies((word >> 9) & 1, true);
        if (cmd == MCMD_JOINT && (word & 0x100)) {   // next windows, while the MMAs run
          spec_copies((word >> 9) & 1);
          __syncwarp();
          if (lane == 0) mbar_arrive(bar(BAR_SPEC));
        }
      }
    }
  }

  __device__ void init_barriers() {
    if (tid == 0) {
      for (int i = 0; i < NBARS; ++i) mbar_init(bars + i, 1);
      fence_mbar_init();
    }
  }

  // -------------------------------------------------------------------------
  // This CTA's slice of [W_out; W_dur]: rows tile0*8 ... (8 per warp) into the
  // warp's registers once per kernel (bf16 path); bias slice (fp32) in smem.
  // -------------------------------------------------------------------------
  __device__ void load_weight_slice() {
    const int nrows = L.tiles_max * 8;
    const int V1 = p.V1, NV = p.V1 + p.nD, H = Hd();
    float *bs = bsl();
    if constexpr (TJ) {   // bias: [0, 64) main rows, [64, 64 + nx) extra rows; [72, 72 + 40) b_pred slice (LSTM)
      if (p.b_pred != nullptr && p.w_hh != nullptr)   // OTF: b_pred + b_enc (both projections per round)
        for (int r = tid; r < TG_UPC; r += NCT)
          bs[72 + r] = to_f32(((const T *)p.b_pred)[d0 + r]) + (OTF ? to_f32(((const T *)p.b_enc)[d0 + r]) : 0.f);
      for (int r = tid; r < 72; r += NCT) {
        const int v = r < 64 ? vm0 + r : vx0 + (r - 64);
        float bv = 0.f;
        if (r < 64 ? r < nmain : r - 64 < nx)
          bv = v < V1 ? to_f32(((const T *)p.b_out)[v]) : to_f32(((const T *)p.b_dur)[v - V1]);
        bs[r] = bv;
      }
    } else
    for (int r = tid; r < nrows; r += NCT) {
      const int v = tile0 * 8 + r;
      float bv = 0.f;
      if (r < ntiles * 8 && v < NV)
        bv = v < V1 ? to_f32(((const T *)p.b_out)[v]) : to_f32(((const T *)p.b_dur)[v - V1]);
      bs[r] = bv;
    }
    if constexpr (TJ) {
      // A operand: the first 8 tiles (64 rows), row r = 32 (vl / 16) + 16 a + vl % 16
      // holds local row vl's K-half a; the 9th tile (if any) for mma.sync
      for (int i = tid; i < 128 * (TJ_H / 16); i += NCT) {
        const int r = i / (TJ_H / 16), c = i % (TJ_H / 16);
        const int vl = 16 * (r >> 5) + (r & 15), a = (r >> 4) & 1, v = vm0 + vl;
        uint4 x = make_uint4(0, 0, 0, 0);
        if (vl < nmain && v < NV) {
          const bf16 *src = v < V1 ? (const bf16 *)p.w_out + (size_t)v * TJ_H : (const bf16 *)p.w_dur + (size_t)(v - V1) * TJ_H;
          x = ldg128_nc(src + a * (TJ_H / 2) + c * 8);
        }
        *reinterpret_cast<uint4 *>(sm + L.off_wa + (r >> 3) * TJ_GRP + c * 128 + (r & 7) * 16) = x;
      }
      for (int i = tid; i < 8 * (TJ_H / 8); i += NCT) {
        const int r = i / (TJ_H / 8), c = i % (TJ_H / 8);
        const int v = vx0 + r;
        uint4 x = make_uint4(0, 0, 0, 0);
        if (r < nx) {
          const bf16 *src = v < V1 ? (const bf16 *)p.w_out + (size_t)v * TJ_H : (const bf16 *)p.w_dur + (size_t)(v - V1) * TJ_H;
          x = ldg128_nc(src + c * 8);
        }
        *reinterpret_cast<uint4 *>(sm + L.off_wx + r * TJ_XROW + c * 16) = x;
      }
      fence_proxy_async_smem();   // the A operand is read by the tensor core
    } else if constexpr (BF) {
      const int KB = H / 32;
      const int v = tile0 * 8 + warp * 8 + g;
      const bool ok = warp < ntiles && v < NV;
      const bf16 *src = ok ? (v < V1 ? (const bf16 *)p.w_out + (size_t)v * H
                                     : (const bf16 *)p.w_dur + (size_t)(v - V1) * H)
                           : nullptr;
#pragma unroll
      for (int kb = 0; kb < KR; ++kb)
        wreg[kb] = (ok && kb < KB) ? ldg128_nc(src + kb * 32 + q * 8) : make_uint4(0, 0, 0, 0);
      wtail = (ok && (H & 31)) ? ldg64_nc(src + KB * 32 + q * 4) : make_uint2(0, 0);
    }
  }

  // -------------------------------------------------------------------------
  // f rows: for every scanning slot, frames [base, base + n) with
  //   base = t (or t + W when speculating that the row keeps scanning),
  //   n = min(WF, L - base),
  // by one bulk (TMA-engine) copy per slot into fbuf[X], completing on BAR_F+X.
  // Called by every consumer thread (the phase bookkeeping is replicated);
  // only warp 0 issues.  Caller guarantees nobody reads fbuf[X] meanwhile.
  // -------------------------------------------------------------------------
  __device__ void wait_f(int X) {
    mbar_wait(bar(BAR_F + X), fph(X));
    phs ^= 1u << X;
    phs &= ~(1u << (2 + X));
  }
  // Speculative next windows (every scanning row keeps scanning): frames
  // t + W .. into fbuf[X].  TJ: the MMA warp issues the copies right after the
  // joint MMAs (the command posted by joint_keys carries X); every consumer
  // thread records the pending copy here.
  int spec_x = -1;
  __device__ void spec_issue(int X) {
    if constexpr (TJ) {
      if (fpend(X)) wait_f(X);
      if (fpend(X ^ 1)) wait_f(X ^ 1);
      spec_x = X;
      phs |= (1u << (2 + X)) | (1u << 13);
    } else {
      issue_f(X, true);
    }
  }
  // MMA warp (all lanes): the copies of a posted speculative request; lane =
  // scanning slot.  fbase / fcnt are written before the (releasing) expect_tx
  // arrive, so a consumer that waited on BAR_F + X sees them.
  // (also the reloads at a tick's start: list = llist, base = t)
  __device__ void spec_copies(int X, bool reload = false) {
    const int n = reload ? rs.nload : rs.nscan;
    uint32_t bytes = 0;
    int s = 0, base = 0, cnt = 0;
    if (lane < n) {
      s = reload ? rs.llist[lane] : rs.slist[lane];
      base = rs.t[s] + (reload ? 0 : rs.wg);
      cnt = rs.L[s] - base;
      if (cnt > p.WF) cnt = p.WF;
      if (cnt < 0) cnt = 0;
      rs.fbase[X][s] = base;
      rs.fcnt[X][s] = cnt;
      bytes = cnt > 0 ? (p.fmap_ok ? (uint32_t)(p.WF * TJ_FROW) : (uint32_t)(cnt * frow_src())) : 0u;
    }
    uint32_t tot = bytes;
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    __syncwarp();
    if (lane == 0) mbar_arrive_expect_tx(bar(BAR_F + X), tot);
    __syncwarp();
    if (lane < n && cnt > 0) {
      if (p.fmap_ok) {
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                smem_u32(fbuf(X) + (size_t)s * L.fss)),
            "l"(&p.fmap), "r"(0), "r"(0), "r"(rs.b[s] * p.T_max + base), "r"(smem_u32(bar(BAR_F + X)))
            : "memory");
      } else {
        const int rb = frow_src(), rst = frow_smem();
        const uint8_t *src = (const uint8_t *)p.f + ((size_t)rs.b[s] * p.T_max + base) * rb;
        for (int i = 0; i < cnt; ++i)
          bulk_g2s(fbuf(X) + (size_t)s * L.fss + (size_t)i * rst, src + (size_t)i * rb, rb, bar(BAR_F + X));
      }
    }
  }

  // TJ tick start: the windows of rs.llist into fbuf[X], issued by the MMA warp
  // (after every reader of fbuf is done: the caller's barrier)
  __device__ void reload_f(int X) {
    if (fpend(X)) wait_f(X);
    if (fpend(X ^ 1)) wait_f(X ^ 1);
    if (tid == 0) post(MCMD_FLOAD | (X << 9));
    phs |= 1u << (2 + X);
  }

  __device__ void issue_f(int X, bool spec, const int *list = nullptr, int nlist = 0) {
    if (fpend(X)) wait_f(X);  // drain a stale speculative copy first
    if (TJ && fpend(X ^ 1)) wait_f(X ^ 1);   // one buffer behind both halves
    const int n = list ? nlist : rs.nscan;
    const uint32_t frb = TJ ? (uint32_t)frow_src() : (uint32_t)(Hd() * sizeof(T));
    if (warp == iw) {
      uint32_t bytes = 0;
      int s = 0, base = 0, cnt = 0;
      if (lane < n) {
        s = list ? list[lane] : rs.slist[lane];
        base = rs.t[s] + (spec ? p.W : 0);
        cnt = rs.L[s] - base;
        if (cnt > p.WF) cnt = p.WF;
        if (cnt < 0) cnt = 0;
        bytes = (uint32_t)cnt * frb;
      }
      if (TJ && p.fmap_ok && cnt > 0) bytes = (uint32_t)(p.WF * TJ_FROW);   // whole boxes
      uint32_t tot = bytes;
      for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
      if (lane == 0) mbar_arrive_expect_tx(bar(BAR_F + X), tot);
      __syncwarp();
      if (lane < n) {
        rs.fbase[X][s] = base;
        rs.fcnt[X][s] = cnt;
        if (cnt > 0) {
          const uint8_t *src = (const uint8_t *)p.f + ((size_t)rs.b[s] * p.T_max + base) * frb;
          if constexpr (TJ) {   // padded rows: one tensor copy per slot (else one bulk copy per frame)
            if (p.fmap_ok) {
              asm volatile(
                  "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                      smem_u32(fbuf(X) + (size_t)s * L.fss)),
                  "l"(&p.fmap), "r"(0), "r"(0), "r"(rs.b[s] * p.T_max + base), "r"(smem_u32(bar(BAR_F + X)))
                  : "memory");
            } else {
              for (int i = 0; i < cnt; ++i)
                bulk_g2s(fbuf(X) + (size_t)s * L.fss + (size_t)i * frow_smem(), src + (size_t)i * frb, frb, bar(BAR_F + X));
            }
          } else {
            bulk_g2s(fbuf(X) + (size_t)s * p.WF * frb, src, bytes, bar(BAR_F + X));
          }
        }
      }
      __syncwarp();   // reconverge before the caller's (aligned) CTA barrier
    }
    phs |= 1u << (2 + X);
  }

  // warp 0: the live joint rows of the round (window frames of scanning slots
  // that exist): z row index and the element offset of their f row in fbuf[X].
  __device__ void plan_z(int X) {
    if (warp != 0) return;
    const int W = p.W;
    bool live = false;
    int src = 0, dst = 0;
    if (lane < rs.nscan * W) {
      const int s = rs.slist[lane / W], j = lane % W;
      const int fr = rs.t[s] + j - rs.fbase[X][s];
      live = rs.t[s] + j < rs.L[s] && fr >= 0 && fr < rs.fcnt[X][s];
      src = TJ ? (s * L.fss + fr * frow_smem()) / 2 : (s * p.WF + fr) * Hd();
      dst = s * W + j;
    }
    const unsigned m = __ballot_sync(0xffffffffu, live);
    if (live) {
      const int k = __popc(m & ((1u << lane) - 1u));
      rs.zsrc[k] = src;
      rs.zdst[k] = dst;
    }
    // per slot: its live rows are frames j = 0 .. zcnt-1 at compact rows zbeg + j
    if (lane < p.R) rs.zcnt[lane] = 0;
    __syncwarp();
    if (lane < rs.nscan) {
      const int s = rs.slist[lane], b0 = lane * W;
      rs.zbeg[s] = __popc(m & ((1u << b0) - 1u));
      rs.zcnt[s] = __popc((m >> b0) & ((1u << W) - 1u));
    }
    if (lane == 0) rs.nz = __popc(m);
  }

  // TJ tick schedule (warp 0, lane = slot): the next round's plan, made when
  // the round's decisions are taken.  Every row that scans in the next round
  // has its window at base = t (a continuing row's speculative window starts
  // at t, every other row is reloaded at t), so frame j of slot s is f row j of
  // its fbuf slot: the plan depends only on (t, L) per slot.
  __device__ void plan_next_tj(bool scan_next, int t, int Ls) {
    const int W = rs.wg;
    int cnt = 0;
    if (scan_next) cnt = min(W, Ls - t);
    int incl = cnt;   // inclusive scan over the slots (cnt = 0 on lanes >= R)
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
      if (2 * o >= p.R) break;   // uniform: lanes < R hold their full prefix sums
    }
    const int total = __shfl_sync(0xffffffffu, incl, p.R - 1);
    const int beg = incl - cnt;
    if (lane < p.R) {
      rs.zbeg[lane] = beg;
      rs.zcnt[lane] = cnt;
    }
    if (!lean()) {
      for (int j = 0; j < cnt; ++j) {
        rs.zsrc[beg + j] = (lane * L.fss + j * frow_smem()) / 2;
        rs.zdst[beg + j] = lane * W + j;
      }
    }
    if (lane == 0) rs.nz = total;
  }

  // z[jr] = ReLU(f[b_s, t_s + j] + g_s) for the live joint rows.  Other joint
  // rows keep stale values: an MMA output row depends only on its own A row
  // and those rows are never read.  Warp per joint row, 8 columns per lane.
  // tick: the TJ tick schedule's plan (plan_next_tj), where compact row zbeg[s] + j
  // is frame j of slot s's window, row j of its f buffer slot
  __device__ void build_z(int X, bool tick = false) {
    const int H = Hd(), W = p.W;
    const int nz = rs.nz;
    if constexpr (TJ) {
      // work unit = (scanning slot, 16-chunk block b): lane = (row parity h =
      // lane / 16, chunk 16b + lane % 16): g once, then window rows h, h + 2, ..
      // (compact rows zbeg + j).  Units are dealt to warps so that the four
      // sub-partitions (3, 3, 2, 2 consumer warps) get equal shares.
      (void)nz;
      constexpr int NBLK = TJ_H / 8 / 16;   // 5
      const int nu = rs.nscan * NBLK;
      const int pos = (int)((0x9832761054ull >> (4 * warp)) & 0xF);   // warps 2,3,6,7,0,1,4,5,8,9 -> 0..9
      const int h = lane >> 4, c = (lane & 15);
      const uint32_t fb = smem_u32(fbuf(X)), zb = smem_u32(zs()), gb = smem_u32(gs());
      for (int u = pos; u < nu; u += NW) {
        const int s = rs.slist[u / NBLK], cc = 16 * (u % NBLK) + c;
        const int kb0 = rs.zbeg[s], cnt = rs.zcnt[s];
        // per-lane part of the swizzled z address of chunk cc, and its 16-byte slot j
        const int a = cc >= 40 ? 1 : 0, c40 = cc - 40 * a;
        const uint32_t zl = zb + (uint32_t)((c40 >> 3) * 8192 + a * 4096);
        const uint32_t jx = (uint32_t)((c40 & 7) << 4);
        const uint4 g0 = lds128_u32(gb + (uint32_t)(s * TJ_H * 4 + cc * 16));
        const uint4 g1 = lds128_u32(gb + (uint32_t)(s * TJ_H * 4 + TJ_H * 2 + cc * 16));
        uint4 f[4];
        int kk[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int j = h + 2 * i;
          kk[i] = kb0 + j;
          if (j < cnt)
            f[i] = lds128_u32(fb + (tick ? (uint32_t)(s * L.fss + j * frow_smem())
                                         : (uint32_t)(rs.zsrc[kb0 + j] * 2)) + (uint32_t)(cc * 16));
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (h + 2 * i < cnt) {
            const int k = kk[i], r = k & 7;
            const uint32_t za = zl + (uint32_t)((k >> 3) * 1024 + r * 128) + (jx ^ (uint32_t)(r << 4));
            sts128_u32(za, relu_add_bf16x8_2(f[i], g0, g1));
          }
        }
      }
      tl_round_(11);
      fence_proxy_async_smem();   // z is read by the tensor core
      return;
    }
    if constexpr (BF) {
      // one joint row per warp pass, up to 3 16-byte chunks per lane (H <= 768):
      // all shared loads of the row are issued before any store (the compiler
      // cannot prove that z does not alias f / g)
      const int NCH = H / 8;
      for (int k = warp; k < nz; k += NW) {
        const int s = rs.zdst[k] / W;
        const uint4 *frp = reinterpret_cast<const uint4 *>(fbuf(X)) + rs.zsrc[k] / 8;
        const float4 *gr0 = reinterpret_cast<const float4 *>(gs() + (size_t)s * H);   // plane 0
        const float4 *gr1 = gr0 + H / 8;                                               // plane 1
        uint4 *zr = reinterpret_cast<uint4 *>(zs() + (size_t)k * zstride());
        uint4 fv[3];
        float4 ga[3], gb[3];
#pragma unroll
        for (int u = 0; u < 3; ++u) {
          const int c = lane + 32 * u;
          if (c < NCH) {
            fv[u] = frp[c];
            ga[u] = gr0[c];
            gb[u] = gr1[c];
          }
        }
#pragma unroll
        for (int u = 0; u < 3; ++u) {
          const int c = lane + 32 * u;
          if (c < NCH) {
            const uint4 f = fv[u];
            const float4 g0 = ga[u], g1 = gb[u];
            uint4 o;
            o.x = pack_bf16x2(fmaxf(bf16_lo(f.x) + g0.x, 0.f), fmaxf(bf16_hi(f.x) + g0.y, 0.f));
            o.y = pack_bf16x2(fmaxf(bf16_lo(f.y) + g0.z, 0.f), fmaxf(bf16_hi(f.y) + g0.w, 0.f));
            o.z = pack_bf16x2(fmaxf(bf16_lo(f.z) + g1.x, 0.f), fmaxf(bf16_hi(f.z) + g1.y, 0.f));
            o.w = pack_bf16x2(fmaxf(bf16_lo(f.w) + g1.z, 0.f), fmaxf(bf16_hi(f.w) + g1.w, 0.f));
            zr[c] = o;
          }
        }
      }
    } else {
      for (int k = warp; k < nz; k += NW) {
        const int s = rs.zdst[k] / W;
        const float4 *frp = reinterpret_cast<const float4 *>(fbuf(X)) + rs.zsrc[k] / 4;
        const float4 *gr = reinterpret_cast<const float4 *>(gs() + (size_t)s * H);
        float4 *zr = reinterpret_cast<float4 *>(zs() + (size_t)k * zstride());
        for (int c = lane; c < H / 4; c += 32) {
          const float4 fv = frp[c], gv = gr[c];
          zr[c] = make_float4(fmaxf(fv.x + gv.x, 0.f), fmaxf(fv.y + gv.y, 0.f), fmaxf(fv.z + gv.z, 0.f),
                              fmaxf(fv.w + gv.w, 0.f));
        }
      }
    }
  }

  // OTF (replaces build_z): the round's z rows with both projections applied
  // now (OTF_* above).  Per pass of 16 joint rows, warp w sums its K blocks --
  // h' (kb = w, w + 10: W_pred fragments in registers, h' of the row's slot from
  // the h buffer) and the encoder row (kb = w, w + 10, .. < D_e / 32: W_enc
  // fragments through L2) -- for the CTA's 40 output dims (3 m16 tiles, rows
  // 40..47 zero) x 2 n8 tiles, as partials P[w][row][dim]; one thread per
  // (row, 16-byte chunk) then sums the 10 partials in warp order, adds
  // b_enc + b_pred, applies ReLU, rounds to bf16 and stores the chunk into its
  // own z and every other CTA's z (st.async, tx on BAR_Z).  Remote writes are
  // safe: a CTA projects round r + 1 only after every CTA's round-r keys, which
  // each CTA sends after its joint MMAs (the readers of z) completed; the gate
  // scratch in z (predictor step) is read before the h' slices that another
  // CTA waits for are sent.
  __device__ __forceinline__ uint32_t zph() const { return (phs >> 14) & 1u; }
  __device__ void project_z(int X) {
    if constexpr (OTF) {
      constexpr int CPC = TJ_H / 8 / TJ_C;   // 16-byte z chunks per CTA (5)
      const int nz = rs.nz, KBE = p.De / 32;
      if (tid == 0) mbar_arrive_expect_tx(bar(BAR_Z), (uint32_t)((C - 1) * nz * CPC * 16));
      const uint32_t fb = smem_u32(fbuf(X)), hb = smem_u32(hbuf()), zb = smem_u32(zs()), bz = smem_u32(bar(BAR_Z));
      float *P = gs();
      const bf16 *we = (const bf16 *)p.w_enc;
      for (int k0 = 0; k0 < nz; k0 += OTF_ROWS) {
        float acc[3][2][4];
#pragma unroll
        for (int t = 0; t < 3; ++t)
#pragma unroll
          for (int nb = 0; nb < 2; ++nb) acc[t][nb][0] = acc[t][nb][1] = acc[t][nb][2] = acc[t][nb][3] = 0.f;
        uint32_t er[2], hr[2];
#pragma unroll
        for (int nb = 0; nb < 2; ++nb) {
          int k = k0 + 8 * nb + g;
          if (k >= nz) k = nz - 1;   // rows past nz: any valid row (outputs never stored)
          er[nb] = fb + (uint32_t)(rs.zsrc[k] * 2);
          hr[nb] = hb + (uint32_t)(16 * (rs.zdst[k] / rs.wg));
        }
        const int nbn = (nz - k0) > 8 ? 2 : 1;
        // W_enc fragments of this warp's first two encoder K blocks: issued
        // first, so their L2 latency overlaps the h' part (register weights)
        constexpr int NEI = (OTF_MAX_DE / 32 + MAX_NW - 1) / MAX_NW;
        uint4 wa[2][3], wb[2][3];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int kb = warp + MAX_NW * i;
#pragma unroll
          for (int t = 0; t < 3; ++t) {
            const int r0 = 16 * t + g, r1 = r0 + 8;
            const bf16 *src = we + (size_t)(d0 + r0) * p.De + (4 * kb + q) * 8;
            wa[i][t] = (kb < KBE && r0 < TG_UPC) ? ldg128_nc(src) : make_uint4(0, 0, 0, 0);
            wb[i][t] = (kb < KBE && r1 < TG_UPC) ? ldg128_nc(src + (size_t)8 * p.De) : make_uint4(0, 0, 0, 0);
          }
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {   // h' . W_pred^T (registers)
          const int kb = warp + MAX_NW * i;
          if (kb < TG_P / 32) {
            uint4 x[2];
#pragma unroll
            for (int nb = 0; nb < 2; ++nb)
              if (nb < nbn) x[nb] = lds128_u32(hr[nb] + (uint32_t)hoff(0, 4 * kb + q));
#pragma unroll
            for (int t = 0; t < 3; ++t) {
              const uint4 ua = wpr[i][t][0], ub = wpr[i][t][1];
#pragma unroll
              for (int nb = 0; nb < 2; ++nb)
                if (nb < nbn) {
                  mma_bf16_16816(acc[t][nb], ua.x, ub.x, ua.y, ub.y, x[nb].x, x[nb].y);
                  mma_bf16_16816(acc[t][nb], ua.z, ub.z, ua.w, ub.w, x[nb].z, x[nb].w);
                }
            }
          }
        }
#pragma unroll
        for (int i = 0; i < NEI; ++i) {   // e . W_enc^T (L2)
          const int kb = warp + MAX_NW * i;
          if (kb < KBE) {
            uint4 ua[3], ub[3], x[2];
#pragma unroll
            for (int t = 0; t < 3; ++t) {
              if (i < 2) {
                ua[t] = wa[i][t];
                ub[t] = wb[i][t];
              } else {
                const int r0 = 16 * t + g, r1 = r0 + 8;
                const bf16 *src = we + (size_t)(d0 + r0) * p.De + (4 * kb + q) * 8;
                ua[t] = r0 < TG_UPC ? ldg128_nc(src) : make_uint4(0, 0, 0, 0);
                ub[t] = r1 < TG_UPC ? ldg128_nc(src + (size_t)8 * p.De) : make_uint4(0, 0, 0, 0);
              }
            }
#pragma unroll
            for (int nb = 0; nb < 2; ++nb)
              if (nb < nbn) x[nb] = lds128_u32(er[nb] + (uint32_t)((4 * kb + q) * 16));
#pragma unroll
            for (int t = 0; t < 3; ++t)
#pragma unroll
              for (int nb = 0; nb < 2; ++nb)
                if (nb < nbn) {
                  mma_bf16_16816(acc[t][nb], ua[t].x, ub[t].x, ua[t].y, ub[t].y, x[nb].x, x[nb].y);
                  mma_bf16_16816(acc[t][nb], ua[t].z, ub[t].z, ua[t].w, ub[t].w, x[nb].z, x[nb].w);
                }
          }
        }
        // partials: acc[t][nb][e] = (dim 16t + g + 8(e >> 1), row 8nb + 2q + (e & 1))
#pragma unroll
        for (int t = 0; t < 3; ++t)
#pragma unroll
          for (int nb = 0; nb < 2; ++nb)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int d = 16 * t + g + 8 * (e >> 1), i = 8 * nb + 2 * q + (e & 1);
              if (d < TG_UPC && nb < nbn) P[(warp * OTF_ROWS + i) * OTF_PS + d] = acc[t][nb][e];
            }
        sync();
        if (tid < OTF_ROWS * CPC) {
          const int i = tid / CPC, c = tid % CPC, k = k0 + i;
          if (k < nz) {
            float4 s0 = make_float4(0.f, 0.f, 0.f, 0.f), s1 = s0;
#pragma unroll
            for (int w = 0; w < MAX_NW; ++w) {   // fixed warp order
              const float4 a = *reinterpret_cast<const float4 *>(P + (w * OTF_ROWS + i) * OTF_PS + 8 * c);
              const float4 b = *reinterpret_cast<const float4 *>(P + (w * OTF_ROWS + i) * OTF_PS + 8 * c + 4);
              s0.x += a.x; s0.y += a.y; s0.z += a.z; s0.w += a.w;
              s1.x += b.x; s1.y += b.y; s1.z += b.z; s1.w += b.w;
            }
            const float *bp = bsl() + 72 + 8 * c;   // b_enc + b_pred slice
            uint4 o;
            o.x = pack_relu_bf16x2(s0.x + bp[0], s0.y + bp[1]);
            o.y = pack_relu_bf16x2(s0.z + bp[2], s0.w + bp[3]);
            o.z = pack_relu_bf16x2(s1.x + bp[4], s1.y + bp[5]);
            o.w = pack_relu_bf16x2(s1.z + bp[6], s1.w + bp[7]);
            const uint32_t za = zb + (uint32_t)zoff(k, CPC * rank + c);
            sts128_u32(za, o);
            const uint64_t lo = ((uint64_t)o.y << 32) | o.x, hi = ((uint64_t)o.w << 32) | o.z;
#pragma unroll 16
            for (int cc = 1; cc < C; ++cc) {
              const uint32_t dr = (uint32_t)((rank + cc) % C);
              st_async_u64x2(mapa_u32(za, dr), lo, hi, mapa_u32(bz, dr));
            }
          }
        }
        sync();   // P is reused by the next pass
      }
      mbar_wait(bar(BAR_Z), zph());
      phs ^= 1u << 14;
      fence_proxy_async_smem();   // z (local stores + the other CTAs' st.async) is read by the tensor core
    }
  }

  // -------------------------------------------------------------------------
  // Joint + fused argmax over this CTA's vocabulary slice for joint rows
  // [0, MT*16).  Writes per-warp keys wkey[warp][jr] = {token key, duration key}.
  // If `logits` != nullptr (debug), also writes raw logits [row_base + jr][v].
  // -------------------------------------------------------------------------
  template <int MT>
  __device__ __forceinline__ void joint_mma(float (&acc)[2][2][4]) const {
    const int KB = Hd() / 32;
    const uint8_t *a0 = zs() + (size_t)g * zstride() + q * 16;
    const uint8_t *a1 = a0 + (size_t)8 * zstride();
    const uint8_t *a2 = a0 + (size_t)16 * zstride();
    const uint8_t *a3 = a0 + (size_t)24 * zstride();
    if (KB == KR) {
      // hot path (H = 640): fully unrolled, no guards, loads can be hoisted
#pragma unroll
      for (int kb = 0; kb < KR; ++kb) {
        const uint4 b = wreg[kb];
        const uint4 x0 = lds128(a0 + kb * 64), x1 = lds128(a1 + kb * 64);
        mma_bf16_16816(acc[0][kb & 1], x0.x, x1.x, x0.y, x1.y, b.x, b.y);
        mma_bf16_16816(acc[0][kb & 1], x0.z, x1.z, x0.w, x1.w, b.z, b.w);
        if (MT > 1) {
          const uint4 x2 = lds128(a2 + kb * 64), x3 = lds128(a3 + kb * 64);
          mma_bf16_16816(acc[1][kb & 1], x2.x, x3.x, x2.y, x3.y, b.x, b.y);
          mma_bf16_16816(acc[1][kb & 1], x2.z, x3.z, x2.w, x3.w, b.z, b.w);
        }
      }
    } else {
#pragma unroll
      for (int kb = 0; kb < KR; ++kb) {
        if (kb < KB) {
          const uint4 b = wreg[kb];
          const uint4 x0 = lds128(a0 + kb * 64), x1 = lds128(a1 + kb * 64);
          mma_bf16_16816(acc[0][kb & 1], x0.x, x1.x, x0.y, x1.y, b.x, b.y);
          mma_bf16_16816(acc[0][kb & 1], x0.z, x1.z, x0.w, x1.w, b.z, b.w);
          if (MT > 1) {
            const uint4 x2 = lds128(a2 + kb * 64), x3 = lds128(a3 + kb * 64);
            mma_bf16_16816(acc[1][kb & 1], x2.x, x3.x, x2.y, x3.y, b.x, b.y);
            mma_bf16_16816(acc[1][kb & 1], x2.z, x3.z, x2.w, x3.w, b.z, b.w);
          }
        }
      }
      if (Hd() & 31) {
        const int o = KB * 64 - q * 8;
        const uint2 x0 = lds64(a0 + o), x1 = lds64(a1 + o);
        mma_bf16_16816(acc[0][0], x0.x, x1.x, x0.y, x1.y, wtail.x, wtail.y);
        if (MT > 1) {
          const uint2 x2 = lds64(a2 + o), x3 = lds64(a3 + o);
          mma_bf16_16816(acc[1][0], x2.x, x3.x, x2.y, x3.y, wtail.x, wtail.y);
        }
      }
    }
  }

  // TJ butterfly: 32-lane keys/partials, lane l keeps column l after the 4 steps
  // (xor 8, 4, 2, 1 inside each 16-lane half; lane l's half = column block l / 16).
  template <int NK>
  __device__ __forceinline__ static void bfly_max(uint64_t (&x)[NK], int lane) {
#pragma unroll
    for (int w = 8; w >= 1; w >>= 1) {
      const bool b = (lane & w) != 0;
#pragma unroll
      for (int i = 0; i < w; ++i) {
        const uint64_t lo = x[i], hi = x[i + w];
        const uint64_t r = shfl_xor_u64(b ? lo : hi, w);
        x[i] = umax64(b ? hi : lo, r);
      }
    }
  }
  template <int NK>
  __device__ __forceinline__ static void bfly_lse(uint64_t (&x)[NK], int lane) {
#pragma unroll
    for (int w = 8; w >= 1; w >>= 1) {
      const bool b = (lane & w) != 0;
#pragma unroll
      for (int i = 0; i < w; ++i) {
        const uint64_t lo = x[i], hi = x[i + w];
        const uint64_t r = shfl_xor_u64(b ? lo : hi, w);
        x[i] = lse_combine(b ? hi : lo, r);
      }
    }
  }
  template <int NK>
  __device__ __forceinline__ static void bfly8_max(uint64_t (&x)[NK], int lane) {
#pragma unroll
    for (int w = 4; w >= 1; w >>= 1) {
      const bool b = (lane & w) != 0;
#pragma unroll
      for (int i = 0; i < w; ++i) {
        const uint64_t lo = x[i], hi = x[i + w];
        const uint64_t r = shfl_xor_u64(b ? lo : hi, w);
        x[i] = umax64(b ? hi : lo, r);
      }
    }
    x[0] = umax64(x[0], shfl_xor_u64(x[0], 8));
  }
  template <int NK>
  __device__ __forceinline__ static void bfly8_lse(uint64_t (&x)[NK], int lane) {
#pragma unroll
    for (int w = 4; w >= 1; w >>= 1) {
      const bool b = (lane & w) != 0;
#pragma unroll
      for (int i = 0; i < w; ++i) {
        const uint64_t lo = x[i], hi = x[i + w];
        const uint64_t r = shfl_xor_u64(b ? lo : hi, w);
        x[i] = lse_combine(b ? hi : lo, r);
      }
    }
    // the two 8-lane groups, combined in a fixed (group 0, group 1) order on both sides
    const uint64_t o = shfl_xor_u64(x[0], 8);
    x[0] = (lane & 8) ? lse_combine(o, x[0]) : lse_combine(x[0], o);
  }
  __device__ __forceinline__ int nkw() const {
    if constexpr (TJ) return xall ? TJ_NKW + 4 : nx > 0 ? TJ_NKW : TJ_NKW - 1;
    else return NW;
  }

  // TJ joint: the MMA warp runs D' = A . z^T (posted here); warps 0-3 read D'
  // (lane quarter q = vocabulary rows 16q .. 16q + 15, both K-halves), warps
  // 4-5 the extra tile on mma.sync; per-partial keys -> wkey[0..4][jr].
  __device__ void joint_keys_tj(int nrows_valid, float *logits, int row_base) {
    const int V1 = p.V1, NV = p.V1 + p.nD;
    uint64_t *wk = wkey();
#ifdef LL_TIMELINE
    if (tid == 0 && tl != nullptr && tl_round < TL_N) {   // is the background gate batch still running?
      const bool pend = (phs & (1u << 8)) && !mbar_test_wait(smem_u32(bar(BAR_GATE)), (phs >> 9) & 1u);
      tl[((size_t)tl_round * TL_PH + 14) * MAX_NW + 7] = pend ? 2 : 1;
      tl[((size_t)tl_round * TL_PH + 14) * MAX_NW + 8] = clock64();
    }
#endif
    if (tid == 0) post(MCMD_JOINT | (spec_x >= 0 ? 0x100 | (spec_x << 9) : 0));
    spec_x = -1;
    // extra rows (<= 8 per CTA, rows vx0 ..): after the MMAs (the tensor pipe and
    // shared memory are busy with them until then), warps 8 and 9 take joint
    // rows 0-15 / 16-31 on mma.sync: z rows as the m16 A operand (ldmatrix from
    // the swizzled z), the extra weight rows as the n8 B operand, 4 chains
    if (TM != 1 && xall) {   // (compiled out of the RNN-T kernels)
      // 3..8 extra rows (TDT: token 1024 + 5 duration rows): every CTA, for its
      // joint rows k = rank + 16 h only, dealt over the 10 consumer warps while
      // the MMAs run (warps 0-7 idle until BAR_JOINT): warp w takes h = w & 1
      // and the extra rows {w / 2, w / 2 + 5}, its keys are partial 4 + w / 2
      // (the other joint rows of that partial: neutral), reduced with the rest
      // in exchange_keys
      const int hf = warp & 1, j = warp >> 1;
      uint64_t *wkj = wk + (size_t)(4 + j) * L.JR * wks();
      for (int k = 16 * hf + lane; k < min(L.JR, 16 * hf + 16); k += 32) {   // neutral partials
        if (k == rank + 16 * hf) continue;
        uint64_t *dst = wkj + (size_t)k * wks();
        *reinterpret_cast<uint4 *>(dst) = make_uint4(0, 0, 0, 0);
        if constexpr (SC) {
          const uint64_t e = lse_empty();
          *reinterpret_cast<uint4 *>(dst + 2) = make_uint4((uint32_t)e, (uint32_t)(e >> 32), (uint32_t)e, (uint32_t)(e >> 32));
        }
      }
      const int k = rank + 16 * hf;
      const uint32_t zb = smem_u32(zs()), wb = smem_u32(sm + L.off_wx);
      uint4 zc[3];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const int c = lane + 32 * i;
        zc[i] = c < TJ_H / 8 ? lds128_u32(zb + (uint32_t)zoff(k, c)) : make_uint4(0, 0, 0, 0);
      }
      uint64_t tk2 = 0, dk2 = 0;
      [[maybe_unused]] uint64_t tl2 = lse_empty(), dl2 = lse_empty();
#pragma unroll
      for (int xx = 0; xx < 2; ++xx) {
        const int x = j + 5 * xx;
        if (x < nx) {
          float d = 0.f;
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            const int c = lane + 32 * i;
            if (c < TJ_H / 8) d += dot_bf16x8(zc[i], lds128_u32(wb + (uint32_t)(x * TJ_XROW + c * 16)));
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
          const float val = d + bsl()[64 + x];
          const int v2 = vx0 + x;
          if (logits != nullptr && lane == 0 && k < nrows_valid) logits[(size_t)(row_base + k) * NV + v2] = val;
          if (v2 < V1) tk2 = umax64(tk2, pack_key(val, v2));
          else dk2 = umax64(dk2, pack_key(val, v2 - V1));
          if constexpr (SC) {
            if (v2 < V1) tl2 = lse_combine(tl2, lse_pack(val, 1.f));
            else dl2 = lse_combine(dl2, lse_pack(val, 1.f));
          }
        }
      }
      if (lane == 0 && k < L.JR) {
        uint64_t *dst = wkj + (size_t)k * wks();
        *reinterpret_cast<uint4 *>(dst) =
            make_uint4((uint32_t)tk2, (uint32_t)(tk2 >> 32), (uint32_t)dk2, (uint32_t)(dk2 >> 32));
        if constexpr (SC)
          *reinterpret_cast<uint4 *>(dst + 2) =
              make_uint4((uint32_t)tl2, (uint32_t)(tl2 >> 32), (uint32_t)dl2, (uint32_t)(dl2 >> 32));
      }
    } else if (xrep) {
      // the extra row(s) (1 for the FC RNN-T) on CUDA cores WHILE the
      // MMAs run, for this CTA's joint rows only: warp 8 row k = rank, warp 9
      // row k = rank + 16; every CTA evaluates 2 rows instead of one CTA all 32
      // after the MMAs (that tail, ~1.5K cycles on rank 0, held every round of
      // the cluster).  Lanes split the 80 z chunks; a fixed xor butterfly sums.
      if (warp >= 8) {
        const int hf = warp - 8;
        for (int k = 16 * hf + lane; k < min(L.JR, 16 * hf + 16); k += 32) {   // neutral partials
          if (k == rank + 16 * hf) continue;
          uint64_t *dst = wk + ((size_t)4 * L.JR + k) * wks();
          *reinterpret_cast<uint4 *>(dst) = make_uint4(0, 0, 0, 0);
          if constexpr (SC) {
            const uint64_t e = lse_empty();
            *reinterpret_cast<uint4 *>(dst + 2) = make_uint4((uint32_t)e, (uint32_t)(e >> 32), (uint32_t)e, (uint32_t)(e >> 32));
          }
        }
        const uint32_t zb = smem_u32(zs()), wb = smem_u32(sm + L.off_wx);
        {
          const int k = rank + 16 * hf;
          uint4 zc[3];
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            const int c = lane + 32 * i;
            zc[i] = c < TJ_H / 8 ? lds128_u32(zb + (uint32_t)zoff(k, c)) : make_uint4(0, 0, 0, 0);
          }
          uint64_t tk2 = 0, dk2 = 0;
          [[maybe_unused]] uint64_t tl2 = lse_empty(), dl2 = lse_empty();
#pragma unroll 1
          for (int x = 0; x < nx; ++x) {
            float d = 0.f;
#pragma unroll
            for (int i = 0; i < 3; ++i) {
              const int c = lane + 32 * i;
              if (c < TJ_H / 8) d += dot_bf16x8(zc[i], lds128_u32(wb + (uint32_t)(x * TJ_XROW + c * 16)));
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
            const float val = d + bsl()[64 + x];
            const int v2 = vx0 + x;
            if (logits != nullptr && lane == 0 && k < nrows_valid) logits[(size_t)(row_base + k) * NV + v2] = val;
            if (v2 < V1) tk2 = umax64(tk2, pack_key(val, v2));
            else dk2 = umax64(dk2, pack_key(val, v2 - V1));
            if constexpr (SC) {
              if (v2 < V1) tl2 = lse_combine(tl2, lse_pack(val, 1.f));
              else dl2 = lse_combine(dl2, lse_pack(val, 1.f));
            }
          }
          if (lane == 0 && k < L.JR) {
            uint64_t *dst = wk + ((size_t)4 * L.JR + k) * wks();
            *reinterpret_cast<uint4 *>(dst) =
                make_uint4((uint32_t)tk2, (uint32_t)(tk2 >> 32), (uint32_t)dk2, (uint32_t)(dk2 >> 32));
            if constexpr (SC)
              *reinterpret_cast<uint4 *>(dst + 2) =
                  make_uint4((uint32_t)tl2, (uint32_t)(tl2 >> 32), (uint32_t)dl2, (uint32_t)(dl2 >> 32));
          }
        }
      }
    } else if ((warp == 8 || (warp == 9 && rs.nz > 16)) && nx > 0) {
      const int m0 = 16 * (warp - 8);
      mbar_wait(bar(BAR_JOINT), jph());
      float acc[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
      const int mi = lane >> 3, rr = lane & 7, kz = m0 + 8 * (mi & 1) + rr;
      const uint32_t zb = smem_u32(zs()), wb = smem_u32(sm + L.off_wx) + (uint32_t)(g * TJ_XROW + 4 * q);
#pragma unroll 8
      for (int kk = 0; kk < TJ_H / 16; ++kk) {
        const int c = 2 * kk + (mi >> 1);
        uint32_t a0, a1, a2, a3, b0, b1;
        ldmatrix_x4(zb + (uint32_t)zoff(kz, c), a0, a1, a2, a3);
        asm volatile("ld.shared.u32 %0, [%2];\n ld.shared.u32 %1, [%2 + 16];" : "=r"(b0), "=r"(b1) : "r"(wb + (uint32_t)(32 * kk)));
        mma_bf16_16816(acc[kk & 3], a0, a1, a2, a3, b0, b1);
      }
      uint64_t tk2[2] = {0, 0}, dk2[2] = {0, 0};
      [[maybe_unused]] uint64_t tl2[2] = {lse_empty(), lse_empty()}, dl2[2] = {lse_empty(), lse_empty()};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int i = 2 * q + (e & 1), v2 = vx0 + i, hr = e >> 1;
        if (i < nx) {
          const float val = ((acc[0][e] + acc[1][e]) + (acc[2][e] + acc[3][e])) + bsl()[64 + i];
          const int k = m0 + g + 8 * hr;
          if (logits != nullptr && k < nrows_valid) logits[(size_t)(row_base + k) * NV + v2] = val;
          if (v2 < V1) tk2[hr] = umax64(tk2[hr], pack_key(val, v2));
          else dk2[hr] = umax64(dk2[hr], pack_key(val, v2 - V1));
          if constexpr (SC) {
            if (v2 < V1) tl2[hr] = lse_combine(tl2[hr], lse_pack(val, 1.f));
            else dl2[hr] = lse_combine(dl2[hr], lse_pack(val, 1.f));
          }
        }
      }
#pragma unroll
      for (int hr = 0; hr < 2; ++hr) {
#pragma unroll
        for (int o = 1; o <= 2; o <<= 1) {
          tk2[hr] = umax64(tk2[hr], shfl_xor_u64(tk2[hr], o));
          dk2[hr] = umax64(dk2[hr], shfl_xor_u64(dk2[hr], o));
          if constexpr (SC) {   // fixed order: the lower lane's subset first
            const uint64_t ot = shfl_xor_u64(tl2[hr], o), od = shfl_xor_u64(dl2[hr], o);
            tl2[hr] = (lane & o) ? lse_combine(ot, tl2[hr]) : lse_combine(tl2[hr], ot);
            dl2[hr] = (lane & o) ? lse_combine(od, dl2[hr]) : lse_combine(dl2[hr], od);
          }
        }
        const int k = m0 + g + 8 * hr;
        if (q == 0 && k < L.JR) {
          uint64_t *dst = wk + ((size_t)4 * L.JR + k) * wks();   // partial 4: the extra rows
          uint4 e;
          e.x = (uint32_t)tk2[hr]; e.y = (uint32_t)(tk2[hr] >> 32); e.z = (uint32_t)dk2[hr]; e.w = (uint32_t)(dk2[hr] >> 32);
          *reinterpret_cast<uint4 *>(dst) = e;
          if constexpr (SC) {
            uint4 f;
            f.x = (uint32_t)tl2[hr]; f.y = (uint32_t)(tl2[hr] >> 32); f.z = (uint32_t)dl2[hr]; f.w = (uint32_t)(dl2[hr] >> 32);
            *reinterpret_cast<uint4 *>(dst + 2) = f;
          }
        }
      }
    }
    if (warp < 8) {
      // warp w: lane quarter q = w % 4 (vocabulary rows 16q .. 16q + 15, both
      // K-halves), joint-row half h = w / 4 (rows 16h .. 16h + 15)
      const int qd = warp & 3, h = warp >> 2;
      mbar_wait(bar(BAR_JOINT), jph());
      tl_round_(12);
      tc_fence_after();
      uint32_t lo[16], hi[16];
      const uint32_t ta = tmem + ((uint32_t)(32 * qd) << 16) + TJ_COL_D + 16u * h;
      tmem_ld16(ta, lo);
      tmem_ld16(ta + 32, hi);
      tmem_wait_ld();
      const int a = lane >> 4, vl = 16 * qd + (lane & 15), v = vm0 + vl;
      const int kind = vl < nmain ? (v < V1 ? 1 : 2) : 0;
      const float bias = bsl()[vl];
      const bool dmain = is_tdt() && vm0 + nmain > V1;   // duration rows among the main rows
      // joint rows k = 16h + 8a + i (i < 8): K-half partials of lanes l, l ^ 16 (lo + hi)
      uint64_t tk[8], dk[8];
      [[maybe_unused]] uint64_t tl[8], dl[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t send = a ? hi[i] : lo[i + 8];
        const float recv = __uint_as_float(__shfl_xor_sync(0xffffffffu, send, 16));
        const float val = (a ? recv + __uint_as_float(hi[i + 8]) : __uint_as_float(lo[i]) + recv) + bias;
        const int k = 16 * h + 8 * a + i;
        if (logits != nullptr && kind && k < nrows_valid) logits[(size_t)(row_base + k) * NV + v] = val;
        tk[i] = kind == 1 ? pack_key(val, v) : 0ull;
        dk[i] = kind == 2 ? pack_key(val, v - V1) : 0ull;
        if constexpr (SC) {
          tl[i] = kind == 1 ? lse_pack(val, 1.f) : lse_empty();
          dl[i] = kind == 2 ? lse_pack(val, 1.f) : lse_empty();
        }
      }
      // 8 columns over the 16 lanes of the half: xor 4, 2, 1 keep one column
      // (l & 7), xor 8 merges the two 8-lane groups
      bfly8_max(tk, lane);
      if (dmain) bfly8_max(dk, lane);
      if constexpr (SC) {
        bfly8_lse(tl, lane);
        if (dmain) bfly8_lse(dl, lane);
      }
      tl_round_(13);
      const int kc = 16 * h + 8 * a + (lane & 7);
      if ((lane & 8) == 0 && kc < L.JR) {
        uint64_t *dst = wk + ((size_t)qd * L.JR + kc) * wks();
        uint4 e;
        const uint64_t d0 = dmain ? dk[0] : 0ull;
        e.x = (uint32_t)tk[0]; e.y = (uint32_t)(tk[0] >> 32); e.z = (uint32_t)d0; e.w = (uint32_t)(d0 >> 32);
        *reinterpret_cast<uint4 *>(dst) = e;
        if constexpr (SC) {
          const uint64_t l0 = dmain ? dl[0] : lse_empty();
          uint4 f;
          f.x = (uint32_t)tl[0]; f.y = (uint32_t)(tl[0] >> 32); f.z = (uint32_t)l0; f.w = (uint32_t)(l0 >> 32);
          *reinterpret_cast<uint4 *>(dst + 2) = f;
        }
      }
    }
    tc_fence_before();   // D' reads ordered before the next joint (through the exchange barrier)
    phs ^= 1u << 11;
  }

  __device__ void joint_keys(int MT, int nrows_valid, float *logits, int row_base) {
    if constexpr (TJ) {
      (void)MT;
      joint_keys_tj(nrows_valid, logits, row_base);
      return;
    }
    const int V1 = p.V1, NV = p.V1 + p.nD, H = Hd();
    uint64_t *wk = wkey();
    if constexpr (BF) {
      float acc[2][2][4];  // [m-tile][K chain][frag]
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[a][c][e] = 0.f;
      if (warp < ntiles) {
        if (MT > 1) joint_mma<2>(acc);
        else joint_mma<1>(acc);
      }
      uint64_t tk[2][2], dk[2][2];
      [[maybe_unused]] uint64_t tl[2][2], dl[2][2];   // SC: log-sum-exp partials (token, duration)
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          tk[mt][rr] = 0;
          dk[mt][rr] = 0;
          [[maybe_unused]] float vv[2];
          [[maybe_unused]] int kind[2];   // 0 none, 1 token, 2 duration
#pragma unroll
          for (int e2 = 0; e2 < 2; ++e2) {
            const int e = rr * 2 + e2;
            const int lr = warp * 8 + 2 * q + e2;     // local vocab row
            const int v = tile0 * 8 + lr;
            if constexpr (SC) kind[e2] = 0;
            if (warp < ntiles && v < NV) {
              const float val = (acc[mt][0][e] + acc[mt][1][e]) + bsl()[lr];
              if (v < V1) tk[mt][rr] = umax64(tk[mt][rr], pack_key(val, v));
              else dk[mt][rr] = umax64(dk[mt][rr], pack_key(val, v - V1));
              if constexpr (SC) {
                vv[e2] = val;
                kind[e2] = v < V1 ? 1 : 2;
              }
              const int jr = mt * 16 + g + rr * 8;
              if (logits != nullptr && mt < MT && jr < nrows_valid) logits[(size_t)(row_base + jr) * NV + v] = val;
            }
          }
          tk[mt][rr] = umax64(tk[mt][rr], shfl_xor_u64(tk[mt][rr], 1));
          tk[mt][rr] = umax64(tk[mt][rr], shfl_xor_u64(tk[mt][rr], 2));
          if (is_tdt()) {
            dk[mt][rr] = umax64(dk[mt][rr], shfl_xor_u64(dk[mt][rr], 1));
            dk[mt][rr] = umax64(dk[mt][rr], shfl_xor_u64(dk[mt][rr], 2));
          }
          if constexpr (SC) {
            // the warp's partial over its 8 vocabulary rows: the max is the key's
            // value (exact), then the sum of exp(v - max) over the 4 lanes of the row
            const float mt_ = tk[mt][rr] ? key_value(tk[mt][rr]) : -INFINITY;
            float st_ = 0.f, sd_ = 0.f;
            const float md_ = dk[mt][rr] ? key_value(dk[mt][rr]) : -INFINITY;
#pragma unroll
            for (int e2 = 0; e2 < 2; ++e2) {
              if (kind[e2] == 1) st_ += __expf(vv[e2] - mt_);
              if (kind[e2] == 2) sd_ += __expf(vv[e2] - md_);
            }
            st_ += __shfl_xor_sync(0xffffffffu, st_, 1);
            st_ += __shfl_xor_sync(0xffffffffu, st_, 2);
            tl[mt][rr] = mt_ == -INFINITY ? lse_empty() : lse_pack(mt_, st_);
            if (is_tdt()) {
              sd_ += __shfl_xor_sync(0xffffffffu, sd_, 1);
              sd_ += __shfl_xor_sync(0xffffffffu, sd_, 2);
              dl[mt][rr] = md_ == -INFINITY ? lse_empty() : lse_pack(md_, sd_);
            } else {
              dl[mt][rr] = lse_empty();
            }
          }
        }
      if (q == 0) {
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int rr = 0; rr < 2; ++rr) {
            const int jr = mt * 16 + g + rr * 8;
            if (mt < MT && jr < L.JR) {
              uint4 e;
              e.x = (uint32_t)tk[mt][rr]; e.y = (uint32_t)(tk[mt][rr] >> 32);
              e.z = (uint32_t)dk[mt][rr]; e.w = (uint32_t)(dk[mt][rr] >> 32);
              uint64_t *dst = wk + ((size_t)warp * L.JR + jr) * wks();
              *reinterpret_cast<uint4 *>(dst) = e;
              if constexpr (SC) {
                uint4 f;
                f.x = (uint32_t)tl[mt][rr]; f.y = (uint32_t)(tl[mt][rr] >> 32);
                f.z = (uint32_t)dl[mt][rr]; f.w = (uint32_t)(dl[mt][rr] >> 32);
                *reinterpret_cast<uint4 *>(dst + 2) = f;
              }
            }
          }
      }
    } else {
      // fp32 SIMT: one warp per vocabulary row, lanes split K in a fixed order,
      // butterfly reduction; lane jr keeps the best key of joint row jr.
      uint64_t tkey = 0, dkey = 0;
      [[maybe_unused]] uint64_t tlse = lse_empty(), dlse = lse_empty();   // SC
      const int nrows = ntiles * 8;
      const int zst = zstride() / 4;
      const float *z = (const float *)zs();
      const int M = L.JR;
      for (int lr = warp; lr < nrows; lr += NW) {
        const int v = tile0 * 8 + lr;
        if (v >= NV) break;
        const float *wr = v < V1 ? (const float *)p.w_out + (size_t)v * H
                                 : (const float *)p.w_dur + (size_t)(v - V1) * H;
        float acc[MAX_JR];
#pragma unroll
        for (int i = 0; i < MAX_JR; ++i) acc[i] = 0.f;
        for (int k = lane; k < H; k += 32) {
          const float w = __ldg(wr + k);
#pragma unroll
          for (int i = 0; i < MAX_JR; ++i)
            if (i < M) acc[i] = fmaf(w, z[(size_t)i * zst + k], acc[i]);
        }
        float mine = 0.f;
#pragma unroll
        for (int i = 0; i < MAX_JR; ++i) {
          if (i < M) {
            float s = acc[i];
            s += __shfl_xor_sync(0xffffffffu, s, 16);
            s += __shfl_xor_sync(0xffffffffu, s, 8);
            s += __shfl_xor_sync(0xffffffffu, s, 4);
            s += __shfl_xor_sync(0xffffffffu, s, 2);
            s += __shfl_xor_sync(0xffffffffu, s, 1);
            if (lane == i) mine = s;
          }
        }
        if (lane < M) {
          const float val = mine + bsl()[lr];
          if (v < V1) tkey = umax64(tkey, pack_key(val, v));
          else dkey = umax64(dkey, pack_key(val, v - V1));
          if constexpr (SC) {
            if (v < V1) tlse = lse_combine(tlse, lse_pack(val, 1.f));
            else dlse = lse_combine(dlse, lse_pack(val, 1.f));
          }
          if (logits != nullptr && lane < nrows_valid) logits[(size_t)(row_base + lane) * NV + v] = val;
        }
      }
      if (lane < L.JR) {
        wk[((size_t)warp * L.JR + lane) * wks() + 0] = tkey;
        wk[((size_t)warp * L.JR + lane) * wks() + 1] = dkey;
        if constexpr (SC) {
          wk[((size_t)warp * L.JR + lane) * wks() + 2] = tlse;
          wk[((size_t)warp * L.JR + lane) * wks() + 3] = dlse;
        }
      }
    }
  }

  // Reduce per-warp keys of the live joint rows and st.async this CTA's
  // partial to every CTA of the cluster; each CTA's BAR_X+par completes when
  // all C partials of all live rows have landed.  The partial buffers are
  // double-buffered by round parity, and a CTA can be at most one round ahead
  // of any other (it needs everyone's partials to leave a round).
  __device__ void exchange_keys() {
    // TG: the other CTAs write their next h' slices into this CTA's h buffer
    // only after this round's partial keys arrive, so the gate batch reading
    // the buffer completes first
#ifdef LL_TIMELINE
    const bool gpend = (phs & (1u << 8)) != 0;
#endif
    gate_wait();
#ifdef LL_TIMELINE
    if (tid == 0 && tl != nullptr && tl_round < TL_N && gpend) tl[((size_t)tl_round * TL_PH + 14) * MAX_NW + 9] = clock64();
#endif
    const int nz = rs.nz;
    if (tid == 0) mbar_arrive_expect_tx(bar(BAR_X + par()), (uint32_t)(C * nz * 8 * pks()));
    sync();
    const uint64_t *wk = wkey();
    uint64_t *pt = part(par());
    if (tid < nz) {
      const int jr = tid;                       // compact joint row
      uint64_t tkey = 0, dkey = 0;
      [[maybe_unused]] uint64_t tl = lse_empty(), dl = lse_empty();
      const int nk = nkw();
#pragma unroll
      for (int w = 0; w < MAX_NW; ++w) {
        if (w < nk) {
          const uint64_t *e = wk + ((size_t)w * L.JR + jr) * wks();
          if (is_tdt()) {
            const uint4 v = *reinterpret_cast<const uint4 *>(e);
            tkey = umax64(tkey, ((uint64_t)v.y << 32) | v.x);
            dkey = umax64(dkey, ((uint64_t)v.w << 32) | v.z);
          } else {   // RNN-T: the token key only
            tkey = umax64(tkey, e[0]);
          }
          if constexpr (SC) {
            tl = lse_combine(tl, e[2]);
            if (is_tdt()) dl = lse_combine(dl, e[3]);
          }
        }
      }
      const uint32_t slot = smem_u32(pt + ((size_t)rank * L.JR + jr) * pks());
      const uint32_t bb = smem_u32(bar(BAR_X + par()));
      // partial: (token key, duration key) or, with scores, (token key, token lse)
      // for RNN-T and (token key, duration key, token lse, duration lse) for TDT
      const uint64_t second = (SC && !is_tdt()) ? tl : dkey;
#pragma unroll 16
      for (int d = 0; d < C; ++d) {
        const int dst = (rank + d) % C;
        if (TJ && !SC && !is_tdt()) st_async_u64(mapa_u32(slot, (uint32_t)dst), tkey, mapa_u32(bb, (uint32_t)dst));
        else st_async_u64x2(mapa_u32(slot, (uint32_t)dst), tkey, second, mapa_u32(bb, (uint32_t)dst));
        if (SC && is_tdt()) st_async_u64x2(mapa_u32(slot + 16, (uint32_t)dst), tl, dl, mapa_u32(bb, (uint32_t)dst));
      }
    }
  }
  __device__ void exchange_wait() {
    mbar_wait(bar(BAR_X + par()), xph(par()));
    phs ^= 1u << (4 + par());
  }

  // Final argmax of joint row jr from the C partials (after exchange_keys).
  __device__ void final_keys(int jr, int &y, int &di) const {
    const uint64_t *pt = part(par());
    uint64_t tkey = 0, dkey = 0;
#pragma unroll
    for (int r = 0; r < MAX_C; ++r) {
      if (r < C) {
        const uint4 v = *reinterpret_cast<const uint4 *>(pt + ((size_t)r * L.JR + jr) * pks());
        tkey = umax64(tkey, ((uint64_t)v.y << 32) | v.x);
        dkey = umax64(dkey, ((uint64_t)v.w << 32) | v.z);
      }
    }
    y = key_index(tkey);
    di = is_tdt() ? key_index(dkey) : 0;
  }

  // Apply the decisions of one round (warp 0): lane k resolves live joint row
  // k from the C partial keys (a fixed-order max, so the result is independent
  // of arrival order), then lane s walks slot s's window in frame order (Alg. 3
  // lines 9-11 and 15-19 for each frame; TDT: blank advances by max(d, 1),
  // PAPER.md:213).  decide() also rebuilds the scanning list and checks the
  // speculative window.
  __device__ int resolve_rows_w0() {
    // TJ: the MMA warp read this round's row state for the speculative copies
    // and wrote their fbase / fcnt: done before warp 0 changes / reads them
    if (TJ && (phs & (1u << 13))) mbar_wait(bar(BAR_SPEC), (phs >> 12) & 1u);
    const uint64_t *pt = part(par());
    const int nz = rs.nz;
    int dec = 0;
    if (lane < nz) {
      uint64_t tkey = 0, dkey = 0;
      [[maybe_unused]] uint64_t tl = lse_empty(), dl = lse_empty();
#pragma unroll 16
      for (int r = 0; r < C; ++r) {
        const uint64_t *e = pt + ((size_t)r * L.JR + lane) * pks();
        if (is_tdt()) {
          const uint4 v = *reinterpret_cast<const uint4 *>(e);
          tkey = umax64(tkey, ((uint64_t)v.y << 32) | v.x);
          dkey = umax64(dkey, ((uint64_t)v.w << 32) | v.z);
          if constexpr (SC) {
            tl = lse_combine(tl, e[2]);
            dl = lse_combine(dl, e[3]);
          }
        } else {     // RNN-T: the token key only (+ its lse with scores)
          tkey = umax64(tkey, e[0]);
          if constexpr (SC) tl = lse_combine(tl, e[1]);
        }
      }
      dec = key_index(tkey) | ((is_tdt() ? key_index(dkey) : 0) << 24);
      if (!lean()) rs.dec[rs.zdst[lane]] = dec;
      if constexpr (SC) {   // log-probability of this row's decision (token [+ duration])
        float lp = key_value(tkey) - lse_value(tl);
        if (is_tdt()) lp += key_value(dkey) - lse_value(dl);
        rs.lp[rs.zdst[lane]] = lp;
      }
    }
    __syncwarp();
    return dec;   // lane k: decision of compact joint row k
  }

  // RNN-T decisions of a round without a per-slot loop: a ballot marks the
  // non-blank joint rows; slot s's window occupies compact rows zbeg[s] ..
  // zbeg[s] + zcnt[s] - 1 in frame order (plan_z), so its first non-blank frame
  // is the lowest set bit of that range (Alg. 3 lines 9-11 / 15-19 for every
  // frame of the window at once); `dec` is lane k's decision (resolve_rows_w0).
  __device__ void decide_rnnt(int dec, unsigned *algevals, int Xnext) {
    if (warp != 0) return;
    const int W = p.W;
    const unsigned nb = __ballot_sync(0xffffffffu, lane < rs.nz && (dec & 0xFFFFFF) != p.blank);
    const bool scan = lane < p.R && rs.scanning[lane];
    int b0 = 0, c = 0;
    unsigned m = 0;
    if (scan) {
      b0 = rs.zbeg[lane];
      c = rs.zcnt[lane];
      m = (nb >> b0) & ((1u << c) - 1u);   // c <= W <= 8
    }
    const bool found = m != 0u;
    const int pos = found ? __ffs(m) - 1 : c;
    const int y = __shfl_sync(0xffffffffu, dec, found ? b0 + pos : 0) & 0xFFFFFF;
    int used = scan ? (found ? pos + 1 : c) : 0;
    bool sc = false;
    if (scan) {
      const int s = lane, t0 = rs.t[s];
      if (found) {
        rs.found[s] = 1;
        rs.fy[s] = y;
        rs.ft[s] = t0 + pos;
        rs.fd[s] = 0;
      }
      rs.t[s] = t0 + pos;
      // the per-frame label counter restarts whenever t advanced (reading A6/A14)
      if (pos > 0 || !found) rs.k[s] = 0;
      if (!found) {
        if (t0 + pos >= rs.L[s]) rs.active[s] = 0;
        else sc = true;
      }
      rs.scanning[s] = sc;
    }
    const unsigned ms = __ballot_sync(0xffffffffu, sc);
    if (sc) rs.slist[__popc(ms & ((1u << lane) - 1u))] = lane;
    bool ok = true;
    if (sc) {
      const int s = lane;
      int need = rs.L[s] - rs.t[s];
      if (need > W) need = W;
      ok = Xnext >= 0 && rs.t[s] >= rs.fbase[Xnext][s] && rs.t[s] + need <= rs.fbase[Xnext][s] + rs.fcnt[Xnext][s];
    }
    const bool all_ok = __all_sync(0xffffffffu, ok);
    used = __reduce_add_sync(0xffffffffu, used);
    if (lane == 0) {
      rs.nscan = __popc(ms);
      rs.ready = all_ok;
      *algevals += (unsigned)used;
    }
    __syncwarp();
    if (all_ok && Xnext >= 0) plan_z(Xnext);
  }

  // Tick schedule, RNN-T: decide_rnnt(dec, algevals, -1) + append_found(false)
  // + rebuild_lists + the next predictor's E' fetch in one pass of warp 0, with
  // each row's state in lane s's registers (one shared-memory load and one
  // store per field instead of a store / reload chain across the phases).
  __device__ void finish_round_rnnt(int dec, unsigned *algevals, bool eprime) {
    const unsigned FULL = 0xffffffffu;
    const unsigned nb = __ballot_sync(FULL, lane < rs.nz && (dec & 0xFFFFFF) != p.blank);
    const bool inr = lane < p.R;
    int t = 0, k = 0, Ls = 0, len = 0, b = 0, b0 = 0, c = 0;
    bool act = false, scan = false, needp = false;
    if (inr) {
      t = rs.t[lane]; k = rs.k[lane]; Ls = rs.L[lane]; len = rs.len[lane]; b = rs.b[lane];
      act = rs.active[lane]; scan = rs.scanning[lane]; needp = rs.needp[lane];
      b0 = rs.zbeg[lane]; c = rs.zcnt[lane];
    }
    tl_sub(1);
    [[maybe_unused]] const int t_round = t;   // window base of this round (TJ: the speculative next window starts at t_round + W)
    // decisions of the window (Alg. 3 lines 9-11 / 15-19): first non-blank frame
    const unsigned m = scan ? (nb >> b0) & ((1u << c) - 1u) : 0u;   // c <= W <= 8
    const bool found = m != 0u;
    const int pos = found ? __ffs(m) - 1 : c;
    const int y = __shfl_sync(FULL, dec, found ? b0 + pos : 0) & 0xFFFFFF;
    const int used = scan ? (found ? pos + 1 : c) : 0;
    if constexpr (SC) {   // greedy score: every decision used (blanks included)
      float add = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j < used) add += rs.lp[lane * p.W + j];
      if (scan) rs.score[lane] += add;
    }
    if (scan) {
      t += pos;
      // the per-frame label counter restarts whenever t advanced (reading A6/A14)
      if (pos > 0 || !found) k = 0;
      scan = false;
      if (!found) {
        if (t >= Ls) act = false;
        else scan = true;
      }
    }
    // masked append (Alg. 3 line 21) + max-symbols guard
    if (found) {
      if (rank == 0) {
        if (len < p.cap) {
          p.out_tokens[(size_t)b * p.cap + len] = y;
          p.out_timestamps[(size_t)b * p.cap + len] = t;
          if (p.out_durations) p.out_durations[(size_t)b * p.cap + len] = 0;
        } else {
          atomicOr(p.status, 2);
        }
      }
      len += 1;
      k += 1;
      if (k == p.max_sym) {
        t += 1;
        k = 0;
      }
      act = t < Ls;
      needp = act;
    }
    if (inr) {
      rs.t[lane] = t; rs.k[lane] = k; rs.len[lane] = len;
      rs.active[lane] = act; rs.scanning[lane] = scan; rs.needp[lane] = needp;
      if (found) {
        rs.last[lane] = y;
#pragma unroll
        for (int cc = MAX_CTX - 1; cc > 0; --cc) rs.ctx[cc][lane] = rs.ctx[cc - 1][lane];
        rs.ctx[0][lane] = y;
      }
    }
    tl_sub(2);
    // compacted lists (ascending slot order) and counters
    const unsigned ms = __ballot_sync(FULL, inr && scan);
    const unsigned mp = __ballot_sync(FULL, inr && needp);
    const unsigned ma = __ballot_sync(FULL, inr && act);
    const unsigned below = (1u << lane) - 1u;
    if (inr && scan) rs.slist[__popc(ms & below)] = lane;
    if (inr && needp) rs.plist[__popc(mp & below)] = lane;
    const int tot = __reduce_add_sync(FULL, used);
    if (lane == 0) {
      rs.nscan = __popc(ms);
      rs.npred = __popc(mp);
      rs.nactive = __popc(ma);
      rs.ready = ms == 0u;
      *algevals += (unsigned)tot;
    }
    tl_sub(3);
    if constexpr (TJ) {
      plan_next_tj(inr && act && (scan || needp), t, Ls);
      tl_sub(4);
      // the next tick's reloads: rows that found a label, and scanning rows whose
      // speculative window (t_round + W) does not start at their new t (TDT jumps)
      const bool ld = inr && act && (needp || (scan && !(p.spec_prefetch && t == t_round + rs.wg)));
      const unsigned ml = __ballot_sync(FULL, ld);
      if (ld) rs.llist[__popc(ml & below)] = lane;
      if (lane == 0) rs.nload = __popc(ml);
    }
    __syncwarp();
    tl_sub(5);
    if (eprime && mp != 0u) {   // the next predictor's E'[y] slices, from the lanes' registers
      const uint32_t segb = (uint32_t)(4 * upc() * 4);
      if (lane == 0) mbar_arrive_expect_tx(bar(BAR_E), (uint32_t)__popc(mp) * segb);
      __syncwarp();
      if (inr && needp)
        bulk_g2s(es() + (size_t)lane * 4 * upc(), p.tab + (size_t)y * 4 * Pd() + (size_t)rank * 4 * upc(), segb,
                 bar(BAR_E));
    }
    tl_sub(6);
  }

  // Tick schedule: decide / decide_rnnt (Xnext = -1) + append_found +
  // rebuild_lists + the next predictor's E' fetch in one pass of warp 0, with
  // each row's state in lane s's registers (one shared-memory load and one
  // store per field instead of a store / reload chain across the phases).
  // TD (TDT): the window's decisions follow the duration chain t += max(d, 1)
  // (decide), a label with d > 0 advances t by d (append_found).  The RNN-T
  // kernels use finish_round_rnnt above (measured 0.5% faster than
  // finish_round<false>).
  template <bool TD>
  __device__ void finish_round(int dec, unsigned *algevals, bool eprime) {
    const unsigned FULL = 0xffffffffu;
    const bool inr = lane < p.R;
    int t = 0, k = 0, Ls = 0, len = 0, b = 0, b0 = 0, c = 0;
    bool act = false, scan = false, needp = false;
    if (inr) {
      t = rs.t[lane]; k = rs.k[lane]; Ls = rs.L[lane]; len = rs.len[lane]; b = rs.b[lane];
      act = rs.active[lane]; scan = rs.scanning[lane]; needp = rs.needp[lane];
      b0 = rs.zbeg[lane]; c = rs.zcnt[lane];
    }
    [[maybe_unused]] const int t_round = t;   // window base of this round (TJ: the speculative next window starts at t_round + W)
    // decisions of the window (Alg. 3 lines 9-11 / 15-19): first non-blank frame
    bool found = false;
    int pos = 0, y = 0, d = 0, used = 0;
    if constexpr (TD) {
      (void)dec; (void)b0; (void)c;
      if (scan) {
        const int W = rs.wg;   // logical rows s * W + j (plan_next_tj)
        [[maybe_unused]] float add = 0.f;
        while (pos < W && t + pos < Ls) {
          const int ee = rs.dec[lane * W + pos];
          const int yy = ee & 0xFFFFFF, dd = p.durations[ee >> 24];
          ++used;
          if constexpr (SC) add += rs.lp[lane * W + pos];
          if (yy != p.blank) {
            found = true;
            y = yy;
            d = dd;
            break;
          }
          pos += dd > 1 ? dd : 1;
        }
        if constexpr (SC) rs.score[lane] += add;
      }
    } else {
      const unsigned nb = __ballot_sync(FULL, lane < rs.nz && (dec & 0xFFFFFF) != p.blank);
      const unsigned m = scan ? (nb >> b0) & ((1u << c) - 1u) : 0u;   // c <= W <= 8
      found = m != 0u;
      pos = found ? __ffs(m) - 1 : c;
      y = __shfl_sync(FULL, dec, found ? b0 + pos : 0) & 0xFFFFFF;
      used = scan ? (found ? pos + 1 : c) : 0;
      if constexpr (SC) {
        float add = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (j < used) add += rs.lp[lane * rs.wg + j];
        if (scan) rs.score[lane] += add;
      }
    }
    if (scan) {
      t += pos;
      // the per-frame label counter restarts whenever t advanced (reading A6/A14)
      if (pos > 0 || !found) k = 0;
      scan = false;
      if (!found) {
        if (t >= Ls) act = false;
        else scan = true;
      }
    }
    // masked append (Alg. 3 line 21) + max-symbols guard
    if (found) {
      if (rank == 0) {
        if (len < p.cap) {
          p.out_tokens[(size_t)b * p.cap + len] = y;
          p.out_timestamps[(size_t)b * p.cap + len] = t;
          if (p.out_durations) p.out_durations[(size_t)b * p.cap + len] = d;
        } else {
          atomicOr(p.status, 2);
        }
      }
      len += 1;
      if (TD && d > 0) {
        t += d;
        k = 0;
      } else {
        k += 1;
        if (k == p.max_sym) {
          t += 1;
          k = 0;
        }
      }
      act = t < Ls;
      needp = act;
    }
    if (inr) {
      rs.t[lane] = t; rs.k[lane] = k; rs.len[lane] = len;
      rs.active[lane] = act; rs.scanning[lane] = scan; rs.needp[lane] = needp;
      if (found) {
        rs.last[lane] = y;
#pragma unroll
        for (int cc = MAX_CTX - 1; cc > 0; --cc)
          if (cc < p.context) rs.ctx[cc][lane] = rs.ctx[cc - 1][lane];   // stateless context > 1 only
        rs.ctx[0][lane] = y;
      }
    }
    // compacted lists (ascending slot order) and counters
    const unsigned ms = __ballot_sync(FULL, inr && scan);
    const unsigned mp = __ballot_sync(FULL, inr && needp);
    const unsigned ma = __ballot_sync(FULL, inr && act);
    const unsigned below = (1u << lane) - 1u;
    if (inr && scan) rs.slist[__popc(ms & below)] = lane;
    if (inr && needp) rs.plist[__popc(mp & below)] = lane;
    const int tot = __reduce_add_sync(FULL, used);
    if (lane == 0) {
      rs.nscan = __popc(ms);
      rs.npred = __popc(mp);
      rs.nactive = __popc(ma);
      rs.ready = ms == 0u;
      *algevals += (unsigned)tot;
    }
    if constexpr (TJ) {
      plan_next_tj(inr && act && (scan || needp), t, Ls);
      // the next tick's reloads: rows that found a label, and scanning rows whose
      // speculative window (t_round + W) does not start at their new t (TDT jumps)
      const bool ld = inr && act && (needp || (scan && !(p.spec_prefetch && t == t_round + rs.wg)));
      const unsigned ml = __ballot_sync(FULL, ld);
      if (ld) rs.llist[__popc(ml & below)] = lane;
      if (lane == 0) rs.nload = __popc(ml);
    }
    __syncwarp();
    if (eprime && mp != 0u) issue_eprime(rs.plist, __popc(mp));
  }

  __device__ void decide(unsigned *algevals, int Xnext) {
    if (warp != 0) return;
    const int W = p.W;
    int used = 0;
    bool sc = false;
    // walk each slot's window (decisions resolved by resolve_rows)
    if (lane < p.R && rs.scanning[lane]) {
      const int s = lane;
      const int t0 = rs.t[s], Ls = rs.L[s];
      int pos = 0;
      bool found = false;
      while (pos < W && t0 + pos < Ls) {
        const int ee = rs.dec[s * W + pos];
        const int y = ee & 0xFFFFFF, d = is_tdt() ? p.durations[ee >> 24] : 0;
        ++used;
        if (y != p.blank) {
          rs.found[s] = 1;
          rs.fy[s] = y;
          rs.ft[s] = t0 + pos;
          rs.fd[s] = d;
          found = true;
          break;
        }
        pos += is_tdt() ? (d > 1 ? d : 1) : 1;
      }
      rs.t[s] = t0 + pos;
      // the per-frame label counter restarts whenever t advanced (reading A6/A14)
      if (pos > 0 || !found) rs.k[s] = 0;
      if (!found) {
        if (rs.t[s] >= Ls) rs.active[s] = 0;
        else sc = true;
      }
      rs.scanning[s] = sc;
    }
    // rebuild the scanning list (ascending slot order) and check that the
    // speculative window in fbuf[Xnext] covers every row that keeps scanning
    const unsigned ms = __ballot_sync(0xffffffffu, sc);
    if (sc) rs.slist[__popc(ms & ((1u << lane) - 1u))] = lane;
    bool ok = true;
    if (sc) {
      const int s = lane;
      int need = rs.L[s] - rs.t[s];
      if (need > W) need = W;
      ok = Xnext >= 0 && rs.t[s] >= rs.fbase[Xnext][s] && rs.t[s] + need <= rs.fbase[Xnext][s] + rs.fcnt[Xnext][s];
    }
    const bool all_ok = __all_sync(0xffffffffu, ok);
    for (int o = 16; o > 0; o >>= 1) used += __shfl_xor_sync(0xffffffffu, used, o);
    if (lane == 0) {
      rs.nscan = __popc(ms);
      rs.ready = all_ok;
    }
    if (lane == 0) *algevals += (unsigned)used;
    __syncwarp();
    // the next round's joint-row plan (only valid if the window is ready)
    if (all_ok && Xnext >= 0) plan_z(Xnext);
  }

  // Frame-looping baseline (Alg. 2), warp 0: the one-frame
  // decisions of a round at the common frame t.  Blank -> the row is done with
  // this frame; label -> append (t), predictor update before the row's next
  // evaluation, k += 1, and after the m-th label the row is done with this frame
  // without a blank evaluation (guard, reading A6).
  __device__ void decide_fl(unsigned *algevals) {
    if (warp != 0) return;
    int used = 0;
    if (lane < p.R && rs.scanning[lane]) {
      const int s = lane;
      const int y = rs.dec[s * p.W] & 0xFFFFFF;
      used = 1;
      if (y == p.blank) {
        rs.scanning[s] = 0;
      } else {
        const int pos = rs.len[s];
        if (rank == 0) {
          if (pos < p.cap) {
            p.out_tokens[(size_t)rs.b[s] * p.cap + pos] = y;
            p.out_timestamps[(size_t)rs.b[s] * p.cap + pos] = rs.t[s];
          } else {
            atomicOr(p.status, 2);
          }
        }
        rs.len[s] = pos + 1;
        rs.last[s] = y;
        for (int c = MAX_CTX - 1; c > 0; --c) rs.ctx[c][s] = rs.ctx[c - 1][s];
        rs.ctx[0][s] = y;
        rs.needp[s] = 1;
        rs.k[s] += 1;
        if (rs.k[s] == p.max_sym) rs.scanning[s] = 0;
      }
    }
    used = __reduce_add_sync(0xffffffffu, used);
    if (lane == 0) *algevals += (unsigned)used;
    __syncwarp();
  }

  // Append + time rules + guard for the slots that found a label this round
  // (BatchedHyps.add_results; readings A6, A13, A14): warp 0,
  // lane = slot.  The slot then needs a predictor update before it scans again.
  __device__ void append_found(bool tdt) {
    if (warp != 0 || lane >= p.R) return;
    const int s = lane;
    if (!rs.found[s]) return;
    const int b = rs.b[s];
    const int pos = rs.len[s];
    if (rank == 0) {
      if (pos < p.cap) {
        p.out_tokens[(size_t)b * p.cap + pos] = rs.fy[s];
        p.out_timestamps[(size_t)b * p.cap + pos] = rs.ft[s];
        if (p.out_durations) p.out_durations[(size_t)b * p.cap + pos] = rs.fd[s];
      } else {
        atomicOr(p.status, 2);
      }
    }
    rs.len[s] = pos + 1;
    if (tdt && rs.fd[s] > 0) {
      rs.t[s] += rs.fd[s];
      rs.k[s] = 0;
    } else {
      rs.k[s] += 1;
      if (rs.k[s] == p.max_sym) {
        rs.t[s] += 1;
        rs.k[s] = 0;
      }
    }
    rs.active[s] = rs.t[s] < rs.L[s];
    rs.needp[s] = rs.active[s];
    rs.last[s] = rs.fy[s];
    for (int c = MAX_CTX - 1; c > 0; --c) rs.ctx[c][s] = rs.ctx[c - 1][s];
    rs.ctx[0][s] = rs.fy[s];
    rs.found[s] = 0;
  }

  // warp 0: rebuild the compacted scanning / predictor lists (ascending slot order)
  // GUARDED: the counters are written only when they change, for call sites
  // where other warps may still be reading them (no barrier since their last
  // read); the hot per-tick sites follow a CTA barrier and write unguarded.
  template <bool GUARDED = true>
  __device__ void rebuild_lists() {
    if (warp == 0) {
      const bool sc = lane < p.R && rs.scanning[lane];
      const bool pr = lane < p.R && rs.needp[lane];
      const bool ac = lane < p.R && rs.active[lane];
      const unsigned ms = __ballot_sync(0xffffffffu, sc);
      const unsigned mp = __ballot_sync(0xffffffffu, pr);
      const unsigned ma = __ballot_sync(0xffffffffu, ac);
      const unsigned below = (1u << lane) - 1u;
      if (sc) rs.slist[__popc(ms & below)] = lane;
      if (pr) rs.plist[__popc(mp & below)] = lane;
      if constexpr (GUARDED) {   // one lane per counter: the three compares are one load
        if (lane < 3) {
          int *cnt = lane == 0 ? &rs.nscan : lane == 1 ? &rs.npred : &rs.nactive;
          const int v = __popc(lane == 0 ? ms : lane == 1 ? mp : ma);
          if (*cnt != v) *cnt = v;
        }
      } else if (lane == 0) {
        rs.nscan = __popc(ms);
        rs.npred = __popc(mp);
        rs.nactive = __popc(ma);
      }
    }
  }

  // -------------------------------------------------------------------------
  // bf16 LSTM predictor.  Tile sequence of one step (identical every step):
  //   n_local in [0, NG):        W_hh rows {gate*P + u0 + 2n + c/4 : gate = c%4}, c < 8
  //   n_local in [NG, NG + NPT): W_pred rows d0 + 8(n - NG) + c
  // A producer warp streams the tiles through the NS-slot ring (bulk copies);
  // consumer warp w takes tiles w, w + NW, ... of each phase.
  // -------------------------------------------------------------------------
  __device__ int ng() const { return upc() / 2; }
  __device__ int npt() const { return dpc() / 8; }

  // W_hh tile PAIRS: pair pp (units u0 + 4pp .. u0 + 4pp + 3) is two 8-row
  // tiles, half 0 = gates (i, f) and half 1 = gates (g, o), row c of a half =
  // unit 4pp + c/2, gate 2*half + (c & 1) (packed by pack_lstm_stream).
  // Pair pp belongs to warp pp % NW; a warp can only reach TMEM lane quarter
  // warp % 4, so the quarter's columns are shared by its warps: the warp's m-th
  // pair (m = pp / NW) sits in pair slot m * nq + warp / 4 (2 * tcols columns).
  // Thread (g, q) holds, for every 32-wide K block kb, the m16 A fragments of
  // the pair interleaved in columns 8kb..8kb+7: (h0.x, h1.x, h0.y, h1.y, h0.z,
  // h1.z, h0.w, h1.w), h0/h1 = the 16-byte chunk 4kb + q of row g of half 0/1,
  // so each fragment is 4 consecutive registers of one tcgen05.ld (+4 columns
  // for a 16-wide tail).
  __device__ int tcols() const { return 4 * (Pd() / 32) + ((Pd() & 31) ? 2 : 0); }
  __device__ int npairs() const { return upc() / 4; }
  __device__ int quarter_warps(int qd) const { return (NW - qd + 3) / 4; }
  __device__ uint32_t pair_taddr(int pp) const {
    const int w = pp % NW, qd = w & 3;
    const int slot = (pp / NW) * quarter_warps(qd) + (w >> 2);
    return tmem + ((uint32_t)(32 * qd) << 16) + (uint32_t)(slot * 2 * tcols());
  }

  // Kernel start: W_hh tiles of this CTA from the packed stream into TMEM,
  // W_pred tiles into shared memory (one bulk copy).
  __device__ void load_lstm_weights() {
    if constexpr (TG) {
      // W_hh rows of this CTA's 40 units into TMEM in the A-operand layout (TG_*
      // above): warps 0-3 the main rows of lane quarter q = warp (unit 8q +
      // lane/4, gate lane%4), warps 4-7 the K-quarter j = warp - 4 of the folded
      // rows (unit 32 + lane/4, gate lane%4); one 32-bit column = 2 bf16 K elements
      if (warp < 8) {
        const int qd = warp & 3;
        const bool fold = warp >= 4;
        const int unit = (fold ? 32 : 8 * qd) + (lane >> 2), gate = lane & 3;
        const bf16 *src = (const bf16 *)p.w_hh + ((size_t)gate * TG_P + u0 + unit) * TG_P + (fold ? (TG_P / 4) * qd : 0);
        const uint32_t ta = tmem + ((uint32_t)(32 * qd) << 16) + (fold ? TG_COL_FOLD : 0u);
        const int ncols = fold ? TG_P / 8 : TG_P / 2;
        for (int c0 = 0; c0 < ncols; c0 += 16) {
          uint32_t r[16];
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const uint4 x = ldg128_nc(src + 2 * c0 + 8 * v);
            r[4 * v] = x.x; r[4 * v + 1] = x.y; r[4 * v + 2] = x.z; r[4 * v + 3] = x.w;
          }
          tmem_st16(ta + (uint32_t)c0, r);
        }
      }
      tmem_wait_st();
      // W_pred into registers: warp w's K blocks kb = w, w + 10 (16-byte chunk
      // 4 kb + q) of rows 16t + g (tile 2t) and 16t + 8 + g (tile 2t + 1)
      if (warp < NW) {
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int t = 0; t < 3; ++t)
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
              const int row = 16 * t + 8 * hf + g, kb = warp + MAX_NW * i;
              wpr[i][t][hf] = (row < TG_UPC && kb < TG_P / 32)
                                  ? ldg128_nc((const bf16 *)p.w_pred + (size_t)(d0 + row) * TG_P + (4 * kb + q) * 8)
                                  : make_uint4(0, 0, 0, 0);
            }
      }
      return;
    }
    const int NG = ng(), NPT = npt(), KB = Pd() / 32;
    const int sw = ((g & 1) && (Pd() % 64) == 0) ? 4 : 0;
    for (int n = 2 * warp; n < NG; n += 2 * NW) {   // stream tiles n (half 0), n + 1 (half 1) = pair n / 2
      const uint32_t ta = pair_taddr(n / 2);
      const uint8_t *row0 =
          reinterpret_cast<const uint8_t *>(p.wst + (((size_t)rank * (NG + NPT) + n) * 8 + g) * Pd());
      const uint8_t *row1 = row0 + (size_t)8 * Pd() * 2;
      for (int c2 = 0; c2 < KB; c2 += 2) {
        uint32_t r[16];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int kb = c2 + u;
          uint4 v0 = make_uint4(0, 0, 0, 0), v1 = make_uint4(0, 0, 0, 0);
          if (kb < KB) {
            v0 = ldg128_nc(row0 + (((kb * 4 + q) ^ sw) * 16));
            v1 = ldg128_nc(row1 + (((kb * 4 + q) ^ sw) * 16));
          }
          r[8 * u + 0] = v0.x; r[8 * u + 1] = v1.x; r[8 * u + 2] = v0.y; r[8 * u + 3] = v1.y;
          r[8 * u + 4] = v0.z; r[8 * u + 5] = v1.z; r[8 * u + 6] = v0.w; r[8 * u + 7] = v1.w;
        }
        if (c2 + 2 <= KB) {
          tmem_st16(ta + 8 * c2, r);
        } else {   // odd last block: 8 columns
          asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta + 8 * c2),
                       "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                       : "memory");
        }
      }
      if (Pd() & 31) {
        const uint2 v0 = ldg64_nc(row0 + KB * 64 + q * 8), v1 = ldg64_nc(row1 + KB * 64 + q * 8);
        asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(ta + 8 * KB), "r"(v0.x),
                     "r"(v1.x), "r"(v0.y), "r"(v1.y)
                     : "memory");
      }
    }
    tmem_wait_st();
    if (warp == 0) {
      const uint32_t bytes = (uint32_t)(NPT * 8 * Pd() * 2);
      if (lane == 0) {
        mbar_arrive_expect_tx(bar(BAR_FULL), bytes);
        bulk_g2s(ringslot(0), p.wst + ((size_t)rank * (NG + NPT) + NG) * 8 * Pd(), bytes, bar(BAR_FULL));
      }
      mbar_wait(bar(BAR_FULL), 0);
    }
  }

  // Gate GEMM of W_hh tile pair pp against NB groups of 8 predictor rows, as
  // m16n8k16 MMAs with the WEIGHTS as the A operand (16 gate rows: half 0 ->
  // rows 0-7, half 1 -> rows 8-15) and h as the B operand (8 rows per group),
  // so one MMA covers 16 gate rows of <= 8 predictor rows.  A fragments come
  // from TMEM (tcgen05.ld, both halves of a 4-block chunk, one wait), B
  // fragments from shared memory (one 16-byte load per row and K block, the K
  // permutation of common.cuh).  Two accumulator chains over K, summed by the
  // caller in a fixed order.
  template <int NB>
  __device__ __forceinline__ void gates_pair(float (&acc)[NB][2][4], int pp, const uint8_t *const *hrow) const {
    const int KB = Pd() / 32;
    const uint32_t ta = pair_taddr(pp);
#pragma unroll 1
    for (int c4 = 0; c4 < KB; c4 += 4) {
      uint32_t r[32];
      if (c4 + 4 <= KB) {
        tmem_ld32(ta + 8 * c4, r);
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (c4 + u < KB) {
            uint32_t t[8];
            tmem_ld8(ta + 8 * (c4 + u), t);
#pragma unroll
            for (int e = 0; e < 8; ++e) r[8 * u + e] = t[e];
          }
        }
      }
      tmem_wait_ld();
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int kb = c4 + u;
        if (kb < KB) {
#pragma unroll
          for (int nb = 0; nb < NB; ++nb) {
            const uint4 x = lds128(hrow[nb] + kb * 64);
            mma_bf16_16816(acc[nb][u & 1], r[8 * u], r[8 * u + 1], r[8 * u + 2], r[8 * u + 3], x.x, x.y);
            mma_bf16_16816(acc[nb][u & 1], r[8 * u + 4], r[8 * u + 5], r[8 * u + 6], r[8 * u + 7], x.z, x.w);
          }
        }
      }
    }
    if (Pd() & 31) {   // 16-wide K tail: lane q owns columns [4q, 4q + 4) of the block
      uint4 t;
      tmem_ld4(ta + 8 * KB, t);
      tmem_wait_ld();
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) {
        const uint2 x = lds64(hrow[nb] + KB * 64 - q * 8);
        mma_bf16_16816(acc[nb][0], t.x, t.y, t.z, t.w, x.x, x.y);
      }
    }
  }

  // W_pred part of the predictor: partial g = W_pred[this CTA's rows, K blocks
  // of this warp] h' for NB groups of 8 rows.  A = W_pred m-tiles (tiles 2t,
  // 2t+1 of the resident smem copy, rows >= DPC read as zero), B = h' rows.
  // K blocks are split over the warps: warp w takes kb = w, w + NW, ... (and
  // warp 0 the 16-wide tail).
  // hrow[nb]: the row's chunk-q address (hsrow + q * 16), or (TG) the h
  // buffer + 16 * slot (chunk offsets from hoff).
  template <int NB>
  __device__ __forceinline__ void wpred_partial(float (&acc)[3][NB][4], const uint8_t *const *hrow) const {
    const int KB = Pd() / 32, NPT = npt();
    const int sw = ((g & 1) && (Pd() % 64) == 0) ? 4 : 0;
#pragma unroll
    for (int t = 0; t < 3; ++t)
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) acc[t][nb][0] = acc[t][nb][1] = acc[t][nb][2] = acc[t][nb][3] = 0.f;
#pragma unroll
    for (int i = 0; i < (KB + MAX_NW - 1) / MAX_NW; ++i) {   // K blocks warp, warp + NW, ...
      const int kb = warp + i * NW;
      if (kb >= KB) break;
      uint4 x[NB];
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) {
        if constexpr (TG) x[nb] = lds128(hrow[nb] + hoff(0, 4 * kb + q));
        else x[nb] = lds128(hrow[nb] + kb * 64);
      }
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        if (2 * t < NPT) {
          uint4 wa, wb;
          if constexpr (TG) {
            wa = wpr[i][t][0];
            wb = wpr[i][t][1];
          } else {
            const uint32_t co = (uint32_t)(((kb * 4 + q) ^ sw) * 16);
            wa = lds128(ringslot(2 * t) + (size_t)g * Pd() * 2 + co);
            wb = 2 * t + 1 < NPT ? lds128(ringslot(2 * t + 1) + (size_t)g * Pd() * 2 + co) : make_uint4(0, 0, 0, 0);
          }
#pragma unroll
          for (int nb = 0; nb < NB; ++nb) {
            mma_bf16_16816(acc[t][nb], wa.x, wb.x, wa.y, wb.y, x[nb].x, x[nb].y);
            mma_bf16_16816(acc[t][nb], wa.z, wb.z, wa.w, wb.w, x[nb].z, x[nb].w);
          }
        }
      }
    }
    if ((Pd() & 31) && warp == 0) {
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        if (2 * t < NPT) {
          const uint2 wa = lds64(ringslot(2 * t) + (size_t)g * Pd() * 2 + KB * 64 + q * 8);
          const uint2 wb = 2 * t + 1 < NPT ? lds64(ringslot(2 * t + 1) + (size_t)g * Pd() * 2 + KB * 64 + q * 8)
                                           : make_uint2(0, 0);
#pragma unroll
          for (int nb = 0; nb < NB; ++nb) {
            const uint2 x = lds64(hrow[nb] + KB * 64 - q * 8);
            mma_bf16_16816(acc[t][nb], wa.x, wb.x, wa.y, wb.y, x.x, x.y);
          }
        }
      }
    }
  }

  // broadcast `nbytes16` 16-byte chunks starting at local smem `src` (same
  // offset in every CTA) to the other CTAs, completing tx on barrier `bi`.
  __device__ void bcast_rows(const uint8_t *base, int row_stride, int col_off, int row_bytes, int nrows,
                             const int *rows, int bi) {
    const int chunks = row_bytes / 16;
    const int total = nrows * chunks * (C - 1);
    const uint32_t bb = smem_u32(bar(bi));
    for (int idx = tid; idx < total; idx += NCT) {
      const int d = idx % (C - 1), rem = idx / (C - 1);
      const int c = rem % chunks, i = rem / chunks;
      const int dst = (rank + 1 + d) % C;
      const uint8_t *src = base + (size_t)rows[i] * row_stride + col_off + c * 16;
      const uint4 v = *reinterpret_cast<const uint4 *>(src);
      const uint32_t la = smem_u32(src);
      st_async_u64x2(mapa_u32(la, (uint32_t)dst), ((uint64_t)v.y << 32) | v.x, ((uint64_t)v.w << 32) | v.z,
                     mapa_u32(bb, (uint32_t)dst));
    }
  }

  // Gate epilogue for n8 row group nb of pair pp: the two chains summed, gates
  // of a unit paired across lanes g and g ^ 1 (one shuffle each way), the cell
  // update (PyTorch LSTM, reading A9) for predictor row 8nb + 2q (even g) or
  // 8nb + 2q + 1 (odd g): c' = s(f) c + s(i) tanh(g), h' = s(o) tanh(c').
  __device__ __forceinline__ void gate_epilogue(const float (&a)[2][4], int pp, int nb, int n) const {
    float v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) v[e] = a[0][e] + a[1][e];
    const bool ev = (g & 1) == 0;
    // even g holds (i, g) of rows 2q, 2q+1; odd g holds (f, o)
    const float r0 = __shfl_xor_sync(0xffffffffu, ev ? v[1] : v[0], 4);
    const float r1 = __shfl_xor_sync(0xffffffffu, ev ? v[3] : v[2], 4);
    const int i = 8 * nb + 2 * q + (ev ? 0 : 1);
    if (i < n) {
      const int ul = 4 * pp + (g >> 1);                 // unit within this CTA's slice
      const int s = rs.plist[i];
      const float *ep = es() + (size_t)s * 4 * upc() + ul;
      const float gi = (ev ? v[0] : r0) + ep[0];
      const float gf = (ev ? r0 : v[1]) + ep[upc()];
      const float gg = (ev ? v[2] : r1) + ep[2 * upc()];
      const float go = (ev ? r1 : v[3]) + ep[3 * upc()];
      float *cp = cs() + (size_t)s * upc() + ul;
      const float cn = sigmoidf_(gf) * *cp + sigmoidf_(gi) * tanhf(gg);
      *cp = cn;
      reinterpret_cast<bf16 *>(hsrow(rs.hpar[s] ^ 1, s))[u0 + ul] = __float2bfloat16_rn(sigmoidf_(go) * tanhf(cn));
    }
  }

  // Gate GEMM + epilogue for row groups nb0 .. nb0 + NB - 1 (NB <= 2 per pass
  // keeps the accumulators and both TMEM fragments in registers).
  template <int NB>
  __device__ __forceinline__ void gates_all(int n, int nb0, bool &e_ready) {
    const uint8_t *hrow[NB];
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) {
      const int i = 8 * (nb0 + nb) + g;
      const int s = rs.plist[i < n ? i : 0];
      hrow[nb] = hsrow(rs.hpar[s], s) + q * 16;
    }
    for (int pp = warp; pp < npairs(); pp += NW) {
      float acc[NB][2][4];
#pragma unroll
      for (int nb = 0; nb < NB; ++nb)
#pragma unroll
        for (int c = 0; c < 2; ++c) acc[nb][c][0] = acc[nb][c][1] = acc[nb][c][2] = acc[nb][c][3] = 0.f;
      gates_pair<NB>(acc, pp, hrow);
      if (pp == warp && nb0 == 0) tl_pred(1);
      if (!e_ready) {
        mbar_wait(bar(BAR_E), hph());
        e_ready = true;
      }
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) gate_epilogue(acc[nb], pp, nb0 + nb, n);
    }
  }

  // Partial W_pred products of NB row groups (rows 8*nb0 ...) -> shared memory
  // (the z region, idle during the predictor): wpart[warp][t][nb][lane][4].
  template <int NB>
  __device__ __forceinline__ void wpred_store(int nb0, int n) {
    const uint8_t *hrow[NB];
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) {
      const int i = 8 * (nb0 + nb) + g;
      const int s = rs.plist[i < n ? i : 0];
      if constexpr (TG) hrow[nb] = hbuf() + 16 * s;
      else hrow[nb] = hsrow(rs.hpar[s] ^ 1, s) + q * 16;
    }
    float acc[3][NB][4];
    wpred_partial<NB>(acc, hrow);
    if constexpr (TG) {   // (NB = 1) partials as P[warp][row i][dim d] (row stride 44: conflict-free)
      float *P = reinterpret_cast<float *>(zs()) + warp * 8 * 44;
#pragma unroll
      for (int t = 0; t < 3; ++t)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int d = 16 * t + g + 8 * (e >> 1), i = 2 * q + (e & 1);
          if (d < TG_UPC) P[i * 44 + d] = acc[t][0][e];
        }
      return;
    }
    float4 *wp = reinterpret_cast<float4 *>(zs());
#pragma unroll
    for (int t = 0; t < 3; ++t)
#pragma unroll
      for (int nb = 0; nb < NB; ++nb)
        wp[((warp * 3 + t) * 2 + nb) * 32 + lane] = make_float4(acc[t][nb][0], acc[t][nb][1], acc[t][nb][2],
                                                                acc[t][nb][3]);
  }

  // E'[y] slices (this CTA's 4 x UPC gate inputs) of `n` slots into es[slot]
  // by one bulk copy each, completing on BAR_E (one warp; lane 0 arms it).
  // The E' table's columns are CTA-major, so each slice is contiguous.
  __device__ void issue_eprime(const int *slots, int n) {
    const uint32_t segb = (uint32_t)(4 * upc() * 4);
    if (lane == 0) mbar_arrive_expect_tx(bar(BAR_E), (uint32_t)n * segb);
    __syncwarp();
    if (lane < n) {
      const int s = slots[lane];
      bulk_g2s(es() + (size_t)s * 4 * upc(), p.tab + (size_t)rs.last[s] * 4 * Pd() + (size_t)rank * 4 * upc(), segb,
               bar(BAR_E));
    }
  }

  // eprefetched: the E' slices of this step were issued when the labels were
  // decided (tick schedule); otherwise they are fetched here.
  __device__ void predictor_lstm_tmem(bool eprefetched = false) {
    tl_pred(0);
    const int n = rs.npred;
    const int P = Pd(), H = Hd();

    // arm the h' / g exchange barriers for this step (tx from the other CTAs)
    if (tid == 0 && C > 1) {
      mbar_arrive_expect_tx(bar(BAR_H), (uint32_t)((C - 1) * n * upc() * 2));
      if (!OTF) mbar_arrive_expect_tx(bar(BAR_G), (uint32_t)((C - 1) * n * dpc() * 4));
    }
    // (1) gates = E'[y] + W_hh h; fused cell update for this CTA's units.
    // E'[y_i] slices of this CTA's units (4 gates x UPC floats per row) are
    // staged into shared memory by bulk copies that overlap the gate GEMM.
    // (the table's columns are CTA-major: one bulk copy per predictor row)
    if (!eprefetched && warp == NW - 1) issue_eprime(rs.plist, n);
    if constexpr (TG) {
      // W_hh h from the background gate batch (zero on the group's first step)
      gate_wait();
      tc_fence_after();
      const bool dvalid = (phs >> 10) & 1u;
      float *gb = reinterpret_cast<float *>(zs());   // [40 units][36]: gate g at 8g + slot (main units)
      float *fb = gb + TG_UPC * 36;                  // [4 quarters][8 units][4 gates][8 slots] (fold partials)
      if (warp < 8) {
        uint32_t r[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        const int qd = warp & 3;
        if (dvalid) {
          tmem_ld8(tmem + ((uint32_t)(32 * qd) << 16) + (warp < 4 ? TG_COL_DMAIN : TG_COL_DFOLD + 8u * qd), r);
          tmem_wait_ld();
        }
        float *dst = warp < 4 ? gb + (8 * qd + (lane >> 2)) * 36 + (lane & 3) * 8 : fb + (qd * 32 + lane) * 8;
        reinterpret_cast<float4 *>(dst)[0] = make_float4(__uint_as_float(r[0]), __uint_as_float(r[1]),
                                                         __uint_as_float(r[2]), __uint_as_float(r[3]));
        reinterpret_cast<float4 *>(dst)[1] = make_float4(__uint_as_float(r[4]), __uint_as_float(r[5]),
                                                         __uint_as_float(r[6]), __uint_as_float(r[7]));
      }
      tc_fence_before();
      mbar_wait(bar(BAR_E), hph());
      sync();
      tl_pred(1);
      // cell update, one thread per (unit, slot): gates = E'[y] + W_hh h (the
      // folded units sum their 4 K-quarter partials in a fixed order), PyTorch
      // LSTM (reading A9): c' = s(f) c + s(i) tanh(g), h' = s(o) tanh(c')
      {
        const int ul = tid >> 3, s = tid & 7;
        if (s < p.R && rs.needp[s]) {
          float gt[4];
          if (ul < 32) {
#pragma unroll
            for (int gg = 0; gg < 4; ++gg) gt[gg] = gb[ul * 36 + gg * 8 + s];
          } else {
#pragma unroll
            for (int gg = 0; gg < 4; ++gg) {
              const int row = ((ul - 32) * 4 + gg) * 8 + s;
              gt[gg] = ((fb[row] + fb[256 + row]) + fb[512 + row]) + fb[768 + row];
            }
          }
          const float *ep = es() + (size_t)s * 4 * TG_UPC + ul;
          float *cp = cs() + (size_t)s * TG_UPC + ul;
          const float gi = gt[0] + ep[0], gf = gt[1] + ep[TG_UPC], gg = gt[2] + ep[2 * TG_UPC],
                      go = gt[3] + ep[3 * TG_UPC];
          const float cn = sigmoidf_(gf) * *cp + sigmoidf_(gi) * tanhf_(gg);
          *cp = cn;
          const int k = u0 + ul;
          *reinterpret_cast<bf16 *>(hbuf() + hoff(s, k >> 3) + (k & 7) * 2) = __float2bfloat16_rn(sigmoidf_(go) * tanhf_(cn));
        }
      }
      tl_pred(2);
      sync();
      tl_pred_bar(3);
      // h' slices (this CTA's 5 chunks of every predicted row) to every other CTA
      if (C > 1) {
        const int total = n * 5 * (C - 1);
        const uint32_t bb = smem_u32(bar(BAR_H));
        for (int idx = tid; idx < total; idx += NCT) {
          const int d = idx % (C - 1), rem = idx / (C - 1);
          const int c = 5 * rank + rem % 5, s = rs.plist[rem / 5];
          const uint8_t *src = hbuf() + hoff(s, c);
          const uint4 v = *reinterpret_cast<const uint4 *>(src);
          const uint32_t dst = (uint32_t)((rank + 1 + d) % C);
          st_async_u64x2(mapa_u32(smem_u32(src), dst), ((uint64_t)v.y << 32) | v.x, ((uint64_t)v.w << 32) | v.z,
                         mapa_u32(bb, dst));
        }
        mbar_wait(bar(BAR_H), hph());
      }
      // the h buffer (local writes + the other CTAs' st.async) -> async proxy
      fence_proxy_async_smem();
      tl_pred(4);
    } else {
    {
      bool e_ready = false;
      for (int nb0 = 0; nb0 * 8 < n; nb0 += 2) {
        if (n - nb0 * 8 > 8) gates_all<2>(n, nb0, e_ready);
        else gates_all<1>(n, nb0, e_ready);
      }
      if (!e_ready) mbar_wait(bar(BAR_E), hph());  // keep every thread's view of the phase in step
    }
    tl_pred(2);
    // (2) exchange the h' slices (this CTA's units) with every CTA
    sync();
    tl_pred_bar(3);
    if (C > 1) {
      // rows: slot ids; the destination row is the slot's NEXT parity
      if (tid < n) {
        const int s = rs.plist[tid];
        rs.zsrc[tid] = (rs.hpar[s] ^ 1) * p.R + s;  // row index into hs
      }
      sync();
      bcast_rows(sm + L.off_hs, hstride(), u0 * 2, upc() * 2, n, rs.zsrc, BAR_H);
      mbar_wait(bar(BAR_H), hph());
    }
    tl_pred(4);
    }
    if constexpr (OTF) {   // no g: the rounds apply W_pred themselves (project_z)
      sync();              // h' complete in every thread's view (fence.proxy.async above)
      gate_request();      // W_hh h' for the next step, in the background
      phs ^= 1u << 6;
      tl_next_step();
      return;
    }
    // (3) g = W_pred h' + b_pred for this CTA's output dims: K split over the
    // warps (partials in shared memory), then one thread per (row, 4 dims)
    // sums the partials in a fixed warp order, adds the bias, stores g locally
    // and st.async's it to every other CTA (completing tx on their BAR_G).
    const uint32_t bg = smem_u32(bar(BAR_G));
    for (int nb0 = 0; nb0 * 8 < n; nb0 += 2) {
      if (n - nb0 * 8 > 8) wpred_store<2>(nb0, n);
      else wpred_store<1>(nb0, n);
      if (nb0 == 0) tl_pred(9);
      sync();
      if (nb0 == 0) tl_pred_bar(10);
      if constexpr (TG) {
        if (nb0 == 0) gate_request();   // W_hh h' for the next step, in the background
      }
      const int nrows = min(16, n - nb0 * 8);
      const int D4 = dpc() / 4;
      const float4 *wp = reinterpret_cast<const float4 *>(zs());
      if constexpr (TG) {   // one thread per (row, 4 dims): 10 float4 partials in a fixed warp order
        if (tid < nrows * D4) {
          const int i = tid / D4, d = (tid % D4) * 4;
          const float *P = reinterpret_cast<const float *>(zs()) + i * 44 + d;
          float4 pw[MAX_NW];
#pragma unroll
          for (int w = 0; w < MAX_NW; ++w) pw[w] = *reinterpret_cast<const float4 *>(P + w * 8 * 44);
          float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int w = 0; w < MAX_NW; ++w) {
            acc.x += pw[w].x; acc.y += pw[w].y; acc.z += pw[w].z; acc.w += pw[w].w;
          }
          const float4 bp = *reinterpret_cast<const float4 *>(bsl() + 72 + d);   // b_pred slice (smem)
          const float o0 = acc.x + bp.x, o1 = acc.y + bp.y, o2 = acc.z + bp.z, o3 = acc.w + bp.w;
          const int s = rs.plist[i];
          float *dst = gs() + (size_t)s * H + goff(d0 + d);
          *reinterpret_cast<float4 *>(dst) = make_float4(o0, o1, o2, o3);
          const uint64_t lo = ((uint64_t)__float_as_uint(o1) << 32) | __float_as_uint(o0);
          const uint64_t hi2 = ((uint64_t)__float_as_uint(o3) << 32) | __float_as_uint(o2);
          const uint32_t la = smem_u32(dst);
#pragma unroll 16
          for (int c = 1; c < C; ++c) {
            const uint32_t dr = (uint32_t)((rank + c) % C);
            st_async_u64x2(mapa_u32(la, dr), lo, hi2, mapa_u32(bg, dr));
          }
        }
      } else
      for (int idx = tid; idx < nrows * D4; idx += NCT) {
        const int ii = idx / D4, d = (idx % D4) * 4;    // row within the pass, first of 4 dims
        const int i = nb0 * 8 + ii, nb = ii >> 3, il = ii & 7;
        const int t = d >> 4, hi = (d >> 3) & 1, gq = d & 7, qq = il >> 1, e = hi * 2 + (il & 1);
        float out[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int ln = (gq + j) * 4 + qq;
          float part[MAX_NW];
#pragma unroll
          for (int w = 0; w < MAX_NW; ++w)   // all loads first, then a fixed-order sum
            part[w] = w < NW ? reinterpret_cast<const float *>(wp + ((w * 3 + t) * 2 + nb) * 32 + ln)[e] : 0.f;
          float acc = 0.f;
#pragma unroll
          for (int w = 0; w < MAX_NW; ++w) acc += part[w];
          out[j] = acc + __bfloat162float(((const bf16 *)p.b_pred)[d0 + d + j]);
        }
        const int s = rs.plist[i];
        float *dst = gs() + (size_t)s * H + goff(d0 + d);
        *reinterpret_cast<float4 *>(dst) = make_float4(out[0], out[1], out[2], out[3]);
        const uint64_t lo = ((uint64_t)__float_as_uint(out[1]) << 32) | __float_as_uint(out[0]);
        const uint64_t hi2 = ((uint64_t)__float_as_uint(out[3]) << 32) | __float_as_uint(out[2]);
        const uint32_t la = smem_u32(dst);
#pragma unroll 16
        for (int c = 1; c < C; ++c) {
          const uint32_t dr = (uint32_t)((rank + c) % C);
          st_async_u64x2(mapa_u32(la, dr), lo, hi2, mapa_u32(bg, dr));
        }
      }
      sync();   // partial buffer reused by the next pass
    }
    tl_pred_bar(5);
    tl_pred_bar(6);
    // (4) the other CTAs' g slices
    if (C > 1) mbar_wait(bar(BAR_G), hph());
    phs ^= 1u << 6;
    if (!TG && warp == 0 && lane < n) {
      const int s = rs.plist[lane];
      rs.hpar[s] ^= 1;
    }
    sync();
    tl_pred_bar(7);
    tl_next_step();
  }

  // -------------------------------------------------------------------------
  // fp32 predictor (LL_F32): SIMT, h / g through global memory + cluster barriers.
  // -------------------------------------------------------------------------
  __device__ __forceinline__ void warp_dot_f32(float (&acc)[MAX_R], const float *wr, int K, int M) const {
    const float *z = (const float *)zs();
    const int zst = zstride() / 4;
#pragma unroll
    for (int i = 0; i < MAX_R; ++i) acc[i] = 0.f;
    for (int k = lane; k < K; k += 32) {
      const float w = __ldg(wr + k);
#pragma unroll
      for (int i = 0; i < MAX_R; ++i)
        if (i < M) acc[i] = fmaf(w, z[(size_t)i * zst + k], acc[i]);
    }
#pragma unroll
    for (int i = 0; i < MAX_R; ++i) {
      if (i < M) {
        float s = acc[i];
        s += __shfl_xor_sync(0xffffffffu, s, 16);
        s += __shfl_xor_sync(0xffffffffu, s, 8);
        s += __shfl_xor_sync(0xffffffffu, s, 4);
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        acc[i] = s;
      }
    }
  }

  // h rows of layer `layer` ([layers][2][B][P] in global memory) into z rows 0..n-1
  __device__ void load_h_rows_f32(int n, int which /*0: current hpar, 1: next*/, int layer = 0) {
    const int P = Pd();
    float *z = (float *)zs();
    const int zst = zstride() / 4;
    for (int idx = tid; idx < n * P; idx += NCT) {
      const int i = idx / P, c = idx % P;
      const int s = rs.plist[i];
      float v = 0.f;
      if (!(which == 0 && rs.hzero[s])) {
        const int hp = which == 0 ? rs.hpar[s] : (rs.hpar[s] ^ 1);
        v = __ldcg((const float *)p.h + (((size_t)layer * 2 + hp) * p.B + rs.b[s]) * P + c);
      }
      z[(size_t)i * zst + c] = v;
    }
    sync();
  }

  __device__ void predictor_lstm_f32() {
    const int n = rs.npred, P = Pd(), H = Hd();
    const float *tab = p.tab;
    load_h_rows_f32(n, 0);
    for (int uu = warp; uu < upc(); uu += NW) {
      const int unit = u0 + uu;
      float mine[4] = {0.f, 0.f, 0.f, 0.f};
      float acc[MAX_R];
#pragma unroll
      for (int gi = 0; gi < 4; ++gi) {
        warp_dot_f32(acc, (const float *)p.w_hh + ((size_t)gi * P + unit) * P, P, n);
#pragma unroll
        for (int i = 0; i < MAX_R; ++i)
          if (lane == i) mine[gi] = acc[i];
      }
      if (lane < n) {
        const int s = rs.plist[lane];
        const int y = rs.last[s];
        float gate[4];
#pragma unroll
        for (int gi = 0; gi < 4; ++gi) gate[gi] = mine[gi] + tab[(size_t)y * 4 * P + (size_t)gi * P + unit];
        float *cp = cs() + (size_t)s * upc() + uu;
        const float cn = sigmoidf_(gate[1]) * *cp + sigmoidf_(gate[0]) * tanhf(gate[2]);
        *cp = cn;
        ((float *)p.h)[((size_t)(rs.hpar[s] ^ 1) * p.B + rs.b[s]) * P + unit] = sigmoidf_(gate[3]) * tanhf(cn);
      }
    }
    __threadfence();
    if (C > 1) cluster_sync_all(); else sync();
    // layers 2..L (PyTorch nn.LSTM stacking, reading A9): x = the new h of the
    // layer below; gates = (W_ih x + b_ih) + (W_hh h + b_hh), the input side
    // first into shared memory, then the recurrent side and the cell update
    for (int layer = 1; layer < p.layers; ++layer) {
      const size_t lw = (size_t)(layer - 1) * 4 * P;
      const float *wih = (const float *)p.w_ih_rest + lw * P, *whh = (const float *)p.w_hh_rest + lw * P;
      const float *bih = (const float *)p.b_ih_rest + lw, *bhh = (const float *)p.b_hh_rest + lw;
      float *part = es();   // [slot i][gate][unit] input-side partials
      load_h_rows_f32(n, 1, layer - 1);
      for (int uu = warp; uu < upc(); uu += NW) {
        const int unit = u0 + uu;
#pragma unroll
        for (int gi = 0; gi < 4; ++gi) {
          float acc[MAX_R];
          warp_dot_f32(acc, wih + ((size_t)gi * P + unit) * P, P, n);
#pragma unroll
          for (int i = 0; i < MAX_R; ++i)
            if (i < n && lane == i) part[((size_t)i * 4 + gi) * upc() + uu] = acc[i] + bih[gi * P + unit];
        }
      }
      sync();
      load_h_rows_f32(n, 0, layer);
      for (int uu = warp; uu < upc(); uu += NW) {
        const int unit = u0 + uu;
        float mine[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int gi = 0; gi < 4; ++gi) {
          float acc[MAX_R];
          warp_dot_f32(acc, whh + ((size_t)gi * P + unit) * P, P, n);
#pragma unroll
          for (int i = 0; i < MAX_R; ++i)
            if (lane == i) mine[gi] = acc[i];
        }
        if (lane < n) {
          const int s = rs.plist[lane];
          float gate[4];
#pragma unroll
          for (int gi = 0; gi < 4; ++gi)
            gate[gi] = part[((size_t)lane * 4 + gi) * upc() + uu] + (mine[gi] + bhh[gi * P + unit]);
          float *cp = cs() + ((size_t)layer * p.R + s) * upc() + uu;
          const float cn = sigmoidf_(gate[1]) * *cp + sigmoidf_(gate[0]) * tanhf(gate[2]);
          *cp = cn;
          ((float *)p.h)[(((size_t)layer * 2 + (rs.hpar[s] ^ 1)) * p.B + rs.b[s]) * P + unit] = sigmoidf_(gate[3]) * tanhf(cn);
        }
      }
      __threadfence();
      if (C > 1) cluster_sync_all(); else sync();
    }
    load_h_rows_f32(n, 1, p.layers - 1);
    for (int dd = warp; dd < dpc(); dd += NW) {
      const int d = d0 + dd;
      float acc[MAX_R];
      warp_dot_f32(acc, (const float *)p.w_pred + (size_t)d * P, P, n);
      const float bv = ((const float *)p.b_pred)[d];
#pragma unroll
      for (int i = 0; i < MAX_R; ++i)
        if (i < n && lane == i) p.gglob[(size_t)rs.b[rs.plist[i]] * H + d] = acc[i] + bv;
    }
    __threadfence();
    if (C > 1) cluster_sync_all(); else sync();
    for (int idx = tid; idx < n * H; idx += NCT) {
      const int i = idx / H, c = idx % H;
      const int s = rs.plist[i];
      gs()[(size_t)s * H + c] = __ldcg(p.gglob + (size_t)rs.b[s] * H + c);
    }
    sync();
    if (warp == 0 && lane < n) {
      const int s = rs.plist[lane];
      rs.hpar[s] ^= 1;
      rs.hzero[s] = 0;
    }
    sync();
  }

  __device__ void predictor_stateless() {
    const int n = rs.npred, H = Hd(), V1 = p.V1;
    const int c4 = H / 4;
    for (int idx = tid; idx < n * c4; idx += NCT) {
      const int i = idx / c4, c = idx % c4;
      const int s = rs.plist[i];
      float4 acc = *reinterpret_cast<const float4 *>(p.tab + (size_t)rs.ctx[0][s] * H + c * 4);
      for (int kk = 1; kk < p.context; ++kk) {
        const float4 v = *reinterpret_cast<const float4 *>(p.tab + ((size_t)kk * V1 + rs.ctx[kk][s]) * H + c * 4);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
      *reinterpret_cast<float4 *>(gs() + (size_t)s * H + goff(c * 4)) = acc;
    }
    sync();   // every warp is done with plist / npred before warp 0 rebuilds the lists
  }

  // -------------------------------------------------------------------------
  // Group index broadcast without a cluster barrier: rank 0 takes the next
  // group from the work counter and st.async's it to every CTA (BAR_GRP+gp);
  // every CTA acknowledges to rank 0 (BAR_ACK+gp), and rank 0 reuses a
  // broadcast buffer only after all acknowledgements of its previous use.
  // -------------------------------------------------------------------------
  __device__ int next_group(int k) {
    const int gp = k & 1;
    const uint32_t ph = (uint32_t)((k >> 1) & 1);
    if (tid == 0) {
      mbar_arrive_expect_tx(bar(BAR_GRP + gp), 4);
      if (rank == 0) {
        if (k >= 2) mbar_wait(bar(BAR_ACK + gp), ph ^ 1u);
        mbar_arrive_expect_tx(bar(BAR_ACK + gp), (uint32_t)(4 * C));
        const int gi = atomicAdd(p.group_counter, 1);
        const uint32_t slot = smem_u32(&rs.grp[gp]), bb = smem_u32(bar(BAR_GRP + gp));
        for (int r = 0; r < C; ++r) st_async_u32(mapa_u32(slot, (uint32_t)r), (uint32_t)gi, mapa_u32(bb, (uint32_t)r));
      }
    }
    mbar_wait(bar(BAR_GRP + gp), ph);
    const int grp = rs.grp[gp];
    sync();
    if (tid == 0) {
      const uint32_t slot = smem_u32(&rs.ack[gp]), bb = smem_u32(bar(BAR_ACK + gp));
      st_async_u32(mapa_u32(slot, 0), 1u, mapa_u32(bb, 0));
    }
    return grp;
  }
  __device__ void final_acks(int k) {
    // rank 0 waits for the acknowledgements of the last two broadcasts
    if (rank == 0 && tid == 0) {
      for (int kk = k - 1; kk <= k; ++kk)
        if (kk >= 0) mbar_wait(bar(BAR_ACK + (kk & 1)), (uint32_t)((kk >> 1) & 1));
    }
  }
};

// ---------------------------------------------------------------------------
// W_ih / b_ih / b_hh with the 4P gate rows in CTA-major order: row
// r*4*UPC + gate*UPC + ul  <-  gate*P + r*UPC + ul (the E' table GEMM then
// produces, per vocabulary row, one contiguous 4*UPC-float slice per CTA).
// ---------------------------------------------------------------------------
__global__ void permute_gate_rows(const bf16 *w_ih, const bf16 *b_ih, const bf16 *b_hh, bf16 *w_out, bf16 *bi_out,
                                  bf16 *bh_out, int P, int C, int UPC) {
  const int chunks = P / 8;
  const long long total = (long long)4 * P * chunks;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(i % chunks);
    const int dst = (int)(i / chunks);
    const int r = dst / (4 * UPC), gate = (dst / UPC) % 4, ul = dst % UPC;
    const int src = gate * P + r * UPC + ul;
    reinterpret_cast<uint4 *>(w_out + (size_t)dst * P)[j] = reinterpret_cast<const uint4 *>(w_ih + (size_t)src * P)[j];
    if (j == 0) {
      bi_out[dst] = b_ih[src];
      bh_out[dst] = b_hh[src];
    }
  }
}

// ---------------------------------------------------------------------------
// Pack the bf16 LSTM weights into the per-CTA tile stream: for cluster rank r,
// tiles n < NG are W_hh tile pairs (n = 2 * pair + half): row c is unit
// r*UPC + 4*pair + c/2, gate 2*half + (c & 1) (gate order i, f, g, o); tiles
// NG + k are W_pred rows r*DPC + 8k + c.  Rows are stored unpadded; in odd rows
// the 16-byte chunk j is stored at j ^ 4 (bank swizzle).  One thread per
// 16-byte chunk.
// ---------------------------------------------------------------------------
__global__ void pack_lstm_stream(const bf16 *w_hh, const bf16 *w_pred, bf16 *wst, int P, int C, int UPC, int DPC) {
  const int NG = UPC / 2, NPT = DPC / 8, NT = NG + NPT;
  const int chunks = P / 8;
  const long long total = (long long)C * NT * 8 * chunks;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(i % chunks);
    const long long rowid = i / chunks;
    const int c = (int)(rowid % 8);
    const int n = (int)((rowid / 8) % NT);
    const int r = (int)(rowid / (8 * NT));
    const bf16 *src;
    if (n < NG) src = w_hh + ((size_t)(2 * (n & 1) + (c & 1)) * P + r * UPC + 4 * (n >> 1) + (c >> 1)) * P;
    else src = w_pred + (size_t)(r * DPC + 8 * (n - NG) + c) * P;
    const int jd = (c & 1) && (P % 64) == 0 ? (j ^ 4) : j;
    reinterpret_cast<uint4 *>(wst + (size_t)rowid * P)[jd] = reinterpret_cast<const uint4 *>(src)[j];
  }
}

// ---------------------------------------------------------------------------
// The decode kernel.  PRED: 0 = LSTM, 1 = stateless.
// ---------------------------------------------------------------------------
// LM (loop mode): 0 = label-looping, schedule chosen at run time (p.sched);
// 1 = label-looping, per-row ticks only; 2 = label-looping, the batched outer
// loop of Alg. 3 only; 3 = the frame-looping baseline (Alg. 2).  Separate
// instantiations, so a kernel carries only the control code it runs.
// TM: 0 = RNN-T / TDT chosen at run time (p.tdt), 1 = RNN-T only, 2 = TDT only
// (the FC instantiations carry only the code of their model family).
// DBG: 1 = the probe hook (ll.h ll_options): the same kernel also writes the
// logits of every joint row and g after every predictor step (parity tests).
// SC: 1 = greedy scores (N2), per-row tick schedule only.
template <typename T, int PRED, int KR, int HC = 0, int PC = 0, int CC = 0, int LM = 0, int TM = 0, int DBG = 0,
          int SC = 0>
__global__ void __launch_bounds__(MAX_NW * 32 + (sizeof(T) == 2 && HC == TJ_H && PC == TJ_H && CC == TJ_C ? 32 : 0), 1)
    decode_kernel(const __grid_constant__ DecodeParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ RowState rs;
  __shared__ __align__(8) uint64_t s_bars[NBARS];
  // LM: 0 runtime schedule (p.sched), 1 per-row ticks, 2 Alg. 3 batched outer
  // loop, 3 frame-looping baseline (Alg. 2), 4 per-row ticks with on-the-fly
  // projections (OTF, FC LSTM only)
  using CtxT = Ctx<T, KR, HC, PC, CC, TM, SC, (LM == 4 ? 1 : 0)>;
  static_assert(LM != 4 || (PRED == 0 && CtxT::TG && SC == 0 && DBG == 0), "OTF: the FC LSTM tick kernel only");
  CtxT cx(p, smem, rs, PRED == 0, s_bars);
  // TJ: an 11th warp issues the tcgen05 joint (and, LSTM, the background gate
  // batches), outside the consumer barrier
  constexpr bool MMAW = CtxT::TJ;
  constexpr bool TGK = PRED == 0 && CtxT::TG;
  const bool tdt = TM == 0 ? p.tdt != 0 : TM == 2;
  const int C = cx.C, rank = cx.rank, tid = cx.tid, lane = cx.lane, warp = cx.warp;
  const int R = p.R;
  constexpr bool RING = sizeof(T) == 2 && PRED == 0;
  // statistics: counted by thread 0 only, in shared memory (no registers held)
  __shared__ unsigned s_cnt[SC_N];
  if (tid < SC_N) s_cnt[tid] = 0;
  const bool t0 = tid == 0;
  if constexpr (MMAW) {   // the swizzled operands need a 1024-byte aligned base (uniform: every CTA alike)
    if (smem_u32(smem) & 1023u) {
      if (tid == 0 && rank == 0) atomicOr(p.status, 4);
      return;
    }
    if (warp == MAX_NW - 1 && lane == 0 && p.fmap_ok)
      asm volatile("prefetch.tensormap [%0];" ::"l"(&p.fmap) : "memory");
  }

  __shared__ uint32_t s_tmem;
  cx.init_barriers();
  cx.load_weight_slice();
  if constexpr (RING || MMAW) {
    if (warp == 0) tmem_alloc(&s_tmem, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    cx.tmem = s_tmem;
    if constexpr (RING) cx.load_lstm_weights();
    tc_fence_before();
  }
  __syncthreads();
  if (C > 1) cluster_sync_all();  // barriers initialised cluster-wide before any st.async
  if constexpr (RING || MMAW) tc_fence_after();

  if (MMAW && warp == MAX_NW) {
    cx.mma_warp_loop();
  } else {
    int cur = 0;                  // f buffer of the current round
#ifndef LL_DEBUG_TRACE
#define LL_PHASE(k)
#else
#define LL_PHASE(k)                              \
  if (p.trace && tid == 0) {                     \
    p.trace[blockIdx.x * 8 + 0] = (k);           \
    p.trace[blockIdx.x * 8 + 1] = s_cnt[SC_ROUNDS];    \
    p.trace[blockIdx.x * 8 + 2] = s_cnt[SC_OUTER];     \
    p.trace[blockIdx.x * 8 + 3] = (unsigned)k_grp;     \
    p.trace[blockIdx.x * 8 + 4] = (unsigned)rs.nz;     \
    p.trace[blockIdx.x * 8 + 5] = (unsigned)rs.nscan;  \
    p.trace[blockIdx.x * 8 + 6] = cx.phs | ((unsigned)cur << 16); \
  }
#endif

    int k = 0, k_grp = 0;
    for (;; ++k) {
      const int grp = cx.next_group(k);
      k_grp = grp;
      if (grp >= p.n_groups) break;
      if (t0) s_cnt[SC_GROUPS]++;
      // ---- group init (warp 0: lane = row slot) -----------------------------
      int gb = grp * R + lane, gsize = R;   // this slot's utterance, the group's size
      if (warp == 0 && p.perm != nullptr && gb < p.B) gb = p.perm[gb];
      if (warp == 0) {
        if (p.gp_small > 0) {
          // unequal groups: utterance i (lane i, B <= 32) ranked by (length desc, i)
          int Li = 0;
          if (lane < p.B) {
            Li = p.lengths[lane];
            if (Li < 0 || Li > p.T_max) Li = 0;
          }
          int rk = 0;
          for (int j = 0; j < p.B; ++j) {
            const int Lj = __shfl_sync(0xffffffffu, Li, j);
            rk += (Lj > Li || (Lj == Li && j < lane)) ? 1 : 0;
          }
          const int xs = p.gp_small, rsz = p.gp_rsmall;
          const int start = grp < xs ? grp * rsz : xs * rsz + (grp - xs) * R;
          gsize = grp < xs ? rsz : R;
          if (lane < p.B && rk >= start && rk < start + gsize) rs.zsrc[rk - start] = lane;   // scratch
          __syncwarp();
          gb = lane < gsize ? rs.zsrc[lane] : p.B;
          __syncwarp();
          if (lane == 0) rs.wg = grp < xs ? p.gp_wsmall : p.W;
        } else if (lane == 0) {
          rs.wg = p.W;
        }
      }
      if (warp == 0 && lane < R) {
        const int b = lane < gsize ? gb : p.B;
        int L = 0;
        if (b < p.B) {
          L = p.lengths[b];
          if (L < 0 || L > p.T_max) {
            if (rank == 0) atomicOr(p.status, 1);
            L = 0;
          }
        }
        rs.b[lane] = b < p.B ? b : p.B;   // p.B: no utterance in this slot (never addressed: L = 0)
        rs.L[lane] = L;
        rs.t[lane] = 0; rs.k[lane] = 0; rs.len[lane] = 0;
        rs.last[lane] = p.blank;
        rs.hpar[lane] = 0; rs.hzero[lane] = 1;
        for (int c = 0; c < MAX_CTX; ++c) rs.ctx[c][lane] = p.blank;
        rs.active[lane] = L > 0;
        rs.needp[lane] = L > 0;
        rs.scanning[lane] = 0;
        rs.found[lane] = 0;
        rs.score[lane] = 0.f;
      }
      if constexpr (DBG != 0) {   // test hook: skew the cluster's CTAs at group starts
        if (p.probe_stall > 0 && (rank & 1)) {
          const long long c0 = clock64();
          while (clock64() - c0 < p.probe_stall) {
          }
        }
      }
      if constexpr (PRED == 0) {
        // LSTM initial state h = c = 0 (reading A8)
        for (int i = tid; i < R * cx.L.UPC * max(p.layers, 1); i += cx.NCT) cx.cs()[i] = 0.f;
        if constexpr (TGK) {
          // h = 0 means W_hh h = 0: the group's first step skips the
          // pre-activations (bit 10 cleared) and writes h' of every active
          // slot.  The h buffer is NOT zeroed here: the other CTAs may already
          // be st.async'ing this group's first h' slices into it (they only
          // wait for the group index), and no reader uses an inactive slot's
          // h (its gate / W_pred columns are never read)
          cx.gate_wait();
          cx.phs &= ~(1u << 10);
        } else if constexpr (RING) {
          for (int i = tid; i < R * cx.Pd() / 8; i += cx.NCT) {
            const int s = i / (cx.Pd() / 8), c = i % (cx.Pd() / 8);
            *reinterpret_cast<uint4 *>(cx.hsrow(0, s) + c * 16) = make_uint4(0, 0, 0, 0);
          }
        }
      }
      __syncwarp();
      cx.rebuild_lists();
      cx.sync();

      // ---- frame-looping baseline (Alg. 2): frames in lockstep ----------------
      if constexpr (LM == 3) {
        if (warp == 0 && lane < R) rs.scanning[lane] = rs.active[lane];
        __syncwarp();
        cx.rebuild_lists();
        cx.sync();
        while (rs.nactive > 0) {
          if (t0) s_cnt[SC_OUTER]++;
          if (rs.npred > 0) {          // rows that emitted a label: predictor update
            if (t0) {
              s_cnt[SC_PRED]++;
              s_cnt[SC_PREDROWS] += rs.npred;
            }
            if constexpr (PRED == 1) cx.predictor_stateless();
            else if constexpr (RING) cx.predictor_lstm_tmem();
            else cx.predictor_lstm_f32();
            if (warp == 0 && lane < R) rs.needp[lane] = 0;
            __syncwarp();
          }
          if (rs.nscan == 0) {         // every row is done with frame t: t += 1 for all (line 22)
            cx.sync();                 // every warp has read the counters rebuilt below
            if (warp == 0 && lane < R && rs.active[lane]) {
              rs.t[lane] += 1;
              rs.k[lane] = 0;
              rs.active[lane] = rs.t[lane] < rs.L[lane];
              rs.scanning[lane] = rs.active[lane];
            }
            __syncwarp();
            cx.rebuild_lists();
            cx.sync();
            continue;
          }
          // one joint round at frame t for the rows still scanning it (lines 7-8 / 18-19)
          if (cx.fpend(cur)) cur ^= 1;
          cx.issue_f(cur, false);
          cx.sync();
          cx.wait_f(cur);
          cx.plan_z(cur);
          cx.sync();
          cx.build_z(cur);
          cx.sync();
          cx.joint_keys((rs.nz + 15) / 16, 0, nullptr, 0);
          cx.exchange_keys();
          if (warp == 0) {
            cx.exchange_wait();
            if (t0) {
              s_cnt[SC_ROUNDS]++;
              s_cnt[SC_ROWEVALS] += rs.nz;
            }
            cx.resolve_rows_w0();
            cx.decide_fl(s_cnt + SC_ALGEVALS);
          }
          cx.flip_par();
          cx.sync();
          cx.rebuild_lists();
          cx.sync();
        }
      } else
      // ---- per-row schedule (exact reordering of Alg. 3, utterances being
      // independent): a TICK runs the predictor for the rows that found a label
      // in the previous tick, then one joint round for every row that scans
      // (continuing rows and the rows just updated).  A row never waits for the
      // other rows of its group to find their labels.
      if (LM == 1 || LM == 4 || (LM == 0 && p.sched == 1)) {
        if (warp == 0 && lane < R) {
          rs.scanning[lane] = 0;
          rs.found[lane] = 0;
        }
        __syncwarp();
        cx.rebuild_lists();
        __syncwarp();
        if constexpr (RING) {          // SOS inputs of the first predictor step
          if (warp == 0 && rs.npred > 0) cx.issue_eprime(rs.plist, rs.npred);
        }
        if constexpr (CtxT::TJ) {      // the first round's plan and windows (every active row scans from t = 0)
          if (warp == 0) {
            const bool act0 = lane < R && rs.active[lane];
            cx.plan_next_tj(act0, 0, lane < R ? rs.L[lane] : 0);
            const unsigned ml = __ballot_sync(0xffffffffu, act0);
            if (act0) rs.llist[__popc(ml & ((1u << lane) - 1u))] = lane;
            if (lane == 0) rs.nload = __popc(ml);
          }
        }
        cx.sync();
        bool have_spec = false;        // fbuf[cur ^ 1] holds the previous tick's speculative windows
        [[maybe_unused]] int dbg_l = 0, dbg_gr = 0;   // probe rows written by this cluster
        while (rs.nactive > 0) {
          if (t0) s_cnt[SC_OUTER]++;
          cx.tl_pred(11);
          if (have_spec) {
            cx.wait_f(cur ^ 1);
            cur ^= 1;
          }
          // (1) windows: a continuing row whose speculative window starts at its t
          // reuses it; every other row about to scan gets a fresh window
          // (TJ: the reload list was made with the decisions, finish_round*)
          if (CtxT::TJ && rs.nload > 0) cx.reload_f(cur);
          if (!CtxT::TJ && warp == 0) {
            bool ld = false;
            if (lane < R) {
              const int s = lane;
              const bool cont = rs.scanning[s], np = rs.needp[s];
              const bool reuse = have_spec && cont && rs.fbase[cur][s] == rs.t[s];
              ld = (cont || np) && !reuse;
            }
            const unsigned ml = __ballot_sync(0xffffffffu, ld);
            if (ld) rs.llist[__popc(ml & ((1u << lane) - 1u))] = lane;
            if (lane == 0) rs.nload = __popc(ml);
          }
          if constexpr (!CtxT::TJ) {
            cx.sync();
            cx.tl_pred_bar(12);
            if (rs.nload > 0) cx.issue_f(cur, false, rs.llist, rs.nload);
          }
          cx.tl_pred_bar(8);
          // (2) predictor (Alg. 3 line 6) for the rows that found a label
          if (rs.npred > 0) {
            if (t0) {
              s_cnt[SC_PRED]++;
              s_cnt[SC_PREDROWS] += rs.npred;
            }
            if constexpr (PRED == 1) cx.predictor_stateless();
            else if constexpr (RING) cx.predictor_lstm_tmem(true);
            else cx.predictor_lstm_f32();
            if constexpr (DBG != 0) {    // probe: g rows of the predicted slots (rank 0 writes)
              const int n = rs.npred, H = cx.Hd(), region = blockIdx.x / C;
              if (rank == 0) {
                for (int idx = tid; idx < n * H; idx += cx.NCT) {
                  const int i = idx / H, d = idx % H, row = dbg_gr + i;
                  if (row < p.probe_rows)
                    p.probe_g[((size_t)region * p.probe_rows + row) * H + d] =
                        cx.gs()[(size_t)rs.plist[i] * H + cx.goff(d & ~3) + (d & 3)];
                }
                if (tid < n && dbg_gr + tid < p.probe_rows) {
                  const int s = rs.plist[tid];
                  *reinterpret_cast<int4 *>(p.probe_gmeta + ((size_t)region * p.probe_rows + dbg_gr + tid) * 4) =
                      make_int4(rs.b[s], rs.len[s], 0, 0);
                }
                if (t0) p.probe_counts[2 * region + 1] = dbg_gr + n;
              }
              dbg_gr += n;
              cx.sync();
            }
            // the predicted rows scan from now on (with no predictor rows the
            // lists are unchanged, and rewriting the counters here would race
            // with the other warps' read of npred above: no barrier separates them)
            if (warp == 0 && lane < R) {
              rs.scanning[lane] = rs.scanning[lane] || rs.needp[lane];
              rs.needp[lane] = 0;
            }
            __syncwarp();
            cx.template rebuild_lists<false>();   // after the predictor's / round's barriers
          }
          if (cx.fpend(cur)) cx.wait_f(cur);
          cx.tl_pred(13);
          cx.sync();
          have_spec = false;
          if (rs.nscan > 0) {
            // (3) one joint round (Alg. 3 lines 7-19 over a W-frame window)
            cx.tl_round_(0);
            if constexpr (!CtxT::TJ) {   // TJ: planned with the previous decisions (plan_next_tj)
              cx.plan_z(cur);
              cx.sync();
            }
            cx.tl_round_bar(1);
#ifdef LL_EXP1
            cx.gate_wait();   // experiment: no gate batch in flight during build_z
            cx.sync();
            cx.tl_round_bar(1);
#endif
            if constexpr (LM == 4) cx.project_z(cur);
            else cx.build_z(cur, CtxT::TJ);
            cx.tl_round_(2);
            cx.sync();
            cx.tl_round_bar(15);
            if (p.spec_prefetch) {
              cx.spec_issue(cur ^ 1);
              have_spec = true;
            }
            cx.tl_round_bar(3);
            if constexpr (DBG != 0) {    // probe: logits + (b, t, labels so far) of every joint row
              const int nz = rs.nz, NV = p.V1 + p.nD, region = blockIdx.x / C;
              if (rank == 0 && warp == 0 && lane < nz && dbg_l + lane < p.probe_rows) {
                const int s = rs.zdst[lane] / p.W, j = rs.zdst[lane] % p.W;
                *reinterpret_cast<int4 *>(p.probe_lmeta + ((size_t)region * p.probe_rows + dbg_l + lane) * 4) =
                    make_int4(rs.b[s], rs.t[s] + j, rs.len[s], 0);
              }
              if (rank == 0 && t0) p.probe_counts[2 * region] = dbg_l + nz;
              cx.joint_keys((nz + 15) / 16, max(0, min(nz, p.probe_rows - dbg_l)),
                            p.probe_logits + (size_t)region * p.probe_rows * NV, dbg_l);
              dbg_l += nz;
            } else {
              cx.joint_keys((rs.nz + 15) / 16, 0, nullptr, 0);
            }
            cx.tl_round_(4);
            cx.exchange_keys();
            cx.tl_round_(5);
            if (warp == 0) {
              cx.exchange_wait();
              cx.tl_round_(6);
              if (t0) {
                s_cnt[SC_ROUNDS]++;
                s_cnt[SC_ROWEVALS] += rs.nz;
              }
              const int dec = cx.resolve_rows_w0();
              cx.tl_round_(7);
              cx.tl_round_(8);
              // decide + append + list rebuild + next predictor's E' fetch
              // (after the predictor's / round's barriers)
              if (tdt) cx.template finish_round<true>(dec, s_cnt + SC_ALGEVALS, RING);
              else cx.finish_round_rnnt(dec, s_cnt + SC_ALGEVALS, RING);
              cx.tl_round_(9);
            }
            cx.flip_par();
            cx.sync();
            cx.tl_round_bar(10);
            cx.tl_next_round();
          }
        }
      } else
      // ---- outer loop over labels (Alg. 3 line 5) -----------------------------
      while (rs.nactive > 0) {
        if (t0) s_cnt[SC_OUTER]++;
        if (warp == 0 && lane < R) {
          rs.scanning[lane] = rs.active[lane];
          rs.found[lane] = 0;
        }
        __syncwarp();
        cx.rebuild_lists();
        cx.sync();
        // first window of every active row, overlapping the predictor phase
        if (cx.fpend(cur)) cur ^= 1;
        cx.issue_f(cur, false);
        cx.sync();                     // fbase/fcnt (written by the issuing warp) visible to warp 0
        LL_PHASE(11);
        cx.tl_pred_bar(8);
        // predictor (Alg. 3 line 6): only rows that found a label and stay active
        if (rs.npred > 0) {
          if (t0) {
            s_cnt[SC_PRED]++;
            s_cnt[SC_PREDROWS] += rs.npred;
          }
          if constexpr (PRED == 1) cx.predictor_stateless();
          else if constexpr (RING) cx.predictor_lstm_tmem();
          else cx.predictor_lstm_f32();
        }
        LL_PHASE(10);
        // ---- frame loop: rounds of W-frame windows until no row scans ---------
        bool planned = false;          // first round: plan after the predictor phase
        while (rs.nscan > 0) {
          cx.tl_round_(0);
          cx.wait_f(cur);
          if (!planned) {
            cx.plan_z(cur);
            cx.sync();                 // plan visible, predictor's g written
          }
          LL_PHASE(0);
          cx.tl_round_bar(1);
          cx.build_z(cur);
          LL_PHASE(1);
          cx.tl_round_(2);
          cx.sync();
          // speculative: a row whose window is all blank needs the next window
          if (p.spec_prefetch) cx.spec_issue(cur ^ 1);
          LL_PHASE(2);
          cx.tl_round_bar(3);
          cx.joint_keys((rs.nz + 15) / 16, 0, nullptr, 0);
          LL_PHASE(3);
          cx.tl_round_(4);
          cx.exchange_keys();
          LL_PHASE(4);
          cx.tl_round_(5);
          if (warp == 0) {
            // warp 0 alone: cross-CTA argmax, decisions, next round's plan
            cx.exchange_wait();
            LL_PHASE(5);
            cx.tl_round_(6);
            if (t0) {
              s_cnt[SC_ROUNDS]++;
              s_cnt[SC_ROWEVALS] += rs.nz;
            }
            const int dec = cx.resolve_rows_w0();
            cx.tl_round_(7);
            cx.tl_round_(8);
            if (tdt) cx.decide(s_cnt + SC_ALGEVALS, p.spec_prefetch ? (cur ^ 1) : -1);
            else cx.decide_rnnt(dec, s_cnt + SC_ALGEVALS, p.spec_prefetch ? (cur ^ 1) : -1);
            LL_PHASE(8);
            cx.tl_round_(9);
          }
          cx.flip_par();
          cx.sync();
          planned = false;
          if (rs.nscan > 0) {
            cur ^= 1;
            // TDT may jump past the prefetched frames (or no speculation): reload
            if (!rs.ready) {
              cx.issue_f(cur, false);
              cx.sync();                 // fbase/fcnt visible to warp 0's plan_z
            } else {
              planned = true;            // decide() planned the next round from fbuf[cur]
            }
          } else if (p.spec_prefetch) {
            cur ^= 1;                    // the other buffer holds a stale speculative copy
          }
          LL_PHASE(9);
          cx.tl_round_bar(10);
          cx.tl_next_round();
        }
        // ---- append + time rules + guard (BatchedHyps.add_results, :196-199) --
        if (warp == 0 && lane < R) {
          const int s = lane;
          rs.needp[s] = 0;
          if (rs.found[s]) {
            const int b = rs.b[s];
            const int pos = rs.len[s];
            if (rank == 0) {
              if (pos < p.cap) {
                p.out_tokens[(size_t)b * p.cap + pos] = rs.fy[s];
                p.out_timestamps[(size_t)b * p.cap + pos] = rs.ft[s];
                if (p.out_durations) p.out_durations[(size_t)b * p.cap + pos] = rs.fd[s];
              } else {
                atomicOr(p.status, 2);
              }
            }
            rs.len[s] = pos + 1;
            if (tdt && rs.fd[s] > 0) {
              rs.t[s] += rs.fd[s];
              rs.k[s] = 0;
            } else {
              rs.k[s] += 1;
              if (rs.k[s] == p.max_sym) {
                rs.t[s] += 1;
                rs.k[s] = 0;
              }
            }
            rs.active[s] = rs.t[s] < rs.L[s];
            rs.needp[s] = rs.active[s];
            rs.last[s] = rs.fy[s];
            for (int c = MAX_CTX - 1; c > 0; --c) rs.ctx[c][s] = rs.ctx[c - 1][s];
            rs.ctx[0][s] = rs.fy[s];
            rs.found[s] = 0;
          }
        }
        __syncwarp();
        cx.rebuild_lists();
        cx.sync();
      }
      // ---- group done: lengths, statistics -----------------------------------
      if (rank == 0 && warp == 0) {
        const int b = lane < R ? rs.b[lane] : p.B;   // the slot's utterance (unequal groups: length-sorted)
        int tot = 0;
        if (b < p.B) {
          p.out_lengths[b] = rs.len[lane];
          if constexpr (SC) p.out_scores[b] = rs.score[lane];
          tot = rs.len[lane];
        }
        for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
        if (t0) s_cnt[SC_LABELS] += tot;
      }
    }
    cx.final_acks(k);
    // drain outstanding f bulk copies before the CTA exits
    if (cx.fpend(0)) cx.wait_f(0);
    if (cx.fpend(1)) cx.wait_f(1);
    if constexpr (MMAW) {
      cx.gate_wait();
      if (tid == 0) cx.post(MCMD_EXIT);
    }
    cx.sync();
#undef LL_PHASE
    if (rank == 0 && tid == 0 && p.stats) {
      atomicAdd(p.stats + 0, (unsigned long long)s_cnt[SC_OUTER]);
      atomicAdd(p.stats + 1, (unsigned long long)s_cnt[SC_ROUNDS]);
      atomicAdd(p.stats + 2, (unsigned long long)s_cnt[SC_ALGEVALS]);
      atomicAdd(p.stats + 3, (unsigned long long)s_cnt[SC_PRED]);
      atomicAdd(p.stats + 4, (unsigned long long)s_cnt[SC_PREDROWS]);
      atomicAdd(p.stats + 5, (unsigned long long)s_cnt[SC_LABELS]);
      atomicAdd(p.stats + 6, (unsigned long long)s_cnt[SC_GROUPS]);
      atomicAdd(p.stats + 8, (unsigned long long)s_cnt[SC_ROWEVALS]);
      // the longest dependent chain of one cluster (its joint rounds + predictor
      // steps, over every group it decoded): the critical path of the launch
      {
        const unsigned long long r = min(s_cnt[SC_ROUNDS], 0xFFFFFu), pr = min(s_cnt[SC_PRED], 0xFFFFFu);
        atomicMax(p.stats + 11, ((r + pr) << 40) | (r << 20) | pr);
      }
      if (blockIdx.x == 0) {
        p.stats[7] = (unsigned long long)C;
        p.stats[9] = (unsigned long long)p.W;
        p.stats[10] = (unsigned long long)p.R;
        p.stats[12] = (unsigned long long)p.n_launch;
      }
    }
  }
  if constexpr (RING || MMAW) tc_fence_before();
  __syncthreads();
  if constexpr (RING || MMAW) {
    tc_fence_after();
    if (warp == 0) tmem_dealloc(cx.tmem, 512);
  }
  if (C > 1) cluster_sync_all();  // no CTA exits while peers may still st.async into it
}

// ---------------------------------------------------------------------------
// ll_debug_joint: the same joint / argmax / cross-CTA path on given rows.
// f rows [n][H] (workspace, produced by the encoder projection) + g [n][H].
// Runs with W = 1: every row is one slot with one frame.
// ---------------------------------------------------------------------------
template <typename T, int KR>
__global__ void __launch_bounds__(MAX_NW * 32, 1) debug_joint_kernel(const __grid_constant__ DecodeParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ RowState rs;
  __shared__ __align__(8) uint64_t s_bars[NBARS];
  Ctx<T, KR> cx(p, smem, rs, false, s_bars);
  const int C = cx.C, tid = cx.tid, warp = cx.warp, lane = cx.lane, R = p.R;
  cx.init_barriers();
  cx.load_weight_slice();
  __syncthreads();
  if (C > 1) cluster_sync_all();
  const int cluster_id = blockIdx.x / C, n_clusters = gridDim.x / C;
  for (int base = cluster_id * R; base < p.dbg_n; base += n_clusters * R) {
    const int M = min(R, p.dbg_n - base), MT = (M + 15) / 16;
    if (warp == 0 && lane < R) {
      rs.b[lane] = base + (lane < M ? lane : 0);
      rs.t[lane] = 0;
      rs.L[lane] = 1;
      rs.scanning[lane] = lane < M;
      rs.needp[lane] = 0;
      rs.active[lane] = lane < M;
    }
    __syncwarp();
    cx.rebuild_lists();
    for (int idx = tid; idx < M * p.H; idx += blockDim.x) {
      const int i = idx / p.H, c = idx % p.H;
      cx.gs()[(size_t)i * p.H + cx.goff(c & ~3) + (c & 3)] = p.dbg_g[(size_t)(base + i) * p.H + c];
    }
    __syncthreads();
    cx.issue_f(0, false);   // the workspace holds f as [n][1][H] (T_max = 1)
    __syncthreads();
    cx.wait_f(0);
    cx.plan_z(0);
    __syncthreads();
    cx.build_z(0);
    __syncthreads();
    cx.joint_keys(MT, M, p.dbg_logits, base);
    cx.exchange_keys();
    cx.exchange_wait();
    if (cx.rank == 0 && warp == 0 && lane < M) {
      int y, di;
      cx.final_keys(lane, y, di);
      p.dbg_argmax[base + lane] = y;
      if (p.dbg_dargmax) p.dbg_dargmax[base + lane] = di;
    }
    cx.flip_par();
    __syncthreads();
  }
  if (C > 1) cluster_sync_all();  // no CTA exits while peers may still st.async into it
}

}  // namespace ll
