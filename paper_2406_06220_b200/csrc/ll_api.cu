// ll_api.cu -- host side of the C ABI declared in include/ll.h.
//
// Validation (synchronous, nothing enqueued on error), workspace carving,
// cluster-size selection and the launches:
//   1. encoder projection f = W_enc enc + b_enc over all B*T_max frames
//      (Alg. 3 line 2; precompute)
//   2. model tables (LSTM E' = W_ih Emb + b_ih + b_hh; stateless G_k)
//   3. the persistent cluster decode kernel (decode.cuh)
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <unordered_map>

#include <cudaTypedefs.h>

#include "../../include/ll.h"
#include "decode.cuh"
#include "gemm_tc.cuh"
#include "linear.cuh"

using namespace ll;

namespace {

constexpr size_t HDR_BYTES = 4096;  // [0] status, [1] group counter, [16..] stats (u64 x 8 at byte 64)
// rows per group when the batch spans many waves (measured under the per-row
// tick schedule: LSTM sweep best at 8, stateless config 4 at 16)
constexpr int RPREF_MANY_LSTM = 8, RPREF_MANY_STATELESS = 16;
constexpr size_t SMEM_LIMIT = 232448;

struct Ws {
  size_t f, tab, h, g, wst, wih, perm, total;
};

size_t esize(ll_dtype d) { return d == LL_BF16 ? 2 : 4; }
inline int nlayers(const ll_predictor *pr) {
  return (pr && pr->kind == LL_PRED_LSTM && pr->num_layers > 1) ? pr->num_layers : 1;
}

// Workspace regions (256-B aligned).  The weight-only tables come first so
// that their offsets do not depend on the batch shape (ll_prepare).
Ws ws_layout(int B, int T, const ll_predictor *pr, const ll_joint *jn, ll_dtype dt) {
  Ws w;
  const size_t H = jn->joint_dim, P = jn->pred_dim, V1 = jn->num_outputs;
  size_t o = HDR_BYTES;
  w.tab = o;
  if (pr->kind == LL_PRED_LSTM)
    o = align_up(o + V1 * 4 * P * 4, 256);
  else
    o = align_up(o + (size_t)pr->context * V1 * H * 4, 256);
  w.wst = o;  // packed LSTM weight stream (bf16): (4P + H) rows of P
  if (pr->kind == LL_PRED_LSTM && dt == LL_BF16) o = align_up(o + (4 * P + H) * P * 2, 256);
  w.wih = o;  // bf16 LSTM: W_ih and b_ih, b_hh with gate rows permuted CTA-major (E' table columns)
  if (pr->kind == LL_PRED_LSTM && dt == LL_BF16) o = align_up(o + 4 * P * P * 2 + 2 * 4 * P * 2, 256);
  w.f = o;
  o = align_up(o + (size_t)B * T * H * esize(dt) + 256, 256);   // + slack: the padded f-row boxes read 16 B past a row
  w.h = o;   // [layers][2][B][P]
  if (pr->kind == LL_PRED_LSTM) o = align_up(o + (size_t)nlayers(pr) * 2 * B * P * esize(dt), 256);
  w.g = o;
  if (pr->kind == LL_PRED_LSTM) o = align_up(o + (size_t)B * H * 4, 256);
  w.perm = o;   // utterances ranked by length (groups of similar lengths, longest first)
  o = align_up(o + (size_t)B * 4, 256);
  w.total = o;
  return w;
}

thread_local cudaEvent_t g_ev_before = nullptr, g_ev_after = nullptr;
// kernels launched by the current public decode call of this thread (reported
// by ll_stats [12]; every launch site counts itself)
thread_local int g_nlaunch = 0;

// Test / debug options of this host thread (ll_set_options; ll.h).  The
// production path reads no environment variable.
ll_options default_options() {
  ll_options o;
  memset(&o, 0, sizeof(o));
  o.schedule = -1;
  o.spec_prefetch = -1;
  o.group_plan = -1;
  return o;
}
thread_local ll_options g_opt = default_options();

ll_status check_model(const ll_predictor *pr, const ll_joint *jn, ll_dtype dt, ll_prec prec,
                      int nD, bool need_pred) {
  if (!jn) return LL_ERR_INVALID_ARGUMENT;
  if (dt != LL_BF16 && dt != LL_F32) return LL_ERR_INVALID_ARGUMENT;
  if (prec != LL_PREC_FAST && prec != LL_PREC_EXACT) return LL_ERR_INVALID_ARGUMENT;
  if (jn->enc_dim <= 0 || jn->pred_dim <= 0 || jn->joint_dim <= 0 || jn->num_outputs < 1)
    return LL_ERR_INVALID_ARGUMENT;
  if (!jn->w_enc || !jn->b_enc || !jn->w_out || !jn->b_out) return LL_ERR_INVALID_ARGUMENT;
  if (nD < 0 || nD > MAX_DUR) return LL_ERR_INVALID_ARGUMENT;
  if (nD > 0 && (!jn->w_dur || !jn->b_dur)) return LL_ERR_INVALID_ARGUMENT;
  if (need_pred) {
    if (!pr) return LL_ERR_INVALID_ARGUMENT;
    if (!jn->w_pred || !jn->b_pred || !pr->embedding) return LL_ERR_INVALID_ARGUMENT;
    if (pr->num_tokens != jn->num_outputs || pr->hidden != jn->pred_dim) return LL_ERR_INVALID_ARGUMENT;
    if (pr->kind == LL_PRED_LSTM) {
      if (!pr->w_ih || !pr->w_hh || !pr->b_ih || !pr->b_hh) return LL_ERR_INVALID_ARGUMENT;
      if (pr->num_layers < 0 || pr->num_layers > MAX_LAYERS) return LL_ERR_INVALID_ARGUMENT;
      if (pr->num_layers > 1 && (!pr->w_ih_rest || !pr->w_hh_rest || !pr->b_ih_rest || !pr->b_hh_rest))
        return LL_ERR_INVALID_ARGUMENT;   // bf16 with > 1 layer: widened to fp32 (see widened() below)
    } else if (pr->kind == LL_PRED_STATELESS) {
      if (pr->context < 1) return LL_ERR_INVALID_ARGUMENT;
      if (pr->context > MAX_CTX || pr->hidden % pr->context) return LL_ERR_UNSUPPORTED;
    } else {
      return LL_ERR_INVALID_ARGUMENT;
    }
  }
  if (jn->enc_dim % 16 || jn->pred_dim % 16 || jn->joint_dim % 16) return LL_ERR_UNSUPPORTED;
  if (need_pred && pr->kind == LL_PRED_STATELESS && (jn->pred_dim / pr->context) % 8)
    return LL_ERR_UNSUPPORTED;
  return LL_OK;
}

// Decode configuration: cluster size C, rows per group R, window W (R*W <= 32
// joint rows per round), buffered frames WF = W + max_duration - 1.
struct Config {
  int C, R, W, WF, NS;
  Layout L;
};

static int pow2ceil(int x) {
  int r = 1;
  while (r < x) r <<= 1;
  return r;
}

// Candidate (C, R, W) in preference order; the first that fits wins.  The
// preferred R spreads the batch over the ~8 concurrently resident 16-CTA
// clusters of a B200 (small groups = fewer rounds per group), W = 32 / R.
// nclusters: how many clusters of the chosen size can be resident (0: unknown,
// assume 8).  R is chosen so that all groups of the batch run in one wave.
bool choose_config(bool bf, bool lstm, int H, int P, int V1, int nD, int maxd, int B, Config &cf,
                   int nclusters = 0, int sc = 0, int layers = 1, int otf_de = 0) {
  const int forceC = g_opt.cluster_size;
  const int forceR = g_opt.group_rows;
  const int forceW = g_opt.window;
  const bool ring = bf && lstm;
  if (bf && H > KREG * 32 + 16) return false;        // joint slice must fit the register tile
  const int ncl = nclusters > 0 ? nclusters : 8;
  int Rpref = forceR ? forceR : (B + ncl - 1) / ncl;
  // throughput mode: when one wave would need more than 8 rows per group, run
  // many waves of small groups instead (groups are taken from a work counter,
  // so the clusters stay busy; small groups keep the multi-frame window wide)
  if (!forceR && Rpref > 8) Rpref = lstm ? RPREF_MANY_LSTM : RPREF_MANY_STATELESS;
  if (Rpref < 1) Rpref = 1;
  if (Rpref > MAX_R) Rpref = MAX_R;
  // clusters of >= 2 CTAs: the kernels' DSMEM traffic (st.async to mapa'd
  // addresses) is defined for real clusters (compute-sanitizer rejects a
  // 1-CTA cluster)
  for (int C = 2; C <= MAX_C; C *= 2) {
    if (forceC && C != forceC) continue;
    const int NT = (V1 + nD + 7) / 8;
    if (bf && (NT + C - 1) / C > MAX_NW) continue;   // one vocab tile per warp
    if (bf) {
      if (H % (8 * C)) continue;
      if (lstm && P % (8 * C)) continue;             // h' slice: whole 16-byte chunks
      if (ring) {
        // W_hh tile pairs of a CTA must fit TMEM (512 columns): warp w holds
        // 2 * ceil(pairs / NW) tiles in lane quarter w % 4, shared by <= 3 warps
        const int pairs = P / C / 4, tcols = 4 * (P / 32) + ((P & 31) ? 2 : 0);
        if (2 * ((pairs + MAX_NW - 1) / MAX_NW) * 3 * tcols > 512) continue;
        if (H / C > 48) continue;                    // W_pred: <= 3 m16 tiles per CTA
      }
    } else {
      if (H % C) continue;
      if (lstm && P % C) continue;
    }
    for (int R = Rpref; R >= 1; --R) {
      if (forceR && R != forceR) continue;
      if (tg_shape(bf, lstm, H, P, C) && R > TG_NH) continue;   // gate batch: one N=8 B operand
      int W = forceW ? forceW : MAX_JR / R;
      if (W > 8) W = 8;
      if (W < 1) W = 1;
      if (R * W > MAX_JR) continue;
      for (; W >= 1; W = tj_shape(bf, H, P, C) ? W - 1 : W >> 1) {
        // TJ (tcgen05 joint, ~1K cycles per round whatever the row count):
        // fewer rows per group with a real window beat one-frame rounds
        if (tj_shape(bf, H, P, C) && !forceW && !forceR && W == 1 && R > 1) break;
        cf.C = C; cf.R = R; cf.W = W; cf.WF = W + (maxd > 1 ? maxd - 1 : 0);
        cf.NS = 0;
        cf.L = make_layout(bf, lstm, H, P, V1, nD, R, W, cf.WF, C, 0, sc, true, layers,
                           otf_de && tg_shape(bf, lstm, H, P, C) ? otf_de : 0);
        if (cf.L.total + sizeof(RowState) + 1024 <= SMEM_LIMIT) return true;
        if (forceW) break;
      }
    }
  }
  return false;
}

// Resident clusters of size C for the decode kernel (1 CTA per SM).
// Register-tile width of the joint weight slice: KREG_SMALL K blocks for small
// joints, KREG (H <= 656) otherwise; fp32 keeps no weights in registers.
inline int kreg_for(bool bf, int H) { return !bf ? 1 : (H <= KREG_SMALL * 32 + 16 ? KREG_SMALL : KREG); }
// Production shape (FastConformer joint, BASELINE configs 2-5): H = P = 640 in
// 16-CTA clusters, compiled with those dims fixed.
constexpr int FC_H = 640, FC_P = 640, FC_C = 16;
inline bool is_fc(bool bf, int H, int P, int C) { return bf && H == FC_H && P == FC_P && C == FC_C; }

template <typename T, int PRED, int KR, int HC = 0, int PC = 0, int CC = 0, int LM = 0, int TM = 0>
int max_clusters(int C, const Layout &L) {
  auto kern = decode_kernel<T, PRED, KR, HC, PC, CC, LM, TM>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
  if (C > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(L.NTH);
  cfg.dynamicSmemBytes = L.total;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3(C);
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, (void *)kern, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

template <typename T, int PRED, int KR, int HC = 0, int PC = 0, int CC = 0, int LM = 0, int TM = 0, int DBG = 0,
          int SC = 0>
ll_status launch_decode(const DecodeParams &p, int C, const Layout &L, int n_groups, cudaStream_t st,
                        int &used_clusters) {
  auto kern = decode_kernel<T, PRED, KR, HC, PC, CC, LM, TM, DBG, SC>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total) != cudaSuccess)
    return LL_ERR_CUDA;
  if (C > 8 && cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
    return LL_ERR_CUDA;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(L.NTH);
  cfg.dynamicSmemBytes = L.total;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int max_clusters = 0;
  cfg.gridDim = dim3(C);
  if (cudaOccupancyMaxActiveClusters(&max_clusters, (void *)kern, &cfg) != cudaSuccess || max_clusters < 1) {
    cudaGetLastError();
    return LL_ERR_UNSUPPORTED;
  }
  if (g_opt.max_clusters > 0) max_clusters = std::min(max_clusters, g_opt.max_clusters);
  if (p.probe_logits && p.probe_regions > 0) max_clusters = std::min(max_clusters, p.probe_regions);
  used_clusters = std::min(n_groups, max_clusters);
  cfg.gridDim = dim3(used_clusters * C);
  if (cudaLaunchKernelEx(&cfg, kern, p) != cudaSuccess) return LL_ERR_CUDA;
  return LL_OK;
}

template <typename T, int KR>
ll_status launch_debug(const DecodeParams &p, int C, const Layout &L, int n_chunks, cudaStream_t st) {
  auto kern = debug_joint_kernel<T, KR>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total) != cudaSuccess)
    return LL_ERR_CUDA;
  if (C > 8 && cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
    return LL_ERR_CUDA;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(L.NTH);
  cfg.dynamicSmemBytes = L.total;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int max_clusters = 0;
  cfg.gridDim = dim3(C);
  if (cudaOccupancyMaxActiveClusters(&max_clusters, (void *)kern, &cfg) != cudaSuccess || max_clusters < 1) {
    cudaGetLastError();
    return LL_ERR_UNSUPPORTED;
  }
  cfg.gridDim = dim3(std::min(n_chunks, max_clusters) * C);
  if (cudaLaunchKernelEx(&cfg, kern, p) != cudaSuccess) return LL_ERR_CUDA;
  return LL_OK;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void *f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    fn = (PFN_cuTensorMapEncodeTiled_v12000)f;
  }
  return fn;
}

// 2-D bf16 tensor map over a row-major [rows, cols] matrix with leading
// dimension ld (elements): 64-column x box_rows boxes, 128-byte swizzle.
bool make_map_bf16(CUtensorMap *m, const void *base, uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box_rows) {
  PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
  if (!enc) return false;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {ld * 2};
  const cuuint32_t box[2] = {TC_BK, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 3-D bf16 tensor map over Bu segments of T rows of a row-major matrix with
// leading dimension ld (elements), segment stride T * ld: 64-column x box_rows x
// 1 boxes, 128-byte swizzle; rows past T in a segment are zero-filled.
bool make_map3_bf16(CUtensorMap *m, const void *base, uint64_t T, uint64_t Bu, uint64_t cols, uint64_t ld,
                    uint32_t box_rows) {
  PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
  if (!enc) return false;
  const cuuint64_t dims[3] = {cols, T, Bu};
  const cuuint64_t strides[2] = {ld * 2, T * ld * 2};
  const cuuint32_t box[3] = {TC_BK, box_rows, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// TJ f boxes (DecodeParams::fmap): {8 elements, 81 chunks, frames}, chunk stride
// 16 B, frame stride 2H; box {8, 81, WF} -> WF padded 1296-byte rows.
bool make_fmap(CUtensorMap *m, const void *f, uint64_t frames, int H, int WF) {
  PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
  if (!enc || H != TJ_H || WF < 1 || WF > 255) return false;
  const cuuint64_t dims[3] = {8, (cuuint64_t)(TJ_FROW / 16), frames};
  const cuuint64_t strides[2] = {16, (cuuint64_t)H * 2};
  const cuuint32_t box[3] = {8, (cuuint32_t)(TJ_FROW / 16), (cuuint32_t)WF};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(f), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// tcgen05 GEMM (gemm_tc.cuh) when the shape fits its tiles; false = not taken.
bool linear_tc(const void *X, int64_t ldx, const void *W, int64_t ldw, const void *bias, const void *bias2, void *Y,
               int64_t ldy, int M, int N, int K, bool out_bf16, cudaStream_t st, ll_status &s,
               const int *lengths = nullptr, int T = 0) {
  if (g_opt.gemm_mma_sync) return false;
  if (K % TC_BK || N % TC_BNQ || (ldx * 2) % 16 || (ldw * 2) % 16 || ((uintptr_t)X & 15) || ((uintptr_t)W & 15))
    return false;
  if ((out_bf16 && (ldy * 2) % 16) || (!out_bf16 && (ldy * 4) % 16) || ((uintptr_t)Y & 15)) return false;
  static int nsm = 0, attr_done = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (nsm < 1) nsm = 1;
  }
  // rows as segments: the encoder frames of each utterance (lengths), else one segment
  if (lengths && (T < 1 || M % T)) return false;
  const int Tseg = lengths ? T : M, Bu = lengths ? M / T : 1;
  // 128 x 256 tiles, unless that leaves fewer than two tiles per SM (then 128 x 128);
  // mt: M tiles at full lengths (an upper bound of the used ones)
  const int mt = Bu * ((Tseg + TC_BM - 1) / TC_BM);
  const int bn = mt * ((N + TC_BN - 1) / TC_BN) >= 2 * nsm ? TC_BN : TC_BNQ;
  CUtensorMap mx, mw;
  if (!make_map3_bf16(&mx, X, (uint64_t)Tseg, (uint64_t)Bu, (uint64_t)K, (uint64_t)ldx, TC_BM) ||
      !make_map_bf16(&mw, W, (uint64_t)N, (uint64_t)K, (uint64_t)ldw, (uint32_t)bn))
    return false;
  TcGemmArgs a{bias, bias2, Y, ldy, M, N, K, lengths, Tseg, Bu, bn};
  if (!attr_done) {   // once per process (not on every call)
    cudaFuncSetAttribute(gemm_tc_kernel<bf16>, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM);
    cudaFuncSetAttribute(gemm_tc_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM);
    attr_done = 1;
  }
  const int ntiles = mt * ((N + bn - 1) / bn);
  dim3 grid(std::min(ntiles, nsm));
  ++g_nlaunch;
  if (out_bf16) gemm_tc_kernel<bf16><<<grid, TC_THREADS, TC_SMEM, st>>>(mx, mw, a);
  else gemm_tc_kernel<float><<<grid, TC_THREADS, TC_SMEM, st>>>(mx, mw, a);
  s = cudaPeekAtLastError() == cudaSuccess ? LL_OK : LL_ERR_CUDA;
  return true;
}

// lengths / T: ragged encoder rows (row b*T + t used iff t < lengths[b]); tcgen05 path only
ll_status linear(bool bf, const void *X, int64_t ldx, const void *W, int64_t ldw, const void *bias,
                 const void *bias2, void *Y, int64_t ldy, int M, int N, int K, bool out_bf16,
                 cudaStream_t st, const int *lengths = nullptr, int T = 0) {
  if (M <= 0 || N <= 0) return LL_OK;
  if (bf) {
    ll_status s;
    if (linear_tc(X, ldx, W, ldw, bias, bias2, Y, ldy, M, N, K, out_bf16, st, s, lengths, T)) return s;
  }
  LinearArgs a{X, ldx, W, ldw, bias, bias2, Y, ldy, M, N, K};
  ++g_nlaunch;
  if (bf) {
    dim3 grid((N + LB_N - 1) / LB_N, (M + LB_M - 1) / LB_M);
    if (out_bf16)
      linear_bf16_kernel<bf16><<<grid, 256, 0, st>>>(a);
    else
      linear_bf16_kernel<float><<<grid, 256, 0, st>>>(a);
  } else {
    dim3 grid((N + 63) / 64, (M + 63) / 64);
    linear_f32_kernel<<<grid, 256, 0, st>>>(a);
  }
  return cudaPeekAtLastError() == cudaSuccess ? LL_OK : LL_ERR_CUDA;
}

// Cluster size / group rows / window for a call: choose_config, then again
// with the number of clusters that can actually be resident.
bool decode_config(bool bf, bool lstm, int H, int P, int V1, int nD, int maxd, int B, Config &cf, int sc = 0,
                   int layers = 1, int otf_de = 0) {
  if (!choose_config(bf, lstm, H, P, V1, nD, maxd, B, cf, 0, sc, layers, otf_de)) return false;
  int ncl = 0;
  if (otf_de && cf.L.otf)
    ncl = max_clusters<bf16, 0, KREG, FC_H, FC_P, FC_C, 4, 1>(cf.C, cf.L);
  else if (is_fc(bf, H, P, cf.C))
    ncl = lstm ? max_clusters<bf16, 0, KREG, FC_H, FC_P, FC_C, 1, 1>(cf.C, cf.L)
               : max_clusters<bf16, 1, KREG, FC_H, FC_P, FC_C, 1, 1>(cf.C, cf.L);
  else if (bf && kreg_for(bf, H) == KREG)
    ncl = lstm ? max_clusters<bf16, 0, KREG>(cf.C, cf.L) : max_clusters<bf16, 1, KREG>(cf.C, cf.L);
  else if (bf)
    ncl = lstm ? max_clusters<bf16, 0, KREG_SMALL>(cf.C, cf.L) : max_clusters<bf16, 1, KREG_SMALL>(cf.C, cf.L);
  else
    ncl = lstm ? max_clusters<float, 0, 1>(cf.C, cf.L) : max_clusters<float, 1, 1>(cf.C, cf.L);
  return !(ncl > 0 && !choose_config(bf, lstm, H, P, V1, nD, maxd, B, cf, ncl, sc, layers, otf_de));
}

// ---------------------------------------------------------------------------
// Weight-only model tables of a call (E' or G_k, the packed W_hh / W_pred
// stream) and the registry that lets ll_prepare build them once per
// workspace: a decode whose weights / shapes / cluster config match the
// fingerprint ll_prepare recorded for its workspace skips rebuilding them.
// ---------------------------------------------------------------------------
struct TableKey {
  const void *ptr[8];
  int dims[10];
  size_t ws_bytes;
  bool operator==(const TableKey &o) const { return memcmp(this, &o, sizeof(TableKey)) == 0; }
};

TableKey table_key(const ll_predictor *pr, const ll_joint *jn, ll_dtype dt, int C, const Layout &L,
                   size_t ws_bytes) {
  TableKey k;
  memset(&k, 0, sizeof(k));
  k.ws_bytes = ws_bytes;
  k.ptr[0] = pr->embedding; k.ptr[1] = pr->w_ih; k.ptr[2] = pr->w_hh; k.ptr[3] = pr->b_ih;
  k.ptr[4] = pr->b_hh; k.ptr[5] = jn->w_pred; k.ptr[6] = jn->b_pred;
  k.dims[0] = pr->kind; k.dims[1] = pr->num_tokens; k.dims[2] = pr->hidden; k.dims[3] = pr->context;
  k.dims[4] = jn->joint_dim; k.dims[5] = (int)dt; k.dims[6] = jn->num_outputs; k.dims[8] = C;
  k.dims[9] = L.UPC * 1000 + L.DPC;
  return k;
}

std::mutex g_prep_mu;
std::unordered_map<const void *, TableKey> g_prepared;   // workspace -> tables it holds

ll_status build_tables(bool bf, const ll_predictor *pr, const ll_joint *jn, ll_dtype dt, const Ws &w, uint8_t *ws,
                       int C, const Layout &L, cudaStream_t st) {
  const bool lstm = pr->kind == LL_PRED_LSTM, ring = bf && lstm;
  const int H = jn->joint_dim, P = jn->pred_dim, V1 = jn->num_outputs;
  ll_status s = LL_OK;
  float *tab = (float *)(ws + w.tab);
  if (lstm && ring) {
    // E' = Emb W_ih^T + b_ih + b_hh with its 4P columns ordered CTA-major (rank r:
    // gates i,f,g,o of units r*UPC ...), so the decode kernel fetches a predictor
    // row's slice with ONE bulk copy of 4*UPC floats
    bf16 *wih = (bf16 *)(ws + w.wih);
    bf16 *bih = wih + (size_t)4 * P * P, *bhh = bih + 4 * P;
    ++g_nlaunch;
    permute_gate_rows<<<296, 256, 0, st>>>((const bf16 *)pr->w_ih, (const bf16 *)pr->b_ih, (const bf16 *)pr->b_hh,
                                           wih, bih, bhh, P, C, L.UPC);
    if (cudaPeekAtLastError() != cudaSuccess) return LL_ERR_CUDA;
    s = linear(bf, pr->embedding, P, wih, P, bih, bhh, tab, 4 * P, V1, 4 * P, P, false, st);
  } else if (lstm) {
    s = linear(bf, pr->embedding, P, pr->w_ih, P, pr->b_ih, pr->b_hh, tab, 4 * P, V1, 4 * P, P, false, st);
  } else {
    const int c = pr->context, Pc = P / c;
    for (int k = 0; k < c && s == LL_OK; ++k) {
      const uint8_t *emb = (const uint8_t *)pr->embedding + (size_t)k * V1 * Pc * esize(dt);
      const uint8_t *wp = (const uint8_t *)jn->w_pred + (size_t)k * Pc * esize(dt);
      s = linear(bf, emb, Pc, wp, P, k == 0 ? jn->b_pred : nullptr, nullptr, tab + (size_t)k * V1 * H, H,
                 V1, H, Pc, false, st);
    }
  }
  if (s != LL_OK) return s;
  if (ring) {
    // contiguous per-CTA tile stream of W_hh / W_pred
    ++g_nlaunch;
    pack_lstm_stream<<<296, 256, 0, st>>>((const bf16 *)pr->w_hh, (const bf16 *)jn->w_pred,
                                          (bf16 *)(ws + w.wst), P, C, L.UPC, L.DPC);
    if (cudaPeekAtLastError() != cudaSuccess) return LL_ERR_CUDA;
  }
  return LL_OK;
}

// Utterances ranked by (length desc, index): perm[rank] = b.  Groups of
// consecutive ranks then hold utterances of similar lengths (a group runs as
// long as its longest row) and the work counter hands out the longest groups
// first (LPT).  O(B^2) comparisons through shared-memory tiles: ~µs at B = 512.
__global__ void rank_lengths_kernel(const int *lengths, int B, int T_max, int *perm) {
  __shared__ int tile[256];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  int Li = 0;
  if (i < B) {
    Li = lengths[i];
    if (Li < 0 || Li > T_max) Li = 0;
  }
  int rk = 0;
  for (int j0 = 0; j0 < B; j0 += 256) {
    __syncthreads();
    if (j0 + threadIdx.x < B) {
      int L = lengths[j0 + threadIdx.x];
      tile[threadIdx.x] = (L < 0 || L > T_max) ? 0 : L;
    }
    __syncthreads();
    const int n = min(256, B - j0);
    for (int j = 0; j < n; ++j) {
      const int Lj = tile[j];
      rk += (Lj > Li || (Lj == Li && j0 + j < i)) ? 1 : 0;
    }
  }
  if (i < B) perm[rk] = i;
}

// ---------------------------------------------------------------------------
// LL_PREC_EXACT with bf16 inputs, and bf16 LSTM predictors of more than one
// layer: the call runs the fp32 kernels on fp32 copies of the bf16 values.
// Every bf16 value is an fp32 value, so this is the same model computed with
// fp32 f, g, h, c and z (the fp32 tolerance class, 1e-5 on the logits) instead
// of bf16-rounded f / h / z.  The copies (one widening kernel per array) sit
// BEHIND the fp32 call's own workspace, whose header (status, stats) stays at
// the front for ll_sync / ll_stats.  The model tables are rebuilt on every
// such call (ll_prepare records nothing for them).
// ---------------------------------------------------------------------------
__global__ void widen_bf16_kernel(const bf16 *src, float *dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = __bfloat162float(src[i]);
}

inline bool widened(const ll_predictor *pr, ll_dtype dt, ll_prec prec) {
  return dt == LL_BF16 && (prec == LL_PREC_EXACT || (pr && nlayers(pr) > 1));
}

struct WideArr {
  const void *src;
  const void **dst;   // the pointer field of the fp32 copy of the model struct
  size_t n;
};

// The weight arrays of (pr, jn) in a fixed order (NULL fields skipped); the
// destinations are the matching fields of pr32 / jn32 (pr may be NULL).
int wide_arrays(const ll_predictor *pr, const ll_joint *jn, int nD, ll_predictor *pr32, ll_joint *jn32,
                WideArr *a) {
  const size_t H = jn->joint_dim, P = jn->pred_dim, V1 = jn->num_outputs, De = jn->enc_dim;
  int k = 0;
  auto add = [&](const void *src, const void **dst, size_t n) {
    if (src) a[k++] = WideArr{src, dst, n};
  };
  add(jn->w_enc, &jn32->w_enc, H * De);
  add(jn->b_enc, &jn32->b_enc, H);
  add(jn->w_pred, &jn32->w_pred, H * P);
  add(jn->b_pred, &jn32->b_pred, H);
  add(jn->w_out, &jn32->w_out, V1 * H);
  add(jn->b_out, &jn32->b_out, V1);
  if (nD > 0) {
    add(jn->w_dur, &jn32->w_dur, (size_t)nD * H);
    add(jn->b_dur, &jn32->b_dur, (size_t)nD);
  }
  if (pr) {
    add(pr->embedding, &pr32->embedding, V1 * P);   // LSTM [V1, P]; stateless [ctx][V1, P / ctx]
    if (pr->kind == LL_PRED_LSTM) {
      const size_t Lr = (size_t)nlayers(pr) - 1;
      add(pr->w_ih, &pr32->w_ih, 4 * P * P);
      add(pr->w_hh, &pr32->w_hh, 4 * P * P);
      add(pr->b_ih, &pr32->b_ih, 4 * P);
      add(pr->b_hh, &pr32->b_hh, 4 * P);
      if (Lr > 0) {
        add(pr->w_ih_rest, &pr32->w_ih_rest, Lr * 4 * P * P);
        add(pr->w_hh_rest, &pr32->w_hh_rest, Lr * 4 * P * P);
        add(pr->b_ih_rest, &pr32->b_ih_rest, Lr * 4 * P);
        add(pr->b_hh_rest, &pr32->b_hh_rest, Lr * 4 * P);
      }
    }
  }
  return k;
}
constexpr int MAX_WIDE = 24;

// bytes of the fp32 copies: the weights + the encoder rows [B, T, D_e]
size_t wide_bytes(int B, int T, const ll_predictor *pr, const ll_joint *jn, int nD) {
  ll_predictor p2 = pr ? *pr : ll_predictor{};
  ll_joint j2 = *jn;
  WideArr a[MAX_WIDE];
  const int na = wide_arrays(pr, jn, nD, pr ? &p2 : nullptr, &j2, a);
  size_t o = 0;
  for (int i = 0; i < na; ++i) o = align_up(o + a[i].n * 4, 256);
  return align_up(o + (size_t)B * T * jn->enc_dim * 4, 256);
}

// Widen into ws (256-aligned): fills pr32 / jn32 (copies of pr / jn with the
// fp32 pointers) and returns the fp32 encoder rows.
float *widen_all(const void *enc, size_t enc_n, const ll_predictor *pr, const ll_joint *jn, int nD,
                 ll_predictor *pr32, ll_joint *jn32, uint8_t *ws, cudaStream_t st, ll_status &s) {
  if (pr) *pr32 = *pr;
  *jn32 = *jn;
  WideArr a[MAX_WIDE];
  const int na = wide_arrays(pr, jn, nD, pr32, jn32, a);
  size_t o = 0;
  auto widen = [&](const void *src, float *dst, size_t n) {
    if (n == 0) return;
    const int blocks = (int)std::min<size_t>((n + 255) / 256, 4096);
    ++g_nlaunch;
    widen_bf16_kernel<<<blocks, 256, 0, st>>>((const bf16 *)src, dst, n);
  };
  for (int i = 0; i < na; ++i) {
    float *d = (float *)(ws + o);
    *a[i].dst = d;
    widen(a[i].src, d, a[i].n);
    o = align_up(o + a[i].n * 4, 256);
  }
  float *enc32 = (float *)(ws + o);
  widen(enc, enc32, enc_n);
  s = cudaPeekAtLastError() == cudaSuccess ? LL_OK : LL_ERR_CUDA;
  return enc32;
}

ll_status decode_impl(bool tdt, bool frame_looping, const void *enc, ll_dtype dt, ll_prec prec, int32_t B, int32_t T_max,
                      const int32_t *lengths, const ll_predictor *pr, const ll_joint *jn,
                      int32_t blank_id, int32_t max_symbols, const int32_t *durations, int32_t nD,
                      int32_t *out_tokens, int32_t *out_timestamps, int32_t *out_durations,
                      int32_t *out_lengths, int32_t cap, void *workspace, size_t workspace_bytes,
                      ll_stream stream, float *out_scores = nullptr) {
  if (B < 0 || T_max < 0 || cap < 0) return LL_ERR_INVALID_ARGUMENT;
  if (!workspace || ((uintptr_t)workspace & 255)) return LL_ERR_INVALID_ARGUMENT;
  if (B > 0 && (!enc || !lengths || !out_tokens || !out_timestamps || !out_lengths))
    return LL_ERR_INVALID_ARGUMENT;
  if (tdt) {
    if (nD < 1 || !durations) return LL_ERR_INVALID_ARGUMENT;
    for (int i = 0; i < nD; ++i)
      if (durations[i] < 0) return LL_ERR_INVALID_ARGUMENT;
  } else {
    nD = 0;
  }
  ll_status s = check_model(pr, jn, dt, prec, nD, true);
  if (s != LL_OK) return s;
  if (blank_id < 0 || blank_id >= jn->num_outputs) return LL_ERR_INVALID_ARGUMENT;
  if (max_symbols < 1) return LL_ERR_INVALID_ARGUMENT;
  if (workspace_bytes < ll_workspace_size(B, T_max, pr, jn, dt, prec, nD)) return LL_ERR_WORKSPACE;
  const bool bf = dt == LL_BF16;
  const bool lstm = pr->kind == LL_PRED_LSTM;
  const int H = jn->joint_dim, P = jn->pred_dim, V1 = jn->num_outputs, De = jn->enc_dim;
  int maxd = 1;
  for (int i = 0; i < nD; ++i) maxd = durations[i] > maxd ? durations[i] : maxd;
  if (widened(pr, dt, prec)) {   // fp32 kernels on fp32 copies (see widened() above)
    if (g_opt.projections == 1 || g_opt.probe_logits) return LL_ERR_UNSUPPORTED;   // bf16 FC kernels only
    {
      Config c32;
      if (!decode_config(false, lstm, H, P, V1, nD, maxd, B, c32, out_scores != nullptr, nlayers(pr)))
        return LL_ERR_UNSUPPORTED;
    }
    const size_t inner = align_up(ws_layout(B, T_max, pr, jn, LL_F32).total, 256);
    ll_predictor pr32;
    ll_joint jn32;
    ll_status ws_s = LL_OK;
    float *enc32 = widen_all(enc, (size_t)B * T_max * De, pr, jn, nD, &pr32, &jn32, (uint8_t *)workspace + inner,
                             (cudaStream_t)stream, ws_s);
    if (ws_s != LL_OK) return ws_s;
    ll_release(workspace);   // the fp32 tables are rebuilt from the fresh copies
    return decode_impl(tdt, frame_looping, enc32, LL_F32, LL_PREC_FAST, B, T_max, lengths, &pr32, &jn32, blank_id,
                       max_symbols, durations, nD, out_tokens, out_timestamps, out_durations, out_lengths, cap,
                       workspace, inner, stream, out_scores);
  }
  // greedy scores (N2): the per-row tick schedule's SC kernels
  const int sc = out_scores != nullptr;
  if (sc && (frame_looping || g_opt.schedule == 0 || g_opt.probe_logits)) return LL_ERR_UNSUPPORTED;
  Config cf;
  const int nl = nlayers(pr);
  // on-the-fly projections (ll_options.projections = 1; Table 3's ablation arm)
  const bool otf = g_opt.projections == 1;
  if (otf && (!bf || !lstm || nl != 1 || frame_looping || sc || g_opt.probe_logits || g_opt.schedule == 0 ||
              H != FC_H || P != FC_P || De % 32 || De > OTF_MAX_DE))
    return LL_ERR_UNSUPPORTED;
  if (!decode_config(bf, lstm, H, P, V1, nD, maxd, B, cf, sc, nl, otf ? De : 0)) return LL_ERR_UNSUPPORTED;
  if (otf && !cf.L.otf) return LL_ERR_UNSUPPORTED;   // not the FC cluster shape
  if (frame_looping) {   // Alg. 2 evaluates one frame per joint call
    cf.W = 1;
    cf.WF = 1;
    cf.L = make_layout(bf, lstm, H, P, V1, nD, cf.R, 1, 1, cf.C, 0, 0, true, nl);
  }
  // Length-sorted unequal groups: a one-wave RNN-T FC tick
  // decode of n groups of R rows has n R - B spare slots; making those groups
  // one row smaller lets them take wider windows, and the longest utterances
  // (dealt by length) go there -- the critical group needs fewer ticks
  int gp_small = 0, gp_rsmall = 0, gp_wsmall = 0;
  if (g_opt.group_plan != 0 && !sc && !frame_looping && !g_opt.probe_logits && bf &&
      is_fc(bf, H, P, cf.C) && !g_opt.group_rows && !g_opt.window && (g_opt.schedule < 0 || g_opt.schedule == 1) &&
      B <= 32 && cf.R >= 3) {
    const int ng = (B + cf.R - 1) / cf.R, xs = ng * cf.R - B, rsm = cf.R - 1;
    int wsm = MAX_JR / rsm;
    if (wsm > 8) wsm = 8;
    for (; xs > 0 && xs < ng && wsm > cf.W; --wsm) {   // the widest window whose buffers fit
      const int wfs = wsm + (maxd > 1 ? maxd - 1 : 0);   // TDT: the window plus the largest jump
      const Layout L2 = make_layout(bf, lstm, H, P, V1, nD, cf.R, cf.W, wfs, cf.C, 0, 0, true, nl, otf ? De : 0,
                                    rsm * wsm);
      if (L2.total + sizeof(RowState) + 1024 <= SMEM_LIMIT) {
        cf.L = L2;
        cf.WF = wfs;
        gp_small = xs;
        gp_rsmall = rsm;
        gp_wsmall = wsm;
        break;
      }
    }
  }
  const int C = cf.C, R = cf.R;
  const Layout &L = cf.L;

  cudaStream_t st = (cudaStream_t)stream;
  const bool ring = bf && lstm;
  uint8_t *ws = (uint8_t *)workspace;
  const Ws w = ws_layout(B, T_max, pr, jn, dt);
  if (cudaMemsetAsync(ws, 0, HDR_BYTES, st) != cudaSuccess) return LL_ERR_CUDA;
  if (B == 0) return LL_OK;

  // (1) encoder projection for all frames: f [B*T_max, H]
  // (frames t >= lengths[b] are never read: the tcgen05 GEMM skips tiles of
  // padding frames; a length > T_max is clamped here and reported by the decode)
  // -- not under OTF: the decode kernel projects the encoder rows it evaluates
  if (!otf) {
    s = linear(bf, enc, De, jn->w_enc, De, jn->b_enc, nullptr, ws + w.f, H, B * T_max, H, De, bf, st, lengths, T_max);
    if (s != LL_OK) return s;
  }
  // (2) model tables (weight-only; skipped if ll_prepare built exactly these
  // into this workspace)
  float *tab = (float *)(ws + w.tab);
  {
    const TableKey key = table_key(pr, jn, dt, C, L, workspace_bytes);
    bool cached = false;
    {
      std::lock_guard<std::mutex> lk(g_prep_mu);
      auto it = g_prepared.find(workspace);
      if (it != g_prepared.end()) {
        cached = it->second == key;
        if (!cached) g_prepared.erase(it);   // about to be overwritten with other tables
      }
    }
    if (!cached) {
      s = build_tables(bf, pr, jn, dt, w, ws, C, L, st);
      if (s != LL_OK) return s;
    }
  }
  // (3) decode
  DecodeParams p;
  memset(&p, 0, sizeof(p));
  p.B = B; p.T_max = T_max; p.H = H; p.P = P; p.V1 = V1; p.nD = nD;
  p.blank = blank_id; p.max_sym = max_symbols; p.tdt = tdt ? 1 : 0;
  for (int i = 0; i < nD; ++i) p.durations[i] = durations[i];
  p.context = lstm ? 1 : pr->context;
  p.R = R;
  p.W = cf.W;
  p.WF = cf.WF;
  p.NS = cf.NS;
  p.n_groups = (B + R - 1) / R;
  p.cap = cap;
  p.L = L;
  p.spec_prefetch = frame_looping ? 0 : (g_opt.spec_prefetch < 0 ? 1 : g_opt.spec_prefetch);
  p.gp_small = gp_small;
  p.gp_rsmall = gp_rsmall;
  p.gp_wsmall = gp_wsmall;
  // more than one group and no unequal plan: groups of length-ranked utterances
  if (g_opt.group_plan != 0 && gp_small == 0 && p.n_groups > 1 && B <= 65536) {   // O(B^2) ranking
    int *perm = (int *)(ws + w.perm);
    ++g_nlaunch;
    rank_lengths_kernel<<<(B + 255) / 256, 256, 0, st>>>(lengths, B, T_max, perm);
    if (cudaPeekAtLastError() != cudaSuccess) return LL_ERR_CUDA;
    p.perm = perm;
  }
  p.frame_looping = frame_looping ? 1 : 0;
  p.sched = g_opt.schedule < 0 ? 1 : g_opt.schedule;
  p.lengths = lengths;
  p.f = otf ? enc : (const void *)(ws + w.f);
  if (L.tj && bf && !otf) p.fmap_ok = make_fmap(&p.fmap, ws + w.f, (uint64_t)B * T_max, H, cf.WF) ? 1 : 0;
  if (otf) {   // encoder rows by one bulk copy per frame (fmap_ok = 0)
    p.De = De;
    p.w_enc = jn->w_enc;
    p.b_enc = jn->b_enc;
  }
  p.w_out = jn->w_out; p.b_out = jn->b_out; p.w_dur = jn->w_dur; p.b_dur = jn->b_dur;
  p.w_pred = jn->w_pred; p.b_pred = jn->b_pred; p.w_hh = lstm ? pr->w_hh : nullptr;
  p.layers = lstm ? nl : 1;
  if (lstm && nl > 1) {
    p.w_ih_rest = pr->w_ih_rest; p.w_hh_rest = pr->w_hh_rest; p.b_ih_rest = pr->b_ih_rest; p.b_hh_rest = pr->b_hh_rest;
  }
  p.tab = tab;
  p.wst = ring ? (const bf16 *)(ws + w.wst) : nullptr;
  p.h = lstm ? (void *)(ws + w.h) : nullptr;
  p.gglob = lstm ? (float *)(ws + w.g) : nullptr;
  p.out_tokens = out_tokens; p.out_timestamps = out_timestamps;
  p.out_durations = tdt ? out_durations : nullptr;
  p.out_lengths = out_lengths;
  p.out_scores = out_scores;
  p.status = (int *)ws;
  p.group_counter = (int *)ws + 1;
  p.stats = (unsigned long long *)(ws + 64);
  // debug builds only: per-warp clock64 timeline of block 0 ([2][TL_N][TL_PH][MAX_NW]
  // u64, tools/timeline.py) and host-mapped progress markers (tools/hang_trace.py)
  p.prof = (unsigned long long *)g_opt.timeline;
  p.trace = (volatile unsigned *)g_opt.trace;
  // probe (parity tests): the FC tick-schedule kernels with the probe hook
  const bool probe = g_opt.probe_logits != nullptr;
  if (probe) {
    if (frame_looping || p.sched != 1 || !is_fc(bf, H, P, C) || !g_opt.probe_lmeta || !g_opt.probe_g ||
        !g_opt.probe_gmeta || !g_opt.probe_counts || g_opt.probe_rows < 1 || g_opt.probe_regions < 1)
      return LL_ERR_UNSUPPORTED;
    p.probe_logits = g_opt.probe_logits; p.probe_lmeta = g_opt.probe_lmeta;
    p.probe_g = g_opt.probe_g; p.probe_gmeta = g_opt.probe_gmeta; p.probe_counts = g_opt.probe_counts;
    p.probe_rows = g_opt.probe_rows; p.probe_regions = g_opt.probe_regions;
    p.probe_stall = g_opt.probe_stall;
    if (cudaMemsetAsync(p.probe_counts, 0, sizeof(int) * 2 * p.probe_regions, st) != cudaSuccess) return LL_ERR_CUDA;
  }
  int used = 0;
  p.n_launch = g_nlaunch + 1;   // this call's kernels, the decode kernel included (ll_stats [12])
  if (g_ev_before && cudaEventRecord(g_ev_before, st) != cudaSuccess) return LL_ERR_CUDA;
  if (otf) {             // on-the-fly projections (Table 3's ablation arm)
    s = tdt ? launch_decode<bf16, 0, KREG, FC_H, FC_P, FC_C, 4, 2>(p, C, L, p.n_groups, st, used)
            : launch_decode<bf16, 0, KREG, FC_H, FC_P, FC_C, 4, 1>(p, C, L, p.n_groups, st, used);
  } else if (frame_looping) {   // Alg. 2 baseline instantiations
    if (is_fc(bf, H, P, C))
      s = lstm ? launch_decode<bf16, 0, KREG, FC_H, FC_P, FC_C, 3, 1>(p, C, L, p.n_groups, st, used)
               : launch_decode<bf16, 1, KREG, FC_H, FC_P, FC_C, 3, 1>(p, C, L, p.n_groups, st, used);
    else if (bf && kreg_for(bf, H) == KREG)
      s = lstm ? launch_decode<bf16, 0, KREG, 0, 0, 0, 3>(p, C, L, p.n_groups, st, used)
               : launch_decode<bf16, 1, KREG, 0, 0, 0, 3>(p, C, L, p.n_groups, st, used);
    else if (bf)
      s = lstm ? launch_decode<bf16, 0, KREG_SMALL, 0, 0, 0, 3>(p, C, L, p.n_groups, st, used)
               : launch_decode<bf16, 1, KREG_SMALL, 0, 0, 0, 3>(p, C, L, p.n_groups, st, used);
    else
      s = lstm ? launch_decode<float, 0, 1, 0, 0, 0, 3>(p, C, L, p.n_groups, st, used)
               : launch_decode<float, 1, 1, 0, 0, 0, 3>(p, C, L, p.n_groups, st, used);
  } else if (sc) {      // greedy scores: tick-schedule kernels with the score epilogue
    if (is_fc(bf, H, P, C)) {
      if (lstm)
        s = tdt ? launch_decode<bf16, 0, KREG, FC_H, FC_P, FC_C, 1, 2, 0, 1>(p, C, L, p.n_groups, st, used)
                : launch_decode<bf16, 0, KREG, FC_H, FC_P, FC_C, 1, 1, 0, 1>(p, C, L, p.n_groups, st, used);
      else
        s = tdt ? launch_decode<bf16, 1, KREG, FC_H, FC_P, FC_C, 1, 2, 0, 1>(p, C, L, p.n_groups, st, used)
                : launch_decode<bf16, 1, KREG, FC_H, FC_P, FC_C, 1, 1, 0, 1>(p, C, L, p.n_groups, st, used);
    } else if (bf && kreg_for(bf, H) == KREG) {
      s = lstm ? launch_decode<bf16, 0, KREG, 0, 0, 0, 1, 0, 0, 1>(p, C, L, p.n_groups, st, used)
               : launch_decode<bf16, 1, KREG, 0, 0, 0, 1, 0, 0, 1>(p, C, L, p.n_groups, st, used);
    } else if (bf) {
      s = lstm ? launch_decode<bf16, 0, KREG_SMALL, 0, 0, 0, 1, 0, 0, 1>(p, C, L, p.n_groups, st, used)
               : launch_decode<bf16, 1, KREG_SMALL, 0, 0, 0, 1, 0, 0, 1>(p, C, L, p.n_groups, st, used);
    } else {
      s = lstm ? launch_decode<float, 0, 1, 0, 0, 0, 1, 0, 0, 1>(p, C, L, p.n_groups, st, used)
               : launch_decode<float, 1, 1, 0, 0, 0, 1, 0, 0, 1>(p, C, L, p.n_groups, st, used);
    }
  } else if (probe) {   // the production FC tick kernels + the probe hook (ll.h ll_options)
    if (lstm)
      s = tdt ? launch_decode<bf16, 0, KREG, FC_H, FC_P, FC_C, 1, 2, 1>(p, C, L, p.n_groups, st, used)
              : launch_decode<bf16, 0, KREG, FC_H, FC_P, FC_C, 1, 1, 1>(p, C, L, p.n_groups, st, used);
    else
      s = tdt ? launch_decode<bf16, 1, KREG, FC_H, FC_P, FC_C, 1, 2, 1>(p, C, L, p.n_groups, st, used)
              : launch_decode<bf16, 1, KREG, FC_H, FC_P, FC_C, 1, 1, 1>(p, C, L, p.n_groups, st, used);
  } else if (is_fc(bf, H, P, C)) {   // one instantiation per (predictor, family, schedule)
    const int k = (tdt ? 2 : 0) + (p.sched == 1 ? 0 : 1);
    if (lstm) {
      if (k == 0) s = launch_decode<bf16, 0, KREG, FC_H, FC_P, FC_C, 1, 1>(p, C, L, p.n_groups, st, used);
      else if (k == 1) s = launch_decode<bf16, 0, KREG, FC_H, FC_P, FC_C, 2, 1>(p, C, L, p.n_groups, st, used);
      else if (k == 2) s = launch_decode<bf16, 0, KREG, FC_H, FC_P, FC_C, 1, 2>(p, C, L, p.n_groups, st, used);
      else s = launch_decode<bf16, 0, KREG, FC_H, FC_P, FC_C, 2, 2>(p, C, L, p.n_groups, st, used);
    } else {
      if (k == 0) s = launch_decode<bf16, 1, KREG, FC_H, FC_P, FC_C, 1, 1>(p, C, L, p.n_groups, st, used);
      else if (k == 1) s = launch_decode<bf16, 1, KREG, FC_H, FC_P, FC_C, 2, 1>(p, C, L, p.n_groups, st, used);
      else if (k == 2) s = launch_decode<bf16, 1, KREG, FC_H, FC_P, FC_C, 1, 2>(p, C, L, p.n_groups, st, used);
      else s = launch_decode<bf16, 1, KREG, FC_H, FC_P, FC_C, 2, 2>(p, C, L, p.n_groups, st, used);
    }
  }
  else if (bf && kreg_for(bf, H) == KREG)
    s = lstm ? launch_decode<bf16, 0, KREG>(p, C, L, p.n_groups, st, used)
             : launch_decode<bf16, 1, KREG>(p, C, L, p.n_groups, st, used);
  else if (bf)
    s = lstm ? launch_decode<bf16, 0, KREG_SMALL>(p, C, L, p.n_groups, st, used)
             : launch_decode<bf16, 1, KREG_SMALL>(p, C, L, p.n_groups, st, used);
  else
    s = lstm ? launch_decode<float, 0, 1>(p, C, L, p.n_groups, st, used)
             : launch_decode<float, 1, 1>(p, C, L, p.n_groups, st, used);
  if (s == LL_OK && g_ev_after && cudaEventRecord(g_ev_after, st) != cudaSuccess) return LL_ERR_CUDA;
  return s;
}

}  // namespace

extern "C" {

ll_status ll_set_timing_events(void *ev_before_decode, void *ev_after_decode) {
  if ((ev_before_decode == nullptr) != (ev_after_decode == nullptr)) return LL_ERR_INVALID_ARGUMENT;
  g_ev_before = (cudaEvent_t)ev_before_decode;
  g_ev_after = (cudaEvent_t)ev_after_decode;
  return LL_OK;
}

const char *ll_version(void) { return "ll 0.2 (sm_100a, label-looping arXiv 2406.06220)"; }

ll_status ll_release(void *workspace) {
  if (!workspace) return LL_OK;
  std::lock_guard<std::mutex> lk(g_prep_mu);
  g_prepared.erase(workspace);
  return LL_OK;
}

ll_status ll_set_options(const ll_options *o) {
  if (!o) {
    g_opt = default_options();
    return LL_OK;
  }
  if (o->cluster_size < 0 || o->cluster_size > MAX_C || o->group_rows < 0 || o->group_rows > MAX_R ||
      o->window < 0 || o->window > 8 || o->max_clusters < 0 || o->schedule < -1 || o->schedule > 1 ||
      o->spec_prefetch < -1 || o->spec_prefetch > 1 || o->probe_rows < 0 || o->probe_regions < 0 ||
      o->projections < 0 || o->projections > 1 || o->probe_stall < 0 || o->group_plan < -1 ||
      o->group_plan > 1)
    return LL_ERR_INVALID_ARGUMENT;
  g_opt = *o;
  return LL_OK;
}

const char *ll_status_string(ll_status s) {
  switch (s) {
    case LL_OK: return "LL_OK";
    case LL_ERR_INVALID_ARGUMENT: return "LL_ERR_INVALID_ARGUMENT";
    case LL_ERR_UNSUPPORTED: return "LL_ERR_UNSUPPORTED";
    case LL_ERR_WORKSPACE: return "LL_ERR_WORKSPACE";
    case LL_ERR_CUDA: return "LL_ERR_CUDA";
    case LL_ERR_CAPACITY: return "LL_ERR_CAPACITY";
    default: return "LL_ERR_UNKNOWN";
  }
}

size_t ll_workspace_size(int32_t B, int32_t T_max, const ll_predictor *pred, const ll_joint *joint,
                         ll_dtype dtype, ll_prec prec, int32_t num_durations) {
  if (B < 0 || T_max < 0 || !pred || !joint) return 0;
  if (check_model(pred, joint, dtype, prec, num_durations, false) == LL_ERR_INVALID_ARGUMENT) return 0;
  if (pred->kind != LL_PRED_LSTM && pred->kind != LL_PRED_STATELESS) return 0;
  if (pred->kind == LL_PRED_STATELESS && pred->context < 1) return 0;
  if (widened(pred, dtype, prec))   // the fp32 call's workspace, then the fp32 copies
    return align_up(ws_layout(B, T_max, pred, joint, LL_F32).total, 256) +
           wide_bytes(B, T_max, pred, joint, num_durations > 0 ? num_durations : 0);
  return ws_layout(B, T_max, pred, joint, dtype).total;
}

ll_status ll_decode_rnnt(const void *enc, ll_dtype dtype, ll_prec prec, int32_t B, int32_t T_max,
                         const int32_t *lengths, const ll_predictor *pred, const ll_joint *joint,
                         int32_t blank_id, int32_t max_symbols, int32_t *out_tokens,
                         int32_t *out_timestamps, int32_t *out_lengths, int32_t out_capacity,
                         void *workspace, size_t workspace_bytes, ll_stream stream) {
  g_nlaunch = 0;
  return decode_impl(false, false, enc, dtype, prec, B, T_max, lengths, pred, joint, blank_id, max_symbols,
                     nullptr, 0, out_tokens, out_timestamps, nullptr, out_lengths, out_capacity, workspace,
                     workspace_bytes, stream);
}

ll_status ll_decode_rnnt_scores(const void *enc, ll_dtype dtype, ll_prec prec, int32_t B, int32_t T_max,
                                const int32_t *lengths, const ll_predictor *pred, const ll_joint *joint,
                                int32_t blank_id, int32_t max_symbols, int32_t *out_tokens,
                                int32_t *out_timestamps, int32_t *out_lengths, int32_t out_capacity,
                                float *out_scores, void *workspace, size_t workspace_bytes, ll_stream stream) {
  g_nlaunch = 0;
  if (B > 0 && !out_scores) return LL_ERR_INVALID_ARGUMENT;
  return decode_impl(false, false, enc, dtype, prec, B, T_max, lengths, pred, joint, blank_id, max_symbols,
                     nullptr, 0, out_tokens, out_timestamps, nullptr, out_lengths, out_capacity, workspace,
                     workspace_bytes, stream, out_scores);
}

ll_status ll_decode_tdt_scores(const void *enc, ll_dtype dtype, ll_prec prec, int32_t B, int32_t T_max,
                               const int32_t *lengths, const ll_predictor *pred, const ll_joint *joint,
                               int32_t blank_id, int32_t max_symbols, const int32_t *durations,
                               int32_t num_durations, int32_t *out_tokens, int32_t *out_timestamps,
                               int32_t *out_durations, int32_t *out_lengths, int32_t out_capacity,
                               float *out_scores, void *workspace, size_t workspace_bytes, ll_stream stream) {
  g_nlaunch = 0;
  if (B > 0 && !out_scores) return LL_ERR_INVALID_ARGUMENT;
  return decode_impl(true, false, enc, dtype, prec, B, T_max, lengths, pred, joint, blank_id, max_symbols,
                     durations, num_durations, out_tokens, out_timestamps, out_durations, out_lengths,
                     out_capacity, workspace, workspace_bytes, stream, out_scores);
}

ll_status ll_decode_rnnt_frame_looping(const void *enc, ll_dtype dtype, ll_prec prec, int32_t B, int32_t T_max,
                                       const int32_t *lengths, const ll_predictor *pred, const ll_joint *joint,
                                       int32_t blank_id, int32_t max_symbols, int32_t *out_tokens,
                                       int32_t *out_timestamps, int32_t *out_lengths, int32_t out_capacity,
                                       void *workspace, size_t workspace_bytes, ll_stream stream) {
  g_nlaunch = 0;
  return decode_impl(false, true, enc, dtype, prec, B, T_max, lengths, pred, joint, blank_id, max_symbols,
                     nullptr, 0, out_tokens, out_timestamps, nullptr, out_lengths, out_capacity, workspace,
                     workspace_bytes, stream);
}

ll_status ll_decode_tdt(const void *enc, ll_dtype dtype, ll_prec prec, int32_t B, int32_t T_max,
                        const int32_t *lengths, const ll_predictor *pred, const ll_joint *joint,
                        int32_t blank_id, int32_t max_symbols, const int32_t *durations,
                        int32_t num_durations, int32_t *out_tokens, int32_t *out_timestamps,
                        int32_t *out_durations, int32_t *out_lengths, int32_t out_capacity,
                        void *workspace, size_t workspace_bytes, ll_stream stream) {
  g_nlaunch = 0;
  return decode_impl(true, false, enc, dtype, prec, B, T_max, lengths, pred, joint, blank_id, max_symbols,
                     durations, num_durations, out_tokens, out_timestamps, out_durations, out_lengths,
                     out_capacity, workspace, workspace_bytes, stream);
}

ll_status ll_prepare(const ll_predictor *pred, const ll_joint *joint, ll_dtype dtype, ll_prec prec, int32_t B,
                     int32_t T_max, const int32_t *durations, int32_t num_durations, void *workspace,
                     size_t workspace_bytes, ll_stream stream) {
  if (B < 0 || T_max < 0) return LL_ERR_INVALID_ARGUMENT;
  if (!workspace || ((uintptr_t)workspace & 255)) return LL_ERR_INVALID_ARGUMENT;
  const int nD = durations ? num_durations : 0;
  if (durations) {
    if (nD < 1) return LL_ERR_INVALID_ARGUMENT;
    for (int i = 0; i < nD; ++i)
      if (durations[i] < 0) return LL_ERR_INVALID_ARGUMENT;
  }
  ll_status s = check_model(pred, joint, dtype, prec, nD, true);
  if (s != LL_OK) return s;
  if (workspace_bytes < ll_workspace_size(B, T_max, pred, joint, dtype, prec, nD)) return LL_ERR_WORKSPACE;
  if (widened(pred, dtype, prec)) return LL_OK;   // tables rebuilt by every such decode (no record)
  const bool bf = dtype == LL_BF16, lstm = pred->kind == LL_PRED_LSTM;
  int maxd = 1;
  for (int i = 0; i < nD; ++i) maxd = durations[i] > maxd ? durations[i] : maxd;
  Config cf;
  if (!decode_config(bf, lstm, joint->joint_dim, joint->pred_dim, joint->num_outputs, nD, maxd, B, cf, 0,
                     nlayers(pred)))
    return LL_ERR_UNSUPPORTED;
  const Ws w = ws_layout(B, T_max, pred, joint, dtype);
  s = build_tables(bf, pred, joint, dtype, w, (uint8_t *)workspace, cf.C, cf.L, (cudaStream_t)stream);
  if (s != LL_OK) return s;
  std::lock_guard<std::mutex> lk(g_prep_mu);
  g_prepared[workspace] = table_key(pred, joint, dtype, cf.C, cf.L, workspace_bytes);
  return LL_OK;
}

ll_status ll_sync(void *workspace, ll_stream stream) {
  if (!workspace) return LL_ERR_INVALID_ARGUMENT;
  if (cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) return LL_ERR_CUDA;
  int status = 0;
  if (cudaMemcpy(&status, workspace, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess) return LL_ERR_CUDA;
  if (status & 4) return LL_ERR_CUDA;        // internal: misaligned shared-memory operand base
  if (status & 2) return LL_ERR_CAPACITY;
  if (status & 1) return LL_ERR_INVALID_ARGUMENT;
  return LL_OK;
}

ll_status ll_stats(const void *workspace, uint64_t *out, ll_stream stream) {
  if (!workspace || !out) return LL_ERR_INVALID_ARGUMENT;
  if (cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) return LL_ERR_CUDA;
  if (cudaMemcpy(out, (const uint8_t *)workspace + 64, 13 * sizeof(uint64_t), cudaMemcpyDeviceToHost) !=
      cudaSuccess)
    return LL_ERR_CUDA;
  return LL_OK;
}

ll_status ll_debug_joint(const void *enc_rows, const float *g_rows, int32_t n, const ll_joint *joint,
                         ll_dtype dtype, ll_prec prec, int32_t num_durations, float *out_logits,
                         int32_t *out_argmax, int32_t *out_dur_argmax, void *workspace,
                         size_t workspace_bytes, ll_stream stream) {
  if (n < 0) return LL_ERR_INVALID_ARGUMENT;
  if (!workspace || ((uintptr_t)workspace & 255)) return LL_ERR_INVALID_ARGUMENT;
  ll_status s = check_model(nullptr, joint, dtype, prec, num_durations, false);
  if (s != LL_OK) return s;
  if (n > 0 && (!enc_rows || !g_rows || !out_argmax)) return LL_ERR_INVALID_ARGUMENT;
  {   // this call overwrites the workspace with its own layout: drop any prepared tables
    std::lock_guard<std::mutex> lk(g_prep_mu);
    g_prepared.erase(workspace);
  }
  ll_predictor dummy = {};
  dummy.kind = LL_PRED_STATELESS;
  dummy.context = 1;
  dummy.num_tokens = joint->num_outputs;
  dummy.hidden = joint->pred_dim;
  if (workspace_bytes < ll_workspace_size(n, 1, &dummy, joint, dtype, prec, num_durations))
    return LL_ERR_WORKSPACE;
  ll_release(workspace);   // its f rows overwrite the region prepared tables would occupy
  if (dtype == LL_BF16 && prec == LL_PREC_EXACT) {   // the fp32 joint on fp32 copies (see widened())
    if (n == 0) return LL_OK;
    const size_t inner = align_up(ws_layout(n, 1, &dummy, joint, LL_F32).total, 256);
    ll_joint jn32;
    ll_status ws_s = LL_OK;
    float *rows32 = widen_all(enc_rows, (size_t)n * joint->enc_dim, nullptr, joint, num_durations, nullptr, &jn32,
                              (uint8_t *)workspace + inner, (cudaStream_t)stream, ws_s);
    if (ws_s != LL_OK) return ws_s;
    return ll_debug_joint(rows32, g_rows, n, &jn32, LL_F32, LL_PREC_FAST, num_durations, out_logits, out_argmax,
                          out_dur_argmax, workspace, inner, stream);
  }
  const bool bf = dtype == LL_BF16;
  const int H = joint->joint_dim, V1 = joint->num_outputs, De = joint->enc_dim;
  Config cf;
  if (!choose_config(bf, false, H, joint->pred_dim, V1, num_durations, 1, 16 * 8, cf)) return LL_ERR_UNSUPPORTED;
  cf.R = 16; cf.W = 1; cf.WF = 1; cf.NS = 0;
  cf.L = make_layout(bf, false, H, joint->pred_dim, V1, num_durations, 16, 1, 1, cf.C, 0, 0, false);
  const int C = cf.C, R = cf.R;
  const Layout &L = cf.L;
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t *ws = (uint8_t *)workspace;
  const Ws w = ws_layout(n, 1, &dummy, joint, dtype);
  if (n == 0) return LL_OK;
  s = linear(bf, enc_rows, De, joint->w_enc, De, joint->b_enc, nullptr, ws + w.f, H, n, H, De, bf, st);
  if (s != LL_OK) return s;
  DecodeParams p;
  memset(&p, 0, sizeof(p));
  p.B = n; p.T_max = 1; p.H = H; p.P = joint->pred_dim; p.V1 = V1; p.nD = num_durations;
  p.tdt = num_durations > 0 ? 1 : 0;   // the joint's duration head
  p.R = R;
  p.W = 1;
  p.WF = 1;
  p.f = ws + w.f;
  p.w_out = joint->w_out; p.b_out = joint->b_out; p.w_dur = joint->w_dur; p.b_dur = joint->b_dur;
  p.dbg_g = g_rows; p.dbg_logits = out_logits; p.dbg_argmax = out_argmax; p.dbg_dargmax = out_dur_argmax;
  p.L = L;
  p.dbg_n = n;
  const int chunks = (n + R - 1) / R;
  if (bf && kreg_for(bf, H) == KREG) return launch_debug<bf16, KREG>(p, C, L, chunks, st);
  if (bf) return launch_debug<bf16, KREG_SMALL>(p, C, L, chunks, st);
  return launch_debug<float, 1>(p, C, L, chunks, st);
}

}  // extern "C"
