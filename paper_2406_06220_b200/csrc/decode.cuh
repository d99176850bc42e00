// decode.cuh -- persistent thread-block-cluster kernel for batched label-looping
// greedy decoding of RNN-T and TDT (arXiv 2406.06220, Alg. 3 PAPER.md:129-159,
// TDT PAPER.md:211-213).
//
// One cluster of C CTAs decodes one GROUP of up to R utterances at a time
// (groups are taken from a device work counter, so any number of clusters /
// groups works).  Inside a group the control loop of Alg. 3 runs entirely on
// the device:
//
//   outer step (label loop, Alg. 3 line 5):
//     predictor phase   rows that found a label and are still active:
//                       LSTM  gates = E'[y] + W_hh h  (tensor cores, W_hh streamed
//                             from L2, gate nonlinearities + cell update fused in the
//                             epilogue; c stays in the owner CTA), g = W_pred h' + b_pred
//                       stateless  g = sum_k G_k[ctx_k]  (precomputed tables)
//     scan (frame loop, Alg. 3 lines 7-19), one ROUND per inner iteration:
//       z = ReLU(f[b, t_b] + g_b) for the scanning rows (compacted), bf16
//       joint GEMM [M x H] x [H x slice of V+1(+|D|)] on the CTA's resident
//       weight slice, argmax fused into the epilogue (packed 64-bit keys, warp
//       shuffles), per-CTA partial keys broadcast to every CTA through
//       distributed shared memory, one cluster barrier, then every CTA reduces
//       the C partials and applies the same time rules -> replicated row state.
//       Next frame rows f[b, t+1] are prefetched speculatively (RNN-T).
//     append + time rules + guard (BatchedHyps add_results):
//       masked append into the caller's preallocated [B, cap] buffers, lanes =
//       rows of the group (no atomics: each row has one owner lane).
//
// Weights stay resident in shared memory (joint slice) for the whole kernel;
// no host synchronisation happens until the caller's ll_sync.
#pragma once
#include "common.cuh"

namespace ll {

constexpr int MAX_R = 32;        // rows per group (<= 32: one lane per row)
constexpr int MAX_DUR = 16;
constexpr int MAX_CTX = 4;
constexpr int MAX_NW = 12;       // warps per CTA (<= 384 threads: up to 168 registers)

struct DecodeParams {
  int B, T_max, H, P, V1, nD;
  int blank, max_sym, tdt;
  int durations[MAX_DUR];
  int context;
  int R, n_groups, cap;
  int spec_prefetch;             // speculative next-frame prefetch (RNN-T)
  const int *lengths;
  const void *f;                 // [B, T_max, H] bf16 (bf16 path) / f32
  const void *w_out, *b_out, *w_dur, *b_dur;
  const void *w_pred, *b_pred, *w_hh;
  const float *tab;              // LSTM: E' [V1][4P]; stateless: G [ctx][V1][H] (b_pred in G_0)
  void *h;                       // LSTM: [2][B][P] (bf16 / f32)
  float *gglob;                  // LSTM: [B][H]
  int *out_tokens, *out_timestamps, *out_durations, *out_lengths;
  int *status;                   // bit0 bad length, bit1 capacity
  int *group_counter;
  unsigned long long *stats;     // see ll.h ll_stats
  // ll_debug_joint mode
  const float *dbg_g;
  float *dbg_logits;
  int *dbg_argmax, *dbg_dargmax;
  int dbg_n;
};

// Shared-memory layout (identical on host and device).
struct Layout {
  int wstride, zstride, tiles_max, UPC, DPC, NW;
  size_t off_w, off_b, off_z, off_f, off_g, off_c, off_part, off_wkey, total;
};

__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

__host__ __device__ inline Layout make_layout(bool bf, int H, int P, int V1, int nD, int R, int C,
                                              bool lstm) {
  Layout L;
  const int NT = (V1 + nD + 7) / 8;
  L.tiles_max = (NT + C - 1) / C;
  L.UPC = lstm ? P / C : 0;
  L.DPC = H / C;
  int nw = bf ? L.tiles_max : 8;
  if (nw < 8) nw = 8;
  if (nw > MAX_NW) nw = MAX_NW;
  L.NW = nw;
  const int K = H > P ? H : P;
  L.wstride = bf ? (int)(align_up((size_t)H * 2, 128) + 64) : 0;
  L.zstride = bf ? (int)(align_up((size_t)K * 2, 128) + 64) : K * 4;
  size_t o = 0;
  L.off_w = o;    o = align_up(o + (bf ? (size_t)L.tiles_max * 8 * L.wstride : 0), 128);
  L.off_b = o;    o = align_up(o + (size_t)L.tiles_max * 8 * 4, 128);
  L.off_z = o;    o = align_up(o + (size_t)R * L.zstride, 128);
  L.off_f = o;    o = align_up(o + (size_t)2 * R * H * (bf ? 2 : 4), 128);
  L.off_g = o;    o = align_up(o + (size_t)R * H * 4, 128);
  L.off_c = o;    o = align_up(o + (size_t)R * (lstm ? L.UPC : 0) * 4, 128);
  L.off_part = o; o = align_up(o + (size_t)2 * C * R * 16, 128);
  L.off_wkey = o; o = align_up(o + (size_t)L.NW * R * 16, 128);
  L.total = o;
  return L;
}

struct RowState {
  int b[MAX_R], L[MAX_R], t[MAX_R], k[MAX_R], len[MAX_R], last[MAX_R], hpar[MAX_R], hzero[MAX_R];
  int ctx[MAX_CTX][MAX_R];
  int active[MAX_R], scanning[MAX_R], found[MAX_R], needp[MAX_R];
  int fy[MAX_R], ft[MAX_R], fd[MAX_R];
  int slist[MAX_R], plist[MAX_R];
  int nscan, npred, nactive;
  int grp;
};

// Per-CTA context of the cluster kernel.
template <typename T>
struct Ctx {
  static constexpr bool BF = sizeof(T) == 2;
  const DecodeParams &p;
  Layout L;
  uint8_t *sm;
  RowState &rs;
  int C, rank, tid, warp, lane, NW, g, q;
  int tile0, ntiles;          // vocab n8 tiles owned by this CTA
  int u0, d0;                 // LSTM units / W_pred output dims owned
  int par;                    // DSMEM partial-buffer parity
  __device__ Ctx(const DecodeParams &p_, uint8_t *sm_, RowState &rs_, bool lstm)
      : p(p_), sm(sm_), rs(rs_) {
    C = (int)cluster_size();
    rank = (int)cluster_rank();
    L = make_layout(BF, p.H, p.P, p.V1, p.nD, p.R, C, lstm);
    tid = threadIdx.x; warp = tid >> 5; lane = tid & 31; NW = blockDim.x >> 5;
    g = lane >> 2; q = lane & 3;
    const int NT = (p.V1 + p.nD + 7) / 8;
    const int base = NT / C, rem = NT % C;
    ntiles = base + (rank < rem ? 1 : 0);
    tile0 = rank * base + (rank < rem ? rank : rem);
    u0 = rank * L.UPC;
    d0 = rank * L.DPC;
    par = 0;
  }
  __device__ uint8_t *wsl() const { return sm + L.off_w; }
  __device__ float *bsl() const { return (float *)(sm + L.off_b); }
  __device__ uint8_t *zs() const { return sm + L.off_z; }
  __device__ uint8_t *fbuf(int cur) const {
    return sm + L.off_f + (size_t)cur * p.R * p.H * sizeof(T);
  }
  __device__ float *gs() const { return (float *)(sm + L.off_g); }
  __device__ float *cs() const { return (float *)(sm + L.off_c); }
  __device__ uint64_t *part(int pr) const {
    return (uint64_t *)(sm + L.off_part) + (size_t)pr * C * p.R * 2;
  }
  __device__ uint64_t *wkey() const { return (uint64_t *)(sm + L.off_wkey); }

  // -------------------------------------------------------------------------
  // Load this CTA's slice of [W_out; W_dur] (rows tile0*8 ...) into shared
  // memory once per kernel (bf16 path), and the matching bias slice (fp32).
  // -------------------------------------------------------------------------
  __device__ void load_weight_slice() {
    const int nrows = L.tiles_max * 8;
    const int V1 = p.V1, NV = p.V1 + p.nD, H = p.H;
    float *bs = bsl();
    for (int r = tid; r < nrows; r += blockDim.x) {
      const int v = tile0 * 8 + r;
      float bv = 0.f;
      if (r < ntiles * 8 && v < NV) {
        bv = v < V1 ? to_f32(((const T *)p.b_out)[v]) : to_f32(((const T *)p.b_dur)[v - V1]);
      }
      bs[r] = bv;
    }
    if constexpr (BF) {
      const int chunks = H / 8;  // 16-byte chunks per row
      for (int idx = tid; idx < nrows * chunks; idx += blockDim.x) {
        const int r = idx / chunks, c = idx % chunks;
        const int v = tile0 * 8 + r;
        uint4 val = make_uint4(0, 0, 0, 0);
        if (r < ntiles * 8 && v < NV) {
          const bf16 *src = v < V1 ? (const bf16 *)p.w_out + (size_t)v * H
                                   : (const bf16 *)p.w_dur + (size_t)(v - V1) * H;
          val = ldg128_nc(src + c * 8);
        }
        *reinterpret_cast<uint4 *>(wsl() + (size_t)r * L.wstride + c * 16) = val;
      }
    }
  }

  // f rows f[b, t] of the listed row slots into fbuf[cur][slot] (cp.async).
  __device__ void issue_f_loads(int cur, const int *slots, const int *tt, int n) {
    const int chunks = p.H * (int)sizeof(T) / 16;
    for (int idx = tid; idx < n * chunks; idx += blockDim.x) {
      const int i = idx / chunks, c = idx % chunks;
      const int s = slots[i];
      const int b = rs.b[s];
      const uint8_t *src = (const uint8_t *)p.f + ((size_t)b * p.T_max + tt[i]) * p.H * sizeof(T);
      cp_async16(fbuf(cur) + (size_t)s * p.H * sizeof(T) + c * 16, src + c * 16);
    }
    cp_async_commit();
  }

  // z[i] = ReLU(f[slot_i] + g[slot_i]) for i < M; rows M..Mpad-1 zero.
  __device__ void build_z(int cur, int M, int Mpad) {
    const int H = p.H;
    if constexpr (BF) {
      const int pairs = H / 2;
      for (int idx = tid; idx < Mpad * pairs; idx += blockDim.x) {
        const int i = idx / pairs, c = idx % pairs;
        uint32_t out = 0;
        if (i < M) {
          const int s = rs.slist[i];
          const uint32_t fw = *reinterpret_cast<const uint32_t *>(fbuf(cur) + ((size_t)s * H + 2 * c) * 2);
          const float2 gv = *reinterpret_cast<const float2 *>(gs() + (size_t)s * H + 2 * c);
          out = pack_bf16x2(fmaxf(bf16_lo(fw) + gv.x, 0.f), fmaxf(bf16_hi(fw) + gv.y, 0.f));
        }
        *reinterpret_cast<uint32_t *>(zs() + (size_t)i * L.zstride + c * 4) = out;
      }
    } else {
      for (int idx = tid; idx < Mpad * H; idx += blockDim.x) {
        const int i = idx / H, c = idx % H;
        float out = 0.f;
        if (i < M) {
          const int s = rs.slist[i];
          out = fmaxf(((const float *)fbuf(cur))[(size_t)s * H + c] + gs()[(size_t)s * H + c], 0.f);
        }
        ((float *)zs())[(size_t)i * (L.zstride / 4) + c] = out;
      }
    }
  }

  // -------------------------------------------------------------------------
  // Joint + fused argmax over this CTA's vocabulary slice.  Writes per-warp
  // keys wkey[warp][i] = {token key, duration key} for rows i < Mpad.
  // If `logits` != nullptr (debug), also writes raw logits [row_base+i][v].
  // -------------------------------------------------------------------------
  __device__ void joint_keys(int M, int MT, float *logits, int row_base) {
    const int V1 = p.V1, NV = p.V1 + p.nD, H = p.H;
    uint64_t *wk = wkey();
    if constexpr (BF) {
      uint64_t tk[2][2], dk[2][2];
#pragma unroll
      for (int a = 0; a < 2; ++a) tk[a][0] = tk[a][1] = dk[a][0] = dk[a][1] = 0;
      const int KB = H / 32;
      const bool tail = (H & 31) != 0;
      for (int j = warp; j < ntiles; j += NW) {
        float acc[2][4];
#pragma unroll
        for (int a = 0; a < 2; ++a) acc[a][0] = acc[a][1] = acc[a][2] = acc[a][3] = 0.f;
        const uint8_t *brow = wsl() + (size_t)(j * 8 + g) * L.wstride;
        const uint8_t *a0row = zs() + (size_t)g * L.zstride;
        const uint8_t *a1row = zs() + (size_t)(g + 8) * L.zstride;
        const uint8_t *a2row = zs() + (size_t)(g + 16) * L.zstride;
        const uint8_t *a3row = zs() + (size_t)(g + 24) * L.zstride;
#pragma unroll 4
        for (int kb = 0; kb < KB; ++kb) {
          const uint4 b = lds128(brow + kb * 64 + q * 16);
          const uint4 x0 = lds128(a0row + kb * 64 + q * 16);
          const uint4 x1 = lds128(a1row + kb * 64 + q * 16);
          mma_bf16_16816(acc[0], x0.x, x1.x, x0.y, x1.y, b.x, b.y);
          mma_bf16_16816(acc[0], x0.z, x1.z, x0.w, x1.w, b.z, b.w);
          if (MT > 1) {
            const uint4 x2 = lds128(a2row + kb * 64 + q * 16);
            const uint4 x3 = lds128(a3row + kb * 64 + q * 16);
            mma_bf16_16816(acc[1], x2.x, x3.x, x2.y, x3.y, b.x, b.y);
            mma_bf16_16816(acc[1], x2.z, x3.z, x2.w, x3.w, b.z, b.w);
          }
        }
        if (tail) {
          const uint2 b = lds64(brow + KB * 64 + q * 8);
          const uint2 x0 = lds64(a0row + KB * 64 + q * 8);
          const uint2 x1 = lds64(a1row + KB * 64 + q * 8);
          mma_bf16_16816(acc[0], x0.x, x1.x, x0.y, x1.y, b.x, b.y);
          if (MT > 1) {
            const uint2 x2 = lds64(a2row + KB * 64 + q * 8);
            const uint2 x3 = lds64(a3row + KB * 64 + q * 8);
            mma_bf16_16816(acc[1], x2.x, x3.x, x2.y, x3.y, b.x, b.y);
          }
        }
        // epilogue: bias, keys (and debug logits)
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          if (mt >= MT) break;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int rr = e >> 1;                       // 0: row g, 1: row g+8
            const int lr = (j * 8 + 2 * q + (e & 1));    // local vocab row
            const int v = tile0 * 8 + lr;
            const float val = acc[mt][e] + bsl()[lr];
            const int i = mt * 16 + g + rr * 8;
            if (v < V1) tk[mt][rr] = umax64(tk[mt][rr], pack_key(val, v));
            else if (v < NV) dk[mt][rr] = umax64(dk[mt][rr], pack_key(val, v - V1));
            if (logits != nullptr && i < M && v < NV)
              logits[(size_t)(row_base + i) * NV + v] = val;
          }
        }
      }
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          tk[mt][rr] = umax64(tk[mt][rr], shfl_xor_u64(tk[mt][rr], 1));
          tk[mt][rr] = umax64(tk[mt][rr], shfl_xor_u64(tk[mt][rr], 2));
          dk[mt][rr] = umax64(dk[mt][rr], shfl_xor_u64(dk[mt][rr], 1));
          dk[mt][rr] = umax64(dk[mt][rr], shfl_xor_u64(dk[mt][rr], 2));
        }
      if (q == 0) {
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int rr = 0; rr < 2; ++rr) {
            const int i = mt * 16 + g + rr * 8;
            if (i < p.R) {
              wk[((size_t)warp * p.R + i) * 2 + 0] = tk[mt][rr];
              wk[((size_t)warp * p.R + i) * 2 + 1] = dk[mt][rr];
            }
          }
      }
    } else {
      // fp32 SIMT: one warp per vocabulary row, lanes split K in a fixed order,
      // butterfly reduction; lane i keeps the best key of batch row i.
      uint64_t tkey = 0, dkey = 0;
      const int nrows = ntiles * 8;
      const int zst = L.zstride / 4;
      const float *z = (const float *)zs();
      for (int lr = warp; lr < nrows; lr += NW) {
        const int v = tile0 * 8 + lr;
        if (v >= NV) break;
        const float *wr = v < V1 ? (const float *)p.w_out + (size_t)v * H
                                 : (const float *)p.w_dur + (size_t)(v - V1) * H;
        float acc[MAX_R];
#pragma unroll
        for (int i = 0; i < MAX_R; ++i) acc[i] = 0.f;
        for (int k = lane; k < H; k += 32) {
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
        const float bv = bsl()[lr];
#pragma unroll
        for (int i = 0; i < MAX_R; ++i) {
          if (i < M && lane == i) {
            const float val = acc[i] + bv;
            if (v < V1) tkey = umax64(tkey, pack_key(val, v));
            else dkey = umax64(dkey, pack_key(val, v - V1));
            if (logits != nullptr) logits[(size_t)(row_base + i) * NV + v] = val;
          }
        }
      }
      if (lane < p.R) {
        wk[((size_t)warp * p.R + lane) * 2 + 0] = tkey;
        wk[((size_t)warp * p.R + lane) * 2 + 1] = dkey;
      }
    }
  }

  // Reduce per-warp keys and broadcast this CTA's partial to every CTA of the
  // cluster (distributed shared memory), then one cluster barrier.
  __device__ void exchange_keys(int M) {
    __syncthreads();
    const uint64_t *wk = wkey();
    uint64_t *pt = part(par);
    for (int idx = tid; idx < M * C; idx += blockDim.x) {
      const int i = idx / C, dst = idx % C;
      uint64_t tkey = 0, dkey = 0;
      for (int w = 0; w < NW; ++w) {
        tkey = umax64(tkey, wk[((size_t)w * p.R + i) * 2 + 0]);
        dkey = umax64(dkey, wk[((size_t)w * p.R + i) * 2 + 1]);
      }
      uint64_t *slot = pt + ((size_t)rank * p.R + i) * 2;
      if (C == 1) {
        slot[0] = tkey;
        slot[1] = dkey;
      } else {
        st_dsmem_u64x2(dsmem_addr(slot, (uint32_t)dst), tkey, dkey);
      }
    }
    if (C > 1) cluster_sync_all(); else __syncthreads();
  }

  // Final argmax of compact row i from the C partials (after exchange_keys).
  __device__ void final_keys(int i, int &y, int &di) const {
    const uint64_t *pt = part(par);
    uint64_t tkey = 0, dkey = 0;
    for (int r = 0; r < C; ++r) {
      tkey = umax64(tkey, pt[((size_t)r * p.R + i) * 2 + 0]);
      dkey = umax64(dkey, pt[((size_t)r * p.R + i) * 2 + 1]);
    }
    y = key_index(tkey);
    di = p.nD > 0 ? key_index(dkey) : 0;
  }

  // -------------------------------------------------------------------------
  // Warp GEMM with B streamed from global memory (weights read-only, L2
  // resident): acc[mt] += A(zs rows mt*16..) . B(row brow)^T over K.
  // Register double buffer of KCH 32-wide K blocks per lane.
  // -------------------------------------------------------------------------
  template <int KCH>
  __device__ __forceinline__ void warp_mma_gB(float (&acc)[2][4], const bf16 *brow, int K, int MT) const {
    const int KB = K / 32;
    const int nch = (KB + KCH - 1) / KCH;
    const uint8_t *a0row = zs() + (size_t)g * L.zstride;
    const uint8_t *a1row = zs() + (size_t)(g + 8) * L.zstride;
    const uint8_t *a2row = zs() + (size_t)(g + 16) * L.zstride;
    const uint8_t *a3row = zs() + (size_t)(g + 24) * L.zstride;
    uint4 b0[KCH], b1[KCH];
    auto load = [&](uint4(&buf)[KCH], int ch) {
#pragma unroll
      for (int c = 0; c < KCH; ++c) {
        const int kb = ch * KCH + c;
        if (kb < KB) buf[c] = ldg128_nc(brow + kb * 32 + q * 8);
      }
    };
    auto compute = [&](uint4(&buf)[KCH], int ch) {
#pragma unroll
      for (int c = 0; c < KCH; ++c) {
        const int kb = ch * KCH + c;
        if (kb < KB) {
          const uint4 b = buf[c];
          const uint4 x0 = lds128(a0row + kb * 64 + q * 16);
          const uint4 x1 = lds128(a1row + kb * 64 + q * 16);
          mma_bf16_16816(acc[0], x0.x, x1.x, x0.y, x1.y, b.x, b.y);
          mma_bf16_16816(acc[0], x0.z, x1.z, x0.w, x1.w, b.z, b.w);
          if (MT > 1) {
            const uint4 x2 = lds128(a2row + kb * 64 + q * 16);
            const uint4 x3 = lds128(a3row + kb * 64 + q * 16);
            mma_bf16_16816(acc[1], x2.x, x3.x, x2.y, x3.y, b.x, b.y);
            mma_bf16_16816(acc[1], x2.z, x3.z, x2.w, x3.w, b.z, b.w);
          }
        }
      }
    };
    if (nch > 0) load(b0, 0);
    for (int ch = 0; ch < nch; ch += 2) {
      if (ch + 1 < nch) load(b1, ch + 1);
      compute(b0, ch);
      if (ch + 1 < nch) {
        if (ch + 2 < nch) load(b0, ch + 2);
        compute(b1, ch + 1);
      }
    }
    if (K & 31) {
      const uint2 b = ldg64_nc(brow + KB * 32 + q * 4);
      const uint2 x0 = lds64(a0row + KB * 64 + q * 8);
      const uint2 x1 = lds64(a1row + KB * 64 + q * 8);
      mma_bf16_16816(acc[0], x0.x, x1.x, x0.y, x1.y, b.x, b.y);
      if (MT > 1) {
        const uint2 x2 = lds64(a2row + KB * 64 + q * 8);
        const uint2 x3 = lds64(a3row + KB * 64 + q * 8);
        mma_bf16_16816(acc[1], x2.x, x3.x, x2.y, x3.y, b.x, b.y);
      }
    }
  }

  // SIMT (fp32) warp dot products: out[i] = sum_k A[i][k] W[k] for i < M,
  // lanes split K, butterfly reduction (every lane ends with all sums).
  __device__ __forceinline__ void warp_dot_f32(float (&acc)[MAX_R], const float *wr, int K, int M) const {
    const float *z = (const float *)zs();
    const int zst = L.zstride / 4;
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

  // A operand rows (zs) <- h rows of the predictor list (global, written by
  // every CTA of the cluster), zeros for padding / initial state.
  __device__ void load_h_rows(int n, int npad, int which /*0: current hpar, 1: next*/) {
    const int P = p.P;
    const int chunks = P * (int)sizeof(T) / 16;
    for (int idx = tid; idx < npad * chunks; idx += blockDim.x) {
      const int i = idx / chunks, c = idx % chunks;
      uint8_t *dst = zs() + (size_t)i * L.zstride + c * 16;
      bool zero = i >= n;
      int s = 0;
      if (!zero) {
        s = rs.plist[i];
        if (which == 0 && rs.hzero[s]) zero = true;
      }
      if (zero) {
        *reinterpret_cast<uint4 *>(dst) = make_uint4(0, 0, 0, 0);
      } else {
        const int hp = which == 0 ? rs.hpar[s] : (rs.hpar[s] ^ 1);
        const uint8_t *src = (const uint8_t *)p.h + (((size_t)hp * p.B + rs.b[s]) * P) * sizeof(T);
        cp_async16(dst, src + c * 16);
      }
    }
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
  }

  // -------------------------------------------------------------------------
  // Predictor phase (Alg. 3 line 6 + projection) for the rows in
  // rs.plist.  Leaves g rows in gs() (cp.async in flight; the scan waits).
  // -------------------------------------------------------------------------
  __device__ void predictor_lstm() {
    const int n = rs.npred, MT = (n + 15) / 16, npad = MT * 16;
    const int P = p.P, H = p.H;
    const float *tab = p.tab;  // E' [V1][4P]
    // (1) gates = E'[y] + W_hh h, fused LSTM cell update for this CTA's units
    load_h_rows(n, npad, 0);
    if constexpr (BF) {
      const int ntile = L.UPC / 2;
      for (int j = warp; j < ntile; j += NW) {
        const int ucol = u0 + 2 * j + (g >> 2);
        const bf16 *brow = (const bf16 *)p.w_hh + ((size_t)(g & 3) * P + ucol) * P;
        float acc[2][4];
#pragma unroll
        for (int a = 0; a < 2; ++a) acc[a][0] = acc[a][1] = acc[a][2] = acc[a][3] = 0.f;
        warp_mma_gB<6>(acc, brow, P, MT);
        const int unit = u0 + 2 * j + (q >> 1);
        const int gate0 = (q & 1) * 2;  // q even: (i, f); q odd: (g, o)
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          if (mt >= MT) break;
#pragma unroll
          for (int rr = 0; rr < 2; ++rr) {
            const int i = mt * 16 + g + rr * 8;
            const bool valid = i < n;
            const int s = valid ? rs.plist[i] : 0;
            const int y = valid ? rs.last[s] : 0;
            float v0 = acc[mt][rr * 2 + 0], v1 = acc[mt][rr * 2 + 1];
            if (valid) {
              v0 += tab[(size_t)y * 4 * P + (size_t)(gate0 + 0) * P + unit];
              v1 += tab[(size_t)y * 4 * P + (size_t)(gate0 + 1) * P + unit];
            }
            const float o0 = __shfl_xor_sync(0xffffffffu, v0, 1);
            const float o1 = __shfl_xor_sync(0xffffffffu, v1, 1);
            if (valid && (q & 1) == 0) {
              const float ig = sigmoidf_(v0), fg = sigmoidf_(v1), gg = tanhf(o0), og = sigmoidf_(o1);
              float *cp = cs() + (size_t)s * L.UPC + (unit - u0);
              const float cn = fg * (rs.hzero[s] ? 0.f : *cp) + ig * gg;
              *cp = cn;
              const float hn = og * tanhf(cn);
              ((bf16 *)p.h)[((size_t)(rs.hpar[s] ^ 1) * p.B + rs.b[s]) * P + unit] = __float2bfloat16_rn(hn);
            }
          }
        }
      }
    } else {
      for (int uu = warp; uu < L.UPC; uu += NW) {
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
          float *cp = cs() + (size_t)s * L.UPC + uu;
          const float cn = sigmoidf_(gate[1]) * (rs.hzero[s] ? 0.f : *cp) + sigmoidf_(gate[0]) * tanhf(gate[2]);
          *cp = cn;
          ((float *)p.h)[((size_t)(rs.hpar[s] ^ 1) * p.B + rs.b[s]) * P + unit] = sigmoidf_(gate[3]) * tanhf(cn);
        }
      }
    }
    __threadfence();
    if (C > 1) cluster_sync_all(); else __syncthreads();
    // (2) g = W_pred h' + b_pred for this CTA's output dims
    load_h_rows(n, npad, 1);
    if constexpr (BF) {
      const int ntile = L.DPC / 8;
      for (int j = warp; j < ntile; j += NW) {
        const bf16 *brow = (const bf16 *)p.w_pred + (size_t)(d0 + j * 8 + g) * P;
        float acc[2][4];
#pragma unroll
        for (int a = 0; a < 2; ++a) acc[a][0] = acc[a][1] = acc[a][2] = acc[a][3] = 0.f;
        warp_mma_gB<6>(acc, brow, P, MT);
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          if (mt >= MT) break;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int i = mt * 16 + g + (e >> 1) * 8;
            const int d = d0 + j * 8 + 2 * q + (e & 1);
            if (i < n) {
              const int s = rs.plist[i];
              p.gglob[(size_t)rs.b[s] * H + d] = acc[mt][e] + __bfloat162float(((const bf16 *)p.b_pred)[d]);
            }
          }
        }
      }
    } else {
      for (int dd = warp; dd < L.DPC; dd += NW) {
        const int d = d0 + dd;
        float acc[MAX_R];
        warp_dot_f32(acc, (const float *)p.w_pred + (size_t)d * P, P, n);
        const float bv = ((const float *)p.b_pred)[d];
#pragma unroll
        for (int i = 0; i < MAX_R; ++i)
          if (i < n && lane == i) p.gglob[(size_t)rs.b[rs.plist[i]] * H + d] = acc[i] + bv;
      }
    }
    __threadfence();
    if (C > 1) cluster_sync_all(); else __syncthreads();
    // (3) every CTA pulls the full g rows
    const int chunks = H * 4 / 16;
    for (int idx = tid; idx < n * chunks; idx += blockDim.x) {
      const int i = idx / chunks, c = idx % chunks;
      const int s = rs.plist[i];
      cp_async16((uint8_t *)(gs() + (size_t)s * H) + c * 16,
                 (const uint8_t *)(p.gglob + (size_t)rs.b[s] * H) + c * 16);
    }
    cp_async_commit();
    __syncthreads();
    if (warp == 0 && lane < n) {
      const int s = rs.plist[lane];
      rs.hpar[s] ^= 1;
      rs.hzero[s] = 0;
    }
    __syncthreads();
  }

  __device__ void predictor_stateless() {
    const int n = rs.npred, H = p.H, V1 = p.V1;
    const int c4 = H / 4;
    for (int idx = tid; idx < n * c4; idx += blockDim.x) {
      const int i = idx / c4, c = idx % c4;
      const int s = rs.plist[i];
      float4 acc = *reinterpret_cast<const float4 *>(p.tab + (size_t)rs.ctx[0][s] * H + c * 4);
      for (int kk = 1; kk < p.context; ++kk) {
        const float4 v = *reinterpret_cast<const float4 *>(p.tab + ((size_t)kk * V1 + rs.ctx[kk][s]) * H + c * 4);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
      *reinterpret_cast<float4 *>(gs() + (size_t)s * H + c * 4) = acc;
    }
  }

  // warp 0: rebuild the compacted scanning / predictor lists (ascending slot order)
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
      if (lane == 0) {
        rs.nscan = __popc(ms);
        rs.npred = __popc(mp);
        rs.nactive = __popc(ma);
      }
    }
  }
};

// ---------------------------------------------------------------------------
// The decode kernel.  PRED: 0 = LSTM, 1 = stateless.
// ---------------------------------------------------------------------------
template <typename T, int PRED>
__global__ void __launch_bounds__(MAX_NW * 32, 1) decode_kernel(const __grid_constant__ DecodeParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ RowState rs;
  __shared__ int s_grp;
  __shared__ int s_tt[MAX_R];
  Ctx<T> cx(p, smem, rs, PRED == 0);
  const int C = cx.C, rank = cx.rank, tid = cx.tid, lane = cx.lane, warp = cx.warp;
  const int R = p.R;
  unsigned long long st_outer = 0, st_rounds = 0, st_rowevals = 0, st_pred = 0, st_predrows = 0,
                     st_labels = 0, st_groups = 0;

  cx.load_weight_slice();
  __syncthreads();

  for (;;) {
    if (rank == 0 && tid == 0) {
      const int gi = atomicAdd(p.group_counter, 1);
      if (C == 1) s_grp = gi;
      else
        for (int r = 0; r < C; ++r) st_dsmem_u32(dsmem_addr(&s_grp, (uint32_t)r), (uint32_t)gi);
    }
    if (C > 1) cluster_sync_all(); else __syncthreads();
    const int grp = s_grp;
    if (grp >= p.n_groups) break;
    st_groups++;

    // ---- group init (warp 0: lane = row slot) -------------------------------
    if (warp == 0 && lane < R) {
      const int b = grp * R + lane;
      int L = 0;
      if (b < p.B) {
        L = p.lengths[b];
        if (L < 0 || L > p.T_max) {
          if (rank == 0) atomicOr(p.status, 1);
          L = 0;
        }
      }
      rs.b[lane] = b < p.B ? b : 0;
      rs.L[lane] = L;
      rs.t[lane] = 0; rs.k[lane] = 0; rs.len[lane] = 0;
      rs.last[lane] = p.blank;
      rs.hpar[lane] = 0; rs.hzero[lane] = 1;
      for (int c = 0; c < MAX_CTX; ++c) rs.ctx[c][lane] = p.blank;
      rs.active[lane] = L > 0;
      rs.needp[lane] = L > 0;
      rs.scanning[lane] = 0;
      rs.found[lane] = 0;
    }
    __syncwarp();
    cx.rebuild_lists();
    __syncthreads();

    // ---- outer loop over labels (Alg. 3 line 5) -------------------------------
    while (rs.nactive > 0) {
      st_outer++;
      // first-round f rows of every active row (overlaps the predictor phase)
      if (warp == 0 && lane < R) {
        rs.scanning[lane] = rs.active[lane];
        rs.found[lane] = 0;
      }
      __syncwarp();
      cx.rebuild_lists();
      __syncthreads();
      cp_async_wait_all();
      if (tid < rs.nscan) s_tt[tid] = rs.t[rs.slist[tid]];
      __syncthreads();
      int cur = 0;
      cx.issue_f_loads(cur, rs.slist, s_tt, rs.nscan);
      // predictor (Alg. 3 line 6): only rows that found a label and stay active
      if (rs.npred > 0) {
        st_pred++;
        st_predrows += rs.npred;
        if constexpr (PRED == 0) cx.predictor_lstm();
        else cx.predictor_stateless();
      }
      // ---- frame loop: joint rounds until no row scans (Alg. 3 lines 7-19) ----
      while (rs.nscan > 0) {
        const int M = rs.nscan, MT = (M + 15) / 16;
        cp_async_wait_all();
        __syncthreads();
        cx.build_z(cur, M, MT * 16);
        __syncthreads();
        if (!p.tdt && p.spec_prefetch) {
          // speculative: a row that predicts blank needs f[b, t+1] next round
          if (tid < M) {
            const int s = rs.slist[tid];
            s_tt[tid] = rs.t[s] + 1 < rs.L[s] ? rs.t[s] + 1 : rs.t[s];
          }
          __syncthreads();
          cx.issue_f_loads(cur ^ 1, rs.slist, s_tt, M);
        }
        cx.joint_keys(M, MT, nullptr, 0);
        cx.exchange_keys(M);
        st_rounds++;
        st_rowevals += M;
        // decisions (replicated in every CTA)
        if (warp == 0 && lane < M) {
          int y, di;
          cx.final_keys(lane, y, di);
          const int s = rs.slist[lane];
          const int d = p.tdt ? p.durations[di] : 0;
          if (y == p.blank) {
            rs.t[s] += p.tdt ? (d > 1 ? d : 1) : 1;
            rs.k[s] = 0;
            if (rs.t[s] >= rs.L[s]) {
              rs.active[s] = 0;
              rs.scanning[s] = 0;
            }
          } else {
            rs.found[s] = 1;
            rs.fy[s] = y;
            rs.ft[s] = rs.t[s];
            rs.fd[s] = d;
            rs.scanning[s] = 0;
          }
        }
        cx.par ^= 1;
        __syncwarp();
        cx.rebuild_lists();
        __syncthreads();
        cur ^= 1;
        if (p.tdt || !p.spec_prefetch) {
          if (tid < rs.nscan) s_tt[tid] = rs.t[rs.slist[tid]];
          __syncthreads();
          cx.issue_f_loads(cur, rs.slist, s_tt, rs.nscan);
        }
      }
      // ---- append + time rules + guard (BatchedHyps.add_results, :196-199) ----
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
          if (p.tdt && rs.fd[s] > 0) {
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
      __syncthreads();
    }
    // ---- group done: lengths, statistics -------------------------------------
    if (rank == 0 && warp == 0 && lane < R) {
      const int b = grp * R + lane;
      if (b < p.B) {
        p.out_lengths[b] = rs.len[lane];
      }
    }
    if (rank == 0 && warp == 0) {
      int tot = 0;
      if (lane < R && grp * R + lane < p.B) tot = rs.len[lane];
      for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
      st_labels += tot;
    }
    if (C > 1) cluster_sync_all(); else __syncthreads();
  }
  if (rank == 0 && tid == 0 && p.stats) {
    atomicAdd(p.stats + 0, st_outer);
    atomicAdd(p.stats + 1, st_rounds);
    atomicAdd(p.stats + 2, st_rowevals);
    atomicAdd(p.stats + 3, st_pred);
    atomicAdd(p.stats + 4, st_predrows);
    atomicAdd(p.stats + 5, st_labels);
    atomicAdd(p.stats + 6, st_groups);
    if (blockIdx.x == 0) p.stats[7] = (unsigned long long)C;
  }
}

// ---------------------------------------------------------------------------
// ll_debug_joint: the same joint / argmax / cross-CTA path on given rows.
// f rows [n][H] (workspace, produced by the encoder projection) + g [n][H].
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(MAX_NW * 32, 1) debug_joint_kernel(const __grid_constant__ DecodeParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ RowState rs;
  __shared__ int s_tt[MAX_R];
  Ctx<T> cx(p, smem, rs, false);
  const int C = cx.C, tid = cx.tid, warp = cx.warp, lane = cx.lane, R = p.R;
  cx.load_weight_slice();
  __syncthreads();
  const int cluster_id = blockIdx.x / C, n_clusters = gridDim.x / C;
  for (int base = cluster_id * R; base < p.dbg_n; base += n_clusters * R) {
    const int M = min(R, p.dbg_n - base), MT = (M + 15) / 16;
    if (warp == 0 && lane < R) {
      rs.b[lane] = base + (lane < M ? lane : 0);
      rs.slist[lane] = lane;
    }
    __syncthreads();
    if (tid < M) s_tt[tid] = 0;
    // f rows: the workspace holds [n][1][H]; T_max = 1 in debug mode
    __syncthreads();
    cx.issue_f_loads(0, rs.slist, s_tt, M);
    for (int idx = tid; idx < M * p.H; idx += blockDim.x) {
      const int i = idx / p.H, c = idx % p.H;
      cx.gs()[(size_t)i * p.H + c] = p.dbg_g[(size_t)(base + i) * p.H + c];
    }
    cp_async_wait_all();
    __syncthreads();
    cx.build_z(0, M, MT * 16);
    __syncthreads();
    cx.joint_keys(M, MT, p.dbg_logits, base);
    cx.exchange_keys(M);
    if (cx.rank == 0 && warp == 0 && lane < M) {
      int y, di;
      cx.final_keys(lane, y, di);
      p.dbg_argmax[base + lane] = y;
      if (p.dbg_dargmax) p.dbg_dargmax[base + lane] = di;
    }
    cx.par ^= 1;
    if (C > 1) cluster_sync_all(); else __syncthreads();
  }
}

}  // namespace ll
