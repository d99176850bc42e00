// ll_gather.cu -- the multi-GPU exchange of include/ll.h: gathering the ragged
// hypotheses of every rank on one root (SURVEY.md §8(b) ll_gather_ragged,
// §8(e); north_star "NCCL is used only to gather the ragged results").
//
// Decoding itself shards with no collective (utterances are independent,
// Alg. 1).  Each rank packs its rows into one int32 record on
// the device (two kernels: a single-block scan of the row lengths that writes
// the record header, then one CTA per row copying its ragged fields), the
// record sizes are all-gathered, and the records travel to the root with
// ncclSend / ncclRecv inside one NCCL group.
//
// NCCL is bound at run time with dlopen/dlsym so that libll loads without it
// and uses the same libnccl as the rest of the process (PyTorch's, when
// torch.distributed is initialised).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <stdint.h>
#include <string.h>

#include <mutex>
#include <type_traits>
#include <vector>

#include "../../include/ll.h"

namespace {

constexpr int MAX_RANKS = 4096;
constexpr size_t HDR = 16 * MAX_RANKS + 256;   // [0] own (size, capacity); [16..] gathered pairs

struct Nccl {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *);
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*CommCount)(const ncclComm_t, int *);
  ncclResult_t (*CommUserRank)(const ncclComm_t, int *);
  ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
};

const Nccl &nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    // the copy already in the process (PyTorch's) first, then the loader path
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
    if (!h) return;
    bool all = true;
    auto sym = [&](auto &fp, const char *name) {
      fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
      all = all && fp;
    };
    sym(n.GetUniqueId, "ncclGetUniqueId");
    sym(n.CommInitRank, "ncclCommInitRank");
    sym(n.CommDestroy, "ncclCommDestroy");
    sym(n.CommCount, "ncclCommCount");
    sym(n.CommUserRank, "ncclCommUserRank");
    sym(n.AllGather, "ncclAllGather");
    sym(n.Send, "ncclSend");
    sym(n.Recv, "ncclRecv");
    sym(n.GroupStart, "ncclGroupStart");
    sym(n.GroupEnd, "ncclGroupEnd");
    n.ok = all;
  });
  return n;
}

// Record header: rec[0] = B, rec[1+i] = ids[i], rec[1+B+i] = lens[i]; off[i] =
// exclusive prefix sum of lens; hdr[0] = record size, hdr[1] = root capacity.
__global__ void __launch_bounds__(1024) pack_header_kernel(int32_t B, const int32_t *__restrict__ ids,
                                                           const int32_t *__restrict__ lengths, int32_t cap,
                                                           int32_t nfields, int64_t root_capacity,
                                                           int32_t *__restrict__ rec, int64_t *__restrict__ off,
                                                           int64_t *__restrict__ hdr) {
  __shared__ int64_t wsum[32];
  __shared__ int64_t carry;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    rec[0] = B;
    carry = 0;
  }
  __syncthreads();
  for (int base = 0; base < B; base += 1024) {
    const int i = base + tid;
    int64_t v = 0;
    if (i < B) {
      const int32_t len = min(max(lengths[i], 0), cap);
      rec[1 + i] = ids[i];
      rec[1 + B + i] = len;
      v = len;
    }
    int64_t x = v;   // inclusive warp scan
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int64_t w = wsum[lane];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, w, d);
        if (lane >= d) w += y;
      }
      wsum[lane] = w;   // inclusive over warps
    }
    __syncthreads();
    const int64_t excl = carry + (warp ? wsum[warp - 1] : 0) + x - v;
    if (i < B) off[i] = excl;
    __syncthreads();
    if (tid == 0) carry += wsum[31];
    __syncthreads();
  }
  if (tid == 0) {
    off[B] = carry;   // total ragged entries per field
    hdr[0] = 1 + 2 * (int64_t)B + (int64_t)nfields * carry;
    hdr[1] = root_capacity;
  }
}

// One CTA per row: field k of row i goes to rec[1 + 2B + k*total + off[i] + j].
__global__ void __launch_bounds__(128) pack_fields_kernel(int32_t B, int32_t cap, const int32_t *__restrict__ tokens,
                                                          const int32_t *__restrict__ timestamps,
                                                          const int32_t *__restrict__ durations,
                                                          int32_t *__restrict__ rec, const int64_t *__restrict__ off) {
  const int i = blockIdx.x;
  const int64_t total = off[B], o = off[i];
  const int32_t len = rec[1 + B + i];
  int32_t *dst = rec + 1 + 2 * (int64_t)B + o;
  const int64_t src = (int64_t)i * cap;
  for (int j = threadIdx.x; j < len; j += blockDim.x) {
    dst[j] = tokens[src + j];
    dst[total + j] = timestamps[src + j];
    if (durations) dst[2 * total + j] = durations[src + j];
  }
}

size_t record_elems(int32_t B, int32_t cap, int nfields) {
  return 1 + 2 * (size_t)B + (size_t)nfields * (size_t)B * (size_t)cap;
}

}  // namespace

extern "C" {

ll_status ll_nccl_unique_id(void *id_out) {
  if (!id_out) return LL_ERR_INVALID_ARGUMENT;
  const Nccl &n = nccl();
  if (!n.ok) return LL_ERR_UNSUPPORTED;
  ncclUniqueId id;
  if (n.GetUniqueId(&id) != ncclSuccess) return LL_ERR_CUDA;
  memcpy(id_out, &id, sizeof(id));
  return LL_OK;
}

ll_status ll_nccl_comm_init(void **comm_out, int32_t nranks, const void *id, int32_t rank) {
  if (!comm_out || !id || nranks < 1 || rank < 0 || rank >= nranks) return LL_ERR_INVALID_ARGUMENT;
  if (nranks > MAX_RANKS) return LL_ERR_UNSUPPORTED;
  const Nccl &n = nccl();
  if (!n.ok) return LL_ERR_UNSUPPORTED;
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  if (n.CommInitRank(&c, nranks, uid, rank) != ncclSuccess) return LL_ERR_CUDA;
  *comm_out = c;
  return LL_OK;
}

ll_status ll_nccl_comm_destroy(void *comm) {
  if (!comm) return LL_OK;
  const Nccl &n = nccl();
  if (!n.ok) return LL_ERR_UNSUPPORTED;
  return n.CommDestroy((ncclComm_t)comm) == ncclSuccess ? LL_OK : LL_ERR_CUDA;
}

size_t ll_gather_workspace_size(int32_t B, int32_t out_capacity, int32_t with_durations) {
  if (B < 0 || out_capacity < 0) return 0;
  const size_t rec = record_elems(B, out_capacity, with_durations ? 3 : 2) * sizeof(int32_t);
  return HDR + ((rec + 255) & ~(size_t)255) + ((size_t)B + 1) * sizeof(int64_t);
}

ll_status ll_gather_ragged(void *comm, int32_t root, int32_t B, const int32_t *utt_ids, const int32_t *lengths,
                           const int32_t *tokens, const int32_t *timestamps, const int32_t *durations,
                           int32_t out_capacity, int32_t *root_buf, int64_t root_capacity, int64_t *root_used,
                           void *workspace, size_t workspace_bytes, ll_stream stream) {
  if (!comm || !root_used || !workspace || B < 0 || out_capacity < 0 || root_capacity < 0)
    return LL_ERR_INVALID_ARGUMENT;
  if (B > 0 && (!utt_ids || !lengths || (out_capacity > 0 && (!tokens || !timestamps))))
    return LL_ERR_INVALID_ARGUMENT;
  const Nccl &n = nccl();
  if (!n.ok) return LL_ERR_UNSUPPORTED;
  int nranks = 0, rank = 0;
  if (n.CommCount((ncclComm_t)comm, &nranks) != ncclSuccess || n.CommUserRank((ncclComm_t)comm, &rank) != ncclSuccess)
    return LL_ERR_CUDA;
  if (root < 0 || root >= nranks) return LL_ERR_INVALID_ARGUMENT;
  if (nranks > MAX_RANKS) return LL_ERR_UNSUPPORTED;
  if (rank == root && !root_buf) return LL_ERR_INVALID_ARGUMENT;
  const int nfields = durations ? 3 : 2;
  if (workspace_bytes < ll_gather_workspace_size(B, out_capacity, durations != nullptr)) return LL_ERR_WORKSPACE;

  cudaStream_t st = (cudaStream_t)stream;
  uint8_t *ws = (uint8_t *)workspace;
  int64_t *hdr = (int64_t *)ws, *gathered = hdr + 2;
  int32_t *rec = (int32_t *)(ws + HDR);
  const size_t rec_bytes = (record_elems(B, out_capacity, nfields) * sizeof(int32_t) + 255) & ~(size_t)255;
  int64_t *off = (int64_t *)(ws + HDR + rec_bytes);

  pack_header_kernel<<<1, 1024, 0, st>>>(B, utt_ids, lengths, out_capacity, nfields, root_capacity, rec, off, hdr);
  if (B > 0 && out_capacity > 0)
    pack_fields_kernel<<<B, 128, 0, st>>>(B, out_capacity, tokens, timestamps, durations, rec, off);
  if (cudaGetLastError() != cudaSuccess) return LL_ERR_CUDA;

  // every rank learns every record size and the root's capacity
  if (n.AllGather(hdr, gathered, 2, ncclInt64, (ncclComm_t)comm, st) != ncclSuccess) return LL_ERR_CUDA;
  std::vector<int64_t> pairs(2 * (size_t)nranks);
  if (cudaMemcpyAsync(pairs.data(), gathered, pairs.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, st) !=
          cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return LL_ERR_CUDA;
  int64_t total = 0;
  std::vector<int64_t> at(nranks);
  for (int r = 0; r < nranks; ++r) {
    at[r] = total;
    total += pairs[2 * r];
  }
  *root_used = total;
  if (total > pairs[2 * root + 1]) return LL_ERR_CAPACITY;

  if (n.GroupStart() != ncclSuccess) return LL_ERR_CUDA;
  bool ok = true;
  if (rank == root) {
    for (int r = 0; r < nranks; ++r) {
      if (r == root)
        ok = ok && cudaMemcpyAsync(root_buf + at[r], rec, pairs[2 * r] * sizeof(int32_t), cudaMemcpyDeviceToDevice,
                                   st) == cudaSuccess;
      else
        ok = ok && n.Recv(root_buf + at[r], (size_t)pairs[2 * r], ncclInt32, r, (ncclComm_t)comm, st) == ncclSuccess;
    }
  } else {
    ok = n.Send(rec, (size_t)pairs[2 * rank], ncclInt32, root, (ncclComm_t)comm, st) == ncclSuccess;
  }
  if (n.GroupEnd() != ncclSuccess) ok = false;
  return ok ? LL_OK : LL_ERR_CUDA;
}

}  // extern "C"
