// shard.cu -- vocab-sharded lm_head (BASELINE configs[4]): the
// per-row partial argmax over a shard's vocabulary columns, its exact merge,
// the column scatter that reassembles full draft-logits rows, and the NCCL
// entry points (loaded at run time with dlopen, so the library links and loads
// without NCCL; torch's already-loaded libnccl.so.2 is reused when present).
//
// Greedy verification needs only the argmax of each verify row (P:378 walk,
// reading R8: lowest id among maxima). The argmax over V is the best of the
// shards' partial argmaxes under the same (value desc, id asc) order, so the
// merge is exact: bit-identical to the unsharded argmax whenever the logits
// themselves are.
#include <dlfcn.h>
#include <algorithm>
#include <cstring>
#include <string>
#include <type_traits>
#include <nccl.h>
#include "kernels.cuh"

// ------------------------------------------------------------------ kernels
// partial argmax of rows x[r, 0:w) (row stride ld) -> (value, col0 + index)
__global__ void __launch_bounds__(512) argmax_part_kernel(const float* __restrict__ x, int ld, int w, int col0,
                                                          float* __restrict__ outv, int32_t* __restrict__ outi) {
  pdl_wait();
  pdl_trigger();
  __shared__ float sv[32];
  __shared__ int si[32];
  const int r = blockIdx.x;
  const float* xr = x + (size_t)r * ld;
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int i = threadIdx.x; i < w; i += blockDim.x) {
    const float v = xr[i];
    if (better(v, col0 + i, bv, bi)) { bv = v; bi = col0 + i; }
  }
  warp_argmax(bv, bi);
  const int wp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { sv[wp] = bv; si[wp] = bi; }
  __syncthreads();
  if (wp == 0) {
    const int nw = blockDim.x >> 5;
    bv = lane < nw ? sv[lane] : -INFINITY;
    bi = lane < nw ? si[lane] : 0x7fffffff;
    warp_argmax(bv, bi);
    if (lane == 0) { outv[r] = bv; outi[r] = bi; }
  }
}

// out[m] = best over shards s of (pv, pi)[s * stride + row0 + m]; -1 for inactive rows
__global__ void argmax_merge_kernel(const float* __restrict__ pv, const int32_t* __restrict__ pi, int S,
                                    int stride, int row0, int M, const int32_t* __restrict__ pos,
                                    int32_t* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= M) return;
  if (pos && pos[m] < 0) { out[m] = -1; return; }
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int s = 0; s < S; ++s) {
    const size_t e = (size_t)s * stride + row0 + m;
    if (better(pv[e], pi[e], bv, bi)) { bv = pv[e]; bi = pi[e]; }
  }
  out[m] = bi;
}

// dst[r, lo_s + j] = src_s[r, j] for shard s = blockIdx.y, src_s = src + s * src_stride, row stride w_s
struct ShardCols {
  int lo[HSD_MAX_SHARDS + 1];
};
__global__ void scatter_cols_kernel(const float* __restrict__ src, size_t src_stride, int rows, ShardCols sc,
                                    float* __restrict__ dst, int ld) {
  pdl_wait();
  pdl_trigger();
  const int s = blockIdx.y, w = sc.lo[s + 1] - sc.lo[s];
  const float* sp = src + (size_t)s * src_stride;
  for (int r = blockIdx.x; r < rows; r += gridDim.x) {
    const float* a = sp + (size_t)r * w;
    float* d = dst + (size_t)r * ld + sc.lo[s];
    for (int j = threadIdx.x; j < w; j += blockDim.x) d[j] = a[j];
  }
}

void launch_argmax_part(const float* x, int rows, int ld, int w, int col0, float* outv, int32_t* outi,
                        cudaStream_t st) {
  if (rows > 0) launch_k(argmax_part_kernel, rows, 512, 0, st, x, ld, w, col0, outv, outi);
}
void launch_argmax_merge(const float* pv, const int32_t* pi, int S, int stride, int row0, int M,
                         const int32_t* pos, int32_t* out, cudaStream_t st) {
  if (M > 0) launch_k(argmax_merge_kernel, (M + 127) / 128, 128, 0, st, pv, pi, S, stride, row0, M, pos, out);
}
void launch_scatter_cols(const float* src, size_t src_stride, int rows, int S, const int* lo, float* dst, int ld,
                         cudaStream_t st) {
  if (rows <= 0 || S <= 0) return;
  ShardCols sc{};
  for (int s = 0; s <= S && s <= HSD_MAX_SHARDS; ++s) sc.lo[s] = lo[s];
  launch_k(scatter_cols_kernel, dim3(std::min(rows, 1024), S), 256, 0, st, src, src_stride, rows, sc, dst, ld);
}

// ------------------------------------------------------------------ NCCL (dlopen)
namespace {
struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi& api() {
  static NcclApi a = [] {
    NcclApi x;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      x.err = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
      return x;
    }
    bool all = true;
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn) all = false;
    };
    sym(x.GetUniqueId, "ncclGetUniqueId");
    sym(x.CommInitRank, "ncclCommInitRank");
    sym(x.CommDestroy, "ncclCommDestroy");
    sym(x.AllGather, "ncclAllGather");
    sym(x.Send, "ncclSend");
    sym(x.Recv, "ncclRecv");
    sym(x.GroupStart, "ncclGroupStart");
    sym(x.GroupEnd, "ncclGroupEnd");
    sym(x.GetErrorString, "ncclGetErrorString");
    x.ok = all;
    if (!all) x.err = "libnccl.so.2 lacks a required symbol";
    return x;
  }();
  return a;
}
std::string nerr(ncclResult_t r) {
  return api().GetErrorString ? api().GetErrorString(r) : ("nccl error " + std::to_string((int)r));
}
}  // namespace

bool shard_nccl_unique_id(uint8_t* out, std::string& err) {
  if (!api().ok) { err = api().err; return false; }
  ncclUniqueId id;
  const ncclResult_t r = api().GetUniqueId(&id);
  if (r != ncclSuccess) { err = "ncclGetUniqueId: " + nerr(r); return false; }
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  memcpy(out, &id, 128);
  return true;
}

bool shard_nccl_init(void** comm, int nranks, const uint8_t* id_bytes, int rank, std::string& err) {
  if (!api().ok) { err = api().err; return false; }
  ncclUniqueId id;
  memcpy(&id, id_bytes, 128);
  ncclComm_t c = nullptr;
  const ncclResult_t r = api().CommInitRank(&c, nranks, id, rank);
  if (r != ncclSuccess) { err = "ncclCommInitRank: " + nerr(r); return false; }
  *comm = c;
  return true;
}

void shard_nccl_destroy(void* comm) {
  if (comm && api().ok) api().CommDestroy((ncclComm_t)comm);
}

// all-gather `bytes` per rank (recv holds nranks blocks, rank order)
bool shard_allgather(const void* send, void* recv, size_t bytes, void* comm, cudaStream_t st, std::string& err) {
  const ncclResult_t r = api().AllGather(send, recv, bytes, ncclUint8, (ncclComm_t)comm, st);
  if (r != ncclSuccess) { err = "ncclAllGather: " + nerr(r); return false; }
  return true;
}

// all-to-all of variable blocks: send_off/send_bytes[r] to rank r, recv_off/recv_bytes[r] from rank r
bool shard_alltoallv(const char* send, const size_t* send_off, const size_t* send_bytes, char* recv,
                     const size_t* recv_off, const size_t* recv_bytes, int nranks, void* comm, cudaStream_t st,
                     std::string& err) {
  ncclResult_t r = api().GroupStart();
  for (int p = 0; p < nranks && r == ncclSuccess; ++p) {
    r = api().Send(send + send_off[p], send_bytes[p], ncclUint8, p, (ncclComm_t)comm, st);
    if (r == ncclSuccess) r = api().Recv(recv + recv_off[p], recv_bytes[p], ncclUint8, p, (ncclComm_t)comm, st);
  }
  const ncclResult_t e = api().GroupEnd();
  if (r == ncclSuccess) r = e;
  if (r != ncclSuccess) { err = "nccl send/recv: " + nerr(r); return false; }
  return true;
}
