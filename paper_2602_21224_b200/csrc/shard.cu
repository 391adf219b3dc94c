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

// ------------------------------------------------------------ stochastic partials
// Stochastic acceptance (R13) reads, per visited verify row: lse_v(l_v / T), the
// logits of the row's child tokens, and the Gumbel-max of l_v / T + G_v over V
// minus the rejected children. Over a vocab shard's columns each row yields a
// record [m, z, gv[KG], gi[KG], tl[T]]: (m, z) = (max, sum exp(. - m)) of l / T;
// the shard's KG best (l_v / T + G_v, v) in (value desc, token asc) order, G_v from
// the walk's own Philox stream (v / 4, slot, step, req); tl[s] = the logit of tree
// slot s's token if this shard owns it, else -inf. The merge is exact up to the
// order of the lse sum: lse = M + log sum_s z_s e^(m_s - M); each tree token has one
// owner; the global top-KG is contained in the union of the shards' top-KG lists.
// A rejected set has at most (children of a node) <= k + B_r < KG tokens, so the
// best non-rejected candidate is in the merged list.
constexpr int KG = HSD_SHARD_KG;
__host__ __device__ inline int stoch_rec(int T) { return 2 + 2 * KG + T; }

// one CTA per row; x rows of width w (stride ld) are columns [col0, col0 + w)
__global__ void __launch_bounds__(256) stoch_part_kernel(const float* __restrict__ x, int ld, int w, int col0,
                                                         int T, const int32_t* __restrict__ tree_tok,
                                                         const int32_t* __restrict__ req_id,
                                                         const int32_t* __restrict__ step, uint32_t seed, float invT,
                                                         float* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  __shared__ float sm[8], sz[8];
  __shared__ float cv[256 * 2];
  __shared__ int ci[256 * 2];
  const int r = blockIdx.x, rq = r / T, slot = r % T;
  const float* xr = x + (size_t)r * ld;
  float* rec = out + (size_t)r * stoch_rec(T);
  const uint32_t rqg = (uint32_t)req_id[rq], st = (uint32_t)*step;
  // (1) max / sum of l / T, and this thread's top-KG Gumbel scores (sorted, registers)
  float m = -INFINITY, zs = 0.f;
  float tv[KG];
  int ti[KG];
#pragma unroll
  for (int k = 0; k < KG; ++k) { tv[k] = -INFINITY; ti[k] = 0x7fffffff; }
  const int v0 = col0 & ~3;                       // whole Philox blocks
  for (int b4 = v0 / 4 + threadIdx.x; b4 * 4 < col0 + w; b4 += blockDim.x) {
    const u32x4 c = {(uint32_t)b4, (uint32_t)slot, st, rqg};
    const u32x4 rr = philox4x32_10(c, seed, TAG_GUMBEL);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int v = b4 * 4 + q;
      if (v < col0 || v >= col0 + w) continue;
      const float t = xr[v - col0] * invT;
      if (t > m) { zs = zs * expf(m - t) + 1.f; m = t; }
      else zs += expf(t - m);
      const float g = t - logf(-logf(unit_open(lane_of(rr, q))));
      if (better(g, v, tv[KG - 1], ti[KG - 1])) {   // insert into the sorted list
        float cvv = g;
        int cii = v;
#pragma unroll
        for (int k = 0; k < KG; ++k) {
          if (better(cvv, cii, tv[k], ti[k])) {
            const float ov = tv[k];
            const int oi = ti[k];
            tv[k] = cvv; ti[k] = cii;
            cvv = ov; cii = oi;
          }
        }
      }
    }
  }
  // block (max, sum)
  float M = m;
  for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
  const int wp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) sm[wp] = M;
  __syncthreads();
  M = sm[0];
  for (int i = 1; i < (int)(blockDim.x >> 5); ++i) M = fmaxf(M, sm[i]);
  float zz = m == -INFINITY ? 0.f : zs * expf(m - M);
  for (int o = 16; o > 0; o >>= 1) zz += __shfl_xor_sync(0xffffffffu, zz, o);
  if (lane == 0) sz[wp] = zz;
  // (2) block top-KG: KG rounds, each takes the best head among the threads' lists
  int head = 0;
  for (int k = 0; k < KG; ++k) {
    float bv = head < KG ? tv[0] : -INFINITY;
    int bi = head < KG ? ti[0] : 0x7fffffff;
#pragma unroll
    for (int q = 1; q < KG; ++q)
      if (q == head) { bv = tv[q]; bi = ti[q]; }
    float wv = bv;
    int wi = bi;
    warp_argmax(wv, wi);
    __syncthreads();
    if (lane == 0) { cv[wp] = wv; ci[wp] = wi; }
    __syncthreads();
    if (wp == 0) {
      float v2 = lane < (int)(blockDim.x >> 5) ? cv[lane] : -INFINITY;
      int i2 = lane < (int)(blockDim.x >> 5) ? ci[lane] : 0x7fffffff;
      warp_argmax(v2, i2);
      if (lane == 0) { cv[256] = v2; ci[256] = i2; }
    }
    __syncthreads();
    if (ci[256] == bi && bi != 0x7fffffff) ++head;   // the winner's owner advances (indices are unique)
    if (threadIdx.x == 0) { rec[2 + k] = cv[256]; ((int*)rec)[2 + KG + k] = ci[256]; }
  }
  if (threadIdx.x == 0) {
    float z = 0.f;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) z += sz[i];
    rec[0] = M;
    rec[1] = z;
  }
  // (3) tree-token logits owned by this shard
  for (int s2 = threadIdx.x; s2 < T; s2 += blockDim.x) {
    const int t = tree_tok[(size_t)rq * T + s2];
    rec[2 + 2 * KG + s2] = (t >= col0 && t < col0 + w) ? xr[t - col0] : -INFINITY;
  }
}

// merge G shard records of rows [row0, row0 + M) (record stride per shard `sstride`
// rows) into lse / tl / (gv, gi) of this rank's M rows
__global__ void stoch_merge_kernel(const float* __restrict__ part, int G, size_t sstride, int row0, int M, int T,
                                   float* __restrict__ lse, float* __restrict__ tl, float* __restrict__ gv,
                                   int32_t* __restrict__ gi) {
  pdl_wait();
  pdl_trigger();
  const int m = blockIdx.x;
  if (m >= M) return;
  const int R = stoch_rec(T);
  auto recp = [&](int s) { return part + ((size_t)s * sstride + row0 + m) * R; };
  if (threadIdx.x == 0) {
    float Mx = -INFINITY;
    for (int s = 0; s < G; ++s) if (recp(s)[1] > 0.f) Mx = fmaxf(Mx, recp(s)[0]);
    float Z = 0.f;
    for (int s = 0; s < G; ++s) if (recp(s)[1] > 0.f) Z += recp(s)[1] * expf(recp(s)[0] - Mx);
    lse[m] = Mx + logf(Z);
    // G sorted lists -> the KG best (G-way merge by heads)
    int hd[HSD_MAX_SHARDS];
    for (int s = 0; s < G; ++s) hd[s] = 0;
    for (int k = 0; k < KG; ++k) {
      float bv = -INFINITY;
      int bi = 0x7fffffff, bs = -1;
      for (int s = 0; s < G; ++s) {
        if (hd[s] >= KG) continue;
        const float v = recp(s)[2 + hd[s]];
        const int i = ((const int*)recp(s))[2 + KG + hd[s]];
        if (better(v, i, bv, bi)) { bv = v; bi = i; bs = s; }
      }
      if (bs >= 0) ++hd[bs];
      gv[(size_t)m * KG + k] = bv;
      gi[(size_t)m * KG + k] = bi;
    }
  }
  for (int s2 = threadIdx.x; s2 < T; s2 += blockDim.x) {
    float v = -INFINITY;
    for (int s = 0; s < G; ++s) v = fmaxf(v, recp(s)[2 + 2 * KG + s2]);
    tl[(size_t)m * T + s2] = v;
  }
}

void launch_stoch_part(const float* x, int rows, int ld, int w, int col0, int T, const int32_t* tree_tok,
                       const int32_t* req_id, const int32_t* step, uint32_t seed, float temperature, float* out,
                       cudaStream_t st) {
  if (rows > 0)
    launch_k(stoch_part_kernel, rows, 256, 0, st, x, ld, w, col0, T, tree_tok, req_id, step, seed, 1.0f / temperature,
             out);
}
void launch_stoch_merge(const float* part, int G, size_t sstride, int row0, int M, int T, float* lse, float* tl,
                        float* gv, int32_t* gi, cudaStream_t st) {
  if (M > 0) launch_k(stoch_merge_kernel, M, 128, 0, st, part, G, sstride, row0, M, T, lse, tl, gv, gi);
}
size_t stoch_record_floats(int T) { return (size_t)stoch_rec(T); }

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
