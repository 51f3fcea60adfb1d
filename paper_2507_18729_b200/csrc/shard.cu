// shard.cu -- row e of the hot path: the address-sharded
// multi-GPU mode.
//
// A sector's nine counts depend only on the records that touch it (the
// per-sector bitmasks are independent; S:292-300 merge = OR, S:332 shards "by
// sector key ... combined with merge"), so the reduction shards by sector:
//   * every rank decodes its own slice of the trace into keys (a2/a3);
//   * pc ids are unified (the union of the ranks' (launch, pc) sites, ids in
//     order of first appearance in the union, sorted within each build);
//   * keys move to the owner of their sector, owner(g) = (g >> 11) % nranks
//     (2048-sector chunks = one indicator tile, block-cyclic so that a hot
//     object spreads over all ranks), in ONE all-to-all exchange;
//   * each owner counts its sectors (a4/a5) into its part of the dense arrays,
//     histograms its sectors and tiles (a6/a7), and the per-object / per-pc
//     partial sums are combined with all-reduce (sum, or max for the largest
//     sector count).
// The result is bit-identical to one rank reducing the whole trace.
//
// Transport: NcclComm (NCCL over NVLink/NVSwitch, one process per GPU) or
// LocalComm (several contexts of one process on one device, each driven by
// its own host thread; the same algorithm with device-to-device copies --
// used to test the sharded path on a single GPU).
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>

#include "shard.cuh"

namespace thermo {

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------
constexpr int kShardThreads = 256;
constexpr int kShardPer = 8;  // keys per thread per tile

__device__ __forceinline__ unsigned lanemask_lt_s() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// per-owner key counts
__global__ void __launch_bounds__(kShardThreads) shard_count_kernel(const ull* __restrict__ keys, ull n, KeyLayout kl,
                                                                    uint32_t nranks, ull* __restrict__ counts) {
  __shared__ uint32_t s[kMaxRanks];
  if (threadIdx.x < kMaxRanks) s[threadIdx.x] = 0;
  __syncthreads();
  const ull stride = (ull)gridDim.x * blockDim.x;
  const ull nt = (n + 31) / 32 * 32;
  for (ull i = (ull)blockIdx.x * blockDim.x + threadIdx.x; i < nt; i += stride) {
    const bool in = i < n;
    const uint32_t o = in ? shard_owner(key_g(keys[i], kl), nranks) : 0u;
    const unsigned peers = __match_any_sync(0xFFFFFFFFu, in ? o : 0xFFFFFFFFu);
    if (in && (__ffs(peers) - 1) == (int)(threadIdx.x & 31)) atomicAdd(&s[o], (uint32_t)__popc(peers));
  }
  __syncthreads();
  if (threadIdx.x < nranks && s[threadIdx.x]) atomicAdd(&counts[threadIdx.x], (ull)s[threadIdx.x]);
}

// scatter keys into owner buckets (cursor[o] = next free slot of bucket o),
// rewriting rank-local pc ids to job-wide ones on the way
__global__ void __launch_bounds__(kShardThreads) shard_scatter_kernel(const ull* __restrict__ keys, ull n, KeyLayout kl,
                                                                      uint32_t nranks, const uint32_t* __restrict__ pc_map,
                                                                      ull* __restrict__ cursor, ull* __restrict__ out) {
  __shared__ uint32_t s_cnt[kMaxRanks];
  __shared__ ull s_base[kMaxRanks];
  const int lane = threadIdx.x & 31;
  const unsigned lt = lanemask_lt_s();
  const ull tile = (ull)kShardThreads * kShardPer;
  for (ull t0 = (ull)blockIdx.x * tile; t0 < n; t0 += (ull)gridDim.x * tile) {
    if (threadIdx.x < kMaxRanks) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    ull k[kShardPer];
    uint32_t own[kShardPer], rk[kShardPer];
#pragma unroll
    for (int u = 0; u < kShardPer; ++u) {
      const ull i = t0 + (ull)u * kShardThreads + threadIdx.x;
      const bool in = i < n;
      ull key = in ? keys[i] : 0;
      if (in && pc_map && kl.P) {
        const ull pm = ((1ull << kl.P) - 1) << 8;
        key = (key & ~pm) | ((ull)pc_map[key_pcid(key, kl)] << 8);
      }
      own[u] = in ? shard_owner(key_g(key, kl), nranks) : 0xFFFFFFFFu;
      if (in) {  // the owner counts into its own chunks: global sector -> its local index
        const uint32_t gs = 8 + kl.P + kl.L + kl.W;
        key = (key & ((1ull << gs) - 1)) | (shard_local(key_g(key, kl), nranks) << gs);
      }
      k[u] = key;
      const unsigned peers = __match_any_sync(0xFFFFFFFFu, own[u]);
      const int leader = __ffs(peers) - 1;
      uint32_t base = 0;
      if (in && lane == leader) base = atomicAdd(&s_cnt[own[u]], (uint32_t)__popc(peers));
      base = __shfl_sync(0xFFFFFFFFu, base, leader);
      rk[u] = base + __popc(peers & lt);
    }
    __syncthreads();
    if (threadIdx.x < nranks) s_base[threadIdx.x] = s_cnt[threadIdx.x] ? atomicAdd(&cursor[threadIdx.x], (ull)s_cnt[threadIdx.x]) : 0;
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kShardPer; ++u)
      if (own[u] != 0xFFFFFFFFu) out[s_base[own[u]] + rk[u]] = k[u];
    __syncthreads();
  }
}

__global__ void reduce_pair_kernel(ull* __restrict__ dst, const ull* __restrict__ src, size_t n, int op_max) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const ull a = dst[i], b = src[i];
    dst[i] = op_max ? (a > b ? a : b) : a + b;
  }
}

static void launch_reduce_pair(ull* dst, const ull* src, size_t n, bool op_max, cudaStream_t s) {
  if (!n) return;
  const unsigned grid = (unsigned)std::min<size_t>((n + 255) / 256, 1024);
  reduce_pair_kernel<<<grid, 256, 0, s>>>(dst, src, n, op_max ? 1 : 0);
}

cudaError_t shard_partition(const ull* keys, ull n, KeyLayout kl, uint32_t nranks, const uint32_t* pc_map,
                            ull* out, ull* d_tmp /*[2 * kMaxRanks]*/, ull* h_counts /*[nranks]*/, int num_sms,
                            cudaStream_t s) {
  cudaError_t e;
  if ((e = cudaMemsetAsync(d_tmp, 0, 2 * kMaxRanks * sizeof(ull), s))) return e;
  if (n) {
    const unsigned grid = (unsigned)std::min<ull>((n + kShardThreads - 1) / kShardThreads, (ull)num_sms * 8);
    shard_count_kernel<<<grid, kShardThreads, 0, s>>>(keys, n, kl, nranks, d_tmp);
  }
  if ((e = cudaMemcpyAsync(h_counts, d_tmp, nranks * sizeof(ull), cudaMemcpyDeviceToHost, s))) return e;
  if ((e = cudaStreamSynchronize(s))) return e;
  ull cur[kMaxRanks] = {0};
  for (uint32_t q = 1; q < nranks; ++q) cur[q] = cur[q - 1] + h_counts[q - 1];
  if ((e = cudaMemcpyAsync(d_tmp + kMaxRanks, cur, nranks * sizeof(ull), cudaMemcpyHostToDevice, s))) return e;
  if (n) {
    const ull tile = (ull)kShardThreads * kShardPer;
    const unsigned grid = (unsigned)std::min<ull>((n + tile - 1) / tile, (ull)num_sms * 8);
    shard_scatter_kernel<<<grid, kShardThreads, 0, s>>>(keys, n, kl, nranks, pc_map, d_tmp + kMaxRanks, out);
  }
  if ((e = cudaGetLastError())) return e;
  return cudaStreamSynchronize(s);  // cur[] lives on the host stack
}

double comm_timeout_s() {
  const char* e = getenv("THERMO_COMM_TIMEOUT_S");
  const double v = e ? atof(e) : 0.0;
  return v > 0 ? v : 600.0;
}

// ---------------------------------------------------------------------------
// NCCL transport (one process per GPU)
// ---------------------------------------------------------------------------
namespace {

int nccl_fail(std::string* msg, const char* what, ncclResult_t r) {
  if (msg) *msg = std::string(what) + ": " + ncclGetErrorString(r);
  return 2;
}
int cuda_fail(std::string* msg, const char* what, cudaError_t e) {
  if (msg) *msg = std::string(what) + ": " + cudaGetErrorString(e);
  return 1;
}
#define NCK(call, what)                                  \
  do {                                                   \
    ncclResult_t r_ = (call);                            \
    if (r_ != ncclSuccess) return nccl_fail(&err, what, r_); \
  } while (0)
#define CCK(call, what)                                  \
  do {                                                   \
    cudaError_t e_ = (call);                             \
    if (e_ != cudaSuccess) return cuda_fail(&err, what, e_); \
  } while (0)

class NcclComm final : public Comm {
 public:
  ncclComm_t comm = nullptr;
  unsigned char* scratch = nullptr;
  size_t scratch_bytes = 0;

  ~NcclComm() override {
    if (scratch) cudaFree(scratch);
    if (comm) ncclCommDestroy(comm);
  }
  void abort() override {
    if (comm) ncclCommAbort(comm);
    comm = nullptr;
  }
  // poll the stream and NCCL's asynchronous error state until the queued work
  // completes, an error shows, or the deadline passes (then abort the comm)
  int wait(cudaStream_t s) override {
    if (!comm) { err = "communicator aborted"; return 2; }
    const auto t0 = std::chrono::steady_clock::now();
    const double lim = comm_timeout_s();
    for (unsigned it = 0;; ++it) {
      const cudaError_t q = cudaStreamQuery(s);
      if (q == cudaSuccess) return 0;
      if (q != cudaErrorNotReady) return cuda_fail(&err, "stream wait", q);
      ncclResult_t ar = ncclSuccess;
      const ncclResult_t r = ncclCommGetAsyncError(comm, &ar);
      if (r != ncclSuccess || (ar != ncclSuccess && ar != ncclInProgress)) {
        nccl_fail(&err, "ncclCommGetAsyncError", r != ncclSuccess ? r : ar);
        abort();
        return 2;
      }
      if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > lim) {
        err = "collective timed out (THERMO_COMM_TIMEOUT_S); communicator aborted";
        abort();
        return 2;
      }
      if (it > 64) std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
  }
  int allreduce(ull* d, size_t n, bool op_max, cudaStream_t s) override {
    if (!n) return 0;
    if (!comm) { err = "communicator aborted"; return 2; }
    NCK(ncclAllReduce(d, d, n, ncclUint64, op_max ? ncclMax : ncclSum, comm, s), "ncclAllReduce");
    return 0;
  }
  int allgather_host(const void* mine, size_t bytes, void* all, cudaStream_t s) override {
    if (!bytes) return 0;
    const size_t need = bytes * (size_t)nranks;
    if (scratch_bytes < need) {
      if (scratch) cudaFree(scratch);
      scratch = nullptr;
      scratch_bytes = 0;
      CCK(cudaMalloc(&scratch, need), "cudaMalloc (allgather scratch)");
      scratch_bytes = need;
    }
    if (!comm) { err = "communicator aborted"; return 2; }
    CCK(cudaMemcpyAsync(scratch + (size_t)rank * bytes, mine, bytes, cudaMemcpyHostToDevice, s), "allgather H2D");
    NCK(ncclAllGather(scratch + (size_t)rank * bytes, scratch, bytes, ncclUint8, comm, s), "ncclAllGather");
    CCK(cudaMemcpyAsync(all, scratch, need, cudaMemcpyDeviceToHost, s), "allgather D2H");
    return wait(s);
  }
  int alltoallv(const ull* send, const ull* scnt, const ull* sdispl, ull* recv, const ull* rcnt, const ull* rdispl,
                cudaStream_t s) override {
    if (!comm) { err = "communicator aborted"; return 2; }
    NCK(ncclGroupStart(), "ncclGroupStart");
    for (int q = 0; q < nranks; ++q) {
      if (q == rank) {
        if (scnt[q])
          CCK(cudaMemcpyAsync(recv + rdispl[q], send + sdispl[q], scnt[q] * sizeof(ull), cudaMemcpyDeviceToDevice, s),
              "alltoallv self copy");
        continue;
      }
      if (scnt[q]) NCK(ncclSend(send + sdispl[q], scnt[q], ncclUint64, q, comm, s), "ncclSend");
      if (rcnt[q]) NCK(ncclRecv(recv + rdispl[q], rcnt[q], ncclUint64, q, comm, s), "ncclRecv");
    }
    NCK(ncclGroupEnd(), "ncclGroupEnd");
    return 0;
  }
};

// ---------------------------------------------------------------------------
// in-process transport: nranks contexts on one device, one host thread each
// ---------------------------------------------------------------------------
struct LocalGroup {
  int P;
  int refs;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long gen = 0;
  bool poisoned = false;  // a rank failed inside a collective, or a barrier timed out
  std::vector<const void*> dptr, hptr;
  std::vector<const ull*> m1, m2;
  explicit LocalGroup(int p) : P(p), refs(p), dptr(p), hptr(p), m1(p), m2(p) {}
  // false once the group is poisoned (then every later barrier fails at once)
  bool barrier() {
    std::unique_lock<std::mutex> l(m);
    if (poisoned) return false;
    const unsigned long g = gen;
    if (++arrived == P) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    const auto lim = std::chrono::duration<double>(comm_timeout_s());
    if (!cv.wait_for(l, lim, [&] { return gen != g || poisoned; })) poisoned = true;
    if (poisoned) {
      cv.notify_all();
      return false;
    }
    return true;
  }
  void poison() {
    std::lock_guard<std::mutex> l(m);
    poisoned = true;
    cv.notify_all();
  }
};

class LocalComm final : public Comm {
 public:
  LocalGroup* g = nullptr;
  ull *snap = nullptr, *tmp = nullptr;
  size_t cap = 0;

  ~LocalComm() override {
    if (snap) cudaFree(snap);
    if (tmp) cudaFree(tmp);
    if (g) {
      bool last;
      {
        std::lock_guard<std::mutex> l(g->m);
        last = --g->refs == 0;
      }
      if (last) delete g;
    }
  }
  int allreduce(ull* d, size_t n, bool op_max, cudaStream_t s) override {
    if (!n) return 0;
    if (cap < n) {
      if (snap) cudaFree(snap);
      if (tmp) cudaFree(tmp);
      snap = tmp = nullptr;
      cap = 0;
      CCK(cudaMalloc(&snap, n * sizeof(ull)), "cudaMalloc (allreduce)");
      CCK(cudaMalloc(&tmp, n * sizeof(ull)), "cudaMalloc (allreduce)");
      cap = n;
    }
    CCK(cudaMemcpyAsync(snap, d, n * sizeof(ull), cudaMemcpyDeviceToDevice, s), "allreduce snapshot");
    CCK(cudaStreamSynchronize(s), "allreduce sync");
    g->dptr[rank] = snap;
    if (!g->barrier()) return peer_fail();
    for (int q = 0; q < nranks; ++q) {
      if (q == rank) continue;
      CCK(cudaMemcpyAsync(tmp, g->dptr[q], n * sizeof(ull), cudaMemcpyDeviceToDevice, s), "allreduce copy");
      launch_reduce_pair(d, tmp, n, op_max, s);
    }
    CCK(cudaStreamSynchronize(s), "allreduce sync");
    if (!g->barrier()) return peer_fail();  // peers done reading my snapshot
    return 0;
  }
  int allgather_host(const void* mine, size_t bytes, void* all, cudaStream_t) override {
    g->hptr[rank] = mine;
    if (!g->barrier()) return peer_fail();
    for (int q = 0; q < nranks; ++q) std::memcpy(static_cast<char*>(all) + (size_t)q * bytes, g->hptr[q], bytes);
    if (!g->barrier()) return peer_fail();
    return 0;
  }
  int alltoallv(const ull* send, const ull* scnt, const ull* sdispl, ull* recv, const ull* rcnt, const ull* rdispl,
                cudaStream_t s) override {
    CCK(cudaStreamSynchronize(s), "alltoallv sync");
    g->dptr[rank] = send;
    g->m1[rank] = scnt;
    g->m2[rank] = sdispl;
    if (!g->barrier()) return peer_fail();
    for (int q = 0; q < nranks; ++q) {
      const ull cnt = g->m1[q][rank];
      if (cnt != rcnt[q]) {
        err = "alltoallv: receive count mismatch";
        g->poison();
        return 2;
      }
      if (cnt)
        CCK(cudaMemcpyAsync(recv + rdispl[q], static_cast<const ull*>(g->dptr[q]) + g->m2[q][rank], cnt * sizeof(ull),
                            cudaMemcpyDeviceToDevice, s),
            "alltoallv copy");
    }
    CCK(cudaStreamSynchronize(s), "alltoallv sync");
    if (!g->barrier()) return peer_fail();
    return 0;
  }
  int wait(cudaStream_t s) override {
    CCK(cudaStreamSynchronize(s), "stream wait");
    return 0;
  }
  void abort() override { g->poison(); }
  int peer_fail() {
    err = "a peer rank failed inside the collective, or it timed out (THERMO_COMM_TIMEOUT_S)";
    return 2;
  }
};

}  // namespace

int nccl_unique_id(void* out128, std::string* msg) {
  ncclUniqueId id;
  const ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(msg, "ncclGetUniqueId", r);
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out128, &id, 128);
  return 0;
}

Comm* make_nccl_comm(const void* id128, int rank, int nranks, std::string* msg) {
  ncclUniqueId id;
  std::memcpy(&id, id128, 128);
  NcclComm* c = new NcclComm();
  c->rank = rank;
  c->nranks = nranks;
  const ncclResult_t r = ncclCommInitRank(&c->comm, nranks, id, rank);
  if (r != ncclSuccess) {
    nccl_fail(msg, "ncclCommInitRank", r);
    c->comm = nullptr;
    delete c;
    return nullptr;
  }
  return c;
}

std::vector<Comm*> make_local_comms(int nranks) {
  LocalGroup* g = new LocalGroup(nranks);
  std::vector<Comm*> v;
  for (int r = 0; r < nranks; ++r) {
    LocalComm* c = new LocalComm();
    c->g = g;
    c->rank = r;
    c->nranks = nranks;
    v.push_back(c);
  }
  return v;
}

}  // namespace thermo
