// shard.cuh -- the address-sharded multi-GPU mode (row e): sector
// ownership, key partitioning and the transport interface.  See shard.cu.
#pragma once

#include <string>
#include <vector>

#include "thermo_internal.cuh"

namespace thermo {

// collective transport; every call is made by all ranks in the same order.
// Returns 0, 1 (CUDA error) or 2 (NCCL error) with `err` set.
class Comm {
 public:
  int rank = 0, nranks = 1;
  std::string err;
  virtual ~Comm() {}
  // element-wise sum (or max) of n u64 across ranks, in place, stream-ordered
  virtual int allreduce(ull* d, size_t n, bool op_max, cudaStream_t s) = 0;
  // host bytes of every rank -> all[r * bytes, (r + 1) * bytes); equal sizes
  virtual int allgather_host(const void* mine, size_t bytes, void* all, cudaStream_t s) = 0;
  // send[sdispl[q] .. + scnt[q]) goes to rank q; rank q's part lands at
  // recv[rdispl[q] .. + rcnt[q]).  Counts and displacements are host arrays.
  virtual int alltoallv(const ull* send, const ull* scnt, const ull* sdispl, ull* recv, const ull* rcnt,
                        const ull* rdispl, cudaStream_t s) = 0;
  // wait for the stream (and the collectives queued on it) to complete; a
  // hung or failed peer makes it return 2 after the timeout
  // (THERMO_COMM_TIMEOUT_S, default 600 s) instead of blocking forever
  virtual int wait(cudaStream_t s) = 0;
  // a rank that fails inside a collective call aborts the group, so that its
  // peers' pending and later collectives return an error instead of hanging
  virtual void abort() = 0;
};

double comm_timeout_s();

int nccl_unique_id(void* out128, std::string* msg);
Comm* make_nccl_comm(const void* id128, int rank, int nranks, std::string* msg);
std::vector<Comm*> make_local_comms(int nranks);

// partition keys by owner into out (bucket q at [sum of counts < q, ...)),
// rewriting pc ids through pc_map (null: keep); h_counts receives the bucket
// sizes.  d_tmp: device scratch of 2 * kMaxRanks u64.  Synchronizes s.
cudaError_t shard_partition(const ull* keys, ull n, KeyLayout kl, uint32_t nranks, const uint32_t* pc_map,
                            ull* out, ull* d_tmp, ull* h_counts, int num_sms, cudaStream_t s);

}  // namespace thermo
