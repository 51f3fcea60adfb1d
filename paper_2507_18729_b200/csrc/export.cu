// export.cu -- SURVEY §8f item 3: run compression of an object's heat-map rows
// (Fig. 4 caption: "consecutive memory regions with identical temperatures are
// compressed, and the number of occurrences is indicated").
//
// A row is the sector's 9-tuple (8 word temperatures, words past the object's
// end read as 0, then the sector temperature).  A run starts at the object's
// first sector and wherever a row differs from the previous one.  Three passes
// over the object's rows: (1) per-block counts of run starts, (2) one-block
// exclusive scan of the block counts, (3) each start writes its run (start
// sector, 9 temperatures) at its rank; (4) counts = next start - start.
#include "thermo_internal.cuh"

namespace thermo {

constexpr int kRunThreads = 256;
constexpr int kRunPer = 8;                          // sectors per thread
constexpr ull kRunBlock = kRunThreads * kRunPer;   // sectors per block

struct RunRow {
  uint32_t t[9];
};

__device__ __forceinline__ RunRow run_row(const uint32_t* wc, const uint32_t* sc, ull g0, ull nw, ull s) {
  RunRow r;
#pragma unroll
  for (int b = 0; b < 8; ++b) r.t[b] = 8 * s + b < nw ? wc[8 * (g0 + s) + b] : 0u;
  r.t[8] = sc[g0 + s];
  return r;
}

__device__ __forceinline__ bool run_head(const uint32_t* wc, const uint32_t* sc, ull g0, ull nw, ull s) {
  if (s == 0) return true;
  const RunRow a = run_row(wc, sc, g0, nw, s), b = run_row(wc, sc, g0, nw, s - 1);
  bool diff = false;
#pragma unroll
  for (int k = 0; k < 9; ++k) diff |= a.t[k] != b.t[k];
  return diff;
}

__global__ void __launch_bounds__(kRunThreads) run_count_kernel(const uint32_t* __restrict__ wc,
                                                                const uint32_t* __restrict__ sc, ull g0, ull ns, ull nw,
                                                                uint32_t* __restrict__ bcount) {
  __shared__ uint32_t s_cnt;
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  uint32_t c = 0;
  const ull base = (ull)blockIdx.x * kRunBlock + (ull)threadIdx.x * kRunPer;
  for (int k = 0; k < kRunPer; ++k) {
    const ull s = base + k;
    if (s < ns && run_head(wc, sc, g0, nw, s)) ++c;
  }
  c = __reduce_add_sync(0xFFFFFFFFu, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(&s_cnt, c);
  __syncthreads();
  if (threadIdx.x == 0) bcount[blockIdx.x] = s_cnt;
}

// exclusive scan of nb block counts in place (one block); total -> *total
__global__ void run_scan_kernel(uint32_t* bcount, ull nb, ull* total) {
  __shared__ ull carry;
  __shared__ ull wsum[kRunThreads / 32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (ull b0 = 0; b0 < nb; b0 += kRunThreads) {
    const ull i = b0 + threadIdx.x;
    const ull v = i < nb ? bcount[i] : 0;
    ull incl = v;
    for (int d = 1; d < 32; d <<= 1) {
      const ull o = __shfl_up_sync(0xFFFFFFFFu, incl, d);
      if (lane >= d) incl += o;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    ull pre = carry;
    for (int k = 0; k < w; ++k) pre += wsum[k];
    if (i < nb) bcount[i] = (uint32_t)(pre + incl - v);
    __syncthreads();
    if (threadIdx.x == kRunThreads - 1) carry = pre + incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

__global__ void __launch_bounds__(kRunThreads) run_emit_kernel(const uint32_t* __restrict__ wc,
                                                               const uint32_t* __restrict__ sc, ull g0, ull ns, ull nw,
                                                               const uint32_t* __restrict__ boff,
                                                               thermo_run* __restrict__ out) {
  __shared__ uint32_t wsum[kRunThreads / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const ull base = (ull)blockIdx.x * kRunBlock + (ull)threadIdx.x * kRunPer;
  uint32_t heads = 0;  // bit k: sector base + k starts a run
  for (int k = 0; k < kRunPer; ++k) {
    const ull s = base + k;
    if (s < ns && run_head(wc, sc, g0, nw, s)) heads |= 1u << k;
  }
  const uint32_t c = __popc(heads);
  uint32_t incl = c;
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, incl, d);
    if (lane >= d) incl += o;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  uint32_t pre = boff[blockIdx.x];
  for (int k = 0; k < w; ++k) pre += wsum[k];
  pre += incl - c;
  for (int k = 0; k < kRunPer; ++k) {
    if (!((heads >> k) & 1u)) continue;
    const ull s = base + k;
    thermo_run r;
    r.start = s;
    r.count = 0;
    const RunRow row = run_row(wc, sc, g0, nw, s);
#pragma unroll
    for (int b = 0; b < 9; ++b) r.temp[b] = row.t[b];
    r.reserved = 0;
    out[pre++] = r;
  }
}

__global__ void run_len_kernel(thermo_run* runs, ull n, ull ns) {
  const ull i = (ull)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) runs[i].count = (i + 1 < n ? runs[i + 1].start : ns) - runs[i].start;
}

cudaError_t compress_runs(const uint32_t* wc, const uint32_t* sc, ull g0, ull ns, ull nw, uint32_t* scratch,
                          ull* d_total, thermo_run* out, ull out_cap, ull* n_runs, cudaStream_t s) {
  cudaError_t e;
  const ull nb = (ns + kRunBlock - 1) / kRunBlock;
  if (!nb) { *n_runs = 0; return cudaSuccess; }
  run_count_kernel<<<(unsigned)nb, kRunThreads, 0, s>>>(wc, sc, g0, ns, nw, scratch);
  run_scan_kernel<<<1, kRunThreads, 0, s>>>(scratch, nb, d_total);
  if ((e = cudaMemcpyAsync(n_runs, d_total, sizeof(ull), cudaMemcpyDeviceToHost, s))) return e;
  if ((e = cudaStreamSynchronize(s))) return e;
  if (!out || *n_runs > out_cap) return cudaSuccess;  // sizing call
  run_emit_kernel<<<(unsigned)nb, kRunThreads, 0, s>>>(wc, sc, g0, ns, nw, scratch, out);
  run_len_kernel<<<(unsigned)((*n_runs + 255) / 256), 256, 0, s>>>(out, *n_runs, ns);
  return cudaGetLastError();
}

}  // namespace thermo
