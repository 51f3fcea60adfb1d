// sort.cu -- row a4 (sort path): onesweep LSD radix sort of the 64-bit
// (sector, launch, warp | mask) keys on the prefix bits, replacing the paper's
// host-side sector_history_map (§IV-B2).  Sorting brings every
// (sector, launch, warp) tuple's copies together so a5 can count distinct
// warps per word and per sector with one segmented pass.
//
// One upfront pass histograms every 8-bit digit; each digit pass is then a
// single kernel: tiles take ids from an atomic counter, rank their keys with
// warp-level match (8 ballots), publish per-digit counts and resolve their
// global offsets by decoupled look-back, stage the tile in shared memory in
// digit order and write it out coalesced.  Status words carry an epoch so the
// look-back array never needs clearing.
#include "thermo_internal.cuh"

namespace thermo {

constexpr unsigned SFULL = 0xFFFFFFFFu;
constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kKPT = 16;                           // keys per thread
constexpr int kTile = kSortThreads * kKPT;         // 4096 keys per tile
constexpr int kMaxPasses = 7;
constexpr ull kFlagAgg = 1ull, kFlagInc = 2ull;
// status word: [63:56] epoch | [55:54] flag | [53:0] count
__device__ __forceinline__ ull pack_status(uint32_t epoch, ull flag, ull v) {
  return ((ull)(epoch & 0xFF) << 56) | (flag << 54) | (v & ((1ull << 54) - 1));
}

__device__ __forceinline__ unsigned lanemask_lt_s() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---- upfront histogram of all digit passes --------------------------------
__global__ void __launch_bounds__(256) sort_hist_kernel(const ull* __restrict__ keys, ull n, int lo_bit,
                                                        int passes, uint32_t* __restrict__ ghist) {
  __shared__ uint32_t sh[kMaxPasses][4][256];  // 4 sub-histograms to spread bank/addr conflicts
  for (int i = threadIdx.x; i < kMaxPasses * 4 * 256; i += blockDim.x) (&sh[0][0][0])[i] = 0;
  __syncthreads();
  const int sub = (threadIdx.x >> 5) & 3;
  const ull stride = (ull)gridDim.x * blockDim.x;
  for (ull i = (ull)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    ull k = keys[i];
#pragma unroll
    for (int p = 0; p < kMaxPasses; ++p) {
      if (p < passes) atomicAdd(&sh[p][sub][(k >> (lo_bit + 8 * p)) & 255], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * 256; i += blockDim.x) {
    int p = i >> 8, d = i & 255;
    uint32_t v = sh[p][0][d] + sh[p][1][d] + sh[p][2][d] + sh[p][3][d];
    if (v) atomicAdd(&ghist[p * 256 + d], v);
  }
}

// exclusive scan of each pass's histogram in place (one block, 256 threads)
__global__ void sort_scan_kernel(uint32_t* hist, int passes) {
  __shared__ uint32_t s[256];
  for (int p = 0; p < passes; ++p) {
    uint32_t v = hist[p * 256 + threadIdx.x];
    s[threadIdx.x] = v;
    __syncthreads();
    for (int d = 1; d < 256; d <<= 1) {
      uint32_t t = threadIdx.x >= d ? s[threadIdx.x - d] : 0;
      __syncthreads();
      s[threadIdx.x] += t;
      __syncthreads();
    }
    hist[p * 256 + threadIdx.x] = s[threadIdx.x] - v;
    __syncthreads();
  }
}

// ---- one digit pass ----------------------------------------------------------
__global__ void __launch_bounds__(kSortThreads, 3) onesweep_kernel(const ull* __restrict__ in, ull* __restrict__ out,
                                                                ull n, int shift,
                                                                const uint32_t* __restrict__ gofs,
                                                                ull* __restrict__ status,
                                                                uint32_t* __restrict__ tile_ctr, uint32_t epoch) {
  __shared__ uint32_t s_tile;
  __shared__ uint32_t whist[kSortWarps][256];
  __shared__ uint32_t blk_ofs[256];
  __shared__ ull glob_base[256];
  __shared__ ull stage[kTile];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
  for (int i = threadIdx.x; i < kSortWarps * 256; i += kSortThreads) (&whist[0][0])[i] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  const ull base = (ull)tile * kTile;
  const ull wbase = base + (ull)w * 32 * kKPT;

  ull k[kKPT];
  uint32_t rank[kKPT];
#pragma unroll
  for (int r = 0; r < kKPT; ++r) {
    ull idx = wbase + (ull)r * 32 + lane;
    k[r] = idx < n ? in[idx] : kEmptyKey;
  }
  // ---- warp-level ranking (stable: rounds in key order, lanes in order) ----
  const unsigned lt = lanemask_lt_s();
#pragma unroll
  for (int r = 0; r < kKPT; ++r) {
    ull idx = wbase + (ull)r * 32 + lane;
    const bool valid = idx < n;
    const uint32_t d = (uint32_t)(k[r] >> shift) & 255u;
    const unsigned peers = __match_any_sync(SFULL, valid ? d : 0x100u + lane);
    uint32_t old = 0;
    const int leader = __ffs(peers) - 1;
    if (valid && lane == leader) old = whist[w][d];
    // each lane fetches from its own leader: shfl with per-lane source
    old = __shfl_sync(SFULL, old, valid ? leader : lane);
    rank[r] = old + __popc(peers & lt);
    __syncwarp();
    if (valid && lane == leader) whist[w][d] = old + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // ---- per digit: exclusive offsets across warps, tile count ----
  const int t = threadIdx.x;  // digit
  uint32_t tot = 0;
#pragma unroll
  for (int ww = 0; ww < kSortWarps; ++ww) {
    uint32_t c = whist[ww][t];
    whist[ww][t] = tot;
    tot += c;
  }
  // ---- decoupled look-back for this digit ----
  volatile ull* vs = status;
  if (tile == 0) {
    vs[(ull)tile * 256 + t] = pack_status(epoch, kFlagInc, tot);
  } else {
    vs[(ull)tile * 256 + t] = pack_status(epoch, kFlagAgg, tot);
  }
  ull prefix = 0;
  if (tile > 0) {
    // look back 4 predecessors per step (independent loads in flight)
    const uint32_t ep8 = epoch & 0xFF;
    long long tp = (long long)tile - 1;
    while (tp >= 0) {
      ull s[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) s[j] = tp - j >= 0 ? vs[(ull)(tp - j) * 256 + t] : pack_status(ep8, kFlagInc, 0);
      bool stop = false;
      int used = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (stop) continue;
        const ull flag = (s[j] >> 54) & 3ull;
        if ((uint32_t)(s[j] >> 56) != ep8 || flag == 0) { stop = true; continue; }  // not ready: retry from here
        prefix += s[j] & ((1ull << 54) - 1);
        ++used;
        if (flag == kFlagInc) { stop = true; used = 1 << 20; }
      }
      if (used >= (1 << 20)) break;
      tp -= used;
    }
    __threadfence();
    vs[(ull)tile * 256 + t] = pack_status(epoch, kFlagInc, prefix + tot);
  }
  // ---- block exclusive scan of tot over digits ----
  blk_ofs[t] = tot;
  __syncthreads();
  for (int d = 1; d < 256; d <<= 1) {
    uint32_t v = t >= d ? blk_ofs[t - d] : 0;
    __syncthreads();
    blk_ofs[t] += v;
    __syncthreads();
  }
  const uint32_t excl = blk_ofs[t] - tot;
  __syncthreads();
  blk_ofs[t] = excl;
  glob_base[t] = (ull)gofs[t] + prefix;
  __syncthreads();
  // ---- stage in digit order, then write out coalesced ----
#pragma unroll
  for (int r = 0; r < kKPT; ++r) {
    ull idx = wbase + (ull)r * 32 + lane;
    if (idx < n) {
      uint32_t d = (uint32_t)(k[r] >> shift) & 255u;
      stage[blk_ofs[d] + whist[w][d] + rank[r]] = k[r];
    }
  }
  __syncthreads();
  const ull cnt = (n - base) < (ull)kTile ? (n - base) : (ull)kTile;
  for (uint32_t i = threadIdx.x; i < cnt; i += kSortThreads) {
    ull key = stage[i];
    uint32_t d = (uint32_t)(key >> shift) & 255u;
    out[glob_base[d] + (i - blk_ofs[d])] = key;
  }
}

ull* radix_sort_keys(ull* keys, ull n, int lo_bit, int nbits, SortWorkspace& ws, int num_sms, cudaStream_t s,
                     cudaError_t* err) {
  *err = cudaSuccess;
  if (n <= 1 || nbits <= 0) return keys;
  int passes = (nbits + 7) / 8;
  if (passes > kMaxPasses) { *err = cudaErrorInvalidValue; return keys; }
  ull tiles = (n + kTile - 1) / kTile;
  // workspace
  if (ws.alt_cap < n) {
    if (ws.alt) cudaFree(ws.alt);
    ws.alt_cap = n + n / 8;
    *err = cudaMalloc(&ws.alt, ws.alt_cap * sizeof(ull));
    if (*err) { ws.alt = nullptr; ws.alt_cap = 0; return keys; }
  }
  if (ws.status_cap < tiles * 256) {
    if (ws.status) cudaFree(ws.status);
    ws.status_cap = tiles * 256 + tiles * 32;
    *err = cudaMalloc(&ws.status, ws.status_cap * sizeof(ull));
    if (*err) { ws.status = nullptr; ws.status_cap = 0; return keys; }
    cudaMemsetAsync(ws.status, 0, ws.status_cap * sizeof(ull), s);
    ws.epoch = 0;
  }
  if (!ws.hist) {
    *err = cudaMalloc(&ws.hist, kMaxPasses * 256 * sizeof(uint32_t));
    if (*err) return keys;
    *err = cudaMalloc(&ws.counters, 8 * sizeof(uint32_t));
    if (*err) return keys;
  }
  cudaMemsetAsync(ws.hist, 0, kMaxPasses * 256 * sizeof(uint32_t), s);
  cudaMemsetAsync(ws.counters, 0, 8 * sizeof(uint32_t), s);
  unsigned hgrid = (unsigned)std::min<ull>((n + 255) / 256, (ull)num_sms * 8);
  sort_hist_kernel<<<hgrid, 256, 0, s>>>(keys, n, lo_bit, passes, ws.hist);
  sort_scan_kernel<<<1, 256, 0, s>>>(ws.hist, passes);
  ws.launches += 2 + passes;
  ull* src = keys;
  ull* dst = ws.alt;
  for (int p = 0; p < passes; ++p) {
    ws.epoch = (ws.epoch + 1) & 0xFF;
    if (ws.epoch == 0) {  // epoch wrapped: clear the status array once
      cudaMemsetAsync(ws.status, 0, ws.status_cap * sizeof(ull), s);
      ws.epoch = 1;
    }
    onesweep_kernel<<<(unsigned)tiles, kSortThreads, 0, s>>>(src, dst, n, lo_bit + 8 * p, ws.hist + p * 256,
                                                            ws.status, ws.counters + p, ws.epoch);
    ull* t = src; src = dst; dst = t;
  }
  *err = cudaGetLastError();
  return src;
}

}  // namespace thermo
