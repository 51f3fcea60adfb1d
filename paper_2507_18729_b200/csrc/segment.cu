// segment.cu -- rows a4 + a5 (+ the per-pc part of a6), "sector-segmented"
// dedup path: a counting sort of the keys by sector id, then one CTA per chunk
// of consecutive sectors deduplicates its keys in shared memory, writes the
// chunk's dense word/sector counts (the paper's popcount flush) and,
// from the same keys, the per-pc level histograms (G11).
//
// Why: a5 only needs the keys grouped per sector, and the sector range is
// small (SGEMM: 163,840 sectors), so an exact counting sort by sector
// (histogram, scan, scatter) groups them in ~3 streaming passes instead of one
// LSD pass per 8 key bits; the (launch, warp) and (pc) dedup then runs in a
// shared-memory hash set per chunk (one insert per key, no sort).  Sectors with more keys than a chunk holds make the caller
// fall back to the onesweep path (thermo_api.cu).
#include "thermo_internal.cuh"

namespace thermo {

constexpr unsigned GFULL = 0xFFFFFFFFu;
constexpr int kSegThreads = 256;
constexpr int kSegWarps = kSegThreads / 32;
constexpr int kSegCap = 2048;            // chunk window (keys); a chunk holds < 2 * kSegCap keys
constexpr int kScanBlock = 2048;         // scan elements per block (256 threads x 8)

__device__ __forceinline__ unsigned lanemask_lt_g() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
__device__ __forceinline__ int level_of_g(uint32_t c) { return 32 - __clz(c); }

// ---- 1. per-sector key histogram ----------------------------------------------
__global__ void seg_hist_kernel(const ull* __restrict__ keys, ull n, KeyLayout kl, uint32_t* __restrict__ cnt) {
  const ull stride = (ull)gridDim.x * blockDim.x;
  for (ull i = (ull)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) atomicAdd(&cnt[key_g(keys[i], kl)], 1u);
}

// ---- 2. exclusive scan of the S_tot counts (3 phases) ----------------------------
// a "big" sector (>= kSegCap keys) does not fit a chunk: its keys go to a
// separate buffer (hash path) and its segment here is empty
__device__ __forceinline__ uint32_t seg_len(uint32_t c) { return c >= (uint32_t)kSegCap ? 0u : c; }

__global__ void seg_scan_reduce(const uint32_t* __restrict__ in, ull n, ull* __restrict__ bsum,
                                uint32_t* __restrict__ maxc, ull* __restrict__ nbig) {
  __shared__ ull s[kSegWarps];
  __shared__ uint32_t smax[kSegWarps];
  const ull base = (ull)blockIdx.x * kScanBlock;
  ull t = 0, big = 0;
  uint32_t mx = 0;
  for (int i = threadIdx.x; i < kScanBlock; i += kSegThreads) {
    const ull j = base + i;
    const uint32_t v = j < n ? in[j] : 0u;
    t += seg_len(v);
    big += v - seg_len(v);
    mx = v > mx ? v : mx;
  }
  for (int d = 16; d; d >>= 1) big += __shfl_xor_sync(GFULL, big, d);
  if ((threadIdx.x & 31) == 0 && big) atomicAdd(nbig, big);
  for (int d = 16; d; d >>= 1) {
    t += __shfl_xor_sync(GFULL, t, d);
    const uint32_t o = __shfl_xor_sync(GFULL, mx, d);
    mx = o > mx ? o : mx;
  }
  if ((threadIdx.x & 31) == 0) { s[threadIdx.x >> 5] = t; smax[threadIdx.x >> 5] = mx; }
  __syncthreads();
  if (threadIdx.x == 0) {
    ull a = 0;
    uint32_t m = 0;
    for (int i = 0; i < kSegWarps; ++i) { a += s[i]; m = smax[i] > m ? smax[i] : m; }
    bsum[blockIdx.x] = a;
    atomicMax(maxc, m);
  }
}

// one block: exclusive scan of the block sums; writes the grand total to *total
__global__ void seg_scan_blocks(ull* bsum, ull nb, ull* total) {
  __shared__ ull carry;
  __shared__ ull ws[kSegWarps];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (ull b0 = 0; b0 < nb; b0 += kSegThreads) {
    const ull i = b0 + threadIdx.x;
    const ull v = i < nb ? bsum[i] : 0;
    ull incl = v;
    for (int d = 1; d < 32; d <<= 1) {
      const ull o = __shfl_up_sync(GFULL, incl, d);
      if (lane >= d) incl += o;
    }
    if (lane == 31) ws[w] = incl;
    __syncthreads();
    ull wpre = 0;
    for (int k = 0; k < w; ++k) wpre += ws[k];
    const ull c = carry;
    if (i < nb) bsum[i] = c + wpre + incl - v;
    __syncthreads();
    if (threadIdx.x == kSegThreads - 1) carry = c + wpre + incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

// off[j] = exclusive prefix of cnt; dst[j] = the chunk sector j's keys go to
// (the one its segment starts in; ~0 for a big sector)
__global__ void seg_scan_apply(const uint32_t* __restrict__ in, ull n, const ull* __restrict__ bsum,
                               ull* __restrict__ off, uint32_t* __restrict__ dst) {
  __shared__ ull ws[kSegWarps];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const ull base = (ull)blockIdx.x * kScanBlock + (ull)threadIdx.x * 8;
  uint32_t v[8];
  bool bg[8];
  ull t = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const ull j = base + k;
    const uint32_t c = j < n ? in[j] : 0u;
    v[k] = seg_len(c);
    bg[k] = c >= (uint32_t)kSegCap;
    t += v[k];
  }
  ull incl = t;
  for (int d = 1; d < 32; d <<= 1) {
    const ull o = __shfl_up_sync(GFULL, incl, d);
    if (lane >= d) incl += o;
  }
  if (lane == 31) ws[w] = incl;
  __syncthreads();
  ull pre = bsum[blockIdx.x];
  for (int k = 0; k < w; ++k) pre += ws[k];
  pre += incl - t;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const ull j = base + k;
    if (j < n) {
      off[j] = pre;
      dst[j] = bg[k] ? 0xFFFFFFFFu : (uint32_t)(pre / (ull)kSegCap);
    }
    pre += v[k];
  }
}

// ---- 3. scatter keys into their sector's segment ------------------------------------
// 8 keys per thread with their 8 cursor atomics in flight together: the
// atomics' latency (contended cursors of hot sectors), not bandwidth, bounds it
constexpr int kScatterPer = 8;
__global__ void __launch_bounds__(256) seg_scatter_kernel(const ull* __restrict__ keys, ull n, KeyLayout kl,
                                                          const uint32_t* __restrict__ dst, ull* __restrict__ cur,
                                                          ull* __restrict__ out, ull* __restrict__ big,
                                                          ull* __restrict__ nbig_ctr) {
  const int lane = threadIdx.x & 31;
  unsigned lt;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
  const ull tile = (ull)blockDim.x * kScatterPer;
  for (ull t0 = (ull)blockIdx.x * tile; t0 < n; t0 += (ull)gridDim.x * tile) {
    ull k[kScatterPer], pos[kScatterPer];
    uint32_t d[kScatterPer];
    const ull i0 = t0 + threadIdx.x;
#pragma unroll
    for (int u = 0; u < kScatterPer; ++u) k[u] = i0 + (ull)u * blockDim.x < n ? keys[i0 + (ull)u * blockDim.x] : 0;
    // one 4-byte read per key: the key's chunk (chunk cursors stay
    // cache-resident however many sectors there are) or ~0 for a big sector
#pragma unroll
    for (int u = 0; u < kScatterPer; ++u) d[u] = i0 + (ull)u * blockDim.x < n ? dst[key_g(k[u], kl)] : 0xFFFFFFFEu;
    // warp-aggregated cursor atomics: lanes holding keys of the same chunk take
    // consecutive positions from one atomic by their lowest lane
    unsigned peers[kScatterPer];
#pragma unroll
    for (int u = 0; u < kScatterPer; ++u) peers[u] = __match_any_sync(GFULL, d[u]);
#pragma unroll
    for (int u = 0; u < kScatterPer; ++u) {
      pos[u] = 0;
      if (d[u] < 0xFFFFFFFEu && lane == __ffs(peers[u]) - 1) pos[u] = atomicAdd(&cur[d[u]], (ull)__popc(peers[u]));
    }
#pragma unroll
    for (int u = 0; u < kScatterPer; ++u)
      pos[u] = __shfl_sync(GFULL, pos[u], __ffs(peers[u]) - 1) + __popc(peers[u] & lt);
#pragma unroll
    for (int u = 0; u < kScatterPer; ++u) {
      const bool isbig = d[u] == 0xFFFFFFFFu;
      const unsigned bb = __ballot_sync(GFULL, isbig);  // big keys: one append per warp
      if (bb) {
        ull b0 = 0;
        if (lane == __ffs(bb) - 1) b0 = atomicAdd(nbig_ctr, (ull)__popc(bb));
        b0 = __shfl_sync(GFULL, b0, __ffs(bb) - 1);
        if (isbig) big[b0 + __popc(bb & lt)] = k[u];
      }
      if (d[u] < 0xFFFFFFFEu) out[pos[u]] = k[u];
    }
  }
}

// ---- 4. per-chunk shared-memory dedup + count --------------------------------------
// chunk c owns the sectors whose segment starts in [c*kSegCap, (c+1)*kSegCap);
// their keys lie in [off[s0], off[s1]) and number < 2*kSegCap when every
// sector has < kSegCap keys (checked by the caller).
__device__ __forceinline__ ull first_sector_at(const ull* off, ull nsec, ull pos) {
  ull lo = 0, hi = nsec;  // smallest s with off[s] >= pos (off[nsec] = total)
  while (lo < hi) {
    const ull mid = (lo + hi) >> 1;
    if (off[mid] >= pos) hi = mid; else lo = mid + 1;
  }
  return lo;
}

// chunk cursors: chunk c's keys start where its first sector's segment does
// (and each chunk's first sector, so the chunk kernel needs no search)
__global__ void seg_chunk_cursor_kernel(const ull* __restrict__ off, ull nsec, ull nchunks, ull* __restrict__ cur,
                                        ull* __restrict__ cs0) {
  const ull c = (ull)blockIdx.x * blockDim.x + threadIdx.x;
  if (c <= nchunks) {
    const ull s = first_sector_at(off, nsec, c * kSegCap);
    cs0[c] = s;
    if (c < nchunks) cur[c] = off[s];
  }
}


// per-block (pc, level) bin table in shared memory: open addressing on the
// bin id; a full table falls back to the global atomic
constexpr int kPcBins = 512;
__device__ __forceinline__ void bin_add(uint32_t* tbin, uint32_t* tcnt, ull* g, uint32_t bin, uint32_t v) {
  uint32_t h = (bin * 0x9E3779B1u) >> (32 - 9);
  for (int probe = 0; probe < 16; ++probe) {
    uint32_t cur = tbin[h];
    if (cur == 0xFFFFFFFFu) {
      cur = atomicCAS(&tbin[h], 0xFFFFFFFFu, bin);
      if (cur == 0xFFFFFFFFu) cur = bin;
    }
    if (cur == bin) { atomicAdd(&tcnt[h], v); return; }
    h = (h + 1) & (kPcBins - 1);
  }
  atomicAdd(&g[bin], (ull)v);
}

// chunk hash set in shared memory: slot = (id << 8 | mask), id = the key's
// (sector, launch, warp) or (sector, pc id) with the sector relative to the
// chunk's first; insert ORs the mask into the id's slot (the OR of a
// word's accesses is idempotent)
constexpr int kHSlots = 5120;  // > 1.25 x the chunk's < 2 * kSegCap keys (typically ~2/3 of that)
constexpr int kHWin = 1024;    // chunks spanning at most this many sectors count them in shared memory
constexpr ull kHEmpty = ~0ull;
// insert returns true when the id takes a new slot (*slot); the caller appends
// new slots to the chunk's list (one atomic per warp), so the scans visit
// occupied slots only.  The mask lives in the slot's low 32-bit word: the OR
// is a native 32-bit shared atomic (a 64-bit atomicOr is a CAS loop)
__device__ __forceinline__ bool hset_or(ull* tab, ull id, uint32_t m, uint32_t& slot) {
  const uint32_t hx = (uint32_t)((id * 0x9E3779B97F4A7C15ull) >> 32);
  uint32_t h = __umulhi(hx, (uint32_t)kHSlots);
  const ull v = (id << 8) | m;
  for (;;) {
    ull cur = tab[h];
    if (cur == kHEmpty) {
      cur = atomicCAS(&tab[h], kHEmpty, v);
      if (cur == kHEmpty) {
        slot = h;
        return true;
      }
    }
    if ((cur >> 8) == id) {
      if (((uint32_t)cur & m) != m) atomicOr(reinterpret_cast<uint32_t*>(&tab[h]), m);
      return false;
    }
    h = h + 1 == (uint32_t)kHSlots ? 0u : h + 1;
  }
}

// one insert pass over the chunk's keys seg[k0, k0 + nk): id = (sector - s0) <<
// A | (key >> B) & M, mask = the key's low 8 bits.  Each warp takes 32 x kIns
// consecutive keys per iteration, all loads in flight before the inserts
constexpr int kIns = 4;
__device__ __forceinline__ void chunk_insert_pass(ull* tab, uint16_t* list, uint32_t* nlist, const ull* __restrict__ seg,
                                                  ull k0, uint32_t nk, ull s0, const KeyLayout& kl, uint32_t filter,
                                                  uint32_t A, uint32_t B, ull M) {
  const int lane = threadIdx.x & 31;
  unsigned lt;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
  for (uint32_t wb = (threadIdx.x >> 5) * 32u * kIns; wb < nk; wb += (uint32_t)kSegThreads * kIns) {
    ull kk[kIns];
#pragma unroll
    for (int u = 0; u < kIns; ++u) {
      const uint32_t i = wb + u * 32u + lane;
      kk[u] = i < nk ? seg[k0 + i] : 0ull;
    }
#pragma unroll
    for (int u = 0; u < kIns; ++u) {
      const ull k = kk[u];
      bool ok = wb + u * 32u + lane < nk;
      if (filter != THERMO_ALL_LAUNCHES) ok = ok && key_launch(k, kl) == filter;
      uint32_t slot = 0;
      const bool nw = ok && hset_or(tab, ((key_g(k, kl) - s0) << A) | ((k >> B) & M), (uint32_t)k & 0xFFu, slot);
      const unsigned b = __ballot_sync(GFULL, nw);
      if (b) {
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(nlist, (uint32_t)__popc(b));
        base = __shfl_sync(GFULL, base, 0);
        if (nw) list[base + __popc(b & lt)] = (uint16_t)slot;
      }
    }
  }
}

// chunk c owns the sectors [cs0[c], cs0[c + 1]) (those whose segment starts in
// [c kSegCap, (c + 1) kSegCap)); their keys are seg[off[s0], off[s1]), fewer
// than 2 kSegCap.  (a) distinct (sector, launch, warp) with OR-ed masks in a
// shared-memory hash set -> sector count = #entries, word b's count = #entries
// with bit b (the popcount flush of P:328, G6), summed per sector in shared
// memory (or, for a chunk spanning > kHWin sectors, with warp-aggregated
// global atomics); (b) distinct (sector, pc id) with OR-ed masks -> per-pc
// level histograms (G11)
__global__ void __launch_bounds__(kSegThreads, 3) seg_chunk_kernel(const ull* __restrict__ seg, const ull* __restrict__ off,
                                                               ull nsec, KeyLayout kl, uint32_t filter,
                                                               uint32_t* __restrict__ wc, uint32_t* __restrict__ sc,
                                                               const uint32_t* __restrict__ site_of,
                                                               ull* __restrict__ pc_hist, DevCounters* ctr,
                                                               const ull* __restrict__ cs0) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ull* tab = reinterpret_cast<ull*>(smem_raw);                    // [kHSlots]
  uint32_t* cnt = reinterpret_cast<uint32_t*>(tab + kHSlots);     // [kHWin][5]: words (2b, 2b+1) as u16 pairs, sector
  uint32_t* tbin = cnt + kHWin * 5;                               // [kPcBins]
  uint32_t* tcnt = tbin + kPcBins;                                // [kPcBins]
  uint16_t* list = reinterpret_cast<uint16_t*>(tcnt + kPcBins);   // [2 kSegCap] occupied slots
  __shared__ uint32_t s_n[2];
  const int lane = threadIdx.x & 31;
  const ull c = blockIdx.x;
  const ull s0 = cs0[c], s1 = cs0[c + 1];
  if (s0 >= s1) return;
  const ull k0 = off[s0];
  const uint32_t nk = (uint32_t)(off[s1] - k0);  // < 2 kSegCap
  const ull win = s1 - s0;
  const bool local = win <= (ull)kHWin;
  const uint32_t LW = kl.L + kl.W, RS = 8 + kl.P;
  const ull lwmask = (1ull << LW) - 1;
  for (int i = threadIdx.x; i < kHSlots; i += kSegThreads) tab[i] = kHEmpty;
  if (threadIdx.x < 2) s_n[threadIdx.x] = 0;
  if (local)
    for (uint32_t i = threadIdx.x; i < (uint32_t)win * 5; i += kSegThreads) cnt[i] = 0;
  __syncthreads();
  // ---- (a) distinct (sector, launch, warp) ----
  chunk_insert_pass(tab, list, &s_n[0], seg, k0, nk, s0, kl, filter, LW, RS, lwmask);
  __syncthreads();
  const uint32_t nent = s_n[0];
  for (uint32_t base = threadIdx.x & ~31u; base < nent; base += kSegThreads) {  // warp-uniform trip count
    const uint32_t i = base + lane;
    const bool occ = i < nent;
    const ull v = occ ? tab[list[i]] : kHEmpty;
    const uint32_t gl = occ ? (uint32_t)(v >> (8 + LW)) : 0xFFFFFFFFu;
    const uint32_t m = occ ? (uint32_t)v & 0xFFu : 0u;
    const unsigned peers = __match_any_sync(GFULL, gl);
    uint32_t cb[8];
#pragma unroll
    for (int b = 0; b < 8; ++b) cb[b] = __popc(__ballot_sync(GFULL, (m >> b) & 1u) & peers);
    if (occ && lane == __ffs(peers) - 1) {
      const uint32_t cs = __popc(peers);
      if (local) {
        uint32_t* cg = cnt + gl * 5;
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (cb[2 * j] | cb[2 * j + 1]) atomicAdd(&cg[j], cb[2 * j] | (cb[2 * j + 1] << 16));
        atomicAdd(&cg[4], cs);
      } else {
        const ull g = s0 + gl;
        atomicAdd(&sc[g], cs);
#pragma unroll
        for (int b = 0; b < 8; ++b)
          if (cb[b]) atomicAdd(&wc[8 * g + b], cb[b]);
      }
    }
  }
  if (threadIdx.x == 0 && nent) atomicAdd(&ctr->distinct_pairs, (ull)nent);
  __syncthreads();
  if (local) {  // the chunk owns its sectors: plain stores of the nonzero rows
    for (uint32_t j = threadIdx.x; j < (uint32_t)win; j += kSegThreads) {
      const uint32_t* cg = cnt + j * 5;
      if (cg[4] == 0) continue;
      const ull g = s0 + j;
      sc[g] = cg[4];
      uint4 lo, hi;
      lo.x = cg[0] & 0xFFFFu; lo.y = cg[0] >> 16; lo.z = cg[1] & 0xFFFFu; lo.w = cg[1] >> 16;
      hi.x = cg[2] & 0xFFFFu; hi.y = cg[2] >> 16; hi.z = cg[3] & 0xFFFFu; hi.w = cg[3] >> 16;
      reinterpret_cast<uint4*>(wc + 8 * g)[0] = lo;
      reinterpret_cast<uint4*>(wc + 8 * g)[1] = hi;
    }
  }
  if (!pc_hist) return;
  // ---- (b) distinct (sector, pc id) -> per-pc level histograms ----
  for (int i = threadIdx.x; i < kHSlots; i += kSegThreads) tab[i] = kHEmpty;
  for (int i = threadIdx.x; i < kPcBins; i += kSegThreads) { tbin[i] = 0xFFFFFFFFu; tcnt[i] = 0; }
  __syncthreads();
  const ull pmask = (1ull << kl.P) - 1;
  chunk_insert_pass(tab, list, &s_n[1], seg, k0, nk, s0, kl, filter, kl.P, 8, pmask);
  __syncthreads();
  const uint32_t npc = s_n[1];
  for (uint32_t base = threadIdx.x & ~31u; base < npc; base += kSegThreads) {
    const uint32_t i = base + lane;
    const bool head = i < npc;
    const ull v = head ? tab[list[i]] : kHEmpty;
    const uint32_t gl = (uint32_t)(v >> (8 + kl.P));
    const uint32_t pcid = (uint32_t)((v >> 8) & pmask);
    const uint32_t m = (uint32_t)v & 0xFFu;
    const uint32_t* cg = cnt + gl * 5;
    const ull g = s0 + gl;
    {
      const uint32_t scv = head ? (local ? cg[4] : __ldcg(&sc[g])) : 0u;
      const uint32_t bin = head ? (pcid * 2 + 1) * kLevels + level_of_g(scv) : 0xFFFFFFFFu;
      const unsigned mm = __match_any_sync(GFULL, bin);
      if (head && (__ffs(mm) - 1) == lane) bin_add(tbin, tcnt, pc_hist, bin, __popc(mm));
    }
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const bool hb = head && ((m >> b) & 1u);
      uint32_t wv = 0;
      if (hb) wv = local ? ((cg[b >> 1] >> (16 * (b & 1))) & 0xFFFFu) : __ldcg(&wc[8 * g + b]);
      const uint32_t bin = hb ? (pcid * 2) * kLevels + level_of_g(wv) : 0xFFFFFFFFu;
      const unsigned mm = __match_any_sync(GFULL, bin);
      if (hb && (__ffs(mm) - 1) == lane) bin_add(tbin, tcnt, pc_hist, bin, __popc(mm));
    }
  }
  if (threadIdx.x == 0 && npc) atomicAdd(&ctr->distinct_pc, (ull)npc);
  __syncthreads();
  for (int i = threadIdx.x; i < kPcBins; i += kSegThreads)
    if (tbin[i] != 0xFFFFFFFFu && tcnt[i]) atomicAdd(&pc_hist[tbin[i]], (ull)tcnt[i]);
  (void)site_of;
  (void)nsec;
}

static size_t segment_chunk_smem() {
  return (size_t)kHSlots * sizeof(ull) + ((size_t)kHWin * 5 + 2 * kPcBins) * sizeof(uint32_t) +
         2 * kSegCap * sizeof(uint16_t);
}
ull segment_chunk_cap() { return kSegCap; }

// phases 1-2; syncs once so the caller can read the largest per-sector count
cudaError_t segment_reserve(SegWorkspace& ws, ull nsec) {
  cudaError_t e;
  if (ws.cap_sec < nsec + 1) {
    cudaFree(ws.cnt); cudaFree(ws.off); cudaFree(ws.cur); cudaFree(ws.bsum); cudaFree(ws.cs0); cudaFree(ws.dst);
    ws.cnt = nullptr; ws.off = ws.cur = ws.bsum = ws.cs0 = nullptr;
    ws.dst = nullptr;
    ws.cap_sec = 0;
    if ((e = cudaMalloc(&ws.cnt, (nsec + 1) * sizeof(uint32_t)))) return e;
    if ((e = cudaMalloc(&ws.off, (nsec + 1) * sizeof(ull)))) return e;
    if ((e = cudaMalloc(&ws.cur, (nsec + 1) * sizeof(ull)))) return e;
    if ((e = cudaMalloc(&ws.cs0, (nsec + 2) * sizeof(ull)))) return e;
    if ((e = cudaMalloc(&ws.dst, (nsec + 1) * sizeof(uint32_t)))) return e;
    if ((e = cudaMalloc(&ws.bsum, ((nsec + kScanBlock) / kScanBlock + 1) * sizeof(ull)))) return e;
    ws.cap_sec = nsec + 1;
  }
  if (!ws.maxc && (e = cudaMalloc(&ws.maxc, 4 * sizeof(ull)))) return e;  // maxc, big total, big cursor
  return cudaSuccess;
}

cudaError_t segment_prepare(const ull* keys, ull n, KeyLayout kl, ull nsec, SegWorkspace& ws, int num_sms,
                            cudaStream_t s, uint32_t* max_per_sector, ull* n_big, bool counted) {
  cudaError_t e;
  if ((e = segment_reserve(ws, nsec))) return e;
  cudaMemsetAsync(ws.maxc, 0, 4 * sizeof(ull), s);  // maxc, big-key total, big-key cursor
  if (!counted) {
    cudaMemsetAsync(ws.cnt, 0, (nsec + 1) * sizeof(uint32_t), s);
    if (n) {
      const unsigned grid = (unsigned)std::min<ull>((n + 255) / 256, (ull)num_sms * 16);
      seg_hist_kernel<<<grid, 256, 0, s>>>(keys, n, kl, ws.cnt);
      ws.launches += 1;
    }
  }
  const ull nb = (nsec + kScanBlock - 1) / kScanBlock;
  seg_scan_reduce<<<(unsigned)nb, kSegThreads, 0, s>>>(ws.cnt, nsec, ws.bsum, ws.maxc,
                                                       reinterpret_cast<ull*>(ws.maxc) + 1);
  seg_scan_blocks<<<1, kSegThreads, 0, s>>>(ws.bsum, nb, ws.off + nsec);
  seg_scan_apply<<<(unsigned)nb, kSegThreads, 0, s>>>(ws.cnt, nsec, ws.bsum, ws.off, ws.dst);
  ws.launches += 3;
  ull hv[2];
  if ((e = cudaMemcpyAsync(hv, ws.maxc, 2 * sizeof(ull), cudaMemcpyDeviceToHost, s))) return e;
  if ((e = cudaStreamSynchronize(s))) return e;
  *max_per_sector = (uint32_t)hv[0];
  *n_big = hv[1];
  return cudaSuccess;
}

// phases 3-4: keys -> out (grouped by sector) -> dense counts (+ per-pc histograms)
cudaError_t segment_count(const ull* keys, ull n, ull* out, ull* big, KeyLayout kl, ull nsec, uint32_t filter,
                          SegWorkspace& ws, uint32_t* wc, uint32_t* sc, const uint32_t* site_of, ull* pc_hist,
                          DevCounters* ctr, int num_sms, cudaStream_t s) {
  if (n) {
    const unsigned grid = (unsigned)std::min<ull>((n + 256 * kScatterPer - 1) / (256 * kScatterPer), (ull)num_sms * 8);
    const ull nch = (n + kSegCap - 1) / kSegCap;  // <= nsec + 1 = the cursor array's size
    seg_chunk_cursor_kernel<<<(unsigned)((nch + 256) / 256), 256, 0, s>>>(ws.off, nsec, nch, ws.cur, ws.cs0);
    seg_scatter_kernel<<<grid, 256, 0, s>>>(keys, n, kl, ws.dst, ws.cur, out, big,
                                            reinterpret_cast<ull*>(ws.maxc) + 2);
  }
  const size_t smem = segment_chunk_smem();
  smem_optin((const void*)seg_chunk_kernel, (int)smem);
  const ull chunks = (n + kSegCap - 1) / kSegCap;
  if (chunks)
    seg_chunk_kernel<<<(unsigned)chunks, kSegThreads, smem, s>>>(out, ws.off, nsec, kl, filter, wc, sc, site_of,
                                                                  pc_hist, ctr, ws.cs0);
  ws.launches += 2;
  return cudaGetLastError();
}

}  // namespace thermo
