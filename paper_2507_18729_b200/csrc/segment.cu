// segment.cu -- rows a4 + a5 (+ the per-pc part of a6), "sector-segmented"
// dedup path: a counting sort of the keys by sector id, then shared-memory
// sets per chunk of consecutive sectors, which write the chunk's dense word /
// sector counts (the paper's popcount flush) and, from the same keys,
// the per-pc level histograms (G11).
//
// Why: a5 only needs the keys grouped per sector.  The decoder counts keys per
// sector as it writes them; scans give every sector its segment; two
// onesweep-style partition passes (coarse buckets balanced by key count, then
// chunks) move the keys there with coalesced writes; one CTA per chunk (< 4096
// keys) dedups in shared memory.  Sectors with >= 2048 keys (hot sectors, e.g.
// SpMV's power-law x columns) get their own segments and are reduced by one CTA
// per (sector, warp-hash pass) in seg_big_kernel.
#include "thermo_internal.cuh"

namespace thermo {

constexpr unsigned GFULL = 0xFFFFFFFFu;
constexpr int kSegThreads = 256;
constexpr int kSegWarps = kSegThreads / 32;
constexpr int kSegCap = 2048;            // chunk window (keys); a chunk holds < 2 * kSegCap keys
constexpr int kChunkSec = 1024;          // a chunk spans at most this many sectors (its rows fit the CTA)
// chunk of sector j with normal-key prefix off: both terms are non-decreasing
// in j, so a chunk (the sectors with one value) lies in one kSegCap window of
// keys (< 2 kSegCap keys) and in one kChunkSec block of sectors
__host__ __device__ __forceinline__ ull chunk_of(ull off, ull j) { return off / kSegCap + j / kChunkSec; }
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

constexpr int kGroup = 64;               // sectors per coarse-bucket granule
// ---- 2. exclusive scans of the S_tot counts (3 phases) ---------------------------
// Per sector g with c = cnt[g] keys, three running sums:
//   NL  normal keys  (c < kSegCap)   -> off[g], the sector's segment in the chunked layout
//   BS  big sectors  (c >= kSegCap)  -> the sector's big index i (its keys go to `big`)
//   BK  big keys                     -> boff[i], the sector's segment in `big`
// and, at every coarse bucket boundary (g % 2^cs == 0), the bucket's first key
// in the coarse layout (NL + BK) and its (NL, BS) starts.
__device__ __forceinline__ uint32_t seg_len(uint32_t c) { return c >= (uint32_t)kSegCap ? 0u : c; }

struct Sum3 {
  ull nl, bs, bk;
};
__device__ __forceinline__ Sum3 sum3_of(uint32_t c) {
  const bool big = c >= (uint32_t)kSegCap;
  return Sum3{big ? 0ull : (ull)c, big ? 1ull : 0ull, big ? (ull)c : 0ull};
}
__device__ __forceinline__ Sum3 warp_incl_scan3(Sum3 v, int lane) {
  for (int d = 1; d < 32; d <<= 1) {
    const ull a = __shfl_up_sync(GFULL, v.nl, d), b = __shfl_up_sync(GFULL, v.bs, d),
              c = __shfl_up_sync(GFULL, v.bk, d);
    if (lane >= d) { v.nl += a; v.bs += b; v.bk += c; }
  }
  return v;
}

__global__ void seg_scan_reduce(const uint32_t* __restrict__ in, ull n, ull* __restrict__ bsum3,
                                uint32_t* __restrict__ maxc) {
  __shared__ ull s[3][kSegWarps];
  __shared__ uint32_t smax[kSegWarps];
  const ull base = (ull)blockIdx.x * kScanBlock;
  Sum3 t{0, 0, 0};
  uint32_t mx = 0;
  // 16-byte loads: thread t reads counts [4 t, 4 t + 4) and [1024 + 4 t, ...)
  for (int i = threadIdx.x * 4; i < kScanBlock; i += kSegThreads * 4) {
    const ull j = base + i;
    uint32_t v[4];
    if (j + 4 <= n) {
      const uint4 q4 = *reinterpret_cast<const uint4*>(in + j);
      v[0] = q4.x; v[1] = q4.y; v[2] = q4.z; v[3] = q4.w;
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k] = j + k < n ? in[j + k] : 0u;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const Sum3 q = sum3_of(v[k]);
      t.nl += q.nl; t.bs += q.bs; t.bk += q.bk;
      mx = v[k] > mx ? v[k] : mx;
    }
  }
  for (int d = 16; d; d >>= 1) {
    t.nl += __shfl_xor_sync(GFULL, t.nl, d);
    t.bs += __shfl_xor_sync(GFULL, t.bs, d);
    t.bk += __shfl_xor_sync(GFULL, t.bk, d);
    const uint32_t o = __shfl_xor_sync(GFULL, mx, d);
    mx = o > mx ? o : mx;
  }
  if ((threadIdx.x & 31) == 0) {
    s[0][threadIdx.x >> 5] = t.nl; s[1][threadIdx.x >> 5] = t.bs; s[2][threadIdx.x >> 5] = t.bk;
    smax[threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    ull a = 0;
    for (int i = 0; i < kSegWarps; ++i) a += s[threadIdx.x][i];
    bsum3[3 * blockIdx.x + threadIdx.x] = a;
  }
  if (threadIdx.x == 0) {
    uint32_t m = 0;
    for (int i = 0; i < kSegWarps; ++i) m = smax[i] > m ? smax[i] : m;
    atomicMax(maxc, m);
  }
}

// one block: exclusive scan of the block sums (three columns); totals -> tot[0..3)
constexpr int kScanBT = 1024;  // seg_scan_blocks threads: each scans a contiguous run of block sums
__global__ void __launch_bounds__(kScanBT) seg_scan_blocks(ull* bsum3, ull nb, ull* tot, ull nsec, ull* cs0,
                                                           ull* cko) {
  __shared__ ull ws[3][kScanBT / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const ull per = (nb + kScanBT - 1) / kScanBT;
  const ull i0 = (ull)threadIdx.x * per, i1 = i0 + per < nb ? i0 + per : nb;
  Sum3 t{0, 0, 0};
  for (ull i = i0; i < i1; ++i) { t.nl += bsum3[3 * i]; t.bs += bsum3[3 * i + 1]; t.bk += bsum3[3 * i + 2]; }
  const Sum3 incl = warp_incl_scan3(t, lane);
  if (lane == 31) { ws[0][w] = incl.nl; ws[1][w] = incl.bs; ws[2][w] = incl.bk; }
  __syncthreads();
  Sum3 pre{0, 0, 0}, all{0, 0, 0};
  for (int k = 0; k < kScanBT / 32; ++k) {
    if (k < w) { pre.nl += ws[0][k]; pre.bs += ws[1][k]; pre.bk += ws[2][k]; }
    all.nl += ws[0][k]; all.bs += ws[1][k]; all.bk += ws[2][k];
  }
  pre.nl += incl.nl - t.nl; pre.bs += incl.bs - t.bs; pre.bk += incl.bk - t.bk;
  for (ull i = i0; i < i1; ++i) {
    const Sum3 v{bsum3[3 * i], bsum3[3 * i + 1], bsum3[3 * i + 2]};
    bsum3[3 * i] = pre.nl; bsum3[3 * i + 1] = pre.bs; bsum3[3 * i + 2] = pre.bk;
    pre.nl += v.nl; pre.bs += v.bs; pre.bk += v.bk;
  }
  if (threadIdx.x == 0) { tot[0] = all.nl; tot[1] = all.bs; tot[2] = all.bk; }
  (void)nsec; (void)cs0; (void)cko;
}

// With off[g] = the normal-key prefix at sector g (the sector's segment in the
// chunked layout, never stored): dst[g] = chunk_of(off[g], g) of g's normal
// keys, or 0x80000000 | big index for a big sector (then bg[i] = g, boff[i] =
// big-key prefix); the chunks (chunk_of(g - 1), chunk_of(g)] start at g
// (at most two: a normal segment is shorter than kSegCap): cs0[c] = g, cko[c]
// = off[g]; after the last sector the end of the table (cs0 = n, cko = NL) and
// the chunk count -> *nch;
// gpre[q] = (NL, BS, BK) at the first sector of group q (kGroup sectors)
__global__ void seg_scan_apply(const uint32_t* __restrict__ in, ull n, const ull* __restrict__ bsum3,
                               ull* __restrict__ cs0, ull* __restrict__ cko, uint32_t* __restrict__ dst,
                               ull* __restrict__ bg, ull* __restrict__ boff, ull* __restrict__ gpre,
                               ull* __restrict__ nch) {
  __shared__ ull ws[3][kSegWarps];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const ull base = (ull)blockIdx.x * kScanBlock + (ull)threadIdx.x * 8;
  uint32_t v[8];
  if (base + 8 <= n) {  // two 16-byte loads (32-byte aligned)
    const uint4 a0 = reinterpret_cast<const uint4*>(in + base)[0], a1 = reinterpret_cast<const uint4*>(in + base)[1];
    v[0] = a0.x; v[1] = a0.y; v[2] = a0.z; v[3] = a0.w; v[4] = a1.x; v[5] = a1.y; v[6] = a1.z; v[7] = a1.w;
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = base + k < n ? in[base + k] : 0u;
  }
  Sum3 t{0, 0, 0};
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const Sum3 q = sum3_of(v[k]);
    t.nl += q.nl; t.bs += q.bs; t.bk += q.bk;
  }
  const Sum3 incl = warp_incl_scan3(t, lane);
  if (lane == 31) { ws[0][w] = incl.nl; ws[1][w] = incl.bs; ws[2][w] = incl.bk; }
  __syncthreads();
  Sum3 pre{bsum3[3 * blockIdx.x], bsum3[3 * blockIdx.x + 1], bsum3[3 * blockIdx.x + 2]};
  for (int k = 0; k < w; ++k) { pre.nl += ws[0][k]; pre.bs += ws[1][k]; pre.bk += ws[2][k]; }
  pre.nl += incl.nl - t.nl; pre.bs += incl.bs - t.bs; pre.bk += incl.bk - t.bk;
  uint32_t vprev = (base > 0 && base - 1 < n) ? in[base - 1] : 0u;  // the previous sector's keys
  uint32_t dd[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const ull j = base + k;
    if (j < n) {
      const ull c = chunk_of(pre.nl, j);
      for (ull cc = j == 0 ? 0 : chunk_of(pre.nl - seg_len(vprev), j - 1) + 1; cc <= c; ++cc) {
        cs0[cc] = j;
        cko[cc] = pre.nl;
      }
      if (j == n - 1) {
        cs0[c + 1] = n;
        cko[c + 1] = pre.nl + seg_len(v[k]);
        *nch = c + 1;
      }
      const bool big = v[k] >= (uint32_t)kSegCap;
      if (big) {
        dd[k] = 0x80000000u | (uint32_t)pre.bs;
        bg[pre.bs] = j;
        boff[pre.bs] = pre.bk;
      } else {
        dd[k] = (uint32_t)c;
      }
      if ((j & (kGroup - 1)) == 0) {
        gpre[3 * (j / kGroup)] = pre.nl;
        gpre[3 * (j / kGroup) + 1] = pre.bs;
        gpre[3 * (j / kGroup) + 2] = pre.bk;
      }
    }
    const Sum3 q = sum3_of(v[k]);
    pre.nl += q.nl; pre.bs += q.bs; pre.bk += q.bk;
    vprev = v[k];
  }
  if (base + 8 <= n) {
    reinterpret_cast<uint4*>(dst + base)[0] = make_uint4(dd[0], dd[1], dd[2], dd[3]);
    reinterpret_cast<uint4*>(dst + base)[1] = make_uint4(dd[4], dd[5], dd[6], dd[7]);
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (base + k < n) dst[base + k] = dd[k];
  }
}

// coarse buckets balanced by key count: group q (kGroup sectors) goes to
// bucket cb[q] = (keys before q) * ncoarse / n, non-decreasing in q; bucket b
// starts at its first group's prefixes (cstart = all keys, cinfo = (NL, BS,
// first sector));
// buckets no group maps to are empty (the next group's / the totals' start)
__global__ void seg_groups_kernel(const ull* __restrict__ gpre, ull ngroups, const ull* __restrict__ tot,
                                  uint32_t ncoarse, uint16_t* __restrict__ cb, ull* __restrict__ cstart,
                                  ull* __restrict__ cinfo, ull nsec) {
  const ull q = (ull)blockIdx.x * blockDim.x + threadIdx.x;
  if (q > ngroups) return;
  const ull n = tot[0] + tot[2];
  auto bucket = [&](ull qq) -> uint32_t {
    if (qq >= ngroups) return ncoarse;
    const ull p = gpre[3 * qq] + gpre[3 * qq + 2];
    const ull b = n ? (ull)(((unsigned __int128)p * ncoarse) / n) : 0ull;
    return (uint32_t)(b < ncoarse ? b : ncoarse - 1);
  };
  const uint32_t bq = bucket(q);
  if (q < ngroups) cb[q] = (uint16_t)bq;
  const uint32_t bp = q == 0 ? 0u : bucket(q - 1) + 1;  // buckets (bucket(q-1), bucket(q)] start here
  const ull nl = q < ngroups ? gpre[3 * q] : tot[0], bs = q < ngroups ? gpre[3 * q + 1] : tot[1];
  const ull all = q < ngroups ? gpre[3 * q] + gpre[3 * q + 2] : n;
  const ull g0 = q < ngroups ? q * kGroup : nsec;
  for (uint32_t b = bp; b <= bq; ++b) {
    cstart[b] = all;
    cinfo[3 * b] = nl;
    cinfo[3 * b + 1] = bs;
    cinfo[3 * b + 2] = g0;
  }
}

// ---- 3. two-pass partition of the keys into chunks and big sectors ----------------
// A single scatter to ~n / 2048 chunk cursors writes 8-byte keys to random
// places through a dependent key -> chunk -> cursor-atomic chain (ncu: 9 %
// issue-active, long-scoreboard bound).  Instead, two onesweep-style passes
// with <= 4096 destinations each: a tile of 4096 keys is ranked by destination
// in shared memory, takes one cursor atomic per destination present, is staged
// in destination order and written out in runs.
//   pass 1: coarse bucket b = cb[g / kGroup] (<= kCoarse buckets balanced by
//           key count, so each holds about n / kCoarse keys), into `tmp`;
//   pass 2: per coarse bucket, the key's chunk or big sector, into `out` / `big`
//           (a bucket's chunks and big sectors are consecutive ids, and the
//           chunk-of-sector lookups stay within the bucket's sector range).
constexpr int kCoarse = 1024;
constexpr int kPT = 512;                 // partition threads (16 warps: two CTAs fill an SM's 32 warps)
constexpr int kPPer = 8;                 // keys per thread
constexpr int kPTile = kPT * kPPer;      // 4096 keys per tile
constexpr int kFPer = 4;                 // pass 2: keys per thread
constexpr int kFTile = kPT * kFPer;      // pass-2 tile (2048 keys): smaller tiles, three CTAs per SM
constexpr int kFineBins = 2048;          // pass-2 destinations per bucket (more: direct scatter)

// block-wide exclusive scan of cnt[0, nbins) into excl (nbins <= kFineBins), returns the total
__device__ __forceinline__ uint32_t block_excl_scan(const uint32_t* cnt, uint32_t* excl, uint32_t nbins,
                                                    uint32_t* wsum) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  constexpr int per = kFineBins / kPT;  // 16 bins per thread
  const uint32_t b0 = threadIdx.x * per;
  uint32_t loc[per];
  uint32_t t = 0;
#pragma unroll
  for (int k = 0; k < per; ++k) {
    loc[k] = b0 + k < nbins ? cnt[b0 + k] : 0u;
    t += loc[k];
  }
  uint32_t incl = t;
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t o = __shfl_up_sync(GFULL, incl, d);
    if (lane >= d) incl += o;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  uint32_t pre = 0, tot = 0;
  for (int k = 0; k < kPT / 32; ++k) {
    pre += k < w ? wsum[k] : 0u;
    tot += wsum[k];
  }
  pre += incl - t;
#pragma unroll
  for (int k = 0; k < per; ++k) {
    if (b0 + k < nbins) excl[b0 + k] = pre;
    pre += loc[k];
  }
  __syncthreads();
  return tot;
}

// pass 1 needs only kCoarse bins; two tile buffers: the next tile's keys land
// (cp.async) while the current one is ranked, staged and written
struct CoarseSmem {
  uint32_t cnt[kCoarse];
  uint32_t excl[kCoarse];
  ull base[kCoarse];
  ull buf[2][kPTile];   // [cur]: this tile's keys, then its staged order; [cur ^ 1]: the next tile
  uint16_t sd[kPTile];
  uint32_t wsum[kPT / 32];
};

// this thread's share of tile t0's keys -> dst (8-byte cp.async, zero-filled past n)
__device__ __forceinline__ void tile_prefetch(ull* dst, const ull* __restrict__ keys, ull t0, ull n) {
#pragma unroll
  for (int u = 0; u < kPPer; ++u) {
    const uint32_t j = u * kPT + threadIdx.x;
    const ull i = t0 + j;
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst + j);
    const ull* src = keys + (i < n ? i : 0);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(i < n ? 8 : 0)
                 : "memory");
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
struct PartSmem {
  uint32_t cnt[kFineBins];
  uint32_t excl[kFineBins];
  ull base[kFineBins];
  ull stage[kFTile];
  uint16_t sd[kFTile];  // pass 2: the staged key's destination
  uint32_t wsum[kPT / 32];
};

// pass 1: tiles of 4096 keys -> coarse buckets (persistent, double-buffered)
__global__ void __launch_bounds__(kPT, 2) seg_coarse_kernel(const ull* __restrict__ keys, ull n, KeyLayout kl,
                                                         const uint16_t* __restrict__ cb, uint32_t ncoarse,
                                                         ull* __restrict__ ccur, ull* __restrict__ tmp) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CoarseSmem& sm = *reinterpret_cast<CoarseSmem*>(smem_raw);
  const int lane = threadIdx.x & 31;
  unsigned lt;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
  const ull stride = (ull)gridDim.x * kPTile;
  ull t0 = (ull)blockIdx.x * kPTile;
  for (uint32_t i = threadIdx.x; i < ncoarse; i += kPT) sm.cnt[i] = 0;
  if (t0 < n) tile_prefetch(sm.buf[0], keys, t0, n);
  int cur = 0;
  for (; t0 < n; t0 += stride) {
    if (t0 + stride < n) tile_prefetch(sm.buf[cur ^ 1], keys, t0 + stride, n);
    else asm volatile("cp.async.commit_group;\n" ::: "memory");
    asm volatile("cp.async.wait_group 1;\n" ::: "memory");  // this tile's keys (own copies) landed
    __syncthreads();                                          // everyone's
    ull k[kPPer];
    uint32_t b[kPPer], r[kPPer];
#pragma unroll
    for (int u = 0; u < kPPer; ++u) {
      const ull i = t0 + (ull)u * kPT + threadIdx.x;
      k[u] = sm.buf[cur][u * kPT + threadIdx.x];
      b[u] = i < n ? (uint32_t)cb[key_g(k[u], kl) / kGroup] : 0xFFFFFFFFu;
    }
    // rank within the bucket: one shared atomic per key (the order within a
    // bucket is free; with ~1024 buckets a warp's keys rarely share one, so a
    // match_any aggregation costs more than it saves)
#pragma unroll
    for (int u = 0; u < kPPer; ++u) r[u] = b[u] != 0xFFFFFFFFu ? atomicAdd(&sm.cnt[b[u]], 1u) : 0u;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < ncoarse; i += kPT)
      if (sm.cnt[i]) sm.base[i] = atomicAdd(&ccur[i], (ull)sm.cnt[i]);
    const uint32_t tot = block_excl_scan(sm.cnt, sm.excl, ncoarse, sm.wsum);
    ull* const stage = sm.buf[cur];  // every thread has its keys in registers by now
#pragma unroll
    for (int u = 0; u < kPPer; ++u)
      if (b[u] != 0xFFFFFFFFu) {
        const uint32_t q = sm.excl[b[u]] + r[u];
        stage[q] = k[u];
        sm.sd[q] = (uint16_t)b[u];
      }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < tot; i += kPT) {
      const uint32_t bb = sm.sd[i];
      tmp[sm.base[bb] + (i - sm.excl[bb])] = stage[i];
    }
    for (uint32_t i = threadIdx.x; i < ncoarse; i += kPT) sm.cnt[i] = 0;
    __syncthreads();  // stage read out, counters clear: buf[cur] takes the tile after next
    cur ^= 1;
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

// tiles of every coarse bucket (tpre[b] = first tile of bucket b) and the
// sentinels of the bucket tables; one block
__global__ void seg_tiles_kernel(const ull* __restrict__ tot, uint32_t ncoarse, ull* __restrict__ cstart,
                                 ull* __restrict__ cinfo, ull* __restrict__ ccur, ull* __restrict__ tpre,
                                 ull nsec) {
  __shared__ ull carry;
  __shared__ ull wsum[kSegWarps];
  if (threadIdx.x == 0) carry = 0;
  (void)nsec;
  (void)cinfo;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (uint32_t b0 = 0; b0 < ncoarse; b0 += kSegThreads) {
    const uint32_t b = b0 + threadIdx.x;
    ull v = 0;
    if (b < ncoarse) {
      v = (cstart[b + 1] - cstart[b] + kFTile - 1) / kFTile;
      ccur[b] = cstart[b];
    }
    ull incl = v;
    for (int d = 1; d < 32; d <<= 1) {
      const ull o = __shfl_up_sync(GFULL, incl, d);
      if (lane >= d) incl += o;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    ull pre = carry;
    for (int k = 0; k < w; ++k) pre += wsum[k];
    if (b < ncoarse) tpre[b] = pre + incl - v;
    __syncthreads();
    if (threadIdx.x == kSegThreads - 1) carry = pre + incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) tpre[ncoarse] = carry;
}

// tbk[t] = the coarse bucket of pass-2 tile t (one thread per bucket)
__global__ void seg_tilemap_kernel(const ull* __restrict__ tpre, uint32_t ncoarse, uint32_t* __restrict__ tbk) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= ncoarse) return;
  for (ull t = tpre[b]; t < tpre[b + 1]; ++t) tbk[t] = b;
}

// pass 2: tile t of coarse bucket b -> its chunks (out) and big sectors (big)
__global__ void __launch_bounds__(kPT, 3) seg_fine_kernel(const ull* __restrict__ tmp, KeyLayout kl,
                                                       uint32_t ncoarse, const ull* __restrict__ cstart,
                                                       const ull* __restrict__ cinfo, const ull* __restrict__ tpre,
                                                       const uint32_t* __restrict__ tbk,
                                                       const uint32_t* __restrict__ dst, ull* __restrict__ cur,
                                                       ull* __restrict__ bcur, ull* __restrict__ out,
                                                       ull* __restrict__ big) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PartSmem& sm = *reinterpret_cast<PartSmem*>(smem_raw);
  const int lane = threadIdx.x & 31;
  unsigned lt;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
  const ull t = blockIdx.x;
  if (t >= tpre[ncoarse]) return;
  const uint32_t b = tbk[t];  // bucket b: tpre[b] <= t < tpre[b + 1]
  const ull k0 = cstart[b] + (t - tpre[b]) * kFTile;
  const ull k1 = k0 + kFTile < cstart[b + 1] ? k0 + kFTile : cstart[b + 1];
  const ull nl0 = cinfo[3 * b], nl1 = cinfo[3 * b + 3];
  const ull bs0 = cinfo[3 * b + 1], bs1 = cinfo[3 * b + 4];
  // the bucket's chunks lie in [chunk_of(nl0, g0), chunk_of(nl1, g1)] (monotone)
  const ull c_lo = chunk_of(nl0, cinfo[3 * b + 2]);
  const uint32_t nbn = nl1 > nl0 ? (uint32_t)(chunk_of(nl1, cinfo[3 * b + 5]) - c_lo + 1) : 0u;  // chunk bins
  const uint32_t nbins = nbn + (uint32_t)(bs1 - bs0);
  ull k[kFPer];
  uint32_t d[kFPer];  // destination, ~0 = none; below kFineBins bins: | rank << 16
#pragma unroll
  for (int u = 0; u < kFPer; ++u) {
    const ull i = k0 + (ull)u * kPT + threadIdx.x;
    k[u] = i < k1 ? tmp[i] : 0ull;
  }
#pragma unroll
  for (int u = 0; u < kFPer; ++u) {
    const ull i = k0 + (ull)u * kPT + threadIdx.x;
    uint32_t dd = 0xFFFFFFFFu;
    if (i < k1) {
      const uint32_t x = dst[key_g(k[u], kl)];
      dd = (x & 0x80000000u) ? nbn + ((x & 0x7FFFFFFFu) - (uint32_t)bs0) : x - (uint32_t)c_lo;
    }
    d[u] = dd;
  }
  if (nbins > (uint32_t)kFineBins) {
    // too many destinations for one tile's histogram: per-key cursor atomics
    // (warp-aggregated), written directly
#pragma unroll
    for (int u = 0; u < kFPer; ++u) {
      const unsigned peers = __match_any_sync(GFULL, d[u]);
      const int ldr = __ffs(peers) - 1;
      ull p0 = 0;
      if (d[u] != 0xFFFFFFFFu && lane == ldr) {
        ull* c = d[u] < nbn ? &cur[c_lo + d[u]] : &bcur[bs0 + d[u] - nbn];
        p0 = atomicAdd(c, (ull)__popc(peers));
      }
      const ull pos = __shfl_sync(GFULL, p0, ldr) + __popc(peers & lt);
      if (d[u] != 0xFFFFFFFFu) (d[u] < nbn ? out : big)[pos] = k[u];
    }
    return;
  }
  for (uint32_t i = threadIdx.x; i < nbins; i += kPT) sm.cnt[i] = 0;
  __syncthreads();
  // rank within the destination: one shared atomic per key (order within a
  // destination is free)
#pragma unroll
  for (int u = 0; u < kFPer; ++u)
    if (d[u] != 0xFFFFFFFFu) d[u] |= atomicAdd(&sm.cnt[d[u]], 1u) << 16;
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < nbins; i += kPT)
    if (sm.cnt[i]) sm.base[i] = atomicAdd(i < nbn ? &cur[c_lo + i] : &bcur[bs0 + i - nbn], (ull)sm.cnt[i]);
  const uint32_t tot = block_excl_scan(sm.cnt, sm.excl, nbins, sm.wsum);
  // stage in destination order (with each key's destination), then write runs
#pragma unroll
  for (int u = 0; u < kFPer; ++u)
    if (d[u] != 0xFFFFFFFFu) {
      const uint32_t dd = d[u] & 0xFFFFu;
      const uint32_t q = sm.excl[dd] + (d[u] >> 16);
      sm.stage[q] = k[u];
      sm.sd[q] = (uint16_t)dd;
    }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < tot; i += kPT) {
    const uint32_t dd = sm.sd[i];
    (dd < nbn ? out : big)[sm.base[dd] + (i - sm.excl[dd])] = sm.stage[i];
  }
}

// ---- 4. per-chunk shared-memory dedup + count --------------------------------------
// chunk c owns the sectors g with chunk_of(off[g], g) = c: at most kChunkSec of
// them, whose segments start in one kSegCap window; their keys lie in
// [cko[c], cko[c + 1]) and number < 2*kSegCap (every normal sector has fewer
// than kSegCap keys).

// per-block (pc, level) bin table in shared memory: open addressing on the
// bin id; a full table falls back to the global atomic
constexpr int kPcBins = 512;
constexpr uint32_t kFewPcs = 8;  // direct bins + byte masks up to this many pc ids (8 x 2 x 33 <= 2 kPcBins)
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
static_assert(kHWin >= kChunkSec, "every chunk counts its sectors in shared memory");
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

// the same insert reporting what it added (the pass-(a) counts form as the
// entries do): 0x100 | m for a new entry (*slot), else the mask bits the
// entry gained (exact: bits only accumulate; the OR returns the old mask)
__device__ __forceinline__ uint32_t hset_or_new(ull* tab, ull id, uint32_t m, uint32_t& slot) {
  const uint32_t hx = (uint32_t)((id * 0x9E3779B97F4A7C15ull) >> 32);
  uint32_t h = __umulhi(hx, (uint32_t)kHSlots);
  const ull v = (id << 8) | m;
  for (;;) {
    ull cur = tab[h];
    if (cur == kHEmpty) {
      cur = atomicCAS(&tab[h], kHEmpty, v);
      if (cur == kHEmpty) {
        slot = h;
        return 0x100u | m;
      }
    }
    if ((cur >> 8) == id) {
      if (((uint32_t)cur & m) == m) return 0u;
      return m & ~atomicOr(reinterpret_cast<uint32_t*>(&tab[h]), m);
    }
    h = h + 1 == (uint32_t)kHSlots ? 0u : h + 1;
  }
}

// the chunk's keys, held in registers for both insert passes: thread t holds
// keys t, t + 256, ... (a chunk holds < 2 kSegCap = 16 x 256 keys)
constexpr int kKPT = 2 * kSegCap / kSegThreads;
__device__ __forceinline__ void chunk_load(ull (&kk)[kKPT], const ull* __restrict__ seg, ull k0, uint32_t nk) {
#pragma unroll
  for (int j = 0; j < kKPT; ++j) {
    const uint32_t i = j * kSegThreads + threadIdx.x;
    kk[j] = i < nk ? __ldcs(&seg[k0 + i]) : 0ull;  // (streamed: read once)
  }
}
// one insert pass over the chunk's keys kk: id = (sector - s0) << A | (key >> B)
// & M, mask = the key's low 8 bits; new slots appended to `list`
__device__ __forceinline__ void chunk_insert_regs(ull* tab, uint16_t* list, uint32_t* nlist, const ull (&kk)[kKPT],
                                                  uint32_t nk, ull s0, const KeyLayout& kl, uint32_t filter,
                                                  uint32_t A, uint32_t B, ull M) {
  const int lane = threadIdx.x & 31;
  unsigned lt;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
  const uint32_t jmax = (nk + kSegThreads - 1) / kSegThreads;  // (uniform)
#pragma unroll
  for (int j = 0; j < kKPT; ++j) {
    if ((uint32_t)j >= jmax) break;
    const ull k = kk[j];
    bool ok = j * kSegThreads + threadIdx.x < nk;
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

// pass (a) over the chunk's keys kk: id = (sector - s0) << LW | (launch, warp),
// OR-ed masks; each insert adds what it created to the sector's counters in
// cnt ([sector][5]: words (2b, 2b+1) as u16 pairs, the sector count): a new
// entry is a new warp of the sector, each bit it gains a new (warp, word)
// (P:328 flush); with pcm (<= 8 pc ids), each key also ORs its word mask into
// the (sector, pc) byte pcm[2 (sector - s0) + pc / 4] byte pc % 4; returns the
// entries this thread created
__device__ __forceinline__ uint32_t chunk_insert_count(ull* tab, const ull (&kk)[kKPT], uint32_t nk, ull s0,
                                                       const KeyLayout& kl, uint32_t filter, uint32_t LW, uint32_t RS,
                                                       ull M, uint32_t* cnt, uint32_t* pcm) {
  const uint32_t jmax = (nk + kSegThreads - 1) / kSegThreads;  // (uniform)
  uint32_t fresh = 0;  // entries this thread created
#pragma unroll
  for (int j = 0; j < kKPT; ++j) {
    if ((uint32_t)j >= jmax) break;
    const ull k = kk[j];
    bool ok = j * kSegThreads + threadIdx.x < nk;
    if (filter != THERMO_ALL_LAUNCHES) ok = ok && key_launch(k, kl) == filter;
    uint32_t slot = 0, r = 0;
    if (ok) {
      const uint32_t gl = (uint32_t)(key_g(k, kl) - s0);
      r = hset_or_new(tab, ((ull)gl << LW) | ((k >> RS) & M), (uint32_t)k & 0xFFu, slot);
      uint32_t* cg = cnt + gl * 5;
      if (r & 0x100u) atomicAdd(&cg[4], 1u);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t add = ((r >> (2 * q)) & 1u) | (((r >> (2 * q + 1)) & 1u) << 16);
        if (add) atomicAdd(&cg[q], add);
      }
      if (pcm) {  // <= 8 pc ids: the key's word mask into its (sector, pc) byte
        const uint32_t pcid = (uint32_t)(k >> 8) & 7u;
        atomicOr(&pcm[2 * gl + (pcid >> 2)], ((uint32_t)k & 0xFFu) << (8 * (pcid & 3u)));
      }
    }
    fresh += (r >> 8) & 1u;
  }
  return fresh;
}

// chunk c owns the sectors [cs0[c], cs0[c + 1]) (at most kChunkSec); their
// keys are seg[cko[c], cko[c + 1]), fewer than 2 kSegCap.  (a) distinct
// (sector, launch, warp) with OR-ed masks in a shared-memory hash set ->
// sector count = #entries, word b's count = #entries with bit b (the popcount
// flush of P:328, G6), summed per sector in shared memory and stored as the
// chunk's rows; (b) distinct (sector, pc id) with OR-ed masks -> per-pc level
// histograms (G11)
// Persistent: a CTA takes chunks from a counter until none are left, so the
// table and the per-pc bin table are initialised once per CTA (between chunks
// only the slots a pass used are cleared) and the bins are flushed once.
__global__ void __launch_bounds__(kSegThreads, 3) seg_chunk_kernel(const ull* __restrict__ seg, const ull* __restrict__ cko,
                                                               ull nsec, KeyLayout kl, uint32_t filter,
                                                               uint32_t* __restrict__ wc, uint32_t* __restrict__ sc,
                                                               const uint32_t* __restrict__ site_of,
                                                               ull* __restrict__ pc_hist, DevCounters* ctr,
                                                               const ull* __restrict__ cs0, ull nchunks,
                                                               ull* __restrict__ chunk_ctr, uint32_t few_pcs) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ull* tab = reinterpret_cast<ull*>(smem_raw);                    // [kHSlots]
  uint32_t* cnt = reinterpret_cast<uint32_t*>(tab + kHSlots);     // [kHWin][5]: words (2b, 2b+1) as u16 pairs, sector
  uint32_t* tbin = cnt + kHWin * 5;                               // [kPcBins]
  uint32_t* tcnt = tbin + kPcBins;                                // [kPcBins]
  uint16_t* list = reinterpret_cast<uint16_t*>(tcnt + kPcBins);   // [2 kSegCap] occupied slots
  __shared__ uint32_t s_n[2];
  __shared__ ull s_c;
  const int lane = threadIdx.x & 31;
  const uint32_t LW = kl.L + kl.W, RS = 8 + kl.P;
  const ull lwmask = (1ull << LW) - 1;
  const ull pmask = (1ull << kl.P) - 1;
  for (int i = threadIdx.x; i < kHSlots; i += kSegThreads) tab[i] = kHEmpty;
  // few_pcs (at most kFewPcs pc ids in the job): the bin region is a direct
  // [pc][word | sector][level] table, and a chunk collects its (sector, pc)
  // word masks as bytes (one shared OR per key) instead of the second set
  uint32_t* const dir = tbin;  // [kFewPcs * 2 * kLevels] <= 2 kPcBins
  if (few_pcs) {
    for (int i = threadIdx.x; i < 2 * kPcBins; i += kSegThreads) dir[i] = 0;
  } else {
    for (int i = threadIdx.x; i < kPcBins; i += kSegThreads) { tbin[i] = 0xFFFFFFFFu; tcnt[i] = 0; }
  }
  ull distinct = 0, distinct_pc = 0;  // this thread's running totals (distinct_pc: thread 0's on the hashed path)
  for (;;) {
    __syncthreads();  // the previous chunk is done with s_c, s_n and its table slots
    if (threadIdx.x == 0) {
      s_c = atomicAdd(chunk_ctr, 1ull);
      s_n[0] = s_n[1] = 0;
    }
    __syncthreads();
    const ull c = s_c;
    if (c >= nchunks) break;
    const ull s0 = cs0[c], s1 = cs0[c + 1];
    if (s0 >= s1) continue;  // (uniform)
    const ull k0 = cko[c];
    const uint32_t nk = (uint32_t)(cko[c + 1] - k0);  // < 2 kSegCap
    const ull win = s1 - s0;  // <= kChunkSec <= kHWin: the chunk's rows are counted in shared memory
    // few pc ids: the (sector, pc) byte masks live in the list region (the
    // hashed per-pc pass's, unused then)
    uint32_t* const pcm = (few_pcs && pc_hist) ? reinterpret_cast<uint32_t*>(list) : nullptr;
    for (uint32_t i = threadIdx.x; i < (uint32_t)win * 5; i += kSegThreads) cnt[i] = 0;
    if (pcm)
      for (uint32_t i = threadIdx.x; i < 2 * (uint32_t)win; i += kSegThreads) pcm[i] = 0;
    __syncthreads();
    // ---- (a) distinct (sector, launch, warp) ----
    ull kk[kKPT];
    chunk_load(kk, seg, k0, nk);
    distinct += chunk_insert_count(tab, kk, nk, s0, kl, filter, LW, RS, lwmask, cnt, pcm);
    __syncthreads();
    // the chunk owns its sectors: plain stores of every row, zeros included
    // (the build does not clear the dense rows on this path; a big sector's
    // row is zero here and its passes add to it afterwards)
    for (uint32_t j = threadIdx.x; j < (uint32_t)win; j += kSegThreads) {
      const uint32_t* cg = cnt + j * 5;
      const ull g = s0 + j;
      sc[g] = cg[4];
      uint4 lo, hi;
      lo.x = cg[0] & 0xFFFFu; lo.y = cg[0] >> 16; lo.z = cg[1] & 0xFFFFu; lo.w = cg[1] >> 16;
      hi.x = cg[2] & 0xFFFFu; hi.y = cg[2] >> 16; hi.z = cg[3] & 0xFFFFu; hi.w = cg[3] >> 16;
      reinterpret_cast<uint4*>(wc + 8 * g)[0] = lo;
      reinterpret_cast<uint4*>(wc + 8 * g)[1] = hi;
    }
    for (uint32_t i = threadIdx.x; i < (uint32_t)kHSlots; i += kSegThreads) tab[i] = kHEmpty;  // (a)'s entries
    if (!pc_hist) continue;  // (uniform)
    if (pcm) {
      // ---- (b') the chunk's (sector, pc) word-mask bytes (filled by pass (a))
      // binned at the sectors' and words' levels ----
      uint32_t npcs = 0;
      for (uint32_t j = threadIdx.x; j < (uint32_t)win; j += kSegThreads) {
        const uint32_t p0 = pcm[2 * j], p1 = pcm[2 * j + 1];
        if ((p0 | p1) == 0) continue;
        const uint32_t* cg = cnt + j * 5;
        const uint32_t ls = level_of_g(cg[4]);
        uint32_t lw[8];
#pragma unroll
        for (int b = 0; b < 8; ++b) lw[b] = level_of_g((cg[b >> 1] >> (16 * (b & 1))) & 0xFFFFu);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint32_t m = ((q < 4 ? p0 : p1) >> (8 * (q & 3))) & 0xFFu;
          if (!m) continue;
          ++npcs;
          atomicAdd(&dir[(q * 2 + 1) * kLevels + ls], 1u);
#pragma unroll
          for (int b = 0; b < 8; ++b)
            if ((m >> b) & 1u) atomicAdd(&dir[(q * 2) * kLevels + lw[b]], 1u);
        }
      }
      distinct_pc += npcs;  // (per thread: summed below)
      continue;
    }
    __syncthreads();
    // ---- (b) distinct (sector, pc id) -> per-pc level histograms ----
    chunk_insert_regs(tab, list, &s_n[1], kk, nk, s0, kl, filter, kl.P, 8, pmask);
    __syncthreads();
    const uint32_t npc = s_n[1];
    for (uint32_t base = threadIdx.x & ~31u; base < npc; base += kSegThreads) {
      const uint32_t i = base + lane;
      const bool head = i < npc;
      const ull v = head ? tab[list[i]] : kHEmpty;
      const uint32_t gl = (uint32_t)(v >> (8 + kl.P));
      const uint32_t pcid = (uint32_t)((v >> 8) & pmask);
      const uint32_t m = (uint32_t)v & 0xFFu;
      const uint32_t* cg = cnt + (head ? gl : 0u) * 5;
      {
        const uint32_t scv = head ? cg[4] : 0u;
        const uint32_t bin = head ? (pcid * 2 + 1) * kLevels + level_of_g(scv) : 0xFFFFFFFFu;
        const unsigned mm = __match_any_sync(GFULL, bin);
        if (head && (__ffs(mm) - 1) == lane) bin_add(tbin, tcnt, pc_hist, bin, __popc(mm));
      }
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const bool hb = head && ((m >> b) & 1u);
        const uint32_t wv = hb ? ((cg[b >> 1] >> (16 * (b & 1))) & 0xFFFFu) : 0u;
        const uint32_t bin = hb ? (pcid * 2) * kLevels + level_of_g(wv) : 0xFFFFFFFFu;
        const unsigned mm = __match_any_sync(GFULL, bin);
        if (hb && (__ffs(mm) - 1) == lane) bin_add(tbin, tcnt, pc_hist, bin, __popc(mm));
      }
    }
    if (threadIdx.x == 0) distinct_pc += npc;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < npc; i += kSegThreads) tab[list[i]] = kHEmpty;
  }
  for (int d = 16; d; d >>= 1) distinct += __shfl_xor_sync(GFULL, distinct, d);
  if (lane == 0 && distinct) atomicAdd(&ctr->distinct_pairs, distinct);
  for (int d = 16; d; d >>= 1) distinct_pc += __shfl_xor_sync(GFULL, distinct_pc, d);
  if (lane == 0 && distinct_pc) atomicAdd(&ctr->distinct_pc, distinct_pc);
  if (pc_hist) {
    __syncthreads();
    if (few_pcs) {
      for (int i = threadIdx.x; i < 2 * kPcBins; i += kSegThreads)
        if (dir[i]) atomicAdd(&pc_hist[i], (ull)dir[i]);
    } else {
      for (int i = threadIdx.x; i < kPcBins; i += kSegThreads)
        if (tbin[i] != 0xFFFFFFFFu && tcnt[i]) atomicAdd(&pc_hist[tbin[i]], (ull)tcnt[i]);
    }
  }
  (void)site_of;
  (void)nsec;
}

// ---- 5. big sectors (>= kSegCap keys: the hot x sectors of SpMV hold up to
// 620 k keys of 138 k warps) ---------------------------------------------------
// A big sector's keys big[boff[i], boff[i + 1]) are split into P_i = ceil(K_i /
// kBigFill) passes by a hash of the (launch, warp) id, so that every distinct
// warp lands in exactly one pass; one CTA per (sector, pass) collects its
// warps' OR-ed masks in a shared-memory hash set and adds its entries to the
// sector's counts (P:325 flush: sector count = distinct warps, word count =
// those with the bit).  A second kernel, once the counts are final, collects
// the sector's distinct pc ids (split the same way) and bins them at the
// sector's and words' levels (G11).  All CTAs run in parallel: a CTA re-reads
// its sector's keys (L2-resident) instead of one CTA looping over P passes.
constexpr int kBigSlots = 4096;          // 32 KB table
constexpr uint32_t kBigFill = 3072;      // keys per pass (load <= 3/4)
__device__ __forceinline__ uint32_t big_pass_of(ull id, uint32_t P) {
  return P <= 1 ? 0u : __umulhi((uint32_t)((id * 0xD6E8FEB86659FD93ull) >> 32), P);
}
// table of tb = log2(slots) bits, sized to the pass's keys (a CTA clears and
// scans only what it uses)
// returns false when the table is full (the pass drew far more distinct ids
// than its share: reported as a hash overflow, never a wrong count)
__device__ __forceinline__ bool big_or(ull* tab, uint32_t tb, ull id, uint32_t m) {
  const uint32_t tmask = (1u << tb) - 1;
  uint32_t h = (uint32_t)((id * 0x9E3779B97F4A7C15ull) >> (64 - tb));
  const ull v = (id << 8) | m;
  for (uint32_t probe = 0; probe <= tmask; ++probe) {
    ull cur = tab[h];
    if (cur == kHEmpty) {
      cur = atomicCAS(&tab[h], kHEmpty, v);
      if (cur == kHEmpty) return true;
    }
    if ((cur >> 8) == id) {
      if (((uint32_t)cur & m) != m) atomicOr(reinterpret_cast<uint32_t*>(&tab[h]), m);
      return true;
    }
    h = (h + 1) & tmask;
  }
  return false;
}
// f(key) over big[b0, b0 + K), kBigUnroll loads in flight per thread (the
// keys are re-read from L2 by each pass of the sector: latency-bound with one
// load at a time)
constexpr int kBigUnroll = 4;
template <typename F>
__device__ __forceinline__ void big_for_keys(const ull* __restrict__ big, ull b0, uint32_t K, F f) {
  for (uint32_t base = 0; base < K; base += kSegThreads * kBigUnroll) {
    ull kk[kBigUnroll];
#pragma unroll
    for (int u = 0; u < kBigUnroll; ++u) {
      const uint32_t j = base + u * kSegThreads + threadIdx.x;
      kk[u] = j < K ? big[b0 + j] : 0ull;
    }
#pragma unroll
    for (int u = 0; u < kBigUnroll; ++u)
      if (base + u * kSegThreads + threadIdx.x < K) f(kk[u]);
  }
}
// f(key) over the keys of big[b0, b0 + K) that keep(key) selects: a pass of
// a P-pass sector keeps ~1/P of what it reads, so each warp first compacts its
// selected keys into its own 64-key buffer and inserts them 32 at a time with
// every lane busy (filtering in place leaves most lanes idle in the insert)
constexpr int kBigWBuf = 64;
template <typename Keep, typename F>
__device__ __forceinline__ void big_for_kept(const ull* __restrict__ big, ull b0, uint32_t K, ull* wbuf, Keep keep,
                                             F f) {
  const int lane = threadIdx.x & 31;
  unsigned lt;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
  uint32_t wn = 0;  // keys in the warp's buffer (uniform, < 32 between appends)
  const uint32_t K32 = (K + 31) & ~31u;  // whole warps iterate (inactive lanes keep nothing)
  for (uint32_t base = 0; base < K32; base += kSegThreads * kBigUnroll) {
    ull kk[kBigUnroll];
#pragma unroll
    for (int u = 0; u < kBigUnroll; ++u) {
      const uint32_t j = base + u * kSegThreads + threadIdx.x;
      kk[u] = j < K ? big[b0 + j] : 0ull;
    }
#pragma unroll
    for (int u = 0; u < kBigUnroll; ++u) {
      const bool ok = base + u * kSegThreads + threadIdx.x < K && keep(kk[u]);
      const unsigned b = __ballot_sync(GFULL, ok);
      if (ok) wbuf[wn + __popc(b & lt)] = kk[u];
      wn += __popc(b);
      if (wn >= 32) {  // (uniform)
        __syncwarp();
        const ull k = wbuf[lane];
        const ull k2 = wbuf[32 + lane];
        __syncwarp();
        if ((uint32_t)lane < wn - 32) wbuf[lane] = k2;
        wn -= 32;
        __syncwarp();
        f(k);
      }
    }
  }
  __syncwarp();
  if ((uint32_t)lane < wn) f(wbuf[lane]);
}
__device__ __forceinline__ uint32_t big_table_bits(uint32_t keys_per_pass) {
  uint32_t tb = 8;
  while ((1u << tb) * 3u < keys_per_pass * 4u && (1u << tb) < (uint32_t)kBigSlots) ++tb;
  return tb;
}

// passes of every big sector: pre[i] = first CTA of sector i (pre[n] = total);
// kind 0: main-key passes ceil(K / fill), kind 1: pc passes ceil(min(K, npc) / fill)
constexpr int kPlanT = 1024;  // seg_big_plan_kernel threads: each scans a contiguous run of big sectors
__global__ void __launch_bounds__(kPlanT) seg_big_plan_kernel(const ull* __restrict__ boff, const ull* __restrict__ tot,
                                                              ull npc, ull* __restrict__ pre_main,
                                                              ull* __restrict__ pre_pc) {
  __shared__ ull ws[2][kPlanT / 32];
  const ull nbs = tot[1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const ull per = (nbs + kPlanT - 1) / kPlanT;
  const ull i0 = (ull)threadIdx.x * per, i1 = i0 + per < nbs ? i0 + per : nbs;
  auto passes = [&](ull i, ull& v0, ull& v1) {
    const ull K = (i + 1 < nbs ? boff[i + 1] : tot[2]) - boff[i];
    v0 = (K + kBigFill - 1) / kBigFill;
    const ull kp = K < npc ? K : npc;
    // one-pass sectors bin their pc ids in the main kernel (counts final there)
    v1 = v0 == 1 ? 0 : (kp + kBigFill - 1) / kBigFill;
  };
  ull t0 = 0, t1 = 0;
  for (ull i = i0; i < i1; ++i) {
    ull v0, v1;
    passes(i, v0, v1);
    t0 += v0;
    t1 += v1;
  }
  ull c0 = t0, c1 = t1;  // inclusive warp scans
  for (int d = 1; d < 32; d <<= 1) {
    const ull a0 = __shfl_up_sync(GFULL, c0, d), a1 = __shfl_up_sync(GFULL, c1, d);
    if (lane >= d) { c0 += a0; c1 += a1; }
  }
  if (lane == 31) { ws[0][w] = c0; ws[1][w] = c1; }
  __syncthreads();
  ull p0 = c0 - t0, p1 = c1 - t1, all0 = 0, all1 = 0;
  for (int k = 0; k < kPlanT / 32; ++k) {
    if (k < w) { p0 += ws[0][k]; p1 += ws[1][k]; }
    all0 += ws[0][k];
    all1 += ws[1][k];
  }
  for (ull i = i0; i < i1; ++i) {
    ull v0, v1;
    passes(i, v0, v1);
    pre_main[i] = p0;
    pre_pc[i] = p1;
    p0 += v0;
    p1 += v1;
  }
  if (threadIdx.x == 0) { pre_main[nbs] = all0; pre_pc[nbs] = all1; }
}

// CTA t -> (big sector i, pass p): pre[i] <= t < pre[i + 1]
__device__ __forceinline__ bool big_cta(const ull* pre, ull nbs, ull t, ull& i, uint32_t& p, uint32_t& P) {
  if (t >= pre[nbs]) return false;
  ull lo = 0, hi = nbs;
  while (hi - lo > 1) {
    const ull mid = (lo + hi) >> 1;
    if (pre[mid] <= t) lo = mid; else hi = mid;
  }
  i = lo;
  p = (uint32_t)(t - pre[lo]);
  P = (uint32_t)(pre[lo + 1] - pre[lo]);
  return true;
}

__global__ void __launch_bounds__(kSegThreads) seg_big_kernel(const ull* __restrict__ big,
                                                             const ull* __restrict__ boff,
                                                             const ull* __restrict__ bg, const ull* __restrict__ tot,
                                                             const ull* __restrict__ pre, KeyLayout kl,
                                                             uint32_t filter, uint32_t* __restrict__ wc,
                                                             uint32_t* __restrict__ sc,
                                                             const uint32_t* __restrict__ site_of,
                                                             ull* __restrict__ pc_hist, DevCounters* ctr,
                                                             uint32_t few_pcs, uint32_t* __restrict__ bpcm) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ull* tab = reinterpret_cast<ull*>(smem_raw);  // [kBigSlots], then [warps][kBigWBuf] compaction buffers
  __shared__ uint32_t s_cnt[9];
  __shared__ uint32_t s_pcm[2];  // few_pcs: the pass's (pc, word) bytes (pc q: byte q)
  const ull nbs = tot[1];
  ull i;
  uint32_t p, P;
  if (!big_cta(pre, nbs, blockIdx.x, i, p, P)) return;
  const ull g = bg[i];
  const ull b0 = boff[i], b1 = (i + 1 < nbs) ? boff[i + 1] : tot[2];
  const uint32_t K = (uint32_t)(b1 - b0);
  const uint32_t LW = kl.L + kl.W, RS = 8 + kl.P;
  const ull lwmask = (1ull << LW) - 1;
  if (threadIdx.x < 9) s_cnt[threadIdx.x] = 0;
  if (threadIdx.x < 2) s_pcm[threadIdx.x] = 0;
  const uint32_t tb = big_table_bits((K + P - 1) / P + 64);
  // few_pcs: each key ORs its word mask into its pc's byte of a register
  // (pc ids < 8), so the per-pc facts need no second pass over the keys
  ull pm = 0;
  const int T = 1 << tb;
  for (int j = threadIdx.x; j < T; j += kSegThreads) tab[j] = kHEmpty;
  __syncthreads();
  auto insert = [&](ull k) {
    if (!big_or(tab, tb, (k >> RS) & lwmask, (uint32_t)k & 0xFFu)) atomicAdd(&ctr->hash_fail, 1ull);
    if (few_pcs) pm |= (ull)((uint32_t)k & 0xFFu) << (8 * ((uint32_t)(k >> 8) & 7u));
  };
  if (P == 1) {
    big_for_keys(big, b0, K, [&](ull k) {
      if (filter != THERMO_ALL_LAUNCHES && key_launch(k, kl) != filter) return;
      insert(k);
    });
  } else {
    big_for_kept(
        big, b0, K, tab + kBigSlots + (threadIdx.x >> 5) * kBigWBuf,
        [&](ull k) {
          return (filter == THERMO_ALL_LAUNCHES || key_launch(k, kl) == filter) &&
                 big_pass_of((k >> RS) & lwmask, P) == p;
        },
        insert);
  }
  if (few_pcs) {
    for (int d = 16; d; d >>= 1) pm |= __shfl_xor_sync(GFULL, pm, d);
    if ((threadIdx.x & 31) == 0 && pm) {
      atomicOr(&s_pcm[0], (uint32_t)pm);
      atomicOr(&s_pcm[1], (uint32_t)(pm >> 32));
    }
  }
  __syncthreads();
  uint32_t cw[8] = {0, 0, 0, 0, 0, 0, 0, 0}, cs = 0;
  for (int j = threadIdx.x; j < T; j += kSegThreads) {
    const ull v = tab[j];
    if (v == kHEmpty) continue;
    ++cs;
#pragma unroll
    for (int b = 0; b < 8; ++b) cw[b] += ((uint32_t)v >> b) & 1u;
  }
  for (int d = 16; d; d >>= 1) {
    cs += __shfl_xor_sync(GFULL, cs, d);
#pragma unroll
    for (int b = 0; b < 8; ++b) cw[b] += __shfl_xor_sync(GFULL, cw[b], d);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&s_cnt[8], cs);
#pragma unroll
    for (int b = 0; b < 8; ++b) atomicAdd(&s_cnt[b], cw[b]);
  }
  __syncthreads();
  if (threadIdx.x < 9 && s_cnt[threadIdx.x]) {
    // several passes of one sector add up (the dense arrays start at 0)
    atomicAdd(threadIdx.x == 8 ? &sc[g] : &wc[8 * g + threadIdx.x], s_cnt[threadIdx.x]);
    if (threadIdx.x == 8) atomicAdd(&ctr->distinct_pairs, (ull)s_cnt[8]);
  }
  if (few_pcs) {
    // the (pc, word) bytes: binned here for a one-pass sector (its counts are
    // final), OR-ed into the sector's slot for several passes (binned by
    // seg_big_pcbin_kernel once every pass has added its counts)
    if (P != 1) {
      if (threadIdx.x < 2 && s_pcm[threadIdx.x]) atomicOr(&bpcm[2 * i + threadIdx.x], s_pcm[threadIdx.x]);
      return;
    }
    if (threadIdx.x < 8) {
      const uint32_t q = threadIdx.x, m = (s_pcm[q >> 2] >> (8 * (q & 3))) & 0xFFu;
      if (m) {
        atomicAdd(&pc_hist[(q * 2 + 1) * kLevels + level_of_g(s_cnt[8])], 1ull);
        for (uint32_t r = m; r; r &= r - 1)
          atomicAdd(&pc_hist[(q * 2) * kLevels + level_of_g(s_cnt[__ffs(r) - 1])], 1ull);
        atomicAdd(&ctr->distinct_pc, 1ull);
      }
    }
    return;
  }
  if (P != 1 || !pc_hist || !kl.P) return;
  // ---- one-pass sector: its counts are final here, so its distinct pc ids
  // (at most K <= kBigFill) are binned at once (G11) ----
  const ull pmask = (1ull << kl.P) - 1;
  const uint32_t scnt = s_cnt[8];
  __syncthreads();
  for (int j = threadIdx.x; j < T; j += kSegThreads) tab[j] = kHEmpty;
  __syncthreads();
  big_for_keys(big, b0, K, [&](ull k) {
    const ull id = (k >> 8) & pmask;
    if (filter != THERMO_ALL_LAUNCHES && (site_of[id] >> 20) != filter) return;
    if (!big_or(tab, tb, id, (uint32_t)k & 0xFFu)) atomicAdd(&ctr->hash_fail, 1ull);
  });
  __syncthreads();
  uint32_t npc = 0;
  for (int j = threadIdx.x; j < T; j += kSegThreads) {
    const ull v = tab[j];
    if (v == kHEmpty) continue;
    ++npc;
    const uint32_t pcid = (uint32_t)(v >> 8);
    atomicAdd(&pc_hist[(pcid * 2 + 1) * kLevels + level_of_g(scnt)], 1ull);
    for (uint32_t m = (uint32_t)v & 0xFFu; m; m &= m - 1)
      atomicAdd(&pc_hist[(pcid * 2) * kLevels + level_of_g(s_cnt[__ffs(m) - 1])], 1ull);
  }
  for (int d = 16; d; d >>= 1) npc += __shfl_xor_sync(GFULL, npc, d);
  if ((threadIdx.x & 31) == 0 && npc) atomicAdd(&ctr->distinct_pc, (ull)npc);
}

__global__ void __launch_bounds__(kSegThreads) seg_big_pc_kernel(const ull* __restrict__ big,
                                                                const ull* __restrict__ boff,
                                                                const ull* __restrict__ bg,
                                                                const ull* __restrict__ tot,
                                                                const ull* __restrict__ pre, KeyLayout kl,
                                                                uint32_t filter, const uint32_t* __restrict__ wc,
                                                                const uint32_t* __restrict__ sc,
                                                                const uint32_t* __restrict__ site_of,
                                                                ull* __restrict__ pc_hist, DevCounters* ctr) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ull* tab = reinterpret_cast<ull*>(smem_raw);  // [kBigSlots], then [warps][kBigWBuf] compaction buffers
  const ull nbs = tot[1];
  ull i;
  uint32_t p, P;
  if (!big_cta(pre, nbs, blockIdx.x, i, p, P)) return;
  const ull g = bg[i];
  const ull b0 = boff[i], b1 = (i + 1 < nbs) ? boff[i + 1] : tot[2];
  const uint32_t K = (uint32_t)(b1 - b0);
  const ull pmask = (1ull << kl.P) - 1;
  const uint32_t kp = K < (1u << kl.P) ? K : (1u << kl.P);
  const uint32_t tb = big_table_bits((kp + P - 1) / P + 64);
  const int T = 1 << tb;
  for (int j = threadIdx.x; j < T; j += kSegThreads) tab[j] = kHEmpty;
  __syncthreads();
  if (P == 1) {
    big_for_keys(big, b0, K, [&](ull k) {
      const ull id = (k >> 8) & pmask;
      if (filter != THERMO_ALL_LAUNCHES && (site_of[id] >> 20) != filter) return;
      if (!big_or(tab, tb, id, (uint32_t)k & 0xFFu)) atomicAdd(&ctr->hash_fail, 1ull);
    });
  } else {
    big_for_kept(
        big, b0, K, tab + kBigSlots + (threadIdx.x >> 5) * kBigWBuf,
        [&](ull k) {
          const ull id = (k >> 8) & pmask;
          return (filter == THERMO_ALL_LAUNCHES || (site_of[id] >> 20) == filter) && big_pass_of(id, P) == p;
        },
        [&](ull k) {
          if (!big_or(tab, tb, (k >> 8) & pmask, (uint32_t)k & 0xFFu)) atomicAdd(&ctr->hash_fail, 1ull);
        });
  }
  __syncthreads();
  const uint32_t scnt = sc[g];
  uint32_t npc = 0;
  for (int j = threadIdx.x; j < T; j += kSegThreads) {
    const ull v = tab[j];
    if (v == kHEmpty) continue;
    ++npc;
    const uint32_t pcid = (uint32_t)(v >> 8);
    atomicAdd(&pc_hist[(pcid * 2 + 1) * kLevels + level_of_g(scnt)], 1ull);
    for (uint32_t m = (uint32_t)v & 0xFFu; m; m &= m - 1)
      atomicAdd(&pc_hist[(pcid * 2) * kLevels + level_of_g(wc[8 * g + __ffs(m) - 1])], 1ull);
  }
  for (int d = 16; d; d >>= 1) npc += __shfl_xor_sync(GFULL, npc, d);
  if ((threadIdx.x & 31) == 0 && npc) atomicAdd(&ctr->distinct_pc, (ull)npc);
}

// few_pcs, big sectors of several passes: their (pc, word) bytes against the
// final counts (one thread per big sector)
__global__ void seg_big_pcbin_kernel(const ull* __restrict__ pre, const ull* __restrict__ bg,
                                     const ull* __restrict__ tot, const uint32_t* __restrict__ bpcm,
                                     const uint32_t* __restrict__ wc, const uint32_t* __restrict__ sc,
                                     ull* __restrict__ pc_hist, DevCounters* ctr) {
  const ull i = (ull)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= tot[1] || pre[i + 1] - pre[i] <= 1) return;
  const ull g = bg[i];
  const uint32_t p0 = bpcm[2 * i], p1 = bpcm[2 * i + 1];
  if ((p0 | p1) == 0) return;
  uint32_t w[8];
#pragma unroll
  for (int b = 0; b < 8; ++b) w[b] = wc[8 * g + b];
  const uint32_t ls = level_of_g(sc[g]);
  ull npc = 0;
  for (int q = 0; q < 8; ++q) {
    const uint32_t m = ((q < 4 ? p0 : p1) >> (8 * (q & 3))) & 0xFFu;
    if (!m) continue;
    ++npc;
    atomicAdd(&pc_hist[(q * 2 + 1) * kLevels + ls], 1ull);
    for (uint32_t r = m; r; r &= r - 1) atomicAdd(&pc_hist[(q * 2) * kLevels + level_of_g(w[__ffs(r) - 1])], 1ull);
  }
  atomicAdd(&ctr->distinct_pc, npc);
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
    cudaFree(ws.cnt); cudaFree(ws.cko); cudaFree(ws.cur); cudaFree(ws.bsum); cudaFree(ws.cs0); cudaFree(ws.dst);
    ws.cnt = nullptr; ws.cko = ws.cur = ws.bsum = ws.cs0 = nullptr;
    ws.dst = nullptr;
    ws.cap_sec = 0;
    if ((e = cudaMalloc(&ws.cnt, (nsec + 1) * sizeof(uint32_t)))) return e;
    // chunks: chunk_of(NL, nsec) + 1 <= nsec + nsec / kChunkSec + 1 (NL < kSegCap nsec)
    if ((e = cudaMalloc(&ws.cko, (nsec + nsec / kChunkSec + 3) * sizeof(ull)))) return e;
    if ((e = cudaMalloc(&ws.cur, (nsec + nsec / kChunkSec + 3) * sizeof(ull)))) return e;
    if ((e = cudaMalloc(&ws.cs0, (nsec + nsec / kChunkSec + 3) * sizeof(ull)))) return e;
    if ((e = cudaMalloc(&ws.dst, (nsec + 1) * sizeof(uint32_t)))) return e;
    if ((e = cudaMalloc(&ws.bsum, 3 * ((nsec + kScanBlock) / kScanBlock + 1) * sizeof(ull)))) return e;
    cudaFree(ws.gpre); cudaFree(ws.cb);
    ws.gpre = nullptr; ws.cb = nullptr;
    if ((e = cudaMalloc(&ws.gpre, 3 * ((nsec + kGroup - 1) / kGroup + 1) * sizeof(ull)))) return e;
    if ((e = cudaMalloc(&ws.cb, ((nsec + kGroup - 1) / kGroup + 1) * sizeof(uint16_t)))) return e;
    ws.cap_sec = nsec + 1;
  }
  if (!ws.maxc && (e = cudaMalloc(&ws.maxc, 8 * sizeof(ull)))) return e;  // maxc | totals NL, BS, BK
  if (!ws.cstart) {
    if ((e = cudaMalloc(&ws.cstart, (kCoarse + 1) * sizeof(ull)))) return e;
    if ((e = cudaMalloc(&ws.cinfo, 3 * (kCoarse + 1) * sizeof(ull)))) return e;
    if ((e = cudaMalloc(&ws.ccur, kCoarse * sizeof(ull)))) return e;
    if ((e = cudaMalloc(&ws.tpre, (kCoarse + 1) * sizeof(ull)))) return e;
  }
  return cudaSuccess;
}

cudaError_t segment_prepare(const ull* keys, ull n, KeyLayout kl, ull nsec, SegWorkspace& ws, int num_sms,
                            cudaStream_t s, uint32_t* max_per_sector, ull* n_big, bool counted) {
  cudaError_t e;
  if ((e = segment_reserve(ws, nsec))) return e;
  cudaMemsetAsync(ws.maxc, 0, 8 * sizeof(ull), s);
  if (!counted) {
    cudaMemsetAsync(ws.cnt, 0, (nsec + 1) * sizeof(uint32_t), s);
    if (n) {
      const unsigned grid = (unsigned)std::min<ull>((n + 255) / 256, (ull)num_sms * 16);
      seg_hist_kernel<<<grid, 256, 0, s>>>(keys, n, kl, ws.cnt);
      ws.launches += 1;
    }
  }
  // big-sector tables: their number is known only after the scan; bound it by
  // the sectors holding >= kSegCap of the n keys
  const ull nbig_cap = std::min<ull>(nsec, n / kSegCap) + 2;
  if (ws.big_cap < nbig_cap) {
    cudaFree(ws.bg); cudaFree(ws.boff); cudaFree(ws.bcur); cudaFree(ws.bpre); cudaFree(ws.bpcm);
    ws.bg = ws.boff = ws.bcur = ws.bpre = nullptr;
    ws.bpcm = nullptr;
    ws.big_cap = 0;
    if ((e = cudaMalloc(&ws.bg, nbig_cap * sizeof(ull)))) return e;
    if ((e = cudaMalloc(&ws.boff, nbig_cap * sizeof(ull)))) return e;
    if ((e = cudaMalloc(&ws.bcur, nbig_cap * sizeof(ull)))) return e;
    if ((e = cudaMalloc(&ws.bpre, 2 * nbig_cap * sizeof(ull)))) return e;
    if ((e = cudaMalloc(&ws.bpcm, 2 * nbig_cap * sizeof(uint32_t)))) return e;
    ws.big_cap = nbig_cap;
  }
  const ull ngroups = (nsec + kGroup - 1) / kGroup;
  ws.ncoarse = (uint32_t)std::min<ull>(kCoarse, ngroups);
  ull* tot = reinterpret_cast<ull*>(ws.maxc) + 1;
  const ull nb = (nsec + kScanBlock - 1) / kScanBlock;
  seg_scan_reduce<<<(unsigned)nb, kSegThreads, 0, s>>>(ws.cnt, nsec, ws.bsum, ws.maxc);
  seg_scan_blocks<<<1, kScanBT, 0, s>>>(ws.bsum, nb, tot, nsec, ws.cs0, ws.cko);
  seg_scan_apply<<<(unsigned)nb, kSegThreads, 0, s>>>(ws.cnt, nsec, ws.bsum, ws.cs0, ws.cko, ws.dst, ws.bg, ws.boff,
                                                      ws.gpre, tot + 3);
  seg_groups_kernel<<<(unsigned)((ngroups + 256) / 256), 256, 0, s>>>(ws.gpre, ngroups, tot, ws.ncoarse, ws.cb,
                                                                      ws.cstart, ws.cinfo, nsec);
  seg_tiles_kernel<<<1, kSegThreads, 0, s>>>(tot, ws.ncoarse, ws.cstart, ws.cinfo, ws.ccur, ws.tpre, nsec);
  ws.launches += 5;
  ull hv[5];
  if ((e = cudaMemcpyAsync(hv, ws.maxc, 5 * sizeof(ull), cudaMemcpyDeviceToHost, s))) return e;
  if ((e = cudaStreamSynchronize(s))) return e;
  *max_per_sector = (uint32_t)hv[0];
  *n_big = hv[3];         // keys of big sectors
  ws.n_normal = hv[1];  // keys of normal sectors (the chunks')
  ws.n_chunks = hv[4];
  ws.n_bigsec = hv[2];
  ws.n_big_keys = hv[3];
  if (ws.n_bigsec)  // big-sector cursors start at their segments
    if ((e = cudaMemcpyAsync(ws.bcur, ws.boff, ws.n_bigsec * sizeof(ull), cudaMemcpyDeviceToDevice, s))) return e;
  return cudaSuccess;
}

// phases 3-5: keys -> tmp (coarse buckets) -> out (chunks) / big (big sectors)
// -> dense counts (+ per-pc histograms)
cudaError_t segment_count(const ull* keys, ull n, ull* out, ull* big, KeyLayout kl, ull nsec, uint32_t filter,
                          SegWorkspace& ws, uint32_t* wc, uint32_t* sc, const uint32_t* site_of, ull* pc_hist,
                          ull n_pc, DevCounters* ctr, int num_sms, cudaStream_t s) {
  cudaError_t e;
  if (n && ws.tmp_cap < n) {
    cudaFree(ws.tmp);
    ws.tmp = nullptr;
    ws.tmp_cap = 0;
    if ((e = cudaMalloc(&ws.tmp, (n + n / 8 + 1024) * sizeof(ull)))) return e;
    ws.tmp_cap = n + n / 8 + 1024;
  }
  const size_t psm = sizeof(PartSmem), csm = sizeof(CoarseSmem);
  smem_optin((const void*)seg_coarse_kernel, (int)csm);
  smem_optin((const void*)seg_fine_kernel, (int)psm);
  for (int k = 0; k < 4; ++k) ws.ran[k] = false;
  if (ws.ev[0]) cudaEventRecord(ws.ev[0], s);
  if (n) {
    // chunk cursors start at the chunks' first keys
    const ull nch = ws.n_chunks;
    if (nch && (e = cudaMemcpyAsync(ws.cur, ws.cko, nch * sizeof(ull), cudaMemcpyDeviceToDevice, s))) return e;
    const unsigned g1 = (unsigned)std::min<ull>((n + kPTile - 1) / kPTile, (ull)num_sms * 2);
    seg_coarse_kernel<<<g1, kPT, csm, s>>>(keys, n, kl, ws.cb, ws.ncoarse, ws.ccur, ws.tmp);
    if (ws.ev[1]) cudaEventRecord(ws.ev[1], s);
    const ull g2 = (n + kFTile - 1) / kFTile + ws.ncoarse;  // >= the tiles of all buckets
    if (ws.tbk_cap < g2) {
      cudaFree(ws.tbk);
      ws.tbk = nullptr;
      ws.tbk_cap = 0;
      if ((e = cudaMalloc(&ws.tbk, g2 * sizeof(uint32_t)))) return e;
      ws.tbk_cap = g2;
    }
    seg_tilemap_kernel<<<(ws.ncoarse + 255) / 256, 256, 0, s>>>(ws.tpre, ws.ncoarse, ws.tbk);
    seg_fine_kernel<<<(unsigned)g2, kPT, psm, s>>>(ws.tmp, kl, ws.ncoarse, ws.cstart, ws.cinfo, ws.tpre, ws.tbk, ws.dst,
                                                   ws.cur, ws.bcur, out, big);
    if (ws.ev[2]) cudaEventRecord(ws.ev[2], s);
    ws.launches += 4;
    ws.ran[0] = ws.ran[1] = true;
  }
  const size_t smem = segment_chunk_smem();
  smem_optin((const void*)seg_chunk_kernel, (int)smem);
  const ull chunks = ws.n_chunks;
  if (chunks) {
    if (ws.ev[2] && !n) cudaEventRecord(ws.ev[2], s);
    if (!ws.chunk_ctr && (e = cudaMalloc(&ws.chunk_ctr, sizeof(ull)))) return e;
    cudaMemsetAsync(ws.chunk_ctr, 0, sizeof(ull), s);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, seg_chunk_kernel, kSegThreads, smem);
    const ull grid = std::min<ull>(chunks, (ull)num_sms * (per_sm < 1 ? 1 : per_sm));
    seg_chunk_kernel<<<(unsigned)grid, kSegThreads, smem, s>>>(out, ws.cko, nsec, kl, filter, wc, sc, site_of,
                                                               pc_hist, ctr, ws.cs0, chunks, ws.chunk_ctr,
                                                               pc_hist && n_pc <= kFewPcs ? 1u : 0u);
    ws.launches += 1;
    ws.ran[2] = true;
  }
  if (ws.ev[3]) cudaEventRecord(ws.ev[3], s);
  if (ws.n_bigsec) {
    const ull* tot = reinterpret_cast<ull*>(ws.maxc) + 1;
    const ull npc = pc_hist ? (1ull << kl.P) : 0ull;
    seg_big_plan_kernel<<<1, kPlanT, 0, s>>>(ws.boff, tot, npc, ws.bpre, ws.bpre + ws.big_cap);
    // CTAs: at most one per kBigFill keys plus one per sector
    const ull grid = ws.n_big_keys / kBigFill + ws.n_bigsec + 1;
    const size_t bsm = ((size_t)kBigSlots + kSegWarps * kBigWBuf) * sizeof(ull);
    smem_optin((const void*)seg_big_kernel, (int)bsm);
    smem_optin((const void*)seg_big_pc_kernel, (int)bsm);
    const uint32_t few = pc_hist && kl.P && n_pc <= kFewPcs ? 1u : 0u;
    if (few) cudaMemsetAsync(ws.bpcm, 0, 2 * ws.n_bigsec * sizeof(uint32_t), s);
    seg_big_kernel<<<(unsigned)grid, kSegThreads, bsm, s>>>(big, ws.boff, ws.bg, tot, ws.bpre, kl, filter, wc, sc,
                                                             site_of, pc_hist, ctr, few, ws.bpcm);
    ws.launches += 2;
    if (few) {
      seg_big_pcbin_kernel<<<(unsigned)((ws.n_bigsec + 255) / 256), 256, 0, s>>>(ws.bpre, ws.bg, tot, ws.bpcm, wc, sc,
                                                                                pc_hist, ctr);
      ws.launches += 1;
    } else if (pc_hist && kl.P) {
      seg_big_pc_kernel<<<(unsigned)grid, kSegThreads, bsm, s>>>(big, ws.boff, ws.bg, tot, ws.bpre + ws.big_cap,
                                                                  kl, filter, wc, sc, site_of, pc_hist, ctr);
      ws.launches += 1;
    }
    ws.ran[3] = true;
  }
  if (ws.ev[4]) cudaEventRecord(ws.ev[4], s);
  return cudaGetLastError();
}

}  // namespace thermo
