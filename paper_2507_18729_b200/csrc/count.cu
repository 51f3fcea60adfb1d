// count.cu -- rows a4 (hash path), a5 (segmented distinct-warp count and
// word->sector roll-up), a6 (heat-level histograms per object and per PC).
//
// a5 is the paper's flush (§IV-B2: "count the number of 1s in the
// bitmasks"): after dedup every distinct (sector g, launch, warp) tuple appears
// once with the OR of its word masks, so
//     sector_count[g]      = number of distinct tuples of g          (P:325 9th mask)
//     word_count[8g + b]   = number of those tuples with bit b set    (P:325 word masks)
// Levels are bit_width(count) (G10, P:351 legend).  Per-PC rows count
// distinct (launch, pc, word) pairs at the word's level (G11).
#include "thermo_internal.cuh"

namespace thermo {

constexpr unsigned CFULL = 0xFFFFFFFFu;

__device__ __forceinline__ ull mix64(ull x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return x;
}
__device__ __forceinline__ int level_of(uint32_t c) { return 32 - __clz(c); }

// ---- a4 hash path: open addressing, linear probing, slot = prefix<<8 | mask ----
__global__ void hash_insert_kernel(const ull* __restrict__ keys, ull n, ull* __restrict__ table, ull cap_mask,
                                   uint32_t drop_low, DevCounters* ctr) {
  const ull stride = (ull)gridDim.x * blockDim.x;
  for (ull i = (ull)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const ull m = keys[i] & 0xFFull;
    const ull pre = (keys[i] >> 8) >> drop_low;
    const ull key = (pre << 8) | m;
    ull h = mix64(pre) & cap_mask;
    bool done = false;
    for (ull probe = 0; probe <= cap_mask && !done; ++probe) {
      ull cur = table[h];
      if (cur == kEmptyKey) {
        ull old = atomicCAS(&table[h], kEmptyKey, key);
        if (old == kEmptyKey) { done = true; break; }
        cur = old;
      }
      if ((cur >> 8) == pre) {
        if ((cur & m) != m) atomicOr(&table[h], m);
        done = true;
        break;
      }
      h = (h + 1) & cap_mask;
    }
    if (!done) atomicAdd(&ctr->hash_fail, 1ull);
  }
}

void launch_hash_insert(const ull* keys, ull n, ull* table, ull cap_mask, uint32_t drop_low, DevCounters* ctr,
                        int num_sms, cudaStream_t s) {
  if (!n) return;
  unsigned grid = (unsigned)std::min<ull>((n + 255) / 256, (ull)num_sms * 16);
  hash_insert_kernel<<<grid, 256, 0, s>>>(keys, n, table, cap_mask, drop_low, ctr);
}

// pc keys [pcid : P][g : S][mask : 8] from keys [g][launch, warp][pcid][mask]
__global__ void pc_extract_kernel(const ull* __restrict__ keys, ull n, KeyLayout kl, ull* __restrict__ out) {
  const ull stride = (ull)gridDim.x * blockDim.x;
  for (ull i = (ull)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const ull k = keys[i];
    out[i] = ((((ull)key_pcid(k, kl) << kl.S) | key_g(k, kl)) << 8) | (k & 0xFF);
  }
}

void launch_pc_extract(const ull* keys, ull n, KeyLayout kl, ull* pckeys, int num_sms, cudaStream_t s) {
  if (!n) return;
  unsigned grid = (unsigned)std::min<ull>((n + 255) / 256, (ull)num_sms * 16);
  pc_extract_kernel<<<grid, 256, 0, s>>>(keys, n, kl, pckeys);
}

// ---- a5 on sorted keys ------------------------------------------------------
// packed per-sector contribution: field 0 = sector count, fields 1..8 = word
// counts, 6 bits each (a warp adds at most 32 per field)
__device__ __forceinline__ ull pack_contrib(uint32_t m) {
  ull v = 1ull;
#pragma unroll
  for (int b = 0; b < 8; ++b) v |= (ull)((m >> b) & 1u) << (6 * (b + 1));
  return v;
}

__device__ __forceinline__ void flush_contrib(ull v, ull g, uint32_t* wc, uint32_t* sc) {
  uint32_t c0 = (uint32_t)(v & 63);
  if (c0) atomicAdd(&sc[g], c0);
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    uint32_t c = (uint32_t)((v >> (6 * (b + 1))) & 63);
    if (c) atomicAdd(&wc[8 * g + b], c);
  }
}

__global__ void __launch_bounds__(256) count_sorted_kernel(const ull* __restrict__ keys, ull n, KeyLayout kl,
                                                           uint32_t filter, uint32_t* __restrict__ wc,
                                                           uint32_t* __restrict__ sc, DevCounters* ctr) {
  const int lane = threadIdx.x & 31;
  const ull nw = (n + 31) / 32;
  const ull wstride = ((ull)gridDim.x * blockDim.x) >> 5;
  const int RS = 8 + kl.P;  // a run is one (g, launch, warp): the pc id is ignored
  ull distinct = 0;
  for (ull wi = ((ull)blockIdx.x * blockDim.x + threadIdx.x) >> 5; wi < nw; wi += wstride) {
    const ull i = wi * 32 + lane;
    const ull key = i < n ? keys[i] : kEmptyKey;
    const ull pre = key >> RS;
    bool valid = key != kEmptyKey;
    if (filter != THERMO_ALL_LAUNCHES) valid &= key_launch(key, kl) == filter;
    ull prev = __shfl_up_sync(CFULL, pre, 1);
    if (lane == 0) prev = i > 0 && i - 1 < n ? (keys[i - 1] >> RS) : ~0ull;
    const bool head = valid && pre != prev;
    uint32_t m = (uint32_t)(key & 0xFF);
    if (head) {  // OR the run (duplicates are adjacent after the sort)
      for (ull j = i + 1; j < n; ++j) {
        ull kj = keys[j];
        if ((kj >> RS) != pre) break;
        m |= (uint32_t)(kj & 0xFF);
      }
    }
    ull v = head ? pack_contrib(m) : 0ull;
    distinct += head ? 1 : 0;
    const ull g = key == kEmptyKey ? ~0ull : key_g(key, kl);
    // reverse segmented sum over equal g (contiguous after the sort)
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      ull ov = __shfl_down_sync(CFULL, v, d);
      ull og = __shfl_down_sync(CFULL, g, d);
      if (lane + d < 32 && og == g) v += ov;
    }
    const ull pg = __shfl_up_sync(CFULL, g, 1);
    const bool ghead = lane == 0 || pg != g;
    if (ghead && v && key != kEmptyKey) flush_contrib(v, g, wc, sc);
  }
  for (int d = 16; d; d >>= 1) distinct += __shfl_xor_sync(CFULL, distinct, d);
  if (lane == 0 && distinct) atomicAdd(&ctr->distinct_pairs, distinct);
}

void launch_count_sorted(const ull* keys, ull n, KeyLayout kl, uint32_t launch_filter, uint32_t* word_cnt,
                         uint32_t* sector_cnt, DevCounters* ctr, int num_sms, cudaStream_t s) {
  if (!n) return;
  unsigned grid = (unsigned)std::min<ull>((n + 255) / 256, (ull)num_sms * 16);
  count_sorted_kernel<<<grid, 256, 0, s>>>(keys, n, kl, launch_filter, word_cnt, sector_cnt, ctr);
}

// ---- a5 on the hash table -----------------------------------------------------
__global__ void __launch_bounds__(256) count_hash_kernel(const ull* __restrict__ table, ull cap, KeyLayout kl,
                                                         uint32_t filter, uint32_t* __restrict__ wc,
                                                         uint32_t* __restrict__ sc, DevCounters* ctr) {
  const int LW = kl.L + kl.W;
  const ull stride = (ull)gridDim.x * blockDim.x;
  ull distinct = 0;
  for (ull i = (ull)blockIdx.x * blockDim.x + threadIdx.x; i < cap; i += stride) {
    const ull v = table[i];
    if (v == kEmptyKey) continue;
    const ull pre = v >> 8;
    if (filter != THERMO_ALL_LAUNCHES) {
      uint32_t la = kl.L ? (uint32_t)((pre >> kl.W) & ((1ull << kl.L) - 1)) : 0u;
      if (la != filter) continue;
    }
    const ull g = pre >> LW;
    const uint32_t m = (uint32_t)(v & 0xFF);
    ++distinct;
    atomicAdd(&sc[g], 1u);
#pragma unroll
    for (int b = 0; b < 8; ++b)
      if ((m >> b) & 1u) atomicAdd(&wc[8 * g + b], 1u);
  }
  for (int d = 16; d; d >>= 1) distinct += __shfl_xor_sync(CFULL, distinct, d);
  if ((threadIdx.x & 31) == 0 && distinct) atomicAdd(&ctr->distinct_pairs, distinct);
}

void launch_count_hash(const ull* table, ull cap, KeyLayout kl, uint32_t launch_filter, uint32_t* word_cnt,
                       uint32_t* sector_cnt, DevCounters* ctr, int num_sms, cudaStream_t s) {
  unsigned grid = (unsigned)std::min<ull>((cap + 255) / 256, (ull)num_sms * 16);
  count_hash_kernel<<<grid, 256, 0, s>>>(table, cap, kl, launch_filter, word_cnt, sector_cnt, ctr);
}

// ---- a6: per-object level histograms, smem-privatised, warp-aggregated ------
__device__ __forceinline__ uint32_t obj_of_sector(const ull* soff, uint32_t n, ull g) {
  // last o with soff[o] <= g (soff ascending, soff[n] = total)
  uint32_t lo = 0, hi = n;
  while (hi - lo > 1) {
    uint32_t mid = (lo + hi) >> 1;
    if (soff[mid] <= g) lo = mid; else hi = mid;
  }
  return lo;
}

// w: every lane of the call adds w to its bin
__device__ __forceinline__ void agg_add(uint32_t* s_hist, ull* g_hist, bool use_smem, uint32_t bin, bool has,
                                        uint32_t w = 1u) {
  const uint32_t key = has ? bin : 0xFFFFFFFFu;
  const unsigned m = __match_any_sync(CFULL, key);
  const int lane = threadIdx.x & 31;
  if (has && (__ffs(m) - 1) == lane) {
    if (use_smem) atomicAdd(&s_hist[bin], w * (uint32_t)__popc(m));
    else atomicAdd(&g_hist[bin], (ull)w * __popc(m));
  }
}

// a6 per-object histograms over the dense rows, one sector per lane (the 8
// word counts as two 16-byte loads, a warp reads 1 KB contiguous); the
// object is looked up once per warp while its 32 sectors stay inside it.
// sharded mode: lane sector l < n_local is the rank's local index (global
// g = shard_global(l)); one rank: l = g, n_local = total
__global__ void __launch_bounds__(256) object_hist_kernel(const uint32_t* __restrict__ wc,
                                                          const uint32_t* __restrict__ sc, const ull* __restrict__ soff,
                                                          const ull* __restrict__ nwords, uint32_t nobj,
                                                          ull* __restrict__ hist, ull total, ull n_local,
                                                          int use_smem, uint32_t rank, uint32_t nranks) {
  extern __shared__ uint32_t s_hist[];  // [nobj][2][33] when use_smem
  const uint32_t nb = nobj * 2 * kLevels;
  if (use_smem) {
    for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) s_hist[i] = 0;
    __syncthreads();
  }
  const uint32_t lane = threadIdx.x & 31;
  const ull wstride = (ull)gridDim.x * blockDim.x;
  uint32_t o0 = 0;
  ull olo = 1, ohi = 0;  // sectors [olo, ohi) of object o0 (the last one looked up)
  for (ull l0 = ((ull)blockIdx.x * blockDim.x + (threadIdx.x & ~31u)); l0 < n_local; l0 += wstride) {
    // a warp's 32 local sectors lie in one 2048-sector chunk: contiguous globally
    const ull g0 = shard_global(l0, rank, nranks);
    const ull l = l0 + lane;
    const ull g = g0 + lane;
    const bool in = l < n_local && g < total;
    const ull glast = (g0 + 31 < total ? g0 + 31 : total - 1);
    if (g0 >= total) continue;
    // warp-uniform object when the first and last sector of the 32 agree
    if (g0 < olo || g0 >= ohi) {  // (uniform) search only when leaving the object
      o0 = obj_of_sector(soff, nobj, g0);
      olo = soff[o0];
      ohi = soff[o0 + 1];
    }
    const bool uni = glast < ohi;
    const uint32_t o = uni ? o0 : (g < total ? obj_of_sector(soff, nobj, g) : 0u);
    uint4 lo = make_uint4(0, 0, 0, 0), hi = lo;
    uint32_t c = 0;
    if (in) {
      lo = reinterpret_cast<const uint4*>(wc + 8 * l)[0];
      hi = reinterpret_cast<const uint4*>(wc + 8 * l)[1];
      c = sc[l];
    }
    const ull nwo = nwords[o];
    const ull wl0 = in ? (g - soff[o]) * 8 : 0;
    const uint32_t x[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
    // bins aggregated over the warp's lanes (match_any), one atomic per distinct bin
    agg_add(s_hist, hist, use_smem, (o * 2 + 1) * kLevels + (in ? level_of(c) : 0), in);
    // a sector whose 8 words (all the object's) share one level adds 8 to one
    // bin: one aggregation for those lanes instead of eight
    const uint32_t lw0 = level_of(x[0]);
    bool same8 = in && wl0 + 8 <= nwo;
#pragma unroll
    for (int b = 1; b < 8; ++b) same8 = same8 && level_of(x[b]) == lw0;
    agg_add(s_hist, hist, use_smem, (o * 2) * kLevels + (same8 ? lw0 : 0), same8, 8u);
    if (__any_sync(CFULL, in && !same8)) {
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const bool hw = in && !same8 && wl0 + b < nwo;
        agg_add(s_hist, hist, use_smem, (o * 2) * kLevels + (hw ? level_of(x[b]) : 0), hw);
      }
    }
  }
  if (use_smem) {
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x)
      if (s_hist[i]) atomicAdd(&hist[i], (ull)s_hist[i]);
  }
}

void launch_object_hist(const uint32_t* word_cnt, const uint32_t* sector_cnt, ObjTable obj, const ull* obj_nwords,
                        ull* hist, ull total_sectors, ull n_local, uint32_t rank, uint32_t nranks, int num_sms,
                        cudaStream_t s) {
  const uint32_t nb = obj.n * 2 * kLevels;
  const int use_smem = nb * sizeof(uint32_t) <= 96 * 1024;
  size_t smem = use_smem ? nb * sizeof(uint32_t) : 0;
  smem_optin((const void*)object_hist_kernel, 96 * 1024);
  unsigned grid = (unsigned)std::min<ull>((n_local + 255) / 256, (ull)num_sms * 8);
  if (grid < 1) grid = 1;
  object_hist_kernel<<<grid, 256, smem, s>>>(word_cnt, sector_cnt, obj.soff, obj_nwords, obj.n, hist,
                                              total_sectors, n_local, use_smem, rank, nranks);
}

// ---- a6: per-PC histograms ---------------------------------------------------------
// per-block bin table in shared memory (a few hundred hot (pc, level) bins take
// every update; only the table's overflow goes to the global histogram)
constexpr int kPcTab = 1024;
__device__ __forceinline__ void pc_bin_add(uint32_t* tbin, uint32_t* tcnt, ull* g, uint32_t bin, uint32_t v) {
  uint32_t h = (bin * 0x9E3779B1u) >> (32 - 10);
  for (int probe = 0; probe < 16; ++probe) {
    uint32_t cur = tbin[h];
    if (cur == 0xFFFFFFFFu) {
      cur = atomicCAS(&tbin[h], 0xFFFFFFFFu, bin);
      if (cur == 0xFFFFFFFFu) cur = bin;
    }
    if (cur == bin) { atomicAdd(&tcnt[h], v); return; }
    h = (h + 1) & (kPcTab - 1);
  }
  atomicAdd(&g[bin], (ull)v);
}
__device__ __forceinline__ void pc_tab_init(uint32_t* tbin, uint32_t* tcnt) {
  for (int i = threadIdx.x; i < kPcTab; i += blockDim.x) { tbin[i] = 0xFFFFFFFFu; tcnt[i] = 0; }
  __syncthreads();
}
__device__ __forceinline__ void pc_tab_flush(const uint32_t* tbin, const uint32_t* tcnt, ull* g) {
  __syncthreads();
  for (int i = threadIdx.x; i < kPcTab; i += blockDim.x)
    if (tbin[i] != 0xFFFFFFFFu && tcnt[i]) atomicAdd(&g[tbin[i]], (ull)tcnt[i]);
}

__device__ __forceinline__ void pc_contrib(ull pre, uint32_t m, bool head, KeyLayout kl, const uint32_t* site_of,
                                           uint32_t filter, const uint32_t* wc, const uint32_t* sc, ull* pc_hist,
                                           ull& distinct, uint32_t* tbin, uint32_t* tcnt) {
  const ull g = pre & ((1ull << kl.S) - 1);
  const uint32_t pcid = (uint32_t)(pre >> kl.S);
  bool ok = head;
  if (ok && filter != THERMO_ALL_LAUNCHES) ok = (site_of[pcid] >> 20) == filter;
  distinct += ok ? 1 : 0;
  if (!__any_sync(CFULL, ok)) return;  // warp-uniform: nothing to add
  // sector bin then word bins, each aggregated across the warp
  {
    const uint32_t bin = ok ? (pcid * 2 + 1) * kLevels + level_of(sc[g]) : 0xFFFFFFFFu;
    const unsigned mm = __match_any_sync(CFULL, bin);
    if (ok && (__ffs(mm) - 1) == (int)(threadIdx.x & 31)) pc_bin_add(tbin, tcnt, pc_hist, bin, __popc(mm));
  }
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const bool hb = ok && ((m >> b) & 1u);
    const uint32_t bin = hb ? (pcid * 2) * kLevels + level_of(wc[8 * g + b]) : 0xFFFFFFFFu;
    const unsigned mm = __match_any_sync(CFULL, bin);
    if (hb && (__ffs(mm) - 1) == (int)(threadIdx.x & 31)) pc_bin_add(tbin, tcnt, pc_hist, bin, __popc(mm));
  }
}

__global__ void __launch_bounds__(256) pc_hist_sorted_kernel(const ull* __restrict__ keys, ull n, KeyLayout kl,
                                                             const uint32_t* __restrict__ site_of, uint32_t filter,
                                                             const uint32_t* __restrict__ wc,
                                                             const uint32_t* __restrict__ sc,
                                                             ull* __restrict__ pc_hist, DevCounters* ctr) {
  __shared__ uint32_t tbin[kPcTab], tcnt[kPcTab];
  pc_tab_init(tbin, tcnt);
  const int lane = threadIdx.x & 31;
  const ull nw = (n + 31) / 32;
  const ull wstride = ((ull)gridDim.x * blockDim.x) >> 5;
  ull distinct = 0;
  for (ull wi = ((ull)blockIdx.x * blockDim.x + threadIdx.x) >> 5; wi < nw; wi += wstride) {
    const ull i = wi * 32 + lane;
    const ull key = i < n ? keys[i] : kEmptyKey;
    const ull pre = key >> 8;
    ull prev = __shfl_up_sync(CFULL, pre, 1);
    if (lane == 0) prev = i > 0 && i - 1 < n ? (keys[i - 1] >> 8) : ~0ull;
    const bool head = key != kEmptyKey && pre != prev;
    uint32_t m = (uint32_t)(key & 0xFF);
    if (head) {
      for (ull j = i + 1; j < n; ++j) {
        ull kj = keys[j];
        if ((kj >> 8) != pre) break;
        m |= (uint32_t)(kj & 0xFF);
      }
    }
    pc_contrib(pre, m, head, kl, site_of, filter, wc, sc, pc_hist, distinct, tbin, tcnt);
  }
  for (int d = 16; d; d >>= 1) distinct += __shfl_xor_sync(CFULL, distinct, d);
  if (lane == 0 && distinct) atomicAdd(&ctr->distinct_pc, distinct);
  pc_tab_flush(tbin, tcnt, pc_hist);
}

void launch_pc_hist_sorted(const ull* pckeys, ull n, KeyLayout kl, const uint32_t* site_of, uint32_t launch_filter,
                           const uint32_t* word_cnt, const uint32_t* sector_cnt, ull* pc_hist, DevCounters* ctr,
                           int num_sms, cudaStream_t s) {
  if (!n) return;
  unsigned grid = (unsigned)std::min<ull>((n + 255) / 256, (ull)num_sms * 16);
  pc_hist_sorted_kernel<<<grid, 256, 0, s>>>(pckeys, n, kl, site_of, launch_filter, word_cnt, sector_cnt, pc_hist,
                                              ctr);
}

__global__ void __launch_bounds__(256) pc_hist_hash_kernel(const ull* __restrict__ table, ull cap, KeyLayout kl,
                                                           const uint32_t* __restrict__ site_of, uint32_t filter,
                                                           const uint32_t* __restrict__ wc,
                                                           const uint32_t* __restrict__ sc,
                                                           ull* __restrict__ pc_hist, DevCounters* ctr) {
  __shared__ uint32_t tbin[kPcTab], tcnt[kPcTab];
  pc_tab_init(tbin, tcnt);
  const ull stride = (ull)gridDim.x * blockDim.x;
  const ull nthreads = (cap + 255) / 256 * 256;
  ull distinct = 0;
  for (ull i = (ull)blockIdx.x * blockDim.x + threadIdx.x; i < nthreads; i += stride) {
    const ull v = i < cap ? table[i] : kEmptyKey;
    pc_contrib(v >> 8, (uint32_t)(v & 0xFF), v != kEmptyKey, kl, site_of, filter, wc, sc, pc_hist, distinct, tbin,
               tcnt);
  }
  for (int d = 16; d; d >>= 1) distinct += __shfl_xor_sync(CFULL, distinct, d);
  if ((threadIdx.x & 31) == 0 && distinct) atomicAdd(&ctr->distinct_pc, distinct);
  pc_tab_flush(tbin, tcnt, pc_hist);
}

void launch_pc_hist_hash(const ull* table, ull cap, KeyLayout kl, const uint32_t* site_of, uint32_t launch_filter,
                         const uint32_t* word_cnt, const uint32_t* sector_cnt, ull* pc_hist, DevCounters* ctr,
                         int num_sms, cudaStream_t s) {
  unsigned grid = (unsigned)std::min<ull>((cap + 255) / 256, (ull)num_sms * 16);
  pc_hist_hash_kernel<<<grid, 256, 0, s>>>(table, cap, kl, site_of, launch_filter, word_cnt, sector_cnt, pc_hist,
                                            ctr);
}

}  // namespace thermo
