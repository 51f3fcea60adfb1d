// decode.cu -- rows a2 + a3 of the hot path: record decode, word
// expansion, object resolution, (sector, launch, warp, word-mask) key packing
// with warp-level pre-dedup, the (pc, sector, mask) stream, and the
// per-instruction misalignment statistics.
//
// Paper passages: record attributes P:283-292 (§IV-B1); tag/offset
// processing P:323-325 (§IV-B2, G3/G4); "1 << warp_id ... |=" P:325 -- the OR
// is idempotent, so merging identical (sector, warp) tuples anywhere before the
// count is exact (S:292-300 merge = OR); misalignment P:435-446 (Fig. 6),
// instruction grouping G24.
//
// Execution model: a persistent grid; each warp owns contiguous record ranges
// [heads[r], heads[r+1]) that start at explicit instruction heads (found by
// find_heads), and walks them one warp-instruction ("view") at a time: lane l
// handles record p + l of the view, so lane l sees lane l of consecutive
// instructions and a per-lane register cache catches a lane's repeats across
// instructions (e.g. GEMM's A[row][k..k+7] in one sector, Listing 1).
#include <cstdlib>

#include "thermo_internal.cuh"

namespace thermo {

constexpr unsigned FULL = 0xFFFFFFFFu;
constexpr int kDecWarps = 8;            // warps per block
constexpr int kStage = 256;             // staged keys per warp before a flush
constexpr int kFlushAt = kStage - 64;   // a view emits <= 64 keys per stream
constexpr int kCacheMain = 4;           // per-lane LRU cache entries (main keys)
constexpr int kCachePc = 4;             // per-lane LRU cache entries (pc keys)
constexpr int kInstrSlots = 64;         // per-block (launch, object) counter table
constexpr int kPcSlots = 64;            // per-block (site -> pc id) cache
constexpr ull kNoPrefix = ~0ull;

// ---------------------------------------------------------------------------
// find_heads: heads[r] = first explicit instruction head at or after r*range_len
// (record 0 of the call always is one); heads[n_ranges] = n.
// ---------------------------------------------------------------------------
__global__ void find_heads_kernel(const uint4* __restrict__ recs, ull n, ull range_len, uint32_t n_ranges,
                                  ull* __restrict__ heads) {
  const int lane = threadIdx.x & 31;
  const uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r > n_ranges) return;
  if (r == 0) { if (lane == 0) heads[0] = 0; return; }
  if (r == n_ranges) { if (lane == 0) heads[r] = n; return; }
  ull p = (ull)r * range_len;
  ull found = n;
  for (; p < n; p += 32) {
    ull i = p + lane;
    bool st = false;
    if (i < n) st = (__ldg(&recs[i].y) >> 23) & 1u;
    unsigned b = __ballot_sync(FULL, st);
    if (b) { found = p + (__ffs(b) - 1); break; }
  }
  if (lane == 0) heads[r] = found;
}

void launch_find_heads(const uint4* recs, ull n, ull range_len, uint32_t n_ranges, ull* heads, cudaStream_t s) {
  ull threads = ((ull)n_ranges + 1) * 32;
  find_heads_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(recs, n, range_len, n_ranges, heads);
}

// ---------------------------------------------------------------------------
// small device helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

__device__ __forceinline__ ull warp_min64(ull v) {
  for (int d = 16; d; d >>= 1) { ull o = __shfl_xor_sync(FULL, v, d); v = o < v ? o : v; }
  return v;
}
__device__ __forceinline__ ull warp_max64(ull v) {
  for (int d = 16; d; d >>= 1) { ull o = __shfl_xor_sync(FULL, v, d); v = o > v ? o : v; }
  return v;
}

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

// last object with lo <= x, or -1 if x lies in no object
__device__ __forceinline__ int obj_lookup(const ull* s_lo, const ull* s_hi, uint32_t n, int steps, ull x) {
  uint32_t lo = 0, hi = n;
  for (int i = 0; i < steps; ++i) {
    uint32_t mid = (lo + hi) >> 1;
    bool le = s_lo[mid] <= x;
    lo = le ? mid : lo;
    hi = le ? hi : mid;
  }
  return (n > 0 && x >= s_lo[lo] && x < s_hi[lo]) ? (int)lo : -1;
}

// merge equal prefixes held by adjacent lanes: the first lane of each run gets
// the OR of the run's masks, the others drop their key (P:325 OR idempotent)
__device__ __forceinline__ void adjacent_merge(ull& prefix, uint32_t& mask, bool& has, int lane) {
  ull pp = __shfl_up_sync(FULL, prefix, 1);
  bool ph = __shfl_up_sync(FULL, has, 1);
  bool same = lane > 0 && has && ph && pp == prefix;
  unsigned sb = __ballot_sync(FULL, same);
  if (sb == 0) return;
  unsigned hb = __ballot_sync(FULL, has);
  if (sb == (hb & (hb - 1))) {  // every key equals its predecessor: one run
    uint32_t orm = __reduce_or_sync(FULL, has ? mask : 0u);
    if (same) has = false; else if (has) mask = orm;
    return;
  }
  for (int d = 1; d < 32; d <<= 1) {  // reverse segmented OR (Kogge-Stone)
    ull np = __shfl_down_sync(FULL, prefix, d);
    uint32_t nm = __shfl_down_sync(FULL, mask, d);
    bool nh = __shfl_down_sync(FULL, has, d);
    if (lane + d < 32 && nh && has && np == prefix) mask |= nm;
  }
  if (same) has = false;
}

// per-lane LRU cache of (prefix, mask): returns the evicted key (or kEmptyKey)
template <int C>
struct LaneCache {
  ull p[C];
  uint32_t m[C];
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int i = 0; i < C; ++i) { p[i] = kNoPrefix; m[i] = 0; }
  }
  // FIFO replacement (cheaper than LRU; a hit ORs the mask in place)
  __device__ __forceinline__ ull put(ull prefix, uint32_t mask) {
    bool hit = false;
#pragma unroll
    for (int i = 0; i < C; ++i) {
      const bool h = p[i] == prefix;
      m[i] |= h ? mask : 0u;
      hit |= h;
    }
    ull ev = kEmptyKey;
    if (!hit) {
      if (p[C - 1] != kNoPrefix) ev = (p[C - 1] << 8) | m[C - 1];
#pragma unroll
      for (int i = C - 1; i > 0; --i) { p[i] = p[i - 1]; m[i] = m[i - 1]; }
      p[0] = prefix; m[0] = mask;
    }
    return ev;
  }
};

// per-warp staging buffer in shared memory; flushed to global with one atomic
struct Stage {
  ull* s;        // smem [kStage]
  uint32_t cnt;  // warp-uniform
  __device__ __forceinline__ void push(ull key, bool has, ull* g, ull* gcount, int lane) {
    unsigned b = __ballot_sync(FULL, has);
    if (!b) return;
    if (has) s[cnt + __popc(b & lanemask_lt())] = key;
    cnt += __popc(b);
    if (cnt > (uint32_t)kFlushAt) flush(g, gcount, lane);
  }
  __device__ __forceinline__ void flush(ull* g, ull* gcount, int lane) {
    __syncwarp();
    if (cnt == 0) return;
    ull base = 0;
    if (lane == 0) base = atomicAdd(gcount, (ull)cnt);
    base = __shfl_sync(FULL, base, 0);
    for (uint32_t i = lane; i < cnt; i += 32) g[base + i] = s[i];
    __syncwarp();
    cnt = 0;
  }
};

// (launch, pc) -> dense pc id; inserts on first sight (G11)
__device__ uint32_t pc_lookup_global(const PcMap& pm, uint32_t site, DevCounters* ctr) {
  ull key = (ull)site + 1ull;
  uint32_t h = hash32(site) & pm.cap_mask;
  ull* keys = pm.keys;
  for (uint32_t probe = 0; probe <= pm.cap_mask; ++probe) {
    ull cur = *((volatile ull*)&keys[h]);
    if (cur == 0) {
      ull old = atomicCAS(&keys[h], 0ull, key);
      if (old == 0) {
        ull id = atomicAdd(&ctr->pc_count, 1ull);
        uint32_t v;
        if (id >= pm.max_pcs) { atomicAdd(&ctr->pc_overflow, 1ull); v = kPcNone - 1; }
        else { pm.site_of[id] = site; v = (uint32_t)id; }
        __threadfence();
        atomicExch(&pm.vals[h], v);
        return v;
      }
      cur = old;
    }
    if (cur == key) {
      uint32_t v;
      while ((v = *((volatile uint32_t*)&pm.vals[h])) == kPcNone) { }
      return v;
    }
    h = (h + 1) & pm.cap_mask;
  }
  return kPcNone - 1;
}

__device__ __forceinline__ uint32_t pc_lookup(ull* s_pc, const PcMap& pm, uint32_t site, DevCounters* ctr) {
  uint32_t h = hash32(site) & (kPcSlots - 1);
  ull e = *((volatile ull*)&s_pc[h]);
  if ((uint32_t)(e >> 32) == site && (uint32_t)e != kPcNone) return (uint32_t)e;
  uint32_t id = pc_lookup_global(pm, site, ctr);
  s_pc[h] = ((ull)site << 32) | id;
  return id;
}

__device__ __forceinline__ void instr_flush(uint32_t* s_ikey, ull* s_ival, ull* g_ctr, uint32_t key, uint32_t ni,
                                            uint32_t nm) {
  uint32_t h = hash32(key) & (kInstrSlots - 1);
  for (int probe = 0; probe < kInstrSlots; ++probe) {
    uint32_t cur = s_ikey[h];
    if (cur == 0) {
      cur = atomicCAS(&s_ikey[h], 0u, key);
      if (cur == 0) cur = key;
    }
    if (cur == key) {
      atomicAdd(&s_ival[2 * h], (ull)ni);
      if (nm) atomicAdd(&s_ival[2 * h + 1], (ull)nm);
      return;
    }
    h = (h + 1) & (kInstrSlots - 1);
  }
  atomicAdd(&g_ctr[2 * (key - 1)], (ull)ni);
  if (nm) atomicAdd(&g_ctr[2 * (key - 1) + 1], (ull)nm);
}

__device__ __forceinline__ void instr_add(uint32_t* s_ikey, ull* s_ival, ull* g_ctr, uint32_t key, bool mis) {
  uint32_t h = hash32(key) & (kInstrSlots - 1);
  for (int probe = 0; probe < kInstrSlots; ++probe) {
    uint32_t cur = s_ikey[h];
    if (cur == 0) {
      cur = atomicCAS(&s_ikey[h], 0u, key);
      if (cur == 0) cur = key;
    }
    if (cur == key) {
      atomicAdd(&s_ival[2 * h], 1ull);
      if (mis) atomicAdd(&s_ival[2 * h + 1], 1ull);
      return;
    }
    h = (h + 1) & (kInstrSlots - 1);
  }
  atomicAdd(&g_ctr[2 * (key - 1)], 1ull);
  if (mis) atomicAdd(&g_ctr[2 * (key - 1) + 1], 1ull);
}

// per-warp register cache of the (launch, object) misalignment counters; all
// lanes hold identical copies (warp-uniform), lane 0 flushes evictions
struct InstrCache {
  uint32_t k0, k1;
  uint32_t i0, m0, i1, m1;
  __device__ __forceinline__ void init() { k0 = k1 = 0; i0 = m0 = i1 = m1 = 0; }
  __device__ __forceinline__ void add(uint32_t key, bool mis, uint32_t* s_ikey, ull* s_ival, ull* g, int lane) {
    if (key == k0) { ++i0; m0 += mis; return; }
    if (key == k1) { ++i1; m1 += mis; return; }
    if (k1 && lane == 0) instr_flush(s_ikey, s_ival, g, k1, i1, m1);
    k1 = k0; i1 = i0; m1 = m0;
    k0 = key; i0 = 1; m0 = mis;
  }
  __device__ __forceinline__ void drain(uint32_t* s_ikey, ull* s_ival, ull* g, int lane) {
    if (lane == 0) {
      if (k0) instr_flush(s_ikey, s_ival, g, k0, i0, m0);
      if (k1) instr_flush(s_ikey, s_ival, g, k1, i1, m1);
    }
    init();
  }
};

// ---------------------------------------------------------------------------
// the decode kernel
// ---------------------------------------------------------------------------
template <int MINB>
__global__ void __launch_bounds__(kDecWarps * 32, MINB) decode_kernel(DecodeArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t nobj = a.obj.n;
  ull* s_lo = reinterpret_cast<ull*>(smem);
  ull* s_hi = s_lo + nobj;
  ull* s_soff = s_hi + nobj;
  ull* s_stage = s_soff + nobj;                       // [kDecWarps][2][kStage]
  ull* s_ival = s_stage + kDecWarps * 2 * kStage;     // [kInstrSlots][2]
  ull* s_pc = s_ival + 2 * kInstrSlots;               // [kPcSlots]
  uint32_t* s_ikey = reinterpret_cast<uint32_t*>(s_pc + kPcSlots);  // [kInstrSlots]

  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  for (uint32_t i = threadIdx.x; i < nobj; i += blockDim.x) {
    s_lo[i] = a.obj.lo[i];
    s_hi[i] = a.obj.hi[i];
    s_soff[i] = a.obj.soff[i];
  }
  for (int i = threadIdx.x; i < kInstrSlots; i += blockDim.x) {
    s_ikey[i] = 0;
    s_ival[2 * i] = 0;
    s_ival[2 * i + 1] = 0;
  }
  for (int i = threadIdx.x; i < kPcSlots; i += blockDim.x) s_pc[i] = ((ull)0xFFFFFFFFu << 32) | kPcNone;
  __syncthreads();

  int steps = 0;
  while ((1u << steps) < nobj) ++steps;
  const uint32_t LW = a.kl.L + a.kl.W;
  const uint32_t S = a.kl.S;
  const unsigned lt = lanemask_lt();

  Stage st_main{s_stage + (wib * 2 + 0) * kStage, 0};
  Stage st_pc{s_stage + (wib * 2 + 1) * kStage, 0};
  LaneCache<kCacheMain> cmain;
  LaneCache<kCachePc> cpc;
  cmain.init();
  cpc.init();
  InstrCache icache;
  icache.init();

  ull n_invalid = 0, n_oor = 0, n_mapped = 0, n_unmapped = 0;
  uint32_t cur_launch = 0xFFFFFFFFu;   // launch the mapped/unmapped counters belong to
  int hint = 0;                        // per-lane last object (lookup hint)

  const uint32_t gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;

  for (uint32_t r = gwarp; r < a.n_ranges; r += nwarps) {
    const ull end = a.heads[r + 1];
    ull p = a.heads[r];
    uint4 cur = make_uint4(0, 0, 0, 0);
    if (p + lane < end) cur = ld_stream(&a.recs[p + lane]);
    uint4 nx1 = make_uint4(0, 0, 0, 0);  // speculative: the view after a full one
    if (p + 32 + lane < end) nx1 = ld_stream(&a.recs[p + 32 + lane]);
    while (p < end) {
      // ---- view = one warp instruction: records [p, p + len) ----
      const bool st = (cur.y >> 23) & 1u;
      const unsigned sb = __ballot_sync(FULL, st) & ~1u;
      uint32_t len = sb ? (uint32_t)(__ffs(sb) - 1) : 32u;
      if ((ull)len > end - p) len = (uint32_t)(end - p);
      const ull pn = p + len;
      uint4 nxt, nx2 = make_uint4(0, 0, 0, 0);
      if (len == 32) {
        nxt = nx1;
        if (pn + 32 + lane < end) nx2 = ld_stream(&a.recs[pn + 32 + lane]);
      } else {
        nxt = make_uint4(0, 0, 0, 0);
        if (pn + lane < end) nxt = ld_stream(&a.recs[pn + lane]);
        if (pn + 32 + lane < end) nx2 = ld_stream(&a.recs[pn + 32 + lane]);
      }

      const bool act = lane < (int)len;
      const ull af = ((ull)cur.y << 32) | cur.x;
      const uint32_t warp_id = cur.z, site = cur.w;
      const ull addr = af & ((1ull << 48) - 1);
      const uint32_t l2s = (uint32_t)(af >> 48) & 7u, kind = (uint32_t)(af >> 51) & 3u;
      const uint32_t space = (uint32_t)(af >> 53) & 3u, resv = (uint32_t)(af >> 56);
      const ull size = 1ull << (l2s > 4 ? 0 : l2s);
      bool valid = act && l2s <= 4 && kind <= 2 && space <= 2 && resv == 0 && addr + size <= (1ull << 48);
      const uint32_t launch = site >> 20;
      const bool oor = valid && (launch >= a.max_launches || warp_id >= a.max_warps);
      valid = valid && !oor;
      const ull lo = ((ull)space << 48) | addr;
      const ull hi = lo + size - 1;
      const ull sa = lo >> 5, sbk = hi >> 5;
      const bool strad = sbk != sa;

      // ---- fast path: one uniform instruction (same warp, pc, launch, space,
      //      size on every active lane), all valid, no sector straddle ----
      const uint32_t cur_y0 = __shfl_sync(FULL, cur.y, 0);
      const uint32_t warp0 = __shfl_sync(FULL, warp_id, 0), site0 = __shfl_sync(FULL, site, 0);
      const bool odd = act && (!valid || strad || warp_id != warp0 || site != site0 ||
                               ((cur.y ^ cur_y0) & 0x007F0000u) != 0);  // size/kind/space bits
      const unsigned oddb = __ballot_sync(FULL, odd);

      if (oddb == 0) {
        // ======================= FAST PATH =======================
        // object of each lane's sector: hint, else binary search
        const ull x = sa << 5;
        int o = hint;
        if (!(x >= s_lo[o] && x < s_hi[o])) o = obj_lookup(s_lo, s_hi, nobj, steps, x);
        hint = o >= 0 ? o : hint;
        uint32_t fa = 0;
        ull g = 0;
        const uint32_t wa = (uint32_t)(lo >> 2) & 7u, wb = (uint32_t)(hi >> 2) & 7u;
        const uint32_t ma = act ? ((0xFFu << wa) & (0xFFu >> (7 - wb))) : 0u;
        if (o >= 0) {
          const ull lim = s_hi[o] - x;
          const uint32_t allow = lim >= 32 ? 0xFFu : ((1u << ((lim + 3) >> 2)) - 1u);
          fa = ma & allow;
          g = s_soff[o] + (sa - (s_lo[o] >> 5));
        }
        // per-launch mapped / unmapped word counters (launch is uniform here)
        if (launch != cur_launch) {
          if (cur_launch != 0xFFFFFFFFu && (n_mapped | n_unmapped)) {
            atomicAdd(&a.launch_ctr[2 * cur_launch], n_unmapped);
            atomicAdd(&a.launch_ctr[2 * cur_launch + 1], n_mapped);
          }
          cur_launch = launch;
          n_mapped = n_unmapped = 0;
        }
        n_mapped += __popc(fa);
        n_unmapped += __popc(ma) - __popc(fa);
        // main keys: adjacent-lane merge on the sector (lw is uniform)
        const ull lw = ((ull)launch << a.kl.W) | warp_id;
        bool has = fa != 0;
        uint32_t mk = fa;
        {
          const ull pg = __shfl_up_sync(FULL, g, 1);
          const bool ph = __shfl_up_sync(FULL, has, 1);
          const bool same = lane > 0 && has && ph && pg == g;
          const unsigned sbm = __ballot_sync(FULL, same);
          if (sbm) {
            const unsigned hb = __ballot_sync(FULL, has);
            if (sbm == (hb & (hb - 1))) {
              const uint32_t orm = __reduce_or_sync(FULL, has ? mk : 0u);
              if (has) mk = orm;
            } else {
              for (int d = 1; d < 32; d <<= 1) {
                const ull ng = __shfl_down_sync(FULL, g, d);
                const uint32_t nm = __shfl_down_sync(FULL, mk, d);
                const bool nh = __shfl_down_sync(FULL, has, d);
                if (lane + d < 32 && nh && has && ng == g) mk |= nm;
              }
            }
            has = has && !same;
          }
        }
        {
          const ull e1 = has ? cmain.put((g << LW) | lw, mk) : kEmptyKey;
          st_main.push(e1, e1 != kEmptyKey, a.keys, &a.ctr->n_keys, lane);
        }
        // pc keys: same runs, same masks (pc is uniform)
        uint32_t pcid = kPcNone;
        if (a.track_pc && __any_sync(FULL, has)) {
          uint32_t id = 0;
          if (lane == 0) id = pc_lookup(s_pc, a.pcmap, site0, a.ctr);
          pcid = __shfl_sync(FULL, id, 0);
          if (pcid < a.pcmap.max_pcs) {
            const ull e2 = has ? cpc.put(((ull)pcid << S) | g, mk) : kEmptyKey;
            st_pc.push(e2, e2 != kEmptyKey, a.pckeys, &a.ctr->n_pckeys, lane);
          }
        }
        // instruction statistics (G24): monotone starts -> count
        // sector changes; otherwise distinct sectors by match
        {
          const uint32_t fa0 = __shfl_sync(FULL, fa, 0);
          const int o0 = __shfl_sync(FULL, o, 0);
          const uint32_t wa0 = __shfl_sync(FULL, wa, 0);
          if (o0 >= 0 && ((fa0 >> wa0) & 1u)) {
            const ull plo = __shfl_up_sync(FULL, lo, 1);
            const unsigned down = __ballot_sync(FULL, act && lane > 0 && lo < plo);
            uint32_t distinct;
            ull mn, mx;
            if (down == 0) {  // sizes are uniform: first lane has the min, last lane the max
              distinct = __popc(__ballot_sync(FULL, act && (lane == 0 || (plo >> 5) != sa)));
              mn = __shfl_sync(FULL, lo, 0);
              mx = __shfl_sync(FULL, hi, len - 1);
            } else {
              const ull key = act ? sa : (0xFFFF000000000000ull | (ull)lane);
              const unsigned m = __match_any_sync(FULL, key);
              distinct = __popc(__ballot_sync(FULL, act && (__ffs(m) - 1 == lane)));
              mn = warp_min64(act ? lo : ~0ull);
              mx = warp_max64(act ? hi : 0ull);
            }
            const bool mis = distinct > (mx - mn + 1 + 31) / 32;
            icache.add(launch * nobj + (uint32_t)o0 + 1u, mis, s_ikey, s_ival, a.instr_ctr, lane);
          }
        }
      } else {
        // ======================= GENERAL PATH =======================
        n_invalid += (act && !valid && !oor) ? 1 : 0;
        n_oor += oor ? 1 : 0;
        const uint32_t wa = (uint32_t)(lo >> 2) & 7u, wb = (uint32_t)(hi >> 2) & 7u;
        uint32_t ma = (0xFFu << wa) & 0xFFu;
        uint32_t mb = 0;
        if (strad) mb = 0xFFu >> (7 - wb); else ma &= 0xFFu >> (7 - wb);
        int oa = -1, ob = -1;
        ull ga = 0, gb = 0;
        uint32_t fa = 0, fb = 0;
        int first_obj = -1;
        if (valid) {
          oa = obj_lookup(s_lo, s_hi, nobj, steps, sa << 5);
          if (oa >= 0) {
            ull lim = s_hi[oa] - (sa << 5);
            uint32_t allow = lim >= 32 ? 0xFFu : ((1u << ((lim + 3) >> 2)) - 1u);
            fa = ma & allow;
            ga = s_soff[oa] + (sa - (s_lo[oa] >> 5));
            if ((fa >> wa) & 1u) first_obj = oa;
          }
          if (strad) {
            ob = obj_lookup(s_lo, s_hi, nobj, steps, sbk << 5);
            if (ob >= 0) {
              ull lim = s_hi[ob] - (sbk << 5);
              uint32_t allow = lim >= 32 ? 0xFFu : ((1u << ((lim + 3) >> 2)) - 1u);
              fb = mb & allow;
              gb = s_soff[ob] + (sbk - (s_lo[ob] >> 5));
            }
          }
          if (launch != cur_launch) {
            if (cur_launch != 0xFFFFFFFFu && (n_mapped | n_unmapped)) {
              atomicAdd(&a.launch_ctr[2 * cur_launch], n_unmapped);
              atomicAdd(&a.launch_ctr[2 * cur_launch + 1], n_mapped);
            }
            cur_launch = launch;
            n_mapped = n_unmapped = 0;
          }
          const uint32_t mapped = __popc(fa) + __popc(fb);
          n_mapped += mapped;
          n_unmapped += __popc(ma) + __popc(mb) - mapped;
        }
        {
          const ull lw = ((ull)launch << a.kl.W) | warp_id;
          ull pa = fa ? ((ga << LW) | lw) : kNoPrefix;
          ull pb = fb ? ((gb << LW) | lw) : kNoPrefix;
          bool ha = fa != 0, hb = fb != 0;
          uint32_t mA = fa, mB = fb;
          adjacent_merge(pa, mA, ha, lane);
          if (__any_sync(FULL, hb)) adjacent_merge(pb, mB, hb, lane);
          ull e1 = ha ? cmain.put(pa, mA) : kEmptyKey;
          st_main.push(e1, e1 != kEmptyKey, a.keys, &a.ctr->n_keys, lane);
          if (__any_sync(FULL, hb)) {
            ull e2 = hb ? cmain.put(pb, mB) : kEmptyKey;
            st_main.push(e2, e2 != kEmptyKey, a.keys, &a.ctr->n_keys, lane);
          }
        }
        if (a.track_pc) {
          const unsigned vb = __ballot_sync(FULL, fa | fb);
          uint32_t pcid = kPcNone;
          if (vb) {
            const int f = __ffs(vb) - 1;
            const uint32_t sitef = __shfl_sync(FULL, site, f);
            const bool other = (fa | fb) && site != sitef;
            if (__ballot_sync(FULL, other) == 0) {
              uint32_t id = 0;
              if (lane == f) id = pc_lookup(s_pc, a.pcmap, sitef, a.ctr);
              pcid = __shfl_sync(FULL, id, f);
            } else if (fa | fb) {
              pcid = pc_lookup(s_pc, a.pcmap, site, a.ctr);
            }
          }
          const bool okpc = pcid < a.pcmap.max_pcs;
          ull qa = (fa && okpc) ? (((ull)pcid << S) | ga) : kNoPrefix;
          ull qb = (fb && okpc) ? (((ull)pcid << S) | gb) : kNoPrefix;
          bool ha = fa && okpc, hb = fb && okpc;
          uint32_t mA = fa, mB = fb;
          adjacent_merge(qa, mA, ha, lane);
          if (__any_sync(FULL, hb)) adjacent_merge(qb, mB, hb, lane);
          ull e1 = ha ? cpc.put(qa, mA) : kEmptyKey;
          st_pc.push(e1, e1 != kEmptyKey, a.pckeys, &a.ctr->n_pckeys, lane);
          if (__any_sync(FULL, hb)) {
            ull e2 = hb ? cpc.put(qb, mB) : kEmptyKey;
            st_pc.push(e2, e2 != kEmptyKey, a.pckeys, &a.ctr->n_pckeys, lane);
          }
        }
        // instruction statistics, general case
        const unsigned vbm = __ballot_sync(FULL, valid);
        if (vbm) {
          const int f = __ffs(vbm) - 1;
          const int i_obj = __shfl_sync(FULL, first_obj, f);
          const uint32_t i_launch = __shfl_sync(FULL, launch, f);
          if (i_obj >= 0) {
            const ull mn = warp_min64(valid ? lo : ~0ull);
            const ull mx = warp_max64(valid ? hi : 0ull);
            uint32_t distinct;
            const unsigned sbm = __ballot_sync(FULL, valid && strad);
            if (sbm == 0) {
              const ull key = valid ? sa : (0xFFFF000000000000ull | (ull)lane);
              const unsigned m = __match_any_sync(FULL, key);
              distinct = __popc(__ballot_sync(FULL, valid && (__ffs(m) - 1 == lane)));
            } else {
              bool dup_a = false, dup_b = !strad;
              for (int j = 0; j < 32; ++j) {
                const ull aj = __shfl_sync(FULL, sa, j), bj = __shfl_sync(FULL, sbk, j);
                const bool vj = __shfl_sync(FULL, valid, j);
                if (vj && j < lane) {
                  dup_a |= (sa == aj) || (sa == bj);
                  dup_b |= (sbk == aj) || (sbk == bj);
                }
              }
              distinct = __popc(__ballot_sync(FULL, valid && !dup_a)) +
                         __popc(__ballot_sync(FULL, valid && !dup_b));
            }
            const bool mis = distinct > (mx - mn + 1 + 31) / 32;
            icache.add(i_launch * nobj + (uint32_t)i_obj + 1u, mis, s_ikey, s_ival, a.instr_ctr, lane);
          }
        }
      }
      (void)lt;
      cur = nxt;
      nx1 = nx2;
      p = pn;
    }
  }
  // ---- drain the lane caches and staging buffers ----
#pragma unroll
  for (int i = 0; i < kCacheMain; ++i) {
    bool h = cmain.p[i] != kNoPrefix;
    st_main.push((cmain.p[i] << 8) | cmain.m[i], h, a.keys, &a.ctr->n_keys, lane);
  }
  st_main.flush(a.keys, &a.ctr->n_keys, lane);
#pragma unroll
  for (int i = 0; i < kCachePc; ++i) {
    bool h = cpc.p[i] != kNoPrefix;
    st_pc.push((cpc.p[i] << 8) | cpc.m[i], h, a.pckeys, &a.ctr->n_pckeys, lane);
  }
  st_pc.flush(a.pckeys, &a.ctr->n_pckeys, lane);
  icache.drain(s_ikey, s_ival, a.instr_ctr, lane);
  if (cur_launch != 0xFFFFFFFFu && (n_mapped | n_unmapped)) {
    atomicAdd(&a.launch_ctr[2 * cur_launch], n_unmapped);
    atomicAdd(&a.launch_ctr[2 * cur_launch + 1], n_mapped);
  }
  for (int d = 16; d; d >>= 1) {
    n_invalid += __shfl_xor_sync(FULL, n_invalid, d);
    n_oor += __shfl_xor_sync(FULL, n_oor, d);
  }
  if (lane == 0) {
    if (n_invalid) atomicAdd(&a.ctr->invalid, n_invalid);
    if (n_oor) atomicAdd(&a.ctr->out_of_range, n_oor);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kInstrSlots; i += blockDim.x) {
    uint32_t k = s_ikey[i];
    if (k) {
      atomicAdd(&a.instr_ctr[2 * (k - 1)], s_ival[2 * i]);
      if (s_ival[2 * i + 1]) atomicAdd(&a.instr_ctr[2 * (k - 1) + 1], s_ival[2 * i + 1]);
    }
  }
}

template <int MINB>
static void launch_decode_t(const DecodeArgs& a, int num_sms, cudaStream_t s, size_t smem) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(decode_kernel<MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, decode_kernel<MINB>, kDecWarps * 32, smem);
  if (per_sm < 1) per_sm = 1;
  ull want = ((ull)a.n_ranges + kDecWarps - 1) / kDecWarps;
  ull grid = (ull)num_sms * per_sm;
  if (want < grid) grid = want;
  if (grid < 1) grid = 1;
  decode_kernel<MINB><<<(unsigned)grid, kDecWarps * 32, smem, s>>>(a);
}

void launch_decode(const DecodeArgs& a, int num_sms, cudaStream_t s) {
  size_t smem = (size_t)a.obj.n * 3 * sizeof(ull) + (size_t)kDecWarps * 2 * kStage * sizeof(ull) +
                2 * kInstrSlots * sizeof(ull) + kPcSlots * sizeof(ull) + kInstrSlots * sizeof(uint32_t);
  static int minb = -1;
  if (minb < 0) {
    const char* e = getenv("THERMO_DECODE_MINB");
    minb = e ? atoi(e) : 3;
  }
  if (minb == 2) launch_decode_t<2>(a, num_sms, s, smem);
  else if (minb == 4) launch_decode_t<4>(a, num_sms, s, smem);
  else launch_decode_t<3>(a, num_sms, s, smem);
}

}  // namespace thermo
