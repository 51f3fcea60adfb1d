// decode_common.cuh -- pieces shared by the fast and the general decode
// kernels (rows a2 + a3): constants, warp helpers, object lookup,
// the (launch, pc) -> pc id map, per-warp staging / dedup tables and the
// misalignment counter caches.  See decode.cu for the paper passages.
#pragma once
#include <cstdlib>

#include "thermo_internal.cuh"

namespace thermo {

constexpr unsigned FULL = 0xFFFFFFFFu;
constexpr int kDecWarps = 8;            // warps per block
constexpr int kStage = 256;             // staged keys per warp before a flush
constexpr int kFlushAt = kStage - 32;   // flush when the next push may not fit
constexpr int kInstrSlots = 64;         // per-block (launch, object) counter table
constexpr int kPcSlots = 64;            // per-block (site -> pc id) cache
constexpr uint32_t kNoG = 0xFFFFFFFFu;  // empty cache entry (sector ids are < 2^31)


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


// word mask of a sector restricted to the object's words (tail sector of an
// object whose length is not a multiple of 32 bytes, G9)
__device__ __forceinline__ uint32_t allow_mask(ull hi_obj, ull sector_start) {
  const ull lim = hi_obj - sector_start;
  return lim >= 32 ? 0xFFu : ((1u << ((lim + 3) >> 2)) - 1u);
}

// merge equal 64-bit prefixes held by adjacent lanes (general path): the first
// lane of each run gets the OR of the run's masks, the others drop their key
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

// merge equal 64-bit prefixes held by ANY lanes of the view (general path:
// a view of packed short instructions holds one source warp's consecutive
// col[e], col[e+1] loads on non-adjacent lanes): the lowest lane of each
// group gets the OR of the group's masks (through the warp's 32-word scratch),
// the others drop their key
__device__ __forceinline__ void group_merge(ull prefix, uint32_t& mask, bool& has, uint32_t* scr, int lane) {
  const unsigned grp = __match_any_sync(FULL, has ? prefix : ~0ull);
  if (!__any_sync(FULL, has && grp != (1u << lane))) return;
  const int ldr = __ffs(grp) - 1;
  if (has && ldr == lane) scr[lane] = mask;
  __syncwarp();
  if (has && ldr != lane) atomicOr(&scr[ldr], mask);
  __syncwarp();
  if (has && ldr == lane) mask = scr[lane];
  has = has && ldr == lane;
  __syncwarp();
}

// same with the groups given: grp = the lanes holding a key equal to this
// lane's (computed by the caller's match, restricted to lanes that have one)
__device__ __forceinline__ void group_merge_grp(unsigned grp, uint32_t& mask, bool& has, uint32_t* scr, int lane) {
  if (!__any_sync(FULL, has && grp != (1u << lane))) return;
  const int ldr = __ffs(grp) - 1;
  if (has && ldr == lane) scr[lane] = mask;
  __syncwarp();
  if (has && ldr != lane) atomicOr(&scr[ldr], mask);
  __syncwarp();
  if (has && ldr == lane) mask = scr[lane];
  has = has && ldr == lane;
  __syncwarp();
}

// same on 32-bit sector ids (fast path: launch/warp are uniform)
// (g < 2^31 where has: the previous lane's g is shuffled as kNoG when it has no key)
__device__ __forceinline__ void adjacent_merge32(uint32_t g, uint32_t& mask, bool& has, int lane) {
  const uint32_t pg = __shfl_up_sync(FULL, has ? g : kNoG, 1);
  const bool same = lane > 0 && has && pg == g;
  const unsigned sb = __ballot_sync(FULL, same);
  if (sb == 0) return;
  const unsigned hb = __ballot_sync(FULL, has);
  if (sb == (hb & (hb - 1))) {
    const uint32_t orm = __reduce_or_sync(FULL, has ? mask : 0u);
    if (has) mask = orm;
  } else {
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t ng = __shfl_down_sync(FULL, g, d);
      const uint32_t nm = __shfl_down_sync(FULL, mask, d);
      const bool nh = __shfl_down_sync(FULL, has, d);
      if (lane + d < 32 && nh && has && ng == g) mask |= nm;
    }
  }
  has = has && !same;
}



// per-warp staging buffer in shared memory; flushed to global with one atomic
// (seg_cnt != null: also count the flushed keys per sector, the SEGMENT
// path's histogram, so that build does not re-read the keys for it)
struct Stage {
  ull* s;        // smem [kStage]
  uint32_t cnt;  // warp-uniform
  uint32_t* seg_cnt;
  uint32_t gshift;  // key >> gshift = sector id
  __device__ __forceinline__ void flush(ull* g, ull* gcount, int lane) {
    __syncwarp();
    if (cnt == 0) return;
    ull base = 0;
    if (lane == 0) base = atomicAdd(gcount, (ull)cnt);
    base = __shfl_sync(FULL, base, 0);
    for (uint32_t i = lane; i < cnt; i += 32) {
      const ull k = s[i];
      g[base + i] = k;
      if (seg_cnt) atomicAdd(&seg_cnt[k >> gshift], 1u);
    }
    __syncwarp();
    cnt = 0;
  }
};
// push the lanes' keys for which HAS holds; KEY is evaluated only on them
// (needs `lane_lt` = lanemask_lt() and `lane` in scope)
#define STAGE_PUSH(st, HAS, KEY, gbuf, gcnt)                              \
  do {                                                                    \
    const bool has_ = (HAS);                                              \
    const unsigned b_ = __ballot_sync(FULL, has_);                        \
    if (b_) {                                                             \
      if (has_) (st).s[(st).cnt + __popc(b_ & lane_lt)] = (KEY);          \
      (st).cnt += __popc(b_);                                             \
      if ((st).cnt > (uint32_t)kFlushAt) (st).flush((gbuf), (gcnt), lane); \
    }                                                                     \
  } while (0)

// (launch, pc) -> dense pc id; inserts on first sight (G11)
static __device__ uint32_t pc_lookup_global(const PcMap& pm, uint32_t site, DevCounters* ctr) {
  const ull key = (ull)site + 1ull;
  uint32_t h = hash32(site) & pm.cap_mask;
  for (uint32_t probe = 0; probe <= pm.cap_mask; ++probe) {
    ull cur = *((volatile ull*)&pm.keys[h]);
    if (cur == 0) {
      const ull old = atomicCAS(&pm.keys[h], 0ull, key);
      if (old == 0) {
        const ull id = atomicAdd(&ctr->pc_count, 1ull);
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

static __device__ __noinline__ uint32_t pc_lookup(ull* s_pc, const PcMap& pm, uint32_t site, DevCounters* ctr) {
  // the block's warps share the cache: atomic 64-bit read (a CAS that never
  // changes the value) and exchange, so an entry is never seen torn
  const uint32_t h = hash32(site) & (kPcSlots - 1);
  const ull e = atomicCAS(&s_pc[h], 0ull, 0ull);
  if ((uint32_t)(e >> 32) == site && (uint32_t)e != kPcNone) return (uint32_t)e;
  const uint32_t id = pc_lookup_global(pm, site, ctr);
  atomicExch(&s_pc[h], ((ull)site << 32) | id);
  return id;
}

static __device__ __noinline__ void instr_flush(uint32_t* s_ikey, ull* s_ival, ull* g_ctr, uint32_t key, uint32_t ni,
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

// shared-memory layout common to both decode kernels: object table, one
// per-warp key staging buffer, the block's (launch, object) counter table and
// (site -> pc id) cache
constexpr int kRingChunks = 8;          // fast kernel: per-warp record ring of 8 x 32 records (4 KB)
constexpr int kAhead = 6;               // chunks in flight ahead of the current one (cp.async)
constexpr uint32_t kShortView = 8;      // instructions shorter than this are packed for the general kernel
constexpr size_t kWarpCache = 12 * 16;  // four window-cache entries (4 x 2 uint4) + pc-id cache (view kernel: 8 sites in 4 uint4)
constexpr int kDeferBuf = 32;           // fast kernel: deferred-view descriptors staged per warp
// + 32 words of merge scratch (lane decoder)
constexpr size_t kOffScratch = kStage * sizeof(ull) + kRingChunks * 32 * 16 + kWarpCache + kDeferBuf * sizeof(ull);
constexpr size_t kWarpRegion = kOffScratch + 32 * sizeof(uint32_t);
// fixed-size parts first, at compile-time offsets (addresses are immediates,
// nothing to keep in registers); the object table (3 x n u64) last
constexpr size_t kOffIval = 0;                                         // [kInstrSlots][2] u64
constexpr size_t kOffPc = kOffIval + 2 * kInstrSlots * sizeof(ull);    // [kPcSlots] u64
constexpr size_t kOffIkey = kOffPc + kPcSlots * sizeof(ull);           // [kInstrSlots] u32
constexpr size_t kOffWarp = (kOffIkey + kInstrSlots * sizeof(uint32_t) + 15) & ~(size_t)15;  // [kDecWarps]
constexpr int kInstrDirect = 1024;      // (launch, object) counters addressed directly (launch * n_obj + obj)
constexpr size_t kOffIdir = kOffWarp + (size_t)kDecWarps * kWarpRegion;  // [kInstrDirect][2] u32: instrs, misaligned
constexpr size_t kOffObj = kOffIdir + kInstrDirect * sizeof(ull);       // lo, hi, soff [n] u64 each
static_assert(kOffWarp % 16 == 0 && kWarpRegion % 16 == 0, "128-bit ring loads need 16-byte alignment");
struct Smem {
  ull *lo, *hi, *soff, *ival, *pc;
  uint32_t* idir;  // [kInstrDirect][2]: instructions, misaligned ones
  unsigned char* warp;  // [kDecWarps][kWarpRegion]
  uint32_t* ikey;
};
__device__ __forceinline__ Smem smem_setup(unsigned char* smem, const DecodeArgs& a) {
  const uint32_t nobj = a.obj.n;
  Smem m;
  m.ival = reinterpret_cast<ull*>(smem + kOffIval);
  m.pc = reinterpret_cast<ull*>(smem + kOffPc);
  m.ikey = reinterpret_cast<uint32_t*>(smem + kOffIkey);
  m.warp = smem + kOffWarp;
  m.idir = reinterpret_cast<uint32_t*>(smem + kOffIdir);
  m.lo = reinterpret_cast<ull*>(smem + kOffObj);
  m.hi = m.lo + nobj;
  m.soff = m.hi + nobj;
  for (uint32_t i = threadIdx.x; i < nobj; i += blockDim.x) {
    m.lo[i] = a.obj.lo[i];
    m.hi[i] = a.obj.hi[i];
    m.soff[i] = a.obj.soff[i];
  }
  for (int i = threadIdx.x; i < kInstrSlots; i += blockDim.x) {
    m.ikey[i] = 0;
    m.ival[2 * i] = 0;
    m.ival[2 * i + 1] = 0;
  }
  for (int i = threadIdx.x; i < kPcSlots; i += blockDim.x) m.pc[i] = ((ull)0xFFFFFFFFu << 32) | kPcNone;
  for (int i = threadIdx.x; i < 2 * kInstrDirect; i += blockDim.x) m.idir[i] = 0;
  __syncthreads();
  return m;
}

// n warp instructions of (launch, object) key1 - 1 = launch * n_obj + obj, nm
// of them misaligned, from the calling lane: two 32-bit shared atomics in the
// block's direct table (native; a 64-bit shared atomicAdd is a CAS loop on
// sm_100a; a block counts < 2^32 instructions per ingest call), or, for ids
// past the table, the hashed one
__device__ __forceinline__ void instr_add_n(const Smem& m, uint32_t key1, uint32_t n, uint32_t nm, ull* g) {
  if (key1 - 1u < (uint32_t)kInstrDirect) {
    atomicAdd(&m.idir[2 * (key1 - 1u)], n);
    if (nm) atomicAdd(&m.idir[2 * (key1 - 1u) + 1], nm);
  } else {
    instr_flush(m.ikey, m.ival, g, key1, n, nm);
  }
}
// one warp instruction (warp-uniform arguments), counted by lane 0
__device__ __forceinline__ void instr_add(const Smem& m, uint32_t key1, bool mis, ull* g, int lane) {
  if (lane == 0) instr_add_n(m, key1, 1u, mis ? 1u : 0u, g);
}

// deferred views staged per warp in shared memory, appended to the global
// list with one atomic per 32 (a per-view atomic on the one counter serialises
// in L2 when most instructions are short, e.g. SpMV)
struct DeferBuf {
  ull* s;        // smem [kDeferBuf]
  uint32_t n;    // warp-uniform
  __device__ __forceinline__ void flush(ull* g, ull* gcount, int lane) {
    __syncwarp();
    if (n == 0) return;
    ull base = 0;
    if (lane == 0) base = atomicAdd(gcount, (ull)n);
    base = __shfl_sync(FULL, base, 0);
    if ((uint32_t)lane < n) g[base + lane] = s[lane];
    __syncwarp();
    n = 0;
  }
  __device__ __forceinline__ void push(ull e, ull* g, ull* gcount, int lane) {
    if (lane == 0) s[n] = e;
    if (++n == (uint32_t)kDeferBuf) flush(g, gcount, lane);
  }
};

// (launch, object) ids k < 32 counted in registers, lane k holding id k: one
// predicated add per instruction instead of a shared atomic; flushed with
// global atomics when the warp ends (a warp counts < 2^32 instructions per
// ingest call)
struct InstrRegs {
  uint32_t n = 0, m = 0;
  __device__ __forceinline__ void add(const Smem& sm, uint32_t k, bool mis, ull* g, int lane) {
    if (k < 32u) {
      const bool me = (uint32_t)lane == k;
      n += me;
      m += me & mis;
    } else {
      instr_add(sm, k + 1u, mis, g, lane);
    }
  }
  __device__ __forceinline__ void flush(ull* g, int lane) {
    if (n) atomicAdd(&g[2 * lane], (ull)n);
    if (m) atomicAdd(&g[2 * lane + 1], (ull)m);
  }
};

__device__ __forceinline__ void smem_flush_instr(const Smem& m, ull* g) {
  __syncthreads();
  for (int i = threadIdx.x; i < kInstrDirect; i += blockDim.x) {
    const uint32_t n = m.idir[2 * i], nm = m.idir[2 * i + 1];
    if (n) atomicAdd(&g[2 * i], (ull)n);
    if (nm) atomicAdd(&g[2 * i + 1], (ull)nm);
  }
  for (int i = threadIdx.x; i < kInstrSlots; i += blockDim.x) {
    const uint32_t k = m.ikey[i];
    if (k) {
      atomicAdd(&g[2 * (k - 1)], m.ival[2 * i]);
      if (m.ival[2 * i + 1]) atomicAdd(&g[2 * (k - 1) + 1], m.ival[2 * i + 1]);
    }
  }
}

__device__ __forceinline__ void flush_launch_ctr(ull* lc, uint32_t launch, ull& unmapped, ull& mapped) {
  if (launch != 0xFFFFFFFFu && (mapped | unmapped)) {
    atomicAdd(&lc[2 * launch], unmapped);
    atomicAdd(&lc[2 * launch + 1], mapped);
  }
  unmapped = mapped = 0;
}

// ---- window-interval object cache (fast decode kernels) ----
// one interval of a 4 GiB window: [blo, blo + bn) in 32-bit offsets
struct WinEnt {
  uint32_t H;       // window id (space << 16 | addr[32,48)); 0xFFFFFFFF = empty
  uint32_t blo, bn;
  uint32_t sbase;   // sector id of the sector at blo (objects)
  uint32_t tail_s;  // offset of the object's partial last sector, 1 if none
  uint32_t tail_m;  // its allowed words
  int oid;          // object index, -1 for a gap
};

// the interval of window H holding the sector at offset xs (xs % 32 == 0)
__device__ __forceinline__ WinEnt win_lookup(const ull* s_lo, const ull* s_hi, const ull* s_soff, uint32_t n,
                                             int steps, uint32_t H, uint32_t xs) {
  const ull wlo = (ull)H << 32, wend = wlo + (1ull << 32);
  const ull X = wlo | xs;
  int i = -1;  // last object with lo <= X
  {
    uint32_t lo = 0, hi = n;
    for (int k = 0; k < steps; ++k) {
      const uint32_t mid = (lo + hi) >> 1;
      const bool le = s_lo[mid] <= X;
      lo = le ? mid : lo;
      hi = le ? hi : mid;
    }
    if (n > 0 && s_lo[lo] <= X) i = (int)lo;
  }
  WinEnt e;
  e.H = H;
  e.tail_s = 1;
  e.tail_m = 0xFFu;
  ull a, b;
  if (i >= 0 && X < s_hi[i]) {  // a sector of object i
    const ull olo = s_lo[i], ohi = s_hi[i];
    const ull ohi32 = (ohi + 31) & ~31ull;
    a = olo > wlo ? olo : wlo;
    b = ohi32 < wend ? ohi32 : wend;
    e.oid = i;
    e.sbase = (uint32_t)(s_soff[i] + ((a - olo) >> 5));
    const ull ts = ohi & ~31ull;
    if ((ohi & 31) && ts >= wlo && ts < wend) {
      e.tail_s = (uint32_t)(ts - wlo);
      e.tail_m = (1u << (((uint32_t)(ohi & 31) + 3) >> 2)) - 1u;
    }
  } else {  // the gap between objects i and i + 1
    const ull glo = i >= 0 ? ((s_hi[i] + 31) & ~31ull) : 0ull;
    const ull ghi = (uint32_t)(i + 1) < n ? s_lo[i + 1] : ~0ull;
    a = glo > wlo ? glo : wlo;
    b = ghi < wend ? ghi : wend;
    e.oid = -1;
    e.sbase = 0;
  }
  e.blo = (uint32_t)(a - wlo);
  const ull len = b > a ? b - a : 0;
  e.bn = len > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)len;  // xs - blo <= 0xFFFFFFE0 then always passes
  return e;
}

__device__ __forceinline__ bool win_has(const WinEnt& e, uint32_t H, uint32_t xs) {
  return (e.H == H) & (xs - e.blo < e.bn);
}

// full key of a lane entry (pc id << 32 | g) -> mask: [g][launch, warp][pc id][mask]
__device__ __forceinline__ ull entry_key(ull c, uint32_t m, ull tag, uint32_t SH, uint32_t P) {
  return ((((c & 0xFFFFFFFFull) << SH) | (tag << P) | (c >> 32)) << 8) | m;
}

// same with the (launch, warp) field pre-shifted: tag8 = tag << (P + 8), SH8 = SH + 8
__device__ __forceinline__ ull entry_key8(ull c, uint32_t m, ull tag8, uint32_t SH8) {
  return ((c & 0xFFFFFFFFull) << SH8) | tag8 | (((uint32_t)(c >> 32) << 8) | m);
}

size_t decode_smem(const DecodeArgs& a);

}  // namespace thermo
