// decode_fast.cu -- the fast decode kernel (rows a2 + a3): one
// warp instruction ("view") per iteration when every active record of it
// shares warp, pc, launch, space and size (what a collector emits for one
// instruction); any other view is deferred to decode_general_kernel
// (decode.cu), which produces the same keys and counters.
//
// Per view: decode, object resolution through a two-entry
// warp-uniform object cache, word mask (G3/G4), adjacent-lane
// merge, insert of (pc id, sector) -> word mask into the warp's shared-memory
// table (emitted as keys when the source warp changes, P:325's OR being
// idempotent), and the instruction's distinct-sector / span test for the
// misalignment indicator (G24).  Boolean conditions use bitwise
// operators so they compile to predicates rather than branches.
#include "decode_common.cuh"

namespace thermo {

template <int MINB>
__global__ void __launch_bounds__(kDecWarps * 32, MINB) decode_kernel(DecodeArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const Smem sm = smem_setup(smem, a);
  const uint32_t nobj = a.obj.n;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  int steps = 0;
  while ((1u << steps) < nobj) ++steps;
  const uint32_t LW = a.kl.L + a.kl.W, P = a.kl.P, W = a.kl.W;
  const uint32_t max_launches = a.max_launches, max_warps = a.max_warps;
  ull* const gkeys = a.keys;
  ull* const gnk = &a.ctr->n_keys;

  WarpTable tab;
  tab.init(sm.warp + wib * kWarpRegion, lane);
  InstrCache icache;
  icache.init();

  ull n_mapped = 0, n_unmapped = 0;
  uint32_t cur_launch = 0xFFFFFFFFu;
  // warp-uniform object cache: [lo, hi) and sector base (soff - lo/32) of two objects
  ull olo0 = 1, ohi0 = 0, ob0 = 0, olo1 = 1, ohi1 = 0, ob1 = 0;
  int oi0 = -1, oi1 = -1;
  bool last1 = false;                                                // entry 1 used last
  uint32_t ps0 = 0xFFFFFFFFu, pi0 = 0, ps1 = 0xFFFFFFFFu, pi1 = 0;  // site -> pc id cache

  const uint32_t gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;

  for (uint32_t r = gwarp; r < a.n_ranges; r += nwarps) {
    const ull end = a.heads[r + 1];
    ull p = a.heads[r];
    uint4 cur = make_uint4(0, 0, 0, 0);
    if (p + lane < end) cur = ld_stream(&a.recs[p + lane]);
    while (p < end) {
      // ---- view = one warp instruction: records [p, p + len) ----
      const unsigned sb = __ballot_sync(FULL, (cur.y >> 23) & 1u) & ~1u;
      const ull rem = end - p;
      uint32_t len = sb ? (uint32_t)(__ffs(sb) - 1) : 32u;
      len = rem < len ? (uint32_t)rem : len;
      const ull pn = p + len;
      uint4 nxt = make_uint4(0, 0, 0, 0);
      if (pn + lane < end) nxt = ld_stream(&a.recs[pn + lane]);  // next view, in flight during this one

      const bool act = lane < (int)len;
      const uint32_t y0 = __shfl_sync(FULL, cur.y, 0);
      const uint32_t z0 = __shfl_sync(FULL, cur.z, 0), w0 = __shfl_sync(FULL, cur.w, 0);
      const uint32_t l2s = (y0 >> 16) & 7u;
      const uint32_t launch0 = w0 >> 20;
      const bool ok0 = (l2s <= 4) & (((y0 >> 19) & 3u) != 3u) & (((y0 >> 21) & 3u) != 3u) & ((y0 >> 24) == 0) &
                       (launch0 < max_launches) & (z0 < max_warps);
      const uint32_t size = 1u << l2s;
      // uniform instruction, no sector straddle, no 2^48 overflow risk
      const bool odd = act & ((cur.z != z0) | (cur.w != w0) | (((cur.y ^ y0) & 0xFF7F0000u) != 0) |
                              ((cur.x & 31u) + size > 32u) | ((cur.y & 0xFFFFu) == 0xFFFFu));
      if (!ok0 || __ballot_sync(FULL, odd) != 0) {
        if (lane == 0) {  // defer the view to the general kernel
          const ull slot = atomicAdd(&a.ctr->n_deferred, 1ull);
          a.deferred[slot] = (p << 7) | len;
        }
        cur = nxt;
        p = pn;
        continue;
      }
      // ---- object of lane 0's sector: two-entry uniform cache; lanes verify ----
      const ull spc = (ull)((y0 >> 21) & 3u) << 48;
      const ull lo = spc | ((ull)(cur.y & 0xFFFFu) << 32) | cur.x;  // space | byte address
      const ull xs = lo & ~31ull;                                   // sector start
      const ull x0 = __shfl_sync(FULL, xs, 0);
      const bool in0 = (x0 >= olo0) & (x0 < ohi0), in1 = (x0 >= olo1) & (x0 < ohi1);
      if (!(in0 | in1)) {  // uniform miss: replace the entry not used last
        const int o = obj_lookup(sm.lo, sm.hi, nobj, steps, x0);
        const ull nlo = o >= 0 ? sm.lo[o] : 1, nhi = o >= 0 ? sm.hi[o] : 0;
        const ull nb = o >= 0 ? sm.soff[o] - (sm.lo[o] >> 5) : 0;
        if (last1) { olo0 = nlo; ohi0 = nhi; ob0 = nb; oi0 = o; last1 = false; }
        else { olo1 = nlo; ohi1 = nhi; ob1 = nb; oi1 = o; last1 = true; }
      } else {
        last1 = !in0;
      }
      const ull wlo = last1 ? olo1 : olo0;
      ull ohi = last1 ? ohi1 : ohi0, ob = last1 ? ob1 : ob0;
      const int oiw = last1 ? oi1 : oi0;
      bool mapped = (xs >= wlo) & (xs < ohi);
      if (__ballot_sync(FULL, act & !mapped)) {  // lanes outside lane 0's object (rare)
        if (act & !mapped) {
          const int o = obj_lookup(sm.lo, sm.hi, nobj, steps, xs);
          mapped = o >= 0;
          if (mapped) { ohi = sm.hi[o]; ob = sm.soff[o] - (sm.lo[o] >> 5); }
        }
      }
      // ---- word mask, restricted to the object's words (G9) ----
      const uint32_t wa = (cur.x >> 2) & 7u, wb = ((cur.x + size - 1u) >> 2) & 7u;
      const uint32_t ma = act ? ((0xFFu << wa) & (0xFFu >> (7u - wb))) : 0u;
      const ull lim = ohi - xs;
      const uint32_t allow = lim >= 32 ? 0xFFu : ((1u << ((uint32_t)(lim + 3) >> 2)) - 1u);
      const uint32_t fa = (act & mapped) ? (ma & allow) : 0u;
      const uint32_t g = (uint32_t)((xs >> 5) + ob);
      if (launch0 != cur_launch) {
        flush_launch_ctr(a.launch_ctr, cur_launch, n_unmapped, n_mapped);
        cur_launch = launch0;
      }
      n_mapped += __popc(fa);
      n_unmapped += __popc(ma) - __popc(fa);
      // ---- keys: adjacent-lane merge, then the warp's dedup table ----
      bool has = fa != 0;
      uint32_t mk = fa;
      adjacent_merge32(g, mk, has, lane);
      if (__any_sync(FULL, has)) {
        const ull lw = ((ull)launch0 << W) | z0;
        if ((lw != tab.tag) | (tab.count > (uint32_t)kTabFlush)) {
          tab.flush(gkeys, gnk, LW, P, lane);
          tab.tag = lw;
        }
        uint32_t pcid = 0;
        if (a.track_pc) {
          if (w0 == ps0) {
            pcid = pi0;
          } else if (w0 == ps1) {
            pcid = pi1; ps1 = ps0; pi1 = pi0; ps0 = w0; pi0 = pcid;
          } else {
            uint32_t id = 0;
            if (lane == 0) id = pc_lookup(sm.pc, a.pcmap, w0, a.ctr);
            pcid = __shfl_sync(FULL, id, 0);
            ps1 = ps0; pi1 = pi0; ps0 = w0; pi0 = pcid;
          }
          pcid = pcid < a.pcmap.max_pcs ? pcid : 0u;  // overflow is reported at build (ERANGE)
        }
        bool fresh = false;
        if (has) fresh = tab.insert(((ull)pcid << 32) | g, mk);
        tab.count += __popc(__ballot_sync(FULL, fresh));
      }
      // ---- instruction statistics (G24) ----
      const uint32_t fa0 = __shfl_sync(FULL, fa, 0);
      const uint32_t xl0 = __shfl_sync(FULL, cur.x, 0);
      const uint32_t wa0 = (xl0 >> 2) & 7u;
      if ((oiw >= 0) & ((fa0 >> wa0) & 1u)) {  // lane 0's first word is mapped (warp-uniform)
        // offsets from lane 0 (32-bit when the instruction spans < 2 GiB, else the 64-bit path)
        const ull rel64 = lo - __shfl_sync(FULL, lo, 0);
        const uint32_t rel = (uint32_t)rel64;
        const uint32_t prel = __shfl_up_sync(FULL, rel, 1);
        const bool down = act & (lane > 0) & (((rel64 >> 31) != 0) | (rel < prel));
        uint32_t distinct;
        bool mis;
        if (__ballot_sync(FULL, down) == 0) {
          // monotone starts, uniform size: count sector changes; span = rel(last) + size
          const uint32_t s0 = xl0 & 31u;  // lane 0's byte offset in its sector
          const uint32_t sec = (rel + s0) >> 5, psec = (prel + s0) >> 5;
          distinct = __popc(__ballot_sync(FULL, act & ((lane == 0) | (sec != psec))));
          const uint32_t span = __shfl_sync(FULL, rel, len - 1) + size;
          mis = distinct > (span + 31) / 32;
        } else {
          const unsigned m = __match_any_sync(FULL, act ? (lo >> 5) : (0xFFFF000000000000ull | (ull)lane));
          distinct = __popc(__ballot_sync(FULL, act & (__ffs(m) - 1 == lane)));
          const ull mn = warp_min64(act ? lo : ~0ull);
          const ull mx = warp_max64(act ? lo : 0ull) + size - 1;
          mis = distinct > (mx - mn + 1 + 31) / 32;
        }
        icache.add(launch0 * nobj + (uint32_t)oiw + 1u, mis, sm.ikey, sm.ival, a.instr_ctr, lane);
      }
      cur = nxt;
      p = pn;
    }
  }
  tab.flush(gkeys, gnk, LW, P, lane);
  icache.drain(sm.ikey, sm.ival, a.instr_ctr, lane);
  flush_launch_ctr(a.launch_ctr, cur_launch, n_unmapped, n_mapped);
  smem_flush_instr(sm, a.instr_ctr);
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
  const ull want = ((ull)a.n_ranges + kDecWarps - 1) / kDecWarps;
  ull grid = (ull)num_sms * per_sm;
  if (want < grid) grid = want;
  if (grid < 1) grid = 1;
  decode_kernel<MINB><<<(unsigned)grid, kDecWarps * 32, smem, s>>>(a);
}

void launch_decode(const DecodeArgs& a, int num_sms, cudaStream_t s) {
  static int batch = -1;
  if (batch < 0) {
    const char* e = getenv("THERMO_DECODE");
    batch = (e && e[0] == 'b') ? 1 : 0;
  }
  if (batch) {
    launch_decode_batch(a, num_sms, s);
    return;
  }
  const size_t smem = decode_smem(a);
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
