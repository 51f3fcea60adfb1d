// decode_warp.cu -- rows a2 + a3 for warp-instruction records (SURVEY §8f
// item 4): thermo_warp_record = one warp instruction with its 32 lane
// addresses, the collector's native unit ("32-element array"),
// 272 B per instruction = 8.5 B per lane for full warps instead of 16.
//
// One instruction per warp iteration: lane l loads its address (one coalesced
// 256-byte read per instruction) and the 16-byte header is read once; warp,
// pc, launch, size, kind and space are uniform by construction, so the
// per-lane record path's uniformity tests disappear.  Everything after that is
// the fast per-lane kernel's (decode_fast.cu): window-interval object cache,
// word mask, adjacent-lane merge, two-entry LRU dedup, key stage, misalignment
// statistics (active lanes may be any subset of the warp).  Instructions the
// fast path does not take (invalid header, an address with bits >= 48, lanes
// in different 4 GiB windows, a sector-straddling access) are spilled as the
// per-lane records they stand for and reduced by the per-lane kernels.
#include "decode_common.cuh"

namespace thermo {

constexpr ull kWarpRange = 256;  // instructions per work range (8192 lane records for full warps)

struct WarpDecodeArgs {
  DecodeArgs a;             // object table, key layout, outputs (as the per-lane kernels)
  const uint4* wrec;        // [n_instr][17] 272-byte records
  ull n_instr;
  uint4* spill;             // [32 n_instr] per-lane records of spilled instructions
  ull* spill_ctr;           // [2]: spilled records, lane records seen
};

template <int MINB>
__global__ void __launch_bounds__(kDecWarps * 32, MINB) decode_warp_kernel(WarpDecodeArgs wa) {
  const DecodeArgs& a = wa.a;
  extern __shared__ __align__(16) unsigned char smem[];
  const Smem sm = smem_setup(smem, a);
  const uint32_t nobj = a.obj.n;
  const int lane = threadIdx.x & 31;
  const unsigned lane_lt = lanemask_lt();
  const int wib = threadIdx.x >> 5;
  int steps = 0;
  while ((1u << steps) < nobj) ++steps;
  const uint32_t P = a.kl.P, W = a.kl.W;
  const uint32_t SH = a.kl.L + a.kl.W + P;
  const uint32_t max_launches = a.max_launches, max_warps = a.max_warps;
  ull* const gkeys = a.keys;
  ull* const gnk = &a.ctr->n_keys;
  Stage st{reinterpret_cast<ull*>(sm.warp + wib * kWarpRegion), 0, a.seg_cnt, 8 + a.kl.P + a.kl.L + a.kl.W};

  uint32_t lane_mapped = 0, lane_unmapped = 0;
  uint32_t cur_launch = 0xFFFFFFFFu;
  InstrRegs ir;  // (launch, object) instruction counters for ids < 32
  WinEnt e0, e1;
  e0.H = e1.H = 0xFFFFFFFFu;
  e0.blo = e1.blo = 0;
  e0.bn = e1.bn = 0;
  e0.sbase = e1.sbase = 0;
  e0.tail_s = e1.tail_s = 1;
  e0.tail_m = e1.tail_m = 0xFFu;
  e0.oid = e1.oid = -1;
  bool last1 = false;
  uint32_t ps0 = 0xFFFFFFFFu, pi0 = 0, ps1 = 0xFFFFFFFFu, pi1 = 0;
  ull c0 = 0, c1 = 0;
  uint32_t m0 = 0, m1 = 0;
  ull tag = 0;
  ull lanes_seen = 0;

  const ull gwarp = ((ull)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const ull nwarps = ((ull)gridDim.x * blockDim.x) >> 5;
  // contiguous ranges of instructions per warp: consecutive instructions of a
  // source warp meet the same lanes' LRU entries (the A[row][k..k+7] reuse)
  const ull n_rng = (wa.n_instr + kWarpRange - 1) / kWarpRange;
  for (ull r = gwarp; r < n_rng; r += nwarps) {
  const ull i0 = r * kWarpRange, i1 = i0 + kWarpRange < wa.n_instr ? i0 + kWarpRange : wa.n_instr;
  // software pipeline: the next instruction's header and address are in flight
  uint4 hdr = ld_stream(wa.wrec + i0 * 17);
  ull adr = reinterpret_cast<const ull*>(wa.wrec + i0 * 17 + 1)[lane];
  for (ull i = i0; i < i1; ++i) {
    const uint4 h = hdr;
    const ull addr = adr;
    if (i + 1 < i1) {
      hdr = ld_stream(wa.wrec + (i + 1) * 17);
      adr = reinterpret_cast<const ull*>(wa.wrec + (i + 1) * 17 + 1)[lane];
    }
    const uint32_t z0 = h.x, w0 = h.y, amask = h.z, flags = h.w;
    if (amask == 0) continue;  // no lane executed it: no records
    lanes_seen += __popc(amask);
    if (out_of_scope(a, z0, w0 >> 20)) continue;  // outside the sampled block (G28) or the launch whitelist
    const bool act = (amask >> lane) & 1u;
    const int f = __ffs(amask) - 1;  // the instruction's first record
    const uint32_t l2s = flags & 7u, kind = (flags >> 3) & 3u, space = (flags >> 5) & 3u;
    const uint32_t launch0 = w0 >> 20;
    const bool ok0 = (l2s <= 4) & (kind != 3) & (space != 3) & ((flags >> 7) == 0) & (launch0 < max_launches) &
                     (z0 < max_warps);
    const uint32_t size = 1u << l2s;
    const uint32_t x = (uint32_t)addr;
    const uint32_t hi = (uint32_t)(addr >> 32);  // addr[32, 64)
    const uint32_t hi0 = __shfl_sync(FULL, hi, f);
    const bool odd = act & ((hi != hi0) | ((x & 31u) + size > 32u));
    if (!ok0 || (hi0 >> 16) != 0 || __ballot_sync(FULL, odd) != 0) {
      // spill: the per-lane records of this instruction (first active lane
      // carries instr_start), reduced later by the per-lane kernels
      ull base = 0;
      if (lane == f) base = atomicAdd(&wa.spill_ctr[0], (ull)__popc(amask));
      base = __shfl_sync(FULL, base, f);
      if (act) {
        const ull resv = ((addr >> 48) != 0 || (flags >> 7) != 0) ? 1ull : 0ull;
        const ull af = (addr & ((1ull << 48) - 1)) | ((ull)l2s << 48) | ((ull)kind << 51) | ((ull)space << 53) |
                       ((ull)(lane == f) << 55) | (resv << 56);
        wa.spill[base + __popc(amask & lane_lt)] = make_uint4((uint32_t)af, (uint32_t)(af >> 32), z0, w0);
      }
      continue;
    }
    // ---- interval of the first record's sector (uniform cache), lanes test theirs ----
    const uint32_t H = (space << 16) | (hi0 & 0xFFFFu);
    const uint32_t xs = x & ~31u;
    const uint32_t x0 = __shfl_sync(FULL, x, f);
    const uint32_t xs0 = x0 & ~31u;
    // broadcast instruction (every active lane on the first one's address): no
    // interval check, the merge leaves the first lane's key, never misaligned
    const bool bcast = __ballot_sync(FULL, act & (x != x0)) == 0;
    const bool h0 = win_has(e0, H, xs0), h1 = win_has(e1, H, xs0);
    if (!(h0 | h1)) {
      const WinEnt ne = win_lookup(sm.lo, sm.hi, sm.soff, nobj, steps, H, xs0);
      if (last1) { e0 = ne; last1 = false; } else { e1 = ne; last1 = true; }
    } else {
      last1 = !h0;
    }
    uint32_t blo = last1 ? e1.blo : e0.blo;
    uint32_t sbase = last1 ? e1.sbase : e0.sbase;
    uint32_t tail_s = last1 ? e1.tail_s : e0.tail_s, tail_m = last1 ? e1.tail_m : e0.tail_m;
    const int oid0 = last1 ? e1.oid : e0.oid;
    int oid = oid0;
    const bool inw = xs - blo < (last1 ? e1.bn : e0.bn);
    if (!bcast && __ballot_sync(FULL, act & !inw)) {
      if (act & !inw) {
        const WinEnt le = win_lookup(sm.lo, sm.hi, sm.soff, nobj, steps, H, xs);
        blo = le.blo; sbase = le.sbase; tail_s = le.tail_s; tail_m = le.tail_m; oid = le.oid;
      }
    }
    // ---- word mask, restricted to the object's words (G9) ----
    const uint32_t words = ((x & 3u) + size + 3u) >> 2;
    const uint32_t ma = (((1u << words) - 1u) << ((x >> 2) & 7u)) & (0u - (uint32_t)act);
    const uint32_t fa = (oid >= 0) ? (ma & (xs == tail_s ? tail_m : 0xFFu)) : 0u;
    if (launch0 != cur_launch) {
      if (cur_launch != 0xFFFFFFFFu) {
        const uint32_t um = __reduce_add_sync(FULL, lane_unmapped), mm = __reduce_add_sync(FULL, lane_mapped);
        if (lane == 0 && (um | mm)) {
          atomicAdd(&a.launch_ctr[2 * cur_launch], (ull)um);
          atomicAdd(&a.launch_ctr[2 * cur_launch + 1], (ull)mm);
        }
      }
      lane_mapped = lane_unmapped = 0;
      cur_launch = launch0;
    }
    const uint32_t pf = __popc(fa);
    lane_mapped += pf;
    lane_unmapped += __popc(ma) - pf;
    // ---- keys: adjacent-lane merge, then this lane's (pc id, sector) entries ----
    bool has = fa != 0;
    uint32_t mk = fa;
    const uint32_t g = sbase + ((xs - blo) >> 5);
    if (a.acc) {
      for (uint32_t m = fa; m; m &= m - 1) atomicAdd(&a.acc[8ull * g + (__ffs(m) - 1)], 1u);
    }
    if (bcast) has = has & (lane == f);
    else adjacent_merge32(g, mk, has, lane);
    if (__any_sync(FULL, has)) {
      const ull lw = ((ull)launch0 << W) | z0;
      if (lw != tag) {
        STAGE_PUSH(st, m0 != 0, entry_key(c0, m0, tag, SH, P), gkeys, gnk);
        STAGE_PUSH(st, m1 != 0, entry_key(c1, m1, tag, SH, P), gkeys, gnk);
        m0 = m1 = 0;
        tag = lw;
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
        pcid = pcid < a.pcmap.max_pcs ? pcid : 0u;
      }
      const ull ck = ((ull)pcid << 32) | g;
      const bool hit0 = c0 == ck, hit1 = c1 == ck;
      STAGE_PUSH(st, has & !hit0 & !hit1 & (m1 != 0), entry_key(c1, m1, tag, SH, P), gkeys, gnk);
      const uint32_t mprev = hit0 ? m0 : (hit1 ? m1 : 0u);
      const bool shift = has & !hit0;
      c1 = shift ? c0 : c1;
      m1 = shift ? m0 : m1;
      c0 = has ? ck : c0;
      m0 = has ? (mprev | mk) : m0;
    }
    // ---- instruction statistics (G24): active lanes ----
    const uint32_t fa0 = __shfl_sync(FULL, fa, f);
    const bool first_mapped = (oid0 >= 0) & ((fa0 >> ((x0 >> 2) & 7u)) & 1u);  // the first record's first word
    if (first_mapped & bcast) {
      ir.add(sm, launch0 * nobj + (uint32_t)oid0, false, a.instr_ctr, lane);
    } else if (first_mapped & (amask == FULL) &&
               __ballot_sync(FULL, (lane > 0) & (x < __shfl_up_sync(FULL, x, 1))) == 0) {
      // all lanes active, non-decreasing offsets: count sector changes; span = last - first + size
      const uint32_t px = __shfl_up_sync(FULL, x, 1);
      const uint32_t distinct = __popc(__ballot_sync(FULL, (lane == 0) | ((x >> 5) != (px >> 5))));
      const ull span = (ull)(__shfl_sync(FULL, x, 31) - x0) + size;
      ir.add(sm, launch0 * nobj + (uint32_t)oid0, distinct > (span + 31) / 32, a.instr_ctr, lane);
    } else if (first_mapped) {
      const unsigned m = __match_any_sync(FULL, act ? (x >> 5) : (0xF8000000u | (uint32_t)lane));
      const uint32_t distinct = __popc(__ballot_sync(FULL, act & (__ffs(m) - 1 == lane)));
      const uint32_t mn = __reduce_min_sync(FULL, act ? x : 0xFFFFFFFFu);
      const uint32_t mx = __reduce_max_sync(FULL, act ? x : 0u);
      const ull span = (ull)(mx - mn) + size;
      ir.add(sm, launch0 * nobj + (uint32_t)oid0, distinct > (span + 31) / 32, a.instr_ctr, lane);
    }
  }
  }
  STAGE_PUSH(st, m0 != 0, entry_key(c0, m0, tag, SH, P), gkeys, gnk);
  STAGE_PUSH(st, m1 != 0, entry_key(c1, m1, tag, SH, P), gkeys, gnk);
  st.flush(gkeys, gnk, lane);
  if (cur_launch != 0xFFFFFFFFu) {
    const uint32_t um = __reduce_add_sync(FULL, lane_unmapped), mm = __reduce_add_sync(FULL, lane_mapped);
    if (lane == 0 && (um | mm)) {
      atomicAdd(&a.launch_ctr[2 * cur_launch], (ull)um);
      atomicAdd(&a.launch_ctr[2 * cur_launch + 1], (ull)mm);
    }
  }
  if (lane == 0 && lanes_seen) atomicAdd(&wa.spill_ctr[1], lanes_seen);
  ir.flush(a.instr_ctr, lane);
  smem_flush_instr(sm, a.instr_ctr);
}

void launch_decode_warp(const DecodeArgs& a, const uint4* wrec, ull n_instr, uint4* spill, ull* spill_ctr,
                        int num_sms, cudaStream_t s) {
  WarpDecodeArgs wa{a, wrec, n_instr, spill, spill_ctr};
  const size_t smem = decode_smem(a);
  smem_optin((const void*)decode_warp_kernel<3>, 200 * 1024);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, decode_warp_kernel<3>, kDecWarps * 32, smem);
  if (per_sm < 1) per_sm = 1;
  const ull want = ((n_instr + kWarpRange - 1) / kWarpRange + kDecWarps - 1) / kDecWarps;
  ull grid = (ull)num_sms * per_sm;
  if (want < grid) grid = want;
  if (grid < 1) grid = 1;
  decode_warp_kernel<3><<<(unsigned)grid, kDecWarps * 32, smem, s>>>(wa);
}

}  // namespace thermo
