// decode_fast.cu -- the fast decode kernel (rows a2 + a3): one
// warp instruction ("view", lane l = record p + l) per iteration when all its
// records share warp, pc, launch, size, kind, space and the upper 16 address
// bits, and none straddles a sector -- what a collector emits for one
// instruction.  Any other view is deferred to
// decode_general_kernel (decode.cu), which produces the same keys and counters.
//
// The kernel is issue-bound, so it is written for instruction economy:
//  * addresses are handled as 32-bit offsets inside the view's uniform 4 GiB
//    window H = (space, addr[32,48));
//  * object resolution goes through a two-entry warp-uniform cache
//    of window intervals: either the part of an object inside the window, with
//    the sector id of its first sector and the allowed words of its partial
//    last sector (G9), or the gap between two objects.  A lane's test is one
//    subtraction and one compare; its sector id g one shift and one add;
//  * word mask (G3/G4): ((1 << words) - 1) << first word;
//  * pre-dedup (P:325's OR is idempotent): lanes holding the same sector merge
//    into the run's first lane; each lane then keeps, in registers, its two
//    most recent (pc id, sector) -> mask entries and emits a key only when an
//    entry is replaced (A[row][k..k+7] of Listing 1 hit the same lane's
//    entry for 8 consecutive k) or the source warp changes.  Keys go through a
//    256-entry per-warp shared-memory stage flushed with one global atomic;
//  * the misalignment test of the instruction (G24) counts sector
//    changes with one ballot when the offsets are non-decreasing.
#include "decode_common.cuh"

namespace thermo {

// record ring: chunk c = records [32c, 32c + 32) of the range (offsets from its
// first record) lives in ring slot c % kRingChunks; lane l copies record
// 32c + l with cp.async, zero-filled at or past the range end
// ring_lane: shared address of this lane's slot in chunk slot 0; src_lane:
// the range's record `lane`
__device__ __forceinline__ void ring_issue(uint32_t ring_lane, const uint4* src_lane, uint32_t c, uint32_t rlen,
                                           int lane) {
  const bool in = c * 32 + lane < rlen;
  const uint32_t dst = ring_lane + (c & (kRingChunks - 1)) * 512;
  const uint4* src = in ? src_lane + c * 32 : src_lane;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(in ? 16 : 0) : "memory");
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}

// FEAT: compile-time features (1: access counts, 2: sampled-block filter), so
// the common configuration carries none of their per-view tests
template <int MINB, int FEAT>
__global__ void __launch_bounds__(kDecWarps * 32, MINB) decode_kernel(DecodeArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const Smem sm = smem_setup(smem, a);
  const uint32_t nobj = a.obj.n;
  const int lane = threadIdx.x & 31;
  const unsigned lane_lt = lanemask_lt();
  const int wib = threadIdx.x >> 5;
  int steps = 0;
  while ((1u << steps) < nobj) ++steps;
  const uint32_t P = a.kl.P, W = a.kl.W;
  const uint32_t SH8 = a.kl.L + a.kl.W + P + 8;
  const uint32_t max_launches = a.max_launches, max_warps = a.max_warps;
  ull* const gkeys = a.keys;
  ull* const gnk = &a.ctr->n_keys;
  Stage st{reinterpret_cast<ull*>(sm.warp + wib * kWarpRegion), 0, a.seg_cnt, 8 + a.kl.P + a.kl.L + a.kl.W};
  uint4* const ring = reinterpret_cast<uint4*>(sm.warp + wib * kWarpRegion + kStage * sizeof(ull));
  const uint32_t ring_lane = (uint32_t)__cvta_generic_to_shared(ring + lane);
  // warp-uniform caches kept in shared memory (registers are the kernel's
  // occupancy limit): window entries e = 0..3 as {H, blo, bn, sbase},
  // {tail_s, tail_m, oid, -} at wc[2e], wc[2e + 1] (four: SpMV's col / val / x
  // loads alternate between three objects); site -> pc id cache
  // {site0, id0, site1, id1} ... {site6, id6, site7, id7} at wc[8..11] (the
  // stencil's six loads and store cycle through six pcs)
  uint4* const wc = ring + kRingChunks * 32;
  if (lane < 4) {
    wc[2 * lane] = make_uint4(0xFFFFFFFFu, 0, 0, 0);
    wc[2 * lane + 1] = make_uint4(1, 0xFFu, 0xFFFFFFFFu, 0);
  }
  if (lane < 4) wc[8 + lane] = make_uint4(0xFFFFFFFFu, 0, 0xFFFFFFFFu, 0);
  uint32_t win_rr = 0, pc_rr = 0;  // round-robin replacement (uniform)
  DeferBuf dq{reinterpret_cast<ull*>(wc + 12), 0};
  __syncwarp();

  uint32_t lane_mapped = 0, lane_unmapped = 0;  // this lane's word counts for cur_launch
  uint32_t cur_launch = 0xFFFFFFFFu;
  InstrRegs ir;  // (launch, object) instruction counters for ids < 32
  // this lane's two most recent dedup entries: (pc id << 32 | g) -> mask
  ull c0 = 0, c1 = 0;
  uint32_t m0 = 0, m1 = 0;
  ull tag = 0;  // (launch << W | warp) of the entries (uniform)
  ull tag8 = 0;  // tag << (P + 8), its place in a key

  const uint32_t gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;

  // ranges are handed out dynamically (their costs differ: SpMV rows), so the
  // warps finish together instead of waiting for the slowest static share
  (void)gwarp;
  (void)nwarps;
  for (;;) {
    uint32_t r = 0;
    if (lane == 0) r = (uint32_t)atomicAdd(&a.ctr->next_range, 1ull);
    r = __shfl_sync(FULL, r, 0);
    if (r >= a.n_ranges) break;
    const ull p0 = a.heads[r];
    const uint32_t rlen = (uint32_t)(a.heads[r + 1] - p0);  // ingest calls hold < 2^32 records
    const uint4* const rbase = a.recs + p0;
    // keep kAhead chunks in flight ahead of the one holding the view (~3 KB per warp)
    uint32_t issued = 0;
    const uint4* const src_lane = rbase + lane;
    for (int k = 0; k <= kAhead; ++k) ring_issue(ring_lane, src_lane, issued++, rlen, lane);
    uint32_t off = 0;  // the view's first record, from p0
    while (off < rlen) {
      if (issued <= (off >> 5) + kAhead) ring_issue(ring_lane, src_lane, issued++, rlen, lane);
      asm volatile("cp.async.wait_group %0;\n" ::"n"(kAhead - 1) : "memory");  // the view's 2 chunks landed
      __syncwarp();
      const uint32_t rem = rlen - off;
      // records at or past the range end were zero-filled by cp.async
      const uint4 cur = ring[(off + lane) & (kRingChunks * 32 - 1)];
      // ---- view = one warp instruction: records [off, off + len) ----
      const unsigned sb = __ballot_sync(FULL, (cur.y >> 23) & 1u) & ~1u;
      uint32_t len = sb ? (uint32_t)(__ffs(sb) - 1) : 32u;
      len = rem < len ? rem : len;
      if (len < kShortView) {
        // short instructions (divergent loops, e.g. SpMV rows): pack the whole
        // instructions of the next 32 records into one general-path view
        const uint32_t span = rem <= 32 ? rem : (sb ? 31u - __clz(sb) : 0u);  // to the last head / range end
        if (span > len) {
          dq.push(((p0 + off) << 7) | span, a.deferred, &a.ctr->n_deferred, lane);
          off += span;
          continue;
        }
      }
      const uint32_t offn = off + len;

      const bool act = lane < (int)len;
      const uint32_t y0 = __shfl_sync(FULL, cur.y, 0);
      const uint32_t z0 = __shfl_sync(FULL, cur.z, 0), w0 = __shfl_sync(FULL, cur.w, 0);
      const uint32_t l2s = (y0 >> 16) & 7u;
      const uint32_t launch0 = w0 >> 20;
      const bool ok0 = (l2s <= 4) & (((y0 >> 19) & 3u) != 3u) & (((y0 >> 21) & 3u) != 3u) & ((y0 >> 24) == 0) &
                       (launch0 < max_launches) & (z0 < max_warps);
      const uint32_t size = 1u << l2s;
      const uint32_t x = cur.x;
      // uniform instruction (upper address bits included), no sector straddle
      const bool odd = act & ((cur.z != z0) | (cur.w != w0) | (((cur.y ^ y0) & 0xFF7FFFFFu) != 0) |
                              ((x & 31u) + size > 32u));
      if ((FEAT & 2) && out_of_scope(a, z0, launch0) && __ballot_sync(FULL, odd) == 0) {
        off = offn;  // an instruction outside the sampled block or the launch whitelist: never traced
        continue;
      }
      if (!ok0 || __ballot_sync(FULL, odd) != 0) {
        dq.push(((p0 + off) << 7) | len, a.deferred, &a.ctr->n_deferred, lane);  // to the general kernel
        off = offn;
        continue;
      }
      // ---- interval of lane 0's sector (uniform cache), lanes test theirs ----
      const uint32_t H = ((y0 >> 5) & 0x30000u) | (y0 & 0xFFFFu);  // space << 16 | addr[32,48)
      const uint32_t xs = x & ~31u;
      const uint32_t x0 = __shfl_sync(FULL, x, 0);
      const uint32_t xs0 = x0 & ~31u;
      // broadcast instruction: every lane on lane 0's address (B[k][col] of
      // Listing 1); its lanes are all in lane 0's interval, merge into lane 0
      // and span one sector run (never misaligned), so those steps are skipped
      const bool bcast = __ballot_sync(FULL, act & (x != x0)) == 0;
      // lane e < 4 tests window entry e; one ballot finds the hit
      uint4 Ae = make_uint4(0, 0, 0, 0);
      if (lane < 4) Ae = wc[2 * lane];
      const unsigned hits = __ballot_sync(FULL, (lane < 4) & (Ae.x == H) & (xs0 - Ae.y < Ae.z));
      uint32_t blo, bn, sbase, tail_s, tail_m;
      int oid0;
      if (!hits) {  // uniform miss: replace the round-robin entry
        const WinEnt ne = win_lookup(sm.lo, sm.hi, sm.soff, nobj, steps, H, xs0);
        const uint32_t e = win_rr;
        win_rr = (win_rr + 1) & 3u;
        __syncwarp();  // every lane has read the entries before lane 0 replaces one
        if (lane == 0) {
          wc[2 * e] = make_uint4(ne.H, ne.blo, ne.bn, ne.sbase);
          wc[2 * e + 1] = make_uint4(ne.tail_s, ne.tail_m, (uint32_t)ne.oid, 0);
        }
        __syncwarp();  // and the warp sees it from the next view on
        blo = ne.blo; bn = ne.bn; sbase = ne.sbase; tail_s = ne.tail_s; tail_m = ne.tail_m; oid0 = ne.oid;
      } else {
        const uint32_t e = __ffs(hits) - 1;
        const uint4 A = wc[2 * e];
        const uint4 B = wc[2 * e + 1];
        blo = A.y; bn = A.z; sbase = A.w; tail_s = B.x; tail_m = B.y; oid0 = (int)B.z;
      }
      // lane 0's first word is mapped (uniform, from lane 0's interval): its
      // instruction is counted in the statistics below
      const bool first_mapped = (oid0 >= 0) & ((xs0 != tail_s) | ((tail_m >> ((x0 >> 2) & 7u)) & 1u));
      int oid = oid0;
      const bool inw = xs - blo < bn;
      if (!bcast && __ballot_sync(FULL, act & !inw)) {  // lanes outside lane 0's interval (rare)
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
      if (FEAT & 1) {  // access counts: every lane's every mapped word (before the merge)
        for (uint32_t m = fa; m; m &= m - 1) atomicAdd(&a.acc[8ull * g + (__ffs(m) - 1)], 1u);
      }
      // stride instruction: every active lane's sector strictly above the
      // previous lane's (A[row][k] of Listing 1): no two lanes share a sector,
      // so the merge has nothing to do and the distinct sectors are the lanes
      uint32_t px = 0;
      bool stride = false;
      if (!bcast) {
        px = __shfl_up_sync(FULL, x, 1);
        const unsigned actm = len >= 32 ? FULL : ((1u << len) - 1u);
        stride = __ballot_sync(FULL, act & (lane > 0) & ((x >> 5) > (px >> 5))) == (actm & ~1u);
      }
      if (bcast) has = has & (lane == 0);  // the run of equal sectors is the whole view
      else if (!stride) adjacent_merge32(g, mk, has, lane);
      if (__any_sync(FULL, has)) {
        const ull lw = ((ull)launch0 << W) | z0;
        if (lw != tag) {  // new source warp: every entry leaves as a key
          STAGE_PUSH(st, m0 != 0, entry_key8(c0, m0, tag8, SH8), gkeys, gnk);
          STAGE_PUSH(st, m1 != 0, entry_key8(c1, m1, tag8, SH8), gkeys, gnk);
          m0 = m1 = 0;
          tag = lw;
          tag8 = lw << (P + 8);
        }
        uint32_t pcid = 0;
        if (a.track_pc) {
          // eight cached sites (uniform): lane e < 8 tests entry e
          const uint32_t* const pcw = reinterpret_cast<const uint32_t*>(wc + 8);
          const unsigned ph = __ballot_sync(FULL, (lane < 8) && pcw[2 * (lane & 7)] == w0);
          if (ph) {
            pcid = pcw[2 * (__ffs(ph) - 1) + 1];
          } else {
            uint32_t id = 0;
            __syncwarp();  // (as for the window entries)
            if (lane == 0) {
              id = pc_lookup(sm.pc, a.pcmap, w0, a.ctr);
              id = id < a.pcmap.max_pcs ? id : 0u;  // overflow is reported at build (ERANGE)
              reinterpret_cast<uint32_t*>(wc + 8)[2 * pc_rr] = w0;
              reinterpret_cast<uint32_t*>(wc + 8)[2 * pc_rr + 1] = id;
            }
            pc_rr = (pc_rr + 1) & 7u;
            __syncwarp();
            pcid = __shfl_sync(FULL, id, 0);
          }
        }
        // two-entry LRU of (pc id, sector) -> mask; entry 0 is the most recent
        const ull ck = ((ull)pcid << 32) | g;
        const bool hit0 = c0 == ck, hit1 = c1 == ck;
        // a replaced entry leaves as a key
        STAGE_PUSH(st, has & !hit0 & !hit1 & (m1 != 0), entry_key8(c1, m1, tag8, SH8), gkeys, gnk);
        const uint32_t mprev = hit0 ? m0 : (hit1 ? m1 : 0u);
        const bool shift = has & !hit0;  // entry 0 moves to slot 1 (selects, no branch)
        c1 = shift ? c0 : c1;
        m1 = shift ? m0 : m1;
        c0 = has ? ck : c0;
        m0 = has ? (mprev | mk) : m0;
      }
      // ---- instruction statistics (G24) ----
      if (first_mapped & bcast) {  // one address: distinct = 1 <= ceil(size / 32) sectors
        ir.add(sm, launch0 * nobj + (uint32_t)oid0, false, a.instr_ctr, lane);
      } else if (first_mapped & stride) {  // len distinct sectors over [x0, x_last + size)
        const uint32_t d = __shfl_sync(FULL, x, len - 1) - x0;
        const uint32_t need = (d >> 5) + (((d & 31u) + size + 31u) >> 5);  // ceil((d + size) / 32)
        ir.add(sm, launch0 * nobj + (uint32_t)oid0, len > need, a.instr_ctr, lane);
      } else if (first_mapped) {
        const bool down = act & (lane > 0) & (x < px);
        uint32_t distinct;
        ull span;
        if (__ballot_sync(FULL, down) == 0) {
          // non-decreasing offsets in one window: count sector changes; span = last - first + size
          distinct = __popc(__ballot_sync(FULL, act & ((lane == 0) | ((x >> 5) != (px >> 5)))));
          span = (ull)(__shfl_sync(FULL, x, len - 1) - x0) + size;
        } else {
          const unsigned m = __match_any_sync(FULL, act ? (x >> 5) : (0xF8000000u | (uint32_t)lane));
          distinct = __popc(__ballot_sync(FULL, act & (__ffs(m) - 1 == lane)));
          const uint32_t mn = __reduce_min_sync(FULL, act ? x : 0xFFFFFFFFu);
          const uint32_t mx = __reduce_max_sync(FULL, act ? x : 0u);
          span = (ull)(mx - mn) + size;
        }
        ir.add(sm, launch0 * nobj + (uint32_t)oid0, distinct > (span + 31) / 32, a.instr_ctr, lane);
      }
      off = offn;
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");  // no copy may land in the next range's slots
    __syncwarp();
  }
  STAGE_PUSH(st, m0 != 0, entry_key8(c0, m0, tag8, SH8), gkeys, gnk);
  STAGE_PUSH(st, m1 != 0, entry_key8(c1, m1, tag8, SH8), gkeys, gnk);
  st.flush(gkeys, gnk, lane);
  dq.flush(a.deferred, &a.ctr->n_deferred, lane);
  if (cur_launch != 0xFFFFFFFFu) {
    const uint32_t um = __reduce_add_sync(FULL, lane_unmapped), mm = __reduce_add_sync(FULL, lane_mapped);
    if (lane == 0 && (um | mm)) {
      atomicAdd(&a.launch_ctr[2 * cur_launch], (ull)um);
      atomicAdd(&a.launch_ctr[2 * cur_launch + 1], (ull)mm);
    }
  }
  ir.flush(a.instr_ctr, lane);
  smem_flush_instr(sm, a.instr_ctr);
}

template <int MINB, int FEAT>
static void launch_decode_t(const DecodeArgs& a, int num_sms, cudaStream_t s, size_t smem) {
  smem_optin((const void*)decode_kernel<MINB, FEAT>, 200 * 1024);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, decode_kernel<MINB, FEAT>, kDecWarps * 32, smem);
  if (per_sm < 1) per_sm = 1;
  const ull want = ((ull)a.n_ranges + kDecWarps - 1) / kDecWarps;
  ull grid = (ull)num_sms * per_sm;
  if (want < grid) grid = want;
  if (grid < 1) grid = 1;
  decode_kernel<MINB, FEAT><<<(unsigned)grid, kDecWarps * 32, smem, s>>>(a);
}

void launch_decode(const DecodeArgs& a, int num_sms, cudaStream_t s) {
  const size_t smem = decode_smem(a);
  const int feat = (a.acc ? 1 : 0) | ((a.block_warps || a.wl) ? 2 : 0);
  static const int minb = getenv("THERMO_DEC_MINB") ? atoi(getenv("THERMO_DEC_MINB")) : 3;
  switch (feat) {
    case 0:
      if (minb == 4) launch_decode_t<4, 0>(a, num_sms, s, smem);
      else if (minb == 2) launch_decode_t<2, 0>(a, num_sms, s, smem);
      else launch_decode_t<3, 0>(a, num_sms, s, smem);
      break;
    case 1: launch_decode_t<3, 1>(a, num_sms, s, smem); break;
    case 2: launch_decode_t<3, 2>(a, num_sms, s, smem); break;
    default: launch_decode_t<3, 3>(a, num_sms, s, smem); break;
  }
}

}  // namespace thermo
