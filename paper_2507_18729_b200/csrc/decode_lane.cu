// decode_lane.cu -- the lane-per-record decode kernel (rows a2 + a3, SURVEY
// §8a), the default decoder.  A window is up to 32 consecutive records holding
// whole instructions (G24: all 32 when record 32 starts an instruction, else
// it ends at the last instruction head within 32 records, or after 32 records
// of one instruction); lane l reduces record l of
// the window.  Unlike the view-per-instruction kernel (decode_fast.cu), a
// window of many short instructions -- divergent loops, 62 % of SpMV's
// instructions have one active lane -- is reduced in place from the record
// ring instead of being deferred to the general kernel, which re-reads it.
//
//  * records stream through the per-warp cp.async ring (decode_fast.cu's);
//    work ranges of whole instructions are handed out dynamically;
//  * object resolution: four warp-uniform window intervals in
//    shared memory (the part of an object, or the gap between two, inside the
//    4 GiB window (space, addr[32,48)) of the records); each lane tests its own
//    sector offset against them (one subtraction and one compare each), misses
//    are looked up once per distinct interval and installed round-robin;
//  * word mask (G3/G4), sector id g = sbase + (offset - blo) / 32;
//  * pc ids (G11): four cached (launch, pc) sites, misses looked up once per
//    distinct site;
//  * pre-dedup (P:325's OR is idempotent): a window of one instruction merges
//    adjacent equal sectors (broadcast: the whole window is one key) as
//    decode_fast.cu does; a window of several instructions merges equal keys
//    anywhere (match_any); each lane then keeps its four most recent keys with
//    their OR-ed masks in registers and emits a key when it is replaced;
//  * instruction statistics (G24): a one-instruction window
//    takes decode_fast.cu's uniform tests (broadcast, stride, non-decreasing);
//    a window of one-record instructions is never misaligned (no record
//    straddles a sector here); otherwise segmented 32-bit scans per
//    instruction.  Counters per (launch, object) are aggregated per window.
// Windows with an invalid / out-of-range / out-of-scope record, a sector
// straddle, several 4 GiB windows or several launches are deferred whole to
// decode_general_kernel (decode.cu), which produces the same keys and counters.
#include "decode_common.cuh"

namespace thermo {

__device__ __forceinline__ void lane_ring_issue(uint32_t ring_lane, const uint4* src_lane, uint32_t c, uint32_t rlen,
                                                int lane) {
  const bool in = c * 32 + lane < rlen;
  const uint32_t dst = ring_lane + (c & (kRingChunks - 1)) * 512;
  const uint4* src = in ? src_lane + c * 32 : src_lane;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(in ? 16 : 0) : "memory");
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}

template <int MINB, int FEAT>
__global__ void __launch_bounds__(kDecWarps * 32, MINB) decode_lane_kernel(DecodeArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const Smem sm = smem_setup(smem, a);
  const uint32_t nobj = a.obj.n;
  const int lane = threadIdx.x & 31;
  const unsigned lane_lt = lanemask_lt();
  const int wib = threadIdx.x >> 5;
  int steps = 0;
  while ((1u << steps) < nobj) ++steps;
  const uint32_t P = a.kl.P, W = a.kl.W, LW = a.kl.L + a.kl.W;
  const uint32_t max_launches = a.max_launches, max_warps = a.max_warps;
  ull* const gkeys = a.keys;
  ull* const gnk = &a.ctr->n_keys;
  Stage st{reinterpret_cast<ull*>(sm.warp + wib * kWarpRegion), 0, a.seg_cnt, 8 + a.kl.P + a.kl.L + a.kl.W};
  uint4* const ring = reinterpret_cast<uint4*>(sm.warp + wib * kWarpRegion + kStage * sizeof(ull));
  const uint32_t ring_lane = (uint32_t)__cvta_generic_to_shared(ring + lane);
  // warp-uniform caches in shared memory: window entries e = 0..3 as
  // {H, blo, bn, sbase}, {tail_s, tail_m, oid, -} at wc[2e], wc[2e + 1];
  // sites {site0, id0, site1, id1} {site2, id2, site3, id3} at wc[8], wc[9]
  uint4* const wc = ring + kRingChunks * 32;
  if (lane < 4) {
    wc[2 * lane] = make_uint4(0xFFFFFFFFu, 0, 0, 0);
    wc[2 * lane + 1] = make_uint4(1, 0xFFu, 0xFFFFFFFFu, 0);
  }
  if (lane == 0) wc[8] = wc[9] = make_uint4(0xFFFFFFFFu, 0, 0xFFFFFFFFu, 0);
  uint32_t win_rr = 0, pc_rr = 0;  // round-robin replacement (uniform)
  DeferBuf dq{reinterpret_cast<ull*>(wc + 12), 0};
  uint32_t* const scr = reinterpret_cast<uint32_t*>(sm.warp + wib * kWarpRegion + kOffScratch);  // merge scratch
  __syncwarp();

  uint32_t lane_mapped = 0, lane_unmapped = 0;  // this lane's word counts for cur_launch
  uint32_t cur_launch = 0xFFFFFFFFu;
  InstrRegs ir;  // (launch, object) instruction counters for ids < 32
  // this lane's four most recent keys (full prefix) with their OR-ed masks
  ull c0 = ~0ull, c1 = ~0ull, c2 = ~0ull, c3 = ~0ull;
  uint32_t m0 = 0, m1 = 0, m2 = 0, m3 = 0;

  for (;;) {
    uint32_t r = 0;
    if (lane == 0) r = (uint32_t)atomicAdd(&a.ctr->next_range, 1ull);
    r = __shfl_sync(FULL, r, 0);
    if (r >= a.n_ranges) break;
    const ull p0 = a.heads[r];
    const uint32_t rlen = (uint32_t)(a.heads[r + 1] - p0);  // ingest calls hold < 2^32 records
    uint32_t issued = 0;
    const uint4* const src_lane = a.recs + p0 + lane;
    for (int k = 0; k <= kAhead; ++k) lane_ring_issue(ring_lane, src_lane, issued++, rlen, lane);
    uint32_t off = 0;  // the window's first record, from p0
    while (off < rlen) {
      if (issued <= (off >> 5) + kAhead) lane_ring_issue(ring_lane, src_lane, issued++, rlen, lane);
      asm volatile("cp.async.wait_group %0;\n" ::"n"(kAhead - 1) : "memory");  // the window's 2 chunks landed
      __syncwarp();
      const uint32_t rem = rlen - off;
      // records at or past the range end were zero-filled by cp.async
      const uint4 cur = ring[(off + lane) & (kRingChunks * 32 - 1)];
      // record off + 32 (in the window's second chunk, landed): when it starts
      // an instruction, the 32 records hold whole instructions
      const uint32_t y32 = ring[(off + 32) & (kRingChunks * 32 - 1)].y;
      // ---- window: the whole instructions within the next 32 records ----
      const unsigned hb_all = __ballot_sync(FULL, (cur.y >> 23) & 1u) | 1u;  // lane 0 starts one
      uint32_t span;
      if (rem <= 32) span = rem;
      else if ((y32 >> 23) & 1u) span = 32u;
      else span = (hb_all & ~1u) ? 31u - __clz(hb_all & ~1u) : 32u;
      const unsigned actm = span >= 32 ? FULL : ((1u << span) - 1u);
      const bool act = lane < (int)span;
      const unsigned hb = hb_all & actm;  // instruction heads of the window

      const uint32_t x = cur.x, y = cur.y, z = cur.z, w = cur.w;
      const uint32_t l2s = (y >> 16) & 7u;
      const uint32_t size = 1u << (l2s & 7u);
      const uint32_t launch = w >> 20;
      const uint32_t H = ((y >> 5) & 0x30000u) | (y & 0xFFFFu);  // space << 16 | addr[32,48)
      const uint32_t H0 = __shfl_sync(FULL, H, 0), launch0 = __shfl_sync(FULL, launch, 0);
      bool odd = (l2s > 4) | (((y >> 19) & 3u) == 3u) | (((y >> 21) & 3u) == 3u) | ((y >> 24) != 0) |
                 (launch >= max_launches) | (z >= max_warps) | ((x & 31u) + size > 32u) | (H != H0) |
                 (launch != launch0);
      if (FEAT & 2) {  // sampled block / launch whitelist: a window entirely out of scope was never traced
        const bool oos = out_of_scope(a, z, launch);
        if (__ballot_sync(FULL, act & !oos) == 0) {
          off += span;
          continue;
        }
        odd |= oos;  // a mixed window: the general kernel filters per record
      }
      if (__ballot_sync(FULL, act & odd)) {
        dq.push(((p0 + off) << 7) | span, a.deferred, &a.ctr->n_deferred, lane);  // to the general kernel
        off += span;
        continue;
      }
      const uint32_t xs = x & ~31u;
      // the window is one instruction of uniform warp, pc and size (what a
      // collector emits): decode_fast.cu's uniform shortcuts apply
      const uint32_t x0 = __shfl_sync(FULL, x, 0);
      const uint32_t z0 = __shfl_sync(FULL, z, 0), w0 = __shfl_sync(FULL, w, 0), l0 = __shfl_sync(FULL, l2s, 0);
      const bool one = hb == 1u && __ballot_sync(FULL, act & ((z != z0) | (w != w0) | (l2s != l0))) == 0;
      const bool bcast = one && __ballot_sync(FULL, act & (x != x0)) == 0;
      // a window of several instructions of one source warp: one match over
      // (site, sector offset) groups equal keys (the merge: launch, warp and
      // window are uniform, the site fixes the pc id, the offset the sector)
      // and equal sectors of an instruction (the statistics); 0 = not taken
      unsigned grp = 0;
      if (!one && __ballot_sync(FULL, act & (z != z0)) == 0)
        grp = __match_any_sync(FULL, act ? (((ull)w << 32) | (x >> 5)) : (0xFFFFFFFF80000000ull | (ull)lane));
      // ---- window interval of each lane's sector (four uniform entries) ----
      uint32_t blo = 0, bn = 0, sbase = 0, tail_s = 1, tail_m = 0xFFu;
      int oid = -1;
      bool hit = false;
      if (one) {  // lane 0's interval (lanes e < 4 test entry e), then every lane tests it
        uint4 Ae = make_uint4(0, 0, 0, 0);
        if (lane < 4) Ae = wc[2 * lane];
        const uint32_t xs0 = x0 & ~31u;
        const unsigned hits = __ballot_sync(FULL, (lane < 4) & (Ae.x == H0) & (xs0 - Ae.y < Ae.z));
        if (hits) {
          const uint32_t e = __ffs(hits) - 1;
          const uint4 A = wc[2 * e], B = wc[2 * e + 1];
          blo = A.y; bn = A.z; sbase = A.w; tail_s = B.x; tail_m = B.y; oid = (int)B.z;
          hit = xs - blo < bn;
        }
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint4 A = wc[2 * e];
          const bool h = !hit && (A.x == H0) && (xs - A.y < A.z);
          if (h) {
            const uint4 B = wc[2 * e + 1];
            blo = A.y; bn = A.z; sbase = A.w; tail_s = B.x; tail_m = B.y; oid = (int)B.z;
          }
          hit = hit || h;
        }
      }
      unsigned miss = __ballot_sync(FULL, act & !hit);
      while (miss) {  // (uniform) the lowest missing lane's interval, installed round-robin
        const uint32_t xl = __shfl_sync(FULL, xs, __ffs(miss) - 1);
        const WinEnt ne = win_lookup(sm.lo, sm.hi, sm.soff, nobj, steps, H0, xl);
        const uint32_t e = win_rr;
        win_rr = (win_rr + 1) & 3u;
        __syncwarp();  // every lane has read the entries before lane 0 replaces one
        if (lane == 0) {
          wc[2 * e] = make_uint4(ne.H, ne.blo, ne.bn, ne.sbase);
          wc[2 * e + 1] = make_uint4(ne.tail_s, ne.tail_m, (uint32_t)ne.oid, 0);
        }
        __syncwarp();
        if (act && !hit && (xs - ne.blo < ne.bn)) {
          blo = ne.blo; bn = ne.bn; sbase = ne.sbase; tail_s = ne.tail_s; tail_m = ne.tail_m; oid = ne.oid;
          hit = true;
        }
        miss = __ballot_sync(FULL, act & !hit);
      }
      (void)bn;
      // ---- word mask, restricted to the object's words (G9) ----
      const uint32_t wfirst = (x >> 2) & 7u;
      const uint32_t words = ((x & 3u) + size + 3u) >> 2;
      const uint32_t ma = act ? (((1u << words) - 1u) << wfirst) : 0u;
      const uint32_t fa = (oid >= 0) ? (ma & (xs == tail_s ? tail_m : 0xFFu)) : 0u;
      // the record's first word is mapped: it attributes its instruction (G24)
      const bool fm = act & (oid >= 0) & ((xs != tail_s) | ((tail_m >> wfirst) & 1u));
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
      const uint32_t g = sbase + ((xs - blo) >> 5);
      if (FEAT & 1) {  // access counts: every lane's every mapped word (before any merge)
        for (uint32_t m = fa; m; m &= m - 1) atomicAdd(&a.acc[8ull * g + (__ffs(m) - 1)], 1u);
      }
      bool has = fa != 0;
      uint32_t mk = fa;
      if (__any_sync(FULL, has)) {
        // ---- pc id of each lane (four uniform cached sites) ----
        uint32_t pcid = 0;
        if (a.track_pc) {
          const uint4 q0 = wc[8], q1 = wc[9];
          uint32_t id = 0xFFFFFFFFu;
          id = (w == q0.x) ? q0.y : id;
          id = (id == 0xFFFFFFFFu && w == q0.z) ? q0.w : id;
          id = (id == 0xFFFFFFFFu && w == q1.x) ? q1.y : id;
          id = (id == 0xFFFFFFFFu && w == q1.z) ? q1.w : id;
          unsigned pm = __ballot_sync(FULL, has & (id == 0xFFFFFFFFu));
          while (pm) {  // (uniform) one lookup per missing site, by its lowest lane
            const int ll = __ffs(pm) - 1;
            const uint32_t sl = __shfl_sync(FULL, w, ll);
            uint32_t v = 0;
            __syncwarp();
            if (lane == ll) {
              v = pc_lookup(sm.pc, a.pcmap, sl, a.ctr);
              v = v < a.pcmap.max_pcs ? v : 0u;  // overflow is reported at build (ERANGE)
              reinterpret_cast<uint32_t*>(wc + 8)[2 * pc_rr] = sl;
              reinterpret_cast<uint32_t*>(wc + 8)[2 * pc_rr + 1] = v;
            }
            __syncwarp();
            v = __shfl_sync(FULL, v, ll);
            pc_rr = (pc_rr + 1) & 3u;
            if (has && w == sl) id = v;
            pm = __ballot_sync(FULL, has & (id == 0xFFFFFFFFu));
          }
          pcid = id;
        }
        const ull pre = ((((ull)g << LW) | ((ull)launch << W) | z) << P) | pcid;
        // ---- merge the window's equal keys ----
        if (bcast) {
          has = has && lane == 0;  // the run of equal sectors is the whole window
        } else if (one) {
          adjacent_merge32(g, mk, has, lane);  // one instruction: warp, launch and pc are uniform
        } else if (grp) {
          group_merge_grp(grp & __ballot_sync(FULL, has), mk, has, scr, lane);
        } else {
          group_merge(pre, mk, has, scr, lane);
        }
        // ---- this lane's four most recent keys ----
        // (move-to-front over four entries: SpMV's col / val / x loads of one
        // lane cycle through three keys, which a two-entry LRU thrashes)
        const bool hit0 = c0 == pre, hit1 = c1 == pre, hit2 = c2 == pre, hit3 = c3 == pre;
        const bool s1 = has & !hit0, s2 = s1 & !hit1, s3 = s2 & !hit2;
        STAGE_PUSH(st, s3 & !hit3 & (m3 != 0), (c3 << 8) | m3, gkeys, gnk);
        const uint32_t mprev = hit0 ? m0 : (hit1 ? m1 : (hit2 ? m2 : (hit3 ? m3 : 0u)));
        c3 = s3 ? c2 : c3;
        m3 = s3 ? m2 : m3;
        c2 = s2 ? c1 : c2;
        m2 = s2 ? m1 : m2;
        c1 = s1 ? c0 : c1;
        m1 = s1 ? m0 : m1;
        c0 = has ? pre : c0;
        m0 = has ? (mprev | mk) : m0;
      }
      // ---- instruction statistics (G24) ----
      if (one) {
        const bool fm0 = __shfl_sync(FULL, fm, 0);
        const int oid0 = __shfl_sync(FULL, oid, 0);
        if (fm0) {
          bool mis;
          if (bcast) {
            mis = false;  // one address: distinct = 1 <= ceil(size / 32)
          } else {
            const uint32_t px = __shfl_up_sync(FULL, x, 1);
            if (__ballot_sync(FULL, act & (lane > 0) & (x < px)) == 0) {
              // non-decreasing offsets: count sector changes; span = last - first + size
              const uint32_t distinct = __popc(__ballot_sync(FULL, act & ((lane == 0) | ((x >> 5) != (px >> 5)))));
              const ull sp = (ull)(__shfl_sync(FULL, x, span - 1) - x0) + size;
              mis = distinct > (sp + 31) / 32;
            } else {
              const unsigned m = __match_any_sync(FULL, act ? (x >> 5) : (0xF8000000u | (uint32_t)lane));
              const uint32_t distinct = __popc(__ballot_sync(FULL, act & (__ffs(m) - 1 == lane)));
              const uint32_t mn = __reduce_min_sync(FULL, act ? x : 0xFFFFFFFFu);
              const uint32_t mx = __reduce_max_sync(FULL, act ? x : 0u);
              mis = distinct > ((ull)(mx - mn) + size + 31) / 32;
            }
          }
          ir.add(sm, launch0 * nobj + (uint32_t)oid0, mis, a.instr_ctr, lane);
        }
      } else {
        // several instructions: lanes [s, e) between consecutive heads
        const bool head = act & ((hb >> lane) & 1u);
        bool mis = false;
        if ((hb | ~actm) != FULL) {  // some instruction has several records
          const unsigned le = lane_lt | (1u << lane);
          const int s0 = 31 - __clz(hb & le);
          const unsigned after = hb & ~le;
          const int e0 = after ? __ffs(after) - 1 : (int)span;
          const unsigned segm = (e0 >= 32 ? FULL : ((1u << e0) - 1u)) & ~((1u << s0) - 1u);
          // min / max byte offset over the instruction: segmented 32-bit scans
          uint32_t mn = act ? x : 0xFFFFFFFFu, mx = act ? x + size - 1 : 0u;
          for (int d = 1; d < 32; d <<= 1) {
            const uint32_t omn = __shfl_down_sync(FULL, mn, d), omx = __shfl_down_sync(FULL, mx, d);
            if (lane + d < e0) { mn = omn < mn ? omn : mn; mx = omx > mx ? omx : mx; }
          }
          // (an instruction's records share the site: grp & segm = its lanes on this sector)
          const unsigned m = grp ? grp : __match_any_sync(FULL, act ? (x >> 5) : (0xF8000000u | (uint32_t)lane));
          const uint32_t distinct = __popc(__ballot_sync(FULL, act && (__ffs(m & segm) - 1 == lane)) & segm);
          mis = distinct > ((ull)(mx - mn) + 1 + 31) / 32;  // (valid at lane s0: its instruction's values)
        }
        // one update per distinct (launch, object) of the window's counted instructions
        const bool counted = head & fm;
        const uint32_t key1 = counted ? launch0 * nobj + (uint32_t)oid + 1u : 0u;
        const unsigned peers = __match_any_sync(FULL, key1);
        const unsigned misb = __ballot_sync(FULL, counted && mis);
        if (counted && lane == __ffs(peers) - 1)
          instr_add_n(sm, key1, (uint32_t)__popc(peers), (uint32_t)__popc(peers & misb), a.instr_ctr);
      }
      off += span;
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");  // no copy may land in the next range's slots
    __syncwarp();
  }
  STAGE_PUSH(st, m0 != 0, (c0 << 8) | m0, gkeys, gnk);
  STAGE_PUSH(st, m1 != 0, (c1 << 8) | m1, gkeys, gnk);
  STAGE_PUSH(st, m2 != 0, (c2 << 8) | m2, gkeys, gnk);
  STAGE_PUSH(st, m3 != 0, (c3 << 8) | m3, gkeys, gnk);
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
static int lane_per_sm(size_t smem) {
  smem_optin((const void*)decode_lane_kernel<MINB, FEAT>, 200 * 1024);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, decode_lane_kernel<MINB, FEAT>, kDecWarps * 32, smem);
  return per_sm < 1 ? 1 : per_sm;
}

template <int MINB, int FEAT>
static void launch_lane_t(const DecodeArgs& a, int num_sms, cudaStream_t s, size_t smem) {
  const int per_sm = lane_per_sm<MINB, FEAT>(smem);
  const ull want = ((ull)a.n_ranges + kDecWarps - 1) / kDecWarps;
  ull grid = (ull)num_sms * per_sm;
  if (want < grid) grid = want;
  if (grid < 1) grid = 1;
  decode_lane_kernel<MINB, FEAT><<<(unsigned)grid, kDecWarps * 32, smem, s>>>(a);
}

void launch_decode_lane(const DecodeArgs& a, int num_sms, cudaStream_t s) {
  const size_t smem = decode_smem(a);
  const int feat = (a.acc ? 1 : 0) | ((a.block_warps || a.wl) ? 2 : 0);
  switch (feat) {
    case 0: launch_lane_t<3, 0>(a, num_sms, s, smem); break;
    case 1: launch_lane_t<3, 1>(a, num_sms, s, smem); break;
    case 2: launch_lane_t<3, 2>(a, num_sms, s, smem); break;
    default: launch_lane_t<3, 3>(a, num_sms, s, smem); break;
  }
}

}  // namespace thermo
