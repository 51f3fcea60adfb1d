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
// find_heads) and walks them one warp instruction ("view") at a time: lane l
// handles record p + l of the view, so lane l sees lane l of consecutive
// instructions.  A view whose records share warp, pc, launch, space and size
// (every instruction a collector emits) takes the fast path, where
// those fields are warp-uniform; anything else takes the general path.
//
// Keys (a3): [ g : S ][ launch, warp : L+W ][ pc id : P ][ word mask : 8 ] --
// one key stream carries both the (sector, warp) and the (pc, sector) facts.
// Pre-dedup: (1) adjacent lanes holding the same sector merge into the first
// lane (B[k][col] in Listing 1: all 32 lanes on one word); (2) a per-warp
// shared-memory table of (pc id, sector) -> word mask holds one source warp's
// keys across its instructions (A[row][k..k+7] share a sector; stencil rows
// overlap between lanes) and is emitted when the source warp changes.
#include "decode_common.cuh"

namespace thermo {


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

// instruction heads among sampled 32-record chunks (every stride-th chunk):
// out[0] += records sampled, out[1] += heads among them
__global__ void head_sample_kernel(const uint4* __restrict__ recs, ull n, ull stride, uint32_t nsample,
                                   ull* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const uint32_t c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (c >= nsample) return;
  const ull i = (ull)c * stride * 32 + lane;
  const bool in = i < n;
  const bool st = in && ((__ldg(&recs[i].y) >> 23) & 1u);
  const unsigned b = __ballot_sync(FULL, st), v = __ballot_sync(FULL, in);
  if (lane == 0 && v) {
    atomicAdd(&out[0], (ull)__popc(v));
    atomicAdd(&out[1], (ull)__popc(b));
  }
}

void launch_head_sample(const uint4* recs, ull n, ull* out, cudaStream_t s) {
  const ull chunks = (n + 31) / 32;
  const uint32_t nsample = (uint32_t)std::min<ull>(chunks, 4096);
  const ull stride = chunks / nsample;
  head_sample_kernel<<<(nsample * 32 + 255) / 256, 256, 0, s>>>(recs, n, stride, nsample, out);
}

void launch_find_heads(const uint4* recs, ull n, ull range_len, uint32_t n_ranges, ull* heads, cudaStream_t s) {
  ull threads = ((ull)n_ranges + 1) * 32;
  find_heads_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(recs, n, range_len, n_ranges, heads);
}

// ---------------------------------------------------------------------------
// general decode kernel: deferred views (mixed warps / pcs / sizes, invalid or
// straddling records); one warp per view, grid-stride
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kDecWarps * 32) decode_general_kernel(DecodeArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const Smem sm = smem_setup(smem, a);
  const uint32_t nobj = a.obj.n;
  const int lane = threadIdx.x & 31;
  const unsigned lane_lt = lanemask_lt();
  const int wib = threadIdx.x >> 5;
  int steps = 0;
  while ((1u << steps) < nobj) ++steps;
  const uint32_t LW = a.kl.L + a.kl.W, P = a.kl.P;

  Stage st{reinterpret_cast<ull*>(sm.warp + wib * kWarpRegion), 0, a.seg_cnt, 8 + a.kl.P + a.kl.L + a.kl.W};
  ull n_invalid = 0, n_oor = 0, n_mapped = 0, n_unmapped = 0;
  uint32_t cur_launch = 0xFFFFFFFFu;

  // each warp takes a contiguous run of the deferred list (the fast kernel
  // appends a warp's views 32 at a time, in trace order); the descriptors of
  // the next 32 views are loaded together and the next view's records are in
  // flight while the current one is reduced
  const ull n_views = *((volatile ull*)&a.ctr->n_deferred);
  const ull gwarp = ((ull)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const ull nwarps = ((ull)gridDim.x * blockDim.x) >> 5;
  const ull per = ((n_views + 31) / 32 + nwarps - 1) / nwarps * 32;
  const ull v0 = gwarp * per < n_views ? gwarp * per : n_views;
  const ull v1 = v0 + per < n_views ? v0 + per : n_views;
  ull dq = 0, vb = v0, e_nxt = 0;
  uint4 nxt = make_uint4(0, 0, 0, 0);
  if (v0 < v1) {
    dq = v0 + lane < v1 ? a.deferred[v0 + lane] : 0ull;
    e_nxt = __shfl_sync(FULL, dq, 0);
    if (lane < (int)(e_nxt & 63)) nxt = ld_stream(&a.recs[(e_nxt >> 7) + lane]);
  }
  for (ull v = v0; v < v1; ++v) {
    // deferred view: p << 7 | stats_only << 6 | len (len <= 32).  stats_only:
    // the fast kernel already emitted this view's keys and word counters; only
    // the instruction statistics remain (a non-monotone instruction).  A view
    // may hold several whole instructions (short ones packed together by the
    // fast kernel): they start at the view's first record and at every
    // instr_start record inside it (G24)
    const ull e = e_nxt;
    const uint4 cur = nxt;
    if (v + 1 < v1) {
      if (v + 1 - vb >= 32) {
        vb = v + 1;
        dq = vb + lane < v1 ? a.deferred[vb + lane] : 0ull;
      }
      e_nxt = __shfl_sync(FULL, dq, (int)(v + 1 - vb));
      nxt = make_uint4(0, 0, 0, 0);
      if (lane < (int)(e_nxt & 63)) nxt = ld_stream(&a.recs[(e_nxt >> 7) + lane]);
    }
    const bool keys_too = ((e >> 6) & 1u) == 0;
    const uint32_t len = (uint32_t)(e & 63);
    const bool act = lane < (int)len;
    const ull af = ((ull)cur.y << 32) | cur.x;
    const uint32_t warp_id = cur.z, site = cur.w;
    const ull addr = af & ((1ull << 48) - 1);
    const uint32_t l2s = (cur.y >> 16) & 7u, kind = (cur.y >> 19) & 3u;
    const uint32_t space = (cur.y >> 21) & 3u, resv = cur.y >> 24;
    const ull size = 1ull << (l2s > 4 ? 0 : l2s);
    const bool traced = act && !out_of_scope(a, warp_id, site >> 20);  // sampled block, launch whitelist
    bool valid = traced && l2s <= 4 && kind <= 2 && space <= 2 && resv == 0 && addr + size <= (1ull << 48);
    const uint32_t launch = site >> 20;
    const bool oor = valid && (launch >= a.max_launches || warp_id >= a.max_warps);
    valid = valid && !oor;
    n_invalid += (traced && !valid && !oor) ? 1 : 0;
    n_oor += oor ? 1 : 0;
    const ull lo = ((ull)space << 48) | addr;
    const ull hi = lo + size - 1;
    const ull sa = lo >> 5, sbk = hi >> 5;
    const bool strad = sbk != sa;
    const uint32_t wa = (uint32_t)(lo >> 2) & 7u, wb = (uint32_t)(hi >> 2) & 7u;
    uint32_t ma = (0xFFu << wa) & 0xFFu;
    uint32_t mb = 0;
    if (strad) mb = 0xFFu >> (7 - wb); else ma &= 0xFFu >> (7 - wb);
    uint32_t ga = kNoG, gb = kNoG, fa = 0, fb = 0;
    int first_obj = -1;
    if (valid) {
      const int oa = obj_lookup(sm.lo, sm.hi, nobj, steps, sa << 5);
      if (oa >= 0) {
        fa = ma & allow_mask(sm.hi[oa], sa << 5);
        ga = (uint32_t)(sm.soff[oa] + (sa - (sm.lo[oa] >> 5)));
        if ((fa >> wa) & 1u) first_obj = oa;
      }
      if (strad) {
        const int ob = obj_lookup(sm.lo, sm.hi, nobj, steps, sbk << 5);
        if (ob >= 0) {
          fb = mb & allow_mask(sm.hi[ob], sbk << 5);
          gb = (uint32_t)(sm.soff[ob] + (sbk - (sm.lo[ob] >> 5)));
        }
      }
      if (keys_too) {
        if (launch != cur_launch) {
          flush_launch_ctr(a.launch_ctr, cur_launch, n_unmapped, n_mapped);
          cur_launch = launch;
        }
        const uint32_t mapped = __popc(fa) + __popc(fb);
        n_mapped += mapped;
        n_unmapped += __popc(ma) + __popc(mb) - mapped;
      }
    }
    if (!keys_too) { fa = fb = 0; }  // keys and counters came from the fast kernel
    if (a.acc) {  // access counts (track_access)
      for (uint32_t m = fa; m; m &= m - 1) atomicAdd(&a.acc[8ull * ga + (__ffs(m) - 1)], 1u);
      for (uint32_t m = fb; m; m &= m - 1) atomicAdd(&a.acc[8ull * gb + (__ffs(m) - 1)], 1u);
    }
    // pc id of each lane (usually one per view)
    uint32_t pcid = 0;
    if (a.track_pc) {
      const unsigned vb = __ballot_sync(FULL, fa | fb);
      if (vb) {
        const int f = __ffs(vb) - 1;
        const uint32_t sitef = __shfl_sync(FULL, site, f);
        const bool other = (fa | fb) && site != sitef;
        if (__ballot_sync(FULL, other) == 0) {
          uint32_t id = 0;
          if (lane == f) id = pc_lookup(sm.pc, a.pcmap, sitef, a.ctr);
          pcid = __shfl_sync(FULL, id, f);
        } else if (fa | fb) {
          pcid = pc_lookup(sm.pc, a.pcmap, site, a.ctr);
        }
      }
      if (pcid >= a.pcmap.max_pcs) pcid = 0;  // overflow is reported at build (ERANGE)
    }
    const ull lw = ((ull)launch << a.kl.W) | warp_id;
    {
      ull pa = fa ? (((((ull)ga << LW) | lw) << P) | pcid) : ~0ull;
      ull pb = fb ? (((((ull)gb << LW) | lw) << P) | pcid) : ~0ull;
      bool ha = fa != 0, hb = fb != 0;
      uint32_t mA = fa, mB = fb;
      // (the general kernel does not use the warp's record ring: its first 32
      // words are the merge scratch)
      uint32_t* const scr = reinterpret_cast<uint32_t*>(sm.warp + wib * kWarpRegion + kStage * sizeof(ull));
      group_merge(pa, mA, ha, scr, lane);
      if (__any_sync(FULL, hb)) group_merge(pb, mB, hb, scr, lane);
      STAGE_PUSH(st, ha, (pa << 8) | mA, a.keys, &a.ctr->n_keys);
      STAGE_PUSH(st, hb, (pb << 8) | mB, a.keys, &a.ctr->n_keys);
    }
    // instruction statistics, general case (G24), per
    // instruction of the view: lanes [s, e) between consecutive heads
    const unsigned hb = __ballot_sync(FULL, act && (lane == 0 || ((cur.y >> 23) & 1u)));
    const unsigned vbm = __ballot_sync(FULL, valid);
    if (vbm) {
      const unsigned le = lane_lt | (1u << lane);
      const int s0 = 31 - __clz(hb & le);  // this lane's instruction starts here (lane 0 is a head)
      const unsigned after = hb & ~le;
      const int e0 = after ? __ffs(after) - 1 : 32;
      const unsigned segm = (e0 >= 32 ? FULL : ((1u << e0) - 1u)) & ~((1u << s0) - 1u);
      const unsigned svalid = vbm & segm;
      const int f = svalid ? __ffs(svalid) - 1 : lane;
      const int i_obj = __shfl_sync(FULL, first_obj, f);
      const uint32_t i_launch = __shfl_sync(FULL, launch, f);
      // min / max byte over the instruction's valid records: segmented scans
      ull mn = valid ? lo : ~0ull, mx = valid ? hi : 0ull;
      uint32_t distinct;
      const bool any_strad = __ballot_sync(FULL, valid && strad) != 0;
      // every instruction of the view is one record (SpMV's divergent rows):
      // its min and max are its own bytes, and it touches one sector
      const bool all_single = !any_strad && __all_sync(FULL, !valid || segm == (1u << lane));
      // all valid bytes in one 4 GiB window (space, addr[32, 48)): 32-bit scans
      const uint32_t hw0 = __shfl_sync(FULL, (uint32_t)(lo >> 32), f);
      const bool win32 = __all_sync(FULL, !valid || (((uint32_t)(lo >> 32) == hw0) && ((uint32_t)(hi >> 32) == hw0)));
      if (all_single) {
        distinct = 1;
      } else if (win32 && !any_strad) {
        uint32_t mn32 = valid ? (uint32_t)lo : 0xFFFFFFFFu, mx32 = valid ? (uint32_t)hi : 0u;
        for (int d = 1; d < 32; d <<= 1) {
          const uint32_t omn = __shfl_down_sync(FULL, mn32, d), omx = __shfl_down_sync(FULL, mx32, d);
          if (lane + d < e0) { mn32 = omn < mn32 ? omn : mn32; mx32 = omx > mx32 ? omx : mx32; }
        }
        mn = ((ull)hw0 << 32) | mn32;
        mx = ((ull)hw0 << 32) | mx32;
        const unsigned m = __match_any_sync(FULL, valid ? ((uint32_t)lo >> 5) : (0xF8000000u | (uint32_t)lane));
        distinct = __popc(__ballot_sync(FULL, valid && (__ffs(m & segm) - 1 == lane)) & segm);
      } else {
        for (int d = 1; d < 32; d <<= 1) {
          const ull omn = __shfl_down_sync(FULL, mn, d), omx = __shfl_down_sync(FULL, mx, d);
          if (lane + d < e0) { mn = omn < mn ? omn : mn; mx = omx > mx ? omx : mx; }
        }
      }
      // (lane s0 now holds its instruction's min and max)
      if (all_single || (win32 && !any_strad)) {
      } else if (!any_strad) {
        const unsigned m = __match_any_sync(FULL, valid ? sa : (0xFFFF000000000000ull | (ull)lane));
        distinct = __popc(__ballot_sync(FULL, valid && (__ffs(m & segm) - 1 == lane)) & segm);
      } else {
        bool dup_a = false, dup_b = !strad;
        for (int j = 0; j < 32; ++j) {
          const ull aj = __shfl_sync(FULL, sa, j), bj = __shfl_sync(FULL, sbk, j);
          const bool vj = __shfl_sync(FULL, valid, j);
          if (vj && j < lane && j >= s0) {
            dup_a |= (sa == aj) || (sa == bj);
            dup_b |= (sbk == aj) || (sbk == bj);
          }
        }
        distinct = __popc(__ballot_sync(FULL, valid && !dup_a) & segm) +
                   __popc(__ballot_sync(FULL, valid && !dup_b) & segm);
      }
      const bool mis = svalid && i_obj >= 0 && distinct > (mx - mn + 1 + 31) / 32;
      const bool counted = svalid && i_obj >= 0;
      // counter updates aggregated over the view's instructions (lane s0 of
      // each holds its (launch, object) and misalignment): one update per
      // distinct (launch, object), by its lowest head lane
      const bool head = counted && lane == s0;
      const uint32_t key1 = head ? i_launch * nobj + (uint32_t)i_obj + 1u : 0u;
      const unsigned peers = __match_any_sync(FULL, key1);
      const unsigned misb = __ballot_sync(FULL, head && mis);
      if (head && lane == __ffs(peers) - 1)
        instr_add_n(sm, key1, (uint32_t)__popc(peers), (uint32_t)__popc(peers & misb), a.instr_ctr);
    }
  }
  st.flush(a.keys, &a.ctr->n_keys, lane);
  flush_launch_ctr(a.launch_ctr, cur_launch, n_unmapped, n_mapped);
  for (int d = 16; d; d >>= 1) {
    n_invalid += __shfl_xor_sync(FULL, n_invalid, d);
    n_oor += __shfl_xor_sync(FULL, n_oor, d);
  }
  if (lane == 0) {
    if (n_invalid) atomicAdd(&a.ctr->invalid, n_invalid);
    if (n_oor) atomicAdd(&a.ctr->out_of_range, n_oor);
  }
  smem_flush_instr(sm, a.instr_ctr);
}


size_t decode_smem(const DecodeArgs& a) {
  return kOffObj + (size_t)a.obj.n * 3 * sizeof(ull);
}



void launch_decode_general(const DecodeArgs& a, int num_sms, cudaStream_t s) {
  const size_t smem = decode_smem(a);
  smem_optin((const void*)decode_general_kernel, 200 * 1024);
  // the deferred count is read on the device: a full persistent grid (the
  // kernel waits on record loads, so every resident warp helps)
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, decode_general_kernel, kDecWarps * 32, smem);
  if (per_sm < 1) per_sm = 1;
  ull grid = (a.n_ranges + kDecWarps - 1) / kDecWarps;
  const ull cap = (ull)num_sms * per_sm;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  decode_general_kernel<<<(unsigned)grid, kDecWarps * 32, smem, s>>>(a);
}

}  // namespace thermo
