// indicators.cu -- row a7: the per-object pattern indicators and labels read
// from the heat map (§IV-C; rules S:356-409 as exact integer
// inequalities).
//
//   per touched sector (c = sector count, mw = max word count):
//     hot       c >= theta_hot and alpha_den*c <= alpha_num*mw
//     false-sh. beta_den*c >= beta_num*mw and c >= fs_min
//   per object: T, TW, hot, fs, sum x, sum x^2 (u128), words <= smem_cap,
//   max sector count, gaps between consecutive touched words and the gap value
//   holding a strict majority (parallel Boyer-Moore vote + exact verify count;
//   exact because any value with >= 3/4 of the gaps is the majority), and the
//   misalignment counters gathered by the decoder.
//
// Tiles never span objects: tile t covers sectors [tile_first, tile_end) of
// object tile_obj.  Pass 1 (mode 0) accumulates sums and per-tile votes, the
// stitch kernel orders tiles per object (cross-tile gaps, vote merge), pass 2
// (mode 1) counts the gaps equal to the object's candidate, finalize applies
// the label rules.
#include "thermo_internal.cuh"

namespace thermo {

constexpr unsigned IFULL = 0xFFFFFFFFu;
constexpr int kIndThreads = 256;
constexpr int kSecPerThread = 8;
constexpr ull kNone = ~0ull;
typedef unsigned __int128 u128;

struct Vote {
  ull c, n;
};
__device__ __forceinline__ Vote vote_merge(Vote a, Vote b) {
  if (a.n == 0) return b;
  if (b.n == 0) return a;
  if (a.c == b.c) return Vote{a.c, a.n + b.n};
  return a.n >= b.n ? Vote{a.c, a.n - b.n} : Vote{b.c, b.n - a.n};
}
__device__ __forceinline__ void vote_add(Vote& v, ull x) { v = vote_merge(v, Vote{x, 1}); }
__device__ __forceinline__ Vote warp_vote(Vote v) {
  for (int d = 16; d; d >>= 1) {
    Vote o{__shfl_xor_sync(IFULL, v.c, d), __shfl_xor_sync(IFULL, v.n, d)};
    v = vote_merge(v, o);
  }
  return v;
}
__device__ __forceinline__ ull warp_sum(ull v) {
  for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(IFULL, v, d);
  return v;
}
__device__ __forceinline__ ull warp_max(ull v) {
  for (int d = 16; d; d >>= 1) { ull o = __shfl_xor_sync(IFULL, v, d); v = o > v ? o : v; }
  return v;
}
__device__ __forceinline__ ull warp_min(ull v) {
  for (int d = 16; d; d >>= 1) { ull o = __shfl_xor_sync(IFULL, v, d); v = o < v ? o : v; }
  return v;
}

__device__ __forceinline__ void atomic_add_u128(ull* lo, ull* hi, u128 v) {
  ull vlo = (ull)v, vhi = (ull)(v >> 64);
  ull old = atomicAdd(lo, vlo);
  if (old + vlo < old) vhi += 1;  // carry
  if (vhi) atomicAdd(hi, vhi);
}

// exclusive "last touched position before me" across the block: max-scan,
// positions grow with the thread index so max == nearest previous
__device__ ull block_prev_last(ull last_or_none, ull* s_w) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  ull v = last_or_none == kNone ? 0 : last_or_none + 1;  // 0 = none
  ull incl = v;
  for (int d = 1; d < 32; d <<= 1) {
    ull o = __shfl_up_sync(IFULL, incl, d);
    if (lane >= d) incl = o > incl ? o : incl;
  }
  if (lane == 31) s_w[w] = incl;
  __syncthreads();
  ull carry = 0;
  for (int i = 0; i < w; ++i) carry = s_w[i] > carry ? s_w[i] : carry;
  __syncthreads();
  ull ex = __shfl_up_sync(IFULL, incl, 1);
  if (lane == 0) ex = 0;
  ex = ex > carry ? ex : carry;
  return ex == 0 ? kNone : ex - 1;
}

// mode 0: sums + votes; mode 1: verify count of gaps == candidate
__global__ void __launch_bounds__(kIndThreads, 4) indicator_tile_kernel(IndicatorArgs a, int mode) {
  __shared__ ull s_w[kIndThreads / 32];
  __shared__ ull s_red[kIndThreads / 32][13];
  const uint32_t tile = blockIdx.x;
  const uint32_t o = (uint32_t)a.tile_obj[tile];
  const ull g0 = a.tile_first[tile], g1 = a.tile_end[tile];
  if (shard_owner(g0, a.nranks) != a.rank) {  // another rank's tile (sharded mode)
    if (mode == 0 && threadIdx.x < kTileInfo) a.tile_info[(ull)tile * kTileInfo + threadIdx.x] = 0;  // sum identity
    return;
  }
  if (mode == 1) {
    // a tile whose gaps all equal the object's candidate (its vote never lost
    // a count: cnt = touched words - 1) needs no re-scan: its verify count is
    // its gaps, plus the gap from the previous touched word if that is equal
    const ull* ti = a.tile_info + (ull)tile * kTileInfo;
    const ull cand0 = a.ind[(ull)o * kIndFields + F_CAND];
    if (a.ind[(ull)o * kIndFields + F_CANDCNT] == 0) return;
    const ull tw = ti[4];
    if (tw == 0) return;
    if (ti[2] == cand0 && ti[3] == tw - 1) {
      if (threadIdx.x == 0) {
        const ull tp = a.tile_prev[tile];
        const ull v = (tw - 1) + ((tp != kNone && ti[0] - tp == cand0) ? 1 : 0);
        if (v) atomicAdd(&a.ind[(ull)o * kIndFields + F_VERIFY], v);
      }
      return;
    }
  }
  const ull soff = a.obj.soff[o];
  const ull nw = a.obj_nwords[o];
  const thermo_params& P = a.prm;
  // the rows of an owned tile (one 2048-sector chunk) at their local index
  const long long ldelta = (long long)shard_local(g0, a.nranks) - (long long)g0;
  const uint32_t* const sector_cnt = a.sector_cnt + ldelta;
  const uint32_t* const word_cnt = a.word_cnt + 8 * ldelta;
  const ull cand = mode ? a.ind[(ull)o * kIndFields + F_CAND] : 0;
  // no surviving vote: no gap holds a majority, the verify count is not needed
  if (mode == 1 && a.ind[(ull)o * kIndFields + F_CANDCNT] == 0) return;

  // Boyer-Moore summaries of the gaps inside one sector, by its touched-word
  // mask: the gaps between consecutive set bits of m, voted in order (any
  // pairing summary keeps a strict majority as its candidate, and the later
  // count / bounds are exact): s_bm[m] = candidate << 4 | count
  __shared__ uint8_t s_bm[256];
  {
    const uint32_t m = threadIdx.x & 255u;
    uint32_t c = 0, n = 0;
    for (uint32_t r = m; r & (r - 1); r &= r - 1) {
      const uint32_t gap = (uint32_t)(__ffs(r & (r - 1)) - __ffs(r));
      if (n == 0) { c = gap; n = 1; } else if (c == gap) ++n; else --n;
    }
    if (threadIdx.x < 256) s_bm[m] = (uint8_t)((c << 4) | n);
  }
  __syncthreads();
  uint32_t T = 0, TW = 0, hot = 0, fs = 0, le1 = 0, maxsec = 0;
  ull sumx = 0, verify = 0;
  u128 sumx2 = 0;
  Vote vt{0, 0};
  ull first = kNone, last = kNone;
  const ull gs = g0 + (ull)threadIdx.x * kSecPerThread;
  // software pipeline: the next sector's count and 8 word counts (two 16-byte
  // loads; rows are 32-byte aligned) are in flight while this one is scanned
  uint32_t c_n = 0;
  uint4 lo_n = make_uint4(0, 0, 0, 0), hi_n = lo_n;
  if (gs < g1) {
    c_n = sector_cnt[gs];
    lo_n = reinterpret_cast<const uint4*>(word_cnt + 8 * gs)[0];
    hi_n = reinterpret_cast<const uint4*>(word_cnt + 8 * gs)[1];
  }
  const uint32_t smem_cap = (uint32_t)(P.smem_cap < 0xFFFFFFFFull ? P.smem_cap : 0xFFFFFFFFull);
  for (int i = 0; i < kSecPerThread; ++i) {
    const ull g = gs + i;
    if (g >= g1) break;
    const uint32_t c = c_n;
    const uint4 lo = lo_n, hi = hi_n;
    if (i + 1 < kSecPerThread && g + 1 < g1) {
      c_n = sector_cnt[g + 1];
      lo_n = reinterpret_cast<const uint4*>(word_cnt + 8 * (g + 1))[0];
      hi_n = reinterpret_cast<const uint4*>(word_cnt + 8 * (g + 1))[1];
    }
    const uint32_t xs[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
    const ull wl0 = (g - soff) * 8;
    // the object's words of this sector (its partial last sector, G9)
    const uint32_t vm = wl0 + 8 <= nw ? 0xFFu : (wl0 >= nw ? 0u : (1u << (uint32_t)(nw - wl0)) - 1u);
    uint32_t mw = 0, tm = 0, lm = 0;
    ull s1 = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const uint32_t x = ((vm >> b) & 1u) ? xs[b] : 0u;
      mw = x > mw ? x : mw;
      tm |= (x != 0u) << b;
      lm |= (x != 0u && x <= smem_cap) << b;
      s1 += x;
    }
    if (tm) {
      TW += __popc(tm);
      le1 += __popc(lm);
      sumx += s1;
      if (mw < (1u << 30)) {  // 8 squares below 2^63: one 64-bit sum per sector
        ull s2 = 0;
#pragma unroll
        for (int b = 0; b < 8; ++b) s2 += ((vm >> b) & 1u) ? (ull)xs[b] * xs[b] : 0ull;
        sumx2 += s2;
      } else {
#pragma unroll
        for (int b = 0; b < 8; ++b) sumx2 += ((vm >> b) & 1u) ? (u128)((ull)xs[b] * xs[b]) : (u128)0;
      }
      const ull wf = wl0 + (uint32_t)(__ffs(tm) - 1);
      if (last != kNone) {  // the gap from the previous touched word of this thread
        const ull gap = wf - last;
        if (mode == 0) vote_add(vt, gap);
        verify += gap == (mode == 0 ? 1ull : cand) ? 1 : 0;  // (mode 0: the gaps of 1, exactly)
      } else {
        first = wf;
      }
      if (mode == 0) {  // the gaps inside the sector: their summary, their 1s
        const uint32_t e = s_bm[tm];
        if (e & 15u) vt = vote_merge(vt, Vote{(ull)(e >> 4), (ull)(e & 15u)});
        verify += __popc(tm & (tm >> 1));
      } else if (cand < 8) {
        for (uint32_t r = tm; r & (r - 1); r &= r - 1)
          verify += (ull)(__ffs(r & (r - 1)) - __ffs(r)) == cand ? 1 : 0;
      }
      last = wl0 + (uint32_t)(31 - __clz(tm));
    }
    if (c == 0) continue;
    ++T;
    maxsec = c > maxsec ? c : maxsec;
    if (c >= P.theta_hot && P.alpha_den * c <= P.alpha_num * (ull)mw) ++hot;
    if (P.beta_den * c >= P.beta_num * (ull)mw && c >= P.fs_min) ++fs;
  }
  // gap from the previous touched word in this tile (another thread)
  const ull prev = block_prev_last(last, s_w);
  if (first != kNone && prev != kNone) {
    const ull gap = first - prev;
    if (mode == 0) vote_add(vt, gap);
    verify += gap == (mode == 0 ? 1ull : cand) ? 1 : 0;
  }
  // the tile's first gap (crossing the previous tile) in verify mode
  if (mode == 1 && first != kNone && prev == kNone) {
    const ull tp = a.tile_prev[tile];
    if (tp != kNone) verify += (first - tp) == cand ? 1 : 0;
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (mode == 1) {
    verify = warp_sum(verify);
    if (lane == 0) s_red[w][0] = verify;
    __syncthreads();
    if (threadIdx.x == 0) {
      ull s = 0;
      for (int i = 0; i < kIndThreads / 32; ++i) s += s_red[i][0];
      if (s) atomicAdd(&a.ind[(ull)o * kIndFields + F_VERIFY], s);
    }
    return;
  }
  // ---- block reduction of the sums and votes ----
  T = warp_sum(T); TW = warp_sum(TW); hot = warp_sum(hot); fs = warp_sum(fs); sumx = warp_sum(sumx);
  le1 = warp_sum(le1); maxsec = warp_max(maxsec);
  ull s2lo = (ull)sumx2, s2hi = (ull)(sumx2 >> 64);
  for (int d = 16; d; d >>= 1) {  // u128 warp sum
    ull olo = __shfl_xor_sync(IFULL, s2lo, d), ohi = __shfl_xor_sync(IFULL, s2hi, d);
    ull nlo = s2lo + olo;
    s2hi = s2hi + ohi + (nlo < s2lo ? 1 : 0);
    s2lo = nlo;
  }
  vt = warp_vote(vt);
  verify = warp_sum(verify);
  const ull tfirst = warp_min(first);
  const ull tlast = warp_max(last == kNone ? 0 : last + 1);
  if (lane == 0) {
    ull* r = s_red[w];
    r[0] = T; r[1] = TW; r[2] = hot; r[3] = fs; r[4] = sumx; r[5] = le1; r[6] = maxsec;
    r[7] = s2lo; r[8] = s2hi; r[9] = vt.c; r[10] = vt.n; r[11] = tfirst; r[12] = verify;
    s_w[w] = tlast;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    ull acc[12] = {0};
    acc[11] = kNone;
    Vote bv{0, 0};
    ull bl = 0, ones = 0;
    u128 s2 = 0;
    for (int i = 0; i < kIndThreads / 32; ++i) {
      const ull* r = s_red[i];
      ones += r[12];
      for (int f = 0; f < 6; ++f) acc[f] += r[f];
      acc[6] = r[6] > acc[6] ? r[6] : acc[6];
      s2 += ((u128)r[8] << 64) | r[7];
      bv = vote_merge(bv, Vote{r[9], r[10]});
      acc[11] = r[11] < acc[11] ? r[11] : acc[11];
      bl = s_w[i] > bl ? s_w[i] : bl;
    }
    ull* ind = a.ind + (ull)o * kIndFields;
    if (acc[0]) atomicAdd(&ind[F_T], acc[0]);
    if (acc[1]) atomicAdd(&ind[F_TW], acc[1]);
    if (acc[2]) atomicAdd(&ind[F_HOT], acc[2]);
    if (acc[3]) atomicAdd(&ind[F_FS], acc[3]);
    if (acc[4]) atomicAdd(&ind[F_SUMX], acc[4]);
    if (acc[5]) atomicAdd(&ind[F_LE1], acc[5]);
    if (acc[6]) atomicMax(&ind[F_MAXSEC], acc[6]);
    if (s2) atomic_add_u128(&ind[F_SUMX2_LO], &ind[F_SUMX2_HI], s2);
    ull* ti = a.tile_info + (ull)tile * kTileInfo;
    ti[0] = acc[11];
    ti[1] = bl == 0 ? kNone : bl - 1;
    ti[2] = bv.c;
    ti[3] = bv.n;
    ti[4] = acc[1];
    ti[5] = ones;
  }
}

// one block per object: order the object's tiles, add the cross-tile gaps to
// the vote, merge the tile votes, record each tile's predecessor word
constexpr int kStitchT = 1024;  // a block per object walks its tiles in order, 1024 at a time
__global__ void __launch_bounds__(kStitchT) indicator_stitch_kernel(IndicatorArgs a, const uint32_t* obj_tile0) {
  __shared__ ull s_w[kStitchT / 32];
  __shared__ ull s_vc[kStitchT / 32], s_vn[kStitchT / 32];
  __shared__ ull s_carry;
  const uint32_t o = blockIdx.x;
  const uint32_t t0 = obj_tile0[o], t1 = obj_tile0[o + 1];
  if (threadIdx.x == 0) s_carry = kNone;
  __syncthreads();
  Vote vt{0, 0};
  for (uint32_t base = t0; base < t1; base += kStitchT) {
    const uint32_t t = base + threadIdx.x;
    ull first = kNone, last = kNone;
    Vote tv{0, 0};
    if (t < t1) {
      const ull* ti = a.tile_info + (ull)t * kTileInfo;
      first = ti[0]; last = ti[1]; tv = Vote{ti[2], ti[3]};
    }
    ull prev = block_prev_last(last, s_w);
    const ull carry = s_carry;
    if (prev == kNone) prev = carry;
    if (t < t1) {
      a.tile_prev[t] = prev;
      vt = vote_merge(vt, tv);
      if (first != kNone && prev != kNone) vote_add(vt, first - prev);
    }
    // new carry = last touched in this chunk (or the old carry)
    ull cl = warp_max(last == kNone ? 0 : last + 1);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) s_w[w] = cl;
    __syncthreads();
    if (threadIdx.x == 0) {
      ull m = 0;
      for (int i = 0; i < kStitchT / 32; ++i) m = s_w[i] > m ? s_w[i] : m;
      if (m) s_carry = m - 1;
    }
    __syncthreads();
  }
  vt = warp_vote(vt);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) { s_vc[w] = vt.c; s_vn[w] = vt.n; }
  __syncthreads();
  if (threadIdx.x == 0) {
    Vote v{0, 0};
    for (int i = 0; i < kStitchT / 32; ++i) v = vote_merge(v, Vote{s_vc[i], s_vn[i]});
    s_vc[0] = v.c;
    s_vn[0] = v.n;
  }
  __syncthreads();
  const ull x = s_vc[0], xn = s_vn[0];
  // An upper bound on the candidate's gap count, from the tile summaries: a
  // Boyer-Moore summary (c, n) of N values was formed by cancelling pairs of
  // different values, so a value v occurs at most (N + n) / 2 times if v == c
  // and n > 0, else at most (N - n) / 2; each cross-tile gap counts 1 if it
  // equals the candidate.  When twice the bound is at most the object's gap
  // count, no gap value can hold a strict majority: the verify scan is
  // skipped (F_CANDCNT = 0) and no dominant gap is reported, as with the count
  // A candidate of 1 (every word after the previous one: the contiguous
  // pattern) needs no verify scan either: the tiles counted their gaps of 1
  // exactly (tile_info[5]), plus the cross-tile gaps of 1 -- F_VERIFY directly
  // (rank 0's copy: the sharded mode sums the ranks' verify counts)
  ull ub = 0, ng = 0, n1 = 0;
  if (xn) {
    for (uint32_t t = t0 + threadIdx.x; t < t1; t += kStitchT) {
      const ull* ti = a.tile_info + (ull)t * kTileInfo;
      const ull G = ti[4] ? ti[4] - 1 : 0;  // the tile's own gaps (touched words - 1)
      const ull c = ti[2], n = ti[3];
      ub += (n && c == x) ? (G + n) / 2 : (G - n) / 2;
      ng += G;
      n1 += ti[5];
      const ull first = ti[0], prev = a.tile_prev[t];
      if (first != kNone && prev != kNone) {
        ++ng;
        ub += first - prev == x ? 1 : 0;
        n1 += first - prev == 1 ? 1 : 0;
      }
    }
  }
  ub = warp_sum(ub);
  ng = warp_sum(ng);
  n1 = warp_sum(n1);
  __syncthreads();
  if (lane == 0) { s_w[w] = ub; s_vn[w] = ng; s_vc[w] = n1; }
  __syncthreads();
  if (threadIdx.x == 0) {
    ull U = 0, N = 0, N1 = 0;
    for (int i = 0; i < kStitchT / 32; ++i) { U += s_w[i]; N += s_vn[i]; N1 += s_vc[i]; }
    ull* ind = a.ind + (ull)o * kIndFields;
    const bool possible = xn && 2 * U > N;
    ind[F_CAND] = possible ? x : 0;
    ind[F_CANDCNT] = possible && x != 1 ? xn : 0;  // 0: no verify scan of this object
    if (possible && x == 1) ind[F_VERIFY] = a.rank == 0 ? N1 : 0;
  }
}

// labels (one thread per object)
__global__ void indicator_finalize_kernel(IndicatorArgs a) {
  const uint32_t o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= a.obj.n) return;
  ull* r = a.ind + (ull)o * kIndFields;
  const thermo_params& P = a.prm;
  r[F_NWORDS] = a.obj_nwords[o];
  r[F_NSECTORS] = a.obj.soff[o + 1] - a.obj.soff[o];
  ull instrs = 0, mis = 0;
  for (uint32_t la = 0; la < a.max_launches; ++la) {
    if (a.launch_filter != THERMO_ALL_LAUNCHES && la != a.launch_filter) continue;
    const ull* c = a.instr_ctr + 2 * ((ull)la * a.obj.n + o);
    instrs += c[0];
    mis += c[1];
  }
  r[F_INSTRS] = instrs;
  r[F_MIS] = mis;
  const ull T = r[F_T], TW = r[F_TW];
  const ull gaps = TW ? TW - 1 : 0;
  r[F_GAPS] = gaps;
  const ull ver = r[F_VERIFY];
  if (gaps && 2 * ver > gaps) { r[F_DOMGAP] = r[F_CAND]; r[F_DOMCNT] = ver; }
  else { r[F_DOMGAP] = 0; r[F_DOMCNT] = 0; }
  uint32_t L = 0;
  if (T >= 1 && P.hot_frac_den * r[F_HOT] >= P.hot_frac_num * T) {
    const u128 S1 = r[F_SUMX], n = TW;
    const u128 S2 = ((u128)r[F_SUMX2_HI] << 64) | r[F_SUMX2_LO];
    const u128 var_num = n * S2 - S1 * S1;
    const u128 lhs = (u128)P.cv_den * P.cv_den * var_num;
    const u128 rhs = (u128)P.cv_num * P.cv_num * S1 * S1;
    L |= (TW >= 1 && lhs > rhs) ? THERMO_LABEL_RANDOM_HOT : THERMO_LABEL_HOT;
  }
  const bool global = a.obj_space[o] == 0;
  if (global && T >= 1 && P.fs_frac_den * r[F_FS] >= P.fs_frac_num * T) L |= THERMO_LABEL_FALSE_SHARING;
  if (a.obj_space[o] == 1 && TW >= 1 && P.smem_cov_den * r[F_LE1] >= P.smem_cov_num * TW)
    L |= r[F_MAXSEC] == 1 ? THERMO_LABEL_SMEM_THREAD_LOCAL : THERMO_LABEL_SMEM_WARP_PRIVATE;
  if (instrs >= 1 && P.mis_frac_den * mis >= P.mis_frac_num * instrs) L |= THERMO_LABEL_MISALIGNED;
  if (global && T >= P.strided_min_sectors && P.gamma_den * TW <= P.gamma_num * 8 * T && gaps >= 1 &&
      P.dom_den * r[F_DOMCNT] >= P.dom_num * gaps)
    L |= THERMO_LABEL_STRIDED;
  r[F_LABELS] = L;
}

// sharded mode: per-object partial sums <-> reducible arrays
__global__ void indicator_pack_kernel(ull* ind, uint32_t n, ull* sums, ull* maxs, ull* verify, int dir) {
  const uint32_t o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= n) return;
  ull* r = ind + (ull)o * kIndFields;
  static constexpr int kSumF[6] = {F_T, F_TW, F_HOT, F_FS, F_SUMX, F_LE1};
  if (dir == 0) {
    if (sums) {
      ull* d = sums + (ull)o * kIndSumFields;
      for (int f = 0; f < 6; ++f) d[f] = r[kSumF[f]];
      d[6] = r[F_SUMX2_LO] & 0xFFFFFFFFull; d[7] = r[F_SUMX2_LO] >> 32;
      d[8] = r[F_SUMX2_HI] & 0xFFFFFFFFull; d[9] = r[F_SUMX2_HI] >> 32;
      maxs[o] = r[F_MAXSEC];
    }
    if (verify) verify[o] = r[F_VERIFY];
  } else {
    if (sums) {
      const ull* d = sums + (ull)o * kIndSumFields;
      for (int f = 0; f < 6; ++f) r[kSumF[f]] = d[f];
      const u128 v = (u128)d[6] + ((u128)d[7] << 32) + ((u128)d[8] << 64) + ((u128)d[9] << 96);
      r[F_SUMX2_LO] = (ull)v;
      r[F_SUMX2_HI] = (ull)(v >> 64);
      r[F_MAXSEC] = maxs[o];
    }
    if (verify) r[F_VERIFY] = verify[o];
  }
}

void launch_indicator_pack(ull* ind, uint32_t n, ull* sums, ull* maxs, ull* verify, int dir, cudaStream_t s) {
  indicator_pack_kernel<<<(n + 127) / 128, 128, 0, s>>>(ind, n, sums, maxs, verify, dir);
}

void launch_indicator_tiles(const IndicatorArgs& a, int mode, cudaStream_t s) {
  if (a.n_tiles) indicator_tile_kernel<<<a.n_tiles, kIndThreads, 0, s>>>(a, mode);
}

void launch_indicator_stitch(const IndicatorArgs& a, cudaStream_t s) {
  // obj_tile0: first tile of each object, derived from tile_obj on the host side
  // and stored right after tile_prev (see thermo_api.cu)
  const uint32_t* obj_tile0 = reinterpret_cast<const uint32_t*>(a.tile_prev + a.n_tiles);
  indicator_stitch_kernel<<<a.obj.n, kStitchT, 0, s>>>(a, obj_tile0);
}

void launch_indicator_finalize(const IndicatorArgs& a, cudaStream_t s) {
  indicator_finalize_kernel<<<(a.obj.n + 127) / 128, 128, 0, s>>>(a);
}

void launch_indicators(const IndicatorArgs& a, int num_sms, cudaStream_t s) {
  (void)num_sms;
  launch_indicator_tiles(a, 0, s);
  launch_indicator_stitch(a, s);
  launch_indicator_tiles(a, 1, s);
  launch_indicator_finalize(a, s);
}

}  // namespace thermo
