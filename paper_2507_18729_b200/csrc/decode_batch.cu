// decode_fast.cu -- the fast decode kernel (rows a2 + a3).
//
// Work mapping ("transposed"): a warp stages a batch of up to 1024 consecutive
// records in shared memory with coalesced 128-bit loads, finds the warp
// instructions in it (runs starting at instr_start, G24), and then each LANE
// walks one whole instruction sequentially -- scalar code with no warp
// collectives in the inner loop.  Per record: decode, object
// resolution through a per-lane object cache, word mask (P:324,
// G3/G4), merge with the previous record of the instruction (same sector ->
// OR the masks; P:325 is idempotent), insert of the (sector, launch, warp, pc)
// key into the warp's shared-memory dedup table, and the running
// distinct-sector / span statistics of the instruction.
//
// An instruction takes this path when all its records share warp, pc, launch,
// size, kind and space and none straddles a sector (what a collector emits
// for one instruction); otherwise it is deferred whole to
// decode_general_kernel (decode.cu).  A monotone-address instruction gets its
// misalignment test here; a non-monotone one is deferred "stats only".
#include "decode_common.cuh"

namespace thermo {

constexpr int kFW = 4;                 // warps per block
constexpr int kBatch = 1024;           // records per batch (32 chunks of 32)
constexpr int kBatchSlots = kBatch + kBatch / 32;  // one pad slot per 32 (bank spread)
constexpr int kFTab = 1024;            // dedup table entries per warp
constexpr int kFTabFlush = 512;        // flush at batch boundaries when this full
constexpr int kMaxInstr = 64;          // heads remembered per batch

__device__ __forceinline__ uint32_t slot_of(uint32_t idx) { return idx + (idx >> 5); }

// per-warp dedup table: full 56-bit key prefix -> word mask
struct FastTable {
  ull* key;        // [kFTab], ~0 = empty
  uint32_t* msk;   // [kFTab]
  __device__ __forceinline__ void init(ull* k, uint32_t* m, int lane) {
    key = k;
    msk = m;
    for (int i = lane; i < kFTab; i += 32) { key[i] = ~0ull; msk[i] = 0; }
    __syncwarp();
  }
  // lane-divergent insert; false if the table is full (caller emits directly)
  __device__ __forceinline__ bool insert(ull k, uint32_t m, uint32_t& fresh) {
    uint32_t h = ((uint32_t)k * 0x9E3779B1u ^ (uint32_t)(k >> 32) * 0x85EBCA6Bu) >> (32 - 10);
#pragma unroll 1
    for (int probe = 0; probe < 64; ++probe) {
      ull cur = key[h];
      if (cur == ~0ull) {
        cur = atomicCAS(&key[h], ~0ull, k);
        if (cur == ~0ull) { atomicOr(&msk[h], m); ++fresh; return true; }
      }
      if (cur == k) {
        if ((msk[h] & m) != m) atomicOr(&msk[h], m);
        return true;
      }
      h = (h + 1) & (kFTab - 1);
    }
    return false;
  }
  // emit every entry as a key (prefix << 8 | mask) and clear (warp-collective)
  __device__ __forceinline__ void flush(uint32_t count, ull* gkeys, ull* gcount, int lane) {
    __syncwarp();
    if (count == 0) return;
    ull base = 0;
    if (lane == 0) base = atomicAdd(gcount, (ull)count);
    base = __shfl_sync(FULL, base, 0);
    const unsigned lt = lanemask_lt();
    uint32_t pos = 0;
    for (int i = lane; i < kFTab; i += 32) {
      const ull k = key[i];
      const bool v = k != ~0ull;
      const unsigned b = __ballot_sync(FULL, v);
      if (v) {
        gkeys[base + pos + __popc(b & lt)] = (k << 8) | msk[i];
        key[i] = ~0ull;
        msk[i] = 0;
      }
      pos += __popc(b);
    }
    __syncwarp();
  }
};

// per-lane (launch, object) misalignment counter cache (lanes diverge)
struct LaneInstr {
  uint32_t k0, i0, m0;
  __device__ __forceinline__ void init() { k0 = 0; i0 = m0 = 0; }
  __device__ __forceinline__ void add(uint32_t key, uint32_t mis, uint32_t* s_ikey, ull* s_ival, ull* g) {
    if (key != k0) {
      if (k0) instr_flush(s_ikey, s_ival, g, k0, i0, m0);
      k0 = key; i0 = 0; m0 = 0;
    }
    ++i0;
    m0 += mis;
  }
  __device__ __forceinline__ void drain(uint32_t* s_ikey, ull* s_ival, ull* g) {
    if (k0) instr_flush(s_ikey, s_ival, g, k0, i0, m0);
    init();
  }
};

__device__ __forceinline__ void defer_view(const DecodeArgs& a, ull p, uint32_t len, bool stats_only) {
  const ull slot = atomicAdd(&a.ctr->n_deferred, 1ull);
  a.deferred[slot] = (p << 7) | ((ull)stats_only << 6) | len;
}

__global__ void __launch_bounds__(kFW * 32, 2) decode_fast_kernel(DecodeArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t nobj = a.obj.n;
  ull* s_lo = reinterpret_cast<ull*>(smem);
  ull* s_hi = s_lo + nobj;
  ull* s_soff = s_hi + nobj;
  ull* s_ival = s_soff + nobj;                                  // [kInstrSlots][2]
  ull* s_pc = s_ival + 2 * kInstrSlots;                         // [kPcSlots]
  uint32_t* s_ikey = reinterpret_cast<uint32_t*>(s_pc + kPcSlots);
  unsigned char* wbase = reinterpret_cast<unsigned char*>(s_ikey + kInstrSlots);
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const size_t per_warp = (size_t)kBatchSlots * 8 + (size_t)kFTab * 12 + kMaxInstr * 12 + 16;
  unsigned char* wreg = wbase + wib * per_warp;
  ull* buf = reinterpret_cast<ull*>(wreg);                                  // addr_flags per record
  ull* tkey = buf + kBatchSlots;
  uint32_t* tmsk = reinterpret_cast<uint32_t*>(tkey + kFTab);
  uint32_t* hstart = tmsk + kFTab;                                          // head record index
  uint32_t* hwarp = hstart + kMaxInstr;                                     // head's warp id
  uint32_t* hsite = hwarp + kMaxInstr;                                      // head's site
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
  const uint32_t LW = a.kl.L + a.kl.W, P = a.kl.P, W = a.kl.W;
  const uint32_t max_launches = a.max_launches, max_warps = a.max_warps;
  const unsigned lt = lanemask_lt();
  FastTable tab;
  tab.init(tkey, tmsk, lane);
  uint32_t tab_count = 0;  // warp-uniform
  LaneInstr li;
  li.init();
  ull n_mapped = 0, n_unmapped = 0;
  uint32_t cur_launch = 0xFFFFFFFFu;
  // per-lane object cache and (site -> pc id) cache
  ull olo = 1, ohi = 0, obase = 0;
  int oidx = -1;
  uint32_t csite = 0xFFFFFFFFu, cpcid = 0;

  const uint32_t gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t r = gwarp; r < a.n_ranges; r += nwarps) {
    const ull end = a.heads[r + 1];
    ull p = a.heads[r];
    while (p < end) {
      const uint32_t nrec = (uint32_t)(end - p < (ull)kBatch ? end - p : (ull)kBatch);
      // ---- stage: coalesced loads, head detection, predecessor check ----
      uint32_t nheads = 0;          // warp-uniform
      uint32_t pz = 0, pw = 0;      // previous chunk's last record warp / site
#pragma unroll 1
      for (uint32_t c0 = 0; c0 < 32; c0 += 8) {
        uint4 rr[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t idx = (c0 + u) * 32 + lane;
          rr[u] = idx < nrec ? ld_stream(&a.recs[p + idx]) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t idx = (c0 + u) * 32 + lane;
          const bool inb = idx < nrec;
          const bool head = inb & ((((rr[u].y >> 23) & 1u) != 0) | (idx == 0));
          const unsigned hb = __ballot_sync(FULL, head);
          uint32_t uz = __shfl_up_sync(FULL, rr[u].z, 1), uw = __shfl_up_sync(FULL, rr[u].w, 1);
          if (lane == 0) { uz = pz; uw = pw; }
          pz = __shfl_sync(FULL, rr[u].z, 31);
          pw = __shfl_sync(FULL, rr[u].w, 31);
          // bit 63 (a reserved bit) marks "warp or site differs from the predecessor"
          const bool diff = inb & !head & ((rr[u].z != uz) | (rr[u].w != uw));
          if (inb) buf[slot_of(idx)] = (((ull)rr[u].y << 32) | rr[u].x) | ((ull)diff << 63);
          if (head) {
            const uint32_t k = nheads + __popc(hb & lt);
            if (k < kMaxInstr) { hstart[k] = idx; hwarp[k] = rr[u].z; hsite[k] = rr[u].w; }
          }
          nheads += __popc(hb);
        }
      }
      __syncwarp();
      // complete instructions: those followed by another head, or all of them at the range end
      const uint32_t nh = nheads < kMaxInstr ? nheads : kMaxInstr;
      const bool at_end = p + nrec == end && nheads <= kMaxInstr;
      uint32_t ninst = at_end ? nh : (nh > 0 ? nh - 1 : 0);
      ninst = ninst < 32 ? ninst : 32;
      const uint32_t consumed = ninst < nh ? hstart[ninst] : nrec;
      if (ninst == 0) {
        // a run longer than the batch without instr_start: split every 32 (G24), defer
        if (lane == 0)
          for (uint32_t q = 0; q < nrec; q += 32) defer_view(a, p + q, nrec - q < 32 ? nrec - q : 32, false);
        p += nrec;
        continue;
      }
      // ---- lane i walks instruction i ----
      uint32_t fresh = 0;  // new table entries created by this lane
      if (lane < (int)ninst) {
        const uint32_t s = hstart[lane];
        const uint32_t e = (uint32_t)lane + 1 < nh ? hstart[lane + 1] : nrec;
        const uint32_t len = e - s;
        const ull y0 = buf[slot_of(s)];
        const uint32_t z0 = hwarp[lane], w0 = hsite[lane];
        const uint32_t yh = (uint32_t)(y0 >> 32);
        const uint32_t l2s = (yh >> 16) & 7u;
        const uint32_t launch = w0 >> 20;
        bool ok = (len <= 32) & (l2s <= 4) & (((yh >> 19) & 3u) != 3u) & (((yh >> 21) & 3u) != 3u) &
                  ((yh >> 24) == 0) & (launch < max_launches) & (z0 < max_warps);
        if (!ok) {
          for (uint32_t q = 0; q < len; q += 32) defer_view(a, p + s + q, len - q < 32 ? len - q : 32, false);
        } else {
          const uint32_t size = 1u << l2s;
          const ull spc = (ull)((yh >> 21) & 3u) << 48;
          const ull lwp = ((((ull)launch << W) | z0) << P);
          uint32_t pcid = 0;
          if (a.track_pc) {
            if (w0 != csite) { cpcid = pc_lookup(s_pc, a.pcmap, w0, a.ctr); csite = w0; }
            pcid = cpcid < a.pcmap.max_pcs ? cpcid : 0u;
          }
          uint32_t prev_g = kNoG, prev_m = 0;
          ull prev_lo = 0;
          uint32_t distinct = 0, mapped_w = 0, unmapped_w = 0;
          bool mono = true, first_mapped = false;
          int first_obj = -1;
          uint32_t j = 0;
          for (; j < len; ++j) {
            const ull af = buf[slot_of(s + j)];
            const uint32_t yj = (uint32_t)(af >> 32), xj = (uint32_t)af;
            // uniform with the head, no straddle, no overflow, same warp/site as predecessor
            if (((yj ^ yh) & 0xFF7F0000u) | (uint32_t)((xj & 31u) + size > 32u) |
                (uint32_t)((yj & 0xFFFFu) == 0xFFFFu) | (uint32_t)(af >> 63))
              break;
            const ull lo = spc | (af & 0xFFFFFFFFFFFFull);
            const ull xs = lo & ~31ull;
            if (!((xs >= olo) & (xs < ohi))) {
              const int o = obj_lookup(s_lo, s_hi, nobj, steps, xs);
              oidx = o;
              if (o >= 0) { olo = s_lo[o]; ohi = s_hi[o]; obase = s_soff[o] - (s_lo[o] >> 5); }
              else { olo = 1; ohi = 0; obase = 0; }
            }
            const uint32_t wa = (xj >> 2) & 7u, wb = ((xj + size - 1u) >> 2) & 7u;
            const uint32_t ma = (0xFFu << wa) & (0xFFu >> (7u - wb));
            const bool mapped = (xs >= olo) & (xs < ohi);
            const ull lim = ohi - xs;
            const uint32_t allow = lim >= 32 ? 0xFFu : ((1u << ((uint32_t)(lim + 3) >> 2)) - 1u);
            const uint32_t fa = mapped ? (ma & allow) : 0u;
            mapped_w += __popc(fa);
            unmapped_w += __popc(ma) - __popc(fa);
            if (j == 0) { first_mapped = (fa >> wa) & 1u; first_obj = mapped ? oidx : -1; }
            // merge with the previous record's sector, else hand that one to the table
            const uint32_t g = (uint32_t)((xs >> 5) + obase);
            if (fa) {
              if (g == prev_g) {
                prev_m |= fa;
              } else {
                if (prev_m && !tab.insert(((ull)prev_g << (LW + P)) | lwp | pcid, prev_m, fresh)) {
                  const ull at = atomicAdd(&a.ctr->n_keys, 1ull);
                  a.keys[at] = ((((ull)prev_g << (LW + P)) | lwp | pcid) << 8) | prev_m;
                }
                prev_g = g;
                prev_m = fa;
              }
            }
            // instruction statistics (monotone addresses)
            mono = mono & ((j == 0) | (lo >= prev_lo));
            distinct += ((j == 0) | ((lo >> 5) != (prev_lo >> 5))) ? 1u : 0u;
            prev_lo = lo;
          }
          if (prev_m && !tab.insert(((ull)prev_g << (LW + P)) | lwp | pcid, prev_m, fresh)) {
            const ull at = atomicAdd(&a.ctr->n_keys, 1ull);
            a.keys[at] = ((((ull)prev_g << (LW + P)) | lwp | pcid) << 8) | prev_m;
          }
          // a break at j < len: a record differs from the head (non-uniform instruction)
          const bool uniform = j == len;
          if (!uniform) {
            defer_view(a, p + s, len, false);  // keys emitted so far are correct duplicates
          } else {
            if (launch != cur_launch) {
              flush_launch_ctr(a.launch_ctr, cur_launch, n_unmapped, n_mapped);
              cur_launch = launch;
            }
            n_mapped += mapped_w;
            n_unmapped += unmapped_w;
            if (!mono) {
              defer_view(a, p + s, len, true);  // exact distinct sectors in the general kernel
            } else if (first_obj >= 0 && first_mapped) {
              const ull span = prev_lo - (spc | (buf[slot_of(s)] & 0xFFFFFFFFFFFFull)) + size;
              li.add(launch * nobj + (uint32_t)first_obj + 1u, distinct > (span + 31) / 32 ? 1u : 0u, s_ikey,
                     s_ival, a.instr_ctr);
            }
          }
        }
      }
      tab_count += __reduce_add_sync(FULL, fresh);  // implies __syncwarp
      p += consumed;
      if (tab_count > (uint32_t)kFTabFlush) {
        tab.flush(tab_count, a.keys, &a.ctr->n_keys, lane);
        tab_count = 0;
      }
    }
  }
  tab.flush(tab_count, a.keys, &a.ctr->n_keys, lane);
  li.drain(s_ikey, s_ival, a.instr_ctr);
  flush_launch_ctr(a.launch_ctr, cur_launch, n_unmapped, n_mapped);
  __syncthreads();
  for (int i = threadIdx.x; i < kInstrSlots; i += blockDim.x) {
    const uint32_t k = s_ikey[i];
    if (k) {
      atomicAdd(&a.instr_ctr[2 * (k - 1)], s_ival[2 * i]);
      if (s_ival[2 * i + 1]) atomicAdd(&a.instr_ctr[2 * (k - 1) + 1], s_ival[2 * i + 1]);
    }
  }
}

static size_t fast_smem(const DecodeArgs& a) {
  const size_t per_warp = (size_t)kBatchSlots * 8 + (size_t)kFTab * 12 + kMaxInstr * 12 + 16;
  return (size_t)a.obj.n * 3 * sizeof(ull) + 2 * kInstrSlots * sizeof(ull) + kPcSlots * sizeof(ull) +
         kInstrSlots * sizeof(uint32_t) + kFW * per_warp;
}

void launch_decode_batch(const DecodeArgs& a, int num_sms, cudaStream_t s) {
  const size_t smem = fast_smem(a);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(decode_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, decode_fast_kernel, kFW * 32, smem);
  if (per_sm < 1) per_sm = 1;
  const ull want = ((ull)a.n_ranges + kFW - 1) / kFW;
  ull grid = (ull)num_sms * per_sm;
  if (want < grid) grid = want;
  if (grid < 1) grid = 1;
  decode_fast_kernel<<<(unsigned)grid, kFW * 32, smem, s>>>(a);
}

}  // namespace thermo
