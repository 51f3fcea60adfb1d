// thermo_internal.cuh -- shared declarations of libthermo's CUDA implementation.
//
// Citation keys: P:n = PAPER.md line n; S:n = SPEC.md line n; G# = DESIGN.md
// "Readings".  Nothing in this directory includes or links anything under
// oracle/ (the test oracle); the two share no code.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <mutex>
#include <set>
#include <string>
#include <utility>
#include <unordered_map>
#include <vector>

#include "../../include/thermo.h"

namespace thermo {

typedef unsigned long long ull;

constexpr int kLevels = THERMO_LEVELS;
constexpr ull kEmptyKey = ~0ull;  // sentinel key (prefix all-ones is reserved)
constexpr uint32_t kPcNone = 0xFFFFFFFFu;

// Opt a kernel in to `bytes` of dynamic shared memory on the CURRENT device.
// cudaFuncSetAttribute applies per device (context), so the opt-in is cached per
// (kernel, device) under a lock: contexts on several devices, or in-process
// shards driven from several host threads, each get it exactly once.
inline void smem_optin(const void* func, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (done.insert(std::make_pair(func, dev)).second)
    cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

// ---- device-resident counters (one struct per context) -------------------
struct DevCounters {
  ull n_keys;          // main keys emitted (after pre-dedup)
  ull n_pckeys;        // pc keys emitted
  ull invalid;         // invalid records
  ull out_of_range;    // launch/warp beyond the declared widths
  ull pc_count;        // distinct (launch, pc) pairs assigned an id
  ull pc_overflow;     // (launch, pc) pairs beyond max_pcs
  ull distinct_pairs;  // set by the count kernels
  ull distinct_pc;     // set by the per-pc kernel
  ull hash_fail;       // hash-table insert failures (probe limit)
  ull n_deferred;      // views deferred to the general decode kernel (per call)
  ull next_range;      // decode work ranges handed out so far (per call)
  ull pad[5];
};

// ---- object table in device memory, sorted by (space << 48 | base) -------
struct ObjTable {
  const ull* lo;    // space << 48 | base           [n]
  const ull* hi;    // lo + len                     [n]
  const ull* soff;  // first global sector index    [n + 1]
  uint32_t n;
};

// ---- (launch, pc) -> dense pc id map (open addressing, global memory) ----
struct PcMap {
  ull* keys;         // site + 1 (0 = empty)      [cap]
  uint32_t* vals;    // pc id, kPcNone = pending   [cap]
  uint32_t* site_of; // pc id -> site              [max_pcs]
  uint32_t cap_mask;
  uint32_t max_pcs;
};

// ---- sector ownership in the sharded mode (shard.cu, row e) ---------------
constexpr int kShardShift = 11;  // ownership chunk: 2048 sectors = one indicator tile
constexpr int kMaxRanks = 64;
// owner rank of global sector g (block-cyclic over 2048-sector chunks)
__host__ __device__ __forceinline__ uint32_t shard_owner(unsigned long long g, uint32_t nranks) {
  return nranks <= 1 ? 0u : (uint32_t)((g >> kShardShift) % nranks);
}
// local index of global sector g on its owner: the owned chunks packed in
// chunk order (l = ((g >> c) / P) << c | (g & (2^c - 1))); an
// owner's dense rows and count workspace cover only its chunks
__host__ __device__ __forceinline__ unsigned long long shard_local(unsigned long long g, uint32_t nranks) {
  return nranks <= 1 ? g
                     : (((g >> kShardShift) / nranks) << kShardShift) | (g & ((1ull << kShardShift) - 1));
}
__host__ __device__ __forceinline__ unsigned long long shard_global(unsigned long long l, uint32_t rank,
                                                                   uint32_t nranks) {
  return nranks <= 1 ? l
                     : ((((l >> kShardShift) * nranks) + rank) << kShardShift) | (l & ((1ull << kShardShift) - 1));
}

// ---- key layout -----------------------------------------------------------
// key:     [ g : S ][ launch : L ][ warp : W ][ pcid : P ][ mask : 8 ]  (S+L+W+P <= 56)
//          one stream carries the (sector, warp) and the (pc, sector) facts
// pc key:  [ pcid : P ][ g : S ][ mask : 8 ]   (derived at build for the sort/hash paths)
struct KeyLayout {
  uint32_t S, L, W, P;
};
__host__ __device__ __forceinline__ ull key_g(ull key, const KeyLayout& k) { return key >> (8 + k.P + k.L + k.W); }
__host__ __device__ __forceinline__ uint32_t key_launch(ull key, const KeyLayout& k) {
  return k.L ? (uint32_t)((key >> (8 + k.P + k.W)) & ((1ull << k.L) - 1)) : 0u;
}
__host__ __device__ __forceinline__ uint32_t key_pcid(ull key, const KeyLayout& k) {
  return k.P ? (uint32_t)((key >> 8) & ((1ull << k.P) - 1)) : 0u;
}

struct DecodeArgs {
  const uint4* recs;
  ull n;                  // records in this ingest call
  const ull* heads;       // [n_ranges + 1] range boundaries (explicit heads)
  uint32_t n_ranges;
  ObjTable obj;
  KeyLayout kl;
  uint32_t max_launches, max_warps;
  int track_pc;
  PcMap pcmap;
  ull* keys;              // key buffer (append)
  DevCounters* ctr;
  ull* instr_ctr;         // [max_launches * n_obj * 2] (instrs, misaligned)
  ull* launch_ctr;        // [max_launches * 2] (unmapped words, mapped word accesses)
  ull* deferred;          // [n] p << 7 | stats_only << 6 | len of deferred views
  uint32_t* seg_cnt;      // [S_tot] keys per sector (SEGMENT histogram), or null
  uint32_t* acc;          // [8 S_tot] lane accesses per word (track_access), or null
  uint32_t block_warps, block_id;  // sampled-block mode (0: whole grid)
  const uint32_t* wl;               // launch whitelist bitmask [128], or null: every launch
};

// outside the traced scope: a warp outside the sampled block or a launch
// outside the whitelist (launch < 4096 for any record: site >> 20)
__device__ __forceinline__ bool out_of_scope(const DecodeArgs& a, uint32_t warp, uint32_t launch) {
  return (a.block_warps && warp / a.block_warps != a.block_id) ||
         (a.wl && !((a.wl[(launch >> 5) & 127u] >> (launch & 31u)) & 1u));
}

// ---- kernels (launch wrappers live in the .cu files) ----------------------
void launch_find_heads(const uint4* recs, ull n, ull range_len, uint32_t n_ranges, ull* heads,
                       cudaStream_t s);
void launch_decode(const DecodeArgs& a, int num_sms, cudaStream_t s);
// the lane-per-record decoder (decode_lane.cu): windows of whole instructions
void launch_decode_lane(const DecodeArgs& a, int num_sms, cudaStream_t s);
// records and instruction heads of a sample of 32-record chunks (out[0], out[1] +=)
void launch_head_sample(const uint4* recs, ull n, ull* out, cudaStream_t s);
void launch_decode_general(const DecodeArgs& a, int num_sms, cudaStream_t s);
// warp-instruction records (decode_warp.cu); spill_ctr[0] = spilled per-lane
// records written to spill, spill_ctr[1] += lane records seen
void launch_decode_warp(const DecodeArgs& a, const uint4* wrec, ull n_instr, uint4* spill, ull* spill_ctr,
                        int num_sms, cudaStream_t s);

// onesweep LSD radix sort of u64 keys on bits [lo_bit, lo_bit + nbits)
struct SortWorkspace {
  ull* alt = nullptr;        size_t alt_cap = 0;
  ull* status = nullptr;     size_t status_cap = 0;   // tiles * 256
  uint32_t* hist = nullptr;  // [8 * 256] digit histograms
  uint32_t* counters = nullptr;  // [8] tile counters
  uint32_t epoch = 0;
  ull launches = 0;  // kernels launched (for stats)
};
// returns pointer to the sorted keys (either keys or ws.alt)
ull* radix_sort_keys(ull* keys, ull n, int lo_bit, int nbits, SortWorkspace& ws, int num_sms,
                     cudaStream_t s, cudaError_t* err);

// sector-segmented dedup (segment.cu): counting sort by sector + per-chunk
// shared-memory dedup and count
struct SegWorkspace {
  uint32_t* cnt = nullptr;   // [S_tot + 1] keys per sector
  ull* cko = nullptr;        // [chunks + 1] first key of each chunk (+ end = the normal keys)
  ull* cur = nullptr;        // [S_tot + 1] scatter cursors (one per chunk)
  ull* cs0 = nullptr;        // [chunks + 1 <= S_tot + 2] first sector of each chunk (+ end)
  uint32_t* dst = nullptr;   // [S_tot + 1] chunk of each sector's keys (~0: a big sector's, hash path)
  ull* bsum = nullptr;       // scan block sums
  uint32_t* maxc = nullptr;  // [8 u64]: max keys in one sector | totals: normal keys, big sectors, big keys
  ull cap_sec = 0;
  ull launches = 0;
  // two-pass partition (coarse buckets balanced by key count, then chunks / big sectors)
  uint32_t ncoarse = 0;
  ull* gpre = nullptr;       // [groups][3] (NL, BS, BK) at each 64-sector group
  uint16_t* cb = nullptr;    // [groups] coarse bucket of each group
  ull* cstart = nullptr;     // [ncoarse + 1] first key of each coarse bucket
  ull* cinfo = nullptr;      // [ncoarse + 1][3] normal keys / big sectors before the bucket, its first sector
  ull* ccur = nullptr;       // [ncoarse] pass-1 cursors
  ull* tpre = nullptr;       // [ncoarse + 1] first pass-2 tile of each bucket
  uint32_t* tbk = nullptr;   // [pass-2 tiles] bucket of each tile
  ull tbk_cap = 0;
  ull* tmp = nullptr;        // pass-1 output
  size_t tmp_cap = 0;
  ull* bg = nullptr;         // [n big sectors] sector id of big sector i
  ull* boff = nullptr;       // [n big sectors] its first key in `big`
  ull* bcur = nullptr;       // [n big sectors] pass-2 cursors
  ull* bpre = nullptr;       // [2][big_cap] first CTA of each big sector (main, pc passes)
  uint32_t* bpcm = nullptr;  // [big_cap][2] <= 8 pc ids: each big sector's (pc, word) bytes, OR-ed by its passes
  ull big_cap = 0, n_bigsec = 0, n_big_keys = 0, n_normal = 0, n_chunks = 0;
  ull* chunk_ctr = nullptr;  // persistent chunk kernel: chunks handed out
  // per-kernel timers (created by the caller): before coarse, after coarse,
  // after fine, after chunk, after big; ran[] says which intervals ran
  cudaEvent_t ev[5] = {};
  bool ran[4] = {false, false, false, false};
};
// counted: ws.cnt already holds the keys per sector (counted by the decoder)
cudaError_t segment_reserve(SegWorkspace& ws, ull nsec);
// n_big: keys of sectors too big for a chunk (they go to the hash path)
cudaError_t segment_prepare(const ull* keys, ull n, KeyLayout kl, ull nsec, SegWorkspace& ws, int num_sms,
                            cudaStream_t s, uint32_t* max_per_sector, ull* n_big, bool counted);
// scatter + per-chunk dedup: dense counts (a5) and, if pc_hist != null, the
// per-pc histograms (a6) of the chunk's sectors
// big: receives the keys of the big sectors (capacity n_big from prepare)
cudaError_t segment_count(const ull* keys, ull n, ull* out, ull* big, KeyLayout kl, ull nsec, uint32_t filter,
                          SegWorkspace& ws, uint32_t* wc, uint32_t* sc, const uint32_t* site_of, ull* pc_hist,
                          ull n_pc, DevCounters* ctr, int num_sms, cudaStream_t s);
ull segment_chunk_cap();

// hash-set dedup: insert keys (prefix<<8 | mask) into table; EMPTY = ~0.
// drop_low: prefix bits dropped before inserting (the pc id of main keys)
void launch_hash_insert(const ull* keys, ull n, ull* table, ull cap_mask, uint32_t drop_low, DevCounters* ctr,
                        int num_sms, cudaStream_t s);
// derive pc keys [pcid : P][g : S][mask : 8] from keys (sort / hash paths)
void launch_pc_extract(const ull* keys, ull n, KeyLayout kl, ull* pckeys, int num_sms, cudaStream_t s);

// segmented count (a5) -> dense arrays
void launch_count_sorted(const ull* keys, ull n, KeyLayout kl, uint32_t launch_filter, uint32_t* word_cnt,
                         uint32_t* sector_cnt, DevCounters* ctr, int num_sms, cudaStream_t s);
void launch_count_hash(const ull* table, ull cap, KeyLayout kl, uint32_t launch_filter, uint32_t* word_cnt,
                       uint32_t* sector_cnt, DevCounters* ctr, int num_sms, cudaStream_t s);

// DENSE dedup (sampled-block mode, <= 64 warps in scope): keys OR-ed into one
// u64 warp mask per (launch, word) [L][S_tot][8], then popcounts -> dense arrays
void launch_dense_or(const ull* keys, ull n, KeyLayout kl, uint32_t warp0, ull S_tot, ull* dm, int num_sms,
                     cudaStream_t s);
void launch_dense_count(const ull* dm, uint32_t L, ull S_tot, uint32_t filter, uint32_t* wc, uint32_t* sc,
                        DevCounters* ctr, int num_sms, cudaStream_t s);

// a6 histograms over dense arrays, per object
// (sharded mode: only the sectors rank owns; nranks = 1: all)
// (sharded mode: rows of the rank's own chunks, local indices [0, n_local))
void launch_object_hist(const uint32_t* word_cnt, const uint32_t* sector_cnt, ObjTable obj,
                        const ull* obj_nwords, ull* hist /*[n_obj][2][33]*/, ull total_sectors, ull n_local,
                        uint32_t rank, uint32_t nranks, int num_sms, cudaStream_t s);
// a6 per-pc histograms from deduped pc keys
void launch_pc_hist_sorted(const ull* pckeys, ull n, KeyLayout kl, const uint32_t* site_of,
                           uint32_t launch_filter, const uint32_t* word_cnt, const uint32_t* sector_cnt,
                           ull* pc_hist /*[max_pcs][2][33]*/, DevCounters* ctr, int num_sms, cudaStream_t s);
void launch_pc_hist_hash(const ull* table, ull cap, KeyLayout kl, const uint32_t* site_of,
                         uint32_t launch_filter, const uint32_t* word_cnt, const uint32_t* sector_cnt,
                         ull* pc_hist, DevCounters* ctr, int num_sms, cudaStream_t s);

// a7 indicators
struct IndicatorArgs {
  const uint32_t* word_cnt;
  const uint32_t* sector_cnt;
  ObjTable obj;
  const ull* obj_nwords;     // [n]
  const uint32_t* obj_space; // [n]
  const ull* tile_obj;       // [n_tiles] object of tile
  const ull* tile_first;     // [n_tiles] first sector (global) of tile
  const ull* tile_end;       // [n_tiles] end sector (global, exclusive)
  uint32_t n_tiles;
  const ull* instr_ctr;      // [max_launches * n * 2]
  uint32_t max_launches, launch_filter;
  thermo_params prm;
  ull* ind;                  // [n][kIndFields] accumulators
  ull* tile_info;            // [n_tiles][kTileInfo] first touched, last touched, cand, cnt, touched words, gaps of 1
  ull* tile_prev;            // [n_tiles] last touched word before the tile (or ~0)
  uint32_t rank, nranks;     // sharded mode: tiles of other ranks are skipped
};
constexpr int kIndFields = 24;
constexpr int kTileInfo = 6;
enum IndField {
  F_NWORDS, F_NSECTORS, F_T, F_TW, F_HOT, F_FS, F_SUMX, F_SUMX2_LO, F_SUMX2_HI, F_LE1, F_MAXSEC,
  F_INSTRS, F_MIS, F_GAPS, F_DOMGAP, F_DOMCNT, F_LABELS, F_CAND, F_CANDCNT, F_VERIFY, F_PAD0,
  F_PAD1, F_PAD2, F_PAD3
};
void launch_indicators(const IndicatorArgs& a, int num_sms, cudaStream_t s);

// run compression of one object's rows (export.cu): sectors [g0, g0 + ns) of the
// dense arrays, nw words; scratch: ceil(ns / 2048) u32; out NULL = count only
cudaError_t compress_runs(const uint32_t* wc, const uint32_t* sc, ull g0, ull ns, ull nw, uint32_t* scratch,
                          ull* d_total, thermo_run* out, ull out_cap, ull* n_runs, cudaStream_t s);
// the same in steps, for the sharded mode (partial sums combined in between):
// tiles (mode 0: sums + votes, 1: verify), stitch, finalize
void launch_indicator_tiles(const IndicatorArgs& a, int mode, cudaStream_t s);
void launch_indicator_stitch(const IndicatorArgs& a, cudaStream_t s);
void launch_indicator_finalize(const IndicatorArgs& a, cudaStream_t s);
// per-object partial sums <-> a reducible array: sums [n][10] (T, TW, hot, fs,
// sum x, le1, sum x^2 as four 32-bit limbs), maxima [n] (largest sector
// count); dir 0 packs, 1 unpacks.  verify: F_VERIFY <-> [n]
constexpr int kIndSumFields = 10;
void launch_indicator_pack(ull* ind, uint32_t n, ull* sums, ull* maxs, ull* verify, int dir, cudaStream_t s);

}  // namespace thermo
