/*
 * thermo.h -- C ABI of libthermo, a B200-native (sm_100a) implementation of the
 * data-parallel hot path of cuThermo (arXiv 2507.18729): the reduction of a
 * GPU memory-access trace into the paper's word-sector heat map of distinct
 * warp counts, heat-level histograms per object and per PC, and the sharing /
 * inefficiency indicators the paper's five patterns are read from.
 *
 * Citation keys: P:n = PAPER.md line n (section named alongside);
 *                S:n = SPEC.md line n;  G# = DESIGN.md "Readings" entry.
 *
 * General conventions
 *   - Every entry point returns a thermo_status; no exception crosses the ABI.
 *     CUDA / NCCL failures are sticky: once a context has returned
 *     THERMO_ECUDA or THERMO_ENCCL every later call returns the same code.
 *     thermo_last_error() gives a per-context message for the last failure.
 *   - A context is bound to one device and one CUDA stream and is NOT
 *     thread-safe; distinct contexts are independent.
 *   - All device work is stream-ordered on the context stream.  Queries are
 *     synchronous (they copy small results to caller-owned HOST buffers).
 *   - State machine: create -> register_objects (exactly once) -> ingest_trace*
 *     -> build_heatmap -> query_* / classify.  build_heatmap may be repeated
 *     (e.g. with another launch filter); ingest after build invalidates the
 *     build (queries then return THERMO_ESTATE until the next build).
 *     Out-of-order calls return THERMO_ESTATE.
 */
#ifndef THERMO_H_
#define THERMO_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define THERMO_ABI_VERSION 6u
#define THERMO_ALL_LAUNCHES 0xFFFFFFFFu
#define THERMO_LEVELS 33        /* heat levels 0..32: level(c) = bit_width(c) (G10) */
#define THERMO_MAX_OBJECTS 1024

/*
 * One lane's memory access: the paper's per-instruction record (P:283-292,
 * §IV-B1: pc, address[32], size, active_mask, access_flags, warp_id,
 * block_id) flattened to one 16-byte record per active lane.  16-byte aligned,
 * little-endian.
 *
 *   addr_flags bits [0,48)  byte address (G5)
 *              bits [48,51) log2(access size): 0..4 = 1,2,4,8,16 bytes (G4)
 *              bits [51,53) kind: 0 load, 1 store, 2 atomic (G7: all count)
 *              bits [53,55) space: 0 global, 1 shared, 2 local
 *              bit  55      instr_start: first record of a warp instruction (G24)
 *              bits [56,64) reserved, must be 0
 *   warp       global warp id within its launch
 *              (= linear_block_id * warps_per_block + warp_in_block; G1)
 *   site       bits [0,20) pc >> 4 (SASS instructions are 16 B), bits [20,32) launch id
 *
 * A record is INVALID (skipped and counted, never fatal) if log2size > 4,
 * kind > 2, space > 2, reserved != 0, or addr + size > 2^48.
 * An instruction (for the misalignment indicator) is a run of
 * records starting at a record with instr_start = 1 or at the first record of
 * an ingest call, of at most 32 records (32 lane addresses); a longer
 * run is split every 32 records (G24).
 */
typedef struct {
  uint64_t addr_flags;
  uint32_t warp;
  uint32_t site;
} thermo_record;

/*
 * Warp-instruction record (the
 * collector's native unit, one warp instruction with its 32 lane addresses).
 * By definition it stands for the per-lane thermo_records of its active lanes
 * in lane order, the first one carrying instr_start, each with
 *   addr_flags = addr[0,48) | log2size | kind | space | instr_start | reserved,
 * where reserved != 0 (an invalid record) iff addr has bits >= 48 set or
 * flags has bits >= 7 set.  272 bytes, 16-byte aligned.  Full warps take
 * 8.5 B per lane instead of 16.
 */
typedef struct {
  uint32_t warp;       /* global warp id within its launch                          */
  uint32_t site;       /* [0,20) pc >> 4 | [20,32) launch id                        */
  uint32_t active;     /* bit l: lane l executed the access                         */
  uint32_t flags;      /* [0,3) log2(size) | [3,5) kind | [5,7) space | [7,32) 0    */
  uint64_t addr[32];   /* byte address of lane l (inactive lanes: ignored)          */
} thermo_warp_record;

/*
 * A registered data object ("memory registration"; P:329 region
 * config).  base must be 32-byte aligned (G9), len > 0, base + len <= 2^48, and
 * objects of one space must not overlap.  id is the caller's handle
 * used by the queries; ids must be unique.
 * A word (4 B) belongs to the object iff its first byte lies in [base, base+len);
 * n_words = ceil(len/4), n_sectors = ceil(len/32).
 */
typedef struct {
  uint64_t base;
  uint64_t len;
  uint32_t space;
  uint32_t id;
} thermo_object;

typedef enum { THERMO_WORD = 1, THERMO_SECTOR = 2, THERMO_BOTH = 3 } thermo_granularity;

typedef enum {
  THERMO_OK = 0,
  THERMO_EINVAL = -1,  /* bad argument / malformed object table           */
  THERMO_ENOMEM = -2,  /* device or pinned-host allocation failed          */
  THERMO_ERANGE = -3,  /* key width overflow, id out of declared range, cap too small */
  THERMO_ESTATE = -4,  /* call out of order                                */
  THERMO_ECUDA = -5,   /* CUDA error (sticky)                              */
  THERMO_ENCCL = -6    /* NCCL error (sticky)                              */
} thermo_status;

/* dedup paths for the main (sector, launch, warp) keys (a4):
 *   SORT     onesweep LSD radix sort on all key bits
 *   HASH     open-addressing hash set in HBM
 *   SEGMENT  counting sort by sector + per-chunk shared-memory dedup; the
 *            keys of sectors holding >= 2048 keys take a hash-set side path
 *   DENSE    sampled-block mode only (1 <= block_warps <= 64, SURVEY §8f item
 *            1): the paper's per-word warp bitmask as one u64 per
 *            (launch, word) in device memory (64 B per sector per launch),
 *            OR-ed from the keys and popcounted; no sort, no hash
 *   AUTO     DENSE in sampled-block mode with block_warps <= 64 when its masks
 *            take <= 4 GiB; else SEGMENT up to 2^30 registered sectors (its
 *            workspace is 28 B per sector), HASH beyond (chosen by
 *            measurement)
 * thermo_create returns THERMO_EINVAL for DENSE outside sampled-block mode or
 * with block_warps > 64. */
typedef enum {
  THERMO_DEDUP_AUTO = 0, THERMO_DEDUP_SORT = 1, THERMO_DEDUP_HASH = 2, THERMO_DEDUP_SEGMENT = 3,
  THERMO_DEDUP_DENSE = 4
} thermo_dedup;

/*
 * Context configuration.  max_launches / max_warps_per_launch fix the bit
 * widths L, W of the (sector, launch, warp) key; records whose launch or warp
 * id exceeds them are counted in stats.out_of_range and make build return
 * THERMO_ERANGE.  max_pcs bounds the number of distinct (launch, pc) pairs.
 */
typedef struct {
  uint32_t max_launches;          /* >= 1; launch ids < max_launches (<= 4096)      */
  uint32_t max_warps_per_launch;  /* >= 1; warp ids < this                           */
  uint32_t max_pcs;               /* >= 1; distinct (launch, pc) pairs (<= 65536)    */
  uint32_t dedup;                 /* thermo_dedup                                    */
  uint32_t track_pc;              /* 1: maintain per-PC histograms (G11)             */
  uint32_t track_access;          /* 1: also count lane accesses per word (the Fig. 3
                                     baseline; thermo_query_access)       */
  uint64_t expected_pairs;        /* hash sizing hint: distinct (sector,warp) pairs; 0 = auto */
  uint32_t block_warps;           /* sampled-block mode:
                                     0 = the whole grid; else warps per thread block, and
                                     only records of warps in block `block_id`
                                     (warp / block_warps == block_id) are reduced -- the
                                     others are treated as never traced              */
  uint32_t block_id;
} thermo_config;

/*
 * Pattern-rule parameters as exact rationals (SPEC PatternParams; G12).
 * Defaults (thermo_default_params): theta_hot 16, alpha 5/4, beta 4/1, fs_min 4,
 * smem_cap 1, smem_cov 9/10, gamma 1/2, strided_min_sectors 4, dom 3/4,
 * hot_frac 1/2, fs_frac 1/4, mis_frac 1/10, cv 1/2.
 */
typedef struct {
  uint64_t theta_hot, alpha_num, alpha_den, beta_num, beta_den, fs_min;
  uint64_t smem_cap, smem_cov_num, smem_cov_den, gamma_num, gamma_den;
  uint64_t strided_min_sectors, dom_num, dom_den, hot_frac_num, hot_frac_den;
  uint64_t fs_frac_num, fs_frac_den, mis_frac_num, mis_frac_den, cv_num, cv_den;
} thermo_params;

/* label bits of thermo_indicators.labels (§IV-C) */
#define THERMO_LABEL_HOT 1u
#define THERMO_LABEL_RANDOM_HOT 2u               /* P:404 random variant */
#define THERMO_LABEL_FALSE_SHARING 4u
#define THERMO_LABEL_SMEM_THREAD_LOCAL 8u
#define THERMO_LABEL_SMEM_WARP_PRIVATE 16u
#define THERMO_LABEL_MISALIGNED 32u
#define THERMO_LABEL_STRIDED 64u

/* Per-object indicator sums and labels. */
typedef struct {
  uint32_t object_id;
  uint32_t labels;             /* THERMO_LABEL_* bits                         */
  uint64_t n_words, n_sectors;
  uint64_t touched_sectors;    /* T: sectors with count >= 1                   */
  uint64_t touched_words;      /* TW: words with count >= 1                    */
  uint64_t hot_sectors;        /* c >= theta_hot and alpha_den*c <= alpha_num*max_word */
  uint64_t fs_sectors;         /* beta_den*c >= beta_num*max_word and c >= fs_min */
  uint64_t sum_x;              /* sum of nonzero word counts                   */
  uint64_t sum_x2_lo, sum_x2_hi;  /* 128-bit sum of squares of word counts      */
  uint64_t le1_words;          /* touched words with count <= smem_cap         */
  uint64_t max_sector_count;
  uint64_t instrs, misaligned_instrs;  /* instructions attributed to the object (G24) */
  uint64_t gaps;               /* TW - 1 (gaps between consecutive touched words) */
  uint64_t dom_gap, dom_count; /* gap value holding a strict majority of gaps, else 0,0 */
} thermo_indicators;

/* Per-PC heat-level histogram row (G11): distinct (launch, pc, word) pairs
 * binned by the word's level (THERMO_WORD) or distinct (launch, pc, sector)
 * pairs binned by the sector's level (THERMO_SECTOR). */
typedef struct {
  uint32_t launch;
  uint32_t pc;                 /* byte pc (site field << 4) */
  uint64_t hist[THERMO_LEVELS];
} thermo_pc_hist;

typedef struct {
  uint64_t records;            /* records ingested (all calls)                */
  uint64_t invalid;            /* invalid records (skipped)                   */
  uint64_t out_of_range;       /* launch/warp id beyond the declared widths   */
  uint64_t unmapped_words;     /* word accesses outside every object (G8), launch-filtered */
  uint64_t mapped_word_accesses; /* word accesses inside objects, launch-filtered */
  uint64_t keys_emitted;       /* (sector, launch, warp) keys after pre-dedup  */
  uint64_t pc_keys_emitted;    /* (pc, sector) keys after pre-dedup            */
  uint64_t distinct_pairs;     /* distinct (sector, launch, warp) = sum of sector counts */
  uint64_t distinct_pc_pairs;  /* distinct (launch, pc, sector)                */
  uint64_t n_pcs;              /* distinct (launch, pc) pairs seen             */
  uint32_t dedup_used;         /* THERMO_DEDUP_SORT, _HASH, _SEGMENT or _DENSE  */
  uint32_t decoder_used;       /* last ingest: 1 per-instruction view kernel
                                  (+ general kernel), 2 lane-per-record kernel
                                  (chosen by the trace's mean instruction length,
                                  or THERMO_DECODER=view|lane), 3 warp-record
                                  kernel (thermo_ingest_warp_trace); 0 none   */
  double ms_ingest, ms_build, ms_classify;  /* device time of the last calls   */
  /* device time (CUDA events on the context stream) of the phases of the last
   * ingest / build / classify: decode kernel (a2+a3), main-key dedup (a4),
   * segmented count (a5), object histograms (a6), per-pc dedup + histograms
   * (a4+a6), indicators (a7) */
  double ms_decode, ms_dedup, ms_count, ms_hist, ms_pc, ms_indicators;
  uint64_t kernel_launches;    /* libthermo kernels launched since create      */
  /* sharded mode, last build: the key all-to-all's device time on this rank
   * and the bytes it sent to other ranks (NVLink roofline of row e) */
  double ms_exchange;
  uint64_t exchange_bytes;
  /* per-kernel device time of the last ingest / build / classify (CUDA events
   * on the context stream around each kernel or kernel group; 0 if it did not
   * run): THERMO_K_* indices */
  double ms_kernel[9];
  /* sectors this context's dense rows and count workspace cover: all
   * registered sectors, or (sharded mode) the rank's own 2048-sector chunks */
  uint64_t local_sectors;
  /* keys this context counts in its build (sharded mode: the keys it owns
   * after the exchange; one rank: every key) */
  uint64_t local_keys;
} thermo_stats;
enum {
  THERMO_K_DECODE = 0,         /* decode_kernel: fast per-instruction decode (a2+a3)        */
  THERMO_K_DECODE_GENERAL = 1, /* decode_general_kernel: deferred / packed views (a2+a3)     */
  THERMO_K_SEG_SCAN = 2,       /* SEGMENT: per-sector scans, coarse buckets, tiles (a4)      */
  THERMO_K_SEG_COARSE = 3,     /* SEGMENT: partition pass 1, coarse buckets (a4)             */
  THERMO_K_SEG_FINE = 4,       /* SEGMENT: partition pass 2, chunks / big sectors (a4)       */
  THERMO_K_SEG_CHUNK = 5,      /* SEGMENT: per-chunk dedup + count + per-pc bins (a4-a6)     */
  THERMO_K_SEG_BIG = 6,        /* SEGMENT: big-sector plan + count + per-pc bins (a4-a6)     */
  THERMO_K_OBJECT_HIST = 7,    /* object_hist_kernel (a6)                                    */
  THERMO_K_INDICATORS = 8      /* indicator kernels of classify (a7)                         */
};

typedef struct thermo_ctx thermo_ctx;

/* Defaults: max_launches 1, max_warps_per_launch 2^20, max_pcs 4096, AUTO, track_pc 1. */
void thermo_default_config(thermo_config *cfg);
void thermo_default_params(thermo_params *p);
uint32_t thermo_abi_version(void);

/*
 * Create a context on `device` using CUDA stream `stream` (a cudaStream_t
 * passed as void*, NULL = a new blocking stream owned by the context, which is
 * ordered after work queued on the legacy default stream).  Device-resident
 * records written on any OTHER stream must be complete before ingest (pass
 * that stream here, or synchronize).  cfg NULL = defaults.  Ownership: the context owns every device buffer it allocates.
 * Errors: EINVAL (bad cfg), ECUDA, ENOMEM.
 */
thermo_status thermo_create(thermo_ctx **out, int device, void *stream, const thermo_config *cfg);

/*
 * Multi-GPU (address-sharded) context: rank `rank` of `nranks`
 * (1..64), one process per GPU.  nccl_id is a 128-byte ncclUniqueId made by
 * rank 0 with thermo_nccl_unique_id and broadcast by the caller (e.g. over a
 * torch.distributed group).  A sector's counts depend only on the records
 * touching it (S:292-300 merge = OR, S:332 shard by sector), so:
 *   - every rank ingests its own slice of the trace (split the trace at
 *     instr_start records);
 *   - thermo_build_heatmap and thermo_classify are COLLECTIVE: every rank
 *     calls them, in the same order with the same arguments.  Build unifies
 *     the (launch, pc) ids, moves each key to the owner of its sector --
 *     rank (g >> 11) % nranks for global sector index g (2048-sector chunks)
 *     -- in one all-to-all, counts the owned sectors, and sums the
 *     histograms / counters over ranks;
 *   - thermo_query_histogram, thermo_query_per_pc, thermo_classify and
 *     thermo_get_stats (after a build) return job-wide results, identical on
 *     every rank and bit-identical to one rank reducing the whole trace;
 *   - thermo_query_heatmap returns this rank's partition: cells of sectors
 *     owned by other ranks are 0, so the full rows are the element-wise sum
 *     over ranks (thermo_sharding gives the chunk size).
 * Errors additionally: ENCCL (sticky).  nranks == 1 is thermo_create.
 */
thermo_status thermo_create_dist(thermo_ctx **out, int device, void *stream, const thermo_config *cfg,
                                 const void *nccl_id, int rank, int nranks);
/* Writes a fresh 128-byte ncclUniqueId into out128 (call on rank 0).  Errors: EINVAL, ENCCL. */
thermo_status thermo_nccl_unique_id(void *out128);
/*
 * The same sharded mode inside one process on one device: creates nranks
 * contexts (outs[0..nranks), each on its own new stream) whose collectives
 * exchange through device-to-device copies.  Each context must be driven by
 * its own host thread, because a collective call returns only when every
 * rank has made it.  Used to run and test the P-rank algorithm on one GPU.
 * Errors: EINVAL (nranks outside 1..64), ECUDA, ENOMEM.
 */
thermo_status thermo_create_local_shards(thermo_ctx **outs, int device, const thermo_config *cfg, int nranks);
/* rank, nranks and the ownership chunk (sectors) of a context (1 rank: 0, 1). */
thermo_status thermo_sharding(const thermo_ctx *ctx, int *rank, int *nranks, uint32_t *chunk_sectors);

thermo_status thermo_destroy(thermo_ctx *ctx);

/*
 * Drop everything ingested (keys, counters, pc ids) and return to the
 * "registered" state, keeping the object table and all allocations -- for
 * repeated runs over new traces of the same objects.  Errors: ESTATE.
 */
thermo_status thermo_reset(thermo_ctx *ctx);

/*
 * Kernel sampling by whitelist ("kernel sampling is also supported by a
 * whitelist method"): from the next ingest call on, only the
 * records of the n launch ids in `launches` (host array, read during the call)
 * are traced; the others are treated as never traced (counted in
 * stats.records only), like the warps outside the sampled block.  n = 0 traces
 * every launch again.  Combines with sampled-block mode.  Errors: EINVAL (a
 * launch id >= max_launches, or launches == NULL with n > 0), ECUDA.
 */
thermo_status thermo_set_launch_whitelist(thermo_ctx *ctx, const uint32_t *launches, size_t n);

/*
 * Register the data objects.  Called exactly once, before any
 * ingest.  objs is a HOST array of n objects (copied).  Errors: EINVAL
 * (len == 0, base not 32-aligned, base+len > 2^48, space > 2, overlap within a
 * space, duplicate id, n == 0 or n > THERMO_MAX_OBJECTS), ERANGE (total sectors
 * do not fit the key together with the declared launch/warp widths), ESTATE.
 */
thermo_status thermo_register_objects(thermo_ctx *ctx, const thermo_object *objs, size_t n);

/*
 * Ingest n records (the analyzer consumes the collector's
 * buffers).  recs may be a DEVICE pointer (fast path; must stay valid until
 * the context stream passes this call) or a HOST pointer (pinned or pageable;
 * staged through pinned chunks with copies overlapped with decoding; the call
 * returns when the host buffer may be reused).  The first record starts an
 * instruction.  n == 0 is a no-op.  Errors: EINVAL (recs NULL with n > 0,
 * misaligned, a device pointer with n >= 2^32: split such traces at
 * instr_start records), ESTATE, ENOMEM, ECUDA.
 */
thermo_status thermo_ingest_trace(thermo_ctx *ctx, const thermo_record *recs, size_t n);

/*
 * Reduce everything ingested so far into the heat map (the
 * popcount flush): dense per-object word and sector distinct-warp counts,
 * level histograms per object and per PC.  launch_filter selects one launch
 * (the paper's per-kernel heat map, G2) or THERMO_ALL_LAUNCHES (launch-
 * qualified warps of all launches).  g (WORD, SECTOR or BOTH) is checked and
 * recorded; counts and histograms are always produced for both granularities.
 * May be called again (another filter) from the retained keys.  Errors: ESTATE, ERANGE
 * (out-of-range records were ingested, or too many distinct pcs), ECUDA.
 */
thermo_status thermo_build_heatmap(thermo_ctx *ctx, thermo_granularity g, uint32_t launch_filter);

/*
 * Dense heat-map rows of object `object_id` into the HOST buffer out:
 *   THERMO_WORD   n_words   u32 word counts
 *   THERMO_SECTOR n_sectors u32 sector counts
 *   THERMO_BOTH   9*n_sectors u32: per sector its 8 word counts (0 past n_words)
 *                 then the sector count (the paper's 9-cell row)
 * *n_out receives the element count; ERANGE (with *n_out set) if cap is too
 * small.  Errors: EINVAL (unknown id), ESTATE.
 */
thermo_status thermo_query_heatmap(thermo_ctx *ctx, uint32_t object_id, thermo_granularity g,
                                   uint32_t *out, size_t cap, size_t *n_out);

/* Level histogram (THERMO_LEVELS bins, HOST buffer) of one object over all its
 * n_words words (THERMO_WORD) or n_sectors sectors (THERMO_SECTOR); level-0
 * counts untouched ones.  Errors: EINVAL, ESTATE. */
/*
 * One run of the run-compressed heat map (Fig. 4 caption:
 * "consecutive memory regions with identical temperatures are compressed, and
 * the number of occurrences is indicated"): `count` consecutive sectors from
 * object-local sector `start` whose rows are all temp[0..7] (word
 * temperatures, words past the object's end 0) and temp[8] (sector).
 */
typedef struct {
  uint64_t start;
  uint64_t count;
  uint32_t temp[9];
  uint32_t reserved;
} thermo_run;

/*
 * Run-compressed rows of object `object_id` after a build: maximal runs of
 * consecutive sectors with identical rows, untouched sectors included, in
 * sector order; expanding them gives thermo_query_heatmap(BOTH) exactly.  out
 * NULL or cap too small: *n_out = number of runs and ERANGE (out non-NULL).
 * Not available in the sharded mode (rows are partitioned; assemble them).
 * Errors: ESTATE, EINVAL, ERANGE, ECUDA.
 */
thermo_status thermo_query_runs(thermo_ctx *ctx, uint32_t object_id, thermo_run *out, size_t cap, size_t *n_out);

/*
 * Ingest n warp-instruction records (device or host pointer; host records are
 * copied once).  Same result as thermo_ingest_trace on the per-lane records
 * they stand for; each record is one instruction (G24).  Instructions the fast
 * path does not take (invalid header, lanes in different 4 GiB windows,
 * straddling accesses) are reduced through their per-lane records.  Device
 * memory: spill space for the per-lane records of one chunk of instructions
 * (2^20 host / 2^23 device records per chunk: at most 4 GiB).  stats.records counts
 * lane records.  Errors: EINVAL (NULL, misaligned, n >= 2^27), ESTATE, ENOMEM,
 * ECUDA.
 */
thermo_status thermo_ingest_warp_trace(thermo_ctx *ctx, const thermo_warp_record *recs, size_t n);

/*
 * Access counts (Fig. 3: equal access counts,
 * different temperatures): out[w] = number of (record, word) pairs touching
 * word w of object `object_id`, over every ingested launch (G27; the build's
 * launch filter does not apply), n_words values.  Needs a context created
 * with track_access = 1.  Sharded mode: this rank's records only -- the job's
 * counts are the element-wise sum over ranks.  Available after ingest.
 * Errors: ESTATE (track_access off), EINVAL (unknown id), ERANGE (cap), ECUDA.
 */
thermo_status thermo_query_access(thermo_ctx *ctx, uint32_t object_id, uint32_t *out, size_t cap, size_t *n_out);

thermo_status thermo_query_histogram(thermo_ctx *ctx, uint32_t object_id, thermo_granularity g,
                                     uint64_t hist[THERMO_LEVELS]);

/* Per-PC histograms in ascending (launch, pc) order into HOST out[cap].
 * ERANGE (with *n_out set) if cap is too small; ESTATE if track_pc == 0. */
thermo_status thermo_query_per_pc(thermo_ctx *ctx, thermo_granularity g, thermo_pc_hist *out,
                                  size_t cap, size_t *n_out);

/*
 * Pattern indicators and labels per object (rules S:356-409 as
 * exact integer inequalities).  params NULL = defaults.
 * out[cap] HOST, one row per object in registration order.  Errors: ESTATE,
 * ERANGE (cap < number of objects), ECUDA.
 */
thermo_status thermo_classify(thermo_ctx *ctx, const thermo_params *params, thermo_indicators *out,
                              size_t cap, size_t *n_out);

thermo_status thermo_get_stats(thermo_ctx *ctx, thermo_stats *out);

/* Per-context message of the last failure ("" if none).  Valid until the next call. */
const char *thermo_last_error(const thermo_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* THERMO_H_ */
