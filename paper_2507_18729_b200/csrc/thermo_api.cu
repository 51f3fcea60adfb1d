// thermo_api.cu -- the C ABI of libthermo (include/thermo.h) and the host-side
// orchestration of the hot path: object staging (a1), ingest
// (a2/a3 kernels), build (a4/a5/a6 kernels), classify (a7 kernels), queries.
// Host code only launches kernels and moves small results; every step of the
// reduction runs in the kernels of decode.cu, sort.cu, count.cu, indicators.cu.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: ranges cost nothing unless a tool (nsys) attaches

#include "shard.cuh"
#include "thermo_internal.cuh"

namespace {
// one NVTX range per ABI call (SURVEY §5 tracing: nsys timelines per call)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

using namespace thermo;

namespace {

constexpr ull kRangeLen = 8192;          // records per decode work range
constexpr ull kHostChunk = 1ull << 24;   // records per staged host chunk
constexpr ull kWarpChunk = 1ull << 20;   // warp records per staged host chunk (272 MB)
constexpr ull kWarpChunkDev = 1ull << 23;  // warp records per device-resident chunk (spill space <= 4 GiB)
constexpr ull kTileSectors = 2048;       // indicator tile (256 threads x 8 sectors) = 1 << kShardShift
static_assert(kTileSectors == (1ull << kShardShift), "a tile is one ownership chunk");

int bit_width(ull x) { return x ? 64 - __builtin_clzll(x) : 0; }
ull next_pow2(ull x) {
  ull p = 1;
  while (p < x) p <<= 1;
  return p;
}

struct Buf {
  void* p = nullptr;
  size_t bytes = 0;
};

}  // namespace

struct thermo_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaStream_t copy_stream = nullptr;
  thermo_config cfg{};
  int num_sms = 148;
  int state = 0;  // 0 created, 1 registered, 2 ingested, 3 built
  thermo_status sticky = THERMO_OK;
  std::string err;
  int rank = 0, nranks = 1;

  // objects
  std::vector<thermo_object> reg;
  std::vector<uint32_t> sorted_to_reg, reg_to_sorted;
  std::unordered_map<uint32_t, uint32_t> id_to_reg;
  std::vector<ull> h_lo, h_hi, h_soff, h_nwords;
  std::vector<uint32_t> h_space;
  ull S_tot = 0;
  ull S_own = 0;   // sectors of the dense rows / count workspace: S_tot, or (sharded) the owned chunks
  KeyLayout kl{};
  uint32_t n_tiles = 0;

  // device buffers
  ull *d_lo = nullptr, *d_hi = nullptr, *d_soff = nullptr, *d_nwords = nullptr;
  uint32_t* d_space = nullptr;
  uint32_t *d_wc = nullptr, *d_sc = nullptr;
  ull* d_keys = nullptr;
  size_t keys_cap = 0;
  ull* d_pckeys = nullptr;
  size_t pckeys_cap = 0;
  ull n_keys = 0, n_pckeys = 0;
  DevCounters* d_ctr = nullptr;
  ull* d_pc_keys_tab = nullptr;
  uint32_t* d_pc_vals = nullptr;
  uint32_t* d_site_of = nullptr;
  uint32_t pc_cap = 0;
  ull* d_instr = nullptr;
  ull* d_launch_ctr = nullptr;
  ull* d_hist = nullptr;
  ull* d_pchist = nullptr;
  ull* d_ind = nullptr;
  ull *d_tile_obj = nullptr, *d_tile_first = nullptr, *d_tile_end = nullptr;
  ull* d_tile_info = nullptr;
  ull* d_tile_prev = nullptr;  // followed by obj_tile0 (u32[n+1])
  ull* d_heads = nullptr;
  size_t heads_cap = 0;
  ull* d_deferred = nullptr;
  size_t deferred_cap = 0;
  ull* d_table = nullptr;
  size_t table_cap = 0;
  ull* d_pctable = nullptr;
  size_t pctable_cap = 0;
  ull* d_dense = nullptr;  // DENSE dedup: [max_launches][S_tot][8] warp masks
  size_t dense_cap = 0;
  uint32_t* d_wl = nullptr;  // launch whitelist bitmask [128]
  bool wl_on = false;
  SortWorkspace sw, swpc;
  SegWorkspace seg;
  // host staging
  void* h_pinned[2] = {nullptr, nullptr};
  uint4* d_stage[2] = {nullptr, nullptr};
  cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_used[2] = {nullptr, nullptr};
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t evp[8] = {};  // phase timers
  ull launches = 0;         // kernels launched
  float ms_phase[6] = {0, 0, 0, 0, 0, 0};  // decode, dedup, count, hist, pc, indicators
  double ms_kernel[9] = {};                // THERMO_K_* (thermo.h)
  cudaEvent_t evk[4] = {};                 // decode kernel timers
  bool decoder_view = false;               // the last decode ran the view kernel

  uint32_t built_filter = THERMO_ALL_LAUNCHES;
  uint32_t built_gran = THERMO_BOTH;
  uint32_t dedup_used = THERMO_DEDUP_SORT;
  uint32_t decoder_used = 0;  // thermo_stats.decoder_used
  ull records = 0;
  float ms_ingest = 0, ms_build = 0, ms_classify = 0;
  bool hist_valid = false;
  bool seg_counted = false;  // the decoder counts keys per sector (SEGMENT histogram, one rank)
  uint32_t* d_acc = nullptr;  // [8 S_tot] lane accesses per word (track_access)
  uint4* d_spill = nullptr;   // per-lane records of spilled warp instructions
  uint4* d_wstage[2] = {nullptr, nullptr};  // host warp-record staging (kWarpChunk records each)
  size_t spill_cap = 0;
  ull* d_wctr = nullptr;      // [2] spilled records, lane records seen

  // sharded mode (row e, shard.cu); comm == nullptr: one rank
  Comm* comm = nullptr;
  ull n_exch = 0;                            // keys [0, n_exch) are this rank's own (exchanged)
  uint32_t pc_mapped = 0;                    // local pc ids [0, pc_mapped) have job-wide ids
  std::vector<uint32_t> glob_sites;          // job-wide pc id -> site
  std::unordered_map<uint32_t, uint32_t> glob_index;
  uint32_t* d_pcmap = nullptr;               // local pc id -> job-wide id [max_pcs]
  uint32_t* d_site_glob = nullptr;           // job-wide pc id -> site [max_pcs]
  ull* d_tmp = nullptr;                      // [256] small scratch
  ull* d_red = nullptr;                      // reduction scratch
  size_t red_cap = 0;
  ull *d_instr_g = nullptr, *d_launch_g = nullptr;  // job-wide copies (after build)
  ull h_ctr_g[17] = {};                      // job-wide DevCounters + records (after build)
  bool have_glob = false;
  cudaEvent_t evx[2] = {nullptr, nullptr};  // around the key all-to-all
  bool in_collective = false;               // inside build / classify of the sharded mode
  float ms_exchange = 0;
  ull exchange_bytes = 0;
};

namespace {

thermo_status fail(thermo_ctx* c, thermo_status st, const std::string& msg) {
  if (c) {
    c->err = msg;
    if (st == THERMO_ECUDA || st == THERMO_ENCCL) c->sticky = st;
    // a rank failing alone inside a collective call aborts the communicator,
    // so its peers get an error instead of waiting for it forever (sticky
    // ENCCL on every rank from then on)
    if (c->comm && c->in_collective) {
      c->comm->abort();
      c->in_collective = false;
      c->sticky = THERMO_ENCCL;
    }
  }
  return st;
}
// an error every rank of a sharded job detects at the same point (after a
// collective made it job-wide): no abort, not sticky
thermo_status fail_job(thermo_ctx* c, thermo_status st, const std::string& msg) {
  if (c) c->err = msg;
  return st;
}
// marks a sharded build / classify as a collective section
struct CollectiveScope {
  thermo_ctx* c;
  explicit CollectiveScope(thermo_ctx* ctx) : c(ctx) { if (c->comm) c->in_collective = true; }
  ~CollectiveScope() { c->in_collective = false; }
};

#define CK(call)                                                                                  \
  do {                                                                                            \
    cudaError_t e_ = (call);                                                                      \
    if (e_ != cudaSuccess)                                                                        \
      return fail(ctx, THERMO_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));         \
  } while (0)

template <typename T>
cudaError_t dalloc(T** p, size_t n) {
  *p = nullptr;
  if (n == 0) n = 1;
  return cudaMalloc(reinterpret_cast<void**>(p), n * sizeof(T));
}

void dfree(void* p) {
  if (p) cudaFree(p);
}

thermo_status comm_fail(thermo_ctx* ctx, int rc) {
  return fail(ctx, rc == 2 ? THERMO_ENCCL : THERMO_ECUDA, "exchange: " + ctx->comm->err);
}
#define DCK(call)                      \
  do {                                 \
    const int rc_ = (call);            \
    if (rc_) return comm_fail(ctx, rc_); \
  } while (0)

ObjTable obj_table(thermo_ctx* c) { return ObjTable{c->d_lo, c->d_hi, c->d_soff, (uint32_t)c->reg.size()}; }

thermo_status pre(thermo_ctx* ctx) {
  if (!ctx) return THERMO_EINVAL;
  if (ctx->sticky != THERMO_OK) return ctx->sticky;
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return fail(ctx, THERMO_ECUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  ctx->err.clear();
  return THERMO_OK;
}

// grow a device key buffer to hold `need` keys, preserving `keep` keys
thermo_status grow_keys(thermo_ctx* ctx, ull** buf, size_t* cap, ull need, ull keep) {
  if (need <= *cap) return THERMO_OK;
  size_t ncap = std::max<size_t>(need, *cap + *cap / 2);
  ull* nb = nullptr;
  if (cudaMalloc(&nb, ncap * sizeof(ull)) != cudaSuccess) {
    cudaGetLastError();
    ncap = need;
    if (cudaMalloc(&nb, ncap * sizeof(ull)) != cudaSuccess) {
      cudaGetLastError();
      return fail(ctx, THERMO_ENOMEM, "key buffer allocation failed");
    }
  }
  if (keep) CK(cudaMemcpyAsync(nb, *buf, keep * sizeof(ull), cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  dfree(*buf);
  *buf = nb;
  *cap = ncap;
  return THERMO_OK;
}

DecodeArgs decode_args(thermo_ctx* ctx);

// decode one device-resident call (records[0] starts an instruction)
thermo_status decode_device(thermo_ctx* ctx, const uint4* recs, ull n, bool timed = false) {
  if (n == 0) return THERMO_OK;
  const ull n_ranges = (n + kRangeLen - 1) / kRangeLen;
  if (ctx->heads_cap < n_ranges + 1) {
    dfree(ctx->d_heads);
    ctx->heads_cap = n_ranges + 1 + 1024;
    CK(dalloc(&ctx->d_heads, ctx->heads_cap));
  }
  CK(cudaEventRecord(ctx->evp[6], ctx->stream));
  if (ctx->deferred_cap < n) {
    dfree(ctx->d_deferred);
    ctx->deferred_cap = n + n / 4 + 1024;
    CK(dalloc(&ctx->d_deferred, ctx->deferred_cap));
  }
  CK(cudaMemsetAsync(&ctx->d_ctr->n_deferred, 0, 2 * sizeof(ull), ctx->stream));  // + next_range
  launch_find_heads(recs, n, kRangeLen, (uint32_t)n_ranges, ctx->d_heads, ctx->stream);
  DecodeArgs a = decode_args(ctx);
  a.recs = recs;
  a.n = n;
  a.heads = ctx->d_heads;
  a.n_ranges = (uint32_t)n_ranges;
  // Decoder choice by the trace's shape: the view-per-instruction kernel
  // (decode_fast.cu) for long instructions (full warps: SGEMM, stencil), the
  // lane-per-record kernel (decode_lane.cu) for short ones (divergent loops:
  // SpMV), from the mean instruction length of a 4096-chunk sample (measured
  // crossover); THERMO_DECODER=view|lane forces one
  const char* force = getenv("THERMO_DECODER");
  bool view;
  if (force && std::string(force) == "view") {
    view = true;
  } else if (force && std::string(force) == "lane") {
    view = false;
  } else {
    CK(cudaMemsetAsync(ctx->d_tmp + 200, 0, 2 * sizeof(ull), ctx->stream));
    launch_head_sample(recs, n, ctx->d_tmp + 200, ctx->stream);
    ull hv[2];
    CK(cudaMemcpyAsync(hv, ctx->d_tmp + 200, sizeof hv, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    view = hv[1] == 0 || hv[0] >= 16 * hv[1];  // mean instruction length >= 16 records
    ctx->launches += 1;
  }
  CK(cudaEventRecord(ctx->evk[0], ctx->stream));
  if (view) launch_decode(a, ctx->num_sms, ctx->stream);
  else launch_decode_lane(a, ctx->num_sms, ctx->stream);
  ctx->decoder_used = view ? 1u : 2u;
  ctx->decoder_view = view;
  CK(cudaEventRecord(ctx->evk[1], ctx->stream));
  launch_decode_general(a, ctx->num_sms, ctx->stream);
  CK(cudaGetLastError());
  CK(cudaEventRecord(ctx->evk[2], ctx->stream));
  CK(cudaEventRecord(ctx->evp[7], ctx->stream));
  // per-kernel times of a device-resident call (the staged host path keeps its
  // copy / decode overlap and is not timed per kernel)
  if (!timed) return THERMO_OK;
  CK(cudaEventSynchronize(ctx->evk[2]));
  float t0 = 0, t1 = 0;
  cudaEventElapsedTime(&t0, ctx->evk[0], ctx->evk[1]);
  cudaEventElapsedTime(&t1, ctx->evk[1], ctx->evk[2]);
  ctx->ms_kernel[THERMO_K_DECODE] += t0;
  ctx->ms_kernel[THERMO_K_DECODE_GENERAL] += t1;
  ctx->launches += 3;
  return THERMO_OK;
}

// the parts of the decode arguments that do not depend on the records
DecodeArgs decode_args(thermo_ctx* ctx) {
  DecodeArgs a{};
  a.obj = obj_table(ctx);
  a.kl = ctx->kl;
  a.max_launches = ctx->cfg.max_launches;
  a.max_warps = ctx->cfg.max_warps_per_launch;
  a.track_pc = ctx->cfg.track_pc ? 1 : 0;
  a.pcmap = PcMap{ctx->d_pc_keys_tab, ctx->d_pc_vals, ctx->d_site_of, ctx->pc_cap - 1, ctx->cfg.max_pcs};
  a.keys = ctx->d_keys;
  a.ctr = ctx->d_ctr;
  a.instr_ctr = ctx->d_instr;
  a.launch_ctr = ctx->d_launch_ctr;
  a.deferred = ctx->d_deferred;
  a.seg_cnt = ctx->seg_counted ? ctx->seg.cnt : nullptr;
  a.acc = ctx->d_acc;
  a.block_warps = ctx->cfg.block_warps;
  a.block_id = ctx->cfg.block_id;
  a.wl = ctx->wl_on ? ctx->d_wl : nullptr;
  return a;
}

thermo_status sync_counts(thermo_ctx* ctx) {
  ull v[2];
  CK(cudaMemcpyAsync(v, ctx->d_ctr, sizeof v, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->n_keys = v[0];
  ctx->n_pckeys = v[1];
  return THERMO_OK;
}

// =============================================================================
// sharded mode, start of a build: consistent error flags, job-wide pc ids,
// and the exchange of the keys decoded since the last build to their owners
thermo_status dist_exchange(thermo_ctx* ctx, const DevCounters& hc) {
  Comm* c = ctx->comm;
  cudaStream_t s = ctx->stream;
  const uint32_t P = (uint32_t)c->nranks;
  ull flags[2] = {hc.out_of_range, ctx->cfg.track_pc ? hc.pc_overflow : 0ull};
  CK(cudaMemcpyAsync(ctx->d_tmp, flags, sizeof flags, cudaMemcpyHostToDevice, s));
  DCK(c->allreduce(ctx->d_tmp, 2, false, s));
  CK(cudaMemcpyAsync(flags, ctx->d_tmp, sizeof flags, cudaMemcpyDeviceToHost, s));
  DCK(c->wait(s));
  if (flags[0]) return fail_job(ctx, THERMO_ERANGE, "records with launch/warp ids beyond the declared widths (job-wide)");
  if (flags[1]) return fail_job(ctx, THERMO_ERANGE, "more distinct (launch, pc) pairs than max_pcs (job-wide)");
  // ---- job-wide pc ids: union of the new sites of every rank, appended in sorted order ----
  if (ctx->cfg.track_pc) {
    const uint32_t npc = (uint32_t)std::min<ull>(hc.pc_count, ctx->cfg.max_pcs);
    std::vector<uint32_t> mine(npc - ctx->pc_mapped);
    if (!mine.empty())
      CK(cudaMemcpy(mine.data(), ctx->d_site_of + ctx->pc_mapped, mine.size() * 4, cudaMemcpyDeviceToHost));
    ull cnt = mine.size();
    std::vector<ull> cnts(P);
    DCK(c->allgather_host(&cnt, sizeof cnt, cnts.data(), s));
    const ull mx = *std::max_element(cnts.begin(), cnts.end());
    if (mx) {
      std::vector<uint32_t> pad(mx, 0xFFFFFFFFu), all(mx * P);
      std::copy(mine.begin(), mine.end(), pad.begin());
      DCK(c->allgather_host(pad.data(), mx * 4, all.data(), s));
      std::vector<uint32_t> fresh;
      for (uint32_t v : all)
        if (v != 0xFFFFFFFFu && !ctx->glob_index.count(v)) fresh.push_back(v);
      std::sort(fresh.begin(), fresh.end());
      fresh.erase(std::unique(fresh.begin(), fresh.end()), fresh.end());
      for (uint32_t v : fresh) {
        ctx->glob_index[v] = (uint32_t)ctx->glob_sites.size();
        ctx->glob_sites.push_back(v);
      }
      if (ctx->glob_sites.size() > ctx->cfg.max_pcs)
        return fail_job(ctx, THERMO_ERANGE, "more distinct (launch, pc) pairs than max_pcs (job-wide)");
      std::vector<uint32_t> map(mine.size());
      for (size_t i = 0; i < mine.size(); ++i) map[i] = ctx->glob_index[mine[i]];
      if (!map.empty())
        CK(cudaMemcpy(ctx->d_pcmap + ctx->pc_mapped, map.data(), map.size() * 4, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(ctx->d_site_glob, ctx->glob_sites.data(), ctx->glob_sites.size() * 4, cudaMemcpyHostToDevice));
      ctx->pc_mapped = npc;
    }
  }
  // ---- keys [n_exch, n_keys) -> owners (one all-to-all) ----
  const ull n_new = ctx->n_keys - ctx->n_exch;
  if (ctx->sw.alt_cap < n_new) {
    dfree(ctx->sw.alt);
    ctx->sw.alt_cap = n_new + n_new / 8 + 1024;
    CK(dalloc(&ctx->sw.alt, ctx->sw.alt_cap));
  }
  std::vector<ull> scnt(P), sdispl(P, 0), mat((size_t)P * P), rcnt(P), rdispl(P, 0);
  cudaError_t e = shard_partition(ctx->d_keys + ctx->n_exch, n_new, ctx->kl, P,
                                  ctx->cfg.track_pc ? ctx->d_pcmap : nullptr, ctx->sw.alt, ctx->d_tmp, scnt.data(),
                                  ctx->num_sms, s);
  if (e) return fail(ctx, THERMO_ECUDA, std::string("shard partition: ") + cudaGetErrorString(e));
  ctx->launches += 2;
  DCK(c->allgather_host(scnt.data(), P * sizeof(ull), mat.data(), s));
  ull total = 0;
  for (uint32_t q = 0; q < P; ++q) {
    rcnt[q] = mat[(size_t)q * P + ctx->rank];
    rdispl[q] = total;
    total += rcnt[q];
    if (q) sdispl[q] = sdispl[q - 1] + scnt[q - 1];
  }
  thermo_status st = grow_keys(ctx, &ctx->d_keys, &ctx->keys_cap, ctx->n_exch + total + 64, ctx->n_exch);
  if (st) return st;
  if (!ctx->evx[0]) {
    CK(cudaEventCreate(&ctx->evx[0]));
    CK(cudaEventCreate(&ctx->evx[1]));
  }
  CK(cudaEventRecord(ctx->evx[0], s));
  DCK(c->alltoallv(ctx->sw.alt, scnt.data(), sdispl.data(), ctx->d_keys + ctx->n_exch, rcnt.data(), rdispl.data(), s));
  CK(cudaEventRecord(ctx->evx[1], s));
  DCK(c->wait(s));
  cudaEventElapsedTime(&ctx->ms_exchange, ctx->evx[0], ctx->evx[1]);
  ctx->exchange_bytes = 0;
  for (uint32_t q = 0; q < P; ++q)
    if ((int)q != ctx->rank) ctx->exchange_bytes += scnt[q] * sizeof(ull);
  ctx->n_keys = ctx->n_exch + total;
  ctx->n_exch = ctx->n_keys;
  CK(cudaMemcpy(&ctx->d_ctr->n_keys, &ctx->n_keys, sizeof(ull), cudaMemcpyHostToDevice));  // later ingests append
  return THERMO_OK;
}

// sharded mode, end of a build: job-wide histograms and counters
thermo_status dist_combine(thermo_ctx* ctx) {
  Comm* c = ctx->comm;
  cudaStream_t s = ctx->stream;
  const size_t n = ctx->reg.size();
  DCK(c->allreduce(ctx->d_hist, n * 2 * kLevels, false, s));
  if (ctx->cfg.track_pc && !ctx->glob_sites.empty())
    DCK(c->allreduce(ctx->d_pchist, ctx->glob_sites.size() * 2 * kLevels, false, s));
  const size_t ni = (size_t)ctx->cfg.max_launches * n * 2, nl = (size_t)ctx->cfg.max_launches * 2;
  CK(cudaMemcpyAsync(ctx->d_instr_g, ctx->d_instr, ni * 8, cudaMemcpyDeviceToDevice, s));
  CK(cudaMemcpyAsync(ctx->d_launch_g, ctx->d_launch_ctr, nl * 8, cudaMemcpyDeviceToDevice, s));
  DCK(c->allreduce(ctx->d_instr_g, ni, false, s));
  DCK(c->allreduce(ctx->d_launch_g, nl, false, s));
  static_assert(sizeof(DevCounters) == 16 * sizeof(ull), "DevCounters layout");
  CK(cudaMemcpyAsync(ctx->d_tmp, ctx->d_ctr, sizeof(DevCounters), cudaMemcpyDeviceToDevice, s));
  CK(cudaMemcpyAsync(ctx->d_tmp + 16, &ctx->records, sizeof(ull), cudaMemcpyHostToDevice, s));
  DCK(c->allreduce(ctx->d_tmp, 17, false, s));
  CK(cudaMemcpyAsync(ctx->h_ctr_g, ctx->d_tmp, 17 * sizeof(ull), cudaMemcpyDeviceToHost, s));
  DCK(c->wait(s));
  ctx->have_glob = true;
  return THERMO_OK;
}

}  // namespace

// =============================================================================
// C ABI
// =============================================================================
extern "C" {

void thermo_default_config(thermo_config* cfg) {
  if (!cfg) return;
  std::memset(cfg, 0, sizeof *cfg);
  cfg->max_launches = 1;
  cfg->max_warps_per_launch = 1u << 20;
  cfg->max_pcs = 4096;
  cfg->dedup = THERMO_DEDUP_AUTO;
  cfg->track_pc = 1;
}

void thermo_default_params(thermo_params* p) {
  if (!p) return;
  *p = thermo_params{16, 5, 4, 4, 1, 4, 1, 9, 10, 1, 2, 4, 3, 4, 1, 2, 1, 4, 1, 10, 1, 2};
}

uint32_t thermo_abi_version(void) { return THERMO_ABI_VERSION; }

thermo_status thermo_create(thermo_ctx** out, int device, void* stream, const thermo_config* cfg) {
  if (!out) return THERMO_EINVAL;
  *out = nullptr;
  thermo_config c;
  if (cfg) c = *cfg; else thermo_default_config(&c);
  if (c.max_launches < 1 || c.max_launches > 4096 || c.max_warps_per_launch < 1 || c.max_pcs < 1 ||
      c.max_pcs > 65536 || c.dedup > THERMO_DEDUP_DENSE)
    return THERMO_EINVAL;
  if (c.dedup == THERMO_DEDUP_DENSE && (c.block_warps < 1 || c.block_warps > 64)) return THERMO_EINVAL;
  thermo_ctx* ctx = new thermo_ctx();
  ctx->device = device;
  ctx->cfg = c;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) { delete ctx; return THERMO_ECUDA; }
  cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (stream) {
    ctx->stream = static_cast<cudaStream_t>(stream);
  } else {
    // a BLOCKING stream: it waits for work already queued on the legacy default
    // stream (where e.g. torch writes device-resident records by default), so a
    // device trace produced there is complete before the first decode reads it
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamDefault) != cudaSuccess) { delete ctx; return THERMO_ECUDA; }
    ctx->own_stream = true;
  }
  if (cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreate(&ctx->ev0) != cudaSuccess || cudaEventCreate(&ctx->ev1) != cudaSuccess) {
    delete ctx;
    return THERMO_ECUDA;
  }
  for (int i = 0; i < 8; ++i)
    if (cudaEventCreate(&ctx->evp[i]) != cudaSuccess) {
    delete ctx;
    return THERMO_ECUDA;
  }
  for (int i = 0; i < 4; ++i)
    if (cudaEventCreate(&ctx->evk[i]) != cudaSuccess) {
      delete ctx;
      return THERMO_ECUDA;
    }
  for (int i = 0; i < 5; ++i)
    if (cudaEventCreate(&ctx->seg.ev[i]) != cudaSuccess) {
      delete ctx;
      return THERMO_ECUDA;
    }
  for (int i = 0; i < 2; ++i) {
    cudaEventCreateWithFlags(&ctx->ev_copied[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ctx->ev_used[i], cudaEventDisableTiming);
  }
  if (dalloc(&ctx->d_ctr, 1) != cudaSuccess || dalloc(&ctx->d_tmp, 256) != cudaSuccess) {
    thermo_destroy(ctx);
    return THERMO_ENOMEM;
  }
  cudaMemsetAsync(ctx->d_ctr, 0, sizeof(DevCounters), ctx->stream);
  *out = ctx;
  return THERMO_OK;
}

thermo_status thermo_create_dist(thermo_ctx** out, int device, void* stream, const thermo_config* cfg,
                                 const void* nccl_id, int rank, int nranks) {
  if (!out || !nccl_id || nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks) return THERMO_EINVAL;
  *out = nullptr;
  thermo_status st = thermo_create(out, device, stream, cfg);
  // THERMO_FORCE_COMM=1: run the NCCL path even for one rank (tests on one GPU)
  const char* force = getenv("THERMO_FORCE_COMM");
  if (st || (nranks == 1 && !(force && force[0] == '1'))) return st;
  thermo_ctx* ctx = *out;
  std::string msg;
  ctx->comm = make_nccl_comm(nccl_id, rank, nranks, &msg);
  if (!ctx->comm) {
    thermo_destroy(ctx);
    *out = nullptr;
    return THERMO_ENCCL;
  }
  ctx->rank = rank;
  ctx->nranks = nranks;
  return THERMO_OK;
}

thermo_status thermo_create_local_shards(thermo_ctx** outs, int device, const thermo_config* cfg, int nranks) {
  if (!outs || nranks < 1 || nranks > kMaxRanks) return THERMO_EINVAL;
  for (int r = 0; r < nranks; ++r) outs[r] = nullptr;
  for (int r = 0; r < nranks; ++r) {
    const thermo_status st = thermo_create(&outs[r], device, nullptr, cfg);
    if (st) {
      for (int q = 0; q < r; ++q) { thermo_destroy(outs[q]); outs[q] = nullptr; }
      return st;
    }
  }
  if (nranks > 1) {
    std::vector<Comm*> comms = make_local_comms(nranks);
    for (int r = 0; r < nranks; ++r) {
      outs[r]->comm = comms[r];
      outs[r]->rank = r;
      outs[r]->nranks = nranks;
    }
  }
  return THERMO_OK;
}

thermo_status thermo_nccl_unique_id(void* out128) {
  if (!out128) return THERMO_EINVAL;
  std::string msg;
  return nccl_unique_id(out128, &msg) ? THERMO_ENCCL : THERMO_OK;
}

thermo_status thermo_sharding(const thermo_ctx* ctx, int* rank, int* nranks, uint32_t* chunk_sectors) {
  if (!ctx) return THERMO_EINVAL;
  if (rank) *rank = ctx->rank;
  if (nranks) *nranks = ctx->nranks;
  if (chunk_sectors) *chunk_sectors = 1u << kShardShift;
  return THERMO_OK;
}

thermo_status thermo_destroy(thermo_ctx* ctx) {
  if (!ctx) return THERMO_EINVAL;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  void* bufs[] = {ctx->d_lo, ctx->d_hi, ctx->d_soff, ctx->d_nwords, ctx->d_space, ctx->d_wc, ctx->d_sc,
                  ctx->d_keys, ctx->d_pckeys, ctx->d_ctr, ctx->d_pc_keys_tab, ctx->d_pc_vals, ctx->d_site_of,
                  ctx->d_instr, ctx->d_launch_ctr, ctx->d_hist, ctx->d_pchist, ctx->d_ind, ctx->d_tile_obj,
                  ctx->d_tile_first, ctx->d_tile_end, ctx->d_tile_info, ctx->d_tile_prev, ctx->d_heads,
                  ctx->d_table, ctx->d_pctable, ctx->d_dense, ctx->d_wl, ctx->d_deferred, ctx->sw.alt, ctx->sw.status, ctx->sw.hist, ctx->sw.counters,
                  ctx->swpc.alt, ctx->swpc.status, ctx->swpc.hist, ctx->swpc.counters, ctx->seg.cnt, ctx->seg.cko, ctx->seg.cur,
                  ctx->seg.bsum, ctx->seg.maxc, ctx->seg.cs0, ctx->seg.dst, ctx->seg.gpre, ctx->seg.cb,
                  ctx->seg.cstart, ctx->seg.cinfo, ctx->seg.ccur, ctx->seg.tpre, ctx->seg.tbk, ctx->seg.tmp, ctx->seg.bg,
                  ctx->seg.boff, ctx->seg.bcur, ctx->seg.bpre, ctx->seg.bpcm, ctx->seg.chunk_ctr, ctx->d_stage[0],
                  ctx->d_stage[1], ctx->d_pcmap, ctx->d_site_glob, ctx->d_tmp, ctx->d_red, ctx->d_instr_g,
                  ctx->d_launch_g, ctx->d_acc, ctx->d_spill, ctx->d_wctr, ctx->d_wstage[0], ctx->d_wstage[1]};
  for (void* b : bufs) dfree(b);
  for (int i = 0; i < 2; ++i) {
    if (ctx->h_pinned[i]) cudaFreeHost(ctx->h_pinned[i]);
    if (ctx->ev_copied[i]) cudaEventDestroy(ctx->ev_copied[i]);
    if (ctx->ev_used[i]) cudaEventDestroy(ctx->ev_used[i]);
  }
  for (int i = 0; i < 8; ++i)
    if (ctx->evp[i]) cudaEventDestroy(ctx->evp[i]);
  for (int i = 0; i < 4; ++i)
    if (ctx->evk[i]) cudaEventDestroy(ctx->evk[i]);
  for (int i = 0; i < 5; ++i)
    if (ctx->seg.ev[i]) cudaEventDestroy(ctx->seg.ev[i]);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  for (int i = 0; i < 2; ++i)
    if (ctx->evx[i]) cudaEventDestroy(ctx->evx[i]);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  delete ctx->comm;
  delete ctx;
  return THERMO_OK;
}

thermo_status thermo_register_objects(thermo_ctx* ctx, const thermo_object* objs, size_t n) {
  NvtxRange nvtx_("thermo_register_objects");
  thermo_status st = pre(ctx);
  if (st) return st;
  if (ctx->state != 0) return fail(ctx, THERMO_ESTATE, "objects already registered");
  if (!objs || n == 0 || n > THERMO_MAX_OBJECTS) return fail(ctx, THERMO_EINVAL, "need 1..1024 objects");
  std::vector<uint32_t> order(n);
  std::unordered_map<uint32_t, uint32_t> ids;
  for (size_t i = 0; i < n; ++i) {
    const thermo_object& o = objs[i];
    if (o.len == 0 || (o.base & 31) || o.space > 2 || o.base + o.len > (1ull << 48) || o.base + o.len < o.base)
      return fail(ctx, THERMO_EINVAL, "object " + std::to_string(i) + ": need len > 0, base % 32 == 0, space <= 2, base+len <= 2^48");
    if (!ids.emplace(o.id, (uint32_t)i).second) return fail(ctx, THERMO_EINVAL, "duplicate object id");
    order[i] = (uint32_t)i;
  }
  auto key = [&](uint32_t i) { return ((ull)objs[i].space << 48) | objs[i].base; };
  std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return key(a) < key(b); });
  for (size_t j = 1; j < n; ++j) {
    const thermo_object &a = objs[order[j - 1]], &b = objs[order[j]];
    if (a.space == b.space && a.base + a.len > b.base) return fail(ctx, THERMO_EINVAL, "objects overlap");
  }
  ctx->reg.assign(objs, objs + n);
  ctx->id_to_reg = ids;
  ctx->sorted_to_reg = order;
  ctx->reg_to_sorted.assign(n, 0);
  ctx->h_lo.resize(n); ctx->h_hi.resize(n); ctx->h_soff.resize(n + 1); ctx->h_nwords.resize(n);
  ctx->h_space.resize(n);
  ull soff = 0;
  std::vector<ull> tile_obj, tile_first, tile_end;
  std::vector<uint32_t> obj_tile0(n + 1, 0);
  for (size_t j = 0; j < n; ++j) {
    const thermo_object& o = objs[order[j]];
    ctx->reg_to_sorted[order[j]] = (uint32_t)j;
    ctx->h_lo[j] = ((ull)o.space << 48) | o.base;
    ctx->h_hi[j] = ctx->h_lo[j] + o.len;
    ctx->h_soff[j] = soff;
    ctx->h_nwords[j] = (o.len + 3) / 4;
    ctx->h_space[j] = o.space;
    const ull ns = (o.len + 31) / 32;
    obj_tile0[j] = (uint32_t)tile_obj.size();
    // tiles end at the object's end and at global multiples of kTileSectors,
    // so that a tile lies in one ownership chunk of the sharded mode
    for (ull t = soff; t < soff + ns;) {
      const ull te = std::min(soff + ns, (t / kTileSectors + 1) * kTileSectors);
      tile_obj.push_back(j);
      tile_first.push_back(t);
      tile_end.push_back(te);
      t = te;
    }
    soff += ns;
  }
  obj_tile0[n] = (uint32_t)tile_obj.size();
  ctx->h_soff[n] = soff;
  ctx->S_tot = soff;
  if (ctx->nranks > 1) {  // the rank's own 2048-sector chunks only (SURVEY §8e local index)
    const ull nch = (soff + kTileSectors - 1) / kTileSectors;
    const ull own = nch > (ull)ctx->rank ? (nch - ctx->rank + ctx->nranks - 1) / ctx->nranks : 0;
    ctx->S_own = std::max<ull>(1, own) * kTileSectors;
  } else {
    ctx->S_own = soff;
  }
  ctx->n_tiles = (uint32_t)tile_obj.size();
  const thermo_config& c = ctx->cfg;
  KeyLayout kl;
  kl.S = std::max(1, bit_width(soff - 1));
  kl.L = bit_width(c.max_launches - 1);
  kl.W = bit_width(c.max_warps_per_launch - 1);
  kl.P = c.track_pc ? bit_width(c.max_pcs - 1) : 0;
  if (kl.S + kl.L + kl.W + kl.P > 56)
    return fail(ctx, THERMO_ERANGE,
                "key widths exceed 56 bits: sectors " + std::to_string(kl.S) + " + launch " + std::to_string(kl.L) +
                    " + warp " + std::to_string(kl.W) + " + pc " + std::to_string(kl.P) +
                    " (lower max_warps_per_launch / max_pcs)");
  if (soff >= (1ull << 31)) return fail(ctx, THERMO_ERANGE, "more than 2^31 sectors (64 GiB) of registered objects");
  ctx->kl = kl;
  // ---- device tables ----
  CK(dalloc(&ctx->d_lo, n)); CK(dalloc(&ctx->d_hi, n)); CK(dalloc(&ctx->d_soff, n + 1));
  CK(dalloc(&ctx->d_nwords, n)); CK(dalloc(&ctx->d_space, n));
  CK(cudaMemcpy(ctx->d_lo, ctx->h_lo.data(), n * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ctx->d_hi, ctx->h_hi.data(), n * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ctx->d_soff, ctx->h_soff.data(), (n + 1) * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ctx->d_nwords, ctx->h_nwords.data(), n * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ctx->d_space, ctx->h_space.data(), n * 4, cudaMemcpyHostToDevice));
  if (dalloc(&ctx->d_wc, 8 * ctx->S_own) != cudaSuccess || dalloc(&ctx->d_sc, ctx->S_own) != cudaSuccess)
    return fail(ctx, THERMO_ENOMEM, "dense heat-map arrays");
  CK(dalloc(&ctx->d_instr, (size_t)c.max_launches * n * 2));
  CK(dalloc(&ctx->d_launch_ctr, (size_t)c.max_launches * 2));
  CK(dalloc(&ctx->d_hist, n * 2 * kLevels));
  CK(dalloc(&ctx->d_pchist, (size_t)c.max_pcs * 2 * kLevels));
  CK(dalloc(&ctx->d_ind, n * kIndFields));
  const size_t nt = std::max<size_t>(1, ctx->n_tiles);
  CK(dalloc(&ctx->d_tile_obj, nt)); CK(dalloc(&ctx->d_tile_first, nt)); CK(dalloc(&ctx->d_tile_end, nt));
  CK(dalloc(&ctx->d_tile_info, nt * kTileInfo));
  CK(dalloc(&ctx->d_tile_prev, nt + (n + 2) / 2 + 1));
  if (ctx->n_tiles) {
    CK(cudaMemcpy(ctx->d_tile_obj, tile_obj.data(), ctx->n_tiles * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->d_tile_first, tile_first.data(), ctx->n_tiles * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->d_tile_end, tile_end.data(), ctx->n_tiles * 8, cudaMemcpyHostToDevice));
  }
  CK(cudaMemcpy(ctx->d_tile_prev + ctx->n_tiles, obj_tile0.data(), (n + 1) * 4, cudaMemcpyHostToDevice));
  ctx->pc_cap = (uint32_t)next_pow2(std::max<ull>(64, 4ull * c.max_pcs));
  CK(dalloc(&ctx->d_pc_keys_tab, ctx->pc_cap));
  CK(dalloc(&ctx->d_pc_vals, ctx->pc_cap));
  CK(dalloc(&ctx->d_site_of, c.max_pcs));
  CK(segment_reserve(ctx->seg, soff));
  if (c.track_access && dalloc(&ctx->d_acc, 8 * soff) != cudaSuccess)
    return fail(ctx, THERMO_ENOMEM, "access-count array");
  if (ctx->comm) {
    CK(dalloc(&ctx->d_pcmap, c.max_pcs));
    CK(dalloc(&ctx->d_site_glob, c.max_pcs));
    CK(dalloc(&ctx->d_instr_g, (size_t)c.max_launches * n * 2));
    CK(dalloc(&ctx->d_launch_g, (size_t)c.max_launches * 2));
  }
  ctx->state = 1;
  return thermo_reset(ctx);
}

thermo_status thermo_set_launch_whitelist(thermo_ctx* ctx, const uint32_t* launches, size_t n) {
  thermo_status st = pre(ctx);
  if (st) return st;
  if (n && !launches) return fail(ctx, THERMO_EINVAL, "launch whitelist: null array");
  uint32_t bits[128] = {0};
  for (size_t i = 0; i < n; ++i) {
    if (launches[i] >= ctx->cfg.max_launches) return fail(ctx, THERMO_EINVAL, "launch whitelist: id >= max_launches");
    bits[launches[i] >> 5] |= 1u << (launches[i] & 31u);
  }
  if (!ctx->d_wl) CK(dalloc(&ctx->d_wl, 128));
  CK(cudaMemcpyAsync(ctx->d_wl, bits, sizeof bits, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));  // `bits` is on this stack frame
  ctx->wl_on = n > 0;
  return THERMO_OK;
}

thermo_status thermo_reset(thermo_ctx* ctx) {
  thermo_status st = pre(ctx);
  if (st) return st;
  if (ctx->state < 1) return fail(ctx, THERMO_ESTATE, "register objects first");
  const size_t n = ctx->reg.size();
  CK(cudaMemsetAsync(ctx->d_ctr, 0, sizeof(DevCounters), ctx->stream));
  CK(cudaMemsetAsync(ctx->d_instr, 0, (size_t)ctx->cfg.max_launches * n * 2 * 8, ctx->stream));
  CK(cudaMemsetAsync(ctx->d_launch_ctr, 0, (size_t)ctx->cfg.max_launches * 2 * 8, ctx->stream));
  CK(cudaMemsetAsync(ctx->d_pc_keys_tab, 0, (size_t)ctx->pc_cap * 8, ctx->stream));
  CK(cudaMemsetAsync(ctx->d_pc_vals, 0xFF, (size_t)ctx->pc_cap * 4, ctx->stream));
  ctx->n_keys = ctx->n_pckeys = 0;
  ctx->records = 0;
  ctx->state = 1;
  ctx->hist_valid = false;
  // the decoder counts keys per sector as it flushes them (one RED per key,
  // hidden in the issue-bound decode; measured cheaper than a histogram pass
  // over the keys at every sector count: synthetic 2^28 sectors 55.9 -> 52.7 ms)
  ctx->seg_counted = !ctx->comm && ctx->S_tot <= (1ull << 30) &&
                     (ctx->cfg.dedup == THERMO_DEDUP_AUTO || ctx->cfg.dedup == THERMO_DEDUP_SEGMENT);
  if (ctx->seg_counted) CK(cudaMemsetAsync(ctx->seg.cnt, 0, (ctx->S_tot + 1) * sizeof(uint32_t), ctx->stream));
  if (ctx->d_acc) CK(cudaMemsetAsync(ctx->d_acc, 0, 8 * ctx->S_tot * sizeof(uint32_t), ctx->stream));
  ctx->n_exch = 0;
  ctx->pc_mapped = 0;
  ctx->glob_sites.clear();
  ctx->glob_index.clear();
  ctx->have_glob = false;
  return THERMO_OK;
}

thermo_status thermo_ingest_trace(thermo_ctx* ctx, const thermo_record* recs, size_t n) {
  NvtxRange nvtx_("thermo_ingest_trace");
  thermo_status st = pre(ctx);
  if (st) return st;
  if (ctx->state < 1) return fail(ctx, THERMO_ESTATE, "register objects first");
  if (n == 0) return THERMO_OK;
  if (!recs) return fail(ctx, THERMO_EINVAL, "recs is NULL");
  if (reinterpret_cast<uintptr_t>(recs) & 15) return fail(ctx, THERMO_EINVAL, "recs must be 16-byte aligned");
  cudaPointerAttributes attr;
  bool on_device = false, pinned = false;
  if (cudaPointerGetAttributes(&attr, recs) == cudaSuccess) {
    on_device = attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged;
    pinned = attr.type == cudaMemoryTypeHost;
  } else {
    cudaGetLastError();
  }
  if (on_device && n >= (1ull << 32))
    return fail(ctx, THERMO_EINVAL, "a device-resident ingest call holds < 2^32 records (split at instr_start records)");
  // worst case: every record emits two keys (one per sector it touches)
  st = grow_keys(ctx, &ctx->d_keys, &ctx->keys_cap, ctx->n_keys + 2 * (ull)n + 64, ctx->n_keys);
  if (st) return st;
  CK(cudaEventRecord(ctx->ev0, ctx->stream));
  ctx->ms_kernel[THERMO_K_DECODE] = ctx->ms_kernel[THERMO_K_DECODE_GENERAL] = 0;
  if (on_device) {
    st = decode_device(ctx, reinterpret_cast<const uint4*>(recs), n, true);
    if (st) return st;
  } else {
    // staged host ingest: chunks split at explicit instruction heads, copy of
    // chunk k+1 overlapped with decoding of chunk k
    const unsigned char* src = reinterpret_cast<const unsigned char*>(recs);
    for (int i = 0; i < 2; ++i) {
      if (!ctx->d_stage[i]) CK(dalloc(&ctx->d_stage[i], kHostChunk + 4096));
      if (!pinned && !ctx->h_pinned[i]) CK(cudaHostAlloc(&ctx->h_pinned[i], (kHostChunk + 4096) * 16, 0));
    }
    ull pos = 0;
    int k = 0;
    while (pos < n) {
      ull end = n;
      if (pos + kHostChunk < n) {  // cut at the next explicit head (bounded look-ahead)
        const ull lim = std::min<ull>(n, pos + kHostChunk + 4096);
        ull e = pos + kHostChunk;
        while (e < lim) {
          uint32_t hiw;
          std::memcpy(&hiw, src + e * 16 + 4, 4);
          if ((hiw >> 23) & 1u) break;
          ++e;
        }
        end = e < lim ? e : n;  // no head within reach: take the rest in one piece
      }
      const ull cnt = end - pos;
      const int b = k & 1;
      if (cnt > kHostChunk + 4096) {
        // oversize tail (no instruction head in reach): one-off device buffer
        uint4* tmp = nullptr;
        CK(dalloc(&tmp, cnt));
        CK(cudaMemcpyAsync(tmp, src + pos * 16, cnt * 16, cudaMemcpyHostToDevice, ctx->stream));
        st = decode_device(ctx, tmp, cnt);
        CK(cudaStreamSynchronize(ctx->stream));
        dfree(tmp);
        if (st) return st;
        pos = end;
        ++k;
        continue;
      }
      CK(cudaEventSynchronize(ctx->ev_used[b]));  // staging buffer b free again
      const void* hsrc = src + pos * 16;
      if (!pinned) {
        std::memcpy(ctx->h_pinned[b], hsrc, cnt * 16);
        hsrc = ctx->h_pinned[b];
      }
      CK(cudaMemcpyAsync(ctx->d_stage[b], hsrc, cnt * 16, cudaMemcpyHostToDevice, ctx->copy_stream));
      CK(cudaEventRecord(ctx->ev_copied[b], ctx->copy_stream));
      CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_copied[b], 0));
      st = decode_device(ctx, ctx->d_stage[b], cnt);
      if (st) return st;
      CK(cudaEventRecord(ctx->ev_used[b], ctx->stream));
      pos = end;
      ++k;
    }
  }
  CK(cudaEventRecord(ctx->ev1, ctx->stream));
  st = sync_counts(ctx);
  if (st) return st;
  cudaEventElapsedTime(&ctx->ms_ingest, ctx->ev0, ctx->ev1);
  if (on_device) cudaEventElapsedTime(&ctx->ms_phase[0], ctx->evp[6], ctx->evp[7]);
  else ctx->ms_phase[0] = ctx->ms_ingest;
  ctx->records += n;
  ctx->state = 2;
  ctx->hist_valid = false;
  ctx->have_glob = false;
  return THERMO_OK;
}

thermo_status thermo_ingest_warp_trace(thermo_ctx* ctx, const thermo_warp_record* recs, size_t n) {
  NvtxRange nvtx_("thermo_ingest_warp_trace");
  thermo_status st = pre(ctx);
  if (st) return st;
  if (ctx->state < 1) return fail(ctx, THERMO_ESTATE, "register objects first");
  if (n == 0) return THERMO_OK;
  if (!recs) return fail(ctx, THERMO_EINVAL, "recs is NULL");
  if (reinterpret_cast<uintptr_t>(recs) & 15) return fail(ctx, THERMO_EINVAL, "recs must be 16-byte aligned");
  if (n >= (1ull << 27)) return fail(ctx, THERMO_EINVAL, "a warp-record ingest call holds < 2^27 instructions");
  cudaPointerAttributes attr;
  bool on_device = false;
  if (cudaPointerGetAttributes(&attr, recs) == cudaSuccess) {
    on_device = attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged;
  } else {
    cudaGetLastError();
  }
  cudaStream_t s = ctx->stream;
  // host records: chunks of kWarpChunk instructions copied on the copy stream
  // into two device staging buffers, each copy overlapped with the previous
  // chunk's decode (the device path is one chunk)
  // device records are decoded in the same chunks, so the spill space and the
  // key-buffer growth are bounded by one chunk, not by the whole call
  const ull C = std::min<ull>(n, on_device ? kWarpChunkDev : kWarpChunk);
  const ull lanes_max = 32 * C;
  if (ctx->spill_cap < lanes_max) {  // worst case: every instruction of a chunk spills
    dfree(ctx->d_spill);
    ctx->d_spill = nullptr;
    ctx->spill_cap = 0;
    if (dalloc(&ctx->d_spill, lanes_max) != cudaSuccess) return fail(ctx, THERMO_ENOMEM, "spill");
    ctx->spill_cap = lanes_max;
  }
  if (!on_device)
    for (int b = 0; b < 2; ++b)
      if (!ctx->d_wstage[b]) CK(dalloc(&ctx->d_wstage[b], kWarpChunk * 17));
  if (!ctx->d_wctr) CK(dalloc(&ctx->d_wctr, 2));
  CK(cudaEventRecord(ctx->ev0, s));
  CK(cudaEventRecord(ctx->evp[6], s));
  const unsigned char* hsrc = reinterpret_cast<const unsigned char*>(recs);
  auto issue_copy = [&](ull k) -> thermo_status {
    const int b = (int)(k & 1);
    const ull i0 = k * C, cnt = std::min<ull>(C, n - i0);
    CK(cudaEventSynchronize(ctx->ev_used[b]));  // staging buffer b free again
    CK(cudaMemcpyAsync(ctx->d_wstage[b], hsrc + i0 * 272, cnt * 272, cudaMemcpyHostToDevice, ctx->copy_stream));
    CK(cudaEventRecord(ctx->ev_copied[b], ctx->copy_stream));
    return THERMO_OK;
  };
  const ull nchunks = (n + C - 1) / C;
  if (!on_device && (st = issue_copy(0))) return st;
  ull lanes = 0;
  for (ull k = 0; k < nchunks; ++k) {
    const int b = (int)(k & 1);
    const ull i0 = k * C, cnt = std::min<ull>(C, n - i0);
    if (!on_device && k + 1 < nchunks && (st = issue_copy(k + 1))) return st;
    const uint4* drec = reinterpret_cast<const uint4*>(recs) + i0 * 17;
    if (!on_device) {
      CK(cudaStreamWaitEvent(s, ctx->ev_copied[b], 0));
      drec = ctx->d_wstage[b];
    }
    // worst case of this chunk: every lane record emits two keys
    if ((st = sync_counts(ctx))) return st;
    st = grow_keys(ctx, &ctx->d_keys, &ctx->keys_cap, ctx->n_keys + 2 * 32 * cnt + 64, ctx->n_keys);
    if (st) return st;
    CK(cudaMemsetAsync(ctx->d_wctr, 0, 2 * sizeof(ull), s));
    DecodeArgs a = decode_args(ctx);
    launch_decode_warp(a, drec, cnt, ctx->d_spill, ctx->d_wctr, ctx->num_sms, s);
    ctx->decoder_used = 3u;
    ctx->launches += 1;
    CK(cudaGetLastError());
    if (!on_device) CK(cudaEventRecord(ctx->ev_used[b], s));
    ull wc[2];
    CK(cudaMemcpyAsync(wc, ctx->d_wctr, sizeof wc, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (wc[0]) {  // spilled instructions: their per-lane records through the per-lane kernels
      st = decode_device(ctx, ctx->d_spill, wc[0]);
      if (st) return st;
    }
    lanes += wc[1];
  }
  CK(cudaEventRecord(ctx->evp[7], s));
  CK(cudaEventRecord(ctx->ev1, s));
  st = sync_counts(ctx);
  if (st) return st;
  cudaEventElapsedTime(&ctx->ms_ingest, ctx->ev0, ctx->ev1);
  cudaEventElapsedTime(&ctx->ms_phase[0], ctx->evp[6], ctx->evp[7]);
  ctx->records += lanes;
  ctx->state = 2;
  ctx->hist_valid = false;
  ctx->have_glob = false;
  return THERMO_OK;
}

thermo_status thermo_build_heatmap(thermo_ctx* ctx, thermo_granularity g, uint32_t launch_filter) {
  NvtxRange nvtx_("thermo_build_heatmap");
  thermo_status st = pre(ctx);
  if (st) return st;
  // (sharded: a rank may hold an empty slice; build is collective)
  if (ctx->state < (ctx->comm ? 1 : 2)) return fail(ctx, THERMO_ESTATE, "ingest a trace before build");
  if (g < THERMO_WORD || g > THERMO_BOTH) return fail(ctx, THERMO_EINVAL, "bad granularity");
  if (launch_filter != THERMO_ALL_LAUNCHES && launch_filter >= ctx->cfg.max_launches)
    return fail(ctx, THERMO_EINVAL, "launch_filter beyond max_launches");
  CollectiveScope coll(ctx);
  DevCounters hc;
  CK(cudaMemcpyAsync(&hc, ctx->d_ctr, sizeof hc, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (ctx->comm) {  // sharded: job-wide checks, pc ids and the key exchange (collective)
    st = dist_exchange(ctx, hc);
    if (st) return st;
  } else {
    if (hc.out_of_range) return fail(ctx, THERMO_ERANGE, "records with launch/warp ids beyond the declared widths");
    if (ctx->cfg.track_pc && hc.pc_overflow)
      return fail(ctx, THERMO_ERANGE, "more distinct (launch, pc) pairs than max_pcs");
  }
  const uint32_t* site_tab = ctx->comm ? ctx->d_site_glob : ctx->d_site_of;
  const ull n_pc = ctx->comm ? ctx->glob_sites.size() : hc.pc_count;
  const size_t n = ctx->reg.size();
  cudaStream_t s = ctx->stream;
  CK(cudaEventRecord(ctx->ev0, s));
  const ull l0 = ctx->launches;
  CK(cudaMemsetAsync(ctx->d_hist, 0, n * 2 * kLevels * 8, s));
  CK(cudaMemsetAsync(ctx->d_pchist, 0, (size_t)ctx->cfg.max_pcs * 2 * kLevels * 8, s));
  CK(cudaMemsetAsync(&ctx->d_ctr->distinct_pairs, 0, 2 * sizeof(ull), s));
  // AUTO, chosen by measurement: SEGMENT (counting sort by
  // sector + shared-memory hash set per chunk) beats the HBM hash set on every
  // BJ config (SGEMM 4.9 vs 6.3 ms; stencil 2^24 sectors 26 vs 62 ms; SpMV
  // 2^26 sectors 127 vs 170 ms; synthetic 2^28 sectors 60 vs 82 ms); its
  // per-sector workspace (28 B/sector) decides the limit
  uint32_t mode = ctx->cfg.dedup;
  const ull dense_words = (ull)ctx->cfg.max_launches * ctx->S_own * 8;  // DENSE masks (u64 each)
  if (mode == THERMO_DEDUP_AUTO) {
    if (ctx->cfg.block_warps >= 1 && ctx->cfg.block_warps <= 64 && dense_words * 8 <= (4ull << 30))
      mode = THERMO_DEDUP_DENSE;
    else
      mode = ctx->S_own <= (1ull << 30) ? THERMO_DEDUP_SEGMENT : THERMO_DEDUP_HASH;
  }
  if (mode != THERMO_DEDUP_SEGMENT) {  // (SEGMENT's chunk kernel writes every row, zeros included)
    CK(cudaMemsetAsync(ctx->d_wc, 0, 8 * ctx->S_own * sizeof(uint32_t), s));
    CK(cudaMemsetAsync(ctx->d_sc, 0, ctx->S_own * sizeof(uint32_t), s));
  }
  const KeyLayout kl = ctx->kl;
  cudaError_t e = cudaSuccess;
  bool pc_done = false;
  // measurement hook (SORT vs CUB): THERMO_DUMP_KEYS=<path> writes
  // the retained keys (u64, little-endian) and their prefix width to <path> at
  // build; never set in tests or the bench
  if (const char* dump = getenv("THERMO_DUMP_KEYS")) {
    std::vector<ull> hk(ctx->n_keys);
    if (ctx->n_keys) CK(cudaMemcpy(hk.data(), ctx->d_keys, ctx->n_keys * 8, cudaMemcpyDeviceToHost));
    if (FILE* f = fopen(dump, "wb")) {
      const ull hdr[2] = {ctx->n_keys, (ull)(kl.S + kl.L + kl.W + kl.P)};
      fwrite(hdr, 8, 2, f);
      fwrite(hk.data(), 8, hk.size(), f);
      fclose(f);
    }
  }
  // ---- a4 dedup + a5 count (+ a6 per-pc on the segment path) ----
  if (mode == THERMO_DEDUP_SEGMENT) {
    // counting sort by sector (two partition passes) + per-chunk shared-memory
    // dedup; the keys of sectors too big for a chunk (hot sectors: >= 2048
    // keys) are reduced one CTA per sector
    CK(cudaEventRecord(ctx->evp[0], s));
    uint32_t maxc = 0;
    ull n_big = 0;
    e = segment_prepare(ctx->d_keys, ctx->n_keys, kl, ctx->S_own, ctx->seg, ctx->num_sms, s, &maxc, &n_big,
                        ctx->seg_counted);
    if (e) return fail(ctx, THERMO_ECUDA, std::string("segment prepare: ") + cudaGetErrorString(e));
    if (ctx->sw.alt_cap < ctx->n_keys) {
      dfree(ctx->sw.alt);
      ctx->sw.alt_cap = ctx->n_keys + ctx->n_keys / 8 + 1024;
      CK(dalloc(&ctx->sw.alt, ctx->sw.alt_cap));
    }
    if (n_big && ctx->pckeys_cap < n_big) {  // the big keys' buffer (the pc-key buffer is free here)
      dfree(ctx->d_pckeys);
      ctx->pckeys_cap = n_big + n_big / 8 + 1024;
      CK(dalloc(&ctx->d_pckeys, ctx->pckeys_cap));
    }
    CK(cudaEventRecord(ctx->evp[1], s));
    e = segment_count(ctx->d_keys, ctx->n_keys, ctx->sw.alt, ctx->d_pckeys, kl, ctx->S_own, launch_filter, ctx->seg,
                      ctx->d_wc, ctx->d_sc, site_tab, ctx->cfg.track_pc ? ctx->d_pchist : nullptr, n_pc, ctx->d_ctr,
                      ctx->num_sms, s);
    if (e) return fail(ctx, THERMO_ECUDA, std::string("segment count: ") + cudaGetErrorString(e));
    ctx->launches += ctx->seg.launches;
    ctx->seg.launches = 0;
    pc_done = true;
    (void)maxc;
  }
  ctx->dedup_used = mode;
  if (mode == THERMO_DEDUP_SORT) {
    CK(cudaEventRecord(ctx->evp[0], s));
    ull* sorted =
        radix_sort_keys(ctx->d_keys, ctx->n_keys, 8, kl.S + kl.L + kl.W + kl.P, ctx->sw, ctx->num_sms, s, &e);
    CK(cudaEventRecord(ctx->evp[1], s));
    if (e) return fail(ctx, THERMO_ECUDA, std::string("radix sort: ") + cudaGetErrorString(e));
    if (sorted != ctx->d_keys) {  // keep the sorted copy as the retained keys
      std::swap(ctx->d_keys, ctx->sw.alt);
      std::swap(ctx->keys_cap, ctx->sw.alt_cap);
    }
    launch_count_sorted(ctx->d_keys, ctx->n_keys, kl, launch_filter, ctx->d_wc, ctx->d_sc, ctx->d_ctr, ctx->num_sms, s);
    ctx->launches += 1;
  } else if (mode == THERMO_DEDUP_DENSE) {
    // sampled-block mode: the paper's per-word warp bitmask per
    // (launch, word), OR-ed from the keys, then popcounted
    if (ctx->dense_cap < dense_words) {
      dfree(ctx->d_dense);
      ctx->dense_cap = 0;
      CK(dalloc(&ctx->d_dense, dense_words));
      ctx->dense_cap = dense_words;
    }
    CK(cudaEventRecord(ctx->evp[0], s));
    CK(cudaMemsetAsync(ctx->d_dense, 0, dense_words * 8, s));
    launch_dense_or(ctx->d_keys, ctx->n_keys, kl, ctx->cfg.block_id * ctx->cfg.block_warps, ctx->S_own,
                    ctx->d_dense, ctx->num_sms, s);
    CK(cudaEventRecord(ctx->evp[1], s));
    launch_dense_count(ctx->d_dense, ctx->cfg.max_launches, ctx->S_own, launch_filter, ctx->d_wc, ctx->d_sc,
                       ctx->d_ctr, ctx->num_sms, s);
    ctx->launches += 2;
  } else if (mode == THERMO_DEDUP_HASH) {
    ull cap = next_pow2(std::max<ull>(1024, 2 * ctx->n_keys));
    if (ctx->table_cap < cap) {
      dfree(ctx->d_table);
      ctx->table_cap = cap;
      CK(dalloc(&ctx->d_table, cap));
    }
    CK(cudaEventRecord(ctx->evp[0], s));
    CK(cudaMemsetAsync(ctx->d_table, 0xFF, cap * 8, s));
    launch_hash_insert(ctx->d_keys, ctx->n_keys, ctx->d_table, cap - 1, kl.P, ctx->d_ctr, ctx->num_sms, s);
    CK(cudaEventRecord(ctx->evp[1], s));
    ctx->launches += 2;
    launch_count_hash(ctx->d_table, cap, kl, launch_filter, ctx->d_wc, ctx->d_sc, ctx->d_ctr, ctx->num_sms, s);
  }
  CK(cudaGetLastError());
  CK(cudaEventRecord(ctx->evp[2], s));
  // ---- a6 histograms ----
  launch_object_hist(ctx->d_wc, ctx->d_sc, obj_table(ctx), ctx->d_nwords, ctx->d_hist, ctx->S_tot, ctx->S_own,
                     ctx->rank, ctx->nranks, ctx->num_sms, s);
  ctx->launches += 1;
  CK(cudaEventRecord(ctx->evp[3], s));
  if (ctx->cfg.track_pc && !pc_done) {
    // pc keys [pcid][g][mask] derived from the keys; deduplicated by sort
    // (SORT mode) or by a hash table bounded by n_pcs * S_tot (usually L2-sized)
    if (ctx->pckeys_cap < ctx->n_keys) {
      dfree(ctx->d_pckeys);
      ctx->pckeys_cap = ctx->n_keys + ctx->n_keys / 8 + 1024;
      CK(dalloc(&ctx->d_pckeys, ctx->pckeys_cap));
    }
    ctx->n_pckeys = ctx->n_keys;
    launch_pc_extract(ctx->d_keys, ctx->n_keys, kl, ctx->d_pckeys, ctx->num_sms, s);
    ctx->launches += 1;
    if (mode == THERMO_DEDUP_SORT) {
      ull* sorted = radix_sort_keys(ctx->d_pckeys, ctx->n_pckeys, 8, kl.P + kl.S, ctx->swpc, ctx->num_sms, s, &e);
      if (e) return fail(ctx, THERMO_ECUDA, std::string("radix sort (pc): ") + cudaGetErrorString(e));
      if (sorted != ctx->d_pckeys) {
        std::swap(ctx->d_pckeys, ctx->swpc.alt);
        std::swap(ctx->pckeys_cap, ctx->swpc.alt_cap);
      }
      ctx->launches += 1;
      launch_pc_hist_sorted(ctx->d_pckeys, ctx->n_pckeys, kl, site_tab, launch_filter, ctx->d_wc, ctx->d_sc,
                            ctx->d_pchist, ctx->d_ctr, ctx->num_sms, s);
    } else {
      const ull bound = std::min<ull>(ctx->n_pckeys, std::max<ull>(1, n_pc) * ctx->S_own);
      ull cap = next_pow2(std::max<ull>(1024, 2 * bound));
      if (ctx->pctable_cap < cap) {
        dfree(ctx->d_pctable);
        ctx->pctable_cap = cap;
        CK(dalloc(&ctx->d_pctable, cap));
      }
      CK(cudaMemsetAsync(ctx->d_pctable, 0xFF, cap * 8, s));
      launch_hash_insert(ctx->d_pckeys, ctx->n_pckeys, ctx->d_pctable, cap - 1, 0, ctx->d_ctr, ctx->num_sms, s);
      ctx->launches += 2;
      launch_pc_hist_hash(ctx->d_pctable, cap, kl, site_tab, launch_filter, ctx->d_wc, ctx->d_sc,
                          ctx->d_pchist, ctx->d_ctr, ctx->num_sms, s);
    }
  }
  CK(cudaGetLastError());
  CK(cudaEventRecord(ctx->evp[4], s));
  CK(cudaEventRecord(ctx->ev1, s));
  CK(cudaEventSynchronize(ctx->ev1));
  cudaEventElapsedTime(&ctx->ms_build, ctx->ev0, ctx->ev1);
  for (int i = 0; i < 4; ++i) cudaEventElapsedTime(&ctx->ms_phase[1 + i], ctx->evp[i], ctx->evp[i + 1]);
  for (int k = THERMO_K_SEG_SCAN; k <= THERMO_K_OBJECT_HIST; ++k) ctx->ms_kernel[k] = 0;
  ctx->ms_kernel[THERMO_K_SEG_SCAN] = ctx->dedup_used == THERMO_DEDUP_SEGMENT ? ctx->ms_phase[1] : 0.0;
  if (ctx->dedup_used == THERMO_DEDUP_SEGMENT) {
    float t = 0;
    for (int k = 0; k < 4; ++k)
      if (ctx->seg.ran[k] && cudaEventElapsedTime(&t, ctx->seg.ev[k], ctx->seg.ev[k + 1]) == cudaSuccess)
        ctx->ms_kernel[THERMO_K_SEG_COARSE + k] = t;
  }
  ctx->ms_kernel[THERMO_K_OBJECT_HIST] = ctx->ms_phase[3];
  ctx->launches += ctx->sw.launches + ctx->swpc.launches;
  ctx->sw.launches = ctx->swpc.launches = 0;
  (void)l0;
  if (ctx->comm) {
    st = dist_combine(ctx);
    if (st) return st;
  }
  DevCounters hc2;
  CK(cudaMemcpy(&hc2, ctx->d_ctr, sizeof hc2, cudaMemcpyDeviceToHost));
  if (hc2.hash_fail) return fail(ctx, THERMO_ECUDA, "hash table overflow");
  ctx->built_filter = launch_filter;
  ctx->built_gran = g;
  ctx->state = 3;
  ctx->hist_valid = true;
  return THERMO_OK;
}

thermo_status thermo_query_heatmap(thermo_ctx* ctx, uint32_t object_id, thermo_granularity g, uint32_t* out,
                                   size_t cap, size_t* n_out) {
  thermo_status st = pre(ctx);
  if (st) return st;
  if (ctx->state != 3) return fail(ctx, THERMO_ESTATE, "build the heat map first");
  auto it = ctx->id_to_reg.find(object_id);
  if (it == ctx->id_to_reg.end()) return fail(ctx, THERMO_EINVAL, "unknown object id");
  const uint32_t j = ctx->reg_to_sorted[it->second];
  const ull nw = ctx->h_nwords[j], ns = ctx->h_soff[j + 1] - ctx->h_soff[j], so = ctx->h_soff[j];
  size_t need = g == THERMO_WORD ? nw : g == THERMO_SECTOR ? ns : 9 * ns;
  if (n_out) *n_out = need;
  if (!out || cap < need) return fail(ctx, THERMO_ERANGE, "output capacity too small");
  if (ctx->nranks > 1) {
    // sharded: this rank's chunks of the object, from their local rows (one
    // copy of the contiguous local range), other ranks' cells 0
    const ull P = (ull)ctx->nranks, R = (ull)ctx->rank, C = kTileSectors;
    const ull c_lo = so / C, c_hi = (so + ns - 1) / C;
    ull f = c_lo + (R + P - c_lo % P) % P;  // first owned chunk >= c_lo
    std::memset(out, 0, need * 4);
    if (ns == 0 || f > c_hi) return THERMO_OK;
    const ull last = c_hi - (c_hi + P - R) % P;          // last owned chunk <= c_hi (>= f)
    const ull l0 = (f / P) * C, l1 = (last / P + 1) * C;   // local sectors [l0, l1)
    std::vector<uint32_t> hw(8 * (l1 - l0)), hs(l1 - l0);
    CK(cudaMemcpy(hw.data(), ctx->d_wc + 8 * l0, hw.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hs.data(), ctx->d_sc + l0, hs.size() * 4, cudaMemcpyDeviceToHost));
    for (ull c = f; c <= c_hi; c += P) {
      const ull gs0 = std::max(so, c * C), gs1 = std::min(so + ns, (c + 1) * C);
      for (ull gs = gs0; gs < gs1; ++gs) {
        const ull li = shard_local(gs, ctx->nranks) - l0, s2 = gs - so;
        for (int b = 0; b < 8; ++b) {
          const ull w = 8 * s2 + b;
          if (w >= nw) break;
          if (g == THERMO_WORD) out[w] = hw[8 * li + b];
          else if (g == THERMO_BOTH) out[9 * s2 + b] = hw[8 * li + b];
        }
        if (g == THERMO_SECTOR) out[s2] = hs[li];
        else if (g == THERMO_BOTH) out[9 * s2 + 8] = hs[li];
      }
    }
    return THERMO_OK;
  }
  if (g == THERMO_WORD) {
    CK(cudaMemcpy(out, ctx->d_wc + 8 * so, nw * 4, cudaMemcpyDeviceToHost));
  } else if (g == THERMO_SECTOR) {
    CK(cudaMemcpy(out, ctx->d_sc + so, ns * 4, cudaMemcpyDeviceToHost));
  } else {
    CK(cudaMemcpy2D(out, 9 * 4, ctx->d_wc + 8 * so, 8 * 4, 8 * 4, ns, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy2D(out + 8, 9 * 4, ctx->d_sc + so, 4, 4, ns, cudaMemcpyDeviceToHost));
    for (ull s2 = 0; s2 < ns; ++s2)
      for (int b = 0; b < 8; ++b)
        if (8 * s2 + b >= nw) out[9 * s2 + b] = 0;
  }
  return THERMO_OK;
}

thermo_status thermo_query_access(thermo_ctx* ctx, uint32_t object_id, uint32_t* out, size_t cap, size_t* n_out) {
  thermo_status st = pre(ctx);
  if (st) return st;
  if (!ctx->d_acc) return fail(ctx, THERMO_ESTATE, "context created with track_access = 0");
  auto it = ctx->id_to_reg.find(object_id);
  if (it == ctx->id_to_reg.end()) return fail(ctx, THERMO_EINVAL, "unknown object id");
  const uint32_t j = ctx->reg_to_sorted[it->second];
  const ull nw = ctx->h_nwords[j], so = ctx->h_soff[j];
  if (n_out) *n_out = nw;
  if (!out || cap < nw) return fail(ctx, THERMO_ERANGE, "output capacity too small");
  CK(cudaStreamSynchronize(ctx->stream));
  CK(cudaMemcpy(out, ctx->d_acc + 8 * so, nw * 4, cudaMemcpyDeviceToHost));
  return THERMO_OK;
}

thermo_status thermo_query_runs(thermo_ctx* ctx, uint32_t object_id, thermo_run* out, size_t cap, size_t* n_out) {
  thermo_status st = pre(ctx);
  if (st) return st;
  if (ctx->state != 3) return fail(ctx, THERMO_ESTATE, "build the heat map first");
  if (ctx->comm) return fail(ctx, THERMO_ESTATE, "sharded mode: rows are partitioned across ranks");
  auto it = ctx->id_to_reg.find(object_id);
  if (it == ctx->id_to_reg.end()) return fail(ctx, THERMO_EINVAL, "unknown object id");
  const uint32_t j = ctx->reg_to_sorted[it->second];
  const ull ns = ctx->h_soff[j + 1] - ctx->h_soff[j], so = ctx->h_soff[j], nw = ctx->h_nwords[j];
  uint32_t* scratch = nullptr;
  CK(dalloc(&scratch, (ns + 2047) / 2048 + 1));
  ull n = 0;
  cudaError_t e = compress_runs(ctx->d_wc, ctx->d_sc, so, ns, nw, scratch, ctx->d_tmp, nullptr, 0, &n, ctx->stream);
  if (e) { dfree(scratch); return fail(ctx, THERMO_ECUDA, std::string("runs: ") + cudaGetErrorString(e)); }
  if (n_out) *n_out = n;
  if (!out || cap < n) { dfree(scratch); return fail(ctx, THERMO_ERANGE, "output capacity too small"); }
  thermo_run* d_out = nullptr;
  if (dalloc(&d_out, n) != cudaSuccess) { dfree(scratch); return fail(ctx, THERMO_ENOMEM, "runs"); }
  e = compress_runs(ctx->d_wc, ctx->d_sc, so, ns, nw, scratch, ctx->d_tmp, d_out, n, &n, ctx->stream);
  if (!e) e = cudaMemcpyAsync(out, d_out, n * sizeof(thermo_run), cudaMemcpyDeviceToHost, ctx->stream);
  if (!e) e = cudaStreamSynchronize(ctx->stream);
  dfree(scratch);
  dfree(d_out);
  if (e) return fail(ctx, THERMO_ECUDA, std::string("runs: ") + cudaGetErrorString(e));
  return THERMO_OK;
}

thermo_status thermo_query_histogram(thermo_ctx* ctx, uint32_t object_id, thermo_granularity g,
                                     uint64_t hist[THERMO_LEVELS]) {
  thermo_status st = pre(ctx);
  if (st) return st;
  if (ctx->state != 3) return fail(ctx, THERMO_ESTATE, "build the heat map first");
  if (g != THERMO_WORD && g != THERMO_SECTOR) return fail(ctx, THERMO_EINVAL, "granularity must be WORD or SECTOR");
  auto it = ctx->id_to_reg.find(object_id);
  if (it == ctx->id_to_reg.end()) return fail(ctx, THERMO_EINVAL, "unknown object id");
  const uint32_t j = ctx->reg_to_sorted[it->second];
  const size_t off = ((size_t)j * 2 + (g == THERMO_SECTOR ? 1 : 0)) * kLevels;
  CK(cudaMemcpy(hist, ctx->d_hist + off, kLevels * 8, cudaMemcpyDeviceToHost));
  return THERMO_OK;
}

thermo_status thermo_query_per_pc(thermo_ctx* ctx, thermo_granularity g, thermo_pc_hist* out, size_t cap,
                                  size_t* n_out) {
  thermo_status st = pre(ctx);
  if (st) return st;
  if (ctx->state != 3) return fail(ctx, THERMO_ESTATE, "build the heat map first");
  if (!ctx->cfg.track_pc) return fail(ctx, THERMO_ESTATE, "context created with track_pc = 0");
  if (g != THERMO_WORD && g != THERMO_SECTOR) return fail(ctx, THERMO_EINVAL, "granularity must be WORD or SECTOR");
  DevCounters hc;
  CK(cudaMemcpy(&hc, ctx->d_ctr, sizeof hc, cudaMemcpyDeviceToHost));
  const ull npc = ctx->comm ? ctx->glob_sites.size() : std::min<ull>(hc.pc_count, ctx->cfg.max_pcs);
  std::vector<uint32_t> site(npc);
  std::vector<ull> hist(npc * 2 * kLevels);
  if (npc) {
    if (ctx->comm) site = ctx->glob_sites;
    else CK(cudaMemcpy(site.data(), ctx->d_site_of, npc * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hist.data(), ctx->d_pchist, npc * 2 * kLevels * 8, cudaMemcpyDeviceToHost));
  }
  std::vector<uint32_t> ids;
  for (uint32_t i = 0; i < npc; ++i)
    if (ctx->built_filter == THERMO_ALL_LAUNCHES || (site[i] >> 20) == ctx->built_filter) ids.push_back(i);
  std::sort(ids.begin(), ids.end(), [&](uint32_t a, uint32_t b) { return site[a] < site[b]; });
  if (n_out) *n_out = ids.size();
  if (!out || cap < ids.size()) return fail(ctx, THERMO_ERANGE, "output capacity too small");
  for (size_t k = 0; k < ids.size(); ++k) {
    const uint32_t i = ids[k];
    out[k].launch = site[i] >> 20;
    out[k].pc = (site[i] & 0xFFFFFu) << 4;
    const size_t off = ((size_t)i * 2 + (g == THERMO_SECTOR ? 1 : 0)) * kLevels;
    std::memcpy(out[k].hist, hist.data() + off, kLevels * 8);
  }
  return THERMO_OK;
}

thermo_status thermo_classify(thermo_ctx* ctx, const thermo_params* params, thermo_indicators* out, size_t cap,
                              size_t* n_out) {
  NvtxRange nvtx_("thermo_classify");
  thermo_status st = pre(ctx);
  if (st) return st;
  if (ctx->state != 3) return fail(ctx, THERMO_ESTATE, "build the heat map first");
  const size_t n = ctx->reg.size();
  if (n_out) *n_out = n;
  if (!out || cap < n) return fail(ctx, THERMO_ERANGE, "output capacity too small");
  thermo_params p;
  if (params) p = *params; else thermo_default_params(&p);
  if (!p.alpha_den || !p.beta_den || !p.smem_cov_den || !p.gamma_den || !p.dom_den || !p.hot_frac_den ||
      !p.fs_frac_den || !p.mis_frac_den || !p.cv_den)
    return fail(ctx, THERMO_EINVAL, "zero denominator in params");
  cudaStream_t s = ctx->stream;
  CK(cudaEventRecord(ctx->ev0, s));
  CK(cudaMemsetAsync(ctx->d_ind, 0, n * kIndFields * 8, s));
  IndicatorArgs a{};
  a.word_cnt = ctx->d_wc;
  a.sector_cnt = ctx->d_sc;
  a.obj = obj_table(ctx);
  a.obj_nwords = ctx->d_nwords;
  a.obj_space = ctx->d_space;
  a.tile_obj = ctx->d_tile_obj;
  a.tile_first = ctx->d_tile_first;
  a.tile_end = ctx->d_tile_end;
  a.n_tiles = ctx->n_tiles;
  a.instr_ctr = ctx->comm ? ctx->d_instr_g : ctx->d_instr;
  a.max_launches = ctx->cfg.max_launches;
  a.launch_filter = ctx->built_filter;
  a.prm = p;
  a.ind = ctx->d_ind;
  a.tile_info = ctx->d_tile_info;
  a.tile_prev = ctx->d_tile_prev;
  a.rank = (uint32_t)ctx->rank;
  a.nranks = (uint32_t)ctx->nranks;
  if (!ctx->comm) {
    launch_indicators(a, ctx->num_sms, s);
    ctx->launches += ctx->n_tiles ? 4 : 2;
  } else {
    // sharded: each rank scans its own tiles; sums, maxima, tile summaries and
    // verify counts are combined between the steps (collective)
    CollectiveScope coll(ctx);
    Comm* c = ctx->comm;
    const size_t need = n * kIndSumFields + n + 1;
    if (ctx->red_cap < need) {
      dfree(ctx->d_red);
      ctx->d_red = nullptr;
      ctx->red_cap = 0;
      CK(dalloc(&ctx->d_red, need));
      ctx->red_cap = need;
    }
    ull* sums = ctx->d_red;
    ull* maxs = sums + n * kIndSumFields;
    launch_indicator_tiles(a, 0, s);
    launch_indicator_pack(ctx->d_ind, (uint32_t)n, sums, maxs, nullptr, 0, s);
    DCK(c->allreduce(sums, n * kIndSumFields, false, s));
    DCK(c->allreduce(maxs, n, true, s));
    if (ctx->n_tiles) DCK(c->allreduce(ctx->d_tile_info, (size_t)ctx->n_tiles * kTileInfo, false, s));
    launch_indicator_pack(ctx->d_ind, (uint32_t)n, sums, maxs, nullptr, 1, s);
    launch_indicator_stitch(a, s);
    launch_indicator_tiles(a, 1, s);
    launch_indicator_pack(ctx->d_ind, (uint32_t)n, nullptr, nullptr, sums, 0, s);
    DCK(c->allreduce(sums, n, false, s));
    launch_indicator_pack(ctx->d_ind, (uint32_t)n, nullptr, nullptr, sums, 1, s);
    launch_indicator_finalize(a, s);
    ctx->launches += ctx->n_tiles ? 8 : 6;
    DCK(c->wait(s));
  }
  CK(cudaGetLastError());
  CK(cudaEventRecord(ctx->ev1, s));
  std::vector<ull> ind(n * kIndFields);
  CK(cudaMemcpyAsync(ind.data(), ctx->d_ind, n * kIndFields * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  cudaEventElapsedTime(&ctx->ms_classify, ctx->ev0, ctx->ev1);
  ctx->ms_phase[5] = ctx->ms_classify;
  ctx->ms_kernel[THERMO_K_INDICATORS] = ctx->ms_classify;
  for (size_t r = 0; r < n; ++r) {
    const ull* v = ind.data() + ctx->reg_to_sorted[r] * kIndFields;
    thermo_indicators& o = out[r];
    o.object_id = ctx->reg[r].id;
    o.labels = (uint32_t)v[F_LABELS];
    o.n_words = v[F_NWORDS]; o.n_sectors = v[F_NSECTORS];
    o.touched_sectors = v[F_T]; o.touched_words = v[F_TW];
    o.hot_sectors = v[F_HOT]; o.fs_sectors = v[F_FS];
    o.sum_x = v[F_SUMX]; o.sum_x2_lo = v[F_SUMX2_LO]; o.sum_x2_hi = v[F_SUMX2_HI];
    o.le1_words = v[F_LE1]; o.max_sector_count = v[F_MAXSEC];
    o.instrs = v[F_INSTRS]; o.misaligned_instrs = v[F_MIS];
    o.gaps = v[F_GAPS]; o.dom_gap = v[F_DOMGAP]; o.dom_count = v[F_DOMCNT];
  }
  return THERMO_OK;
}

thermo_status thermo_get_stats(thermo_ctx* ctx, thermo_stats* out) {
  thermo_status st = pre(ctx);
  if (st) return st;
  if (!out) return THERMO_EINVAL;
  std::memset(out, 0, sizeof *out);
  DevCounters hc;
  CK(cudaMemcpyAsync(&hc, ctx->d_ctr, sizeof hc, cudaMemcpyDeviceToHost, ctx->stream));
  std::vector<ull> lc;
  if (ctx->state >= 1) {
    lc.resize((size_t)ctx->cfg.max_launches * 2);
    CK(cudaMemcpyAsync(lc.data(), ctx->d_launch_ctr, lc.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  if (ctx->comm && ctx->have_glob) {  // sharded, after a build: job-wide totals
    CK(cudaMemcpy(lc.data(), ctx->d_launch_g, lc.size() * 8, cudaMemcpyDeviceToHost));
    std::memcpy(&hc, ctx->h_ctr_g, sizeof hc);
    hc.pc_count = ctx->glob_sites.size();
  }
  out->records = ctx->comm && ctx->have_glob ? ctx->h_ctr_g[16] : ctx->records;
  out->invalid = hc.invalid;
  out->out_of_range = hc.out_of_range;
  for (uint32_t la = 0; la < ctx->cfg.max_launches && !lc.empty(); ++la) {
    if (ctx->state == 3 && ctx->built_filter != THERMO_ALL_LAUNCHES && la != ctx->built_filter) continue;
    out->unmapped_words += lc[2 * la];
    out->mapped_word_accesses += lc[2 * la + 1];
  }
  out->keys_emitted = hc.n_keys;
  out->pc_keys_emitted = hc.n_pckeys;
  out->distinct_pairs = hc.distinct_pairs;
  out->distinct_pc_pairs = hc.distinct_pc;
  out->n_pcs = hc.pc_count;
  out->dedup_used = ctx->dedup_used;
  out->decoder_used = ctx->decoder_used;
  out->ms_ingest = ctx->ms_ingest;
  out->ms_build = ctx->ms_build;
  out->ms_classify = ctx->ms_classify;
  out->ms_decode = ctx->ms_phase[0];
  out->ms_dedup = ctx->ms_phase[1];
  out->ms_count = ctx->ms_phase[2];
  out->ms_hist = ctx->ms_phase[3];
  out->ms_pc = ctx->ms_phase[4];
  out->ms_indicators = ctx->ms_phase[5];
  out->kernel_launches = ctx->launches;
  out->ms_exchange = ctx->ms_exchange;
  out->exchange_bytes = ctx->exchange_bytes;
  for (int k = 0; k < 9; ++k) out->ms_kernel[k] = ctx->ms_kernel[k];
  out->local_sectors = ctx->S_own;
  out->local_keys = ctx->n_keys;
  return THERMO_OK;
}

const char* thermo_last_error(const thermo_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

}  // extern "C"
