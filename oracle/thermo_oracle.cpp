// =============================================================================
// thermo_oracle.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, single-threaded CPU oracle for the cuThermo heat-map
// reduction (arXiv 2507.18729).  Only tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py may load this library.  The
// product path (paper_2507_18729_b200/, libthermo) never links, imports or
// calls it, and this file shares no code, header, table or constant generator
// with the CUDA path.
//
// Citation keys: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n,
// G# = ambiguity-ledger reading in DESIGN.md (section "Readings").
//
// What it computes (the plain definition, §IV-A1, §IV-B2):
//   * temperature of a 4-byte word  = number of distinct warps that accessed it
//   * temperature of a 32-byte sector = number of distinct warps that accessed
//     any of its 8 words (P:325 ORs every access into the sector's 9th mask)
//   A "warp" is the pair (launch, global warp id) (G1, G2).  Instead of the
//   paper's 64-bit bitmask (which caps warp ids at 63) the oracle keeps an
//   explicit std::set of warps per word -- the definition written out.
//
// Everything else (levels, histograms, per-PC histograms, indicators, labels)
// follows DESIGN.md §Readings step by step; each function names its passage.
// =============================================================================
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <array>
#include <map>
#include <set>
#include <unordered_map>
#include <vector>

namespace {

// ---- record fields (§IV-B1 flattened per lane) --
struct Rec {
  uint64_t addr;     // byte address, 48 bits (G5)
  uint32_t size;     // 1,2,4,8,16 bytes (G4)
  uint32_t kind;     // 0 load, 1 store, 2 atomic (G7: all kinds count)
  uint32_t space;    // 0 global, 1 shared, 2 local
  bool instr_start;  // first lane record of a warp-level instruction (G14/G24)
  bool valid;
  uint32_t warp;     // global warp id within its launch (G1)
  uint32_t pc;       // byte pc
  uint32_t launch;   // launch id (G2)
};

Rec parse(const unsigned char* p) {
  uint64_t af;
  uint32_t warp, site;
  std::memcpy(&af, p, 8);
  std::memcpy(&warp, p + 8, 4);
  std::memcpy(&site, p + 12, 4);
  Rec r;
  r.addr = af & ((uint64_t(1) << 48) - 1);
  uint32_t log2size = uint32_t((af >> 48) & 7);
  r.kind = uint32_t((af >> 51) & 3);
  r.space = uint32_t((af >> 53) & 3);
  r.instr_start = ((af >> 55) & 1) != 0;
  uint32_t reserved = uint32_t(af >> 56);
  r.size = 1u << (log2size > 4 ? 0 : log2size);
  r.valid = log2size <= 4 && r.kind <= 2 && r.space <= 2 && reserved == 0 &&
            r.addr + r.size <= (uint64_t(1) << 48);
  r.warp = warp;
  r.pc = (site & 0xFFFFFu) << 4;
  r.launch = site >> 20;
  return r;
}

struct Obj {
  uint64_t base, len;
  uint32_t space, id;
  uint64_t n_words() const { return (len + 3) / 4; }     // G9
  uint64_t n_sectors() const { return (len + 31) / 32; } // G9
};

// bit_width(c): level 0 = untouched, 1 = one warp, 2 = 2-3, ... (G10)
int level_of(uint64_t c) {
  int l = 0;
  while (c) { ++l; c >>= 1; }
  return l;
}

typedef unsigned __int128 u128;

struct Oracle {
  std::vector<Obj> objs;  // in registration order
  // sampled-block scope: block_warps != 0 keeps
  // only the records of global block `block_id` (warp / block_warps); the others
  // were never traced
  uint32_t block_warps = 0, block_id = 0;
  // kernel sampling by whitelist: when non-empty, only the records of
  // launches l with launch_ok[l] are traced; the others are as never traced
  std::vector<bool> launch_ok;
  // restriction (sampled mode): only these (object index, local sector) pairs
  bool restricted = false;
  std::set<std::pair<uint32_t, uint64_t>> allow;
  // restricted build: the allowed sectors' rows only (8 word counts, sector count)
  std::map<std::pair<uint32_t, uint64_t>, std::array<uint32_t, 9>> sampled;

  // Wset[(o, w)] = set of (launch<<32 | warp)  (written as a set)
  std::unordered_map<uint64_t, std::set<uint64_t>> wset;
  // per-PC: (launch<<32 | pc) -> set of (o, w)        (G11)
  std::map<uint64_t, std::set<std::pair<uint32_t, uint64_t>>> pcset;
  // access counts: lane accesses per word,
  // over every ingested launch (G27)
  std::unordered_map<uint64_t, uint64_t> access;
  // misalignment counters per (launch, o)   (G24)
  std::map<std::pair<uint32_t, uint32_t>, std::pair<uint64_t, uint64_t>> instr;
  // stats
  uint64_t n_records = 0, n_invalid = 0;
  std::map<uint32_t, uint64_t> unmapped_by_launch, mapped_by_launch;

  // ---- results of build() ----
  uint32_t filter = 0xFFFFFFFFu;
  std::vector<std::vector<uint32_t>> word_count, sector_count;  // per object
  std::vector<std::vector<uint64_t>> hist_word, hist_sector;    // per object [33]
  struct PcRow { uint32_t launch, pc; uint64_t hw[33], hs[33]; };
  std::vector<PcRow> pcrows;
  bool built = false;

  static uint64_t wkey(uint32_t o, uint64_t w) { return (uint64_t(o) << 48) | w; }

  // object lookup: the object whose [base, base+len) holds byte 4w in `space`
  // (S:154-162 region_lookup; G8 unmapped words are dropped and counted)
  int lookup(uint32_t space, uint64_t byte) const {
    for (size_t i = 0; i < objs.size(); ++i)
      if (objs[i].space == space && objs[i].base <= byte && byte < objs[i].base + objs[i].len)
        return int(i);
    return -1;
  }

  void ingest(const unsigned char* recs, size_t n) {
    // instruction state (G24): a call starts a new instruction at its first record
    bool in_instr = false, has_valid = false;
    uint32_t i_launch = 0;
    int i_obj = -1;
    uint64_t i_min = 0, i_max = 0;
    std::set<uint64_t> i_sectors;
    auto close_instr = [&]() {
      if (in_instr && has_valid && i_obj >= 0) {
        auto& c = instr[{i_launch, uint32_t(i_obj)}];
        c.first += 1;
        uint64_t span = i_max - i_min + 1;
        if (uint64_t(i_sectors.size()) > (span + 31) / 32) c.second += 1;
      }
      in_instr = false; has_valid = false; i_obj = -1; i_sectors.clear();
    };
    size_t pos = 0;  // record position within the current instruction
    for (size_t k = 0; k < n; ++k) {
      Rec r = parse(recs + 16 * k);
      ++n_records;
      // an instruction has at most 32 lane records ("32-element array");
      // a longer run without instr_start is split every 32 records (G24)
      if (k == 0 || r.instr_start || pos == 32) { close_instr(); in_instr = true; pos = 0; }
      ++pos;
      if (block_warps && r.warp / block_warps != block_id) continue;  // outside the sampled block
      if (!launch_ok.empty() && (r.launch >= launch_ok.size() || !launch_ok[r.launch])) continue;  // not whitelisted
      if (!r.valid) { ++n_invalid; continue; }
      // ---- instruction extent (Fig.6) ----
      uint64_t lo = (uint64_t(r.space) << 48) | r.addr;
      uint64_t hi = lo + r.size - 1;
      for (uint64_t s = lo >> 5; s <= (hi >> 5); ++s) i_sectors.insert(s);
      if (!has_valid) {
        has_valid = true;
        i_launch = r.launch;
        i_obj = lookup(r.space, (r.addr >> 2) << 2);
        i_min = lo; i_max = hi;
      } else {
        i_min = std::min(i_min, lo);
        i_max = std::max(i_max, hi);
      }
      // ---- words touched (G3/G4) ----
      uint64_t w0 = r.addr >> 2, w1 = (r.addr + r.size - 1) >> 2;
      for (uint64_t w = w0; w <= w1; ++w) {
        int o = lookup(r.space, w * 4);
        if (o < 0) { unmapped_by_launch[r.launch] += 1; continue; }
        mapped_by_launch[r.launch] += 1;
        uint64_t wl = w - objs[o].base / 4;  // object-local word index
        if (restricted && !allow.count({uint32_t(o), wl / 8})) continue;
        wset[wkey(uint32_t(o), wl)].insert((uint64_t(r.launch) << 32) | r.warp);
        access[wkey(uint32_t(o), wl)] += 1;  // every access, not distinct warps (Fig. 3 baseline)
        pcset[(uint64_t(r.launch) << 32) | r.pc].insert({uint32_t(o), wl});
      }
    }
    close_instr();
  }

  bool pass(uint64_t lw) const { return filter == 0xFFFFFFFFu || uint32_t(lw >> 32) == filter; }

  size_t filtered_size(const std::set<uint64_t>& s) const {
    size_t c = 0;
    for (uint64_t lw : s) c += pass(lw) ? 1 : 0;
    return c;
  }

  // one sector's row, straight from the sets (G6)
  std::array<uint32_t, 9> sector_row(uint32_t o, uint64_t s) const {
    std::array<uint32_t, 9> row{};
    std::set<uint64_t> u;
    for (uint64_t b = 0; b < 8; ++b) {
      auto it = wset.find(wkey(o, 8 * s + b));
      if (it == wset.end()) continue;
      row[b] = uint32_t(filtered_size(it->second));
      for (uint64_t lw : it->second) if (pass(lw)) u.insert(lw);
    }
    row[8] = uint32_t(u.size());
    return row;
  }

  void build(uint32_t f) {
    filter = f;
    size_t no = objs.size();
    if (restricted) {  // sampled mode: only the allowed sectors' rows (no dense arrays;
      // dense queries, histograms and indicators then read empty / zero)
      word_count.assign(no, {});
      sector_count.assign(no, {});
      hist_word.assign(no, std::vector<uint64_t>(33, 0));
      hist_sector.assign(no, std::vector<uint64_t>(33, 0));
      pcrows.clear();
      sampled.clear();
      for (auto& os : allow) sampled[os] = sector_row(os.first, os.second);
      built = true;
      return;
    }
    word_count.assign(no, {});
    sector_count.assign(no, {});
    hist_word.assign(no, std::vector<uint64_t>(33, 0));
    hist_sector.assign(no, std::vector<uint64_t>(33, 0));
    for (size_t o = 0; o < no; ++o) {
      uint64_t nw = objs[o].n_words(), ns = objs[o].n_sectors();
      word_count[o].assign(nw, 0);
      sector_count[o].assign(ns, 0);
      // word temperature = |Wset| ("count the number of 1s")
      for (uint64_t w = 0; w < nw; ++w) {
        auto it = wset.find(wkey(uint32_t(o), w));
        if (it != wset.end()) word_count[o][w] = uint32_t(filtered_size(it->second));
      }
      // sector temperature = |union of its words' sets| (G6)
      for (uint64_t s = 0; s < ns; ++s) {
        std::set<uint64_t> u;
        for (uint64_t b = 0; b < 8; ++b) {
          auto it = wset.find(wkey(uint32_t(o), 8 * s + b));
          if (it == wset.end()) continue;
          for (uint64_t lw : it->second) if (pass(lw)) u.insert(lw);
        }
        sector_count[o][s] = uint32_t(u.size());
      }
      // histograms of levels (P:351 legend; G10)
      for (uint64_t w = 0; w < nw; ++w) hist_word[o][level_of(word_count[o][w])] += 1;
      for (uint64_t s = 0; s < ns; ++s) hist_sector[o][level_of(sector_count[o][s])] += 1;
    }
    // per-PC histograms (G11): distinct (launch, pc, word) pairs, each adds 1 at
    // the word's level; distinct (launch, pc, sector) pairs likewise.
    pcrows.clear();
    for (auto& kv : pcset) {
      uint32_t launch = uint32_t(kv.first >> 32), pc = uint32_t(kv.first);
      if (filter != 0xFFFFFFFFu && launch != filter) continue;
      PcRow row;
      row.launch = launch; row.pc = pc;
      std::memset(row.hw, 0, sizeof row.hw);
      std::memset(row.hs, 0, sizeof row.hs);
      std::set<std::pair<uint32_t, uint64_t>> sectors;
      for (auto& ow : kv.second) {
        row.hw[level_of(word_count[ow.first][ow.second])] += 1;
        sectors.insert({ow.first, ow.second / 8});
      }
      for (auto& os : sectors) row.hs[level_of(sector_count[os.first][os.second])] += 1;
      pcrows.push_back(row);
    }
    built = true;
  }
};

}  // namespace

// ----------------------------------------------------------------------------
// C ABI used by oracle/__init__.py (ctypes).  Objects: {base, len, space, id}.
// ----------------------------------------------------------------------------
struct orc_object { uint64_t base, len; uint32_t space, id; };

// per-object indicator block written by orc_classify (all u64)
enum {
  I_NWORDS, I_NSECTORS, I_T, I_TW, I_HOT, I_FS, I_SUMX, I_SUMX2_LO, I_SUMX2_HI,
  I_LE1, I_MAXSEC, I_INSTRS, I_MIS, I_GAPS, I_DOMGAP, I_DOMCNT, I_LABELS, I_COUNT
};
// params (u64, exact rationals): see DESIGN.md "Pattern parameters"
enum {
  P_THETA_HOT, P_ALPHA_NUM, P_ALPHA_DEN, P_BETA_NUM, P_BETA_DEN, P_FS_MIN,
  P_SMEM_CAP, P_SMEM_COV_NUM, P_SMEM_COV_DEN, P_GAMMA_NUM, P_GAMMA_DEN,
  P_STRIDED_MIN, P_DOM_NUM, P_DOM_DEN, P_HOTF_NUM, P_HOTF_DEN, P_FSF_NUM,
  P_FSF_DEN, P_MISF_NUM, P_MISF_DEN, P_CV_NUM, P_CV_DEN, P_COUNT
};
enum {
  L_HOT = 1, L_RANDOM_HOT = 2, L_FALSE_SHARING = 4, L_SMEM_THREAD_LOCAL = 8,
  L_SMEM_WARP_PRIVATE = 16, L_MISALIGNED = 32, L_STRIDED = 64
};

extern "C" {

void* orc_new(const orc_object* objs, size_t n) {
  Oracle* o = new Oracle();
  for (size_t i = 0; i < n; ++i)
    o->objs.push_back(Obj{objs[i].base, objs[i].len, objs[i].space, objs[i].id});
  return o;
}

void orc_free(void* h) { delete static_cast<Oracle*>(h); }

// sampled mode: only words of the listed (object index, local sector) pairs are
// recorded; histograms are then meaningless, counts at the listed sectors exact.
void orc_restrict(void* h, const uint32_t* obj_idx, const uint64_t* sectors, size_t n) {
  Oracle* o = static_cast<Oracle*>(h);
  o->restricted = true;
  for (size_t i = 0; i < n; ++i) o->allow.insert({obj_idx[i], sectors[i]});
}

// warp-instruction records (include/thermo.h
// thermo_warp_record): one warp instruction with its 32 lane addresses
// is, by definition, the per-lane records of its active lanes in lane order,
// the first carrying instr_start; written out here and ingested as one call.
void orc_ingest_warp(void* h, const void* recs, size_t n) {
  const unsigned char* p = static_cast<const unsigned char*>(recs);
  std::vector<unsigned char> lanes;
  lanes.reserve(n * 32 * 16);
  for (size_t i = 0; i < n; ++i) {
    const unsigned char* r = p + 272 * i;
    uint32_t warp, site, active, flags;
    std::memcpy(&warp, r, 4);
    std::memcpy(&site, r + 4, 4);
    std::memcpy(&active, r + 8, 4);
    std::memcpy(&flags, r + 12, 4);
    bool first = true;
    for (int l = 0; l < 32; ++l) {
      if (!((active >> l) & 1u)) continue;
      uint64_t addr;
      std::memcpy(&addr, r + 16 + 8 * l, 8);
      const uint64_t reserved = ((addr >> 48) != 0 || (flags >> 7) != 0) ? 1 : 0;
      const uint64_t af = (addr & ((uint64_t(1) << 48) - 1)) | (uint64_t(flags & 7) << 48) |
                          (uint64_t((flags >> 3) & 3) << 51) | (uint64_t((flags >> 5) & 3) << 53) |
                          (uint64_t(first ? 1 : 0) << 55) | (reserved << 56);
      first = false;
      unsigned char q[16];
      std::memcpy(q, &af, 8);
      std::memcpy(q + 8, &warp, 4);
      std::memcpy(q + 12, &site, 4);
      lanes.insert(lanes.end(), q, q + 16);
    }
  }
  static_cast<Oracle*>(h)->ingest(lanes.data(), lanes.size() / 16);
}

// sampled-block scope: only block `block` of `warps_per_block` warps
void orc_block_scope(void* h, uint32_t warps_per_block, uint32_t block) {
  Oracle* o = static_cast<Oracle*>(h);
  o->block_warps = warps_per_block;
  o->block_id = block;
}

// kernel whitelist: only launches listed are traced; n = 0 traces all
void orc_launch_whitelist(void* h, const uint32_t* launches, size_t n) {
  Oracle* o = static_cast<Oracle*>(h);
  o->launch_ok.clear();
  for (size_t i = 0; i < n; ++i) {
    if (launches[i] >= o->launch_ok.size()) o->launch_ok.resize(launches[i] + 1, false);
    o->launch_ok[launches[i]] = true;
  }
}

void orc_ingest(void* h, const void* recs, size_t n) {
  static_cast<Oracle*>(h)->ingest(static_cast<const unsigned char*>(recs), n);
}

void orc_build(void* h, uint32_t launch_filter) { static_cast<Oracle*>(h)->build(launch_filter); }

// dense rows of object index `o` (registration order)
void orc_word_counts(void* h, uint32_t o, uint32_t* out) {
  Oracle* p = static_cast<Oracle*>(h);
  std::copy(p->word_count[o].begin(), p->word_count[o].end(), out);
}
void orc_sector_counts(void* h, uint32_t o, uint32_t* out) {
  Oracle* p = static_cast<Oracle*>(h);
  std::copy(p->sector_count[o].begin(), p->sector_count[o].end(), out);
}
// access counts of object index `o`: number of (record, word) pairs per word,
// all launches (the metric Fig. 3 shows to be blind to sharing)
void orc_access_counts(void* h, uint32_t o, uint32_t* out) {
  Oracle* p = static_cast<Oracle*>(h);
  const uint64_t nw = (p->objs[o].len + 3) / 4;
  for (uint64_t w = 0; w < nw; ++w) {
    auto it = p->access.find(Oracle::wkey(o, w));
    out[w] = it == p->access.end() ? 0u : uint32_t(it->second);
  }
}

// run compression of object `o`'s rows (Fig. 4 caption:
// "consecutive memory regions with identical temperatures are compressed, and
// the number of occurrences is indicated"): maximal runs of
// consecutive sectors whose 9-tuples (8 word temperatures, words past the
// object's end as 0, then the sector's) are identical, untouched sectors
// included.  Writes up to cap runs (start sector, count, 9 temps); returns
// the number of runs.
size_t orc_runs(void* h, uint32_t o, uint64_t* start, uint64_t* count, uint32_t* temps, size_t cap) {
  Oracle* p = static_cast<Oracle*>(h);
  const uint64_t ns = p->sector_count[o].size(), nw = p->word_count[o].size();
  size_t n = 0;
  uint32_t prev[9] = {0};
  for (uint64_t s = 0; s < ns; ++s) {
    uint32_t t[9];
    for (int b = 0; b < 8; ++b) t[b] = 8 * s + b < nw ? p->word_count[o][8 * s + b] : 0;
    t[8] = p->sector_count[o][s];
    if (s > 0 && std::equal(t, t + 9, prev)) {
      if (n - 1 < cap) count[n - 1] += 1;
    } else {
      if (n < cap) {
        start[n] = s;
        count[n] = 1;
        std::copy(t, t + 9, temps + 9 * n);
      }
      ++n;
    }
    std::copy(t, t + 9, prev);
  }
  return n;
}

// counts of selected (object index, local sector) pairs: out[9*i .. 9*i+8] =
// 8 word counts then the sector count (words past n_words read as 0)
void orc_sample(void* h, const uint32_t* obj_idx, const uint64_t* sectors, size_t n, uint32_t* out) {
  Oracle* p = static_cast<Oracle*>(h);
  for (size_t i = 0; i < n; ++i) {
    uint32_t o = obj_idx[i];
    uint64_t s = sectors[i];
    if (p->restricted) {
      auto it = p->sampled.find({o, s});
      for (int b = 0; b < 9; ++b) out[9 * i + b] = it == p->sampled.end() ? 0u : it->second[b];
      continue;
    }
    for (int b = 0; b < 8; ++b) {
      uint64_t w = 8 * s + b;
      out[9 * i + b] = w < p->word_count[o].size() ? p->word_count[o][w] : 0;
    }
    out[9 * i + 8] = p->sector_count[o][s];
  }
}
void orc_hist(void* h, uint32_t o, int sector, uint64_t* out33) {
  Oracle* p = static_cast<Oracle*>(h);
  const auto& v = sector ? p->hist_sector[o] : p->hist_word[o];
  std::copy(v.begin(), v.end(), out33);
}
size_t orc_n_pcs(void* h) { return static_cast<Oracle*>(h)->pcrows.size(); }
// rows are in ascending (launch, pc) order (std::map order; G16)
void orc_pc_row(void* h, size_t i, uint32_t* launch, uint32_t* pc, uint64_t* hw33, uint64_t* hs33) {
  Oracle* p = static_cast<Oracle*>(h);
  const auto& r = p->pcrows[i];
  *launch = r.launch; *pc = r.pc;
  std::memcpy(hw33, r.hw, sizeof r.hw);
  std::memcpy(hs33, r.hs, sizeof r.hs);
}
// stats: [records, invalid, unmapped words, mapped word accesses] (filtered)
void orc_stats(void* h, uint64_t* out4) {
  Oracle* p = static_cast<Oracle*>(h);
  out4[0] = p->n_records;
  out4[1] = p->n_invalid;
  out4[2] = 0; out4[3] = 0;
  for (auto& kv : p->unmapped_by_launch) if (p->filter == 0xFFFFFFFFu || kv.first == p->filter) out4[2] += kv.second;
  for (auto& kv : p->mapped_by_launch) if (p->filter == 0xFFFFFFFFu || kv.first == p->filter) out4[3] += kv.second;
}

// Indicators and labels per object (§IV-C; rules S:356-409; DESIGN.md
// "Pattern indicators").  out[I_COUNT * o + field].
void orc_classify(void* h, const uint64_t* prm, uint64_t* out) {
  Oracle* p = static_cast<Oracle*>(h);
  for (size_t o = 0; o < p->objs.size(); ++o) {
    const auto& wc = p->word_count[o];
    const auto& sc = p->sector_count[o];
    uint64_t* r = out + I_COUNT * o;
    std::memset(r, 0, sizeof(uint64_t) * I_COUNT);
    r[I_NWORDS] = wc.size();
    r[I_NSECTORS] = sc.size();
    uint64_t T = 0, TW = 0, hot = 0, fs = 0, sumx = 0, le1 = 0, maxsec = 0;
    u128 sumx2 = 0;
    for (size_t s = 0; s < sc.size(); ++s) {
      uint64_t c = sc[s];
      if (c == 0) continue;
      ++T;
      maxsec = std::max(maxsec, c);
      uint64_t mw = 0;
      for (size_t b = 0; b < 8; ++b) {
        size_t w = 8 * s + b;
        if (w < wc.size()) mw = std::max<uint64_t>(mw, wc[w]);
      }
      // hot sector: c >= theta_hot and c <= alpha * mw
      if (c >= prm[P_THETA_HOT] && prm[P_ALPHA_DEN] * c <= prm[P_ALPHA_NUM] * mw) ++hot;
      // false-shared sector: c >= beta * mw and c >= fs_min
      if (prm[P_BETA_DEN] * c >= prm[P_BETA_NUM] * mw && c >= prm[P_FS_MIN]) ++fs;
    }
    for (size_t w = 0; w < wc.size(); ++w) {
      uint64_t x = wc[w];
      if (x == 0) continue;
      ++TW;
      sumx += x;
      sumx2 += u128(x) * x;
      if (x <= prm[P_SMEM_CAP]) ++le1;  // P:411 "every word's temperature ... is 1"
    }
    // gaps between consecutive touched words in address order (G15)
    std::map<uint64_t, uint64_t> gapc;
    uint64_t gaps = 0, prev = 0;
    bool have = false;
    for (size_t w = 0; w < wc.size(); ++w) {
      if (wc[w] == 0) continue;
      if (have) { gapc[w - prev] += 1; ++gaps; }
      prev = w; have = true;
    }
    uint64_t domgap = 0, domcnt = 0;
    for (auto& kv : gapc)
      if (kv.second > domcnt) { domcnt = kv.second; domgap = kv.first; }
    if (!(2 * domcnt > gaps)) { domgap = 0; domcnt = 0; }  // report only a strict majority (G16)
    // misalignment counters (instructions attributed to this object)
    uint64_t instrs = 0, mis = 0;
    for (auto& kv : p->instr) {
      if (kv.first.second != o) continue;
      if (p->filter != 0xFFFFFFFFu && kv.first.first != p->filter) continue;
      instrs += kv.second.first;
      mis += kv.second.second;
    }
    r[I_T] = T; r[I_TW] = TW; r[I_HOT] = hot; r[I_FS] = fs; r[I_SUMX] = sumx;
    r[I_SUMX2_LO] = uint64_t(sumx2); r[I_SUMX2_HI] = uint64_t(sumx2 >> 64);
    r[I_LE1] = le1; r[I_MAXSEC] = maxsec; r[I_INSTRS] = instrs; r[I_MIS] = mis;
    r[I_GAPS] = gaps; r[I_DOMGAP] = domgap; r[I_DOMCNT] = domcnt;
    // ---- labels (guards G23) ----
    uint64_t L = 0;
    if (T >= 1 && prm[P_HOTF_DEN] * hot >= prm[P_HOTF_NUM] * T) {
      // Random hot ("random numbers of warps"): CV of nonzero word temps
      // > cv_num/cv_den  <=>  den^2 (n*S2 - S1^2) > num^2 * S1^2     (G13)
      u128 S1 = sumx, n = TW;
      u128 var_num = n * sumx2 - S1 * S1;
      u128 lhs = u128(prm[P_CV_DEN]) * prm[P_CV_DEN] * var_num;
      u128 rhs = u128(prm[P_CV_NUM]) * prm[P_CV_NUM] * S1 * S1;
      L |= (TW >= 1 && lhs > rhs) ? L_RANDOM_HOT : L_HOT;
    }
    // FalseSharing and Strided apply to global-space objects ("pre:
    // rows from global space"); SmemAbuse to shared-space objects.
    const bool global = p->objs[o].space == 0;
    if (global && T >= 1 && prm[P_FSF_DEN] * fs >= prm[P_FSF_NUM] * T) L |= L_FALSE_SHARING;
    if (p->objs[o].space == 1 && TW >= 1 && prm[P_SMEM_COV_DEN] * le1 >= prm[P_SMEM_COV_NUM] * TW)
      L |= (maxsec == 1) ? L_SMEM_THREAD_LOCAL : L_SMEM_WARP_PRIVATE;
    if (instrs >= 1 && prm[P_MISF_DEN] * mis >= prm[P_MISF_NUM] * instrs) L |= L_MISALIGNED;
    if (global && T >= prm[P_STRIDED_MIN] && prm[P_GAMMA_DEN] * TW <= prm[P_GAMMA_NUM] * 8 * T && gaps >= 1 &&
        prm[P_DOM_DEN] * domcnt >= prm[P_DOM_NUM] * gaps)
      L |= L_STRIDED;
    r[I_LABELS] = L;
  }
}

}  // extern "C"
