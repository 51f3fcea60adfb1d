// dense.cu -- DENSE dedup path (rows a4 + a5 in sampled-block mode, SURVEY
// §8f item 1).  With one sampled thread block in scope at most 64
// warps of a launch are traced, so a word's set of warps is the paper's own
// bitmask (`sector_history_map` with `1 << warp_id |=`): one u64 per
// (launch, word) in HBM, OR-ed from the decoder's keys with one atomic per
// mapped word, no sort and no hash.  The flush is a popcount: a word's
// temperature is the popcount of its mask summed over the launches counted
// (warps are (launch, warp) pairs, G1), a sector's the popcount of the OR of
// its 8 word masks (G6).
#include "thermo_internal.cuh"

namespace thermo {

// keys [g : S][launch : L][warp : W][pcid : P][mask : 8]; warp0 = block_id *
// block_warps, so warp - warp0 < block_warps <= 64 (the decoders drop every
// other warp's records in sampled-block mode)
__global__ void __launch_bounds__(256) dense_or_kernel(const ull* __restrict__ keys, ull n, KeyLayout kl,
                                                       uint32_t warp0, ull S_tot, ull* __restrict__ dm) {
  const ull stride = (ull)gridDim.x * blockDim.x;
  const ull wmask = (1ull << kl.W) - 1;
  for (ull i = (ull)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const ull k = keys[i];
    const ull g = key_g(k, kl);
    const uint32_t la = key_launch(k, kl);
    const uint32_t w = (uint32_t)((k >> (8 + kl.P)) & wmask) - warp0;
    const ull bit = 1ull << (w & 63u);
    ull* row = dm + ((ull)la * S_tot + g) * 8;
    for (uint32_t m = (uint32_t)k & 0xFFu; m; m &= m - 1) atomicOr(&row[__ffs(m) - 1], bit);
  }
}

// one sector per thread: 64 B of masks per counted launch -> 8 word counts and
// the sector count (rows of untouched sectors stay as build zeroed them)
__global__ void __launch_bounds__(256) dense_count_kernel(const ull* __restrict__ dm, uint32_t L, ull S_tot,
                                                          uint32_t filter, uint32_t* __restrict__ wc,
                                                          uint32_t* __restrict__ sc, DevCounters* ctr) {
  const ull stride = (ull)gridDim.x * blockDim.x;
  ull pairs = 0;
  for (ull g = (ull)blockIdx.x * blockDim.x + threadIdx.x; g < S_tot; g += stride) {
    uint32_t cw[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    uint32_t cs = 0;
    for (uint32_t l = 0; l < L; ++l) {
      if (filter != THERMO_ALL_LAUNCHES && l != filter) continue;
      const ulonglong2* p = reinterpret_cast<const ulonglong2*>(dm + ((ull)l * S_tot + g) * 8);
      ull o = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const ulonglong2 v = p[q];
        cw[2 * q] += __popcll(v.x);
        cw[2 * q + 1] += __popcll(v.y);
        o |= v.x | v.y;
      }
      cs += __popcll(o);
    }
    if (cs) {
      reinterpret_cast<uint4*>(wc + 8 * g)[0] = make_uint4(cw[0], cw[1], cw[2], cw[3]);
      reinterpret_cast<uint4*>(wc + 8 * g)[1] = make_uint4(cw[4], cw[5], cw[6], cw[7]);
      sc[g] = cs;
      pairs += cs;
    }
  }
  for (int d = 16; d; d >>= 1) pairs += __shfl_xor_sync(0xFFFFFFFFu, pairs, d);
  if ((threadIdx.x & 31) == 0 && pairs) atomicAdd(&ctr->distinct_pairs, pairs);
}

void launch_dense_or(const ull* keys, ull n, KeyLayout kl, uint32_t warp0, ull S_tot, ull* dm, int num_sms,
                     cudaStream_t s) {
  if (!n) return;
  const unsigned grid = (unsigned)std::min<ull>((n + 255) / 256, (ull)num_sms * 16);
  dense_or_kernel<<<grid, 256, 0, s>>>(keys, n, kl, warp0, S_tot, dm);
}

void launch_dense_count(const ull* dm, uint32_t L, ull S_tot, uint32_t filter, uint32_t* wc, uint32_t* sc,
                        DevCounters* ctr, int num_sms, cudaStream_t s) {
  if (!S_tot) return;
  const unsigned grid = (unsigned)std::min<ull>((S_tot + 255) / 256, (ull)num_sms * 16);
  dense_count_kernel<<<grid, 256, 0, s>>>(dm, L, S_tot, filter, wc, sc, ctr);
}

}  // namespace thermo
