// bmt.cu -- sliced block-major tiled (BMT) fp32 hop: signal gathers from
// shared memory, 6-byte matrix entries, no cross-lane reductions.
//
// Why: the row kernel (filter.cu k_hop) streams (col, w) fully coalesced but
// each stored entry gathers a signal row z_j (8-16 B) through L1; on c2/c3
// those scattered gathers keep the L1TEX pipe ~90% busy and cap the kernel at
// ~50-60% of HBM bandwidth (profiles/r01_v2_k_hop_c3.txt).  Netlist graphs
// are banded (nets live in +-W index windows): a tile of rows touches only a
// few column blocks.  BMT stores a reordered copy of the matrix:
//
//   row tiles of kR = 2048 rows x column blocks of kC = 4096 columns (4096 x
//   8192 for short-row graphs, see bmt_shape_for);
//   a SEGMENT = the entries of one (tile, block) pair; segments tile-major,
//   blocks ascending;
//   inside a segment, every row's run of entries goes to one lane of a
//   SLICE of 32 runs (runs sorted by length, longest first, so slices are
//   nearly rectangular); a slice stores its runs lane-interleaved in groups
//   of 4: slot(k, lane) = base + (k/4)*128 + lane*4 + k%4 -- each lane reads
//   4 consecutive entries with one 8-byte (columns) + one 16-byte (weights)
//   load, the warp reads 768 contiguous bytes;
//   entry = u16 column-in-block + f32 weight = 6 B (vs 8 B for int32 col);
//   padding = column kC, which addresses a zero row of the staged block.
//
// Kernel: a CTA owns a tile.  Per segment it stages the block's signal rows
// in shared memory (dense segments; sparse ones -- pad / macro columns -- are
// gathered from L2 directly), then warps take slices: each lane sums its
// row's run sequentially in ascending column order and adds it to the row's
// shared fp32 accumulator (each row has one run per segment, so no two lanes
// touch a row in one segment).  After the last segment the shared row
// epilogue (hop.cuh) runs per row.  Summation order is fixed -> deterministic.
// (A first BMT version summed segment runs with warp segmented scans; it was
// instruction-bound at ~4 instructions per entry -- profiles/r01_bmt_scan_c2.txt.)
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <climits>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>
#include <set>

#include "common.cuh"
#include "hop.cuh"


// records in flight per warp (software-pipeline depth), per signal width; at
// F = 4, 4 on 512-thread CTAs (c3 F=4 pass 1.138 -> 1.117 ms) and 4 on
// 1024-thread ones (round 2, same-box A/B: c3 F=4 pass 1.050 -> 1.035 ms,
// c4 2.149 -> 2.144; round 1 had measured 3 ahead on c4)
#ifndef GIFT_BMT_DEPTH4
#define GIFT_BMT_DEPTH4 4
#endif
#ifndef GIFT_BMT_DEPTH4_512
#define GIFT_BMT_DEPTH4_512 4
#endif
#ifndef GIFT_BMT_DEPTH4_768
#define GIFT_BMT_DEPTH4_768 5
#endif
#ifndef GIFT_BMT_DEPTH2
#define GIFT_BMT_DEPTH2 5
#endif
// segment blocks staged by one bulk async copy (1) or by all threads (0)
#ifndef GIFT_BMT_BULK
#define GIFT_BMT_BULK 1
#endif
// segment hand-off pipelining in the barrier kernel (see FirstSlice)
#ifndef GIFT_BMT_PRE
#define GIFT_BMT_PRE 1
#endif
// threads per CTA of the F = 4 barrier kernel (compile-time; 768 leaves 85
// registers per thread for a deeper record pipeline)
#ifndef GIFT_BMT_THREADS4
#define GIFT_BMT_THREADS4 1024
#endif
template <int FIN, int kThreads>
__host__ __device__ constexpr int bmt_depth() {
  return FIN == 4 ? (kThreads == 512 ? GIFT_BMT_DEPTH4_512 : kThreads == 768 ? GIFT_BMT_DEPTH4_768 : GIFT_BMT_DEPTH4)
                  : GIFT_BMT_DEPTH2;
}

namespace gift {

namespace {

// Tile shape (rows per tile kR, columns per block kC = 2^cb), chosen per graph
// and signal width.  Fewer, larger segments win (per-segment hand-offs and the
// round-up of runs to 4-entry steps cost more than the larger staged block):
// signal widths <= 2 use 8192 x 16384 -- the largest F = 2 footprint,
// (kC + 16) x 8 B + kR x 8 B -- on every graph (per hop, tools/shape_sweep.sh:
// c4 4096x4096 1.87 ms, 4096x8192 1.45, 8192x8192 1.48, 4096x16384 1.36,
// 8192x16384 1.22; c3 2048x4096 0.98, 2048x8192 0.93, 4096x16384 0.89,
// 8192x16384 0.87).  F = 4 needs (kC + 16 + kR) x 16 B and gets a second
// copy: 8192 x 4096 for long rows (c2/c3, ~400 entries: ~80-entry runs even in
// 4096-column blocks, and more rows per segment; F = 4 pass on c3: 2048x4096
// at 2 CTAs per SM 1.12 ms, 4096x4096 1.23, 2048x8192 1.41, 4096x8192 1.10,
// 8192x2048 1.18, 8192x4096 1.04), 4096 x 8192 for short rows (c4, ~70
// entries over a +-40k band: 4096-column blocks left ~6-entry runs and x1.32
// stored slots).
struct BmtShape {
  int kR, cb;
};
BmtShape bmt_shape_for(const Ctx* ctx, int64_t n, double mean_row, bool wide_blocks) {
  BmtShape s = wide_blocks ? BmtShape{8192, 14} : (mean_row >= 160.0 ? BmtShape{8192, 12} : BmtShape{4096, 13});
  if (ctx->opt.tile_rows) s.kR = (int)ctx->opt.tile_rows;  // forced shape (option "tile_rows")
  if (ctx->opt.col_bits) s.cb = (int)ctx->opt.col_bits;    // option "col_bits"
  // Even waves (option "balance").  The default shapes run one CTA per SM and
  // one CTA per tile, so ceil(n / kR) tiles take ceil(tiles / SMs) waves: c3's
  // 269 tiles of 8192 rows on 148 SMs are 2 waves of which the second is 82 %
  // full, and the F = 4 pass -- bound per SM by the shared-memory pipe, not by
  // DRAM -- loses that idle time (the DRAM-bound F = 2 pass does not: fewer
  // SMs share the same bandwidth).  The tile height shrinks to the smallest
  // multiple of 32 that keeps the wave count: 7424 rows = 296 tiles = 2 x 148.
  // Graphs with fewer tiles than SMs get shorter tiles (down to 1024 rows) so
  // every SM has one: c1 (211k rows) runs 147 tiles of 1440 rows, 0.199 ->
  // 0.182 ms per bank; at 105k rows 1024-row tiles beat the row kernel 0.138
  // to 0.181 (profiles/r02_ab_small_tiles.txt).
  if (!ctx->opt.tile_rows && ctx->opt.balance && n > 0) {
    const int64_t sms = ctx->num_sms > 0 ? ctx->num_sms : 148;
    const int64_t waves = (n + (int64_t)s.kR * sms - 1) / ((int64_t)s.kR * sms);
    int64_t kr = (n + waves * sms - 1) / (waves * sms);
    kr = (kr + 31) / 32 * 32;
    s.kR = (int)std::min<int64_t>(s.kR, std::max<int64_t>(kr, 1024));
  }
  return s;
}
constexpr int kPadRows = 16;      // one zero row per bank residue mod 16 (padding never conflicts)
// columns kC .. kC + 15 of a staged block are its zero padding rows
constexpr int kStage = 1024;      // a segment with >= kStage entries stages its block
constexpr int kCodes = 256;       // coded copies: u8 weight codes, 255 = padding (weight 0)
constexpr int kCodeCopies = 16;   // shared-memory copies of the code table (see RecW)
constexpr int kBlock = 256;
constexpr int kWide = 8;          // rows touching > max(kWide, 3 x mean) blocks run on the row kernel
constexpr int kReuseHops = 4;     // GIFT_TILED_ON_REUSE: build once a graph has served this many fp32 hops

__global__ void k_mark_rows(int64_t n, const int64_t* __restrict__ indptr, int32_t* __restrict__ mark) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    if (indptr[r + 1] > indptr[r]) mark[indptr[r]] = (int32_t)r;
}

struct MaxI32 {
  __device__ __forceinline__ int32_t operator()(int32_t a, int32_t b) const { return a > b ? a : b; }
};

__global__ void k_iota64(int64_t n, int64_t* __restrict__ p) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = i;
}

// rows whose entries span many more column blocks than a typical row (pads /
// macros wired all over the die): one CTA would walk every block for them, so
// they stay on the row kernel.  Pass 1 counts blocks per row, pass 2 flags.
__global__ void k_row_nblocks(int64_t n, const int64_t* __restrict__ indptr, const int32_t* __restrict__ col, int cb,
                              uint16_t* __restrict__ nb_out, unsigned long long* __restrict__ total) {
  unsigned long long acc = 0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    int nb = 0, prev = -1;
    for (int64_t k = indptr[r]; k < indptr[r + 1] && nb < 65535; ++k) {
      const int b = col[k] >> cb;
      nb += b != prev;
      prev = b;
    }
    nb_out[r] = (uint16_t)nb;
    acc += nb;
  }
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) atomicAdd(total, acc);
}

__global__ void k_wide_rows(int64_t n, const int64_t* __restrict__ indptr, const uint16_t* __restrict__ nb, int limit,
                            uint8_t* __restrict__ wide, unsigned long long* __restrict__ n_wide,
                            unsigned long long* __restrict__ wide_nnz) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const bool wd = nb[r] > limit;
    wide[r] = wd;
    if (wd) {
      atomicAdd(n_wide, 1ULL);
      atomicAdd(wide_nnz, (unsigned long long)(indptr[r + 1] - indptr[r]));
    }
  }
}

// sort key (tile, block) and payload (weight bits, row in tile, column in block);
// wide rows get the sentinel key and sort past the kept entries
__global__ void k_bmt_keys(int64_t nnz, const int32_t* __restrict__ row_of, const int32_t* __restrict__ col,
                           const float* __restrict__ w, int bb, int kR, int cb, const uint8_t* __restrict__ wide,
                           uint32_t sentinel,
                           uint32_t* __restrict__ key, uint64_t* __restrict__ payload) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t r = (uint32_t)row_of[k], c = (uint32_t)col[k];
    key[k] = wide[r] ? sentinel : (((r / kR) << bb) | (c >> cb));
    const uint32_t packed = ((r % kR) << cb) | (c & ((1u << cb) - 1));
    payload[k] = ((uint64_t)__float_as_uint(w[k]) << 32) | packed;
  }
}

// segment heads (new (tile, block)) and run heads (new (segment, row)), counted
__global__ void k_bmt_heads(int64_t nnz, int cb, const uint32_t* __restrict__ key, const uint64_t* __restrict__ pay,
                            uint8_t* __restrict__ seg_head, uint8_t* __restrict__ run_head,
                            unsigned long long* __restrict__ counts) {
  unsigned long long ns = 0, nr = 0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
    const bool sh = k == 0 || key[k] != key[k - 1];
    const bool rh = sh || ((uint32_t)pay[k] >> cb) != ((uint32_t)pay[k - 1] >> cb);
    seg_head[k] = sh;
    run_head[k] = rh;
    ns += sh;
    nr += rh;
  }
  for (int off = 16; off > 0; off >>= 1) {
    ns += __shfl_xor_sync(0xffffffffu, ns, off);
    nr += __shfl_xor_sync(0xffffffffu, nr, off);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(counts, ns);
    atomicAdd(counts + 1, nr);
  }
}

// per run: sort key (segment, longest first); the stable sort keeps row order among equals
__global__ void k_run_keys(int64_t nruns, const int64_t* __restrict__ run_start, int64_t nnz,
                           const int64_t* __restrict__ seg_start, int64_t nseg, int cb, uint64_t* __restrict__ rkey) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nruns; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = run_start[i], b = i + 1 < nruns ? run_start[i + 1] : nnz;
    int64_t lo = 0, hi = nseg;  // segment = last seg_start <= a
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (seg_start[mid] <= a) lo = mid;
      else hi = mid;
    }
    const uint64_t len = (uint64_t)(b - a);  // <= kC distinct columns in a block
    rkey[i] = ((uint64_t)lo << (cb + 1)) | ((1ull << cb) - len);
  }
}

// first sorted run of every segment
__global__ void k_seg_runs(int64_t nruns, const uint64_t* __restrict__ rkey_s, int64_t nseg, int cb,
                           int64_t* __restrict__ seg_run) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= nruns; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = i < nruns ? (int64_t)(rkey_s[i] >> (cb + 1)) : nseg;
    const int64_t sp = i > 0 ? (int64_t)(rkey_s[i - 1] >> (cb + 1)) : -1;
    for (int64_t t = sp + 1; t <= s; ++t) seg_run[t] = i;
  }
}

__global__ void k_seg_slices(int64_t nseg, const int64_t* __restrict__ seg_run, int64_t* __restrict__ nsl) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nseg; s += (int64_t)gridDim.x * blockDim.x)
    nsl[s] = (seg_run[s + 1] - seg_run[s] + 31) / 32;
}

// slot count of each slice: its longest (first) run rounded up to 4, x 32 lanes
__global__ void k_slice_len(int64_t nseg, const int64_t* __restrict__ seg_run, const int64_t* __restrict__ seg_slice,
                            const uint64_t* __restrict__ rkey_s, int cb, int64_t* __restrict__ slice_slots) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nseg; s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r0 = seg_run[s], r1 = seg_run[s + 1];
    for (int64_t j = 0; r0 + 32 * j < r1; ++j) {
      const int64_t len = (1ll << cb) - (int64_t)(rkey_s[r0 + 32 * j] & ((2ull << cb) - 1));
      slice_slots[seg_slice[s] + j] = ((len + 3) / 4) * 4 * 32;
    }
  }
}

// scatter every run's entries into its slice lane (CTA per segment, thread per run)
__global__ void k_scatter_runs(int64_t nseg, const int64_t* __restrict__ seg_run, const int64_t* __restrict__ seg_slice,
                               const int64_t* __restrict__ run_perm, const int64_t* __restrict__ run_start,
                               int64_t nruns, int64_t nnz, int cb, const uint64_t* __restrict__ pay,
                               const int64_t* __restrict__ slice_off, uint16_t* __restrict__ slice_rows,
                               uint16_t* __restrict__ col, float* __restrict__ w) {
  for (int64_t s = blockIdx.x; s < nseg; s += gridDim.x) {
    const int64_t r0 = seg_run[s], r1 = seg_run[s + 1];
    for (int64_t q = r0 + threadIdx.x; q < r1; q += blockDim.x) {
      const int64_t pos = q - r0;
      const int64_t slice = seg_slice[s] + pos / 32;
      const int lane = (int)(pos % 32);
      const int64_t run = run_perm[q];
      const int64_t a = run_start[run], b = run + 1 < nruns ? run_start[run + 1] : nnz;
      const int64_t base = slice_off[slice] + 4 * lane;
      slice_rows[slice * 32 + lane] = (uint16_t)((uint32_t)pay[a] >> cb);
      for (int64_t k = 0; k < b - a; ++k) {
        const uint64_t p = pay[a + k];
        const int64_t slot = base + (k / 4) * 128 + (k % 4);
        col[slot] = (uint16_t)(p & ((1u << cb) - 1));
        w[slot] = __uint_as_float((uint32_t)(p >> 32));
      }
    }
  }
}

// Bank-conflict-aware step order.  Shared-memory gathers conflict when lanes
// of one wavefront hit the same bank group with different addresses:
//   F = 4 (LDS.128): a wavefront serves 8 lanes  -> want distinct col mod 8
//                    within each 8-lane quarter warp;
//   F = 2 (LDS.64):  a wavefront serves 16 lanes -> want distinct col mod 16
//                    within each 16-lane half warp.
// Random columns average ~2.5 wavefronts per phase.  A lane may take its run's
// entries in any FIXED order (the per-row fp32 sum stays deterministic), so per
// (slice, 16-lane half) a greedy pass reorders the lanes' entries: at every
// step each lane takes an entry whose residue mod 16 is unused in its half and
// whose residue mod 8 is unused in its quarter, preferring its most plentiful
// residue; failing that, one free mod 8 only; failing that, its most plentiful.
// Padding (column kC, residue 0, after the lane's real entries) is a
// wildcard: it can sit on any zero row kC + r, so it takes a residue no other
// lane of its half / quarter uses.
//
// One warp per slice, lane = the slice's lane.  Each lane buckets its own run
// by residue (counting sort into tmp); then the greedy runs as a WAVEFRONT
// over (step, lane): lane l decides step k at iteration k + l, using the
// used-residue masks of step k that lane l - 1 produced one iteration earlier
// (shuffled up within the 16-lane half).  All 16 lanes of a half decide at
// once, in L + 15 iterations instead of 16 L sequential decisions, and the
// per-lane counts / bucket cursors live in registers (unrolled selects, no
// dynamic indexing).  (Earlier versions: one thread per half slice over
// [16][16] count tables, 560 ms of the c3 build; lane-serial decisions with
// shuffles, 350 ms.)
__device__ __forceinline__ int sel16(const int (&v)[16], int r) {
  int x = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) x = (i == r) ? v[i] : x;
  return x;
}

__device__ __forceinline__ void add16(int (&v)[16], int r, int d) {
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] += (i == r) ? d : 0;
}

// residue with the largest count among the set bits of m (-1 if none);
// counts of residue 0 are the real (non-padding) entries only
__device__ __forceinline__ int argmax16(const int (&cnt)[16], int real0, unsigned m) {
  int best = -1, bc = 0;
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const int c = r == 0 ? real0 : cnt[r];
    const bool take = ((m >> r) & 1u) && c > bc;
    bc = take ? c : bc;
    best = take ? r : best;
  }
  return best;
}

__global__ void __launch_bounds__(256) k_slice_schedule(int64_t nslices, int kC, const int64_t* __restrict__ slice_off,
                                                        uint16_t* __restrict__ col, float* __restrict__ w,
                                                        uint16_t* __restrict__ tcol, float* __restrict__ tw) {
  const int lane = threadIdx.x & 31;
  const int hl = lane & 15;  // position in the 16-lane half
  const int q = hl >> 3;     // quarter within the half
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t sl = warp0; sl < nslices; sl += nwarps) {
    const int64_t off = slice_off[sl];
    const int L = (int)((slice_off[sl + 1] - off) / 32);  // slots per lane
    int cnt[16], next[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) cnt[r] = 0;
    int real0 = 0;
    for (int k = 0; k < L; ++k) {
      const int cv = col[off + (k >> 2) * 128 + lane * 4 + (k & 3)];
      add16(cnt, cv & 15, 1);
      real0 += ((cv & 15) == 0 && cv < kC);
    }
    {
      int acc = 0;
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        next[r] = acc;
        acc += cnt[r];
      }
    }
    const int64_t base = off + (int64_t)lane * L;
    {
      int pos[16];
#pragma unroll
      for (int r = 0; r < 16; ++r) pos[r] = next[r];
      for (int k = 0; k < L; ++k) {
        const int64_t slot = off + (k >> 2) * 128 + lane * 4 + (k & 3);
        const uint16_t cv = col[slot];
        const int r = cv & 15;
        const int p = sel16(pos, r);
        tcol[base + p] = cv;
        tw[base + p] = w[slot];
        add16(pos, r, 1);
      }
    }
    int pads = cnt[0] - real0;
    unsigned out16 = 0, out8 = 0;  // masks after this lane's decision (read by lane + 1)
    for (int t = 0; t < L + 15; ++t) {
      unsigned in16 = __shfl_up_sync(0xffffffffu, out16, 1, 16);
      unsigned in8 = __shfl_up_sync(0xffffffffu, out8, 1, 16);
      if (hl == 0) in16 = in8 = 0;
      const int k = t - hl;
      out16 = in16;
      out8 = in8;
      if (k < 0 || k >= L) continue;
      unsigned avail = 0;
#pragma unroll
      for (int r = 0; r < 16; ++r) avail |= ((r == 0 ? real0 : cnt[r]) > 0 ? 1u : 0u) << r;
      const unsigned q8 = (in8 >> (8 * q)) & 0xffu;
      const unsigned blocked = q8 | (q8 << 8);
      int r = argmax16(cnt, real0, avail & ~in16 & ~blocked);
      bool wildcard = false;
      if (r < 0 && pads > 0) {
        // no conflict-free real entry: a padding slot on a free zero row
        const unsigned f16 = ~in16 & ~blocked & 0xffffu, f8 = ~blocked & 0xffffu;
        r = f16 ? __ffs(f16) - 1 : (f8 ? __ffs(f8) - 1 : 0);
        wildcard = true;
      } else {
        if (r < 0) r = argmax16(cnt, real0, avail & ~blocked);
        if (r < 0) r = argmax16(cnt, real0, avail);
        if (r < 0) {  // nothing real left (cannot happen while pads > 0 is handled above)
          r = 0;
          wildcard = true;
        }
      }
      const int64_t slot = off + (k >> 2) * 128 + lane * 4 + (k & 3);
      if (wildcard) {
        pads--;
        add16(cnt, 0, -1);
        col[slot] = (uint16_t)(kC + r);
        w[slot] = 0.f;
      } else {
        const int src = sel16(next, r);
        add16(next, r, 1);
        add16(cnt, r, -1);
        if (r == 0) real0--;
        col[slot] = tcol[base + src];
        w[slot] = tw[base + src];
      }
      out16 = in16 | (1u << r);
      out8 = in8 | (1u << ((r & 7) + 8 * q));
    }
  }
}


// Optimal step order for the F = 4 copy (option "schedule" = 2).  An LDS.128
// wavefront serves the 8 lanes of a quarter warp, conflict-free when their
// columns differ mod 8.  Per (slice, quarter) the entries form a bipartite
// multigraph lanes x residues (M[i][r] = entries of lane i with column = r mod
// 8); ordering them into L steps with distinct residues per step is an edge
// colouring with L colours.  A residue held by more than L entries of the
// quarter forces conflicts: its surplus entries become "fillers" like the
// padding slots (which may sit on the zero row of any residue).  The rest is
// made L-regular by spreading every lane's fillers over the residues with
// slack (north-west corner rule, in closed form from two prefix sums), and an
// L-regular bipartite multigraph splits into L perfect matchings (Birkhoff -
// von Neumann): find a perfect matching in the support (8 x 8 bits, augmenting
// paths), use it for as many steps as its rarest edge allows, repeat.
// Conflicts left = the surplus entries, the lower bound; the greedy wavefront
// schedule leaves 5-9-way conflicts in a slice's last steps.
//
// One warp per slice, lane = the slice's lane (it moves its own entries, as in
// the greedy kernel).  The 8 lanes of a quarter hold one matrix row each and
// run the matching search redundantly on the shared 64-bit support, so they
// stay converged; all exchanges are quarter-wide shuffles.  Small per-lane
// arrays are indexed through unrolled selects (registers, no local memory).
__device__ __forceinline__ int sel8(const int (&v)[8], int r) {
  int x = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) x = (i == r) ? v[i] : x;
  return x;
}
__device__ __forceinline__ void add8(int (&v)[8], int r, int d) {
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] += (i == r) ? d : 0;
}
__device__ __forceinline__ unsigned get4(unsigned x, int i) { return (x >> (4 * i)) & 15u; }
__device__ __forceinline__ unsigned set4(unsigned x, int i, unsigned v) {
  return (x & ~(15u << (4 * i))) | (v << (4 * i));
}

__global__ void __launch_bounds__(256) k_slice_schedule_bvn(int64_t nslices, int kC,
                                                            const int64_t* __restrict__ slice_off,
                                                            uint16_t* __restrict__ col, float* __restrict__ w,
                                                            uint16_t* __restrict__ tcol, float* __restrict__ tw) {
  const int lane = threadIdx.x & 31;
  const int i = lane & 7;    // this lane's row of the quarter's matrix
  const int qb = lane & ~7;  // first lane of the quarter
  const unsigned qmask = 0xffu << qb;
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t sl = warp0; sl < nslices; sl += nwarps) {
    const int64_t off = slice_off[sl];
    const int L = (int)((slice_off[sl + 1] - off) / 32);  // slots per lane
    if (L <= 0) continue;
    // 1. bucket this lane's real entries by residue into its scratch run
    int cnt[8], bst[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) cnt[r] = 0;
    int pads = 0;
    for (int k = 0; k < L; ++k) {
      const int cv = col[off + (k >> 2) * 128 + lane * 4 + (k & 3)];
      if (cv >= kC) ++pads;
      else add8(cnt, cv & 7, 1);
    }
    {
      int acc = 0;
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        bst[r] = acc;
        acc += cnt[r];
      }
    }
    const int64_t base = off + (int64_t)lane * L;
    {
      int pos[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) pos[r] = bst[r];
      for (int k = 0; k < L; ++k) {
        const int64_t slot = off + (k >> 2) * 128 + lane * 4 + (k & 3);
        const int cv = col[slot];
        if (cv >= kC) continue;
        const int p = sel8(pos, cv & 7);
        tcol[base + p] = (uint16_t)cv;
        tw[base + p] = w[slot];
        add8(pos, cv & 7, 1);
      }
    }
    // 2. surplus of every residue (column sum above L), given up lane by lane;
    //    cnt[r] keeps the entries placed as themselves, ovc[r] the surplus
    int ovc[8], S[8];
    int need = pads;  // fillers of this lane = padding + surplus entries
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int v = cnt[r];
      int inc = v;
#pragma unroll
      for (int d = 1; d < 8; d <<= 1) {
        const int t = __shfl_up_sync(qmask, inc, d, 8);
        if (i >= d) inc += t;
      }
      const int tot = __shfl_sync(qmask, inc, 7, 8);
      const int e = tot - L;
      int g = 0;
      if (e > 0) g = min(max(e - (inc - v), 0), v);
      ovc[r] = g;
      cnt[r] = v - g;
      need += g;
      S[r] = e > 0 ? L : tot;
    }
    // 3. A = real + fillers with every row and column sum L: this lane's
    //    fillers are the interval [P, P + need) of the columns' slacks laid end to end
    int A[8];
    {
      int inc = need;
#pragma unroll
      for (int d = 1; d < 8; d <<= 1) {
        const int t = __shfl_up_sync(qmask, inc, d, 8);
        if (i >= d) inc += t;
      }
      const int P = inc - need;
      int Q = 0;
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int slack = L - S[r];
        const int lo = max(P, Q), hi = min(P + need, Q + slack);
        A[r] = cnt[r] + max(hi - lo, 0);
        Q += slack;
      }
    }
    // 4. Birkhoff - von Neumann: perfect matchings of the support, replicated per lane
    unsigned rowm = 0xffffffffu, colm = 0xffffffffu;  // nibble i: residue of lane i / lane of residue i (15: none)
    int used[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) used[r] = 0;
    int k = 0;
    while (k < L) {
      unsigned my = 0;
#pragma unroll
      for (int r = 0; r < 8; ++r) my |= (A[r] > 0 ? 1u : 0u) << r;
      unsigned long long sup = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) sup |= (unsigned long long)__shfl_sync(qmask, my, j, 8) << (8 * j);
      for (int i0 = 0; i0 < 8; ++i0) {
        if (get4(rowm, i0) != 15u) continue;
        unsigned from = 0, queue = 0, seen = 0;
        int qh = 0, qt = 0;
        queue = set4(queue, qt++, (unsigned)i0);
        bool done = false;
        while (qh < qt && !done) {
          const int ii = (int)get4(queue, qh++);
          unsigned cand = (unsigned)(sup >> (8 * ii)) & 0xffu & ~seen;
          while (cand && !done) {
            const int r = __ffs(cand) - 1;
            cand &= cand - 1;
            seen |= 1u << r;
            from = set4(from, r, (unsigned)ii);
            const unsigned cm = get4(colm, r);
            if (cm == 15u) {  // free residue: flip the alternating path back to i0
              int rr = r;
              for (;;) {
                const int i2 = (int)get4(from, rr);
                const unsigned prev = get4(rowm, i2);
                colm = set4(colm, rr, (unsigned)i2);
                rowm = set4(rowm, i2, (unsigned)rr);
                if (i2 == i0) break;
                rr = (int)prev;
              }
              done = true;
            } else {
              queue = set4(queue, qt++, cm);
            }
          }
        }
        if (!done) {  // impossible for a regular multigraph; keep the state consistent anyway
          for (int r = 0; r < 8; ++r)
            if (get4(colm, r) == 15u) {
              colm = set4(colm, r, (unsigned)i0);
              rowm = set4(rowm, i0, (unsigned)r);
              break;
            }
        }
      }
      const int r = (int)get4(rowm, i);  // this lane's residue for the next m steps
      int m = min(max(sel8(A, r), 1), L - k);
#pragma unroll
      for (int d = 4; d > 0; d >>= 1) m = min(m, __shfl_xor_sync(qmask, m, d, 8));
      int nreal = sel8(cnt, r) - sel8(used, r);
      for (int t = 0; t < m; ++t) {
        const int kk = k + t;
        const int64_t slot = off + (kk >> 2) * 128 + lane * 4 + (kk & 3);
        if (nreal > 0) {  // an entry of this residue
          const int p = sel8(bst, r) + sel8(used, r);
          add8(used, r, 1);
          --nreal;
          col[slot] = tcol[base + p];
          w[slot] = tw[base + p];
        } else if (pads > 0) {  // a padding slot, on the zero row of this residue
          --pads;
          col[slot] = (uint16_t)(kC + r);
          w[slot] = 0.f;
        } else {  // a surplus entry: it conflicts wherever it goes
          int rs = -1;
#pragma unroll
          for (int r2 = 7; r2 >= 0; --r2) rs = ovc[r2] > 0 ? r2 : rs;
          if (rs < 0) {
            col[slot] = (uint16_t)(kC + r);
            w[slot] = 0.f;
          } else {
            add8(ovc, rs, -1);
            const int p = sel8(bst, rs) + sel8(cnt, rs) + sel8(ovc, rs);
            col[slot] = tcol[base + p];
            w[slot] = tw[base + p];
          }
        }
      }
      add8(A, r, -m);
      unsigned z = (__ballot_sync(qmask, sel8(A, r) <= 0) >> qb) & 0xffu;
      while (z) {  // used-up edges: lane and residue look for new partners
        const int i2 = __ffs(z) - 1;
        z &= z - 1;
        const unsigned r2 = get4(rowm, i2);
        rowm = set4(rowm, i2, 15u);
        colm = set4(colm, (int)r2, 15u);
      }
      k += m;
    }
  }
}

// entries of sparse segments (fewer than kStage entries: pad / macro columns)
__global__ void k_flag_sparse(int64_t nseg, const int64_t* __restrict__ seg_start, int64_t nnz,
                              uint8_t* __restrict__ sparse, uint8_t* __restrict__ dense) {
  for (int64_t sg = blockIdx.x; sg < nseg; sg += gridDim.x) {
    const int64_t a = seg_start[sg], b = sg + 1 < nseg ? seg_start[sg + 1] : nnz;
    const uint8_t sp = (b - a) < kStage;
    for (int64_t k = a + threadIdx.x; k < b; k += blockDim.x) {
      sparse[k] = sp;
      dense[k] = !sp;
    }
  }
}

// residual entry -> (global row key, payload with global column)
__global__ void k_residual_keys(int64_t m, const uint32_t* __restrict__ key, const uint64_t* __restrict__ pay, int bb,
                                int kR, int cb, uint32_t* __restrict__ rkey, uint64_t* __restrict__ rpay) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t kk = key[k];
    const uint64_t p = pay[k];
    const uint32_t tile = kk >> bb, blk = kk & ((1u << bb) - 1);
    const uint32_t rowl = (uint32_t)p >> cb, coll = (uint32_t)p & ((1u << cb) - 1);
    rkey[k] = tile * (uint32_t)kR + rowl;
    rpay[k] = (p & 0xffffffff00000000ULL) | (uint64_t)((blk << cb) + coll);
  }
}

__global__ void k_residual_split(int64_t m, const uint32_t* __restrict__ rkey, const uint64_t* __restrict__ rpay,
                                 int64_t n, int64_t* __restrict__ rowptr, int32_t* __restrict__ col,
                                 float* __restrict__ w) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k <= m; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = k < m ? (int64_t)rkey[k] : n;
    const int64_t rp = k > 0 ? (int64_t)rkey[k - 1] : -1;
    for (int64_t t = rp + 1; t <= r; ++t) rowptr[t] = k;
    if (k < m) {
      col[k] = (int32_t)(uint32_t)rpay[k];
      w[k] = __uint_as_float((uint32_t)(rpay[k] >> 32));
    }
  }
}

// rows with residual entries, and each tile's range of that list
__global__ void k_has_res(int64_t n, const int64_t* __restrict__ rowptr, uint8_t* __restrict__ flag) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    flag[r] = rowptr[r + 1] > rowptr[r];
}

__global__ void k_tile_res(int64_t ntiles, int kR, const int64_t* __restrict__ rows, int64_t m,
                           int64_t* __restrict__ tile_res) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t <= ntiles; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t key = t * kR;
    int64_t lo = 0, hi = m;  // first row >= key
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (rows[mid] < key) lo = mid + 1;
      else hi = mid;
    }
    tile_res[t] = lo;
  }
}

// ---- u8 weight codes (the copy for signal widths <= 2) ---------------------
// code of w in the ascending table tbl[0, K), -1 if absent
__device__ __forceinline__ int code_of(float w, const float* __restrict__ tbl, int K) {
  int lo = 0, hi = K;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (tbl[mid] < w) lo = mid + 1;
    else hi = mid;
  }
  return (lo < K && tbl[lo] == w) ? lo : -1;
}

__global__ void k_sample_bits(int64_t m, int64_t stride, const float* __restrict__ w, uint32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __float_as_uint(w[i * stride]);
}

// dense entries whose weight has no code join the residual CSR
__global__ void k_flag_uncoded(int64_t nnz, const uint64_t* __restrict__ pay, const float* __restrict__ tbl, int K,
                               uint8_t* __restrict__ sparse, uint8_t* __restrict__ dense) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x)
    if (dense[k] && code_of(__uint_as_float((uint32_t)(pay[k] >> 32)), tbl, K) < 0) {
      dense[k] = 0;
      sparse[k] = 1;
    }
}

// coded layout: one 384-byte record per (slice, step of 4): 32 lanes x 4 u16
// columns, then 32 lanes x 4 u8 codes (255: padding)
__global__ void k_interleave_coded(int64_t total, const uint16_t* __restrict__ col, const float* __restrict__ w,
                                   const float* __restrict__ tbl, int K, uint8_t* __restrict__ data) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = q / 128;
    const int r = (int)(q % 128);  // lane * 4 + j
    uint8_t* rec = data + t * 384;
    reinterpret_cast<uint16_t*>(rec)[r] = col[q];
    const int code = w[q] == 0.f ? 255 : code_of(w[q], tbl, K);
    rec[256 + r] = (uint8_t)(code < 0 ? 255 : code);  // (every kept entry has a code)
  }
}

// final layout: one 768-byte record per (slice, step of 4): 32 lanes x 4 u16
// columns, then 32 lanes x 4 f32 weights -- a warp step reads one contiguous
// record (one DRAM stream per warp instead of two)
__global__ void k_interleave(int64_t total, const uint16_t* __restrict__ col, const float* __restrict__ w,
                             uint8_t* __restrict__ data) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = q / 128;
    const int r = (int)(q % 128);  // lane * 4 + j
    uint8_t* rec = data + t * 768;
    reinterpret_cast<uint16_t*>(rec)[r] = col[q];
    reinterpret_cast<float*>(rec + 256)[r] = w[q];
  }
}

__global__ void k_fill_u16(int64_t m, uint16_t v, uint16_t* __restrict__ p) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}

__global__ void k_seg_meta(int64_t nseg, const int64_t* __restrict__ seg_start, const uint32_t* __restrict__ key_s,
                           int64_t nnz, int bb, int32_t* __restrict__ seg_code, uint32_t* __restrict__ seg_tile) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nseg; s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = seg_start[s], b = s + 1 < nseg ? seg_start[s + 1] : nnz;
    const uint32_t k = key_s[a];
    const int blk = (int)(k & ((1u << bb) - 1));
    seg_code[s] = blk;  // sparse segments were moved to the residual CSR
    (void)b;
    seg_tile[s] = k >> bb;
  }
}

__global__ void k_bmt_tile_ptr(int64_t nseg, const uint32_t* __restrict__ seg_tile, int64_t ntiles,
                               int64_t* __restrict__ tile_seg) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s <= nseg; s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = s < nseg ? (int64_t)seg_tile[s] : ntiles;
    const int64_t tp = s > 0 ? (int64_t)seg_tile[s - 1] : -1;
    for (int64_t tt = tp + 1; tt <= t; ++tt) tile_seg[tt] = s;
  }
}

// estimated cost of a tile for the persistent scheduler: stored slots (6 B
// each), one staged block per dense segment, residual entries (gathered from
// L2) and the per-row epilogue
__global__ void k_tile_cost(int64_t ntiles, int kR, int kC, int64_t n, const int64_t* __restrict__ tile_seg,
                            const int64_t* __restrict__ seg_slice, const int64_t* __restrict__ slice_off,
                            const int64_t* __restrict__ res_rowptr, int64_t* __restrict__ cost) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ntiles; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s0 = tile_seg[t], s1 = tile_seg[t + 1];
    const int64_t slots = slice_off[seg_slice[s1]] - slice_off[seg_slice[s0]];
    const int64_t r0 = t * kR, r1 = min(n, r0 + kR);
    const int64_t res = res_rowptr[r1] - res_rowptr[r0];
    cost[t] = 6 * slots + 8 * (int64_t)kC * (s1 - s0) + 32 * res + 16 * (r1 - r0);
  }
}

struct BmtArgs {
  int64_t ncols;
  int tile_rows;
  int kC;               // columns per staged block
  const uint8_t* data;  // 768-byte step records (k_interleave)
  const uint8_t* wide;  // rows finished by the row kernel instead
  const int64_t* res_rowptr;  // [n + 1] residual (sparse-block) entries per row
  const int32_t* res_col;
  const float* res_w;
  const int64_t* tile_seg;
  const int32_t* seg_code;
  const int64_t* seg_slice;
  const int64_t* slice_off;
  const uint16_t* slice_rows;
  const int32_t* tile_order;  // persistent mode: tiles by decreasing cost
  unsigned* ctr;              // persistent mode: [next tile, finished CTAs]; null = one CTA per tile
  int64_t ntiles;
  const int64_t* res_rows;    // rows with residual entries, ascending
  const int64_t* tile_res;    // [ntiles + 1] range of res_rows per tile
  const float* code_tbl;      // CODED copies: [256] weight of each code (255 = padding, 0)
  int prefetch;               // L2 bulk prefetch of each warp's next slice (option "prefetch")
  int stream;                 // cross-slice record stream (option "stream")
};

// CODED kernels: the code table, 16 copies interleaved (see RecW), after the
// staged blocks and accumulators
template <int kThreads>
__device__ __forceinline__ void stage_code_table(const BmtArgs& b, float* tbl, int tid) {
  for (int i = tid; i < kCodes * kCodeCopies; i += kThreads) tbl[i] = b.code_tbl[i / kCodeCopies];
}

__device__ __forceinline__ uint2 ld_stream_v2u32(const void* p, uint64_t pol) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0, %1}, [%2], %3;"
               : "=r"(r.x), "=r"(r.y)
               : "l"(p), "l"(pol));
  return r;
}

// entry (c, w) of a run: acc += w * z_c from the staged block (c >= kC hits a zero row)
template <int FIN>
__device__ __forceinline__ void gather_fma(float (&acc)[FIN], float w, int c, const float* zs) {
  const float* zp = zs + c * FIN;
  if constexpr (FIN == 4) {
    const float4 q = *reinterpret_cast<const float4*>(zp);
    acc[0] = fmaf(w, q.x, acc[0]); acc[1] = fmaf(w, q.y, acc[1]);
    acc[2] = fmaf(w, q.z, acc[2]); acc[3] = fmaf(w, q.w, acc[3]);
  } else if constexpr (FIN == 2) {
    const float2 q = *reinterpret_cast<const float2*>(zp);
    acc[0] = fmaf(w, q.x, acc[0]); acc[1] = fmaf(w, q.y, acc[1]);
  } else {
    acc[0] = fmaf(w, zp[0], acc[0]);
  }
}

// Record stream of one warp.  Step k of the stream is the 768-byte record at
// base + k * 768: lane l reads its 4 columns (u16) at +8l and its 4 weights at
// +256+16l.  D records are kept in flight by a software pipeline written so the
// compiler needs no register copies: step k's registers are consumed (gathers
// issued, FMAs issued) BEFORE the load of step k + D is issued into the same
// registers.  (The first version issued the reload first; nvcc then renamed
// the destination and copied it back at the loop end, which waited on the
// load just issued -- one full memory latency per unrolled iteration, a third
// of all stall samples in profiles/r02_base_c3.)
template <int FIN>
__device__ __forceinline__ void step_fma(float (&acc)[FIN], uint2 cv, float4 wv, const float* zs) {
  gather_fma<FIN>(acc, wv.x, (int)(cv.x & 0xffffu), zs);
  gather_fma<FIN>(acc, wv.y, (int)(cv.x >> 16), zs);
  gather_fma<FIN>(acc, wv.z, (int)(cv.y & 0xffffu), zs);
  gather_fma<FIN>(acc, wv.w, (int)(cv.y >> 16), zs);
}

// Weight half of a record step.  Plain copies store f32 weights (768-byte
// records: 256 B of u16 columns, then 512 B of weights); CODED copies store a
// u8 code per entry into the graph's table of its 255 most frequent fp32
// weights (384-byte records: 256 B of columns, then 128 B of codes) -- entries
// with other weights live in the residual CSR.  The table sits in shared
// memory 16 times over (copy = lane % 16), so a warp's 32 lookups touch at
// most two addresses per bank.
template <bool CODED>
struct RecW;
template <>
struct RecW<false> {
  float4 v;
};
template <>
struct RecW<true> {
  uint32_t v;
};
template <bool CODED>
__host__ __device__ constexpr int rec_bytes() {
  return CODED ? 384 : 768;
}

// p = the lane's weight slot of a record: +256+16l (f32) or +256+4l (codes)
template <bool CODED>
__device__ __forceinline__ RecW<CODED> ld_w(const uint8_t* p, uint64_t pol) {
  RecW<CODED> r;
  if constexpr (CODED) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r.v) : "l"(p), "l"(pol));
  } else {
    r.v = ld_stream_v4f32(reinterpret_cast<const float*>(p), pol);
  }
  return r;
}

template <bool CODED>
__device__ __forceinline__ float4 weights(RecW<CODED> r, const float* tbl, int lane) {
  if constexpr (CODED) {
    const float* t = tbl + (lane & (kCodeCopies - 1));
    return make_float4(t[(r.v & 0xffu) * kCodeCopies], t[((r.v >> 8) & 0xffu) * kCodeCopies],
                       t[((r.v >> 16) & 0xffu) * kCodeCopies], t[(r.v >> 24) * kCodeCopies]);
  } else {
    (void)tbl;
    (void)lane;
    return r.v;
  }
}

// D record steps in flight (the registers of the software pipeline)
template <int D, bool CODED>
struct RecPipe {
  uint2 cq[D];
  RecW<CODED> wq[D];
};

// first D record loads of a slice (cp / wp: the lane's column / weight slots of
// the slice's first record)
template <int D, bool CODED>
__device__ __forceinline__ void pipe_issue(RecPipe<D, CODED>& p, const uint8_t* cp, const uint8_t* wp, int steps,
                                           uint64_t pol_s) {
  constexpr int RB = rec_bytes<CODED>();
#pragma unroll
  for (int d = 0; d < D; ++d)
    if (d < steps) {
      p.cq[d] = ld_stream_v2u32(cp + d * RB, pol_s);
      p.wq[d] = ld_w<CODED>(wp + d * RB, pol_s);
    }
}

// the rest of the slice: lane = one row's run, summed in its (conflict-
// scheduled) order, then added to the row's accumulator
template <int FIN, int D, bool CODED>
__device__ __forceinline__ void pipe_consume(RecPipe<D, CODED>& p, const uint8_t* cp, const uint8_t* wp, int steps,
                                             int row, const float* zs, float* accs, const float* tbl, int lane,
                                             uint64_t pol_s) {
  constexpr int RB = rec_bytes<CODED>();
  float acc[FIN];
#pragma unroll
  for (int f = 0; f < FIN; ++f) acc[f] = 0.f;
  int rem = steps;
  // steady state: D steps consumed, D reloaded, no predicates
  while (rem >= 2 * D) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      step_fma<FIN>(acc, p.cq[d], weights<CODED>(p.wq[d], tbl, lane), zs);
      p.cq[d] = ld_stream_v2u32(cp + (d + D) * RB, pol_s);
      p.wq[d] = ld_w<CODED>(wp + (d + D) * RB, pol_s);
    }
    cp += D * RB;
    wp += D * RB;
    rem -= D;
  }
  // tail: fewer than 2D steps left
  if (rem > D) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      step_fma<FIN>(acc, p.cq[d], weights<CODED>(p.wq[d], tbl, lane), zs);
      if (d + D < rem) {
        p.cq[d] = ld_stream_v2u32(cp + (d + D) * RB, pol_s);
        p.wq[d] = ld_w<CODED>(wp + (d + D) * RB, pol_s);
      }
    }
    rem -= D;
  }
#pragma unroll
  for (int d = 0; d < D; ++d)
    if (d < rem) step_fma<FIN>(acc, p.cq[d], weights<CODED>(p.wq[d], tbl, lane), zs);
  if (row != 0xffff) {
    // one run per row per segment: no other lane touches this row now
    if constexpr (FIN == 4) {
      float4* ap = reinterpret_cast<float4*>(accs) + row;
      float4 v = *ap;
      v.x += acc[0]; v.y += acc[1]; v.z += acc[2]; v.w += acc[3];
      *ap = v;
    } else if constexpr (FIN == 2) {
      float2* ap = reinterpret_cast<float2*>(accs) + row;
      float2 v = *ap;
      v.x += acc[0]; v.y += acc[1];
      *ap = v;
    } else {
#pragma unroll
      for (int f = 0; f < FIN; ++f) accs[row * FIN + f] += acc[f];
    }
  }
}

// one slice (dynamic mode)
template <int FIN, int D, bool CODED>
__device__ __forceinline__ void run_slice(const BmtArgs& b, int64_t off, int steps, int row, const float* zs,
                                          float* accs, const float* tbl, int lane, uint64_t pol_s) {
  constexpr int RB = rec_bytes<CODED>();
  const uint8_t* cp = b.data + (off / 128) * RB + 8 * lane;              // the lane's 4 columns
  const uint8_t* wp = cp - 8 * lane + 256 + (CODED ? 4 : 16) * lane;     // its 4 weights / codes
  RecPipe<D, CODED> p;
  pipe_issue<D, CODED>(p, cp, wp, steps, pol_s);
  pipe_consume<FIN, D, CODED>(p, cp, wp, steps, row, zs, accs, tbl, lane, pol_s);
}

// Segment hand-off pipelining (the barrier kernel).  A warp's FIRST slice of a
// segment is fixed (slice index = warp index; the shared counter hands out
// the rest from kThreads / 32 on), so everything that slice needs from global
// memory is requested while the segment's signal block is being staged:
// right after the barrier that ends the previous segment the warp loads the
// slice's metadata (offsets, the lanes' rows; the segment's slice range was
// loaded a segment ahead) and issues its first D records; both latencies run
// under the bulk copy of the block, which every warp has to wait for anyway.
// Without this a segment started with three dependent memory latencies
// AFTER the staging (slice range -> slice offsets -> records), ~2.5 us of the
// ~12 us a config-4 segment takes.
// slice metadata loads pinned where they are written (asm volatile), one
// slice ahead of their use.  The row id is still waited for at the end of a
// short slice (9 % of the c4 F = 4 pass's stall samples sit on it): a c4
// slice is ~3 record steps, about one DRAM latency (same time with plain
// loads: profiles/r02_ab_meta.txt)
#ifndef GIFT_BMT_META
#define GIFT_BMT_META 1
#endif
__device__ __forceinline__ int64_t ld_meta_s64(const int64_t* p) {
#if GIFT_BMT_META
  int64_t v;
  asm volatile("ld.global.nc.s64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
#else
  return *p;
#endif
}
__device__ __forceinline__ int ld_meta_u16(const uint16_t* p) {
#if GIFT_BMT_META
  unsigned short v;
  asm volatile("ld.global.nc.u16 %0, [%1];" : "=h"(v) : "l"(p));
  return (int)v;
#else
  return (int)*p;
#endif
}

struct FirstSlice {
  int64_t off = 0, end = 0;  // slot range (raw loads: converted where they are used)
  int row = 0xffff;
};

__device__ __forceinline__ FirstSlice load_first(const BmtArgs& b, int sl0, int nsl, int warp, int lane) {
  FirstSlice f;
  if (warp < nsl) {
    f.off = ld_meta_s64(b.slice_off + sl0 + warp);
    f.end = ld_meta_s64(b.slice_off + sl0 + warp + 1);
    f.row = ld_meta_u16(b.slice_rows + (int64_t)(sl0 + warp) * 32 + lane);
  }
  return f;
}

// segment [sl0, sl0 + nsl) with the warp's first slice `first` already issued into p
template <int FIN, int D, bool CODED>
__device__ __forceinline__ void segment_slices_pre(const BmtArgs& b, int sl0, int nsl, int warp,
                                                   const FirstSlice& first, RecPipe<D, CODED>& p, const float* zs,
                                                   float* accs, int* ctr, const float* tbl, int lane,
                                                   uint64_t pol_s) {
  constexpr int RB = rec_bytes<CODED>();
  auto grab = [&]() {
    int j = 0;
    if (lane == 0) j = atomicAdd(ctr, 1);
    return __shfl_sync(0xffffffffu, j, 0);
  };
  if (warp >= nsl) return;
  int64_t off = first.off, end = first.end;
  int row = first.row;
  bool pre = true;
  for (;;) {
    const int jn = grab();
    int64_t off_n = 0, end_n = 0;
    int row_n = 0xffff;
    if (jn < nsl) {
      off_n = ld_meta_s64(b.slice_off + sl0 + jn);
      end_n = ld_meta_s64(b.slice_off + sl0 + jn + 1);
      row_n = ld_meta_u16(b.slice_rows + (int64_t)(sl0 + jn) * 32 + lane);
    }
    const int steps = (int)((end - off) / 128);
    const uint8_t* cp = b.data + (off / 128) * RB + 8 * lane;
    const uint8_t* wp = cp - 8 * lane + 256 + (CODED ? 4 : 16) * lane;
    if (!pre) pipe_issue<D, CODED>(p, cp, wp, steps, pol_s);
    pre = false;
    pipe_consume<FIN, D, CODED>(p, cp, wp, steps, row, zs, accs, tbl, lane, pol_s);
    if (jn >= nsl) break;
    off = off_n;
    end = end_n;
    row = row_n;
  }
}

// the slices of segment s: warps take them dynamically from *ctr (slices touch
// distinct rows, so the assignment never changes a result)
template <int FIN, int D, bool CODED>
__device__ __forceinline__ void segment_slices(const BmtArgs& b, int64_t s, const float* zs, float* accs, int* ctr,
                                               const float* tbl, int lane, uint64_t pol_s) {
  const int64_t sl0 = b.seg_slice[s];
  const int nsl = (int)(b.seg_slice[s + 1] - sl0);
  auto grab = [&]() {
    int j = 0;
    if (lane == 0) j = atomicAdd(ctr, 1);
    return __shfl_sync(0xffffffffu, j, 0);
  };
  // the next slice's index and metadata are fetched before the current one
  // runs, so their latency hides behind its stream.  Tuning builds' option
  // "prefetch" also bulk-prefetches its records into L2 (c4, whose slices
  // are ~2 record steps, gained 1-2 %; c3's long slices lost 20-40 % to the
  // extra L2 traffic)
  [[maybe_unused]] constexpr int RB = rec_bytes<CODED>();
  int j = grab();
  int64_t off = 0, end = 0;
  int row = 0xffff;
  if (j < nsl) {
    off = b.slice_off[sl0 + j];
    end = b.slice_off[sl0 + j + 1];
    row = b.slice_rows[(sl0 + j) * 32 + lane];
  }
  while (j < nsl) {
    const int jn = grab();
    int64_t off_n = 0, end_n = 0;
    int row_n = 0xffff;
    if (jn < nsl) {
      off_n = b.slice_off[sl0 + jn];
      end_n = b.slice_off[sl0 + jn + 1];
      row_n = b.slice_rows[(sl0 + jn) * 32 + lane];
#ifdef GIFT_TUNING
      if (b.prefetch && lane == 0)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(b.data + (off_n / 128) * RB),
                     "r"((unsigned)((end_n - off_n) / 128 * RB))
                     : "memory");
#endif
    }
    run_slice<FIN, D, CODED>(b, off, (int)((end - off) / 128), row, zs, accs, tbl, lane, pol_s);
    j = jn;
    off = off_n;
    end = end_n;
    row = row_n;
  }
}

// Cross-slice record stream (option "stream"): the warp's D-record pipeline
// runs through every slice the warp takes in a segment instead of restarting
// per slice.  Each pipeline slot carries its record, the lane's row of the
// record's slice and whether the record is that slice's last step; consuming
// a last step flushes the lane's sum into the row accumulator.  The load
// cursor walks the current slice's records and moves to the next slice
// (grabbed, with its metadata, one slice ahead) when it runs out, so a slice
// of 2 record steps (c4) no longer pays a full memory latency of its own.
// Same per-row entry order as segment_slices: results are bit-identical.
template <int FIN, int D, bool CODED>
__device__ __forceinline__ void segment_stream(const BmtArgs& b, int64_t s, const float* zs, float* accs, int* ctr,
                                               const float* tbl, int lane, uint64_t pol_s) {
  constexpr int RB = rec_bytes<CODED>();
  const int64_t sl0 = b.seg_slice[s];
  const int nsl = (int)(b.seg_slice[s + 1] - sl0);
  auto grab = [&]() {
    int j = 0;
    if (lane == 0) j = atomicAdd(ctr, 1);
    return __shfl_sync(0xffffffffu, j, 0);
  };
  // next slice (metadata fetched one slice ahead)
  int nx_steps = 0, nx_row = 0xffff;
  const uint8_t* nx_rec = nullptr;
  auto fetch_next = [&]() {
    const int j = grab();
    nx_steps = 0;
    nx_row = 0xffff;
    if (j < nsl) {
      const int64_t off = b.slice_off[sl0 + j], end = b.slice_off[sl0 + j + 1];
      nx_steps = (int)((end - off) / 128);
      nx_row = b.slice_rows[(sl0 + j) * 32 + lane];
      nx_rec = b.data + (off / 128) * RB;
    }
  };
  // load cursor
  int cur_left = 0, cur_row = 0xffff;
  const uint8_t* cur_cp = nullptr;
  const uint8_t* cur_wp = nullptr;
  auto advance = [&]() {  // make the cursor point at a record, if any is left
    while (cur_left == 0 && nx_steps > 0) {
      cur_left = nx_steps;
      cur_row = nx_row;
      cur_cp = nx_rec + 8 * lane;
      cur_wp = nx_rec + 256 + (CODED ? 4 : 16) * lane;
      fetch_next();
    }
  };
  uint2 cq[D];
  RecW<CODED> wq[D];
  int srow[D];  // lane's row of the slot's slice; bit 16: last step of that slice
  bool sval[D];
  fetch_next();
  advance();
  int inflight = 0;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    sval[d] = cur_left > 0;
    if (sval[d]) {
      cq[d] = ld_stream_v2u32(cur_cp, pol_s);
      wq[d] = ld_w<CODED>(cur_wp, pol_s);
      srow[d] = cur_row | (cur_left == 1 ? 0x10000 : 0);
      cur_cp += RB;
      cur_wp += RB;
      --cur_left;
      ++inflight;
      advance();
    }
  }
  float acc[FIN];
#pragma unroll
  for (int f = 0; f < FIN; ++f) acc[f] = 0.f;
  while (inflight > 0) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      if (sval[d]) {
        step_fma<FIN>(acc, cq[d], weights<CODED>(wq[d], tbl, lane), zs);
        --inflight;
        if (srow[d] & 0x10000) {  // the slice's last step: flush the lane's run sum
          const int row = srow[d] & 0xffff;
          if (row != 0xffff) {
#pragma unroll
            for (int f = 0; f < FIN; ++f) accs[row * FIN + f] += acc[f];
          }
#pragma unroll
          for (int f = 0; f < FIN; ++f) acc[f] = 0.f;
        }
        sval[d] = cur_left > 0;
        if (sval[d]) {
          cq[d] = ld_stream_v2u32(cur_cp, pol_s);
          wq[d] = ld_w<CODED>(cur_wp, pol_s);
          srow[d] = cur_row | (cur_left == 1 ? 0x10000 : 0);
          cur_cp += RB;
          cur_wp += RB;
          --cur_left;
          ++inflight;
          advance();
        }
      }
    }
  }
}

// segment processor: per-slice pipelines or the cross-slice stream
// (compile-time: both in one kernel would share its register budget)
#ifndef GIFT_BMT_STREAM
#define GIFT_BMT_STREAM 0
#endif
template <int FIN, int D, bool CODED>
__device__ __forceinline__ void segment_run(const BmtArgs& b, int64_t s, const float* zs, float* accs, int* ctr,
                                            const float* tbl, int lane, uint64_t pol_s) {
  if constexpr (GIFT_BMT_STREAM)
    segment_stream<FIN, D, CODED>(b, s, zs, accs, ctr, tbl, lane, pol_s);
  else
    segment_slices<FIN, D, CODED>(b, s, zs, accs, ctr, tbl, lane, pol_s);
}

// after the segments: residual entries, then the fused row epilogue
template <int FIN, int FOUT, int kThreads>
__device__ __forceinline__ void bmt_tile_finish(const HopArgs& a, const BmtArgs& b, int64_t tile, int64_t r0,
                                                int nrows, float* accs, int tid, int lane, uint64_t pol_z) {
  __syncthreads();
  // residual entries (sparse blocks: pad / macro columns), 8 lanes per row, from
  // L2; only the tile's rows that have any (a precomputed list)
  {
    constexpr int G = 8;
    const int sub = lane & (G - 1);
    const unsigned gmask = 0xffu << (lane & ~(G - 1));
    const int64_t q1 = b.tile_res[tile + 1];
    for (int64_t q = b.tile_res[tile] + tid / G; q < q1; q += kThreads / G) {
      const int64_t r = b.res_rows[q];
      const int rr = (int)(r - r0);
      const int64_t beg = b.res_rowptr[r], end = b.res_rowptr[r + 1];
      float acc[FIN];
#pragma unroll
      for (int f = 0; f < FIN; ++f) acc[f] = 0.f;
      for (int64_t k = beg + sub; k < end; k += G) {
        const VecF<FIN> zq = ld_z<FIN>(a.zin + (int64_t)b.res_col[k] * FIN, pol_z);
        const float wk = b.res_w[k];
#pragma unroll
        for (int f = 0; f < FIN; ++f) acc[f] = fmaf(wk, zq.v[f], acc[f]);
      }
#pragma unroll
      for (int off = G / 2; off > 0; off >>= 1)
#pragma unroll
        for (int f = 0; f < FIN; ++f) acc[f] += __shfl_xor_sync(gmask, acc[f], off, G);
      if (sub == 0)
#pragma unroll
        for (int f = 0; f < FIN; ++f) accs[rr * FIN + f] += acc[f];
    }
  }
  __syncthreads();
  for (int rr = tid; rr < nrows; rr += kThreads) {
    if (b.wide[r0 + rr]) continue;
    float acc[FIN];
#pragma unroll
    for (int f = 0; f < FIN; ++f) acc[f] = accs[rr * FIN + f];
    row_epilogue<FIN, FOUT>(a, r0 + rr, acc, pol_z);
  }
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* m, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(m)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* m, unsigned bytes) {
  uint64_t state;
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 %0, [%1], %2;"
               : "=l"(state)
               : "r"(smem_addr(m)), "r"(bytes)
               : "memory");
  asm volatile("" ::"l"(state));  // the phase token is not needed
}

__device__ __forceinline__ void mbar_wait(uint64_t* m, unsigned parity) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_addr(m)), "r"(parity)
        : "memory");
  } while (!ok);
}

// segment s's signal block -> dst: one bulk copy of the 16-byte-aligned part,
// the ragged tail (last block of an odd-sized signal) by this thread's own
// stores, which the arrive (release) publishes together with the copy
template <int FIN>
__device__ __forceinline__ void stage_bulk(const HopArgs& a, const BmtArgs& b, int64_t s, float* dst, uint64_t* full,
                                           uint64_t pol) {
  const int64_t cbase = (int64_t)b.seg_code[s] * b.kC;
  const int64_t cend = min(cbase + b.kC, b.ncols);
  const unsigned nf = (unsigned)((cend - cbase) * FIN);
  const unsigned bytes = (nf * 4u) & ~15u;
  const float* src = a.zin + cbase * FIN;
  for (unsigned i = bytes / 4; i < nf; ++i) dst[i] = src[i];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // earlier generic reads of dst before the async write
  mbar_arrive_expect_tx(full, bytes);
  if (bytes)
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(full)), "l"(pol)
        : "memory");
}

// one staging buffer: stage, barrier, slices, barrier.  The block is staged
// by ONE bulk async copy (cp.async.bulk global -> shared, completion on an
// mbarrier) issued by thread 0 -- the warps spend no load / store issue on
// it -- or, for a signal that is not 16-byte aligned, by all threads.
template <int FIN, int FOUT, int kThreads, bool CODED>
__device__ __forceinline__ void bmt_tile(const HopArgs& a, const BmtArgs& b, int64_t tile, int kR, int tid, int lane,
                                         uint64_t pol_s, uint64_t pol_z) {
  extern __shared__ float4 smem_f4[];
  __shared__ int slice_ctr;
  __shared__ uint64_t full;
  const int kC = b.kC;
  float* zs = reinterpret_cast<float*>(smem_f4);  // [(kC + kPadRows) * FIN], rows >= kC stay zero
  float* accs = zs + (kC + kPadRows) * FIN;         // [kR * FIN]
  const float* tbl = accs + kR * FIN;               // CODED: [256 * 16] code table
  const int64_t r0 = tile * kR;
  const int nrows = (int)min((int64_t)kR, a.n - r0);
  const bool bulk = GIFT_BMT_BULK && (reinterpret_cast<uintptr_t>(a.zin) & 15) == 0;
  if (bulk && tid == 0) {  // visible after the first segment's barrier
    mbar_init(&full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  unsigned parity = 0;
  for (int i = tid; i < nrows * FIN; i += kThreads) accs[i] = 0.f;
  const int64_t s_beg = b.tile_seg[tile], s_end = b.tile_seg[tile + 1];
  constexpr int D = bmt_depth<FIN, kThreads>();
  constexpr int RB = rec_bytes<CODED>();
  constexpr bool kPre = !GIFT_BMT_STREAM && GIFT_BMT_PRE;
  const int warp = tid >> 5;
  // slice ranges of this segment [sl0, sl1), the next [sl1, sl2) and the one after
  // (loaded a segment ahead of the addresses they feed)
  int sl0 = 0, sl1 = 0, sl2 = 0;
  FirstSlice cur;
  if (kPre && s_beg < s_end) {
    sl0 = (int)b.seg_slice[s_beg];
    sl1 = (int)b.seg_slice[s_beg + 1];
    sl2 = s_beg + 2 <= s_end ? (int)b.seg_slice[s_beg + 2] : sl1;
  }
  for (int64_t s = s_beg; s < s_end; ++s) {
    const int64_t cbase = (int64_t)b.seg_code[s] * kC;
    const float* zg = a.zin + cbase * FIN;
    // finish the previous segment: its lanes may still read zs and update the
    // accumulators of rows this segment touches again
    __syncthreads();
    const int64_t cend = min(cbase + kC, b.ncols);
    const int nf = (int)((cend - cbase) * FIN);
    if (bulk) {
      if (tid == 0) stage_bulk<FIN>(a, b, s, zs, &full, pol_z);
    } else {
      const int nv = nf / 4;
      const float4* src = reinterpret_cast<const float4*>(zg);
      float4* dst = reinterpret_cast<float4*>(zs);
#pragma unroll 4
      for (int i = tid; i < nv; i += kThreads) dst[i] = src[i];
      for (int i = nv * 4 + tid; i < nf; i += kThreads) zs[i] = zg[i];
    }
    // the warp's first slice: metadata, then its first records, in flight
    // while the block is staged.  (Requesting the metadata one step earlier,
    // when the warp leaves the previous segment, keeps five more registers
    // live across the barrier: spills, c4 step 6.46 -> 6.81 ms.)
    RecPipe<D, CODED> pipe;
    int sl3 = sl2;
    if constexpr (kPre) {
      cur = load_first(b, sl0, sl1 - sl0, warp, lane);
      if (s + 3 <= s_end) sl3 = (int)b.seg_slice[s + 3];
      if (warp < sl1 - sl0) {
        const uint8_t* cp = b.data + (cur.off / 128) * RB + 8 * lane;
        pipe_issue<D, CODED>(pipe, cp, cp - 8 * lane + 256 + (CODED ? 4 : 16) * lane, (int)((cur.end - cur.off) / 128),
                             pol_s);
      }
    }
    for (int i = nf + tid; i < (kC + kPadRows) * FIN; i += kThreads) zs[i] = 0.f;  // short block + padding rows
    if (tid == 0) slice_ctr = kPre ? kThreads / 32 : 0;
    __syncthreads();
    if (bulk) {
      mbar_wait(&full, parity);
      parity ^= 1u;
    }
    if constexpr (kPre) {
      segment_slices_pre<FIN, D, CODED>(b, sl0, sl1 - sl0, warp, cur, pipe, zs, accs, &slice_ctr, tbl, lane, pol_s);
      sl0 = sl1;
      sl1 = sl2;
      sl2 = sl3;
    } else {
      segment_run<FIN, D, CODED>(b, s, zs, accs, &slice_ctr, tbl, lane, pol_s);
    }
  }
  bmt_tile_finish<FIN, FOUT, kThreads>(a, b, tile, r0, nrows, accs, tid, lane, pol_z);
}

// cp.async (16 B, L2 hint) of segment s's signal block into zs; a ragged tail
// (an odd row count at F = 2 in the last block) is copied by plain stores
template <int FIN, int kThreads>
__device__ __forceinline__ void stage_async(const HopArgs& a, const BmtArgs& b, int64_t s, float* zs, int tid,
                                            uint64_t pol) {
  const int64_t cbase = (int64_t)b.seg_code[s] * b.kC;
  const int64_t cend = min(cbase + b.kC, b.ncols);
  const int nf = (int)((cend - cbase) * FIN);
  const int nv = nf / 4;
  const float* zg = a.zin + cbase * FIN;
  const uint32_t dst = (uint32_t)__cvta_generic_to_shared(zs);
  for (int i = tid; i < nv; i += kThreads)
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(dst + 16u * (uint32_t)i),
                 "l"(zg + 4 * (int64_t)i), "l"(pol)
                 : "memory");
  for (int i = nv * 4 + tid; i < nf; i += kThreads) zs[i] = zg[i];
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}

// two staging buffers: segment s + 1's block streams in (cp.async) while the
// warps run segment s's slices; one barrier per segment
template <int FIN, int FOUT, int kThreads, bool CODED>
__device__ __forceinline__ void bmt_tile_db(const HopArgs& a, const BmtArgs& b, int64_t tile, int kR, int tid,
                                            int lane, uint64_t pol_s, uint64_t pol_z) {
  extern __shared__ float4 smem_f4[];
  __shared__ int slice_ctr2[2];
  const int kC = b.kC;
  const int zrows = (kC + kPadRows) * FIN;
  float* zs0 = reinterpret_cast<float*>(smem_f4);
  float* zs1 = zs0 + zrows;
  float* accs = zs1 + zrows;  // [kR * FIN]
  const float* tbl = accs + kR * FIN;  // CODED: code table
  const int64_t r0 = tile * kR;
  const int nrows = (int)min((int64_t)kR, a.n - r0);
  for (int i = tid; i < nrows * FIN; i += kThreads) accs[i] = 0.f;
  for (int i = kC * FIN + tid; i < zrows; i += kThreads) {  // padding rows: zero in both buffers
    zs0[i] = 0.f;
    zs1[i] = 0.f;
  }
  if (tid == 0) slice_ctr2[0] = 0;
  const int64_t s0 = b.tile_seg[tile], s1 = b.tile_seg[tile + 1];
  if (s0 < s1) stage_async<FIN, kThreads>(a, b, s0, zs0, tid, pol_z);
  for (int64_t s = s0; s < s1; ++s) {
    const int buf = (int)((s - s0) & 1);
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    // segment s is staged (every thread's copies), and every warp is done with
    // segment s - 1: its buffer, counter and accumulator updates
    __syncthreads();
    if (s + 1 < s1) {
      stage_async<FIN, kThreads>(a, b, s + 1, buf ? zs0 : zs1, tid, pol_z);
      if (tid == 0) slice_ctr2[buf ^ 1] = 0;
    }
    segment_run<FIN, bmt_depth<FIN, kThreads>(), CODED>(b, s, buf ? zs1 : zs0, accs, &slice_ctr2[buf], tbl, lane,
                                                           pol_s);
  }
  bmt_tile_finish<FIN, FOUT, kThreads>(a, b, tile, r0, nrows, accs, tid, lane, pol_z);
}

template <int FIN, int FOUT, int kThreads, bool DB, bool CODED>
__global__ void __launch_bounds__(kThreads, 1024 / kThreads) k_hop_bmt(HopArgs a, BmtArgs b) {
  const int kR = b.tile_rows;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const uint64_t pol_s = policy_evict_first();
  const uint64_t pol_z = policy_evict_last();
  __shared__ int64_t tile_sh;
  if constexpr (CODED) {  // visible after the first segment's barrier
    extern __shared__ float4 smem_f4[];
    const int zrows = (b.kC + kPadRows) * FIN;
    stage_code_table<kThreads>(b, reinterpret_cast<float*>(smem_f4) + (DB ? 2 : 1) * zrows + kR * FIN, tid);
  }
  if (!b.ctr) {  // one CTA per tile; the block scheduler issues low blockIdx first
    const int64_t tile = b.tile_order ? b.tile_order[blockIdx.x] : blockIdx.x;
    if constexpr (DB)
      bmt_tile_db<FIN, FOUT, kThreads, CODED>(a, b, tile, kR, tid, lane, pol_s, pol_z);
    else
      bmt_tile<FIN, FOUT, kThreads, CODED>(a, b, tile, kR, tid, lane, pol_s, pol_z);
    return;
  }
  // persistent CTAs take tiles costliest first from a global counter (the
  // last CTA to finish resets it for the next launch on the stream); tiles
  // are independent (disjoint output rows), so the assignment never changes
  // a result
  for (;;) {
    if (tid == 0) {
      const unsigned t = atomicAdd(&b.ctr[0], 1u);
      tile_sh = t < (unsigned long long)b.ntiles ? b.tile_order[t] : -1;
    }
    __syncthreads();  // also: the previous tile's epilogue is done with accs
    const int64_t tile = tile_sh;
    __syncthreads();
    if (tile < 0) break;
    if constexpr (DB)
      bmt_tile_db<FIN, FOUT, kThreads, CODED>(a, b, tile, kR, tid, lane, pol_s, pol_z);
    else
      bmt_tile<FIN, FOUT, kThreads, CODED>(a, b, tile, kR, tid, lane, pol_s, pol_z);
  }
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(&b.ctr[1], 1u) == gridDim.x - 1) {
      b.ctr[0] = 0;
      b.ctr[1] = 0;
    }
  }
}

// ---------------------------------------------------------------------------
// Barrier-free segment pipeline (default where it fits in shared memory).
//
// The kernels above end every segment with a CTA barrier: the next block is
// staged into the buffer the slowest warp may still read, and two segments of
// a tile may touch the same row's accumulator.  ncu (profiles/r02_base_c3)
// put 18 % of the F = 2 pass's stall samples on that barrier.  Here:
//   * two signal buffers, filled by one bulk async copy each
//     (cp.async.bulk global -> shared, completion on an mbarrier);
//   * two accumulator banks: segment i adds into bank i % 2;
//   * a warp that finishes segment i bumps done[i % 2]; the LAST warp to do so
//     (every warp has left segment i, so nobody reads buffer i % 2 or adds to
//     bank i % 2 any more) issues the copy of segment i + 2 into that buffer.
// A warp may thus run one segment ahead of the slowest warp; it waits only if
// it gets two ahead.  A row's sum is (bank 0 + bank 1) + residual: fixed
// order, so the result stays deterministic (it is a different, equally valid
// fp32 association than the single-bank kernels).
// ---------------------------------------------------------------------------
template <int FIN, int FOUT, int kThreads, bool CODED>
__global__ void __launch_bounds__(kThreads, 1024 / kThreads) k_hop_bmt_nb(HopArgs a, BmtArgs b) {
  extern __shared__ float4 smem_f4[];
  __shared__ uint64_t full[2];
  __shared__ int slice_ctr[2];
  __shared__ int done[2];
  constexpr int NW = kThreads / 32;
  const int tid = threadIdx.x, lane = tid & 31;
  const int kR = b.tile_rows, kC = b.kC;
  const uint64_t pol_s = policy_evict_first();
  const uint64_t pol_z = policy_evict_last();
  const int zrows = (kC + kPadRows) * FIN;
  float* zs[2];
  zs[0] = reinterpret_cast<float*>(smem_f4);
  zs[1] = zs[0] + zrows;
  float* acc[2];
  acc[0] = zs[1] + zrows;
  acc[1] = acc[0] + kR * FIN;
  float* tbl = acc[1] + kR * FIN;  // CODED: code table
  if constexpr (CODED) stage_code_table<kThreads>(b, tbl, tid);  // visible after the barrier below
  const int64_t tile = b.tile_order ? b.tile_order[blockIdx.x] : blockIdx.x;
  const int64_t r0 = tile * kR;
  const int nrows = (int)min((int64_t)kR, a.n - r0);
  for (int i = tid; i < nrows * FIN; i += kThreads) {
    acc[0][i] = 0.f;
    acc[1][i] = 0.f;
  }
  for (int i = kC * FIN + tid; i < zrows; i += kThreads) {  // zero padding rows of both buffers
    zs[0][i] = 0.f;
    zs[1][i] = 0.f;
  }
  const int64_t s0 = b.tile_seg[tile];
  const int nseg = (int)(b.tile_seg[tile + 1] - s0);
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    slice_ctr[0] = slice_ctr[1] = 0;
    done[0] = done[1] = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (int i = 0; i < 2 && i < nseg; ++i) stage_bulk<FIN>(a, b, s0 + i, zs[i], &full[i], pol_z);
  for (int i = 0; i < nseg; ++i) {
    const int buf = i & 1;
    mbar_wait(&full[buf], (unsigned)(i >> 1) & 1u);
    segment_run<FIN, bmt_depth<FIN, kThreads>(), CODED>(b, s0 + i, zs[buf], acc[buf], &slice_ctr[buf], tbl, lane,
                                                           pol_s);
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      if (atomicAdd(&done[buf], 1) == NW - 1) {  // every warp has left segment i
        __threadfence_block();
        done[buf] = 0;
        slice_ctr[buf] = 0;
        if (i + 2 < nseg) stage_bulk<FIN>(a, b, s0 + i + 2, zs[buf], &full[buf], pol_z);
      }
    }
  }
  __syncthreads();
  for (int i = tid; i < nrows * FIN; i += kThreads) acc[0][i] += acc[1][i];
  bmt_tile_finish<FIN, FOUT, kThreads>(a, b, tile, r0, nrows, acc[0], tid, lane, pol_z);
}

constexpr size_t kCodeTableBytes = (size_t)kCodes * kCodeCopies * sizeof(float);

size_t bmt_smem_nb(int fin, int kR, int kC, bool coded) {
  return 2 * ((size_t)(kC + kPadRows) * fin * 4 + (size_t)kR * fin * 4) + (coded ? kCodeTableBytes : 0);
}

size_t bmt_smem(int fin, int kR, int kC, bool coded = false) {
  return (size_t)(kC + kPadRows) * fin * 4 + (size_t)kR * fin * 4 + (coded ? kCodeTableBytes : 0);
}

#ifdef GIFT_TUNING
size_t bmt_smem_db(int fin, int kR, int kC, bool coded) {
  return bmt_smem(fin, kR, kC, coded) + (size_t)(kC + kPadRows) * fin * 4;
}
#endif

template <int FIN, int FOUT, bool DB, bool CODED>
void launch_bmt_k(Ctx* ctx, const HopArgs& a, const BmtArgs& b, int64_t ntiles, int tpb, size_t smem) {
  constexpr int kBig = FIN == 4 ? GIFT_BMT_THREADS4 : 1024;  // the one-CTA-per-SM shape
#ifdef GIFT_TUNING
  auto kern = tpb == 1024 ? k_hop_bmt<FIN, FOUT, kBig, DB, CODED> : k_hop_bmt<FIN, FOUT, 512, DB, CODED>;
  if (tpb == 1024) tpb = kBig;
#else
  auto kern = k_hop_bmt<FIN, FOUT, kBig, DB, CODED>;  // default shapes are >= 4096 rows: 1 CTA per SM
  tpb = kBig;
#endif
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> occ;  // resident CTAs per SM per (instance, device)
  int per_sm = 0;
  {
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_pair((const void*)kern, ctx->device);
    auto it = occ.find(key);
    if (it == occ.end()) {
      const int optin = ctx->smem_optin;
      cudaFuncAttributes fa{};
      GIFT_CUDA(cudaFuncGetAttributes(&fa, kern));
      GIFT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     optin - (int)fa.sharedSizeBytes));
      GIFT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, tpb, smem));
      occ[key] = per_sm;
    } else {
      per_sm = it->second;
    }
  }
  unsigned grid = (unsigned)ntiles;
  if (b.ctr) grid = (unsigned)std::min<int64_t>(ntiles, (int64_t)std::max(per_sm, 1) * ctx->num_sms);
  kern<<<grid, tpb, smem, ctx->stream>>>(a, b);
  GIFT_LAUNCH_CHECK(ctx);
}

template <int FIN, int FOUT, int kThreads, bool CODED>
void launch_bmt_nb(Ctx* ctx, const HopArgs& a, const BmtArgs& b, int64_t ntiles, size_t smem) {
  auto kern = k_hop_bmt_nb<FIN, FOUT, kThreads, CODED>;
  // the smem opt-in is a per-device function attribute: set it once per device
  static std::mutex mu;
  static std::set<int> done;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!done.count(ctx->device)) {
      cudaFuncAttributes fa{};
      GIFT_CUDA(cudaFuncGetAttributes(&fa, kern));
      GIFT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     ctx->smem_optin - (int)fa.sharedSizeBytes));
      done.insert(ctx->device);
    }
  }
  kern<<<(unsigned)ntiles, kThreads, smem, ctx->stream>>>(a, b);
  GIFT_LAUNCH_CHECK(ctx);
}

template <int FIN, int FOUT, bool CODED>
void launch_bmt(Ctx* ctx, const HopArgs& a, const BmtArgs& b, int64_t ntiles) {
  // barrier-free pipeline where it keeps the barrier kernel's occupancy:
  // 2 CTAs x 512 threads per SM for 2048-row tiles, 1 x 1024 for taller ones
  // (A/B on B200: c4 F=2 pass 1.83 -> 1.63 ms at 1 x 1024; c3 F=4 pass 1.16 ->
  // 1.25 ms when its 197 KB footprint drops it from 2 x 512 to 1 x 1024).  The
  // bulk copies need a 16-byte aligned signal.
  if (ctx->opt.barrier_free && !b.ctr && ((uintptr_t)a.zin & 15) == 0) {
    const size_t nb = bmt_smem_nb(FIN, b.tile_rows, b.kC, CODED), fixed = 3 * 1024;
#ifdef GIFT_TUNING
    if (b.tile_rows <= 2048 && 2 * (nb + fixed) <= 228 * 1024) {
      launch_bmt_nb<FIN, FOUT, 512, CODED>(ctx, a, b, ntiles, nb);
      return;
    }
#endif
    if ((b.tile_rows > 2048 || ctx->opt.barrier_free > 1) && nb + fixed <= 228 * 1024) {
      launch_bmt_nb<FIN, FOUT, 1024, CODED>(ctx, a, b, ntiles, nb);
      return;
    }
  }
  // the barrier kernel: 1 CTA x 1024 threads per SM on the default (>= 4096-row)
  // tiles.  Tuning builds also have 2 x 512 for 2048-row tiles and a
  // double-buffered (cp.async) variant; neither won on the default shapes
  // (DESIGN.md §4).
  const size_t smem1 = bmt_smem(FIN, b.tile_rows, b.kC, CODED);
#ifdef GIFT_TUNING
  const size_t smem2 = bmt_smem_db(FIN, b.tile_rows, b.kC, CODED);
  const int tpb = (b.tile_rows > 2048 || 2 * (smem1 + 3 * 1024) > 228 * 1024) ? 1024 : 512;
  const int per_sm = tpb == 512 ? 2 : 1;
  const bool db = env_int("GIFT_BMT_DB", 1) && ((uintptr_t)a.zin & 15) == 0 &&
                  (size_t)per_sm * (smem2 + 3 * 1024) <= 228 * 1024;
  if (db) {
    launch_bmt_k<FIN, FOUT, true, CODED>(ctx, a, b, ntiles, tpb, smem2);
    return;
  }
  launch_bmt_k<FIN, FOUT, false, CODED>(ctx, a, b, ntiles, tpb, smem1);
#else
  launch_bmt_k<FIN, FOUT, false, CODED>(ctx, a, b, ntiles, 1024, smem1);
#endif
}

// Coded copies (u8 weight codes, 3-byte entries) are a TUNING-build
// experiment: on B200 the F = 2 pass got slower with them (c3 0.85 -> 0.93 ms,
// c4 1.25 -> 1.34 ms: the per-entry table lookup costs more shared-memory
// issue than the halved record bytes save), so product builds keep fp32
// weights
template <int FIN>
void launch_bmt_out(Ctx* ctx, const HopArgs& a, const BmtArgs& b, int64_t ntiles, int fout, bool coded) {
#ifdef GIFT_TUNING
  if constexpr (FIN <= 2) {
    if (coded) {
      switch (fout) {
        case 0: launch_bmt<FIN, 0, true>(ctx, a, b, ntiles); break;
        case 1: launch_bmt<FIN, 1, true>(ctx, a, b, ntiles); break;
        case 2: launch_bmt<FIN, 2, true>(ctx, a, b, ntiles); break;
        default: launch_bmt<FIN, 4, true>(ctx, a, b, ntiles); break;
      }
      return;
    }
  }
#else
  (void)coded;  // coded copies exist only in tuning builds
#endif
  switch (fout) {
    case 0: launch_bmt<FIN, 0, false>(ctx, a, b, ntiles); break;
    case 1: launch_bmt<FIN, 1, false>(ctx, a, b, ntiles); break;
    case 2: launch_bmt<FIN, 2, false>(ctx, a, b, ntiles); break;
    default: launch_bmt<FIN, 4, false>(ctx, a, b, ntiles); break;
  }
}

template <typename T>
T fetch(Ctx* ctx, const T* d) {
  T h;
  GIFT_CUDA(cudaMemcpyAsync(&h, d, sizeof(T), cudaMemcpyDeviceToHost, ctx->stream));
  GIFT_CUDA(cudaStreamSynchronize(ctx->stream));
  return h;
}

void select_positions(Ctx* ctx, const uint8_t* flags, int64_t n, int64_t* out, int64_t* d_count) {
  thrust::counting_iterator<int64_t> it(0);
  size_t bytes = 0;
  GIFT_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, it, flags, out, d_count, n, ctx->stream));
  DevBuf<char> tmp(ctx, bytes);
  GIFT_CUDA(cub::DeviceSelect::Flagged(tmp.p, bytes, it, flags, out, d_count, n, ctx->stream));
  ctx->launches += 2;
}

void exclusive_sum(Ctx* ctx, const int64_t* in, int64_t* out, int64_t n) {
  size_t bytes = 0;
  GIFT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, ctx->stream));
  DevBuf<char> tmp(ctx, bytes);
  GIFT_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, in, out, n, ctx->stream));
  ctx->launches += 2;
}

// the graph's (up to) 255 most frequent fp32 weights, ascending, into tbl[0, K);
// tbl[255] = 0 (padding).  Returns K.
int build_code_table(Ctx* ctx, const float* w32, int64_t nnz, float* tbl) {
  cudaStream_t st = ctx->stream;
  const int64_t m = std::min<int64_t>(nnz, 1LL << 24);
  const int64_t stride = (nnz + m - 1) / m;
  const int64_t ms = (nnz + stride - 1) / stride;
  DevBuf<uint32_t> smp(ctx, ms), srt(ctx, ms), uniq(ctx, ms);
  DevBuf<int32_t> cnt(ctx, ms);
  DevBuf<int32_t> nruns(ctx, 1);
  k_sample_bits<<<grid_for(ms, kBlock), kBlock, 0, st>>>(ms, stride, w32, smp.p);
  GIFT_LAUNCH_CHECK(ctx);
  size_t bytes = 0;
  GIFT_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, smp.p, srt.p, ms, 0, 32, st));
  {
    DevBuf<char> tmp(ctx, bytes);
    GIFT_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, bytes, smp.p, srt.p, ms, 0, 32, st));
  }
  bytes = 0;
  GIFT_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, bytes, srt.p, uniq.p, cnt.p, nruns.p, ms, st));
  {
    DevBuf<char> tmp(ctx, bytes);
    GIFT_CUDA(cub::DeviceRunLengthEncode::Encode(tmp.p, bytes, srt.p, uniq.p, cnt.p, nruns.p, ms, st));
  }
  ctx->launches += 5;
  const int32_t nr = fetch(ctx, nruns.p);
  std::vector<uint32_t> hu(nr);
  std::vector<int32_t> hc(nr);
  GIFT_CUDA(cudaMemcpyAsync(hu.data(), uniq.p, nr * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  GIFT_CUDA(cudaMemcpyAsync(hc.data(), cnt.p, nr * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  GIFT_CUDA(cudaStreamSynchronize(st));
  std::vector<int32_t> idx(nr);
  for (int32_t i = 0; i < nr; ++i) idx[i] = i;
  const int K = std::min<int32_t>(nr, kCodes - 1);
  // most frequent first, ties by bit pattern: deterministic
  std::partial_sort(idx.begin(), idx.begin() + K, idx.end(), [&](int32_t x, int32_t y) {
    return hc[x] != hc[y] ? hc[x] > hc[y] : hu[x] < hu[y];
  });
  std::vector<float> vals(kCodes, 0.f);
  for (int i = 0; i < K; ++i) memcpy(&vals[i], &hu[idx[i]], sizeof(float));
  std::sort(vals.begin(), vals.begin() + K);
  for (int i = K; i < kCodes; ++i) vals[i] = 0.f;  // unused codes; 255 = padding
  GIFT_CUDA(cudaMemcpyAsync(tbl, vals.data(), kCodes * sizeof(float), cudaMemcpyHostToDevice, st));
  GIFT_CUDA(cudaStreamSynchronize(st));  // vals lives on this stack
  return K;
}

// Build the sliced block-major copy (once per graph; cached on the csr).
bool bmt_build(Ctx* ctx, Csr* c, const float* w32, Csr::Bmt& B, bool wide_blocks) {
  cudaStream_t st = ctx->stream;
  const bool coded = wide_blocks && ctx->opt.codes;  // tuning builds only (see launch_bmt_out)
  const int64_t n = c->n, nnz_all = c->nnz;
  const BmtShape shape = bmt_shape_for(ctx, c->n, c->mean_row, wide_blocks);
  const int kR = shape.kR, cb = shape.cb, kC = 1 << cb;
  const int64_t ntiles = (n + kR - 1) / kR;
  const int64_t nblocks = (n + kC - 1) / kC;
  const int bb = bit_length((uint64_t)(nblocks > 1 ? nblocks - 1 : 1));
  const int key_bits = bb + bit_length((uint64_t)(ntiles > 1 ? ntiles - 1 : 1)) + 1;  // + sentinel bit
  if (key_bits > 32 || c->nnz == 0) return false;
  const uint32_t sentinel = 1u << (key_bits - 1);
  // 0. wide rows -> row kernel
  B.wide = static_cast<uint8_t*>(csr_alloc(ctx, c, n));
  int64_t nwide = 0, nnz = c->nnz;
  {
    DevBuf<unsigned long long> wc(ctx, 3);
    GIFT_CUDA(cudaMemsetAsync(wc.p, 0, 3 * sizeof(unsigned long long), st));
    DevBuf<uint16_t> nb(ctx, n);
    k_row_nblocks<<<grid_for(n, kBlock), kBlock, 0, st>>>(n, c->indptr, c->indices, cb, nb.p, wc.p + 2);
    GIFT_LAUNCH_CHECK(ctx);
    const double mean_nb = (double)fetch(ctx, wc.p + 2) / (double)(n > 0 ? n : 1);
    const int limit = std::max(kWide, (int)(3.0 * mean_nb + 0.5));
    k_wide_rows<<<grid_for(n, kBlock), kBlock, 0, st>>>(n, c->indptr, nb.p, limit, B.wide, wc.p, wc.p + 1);
    GIFT_LAUNCH_CHECK(ctx);
    unsigned long long h[2];
    GIFT_CUDA(cudaMemcpyAsync(h, wc.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    GIFT_CUDA(cudaStreamSynchronize(st));
    nwide = (int64_t)h[0];
    nnz = c->nnz - (int64_t)h[1];  // entries kept in the tiled copy
    B.wide_rows = static_cast<int32_t*>(csr_alloc(ctx, c, (nwide + 1) * sizeof(int32_t)));
    if (nwide > 0) {
      DevBuf<int64_t> nsel1(ctx, 1);
      thrust::counting_iterator<int32_t> it(0);
      size_t bytes = 0;
      GIFT_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, it, B.wide, B.wide_rows, nsel1.p, n, st));
      DevBuf<char> tmp(ctx, bytes);
      GIFT_CUDA(cub::DeviceSelect::Flagged(tmp.p, bytes, it, B.wide, B.wide_rows, nsel1.p, n, st));
      ctx->launches += 2;
    }
  }
  if (nnz == 0) return false;
  // 1. row of every entry (scatter row ids at row starts, max-scan)
  DevBuf<int32_t> row_of(ctx, nnz_all);
  {
    DevBuf<int32_t> mark(ctx, nnz_all);
    GIFT_CUDA(cudaMemsetAsync(mark.p, 0, nnz_all * sizeof(int32_t), st));
    k_mark_rows<<<grid_for(n, kBlock), kBlock, 0, st>>>(n, c->indptr, mark.p);
    GIFT_LAUNCH_CHECK(ctx);
    size_t bytes = 0;
    GIFT_CUDA(cub::DeviceScan::InclusiveScan(nullptr, bytes, mark.p, row_of.p, MaxI32(), nnz_all, st));
    DevBuf<char> tmp(ctx, bytes);
    GIFT_CUDA(cub::DeviceScan::InclusiveScan(tmp.p, bytes, mark.p, row_of.p, MaxI32(), nnz_all, st));
    ctx->launches += 2;
  }
  // 2. stable sort by (tile, block): segments, CSR (row, column) order inside
  DevBuf<uint32_t> key_s(ctx, nnz_all);
  DevBuf<uint64_t> pay_s(ctx, nnz_all);
  {
    DevBuf<uint32_t> key(ctx, nnz_all);
    DevBuf<uint64_t> pay(ctx, nnz_all);
    k_bmt_keys<<<grid_for(nnz_all, kBlock), kBlock, 0, st>>>(nnz_all, row_of.p, c->indices, w32, bb, kR, cb, B.wide, sentinel,
                                                             key.p, pay.p);
    GIFT_LAUNCH_CHECK(ctx);
    row_of.reset();
    size_t bytes = 0;
    GIFT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, key.p, key_s.p, pay.p, pay_s.p, nnz_all, 0, key_bits,
                                              st));
    DevBuf<char> tmp(ctx, bytes);
    GIFT_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, key.p, key_s.p, pay.p, pay_s.p, nnz_all, 0, key_bits,
                                              st));
    ctx->launches += 4;
  }
  // entries [0, nnz) are the kept ones; wide rows' entries sorted past them
  // 2a. coded copy: the graph's 255 most frequent fp32 weights (from a sample of
  //     at most 2^24 entries) become u8 codes; on netlist graphs they cover
  //     ~99 % of the entries (single-net weights 2/m)
  int code_k = 0;
  if (coded) {
    B.code_tbl = static_cast<float*>(csr_alloc(ctx, c, kCodes * sizeof(float)));
    code_k = build_code_table(ctx, w32, nnz_all, B.code_tbl);
    B.coded_values = code_k;
  }
  // 2b. sparse segments -> residual CSR (gathered from L2 by the tile's rows);
  //     dense segments stay in the sliced copy (coded copy: so do only entries
  //     whose weight has a code)
  {
    DevBuf<uint8_t> seg_head(ctx, nnz), run_head(ctx, nnz);
    DevBuf<unsigned long long> cnt0(ctx, 2);
    DevBuf<int64_t> nsel0(ctx, 2);
    GIFT_CUDA(cudaMemsetAsync(cnt0.p, 0, 2 * sizeof(unsigned long long), st));
    k_bmt_heads<<<grid_for(nnz, kBlock), kBlock, 0, st>>>(nnz, cb, key_s.p, pay_s.p, seg_head.p, run_head.p, cnt0.p);
    GIFT_LAUNCH_CHECK(ctx);
    const int64_t nseg0 = (int64_t)fetch(ctx, cnt0.p);
    DevBuf<int64_t> seg0(ctx, nseg0 + 1);
    select_positions(ctx, seg_head.p, nnz, seg0.p, nsel0.p);
    run_head.reset();
    DevBuf<uint8_t>& sparse = seg_head;  // reuse
    DevBuf<uint8_t> dense(ctx, nnz);
    k_flag_sparse<<<(unsigned)std::min<int64_t>(nseg0, 65535), 256, 0, st>>>(nseg0, seg0.p, nnz, sparse.p, dense.p);
    GIFT_LAUNCH_CHECK(ctx);
    if (coded) {
      k_flag_uncoded<<<grid_for(nnz, kBlock), kBlock, 0, st>>>(nnz, pay_s.p, B.code_tbl, code_k, sparse.p, dense.p);
      GIFT_LAUNCH_CHECK(ctx);
    }
    // residual entries
    DevBuf<uint32_t> rk(ctx, nnz);
    DevBuf<uint64_t> rp(ctx, nnz);
    size_t bytes = 0, bytes2 = 0;
    GIFT_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, key_s.p, sparse.p, rk.p, nsel0.p, nnz, st));
    GIFT_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes2, pay_s.p, sparse.p, rp.p, nsel0.p + 1, nnz, st));
    bytes = std::max(bytes, bytes2);
    {
      DevBuf<char> tmp(ctx, bytes);
      GIFT_CUDA(cub::DeviceSelect::Flagged(tmp.p, bytes, key_s.p, sparse.p, rk.p, nsel0.p, nnz, st));
      GIFT_CUDA(cub::DeviceSelect::Flagged(tmp.p, bytes, pay_s.p, sparse.p, rp.p, nsel0.p + 1, nnz, st));
    }
    const int64_t nres = fetch(ctx, nsel0.p);
    B.res_rowptr = static_cast<int64_t*>(csr_alloc(ctx, c, (n + 1) * sizeof(int64_t)));
    B.res_col = static_cast<int32_t*>(csr_alloc(ctx, c, (nres + 1) * sizeof(int32_t)));
    B.res_w = static_cast<float*>(csr_alloc(ctx, c, (nres + 1) * sizeof(float)));
    if (nres > 0) {
      DevBuf<uint32_t> rkey(ctx, nres), rkey_s2(ctx, nres);
      DevBuf<uint64_t> rpay(ctx, nres), rpay_s2(ctx, nres);
      k_residual_keys<<<grid_for(nres, kBlock), kBlock, 0, st>>>(nres, rk.p, rp.p, bb, kR, cb, rkey.p, rpay.p);
      GIFT_LAUNCH_CHECK(ctx);
      const int row_bits = bit_length((uint64_t)(n > 1 ? n - 1 : 1));
      GIFT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, rkey.p, rkey_s2.p, rpay.p, rpay_s2.p, nres, 0,
                                                row_bits, st));
      DevBuf<char> tmp(ctx, bytes);
      GIFT_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, rkey.p, rkey_s2.p, rpay.p, rpay_s2.p, nres, 0,
                                                row_bits, st));
      ctx->launches += 4;
      k_residual_split<<<grid_for(nres + 1, kBlock), kBlock, 0, st>>>(nres, rkey_s2.p, rpay_s2.p, n, B.res_rowptr,
                                                                      B.res_col, B.res_w);
      GIFT_LAUNCH_CHECK(ctx);
    } else {
      GIFT_CUDA(cudaMemsetAsync(B.res_rowptr, 0, (n + 1) * sizeof(int64_t), st));
    }
    B.nres = nres;
    {  // rows with residual entries per tile (the tile epilogue visits only those)
      DevBuf<uint8_t> flag(ctx, n);
      k_has_res<<<grid_for(n, kBlock), kBlock, 0, st>>>(n, B.res_rowptr, flag.p);
      GIFT_LAUNCH_CHECK(ctx);
      const int64_t cap = std::min<int64_t>(n, nres);
      B.res_rows = static_cast<int64_t*>(csr_alloc(ctx, c, (cap + 1) * sizeof(int64_t)));
      int64_t m = 0;
      if (cap > 0) {
        select_positions(ctx, flag.p, n, B.res_rows, nsel0.p);
        m = fetch(ctx, nsel0.p);
      }
      B.tile_res = static_cast<int64_t*>(csr_alloc(ctx, c, (ntiles + 1) * sizeof(int64_t)));
      k_tile_res<<<grid_for(ntiles + 1, kBlock), kBlock, 0, st>>>(ntiles, kR, B.res_rows, m, B.tile_res);
      GIFT_LAUNCH_CHECK(ctx);
    }
    // compact the dense entries (order preserved)
    DevBuf<uint32_t> k2(ctx, nnz - nres + 1);
    DevBuf<uint64_t> p2(ctx, nnz - nres + 1);
    GIFT_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, key_s.p, dense.p, k2.p, nsel0.p, nnz, st));
    GIFT_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes2, pay_s.p, dense.p, p2.p, nsel0.p + 1, nnz, st));
    bytes = std::max(bytes, bytes2);
    {
      DevBuf<char> tmp(ctx, bytes);
      GIFT_CUDA(cub::DeviceSelect::Flagged(tmp.p, bytes, key_s.p, dense.p, k2.p, nsel0.p, nnz, st));
      GIFT_CUDA(cub::DeviceSelect::Flagged(tmp.p, bytes, pay_s.p, dense.p, p2.p, nsel0.p + 1, nnz, st));
    }
    ctx->launches += 8;
    nnz -= nres;
    key_s = std::move(k2);
    pay_s = std::move(p2);
  }
  if (nnz <= 0) return false;
  // 3. segment and run heads; segment index of every entry
  DevBuf<unsigned long long> counts(ctx, 2);
  DevBuf<int64_t> nsel(ctx, 2);
  DevBuf<int64_t> seg_start, run_start;
  int64_t nseg = 0, nruns = 0;
  {
    DevBuf<uint8_t> seg_head(ctx, nnz), run_head(ctx, nnz);
    GIFT_CUDA(cudaMemsetAsync(counts.p, 0, 2 * sizeof(unsigned long long), st));
    k_bmt_heads<<<grid_for(nnz, kBlock), kBlock, 0, st>>>(nnz, cb, key_s.p, pay_s.p, seg_head.p, run_head.p, counts.p);
    GIFT_LAUNCH_CHECK(ctx);
    unsigned long long h[2];
    GIFT_CUDA(cudaMemcpyAsync(h, counts.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    GIFT_CUDA(cudaStreamSynchronize(st));
    nseg = (int64_t)h[0];
    nruns = (int64_t)h[1];
    seg_start = DevBuf<int64_t>(ctx, nseg + 1);
    run_start = DevBuf<int64_t>(ctx, nruns + 1);
    select_positions(ctx, seg_head.p, nnz, seg_start.p, nsel.p);
    select_positions(ctx, run_head.p, nnz, run_start.p, nsel.p + 1);
  }
  if (nseg >= (1LL << 40)) return false;
  // 4. sort runs inside segments: longest first (stable: row order among equal lengths)
  DevBuf<uint64_t> rkey_s(ctx, nruns);
  DevBuf<int64_t> run_perm(ctx, nruns);
  {
    DevBuf<uint64_t> rkey(ctx, nruns);
    DevBuf<int64_t> iota(ctx, nruns);
    k_run_keys<<<grid_for(nruns, kBlock), kBlock, 0, st>>>(nruns, run_start.p, nnz, seg_start.p, nseg, cb, rkey.p);
    GIFT_LAUNCH_CHECK(ctx);
    k_iota64<<<grid_for(nruns, kBlock), kBlock, 0, st>>>(nruns, iota.p);
    GIFT_LAUNCH_CHECK(ctx);
    const int rbits = cb + 1 + bit_length((uint64_t)nseg);
    size_t bytes = 0;
    GIFT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, rkey.p, rkey_s.p, iota.p, run_perm.p, nruns, 0, rbits,
                                              st));
    DevBuf<char> tmp(ctx, bytes);
    GIFT_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, rkey.p, rkey_s.p, iota.p, run_perm.p, nruns, 0, rbits,
                                              st));
    ctx->launches += 4;
  }
  // 5. slices: ceil(runs / 32) per segment; slots from each slice's longest run
  DevBuf<int64_t> seg_run(ctx, nseg + 1), nsl(ctx, nseg + 1);
  k_seg_runs<<<grid_for(nruns + 1, kBlock), kBlock, 0, st>>>(nruns, rkey_s.p, nseg, cb, seg_run.p);
  GIFT_LAUNCH_CHECK(ctx);
  k_seg_slices<<<grid_for(nseg, kBlock), kBlock, 0, st>>>(nseg, seg_run.p, nsl.p);
  GIFT_LAUNCH_CHECK(ctx);
  GIFT_CUDA(cudaMemsetAsync(nsl.p + nseg, 0, sizeof(int64_t), st));
  B.seg_slice = static_cast<int64_t*>(csr_alloc(ctx, c, (nseg + 1) * sizeof(int64_t)));
  exclusive_sum(ctx, nsl.p, B.seg_slice, nseg + 1);
  const int64_t nslices = fetch(ctx, B.seg_slice + nseg);
  DevBuf<int64_t> slots(ctx, nslices + 1);
  GIFT_CUDA(cudaMemsetAsync(slots.p + nslices, 0, sizeof(int64_t), st));
  k_slice_len<<<grid_for(nseg, kBlock), kBlock, 0, st>>>(nseg, seg_run.p, B.seg_slice, rkey_s.p, cb, slots.p);
  GIFT_LAUNCH_CHECK(ctx);
  B.slice_off = static_cast<int64_t*>(csr_alloc(ctx, c, (nslices + 1) * sizeof(int64_t)));
  exclusive_sum(ctx, slots.p, B.slice_off, nslices + 1);
  const int64_t total = fetch(ctx, B.slice_off + nslices);
  // 6. scatter entries into slices; padding = column kC (zero signal row), weight 0
  B.slice_rows = static_cast<uint16_t*>(csr_alloc(ctx, c, (nslices * 32 + 1) * sizeof(uint16_t)));
  DevBuf<uint16_t> colb(ctx, total + 8);
  DevBuf<float> wb(ctx, total + 8);
  uint16_t* const bcol = colb.p;
  float* const bw = wb.p;
  k_fill_u16<<<grid_for(nslices * 32, kBlock), kBlock, 0, st>>>(nslices * 32, 0xffff, B.slice_rows);
  GIFT_LAUNCH_CHECK(ctx);
  k_fill_u16<<<grid_for(total, kBlock), kBlock, 0, st>>>(total, (uint16_t)kC, bcol);
  GIFT_LAUNCH_CHECK(ctx);
  GIFT_CUDA(cudaMemsetAsync(bw, 0, total * sizeof(float), st));
  k_scatter_runs<<<(unsigned)std::min<int64_t>(nseg, 65535), 256, 0, st>>>(
      nseg, seg_run.p, B.seg_slice, run_perm.p, run_start.p, nruns, nnz, cb, pay_s.p, B.slice_off, B.slice_rows, bcol,
      bw);
  GIFT_LAUNCH_CHECK(ctx);
  if (ctx->opt.schedule) {
    DevBuf<uint16_t> tcol(ctx, total + 8);
    DevBuf<float> tw(ctx, total + 8);
    if (ctx->opt.schedule == 2 && !wide_blocks && !coded)  // the F = 4 copy: optimal per quarter warp
      k_slice_schedule_bvn<<<grid_for(nslices * 32, 256, 1LL << 30), 256, 0, st>>>(nslices, kC, B.slice_off, bcol, bw,
                                                                                  tcol.p, tw.p);
    else
      k_slice_schedule<<<grid_for(nslices * 32, 256, 1LL << 30), 256, 0, st>>>(nslices, kC, B.slice_off, bcol, bw,
                                                                              tcol.p, tw.p);
    GIFT_LAUNCH_CHECK(ctx);
  }
  if (coded) {
    B.data = static_cast<uint8_t*>(csr_alloc(ctx, c, (total / 128 + 1) * 384));
    k_interleave_coded<<<grid_for(total, kBlock), kBlock, 0, st>>>(total, bcol, bw, B.code_tbl, code_k, B.data);
  } else {
    B.data = static_cast<uint8_t*>(csr_alloc(ctx, c, (total / 128 + 1) * 768));
    k_interleave<<<grid_for(total, kBlock), kBlock, 0, st>>>(total, bcol, bw, B.data);
  }
  GIFT_LAUNCH_CHECK(ctx);
  B.coded = coded;
  colb.reset();
  wb.reset();
  // 7. segment codes and tile -> segment ranges
  B.seg_code = static_cast<int32_t*>(csr_alloc(ctx, c, (nseg + 1) * sizeof(int32_t)));
  B.tile_seg = static_cast<int64_t*>(csr_alloc(ctx, c, (ntiles + 1) * sizeof(int64_t)));
  DevBuf<uint32_t> seg_tile(ctx, nseg + 1);
  k_seg_meta<<<grid_for(nseg, kBlock), kBlock, 0, st>>>(nseg, seg_start.p, key_s.p, nnz, bb, B.seg_code, seg_tile.p);
  GIFT_LAUNCH_CHECK(ctx);
  k_bmt_tile_ptr<<<grid_for(nseg + 1, kBlock), kBlock, 0, st>>>(nseg, seg_tile.p, ntiles, B.tile_seg);
  GIFT_LAUNCH_CHECK(ctx);
  // 8. persistent-scheduler order: costliest tiles first (host sort of ntiles keys)
  B.tile_order = static_cast<int32_t*>(csr_alloc(ctx, c, (ntiles + 1) * sizeof(int32_t)));
  {
    DevBuf<int64_t> cost(ctx, ntiles);
    k_tile_cost<<<grid_for(ntiles, kBlock), kBlock, 0, st>>>(ntiles, kR, kC, n, B.tile_seg, B.seg_slice, B.slice_off,
                                                            B.res_rowptr, cost.p);
    GIFT_LAUNCH_CHECK(ctx);
    std::vector<int64_t> hc(ntiles);
    GIFT_CUDA(cudaMemcpyAsync(hc.data(), cost.p, ntiles * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    GIFT_CUDA(cudaStreamSynchronize(st));
    // heavy tiles (> 1.25 x the median cost) first, costliest first; the rest
    // keep index order, so CTAs resident together work on neighbouring tiles
    // and share the signal blocks they stage in L2 (a full cost sort scatters
    // them: +12 % DRAM bytes on config 4, whose tiles are uniform)
    std::vector<int64_t> sorted(hc);
    std::nth_element(sorted.begin(), sorted.begin() + ntiles / 2, sorted.end());
    const double heavy = 1.25 * (double)sorted[ntiles / 2];
    std::vector<int32_t> order(ntiles);
    for (int64_t t = 0; t < ntiles; ++t) order[t] = (int32_t)t;
    std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) {
      const bool hx = (double)hc[x] > heavy, hy = (double)hc[y] > heavy;
      if (hx != hy) return hx;
      return hx && hc[x] > hc[y];
    });
    GIFT_CUDA(cudaMemcpyAsync(B.tile_order, order.data(), ntiles * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  }
  GIFT_CUDA(cudaStreamSynchronize(st));
  B.ntiles = ntiles;
  B.tile_rows = kR;
  B.kC = kC;
  B.nwide = nwide;
  B.nseg = nseg;
  B.nslices = nslices;
  B.slots = total;
  return true;
}

}  // namespace

const float* csr_w32_public(Ctx* ctx, Csr* c);
void launch_row_list(Ctx* ctx, cudaStream_t st, const HopArgs& base, const int32_t* rows, int64_t nrows, int fin,
                     int fout, int G);

bool bmt_possible(Ctx* ctx, const Csr* c) {
  if (!ctx->opt.tiled || !c->sorted_rows || !c->square) return false;
  if (ctx->tiled_policy == GIFT_TILED_NEVER && !c->bmt.ready && !c->bmt_wide.ready) return false;
  return c->n >= ctx->opt.tiled_min_rows && c->mean_row >= (double)ctx->opt.tiled_min_mean;
}

bool bmt_hop(Ctx* ctx, Csr* c, const HopArgs& a, int fin, int fout) {
  if (!ctx->opt.tiled || !c->sorted_rows || !c->square) return false;
  // building the tiled copy costs ~a few hops; only resident graphs amortise it
  // signal widths <= 2 use the wide-block copy, F = 4 its own (unless a
  // tuning shape is forced: then one copy serves every width)
  const bool wide_blocks = fin <= 2 && ctx->opt.tile_rows == 0 && ctx->opt.col_bits == 0;
  Csr::Bmt& B = wide_blocks ? c->bmt_wide : c->bmt;
  // build policy (GIFT_TILED_*): a graph filtered once (gift_place on a fresh
  // design, cli.py:203-220) never pays for the copy; one filtered again gets it
  if (!B.ready && (ctx->tiled_policy == GIFT_TILED_NEVER ||
                   (ctx->tiled_policy == GIFT_TILED_ON_REUSE && c->fp32_hops < kReuseHops)))
    return false;
  if (c->n < ctx->opt.tiled_min_rows || c->mean_row < (double)ctx->opt.tiled_min_mean) return false;
  // whole square graphs only; partial sums in (part_in: the high-fanout term)
  // or out (part_out: a shard's local block) pass through the row epilogue
  if (a.row_begin != 0 || a.n != c->n) return false;
  if (!B.ready) {
    B.ready = true;
    // the tiled copy is an optimisation: if device memory runs out while it is
    // built (its temporaries take ~3x the matrix), free what it got and let
    // the row kernel serve this graph
    const size_t mark = c->owned.size();
    try {
      B.ok = bmt_build(ctx, c, csr_w32_public(ctx, c), B, wide_blocks);
    } catch (const GiftException& e) {
      if (e.code != GIFT_ERR_OOM) throw;
      for (size_t i = mark; i < c->owned.size(); ++i) dev_free(ctx, c->owned[i]);
      c->owned.resize(mark);
      B = Csr::Bmt{};
      B.ready = true;
      B.ok = false;
    }
  }
  if (!B.ok) return false;
  // a tuning shape may not fit this signal width's shared-memory footprint
  if (bmt_smem(fin, B.tile_rows, B.kC, B.coded) + 1024 > (size_t)ctx->smem_optin) return false;
  // the wide rows (pads / macros, long rows) run concurrently on a side stream:
  // disjoint output rows, same input signal
  const bool fork = B.nwide > 0;
  if (fork) {
    if (!ctx->side) {
      GIFT_CUDA(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
      GIFT_CUDA(cudaEventCreateWithFlags(&ctx->fork_ev, cudaEventDisableTiming));
      GIFT_CUDA(cudaEventCreateWithFlags(&ctx->join_ev, cudaEventDisableTiming));
    }
    GIFT_CUDA(cudaEventRecord(ctx->fork_ev, ctx->stream));
    GIFT_CUDA(cudaStreamWaitEvent(ctx->side, ctx->fork_ev, 0));
    launch_row_list(ctx, ctx->side, a, B.wide_rows, B.nwide, fin, fout, 32);
    GIFT_CUDA(cudaEventRecord(ctx->join_ev, ctx->side));
  }
  unsigned* ctr = nullptr;
  const int32_t* order = B.tile_order;
#ifdef GIFT_TUNING
  if (!env_int("GIFT_BMT_LPT", 1)) order = nullptr;
  if (env_int("GIFT_BMT_PERSIST", 0)) {
    order = B.tile_order;
    unsigned*& slot = ctx->tile_ctr[ctx->stream];
    if (!slot) {
      GIFT_CUDA(cudaMalloc(&slot, 2 * sizeof(unsigned)));
      GIFT_CUDA(cudaMemsetAsync(slot, 0, 2 * sizeof(unsigned), ctx->stream));
    }
    ctr = slot;
  }
#endif
  BmtArgs b{c->n,         B.tile_rows,  B.kC,         B.data,      B.wide,      B.res_rowptr, B.res_col,     B.res_w,
            B.tile_seg,   B.seg_code,   B.seg_slice, B.slice_off, B.slice_rows, order,         ctr,
            B.ntiles,     B.res_rows,   B.tile_res,  B.code_tbl,  (int)ctx->opt.prefetch,
            (int)ctx->opt.stream};
  switch (fin) {
    case 1: launch_bmt_out<1>(ctx, a, b, B.ntiles, fout, B.coded); break;
    case 2: launch_bmt_out<2>(ctx, a, b, B.ntiles, fout, B.coded); break;
    default: launch_bmt_out<4>(ctx, a, b, B.ntiles, fout, false); break;
  }
  if (fork) GIFT_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->join_ev, 0));
  return true;
}

}  // namespace gift
