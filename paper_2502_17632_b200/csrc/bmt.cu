// bmt.cu -- block-major tiled (BMT) fp32 hop: the signal is gathered from
// shared memory instead of through L1.
//
// Why: the row kernel (filter.cu k_hop) streams (col, w) at full coalescing
// but every stored entry gathers one signal row z_j (8-16 B) from L1/L2; on
// c2/c3 those scattered gathers keep the L1TEX pipe ~90% busy and the kernel
// at ~50-60% of HBM bandwidth (profiles/r01_v2_k_hop_c3.txt).  Netlist
// graphs are banded (nets live in +-W index windows), so a tile of rows only
// touches a few column blocks.  BMT reorders a copy of the matrix so that
// each (row tile, column block) pair is one contiguous SEGMENT:
//
//   tiles of kR = 2048 rows, blocks of kC = 4096 columns;
//   segments ordered tile-major, block ascending; inside a segment entries
//   keep CSR order (row, then column) -- a stable sort by (tile, block);
//   entry = u32 (row in tile << 12 | column in block) + f32 weight: 8 B, the
//   same stream bytes as (int32 col, f32 w).
//
// A CTA owns a tile.  For each segment it stages the 64 KB signal block in
// shared memory (dense segments; sparse ones -- pad / macro columns -- gather
// from L2 directly) and its warps stream the segment: warp-level units are
// row-aligned runs of ~256 entries, so every row of a segment is summed by
// one warp: lane-local segmented scan over 8 entries, a 5-step segmented
// Hillis-Steele scan across lanes, a register carry across chunks.  Row sums
// land in a per-tile shared accumulator (blocks ascending), then the shared
// row epilogue of hop.cuh runs per row.  Fixed reduction tree everywhere ->
// deterministic.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <climits>
#include <cstring>

#include "common.cuh"
#include "hop.cuh"

namespace gift {

namespace {

constexpr int kR = 2048;        // rows per tile (11 bits)
constexpr int kCbits = 12;
constexpr int kC = 1 << kCbits;  // columns per block
constexpr int kThreads = 512;
template <int FIN>
__host__ __device__ constexpr int kVof() { return FIN >= 4 ? 4 : 8; }  // entries per lane per chunk (register budget: 64 at 2 CTAs/SM)
constexpr int kStage = 1024;    // a segment with >= kStage entries stages its block
constexpr int kBlock = 256;

__global__ void k_mark_rows(int64_t n, const int64_t* __restrict__ indptr, int32_t* __restrict__ mark) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    if (indptr[r + 1] > indptr[r]) mark[indptr[r]] = (int32_t)r;
}

struct MaxI32 {
  __device__ __forceinline__ int32_t operator()(int32_t a, int32_t b) const { return a > b ? a : b; }
};

__global__ void k_bmt_keys(int64_t nnz, const int32_t* __restrict__ row_of, const int32_t* __restrict__ col,
                           const float* __restrict__ w, int bb, uint32_t* __restrict__ key,
                           uint64_t* __restrict__ payload) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t r = (uint32_t)row_of[k], c = (uint32_t)col[k];
    key[k] = ((r / kR) << bb) | (c >> kCbits);
    const uint32_t packed = ((r % kR) << kCbits) | (c & (kC - 1));
    payload[k] = ((uint64_t)__float_as_uint(w[k]) << 32) | packed;
  }
}

// segment heads (key change) and unit boundaries (segment heads, plus row
// heads whose row group of D consecutive rows differs from the previous row's)
__global__ void k_bmt_flags(int64_t nnz, const uint32_t* __restrict__ key, const uint64_t* __restrict__ payload,
                            int D, uint8_t* __restrict__ seg_head, uint8_t* __restrict__ unit_head,
                            unsigned long long* __restrict__ row_heads) {
  unsigned long long cnt = 0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
    const bool sh = k == 0 || key[k] != key[k - 1];
    const uint32_t r = (uint32_t)payload[k] >> kCbits;
    const uint32_t rp = k == 0 ? 0xffffffffu : (uint32_t)payload[k - 1] >> kCbits;
    const bool rh = sh || r != rp;
    seg_head[k] = sh;
    unit_head[k] = sh || (rh && (r / D) != (rp / D));
    cnt += rh;
  }
  if (row_heads) atomicAdd(row_heads, cnt);
}

__global__ void k_bmt_split(int64_t nnz, const uint64_t* __restrict__ payload, uint32_t* __restrict__ idx,
                            float* __restrict__ w) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t p = payload[k];
    idx[k] = (uint32_t)p;
    w[k] = __uint_as_float((uint32_t)(p >> 32));
  }
}

__global__ void k_bmt_segs(int64_t nseg, const int64_t* __restrict__ seg_start, const uint32_t* __restrict__ key_s,
                           int64_t nnz, int bb, const int64_t* __restrict__ unit_start, int64_t nunits,
                           int32_t* __restrict__ seg_code, int64_t* __restrict__ seg_unit,
                           uint32_t* __restrict__ seg_tile) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s <= nseg; s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = s < nseg ? seg_start[s] : nnz;
    // first unit starting at or after a (segment starts are unit starts)
    int64_t lo = 0, hi = nunits;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (unit_start[mid] < a) lo = mid + 1;
      else hi = mid;
    }
    seg_unit[s] = lo;
    if (s < nseg) {
      const int64_t b = s + 1 < nseg ? seg_start[s + 1] : nnz;
      const uint32_t k = key_s[a];
      const int blk = (int)(k & ((1u << bb) - 1));
      seg_code[s] = (b - a) >= kStage ? blk : -(blk + 1);
      seg_tile[s] = k >> bb;
    }
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

struct BmtArgs {
  int64_t ncols;
  const int64_t* tile_seg;
  const int32_t* seg_code;
  const int64_t* seg_unit;
  const int64_t* unit_start;
  const uint32_t* idx;
  const float* w;
};

template <int F>
__device__ __forceinline__ void add_to(float (&d)[F], const float (&s)[F]) {
#pragma unroll
  for (int f = 0; f < F; ++f) d[f] += s[f];
}

template <int FIN, int FOUT>
__global__ void __launch_bounds__(kThreads, 2) k_hop_bmt(HopArgs a, BmtArgs b) {
  constexpr int kV = kVof<FIN>();
  extern __shared__ float4 smem_f4[];
  float* zs = reinterpret_cast<float*>(smem_f4);  // [kC * FIN]
  float* accs = zs + kC * FIN;                      // [kR * FIN]
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  constexpr int NW = kThreads / 32;
  const int64_t tile = blockIdx.x;
  const int64_t r0 = tile * kR;
  const int nrows = (int)min((int64_t)kR, a.n - r0);
  const uint64_t pol_s = policy_evict_first();
  const uint64_t pol_z = policy_evict_last();
  for (int i = tid; i < nrows * FIN; i += kThreads) accs[i] = 0.f;
  const int64_t s_end = b.tile_seg[tile + 1];
  for (int64_t s = b.tile_seg[tile]; s < s_end; ++s) {
    const int code = b.seg_code[s];
    const bool staged = code >= 0;
    const int64_t cbase = (int64_t)(staged ? code : -code - 1) * kC;
    __syncthreads();  // previous segment's readers are done with zs
    if (staged) {
      const int64_t cend = min(cbase + kC, b.ncols);
      const float4* src = reinterpret_cast<const float4*>(a.zin + cbase * FIN);
      float4* dst = reinterpret_cast<float4*>(zs);
      const int nv = (int)(((cend - cbase) * FIN + 3) / 4);
#pragma unroll 4
      for (int i = tid; i < nv; i += kThreads) dst[i] = src[i];
    }
    __syncthreads();
    const float* zg = a.zin + cbase * FIN;
    const int64_t u_end = b.seg_unit[s + 1];
    for (int64_t u = b.seg_unit[s] + warp; u < u_end; u += NW) {
      const int64_t us = b.unit_start[u], ue = b.unit_start[u + 1];
      int carry_row = -1;
      float carry[FIN];
#pragma unroll
      for (int f = 0; f < FIN; ++f) carry[f] = 0.f;
      for (int64_t cb = us & ~(int64_t)3; cb < ue; cb += 32 * kV) {
        const int64_t e0 = cb + (int64_t)kV * lane;
        int rowl[kV];
        float p[kV][FIN];
        {
          uint32_t ix[kV];
          float wv[kV];
#pragma unroll
          for (int h = 0; h < kV / 4; ++h) {
            const int64_t e = e0 + 4 * h;
            int4 iv = make_int4(0, 0, 0, 0);
            float4 ww = make_float4(0.f, 0.f, 0.f, 0.f);
            if (e < ue) {
              iv = ld_stream_v4s32(reinterpret_cast<const int32_t*>(b.idx) + e, pol_s);
              ww = ld_stream_v4f32(b.w + e, pol_s);
            }
            ix[4 * h + 0] = (uint32_t)iv.x; ix[4 * h + 1] = (uint32_t)iv.y;
            ix[4 * h + 2] = (uint32_t)iv.z; ix[4 * h + 3] = (uint32_t)iv.w;
            wv[4 * h + 0] = ww.x; wv[4 * h + 1] = ww.y; wv[4 * h + 2] = ww.z; wv[4 * h + 3] = ww.w;
          }
#pragma unroll
          for (int j = 0; j < kV; ++j) {
            const int64_t e = e0 + j;
            const bool valid = e >= us && e < ue;
            rowl[j] = valid ? (int)(ix[j] >> kCbits) : -1;
            const int cl = (int)(ix[j] & (kC - 1));
            float zq[FIN];
#pragma unroll
            for (int f = 0; f < FIN; ++f) zq[f] = 0.f;
            if (valid) {
              if (staged) {
                const float* zp = zs + cl * FIN;
                if constexpr (FIN == 4) {
                  const float4 q = *reinterpret_cast<const float4*>(zp);
                  zq[0] = q.x; zq[1] = q.y; zq[2] = q.z; zq[3] = q.w;
                } else if constexpr (FIN == 2) {
                  const float2 q = *reinterpret_cast<const float2*>(zp);
                  zq[0] = q.x; zq[1] = q.y;
                } else {
                  zq[0] = zp[0];
                }
              } else {
                const VecF<FIN> q = ld_z<FIN>(zg + (int64_t)cl * FIN, pol_z);
#pragma unroll
                for (int f = 0; f < FIN; ++f) zq[f] = q.v[f];
              }
            }
#pragma unroll
            for (int f = 0; f < FIN; ++f) p[j][f] = wv[j] * zq[f];
          }
        }
        // lane-local inclusive segmented scan (rows are sorted inside a unit)
#pragma unroll
        for (int j = 1; j < kV; ++j)
          if (rowl[j] == rowl[j - 1]) add_to<FIN>(p[j], p[j - 1]);
        const int head = rowl[0], tail = rowl[kV - 1];
        // the chunk carry flows into lane 0's first run
        const int c_row = __shfl_sync(0xffffffffu, carry_row, 0);
        float cin[FIN];
#pragma unroll
        for (int f = 0; f < FIN; ++f) cin[f] = 0.f;
        if (lane == 0 && c_row >= 0 && c_row == head) {
#pragma unroll
          for (int f = 0; f < FIN; ++f) cin[f] = carry[f];
        }
        if (lane == 0 && c_row >= 0 && c_row != head) {
          // the carried row ended exactly at the previous chunk boundary
#pragma unroll
          for (int f = 0; f < FIN; ++f) accs[c_row * FIN + f] += carry[f];
        }
        // segmented scan of lane tails: S_l = tail_l + (continues ? S_{l-1} : 0)
        const int prev_tail = __shfl_up_sync(0xffffffffu, tail, 1);
        const bool single = head == tail;
        int flag = (lane == 0) ? 1 : (single && prev_tail == head && head >= 0 ? 0 : 1);
        float sv[FIN];
#pragma unroll
        for (int f = 0; f < FIN; ++f) sv[f] = p[kV - 1][f] + (single ? cin[f] : 0.f);
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const int fu = __shfl_up_sync(0xffffffffu, flag, d);
          float vu[FIN];
#pragma unroll
          for (int f = 0; f < FIN; ++f) vu[f] = __shfl_up_sync(0xffffffffu, sv[f], d);
          if (lane >= d) {
            if (!flag) add_to<FIN>(sv, vu);
            flag |= fu;
          }
        }
        // carry into this lane's first run from the lanes before it
        float pin[FIN];
#pragma unroll
        for (int f = 0; f < FIN; ++f) {
          const float up = __shfl_up_sync(0xffffffffu, sv[f], 1);
          pin[f] = (lane > 0 && prev_tail == head && head >= 0) ? up : cin[f];
        }
        const int next_head = __shfl_down_sync(0xffffffffu, head, 1);
        // run ends: write finished rows; lane 31's tail becomes the chunk carry
#pragma unroll
        for (int j = 0; j < kV; ++j) {
          const int r = rowl[j];
          if (r < 0) continue;
          const bool last_in_lane = j == kV - 1;
          const int nxt = last_in_lane ? (lane < 31 ? next_head : INT_MIN) : rowl[j + 1];
          if (nxt == r) continue;       // the run goes on
          if (nxt == INT_MIN) continue;  // chunk end: carried below
          float v[FIN];
#pragma unroll
          for (int f = 0; f < FIN; ++f) v[f] = p[j][f] + (r == head ? pin[f] : 0.f);
#pragma unroll
          for (int f = 0; f < FIN; ++f) accs[r * FIN + f] += v[f];
        }
        // new carry: lane 31's tail run (including everything before it in this row)
        const int t31 = __shfl_sync(0xffffffffu, tail, 31);
        float tv[FIN];
#pragma unroll
        for (int f = 0; f < FIN; ++f) {
          const float mine = p[kV - 1][f] + (tail == head ? pin[f] : 0.f);
          tv[f] = __shfl_sync(0xffffffffu, mine, 31);
        }
        carry_row = t31;
#pragma unroll
        for (int f = 0; f < FIN; ++f) carry[f] = tv[f];
      }
      if (lane == 0 && carry_row >= 0) {
#pragma unroll
        for (int f = 0; f < FIN; ++f) accs[carry_row * FIN + f] += carry[f];
      }
    }
  }
  __syncthreads();
  for (int rr = tid; rr < nrows; rr += kThreads) {
    float acc[FIN];
#pragma unroll
    for (int f = 0; f < FIN; ++f) acc[f] = accs[rr * FIN + f];
    row_epilogue<FIN, FOUT>(a, r0 + rr, acc, pol_z);
  }
}

size_t bmt_smem(int fin) { return (size_t)kC * fin * 4 + (size_t)kR * fin * 4; }

template <int FIN, int FOUT>
void launch_bmt(Ctx* ctx, const HopArgs& a, const BmtArgs& b, int64_t ntiles) {
  auto kern = k_hop_bmt<FIN, FOUT>;
  static bool configured = false;  // one flag per template instance
  const size_t smem = bmt_smem(FIN);
  if (!configured) {
    GIFT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = true;
  }
  kern<<<(unsigned)ntiles, kThreads, smem, ctx->stream>>>(a, b);
  GIFT_LAUNCH_CHECK(ctx);
}

template <int FIN>
void launch_bmt_out(Ctx* ctx, const HopArgs& a, const BmtArgs& b, int64_t ntiles, int fout) {
  switch (fout) {
    case 0: launch_bmt<FIN, 0>(ctx, a, b, ntiles); break;
    case 1: launch_bmt<FIN, 1>(ctx, a, b, ntiles); break;
    case 2: launch_bmt<FIN, 2>(ctx, a, b, ntiles); break;
    default: launch_bmt<FIN, 4>(ctx, a, b, ntiles); break;
  }
}

template <typename T>
T fetch(Ctx* ctx, const T* d) {
  T h;
  GIFT_CUDA(cudaMemcpyAsync(&h, d, sizeof(T), cudaMemcpyDeviceToHost, ctx->stream));
  GIFT_CUDA(cudaStreamSynchronize(ctx->stream));
  return h;
}

// Build the block-major copy (once per graph; cached on the csr).
bool bmt_build(Ctx* ctx, Csr* c, const float* w32) {
  Csr::Bmt& B = c->bmt;
  cudaStream_t st = ctx->stream;
  const int64_t n = c->n, nnz = c->nnz;
  const int64_t ntiles = (n + kR - 1) / kR;
  const int64_t nblocks = (n + kC - 1) / kC;
  const int bb = bit_length((uint64_t)(nblocks > 1 ? nblocks - 1 : 1));
  const int key_bits = bb + bit_length((uint64_t)(ntiles > 1 ? ntiles - 1 : 1));
  if (key_bits > 32 || nnz >= (1LL << 31) * 2) return false;
  // row of every entry: scatter row ids at row starts, max-scan
  DevBuf<int32_t> mark(ctx, nnz), row_of(ctx, nnz);
  GIFT_CUDA(cudaMemsetAsync(mark.p, 0, nnz * sizeof(int32_t), st));
  k_mark_rows<<<grid_for(n, kBlock), kBlock, 0, st>>>(n, c->indptr, mark.p);
  GIFT_LAUNCH_CHECK(ctx);
  size_t bytes = 0;
  GIFT_CUDA(cub::DeviceScan::InclusiveScan(nullptr, bytes, mark.p, row_of.p, MaxI32(), nnz, st));
  DevBuf<char> tmp(ctx, bytes);
  GIFT_CUDA(cub::DeviceScan::InclusiveScan(tmp.p, bytes, mark.p, row_of.p, MaxI32(), nnz, st));
  ctx->launches += 2;
  mark.reset();
  tmp.reset();
  DevBuf<uint32_t> key(ctx, nnz), key_s(ctx, nnz);
  DevBuf<uint64_t> pay(ctx, nnz), pay_s(ctx, nnz);
  k_bmt_keys<<<grid_for(nnz, kBlock), kBlock, 0, st>>>(nnz, row_of.p, c->indices, w32, bb, key.p, pay.p);
  GIFT_LAUNCH_CHECK(ctx);
  row_of.reset();
  GIFT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, key.p, key_s.p, pay.p, pay_s.p, nnz, 0, key_bits, st));
  tmp = DevBuf<char>(ctx, bytes);
  GIFT_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, key.p, key_s.p, pay.p, pay_s.p, nnz, 0, key_bits, st));
  ctx->launches += 4;
  tmp.reset();
  key.reset();
  pay.reset();
  // unit granularity: D consecutive rows ~ 256 entries
  DevBuf<uint8_t> seg_head(ctx, nnz), unit_head(ctx, nnz);
  DevBuf<unsigned long long> cnt(ctx, 1);
  GIFT_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), st));
  k_bmt_flags<<<grid_for(nnz, kBlock), kBlock, 0, st>>>(nnz, key_s.p, pay_s.p, 1, seg_head.p, unit_head.p, cnt.p);
  GIFT_LAUNCH_CHECK(ctx);
  const unsigned long long row_runs = fetch(ctx, cnt.p);
  const double per_run = row_runs ? (double)nnz / (double)row_runs : 1.0;
  int D = (int)(256.0 / per_run + 0.5);
  D = D < 1 ? 1 : (D > 64 ? 64 : D);
  if (D > 1) {
    k_bmt_flags<<<grid_for(nnz, kBlock), kBlock, 0, st>>>(nnz, key_s.p, pay_s.p, D, seg_head.p, unit_head.p,
                                                          nullptr);
    GIFT_LAUNCH_CHECK(ctx);
  }
  // segment starts and unit starts (positions of the flags)
  const int64_t max_seg = std::min<int64_t>(nnz, ntiles * nblocks) + 1;
  DevBuf<int64_t> seg_start(ctx, max_seg), nsel(ctx, 2);
  thrust::counting_iterator<int64_t> it(0);
  GIFT_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, it, seg_head.p, seg_start.p, nsel.p, nnz, st));
  {
    DevBuf<char> t2(ctx, bytes);
    GIFT_CUDA(cub::DeviceSelect::Flagged(t2.p, bytes, it, seg_head.p, seg_start.p, nsel.p, nnz, st));
  }
  const int64_t nseg = fetch(ctx, nsel.p);
  if (nseg > (int64_t)seg_start.n) throw_error(GIFT_ERR_INTERNAL, "bmt: segment buffer overflow");
  // every unit starts at a row run head, so row_runs bounds the unit count
  B.unit_start = static_cast<int64_t*>(csr_alloc(ctx, c, (row_runs + 2) * sizeof(int64_t)));
  GIFT_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, it, unit_head.p, B.unit_start, nsel.p + 1, nnz, st));
  {
    DevBuf<char> t2(ctx, bytes);
    GIFT_CUDA(cub::DeviceSelect::Flagged(t2.p, bytes, it, unit_head.p, B.unit_start, nsel.p + 1, nnz, st));
  }
  ctx->launches += 4;
  const int64_t nunits = fetch(ctx, nsel.p + 1);
  if (nunits > (int64_t)row_runs) throw_error(GIFT_ERR_INTERNAL, "bmt: unit buffer overflow");
  GIFT_CUDA(cudaMemcpyAsync(B.unit_start + nunits, &nnz, sizeof(int64_t), cudaMemcpyHostToDevice, st));
  seg_head.reset();
  unit_head.reset();
  B.seg_code = static_cast<int32_t*>(csr_alloc(ctx, c, (nseg + 1) * sizeof(int32_t)));
  B.seg_unit = static_cast<int64_t*>(csr_alloc(ctx, c, (nseg + 1) * sizeof(int64_t)));
  B.tile_seg = static_cast<int64_t*>(csr_alloc(ctx, c, (ntiles + 1) * sizeof(int64_t)));
  DevBuf<uint32_t> seg_tile(ctx, nseg + 1);
  k_bmt_segs<<<grid_for(nseg + 1, kBlock), kBlock, 0, st>>>(nseg, seg_start.p, key_s.p, nnz, bb, B.unit_start,
                                                            nunits, B.seg_code, B.seg_unit, seg_tile.p);
  GIFT_LAUNCH_CHECK(ctx);
  k_bmt_tile_ptr<<<grid_for(nseg + 1, kBlock), kBlock, 0, st>>>(nseg, seg_tile.p, ntiles, B.tile_seg);
  GIFT_LAUNCH_CHECK(ctx);
  B.idx = static_cast<uint32_t*>(csr_alloc(ctx, c, nnz * sizeof(uint32_t)));
  B.w = static_cast<float*>(csr_alloc(ctx, c, nnz * sizeof(float)));
  k_bmt_split<<<grid_for(nnz, kBlock), kBlock, 0, st>>>(nnz, pay_s.p, B.idx, B.w);
  GIFT_LAUNCH_CHECK(ctx);
  GIFT_CUDA(cudaStreamSynchronize(st));
  B.ntiles = ntiles;
  B.nseg = nseg;
  B.nunits = nunits;
  return true;
}

}  // namespace

const float* csr_w32_public(Ctx* ctx, Csr* c);

bool bmt_hop(Ctx* ctx, Csr* c, const HopArgs& a, int fin, int fout) {
  if (env_int("GIFT_BMT", 1) == 0 || !c->sorted_rows) return false;
  if (c->n < env_int("GIFT_BMT_MIN_ROWS", 262144) || c->mean_row < env_int("GIFT_BMT_MIN_MEAN", 96)) return false;
  if (a.row_begin != 0 || a.n != c->n || a.part_in || a.part_out) return false;
  Csr::Bmt& B = c->bmt;
  if (!B.ready) {
    B.ready = true;
    B.ok = bmt_build(ctx, c, csr_w32_public(ctx, c));
  }
  if (!B.ok) return false;
  BmtArgs b{c->n, B.tile_seg, B.seg_code, B.seg_unit, B.unit_start, B.idx, B.w};
  switch (fin) {
    case 1: launch_bmt_out<1>(ctx, a, b, B.ntiles, fout); break;
    case 2: launch_bmt_out<2>(ctx, a, b, B.ntiles, fout); break;
    default: launch_bmt_out<4>(ctx, a, b, B.ntiles, fout); break;
  }
  return true;
}

}  // namespace gift
