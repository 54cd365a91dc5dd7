// hf.cu -- implicit clique term for high-fanout nets (opt-in extension).
//
// The reference skips every net with more pins than max_clique_pins
// (graph.py:136-138); it has no star or implicit model (SURVEY.md Appendix
// B.1).  A net e with m pins contributes, in the clique model,
//     A_e = (2/m) (b b^T - diag(b o b)),   b_i = multiplicity of cell i in e
// (pairs p < q of distinct cells, weight 2/m each, symmetrised).  Applied to a
// signal z it costs O(m), not O(m^2):
//     (A_e z)_i = (2/m) b_i (t_e - b_i z_i),   t_e = sum over pins z[cell(p)],
//     d_i      += (2/m) b_i (m - b_i).
// This file keeps the nets above the cap as that implicit term next to the
// explicit (capped) CSR, so A = A_cap + sum_e A_e equals the UNCAPPED clique
// graph in exact arithmetic (checked against the uncapped oracle).  Every
// reduction has a fixed order (block trees per net, per-cell sums over the
// cell's occurrences in net order): results are deterministic.
//
// Layout (Csr::Hf): the selected nets' pin table (net_start / pin_cell), 2/m
// per net, and the pin occurrences grouped by cell -- cells ascending, a
// cell's occurrences in net order -- with the net and the multiplicity b of
// each occurrence.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "common.cuh"
#include "hop.cuh"

namespace gift {

const double* csr_degrees(Ctx* ctx, Csr* c);

namespace {

constexpr int kBlock = 256;
constexpr int kNetBlock = 256;

__global__ void k_hf_flags(int64_t n_nets, const int64_t* __restrict__ net_start, int64_t cap, int64_t upto,
                           uint8_t* __restrict__ flag, int64_t* __restrict__ cnt) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_nets; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = net_start[e + 1] - net_start[e];
    const bool hf = m >= 2 && m > cap && (upto < 0 || m <= upto);
    flag[e] = hf;
    cnt[e] = hf ? m : 0;
  }
}

// pins of the selected nets, and 2/m per net (the reference's IEEE 2.0/m, graph.py:149)
__global__ void k_hf_gather(int64_t nh, const int64_t* __restrict__ ids, const int64_t* __restrict__ net_start,
                            const int32_t* __restrict__ pin_cell, const int64_t* __restrict__ hstart,
                            int32_t* __restrict__ hpin, double* __restrict__ coef64, float* __restrict__ coef32,
                            int32_t* __restrict__ pin_net) {
  for (int64_t h = blockIdx.x; h < nh; h += gridDim.x) {
    const int64_t e = ids[h], a = net_start[e], m = net_start[e + 1] - a, o = hstart[h];
    for (int64_t p = threadIdx.x; p < m; p += blockDim.x) {
      hpin[o + p] = pin_cell[a + p];
      pin_net[o + p] = (int32_t)h;
    }
    if (threadIdx.x == 0) {
      const double cf = __ddiv_rn(2.0, (double)m);
      coef64[h] = cf;
      coef32[h] = (float)cf;
    }
  }
}

// multiplicity of each pin's cell inside its net (O(m^2) per net, shared-memory staged)
__global__ void k_hf_mult(int64_t nh, const int64_t* __restrict__ hstart, const int32_t* __restrict__ hpin,
                          int32_t* __restrict__ mult) {
  __shared__ int32_t sc[4096];
  for (int64_t h = blockIdx.x; h < nh; h += gridDim.x) {
    const int64_t a = hstart[h], m = hstart[h + 1] - a;
    const bool staged = m <= 4096;
    __syncthreads();
    if (staged)
      for (int64_t p = threadIdx.x; p < m; p += blockDim.x) sc[p] = hpin[a + p];
    __syncthreads();
    const int32_t* cells = staged ? sc : hpin + a;
    for (int64_t p = threadIdx.x; p < m; p += blockDim.x) {
      const int32_t c = cells[p];
      int b = 0;
      for (int64_t q = 0; q < m; ++q) b += cells[q] == c;
      mult[a + p] = b;
    }
  }
}

__global__ void k_hf_occ(int64_t P, const int32_t* __restrict__ perm_pin, const int32_t* __restrict__ pin_net,
                         const int32_t* __restrict__ mult, int32_t* __restrict__ occ_net, float* __restrict__ b32,
                         double* __restrict__ b64) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < P; k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p = perm_pin[k];
    occ_net[k] = pin_net[p];
    b32[k] = (float)mult[p];
    b64[k] = (double)mult[p];
  }
}

__global__ void k_iota32(int64_t n, int32_t* __restrict__ p) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = (int32_t)i;
}

__global__ void k_hf_heads(int64_t P, const int32_t* __restrict__ cell_s, uint8_t* __restrict__ head) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < P; k += (int64_t)gridDim.x * blockDim.x)
    head[k] = k == 0 || cell_s[k] != cell_s[k - 1];
}

__global__ void k_hf_cells(int64_t nc, int64_t P, const int64_t* __restrict__ occ_ptr, const int32_t* __restrict__ cell_s,
                           int32_t* __restrict__ cell, int64_t* __restrict__ occ_ptr_out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= nc; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < nc) {
      cell[i] = cell_s[occ_ptr[i]];
      occ_ptr_out[i] = occ_ptr[i];
    } else {
      occ_ptr_out[nc] = P;
    }
  }
}

// d_i += sum over the cell's occurrences of (2/m)(m - b), in net order
__global__ void k_hf_degrees(int64_t nc, const int32_t* __restrict__ cell, const int64_t* __restrict__ occ_ptr,
                             const int32_t* __restrict__ occ_net, const double* __restrict__ b64,
                             const double* __restrict__ coef64, const int64_t* __restrict__ hstart,
                             double* __restrict__ deg) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nc; i += (int64_t)gridDim.x * blockDim.x) {
    double d = 0.0;
    for (int64_t k = occ_ptr[i]; k < occ_ptr[i + 1]; ++k) {
      const int32_t h = occ_net[k];
      const double m = (double)(hstart[h + 1] - hstart[h]);
      d = __dadd_rn(d, __dmul_rn(coef64[h], __dadd_rn(m, -b64[k])));
    }
    deg[cell[i]] = __dadd_rn(deg[cell[i]], d);
  }
}

// ---- per hop ---------------------------------------------------------------
// t_e = sum over the net's pins of u[cell(p)] (F floats per row), fp64
// accumulation, fixed block tree.  u = z (fp32 hop) or s o x (fp64 hop, S set).
template <typename T, int F, bool S>
__global__ void __launch_bounds__(kNetBlock) k_hf_tsum(int64_t nh, const int64_t* __restrict__ hstart,
                                                       const int32_t* __restrict__ hpin, const T* __restrict__ z,
                                                       int64_t ld, int64_t c0, const double* __restrict__ s,
                                                       double* __restrict__ t) {
  __shared__ double red[kNetBlock / 32][F];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int64_t h = blockIdx.x; h < nh; h += gridDim.x) {
    double acc[F];
#pragma unroll
    for (int f = 0; f < F; ++f) acc[f] = 0.0;
    for (int64_t p = hstart[h] + threadIdx.x; p < hstart[h + 1]; p += kNetBlock) {
      const int64_t c = hpin[p];
      const double sc = S ? s[c] : 1.0;
#pragma unroll
      for (int f = 0; f < F; ++f) acc[f] += sc * (double)z[c * ld + c0 + f];
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
#pragma unroll
      for (int f = 0; f < F; ++f) acc[f] += __shfl_xor_sync(0xffffffffu, acc[f], off);
    __syncthreads();
    if (lane == 0)
#pragma unroll
      for (int f = 0; f < F; ++f) red[wid][f] = acc[f];
    __syncthreads();
    if (threadIdx.x < F) {
      double v = 0.0;
      for (int w = 0; w < kNetBlock / 32; ++w) v += red[w][threadIdx.x];
      t[h * F + threadIdx.x] = v;
    }
  }
}

// the same sums with one WARP per net (graphs whose implicit nets are many and
// short -- the factored clique model keeps every net above a few pins
// implicit): lanes stride the net's pins, fixed xor-butterfly, lane f writes
template <typename T, int F, bool S>
__global__ void __launch_bounds__(kBlock) k_hf_tsum_warp(int64_t nh, const int64_t* __restrict__ hstart,
                                                         const int32_t* __restrict__ hpin, const T* __restrict__ z,
                                                         int64_t ld, int64_t c0, const double* __restrict__ s,
                                                         double* __restrict__ t) {
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t h = warp0; h < nh; h += nwarps) {
    double acc[F];
#pragma unroll
    for (int f = 0; f < F; ++f) acc[f] = 0.0;
    const int64_t a = hstart[h], b = hstart[h + 1];
    for (int64_t p = a + lane; p < b; p += 32) {
      const int64_t c = hpin[p];
      const double sc = S ? s[c] : 1.0;
#pragma unroll
      for (int f = 0; f < F; ++f) acc[f] += sc * (double)z[c * ld + c0 + f];
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
#pragma unroll
      for (int f = 0; f < F; ++f) acc[f] += __shfl_xor_sync(0xffffffffu, acc[f], off);
#pragma unroll
    for (int f = 0; f < F; ++f)
      if (lane == f) t[h * F + f] = acc[f];
  }
}

// out[cell] (F values) = sum over occurrences of (2/m)(t_e - b u_cell), in net order
template <typename T, int F, bool S>
__global__ void k_hf_apply(int64_t nc, const int32_t* __restrict__ cell, const int64_t* __restrict__ occ_ptr,
                           const int32_t* __restrict__ occ_net, const double* __restrict__ b64,
                           const double* __restrict__ coef64, const double* __restrict__ t, const T* __restrict__ z,
                           int64_t ld, int64_t c0, const double* __restrict__ s, T* __restrict__ out, int64_t ldo) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nc; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = cell[i];
    const double sc = S ? s[c] : 1.0;
    double u[F], acc[F];
#pragma unroll
    for (int f = 0; f < F; ++f) {
      u[f] = sc * (double)z[c * ld + c0 + f];
      acc[f] = 0.0;
    }
    for (int64_t k = occ_ptr[i]; k < occ_ptr[i + 1]; ++k) {
      const int32_t h = occ_net[k];
      const double cf = coef64[h], b = b64[k];
#pragma unroll
      for (int f = 0; f < F; ++f) acc[f] += cf * (t[h * F + f] - b * u[f]);
    }
#pragma unroll
    for (int f = 0; f < F; ++f) out[c * ldo + f] = (T)acc[f];
  }
}

// ---- fp32 hop of the FACTORED clique model ---------------------------------
// When every net above a few pins is implicit the stored matrix is tiny (rows
// of ~5 entries) and the hop is two kernels over O(pins) data:
//   k_fact_tsum: t'_e = (2/m) * sum of the net's pins' signal rows, 8 lanes
//                per net (fp64, fixed butterfly);
//   k_fact_hop : one thread per row: the row's few stored entries (fp32),
//                then sum over its occurrences in implicit nets of t'_e, in
//                net order, minus D_i z_i with D_i = sum (2/m) b over those
//                occurrences (a per-row constant, computed at attach) -- the
//                same sum of (2/m)(t_e - b z_i), but one 32-byte gather per
//                occurrence and nothing else; fp64 (t_e is ~m signal values:
//                rounding it to fp32 would cost the row sum several ulps);
//                then the shared fused epilogue (hop.cuh).
// Fixed orders everywhere: deterministic.
struct FactArgs {
  int64_t nets;
  const int64_t* net_start;
  const int32_t* pin_cell;
  double* t;  // [nets, F] (2/m) * net sums
  const int32_t* row_occ;
  const int32_t* occ_net;
  const double* row_d;  // [n] D_i
  const double* coef;
  const int2* cw;       // [nnz] stored entries as (column, fp32 weight bits): one 8-byte load each
};

template <int F>
__global__ void __launch_bounds__(kBlock) k_fact_tsum(FactArgs h, const float* __restrict__ z) {
  constexpr int G = 8;
  const int lane = threadIdx.x & 31, sub = lane & (G - 1);
  const unsigned gmask = 0xffu << (lane & ~(G - 1));
  const uint64_t pol_z = policy_evict_last();
  const int64_t g0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
  const int64_t ng = ((int64_t)gridDim.x * blockDim.x) / G;
  for (int64_t e = g0; e < h.nets; e += ng) {
    double acc[F];
#pragma unroll
    for (int f = 0; f < F; ++f) acc[f] = 0.0;
    const int64_t a = h.net_start[e], b = h.net_start[e + 1];
    int64_t p = a + sub;
    for (; p + 3 * G < b; p += 4 * G) {  // four gathers in flight per lane (same summation order)
      const int c0 = h.pin_cell[p], c1 = h.pin_cell[p + G], c2 = h.pin_cell[p + 2 * G], c3 = h.pin_cell[p + 3 * G];
      const VecF<F> q0 = ld_z<F>(z + (int64_t)c0 * F, pol_z), q1 = ld_z<F>(z + (int64_t)c1 * F, pol_z);
      const VecF<F> q2 = ld_z<F>(z + (int64_t)c2 * F, pol_z), q3 = ld_z<F>(z + (int64_t)c3 * F, pol_z);
#pragma unroll
      for (int f = 0; f < F; ++f) acc[f] = (((acc[f] + (double)q0.v[f]) + (double)q1.v[f]) + (double)q2.v[f]) + (double)q3.v[f];
    }
    for (; p < b; p += G) {
      const VecF<F> zq = ld_z<F>(z + (int64_t)h.pin_cell[p] * F, pol_z);
#pragma unroll
      for (int f = 0; f < F; ++f) acc[f] += (double)zq.v[f];
    }
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1)
#pragma unroll
      for (int f = 0; f < F; ++f) acc[f] += __shfl_xor_sync(gmask, acc[f], off, G);
    if (sub == 0)
#pragma unroll
      for (int f = 0; f < F; ++f) h.t[e * F + f] = h.coef[e] * acc[f];
  }
}

template <int F, int FOUT>
__global__ void __launch_bounds__(kBlock) k_fact_hop(HopArgs a, FactArgs h) {
  const uint64_t pol_z = policy_evict_last();
  for (int64_t row = a.row_begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; row < a.n;
       row += (int64_t)gridDim.x * blockDim.x) {
    float acc[F];
#pragma unroll
    for (int f = 0; f < F; ++f) acc[f] = 0.f;
    const int64_t k1 = a.rowptr[row + 1];
    for (int64_t k = a.rowptr[row]; k < k1; ++k) {
      const int2 e = __ldg(h.cw + k);
      const VecF<F> zq = ld_z<F>(a.zin + (int64_t)e.x * F, pol_z);
      const float w = __int_as_float(e.y);
#pragma unroll
      for (int f = 0; f < F; ++f) acc[f] = fmaf(w, zq.v[f], acc[f]);
    }
    const int o1 = h.row_occ[row + 1];
    int o = h.row_occ[row];
    if (o < o1) {
      const VecF<F> zi = ld_z<F>(a.zin + row * F, pol_z);
      double imp[F];
#pragma unroll
      for (int f = 0; f < F; ++f) imp[f] = 0.0;
      for (; o < o1; ++o) {
        const double* tp = h.t + (int64_t)h.occ_net[o] * F;
#pragma unroll
        for (int f = 0; f < F; ++f) imp[f] += tp[f];
      }
      const double d = h.row_d[row];
#pragma unroll
      for (int f = 0; f < F; ++f) imp[f] = fma(-d, (double)zi.v[f], imp[f]);
#pragma unroll
      for (int f = 0; f < F; ++f) acc[f] += (float)imp[f];
    }
    row_epilogue<F, FOUT>(a, row, acc, pol_z);
  }
}

template <int F>
void launch_fact(Ctx* ctx, const HopArgs& a, const FactArgs& h, int fout) {
  cudaStream_t st = ctx->stream;
  k_fact_tsum<F><<<grid_for(h.nets * 8, kBlock, 1LL << 30), kBlock, 0, st>>>(h, a.zin);
  GIFT_LAUNCH_CHECK(ctx);
  const unsigned grid = grid_for(a.n - a.row_begin, kBlock, 1LL << 30);
  switch (fout) {
    case 0: k_fact_hop<F, 0><<<grid, kBlock, 0, st>>>(a, h); break;
    case 1: k_fact_hop<F, 1><<<grid, kBlock, 0, st>>>(a, h); break;
    case 2: k_fact_hop<F, 2><<<grid, kBlock, 0, st>>>(a, h); break;
    default: k_fact_hop<F, 4><<<grid, kBlock, 0, st>>>(a, h); break;
  }
  GIFT_LAUNCH_CHECK(ctx);
}

// stored entries as (column, fp32 weight) pairs (the weights rounded like the hop's w32)
__global__ void k_fact_pack(int64_t nnz, const int32_t* __restrict__ col, const double* __restrict__ v,
                            int2* __restrict__ cw) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x)
    cw[k] = make_int2(col[k], __float_as_int((float)v[k]));
}

// D_i = sum over the row's occurrences of (2/m) b, in net order
__global__ void k_hf_row_d(int64_t n, const int32_t* __restrict__ row_occ, const int32_t* __restrict__ occ_net,
                           const double* __restrict__ b64, const double* __restrict__ coef64,
                           double* __restrict__ row_d) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    double d = 0.0;
    for (int o = row_occ[r]; o < row_occ[r + 1]; ++o) d = fma(coef64[occ_net[o]], b64[o], d);
    row_d[r] = d;
  }
}

__global__ void k_hf_row_counts(int64_t nc, const int32_t* __restrict__ cell, const int64_t* __restrict__ occ_ptr,
                                int32_t* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nc; i += (int64_t)gridDim.x * blockDim.x)
    cnt[cell[i]] = (int32_t)(occ_ptr[i + 1] - occ_ptr[i]);
}

template <typename T, bool S>
void hf_apply_t(Ctx* ctx, const Csr* c, int F, const T* z, int64_t ld, int64_t c0, const double* s, T* out,
                int64_t ldo) {
  const Csr::Hf& H = c->hf;
  if (!H.nets) return;
  cudaStream_t st = ctx->stream;
  double* t = static_cast<double*>(H.tbuf);
  const unsigned gn = (unsigned)std::min<int64_t>(H.nets, 65535);
  const unsigned gc = grid_for(H.cells, kBlock);
  // one warp per net unless the nets are few and long (a fixed choice per
  // graph: the two kernels sum in different orders)
  const bool warp_nets = H.pins < 512 * H.nets;
  const unsigned gw = grid_for(H.nets * 32, kBlock, 1LL << 30);
#define GIFT_HF_CASE(FF)                                                                                         \
  if (warp_nets)                                                                                                   \
    k_hf_tsum_warp<T, FF, S><<<gw, kBlock, 0, st>>>(H.nets, H.net_start, H.pin_cell, z, ld, c0, s, t);            \
  else                                                                                                             \
    k_hf_tsum<T, FF, S><<<gn, kNetBlock, 0, st>>>(H.nets, H.net_start, H.pin_cell, z, ld, c0, s, t);              \
  k_hf_apply<T, FF, S><<<gc, kBlock, 0, st>>>(H.cells, H.cell, H.occ_ptr, H.occ_net, H.occ_b, H.coef, t, z, ld, c0, \
                                              s, out, ldo);
  switch (F) {
    case 1: GIFT_HF_CASE(1) break;
    case 2: GIFT_HF_CASE(2) break;
    case 3: GIFT_HF_CASE(3) break;
    default: GIFT_HF_CASE(4) break;
  }
#undef GIFT_HF_CASE
  GIFT_LAUNCH_CHECK(ctx);
  ctx->launches++;
}

}  // namespace

// Attach the implicit term of the nets with more than `cap` pins -- and, when
// upto >= 0, at most `upto` pins (larger ones stay dropped, like the
// reference's max_clique_pins skip) -- to c, a graph built from the same
// netlist with that cap.  Must run before any derived state (degrees,
// s_sigma) exists: those then include the term.
int64_t csr_attach_high_fanout(Ctx* ctx, Csr* c, int64_t n_nets, const int64_t* d_net_start,
                               const int32_t* d_pin_cell, int64_t cap, int64_t upto) {
  if (cap < 0) throw_error(GIFT_ERR_VALUE, "high-fanout term needs a cap (max_clique_pins >= 0)");
  if (c->hf.nets) throw_error(GIFT_ERR_VALUE, "graph already has a high-fanout term");
  if (c->degrees || !c->s64.empty() || c->bmt.ready || c->bmt_wide.ready)
    throw_error(GIFT_ERR_VALUE, "attach the high-fanout term before the graph is used");
  if (n_nets <= 0) return 0;
  cudaStream_t st = ctx->stream;
  DevBuf<uint8_t> flag(ctx, n_nets);
  DevBuf<int64_t> cnt(ctx, n_nets + 1), ids(ctx, n_nets + 1), nsel(ctx, 1);
  k_hf_flags<<<grid_for(n_nets, kBlock), kBlock, 0, st>>>(n_nets, d_net_start, cap, upto, flag.p, cnt.p);
  GIFT_LAUNCH_CHECK(ctx);
  {
    thrust::counting_iterator<int64_t> it(0);
    size_t bytes = 0;
    GIFT_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, it, flag.p, ids.p, nsel.p, n_nets, st));
    DevBuf<char> tmp(ctx, bytes);
    GIFT_CUDA(cub::DeviceSelect::Flagged(tmp.p, bytes, it, flag.p, ids.p, nsel.p, n_nets, st));
    ctx->launches += 2;
  }
  int64_t nh = 0;
  GIFT_CUDA(cudaMemcpyAsync(&nh, nsel.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GIFT_CUDA(cudaStreamSynchronize(st));
  if (nh == 0) return 0;
  if (nh >= (1LL << 31)) throw_error(GIFT_ERR_TOO_LARGE, "too many high-fanout nets");
  Csr::Hf H;
  // per selected net: pin count -> offsets
  DevBuf<int64_t> hcnt(ctx, nh + 1);
  {
    DevBuf<int64_t> cnt_sel(ctx, nh + 1);
    size_t bytes = 0;
    GIFT_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, cnt.p, flag.p, cnt_sel.p, nsel.p, n_nets, st));
    DevBuf<char> tmp(ctx, bytes);
    GIFT_CUDA(cub::DeviceSelect::Flagged(tmp.p, bytes, cnt.p, flag.p, cnt_sel.p, nsel.p, n_nets, st));
    GIFT_CUDA(cudaMemsetAsync(cnt_sel.p + nh, 0, sizeof(int64_t), st));
    H.net_start = static_cast<int64_t*>(csr_alloc(ctx, c, (nh + 1) * sizeof(int64_t)));
    bytes = 0;
    GIFT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt_sel.p, H.net_start, nh + 1, st));
    DevBuf<char> tmp2(ctx, bytes);
    GIFT_CUDA(cub::DeviceScan::ExclusiveSum(tmp2.p, bytes, cnt_sel.p, H.net_start, nh + 1, st));
    ctx->launches += 4;
  }
  int64_t P = 0;
  GIFT_CUDA(cudaMemcpyAsync(&P, H.net_start + nh, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GIFT_CUDA(cudaStreamSynchronize(st));
  if (P >= (1LL << 31)) throw_error(GIFT_ERR_TOO_LARGE, "too many high-fanout pins");
  H.pin_cell = static_cast<int32_t*>(csr_alloc(ctx, c, P * sizeof(int32_t)));
  H.coef = static_cast<double*>(csr_alloc(ctx, c, nh * sizeof(double)));
  float* coef32 = static_cast<float*>(csr_alloc(ctx, c, nh * sizeof(float)));
  DevBuf<int32_t> pin_net(ctx, P), mult(ctx, P);
  k_hf_gather<<<(unsigned)std::min<int64_t>(nh, 65535), kBlock, 0, st>>>(nh, ids.p, d_net_start, d_pin_cell, H.net_start,
                                                                          H.pin_cell, H.coef, coef32, pin_net.p);
  GIFT_LAUNCH_CHECK(ctx);
  k_hf_mult<<<(unsigned)std::min<int64_t>(nh, 65535), kBlock, 0, st>>>(nh, H.net_start, H.pin_cell, mult.p);
  GIFT_LAUNCH_CHECK(ctx);
  // occurrences grouped by cell (stable: net order inside a cell)
  DevBuf<int32_t> cell_s(ctx, P), perm(ctx, P);
  {
    DevBuf<int32_t> iota(ctx, P);
    k_iota32<<<grid_for(P, kBlock), kBlock, 0, st>>>(P, iota.p);
    GIFT_LAUNCH_CHECK(ctx);
    const int bits = bit_length((uint64_t)(c->n > 1 ? c->n - 1 : 1));
    size_t bytes = 0;
    GIFT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, H.pin_cell, cell_s.p, iota.p, perm.p, P, 0, bits, st));
    DevBuf<char> tmp(ctx, bytes);
    GIFT_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, H.pin_cell, cell_s.p, iota.p, perm.p, P, 0, bits, st));
    ctx->launches += 4;
  }
  H.occ_net = static_cast<int32_t*>(csr_alloc(ctx, c, P * sizeof(int32_t)));
  H.occ_b = static_cast<double*>(csr_alloc(ctx, c, P * sizeof(double)));
  float* b32 = static_cast<float*>(csr_alloc(ctx, c, P * sizeof(float)));
  k_hf_occ<<<grid_for(P, kBlock), kBlock, 0, st>>>(P, perm.p, pin_net.p, mult.p, H.occ_net, b32, H.occ_b);
  GIFT_LAUNCH_CHECK(ctx);
  DevBuf<uint8_t> head(ctx, P);
  k_hf_heads<<<grid_for(P, kBlock), kBlock, 0, st>>>(P, cell_s.p, head.p);
  GIFT_LAUNCH_CHECK(ctx);
  DevBuf<int64_t> starts(ctx, P + 1);
  {
    thrust::counting_iterator<int64_t> it(0);
    size_t bytes = 0;
    GIFT_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, it, head.p, starts.p, nsel.p, P, st));
    DevBuf<char> tmp(ctx, bytes);
    GIFT_CUDA(cub::DeviceSelect::Flagged(tmp.p, bytes, it, head.p, starts.p, nsel.p, P, st));
    ctx->launches += 2;
  }
  int64_t nc = 0;
  GIFT_CUDA(cudaMemcpyAsync(&nc, nsel.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GIFT_CUDA(cudaStreamSynchronize(st));
  H.cell = static_cast<int32_t*>(csr_alloc(ctx, c, (nc + 1) * sizeof(int32_t)));
  H.occ_ptr = static_cast<int64_t*>(csr_alloc(ctx, c, (nc + 1) * sizeof(int64_t)));
  k_hf_cells<<<grid_for(nc + 1, kBlock), kBlock, 0, st>>>(nc, P, starts.p, cell_s.p, H.cell, H.occ_ptr);
  GIFT_LAUNCH_CHECK(ctx);
  H.tbuf = csr_alloc(ctx, c, nh * 4 * sizeof(double));
  H.coef32 = coef32;
  H.occ_b32 = b32;
  {  // occurrence range of every row (occurrences are grouped by cell, cells ascending)
    DevBuf<int32_t> cnt(ctx, c->n + 1);
    GIFT_CUDA(cudaMemsetAsync(cnt.p, 0, (c->n + 1) * sizeof(int32_t), st));
    k_hf_row_counts<<<grid_for(nc, kBlock), kBlock, 0, st>>>(nc, H.cell, H.occ_ptr, cnt.p);
    GIFT_LAUNCH_CHECK(ctx);
    H.row_occ = static_cast<int32_t*>(csr_alloc(ctx, c, (c->n + 1) * sizeof(int32_t)));
    size_t bytes = 0;
    GIFT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt.p, H.row_occ, c->n + 1, st));
    DevBuf<char> tmp(ctx, bytes);
    GIFT_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, cnt.p, H.row_occ, c->n + 1, st));
    ctx->launches += 2;
    if (c->nnz <= 64 * c->n) {  // short stored rows: the factored hop's (column, weight) pairs
      H.cw = csr_alloc(ctx, c, (c->nnz > 0 ? c->nnz : 1) * sizeof(int2));
      if (c->nnz > 0) {
        k_fact_pack<<<grid_for(c->nnz, kBlock), kBlock, 0, st>>>(c->nnz, c->indices, c->values, static_cast<int2*>(H.cw));
        GIFT_LAUNCH_CHECK(ctx);
      }
    }
    H.row_d = static_cast<double*>(csr_alloc(ctx, c, (c->n + 1) * sizeof(double)));
    k_hf_row_d<<<grid_for(c->n, kBlock), kBlock, 0, st>>>(c->n, H.row_occ, H.occ_net, H.occ_b, H.coef, H.row_d);
    GIFT_LAUNCH_CHECK(ctx);
    GIFT_CUDA(cudaStreamSynchronize(st));
  }
  H.nets = nh;
  H.pins = P;
  H.cells = nc;
  c->hf = H;
  return nh;
}

// full degrees = the explicit graph's (numpy order) + the implicit term's
void hf_add_degrees(Ctx* ctx, const Csr* c, double* deg) {
  const Csr::Hf& H = c->hf;
  if (!H.nets) return;
  k_hf_degrees<<<grid_for(H.cells, kBlock), kBlock, 0, ctx->stream>>>(H.cells, H.cell, H.occ_ptr, H.occ_net, H.occ_b,
                                                                      H.coef, H.net_start, deg);
  GIFT_LAUNCH_CHECK(ctx);
}

// out[cell, :F] = (A_hf z)[cell] for the cells with high-fanout pins (fp32
// hop: z has F floats per row, ld = F); other rows of out are left untouched
void hf_apply_f32(Ctx* ctx, const Csr* c, int F, const float* z, float* out) {
  hf_apply_t<float, false>(ctx, c, F, z, F, 0, nullptr, out, F);
}

// The whole fp32 hop (explicit rows + implicit nets + epilogue) as the two
// factored-model kernels; false when the graph is not a factored one (its
// stored rows are long: the tiled / row kernels serve those with part_in)
bool fact_hop_applies(const Ctx* ctx, const Csr* c, const HopArgs& a, int fin) {
  const Csr::Hf& H = c->hf;
  if (!H.nets || !H.row_occ || !H.cw || a.part_in || a.part_out || a.row_list) return false;
  if (fin != 1 && fin != 2 && fin != 4) return false;
  // stored rows long enough for the tiled / row kernels (option "tiled_min_mean",
  // default 32): not the factored regime, the term enters those as partial sums
  return c->mean_row < (double)ctx->opt.tiled_min_mean;
}


bool fact_hop_f32(Ctx* ctx, Csr* c, const HopArgs& a, int fin, int fout) {
  const Csr::Hf& H = c->hf;
  if (!fact_hop_applies(ctx, c, a, fin)) return false;
  FactArgs h{H.nets, H.net_start, H.pin_cell, static_cast<double*>(H.tbuf), H.row_occ, H.occ_net, H.row_d, H.coef,
             static_cast<const int2*>(H.cw)};
  switch (fin) {
    case 1: launch_fact<1>(ctx, a, h, fout); break;
    case 2: launch_fact<2>(ctx, a, h, fout); break;
    case 4: launch_fact<4>(ctx, a, h, fout); break;
    default: return false;
  }
  return true;
}

// out[cell, :nc] = (A_hf (s o x))[cell] over columns c0 .. c0 + nc of x
// (fp64 hop; s = nullptr for the plain adjacency)
void hf_apply_f64(Ctx* ctx, const Csr* c, int nc, const double* x, int64_t ld, int64_t c0, const double* s,
                  double* out) {
  if (s)
    hf_apply_t<double, true>(ctx, c, nc, x, ld, c0, s, out, 4);
  else
    hf_apply_t<double, false>(ctx, c, nc, x, ld, c0, s, out, 4);
}

}  // namespace gift
