// metrics.cu -- the placement-quality consumers of the filter output, on the
// device, reusing the resident CSR and pin table:
//
//   quadratic_wirelength(adj, g)   metrics.py:63-74   S = 1/2 sum_k w_k |g_r - g_c|^2
//   laplacian(adj)                 graph.py:161-164   L = D - A (exact: negation, d - 0)
//   rayleigh_smoothness(L, col)    metrics.py:77-92   R = c^T L c / c^T c, c mean-centred
//   hpwl(design, g)                metrics.py:95-112  sum over nets of (max - min) x and y
//
// All sums are fp64 with a fixed reduction tree (per-row or per-net sequential
// terms, block partials in a fixed grid, partials summed in order), so results
// are deterministic run to run; they match numpy to ~1e-15 relative (numpy's
// own order is pairwise / BLAS-dependent and is not reproduced here).
#include <cub/cub.cuh>

#include <cmath>
#include <cstring>

#include "common.cuh"

namespace gift {

namespace {

constexpr int kBlock = 256;
constexpr int kGrid = 1024;  // fixed -> deterministic partition of every reduction

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double sh[kBlock / 32];
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < kBlock / 32; ++i) t += sh[i];
  return t;
}

// S partials: thread-per-row sequential over the row's entries
__global__ void k_qwl(int64_t n, const int64_t* __restrict__ indptr, const int32_t* __restrict__ idx,
                      const double* __restrict__ val, const double* __restrict__ g, double* __restrict__ part) {
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double xi = g[2 * i], yi = g[2 * i + 1];
    double r = 0.0;
    for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k) {
      const int64_t j = idx[k];
      const double dx = xi - g[2 * j], dy = yi - g[2 * j + 1];
      r += val[k] * (dx * dx + dy * dy);
    }
    acc += r;
  }
  const double t = block_sum(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
}

__global__ void k_sum_partials(int m, const double* __restrict__ part, double scale, double* __restrict__ out) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < m; ++i) t += part[i];
    *out = t * scale;
  }
}

// plain deterministic sum / dot with an optional shift: sum_i (x_i - sx) * (y_i - sy)
__global__ void k_dot(int64_t n, const double* __restrict__ x, const double* __restrict__ y, const double* shift,
                      double* __restrict__ part) {
  const double s = shift ? *shift : 0.0;
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    acc += (x[i] - s) * (y ? (y[i] - s) : 1.0);
  const double t = block_sum(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
}

__global__ void k_center(int64_t n, const double* __restrict__ x, const double* __restrict__ sum,
                         double* __restrict__ out, double* __restrict__ mean_out) {
  const double mean = *sum / (double)n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = x[i] - mean;
  if (blockIdx.x == 0 && threadIdx.x == 0 && mean_out) *mean_out = mean;
}

// HPWL partials: thread per net, min/max over its pins (exact), sum in fixed order
__global__ void k_hpwl(int64_t n_nets, const int64_t* __restrict__ net_start, const int32_t* __restrict__ pin_cell,
                       const double* __restrict__ pdx, const double* __restrict__ pdy, const double* __restrict__ g,
                       double* __restrict__ part) {
  double acc = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_nets; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = net_start[e], b = net_start[e + 1];
    if (a == b) continue;
    double xlo = INFINITY, xhi = -INFINITY, ylo = INFINITY, yhi = -INFINITY;
    for (int64_t p = a; p < b; ++p) {
      const int64_t c = pin_cell[p];
      const double x = g[2 * c] + (pdx ? pdx[p] : 0.0), y = g[2 * c + 1] + (pdy ? pdy[p] : 0.0);
      xlo = fmin(xlo, x); xhi = fmax(xhi, x); ylo = fmin(ylo, y); yhi = fmax(yhi, y);
    }
    acc += (xhi - xlo) + (yhi - ylo);
  }
  const double t = block_sum(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
}

// L = D - A: diagonal d_i - a_ii (or d_i) at its sorted position, dropped when 0;
// off-diagonals -a_ij (csr_minus_csr keeps nonzero results only)
__global__ void k_lap_count(int64_t n, const int64_t* __restrict__ indptr, const int32_t* __restrict__ idx,
                            const double* __restrict__ val, const double* __restrict__ deg, int64_t* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x) {
    if (i == n) { cnt[n] = 0; continue; }
    int64_t c = 0;
    bool diag = false;
    for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k) {
      if (idx[k] == i) { diag = true; c += (deg[i] - val[k]) != 0.0; }
      else c += (-val[k]) != 0.0;
    }
    if (!diag) c += deg[i] != 0.0;
    cnt[i] = c;
  }
}

__global__ void k_lap_fill(int64_t n, const int64_t* __restrict__ indptr, const int32_t* __restrict__ idx,
                           const double* __restrict__ val, const double* __restrict__ deg,
                           const int64_t* __restrict__ optr, int32_t* __restrict__ oidx, double* __restrict__ oval) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t o = optr[i];
    bool diag_done = false;
    for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k) {
      const int64_t j = idx[k];
      if (!diag_done && j > i) {
        if (deg[i] != 0.0) { oidx[o] = (int32_t)i; oval[o] = deg[i]; ++o; }
        diag_done = true;
      }
      double v;
      if (j == i) { v = deg[i] - val[k]; diag_done = true; }
      else v = -val[k];
      if (v != 0.0) { oidx[o] = (int32_t)j; oval[o] = v; ++o; }
    }
    if (!diag_done && deg[i] != 0.0) { oidx[o] = (int32_t)i; oval[o] = deg[i]; }
  }
}

double fetch_d(Ctx* ctx, const double* d) {
  double h;
  GIFT_CUDA(cudaMemcpyAsync(&h, d, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  GIFT_CUDA(cudaStreamSynchronize(ctx->stream));
  return h;
}

}  // namespace

const double* csr_degrees(Ctx* ctx, Csr* c);

double quadratic_wirelength(Ctx* ctx, const Csr* c, const double* g) {
  if (c->nnz == 0) return 0.0;
  DevBuf<double> part(ctx, kGrid + 1);
  k_qwl<<<kGrid, kBlock, 0, ctx->stream>>>(c->n, c->indptr, c->indices, c->values, g, part.p);
  GIFT_LAUNCH_CHECK(ctx);
  k_sum_partials<<<1, 32, 0, ctx->stream>>>(kGrid, part.p, 0.5, part.p + kGrid);
  GIFT_LAUNCH_CHECK(ctx);
  return fetch_d(ctx, part.p + kGrid);
}

double hpwl(Ctx* ctx, int64_t n_nets, const int64_t* net_start, const int32_t* pin_cell, const double* pdx,
            const double* pdy, const double* g) {
  if (n_nets == 0) return 0.0;
  DevBuf<double> part(ctx, kGrid + 1);
  k_hpwl<<<kGrid, kBlock, 0, ctx->stream>>>(n_nets, net_start, pin_cell, pdx, pdy, g, part.p);
  GIFT_LAUNCH_CHECK(ctx);
  k_sum_partials<<<1, 32, 0, ctx->stream>>>(kGrid, part.p, 1.0, part.p + kGrid);
  GIFT_LAUNCH_CHECK(ctx);
  return fetch_d(ctx, part.p + kGrid);
}

void csr_matmul(Ctx* ctx, const Csr* c, int64_t ncols, const double* x, double* y);

// returns (numerator, denominator) of the Rayleigh quotient; col is centred first when asked
void rayleigh_parts(Ctx* ctx, const Csr* lap, const double* col, bool center, double* num, double* den) {
  const int64_t n = lap->n;
  DevBuf<double> c(ctx, n + 1), lc(ctx, n + 1), part(ctx, kGrid + 4);
  if (center) {
    k_dot<<<kGrid, kBlock, 0, ctx->stream>>>(n, col, nullptr, nullptr, part.p);
    GIFT_LAUNCH_CHECK(ctx);
    k_sum_partials<<<1, 32, 0, ctx->stream>>>(kGrid, part.p, 1.0, part.p + kGrid);
    GIFT_LAUNCH_CHECK(ctx);
    k_center<<<grid_for(n, kBlock), kBlock, 0, ctx->stream>>>(n, col, part.p + kGrid, c.p, nullptr);
    GIFT_LAUNCH_CHECK(ctx);
  } else {
    GIFT_CUDA(cudaMemcpyAsync(c.p, col, n * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  }
  csr_matmul(ctx, lap, 1, c.p, lc.p);
  k_dot<<<kGrid, kBlock, 0, ctx->stream>>>(n, c.p, lc.p, nullptr, part.p);
  GIFT_LAUNCH_CHECK(ctx);
  k_sum_partials<<<1, 32, 0, ctx->stream>>>(kGrid, part.p, 1.0, part.p + kGrid + 1);
  GIFT_LAUNCH_CHECK(ctx);
  k_dot<<<kGrid, kBlock, 0, ctx->stream>>>(n, c.p, c.p, nullptr, part.p);
  GIFT_LAUNCH_CHECK(ctx);
  k_sum_partials<<<1, 32, 0, ctx->stream>>>(kGrid, part.p, 1.0, part.p + kGrid + 2);
  GIFT_LAUNCH_CHECK(ctx);
  double h[2];
  GIFT_CUDA(cudaMemcpyAsync(h, part.p + kGrid + 1, 2 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  GIFT_CUDA(cudaStreamSynchronize(ctx->stream));
  *num = h[0];
  *den = h[1];
}

Csr* laplacian(Ctx* ctx, Csr* adj) {
  const double* deg = csr_degrees(ctx, adj);
  const int64_t n = adj->n;
  DevBuf<int64_t> cnt(ctx, n + 1);
  Csr* o = new gift_csr();
  o->device = ctx->device;
  o->n = n;
  o->indptr = static_cast<int64_t*>(csr_alloc(ctx, o, (n + 1) * sizeof(int64_t)));
  k_lap_count<<<grid_for(n + 1, kBlock), kBlock, 0, ctx->stream>>>(n, adj->indptr, adj->indices, adj->values, deg,
                                                                   cnt.p);
  GIFT_LAUNCH_CHECK(ctx);
  size_t bytes = 0;
  GIFT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt.p, o->indptr, n + 1, ctx->stream));
  {
    DevBuf<char> tmp(ctx, bytes);
    GIFT_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, cnt.p, o->indptr, n + 1, ctx->stream));
    ctx->launches += 2;
  }
  int64_t nnz = 0;
  GIFT_CUDA(cudaMemcpyAsync(&nnz, o->indptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
  GIFT_CUDA(cudaStreamSynchronize(ctx->stream));
  o->nnz = nnz;
  o->indices = static_cast<int32_t*>(csr_alloc(ctx, o, (nnz > 0 ? nnz : 1) * sizeof(int32_t)));
  o->values = static_cast<double*>(csr_alloc(ctx, o, (nnz > 0 ? nnz : 1) * sizeof(double)));
  o->has_diagonal = true;
  o->mean_row = n > 0 ? (double)nnz / n : 0.0;
  if (n > 0) {
    k_lap_fill<<<grid_for(n, kBlock), kBlock, 0, ctx->stream>>>(n, adj->indptr, adj->indices, adj->values, deg,
                                                                o->indptr, o->indices, o->values);
    GIFT_LAUNCH_CHECK(ctx);
  }
  return o;
}

}  // namespace gift
