// shard.cu -- device-side row sharding of a resident graph.
//
// A rank that holds the full clique graph on its GPU (built there by
// build_clique_graph, graph.py:120-158) cuts out the rows it owns without
// copying the CSR to the host:
//   row_bounds : nnz-balanced contiguous row blocks, r_k = first row whose
//                (indptr[r] + r) reaches k/P of the total (each row counts once,
//                so empty rows still spread) -- shard.py nnz_balanced_bounds;
//   split_rows : rows [r0, r1) -> LOCAL block (columns in [r0, r1), renumbered
//                col - r0: a square block the tiled hop can serve) and GHOST
//                block (the other columns, renumbered n_local + rank of the
//                column in the sorted list of distinct ghost columns).  Entry
//                order inside each row is kept and values are copied bit for
//                bit, so every row's local / ghost partial sums run over the
//                reference's entries in the reference's order.
#include <cub/cub.cuh>

#include "common.cuh"

namespace gift {

Csr* csr_from_arrays(Ctx* ctx, int64_t n_rows, int64_t nnz, const int64_t* d_indptr, const int32_t* d_indices,
                     const double* d_values);

namespace {

constexpr int kBlock = 256;

// bounds[k] = first row r with indptr[r] + r >= (k * total) / P, total = nnz + n
__global__ void k_row_bounds(int64_t n, const int64_t* __restrict__ indptr, int world, int64_t* __restrict__ bounds) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k > world) return;
  if (k == 0) {
    bounds[0] = 0;
    return;
  }
  if (k == world) {
    bounds[world] = n;
    return;
  }
  const int64_t total = indptr[n] + n;
  const int64_t target = (int64_t)(((__int128)k * total) / world);
  int64_t lo = 0, hi = n;  // first r in [0, n] with indptr[r] + r >= target
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (indptr[mid] + mid < target) lo = mid + 1;
    else hi = mid;
  }
  bounds[k] = lo;
}

// per owned row: entries with owned / ghost columns
__global__ void k_split_counts(int64_t r0, int64_t r1, const int64_t* __restrict__ indptr,
                               const int32_t* __restrict__ col, int64_t* __restrict__ nloc,
                               int64_t* __restrict__ ngh) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < r1 - r0; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t l = 0;
    const int64_t a = indptr[r0 + i], b = indptr[r0 + i + 1];
    for (int64_t k = a; k < b; ++k) l += (col[k] >= r0 && col[k] < r1);
    nloc[i] = l;
    ngh[i] = (b - a) - l;
  }
}

// ghost columns of the block (with repeats), in entry order
__global__ void k_ghost_cols(int64_t r0, int64_t r1, const int64_t* __restrict__ indptr, const int32_t* __restrict__ col,
                             const int64_t* __restrict__ gptr, int32_t* __restrict__ gcol) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < r1 - r0; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t o = gptr[i];
    for (int64_t k = indptr[r0 + i]; k < indptr[r0 + i + 1]; ++k)
      if (col[k] < r0 || col[k] >= r1) gcol[o++] = col[k];
  }
}

__global__ void k_split_fill(int64_t r0, int64_t r1, const int64_t* __restrict__ indptr, const int32_t* __restrict__ col,
                             const double* __restrict__ val, const int64_t* __restrict__ lptr,
                             const int64_t* __restrict__ gptr, const int32_t* __restrict__ gids, int64_t ng,
                             int32_t* __restrict__ lcol, double* __restrict__ lval, int32_t* __restrict__ gcol,
                             double* __restrict__ gval) {
  const int64_t nl = r1 - r0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nl; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo_ = lptr[i], go = gptr[i];
    for (int64_t k = indptr[r0 + i]; k < indptr[r0 + i + 1]; ++k) {
      const int32_t c = col[k];
      if (c >= r0 && c < r1) {
        lcol[lo_] = (int32_t)(c - r0);
        lval[lo_++] = val[k];
      } else {
        int64_t lo = 0, hi = ng;  // rank of c among the distinct ghost columns
        while (lo < hi) {
          const int64_t mid = (lo + hi) >> 1;
          if (gids[mid] < c) lo = mid + 1;
          else hi = mid;
        }
        gcol[go] = (int32_t)(nl + lo);
        gval[go++] = val[k];
      }
    }
  }
}

__global__ void k_i32_to_i64(int64_t n, const int32_t* __restrict__ a, int64_t* __restrict__ b) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

void exclusive_scan_i64(Ctx* ctx, const int64_t* in, int64_t* out, int64_t n) {
  size_t bytes = 0;
  GIFT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, ctx->stream));
  DevBuf<char> tmp(ctx, bytes);
  GIFT_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, in, out, n, ctx->stream));
  ctx->launches += 2;
}

}  // namespace

void csr_row_bounds(Ctx* ctx, const Csr* c, int world, int64_t* h_bounds) {
  if (world < 1) throw_error(GIFT_ERR_VALUE, "world size must be >= 1");
  DevBuf<int64_t> b(ctx, world + 1);
  k_row_bounds<<<(world + 1 + 127) / 128, 128, 0, ctx->stream>>>(c->n, c->indptr, world, b.p);
  GIFT_LAUNCH_CHECK(ctx);
  GIFT_CUDA(cudaMemcpyAsync(h_bounds, b.p, (world + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
  GIFT_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int k = 1; k <= world; ++k)
    if (h_bounds[k] < h_bounds[k - 1]) h_bounds[k] = h_bounds[k - 1];  // monotone (as np.maximum.accumulate)
}

void csr_split_rows(Ctx* ctx, const Csr* c, int64_t r0, int64_t r1, Csr** local, Csr** ghost) {
  if (r0 < 0 || r1 > c->n || r0 > r1) throw_error(GIFT_ERR_VALUE, "bad row range");
  if (!c->square) throw_error(GIFT_ERR_VALUE, "split_rows needs a square (full) graph");
  cudaStream_t st = ctx->stream;
  const int64_t nl = r1 - r0;
  const unsigned grid = grid_for(nl, kBlock);
  DevBuf<int64_t> cl(ctx, nl + 1), cg(ctx, nl + 1), lptr(ctx, nl + 1), gptr(ctx, nl + 1);
  GIFT_CUDA(cudaMemsetAsync(cl.p + nl, 0, sizeof(int64_t), st));
  GIFT_CUDA(cudaMemsetAsync(cg.p + nl, 0, sizeof(int64_t), st));
  if (nl > 0) {
    k_split_counts<<<grid, kBlock, 0, st>>>(r0, r1, c->indptr, c->indices, cl.p, cg.p);
    GIFT_LAUNCH_CHECK(ctx);
  }
  exclusive_scan_i64(ctx, cl.p, lptr.p, nl + 1);
  exclusive_scan_i64(ctx, cg.p, gptr.p, nl + 1);
  int64_t tot[2];
  GIFT_CUDA(cudaMemcpyAsync(&tot[0], lptr.p + nl, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GIFT_CUDA(cudaMemcpyAsync(&tot[1], gptr.p + nl, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GIFT_CUDA(cudaStreamSynchronize(st));
  const int64_t nnz_l = tot[0], nnz_g = tot[1];
  // distinct ghost columns, ascending
  DevBuf<int32_t> gcol_raw(ctx, nnz_g + 1), gcol_s(ctx, nnz_g + 1), gids(ctx, nnz_g + 1);
  DevBuf<int64_t> nsel(ctx, 1);
  int64_t ng = 0;
  if (nnz_g > 0) {
    k_ghost_cols<<<grid, kBlock, 0, st>>>(r0, r1, c->indptr, c->indices, gptr.p, gcol_raw.p);
    GIFT_LAUNCH_CHECK(ctx);
    const int bits = bit_length((uint64_t)(c->n > 1 ? c->n - 1 : 1));
    size_t bytes = 0;
    GIFT_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, gcol_raw.p, gcol_s.p, nnz_g, 0, bits, st));
    {
      DevBuf<char> tmp(ctx, bytes);
      GIFT_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, bytes, gcol_raw.p, gcol_s.p, nnz_g, 0, bits, st));
    }
    bytes = 0;
    GIFT_CUDA(cub::DeviceSelect::Unique(nullptr, bytes, gcol_s.p, gids.p, nsel.p, nnz_g, st));
    {
      DevBuf<char> tmp(ctx, bytes);
      GIFT_CUDA(cub::DeviceSelect::Unique(tmp.p, bytes, gcol_s.p, gids.p, nsel.p, nnz_g, st));
    }
    ctx->launches += 6;
    GIFT_CUDA(cudaMemcpyAsync(&ng, nsel.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    GIFT_CUDA(cudaStreamSynchronize(st));
  }
  DevBuf<int32_t> lcol(ctx, nnz_l + 1), gcol(ctx, nnz_g + 1);
  DevBuf<double> lval(ctx, nnz_l + 1), gval(ctx, nnz_g + 1);
  if (nl > 0) {
    k_split_fill<<<grid, kBlock, 0, st>>>(r0, r1, c->indptr, c->indices, c->values, lptr.p, gptr.p, gids.p, ng, lcol.p,
                                          lval.p, gcol.p, gval.p);
    GIFT_LAUNCH_CHECK(ctx);
  }
  Csr* L = csr_from_arrays(ctx, nl, nnz_l, lptr.p, lcol.p, lval.p);
  Csr* G = nullptr;
  try {
    G = csr_from_arrays(ctx, nl, nnz_g, gptr.p, gcol.p, gval.p);
    G->ext_n = ng;
    G->ext_ids = static_cast<int64_t*>(csr_alloc(ctx, G, (ng > 0 ? ng : 1) * sizeof(int64_t)));
    if (ng > 0) {
      k_i32_to_i64<<<grid_for(ng, kBlock), kBlock, 0, st>>>(ng, gids.p, G->ext_ids);
      GIFT_LAUNCH_CHECK(ctx);
    }
    // the caller's later work on the blocks is ordered after these copies
    csr_touch(ctx, L);
    csr_touch(ctx, G);
  } catch (...) {
    csr_touch(ctx, L);
    csr_destroy(L);
    if (G) {
      csr_touch(ctx, G);
      csr_destroy(G);
    }
    throw;
  }
  *local = L;
  *ghost = G;
}

}  // namespace gift
