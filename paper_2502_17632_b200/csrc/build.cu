// build.cu -- netlist -> clique graph CSR on the GPU, bit-identical to the
// reference build_clique_graph (graph.py:120-158) + SparseSymMatrix
// canonicalisation (graph.py:55-58), and from_coo (graph.py:114-117).
//
// Pipeline:
//   K1  pair counts per net (m(m-1)/2, 0 if m<2 or m>cap)  -> scan -> pair offsets
//       net id per pair by scatter + max-scan (segment expansion)
//   K1b expand: pair t -> (p,q) by integer-exact triu inversion,
//       key = (min<<cb | max) (self pairs -> INVALID key), value 2.0/m (fp64)
//   K2  stable LSD radix sort of the 64-bit keys carrying the pair sequence id
//       (scipy's coo_tocsr is a stable row bucketing -> seq order per row)
//   K3  head flags, unique ids, duplicate sums in seq order (__dadd_rn),
//       order-sensitive keys (>= 3 contributions, not all equal) flag their row,
//       global "some row has a column descent" flag (scipy sorts ALL rows iff so)
//   K3b for flagged rows when the descent flag is set: gather the row in seq
//       order, run the libstdc++ introsort emulation, re-sum its duplicates
//   K4  symmetrise U + U^T: radix sort of transposed keys, merge lower ++ upper
//   K5  degrees (numpy pairwise order) -- in filter.cu, lazily
// All fp64 arithmetic uses explicit-rounding intrinsics (no FMA contraction).
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <cstring>

#include "common.cuh"
#include "introsort.cuh"

namespace gift {

namespace {

constexpr int kBlock = 256;

__global__ void k_pair_counts(int64_t n_nets, const int64_t* __restrict__ net_start, int64_t cap,
                              int64_t* __restrict__ counts, unsigned long long* __restrict__ skipped) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_nets;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t m = net_start[e + 1] - net_start[e];
    int64_t c = 0;
    if (m >= 2) {
      if (cap >= 0 && m > cap) atomicAdd(skipped, 1ULL);  // graph.py:136-138; cap < 0 = None
      else c = m * (m - 1) / 2;
    }
    counts[e] = c;
  }
}

// first pair of every non-empty net gets the net id; max-scan fills the rest
__global__ void k_mark_net_heads(int64_t n_nets, const int64_t* __restrict__ counts,
                                 const int64_t* __restrict__ pair_end, int32_t* __restrict__ netid) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_nets;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t c = counts[e];
    if (c > 0) netid[pair_end[e] - c] = (int32_t)e;
  }
}

struct MaxOp {
  __device__ __forceinline__ int32_t operator()(int32_t a, int32_t b) const { return a > b ? a : b; }
};

// local triu index l of an m x m upper triangle -> (p, q), integer exact
__device__ __forceinline__ void triu_invert(int64_t l, int64_t m, int64_t& p, int64_t& q) {
  // off(p) = p*(2m-p-1)/2 ; find largest p with off(p) <= l
  double b = (double)(2 * m - 1);
  double disc = b * b - 8.0 * (double)l;
  int64_t pp = (int64_t)((b - sqrt(disc > 0 ? disc : 0.0)) * 0.5);
  if (pp < 0) pp = 0;
  if (pp > m - 2) pp = m - 2;
  while (pp > 0 && pp * (2 * m - pp - 1) / 2 > l) --pp;
  while (pp + 1 <= m - 2 && (pp + 1) * (2 * m - pp - 2) / 2 <= l) ++pp;
  p = pp;
  q = l - pp * (2 * m - pp - 1) / 2 + pp + 1;
}

__global__ void k_expand_pairs(int64_t T, const int32_t* __restrict__ netid,
                               const int64_t* __restrict__ pair_end, const int64_t* __restrict__ net_start,
                               const int32_t* __restrict__ pin_cell, int cb, uint64_t* __restrict__ keys,
                               double* __restrict__ pval, uint32_t* __restrict__ seq,
                               unsigned long long* __restrict__ n_invalid, uint32_t n_cells,
                               unsigned long long* __restrict__ bad) {
  const uint64_t invalid = 1ULL << (2 * cb);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < T; t += (int64_t)gridDim.x * blockDim.x) {
    int32_t e = netid[t];
    int64_t s = net_start[e];
    int64_t m = net_start[e + 1] - s;
    int64_t first = pair_end[e] - m * (m - 1) / 2;
    int64_t p, q;
    triu_invert(t - first, m, p, q);
    uint32_t a = (uint32_t)pin_cell[s + p];
    uint32_t b = (uint32_t)pin_cell[s + q];
    uint64_t key;
    if (a >= n_cells || b >= n_cells) {
      atomicAdd(bad, 1ULL);
      a = b = 0;
    }
    if (a == b) {
      key = invalid;
      atomicAdd(n_invalid, 1ULL);
    } else {
      uint64_t lo = a < b ? a : b, hi = a < b ? b : a;
      key = (lo << cb) | hi;
    }
    keys[t] = key;
    pval[t] = __ddiv_rn(2.0, (double)m);  // graph.py:149
    seq[t] = (uint32_t)t;
  }
}

__global__ void k_coo_keys(int64_t T, const int64_t* __restrict__ rows, const int64_t* __restrict__ cols,
                           int64_t n, int cb, uint64_t* __restrict__ keys, uint32_t* __restrict__ seq,
                           unsigned long long* __restrict__ bad) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < T; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = rows[t], c = cols[t];
    if (r < 0 || r >= n || c < 0 || c >= n) {
      atomicAdd(bad, 1ULL);
      r = 0;
      c = 0;
    }
    keys[t] = ((uint64_t)r << cb) | (uint64_t)c;
    seq[t] = (uint32_t)t;
  }
}

// head flags + column-descent detection on the sorted (key, seq) stream
__global__ void k_heads(int64_t Tv, const uint64_t* __restrict__ keys, const uint32_t* __restrict__ seq, int cb,
                        uint32_t* __restrict__ head, int* __restrict__ descent) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < Tv; t += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = keys[t];
    uint32_t h = 1;
    if (t > 0) {
      uint64_t kp = keys[t - 1];
      h = (k != kp);
      // same row, later key but earlier in emission order -> a descent in
      // that row's seq-ordered column sequence (scipy csr_has_sorted_indices)
      if ((k >> cb) == (kp >> cb) && seq[t] < seq[t - 1]) *descent = 1;
    }
    head[t] = h;
  }
}

__global__ void k_unique_starts(int64_t Tv, const uint32_t* __restrict__ head, const uint32_t* __restrict__ uid,
                                const uint64_t* __restrict__ keys, int64_t* __restrict__ ustart,
                                uint64_t* __restrict__ ukey) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < Tv; t += (int64_t)gridDim.x * blockDim.x) {
    if (head[t]) {
      uint32_t u = uid[t] - 1;
      ustart[u] = t;
      ukey[u] = keys[t];
    }
    if (t == Tv - 1) ustart[uid[t]] = Tv;
  }
}

// csr_sum_duplicates: x = v0; x += v1; ... in (stable) seq order
__global__ void k_sum_duplicates(int64_t U, const int64_t* __restrict__ ustart, const uint32_t* __restrict__ seq,
                                 const double* __restrict__ pval, const uint64_t* __restrict__ ukey, int cb,
                                 double* __restrict__ uval, uint8_t* __restrict__ rowflag,
                                 int* __restrict__ anyflag) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < U; u += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = ustart[u], b = ustart[u + 1];
    double v0 = pval[seq[a]];
    double x = v0;
    bool same = true;
    for (int64_t t = a + 1; t < b; ++t) {
      double v = pval[seq[t]];
      same &= (__double_as_longlong(v) == __double_as_longlong(v0));
      x = __dadd_rn(x, v);
    }
    uval[u] = x;
    if (b - a >= 3 && !same) {
      rowflag[ukey[u] >> cb] = 1;
      *anyflag = 1;
    }
  }
}

__global__ void k_flag_pairs(int64_t T, const uint64_t* __restrict__ keys, int cb,
                             const uint8_t* __restrict__ rowflag, uint8_t* __restrict__ f) {
  const uint64_t invalid = 1ULL << (2 * cb);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < T; t += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = keys[t];
    f[t] = (k < invalid) && rowflag[k >> cb];
  }
}

__global__ void k_row_heads(int64_t F, const uint64_t* __restrict__ keys, int cb, uint8_t* __restrict__ h) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < F; t += (int64_t)gridDim.x * blockDim.x)
    h[t] = (t == 0) || ((keys[t] >> cb) != (keys[t - 1] >> cb));
}

__device__ __forceinline__ int64_t lower_bound_u64(const uint64_t* a, int64_t n, uint64_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// K3b: one thread per flagged row; entries [seg_start[r], seg_end) of the
// row-grouped, seq-ordered arrays (fkeys, fseq).  Introsort emulation in the
// scratch KV buffer at the same offsets, then left-to-right duplicate sums
// written over the row's unique values.
__global__ void k_introsort_fixup(int64_t nseg, int64_t F, const int64_t* __restrict__ seg_start,
                                  const uint64_t* __restrict__ fkeys, const uint32_t* __restrict__ fseq,
                                  const double* __restrict__ pval, int cb, KV* __restrict__ work,
                                  const uint64_t* __restrict__ ukey, int64_t U, double* __restrict__ uval,
                                  int* __restrict__ mismatch) {
  const uint64_t cmask = (1ULL << cb) - 1;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nseg; r += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = seg_start[r];
    int64_t b = (r + 1 < nseg) ? seg_start[r + 1] : F;
    KV* w = work + a;
    for (int64_t t = a; t < b; ++t) {
      KV kv;
      kv.k = (uint32_t)(fkeys[t] & cmask);
      kv.pad = 0;
      kv.v = pval[fseq[t]];
      w[t - a] = kv;
    }
    dev_std_sort(w, b - a);
    uint64_t row = fkeys[a] >> cb;
    int64_t u = lower_bound_u64(ukey, U, row << cb);
    int64_t L = b - a, j = 0;
    while (j < L) {
      uint32_t c = w[j].k;
      double x = w[j].v;
      ++j;
      while (j < L && w[j].k == c) {
        x = __dadd_rn(x, w[j].v);
        ++j;
      }
      if (u >= U || ukey[u] != ((row << cb) | c)) *mismatch = 1;
      else uval[u] = x;
      ++u;
    }
  }
}

// row start offsets of a (row<<cb | col)-sorted key array: start[r] = first index with row >= r
__global__ void k_row_starts(int64_t U, const uint64_t* __restrict__ keys, int cb, int64_t n,
                             int64_t* __restrict__ start) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u <= U; u += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = (u < U) ? (int64_t)(keys[u] >> cb) : n;
    int64_t rp = (u > 0) ? (int64_t)(keys[u - 1] >> cb) : -1;
    for (int64_t rr = rp + 1; rr <= r; ++rr) start[rr] = u;
  }
}

__global__ void k_add_ptrs(int64_t n1, const int64_t* __restrict__ a, const int64_t* __restrict__ b,
                           int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n1; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = a[i] + b[i];
}

__global__ void k_transpose_keys(int64_t U, const uint64_t* __restrict__ ukey, int cb, uint64_t* __restrict__ tkey) {
  const uint64_t cmask = (1ULL << cb) - 1;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < U; u += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = ukey[u];
    tkey[u] = ((k & cmask) << cb) | (k >> cb);
  }
}

// U + U^T scatter: row i = [lower part (from U^T, ascending)] ++ [upper part]
__global__ void k_sym_scatter_upper(int64_t U, const uint64_t* __restrict__ ukey, const double* __restrict__ uval,
                                    int cb, const int64_t* __restrict__ indptr, const int64_t* __restrict__ up_start,
                                    const int64_t* __restrict__ lo_start, int32_t* __restrict__ indices,
                                    double* __restrict__ values) {
  const uint64_t cmask = (1ULL << cb) - 1;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < U; u += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = ukey[u];
    int64_t r = (int64_t)(k >> cb);
    int64_t pos = indptr[r] + (lo_start[r + 1] - lo_start[r]) + (u - up_start[r]);
    indices[pos] = (int32_t)(k & cmask);
    values[pos] = uval[u];
  }
}

__global__ void k_sym_scatter_lower(int64_t U, const uint64_t* __restrict__ tkey, const double* __restrict__ tval,
                                    int cb, const int64_t* __restrict__ indptr, const int64_t* __restrict__ lo_start,
                                    int32_t* __restrict__ indices, double* __restrict__ values) {
  const uint64_t cmask = (1ULL << cb) - 1;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < U; t += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = tkey[t];
    int64_t r = (int64_t)(k >> cb);
    int64_t pos = indptr[r] + (t - lo_start[r]);
    indices[pos] = (int32_t)(k & cmask);
    values[pos] = tval[t];
  }
}

__global__ void k_csr_from_sorted(int64_t U, const uint64_t* __restrict__ ukey, const double* __restrict__ uval,
                                  int cb, int32_t* __restrict__ indices, double* __restrict__ values) {
  const uint64_t cmask = (1ULL << cb) - 1;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < U; u += (int64_t)gridDim.x * blockDim.x) {
    indices[u] = (int32_t)(ukey[u] & cmask);
    values[u] = uval[u];
  }
}

__global__ void k_nonzero_flags(int64_t U, const double* __restrict__ v, uint8_t* __restrict__ f) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < U; u += (int64_t)gridDim.x * blockDim.x)
    f[u] = (v[u] != 0.0);
}

__global__ void k_has_diagonal(int64_t U, const uint64_t* __restrict__ ukey, int cb, int* __restrict__ flag) {
  const uint64_t cmask = (1ULL << cb) - 1;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < U; u += (int64_t)gridDim.x * blockDim.x)
    if ((ukey[u] >> cb) == (ukey[u] & cmask)) *flag = 1;
}

// SparseSymMatrix symmetry check (graph.py:61-65): max |A_ij - A_ji| vs
// 1e-12 * (1 + max |A|).  Non-negative doubles order like their bit patterns.
__global__ void k_symmetry(int64_t n, const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                           const double* __restrict__ values, unsigned long long* __restrict__ maxdiff,
                           unsigned long long* __restrict__ maxabs) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double md = 0.0, ma = 0.0;
    for (int64_t jj = indptr[i]; jj < indptr[i + 1]; ++jj) {
      int64_t j = indices[jj];
      double v = values[jj];
      double vt = 0.0;
      int64_t lo = indptr[j], hi = indptr[j + 1];
      while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (indices[mid] < i) lo = mid + 1;
        else hi = mid;
      }
      if (lo < indptr[j + 1] && indices[lo] == i) vt = values[lo];
      double d = fabs(__dsub_rn(v, vt));
      md = d > md ? d : md;
      double av = fabs(v);
      ma = av > ma ? av : ma;
    }
    if (md > 0) atomicMax(maxdiff, (unsigned long long)__double_as_longlong(md));
    if (ma > 0) atomicMax(maxabs, (unsigned long long)__double_as_longlong(ma));
  }
}

struct Scratch {
  Ctx* ctx;
  void* p = nullptr;
  size_t bytes = 0;
  explicit Scratch(Ctx* c) : ctx(c) {}
  void* get(size_t b) {
    if (b > bytes) {
      if (p) dev_free(ctx, p);
      p = dev_alloc(ctx, b);
      bytes = b;
    }
    return p;
  }
  ~Scratch() {
    if (p) dev_free(ctx, p);
  }
};

template <typename T>
T read_scalar(Ctx* ctx, const T* d) {
  T h;
  GIFT_CUDA(cudaMemcpyAsync(&h, d, sizeof(T), cudaMemcpyDeviceToHost, ctx->stream));
  GIFT_CUDA(cudaStreamSynchronize(ctx->stream));
  return h;
}

// ---------------------------------------------------------------------------
// Canonicalise a COO stream (keys in emission/seq order, fp64 value per seq)
// exactly as scipy tocsr(): stable row bucketing, then global descent test,
// introsort fix-up of order-sensitive rows, left-to-right duplicate sums.
// Output: unique sorted keys + values (U entries), owned by the returned bufs.
// ---------------------------------------------------------------------------
struct Canonical {
  DevBuf<uint64_t> ukey;
  DevBuf<double> uval;
  int64_t U = 0;
  bool descent = false;
  int64_t flagged_rows = 0;
};

Canonical canonicalise(Ctx* ctx, int64_t n, int64_t T, DevBuf<uint64_t>& keys, DevBuf<double>& pval,
                       DevBuf<uint32_t>& seq, int cb, int64_t n_invalid) {
  cudaStream_t st = ctx->stream;
  Canonical out;
  const int end_bit = 2 * cb + 1;
  Scratch tmp(ctx);
  DevBuf<uint64_t> keys_s(ctx, T);
  DevBuf<uint32_t> seq_s(ctx, T);
  {
    size_t bytes = 0;
    GIFT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.p, keys_s.p, seq.p, seq_s.p, T, 0, end_bit, st));
    GIFT_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(bytes), bytes, keys.p, keys_s.p, seq.p, seq_s.p, T, 0,
                                              end_bit, st));
    ctx->launches += 4;
  }
  const int64_t Tv = T - n_invalid;  // INVALID (self-pair) keys sort last
  if (Tv <= 0) return out;
  DevBuf<uint32_t> head(ctx, Tv), uid(ctx, Tv);
  DevBuf<int> flags(ctx, 4);
  GIFT_CUDA(cudaMemsetAsync(flags.p, 0, 4 * sizeof(int), st));
  k_heads<<<grid_for(Tv, kBlock), kBlock, 0, st>>>(Tv, keys_s.p, seq_s.p, cb, head.p, flags.p + 0);
  GIFT_LAUNCH_CHECK(ctx);
  {
    size_t bytes = 0;
    GIFT_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, head.p, uid.p, Tv, st));
    GIFT_CUDA(cub::DeviceScan::InclusiveSum(tmp.get(bytes), bytes, head.p, uid.p, Tv, st));
    ctx->launches += 2;
  }
  const int64_t U = (int64_t)read_scalar(ctx, uid.p + (Tv - 1));
  out.U = U;
  DevBuf<int64_t> ustart(ctx, U + 1);
  out.ukey = DevBuf<uint64_t>(ctx, U);
  out.uval = DevBuf<double>(ctx, U);
  k_unique_starts<<<grid_for(Tv, kBlock), kBlock, 0, st>>>(Tv, head.p, uid.p, keys_s.p, ustart.p, out.ukey.p);
  GIFT_LAUNCH_CHECK(ctx);
  DevBuf<uint8_t> rowflag(ctx, n + 1);
  GIFT_CUDA(cudaMemsetAsync(rowflag.p, 0, n + 1, st));
  k_sum_duplicates<<<grid_for(U, kBlock), kBlock, 0, st>>>(U, ustart.p, seq_s.p, pval.p, out.ukey.p, cb, out.uval.p,
                                                           rowflag.p, flags.p + 1);
  GIFT_LAUNCH_CHECK(ctx);
  int hflags[4];
  GIFT_CUDA(cudaMemcpyAsync(hflags, flags.p, sizeof(hflags), cudaMemcpyDeviceToHost, st));
  GIFT_CUDA(cudaStreamSynchronize(st));
  out.descent = hflags[0] != 0;
  // scipy skips csr_sort_indices unless some row has a descent; without the
  // sort the stable (seq-order) sums above ARE the reference's.
  if (!(hflags[0] && hflags[1])) return out;

  // ---- K3b: introsort emulation for rows holding order-sensitive keys ----
  head.reset();
  uid.reset();
  DevBuf<uint8_t> f(ctx, T);
  k_flag_pairs<<<grid_for(T, kBlock), kBlock, 0, st>>>(T, keys.p, cb, rowflag.p, f.p);
  GIFT_LAUNCH_CHECK(ctx);
  DevBuf<int64_t> nsel(ctx, 2);
  int64_t F = 0;
  DevBuf<uint64_t> fkeys(ctx, T);
  DevBuf<uint32_t> fseq(ctx, T);
  {
    size_t bytes = 0;
    GIFT_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, keys.p, f.p, fkeys.p, nsel.p, T, st));
    GIFT_CUDA(cub::DeviceSelect::Flagged(tmp.get(bytes), bytes, keys.p, f.p, fkeys.p, nsel.p, T, st));
    GIFT_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, seq.p, f.p, fseq.p, nsel.p + 1, T, st));
    GIFT_CUDA(cub::DeviceSelect::Flagged(tmp.get(bytes), bytes, seq.p, f.p, fseq.p, nsel.p + 1, T, st));
    ctx->launches += 4;
    F = read_scalar(ctx, nsel.p);
  }
  f.reset();
  DevBuf<uint64_t> fkeys_s(ctx, F);
  DevBuf<uint32_t> fseq_s(ctx, F);
  {
    // stable sort by row only -> each flagged row's entries in seq order
    size_t bytes = 0;
    GIFT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, fkeys.p, fkeys_s.p, fseq.p, fseq_s.p, F, cb,
                                              2 * cb, st));
    GIFT_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(bytes), bytes, fkeys.p, fkeys_s.p, fseq.p, fseq_s.p, F, cb,
                                              2 * cb, st));
    ctx->launches += 4;
  }
  fkeys.reset();
  fseq.reset();
  DevBuf<uint8_t> rh(ctx, F);
  k_row_heads<<<grid_for(F, kBlock), kBlock, 0, st>>>(F, fkeys_s.p, cb, rh.p);
  GIFT_LAUNCH_CHECK(ctx);
  DevBuf<int64_t> seg(ctx, F);
  int64_t nseg = 0;
  {
    size_t bytes = 0;
    thrust::counting_iterator<int64_t> it(0);
    GIFT_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, it, rh.p, seg.p, nsel.p, F, st));
    GIFT_CUDA(cub::DeviceSelect::Flagged(tmp.get(bytes), bytes, it, rh.p, seg.p, nsel.p, F, st));
    ctx->launches += 2;
    nseg = read_scalar(ctx, nsel.p);
  }
  out.flagged_rows = nseg;
  DevBuf<KV> work(ctx, F);
  k_introsort_fixup<<<grid_for(nseg, 64, 1LL << 30), 64, 0, st>>>(nseg, F, seg.p, fkeys_s.p, fseq_s.p, pval.p, cb,
                                                                   work.p, out.ukey.p, U, out.uval.p, flags.p + 2);
  GIFT_LAUNCH_CHECK(ctx);
  GIFT_CUDA(cudaMemcpyAsync(hflags, flags.p, sizeof(hflags), cudaMemcpyDeviceToHost, st));
  GIFT_CUDA(cudaStreamSynchronize(st));
  if (hflags[2]) throw_error(GIFT_ERR_INTERNAL, "introsort fix-up: unique key mismatch");
  return out;
}

Csr* new_csr(Ctx* ctx, int64_t n, int64_t nnz) {
  Csr* c = new gift_csr();
  c->device = ctx->device;
  c->n = n;
  c->nnz = nnz;
  c->indptr = static_cast<int64_t*>(csr_alloc(ctx, c, (n + 1) * sizeof(int64_t)));
  c->indices = static_cast<int32_t*>(csr_alloc(ctx, c, (nnz > 0 ? nnz : 1) * sizeof(int32_t)));
  c->values = static_cast<double*>(csr_alloc(ctx, c, (nnz > 0 ? nnz : 1) * sizeof(double)));
  c->mean_row = n > 0 ? (double)nnz / (double)n : 0.0;
  return c;
}

}  // namespace

// build_clique_graph (graph.py:120-158)
Csr* build_clique_graph(Ctx* ctx, int64_t n, int64_t n_nets, const int64_t* d_net_start, const int32_t* d_pin_cell,
                        int64_t cap, int64_t* n_skipped) {
  if (n < 0 || n_nets < 0) throw_error(GIFT_ERR_VALUE, "negative size");
  if (n >= (1LL << 31)) throw_error(GIFT_ERR_TOO_LARGE, "more than 2^31-1 cells");
  cudaStream_t st = ctx->stream;
  const int cb = bit_length((uint64_t)(n > 1 ? n - 1 : 1));
  int64_t T = 0;
  unsigned long long skipped = 0;
  DevBuf<int64_t> pair_end(ctx, n_nets + 1);
  if (n_nets >= (1LL << 31)) throw_error(GIFT_ERR_TOO_LARGE, "more than 2^31-1 nets");
  DevBuf<unsigned long long> counters(ctx, 3);
  GIFT_CUDA(cudaMemsetAsync(counters.p, 0, 3 * sizeof(unsigned long long), st));
  if (n_nets > 0) {
    DevBuf<int64_t> counts(ctx, n_nets);
    k_pair_counts<<<grid_for(n_nets, kBlock), kBlock, 0, st>>>(n_nets, d_net_start, cap, counts.p, counters.p);
    GIFT_LAUNCH_CHECK(ctx);
    size_t bytes = 0;
    Scratch tmp(ctx);
    GIFT_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, counts.p, pair_end.p, n_nets, st));
    GIFT_CUDA(cub::DeviceScan::InclusiveSum(tmp.get(bytes), bytes, counts.p, pair_end.p, n_nets, st));
    ctx->launches += 2;
    T = read_scalar(ctx, pair_end.p + (n_nets - 1));
    skipped = read_scalar(ctx, counters.p);
    if (T >= (1LL << 32)) throw_error(GIFT_ERR_TOO_LARGE, "more than 2^32 clique pairs; lower max_clique_pins");
    if (T > 0) {
      // segment expansion: net id of every pair
      DevBuf<int32_t> netid_raw(ctx, T), netid(ctx, T);
      GIFT_CUDA(cudaMemsetAsync(netid_raw.p, 0, T * sizeof(int32_t), st));
      k_mark_net_heads<<<grid_for(n_nets, kBlock), kBlock, 0, st>>>(n_nets, counts.p, pair_end.p, netid_raw.p);
      GIFT_LAUNCH_CHECK(ctx);
      GIFT_CUDA(cub::DeviceScan::InclusiveScan(nullptr, bytes, netid_raw.p, netid.p, MaxOp(), T, st));
      GIFT_CUDA(cub::DeviceScan::InclusiveScan(tmp.get(bytes), bytes, netid_raw.p, netid.p, MaxOp(), T, st));
      ctx->launches += 2;
      netid_raw.reset();
      counts.reset();
      DevBuf<uint64_t> keys(ctx, T);
      DevBuf<double> pval(ctx, T);
      DevBuf<uint32_t> seq(ctx, T);
      k_expand_pairs<<<grid_for(T, kBlock), kBlock, 0, st>>>(T, netid.p, pair_end.p, d_net_start, d_pin_cell, cb,
                                                             keys.p, pval.p, seq.p, counters.p + 1,
                                                             (uint32_t)n, counters.p + 2);
      GIFT_LAUNCH_CHECK(ctx);
      netid.reset();
      if (read_scalar(ctx, counters.p + 2))
        throw_error(GIFT_ERR_VALUE, "pin references a cell id out of range [0, n_cells)");
      const int64_t n_invalid = (int64_t)read_scalar(ctx, counters.p + 1);
      Canonical can = canonicalise(ctx, n, T, keys, pval, seq, cb, n_invalid);
      keys.reset();
      pval.reset();
      seq.reset();
      if (n_skipped) *n_skipped = (int64_t)skipped;
      const int64_t U = can.U;
      if (U > 0) {
        // ---- K4: symmetrise ----
        DevBuf<uint64_t> tkey(ctx, U), tkey_s(ctx, U);
        DevBuf<double> tval(ctx, U);
        k_transpose_keys<<<grid_for(U, kBlock), kBlock, 0, st>>>(U, can.ukey.p, cb, tkey.p);
        GIFT_LAUNCH_CHECK(ctx);
        size_t b2 = 0;
        GIFT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b2, tkey.p, tkey_s.p, can.uval.p, tval.p, U, 0, 2 * cb, st));
        GIFT_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(b2), b2, tkey.p, tkey_s.p, can.uval.p, tval.p, U, 0, 2 * cb,
                                                  st));
        ctx->launches += 4;
        tkey.reset();
        DevBuf<int64_t> up_start(ctx, n + 1), lo_start(ctx, n + 1);
        k_row_starts<<<grid_for(U + 1, kBlock), kBlock, 0, st>>>(U, can.ukey.p, cb, n, up_start.p);
        GIFT_LAUNCH_CHECK(ctx);
        k_row_starts<<<grid_for(U + 1, kBlock), kBlock, 0, st>>>(U, tkey_s.p, cb, n, lo_start.p);
        GIFT_LAUNCH_CHECK(ctx);
        Csr* c = new_csr(ctx, n, 2 * U);
        c->has_diagonal = false;
        k_add_ptrs<<<grid_for(n + 1, kBlock), kBlock, 0, st>>>(n + 1, up_start.p, lo_start.p, c->indptr);
        GIFT_LAUNCH_CHECK(ctx);
        k_sym_scatter_upper<<<grid_for(U, kBlock), kBlock, 0, st>>>(U, can.ukey.p, can.uval.p, cb, c->indptr,
                                                                    up_start.p, lo_start.p, c->indices, c->values);
        GIFT_LAUNCH_CHECK(ctx);
        k_sym_scatter_lower<<<grid_for(U, kBlock), kBlock, 0, st>>>(U, tkey_s.p, tval.p, cb, c->indptr, lo_start.p,
                                                                    c->indices, c->values);
        GIFT_LAUNCH_CHECK(ctx);
        return c;
      }
    }
  }
  if (n_skipped) *n_skipped = (int64_t)skipped;
  // no pairs: empty n x n (graph.py:153-154)
  Csr* c = new_csr(ctx, n, 0);
  c->has_diagonal = false;
  GIFT_CUDA(cudaMemsetAsync(c->indptr, 0, (n + 1) * sizeof(int64_t), st));
  return c;
}

// from_coo (graph.py:114-117) + SparseSymMatrix(...) checks (graph.py:55-65)
Csr* csr_from_coo(Ctx* ctx, int64_t n, int64_t T, const int64_t* d_rows, const int64_t* d_cols,
                  const double* d_vals, bool check_symmetric) {
  if (n < 0 || T < 0) throw_error(GIFT_ERR_VALUE, "negative size");
  if (n >= (1LL << 31)) throw_error(GIFT_ERR_TOO_LARGE, "more than 2^31-1 rows");
  if (T >= (1LL << 32)) throw_error(GIFT_ERR_TOO_LARGE, "more than 2^32 entries");
  cudaStream_t st = ctx->stream;
  const int cb = bit_length((uint64_t)(n > 1 ? n - 1 : 1));
  Csr* c = nullptr;
  if (T > 0) {
    DevBuf<uint64_t> keys(ctx, T);
    DevBuf<uint32_t> seq(ctx, T);
    DevBuf<double> pval(ctx, T);
    DevBuf<unsigned long long> bad(ctx, 1);
    GIFT_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(unsigned long long), st));
    GIFT_CUDA(cudaMemcpyAsync(pval.p, d_vals, T * sizeof(double), cudaMemcpyDeviceToDevice, st));
    k_coo_keys<<<grid_for(T, kBlock), kBlock, 0, st>>>(T, d_rows, d_cols, n, cb, keys.p, seq.p, bad.p);
    GIFT_LAUNCH_CHECK(ctx);
    if (read_scalar(ctx, bad.p)) throw_error(GIFT_ERR_VALUE, "row or column index out of range for matrix dimensions");
    Canonical can = canonicalise(ctx, n, T, keys, pval, seq, cb, 0);
    keys.reset();
    seq.reset();
    pval.reset();
    int64_t U = can.U;
    // eliminate_zeros (graph.py:58)
    DevBuf<uint8_t> nz(ctx, U > 0 ? U : 1);
    DevBuf<uint64_t> k2(ctx, U > 0 ? U : 1);
    DevBuf<double> v2(ctx, U > 0 ? U : 1);
    DevBuf<int64_t> nsel(ctx, 2);
    int64_t U2 = 0;
    if (U > 0) {
      k_nonzero_flags<<<grid_for(U, kBlock), kBlock, 0, st>>>(U, can.uval.p, nz.p);
      GIFT_LAUNCH_CHECK(ctx);
      Scratch tmp(ctx);
      size_t bytes = 0;
      GIFT_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, can.ukey.p, nz.p, k2.p, nsel.p, U, st));
      GIFT_CUDA(cub::DeviceSelect::Flagged(tmp.get(bytes), bytes, can.ukey.p, nz.p, k2.p, nsel.p, U, st));
      GIFT_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, can.uval.p, nz.p, v2.p, nsel.p + 1, U, st));
      GIFT_CUDA(cub::DeviceSelect::Flagged(tmp.get(bytes), bytes, can.uval.p, nz.p, v2.p, nsel.p + 1, U, st));
      ctx->launches += 4;
      U2 = read_scalar(ctx, nsel.p);
    }
    c = new_csr(ctx, n, U2);
    if (U2 > 0) {
      k_row_starts<<<grid_for(U2 + 1, kBlock), kBlock, 0, st>>>(U2, k2.p, cb, n, c->indptr);
      GIFT_LAUNCH_CHECK(ctx);
      k_csr_from_sorted<<<grid_for(U2, kBlock), kBlock, 0, st>>>(U2, k2.p, v2.p, cb, c->indices, c->values);
      GIFT_LAUNCH_CHECK(ctx);
      DevBuf<int> diag(ctx, 1);
      GIFT_CUDA(cudaMemsetAsync(diag.p, 0, sizeof(int), st));
      k_has_diagonal<<<grid_for(U2, kBlock), kBlock, 0, st>>>(U2, k2.p, cb, diag.p);
      GIFT_LAUNCH_CHECK(ctx);
      c->has_diagonal = read_scalar(ctx, diag.p) != 0;
    } else {
      GIFT_CUDA(cudaMemsetAsync(c->indptr, 0, (n + 1) * sizeof(int64_t), st));
      c->has_diagonal = false;
    }
  } else {
    c = new_csr(ctx, n, 0);
    GIFT_CUDA(cudaMemsetAsync(c->indptr, 0, (n + 1) * sizeof(int64_t), st));
    c->has_diagonal = false;
  }
  if (check_symmetric && c->nnz > 0) {
    DevBuf<unsigned long long> mx(ctx, 2);
    GIFT_CUDA(cudaMemsetAsync(mx.p, 0, 2 * sizeof(unsigned long long), st));
    k_symmetry<<<grid_for(n, kBlock), kBlock, 0, st>>>(n, c->indptr, c->indices, c->values, mx.p, mx.p + 1);
    GIFT_LAUNCH_CHECK(ctx);
    unsigned long long h[2];
    GIFT_CUDA(cudaMemcpyAsync(h, mx.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    GIFT_CUDA(cudaStreamSynchronize(st));
    double maxdiff, maxabs;
    memcpy(&maxdiff, &h[0], 8);
    memcpy(&maxabs, &h[1], 8);
    if (maxdiff > 1e-12 * (1.0 + maxabs)) {
      csr_destroy(c);
      throw_error(GIFT_ERR_NON_SYMMETRIC, "matrix is not symmetric");
    }
  }
  return c;
}

}  // namespace gift
