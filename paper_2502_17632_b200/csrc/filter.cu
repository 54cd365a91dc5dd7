// filter.cu -- degrees, normalisation and the GiFt filter bank on the GPU.
//
// Reference semantics (giftplace):
//   SparseSymMatrix.degrees      graph.py:89-94   -> k_degrees (numpy pairwise order, fp64)
//   normalized_augmented_adjacency graph.py:167-188 -> k_scale (s = 1/sqrt(d+sigma)),
//                                                   k_normalized_fill (materialised, API only)
//   SparseSymMatrix.matmul       graph.py:96-100  -> k_matvec_exact (csr_matvecs order)
//   gift_filter                  gift.py:73-95    -> bank_fp64_exact / bank_fp32
//   gift_place epilogue          gift.py:112-118  -> fused into the final hop
//
// The fast path (GIFT_PREC_FP32) never materialises A_sigma.  It runs the
// pre-scaled recurrence on the raw clique weights w (one fp32 copy of the
// CSR values serves every sigma):
//     z_0 = s o x ;  y_h = s o (A z_{h-1} + sigma z_{h-1}) ;  z_h = s o y_h
// (y_h == A_sigma^h x), and FUSES the sigma chains of the bank: chains are
// packed side by side in the signal (float4 = two chains of an N x 2 signal)
// so one pass over (col, w) advances every packed chain by one hop.  The
// default bank (0.1 A_2^2 + 0.7 A_4^2 + 0.2 A_4^4, 6 algorithmic hops) reads
// the matrix 4 times.  Term accumulation and the re-pin/clamp epilogue ride
// in the epilogue of the hop that completes them.
#include <cub/cub.cuh>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <set>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cooperative_groups.h>

#include "common.cuh"
#include "hop.cuh"

namespace cg = cooperative_groups;

namespace gift {

// hf.cu: implicit clique term of the nets above the cap (opt-in)
void hf_add_degrees(Ctx* ctx, const Csr* c, double* deg);
void hf_apply_f32(Ctx* ctx, const Csr* c, int F, const float* z, float* out);
bool fact_hop_applies(const Ctx* ctx, const Csr* c, const HopArgs& a, int fin);
bool fact_hop_f32(Ctx* ctx, Csr* c, const HopArgs& a, int fin, int fout);
void hf_apply_f64(Ctx* ctx, const Csr* c, int nc, const double* x, int64_t ld, int64_t c0, const double* s,
                  double* out);

namespace {

constexpr int kBlock = 256;

// ---- numpy pairwise summation (loops_utils.h pairwise_sum), fp64 ---------
__device__ __forceinline__ double pw_leaf(const double* __restrict__ a, int64_t n) {
  if (n < 8) {
    double res = -0.0;
    for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  int64_t i;
  for (i = 8; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, a[i]);
  return res;
}

// explicit-stack form of: n <= 128 -> leaf; else n2 = n/2 - (n/2)%8,
// PW(a, n2) + PW(a + n2, n - n2)
__device__ double pw_sum(const double* __restrict__ a, int64_t n) {
  if (n <= 128) return pw_leaf(a, n);
  int64_t off[48], len[48];
  double partial[48];
  uint8_t stage[48];
  int sp = 1;
  off[0] = 0;
  len[0] = n;
  stage[0] = 0;
  double ret = 0.0;
  while (sp > 0) {
    const int i = sp - 1;
    if (len[i] <= 128) {
      ret = pw_leaf(a + off[i], len[i]);
      --sp;
      continue;
    }
    int64_t n2 = len[i] / 2;
    n2 -= n2 % 8;
    if (stage[i] == 0) {
      stage[i] = 1;
      off[sp] = off[i];
      len[sp] = n2;
      stage[sp] = 0;
      ++sp;
    } else if (stage[i] == 1) {
      partial[i] = ret;
      stage[i] = 2;
      off[sp] = off[i] + n2;
      len[sp] = len[i] - n2;
      stage[sp] = 0;
      ++sp;
    } else {
      ret = __dadd_rn(partial[i], ret);
      --sp;
    }
  }
  return ret;
}

// np.add.reduceat(values, indptr[nonempty]) per row: v0 + PW(v[1:])
__global__ void k_degrees(int64_t n, const int64_t* __restrict__ indptr, const double* __restrict__ values,
                          double* __restrict__ deg) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = indptr[i], L = indptr[i + 1] - a;
    deg[i] = L == 0 ? 0.0 : __dadd_rn(values[a], pw_sum(values + a + 1, L - 1));
  }
}

// graph.py:184: s = 1.0 / np.sqrt(deg + sigma) (three correctly rounded ops)
__global__ void k_scale(int64_t n, const double* __restrict__ deg, double sigma, double* __restrict__ s64,
                        float* __restrict__ s32) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double s = __ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(deg[i], sigma)));
    s64[i] = s;
    if (s32) s32[i] = __double2float_rn(s);
  }
}

__global__ void k_first_isolated(int64_t n, const double* __restrict__ deg, unsigned long long* __restrict__ first) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (deg[i] <= 0) atomicMin(first, (unsigned long long)i);
}

__global__ void k_to_f32(int64_t m, const double* __restrict__ v, float* __restrict__ w) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    w[i] = __double2float_rn(v[i]);
}

// does row i already store a diagonal entry (only from_coo matrices can)?
__device__ __forceinline__ bool row_has_diag(const int64_t* indptr, const int32_t* idx, int64_t i) {
  int64_t lo = indptr[i], hi = indptr[i + 1];
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (idx[mid] < i) lo = mid + 1;
    else hi = mid;
  }
  return lo < indptr[i + 1] && idx[lo] == i;
}

__global__ void k_diag_extra(int64_t n, const int64_t* __restrict__ indptr, const int32_t* __restrict__ idx,
                             bool may_have_diag, int64_t* __restrict__ extra) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x)
    extra[i] = (i < n) ? ((may_have_diag && row_has_diag(indptr, idx, i)) ? 0 : 1) : 0;
}

__global__ void k_shift_ptr(int64_t n1, const int64_t* __restrict__ indptr, const int64_t* __restrict__ off,
                            int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n1; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = indptr[i] + off[i];
}

// graph.py:182-187: A + sigma I (diagonal enters at its sorted position as
// 0 + sigma, or a_ii + sigma), then (a * s_i) * s_j
__global__ void k_normalized_fill(int64_t n, const int64_t* __restrict__ indptr, const int32_t* __restrict__ idx,
                                  const double* __restrict__ val, const double* __restrict__ s, double sigma,
                                  const int64_t* __restrict__ optr, int32_t* __restrict__ oidx,
                                  double* __restrict__ oval) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t k = optr[i];
    const double si = s[i];
    bool diag_done = !(sigma > 0);
    for (int64_t jj = indptr[i]; jj < indptr[i + 1]; ++jj) {
      int64_t j = idx[jj];
      if (!diag_done && j > i) {
        oidx[k] = (int32_t)i;
        oval[k] = __dmul_rn(__dmul_rn(sigma, si), si);
        ++k;
        diag_done = true;
      }
      double a = val[jj];
      if (!diag_done && j == i) {
        a = __dadd_rn(a, sigma);
        diag_done = true;
      }
      oidx[k] = (int32_t)j;
      oval[k] = __dmul_rn(__dmul_rn(a, si), s[j]);
      ++k;
    }
    if (!diag_done) {
      oidx[k] = (int32_t)i;
      oval[k] = __dmul_rn(__dmul_rn(sigma, si), si);
    }
  }
}

// ---- exact fp64 SpMM: scipy csr_matvecs order ------------------------------
// y[i, c] = 0; y[i, c] += a_ij * x[j, c] over ascending storage order, no FMA.
// MODE 0: a_ij = stored value.  MODE 1: on-the-fly A_sigma entry
// (a*s_i)*s_j with the sigma diagonal at its sorted position, i.e. exactly
// the value the reference materialises (graph.py:182-187).
template <int MODE>
__global__ void k_matvec_exact(int64_t n, const int64_t* __restrict__ indptr, const int32_t* __restrict__ idx,
                               const double* __restrict__ val, const double* __restrict__ s, double sigma,
                               int64_t ld, int64_t c0, int nc, const double* __restrict__ x,
                               double* __restrict__ y, const double* __restrict__ extra) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    const double si = MODE ? s[i] : 0.0;
    bool diag_done = MODE ? !(sigma > 0) : true;
    for (int64_t jj = indptr[i]; jj < indptr[i + 1]; ++jj) {
      const int64_t j = idx[jj];
      double a = val[jj];
      if (MODE) {
        if (!diag_done && j > i) {
          const double d = __dmul_rn(__dmul_rn(sigma, si), si);
          for (int c = 0; c < nc; ++c) acc[c] = __dadd_rn(acc[c], __dmul_rn(d, x[i * ld + c0 + c]));
          diag_done = true;
        }
        if (!diag_done && j == i) {
          a = __dadd_rn(a, sigma);
          diag_done = true;
        }
        a = __dmul_rn(__dmul_rn(a, si), s[j]);
      }
      for (int c = 0; c < nc; ++c) acc[c] = __dadd_rn(acc[c], __dmul_rn(a, x[j * ld + c0 + c]));
    }
    if (MODE && !diag_done) {
      const double d = __dmul_rn(__dmul_rn(sigma, si), si);
      for (int c = 0; c < nc; ++c) acc[c] = __dadd_rn(acc[c], __dmul_rn(d, x[i * ld + c0 + c]));
    }
    if (extra)  // implicit high-fanout term (hf.cu): (A_hf (s o x))_i, scaled by s_i
      for (int c = 0; c < nc; ++c) acc[c] = __dadd_rn(acc[c], MODE ? __dmul_rn(si, extra[i * 4 + c]) : extra[i * 4 + c]);
    for (int c = 0; c < nc; ++c) y[i * ld + c0 + c] = acc[c];
  }
}

// out += alpha * p  (numpy: temp = alpha * power; out += temp), elementwise fp64
__global__ void k_axpy_exact(int64_t m, double alpha, const double* __restrict__ p, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __dadd_rn(out[i], __dmul_rn(alpha, p[i]));
}

__global__ void k_load_f64(int64_t m, int in_dtype, const void* __restrict__ g, double* __restrict__ x) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = in_dtype == GIFT_DTYPE_F64 ? static_cast<const double*>(g)[i]
                                      : (double)static_cast<const float*>(g)[i];
}

// gift.py:112-118 on an fp64 [n, 2] result, written in out_dtype
__global__ void k_epilogue_f64(int64_t n, int64_t ncols, const double* __restrict__ res,
                               const uint8_t* __restrict__ fixed_mask, const double* __restrict__ fixed_pos,
                               Region4 reg, int out_dtype, void* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * ncols;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v = res[i];
    if (fixed_mask) {
      const int64_t r = i / 2;
      const int c = (int)(i % 2);
      v = fixed_mask[r] ? fixed_pos[i] : np_clip(v, reg.v[c], reg.v[c + 2]);
    }
    if (out_dtype == GIFT_DTYPE_F64) static_cast<double*>(out)[i] = v;
    else static_cast<float*>(out)[i] = __double2float_rn(v);
  }
}

// One hop for every chain packed in zin.  G lanes own a row; each lane
// streams 4 consecutive (col, w) per 16-byte vector load (aligned down to a
// multiple of 4, out-of-row slots masked), U such chunks in flight, so a lane
// has 2U streaming loads then 4U gathers outstanding.  Lane partials reduce
// with a fixed xor-butterfly (deterministic order); lane 0 runs the epilogue.
template <int FIN, int FOUT, int G, int U>
__device__ __forceinline__ void hop_row(const HopArgs& a, int64_t gi) {
  const int lane = threadIdx.x & (G - 1);
  const int64_t row = a.row_list ? (int64_t)a.row_list[gi] : gi;
  const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1)));
  const uint64_t pol_s = policy_evict_first();
  const uint64_t pol_z = policy_evict_last();
  const int64_t beg = a.rowptr[row], end = a.rowptr[row + 1];
  float acc[FIN];
#pragma unroll
  for (int f = 0; f < FIN; ++f) acc[f] = 0.f;
  const int64_t base = beg & ~(int64_t)3;
  for (int64_t k0 = base + 4 * lane; k0 < end; k0 += 4 * G * U) {
    int4 cv[U];
    float4 wv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t k = k0 + (int64_t)(4 * G) * u;
      if (k < end) {
        cv[u] = ld_stream_v4s32(a.col + k, pol_s);
        wv[u] = ld_stream_v4f32(a.w + k, pol_s);
      } else {
        cv[u] = make_int4(0, 0, 0, 0);
        wv[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    VecF<FIN> zv[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t k = k0 + (int64_t)(4 * G) * u;
      const int cc[4] = {cv[u].x, cv[u].y, cv[u].z, cv[u].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (k + j >= beg && k + j < end) {
          zv[u][j] = ld_z<FIN>(a.zin + (int64_t)cc[j] * FIN, pol_z);
        } else {
#pragma unroll
          for (int f = 0; f < FIN; ++f) zv[u][j].v[f] = 0.f;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const float ww[4] = {wv[u].x, wv[u].y, wv[u].z, wv[u].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
#pragma unroll
        for (int f = 0; f < FIN; ++f) acc[f] = fmaf(ww[j], zv[u][j].v[f], acc[f]);
      }
    }
  }
#pragma unroll
  for (int off = G / 2; off > 0; off >>= 1) {
#pragma unroll
    for (int f = 0; f < FIN; ++f) acc[f] += __shfl_xor_sync(gmask, acc[f], off, G);
  }
  if (lane != 0) return;
  row_epilogue<FIN, FOUT>(a, row, acc, pol_z);
}

template <int FIN, int FOUT, int G, int U>
__global__ void __launch_bounds__(kBlock) k_hop(HopArgs a) {
  const int64_t gi = a.row_begin + (blockIdx.x * (int64_t)kBlock + threadIdx.x) / G;
  if (gi >= a.n) return;  // uniform within a row group
  hop_row<FIN, FOUT, G, U>(a, gi);
}


// z0[i, chn*wcols + cc] = s_chn[i] * g[i, c0 + cc]
struct PrepArgs {
  int64_t n;
  int wcols, nch;
  const float* s[4];
  int in_dtype;
  const void* g;
  int64_t ld, c0;
  float* z;
};

template <int F>
__device__ __forceinline__ void prep_row(const PrepArgs& p, int64_t i) {
  if constexpr (F == 4) {
    // the default bank's first pack (two chains of an N x 2 fp32 signal): one
    // 8-byte load, two scale loads, one 16-byte store -- the same products
    if (p.wcols == 2 && p.nch == 2 && p.in_dtype == GIFT_DTYPE_F32 && p.ld == 2 && p.c0 == 0 &&
        (reinterpret_cast<uintptr_t>(p.g) & 7) == 0) {
      const float2 x = static_cast<const float2*>(p.g)[i];
      const float s0 = p.s[0][i], s1 = p.s[1][i];
      *reinterpret_cast<float4*>(p.z + i * 4) = make_float4(s0 * x.x, s0 * x.y, s1 * x.x, s1 * x.y);
      return;
    }
  }
  float v[F];
#pragma unroll
  for (int f = 0; f < F; ++f) {
    const int chn = f / p.wcols, cc = f - chn * p.wcols;
    float x = 0.f, s = 0.f;
    if (chn < p.nch) {
      const int64_t gi = i * p.ld + p.c0 + cc;
      x = p.in_dtype == GIFT_DTYPE_F64 ? (float)static_cast<const double*>(p.g)[gi]
                                       : static_cast<const float*>(p.g)[gi];
      s = p.s[chn][i];
    }
    v[f] = s * x;
  }
  if constexpr (F == 4) *reinterpret_cast<float4*>(p.z + i * 4) = make_float4(v[0], v[1], v[2], v[3]);
  else if constexpr (F == 2) *reinterpret_cast<float2*>(p.z + i * 2) = make_float2(v[0], v[1]);
  else p.z[i] = v[0];
}

// the default bank's first pack (prep_row's fast path) with four rows in
// flight per thread: the one-row-per-thread kernel ran at ~2.4 TB/s on c4
__host__ __device__ __forceinline__ bool prep_is_default_pack(const PrepArgs& p) {
  return p.wcols == 2 && p.nch == 2 && p.in_dtype == GIFT_DTYPE_F32 && p.ld == 2 && p.c0 == 0 &&
         (reinterpret_cast<uintptr_t>(p.g) & 7) == 0;
}
__global__ void __launch_bounds__(256) k_prep4_rows(PrepArgs p) {
  const float2* __restrict__ g = static_cast<const float2*>(p.g);
  const float* __restrict__ s0 = p.s[0];
  const float* __restrict__ s1 = p.s[1];
  float4* __restrict__ z = reinterpret_cast<float4*>(p.z);
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i + 3 * T < p.n; i += 4 * T) {
    float2 x[4];
    float a[4], b[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      x[u] = g[i + u * T];
      a[u] = s0[i + u * T];
      b[u] = s1[i + u * T];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) z[i + u * T] = make_float4(a[u] * x[u].x, a[u] * x[u].y, b[u] * x[u].x, b[u] * x[u].y);
  }
  for (; i < p.n; i += T) {
    const float2 xv = g[i];
    const float av = s0[i], bv = s1[i];
    z[i] = make_float4(av * xv.x, av * xv.y, bv * xv.x, bv * xv.y);
  }
}

// z0[i, chn*wcols + cc] = s_chn[i] * g[i, c0 + cc]
template <int F>
__global__ void k_prep(PrepArgs p) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p.n; i += (int64_t)gridDim.x * blockDim.x)
    prep_row<F>(p, i);
}

__global__ void k_gather_rows(int64_t n_idx, int F, const int64_t* __restrict__ idx, const float* __restrict__ src,
                              float* __restrict__ dst) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_idx * F; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / F;
    dst[t] = src[idx[r] * F + (t - r * F)];
  }
}

int pow2_ceil(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

template <int FIN, int FOUT>
void launch_hop_g(Ctx* ctx, cudaStream_t st, const HopArgs& a, int G) {
  if (a.n <= a.row_begin) return;
  if (ctx->opt.row_lanes) G = (int)ctx->opt.row_lanes;
  const int64_t threads = (a.n - a.row_begin) * (int64_t)G;
  const unsigned grid = (unsigned)((threads + kBlock - 1) / kBlock);
#ifdef GIFT_TUNING
  if (env_int("GIFT_HOP_U", 1) >= 2) {  // two 4-entry chunks in flight per lane (tuning sweeps)
    switch (G) {
      case 8: k_hop<FIN, FOUT, 8, 2><<<grid, kBlock, 0, st>>>(a); break;
      case 16: k_hop<FIN, FOUT, 16, 2><<<grid, kBlock, 0, st>>>(a); break;
      default: k_hop<FIN, FOUT, 32, 2><<<grid, kBlock, 0, st>>>(a); break;
    }
    GIFT_LAUNCH_CHECK(ctx);
    return;
  }
#endif
  switch (G) {
    case 8: k_hop<FIN, FOUT, 8, 1><<<grid, kBlock, 0, st>>>(a); break;
    case 16: k_hop<FIN, FOUT, 16, 1><<<grid, kBlock, 0, st>>>(a); break;
    default: k_hop<FIN, FOUT, 32, 1><<<grid, kBlock, 0, st>>>(a); break;
  }
  GIFT_LAUNCH_CHECK(ctx);
}

template <int FIN>
void launch_hop_out(Ctx* ctx, cudaStream_t st, const HopArgs& a, int fout, int G) {
  switch (fout) {
    case 0: launch_hop_g<FIN, 0>(ctx, st, a, G); break;
    case 1: launch_hop_g<FIN, 1>(ctx, st, a, G); break;
    case 2: launch_hop_g<FIN, 2>(ctx, st, a, G); break;
    default: launch_hop_g<FIN, 4>(ctx, st, a, G); break;
  }
}

}  // namespace

// row kernel over an explicit row list on stream st (bmt.cu: the wide rows
// it leaves out, on the context's side stream)
void launch_row_list(Ctx* ctx, cudaStream_t st, const HopArgs& base, const int32_t* rows, int64_t nrows, int fin,
                     int fout, int G) {
  HopArgs a = base;
  a.row_list = rows;
  a.row_begin = 0;
  a.n = nrows;
  switch (fin) {
    case 1: launch_hop_out<1>(ctx, st, a, fout, G); break;
    case 2: launch_hop_out<2>(ctx, st, a, fout, G); break;
    default: launch_hop_out<4>(ctx, st, a, fout, G); break;
  }
}

namespace {

void launch_hop(Ctx* ctx, Csr* c, const HopArgs& a, int fin, int fout, int G, bool allow_bmt) {
  ProfScope prof(ctx, fin, a.nch);
  const bool tiled = allow_bmt && bmt_hop(ctx, c, a, fin, fout);
  c->fp32_hops++;
  if (tiled) return;
  switch (fin) {
    case 1: launch_hop_out<1>(ctx, ctx->stream, a, fout, G); break;
    case 2: launch_hop_out<2>(ctx, ctx->stream, a, fout, G); break;
    default: launch_hop_out<4>(ctx, ctx->stream, a, fout, G); break;
  }
}

}  // namespace

// ---------------------------------------------------------------------------
const double* csr_degrees(Ctx* ctx, Csr* c) {
  if (!c->degrees) {
    c->degrees = static_cast<double*>(csr_alloc(ctx, c, (c->n > 0 ? c->n : 1) * sizeof(double)));
    if (c->n > 0) {
      k_degrees<<<grid_for(c->n, kBlock, 1LL << 30), kBlock, 0, ctx->stream>>>(c->n, c->indptr, c->values,
                                                                             c->degrees);
      GIFT_LAUNCH_CHECK(ctx);
      hf_add_degrees(ctx, c, c->degrees);  // + the implicit high-fanout term, if any
    }
  }
  return c->degrees;
}

static const float* csr_w32(Ctx* ctx, Csr* c) {
  if (!c->w32) {
    c->w32 = static_cast<float*>(csr_alloc(ctx, c, (c->nnz > 0 ? c->nnz : 1) * sizeof(float)));
    if (c->nnz > 0) {
      k_to_f32<<<grid_for(c->nnz, kBlock), kBlock, 0, ctx->stream>>>(c->nnz, c->values, c->w32);
      GIFT_LAUNCH_CHECK(ctx);
    }
  }
  return c->w32;
}

const float* csr_w32_public(Ctx* ctx, Csr* c) { return csr_w32(ctx, c); }

// sigma validation + isolated-node check (graph.py:174-180); returns s64
static const double* csr_scale(Ctx* ctx, Csr* c, double sigma) {
  if (!(sigma >= 0)) throw_error(GIFT_ERR_VALUE, "sigma must be >= 0, got " + std::to_string(sigma));
  auto it = c->s64.find(sigma);
  if (it != c->s64.end()) return it->second;
  const double* deg = csr_degrees(ctx, c);
  if (sigma == 0 && c->n > 0) {
    DevBuf<unsigned long long> first(ctx, 1);
    GIFT_CUDA(cudaMemsetAsync(first.p, 0xff, sizeof(unsigned long long), ctx->stream));
    k_first_isolated<<<grid_for(c->n, kBlock), kBlock, 0, ctx->stream>>>(c->n, deg, first.p);
    GIFT_LAUNCH_CHECK(ctx);
    unsigned long long h;
    GIFT_CUDA(cudaMemcpyAsync(&h, first.p, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    GIFT_CUDA(cudaStreamSynchronize(ctx->stream));
    if (h != ~0ULL) {
      throw_error(GIFT_ERR_ISOLATED_NODE,
                  "node " + std::to_string(h) +
                      " has degree 0; normalization with sigma=0 is undefined (use sigma > 0 to absorb isolated nodes)",
                  (int64_t)h);
    }
  }
  double* s64 = static_cast<double*>(csr_alloc(ctx, c, (c->n > 0 ? c->n : 1) * sizeof(double)));
  float* s32 = static_cast<float*>(csr_alloc(ctx, c, (c->n > 0 ? c->n : 1) * sizeof(float)));
  if (c->n > 0) {
    k_scale<<<grid_for(c->n, kBlock), kBlock, 0, ctx->stream>>>(c->n, deg, sigma, s64, s32);
    GIFT_LAUNCH_CHECK(ctx);
  }
  c->s64[sigma] = s64;
  c->s32[sigma] = s32;
  return s64;
}

Csr* normalized_augmented_adjacency(Ctx* ctx, Csr* c, double sigma) {
  if (c->hf.nets)
    throw_error(GIFT_ERR_VALUE, "the graph has an implicit high-fanout term; it cannot be materialised "
                                "(build it with max_clique_pins=None for an explicit operator)");
  const double* s = csr_scale(ctx, c, sigma);
  cudaStream_t st = ctx->stream;
  const int64_t n = c->n;
  DevBuf<int64_t> extra(ctx, n + 1), off(ctx, n + 1);
  int64_t add = 0;
  if (sigma > 0) {
    k_diag_extra<<<grid_for(n + 1, kBlock), kBlock, 0, st>>>(n, c->indptr, c->indices, c->has_diagonal, extra.p);
    GIFT_LAUNCH_CHECK(ctx);
    size_t bytes = 0;
    GIFT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, extra.p, off.p, n + 1, st));
    DevBuf<char> tmp(ctx, bytes);
    GIFT_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, extra.p, off.p, n + 1, st));
    ctx->launches += 2;
    GIFT_CUDA(cudaMemcpyAsync(&add, off.p + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    GIFT_CUDA(cudaStreamSynchronize(st));
  } else {
    GIFT_CUDA(cudaMemsetAsync(off.p, 0, (n + 1) * sizeof(int64_t), st));
  }
  Csr* o = new gift_csr();
  o->device = ctx->device;
  o->n = n;
  o->nnz = c->nnz + add;
  o->indptr = static_cast<int64_t*>(csr_alloc(ctx, o, (n + 1) * sizeof(int64_t)));
  o->indices = static_cast<int32_t*>(csr_alloc(ctx, o, (o->nnz > 0 ? o->nnz : 1) * sizeof(int32_t)));
  o->values = static_cast<double*>(csr_alloc(ctx, o, (o->nnz > 0 ? o->nnz : 1) * sizeof(double)));
  o->has_diagonal = c->has_diagonal || sigma > 0;
  o->mean_row = n > 0 ? (double)o->nnz / n : 0.0;
  k_shift_ptr<<<grid_for(n + 1, kBlock), kBlock, 0, st>>>(n + 1, c->indptr, off.p, o->indptr);
  GIFT_LAUNCH_CHECK(ctx);
  if (n > 0) {
    k_normalized_fill<<<grid_for(n, kBlock), kBlock, 0, st>>>(n, c->indptr, c->indices, c->values, s, sigma,
                                                              o->indptr, o->indices, o->values);
    GIFT_LAUNCH_CHECK(ctx);
  }
  return o;
}

void csr_matmul(Ctx* ctx, const Csr* c, int64_t ncols, const double* x, double* y) {
  if (c->n == 0 || ncols == 0) return;
  DevBuf<double> extra(ctx, c->hf.nets ? c->n * 4 : 0);
  for (int64_t c0 = 0; c0 < ncols; c0 += 4) {
    const int nc = (int)std::min<int64_t>(4, ncols - c0);
    if (c->hf.nets) {
      GIFT_CUDA(cudaMemsetAsync(extra.p, 0, c->n * 4 * sizeof(double), ctx->stream));
      hf_apply_f64(ctx, c, nc, x, ncols, c0, nullptr, extra.p);
    }
    k_matvec_exact<0><<<grid_for(c->n, kBlock, 1LL << 30), kBlock, 0, ctx->stream>>>(
        c->n, c->indptr, c->indices, c->values, nullptr, 0.0, ncols, c0, nc, x, y, c->hf.nets ? extra.p : nullptr);
    GIFT_LAUNCH_CHECK(ctx);
  }
}

// ---------------------------------------------------------------------------
// Bank planning shared by both precisions: terms grouped by sigma in
// first-appearance order, each group's terms sorted by k (stable), as
// gift.py:83-93 does.
struct TermGroup {
  double sigma;
  std::vector<std::pair<int64_t, double>> terms;  // (k, alpha), stable-sorted by k
  int64_t maxk;
};

static std::vector<TermGroup> plan_groups(int n_terms, const double* sigma, const int64_t* k, const double* alpha) {
  if (n_terms <= 0) throw_error(GIFT_ERR_VALUE, "filter needs at least one term");
  std::vector<TermGroup> groups;
  for (int t = 0; t < n_terms; ++t) {
    if (!(sigma[t] >= 0)) throw_error(GIFT_ERR_VALUE, "sigma must be >= 0, got " + std::to_string(sigma[t]));
    if (k[t] < 1) throw_error(GIFT_ERR_VALUE, "power k must be >= 1, got " + std::to_string(k[t]));
    auto it = std::find_if(groups.begin(), groups.end(), [&](const TermGroup& g) { return g.sigma == sigma[t]; });
    if (it == groups.end()) {
      groups.push_back({sigma[t], {}, 0});
      it = groups.end() - 1;
    }
    it->terms.push_back({k[t], alpha[t]});
  }
  for (auto& g : groups) {
    std::stable_sort(g.terms.begin(), g.terms.end(),
                     [](const std::pair<int64_t, double>& a, const std::pair<int64_t, double>& b) {
                       return a.first < b.first;
                     });
    g.maxk = g.terms.back().first;
  }
  return groups;
}

// GIFT_PREC_FP64_EXACT: the reference's operation order, bit for bit.
static void bank_fp64_exact(Ctx* ctx, Csr* c, const std::vector<TermGroup>& groups, int64_t ncols, int in_dtype,
                            const void* g, int out_dtype, void* out, const uint8_t* fixed_mask,
                            const double* fixed_pos, const double* region) {
  cudaStream_t st = ctx->stream;
  const int64_t n = c->n, m = n * ncols;
  for (auto& grp : groups) csr_scale(ctx, c, grp.sigma);  // raise before any work, like the reference would
  if (m == 0) return;
  DevBuf<double> x(ctx, m), pa(ctx, m), pb(ctx, m), acc(ctx, m);
  DevBuf<double> extra(ctx, c->hf.nets ? n * 4 : 0);  // implicit high-fanout term (not in the reference)
  k_load_f64<<<grid_for(m, kBlock), kBlock, 0, st>>>(m, in_dtype, g, x.p);
  GIFT_LAUNCH_CHECK(ctx);
  GIFT_CUDA(cudaMemsetAsync(acc.p, 0, m * sizeof(double), st));
  for (auto& grp : groups) {
    const double* s = c->s64[grp.sigma];
    const double* power = x.p;
    int64_t done = 0;
    for (auto& term : grp.terms) {
      for (int64_t h = done; h < term.first; ++h) {
        double* dst = (power == pa.p) ? pb.p : pa.p;
        for (int64_t c0 = 0; c0 < ncols; c0 += 4) {
          const int nc = (int)std::min<int64_t>(4, ncols - c0);
          if (c->hf.nets) {
            GIFT_CUDA(cudaMemsetAsync(extra.p, 0, n * 4 * sizeof(double), st));
            hf_apply_f64(ctx, c, nc, power, ncols, c0, s, extra.p);
          }
          k_matvec_exact<1><<<grid_for(n, kBlock, 1LL << 30), kBlock, 0, st>>>(
              n, c->indptr, c->indices, c->values, s, grp.sigma, ncols, c0, nc, power, dst,
              c->hf.nets ? extra.p : nullptr);
          GIFT_LAUNCH_CHECK(ctx);
        }
        power = dst;
      }
      done = std::max(done, term.first);
      k_axpy_exact<<<grid_for(m, kBlock), kBlock, 0, st>>>(m, term.second, power, acc.p);
      GIFT_LAUNCH_CHECK(ctx);
    }
  }
  Region4 reg{};
  if (region) memcpy(reg.v, region, sizeof(reg.v));
  k_epilogue_f64<<<grid_for(m, kBlock), kBlock, 0, st>>>(n, ncols, acc.p, fixed_mask, fixed_pos, reg, out_dtype, out);
  GIFT_LAUNCH_CHECK(ctx);
}


// ---- the fp32 bank as a sequence of ops ------------------------------------
// A PREP op writes z0 = s o g for the chains of one pack; a HOP op advances
// every chain packed in zin by one hop (epilogue: next z, term accumulation,
// final re-pin / clamp).  bank_fp32 plans the ops, then either launches them
// one by one (tiled or row kernel per hop) or, for small graphs, runs them all
// in ONE cooperative kernel with a grid-wide barrier between ops.
struct BankOp {
  int kind;  // 0 = prep, 1 = hop
  int F;     // prep: floats per row written
  int fin, fout;
  PrepArgs p;
  HopArgs a;
};
constexpr int kMaxFusedOps = 10;
struct FusedBank {
  int nops;
  BankOp op[kMaxFusedOps];
};

template <int G>
__device__ __forceinline__ void fused_hop(const HopArgs& a, int fin, int fout, int64_t gi) {
#define GIFT_FUSED_CASE(FI, FO) \
  if (fin == FI && fout == FO) { \
    hop_row<FI, FO, G, 1>(a, gi);  \
    return;                        \
  }
  GIFT_FUSED_CASE(4, 4) GIFT_FUSED_CASE(4, 2) GIFT_FUSED_CASE(4, 1) GIFT_FUSED_CASE(4, 0)
  GIFT_FUSED_CASE(2, 2) GIFT_FUSED_CASE(2, 1) GIFT_FUSED_CASE(2, 0) GIFT_FUSED_CASE(2, 4)
  GIFT_FUSED_CASE(1, 1) GIFT_FUSED_CASE(1, 0) GIFT_FUSED_CASE(1, 2) GIFT_FUSED_CASE(1, 4)
#undef GIFT_FUSED_CASE
}

// the whole bank of a small (launch-bound, L2-resident) graph in one launch
template <int G>
__global__ void __launch_bounds__(kBlock) k_bank_fused(const __grid_constant__ FusedBank fb) {
  cg::grid_group grid = cg::this_grid();
  const int64_t tid = blockIdx.x * (int64_t)kBlock + threadIdx.x;
  const int64_t nthreads = (int64_t)gridDim.x * kBlock;
  for (int o = 0; o < fb.nops; ++o) {
    const BankOp& op = fb.op[o];
    if (op.kind == 0) {
      for (int64_t i = tid; i < op.p.n; i += nthreads) {
        if (op.F == 4) prep_row<4>(op.p, i);
        else if (op.F == 2) prep_row<2>(op.p, i);
        else prep_row<1>(op.p, i);
      }
    } else {
      // row groups of G lanes, grid-strided (uniform per group)
      for (int64_t gi = tid / G; gi < op.a.n; gi += nthreads / G) fused_hop<G>(op.a, op.fin, op.fout, gi);
    }
    if (o + 1 < fb.nops) grid.sync();
  }
}

// measured on B200 (profiles/r01_sweep_hop.txt): 8 lanes per row at mean
// row length ~64 (c1), 16 at ~400 (c2/c3); one 4-nnz chunk in flight per lane
static int pick_group_lanes(double mean_row) {
  if (mean_row < 160) return 8;
  return 16;
}

// graphs this small run the bank fused (one cooperative launch); above it the
// per-op launches (replayed as a CUDA graph below the tiled threshold) win:
// c0 (0.66M entries) 0.052 -> 0.042 ms per bank, c1 (13.6M) 0.28 -> 0.32 ms
constexpr int64_t kFusedMaxNnz = 1LL << 21;

// lanes per row of the fp32 bank's row-kernel hops.  Small graphs (the fused
// regime) are latency-bound: a lane streams about one 4-entry chunk, so a hop
// is one load round trip (c0, mean row 64: 16 lanes; 8 lanes took 54 us per
// fused bank, 16 take 39 us).  Larger graphs keep the throughput-tuned
// choice.  The same rule serves fused, graph-replayed and direct launches, so
// they agree bit for bit.
static int bank_lanes(Ctx* ctx, const Csr* c) {
  if (ctx->opt.row_lanes) return (int)ctx->opt.row_lanes;
  if (c->nnz <= kFusedMaxNnz) return std::min(32, std::max(8, pow2_ceil((int)(c->mean_row / 4.0 + 0.5))));
  return pick_group_lanes(c->mean_row);
}

static bool launch_fused(Ctx* ctx, Csr* c, const std::vector<BankOp>& ops, int G) {
  if ((int)ops.size() > kMaxFusedOps || !ctx->opt.fused || c->nnz > kFusedMaxNnz || c->hf.nets ||
      bmt_possible(ctx, c) || ctx->profiling)
    return false;
  FusedBank fb{};
  fb.nops = (int)ops.size();
  for (size_t i = 0; i < ops.size(); ++i) fb.op[i] = ops[i];
  void* kern = G == 32 ? (void*)k_bank_fused<32> : G == 16 ? (void*)k_bank_fused<16> : (void*)k_bank_fused<8>;
  static std::mutex mu;
  static std::map<std::pair<void*, int>, int> grid_of;  // co-resident CTAs (x SMs) per (kernel, device)
  int grid = 0;
  {
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_pair(kern, ctx->device);
    auto it = grid_of.find(key);
    if (it == grid_of.end()) {
      int per_sm = 0;
      GIFT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBlock, 0));
      grid = std::max(per_sm, 1) * ctx->num_sms;
      grid_of[key] = grid;
    } else {
      grid = it->second;
    }
  }
  void* args[] = {&fb};
  GIFT_CUDA(cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(kBlock), args, 0, ctx->stream));
  GIFT_LAUNCH_CHECK(ctx);
  c->fp32_hops += (int64_t)ops.size();
  return true;
}

// ops bank_fp32 plans: per column slice, per pack of chains, one prep + its longest chain's hops
static int64_t bank_ops(const std::vector<TermGroup>& groups, int64_t ncols) {
  int64_t ops = 0;
  for (int64_t c0 = 0; c0 < ncols; c0 += 4) {
    const int per = std::max(1, 4 / (int)std::min<int64_t>(4, ncols - c0));
    for (size_t g0 = 0; g0 < groups.size(); g0 += per) {
      int64_t maxk = 0;
      for (size_t j = g0; j < std::min(groups.size(), g0 + per); ++j) maxk = std::max(maxk, groups[j].maxk);
      ops += 1 + maxk;
    }
  }
  return ops;
}

// GIFT_PREC_FP32: fused pre-scaled bank.
static void bank_fp32(Ctx* ctx, Csr* c, const std::vector<TermGroup>& groups, int64_t ncols, int in_dtype,
                      const void* g, int out_dtype, void* out, const uint8_t* fixed_mask, const double* fixed_pos,
                      const double* region) {
  const int64_t n = c->n;
  for (auto& grp : groups) csr_scale(ctx, c, grp.sigma);
  if (n == 0 || ncols == 0) return;
  const float* w = csr_w32(ctx, c);
  const int G = bank_lanes(ctx, c);
  Region4 reg{};
  if (region) memcpy(reg.v, region, sizeof(reg.v));
  float* zA = static_cast<float*>(scratch(ctx, 0, n * 4 * sizeof(float) + 64));
  float* zB = static_cast<float*>(scratch(ctx, 1, n * 4 * sizeof(float) + 64));
  float* accb = static_cast<float*>(scratch(ctx, 2, n * 4 * sizeof(float) + 64));
  std::vector<BankOp> ops;
  // column slices of <= 4 columns; chains of a slice packed <= 4 floats per row
  for (int64_t c0 = 0; c0 < ncols; c0 += 4) {
    const int wcols = (int)std::min<int64_t>(4, ncols - c0);
    const int per = std::max(1, 4 / wcols);
    bool acc_written = false;
    for (size_t g0 = 0; g0 < groups.size(); g0 += per) {
      const int nch = (int)std::min<size_t>(per, groups.size() - g0);
      const bool last_pack = g0 + nch >= groups.size();
      BankOp prep{};
      prep.kind = 0;
      prep.F = pow2_ceil(wcols * nch);
      prep.p = PrepArgs{n, wcols, nch, {nullptr, nullptr, nullptr, nullptr}, in_dtype, g, ncols, c0, zA};
      int64_t maxk = 0;
      for (int j = 0; j < nch; ++j) {
        prep.p.s[j] = c->s32[groups[g0 + j].sigma];
        maxk = std::max(maxk, groups[g0 + j].maxk);
      }
      ops.push_back(prep);
      // active chains (indices into groups) in packing order
      std::vector<int> active;
      for (int j = 0; j < nch; ++j) active.push_back((int)g0 + j);
      float* zin = zA;
      float* zout = zB;
      for (int64_t h = 1; h <= maxk; ++h) {
        HopArgs a{};
        a.rowptr = c->indptr;
        a.col = c->indices;
        a.w = w;
        a.n = n;
        a.zin = zin;
        a.zout = zout;
        a.wcols = wcols;
        a.nch = (int)active.size();
        std::vector<int> next;
        for (size_t j = 0; j < active.size(); ++j) {
          const TermGroup& grp = groups[active[j]];
          ChainArgs& ch = a.ch[j];
          ch.s = c->s32[grp.sigma];
          ch.sigma = (float)grp.sigma;
          double al = 0.0;
          int has = 0;
          for (auto& t : grp.terms)
            if (t.first == h) {
              al += t.second;
              has = 1;
            }
          ch.has_term = has;
          ch.alpha = (float)al;
          a.any_term |= has;
          if (grp.maxk > h) {
            ch.cont = (int)next.size();
            next.push_back(active[j]);
          } else {
            ch.cont = -1;
          }
        }
        BankOp hop{};
        hop.kind = 1;
        hop.fin = pow2_ceil(wcols * (int)active.size());
        hop.fout = next.empty() ? 0 : pow2_ceil(wcols * (int)next.size());
        a.acc = accb;
        a.acc_read = acc_written ? 1 : 0;
        a.is_final = (last_pack && h == maxk) ? 1 : 0;
        a.out_dtype = out_dtype;
        a.out = out;
        a.out_ld = ncols;
        a.out_c0 = c0;
        a.fixed_mask = fixed_mask;
        a.fixed_pos = fixed_pos;
        a.reg = reg;
        hop.a = a;
        ops.push_back(hop);
        if (a.any_term) acc_written = true;
        active.swap(next);
        std::swap(zin, zout);
      }
    }
  }
  if (launch_fused(ctx, c, ops, G)) return;
  for (BankOp& op : ops) {
    if (op.kind == 0) {
      ProfScope prof(ctx, 0, op.p.nch);
      const unsigned grid = grid_for(n, kBlock, 1LL << 30);
      switch (op.F) {
        case 1: k_prep<1><<<grid, kBlock, 0, ctx->stream>>>(op.p); break;
        case 2: k_prep<2><<<grid, kBlock, 0, ctx->stream>>>(op.p); break;
        default:
          if (prep_is_default_pack(op.p))
            k_prep4_rows<<<grid_for((n + 3) / 4, kBlock, 1LL << 30), kBlock, 0, ctx->stream>>>(op.p);
          else
            k_prep<4><<<grid, kBlock, 0, ctx->stream>>>(op.p);
          break;
      }
      GIFT_LAUNCH_CHECK(ctx);
      continue;
    }
    if (c->hf.nets) {
      if (fact_hop_applies(ctx, c, op.a, op.fin)) {  // factored clique model: two O(pins) kernels
        ProfScope prof(ctx, op.fin, op.a.nch);
        fact_hop_f32(ctx, c, op.a, op.fin, op.fout);
        c->fp32_hops++;
        continue;
      }
      // implicit high-fanout term: its row sums enter the hop as partial sums
      float* part = static_cast<float*>(scratch(ctx, 3, n * 4 * sizeof(float) + 64));
      GIFT_CUDA(cudaMemsetAsync(part, 0, n * op.fin * sizeof(float), ctx->stream));
      hf_apply_f32(ctx, c, op.fin, op.a.zin, part);
      op.a.part_in = part;
    }
    launch_hop(ctx, c, op.a, op.fin, op.fout, G, true);
  }
}

// ---- stepped building blocks for host-driven (sharded) banks ----------------
void scale_vectors(Ctx* ctx, Csr* c, double sigma, const double** s64, const float** s32) {
  const double* s = csr_scale(ctx, c, sigma);
  if (s64) *s64 = s;
  if (s32) *s32 = c->s32[sigma];
}

const float* weights32(Ctx* ctx, Csr* c) { return csr_w32(ctx, c); }

void hop_fp32(Ctx* ctx, Csr* c, const gift_hop_desc* d) {
  if (c->hf.nets) throw_error(GIFT_ERR_VALUE, "the stepped (sharded) hop does not support the high-fanout term");
  if (d->fin != 1 && d->fin != 2 && d->fin != 4) throw_error(GIFT_ERR_VALUE, "fin must be 1, 2 or 4");
  if (d->fout != 0 && d->fout != 1 && d->fout != 2 && d->fout != 4) throw_error(GIFT_ERR_VALUE, "bad fout");
  if (d->nch < 1 || d->nch > 4 || d->wcols < 1 || d->wcols * d->nch > d->fin)
    throw_error(GIFT_ERR_VALUE, "bad chain packing");
  if (d->row_begin < 0 || d->row_end > c->n || d->row_begin > d->row_end) throw_error(GIFT_ERR_VALUE, "bad row range");
  HopArgs a{};
  a.rowptr = c->indptr;
  a.col = c->indices;
  a.w = csr_w32(ctx, c);
  a.n = d->row_end;
  a.row_begin = d->row_begin;
  a.part_in = d->part_in;
  a.part_out = d->part_out;
  a.zin = d->zin;
  a.zout = d->zout;
  a.wcols = d->wcols;
  a.nch = d->nch;
  for (int j = 0; j < d->nch; ++j) {
    a.ch[j].s = d->chain[j].s;
    a.ch[j].sigma = (float)d->chain[j].sigma;
    a.ch[j].cont = d->chain[j].cont;
    a.ch[j].has_term = d->chain[j].has_term;
    a.ch[j].alpha = (float)d->chain[j].alpha;
    a.any_term |= d->chain[j].has_term;
  }
  a.acc = d->acc;
  a.acc_read = d->acc_read;
  a.is_final = d->is_final;
  a.out_dtype = d->out_dtype;
  a.out = d->out;
  a.out_ld = d->out_ld;
  a.out_c0 = d->out_c0;
  a.fixed_mask = d->fixed_mask;
  a.fixed_pos = d->fixed_pos;
  memcpy(a.reg.v, d->region, sizeof(a.reg.v));
  // the tiled hop serves whole square blocks (a shard's local part, which may
  // write partial sums); the ghost part (part_in) stays on the row kernel
  const bool tiled = a.row_begin == 0 && a.n == c->n && !a.part_in;
  launch_hop(ctx, c, a, d->fin, d->fout, pick_group_lanes(c->mean_row), tiled);
}

void pack_fp32(Ctx* ctx, int64_t n, int wcols, int nch, const float* const* s, int in_dtype, const void* g,
               int64_t ld, int64_t c0, int F, float* z) {
  if (n <= 0) return;
  ProfScope prof(ctx, 0, nch);
  const float* sp[4] = {nullptr, nullptr, nullptr, nullptr};
  for (int j = 0; j < nch && j < 4; ++j) sp[j] = s[j];
  const unsigned grid = grid_for(n, kBlock, 1LL << 30);
  const PrepArgs p{n, wcols, nch, {sp[0], sp[1], sp[2], sp[3]}, in_dtype, g, ld, c0, z};
  switch (F) {
    case 1: k_prep<1><<<grid, kBlock, 0, ctx->stream>>>(p); break;
    case 2: k_prep<2><<<grid, kBlock, 0, ctx->stream>>>(p); break;
    case 4: k_prep<4><<<grid, kBlock, 0, ctx->stream>>>(p); break;
    default: throw_error(GIFT_ERR_VALUE, "F must be 1, 2 or 4");
  }
  GIFT_LAUNCH_CHECK(ctx);
}

void gather_rows_f32(Ctx* ctx, int64_t n_idx, int F, const int64_t* idx, const float* src, float* dst) {
  if (n_idx <= 0) return;
  k_gather_rows<<<grid_for(n_idx * F, kBlock), kBlock, 0, ctx->stream>>>(n_idx, F, idx, src, dst);
  GIFT_LAUNCH_CHECK(ctx);
}

// bit 0: some row has a column descent; bit 1: some column >= n_rows (not square)
__global__ void k_block_shape(int64_t n, const int64_t* __restrict__ indptr, const int32_t* __restrict__ col,
                              int* __restrict__ flags) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    int f = 0;
    for (int64_t k = indptr[r]; k < indptr[r + 1]; ++k) {
      if (k > indptr[r] && col[k] < col[k - 1]) f |= 1;
      if (col[k] < 0 || (int64_t)col[k] >= n) f |= 2;
    }
    if (f) atomicOr(flags, f);
  }
}

Csr* csr_from_arrays(Ctx* ctx, int64_t n_rows, int64_t nnz, const int64_t* d_indptr, const int32_t* d_indices,
                     const double* d_values) {
  Csr* c = new gift_csr();
  c->device = ctx->device;
  c->n = n_rows;
  c->nnz = nnz;
  c->indptr = static_cast<int64_t*>(csr_alloc(ctx, c, (n_rows + 1) * sizeof(int64_t)));
  c->indices = static_cast<int32_t*>(csr_alloc(ctx, c, (nnz > 0 ? nnz : 1) * sizeof(int32_t)));
  c->values = static_cast<double*>(csr_alloc(ctx, c, (nnz > 0 ? nnz : 1) * sizeof(double)));
  c->mean_row = n_rows > 0 ? (double)nnz / n_rows : 0.0;
  c->has_diagonal = true;
  GIFT_CUDA(cudaMemcpyAsync(c->indptr, d_indptr, (n_rows + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, ctx->stream));
  if (nnz > 0) {
    GIFT_CUDA(cudaMemcpyAsync(c->indices, d_indices, nnz * sizeof(int32_t), cudaMemcpyDeviceToDevice, ctx->stream));
    GIFT_CUDA(cudaMemcpyAsync(c->values, d_values, nnz * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  }
  // a shard's local block (owned columns, remapped in order) is square with
  // ascending columns and can take the tiled hop; ghost blocks cannot
  DevBuf<int> flags(ctx, 1);
  GIFT_CUDA(cudaMemsetAsync(flags.p, 0, sizeof(int), ctx->stream));
  if (n_rows > 0) {
    k_block_shape<<<grid_for(n_rows, kBlock), kBlock, 0, ctx->stream>>>(n_rows, c->indptr, c->indices, flags.p);
    GIFT_LAUNCH_CHECK(ctx);
  }
  int h = 0;
  GIFT_CUDA(cudaMemcpyAsync(&h, flags.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  GIFT_CUDA(cudaStreamSynchronize(ctx->stream));
  c->sorted_rows = (h & 1) == 0;
  c->square = (h & 2) == 0;
  return c;
}

// ---------------------------------------------------------------------------
// Small graphs are launch-bound (c0: ~5 MB per hop, L2-resident; the bank's
// 6-8 launches plus the host's planning cost more than the hops).  Their fp32
// bank is captured once per (graph, terms, widths, dtypes, epilogue) as a CUDA
// graph over staged buffers and replayed: copy in, one graph launch, copy out.
constexpr int64_t kGraphMaxRows = 262144;  // below the tiled hop's size threshold
constexpr size_t kMaxGraphs = 8;

static uint64_t next_uid() {
  static std::atomic<uint64_t> u{0};
  return ++u;
}

static void free_bank_graph(Ctx* ctx, Ctx::BankGraph& e) {
  if (e.exec) cudaGraphExecDestroy(e.exec);
  dev_free(ctx, e.gin);
  dev_free(ctx, e.gout);
  dev_free(ctx, e.gmask);
  dev_free(ctx, e.gpos);
  e = Ctx::BankGraph{};
}

void free_bank_graphs(Ctx* ctx) {
  for (auto& e : ctx->graphs) free_bank_graph(ctx, e);
  ctx->graphs.clear();
}

static bool bank_graph(Ctx* ctx, Csr* c, const std::vector<TermGroup>& groups, int n_terms, const double* sigma,
                       const int64_t* k, const double* alpha, int64_t ncols, int in_dtype, const void* g,
                       int out_dtype, void* out, const uint8_t* fixed_mask, const double* fixed_pos,
                       const double* region) {
  if (ctx->profiling || c->n <= 0 || c->n >= kGraphMaxRows || ncols <= 0 || !ctx->opt.graphs)
    return false;
  if (bmt_possible(ctx, c)) return false;  // a tiled-copy build cannot run inside a capture
  // the fused cooperative kernel (bank_fp32) is a single launch already
  if (ctx->opt.fused && c->nnz <= kFusedMaxNnz && !c->hf.nets && bank_ops(groups, ncols) <= kMaxFusedOps) return false;
  const int64_t n = c->n;
  const size_t in_b = (size_t)(n * ncols) * (in_dtype == GIFT_DTYPE_F64 ? 8 : 4);
  const size_t out_b = (size_t)(n * ncols) * (out_dtype == GIFT_DTYPE_F64 ? 8 : 4);
  std::vector<double> key = {(double)n_terms, (double)ncols, (double)in_dtype, (double)out_dtype,
                             fixed_mask ? 1.0 : 0.0};
  for (int t = 0; t < n_terms; ++t) {
    key.push_back(sigma[t]);
    key.push_back((double)k[t]);
    key.push_back(alpha[t]);
  }
  if (fixed_mask)
    for (int i = 0; i < 4; ++i) key.push_back(region[i]);
  if (!c->uid) c->uid = next_uid();
  size_t hit = ctx->graphs.size();
  for (size_t i = 0; i < ctx->graphs.size(); ++i)
    if (ctx->graphs[i].uid == c->uid && ctx->graphs[i].key.size() == key.size() &&
        memcmp(ctx->graphs[i].key.data(), key.data(), key.size() * sizeof(double)) == 0)
      hit = i;
  if (hit == ctx->graphs.size()) {
    // everything that may synchronise or allocate happens before the capture
    for (auto& grp : groups) csr_scale(ctx, c, grp.sigma);
    csr_w32(ctx, c);
    for (int slot = 0; slot < 3; ++slot) scratch(ctx, slot, n * 4 * sizeof(float) + 64);
    if (c->hf.nets) scratch(ctx, 3, n * 4 * sizeof(float) + 64);
    Ctx::BankGraph e;
    e.uid = c->uid;
    e.key = key;
    e.gin = dev_alloc(ctx, in_b);
    e.gout = dev_alloc(ctx, out_b);
    if (fixed_mask) {
      e.gmask = static_cast<uint8_t*>(dev_alloc(ctx, n));
      e.gpos = static_cast<double*>(dev_alloc(ctx, 2 * n * sizeof(double)));
    }
    if (!ctx->cap_stream) GIFT_CUDA(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
    // the capture stream must see the buffers' allocations (stream-ordered pool)
    cudaEvent_t ready;
    GIFT_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    GIFT_CUDA(cudaEventRecord(ready, ctx->stream));
    GIFT_CUDA(cudaStreamWaitEvent(ctx->cap_stream, ready, 0));
    GIFT_CUDA(cudaStreamSynchronize(ctx->cap_stream));
    cudaEventDestroy(ready);
    cudaStream_t user = ctx->stream;
    const int64_t l0 = ctx->launches;
    cudaGraph_t graph = nullptr;
    ctx->stream = ctx->cap_stream;
    try {
      GIFT_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
      bank_fp32(ctx, c, groups, ncols, in_dtype, e.gin, out_dtype, e.gout, e.gmask, e.gpos, region);
      GIFT_CUDA(cudaStreamEndCapture(ctx->stream, &graph));
      GIFT_CUDA(cudaGraphInstantiate(&e.exec, graph, 0));
    } catch (...) {
      cudaGraph_t dummy = nullptr;
      cudaStreamEndCapture(ctx->stream, &dummy);
      if (dummy) cudaGraphDestroy(dummy);
      if (graph) cudaGraphDestroy(graph);
      cudaGetLastError();
      ctx->stream = user;
      free_bank_graph(ctx, e);
      throw;
    }
    ctx->stream = user;
    cudaGraphDestroy(graph);
    e.kernels = ctx->launches - l0;
    ctx->launches = l0;
    if (ctx->graphs.size() >= kMaxGraphs) {
      free_bank_graph(ctx, ctx->graphs.front());
      ctx->graphs.erase(ctx->graphs.begin());
    }
    ctx->graphs.push_back(std::move(e));
    hit = ctx->graphs.size() - 1;
  } else if (hit + 1 != ctx->graphs.size()) {  // most recent last
    Ctx::BankGraph e = std::move(ctx->graphs[hit]);
    ctx->graphs.erase(ctx->graphs.begin() + hit);
    ctx->graphs.push_back(std::move(e));
    hit = ctx->graphs.size() - 1;
  }
  Ctx::BankGraph& e = ctx->graphs[hit];
  cudaStream_t st = ctx->stream;
  GIFT_CUDA(cudaMemcpyAsync(e.gin, g, in_b, cudaMemcpyDefault, st));
  if (fixed_mask) {
    GIFT_CUDA(cudaMemcpyAsync(e.gmask, fixed_mask, n, cudaMemcpyDefault, st));
    GIFT_CUDA(cudaMemcpyAsync(e.gpos, fixed_pos, 2 * n * sizeof(double), cudaMemcpyDefault, st));
  }
  GIFT_CUDA(cudaGraphLaunch(e.exec, st));
  GIFT_CUDA(cudaMemcpyAsync(out, e.gout, out_b, cudaMemcpyDefault, st));
  ctx->launches += e.kernels;
  c->fp32_hops += 4;
  return true;
}

void filter(Ctx* ctx, Csr* c, int n_terms, const double* sigma, const int64_t* k, const double* alpha, int64_t ncols,
            int in_dtype, const void* g, int out_dtype, void* out, const uint8_t* fixed_mask, const double* fixed_pos,
            const double* region, int precision) {
  if (ncols < 0) throw_error(GIFT_ERR_DIMENSION, "negative column count");
  if (fixed_mask && ncols != 2) throw_error(GIFT_ERR_DIMENSION, "the placement epilogue needs an N x 2 signal");
  if (fixed_mask && !region) throw_error(GIFT_ERR_VALUE, "region required with a fixed mask");
  if (in_dtype != GIFT_DTYPE_F32 && in_dtype != GIFT_DTYPE_F64) throw_error(GIFT_ERR_VALUE, "bad input dtype");
  if (out_dtype != GIFT_DTYPE_F32 && out_dtype != GIFT_DTYPE_F64) throw_error(GIFT_ERR_VALUE, "bad output dtype");
  auto groups = plan_groups(n_terms, sigma, k, alpha);
  if (precision == GIFT_PREC_FP64_EXACT)
    bank_fp64_exact(ctx, c, groups, ncols, in_dtype, g, out_dtype, out, fixed_mask, fixed_pos, region);
  else if (precision == GIFT_PREC_FP32) {
    if (!bank_graph(ctx, c, groups, n_terms, sigma, k, alpha, ncols, in_dtype, g, out_dtype, out, fixed_mask,
                    fixed_pos, region))
      bank_fp32(ctx, c, groups, ncols, in_dtype, g, out_dtype, out, fixed_mask, fixed_pos, region);
  } else
    throw_error(GIFT_ERR_VALUE, "unknown precision");
}

}  // namespace gift
