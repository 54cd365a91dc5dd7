// hop.cuh -- pieces shared by the fp32 hop kernels (filter.cu row kernel,
// bmt.cu block-major tiled kernel): the hop descriptor, cached-load helpers
// and the fused row epilogue (next-hop signal, term accumulation, gift_place
// re-pin / clamp).
#pragma once

#include <stdint.h>

#include <cstdlib>

#include "common.cuh"

namespace gift {

// environment knobs of -DGIFT_TUNING builds (tools/ sweeps); the default
// build takes its options from gift_ctx_set_option only
inline int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}

// np.clip for floats: MIN(MAX(x, lo), hi), NaN passes, PyArray_MAX(a,b) = a > b ? a : b
__device__ __forceinline__ double np_clip(double x, double lo, double hi) {
  double t = isnan(x) ? x : (x > lo ? x : lo);
  return isnan(t) ? t : (t < hi ? t : hi);
}

struct Region4 {
  double v[4];
};

// ---- fp32 fused hop ---------------------------------------------------------
struct ChainArgs {
  const float* s;  // fp32 s_sigma
  float sigma;
  int cont;        // slot of this chain in zout, -1 if the chain ends here
  int has_term;    // a term of this chain completes at this hop
  float alpha;     // its weight (sum if several terms share k)
};

struct HopArgs {
  const int64_t* rowptr;
  const int32_t* col;
  const float* w;
  int64_t n;          // one past the last row processed
  int64_t row_begin;  // first row processed
  const int32_t* row_list;  // when set: process rows row_list[row_begin .. n) instead of [row_begin, n)
  const float* part_in;  // [rows, FIN] partial sums added before the epilogue (split hop), or null
  float* part_out;       // write the raw row sums here and skip the epilogue (split hop), or null
  const float* zin;  // [n, FIN]
  float* zout;       // [n, FOUT]
  int wcols;         // signal columns per chain
  int nch;           // chains packed in zin
  ChainArgs ch[4];
  float* acc;        // [n, wcols] fp32 bank accumulator
  int acc_read;      // 0: first write (out = zeros + ...)
  int is_final;
  int out_dtype;
  void* out;
  int64_t out_ld;
  int64_t out_c0;
  const uint8_t* fixed_mask;
  const double* fixed_pos;
  Region4 reg;
  int any_term;
};

template <int F>
struct VecF;
template <>
struct VecF<1> {
  float v[1];
};
template <>
struct VecF<2> {
  float v[2];
};
template <>
struct VecF<4> {
  float v[4];
};

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// gathered signal rows: L1-allocating, keep in L2
template <int F>
__device__ __forceinline__ VecF<F> ld_z(const float* p, uint64_t pol);
template <>
__device__ __forceinline__ VecF<1> ld_z<1>(const float* p, uint64_t pol) {
  VecF<1> r;
  asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(r.v[0]) : "l"(p), "l"(pol));
  return r;
}
template <>
__device__ __forceinline__ VecF<2> ld_z<2>(const float* p, uint64_t pol) {
  VecF<2> r;
  asm volatile("ld.global.nc.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;"
               : "=f"(r.v[0]), "=f"(r.v[1])
               : "l"(p), "l"(pol));
  return r;
}
template <>
__device__ __forceinline__ VecF<4> ld_z<4>(const float* p, uint64_t pol) {
  VecF<4> r;
  asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
               : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3])
               : "l"(p), "l"(pol));
  return r;
}

__device__ __forceinline__ int4 ld_stream_v4s32(const int32_t* p, uint64_t pol) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.b32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ float4 ld_stream_v4f32(const float* p, uint64_t pol) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p), "l"(pol));
  return r;
}

// Row epilogue shared by every hop kernel: y = s o (A z + sigma z) per packed
// chain; next-hop signal z' = s o y; completed terms accumulate alpha * y;
// the final hop re-pins fixed rows and clamps movable rows (gift.py:112-118).
template <int FIN, int FOUT>
__device__ __forceinline__ void row_epilogue(const HopArgs& a, int64_t row, float (&acc)[FIN], uint64_t pol_z) {
  if (a.part_out) {
#pragma unroll
    for (int f = 0; f < FIN; ++f) a.part_out[row * FIN + f] = acc[f];
    return;
  }
  if (a.part_in) {
#pragma unroll
    for (int f = 0; f < FIN; ++f) acc[f] = a.part_in[row * FIN + f] + acc[f];
  }
  const VecF<FIN> zi = ld_z<FIN>(a.zin + row * FIN, pol_z);
  float o[4] = {0.f, 0.f, 0.f, 0.f};
  if (a.any_term && a.acc_read)
    for (int cc = 0; cc < a.wcols; ++cc) o[cc] = a.acc[row * a.wcols + cc];
  float zo[FOUT > 0 ? FOUT : 1];
#pragma unroll
  for (int f = 0; f < (FOUT > 0 ? FOUT : 1); ++f) zo[f] = 0.f;
#pragma unroll
  for (int f = 0; f < FIN; ++f) {
    const int chn = f / a.wcols;
    if (chn >= a.nch) break;
    const int cc = f - chn * a.wcols;
    const ChainArgs& ch = a.ch[chn];
    const float si = ch.s[row];
    const float y = si * (acc[f] + ch.sigma * zi.v[f]);
    if (FOUT > 0 && ch.cont >= 0) zo[(ch.cont * a.wcols + cc) % (FOUT > 0 ? FOUT : 1)] = si * y;
    if (ch.has_term) o[cc] = fmaf(ch.alpha, y, o[cc]);
  }
  if constexpr (FOUT == 4) *reinterpret_cast<float4*>(a.zout + row * 4) = make_float4(zo[0], zo[1], zo[2], zo[3]);
  else if constexpr (FOUT == 2) *reinterpret_cast<float2*>(a.zout + row * 2) = make_float2(zo[0], zo[1]);
  else if constexpr (FOUT == 1) a.zout[row] = zo[0];
  if (!a.any_term) return;
  if (!a.is_final) {
    for (int cc = 0; cc < a.wcols; ++cc) a.acc[row * a.wcols + cc] = o[cc];
    return;
  }
  if (a.wcols == 2 && a.out_ld == 2 && a.out_dtype == GIFT_DTYPE_F64 && ((uintptr_t)a.out & 15) == 0) {
    // the common N x 2 placement: one 16-byte store per row (the output may be
    // mapped host memory, where full-width writes matter most)
    double v0 = (double)o[0], v1 = (double)o[1];
    if (a.fixed_mask) {
      if (a.fixed_mask[row]) {
        v0 = a.fixed_pos[row * 2];
        v1 = a.fixed_pos[row * 2 + 1];
      } else {
        v0 = np_clip(v0, a.reg.v[0], a.reg.v[2]);
        v1 = np_clip(v1, a.reg.v[1], a.reg.v[3]);
      }
    }
    reinterpret_cast<double2*>(a.out)[row] = make_double2(v0, v1);
    return;
  }
  if (a.wcols == 2 && a.out_ld == 2 && a.out_dtype == GIFT_DTYPE_F32 && ((uintptr_t)a.out & 7) == 0) {
    // N x 2 fp32 placement: one 8-byte store per row
    double v0 = (double)o[0], v1 = (double)o[1];
    if (a.fixed_mask) {
      if (a.fixed_mask[row]) {
        v0 = a.fixed_pos[row * 2];
        v1 = a.fixed_pos[row * 2 + 1];
      } else {
        v0 = np_clip(v0, a.reg.v[0], a.reg.v[2]);
        v1 = np_clip(v1, a.reg.v[1], a.reg.v[3]);
      }
    }
    reinterpret_cast<float2*>(a.out)[row] = make_float2(__double2float_rn(v0), __double2float_rn(v1));
    return;
  }
  for (int cc = 0; cc < a.wcols; ++cc) {
    double v = (double)o[cc];
    if (a.fixed_mask) v = a.fixed_mask[row] ? a.fixed_pos[row * 2 + cc] : np_clip(v, a.reg.v[cc], a.reg.v[cc + 2]);
    const int64_t oi = row * a.out_ld + a.out_c0 + cc;
    if (a.out_dtype == GIFT_DTYPE_F64) static_cast<double*>(a.out)[oi] = v;
    else static_cast<float*>(a.out)[oi] = __double2float_rn(v);
  }
}


struct Csr;
// block-major tiled hop (bmt.cu); false when not applicable -> caller uses the row kernel
bool bmt_hop(Ctx* ctx, Csr* c, const HopArgs& a, int fin, int fout);
// whether bmt_hop could ever serve (or build a tiled copy for) this graph
bool bmt_possible(Ctx* ctx, const Csr* c);

}  // namespace gift
