// plio.cu -- Bookshelf .pl writer on the device.
//
// Reference: write_placement, giftplace/netlist.py:503-522.  The text is
//   "UCLA pl 1.0\n\n" then one line per cell in cell order:
//   f"{name}\t{llx:.6f}\t{lly:.6f}\t: N{' /FIXED' if fixed else ''}\n"
// with llx = cx - width / 2.0, lly = cy - height / 2.0 in fp64
// (netlist.py:516-520, PL_PRECISION = 6 at :29).  Python's "%.6f" is the
// correctly rounded decimal of the exact binary value, ties to even, with
// the sign kept for negative zero and for negatives that round to zero
// ("-0.000000"), and "nan" / "inf" / "-inf" for non-finite values.
//
// Device layout: one thread per cell.  Pass 1 computes each line's byte
// length, a CUB exclusive scan turns lengths into offsets, pass 2 writes the
// bytes.  Byte work, HBM/latency bound; the text buffer is the only large
// allocation (~35-45 B per cell).
//
// Exact formatting: x = m * 2^e (m < 2^53).  N = round_half_even(|x| * 10^6)
// is computed exactly in 128-bit integers: a = m * 10^6 < 2^73, then a << e
// (e >= 0) or a >> -e with the shifted-out remainder deciding the rounding.
// |x| must be < 2^107 (~1.6e32) so a << e fits; larger finite values are
// rejected with GIFT_ERR_VALUE rather than printed wrong.
#include <cub/cub.cuh>

#include <climits>
#include <cstring>
#include <string>

#include "common.cuh"

namespace gift {

namespace {

constexpr int kBlock = 256;
constexpr char kHeader[] = "UCLA pl 1.0\n\n";
constexpr int kHeaderLen = sizeof(kHeader) - 1;
__constant__ char c_header[kHeaderLen + 1] = "UCLA pl 1.0\n\n";

typedef unsigned __int128 u128;

struct Fixed6 {
  bool neg;
  int kind;  // 0 finite, 1 nan, 2 inf
  u128 ip;   // integer part
  uint32_t fp;  // 6 fractional digits
  bool range_error;
};

__device__ __forceinline__ Fixed6 decompose(double x) {
  Fixed6 r{};
  const unsigned long long bits = (unsigned long long)__double_as_longlong(x);
  r.neg = (bits >> 63) != 0;
  const int E = (int)((bits >> 52) & 0x7ff);
  const unsigned long long frac = bits & ((1ull << 52) - 1);
  if (E == 0x7ff) {
    r.kind = frac ? 1 : 2;
    if (r.kind == 1) r.neg = false;  // Python prints "nan" whatever the sign bit
    return r;
  }
  const unsigned long long m = E ? (frac | (1ull << 52)) : frac;
  const int e = E ? E - 1075 : -1074;
  const u128 a = (u128)m * 1000000u;
  u128 q;
  if (e >= 0) {
    if (e > 54) {
      r.range_error = true;
      return r;
    }
    q = a << e;
  } else {
    const int s = -e;
    if (s >= 127) {
      q = 0;  // a < 2^73 <= half: rounds to zero
    } else {
      q = a >> s;
      const u128 rem = a & (((u128)1 << s) - 1);
      const u128 half = (u128)1 << (s - 1);
      if (rem > half || (rem == half && (q & 1))) ++q;
    }
  }
  r.ip = q / 1000000u;
  r.fp = (uint32_t)(q % 1000000u);
  return r;
}

__device__ __forceinline__ int udigits(u128 v) {
  int d = 1;
  while (v >= 10) {
    v /= 10;
    ++d;
  }
  return d;
}

__device__ __forceinline__ int fixed6_len(const Fixed6& f) {
  if (f.kind == 1) return 3;
  if (f.kind == 2) return f.neg ? 4 : 3;
  return (f.neg ? 1 : 0) + udigits(f.ip) + 7;
}

__device__ __forceinline__ char* put_udec(char* p, u128 v) {
  char tmp[40];
  int k = 0;
  do {
    tmp[k++] = (char)('0' + (int)(v % 10));
    v /= 10;
  } while (v);
  while (k) *p++ = tmp[--k];
  return p;
}

__device__ __forceinline__ char* put_fixed6(char* p, const Fixed6& f) {
  if (f.kind == 1) {
    p[0] = 'n'; p[1] = 'a'; p[2] = 'n';
    return p + 3;
  }
  if (f.neg) *p++ = '-';
  if (f.kind == 2) {
    p[0] = 'i'; p[1] = 'n'; p[2] = 'f';
    return p + 3;
  }
  p = put_udec(p, f.ip);
  *p++ = '.';
  uint32_t v = f.fp;
  for (int i = 5; i >= 0; --i) {
    p[i] = (char)('0' + v % 10);
    v /= 10;
  }
  return p + 6;
}

struct PlArgs {
  int64_t n;
  const double* pos;     // [n, 2] centres
  const double* width;   // [n] or null (1.0)
  const double* height;  // [n] or null (1.0)
  const uint8_t* fixed;  // [n] or null (none fixed)
  const char* names;     // concatenated names or null
  const int64_t* name_off;  // [n + 1]
  const char* prefix;    // device copy of the generated-name prefix
  int prefix_len;
};

__device__ __forceinline__ void corners(const PlArgs& a, int64_t i, double& llx, double& lly) {
  const double w = a.width ? a.width[i] : 1.0;
  const double h = a.height ? a.height[i] : 1.0;
  llx = __dsub_rn(a.pos[2 * i], __ddiv_rn(w, 2.0));
  lly = __dsub_rn(a.pos[2 * i + 1], __ddiv_rn(h, 2.0));
}

__device__ __forceinline__ int64_t name_len(const PlArgs& a, int64_t i) {
  if (a.names) return a.name_off[i + 1] - a.name_off[i];
  return a.prefix_len + udigits((u128)i);
}

__global__ void k_pl_len(PlArgs a, int64_t* __restrict__ len, int* __restrict__ err) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * blockDim.x) {
    double llx, lly;
    corners(a, i, llx, lly);
    const Fixed6 fx = decompose(llx), fy = decompose(lly);
    if (fx.range_error || fy.range_error) atomicMin(err, (int)min(i, (int64_t)INT_MAX - 1));
    const bool fixed = a.fixed && a.fixed[i];
    len[i] = name_len(a, i) + 1 + fixed6_len(fx) + 1 + fixed6_len(fy) + 4 + (fixed ? 7 : 0) + 1;
  }
}

__global__ void k_pl_write(PlArgs a, const int64_t* __restrict__ off, char* __restrict__ out) {
  if (blockIdx.x == 0 && threadIdx.x < kHeaderLen) out[threadIdx.x] = c_header[threadIdx.x];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * blockDim.x) {
    double llx, lly;
    corners(a, i, llx, lly);
    const Fixed6 fx = decompose(llx), fy = decompose(lly);
    char* p = out + kHeaderLen + off[i];
    if (a.names) {
      for (int64_t k = a.name_off[i]; k < a.name_off[i + 1]; ++k) *p++ = a.names[k];
    } else {
      for (int k = 0; k < a.prefix_len; ++k) *p++ = a.prefix[k];
      p = put_udec(p, (u128)i);
    }
    *p++ = '\t';
    p = put_fixed6(p, fx);
    *p++ = '\t';
    p = put_fixed6(p, fy);
    p[0] = '\t'; p[1] = ':'; p[2] = ' '; p[3] = 'N';
    p += 4;
    if (a.fixed && a.fixed[i]) {
      const char* s = " /FIXED";
      for (int k = 0; k < 7; ++k) p[k] = s[k];
      p += 7;
    }
    *p = '\n';
  }
}

}  // namespace

// Size (d_out == nullptr) or write the .pl text; returns the exact byte count.
int64_t format_placement(Ctx* ctx, int64_t n, const double* pos, const double* width, const double* height,
                         const uint8_t* fixed, const char* names, const int64_t* name_off, const char* prefix,
                         char* out, int64_t cap) {
  cudaStream_t st = ctx->stream;
  const int plen = prefix ? (int)strlen(prefix) : 0;
  if (!names && plen > 256) throw_error(GIFT_ERR_VALUE, "name prefix longer than 256 bytes");
  if (names && !name_off) throw_error(GIFT_ERR_VALUE, "names given without name offsets");
  if (n == 0) {
    if (out) {
      if (cap < kHeaderLen) throw_error(GIFT_ERR_VALUE, "output buffer too small");
      GIFT_CUDA(cudaMemcpyAsync(out, kHeader, kHeaderLen, cudaMemcpyHostToDevice, st));
      GIFT_CUDA(cudaStreamSynchronize(st));
    }
    return kHeaderLen;
  }
  DevBuf<char> dprefix(ctx, plen + 1);
  if (plen) GIFT_CUDA(cudaMemcpyAsync(dprefix.p, prefix, plen, cudaMemcpyHostToDevice, st));
  PlArgs a{n, pos, width, height, fixed, names, name_off, dprefix.p, plen};
  DevBuf<int64_t> len(ctx, n + 1), off(ctx, n + 1);
  DevBuf<int> err(ctx, 1);
  const int big = INT_MAX;
  GIFT_CUDA(cudaMemcpyAsync(err.p, &big, sizeof(int), cudaMemcpyHostToDevice, st));
  GIFT_CUDA(cudaMemsetAsync(len.p + n, 0, sizeof(int64_t), st));
  k_pl_len<<<grid_for(n, kBlock), kBlock, 0, st>>>(a, len.p, err.p);
  GIFT_LAUNCH_CHECK(ctx);
  size_t bytes = 0;
  GIFT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, len.p, off.p, n + 1, st));
  {
    DevBuf<char> tmp(ctx, bytes);
    GIFT_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, len.p, off.p, n + 1, st));
  }
  ctx->launches += 1;
  int64_t total = 0;
  int h_err = 0;
  GIFT_CUDA(cudaMemcpyAsync(&total, off.p + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GIFT_CUDA(cudaMemcpyAsync(&h_err, err.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  GIFT_CUDA(cudaStreamSynchronize(st));
  if (h_err != INT_MAX)
    throw_error(GIFT_ERR_VALUE, "cell " + std::to_string(h_err) +
                                    ": |coordinate| >= 2^107 is outside the .pl formatter's exact range");
  total += kHeaderLen;
  if (!out) return total;
  if (cap < total) throw_error(GIFT_ERR_VALUE, "output buffer too small for the .pl text");
  k_pl_write<<<grid_for(n, kBlock), kBlock, 0, st>>>(a, off.p, out);
  GIFT_LAUNCH_CHECK(ctx);
  GIFT_CUDA(cudaStreamSynchronize(st));
  return total;
}

}  // namespace gift
