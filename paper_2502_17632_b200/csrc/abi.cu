// abi.cu -- extern "C" entry points of libgiftb200.so (include/gift_b200.h)
// plus the context / memory / error plumbing declared in common.cuh.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "common.cuh"

namespace gift {

// implemented in build.cu / filter.cu
Csr* build_clique_graph(Ctx* ctx, int64_t n, int64_t n_nets, const int64_t* d_net_start, const int32_t* d_pin_cell,
                        int64_t cap, int64_t* n_skipped);
Csr* csr_from_coo(Ctx* ctx, int64_t n, int64_t T, const int64_t* d_rows, const int64_t* d_cols, const double* d_vals,
                  bool check_symmetric);
const double* csr_degrees(Ctx* ctx, Csr* c);
Csr* normalized_augmented_adjacency(Ctx* ctx, Csr* c, double sigma);
void csr_matmul(Ctx* ctx, const Csr* c, int64_t ncols, const double* x, double* y);
void filter(Ctx* ctx, Csr* c, int n_terms, const double* sigma, const int64_t* k, const double* alpha, int64_t ncols,
            int in_dtype, const void* g, int out_dtype, void* out, const uint8_t* fixed_mask, const double* fixed_pos,
            const double* region, int precision);

void scale_vectors(Ctx* ctx, Csr* c, double sigma, const double** s64, const float** s32);
const float* weights32(Ctx* ctx, Csr* c);
void hop_fp32(Ctx* ctx, Csr* c, const gift_hop_desc* d);
void pack_fp32(Ctx* ctx, int64_t n, int wcols, int nch, const float* const* s, int in_dtype, const void* g,
               int64_t ld, int64_t c0, int F, float* z);
void gather_rows_f32(Ctx* ctx, int64_t n_idx, int F, const int64_t* idx, const float* src, float* dst);
Csr* csr_from_arrays(Ctx* ctx, int64_t n_rows, int64_t nnz, const int64_t* d_indptr, const int32_t* d_indices,
                     const double* d_values);
void csr_row_bounds(Ctx* ctx, const Csr* c, int world, int64_t* h_bounds);
void free_bank_graphs(Ctx* ctx);
int64_t csr_attach_high_fanout(Ctx* ctx, Csr* c, int64_t n_nets, const int64_t* d_net_start, const int32_t* d_pin_cell,
                               int64_t cap, int64_t upto);
void csr_split_rows(Ctx* ctx, const Csr* c, int64_t r0, int64_t r1, Csr** local, Csr** ghost);
void* peer_alloc(Ctx* ctx, size_t bytes, cudaIpcMemHandle_t* handle);
void* peer_open(Ctx* ctx, const cudaIpcMemHandle_t& handle);
void pull_rows_f32(Ctx* ctx, int64_t n, int F, const void* const* d_peers, const int32_t* d_src_rank,
                   const int64_t* d_src_row, float* d_dst);
void pull_join(Ctx* ctx);

double quadratic_wirelength(Ctx* ctx, const Csr* c, const double* g);
double hpwl(Ctx* ctx, int64_t n_nets, const int64_t* net_start, const int32_t* pin_cell, const double* pdx,
            const double* pdy, const double* g);
void rayleigh_parts(Ctx* ctx, const Csr* lap, const double* col, bool center, double* num, double* den);
Csr* laplacian(Ctx* ctx, Csr* adj);
struct Bookshelf;
Bookshelf* bookshelf_parse(Ctx* ctx, const char* h_nodes, int64_t n_nodes, const char* h_nets, int64_t n_nets,
                           const char* h_pl, int64_t n_pl);
void bookshelf_destroy(Ctx* ctx, Bookshelf* B);
int64_t format_placement(Ctx* ctx, int64_t n, const double* pos, const double* width, const double* height,
                         const uint8_t* fixed, const char* names, const int64_t* name_off, const char* prefix,
                         char* out, int64_t cap);

static thread_local Error t_err{GIFT_OK, "", -1};

void set_error(int code, const std::string& msg, int64_t arg) { t_err = Error{code, msg, arg}; }

int fail(int code, const std::string& msg, int64_t arg) {
  set_error(code, msg, arg);
  return code;
}

void throw_error(int code, const std::string& msg, int64_t arg) { throw GiftException{code, msg, arg}; }

void check_cuda(cudaError_t e, const char* what, const char* file, int line) {
  if (e == cudaSuccess) return;
  cudaGetLastError();  // clear sticky non-fatal state
  const int code = (e == cudaErrorMemoryAllocation) ? GIFT_ERR_OOM : GIFT_ERR_CUDA;
  throw_error(code, std::string(cudaGetErrorString(e)) + " in " + what + " (" + file + ":" + std::to_string(line) + ")");
}

void* dev_alloc(Ctx* ctx, size_t bytes) {
  void* p = nullptr;
  if (bytes == 0) bytes = 16;
  check_cuda(cudaMallocAsync(&p, bytes, ctx->stream), "cudaMallocAsync", __FILE__, __LINE__);
  return p;
}

void dev_free(Ctx* ctx, void* p) {
  if (p) cudaFreeAsync(p, ctx->stream);
}

void* scratch(Ctx* ctx, int slot, size_t bytes) {
  if (ctx->scratch_bytes[slot] < bytes) {
    // forget the old arena before allocating: if the allocation throws, the
    // context must not keep a pointer it already freed
    void* old = ctx->scratch[slot];
    ctx->scratch[slot] = nullptr;
    ctx->scratch_bytes[slot] = 0;
    dev_free(ctx, old);
    void* p = dev_alloc(ctx, bytes);
    ctx->scratch[slot] = p;
    ctx->scratch_bytes[slot] = bytes;
  }
  return ctx->scratch[slot];
}

void* pinned(Ctx* ctx, size_t bytes) {
  if (ctx->pinned_bytes < bytes) {
    void* old = ctx->pinned;
    ctx->pinned = nullptr;
    ctx->pinned_bytes = 0;
    if (old) cudaFreeHost(old);
    void* p = nullptr;
    check_cuda(cudaMallocHost(&p, bytes), "cudaMallocHost", __FILE__, __LINE__);
    ctx->pinned = p;
    ctx->pinned_bytes = bytes;
  }
  return ctx->pinned;
}

void set_option(Ctx* ctx, const std::string& name, int64_t v) {
  auto bad = [&]() { throw_error(GIFT_ERR_VALUE, "bad value " + std::to_string(v) + " for option " + name); };
  Ctx::Options& o = ctx->opt;
  if (name == "tiled") {
    if (v != 0 && v != 1) bad();
    o.tiled = v;
  } else if (name == "tiled_min_rows") {
    if (v < 0) bad();
    o.tiled_min_rows = v;
  } else if (name == "tiled_min_mean") {
    if (v < 0) bad();
    o.tiled_min_mean = v;
  } else if (name == "tile_rows") {
    const int64_t lo = 1024;
    if (v != 0 && (v < lo || v > 16384 || v % 32 != 0)) bad();
    o.tile_rows = v;
  } else if (name == "col_bits") {
    if (v != 0 && (v < 11 || v > 14)) bad();
    o.col_bits = v;
  } else if (name == "schedule" && v == 2) {
    o.schedule = 2;  // optimal (edge-colouring) step order in the F = 4 tiled copy
  } else if (name == "barrier_free" && v == 2) {
    o.barrier_free = 2;  // also on tiles of <= 2048 rows at one 1024-thread CTA per SM
  } else if (name == "barrier_free" || name == "graphs" || name == "zero_copy" || name == "schedule" ||
             name == "fused" || name == "stream" || name == "balance") {
    if (v != 0 && v != 1) bad();
    (name == "barrier_free" ? o.barrier_free
     : name == "balance"    ? o.balance
     : name == "graphs"     ? o.graphs
     : name == "zero_copy"  ? o.zero_copy
     : name == "fused"      ? o.fused
     : name == "stream"     ? o.stream
                            : o.schedule) = v;
  } else if (name == "prefetch") {
#ifdef GIFT_TUNING
    if (v != 0 && v != 1) bad();
#else
    if (v != 0) throw_error(GIFT_ERR_VALUE, "option prefetch: only in -DGIFT_TUNING builds");
#endif
    o.prefetch = v;
  } else if (name == "codes") {
#ifdef GIFT_TUNING
    if (v != 0 && v != 1) bad();
#else
    if (v != 0) throw_error(GIFT_ERR_VALUE, "option codes: u8 weight codes exist only in -DGIFT_TUNING builds");
#endif
    o.codes = v;
  } else if (name == "implicit_above") {
    if (v != 0 && v < 2) bad();
    o.implicit_above = v;
  } else if (name == "row_lanes") {
    if (v != 0 && v != 8 && v != 16 && v != 32) bad();
    o.row_lanes = v;
  } else {
    throw_error(GIFT_ERR_VALUE, "unknown option " + name);
  }
}

#ifdef GIFT_TUNING
// tuning builds: the GIFT_* environment variables of the sweep tools (tools/)
static void options_from_env(Ctx* ctx) {
  const std::pair<const char*, const char*> names[] = {
      {"GIFT_BMT", "tiled"},          {"GIFT_BMT_MIN_ROWS", "tiled_min_rows"}, {"GIFT_BMT_MIN_MEAN", "tiled_min_mean"},
      {"GIFT_BMT_TILE_ROWS", "tile_rows"}, {"GIFT_BMT_COL_BITS", "col_bits"}, {"GIFT_BMT_NB", "barrier_free"},
      {"GIFT_GRAPHS", "graphs"},      {"GIFT_ZERO_COPY", "zero_copy"},        {"GIFT_BMT_SCHEDULE", "schedule"},
      {"GIFT_HOP_G", "row_lanes"},    {"GIFT_FUSED", "fused"},                 {"GIFT_CODES", "codes"}};
  for (auto& nv : names) {
    const char* v = std::getenv(nv.first);
    if (v && *v) set_option(ctx, nv.second, std::atoll(v));
  }
}
#endif

void* csr_alloc(Ctx* ctx, Csr* c, size_t bytes) {
  void* p = dev_alloc(ctx, bytes + 64);  // vector loads may read up to 3 elements past the end
  c->owned.push_back(p);
  return p;
}

// one non-blocking stream per device that returns freed graphs to the pool
static cudaStream_t free_stream(int device) {
  static std::mutex mu;
  static std::map<int, cudaStream_t> streams;
  std::lock_guard<std::mutex> lk(mu);
  auto it = streams.find(device);
  if (it != streams.end()) return it->second;
  cudaStream_t s = nullptr;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  streams[device] = s;
  return s;
}

// The arrays are freed in stream order after the last entry point that used
// them (its stream recorded c->last_use): no host wait, no device-wide sync.
void csr_destroy(Csr* c) {
  if (!c) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(c->device);
  cudaStream_t fs = free_stream(c->device);
  if (c->last_use) {
    cudaStreamWaitEvent(fs, c->last_use, 0);
    cudaEventDestroy(c->last_use);
  }
  for (void* p : c->owned) cudaFreeAsync(p, fs);
  cudaSetDevice(prev);
  delete static_cast<gift_csr*>(c);
}

// marks c as used by work enqueued on ctx->stream (see csr_destroy)
void csr_touch(Ctx* ctx, Csr* c) {
  if (!c) return;
  if (!c->last_use) GIFT_CUDA(cudaEventCreateWithFlags(&c->last_use, cudaEventDisableTiming));
  GIFT_CUDA(cudaEventRecord(c->last_use, ctx->stream));
}

}  // namespace gift

using gift::GiftException;

#define GIFT_API_BEGIN try {
#define GIFT_API_END                                     \
  return GIFT_OK;                                        \
  }                                                      \
  catch (const GiftException& e) {                       \
    return gift::fail(e.code, e.msg, e.arg);             \
  }                                                      \
  catch (const std::exception& e) {                      \
    return gift::fail(GIFT_ERR_INTERNAL, e.what());      \
  }                                                      \
  catch (...) {                                          \
    return gift::fail(GIFT_ERR_INTERNAL, "unknown error"); \
  }

namespace {
struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

void require(bool ok, int code, const char* msg) {
  if (!ok) gift::throw_error(code, msg);
}

// An entry point that works on (ctx, csr): switches to the context's device,
// serialises on the context and the graph (lock order ctx -> csr), and on
// exit records that csr was used on ctx->stream (csr_destroy orders its
// frees after that).
struct ApiScope {
  DeviceGuard dev;
  std::unique_lock<std::recursive_mutex> lc, lg;
  gift::Ctx* ctx;
  gift::Csr* csr;
  ApiScope(gift::Ctx* c, const gift::Csr* g)
      : dev(c->device), lc(c->mu), ctx(c), csr(const_cast<gift::Csr*>(g)) {
    if (csr) lg = std::unique_lock<std::recursive_mutex>(csr->mu);
  }
  ~ApiScope() {
    try {
      gift::csr_touch(ctx, csr);
    } catch (...) {
    }
  }
};
}  // namespace

extern "C" {

const char* gift_last_error(void) { return gift::t_err.msg.c_str(); }
int64_t gift_last_error_arg(void) { return gift::t_err.arg; }
const char* gift_version(void) { return "giftb200 0.1 sm_100a"; }

int gift_ctx_create(int device, gift_ctx** out) {
  GIFT_API_BEGIN
  require(out != nullptr, GIFT_ERR_VALUE, "null output pointer");
  int count = 0;
  GIFT_CUDA(cudaGetDeviceCount(&count));
  require(device >= 0 && device < count, GIFT_ERR_VALUE, "device ordinal out of range");
  DeviceGuard g(device);
  GIFT_CUDA(cudaFree(nullptr));  // establish the primary context
  cudaMemPool_t pool;
  GIFT_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t thr = UINT64_MAX;
  GIFT_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  auto* c = new gift_ctx();
  c->device = device;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  cudaDeviceGetAttribute(&c->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
#ifdef GIFT_TUNING
  try {
    gift::options_from_env(c);
  } catch (...) {
    delete c;
    throw;
  }
#endif
  *out = c;
  GIFT_API_END
}

int gift_ctx_destroy(gift_ctx* ctx) {
  GIFT_API_BEGIN
  if (!ctx) return GIFT_OK;
  ApiScope g(ctx, nullptr);
  cudaStreamSynchronize(ctx->stream);
  for (int i = 0; i < 4; ++i)
    if (ctx->scratch[i]) cudaFree(ctx->scratch[i]);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  for (auto& kv : ctx->tile_ctr) cudaFree(kv.second);
  gift::free_bank_graphs(ctx);
  if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
  if (ctx->pull) {
    cudaStreamSynchronize(ctx->pull);
    cudaStreamDestroy(ctx->pull);
    cudaEventDestroy(ctx->pull_fork);
    cudaEventDestroy(ctx->pull_done);
  }
  if (ctx->side) {
    cudaStreamSynchronize(ctx->side);
    cudaStreamDestroy(ctx->side);
    cudaEventDestroy(ctx->fork_ev);
    cudaEventDestroy(ctx->join_ev);
  }
  delete ctx;
  GIFT_API_END
}

int gift_ctx_set_stream(gift_ctx* ctx, void* stream) {
  GIFT_API_BEGIN
  require(ctx != nullptr, GIFT_ERR_VALUE, "null context");
  ctx->stream = static_cast<cudaStream_t>(stream);
  GIFT_API_END
}

int64_t gift_ctx_launch_count(const gift_ctx* ctx) { return ctx ? ctx->launches : 0; }

int gift_ctx_set_profiling(gift_ctx* ctx, int on) {
  GIFT_API_BEGIN
  require(ctx != nullptr, GIFT_ERR_VALUE, "null context");
  ctx->profiling = on != 0;
  GIFT_API_END
}

int gift_ctx_profile_drain(gift_ctx* ctx, int max_records, int* h_kind, int* h_units, float* h_ms, int* n_records) {
  GIFT_API_BEGIN
  require(ctx != nullptr, GIFT_ERR_VALUE, "null context");
  ApiScope g(ctx, nullptr);
  GIFT_CUDA(cudaStreamSynchronize(ctx->stream));
  int k = 0;
  for (auto& r : ctx->recs) {
    if (k < max_records) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, r.a, r.b);
      if (h_kind) h_kind[k] = r.kind;
      if (h_units) h_units[k] = r.units;
      if (h_ms) h_ms[k] = ms;
      ++k;
    }
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  ctx->recs.clear();
  if (n_records) *n_records = k;
  GIFT_API_END
}

int gift_build_clique_graph(gift_ctx* ctx, int64_t n_cells, int64_t n_nets, const int64_t* d_net_start,
                            const int32_t* d_pin_cell, int64_t max_clique_pins, gift_csr** out,
                            int64_t* n_skipped) {
  GIFT_API_BEGIN
  require(ctx && out, GIFT_ERR_VALUE, "null argument");
  ApiScope g(ctx, nullptr);
  *out = static_cast<gift_csr*>(
      gift::build_clique_graph(ctx, n_cells, n_nets, d_net_start, d_pin_cell, max_clique_pins, n_skipped));
  GIFT_API_END
}

int gift_csr_from_coo(gift_ctx* ctx, int64_t n, int64_t nnz, const int64_t* d_rows, const int64_t* d_cols,
                      const double* d_vals, int check_symmetric, gift_csr** out) {
  GIFT_API_BEGIN
  require(ctx && out, GIFT_ERR_VALUE, "null argument");
  ApiScope g(ctx, nullptr);
  *out = static_cast<gift_csr*>(gift::csr_from_coo(ctx, n, nnz, d_rows, d_cols, d_vals, check_symmetric != 0));
  GIFT_API_END
}

int gift_csr_destroy(gift_csr* csr) {
  GIFT_API_BEGIN
  gift::csr_destroy(csr);
  GIFT_API_END
}

int gift_csr_shape(const gift_csr* csr, int64_t* n, int64_t* nnz) {
  GIFT_API_BEGIN
  require(csr != nullptr, GIFT_ERR_VALUE, "null csr");
  if (n) *n = csr->n;
  if (nnz) *nnz = csr->nnz;
  GIFT_API_END
}

int gift_csr_arrays(const gift_csr* csr, const int64_t** d_indptr, const int32_t** d_indices,
                    const double** d_values) {
  GIFT_API_BEGIN
  require(csr != nullptr, GIFT_ERR_VALUE, "null csr");
  if (d_indptr) *d_indptr = csr->indptr;
  if (d_indices) *d_indices = csr->indices;
  if (d_values) *d_values = csr->values;
  GIFT_API_END
}

int gift_csr_download(gift_ctx* ctx, const gift_csr* csr, int64_t* h_indptr, int32_t* h_indices,
                      double* h_values) {
  GIFT_API_BEGIN
  require(ctx && csr, GIFT_ERR_VALUE, "null argument");
  ApiScope g(ctx, csr);
  if (h_indptr)
    GIFT_CUDA(cudaMemcpyAsync(h_indptr, csr->indptr, (csr->n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost,
                              ctx->stream));
  if (h_indices && csr->nnz)
    GIFT_CUDA(cudaMemcpyAsync(h_indices, csr->indices, csr->nnz * sizeof(int32_t), cudaMemcpyDeviceToHost,
                              ctx->stream));
  if (h_values && csr->nnz)
    GIFT_CUDA(cudaMemcpyAsync(h_values, csr->values, csr->nnz * sizeof(double), cudaMemcpyDeviceToHost,
                              ctx->stream));
  GIFT_CUDA(cudaStreamSynchronize(ctx->stream));
  GIFT_API_END
}

int gift_csr_degrees(gift_ctx* ctx, gift_csr* csr, const double** d_degrees) {
  GIFT_API_BEGIN
  require(ctx && csr && d_degrees, GIFT_ERR_VALUE, "null argument");
  ApiScope g(ctx, csr);
  *d_degrees = gift::csr_degrees(ctx, csr);
  GIFT_API_END
}

int gift_normalized_augmented_adjacency(gift_ctx* ctx, gift_csr* adj, double sigma, gift_csr** out) {
  GIFT_API_BEGIN
  require(ctx && adj && out, GIFT_ERR_VALUE, "null argument");
  ApiScope g(ctx, adj);
  *out = static_cast<gift_csr*>(gift::normalized_augmented_adjacency(ctx, adj, sigma));
  GIFT_API_END
}

int gift_csr_matmul(gift_ctx* ctx, const gift_csr* csr, int64_t ncols, const double* d_x, double* d_y) {
  GIFT_API_BEGIN
  require(ctx && csr, GIFT_ERR_VALUE, "null argument");
  require(ncols >= 0, GIFT_ERR_DIMENSION, "negative column count");
  ApiScope g(ctx, csr);
  gift::csr_matmul(ctx, csr, ncols, d_x, d_y);
  GIFT_API_END
}

int gift_filter(gift_ctx* ctx, gift_csr* adj, int n_terms, const double* h_sigma, const int64_t* h_k,
                const double* h_alpha, int64_t ncols, int in_dtype, const void* d_g, int out_dtype, void* d_out,
                const uint8_t* d_fixed_mask, const double* d_fixed_pos, const double* h_region, int precision) {
  GIFT_API_BEGIN
  require(ctx && adj, GIFT_ERR_VALUE, "null argument");
  ApiScope g(ctx, adj);
  gift::filter(ctx, adj, n_terms, h_sigma, h_k, h_alpha, ncols, in_dtype, d_g, out_dtype, d_out, d_fixed_mask,
               d_fixed_pos, h_region, precision);
  GIFT_API_END
}

// device address of a page-locked, mapped host buffer; nullptr for pageable memory
static void* mapped_host(const void* h) {
  if (!h) return nullptr;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, h) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return (at.type == cudaMemoryTypeHost && at.devicePointer) ? at.devicePointer : nullptr;
}

int gift_filter_host(gift_ctx* ctx, gift_csr* adj, int n_terms, const double* h_sigma, const int64_t* h_k,
                     const double* h_alpha, int64_t ncols, int in_dtype, const void* h_g, int out_dtype, void* h_out,
                     const uint8_t* h_fixed_mask, const double* h_fixed_pos, const double* h_region, int precision) {
  GIFT_API_BEGIN
  require(ctx && adj, GIFT_ERR_VALUE, "null argument");
  ApiScope g(ctx, adj);
  cudaStream_t st = ctx->stream;
  const int64_t n = adj->n;
  const size_t in_b = (size_t)(n * ncols) * (in_dtype == GIFT_DTYPE_F64 ? 8 : 4);
  const size_t out_b = (size_t)(n * ncols) * (out_dtype == GIFT_DTYPE_F64 ? 8 : 4);
  // Pinned (page-locked, mapped) host buffers are used in place: the fused
  // fp32 bank writes each output row exactly once, from its final hop, so the
  // placement streams to the host while that hop runs instead of after it;
  // fixed centres are read only for fixed rows.  Pageable buffers are staged.
  const bool zc = ctx->opt.zero_copy != 0;
  void* z_out = (zc && precision == GIFT_PREC_FP32) ? mapped_host(h_out) : nullptr;
  const double* z_pos = (zc && h_fixed_mask) ? static_cast<const double*>(mapped_host(h_fixed_pos)) : nullptr;
  gift::DevBuf<char> dg(ctx, in_b), dout(ctx, z_out ? 0 : out_b);
  gift::DevBuf<uint8_t> dmask(ctx, h_fixed_mask ? n : 0);
  gift::DevBuf<double> dpos(ctx, (h_fixed_mask && !z_pos) ? 2 * n : 0);
  GIFT_CUDA(cudaMemcpyAsync(dg.p, h_g, in_b, cudaMemcpyHostToDevice, st));
  if (h_fixed_mask) {
    GIFT_CUDA(cudaMemcpyAsync(dmask.p, h_fixed_mask, n, cudaMemcpyHostToDevice, st));
    if (!z_pos) GIFT_CUDA(cudaMemcpyAsync(dpos.p, h_fixed_pos, 2 * n * sizeof(double), cudaMemcpyHostToDevice, st));
  }
  gift::filter(ctx, adj, n_terms, h_sigma, h_k, h_alpha, ncols, in_dtype, dg.p, out_dtype, z_out ? z_out : dout.p,
               h_fixed_mask ? dmask.p : nullptr, h_fixed_mask ? (z_pos ? z_pos : dpos.p) : nullptr, h_region,
               precision);
  if (!z_out) GIFT_CUDA(cudaMemcpyAsync(h_out, dout.p, out_b, cudaMemcpyDeviceToHost, st));
  GIFT_CUDA(cudaStreamSynchronize(st));
  GIFT_API_END
}

int gift_place_host(gift_ctx* ctx, int64_t n_cells, int64_t n_nets, const int64_t* h_net_start,
                    const int32_t* h_pin_cell, int64_t max_clique_pins, int n_terms, const double* h_sigma,
                    const int64_t* h_k, const double* h_alpha, const float* h_g, const uint8_t* h_fixed_mask,
                    const double* h_fixed_pos, const double* h_region, int out_dtype, void* h_out, int precision,
                    int64_t* nnz_out) {
  GIFT_API_BEGIN
  require(ctx && h_net_start, GIFT_ERR_VALUE, "null argument");
  ApiScope g(ctx, nullptr);
  cudaStream_t st = ctx->stream;
  int64_t n_pins = h_net_start[n_nets];
  gift::DevBuf<int64_t> dns(ctx, n_nets + 1);
  gift::DevBuf<int32_t> dpc(ctx, n_pins);
  GIFT_CUDA(cudaMemcpyAsync(dns.p, h_net_start, (n_nets + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  if (n_pins) GIFT_CUDA(cudaMemcpyAsync(dpc.p, h_pin_cell, n_pins * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  // option "implicit_above" = T > 0: the factored clique model -- nets with
  // T < pins <= max_clique_pins are applied as the O(pins) implicit term and
  // only the smaller ones are expanded into matrix entries (same operator)
  const int64_t T = ctx->opt.implicit_above;
  const bool factored = T >= 2 && (max_clique_pins < 0 || T < max_clique_pins);
  gift::Csr* c = gift::build_clique_graph(ctx, n_cells, n_nets, dns.p, dpc.p, factored ? T : max_clique_pins, nullptr);
  try {
    if (factored) gift::csr_attach_high_fanout(ctx, c, n_nets, dns.p, dpc.p, T, max_clique_pins < 0 ? -1 : max_clique_pins);
  } catch (...) {
    gift::csr_touch(ctx, c);
    gift::csr_destroy(c);
    throw;
  }
  dns.reset();
  dpc.reset();
  try {
    const int64_t n = n_cells;
    const size_t out_b = (size_t)(n * 2) * (out_dtype == GIFT_DTYPE_F64 ? 8 : 4);
    // pinned host buffers in place, as in gift_filter_host
    const bool zc = ctx->opt.zero_copy != 0;
    void* z_out = (zc && precision == GIFT_PREC_FP32) ? mapped_host(h_out) : nullptr;
    const double* z_pos = (zc && h_fixed_mask) ? static_cast<const double*>(mapped_host(h_fixed_pos)) : nullptr;
    gift::DevBuf<float> dg(ctx, 2 * n);
    gift::DevBuf<char> dout(ctx, z_out ? 0 : out_b);
    gift::DevBuf<uint8_t> dmask(ctx, n);
    gift::DevBuf<double> dpos(ctx, z_pos ? 0 : 2 * n);
    GIFT_CUDA(cudaMemcpyAsync(dg.p, h_g, 2 * n * sizeof(float), cudaMemcpyHostToDevice, st));
    if (h_fixed_mask) {
      GIFT_CUDA(cudaMemcpyAsync(dmask.p, h_fixed_mask, n, cudaMemcpyHostToDevice, st));
      if (!z_pos) GIFT_CUDA(cudaMemcpyAsync(dpos.p, h_fixed_pos, 2 * n * sizeof(double), cudaMemcpyHostToDevice, st));
    }
    // a one-shot graph: under the default policy (GIFT_TILED_ON_REUSE) its
    // single bank runs the row kernel and no tiled copy is built
    gift::filter(ctx, c, n_terms, h_sigma, h_k, h_alpha, 2, GIFT_DTYPE_F32, dg.p, out_dtype,
                 z_out ? z_out : dout.p, h_fixed_mask ? dmask.p : nullptr,
                 h_fixed_mask ? (z_pos ? z_pos : dpos.p) : nullptr, h_region, precision);
    if (!z_out) GIFT_CUDA(cudaMemcpyAsync(h_out, dout.p, out_b, cudaMemcpyDeviceToHost, st));
    GIFT_CUDA(cudaStreamSynchronize(st));
    if (nnz_out) *nnz_out = c->nnz;
  } catch (...) {
    gift::csr_touch(ctx, c);
    gift::csr_destroy(c);
    throw;
  }
  gift::csr_destroy(c);
  GIFT_API_END
}

int gift_csr_scale(gift_ctx* ctx, gift_csr* csr, double sigma, const double** d_s64, const float** d_s32) {
  GIFT_API_BEGIN
  require(ctx && csr, GIFT_ERR_VALUE, "null argument");
  ApiScope g(ctx, csr);
  gift::scale_vectors(ctx, csr, sigma, d_s64, d_s32);
  GIFT_API_END
}

int gift_csr_weights32(gift_ctx* ctx, gift_csr* csr, const float** d_w32) {
  GIFT_API_BEGIN
  require(ctx && csr && d_w32, GIFT_ERR_VALUE, "null argument");
  ApiScope g(ctx, csr);
  *d_w32 = gift::weights32(ctx, csr);
  GIFT_API_END
}

int gift_csr_from_arrays(gift_ctx* ctx, int64_t n_rows, int64_t nnz, const int64_t* d_indptr,
                         const int32_t* d_indices, const double* d_values, gift_csr** out) {
  GIFT_API_BEGIN
  require(ctx && out && d_indptr, GIFT_ERR_VALUE, "null argument");
  require(n_rows >= 0 && nnz >= 0, GIFT_ERR_VALUE, "negative size");
  ApiScope g(ctx, nullptr);
  *out = static_cast<gift_csr*>(gift::csr_from_arrays(ctx, n_rows, nnz, d_indptr, d_indices, d_values));
  GIFT_API_END
}

int gift_hop_fp32(gift_ctx* ctx, gift_csr* csr, const gift_hop_desc* desc) {
  GIFT_API_BEGIN
  require(ctx && csr && desc, GIFT_ERR_VALUE, "null argument");
  ApiScope g(ctx, csr);
  gift::hop_fp32(ctx, csr, desc);
  GIFT_API_END
}

int gift_pack_fp32(gift_ctx* ctx, int64_t n, int wcols, int nch, const float* const* h_s, int in_dtype,
                   const void* d_g, int64_t ld, int64_t c0, int F, float* d_z) {
  GIFT_API_BEGIN
  require(ctx && h_s, GIFT_ERR_VALUE, "null argument");
  require(nch >= 1 && nch <= 4 && wcols * nch <= F, GIFT_ERR_VALUE, "bad packing");
  ApiScope g(ctx, nullptr);
  gift::pack_fp32(ctx, n, wcols, nch, h_s, in_dtype, d_g, ld, c0, F, d_z);
  GIFT_API_END
}

int gift_gather_rows_f32(gift_ctx* ctx, int64_t n_idx, int F, const int64_t* d_idx, const float* d_src,
                         float* d_dst) {
  GIFT_API_BEGIN
  require(ctx, GIFT_ERR_VALUE, "null argument");
  ApiScope g(ctx, nullptr);
  gift::gather_rows_f32(ctx, n_idx, F, d_idx, d_src, d_dst);
  GIFT_API_END
}

static_assert(sizeof(cudaIpcMemHandle_t) == GIFT_PEER_HANDLE_BYTES, "IPC handle size");

int gift_peer_alloc(gift_ctx* ctx, int64_t bytes, void** d_ptr, unsigned char* h_handle) {
  GIFT_API_BEGIN
  require(ctx && d_ptr && bytes >= 0, GIFT_ERR_VALUE, "null argument");
  ApiScope g(ctx, nullptr);
  cudaIpcMemHandle_t h;
  *d_ptr = gift::peer_alloc(ctx, (size_t)bytes, h_handle ? &h : nullptr);
  if (h_handle) memcpy(h_handle, &h, sizeof(h));
  GIFT_API_END
}

int gift_peer_open(gift_ctx* ctx, const unsigned char* h_handle, void** d_ptr) {
  GIFT_API_BEGIN
  require(ctx && d_ptr && h_handle, GIFT_ERR_VALUE, "null argument");
  ApiScope g(ctx, nullptr);
  cudaIpcMemHandle_t h;
  memcpy(&h, h_handle, sizeof(h));
  *d_ptr = gift::peer_open(ctx, h);
  GIFT_API_END
}

int gift_peer_close(gift_ctx* ctx, void* d_ptr) {
  GIFT_API_BEGIN
  require(ctx != nullptr, GIFT_ERR_VALUE, "null argument");
  ApiScope g(ctx, nullptr);
  if (d_ptr) GIFT_CUDA(cudaIpcCloseMemHandle(d_ptr));
  GIFT_API_END
}

int gift_peer_free(gift_ctx* ctx, void* d_ptr) {
  GIFT_API_BEGIN
  require(ctx != nullptr, GIFT_ERR_VALUE, "null argument");
  ApiScope g(ctx, nullptr);
  if (d_ptr) {
    GIFT_CUDA(cudaStreamSynchronize(ctx->stream));
    if (ctx->pull) GIFT_CUDA(cudaStreamSynchronize(ctx->pull));
    GIFT_CUDA(cudaFree(d_ptr));
  }
  GIFT_API_END
}

int gift_pull_rows_f32(gift_ctx* ctx, int64_t n_rows, int F, const void* const* d_peers, const int32_t* d_src_rank,
                       const int64_t* d_src_row, float* d_dst) {
  GIFT_API_BEGIN
  require(ctx != nullptr && n_rows >= 0, GIFT_ERR_VALUE, "null argument");
  require(n_rows == 0 || (d_peers && d_src_rank && d_src_row && d_dst), GIFT_ERR_VALUE, "null argument");
  ApiScope g(ctx, nullptr);
  gift::pull_rows_f32(ctx, n_rows, F, d_peers, d_src_rank, d_src_row, d_dst);
  GIFT_API_END
}

int gift_pull_join(gift_ctx* ctx) {
  GIFT_API_BEGIN
  require(ctx != nullptr, GIFT_ERR_VALUE, "null argument");
  ApiScope g(ctx, nullptr);
  gift::pull_join(ctx);
  GIFT_API_END
}

int gift_quadratic_wirelength(gift_ctx* ctx, const gift_csr* adj, const double* d_g, double* h_out) {
  GIFT_API_BEGIN
  require(ctx && adj && h_out, GIFT_ERR_VALUE, "null argument");
  ApiScope g(ctx, adj);
  *h_out = gift::quadratic_wirelength(ctx, adj, d_g);
  GIFT_API_END
}

int gift_laplacian(gift_ctx* ctx, gift_csr* adj, gift_csr** out) {
  GIFT_API_BEGIN
  require(ctx && adj && out, GIFT_ERR_VALUE, "null argument");
  ApiScope g(ctx, adj);
  *out = static_cast<gift_csr*>(gift::laplacian(ctx, adj));
  GIFT_API_END
}

int gift_rayleigh_parts(gift_ctx* ctx, const gift_csr* lap, const double* d_col, int center, double* h_num,
                        double* h_den) {
  GIFT_API_BEGIN
  require(ctx && lap && h_num && h_den, GIFT_ERR_VALUE, "null argument");
  ApiScope g(ctx, lap);
  gift::rayleigh_parts(ctx, lap, d_col, center != 0, h_num, h_den);
  GIFT_API_END
}

int gift_hpwl(gift_ctx* ctx, int64_t n_nets, const int64_t* d_net_start, const int32_t* d_pin_cell,
              const double* d_pin_dx, const double* d_pin_dy, const double* d_g, double* h_out) {
  GIFT_API_BEGIN
  require(ctx && h_out, GIFT_ERR_VALUE, "null argument");
  ApiScope g(ctx, nullptr);
  *h_out = gift::hpwl(ctx, n_nets, d_net_start, d_pin_cell, d_pin_dx, d_pin_dy, d_g);
  GIFT_API_END
}

int gift_format_placement(gift_ctx* ctx, int64_t n, const double* d_pos, const double* d_width,
                          const double* d_height, const uint8_t* d_fixed, const char* d_names,
                          const int64_t* d_name_off, const char* h_name_prefix, char* d_out, int64_t cap,
                          int64_t* h_len) {
  GIFT_API_BEGIN
  require(ctx && h_len && n >= 0, GIFT_ERR_VALUE, "null argument");
  require(n == 0 || d_pos, GIFT_ERR_VALUE, "null positions");
  ApiScope g(ctx, nullptr);
  *h_len = gift::format_placement(ctx, n, d_pos, d_width, d_height, d_fixed, d_names, d_name_off, h_name_prefix,
                                  d_out, cap);
  GIFT_API_END
}

struct gift_bookshelf {
  gift::Bookshelf* b;
};

int gift_ctx_set_tiled_policy(gift_ctx* ctx, int policy) {
  GIFT_API_BEGIN
  require(ctx != nullptr, GIFT_ERR_VALUE, "null context");
  require(policy == GIFT_TILED_NEVER || policy == GIFT_TILED_ON_REUSE || policy == GIFT_TILED_ALWAYS, GIFT_ERR_VALUE,
          "unknown tiled policy");
  std::lock_guard<std::recursive_mutex> lk(ctx->mu);
  ctx->tiled_policy = policy;
  GIFT_API_END
}

int gift_csr_attach_high_fanout(gift_ctx* ctx, gift_csr* csr, int64_t n_nets, const int64_t* d_net_start,
                                const int32_t* d_pin_cell, int64_t max_clique_pins, int64_t* n_implicit) {
  GIFT_API_BEGIN
  require(ctx && csr && d_net_start, GIFT_ERR_VALUE, "null argument");
  ApiScope g(ctx, csr);
  const int64_t k = gift::csr_attach_high_fanout(ctx, csr, n_nets, d_net_start, d_pin_cell, max_clique_pins, -1);
  if (n_implicit) *n_implicit = k;
  GIFT_API_END
}

int gift_csr_attach_implicit_nets(gift_ctx* ctx, gift_csr* csr, int64_t n_nets, const int64_t* d_net_start,
                                  const int32_t* d_pin_cell, int64_t above, int64_t upto, int64_t* n_implicit) {
  GIFT_API_BEGIN
  require(ctx && csr && d_net_start, GIFT_ERR_VALUE, "null argument");
  require(above >= 1 && (upto < 0 || upto >= above), GIFT_ERR_VALUE, "implicit nets: need 1 <= above <= upto");
  ApiScope g(ctx, csr);
  const int64_t k = gift::csr_attach_high_fanout(ctx, csr, n_nets, d_net_start, d_pin_cell, above, upto);
  if (n_implicit) *n_implicit = k;
  GIFT_API_END
}

int gift_csr_row_bounds(gift_ctx* ctx, const gift_csr* csr, int world, int64_t* h_bounds) {
  GIFT_API_BEGIN
  require(ctx && csr && h_bounds, GIFT_ERR_VALUE, "null argument");
  ApiScope g(ctx, csr);
  gift::csr_row_bounds(ctx, csr, world, h_bounds);
  GIFT_API_END
}

int gift_csr_split_rows(gift_ctx* ctx, const gift_csr* csr, int64_t r0, int64_t r1, gift_csr** local,
                        gift_csr** ghost) {
  GIFT_API_BEGIN
  require(ctx && csr && local && ghost, GIFT_ERR_VALUE, "null argument");
  ApiScope g(ctx, csr);
  gift::Csr *L = nullptr, *G = nullptr;
  gift::csr_split_rows(ctx, csr, r0, r1, &L, &G);
  *local = static_cast<gift_csr*>(L);
  *ghost = static_cast<gift_csr*>(G);
  GIFT_API_END
}

int gift_csr_ext_ids(const gift_csr* ghost, const int64_t** d_ids, int64_t* n_ids) {
  GIFT_API_BEGIN
  require(ghost && d_ids && n_ids, GIFT_ERR_VALUE, "null argument");
  *d_ids = ghost->ext_ids;
  *n_ids = ghost->ext_n;
  GIFT_API_END
}

int gift_ctx_set_option(gift_ctx* ctx, const char* name, int64_t value) {
  GIFT_API_BEGIN
  require(ctx && name, GIFT_ERR_VALUE, "null argument");
  std::lock_guard<std::recursive_mutex> lk(ctx->mu);
  gift::set_option(ctx, name, value);
  GIFT_API_END
}

int gift_csr_tiled_info(const gift_csr* csr, int which, int64_t* h_info) {
  GIFT_API_BEGIN
  require(csr && h_info, GIFT_ERR_VALUE, "null argument");
  require(which == 0 || which == 1, GIFT_ERR_VALUE, "which must be 0 (F = 4 copy) or 1 (F <= 2 copy)");
  gift::Csr* c = const_cast<gift_csr*>(csr);
  std::lock_guard<std::recursive_mutex> lk(c->mu);
  const gift::Csr::Bmt& B = which == 0 ? c->bmt : c->bmt_wide;
  const int64_t v[10] = {B.ready, B.ok,     B.tile_rows, B.kC,    B.nseg,
                         B.nslices, B.slots, B.nwide,  B.coded, B.coded_values};
  for (int i = 0; i < 10; ++i) h_info[i] = v[i];
  GIFT_API_END
}

int gift_bookshelf_parse(gift_ctx* ctx, const char* h_nodes, int64_t nodes_len, const char* h_nets,
                         int64_t nets_len, const char* h_pl, int64_t pl_len, gift_bookshelf** out) {
  GIFT_API_BEGIN
  require(ctx && out, GIFT_ERR_VALUE, "null argument");
  require(nodes_len >= 0 && nets_len >= 0 && pl_len >= 0, GIFT_ERR_VALUE, "negative length");
  require((h_nodes || !nodes_len) && (h_nets || !nets_len) && (h_pl || !pl_len), GIFT_ERR_VALUE, "null text");
  *out = nullptr;
  ApiScope g(ctx, nullptr);
  gift::Bookshelf* b = gift::bookshelf_parse(ctx, h_nodes, nodes_len, h_nets, nets_len, h_pl, pl_len);
  *out = new gift_bookshelf{b};
  GIFT_API_END
}

int gift_bookshelf_info(const gift_bookshelf* bs, int64_t* h_sizes, double* h_bbox) {
  GIFT_API_BEGIN
  require(bs && bs->b, GIFT_ERR_VALUE, "null handle");
  const gift::Bookshelf& B = *bs->b;
  if (h_sizes) {
    const int64_t v[10] = {B.n_cells, B.n_nets, B.n_pins, B.n_fixed, B.n_terminals_decl,
                           B.cell_name_bytes, B.net_name_bytes, B.pl_unknown, B.n_placed, 0};
    for (int i = 0; i < 10; ++i) h_sizes[i] = v[i];
  }
  if (h_bbox)
    for (int i = 0; i < 4; ++i) h_bbox[i] = B.bbox[i];
  GIFT_API_END
}

int gift_bookshelf_device(const gift_bookshelf* bs, const int64_t** d_net_start, const int32_t** d_pin_cell,
                          const double** d_pin_dx, const double** d_pin_dy, const double** d_width,
                          const double** d_height, const uint8_t** d_fixed, const double** d_fixed_pos) {
  GIFT_API_BEGIN
  require(bs && bs->b, GIFT_ERR_VALUE, "null handle");
  const gift::Bookshelf& B = *bs->b;
  if (d_net_start) *d_net_start = B.net_start;
  if (d_pin_cell) *d_pin_cell = B.pin_cell;
  if (d_pin_dx) *d_pin_dx = B.pin_dx;
  if (d_pin_dy) *d_pin_dy = B.pin_dy;
  if (d_width) *d_width = B.width;
  if (d_height) *d_height = B.height;
  if (d_fixed) *d_fixed = B.fixed;
  if (d_fixed_pos) *d_fixed_pos = B.fixed_pos;
  GIFT_API_END
}

int gift_bookshelf_copy(gift_ctx* ctx, const gift_bookshelf* bs, int64_t* h_net_start, int32_t* h_pin_cell,
                        double* h_pin_dx, double* h_pin_dy, double* h_width, double* h_height, uint8_t* h_fixed,
                        double* h_fixed_pos, char* h_cell_names, int64_t* h_cell_name_off, char* h_net_names,
                        int64_t* h_net_name_off) {
  GIFT_API_BEGIN
  require(ctx && bs && bs->b, GIFT_ERR_VALUE, "null handle");
  ApiScope g(ctx, nullptr);
  const gift::Bookshelf& B = *bs->b;
  cudaStream_t st = ctx->stream;
  auto cp = [&](void* dst, const void* src, int64_t bytes) {
    if (dst && bytes > 0) GIFT_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToHost, st));
  };
  cp(h_net_start, B.net_start, (B.n_nets + 1) * 8);
  cp(h_pin_cell, B.pin_cell, B.n_pins * 4);
  cp(h_pin_dx, B.pin_dx, B.n_pins * 8);
  cp(h_pin_dy, B.pin_dy, B.n_pins * 8);
  cp(h_width, B.width, B.n_cells * 8);
  cp(h_height, B.height, B.n_cells * 8);
  cp(h_fixed, B.fixed, B.n_cells);
  cp(h_fixed_pos, B.fixed_pos, B.n_cells * 16);
  cp(h_cell_names, B.cell_names, B.cell_name_bytes);
  cp(h_cell_name_off, B.cell_name_off, (B.n_cells + 1) * 8);
  cp(h_net_names, B.net_names, B.net_name_bytes);
  cp(h_net_name_off, B.net_name_off, (B.n_nets + 1) * 8);
  GIFT_CUDA(cudaStreamSynchronize(st));
  GIFT_API_END
}

int gift_bookshelf_destroy(gift_ctx* ctx, gift_bookshelf* bs) {
  GIFT_API_BEGIN
  if (!bs) return GIFT_OK;
  require(ctx, GIFT_ERR_VALUE, "null context");
  ApiScope g(ctx, nullptr);
  cudaStreamSynchronize(ctx->stream);
  gift::bookshelf_destroy(ctx, bs->b);
  delete bs;
  GIFT_API_END
}

}  // extern "C"
