// common.cuh -- shared state, error plumbing and device-memory helpers of
// libgiftb200.so (the C ABI in include/gift_b200.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/gift_b200.h"

namespace gift {

// ---- error plumbing --------------------------------------------------------
struct Error {
  int code;
  std::string msg;
  int64_t arg;
};

void set_error(int code, const std::string& msg, int64_t arg = -1);
int fail(int code, const std::string& msg, int64_t arg = -1);

// Throwable error used inside the library; the ABI layer converts it into a
// status code + thread-local message (no C++ exception crosses the ABI).
struct GiftException {
  int code;
  std::string msg;
  int64_t arg;
};

[[noreturn]] void throw_error(int code, const std::string& msg, int64_t arg = -1);
void check_cuda(cudaError_t e, const char* what, const char* file, int line);

#define GIFT_CUDA(x) ::gift::check_cuda((x), #x, __FILE__, __LINE__)
#define GIFT_LAUNCH_CHECK(ctx)                                   \
  do {                                                           \
    ::gift::check_cuda(cudaGetLastError(), "kernel launch", __FILE__, __LINE__); \
    (ctx)->launches++;                                           \
  } while (0)

// ---- context ---------------------------------------------------------------
struct Ctx {
  int device = 0;
  cudaStream_t stream = 0;
  cudaStream_t side = nullptr;    // forked work (BMT wide rows), joined back with events
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  // ghost-row pull from peer memory (peer.cu): its own forked stream
  cudaStream_t pull = nullptr;
  cudaEvent_t pull_fork = nullptr, pull_done = nullptr;
  bool pull_pending = false;
  int64_t launches = 0;
  int num_sms = 148;
  int smem_optin = 0;             // max dynamic shared memory per block (opt-in), this device
  int tiled_policy = GIFT_TILED_ON_REUSE;  // when the fp32 hop builds the tiled (BMT) copy of a graph
  // kernel-selection options (gift_ctx_set_option; a -DGIFT_TUNING build also
  // reads them from GIFT_* environment variables at context creation)
  struct Options {
    int64_t tiled = 1;              // "tiled": 0 = row kernel only
    int64_t tiled_min_rows = 98304;   // "tiled_min_rows": smaller graphs stay on the row kernel (measured
                                      // crossover with wave-balanced tiles: between 53k and 105k rows)
    int64_t tiled_min_mean = 32;    // "tiled_min_mean": mean row length below which too
    int64_t tile_rows = 0;          // "tile_rows": force the tile height (multiple of 32 in 2048..16384), 0 = per graph
    int64_t balance = 1;            // "balance": shrink the default tile height to fill whole waves of SMs
    int64_t col_bits = 0;           // "col_bits": force log2 of the block width (11..14), 0 = per graph
    int64_t barrier_free = 1;       // "barrier_free": the bulk-copy pipeline where it fits
    int64_t graphs = 1;             // "graphs": replay small-graph banks as CUDA graphs
    int64_t fused = 1;              // "fused": small-graph banks as one cooperative kernel
    int64_t zero_copy = 1;          // "zero_copy": *_host calls use pinned buffers in place
    int64_t schedule = 2;           // "schedule": bank-conflict-aware entry order in the tiled copy (1: greedy
                                    // everywhere; 2: edge-colouring optimum in the F = 4 copy, greedy in the other)
    int64_t implicit_above = 0;     // "implicit_above": gift_place_host builds the factored clique model (0 = off)
    int64_t row_lanes = 0;          // "row_lanes": force lanes per row of the row kernel (8 / 16 / 32)
    int64_t codes = 0;              // "codes" (tuning builds): u8 weight codes in the F <= 2 tiled copy
    int64_t prefetch = 0;           // "prefetch": tiled hop prefetches each warp's next slice into L2
    int64_t stream = 0;             // "stream": tiled hop pipelines records across a warp's slices
  } opt;
  std::recursive_mutex mu;        // entry points serialise on the context (scratch, stream, logs)
  // persistent BMT tile scheduler counters [next tile, finished CTAs], one
  // pair per stream (launches on one stream never overlap; self-resetting)
  std::map<cudaStream_t, unsigned*> tile_ctr;
  // grow-only scratch arenas, reused across calls on this context
  void* scratch[4] = {nullptr, nullptr, nullptr, nullptr};
  size_t scratch_bytes[4] = {0, 0, 0, 0};
  // pinned host staging for the *_host entry points
  void* pinned = nullptr;
  size_t pinned_bytes = 0;
  // launch timing (gift_ctx_set_profiling)
  bool profiling = false;
  struct Rec {
    int kind;
    int units;
    cudaEvent_t a, b;
  };
  std::vector<Rec> recs;
  // small-graph fp32 banks replayed as CUDA graphs (filter.cu), most recent last
  struct BankGraph {
    uint64_t uid = 0;             // Csr::uid the graph was captured on
    std::vector<double> key;      // terms, widths, dtypes, epilogue
    cudaGraphExec_t exec = nullptr;
    void* gin = nullptr;          // staged input / output / mask / fixed centres
    void* gout = nullptr;
    uint8_t* gmask = nullptr;
    double* gpos = nullptr;
    int64_t kernels = 0;          // launches inside the graph
  };
  std::vector<BankGraph> graphs;
  cudaStream_t cap_stream = nullptr;  // private stream the graphs are captured on
};

// brackets one launch with events when ctx->profiling (see gift_ctx_set_profiling)
struct ProfScope {
  Ctx* ctx;
  Ctx::Rec rec;
  bool on;
  ProfScope(Ctx* c, int kind, int units) : ctx(c), on(c->profiling) {
    if (!on) return;
    rec.kind = kind;
    rec.units = units;
    cudaEventCreate(&rec.a);
    cudaEventCreate(&rec.b);
    cudaEventRecord(rec.a, c->stream);
  }
  ~ProfScope() {
    if (!on) return;
    cudaEventRecord(rec.b, ctx->stream);
    ctx->recs.push_back(rec);
  }
};

// stream-ordered device allocation (default mempool, release threshold max)
void* dev_alloc(Ctx* ctx, size_t bytes);
void dev_free(Ctx* ctx, void* p);
void* scratch(Ctx* ctx, int slot, size_t bytes);
void* pinned(Ctx* ctx, size_t bytes);

// RAII device buffer bound to a context stream
template <typename T>
struct DevBuf {
  Ctx* ctx = nullptr;
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(Ctx* c, size_t count) : ctx(c), n(count) {
    p = static_cast<T*>(dev_alloc(c, count * sizeof(T) + 16));
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : ctx(o.ctx), p(o.p), n(o.n) { o.p = nullptr; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    reset();
    ctx = o.ctx; p = o.p; n = o.n; o.p = nullptr;
    return *this;
  }
  ~DevBuf() { reset(); }
  void reset() {
    if (p) dev_free(ctx, p);
    p = nullptr;
  }
  T* release() { T* q = p; p = nullptr; return q; }
};

// ---- CSR -------------------------------------------------------------------
// Symmetric CSR, immutable after construction (graph.py:48-111).
// Structure and fp64 values are the reference's bit for bit; derived arrays
// (degrees, fp32 hop weights, per-sigma scale vectors) are computed lazily
// and cached, as SparseSymMatrix caches `degrees` (graph.py:89-94).
struct Csr {
  int device = 0;
  int64_t n = 0;
  int64_t nnz = 0;
  int64_t* indptr = nullptr;   // [n+1]
  int32_t* indices = nullptr;  // [nnz]
  double* values = nullptr;    // [nnz]
  bool has_diagonal = true;    // false when built by build_clique_graph (no self pairs)
  double* degrees = nullptr;   // [n], lazy
  float* w32 = nullptr;        // [nnz] fp32 weights for the fast hop, lazy
  double mean_row = 0.0;
  std::map<double, double*> s64;  // sigma -> 1/sqrt(d+sigma)   (fp64, exact)
  std::map<double, float*> s32;   // sigma -> fp32 rounding of s64
  bool sorted_rows = true;        // columns ascending within every row (canonical CSR)
  bool square = true;             // every column < n (a full graph, or a shard's local block)
  // sliced block-major copy of the matrix for the fp32 hop (bmt.cu), lazy
  struct Bmt {
    bool ready = false, ok = false;
    int64_t ntiles = 0, nseg = 0, nslices = 0, slots = 0, nwide = 0;
    int tile_rows = 2048;
    int kC = 4096;                  // columns per staged block
    uint8_t* wide = nullptr;        // [n] rows left to the row kernel (span > kWide blocks)
    int32_t* wide_rows = nullptr;   // [nwide]
    int64_t nres = 0;               // entries in sparse (tile, block) segments
    int64_t* res_rowptr = nullptr;  // [n + 1] residual CSR of those entries
    int32_t* res_col = nullptr;
    float* res_w = nullptr;
    int64_t* tile_seg = nullptr;    // [ntiles + 1] segment range of each row tile
    int32_t* tile_order = nullptr;  // [ntiles] tiles by decreasing estimated cost (persistent CTAs take them in order)
    int64_t* res_rows = nullptr;    // rows with residual entries
    int64_t* tile_res = nullptr;    // [ntiles + 1] range of res_rows per tile
    int32_t* seg_code = nullptr;    // [nseg] staged column block, or -(block + 1): gather from L2
    int64_t* seg_slice = nullptr;   // [nseg + 1] slice range of each segment
    int64_t* slice_off = nullptr;   // [nslices + 1] first slot of each slice
    uint16_t* slice_rows = nullptr; // [nslices * 32] row in tile per lane (0xffff: none)
    uint8_t* data = nullptr;        // [slots / 128] records: 32x4 u16 columns (kC = padding), then
                                    // 32x4 f32 weights (768 B) or, coded, 32x4 u8 weight codes (384 B)
    bool coded = false;             // weights as u8 codes into code_tbl
    float* code_tbl = nullptr;      // [256] fp32 weight of each code; 255 = padding (0)
    int64_t coded_values = 0;       // distinct weights the table holds (<= 255)
  } bmt, bmt_wide;  // bmt_wide: signal widths <= 2; bmt: F = 4 (bmt.cu bmt_shape_for)
  int64_t fp32_hops = 0;          // fp32 hop launches served (tiled-copy policy: build on reuse)
  uint64_t uid = 0;               // identity for cached CUDA graphs (0 = none yet; never reused)
  // implicit clique term of the nets above the cap (hf.cu; opt-in extension)
  struct Hf {
    int64_t nets = 0, pins = 0, cells = 0;
    int64_t* net_start = nullptr;  // [nets + 1] the selected nets' pin table
    int32_t* pin_cell = nullptr;   // [pins]
    double* coef = nullptr;        // [nets] 2/m
    int32_t* cell = nullptr;       // [cells] cells with high-fanout pins, ascending
    int64_t* occ_ptr = nullptr;    // [cells + 1] their pin occurrences (net order)
    int32_t* occ_net = nullptr;    // [pins] net of each occurrence
    double* occ_b = nullptr;       // [pins] multiplicity of the cell in that net
    void* tbuf = nullptr;          // [nets * 4] fp64 per-hop net sums
    // fp32 hop of the factored clique model (hf.cu k_fact_*)
    float* coef32 = nullptr;       // [nets] 2/m
    float* occ_b32 = nullptr;      // [pins] multiplicities
    int32_t* row_occ = nullptr;    // [n + 1] occurrence range of every row (cells without any: empty)
    double* row_d = nullptr;       // [n] sum over the row's occurrences of (2/m) b
    void* cw = nullptr;            // [nnz] (column, fp32 weight) pairs of the stored entries (lazy)
  } hf;
  int64_t ext_n = 0;              // ghost block of a row shard: its columns >= n index these
  int64_t* ext_ids = nullptr;     // [ext_n] global ids of the ghost columns, ascending
  std::vector<void*> owned;       // everything above, freed on destroy
  std::recursive_mutex mu;        // lazy derived state (degrees, w32, s_sigma, tiled copies)
  cudaEvent_t last_use = nullptr; // recorded on the using stream by every entry point; destroy waits on it
};

// a parsed Bookshelf design (bookshelf.cu): device arrays owned by the handle
struct Bookshelf {
  int64_t n_cells = 0, n_nets = 0, n_pins = 0, n_terminals_decl = -1, n_fixed = 0;
  int64_t cell_name_bytes = 0, net_name_bytes = 0, pl_unknown = 0, n_placed = 0;
  double bbox[4] = {0, 0, 0, 0};
  std::vector<void*> owned;
  int64_t* net_start = nullptr;
  int32_t* pin_cell = nullptr;
  double *pin_dx = nullptr, *pin_dy = nullptr, *width = nullptr, *height = nullptr, *fixed_pos = nullptr;
  uint8_t* fixed = nullptr;
  char *cell_names = nullptr, *net_names = nullptr;
  int64_t *cell_name_off = nullptr, *net_name_off = nullptr;
};

void* csr_alloc(Ctx* ctx, Csr* c, size_t bytes);
void csr_destroy(Csr* c);
void csr_touch(Ctx* ctx, Csr* c);
void set_option(Ctx* ctx, const std::string& name, int64_t value);

// ---- launch helpers --------------------------------------------------------
inline unsigned grid_for(int64_t work, int block, int64_t cap = 148LL * 64) {
  int64_t g = (work + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}

inline int bit_length(uint64_t v) { return v == 0 ? 0 : 64 - __builtin_clzll(v); }

}  // namespace gift

struct gift_ctx : gift::Ctx {};
struct gift_csr : gift::Csr {};
