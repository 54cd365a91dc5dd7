/*
 * gift_b200.h -- C ABI of the B200-native GiFt hot path (libgiftb200.so).
 *
 * The reference (`giftplace`, pure Python on numpy/scipy) has no FFI; its
 * operator API for this path is the set of Python functions re-exported at
 * giftplace/__init__.py:26-38.  Each entry point below replaces one of them
 * (file:line cited per function) or the scipy/numpy routine it delegates to.
 * The Python package paper_2502_17632_b200 binds this header with ctypes
 * (see INTEGRATION.md for the binding a maintainer would add to giftplace).
 *
 * Conventions
 *  - Plain C types only.  Pointers prefixed d_ are DEVICE pointers (CUDA
 *    global memory of the context's device); h_ are HOST pointers.
 *  - Every function returns a status code (GIFT_OK == 0).  On failure a
 *    thread-local message is available from gift_last_error() and, for
 *    GIFT_ERR_ISOLATED_NODE, the node id from gift_last_error_arg().  The
 *    Python shim re-raises the reference's exception classes:
 *      GIFT_ERR_VALUE         -> ValueError             (graph.py:42-45,174-175,201-202; gift.py:44-45)
 *      GIFT_ERR_DIMENSION     -> DimensionMismatchError (graph.py:98-99; gift.py:80-81)
 *      GIFT_ERR_ISOLATED_NODE -> IsolatedNodeError(node) (graph.py:177-180)
 *      GIFT_ERR_NON_SYMMETRIC -> NonSymmetricError      (graph.py:59-65)
 *  - All work is enqueued on the context's CUDA stream (gift_ctx_set_stream);
 *    functions that must return a host-visible scalar (nnz after a build, an
 *    error found on the device) synchronise that stream.
 *  - Deterministic: identical inputs give bit-identical outputs.
 *    No floating-point atomics anywhere.
 *  - Exactness: CSR structure, fp64 values and fp64 degrees are bit-identical
 *    to the reference (scipy/numpy operation order).
 *    GIFT_PREC_FP64_EXACT filter output is bit-identical to gift_filter /
 *    gift_place; GIFT_PREC_FP32 is the fast fused path (<= 1e-5 rel-L2).
 */
#ifndef GIFT_B200_H
#define GIFT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GIFT_OK 0
#define GIFT_ERR_VALUE 1
#define GIFT_ERR_DIMENSION 2
#define GIFT_ERR_ISOLATED_NODE 3
#define GIFT_ERR_NON_SYMMETRIC 4
#define GIFT_ERR_TOO_LARGE 5
#define GIFT_ERR_CUDA 6
#define GIFT_ERR_OOM 7
#define GIFT_ERR_INTERNAL 8
#define GIFT_ERR_PARSE 9 /* Bookshelf reader: message "<file>\t<lineno>\t<code>\t<value>\t<text>" */

#define GIFT_PREC_FP32 0        /* fused fp32 bank: pre-scaled recurrence, chains fused */
#define GIFT_PREC_FP64_EXACT 1  /* reference operation order, fp64, bit-exact */

#define GIFT_DTYPE_F32 0
#define GIFT_DTYPE_F64 1

/* When the fp32 bank builds the tiled (block-major, BMT) copy of a graph --
 * a one-time reordering (~ a few hops of work) that makes later hops faster: */
#define GIFT_TILED_NEVER 0     /* row kernel only */
#define GIFT_TILED_ON_REUSE 1  /* default: the first bank on a graph runs the row kernel;
                                  the copy is built when the graph is filtered again */
#define GIFT_TILED_ALWAYS 2    /* build on the first fp32 hop */

typedef struct gift_ctx gift_ctx; /* device + stream + workspace */
typedef struct gift_csr gift_csr; /* immutable symmetric CSR (SparseSymMatrix, graph.py:48-111) */
typedef struct gift_bookshelf gift_bookshelf; /* a parsed design (parse_design, netlist.py:418-458) */

/* ---- context --------------------------------------------------------- */
int gift_ctx_create(int device, gift_ctx** out);
int gift_ctx_destroy(gift_ctx* ctx);
/* stream: a cudaStream_t (0 = legacy default stream). */
int gift_ctx_set_stream(gift_ctx* ctx, void* stream);
const char* gift_last_error(void);
int64_t gift_last_error_arg(void);
const char* gift_version(void);
/* Tiled-copy policy of this context (GIFT_TILED_*). */
int gift_ctx_set_tiled_policy(gift_ctx* ctx, int policy);
/* Kernel-selection options of this context (results stay within the fp32
 * tolerance whatever they are; defaults are the tuned choices):
 *   "tiled" 0/1, "tiled_min_rows", "tiled_min_mean" (when the tiled hop applies),
 *   "tile_rows" 0 or a multiple of 32 in 2048..16384 and "col_bits" 0/11..14
 *   (force a tile shape), "balance" 0/1 (default tile heights shrink so the
 *   tiles fill whole waves of SMs), "implicit_above" 0 / T >= 2 (gift_place_host
 *   builds the factored clique model: nets with T < pins <= max_clique_pins
 *   as the implicit term, see gift_csr_attach_implicit_nets),
 *   "barrier_free" 0/1, "fused" 0/1 (small banks as one cooperative kernel),
 *   "graphs" 0/1 (CUDA-graph replay of small banks the fused kernel does not take),
 *   "zero_copy" 0/1 (pinned host buffers used in place), "schedule" 0/1/2
 *   (entry order inside the tiled copies: none / greedy / greedy + the
 *   edge-colouring optimum for the two-chain copy, the default),
 *   "row_lanes" 0/8/16/32, "codes" 0 (1 only in -DGIFT_TUNING builds: u8
 *   weight codes in the F <= 2 tiled copy, an experiment that measured slower),
 *   "prefetch" 0 (1 only in tuning builds: L2 bulk prefetch of each warp's
 *   next slice, measured slower on long-slice graphs).
 *   Unknown names or values: GIFT_ERR_VALUE. */
int gift_ctx_set_option(gift_ctx* ctx, const char* name, int64_t value);
/* Number of kernels this library launched on ctx since creation (for the bench's gpu_launches). */
int64_t gift_ctx_launch_count(const gift_ctx* ctx);
/* Launch timing: when on, every filter-bank kernel is bracketed by CUDA
 * events on the context stream.  gift_ctx_profile_drain synchronises, writes
 * up to max_records (kind, units, milliseconds) triples and clears the log.
 * kind: 0 = signal pack (z0 = s o g), F = hop kernel with F floats per row
 * (1/2/4); units = algorithmic hops the launch performs (chains it advances). */
int gift_ctx_set_profiling(gift_ctx* ctx, int on);
int gift_ctx_profile_drain(gift_ctx* ctx, int max_records, int* h_kind, int* h_units, float* h_ms,
                           int* n_records);

/* ---- graph construction --------------------------------------------- */
/* build_clique_graph(design, max_clique_pins)  graph.py:120-158.
 * d_net_start: int64[n_nets+1] (Design.pin_table net_start, netlist.py:142-166),
 * d_pin_cell:  int32[n_pins] cell ids in [0, n_cells).
 * max_clique_pins < 0 means None (no cap); a cap >= 0 skips every net with
 * more pins than it (cap 0 or 1 skips all nets, as the reference does).  *n_skipped (host, nullable)
 * receives the number of nets skipped by the cap (graph.py:150-151). */
int gift_build_clique_graph(gift_ctx* ctx, int64_t n_cells, int64_t n_nets,
                            const int64_t* d_net_start, const int32_t* d_pin_cell,
                            int64_t max_clique_pins, gift_csr** out, int64_t* n_skipped);

/* Opt-in extension (not in the reference): keep the nets with more than
 * max_clique_pins pins -- which build_clique_graph skips (graph.py:136-138) --
 * as an implicit O(pins) clique term of csr, a graph built from the same
 * netlist with the same cap: A_e = (2/m)(b b^T - diag(b o b)) per net
 * (b = cell multiplicities).  Afterwards degrees, s_sigma, the filter bank
 * (both precisions) and matmul use A_cap + A_implicit, which equals the
 * uncapped clique graph in exact arithmetic (no bit-exact contract for the
 * implicit part; fp32 bank within 1e-5 of the uncapped reference).  Must be
 * called before the graph is used; normalized_augmented_adjacency and the
 * stepped hop refuse such a graph.  *n_implicit (nullable): nets kept. */
int gift_csr_attach_high_fanout(gift_ctx* ctx, gift_csr* csr, int64_t n_nets, const int64_t* d_net_start,
                                const int32_t* d_pin_cell, int64_t max_clique_pins, int64_t* n_implicit);
/* The factored clique model (opt-in): the same implicit term for every net
 * with above < pins <= upto (upto < 0: no upper bound), attached to a graph
 * built with max_clique_pins = above.  With upto = the reference's cap the
 * operator A_explicit(pins <= above) + A_implicit(above < pins <= upto) equals
 * the reference's capped clique graph (graph.py:132-158) in exact arithmetic,
 * at O(pins) per hop for the implicit nets instead of O(pins^2) stored
 * entries: on config 3 ~9M explicit entries + ~9M pin occurrences replace
 * 866M entries.  Same caveats as gift_csr_attach_high_fanout. */
int gift_csr_attach_implicit_nets(gift_ctx* ctx, gift_csr* csr, int64_t n_nets, const int64_t* d_net_start,
                                  const int32_t* d_pin_cell, int64_t above, int64_t upto, int64_t* n_implicit);

/* from_coo(n, rows, cols, vals)  graph.py:114-117, followed by the
 * SparseSymMatrix checks (graph.py:55-65) when check_symmetric != 0.
 * Duplicates summed in scipy order, explicit zeros dropped. */
int gift_csr_from_coo(gift_ctx* ctx, int64_t n, int64_t nnz, const int64_t* d_rows,
                      const int64_t* d_cols, const double* d_vals, int check_symmetric,
                      gift_csr** out);

/* Frees csr once the work already enqueued on it has finished (no host wait,
 * no device-wide synchronisation). */
int gift_csr_destroy(gift_csr* csr);
/* State of the tiled copies of csr (which: 0 = the F = 4 copy, 1 = the copy for
 * signal widths <= 2): h_info[10] = {built, usable, tile_rows, block_cols,
 * segments, slices, stored slots, rows left to the row kernel, weights coded
 * (u8 codes), distinct weights in the code table}. */
int gift_csr_tiled_info(const gift_csr* csr, int which, int64_t* h_info);
int gift_csr_shape(const gift_csr* csr, int64_t* n, int64_t* nnz);
/* Device views (owned by csr): indptr int64[n+1], indices int32[nnz], values fp64[nnz]
 * (SparseSymMatrix.indptr/.indices/.values, graph.py:77-87). */
int gift_csr_arrays(const gift_csr* csr, const int64_t** d_indptr, const int32_t** d_indices,
                    const double** d_values);
/* Copies to caller-allocated HOST arrays (any pointer may be NULL). */
int gift_csr_download(gift_ctx* ctx, const gift_csr* csr, int64_t* h_indptr, int32_t* h_indices,
                      double* h_values);
/* SparseSymMatrix.degrees (graph.py:89-94): fp64 row sums in numpy
 * np.add.reduceat order; computed once and cached on csr. */
int gift_csr_degrees(gift_ctx* ctx, gift_csr* csr, const double** d_degrees);

/* ---- operators ------------------------------------------------------ */
/* normalized_augmented_adjacency(adj, sigma)  graph.py:167-188, materialised. */
int gift_normalized_augmented_adjacency(gift_ctx* ctx, gift_csr* adj, double sigma, gift_csr** out);
/* SparseSymMatrix.matmul(g) (graph.py:96-100): y = A x, fp64, x/y row-major
 * [n, ncols], scipy csr_matvecs order (bit-exact). */
int gift_csr_matmul(gift_ctx* ctx, const gift_csr* csr, int64_t ncols, const double* d_x, double* d_y);

/* ---- filter bank ---------------------------------------------------- */
/* gift_filter(adj, g, config)  gift.py:73-95, optionally fused with the
 * gift_place epilogue gift.py:112-118 (re-pin fixed rows, np.clip movable
 * rows to region) when d_fixed_mask != NULL.
 *   terms: n_terms triples (h_sigma[t], h_k[t], h_alpha[t]) (FilterTerm, graph.py:33-45)
 *   d_g:    [n, ncols] row-major, dtype in_dtype
 *   d_out:  [n, ncols] row-major, dtype out_dtype
 *   d_fixed_mask: uint8[n] or NULL; d_fixed_pos: fp64[n, 2] (rows read only where
 *   fixed); h_region: fp64[4] = xmin, ymin, xmax, ymax.  The epilogue needs ncols == 2.
 *   precision: GIFT_PREC_FP32 or GIFT_PREC_FP64_EXACT. */
int gift_filter(gift_ctx* ctx, gift_csr* adj, int n_terms, const double* h_sigma,
                const int64_t* h_k, const double* h_alpha, int64_t ncols, int in_dtype,
                const void* d_g, int out_dtype, void* d_out, const uint8_t* d_fixed_mask,
                const double* d_fixed_pos, const double* h_region, int precision);

/* Same, with HOST buffers: copies h_g in, runs the bank + epilogue and copies
 * the result out on the context stream (the end-to-end call a host
 * integration makes; returns after the result is in h_out). */
int gift_filter_host(gift_ctx* ctx, gift_csr* adj, int n_terms, const double* h_sigma,
                     const int64_t* h_k, const double* h_alpha, int64_t ncols, int in_dtype,
                     const void* h_g, int out_dtype, void* h_out, const uint8_t* h_fixed_mask,
                     const double* h_fixed_pos, const double* h_region, int precision);

/* Netlist in, positions out: H2D pin table + signal, build_clique_graph,
 * bank, epilogue, D2H (gift.py:98-119 composed with graph.py:120-158).
 * Returns the graph's nnz in *nnz_out (nullable). */
int gift_place_host(gift_ctx* ctx, int64_t n_cells, int64_t n_nets, const int64_t* h_net_start,
                    const int32_t* h_pin_cell, int64_t max_clique_pins, int n_terms,
                    const double* h_sigma, const int64_t* h_k, const double* h_alpha,
                    const float* h_g, const uint8_t* h_fixed_mask, const double* h_fixed_pos,
                    const double* h_region, int out_dtype, void* h_out, int precision,
                    int64_t* nnz_out);

/* ---- stepped bank (host-driven, e.g. row-sharded over ranks) ---------- */
/* The fused fp32 bank of gift_filter, exposed one kernel at a time so a host
 * driver can interleave a halo exchange between hops (paper_2502_17632_b200/
 * shard.py).  Rows of the CSR are the rows a rank owns; column ids index a
 * signal buffer that holds the owned rows first and then the ghost rows the
 * exchange writes. */
typedef struct gift_chain_desc {
  const float* s;  /* fp32 s_sigma = 1/sqrt(d + sigma) of the rows processed (indexed by row) */
  double sigma;
  int cont;        /* slot of this chain in zout, -1 when the chain ends at this hop */
  int has_term;    /* a FilterTerm of this chain completes at this hop */
  double alpha;    /* its weight */
} gift_chain_desc;

typedef struct gift_hop_desc {
  int64_t row_begin, row_end; /* rows processed */
  int fin, fout;              /* floats per signal row in / out (1, 2, 4; fout 0 = none) */
  int wcols, nch;             /* signal columns per chain, chains packed in zin */
  const float* zin;           /* [*, fin], indexed by column id */
  float* zout;                /* [*, fout], indexed by row */
  const float* part_in;       /* split hop: partial row sums [*, fin] added first, or NULL */
  float* part_out;            /* split hop: write raw row sums here, no epilogue, or NULL */
  gift_chain_desc chain[4];
  float* acc;                 /* [*, wcols] fp32 bank accumulator */
  int acc_read, is_final;
  int out_dtype;
  void* out;
  int64_t out_ld, out_c0;
  const uint8_t* fixed_mask;
  const double* fixed_pos;
  double region[4];
} gift_hop_desc;

int gift_csr_scale(gift_ctx* ctx, gift_csr* csr, double sigma, const double** d_s64, const float** d_s32);
int gift_csr_weights32(gift_ctx* ctx, gift_csr* csr, const float** d_w32);
/* A (possibly rectangular) row block: copies caller arrays, no canonicalisation. */
int gift_csr_from_arrays(gift_ctx* ctx, int64_t n_rows, int64_t nnz, const int64_t* d_indptr,
                         const int32_t* d_indices, const double* d_values, gift_csr** out);
int gift_hop_fp32(gift_ctx* ctx, gift_csr* csr, const gift_hop_desc* desc);
/* z[i, j*wcols + c] = s_j[i] * g[i*ld + c0 + c] for j < nch, c < wcols; F floats per row. */
int gift_pack_fp32(gift_ctx* ctx, int64_t n, int wcols, int nch, const float* const* h_s, int in_dtype,
                   const void* d_g, int64_t ld, int64_t c0, int F, float* d_z);
/* Row sharding of a resident graph (shard.py), all on the device:
 * nnz-balanced contiguous row bounds for `world` ranks (h_bounds[world + 1],
 * host), and the split of rows [r0, r1) into a LOCAL block (columns in
 * [r0, r1), renumbered col - r0) and a GHOST block (other columns, renumbered
 * (r1 - r0) + rank among the block's distinct ghost columns; their global ids
 * from gift_csr_ext_ids).  Entry order and fp64 values are kept bit for bit. */
int gift_csr_row_bounds(gift_ctx* ctx, const gift_csr* csr, int world, int64_t* h_bounds);
int gift_csr_split_rows(gift_ctx* ctx, const gift_csr* csr, int64_t r0, int64_t r1, gift_csr** local,
                        gift_csr** ghost);
int gift_csr_ext_ids(const gift_csr* ghost, const int64_t** d_ids, int64_t* n_ids);
/* dst[r, :] = src[idx[r], :] for F floats per row (halo send buffers). */
int gift_gather_rows_f32(gift_ctx* ctx, int64_t n_idx, int F, const int64_t* d_idx, const float* d_src,
                         float* d_dst);
/* Ghost rows over NVLink peer memory instead of a collective (csrc/peer.cu;
 * the reference has no distributed code -- this shards gift.py:73-95 over
 * GPUs).  A rank's signal buffers live in plain device allocations
 * (gift_peer_alloc, zero-filled) whose CUDA IPC handle (64 bytes) the other
 * ranks' processes open once (gift_peer_open: peer access over NVLink).
 * gift_pull_rows_f32 copies, for every ghost row i,
 *   dst[i, :F] = peers[src_rank[i]][src_row[i], :F]
 * (d_peers: device array of one base pointer per rank) on a stream forked
 * from the context's stream; gift_pull_join makes the context's stream wait
 * for it, so work enqueued in between (the local part of the hop) overlaps
 * the transfer.  The caller orders ranks with a per-hop barrier (shard.py). */
#define GIFT_PEER_HANDLE_BYTES 64
int gift_peer_alloc(gift_ctx* ctx, int64_t bytes, void** d_ptr, unsigned char* h_handle);
int gift_peer_open(gift_ctx* ctx, const unsigned char* h_handle, void** d_ptr);
int gift_peer_close(gift_ctx* ctx, void* d_ptr);
int gift_peer_free(gift_ctx* ctx, void* d_ptr);
int gift_pull_rows_f32(gift_ctx* ctx, int64_t n_rows, int F, const void* const* d_peers, const int32_t* d_src_rank,
                       const int64_t* d_src_row, float* d_dst);
int gift_pull_join(gift_ctx* ctx);

/* ---- placement metrics: consumers of the filter output --
 * fp64, fixed reduction trees (deterministic; numpy's pairwise / BLAS order
 * is not reproduced, agreement ~1e-15 relative). */
/* quadratic_wirelength(adj, g)  metrics.py:63-74; d_g fp64 [n, 2]. */
int gift_quadratic_wirelength(gift_ctx* ctx, const gift_csr* adj, const double* d_g, double* h_out);
/* laplacian(adj) = D - A  graph.py:161-164 (bit-exact: zeros dropped like csr_minus_csr). */
int gift_laplacian(gift_ctx* ctx, gift_csr* adj, gift_csr** out);
/* rayleigh_smoothness(lap, col, center)  metrics.py:77-92 -> numerator c^T L c and
 * denominator c^T c (the caller raises ZeroSignalError on a ~0 denominator). */
int gift_rayleigh_parts(gift_ctx* ctx, const gift_csr* lap, const double* d_col, int center, double* h_num,
                        double* h_den);
/* hpwl(design, g)  metrics.py:95-112; pin offsets nullable (zero). */
int gift_hpwl(gift_ctx* ctx, int64_t n_nets, const int64_t* d_net_start, const int32_t* d_pin_cell,
              const double* d_pin_dx, const double* d_pin_dy, const double* d_g, double* h_out);

/* ---- .pl writer: write_placement  netlist.py:503-522 --
 * Formats the Bookshelf placement text byte-identically to the reference:
 * "UCLA pl 1.0\n\n", then per cell i in order
 * "<name>\t<llx>\t<lly>\t: N[ /FIXED]\n" with llx = cx - width/2,
 * lly = cy - height/2 (fp64) printed like Python's f"{v:.6f}" (correctly
 * rounded, ties to even, "-0.000000", "nan", "inf").  d_pos: fp64 [n, 2]
 * centres; d_width/d_height nullable (1.0); d_fixed nullable (no /FIXED).
 * Names: d_names + d_name_off[n + 1] (concatenated bytes), or, when d_names is
 * NULL, "<h_name_prefix><i>" (the FlatDesign / benchgen convention "c<i>").
 * d_out == NULL: only *h_len = exact text size.  Otherwise d_out must hold
 * cap >= that size; the text is written and *h_len set.  |coordinate| >= 2^107
 * is rejected (GIFT_ERR_VALUE) instead of printed inexactly. */
int gift_format_placement(gift_ctx* ctx, int64_t n, const double* d_pos, const double* d_width,
                          const double* d_height, const uint8_t* d_fixed, const char* d_names,
                          const int64_t* d_name_off, const char* h_name_prefix, char* d_out, int64_t cap,
                          int64_t* h_len);

/* ---- Bookshelf reader: parse_design  netlist.py:418-458 --
 * Parses the .nodes, .nets and .pl texts (host bytes, as read from disk; the
 * .aux manifest and .scl rows are the caller's) on the device with the
 * reference's semantics: data lines (comments, blanks, "UCLA" headers
 * skipped; universal newlines), cell ids in .nodes order, NetDegree blocks,
 * pin offsets after the first ':' token, the last .pl line of a cell wins,
 * fixed = "terminal" or /FIXED, fixed centre = lower-left + size / 2.
 * Numbers follow Python float()/int() exactly.  On the first malformed line
 * (in line order, as the reference raises) the call fails with
 * GIFT_ERR_PARSE and gift_last_error() = "<file 0/1/2>\t<lineno>\t<code>\t
 * <value>\t<text>" (codes in paper_2502_17632_b200/bookshelf.py). */
int gift_bookshelf_parse(gift_ctx* ctx, const char* h_nodes, int64_t nodes_len, const char* h_nets,
                         int64_t nets_len, const char* h_pl, int64_t pl_len, gift_bookshelf** out);
/* h_sizes[10] = n_cells, n_nets, n_pins, n_fixed, NumTerminals declared (-1: none),
 * cell-name bytes, net-name bytes, .pl lines naming undeclared cells, cells with a
 * .pl line, 0;  h_bbox[4] = lower-left/upper-right of the placed rectangles. */
int gift_bookshelf_info(const gift_bookshelf* bs, int64_t* h_sizes, double* h_bbox);
/* Device views (valid until destroy): the pin table feeds gift_build_clique_graph. */
int gift_bookshelf_device(const gift_bookshelf* bs, const int64_t** d_net_start, const int32_t** d_pin_cell,
                          const double** d_pin_dx, const double** d_pin_dy, const double** d_width,
                          const double** d_height, const uint8_t** d_fixed, const double** d_fixed_pos);
/* Copy out to host arrays (each pointer nullable): net_start [n_nets+1], pin_cell /
 * pin_dx / pin_dy [n_pins], width / height / fixed [n_cells], fixed_pos [n_cells, 2]
 * (NaN on movable rows), names as bytes + [count+1] offsets. */
int gift_bookshelf_copy(gift_ctx* ctx, const gift_bookshelf* bs, int64_t* h_net_start, int32_t* h_pin_cell,
                        double* h_pin_dx, double* h_pin_dy, double* h_width, double* h_height, uint8_t* h_fixed,
                        double* h_fixed_pos, char* h_cell_names, int64_t* h_cell_name_off, char* h_net_names,
                        int64_t* h_net_name_off);
int gift_bookshelf_destroy(gift_ctx* ctx, gift_bookshelf* bs);

#ifdef __cplusplus
}
#endif
#endif /* GIFT_B200_H */
