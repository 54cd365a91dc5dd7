// peer.cu -- ghost rows read straight from the neighbours' signal buffers
// (NVLink peer memory) for the row-sharded bank (shard.py).
//
// One process per GPU.  A rank keeps its two signal buffers [owned rows |
// ghost rows] x F floats in plain cudaMalloc allocations and publishes their
// CUDA IPC handles; every other rank opens them once, which maps the memory
// into its address space with peer access over NVLink / NVSwitch.  Per hop a
// rank then PULLS the rows its ghost block references from the owners'
// buffers with one kernel of peer loads -- no pack kernel on the owner, no
// staging buffer, no collective on the data path -- on a forked stream, so
// the transfer runs under the local part of the hop; the ghost part of the
// hop joins it.  Ordering between ranks (an owner's rows are complete before
// anyone pulls them, and are not overwritten while someone still pulls) is a
// stream-ordered barrier per hop, issued by the host side (shard.py).
//
// The pull moves each ghost row once per hop (halo + fixed objects: ~1e5
// rows of 8-16 B at c4), whereas gathering peer rows from inside the ghost
// hop would cross the link once per matrix entry that references them
// (~40x more bytes on c4), so the hop kernels keep reading local memory.
#include <cuda_runtime.h>

#include "common.cuh"

namespace gift {

namespace {

constexpr int kBlock = 256;

// dst[i, :] = peers[src_rank[i]][src_row[i], :], V = one row (float / float2 /
// float4).  Ghost ids are grouped by owner and ascending, so consecutive
// threads mostly read consecutive peer rows (the halo): coalesced link reads.
// ld.global.cg: peer lines must not linger in this SM's L1 across hops.
template <typename V>
__global__ void k_pull_rows(int64_t n, const V* const* __restrict__ peers, const int32_t* __restrict__ src_rank,
                            const int64_t* __restrict__ src_row, V* __restrict__ dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const V* base = peers[src_rank[i]];
    dst[i] = __ldcg(base + src_row[i]);
  }
}

void ensure_pull_stream(Ctx* ctx) {
  if (ctx->pull) return;
  GIFT_CUDA(cudaStreamCreateWithFlags(&ctx->pull, cudaStreamNonBlocking));
  GIFT_CUDA(cudaEventCreateWithFlags(&ctx->pull_fork, cudaEventDisableTiming));
  GIFT_CUDA(cudaEventCreateWithFlags(&ctx->pull_done, cudaEventDisableTiming));
}

}  // namespace

// plain device allocation (IPC handles do not exist for pool memory), zeroed
void* peer_alloc(Ctx* ctx, size_t bytes, cudaIpcMemHandle_t* handle) {
  void* p = nullptr;
  GIFT_CUDA(cudaMalloc(&p, bytes > 0 ? bytes : 16));
  GIFT_CUDA(cudaMemsetAsync(p, 0, bytes > 0 ? bytes : 16, ctx->stream));
  GIFT_CUDA(cudaStreamSynchronize(ctx->stream));
  if (handle) {
    const cudaError_t e = cudaIpcGetMemHandle(handle, p);
    if (e != cudaSuccess) {
      cudaFree(p);
      GIFT_CUDA(e);
    }
  }
  return p;
}

void* peer_open(Ctx* ctx, const cudaIpcMemHandle_t& handle) {
  (void)ctx;
  void* p = nullptr;
  GIFT_CUDA(cudaIpcOpenMemHandle(&p, handle, cudaIpcMemLazyEnablePeerAccess));
  return p;
}

// starts the pull on the context's pull stream, ordered after everything
// already enqueued on ctx->stream; pull_join makes ctx->stream wait for it
void pull_rows_f32(Ctx* ctx, int64_t n, int F, const void* const* d_peers, const int32_t* d_src_rank,
                   const int64_t* d_src_row, float* d_dst) {
  if (F != 1 && F != 2 && F != 4) throw_error(GIFT_ERR_VALUE, "pull_rows_f32: F must be 1, 2 or 4");
  ensure_pull_stream(ctx);
  GIFT_CUDA(cudaEventRecord(ctx->pull_fork, ctx->stream));
  GIFT_CUDA(cudaStreamWaitEvent(ctx->pull, ctx->pull_fork, 0));
  if (n > 0) {
    const unsigned grid = grid_for(n, kBlock);
    if (F == 4)
      k_pull_rows<float4><<<grid, kBlock, 0, ctx->pull>>>(n, reinterpret_cast<const float4* const*>(d_peers), d_src_rank,
                                                          d_src_row, reinterpret_cast<float4*>(d_dst));
    else if (F == 2)
      k_pull_rows<float2><<<grid, kBlock, 0, ctx->pull>>>(n, reinterpret_cast<const float2* const*>(d_peers), d_src_rank,
                                                          d_src_row, reinterpret_cast<float2*>(d_dst));
    else
      k_pull_rows<float><<<grid, kBlock, 0, ctx->pull>>>(n, reinterpret_cast<const float* const*>(d_peers), d_src_rank,
                                                         d_src_row, d_dst);
    GIFT_LAUNCH_CHECK(ctx);
  }
  GIFT_CUDA(cudaEventRecord(ctx->pull_done, ctx->pull));
  ctx->pull_pending = true;
}

void pull_join(Ctx* ctx) {
  if (!ctx->pull_pending) return;
  GIFT_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->pull_done, 0));
  ctx->pull_pending = false;
}

}  // namespace gift
