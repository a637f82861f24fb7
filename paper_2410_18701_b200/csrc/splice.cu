// splice.cu -- the K/V byte movement of the splice: a5 embedding of prefilled
// K/V, a6 extraction to a stash, a7 compaction moves.
//
// In the slot-relative layout every one of these is, per (layer, kv head, K|V),
// one contiguous run of `rows * head_dim` bf16 on both sides, so the whole
// splice of an iteration is a batch of equal-shape contiguous copies: ONE launch,
// grid (pieces, layer*kv_head*2, job), 16-B vector loads/stores, 4 loads in
// flight per thread before the stores (bytes in flight ~ 64 KB per SM).
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace baton {
namespace {

constexpr int CP_THREADS = 256;
constexpr int CP_UNROLL = 4;
constexpr int CP_PIECE_VEC = CP_THREADS * CP_UNROLL;   // 16-B vectors per block piece (16 KB)

struct CopyParams {
    CopyJob jobs[MAX_SPLICE_JOBS];
    int kv_heads, vec_per_row, elems_per_row;
};

__global__ void __launch_bounds__(CP_THREADS) kv_copy_kernel(const __grid_constant__ CopyParams p) {
    const CopyJob &j = p.jobs[blockIdx.z];
    const int seg = blockIdx.y;            // ((layer * kv_heads) + head) * 2 + kv
    const int kv = seg & 1;
    const int lh = seg >> 1;
    const int layer = lh / p.kv_heads;
    const int head = lh - layer * p.kv_heads;
    const int64_t nvec = (int64_t)j.rows * p.vec_per_row;
    const int64_t v0 = (int64_t)blockIdx.x * CP_PIECE_VEC;
    if (v0 >= nvec) return;
    const __nv_bfloat16 *src =
        static_cast<const __nv_bfloat16 *>(kv ? j.src_v : j.src_k) + layer * j.src_ls + head * j.src_hs;
    __nv_bfloat16 *dst =
        static_cast<__nv_bfloat16 *>(kv ? j.dst_v : j.dst_k) + layer * j.dst_ls + head * j.dst_hs;
    const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
    uint4 *d4 = reinterpret_cast<uint4 *>(dst);
    uint4 r[CP_UNROLL];
#pragma unroll
    for (int u = 0; u < CP_UNROLL; ++u) {
        const int64_t i = v0 + u * CP_THREADS + threadIdx.x;
        if (i < nvec) r[u] = __ldcs(s4 + i);           // streamed: read once
    }
#pragma unroll
    for (int u = 0; u < CP_UNROLL; ++u) {
        const int64_t i = v0 + u * CP_THREADS + threadIdx.x;
        if (i < nvec) d4[i] = r[u];
    }
}

struct ShapeAppendParams {
    __nv_bfloat16 *k, *v;
    const __nv_bfloat16 *kn, *vn;
    int32_t row0[MAX_SLOTS];
    int layers, slots, kv_heads, vec_per_row, max_ctx, W;
};

// grid-stride over (layer, slot, token, kv head, 16-B vector) of the token-major
// source; each destination row is contiguous in the slot-relative cache
__global__ void __launch_bounds__(256) shape_append_kernel(const __grid_constant__ ShapeAppendParams p) {
    const int64_t per_tok = (int64_t)p.kv_heads * p.vec_per_row;
    const int64_t total = (int64_t)p.layers * p.slots * p.W * per_tok;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t tok = i / per_tok;                 // (layer, slot, t)
        const int rem = (int)(i - tok * per_tok);
        const int g = rem / p.vec_per_row, c = rem - g * p.vec_per_row;
        const int t = (int)(tok % p.W);
        const int64_t ls = tok / p.W;
        const int b = (int)(ls % p.slots), l = (int)(ls / p.slots);
        const int r0 = p.row0[b];
        if (r0 < 0) continue;
        const size_t dst = ((((size_t)l * p.slots + b) * p.kv_heads + g) * p.max_ctx + r0 + t) * p.vec_per_row + c;
        reinterpret_cast<uint4 *>(p.k)[dst] = reinterpret_cast<const uint4 *>(p.kn)[i];
        reinterpret_cast<uint4 *>(p.v)[dst] = reinterpret_cast<const uint4 *>(p.vn)[i];
    }
}

}  // namespace

cudaError_t launch_shape_append(void *k_cache, void *v_cache, const void *k_new, const void *v_new,
                                const int32_t *row0, int layers, int slots, int kv_heads, int head_dim,
                                int max_ctx, int W, cudaStream_t s) {
    if (slots > MAX_SLOTS || head_dim % 8) return cudaErrorInvalidValue;
    ShapeAppendParams p;
    p.k = static_cast<__nv_bfloat16 *>(k_cache);
    p.v = static_cast<__nv_bfloat16 *>(v_cache);
    p.kn = static_cast<const __nv_bfloat16 *>(k_new);
    p.vn = static_cast<const __nv_bfloat16 *>(v_new);
    for (int b = 0; b < slots; ++b) p.row0[b] = row0[b];
    p.layers = layers;
    p.slots = slots;
    p.kv_heads = kv_heads;
    p.vec_per_row = head_dim / 8;
    p.max_ctx = max_ctx;
    p.W = W;
    const int64_t total = (int64_t)layers * slots * W * kv_heads * p.vec_per_row;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t blocks = std::min<int64_t>((total + 255) / 256, (int64_t)sms * 8);
    shape_append_kernel<<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_kv_copy(const CopyJob *jobs, int njobs, int layers, int kv_heads, int head_dim,
                           cudaStream_t s) {
    if (njobs <= 0) return cudaSuccess;
    if (njobs > MAX_SPLICE_JOBS) return cudaErrorInvalidValue;
    CopyParams p;
    int max_rows = 0;
    for (int i = 0; i < njobs; ++i) {
        p.jobs[i] = jobs[i];
        if (jobs[i].rows > max_rows) max_rows = jobs[i].rows;
    }
    if (max_rows == 0) return cudaSuccess;
    p.kv_heads = kv_heads;
    p.vec_per_row = head_dim / 8;
    p.elems_per_row = head_dim;
    const int64_t nvec = (int64_t)max_rows * p.vec_per_row;
    const unsigned pieces = (unsigned)((nvec + CP_PIECE_VEC - 1) / CP_PIECE_VEC);
    dim3 grid(pieces, layers * kv_heads * 2, njobs);
    kv_copy_kernel<<<grid, CP_THREADS, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace baton
