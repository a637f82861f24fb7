// keygen.cu -- HARNESS ONLY (not a step of the Baton method): the counter-based
// synthetic value generator of SURVEY.md §8(d), bit-identical to
// baton_inputs/keygen.py (cross-checked in tests/test_gpu_keygen.py).  It lets the
// GPU harness materialise a query's q/k/v history in HBM without a host round trip.
//
//   ctr = (((((kind*128 + layer)*2^20 + qid)*4096 + pos)*64 + head)*128 + dim)
//   u   = splitmix64_mix(seed*PHI + ctr)
//   x   = (int(u >> 40) - 2^23) * 2^(s-23)       -> bf16 RNE
#include "common.cuh"
#include "kernels.h"

namespace baton {
namespace {

constexpr uint64_t PHI = 0x9E3779B97F4A7C15ull;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint16_t keyed_bf16(uint64_t seed, uint64_t kind, uint64_t layer,
                                               uint64_t qid, uint64_t pos, uint64_t head,
                                               uint64_t dim, float scale) {
    uint64_t c = ((((kind * 128 + layer) * (1ull << 20) + qid) * 4096 + pos) * 64 + head) * 128 + dim;
    uint64_t u = mix64(seed * PHI + c);
    int32_t iv = (int32_t)(u >> 40) - (1 << 23);
    float x = (float)iv * scale;   // exact: |iv| < 2^23, scale a power of two
    __nv_bfloat16 h = __float2bfloat16_rn(x);
    return *reinterpret_cast<uint16_t *>(&h);
}

// out[layer][slot][head][dim] for layers [layer0, layer0+layers); qid < 0 -> zeros
__global__ void keygen_tokens_kernel(uint16_t *out, const int32_t *qids, const int32_t *pos,
                                     int n_slots, int heads, int head_dim, int kind, int layer0,
                                     uint64_t seed, float scale, int64_t total) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = i;
        const int d = r % head_dim;
        r /= head_dim;
        const int h = r % heads;
        r /= heads;
        const int b = r % n_slots;
        const int l = (int)(r / n_slots);
        const int q = qids[b];
        out[i] = q < 0 ? 0 : keyed_bf16(seed, kind, layer0 + l, q, pos[b], h, d, scale);
    }
}

// out + l*layer_stride + h*head_stride + p*head_dim + d, positions [pos_begin, pos_begin+n)
__global__ void keygen_history_kernel(uint16_t *out, int layers, int heads, int head_dim, int qid,
                                      int pos_begin, int n, int kind, uint64_t seed, float scale,
                                      int64_t head_stride, int64_t layer_stride, int64_t total) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = i;
        const int d = r % head_dim;
        r /= head_dim;
        const int p = r % n;
        r /= n;
        const int h = r % heads;
        const int l = (int)(r / heads);
        out[l * layer_stride + h * head_stride + (int64_t)p * head_dim + d] =
            keyed_bf16(seed, kind, l, qid, pos_begin + p, h, d, scale);
    }
}

}  // namespace

cudaError_t launch_keygen_tokens(void *out, const int32_t *qids, const int32_t *pos, int layers,
                                 int n_slots, int heads, int head_dim, int kind, int layer0,
                                 uint64_t seed, int scale_exp, cudaStream_t s) {
    const int64_t total = (int64_t)layers * n_slots * heads * head_dim;
    if (total == 0) return cudaSuccess;
    const float scale = ldexpf(1.0f, scale_exp - 23);
    const int blocks = (int)((total + 255) / 256 < 148 * 16 ? (total + 255) / 256 : 148 * 16);
    keygen_tokens_kernel<<<blocks, 256, 0, s>>>(static_cast<uint16_t *>(out), qids, pos, n_slots,
                                                heads, head_dim, kind, layer0, seed, scale, total);
    return cudaGetLastError();
}

cudaError_t launch_keygen_history(void *out, int layers, int heads, int head_dim, int qid,
                                  int pos_begin, int n, int kind, uint64_t seed, int scale_exp,
                                  int64_t head_stride, int64_t layer_stride, cudaStream_t s) {
    const int64_t total = (int64_t)layers * heads * n * head_dim;
    if (total == 0) return cudaSuccess;
    const float scale = ldexpf(1.0f, scale_exp - 23);
    const int blocks = (int)((total + 255) / 256 < 148 * 16 ? (total + 255) / 256 : 148 * 16);
    keygen_history_kernel<<<blocks, 256, 0, s>>>(static_cast<uint16_t *>(out), layers, heads,
                                                 head_dim, qid, pos_begin, n, kind, seed, scale,
                                                 head_stride, layer_stride, total);
    return cudaGetLastError();
}

}  // namespace baton
