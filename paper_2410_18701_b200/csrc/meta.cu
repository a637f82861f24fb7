// meta.cu -- a1 mask update, a2 KV append, and the mask/metadata side of the
// splice (a4 remove+release, a5 insert, a7 compaction).
//
// The device keeps the paper's logical state: S (shared seq_length),
// lens/pad_start per slot (pad_start = the paper's `index`) and the 0-1
// attention_mask [slots][max_ctx] in logical columns.  Splice kernels get
// the authoritative post-operation metadata from the host mirror as kernel
// parameters; the decode-step kernels (mask update, append) read and advance the
// device copies so that a whole decode iteration can be captured in a CUDA graph.
#include "common.cuh"
#include "kernels.h"

namespace baton {
namespace {

// a1 -- P:L96 "add a column with the value of all 1" (0 for empty rows, C6)
__global__ void mask_update_kernel(uint8_t *__restrict__ mask, int32_t *__restrict__ S,
                                   int32_t *__restrict__ lens, int slots, int max_ctx) {
    griddep_wait();
    griddep_launch_dependents();
    const int s_old = *S;
    for (int b = threadIdx.x; b < slots; b += blockDim.x) {
        const int L = lens[b];
        const bool occ = L > 0;
        mask[(size_t)b * max_ctx + s_old] = occ ? 1 : 0;
        if (occ) lens[b] = L + 1;
    }
    __syncthreads();
    if (threadIdx.x == 0) *S = s_old + 1;
}

// a2 -- P:L96 "appends ... to KV_Cache": row lens[b]-1 of every kv head of b.
__global__ void append_kv_kernel(uint4 *__restrict__ k, uint4 *__restrict__ v,
                                 const uint4 *__restrict__ kn, const uint4 *__restrict__ vn,
                                 const int32_t *__restrict__ lens, int kv_heads, int vec_per_row,
                                 int max_ctx) {
    griddep_wait();
    griddep_launch_dependents();
    const int b = blockIdx.x, g = blockIdx.y;
    const int L = lens[b];
    if (L <= 0) return;
    const size_t dst = (((size_t)b * kv_heads + g) * max_ctx + (L - 1)) * vec_per_row;
    const size_t src = ((size_t)b * kv_heads + g) * vec_per_row;
    for (int i = threadIdx.x; i < vec_per_row; i += blockDim.x) {
        k[dst + i] = kn[src + i];
        v[dst + i] = vn[src + i];
    }
}

struct MaskSpliceParams {
    uint8_t *mask;
    int32_t *d_S, *d_lens, *d_pad;
    int slots, max_ctx, nops, S;
    int32_t lens[MAX_SLOTS];
    int32_t pad[MAX_SLOTS];
    MaskOp ops[MAX_MASK_OPS];
};

// One CTA per mask row.  The op list is a composition of whole-row transforms
// applied in order:
//   ZERO_ROW    P:L105  the finished query's row := 0
//   SHIFT_LEFT  P:L124  release: column j takes column j+p, tail filled with 0
//   SHIFT_RIGHT P:L137  left expansion by e: column j takes j-e, front filled with 0
//   SET_ROW     P:L137  embedded query: 0 on [0, pad), 1 on [pad, S)
//   SET_CELL    NEXT-1  one column := 1
// Every output column is resolved on its own by walking the list BACKWARDS: a
// shift maps the column to its source column (or to the fill 0), a row op of this
// row fixes the value.  A column that survives every op takes the ORIGINAL row's
// value at its source column.  So the original row is staged once in shared memory
// (max_ctx bytes; the launcher opts in above 48 KB) and no per-op pass or barrier
// is needed.
__global__ void mask_splice_kernel(const __grid_constant__ MaskSpliceParams p) {
    extern __shared__ uint8_t row_buf[];
    const int b = blockIdx.x;
    uint8_t *row = p.mask + (size_t)b * p.max_ctx;
    for (int j = threadIdx.x * 16; j < p.max_ctx; j += blockDim.x * 16)      // max_ctx % 16 == 0
        *reinterpret_cast<uint4 *>(row_buf + j) = *reinterpret_cast<const uint4 *>(row + j);
    __syncthreads();
    for (int j = threadIdx.x; j < p.max_ctx; j += blockDim.x) {
        int c = j;
        int val = -1;
        for (int i = p.nops - 1; i >= 0 && val < 0; --i) {
            const MaskOp op = p.ops[i];
            switch (op.kind) {
                case MOP_ZERO_ROW:
                    if (op.slot == b) val = 0;
                    break;
                case MOP_SHIFT_LEFT:
                    c += op.a;
                    if (c >= p.max_ctx) val = 0;
                    break;
                case MOP_SHIFT_RIGHT:
                    if (c < op.a) val = 0;
                    else c -= op.a;
                    break;
                case MOP_SET_CELL:
                    if (op.slot == b && c == op.a) val = 1;
                    break;
                default:   // MOP_SET_ROW
                    if (op.slot == b) val = (c >= op.a && c < op.b) ? 1 : 0;
                    break;
            }
        }
        row[j] = (uint8_t)(val < 0 ? row_buf[c] : val);
    }
    if (b == 0) {
        for (int s = threadIdx.x; s < p.slots; s += blockDim.x) {
            p.d_lens[s] = p.lens[s];
            p.d_pad[s] = p.pad[s];
        }
        if (threadIdx.x == 0) *p.d_S = p.S;
    }
}

struct MaskMoveParams {
    uint8_t *mask;
    int32_t *d_S, *d_lens, *d_pad;
    int slots, max_ctx, nmoves, S;
    int32_t lens[MAX_SLOTS];
    int32_t pad[MAX_SLOTS];
    int32_t src[MAX_SLOTS];
    int32_t dst[MAX_SLOTS];
};

// a7 -- one CTA per move: copy row src -> dst, then zero src (dst rows are free
// rows, src rows distinct, so moves are independent).  CTA 0 also writes metadata.
__global__ void mask_move_kernel(const __grid_constant__ MaskMoveParams p) {
    const int i = blockIdx.x;
    if (i < p.nmoves) {
        uint8_t *s = p.mask + (size_t)p.src[i] * p.max_ctx;
        uint8_t *d = p.mask + (size_t)p.dst[i] * p.max_ctx;
        for (int j = threadIdx.x; j < p.max_ctx; j += blockDim.x) {
            d[j] = s[j];
            s[j] = 0;
        }
    }
    if (i == 0) {
        for (int s = threadIdx.x; s < p.slots; s += blockDim.x) {
            p.d_lens[s] = p.lens[s];
            p.d_pad[s] = p.pad[s];
        }
        if (threadIdx.x == 0) *p.d_S = p.S;
    }
}

}  // namespace

cudaError_t launch_mask_update(uint8_t *mask, int32_t *S, int32_t *lens, int slots, int max_ctx,
                               cudaStream_t s) {
    return launch_pdl(mask_update_kernel, dim3(1), dim3(256), 0, s, mask, S, lens, slots, max_ctx);
}

cudaError_t launch_append_kv(void *k_layer, void *v_layer, const void *k_new, const void *v_new,
                             const int32_t *lens, int slots, int kv_heads, int head_dim,
                             int max_ctx, cudaStream_t s) {
    const int vpr = head_dim / 8;
    return launch_pdl(append_kv_kernel, dim3(slots, kv_heads), dim3(vpr < 32 ? 32 : vpr), 0, s,
                      static_cast<uint4 *>(k_layer), static_cast<uint4 *>(v_layer),
                      static_cast<const uint4 *>(k_new), static_cast<const uint4 *>(v_new), lens,
                      kv_heads, vpr, max_ctx);
}

cudaError_t launch_mask_splice(uint8_t *mask, int slots, int max_ctx, const MaskOp *ops, int nops,
                               int32_t *d_S, int32_t *d_lens, int32_t *d_pad, int S,
                               const int32_t *lens, const int32_t *pad, cudaStream_t s) {
    if (slots > MAX_SLOTS || nops > MAX_MASK_OPS) return cudaErrorInvalidValue;
    MaskSpliceParams p;
    p.mask = mask;
    p.d_S = d_S;
    p.d_lens = d_lens;
    p.d_pad = d_pad;
    p.slots = slots;
    p.max_ctx = max_ctx;
    p.nops = nops;
    p.S = S;
    for (int i = 0; i < slots; ++i) {
        p.lens[i] = lens[i];
        p.pad[i] = pad[i];
    }
    for (int i = 0; i < nops; ++i) p.ops[i] = ops[i];
    cudaError_t e = ensure_smem_attr(mask_splice_kernel, (size_t)max_ctx);
    if (e != cudaSuccess) return e;
    mask_splice_kernel<<<slots, 256, max_ctx, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_mask_move(uint8_t *mask, int slots, int max_ctx, const int32_t *src,
                             const int32_t *dst, int nmoves, int32_t *d_S, int32_t *d_lens,
                             int32_t *d_pad, int S, const int32_t *lens, const int32_t *pad,
                             cudaStream_t s) {
    if (slots > MAX_SLOTS || nmoves > MAX_SLOTS) return cudaErrorInvalidValue;
    MaskMoveParams p;
    p.mask = mask;
    p.d_S = d_S;
    p.d_lens = d_lens;
    p.d_pad = d_pad;
    p.slots = slots;
    p.max_ctx = max_ctx;
    p.nmoves = nmoves;
    p.S = S;
    for (int i = 0; i < slots; ++i) {
        p.lens[i] = lens[i];
        p.pad[i] = pad[i];
    }
    for (int i = 0; i < nmoves; ++i) {
        p.src[i] = src[i];
        p.dst[i] = dst[i];
    }
    mask_move_kernel<<<nmoves > 0 ? nmoves : 1, 256, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace baton
