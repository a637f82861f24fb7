// decode_gqa.cu -- a3 dispatch for grouped-query attention (configs[3]: 64 q heads
// / 8 kv heads) and the split-K merge of its partials.
//
// The attention itself is decode_gqa_tc_kernel (decode_gqa_tc.cu: tcgen05.mma with
// TMEM accumulators, one work item = (slot, kv head, 256-key chunk)).  A (slot, q
// head) with one chunk is written by it directly; otherwise its chunks leave fp32
// split-K partials (same workspace layout as decode_attention.cu) and
// decode_combine_kernel, PDL-chained behind the attention launch, merges them in
// ascending chunk order.  The combine triggers its dependents right after its start,
// so the NEXT layer's launch streams its first K/V ring while the combine runs.
//
// The round-1 mma.sync kernel and the pipeline sweep variants live in
// csrc/experiments/ and are compiled only with BATON_EXPERIMENTS=1
// (python -m paper_2410_18701_b200.build --experiments).
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "gqa_merge.cuh"
#include "sched.cuh"
#include "tma.h"

namespace baton {

namespace {

constexpr int D = 128;
constexpr int GS = 8;                       // q heads per kv head

BATON_DEV uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 b = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t *>(&b);
}

// Split-K merge for multi-chunk queries.  Grid = one 4-warp CTA per SM (a GQA CTA
// keeps two warps on one SM sub-partition; more combine warps resident there would
// block the next layer's CTA from entering until the combine drains).  The merge
// itself is gqa_merge_pairs (gqa_merge.cuh), shared with the decode-step path that
// runs it at the start of the next layer's launch.
__global__ void __launch_bounds__(128) decode_combine_kernel(const int32_t *__restrict__ lens,
                                                             const float *__restrict__ partial,
                                                             __nv_bfloat16 *__restrict__ out, int B,
                                                             int Hq, int max_chunks) {
    // Trigger at once: the next layer's launch may begin its early phase (work list,
    // K/V ring) while this combine -- and the attention launch before it -- finish.
    // Safe because that phase reads only lens/pad/mask and cache rows other than
    // lens-1, which neither launch writes; everything it writes waits for us.
    griddep_launch_dependents();
    griddep_wait();
    gqa_merge_pairs(lens, partial, out, B, Hq, max_chunks, blockIdx.x * 4 + (threadIdx.x >> 5),
                    gridDim.x * 4, threadIdx.x & 31);
}

#if BATON_EXPERIMENTS
// The same merge, started before the attention grid completes: a CTA owns whole
// (slot, kv group)s -- 4 warps x 2 pairs = the group's 8 q heads -- and polls the
// group's ticket (chunks published by the attention kernel's P.V issuers, release
// -> acquire) instead of waiting for the grid, so the merges run under the attention
// tail.  The CTA resets the ticket once all 4 warps have merged the group.  Resident
// beside the attention CTA (128 threads x 72 registers fit next to 384 x 144).
__global__ void __launch_bounds__(128) decode_combine_spin_kernel(const int32_t *__restrict__ lens,
                                                                  const float *__restrict__ partial,
                                                                  int32_t *tickets,
                                                                  __nv_bfloat16 *__restrict__ out, int B,
                                                                  int Hq, int max_chunks) {
    griddep_launch_dependents();
    const int lane = threadIdx.x & 31, hl = lane & 15, w = threadIdx.x >> 5;
    const int groups = B * (Hq / GS);
    constexpr int R = D + PREC_PAD, NB = 8;
    for (int gi = blockIdx.x; gi < groups; gi += gridDim.x) {
        const int b = gi / (Hq / GS);
        const int L = lens[b];
        const int nch = (L + CHUNK - 1) / CHUNK;
        if (nch <= 1) continue;                                   // uniform over the CTA
        const int bh0 = gi * GS;
        int32_t *tk = tickets + bh0;
        if (lane == 0) {
            const long long t0 = clock64();
            while (ld_acquire_gpu(tk) < nch) {
                __nanosleep(256);
                if (clock64() - t0 > 60000000000LL) {   // ~30 s: a missing publish traps, not hangs
                    printf("baton watchdog: combine waits on ticket %d (%d of %d)\n", bh0, *tk, nch);
                    __trap();
                }
            }
        }
        __syncwarp();
        const int pair = bh0 + 2 * w + (lane >> 4);
        const float *pp = partial + (size_t)pair * max_chunks * R + hl * 8;
        float Mc = -INFINITY, Lc = 0.f, Oc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        for (int c0 = 0; c0 < nch; c0 += NB) {
            float m[NB], l[NB];
            float4 va[NB], vb[NB];
#pragma unroll
            for (int j = 0; j < NB; ++j) {
                const bool ok = c0 + j < nch;
                const float *r = pp + (ok ? c0 + j : c0) * R;
                m[j] = ok ? __ldcg(r - hl * 8 + D) : -INFINITY;
                l[j] = ok ? __ldcg(r - hl * 8 + D + 1) : 0.f;
                va[j] = __ldcg(reinterpret_cast<const float4 *>(r));
                vb[j] = __ldcg(reinterpret_cast<const float4 *>(r + 4));
            }
            float Mn = Mc;
#pragma unroll
            for (int j = 0; j < NB; ++j) Mn = fmaxf(Mn, m[j]);
            const float al = (Mc == -INFINITY) ? 0.f : ex2(Mc - Mn);
            Lc *= al;
#pragma unroll
            for (int i = 0; i < 8; ++i) Oc[i] *= al;
#pragma unroll
            for (int j = 0; j < NB; ++j) {
                const float f = (m[j] == -INFINITY) ? 0.f : ex2(m[j] - Mn);
                Lc = fmaf(f, l[j], Lc);
                Oc[0] = fmaf(f, va[j].x, Oc[0]);
                Oc[1] = fmaf(f, va[j].y, Oc[1]);
                Oc[2] = fmaf(f, va[j].z, Oc[2]);
                Oc[3] = fmaf(f, va[j].w, Oc[3]);
                Oc[4] = fmaf(f, vb[j].x, Oc[4]);
                Oc[5] = fmaf(f, vb[j].y, Oc[5]);
                Oc[6] = fmaf(f, vb[j].z, Oc[6]);
                Oc[7] = fmaf(f, vb[j].w, Oc[7]);
            }
            Mc = Mn;
        }
        const float inv = Lc > 0.f ? 1.f / Lc : 0.f;
        uint4 wv;
        wv.x = pack_bf16(Oc[0] * inv, Oc[1] * inv);
        wv.y = pack_bf16(Oc[2] * inv, Oc[3] * inv);
        wv.z = pack_bf16(Oc[4] * inv, Oc[5] * inv);
        wv.w = pack_bf16(Oc[6] * inv, Oc[7] * inv);
        *reinterpret_cast<uint4 *>(out + (size_t)pair * D + hl * 8) = wv;
        __syncthreads();                                          // all 8 heads observed the ticket
        if (threadIdx.x == 0) *tk = 0;                            // ready for the next launch
    }
}

#endif  // BATON_EXPERIMENTS

}  // namespace

#if BATON_EXPERIMENTS
cudaError_t launch_gqa_combine_spin(const DecodeArgs &a, cudaStream_t s) {
    const int num_sms = device_sms();
    return launch_pdl(decode_combine_spin_kernel, dim3(num_sms), dim3(128), 0, s, a.lens,
                      (const float *)a.partial, a.tickets, static_cast<__nv_bfloat16 *>(a.out), a.slots,
                      a.q_heads, a.max_chunks);
}
#endif

bool gqa_supported(int q_heads, int kv_heads, int head_dim) {
    return head_dim == D && kv_heads > 0 && q_heads == GS * kv_heads;
}

cudaError_t launch_gqa_combine(const DecodeArgs &a, cudaStream_t s) {
    const int num_sms = device_sms();
    return launch_pdl(decode_combine_kernel, dim3(num_sms), dim3(128), 0, s, a.lens,
                      (const float *)a.partial, static_cast<__nv_bfloat16 *>(a.out), a.slots,
                      a.q_heads, a.max_chunks);
}

#if BATON_EXPERIMENTS
cudaError_t launch_gqa_experiment(int variant, const DecodeArgs &a, cudaStream_t s);
#endif

cudaError_t launch_decode_gqa(const DecodeArgs &a, cudaStream_t s) {
    // tcgen05 kernel + the PDL combine.  Experiment builds: BATON_GQA_VARIANT selects
    // the mma.sync kernel's sweep variants (0, 1, 5, 6, 9, 10) or the tcgen05 kernel
    // with the in-kernel last-arriver merge (21, needs max_chunks <= 32;
    // profiles/r01_gqa_engine_sweep.md)
#if BATON_EXPERIMENTS
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("BATON_GQA_VARIANT");
        v = e ? atoi(e) : 20;
    }
    if (v == 21 && a.max_chunks <= 32) return launch_decode_gqa_tc(a, s, true);
    // 22: the attention launch alone, no split-K merge (WRONG outputs for multi-chunk
    // queries; measures what the combine hop costs in the decode-step chain)
    if (v == 22) return launch_decode_gqa_tc(a, s, false);
    // 23: published tickets + a combine that merges each (slot, kv group) as soon as it
    // is complete, under the attention tail
    if (v == 23) {
        cudaError_t e = launch_decode_gqa_tc(a, s, false, true);
        if (e != cudaSuccess || a.dry) return e;
        return launch_gqa_combine_spin(a, s);
    }
    if (v != 20 && v != 21) return launch_gqa_experiment(v, a, s);
#endif
    cudaError_t e = launch_decode_gqa_tc(a, s, false);
    if (e != cudaSuccess || a.dry || a.defer_merge) return e;
    return launch_gqa_combine(a, s);
}

}  // namespace baton
