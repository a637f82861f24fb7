// gqa_merge.cuh -- the split-K merge of the GQA decode (a3): for every (slot, q head)
// whose live length spans more than one 256-key chunk, combine the chunk partials
// (o[D], m, l; fp32, written by decode_gqa_tc_kernel) in ascending chunk order -- a
// query's result depends only on its own history (batch invariance) --
// and write the bf16 output row.  Single-chunk queries were written by the attention
// kernel itself.
//
// Warp-collective: warp `gw` of `nw` takes (slot, q head) pairs 2 gw, 2 gw + 1, then
// strides by 2 nw; 16 lanes x 8 dims per pair, eight chunks per L2 round trip with an
// online max.  Used by decode_combine_kernel (its own launch) and, in the decode-step
// graph, by the NEXT layer's attention launch right after its griddepcontrol.wait.
#pragma once
#include "common.cuh"
#include "kernels.h"

namespace baton {

BATON_DEV uint32_t gqa_pack_bf16(float lo, float hi) {
    __nv_bfloat162 b = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t *>(&b);
}

BATON_DEV void gqa_merge_pairs(const int32_t *__restrict__ lens, const float *__restrict__ partial,
                               __nv_bfloat16 *__restrict__ out, int B, int Hq, int max_chunks, int gw,
                               int nw, int lane) {
    constexpr int D = 128, R = D + PREC_PAD, NB = 8;
    const int hl = lane & 15;
    const int npairs = B * Hq;
    for (; gw * 2 < npairs; gw += nw) {
        const int pair = gw * 2 + (lane >> 4);
        const int L = pair < npairs ? lens[pair / Hq] : 0;
        const int nch = (L + CHUNK - 1) / CHUNK;
        if (pair >= npairs || nch <= 1) continue;
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
        uint4 w;
        w.x = gqa_pack_bf16(Oc[0] * inv, Oc[1] * inv);
        w.y = gqa_pack_bf16(Oc[2] * inv, Oc[3] * inv);
        w.z = gqa_pack_bf16(Oc[4] * inv, Oc[5] * inv);
        w.w = gqa_pack_bf16(Oc[6] * inv, Oc[7] * inv);
        *reinterpret_cast<uint4 *>(out + (size_t)pair * D + hl * 8) = w;
    }
}

}  // namespace baton
