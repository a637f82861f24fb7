/*
 * baton_keygen.h -- HARNESS entry points of libbaton (not steps of the Baton
 * method): the counter-based synthetic value generator of SURVEY.md §8(d),
 * bit-identical to baton_inputs/keygen.py.  The benchmark and the full-size
 * parity tests use it to put a query's keyed q/k/v history directly in HBM.
 *
 *   value(seed, kind, layer, qid, pos, head, dim):
 *     ctr = (((((kind*128 + layer)*2^20 + qid)*4096 + pos)*64 + head)*128 + dim)
 *     u   = splitmix64_mix(seed * 0x9E3779B97F4A7C15 + ctr)   (mod 2^64)
 *     x   = (int(u >> 40) - 2^23) * 2^(scale_exp - 23)  -> bf16 round-to-nearest-even
 *   kind: 0 = q, 1 = k, 2 = v.  Field limits: layer < 128, qid < 2^20, pos < 4096,
 *   head < 64, dim < 128.
 * Same error conventions as baton.h.
 */
#ifndef BATON_KEYGEN_H
#define BATON_KEYGEN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* out: device bf16 [layers][n_slots][heads][head_dim] for layers layer0 ..
 * layer0+layers-1; qids, pos: DEVICE int32[n_slots]; a slot with qid < 0 gets zeros. */
int baton_keygen_tokens(void *out, const int32_t *qids, const int32_t *pos, int layers,
                        int n_slots, int heads, int head_dim, int kind, int layer0, uint64_t seed,
                        int scale_exp, void *stream);

/* One query's history for positions [pos_begin, pos_begin + n), layers 0..layers-1:
 * element (l, h, p, d) goes to out + l*layer_stride + h*head_stride + p*head_dim + d
 * (strides in elements).  Dense [layers][heads][n][head_dim]: head_stride = n*head_dim,
 * layer_stride = heads*n*head_dim. */
int baton_keygen_history(void *out, int layers, int heads, int head_dim, int qid, int pos_begin,
                         int n, int kind, uint64_t seed, int scale_exp, int64_t head_stride,
                         int64_t layer_stride, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* BATON_KEYGEN_H */
