/* TEST INFRASTRUCTURE ONLY — types shared by the CPU numeric oracle
 * (llama_ref.c, the checker) and the batched CPU baseline (cpu_decode.c,
 * bench.py's cpu_baseline / --impl reference legs). */
#ifndef MESH_LLAMA_REF_H
#define MESH_LLAMA_REF_H

#include <stdint.h>
#include <string.h>

typedef struct {
    int n_layers, d, n_heads, n_kv, dh, ff, vocab, tied, max_seq;
    float rope_theta, eps;
} ora_shape;

typedef struct {
    uint16_t *wq, *wk, *wv, *wo, *wg, *wu, *wd; /* logical row-major per layer */
    float *ga, *gm;
} ora_layer;

typedef struct ora_model {
    ora_shape s;
    uint64_t seed;
    int round_act;
    uint16_t* emb;
    uint16_t* lm; /* == emb when tied */
    float* gf;
    ora_layer* layers;
    float* cosv; /* [max_seq][dh/2] */
    float* sinv;
} ora_model;

typedef struct ora_seq {
    int len;
    float* k; /* [L][max_seq][n_kv][dh] (values already rounded when round_act) */
    float* v;
} ora_seq;

static inline uint16_t f2bf(float f) { /* round to nearest even */
    uint32_t u;
    memcpy(&u, &f, 4);
    if ((u & 0x7f800000u) == 0x7f800000u) return (uint16_t)(u >> 16); /* inf / nan passthrough */
    uint32_t lsb = (u >> 16) & 1u;
    u += 0x7fffu + lsb;
    return (uint16_t)(u >> 16);
}
static inline float bf2f(uint16_t b) {
    uint32_t u = (uint32_t)b << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

#endif
