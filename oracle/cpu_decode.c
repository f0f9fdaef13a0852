/* TEST INFRASTRUCTURE ONLY — batched CPU decode: the reported CPU baseline
 * (bench.py cpu_baseline and --impl reference legs), NOT the checker.
 *
 * The reference LLM-Mesh artifact prices token steps from tables and has no
 * model arithmetic; its paper ran CPU instances on OpenVINO
 * (PAPER.md:574). So the CPU path that executes the co-located token step is
 * this restatement: the same Llama decoder as llama_ref.c over the same
 * generated weights, but written the way a CPU serving engine runs a decode
 * step: one pass over each weight row serves all B sequences of the batch,
 * fp32 accumulation in 16 independent lanes (AVX2/FMA), OpenMP over rows and
 * over (sequence, head) for attention. Numerics follow llama_ref.c's
 * round_act contract except for accumulation order/precision (fp32 here,
 * double in the checker), which is why the tests never use it. */
#include <math.h>
#include <stdlib.h>

#include "llama_ref.h"

#ifdef _OPENMP
#include <omp.h>
#endif

static inline float rbf_(float f) { return bf2f(f2bf(f)); }

/* Y[b][r] = sum_c W[r][c] X[b][c] for b < B; W bf16 [rows][cols], cols % 16 == 0 */
static void gemv_batch(const uint16_t* W, const float* X, float* Y, int rows, int cols, int B) {
#pragma omp parallel
    {
        float* wf = (float*)aligned_alloc(64, ((size_t)cols * 4 + 63) / 64 * 64);
#pragma omp for schedule(static)
        for (int r = 0; r < rows; ++r) {
            const uint16_t* w = W + (size_t)r * cols;
            for (int c = 0; c < cols; ++c) wf[c] = bf2f(w[c]);
            for (int b = 0; b < B; ++b) {
                const float* x = X + (size_t)b * cols;
                float acc[16] = {0};
                for (int c = 0; c < cols; c += 16)
                    for (int j = 0; j < 16; ++j) acc[j] += wf[c + j] * x[c + j];
                float t = 0.f;
                for (int j = 0; j < 16; ++j) t += acc[j];
                Y[(size_t)b * rows + r] = t;
            }
        }
        free(wf);
    }
}

static void norm_batch(const ora_model* m, const float* H, const float* gamma, float* A, float* rs, int B) {
    const int d = m->s.d;
    for (int b = 0; b < B; ++b) {
        const float* h = H + (size_t)b * d;
        float* a = A + (size_t)b * d;
        float ss = 0.f;
        for (int i = 0; i < d; ++i) ss += h[i] * h[i];
        rs[b] = 1.0f / sqrtf(ss / d + m->s.eps);
        for (int i = 0; i < d; ++i) a[i] = m->round_act ? rbf_(h[i] * gamma[i]) : h[i] * gamma[i];
    }
}

/* One decode step for B sequences (each fed tokens[b] at its own position);
 * next[b] = greedy next token. Returns 0, or -1 if a sequence is full. */
int ora_feed_batch(const ora_model* m, ora_seq** seqs, int B, const int* tokens, int* next) {
    const ora_shape* s = &m->s;
    const int d = s->d, H = s->n_heads, KV = s->n_kv, dh = s->dh, half = dh / 2, ff = s->ff, gq = H / KV;
    for (int b = 0; b < B; ++b)
        if (seqs[b]->len >= s->max_seq) return -1;
    const int wmax = d > ff ? d : ff;
    float* Hs = (float*)malloc(sizeof(float) * B * d);
    float* A = (float*)malloc(sizeof(float) * B * wmax);
    float* Q = (float*)malloc(sizeof(float) * B * H * dh);
    float* K = (float*)malloc(sizeof(float) * B * KV * dh);
    float* V = (float*)malloc(sizeof(float) * B * KV * dh);
    float* AT = (float*)malloc(sizeof(float) * B * H * dh);
    float* O = (float*)malloc(sizeof(float) * B * d);
    float* G = (float*)malloc(sizeof(float) * B * ff);
    float* U = (float*)malloc(sizeof(float) * B * ff);
    float* rs = (float*)malloc(sizeof(float) * B);
    for (int b = 0; b < B; ++b)
        for (int i = 0; i < d; ++i) Hs[(size_t)b * d + i] = bf2f(m->emb[(size_t)tokens[b] * d + i]);
    for (int l = 0; l < s->n_layers; ++l) {
        const ora_layer* L = &m->layers[l];
        norm_batch(m, Hs, L->ga, A, rs, B);
        gemv_batch(L->wq, A, Q, H * dh, d, B);
        gemv_batch(L->wk, A, K, KV * dh, d, B);
        gemv_batch(L->wv, A, V, KV * dh, d, B);
        for (int b = 0; b < B; ++b) {
            ora_seq* q = seqs[b];
            const int pos = q->len;
            const float* cs = m->cosv + (size_t)pos * half;
            const float* sn = m->sinv + (size_t)pos * half;
            float* qv = Q + (size_t)b * H * dh;
            float* kv = K + (size_t)b * KV * dh;
            float* vv = V + (size_t)b * KV * dh;
            for (int i = 0; i < H * dh; ++i) qv[i] *= rs[b];
            for (int i = 0; i < KV * dh; ++i) {
                kv[i] *= rs[b];
                vv[i] *= rs[b];
            }
            for (int hh = 0; hh < H; ++hh)
                for (int i = 0; i < half; ++i) {
                    float x1 = qv[hh * dh + i], x2 = qv[hh * dh + i + half];
                    qv[hh * dh + i] = x1 * cs[i] - x2 * sn[i];
                    qv[hh * dh + i + half] = x2 * cs[i] + x1 * sn[i];
                }
            for (int hh = 0; hh < KV; ++hh)
                for (int i = 0; i < half; ++i) {
                    float x1 = kv[hh * dh + i], x2 = kv[hh * dh + i + half];
                    kv[hh * dh + i] = x1 * cs[i] - x2 * sn[i];
                    kv[hh * dh + i + half] = x2 * cs[i] + x1 * sn[i];
                }
            float* kc = q->k + (size_t)l * s->max_seq * KV * dh;
            float* vc = q->v + (size_t)l * s->max_seq * KV * dh;
            for (int i = 0; i < KV * dh; ++i) {
                kc[(size_t)pos * KV * dh + i] = m->round_act ? rbf_(kv[i]) : kv[i];
                vc[(size_t)pos * KV * dh + i] = m->round_act ? rbf_(vv[i]) : vv[i];
            }
        }
        const float scale = 1.0f / sqrtf((float)dh);
#pragma omp parallel for schedule(dynamic)
        for (int bh = 0; bh < B * H; ++bh) {
            const int b = bh / H, hh = bh % H, kh = hh / gq;
            const ora_seq* q = seqs[b];
            const int len = q->len + 1;
            const float* kc = q->k + (size_t)l * s->max_seq * KV * dh;
            const float* vc = q->v + (size_t)l * s->max_seq * KV * dh;
            const float* qv = Q + ((size_t)b * H + hh) * dh;
            float* sc = (float*)malloc(sizeof(float) * len);
            float mx = -INFINITY;
            for (int t = 0; t < len; ++t) {
                const float* kr = kc + ((size_t)t * KV + kh) * dh;
                float dot = 0.f;
                for (int i = 0; i < dh; ++i) dot += qv[i] * kr[i];
                sc[t] = dot * scale;
                if (sc[t] > mx) mx = sc[t];
            }
            float den = 0.f;
            for (int t = 0; t < len; ++t) {
                sc[t] = expf(sc[t] - mx);
                den += sc[t];
            }
            float* at = AT + ((size_t)b * H + hh) * dh;
            for (int i = 0; i < dh; ++i) at[i] = 0.f;
            for (int t = 0; t < len; ++t) {
                const float* vr = vc + ((size_t)t * KV + kh) * dh;
                for (int i = 0; i < dh; ++i) at[i] += sc[t] * vr[i];
            }
            for (int i = 0; i < dh; ++i) at[i] = m->round_act ? rbf_(at[i] / den) : at[i] / den;
            free(sc);
        }
        gemv_batch(L->wo, AT, O, d, H * dh, B);
        for (size_t i = 0; i < (size_t)B * d; ++i) Hs[i] += O[i];
        norm_batch(m, Hs, L->gm, A, rs, B);
        gemv_batch(L->wg, A, G, ff, d, B);
        gemv_batch(L->wu, A, U, ff, d, B);
        for (int b = 0; b < B; ++b)
            for (int i = 0; i < ff; ++i) {
                float gt = G[(size_t)b * ff + i] * rs[b], up = U[(size_t)b * ff + i] * rs[b];
                float act = gt / (1.0f + expf(-gt)) * up;
                A[(size_t)b * ff + i] = m->round_act ? rbf_(act) : act;
            }
        gemv_batch(L->wd, A, O, d, ff, B);
        for (size_t i = 0; i < (size_t)B * d; ++i) Hs[i] += O[i];
    }
    norm_batch(m, Hs, m->gf, A, rs, B);
    float* LG = (float*)malloc(sizeof(float) * (size_t)B * s->vocab);
    gemv_batch(m->lm, A, LG, s->vocab, d, B);
    for (int b = 0; b < B; ++b) {
        const float* lg = LG + (size_t)b * s->vocab;
        int best = 0;
        for (int v = 1; v < s->vocab; ++v)
            if (lg[v] * rs[b] > lg[best] * rs[b]) best = v;
        next[b] = best;
        seqs[b]->len += 1;
    }
    free(LG); free(Hs); free(A); free(Q); free(K); free(V); free(AT); free(O); free(G); free(U); free(rs);
    return 0;
}
