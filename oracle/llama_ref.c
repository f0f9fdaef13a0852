/* TEST INFRASTRUCTURE ONLY — CPU restatement (numeric oracle) of the token
 * step the B200 data plane executes. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it; the product never does.
 *
 * The reference LLM-Mesh artifact has no model arithmetic at all (SURVEY 0, 8c:
 * "logits/outputs: parity unpinned"): its step cost is a table lookup
 * (proj/src/perfmodel.cpp:55-100). This file therefore restates the standard
 * Llama decoder the paper's engines ran (vLLM/OpenVINO) and is
 * pinned instead against Hugging Face transformers' LlamaForCausalLM on golden
 * vectors (tests/golden/make_llama_golden.py, round_act = 0 mode).
 *
 * Numerics contract shared with the GPU path (round_act = 1):
 *   weights, embeddings, KV cache: bf16 (RNE); residual stream h: fp32;
 *   normed GEMV input  a = bf16(h * gamma), output scaled by rs = 1/sqrt(mean(h^2)+eps);
 *   q, k roped in fp32 (rotate-half, table cos/sin computed in double -> float),
 *   attention in fp32 over bf16 K/V, its output rounded to bf16 before W_o
 *   (the GPU decode kernel feeds q and the softmax weights to the tensor cores
 *   as bf16; that rounding is inside the parity tolerance, not restated here);
 *   silu(gate) * up rounded to bf16 before W_down; logits fp32; greedy argmax
 *   with ties to the lowest id.
 * The generator below must stay bit-identical to csrc/gpu/model.cuh.
 */
#include "llama_ref.h"

#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

enum { T_EMB = 0, T_WQ = 1, T_WK = 2, T_WV = 3, T_WO = 4, T_WGATE = 5, T_WUP = 6, T_WDOWN = 7, T_LM = 8,
       T_GATTN = 9, T_GMLP = 10, T_GFINAL = 11 };

static uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
static uint64_t tensor_key(uint64_t seed, uint32_t tensor, uint32_t layer) {
    return splitmix64(seed ^ ((uint64_t)tensor << 56) ^ ((uint64_t)layer << 40) ^ 0x5eedull);
}
static int32_t elem_i24(uint64_t key, uint64_t index) { return (int32_t)(splitmix64(key + index) >> 40) - (1 << 23); }
static float weight_value(uint64_t key, uint64_t index) { return (float)elem_i24(key, index) * (1.0f / 268435456.0f); }
static float gain_value(uint64_t key, uint64_t index) { return 1.0f + (float)elem_i24(key, index) * (1.0f / 134217728.0f); }

static float rbf(float f) { return bf2f(f2bf(f)); }

int ora_prompt_token(uint64_t seed, int64_t request, int pos, int vocab) {
    uint64_t h = splitmix64(splitmix64(seed ^ 0x70726f6d7074ull) + (uint64_t)request * 0x100000001b3ull + (uint64_t)pos);
    return (int)(h % (uint64_t)vocab);
}
float ora_weight(uint64_t seed, int tensor, int layer, uint64_t index) {
    uint64_t key = tensor_key(seed, (uint32_t)tensor, (uint32_t)layer);
    if (tensor >= T_GATTN) return gain_value(key, index);
    return rbf(weight_value(key, index));
}

static uint16_t* gen_matrix(uint64_t seed, int tensor, int layer, size_t n) {
    uint16_t* m = (uint16_t*)malloc(n * sizeof(uint16_t));
    uint64_t key = tensor_key(seed, (uint32_t)tensor, (uint32_t)layer);
#pragma omp parallel for schedule(static)
    for (long long i = 0; i < (long long)n; ++i) m[i] = f2bf(weight_value(key, (uint64_t)i));
    return m;
}
/* Bulk generator exports for the numpy restatement (oracle/llama_np.py). */
void ora_gen_bf16(uint64_t seed, int tensor, int layer, uint64_t n, uint16_t* out) {
    uint64_t key = tensor_key(seed, (uint32_t)tensor, (uint32_t)layer);
#pragma omp parallel for schedule(static)
    for (long long i = 0; i < (long long)n; ++i) out[i] = f2bf(weight_value(key, (uint64_t)i));
}
void ora_gen_gain(uint64_t seed, int tensor, int layer, int n, float* out) {
    uint64_t key = tensor_key(seed, (uint32_t)tensor, (uint32_t)layer);
    for (int i = 0; i < n; ++i) out[i] = gain_value(key, (uint64_t)i);
}
static float* gen_gain(uint64_t seed, int tensor, int layer, int n) {
    float* g = (float*)malloc((size_t)n * sizeof(float));
    uint64_t key = tensor_key(seed, (uint32_t)tensor, (uint32_t)layer);
    for (int i = 0; i < n; ++i) g[i] = gain_value(key, (uint64_t)i);
    return g;
}

ora_model* ora_create(const ora_shape* s, uint64_t seed, int round_act) {
    ora_model* m = (ora_model*)calloc(1, sizeof(ora_model));
    m->s = *s;
    m->seed = seed;
    m->round_act = round_act;
    size_t d = (size_t)s->d, qd = (size_t)s->n_heads * s->dh, kd = (size_t)s->n_kv * s->dh;
    m->emb = gen_matrix(seed, T_EMB, 0, (size_t)s->vocab * d);
    m->lm = s->tied ? m->emb : gen_matrix(seed, T_LM, 0, (size_t)s->vocab * d);
    m->gf = gen_gain(seed, T_GFINAL, 0, s->d);
    m->layers = (ora_layer*)calloc((size_t)s->n_layers, sizeof(ora_layer));
    for (int l = 0; l < s->n_layers; ++l) {
        ora_layer* L = &m->layers[l];
        L->wq = gen_matrix(seed, T_WQ, l, qd * d);
        L->wk = gen_matrix(seed, T_WK, l, kd * d);
        L->wv = gen_matrix(seed, T_WV, l, kd * d);
        L->wo = gen_matrix(seed, T_WO, l, d * qd);
        L->wg = gen_matrix(seed, T_WGATE, l, (size_t)s->ff * d);
        L->wu = gen_matrix(seed, T_WUP, l, (size_t)s->ff * d);
        L->wd = gen_matrix(seed, T_WDOWN, l, d * (size_t)s->ff);
        L->ga = gen_gain(seed, T_GATTN, l, s->d);
        L->gm = gen_gain(seed, T_GMLP, l, s->d);
    }
    int half = s->dh / 2;
    m->cosv = (float*)malloc((size_t)s->max_seq * half * sizeof(float));
    m->sinv = (float*)malloc((size_t)s->max_seq * half * sizeof(float));
    for (int p = 0; p < s->max_seq; ++p)
        for (int i = 0; i < half; ++i) {
            double inv = pow((double)s->rope_theta, -2.0 * i / (double)s->dh);
            double ang = (double)p * inv;
            m->cosv[(size_t)p * half + i] = (float)cos(ang);
            m->sinv[(size_t)p * half + i] = (float)sin(ang);
        }
    return m;
}

void ora_free(ora_model* m) {
    if (!m) return;
    for (int l = 0; l < m->s.n_layers; ++l) {
        ora_layer* L = &m->layers[l];
        free(L->wq); free(L->wk); free(L->wv); free(L->wo); free(L->wg); free(L->wu); free(L->wd);
        free(L->ga); free(L->gm);
    }
    free(m->layers);
    if (m->lm != m->emb) free(m->lm);
    free(m->emb);
    free(m->gf);
    free(m->cosv);
    free(m->sinv);
    free(m);
}

ora_seq* ora_seq_new(const ora_model* m) {
    ora_seq* q = (ora_seq*)calloc(1, sizeof(ora_seq));
    size_t n = (size_t)m->s.n_layers * m->s.max_seq * m->s.n_kv * m->s.dh;
    q->k = (float*)calloc(n, sizeof(float));
    q->v = (float*)calloc(n, sizeof(float));
    return q;
}
void ora_seq_free(ora_seq* q) {
    if (!q) return;
    free(q->k);
    free(q->v);
    free(q);
}
int ora_seq_len(const ora_seq* q) { return q->len; }

/* y[r] = sum_c W[r][c] * x[c] (W bf16 row-major [rows][cols]) accumulated in double */
static void gemv(const uint16_t* W, const float* x, float* y, int rows, int cols) {
#pragma omp parallel for schedule(static)
    for (int r = 0; r < rows; ++r) {
        const uint16_t* w = W + (size_t)r * cols;
        double acc = 0.0;
        for (int c = 0; c < cols; ++c) acc += (double)bf2f(w[c]) * (double)x[c];
        y[r] = (float)acc;
    }
}

/* Normed GEMV input: a = bf16(h * gamma) (or fp32 when round_act == 0), rs = 1/sqrt(mean h^2 + eps). */
static float norm_input(const ora_model* m, const float* h, const float* gamma, float* a) {
    int d = m->s.d;
    double ss = 0.0;
    for (int i = 0; i < d; ++i) ss += (double)h[i] * (double)h[i];
    float rs = (float)(1.0 / sqrt(ss / d + (double)m->s.eps));
    for (int i = 0; i < d; ++i) a[i] = m->round_act ? rbf(h[i] * gamma[i]) : h[i] * gamma[i];
    return rs;
}

/* Feeds `token` at position q->len; returns the greedy next token, optional logits[vocab]. */
int ora_feed(const ora_model* m, ora_seq* q, int token, float* logits_out) {
    const ora_shape* s = &m->s;
    const int d = s->d, H = s->n_heads, KV = s->n_kv, dh = s->dh, half = dh / 2, ff = s->ff, gq = H / KV;
    const int pos = q->len;
    if (pos >= s->max_seq) return -1;
    float* h = (float*)malloc(sizeof(float) * d);
    float* a = (float*)malloc(sizeof(float) * (d > ff ? d : ff));
    float* qv = (float*)malloc(sizeof(float) * H * dh);
    float* kv = (float*)malloc(sizeof(float) * KV * dh);
    float* vv = (float*)malloc(sizeof(float) * KV * dh);
    float* att = (float*)malloc(sizeof(float) * H * dh);
    float* o = (float*)malloc(sizeof(float) * d);
    float* g = (float*)malloc(sizeof(float) * ff);
    float* u = (float*)malloc(sizeof(float) * ff);
    float* sc = (float*)malloc(sizeof(float) * (pos + 1));
    for (int i = 0; i < d; ++i) h[i] = bf2f(m->emb[(size_t)token * d + i]);
    const float* cs = m->cosv + (size_t)pos * half;
    const float* sn = m->sinv + (size_t)pos * half;
    for (int l = 0; l < s->n_layers; ++l) {
        const ora_layer* L = &m->layers[l];
        float rs = norm_input(m, h, L->ga, a);
        gemv(L->wq, a, qv, H * dh, d);
        gemv(L->wk, a, kv, KV * dh, d);
        gemv(L->wv, a, vv, KV * dh, d);
        for (int i = 0; i < H * dh; ++i) qv[i] *= rs;
        for (int i = 0; i < KV * dh; ++i) {
            kv[i] *= rs;
            vv[i] *= rs;
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
            kc[(size_t)pos * KV * dh + i] = m->round_act ? rbf(kv[i]) : kv[i];
            vc[(size_t)pos * KV * dh + i] = m->round_act ? rbf(vv[i]) : vv[i];
        }
        const double scale = 1.0 / sqrt((double)dh);
        for (int hh = 0; hh < H; ++hh) {
            int kh = hh / gq;
            double mx = -INFINITY;
            for (int t = 0; t <= pos; ++t) {
                const float* kr = kc + ((size_t)t * KV + kh) * dh;
                double dot = 0.0;
                for (int i = 0; i < dh; ++i) dot += (double)qv[hh * dh + i] * (double)kr[i];
                sc[t] = (float)(dot * scale);
                if (sc[t] > mx) mx = sc[t];
            }
            double den = 0.0;
            for (int t = 0; t <= pos; ++t) den += exp((double)sc[t] - mx);
            for (int i = 0; i < dh; ++i) {
                double acc = 0.0;
                for (int t = 0; t <= pos; ++t)
                    acc += exp((double)sc[t] - mx) * (double)vc[((size_t)t * KV + kh) * dh + i];
                float r = (float)(acc / den);
                att[hh * dh + i] = m->round_act ? rbf(r) : r;
            }
        }
        gemv(L->wo, att, o, d, H * dh);
        for (int i = 0; i < d; ++i) h[i] += o[i];
        rs = norm_input(m, h, L->gm, a);
        gemv(L->wg, a, g, ff, d);
        gemv(L->wu, a, u, ff, d);
        for (int i = 0; i < ff; ++i) {
            float gt = g[i] * rs, up = u[i] * rs;
            float act = gt / (1.0f + expf(-gt)) * up;
            a[i] = m->round_act ? rbf(act) : act;
        }
        gemv(L->wd, a, o, d, ff);
        for (int i = 0; i < d; ++i) h[i] += o[i];
    }
    float rs = norm_input(m, h, m->gf, a);
    float* lg = (float*)malloc(sizeof(float) * s->vocab);
    gemv(m->lm, a, lg, s->vocab, d);
    int best = 0;
    for (int v = 0; v < s->vocab; ++v) {
        lg[v] *= rs;
        if (lg[v] > lg[best]) best = v;
    }
    if (logits_out) memcpy(logits_out, lg, sizeof(float) * s->vocab);
    free(lg); free(h); free(a); free(qv); free(kv); free(vv); free(att); free(o); free(g); free(u); free(sc);
    q->len = pos + 1;
    return best;
}

int ora_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
