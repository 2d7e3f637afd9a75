/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference GAS training hot path.
 * See gas_oracle.h for the contract. Compiled with -ffp-contract=off: the reference is
 * built without -march (x86-64 baseline, no FMA), so every a*b+c is two roundings
 * (SURVEY.md Appendix A.8). Citations are to /root/reference/proj/.
 */
#include "gas_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------ */
/* rng.hpp                                                                               */
/* ------------------------------------------------------------------------------------ */

uint64_t go_mix64(uint64_t x) { /* include/gas/rng.hpp:11-16 (splitmix64 finalizer) */
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

uint64_t go_derive_seed(uint64_t s, uint64_t a, uint64_t b, uint64_t c) { /* rng.hpp:18-21 */
    return go_mix64(go_mix64(go_mix64(s ^ go_mix64(a)) ^ go_mix64(b)) ^ go_mix64(c));
}

/* std::mt19937_64 (the engine behind gas::Rng, rng.hpp:23-65), written out. */
typedef struct {
    uint64_t mt[312];
    int mti;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i) g->mt[i] = 6364136223846793005ull * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->mti = 312;
}

static uint64_t mt64_next(mt64* g) {
    const uint64_t UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull, A = 0xB5026F5AA96619E9ull;
    if (g->mti >= 312) {
        int i;
        for (i = 0; i < 312 - 156; ++i) {
            uint64_t x = (g->mt[i] & UM) | (g->mt[i + 1] & LM);
            g->mt[i] = g->mt[i + 156] ^ (x >> 1) ^ ((x & 1ull) ? A : 0ull);
        }
        for (; i < 311; ++i) {
            uint64_t x = (g->mt[i] & UM) | (g->mt[i + 1] & LM);
            g->mt[i] = g->mt[i + (156 - 312)] ^ (x >> 1) ^ ((x & 1ull) ? A : 0ull);
        }
        uint64_t x = (g->mt[311] & UM) | (g->mt[0] & LM);
        g->mt[311] = g->mt[155] ^ (x >> 1) ^ ((x & 1ull) ? A : 0ull);
        g->mti = 0;
    }
    uint64_t x = g->mt[g->mti++];
    x ^= (x >> 29) & 0x5555555555555555ull;
    x ^= (x << 17) & 0x71D67FFFEDA60000ull;
    x ^= (x << 37) & 0xFFF7EEE000000000ull;
    x ^= (x >> 43);
    return x;
}

static double mt64_double(mt64* g) { return (double)(mt64_next(g) >> 11) * 0x1.0p-53; } /* rng.hpp:30-32 */

static uint64_t mt64_below(mt64* g, uint64_t n) { /* rng.hpp:35-43 */
    if (n <= 1) return 0;
    uint64_t limit = ~(uint64_t)0 - (~(uint64_t)0 % n);
    uint64_t x;
    do { x = mt64_next(g); } while (x >= limit);
    return x % n;
}

void go_glorot(int64_t rows, int64_t cols, uint64_t seed, float* out) { /* src/nn.cpp:65-70 */
    const double bound = sqrt(6.0 / (double)(rows + cols));
    mt64 g;
    mt64_seed(&g, seed);
    for (int64_t i = 0; i < rows * cols; ++i) out[i] = (float)((mt64_double(&g) * 2.0 - 1.0) * bound);
}

void go_epoch_order(int32_t nb, uint64_t model_seed, int64_t epoch, int32_t* out) {
    /* src/trainer.cpp:395-400: iota, then Rng(derive_seed(seed ^ "ordr", epoch)).shuffle */
    for (int32_t i = 0; i < nb; ++i) out[i] = i;
    mt64 g;
    mt64_seed(&g, go_derive_seed(model_seed ^ 0x6f726472ull, (uint64_t)epoch, 0, 0));
    for (int64_t i = nb; i > 1; --i) { /* rng.hpp:56-62 Fisher-Yates */
        int64_t j = (int64_t)mt64_below(&g, (uint64_t)i);
        int32_t t = out[i - 1];
        out[i - 1] = out[j];
        out[j] = t;
    }
}

void go_free(void* p) { free(p); }

/* ------------------------------------------------------------------------------------ */
/* graph.cpp                                                                             */
/* ------------------------------------------------------------------------------------ */

static int cmp_i32(const void* a, const void* b) {
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}

int go_build_graph(const int32_t* u, const int32_t* v, int64_t m, int32_t n, int symmetrize,
                   int64_t* row_offsets, int32_t** cols_out, int64_t* nnz_out) {
    /* src/graph.cpp:25-61: row v collects sources w of edges w->v (+ reverse when
     * symmetrizing, self-loops once), each row sorted and deduplicated. */
    if (n < 0) return 1;
    for (int64_t i = 0; i < m; ++i)
        if (u[i] < 0 || u[i] >= n || v[i] < 0 || v[i] >= n) return 1;
    int64_t* cnt = calloc((size_t)n + 1, sizeof(int64_t));
    for (int64_t i = 0; i < m; ++i) {
        cnt[v[i] + 1]++;
        if (symmetrize && u[i] != v[i]) cnt[u[i] + 1]++;
    }
    for (int32_t r = 0; r < n; ++r) cnt[r + 1] += cnt[r];
    int32_t* buf = malloc(sizeof(int32_t) * (size_t)(cnt[n] > 0 ? cnt[n] : 1));
    int64_t* pos = malloc(sizeof(int64_t) * ((size_t)n + 1));
    memcpy(pos, cnt, sizeof(int64_t) * ((size_t)n + 1));
    for (int64_t i = 0; i < m; ++i) {
        buf[pos[v[i]]++] = u[i];
        if (symmetrize && u[i] != v[i]) buf[pos[u[i]]++] = v[i];
    }
    /* rows sorted and deduplicated in place (in parallel), then compacted in row order */
#pragma omp parallel for schedule(dynamic, 256)
    for (int32_t r = 0; r < n; ++r) {
        int64_t b = cnt[r], e = cnt[r + 1], k = b;
        qsort(buf + b, (size_t)(e - b), sizeof(int32_t), cmp_i32);
        for (int64_t i = b; i < e; ++i)
            if (i == b || buf[i] != buf[i - 1]) buf[k++] = buf[i];
        pos[r] = k - b;
    }
    row_offsets[0] = 0;
    int64_t w = 0;
    for (int32_t r = 0; r < n; ++r) {
        if (w != cnt[r]) memmove(buf + w, buf + cnt[r], sizeof(int32_t) * (size_t)pos[r]);
        w += pos[r];
        row_offsets[r + 1] = w;
    }
    free(cnt);
    free(pos);
    *cols_out = buf;
    *nnz_out = w;
    return 0;
}

int go_plan_make(int32_t n, const int64_t* ro, const int32_t* cols, const int32_t* batch, int64_t nb,
                 go_plan* p) {
    /* src/graph.cpp:78-134 */
    memset(p, 0, sizeof(*p));
    if (nb <= 0) return 1;
    for (int64_t i = 0; i < nb; ++i) {
        if (batch[i] < 0 || batch[i] >= n) return 1;
        if (i > 0 && batch[i] <= batch[i - 1]) return 1;
    }
    uint8_t* in_batch = calloc((size_t)n, 1);
    uint8_t* in_ext = calloc((size_t)n, 1);
    int32_t* g2l = malloc(sizeof(int32_t) * (size_t)n);
    for (int64_t i = 0; i < nb; ++i) in_batch[batch[i]] = in_ext[batch[i]] = 1;
    for (int64_t i = 0; i < nb; ++i)
        for (int64_t e = ro[batch[i]]; e < ro[batch[i] + 1]; ++e) in_ext[cols[e]] = 1;
    int32_t next = 0;
    for (int32_t v = 0; v < n; ++v) next += in_ext[v];
    p->nb = (int32_t)nb;
    p->next = next;
    p->nhalo = next - (int32_t)nb;
    p->batch = malloc(sizeof(int32_t) * (size_t)nb);
    memcpy(p->batch, batch, sizeof(int32_t) * (size_t)nb);
    p->extended = malloc(sizeof(int32_t) * (size_t)next);
    p->is_halo = malloc((size_t)next);
    p->halo = malloc(sizeof(int32_t) * (size_t)(p->nhalo + 1));
    p->batch_local_rows = malloc(sizeof(int32_t) * (size_t)nb);
    p->halo_local_rows = malloc(sizeof(int32_t) * (size_t)(p->nhalo + 1));
    int32_t k = 0, kb = 0, kh = 0;
    for (int32_t v = 0; v < n; ++v) {
        if (!in_ext[v]) continue;
        p->extended[k] = v;
        p->is_halo[k] = !in_batch[v];
        g2l[v] = k;
        if (in_batch[v]) p->batch_local_rows[kb++] = k;
        else {
            p->halo[kh] = v;
            p->halo_local_rows[kh++] = k;
        }
        ++k;
    }
    /* Local CSR: in-edges of batch rows only (graph.cpp:114-133). */
    p->local_rowptr = calloc((size_t)next + 1, sizeof(int64_t));
    for (int32_t i = 0; i < next; ++i) {
        int64_t deg = p->is_halo[i] ? 0 : ro[p->extended[i] + 1] - ro[p->extended[i]];
        p->local_rowptr[i + 1] = p->local_rowptr[i] + deg;
    }
    p->local_cols = malloc(sizeof(int32_t) * (size_t)(p->local_rowptr[next] + 1));
    for (int32_t i = 0; i < next; ++i) {
        if (p->is_halo[i]) continue;
        int64_t pos = p->local_rowptr[i];
        for (int64_t e = ro[p->extended[i]]; e < ro[p->extended[i] + 1]; ++e) p->local_cols[pos++] = g2l[cols[e]];
    }
    /* build_plan_aggregation, src/layers.cpp:42-70. */
    int64_t tot = 0;
    for (int64_t i = 0; i < nb; ++i) tot += ro[batch[i] + 1] - ro[batch[i]];
    p->gcn_rowptr = malloc(sizeof(int64_t) * (size_t)(nb + 1));
    p->sum_rowptr = malloc(sizeof(int64_t) * (size_t)(nb + 1));
    p->gcn_cols = malloc(sizeof(int32_t) * (size_t)(tot + nb));
    p->gcn_coeffs = malloc(sizeof(float) * (size_t)(tot + nb));
    p->sum_cols = malloc(sizeof(int32_t) * (size_t)(tot + 1));
    p->sum_coeffs = malloc(sizeof(float) * (size_t)(tot + 1));
    int64_t eg = 0, es = 0;
    p->gcn_rowptr[0] = p->sum_rowptr[0] = 0;
    for (int64_t i = 0; i < nb; ++i) {
        const int32_t v = batch[i], lv = p->batch_local_rows[i];
        const double cv = sqrt((double)(ro[v + 1] - ro[v]) + 1.0);
        int self_seen = 0;
        for (int64_t e = ro[v]; e < ro[v + 1]; ++e) {
            const int32_t w = cols[e];
            const double cw = sqrt((double)(ro[w + 1] - ro[w]) + 1.0);
            p->gcn_cols[eg] = g2l[w];
            p->gcn_coeffs[eg++] = (float)(1.0 / (cw * cv));
            p->sum_cols[es] = g2l[w];
            p->sum_coeffs[es++] = 1.0f;
            if (w == v) self_seen = 1;
        }
        if (!self_seen) {
            p->gcn_cols[eg] = lv;
            p->gcn_coeffs[eg++] = (float)(1.0 / (cv * cv));
        }
        p->gcn_rowptr[i + 1] = eg;
        p->sum_rowptr[i + 1] = es;
    }
    free(in_batch);
    free(in_ext);
    free(g2l);
    return 0;
}

void go_plan_free(go_plan* p) {
    free(p->batch); free(p->extended); free(p->halo); free(p->is_halo);
    free(p->batch_local_rows); free(p->halo_local_rows); free(p->local_rowptr); free(p->local_cols);
    free(p->gcn_rowptr); free(p->gcn_cols); free(p->gcn_coeffs);
    free(p->sum_rowptr); free(p->sum_cols); free(p->sum_coeffs);
    memset(p, 0, sizeof(*p));
}

/* ------------------------------------------------------------------------------------ */
/* tensor.cpp ops                                                                        */
/* ------------------------------------------------------------------------------------ */

void go_aggregate_fwd(const int64_t* rp, int64_t m, const int32_t* cols, const float* coeffs,
                      const float* x, int64_t d, float* y) {
    /* src/tensor.cpp:514-530: sequential CSR order, double accumulator, cast to float. */
    double* acc = malloc(sizeof(double) * (size_t)(d > 0 ? d : 1));
    for (int64_t r = 0; r < m; ++r) {
        for (int64_t j = 0; j < d; ++j) acc[j] = 0.0;
        for (int64_t e = rp[r]; e < rp[r + 1]; ++e) {
            const double c = coeffs[e];
            const float* src = x + (int64_t)cols[e] * d;
            for (int64_t j = 0; j < d; ++j) acc[j] += c * (double)src[j];
        }
        for (int64_t j = 0; j < d; ++j) y[r * d + j] = (float)acc[j];
    }
    free(acc);
}

void go_aggregate_bwd(const int64_t* rp, int64_t m, const int32_t* cols, const float* coeffs,
                      const float* gy, int64_t d, float* gx) {
    /* src/tensor.cpp:531-549: r ascending, row order, float mul then float add. */
    for (int64_t r = 0; r < m; ++r)
        for (int64_t e = rp[r]; e < rp[r + 1]; ++e) {
            const float c = coeffs[e];
            float* g = gx + (int64_t)cols[e] * d;
            for (int64_t j = 0; j < d; ++j) g[j] += c * gy[r * d + j];
        }
}

void go_matmul_fwd(const float* a, int64_t m, int64_t k, const float* b, int64_t n, float* y) {
    /* src/tensor.cpp:148-167: double accumulation per row, zero entries of a skipped. */
    double* acc = malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    for (int64_t i = 0; i < m; ++i) {
        for (int64_t j = 0; j < n; ++j) acc[j] = 0.0;
        for (int64_t t = 0; t < k; ++t) {
            const double av = a[i * k + t];
            if (av == 0.0) continue;
            for (int64_t j = 0; j < n; ++j) acc[j] += av * (double)b[t * n + j];
        }
        for (int64_t j = 0; j < n; ++j) y[i * n + j] = (float)acc[j];
    }
    free(acc);
}

void go_matmul_bwd(const float* a, const float* b, const float* gy, int64_t m, int64_t k, int64_t n,
                   float* ga, float* gb) {
    /* src/tensor.cpp:169-204 */
    if (ga)
        for (int64_t i = 0; i < m; ++i)
            for (int64_t t = 0; t < k; ++t) {
                double acc = 0.0;
                for (int64_t j = 0; j < n; ++j) acc += (double)gy[i * n + j] * (double)b[t * n + j];
                ga[i * k + t] += (float)acc;
            }
    if (gb) {
        double* acc = calloc((size_t)(k * n > 0 ? k * n : 1), sizeof(double));
        for (int64_t i = 0; i < m; ++i)
            for (int64_t t = 0; t < k; ++t) {
                const double av = a[i * k + t];
                if (av == 0.0) continue;
                for (int64_t j = 0; j < n; ++j) acc[t * n + j] += av * (double)gy[i * n + j];
            }
        for (int64_t e = 0; e < k * n; ++e) gb[e] += (float)acc[e];
        free(acc);
    }
}

float go_softmax_ce(const float* logits, int64_t m, int64_t n, const int32_t* rows, const int32_t* labels,
                    int64_t r, float* gl) {
    /* src/tensor.cpp:597-647 */
    (void)m;
    double total = 0.0;
    for (int64_t i = 0; i < r; ++i) {
        const float* row = logits + (int64_t)rows[i] * n;
        float mx = row[0];
        for (int64_t j = 1; j < n; ++j) mx = row[j] > mx ? row[j] : mx;
        double denom = 0.0;
        for (int64_t j = 0; j < n; ++j) denom += exp((double)row[j] - mx);
        total += log(denom) - ((double)row[labels[i]] - mx);
    }
    const float loss = (float)(total / (double)r);
    if (gl) {
        const float gy = 1.0f, inv_m = 1.0f / (float)r;
        for (int64_t i = 0; i < r; ++i) {
            const float* row = logits + (int64_t)rows[i] * n;
            float* g = gl + (int64_t)rows[i] * n;
            float mx = row[0];
            for (int64_t j = 1; j < n; ++j) mx = row[j] > mx ? row[j] : mx;
            double denom = 0.0;
            for (int64_t j = 0; j < n; ++j) denom += exp((double)row[j] - mx);
            for (int64_t j = 0; j < n; ++j) {
                double p = exp((double)row[j] - mx) / denom;
                double delta = (j == labels[i]) ? 1.0 : 0.0;
                g[j] += gy * inv_m * (float)(p - delta);
            }
        }
    }
    return loss;
}

/* ------------------------------------------------------------------------------------ */
/* nn.cpp                                                                                */
/* ------------------------------------------------------------------------------------ */

void go_adam_step(float* p, float* m, float* v, const float* g, int64_t size, int64_t t, go_adam_cfg c) {
    /* src/nn.cpp:20-41 (t already incremented by the caller) */
    const double bc1 = 1.0 - pow((double)c.beta1, (double)t);
    const double bc2 = 1.0 - pow((double)c.beta2, (double)t);
    for (int64_t e = 0; e < size; ++e) {
        const double ge = g ? (double)g[e] : 0.0;
        const double mm = (double)c.beta1 * m[e] + (1.0 - (double)c.beta1) * ge;
        const double vv = (double)c.beta2 * v[e] + (1.0 - (double)c.beta2) * ge * ge;
        m[e] = (float)mm;
        v[e] = (float)vv;
        const double mhat = mm / bc1, vhat = vv / bc2;
        p[e] = (float)(p[e] - (double)c.lr * mhat / (sqrt(vhat) + (double)c.eps));
    }
}

double go_grad_clip(float* g, int64_t size, double max_norm) { /* src/nn.cpp:47-63 */
    double acc = 0.0;
    for (int64_t e = 0; e < size; ++e) acc += (double)g[e] * g[e];
    const double norm = sqrt(acc);
    if (norm > max_norm) {
        const float s = (float)(max_norm / norm);
        for (int64_t e = 0; e < size; ++e) g[e] *= s;
    }
    return norm;
}

/* ------------------------------------------------------------------------------------ */
/* trainer.cpp: GAS session                                                              */
/* ------------------------------------------------------------------------------------ */

typedef struct { float* v; int64_t rows, cols; } ptensor; /* one parameter (views into flat) */

struct go_session {
    go_spec spec;
    int32_t n, in_dim, num_classes, num_parts, hist_dim, L;
    int64_t* ro;
    int32_t* cols;
    float* x;
    int32_t* labels;
    uint8_t* train;
    go_plan* plans;
    /* parameters, flat, in Model::params() order (trainer.cpp:122-127) */
    int32_t np;
    ptensor prm[300];
    float* flat;
    int64_t nflat;
    float *adam_m, *adam_v;
    int64_t adam_t;
    /* named views */
    int32_t i_hw1, i_hb1, i_hw2, i_hb2, i_layer0, i_ow, i_ob;
    float** hist; /* L-1 tables n x hist_dim */
    int64_t store_step;
};

static int add_param(go_session* s, int64_t r, int64_t c) {
    s->prm[s->np].rows = r;
    s->prm[s->np].cols = c;
    s->nflat += r * c;
    return s->np++;
}

int go_session_create(int32_t n, const int64_t* ro, const int32_t* cols, const float* features, int32_t in_dim,
                      const int32_t* labels, const uint8_t* train_mask, int32_t num_classes,
                      const int32_t* assignment, int32_t num_parts, const go_spec* spec, go_session** out) {
    if (spec->dropout != 0.0f) return 1; /* dropout streams are not restated (SURVEY §7 hard part 7) */
    if (spec->kind != 0 && spec->kind != 2 && spec->kind != 3) return 1;
    if (spec->num_layers < 1 || spec->num_layers > 256) return 1;
    go_session* s = calloc(1, sizeof(go_session));
    s->spec = *spec;
    s->n = n;
    s->in_dim = in_dim;
    s->num_classes = num_classes;
    s->num_parts = num_parts;
    s->L = spec->num_layers;
    const int64_t nnz = ro[n];
    s->ro = malloc(sizeof(int64_t) * ((size_t)n + 1));
    memcpy(s->ro, ro, sizeof(int64_t) * ((size_t)n + 1));
    s->cols = malloc(sizeof(int32_t) * (size_t)(nnz + 1));
    memcpy(s->cols, cols, sizeof(int32_t) * (size_t)nnz);
    s->x = malloc(sizeof(float) * (size_t)n * (size_t)in_dim);
    memcpy(s->x, features, sizeof(float) * (size_t)n * (size_t)in_dim);
    s->labels = malloc(sizeof(int32_t) * (size_t)n);
    memcpy(s->labels, labels, sizeof(int32_t) * (size_t)n);
    s->train = malloc((size_t)n);
    memcpy(s->train, train_mask, (size_t)n);

    /* BatchSchedule::build (trainer.cpp:253-262): one plan per part, part order. */
    int32_t* cnt = calloc((size_t)num_parts, sizeof(int32_t));
    for (int32_t v = 0; v < n; ++v) {
        if (assignment[v] < 0 || assignment[v] >= num_parts) { free(cnt); go_session_free(s); return 1; }
        cnt[assignment[v]]++;
    }
    s->plans = calloc((size_t)num_parts, sizeof(go_plan));
    int32_t* nodes = malloc(sizeof(int32_t) * (size_t)n);
    for (int32_t p = 0; p < num_parts; ++p) {
        int32_t k = 0;
        for (int32_t v = 0; v < n; ++v)
            if (assignment[v] == p) nodes[k++] = v;
        if (go_plan_make(n, ro, cols, nodes, k, &s->plans[p]) != 0) {
            free(nodes); free(cnt); go_session_free(s); return 1;
        }
    }
    free(nodes);
    free(cnt);

    /* Model::build (trainer.cpp:55-129) */
    const int32_t L = s->L, H = spec->hidden, C = num_classes;
    s->i_hw1 = s->i_hb1 = s->i_hw2 = s->i_hb2 = s->i_ow = s->i_ob = -1;
    if (spec->kind == 2) { /* APPNP: head_w1, head_b1, head_w2, head_b2 */
        s->i_hw1 = add_param(s, in_dim, H);
        s->i_hb1 = add_param(s, 1, H);
        s->i_hw2 = add_param(s, H, C);
        s->i_hb2 = add_param(s, 1, C);
        s->i_layer0 = s->np;
        s->hist_dim = C;
    } else if (spec->kind == 3) { /* GCNII: head_w1, head_b1, W_1..W_L, out_w, out_b */
        s->i_hw1 = add_param(s, in_dim, H);
        s->i_hb1 = add_param(s, 1, H);
        s->i_layer0 = s->np;
        for (int32_t l = 1; l <= L; ++l) add_param(s, H, H);
        s->i_ow = add_param(s, H, C);
        s->i_ob = add_param(s, 1, C);
        s->hist_dim = H;
    } else { /* GCN: W_1..W_L */
        s->i_layer0 = s->np;
        for (int32_t l = 1; l <= L; ++l) add_param(s, l == 1 ? in_dim : H, l == L ? C : H);
        s->hist_dim = H;
    }
    if (L < 2) s->hist_dim = 0;
    s->flat = calloc((size_t)s->nflat + 1, sizeof(float));
    s->adam_m = calloc((size_t)s->nflat + 1, sizeof(float));
    s->adam_v = calloc((size_t)s->nflat + 1, sizeof(float));
    int64_t off = 0;
    for (int32_t i = 0; i < s->np; ++i) {
        s->prm[i].v = s->flat + off;
        off += s->prm[i].rows * s->prm[i].cols;
    }
    const uint64_t seed = spec->seed;
    if (spec->kind == 2 || spec->kind == 3) {
        go_glorot(in_dim, H, go_derive_seed(seed, 20, 1, 0), s->prm[s->i_hw1].v);
        if (spec->kind == 2) go_glorot(H, C, go_derive_seed(seed, 20, 2, 0), s->prm[s->i_hw2].v);
    }
    if (spec->kind == 0 || spec->kind == 3)
        for (int32_t l = 1; l <= L; ++l) { /* Layer::build(cfg, derive_seed(seed,10,l)); glorot(derive_seed(.,1)) */
            ptensor* w = &s->prm[s->i_layer0 + l - 1];
            go_glorot(w->rows, w->cols, go_derive_seed(go_derive_seed(seed, 10, (uint64_t)l, 0), 1, 0, 0), w->v);
        }
    if (spec->kind == 3) go_glorot(H, C, go_derive_seed(seed, 30, 1, 0), s->prm[s->i_ow].v);

    /* HistoryStore(L-1, n, d): zero tables (history.cpp:10-20) */
    s->hist = calloc((size_t)(L > 1 ? L - 1 : 1), sizeof(float*));
    for (int32_t l = 0; l < L - 1; ++l) s->hist[l] = calloc((size_t)n * (size_t)s->hist_dim + 1, sizeof(float));
    *out = s;
    return 0;
}

void go_session_free(go_session* s) {
    if (!s) return;
    if (s->plans)
        for (int32_t p = 0; p < s->num_parts; ++p) go_plan_free(&s->plans[p]);
    free(s->plans);
    if (s->hist)
        for (int32_t l = 0; l < s->L - 1; ++l) free(s->hist[l]);
    free(s->hist);
    free(s->ro); free(s->cols); free(s->x); free(s->labels); free(s->train);
    free(s->flat); free(s->adam_m); free(s->adam_v);
    free(s);
}

int64_t go_session_num_param_floats(const go_session* s) { return s->nflat; }
void go_session_get_params(const go_session* s, float* o) { memcpy(o, s->flat, sizeof(float) * (size_t)s->nflat); }
void go_session_set_params(go_session* s, const float* in) { memcpy(s->flat, in, sizeof(float) * (size_t)s->nflat); }
int32_t go_session_history_dim(const go_session* s) { return s->hist_dim; }
void go_session_get_history(const go_session* s, int32_t l, float* o) {
    memcpy(o, s->hist[l - 1], sizeof(float) * (size_t)s->n * (size_t)s->hist_dim);
}
void go_session_set_history(go_session* s, int32_t l, const float* in) { /* fill_layer, history.cpp:61-67 */
    memcpy(s->hist[l - 1], in, sizeof(float) * (size_t)s->n * (size_t)s->hist_dim);
}
int64_t go_session_store_step(const go_session* s) { return s->store_step; }

static float* zalloc(int64_t count) { return calloc((size_t)(count > 0 ? count : 1), sizeof(float)); }

/* out[i, :] += bias (add_rowvec fwd, tensor.cpp:277-307) */
static void rowvec_fwd(float* y, const float* x, const float* b, int64_t m, int64_t n) {
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) y[i * n + j] = x[i * n + j] + b[j];
}
/* add_rowvec bwd for the bias: gb[j] += float(sum_i double(gy[i,j])) */
static void rowvec_bwd_bias(const float* gy, int64_t m, int64_t n, float* gb) {
    for (int64_t j = 0; j < n; ++j) {
        double acc = 0.0;
        for (int64_t i = 0; i < m; ++i) acc += gy[i * n + j];
        gb[j] += (float)acc;
    }
}
static void relu_fwd(float* y, const float* x, int64_t sz) {
    for (int64_t i = 0; i < sz; ++i) y[i] = x[i] > 0.0f ? x[i] : 0.0f;
}
/* relu bwd (tensor.cpp:363-369): g[i] += gy[i] where x[i] > 0 */
static void relu_bwd(const float* x, const float* gy, float* g, int64_t sz) {
    for (int64_t i = 0; i < sz; ++i)
        if (x[i] > 0.0f) g[i] += gy[i];
}

/* Model::forward (trainer.cpp:174-251) + run_batch (:295-339) + advance_step (:426). */
/* run_batch (trainer.cpp:295-339) up to, not including, the optimizer: forward (pushes into
 * the tables when `push`), loss, backward. gflat (nflat floats, zeroed) receives the
 * pre-clip gradients when *stepped. */
static int batch_core(go_session* s, int32_t part, int train, int push, float* acts_out, float* logits_out,
                      double* loss_out, float* gflat, int* stepped) {
    if (part < 0 || part >= s->num_parts) return 1;
    const go_plan* P = &s->plans[part];
    const int32_t L = s->L, nb = P->nb, ne = P->next, F = s->in_dim, H = s->spec.hidden, C = s->num_classes;
    const int32_t kind = s->spec.kind, hd = s->hist_dim;
    const float alpha = s->spec.alpha, beta = s->spec.beta;

    /* x_ext = gather_features(X, V_b) (trainer.cpp:20-27, :190) */
    float* xe = zalloc((int64_t)ne * F);
    for (int32_t i = 0; i < ne; ++i) memcpy(xe + (int64_t)i * F, s->x + (int64_t)P->extended[i] * F, sizeof(float) * F);

    /* head (APPNP/GCNII, trainer.cpp:142-163), over all V_b rows */
    float *hz1 = NULL, *hr1 = NULL, *hz2 = NULL, *h0 = NULL;
    int32_t d0 = F;
    if (kind == 2 || kind == 3) {
        hz1 = zalloc((int64_t)ne * H);
        float* mm1 = zalloc((int64_t)ne * H);
        go_matmul_fwd(xe, ne, F, s->prm[s->i_hw1].v, H, mm1);
        rowvec_fwd(hz1, mm1, s->prm[s->i_hb1].v, ne, H);
        free(mm1);
        hr1 = zalloc((int64_t)ne * H);
        relu_fwd(hr1, hz1, (int64_t)ne * H);
        if (kind == 2) {
            float* mm2 = zalloc((int64_t)ne * C);
            go_matmul_fwd(hr1, ne, H, s->prm[s->i_hw2].v, C, mm2);
            hz2 = zalloc((int64_t)ne * C);
            rowvec_fwd(hz2, mm2, s->prm[s->i_hb2].v, ne, C);
            free(mm2);
            h0 = hz2;
            d0 = C;
        } else {
            h0 = hr1;
            d0 = H;
        }
    }

    /* per-layer saved state */
    float** hin = calloc((size_t)L + 1, sizeof(float*));   /* layer input, V_b x din */
    float** agg = calloc((size_t)L + 1, sizeof(float*));   /* aggregate output, nb x din */
    float** mix = calloc((size_t)L + 1, sizeof(float*));   /* GCNII mixed, nb x H */
    float** wt = calloc((size_t)L + 1, sizeof(float*));    /* GCNII w_tilde */
    float** outp = calloc((size_t)L + 1, sizeof(float*));  /* layer output, nb x dout */
    float** act = calloc((size_t)L + 1, sizeof(float*));   /* post-activation (nb x dout) */
    int32_t* din = calloc((size_t)L + 1, sizeof(int32_t));
    int32_t* dout = calloc((size_t)L + 1, sizeof(int32_t));
    float* fin_relu = NULL; /* GCNII final relu */
    float* logits = NULL;

    float* h = (kind == 0) ? xe : h0;
    int32_t dh = (kind == 0) ? F : d0;
    for (int32_t l = 1; l <= L; ++l) {
        hin[l] = h;
        din[l] = dh;
        agg[l] = zalloc((int64_t)nb * dh);
        go_aggregate_fwd(P->gcn_rowptr, nb, P->gcn_cols, P->gcn_coeffs, h, dh, agg[l]);
        if (kind == 0) { /* gcn_forward, layers.cpp:137-140 */
            const ptensor* W = &s->prm[s->i_layer0 + l - 1];
            dout[l] = (int32_t)W->cols;
            outp[l] = zalloc((int64_t)nb * dout[l]);
            go_matmul_fwd(agg[l], nb, dh, W->v, W->cols, outp[l]);
        } else { /* appnp (layers.cpp:152-158) / gcnii (:160-168): alpha*h0[B] + (1-alpha)*agg */
            const int32_t d = dh;
            float* m = zalloc((int64_t)nb * d);
            for (int32_t i = 0; i < nb; ++i)
                for (int32_t j = 0; j < d; ++j) {
                    const float a = h0[(int64_t)P->batch_local_rows[i] * d + j] * alpha;
                    const float b = agg[l][(int64_t)i * d + j] * (1.0f - alpha);
                    m[(int64_t)i * d + j] = a + b;
                }
            if (kind == 2) {
                dout[l] = d;
                outp[l] = m;
            } else {
                mix[l] = m;
                const ptensor* W = &s->prm[s->i_layer0 + l - 1];
                wt[l] = zalloc((int64_t)H * H);
                for (int64_t e = 0; e < (int64_t)H * H; ++e) {
                    const float id = ((e / H) == (e % H)) ? 1.0f : 0.0f;
                    wt[l][e] = id * (1.0f - beta) + W->v[e] * beta;
                }
                dout[l] = H;
                outp[l] = zalloc((int64_t)nb * H);
                go_matmul_fwd(m, nb, H, wt[l], H, outp[l]);
            }
        }
        if (l == L) {
            if (kind == 3) { /* trainer.cpp:221-227: relu, out_w, out_b */
                fin_relu = zalloc((int64_t)nb * H);
                relu_fwd(fin_relu, outp[l], (int64_t)nb * H);
                float* mm = zalloc((int64_t)nb * C);
                go_matmul_fwd(fin_relu, nb, H, s->prm[s->i_ow].v, C, mm);
                logits = zalloc((int64_t)nb * C);
                rowvec_fwd(logits, mm, s->prm[s->i_ob].v, nb, C);
                free(mm);
            } else {
                logits = outp[l];
            }
            break;
        }
        /* act = relu(out) for GCN/GCNII, identity for APPNP (trainer.cpp:232, :36-38) */
        if (kind == 2) act[l] = outp[l];
        else {
            act[l] = zalloc((int64_t)nb * dout[l]);
            relu_fwd(act[l], outp[l], (int64_t)nb * dout[l]);
        }
        /* push (history.cpp:28-42), pull (:44-55), compose_rows (tensor.cpp:459-512) */
        float* tab = s->hist[l - 1];
        if (push)
            for (int32_t i = 0; i < nb; ++i)
                memcpy(tab + (int64_t)P->batch[i] * hd, act[l] + (int64_t)i * hd, sizeof(float) * hd);
        float* comp = zalloc((int64_t)ne * hd);
        for (int32_t i = 0; i < nb; ++i)
            memcpy(comp + (int64_t)P->batch_local_rows[i] * hd, act[l] + (int64_t)i * hd, sizeof(float) * hd);
        for (int32_t i = 0; i < P->nhalo; ++i)
            memcpy(comp + (int64_t)P->halo_local_rows[i] * hd, tab + (int64_t)P->halo[i] * hd, sizeof(float) * hd);
        h = comp;
        dh = hd;
        if (acts_out) memcpy(acts_out + (int64_t)(l - 1) * nb * hd, act[l], sizeof(float) * (size_t)nb * hd);
    }
    if (logits_out) memcpy(logits_out, logits, sizeof(float) * (size_t)nb * C);

    /* run_batch: training rows of B_b (trainer.cpp:273-287, :313-317) */
    int32_t* rows = malloc(sizeof(int32_t) * (size_t)nb);
    int32_t* lab = malloc(sizeof(int32_t) * (size_t)nb);
    int32_t r = 0;
    for (int32_t i = 0; i < nb; ++i)
        if (s->train[P->batch[i]]) {
            rows[r] = i;
            lab[r++] = s->labels[P->batch[i]];
        }
    *stepped = 0;
    *loss_out = 0.0;
    if (r > 0) {
        float loss = go_softmax_ce(logits, nb, C, rows, lab, r, NULL);
        if (train && s->spec.l2_weight > 0.0f) { /* l2_penalty (tensor.cpp:649-678), recorded after CE */
            double acc = 0.0;
            for (int64_t e = 0; e < s->nflat; ++e) acc += (double)s->flat[e] * s->flat[e];
            loss = loss + (float)(s->spec.l2_weight * acc);
            /* its closure runs before CE's: g = 0 + 1*2*w*v */
            for (int64_t e = 0; e < s->nflat; ++e) gflat[e] += 1.0f * 2.0f * s->spec.l2_weight * s->flat[e];
        }
        *loss_out = loss;
        if (train) {
            float* gl = zalloc((int64_t)nb * C);
            go_softmax_ce(logits, nb, C, rows, lab, r, gl);
            float* g_out = NULL;
            if (kind == 3) { /* GCNII output head bwd */
                go_matmul_bwd(fin_relu, s->prm[s->i_ow].v, gl, nb, H, C, NULL, gflat + (s->prm[s->i_ow].v - s->flat));
                rowvec_bwd_bias(gl, nb, C, gflat + (s->prm[s->i_ob].v - s->flat));
                float* gr = zalloc((int64_t)nb * H);
                go_matmul_bwd(fin_relu, s->prm[s->i_ow].v, gl, nb, H, C, gr, NULL);
                g_out = zalloc((int64_t)nb * H);
                relu_bwd(outp[L], gr, g_out, (int64_t)nb * H);
                free(gr);
                free(gl);
            } else {
                g_out = gl;
            }
            float* g_h0 = (kind == 2 || kind == 3) ? zalloc((int64_t)ne * d0) : NULL;
            for (int32_t l = L; l >= 1; --l) {
                const int32_t di = din[l], dd = dout[l];
                float* g_agg = zalloc((int64_t)nb * di);
                if (kind == 0) {
                    const ptensor* W = &s->prm[s->i_layer0 + l - 1];
                    go_matmul_bwd(agg[l], W->v, g_out, nb, di, dd, g_agg, gflat + (W->v - s->flat));
                } else {
                    float* g_mix = g_out; /* APPNP: out is the mix */
                    if (kind == 3) {
                        const ptensor* W = &s->prm[s->i_layer0 + l - 1];
                        g_mix = zalloc((int64_t)nb * H);
                        float* g_wt = zalloc((int64_t)H * H);
                        go_matmul_bwd(mix[l], wt[l], g_out, nb, H, H, g_mix, g_wt);
                        float* gW = gflat + (W->v - s->flat);
                        for (int64_t e = 0; e < (int64_t)H * H; ++e) gW[e] += beta * g_wt[e];
                        free(g_wt);
                    }
                    /* add -> scale(h0b, a) -> select_rows ; scale(prop, 1-a) */
                    for (int32_t i = 0; i < nb; ++i)
                        for (int32_t j = 0; j < di; ++j) {
                            const float g = g_mix[(int64_t)i * di + j];
                            g_h0[(int64_t)P->batch_local_rows[i] * di + j] += alpha * g;
                            g_agg[(int64_t)i * di + j] += (1.0f - alpha) * g;
                        }
                    if (kind == 3) free(g_mix);
                }
                if (l == 1) {
                    if (kind != 0) /* h_in = h0: halo rows get gradient too (Appendix A.7) */
                        go_aggregate_bwd(P->gcn_rowptr, nb, P->gcn_cols, P->gcn_coeffs, g_agg, di, g_h0);
                    free(g_agg);
                    break;
                }
                float* g_h = zalloc((int64_t)ne * di);
                go_aggregate_bwd(P->gcn_rowptr, nb, P->gcn_cols, P->gcn_coeffs, g_agg, di, g_h);
                free(g_agg);
                /* compose bwd -> act_{l-1}; relu bwd -> out_{l-1} */
                float* g_prev = zalloc((int64_t)nb * di);
                if (kind == 2) {
                    for (int32_t i = 0; i < nb; ++i)
                        for (int32_t j = 0; j < di; ++j)
                            g_prev[(int64_t)i * di + j] += g_h[(int64_t)P->batch_local_rows[i] * di + j];
                } else {
                    float* g_act = zalloc((int64_t)nb * di);
                    for (int32_t i = 0; i < nb; ++i)
                        for (int32_t j = 0; j < di; ++j)
                            g_act[(int64_t)i * di + j] += g_h[(int64_t)P->batch_local_rows[i] * di + j];
                    relu_bwd(outp[l - 1], g_act, g_prev, (int64_t)nb * di);
                    free(g_act);
                }
                free(g_h);
                free(g_out);
                g_out = g_prev;
            }
            free(g_out);
            if (kind == 2 || kind == 3) { /* head bwd over all V_b rows */
                float* g_z1;
                if (kind == 2) {
                    rowvec_bwd_bias(g_h0, ne, C, gflat + (s->prm[s->i_hb2].v - s->flat));
                    float* g_r1 = zalloc((int64_t)ne * H);
                    go_matmul_bwd(hr1, s->prm[s->i_hw2].v, g_h0, ne, H, C, g_r1, gflat + (s->prm[s->i_hw2].v - s->flat));
                    g_z1 = zalloc((int64_t)ne * H);
                    relu_bwd(hz1, g_r1, g_z1, (int64_t)ne * H);
                    free(g_r1);
                } else {
                    g_z1 = zalloc((int64_t)ne * H);
                    relu_bwd(hz1, g_h0, g_z1, (int64_t)ne * H);
                }
                rowvec_bwd_bias(g_z1, ne, H, gflat + (s->prm[s->i_hb1].v - s->flat));
                go_matmul_bwd(xe, s->prm[s->i_hw1].v, g_z1, ne, F, H, NULL, gflat + (s->prm[s->i_hw1].v - s->flat));
                free(g_z1);
                free(g_h0);
            }
            *stepped = 1;
        }
    }
    free(rows);
    free(lab);

    /* cleanup */
    for (int32_t l = 1; l <= L; ++l) {
        free(agg[l]);
        if (kind == 3) { free(mix[l]); free(wt[l]); }
        if (act[l] && act[l] != outp[l]) free(act[l]);
        free(outp[l]);
        if (l >= 2) free(hin[l]);
    }
    if (kind == 3) { free(fin_relu); free(logits); }
    free(hin); free(agg); free(mix); free(wt); free(outp); free(act); free(din); free(dout);
    free(xe); free(hz1); free(hr1); free(hz2);
    return 0;
}

/* grad_clip + AdamState::step (trainer.cpp:328-333, nn.cpp:20-63) */
static void optimizer_step(go_session* s, float* g) {
    if (s->spec.clip_max_norm > 0.0f) go_grad_clip(g, s->nflat, s->spec.clip_max_norm);
    s->adam_t++;
    go_adam_cfg cfg = {s->spec.lr, s->spec.beta1, s->spec.beta2, s->spec.eps};
    go_adam_step(s->flat, s->adam_m, s->adam_v, g, s->nflat, s->adam_t, cfg);
}

int go_session_batch(go_session* s, int32_t part, int64_t epoch, int train, int push, float* acts_out,
                     float* logits_out, double* loss_out, float* grads_out, int* stepped) {
    (void)epoch; /* only seeds dropout, which is not restated (must be 0) */
    float* g = zalloc(s->nflat);
    const int rc = batch_core(s, part, train, push, acts_out, logits_out, loss_out, g, stepped);
    if (!rc && *stepped) {
        if (grads_out) memcpy(grads_out, g, sizeof(float) * (size_t)s->nflat);
        optimizer_step(s, g);
    }
    free(g);
    if (!rc) s->store_step++; /* advance_step once per batch (trainer.cpp:426) */
    return rc;
}

/* ---- data-parallel GAS step — no reference counterpart; at k = 1 it IS
 * gas_epoch. A step takes k consecutive batches of the seeded epoch order (rank j gets the
 * j-th). Every batch sees the start-of-step parameters and histories (its own rows are
 * fresh through compose_rows; its pushes are staged and committed after the step, Jacobi
 * semantics); gradients are summed in rank order, divided by the number of batches that
 * had training rows, then clipped and applied once. ---- */
int go_session_dp_batch(go_session* s, int32_t part, float* grads_out, float* acts_out, double* loss, int* stepped) {
    memset(grads_out, 0, sizeof(float) * (size_t)s->nflat);
    return batch_core(s, part, 1, 0, acts_out, NULL, loss, grads_out, stepped);
}

void go_session_dp_commit(go_session* s, int32_t part, const float* acts) {
    const go_plan* P = &s->plans[part];
    const int32_t hd = s->hist_dim;
    for (int32_t l = 1; l < s->L; ++l)
        for (int32_t i = 0; i < P->nb; ++i)
            memcpy(s->hist[l - 1] + (int64_t)P->batch[i] * hd, acts + ((int64_t)(l - 1) * P->nb + i) * hd,
                   sizeof(float) * (size_t)hd);
}

void go_session_dp_apply(go_session* s, const float* grad_sum, int32_t count, int32_t batches) {
    if (count > 0) {
        float* g = zalloc(s->nflat);
        for (int64_t e = 0; e < s->nflat; ++e) g[e] = grad_sum[e] / (float)count;
        optimizer_step(s, g);
        free(g);
    }
    s->store_step += batches;
}

int go_session_dp_epoch(go_session* s, int64_t epoch, int shuffle, int32_t k, double* loss) {
    if (k < 1) return 1;
    int32_t* order = malloc(sizeof(int32_t) * (size_t)s->num_parts);
    if (shuffle) go_epoch_order(s->num_parts, s->spec.seed, epoch, order);
    else for (int32_t i = 0; i < s->num_parts; ++i) order[i] = i;
    float* gsum = zalloc(s->nflat);
    float* g = zalloc(s->nflat);
    float** acts = calloc((size_t)k, sizeof(float*));
    double sum = 0.0;
    int64_t cnt = 0;
    int rc = 0;
    for (int32_t s0 = 0; s0 < s->num_parts && !rc; s0 += k) {
        const int32_t kk = s->num_parts - s0 < k ? s->num_parts - s0 : k;
        memset(gsum, 0, sizeof(float) * (size_t)s->nflat);
        int32_t count = 0;
        for (int32_t j = 0; j < kk && !rc; ++j) {
            const go_plan* P = &s->plans[order[s0 + j]];
            acts[j] = zalloc((int64_t)(s->L > 1 ? s->L - 1 : 0) * P->nb * s->hist_dim);
            double l = 0.0;
            int stepped = 0;
            rc = go_session_dp_batch(s, order[s0 + j], g, acts[j], &l, &stepped);
            if (stepped) {
                for (int64_t e = 0; e < s->nflat; ++e) gsum[e] += g[e];
                ++count;
                sum += l;
                ++cnt;
            }
        }
        for (int32_t j = 0; j < kk; ++j) {
            if (!rc) go_session_dp_commit(s, order[s0 + j], acts[j]);
            free(acts[j]);
            acts[j] = NULL;
        }
        if (!rc) go_session_dp_apply(s, gsum, count, kk);
    }
    free(acts);
    free(gsum);
    free(g);
    free(order);
    *loss = cnt > 0 ? sum / (double)cnt : 0.0;
    return rc;
}

int go_session_epoch(go_session* s, int64_t epoch, int shuffle, double* loss) { /* trainer.cpp:386-442 */
    int32_t* order = malloc(sizeof(int32_t) * (size_t)s->num_parts);
    if (shuffle) go_epoch_order(s->num_parts, s->spec.seed, epoch, order);
    else for (int32_t i = 0; i < s->num_parts; ++i) order[i] = i;
    double sum = 0.0;
    int64_t cnt = 0;
    for (int32_t oi = 0; oi < s->num_parts; ++oi) {
        double l = 0.0;
        int stepped = 0;
        int rc = go_session_batch(s, order[oi], epoch, 1, 1, NULL, NULL, &l, NULL, &stepped);
        if (rc) { free(order); return rc; }
        if (stepped) { sum += l; ++cnt; }
    }
    free(order);
    *loss = cnt > 0 ? sum / (double)cnt : 0.0;
    return 0;
}

/* ------------------------------------------------------------------------------------ */
/* Synthetic workload generator (not a reference algorithm: the bench's input generator, */
/* restated here so bench.py's reference arm builds the same graph and features without */
/* loading the product library; tests/test_workloads.py checks it equals                */
/* gasb_synth_pairs / gasb_synth_features bit for bit).                                  */
/* ------------------------------------------------------------------------------------ */

static double syn_u01(uint64_t seed, uint64_t a, uint64_t b) {
    return (double)(go_mix64(go_mix64(seed ^ go_mix64(a)) ^ go_mix64(b)) >> 11) * 0x1.0p-53;
}

static int32_t syn_sample(const double* cum, int64_t lo, int64_t hi, double target) {
    int64_t a = lo, b = hi - 1;
    while (a < b) {
        int64_t mid = (a + b) >> 1;
        if (cum[mid + 1] > target) b = mid;
        else a = mid + 1;
    }
    return (int32_t)a;
}

typedef struct { uint64_t key; int32_t v; } syn_key;
static int cmp_key(const void* a, const void* b) {
    const syn_key *x = (const syn_key*)a, *y = (const syn_key*)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return (x->v > y->v) - (x->v < y->v);
}

int go_synth_pairs(int32_t n, int32_t K, int64_t m, double intra, double gamma, double wmin, double wmax,
                   uint64_t seed, int32_t* src, int32_t* dst, int32_t* community) {
    if (n <= 0 || K <= 0 || K > n || !(gamma > 1.0) || !(wmin > 0.0) || wmax < wmin) return 1;
    double* w = malloc(sizeof(double) * (size_t)n);
    syn_key* key = malloc(sizeof(syn_key) * (size_t)n);
    int32_t* comm = malloc(sizeof(int32_t) * (size_t)n);
    double* cum = calloc((size_t)n + 1, sizeof(double));
    int64_t* cstart = calloc((size_t)K + 1, sizeof(int64_t));
    int64_t* fill = malloc(sizeof(int64_t) * (size_t)K);
    int32_t* members = malloc(sizeof(int32_t) * (size_t)n);
    double* ccum = calloc((size_t)n + (size_t)K, sizeof(double));
#pragma omp parallel for schedule(static)
    for (int32_t v = 0; v < n; ++v) {
        const double u = syn_u01(seed, 0x77656967ull, (uint64_t)v);
        const double x = wmin * pow(1.0 - u, -1.0 / (gamma - 1.0));
        w[v] = x < wmax ? x : wmax;
    }
    for (int32_t v = 0; v < n; ++v) {
        key[v].key = go_mix64(seed ^ go_mix64(0x636f6d6dull ^ go_mix64((uint64_t)v)));
        key[v].v = v;
    }
    qsort(key, (size_t)n, sizeof(syn_key), cmp_key);
    for (int32_t r = 0; r < n; ++r) comm[key[r].v] = r % K;
    for (int32_t v = 0; v < n; ++v) cum[v + 1] = cum[v] + w[v];
    for (int32_t v = 0; v < n; ++v) cstart[comm[v] + 1]++;
    for (int32_t c = 0; c < K; ++c) cstart[c + 1] += cstart[c];
    for (int32_t c = 0; c < K; ++c) fill[c] = cstart[c];
    for (int32_t v = 0; v < n; ++v) members[fill[comm[v]]++] = v;
    for (int32_t c = 0; c < K; ++c) {
        double* cc = ccum + cstart[c] + c;
        cc[0] = 0.0;
        for (int64_t i = cstart[c]; i < cstart[c + 1]; ++i) cc[i - cstart[c] + 1] = cc[i - cstart[c]] + w[members[i]];
    }
    const double W = cum[n];
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i) {
        const uint64_t ui = (uint64_t)i;
        const int32_t u = syn_sample(cum, 0, n, syn_u01(seed, ui, 1) * W);
        int32_t v;
        if (syn_u01(seed, ui, 2) < intra) {
            const int32_t c = comm[u];
            const double* cc = ccum + cstart[c] + c;
            const int64_t sz = cstart[c + 1] - cstart[c];
            v = members[cstart[c] + syn_sample(cc, 0, sz, syn_u01(seed, ui, 3) * cc[sz])];
        } else {
            v = syn_sample(cum, 0, n, syn_u01(seed, ui, 3) * W);
        }
        src[i] = u;
        dst[i] = v;
    }
    if (community) memcpy(community, comm, sizeof(int32_t) * (size_t)n);
    free(w); free(key); free(comm); free(cum); free(cstart); free(fill); free(members); free(ccum);
    return 0;
}

void go_synth_features(int64_t n, int32_t dim, int64_t ld, uint64_t seed, float* out) {
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < n; ++v) {
        float* row = out + v * ld;
        for (int32_t j = 0; j < dim; ++j) {
            const uint64_t c = (uint64_t)v * (uint64_t)dim + (uint64_t)j;
            double u1 = syn_u01(seed, c, 0x6e31ull);
            if (u1 <= 0.0) u1 = 0x1.0p-53;
            const double u2 = syn_u01(seed, c, 0x6e32ull);
            row[j] = (float)(sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2));
        }
        for (int64_t j = dim; j < ld; ++j) row[j] = 0.0f;
    }
}
