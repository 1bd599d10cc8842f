/* TEST INFRASTRUCTURE ONLY — see stagger_oracle.h.
 *
 * Plain-C, fp64 restatement of the reference hot path.  Each function cites
 * the reference file:line it follows (paths relative to
 * /root/reference/proj/core).  Arithmetic is written in the reference's
 * operation order and compiled with -ffp-contract=off so results are
 * bit-identical to the reference build (checked in tests/test_oracle.py).
 */
#include "stagger_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[512];

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

const char* orc_last_error(void) { return g_err; }

/* ---- RNG -------------------------------------------------------------- */

/* std::mt19937_64 (fixed by the C++ standard; rng.hpp:19-24 uses it). */
#define MT_N 312
#define MT_M 156
#define MT_A 0xB5026F5AA96619E9ULL
#define MT_UM 0xFFFFFFFF80000000ULL
#define MT_LM 0x7FFFFFFFULL

void orc_rng_init(orc_rng* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->mti = MT_N;
    r->spare = 0.0;
    r->has_spare = 0;
}

static void mt_twist(orc_rng* r) {
    for (int i = 0; i < MT_N; ++i) {
        const uint64_t x = (r->mt[i] & MT_UM) | (r->mt[(i + 1) % MT_N] & MT_LM);
        uint64_t xa = x >> 1;
        if (x & 1ULL) xa ^= MT_A;
        r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
    }
    r->mti = 0;
}

uint64_t orc_rng_next_u64(orc_rng* r) {
    if (r->mti >= MT_N) mt_twist(r);
    uint64_t x = r->mt[r->mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}

/* rng.hpp:26-28 */
double orc_rng_uniform(orc_rng* r) { return (double)(orc_rng_next_u64(r) >> 11) * 0x1.0p-53; }

/* rng.hpp:31-43: Box-Muller, cos first, sin cached */
double orc_rng_gaussian(orc_rng* r) {
    if (r->has_spare) {
        r->has_spare = 0;
        return r->spare;
    }
    const double u1 = orc_rng_uniform(r);
    const double u2 = orc_rng_uniform(r);
    const double rad = sqrt(-2.0 * log1p(-u1));
    const double a = 2.0 * 3.14159265358979323846 * u2;
    r->spare = rad * sin(a);
    r->has_spare = 1;
    return rad * cos(a);
}

/* rng.cpp:14-20 */
uint64_t orc_derive_seed(uint64_t seed, uint64_t tag) {
    uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (tag + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

void orc_rng_uniforms(uint64_t seed, int n, double* out) {
    orc_rng r;
    orc_rng_init(&r, seed);
    for (int i = 0; i < n; ++i) out[i] = orc_rng_uniform(&r);
}

void orc_rng_u64(uint64_t seed, int n, uint64_t* out) {
    orc_rng r;
    orc_rng_init(&r, seed);
    for (int i = 0; i < n; ++i) out[i] = orc_rng_next_u64(&r);
}

/* rng.cpp:7-12 */
static int sample_into(orc_rng* r, int d, double* out) {
    if (d <= 0) return fail(1, "sample_gaussian: d must be >= 1");
    for (int i = 0; i < d; ++i) out[i] = orc_rng_gaussian(r);
    return 0;
}

int orc_sample_gaussian(uint64_t seed, int d, double* out) {
    orc_rng r;
    orc_rng_init(&r, seed);
    return sample_into(&r, d, out);
}

/* ---- schedule ------------------------------------------------------------ */

/* schedule.cpp:29-58 (alpha_bar_table :15-25) */
int orc_build_schedule(int n, int t_grid, double entry, int* taus, double* alphas,
                       double* betas) {
    if (n < 1) return fail(1, "build_schedule: n must be >= 1");
    if (t_grid < 1) return fail(1, "build_schedule: t_grid must be >= 1");
    if (n > t_grid) return fail(1, "build_schedule: n exceeds t_grid");
    if (!(entry > 0.0 && entry <= 1.0))
        return fail(1, "build_schedule: entry_strength must lie in (0,1]");
    const long tau0 = lround(entry * (t_grid - 1));
    if (n > tau0 + 1)
        return fail(1, "build_schedule: n exceeds the usable range below the entry index");
    double* table = (double*)malloc(sizeof(double) * (size_t)t_grid);
    double prod = 1.0;
    for (int t = 0; t < t_grid; ++t) {
        const double frac = t_grid > 1 ? (double)t / (t_grid - 1) : 0.0;
        const double rate = 1e-4 + (2e-2 - 1e-4) * frac;
        prod *= 1.0 - rate;
        table[t] = prod;
    }
    const double stride = (double)(tau0 + 1) / n;
    for (int i = 0; i < n; ++i) {
        const long long tau = llround((double)tau0 - stride * i);
        taus[i] = (int)tau;
        alphas[i] = table[tau];
        betas[i] = 1.0 - table[tau];
    }
    free(table);
    for (int i = 1; i < n; ++i)
        if (taus[i] >= taus[i - 1]) return fail(2, "build_schedule: taus must strictly decrease");
    return 0;
}

/* schedule.cpp:80-89 (LcmParams defaults sigma_data 0.5, s 10: schedule.hpp:36-41) */
void orc_lcm_coefficients(int tau, double alpha, double beta, int mode, double* c_skip,
                          double* c_out) {
    (void)alpha;
    (void)beta;
    if (mode == 1) {
        *c_skip = tau == 0 ? 1.0 : 0.0;
        *c_out = tau == 0 ? 0.0 : 1.0;
        return;
    }
    const double sigma = 0.5, s = 10.0;
    const double st = s * tau;
    const double sig2 = sigma * sigma;
    *c_skip = sig2 / (st * st + sig2);
    *c_out = sigma * st / sqrt(sig2 + st * st);
}

/* ---- SSF ---------------------------------------------------------------- */

/* ssf.cpp:8-20 */
double orc_cosine(const double* a, const double* b, int d) {
    double dot = 0.0, na = 0.0, nb = 0.0;
    for (int i = 0; i < d; ++i) {
        dot += a[i] * b[i];
        na += a[i] * a[i];
        nb += b[i] * b[i];
    }
    na = sqrt(na);
    nb = sqrt(nb);
    if (na < 1e-12 || nb < 1e-12) return 0.0;
    return dot / (na * nb);
}

/* ssf.cpp:26-32 */
double orc_skip_probability(double sim, double eta) {
    const double p = (sim - eta) / (1.0 - eta);
    if (p <= 0.0) return 0.0;
    return p >= 1.0 ? 1.0 : p;
}

struct orc_ssf {
    double eta;
    orc_rng rng;
    double* ref;
    int d;
    int max_skip;
    int run;
    uint64_t examined, skipped;
};

int orc_ssf_create(double eta, uint64_t rng_seed, int max_skip, orc_ssf** out) {
    if (!(eta >= 0.0 && eta < 1.0)) return fail(1, "SsfState: eta must lie in [0,1)");
    orc_ssf* s = (orc_ssf*)calloc(1, sizeof *s);
    s->eta = eta;
    orc_rng_init(&s->rng, rng_seed);
    s->max_skip = max_skip;
    *out = s;
    return 0;
}

void orc_ssf_destroy(orc_ssf* s) {
    if (!s) return;
    free(s->ref);
    free(s);
}

/* ssf.cpp:39-54 (+ max_skip extension, off when max_skip <= 0) */
int orc_ssf_gate(orc_ssf* s, const double* payload, int d) {
    s->examined += 1;
    if (!s->ref) {
        s->ref = (double*)malloc(sizeof(double) * (size_t)d);
        memcpy(s->ref, payload, sizeof(double) * (size_t)d);
        s->d = d;
        s->run = 0;
        return 0;
    }
    if (d != s->d) return -fail(1, "cosine_similarity: dimension mismatch");
    const double sim = orc_cosine(payload, s->ref, d);
    const double p = orc_skip_probability(sim, s->eta);
    const double u = orc_rng_uniform(&s->rng);
    int skip = u < p;
    if (skip && s->max_skip > 0 && s->run >= s->max_skip) skip = 0;
    if (skip) {
        s->skipped += 1;
        s->run += 1;
        return 1;
    }
    memcpy(s->ref, payload, sizeof(double) * (size_t)d);
    s->run = 0;
    return 0;
}

void orc_ssf_counters(orc_ssf* s, uint64_t* examined, uint64_t* skipped) {
    *examined = s->examined;
    *skipped = s->skipped;
}

/* ---- engine ------------------------------------------------------------- */

typedef struct {
    int64_t seq;
    double* x0;
    double* cur;
    double* x0_ref;
    int step;
    int init;
    int64_t ingest_tick;
} slot_t;

struct orc_engine {
    orc_cfg cfg;
    int n, d;
    int* tau;
    double *alpha, *beta;
    double* eps_cached; /* n x d */
    double* cond;
    double* neg;
    slot_t* fl; /* oldest first */
    int count;
    int64_t ticks, last_seq;
    uint64_t calls, evals;
    double *scratch_eps, *scratch_neg;
};

static int validate(const orc_cfg* c) {
    if (c->n_steps < 1) return fail(1, "invalid config: n_steps must be >= 1");
    if (!(c->eta >= 0.0 && c->eta < 1.0)) return fail(1, "invalid config: eta out of range");
    if (!(c->gamma >= 0.0)) return fail(1, "invalid config: gamma must be >= 0");
    if (!(c->delta >= 0.0 && c->delta <= 1.0)) return fail(1, "invalid config: delta");
    if (c->d_latent < 1) return fail(1, "invalid config: d_latent must be >= 1");
    if (c->t_grid < 1) return fail(1, "invalid config: t_grid must be >= 1");
    if (c->n_steps > c->t_grid) return fail(1, "invalid config: n_steps must not exceed t_grid");
    if (!(c->entry_strength > 0.0 && c->entry_strength <= 1.0))
        return fail(1, "invalid config: entry_strength");
    if (!(c->data_variance > 0.0)) return fail(1, "invalid config: data_variance must be > 0");
    if (c->queue_capacity < 1) return fail(1, "invalid config: queue_capacity must be >= 1");
    if (c->codec != 0) return fail(1, "oracle restates the identity codec only");
    return 0;
}

int orc_engine_create(const orc_cfg* c, const double* cond, const double* neg, orc_engine** out) {
    int st = validate(c);
    if (st) return st;
    const int needs_neg = c->guidance_mode == 1 || c->guidance_mode == 3;
    if (needs_neg && !neg)
        return fail(1, "invalid config: negative_condition is required for cfg/onetime_negative modes");
    orc_engine* e = (orc_engine*)calloc(1, sizeof *e);
    e->cfg = *c;
    e->n = c->n_steps;
    e->d = c->d_latent;
    e->tau = (int*)malloc(sizeof(int) * (size_t)e->n);
    e->alpha = (double*)malloc(sizeof(double) * (size_t)e->n);
    e->beta = (double*)malloc(sizeof(double) * (size_t)e->n);
    st = orc_build_schedule(e->n, c->t_grid, c->entry_strength, e->tau, e->alpha, e->beta);
    if (st) {
        orc_engine_destroy(e);
        return st;
    }
    /* precompute.cpp:7-21: one Rng(derive_seed(seed, kStreamNoiseCache=1)), n draws of d */
    e->eps_cached = (double*)malloc(sizeof(double) * (size_t)e->n * (size_t)e->d);
    orc_rng r;
    orc_rng_init(&r, orc_derive_seed(c->seed, 1));
    for (int i = 0; i < e->n; ++i) sample_into(&r, e->d, e->eps_cached + (size_t)i * (size_t)e->d);
    e->cond = (double*)malloc(sizeof(double) * (size_t)e->d);
    memcpy(e->cond, cond, sizeof(double) * (size_t)e->d);
    if (neg) {
        e->neg = (double*)malloc(sizeof(double) * (size_t)e->d);
        memcpy(e->neg, neg, sizeof(double) * (size_t)e->d);
    }
    e->fl = (slot_t*)calloc((size_t)e->n + 1, sizeof(slot_t));
    e->last_seq = -1;
    e->scratch_eps = (double*)malloc(sizeof(double) * (size_t)e->d);
    e->scratch_neg = (double*)malloc(sizeof(double) * (size_t)e->d);
    *out = e;
    return 0;
}

static void free_slot(slot_t* s) {
    free(s->x0);
    free(s->cur);
    free(s->x0_ref);
    memset(s, 0, sizeof *s);
}

void orc_engine_destroy(orc_engine* e) {
    if (!e) return;
    if (e->fl)
        for (int i = 0; i < e->count; ++i) free_slot(&e->fl[i]);
    free(e->fl);
    free(e->tau);
    free(e->alpha);
    free(e->beta);
    free(e->eps_cached);
    free(e->cond);
    free(e->neg);
    free(e->scratch_eps);
    free(e->scratch_neg);
    free(e);
}

/* engine.cpp:53-76 */
int orc_engine_ingest(orc_engine* e, int64_t seq, const double* x0) {
    for (int i = 0; i < e->d; ++i)
        if (!isfinite(x0[i])) return fail(1, "ingest: non-finite latent");
    if (seq <= e->last_seq) return fail(1, "ingest: seq ids must strictly increase");
    for (int i = 0; i < e->count; ++i)
        if (e->fl[i].step == 0) return fail(2, "ingest: step-0 slot already occupied, tick first");
    slot_t* s = &e->fl[e->count++];
    const size_t bytes = sizeof(double) * (size_t)e->d;
    s->seq = seq;
    s->x0 = (double*)malloc(bytes);
    memcpy(s->x0, x0, bytes);
    s->cur = (double*)malloc(bytes);
    s->x0_ref = (double*)malloc(bytes);
    /* forward_diffuse (schedule.cpp:60-67) with eps_cached[0] */
    const double sa = sqrt(e->alpha[0]), sb = sqrt(e->beta[0]);
    for (int i = 0; i < e->d; ++i) s->cur[i] = sa * x0[i] + sb * e->eps_cached[i];
    s->step = 0;
    s->init = 0;
    s->ingest_tick = e->ticks;
    e->last_seq = seq;
    return 0;
}

/* AnalyticGaussianModel::do_predict (denoiser.cpp:26-43) */
static void analytic(const orc_engine* e, const double* x, double alpha, double beta,
                     const double* mu, double* out) {
    const double scale = sqrt(beta) / (alpha * e->cfg.data_variance + beta);
    const double sa = sqrt(alpha);
    for (int i = 0; i < e->d; ++i) out[i] = scale * (x[i] - sa * mu[i]);
}

/* combine_row (engine.cpp:17-32) -> cfg_combine / virtual_residual_noise / rcfg_combine
 * (guidance.cpp:19-48), in place on eps_c. */
static void combine(const orc_engine* e, const double* cur, double alpha, double beta,
                    double* eps_c, const double* eps_n, const double* x0_ref) {
    const double g = e->cfg.gamma, dl = e->cfg.delta;
    switch (e->cfg.guidance_mode) {
        case 0:
            return;
        case 1:
            for (int i = 0; i < e->d; ++i) eps_c[i] = eps_n[i] + g * (eps_c[i] - eps_n[i]);
            return;
        default: {
            if (beta <= 0.0) return;
            const double sa = sqrt(alpha), sb = sqrt(beta);
            for (int i = 0; i < e->d; ++i) {
                const double ev = (cur[i] - sa * x0_ref[i]) / sb;
                const double dv = dl * ev;
                eps_c[i] = dv + g * (eps_c[i] - dv);
            }
        }
    }
}

/* consistency_step (schedule.cpp:91-107) into out (may alias x) */
static void consistency(const orc_engine* e, const double* x, int step, int next,
                        const double* eps, double* out) {
    double cs, co;
    orc_lcm_coefficients(e->tau[step], e->alpha[step], e->beta[step], e->cfg.lcm_mode, &cs, &co);
    const double sa = sqrt(e->alpha[step]), sb = sqrt(e->beta[step]);
    const int terminal = next >= e->n;
    const double na = terminal ? 1.0 : e->alpha[next], nb = terminal ? 0.0 : e->beta[next];
    const double nsa = sqrt(na), nsb = sqrt(nb);
    const double* renoise = terminal ? NULL : e->eps_cached + (size_t)next * (size_t)e->d;
    for (int i = 0; i < e->d; ++i) {
        const double px0 = (x[i] - sb * eps[i]) / sa;
        const double x0_hat = cs * x[i] + co * px0;
        out[i] = terminal ? x0_hat : nsa * x0_hat + nsb * renoise[i];
    }
}

/* Cross-frame (Stream Batch) attention, engine.cpp:139-149 with attention.cpp:12-95:
 * every in-flight frame's guided eps is replaced by attention of its current latent
 * (lifted to kAttentionTokens = 4 identical token rows of width d) over keys = the
 * in-flight currents and values = their eps (the batch ordered by step index), then
 * unlifted by averaging the token rows.  The arithmetic follows the reference loop
 * for loop (fp64, sequential sums), so the result matches the reference build. */
static int tick_cross_frame(orc_engine* e, uint64_t rows, int64_t* emitted_seq, double* x0_hat, int64_t* ingest_tick,
                            int64_t* emit_tick, uint64_t* calls, uint64_t* evals) {
    const int b = e->count, d = e->d, mode = e->cfg.guidance_mode;
    enum { kTokens = 4 };
    double* eps = (double*)malloc(sizeof(double) * (size_t)b * (size_t)d);
    for (int i = 0; i < b; ++i) {
        slot_t* f = &e->fl[i];
        const double a = e->alpha[f->step], be = e->beta[f->step];
        double* ei = eps + (size_t)i * (size_t)d;
        analytic(e, f->cur, a, be, e->cond, ei);
        if (mode == 1) analytic(e, f->cur, a, be, e->neg, e->scratch_neg);
        combine(e, f->cur, a, be, ei, e->scratch_neg, mode == 3 ? f->x0_ref : f->x0);
    }
    /* build_attention_batch: frames ordered by step index (distinct per frame) */
    int* ord = (int*)malloc(sizeof(int) * (size_t)b);
    for (int i = 0; i < b; ++i) ord[i] = i;
    for (int i = 1; i < b; ++i)
        for (int j = i; j > 0 && e->fl[ord[j]].step < e->fl[ord[j - 1]].step; --j) {
            const int t = ord[j];
            ord[j] = ord[j - 1];
            ord[j - 1] = t;
        }
    const int nk = b * kTokens;
    const double inv_sqrt_d = 1.0 / sqrt((double)d);
    double* scores = (double*)malloc(sizeof(double) * (size_t)nk);
    double* out = (double*)malloc(sizeof(double) * (size_t)d);
    double* mixed = (double*)malloc(sizeof(double) * (size_t)b * (size_t)d);
    for (int i = 0; i < b; ++i) {
        const double* q = e->fl[i].cur;  /* every token row of the lifted query is cur_i */
        memset(out, 0, sizeof(double) * (size_t)d);
        double max_score = -INFINITY;
        for (int k = 0; k < nk; ++k) {
            const double* kr = e->fl[ord[k / kTokens]].cur;
            double dot = 0.0;
            for (int c = 0; c < d; ++c) dot += q[c] * kr[c];
            scores[k] = dot * inv_sqrt_d;
            max_score = scores[k] > max_score ? scores[k] : max_score;
        }
        double denom = 0.0;
        for (int k = 0; k < nk; ++k) {
            scores[k] = exp(scores[k] - max_score);
            denom += scores[k];
        }
        for (int k = 0; k < nk; ++k) {
            const double w = scores[k] / denom;
            const double* vr = eps + (size_t)ord[k / kTokens] * (size_t)d;
            for (int c = 0; c < d; ++c) out[c] += w * vr[c];
        }
        /* unlift_tokens: the kTokens identical rows summed in order, divided by kTokens */
        double* mi = mixed + (size_t)i * (size_t)d;
        for (int c = 0; c < d; ++c) {
            double sum = 0.0;
            for (int t = 0; t < kTokens; ++t) sum += out[c];
            mi[c] = sum / (double)kTokens;
        }
    }
    e->ticks += 1;
    e->calls += 1;
    e->evals += rows;
    *emitted_seq = -1;
    int emit_index = -1, st = 0;
    for (int i = 0; i < b && !st; ++i) {
        slot_t* f = &e->fl[i];
        const int next = f->step + 1;
        consistency(e, f->cur, f->step, next, mixed + (size_t)i * (size_t)d, f->cur);
        f->step = next;
        if (f->step == e->n) {
            for (int k = 0; k < d; ++k)
                if (!isfinite(f->cur[k])) st = fail(3, "tick: non-finite latent at emission");
            if (st) break;
            *emitted_seq = f->seq;
            if (x0_hat) memcpy(x0_hat, f->cur, sizeof(double) * (size_t)d);
            *ingest_tick = f->ingest_tick;
            *emit_tick = e->ticks;
            emit_index = i;
        }
    }
    free(eps);
    free(ord);
    free(scores);
    free(out);
    free(mixed);
    if (st) return st;
    if (emit_index >= 0) {
        free_slot(&e->fl[emit_index]);
        for (int i = emit_index; i + 1 < e->count; ++i) e->fl[i] = e->fl[i + 1];
        memset(&e->fl[e->count - 1], 0, sizeof(slot_t));
        e->count -= 1;
    }
    *calls = 1;
    *evals = rows;
    return 0;
}

/* engine.cpp:78-195 */
int orc_engine_tick(orc_engine* e, int64_t* emitted_seq, double* x0_hat, int64_t* ingest_tick,
                    int64_t* emit_tick, uint64_t* calls, uint64_t* evals) {
    if (e->count == 0) return fail(2, "tick: no in-flight frames");
    const int b = e->count;
    const int mode = e->cfg.guidance_mode;
    uint64_t rows = (uint64_t)b;
    if (mode == 1) rows += (uint64_t)b;
    /* onetime init rows: x0_ref = predict_x0(current, steps[0], eps_neg) (engine.cpp:122-126) */
    if (mode == 3) {
        for (int i = 0; i < b; ++i) {
            slot_t* f = &e->fl[i];
            if (f->step == 0 && !f->init) {
                rows += 1;
                analytic(e, f->cur, e->alpha[0], e->beta[0], e->neg, e->scratch_neg);
                if (e->alpha[0] <= 0.0) return fail(1, "predict_x0: singular step (alpha = 0)");
                const double sa = sqrt(e->alpha[0]), sb = sqrt(e->beta[0]);
                for (int k = 0; k < e->d; ++k) f->x0_ref[k] = (f->cur[k] - sb * e->scratch_neg[k]) / sa;
                f->init = 1;
            }
        }
    }
    if (e->cfg.cross_frame_attention) return tick_cross_frame(e, rows, emitted_seq, x0_hat, ingest_tick, emit_tick, calls, evals);
    /* eps rows per frame, then the consistency transition.  The reference
     * computes all eps before any update; per-frame rows are independent so
     * the interleaving does not change any value. */
    e->ticks += 1;
    e->calls += 1;
    e->evals += rows;
    *emitted_seq = -1;
    int emit_index = -1;
    for (int i = 0; i < b; ++i) {
        slot_t* f = &e->fl[i];
        const double a = e->alpha[f->step], be = e->beta[f->step];
        analytic(e, f->cur, a, be, e->cond, e->scratch_eps);
        if (mode == 1) analytic(e, f->cur, a, be, e->neg, e->scratch_neg);
        const double* x0_ref = mode == 3 ? f->x0_ref : f->x0;
        combine(e, f->cur, a, be, e->scratch_eps, e->scratch_neg, x0_ref);
        const int next = f->step + 1;
        consistency(e, f->cur, f->step, next, e->scratch_eps, f->cur);
        f->step = next;
        if (f->step == e->n) {
            for (int k = 0; k < e->d; ++k)
                if (!isfinite(f->cur[k])) return fail(3, "tick: non-finite latent at emission");
            *emitted_seq = f->seq;
            if (x0_hat) memcpy(x0_hat, f->cur, sizeof(double) * (size_t)e->d);
            *ingest_tick = f->ingest_tick;
            *emit_tick = e->ticks;
            emit_index = i;
        }
    }
    if (emit_index >= 0) {
        free_slot(&e->fl[emit_index]);
        for (int i = emit_index; i + 1 < e->count; ++i) e->fl[i] = e->fl[i + 1];
        memset(&e->fl[e->count - 1], 0, sizeof(slot_t));
        e->count -= 1;
    }
    *calls = 1;
    *evals = rows;
    return 0;
}

int orc_engine_idle(orc_engine* e) { return e->count == 0; }
int64_t orc_engine_ticks(orc_engine* e) { return e->ticks; }
int orc_engine_inflight(orc_engine* e) { return e->count; }

/* engine.cpp:205-211 */
int64_t orc_engine_min_inflight_seq(orc_engine* e) {
    int64_t m = INT64_MAX;
    for (int i = 0; i < e->count; ++i)
        if (e->fl[i].seq < m) m = e->fl[i].seq;
    return m;
}

static int cmp_int(const void* a, const void* b) { return *(const int*)a - *(const int*)b; }

/* engine.cpp:197-203 */
int orc_engine_step_indices(orc_engine* e, int* out) {
    for (int i = 0; i < e->count; ++i) out[i] = e->fl[i].step;
    qsort(out, (size_t)e->count, sizeof(int), cmp_int);
    return e->count;
}

void orc_engine_counters(orc_engine* e, uint64_t* calls, uint64_t* evals) {
    *calls = e->calls;
    *evals = e->evals;
}

void orc_engine_eps_cached(orc_engine* e, int step, double* out) {
    memcpy(out, e->eps_cached + (size_t)step * (size_t)e->d, sizeof(double) * (size_t)e->d);
}

/* run_sequential_reference (engine.cpp:213-238) with guided_eps (guidance.cpp:64-103) */
int orc_sequential(const orc_cfg* c, const double* cond, const double* neg, const double* x0,
                   double* out) {
    orc_engine* e = NULL;
    int st = orc_engine_create(c, cond, neg, &e);
    if (st) return st;
    const int d = e->d, n = e->n, mode = c->guidance_mode;
    double* x = out;
    double* x0_ref = (double*)malloc(sizeof(double) * (size_t)d);
    const double sa0 = sqrt(e->alpha[0]), sb0 = sqrt(e->beta[0]);
    for (int i = 0; i < d; ++i) x[i] = sa0 * x0[i] + sb0 * e->eps_cached[i];
    if (mode == 3) { /* init_onetime_negative (guidance.cpp:50-62) */
        analytic(e, x, e->alpha[0], e->beta[0], e->neg, e->scratch_neg);
        for (int i = 0; i < d; ++i) x0_ref[i] = (x[i] - sb0 * e->scratch_neg[i]) / sa0;
    }
    for (int s = 0; s < n; ++s) {
        const double a = e->alpha[s], be = e->beta[s];
        analytic(e, x, a, be, e->cond, e->scratch_eps);
        if (mode == 1) analytic(e, x, a, be, e->neg, e->scratch_neg);
        combine(e, x, a, be, e->scratch_eps, e->scratch_neg, mode == 3 ? x0_ref : x0);
        consistency(e, x, s, s + 1, e->scratch_eps, x);
    }
    free(x0_ref);
    orc_engine_destroy(e);
    return 0;
}

/* ---- pipeline ----------------------------------------------------------- */

/* BoundedQueue drop-oldest FIFO (queue.hpp:23-40) over opaque items. */
typedef struct {
    int64_t* seq;
    double** payload; /* owned; NULL for skip tokens / stale */
    int* skip;
    int head, size, cap, ring;
    uint64_t dropped;
} q_t;

static void q_init(q_t* q, int cap) {
    q->cap = cap;
    q->ring = cap + 1;
    q->seq = (int64_t*)calloc((size_t)q->ring, sizeof(int64_t));
    q->payload = (double**)calloc((size_t)q->ring, sizeof(double*));
    q->skip = (int*)calloc((size_t)q->ring, sizeof(int));
    q->head = q->size = 0;
    q->dropped = 0;
}

static void q_push(q_t* q, int64_t seq, double* payload, int skip) {
    const int tail = (q->head + q->size) % q->ring;
    q->seq[tail] = seq;
    q->payload[tail] = payload;
    q->skip[tail] = skip;
    q->size += 1;
    if (q->size > q->cap) {
        free(q->payload[q->head]);
        q->head = (q->head + 1) % q->ring;
        q->size -= 1;
        q->dropped += 1;
    }
}

static int q_pop(q_t* q, int64_t* seq, double** payload, int* skip) {
    if (q->size == 0) return 0;
    *seq = q->seq[q->head];
    *payload = q->payload[q->head];
    *skip = q->skip[q->head];
    q->head = (q->head + 1) % q->ring;
    q->size -= 1;
    return 1;
}

static void q_free(q_t* q) {
    int64_t s;
    double* p;
    int k;
    while (q_pop(q, &s, &p, &k)) free(p);
    free(q->seq);
    free(q->payload);
    free(q->skip);
}

typedef struct {
    int64_t* seq;
    double* payload;
    int cap, count, d;
} sink_t;

static void sink_put(sink_t* s, int64_t seq, const double* payload) {
    if (s->count < s->cap) {
        s->seq[s->count] = seq;
        if (s->payload)
            memcpy(s->payload + (size_t)s->count * (size_t)s->d, payload, sizeof(double) * (size_t)s->d);
    }
    s->count += 1;
}

/* run_pipeline deterministic mode (pipeline.cpp:152-214, EngineStage :39-133,
 * report :288-339) with the identity codec. */
int orc_run_pipeline(const orc_cfg* c, const double* cond_in, const double* neg,
                     const double* frames, int nframes, int d, int max_skip, int64_t* out_seq,
                     double* out_payload, int out_cap, int* n_out, int* decisions,
                     orc_report* rep) {
    memset(rep, 0, sizeof *rep);
    int st = validate(c);
    if (st) return st;
    const size_t bytes = sizeof(double) * (size_t)c->d_latent;
    double* cond = (double*)malloc(bytes);
    if (cond_in) {
        memcpy(cond, cond_in, bytes);
    } else { /* resolve_condition (pipeline.cpp:30-34) */
        orc_rng r;
        orc_rng_init(&r, orc_derive_seed(c->seed, 4));
        sample_into(&r, c->d_latent, cond);
    }
    orc_engine* e = NULL;
    st = orc_engine_create(c, cond, neg, &e);
    free(cond);
    if (st) return st;
    orc_ssf* ssf = NULL;
    if (c->ssf_enabled) orc_ssf_create(c->eta, orc_derive_seed(c->seed, 2), max_skip, &ssf);

    q_t in_q, out_q;
    q_init(&in_q, c->queue_capacity);
    q_init(&out_q, c->queue_capacity * 8);
    sink_t sink = {out_seq, out_payload, out_cap, 0, c->d_latent};

    int64_t* pending = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nframes + 1));
    int p_head = 0, p_tail = 0;
    double* last_output = NULL;
    int64_t* lats = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nframes + 1));
    int n_lats = 0;
    int next_frame = 0, source_done = 0;
    double* xhat = (double*)malloc(bytes);

#define FLUSH_BELOW(limit)                                                  \
    while (p_head < p_tail && pending[p_head] < (limit)) {                  \
        const int64_t sq = pending[p_head++];                               \
        if (!last_output) {                                                 \
            rep->stale_skips += 1;                                          \
            continue;                                                       \
        }                                                                   \
        double* dup = (double*)malloc(bytes);                               \
        memcpy(dup, last_output, bytes);                                    \
        rep->duplicates += 1;                                               \
        q_push(&out_q, sq, dup, 0);                                         \
    }
#define DRAIN()                                                             \
    {                                                                       \
        int64_t sq;                                                         \
        double* pl;                                                         \
        int sk;                                                             \
        while (q_pop(&out_q, &sq, &pl, &sk)) {                              \
            sink_put(&sink, sq, pl);                                        \
            free(pl);                                                       \
            rep->frames_out += 1;                                           \
        }                                                                   \
    }

    for (;;) {
        /* pre_step (pipeline.cpp:173-186) */
        if (!source_done) {
            if (next_frame >= nframes) {
                source_done = 1;
            } else {
                const double* f = frames + (size_t)next_frame * (size_t)d;
                rep->frames_in += 1;
                int skip = 0;
                if (ssf) {
                    const int g = orc_ssf_gate(ssf, f, d);
                    if (g < 0) {
                        rep->incomplete = 1;
                        break;
                    }
                    skip = g;
                }
                if (decisions) decisions[next_frame] = skip;
                double* payload = NULL;
                if (!skip) {
                    payload = (double*)malloc(sizeof(double) * (size_t)d);
                    memcpy(payload, f, sizeof(double) * (size_t)d);
                }
                q_push(&in_q, next_frame, payload, skip);
                next_frame += 1;
            }
        }
        /* dequeue -> EngineStage::on_item (pipeline.cpp:55-61) */
        {
            int64_t sq;
            double* pl;
            int sk;
            if (q_pop(&in_q, &sq, &pl, &sk)) {
                if (sk) {
                    pending[p_tail++] = sq;
                } else {
                    const int ist = d != c->d_latent ? fail(1, "ingest: latent length != d_latent")
                                                     : orc_engine_ingest(e, sq, pl);
                    free(pl);
                    if (ist) {
                        rep->incomplete = 1;
                        break;
                    }
                }
            }
        }
        /* tick_once (pipeline.cpp:65-76) */
        if (!orc_engine_idle(e)) {
            int64_t es, it, et;
            uint64_t ca, ev;
            if (orc_engine_tick(e, &es, xhat, &it, &et, &ca, &ev)) {
                rep->incomplete = 1;
                break;
            }
            if (es >= 0) {
                FLUSH_BELOW(es);
                lats[n_lats++] = et - it;
                double* outp = (double*)malloc(bytes);
                memcpy(outp, xhat, bytes);
                if (!last_output) last_output = (double*)malloc(bytes);
                memcpy(last_output, xhat, bytes);
                q_push(&out_q, es, outp, 0);
            }
        }
        /* flush_ready_skips (pipeline.cpp:80-82) */
        {
            const int64_t lim = orc_engine_min_inflight_seq(e);
            FLUSH_BELOW(lim);
        }
        DRAIN();
        if (source_done && in_q.size == 0 && orc_engine_idle(e)) {
            FLUSH_BELOW(INT64_MAX);
            DRAIN();
            break;
        }
    }
#undef FLUSH_BELOW
#undef DRAIN

    rep->input_drops = in_q.dropped;
    rep->output_drops = out_q.dropped;
    rep->ticks = (uint64_t)e->ticks;
    rep->denoiser_calls = e->calls;
    rep->element_evals = e->evals;
    if (ssf) {
        rep->ssf_examined = ssf->examined;
        rep->ssf_skipped = ssf->skipped;
        rep->skip_rate = ssf->examined == 0 ? 0.0 : (double)ssf->skipped / (double)ssf->examined;
    }
    if (n_lats > 0) {
        int64_t lo = lats[0], hi = lats[0], sum = 0;
        for (int i = 0; i < n_lats; ++i) {
            lo = lats[i] < lo ? lats[i] : lo;
            hi = lats[i] > hi ? lats[i] : hi;
            sum += lats[i];
        }
        rep->latency_ticks_min = lo;
        rep->latency_ticks_max = hi;
        rep->latency_ticks_mean = (double)sum / (double)n_lats;
    }
    if (rep->frames_out > 0) {
        rep->mean_frame_time_ms = (double)rep->ticks / (double)rep->frames_out;
        rep->throughput_fps = 1000.0 / rep->mean_frame_time_ms;
        rep->wall_ms = (double)rep->ticks;
    }
    *n_out = sink.count;
    free(xhat);
    free(lats);
    free(pending);
    free(last_output);
    q_free(&in_q);
    q_free(&out_q);
    orc_ssf_destroy(ssf);
    orc_engine_destroy(e);
    return 0;
}

/* ---- StreamGenerator (stream_gen.cpp:11-71), defaults noise 1.0, period 20, static 0.5 */
int orc_stream_frames(int kind, int d, uint64_t seed, int nframes, double* out) {
    if (d < 1) return fail(1, "StreamGenerator: d must be >= 1");
    orc_rng r;
    orc_rng_init(&r, orc_derive_seed(seed, 3));
    const int period = 20;
    const int dynamic_len = period - (int)lround(period * 0.5);
    const double target = sqrt((double)d);
    double* state = (double*)malloc(sizeof(double) * (size_t)d);
    double* step = (double*)malloc(sizeof(double) * (size_t)d);
    /* randomize_state */
    sample_into(&r, d, state);
    {
        double norm = 0.0;
        for (int i = 0; i < d; ++i) norm += state[i] * state[i];
        norm = sqrt(norm);
        if (norm < 1e-12) norm = 1.0;
        for (int i = 0; i < d; ++i) state[i] *= target / norm;
    }
    for (int64_t seq = 0; seq < nframes; ++seq) {
        int walk = 0;
        if (kind == 1) walk = seq > 0;
        if (kind == 2) walk = seq > 0 && (int)(seq % period) < dynamic_len;
        if (walk) {
            sample_into(&r, d, step);
            double norm = 0.0;
            for (int i = 0; i < d; ++i) {
                state[i] += 1.0 * step[i];
                norm += state[i] * state[i];
            }
            norm = sqrt(norm);
            if (norm < 1e-12) {
                sample_into(&r, d, state);
                double n2 = 0.0;
                for (int i = 0; i < d; ++i) n2 += state[i] * state[i];
                n2 = sqrt(n2);
                if (n2 < 1e-12) n2 = 1.0;
                for (int i = 0; i < d; ++i) state[i] *= target / n2;
            } else {
                for (int i = 0; i < d; ++i) state[i] *= target / norm;
            }
        }
        memcpy(out + (size_t)seq * (size_t)d, state, sizeof(double) * (size_t)d);
    }
    free(state);
    free(step);
    return 0;
}
