/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY (see oracle.h for the contract).
 *
 * f64 CPU restatement of the reference path.  Every routine mirrors the
 * evaluation ORDER of the reference (tape.hpp / optim.hpp / rng.hpp) so that
 * it is bit-identical to the reference built from /root/reference headers
 * (oracle/_ref/libmtref.so); tests/test_oracle.py checks that.  Build with
 * -ffp-contract=off (FMA contraction changes the
 * bits of Rng::uniform(lo,hi), rng.hpp:22).
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ======================================================================= */
/* RNG -- mt::Rng, rng.hpp:13-75 (std::mt19937_64 + hand-rolled dists)     */
/* ======================================================================= */
#define MT_N 312
#define MT_M 156
#define MT_UPPER 0xFFFFFFFF80000000ULL
#define MT_LOWER 0x000000007FFFFFFFULL

size_t orc_rng_sizeof(void) { return sizeof(orc_rng); }

/* std::mt19937_64 seeding (rng.hpp:15 constructs gen_(seed)) */
void orc_rng_seed(orc_rng* r, uint64_t seed) {
    r->state[0] = seed;
    for (int i = 1; i < MT_N; ++i) {
        uint64_t prev = r->state[i - 1];
        r->state[i] = 6364136223846793005ULL * (prev ^ (prev >> 62)) + (uint64_t)i;
    }
    r->pos = MT_N;
    r->has_spare = 0;
    r->spare = 0.0;
}

static void mt_regenerate(orc_rng* r) {
    uint64_t* s = r->state;
    for (int i = 0; i < MT_N; ++i) {
        uint64_t y = (s[i] & MT_UPPER) | (s[(i + 1) % MT_N] & MT_LOWER);
        uint64_t v = s[(i + MT_M) % MT_N] ^ (y >> 1);
        if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
        s[i] = v;
    }
    r->pos = 0;
}

/* Rng::next_u64 (rng.hpp:17) */
uint64_t orc_rng_next(orc_rng* r) {
    if (r->pos >= MT_N) mt_regenerate(r);
    uint64_t y = r->state[r->pos++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

/* Rng::uniform -- 53 random bits (rng.hpp:20) */
double orc_rng_uniform(orc_rng* r) { return (double)(orc_rng_next(r) >> 11) * 0x1.0p-53; }

/* Rng::uniform(lo,hi) (rng.hpp:22); needs -ffp-contract=off */
double orc_rng_uniform_range(orc_rng* r, double lo, double hi) {
    double u = orc_rng_uniform(r);
    double span = hi - lo;
    double t = span * u;
    return lo + t;
}

/* Rng::normal -- Box-Muller with cached spare (rng.hpp:24-37) */
double orc_rng_normal(orc_rng* r) {
    if (r->has_spare) {
        r->has_spare = 0;
        return r->spare;
    }
    double u = 1.0 - orc_rng_uniform(r);
    double v = orc_rng_uniform(r);
    double rad = sqrt(-2.0 * log(u));
    double ang = 6.28318530717958647692 * v;
    r->spare = rad * sin(ang);
    r->has_spare = 1;
    return rad * cos(ang);
}

/* Rng::below -- rejection sampling (rng.hpp:39-46) */
uint64_t orc_rng_below(orc_rng* r, uint64_t n) {
    if (n == 0) return 0;
    uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    uint64_t x;
    do {
        x = orc_rng_next(r);
    } while (x >= limit);
    return x % n;
}

/* Rng::permutation = iota + Fisher-Yates from the top (rng.hpp:50-63) */
void orc_rng_permutation(orc_rng* r, size_t n, uint64_t* out) {
    for (size_t i = 0; i < n; ++i) out[i] = i;
    for (size_t i = n; i > 1; --i) {
        size_t j = (size_t)orc_rng_below(r, i);
        uint64_t t = out[i - 1];
        out[i - 1] = out[j];
        out[j] = t;
    }
}

/* Rng::split consumes one parent draw (rng.hpp:65-69) */
void orc_rng_split(orc_rng* parent, uint64_t stream, orc_rng* child) {
    uint64_t s = orc_rng_next(parent) ^ (0x9e3779b97f4a7c15ULL * (stream + 1));
    orc_rng_seed(child, s);
}

void orc_rng_fill_normal(orc_rng* r, double* out, size_t n) {
    for (size_t i = 0; i < n; ++i) out[i] = orc_rng_normal(r);
}

void orc_rng_fill_uniform_range(orc_rng* r, double* out, size_t n, double lo, double hi) {
    for (size_t i = 0; i < n; ++i) out[i] = orc_rng_uniform_range(r, lo, hi);
}

/* ======================================================================= */
/* Dense loops -- detail::mm_acc / mm_nt_acc / mm_tn_acc (tape.hpp:36-78)  */
/* ======================================================================= */
void orc_mm_acc(const double* a, const double* b, double* c, size_t M, size_t K, size_t N) {
    for (size_t i = 0; i < M; ++i)
        for (size_t p = 0; p < K; ++p) {
            const double av = a[i * K + p];
            for (size_t j = 0; j < N; ++j) c[i * N + j] += av * b[p * N + j];
        }
}

void orc_mm_nt_acc(const double* a, const double* b, double* c, size_t M, size_t N, size_t K) {
    for (size_t i = 0; i < M; ++i)
        for (size_t j = 0; j < N; ++j) {
            double acc = 0.0;
            for (size_t q = 0; q < K; ++q) acc += a[i * K + q] * b[j * K + q];
            c[i * N + j] += acc;
        }
}

/* optim.hpp:49-63: m = b1 m + (1-b1) g; v = b2 v + (1-b2) g g;
 * w -= lr (m / bc1) / (sqrt(v / bc2) + eps), bc = 1 - beta^step.        */
void orc_adam_update(double* w, const double* g, double* m, double* v, size_t n, double lr,
                     double beta1, double beta2, double eps, uint64_t step) {
    const double bc1 = 1.0 - pow(beta1, (double)step);
    const double bc2 = 1.0 - pow(beta2, (double)step);
    for (size_t i = 0; i < n; ++i) {
        m[i] = beta1 * m[i] + (1.0 - beta1) * g[i];
        v[i] = beta2 * v[i] + (1.0 - beta2) * g[i] * g[i];
        const double mhat = m[i] / bc1;
        const double vhat = v[i] / bc2;
        w[i] -= lr * mhat / (sqrt(vhat) + eps);
    }
}

void orc_mm_tn_acc(const double* a, const double* g, double* c, size_t M, size_t K, size_t N) {
    for (size_t i = 0; i < M; ++i)
        for (size_t p = 0; p < K; ++p) {
            const double av = a[i * K + p];
            if (av == 0.0) continue; /* tape.hpp:73 */
            for (size_t j = 0; j < N; ++j) c[p * N + j] += av * g[i * N + j];
        }
}

/* ======================================================================= */
/* MLP                                                                     */
/* ======================================================================= */
static int all_finite(const double* x, size_t n) {
    for (size_t i = 0; i < n; ++i)
        if (!isfinite(x[i])) return 0;
    return 1;
}

/* Tape::add_bias forward (tape.hpp:204-221): out = x; out[i] += b[i % h] */
static void add_bias_fwd(double* z, const double* b, size_t rows, size_t h) {
    for (size_t i = 0; i < rows * h; ++i) z[i] += b[i % h];
}

/* Tape::relu forward (tape.hpp:342-352) */
static void relu_fwd(const double* z, double* out, size_t n) {
    for (size_t i = 0; i < n; ++i) out[i] = z[i] > 0.0 ? z[i] : 0.0;
}

/* Tape::cross_entropy_weighted forward + backward (tape.hpp:475-520).
 * grad_in is the incoming scalar gradient of the CE node (1.0 here).
 * dlogits must be zero-initialised; it receives (g/denom)*w_i*(P - onehot). */
static int ce_weighted(const double* x, size_t b, size_t n, const int32_t* labels,
                       const double* weights, double denom, double grad_in, double* loss_out,
                       double* dlogits) {
    if (denom <= 0.0) return 2;
    for (size_t i = 0; i < b; ++i)
        if (labels[i] < 0 || (size_t)labels[i] >= n) return 2;
    double* probs = (double*)malloc(sizeof(double) * b * n);
    double loss = 0.0;
    for (size_t i = 0; i < b; ++i) {
        const double* row = x + i * n;
        double mx = row[0];
        for (size_t j = 1; j < n; ++j) mx = row[j] > mx ? row[j] : mx;
        double z = 0.0;
        for (size_t j = 0; j < n; ++j) z += exp(row[j] - mx);
        const double lse = mx + log(z);
        const double wi = weights ? weights[i] : 1.0;
        loss += wi * (lse - row[labels[i]]);
        for (size_t j = 0; j < n; ++j) probs[i * n + j] = exp(row[j] - lse);
    }
    loss /= denom;
    *loss_out = loss;
    if (dlogits) {
        const double g = grad_in / denom;
        for (size_t i = 0; i < b; ++i) {
            const double wi = g * (weights ? weights[i] : 1.0);
            if (wi == 0.0) continue;
            for (size_t j = 0; j < n; ++j) dlogits[i * n + j] += wi * probs[i * n + j];
            dlogits[i * n + labels[i]] -= wi;
        }
    }
    free(probs);
    return isfinite(loss) ? 0 : 5;
}

typedef struct {
    double** z;  /* pre-activation per layer [rows, dims[l+1]] */
    double** h;  /* h[0] = X (borrowed); h[l+1] = relu(z[l]) for l < L-1 */
} branch_fwd;

static int branch_forward(int L, const int* dims, const double* const* W, const double* const* b,
                          const double* Wh, const double* bh, const double* X, size_t rows,
                          branch_fwd* f) {
    f->z = (double**)calloc((size_t)L, sizeof(double*));
    f->h = (double**)calloc((size_t)L, sizeof(double*));
    f->h[0] = (double*)X;
    for (int l = 0; l < L; ++l) {
        const size_t k = (size_t)dims[l], n = (size_t)dims[l + 1];
        const double* Wl = (l == L - 1) ? Wh : W[l];
        const double* bl = (l == L - 1) ? bh : b[l];
        f->z[l] = (double*)calloc(rows * n, sizeof(double));
        orc_mm_acc(f->h[l], Wl, f->z[l], rows, k, n);
        if (!all_finite(f->z[l], rows * n)) return 5; /* tape.hpp:916 */
        add_bias_fwd(f->z[l], bl, rows, n);
        if (!all_finite(f->z[l], rows * n)) return 5;
        if (l < L - 1) {
            f->h[l + 1] = (double*)malloc(sizeof(double) * rows * n);
            relu_fwd(f->z[l], f->h[l + 1], rows * n);
        }
    }
    return 0;
}

static void branch_free(int L, branch_fwd* f) {
    if (!f->z) return;
    for (int l = 0; l < L; ++l) {
        free(f->z[l]);
        if (l > 0) free(f->h[l]);
    }
    free(f->z);
    free(f->h);
    f->z = NULL;
    f->h = NULL;
}

/* Reverse sweep of one branch given d(logits), accumulating into the param
 * gradient buffers gW/gb (running sums, as the Tape's shared param node
 * grads).  gWh/gbh receive the head's gradient.  dh_inject (optional) is
 * the gradient already sitting on h[L-1] before the head matmul's backward
 * adds to it (the sum(mul(h, constant(G))) injection, tape.hpp:153-171,
 * 406-416).  Layers < frozen receive no gradient.                          */
static void branch_backward(int L, const int* dims, int frozen, const double* const* W,
                            const double* Wh, const branch_fwd* f, size_t rows,
                            const double* dlogits, const double* dh_inject, double* const* gW,
                            double* const* gb, double* gWh, double* gbh) {
    size_t n = (size_t)dims[L];
    double* g = (double*)malloc(sizeof(double) * rows * n);
    memcpy(g, dlogits, sizeof(double) * rows * n);
    for (int l = L - 1; l >= 0; --l) {
        const size_t k = (size_t)dims[l];
        n = (size_t)dims[l + 1];
        const double* Wl = (l == L - 1) ? Wh : W[l];
        double* gWl = (l == L - 1) ? gWh : gW[l];
        double* gbl = (l == L - 1) ? gbh : gb[l];
        /* add_bias backward: accum(parent, g) -> 0 + g; gb[i%h] += g[i] */
        double* gmm = (double*)malloc(sizeof(double) * rows * n);
        for (size_t i = 0; i < rows * n; ++i) gmm[i] = 0.0 + g[i];
        if (l >= frozen)
            for (size_t i = 0; i < rows * n; ++i) gbl[i % n] += g[i];
        free(g);
        g = NULL;
        /* matmul backward: dX via mm_nt_acc, then dW via mm_tn_acc (tape.hpp:238-244) */
        double* gh = NULL;
        if (l > 0 && l > frozen) {
            gh = (double*)calloc(rows * k, sizeof(double));
            if (l == L - 1 && dh_inject)
                for (size_t i = 0; i < rows * k; ++i) gh[i] += 1.0 * dh_inject[i];
            orc_mm_nt_acc(gmm, Wl, gh, rows, k, n);
        }
        if (l >= frozen) orc_mm_tn_acc(f->h[l], gmm, gWl, rows, k, n);
        free(gmm);
        if (!gh) break;
        /* relu backward (tape.hpp:345-350): strictly x > 0 */
        g = (double*)calloc(rows * k, sizeof(double));
        const double* zin = f->z[l - 1];
        for (size_t i = 0; i < rows * k; ++i)
            if (zin[i] > 0.0) g[i] += gh[i];
        free(gh);
    }
    free(g);
}

int orc_mlp_forward(int n_layers, const int* dims, int head, const double* const* W,
                    const double* const* b, const double* X, int B, double* logits,
                    double* hidden_last) {
    if (n_layers < 1 || B < 1) return 1;
    const int L = n_layers;
    const double* Wh = W[L - 1 + (head ? 1 : 0)];
    const double* bh = b[L - 1 + (head ? 1 : 0)];
    branch_fwd f = {0};
    int st = branch_forward(L, dims, W, b, Wh, bh, X, (size_t)B, &f);
    if (st == 0) {
        memcpy(logits, f.z[L - 1], sizeof(double) * (size_t)B * (size_t)dims[L]);
        if (hidden_last && L > 1)
            memcpy(hidden_last, f.h[L - 1], sizeof(double) * (size_t)B * (size_t)dims[L - 1]);
    }
    branch_free(L, &f);
    return st;
}

int orc_mlp_train_step(int n_layers, const int* dims, int n_heads, int frozen_layers,
                       double* const* W, double* const* b, const double* X, int B, int src_rows,
                       const int32_t* y, const double* w, const double* denoms, double lr,
                       const double* dH_inject, double* loss_out, double* const* dW_out,
                       double* const* db_out) {
    const int L = n_layers;
    if (L < 1 || B < 1 || (n_heads != 1 && n_heads != 2)) return 1;
    if (n_heads == 2 && (src_rows <= 0 || src_rows >= B || L < 2 || dH_inject)) return 1;
    const int n_mats = L + n_heads - 1;
    const size_t C = (size_t)dims[L];
    /* parameter-gradient buffers (Parameter::grad after zero_grads) */
    double** gW = (double**)calloc((size_t)n_mats, sizeof(double*));
    double** gb = (double**)calloc((size_t)n_mats, sizeof(double*));
    for (int i = 0; i < n_mats; ++i) {
        const int l = i < L ? i : L - 1;
        gW[i] = (double*)calloc((size_t)dims[l] * (size_t)dims[l + 1], sizeof(double));
        gb[i] = (double*)calloc((size_t)dims[l + 1], sizeof(double));
    }
    int st = 0;
    double loss = 0.0;
    if (n_heads == 1) {
        branch_fwd f = {0};
        st = branch_forward(L, dims, (const double* const*)W, (const double* const*)b, W[L - 1],
                            b[L - 1], X, (size_t)B, &f);
        double* dl = (double*)calloc((size_t)B * C, sizeof(double));
        if (st == 0) st = ce_weighted(f.z[L - 1], (size_t)B, C, y, w, denoms[0], 1.0, &loss, dl);
        if (st == 0)
            branch_backward(L, dims, frozen_layers, (const double* const*)W, W[L - 1], &f,
                            (size_t)B, dl, dH_inject, gW, gb, gW[L - 1], gb[L - 1]);
        free(dl);
        branch_free(L, &f);
    } else {
        /* parameter-based: src branch (head 0) built first, tgt branch
         * (head 1) second; loss = add(CE_s, CE_t).  The reverse sweep visits
         * the tgt branch first, so the shared trunk gradients accumulate tgt
         * rows then src rows. */
        const size_t ns = (size_t)src_rows, nt = (size_t)B - ns;
        const size_t d0 = (size_t)dims[0];
        branch_fwd fs = {0}, ft = {0};
        st = branch_forward(L, dims, (const double* const*)W, (const double* const*)b, W[L - 1],
                            b[L - 1], X, ns, &fs);
        if (st == 0)
            st = branch_forward(L, dims, (const double* const*)W, (const double* const*)b, W[L],
                                b[L], X + ns * d0, nt, &ft);
        double* dls = (double*)calloc(ns * C, sizeof(double));
        double* dlt = (double*)calloc(nt * C, sizeof(double));
        double ls = 0.0, lt = 0.0;
        if (st == 0) st = ce_weighted(fs.z[L - 1], ns, C, y, w, denoms[0], 1.0, &ls, dls);
        if (st == 0)
            st = ce_weighted(ft.z[L - 1], nt, C, y + ns, w ? w + ns : NULL, denoms[1], 1.0, &lt,
                             dlt);
        if (st == 0) {
            loss = ls + lt;
            branch_backward(L, dims, frozen_layers, (const double* const*)W, W[L], &ft, nt, dlt,
                            NULL, gW, gb, gW[L], gb[L]);
            branch_backward(L, dims, frozen_layers, (const double* const*)W, W[L - 1], &fs, ns,
                            dls, NULL, gW, gb, gW[L - 1], gb[L - 1]);
        }
        free(dls);
        free(dlt);
        branch_free(L, &fs);
        branch_free(L, &ft);
    }
    if (st == 0) {
        /* sink: Parameter::grad.add_(node grad) onto zeroed grads (tape.hpp:882-885),
         * then optimizer_step SGD (optim.hpp:46-48) on trainable params */
        for (int i = 0; i < n_mats; ++i) {
            const int l = i < L ? i : L - 1;
            if (l < frozen_layers) continue;
            const size_t nw = (size_t)dims[l] * (size_t)dims[l + 1], nb = (size_t)dims[l + 1];
            for (size_t j = 0; j < nw; ++j) gW[i][j] = 0.0 + gW[i][j];
            for (size_t j = 0; j < nb; ++j) gb[i][j] = 0.0 + gb[i][j];
            if (dW_out && dW_out[i]) memcpy(dW_out[i], gW[i], sizeof(double) * nw);
            if (db_out && db_out[i]) memcpy(db_out[i], gb[i], sizeof(double) * nb);
            for (size_t j = 0; j < nw; ++j) W[i][j] -= lr * gW[i][j];
            for (size_t j = 0; j < nb; ++j) b[i][j] -= lr * gb[i][j];
            if (!all_finite(W[i], nw) || !all_finite(b[i], nb)) st = 5; /* optim.hpp:65-66 */
        }
        if (loss_out) *loss_out = loss;
    }
    for (int i = 0; i < n_mats; ++i) {
        free(gW[i]);
        free(gb[i]);
    }
    free(gW);
    free(gb);
    return st;
}

void orc_mlp_init(orc_rng* r, int n_mats, const int* fan_in, const int* fan_out, double* const* W,
                  double* const* b) {
    for (int i = 0; i < n_mats; ++i) {
        const double lim = 1.0 / sqrt((double)fan_in[i]);
        orc_rng_fill_uniform_range(r, W[i], (size_t)fan_in[i] * (size_t)fan_out[i], -lim, lim);
        memset(b[i], 0, sizeof(double) * (size_t)fan_out[i]);
    }
}

/* ======================================================================= */
/* Multi-bandwidth Gaussian MMD (no reference code)  */
/* ======================================================================= */
double orc_mmd_beta(const double* Xs, size_t m, const double* Xt, size_t n, size_t d) {
    const size_t N = m + n;
    double s2 = 0.0;
    double* s = (double*)calloc(d, sizeof(double));
    for (size_t i = 0; i < N; ++i) {
        const double* z = i < m ? Xs + i * d : Xt + (i - m) * d;
        for (size_t k = 0; k < d; ++k) {
            s2 += z[k] * z[k];
            s[k] += z[k];
        }
    }
    double ss = 0.0;
    for (size_t k = 0; k < d; ++k) ss += s[k] * s[k];
    free(s);
    const double Nd = (double)N;
    return (2.0 * Nd * s2 - 2.0 * ss) / (Nd * Nd - Nd);
}

int orc_mmd_gaussian(const double* Xs, size_t m, const double* Xt, size_t n, size_t d,
                     const double* mult, int nb, double beta_in, double* value, double* beta_out,
                     double* gXs, double* gXt) {
    if (m == 0 || n == 0 || d == 0 || nb <= 0 || nb > 16) return 1;
    const double beta = beta_in > 0.0 ? beta_in : orc_mmd_beta(Xs, m, Xt, n, d);
    if (!(beta > 0.0) || !isfinite(beta)) return 2;
    if (beta_out) *beta_out = beta;
    double inv_s[16];
    for (int q = 0; q < nb; ++q) inv_s[q] = 1.0 / (beta * mult[q]);
    const size_t N = m + n;
    const double cSS = 1.0 / ((double)m * (double)m), cTT = 1.0 / ((double)n * (double)n),
                 cST = -2.0 / ((double)m * (double)n);
    double sum_ss = 0.0, sum_tt = 0.0, sum_st = 0.0;
    for (size_t i = 0; i < N; ++i) {
        const int di = i >= m;
        const double* zi = di ? Xt + (i - m) * d : Xs + i * d;
        double* gi = di ? (gXt ? gXt + (i - m) * d : NULL) : (gXs ? gXs + i * d : NULL);
        if (gi) memset(gi, 0, sizeof(double) * d);
        for (size_t j = 0; j < N; ++j) {
            const int dj = j >= m;
            const double* zj = dj ? Xt + (j - m) * d : Xs + j * d;
            double d2 = 0.0;
            for (size_t k = 0; k < d; ++k) {
                const double t = zi[k] - zj[k];
                d2 += t * t;
            }
            double kv = 0.0, A = 0.0;
            for (int q = 0; q < nb; ++q) {
                const double e = exp(-d2 * inv_s[q]);
                kv += e;
                A += 2.0 * inv_s[q] * e;
            }
            double c;
            if (!di && !dj) {
                sum_ss += kv;
                c = -2.0 * cSS;
            } else if (di && dj) {
                sum_tt += kv;
                c = -2.0 * cTT;
            } else {
                if (!di) sum_st += kv;
                c = -cST; /* 2/(mn) */
            }
            if (gi && i != j) {
                const double f = c * A;
                for (size_t k = 0; k < d; ++k) gi[k] += f * (zi[k] - zj[k]);
            }
        }
    }
    *value = cSS * sum_ss + cTT * sum_tt + cST * sum_st;
    return isfinite(*value) ? 0 : 5;
}

/* ======================================================================= */
/* Attack stage                                                            */
/* ======================================================================= */
void orc_softmax(const double* logits, size_t rows, int C, double* probs) {
    const size_t n = (size_t)C;
    for (size_t r = 0; r < rows; ++r) {
        const double* x = logits + r * n;
        double* row = probs + r * n;
        double mx = x[0];
        for (size_t j = 1; j < n; ++j) mx = x[j] > mx ? x[j] : mx;
        double z = 0.0;
        for (size_t j = 0; j < n; ++j) {
            row[j] = exp(x[j] - mx);
            z += row[j];
        }
        const double inv = 1.0 / z;
        for (size_t j = 0; j < n; ++j) row[j] *= inv;
    }
}

int orc_posterior_features(const double* logits, size_t rows, int C, int k, const int32_t* labels,
                           double* feats) {
    if (k < 1 || k > C || C > 64) return 1;
    const size_t nf = (size_t)k + (labels ? 1 : 0);
    double p[64];
    for (size_t r = 0; r < rows; ++r) {
        orc_softmax(logits + r * (size_t)C, 1, C, p);
        double* out = feats + r * nf;
        /* partial selection sort, descending */
        for (int a = 0; a < k; ++a) {
            int best = a;
            for (int j = a + 1; j < C; ++j)
                if (p[j] > p[best]) best = j;
            double t = p[a];
            p[a] = p[best];
            p[best] = t;
            out[a] = p[a];
        }
        if (labels) {
            const double* x = logits + r * (size_t)C;
            if (labels[r] < 0 || labels[r] >= C) return 2;
            double mx = x[0];
            for (int j = 1; j < C; ++j) mx = x[j] > mx ? x[j] : mx;
            double z = 0.0;
            for (int j = 0; j < C; ++j) z += exp(x[j] - mx);
            out[k] = mx + log(z) - x[labels[r]];
        }
    }
    return 0;
}

typedef struct {
    double s;
    uint8_t l;
} scored;

static int cmp_scored(const void* a, const void* b) {
    const double x = ((const scored*)a)->s, y = ((const scored*)b)->s;
    return (x > y) - (x < y);
}

int orc_auc(const double* scores, const uint8_t* labels, size_t n, double* auc) {
    if (n == 0) return 1;
    scored* v = (scored*)malloc(sizeof(scored) * n);
    size_t npos = 0;
    for (size_t i = 0; i < n; ++i) {
        v[i].s = scores[i];
        v[i].l = labels[i] ? 1 : 0;
        npos += v[i].l;
    }
    const size_t nneg = n - npos;
    if (npos == 0 || nneg == 0) {
        free(v);
        return 2;
    }
    qsort(v, n, sizeof(scored), cmp_scored);
    double rank_sum = 0.0;
    size_t i = 0;
    while (i < n) {
        size_t j = i;
        size_t pos_in_group = 0;
        while (j < n && v[j].s == v[i].s) pos_in_group += v[j++].l;
        /* ranks i+1 .. j, mid-rank (i+1+j)/2 */
        rank_sum += (double)pos_in_group * 0.5 * ((double)(i + 1) + (double)j);
        i = j;
    }
    free(v);
    const double np = (double)npos, nn = (double)nneg;
    *auc = (rank_sum - np * (np + 1.0) * 0.5) / (np * nn);
    return 0;
}

double orc_accuracy(const double* scores, const uint8_t* labels, size_t n, double threshold) {
    size_t ok = 0;
    for (size_t i = 0; i < n; ++i) ok += ((scores[i] > threshold) == (labels[i] != 0));
    return n ? (double)ok / (double)n : 0.0;
}

void orc_synth(orc_rng* r, int C, int d, size_t n, const double* mu, const double* shift,
               double* X, int32_t* y) {
    for (size_t i = 0; i < n; ++i) {
        const int c = (int)orc_rng_below(r, (uint64_t)C);
        y[i] = c;
        double* x = X + i * (size_t)d;
        const double* m = mu + (size_t)c * (size_t)d;
        for (int k = 0; k < d; ++k) {
            double v = m[k] + orc_rng_normal(r);
            if (shift) v = v + shift[k];
            x[k] = v;
        }
    }
}

/* ======================================================================= */
/* Counter-based generator -- see oracle.h             */
/* ======================================================================= */
static uint64_t mulhilo64(uint64_t a, uint64_t b, uint64_t* hi) {
    const unsigned __int128 p = (unsigned __int128)a * b;
    *hi = (uint64_t)(p >> 64);
    return (uint64_t)p;
}

void orc_philox4x64(const uint64_t ctr[4], const uint64_t key[2], uint64_t out[4]) {
    uint64_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint64_t k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; ++r) {
        uint64_t hi0, hi1;
        const uint64_t lo0 = mulhilo64(0xD2E7470EE14C6C93ULL, c0, &hi0);
        const uint64_t lo1 = mulhilo64(0xCA5A826395121157ULL, c2, &hi1);
        const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
        k0 += 0x9E3779B97F4A7C15ULL;
        k1 += 0xBB67AE8584CAA73BULL;
    }
    out[0] = c0;
    out[1] = c1;
    out[2] = c2;
    out[3] = c3;
}

static void box_muller(uint64_t wa, uint64_t wb, double* za, double* zb) {
    const double u1 = (double)((wa >> 40) + 1) * 0x1p-24;
    const double u2 = (double)(wb >> 40) * 0x1p-24;
    const double r = sqrt(-2.0 * log(u1));
    const double t = 2.0 * 3.14159265358979323846 * u2;
    *za = r * cos(t);
    *zb = r * sin(t);
}

void orc_counter_normals(uint64_t seed, uint64_t stream, size_t first, size_t count, double* z) {
    const uint64_t key[2] = {seed, stream};
    for (size_t e = first; e < first + count;) {
        const uint64_t ctr[4] = {(uint64_t)(e / 4), 0, 0, 0};
        uint64_t w[4];
        double v[4];
        orc_philox4x64(ctr, key, w);
        box_muller(w[0], w[1], &v[0], &v[1]);
        box_muller(w[2], w[3], &v[2], &v[3]);
        for (size_t j = e % 4; j < 4 && e < first + count; ++j, ++e) z[e - first] = v[j];
    }
}

void orc_synth_counter(uint64_t seed, uint64_t stream, int C, int d, size_t n, const double* mu,
                       const double* shift, double* X, int32_t* y) {
    const uint64_t key[2] = {seed, stream};
    for (size_t i = 0; i < n; ++i) {
        const uint64_t ctr[4] = {(uint64_t)(i / 4), 1, 0, 0};
        uint64_t w[4], hi;
        orc_philox4x64(ctr, key, w);
        (void)mulhilo64(w[i % 4], (uint64_t)C, &hi);
        y[i] = (int32_t)hi;
    }
    orc_counter_normals(seed, stream, 0, n * (size_t)d, X);
    for (size_t i = 0; i < n; ++i) {
        const double* m = mu + (size_t)y[i] * (size_t)d;
        double* x = X + i * (size_t)d;
        for (int k = 0; k < d; ++k) {
            double v = m[k] + x[k];
            if (shift) v = v + shift[k];
            x[k] = v;
        }
    }
}
