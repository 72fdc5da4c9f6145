// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Thin extern "C" shim over the UNMODIFIED reference headers in
// /root/reference/proj/include/minitransfer (included, never copied).  It is
// compiled by oracle/Makefile into oracle/_ref/libmtref.so and used by the
// tests to pin the C restatement in oracle.c, to mint golden fixtures, and by
// bench.py --impl reference as the reference CPU arm.  The reference has no
// MMD, so the MMD gradient is injected into the reference Tape with
// sum(mul(h, constant(G))) (tape.hpp:153-171, 406-416), G coming from the C
// restatement orc_mmd_gaussian (oracle.c).
#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#ifndef MTREF_FLAGS
#define MTREF_FLAGS "(flags not recorded)"
#endif

#include "minitransfer/optim.hpp"
#include "minitransfer/rng.hpp"
#include "minitransfer/tape.hpp"
#include "minitransfer/tensor.hpp"

extern "C" {
#include "oracle.h"
}

namespace {

thread_local std::string g_err;

int status_of(const std::exception& e) {
    if (dynamic_cast<const mt::ShapeError*>(&e)) return 1;
    if (dynamic_cast<const mt::ValueError*>(&e)) return 2;
    if (dynamic_cast<const mt::ConfigError*>(&e)) return 3;
    if (dynamic_cast<const mt::DataError*>(&e)) return 4;
    return 5;
}

mt::Tensor mat(const double* p, std::size_t r, std::size_t c) {
    return mt::Tensor({r, c}, std::vector<double>(p, p + r * c));
}

struct Net {
    int L;
    std::vector<int> dims;
    int n_heads;
    std::vector<mt::Parameter> W, b;  // L + n_heads - 1 entries
};

Net make_net(int L, const int* dims, int n_heads, double* const* W, double* const* b) {
    Net n{L, std::vector<int>(dims, dims + L + 1), n_heads, {}, {}};
    const int n_mats = L + n_heads - 1;
    for (int i = 0; i < n_mats; ++i) {
        const int l = i < L ? i : L - 1;
        const std::size_t k = dims[l], o = dims[l + 1];
        n.W.emplace_back("W" + std::to_string(i), mat(W[i], k, o));
        n.b.emplace_back("b" + std::to_string(i),
                         mt::Tensor({o}, std::vector<double>(b[i], b[i] + o)));
    }
    return n;
}

// matmul -> add_bias -> relu chain; the head index picks W[L-1] or W[L].
mt::Var chain(mt::Tape& t, const Net& n, const std::vector<mt::Var>& pw,
              const std::vector<mt::Var>& pb, mt::Var x, int head, mt::Var* h_last) {
    mt::Var h = x;
    for (int l = 0; l < n.L; ++l) {
        const int i = (l == n.L - 1) ? l + head : l;
        mt::Var z = t.add_bias(t.matmul(h, pw[i]), pb[i]);
        if (l == n.L - 1) {
            if (h_last) *h_last = h;
            return z;
        }
        h = t.relu(z);
    }
    return h;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// ---- mt::Rng (rng.hpp) ----------------------------------------------------
void* ref_rng_create(uint64_t seed) { return new mt::Rng(seed); }
void ref_rng_destroy(void* r) { delete static_cast<mt::Rng*>(r); }
uint64_t ref_rng_next(void* r) { return static_cast<mt::Rng*>(r)->next_u64(); }
double ref_rng_uniform(void* r) { return static_cast<mt::Rng*>(r)->uniform(); }
double ref_rng_uniform_range(void* r, double lo, double hi) {
    return static_cast<mt::Rng*>(r)->uniform(lo, hi);
}
double ref_rng_normal(void* r) { return static_cast<mt::Rng*>(r)->normal(); }
uint64_t ref_rng_below(void* r, uint64_t n) { return static_cast<mt::Rng*>(r)->below(n); }
void ref_rng_permutation(void* r, std::size_t n, uint64_t* out) {
    auto p = static_cast<mt::Rng*>(r)->permutation(n);
    for (std::size_t i = 0; i < n; ++i) out[i] = p[i];
}
void* ref_rng_split(void* r, uint64_t stream) {
    return new mt::Rng(static_cast<mt::Rng*>(r)->split(stream));
}

// ---- Adam through mt::optimizer_step (optim.hpp:30-68) ---------------------
// `steps` consecutive updates of one parameter with the given gradients
// (g_seq [steps][n]); the OptimizerState persists across them.
int ref_adam_sequence(double* w, const double* g_seq, size_t n, int steps, double lr, double beta1,
                      double beta2, double eps) {
    try {
        mt::Parameter p("p", mt::Tensor({n}, std::vector<double>(w, w + n)));
        mt::OptimizerState st = mt::OptimizerState::adam(lr);
        st.beta1 = beta1;
        st.beta2 = beta2;
        st.epsilon = eps;
        std::vector<mt::Parameter*> ps{&p};
        for (int s = 0; s < steps; ++s) {
            for (size_t i = 0; i < n; ++i) p.grad[i] = g_seq[(size_t)s * n + i];
            mt::optimizer_step(st, ps);
        }
        for (size_t i = 0; i < n; ++i) w[i] = p.value[i];
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 5;
    }
}

// ---- Tape MLP step: the reference composition of the path ----------------
// Same argument meaning as orc_mlp_train_step (oracle.h).
int ref_mlp_train_step(int L, const int* dims, int n_heads, int frozen, double* const* W,
                       double* const* b, const double* X, int B, int src_rows, const int32_t* y,
                       const double* w, const double* denoms, double lr, const double* dH_inject,
                       double* loss_out, double* const* dW_out, double* const* db_out) {
    try {
        Net n = make_net(L, dims, n_heads, W, b);
        const int n_mats = L + n_heads - 1;
        std::vector<mt::Parameter*> trainable;
        for (int i = 0; i < n_mats; ++i) {
            const int l = i < L ? i : L - 1;
            if (l >= frozen) {
                trainable.push_back(&n.W[i]);
                trainable.push_back(&n.b[i]);
            }
        }
        mt::zero_grads(trainable);
        double loss_val = 0.0;
        {
            mt::Tape t;
            std::vector<mt::Var> pw, pb;
            for (int i = 0; i < n_mats; ++i) {
                const int l = i < L ? i : L - 1;
                if (l >= frozen) {
                    pw.push_back(t.param(n.W[i]));
                    pb.push_back(t.param(n.b[i]));
                } else {
                    pw.push_back(t.constant(n.W[i].value));
                    pb.push_back(t.constant(n.b[i].value));
                }
            }
            const std::size_t d0 = dims[0];
            std::vector<int> labels(y, y + B);
            std::vector<double> wts(B, 1.0);
            if (w) wts.assign(w, w + B);
            if (n_heads == 1) {
                mt::Var x = t.constant(mat(X, B, d0));
                mt::Var h_last;
                mt::Var logits = chain(t, n, pw, pb, x, 0, &h_last);
                mt::Var loss = t.cross_entropy_weighted(logits, labels, wts, denoms[0]);
                loss_val = t.value(loss).item();
                if (dH_inject) {
                    const std::size_t hd = dims[L - 1];
                    mt::Var g = t.constant(mat(dH_inject, B, hd));
                    loss = t.add(loss, t.sum(t.mul(h_last, g)));
                }
                t.backward(loss);
            } else {
                const std::size_t ns = src_rows, nt = B - src_rows;
                mt::Var xs = t.constant(mat(X, ns, d0));
                mt::Var xt = t.constant(mat(X + ns * d0, nt, d0));
                mt::Var ls = chain(t, n, pw, pb, xs, 0, nullptr);
                mt::Var lt = chain(t, n, pw, pb, xt, 1, nullptr);
                std::vector<int> ys(labels.begin(), labels.begin() + ns),
                    yt(labels.begin() + ns, labels.end());
                std::vector<double> ws(wts.begin(), wts.begin() + ns),
                    wt(wts.begin() + ns, wts.end());
                mt::Var cs = t.cross_entropy_weighted(ls, ys, ws, denoms[0]);
                mt::Var ct = t.cross_entropy_weighted(lt, yt, wt, denoms[1]);
                mt::Var loss = t.add(cs, ct);
                loss_val = t.value(loss).item();
                t.backward(loss);
            }
        }
        mt::OptimizerState st = mt::OptimizerState::sgd(lr);
        int k = 0;
        for (int i = 0; i < n_mats; ++i) {
            const int l = i < L ? i : L - 1;
            if (l < frozen) continue;
            if (dW_out && dW_out[i])
                std::memcpy(dW_out[i], n.W[i].grad.data(), sizeof(double) * n.W[i].grad.size());
            if (db_out && db_out[i])
                std::memcpy(db_out[i], n.b[i].grad.data(), sizeof(double) * n.b[i].grad.size());
            ++k;
        }
        mt::optimizer_step(st, trainable);
        for (int i = 0; i < n_mats; ++i) {
            std::memcpy(W[i], n.W[i].value.data(), sizeof(double) * n.W[i].value.size());
            std::memcpy(b[i], n.b[i].value.data(), sizeof(double) * n.b[i].value.size());
        }
        if (loss_out) *loss_out = loss_val;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return status_of(e);
    }
}

int ref_mlp_forward(int L, const int* dims, int head, double* const* W, double* const* b,
                    const double* X, int B, double* logits, double* hidden_last) {
    try {
        Net n = make_net(L, dims, head ? 2 : 1, W, b);
        mt::Tape t;
        std::vector<mt::Var> pw, pb;
        for (std::size_t i = 0; i < n.W.size(); ++i) {
            pw.push_back(t.param(n.W[i]));
            pb.push_back(t.param(n.b[i]));
        }
        mt::Var x = t.constant(mat(X, B, dims[0]));
        mt::Var h_last;
        mt::Var z = chain(t, n, pw, pb, x, head, &h_last);
        std::memcpy(logits, t.value(z).data(), sizeof(double) * t.value(z).size());
        if (hidden_last && L > 1)
            std::memcpy(hidden_last, t.value(h_last).data(),
                        sizeof(double) * t.value(h_last).size());
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return status_of(e);
    }
}

int ref_softmax(const double* logits, std::size_t rows, int C, double* probs) {
    try {
        mt::Tape t;
        mt::Var p = t.softmax(t.constant(mat(logits, rows, C)));
        std::memcpy(probs, t.value(p).data(), sizeof(double) * rows * C);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return status_of(e);
    }
}

// grad_check (optim.hpp:81-117) of loss = lam * MMD(h(Xs), h(Xt)) for a
// one-layer tanh encoder h = tanh(X W + b), with beta frozen (detached).  The
// loss value is MMD itself via add_scalar; the gradient is the injected G.
double ref_grad_check_mmd(int d_in, int d_h, const double* Xs, int m, const double* Xt, int n,
                          const double* W0, const double* b0, const double* mult, int nb,
                          double lam, double beta) {
    mt::Parameter W("W", mat(W0, d_in, d_h));
    mt::Parameter b("b", mt::Tensor({(std::size_t)d_h}, std::vector<double>(b0, b0 + d_h)));
    auto build = [&](mt::Tape& t) {
        mt::Var w = t.param(W), bb = t.param(b);
        mt::Var hs = t.tanh(t.add_bias(t.matmul(t.constant(mat(Xs, m, d_in)), w), bb));
        mt::Var ht = t.tanh(t.add_bias(t.matmul(t.constant(mat(Xt, n, d_in)), w), bb));
        const mt::Tensor& Hs = t.value(hs);
        const mt::Tensor& Ht = t.value(ht);
        std::vector<double> gs((std::size_t)m * d_h), gt((std::size_t)n * d_h);
        double v = 0.0;
        orc_mmd_gaussian(Hs.data(), m, Ht.data(), n, d_h, mult, nb, beta, &v, nullptr, gs.data(),
                         gt.data());
        for (double& g : gs) g *= lam;
        for (double& g : gt) g *= lam;
        mt::Var inj = t.add(t.sum(t.mul(hs, t.constant(mt::Tensor({(std::size_t)m, (std::size_t)d_h}, gs)))),
                            t.sum(t.mul(ht, t.constant(mt::Tensor({(std::size_t)n, (std::size_t)d_h}, gt)))));
        return t.add_scalar(inj, lam * v - t.value(inj).item());
    };
    return mt::grad_check(build, {&W, &b}, 1e-5);
}

// ======================================================================
// CPU baseline arms (bench.py cpu_baseline / --impl reference).
//
// Every arm is built from the reference's own code: the Tape ops, backward
// and optimizer_step for the models (one Tape per model per step, one model
// per std::thread: tape.hpp:84-85) and the Tape's own matmul
// primitives detail::mm_acc / mm_tn_acc (tape.hpp:36-48, 65-78) for the MMD
// Gram and gradient products.  The reference has no MMD: it is restated out
// of the Tape over UNIQUE pairs (each unordered pair's exp once, the kernel
// matrix symmetric) and injected into the SAME Tape with
// sum(mul(h, constant(G))) (tape.hpp:153-171, 406-416), as SURVEY.md 8(c)
// prescribes.  Model init and data generation happen before the timed region.
// ======================================================================

// Raw unique-pair MMD partials of the joint sample Z [N][d] (rows [0, m) the
// source): tile pairs (I, J >= I) with I over [ilo, ihi) (tile-aligned).
// sums[0..2] += kernel sums over unordered pairs i < j (ss, tt, st); the
// gradient pair terms f_ij (z_i - z_j) go to gI[i] and f_ij (z_j - z_i) to
// gJ[j] (absolute row indices, stride d; the same buffer or two), caller-zeroed.
struct MmdTileWork {
    std::vector<double> ZJt, S, F, tmp;
};
static void mmd_tile_pair(const double* Z, const double* norms, size_t N, size_t m, size_t d,
                          const double* inv_s, int nb, const double coef[3], size_t a0, size_t a1,
                          size_t b0, size_t b1, double* gI, double* gJ, double sums[3],
                          MmdTileWork& w) {
    const size_t nI = a1 - a0, nJ = b1 - b0;
    w.ZJt.assign(d * nJ, 0.0);
    for (size_t j = 0; j < nJ; ++j)
        for (size_t k = 0; k < d; ++k) w.ZJt[k * nJ + j] = Z[(b0 + j) * d + k];
    w.S.assign(nI * nJ, 0.0);
    mt::detail::mm_acc(Z + a0 * d, w.ZJt.data(), w.S.data(), nI, d, nJ);  // Z_I Z_J^T
    w.F.assign(nI * nJ, 0.0);
    std::vector<double> rs(nI, 0.0), cs(nJ, 0.0);
    for (size_t i = 0; i < nI; ++i) {
        const size_t gi = a0 + i;
        const bool si = gi < m;
        for (size_t j = 0; j < nJ; ++j) {
            const size_t gj = b0 + j;
            if (gj <= gi) continue;  // unordered pairs i < j only
            double d2 = norms[gi] + norms[gj] - 2.0 * w.S[i * nJ + j];
            if (d2 < 0.0) d2 = 0.0;
            double kv = 0.0, A = 0.0;
            for (int q = 0; q < nb; ++q) {
                const double e = std::exp(-d2 * inv_s[q]);
                kv += e;
                A += 2.0 * inv_s[q] * e;
            }
            const bool sj = gj < m;
            const int cls = (si && sj) ? 0 : (!si && !sj) ? 1 : 2;
            sums[cls] += kv;
            const double f = coef[cls] * A;
            w.F[i * nJ + j] = f;
            rs[i] += f;
            cs[j] += f;
        }
    }
    // g_i += f_ij (z_i - z_j), g_j += f_ij (z_j - z_i)
    w.tmp.assign(nI * d, 0.0);
    mt::detail::mm_acc(w.F.data(), Z + b0 * d, w.tmp.data(), nI, nJ, d);  // F Z_J
    for (size_t i = 0; i < nI; ++i)
        for (size_t k = 0; k < d; ++k)
            gI[(a0 + i) * d + k] += rs[i] * Z[(a0 + i) * d + k] - w.tmp[i * d + k];
    w.tmp.assign(nJ * d, 0.0);
    mt::detail::mm_tn_acc(w.F.data(), Z + a0 * d, w.tmp.data(), nI, nJ, d);  // F^T Z_I
    for (size_t j = 0; j < nJ; ++j)
        for (size_t k = 0; k < d; ++k)
            gJ[(b0 + j) * d + k] += cs[j] * Z[(b0 + j) * d + k] - w.tmp[j * d + k];
}

// detached beta (SURVEY.md Appendix A closed form) and the pair coefficients
static void mmd_setup(const double* Z, size_t N, size_t m, size_t d, const double* mult, int nb,
                      std::vector<double>& norms, double* inv_s, double coef[3], double* beta_out) {
    norms.assign(N, 0.0);
    std::vector<double> col(d, 0.0);
    double sn = 0.0;
    for (size_t i = 0; i < N; ++i) {
        double s = 0.0;
        for (size_t k = 0; k < d; ++k) {
            s += Z[i * d + k] * Z[i * d + k];
            col[k] += Z[i * d + k];
        }
        norms[i] = s;
        sn += s;
    }
    double c2 = 0.0;
    for (size_t k = 0; k < d; ++k) c2 += col[k] * col[k];
    const double Nd = (double)N;
    const double beta = (2.0 * Nd * sn - 2.0 * c2) / (Nd * Nd - Nd);
    for (int q = 0; q < nb; ++q) inv_s[q] = 1.0 / (beta * mult[q]);
    const double n = (double)(N - m), mm = (double)m;
    coef[0] = -2.0 / (mm * mm);  // -2 cSS
    coef[1] = -2.0 / (n * n);    // -2 cTT
    coef[2] = 2.0 / (mm * n);    // -cST
    if (beta_out) *beta_out = beta;
}

constexpr size_t kMmdTile = 128;

// Full MMD^2 + gradient of one joint sample, single thread (a C2 model step).
static double mmd_full(const double* Z, size_t N, size_t m, size_t d, const double* mult, int nb,
                       double* g /* [N][d], overwritten */) {
    std::vector<double> norms;
    double inv_s[16], coef[3];
    mmd_setup(Z, N, m, d, mult, nb, norms, inv_s, coef, nullptr);
    std::fill(g, g + N * d, 0.0);
    double sums[3] = {0.0, 0.0, 0.0};
    MmdTileWork w;
    for (size_t a0 = 0; a0 < N; a0 += kMmdTile)
        for (size_t b0 = a0; b0 < N; b0 += kMmdTile)
            mmd_tile_pair(Z, norms.data(), N, m, d, inv_s, nb, coef, a0, std::min(N, a0 + kMmdTile), b0,
                          std::min(N, b0 + kMmdTile), g, g, sums, w);
    const double n = (double)(N - m), mm = (double)m;
    // V-statistic: ordered double sums = 2 x unordered + the nb-valued diagonal
    return (2.0 * sums[0] + mm * nb) / (mm * mm) + (2.0 * sums[1] + n * nb) / (n * n) -
           2.0 * sums[2] / (mm * n);
}

namespace {
struct Barrier {  // one-shot start line for the timed region
    std::mutex mu;
    std::condition_variable cv;
    int waiting = 0, total;
    explicit Barrier(int n) : total(n) {}
    void arrive_and_wait() {
        std::unique_lock<std::mutex> lk(mu);
        if (++waiting == total) cv.notify_all();
        else cv.wait(lk, [&] { return waiting >= total; });
    }
};
using Clock = std::chrono::steady_clock;
}  // namespace

// CPU C2/C1 arm: `threads` independent models, one per std::thread, each
// running `steps` SGD steps (lr 0.05) of dims on its own fixed synthetic
// batch of B rows; mmd_lambda > 0 adds lambda * MMD^2(h_src, h_tgt) on the
// last hidden layer, injected into the step's own Tape.  Init + data before
// the timed region; returns the seconds from the common start line until the
// last thread finishes its steps.
double ref_bench_train_heads(int threads, int L, const int* dims, int n_heads, int B, int src_rows,
                             int steps, double mmd_lambda, uint64_t seed);
double ref_bench_train(int threads, int L, const int* dims, int B, int src_rows, int steps,
                       double mmd_lambda, uint64_t seed) {
    return ref_bench_train_heads(threads, L, dims, 1, B, src_rows, steps, mmd_lambda, seed);
}

// n_heads == 2: the parameter-based paradigm (shared trunk, a source head and
// a target head; rows [0, src_rows) through head 0, the rest through head 1,
// CE of each head over its own rows)
double ref_bench_train_heads(int threads, int L, const int* dims, int n_heads, int B, int src_rows,
                             int steps, double mmd_lambda, uint64_t seed) {
    Barrier start(threads + 1);
    std::vector<std::thread> pool;
    std::vector<Clock::time_point> done(threads);
    for (int th = 0; th < threads; ++th) {
        pool.emplace_back([=, &start, &done]() {
            mt::Rng rng(seed + th);
            std::vector<mt::Parameter> W, b;
            for (int i = 0; i < L + n_heads - 1; ++i) {
                const int l = i < L ? i : L - 1;
                const double lim = 1.0 / std::sqrt((double)dims[l]);
                std::vector<double> w((std::size_t)dims[l] * dims[l + 1]);
                for (double& v : w) v = rng.uniform(-lim, lim);
                W.emplace_back("W" + std::to_string(i), mt::Tensor({(std::size_t)dims[l], (std::size_t)dims[l + 1]}, w));
                b.emplace_back("b" + std::to_string(i),
                               mt::Tensor({(std::size_t)dims[l + 1]}, std::vector<double>(dims[l + 1], 0.0)));
            }
            std::vector<mt::Parameter*> params;
            for (std::size_t i = 0; i < W.size(); ++i) {
                params.push_back(&W[i]);
                params.push_back(&b[i]);
            }
            std::vector<double> X((std::size_t)B * dims[0]);
            for (double& v : X) v = rng.normal();
            std::vector<int> y(B);
            for (auto& v : y) v = (int)rng.below(dims[L]);
            const std::vector<double> wts(B, 1.0);
            const mt::Tensor Xt({(std::size_t)B, (std::size_t)dims[0]}, X);
            const std::size_t ns = src_rows, nt = B - src_rows;
            const mt::Tensor Xs2({ns ? ns : 1, (std::size_t)dims[0]},
                                 std::vector<double>(X.begin(), X.begin() + (ns ? ns : 1) * dims[0]));
            const mt::Tensor Xt2({nt ? nt : 1, (std::size_t)dims[0]},
                                 std::vector<double>(X.begin() + ns * dims[0],
                                                     X.begin() + (ns + (nt ? nt : 1)) * dims[0]));
            const std::vector<int> ys(y.begin(), y.begin() + ns), yt(y.begin() + ns, y.end());
            const std::vector<double> ws(ns, 1.0), wt2(nt, 1.0);
            const std::size_t hd = dims[L - 1];
            std::vector<double> G((std::size_t)B * hd);
            const double mult[5] = {0.25, 0.5, 1.0, 2.0, 4.0};
            mt::OptimizerState st = mt::OptimizerState::sgd(0.05);
            start.arrive_and_wait();
            for (int s = 0; s < steps; ++s) {
                mt::zero_grads(params);
                mt::Tape t;
                std::vector<mt::Var> pw, pb;
                for (std::size_t i = 0; i < W.size(); ++i) {
                    pw.push_back(t.param(W[i]));
                    pb.push_back(t.param(b[i]));
                }
                if (n_heads == 2) {  // parameter-based: two heads over the shared trunk
                    auto run = [&](const mt::Tensor& x, int head) {
                        mt::Var h = t.constant(x);
                        for (int l = 0; l < L; ++l) {
                            const int i = (l == L - 1) ? l + head : l;
                            mt::Var z = t.add_bias(t.matmul(h, pw[i]), pb[i]);
                            h = (l == L - 1) ? z : t.relu(z);
                        }
                        return h;
                    };
                    mt::Var loss = t.add(t.cross_entropy_weighted(run(Xs2, 0), ys, ws, (double)ns),
                                         t.cross_entropy_weighted(run(Xt2, 1), yt, wt2, (double)nt));
                    t.backward(loss);
                    mt::optimizer_step(st, params);
                    continue;
                }
                mt::Var h = t.constant(Xt), h_last = h;
                for (int l = 0; l < L; ++l) {
                    mt::Var z = t.add_bias(t.matmul(h, pw[l]), pb[l]);
                    if (l == L - 1) {
                        h_last = h;
                        h = z;
                    } else {
                        h = t.relu(z);
                    }
                }
                mt::Var loss = t.cross_entropy_weighted(h, y, wts, (double)B);
                if (mmd_lambda > 0.0) {
                    mmd_full(t.value(h_last).data(), B, src_rows, hd, mult, 5, G.data());
                    for (double& v : G) v *= mmd_lambda;
                    loss = t.add(loss, t.sum(t.mul(h_last, t.constant(mt::Tensor({(std::size_t)B, hd}, G)))));
                }
                t.backward(loss);
                mt::optimizer_step(st, params);
            }
            done[th] = Clock::now();
        });
    }
    start.arrive_and_wait();
    const auto t0 = Clock::now();
    for (auto& t : pool) t.join();
    Clock::time_point t1 = t0;
    for (auto& d : done) t1 = std::max(t1, d);
    return std::chrono::duration<double>(t1 - t0).count();
}

// CPU C4 arm: the joint sample Z = [Xs; Xt] (Xs ~ N(0, I), Xt ~ N(0.1, I),
// f64, drawn before the timed region) and the unordered pairs whose smaller
// index lies in the first `slice_rows` source rows (a bounded slice of the
// full evaluation): value partials + gradient over those pairs, threads over
// J tiles (each thread owns its J rows' gradient; the slice rows' gradient is
// per thread, summed in thread order at the end).  *pairs_out = the slice's
// unique pair count.  Returns the timed seconds.
double ref_bench_mmd(int threads, int64_t m, int64_t n, int d, int64_t slice_rows, uint64_t seed,
                     double* pairs_out, double* sums_out) {
    const size_t N = (size_t)(m + n), D = (size_t)d;
    std::vector<double> Z(N * D);
    {
        std::vector<std::thread> gen;
        const size_t per = (N + threads - 1) / threads;
        for (int th = 0; th < threads; ++th)
            gen.emplace_back([&, th]() {
                mt::Rng r(seed + 1000 + th);
                for (size_t i = th * per; i < std::min(N, (th + 1) * per); ++i)
                    for (size_t k = 0; k < D; ++k) Z[i * D + k] = r.normal() + (i >= (size_t)m ? 0.1 : 0.0);
            });
        for (auto& t : gen) t.join();
    }
    const size_t S = (size_t)slice_rows;
    const double mult[5] = {0.25, 0.5, 1.0, 2.0, 4.0};
    std::vector<double> norms;
    double inv_s[16], coef[3];
    std::vector<double> g(N * D, 0.0);
    std::vector<std::vector<double>> gslice(threads, std::vector<double>(S * D, 0.0));
    std::vector<std::array<double, 3>> sums(threads, std::array<double, 3>{0.0, 0.0, 0.0});
    Barrier start(threads + 1);
    std::vector<std::thread> pool;
    const size_t nJ = (N + kMmdTile - 1) / kMmdTile;
    std::vector<Clock::time_point> done(threads);
    const auto t0 = Clock::now();
    mmd_setup(Z.data(), N, (size_t)m, D, mult, 5, norms, inv_s, coef, nullptr);  // O(Nd), timed
    for (int th = 0; th < threads; ++th)
        pool.emplace_back([&, th]() {
            MmdTileWork w;
            double acc[3] = {0.0, 0.0, 0.0};
            for (size_t jt = th; jt < nJ; jt += threads) {
                const size_t b0 = jt * kMmdTile, b1 = std::min(N, b0 + kMmdTile);
                for (size_t a0 = 0; a0 < S && a0 <= b0; a0 += kMmdTile)
                    mmd_tile_pair(Z.data(), norms.data(), N, (size_t)m, D, inv_s, 5, coef, a0,
                                  std::min(S, a0 + kMmdTile), b0, b1, gslice[th].data(), g.data(), acc, w);
            }
            for (int c = 0; c < 3; ++c) sums[th][c] = acc[c];
            done[th] = Clock::now();
        });
    for (auto& t : pool) t.join();
    for (int th = 0; th < threads; ++th)  // slice rows: ascending thread order
        for (size_t e = 0; e < S * D; ++e) g[e] += gslice[th][e];
    const double secs = std::chrono::duration<double>(Clock::now() - t0).count();
    double tot[3] = {0.0, 0.0, 0.0};
    for (int th = 0; th < threads; ++th)
        for (int c = 0; c < 3; ++c) tot[c] += sums[th][c];
    if (sums_out)
        for (int c = 0; c < 3; ++c) sums_out[c] = tot[c];
    double pairs = 0.0;
    for (size_t i = 0; i < S; ++i) pairs += (double)(N - 1 - i);
    if (pairs_out) *pairs_out = pairs;
    return secs;
}

// CPU attack arm (C5 attack stage): Q queried 10-class logit rows (drawn
// before the timed region; members' class-0 logit +1) -> posteriors
// (Tape::softmax, tape.hpp:433-464) -> top-3 sorted features -> the attack
// MLP 3-64-2 (Tape matmul / add_bias / relu / softmax) -> member probability
// -> mid-rank AUC over std::sort'ed scores.  Rows are split into chunks over
// the threads (one Tape per chunk); the sort and rank-sum run on one thread.
// Returns the timed seconds of `reps` evaluations; *auc_out the AUC.
double ref_bench_attack(int threads, int64_t Q, int reps, uint64_t seed, double* auc_out) {
    const size_t q = (size_t)Q, C = 10, K = 3, H = 64;
    std::vector<double> logits(q * C);
    std::vector<uint8_t> lab(q);
    mt::Rng r(seed);
    for (size_t i = 0; i < q; ++i) {
        lab[i] = r.uniform() < 0.5;
        for (size_t c = 0; c < C; ++c) logits[i * C + c] = r.normal() + ((lab[i] && c == 0) ? 1.0 : 0.0);
    }
    std::vector<double> W0(K * H), b0(H, 0.0), W1(H * 2), b1(2, 0.0);
    for (double& v : W0) v = r.uniform(-1.0 / std::sqrt(3.0), 1.0 / std::sqrt(3.0));
    for (double& v : W1) v = r.uniform(-0.125, 0.125);
    const mt::Tensor tW0({K, H}, W0), tb0({H}, b0), tW1({H, 2}, W1), tb1({2}, b1);
    std::vector<double> score(q);
    const size_t chunk = 4096;
    double auc = 0.0;
    const auto t0 = Clock::now();
    for (int rep = 0; rep < reps; ++rep) {
        std::vector<std::thread> pool;
        std::atomic<size_t> next{0};
        for (int th = 0; th < threads; ++th)
            pool.emplace_back([&]() {
                for (size_t c0; (c0 = next.fetch_add(chunk)) < q;) {
                    const size_t rows = std::min(chunk, q - c0);
                    mt::Tape t;
                    mt::Var p = t.softmax(t.constant(mat(logits.data() + c0 * C, rows, C)));
                    const mt::Tensor& P = t.value(p);
                    std::vector<double> F(rows * K);
                    for (size_t i = 0; i < rows; ++i) {
                        double row[10];
                        std::copy(P.data() + i * C, P.data() + (i + 1) * C, row);
                        std::partial_sort(row, row + K, row + C, std::greater<double>());
                        std::copy(row, row + K, F.data() + i * K);
                    }
                    mt::Var h = t.relu(t.add_bias(t.matmul(t.constant(mt::Tensor({rows, K}, F)),
                                                           t.constant(tW0)), t.constant(tb0)));
                    mt::Var s = t.softmax(t.add_bias(t.matmul(h, t.constant(tW1)), t.constant(tb1)));
                    const mt::Tensor& S = t.value(s);
                    for (size_t i = 0; i < rows; ++i) score[c0 + i] = S.data()[i * 2 + 1];
                }
            });
        for (auto& t : pool) t.join();
        // mid-rank Mann-Whitney AUC
        std::vector<std::pair<double, uint8_t>> v(q);
        for (size_t i = 0; i < q; ++i) v[i] = {score[i], lab[i]};
        std::sort(v.begin(), v.end());
        double rpos = 0.0, npos = 0.0;
        for (size_t i = 0; i < q;) {
            size_t e = i;
            while (e < q && v[e].first == v[i].first) ++e;
            const double mid = 0.5 * (double)(i + 1 + e);  // ranks i+1 .. e
            for (size_t k = i; k < e; ++k)
                if (v[k].second) {
                    rpos += mid;
                    npos += 1.0;
                }
            i = e;
        }
        const double nneg = (double)q - npos;
        auc = (rpos - npos * (npos + 1.0) / 2.0) / (npos * nneg);
    }
    const double secs = std::chrono::duration<double>(Clock::now() - t0).count();
    if (auc_out) *auc_out = auc;
    return secs;
}

// how this shim was built (recorded in cpu_baseline)
const char* ref_build_info(void) {
    static const std::string s = std::string("g++ ") + __VERSION__ + ", " + MTREF_FLAGS;
    return s.c_str();
}

}  // extern "C"
