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
#include <chrono>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

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

// CPU baseline arm: `threads` independent models, one Tape per std::thread
// (tape.hpp:84-85), each running `steps` SGD steps of the given
// paradigm on a fixed synthetic batch.  mmd_lambda > 0 adds the
// mapping-based MMD term on the last hidden layer (src rows vs tgt rows).
// Returns wall seconds.
double ref_bench_train(int threads, int L, const int* dims, int B, int src_rows, int steps,
                       double mmd_lambda, uint64_t seed) {
    std::vector<std::thread> pool;
    auto t0 = std::chrono::steady_clock::now();
    for (int th = 0; th < threads; ++th) {
        pool.emplace_back([=]() {
            mt::Rng rng(seed + th);
            const std::size_t d0 = dims[0];
            std::vector<std::vector<double>> W(L), b(L);
            std::vector<double*> Wp(L), bp(L);
            for (int l = 0; l < L; ++l) {
                const double lim = 1.0 / std::sqrt((double)dims[l]);
                W[l].resize((std::size_t)dims[l] * dims[l + 1]);
                for (double& v : W[l]) v = rng.uniform(-lim, lim);
                b[l].assign(dims[l + 1], 0.0);
                Wp[l] = W[l].data();
                bp[l] = b[l].data();
            }
            std::vector<double> X((std::size_t)B * d0);
            for (double& v : X) v = rng.normal();
            std::vector<int32_t> y(B);
            for (auto& v : y) v = (int32_t)rng.below(dims[L]);
            const double denom = B;
            const std::size_t hd = dims[L - 1];
            std::vector<double> G((std::size_t)B * hd), H((std::size_t)B * hd),
                logits((std::size_t)B * dims[L]);
            const double mult[5] = {0.25, 0.5, 1.0, 2.0, 4.0};
            for (int s = 0; s < steps; ++s) {
                const double* inj = nullptr;
                if (mmd_lambda > 0.0) {
                    ref_mlp_forward(L, dims, 0, Wp.data(), bp.data(), X.data(), B, logits.data(),
                                    H.data());
                    double v = 0.0;
                    orc_mmd_gaussian(H.data(), src_rows, H.data() + (std::size_t)src_rows * hd,
                                     B - src_rows, hd, mult, 5, 0.0, &v, nullptr, G.data(),
                                     G.data() + (std::size_t)src_rows * hd);
                    for (double& g : G) g *= mmd_lambda;
                    inj = G.data();
                }
                double loss = 0.0;
                ref_mlp_train_step(L, dims, 1, 0, Wp.data(), bp.data(), X.data(), B, src_rows,
                                   y.data(), nullptr, &denom, 0.05, inj, &loss, nullptr, nullptr);
            }
        });
    }
    for (auto& t : pool) t.join();
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // extern "C"
