// sweep.cpp -- the shadow-training + membership-attack sweep in C++ (SURVEY.md
// 8(a) rows a17 / a18; Appendix A), the native host driver
// behind mtk_sweep_run and mt::gpu::run_shadow_sweep.
//
// It is the same composition as paper_2011_09463_b200/sweep.py (whose module
// docstring pins the definitions: data, per-model streams, member splits,
// paradigms, attack), call for call on the same library entry points, so the
// two drivers give bit-identical AUC / accuracy on one device.  Differences
// are in the plumbing only: whole epochs run through mtk_bank_train_epoch
// (device-side batch gather + step, no host round trip per step), and the
// ranks' feature blocks move device to device through mtk_allgather.
//
// All sampling is host-side mt::Rng (rng.hpp:13-75, bit-exact): root =
// Rng(seed); data = root.split(0); model k (0 = target, 1..S shadows) =
// root.split(k + 1) in ascending k on every rank; stream M drives the attack.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "internal.h"

namespace mtk {
namespace {

// C-ABI status -> the Failure the guard() converts back
void ck(int st, const char* what) {
    if (st != MTK_OK) fail(st, std::string(what) + ": " + mtk_last_error());
}

struct Dev {  // owning device buffer
    void* p = nullptr;
    size_t bytes = 0;
    Dev() = default;
    explicit Dev(size_t b) : bytes(b) {
        if (b) MTK_CUDA(cudaMalloc(&p, b));
    }
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
    Dev(Dev&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; }
    Dev& operator=(Dev&& o) noexcept {
        std::swap(p, o.p);
        std::swap(bytes, o.bytes);
        return *this;
    }
    ~Dev() {
        if (p) cudaFree(p);
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

template <class T>
Dev upload(const std::vector<T>& h, cudaStream_t s) {
    Dev d(h.size() * sizeof(T));
    if (!h.empty()) {
        MTK_CUDA(cudaMemcpyAsync(d.p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, s));
        MTK_CUDA(cudaStreamSynchronize(s));  // h may die after the call
    }
    return d;
}

struct Rng {  // owning mtk_rng
    mtk_rng* h = nullptr;
    explicit Rng(uint64_t seed) { ck(mtk_rng_create(seed, &h), "rng"); }
    Rng(Rng&& o) noexcept : h(o.h) { o.h = nullptr; }
    Rng(const Rng&) = delete;
    explicit Rng(mtk_rng* x) : h(x) {}
    ~Rng() {
        if (h) mtk_rng_destroy(h);
    }
    Rng split(uint64_t stream) {
        mtk_rng* c = nullptr;
        ck(mtk_rng_split(h, stream, &c), "rng split");
        return Rng(c);
    }
    std::vector<uint64_t> permutation(uint64_t n) {
        std::vector<uint64_t> p(n);
        ck(mtk_rng_permutation(h, n, p.data()), "permutation");
        return p;
    }
    std::vector<double> normals(uint64_t n) {
        std::vector<double> v(n);
        ck(mtk_rng_fill_normal(h, v.data(), n), "normals");
        return v;
    }
};

struct Bank {  // owning mtk_bank
    mtk_bank* h = nullptr;
    Bank(mtk_ctx* c, int G, const std::vector<int>& dims, int heads) {
        ck(mtk_bank_create(c, G, (int)dims.size() - 1, dims.data(), heads, &h), "bank");
    }
    Bank(const Bank&) = delete;
    ~Bank() {
        if (h) mtk_bank_destroy(h);
    }
};

// batch_iter semantics: consecutive slices of the seeded
// order; the short last batch is padded with weight-0 copies of its last row
struct Batch {
    std::vector<int64_t> idx;
    std::vector<float> w;
    double wsum;
};
std::vector<Batch> batches(const std::vector<uint64_t>& order, int B) {
    std::vector<Batch> out;
    for (size_t s = 0; s < order.size(); s += (size_t)B) {
        Batch b;
        const size_t n = std::min((size_t)B, order.size() - s);
        for (size_t i = 0; i < (size_t)B; ++i) {
            b.idx.push_back((int64_t)order[s + std::min(i, n - 1)]);
            b.w.push_back(i < n ? 1.f : 0.f);
        }
        b.wsum = (double)n;
        out.push_back(std::move(b));
    }
    return out;
}

struct Pool {  // a device-resident population: X [rows, d] fp32, y [rows] int32
    Dev X, y;
    int64_t rows = 0;
};

}  // namespace
}  // namespace mtk

using namespace mtk;

extern "C" {

void mtk_sweep_config_default(mtk_sweep_config* c) {
    if (!c) return;
    std::memset(c, 0, sizeof(*c));
    c->paradigm = MTK_PARADIGM_MODEL;
    c->n_layers = 2;
    c->dims[0] = 784;
    c->dims[1] = 256;
    c->dims[2] = 10;
    c->n_shadows = 4;
    c->pool = 8192;
    c->members = 2048;
    c->source_pool = 16384;
    c->source_per_model = 4096;
    c->batch = 128;
    c->epochs = 10;
    c->pretrain_epochs = 2;
    c->frozen_layers = 0;
    c->lr = 0.05;
    c->optimizer = 0;
    c->mmd_lambda = 1.0;
    c->mu_scale = 0.1;
    c->shift_scale = 0.5;
    c->k = 3;
    c->attack_hidden = 64;
    c->attack_epochs = 30;
    c->attack_batch = 1024;
    c->attack_lr = 0.1;
    c->attack_optimizer = 0;
    c->data_rng = 0;
    c->seed = 20110946ULL;
}

int mtk_sweep_run(mtk_ctx* ctx, const mtk_sweep_config* cfg, mtk_comm* comm, mtk_sweep_result* out) {
    return guard_on(ctx, [&] {
        need(ctx && cfg && out, MTK_VALUE_ERROR, "sweep: null argument");
        const auto t0 = std::chrono::steady_clock::now();
        const mtk_sweep_config& c = *cfg;
        // ---- validation (sweep.py SweepConfig.validate) ----
        need(c.paradigm >= 0 && c.paradigm <= 2, MTK_CONFIG_ERROR, "sweep: unknown paradigm");
        need(c.n_layers >= 1 && c.n_layers < MTK_SWEEP_MAX_LAYERS, MTK_CONFIG_ERROR, "sweep: bad layer count");
        need(c.paradigm == MTK_PARADIGM_MODEL || c.n_layers >= 2, MTK_CONFIG_ERROR,
             "sweep: transfer paradigms need a hidden layer");
        need(2LL * c.members <= c.pool, MTK_CONFIG_ERROR, "sweep: members + non-members exceed the pool");
        need(c.source_per_model <= c.source_pool, MTK_CONFIG_ERROR, "sweep: source_per_model exceeds source_pool");
        need(c.n_shadows >= 1 && c.members >= 1 && c.batch >= 1 && c.attack_batch >= 1 && c.epochs >= 0,
             MTK_CONFIG_ERROR, "sweep: counts must be positive");
        const std::vector<int> dims(c.dims, c.dims + c.n_layers + 1);
        const int C = dims.back(), d = dims[0];
        need(c.k >= 1 && c.k <= C, MTK_CONFIG_ERROR, "sweep: k must be in [1, C]");
        need(c.optimizer == 0 || c.optimizer == 1, MTK_CONFIG_ERROR, "sweep: optimizer is 0 (SGD) or 1 (Adam)");
        need(c.attack_optimizer == 0 || c.attack_optimizer == 1, MTK_CONFIG_ERROR,
             "sweep: attack_optimizer is 0 (SGD) or 1 (Adam)");
        need(c.data_rng == 0 || c.data_rng == 1, MTK_CONFIG_ERROR, "sweep: data_rng is 0 (host) or 1 (counter)");
        int world = 1, rank = 0;
        if (comm) ck(mtk_comm_info(comm, &world, &rank, nullptr, nullptr), "comm_info");
        cudaStream_t st = ctx->stream;

        // ---- population (sweep.py Population) ----
        Rng root(c.seed);
        Rng data = root.split(0);
        std::vector<double> mu = data.normals((uint64_t)C * d), shift = data.normals((uint64_t)d);
        for (double& v : mu) v = c.mu_scale * v;
        for (double& v : shift) v = c.shift_scale * v;
        Pool tgt, src;
        tgt.rows = c.pool;
        src.rows = c.source_pool;
        tgt.X = Dev((size_t)tgt.rows * d * 4);
        tgt.y = Dev((size_t)tgt.rows * 4);
        src.X = Dev((size_t)src.rows * d * 4);
        src.y = Dev((size_t)src.rows * 4);
        if (c.data_rng == 1) {  // device counter-based pools (mtk_synth_counter, 8(f) f3)
            std::vector<float> mu32(mu.begin(), mu.end()), sh32(shift.begin(), shift.end());
            Dev dmu = upload(mu32, st), dsh = upload(sh32, st);
            ck(mtk_synth_counter(ctx, c.seed, 1, C, d, tgt.rows, dmu.as<float>(), dsh.as<float>(),
                                 tgt.X.as<float>(), tgt.y.as<int32_t>()), "synth_counter");
            ck(mtk_synth_counter(ctx, c.seed, 2, C, d, src.rows, dmu.as<float>(), nullptr, src.X.as<float>(),
                                 src.y.as<int32_t>()), "synth_counter");
            MTK_CUDA(cudaStreamSynchronize(st));
        } else {
            for (Pool* p : {&tgt, &src}) {
                std::vector<float> X((size_t)p->rows * d);
                std::vector<int32_t> y((size_t)p->rows);
                ck(mtk_synth(data.h, C, d, (uint64_t)p->rows, mu.data(), p == &tgt ? shift.data() : nullptr,
                             nullptr, X.data(), y.data()),
                   "synth");
                MTK_CUDA(cudaMemcpyAsync(p->X.p, X.data(), X.size() * 4, cudaMemcpyHostToDevice, st));
                MTK_CUDA(cudaMemcpyAsync(p->y.p, y.data(), y.size() * 4, cudaMemcpyHostToDevice, st));
                MTK_CUDA(cudaStreamSynchronize(st));
            }
        }
        // one combined pool [source; target] for the co-training paradigms'
        // epochs (a step's batch is source rows then member rows)
        Pool both;
        both.rows = src.rows + tgt.rows;
        both.X = Dev((size_t)both.rows * d * 4);
        both.y = Dev((size_t)both.rows * 4);
        MTK_CUDA(cudaMemcpyAsync(both.X.p, src.X.p, src.X.bytes, cudaMemcpyDeviceToDevice, st));
        MTK_CUDA(cudaMemcpyAsync(both.X.as<char>() + src.X.bytes, tgt.X.p, tgt.X.bytes, cudaMemcpyDeviceToDevice, st));
        MTK_CUDA(cudaMemcpyAsync(both.y.p, src.y.p, src.y.bytes, cudaMemcpyDeviceToDevice, st));
        MTK_CUDA(cudaMemcpyAsync(both.y.as<char>() + src.y.bytes, tgt.y.p, tgt.y.bytes, cudaMemcpyDeviceToDevice, st));

        const int M = 1 + c.n_shadows;
        std::vector<Rng> streams;
        for (int kk = 0; kk <= M; ++kk) streams.push_back(root.split((uint64_t)kk + 1));
        const int lo = rank * M / world, hi = (rank + 1) * M / world, G = hi - lo;
        need(G >= 1, MTK_CONFIG_ERROR, "sweep: more ranks than models");

        // ---- train_bank ----
        const bool two = c.paradigm == MTK_PARADIGM_PARAMETER;
        Bank bank(ctx, G, dims, two ? 2 : 1);
        std::vector<std::vector<uint64_t>> mem(G), non(G), srcs(G);
        for (int g = 0; g < G; ++g) {
            Rng& r = streams[lo + g];
            std::vector<uint64_t> perm = r.permutation((uint64_t)c.pool);
            mem[g].assign(perm.begin(), perm.begin() + c.members);
            non[g].assign(perm.begin() + c.members, perm.begin() + 2 * (size_t)c.members);
            ck(mtk_bank_init_params(bank.h, g, r.h), "init_params");
            std::vector<uint64_t> sp = r.permutation((uint64_t)c.source_pool);
            srcs[g].assign(sp.begin(), sp.begin() + c.source_per_model);
        }
        const int B = c.batch;
        mtk_step tmpl{};
        tmpl.lr = c.lr;
        tmpl.optimizer = c.optimizer;
        // one epoch: per model the batches of `orders`, row r of step t mapped
        // through rowmap(g, t, idx) to pool rows; [nsteps][G][rows] on the device
        auto run_epoch = [&](const Pool& pool, int rows, int nsteps,
                             const std::function<void(int g, int t, int64_t* ix, float* w)>& fill,
                             const std::vector<double>& denom0, mtk_step s) {
            std::vector<int64_t> ix((size_t)nsteps * G * rows);
            std::vector<float> w((size_t)nsteps * G * rows);
            for (int t = 0; t < nsteps; ++t)
                for (int g = 0; g < G; ++g)
                    fill(g, t, ix.data() + ((size_t)t * G + g) * rows, w.data() + ((size_t)t * G + g) * rows);
            Dev dix = upload(ix, st), dw = upload(w, st);
            s.B = rows;
            ck(mtk_bank_train_epoch(bank.h, &s, pool.X.as<float>(), pool.y.as<int32_t>(), pool.rows,
                                    dix.as<int64_t>(), dw.as<float>(), denom0.data(), nsteps),
               "train_epoch");
        };
        auto model_orders = [&](uint64_t n) {
            std::vector<std::vector<Batch>> o;
            for (int g = 0; g < G; ++g) o.push_back(batches(streams[lo + g].permutation(n), B));
            return o;
        };
        if (c.paradigm == MTK_PARADIGM_MODEL && c.pretrain_epochs > 0) {
            for (int e = 0; e < c.pretrain_epochs; ++e) {
                auto orders = model_orders((uint64_t)c.source_per_model);
                const int nsteps = (int)orders[0].size();
                std::vector<double> den;
                for (int t = 0; t < nsteps; ++t) den.push_back(orders[0][t].wsum);
                run_epoch(src, B, nsteps, [&](int g, int t, int64_t* ix, float* w) {
                    for (int r = 0; r < B; ++r) {
                        ix[r] = (int64_t)srcs[g][orders[g][t].idx[r]];
                        w[r] = orders[g][t].w[r];
                    }
                }, den, tmpl);
            }
        }
        for (int e = 0; e < c.epochs; ++e) {
            auto orders = model_orders((uint64_t)c.members);
            const int nsteps = (int)orders[0].size();
            if (c.paradigm == MTK_PARADIGM_MODEL) {
                std::vector<double> den;
                for (int t = 0; t < nsteps; ++t) den.push_back(orders[0][t].wsum);
                mtk_step s = tmpl;
                s.frozen_layers = c.frozen_layers;
                run_epoch(tgt, B, nsteps, [&](int g, int t, int64_t* ix, float* w) {
                    for (int r = 0; r < B; ++r) {
                        ix[r] = (int64_t)mem[g][orders[g][t].idx[r]];
                        w[r] = orders[g][t].w[r];
                    }
                }, den, s);
                continue;
            }
            // co-training: a source batch rides along with every member batch
            auto fill = [&](int g, int t, int64_t* ix, float* w) {
                for (int r = 0; r < B; ++r) {
                    ix[r] = (int64_t)srcs[g][((int64_t)t * B + r) % c.source_per_model];
                    w[r] = 1.f;
                    ix[B + r] = src.rows + (int64_t)mem[g][orders[g][t].idx[r]];
                    w[B + r] = orders[g][t].w[r];
                }
            };
            mtk_step s = tmpl;
            s.src_rows = B;
            if (c.paradigm == MTK_PARADIGM_MAPPING) {
                s.mmd_lambda = c.mmd_lambda;
                std::vector<double> den;
                for (int t = 0; t < nsteps; ++t) den.push_back((double)B + orders[0][t].wsum);
                run_epoch(both, 2 * B, nsteps, fill, den, s);
            } else {
                // parameter-based: head denominators (B, member weight sum); the
                // per-step override covers head 0 only, so runs of steps with
                // equal member sums go in one call each
                int t0 = 0;
                while (t0 < nsteps) {
                    int t1 = t0 + 1;
                    while (t1 < nsteps && orders[0][t1].wsum == orders[0][t0].wsum) ++t1;
                    mtk_step sp = s;
                    sp.denom[1] = orders[0][t0].wsum;
                    std::vector<double> den(t1 - t0, (double)B);
                    run_epoch(both, 2 * B, t1 - t0,
                              [&](int g, int t, int64_t* ix, float* w) { fill(g, t0 + t, ix, w); }, den, sp);
                    t0 = t1;
                }
            }
        }

        // ---- query_features: top-k posteriors of each model on its members
        // and non-members (the target-domain head) ----
        const int Q = 2 * c.members, kf = c.k;
        Dev Xq((size_t)G * Q * d * 4), lq((size_t)G * Q * C * 4);
        {
            std::vector<int64_t> qi((size_t)G * Q);
            for (int g = 0; g < G; ++g) {
                std::copy(mem[g].begin(), mem[g].end(), qi.begin() + (size_t)g * Q);
                std::copy(non[g].begin(), non[g].end(), qi.begin() + (size_t)g * Q + c.members);
            }
            Dev dqi = upload(qi, st);
            ck(mtk_gather_rows(ctx, tgt.X.p, tgt.rows, d, dqi.as<int64_t>(), G, Q, Xq.p, Q, 0), "gather_rows");
            ck(mtk_bank_forward(bank.h, Xq.as<float>(), Q, two ? 1 : 0, lq.as<float>(), nullptr), "forward");
            MTK_CUDA(cudaStreamSynchronize(st));
        }
        const int gmax = (M + world - 1) / world;  // the largest rank block (padded for the all-gather)
        const size_t blk = (size_t)gmax * Q * kf;
        Dev F(blk * 4);
        MTK_CUDA(cudaMemsetAsync(F.p, 0, F.bytes, st));
        ck(mtk_posterior_features(ctx, lq.as<float>(), (int64_t)G * Q, C, kf, nullptr, F.as<float>()), "features");
        // all ranks' blocks, padded to gmax models, in rank order -> [M][Q][k] in model order
        Dev Fall((size_t)M * Q * kf * 4);
        if (world > 1) {
            Dev gathered((size_t)world * blk * 4);
            ck(mtk_allgather(comm, ctx, F.p, gathered.p, blk * 4), "allgather");
            for (int r = 0; r < world; ++r) {
                const int rl = r * M / world, rh = (r + 1) * M / world;
                MTK_CUDA(cudaMemcpyAsync(Fall.as<float>() + (size_t)rl * Q * kf, gathered.as<float>() + r * blk,
                                         (size_t)(rh - rl) * Q * kf * 4, cudaMemcpyDeviceToDevice, st));
            }
            MTK_CUDA(cudaStreamSynchronize(st));
        } else {
            MTK_CUDA(cudaMemcpyAsync(Fall.p, F.p, Fall.bytes, cudaMemcpyDeviceToDevice, st));
        }

        // ---- train_attack on the shadows' features (member 1 / non-member 0) ----
        const int64_t ntr = (int64_t)c.n_shadows * Q;
        std::vector<int32_t> ltr((size_t)ntr);
        for (int64_t i = 0; i < ntr; ++i) ltr[(size_t)i] = (i % Q) < c.members ? 1 : 0;
        Dev dl = upload(ltr, st);
        const std::vector<int> adims = {kf, c.attack_hidden, 2};
        Bank att(ctx, 1, adims, 1);
        Rng& ar = streams[M];
        ck(mtk_bank_init_params(att.h, 0, ar.h), "init_params");
        const float* Ftr = Fall.as<float>() + (size_t)Q * kf;  // models 1 .. M-1
        for (int e = 0; e < c.attack_epochs; ++e) {
            std::vector<Batch> bl = batches(ar.permutation((uint64_t)ntr), c.attack_batch);
            const int nb = (int)bl.size();
            std::vector<int64_t> ix;
            std::vector<float> w;
            std::vector<double> den;
            for (auto& b : bl) {
                ix.insert(ix.end(), b.idx.begin(), b.idx.end());
                w.insert(w.end(), b.w.begin(), b.w.end());
                den.push_back(b.wsum);
            }
            Dev dix = upload(ix, st), dw = upload(w, st);
            mtk_step s{};
            s.B = c.attack_batch;
            s.lr = c.attack_lr;
            s.optimizer = c.attack_optimizer;
            ck(mtk_bank_train_epoch(att.h, &s, Ftr, dl.as<int32_t>(), ntr, dix.as<int64_t>(), dw.as<float>(),
                                    den.data(), nb),
               "attack train_epoch");
        }

        // ---- score the target's members / non-members: AUC + accuracy ----
        std::vector<uint8_t> lab((size_t)Q);
        for (int i = 0; i < Q; ++i) lab[(size_t)i] = i < c.members ? 1 : 0;
        Dev dlab = upload(lab, st), alog((size_t)Q * 2 * 4), sc((size_t)Q * 4);
        ck(mtk_bank_forward(att.h, Fall.as<float>(), Q, 0, alog.as<float>(), nullptr), "attack forward");
        ck(mtk_posterior_column(ctx, alog.as<float>(), Q, 2, 1, sc.as<float>()), "posterior_column");
        double auc = 0.0, acc = 0.0;
        ck(mtk_auc(ctx, sc.as<float>(), dlab.as<uint8_t>(), Q, &auc, &acc), "auc");
        out->auc = auc;
        out->accuracy = acc;
        out->models = M;
        out->rank_model_begin = lo;
        out->rank_model_end = hi;
        out->n_queries = Q;
        out->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}

}  // extern "C"
