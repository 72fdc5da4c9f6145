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
#include <cstdio>
#include <cstdlib>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <functional>
#include <future>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
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

// The per-epoch batch indices and weights are built straight into pinned
// host blocks (the context's recycled pool, Ctx::host_pool) on the worker
// thread and copied to persistent device buffers: no staging copy, no
// synchronising pageable transfer, no per-epoch cudaMalloc / cudaFree
// (cudaFree synchronises the device, which serialised the host and device
// pipelines), and no pinning / unpinning per sweep.
using PinnedPool = HostBlockPool;
template <class T>
struct PinnedVec {  // a fixed-size array in a pooled pinned block (bytes: the block's size)
    PinnedPool* pool = nullptr;
    T* p = nullptr;
    size_t n = 0, bytes = 0;
    PinnedVec() = default;
    PinnedVec(PinnedPool& pl, size_t count) : pool(&pl), n(count) {
        p = static_cast<T*>(pl.get(std::max<size_t>(count * sizeof(T), 1), &bytes));
    }
    PinnedVec(PinnedVec&& o) noexcept : pool(o.pool), p(o.p), n(o.n), bytes(o.bytes) { o.p = nullptr; }
    PinnedVec& operator=(PinnedVec&& o) noexcept {
        std::swap(pool, o.pool);
        std::swap(p, o.p);
        std::swap(n, o.n);
        std::swap(bytes, o.bytes);
        return *this;
    }
    PinnedVec(const PinnedVec&) = delete;
    ~PinnedVec() {
        if (p) pool->put(p, bytes);
    }
    T* data() const { return p; }
    size_t size() const { return n; }
    T& operator[](size_t i) const { return p[i]; }
};
// a grow-only device buffer
struct DevBuf {
    Dev d;
    template <class T>
    T* fit(size_t count) {
        if (d.bytes < count * sizeof(T)) d = Dev(count * sizeof(T));
        return d.as<T>();
    }
};
// one epoch call's indices / weights -> device (stream-ordered; the caller's
// train_epoch synchronises before the pinned blocks are recycled)
template <class F>
void with_uploaded(const PinnedVec<int64_t>& ix, const PinnedVec<float>& w, DevBuf& dix, DevBuf& dw,
                   cudaStream_t st, F&& run) {
    int64_t* di = dix.fit<int64_t>(ix.size());
    float* dwp = dw.fit<float>(w.size());
    MTK_CUDA(cudaMemcpyAsync(di, ix.data(), ix.size() * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    MTK_CUDA(cudaMemcpyAsync(dwp, w.data(), w.size() * sizeof(float), cudaMemcpyHostToDevice, st));
    try {
        run(di, dwp);
    } catch (...) {
        cudaStreamSynchronize(st);  // the copies read the pinned blocks
        throw;
    }
}

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

// batch_iter semantics over one seeded order: consecutive
// slices; the short last batch is padded with weight-0 copies of its last row
struct Batches {
    std::vector<uint64_t> order;
    int B;
    int steps() const { return (int)((order.size() + B - 1) / B); }
    int rows(int t) const { return (int)std::min<size_t>((size_t)B, order.size() - (size_t)t * B); }
    int64_t idx(int t, int r) const { return (int64_t)order[(size_t)t * B + std::min(r, rows(t) - 1)]; }
    float w(int t, int r) const { return r < rows(t) ? 1.f : 0.f; }
    double wsum(int t) const { return (double)rows(t); }
};

// Host-prepared work in order: item e + 1 is built on a worker thread while
// item e runs (exceptions surface at get()).  The builders must only touch
// state no consumer uses (here: the per-model RNG streams).
template <class T, class F>
void run_pipelined(std::vector<std::function<std::vector<T>()>>& items, F&& consume) {
    if (items.empty()) return;
    std::future<std::vector<T>> next = std::async(std::launch::async, items[0]);
    for (size_t e = 0; e < items.size(); ++e) {
        std::vector<T> cur = next.get();
        if (e + 1 < items.size()) next = std::async(std::launch::async, items[e + 1]);
        for (T& x : cur) consume(x);
    }
}

// f(i) for i in [0, n) on all host cores (contiguous ranges; f must only
// touch state of its own i -- here: model g's stream, rows of step t)
template <class F>
void parallel_for(int n, F&& f) {
    unsigned nt = std::thread::hardware_concurrency();
    nt = std::max(1u, std::min({nt, 16u, (unsigned)std::max(n, 1)}));
    if (nt == 1 || n < 8) {
        for (int i = 0; i < n; ++i) f(i);
        return;
    }
    auto range = [&](int a, int b) {
        for (int i = a; i < b; ++i) f(i);
    };
    std::vector<std::future<void>> parts;
    for (unsigned t = 1; t < nt; ++t)
        parts.push_back(std::async(std::launch::async, range, (int)((long long)n * t / nt),
                                   (int)((long long)n * (t + 1) / nt)));
    range(0, (int)((long long)n / nt));
    for (auto& p : parts) p.get();
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
        const char* trace_env = getenv("MTK_SWEEP_TRACE");  // phase wall times to stderr
        auto trace = [&](const char* what) {
            if (!trace_env) return;
            MTK_CUDA(cudaStreamSynchronize(ctx->stream));
            std::fprintf(stderr, "sweep %-14s %8.3f s\n", what,
                         std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
        };
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
            // drawn straight into recycled pinned blocks; each pool's upload
            // overlaps the next pool's draws
            PinnedPool& hp = ctx->host_pool();
            PinnedVec<float> X[2];
            PinnedVec<int32_t> y[2];
            int i = 0;
            try {
                for (Pool* p : {&tgt, &src}) {
                    X[i] = PinnedVec<float>(hp, (size_t)p->rows * d);
                    y[i] = PinnedVec<int32_t>(hp, (size_t)p->rows);
                    ck(mtk_synth(data.h, C, d, (uint64_t)p->rows, mu.data(), p == &tgt ? shift.data() : nullptr,
                                 nullptr, X[i].data(), y[i].data()),
                       "synth");
                    MTK_CUDA(cudaMemcpyAsync(p->X.p, X[i].data(), X[i].size() * 4, cudaMemcpyHostToDevice, st));
                    MTK_CUDA(cudaMemcpyAsync(p->y.p, y[i].data(), y[i].size() * 4, cudaMemcpyHostToDevice, st));
                    ++i;
                }
            } catch (...) {
                cudaStreamSynchronize(st);  // queued copies still read the blocks
                throw;
            }
            MTK_CUDA(cudaStreamSynchronize(st));  // before the blocks are recycled
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

        trace("population");
        const int M = 1 + c.n_shadows;
        std::vector<Rng> streams;
        for (int kk = 0; kk <= M; ++kk) streams.push_back(root.split((uint64_t)kk + 1));
        const int lo = rank * M / world, hi = (rank + 1) * M / world, G = hi - lo;
        need(G >= 1, MTK_CONFIG_ERROR, "sweep: more ranks than models");

        // ---- train_bank ----
        const bool two = c.paradigm == MTK_PARADIGM_PARAMETER;
        Bank bank(ctx, G, dims, two ? 2 : 1);
        std::vector<std::vector<uint64_t>> mem(G), non(G), srcs(G);
        // Each model's stream draws its member split, its weights (exactly as
        // mtk_bank_init_params: uniform(-1/sqrt(fan_in), +) per matrix, zero
        // biases) and its source subset, in that order.  The streams are
        // independent, so the models are drawn on all host cores (up to 0.7 s
        // on one core for 257 models of 1024-512-256-10) into one pinned
        // [matrix][model] block, uploaded with one copy per matrix.
        PinnedPool& pinned = ctx->host_pool();
        const int L = (int)dims.size() - 1, n_mats = L + (two ? 1 : 0);
        auto fan = [&](int i, int io) { return dims[(i < L ? i : L - 1) + io]; };
        std::vector<size_t> mat_off(n_mats + 1, 0);  // floats of matrices 0..i-1, all models
        for (int i = 0; i < n_mats; ++i) mat_off[i + 1] = mat_off[i] + (size_t)G * fan(i, 0) * fan(i, 1);
        {
            PinnedVec<float> hw(pinned, mat_off[n_mats]);
            auto draw_models = [&](int g0, int g1) {
                for (int g = g0; g < g1; ++g) {
                    Rng& r = streams[lo + g];
                    std::vector<uint64_t> perm = r.permutation((uint64_t)c.pool);
                    mem[g].assign(perm.begin(), perm.begin() + c.members);
                    non[g].assign(perm.begin() + c.members, perm.begin() + 2 * (size_t)c.members);
                    for (int i = 0; i < n_mats; ++i) {
                        const size_t nw = (size_t)fan(i, 0) * fan(i, 1);
                        const double lim = 1.0 / std::sqrt((double)fan(i, 0));
                        float* w = hw.data() + mat_off[i] + (size_t)g * nw;
                        for (size_t j = 0; j < nw; ++j) w[j] = (float)mtk_rng_uniform(r.h, -lim, lim);
                    }
                    std::vector<uint64_t> sp = r.permutation((uint64_t)c.source_pool);
                    srcs[g].assign(sp.begin(), sp.begin() + c.source_per_model);
                }
            };
            unsigned nt = std::thread::hardware_concurrency();
            nt = std::max(1u, std::min({nt, 32u, (unsigned)G}));
            std::vector<std::future<void>> parts;
            for (unsigned t = 1; t < nt; ++t)
                parts.push_back(std::async(std::launch::async, draw_models, (int)((long long)G * t / nt),
                                           (int)((long long)G * (t + 1) / nt)));
            draw_models(0, (int)((long long)G / nt));
            for (auto& f : parts) f.get();  // (rethrows a worker's failure)
            for (int i = 0; i < n_mats; ++i) {
                float *Wd = nullptr, *bd = nullptr;
                ck(mtk_bank_param_device(bank.h, i, &Wd, &bd), "param_device");
                MTK_CUDA(cudaMemcpyAsync(Wd, hw.data() + mat_off[i], (mat_off[i + 1] - mat_off[i]) * 4,
                                         cudaMemcpyHostToDevice, st));
                MTK_CUDA(cudaMemsetAsync(bd, 0, (size_t)G * fan(i, 1) * 4, st));
            }
            MTK_CUDA(cudaStreamSynchronize(st));  // before the pinned block is recycled
        }
        const int B = c.batch;
        mtk_step tmpl{};
        tmpl.lr = c.lr;
        tmpl.optimizer = c.optimizer;
        // Each epoch becomes one or more train_epoch calls whose batch indices
        // [nsteps][G][rows] are built on the host; a worker thread builds epoch
        // e + 1 (the per-model streams advance in the same order as before)
        // while the device trains epoch e.
        struct Call {
            const Pool* pool;
            int rows, nsteps;
            PinnedVec<int64_t> ix;
            PinnedVec<float> w;
            std::vector<double> den;
            mtk_step s;
        };
        DevBuf dix_buf, dw_buf;
        auto make_call = [&](const Pool& pool, int rows, int nsteps,
                             const std::function<void(int g, int t, int64_t* ix, float* w)>& fill,
                             std::vector<double> denom0, mtk_step s) {
            Call cl{&pool, rows, nsteps, PinnedVec<int64_t>(pinned, (size_t)nsteps * G * rows),
                    PinnedVec<float>(pinned, (size_t)nsteps * G * rows), std::move(denom0), s};
            parallel_for(G, [&](int g) {  // the fills read model g's state only
                for (int t = 0; t < nsteps; ++t)
                    fill(g, t, cl.ix.data() + ((size_t)t * G + g) * rows, cl.w.data() + ((size_t)t * G + g) * rows);
            });
            cl.s.B = rows;
            return cl;
        };
        auto model_orders = [&](uint64_t n) {  // one permutation per model stream (independent)
            std::vector<Batches> o(G, Batches{{}, B});
            parallel_for(G, [&](int g) { o[g].order = streams[lo + g].permutation(n); });
            return o;
        };
        std::vector<std::function<std::vector<Call>()>> epochs;
        if (c.paradigm == MTK_PARADIGM_MODEL)
            for (int e = 0; e < c.pretrain_epochs; ++e)
                epochs.push_back([&]() {
                    auto orders = model_orders((uint64_t)c.source_per_model);
                    const int nsteps = orders[0].steps();
                    std::vector<double> den;
                    for (int t = 0; t < nsteps; ++t) den.push_back(orders[0].wsum(t));
                    std::vector<Call> v;
                    v.push_back(make_call(src, B, nsteps, [&](int g, int t, int64_t* ix, float* w) {
                        for (int r = 0; r < B; ++r) {
                            ix[r] = (int64_t)srcs[g][orders[g].idx(t, r)];
                            w[r] = orders[g].w(t, r);
                        }
                    }, den, tmpl));
                    return v;
                });
        for (int e = 0; e < c.epochs; ++e)
            epochs.push_back([&]() {
                auto orders = model_orders((uint64_t)c.members);
                const int nsteps = orders[0].steps();
                std::vector<Call> v;
                if (c.paradigm == MTK_PARADIGM_MODEL) {
                    std::vector<double> den;
                    for (int t = 0; t < nsteps; ++t) den.push_back(orders[0].wsum(t));
                    mtk_step s = tmpl;
                    s.frozen_layers = c.frozen_layers;
                    v.push_back(make_call(tgt, B, nsteps, [&](int g, int t, int64_t* ix, float* w) {
                        for (int r = 0; r < B; ++r) {
                            ix[r] = (int64_t)mem[g][orders[g].idx(t, r)];
                            w[r] = orders[g].w(t, r);
                        }
                    }, den, s));
                    return v;
                }
                // co-training: a source batch rides along with every member batch
                auto fill = [&](int g, int t, int64_t* ix, float* w) {
                    for (int r = 0; r < B; ++r) {
                        ix[r] = (int64_t)srcs[g][((int64_t)t * B + r) % c.source_per_model];
                        w[r] = 1.f;
                        ix[B + r] = src.rows + (int64_t)mem[g][orders[g].idx(t, r)];
                        w[B + r] = orders[g].w(t, r);
                    }
                };
                mtk_step s = tmpl;
                s.src_rows = B;
                if (c.paradigm == MTK_PARADIGM_MAPPING) {
                    s.mmd_lambda = c.mmd_lambda;
                    std::vector<double> den;
                    for (int t = 0; t < nsteps; ++t) den.push_back((double)B + orders[0].wsum(t));
                    v.push_back(make_call(both, 2 * B, nsteps, fill, den, s));
                    return v;
                }
                // parameter-based: head denominators (B, member weight sum); the
                // per-step override covers head 0 only, so runs of steps with
                // equal member sums go in one call each
                int t0 = 0;
                while (t0 < nsteps) {
                    int t1 = t0 + 1;
                    while (t1 < nsteps && orders[0].wsum(t1) == orders[0].wsum(t0)) ++t1;
                    mtk_step sp = s;
                    sp.denom[1] = orders[0].wsum(t0);
                    v.push_back(make_call(both, 2 * B, t1 - t0,
                                          [&](int g, int t, int64_t* ix, float* w) { fill(g, t0 + t, ix, w); },
                                          std::vector<double>(t1 - t0, (double)B), sp));
                    t0 = t1;
                }
                return v;
            });
        run_pipelined(epochs, [&](Call& cl) {
            with_uploaded(cl.ix, cl.w, dix_buf, dw_buf, st, [&](const int64_t* dix, const float* dw) {
                ck(mtk_bank_train_epoch(bank.h, &cl.s, cl.pool->X.as<float>(), cl.pool->y.as<int32_t>(),
                                        cl.pool->rows, dix, dw, cl.den.data(), cl.nsteps),
                   "train_epoch");
            });
        });

        trace("training");
        // ---- query_features: top-k posteriors of each model on its members
        // and non-members (the target-domain head) ----
        const int Q = 2 * c.members, kf = c.k;
        trace("features: start");
        // in chunks of the training batch's rows: the bank's activation
        // buffers (sized by training) are reused; a whole-Q forward would
        // allocate them for 4096 rows x 257 models (GBs, per sweep)
        const int qb = std::min(Q, c.paradigm == MTK_PARADIGM_MODEL ? B : 2 * B);
        const int nchunk = (Q + qb - 1) / qb;
        Dev lq((size_t)G * Q * C * 4), lc((size_t)G * qb * C * 4);
        {
            // chunk-major indices: chunk k holds [G][rows of the chunk]
            std::vector<int64_t> qi((size_t)G * Q);
            size_t o = 0;
            for (int k = 0; k < nchunk; ++k) {
                const int q0 = k * qb, nq = std::min(qb, Q - q0);
                for (int g = 0; g < G; ++g)
                    for (int q = q0; q < q0 + nq; ++q)
                        qi[o++] = (int64_t)(q < c.members ? mem[g][q] : non[g][q - c.members]);
            }
            Dev dqi = upload(qi, st);
            float* Xc = static_cast<float*>(ctx->sweep_buf((size_t)G * qb * d * 4));  // reused across sweeps
            for (int k = 0; k < nchunk; ++k) {
                const int q0 = k * qb, nq = std::min(qb, Q - q0);
                ck(mtk_gather_rows(ctx, tgt.X.p, tgt.rows, d, dqi.as<int64_t>() + (size_t)G * q0, G, nq, Xc, nq, 0),
                   "gather_rows");
                ck(mtk_bank_forward(bank.h, Xc, nq, two ? 1 : 0, lc.as<float>(), nullptr), "forward");
                MTK_CUDA(cudaMemcpy2DAsync(lq.as<float>() + (size_t)q0 * C, (size_t)Q * C * 4, lc.p,
                                           (size_t)nq * C * 4, (size_t)nq * C * 4, G, cudaMemcpyDeviceToDevice,
                                           st));
            }
            MTK_CUDA(cudaStreamSynchronize(st));
        }
        trace("features: posteriors");
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

        trace("features");
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
        struct AttCall {
            PinnedVec<int64_t> ix;
            PinnedVec<float> w;
            std::vector<double> den;
        };
        // Three stages: a thread draws each epoch's Fisher-Yates targets from
        // the attack stream (sequential, up to two epochs ahead); the epoch
        // builder applies the swaps and fills the batch indices; the caller
        // trains.  The permutations are the stream's own (rng_host.cpp).
        const bool staged = ntr >= 2 && ntr < (int64_t(1) << 32);
        std::mutex qm;
        std::condition_variable qcv;
        std::deque<std::vector<uint32_t>> tq;
        bool tstop = false;
        std::thread tthread;
        if (staged)
            tthread = std::thread([&] {
                std::vector<uint64_t> raw((size_t)ntr - 1);
                for (int e = 0; e < c.attack_epochs; ++e) {
                    std::vector<uint32_t> js((size_t)ntr - 1);
                    rng_permutation_targets(ar.h, (uint64_t)ntr, js.data(), raw.data());
                    std::unique_lock<std::mutex> lk(qm);
                    qcv.wait(lk, [&] { return tq.size() < 2 || tstop; });
                    if (tstop) return;
                    tq.push_back(std::move(js));
                    qcv.notify_all();
                }
            });
        struct JoinTargets {  // on every exit path
            std::thread& t;
            std::mutex& m;
            std::condition_variable& cv;
            bool& stop;
            ~JoinTargets() {
                {
                    std::lock_guard<std::mutex> lk(m);
                    stop = true;
                }
                cv.notify_all();
                if (t.joinable()) t.join();
            }
        } join_targets{tthread, qm, qcv, tstop};
        std::vector<uint64_t> order_buf(staged ? (size_t)ntr : 0);
        std::vector<uint32_t> swap_buf(staged ? (size_t)ntr : 0);
        auto next_order = [&]() -> std::vector<uint64_t> {
            if (!staged) return ar.permutation((uint64_t)ntr);
            std::vector<uint32_t> js;
            {
                std::unique_lock<std::mutex> lk(qm);
                qcv.wait(lk, [&] { return !tq.empty(); });
                js = std::move(tq.front());
                tq.pop_front();
            }
            qcv.notify_all();
            order_buf.resize((size_t)ntr);
            permutation_apply((uint64_t)ntr, js.data(), swap_buf.data(), order_buf.data());
            return std::move(order_buf);  // (handed back after the fill)
        };
        std::vector<std::function<std::vector<AttCall>()>> aep(c.attack_epochs, [&]() {
            Batches bl{next_order(), c.attack_batch};
            const int nb = bl.steps();
            AttCall a{PinnedVec<int64_t>(pinned, (size_t)nb * c.attack_batch),
                      PinnedVec<float>(pinned, (size_t)nb * c.attack_batch), std::vector<double>(nb)};
            parallel_for(nb, [&](int t) {
                for (int r = 0; r < c.attack_batch; ++r) {
                    a.ix[(size_t)t * c.attack_batch + r] = bl.idx(t, r);
                    a.w[(size_t)t * c.attack_batch + r] = bl.w(t, r);
                }
                a.den[t] = bl.wsum(t);
            });
            if (staged) order_buf = std::move(bl.order);  // the next epoch's swap output
            std::vector<AttCall> v;
            v.push_back(std::move(a));
            return v;
        });
        run_pipelined(aep, [&](AttCall& a) {
            mtk_step s{};
            s.B = c.attack_batch;
            s.lr = c.attack_lr;
            s.optimizer = c.attack_optimizer;
            with_uploaded(a.ix, a.w, dix_buf, dw_buf, st, [&](const int64_t* dix, const float* dw) {
                ck(mtk_bank_train_epoch(att.h, &s, Ftr, dl.as<int32_t>(), ntr, dix, dw, a.den.data(),
                                        (int)a.den.size()),
                   "attack train_epoch");
            });
        });

        trace("attack train");
        // ---- score the target's members / non-members: AUC + accuracy ----
        std::vector<uint8_t> lab((size_t)Q);
        for (int i = 0; i < Q; ++i) lab[(size_t)i] = i < c.members ? 1 : 0;
        Dev dlab = upload(lab, st), alog((size_t)Q * 2 * 4), sc((size_t)Q * 4);
        ck(mtk_bank_forward(att.h, Fall.as<float>(), Q, 0, alog.as<float>(), nullptr), "attack forward");
        ck(mtk_posterior_column(ctx, alog.as<float>(), Q, 2, 1, sc.as<float>()), "posterior_column");
        double auc = 0.0, acc = 0.0;
        ck(mtk_auc(ctx, sc.as<float>(), dlab.as<uint8_t>(), Q, &auc, &acc), "auc");
        trace("attack score");
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
