// capi.cu -- the C ABI (include/minitransfer/mtk.h): contexts, the grouped
// model bank, the MMD and attack entry points.
//
// One bank step runs, for all G models at once, the reference composition
//   forward : matmul -> add_bias -> relu ... -> cross_entropy_weighted
//             (tape.hpp:225-290, 204-221, 342-352, 475-520)
//   backward: Tape::backward reverse sweep (tape.hpp:870-886)
//   update  : optimizer_step SGD (optim.hpp:46-48)
// as a fixed schedule of fused kernels (no device tape):
//   per layer  FWD gemm (+bias, +ReLU)            -> H[l+1]
//   head       CE (softmax, loss, dlogits)        -> dZ_L
//   [mapping]  MMD beta, pairs, finish            -> lambda * dMMD/dH_{L-1}
//   per layer  DX gemm (+inject, *ReLU mask) then DW gemm (+SGD) + bias SGD
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "internal.h"

namespace {
thread_local std::string tl_last_error;
}

extern "C" void mtk_internal_set_error(const char* msg) { tl_last_error = msg ? msg : ""; }

namespace mtk {

double* Ctx::scratch(size_t bytes) {
    if (bytes > scratch_bytes) {
        if (d_scratch) MTK_CUDA(cudaFree(d_scratch));
        d_scratch = nullptr;
        MTK_CUDA(cudaMalloc(&d_scratch, bytes));
        scratch_bytes = bytes;
    }
    return d_scratch;
}

void* Ctx::pinned_buf(size_t bytes) {
    if (bytes > pinned_bytes) {
        if (pinned) MTK_CUDA(cudaFreeHost(pinned));
        pinned = nullptr;
        MTK_CUDA(cudaMallocHost(&pinned, bytes));
        pinned_bytes = bytes;
    }
    return pinned;
}

void Ctx::check_flags() {
    if (!pinned_flags) MTK_CUDA(cudaMallocHost(&pinned_flags, 64));
    int* h = pinned_flags;
    MTK_CUDA(cudaMemcpyAsync(h, d_flags, sizeof(int), cudaMemcpyDeviceToHost, stream));
    MTK_CUDA(cudaStreamSynchronize(stream));
    const int f = *h;
    if (f) {
        MTK_CUDA(cudaMemsetAsync(d_flags, 0, sizeof(int), stream));
        MTK_CUDA(cudaStreamSynchronize(stream));
        if (f & kFlagBadLabel) fail(MTK_VALUE_ERROR, "label out of range [0, C)");
        fail(MTK_ERROR, "non-finite values produced on the device");
    }
}

cudaEvent_t Ctx::take_event() {
    if (!event_pool.empty()) {
        cudaEvent_t e = event_pool.back();
        event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    MTK_CUDA(cudaEventCreate(&e));
    return e;
}

void Ctx::collect_phases() {
    if (pending.empty()) return;
    MTK_CUDA(cudaStreamSynchronize(stream));
    for (auto& p : pending) {
        float ms = 0.f;
        MTK_CUDA(cudaEventElapsedTime(&ms, p.second.first, p.second.second));
        phase_ms[p.first] += ms;
        event_pool.push_back(p.second.first);
        event_pool.push_back(p.second.second);
    }
    pending.clear();
}

PhaseScope::PhaseScope(Ctx& ctx, int phase, int launches) : c(ctx), ph(phase), n(launches) {
    if (c.timing) {
        a = c.take_event();
        MTK_CUDA(cudaEventRecord(a, c.stream));
    }
}

PhaseScope::~PhaseScope() {
    if (!a) return;
    cudaEvent_t b = c.take_event();
    cudaEventRecord(b, c.stream);
    c.pending.push_back({ph, {a, b}});
    c.phase_launches[ph] += n;
}

inline void after_launch(Ctx& c, int n = 1) {
    c.launches += n;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) fail(MTK_ERROR, std::string("kernel launch: ") + cudaGetErrorString(e));
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return MTK_OK;
    } catch (const Failure& e) {
        tl_last_error = e.what();
        return e.status;
    } catch (const std::bad_alloc&) {
        tl_last_error = "host allocation failed";
        return MTK_ERROR;
    } catch (const std::exception& e) {
        tl_last_error = e.what();
        return MTK_ERROR;
    }
}

void need(bool ok, int status, const char* msg) {
    if (!ok) fail(status, msg);
}

}  // namespace mtk

using namespace mtk;

struct mtk_bank {
    mtk_ctx* ctx = nullptr;
    int G = 0, L = 0, n_heads = 1, n_mats = 0;
    std::vector<int> dims;
    std::vector<float*> W, b, gW, gb;
    bool keep_grads = false;
    int capB = 0;
    std::vector<float*> H;  // H[l], l in [1, L): post-ReLU output of layer l-1
    float* logits = nullptr;
    float* dZa = nullptr;
    float* dZb = nullptr;
    double* row_loss = nullptr;
    double* loss = nullptr;
    double* mmd = nullptr;
    double* beta = nullptr;
    float* gH = nullptr;
    double* mmd_part = nullptr;
    size_t mmd_part_bytes = 0;
    float* Xs = nullptr;
    int32_t* ys = nullptr;
    float* ws = nullptr;
    int stageB = 0;

    int fan_in(int i) const { return dims[i < L ? i : L - 1]; }
    int fan_out(int i) const { return dims[(i < L ? i : L - 1) + 1]; }
    int maxd() const {
        int m = 0;
        for (int v : dims) m = std::max(m, v);
        return m;
    }

    ~mtk_bank() {
        for (auto* p : W) cudaFree(p);
        for (auto* p : b) cudaFree(p);
        for (auto* p : gW) cudaFree(p);
        for (auto* p : gb) cudaFree(p);
        free_acts();
        cudaFree(Xs);
        cudaFree(ys);
        cudaFree(ws);
    }
    void free_acts() {
        for (auto* p : H) cudaFree(p);
        H.clear();
        cudaFree(logits);
        cudaFree(dZa);
        cudaFree(dZb);
        cudaFree(row_loss);
        cudaFree(gH);
        logits = dZa = dZb = gH = nullptr;
        row_loss = nullptr;
    }
    void ensure(int B) {
        if (B <= capB) return;
        MTK_CUDA(cudaStreamSynchronize(ctx->stream));
        free_acts();
        const size_t GB = (size_t)G * B;
        H.assign(L, nullptr);
        for (int l = 1; l < L; ++l) MTK_CUDA(cudaMalloc(&H[l], GB * dims[l] * sizeof(float)));
        MTK_CUDA(cudaMalloc(&logits, GB * dims[L] * sizeof(float)));
        MTK_CUDA(cudaMalloc(&dZa, GB * maxd() * sizeof(float)));
        MTK_CUDA(cudaMalloc(&dZb, GB * maxd() * sizeof(float)));
        MTK_CUDA(cudaMalloc(&row_loss, GB * sizeof(double)));
        if (L > 1) MTK_CUDA(cudaMalloc(&gH, GB * dims[L - 1] * sizeof(float)));
        capB = B;
    }
    void ensure_stage(int B) {
        if (B <= stageB) return;
        MTK_CUDA(cudaStreamSynchronize(ctx->stream));
        cudaFree(Xs);
        cudaFree(ys);
        cudaFree(ws);
        const size_t GB = (size_t)G * B;
        MTK_CUDA(cudaMalloc(&Xs, GB * dims[0] * sizeof(float)));
        MTK_CUDA(cudaMalloc(&ys, GB * sizeof(int32_t)));
        MTK_CUDA(cudaMalloc(&ws, GB * sizeof(float)));
        stageB = B;
    }
};

namespace {

// ---- GEMM builders (row range [r0, r0+rows) of every model) ----------------
Gemm fwd_gemm(mtk_bank& k, int mat, const float* in, int B, int r0, int rows, float* out,
              bool relu) {
    const int fi = k.fan_in(mat), fo = k.fan_out(mat);
    Gemm g;
    g.G = k.G;
    g.M = rows;
    g.N = fo;
    g.K = fi;
    g.A = in + (size_t)r0 * fi;
    g.a_gs = (long long)B * fi;
    g.a_ms = fi;
    g.a_ks = 1;
    g.B = k.W[mat];
    g.b_gs = (long long)fi * fo;
    g.b_ks = fo;
    g.b_ns = 1;
    g.C = out + (size_t)r0 * fo;
    g.c_gs = (long long)B * fo;
    g.ldc = fo;
    g.epi = relu ? Epi::kBiasRelu : Epi::kBias;
    g.bias = k.b[mat];
    g.bias_gs = fo;
    g.flags = k.ctx->d_flags;
    return g;
}

Gemm dx_gemm(mtk_bank& k, int mat, const float* dz, int B, int r0, int rows, float* out,
             const float* mask, const float* add) {
    const int fi = k.fan_in(mat), fo = k.fan_out(mat);
    Gemm g;
    g.G = k.G;
    g.M = rows;
    g.N = fi;
    g.K = fo;
    g.A = dz + (size_t)r0 * fo;
    g.a_gs = (long long)B * fo;
    g.a_ms = fo;
    g.a_ks = 1;
    g.B = k.W[mat];
    g.b_gs = (long long)fi * fo;
    g.b_ks = 1;
    g.b_ns = fo;
    g.C = out + (size_t)r0 * fi;
    g.c_gs = (long long)B * fi;
    g.ldc = fi;
    g.epi = Epi::kMask;
    g.mask = mask + (size_t)r0 * fi;
    g.add = add ? add + (size_t)r0 * fi : nullptr;
    g.flags = k.ctx->d_flags;
    return g;
}

Gemm dw_gemm(mtk_bank& k, int mat, const float* in, const float* dz, int B, int r0, int rows,
             float lr) {
    const int fi = k.fan_in(mat), fo = k.fan_out(mat);
    Gemm g;
    g.G = k.G;
    g.M = fi;
    g.N = fo;
    g.K = rows;
    g.A = in + (size_t)r0 * fi;
    g.a_gs = (long long)B * fi;
    g.a_ms = 1;
    g.a_ks = fi;
    g.B = dz + (size_t)r0 * fo;
    g.b_gs = (long long)B * fo;
    g.b_ks = fo;
    g.b_ns = 1;
    g.C = k.W[mat];
    g.c_gs = (long long)fi * fo;
    g.ldc = fo;
    g.epi = Epi::kSgd;
    g.lr = lr;
    g.grad_out = k.keep_grads ? k.gW[mat] : nullptr;
    g.flags = k.ctx->d_flags;
    return g;
}

void run_forward(mtk_bank& k, const float* X, int B, int head_all, int src_rows) {
    Ctx& c = *k.ctx;
    const float* h = X;
    for (int l = 0; l < k.L; ++l) {
        PhaseScope ph(c, kPhFwd, (l == k.L - 1 && head_all < 0) ? 2 : 1);
        if (l < k.L - 1) {
            launch_gemm(fwd_gemm(k, l, h, B, 0, B, k.H[l + 1], true), c.stream);
            after_launch(c);
            h = k.H[l + 1];
        } else if (head_all >= 0) {
            launch_gemm(fwd_gemm(k, l + head_all, h, B, 0, B, k.logits, false), c.stream);
            after_launch(c);
        } else {  // two heads split by rows
            launch_gemm(fwd_gemm(k, l, h, B, 0, src_rows, k.logits, false), c.stream);
            launch_gemm(fwd_gemm(k, l + 1, h, B, src_rows, B - src_rows, k.logits, false),
                        c.stream);
            after_launch(c, 2);
        }
    }
}

void train_step(mtk_bank& k, const mtk_step& s, double* loss_host, double* mmd_host) {
    Ctx& c = *k.ctx;
    const int B = s.B, L = k.L;
    need(B >= 1, MTK_SHAPE_ERROR, "train_step: B must be >= 1");
    need(s.X && s.y, MTK_VALUE_ERROR, "train_step: X and y are required");
    need(std::isfinite(s.lr), MTK_VALUE_ERROR, "train_step: lr must be finite");
    need(s.frozen_layers >= 0 && s.frozen_layers <= L, MTK_CONFIG_ERROR,
         "train_step: frozen_layers out of range");
    const bool two = k.n_heads == 2;
    const bool use_mmd = s.mmd_lambda > 0.0;
    if (two || use_mmd)
        need(s.src_rows > 0 && s.src_rows < B, MTK_SHAPE_ERROR,
             "train_step: src_rows must split the batch into two non-empty parts");
    need(!(two && use_mmd), MTK_CONFIG_ERROR, "train_step: MMD with two heads is not supported");
    need(!use_mmd || L >= 2, MTK_CONFIG_ERROR, "train_step: MMD needs a hidden layer");
    const int nb = s.mmd_nb > 0 ? s.mmd_nb : 5;
    need(nb <= 8, MTK_CONFIG_ERROR, "train_step: at most 8 MMD bandwidths");
    k.ensure(B);
    const int src = (two || use_mmd) ? s.src_rows : B;
    need(s.denom[0] >= 0 && s.denom[1] >= 0 && !std::isnan(s.denom[0]) && !std::isnan(s.denom[1]),
         MTK_VALUE_ERROR, "cross_entropy: denominator must be positive");
    const double d0 = s.denom[0] > 0 ? s.denom[0] : (double)(two ? src : B);
    const double d1 = s.denom[1] > 0 ? s.denom[1] : (double)(B - src);
    need(d0 > 0 && (!two || d1 > 0), MTK_VALUE_ERROR,
         "cross_entropy: denominator must be positive");
    const float lr = (float)s.lr;

    run_forward(k, s.X, B, two ? -1 : 0, src);

    CeArgs ce{k.G,      B,          k.dims[L], two ? src : B, k.logits, s.y, s.w,
              (float)(1.0 / d0), (float)(1.0 / (two ? d1 : d0)), k.dZa, k.row_loss, k.loss,
              c.d_flags};
    {
        PhaseScope ph(c, kPhCe, 2);
        launch_ce(ce, c.stream);
        after_launch(c, 2);
    }

    if (use_mmd) {
        MmdArgs a;
        a.G = k.G;
        a.m = src;
        a.n = B - src;
        a.d = k.dims[L - 1];
        a.Xs = k.H[L - 1];
        a.xs_gs = (long long)B * a.d;
        a.Xt = k.H[L - 1] + (size_t)src * a.d;
        a.xt_gs = a.xs_gs;
        a.nb = nb;
        for (int q = 0; q < 8; ++q)
            a.mult[q] = s.mmd_nb > 0 ? (float)s.mmd_mult[q] : a.mult[q];
        a.beta = k.beta;
        a.gXs = k.gH;
        a.gs_gs = a.xs_gs;
        a.gXt = k.gH + (size_t)src * a.d;
        a.gt_gs = a.xs_gs;
        a.grad_scale = (float)s.mmd_lambda;
        a.flags = c.d_flags;
        const int nblk = mmd_blocks_per_group(a);
        const size_t pbytes = (size_t)k.G * nblk * 3 * sizeof(double);
        if (pbytes > k.mmd_part_bytes) {
            MTK_CUDA(cudaStreamSynchronize(c.stream));
            cudaFree(k.mmd_part);
            MTK_CUDA(cudaMalloc(&k.mmd_part, pbytes));
            k.mmd_part_bytes = pbytes;
        }
        a.partial = k.mmd_part;
        const long long N = a.m + a.n;
        double* sc = c.scratch((size_t)k.G * ((N + 255) / 256) * (a.d + 1) * sizeof(double));
        {
            PhaseScope ph(c, kPhMmdBeta, 2);
            launch_mmd_beta(a, k.beta, sc, c.stream);
            after_launch(c, 2);
        }
        {
            PhaseScope ph(c, kPhMmdPairs, 1);
            launch_mmd_pairs(a, c.stream);
            after_launch(c, 1);
        }
        {
            PhaseScope ph(c, kPhOther, 1);
            launch_mmd_finish(a, k.mmd, nullptr, c.stream);
            after_launch(c, 1);
        }
    }

    // backward sweep, layer L-1 down to 0
    float* cur = k.dZa;
    float* nxt = k.dZb;
    for (int l = L - 1; l >= 0; --l) {
        const bool trainable = l >= s.frozen_layers;
        const bool need_dx = l > 0 && l > s.frozen_layers;
        const float* in = l == 0 ? s.X : k.H[l];
        const float* add = (l == L - 1 && use_mmd) ? k.gH : nullptr;
        if (need_dx) {
            PhaseScope ph(c, kPhDx, (l == L - 1 && two) ? 2 : 1);
            if (l == L - 1 && two) {
                launch_gemm(dx_gemm(k, l, cur, B, 0, src, nxt, k.H[l], nullptr), c.stream);
                launch_gemm(dx_gemm(k, l + 1, cur, B, src, B - src, nxt, k.H[l], nullptr),
                            c.stream);
                after_launch(c, 2);
            } else {
                launch_gemm(dx_gemm(k, l, cur, B, 0, B, nxt, k.H[l], add), c.stream);
                after_launch(c);
            }
        }
        if (trainable) {
            const int fo = k.dims[l + 1];
            const bool split = (l == L - 1 && two);
            {
                PhaseScope ph(c, kPhDw, split ? 2 : 1);
                if (split) {
                    launch_gemm(dw_gemm(k, l, in, cur, B, 0, src, lr), c.stream);
                    launch_gemm(dw_gemm(k, l + 1, in, cur, B, src, B - src, lr), c.stream);
                } else {
                    launch_gemm(dw_gemm(k, l, in, cur, B, 0, B, lr), c.stream);
                }
                after_launch(c, split ? 2 : 1);
            }
            PhaseScope ph(c, kPhBias, split ? 2 : 1);
            if (split) {
                launch_bias_sgd(k.G, src, fo, cur, (long long)B * fo, k.b[l], fo, lr,
                                k.keep_grads ? k.gb[l] : nullptr, c.d_flags, c.stream);
                launch_bias_sgd(k.G, B - src, fo, cur + (size_t)src * fo, (long long)B * fo,
                                k.b[l + 1], fo, lr, k.keep_grads ? k.gb[l + 1] : nullptr,
                                c.d_flags, c.stream);
            } else {
                launch_bias_sgd(k.G, B, fo, cur, (long long)B * fo, k.b[l], fo, lr,
                                k.keep_grads ? k.gb[l] : nullptr, c.d_flags, c.stream);
            }
            after_launch(c, split ? 2 : 1);
        }
        std::swap(cur, nxt);
    }

    if (loss_host || mmd_host) {
        double* h = static_cast<double*>(c.pinned_buf(2 * k.G * sizeof(double) + 64));
        if (loss_host)
            MTK_CUDA(cudaMemcpyAsync(h, k.loss, k.G * sizeof(double), cudaMemcpyDeviceToHost,
                                     c.stream));
        if (mmd_host && use_mmd)
            MTK_CUDA(cudaMemcpyAsync(h + k.G, k.mmd, k.G * sizeof(double),
                                     cudaMemcpyDeviceToHost, c.stream));
        c.check_flags();
        if (loss_host) std::memcpy(loss_host, h, k.G * sizeof(double));
        if (mmd_host) {
            if (use_mmd)
                std::memcpy(mmd_host, h + k.G, k.G * sizeof(double));
            else
                for (int g = 0; g < k.G; ++g) mmd_host[g] = 0.0;
        }
    }
}

void check_bank(mtk_bank* k) { need(k != nullptr, MTK_VALUE_ERROR, "null bank"); }
void check_model(mtk_bank* k, int model) {
    check_bank(k);
    need(model >= 0 && model < k->G, MTK_VALUE_ERROR, "model index out of range");
}

}  // namespace

extern "C" {

int mtk_version(void) { return 100; }

const char* mtk_last_error(void) { return tl_last_error.c_str(); }

int mtk_ctx_create(int device, void* stream, mtk_ctx** out) {
    return guard([&] {
        need(out != nullptr, MTK_VALUE_ERROR, "mtk_ctx_create: null out");
        int n = 0;
        MTK_CUDA(cudaGetDeviceCount(&n));
        need(device >= 0 && device < n, MTK_VALUE_ERROR, "mtk_ctx_create: no such device");
        MTK_CUDA(cudaSetDevice(device));
        std::unique_ptr<mtk_ctx> c(new mtk_ctx());
        c->device = device;
        // the context runs on exactly the stream it is given; NULL is the
        // legacy default stream (what torch uses unless told otherwise)
        c->stream = static_cast<cudaStream_t>(stream);
        MTK_CUDA(cudaMalloc(&c->d_flags, 64));
        MTK_CUDA(cudaMemsetAsync(c->d_flags, 0, 64, c->stream));
        c->pinned_buf(4096);
        *out = c.release();
    });
}

int mtk_ctx_destroy(mtk_ctx* c) {
    return guard([&] {
        if (!c) return;
        cudaStreamSynchronize(c->stream);
        cudaFree(c->d_flags);
        cudaFree(c->d_scratch);
        if (c->pinned) cudaFreeHost(c->pinned);
        if (c->pinned_flags) cudaFreeHost(c->pinned_flags);
        if (c->own_stream) cudaStreamDestroy(c->stream);
        delete c;
    });
}

int mtk_ctx_synchronize(mtk_ctx* c) {
    return guard([&] {
        need(c != nullptr, MTK_VALUE_ERROR, "null ctx");
        c->check_flags();
    });
}

int mtk_ctx_launch_count(mtk_ctx* c, uint64_t* out) {
    return guard([&] {
        need(c && out, MTK_VALUE_ERROR, "null argument");
        *out = c->launches;
    });
}

int mtk_ctx_set_timing(mtk_ctx* c, int on) {
    return guard([&] {
        need(c != nullptr, MTK_VALUE_ERROR, "null ctx");
        c->collect_phases();
        c->timing = on != 0;
    });
}

int mtk_ctx_phase_times(mtk_ctx* c, double* ms_host, uint64_t* launches_host) {
    return guard([&] {
        need(c != nullptr, MTK_VALUE_ERROR, "null ctx");
        c->collect_phases();
        for (int i = 0; i < kNumPhases; ++i) {
            if (ms_host) ms_host[i] = c->phase_ms[i];
            if (launches_host) launches_host[i] = c->phase_launches[i];
            c->phase_ms[i] = 0.0;
            c->phase_launches[i] = 0;
        }
    });
}

int mtk_bank_create(mtk_ctx* c, int G, int n_layers, const int* dims, int n_heads,
                    mtk_bank** out) {
    return guard([&] {
        need(c && dims && out, MTK_VALUE_ERROR, "mtk_bank_create: null argument");
        need(G >= 1 && n_layers >= 1, MTK_SHAPE_ERROR, "mtk_bank_create: zero dimension");
        need(n_heads == 1 || n_heads == 2, MTK_CONFIG_ERROR, "mtk_bank_create: n_heads is 1 or 2");
        need(n_heads == 1 || n_layers >= 2, MTK_CONFIG_ERROR,
             "mtk_bank_create: two heads need a shared trunk");
        for (int i = 0; i <= n_layers; ++i)
            need(dims[i] >= 1, MTK_SHAPE_ERROR, "mtk_bank_create: zero dimension in dims");
        MTK_CUDA(cudaSetDevice(c->device));
        std::unique_ptr<mtk_bank> k(new mtk_bank());
        k->ctx = c;
        k->G = G;
        k->L = n_layers;
        k->n_heads = n_heads;
        k->dims.assign(dims, dims + n_layers + 1);
        k->n_mats = n_layers + n_heads - 1;
        for (int i = 0; i < k->n_mats; ++i) {
            float *w = nullptr, *bb = nullptr;
            MTK_CUDA(cudaMalloc(&w, (size_t)G * k->fan_in(i) * k->fan_out(i) * sizeof(float)));
            MTK_CUDA(cudaMalloc(&bb, (size_t)G * k->fan_out(i) * sizeof(float)));
            MTK_CUDA(cudaMemsetAsync(w, 0, (size_t)G * k->fan_in(i) * k->fan_out(i) * 4, c->stream));
            MTK_CUDA(cudaMemsetAsync(bb, 0, (size_t)G * k->fan_out(i) * 4, c->stream));
            k->W.push_back(w);
            k->b.push_back(bb);
        }
        MTK_CUDA(cudaMalloc(&k->loss, G * sizeof(double)));
        MTK_CUDA(cudaMalloc(&k->mmd, G * sizeof(double)));
        MTK_CUDA(cudaMalloc(&k->beta, G * sizeof(double)));
        MTK_CUDA(cudaStreamSynchronize(c->stream));
        *out = k.release();
    });
}

int mtk_bank_destroy(mtk_bank* k) {
    return guard([&] {
        if (!k) return;
        cudaStreamSynchronize(k->ctx->stream);
        delete k;
    });
}

int mtk_bank_set_params(mtk_bank* k, int model, const double* const* W, const double* const* b) {
    return guard([&] {
        check_model(k, model);
        need(W && b, MTK_VALUE_ERROR, "set_params: null arrays");
        std::vector<float> tmp;
        for (int i = 0; i < k->n_mats; ++i) {
            const size_t nw = (size_t)k->fan_in(i) * k->fan_out(i), nbias = k->fan_out(i);
            need(W[i] && b[i], MTK_VALUE_ERROR, "set_params: null matrix");
            tmp.assign(W[i], W[i] + nw);
            MTK_CUDA(cudaMemcpy(k->W[i] + model * nw, tmp.data(), nw * 4, cudaMemcpyHostToDevice));
            tmp.assign(b[i], b[i] + nbias);
            MTK_CUDA(cudaMemcpy(k->b[i] + model * nbias, tmp.data(), nbias * 4,
                                cudaMemcpyHostToDevice));
        }
    });
}

int mtk_bank_get_params(mtk_bank* k, int model, double* const* W, double* const* b) {
    return guard([&] {
        check_model(k, model);
        MTK_CUDA(cudaStreamSynchronize(k->ctx->stream));
        std::vector<float> tmp;
        for (int i = 0; i < k->n_mats; ++i) {
            const size_t nw = (size_t)k->fan_in(i) * k->fan_out(i), nbias = k->fan_out(i);
            if (W && W[i]) {
                tmp.resize(nw);
                MTK_CUDA(cudaMemcpy(tmp.data(), k->W[i] + model * nw, nw * 4,
                                    cudaMemcpyDeviceToHost));
                for (size_t j = 0; j < nw; ++j) W[i][j] = tmp[j];
            }
            if (b && b[i]) {
                tmp.resize(nbias);
                MTK_CUDA(cudaMemcpy(tmp.data(), k->b[i] + model * nbias, nbias * 4,
                                    cudaMemcpyDeviceToHost));
                for (size_t j = 0; j < nbias; ++j) b[i][j] = tmp[j];
            }
        }
    });
}

int mtk_bank_init_params(mtk_bank* k, int model, mtk_rng* r) {
    return guard([&] {
        check_model(k, model);
        need(r != nullptr, MTK_VALUE_ERROR, "init_params: null rng");
        std::vector<std::vector<double>> W(k->n_mats), b(k->n_mats);
        std::vector<const double*> pw, pb;
        for (int i = 0; i < k->n_mats; ++i) {
            const double lim = 1.0 / std::sqrt((double)k->fan_in(i));
            W[i].resize((size_t)k->fan_in(i) * k->fan_out(i));
            for (double& v : W[i]) v = mtk_rng_uniform(r, -lim, lim);
            b[i].assign(k->fan_out(i), 0.0);
            pw.push_back(W[i].data());
            pb.push_back(b[i].data());
        }
        const int st = mtk_bank_set_params(k, model, pw.data(), pb.data());
        if (st) fail(st, tl_last_error);
    });
}

int mtk_bank_param_device(mtk_bank* k, int mat, float** W, float** b) {
    return guard([&] {
        check_bank(k);
        need(mat >= 0 && mat < k->n_mats, MTK_VALUE_ERROR, "param_device: bad matrix index");
        if (W) *W = k->W[mat];
        if (b) *b = k->b[mat];
    });
}

int mtk_bank_forward(mtk_bank* k, const float* X, int B, int head, float* logits,
                     float* hidden_last) {
    return guard([&] {
        check_bank(k);
        need(X && logits, MTK_VALUE_ERROR, "forward: null argument");
        need(B >= 1, MTK_SHAPE_ERROR, "forward: B must be >= 1");
        need(head >= 0 && head < k->n_heads, MTK_VALUE_ERROR, "forward: bad head index");
        k->ensure(B);
        Ctx& c = *k->ctx;
        run_forward(*k, X, B, head, 0);
        const size_t GB = (size_t)k->G * B;
        MTK_CUDA(cudaMemcpyAsync(logits, k->logits, GB * k->dims[k->L] * 4,
                                 cudaMemcpyDeviceToDevice, c.stream));
        if (hidden_last && k->L > 1)
            MTK_CUDA(cudaMemcpyAsync(hidden_last, k->H[k->L - 1], GB * k->dims[k->L - 1] * 4,
                                     cudaMemcpyDeviceToDevice, c.stream));
    });
}

int mtk_bank_train_step(mtk_bank* k, const mtk_step* s, double* loss_host, double* mmd_host) {
    return guard([&] {
        check_bank(k);
        need(s != nullptr, MTK_VALUE_ERROR, "train_step: null step");
        train_step(*k, *s, loss_host, mmd_host);
    });
}

int mtk_bank_train_step_host(mtk_bank* k, const mtk_step* s, const float* X_host,
                             const int32_t* y_host, const float* w_host, double* loss_host,
                             double* mmd_host) {
    return guard([&] {
        check_bank(k);
        need(s && X_host && y_host, MTK_VALUE_ERROR, "train_step_host: null argument");
        need(s->B >= 1, MTK_SHAPE_ERROR, "train_step_host: B must be >= 1");
        k->ensure_stage(s->B);
        Ctx& c = *k->ctx;
        const size_t GB = (size_t)k->G * s->B;
        MTK_CUDA(cudaMemcpyAsync(k->Xs, X_host, GB * k->dims[0] * 4, cudaMemcpyHostToDevice,
                                 c.stream));
        MTK_CUDA(cudaMemcpyAsync(k->ys, y_host, GB * 4, cudaMemcpyHostToDevice, c.stream));
        if (w_host)
            MTK_CUDA(cudaMemcpyAsync(k->ws, w_host, GB * 4, cudaMemcpyHostToDevice, c.stream));
        mtk_step d = *s;
        d.X = k->Xs;
        d.y = k->ys;
        d.w = w_host ? k->ws : nullptr;
        train_step(*k, d, loss_host, mmd_host);
    });
}

int mtk_bank_set_keep_grads(mtk_bank* k, int on) {
    return guard([&] {
        check_bank(k);
        k->keep_grads = on != 0;
        if (k->keep_grads && k->gW.empty()) {
            for (int i = 0; i < k->n_mats; ++i) {
                float *w = nullptr, *bb = nullptr;
                MTK_CUDA(cudaMalloc(&w, (size_t)k->G * k->fan_in(i) * k->fan_out(i) * 4));
                MTK_CUDA(cudaMalloc(&bb, (size_t)k->G * k->fan_out(i) * 4));
                MTK_CUDA(cudaMemset(w, 0, (size_t)k->G * k->fan_in(i) * k->fan_out(i) * 4));
                MTK_CUDA(cudaMemset(bb, 0, (size_t)k->G * k->fan_out(i) * 4));
                k->gW.push_back(w);
                k->gb.push_back(bb);
            }
        }
    });
}

int mtk_bank_get_grads(mtk_bank* k, int model, double* const* dW, double* const* db) {
    return guard([&] {
        check_model(k, model);
        need(!k->gW.empty(), MTK_CONFIG_ERROR, "get_grads: call mtk_bank_set_keep_grads first");
        MTK_CUDA(cudaStreamSynchronize(k->ctx->stream));
        std::vector<float> tmp;
        for (int i = 0; i < k->n_mats; ++i) {
            const size_t nw = (size_t)k->fan_in(i) * k->fan_out(i), nbias = k->fan_out(i);
            if (dW && dW[i]) {
                tmp.resize(nw);
                MTK_CUDA(cudaMemcpy(tmp.data(), k->gW[i] + model * nw, nw * 4,
                                    cudaMemcpyDeviceToHost));
                for (size_t j = 0; j < nw; ++j) dW[i][j] = tmp[j];
            }
            if (db && db[i]) {
                tmp.resize(nbias);
                MTK_CUDA(cudaMemcpy(tmp.data(), k->gb[i] + model * nbias, nbias * 4,
                                    cudaMemcpyDeviceToHost));
                for (size_t j = 0; j < nbias; ++j) db[i][j] = tmp[j];
            }
        }
    });
}

// ---- MMD -------------------------------------------------------------------
static MmdArgs mmd_args(mtk_ctx* c, const float* Xs, int64_t m, const float* Xt, int64_t n, int d,
                        const double* mult, int nb) {
    need(c && Xs && Xt, MTK_VALUE_ERROR, "mmd: null argument");
    need(m >= 1 && n >= 1 && d >= 1, MTK_SHAPE_ERROR, "mmd: zero dimension");
    need(nb >= 0 && nb <= 8, MTK_CONFIG_ERROR, "mmd: at most 8 bandwidths");
    MmdArgs a;
    a.m = m;
    a.n = n;
    a.d = d;
    a.Xs = Xs;
    a.Xt = Xt;
    if (nb > 0) {
        need(mult != nullptr, MTK_VALUE_ERROR, "mmd: null bandwidth multipliers");
        a.nb = nb;
        for (int q = 0; q < nb; ++q) {
            need(mult[q] > 0, MTK_VALUE_ERROR, "mmd: bandwidth multipliers must be positive");
            a.mult[q] = (float)mult[q];
        }
    }
    a.flags = c->d_flags;
    return a;
}

int mtk_mmd_beta(mtk_ctx* c, const float* Xs, int64_t m, const float* Xt, int64_t n, int d,
                 double* beta_host) {
    return guard([&] {
        MmdArgs a = mmd_args(c, Xs, m, Xt, n, d, nullptr, 0);
        const long long N = m + n;
        const size_t part = (size_t)((N + 255) / 256) * (d + 1) * sizeof(double);
        double* sc = c->scratch(part + 64);
        double* beta_d = sc + part / sizeof(double);
        launch_mmd_beta(a, beta_d, sc, c->stream);
        after_launch(*c, 2);
        double* h = static_cast<double*>(c->pinned_buf(4096));
        MTK_CUDA(cudaMemcpyAsync(h, beta_d, 8, cudaMemcpyDeviceToHost, c->stream));
        c->check_flags();
        *beta_host = h[0];
    });
}

static void mmd_run(mtk_ctx* c, MmdArgs& a, double beta, bool want_value, double* value_host,
                    double* beta_host, double* sums_host) {
    const long long N = a.m + a.n;
    const int nblk = mmd_blocks_per_group(a);
    const size_t part_beta = (size_t)((N + 255) / 256) * (a.d + 1) * sizeof(double);
    const size_t part_pairs = (size_t)nblk * 3 * sizeof(double);
    const size_t bytes = part_beta + part_pairs + 64 * sizeof(double);
    double* sc = c->scratch(bytes);
    double* beta_d = sc;
    double* out_d = sc + 8;
    double* sums_d = sc + 16;
    double* part_d = sc + 64;
    double* bscratch = part_d + nblk * 3;
    if (beta > 0) {
        MTK_CUDA(cudaMemcpyAsync(beta_d, &beta, sizeof(double), cudaMemcpyHostToDevice, c->stream));
    } else {
        launch_mmd_beta(a, beta_d, bscratch, c->stream);
        after_launch(*c, 2);
    }
    a.beta = beta_d;
    a.partial = part_d;
    launch_mmd_pairs(a, c->stream);
    launch_mmd_finish(a, want_value ? out_d : nullptr, sums_d, c->stream);
    after_launch(*c, 2);
    double* h = static_cast<double*>(c->pinned_buf(4096));
    MTK_CUDA(cudaMemcpyAsync(h, sc, 24 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    c->check_flags();
    need(std::isfinite(h[0]) && h[0] > 0, MTK_VALUE_ERROR, "mmd: bandwidth must be positive");
    if (beta_host) *beta_host = h[0];
    if (value_host) *value_host = h[8];
    if (sums_host)
        for (int q = 0; q < 3; ++q) sums_host[q] = h[16 + q];
}

int mtk_mmd_gaussian(mtk_ctx* c, const float* Xs, int64_t m, const float* Xt, int64_t n, int d,
                     const double* mult, int nb, double beta, double* value_host,
                     double* beta_host, float* gXs, float* gXt) {
    return guard([&] {
        MmdArgs a = mmd_args(c, Xs, m, Xt, n, d, mult, nb);
        need(value_host != nullptr, MTK_VALUE_ERROR, "mmd: null value");
        a.gXs = gXs;
        a.gXt = gXt;
        mmd_run(c, a, beta, true, value_host, beta_host, nullptr);
    });
}

int mtk_mmd_gaussian_rows(mtk_ctx* c, const float* Xs, int64_t m, const float* Xt, int64_t n,
                          int d, const double* mult, int nb, double beta, int64_t row_begin,
                          int64_t row_end, double* partial_host, float* gXs, float* gXt) {
    return guard([&] {
        MmdArgs a = mmd_args(c, Xs, m, Xt, n, d, mult, nb);
        need(beta > 0, MTK_VALUE_ERROR, "mmd_rows: beta must be given (> 0)");
        need(partial_host != nullptr, MTK_VALUE_ERROR, "mmd_rows: null partial");
        need(row_begin >= 0 && row_begin <= row_end && row_end <= m + n, MTK_SHAPE_ERROR,
             "mmd_rows: bad row range");
        a.row_begin = row_begin;
        a.row_end = row_end;
        a.gXs = gXs;
        a.gXt = gXt;
        if (row_end == row_begin) {
            partial_host[0] = partial_host[1] = partial_host[2] = 0.0;
            return;
        }
        mmd_run(c, a, beta, false, nullptr, nullptr, partial_host);
    });
}

// ---- attack stage ----------------------------------------------------------
int mtk_softmax(mtk_ctx* c, const float* logits, int64_t rows, int C, float* probs) {
    return guard([&] {
        need(c && logits && probs, MTK_VALUE_ERROR, "softmax: null argument");
        need(rows >= 1 && C >= 1, MTK_SHAPE_ERROR, "softmax: zero dimension");
        launch_softmax(logits, rows, C, probs, c->stream);
        after_launch(*c);
    });
}

int mtk_posterior_features(mtk_ctx* c, const float* logits, int64_t rows, int C, int k,
                           const int32_t* labels, float* feats) {
    return guard([&] {
        need(c && logits && feats, MTK_VALUE_ERROR, "features: null argument");
        need(rows >= 1 && C >= 1, MTK_SHAPE_ERROR, "features: zero dimension");
        need(k >= 1 && k <= C, MTK_VALUE_ERROR, "features: k must be in [1, C]");
        launch_features(logits, rows, C, k, labels, feats, c->d_flags, c->stream);
        after_launch(*c);
    });
}

int mtk_posterior_column(mtk_ctx* c, const float* logits, int64_t rows, int C, int col,
                         float* out) {
    return guard([&] {
        need(c && logits && out, MTK_VALUE_ERROR, "posterior_column: null argument");
        need(rows >= 1 && C >= 1, MTK_SHAPE_ERROR, "posterior_column: zero dimension");
        need(col >= 0 && col < C, MTK_VALUE_ERROR, "posterior_column: column out of range");
        launch_column(logits, rows, C, col, out, c->stream);
        after_launch(*c);
    });
}

int mtk_auc(mtk_ctx* c, const float* scores, const uint8_t* labels, int64_t n, double* auc_host,
            double* acc_host) {
    return guard([&] {
        need(c && scores && labels, MTK_VALUE_ERROR, "auc: null argument");
        need(n >= 1, MTK_SHAPE_ERROR, "auc: zero rows");
        auc_device(*c, scores, labels, n, auc_host, acc_host);
        c->check_flags();
    });
}

int mtk_diag_gemm_tf32x3(mtk_ctx* c, int a_mn, int b_mn, int G, int M, int N, int K,
                         const float* A, const float* B, float* Cm) {
    return guard([&] {
        need(c && A && B && Cm, MTK_VALUE_ERROR, "diag_gemm: null argument");
        need(G >= 1 && M >= 1 && N >= 1 && K >= 1, MTK_SHAPE_ERROR, "diag_gemm: zero dimension");
        const size_t na = (size_t)G * M * K, nb = (size_t)G * K * N;
        float* buf = nullptr;
        MTK_CUDA(cudaMallocAsync(&buf, (2 * na + 2 * nb + 64) * sizeof(float), c->stream));
        float* ahi = buf;
        float* alo = ahi + na;
        float* bhi = alo + na;
        float* blo = bhi + nb;
        launch_split(A, ahi, alo, (long long)na, c->stream);
        launch_split(B, bhi, blo, (long long)nb, c->stream);
        after_launch(*c, 2);
        UmmaGemm u;
        u.G = G;
        u.M = M;
        u.N = N;
        u.K = K;
        u.a_mn = a_mn;
        u.b_mn = b_mn;
        u.a_hi = ahi;
        u.a_lo = alo;
        u.a_rs = a_mn ? M : K;
        u.a_gs = (long long)M * K;
        u.b_hi = bhi;
        u.b_lo = blo;
        u.b_rs = b_mn ? N : K;
        u.b_gs = (long long)K * N;
        u.epi = Epi::kStore;
        u.C = Cm;
        u.c_gs = (long long)M * N;
        u.ldc = N;
        u.flags = c->d_flags;
        if (getenv("MTK_UMMA_DEBUG")) u.dbg = reinterpret_cast<float*>(strtoull(getenv("MTK_UMMA_DEBUG"), nullptr, 0));
        launch_umma(u, c->stream);
        after_launch(*c);
        MTK_CUDA(cudaFreeAsync(buf, c->stream));
        c->check_flags();
    });
}

}  // extern "C"
