// bank.cu -- the grouped shadow-model bank (C ABI mtk_bank_*).
//
// One bank step runs, for all G models at once, the reference composition
//   forward : matmul -> add_bias -> relu ... -> cross_entropy_weighted
//             (tape.hpp:225-290, 204-221, 342-352, 475-520)
//   backward: Tape::backward reverse sweep (tape.hpp:870-886)
//   update  : optimizer_step SGD (optim.hpp:46-48)
// as a fixed schedule of fused kernels (no device tape):
//   per layer    FWD gemm (+bias, +ReLU)             -> H[l+1]
//   head         CE (softmax, loss, dlogits)         -> dZ_{L-1}
//   [mapping]    MMD beta, pairs, finish             -> lambda * dMMD/dH_{L-1}
//   per layer    DX gemm (+inject, *ReLU mask) then DW gemm (+SGD) + bias SGD
// Layers whose in/out widths are >= 32 and multiples of 4 ("tc layers") run
// their three GEMMs on the tcgen05 3xTF32 path (k_umma.cu); narrow layers
// (the 10-class head, the 3-feature attack input) use the SIMT kernel.
//
// HBM layout per bank (row-major fp32; the tensor-core kernels split
// operands into tf32 hi/lo on chip, so nothing else is stored):
//   W[i]  [G, fan_in, fan_out];  b[i] [G, fan_out]
//   H[l]  [G, B, dims[l]] post-ReLU activations (ReLU mask = H > 0)
//   dZ    two ping-pong [G, B, max dim] gradient buffers
#include <cerrno>
#include <cmath>
#include <functional>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "internal.h"

using namespace mtk;

namespace {

// one device fp32 array (kept as a struct so the layer plumbing stays typed)
struct Plane3 {
    float* f = nullptr;
    // post-ReLU activations only: the ReLU mask as bits, [G][rows][ceil(cols / 32)]
    // words (bit j of word w = column 32 w + j > 0), written by the tcgen05
    // FWD epilogue and read by the DX epilogue instead of the fp32 plane
    uint32_t* bits = nullptr;
};

void free3(Plane3& p, bool own_f = true) {
    if (own_f) cudaFree(p.f);
    cudaFree(p.bits);
    p = Plane3{};
}
inline int mask_words(int cols) { return (cols + 31) / 32; }

void alloc3(Plane3& p, size_t n) { MTK_CUDA(cudaMalloc(&p.f, n * sizeof(float))); }

}  // namespace

struct mtk_bank {
    mtk_ctx* ctx = nullptr;
    int G = 0, L = 0, n_heads = 1, n_mats = 0;
    std::vector<int> dims;
    std::vector<bool> tc;  // per layer: tensor-core path
    std::vector<Plane3> W;
    std::vector<float*> b, gW, gb;
    std::vector<float*> mW, vW, mb, vb;  // Adam moments (allocated on first Adam step)
    unsigned long long adam_t = 0;       // OptimizerState::step (optim.hpp:41)
    float* adam_g = nullptr;             // gradient scratch for Adam on the GEMM paths
    size_t adam_g_elems = 0;
    float* adam_grad(int mat) {
        const size_t n = (size_t)G * fan_in(mat) * fan_out(mat);
        if (n > adam_g_elems) {
            MTK_CUDA(cudaStreamSynchronize(ctx->stream));
            cudaFree(adam_g);
            MTK_CUDA(cudaMalloc(&adam_g, n * sizeof(float)));
            adam_g_elems = n;
        }
        return adam_g;
    }
    bool keep_grads = false;
    bool no_update = false;  // compute_grads: store gradients, never write a parameter
    int capB = 0;
    std::vector<Plane3> H;    // H[l], l in [1, L)
    Plane3 dZ[2];
    float* logits = nullptr;
    double* row_loss = nullptr;
    double* loss = nullptr;
    double* mmd = nullptr;
    double* beta = nullptr;
    float* gH = nullptr;
    // [G][ceil(B/32)][max dim] bias-gradient partials: layer j's from the
    // producer of its dZ (CE, a DX epilogue, the fused MMD gradient GEMM) in
    // colsum[j % 3], so a bias update on the side stream can lag two layers
    float* colsum[3] = {nullptr, nullptr, nullptr};
    Plane3 dlog;              // dlogits [G][B][C] (own buffer: the side-stream head dW reads it late)
    double* loss_part = nullptr;  // [G][ceil(B/32)] CE loss partials
    double* mmd_part = nullptr;
    size_t mmd_part_bytes = 0;
    // skinny dW partial sums: [0] for the main stream, [1] for the side stream
    // (the head dW there can overlap a narrow-input layer's dW on the main stream)
    float* head_scratch[2] = {nullptr, nullptr};
    size_t head_scratch_bytes[2] = {0, 0};
    void* mmd_z = nullptr;     // tf32 planes + norms of the MMD sample (tc path)
    size_t mmd_z_bytes = 0;
    bool tc_mmd = true;
    float* Xs = nullptr;
    int32_t* ys = nullptr;
    float* ws = nullptr;
    int stageB = 0;
    // pipelined host steps: two staging slots filled on a copy stream
    struct Slot {
        float* X = nullptr;
        int32_t* y = nullptr;
        float* w = nullptr;
        double* res = nullptr;  // pinned [2G]: loss, mmd
        cudaEvent_t copied = nullptr, consumed = nullptr, done = nullptr;
        bool mmd = false;
    } slot[2];
    int slotB = 0, next_slot = 0, last_slot = -1;
    cudaStream_t copy_stream = nullptr;

    int layer_of(int i) const { return i < L ? i : L - 1; }
    int fan_in(int i) const { return dims[layer_of(i)]; }
    int fan_out(int i) const { return dims[layer_of(i) + 1]; }
    bool any_tc() const {
        for (bool t : tc)
            if (t) return true;
        return false;
    }
    int maxd() const {
        int m = 0;
        for (int v : dims) m = std::max(m, v);
        return m;
    }

    ~mtk_bank() {
        for (auto& p : W) free3(p);
        for (auto* p : b) cudaFree(p);
        for (auto* p : gW) cudaFree(p);
        for (auto* p : gb) cudaFree(p);
        for (auto* p : mW) cudaFree(p);
        for (auto* p : vW) cudaFree(p);
        for (auto* p : mb) cudaFree(p);
        for (auto* p : vb) cudaFree(p);
        cudaFree(adam_g);
        free_acts();
        cudaFree(loss);
        cudaFree(mmd);
        cudaFree(beta);
        cudaFree(mmd_part);
        cudaFree(mmd_z);
        cudaFree(head_scratch[0]);
        cudaFree(head_scratch[1]);
        cudaFree(Xs);
        cudaFree(ys);
        cudaFree(ws);
        free_slots();
        if (copy_stream) cudaStreamDestroy(copy_stream);
        for (auto& sl : slot) {
            if (sl.copied) cudaEventDestroy(sl.copied);
            if (sl.consumed) cudaEventDestroy(sl.consumed);
            if (sl.done) cudaEventDestroy(sl.done);
            if (sl.res) cudaFreeHost(sl.res);
        }
    }
    void ensure_adam() {
        if (!mW.empty()) return;
        for (int i = 0; i < n_mats; ++i) {
            const size_t nw = (size_t)G * fan_in(i) * fan_out(i), nb = (size_t)G * fan_out(i);
            float *a, *b2, *c2, *d2;
            MTK_CUDA(cudaMalloc(&a, nw * sizeof(float)));
            MTK_CUDA(cudaMalloc(&b2, nw * sizeof(float)));
            MTK_CUDA(cudaMalloc(&c2, nb * sizeof(float)));
            MTK_CUDA(cudaMalloc(&d2, nb * sizeof(float)));
            mW.push_back(a);
            vW.push_back(b2);
            mb.push_back(c2);
            vb.push_back(d2);
        }
        reset_adam();
    }
    void reset_adam() {
        for (int i = 0; i < (int)mW.size(); ++i) {
            const size_t nw = (size_t)G * fan_in(i) * fan_out(i), nb = (size_t)G * fan_out(i);
            MTK_CUDA(cudaMemsetAsync(mW[i], 0, nw * sizeof(float), ctx->stream));
            MTK_CUDA(cudaMemsetAsync(vW[i], 0, nw * sizeof(float), ctx->stream));
            MTK_CUDA(cudaMemsetAsync(mb[i], 0, nb * sizeof(float), ctx->stream));
            MTK_CUDA(cudaMemsetAsync(vb[i], 0, nb * sizeof(float), ctx->stream));
        }
        adam_t = 0;
    }
    void free_slots() {
        for (auto& sl : slot) {
            cudaFree(sl.X);
            cudaFree(sl.y);
            cudaFree(sl.w);
            sl.X = nullptr;
            sl.y = nullptr;
            sl.w = nullptr;
        }
    }
    void ensure_slots(int B) {
        if (!copy_stream) {
            MTK_CUDA(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
            for (auto& sl : slot) {
                MTK_CUDA(cudaEventCreateWithFlags(&sl.copied, cudaEventDisableTiming));
                MTK_CUDA(cudaEventCreateWithFlags(&sl.consumed, cudaEventDisableTiming));
                MTK_CUDA(cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming));
                MTK_CUDA(cudaMallocHost(&sl.res, 2 * G * sizeof(double)));
            }
        }
        if (B <= slotB) return;
        MTK_CUDA(cudaStreamSynchronize(ctx->stream));
        MTK_CUDA(cudaStreamSynchronize(copy_stream));
        free_slots();
        const size_t GB = (size_t)G * B;
        for (auto& sl : slot) {
            MTK_CUDA(cudaMalloc(&sl.X, GB * dims[0] * sizeof(float)));
            MTK_CUDA(cudaMalloc(&sl.y, GB * sizeof(int32_t)));
            MTK_CUDA(cudaMalloc(&sl.w, GB * sizeof(float)));
        }
        slotB = B;
    }
    void free_acts() {
        for (auto& p : H) free3(p);
        H.clear();
        free3(dZ[0]);
        free3(dZ[1]);
        cudaFree(logits);
        cudaFree(row_loss);
        cudaFree(gH);
        for (auto& cs : colsum) {
            cudaFree(cs);
            cs = nullptr;
        }
        free3(dlog);
        cudaFree(loss_part);
        loss_part = nullptr;
        logits = nullptr;
        gH = nullptr;
        row_loss = nullptr;
    }
    void ensure(int B) {
        if (B <= capB) return;
        MTK_CUDA(cudaStreamSynchronize(ctx->stream));
        free_acts();
        const size_t GB = (size_t)G * B;
        H.assign(L, Plane3{});
        for (int l = 1; l < L; ++l) {
            alloc3(H[l], GB * dims[l]);
            // the mask bits, when both the FWD producing H[l] and the DX reading it are tcgen05 GEMMs
            const char* nb = getenv("MTK_NO_MASK_BITS");  // A/B at bank allocation
            // (and for the last hidden layer: the MMD gradient GEMM's fused head DX reads them)
            if (tc[l - 1] && (tc[l] || l == L - 1) && !(nb && nb[0] == '1'))
                MTK_CUDA(cudaMalloc(&H[l].bits, GB * mask_words(dims[l]) * sizeof(uint32_t)));
        }
        for (auto& z : dZ) alloc3(z, GB * maxd());
        MTK_CUDA(cudaMalloc(&logits, GB * dims[L] * sizeof(float)));
        MTK_CUDA(cudaMalloc(&row_loss, GB * sizeof(double)));
        if (L > 1) MTK_CUDA(cudaMalloc(&gH, GB * dims[L - 1] * sizeof(float)));
        for (auto& cs : colsum) MTK_CUDA(cudaMalloc(&cs, (size_t)G * ((B + 31) / 32) * maxd() * sizeof(float)));
        alloc3(dlog, GB * dims[L]);
        MTK_CUDA(cudaMalloc(&loss_part, (size_t)G * ((B + 31) / 32) * sizeof(double)));
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

// ---- GEMM dispatch over row range [r0, r0+rows) of every model -------------
// FWD: out[r, n] = sum_k in[r, k] W[k, n] (+bias, ReLU)
// returns true when `ce` (optional) was computed by the same launch (skinny head)
bool gemm_fwd(mtk_bank& k, int mat, const Plane3& in, int B, int r0, int rows, const Plane3& out,
              bool relu, const CeArgs* ce = nullptr) {
    Ctx& c = *k.ctx;
    const int fi = k.fan_in(mat), fo = k.fan_out(mat);
    if (k.tc[k.layer_of(mat)]) {
        UmmaGemm u;
        u.G = k.G;
        u.M = rows;
        u.N = fo;
        u.K = fi;
        u.a_mn = 0;
        u.a = in.f + (size_t)r0 * fi;
        u.a_rs = fi;
        u.a_gs = (long long)B * fi;
        u.b_mn = 1;
        u.b = k.W[mat].f;
        u.b_rs = fo;
        u.b_gs = (long long)fi * fo;
        u.epi = relu ? Epi::kBiasRelu : Epi::kBias;
        u.C = out.f + (size_t)r0 * fo;
        u.c_gs = (long long)B * fo;
        u.ldc = fo;
        u.bias = k.b[mat];
        u.bias_gs = fo;
        if (relu && out.bits) {
            const int wd = mask_words(fo);
            u.mbits = out.bits + (size_t)r0 * wd;
            u.mb_gs = (long long)B * wd;
            u.mb_ld = wd;
        }
        u.flags = c.d_flags;
        launch_umma(u, c.stream);
    } else if (head_fwd_ok(fi, fo)) {
        HeadFwd h;
        h.G = k.G;
        h.rows = rows;
        h.K = fi;
        h.N = fo;
        h.A = in.f + (size_t)r0 * fi;
        h.a_gs = (long long)B * fi;
        h.lda = fi;
        h.W = k.W[mat].f;
        h.w_gs = (long long)fi * fo;
        h.bias = k.b[mat];
        h.bias_gs = fo;
        h.C = out.f + (size_t)r0 * fo;
        h.c_gs = (long long)B * fo;
        h.ldc = fo;
        h.relu = relu ? 1 : 0;
        h.flags = c.d_flags;
        h.ce = (ce && r0 == 0 && rows == B && !relu) ? ce : nullptr;
        launch_head_fwd(h, c.stream);
        return h.ce != nullptr;
    } else {
        Gemm g;
        g.G = k.G;
        g.M = rows;
        g.N = fo;
        g.K = fi;
        g.A = in.f + (size_t)r0 * fi;
        g.a_gs = (long long)B * fi;
        g.a_ms = fi;
        g.a_ks = 1;
        g.B = k.W[mat].f;
        g.b_gs = (long long)fi * fo;
        g.b_ks = fo;
        g.b_ns = 1;
        g.C = out.f + (size_t)r0 * fo;
        g.c_gs = (long long)B * fo;
        g.ldc = fo;
        g.epi = relu ? Epi::kBiasRelu : Epi::kBias;
        g.bias = k.b[mat];
        g.bias_gs = fo;
        g.flags = c.d_flags;
        launch_gemm(g, c.stream);
    }
    return false;
}

// DX: out[r, p] = (sum_j dz[r, j] W[p, j] + add[r, p]) * (mask[r, p] > 0)
// returns true when `colsum` received the per-32-row-block column sums of out
// (the next layer's bias gradient), false when the caller must reduce it
bool gemm_dx(mtk_bank& k, int mat, const Plane3& dz, int B, int r0, int rows, const Plane3& out,
             const float* mask, const float* add, float* colsum = nullptr, const uint32_t* mbits = nullptr) {
    Ctx& c = *k.ctx;
    const int fi = k.fan_in(mat), fo = k.fan_out(mat);
    if (k.tc[k.layer_of(mat)]) {
        UmmaGemm u;
        u.G = k.G;
        u.M = rows;
        u.N = fi;
        u.K = fo;
        u.a_mn = 0;
        u.a = dz.f + (size_t)r0 * fo;
        u.a_rs = fo;
        u.a_gs = (long long)B * fo;
        u.b_mn = 0;  // B(k=j, n=p) = W[p][j]: rows p, contiguous j
        u.b = k.W[mat].f;
        u.b_rs = fo;
        u.b_gs = (long long)fi * fo;
        u.epi = Epi::kMask;
        u.C = out.f + (size_t)r0 * fi;
        u.c_gs = (long long)B * fi;
        u.ldc = fi;
        u.mask = mask + (size_t)r0 * fi;
        if (mbits) {  // the mask as bits (written by the FWD epilogue of the layer below)
            const int wd = mask_words(fi);
            u.mbits = const_cast<uint32_t*>(mbits) + (size_t)r0 * wd;
            u.mb_gs = (long long)B * wd;
            u.mb_ld = wd;
        }
        u.add = add ? add + (size_t)r0 * fi : nullptr;
        u.colsum = colsum;
        u.flags = c.d_flags;
        launch_umma(u, c.stream);
        return colsum != nullptr;
    } else if (head_dx_ok(fi, fo)) {
        HeadDx h;
        h.G = k.G;
        h.rows = rows;
        h.K = fi;
        h.N = fo;
        h.dZ = dz.f + (size_t)r0 * fo;
        h.dz_gs = (long long)B * fo;
        h.lddz = fo;
        h.W = k.W[mat].f;
        h.w_gs = (long long)fi * fo;
        h.C = out.f + (size_t)r0 * fi;
        h.c_gs = (long long)B * fi;
        h.ldc = fi;
        h.mask = mask + (size_t)r0 * fi;
        h.add = add ? add + (size_t)r0 * fi : nullptr;
        h.colsum = colsum;
        launch_head_dx(h, c.stream);
        return colsum != nullptr;
    } else {
        Gemm g;
        g.G = k.G;
        g.M = rows;
        g.N = fi;
        g.K = fo;
        g.A = dz.f + (size_t)r0 * fo;
        g.a_gs = (long long)B * fo;
        g.a_ms = fo;
        g.a_ks = 1;
        g.B = k.W[mat].f;
        g.b_gs = (long long)fi * fo;
        g.b_ks = 1;
        g.b_ns = fo;
        g.C = out.f + (size_t)r0 * fi;
        g.c_gs = (long long)B * fi;
        g.ldc = fi;
        g.epi = Epi::kMask;
        g.mask = mask + (size_t)r0 * fi;
        g.add = add ? add + (size_t)r0 * fi : nullptr;
        g.flags = c.d_flags;
        launch_gemm(g, c.stream);
        return false;
    }
}

// DW + SGD: W[p, j] -= lr * sum_r in[r, p] dz[r, j]
void gemm_dw(mtk_bank& k, int mat, const Plane3& in, const Plane3& dz, int B, int r0, int rows,
             float lr, AdamArgs adam, cudaStream_t st = nullptr) {
    Ctx& c = *k.ctx;
    if (!st) st = c.stream;
    const int fi = k.fan_in(mat), fo = k.fan_out(mat);
    if (adam.on) {
        adam.m = k.mW[mat];
        adam.v = k.vW[mat];
    }
    // Adam on the GEMM paths: the epilogue stores the gradient, adam_apply updates
    const bool adam_gemm = (adam.on || adam.store_only) &&
                           (k.tc[k.layer_of(mat)] || (!head_dw_ok(fo) && !head_dw_ok(fi)));
    float* gbuf = nullptr;
    if (adam_gemm) {
        gbuf = k.keep_grads ? k.gW[mat] : k.adam_grad(mat);
    }
    if (k.tc[k.layer_of(mat)]) {
        UmmaGemm u;
        u.G = k.G;
        u.M = fi;
        u.N = fo;
        u.K = rows;
        u.a_mn = 1;  // A(m=p, k=r) = in[r][p]
        u.a = in.f + (size_t)r0 * fi;
        u.a_rs = fi;
        u.a_gs = (long long)B * fi;
        u.b_mn = 1;  // B(k=r, n=j) = dz[r][j]
        u.b = dz.f + (size_t)r0 * fo;
        u.b_rs = fo;
        u.b_gs = (long long)B * fo;
        u.epi = adam_gemm ? Epi::kStore : Epi::kSgd;
        u.C = adam_gemm ? gbuf : k.W[mat].f;
        u.c_gs = (long long)fi * fo;
        u.ldc = fo;
        u.lr = lr;
        u.grad_out = (!adam_gemm && k.keep_grads) ? k.gW[mat] : nullptr;
        u.flags = c.d_flags;
        launch_umma(u, st);
        if (adam_gemm && !adam.store_only)
            launch_adam_apply(k.W[mat].f, gbuf, (long long)k.G * fi * fo, lr, adam, c.d_flags, st);
    } else if (head_dw_ok(fo) || head_dw_ok(fi)) {
        // narrow output (the heads): reduce over rows with the fo-wide dZ as the
        // register-blocked operand; narrow input (the attack model's k -> H
        // layer): the same kernel on the transposed product dW^T = dZ^T X
        const bool tr = !head_dw_ok(fo);
        HeadDw h;
        h.G = k.G;
        h.rows = rows;
        h.K = tr ? fo : fi;
        h.N = tr ? fi : fo;
        h.A = tr ? dz.f + (size_t)r0 * fo : in.f + (size_t)r0 * fi;
        h.a_gs = (long long)B * (tr ? fo : fi);
        h.lda = tr ? fo : fi;
        h.dZ = tr ? in.f + (size_t)r0 * fi : dz.f + (size_t)r0 * fo;
        h.dz_gs = (long long)B * (tr ? fi : fo);
        h.lddz = tr ? fi : fo;
        h.trans = tr ? 1 : 0;
        h.W = k.W[mat].f;
        h.w_gs = (long long)fi * fo;
        h.lr = lr;
        h.adam = adam;
        h.grad_out = k.keep_grads ? k.gW[mat] : nullptr;
        h.flags = c.d_flags;
        const size_t hb = head_dw_scratch_bytes(k.G, fi, fo);
        const int hs = st == c.stream ? 0 : 1;
        if (hb > k.head_scratch_bytes[hs]) {
            MTK_CUDA(cudaStreamSynchronize(st));  // (the side stream's own prior work)
            MTK_CUDA(cudaStreamSynchronize(c.stream));
            cudaFree(k.head_scratch[hs]);
            MTK_CUDA(cudaMalloc(&k.head_scratch[hs], hb));
            k.head_scratch_bytes[hs] = hb;
        }
        h.partial = k.head_scratch[hs];
        launch_head_dw(h, st);
    } else {
        Gemm g;
        g.G = k.G;
        g.M = fi;
        g.N = fo;
        g.K = rows;
        g.A = in.f + (size_t)r0 * fi;
        g.a_gs = (long long)B * fi;
        g.a_ms = 1;
        g.a_ks = fi;
        g.B = dz.f + (size_t)r0 * fo;
        g.b_gs = (long long)B * fo;
        g.b_ks = fo;
        g.b_ns = 1;
        g.C = adam_gemm ? gbuf : k.W[mat].f;
        g.c_gs = (long long)fi * fo;
        g.ldc = fo;
        g.epi = adam_gemm ? Epi::kStore : Epi::kSgd;
        g.lr = lr;
        g.grad_out = (!adam_gemm && k.keep_grads) ? k.gW[mat] : nullptr;
        g.flags = c.d_flags;
        launch_gemm(g, st);
        if (adam_gemm && !adam.store_only)
            launch_adam_apply(k.W[mat].f, gbuf, (long long)k.G * fi * fo, lr, adam, c.d_flags, st);
    }
}

Plane3 input_plane(mtk_bank& k, const float* X, int B) {
    (void)B;
    Plane3 in;
    in.f = const_cast<float*>(X);
    return in;
}

// after_hidden (optional) runs once the last hidden layer's forward is enqueued
// returns true when the head launch also ran `ce` (optional, single head)
bool run_forward(mtk_bank& k, const Plane3& X, int B, int head_all, int src_rows,
                 const std::function<void()>& after_hidden = {}, const CeArgs* ce = nullptr) {
    bool ce_done = false;
    Ctx& c = *k.ctx;
    Plane3 h = X;
    Plane3 lg;
    lg.f = k.logits;
    for (int l = 0; l < k.L; ++l) {
        PhaseScope ph(c, kPhFwd, (l == k.L - 1 && head_all < 0) ? 2 : 1);
        if (l < k.L - 1) {
            gemm_fwd(k, l, h, B, 0, B, k.H[l + 1], true);
            after_launch(c);
            h = k.H[l + 1];
            if (l == k.L - 2 && after_hidden) after_hidden();
        } else if (head_all >= 0) {
            ce_done = gemm_fwd(k, l + head_all, h, B, 0, B, lg, false, ce);
            after_launch(c);
        } else {  // two heads split by rows
            gemm_fwd(k, l, h, B, 0, src_rows, lg, false);
            gemm_fwd(k, l + 1, h, B, src_rows, B - src_rows, lg, false);
            after_launch(c, 2);
        }
    }
    return ce_done;
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
    need(s.denom[0] >= 0 && s.denom[1] >= 0 && !std::isnan(s.denom[0]) && !std::isnan(s.denom[1]),
         MTK_VALUE_ERROR, "cross_entropy: denominator must be positive");
    k.ensure(B);
    const int src = (two || use_mmd) ? s.src_rows : B;
    const double d0 = s.denom[0] > 0 ? s.denom[0] : (double)(two ? src : B);
    const double d1 = s.denom[1] > 0 ? s.denom[1] : (double)(B - src);
    const float lr = (float)s.lr;
    need(s.optimizer == 0 || s.optimizer == 1, MTK_CONFIG_ERROR,
         "train_step: optimizer must be 0 (SGD) or 1 (Adam)");
    AdamArgs adam;
    if (s.optimizer == 1) {
        const double b1 = s.adam_beta1 > 0 ? s.adam_beta1 : 0.9;
        const double b2 = s.adam_beta2 > 0 ? s.adam_beta2 : 0.999;
        const double eps = s.adam_eps > 0 ? s.adam_eps : 1e-8;
        need(b1 < 1.0 && b2 < 1.0 && std::isfinite(eps), MTK_CONFIG_ERROR,
             "train_step: Adam betas must lie in [0, 1)");
        k.ensure_adam();
        k.adam_t += 1;  // optim.hpp:41, once per optimizer_step
        adam.on = 1;
        adam.b1 = (float)b1;
        adam.b2 = (float)b2;
        adam.eps = (float)eps;
        adam.bc1 = (float)(1.0 - std::pow(b1, (double)k.adam_t));
        adam.bc2 = (float)(1.0 - std::pow(b2, (double)k.adam_t));
    }
    if (k.no_update) {  // mtk_bank_compute_grads: gradients out, parameters untouched
        adam = AdamArgs();
        adam.store_only = 1;
    }
    auto bias_adam = [&](int mat) {
        AdamArgs a = adam;
        if (a.on) {
            a.m = k.mb[mat];
            a.v = k.vb[mat];
        }
        return a;
    };

    const Plane3 X = input_plane(k, s.X, B);
    // Side stream (Ctx::fork/join): the MMD prep pass beside the head forward +
    // CE; the bias updates and the skinny head dW beside the DW GEMMs.
    const char* nse = getenv("MTK_NO_SIDE");  // A/B (read per call)
    const bool side = !(nse && nse[0] == '1');
    cudaEvent_t bias_done[3] = {nullptr, nullptr, nullptr};  // side: last reader of colsum[j % 3]
    auto before_colsum_write = [&](int layer) {  // main: about to overwrite colsum[layer % 3]
        cudaEvent_t& e = bias_done[layer % 3];
        if (e) MTK_CUDA(cudaStreamWaitEvent(c.stream, e, 0));
        e = nullptr;
    };

    static const bool no_colsum = getenv("MTK_NO_COLSUM") != nullptr;  // A/B diagnostics
    MmdArgs a;
    bool prep_on_side = false;
    if (use_mmd) {
        a.G = k.G;
        a.m = src;
        a.n = B - src;
        a.d = k.dims[L - 1];
        a.Xs = k.H[L - 1].f;
        a.xs_gs = (long long)B * a.d;
        a.Xt = k.H[L - 1].f + (size_t)src * a.d;
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
        a.tc = k.tc_mmd && mmd_tc_supported(a);
        // The head's DX (dZ of the last hidden layer = (lambda*g + dlogits W^T) * (h > 0))
        // is fused into the MMD gradient GEMM (an extra K block + the masked
        // epilogue) when that GEMM runs (materialised-W path) and the head is skinny.
        const char* nhf = getenv("MTK_NO_HEAD_FUSE");  // A/B (read per call)
        const bool no_head_fuse = nhf && nhf[0] == '1';
        const int hl = L - 1;
        if (a.tc && !two && !no_head_fuse && hl > 0 && hl > s.frozen_layers && !k.tc[k.layer_of(hl)] &&
            head_dx_ok(k.fan_in(hl), k.fan_out(hl))) {
            const int fi = k.fan_in(hl), fo = k.fan_out(hl);
            a.hd_dz = k.dlog.f;
            a.hd_dz_gs = (long long)B * fo;
            a.hd_n = fo;
            a.hd_W = k.W[hl].f;
            a.hd_w_gs = (long long)fi * fo;
            a.hd_out = k.dZ[1].f;
            a.hd_colsum = (hl - 1 >= s.frozen_layers && !no_colsum) ? k.colsum[(hl - 1) % 3] : nullptr;
            if (k.H[hl].bits) {
                a.hd_zbits = k.H[hl].bits;
                a.hd_zbits_ld = mask_words(fi);
                a.hd_zbits_gs = (long long)B * a.hd_zbits_ld;
            }
            if (!mmd_head_fusable(a)) a.hd_n = 0;
        }
        if (const char* t = getenv("MTK_MMD_TRACE"))  // diagnostics (tools/mmd_trace.py)
            a.trace = reinterpret_cast<unsigned long long*>(strtoull(t, nullptr, 0));
        const int nblk = mmd_blocks_per_group(a);
        const size_t pbytes = (size_t)k.G * nblk * 3 * sizeof(double);
        if (pbytes > k.mmd_part_bytes) {
            MTK_CUDA(cudaStreamSynchronize(c.stream));
            cudaFree(k.mmd_part);
            MTK_CUDA(cudaMalloc(&k.mmd_part, pbytes));
            k.mmd_part_bytes = pbytes;
        }
        a.partial = k.mmd_part;
        if (a.tc) {
            a.beta_out = k.beta;  // fused into the prep pass of launch_mmd_tc
            const size_t zb = mmd_tc_scratch_bytes(a);
            if (zb > k.mmd_z_bytes) {
                MTK_CUDA(cudaStreamSynchronize(c.stream));
                cudaFree(k.mmd_z);
                MTK_CUDA(cudaMalloc(&k.mmd_z, zb));
                k.mmd_z_bytes = zb;
            }
            prep_on_side = side;
        }
    }
    // the prep pass only needs the last hidden layer: it forks off after that
    // layer's forward GEMM and runs beside the head forward and CE
    Plane3* cur = &k.dlog;
    Plane3* nxt = &k.dZ[1];
    Plane3* spare = &k.dZ[0];  // becomes nxt after the head (dlogits keep their own buffer)
    CeArgs ce{k.G,      B,          k.dims[L], two ? src : B, k.logits, s.y, s.w,
              (float)(1.0 / d0), (float)(1.0 / (two ? d1 : d0)), cur->f, k.row_loss, k.loss,
              c.d_flags, k.loss_part};
    // the head's bias gradient comes out of the CE kernel as column partials
    ce.colsum = (!two && L - 1 >= s.frozen_layers && !no_colsum) ? k.colsum[(L - 1) % 3] : nullptr;
    const char* nhc = getenv("MTK_NO_HEAD_CE");  // A/B (read per call)
    const bool fuse_ce = side && !(nhc && nhc[0] == '1');
    // the skinny head's forward also runs the CE rows (fuse_ce), and the MMD
    // prep pass forks off after the last hidden layer to run beside them
    const bool ce_done = run_forward(k, X, B, two ? -1 : 0, src, prep_on_side ? [&] {
        c.fork();
        PhaseScope ph(c, kPhMmdBeta, 2, c.side);  // prep pass: tf32 planes, norms, beta
        launch_mmd_tc(a, k.mmd_z, c.side, kMmdPrep);
        after_launch(c, 2);
    } : std::function<void()>(), fuse_ce ? &ce : nullptr);
    // the loss finish only feeds the host read-back: it joins the first side
    // segment of the backward sweep (a fork here would make the MMD's join wait)
    bool ce_loss_pending = ce_done;
    auto launch_ce_loss_side = [&] {
        if (!ce_loss_pending) return;
        PhaseScope ph(c, kPhCe, 1, c.side);
        launch_ce_loss(ce, c.side);
        after_launch(c, 1);
        ce_loss_pending = false;
    };
    if (!ce_done) {
        PhaseScope ph(c, kPhCe, 2);
        launch_ce(ce, c.stream);
        after_launch(c, 2);
    }

    const bool head_fused = use_mmd && a.hd_n > 0;
    const bool head_fused_colsum = head_fused && a.hd_colsum != nullptr;
    if (use_mmd) {
        if (a.tc && !prep_on_side) {
            PhaseScope ph(c, kPhMmdBeta, 2);  // prep pass: tf32 planes, norms, beta
            launch_mmd_tc(a, k.mmd_z, c.stream, kMmdPrep);
            after_launch(c, 2);
        } else if (!a.tc) {
            double* sc = c.scratch(mmd_beta_scratch_bytes(a));
            PhaseScope ph(c, kPhMmdBeta, 2);
            launch_mmd_beta(a, k.beta, sc, c.stream);
            after_launch(c, 2);
        }
        c.join();  // the prep pass
        if (head_fused && a.hd_colsum) before_colsum_write(L - 2);
        {
            PhaseScope ph(c, kPhMmdPairs, 1);
            if (a.tc) launch_mmd_tc(a, k.mmd_z, c.stream, kMmdPairs);
            else launch_mmd_pairs(a, c.stream);
            after_launch(c, 1);
        }
        {
            // the MMD value only feeds the host read-back: side stream (joined
            // with the step's other side work)
            if (side) c.fork();
            PhaseScope ph(c, kPhOther, 1, side ? c.side : nullptr);
            launch_mmd_finish(a, k.mmd, nullptr, side ? c.side : c.stream);
            after_launch(c, 1);
        }
    }

    // backward sweep, layer L-1 down to 0.  A DX launch also reduces its
    // output's columns per 32-row block when the layer below is trainable,
    // so that layer's bias update needs no second pass over dZ.  Bias updates
    // from those partials and the skinny head dW go to the side stream once
    // the layer's DX is enqueued; they overlap the DW GEMMs.
    bool colsum_ready = ce.colsum != nullptr;
    for (int l = L - 1; l >= 0; --l) {
        const bool trainable = l >= s.frozen_layers;
        const bool need_dx = l > 0 && l > s.frozen_layers;
        const Plane3& in = l == 0 ? X : k.H[l];
        const float* add = (l == L - 1 && use_mmd) ? k.gH : nullptr;
        const Plane3 out = *nxt;
        const bool split = (l == L - 1 && two);
        const int fo = k.dims[l + 1];
        bool next_colsum = false;
        const bool fused_here = head_fused && l == L - 1;  // DX done with the MMD
        if (fused_here) next_colsum = head_fused_colsum;
        // bias from column partials: deferred to the side stream (below)
        const bool bias_side = side && trainable && colsum_ready && !split;
        if (trainable && !bias_side) {
            PhaseScope ph(c, kPhBias, split ? 2 : 1);
            if (colsum_ready && !split) {
                launch_bias_from_partials(k.G, (B + 31) / 32, fo, k.colsum[l % 3], k.b[l], lr, bias_adam(l),
                                          k.keep_grads ? k.gb[l] : nullptr, c.d_flags, c.stream);
            } else if (split) {
                launch_bias_sgd(k.G, src, fo, cur->f, (long long)B * fo, k.b[l], fo, lr, bias_adam(l),
                                k.keep_grads ? k.gb[l] : nullptr, c.d_flags, c.stream);
                launch_bias_sgd(k.G, B - src, fo, cur->f + (size_t)src * fo, (long long)B * fo,
                                k.b[l + 1], fo, lr, bias_adam(l + 1),
                                k.keep_grads ? k.gb[l + 1] : nullptr, c.d_flags, c.stream);
            } else {
                launch_bias_sgd(k.G, B, fo, cur->f, (long long)B * fo, k.b[l], fo, lr, bias_adam(l),
                                k.keep_grads ? k.gb[l] : nullptr, c.d_flags, c.stream);
            }
            after_launch(c, split ? 2 : 1);
        }
        if (need_dx && !fused_here) {
            PhaseScope ph(c, kPhDx, split ? 2 : 1);
            if (split) {
                gemm_dx(k, l, *cur, B, 0, src, out, k.H[l].f, nullptr, nullptr, k.H[l].bits);
                gemm_dx(k, l + 1, *cur, B, src, B - src, out, k.H[l].f, nullptr, nullptr, k.H[l].bits);
                after_launch(c, 2);
            } else {
                const bool below_trainable = l - 1 >= s.frozen_layers && !no_colsum;
                if (below_trainable) before_colsum_write(l - 1);
                const bool have = gemm_dx(k, l, *cur, B, 0, B, out, k.H[l].f, add,
                                          below_trainable ? k.colsum[(l - 1) % 3] : nullptr, k.H[l].bits);
                after_launch(c);
                next_colsum = have;
            }
        }
        // the head's dW reads only dlogits (own buffer), H and its own W: side stream
        const bool dw_side = side && trainable && l == L - 1 && !split && !k.tc[k.layer_of(l)] &&
                             (head_dw_ok(fo) || head_dw_ok(k.dims[l]));
        if (bias_side || dw_side) {
            c.fork();
            launch_ce_loss_side();
            if (bias_side) {
                PhaseScope ph(c, kPhBias, 1, c.side);
                launch_bias_from_partials(k.G, (B + 31) / 32, fo, k.colsum[l % 3], k.b[l], lr, bias_adam(l),
                                          k.keep_grads ? k.gb[l] : nullptr, c.d_flags, c.side);
                after_launch(c, 1);
                bias_done[l % 3] = c.record(c.side);
            }
            if (dw_side) {
                PhaseScope ph(c, kPhDw, 1, c.side);
                gemm_dw(k, l, in, *cur, B, 0, B, lr, adam, c.side);
                after_launch(c, 1);
            }
        }
        if (trainable && !dw_side) {
            PhaseScope ph(c, kPhDw, split ? 2 : 1);
            if (split) {
                gemm_dw(k, l, in, *cur, B, 0, src, lr, adam);
                gemm_dw(k, l + 1, in, *cur, B, src, B - src, lr, adam);
            } else {
                gemm_dw(k, l, in, *cur, B, 0, B, lr, adam);
            }
            after_launch(c, split ? 2 : 1);
        }
        colsum_ready = next_colsum;
        if (l == L - 1) {  // dlogits -> dZ[1] -> dZ[0] -> dZ[1] ...
            cur = nxt;
            nxt = spare;
        } else {
            std::swap(cur, nxt);
        }
    }
    if (ce_loss_pending) {
        c.fork();
        launch_ce_loss_side();
    }
    c.join();  // every side-stream launch of this step

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

bool tc_eligible(int fi, int fo) { return fi >= 32 && fo >= 32 && fi % 4 == 0 && fo % 4 == 0; }

}  // namespace

extern "C" {

int mtk_bank_create(mtk_ctx* c, int G, int n_layers, const int* dims, int n_heads,
                    mtk_bank** out) {
    return guard_on(c, [&] {
        need(c && dims && out, MTK_VALUE_ERROR, "mtk_bank_create: null argument");
        need(G >= 1 && n_layers >= 1, MTK_SHAPE_ERROR, "mtk_bank_create: zero dimension");
        need(n_heads == 1 || n_heads == 2, MTK_CONFIG_ERROR, "mtk_bank_create: n_heads is 1 or 2");
        need(n_heads == 1 || n_layers >= 2, MTK_CONFIG_ERROR,
             "mtk_bank_create: two heads need a shared trunk");
        for (int i = 0; i <= n_layers; ++i)
            need(dims[i] >= 1, MTK_SHAPE_ERROR, "mtk_bank_create: zero dimension in dims");
        std::unique_ptr<mtk_bank> k(new mtk_bank());
        k->ctx = c;
        k->G = G;
        k->L = n_layers;
        k->n_heads = n_heads;
        k->dims.assign(dims, dims + n_layers + 1);
        const char* env = getenv("MTK_DISABLE_TC");
        const bool allow_tc = !(env && env[0] == '1');
        for (int l = 0; l < n_layers; ++l)
            k->tc.push_back(allow_tc && tc_eligible(dims[l], dims[l + 1]));
        k->tc_mmd = allow_tc;
        k->n_mats = n_layers + n_heads - 1;
        for (int i = 0; i < k->n_mats; ++i) {
            const size_t nw = (size_t)G * k->fan_in(i) * k->fan_out(i);
            Plane3 w;
            alloc3(w, nw);
            MTK_CUDA(cudaMemsetAsync(w.f, 0, nw * 4, c->stream));
            float* bb = nullptr;
            MTK_CUDA(cudaMalloc(&bb, (size_t)G * k->fan_out(i) * sizeof(float)));
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
    return guard_on(k ? k->ctx : nullptr, [&] {
        if (!k) return;
        cudaStreamSynchronize(k->ctx->stream);
        delete k;
    });
}

int mtk_bank_set_params(mtk_bank* k, int model, const double* const* W, const double* const* b) {
    return guard_on(k ? k->ctx : nullptr, [&] {
        check_model(k, model);
        need(W && b, MTK_VALUE_ERROR, "set_params: null arrays");
        std::vector<float> tmp;
        for (int i = 0; i < k->n_mats; ++i) {
            const size_t nw = (size_t)k->fan_in(i) * k->fan_out(i), nbias = k->fan_out(i);
            need(W[i] && b[i], MTK_VALUE_ERROR, "set_params: null matrix");
            tmp.assign(W[i], W[i] + nw);
            MTK_CUDA(cudaMemcpyAsync(k->W[i].f + model * nw, tmp.data(), nw * 4,
                                     cudaMemcpyHostToDevice, k->ctx->stream));
            MTK_CUDA(cudaStreamSynchronize(k->ctx->stream));
            tmp.assign(b[i], b[i] + nbias);
            MTK_CUDA(cudaMemcpyAsync(k->b[i] + model * nbias, tmp.data(), nbias * 4,
                                     cudaMemcpyHostToDevice, k->ctx->stream));
            MTK_CUDA(cudaStreamSynchronize(k->ctx->stream));
        }
        MTK_CUDA(cudaStreamSynchronize(k->ctx->stream));
    });
}

int mtk_bank_get_params(mtk_bank* k, int model, double* const* W, double* const* b) {
    return guard_on(k ? k->ctx : nullptr, [&] {
        check_model(k, model);
        MTK_CUDA(cudaStreamSynchronize(k->ctx->stream));
        std::vector<float> tmp;
        for (int i = 0; i < k->n_mats; ++i) {
            const size_t nw = (size_t)k->fan_in(i) * k->fan_out(i), nbias = k->fan_out(i);
            if (W && W[i]) {
                tmp.resize(nw);
                MTK_CUDA(cudaMemcpy(tmp.data(), k->W[i].f + model * nw, nw * 4,
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
    return guard_on(k ? k->ctx : nullptr, [&] {
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
        if (st) fail(st, last_error());
    });
}

int mtk_bank_param_device(mtk_bank* k, int mat, float** W, float** b) {
    return guard_on(k ? k->ctx : nullptr, [&] {
        check_bank(k);
        need(mat >= 0 && mat < k->n_mats, MTK_VALUE_ERROR, "param_device: bad matrix index");
        if (W) *W = k->W[mat].f;
        if (b) *b = k->b[mat];
    });
}

int mtk_bank_forward(mtk_bank* k, const float* X, int B, int head, float* logits,
                     float* hidden_last) {
    return guard_on(k ? k->ctx : nullptr, [&] {
        check_bank(k);
        need(X && logits, MTK_VALUE_ERROR, "forward: null argument");
        need(B >= 1, MTK_SHAPE_ERROR, "forward: B must be >= 1");
        need(head >= 0 && head < k->n_heads, MTK_VALUE_ERROR, "forward: bad head index");
        Ctx& c = *k->ctx;
        if (k->L == 2 && k->n_heads == 1 && !hidden_last &&
            small2_forward_ok(k->dims[0], k->dims[1], k->dims[2])) {
            // attack-model shape: one fused kernel, hidden layer kept in registers
            launch_small2_forward(X, k->G, B, k->dims[0], k->dims[1], k->dims[2], k->W[0].f, k->b[0],
                                  k->W[1].f, k->b[1], logits, c.stream);
            after_launch(c);
            return;
        }
        k->ensure(B);
        const Plane3 in = input_plane(*k, X, B);
        run_forward(*k, in, B, head, 0);
        const size_t GB = (size_t)k->G * B;
        MTK_CUDA(cudaMemcpyAsync(logits, k->logits, GB * k->dims[k->L] * 4,
                                 cudaMemcpyDeviceToDevice, c.stream));
        if (hidden_last && k->L > 1)
            MTK_CUDA(cudaMemcpyAsync(hidden_last, k->H[k->L - 1].f, GB * k->dims[k->L - 1] * 4,
                                     cudaMemcpyDeviceToDevice, c.stream));
    });
}

int mtk_attack_auc(mtk_bank* k, const float* logits, int64_t rows, int C, const uint8_t* labels,
                   double* auc_host, double* acc_host, float* scores_out) {
    return guard_on(k ? k->ctx : nullptr, [&] {
        check_bank(k);
        need(logits && labels, MTK_VALUE_ERROR, "attack_auc: null argument");
        need(rows >= 1 && C >= 1, MTK_SHAPE_ERROR, "attack_auc: zero dimension");
        need(k->G == 1 && k->n_heads == 1 && k->dims[k->L] >= 2, MTK_CONFIG_ERROR,
             "attack_auc: one attack model (G = 1) with one head of >= 2 outputs");
        const int kf = k->dims[0];
        need(kf <= C, MTK_SHAPE_ERROR, "attack_auc: more features than classes");
        Ctx& c = *k->ctx;
        if (k->L == 2 && attack_fused_ok(C, kf, k->dims[1], k->dims[2])) {
            bool clear = false;
            attack_auc_fused(c, logits, rows, C, k->W[0].f, k->b[0], k->W[1].f, k->b[1], labels, scores_out,
                             auc_host, acc_host, &clear);
            if (!clear) c.check_flags();
            return;
        }
        // any other attack-model shape: the four-call composition on the device
        need(rows <= 0x7fffffffLL, MTK_SHAPE_ERROR, "attack_auc: too many rows");
        const int O = k->dims[k->L];
        auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
        const size_t fb = al((size_t)rows * kf * 4), ob = al((size_t)rows * O * 4), sb = al((size_t)rows * 4);
        float* buf = nullptr;
        MTK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&buf), fb + ob + sb, c.stream));
        float* feats = buf;
        float* out = reinterpret_cast<float*>(reinterpret_cast<char*>(buf) + fb);
        float* sc = scores_out ? scores_out : reinterpret_cast<float*>(reinterpret_cast<char*>(buf) + fb + ob);
        launch_features(logits, rows, C, kf, nullptr, feats, c.d_flags, c.stream);
        const int e = mtk_bank_forward(k, feats, (int)rows, 0, out, nullptr);
        if (e != MTK_OK) fail(e, last_error());
        launch_column(out, rows, O, 1, sc, c.stream);
        auc_device(c, sc, labels, rows, auc_host, acc_host);
        MTK_CUDA(cudaFreeAsync(buf, c.stream));
        c.check_flags();
    });
}

int mtk_bank_train_step(mtk_bank* k, const mtk_step* s, double* loss_host, double* mmd_host) {
    return guard_on(k ? k->ctx : nullptr, [&] {
        check_bank(k);
        need(s != nullptr, MTK_VALUE_ERROR, "train_step: null step");
        train_step(*k, *s, loss_host, mmd_host);
    });
}

int mtk_bank_train_epoch(mtk_bank* k, const mtk_step* tmpl, const float* X_pool, const int32_t* y_pool,
                         int64_t pool_rows, const int64_t* idx, const float* w, const double* denom0,
                         int nsteps) {
    return guard_on(k ? k->ctx : nullptr, [&] {
        check_bank(k);
        need(tmpl && X_pool && y_pool && idx, MTK_VALUE_ERROR, "train_epoch: null argument");
        need(nsteps >= 0 && tmpl->B >= 1 && pool_rows >= 1, MTK_SHAPE_ERROR, "train_epoch: bad shape");
        k->ensure_stage(tmpl->B);
        Ctx& c = *k->ctx;
        const int B = tmpl->B, G = k->G;
        // the attack model under SGD: every step of the epoch in one launch
        const char* nse = getenv("MTK_NO_SMALL_EPOCH");  // A/B (read per call)
        if (!(nse && nse[0] == '1') && k->L == 2 && k->n_heads == 1 &&
            small2_epoch_ok(k->dims[0], k->dims[1], k->dims[2], B) && tmpl->optimizer == 0 &&
            tmpl->frozen_layers == 0 && !(tmpl->mmd_lambda > 0.0) && !k->keep_grads && nsteps > 0) {
            need(std::isfinite(tmpl->lr), MTK_VALUE_ERROR, "train_step: lr must be finite");
            std::vector<double> den(nsteps);
            for (int s = 0; s < nsteps; ++s) {
                const double d = denom0 ? denom0[s] : tmpl->denom[0];
                need(d >= 0 && !std::isnan(d), MTK_VALUE_ERROR, "cross_entropy: denominator must be positive");
                den[s] = d > 0 ? d : (double)B;
            }
            double* dden = c.scratch((size_t)nsteps * sizeof(double));
            MTK_CUDA(cudaMemcpyAsync(dden, den.data(), (size_t)nsteps * sizeof(double), cudaMemcpyHostToDevice,
                                     c.stream));
            SmallEpoch e;
            e.G = G;
            e.B = B;
            e.nsteps = nsteps;
            e.W0 = k->W[0].f;
            e.b0 = k->b[0];
            e.W1 = k->W[1].f;
            e.b1 = k->b[1];
            e.X = X_pool;
            e.y = y_pool;
            e.pool_rows = pool_rows;
            e.idx = idx;
            e.w = w;
            e.denom = dden;
            e.lr = (float)tmpl->lr;
            e.flags = c.d_flags;
            launch_small2_epoch(e, c.stream);
            after_launch(c);
            c.check_flags();  // also keeps the host denominators alive until the copy is done
            return;
        }
        for (int s = 0; s < nsteps; ++s) {
            const int64_t* ix = idx + (size_t)s * G * B;
            launch_gather_rows(reinterpret_cast<const uint32_t*>(X_pool), pool_rows, k->dims[0],
                               reinterpret_cast<const long long*>(ix), G, B,
                               reinterpret_cast<uint32_t*>(k->Xs), B, 0, c.d_flags, c.stream);
            launch_gather_rows(reinterpret_cast<const uint32_t*>(y_pool), pool_rows, 1,
                               reinterpret_cast<const long long*>(ix), G, B,
                               reinterpret_cast<uint32_t*>(k->ys), B, 0, c.d_flags, c.stream);
            after_launch(c, 2);
            mtk_step st = *tmpl;
            st.X = k->Xs;
            st.y = k->ys;
            st.w = w ? w + (size_t)s * G * B : nullptr;
            if (denom0) st.denom[0] = denom0[s];
            train_step(*k, st, nullptr, nullptr);
        }
        c.check_flags();
    });
}

int mtk_bank_train_step_host(mtk_bank* k, const mtk_step* s, const float* X_host,
                             const int32_t* y_host, const float* w_host, double* loss_host,
                             double* mmd_host) {
    return guard_on(k ? k->ctx : nullptr, [&] {
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

int mtk_bank_train_step_host_async(mtk_bank* k, const mtk_step* s, const float* X_host,
                                   const int32_t* y_host, const float* w_host) {
    return guard_on(k ? k->ctx : nullptr, [&] {
        check_bank(k);
        need(s && X_host && y_host, MTK_VALUE_ERROR, "train_step_host_async: null argument");
        need(s->B >= 1, MTK_SHAPE_ERROR, "train_step_host_async: B must be >= 1");
        k->ensure_slots(s->B);
        Ctx& c = *k->ctx;
        auto& sl = k->slot[k->next_slot];
        const size_t GB = (size_t)k->G * s->B;
        // the slot's previous step must have finished reading its inputs
        MTK_CUDA(cudaStreamWaitEvent(k->copy_stream, sl.consumed, 0));
        MTK_CUDA(cudaMemcpyAsync(sl.X, X_host, GB * k->dims[0] * 4, cudaMemcpyHostToDevice,
                                 k->copy_stream));
        MTK_CUDA(cudaMemcpyAsync(sl.y, y_host, GB * 4, cudaMemcpyHostToDevice, k->copy_stream));
        if (w_host)
            MTK_CUDA(cudaMemcpyAsync(sl.w, w_host, GB * 4, cudaMemcpyHostToDevice, k->copy_stream));
        MTK_CUDA(cudaEventRecord(sl.copied, k->copy_stream));
        MTK_CUDA(cudaStreamWaitEvent(c.stream, sl.copied, 0));
        mtk_step d = *s;
        d.X = sl.X;
        d.y = sl.y;
        d.w = w_host ? sl.w : nullptr;
        train_step(*k, d, nullptr, nullptr);
        MTK_CUDA(cudaEventRecord(sl.consumed, c.stream));
        MTK_CUDA(cudaMemcpyAsync(sl.res, k->loss, k->G * sizeof(double), cudaMemcpyDeviceToHost,
                                 c.stream));
        sl.mmd = s->mmd_lambda > 0.0;
        if (sl.mmd)
            MTK_CUDA(cudaMemcpyAsync(sl.res + k->G, k->mmd, k->G * sizeof(double),
                                     cudaMemcpyDeviceToHost, c.stream));
        MTK_CUDA(cudaEventRecord(sl.done, c.stream));
        k->last_slot = k->next_slot;
        k->next_slot ^= 1;
    });
}

int mtk_bank_step_result(mtk_bank* k, int which, double* loss_host, double* mmd_host) {
    return guard_on(k ? k->ctx : nullptr, [&] {
        check_bank(k);
        need(k->last_slot >= 0, MTK_CONFIG_ERROR, "step_result: no asynchronous step enqueued");
        need(which == 0 || which == 1, MTK_VALUE_ERROR, "step_result: which is 0 (last) or 1");
        const int idx = which == 0 ? k->last_slot : (k->last_slot ^ 1);
        auto& sl = k->slot[idx];
        MTK_CUDA(cudaEventSynchronize(sl.done));
        if (loss_host) std::memcpy(loss_host, sl.res, k->G * sizeof(double));
        if (mmd_host) {
            if (sl.mmd)
                std::memcpy(mmd_host, sl.res + k->G, k->G * sizeof(double));
            else
                for (int g = 0; g < k->G; ++g) mmd_host[g] = 0.0;
        }
        if (which == 0) k->ctx->check_flags();
    });
}

int mtk_bank_reset_optimizer(mtk_bank* k) {
    return guard_on(k ? k->ctx : nullptr, [&] {
        need(k != nullptr, MTK_VALUE_ERROR, "reset_optimizer: null bank");
        k->reset_adam();
    });
}

int mtk_bank_set_keep_grads(mtk_bank* k, int on) {
    return guard_on(k ? k->ctx : nullptr, [&] {
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
    return guard_on(k ? k->ctx : nullptr, [&] {
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

// ---- data-parallel training of a replicated bank --------

namespace {

int layer_of(const mtk_bank& k, int mat) { return mat < k.L ? mat : k.L - 1; }

// the gradient-arena layout: per matrix i, dW_i then db_i, every segment
// starting on a 128-byte boundary (the GEMM epilogues store 16-byte vectors)
constexpr long long kArenaAlign = 32;  // floats
long long arena_round(long long n) { return (n + kArenaAlign - 1) / kArenaAlign * kArenaAlign; }

std::vector<DpSegment> arena_segments(mtk_bank& k, int frozen_layers, bool adam) {
    std::vector<DpSegment> v;
    long long off = 0;
    for (int i = 0; i < k.n_mats; ++i) {
        const int fz = layer_of(k, i) < frozen_layers;
        DpSegment w, b;
        w.p = k.W[i].f;
        w.n = (long long)k.G * k.fan_in(i) * k.fan_out(i);
        w.off = off;
        w.frozen = fz;
        off = arena_round(off + w.n);
        b.p = k.b[i];
        b.n = (long long)k.G * k.fan_out(i);
        b.off = off;
        b.frozen = fz;
        off = arena_round(off + b.n);
        if (adam) {
            w.m = k.mW[i];
            w.v = k.vW[i];
            b.m = k.mb[i];
            b.v = k.vb[i];
        }
        v.push_back(w);
        v.push_back(b);
    }
    return v;
}

long long arena_floats(mtk_bank& k) {
    const auto v = arena_segments(k, 0, false);
    return v.empty() ? 0 : arena_round(v.back().off + v.back().n);
}

std::vector<DpSegments> segment_chunks(const std::vector<DpSegment>& v) {
    std::vector<DpSegments> out;
    for (size_t i = 0; i < v.size(); i += kMaxDpSegments) {
        DpSegments s;
        for (size_t j = i; j < v.size() && j < i + kMaxDpSegments; ++j) s.s[s.count++] = v[j];
        out.push_back(s);
    }
    return out;
}

}  // namespace

int mtk_bank_grad_size(mtk_bank* k, int64_t* n_floats) {
    return guard_on(k ? k->ctx : nullptr, [&] {
        check_bank(k);
        need(n_floats != nullptr, MTK_VALUE_ERROR, "grad_size: null out");
        *n_floats = arena_floats(*k);
    });
}

int mtk_bank_compute_grads(mtk_bank* k, const mtk_step* s, float* grads, double* loss_host,
                           double* mmd_host) {
    return guard_on(k ? k->ctx : nullptr, [&] {
        check_bank(k);
        need(s != nullptr && grads != nullptr, MTK_VALUE_ERROR, "compute_grads: null argument");
        need(((uintptr_t)grads & 127) == 0, MTK_VALUE_ERROR,
             "compute_grads: the gradient arena must be 128-byte aligned");
        need(s->frozen_layers >= 0 && s->frozen_layers <= k->L, MTK_CONFIG_ERROR,
             "train_step: frozen_layers out of range");
        // the step's own forward/backward in no-update mode: the epilogues
        // store the gradients into the caller's arena and never write a
        // parameter (so a non-finite gradient cannot corrupt the replica)
        const std::vector<DpSegment> segs = arena_segments(*k, s->frozen_layers, false);
        std::vector<float*> saved_w, saved_b;
        saved_w.swap(k->gW);
        saved_b.swap(k->gb);
        const bool saved_keep = k->keep_grads;
        for (int i = 0; i < k->n_mats; ++i) {
            k->gW.push_back(grads + segs[2 * i].off);
            k->gb.push_back(grads + segs[2 * i + 1].off);
        }
        k->keep_grads = true;
        k->no_update = true;
        struct Restore {
            mtk_bank* k;
            std::vector<float*>& w;
            std::vector<float*>& b;
            bool keep;
            ~Restore() {
                k->gW.swap(w);
                k->gb.swap(b);
                k->keep_grads = keep;
                k->no_update = false;
            }
        } restore{k, saved_w, saved_b, saved_keep};
        for (const DpSegment& sg : segs)  // frozen matrices report zero gradients
            if (sg.frozen)
                MTK_CUDA(cudaMemsetAsync(grads + sg.off, 0, sg.n * sizeof(float), k->ctx->stream));
        mtk_step g = *s;
        g.lr = 0.0;
        g.optimizer = 0;
        train_step(*k, g, loss_host, mmd_host);
    });
}

int mtk_bank_dp_apply(mtk_bank* k, const mtk_step* s, const float* parts, int n_parts,
                      int64_t part_stride) {
    return guard_on(k ? k->ctx : nullptr, [&] {
        check_bank(k);
        need(s != nullptr && parts != nullptr, MTK_VALUE_ERROR, "dp_apply: null argument");
        need(n_parts >= 1, MTK_CONFIG_ERROR, "dp_apply: n_workers must be >= 1");
        need(part_stride >= arena_floats(*k) || n_parts == 1, MTK_SHAPE_ERROR,
             "dp_apply: part_stride is smaller than the gradient arena");
        need(((uintptr_t)parts & 15) == 0, MTK_VALUE_ERROR, "dp_apply: parts must be 16-byte aligned");
        need(std::isfinite(s->lr), MTK_VALUE_ERROR, "train_step: lr must be finite");
        need(s->frozen_layers >= 0 && s->frozen_layers <= k->L, MTK_CONFIG_ERROR,
             "train_step: frozen_layers out of range");
        need(s->optimizer == 0 || s->optimizer == 1, MTK_CONFIG_ERROR,
             "train_step: optimizer must be 0 (SGD) or 1 (Adam)");
        AdamArgs adam;
        if (s->optimizer == 1) {
            const double b1 = s->adam_beta1 > 0 ? s->adam_beta1 : 0.9;
            const double b2 = s->adam_beta2 > 0 ? s->adam_beta2 : 0.999;
            const double eps = s->adam_eps > 0 ? s->adam_eps : 1e-8;
            need(b1 < 1.0 && b2 < 1.0 && std::isfinite(eps), MTK_CONFIG_ERROR,
                 "train_step: Adam betas must lie in [0, 1)");
            k->ensure_adam();
            k->adam_t += 1;  // one optimizer_step per dp_step (optim.hpp:41)
            adam.on = 1;
            adam.b1 = (float)b1;
            adam.b2 = (float)b2;
            adam.eps = (float)eps;
            adam.bc1 = (float)(1.0 - std::pow(b1, (double)k->adam_t));
            adam.bc2 = (float)(1.0 - std::pow(b2, (double)k->adam_t));
        }
        Ctx& c = *k->ctx;
        const auto segs = arena_segments(*k, s->frozen_layers, adam.on != 0);
        for (const DpSegments& ch : segment_chunks(segs))
            launch_dp_reduce_apply(ch, parts, n_parts, (long long)part_stride, (float)s->lr, adam,
                                   c.d_flags, c.stream);
        after_launch(c);
    });
}

int mtk_bank_fingerprint(mtk_bank* k, uint64_t* out_host) {
    return guard_on(k ? k->ctx : nullptr, [&] {
        check_bank(k);
        need(out_host != nullptr, MTK_VALUE_ERROR, "fingerprint: null out");
        Ctx& c = *k->ctx;
        auto* d = reinterpret_cast<unsigned long long*>(c.scratch(sizeof(unsigned long long)));
        MTK_CUDA(cudaMemsetAsync(d, 0, sizeof(unsigned long long), c.stream));
        for (const DpSegments& ch : segment_chunks(arena_segments(*k, 0, false)))
            launch_fingerprint(ch, d, c.stream);
        after_launch(c);
        auto* h = static_cast<unsigned long long*>(c.pinned_buf(sizeof(unsigned long long)));
        MTK_CUDA(cudaMemcpyAsync(h, d, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c.stream));
        c.join();
            MTK_CUDA(cudaStreamSynchronize(c.stream));
        *out_host = *h;
    });
}

int mtk_bank_tc_layers(mtk_bank* k, int* out_host) {
    return guard_on(k ? k->ctx : nullptr, [&] {
        check_bank(k);
        need(out_host != nullptr, MTK_VALUE_ERROR, "tc_layers: null out");
        for (int l = 0; l < k->L; ++l) out_host[l] = k->tc[l] ? 1 : 0;
    });
}

}  // extern "C"

// ---- checkpoint / resume ---------------------------------------------------
namespace {

// version 2: the SHA-256 covers the header's config lines (G, dims, heads,
// Adam flag and step count) as well as the payload, so a corrupted step count
// cannot silently change Adam's bias correction on resume
constexpr int kCkptVersion = 2;
const char kCkptMagic[] = "MTKBANK";

std::string hex32(const uint8_t* d) {
    static const char* x = "0123456789abcdef";
    std::string s;
    for (int i = 0; i < 32; ++i) {
        s += x[d[i] >> 4];
        s += x[d[i] & 15];
    }
    return s;
}

void put_u32(std::string& o, uint32_t v) {
    for (int i = 0; i < 4; ++i) o += (char)((v >> (8 * i)) & 0xff);
}
void put_u64(std::string& o, uint64_t v) {
    for (int i = 0; i < 8; ++i) o += (char)((v >> (8 * i)) & 0xff);
}
// little-endian fp32 record: name, rank, dims, byte count, data
void put_tensor(std::string& o, const std::string& name, const std::vector<uint64_t>& shape,
                const std::vector<float>& v) {
    put_u32(o, (uint32_t)name.size());
    o += name;
    put_u32(o, (uint32_t)shape.size());
    for (uint64_t d : shape) put_u64(o, d);
    put_u64(o, (uint64_t)v.size() * 4);
    for (float f : v) {
        uint32_t u;
        std::memcpy(&u, &f, 4);
        put_u32(o, u);
    }
}

struct Reader {
    const std::string& s;
    size_t pos;
    uint32_t u32() {
        need(pos + 4 <= s.size(), MTK_CHECKPOINT_ERROR, "checkpoint: record overruns the payload");
        uint32_t v = 0;
        for (int i = 0; i < 4; ++i) v |= (uint32_t)(uint8_t)s[pos + i] << (8 * i);
        pos += 4;
        return v;
    }
    uint64_t u64() {
        const uint64_t lo = u32(), hi = u32();
        return lo | (hi << 32);
    }
    // the next record, which must be `name` with `shape`
    void tensor(const std::string& name, const std::vector<uint64_t>& shape, std::vector<float>& out) {
        const uint32_t nl = u32();
        need(pos + nl <= s.size(), MTK_CHECKPOINT_ERROR, "checkpoint: record overruns the payload");
        const std::string got = s.substr(pos, nl);
        pos += nl;
        need(got == name, MTK_CHECKPOINT_ERROR, "checkpoint: expected tensor " + name + ", found " + got);
        const uint32_t rank = u32();
        need(rank == shape.size(), MTK_CHECKPOINT_ERROR, "checkpoint: rank mismatch for " + name);
        size_t n = 1;
        for (uint64_t d : shape) {
            need(u64() == d, MTK_CHECKPOINT_ERROR, "checkpoint: shape mismatch for " + name);
            n *= d;
        }
        need(u64() == n * 4, MTK_CHECKPOINT_ERROR, "checkpoint: byte count mismatch for " + name);
        out.resize(n);
        for (size_t i = 0; i < n; ++i) {
            const uint32_t u = u32();
            std::memcpy(&out[i], &u, 4);
        }
    }
};

// SHA-256 over the canonical header text (magic .. payload line, each line
// '\n'-terminated) followed by the payload
void digest_of(const std::string& hdr_core, const std::string& pay, uint8_t out[32]) {
    std::string all;
    all.reserve(hdr_core.size() + pay.size());
    all += hdr_core;
    all += pay;
    sha256(all.data(), all.size(), out);
}

// strict decimal integer in [lo, hi]: the whole word, no sign tricks, no overflow
long long parse_int(const std::string& w, long long lo, long long hi, const char* what) {
    bool ok = !w.empty() && w.size() <= 19;
    for (char ch : w) ok = ok && ch >= '0' && ch <= '9';
    long long v = 0;
    if (ok) {
        errno = 0;
        char* end = nullptr;
        v = std::strtoll(w.c_str(), &end, 10);
        ok = errno == 0 && end && *end == '\0' && v >= lo && v <= hi;
    }
    need(ok, MTK_CHECKPOINT_ERROR, std::string("checkpoint: malformed ") + what + " '" + w + "'");
    return v;
}

std::vector<float> d2h(const float* d, size_t n, cudaStream_t s) {
    std::vector<float> h(n);
    MTK_CUDA(cudaMemcpyAsync(h.data(), d, n * 4, cudaMemcpyDeviceToHost, s));
    MTK_CUDA(cudaStreamSynchronize(s));
    return h;
}

}  // namespace

int mtk_bank_save(mtk_bank* k, const char* path) {
    return guard_on(k ? k->ctx : nullptr, [&] {
        check_bank(k);
        need(path != nullptr, MTK_VALUE_ERROR, "save: null path");
        Ctx& c = *k->ctx;
        c.check_flags();
        std::string pay;
        const bool adam = !k->mW.empty();
        for (int i = 0; i < k->n_mats; ++i) {
            const uint64_t G = k->G, fi = k->fan_in(i), fo = k->fan_out(i);
            const std::string n = std::to_string(i);
            put_tensor(pay, "W" + n, {G, fi, fo}, d2h(k->W[i].f, G * fi * fo, c.stream));
            put_tensor(pay, "b" + n, {G, fo}, d2h(k->b[i], G * fo, c.stream));
            if (adam) {
                put_tensor(pay, "mW" + n, {G, fi, fo}, d2h(k->mW[i], G * fi * fo, c.stream));
                put_tensor(pay, "vW" + n, {G, fi, fo}, d2h(k->vW[i], G * fi * fo, c.stream));
                put_tensor(pay, "mb" + n, {G, fo}, d2h(k->mb[i], G * fo, c.stream));
                put_tensor(pay, "vb" + n, {G, fo}, d2h(k->vb[i], G * fo, c.stream));
            }
        }
        std::string hdr = std::string(kCkptMagic) + " " + std::to_string(kCkptVersion) + "\n";
        hdr += "G " + std::to_string(k->G) + "\n";
        hdr += "dims";
        for (int v : k->dims) hdr += " " + std::to_string(v);
        hdr += "\nheads " + std::to_string(k->n_heads) + "\n";
        hdr += "adam " + std::to_string(adam ? 1 : 0) + " " + std::to_string(k->adam_t) + "\n";
        hdr += "payload " + std::to_string(pay.size()) + "\n";
        uint8_t dg[32];
        digest_of(hdr, pay, dg);  // the header lines so far + the payload
        hdr += "sha256 " + hex32(dg) + "\n\n";
        FILE* f = std::fopen(path, "wb");
        need(f != nullptr, MTK_DATA_ERROR, std::string("save: cannot open ") + path);
        const bool ok = std::fwrite(hdr.data(), 1, hdr.size(), f) == hdr.size() &&
                        std::fwrite(pay.data(), 1, pay.size(), f) == pay.size();
        std::fclose(f);
        need(ok, MTK_DATA_ERROR, std::string("save: write failed for ") + path);
    });
}

int mtk_bank_load(mtk_ctx* c, const char* path, mtk_bank** out) {
    return guard_on(c, [&] {
        need(c && path && out, MTK_VALUE_ERROR, "load: null argument");
        *out = nullptr;
        FILE* f = std::fopen(path, "rb");
        need(f != nullptr, MTK_DATA_ERROR, std::string("load: cannot open ") + path);
        std::string all;
        char buf[1 << 16];
        size_t got;
        while ((got = std::fread(buf, 1, sizeof(buf), f)) > 0) all.append(buf, got);
        std::fclose(f);
        const size_t he = all.find("\n\n");
        need(he != std::string::npos, MTK_TRUNCATED_ERROR, "checkpoint: truncated header");
        std::vector<std::string> lines;
        for (size_t p = 0; p < he;) {
            const size_t e = all.find('\n', p);
            lines.push_back(all.substr(p, (e == std::string::npos || e > he ? he : e) - p));
            p = (e == std::string::npos) ? he : e + 1;
        }
        auto words = [](const std::string& l) {
            std::vector<std::string> w;
            size_t p = 0;
            while (p < l.size()) {
                const size_t e = l.find(' ', p);
                const size_t q = e == std::string::npos ? l.size() : e;
                if (q > p) w.push_back(l.substr(p, q - p));
                p = q + 1;
            }
            return w;
        };
        need(!lines.empty(), MTK_CHECKPOINT_ERROR, "checkpoint: empty header");
        auto l0 = words(lines[0]);
        need(l0.size() == 2 && l0[0] == kCkptMagic, MTK_CHECKPOINT_ERROR, "checkpoint: not a bank checkpoint");
        const long long ver = parse_int(l0[1], 0, 1LL << 30, "format_version");
        need(ver == kCkptVersion, MTK_VERSION_ERROR,
             "checkpoint: format_version " + l0[1] + " in file, this library reads version " +
                 std::to_string(kCkptVersion));
        // exactly: magic, G, dims, heads, adam, payload, sha256 -- in that order
        const char* keys[] = {"G", "dims", "heads", "adam", "payload", "sha256"};
        need(lines.size() == 7, MTK_CHECKPOINT_ERROR, "checkpoint: malformed header (line count)");
        std::vector<std::vector<std::string>> hw;
        for (size_t i = 1; i < 7; ++i) {
            hw.push_back(words(lines[i]));
            need(!hw.back().empty() && hw.back()[0] == keys[i - 1], MTK_CHECKPOINT_ERROR,
                 std::string("checkpoint: malformed header (expected '") + keys[i - 1] + "')");
        }
        need(hw[0].size() == 2 && hw[1].size() >= 3 && hw[2].size() == 2 && hw[3].size() == 3 &&
                 hw[4].size() == 2 && hw[5].size() == 2 && hw[5][1].size() == 64,
             MTK_CHECKPOINT_ERROR, "checkpoint: malformed header (field count)");
        const int G = (int)parse_int(hw[0][1], 1, 1 << 20, "G");
        std::vector<int> dims;
        for (size_t j = 1; j < hw[1].size(); ++j) dims.push_back((int)parse_int(hw[1][j], 1, 1 << 24, "dims"));
        const int heads = (int)parse_int(hw[2][1], 1, 2, "heads");
        const int adam = (int)parse_int(hw[3][1], 0, 1, "adam flag");
        const unsigned long long adam_t = (unsigned long long)parse_int(hw[3][2], 0, 1LL << 62, "adam step");
        const unsigned long long paybytes = (unsigned long long)parse_int(hw[4][1], 0, 1LL << 62, "payload size");
        const std::string digest = hw[5][1];
        const size_t sha_at = all.rfind("\nsha256 ", he);
        need(sha_at != std::string::npos, MTK_CHECKPOINT_ERROR, "checkpoint: malformed header (sha256)");
        const std::string hdr_core = all.substr(0, sha_at + 1);
        const std::string pay = all.substr(he + 2);
        need(pay.size() >= paybytes, MTK_TRUNCATED_ERROR,
             "checkpoint: truncated payload (" + std::to_string(pay.size()) + " of " +
                 std::to_string(paybytes) + " bytes)");
        need(pay.size() == paybytes, MTK_CHECKPOINT_ERROR, "checkpoint: trailing bytes after the payload");
        uint8_t dg[32];
        digest_of(hdr_core, pay, dg);
        need(hex32(dg) == digest, MTK_DIGEST_ERROR, "checkpoint: header/payload SHA-256 mismatch");
        mtk_bank* k = nullptr;
        const int st = mtk_bank_create(c, G, (int)dims.size() - 1, dims.data(), heads, &k);
        if (st != MTK_OK) fail(st, mtk_last_error());
        std::unique_ptr<mtk_bank> own(k);
        Reader rd{pay, 0};
        std::vector<float> v;
        Ctx& cx = *k->ctx;
        auto h2d = [&](float* d) {
            MTK_CUDA(cudaMemcpyAsync(d, v.data(), v.size() * 4, cudaMemcpyHostToDevice, cx.stream));
            MTK_CUDA(cudaStreamSynchronize(cx.stream));
        };
        if (adam) k->ensure_adam();
        for (int i = 0; i < k->n_mats; ++i) {
            const uint64_t g = k->G, fi = k->fan_in(i), fo = k->fan_out(i);
            const std::string n = std::to_string(i);
            rd.tensor("W" + n, {g, fi, fo}, v);
            h2d(k->W[i].f);
            rd.tensor("b" + n, {g, fo}, v);
            h2d(k->b[i]);
            if (adam) {
                rd.tensor("mW" + n, {g, fi, fo}, v);
                h2d(k->mW[i]);
                rd.tensor("vW" + n, {g, fi, fo}, v);
                h2d(k->vW[i]);
                rd.tensor("mb" + n, {g, fo}, v);
                h2d(k->mb[i]);
                rd.tensor("vb" + n, {g, fo}, v);
                h2d(k->vb[i]);
            }
        }
        need(rd.pos == pay.size(), MTK_CHECKPOINT_ERROR, "checkpoint: unexpected records after the last tensor");
        k->adam_t = adam_t;
        *out = own.release();
    });
}

int mtk_bank_info(mtk_bank* k, int* G, int* n_layers, int* dims_out, int* n_heads) {
    return guard_on(k ? k->ctx : nullptr, [&] {
        check_bank(k);
        if (G) *G = k->G;
        if (n_layers) *n_layers = k->L;
        if (dims_out)
            for (size_t i = 0; i < k->dims.size(); ++i) dims_out[i] = k->dims[i];
        if (n_heads) *n_heads = k->n_heads;
    });
}
