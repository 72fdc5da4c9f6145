// internal.h -- shared declarations of libmtk (host side + kernel launchers).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <mutex>
#include <vector>

#include "minitransfer/mtk.h"

namespace mtk {

// Exceptions carry the C-ABI status; capi.cu converts them at the boundary.
struct Failure : std::runtime_error {
    int status;
    Failure(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};
[[noreturn]] inline void fail(int s, const std::string& m) { throw Failure(s, m); }
void sha256(const void* data, size_t len, uint8_t out[32]);

#define MTK_CUDA(call)                                                                   \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess)                                                           \
            ::mtk::fail(MTK_ERROR, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// Device-side deferred error bits (checked at synchronizing calls).
enum : int { kFlagNonFinite = 1, kFlagBadLabel = 2, kFlagBadIndex = 4 };

// Phases of the bank step, for optional CUDA-event timing (mtk_ctx_set_timing).
enum Phase : int { kPhFwd = 0, kPhCe, kPhMmdBeta, kPhMmdPairs, kPhDx, kPhDw, kPhBias, kPhOther,
                   kPhSide, kNumPhases };

// Pinned host blocks, recycled (grow-only; thread-safe: the sweep's worker
// thread takes blocks while the caller's thread returns them).  Portable, so
// a thread with another device current may allocate.
class HostBlockPool {
    std::mutex mu_;
    std::vector<std::pair<void*, size_t>> free_;
    std::vector<void*> all_;

public:
    HostBlockPool() = default;
    HostBlockPool(const HostBlockPool&) = delete;
    HostBlockPool& operator=(const HostBlockPool&) = delete;
    // the smallest free block of >= bytes, else a new one; *cap = its size
    void* get(size_t bytes, size_t* cap);
    void put(void* p, size_t cap);
    ~HostBlockPool();
};

struct Ctx {
    int device = 0;
    bool timing = false;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
    std::vector<cudaEvent_t> event_pool;
    double phase_ms[kNumPhases] = {0};
    uint64_t phase_launches[kNumPhases] = {0};
    cudaEvent_t take_event();
    void collect_phases();
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int* d_flags = nullptr;          // deferred error bits
    double* d_scratch = nullptr;     // small fp64 reduction scratch
    size_t scratch_bytes = 0;
    uint64_t launches = 0;
    void* pinned = nullptr;          // host staging for small results
    int* pinned_flags = nullptr;     // dedicated host word for check_flags()
    size_t pinned_bytes = 0;
    double* scratch(size_t bytes);
    // grow-only device workspace for the large per-call buffers (AUC sort,
    // MMD planes / partial slots); stream-ordered reuse, no per-call malloc
    void* big(size_t bytes);
    void* d_big = nullptr;
    size_t big_bytes = 0;
    void* pinned_buf(size_t bytes);
    // AUC level-2 class histograms (auc.cuh): grow-only, zeroed when allocated
    // and left zeroed by every call
    uint32_t* auc_l2(size_t bytes);
    uint32_t* d_auc_l2 = nullptr;
    // AUC mailbox: mapped pinned host memory the last AUC kernel writes its
    // counters to, then a sequence number; the host spins on it instead of a
    // D2H copy + stream synchronize (k_attack.cu)
    unsigned long long* auc_mail = nullptr;      // host view, 16 words
    unsigned long long* auc_mail_dev = nullptr;  // device view
    unsigned long long auc_seq = 0;
    bool auc_fast_hint = true;        // the previous AUC took the full-resolution path (k_attack.cu)
    bool auc_win_valid = false;       // speculative full-resolution window from the previous call's keys
    uint32_t auc_win_lo = 0;
    int auc_parity = 0;               // which of the two counter blocks this call uses
    size_t auc_l2_bytes = 0;
    HostBlockPool* host_blocks = nullptr;  // the native sweep's pinned staging (sweep.cpp)
    HostBlockPool& host_pool();
    // grow-only device workspace of the native sweep (one chunk of query rows
    // of every model: G x rows x d floats -- allocated once per context)
    void* sweep_buf(size_t bytes);
    void* d_sweep = nullptr;
    size_t sweep_bytes = 0;
    void check_flags();               // synchronizes; throws on a set flag
    // Side stream for short, latency-bound kernels that do not feed the next
    // main-stream launch (bias updates, the skinny head dW, the MMD prep pass):
    // they run beside the persistent GEMMs, on the SMs those leave idle in
    // their last partial wave.  Ordering is by events only.
    cudaStream_t side = nullptr;
    cudaEvent_t ev_ring[32] = {};
    int ev_next = 0;
    bool side_pending = false;        // side work not yet joined into the main stream
    cudaEvent_t record(cudaStream_t s);  // a fresh (no-timing) event recorded on s
    void fork();                      // side waits for all main-stream work so far
    void join();                      // main waits for all side-stream work so far
};

// RAII: records start/stop events around a launch group when timing is on.
struct PhaseScope {
    Ctx& c;
    int ph;
    int n;
    cudaStream_t st;
    cudaEvent_t a = nullptr;
    PhaseScope(Ctx& ctx, int phase, int launches = 1, cudaStream_t s = nullptr);  // s: side -> kPhSide
    ~PhaseScope();
};

// Grouped GEMM description.  Per group g:
//   C(m,n) = sum_k A(m,k) * B(k,n)
//   A(m,k) = A[g*a_gs + m*a_ms + k*a_ks]; B(k,n) = B[g*b_gs + k*b_ks + n*b_ns]
// Epilogues operate on row-major outputs C[g*c_gs + m*ldc + n].
// Parameter update applied by the dW / db epilogues (optim.hpp:30-68):
// SGD w -= lr g (:46-48), or Adam (:49-63) with moments m, v laid out like
// the parameter and host-computed bias corrections bc1 = 1 - b1^t,
// bc2 = 1 - b2^t (fp32 here, f64 in the reference).
struct AdamArgs {
    int on = 0;
    // no parameter update at all (mtk_bank_compute_grads): the epilogues store
    // the gradient only and every update site leaves w untouched, so a
    // non-finite gradient cannot reach the parameters
    int store_only = 0;
    float b1 = 0.9f, b2 = 0.999f, eps = 1e-8f, bc1 = 1.f, bc2 = 1.f;
    float* m = nullptr;
    float* v = nullptr;
};
#ifdef __CUDACC__
// For the simple (not unrolled) update loops: bias, skinny-head dW, adam_apply.
// The tensor-core / SIMT GEMM epilogues do SGD only; under Adam they store the
// gradient and launch_adam_apply updates (keeps Adam's division / sqrt slow
// paths out of the unrolled epilogues).
// SGD w - lr*g as one explicit fused multiply-add, so every update site (GEMM
// epilogues, bias kernels, dp_apply) rounds identically whatever nvcc's
// contraction choices are.
__device__ __forceinline__ float sgd_update(float w, float g, float lr) { return __fmaf_rn(-lr, g, w); }
__device__ __forceinline__ float param_update(float w, float g, float lr, const AdamArgs& a,
                                              long long idx) {
    if (a.store_only) return w;
    if (!a.on) return sgd_update(w, g, lr);
    const float m = a.b1 * a.m[idx] + (1.f - a.b1) * g;
    const float v = a.b2 * a.v[idx] + (1.f - a.b2) * g * g;
    a.m[idx] = m;
    a.v[idx] = v;
    const float mhat = m / a.bc1, vhat = v / a.bc2;
    return w - lr * mhat / (sqrtf(vhat) + a.eps);
}
#endif

enum class Epi : int {
    kBias = 0,      // C = acc + bias[n]
    kBiasRelu = 1,  // C = max(acc + bias[n], 0)
    kMask = 2,      // C = (acc + add[m,n]) * (mask[m,n] > 0)      (dX through ReLU)
    kSgd = 3,       // C(=W) -= lr * acc ; optionally grad_out = acc  (dW + SGD)
    kStore = 4,     // C = acc (diagnostics)
    kNone = 5,      // no output (diagnostics: epilogue without global traffic)
    kMmdGrad = 6,   // C = scale * (add[m,n] * rowvec[m] - acc)   (MMD gradient from V = W.Z)
    kMmdGradW = 7,  // C = -scale * acc [* ReLU mask bits]         (V' = W'.Z, W' = W - diag(Wsum))
};

struct Gemm {
    int G = 1, M = 0, N = 0, K = 0;
    const float* A = nullptr;
    long long a_gs = 0, a_ms = 0, a_ks = 0;
    const float* B = nullptr;
    long long b_gs = 0, b_ks = 0, b_ns = 0;
    float* C = nullptr;
    long long c_gs = 0, ldc = 0;
    Epi epi = Epi::kBias;
    const float* bias = nullptr;  // [G, N] stride bias_gs
    long long bias_gs = 0;
    const float* add = nullptr;   // kMask: optional addend, same layout as C
    const float* mask = nullptr;  // kMask: mask source, same layout as C
    float lr = 0.f;               // kSgd
    float* grad_out = nullptr;    // kSgd: optional copy of acc, same layout as C
    int* flags = nullptr;
};

void launch_gemm(const Gemm& g, cudaStream_t s);
// W[i] -= Adam step from grad[i], i < n (moments in a.m / a.v); non-finite -> flags
void launch_adam_apply(float* W, const float* grad, long long n, float lr, const AdamArgs& a,
                       int* flags, cudaStream_t s);

// data-parallel step (k_dp.cu): one segment per parameter array (W_i, b_i)
// of a bank, at float offset `off` of the gradient arena.
struct DpSegment {
    float* p = nullptr;  // parameters (device)
    float* m = nullptr;  // Adam moments (or null)
    float* v = nullptr;
    long long off = 0, n = 0;
    int frozen = 0;
};
constexpr int kMaxDpSegments = 40;
struct DpSegments {
    DpSegment s[kMaxDpSegments];
    int count = 0;
};
// p_seg = optimizer_step(p_seg, (sum_{r ascending} parts[r*stride + off + j]) / n)
void launch_dp_reduce_apply(const DpSegments& segs, const float* parts, int n_parts,
                            long long part_stride, float lr, const AdamArgs& adam, int* flags,
                            cudaStream_t s);
// *out += order-independent 64-bit hash of every segment's parameter bits
void launch_fingerprint(const DpSegments& segs, unsigned long long* out, cudaStream_t s);

// counter-based synthetic data (k_rng.cu; contract in mtk.h / oracle.h)
void launch_philox_fill(uint64_t seed, uint64_t stream, uint64_t c0, uint64_t c1, long long nblocks,
                        uint64_t* out, cudaStream_t s);
void launch_counter_normals(uint64_t seed, uint64_t stream, long long first, long long count,
                            float* out, cudaStream_t s);
void launch_synth_counter(uint64_t seed, uint64_t stream, int C, int d, long long n,
                          const float* mu, const float* shift, float* X, int32_t* y,
                          cudaStream_t s);

// tcgen05 3xTF32 grouped GEMM (k_umma.cu).  Operands are plain fp32; element
// (r, c) sits at base[g*gs + r*rs + c], c being the contiguous index: for a
// K-major operand r = m (or n) and c = k, for an MN-major operand r = k and
// c = m (or n).  Row strides must be multiples of 4 elements (TMA).
struct UmmaGemm {
    int G = 1, M = 0, N = 0, K = 0;
    int a_mn = 0, b_mn = 0;
    const float* a = nullptr;
    long long a_rs = 0, a_gs = 0;
    const float* b = nullptr;
    long long b_rs = 0, b_gs = 0;
    Epi epi = Epi::kStore;
    float* C = nullptr;
    long long c_gs = 0, ldc = 0;
    const float* bias = nullptr;
    long long bias_gs = 0;
    const float* add = nullptr;
    const float* mask = nullptr;
    float lr = 0.f;
    float* grad_out = nullptr;
    float* colsum = nullptr;  // kMask: per-32-row-block column sums [G][ceil(M/32)][N]
    const float* rowvec = nullptr;  // kMmdGrad: per-row scalar [G][M]
    float scale = 1.f;              // kMmdGrad
    int zmask = 0;                  // kMmdGrad: C *= (add > 0) (the fused head DX)
    // optional second B operand: rows k >= ksplit of B are rows k - ksplit of b2
    // (N-major B only; ksplit % 32 == 0)
    const float* b2 = nullptr;
    long long b2_rs = 0, b2_gs = 0;
    int ksplit = 0;
    // the operands are of one sign (e.g. MMD V = W.Z, W >= 0, Z = post-ReLU
    // h >= 0): accumulate the 3xTF32 corrections separately whatever K is
    int same_sign = 0;
    // SEPC: at most this many leading k-blocks' corrections share the main
    // accumulator while the previous tile's epilogue drains (0: none; the MMD
    // gradient GEMM, whose result is a small difference)
    int sepc_share = 10;
    // ReLU mask bits [G][M][mb_ld words], bit j of word w = column 32 w + j:
    // kBiasRelu writes them (output > 0), kMask reads them instead of `mask`
    uint32_t* mbits = nullptr;
    long long mb_gs = 0, mb_ld = 0;
    int* flags = nullptr;
};
void launch_umma(const UmmaGemm& u, cudaStream_t s);
namespace umma {
bool pdl_enabled();  // programmatic dependent launch (MTK_PDL, default on)
}


// Skinny layers (out width <= 32): k_head.cu
struct CeArgs;
struct HeadFwd {
    int G = 1, rows = 0, K = 0, N = 0;
    const float* A = nullptr;
    long long a_gs = 0, lda = 0;
    const float* W = nullptr;  // [G][K][N]
    long long w_gs = 0;
    const float* bias = nullptr;
    long long bias_gs = 0;
    float* C = nullptr;
    long long c_gs = 0, ldc = 0;
    int relu = 0;
    int* flags = nullptr;
    // optional: softmax-CE of the finished logits rows in the same kernel
    // (ce_kernel's per-row work and per-32-row partials; rows = ce->B, C = N);
    // the loss finish (launch_ce_loss) stays a separate launch
    const CeArgs* ce = nullptr;
};
struct HeadDw {
    int G = 1, rows = 0, K = 0, N = 0;
    const float* A = nullptr;  // [G][rows][K] (stride lda)
    long long a_gs = 0, lda = 0;
    const float* dZ = nullptr; // [G][rows][N] (stride lddz)
    long long dz_gs = 0, lddz = 0;
    float* W = nullptr;        // [G][K][N]  ([G][N][K] with trans)
    long long w_gs = 0;
    int trans = 0;             // W^T layout: the narrow operand is the layer input
    float lr = 0.f;
    AdamArgs adam;
    float* grad_out = nullptr;
    int* flags = nullptr;
    float* partial = nullptr;  // scratch, head_dw_scratch_bytes()
};
struct HeadDx {
    int G = 1, rows = 0, K = 0, N = 0;  // out [rows, K] = dZ [rows, N] . W[K, N]^T
    const float* dZ = nullptr;
    long long dz_gs = 0, lddz = 0;
    const float* W = nullptr;  // [G][K][N]
    long long w_gs = 0;
    float* C = nullptr;
    long long c_gs = 0, ldc = 0;
    const float* mask = nullptr;  // same layout as C
    const float* add = nullptr;
    float* colsum = nullptr;      // per-32-row-block column sums [G][ceil(rows/32)][K], or null
};
bool head_fwd_ok(int K, int N);
// forward-only 2-layer MLP K -> H -> O with K <= 8, O <= 4 (the attack model)
bool small2_forward_ok(int K, int H, int O);
void launch_small2_forward(const float* X, int G, int rows, int K, int H, int O, const float* W0,
                           const float* b0, const float* W1, const float* b1, float* logits,
                           cudaStream_t s);
// whole SGD epochs of the attack model (K=3 -> 64 -> 2, B <= 1024) in one launch
struct SmallEpoch {
    int G, B, nsteps;
    float *W0, *b0, *W1, *b1;  // the bank's parameters (updated in place)
    const float* X;            // pool [pool_rows][3]
    const int32_t* y;          // pool labels
    long long pool_rows;
    const int64_t* idx;        // [nsteps][G][B]
    const float* w;            // [nsteps][G][B] or null
    const double* denom;       // [nsteps] device
    float lr;
    int* flags;
    unsigned long long* trace = nullptr;  // diagnostics (MTK_EPOCH_TRACE): phase stamps of CTA 0
};
bool small2_epoch_ok(int K, int H, int O, int B);
void launch_small2_epoch(const SmallEpoch& p, cudaStream_t s);
bool head_dx_ok(int K, int N);
void launch_head_dx(const HeadDx& p, cudaStream_t s);
size_t head_dw_scratch_bytes(int G, int K, int N);
bool head_dw_ok(int N);
void launch_head_fwd(const HeadFwd& p, cudaStream_t s);
void launch_head_dw(const HeadDw& p, cudaStream_t s);

// Cross-entropy head (tape.hpp:475-520), rows laid out [G, B, C].
struct CeArgs {
    int G, B, C, src_rows;
    const float* logits;
    const int32_t* y;
    const float* w;         // may be null
    float inv_denom0, inv_denom1;  // head 0 rows [0,src_rows), head 1 the rest
    float* dlogits;         // [G,B,C]
    double* row_loss;       // [G,B]  w_i (lse - x_y) / denom_head
    double* loss;           // [G]
    int* flags;
    double* loss_part;      // [G][ceil(B/32)] scratch
    float* colsum = nullptr;  // optional [G][ceil(B/32)][C] dlogits column partials
};
void launch_ce(const CeArgs& a, cudaStream_t s);       // rows + loss finish
void launch_ce_loss(const CeArgs& a, cudaStream_t s);  // the loss finish alone

// Column sums + SGD on a bias: db[g,n] = sum_{rows} dZ[g, r, n]; b -= lr*db
// bias update from per-row-block column partials [G][nrb][N] (fixed order)
void launch_bias_from_partials(int G, int nrb, int N, const float* partial, float* b, float lr,
                               const AdamArgs& adam, float* grad_out, int* flags, cudaStream_t s);
void launch_bias_sgd(int G, int rows, int N, const float* dZ, long long dz_gs, float* b,
                     long long b_gs, float lr, const AdamArgs& adam, float* grad_out, int* flags,
                     cudaStream_t s);

// MMD problem over G independent groups; group g has rows [0,m) in Xs and
// [0,n) in Xt, both row-major with row stride d.
struct MmdArgs {
    int G = 1;
    long long m = 0, n = 0;
    int d = 0;
    const float* Xs = nullptr;
    long long xs_gs = 0;
    const float* Xt = nullptr;
    long long xt_gs = 0;
    int nb = 5;
    float mult[8] = {0.25f, 0.5f, 1.f, 2.f, 4.f, 0.f, 0.f, 0.f};
    const double* beta = nullptr;   // [G] device (detached)
    double* beta_out = nullptr;     // tc path: compute beta here (fused into the prep pass); == beta
    long long row_begin = 0, row_end = -1;  // concatenated-row range (all groups)
    // materialised-W path, one group: this rank owns the 128-row tiles
    // [tile_begin, tile_end) (-1: all); see mtk_mmd_gaussian_tiles
    long long tile_begin = 0, tile_end = -1;
    double* partial = nullptr;      // [G, nblocks_per_group, 3] device
    float* gXs = nullptr;           // optional, layout as Xs, scaled by grad_scale
    long long gs_gs = 0;
    float* gXt = nullptr;
    long long gt_gs = 0;
    float grad_scale = 1.f;
    // optional (materialised-W path only, mmd_head_fusable): fuse the head layer's DX
    // into the gradient GEMM (an extra K block + the epilogue).  hd_out[r, p] = (grad_scale * g[r, p] +
    // sum_j hd_dz[r, j] hd_W[p, j]) * (z[r, p] > 0), laid out as gXs; gXs/gXt are
    // then not written.  hd_colsum (or null) gets per-32-row-block column sums.
    const float* hd_dz = nullptr;   // [G][m+n][hd_n]
    long long hd_dz_gs = 0;
    const float* hd_W = nullptr;    // [G][d][hd_n]
    long long hd_w_gs = 0;
    int hd_n = 0;                   // <= 32
    float* hd_out = nullptr;
    float* hd_colsum = nullptr;
    // optional: the ReLU mask of z (= Xs) as bits [G][m+n][hd_zbits_ld] (the FWD
    // epilogue's); with it the fused head's mask comes from the bits (k_mmd_tc.cu)
    const uint32_t* hd_zbits = nullptr;
    long long hd_zbits_gs = 0, hd_zbits_ld = 0;
    int* flags = nullptr;
    bool tc = false;                // run on the tcgen05 path (k_mmd_tc.cu)
    unsigned long long* trace = nullptr;  // diagnostics (k_mmd_tc.cu)
};
int mmd_blocks_per_group(const MmdArgs& a);  // partial-sum blocks (depends on a.tc)
bool mmd_tc_supported(const MmdArgs& a);
int mmd_tc_blocks_per_group(const MmdArgs& a);
size_t mmd_tc_scratch_bytes(const MmdArgs& a);
// true when launch_mmd_tc fuses the head DX described by a.hd_* (materialised-W
// path, hd_n <= 32, (m + n) % 32 == 0)
bool mmd_head_fusable(const MmdArgs& a);
// true when launch_mmd_tc takes the materialised-W path for these arguments
bool mmd_w_path(const MmdArgs& a);
constexpr int kMmdTileRows = 128;  // W-path tile (mtk_mmd_gaussian_tiles granularity)
// stages: 1 = prep pass (tf32 planes, norms, fused beta), 2 = the pair kernel;
// the same scratch must be passed to both.
constexpr int kMmdPrep = 1, kMmdPairs = 2;
void launch_mmd_tc(const MmdArgs& a, void* scratch, cudaStream_t s, int stages = kMmdPrep | kMmdPairs);
size_t mmd_beta_scratch_bytes(const MmdArgs& a);
void launch_mmd_beta(const MmdArgs& a, double* beta_out, double* scratch, cudaStream_t s);
// beta from partials laid out as beta_partial writes them ([G][P][d+1], P = ceil(N / 32))
void launch_mmd_beta_finish(const MmdArgs& a, const double* part, double* beta_out, cudaStream_t s);
constexpr int kBetaRows = 32;
void launch_mmd_pairs(const MmdArgs& a, cudaStream_t s);
// value[g] = cSS*ss + cTT*tt + cST*st from the per-block partials (fixed order)
void launch_mmd_finish(const MmdArgs& a, double* value, double* sums3, cudaStream_t s);

// attack stage
void launch_gather_rows(const uint32_t* src, long long src_rows, int d, const long long* idx, int G,
                        int nb, uint32_t* out, int out_rows, int row0, int* flags, cudaStream_t s);
void launch_softmax(const float* logits, long long rows, int C, float* probs, cudaStream_t s);
void launch_features(const float* logits, long long rows, int C, int k, const int32_t* labels,
                     float* feats, int* flags, cudaStream_t s);
void launch_column(const float* logits, long long rows, int C, int col, float* out,
                   cudaStream_t s);
// fused attack scoring (k_attack.cu): the [3, 64, 2] attack model over <= 16 classes
bool attack_fused_ok(int C, int K, int H, int O);
void attack_auc_fused(Ctx& ctx, const float* logits, long long rows, int C, const float* W0, const float* b0,
                      const float* W1, const float* b1, const uint8_t* labels, float* score_out, double* auc,
                      double* acc, bool* flags_clear = nullptr);
// flags_clear (optional): set when the context's device flags came back clear
// with the result (the mailbox path), so the caller can skip check_flags
void auc_device(Ctx& ctx, const float* scores, const uint8_t* labels, long long n, double* auc,
                double* acc, bool* flags_clear = nullptr);

std::string& last_error();

// process-wide count of kernels this library launched (mtk_ctx_launch_count)
unsigned long long& launch_counter();
inline void count_launch() { __atomic_add_fetch(&launch_counter(), 1ULL, __ATOMIC_RELAXED); }

inline void after_launch(Ctx& c, int n = 1) {
    (void)c;
    (void)n;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) fail(MTK_ERROR, std::string("kernel launch: ") + cudaGetErrorString(e));
}

template <class F>
inline int guard(F&& f) {
    try {
        f();
        return MTK_OK;
    } catch (const Failure& e) {
        last_error() = e.what();
        return e.status;
    } catch (const std::bad_alloc&) {
        last_error() = "host allocation failed";
        return MTK_ERROR;
    } catch (const std::exception& e) {
        last_error() = e.what();
        return MTK_ERROR;
    }
}

// Per-DEVICE launch state.  cudaFuncSetAttribute(MaxDynamicSharedMemorySize)
// is per device context and the SM count is per device, so neither may be a
// process-wide static: one process may drive several devices from several
// host threads (one ctx per (host thread, device), mtk.h).  Both are cached
// per device under a mutex.
int current_device();
int device_sm_count(int device);
// permutation(n) of mt::Rng (rng.hpp:48-56, rng_host.cpp) in two stages, so
// a caller can pipeline them: the Fisher-Yates targets (the stream's draws,
// js[n - 1], raw[n - 1] scratch), then the swaps (w[n] scratch)
void rng_permutation_targets(mtk_rng* r, uint64_t n, uint32_t* js, uint64_t* raw);
void permutation_apply(uint64_t n, const uint32_t* js, uint32_t* w, uint64_t* out);
// raise `func`'s dynamic shared-memory limit to `bytes` on the current device
// (once per (device, func))
void ensure_smem_attr(const void* func, int bytes);

// Makes `device` current for the duration of one C-ABI call and restores the
// caller's device afterwards, so a ctx-bound entry point always launches on
// its ctx's device whatever the calling thread last selected.
struct DeviceScope {
    int prev = -1;
    explicit DeviceScope(int device);
    ~DeviceScope();
    DeviceScope(const DeviceScope&) = delete;
    DeviceScope& operator=(const DeviceScope&) = delete;
};

// guard() for entry points bound to a context: the ctx's device is current
// inside f (c may be null; f then reports the null argument itself).
template <class F>
inline int guard_on(const Ctx* c, F&& f) {
    return guard([&] {
        DeviceScope ds(c ? c->device : -1);
        f();
    });
}

inline void need(bool ok, int status, const char* msg) {
    if (!ok) fail(status, msg);
}
inline void need(bool ok, int status, const std::string& msg) {
    if (!ok) fail(status, msg);
}

}  // namespace mtk

struct mtk_ctx : mtk::Ctx {};
