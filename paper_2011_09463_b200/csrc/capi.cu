// capi.cu -- the C ABI (include/minitransfer/mtk.h): contexts, error
// reporting, the MMD and attack entry points, diagnostics.  The model bank
// lives in bank.cu.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include "internal.h"

namespace mtk {
std::string& last_error() {
    thread_local std::string e;
    return e;
}
unsigned long long& launch_counter() {
    static unsigned long long n = 0;
    return n;
}

namespace {
constexpr int kMaxDevices = 64;
std::mutex g_dev_mu;
int g_sms[kMaxDevices] = {};
std::set<std::pair<int, const void*>> g_smem_attr;  // (device, kernel) already raised
}  // namespace

int current_device() {
    int dev = 0;
    MTK_CUDA(cudaGetDevice(&dev));
    return dev;
}

int device_sm_count(int device) {
    need(device >= 0 && device < kMaxDevices, MTK_ERROR, "device index out of range");
    std::lock_guard<std::mutex> lk(g_dev_mu);
    if (!g_sms[device]) MTK_CUDA(cudaDeviceGetAttribute(&g_sms[device], cudaDevAttrMultiProcessorCount, device));
    return g_sms[device];
}

void ensure_smem_attr(const void* func, int bytes) {
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(g_dev_mu);
    if (g_smem_attr.count({dev, func})) return;
    MTK_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    g_smem_attr.insert({dev, func});
}

DeviceScope::DeviceScope(int device) {
    if (device < 0) return;
    int cur = -1;
    MTK_CUDA(cudaGetDevice(&cur));
    if (cur != device) {
        MTK_CUDA(cudaSetDevice(device));
        prev = cur;
    }
}

DeviceScope::~DeviceScope() {
    if (prev >= 0) cudaSetDevice(prev);
}
}  // namespace mtk

extern "C" void mtk_internal_set_error(const char* msg) { mtk::last_error() = msg ? msg : ""; }

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

void* Ctx::big(size_t bytes) {
    if (bytes > big_bytes) {
        if (d_big) MTK_CUDA(cudaFree(d_big));  // synchronizes: in-flight users are done
        d_big = nullptr;
        MTK_CUDA(cudaMalloc(&d_big, bytes));
        big_bytes = bytes;
    }
    return d_big;
}

void* Ctx::sweep_buf(size_t bytes) {
    if (bytes > sweep_bytes) {
        if (d_sweep) MTK_CUDA(cudaFree(d_sweep));  // synchronizes: in-flight users are done
        d_sweep = nullptr;
        MTK_CUDA(cudaMalloc(&d_sweep, bytes));
        sweep_bytes = bytes;
    }
    return d_sweep;
}

uint32_t* Ctx::auc_l2(size_t bytes) {
    if (bytes > auc_l2_bytes) {
        if (d_auc_l2) MTK_CUDA(cudaFree(d_auc_l2));  // synchronizes: in-flight users are done
        d_auc_l2 = nullptr;
        MTK_CUDA(cudaMalloc(&d_auc_l2, bytes));
        MTK_CUDA(cudaMemsetAsync(d_auc_l2, 0, bytes, stream));
        auc_l2_bytes = bytes;
    }
    return d_auc_l2;
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
        if (f & kFlagBadIndex) fail(MTK_VALUE_ERROR, "gather_rows: index out of range");
        fail(MTK_ERROR, "non-finite values produced on the device");
    }
}

void* HostBlockPool::get(size_t bytes, size_t* cap) {
    std::lock_guard<std::mutex> lk(mu_);
    size_t best = free_.size();
    for (size_t i = 0; i < free_.size(); ++i)
        if (free_[i].second >= bytes && (best == free_.size() || free_[i].second < free_[best].second)) best = i;
    if (best < free_.size()) {
        void* p = free_[best].first;
        *cap = free_[best].second;
        free_.erase(free_.begin() + (long)best);
        return p;
    }
    void* p = nullptr;
    MTK_CUDA(cudaHostAlloc(&p, bytes, cudaHostAllocPortable));
    all_.push_back(p);
    *cap = bytes;
    return p;
}

void HostBlockPool::put(void* p, size_t cap) {
    std::lock_guard<std::mutex> lk(mu_);
    free_.push_back({p, cap});
}

HostBlockPool::~HostBlockPool() {
    for (void* p : all_) cudaFreeHost(p);
}

HostBlockPool& Ctx::host_pool() {
    if (!host_blocks) host_blocks = new HostBlockPool();
    return *host_blocks;
}

cudaEvent_t Ctx::record(cudaStream_t s) {
    cudaEvent_t& e = ev_ring[ev_next];
    ev_next = (ev_next + 1) % 32;
    if (!e) MTK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    MTK_CUDA(cudaEventRecord(e, s));  // a wait captures the state at call time: reuse is safe
    return e;
}

void Ctx::fork() {
    if (!side) {
        int lo = 0, hi = 0;
        MTK_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        MTK_CUDA(cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, lo));  // lowest priority
    }
    MTK_CUDA(cudaStreamWaitEvent(side, record(stream), 0));
    side_pending = true;
}

void Ctx::join() {
    if (!side_pending) return;
    MTK_CUDA(cudaStreamWaitEvent(stream, record(side), 0));
    side_pending = false;
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

PhaseScope::PhaseScope(Ctx& ctx, int phase, int launches, cudaStream_t s)
    : c(ctx), ph(s && s != ctx.stream ? (int)kPhSide : phase), n(launches), st(s ? s : ctx.stream) {
    if (c.timing) {
        a = c.take_event();
        MTK_CUDA(cudaEventRecord(a, st));
    }
}

PhaseScope::~PhaseScope() {
    if (!a) return;
    cudaEvent_t b = c.take_event();
    cudaEventRecord(b, st);
    c.pending.push_back({ph, {a, b}});
    c.phase_launches[ph] += n;
}

}  // namespace mtk

using namespace mtk;


extern "C" {

int mtk_version(void) { return 100; }

const char* mtk_last_error(void) { return last_error().c_str(); }

int mtk_ctx_create(int device, void* stream, mtk_ctx** out) {
    return guard([&] {
        need(out != nullptr, MTK_VALUE_ERROR, "mtk_ctx_create: null out");
        int n = 0;
        MTK_CUDA(cudaGetDeviceCount(&n));
        need(device >= 0 && device < n, MTK_VALUE_ERROR, "mtk_ctx_create: no such device");
        DeviceScope ds(device);
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
    return guard_on(c, [&] {
        if (!c) return;
        cudaStreamSynchronize(c->stream);
        cudaFree(c->d_flags);
        cudaFree(c->d_scratch);
        cudaFree(c->d_big);
        cudaFree(c->d_auc_l2);
        cudaFree(c->d_sweep);
        if (c->auc_mail) cudaFreeHost(c->auc_mail);
        if (c->pinned) cudaFreeHost(c->pinned);
        if (c->pinned_flags) cudaFreeHost(c->pinned_flags);
        delete c->host_blocks;
        if (c->own_stream) cudaStreamDestroy(c->stream);
        if (c->side) {
            cudaStreamSynchronize(c->side);
            cudaStreamDestroy(c->side);
        }
        for (cudaEvent_t e : c->ev_ring)
            if (e) cudaEventDestroy(e);
        delete c;
    });
}

int mtk_ctx_synchronize(mtk_ctx* c) {
    return guard_on(c, [&] {
        need(c != nullptr, MTK_VALUE_ERROR, "null ctx");
        c->check_flags();
    });
}

int mtk_ctx_launch_count(mtk_ctx* c, uint64_t* out) {
    return guard_on(c, [&] {
        need(c && out, MTK_VALUE_ERROR, "null argument");
        *out = __atomic_load_n(&launch_counter(), __ATOMIC_RELAXED);
    });
}

int mtk_ctx_set_timing(mtk_ctx* c, int on) {
    return guard_on(c, [&] {
        need(c != nullptr, MTK_VALUE_ERROR, "null ctx");
        c->collect_phases();
        c->timing = on != 0;
    });
}

int mtk_ctx_phase_times(mtk_ctx* c, double* ms_host, uint64_t* launches_host) {
    return guard_on(c, [&] {
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
    // one group: the group strides are never stepped, but the materialised-W
    // path checks that [Xs; Xt] (and the gradients) form one [m + n][d] block
    a.xs_gs = a.xt_gs = a.gs_gs = a.gt_gs = (m + n) * (long long)d;
    if (nb > 0) {
        need(mult != nullptr, MTK_VALUE_ERROR, "mmd: null bandwidth multipliers");
        a.nb = nb;
        for (int q = 0; q < nb; ++q) {
            need(mult[q] > 0, MTK_VALUE_ERROR, "mmd: bandwidth multipliers must be positive");
            a.mult[q] = (float)mult[q];
        }
    }
    a.flags = c->d_flags;
    const char* env = getenv("MTK_DISABLE_TC");
    a.tc = !(env && env[0] == '1') && mmd_tc_supported(a);
    if (const char* t = getenv("MTK_MMD_TRACE"))
        a.trace = reinterpret_cast<unsigned long long*>(strtoull(t, nullptr, 0));
    return a;
}

int mtk_mmd_beta(mtk_ctx* c, const float* Xs, int64_t m, const float* Xt, int64_t n, int d,
                 double* beta_host) {
    return guard_on(c, [&] {
        MmdArgs a = mmd_args(c, Xs, m, Xt, n, d, nullptr, 0);
        const size_t part = mmd_beta_scratch_bytes(a);
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
    const int nblk = mmd_blocks_per_group(a);
    const size_t part_beta = mmd_beta_scratch_bytes(a);
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
    } else if (a.tc) {
        a.beta_out = beta_d;  // fused into the prep pass of launch_mmd_tc
    } else {
        launch_mmd_beta(a, beta_d, bscratch, c->stream);
        after_launch(*c, 2);
    }
    a.beta = beta_d;
    a.partial = part_d;
    if (a.tc) {
        void* zs = c->big(mmd_tc_scratch_bytes(a));
        launch_mmd_tc(a, zs, c->stream);
        after_launch(*c, 1);
    } else {
        launch_mmd_pairs(a, c->stream);
    }
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
    return guard_on(c, [&] {
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
    return guard_on(c, [&] {
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

int mtk_mmd_gaussian_tiles(mtk_ctx* c, const float* Xs, int64_t m, const float* Xt, int64_t n, int d,
                           const double* mult, int nb, double beta, int64_t tile_begin, int64_t tile_end,
                           double* tile_partials_host, float* gXs, float* gXt) {
    return guard_on(c, [&] {
        MmdArgs a = mmd_args(c, Xs, m, Xt, n, d, mult, nb);
        need(beta > 0, MTK_VALUE_ERROR, "mmd_tiles: beta must be given (> 0)");
        need(tile_partials_host && gXs && gXt, MTK_VALUE_ERROR, "mmd_tiles: null argument");
        const int64_t T = (m + n + kMmdTileRows - 1) / kMmdTileRows;
        need(tile_begin >= 0 && tile_begin < tile_end && tile_end <= T, MTK_SHAPE_ERROR,
             "mmd_tiles: tile range outside [0, ceil((m + n) / 128))");
        a.gXs = gXs;
        a.gXt = gXt;
        a.tile_begin = tile_begin;
        a.tile_end = tile_end;
        need(a.tc && mmd_w_path(a), MTK_CONFIG_ERROR,
             "mmd_tiles: needs the materialised-W path (Xs, Xt and the gradients each one [m + n, d] "
             "block, d % 4 == 0, d >= 32)");
        const size_t part = (size_t)T * 3 * sizeof(double);
        double* sc = c->scratch(part + 64 * sizeof(double));
        double* beta_d = sc;
        double* part_d = sc + 64;
        MTK_CUDA(cudaMemcpyAsync(beta_d, &beta, sizeof(double), cudaMemcpyHostToDevice, c->stream));
        MTK_CUDA(cudaMemsetAsync(part_d, 0, part, c->stream));
        a.beta = beta_d;
        a.partial = part_d;
        void* zs = c->big(mmd_tc_scratch_bytes(a));
        launch_mmd_tc(a, zs, c->stream);
        after_launch(*c, 1);
        MTK_CUDA(cudaMemcpyAsync(tile_partials_host, part_d, part, cudaMemcpyDeviceToHost, c->stream));
        c->check_flags();
    });
}

int mtk_mmd_value_from_tile_partials(const double* partials, int64_t T, int64_t m, int64_t n,
                                     double* value_host) {
    return guard([&] {
        need(partials && value_host && T >= 1 && m >= 1 && n >= 1, MTK_VALUE_ERROR, "mmd_value: bad argument");
        // mmd_finish_kernel's order and formula, in fp64 (the host is built
        // with -ffp-contract=off): ascending tile rows, then the V-statistic
        double s[3] = {0.0, 0.0, 0.0};
        for (int64_t b = 0; b < T; ++b)
            for (int q = 0; q < 3; ++q) s[q] += partials[b * 3 + q];
        const double md = (double)m, nd = (double)n;
        *value_host = s[0] / (md * md) + s[1] / (nd * nd) - 2.0 * s[2] / (md * nd);
    });
}

// ---- attack stage ----------------------------------------------------------
int mtk_gather_rows(mtk_ctx* c, const void* src, int64_t src_rows, int d, const int64_t* idx, int G,
                    int nb, void* out, int out_rows, int row0) {
    return guard_on(c, [&] {
        need(c && src && idx && out, MTK_VALUE_ERROR, "gather_rows: null argument");
        need(d >= 1 && G >= 0 && nb >= 0 && src_rows >= 1, MTK_SHAPE_ERROR, "gather_rows: bad shape");
        need(row0 >= 0 && row0 + nb <= out_rows, MTK_SHAPE_ERROR, "gather_rows: rows exceed out_rows");
        launch_gather_rows(static_cast<const uint32_t*>(src), src_rows, d,
                           reinterpret_cast<const long long*>(idx), G, nb, static_cast<uint32_t*>(out),
                           out_rows, row0, c->d_flags, c->stream);
        after_launch(*c);
    });
}

int mtk_philox4x64_fill(mtk_ctx* c, uint64_t seed, uint64_t stream, uint64_t ctr0, uint64_t ctr1,
                        int64_t nblocks, uint64_t* out) {
    return guard_on(c, [&] {
        need(c && (out || nblocks == 0), MTK_VALUE_ERROR, "philox: null argument");
        need(nblocks >= 0, MTK_SHAPE_ERROR, "philox: negative block count");
        launch_philox_fill(seed, stream, ctr0, ctr1, nblocks, out, c->stream);
        after_launch(*c);
    });
}

int mtk_counter_normals(mtk_ctx* c, uint64_t seed, uint64_t stream, int64_t first, int64_t count,
                        float* out) {
    return guard_on(c, [&] {
        need(c && (out || count == 0), MTK_VALUE_ERROR, "counter_normals: null argument");
        need(first >= 0 && count >= 0, MTK_SHAPE_ERROR, "counter_normals: negative range");
        launch_counter_normals(seed, stream, first, count, out, c->stream);
        after_launch(*c);
    });
}

int mtk_synth_counter(mtk_ctx* c, uint64_t seed, uint64_t stream, int C, int d, int64_t n,
                      const float* mu, const float* shift, float* X, int32_t* y) {
    return guard_on(c, [&] {
        need(c && mu && X && y, MTK_VALUE_ERROR, "synth_counter: null argument");
        need(C >= 1 && d >= 1 && n >= 1, MTK_SHAPE_ERROR, "synth_counter: zero dimension");
        launch_synth_counter(seed, stream, C, d, n, mu, shift, X, y, c->stream);
        after_launch(*c);
    });
}

int mtk_softmax(mtk_ctx* c, const float* logits, int64_t rows, int C, float* probs) {
    return guard_on(c, [&] {
        need(c && logits && probs, MTK_VALUE_ERROR, "softmax: null argument");
        need(rows >= 1 && C >= 1, MTK_SHAPE_ERROR, "softmax: zero dimension");
        launch_softmax(logits, rows, C, probs, c->stream);
        after_launch(*c);
    });
}

int mtk_posterior_features(mtk_ctx* c, const float* logits, int64_t rows, int C, int k,
                           const int32_t* labels, float* feats) {
    return guard_on(c, [&] {
        need(c && logits && feats, MTK_VALUE_ERROR, "features: null argument");
        need(rows >= 1 && C >= 1, MTK_SHAPE_ERROR, "features: zero dimension");
        need(k >= 1 && k <= C, MTK_VALUE_ERROR, "features: k must be in [1, C]");
        launch_features(logits, rows, C, k, labels, feats, c->d_flags, c->stream);
        after_launch(*c);
    });
}

int mtk_posterior_column(mtk_ctx* c, const float* logits, int64_t rows, int C, int col,
                         float* out) {
    return guard_on(c, [&] {
        need(c && logits && out, MTK_VALUE_ERROR, "posterior_column: null argument");
        need(rows >= 1 && C >= 1, MTK_SHAPE_ERROR, "posterior_column: zero dimension");
        need(col >= 0 && col < C, MTK_VALUE_ERROR, "posterior_column: column out of range");
        launch_column(logits, rows, C, col, out, c->stream);
        after_launch(*c);
    });
}

int mtk_auc(mtk_ctx* c, const float* scores, const uint8_t* labels, int64_t n, double* auc_host,
            double* acc_host) {
    return guard_on(c, [&] {
        need(c && scores && labels, MTK_VALUE_ERROR, "auc: null argument");
        need(n >= 1, MTK_SHAPE_ERROR, "auc: zero rows");
        bool clear = false;
        auc_device(*c, scores, labels, n, auc_host, acc_host, &clear);
        if (!clear) c->check_flags();
    });
}

int mtk_diag_gemm_tf32x3(mtk_ctx* c, int a_mn, int b_mn, int G, int M, int N, int K,
                         const float* A, const float* B, float* Cm) {
    return guard_on(c, [&] {
        need(c && A && B && Cm, MTK_VALUE_ERROR, "diag_gemm: null argument");
        need(G >= 1 && M >= 1 && N >= 1 && K >= 1, MTK_SHAPE_ERROR, "diag_gemm: zero dimension");
        UmmaGemm u;
        u.G = G;
        u.M = M;
        u.N = N;
        u.K = K;
        u.a_mn = a_mn;
        u.b_mn = b_mn;
        u.a = A;
        u.a_rs = a_mn ? M : K;
        u.a_gs = (long long)M * K;
        u.b = B;
        u.b_rs = b_mn ? N : K;
        u.b_gs = (long long)K * N;
        u.epi = Epi::kStore;
        if (const char* e = getenv("MTK_DIAG_EPI")) {  // diagnostics: epilogue variants
            if (e[0] == 's') {  // SGD against C as the master weight, lr = 1e-3
                u.epi = Epi::kSgd;
                u.lr = 1e-3f;
            } else if (e[0] == 'n') {  // epilogue reads TMEM, writes nothing
                u.epi = Epi::kNone;
            } else if (e[0] == 'm') {  // ReLU mask taken from C itself
                u.epi = Epi::kMask;
                u.mask = Cm;
            }
        }
        u.C = Cm;
        u.c_gs = (long long)M * N;
        u.ldc = N;
        u.flags = c->d_flags;
        launch_umma(u, c->stream);
        after_launch(*c);
        c->check_flags();
    });
}

}  // extern "C"
