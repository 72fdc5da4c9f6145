// rng_host.cpp -- host-side bit-exact sampling for the shadow sweep.
//
// Restates the reference's mt::Rng (rng.hpp:13-75) on std::mt19937_64, whose
// output sequence is fixed by the C++ standard, with the same hand-rolled
// distributions, so every draw, permutation, member/non-member split and
// weight initialisation is bit-identical to the reference.  Compiled with
// -ffp-contract=off (rng.hpp:22 changes bits
// under FMA contraction).  Sampling never runs on the device.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <mutex>
#include <thread>
#include <vector>

#include "minitransfer/mtk.h"

struct mtk_rng {
    std::mt19937_64 eng;
    bool cached = false;
    double cache = 0.0;
    explicit mtk_rng(uint64_t seed) : eng(seed) {}

    double unit() { return static_cast<double>(eng() >> 11) * 0x1.0p-53; }  // rng.hpp:20
    double range(double lo, double hi) {                                  // rng.hpp:22
        const double u = unit();
        const double width = hi - lo;
        const double off = width * u;
        return lo + off;
    }
    double gauss() {  // rng.hpp:24-37, Box-Muller pair, second value cached
        if (cached) {
            cached = false;
            return cache;
        }
        const double u1 = 1.0 - unit();
        const double u2 = unit();
        const double rad = std::sqrt(-2.0 * std::log(u1));
        const double theta = 6.28318530717958647692 * u2;
        cache = rad * std::sin(theta);
        cached = true;
        return rad * std::cos(theta);
    }
    uint64_t bounded(uint64_t n) {  // rng.hpp:39-46, unbiased rejection
        if (n == 0) return 0;
        const uint64_t cut = UINT64_MAX - UINT64_MAX % n;
        for (;;) {
            const uint64_t x = eng();
            if (x < cut) return x % n;
        }
    }
};

extern "C" void mtk_internal_set_error(const char* msg);  // capi.cu

namespace {
int set_err(int s, const char* m) {
    mtk_internal_set_error(m);
    return s;
}
}  // namespace

extern "C" {

int mtk_rng_create(uint64_t seed, mtk_rng** out) {
    if (!out) return set_err(MTK_VALUE_ERROR, "mtk_rng_create: null out");
    *out = new mtk_rng(seed);
    return MTK_OK;
}

int mtk_rng_destroy(mtk_rng* r) {
    delete r;
    return MTK_OK;
}

// rng.hpp:65-69: one parent draw xor a stream constant seeds the child
int mtk_rng_split(mtk_rng* parent, uint64_t stream, mtk_rng** out) {
    if (!parent || !out) return set_err(MTK_VALUE_ERROR, "mtk_rng_split: null argument");
    const uint64_t s = parent->eng() ^ (0x9e3779b97f4a7c15ULL * (stream + 1));
    *out = new mtk_rng(s);
    return MTK_OK;
}

uint64_t mtk_rng_next_u64(mtk_rng* r) { return r->eng(); }
double mtk_rng_uniform(mtk_rng* r, double lo, double hi) { return r->range(lo, hi); }
double mtk_rng_normal(mtk_rng* r) { return r->gauss(); }
uint64_t mtk_rng_below(mtk_rng* r, uint64_t n) { return r->bounded(n); }

// rng.hpp:50-63: identity then Fisher-Yates swaps from the top.  The swap
// targets depend only on the stream (bounded(n), bounded(n - 1), ...), so
// they are drawn first, in the same order; the swaps then run with the
// random targets prefetched a few iterations ahead, on a 32-bit working
// array when n < 2^32 (the attack sweep permutes 2^20 rows every epoch:
// the swaps were bound by cache misses).  Same stream use, same result.
}  // extern "C"

namespace mtk {
// the Fisher-Yates targets of permutation(n) (n >= 2, n < 2^32): js[k] =
// bounded(n - k), k = 0 .. n - 2, drawn in stream order -- the raw words in
// one sequential pass, the reductions (two 64-bit divisions each) on all
// cores.  A rejection (a word >= the cut: ~top / 2^64) would shift the
// stream: then the engine is restored and the targets drawn one by one, as
// bounded() does.
void rng_permutation_targets(mtk_rng* r, uint64_t n, uint32_t* js, uint64_t* raw) {
    const std::mt19937_64 saved = r->eng;
    for (uint64_t k = 0; k + 1 < n; ++k) raw[k] = r->eng();
    unsigned nt = std::thread::hardware_concurrency();
    nt = nt == 0 ? 1 : (nt > 16 ? 16 : nt);
    if (n < (1u << 16)) nt = 1;
    std::vector<char> rejected(nt, 0);
    auto part = [&](unsigned t) {
        const uint64_t a = (n - 1) * t / nt, b = (n - 1) * (t + 1) / nt;
        for (uint64_t k = a; k < b; ++k) {
            const uint64_t top = n - k, cut = UINT64_MAX - UINT64_MAX % top;
            if (raw[k] >= cut) rejected[t] = 1;
            js[k] = static_cast<uint32_t>(raw[k] % top);
        }
    };
    std::vector<std::thread> th;
    for (unsigned t = 1; t < nt; ++t) th.emplace_back(part, t);
    part(0);
    for (auto& x : th) x.join();
    bool any = false;
    for (char c : rejected) any |= c != 0;
    if (any) {
        r->eng = saved;
        for (uint64_t k = 0, top = n; top > 1; --top, ++k) js[k] = static_cast<uint32_t>(r->bounded(top));
    }
}

// the swaps of permutation(n) for targets js, top down (w: n words of scratch)
void permutation_apply(uint64_t n, const uint32_t* js, uint32_t* w, uint64_t* out) {
    for (uint64_t i = 0; i < n; ++i) w[i] = static_cast<uint32_t>(i);
    constexpr uint64_t kAhead = 16;
    const uint64_t steps = n - 1;
    for (uint64_t k = 0; k < steps; ++k) {
        if (k + kAhead < steps) __builtin_prefetch(&w[js[k + kAhead]], 1, 0);
        const uint64_t top = n - k, j = js[k];
        const uint32_t t = w[top - 1];
        w[top - 1] = w[j];
        w[j] = t;
    }
    for (uint64_t i = 0; i < n; ++i) out[i] = w[i];
}
}  // namespace mtk

extern "C" {

int mtk_rng_permutation(mtk_rng* r, uint64_t n, uint64_t* out) {
    if (!r || (!out && n)) return set_err(MTK_VALUE_ERROR, "mtk_rng_permutation: null argument");
    if (n < 2 || n >= (1ull << 32)) {
        for (uint64_t i = 0; i < n; ++i) out[i] = i;
        for (uint64_t top = n; top > 1; --top) {
            const uint64_t j = r->bounded(top);
            const uint64_t t = out[top - 1];
            out[top - 1] = out[j];
            out[j] = t;
        }
        return MTK_OK;
    }
    // working buffers reused across calls (fresh 16 MB per call cost ~6 ms of
    // page faults); a concurrent caller takes its own
    static std::mutex mu;
    static std::vector<uint32_t> js_s, w_s;
    static std::vector<uint64_t> raw_s;
    std::unique_lock<std::mutex> lk(mu, std::try_to_lock);
    std::vector<uint32_t> js_l, w_l;
    std::vector<uint64_t> raw_l;
    std::vector<uint32_t>& js = lk.owns_lock() ? js_s : js_l;
    std::vector<uint32_t>& w = lk.owns_lock() ? w_s : w_l;
    std::vector<uint64_t>& raw = lk.owns_lock() ? raw_s : raw_l;
    if (js.size() < n - 1) js.resize(n - 1);
    if (w.size() < n) w.resize(n);
    if (raw.size() < n - 1) raw.resize(n - 1);
    mtk::rng_permutation_targets(r, n, js.data(), raw.data());
    mtk::permutation_apply(n, js.data(), w.data(), out);
    return MTK_OK;
}

int mtk_rng_fill_normal(mtk_rng* r, double* out, uint64_t n) {
    if (!r || (!out && n)) return set_err(MTK_VALUE_ERROR, "mtk_rng_fill_normal: null argument");
    for (uint64_t i = 0; i < n; ++i) out[i] = r->gauss();
    return MTK_OK;
}

// The population draws are sequential (one mt19937_64 stream: a label by
// rejection, then d Box-Muller normals whose pairs straddle rows), but the
// transcendentals dominate (19.3 M normals for the sweep's default pools:
// ~0.4 s on one core).  So the rows go in blocks: the calling thread takes
// every raw draw of block b + 1 -- the labels, and each Box-Muller pair's two
// raw words -- in stream order, while the other host cores turn block b's
// pairs into normals (the same expressions as gauss(), so bit-identical) and
// rows.  Two block-sized word buffers, no whole-stream intermediate arrays.
namespace {
struct SynthBlock {
    uint64_t row0 = 0, rows = 0;
    bool cached_in = false;  // the block's first normal is the pending sin value `carry`
    double carry = 0.0;
    std::vector<uint64_t> words;  // two per new Box-Muller pair, stream order
};
inline void box_muller(uint64_t w1, uint64_t w2, double& c, double& s) {  // gauss(), rng.hpp:24-37
    const double u1 = 1.0 - static_cast<double>(w1 >> 11) * 0x1.0p-53;
    const double u2 = static_cast<double>(w2 >> 11) * 0x1.0p-53;
    const double rad = std::sqrt(-2.0 * std::log(u1));
    const double theta = 6.28318530717958647692 * u2;
    s = rad * std::sin(theta);
    c = rad * std::cos(theta);
}
}  // namespace

int mtk_synth(mtk_rng* r, int C, int d, uint64_t n, const double* mu, const double* shift,
              double* X64, float* X32, int32_t* y) {
    if (!r || !mu || !y) return set_err(MTK_VALUE_ERROR, "mtk_synth: null argument");
    if (C <= 0 || d <= 0) return set_err(MTK_SHAPE_ERROR, "mtk_synth: zero dimension");
    const uint64_t total = n * static_cast<uint64_t>(d);
    unsigned nt = std::thread::hardware_concurrency();
    nt = nt == 0 ? 1 : (nt > 32 ? 32 : nt);
    if (total < (1u << 16)) nt = 1;
    const uint64_t R = std::max<uint64_t>(1, (uint64_t(1) << 20) / static_cast<uint64_t>(d));  // rows per block
    bool cached = r->cached;
    double pending = r->cache;  // the value a cached gauss() call returns
    // sequential: block b's labels and pair words; leaves the cache state
    auto draw = [&](SynthBlock& B, uint64_t row0) {
        B.row0 = row0;
        B.rows = std::min<uint64_t>(R, n - row0);
        B.cached_in = cached;
        B.carry = pending;
        B.words.clear();
        for (uint64_t i = row0; i < row0 + B.rows; ++i) {
            y[i] = static_cast<int32_t>(r->bounded(static_cast<uint64_t>(C)));
            for (int k = 0; k < d; ++k) {
                if (cached) {
                    cached = false;
                } else {
                    B.words.push_back(r->eng());
                    B.words.push_back(r->eng());
                    cached = true;
                }
            }
        }
        if (cached && !B.words.empty()) {  // the block's last pair leaves its sin value pending
            double c, sv;
            const size_t m = B.words.size();
            box_muller(B.words[m - 2], B.words[m - 1], c, sv);
            pending = sv;
        }
    };
    // parallel: block element e (stream order) -> X[row0 + e / d][e % d]
    auto put = [&](const SynthBlock& B, uint64_t e, double g) {
        const uint64_t i = B.row0 + e / static_cast<uint64_t>(d);
        const int k = static_cast<int>(e % static_cast<uint64_t>(d));
        double v = mu[static_cast<size_t>(y[i]) * d + k] + g;
        if (shift) v = v + shift[k];
        if (X64) X64[i * d + k] = v;
        if (X32) X32[i * d + k] = static_cast<float>(v);
    };
    auto form = [&](const SynthBlock& B, size_t pa, size_t pb) {  // pairs [pa, pb) of the block
        const uint64_t elems = B.rows * static_cast<uint64_t>(d);
        const uint64_t off = B.cached_in ? 1 : 0;
        if (pa == 0 && B.cached_in) put(B, 0, B.carry);
        for (size_t p = pa; p < pb; ++p) {
            double c, sv;
            box_muller(B.words[2 * p], B.words[2 * p + 1], c, sv);
            const uint64_t e = off + 2 * p;
            put(B, e, c);
            if (e + 1 < elems) put(B, e + 1, sv);  // else: pending for the next block
        }
    };
    auto form_all = [&](const SynthBlock& B, unsigned threads) {
        const size_t np = B.words.size() / 2;
        if (threads <= 1 || np < 4096) {
            form(B, 0, np);
            return;
        }
        std::vector<std::thread> th;
        for (unsigned t = 1; t < threads; ++t)
            th.emplace_back([&, t] { form(B, np * t / threads, np * (t + 1) / threads); });
        form(B, 0, np / threads);
        for (auto& x : th) x.join();
    };
    SynthBlock blk[2];
    if (n == 0) return MTK_OK;
    draw(blk[0], 0);
    int cur = 0;
    for (uint64_t row0 = 0; row0 < n; row0 += R) {
        const uint64_t next = row0 + R;
        if (next < n && nt > 1) {
            // the other cores form block `cur` while this thread draws the next one
            std::thread former([&, cur] { form_all(blk[cur], nt - 1); });
            draw(blk[cur ^ 1], next);
            former.join();
        } else {
            form_all(blk[cur], nt);
            if (next < n) draw(blk[cur ^ 1], next);
        }
        cur ^= 1;
    }
    // the generator's Box-Muller cache as the sequential draws leave it
    r->cached = cached;
    r->cache = cached ? pending : r->cache;
    return MTK_OK;
}

}  // extern "C"
