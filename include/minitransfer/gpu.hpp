// gpu.hpp -- C++ host wrapper over the C ABI (mtk.h), in the style of the
// reference's header API (namespace mt, exceptions from error.hpp).
//
// Drop-in use next to the reference headers: where `minitransfer/error.hpp`
// and `minitransfer/tape.hpp` are on the include path, failures throw the
// reference's own classes (mt::ShapeError, mt::ValueError, ...) and banks
// exchange parameters as mt::Parameter lists in optimizer_step order
// (W0, b0, W1, b1, ...; optim.hpp:13-14).  Without them, compatible classes
// are declared here.
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "minitransfer/mtk.h"

#if __has_include("minitransfer/tape.hpp")
#include "minitransfer/error.hpp"
#include "minitransfer/tape.hpp"
#define MT_GPU_HAVE_REFERENCE 1
#else
namespace mt {
struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ShapeError : Error {
    using Error::Error;
};
struct ValueError : Error {
    using Error::Error;
};
struct ConfigError : Error {
    using Error::Error;
};
struct DataError : Error {
    using Error::Error;
};
struct CheckpointError : DataError {
    using DataError::DataError;
};
struct VersionError : CheckpointError {
    using CheckpointError::CheckpointError;
};
struct DigestError : CheckpointError {
    using CheckpointError::CheckpointError;
};
struct TruncatedError : CheckpointError {
    using CheckpointError::CheckpointError;
};
}  // namespace mt
#define MT_GPU_HAVE_REFERENCE 0
#endif

namespace mt {
namespace gpu {

// status code -> the reference exception class (error.hpp:10-51)
[[noreturn]] inline void throw_status(int st, const char* what = nullptr) {
    std::string msg = mtk_last_error();
    if (what) msg = std::string(what) + ": " + msg;
    switch (st) {
        case MTK_SHAPE_ERROR: throw ShapeError(msg);
        case MTK_VALUE_ERROR: throw ValueError(msg);
        case MTK_CONFIG_ERROR: throw ConfigError(msg);
        case MTK_DATA_ERROR: throw DataError(msg);
        case MTK_CHECKPOINT_ERROR: throw CheckpointError(msg);
        case MTK_VERSION_ERROR: throw VersionError(msg);
        case MTK_DIGEST_ERROR: throw DigestError(msg);
        case MTK_TRUNCATED_ERROR: throw TruncatedError(msg);
        default: throw Error(msg);
    }
}
inline void check(int st, const char* what = nullptr) {
    if (st != MTK_OK) throw_status(st, what);
}

// One per (host thread, device), like one Tape per thread (tape.hpp:84-85).
class Context {
  public:
    explicit Context(int device = 0, void* cuda_stream = nullptr) {
        check(mtk_ctx_create(device, cuda_stream, &h_), "mtk_ctx_create");
    }
    ~Context() { mtk_ctx_destroy(h_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    void synchronize() { check(mtk_ctx_synchronize(h_), "synchronize"); }
    mtk_ctx* get() const { return h_; }

  private:
    mtk_ctx* h_ = nullptr;
};

// mt::Rng (rng.hpp:13-75), bit-exact, host-side.
class Rng {
  public:
    explicit Rng(uint64_t seed) { check(mtk_rng_create(seed, &h_)); }
    ~Rng() { mtk_rng_destroy(h_); }
    Rng(Rng&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
    Rng(const Rng&) = delete;
    uint64_t next_u64() { return mtk_rng_next_u64(h_); }
    double uniform(double lo = 0.0, double hi = 1.0) { return mtk_rng_uniform(h_, lo, hi); }
    double normal() { return mtk_rng_normal(h_); }
    uint64_t below(uint64_t n) { return mtk_rng_below(h_, n); }
    std::vector<std::size_t> permutation(std::size_t n) {
        std::vector<uint64_t> p(n);
        check(mtk_rng_permutation(h_, n, p.data()));
        return std::vector<std::size_t>(p.begin(), p.end());
    }
    Rng split(uint64_t stream) {
        mtk_rng* c = nullptr;
        check(mtk_rng_split(h_, stream, &c));
        return Rng(c);
    }
    mtk_rng* get() const { return h_; }

  private:
    explicit Rng(mtk_rng* h) : h_(h) {}
    mtk_rng* h_ = nullptr;
};

// G independent MLPs trained as one grouped step (mtk_bank_*).
class Bank {
  public:
    Bank(Context& ctx, int G, const std::vector<int>& dims, int n_heads = 1)
        : G_(G), dims_(dims), n_heads_(n_heads) {
        if (dims.size() < 2) throw ShapeError("Bank: need at least one layer");
        check(mtk_bank_create(ctx.get(), G, (int)dims.size() - 1, dims.data(), n_heads, &h_),
              "mtk_bank_create");
    }
    ~Bank() { mtk_bank_destroy(h_); }
    Bank(const Bank&) = delete;
    Bank& operator=(const Bank&) = delete;

    int n_mats() const { return (int)dims_.size() - 1 + n_heads_ - 1; }
    void init_params(int model, Rng& r) { check(mtk_bank_init_params(h_, model, r.get())); }

    void set_params(int model, const std::vector<const double*>& W,
                    const std::vector<const double*>& b) {
        check(mtk_bank_set_params(h_, model, W.data(), b.data()), "set_params");
    }
    void get_params(int model, const std::vector<double*>& W, const std::vector<double*>& b) {
        check(mtk_bank_get_params(h_, model, W.data(), b.data()), "get_params");
    }
#if MT_GPU_HAVE_REFERENCE
    // params in optimizer_step order: W0, b0, W1, b1, ... (optim.hpp:13-14)
    void set_params(int model, const std::vector<Parameter*>& params) {
        std::vector<const double*> W, b;
        for (std::size_t i = 0; i + 1 < params.size(); i += 2) {
            W.push_back(params[i]->value.data());
            b.push_back(params[i + 1]->value.data());
        }
        set_params(model, W, b);
    }
    void get_params(int model, const std::vector<Parameter*>& params) {
        std::vector<double*> W, b;
        for (std::size_t i = 0; i + 1 < params.size(); i += 2) {
            W.push_back(params[i]->value.data());
            b.push_back(params[i + 1]->value.data());
        }
        get_params(model, W, b);
    }
#endif
    // one SGD step of all G models from device buffers; returns per-model CE loss
    std::vector<double> train_step(const mtk_step& s, std::vector<double>* mmd = nullptr) {
        std::vector<double> loss(G_);
        if (mmd) mmd->resize(G_);
        check(mtk_bank_train_step(h_, &s, loss.data(), mmd ? mmd->data() : nullptr), "train_step");
        return loss;
    }
    // checkpoint / resume: bit-exact, Adam state included
    void save(const std::string& path) { check(mtk_bank_save(h_, path.c_str()), "save"); }
    // a fresh Adam state (OptimizerState, optim.hpp:13-26): zero moments, step 0
    void reset_optimizer() { check(mtk_bank_reset_optimizer(h_), "reset_optimizer"); }
    void forward(const float* X, int B, float* logits, int head = 0, float* hidden = nullptr) {
        check(mtk_bank_forward(h_, X, B, head, logits, hidden), "forward");
    }
    mtk_bank* get() const { return h_; }

  private:
    int G_;
    std::vector<int> dims_;
    int n_heads_;
    mtk_bank* h_ = nullptr;
};

struct MmdResult {
    double value = 0.0;
    double beta = 0.0;
};

// multi-bandwidth Gaussian MMD^2 (biased V-statistic) and gradients (device)
inline MmdResult mmd_gaussian(Context& ctx, const float* Xs, int64_t m, const float* Xt,
                              int64_t n, int d, const std::vector<double>& mult = {},
                              double beta = 0.0, float* gXs = nullptr, float* gXt = nullptr) {
    MmdResult r;
    check(mtk_mmd_gaussian(ctx.get(), Xs, m, Xt, n, d, mult.empty() ? nullptr : mult.data(),
                           (int)mult.size(), beta, &r.value, &r.beta, gXs, gXt),
          "mmd_gaussian");
    return r;
}

inline double auc(Context& ctx, const float* scores, const uint8_t* labels, int64_t n,
                  double* accuracy = nullptr) {
    double a = 0.0;
    check(mtk_auc(ctx.get(), scores, labels, n, &a, accuracy), "auc");
    return a;
}

// the attack evaluation in one call: device logits [rows, C] of the queried
// models -> AUC (and accuracy at 0.5) of `attack` (model 0) as the scorer
inline double attack_auc(Bank& attack, const float* logits, int64_t rows, int C, const uint8_t* labels,
                         double* accuracy = nullptr, float* scores = nullptr) {
    double a = 0.0;
    check(mtk_attack_auc(attack.get(), logits, rows, C, labels, &a, accuracy, scores), "attack_auc");
    return a;
}

}  // namespace gpu
}  // namespace mt
