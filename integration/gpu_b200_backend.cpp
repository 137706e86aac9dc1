// Reference-side binding: an `mpc::backend::Backend` implementation that a
// maintainer drops into the reference (proj/core/src/) to route its batched
// kernels to the B200 back end through the C ABI of include/spdz_b200.h.
//
//   Replaces: GpuStub (proj/core/src/backend.cpp:90-121), which throws
//   BackendUnavailable on every kernel; same interface (backend.hpp:32-49),
//   same error types (backend.hpp:11-19), same ownership (outputs returned by
//   value, mul_mask resizes d_out/e_out, backend.cpp:59-60).
//
// Registration (the reference lacks an injection hook, runtime.cpp:74,97):
//   registry.register_preferred(mpc::backend::make_gpu_b200_backend(device));
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "mpc/backend.hpp"
#include "spdz_b200.h"

namespace mpc::backend {

namespace {

[[noreturn]] void raise(int rc) {
    const std::string msg = spdz_last_error();
    switch (rc) {
        case SPDZ_ERR_LANE_MISMATCH: throw LaneMismatch(msg);
        case SPDZ_ERR_TRIPLE_SHORTAGE: throw TripleShortage(msg);
        case SPDZ_ERR_BACKEND_UNAVAILABLE: throw BackendUnavailable(msg);
        default: throw std::runtime_error(msg);
    }
}

void ok(int rc) {
    if (rc != SPDZ_OK) raise(rc);
}

// The runtime calls the backend concurrently from its worker threads and open
// continuations (runtime.cpp:221-238, 452-465; kernels must be pure, SPDZ_SPEC 473-474).
// A context owns one CUDA stream and its staging buffers, so each call borrows a
// context from a pool for its duration: concurrent calls run on separate streams
// instead of queueing behind one lock.
class CtxPool {
public:
    explicit CtxPool(int device) : device_(device) {}
    ~CtxPool() {
        for (auto* c : free_) spdz_ctx_destroy(c);
    }
    spdz_ctx* acquire() {
        {
            std::lock_guard lk(mu_);
            if (!free_.empty()) {
                spdz_ctx* c = free_.back();
                free_.pop_back();
                return c;
            }
        }
        spdz_ctx* c = nullptr;  // party/alpha are per call (mul_combine carries them)
        ok(spdz_ctx_create(device_, 0, 2, 0, &c));
        return c;
    }
    void release(spdz_ctx* c) {
        std::lock_guard lk(mu_);
        free_.push_back(c);
    }

private:
    int device_;
    std::mutex mu_;
    std::vector<spdz_ctx*> free_;
};

struct Lease {
    CtxPool& pool;
    spdz_ctx* ctx;
    explicit Lease(CtxPool& p) : pool(p), ctx(p.acquire()) {}
    ~Lease() { pool.release(ctx); }
    Lease(const Lease&) = delete;
    Lease& operator=(const Lease&) = delete;
};

class GpuB200Backend : public Backend {
public:
    explicit GpuB200Backend(int device) : pool_(device) {
        Lease l(pool_);
        spdz_capability_t c;
        ok(spdz_capability(l.ctx, &c));
        cap_.name = c.name;
        cap_.min_kernel_size = c.min_kernel_size;  // 1: no CPU fallback
        cap_.threads_per_block = c.threads_per_block;
        cap_.executable = c.executable != 0;
    }

    const BackendCapability& capability() const override { return cap_; }

    spdz::ShareVec add_batch(const spdz::ShareVec& x, const spdz::ShareVec& y) override {
        spdz::ShareVec z;
        z.resize(x.lanes());
        Lease l(pool_);
        ok(spdz_host_add_batch(l.ctx, x.vals.data(), x.macs.data(), x.lanes(), y.vals.data(), y.macs.data(),
                               y.lanes(), z.vals.data(), z.macs.data()));
        return z;
    }

    spdz::ShareVec sub_batch(const spdz::ShareVec& x, const spdz::ShareVec& y) override {
        spdz::ShareVec z;
        z.resize(x.lanes());
        Lease l(pool_);
        ok(spdz_host_sub_batch(l.ctx, x.vals.data(), x.macs.data(), x.lanes(), y.vals.data(), y.macs.data(),
                               y.lanes(), z.vals.data(), z.macs.data()));
        return z;
    }

    void mul_mask(const spdz::ShareVec& x, const spdz::ShareVec& y, const spdz::TripleShares& t,
                  std::vector<uint32_t>& d_out, std::vector<uint32_t>& e_out) override {
        if (x.lanes() != y.lanes())
            throw LaneMismatch("LaneMismatch: " + std::to_string(x.lanes()) + " vs " + std::to_string(y.lanes()));
        d_out.resize(x.lanes());
        e_out.resize(x.lanes());
        const uint32_t* tri[6] = {t.a.vals.data(), t.a.macs.data(), t.b.vals.data(),
                                  t.b.macs.data(), t.c.vals.data(), t.c.macs.data()};
        Lease l(pool_);
        ok(spdz_host_mul_mask(l.ctx, x.vals.data(), y.vals.data(), x.lanes(), tri, t.a.lanes(), d_out.data(),
                              e_out.data()));
    }

    spdz::ShareVec mul_combine(const spdz::TripleShares& t, const std::vector<uint32_t>& d,
                               const std::vector<uint32_t>& e, int party, uint32_t alpha_share) override {
        if (d.size() != e.size())
            throw LaneMismatch("LaneMismatch: " + std::to_string(d.size()) + " vs " + std::to_string(e.size()));
        spdz::ShareVec z;
        z.resize(d.size());
        const uint32_t* tri[6] = {t.a.vals.data(), t.a.macs.data(), t.b.vals.data(),
                                  t.b.macs.data(), t.c.vals.data(), t.c.macs.data()};
        Lease l(pool_);
        ok(spdz_host_mul_combine(l.ctx, tri, t.a.lanes(), d.data(), e.data(), d.size(), party, alpha_share,
                                 z.vals.data(), z.macs.data()));
        return z;
    }

    spdz::ShareVec reduce_add(const spdz::ShareVec& x) override {
        spdz::ShareVec z;
        z.resize(1);
        Lease l(pool_);
        ok(spdz_host_reduce_add(l.ctx, x.vals.data(), x.macs.data(), x.lanes(), z.vals.data(), z.macs.data()));
        return z;
    }

private:
    CtxPool pool_;
    BackendCapability cap_;
};

}  // namespace

std::shared_ptr<Backend> make_gpu_b200_backend(int device) { return std::make_shared<GpuB200Backend>(device); }

}  // namespace mpc::backend
