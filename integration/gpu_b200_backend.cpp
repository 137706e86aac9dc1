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

class GpuB200Backend : public Backend {
public:
    explicit GpuB200Backend(int device) {
        // party/alpha are per call (mul_combine carries them), so one context
        ok(spdz_ctx_create(device, 0, 2, 0, &ctx_));
        spdz_capability_t c;
        ok(spdz_capability(ctx_, &c));
        cap_.name = c.name;
        cap_.min_kernel_size = c.min_kernel_size;  // 1: no CPU fallback
        cap_.threads_per_block = c.threads_per_block;
        cap_.executable = c.executable != 0;
    }
    ~GpuB200Backend() override { spdz_ctx_destroy(ctx_); }

    const BackendCapability& capability() const override { return cap_; }

    spdz::ShareVec add_batch(const spdz::ShareVec& x, const spdz::ShareVec& y) override {
        spdz::ShareVec z;
        z.resize(x.lanes());
        std::lock_guard lk(mu_);  // one stream per context; kernels stay pure
        ok(spdz_host_add_batch(ctx_, x.vals.data(), x.macs.data(), x.lanes(), y.vals.data(), y.macs.data(),
                               y.lanes(), z.vals.data(), z.macs.data()));
        return z;
    }

    spdz::ShareVec sub_batch(const spdz::ShareVec& x, const spdz::ShareVec& y) override {
        spdz::ShareVec z;
        z.resize(x.lanes());
        std::lock_guard lk(mu_);
        ok(spdz_host_sub_batch(ctx_, x.vals.data(), x.macs.data(), x.lanes(), y.vals.data(), y.macs.data(),
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
        std::lock_guard lk(mu_);
        ok(spdz_host_mul_mask(ctx_, x.vals.data(), y.vals.data(), x.lanes(), tri, t.a.lanes(), d_out.data(),
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
        std::lock_guard lk(mu_);
        ok(spdz_host_mul_combine(ctx_, tri, t.a.lanes(), d.data(), e.data(), d.size(), party, alpha_share,
                                 z.vals.data(), z.macs.data()));
        return z;
    }

    spdz::ShareVec reduce_add(const spdz::ShareVec& x) override {
        spdz::ShareVec z;
        z.resize(1);
        std::lock_guard lk(mu_);
        ok(spdz_host_reduce_add(ctx_, x.vals.data(), x.macs.data(), x.lanes(), z.vals.data(), z.macs.data()));
        return z;
    }

private:
    spdz_ctx* ctx_ = nullptr;
    BackendCapability cap_;
    std::mutex mu_;
};

}  // namespace

std::shared_ptr<Backend> make_gpu_b200_backend(int device) { return std::make_shared<GpuB200Backend>(device); }

}  // namespace mpc::backend
