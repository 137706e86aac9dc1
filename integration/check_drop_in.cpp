// Drop-in check: the reference's own protocol_tests.cpp:280-330 scenario with
// the reference's Dealer, BackendRegistry and spdz::beaver_combine, but the
// preferred backend is the B200 one (gpu_b200_backend.cpp) instead of GpuStub.
// Every GPU result is compared bit-for-bit with the reference CpuBackend.
// Exit 0 = all checks passed.  Built by integration/Makefile (needs the
// reference headers and oracle/_ref/libllspdz_ref.so); runs on the GPU box.
#include <atomic>
#include <cstdio>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "mpc/backend.hpp"
#include "mpc/spdz.hpp"

namespace mpc::backend {
std::shared_ptr<Backend> make_gpu_b200_backend(int device);
}

using namespace mpc;

static std::atomic<int> failures{0};
#define CHECK(c)                                                    \
    do {                                                            \
        if (!(c)) {                                                 \
            std::fprintf(stderr, "FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
            ++failures;                                             \
        }                                                           \
    } while (0)

static std::vector<uint32_t> rand_field_vec(size_t n, uint64_t seed) {  // tests/test_util.hpp:46-51
    std::mt19937_64 rng(seed);
    std::vector<uint32_t> v(n);
    for (auto& x : v) x = uint32_t(rng() % kPrime);
    return v;
}

int main() {
    backend::BackendRegistry reg(1);
    auto gpu = backend::make_gpu_b200_backend(0);
    reg.register_preferred(gpu);
    CHECK(gpu->capability().executable);
    CHECK(&reg.select(1) == gpu.get());  // min_kernel_size 1: every size routes to the GPU
    auto cpu = backend::make_cpu_backend();

    for (size_t lanes : {size_t(1), size_t(513), size_t(1) << 20}) {
        spdz::Dealer d(2, 12);
        auto xs = rand_field_vec(lanes, 9), ys = rand_field_vec(lanes, 10);
        auto X = d.share(xs), Y = d.share(ys);
        auto& be = reg.select(lanes);
        auto s = be.add_batch(X[0], Y[0]);
        auto s_ref = cpu->add_batch(X[0], Y[0]);
        CHECK(s.vals == s_ref.vals && s.macs == s_ref.macs);
        auto df = be.sub_batch(X[0], Y[0]);
        auto df_ref = cpu->sub_batch(X[0], Y[0]);
        CHECK(df.vals == df_ref.vals && df.macs == df_ref.macs);
        auto r = be.reduce_add(X[0]);
        auto r_ref = cpu->reduce_add(X[0]);
        CHECK(r.vals == r_ref.vals && r.macs == r_ref.macs);
        auto T = d.triples(lanes);
        std::vector<uint32_t> dv(lanes, 0), ev(lanes, 0);
        for (int i = 0; i < 2; ++i)
            for (size_t j = 0; j < lanes; ++j) {
                dv[j] = fp::add(dv[j], fp::sub(X[i].vals[j], T[i].a.vals[j]));
                ev[j] = fp::add(ev[j], fp::sub(Y[i].vals[j], T[i].b.vals[j]));
            }
        for (int i = 0; i < 2; ++i) {
            std::vector<uint32_t> d0, e0, d1, e1;
            be.mul_mask(X[i], Y[i], T[i], d0, e0);
            cpu->mul_mask(X[i], Y[i], T[i], d1, e1);
            CHECK(d0 == d1 && e0 == e1);
            auto z = be.mul_combine(T[i], dv, ev, i, d.alpha_share(i));
            auto z_ref = spdz::beaver_combine(T[i], dv, ev, i, d.alpha_share(i));
            CHECK(z.vals == z_ref.vals && z.macs == z_ref.macs);
        }
    }
    // concurrent callers (the runtime's worker threads, runtime.cpp:452-465): each thread's
    // Beaver mask/combine through the shared backend equals the CpuBackend's
    {
        std::vector<std::thread> th;
        for (int w = 0; w < 8; ++w)
            th.emplace_back([&, w] {
                const size_t lanes = 4096 + 97 * w;
                spdz::Dealer d(2, 100 + w);
                auto X = d.share(rand_field_vec(lanes, 200 + w)), Y = d.share(rand_field_vec(lanes, 300 + w));
                auto T = d.triples(lanes);
                for (int rep = 0; rep < 4; ++rep)
                    for (int i = 0; i < 2; ++i) {
                        std::vector<uint32_t> d0, e0, d1, e1;
                        gpu->mul_mask(X[i], Y[i], T[i], d0, e0);
                        cpu->mul_mask(X[i], Y[i], T[i], d1, e1);
                        CHECK(d0 == d1 && e0 == e1);
                        auto z = gpu->mul_combine(T[i], d0, e0, i, d.alpha_share(i));
                        auto z_ref = spdz::beaver_combine(T[i], d0, e0, i, d.alpha_share(i));
                        CHECK(z.vals == z_ref.vals && z.macs == z_ref.macs);
                        auto s = gpu->add_batch(X[i], Y[i]);
                        auto s_ref = cpu->add_batch(X[i], Y[i]);
                        CHECK(s.vals == s_ref.vals && s.macs == s_ref.macs);
                    }
            });
        for (auto& t : th) t.join();
    }
    bool threw = false;
    try {
        spdz::ShareVec a, b;
        a.resize(4);
        gpu->add_batch(a, b);
    } catch (const backend::LaneMismatch&) {
        threw = true;
    }
    CHECK(threw);
    threw = false;
    try {
        spdz::Dealer d(2, 3);
        auto T = d.triples(3);
        spdz::ShareVec a;
        a.resize(5);
        std::vector<uint32_t> dd, ee;
        gpu->mul_mask(a, a, T[0], dd, ee);
    } catch (const backend::TripleShortage&) {
        threw = true;
    }
    CHECK(threw);
    std::printf("%s: %d failures\n", failures ? "FAIL" : "PASS", failures.load());
    return failures ? 1 : 0;
}
