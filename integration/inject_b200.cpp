// Reference-side injection point for the demo build of the stock PartyRuntime
// (INTEGRATION.md §3 step 3).  integration/runtime_hook.patch adds to the reference's
// PartyRuntime::Impl constructor (runtime.cpp:91-100)
//     if (auto b = injected_preferred_backend()) registry.register_preferred(std::move(b));
// and this file provides the function: the B200 back end (gpu_b200_backend.cpp) on device
// $SPDZ_B200_DEVICE (default 0) unless SPDZ_B200_INJECT=0.  Every BackendRegistry::select
// of every party then routes the batched ops (add/sub, Beaver mask/combine, reduce_add,
// runtime.cpp:141-142, 209, 231, 259, 273, 392) to the GPU (min_kernel_size = 1).
// At exit it reports how many kernels the B200 library launched (evidence the GPU ran).
#include <cstdio>
#include <cstdlib>
#include <memory>

#include "mpc/backend.hpp"
#include "spdz_b200.h"

namespace mpc::backend {
std::shared_ptr<Backend> make_gpu_b200_backend(int device);
}

namespace mpc::runtime {

std::shared_ptr<backend::Backend> injected_preferred_backend() {
    static const std::shared_ptr<backend::Backend> b = []() -> std::shared_ptr<backend::Backend> {
        const char* on = std::getenv("SPDZ_B200_INJECT");
        if (on && on[0] == '0') return nullptr;
        const char* dev = std::getenv("SPDZ_B200_DEVICE");
        std::atexit([] {
            std::fprintf(stderr, "b200 backend injected: %llu kernels launched\n",
                         (unsigned long long)spdz_kernel_launches());
        });
        return backend::make_gpu_b200_backend(dev ? std::atoi(dev) : 0);
    }();
    return b;
}

}  // namespace mpc::runtime
