// Internal host-side state shared by capi.cu and run.cu.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/spdz_b200.h"
#include "kernels.cuh"

namespace spdzb200 {

// Error with a status code; converted to (code, thread-local message) at the C boundary.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const char* msg);

template <class F>
int guard(F&& f) {
    try {
        f();
        return SPDZ_OK;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.code;
    } catch (const std::bad_alloc& e) {
        set_last_error("out of host memory");
        return SPDZ_ERR_INVALID_ARGUMENT;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return SPDZ_ERR_INVALID_ARGUMENT;
    }
}

inline void need(bool cond, int code, const std::string& msg) {
    if (!cond) throw Error(code, msg);
}

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Error(SPDZ_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// Growable device scratch (never shrinks; reused across calls of one context).
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    int device = 0;
    void* ensure(size_t n) {
        if (n <= bytes) return p;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        cuda_check(cudaMalloc(&p, n), "cudaMalloc(scratch)");
        bytes = n;
        return p;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
};

struct HostPinned {
    void* p = nullptr;
    size_t bytes = 0;
    void* ensure(size_t n) {
        if (n <= bytes) return p;
        if (p) cudaFreeHost(p);
        p = nullptr;
        bytes = 0;
        cuda_check(cudaMallocHost(&p, n), "cudaMallocHost");
        bytes = n;
        return p;
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        bytes = 0;
    }
};

}  // namespace spdzb200

struct spdz_ctx {
    int device = 0;
    int party = 0;
    int n_parties = 2;
    uint32_t alpha = 0;
    uint32_t* d_alpha = nullptr;          // device copy of alpha (read by graph-captured kernels)
    int sms = 148;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    unsigned long long* d_acc = nullptr;  // 16 x u64 accumulators
    unsigned int* d_flag = nullptr;       // dealer rejection flag
    spdzb200::DevBuf scratch;             // host-wrapper staging / opened-E scratch
    spdzb200::DevBuf seg_buf;             // MAC segment + chunk tables
    spdzb200::DevBuf rank_buf;
    spdzb200::HostPinned pinned;
    // caller-driven MAC log (spdz_mac_log_*, runtime.cpp:112-117): device segments, appended
    // from any thread; per batch id the records logged so far (next lane0)
    std::mutex maclog_mu;
    std::vector<spdz_mac_segment_t> maclog;
    std::map<uint64_t, uint64_t> maclog_lanes;
};

namespace spdzb200 {
// throws Error; used by run.cu
void device_guard(const spdz_ctx* ctx);
// ctx->alpha and its device copy (stream-ordered on ctx->stream)
void set_alpha(spdz_ctx* ctx, uint32_t alpha);
uint32_t mac_sigma_impl(spdz_ctx* ctx, const spdz_mac_segment_t* segs, uint64_t n, uint64_t coin);
void mac_sigma_launch(spdz_ctx* ctx, const spdz_mac_segment_t* segs, uint64_t n, uint64_t coin, int acc_slot);
uint32_t mac_sigma_collect(spdz_ctx* ctx, int acc_slot);
void assign_ranks(spdz_mac_segment_t* segs, uint64_t n);
uint32_t host_reduce64(uint64_t v);
uint64_t dealer_draws_triples(int n, uint64_t lanes);
uint64_t dealer_draws_share(int n, uint64_t lanes);
uint64_t dealer_draws_matrix(int n, uint32_t din, uint32_t rows);
uint64_t dealer_draws_masks(int n, uint64_t count);
void dealer_alpha(int n, uint64_t seed, uint32_t* shares, uint32_t* alpha);
void check_dealer_flag(spdz_ctx* ctx);
}  // namespace spdzb200
