// Diagnostics: measured integer-pipe peak of the CUDA cores on this device
// (the denominator for the CUDA-core modular GEMM's roofline; MEASURED_PEAKS
// only holds HBM and bf16 numbers).  Each thread runs 8 independent
// IMAD.WIDE.U32 chains (u64 += u32*u32), so the fma pipe, not latency, bounds it.
#include <cuda_runtime.h>

#include <cstdint>

#include "field.cuh"
#include "internal.hpp"

namespace {

__global__ void __launch_bounds__(256) k_imad_wide_peak(uint32_t iters, uint32_t seed, unsigned long long* sink) {
    uint32_t a[8];
    unsigned long long acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        a[k] = seed * (threadIdx.x + 1) + k * 0x9e3779b9u;
        acc[k] = k;
    }
    const uint32_t b = seed ^ blockIdx.x;
    for (uint32_t i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[k] += (unsigned long long)a[k] * b;  // IMAD.WIDE.U32
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] += (uint32_t)acc[k];                // keep the chains live
    }
    unsigned long long s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s ^= acc[k];
    if (s == 0x123456789ull) sink[0] = s;
}

// out[2i] = rep_mod_p(v_i), out[2i+1] = mac_coeff_rep(v_i) for u64 v_i (edge-case checks of
// the MAC-check record arithmetic against v mod p / reduce(mix64(v)) on the host).
__global__ void k_rep_check(const unsigned long long* in, uint64_t n, uint32_t* out, spdzb200::SigConsts kc) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t l = (uint32_t)in[i], h = (uint32_t)(in[i] >> 32);
        out[2 * i] = spdzb200::rep_mod_p(l, h, kc.five);
        out[2 * i + 1] = spdzb200::mac_coeff_rep(l, h, kc);
    }
}

}  // namespace

using namespace spdzb200;

extern "C" int spdz_diag_rep_check(spdz_ctx* ctx, const uint64_t* d_in, uint64_t n, uint32_t* d_out) {
    return guard([&] {
        need(ctx && (n == 0 || (d_in && d_out)), SPDZ_ERR_INVALID_ARGUMENT, "bad diag args");
        device_guard(ctx);
        if (n == 0) return;
        k_rep_check<<<(int)((n + 255) / 256 < 1024 ? (n + 255) / 256 : 1024), 256, 0, ctx->stream>>>(
            reinterpret_cast<const unsigned long long*>(d_in), n, d_out, spdzb200::SigConsts{});
        cuda_check(cudaGetLastError(), "k_rep_check");
        cuda_check(cudaStreamSynchronize(ctx->stream), "sync");
    });
}

extern "C" int spdz_diag_imad_wide_rate(spdz_ctx* ctx, double* wide_per_s, double* total_int_per_s) {
    return guard([&] {
        need(ctx && wide_per_s, SPDZ_ERR_INVALID_ARGUMENT, "bad diag args");
        device_guard(ctx);
        unsigned long long* sink = ctx->d_acc + 8;
        const uint32_t iters = 4096;
        const int grid = ctx->sms * 8;
        cudaEvent_t e0, e1;
        cuda_check(cudaEventCreate(&e0), "ev");
        cuda_check(cudaEventCreate(&e1), "ev");
        k_imad_wide_peak<<<grid, 256, 0, ctx->stream>>>(64, 7u, sink);  // warm
        cuda_check(cudaEventRecord(e0, ctx->stream), "rec");
        k_imad_wide_peak<<<grid, 256, 0, ctx->stream>>>(iters, 7u, sink);
        cuda_check(cudaEventRecord(e1, ctx->stream), "rec");
        cuda_check(cudaEventSynchronize(e1), "sync");
        float ms = 0;
        cuda_check(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        const double threads = double(grid) * 256;
        *wide_per_s = threads * iters * 8 / (ms / 1e3);
        if (total_int_per_s) *total_int_per_s = threads * iters * 16 / (ms / 1e3);  // + the IADD chain
    });
}

namespace spdzb200 {
void modgemm_tc_debug(uint32_t flags);
void modgemm_tc_timeline(uint64_t* dev_buf);
}

// Diagnostic switches of the tcgen05 GEMM (gemm_tc.cu g_tc_dbg): bit 2 skips the GEMM kernel,
// bit 3 the re-layout kernels (results invalid while set); bits 6/7 force the 32/64-column tile.
extern "C" int spdz_diag_gemm_tc_timeline(void* dev_buf) {
    spdzb200::modgemm_tc_timeline(static_cast<uint64_t*>(dev_buf));
    return 0;
}

extern "C" int spdz_diag_gemm_tc_flags(uint32_t flags) {
    spdzb200::modgemm_tc_debug(flags);
    return 0;
}
