// tcgen05 (5th-gen tensor core) modular GEMM for the secret x public linear
// layer (runtime.cpp:303-334, batched): C = A * B mod p, p = 2^32 - 5.
//
// u32 operands are split into four u8 limbs, A = sum_i 2^(8i) A_i, B = sum_j 2^(8j) B_j,
// so A*B = sum_s 2^(8s) P_s with P_s = sum_{i+j=s} A_i B_j (s = 0..6).  Each P_s is an
// exact u8 x u8 -> s32 tensor-core GEMM accumulated in TMEM (tcgen05.mma kind::i8,
// M = 128, N = BN, K = 32 per instruction); 16 MMAs per K step.  The epilogue reads
// the seven s32 accumulators (tcgen05.ld) and recombines them mod p:
//   2^0, 2^8, 2^16, 2^24, 2^32 = 5, 2^40 = 1280, 2^48 = 327680 (mod p).
// Exactness: P_3 sums 4 limb products over K, 4 * 255^2 * K < 2^31 for K <= 8192.
//
// Operands are staged as u8 limb planes, K-major, padded to the tile (k_split_*),
// copied to shared memory with cp.async in the canonical no-swizzle K-major
// UMMA layout (8-row x 16-byte core matrices), double buffered against the MMAs;
// one elected thread issues the MMAs and tcgen05.commit releases a stage.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "field.cuh"
#include "internal.hpp"

namespace spdzb200 {

namespace {

constexpr int TM = 128;   // rows per CTA tile (UMMA M)
constexpr int TK = 64;    // K bytes (= elements) per stage
constexpr int kThreadsTc = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

// Bounded wait: a protocol bug traps (kernel error) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    uint32_t done = 0;
    for (uint32_t it = 0; it < (1u << 26); ++it) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(phase));
        if (done) return;
    }
    __trap();
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N));
}

// SMEM matrix descriptor, K-major, SWIZZLE_NONE (layout type 0), sm100 version 1.
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // version (Blackwell)
    return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE
}

// Instruction descriptor: kind::i8, D = s32, A = B = u8, both K-major, M = 128, N = BN.
template <int BN>
__device__ __forceinline__ uint32_t idesc_i8() {
    return (2u << 4)                      // c_format = S32
           | (0u << 7) | (0u << 10)       // a/b format = unsigned 8 bit
           | ((uint32_t)(BN >> 3) << 17)  // N >> 3
           | ((uint32_t)(TM >> 4) << 24); // M >> 4
}

__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}

// Shared-memory image of one limb tile (rows x TK bytes), canonical K-major
// no-swizzle layout: byte (r, k) at (r/8)*SBO + (k/16)*LBO + (r%8)*16 + k%16.
constexpr uint32_t kLBO = 128;                 // next 16-byte K chunk
constexpr uint32_t kSBO = (TK / 16) * 128;     // next 8-row group

template <int BN>
struct TcSmem {
    static constexpr uint32_t A_LIMB = TM * TK;              // 8 KB
    static constexpr uint32_t B_LIMB = BN * TK;
    static constexpr uint32_t STAGE = 4 * A_LIMB + 4 * B_LIMB;
    static constexpr uint32_t BYTES = 2 * STAGE + 1024;      // + barriers / tmem slot
    static constexpr uint32_t TMEM_COLS = (7 * BN <= 256) ? 256 : 512;
};

// Copies one K stage of the A and B limb planes into shared memory.
// A limb plane: [Mp][Kp] bytes; B limb plane: [Np][Kp] bytes (both K-major).
template <int BN>
__device__ __forceinline__ void load_stage(uint32_t sbase, const uint8_t* __restrict__ A, const uint8_t* __restrict__ B,
                                           uint64_t Mp, uint64_t Np, uint32_t Kp, uint32_t m0, uint32_t n0,
                                           uint32_t k0) {
    using L = TcSmem<BN>;
    // A: 4 limbs x 128 rows x 4 chunks of 16 B
    for (uint32_t c = threadIdx.x; c < 4u * TM * (TK / 16); c += blockDim.x) {
        const uint32_t limb = c / (TM * (TK / 16));
        const uint32_t rem = c % (TM * (TK / 16));
        const uint32_t r = rem / (TK / 16), kc = rem % (TK / 16);
        const uint8_t* src = A + (uint64_t)limb * Mp * Kp + (uint64_t)(m0 + r) * Kp + k0 + kc * 16;
        const uint32_t dst = sbase + limb * L::A_LIMB + (r >> 3) * kSBO + kc * kLBO + (r & 7) * 16;
        cp_async16(dst, src);
    }
    const uint32_t bbase = sbase + 4 * L::A_LIMB;
    for (uint32_t c = threadIdx.x; c < 4u * BN * (TK / 16); c += blockDim.x) {
        const uint32_t limb = c / (BN * (TK / 16));
        const uint32_t rem = c % (BN * (TK / 16));
        const uint32_t r = rem / (TK / 16), kc = rem % (TK / 16);
        const uint8_t* src = B + (uint64_t)limb * Np * Kp + (uint64_t)(n0 + r) * Kp + k0 + kc * 16;
        const uint32_t dst = bbase + limb * L::B_LIMB + (r >> 3) * kSBO + kc * kLBO + (r & 7) * 16;
        cp_async16(dst, src);
    }
}

// out plane mapping of C[row][col] (see launch_modgemm_tc)
struct TcOut {
    int mode;          // 0: cols [0,batch) -> y0, [batch, 2 batch) -> y1;  1: rows [0,dout) -> y0, rest -> y1
    uint32_t dout, batch;
    uint32_t* y0;
    uint32_t* y1;
};

template <int BN>
__global__ void __launch_bounds__(kThreadsTc, 1) k_modgemm_tc(const uint8_t* __restrict__ A, const uint8_t* __restrict__ B,
                                                               uint32_t M, uint32_t N, uint64_t Mp, uint64_t Np, uint32_t Kp,
                                                               TcOut out) {
    using L = TcSmem<BN>;
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t sbase = (smem_u32(smem) + 1023u) & ~1023u;
    uint8_t* sgen = smem + (sbase - smem_u32(smem));
    uint64_t* bars = reinterpret_cast<uint64_t*>(sgen + 2 * L::STAGE);  // [0..1] stage free, [2] final
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sgen + 2 * L::STAGE + 64);
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t m0 = blockIdx.y * TM, n0 = blockIdx.x * BN;

    if (threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        mbar_init(&bars[2], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(L::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;

    const uint32_t nkb = Kp / TK;
    const uint32_t idesc = idesc_i8<BN>();
    uint32_t uses[2] = {0, 0};
    load_stage<BN>(sbase, A, B, Mp, Np, Kp, m0, n0, 0);
    cp_async_commit();
    uint32_t inited = 0;  // issuing thread: accumulators already written
    for (uint32_t kb = 0; kb < nkb; ++kb) {
        const uint32_t st = kb & 1;
        if (kb + 1 < nkb) {
            const uint32_t ns = st ^ 1;
            if (uses[ns]) mbar_wait(&bars[ns], (uses[ns] - 1) & 1);  // MMAs of kb-1 released it
            load_stage<BN>(sbase + ns * L::STAGE, A, B, Mp, Np, Kp, m0, n0, (kb + 1) * TK);
            cp_async_commit();
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // cp.async writes -> tensor core
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t sa = sbase + st * L::STAGE, sb = sa + 4 * L::A_LIMB;
#pragma unroll
            for (int ks = 0; ks < TK / 32; ++ks) {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const uint64_t ad = smem_desc(sa + i * L::A_LIMB + ks * 2 * kLBO, kLBO, kSBO);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int s = i + j;
                        const uint64_t bd = smem_desc(sb + j * L::B_LIMB + ks * 2 * kLBO, kLBO, kSBO);
                        mma_i8(tmem + s * BN, ad, bd, idesc, (inited >> s) & 1u);
                        inited |= 1u << s;
                    }
                }
            }
            mma_commit(&bars[st]);  // stage st may be overwritten once these MMAs complete
        }
        uses[st] += 1;
        __syncwarp();
    }
    if (threadIdx.x == 0) mma_commit(&bars[2]);
    mbar_wait(&bars[2], 0);
    asm volatile("tcgen05.fence::after_thread_sync;");

    // epilogue: TMEM lane = row (warp w owns lanes 32w..32w+31), column = n
    const uint32_t row = m0 + warp * 32 + lane;
    const uint32_t lane_base = tmem + ((warp * 32u) << 16);
    constexpr uint32_t kPow[7] = {1u, 256u, 65536u, 16777216u, 5u, 1280u, 327680u};
#pragma unroll 1
    for (int cc = 0; cc < BN / 16; ++cc) {
        uint32_t v[7][16];
#pragma unroll
        for (int s = 0; s < 7; ++s) tmem_ld16(lane_base + s * BN + cc * 16, v[s]);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (row < M) {
#pragma unroll
            for (int t = 0; t < 16; ++t) {
                const uint32_t col = n0 + cc * 16 + t;
                if (col >= N) continue;
                unsigned long long acc = 0;
#pragma unroll
                for (int s = 0; s < 7; ++s) acc += (unsigned long long)v[s][t] * kPow[s];
                const uint32_t r = fp_reduce64(acc);
                if (out.mode == 0) {
                    if (col < out.batch) out.y0[(uint64_t)row * out.batch + col] = r;
                    else out.y1[(uint64_t)row * out.batch + (col - out.batch)] = r;
                } else {
                    if (row < out.dout) out.y0[(uint64_t)row * out.batch + col] = r;
                    else out.y1[(uint64_t)(row - out.dout) * out.batch + col] = r;
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(L::TMEM_COLS));
}

// A limb planes (K-major): out[i][m][k] = byte i of A(m, k), zero padded to Mp x Kp.
// A(m, k) = a0[m*K + k] for m < M0, a1[(m-M0)*K + k] for M0 <= m < M (row stacking).
__global__ void k_split_rows(const uint32_t* __restrict__ a0, const uint32_t* __restrict__ a1, uint32_t M0, uint32_t M,
                             uint32_t K, uint64_t Mp, uint32_t Kp, uint8_t* __restrict__ out) {
    const uint64_t total = Mp * Kp / 4;  // 4 k per thread
    const uint64_t plane = Mp * Kp;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t m = (t * 4) / Kp;
        const uint32_t k = (uint32_t)((t * 4) % Kp);
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t kk = k + q;
            w[q] = (m < M && kk < K) ? (m < M0 ? a0[m * K + kk] : a1[(m - M0) * K + kk]) : 0u;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint32_t packed = ((w[0] >> (8 * i)) & 0xFF) | (((w[1] >> (8 * i)) & 0xFF) << 8) |
                                    (((w[2] >> (8 * i)) & 0xFF) << 16) | (((w[3] >> (8 * i)) & 0xFF) << 24);
            reinterpret_cast<uint32_t*>(out + i * plane + m * Kp + k)[0] = packed;
        }
    }
}

// B limb planes transposed to K-major: out[j][n][k] = byte j of B(k, n), zero padded.
// B(k, n) = b0[k*NB + n] for n < NB, b1[k*NB + n - NB] for NB <= n < N (column stacking).
__global__ void k_split_cols_t(const uint32_t* __restrict__ b0, const uint32_t* __restrict__ b1, uint32_t NB, uint32_t N,
                               uint32_t K, uint64_t Np, uint32_t Kp, uint8_t* __restrict__ out) {
    __shared__ uint32_t tile[32][33];
    const uint64_t plane = Np * Kp;
    const uint32_t kt = blockIdx.x * 32, nt = blockIdx.y * 32;
    for (int yy = threadIdx.y; yy < 32; yy += blockDim.y) {  // read rows k, coalesced over n
        const uint32_t k = kt + yy, n = nt + threadIdx.x;
        uint32_t v = 0;
        if (k < K && n < N) v = n < NB ? b0[(uint64_t)k * NB + n] : b1[(uint64_t)k * NB + (n - NB)];
        tile[yy][threadIdx.x] = v;
    }
    __syncthreads();
    for (int yy = threadIdx.y; yy < 32; yy += blockDim.y) {  // write rows n, coalesced over k
        const uint32_t n = nt + yy, k = kt + threadIdx.x;
        if (n < Np && k < Kp) {
            const uint32_t v = tile[threadIdx.x][yy];
#pragma unroll
            for (int j = 0; j < 4; ++j) out[j * plane + (uint64_t)n * Kp + k] = (uint8_t)(v >> (8 * j));
        }
    }
}

template <int BN>
cudaError_t run_tc(cudaStream_t s, const uint8_t* Al, const uint8_t* Bl, uint32_t M, uint32_t N, uint64_t Mp,
                   uint64_t Np, uint32_t Kp, const TcOut& out) {
    using L = TcSmem<BN>;
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(k_modgemm_tc<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::BYTES);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    dim3 grid((unsigned)(Np / BN), (unsigned)(Mp / TM));
    k_modgemm_tc<BN><<<grid, kThreadsTc, L::BYTES, s>>>(Al, Bl, M, N, Mp, Np, Kp, out);
    ++g_kernel_launches;
    return cudaGetLastError();
}

}  // namespace

uint64_t modgemm_tc_scratch_bytes(int mode, uint32_t dout, uint32_t din, uint32_t batch) {
    const uint64_t M = mode == 0 ? dout : 2ull * dout, N = mode == 0 ? 2ull * batch : batch;
    const uint64_t Mp = (M + TM - 1) / TM * TM, Np = (N + 63) / 64 * 64, Kp = (din + TK - 1) / TK * TK;
    return 4 * (Mp + Np) * Kp + 256;
}

bool modgemm_tc_supported(uint32_t din) { return din >= 1 && din <= 8192; }

// Y (dout x batch, two planes) for the secret x public linear layer on tcgen05.
//   mode 0: W public (w0), X secret planes (x0 vals, x1 macs): C = W * [Xv | Xm]
//   mode 1: W secret planes (w0, w1), X public (x0):           C = [Wv ; Wm] * X
cudaError_t launch_modgemm_tc(cudaStream_t s, int mode, uint32_t dout, uint32_t din, uint32_t batch,
                              const uint32_t* w0, const uint32_t* w1, const uint32_t* x0, const uint32_t* x1,
                              uint32_t* y0, uint32_t* y1, uint8_t* scratch, int sms) {
    if (dout == 0 || batch == 0) return cudaSuccess;
    const uint32_t M = mode == 0 ? dout : 2 * dout, N = mode == 0 ? 2 * batch : batch;
    const uint64_t Mp = (M + TM - 1) / TM * TM, Np = (N + 63) / 64 * 64;
    const uint32_t Kp = (din + TK - 1) / TK * TK;
    uint8_t* Al = scratch;
    uint8_t* Bl = scratch + 4 * Mp * Kp;
    // limb planes
    {
        const uint64_t work = Mp * Kp / 4;
        const int grid = (int)std::min<uint64_t>((work + 255) / 256, (uint64_t)sms * 16);
        if (mode == 0) k_split_rows<<<grid, 256, 0, s>>>(w0, w0, M, M, din, Mp, Kp, Al);
        else k_split_rows<<<grid, 256, 0, s>>>(w0, w1, dout, M, din, Mp, Kp, Al);
        ++g_kernel_launches;
        dim3 g2(Kp / 32, (unsigned)((Np + 31) / 32)), b2(32, 8);
        if (mode == 0) k_split_cols_t<<<g2, b2, 0, s>>>(x0, x1, batch, N, din, Np, Kp, Bl);
        else k_split_cols_t<<<g2, b2, 0, s>>>(x0, x0, batch, N, din, Np, Kp, Bl);
        ++g_kernel_launches;
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    TcOut out{mode, dout, batch, y0, y1};
    // narrow N tiles when the 64-wide grid would leave SMs idle
    if ((Mp / TM) * (Np / 64) < (uint64_t)sms) return run_tc<32>(s, Al, Bl, M, N, Mp, Np, Kp, out);
    return run_tc<64>(s, Al, Bl, M, N, Mp, Np, Kp, out);
}

}  // namespace spdzb200
