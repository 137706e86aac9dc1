// tcgen05 (5th-gen tensor core) modular GEMM for the secret x public linear
// layer (runtime.cpp:303-334, batched): C = A * B mod p, p = 2^32 - 5.
//
// u32 operands are split into four u8 limbs, A = sum_i 2^(8i) A_i, B = sum_j 2^(8j) B_j,
// so A*B = sum_s 2^(8s) P_s with P_s = sum_{i+j=s} A_i B_j (s = 0..6).  Each limb
// product is an exact u8 x u8 -> s32 tensor-core product (tcgen05.mma kind::i8, K = 32
// per instruction); the epilogue recombines mod p with
//   2^0, 2^8, 2^16, 2^24, 2^32 = 5, 2^40 = 1280, 2^48 = 327680 (mod p).
// Exactness: P_3 sums 4 limb products over K, 4 * 255^2 * K < 2^31 for K <= 8192.
//
// Main kernel (k_modgemm_tc): a 128 x 64 output tile keeps the seven P_s
// accumulators side by side in TMEM (P_s at columns [64 s, 64 s + 64), 448 of the 512
// columns).  The four B limb tiles are stacked as one N = 256 operand [B_0|B_1|B_2|B_3],
// so one MMA with A_i and destination column 64 i adds A_i B_j into P_{i+j} for all j:
// four N = 256 MMAs per 32-deep K step cover all 16 limb products (the first K step
// initialises the overlapping ranges with an N = 192 / 256 / 64 sequence).  N = 256 per
// instruction keeps the shared-memory operand traffic at 96 B/clk; the 128 x 64 tile
// needs 48 B/clk of L2->SMEM fill at the MMA rate.
//
// Operands are re-laid out once per call (k_tile_both: tile_rows / tile_cols) as u8 limb
// tiles already in the canonical no-swizzle K-major UMMA image (8-row x 16-byte
// core matrices), so each K stage is two 1-D TMA bulk copies (cp.async.bulk +
// mbarrier complete_tx) into a 4-stage ring.  The kernel is persistent (one CTA per
// SM, tiles N-fastest so the B image stays L2-resident): warp 0 produces, one thread
// of warp 1 issues the MMAs, warps 2-5 drain TMEM (tcgen05.ld) and store; the
// producer keeps prefetching the next tile while the epilogue runs.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "async.cuh"
#include "field.cuh"
#include "internal.hpp"

namespace spdzb200 {

namespace {

constexpr int TM = 128;   // rows per CTA tile (UMMA M)
constexpr int TK = 64;    // K bytes (= elements) per stage
constexpr uint32_t kMaxKSlice = 8192;  // 4 * 255^2 * K < 2^31: the s32 P_3 accumulator bound

// SMEM matrix descriptor, K-major, SWIZZLE_NONE (layout type 0), sm100 version 1.
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // version (Blackwell)
    return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE
}

// Instruction descriptor: kind::i8, D = s32, A = B = u8, both K-major, M = BM (128, or 256 for a
// CTA pair), N = BN.
template <int BN, int BM = TM>
__host__ __device__ constexpr uint32_t idesc_i8() {
    return (2u << 4)                      // c_format = S32
           | (0u << 7) | (0u << 10)       // a/b format = unsigned 8 bit
           | ((uint32_t)(BN >> 3) << 17)  // N >> 3
           | ((uint32_t)(BM >> 4) << 24); // M >> 4
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

// diagnostic timeline (spdz_diag_gemm_tc_timeline): per CTA 16 %globaltimer stamps
__device__ __forceinline__ void tl_mark(uint64_t* tl, uint32_t slot) {
    if (tl) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        tl[blockIdx.x * 16 + slot] = t;
    }
}


// Shared-memory image of one limb tile (rows x TK bytes), canonical K-major
// no-swizzle layout: byte (r, k) at (r/8)*SBO + (k/16)*LBO + (r%8)*16 + k%16.
// The split kernels write the operands into global memory already in this image,
// tile by tile, so one K stage is two contiguous 1-D TMA bulk copies.
constexpr uint32_t kLBO = 128;                 // next 16-byte K chunk
constexpr uint32_t kSBO = (TK / 16) * 128;     // next 8-row group

__device__ __forceinline__ uint32_t core_off(uint32_t r, uint32_t k) {
    return (r >> 3) * kSBO + (k >> 4) * kLBO + (r & 7) * 16 + (k & 15);
}

// B-operand transform of the re-layout (tile_cols)
struct TcBx {
    const uint32_t* e;
    uint32_t coef0, coef1;
};

// out plane mapping of C[row][col] (see launch_modgemm_tc)
struct TcOut {
    int mode;          // 0: cols [0,batch) -> y0, [batch, 2 batch) -> y1;  1: rows [0,dout) -> y0, rest -> y1
    uint32_t dout, batch;
    uint32_t* y0;
    uint32_t* y1;
    const uint32_t* add0;  // optional addend planes (same layout as y0/y1, may alias them): y = add + C
    const uint32_t* add1;
};

// ---------------------------------------------------------------------------
// 128 x TN tiles, P_s accumulators, N = 4 TN MMAs, persistent, warp-specialised.
// ---------------------------------------------------------------------------
// TN = 64 for large problems (N = 256 MMAs); TN = 32 (N = 128 MMAs, twice the tiles)
// when the TN = 64 tiling would leave SMs idle.
constexpr int kStages = 4;
constexpr int kThreadsTc = 320;  // warp 0 TMA, warp 1 MMA, warps 2-9 epilogue (two per TMEM lane quarter)
template <int TN>
struct TcSmem {
    static constexpr uint32_t A_LIMB = TM * TK;        // 8 KB
    static constexpr uint32_t B_LIMB = TN * TK;        // 4 KB at TN = 64
    static constexpr uint32_t A_STAGE = 4 * A_LIMB;    // 32 KB
    static constexpr uint32_t B_STAGE = 4 * B_LIMB;    // 16 KB at TN = 64
    static constexpr uint32_t STAGE = A_STAGE + B_STAGE;
    static constexpr uint32_t BYTES = kStages * STAGE + 1024 + 256;
    static constexpr uint32_t TMEM_COLS = 7 * TN <= 256 ? 256 : 512;
};

// sum_s 2^(8s) P_s mod p for 16 columns (2^32 = 5, 2^40 = 1280, 2^48 = 327680 mod p)
__device__ __forceinline__ void tc_recombine16(const uint32_t (&v)[7][16], uint32_t (&r)[16]) {
    constexpr uint32_t kPow[7] = {1u, 256u, 65536u, 16777216u, 5u, 1280u, 327680u};
#pragma unroll
    for (int t = 0; t < 16; ++t) {
        unsigned long long acc = 0;
#pragma unroll
        for (int q = 0; q < 7; ++q) acc += (unsigned long long)v[q][t] * kPow[q];
        r[t] = fp_reduce64(acc);
    }
}

// 16 results of output row `row`, columns col0 .. col0+15 of C, into their plane (+ addend)
__device__ __forceinline__ void tc_store16(const TcOut& out, uint32_t N, uint32_t row, uint32_t col0,
                                           uint32_t (&r)[16]) {
    uint32_t* dst;
    uint32_t lim;  // valid columns in this group
    if (out.mode == 0) {
        const bool hi = col0 >= out.batch;
        dst = hi ? out.y1 + (uint64_t)row * out.batch + (col0 - out.batch) : out.y0 + (uint64_t)row * out.batch + col0;
        lim = hi ? (col0 < N ? N - col0 : 0) : out.batch - col0;
    } else {
        const bool hi = row >= out.dout;
        dst = hi ? out.y1 + (uint64_t)(row - out.dout) * out.batch + col0 : out.y0 + (uint64_t)row * out.batch + col0;
        lim = col0 < N ? N - col0 : 0;
    }
    if (lim >= 16 && (reinterpret_cast<uintptr_t>(dst) & 15u) == 0) {
        if (out.add0) {  // same offset in the addend plane as in the output plane
            const bool hi = out.mode == 0 ? col0 >= out.batch : row >= out.dout;
            const uint32_t* src = (hi ? out.add1 : out.add0) + (dst - (hi ? out.y1 : out.y0));
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const uint4 a = reinterpret_cast<const uint4*>(src)[c];
                r[4 * c] = fp_add(r[4 * c], a.x);
                r[4 * c + 1] = fp_add(r[4 * c + 1], a.y);
                r[4 * c + 2] = fp_add(r[4 * c + 2], a.z);
                r[4 * c + 3] = fp_add(r[4 * c + 3], a.w);
            }
        }
#pragma unroll
        for (int c = 0; c < 4; ++c)
            reinterpret_cast<uint4*>(dst)[c] = make_uint4(r[4 * c], r[4 * c + 1], r[4 * c + 2], r[4 * c + 3]);
    } else {
        // group straddles the plane boundary (mode 0, batch % 16 != 0) or the edge
#pragma unroll
        for (int t = 0; t < 16; ++t) {
            const uint32_t col = col0 + t;
            if (col >= N) break;
            uint64_t off;
            bool hi;
            if (out.mode == 0) {
                hi = col >= out.batch;
                off = (uint64_t)row * out.batch + (hi ? col - out.batch : col);
            } else {
                hi = row >= out.dout;
                off = (uint64_t)(hi ? row - out.dout : row) * out.batch + col;
            }
            uint32_t v = r[t];
            if (out.add0) v = fp_add(v, (hi ? out.add1 : out.add0)[off]);
            (hi ? out.y1 : out.y0)[off] = v;
        }
    }
}

// The seven P_s accumulators of 16 columns (TMEM columns taddr + s TN), issued as one block of
// loads with a single wait: as separate statements ptxas may serialise them (one TMEM round trip
// each) when registers are tight, which measured ~1 us per 16-column chunk in the split-K epilogue.
template <int TN>
__device__ __forceinline__ void tmem_ld16_x7(uint32_t taddr, uint32_t (&v)[7][16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%112];\n"
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%113];\n"
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47}, [%114];\n"
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%115];\n"
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%64,%65,%66,%67,%68,%69,%70,%71,%72,%73,%74,%75,%76,%77,%78,%79}, [%116];\n"
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%80,%81,%82,%83,%84,%85,%86,%87,%88,%89,%90,%91,%92,%93,%94,%95}, [%117];\n"
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%96,%97,%98,%99,%100,%101,%102,%103,%104,%105,%106,%107,%108,%109,%110,%111}, [%118];\n"
        "tcgen05.wait::ld.sync.aligned;\n"
        : "=r"(v[0][0]), "=r"(v[0][1]), "=r"(v[0][2]), "=r"(v[0][3]), "=r"(v[0][4]), "=r"(v[0][5]), "=r"(v[0][6]), "=r"(v[0][7]),
          "=r"(v[0][8]), "=r"(v[0][9]), "=r"(v[0][10]), "=r"(v[0][11]), "=r"(v[0][12]), "=r"(v[0][13]), "=r"(v[0][14]), "=r"(v[0][15]),
          "=r"(v[1][0]), "=r"(v[1][1]), "=r"(v[1][2]), "=r"(v[1][3]), "=r"(v[1][4]), "=r"(v[1][5]), "=r"(v[1][6]), "=r"(v[1][7]),
          "=r"(v[1][8]), "=r"(v[1][9]), "=r"(v[1][10]), "=r"(v[1][11]), "=r"(v[1][12]), "=r"(v[1][13]), "=r"(v[1][14]), "=r"(v[1][15]),
          "=r"(v[2][0]), "=r"(v[2][1]), "=r"(v[2][2]), "=r"(v[2][3]), "=r"(v[2][4]), "=r"(v[2][5]), "=r"(v[2][6]), "=r"(v[2][7]),
          "=r"(v[2][8]), "=r"(v[2][9]), "=r"(v[2][10]), "=r"(v[2][11]), "=r"(v[2][12]), "=r"(v[2][13]), "=r"(v[2][14]), "=r"(v[2][15]),
          "=r"(v[3][0]), "=r"(v[3][1]), "=r"(v[3][2]), "=r"(v[3][3]), "=r"(v[3][4]), "=r"(v[3][5]), "=r"(v[3][6]), "=r"(v[3][7]),
          "=r"(v[3][8]), "=r"(v[3][9]), "=r"(v[3][10]), "=r"(v[3][11]), "=r"(v[3][12]), "=r"(v[3][13]), "=r"(v[3][14]), "=r"(v[3][15]),
          "=r"(v[4][0]), "=r"(v[4][1]), "=r"(v[4][2]), "=r"(v[4][3]), "=r"(v[4][4]), "=r"(v[4][5]), "=r"(v[4][6]), "=r"(v[4][7]),
          "=r"(v[4][8]), "=r"(v[4][9]), "=r"(v[4][10]), "=r"(v[4][11]), "=r"(v[4][12]), "=r"(v[4][13]), "=r"(v[4][14]), "=r"(v[4][15]),
          "=r"(v[5][0]), "=r"(v[5][1]), "=r"(v[5][2]), "=r"(v[5][3]), "=r"(v[5][4]), "=r"(v[5][5]), "=r"(v[5][6]), "=r"(v[5][7]),
          "=r"(v[5][8]), "=r"(v[5][9]), "=r"(v[5][10]), "=r"(v[5][11]), "=r"(v[5][12]), "=r"(v[5][13]), "=r"(v[5][14]), "=r"(v[5][15]),
          "=r"(v[6][0]), "=r"(v[6][1]), "=r"(v[6][2]), "=r"(v[6][3]), "=r"(v[6][4]), "=r"(v[6][5]), "=r"(v[6][6]), "=r"(v[6][7]),
          "=r"(v[6][8]), "=r"(v[6][9]), "=r"(v[6][10]), "=r"(v[6][11]), "=r"(v[6][12]), "=r"(v[6][13]), "=r"(v[6][14]), "=r"(v[6][15])
        : "r"(taddr + 0 * TN), "r"(taddr + 1 * TN), "r"(taddr + 2 * TN), "r"(taddr + 3 * TN),
          "r"(taddr + 4 * TN), "r"(taddr + 5 * TN), "r"(taddr + 6 * TN)
        : "memory");
}

template <int TN>
__global__ void __launch_bounds__(kThreadsTc, 1) k_modgemm_tc(const uint8_t* __restrict__ At,
                                                               const uint8_t* __restrict__ Bt, uint32_t M, uint32_t N,
                                                               uint32_t KB, uint32_t tiles_n, uint32_t n_tiles,
                                                               TcOut out, uint32_t dbg, uint64_t* tl) {
    using L = TcSmem<TN>;
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t sbase = (smem_u32(smem) + 1023u) & ~1023u;
    uint8_t* sgen = smem + (sbase - smem_u32(smem));
    uint64_t* full = reinterpret_cast<uint64_t*>(sgen + kStages * L::STAGE);
    uint64_t* empty = full + kStages;
    uint64_t* tfull = empty + kStages;  // MMAs of a tile done (tcgen05.commit)
    uint64_t* tempty = tfull + 1;        // epilogue drained TMEM (4 warp arrivals)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) tl_mark(tl, 0);

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tfull, 1);
        mbar_init(tempty, 8);
        mbar_fence_init();
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
    if (threadIdx.x == 0) tl_mark(tl, 1);
    // programmatic dependent launch: everything above overlapped the re-layout kernel;
    // its limb images (and any earlier writes) are visible after this
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0) tl_mark(tl, 2);

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer ----
            uint32_t g = 0;
            for (uint32_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
                const uint32_t mt = tile / tiles_n, nt = tile % tiles_n;
                const uint8_t* a_src = At + (uint64_t)mt * KB * L::A_STAGE;
                const uint8_t* b_src = Bt + (uint64_t)nt * KB * L::B_STAGE;
                for (uint32_t kb = 0; kb < KB; ++kb, ++g) {
                    const uint32_t s = g % kStages;
                    if (g >= (uint32_t)kStages) mbar_wait(&empty[s], ((g / kStages) - 1) & 1);
                    const uint32_t dst = sbase + s * L::STAGE;
                    if (dbg & 1) {  // diagnostic: no loads (attribution only, results invalid)
                        mbar_arrive(&full[s]);
                        continue;
                    }
                    mbar_expect_tx(&full[s], L::STAGE);
                    bulk_g2s(dst, a_src + (uint64_t)kb * L::A_STAGE, L::A_STAGE, &full[s]);
                    bulk_g2s(dst + L::A_STAGE, b_src + (uint64_t)kb * L::B_STAGE, L::B_STAGE, &full[s]);
                }
            }
        }
        __syncwarp();  // reconverge before the final (aligned) block barrier
    } else if (warp == 1) {
        if (lane == 0) {  // ---- MMA issuer ----
            constexpr uint32_t id4 = idesc_i8<4 * TN>(), id3 = idesc_i8<3 * TN>(), id1 = idesc_i8<TN>();
            uint32_t g = 0, it = 0;
            for (uint32_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
                if (it > 0) mbar_wait(tempty, (it - 1) & 1);  // epilogue of the previous tile drained TMEM
                asm volatile("tcgen05.fence::after_thread_sync;");
                for (uint32_t kb = 0; kb < KB; ++kb, ++g) {
                    const uint32_t s = g % kStages;
                    mbar_wait(&full[s], (g / kStages) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    if (g == 0) tl_mark(tl, 3);
                    const uint32_t sa = sbase + s * L::STAGE, sb = sa + L::A_STAGE;
                    if (dbg & 2) {  // diagnostic: no MMAs (attribution only, results invalid)
                        mbar_arrive(&empty[s]);
                        continue;
                    }
#pragma unroll
                    for (int ks = 0; ks < TK / 32; ++ks) {
                        const uint64_t bd = smem_desc(sb + ks * 2 * kLBO, kLBO, kSBO);
                        uint64_t ad[4];
#pragma unroll
                        for (int i = 0; i < 4; ++i) ad[i] = smem_desc(sa + i * L::A_LIMB + ks * 2 * kLBO, kLBO, kSBO);
                        if (kb == 0 && ks == 0) {  // initialise P_0..P_6 (overlapping destination ranges)
                            const uint64_t bd3 = smem_desc(sb + 3 * L::B_LIMB + ks * 2 * kLBO, kLBO, kSBO);
                            mma_i8(tmem, ad[0], bd, id3, 0u);             // P0..P2  = A0 [B0|B1|B2]
                            mma_i8(tmem + 3 * TN, ad[3], bd, id4, 0u);    // P3..P6  = A3 [B0..B3]
                            mma_i8(tmem + 3 * TN, ad[0], bd3, id1, 1u);   // P3     += A0 B3
                            mma_i8(tmem + 1 * TN, ad[1], bd, id4, 1u);    // P1..P4 += A1 [B0..B3]
                            mma_i8(tmem + 2 * TN, ad[2], bd, id4, 1u);    // P2..P5 += A2 [B0..B3]
                        } else {
#pragma unroll
                            for (int i = 0; i < 4; ++i) mma_i8(tmem + i * TN, ad[i], bd, id4, 1u);
                        }
                    }
                    mma_commit(&empty[s]);  // frees the stage once these MMAs have read it
                }
                if (dbg & 2) mbar_arrive(tfull);
                else mma_commit(tfull);  // accumulators of this tile complete
            }
            tl_mark(tl, 4);
        }
        __syncwarp();
    } else {  // ---- epilogue: warps 2..9, TMEM lane quarter = warp % 4, 16-column chunks split by (warp-2)/4 ----
        const uint32_t quarter = warp & 3, half = (warp - 2) >> 2;
        const uint32_t lane_base = tmem + ((quarter * 32u) << 16);
        uint32_t it = 0;
        for (uint32_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
            const uint32_t mt = tile / tiles_n, nt = tile % tiles_n;
            const uint32_t row = mt * TM + quarter * 32 + lane;
            mbar_wait(tfull, it & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            if (warp == 2 && lane == 0) tl_mark(tl, 5);
#pragma unroll 1
            for (int cc = half; cc < TN / 16; cc += 2) {
                uint32_t v[7][16];
                tmem_ld16_x7<TN>(lane_base + cc * 16, v);
                if (cc + 2 >= TN / 16) {  // every column of this warp's share is in registers: release TMEM
                    asm volatile("tcgen05.fence::before_thread_sync;");
                    __syncwarp();
                    if (lane == 0) mbar_arrive(tempty);
                }
                const uint32_t col0 = nt * TN + cc * 16;
                if (row >= M) continue;
                uint32_t r[16];
                tc_recombine16(v, r);
                tc_store16(out, N, row, col0, r);
            }
            if (warp == 2 && lane == 0) tl_mark(tl, 6);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x == 0) tl_mark(tl, 7);
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(L::TMEM_COLS));
}

// ---------------------------------------------------------------------------
// CTA-pair variant (tcgen05.mma.cta_group::2, M = 256) for problems whose 128 x 64 tiling
// leaves SMs idle (C3: 1024 x 512 outputs = 64 such tiles).  A pair of CTAs on one TPC owns a
// 256 x TN output tile (TN = 32): each CTA stages its own 128 rows of the four A limbs and two
// of the four stacked B limbs ([B0|B1] in rank 0, [B2|B3] in rank 1), and the leader issues
// N = 4 TN MMAs whose B operand spans both CTAs' shared memory.  Per CTA that is 6 KB of
// operand reads per 64-clock MMA (96 B/clk) instead of the single-CTA N = 128 tile's 8 KB
// (128 B/clk, shared-memory bound: the r02 timeline measured its MMA phase at 7.2 us against
// 4.2 us of tensor work).  The P_s accumulators of each CTA's 128 rows live in its own TMEM;
// every tile starts from TMEM zeroed by the epilogue (tcgen05.st), so all MMAs accumulate —
// the single-CTA kernel's N = 192 / 64 initialisation sequence would split B across the pair
// differently.  Stage hand-off: each CTA's TMA completes on its own full barrier; the peer's
// warp 1 forwards its completion to the leader (remote mbarrier arrive, release.cluster); the
// leader's commits are multicast to both CTAs' empty / accumulator barriers; both CTAs'
// epilogue warps arrive (locally or remotely) on the leader's TMEM-empty barrier.
constexpr int kStages2 = 6;
constexpr int kThreadsTc2 = 320;  // warp 0 TMA, warp 1 MMA (leader) / forwarder (peer), warps 2-9 epilogue
template <int TN>
struct Tc2Smem {
    static constexpr uint32_t A_LIMB = TM * TK;        // 8 KB: this CTA's 128 rows
    static constexpr uint32_t A_STAGE = 4 * A_LIMB;    // 32 KB
    static constexpr uint32_t B_LIMB = TN * TK;        // 2 KB at TN = 32
    static constexpr uint32_t B_STAGE = 2 * B_LIMB;    // this CTA's two limbs of [B0|B1|B2|B3]
    static constexpr uint32_t STAGE = A_STAGE + B_STAGE;
    static constexpr uint32_t BYTES = kStages2 * STAGE + 1024 + 512;
    static constexpr uint32_t TMEM_COLS = 7 * TN <= 256 ? 256 : 512;
};

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// bounded wait with cluster-scope acquire (the arrivals came from the peer CTA)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t phase) {
    uint32_t done = 0;
    for (uint32_t it = 0; it < (1u << 26); ++it) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
        if (done) return;
    }
    __trap();
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mma_i8_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc) {
    asm volatile("tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, 1;" ::"r"(d_tmem), "l"(adesc), "l"(bdesc),
                 "r"(idesc));
}
// arrive on `bar` (same shared offset) in both CTAs of the pair once the issued MMAs complete
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
}
__device__ __forceinline__ void tmem_zero16(uint32_t taddr) {
    const uint32_t z = 0;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr),
        "r"(z)
        : "memory");
}

template <int TN>
__global__ void __launch_bounds__(kThreadsTc2, 1) k_modgemm_tc2(const uint8_t* __restrict__ At,
                                                                 const uint8_t* __restrict__ Bt, uint32_t M, uint32_t N,
                                                                 uint32_t KB, uint32_t tiles_n, uint32_t n_tiles,
                                                                 TcOut out, uint64_t* tl) {
    static_assert(TN == 32, "epilogue assigns one 16-column chunk per warp of each lane quarter");
    using L = Tc2Smem<TN>;
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t sbase = (smem_u32(smem) + 1023u) & ~1023u;
    uint8_t* sgen = smem + (sbase - smem_u32(smem));
    uint64_t* full = reinterpret_cast<uint64_t*>(sgen + kStages2 * L::STAGE);
    uint64_t* empty = full + kStages2;
    uint64_t* pfull = empty + kStages2;  // leader: the peer's stage landed
    uint64_t* tfull = pfull + kStages2;  // both CTAs: the tile's MMAs completed
    uint64_t* tempty = tfull + 1;        // leader: 16 epilogue warps drained and re-zeroed TMEM
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const uint32_t pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    if (threadIdx.x == 0) {
        tl_mark(tl, 0);
        for (int s = 0; s < kStages2; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
            mbar_init(&pfull[s], 1);
        }
        mbar_init(tfull, 1);
        mbar_init(tempty, 16);
        mbar_fence_init();
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(L::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    cluster_sync_all();  // both CTAs: barriers initialised, TMEM allocated
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) {
        uint32_t lead;  // the pair's accumulators sit at the same TMEM address in both CTAs
        asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(lead) : "r"(mapa_shared(smem_u32(tmem_slot), 0)));
        if (lead != tmem) __trap();
        tl_mark(tl, 1);
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0) tl_mark(tl, 2);

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer (both CTAs: own A rows, own two B limbs) ----
            uint32_t g = 0;
            for (uint32_t tile = pair; tile < n_tiles; tile += npairs) {
                const uint32_t mt = tile / tiles_n, nt = tile % tiles_n;
                const uint8_t* a_src = At + (uint64_t)(2 * mt + rank) * KB * L::A_STAGE;
                const uint8_t* b_src = Bt + (uint64_t)nt * KB * (4 * L::B_LIMB) + rank * L::B_STAGE;
                for (uint32_t kb = 0; kb < KB; ++kb, ++g) {
                    const uint32_t s = g % kStages2;
                    if (g >= (uint32_t)kStages2) mbar_wait(&empty[s], ((g / kStages2) - 1) & 1);
                    const uint32_t dst = sbase + s * L::STAGE;
                    mbar_expect_tx(&full[s], L::STAGE);
                    bulk_g2s(dst, a_src + (uint64_t)kb * L::A_STAGE, L::A_STAGE, &full[s]);
                    bulk_g2s(dst + L::A_STAGE, b_src + (uint64_t)kb * (4 * L::B_LIMB), L::B_STAGE, &full[s]);
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0 && rank == 1) {  // ---- peer: forward each landed stage to the leader ----
            const uint32_t lead_pfull = mapa_shared(smem_u32(pfull), 0);
            uint32_t g = 0;
            for (uint32_t tile = pair; tile < n_tiles; tile += npairs)
                for (uint32_t kb = 0; kb < KB; ++kb, ++g) {
                    const uint32_t s = g % kStages2;
                    mbar_wait(&full[s], (g / kStages2) & 1);
                    mbar_arrive_cluster(lead_pfull + s * 8);
                }
        } else if (lane == 0) {  // ---- leader: MMA issuer for the pair ----
            constexpr uint32_t id4 = idesc_i8<4 * TN, 2 * TM>();
            uint32_t g = 0, it = 0;
            for (uint32_t tile = pair; tile < n_tiles; tile += npairs, ++it) {
                mbar_wait_cluster(tempty, it & 1);  // both CTAs' TMEM drained and zeroed
                asm volatile("tcgen05.fence::after_thread_sync;");
                for (uint32_t kb = 0; kb < KB; ++kb, ++g) {
                    const uint32_t s = g % kStages2;
                    mbar_wait(&full[s], (g / kStages2) & 1);
                    mbar_wait_cluster(&pfull[s], (g / kStages2) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    if (g == 0) tl_mark(tl, 3);
                    const uint32_t sa = sbase + s * L::STAGE, sb = sa + L::A_STAGE;
#pragma unroll
                    for (int ks = 0; ks < TK / 32; ++ks) {
                        const uint64_t bd = smem_desc(sb + ks * 2 * kLBO, kLBO, kSBO);
#pragma unroll
                        for (int i = 0; i < 4; ++i)
                            mma_i8_pair(tmem + i * TN, smem_desc(sa + i * L::A_LIMB + ks * 2 * kLBO, kLBO, kSBO), bd,
                                        id4);
                    }
                    mma_commit_pair(&empty[s]);  // frees the stage in both CTAs
                }
                mma_commit_pair(tfull);  // both CTAs' accumulators complete
            }
            tl_mark(tl, 4);
        }
        __syncwarp();
    } else {  // ---- epilogue: warps 2..9; TMEM lane quarter = warp % 4, 16-column chunk = (warp - 2) / 4 ----
        const uint32_t quarter = warp & 3, chunk = (warp - 2) >> 2;
        const uint32_t lane_base = tmem + ((quarter * 32u) << 16) + chunk * 16;
        const uint32_t tempty_addr = rank == 0 ? smem_u32(tempty) : mapa_shared(smem_u32(tempty), 0);
        auto zero_and_release = [&]() {  // the next tile's MMAs accumulate onto zeros
#pragma unroll
            for (int q = 0; q < 7; ++q) tmem_zero16(lane_base + q * TN);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(tempty_addr);
        };
        zero_and_release();
        uint32_t it = 0;
        for (uint32_t tile = pair; tile < n_tiles; tile += npairs, ++it) {
            const uint32_t mt = tile / tiles_n, nt = tile % tiles_n;
            const uint32_t row = (2 * mt + rank) * TM + quarter * 32 + lane;
            mbar_wait(tfull, it & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            if (warp == 2 && lane == 0) tl_mark(tl, 5);
            uint32_t v[7][16];
            tmem_ld16_x7<TN>(lane_base, v);
            zero_and_release();
            if (row < M) {
                uint32_t r[16];
                tc_recombine16(v, r);
                tc_store16(out, N, row, nt * TN + chunk * 16, r);
            }
            if (warp == 2 && lane == 0) tl_mark(tl, 6);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    cluster_sync_all();  // no CTA leaves while its peer may still signal it
    if (threadIdx.x == 0) tl_mark(tl, 7);
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(L::TMEM_COLS));
}

// A (rows, stacked a0 over a1) -> pre-tiled limb image, one thread per 16-byte piece
// of the (128-row x 64-k) block: piece q = (r / 8) * 32 + (k / 16) * 8 + r % 8 sits at
// byte 16 q of each limb image (= core_off), so a warp's four limb stores are 4 x 512
// contiguous bytes; its loads are 64-byte row segments.
// A(m, k) = a0[m*K + k] for m < M0, a1[(m-M0)*K + k] for M0 <= m < M; zero padded.
struct RowsArgs {
    const uint32_t* a0;
    const uint32_t* a1;
    uint32_t M0, M, K, Mp, KB;
    uint8_t* out;
    uint32_t lda;  // row stride of a0/a1 (>= K; larger for a K slice of a wider matrix)
};
__device__ __forceinline__ void tile_rows(const RowsArgs& ra, uint64_t t0, uint64_t stride) {
    const uint32_t *a0 = ra.a0, *a1 = ra.a1;
    const uint32_t M0 = ra.M0, M = ra.M, K = ra.K, Mp = ra.Mp, KB = ra.KB, lda = ra.lda;
    uint8_t* out = ra.out;
    constexpr uint32_t kPieces = TM * TK / 16;  // 512 per block
    const uint64_t pieces = (uint64_t)(Mp / TM) * KB * kPieces;
    const bool v4 = (K % 4) == 0 && (lda % 4) == 0 &&
                    ((reinterpret_cast<uintptr_t>(a0) | reinterpret_cast<uintptr_t>(a1)) & 15u) == 0;
    for (uint64_t t = t0; t < pieces; t += stride) {
        const uint64_t blk = t / kPieces;
        const uint32_t q = (uint32_t)(t % kPieces);
        const uint32_t r = (q / 32) * 8 + (q % 8), kk = ((q / 8) % 4) * 16;
        const uint32_t mt = (uint32_t)(blk / KB), kb = (uint32_t)(blk % KB);
        const uint32_t m = mt * TM + r, k0 = kb * TK + kk;
        uint32_t w[16];
        const uint32_t* row = m < M0 ? a0 + (uint64_t)m * lda : a1 + (uint64_t)(m - M0) * lda;
        if (v4 && m < M && k0 + 16 <= K) {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const uint4 u = __ldg(reinterpret_cast<const uint4*>(row + k0) + c);
                w[4 * c] = u.x;
                w[4 * c + 1] = u.y;
                w[4 * c + 2] = u.z;
                w[4 * c + 3] = u.w;
            }
        } else {
#pragma unroll
            for (int c = 0; c < 16; ++c) w[c] = (m < M && k0 + c < K) ? row[k0 + c] : 0u;
        }
        uint8_t* dst = out + blk * (4u * TM * TK) + 16u * q;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            uint32_t p[4];
#pragma unroll
            for (int c = 0; c < 4; ++c)
                p[c] = __byte_perm(__byte_perm(w[4 * c] >> (8 * i), w[4 * c + 1] >> (8 * i), 0x0040),
                                   __byte_perm(w[4 * c + 2] >> (8 * i), w[4 * c + 3] >> (8 * i), 0x0040), 0x5410);
            *reinterpret_cast<uint4*>(dst + i * (TM * TK)) = make_uint4(p[0], p[1], p[2], p[3]);
        }
    }
}

// B (K x N, columns stacked b0 | b1) -> pre-tiled K-major limb image (transposed):
// block = 64 k x 32 n through shared memory; one thread per (n, 16-k chunk) on the way out.
// With bx.e set, the operand is B + coef * E (E: K x NB, the same plane under both
// halves; coef0 for columns < NB, coef1 after) — the matrix-triple combine's
// B.v + [party 0] E and B.m + alpha_i E, formed on the way into the limb image.
struct ColsArgs {
    const uint32_t* b0;
    const uint32_t* b1;
    uint32_t NB, N, K, KB;
    TcBx bx;
    uint8_t* out;
};
template <int BN>
__device__ __forceinline__ void tile_cols(const ColsArgs& ca, uint32_t kb, uint32_t nt32, uint32_t (&tile)[TK][33]) {
    const uint32_t *b0 = ca.b0, *b1 = ca.b1;
    const uint32_t NB = ca.NB, N = ca.N, K = ca.K, KB = ca.KB;
    const TcBx& bx = ca.bx;
    uint8_t* out = ca.out;
    for (uint32_t e = threadIdx.x; e < TK * 32; e += blockDim.x) {
        const uint32_t kk = e / 32, nn = e % 32;
        const uint32_t k = kb * TK + kk, n = nt32 + nn;
        uint32_t v = 0;
        if (k < K && n < N) {
            const bool hi = n >= NB;
            const uint64_t off = (uint64_t)k * NB + (hi ? n - NB : n);
            v = (hi ? b1 : b0)[off];
            if (bx.e) v = fp_add(v, fp_mul(hi ? bx.coef1 : bx.coef0, bx.e[off]));
        }
        tile[kk][nn] = v;
    }
    __syncthreads();
    for (uint32_t c = threadIdx.x; c < 32 * (TK / 16); c += blockDim.x) {
        const uint32_t nn = c / (TK / 16), kc = c % (TK / 16);
        const uint32_t n = nt32 + nn;
        const uint32_t nt = n / BN, r = n % BN;
        uint8_t* blk = out + ((uint64_t)nt * KB + kb) * (4u * BN * TK);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            uint32_t p[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t base = kc * 16 + 4 * q;
                p[q] = ((tile[base][nn] >> (8 * j)) & 0xFF) | (((tile[base + 1][nn] >> (8 * j)) & 0xFF) << 8) |
                       (((tile[base + 2][nn] >> (8 * j)) & 0xFF) << 16) | (((tile[base + 3][nn] >> (8 * j)) & 0xFF) << 24);
            }
            *reinterpret_cast<uint4*>(blk + j * (BN * TK) + core_off(r, kc * 16)) = make_uint4(p[0], p[1], p[2], p[3]);
        }
    }
}

// Both re-layouts in one launch: blocks [0, row_blocks) split A (grid-strided pieces),
// the rest transpose-split one 64 k x 32 n block of B each.  The first instruction
// lets the dependent GEMM grid launch (programmatic dependent launch): its prologue
// (barrier init, TMEM allocation) overlaps this kernel; it waits before reading.
template <int BN>
__global__ void __launch_bounds__(256) k_tile_both(RowsArgs ra, ColsArgs ca, uint32_t row_blocks, uint32_t col_kb) {
    asm volatile("griddepcontrol.launch_dependents;");
    __shared__ uint32_t tile[TK][33];
    if (blockIdx.x < row_blocks) {
        tile_rows(ra, (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, (uint64_t)row_blocks * blockDim.x);
    } else {
        const uint32_t c = blockIdx.x - row_blocks;
        tile_cols<BN>(ca, c % col_kb, (c / col_kb) * 32, tile);
    }
}

// ---------------------------------------------------------------------------
// Narrow problems (C3: 1024 x 512 outputs, K = 1024): split-K CTA clusters on 128 x 64 tiles
// (k_modgemm_tcs).
// ---------------------------------------------------------------------------
// Per SM the limb GEMM is bound by shared-memory bandwidth (~128 B/clk: operand fills plus the
// MMAs' operand reads) and, in the epilogue, by TMEM reads (~64 B/clk: seven s32 accumulators per
// output).  The persistent kernel's 128 x 32 tiles (the only tiling that fills the SMs at C3) issue
// N = 128 MMAs that read 8 KB per 64 clocks, 208 B/clk with the fills: ~1.6x the tensor time.  Here
// a cluster of two CTAs shares one 128 x 64 output tile and splits K: N = 256 MMAs (96 B/clk) plus
// fills (48 B/clk), 2 x 64 = 128 CTAs at C3, at the price of each CTA draining all 448 accumulator
// columns of its K half (twice the epilogue's TMEM reads).  Each CTA recombines its 64 columns mod
// p, pushes the 32 its peer finalises into the peer's shared memory (st.shared::cluster) and, after
// one cluster barrier, adds the peer's half to its own 32 columns.  Operands: A (W) always from a
// limb image by TMA (prepared once for a public W, or by a re-layout launch of W alone); X split into
// limbs by the 16 worker warps (8 consecutive k of one column per thread, warp-coalesced loads), or,
// when B carries the + coef E transform, from the re-layout launch's image by TMA.  The
// worker warps then drain TMEM, one 16-column chunk each (4 per TMEM lane quarter).
constexpr int kStagesS = 4;
constexpr int kWorkWarps = 16;    // producers, then one 16-column epilogue chunk each (4 per TMEM lane quarter)
constexpr int kThreadsTcs = 32 * (1 + kWorkWarps);  // warp 0: MMA issuer
struct TcsSmem {
    static constexpr uint32_t A_LIMB = TM * TK;      // 8 KB
    static constexpr uint32_t A_STAGE = 4 * A_LIMB;  // 32 KB
    static constexpr uint32_t B_LIMB = 64 * TK;      // 4 KB
    static constexpr uint32_t B_STAGE = 4 * B_LIMB;  // 16 KB
    static constexpr uint32_t STAGE = A_STAGE + B_STAGE;
    static constexpr uint32_t XPITCH = 36;           // exchange row pitch (u32): conflict-free v4 stores
    static constexpr uint32_t XBUF = TM * XPITCH * 4;  // 18 KB
    static constexpr uint32_t BYTES = kStagesS * STAGE + XBUF + 1024 + 256;
};

// 4 u32 words -> their 4 byte-planes: limb[i] = [w0.b_i, w1.b_i, w2.b_i, w3.b_i]
__device__ __forceinline__ void split4(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3, uint32_t (&limb)[4]) {
    const uint32_t t0 = __byte_perm(w0, w1, 0x5140), t1 = __byte_perm(w0, w1, 0x7362);
    const uint32_t t2 = __byte_perm(w2, w3, 0x5140), t3 = __byte_perm(w2, w3, 0x7362);
    limb[0] = __byte_perm(t0, t2, 0x5410);
    limb[1] = __byte_perm(t0, t2, 0x7632);
    limb[2] = __byte_perm(t1, t3, 0x5410);
    limb[3] = __byte_perm(t1, t3, 0x7632);
}

__device__ __forceinline__ void st_cluster_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared::cluster.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
}

struct TcsArgs {
    const uint8_t* a_image;  // A limb image (mt-major blocks of 4 x 128 x 64, KB per row block)
    const uint8_t* b_image;  // B limb image of the re-layout kernel (nt-major blocks of 4 x 64 x 64), or null
    ColsArgs b;              // X (K x N, b0 | b1 columns, row stride NB) when b_image is null
    uint32_t M, N, KB, tiles_n;
    TcOut out;
};

// One stage's B words in registers (worker thread pt in [0, 512)): 8 consecutive k of one column of
// X.  Every load of a stage is issued before any of its words is used (the limb split happens in
// tcs_store_b), and the next stage's loads are in flight while this one is stored.
struct TcsLd {
    uint32_t b[8];
};

__device__ __forceinline__ void tcs_load_b(const ColsArgs& ca, uint32_t nt, uint32_t kb, uint32_t pt, TcsLd& x) {
    const uint32_t n = nt * 64 + (pt & 63), k0 = kb * TK + (pt >> 6) * 8;
    const uint32_t* col = (n >= ca.NB ? ca.b1 + (n - ca.NB) : ca.b0 + n) + (uint64_t)k0 * ca.NB;
    if (n < ca.N && k0 + 8 <= ca.K) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x.b[i] = __ldg(col + (uint64_t)i * ca.NB);
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) x.b[i] = (n < ca.N && k0 + i < ca.K) ? __ldg(col + (uint64_t)i * ca.NB) : 0u;
    }
}

// split the loaded words into the stage's four B limb tiles (canonical K-major no-swizzle image)
__device__ __forceinline__ void tcs_store_b(uint8_t* sb, uint32_t pt, const TcsLd& x) {
    const uint32_t n = pt & 63, kk = (pt >> 6) * 8;
    uint32_t l0[4], l1[4];
    split4(x.b[0], x.b[1], x.b[2], x.b[3], l0);
    split4(x.b[4], x.b[5], x.b[6], x.b[7], l1);
#pragma unroll
    for (int j = 0; j < 4; ++j)
        *reinterpret_cast<uint2*>(sb + j * TcsSmem::B_LIMB + core_off(n, kk)) = make_uint2(l0[j], l1[j]);
}

// Eight output columns c0 .. c0+7 of this thread's TMEM lane: the seven P_s (7 x 8 words, one
// wait), recombined mod p.
template <int TN>
__device__ __forceinline__ void tc_chunk8(uint32_t taddr, uint32_t* r) {
    uint32_t v[7][8];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%56];\n"
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%8,%9,%10,%11,%12,%13,%14,%15}, [%57];\n"
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%16,%17,%18,%19,%20,%21,%22,%23}, [%58];\n"
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%24,%25,%26,%27,%28,%29,%30,%31}, [%59];\n"
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%32,%33,%34,%35,%36,%37,%38,%39}, [%60];\n"
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%40,%41,%42,%43,%44,%45,%46,%47}, [%61];\n"
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%48,%49,%50,%51,%52,%53,%54,%55}, [%62];\n"
        "tcgen05.wait::ld.sync.aligned;\n"
        : "=r"(v[0][0]), "=r"(v[0][1]), "=r"(v[0][2]), "=r"(v[0][3]), "=r"(v[0][4]), "=r"(v[0][5]), "=r"(v[0][6]),
          "=r"(v[0][7]), "=r"(v[1][0]), "=r"(v[1][1]), "=r"(v[1][2]), "=r"(v[1][3]), "=r"(v[1][4]), "=r"(v[1][5]),
          "=r"(v[1][6]), "=r"(v[1][7]), "=r"(v[2][0]), "=r"(v[2][1]), "=r"(v[2][2]), "=r"(v[2][3]), "=r"(v[2][4]),
          "=r"(v[2][5]), "=r"(v[2][6]), "=r"(v[2][7]), "=r"(v[3][0]), "=r"(v[3][1]), "=r"(v[3][2]), "=r"(v[3][3]),
          "=r"(v[3][4]), "=r"(v[3][5]), "=r"(v[3][6]), "=r"(v[3][7]), "=r"(v[4][0]), "=r"(v[4][1]), "=r"(v[4][2]),
          "=r"(v[4][3]), "=r"(v[4][4]), "=r"(v[4][5]), "=r"(v[4][6]), "=r"(v[4][7]), "=r"(v[5][0]), "=r"(v[5][1]),
          "=r"(v[5][2]), "=r"(v[5][3]), "=r"(v[5][4]), "=r"(v[5][5]), "=r"(v[5][6]), "=r"(v[5][7]), "=r"(v[6][0]),
          "=r"(v[6][1]), "=r"(v[6][2]), "=r"(v[6][3]), "=r"(v[6][4]), "=r"(v[6][5]), "=r"(v[6][6]), "=r"(v[6][7])
        : "r"(taddr), "r"(taddr + TN), "r"(taddr + 2 * TN), "r"(taddr + 3 * TN), "r"(taddr + 4 * TN),
          "r"(taddr + 5 * TN), "r"(taddr + 6 * TN)
        : "memory");
    constexpr uint32_t kPow[7] = {1u, 256u, 65536u, 16777216u, 5u, 1280u, 327680u};
#pragma unroll
    for (int t = 0; t < 8; ++t) {
        unsigned long long acc = v[0][t];
#pragma unroll
        for (int q = 1; q < 7; ++q) acc += (unsigned long long)v[q][t] * kPow[q];
        r[t] = fp_reduce64(acc);
    }
}

template <bool kBImg>
__global__ void __launch_bounds__(kThreadsTcs, 1) k_modgemm_tcs(const TcsArgs p, uint64_t* tl) {
    using L = TcsSmem;
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t sbase = (smem_u32(smem) + 1023u) & ~1023u;
    uint8_t* sgen = smem + (sbase - smem_u32(smem));
    uint32_t* xbuf = reinterpret_cast<uint32_t*>(sgen + kStagesS * L::STAGE);
    uint64_t* full = reinterpret_cast<uint64_t*>(sgen + kStagesS * L::STAGE + L::XBUF);
    uint64_t* empty = full + kStagesS;
    uint64_t* tfull = empty + kStagesS;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t ks, kr;  // K split (cluster size) and this CTA's K half
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(ks));
    kr = ks > 1 ? cluster_rank() : 0u;
    const uint32_t tile = blockIdx.x / ks, mt = tile / p.tiles_n, nt = tile % p.tiles_n;
    const uint32_t kper = (p.KB + ks - 1) / ks, kb0 = kr * kper, kb1 = min(p.KB, kb0 + kper);
    const uint32_t nkb = kb1 > kb0 ? kb1 - kb0 : 0;  // the launcher splits only when both halves are non-empty
    if (threadIdx.x == 0) {
        tl_mark(tl, 0);
        for (int s = 0; s < kStagesS; ++s) {
            mbar_init(&full[s], kWorkWarps + 1);  // + the TMA thread's expect_tx arrival
            mbar_init(&empty[s], 1);
        }
        mbar_init(tfull, 1);
        mbar_fence_init();
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    if (ks > 1) cluster_sync_all();  // the peer is running (its shared memory is addressable) and initialised
    else __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) tl_mark(tl, 1);
    asm volatile("griddepcontrol.wait;" ::: "memory");  // inputs written by the previous kernel are visible
    if (threadIdx.x == 0) tl_mark(tl, 2);

    // worker warps 1-16: TMEM lane quarter = warp % 4, 16-column chunk = (warp - 1) / 4
    const uint32_t quarter = warp & 3, cidx = (warp - 1) >> 2;
    const uint32_t lrow = quarter * 32 + lane, row = mt * TM + lrow;
    uint32_t r[16];  // this warp's chunk, mod p
    if (warp == 0) {
        if (lane == 0) {  // ---- MMA issuer ----
            constexpr uint32_t id4 = idesc_i8<256>(), id3 = idesc_i8<192>(), id1 = idesc_i8<64>();
            for (uint32_t g = 0; g < nkb; ++g) {
                const uint32_t s = g % kStagesS;
                mbar_wait(&full[s], (g / kStagesS) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                if (g == 0) tl_mark(tl, 3);
                const uint32_t sa = sbase + s * L::STAGE, sb = sa + L::A_STAGE;
#pragma unroll
                for (int kq = 0; kq < TK / 32; ++kq) {
                    const uint64_t bd = smem_desc(sb + kq * 2 * kLBO, kLBO, kSBO);
                    uint64_t ad[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) ad[i] = smem_desc(sa + i * L::A_LIMB + kq * 2 * kLBO, kLBO, kSBO);
                    if (g == 0 && kq == 0) {  // initialise P_0..P_6 (overlapping destination ranges)
                        const uint64_t bd3 = smem_desc(sb + 3 * L::B_LIMB + kq * 2 * kLBO, kLBO, kSBO);
                        mma_i8(tmem, ad[0], bd, id3, 0u);
                        mma_i8(tmem + 3 * 64, ad[3], bd, id4, 0u);
                        mma_i8(tmem + 3 * 64, ad[0], bd3, id1, 1u);
                        mma_i8(tmem + 1 * 64, ad[1], bd, id4, 1u);
                        mma_i8(tmem + 2 * 64, ad[2], bd, id4, 1u);
                    } else {
#pragma unroll
                        for (int i = 0; i < 4; ++i) mma_i8(tmem + i * 64, ad[i], bd, id4, 1u);
                    }
                }
                mma_commit(&empty[s]);
            }
            mma_commit(tfull);
            tl_mark(tl, 4);
            // every MMA of this CTA is issued: the next kernel in the stream (programmatic dependent
            // launch) may start its prologue on SMs this grid frees; it reads nothing before its
            // griddepcontrol.wait, which waits for this whole grid and its memory
            asm volatile("griddepcontrol.launch_dependents;");
        }
        __syncwarp();
    } else {  // ---- warps 1-16: producers, then epilogue ----
        const uint32_t pt = threadIdx.x - 32;
        auto put = [&](const TcsLd& x, uint32_t g) {
            const uint32_t s = g % kStagesS;
            if (lane == 0 && g >= (uint32_t)kStagesS) mbar_wait(&empty[s], ((g / kStagesS) - 1) & 1);
            __syncwarp();
            if (pt == 0) {
                mbar_expect_tx(&full[s], L::A_STAGE + (kBImg ? L::B_STAGE : 0u));
                bulk_g2s(sbase + s * L::STAGE, p.a_image + ((uint64_t)mt * p.KB + kb0 + g) * L::A_STAGE, L::A_STAGE,
                         &full[s]);
                if (kBImg)
                    bulk_g2s(sbase + s * L::STAGE + L::A_STAGE,
                             p.b_image + ((uint64_t)nt * p.KB + kb0 + g) * L::B_STAGE, L::B_STAGE, &full[s]);
            }
            if (!kBImg) {
                tcs_store_b(sgen + s * L::STAGE + L::A_STAGE, pt, x);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic stores -> tensor-core reads
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[s]);
        };
        TcsLd x0, x1;
        if (!kBImg && nkb > 0) tcs_load_b(p.b, nt, kb0, pt, x0);
        for (uint32_t g = 0; g < nkb; g += 2) {
            if (!kBImg && g + 1 < nkb) tcs_load_b(p.b, nt, kb0 + g + 1, pt, x1);
            put(x0, g);
            if (g + 1 >= nkb) break;
            if (!kBImg && g + 2 < nkb) tcs_load_b(p.b, nt, kb0 + g + 2, pt, x0);
            put(x1, g + 1);
        }
        if (warp == 1 && lane == 0) tl_mark(tl, 8);  // this warp's last stage handed over
        // ---- epilogue: one 16-column chunk per warp, as two 8-column halves ----
        mbar_wait(tfull, 0);
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (warp == 1 && lane == 0) tl_mark(tl, 5);
        const uint32_t taddr = tmem + ((quarter * 32u) << 16) + cidx * 16;
        tc_chunk8<64>(taddr, r);
        tc_chunk8<64>(taddr + 8, r + 8);
        if (ks == 1) {
            if (row < p.M) tc_store16(p.out, p.N, row, nt * 64 + cidx * 16, r);
        } else if ((cidx >> 1) != kr) {  // the peer finalises these columns: push them
            const uint32_t dst = mapa_shared(smem_u32(xbuf + lrow * L::XPITCH + 16 * (cidx & 1)), 1 - kr);
#pragma unroll
            for (int c = 0; c < 4; ++c) st_cluster_v4(dst + 16 * c, r[4 * c], r[4 * c + 1], r[4 * c + 2], r[4 * c + 3]);
            if (warp == 1 && lane == 0) tl_mark(tl, 9);
        }
        if (warp == 1 && lane == 0) tl_mark(tl, 10);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    if (ks > 1) {
        __syncwarp();
        cluster_sync_all();  // every pushed half is in its owner's shared memory
        if (threadIdx.x == 32) tl_mark(tl, 11);
        if (warp > 0 && (cidx >> 1) == kr) {
            const uint4* src = reinterpret_cast<const uint4*>(xbuf + lrow * L::XPITCH + 16 * (cidx & 1));
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const uint4 u = src[c];
                r[4 * c] = fp_add(r[4 * c], u.x);
                r[4 * c + 1] = fp_add(r[4 * c + 1], u.y);
                r[4 * c + 2] = fp_add(r[4 * c + 2], u.z);
                r[4 * c + 3] = fp_add(r[4 * c + 3], u.w);
            }
            if (row < p.M) tc_store16(p.out, p.N, row, nt * 64 + cidx * 16, r);
        }
    }
    if (warp == 1 && lane == 0) tl_mark(tl, 6);
    __syncthreads();
    if (threadIdx.x == 0) tl_mark(tl, 7);
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// Diagnostic switches (attribution experiments, scripts/gemm_probe.py): bit 0 skips the TMA
// loads, bit 1 the MMAs, bit 2 the GEMM kernel, bit 3 the re-layout kernels (results invalid
// while any is set); bit 6 / bit 7 force the 32- / 64-column tile width (results valid).
uint32_t g_tc_dbg = 0;
uint64_t* g_tc_tl = nullptr;  // diagnostic timeline buffer (8 stamps per CTA), or null

// Re-layout both operands into limb images (B tiles BN columns wide), then run
// the GEMM kernel with TN = BN.
template <int BN>
cudaError_t run_tc(cudaStream_t s, int mode, uint32_t dout, uint32_t din, uint32_t lda, uint32_t batch,
                   const uint32_t* w0, const uint32_t* w1, const uint32_t* x0, const uint32_t* x1, const TcBx& bx,
                   uint8_t* scratch, const uint8_t* a_image, const TcOut& out, int sms, bool pair = false) {
    const uint32_t M = mode == 0 ? dout : 2 * dout, N = mode == 0 ? 2 * batch : batch;
    const uint32_t Mp = (M + 2 * TM - 1) / (2 * TM) * (2 * TM), Np = (N + BN - 1) / BN * BN;  // pair tiles: 256 rows
    const uint32_t KB = (din + TK - 1) / TK;
    // a prepared A image (spdz_linear_weights) is used as is: only B is re-laid out
    const uint8_t* At = a_image ? a_image : scratch;
    uint8_t* Bt = a_image ? scratch : scratch + (uint64_t)4 * Mp * KB * TK;
    bool pdl = false;
    if (!(g_tc_dbg & 8)) {  // (diagnostic bit 3 skips the re-layout kernels)
        const uint64_t chunks = (uint64_t)Mp * KB * (TK / 16);
        const uint32_t row_blocks =
            a_image ? 0u : (uint32_t)std::min<uint64_t>((chunks + 255) / 256, (uint64_t)sms * 16);
        const uint32_t col_blocks = KB * ((Np + 31) / 32);
        const RowsArgs ra{w0, mode == 0 ? w0 : w1, mode == 0 ? M : dout, M, din, Mp, KB, scratch, lda};
        const ColsArgs ca{x0, mode == 0 ? x1 : x0, batch, N, din, KB, mode == 0 ? bx : TcBx{}, Bt};
        k_tile_both<BN><<<row_blocks + col_blocks, 256, 0, s>>>(ra, ca, row_blocks, KB);
        ++g_kernel_launches;
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        pdl = true;
    }
    if (g_tc_dbg & 4) return cudaSuccess;  // (diagnostic bit 2 skips the GEMM kernel)
    if (pair) {  // CTA pairs on 256 x 32 tiles (k_modgemm_tc2)
        using L2 = Tc2Smem<32>;
        static bool attr_pair = false;
        if (!attr_pair) {
            cudaError_t e = cudaFuncSetAttribute(k_modgemm_tc2<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 L2::BYTES);
            if (e != cudaSuccess) return e;
            attr_pair = true;
        }
        const uint32_t tiles_n = Np / 32, n_tiles = tiles_n * (Mp / (2 * TM));
        const uint32_t pairs = std::min<uint32_t>(n_tiles, (uint32_t)sms / 2);
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(2 * pairs);
        cfg.blockDim = dim3(kThreadsTc2);
        cfg.dynamicSmemBytes = L2::BYTES;
        cfg.stream = s;
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = pdl ? 2 : 1;
        cudaError_t e = cudaLaunchKernelEx(&cfg, k_modgemm_tc2<32>, (const uint8_t*)At, (const uint8_t*)Bt, M, N, KB,
                                           tiles_n, n_tiles, out, g_tc_tl);
        ++g_kernel_launches;
        if (e != cudaSuccess) return e;
        return cudaGetLastError();
    }
    using L = TcSmem<BN>;
    static bool attr2 = false;
    if (!attr2) {
        cudaError_t e = cudaFuncSetAttribute(k_modgemm_tc<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::BYTES);
        if (e != cudaSuccess) return e;
        attr2 = true;
    }
    const uint32_t tiles_n = Np / BN, n_tiles = tiles_n * ((M + TM - 1) / TM);  // (the image pads M to 256)
    const int grid = (int)std::min<uint32_t>(n_tiles, (uint32_t)sms);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreadsTc);
    cfg.dynamicSmemBytes = L::BYTES;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;  // overlap our prologue with the re-layout kernel's tail
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_modgemm_tc<BN>, (const uint8_t*)At, (const uint8_t*)Bt, M, N, KB,
                                       tiles_n, n_tiles, out, g_tc_dbg & 3u, g_tc_tl);
    ++g_kernel_launches;
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

// Narrow problems: k_modgemm_tcs on 128 x 64 tiles, K split over a 2-CTA cluster when both halves
// get at least one stage and the doubled grid still fits on the SMs (diagnostic bit 11 keeps one CTA).
// A prepared W image: one launch, X split into limbs by the worker warps.  W per call: one re-layout
// launch of W (k_tile_both, PDL-chained), X still split in the kernel (eager 19.3 -> 17.5 us per C3 call
// against re-laying out both, profiles/r02n); with the E transform both operands are re-laid out and
// every stage is two TMA bulk copies.
cudaError_t run_tcs(cudaStream_t s, int mode, uint32_t dout, uint32_t din, uint32_t lda, uint32_t batch,
                    const uint32_t* w0, const uint32_t* w1, const uint32_t* x0, const uint32_t* x1, const TcBx& bx,
                    const uint8_t* a_image, uint8_t* scratch, const TcOut& out, int sms) {
    const uint32_t M = mode == 0 ? dout : 2 * dout, N = mode == 0 ? 2 * batch : batch;
    const uint32_t KB = (din + TK - 1) / TK, tiles_n = (N + 63) / 64, tiles = tiles_n * ((M + TM - 1) / TM);
    const uint32_t ks = (KB >= 2 && 2 * tiles <= (uint32_t)sms && !(g_tc_dbg & 2048)) ? 2 : 1;
    TcsArgs p{};
    p.a_image = a_image;
    p.b = ColsArgs{x0, mode == 0 ? x1 : x0, batch, N, din, KB, mode == 0 ? bx : TcBx{}, nullptr};
    p.M = M;
    p.N = N;
    p.KB = KB;
    p.tiles_n = tiles_n;
    p.out = out;
    // Re-layout launch: the A (W) limb image unless prepared, and the B image only when B carries
    // the + coef E transform (batched secret x secret); otherwise X is split in the kernel's worker
    // warps, as with a prepared W (diagnostic bit 13: the B image by re-layout as well).
    const bool b_relayout = bx.e || (!a_image && (g_tc_dbg & 8192));
    if (!a_image || b_relayout) {
        const uint32_t Mp = (M + 2 * TM - 1) / (2 * TM) * (2 * TM), Np = (N + 63) / 64 * 64;
        uint8_t* At = a_image ? nullptr : scratch;
        uint8_t* Bt = a_image ? scratch : scratch + (uint64_t)4 * Mp * KB * TK;
        const uint64_t chunks = (uint64_t)Mp * KB * (TK / 16);
        const uint32_t row_blocks = a_image ? 0u : (uint32_t)std::min<uint64_t>((chunks + 255) / 256, (uint64_t)sms * 16);
        const RowsArgs ra{w0, mode == 0 ? w0 : w1, mode == 0 ? M : dout, M, din, Mp, KB, At, lda};
        ColsArgs ca = p.b;
        ca.out = Bt;
        const uint32_t col_blocks = b_relayout ? KB * (Np / 32) : 0u;
        k_tile_both<64><<<row_blocks + col_blocks, 256, 0, s>>>(ra, ca, row_blocks, KB);
        ++g_kernel_launches;
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        p.a_image = a_image ? a_image : At;
        p.b_image = b_relayout ? Bt : nullptr;
    }
    static bool attr = false;
    if (!attr) {
        for (auto* f : {k_modgemm_tcs<false>, k_modgemm_tcs<true>}) {
            cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, TcsSmem::BYTES);
            if (e != cudaSuccess) return e;
        }
        attr = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(tiles * ks);
    cfg.blockDim = dim3(kThreadsTcs);
    cfg.dynamicSmemBytes = TcsSmem::BYTES;
    cfg.stream = s;
    cudaLaunchAttribute attrs[2];
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = ks;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // prologue overlaps the previous kernel
    attrs[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = ks > 1 ? attrs : attrs + 1;
    cfg.numAttrs = (ks > 1 ? 1 : 0) + 1;  // programmatic dependent launch after whatever precedes it
    cudaError_t e = p.b_image ? cudaLaunchKernelEx(&cfg, k_modgemm_tcs<true>, p, g_tc_tl)
                              : cudaLaunchKernelEx(&cfg, k_modgemm_tcs<false>, p, g_tc_tl);
    ++g_kernel_launches;
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace

void modgemm_tc_debug(uint32_t flags) { g_tc_dbg = flags; }
void modgemm_tc_timeline(uint64_t* dev_buf) { g_tc_tl = dev_buf; }
uint64_t modgemm_tc_scratch_bytes(int mode, uint32_t dout, uint32_t din, uint32_t batch) {
    din = std::min<uint32_t>(din, kMaxKSlice);  // one K slice at a time
    const uint64_t M = mode == 0 ? dout : 2ull * dout, N = mode == 0 ? 2ull * batch : batch;
    const uint64_t Mp = (M + 2 * TM - 1) / (2 * TM) * (2 * TM), Np = (N + 63) / 64 * 64, Kp = (din + TK - 1) / TK * TK;
    return 4 * (Mp + Np) * Kp + 256;
}

bool modgemm_tc_supported(uint32_t din) { return din >= 1; }  // K > kMaxKSlice runs as K slices

// Y (dout x batch, two planes) for the secret x public linear layer on tcgen05.
//   mode 0: W public (w0), X secret planes (x0 vals, x1 macs): C = W * [Xv | Xm]
//   mode 1: W secret planes (w0, w1), X public (x0):           C = [Wv ; Wm] * X
// Optional (aux): mode 0 right operand X_h + coef_h * E; Y = addend + C.
cudaError_t launch_modgemm_tc(cudaStream_t s, int mode, uint32_t dout, uint32_t din, uint32_t batch,
                              const uint32_t* w0, const uint32_t* w1, const uint32_t* x0, const uint32_t* x1,
                              uint32_t* y0, uint32_t* y1, uint8_t* scratch, int sms, const TcAux* aux) {
    if (dout == 0 || batch == 0) return cudaSuccess;
    const uint64_t M = mode == 0 ? dout : 2ull * dout, N = mode == 0 ? 2ull * batch : batch;
    // K slices of at most kMaxKSlice (the s32 limb-accumulator bound); slice i > 0 adds into
    // the running result through the epilogue addend, so the sum stays exact mod p
    const uint8_t* ai = aux ? aux->a_image : nullptr;
    if (ai && din > kMaxKSlice) return cudaErrorInvalidValue;  // prepared images are single-slice
    for (uint32_t k0 = 0; k0 < din; k0 += kMaxKSlice) {
        const uint32_t kc = std::min<uint32_t>(kMaxKSlice, din - k0);
        TcOut out{mode, dout, batch, y0, y1, aux ? aux->add0 : nullptr, aux ? aux->add1 : nullptr};
        if (k0 > 0) {
            out.add0 = y0;
            out.add1 = y1;
        }
        const uint64_t xo = (uint64_t)k0 * batch;  // X rows k0.. (row-major din x batch)
        TcBx bx{aux && aux->e ? aux->e + xo : nullptr, aux ? aux->coef0 : 0u, aux ? aux->coef1 : 0u};
        const uint32_t* a0 = w0 ? w0 + k0 : nullptr;
        const uint32_t* a1 = w1 ? w1 + k0 : nullptr;
        const uint32_t* b0 = x0 + xo;
        const uint32_t* b1 = x1 ? x1 + xo : nullptr;
        // Problems whose 128 x 64 tiling fills the SMs: the persistent k_modgemm_tc (TN = 64) after one
        // re-layout launch.  Narrower ones (C3): the split-K cluster kernel k_modgemm_tcs, operands split
        // in its producer warps (bit 12 forces it for any shape, bit 11 keeps it on one CTA per tile).
        // Diagnostic comparisons: bit 6 the TN = 32 persistent kernel, bit 7 TN = 64, bit 9 the CTA-pair
        // kernel on 256 x 32 tiles (k_modgemm_tc2; correct, measured slower at C3).
        const uint64_t tiles64 = (M + TM - 1) / TM * ((N + 63) / 64);
        const bool narrow = (g_tc_dbg & (64 | 512)) || (!(g_tc_dbg & 128) && tiles64 < (uint64_t)sms);
        const bool pair = narrow && (g_tc_dbg & 512);
        const bool split = (g_tc_dbg & 4096) || (narrow && !(g_tc_dbg & (64 | 128 | 512)));
        if (split && !(g_tc_dbg & 15)) {
            cudaError_t e = run_tcs(s, mode, dout, kc, din, batch, a0, a1, b0, b1, bx, ai, scratch, out, sms);
            if (e != cudaSuccess) return e;
            continue;
        }
        cudaError_t e = narrow ? run_tc<32>(s, mode, dout, kc, din, batch, a0, a1, b0, b1, bx, scratch, ai, out, sms, pair)
                               : run_tc<64>(s, mode, dout, kc, din, batch, a0, a1, b0, b1, bx, scratch, ai, out, sms);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

// The A-side limb image alone (a public weight matrix prepared once for many calls).
uint64_t modgemm_tc_a_image_bytes(int mode, uint32_t dout, uint32_t din) {
    const uint64_t M = mode == 0 ? dout : 2ull * dout;
    const uint64_t Mp = (M + 2 * TM - 1) / (2 * TM) * (2 * TM), Kp = (din + TK - 1) / TK * TK;
    return 4 * Mp * Kp;
}

cudaError_t launch_tile_a(cudaStream_t s, int mode, uint32_t dout, uint32_t din, const uint32_t* w0,
                          const uint32_t* w1, uint8_t* image, int sms) {
    const uint32_t M = mode == 0 ? dout : 2 * dout;
    const uint32_t Mp = (M + 2 * TM - 1) / (2 * TM) * (2 * TM), KB = (din + TK - 1) / TK;
    const uint64_t chunks = (uint64_t)Mp * KB * (TK / 16);
    const uint32_t row_blocks = (uint32_t)std::min<uint64_t>((chunks + 255) / 256, (uint64_t)sms * 16);
    const RowsArgs ra{w0, mode == 0 ? w0 : w1, mode == 0 ? M : dout, M, din, Mp, KB, image, din};
    k_tile_both<64><<<row_blocks, 256, 0, s>>>(ra, ColsArgs{}, row_blocks, 1);
    ++g_kernel_launches;
    return cudaGetLastError();
}

}  // namespace spdzb200
