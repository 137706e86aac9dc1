// F_p arithmetic for p = 2^32 - 5 (reference: proj/core/include/mpc/field.hpp:10-46)
// and the splitmix64 finaliser (proj/core/include/mpc/hash.hpp:21-26), as
// device inline functions.
//
// Reduction: p is a pseudo-Mersenne prime, 2^32 == 5 (mod p), so a 64-bit
// value v = hi*2^32 + lo folds to 5*hi + lo.  Two folds and one conditional
// subtract give v mod p for every u64 (proof in DESIGN.md §3).  A Barrett
// variant is kept for the ncu comparison the north star asks for
// (`-DSPDZ_REDUCE_BARRETT`); every variant is bit-exact with `v % p`.
#pragma once
#include <cstdint>

#ifndef __CUDACC__
#define __host__
#define __device__
#define __forceinline__ inline
#endif

namespace spdzb200 {

constexpr uint32_t kP = 4294967291u;
constexpr uint64_t kP64 = 4294967291ull;
constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ull;

// t < 6 * 2^32 after one fold of any u64
__host__ __device__ __forceinline__ uint64_t fold1(uint64_t v) {
    return (v & 0xffffffffull) + 5ull * (v >> 32);
}

#if defined(SPDZ_REDUCE_BARRETT)
// Barrett with mu = floor(2^64 / p): q = hi64(v * mu), r = v - q*p in [0, 2p).
__host__ __device__ __forceinline__ uint32_t fp_reduce64(uint64_t v) {
    constexpr uint64_t mu = 4294967301ull;  // floor(2^64 / (2^32 - 5)) = 2^32 + 5 (+0, remainder 25)
#ifdef __CUDA_ARCH__
    uint64_t q = __umul64hi(v, mu);
#else
    uint64_t q = (uint64_t)(((unsigned __int128)v * mu) >> 64);
#endif
    uint64_t r = v - q * kP64;
    while (r >= kP64) r -= kP64;
    return (uint32_t)r;
}
#else
// v mod p for any u64: fold, fold, conditional subtract.
__host__ __device__ __forceinline__ uint32_t fp_reduce64(uint64_t v) {
    uint64_t t = fold1(v);     // < 6 * 2^32
    t = fold1(t);              // < 2^32 + 25 < 2p
    return (uint32_t)(t >= kP64 ? t - kP64 : t);
}
#endif

// field.hpp:14 reduce() of a u32 (payload words from peers may be >= p)
__host__ __device__ __forceinline__ uint32_t fp_reduce32(uint32_t v) { return v >= kP ? v - kP : v; }

// field.hpp:16-20
__host__ __device__ __forceinline__ uint32_t fp_add(uint32_t a, uint32_t b) {
    uint32_t r = a + b;
    // a, b < p: a + b < 2p; carry out of 32 bits implies >= p.
    if (r < a || r >= kP) r -= kP;
    return r;
}

// field.hpp:22-24
__host__ __device__ __forceinline__ uint32_t fp_sub(uint32_t a, uint32_t b) {
    uint32_t r = a - b;
    if (a < b) r += kP;
    return r;
}

// field.hpp:26
__host__ __device__ __forceinline__ uint32_t fp_neg(uint32_t a) { return a == 0 ? 0u : kP - a; }

__host__ __device__ __forceinline__ uint64_t mul_wide(uint32_t a, uint32_t b) { return (uint64_t)a * b; }

// field.hpp:28-30
__host__ __device__ __forceinline__ uint32_t fp_mul(uint32_t a, uint32_t b) { return fp_reduce64(mul_wide(a, b)); }

// Lazy accumulation: acc += a*b folded once (< 6*2^32 per term), so 2^29 terms
// fit in a u64 before a final fp_reduce64.
__host__ __device__ __forceinline__ uint64_t mac_lazy(uint64_t acc, uint32_t a, uint32_t b) {
    return acc + fold1(mul_wide(a, b));
}

// hash.hpp:21-26 finaliser; splitmix64(state) = mix64(state += gamma)
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

// MAC-check coefficient of global record rank j (spdz.cpp:131-135):
// r_j = reduce(splitmix64 stream from coin, draw j) = reduce(mix(coin + (j+1) gamma)).
__host__ __device__ __forceinline__ uint32_t mac_coeff(uint64_t coin, uint64_t j) {
    return fp_reduce64(mix64(coin + (j + 1) * kGamma));
}

#ifdef __CUDACC__
// ---- MAC-check record arithmetic on 32-bit halves (kernels.cu k_mac_sigma) ----
// ~45 instructions per record, split between the ALU pipe (xor/funnel shifts,
// carry chains) and the fma-heavy pipe (multiplies, the h >> s halves of the
// xorshifts, the fold by 5); ncu source-level sampling showed the ALU pipe as
// the throttle when every shift and carry sat there.
struct Acc96 {
    uint32_t w0 = 0, w1 = 0, w2 = 0;
    __device__ __forceinline__ void add(uint64_t v) {
        asm("add.cc.u32 %0, %0, %3;\n\taddc.cc.u32 %1, %1, %4;\n\taddc.u32 %2, %2, 0;"
            : "+r"(w0), "+r"(w1), "+r"(w2)
            : "r"((uint32_t)v), "r"((uint32_t)(v >> 32)));
    }
    __device__ __forceinline__ uint32_t mod() const {  // (w2 2^64 + w1 2^32 + w0) mod p, < 2^38 before the fold
        return fp_reduce64((uint64_t)w0 + 5ull * w1 + 25ull * w2);
    }
};

// Small constants passed as kernel parameters so that ptxas cannot fold
// "h * 2^k" / "h * 5" into ALU shifts/LEAs: the multiplies then run on the
// fma-heavy pipe, which the ALU-bound MAC-check record math leaves idle.
struct SigConsts {
    uint32_t sh30 = 1u << 2, sh27 = 1u << 5, sh31 = 1u << 1, five = 5u;
};

// Which of the three xorshifts take their high-word shift on the ALU pipe (SHF) instead of the
// fma-heavy pipe (umulhi by 2^(32-s)): bit 0 = >> 30, bit 1 = >> 27, bit 2 = >> 31.  The split
// that balances the two pipes is measured (scripts/sigma_ceiling.py).
#ifndef SPDZ_SIGMA_ALU_SHIFTS
#define SPDZ_SIGMA_ALU_SHIFTS 0
#endif
// z ^= z >> s (s < 32); hm = 2^(32-s): h >> s = umulhi(h, hm) on the fma pipe, or a shift
template <bool kAlu>
__device__ __forceinline__ void xorshift_r(uint32_t& l, uint32_t& h, int s, uint32_t hm) {
    l ^= __funnelshift_r(l, h, s);
    h ^= kAlu ? (h >> s) : __umulhi(h, hm);
}
__device__ __forceinline__ void mul_const(uint32_t& l, uint32_t& h, uint32_t cl, uint32_t ch) {  // z *= c (mod 2^64)
    const uint32_t t1 = h * cl, t2 = l * ch, hw = __umulhi(l, cl);
    l = l * cl;
    h = hw + t1 + t2;
}
// r' < 2^32 with r' == (h 2^32 + l) (mod p); not necessarily canonical.
// s = l + 5h < 6 2^32; t = s_lo + 5 s_hi < 2^32 + 25; r' = t_lo + 5 t_hi (t_lo < 25 if t_hi).
__device__ __forceinline__ uint32_t rep_mod_p(uint32_t l, uint32_t h, uint32_t five) {
    const uint64_t s = (uint64_t)h * five + l;
    const uint64_t t = (uint64_t)(uint32_t)(s >> 32) * five + (uint32_t)s;
    return (uint32_t)(t >> 32) * five + (uint32_t)t;
}
// The single-party kernel (k_mac_sigma<1>, the one-party-per-GPU layout) takes the >> 30 and >> 31
// high-word shifts on the ALU: measured in the bench's per-party step, 4.36 -> 4.54 TB/s (bits 0+2;
// all three 4.52; none 4.36), while the co-located two-party kernel keeps all three on the fma
// pipe (profiles/r02zb)
#ifndef SPDZ_SIGMA1_ALU_SHIFTS
#define SPDZ_SIGMA1_ALU_SHIFTS 5
#endif
// r' < 2^32 with r' == mix64(h:l) (mod p)  (hash.hpp:21-26, reduce: field.hpp:14)
template <int ALU = SPDZ_SIGMA_ALU_SHIFTS>
__device__ __forceinline__ uint32_t mac_coeff_rep(uint32_t l, uint32_t h, const SigConsts& kc) {
    xorshift_r<(ALU & 1) != 0>(l, h, 30, kc.sh30);
    mul_const(l, h, 0x1ce4e5b9u, 0xbf58476du);
    xorshift_r<(ALU & 2) != 0>(l, h, 27, kc.sh27);
    mul_const(l, h, 0x133111ebu, 0x94d049bbu);
    xorshift_r<(ALU & 4) != 0>(l, h, 31, kc.sh31);
#ifdef SPDZ_SIGMA_ALU_FIVE
    return rep_mod_p(l, h, 5u);
#else
    return rep_mod_p(l, h, kc.five);
#endif
}
#endif  // __CUDACC__

}  // namespace spdzb200
