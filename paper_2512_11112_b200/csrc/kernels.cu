// sm_100a kernels of the B200 SPDZ online-phase back end.
//
// All hot-path kernels here are HBM-bound integer streams over structure-of-
// arrays share planes: 128-bit vector loads/stores when every
// plane of a call is 16-byte aligned (scalar, still coalesced, otherwise), a
// grid of (148 SMs x 8) 256-thread CTAs striding over the lanes, and modular
// arithmetic by the pseudo-Mersenne fold of field.cuh.  The one dense
// contraction (secret x public linear layer) is a CUDA-core modular GEMM.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "async.cuh"
#include "field.cuh"
#include "kernels.cuh"

namespace spdzb200 {

std::atomic<unsigned long long> g_kernel_launches{0};

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ uint4 ld4(const uint32_t* p, uint64_t g) {
    return __ldcs(reinterpret_cast<const uint4*>(p) + g);
}
__device__ __forceinline__ uint4 ld4_peer(const uint32_t* p, uint64_t g) {
    // peer payloads may live on another GPU (NVLink P2P / IPC): plain load
    return reinterpret_cast<const uint4*>(p)[g];
}
__device__ __forceinline__ void st4(uint32_t* p, uint64_t g, const uint32_t (&v)[4]) {
    reinterpret_cast<uint4*>(p)[g] = make_uint4(v[0], v[1], v[2], v[3]);
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

inline int grid_for(uint64_t work, int sms, int per_sm = 8) {
    uint64_t b = (work + kThreads - 1) / kThreads;
    uint64_t cap = (uint64_t)sms * per_sm;
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return (int)b;
}

inline cudaError_t launched() {
    ++g_kernel_launches;
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Generic lane-parallel map: NI input planes -> NO output planes, `op` applied
// per lane.  Peer planes (NPI of the inputs, starting at PEER0) use plain loads.
// ---------------------------------------------------------------------------
template <int NI, int NO>
struct IO {
    const uint32_t* in[NI > 0 ? NI : 1];
    uint32_t* out[NO];
};

template <int NI, int NO, class Op>
__device__ __forceinline__ void map_group(const IO<NI, NO>& io, uint64_t g, const Op& op, uint32_t (&a)[NI > 0 ? NI : 1][4]) {
    uint32_t o[NO][4];
#pragma unroll
    for (int l = 0; l < 4; ++l) {
        uint32_t ai[NI > 0 ? NI : 1], oi[NO];
#pragma unroll
        for (int k = 0; k < NI; ++k) ai[k] = a[k][l];
        op(ai, oi);
#pragma unroll
        for (int k = 0; k < NO; ++k) o[k][l] = oi[k];
    }
#pragma unroll
    for (int k = 0; k < NO; ++k) st4(io.out[k], g, o[k]);
}

template <int NI, int NO, class Op>
__device__ __forceinline__ void map_load(const IO<NI, NO>& io, uint64_t g, uint32_t (&a)[NI > 0 ? NI : 1][4]) {
#pragma unroll
    for (int k = 0; k < NI; ++k) {
        uint4 v = Op::is_peer(k) ? ld4_peer(io.in[k], g) : ld4(io.in[k], g);
        a[k][0] = v.x;
        a[k][1] = v.y;
        a[k][2] = v.z;
        a[k][3] = v.w;
    }
}

// Ops with few planes (mask, add) keep two 4-lane groups in flight per thread.
template <class Op>
struct MapUnroll {
    static constexpr int value = 1;
};

template <int NI, int NO, class Op>
__global__ void __launch_bounds__(kThreads) k_map(IO<NI, NO> io, uint64_t n, uint64_t n4, Op op_param) {
    Op op = op_param;
    op.prepare();  // e.g. alpha from device memory
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint64_t g = t;
    if (MapUnroll<Op>::value == 2) {
        for (; g + stride < n4; g += 2 * stride) {
            uint32_t a[NI > 0 ? NI : 1][4], b[NI > 0 ? NI : 1][4];
            map_load<NI, NO, Op>(io, g, a);
            map_load<NI, NO, Op>(io, g + stride, b);
            map_group<NI, NO, Op>(io, g, op, a);
            map_group<NI, NO, Op>(io, g + stride, op, b);
        }
    }
    for (; g < n4; g += stride) {
        uint32_t a[NI > 0 ? NI : 1][4];
        map_load<NI, NO, Op>(io, g, a);
        map_group<NI, NO, Op>(io, g, op, a);
    }
    for (uint64_t i = n4 * 4 + t; i < n; i += stride) {
        uint32_t ai[NI > 0 ? NI : 1], oi[NO];
#pragma unroll
        for (int k = 0; k < NI; ++k) ai[k] = io.in[k][i];
        op(ai, oi);
#pragma unroll
        for (int k = 0; k < NO; ++k) io.out[k][i] = oi[k];
    }
}

template <int NI, int NO, class Op>
cudaError_t run_map(cudaStream_t s, const IO<NI, NO>& io, uint64_t n, Op op, int sms) {
    if (n == 0) return cudaSuccess;
    bool al = true;
    for (int k = 0; k < NI; ++k) al = al && aligned16(io.in[k]);
    for (int k = 0; k < NO; ++k) al = al && aligned16(io.out[k]);
    const uint64_t n4 = al ? n / 4 : 0;
    const uint64_t work = n4 ? n4 : n;
    k_map<NI, NO, Op><<<grid_for(work, sms), kThreads, 0, s>>>(io, n, n4, op);
    return launched();
}

// ---- ops ----
struct NoPeer {
    __device__ static constexpr bool is_peer(int) { return false; }
    __device__ void prepare() {}
};
// alpha given by value, or (ap != null) read once per thread from device memory
struct AlphaArg {
    uint32_t alpha;
    const uint32_t* ap;
    __device__ void prepare() {
        if (ap) alpha = __ldg(ap);
    }
};

struct OpAdd : NoPeer {  // backend.cpp:25-37
    __device__ void operator()(const uint32_t* a, uint32_t* o) const {
        o[0] = fp_add(a[0], a[2]);
        o[1] = fp_add(a[1], a[3]);
    }
};
struct OpSub : NoPeer {  // backend.cpp:39-51
    __device__ void operator()(const uint32_t* a, uint32_t* o) const {
        o[0] = fp_sub(a[0], a[2]);
        o[1] = fp_sub(a[1], a[3]);
    }
};

// Both co-located parties' add / sub in one pass: x0.v x0.m y0.v y0.m x1.v x1.m y1.v y1.m -> z0.v z0.m
// z1.v z1.m (the same bytes as two OpAdd launches, one launch)
template <bool SUB>
struct OpAddSub2 : NoPeer {
    __device__ void operator()(const uint32_t* a, uint32_t* o) const {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t x = a[k < 2 ? k : k + 2], y = a[k < 2 ? k + 2 : k + 4];
            o[k] = SUB ? fp_sub(x, y) : fp_add(x, y);
        }
    }
};

// OpAddSub2 followed by the add / sub that consumes its result (SM2: 0 w2 = w + o, 1 w - o, 2 o - w)
// and, with ROOT, the root opening of w2.  Inputs: OpAddSub2's 8, o0.v o0.m o1.v o1.m.  Outputs: w0.v
// w0.m w1.v w1.m, w2 of both parties (4), [both parties' opened outputs].
template <bool SUB, int SM2, bool ROOT>
struct OpAddSub2X : NoPeer {
    __device__ void operator()(const uint32_t* a, uint32_t* o) const {
        OpAddSub2<SUB>{}(a, o);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t w = o[k], q = a[8 + k];
            o[4 + k] = SM2 == 0 ? fp_add(w, q) : SM2 == 1 ? fp_sub(w, q) : fp_sub(q, w);
        }
        if constexpr (ROOT) {
            o[8] = fp_add(o[4], fp_reduce32(o[6]));
            o[9] = fp_add(o[6], fp_reduce32(o[4]));
        }
    }
};

// spdz.cpp:35-75; inputs: xv, xm[, k].  KM: 0 vector k, 1 device scalar
// broadcast (runtime.cpp:36-39), 2 immediate.
template <int OPC, int KM>
struct OpPublic : AlphaArg {
    __device__ static constexpr bool is_peer(int) { return false; }
    int party;
    uint32_t kk;
    const uint32_t* kp;
    __device__ void operator()(const uint32_t* a, uint32_t* o) const {
        const uint32_t k = KM == 0 ? a[2] : (KM == 1 ? __ldg(kp) : kk);
        const uint32_t xv = a[0], xm = a[1];
        if (OPC == 0) {  // add_public
            o[0] = party == 0 ? fp_add(xv, k) : xv;
            o[1] = fp_add(xm, fp_mul(alpha, k));
        } else if (OPC == 1) {  // sub_public
            o[0] = party == 0 ? fp_sub(xv, k) : xv;
            o[1] = fp_sub(xm, fp_mul(alpha, k));
        } else if (OPC == 2) {  // rsub_public
            o[0] = party == 0 ? fp_sub(k, xv) : fp_neg(xv);
            o[1] = fp_sub(fp_mul(alpha, k), xm);
        } else {  // mul_public
            o[0] = fp_mul(xv, k);
            o[1] = fp_mul(xm, k);
        }
    }
};
// spdz.cpp:70-75 share_of_public; input: [k] (KM as OpPublic)
template <int KM>
struct OpShareOfPublic : AlphaArg {
    __device__ static constexpr bool is_peer(int) { return false; }
    int party;
    uint32_t kk;
    const uint32_t* kp;
    __device__ void operator()(const uint32_t* a, uint32_t* o) const {
        const uint32_t k = KM == 0 ? a[0] : (KM == 1 ? __ldg(kp) : kk);
        o[0] = party == 0 ? k : 0u;
        o[1] = fp_mul(alpha, k);
    }
};

struct OpMask : NoPeer {  // backend.cpp:53-65: in xv yv av bv -> d e
    __device__ void operator()(const uint32_t* a, uint32_t* o) const {
        o[0] = fp_sub(a[0], a[2]);
        o[1] = fp_sub(a[1], a[3]);
    }
};

struct OpMask2 : NoPeer {  // both co-located parties: x0 y0 a0 b0 x1 y1 a1 b1 -> d0 e0 d1 e1
    __device__ void operator()(const uint32_t* a, uint32_t* o) const {
        o[0] = fp_sub(a[0], a[2]);
        o[1] = fp_sub(a[1], a[3]);
        o[2] = fp_sub(a[4], a[6]);
        o[3] = fp_sub(a[5], a[7]);
    }
};

// Fused open + Beaver combine.  Inputs: own_d, own_e, peer_d[NP], peer_e[NP],
// a.v a.m b.v b.m c.v c.m.  Outputs: z.v z.m [open_d open_e].
template <int NP, bool LOG>
struct OpCombine : AlphaArg {
    int party;
    __device__ static constexpr bool is_peer(int k) { return k >= 2 && k < 2 + 2 * NP; }
    __device__ void operator()(const uint32_t* in, uint32_t* o) const {
        uint32_t d = in[0], e = in[1];
#pragma unroll
        for (int p = 0; p < NP; ++p) {  // net.cpp:188-189: acc = add(acc, reduce(peer))
            d = fp_add(d, fp_reduce32(in[2 + p]));
            e = fp_add(e, fp_reduce32(in[2 + NP + p]));
        }
        const uint32_t* t = in + 2 + 2 * NP;  // a.v a.m b.v b.m c.v c.m
        // spdz.cpp:83-93, lazily reduced (exact mod p)
        const uint32_t de = fp_mul(d, e);
        uint64_t v = (uint64_t)t[4] + fold1(mul_wide(d, t[2])) + fold1(mul_wide(e, t[0]));
        if (party == 0) v += de;
        uint64_t m = (uint64_t)t[5] + fold1(mul_wide(d, t[3])) + fold1(mul_wide(e, t[1])) +
                     fold1(mul_wide(alpha, de));
        o[0] = fp_reduce64(v);
        o[1] = fp_reduce64(m);
        if (LOG) {
            o[2] = d;
            o[3] = e;
        }
    }
};

// Both parties of a 2-party run in one pass (same GPU): the opened d, e are computed once
// from the two payloads (each read once) and logged once; each party's triple shares give
// its z exactly as OpCombine (spdz.cpp:83-93).  Inputs: d0 e0 d1 e1, party 0's a.v a.m
// b.v b.m c.v c.m, party 1's six planes.  Outputs: z0.v z0.m z1.v z1.m, opened d, e.
// (Payload words are < p here — fault-injected runs take the per-party path — so
// d0 + reduce(d1) == d1 + reduce(d0): one opened value serves both parties.)
struct OpCombine2 {
    uint32_t alpha0, alpha1;
    const uint32_t *ap0, *ap1;
    __device__ static constexpr bool is_peer(int) { return false; }
    __device__ void prepare() {
        if (ap0) alpha0 = __ldg(ap0);
        if (ap1) alpha1 = __ldg(ap1);
    }
    __device__ void operator()(const uint32_t* in, uint32_t* o) const {
        const uint32_t d = fp_add(in[0], fp_reduce32(in[2]));  // net.cpp:188-189
        const uint32_t e = fp_add(in[1], fp_reduce32(in[3]));
        const uint32_t de = fp_mul(d, e);
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            const uint32_t* t = in + 4 + 6 * p;  // a.v a.m b.v b.m c.v c.m of party p
            uint64_t v = (uint64_t)t[4] + fold1(mul_wide(d, t[2])) + fold1(mul_wide(e, t[0]));
            if (p == 0) v += de;
            const uint64_t m = (uint64_t)t[5] + fold1(mul_wide(d, t[3])) + fold1(mul_wide(e, t[1])) +
                               fold1(mul_wide(p == 0 ? alpha0 : alpha1, de));
            o[2 * p] = fp_reduce64(v);
            o[2 * p + 1] = fp_reduce64(m);
        }
        o[4] = d;
        o[5] = e;
    }
};

// OpCombine2 followed, in the same pass, by the next multiply's mask (OpMask2) when that multiply
// consumes this one's product: the fresh z.v of each party is masked from registers instead of
// being re-read by a separate mask launch (runtime.cpp:209-217 for the next node).  ZPOS: which of
// the next multiply's operands is this product (0 = left x, 1 = right y, 2 = both).  Inputs: the 16
// of OpCombine2, then per party [other operand .v (ZPOS < 2)], a'.v, b'.v.  Outputs: the 6 of
// OpCombine2, then d'0 e'0 d'1 e'1.
// ZPOS 3: this product is the circuit's root — its opening (both parties' words, z0 + z1,
// net.cpp:170-215) is written instead (no extra inputs; outputs: the 6 of OpCombine2, then both
// parties' opened outputs).
template <int ZPOS>
struct OpCombine2M : OpCombine2 {
    static constexpr int kPer = ZPOS == 3 ? 0 : (ZPOS == 2 ? 2 : 3);  // extra inputs per party
    __device__ void operator()(const uint32_t* in, uint32_t* o) const {
        OpCombine2::operator()(in, o);
        if constexpr (ZPOS == 3) {
            o[6] = fp_add(o[0], fp_reduce32(o[2]));
            o[7] = fp_add(o[2], fp_reduce32(o[0]));
        } else {
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                const uint32_t* q = in + 16 + kPer * p;
                const uint32_t z = o[2 * p];
                const uint32_t x = ZPOS == 1 ? q[0] : z, y = ZPOS == 0 ? q[0] : z;
                const uint32_t* ab = q + (ZPOS == 2 ? 0 : 1);
                o[6 + 2 * p] = fp_sub(x, ab[0]);
                o[7 + 2 * p] = fp_sub(y, ab[1]);
            }
        }
    }
};
// (one 4-lane group per iteration: two in flight, as OpCombine2 does, measured 12% slower with the
// 22 operand streams; profiles/r02u)

// Input sharing of one private input for both parties of a 2-party run on one GPU
// (preproc.cpp:205-243 with spdz::add_public, spdz.cpp:35-45): x = reduce(raw input),
// diff = x - r (opened by party 0), party 0: (mask.v + diff, mask.m + alpha_0 diff),
// party 1: (mask.v, mask.m + alpha_1 diff).  Inputs: raw x, r (clear mask), party 0's
// mask.v mask.m, party 1's.  Outputs: v0 m0 v1 m1.
struct OpShareInput2 {
    uint32_t alpha0, alpha1;
    const uint32_t *ap0, *ap1;
    __device__ static constexpr bool is_peer(int) { return false; }
    __device__ void prepare() {
        if (ap0) alpha0 = __ldg(ap0);
        if (ap1) alpha1 = __ldg(ap1);
    }
    __device__ void operator()(const uint32_t* in, uint32_t* o) const {
        const uint32_t diff = fp_sub(fp_reduce32(in[0]), in[1]);
        o[0] = fp_add(in[2], diff);
        o[1] = fp_add(in[3], fp_mul(alpha0, diff));
        o[2] = in[4];
        o[3] = fp_add(in[5], fp_mul(alpha1, diff));
    }
};

template <>
struct MapUnroll<OpMask> {
    static constexpr int value = 2;
};
template <>  // two lane groups in flight: 92% -> 95% of HBM in the heavy-chain step (no spills)
struct MapUnroll<OpCombine2> {
    static constexpr int value = 2;
};
template <>
struct MapUnroll<OpAdd> {
    static constexpr int value = 2;
};
template <>
struct MapUnroll<OpSub> {
    static constexpr int value = 2;
};

struct OpDiff : NoPeer {
    __device__ void operator()(const uint32_t* a, uint32_t* o) const { o[0] = fp_sub(a[0], a[1]); }
};

template <int NP>
struct OpOpen {  // net.cpp:170-215
    __device__ static constexpr bool is_peer(int k) { return k >= 1; }
    __device__ void prepare() {}
    __device__ void operator()(const uint32_t* in, uint32_t* o) const {
        uint32_t acc = in[0];
#pragma unroll
        for (int p = 0; p < NP; ++p) acc = fp_add(acc, fp_reduce32(in[1 + p]));
        o[0] = acc;
    }
};

// Root open of two co-located parties: both parties' opened words (identical: z0 + z1) in one
// pass, 8 bytes read and 8 written per lane instead of two OpOpen<1> launches reading 16.
struct OpOpen2 {
    __device__ static constexpr bool is_peer(int k) { return false; }
    __device__ void prepare() {}
    __device__ void operator()(const uint32_t* in, uint32_t* o) const {
        o[0] = fp_add(in[0], fp_reduce32(in[1]));
        o[1] = fp_add(in[1], fp_reduce32(in[0]));
    }
};

template <int NP>
cudaError_t combine_np(cudaStream_t s, const uint32_t* od, const uint32_t* oe, const uint32_t* const* pd,
                       const uint32_t* const* pe, const uint32_t* const tri[6], int party, uint32_t alpha,
                       uint32_t* zv, uint32_t* zm, uint32_t* open_d, uint32_t* open_e, uint64_t n, int sms,
                       const uint32_t* alpha_dev) {
    constexpr int NI = 8 + 2 * NP;
    if (open_d) {
        IO<NI, 4> io;
        io.in[0] = od;
        io.in[1] = oe;
        for (int p = 0; p < NP; ++p) {
            io.in[2 + p] = pd[p];
            io.in[2 + NP + p] = pe[p];
        }
        for (int k = 0; k < 6; ++k) io.in[2 + 2 * NP + k] = tri[k];
        io.out[0] = zv;
        io.out[1] = zm;
        io.out[2] = open_d;
        io.out[3] = open_e;
        return run_map(s, io, n, OpCombine<NP, true>{{alpha, alpha_dev}, party}, sms);
    }
    IO<NI, 2> io;
    io.in[0] = od;
    io.in[1] = oe;
    for (int p = 0; p < NP; ++p) {
        io.in[2 + p] = pd[p];
        io.in[2 + NP + p] = pe[p];
    }
    for (int k = 0; k < 6; ++k) io.in[2 + 2 * NP + k] = tri[k];
    io.out[0] = zv;
    io.out[1] = zm;
    return run_map(s, io, n, OpCombine<NP, false>{{alpha, alpha_dev}, party}, sms);
}

// One party's fused open + combine followed by the next multiply's mask from the fresh product
// (the co-located OpCombine2M, per party: the N-GPU ranks' kernel mix).  Inputs: OpCombine<NP>'s,
// then [the next multiply's other operand .v (ZPOS < 2)], a'.v, b'.v.  Outputs: z.v z.m open_d
// open_e d' e'.
template <int NP, int ZPOS>
struct OpCombineM : OpCombine<NP, true> {
    static constexpr int kX = ZPOS == 2 ? 2 : 3;
    __device__ void operator()(const uint32_t* in, uint32_t* o) const {
        OpCombine<NP, true>::operator()(in, o);
        const uint32_t* q = in + 8 + 2 * NP;
        const uint32_t z = o[0];
        const uint32_t x = ZPOS == 1 ? q[0] : z, y = ZPOS == 0 ? q[0] : z;
        const uint32_t* ab = q + (ZPOS == 2 ? 0 : 1);
        o[4] = fp_sub(x, ab[0]);
        o[5] = fp_sub(y, ab[1]);
    }
};

template <int NP, int ZPOS>
cudaError_t combine_m_np(cudaStream_t s, const uint32_t* od, const uint32_t* oe, const uint32_t* const* pd,
                         const uint32_t* const* pe, const uint32_t* const tri[6], int party, uint32_t alpha,
                         uint32_t* zv, uint32_t* zm, uint32_t* open_d, uint32_t* open_e, const uint32_t* const next[3],
                         uint32_t* const next_de[2], uint64_t n, int sms, const uint32_t* alpha_dev) {
    constexpr int K = OpCombineM<NP, ZPOS>::kX;
    IO<8 + 2 * NP + K, 6> io;
    io.in[0] = od;
    io.in[1] = oe;
    for (int p = 0; p < NP; ++p) {
        io.in[2 + p] = pd[p];
        io.in[2 + NP + p] = pe[p];
    }
    for (int k = 0; k < 6; ++k) io.in[2 + 2 * NP + k] = tri[k];
    int k = 8 + 2 * NP;
    if (ZPOS != 2) io.in[k++] = next[0];
    io.in[k++] = next[1];
    io.in[k] = next[2];
    io.out[0] = zv;
    io.out[1] = zm;
    io.out[2] = open_d;
    io.out[3] = open_e;
    io.out[4] = next_de[0];
    io.out[5] = next_de[1];
    OpCombineM<NP, ZPOS> op;
    op.alpha = alpha;
    op.ap = alpha_dev;
    op.party = party;
    return run_map(s, io, n, op, sms);
}

// One party (one peer) of a 2-party run: OpCombine<1> followed by the private add / sub that
// consumes the product (SM as OpCombine2A) and optionally the mask of the multiply consuming its
// result (NX 1 w left, 2 w right, 3 both).  Inputs: OpCombine<1>'s 10, o.v o.m, [other .v (NX 1, 2)],
// a'.v, b'.v (NX > 0).  Outputs: z.v z.m open_d open_e w.v w.m [d' e'].
template <int SM, int NX>
struct OpCombineA : OpCombine<1, true> {
    static constexpr int kX = 2 + (NX == 0 ? 0 : NX == 3 ? 2 : 3);
    static constexpr int kOut = NX == 0 ? 6 : 8;
    __device__ void operator()(const uint32_t* in, uint32_t* o) const {
        OpCombine<1, true>::operator()(in, o);
        const uint32_t* q = in + 10;
        const uint32_t zv = o[0], zm = o[1];
        const uint32_t wv = SM == 0 ? fp_add(zv, q[0]) : SM == 1 ? fp_sub(zv, q[0]) : fp_sub(q[0], zv);
        const uint32_t wm = SM == 0 ? fp_add(zm, q[1]) : SM == 1 ? fp_sub(zm, q[1]) : fp_sub(q[1], zm);
        o[4] = wv;
        o[5] = wm;
        if constexpr (NX > 0) {
            const uint32_t* r = q + 2;
            const uint32_t x = NX == 2 ? r[0] : wv, y = NX == 1 ? r[0] : wv;
            const uint32_t* ab = r + (NX == 3 ? 0 : 1);
            o[6] = fp_sub(x, ab[0]);
            o[7] = fp_sub(y, ab[1]);
        }
    }
};

template <int SM, int NX>
cudaError_t combine_a(cudaStream_t s, const uint32_t* const in10[10], const uint32_t* const addin[2],
                      const uint32_t* const next[3], uint32_t* const out4[4], uint32_t* const w[2],
                      uint32_t* const next_de[2], int party, uint32_t alpha, const uint32_t* alpha_dev, uint64_t n,
                      int sms) {
    using Op = OpCombineA<SM, NX>;
    IO<10 + Op::kX, Op::kOut> io;
    for (int k = 0; k < 10; ++k) io.in[k] = in10[k];
    int k = 10;
    io.in[k++] = addin[0];
    io.in[k++] = addin[1];
    if constexpr (NX > 0) {
        if (NX != 3) io.in[k++] = next[0];
        io.in[k++] = next[1];
        io.in[k] = next[2];
    }
    for (int j = 0; j < 4; ++j) io.out[j] = out4[j];
    io.out[4] = w[0];
    io.out[5] = w[1];
    if constexpr (NX > 0) {
        io.out[6] = next_de[0];
        io.out[7] = next_de[1];
    }
    Op op;
    op.alpha = alpha;
    op.ap = alpha_dev;
    op.party = party;
    return run_map(s, io, n, op, sms);
}

template <int NP>
cudaError_t open_np(cudaStream_t s, const uint32_t* own, const uint32_t* const* peers, uint32_t* out, uint64_t n,
                    int sms) {
    IO<1 + NP, 1> io;
    io.in[0] = own;
    for (int p = 0; p < NP; ++p) io.in[1 + p] = peers[p];
    io.out[0] = out;
    return run_map(s, io, n, OpOpen<NP>{}, sms);
}

// ---------------------------------------------------------------------------
// Reductions
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block sum of NV u64 values; result valid in thread 0.
template <int NV>
__device__ __forceinline__ void block_sum(unsigned long long (&v)[NV]) {
    __shared__ unsigned long long sh[NV][kThreads / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) sh[k][w] = v[k];
    }
    __syncthreads();
    if (w == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            unsigned long long x = lane < (int)(blockDim.x >> 5) ? sh[k][lane] : 0ull;
            v[k] = warp_sum(x);
        }
    }
    __syncthreads();
}

// backend.cpp:76-84.  Per-thread u64 sums of u32 lanes (<= 2^32 terms safe),
// block tree, fold to < p, one atomic per block.
__global__ void __launch_bounds__(kThreads) k_reduce_add(const uint32_t* __restrict__ xv,
                                                         const uint32_t* __restrict__ xm, uint64_t n,
                                                         unsigned long long* acc) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    unsigned long long s[2] = {0ull, 0ull};
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        s[0] += __ldcs(xv + i);
        s[1] += __ldcs(xm + i);
    }
    s[0] = fp_reduce64(s[0]);
    s[1] = fp_reduce64(s[1]);
    block_sum<2>(s);
    if (threadIdx.x == 0) {
        atomicAdd(acc, (unsigned long long)fp_reduce64(s[0]));
        atomicAdd(acc + 1, (unsigned long long)fp_reduce64(s[1]));
    }
}

__global__ void k_finish_reduce(const unsigned long long* acc, uint32_t* outv, uint32_t* outm) {
    if (threadIdx.x == 0) {
        outv[0] = fp_reduce64(acc[0]);
        outm[0] = fp_reduce64(acc[1]);
    }
}

__global__ void __launch_bounds__(kThreads) k_pair_split(const uint32_t* __restrict__ cv,
                                                         const uint32_t* __restrict__ cm, uint64_t pairs,
                                                         uint32_t* xv, uint32_t* xm, uint32_t* yv, uint32_t* ym) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    // a load at a constant odd offset is a zero-copy view (run_plan.cu), so the
    // pair view is 8-byte aligned only sometimes: the 64-bit path needs both planes aligned
    const bool wide = ((reinterpret_cast<uintptr_t>(cv) | reinterpret_cast<uintptr_t>(cm)) & 7) == 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < pairs; i += stride) {
        uint2 v, m;
        if (wide) {
            v = reinterpret_cast<const uint2*>(cv)[i];
            m = reinterpret_cast<const uint2*>(cm)[i];
        } else {
            v = make_uint2(cv[2 * i], cv[2 * i + 1]);
            m = make_uint2(cm[2 * i], cm[2 * i + 1]);
        }
        xv[i] = v.x;
        yv[i] = v.y;
        xm[i] = m.x;
        ym[i] = m.y;
    }
}

// MAC sigma (spdz.cpp:126-138) in closed form: record of rank j contributes
// r_j * (m_j - alpha x_j), r_j = reduce(mix(coin + (j+1) gamma)).  Order-free, so
// sigma = S_m - alpha * S_x with S_m = sum r_j m_j and S_x = sum r_j x_j (one
// alpha-multiply per thread instead of per record).
//
// The kernel is issue-bound on the fma-heavy pipe (every IMAD variant runs there;
// ncu r01c: fmaheavy 76%, alu 63%, dram 59%), so the per-record arithmetic is
// written on 32-bit halves to keep the IMAD count at the floor (two 64x64-bit
// multiplies by constants = 2 IMAD.WIDE + 4 IMAD, two r*m products = 2 IMAD.WIDE)
// and every add, carry and shift on the ALU pipe:
//  * r' = any representative of mix mod p below 2^32 (not the canonical one):
//    s = lo + 5 hi (< 6 2^32, 2^32 == 5) by shift/add-with-carry, then
//    t = s_lo + 5 s_hi, plus 5 on the (rare) carry out of 32 bits;
//  * S_m, S_x are exact 96-bit sums (add.cc chains); reduced once per thread
//    (2^64 == 25, 2^32 == 5 mod p).
__device__ __forceinline__ void z_step(uint32_t& zl, uint32_t& zh) {  // z += gamma
    asm("add.cc.u32 %0, %0, 0x7f4a7c15;\n\taddc.u32 %1, %1, 0x9e3779b9;" : "+r"(zl), "+r"(zh));
}
__device__ __forceinline__ void sigma_rec(uint32_t zl, uint32_t zh, uint32_t x, uint32_t m, Acc96& sm, Acc96& sx,
                                          const SigConsts& kc) {
    const uint32_t r = mac_coeff_rep<SPDZ_SIGMA1_ALU_SHIFTS>(zl, zh, kc);  // (single-party kernel only)
    sm.add(mul_wide(r, m));
    sx.add(mul_wide(r, x));
}
// four consecutive records starting at state z
__device__ __forceinline__ void sigma_rec4(uint64_t z, const uint4& x, const uint4& m, Acc96& sm, Acc96& sx,
                                           const SigConsts& kc) {
    uint32_t zl = (uint32_t)z, zh = (uint32_t)(z >> 32);
    sigma_rec(zl, zh, x.x, m.x, sm, sx, kc);
    z_step(zl, zh);
    sigma_rec(zl, zh, x.y, m.y, sm, sx, kc);
    z_step(zl, zh);
    sigma_rec(zl, zh, x.z, m.z, sm, sx, kc);
    z_step(zl, zh);
    sigma_rec(zl, zh, x.w, m.w, sm, sx, kc);
}
template <int NP>
struct SigmaOut {
    uint32_t alpha[NP];
    unsigned long long* acc[NP];
};

__device__ __forceinline__ uint4 sub4(const uint4& a, const uint4& b) {
    return make_uint4(fp_sub(a.x, b.x), fp_sub(a.y, b.y), fp_sub(a.z, b.z), fp_sub(a.w, b.w));
}

// Segment table passed by value (no host->device copy, no host sync before the
// launch).  The concatenated record space [0, rec0[n]) is split into one
// contiguous range per CTA (boundaries at multiples of kSigmaAlign records), so
// every CTA does the same work (no tail wave) and walks at most a few segment
// pieces.
//
// Compute-bound, not memory-bound (ncu r01d: the same kernel on L2-resident
// records runs no faster than on HBM; a TMA-staged variant was slower), so the
// block count is the occupancy limit (one wave) and loads are plain 128-bit.
#ifndef SPDZ_SIGMA2_MINB
#define SPDZ_SIGMA2_MINB 3
#endif
#ifndef SPDZ_SIGMA_MINB
#define SPDZ_SIGMA_MINB 4
#endif
template <int NP>
struct SigmaMinBlocks {
    static constexpr int value = NP == 1 ? SPDZ_SIGMA_MINB : SPDZ_SIGMA2_MINB;
};

// NP parties (NP = 1: one party's log; NP = 2: both local parties of a 2-party run,
// whose logs have the same record ranks) — r_j is computed once per record and
// applied to every party's (x_j, m_j), so the 2-party pass costs ~60% of two passes.
template <int NP>
__global__ void __launch_bounds__(kThreads, SigmaMinBlocks<NP>::value)
    k_mac_sigma(MacTableT<NP> tab, uint64_t coin, SigmaOut<NP> so, SigConsts kc) {
    Acc96 sm[NP], sx[NP];
    const uint64_t total = tab.rec0[tab.n];
    const uint64_t units = (total + kSigmaAlign - 1) / kSigmaAlign;
    const uint64_t lo_u = units * blockIdx.x / gridDim.x, hi_u = units * (blockIdx.x + 1) / gridDim.x;
    const uint64_t lo = lo_u * kSigmaAlign, hi = hi_u * kSigmaAlign < total ? hi_u * kSigmaAlign : total;
    uint32_t seg = 0;
    while (seg < tab.n && tab.rec0[seg + 1] <= lo) ++seg;
    for (uint64_t pos = lo; pos < hi && seg < tab.n; ++seg) {
        const MacSegT<NP>& sg = tab.seg[seg];
        const uint64_t s0 = tab.rec0[seg], s1 = tab.rec0[seg + 1] < hi ? tab.rec0[seg + 1] : hi;
        if (s1 <= pos) continue;
        const uint64_t start = pos - s0;
        const uint32_t count = (uint32_t)(s1 - pos);  // < 2^31 (launcher)
        pos = s1;
        const uint32_t *xv[NP], *ma[NP], *mb[NP];
        uintptr_t al = 0;
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            xv[p] = sg.value[p] + start;
            ma[p] = sg.mac_a[p] + start;
            mb[p] = sg.mac_b[p] ? sg.mac_b[p] + start : nullptr;
            al |= reinterpret_cast<uintptr_t>(xv[p]) | reinterpret_cast<uintptr_t>(ma[p]) |
                  reinterpret_cast<uintptr_t>(mb[p]);
        }
        const bool has_b = mb[0] != nullptr;
        const uint64_t z0 = coin + (sg.j0 + start + 1) * kGamma;  // z of record 0 of the piece
        uint32_t done = 0;
        if ((al & 15u) == 0) {
            const uint32_t n4 = count / 4;
            uint32_t g = threadIdx.x;
            if (NP == 1) {
                const uint4* x4 = reinterpret_cast<const uint4*>(xv[0]);
                const uint4* a4 = reinterpret_cast<const uint4*>(ma[0]);
                const uint4* b4 = reinterpret_cast<const uint4*>(mb[0]);
                for (; g + blockDim.x < n4; g += 2 * blockDim.x) {  // 8 records in flight per thread
                    const uint32_t g2 = g + blockDim.x;
                    const uint4 x1 = __ldcs(x4 + g), x2 = __ldcs(x4 + g2);
                    uint4 m1 = __ldcs(a4 + g), m2 = __ldcs(a4 + g2);
                    if (has_b) {
                        m1 = sub4(m1, __ldcs(b4 + g));
                        m2 = sub4(m2, __ldcs(b4 + g2));
                    }
                    sigma_rec4(z0 + (uint64_t)(4 * g) * kGamma, x1, m1, sm[0], sx[0], kc);
                    sigma_rec4(z0 + (uint64_t)(4 * g2) * kGamma, x2, m2, sm[0], sx[0], kc);
                }
            }
            for (; g < n4; g += blockDim.x) {
                uint4 x[NP], m[NP];
#pragma unroll
                for (int p = 0; p < NP; ++p) {
                    // a log shared by both parties is simply read twice (the second read hits in
                    // L1/L2; selecting the first party's registers instead measured 30% slower)
                    x[p] = __ldcs(reinterpret_cast<const uint4*>(xv[p]) + g);
                    m[p] = __ldcs(reinterpret_cast<const uint4*>(ma[p]) + g);
                    if (has_b) m[p] = sub4(m[p], __ldcs(reinterpret_cast<const uint4*>(mb[p]) + g));
                }
                const uint64_t z = z0 + (uint64_t)(4 * g) * kGamma;
                uint32_t zl = (uint32_t)z, zh = (uint32_t)(z >> 32);
#pragma unroll
                for (int l = 0; l < 4; ++l) {
                    const uint32_t r = mac_coeff_rep<NP == 1 ? SPDZ_SIGMA1_ALU_SHIFTS : SPDZ_SIGMA_ALU_SHIFTS>(zl, zh, kc);
#pragma unroll
                    for (int p = 0; p < NP; ++p) {
                        const uint32_t xl = l == 0 ? x[p].x : l == 1 ? x[p].y : l == 2 ? x[p].z : x[p].w;
                        const uint32_t ml = l == 0 ? m[p].x : l == 1 ? m[p].y : l == 2 ? m[p].z : m[p].w;
                        sm[p].add(mul_wide(r, ml));
                        sx[p].add(mul_wide(r, xl));
                    }
                    z_step(zl, zh);
                }
            }
            done = n4 * 4;
        }
        for (uint32_t i = done + threadIdx.x; i < count; i += blockDim.x) {
            const uint64_t z = z0 + (uint64_t)i * kGamma;
            const uint32_t r = mac_coeff_rep<NP == 1 ? SPDZ_SIGMA1_ALU_SHIFTS : SPDZ_SIGMA_ALU_SHIFTS>(
                (uint32_t)z, (uint32_t)(z >> 32), kc);
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                uint32_t mm = __ldcs(ma[p] + i);
                if (has_b) mm = fp_sub(mm, __ldcs(mb[p] + i));
                sm[p].add(mul_wide(r, mm));
                sx[p].add(mul_wide(r, __ldcs(xv[p] + i)));
            }
        }
    }
    // sigma partial of this thread per party: S_m - alpha_p * S_x (mod p)
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        unsigned long long s[1] = {fp_sub(sm[p].mod(), fp_mul(so.alpha[p], sx[p].mod()))};
        block_sum<1>(s);
        if (threadIdx.x == 0) atomicAdd(so.acc[p], (unsigned long long)fp_reduce64(s[0]));
    }
}

__global__ void __launch_bounds__(kThreads) k_mac_sigma_ranked(const uint32_t* __restrict__ value,
                                                               const uint32_t* __restrict__ mac,
                                                               const uint64_t* __restrict__ rank, uint64_t n,
                                                               uint64_t coin, uint32_t alpha,
                                                               unsigned long long* acc) {
    unsigned long long s[1] = {0ull};
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint32_t r = mac_coeff(coin, rank[i]);
        const uint32_t diff = fp_sub(mac[i], fp_mul(alpha, value[i]));
        s[0] = fold1(s[0] + fold1(mul_wide(r, diff)));
    }
    s[0] = fp_reduce64(s[0]);
    block_sum<1>(s);
    if (threadIdx.x == 0) atomicAdd(acc, (unsigned long long)fp_reduce64(s[0]));
}

// ---------------------------------------------------------------------------
// Linear layer: matrix_combine fused with the open of the [D|E] payload.
// One CTA per row (grid-strided); vectorised over the row when aligned.
// E (opened, din words) must already be in opened[cells .. cells+din).
// ---------------------------------------------------------------------------
struct PeerPtrs {
    const uint32_t* p[kMaxPeers];
};

template <int NP, bool V4>
__global__ void __launch_bounds__(kThreads) k_matrix_combine(uint32_t din, uint32_t rows, uint32_t rpt,
                                                             const uint32_t* own,
                                                             PeerPtrs peers_dev,
                                                             const uint32_t* __restrict__ Av,
                                                             const uint32_t* __restrict__ Am,
                                                             const uint32_t* __restrict__ Bv_all,
                                                             const uint32_t* __restrict__ Bm_all,
                                                             const uint32_t* __restrict__ Cv,
                                                             const uint32_t* __restrict__ Cm,
                                                             const uint32_t* __restrict__ biasv,
                                                             const uint32_t* __restrict__ biasm, int party,
                                                             uint32_t alpha, uint32_t* zv, uint32_t* zm,
                                                             uint32_t* opened, const uint32_t* alpha_dev) {
    if (alpha_dev) alpha = __ldg(alpha_dev);  // graph replays follow a re-deal
    const uint64_t cells = (uint64_t)din * rows;
    const uint32_t* peers[NP > 0 ? NP : 1];
#pragma unroll
    for (int p = 0; p < NP; ++p) peers[p] = peers_dev.p[p];
    for (uint32_t r = blockIdx.x; r < rows; r += gridDim.x) {
        const uint64_t base = (uint64_t)r * din;
        const uint64_t tile_off = (uint64_t)(r / rpt) * din;  // B_t / E_t of this row's tile
        const uint32_t* E = opened + cells + tile_off;
        const uint32_t* Bv = Bv_all + tile_off;
        const uint32_t* Bm = Bm_all + tile_off;
        unsigned long long acc[3] = {0ull, 0ull, 0ull};  // v, m, de
        if (V4) {
            const uint32_t n4 = din / 4;
            for (uint32_t g = threadIdx.x; g < n4; g += blockDim.x) {
                const uint64_t gg = base / 4 + g;
                // all loads before the opened-D store (E lives in `opened`: a later load would wait)
                uint4 d4 = ld4(own, gg);
                const uint4 av = ld4(Av, gg), am = ld4(Am, gg);
                const uint4 bv = reinterpret_cast<const uint4*>(Bv)[g], bm = reinterpret_cast<const uint4*>(Bm)[g];
                const uint4 e4 = reinterpret_cast<const uint4*>(E)[g];
                uint32_t d[4] = {d4.x, d4.y, d4.z, d4.w};
#pragma unroll
                for (int p = 0; p < NP; ++p) {
                    uint4 q = ld4_peer(peers[p], gg);
                    d[0] = fp_add(d[0], fp_reduce32(q.x));
                    d[1] = fp_add(d[1], fp_reduce32(q.y));
                    d[2] = fp_add(d[2], fp_reduce32(q.z));
                    d[3] = fp_add(d[3], fp_reduce32(q.w));
                }
                st4(opened, gg, d);
                const uint32_t A0[4] = {av.x, av.y, av.z, av.w}, A1[4] = {am.x, am.y, am.z, am.w};
                const uint32_t B0[4] = {bv.x, bv.y, bv.z, bv.w}, B1[4] = {bm.x, bm.y, bm.z, bm.w};
                const uint32_t Ee[4] = {e4.x, e4.y, e4.z, e4.w};
#pragma unroll
                for (int l = 0; l < 4; ++l) {
                    acc[0] += fold1(mul_wide(d[l], B0[l])) + fold1(mul_wide(A0[l], Ee[l]));
                    acc[1] += fold1(mul_wide(d[l], B1[l])) + fold1(mul_wide(A1[l], Ee[l]));
                    acc[2] += fold1(mul_wide(d[l], Ee[l]));
                }
            }
        } else {
            for (uint32_t c = threadIdx.x; c < din; c += blockDim.x) {
                uint32_t d = own[base + c];
#pragma unroll
                for (int p = 0; p < NP; ++p) d = fp_add(d, fp_reduce32(peers[p][base + c]));
                opened[base + c] = d;
                const uint32_t e = E[c];
                acc[0] += fold1(mul_wide(d, Bv[c])) + fold1(mul_wide(Av[base + c], e));
                acc[1] += fold1(mul_wide(d, Bm[c])) + fold1(mul_wide(Am[base + c], e));
                acc[2] += fold1(mul_wide(d, e));
            }
        }
        // per-thread partial sums are < din/256 * 12 * 2^32: fold before the tree
        acc[0] = fold1(acc[0]);
        acc[1] = fold1(acc[1]);
        acc[2] = fold1(acc[2]);
        block_sum<3>(acc);
        if (threadIdx.x == 0) {
            // spdz.cpp:117-123
            const uint32_t der = fp_reduce64(acc[2]);
            uint32_t vr = fp_reduce64((unsigned long long)Cv[r] + fp_reduce64(acc[0]));
            if (party == 0) vr = fp_add(vr, der);
            uint32_t mr = fp_add(fp_reduce64((unsigned long long)Cm[r] + fp_reduce64(acc[1])), fp_mul(alpha, der));
            if (biasv) {  // linear.cpp:59 add_local(z, b_slice)
                vr = fp_add(vr, biasv[r]);
                mr = fp_add(mr, biasm[r]);
            }
            zv[r] = vr;
            zm[r] = mr;
        }
    }
}

// Both parties of a 2-party linear layer on one GPU (spdz.cpp:98-124 for each party):
// the opened D = D0 + reduce(D1) is computed and logged once, each party's A planes,
// B_t, C and bias give its row result; sum D E (the same for both) is accumulated once.
// G threads per row (G = 32: a warp per row, shuffle reduction, every row in flight at
// once when rows are many; G = 256: a block per row for few long rows).

#ifndef SPDZ_MC2_MINB
#define SPDZ_MC2_MINB 1  // resident blocks per SM the register budget must allow (occupancy experiments)
#endif
template <int G, bool V4>
__global__ void __launch_bounds__(kThreads, SPDZ_MC2_MINB) k_matrix_combine2(MC2Args a) {
    constexpr int RPB = kThreads / G;  // rows per block
    const uint32_t g = threadIdx.x % G, slot = threadIdx.x / G;
    const uint64_t cells = (uint64_t)a.din * a.rows;
    // r is warp-uniform for G = 32 (warp_sum only) and block-uniform for G = 256 (block_sum)
    for (uint32_t r = blockIdx.x * RPB + slot; r < a.rows; r += gridDim.x * RPB) {
        const uint64_t base = (uint64_t)r * a.din;
        const uint64_t toff = (uint64_t)(r / a.rpt) * a.din;
        const uint32_t* E = a.opened + cells + toff;
        unsigned long long acc[5] = {0ull, 0ull, 0ull, 0ull, 0ull};  // v0 m0 v1 m1 de
        if (V4) {
            for (uint32_t c4 = g; c4 < a.din / 4; c4 += G) {
                const uint64_t gg = base / 4 + c4;
                // every load of the iteration issued before the opened-D store: the pointers are
                // not restrict, so a load after the store would wait for it (two round trips)
                const uint4 d0 = ld4(a.D0, gg), d1 = ld4(a.D1, gg);
                const uint4 e4 = reinterpret_cast<const uint4*>(E)[c4];
                uint4 av[2], am[2], bv[2], bm[2];
#pragma unroll
                for (int p = 0; p < 2; ++p) {
                    av[p] = ld4(a.A[p][0], gg);
                    am[p] = ld4(a.A[p][1], gg);
                    bv[p] = reinterpret_cast<const uint4*>(a.B[p][0] + toff)[c4];
                    bm[p] = reinterpret_cast<const uint4*>(a.B[p][1] + toff)[c4];
                }
                const uint32_t d[4] = {fp_add(d0.x, fp_reduce32(d1.x)), fp_add(d0.y, fp_reduce32(d1.y)),
                                       fp_add(d0.z, fp_reduce32(d1.z)), fp_add(d0.w, fp_reduce32(d1.w))};
                const uint32_t e[4] = {e4.x, e4.y, e4.z, e4.w};
#pragma unroll
                for (int l = 0; l < 4; ++l) acc[4] += fold1(mul_wide(d[l], e[l]));
#pragma unroll
                for (int p = 0; p < 2; ++p) {
                    const uint32_t AV[4] = {av[p].x, av[p].y, av[p].z, av[p].w};
                    const uint32_t AM[4] = {am[p].x, am[p].y, am[p].z, am[p].w};
                    const uint32_t BV[4] = {bv[p].x, bv[p].y, bv[p].z, bv[p].w};
                    const uint32_t BM[4] = {bm[p].x, bm[p].y, bm[p].z, bm[p].w};
#pragma unroll
                    for (int l = 0; l < 4; ++l) {
                        acc[2 * p] += fold1(mul_wide(d[l], BV[l])) + fold1(mul_wide(AV[l], e[l]));
                        acc[2 * p + 1] += fold1(mul_wide(d[l], BM[l])) + fold1(mul_wide(AM[l], e[l]));
                    }
                }
                st4(a.opened, gg, d);
            }
        } else {
            for (uint32_t c = g; c < a.din; c += G) {
                const uint32_t d = fp_add(a.D0[base + c], fp_reduce32(a.D1[base + c]));
                a.opened[base + c] = d;
                const uint32_t e = E[c];
                acc[4] += fold1(mul_wide(d, e));
#pragma unroll
                for (int p = 0; p < 2; ++p) {
                    acc[2 * p] += fold1(mul_wide(d, a.B[p][0][toff + c])) + fold1(mul_wide(a.A[p][0][base + c], e));
                    acc[2 * p + 1] += fold1(mul_wide(d, a.B[p][1][toff + c])) + fold1(mul_wide(a.A[p][1][base + c], e));
                }
            }
        }
#pragma unroll
        for (int q = 0; q < 5; ++q) acc[q] = fold1(acc[q]);  // < din/G * 12 * 2^32 before: safe below 2^64
        if (G == 32) {
#pragma unroll
            for (int q = 0; q < 5; ++q) acc[q] = warp_sum(acc[q]);
        } else {
            block_sum<5>(acc);
        }
        if (g == 0) {
            const uint32_t de = fp_reduce64(acc[4]);
            uint32_t vv[2];
#pragma unroll
            for (int p = 0; p < 2; ++p) {  // spdz.cpp:117-123, linear.cpp:59
                uint32_t vr = fp_reduce64((unsigned long long)a.Cc[p][0][r] + fp_reduce64(acc[2 * p]));
                if (p == 0) vr = fp_add(vr, de);
                uint32_t mr = fp_add(fp_reduce64((unsigned long long)a.Cc[p][1][r] + fp_reduce64(acc[2 * p + 1])),
                                     fp_mul(a.alpha_dev[p] ? __ldg(a.alpha_dev[p]) : a.alpha[p], de));
                if (a.bias[p][0]) {
                    vr = fp_add(vr, a.bias[p][0][r]);
                    mr = fp_add(mr, a.bias[p][1][r]);
                }
                a.z[p][0][r] = vr;
                a.z[p][1][r] = mr;
                vv[p] = vr;
            }
            if (a.open_out[0]) {  // the layer is the root: its opening (net.cpp:170-215) for both parties
                a.open_out[0][r] = fp_add(vv[0], fp_reduce32(vv[1]));
                a.open_out[1][r] = fp_add(vv[1], fp_reduce32(vv[0]));
            }
        }
    }
}

// Balanced variant (16-byte path): the dout x din cell space is one flat range of uint4
// groups split evenly over every resident warp of a one-wave grid, so no warp holds more than
// its share (a warp per row leaves a 1.15-wave tail at 4096 rows: 4096 warps on 148 x 24 warp
// slots).  A warp walks its range row segment by row segment; each segment's five lazy sums
// are warp-reduced and added to the row's u64 accumulators (scratch, zero between launches),
// and the warp that completes a row (its lane count reaches din/4) finalises it: C + sums,
// party 0's de, alpha_i de, bias (spdz.cpp:117-123, linear.cpp:59) — then re-zeroes the
// row's scratch.  Sums stay below 2^64: a segment adds < 2^40 and a row has at most din/4
// segments.
__device__ __forceinline__ void mc2_flush(const MC2Args& a, unsigned long long (&lo)[5], unsigned long long (&hi)[5],
                                          uint32_t r, uint32_t seg, uint32_t din4, unsigned long long* acc_rows,
                                          unsigned int* done_rows, uint32_t lane) {
    unsigned long long acc[5];
#pragma unroll
    for (int q = 0; q < 5; ++q) acc[q] = warp_sum(fold1((fold1(hi[q]) << 16) + fold1(lo[q])));
    if (lane == 0) {
        unsigned long long* ar = acc_rows + (uint64_t)r * 5;
#pragma unroll
        for (int q = 0; q < 5; ++q) atomicAdd(ar + q, acc[q]);
        // release: the sums above are visible before the count; acquire: the finaliser sees
        // every other segment's sums (no full fences on the warp's path)
        uint32_t prev;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(prev) : "l"(done_rows + r), "r"(seg)
                     : "memory");
        if (prev + seg == din4) {  // last segment of row r: finalise it
            unsigned long long sum[5];
#pragma unroll
            for (int q = 0; q < 5; ++q) sum[q] = atomicExch(ar + q, 0ull);
            done_rows[r] = 0;
            const uint32_t de = fp_reduce64(sum[4]);
            uint32_t vv[2];
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                uint32_t vr = fp_reduce64((unsigned long long)a.Cc[p][0][r] + fp_reduce64(sum[2 * p]));
                if (p == 0) vr = fp_add(vr, de);
                uint32_t mr = fp_add(fp_reduce64((unsigned long long)a.Cc[p][1][r] + fp_reduce64(sum[2 * p + 1])),
                                     fp_mul(a.alpha_dev[p] ? __ldg(a.alpha_dev[p]) : a.alpha[p], de));
                if (a.bias[p][0]) {
                    vr = fp_add(vr, a.bias[p][0][r]);
                    mr = fp_add(mr, a.bias[p][1][r]);
                }
                a.z[p][0][r] = vr;
                a.z[p][1][r] = mr;
                vv[p] = vr;
            }
            if (a.open_out[0]) {  // the layer is the root: its opening (net.cpp:170-215) for both parties
                a.open_out[0][r] = fp_add(vv[0], fp_reduce32(vv[1]));
                a.open_out[1][r] = fp_add(vv[1], fp_reduce32(vv[0]));
            }
        }
    }
#pragma unroll
    for (int q = 0; q < 5; ++q) lo[q] = hi[q] = 0ull;
}

struct MC2Ld {
    uint4 d0, d1, e4, av[2], am[2], bv[2], bm[2];
};
__device__ __forceinline__ void mc2_load(const MC2Args& a, uint64_t gg, uint32_t c4, const uint4* E4,
                                         const uint4* const (&B4)[2][2], MC2Ld& L) {
    L.d0 = ld4(a.D0, gg);
    L.d1 = ld4(a.D1, gg);
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        L.av[p] = ld4(a.A[p][0], gg);
        L.am[p] = ld4(a.A[p][1], gg);
    }
    L.e4 = E4[c4];
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        L.bv[p] = B4[p][0][c4];
        L.bm[p] = B4[p][1][c4];
    }
}// The nine products per cell (d e; d B.v, d B.m, A.v e, A.m e of each party) with the shared
// operands d and e split into 16-bit halves: every product is then < 2^48 and goes straight into a
// u64 accumulator as one IMAD.WIDE.U32 multiply-add (lo: low halves, hi: high halves, weight
// 2^16), instead of a 64-bit product, its fold and a 64-bit add.  A lane adds at most 2 din/32
// products per accumulator between flushes: below 2^64 for din < 2^20 (launcher).
__device__ __forceinline__ void mc2_compute(const MC2Args& a, uint64_t gg, const MC2Ld& L,
                                            unsigned long long (&lo)[5], unsigned long long (&hi)[5]) {
    const uint4 e4 = L.e4, bv[2] = {L.bv[0], L.bv[1]}, bm[2] = {L.bm[0], L.bm[1]};
    const uint32_t d[4] = {fp_add(L.d0.x, fp_reduce32(L.d1.x)), fp_add(L.d0.y, fp_reduce32(L.d1.y)),
                           fp_add(L.d0.z, fp_reduce32(L.d1.z)), fp_add(L.d0.w, fp_reduce32(L.d1.w))};
    const uint32_t e[4] = {e4.x, e4.y, e4.z, e4.w};
#pragma unroll
    for (int l = 0; l < 4; ++l) {
        const uint32_t dl = d[l] & 0xFFFFu, dh = d[l] >> 16, el = e[l] & 0xFFFFu, eh = e[l] >> 16;
        lo[4] += (unsigned long long)dl * e[l];
        hi[4] += (unsigned long long)dh * e[l];
        const uint32_t BV[2] = {l == 0 ? bv[0].x : l == 1 ? bv[0].y : l == 2 ? bv[0].z : bv[0].w,
                                l == 0 ? bv[1].x : l == 1 ? bv[1].y : l == 2 ? bv[1].z : bv[1].w};
        const uint32_t BM[2] = {l == 0 ? bm[0].x : l == 1 ? bm[0].y : l == 2 ? bm[0].z : bm[0].w,
                                l == 0 ? bm[1].x : l == 1 ? bm[1].y : l == 2 ? bm[1].z : bm[1].w};
        const uint32_t AV[2] = {l == 0 ? L.av[0].x : l == 1 ? L.av[0].y : l == 2 ? L.av[0].z : L.av[0].w,
                                l == 0 ? L.av[1].x : l == 1 ? L.av[1].y : l == 2 ? L.av[1].z : L.av[1].w};
        const uint32_t AM[2] = {l == 0 ? L.am[0].x : l == 1 ? L.am[0].y : l == 2 ? L.am[0].z : L.am[0].w,
                                l == 0 ? L.am[1].x : l == 1 ? L.am[1].y : l == 2 ? L.am[1].z : L.am[1].w};
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            lo[2 * p] += (unsigned long long)dl * BV[p] + (unsigned long long)el * AV[p];
            hi[2 * p] += (unsigned long long)dh * BV[p] + (unsigned long long)eh * AV[p];
            lo[2 * p + 1] += (unsigned long long)dl * BM[p] + (unsigned long long)el * AM[p];
            hi[2 * p + 1] += (unsigned long long)dh * BM[p] + (unsigned long long)eh * AM[p];
        }
    }
    st4(a.opened, gg, d);
}

// Balanced variant (16-byte path): the dout x din cell space is one flat range of uint4
// groups split evenly over every resident warp of a one-wave grid, so no warp holds more than
// its share (a warp per row leaves a 1.15-wave tail at 4096 rows: 4096 warps on 148 x 24 warp
// slots).  A warp walks its range row segment by row segment; each segment's five lazy sums
// are warp-reduced and added to the row's u64 accumulators (scratch, zero between launches),
// and the warp that completes a row (its lane count reaches din/4) finalises it: C + sums,
// party 0's de, alpha_i de, bias (spdz.cpp:117-123, linear.cpp:59) — then re-zeroes the
// row's scratch.  Sums stay below 2^64: a segment adds < 2^40 and a row has at most din/4
// segments.  UNROLL = 2 issues two groups' loads before either group's arithmetic (more
// bytes in flight per warp at the cost of registers; MINB resident blocks per SM).
template <int UNROLL, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) k_matrix_combine2_flat(MC2Args a, unsigned long long* acc_rows,
                                                                         unsigned int* done_rows) {
    const uint32_t din4 = a.din / 4;
    const uint64_t cells = (uint64_t)a.din * a.rows;
    const uint64_t U = (uint64_t)din4 * a.rows;
    const uint64_t warps = (uint64_t)gridDim.x * (kThreads / 32);
    const uint64_t w = (uint64_t)blockIdx.x * (kThreads / 32) + threadIdx.x / 32;
    const uint32_t lane = threadIdx.x & 31;
    uint64_t u0 = U * w / warps;
    const uint64_t u1 = U * (w + 1) / warps;
    while (u0 < u1) {
        const uint32_t r = (uint32_t)(u0 / din4);
        const uint64_t rbase = (uint64_t)r * din4;
        const uint64_t rend = u1 < rbase + din4 ? u1 : rbase + din4;
        const uint64_t toff = (uint64_t)(r / a.rpt) * a.din;
        const uint4* E4 = reinterpret_cast<const uint4*>(a.opened + cells + toff);
        const uint4* const B4[2][2] = {
            {reinterpret_cast<const uint4*>(a.B[0][0] + toff), reinterpret_cast<const uint4*>(a.B[0][1] + toff)},
            {reinterpret_cast<const uint4*>(a.B[1][0] + toff), reinterpret_cast<const uint4*>(a.B[1][1] + toff)}};
        unsigned long long lo[5] = {0ull, 0ull, 0ull, 0ull, 0ull}, hi[5] = {0ull, 0ull, 0ull, 0ull, 0ull};  // v0 m0 v1 m1 de
        uint64_t gg = u0 + lane;
        if (UNROLL == 2) {
            for (; gg + 32 < rend; gg += 64) {
                MC2Ld L0, L1;
                mc2_load(a, gg, (uint32_t)(gg - rbase), E4, B4, L0);
                mc2_load(a, gg + 32, (uint32_t)(gg + 32 - rbase), E4, B4, L1);
                mc2_compute(a, gg, L0, lo, hi);
                mc2_compute(a, gg + 32, L1, lo, hi);
            }
        }
        for (; gg < rend; gg += 32) {
            MC2Ld L0;
            mc2_load(a, gg, (uint32_t)(gg - rbase), E4, B4, L0);
            mc2_compute(a, gg, L0, lo, hi);
        }
        mc2_flush(a, lo, hi, r, (uint32_t)(rend - u0), din4, acc_rows, done_rows, lane);
        u0 = rend;
    }
}

// ---------------------------------------------------------------------------
// CUDA-core modular GEMM: C (MxN) = A (MxK) * B (KxN) mod p, row-major.
// A is split into 16-bit halves when staged to shared memory, so each MAC is
// one IMAD.WIDE.U32 into a u64 (a_half*b < 2^48): 2^15 K-steps between folds.
// 64x64 CTA tile, 16-deep K tile, 256 threads each owning 4x4 outputs.
// ---------------------------------------------------------------------------
constexpr int GT = 64, GK = 16;

__global__ void __launch_bounds__(256) k_modgemm(uint32_t M, uint32_t N, uint32_t K, const uint32_t* A0,
                                                 const uint32_t* A1, const uint32_t* B0, const uint32_t* B1,
                                                 uint32_t* C0, uint32_t* C1) {
    const uint32_t* A = blockIdx.z ? A1 : A0;
    const uint32_t* B = blockIdx.z ? B1 : B0;
    uint32_t* C = blockIdx.z ? C1 : C0;
    __shared__ __align__(16) uint32_t sAl[GK][GT + 4];
    __shared__ __align__(16) uint32_t sAh[GK][GT + 4];
    __shared__ __align__(16) uint32_t sB[GK][GT + 4];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const uint32_t m0 = blockIdx.y * GT, n0 = blockIdx.x * GT;
    unsigned long long lo[4][4], hi[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) lo[i][j] = hi[i][j] = 0ull;
    uint32_t since_fold = 0;
    for (uint32_t k0 = 0; k0 < K; k0 += GK) {
        // stage A tile (GT rows x GK cols) transposed, B tile (GK rows x GT cols)
        for (int idx = threadIdx.x; idx < GT * GK; idx += 256) {
            const int r = idx / GK, c = idx % GK;
            const uint32_t gr = m0 + r, gc = k0 + c;
            const uint32_t a = (gr < M && gc < K) ? A[(uint64_t)gr * K + gc] : 0u;
            sAl[c][r] = a & 0xffffu;
            sAh[c][r] = a >> 16;
            const int br = idx / GT, bc = idx % GT;
            const uint32_t gbr = k0 + br, gbc = n0 + bc;
            sB[br][bc] = (gbr < K && gbc < N) ? B[(uint64_t)gbr * N + gbc] : 0u;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < GK; ++k) {
            const uint4 al4 = *reinterpret_cast<const uint4*>(&sAl[k][ty * 4]);
            const uint4 ah4 = *reinterpret_cast<const uint4*>(&sAh[k][ty * 4]);
            const uint4 b4 = *reinterpret_cast<const uint4*>(&sB[k][tx * 4]);
            const uint32_t al[4] = {al4.x, al4.y, al4.z, al4.w}, ah[4] = {ah4.x, ah4.y, ah4.z, ah4.w};
            const uint32_t b[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    lo[i][j] += mul_wide(al[i], b[j]);
                    hi[i][j] += mul_wide(ah[i], b[j]);
                }
        }
        since_fold += GK;
        if (since_fold >= 32768) {  // keep the u64 accumulators from overflowing
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    lo[i][j] = fold1(lo[i][j]);
                    hi[i][j] = fold1(hi[i][j]);
                }
            since_fold = 0;
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t gr = m0 + ty * 4 + i;
        if (gr >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t gc = n0 + tx * 4 + j;
            if (gc >= N) continue;
            const uint32_t h = fp_reduce64(hi[i][j]);
            C[(uint64_t)gr * N + gc] = fp_reduce64((unsigned long long)fp_reduce64(lo[i][j]) + mul_wide(h, 65536u));
        }
    }
}

// ---------------------------------------------------------------------------
// GPU dealer (spdz.cpp:162-249).  Draw k of the dealer stream (0-based after
// construction) = reduce(mix(seed + (k+1) gamma)); the reference redraws when
// the raw value is >= 2^64 - 25 (spdz.cpp:175-183): flagged, never silently
// shifted.
// ---------------------------------------------------------------------------
constexpr uint64_t kRejectBound = 0xFFFFFFFFFFFFFFE7ull;  // (2^64-1)/p*p = 2^64 - 25

__device__ __forceinline__ uint32_t draw(uint64_t seed, uint64_t k, unsigned int* flag) {
    const uint64_t v = mix64(seed + (k + 1) * kGamma);
    if (v >= kRejectBound) atomicOr(flag, 1u);
    return fp_reduce64(v);
}

// spdz.cpp:185-201 for one lane: party i>=1 gets (val, mac) draws at
// base + 2(i-1), +1; party 0 the remainder.
__device__ __forceinline__ void share_lane(int n, uint64_t seed, uint64_t base, uint32_t alpha, uint32_t x,
                                           uint32_t* vals, uint32_t* macs, uint64_t pstride, uint64_t j,
                                           unsigned int* flag) {
    uint32_t vs = 0, ms = 0;
    for (int i = 1; i < n; ++i) {
        const uint32_t v = draw(seed, base + 2 * (i - 1), flag);
        const uint32_t m = draw(seed, base + 2 * (i - 1) + 1, flag);
        vals[(uint64_t)i * pstride + j] = v;
        macs[(uint64_t)i * pstride + j] = m;
        vs = fp_add(vs, v);
        ms = fp_add(ms, m);
    }
    vals[j] = fp_sub(x, vs);
    macs[j] = fp_sub(fp_mul(alpha, x), ms);
}

// Lanes [j_first, j_first+count) of dealer.triples(S_total) (spdz.cpp:210-225);
// party p's share of local lane j goes to plane[p * pstride + j].
__global__ void k_dealer_triples(int n, uint64_t seed, uint64_t draw0, uint32_t alpha, uint64_t S_total,
                                 uint64_t j_first, uint64_t count, uint64_t pstride, uint32_t* av, uint32_t* am,
                                 uint32_t* bv, uint32_t* bm, uint32_t* cv, uint32_t* cm, unsigned int* flag) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t per = 2ull * (n - 1);
    const uint64_t sa = draw0 + 2 * S_total, sb = sa + per * S_total, sc = sb + per * S_total;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < count; j += stride) {
        const uint64_t g = j_first + j;
        const uint32_t a = draw(seed, draw0 + 2 * g, flag);
        const uint32_t b = draw(seed, draw0 + 2 * g + 1, flag);
        const uint32_t c = fp_mul(a, b);
        share_lane(n, seed, sa + g * per, alpha, a, av, am, pstride, j, flag);
        share_lane(n, seed, sb + g * per, alpha, b, bv, bm, pstride, j, flag);
        share_lane(n, seed, sc + g * per, alpha, c, cv, cm, pstride, j, flag);
    }
}

__global__ void k_dealer_share(int n, uint64_t seed, uint64_t draw0, uint32_t alpha, const uint32_t* clear,
                               uint64_t lanes, uint32_t* vals, uint32_t* macs, uint64_t pstride, unsigned int* flag) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t per = 2ull * (n - 1);
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < lanes; j += stride)
        share_lane(n, seed, draw0 + j * per, alpha, clear[j], vals, macs, pstride, j, flag);
}

__global__ void k_dealer_uniform(uint64_t seed, uint64_t draw0, uint64_t count, uint32_t* out, unsigned int* flag) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < count; j += stride)
        out[j] = draw(seed, draw0 + j, flag);
}

// C[r] = sum_c A[r,c] B[c] mod p (spdz.cpp:239-246)
__global__ void __launch_bounds__(kThreads) k_dealer_matvec(const uint32_t* A, const uint32_t* B, uint32_t din,
                                                            uint32_t rows, uint32_t* C) {
    for (uint32_t r = blockIdx.x; r < rows; r += gridDim.x) {
        unsigned long long s[1] = {0ull};
        for (uint32_t c = threadIdx.x; c < din; c += blockDim.x)
            s[0] += fold1(mul_wide(A[(uint64_t)r * din + c], B[c]));
        s[0] = fold1(s[0]);
        block_sum<1>(s);
        if (threadIdx.x == 0) C[r] = fp_reduce64(s[0]);
    }
}

// triple_store.cpp:274-283: mask j = share_random(1): clear draw, then share draws.
// Masks [m_first, m_first+count) (triple_store.cpp:274-283): mask m = share_random(1):
// one clear draw, then the share draws.  Party p's share of local mask j -> [p * pstride + j].
__global__ void k_dealer_masks(int n, uint64_t seed, uint64_t draw0, uint32_t alpha, uint64_t m_first, uint64_t count,
                               uint64_t pstride, uint32_t* vals, uint32_t* macs, uint32_t* clear, unsigned int* flag) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t per = 1 + 2ull * (n - 1);
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < count; j += stride) {
        const uint64_t base = draw0 + (m_first + j) * per;
        const uint32_t x = draw(seed, base, flag);
        clear[j] = x;
        share_lane(n, seed, base + 1, alpha, x, vals, macs, pstride, j, flag);
    }
}

// public (cleartext) lane ops with scalar broadcast (runtime.cpp:131-136, 168-172)
__global__ void __launch_bounds__(kThreads) k_pub_binop(int op, const uint32_t* a, bool a_b, const uint32_t* b,
                                                        bool b_b, uint32_t* out, uint64_t n) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint32_t a0 = a_b ? a[0] : 0u, b0 = b_b ? b[0] : 0u;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint32_t x = a_b ? a0 : a[i], y = b_b ? b0 : b[i];
        uint32_t z;
        switch (op) {
            case 0: z = fp_add(x, y); break;
            case 1: z = fp_sub(x, y); break;
            case 2: z = fp_mul(x, y); break;
            // 3 + ir::CmpPred: cmp_eval (runtime.cpp:49-58) on the u32 representatives
            case 3: z = x == y; break;
            case 4: z = x != y; break;
            case 5: z = x < y; break;
            case 6: z = x > y; break;
            case 7: z = x <= y; break;
            default: z = x >= y; break;
        }
        out[i] = z;
    }
}

// bcast_share (runtime.cpp:41-47): every lane = lane 0 of the source
__global__ void __launch_bounds__(kThreads) k_bcast2(const uint32_t* sv, const uint32_t* sm, uint32_t* ov,
                                                     uint32_t* om, uint64_t n) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint32_t v = sv[0], m = sm ? sm[0] : 0u;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        ov[i] = v;
        if (om) om[i] = m;
    }
}

// E_t = x.v - B_t.v for every tile t (linear.cpp:44-47), B laid out n_tiles x din
__global__ void __launch_bounds__(kThreads) k_tile_e(const uint32_t* __restrict__ xv, const uint32_t* __restrict__ bv,
                                                     uint32_t din, uint64_t total, uint32_t* __restrict__ out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride)
        out[i] = fp_sub(xv[i % din], bv[i]);
}

// Both parties' linear-layer mask in one launch (linear.cpp:40-47, value planes): D_p = W_p.v
// - A_p.v over every cell, then E_p[t] = x_p.v - B_p.v[t] for every tile, as one grid-strided
// range of uint4 groups (two in flight per thread), so the layer's mask is one kernel instead
// of a D pass plus an E pass per party.
__device__ __forceinline__ uint4 fp_sub4(const uint4 a, const uint4 b) {
    return make_uint4(fp_sub(a.x, b.x), fp_sub(a.y, b.y), fp_sub(a.z, b.z), fp_sub(a.w, b.w));
}
__device__ __forceinline__ void linmask_group(const LinMask2Args& m, uint64_t ud, uint32_t din4, uint64_t g) {
    if (g < ud) {
        const uint4 w0 = ld4(m.w[0], g), a0 = ld4(m.a[0], g), w1 = ld4(m.w[1], g), a1 = ld4(m.a[1], g);
        reinterpret_cast<uint4*>(m.pay[0])[g] = fp_sub4(w0, a0);
        reinterpret_cast<uint4*>(m.pay[1])[g] = fp_sub4(w1, a1);
    } else {
        const uint64_t e = g - ud, c4 = e % din4;
        const uint4 x0 = ld4(m.x[0], c4), b0 = ld4(m.b[0], e), x1 = ld4(m.x[1], c4), b1 = ld4(m.b[1], e);
        const uint4 e0 = fp_sub4(x0, b0), e1 = fp_sub4(x1, b1);
        reinterpret_cast<uint4*>(m.pay[0] + m.cells)[e] = e0;
        reinterpret_cast<uint4*>(m.pay[1] + m.cells)[e] = e1;
        if (m.opened_e)  // both payloads are local: E opened here (net.cpp:170-215 sum) instead of a launch
            reinterpret_cast<uint4*>(m.opened_e)[e] = make_uint4(fp_add(e0.x, e1.x), fp_add(e0.y, e1.y),
                                                                 fp_add(e0.z, e1.z), fp_add(e0.w, e1.w));
    }
}
__global__ void __launch_bounds__(kThreads) k_linear_mask2(LinMask2Args m) {
    const uint64_t ud = m.cells / 4, total = ud + (uint64_t)m.din * m.ntiles / 4;
    const uint32_t din4 = m.din / 4;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; g + stride < total; g += 2 * stride) {  // both groups' loads issue before either's stores
        linmask_group(m, ud, din4, g);
        linmask_group(m, ud, din4, g + stride);
    }
    if (g < total) linmask_group(m, ud, din4, g);
}

__global__ void k_set_word(uint32_t* p, uint32_t v) {
    if (threadIdx.x == 0) *p = v;
}

__global__ void k_xor_word(uint32_t* p, uint32_t mask) {
    if (threadIdx.x == 0) *p ^= mask;
}

}  // namespace

// ===========================================================================
// launchers
// ===========================================================================
cudaError_t launch_add_sub(cudaStream_t s, bool sub, const uint32_t* xv, const uint32_t* xm, const uint32_t* yv,
                           const uint32_t* ym, uint32_t* zv, uint32_t* zm, uint64_t n, int sms) {
    IO<4, 2> io{{xv, xm, yv, ym}, {zv, zm}};
    return sub ? run_map(s, io, n, OpSub{}, sms) : run_map(s, io, n, OpAdd{}, sms);
}

cudaError_t launch_add_sub2(cudaStream_t s, bool sub, const uint32_t* const xy[8], uint32_t* const z[4], uint64_t n,
                            int sms) {
    IO<8, 4> io{{xy[0], xy[1], xy[2], xy[3], xy[4], xy[5], xy[6], xy[7]}, {z[0], z[1], z[2], z[3]}};
    return sub ? run_map(s, io, n, OpAddSub2<true>{}, sms) : run_map(s, io, n, OpAddSub2<false>{}, sms);
}

template <bool SUB, int SM2, bool ROOT>
static cudaError_t add_sub2x(cudaStream_t s, const uint32_t* const xy[8], const uint32_t* const o[4],
                             uint32_t* const z[4], uint32_t* const w[4], uint32_t* const out[2], uint64_t n, int sms) {
    IO<12, ROOT ? 10 : 8> io;
    for (int k = 0; k < 8; ++k) io.in[k] = xy[k];
    for (int k = 0; k < 4; ++k) {
        io.in[8 + k] = o[k];
        io.out[k] = z[k];
        io.out[4 + k] = w[k];
    }
    if constexpr (ROOT) {
        io.out[8] = out[0];
        io.out[9] = out[1];
    }
    return run_map(s, io, n, OpAddSub2X<SUB, SM2, ROOT>{}, sms);
}

cudaError_t launch_add_sub2_chain(cudaStream_t s, bool sub, const uint32_t* const xy[8], uint32_t* const z[4], int sm2,
                                  const uint32_t* const o[4], uint32_t* const w[4], uint32_t* const out[2], uint64_t n,
                                  int sms) {
#define CASE(SB, SM2, R) \
    if (sub == SB && sm2 == SM2 && (out != nullptr) == R) return add_sub2x<SB, SM2, R>(s, xy, o, z, w, out, n, sms);
    CASE(false, 0, false) CASE(false, 1, false) CASE(false, 2, false) CASE(true, 0, false) CASE(true, 1, false)
    CASE(true, 2, false) CASE(false, 0, true) CASE(false, 1, true) CASE(false, 2, true) CASE(true, 0, true)
    CASE(true, 1, true) CASE(true, 2, true)
#undef CASE
    return cudaErrorInvalidValue;
}

template <int OPC>
static cudaError_t public_dispatch(cudaStream_t s, const uint32_t* xv, const uint32_t* xm, const uint32_t* k, int km,
                                   uint32_t kk, int party, uint32_t alpha, const uint32_t* ap, uint32_t* zv,
                                   uint32_t* zm, uint64_t n, int sms) {
    if (km == 0) {
        IO<3, 2> io{{xv, xm, k}, {zv, zm}};
        return run_map(s, io, n, OpPublic<OPC, 0>{{alpha, ap}, party, 0u, k}, sms);
    }
    IO<2, 2> io{{xv, xm}, {zv, zm}};
    if (km == 1) return run_map(s, io, n, OpPublic<OPC, 1>{{alpha, ap}, party, 0u, k}, sms);
    return run_map(s, io, n, OpPublic<OPC, 2>{{alpha, ap}, party, kk, k}, sms);
}

cudaError_t launch_public(cudaStream_t s, int op, const uint32_t* xv, const uint32_t* xm, const uint32_t* k,
                          bool k_bcast, uint32_t k_imm, bool k_is_imm, int party, uint32_t alpha, uint32_t* zv,
                          uint32_t* zm, uint64_t n, int sms, const uint32_t* ap) {
    const int km = k_is_imm ? 2 : (k_bcast ? 1 : 0);
    switch (op) {
        case 0: return public_dispatch<0>(s, xv, xm, k, km, k_imm, party, alpha, ap, zv, zm, n, sms);
        case 1: return public_dispatch<1>(s, xv, xm, k, km, k_imm, party, alpha, ap, zv, zm, n, sms);
        case 2: return public_dispatch<2>(s, xv, xm, k, km, k_imm, party, alpha, ap, zv, zm, n, sms);
        case 3: return public_dispatch<3>(s, xv, xm, k, km, k_imm, party, alpha, ap, zv, zm, n, sms);
        case 4: {
            if (km == 0) {
                IO<1, 2> io{{k}, {zv, zm}};
                return run_map(s, io, n, OpShareOfPublic<0>{{alpha, ap}, party, 0u, k}, sms);
            }
            IO<0, 2> io{{nullptr}, {zv, zm}};
            if (km == 1) return run_map(s, io, n, OpShareOfPublic<1>{{alpha, ap}, party, 0u, k}, sms);
            return run_map(s, io, n, OpShareOfPublic<2>{{alpha, ap}, party, k_imm, k}, sms);
        }
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_mul_mask(cudaStream_t s, const uint32_t* xv, const uint32_t* yv, const uint32_t* av,
                            const uint32_t* bv, uint32_t* d, uint32_t* e, uint64_t n, int sms) {
    IO<4, 2> io{{xv, yv, av, bv}, {d, e}};
    return run_map(s, io, n, OpMask{}, sms);
}

cudaError_t launch_mul_mask2(cudaStream_t s, const uint32_t* const xyab[8], uint32_t* const de[4], uint64_t n,
                             int sms) {
    IO<8, 4> io{{xyab[0], xyab[1], xyab[2], xyab[3], xyab[4], xyab[5], xyab[6], xyab[7]}, {de[0], de[1], de[2], de[3]}};
    return run_map(s, io, n, OpMask2{}, sms);
}

cudaError_t launch_beaver_combine(cudaStream_t s, const uint32_t* own_d, const uint32_t* own_e,
                                  const uint32_t* const* peer_d, const uint32_t* const* peer_e, int n_peers,
                                  const uint32_t* const tri[6], int party, uint32_t alpha, uint32_t* zv, uint32_t* zm,
                                  uint32_t* open_d, uint32_t* open_e, uint64_t n, int sms, const uint32_t* alpha_dev) {
    switch (n_peers) {
#define CASE(NP) \
    case NP:     \
        return combine_np<NP>(s, own_d, own_e, peer_d, peer_e, tri, party, alpha, zv, zm, open_d, open_e, n, sms, alpha_dev);
        CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7)
#undef CASE
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_beaver_combine_mask(cudaStream_t s, const uint32_t* own_d, const uint32_t* own_e,
                                       const uint32_t* const* peer_d, const uint32_t* const* peer_e, int n_peers,
                                       const uint32_t* const tri[6], int party, uint32_t alpha, uint32_t* zv,
                                       uint32_t* zm, uint32_t* open_d, uint32_t* open_e, int zpos,
                                       const uint32_t* const next[3], uint32_t* const next_de[2], uint64_t n, int sms,
                                       const uint32_t* alpha_dev) {
#define CASE(NP, Z)                                                                                              \
    if (n_peers == NP && zpos == Z)                                                                              \
        return combine_m_np<NP, Z>(s, own_d, own_e, peer_d, peer_e, tri, party, alpha, zv, zm, open_d, open_e, next, \
                                   next_de, n, sms, alpha_dev);
    CASE(1, 0) CASE(1, 1) CASE(1, 2) CASE(2, 0) CASE(2, 1) CASE(2, 2) CASE(3, 0) CASE(3, 1) CASE(3, 2)
#undef CASE
    return cudaErrorInvalidValue;
}

cudaError_t launch_beaver_combine_add(cudaStream_t s, const uint32_t* own_d, const uint32_t* own_e,
                                      const uint32_t* peer_d, const uint32_t* peer_e, const uint32_t* const tri[6],
                                      int party, uint32_t alpha, uint32_t* zv, uint32_t* zm, uint32_t* open_d,
                                      uint32_t* open_e, int sm, const uint32_t* const addin[2], uint32_t* const w[2],
                                      int nx, const uint32_t* const next[3], uint32_t* const next_de[2], uint64_t n,
                                      int sms, const uint32_t* alpha_dev) {
    const uint32_t* in10[10] = {own_d, own_e, peer_d, peer_e, tri[0], tri[1], tri[2], tri[3], tri[4], tri[5]};
    uint32_t* const out4[4] = {zv, zm, open_d, open_e};
#define CASE(SM, NX) \
    if (sm == SM && nx == NX) return combine_a<SM, NX>(s, in10, addin, next, out4, w, next_de, party, alpha, alpha_dev, n, sms);
    CASE(0, 0) CASE(0, 1) CASE(0, 2) CASE(0, 3)
    CASE(1, 0) CASE(1, 1) CASE(1, 2) CASE(1, 3)
    CASE(2, 0) CASE(2, 1) CASE(2, 2) CASE(2, 3)
#undef CASE
    return cudaErrorInvalidValue;
}

cudaError_t launch_beaver_combine2(cudaStream_t s, const uint32_t* const de[4], const uint32_t* const tri0[6],
                                   const uint32_t* const tri1[6], const uint32_t alpha[2],
                                   const uint32_t* const alpha_dev[2], uint32_t* const z[4], uint32_t* open_d,
                                   uint32_t* open_e, uint64_t n, int sms) {
    IO<16, 6> io;
    for (int k = 0; k < 4; ++k) io.in[k] = de[k];
    for (int k = 0; k < 6; ++k) {
        io.in[4 + k] = tri0[k];
        io.in[10 + k] = tri1[k];
    }
    for (int k = 0; k < 4; ++k) io.out[k] = z[k];
    io.out[4] = open_d;
    io.out[5] = open_e;
    return run_map(s, io, n, OpCombine2{alpha[0], alpha[1], alpha_dev[0], alpha_dev[1]}, sms);
}

// OpCombine2 followed, in the same pass, by a private add / sub that consumes this product
// (backend.cpp:25-51 on both planes: w = z + o, z - o or o - z; SM = 0 / 1 / 2) and then,
// optionally, the multiply after it that consumes w (its mask: NX = 1 w left, 2 w right, 3 both) or
// the root opening of w (NX = 4).  Inputs: OpCombine2's 16, then per party o.v o.m [the next
// multiply's other operand .v (NX 1, 2), a'.v, b'.v].  Outputs: OpCombine2's 6, w.v w.m of both
// parties, then d'0 e'0 d'1 e'1 (NX 1-3) or both parties' opened outputs (NX 4).
template <int SM, int NX>
struct OpCombine2A : OpCombine2 {
    static constexpr int kMask = NX >= 1 && NX <= 3 ? (NX == 3 ? 2 : 3) : 0;
    static constexpr int kPer = 2 + kMask;  // extra inputs per party
    static constexpr int kOut = 10 + (kMask ? 4 : NX == 4 ? 2 : 0);
    __device__ void operator()(const uint32_t* in, uint32_t* o) const {
        OpCombine2::operator()(in, o);
        uint32_t w[2];
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            const uint32_t* q = in + 16 + kPer * p;
            const uint32_t zv = o[2 * p], zm = o[2 * p + 1];
            const uint32_t wv = SM == 0 ? fp_add(zv, q[0]) : SM == 1 ? fp_sub(zv, q[0]) : fp_sub(q[0], zv);
            const uint32_t wm = SM == 0 ? fp_add(zm, q[1]) : SM == 1 ? fp_sub(zm, q[1]) : fp_sub(q[1], zm);
            o[6 + 2 * p] = wv;
            o[7 + 2 * p] = wm;
            w[p] = wv;
            if constexpr (kMask > 0) {
                const uint32_t* r = q + 2;
                const uint32_t x = NX == 2 ? r[0] : wv, y = NX == 1 ? r[0] : wv;
                const uint32_t* ab = r + (NX == 3 ? 0 : 1);
                o[10 + 2 * p] = fp_sub(x, ab[0]);
                o[11 + 2 * p] = fp_sub(y, ab[1]);
            }
        }
        if constexpr (NX == 4) {
            o[10] = fp_add(w[0], fp_reduce32(w[1]));
            o[11] = fp_add(w[1], fp_reduce32(w[0]));
        }
    }
};

template <int SM, int NX>
static cudaError_t combine2a(cudaStream_t s, const IO<16, 6>& base, const uint32_t* const addin[4],
                            const uint32_t* const nx[6], uint32_t* const w[4], uint32_t* const extra[4],
                            const OpCombine2& op, uint64_t n, int sms) {
    using Op = OpCombine2A<SM, NX>;
    IO<16 + 2 * Op::kPer, Op::kOut> io;
    for (int k = 0; k < 16; ++k) io.in[k] = base.in[k];
    for (int p = 0; p < 2; ++p) {
        int k = 16 + Op::kPer * p;
        io.in[k++] = addin[2 * p];      // o.v
        io.in[k++] = addin[2 * p + 1];  // o.m
        if constexpr (Op::kMask > 0) {
            if (NX != 3) io.in[k++] = nx[3 * p];
            io.in[k++] = nx[3 * p + 1];
            io.in[k] = nx[3 * p + 2];
        }
    }
    for (int k = 0; k < 6; ++k) io.out[k] = base.out[k];
    for (int k = 0; k < 4; ++k) io.out[6 + k] = w[k];
    for (int k = 0; k < Op::kOut - 10; ++k) io.out[10 + k] = extra[k];
    Op f;
    static_cast<OpCombine2&>(f) = op;
    return run_map(s, io, n, f, sms);
}

template <int ZPOS>
static cudaError_t combine2m(cudaStream_t s, const IO<16, 6>& base, const uint32_t* const nx[6],
                            uint32_t* const nde[4], const OpCombine2& op, uint64_t n, int sms) {
    constexpr int K = OpCombine2M<ZPOS>::kPer;
    IO<16 + 2 * K, ZPOS == 3 ? 8 : 10> io;
    for (int k = 0; k < 16; ++k) io.in[k] = base.in[k];
    if constexpr (K > 0) {
        for (int p = 0; p < 2; ++p) {
            int k = 16 + K * p;
            if (ZPOS != 2) io.in[k++] = nx[3 * p];  // the next multiply's other operand
            io.in[k++] = nx[3 * p + 1];             // a'.v
            io.in[k] = nx[3 * p + 2];               // b'.v
        }
    }
    for (int k = 0; k < 6; ++k) io.out[k] = base.out[k];
    for (int k = 0; k < (ZPOS == 3 ? 2 : 4); ++k) io.out[6 + k] = nde[k];
    OpCombine2M<ZPOS> f;
    static_cast<OpCombine2&>(f) = op;
    return run_map(s, io, n, f, sms);
}

cudaError_t launch_beaver_combine2_add(cudaStream_t s, const uint32_t* const de[4], const uint32_t* const tri0[6],
                                       const uint32_t* const tri1[6], const uint32_t alpha[2],
                                       const uint32_t* const alpha_dev[2], uint32_t* const z[4], uint32_t* open_d,
                                       uint32_t* open_e, int sm, const uint32_t* const addin[4], uint32_t* const w[4],
                                       int nx, const uint32_t* const next[6], uint32_t* const extra[4], uint64_t n,
                                       int sms) {
    IO<16, 6> io;
    for (int k = 0; k < 4; ++k) io.in[k] = de[k];
    for (int k = 0; k < 6; ++k) {
        io.in[4 + k] = tri0[k];
        io.in[10 + k] = tri1[k];
    }
    for (int k = 0; k < 4; ++k) io.out[k] = z[k];
    io.out[4] = open_d;
    io.out[5] = open_e;
    const OpCombine2 op{alpha[0], alpha[1], alpha_dev[0], alpha_dev[1]};
#define CASE(SM, NX) \
    if (sm == SM && nx == NX) return combine2a<SM, NX>(s, io, addin, next, w, extra, op, n, sms);
    CASE(0, 0) CASE(0, 1) CASE(0, 2) CASE(0, 3) CASE(0, 4)
    CASE(1, 0) CASE(1, 1) CASE(1, 2) CASE(1, 3) CASE(1, 4)
    CASE(2, 0) CASE(2, 1) CASE(2, 2) CASE(2, 3) CASE(2, 4)
#undef CASE
    return cudaErrorInvalidValue;
}

cudaError_t launch_beaver_combine2_mask(cudaStream_t s, const uint32_t* const de[4], const uint32_t* const tri0[6],
                                        const uint32_t* const tri1[6], const uint32_t alpha[2],
                                        const uint32_t* const alpha_dev[2], uint32_t* const z[4], uint32_t* open_d,
                                        uint32_t* open_e, int zpos, const uint32_t* const next[6],
                                        uint32_t* const next_de[4], uint64_t n, int sms) {
    IO<16, 6> io;
    for (int k = 0; k < 4; ++k) io.in[k] = de[k];
    for (int k = 0; k < 6; ++k) {
        io.in[4 + k] = tri0[k];
        io.in[10 + k] = tri1[k];
    }
    for (int k = 0; k < 4; ++k) io.out[k] = z[k];
    io.out[4] = open_d;
    io.out[5] = open_e;
    const OpCombine2 op{alpha[0], alpha[1], alpha_dev[0], alpha_dev[1]};
    switch (zpos) {
        case 0: return combine2m<0>(s, io, next, next_de, op, n, sms);
        case 1: return combine2m<1>(s, io, next, next_de, op, n, sms);
        case 2: return combine2m<2>(s, io, next, next_de, op, n, sms);
        case 3: return combine2m<3>(s, io, next, next_de, op, n, sms);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_share_input2(cudaStream_t s, const uint32_t* x_raw, const uint32_t* r_clear,
                                const uint32_t* const mask[4], const uint32_t alpha[2],
                                const uint32_t* const alpha_dev[2], uint32_t* const out[4], uint64_t n, int sms) {
    IO<6, 4> io{{x_raw, r_clear, mask[0], mask[1], mask[2], mask[3]}, {out[0], out[1], out[2], out[3]}};
    return run_map(s, io, n, OpShareInput2{alpha[0], alpha[1], alpha_dev[0], alpha_dev[1]}, sms);
}

cudaError_t launch_open_sum(cudaStream_t s, const uint32_t* own, const uint32_t* const* peers, int n_peers,
                            uint32_t* out, uint64_t n, int sms) {
    switch (n_peers) {
#define CASE(NP) \
    case NP: return open_np<NP>(s, own, peers, out, n, sms);
        CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7)
#undef CASE
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_open_sum2(cudaStream_t s, const uint32_t* z0, const uint32_t* z1, uint32_t* out0, uint32_t* out1,
                             uint64_t n, int sms) {
    IO<2, 2> io{{z0, z1}, {out0, out1}};
    return run_map(s, io, n, OpOpen2{}, sms);
}

cudaError_t launch_reduce_add(cudaStream_t s, const uint32_t* xv, const uint32_t* xm, uint64_t n,
                              unsigned long long* acc, int sms) {
    k_reduce_add<<<grid_for(n, sms), kThreads, 0, s>>>(xv, xm, n, acc);
    return launched();
}

cudaError_t launch_finish_reduce(cudaStream_t s, const unsigned long long* acc, uint32_t* outv, uint32_t* outm) {
    k_finish_reduce<<<1, 32, 0, s>>>(acc, outv, outm);
    return launched();
}

cudaError_t launch_pair_split(cudaStream_t s, const uint32_t* cv, const uint32_t* cm, uint64_t pairs, uint32_t* xv,
                              uint32_t* xm, uint32_t* yv, uint32_t* ym, int sms) {
    if (pairs == 0) return cudaSuccess;
    k_pair_split<<<grid_for(pairs, sms), kThreads, 0, s>>>(cv, cm, pairs, xv, xm, yv, ym);
    return launched();
}

template <int NP>
static cudaError_t mac_sigma_np(cudaStream_t s, const MacTableT<NP>& tab, uint64_t coin, const SigmaOut<NP>& so,
                                int sms) {
    const uint64_t units = (tab.rec0[tab.n] + kSigmaAlign - 1) / kSigmaAlign;
    if (units == 0) return cudaSuccess;
    static int per_sm = 0;
    if (per_sm == 0) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mac_sigma<NP>, kThreads, 0) != cudaSuccess ||
            per_sm < 1)
            per_sm = 1;
    }
    const uint64_t cap = (uint64_t)sms * per_sm;
    const int grid = (int)(units < cap ? units : cap);
    if ((units / grid + 1) * kSigmaAlign >= (1ull << 31)) return cudaErrorInvalidValue;  // per-CTA range < 2^31
    k_mac_sigma<NP><<<grid, kThreads, 0, s>>>(tab, coin, so, SigConsts{});
    return launched();
}

cudaError_t launch_mac_sigma(cudaStream_t s, const MacTable& tab, uint64_t coin, uint32_t alpha,
                             unsigned long long* acc, int sms) {
    return mac_sigma_np<1>(s, tab, coin, SigmaOut<1>{{alpha}, {acc}}, sms);
}

cudaError_t launch_mac_sigma2(cudaStream_t s, const MacTableT<2>& tab, uint64_t coin, const uint32_t alpha[2],
                              unsigned long long* const acc[2], int sms) {
    return mac_sigma_np<2>(s, tab, coin, SigmaOut<2>{{alpha[0], alpha[1]}, {acc[0], acc[1]}}, sms);
}

cudaError_t launch_mac_sigma_ranked(cudaStream_t s, const uint32_t* value, const uint32_t* mac,
                                    const uint64_t* rank, uint64_t n, uint64_t coin, uint32_t alpha,
                                    unsigned long long* acc, int sms) {
    if (n == 0) return cudaSuccess;
    k_mac_sigma_ranked<<<grid_for(n, sms), kThreads, 0, s>>>(value, mac, rank, n, coin, alpha, acc);
    return launched();
}

cudaError_t launch_matrix_mask(cudaStream_t s, const uint32_t* wv, const uint32_t* av, uint64_t cells,
                               const uint32_t* xv, const uint32_t* bv, uint32_t din, uint32_t* payload, int sms) {
    // D = W.v - A.v over the tile; E = x.v - B.v (linear.cpp:40-47, value plane)
    IO<2, 1> io_d{{wv, av}, {payload}};
    cudaError_t e = run_map(s, io_d, cells, OpDiff{}, sms);
    if (e != cudaSuccess) return e;
    IO<2, 1> io_e{{xv, bv}, {payload + cells}};
    return run_map(s, io_e, din, OpDiff{}, sms);
}

template <int NP>
static cudaError_t mc_np(cudaStream_t s, uint32_t din, uint32_t rows, uint32_t rpt, const uint32_t* own,
                         const PeerPtrs& peers_dev, const uint32_t* const mt[6], const uint32_t* biasv,
                         const uint32_t* biasm, int party, uint32_t alpha, uint32_t* zv, uint32_t* zm,
                         uint32_t* opened, bool v4, int sms, const uint32_t* alpha_dev) {
    const int grid = (int)(rows < (uint32_t)(sms * 8) ? rows : (uint32_t)(sms * 8));
    if (rows == 0) return cudaSuccess;
    if (v4)
        k_matrix_combine<NP, true><<<grid, kThreads, 0, s>>>(din, rows, rpt, own, peers_dev, mt[0], mt[1], mt[2], mt[3],
                                                             mt[4], mt[5], biasv, biasm, party, alpha, zv, zm, opened,
                                                             alpha_dev);
    else
        k_matrix_combine<NP, false><<<grid, kThreads, 0, s>>>(din, rows, rpt, own, peers_dev, mt[0], mt[1], mt[2], mt[3],
                                                              mt[4], mt[5], biasv, biasm, party, alpha, zv, zm,
                                                              opened, alpha_dev);
    return launched();
}

// `peers` is a HOST array of (device-accessible) peer payload pointers.
cudaError_t launch_matrix_combine(cudaStream_t s, uint32_t din, uint32_t rows, uint32_t rpt, const uint32_t* own,
                                  const uint32_t* const* peers, int n_peers, const uint32_t* const mt[6],
                                  const uint32_t* biasv, const uint32_t* biasm, int party, uint32_t alpha,
                                  uint32_t* zv, uint32_t* zm, uint32_t* opened, int sms, const uint32_t* alpha_dev) {
    const uint64_t cells = (uint64_t)din * rows;
    bool v4 = (din % 4 == 0) && aligned16(own) && aligned16(opened) && aligned16(mt[0]) && aligned16(mt[1]) &&
              aligned16(mt[2]) && aligned16(mt[3]);
    for (int p = 0; p < n_peers; ++p) v4 = v4 && aligned16(peers[p]);
    if (rpt == 0) return cudaErrorInvalidValue;
    (void)cells;
    if (n_peers < 0 || n_peers > kMaxPeers) return cudaErrorInvalidValue;
    PeerPtrs peer_table{};
    for (int p = 0; p < n_peers; ++p) peer_table.p[p] = peers[p];
    switch (n_peers) {
#define CASE(NP) \
    case NP:                                                                                                         \
        return mc_np<NP>(s, din, rows, rpt, own, peer_table, mt, biasv, biasm, party, alpha, zv, zm, opened, v4, sms, \
                         alpha_dev);
        CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7)
#undef CASE
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_matrix_combine2(cudaStream_t s, const MC2Args& a, int sms, unsigned long long* acc_rows,
                                   unsigned int* done_rows) {
    if (a.rows == 0) return cudaSuccess;
    if (a.rpt == 0) return cudaErrorInvalidValue;
    bool v4 = a.din % 4 == 0 && aligned16(a.D0) && aligned16(a.D1) && aligned16(a.opened);
    for (int p = 0; p < 2; ++p)
        v4 = v4 && aligned16(a.A[p][0]) && aligned16(a.A[p][1]) && aligned16(a.B[p][0]) && aligned16(a.B[p][1]);
    static const bool flat_off = std::getenv("SPDZ_MC2_ROWS") != nullptr;  // experiments: the row-per-warp kernel
    static const int unroll = [] {  // SPDZ_MC2_UNROLL=1|2 (experiments; default 2)
        const char* e = std::getenv("SPDZ_MC2_UNROLL");
        return e && std::atoi(e) == 1 ? 1 : 2;
    }();
    if (v4 && acc_rows && done_rows && !flat_off && a.din < (1u << 20)) {  // (the flat kernel's u64 bound)
        auto kern = unroll == 2 ? k_matrix_combine2_flat<2, 2> : k_matrix_combine2_flat<1, 3>;
        static int per_sm[2] = {0, 0};
        int& ps = per_sm[unroll - 1];
        if (!ps) {
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, kern, kThreads, 0) != cudaSuccess || ps < 1) ps = 1;
        }
        const uint64_t units = (uint64_t)(a.din / 4) * a.rows;
        uint64_t grid = (uint64_t)sms * ps;
        const uint64_t need = (units + kThreads - 1) / kThreads;  // small layers: no idle warps
        if (need < grid) grid = need ? need : 1;
        kern<<<(int)grid, kThreads, 0, s>>>(a, acc_rows, done_rows);
        return launched();
    }
    static const int force_g = [] {  // SPDZ_MC2_G=32|256: override the row-group choice (experiments)
        const char* e = std::getenv("SPDZ_MC2_G");
        return e ? std::atoi(e) : 0;
    }();
    const bool warp_rows = force_g ? force_g == 32 : a.rows >= (uint32_t)sms * 8;  // a warp per row fills the GPU
    if (warp_rows) {
        const uint32_t blocks = (a.rows + kThreads / 32 - 1) / (kThreads / 32);
        const int grid = (int)(blocks < (uint32_t)sms * 8 ? blocks : (uint32_t)sms * 8);
        if (v4) k_matrix_combine2<32, true><<<grid, kThreads, 0, s>>>(a);
        else k_matrix_combine2<32, false><<<grid, kThreads, 0, s>>>(a);
    } else {
        const int grid = (int)(a.rows < (uint32_t)sms * 8 ? a.rows : (uint32_t)sms * 8);
        if (v4) k_matrix_combine2<256, true><<<grid, kThreads, 0, s>>>(a);
        else k_matrix_combine2<256, false><<<grid, kThreads, 0, s>>>(a);
    }
    return launched();
}

cudaError_t launch_modgemm(cudaStream_t s, int mode, uint32_t dout, uint32_t din, uint32_t batch,
                           const uint32_t* w0, const uint32_t* w1, const uint32_t* x0, const uint32_t* x1,
                           uint32_t* y0, uint32_t* y1) {
    if (dout == 0 || batch == 0) return cudaSuccess;
    dim3 grid((batch + GT - 1) / GT, (dout + GT - 1) / GT, 2);
    if (mode == 0)  // W public shared by both planes of X
        k_modgemm<<<grid, 256, 0, s>>>(dout, batch, din, w0, w0, x0, x1, y0, y1);
    else  // W secret planes, X public
        k_modgemm<<<grid, 256, 0, s>>>(dout, batch, din, w0, w1, x0, x0, y0, y1);
    return launched();
}

cudaError_t launch_dealer_triples(cudaStream_t s, int n, uint64_t seed, uint64_t draw0, uint32_t alpha,
                                  uint64_t S_total, uint64_t j_first, uint64_t count, uint64_t pstride,
                                  uint32_t* const planes[6], unsigned int* flag, int sms) {
    if (count == 0) return cudaSuccess;
    k_dealer_triples<<<grid_for(count, sms, 16), kThreads, 0, s>>>(n, seed, draw0, alpha, S_total, j_first, count,
                                                                    pstride, planes[0], planes[1], planes[2],
                                                                    planes[3], planes[4], planes[5], flag);
    return launched();
}

cudaError_t launch_dealer_share(cudaStream_t s, int n, uint64_t seed, uint64_t draw0, uint32_t alpha,
                                const uint32_t* clear, uint64_t lanes, uint32_t* vals, uint32_t* macs,
                                uint64_t pstride, unsigned int* flag, int sms) {
    if (lanes == 0) return cudaSuccess;
    k_dealer_share<<<grid_for(lanes, sms, 16), kThreads, 0, s>>>(n, seed, draw0, alpha, clear, lanes, vals, macs,
                                                                  pstride, flag);
    return launched();
}

cudaError_t launch_dealer_uniform(cudaStream_t s, uint64_t seed, uint64_t draw0, uint64_t count, uint64_t,
                                  uint32_t* out, unsigned int* flag, int sms) {
    if (count == 0) return cudaSuccess;
    k_dealer_uniform<<<grid_for(count, sms, 16), kThreads, 0, s>>>(seed, draw0, count, out, flag);
    return launched();
}

cudaError_t launch_dealer_matvec(cudaStream_t s, const uint32_t* A, const uint32_t* B, uint32_t din, uint32_t rows,
                                 uint32_t* C) {
    if (rows == 0) return cudaSuccess;
    k_dealer_matvec<<<rows < 4096 ? rows : 4096, kThreads, 0, s>>>(A, B, din, rows, C);
    return launched();
}

cudaError_t launch_dealer_masks(cudaStream_t s, int n, uint64_t seed, uint64_t draw0, uint32_t alpha,
                                uint64_t m_first, uint64_t count, uint64_t pstride, uint32_t* vals, uint32_t* macs,
                                uint32_t* clear, unsigned int* flag, int sms) {
    if (count == 0) return cudaSuccess;
    k_dealer_masks<<<grid_for(count, sms, 16), kThreads, 0, s>>>(n, seed, draw0, alpha, m_first, count, pstride,
                                                                  vals, macs, clear, flag);
    return launched();
}

cudaError_t launch_pub_binop(cudaStream_t s, int op, const uint32_t* a, bool a_bcast, const uint32_t* b, bool b_bcast,
                             uint32_t* out, uint64_t n, int sms) {
    if (n == 0) return cudaSuccess;
    k_pub_binop<<<grid_for(n, sms), kThreads, 0, s>>>(op, a, a_bcast, b, b_bcast, out, n);
    return launched();
}

cudaError_t launch_bcast(cudaStream_t s, const uint32_t* sv, const uint32_t* sm, uint32_t* ov, uint32_t* om,
                         uint64_t n, int sms) {
    if (n == 0) return cudaSuccess;
    k_bcast2<<<grid_for(n, sms), kThreads, 0, s>>>(sv, sm, ov, om, n);
    return launched();
}

cudaError_t launch_tile_e(cudaStream_t s, const uint32_t* xv, const uint32_t* bv, uint32_t din, uint32_t n_tiles,
                          uint32_t* out, int sms) {
    const uint64_t total = (uint64_t)din * n_tiles;
    if (total == 0) return cudaSuccess;
    k_tile_e<<<grid_for(total, sms), kThreads, 0, s>>>(xv, bv, din, total, out);
    return launched();
}

cudaError_t launch_linear_mask2(cudaStream_t s, const LinMask2Args& m, int sms) {
    bool ok = m.din % 4 == 0 && m.cells % 4 == 0;
    for (int p = 0; p < 2; ++p)
        ok = ok && aligned16(m.w[p]) && aligned16(m.a[p]) && aligned16(m.x[p]) && aligned16(m.b[p]) && aligned16(m.pay[p]);
    ok = ok && aligned16(m.opened_e);
    if (!ok) return cudaErrorInvalidValue;  // caller falls back to the per-plane kernels
    const uint64_t total = m.cells / 4 + (uint64_t)m.din * m.ntiles / 4;
    if (total == 0) return cudaSuccess;
    k_linear_mask2<<<grid_for(total, sms), kThreads, 0, s>>>(m);
    return launched();
}

cudaError_t launch_set_word(cudaStream_t s, uint32_t* p, uint32_t v) {
    k_set_word<<<1, 32, 0, s>>>(p, v);
    return launched();
}

cudaError_t launch_xor_word(cudaStream_t s, uint32_t* p, uint32_t mask) {
    k_xor_word<<<1, 32, 0, s>>>(p, mask);
    return launched();
}

}  // namespace spdzb200
