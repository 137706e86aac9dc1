// Kernel launchers of the B200 SPDZ back end (sm_100a).  Every launcher is
// asynchronous on `stream` and returns cudaGetLastError() of its launch.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

namespace spdzb200 {

constexpr int kMaxPeers = 7;

// Device-side MAC segment descriptor for NP parties whose logs share every record's
// rank (same lengths, same j0): the coefficient stream is computed once for all of them.
template <int NP>
struct MacSegT {
    const uint32_t* value[NP];
    const uint32_t* mac_a[NP];
    const uint32_t* mac_b[NP];  // may be null (then for every party)
    uint64_t len;
    uint64_t j0;
};
constexpr uint32_t kSigmaAlign = 1024;     // CTA record ranges start at multiples of this
constexpr int kMacTableSegs = 384;         // segments per launch (kernel parameter table, < 32 KB for NP = 2)
template <int NP>
struct MacTableT {
    uint32_t n;                            // segments in this table
    MacSegT<NP> seg[kMacTableSegs];
    uint64_t rec0[kMacTableSegs + 1];      // first record of each segment (prefix sums), rec0[n] = total
};
using MacSegDev = MacSegT<1>;
using MacTable = MacTableT<1>;

struct LaunchInfo {
    int sm_count = 148;
};

extern std::atomic<unsigned long long> g_kernel_launches;  // evidence counter (calls may be concurrent)

// elementwise (backend.cpp:25-51, spdz.cpp:35-75)
// both co-located parties: xy = x0.v x0.m y0.v y0.m x1.v x1.m y1.v y1.m, z = z0.v z0.m z1.v z1.m
cudaError_t launch_add_sub2(cudaStream_t s, bool sub, const uint32_t* const xy[8], uint32_t* const z[4], uint64_t n,
                            int sms);
// launch_add_sub2 plus the add / sub consuming its result (sm2: 0 w2 = w + o, 1 w - o, 2 o - w; o =
// o0.v o0.m o1.v o1.m; w = w2 of both parties) and, with out (both parties' outputs), its root opening
cudaError_t launch_add_sub2_chain(cudaStream_t s, bool sub, const uint32_t* const xy[8], uint32_t* const z[4], int sm2,
                                  const uint32_t* const o[4], uint32_t* const w[4], uint32_t* const out[2], uint64_t n,
                                  int sms);
cudaError_t launch_add_sub(cudaStream_t s, bool sub, const uint32_t* xv, const uint32_t* xm, const uint32_t* yv,
                           const uint32_t* ym, uint32_t* zv, uint32_t* zm, uint64_t n, int sms);
// op: 0 add_public 1 sub_public 2 rsub_public 3 mul_public 4 share_of_public (xv/xm unused as inputs)
// alpha_dev (optional): read alpha from device memory instead of the `alpha` argument
// (kernels captured in a CUDA graph stay valid when the MAC key share changes)
cudaError_t launch_public(cudaStream_t s, int op, const uint32_t* xv, const uint32_t* xm, const uint32_t* k,
                          bool k_bcast, uint32_t k_imm, bool k_is_imm, int party, uint32_t alpha, uint32_t* zv,
                          uint32_t* zm, uint64_t n, int sms, const uint32_t* alpha_dev = nullptr);
// backend.cpp:53-65
cudaError_t launch_mul_mask(cudaStream_t s, const uint32_t* xv, const uint32_t* yv, const uint32_t* av,
                            const uint32_t* bv, uint32_t* d, uint32_t* e, uint64_t n, int sms);
// both co-located parties' masks in one pass: xyab = {x0.v y0.v a0.v b0.v x1.v y1.v a1.v b1.v},
// de = {d0 e0 d1 e1}
cudaError_t launch_mul_mask2(cudaStream_t s, const uint32_t* const xyab[8], uint32_t* const de[4], uint64_t n,
                             int sms);
// spdz.cpp:77-96 fused with the open of net.cpp:170-215: d = own_d + sum reduce(peer_d) ...
cudaError_t launch_beaver_combine(cudaStream_t s, const uint32_t* own_d, const uint32_t* own_e,
                                  const uint32_t* const* peer_d, const uint32_t* const* peer_e, int n_peers,
                                  const uint32_t* const tri[6], int party, uint32_t alpha, uint32_t* zv, uint32_t* zm,
                                  uint32_t* open_d, uint32_t* open_e, uint64_t n, int sms,
                                  const uint32_t* alpha_dev = nullptr);
cudaError_t launch_set_word(cudaStream_t s, uint32_t* p, uint32_t v);
// Both parties' matrix combine (spdz.cpp:98-124) in one pass on one GPU (kernels.cu MC2Args).
struct MC2Args {
    uint32_t din, rows, rpt;
    const uint32_t* D0;
    const uint32_t* D1;
    const uint32_t* A[2][2];
    const uint32_t* B[2][2];
    const uint32_t* Cc[2][2];
    const uint32_t* bias[2][2];
    uint32_t alpha[2];
    const uint32_t* alpha_dev[2];  // optional: alpha_i read from device memory (CUDA-graph safe)
    uint32_t* z[2][2];
    uint32_t* opened;
    uint32_t* open_out[2];  // optional: both parties' opened z.v (the layer is the circuit's root)
};
// acc_rows (5 u64 per row) / done_rows (u32 per row): zeroed scratch for the balanced kernel
// (left zeroed); null selects the warp-per-row kernel
cudaError_t launch_matrix_combine2(cudaStream_t s, const MC2Args& a, int sms, unsigned long long* acc_rows = nullptr,
                                   unsigned int* done_rows = nullptr);
// Input sharing for both parties of a 2-party run on one GPU: mask = {v0, m0, v1, m1}
// input-mask shares, out = {v0, m0, v1, m1} input shares (preproc.cpp:205-243).
cudaError_t launch_share_input2(cudaStream_t s, const uint32_t* x_raw, const uint32_t* r_clear,
                                const uint32_t* const mask[4], const uint32_t alpha[2],
                                const uint32_t* const alpha_dev[2], uint32_t* const out[4], uint64_t n, int sms);
// Both parties of a 2-party run on one GPU: de = {d0, e0, d1, e1} payload halves, z = {z0.v,
// z0.m, z1.v, z1.m}; the opened d, e (one copy, identical for both parties) -> open_d/open_e.
// launch_beaver_combine2 plus the private add / sub that consumes the products (sm: 0 w = z + o,
// 1 w = z - o, 2 w = o - z; addin = o.v o.m of party 0, party 1; w = w.v w.m of party 0, party 1) and
// then nx: 0 nothing, 1-3 the mask of the multiply consuming w (w left / right / both; next as in
// launch_beaver_combine2_mask, extra = d'0 e'0 d'1 e'1), 4 the root opening of w (extra = both
// parties' opened outputs)
cudaError_t launch_beaver_combine2_add(cudaStream_t s, const uint32_t* const de[4], const uint32_t* const tri0[6],
                                       const uint32_t* const tri1[6], const uint32_t alpha[2],
                                       const uint32_t* const alpha_dev[2], uint32_t* const z[4], uint32_t* open_d,
                                       uint32_t* open_e, int sm, const uint32_t* const addin[4], uint32_t* const w[4],
                                       int nx, const uint32_t* const next[6], uint32_t* const extra[4], uint64_t n,
                                       int sms);
// launch_beaver_combine of one party of a 2-party run (one peer) plus the private add / sub that
// consumes the product (sm, addin = o.v o.m, w = w.v w.m) and nx 0 nothing / 1-3 the mask of the
// multiply consuming its result (next = other operand .v, a'.v, b'.v; next_de = d', e')
cudaError_t launch_beaver_combine_add(cudaStream_t s, const uint32_t* own_d, const uint32_t* own_e,
                                      const uint32_t* peer_d, const uint32_t* peer_e, const uint32_t* const tri[6],
                                      int party, uint32_t alpha, uint32_t* zv, uint32_t* zm, uint32_t* open_d,
                                      uint32_t* open_e, int sm, const uint32_t* const addin[2], uint32_t* const w[2],
                                      int nx, const uint32_t* const next[3], uint32_t* const next_de[2], uint64_t n,
                                      int sms, const uint32_t* alpha_dev);
// launch_beaver_combine (1-3 peers) plus the next multiply's mask from this party's fresh product
// (zpos as launch_beaver_combine2_mask; next = other operand .v (unused for zpos 2), a'.v, b'.v;
// next_de = d', e')
cudaError_t launch_beaver_combine_mask(cudaStream_t s, const uint32_t* own_d, const uint32_t* own_e,
                                       const uint32_t* const* peer_d, const uint32_t* const* peer_e, int n_peers,
                                       const uint32_t* const tri[6], int party, uint32_t alpha, uint32_t* zv,
                                       uint32_t* zm, uint32_t* open_d, uint32_t* open_e, int zpos,
                                       const uint32_t* const next[3], uint32_t* const next_de[2], uint64_t n, int sms,
                                       const uint32_t* alpha_dev);
// launch_beaver_combine2 plus the next multiply's mask from the fresh products (zpos: the next
// multiply's operand that is this product — 0 left, 1 right, 2 both; next[3p..3p+2] = party p's other
// operand .v (unused for zpos 2), a'.v, b'.v; next_de = d'0 e'0 d'1 e'1).  zpos 3: the product is the
// root — next unused, next_de[0..1] = both parties' opened outputs.
cudaError_t launch_beaver_combine2_mask(cudaStream_t s, const uint32_t* const de[4], const uint32_t* const tri0[6],
                                        const uint32_t* const tri1[6], const uint32_t alpha[2],
                                        const uint32_t* const alpha_dev[2], uint32_t* const z[4], uint32_t* open_d,
                                        uint32_t* open_e, int zpos, const uint32_t* const next[6],
                                        uint32_t* const next_de[4], uint64_t n, int sms);
cudaError_t launch_beaver_combine2(cudaStream_t s, const uint32_t* const de[4], const uint32_t* const tri0[6],
                                   const uint32_t* const tri1[6], const uint32_t alpha[2],
                                   const uint32_t* const alpha_dev[2], uint32_t* const z[4], uint32_t* open_d,
                                   uint32_t* open_e, uint64_t n, int sms);
// net.cpp:170-215
cudaError_t launch_open_sum(cudaStream_t s, const uint32_t* own, const uint32_t* const* peers, int n_peers,
                            uint32_t* out, uint64_t n, int sms);
// backend.cpp:76-84; result folded into acc[0..1] (u64, values < p each) — caller zeroes acc.
cudaError_t launch_reduce_add(cudaStream_t s, const uint32_t* xv, const uint32_t* xm, uint64_t n,
                              unsigned long long* acc, int sms);
// acc (2 x u64) -> out[0] = acc[0] mod p, out[1] = acc[1] mod p
cudaError_t launch_finish_reduce(cudaStream_t s, const unsigned long long* acc, uint32_t* outv, uint32_t* outm);
// pairwise gather for reduce_mul (runtime.cpp:246-255): xs = cur[2i], ys = cur[2i+1]
cudaError_t launch_pair_split(cudaStream_t s, const uint32_t* cv, const uint32_t* cm, uint64_t pairs, uint32_t* xv,
                              uint32_t* xm, uint32_t* yv, uint32_t* ym, int sms);
// MAC sigma partial over chunks; acc (u64) accumulates values < p per block.
cudaError_t launch_mac_sigma(cudaStream_t s, const MacTable& tab, uint64_t coin, uint32_t alpha,
                             unsigned long long* acc, int sms);
// Two parties' sigma partials in one pass (shared coefficients): acc[p] += party p's partial.
cudaError_t launch_mac_sigma2(cudaStream_t s, const MacTableT<2>& tab, uint64_t coin, const uint32_t alpha[2],
                              unsigned long long* const acc[2], int sms);
// MAC sigma over explicit ranks (record form)
cudaError_t launch_mac_sigma_ranked(cudaStream_t s, const uint32_t* value, const uint32_t* mac,
                                    const uint64_t* rank, uint64_t n, uint64_t coin, uint32_t alpha,
                                    unsigned long long* acc, int sms);

// linear layer (linear.cpp:30-61, spdz.cpp:98-124)
cudaError_t launch_matrix_mask(cudaStream_t s, const uint32_t* wv, const uint32_t* av, uint64_t cells,
                               const uint32_t* xv, const uint32_t* bv, uint32_t din, uint32_t* payload, int sms);
// Layer-level: rows = all rows of the layer, tiles of `rpt` rows (last may be
// short); A (rows x din), B (n_tiles x din), C (rows); opened = [D (rows*din) |
// E (n_tiles*din)] with E already opened.  One CTA per row.
cudaError_t launch_matrix_combine(cudaStream_t s, uint32_t din, uint32_t rows, uint32_t rpt, const uint32_t* own,
                                  const uint32_t* const* peers, int n_peers, const uint32_t* const mt[6],
                                  const uint32_t* biasv, const uint32_t* biasm, int party, uint32_t alpha,
                                  uint32_t* zv, uint32_t* zm, uint32_t* opened, int sms,
                                  const uint32_t* alpha_dev = nullptr);
// Both co-located parties' linear mask: pay_p = [W_p.v - A_p.v (cells) | x_p.v - B_p.v[t] (t < ntiles)].
// Needs din % 4 == 0 and 16-byte aligned planes (else cudaErrorInvalidValue: use the per-plane kernels).
struct LinMask2Args {
    const uint32_t* w[2];
    const uint32_t* a[2];
    const uint32_t* x[2];
    const uint32_t* b[2];
    uint32_t* pay[2];
    uint64_t cells;
    uint32_t din, ntiles;
    uint32_t* opened_e;  // optional: the opened E (E_0 + E_1, every tile) written in the same pass
};
// both co-located parties' opened words z0 + z1 (the root open) in one pass
cudaError_t launch_open_sum2(cudaStream_t s, const uint32_t* z0, const uint32_t* z1, uint32_t* out0, uint32_t* out1,
                             uint64_t n, int sms);
cudaError_t launch_linear_mask2(cudaStream_t s, const LinMask2Args& m, int sms);
// E_t = x - B_t for all tiles (B: n_tiles x din)
cudaError_t launch_tile_e(cudaStream_t s, const uint32_t* xv, const uint32_t* bv, uint32_t din, uint32_t n_tiles,
                          uint32_t* out, int sms);
// runtime.cpp:303-334 batched: Y (dout x batch) = W (dout x din) * X (din x batch), two planes.
//   mode 0: W public (w0), X secret planes (x0 vals, x1 macs) -> y0 = W x0, y1 = W x1
//   mode 1: W secret (w0 vals, w1 macs), X public (x0)        -> y0 = w0 X, y1 = w1 X
cudaError_t launch_modgemm(cudaStream_t s, int mode, uint32_t dout, uint32_t din, uint32_t batch,
                           const uint32_t* w0, const uint32_t* w1, const uint32_t* x0, const uint32_t* x1,
                           uint32_t* y0, uint32_t* y1);

// tcgen05 kind::i8 limb GEMM (gemm_tc.cu); scratch >= modgemm_tc_scratch_bytes()
uint64_t modgemm_tc_scratch_bytes(int mode, uint32_t dout, uint32_t din, uint32_t batch);
bool modgemm_tc_supported(uint32_t din);
// Optional extras of the tcgen05 GEMM: mode-0 right operand X_h + coef_h * e (e: din x batch),
// and an addend (planes laid out like y, may alias y): y = add + W X.
struct TcAux {
    const uint32_t* e = nullptr;
    uint32_t coef0 = 0, coef1 = 0;
    const uint32_t* add0 = nullptr;
    const uint32_t* add1 = nullptr;
    const uint8_t* a_image = nullptr;  // prepared A limb image (launch_tile_a): skip its re-layout
};
uint64_t modgemm_tc_a_image_bytes(int mode, uint32_t dout, uint32_t din);
cudaError_t launch_tile_a(cudaStream_t s, int mode, uint32_t dout, uint32_t din, const uint32_t* w0,
                          const uint32_t* w1, uint8_t* image, int sms);
cudaError_t launch_modgemm_tc(cudaStream_t s, int mode, uint32_t dout, uint32_t din, uint32_t batch,
                              const uint32_t* w0, const uint32_t* w1, const uint32_t* x0, const uint32_t* x1,
                              uint32_t* y0, uint32_t* y1, uint8_t* scratch, int sms, const TcAux* aux = nullptr);

// GPU dealer (spdz.cpp:162-249), closed-form splitmix64 stream.
// lanes [j_first, j_first+count) of Dealer::triples(S_total); party p's share of
// local lane j at planes[k][p * pstride + j]
cudaError_t launch_dealer_triples(cudaStream_t s, int n, uint64_t seed, uint64_t draw0, uint32_t alpha,
                                  uint64_t S_total, uint64_t j_first, uint64_t count, uint64_t pstride,
                                  uint32_t* const planes[6], unsigned int* reject_flag, int sms);
cudaError_t launch_dealer_share(cudaStream_t s, int n, uint64_t seed, uint64_t draw0, uint32_t alpha,
                                const uint32_t* clear, uint64_t lanes, uint32_t* vals, uint32_t* macs,
                                uint64_t pstride, unsigned int* reject_flag, int sms);
cudaError_t launch_dealer_uniform(cudaStream_t s, uint64_t seed, uint64_t draw0, uint64_t count, uint64_t stride,
                                  uint32_t* out, unsigned int* reject_flag, int sms);
cudaError_t launch_dealer_matvec(cudaStream_t s, const uint32_t* A, const uint32_t* B, uint32_t din, uint32_t rows,
                                 uint32_t* C);
// masks [m_first, m_first+count); party p's share of local mask j at [p * pstride + j]
cudaError_t launch_dealer_masks(cudaStream_t s, int n, uint64_t seed, uint64_t draw0, uint32_t alpha,
                                uint64_t m_first, uint64_t count, uint64_t pstride, uint32_t* vals, uint32_t* macs,
                                uint32_t* clear, unsigned int* reject_flag, int sms);

// cleartext lane op (0 add 1 sub 2 mul) with scalar broadcast of either side
cudaError_t launch_pub_binop(cudaStream_t s, int op, const uint32_t* a, bool a_bcast, const uint32_t* b, bool b_bcast,
                             uint32_t* out, uint64_t n, int sms);
// out[i] = src[0] (either plane pointer may be null for the MAC plane)
cudaError_t launch_bcast(cudaStream_t s, const uint32_t* sv, const uint32_t* sm, uint32_t* ov, uint32_t* om,
                         uint64_t n, int sms);

// payload fault injection (test hook, net.cpp:241-278 BitFlip)
cudaError_t launch_xor_word(cudaStream_t s, uint32_t* p, uint32_t mask);

}  // namespace spdzb200
