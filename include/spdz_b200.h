/*
 * spdz_b200.h — C ABI of the B200-native SPDZ online-phase back end.
 *
 * This is the drop-in boundary for the reference's back-end plugin
 * `mpc::backend::Backend` (/root/reference/proj/core/include/mpc/backend.hpp:32-49),
 * widened (SURVEY.md §8b "gaps to close") to the other online-phase ops that
 * bypass `Backend` in the reference: public-constant ops (spdz.hpp:131-141),
 * open/reveal (net.hpp:77-81 / net.cpp:61-111), the MAC check
 * (spdz.hpp:168-176, runtime.cpp:467-506) and the linear layer
 * (linear.hpp:248-265, runtime.cpp:283-358).
 *
 * Conventions
 *  - Plain pointers and sizes; no C++ or torch types cross this boundary.
 *  - Field F_p, p = 2^32 - 5 (field.hpp:10).  Elements are uint32 in [0, p).
 *  - Share vectors are structure-of-arrays: one value plane + one MAC plane
 *    (spdz.hpp:19-28).  `spdz_share_t` points at DEVICE memory.
 *  - Device entry points are asynchronous on the context's CUDA stream and
 *    never allocate on the hot path; caller owns every buffer.
 *  - `spdz_host_*` entry points take HOST buffers (the exact call shape of the
 *    reference's `Backend` virtuals) and copy in/out inside the call.
 *  - Every function returns an `spdz_status` (0 = OK).  `spdz_last_error()`
 *    returns the thread-local message; codes map 1:1 onto the reference's
 *    exception types (listed per code).
 *  - A context is owned by one party; distinct contexts may be driven from
 *    distinct threads concurrently (kernels are pure).  One
 *    context is driven by one thread at a time (its stream, staging buffers and
 *    accumulators are not locked), except spdz_mac_log_append (locked).
 *  - A run (spdz_run_*) is driven by one thread at a time; distinct runs, and
 *    distinct meshes (spdz_net_*), may live on distinct threads.
 */
#ifndef SPDZ_B200_H
#define SPDZ_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPDZ_PRIME 4294967291u /* field.hpp:10 */
#define SPDZ_MAX_PARTIES 8

typedef enum spdz_status {
    SPDZ_OK = 0,
    SPDZ_ERR_LANE_MISMATCH = 1,          /* backend::LaneMismatch        backend.hpp:11 */
    SPDZ_ERR_TRIPLE_SHORTAGE = 2,        /* backend::TripleShortage      backend.hpp:14 */
    SPDZ_ERR_BACKEND_UNAVAILABLE = 3,    /* backend::BackendUnavailable  backend.hpp:17 */
    SPDZ_ERR_TRIPLE_EXHAUSTED = 4,       /* spdz::TripleExhausted        triple_store.hpp:14 */
    SPDZ_ERR_TRIPLE_SHAPE_MISMATCH = 5,  /* spdz::TripleShapeMismatch    triple_store.hpp:17 */
    SPDZ_ERR_MASK_EXHAUSTED = 6,         /* spdz::MaskExhausted          triple_store.hpp:20 */
    SPDZ_ERR_PEER_TIMEOUT = 7,           /* net::PeerTimeout             net.hpp:25 */
    SPDZ_ERR_LANE_COUNT_MISMATCH = 8,    /* net::LaneCountMismatch       net.hpp:31 */
    SPDZ_ERR_MALFORMED_SHARE_MESSAGE = 9,/* net::MalformedShareMessage   net.hpp:34 */
    SPDZ_ERR_MAC_CHECK_FAILED = 10,      /* spdz::MacCheckFailed         spdz.hpp:12 */
    SPDZ_ERR_SLICE_TOO_SMALL = 11,       /* linear::SliceTooSmall        linear.hpp:10 */
    SPDZ_ERR_STORE_FORMAT = 12,          /* spdz::StoreFormatError       triple_store.hpp:23 */
    SPDZ_ERR_INSUFFICIENT_TRIPLES = 13,  /* preproc::InsufficientTriples preproc.cpp:182-201 */
    SPDZ_ERR_NET = 14,                   /* net::NetError / ConnectTimeout / IndexCollision net.hpp:19-30
                                            (the message starts with the type's name) */
    SPDZ_ERR_INVALID_ARGUMENT = 20,
    SPDZ_ERR_CUDA = 21,
    SPDZ_ERR_DEALER_REJECTION = 22,      /* GPU dealer hit the 25/2^64 rejection branch */
} spdz_status;

/* One party's authenticated share of a lane vector (spdz.hpp:19-28), device memory. */
typedef struct spdz_share {
    uint32_t* vals;
    uint32_t* macs;
    uint64_t lanes;
} spdz_share_t;

/* Beaver triple shares (spdz.hpp:31-33). */
typedef struct spdz_triple {
    spdz_share_t a, b, c;
} spdz_triple_t;

/* Matrix triple for one linear-layer tile (spdz.hpp:35-43): A rows x din
 * (row-major), B din, C rows. */
typedef struct spdz_mtriple {
    uint32_t din, rows;
    spdz_share_t a, b, c;
} spdz_mtriple_t;

/* Batched matrix triple: the batch-N generalisation of one tile's triple
 * (spdz.hpp:35-43) for W (dout x din) times a secret X (din x batch): A dout x din,
 * B din x batch, C = A B dout x batch, all row-major.  Column j of (B, C) with A is an
 * ordinary matrix triple {A, B[:,j], C[:,j]}. */
typedef struct spdz_bmtriple {
    uint32_t din, dout, batch;
    spdz_share_t a, b, c;
} spdz_bmtriple_t;

/* Backend capability record (backend.hpp:21-27). */
typedef struct spdz_capability {
    char name[32];
    uint64_t min_kernel_size; /* 1: the GPU back end takes every request (no CPU fallback) */
    uint32_t threads_per_block;
    int32_t executable;
    int32_t sm_count;
    int32_t device;
} spdz_capability_t;

/* One contiguous run of opened records for the MAC check.  Record i of the
 * segment is (opened x = value[i], mac share m = mac_a[i] - mac_b[i] (mac_b may
 * be NULL), global rank j = j0 + i).  The rank is the record's position in
 * (batch_id, lane) order over the whole run (spdz.cpp:127-129); the host
 * assigns j0 by sorting segments by batch id (spdz_mac_assign_ranks). */
typedef struct spdz_mac_segment {
    const uint32_t* value;
    const uint32_t* mac_a;
    const uint32_t* mac_b;
    uint64_t len;
    uint64_t j0;       /* global rank of record 0 (filled by spdz_mac_assign_ranks) */
    uint64_t batch_id; /* wire batch id of the opening (runtime.cpp:22-24) */
    uint64_t lane0;    /* lane of record 0 inside its batch (log_open lane, runtime.cpp:115-116) */
    uint64_t batch_len;/* records of the whole batch across all shards (0: infer from the local segments) */
} spdz_mac_segment_t;

typedef struct spdz_ctx spdz_ctx;

/* ---------------- library / context ---------------- */
const char* spdz_last_error(void);
const char* spdz_version(void);
/* Creates a party context on `device` (cudaSetDevice'd on every entry). */
int spdz_ctx_create(int device, int party, int n_parties, uint32_t alpha_share, spdz_ctx** out);
int spdz_ctx_destroy(spdz_ctx* ctx);
/* Launch on an external CUDA stream (cudaStream_t passed as void*; NULL = the
 * legacy default stream), e.g. the caller's framework stream. */
int spdz_ctx_set_stream(spdz_ctx* ctx, void* stream);
/* Back to the context's own non-blocking stream (the default after create). */
int spdz_ctx_use_own_stream(spdz_ctx* ctx);
void* spdz_ctx_stream(spdz_ctx* ctx);
int spdz_ctx_party(const spdz_ctx* ctx);
int spdz_ctx_sync(spdz_ctx* ctx);
/* backend.hpp:35 */
int spdz_capability(const spdz_ctx* ctx, spdz_capability_t* out);
/* Measured CUDA-core integer pipe rate on ctx's device: IMAD.WIDE.U32 per second
 * (the roofline denominator of the CUDA-core modular GEMM) and all integer ops/s. */
int spdz_diag_imad_wide_rate(spdz_ctx* ctx, double* wide_per_s, double* total_int_per_s);
/* Diagnostic: out[2i] = a representative < 2^32 of in[i] mod p, out[2i+1] = one of
 * splitmix64-finaliser(in[i]) mod p (the MAC-check coefficient arithmetic of k_mac_sigma);
 * device pointers, synchronous. */
int spdz_diag_rep_check(spdz_ctx* ctx, const uint64_t* d_in, uint64_t n, uint32_t* d_out);
/* Diagnostic switches of the tcgen05 GEMM: bit 2 skips the GEMM kernel, bit 3 the operand
 * re-layout (results invalid while either is set); bit 6 / bit 7 force the 32- / 64-column
 * output tile (results valid).  Attribution experiments and tests only. */
int spdz_diag_gemm_tc_flags(uint32_t flags);
/* Diagnostic timeline of the tcgen05 GEMM kernel: when dev_buf (device memory, 8 u64 per
 * CTA) is set, every CTA writes %globaltimer at entry, after setup, after the dependent-launch
 * wait, at its first full stage, after its last MMA commit, when the epilogue gets the
 * accumulators, after its stores and at exit.  NULL switches it off. */
int spdz_diag_gemm_tc_timeline(void* dev_buf);
/* Number of kernels this library launched on any context since load (evidence counter). */
uint64_t spdz_kernel_launches(void);

/* ---------------- device buffers and completion events ----------------
 * SoA share buffers in HBM and stream-ordered copies (host buffers must stay valid, and
 * unchanged, until an event recorded after the copy has completed); events let a
 * caller's pump loop poll completion without blocking (runtime.cpp:452-465). */
int spdz_share_alloc(spdz_ctx* ctx, uint64_t lanes, spdz_share_t* out);
int spdz_share_free(spdz_ctx* ctx, spdz_share_t* s);
int spdz_share_upload(spdz_ctx* ctx, spdz_share_t* dst, const uint32_t* host_vals, const uint32_t* host_macs,
                      uint64_t lanes);
int spdz_share_download(spdz_ctx* ctx, const spdz_share_t* src, uint32_t* host_vals, uint32_t* host_macs,
                        uint64_t lanes);
typedef struct spdz_event spdz_event;
int spdz_event_record(spdz_ctx* ctx, spdz_event** out);   /* records on ctx's stream */
int spdz_event_query(spdz_event* ev, int* done);          /* non-blocking: *done = 1 when complete */
int spdz_event_sync(spdz_event* ev);
int spdz_event_wait(spdz_ctx* ctx, spdz_event* ev);       /* ctx's stream waits for ev (other party / device) */
int spdz_event_destroy(spdz_event* ev);

/* ---------------- Backend: batched share ops (device) ---------------- */
/* backend.hpp:37 / backend.cpp:25-37: z = x + y on both planes */
int spdz_add_batch(spdz_ctx* ctx, const spdz_share_t* x, const spdz_share_t* y, spdz_share_t* z);
/* backend.hpp:38 / backend.cpp:39-51 */
int spdz_sub_batch(spdz_ctx* ctx, const spdz_share_t* x, const spdz_share_t* y, spdz_share_t* z);
/* backend.hpp:39-42 / backend.cpp:53-65: d = x.v - a.v, e = y.v - b.v (value planes only) */
int spdz_mul_mask(spdz_ctx* ctx, const spdz_share_t* x, const spdz_share_t* y, const spdz_triple_t* t,
                  uint32_t* d_out, uint32_t* e_out);
/* backend.hpp:43-46 / spdz.cpp:77-96 with already-opened d, e */
int spdz_mul_combine(spdz_ctx* ctx, const spdz_triple_t* t, const uint32_t* d, const uint32_t* e,
                     spdz_share_t* z);
/* backend.hpp:47-48 / backend.cpp:76-84: z (1 lane) = sum of lanes, both planes */
int spdz_reduce_add(spdz_ctx* ctx, const spdz_share_t* x, spdz_share_t* z);

/* ---------------- public-constant ops (spdz.cpp:35-75), in place ----------------
 * `k` is a device vector of x->lanes elements, or of 1 element broadcast over
 * the lanes (runtime.cpp:36-39). */
int spdz_add_public(spdz_ctx* ctx, spdz_share_t* x, const uint32_t* k, uint64_t k_len);
int spdz_sub_public(spdz_ctx* ctx, spdz_share_t* x, const uint32_t* k, uint64_t k_len);
int spdz_rsub_public(spdz_ctx* ctx, spdz_share_t* x, const uint32_t* k, uint64_t k_len);
int spdz_mul_public(spdz_ctx* ctx, spdz_share_t* x, const uint32_t* k, uint64_t k_len);
int spdz_mul_public_scalar(spdz_ctx* ctx, spdz_share_t* x, uint32_t k);
/* spdz.cpp:70-75: out = trivial sharing of public k (out->lanes lanes) */
int spdz_share_of_public(spdz_ctx* ctx, const uint32_t* k, uint64_t k_len, spdz_share_t* out);

/* ---------------- open / reveal (net.cpp:61-111, absorb 170-215) ----------------
 * out[i] = own[i] + sum_p reduce(peers[p][i]) mod p.  Peer pointers may be on
 * this device, on a peer device (P2P over NVLink) or IPC-mapped. */
int spdz_open_sum(spdz_ctx* ctx, const uint32_t* own, const uint32_t* const* peers, int n_peers, uint64_t len,
                  uint32_t* out);

/* Fused Beaver open + combine: opened [d|e] = own_de + sum reduce(peer_de), then
 * z = beaver_combine(t, d, e) (spdz.cpp:77-96).  `own_de`/`peer_de[p]` are the
 * [d | e] payloads (2*lanes words, runtime.cpp:215-217).  If `opened_out` is not
 * NULL the opened [d|e] is written there (the MAC log, runtime.cpp:224). */
int spdz_beaver_open_combine(spdz_ctx* ctx, const spdz_triple_t* t, const uint32_t* own_de,
                             const uint32_t* const* peer_de, int n_peers, spdz_share_t* z,
                             uint32_t* opened_out);

/* ---------------- MAC check (spdz.cpp:126-158, runtime.cpp:467-506) ---------------- */
/* Assigns j0 to each segment: j0 = (records of all smaller batch ids) + lane0
 * (host only). */
int spdz_mac_assign_ranks(spdz_mac_segment_t* segs, uint64_t n_segs);
/* sigma_i = sum_j r_j (m_ij - alpha_i x_j) mod p over the segments (device
 * arrays referenced by host-side descriptors); blocks until the result is on the host. */
int spdz_mac_sigma(spdz_ctx* ctx, const spdz_mac_segment_t* segs, uint64_t n_segs, uint64_t coin,
                   uint32_t* sigma_out);
/* spdz.hpp:168 record form: records in any order (device SoA arrays); ranks are
 * assigned by sorting (batch_id, lane) on the host (compat path). */
int spdz_mac_sigma_records(spdz_ctx* ctx, const uint64_t* host_batch, const uint32_t* host_lane,
                           const uint32_t* dev_value, const uint32_t* dev_mac, uint64_t n, uint64_t coin,
                           uint32_t* sigma_out);
/* The log itself, kept in the context for a caller-driven runtime (log_open,
 * runtime.cpp:112-117, and mac_check, runtime.cpp:467-506): append each opening's
 * device arrays as it completes (from any thread; a batch may arrive in pieces, lanes
 * continue), then one sigma over every record with ranks in (batch_id, lane) order.
 * mac = dev_mac - dev_mac_sub when dev_mac_sub is not NULL (de_macs = x.m - a.m without
 * materialising it).  The arrays must stay valid until spdz_mac_log_sigma returns. */
int spdz_mac_log_append(spdz_ctx* ctx, uint64_t batch_id, const uint32_t* dev_opened, const uint32_t* dev_mac,
                        const uint32_t* dev_mac_sub, uint64_t len);
int spdz_mac_log_size(spdz_ctx* ctx, uint64_t* n_records);
int spdz_mac_log_sigma(spdz_ctx* ctx, uint64_t coin, uint32_t* sigma_out);
int spdz_mac_log_clear(spdz_ctx* ctx);

/* spdz.cpp:140-145 */
uint64_t spdz_commit_sigma(uint32_t sigma, uint64_t nonce);
/* spdz.cpp:147-158: SPDZ_OK or SPDZ_ERR_MAC_CHECK_FAILED */
int spdz_verify_sigmas(const uint32_t* sigmas, const uint64_t* nonces, const uint64_t* commitments, uint64_t n);
/* hash.hpp:11-19 */
uint64_t spdz_fnv1a64(const void* data, uint64_t len, uint64_t seed);

/* ---------------- preprocessing files ---------------- */
typedef struct spdz_store_info {
    int32_t party, n_parties;
    uint32_t alpha_share;
    uint64_t loop_iters, scalar_triples, matrix_triples, input_masks;
} spdz_store_info_t;
/* Validate an MPCT triple-store file (host only, nothing copied): magic, version,
 * prime, every section inside the file, no trailing bytes (triple_store.cpp:196-244). */
int spdz_store_inspect(const char* path, spdz_store_info_t* info);

/* ---------------- linear layer ---------------- */
/* linear.cpp:7-21.  Fills starts/counts (capacity `cap`), returns the tile
 * count via *n_tiles; SPDZ_ERR_SLICE_TOO_SMALL like the reference. */
int spdz_plan_tiles(uint32_t din, uint32_t dout, uint64_t slice, uint32_t* starts, uint32_t* counts, uint64_t cap,
                    uint64_t* n_tiles);
/* linear.cpp:30-49 value plane: payload = [D = W_tile.v - A.v (rows*din) | E = x.v - B.v (din)] */
int spdz_matrix_mask(spdz_ctx* ctx, const spdz_share_t* w_tile, const spdz_share_t* x, const spdz_mtriple_t* mt,
                     uint32_t* payload);
/* linear.cpp:51-61 + spdz.cpp:98-124 fused with the open: opened [D|E] = own +
 * sum reduce(peer); z = matrix_combine(mt, D, E) + b_slice.  b_slice may be NULL.
 * opened_out (rows*din + din words) may be NULL. */
int spdz_matrix_open_combine(spdz_ctx* ctx, const spdz_mtriple_t* mt, const uint32_t* own_payload,
                             const uint32_t* const* peer_payload, int n_peers, const spdz_share_t* b_slice,
                             spdz_share_t* z, uint32_t* opened_out);
/* spdz.cpp:98-124 with already-opened D (rows*din) and E (din). */
int spdz_matrix_combine(spdz_ctx* ctx, const spdz_mtriple_t* mt, const uint32_t* D, const uint32_t* E,
                        spdz_share_t* z);
/* Batched secret x secret linear layer (linear.cpp:30-61 and spdz.cpp:98-124 for `batch`
 * input columns sharing one W and one A):
 *   mask:  payload = [D = W.v - A.v (dout*din) | E = X.v - B.v (din*batch)]
 *   open + combine: opened [D|E] = own + sum reduce(peer) -> opened_out (the MAC-log
 *   values; required), then per column j exactly spdz::matrix_combine({A, B[:,j], C[:,j]},
 *   D, E[:,j]):  Z.v = C.v + D B.v + A.v E (+ D E on party 0),
 *                Z.m = C.m + D B.m + A.m E + alpha_i D E,
 *   as two tcgen05 limb GEMMs: D [B.v + [p0] E | B.m + alpha_i E] and [A.v ; A.m] E
 *   (K sliced by 8192, the s32 limb-accumulator bound). */
int spdz_bmatrix_mask(spdz_ctx* ctx, const spdz_share_t* w, const spdz_share_t* x, const spdz_bmtriple_t* t,
                      uint32_t* payload);
int spdz_bmatrix_open_combine(spdz_ctx* ctx, const spdz_bmtriple_t* t, const uint32_t* own_payload,
                              const uint32_t* const* peer_payload, int n_peers, spdz_share_t* z, uint32_t* opened_out);
/* runtime.cpp:303-334, batched: Y[dout x batch] = W[dout x din] * X[din x batch]
 * on both planes.  w_public != 0: W public (w_vals), X secret (x->vals/x->macs,
 * row-major din x batch).  w_public == 0: W secret (w->vals/w->macs), X public
 * (x_pub).  Y row-major dout x batch.  Bias is a separate spdz_add_batch. */
/* Contraction path of spdz_linear_secret_public: 0 auto (tcgen05 kind::i8 limb GEMM; din
 * beyond 8192 runs as K slices of 8192 accumulated exactly mod p), 1 CUDA-core IMAD.WIDE
 * GEMM, 2 tcgen05 only. */
int spdz_set_gemm_path(int path);
/* A public weight matrix prepared once for many secret x public calls (the layer's weights
 * in an inference loop): its tcgen05 limb image is built at creation, so each call only
 * re-lays out X.  W row-major dout x din (device), din <= 8192. */
typedef struct spdz_linear_weights spdz_linear_weights;
int spdz_linear_weights_create(spdz_ctx* ctx, uint32_t dout, uint32_t din, const uint32_t* w_public,
                               spdz_linear_weights** out);
int spdz_linear_weights_destroy(spdz_linear_weights* w);
int spdz_linear_secret_public_prepared(spdz_ctx* ctx, const spdz_linear_weights* w, uint32_t batch,
                                       const spdz_share_t* x_secret, spdz_share_t* y);
int spdz_linear_secret_public(spdz_ctx* ctx, uint32_t din, uint32_t dout, uint32_t batch, int w_public,
                              const uint32_t* w_vals, const spdz_share_t* w_secret, const spdz_share_t* x_secret,
                              const uint32_t* x_pub, spdz_share_t* y);

/* ---------------- preprocessing: GPU fake dealer (spdz.cpp:162-249) ----------------
 * The dealer is a splitmix64 stream; draw k (0-based after construction) is
 * mix(seed + (k+1)*gamma), so every share is computed independently.  `draw0`
 * is the stream position to start at (n after construction).  Outputs are the
 * share planes of ALL parties, party-major (n * lanes).  Returns
 * SPDZ_ERR_DEALER_REJECTION if any draw hit the rejection branch. */
int spdz_dealer_alpha(int n_parties, uint64_t seed, uint32_t* alpha_shares_out, uint32_t* alpha_out);
int spdz_dealer_triples(spdz_ctx* ctx, int n_parties, uint64_t seed, uint64_t draw0, uint64_t lanes,
                        uint32_t* const planes[6]);
int spdz_dealer_share(spdz_ctx* ctx, int n_parties, uint64_t seed, uint64_t draw0, uint32_t alpha,
                      const uint32_t* clear, uint64_t lanes, uint32_t* vals_out, uint32_t* macs_out);
int spdz_dealer_matrix_triple(spdz_ctx* ctx, int n_parties, uint64_t seed, uint64_t draw0, uint32_t alpha,
                              uint32_t din, uint32_t rows, uint32_t* const planes[6], uint32_t* scratch);
int spdz_dealer_masks(spdz_ctx* ctx, int n_parties, uint64_t seed, uint64_t draw0, uint32_t alpha, uint64_t count,
                      uint32_t* vals_out, uint32_t* macs_out, uint32_t* clear_out);
/* Number of draws each call consumes (to advance draw0). */
uint64_t spdz_dealer_draws_triples(int n_parties, uint64_t lanes);
uint64_t spdz_dealer_draws_share(int n_parties, uint64_t lanes);
uint64_t spdz_dealer_draws_matrix(int n_parties, uint32_t din, uint32_t rows);
uint64_t spdz_dealer_draws_masks(int n_parties, uint64_t count);

/* ---------------- host-buffer Backend (the reference's call shape) ----------------
 * Same semantics as CpuBackend (backend.cpp:16-88) with host vectors; the
 * copies happen inside the call.  `t_lanes` is the triple count the request
 * carries (TripleShortage when != lanes, backend.cpp:56-58). */
int spdz_host_add_batch(spdz_ctx* ctx, const uint32_t* xv, const uint32_t* xm, uint64_t x_lanes, const uint32_t* yv,
                        const uint32_t* ym, uint64_t y_lanes, uint32_t* zv, uint32_t* zm);
int spdz_host_sub_batch(spdz_ctx* ctx, const uint32_t* xv, const uint32_t* xm, uint64_t x_lanes, const uint32_t* yv,
                        const uint32_t* ym, uint64_t y_lanes, uint32_t* zv, uint32_t* zm);
int spdz_host_mul_mask(spdz_ctx* ctx, const uint32_t* xv, const uint32_t* yv, uint64_t lanes,
                       const uint32_t* const tri[6], uint64_t t_lanes, uint32_t* d_out, uint32_t* e_out);
int spdz_host_mul_combine(spdz_ctx* ctx, const uint32_t* const tri[6], uint64_t t_lanes, const uint32_t* d,
                          const uint32_t* e, uint64_t lanes, int party, uint32_t alpha_share, uint32_t* zv,
                          uint32_t* zm);
int spdz_host_reduce_add(spdz_ctx* ctx, const uint32_t* xv, const uint32_t* xm, uint64_t lanes, uint32_t* zv,
                         uint32_t* zm);

/* ---------------- local n-party online phase (runtime.cpp:508-613 shape) ----------------
 * A straight-line circuit executed by n parties, each party on its own CUDA
 * stream (and optionally its own device).  The opening exchange is the peer
 * payload read fused into the combine kernels; per-party streams and events
 * replace the reference's batch-id matching (net.cpp:61-95). */
typedef enum spdz_node_kind {
    SPDZ_NODE_INPUT = 0,   /* operand-free; bound by spdz_run_bind_input */
    SPDZ_NODE_CONST = 1,   /* public constant (cvals) */
    SPDZ_NODE_ADD = 2,     /* AddBatch/Adder      runtime.cpp:364-367 */
    SPDZ_NODE_SUB = 3,     /* SubBatch/Subtract   runtime.cpp:368-371 */
    SPDZ_NODE_MUL = 4,     /* MultBatch/Multiplier runtime.cpp:372-382 */
    SPDZ_NODE_REDUCE_ADD = 5, /* runtime.cpp:383-396 */
    SPDZ_NODE_REDUCE_MUL = 6, /* runtime.cpp:397-410 */
    SPDZ_NODE_LINEAR = 7,  /* runtime.cpp:439-441, operands x, W, b */
    SPDZ_NODE_ROOT = 8,    /* runtime.cpp:442-444 */
    SPDZ_NODE_LOAD = 9,    /* runtime.cpp:419-438: operands (base, start const) -> lane slice view */
    SPDZ_NODE_NOP = 10,    /* BlockLabel and other control nodes of a straight-line graph */
    SPDZ_NODE_CMP_PUBLIC = 11, /* runtime.cpp:411-418: lane 0 of two public operands, const_val = ir::CmpPred
                                  (Eq, Ne, Slt, Sgt, Sle, Sge; compared as u32 field elements) -> public 0/1 */
    /* Control flow (scheduler.cpp): a graph holding a PHI or BRANCH runs block by block
     * from spdz_run_options_t.entry_label, every block a LABEL whose `next` chain lists
     * its nodes in order.  In graphs without them LABEL is a NOP. */
    SPDZ_NODE_PHI = 12,    /* operands[i] taken when the block is entered from phi_labels[i] */
    SPDZ_NODE_BRANCH = 13, /* n_succ 1: jump to succ[0]; 2: operands[0] (public) != 0 ? succ[0] : succ[1] */
    SPDZ_NODE_LABEL = 14,  /* BlockLabel: heads its block's `next` chain */
} spdz_node_kind;

#define SPDZ_NO_NODE 0xFFFFFFFFu

#define SPDZ_MAX_OPERANDS 8

typedef struct spdz_node {
    int32_t kind;
    int32_t is_private;   /* privacy tag (graph_builder.cpp:495) */
    uint32_t lanes;       /* lane count of the node's value */
    uint32_t n_operands;
    uint32_t operands[SPDZ_MAX_OPERANDS]; /* node ids (the index in the node array); a PHI has one per
                                             incoming edge, other nodes at most 3 */
    uint32_t din, dout;   /* LINEAR only */
    uint32_t const_val;   /* CONST only (scalar broadcast) */
    /* control flow (ignored by straight-line graphs) */
    uint32_t next;        /* next node of the enclosing block (circuit::Node::next), SPDZ_NO_NODE ends it */
    uint32_t loop_depth;  /* loops containing the node's block: triples provisioned loop_iters^depth times
                             (preproc.cpp:124-163) */
    uint32_t n_succ;      /* BRANCH */
    uint32_t succ[2];
    uint32_t phi_labels[SPDZ_MAX_OPERANDS]; /* PHI: predecessor block of each operand */
} spdz_node_t;

typedef struct spdz_run_options {
    uint64_t slice;        /* RunOptions.slice (runtime.hpp:12), default 262140 */
    uint64_t dealer_seed;  /* run_local dealer seed (runtime.hpp:54), default 1 */
    int32_t fixed_coin;    /* 1: use `coin` instead of the commit-reveal nonces (tests) */
    uint64_t coin;
    int32_t use_graph;     /* capture the online phase as one CUDA graph on its first run and replay it
                            * (lane-parallel circuits with every party on one stream; else ignored) */
    int32_t devices[SPDZ_MAX_PARTIES]; /* device of each party (-1: device 0) */
    int32_t profile_kernels; /* 1: CUDA-event time every mask / combine / sigma launch */
    int32_t stream_per_party; /* 0 (default): parties on one device share its stream (kernels
                                 serialise, each gets the full HBM); 1: one stream per party */
    /* Lane sharding (multi-GPU): this run holds lanes [shard_offset, shard_offset + L) of
     * every vector node of a global circuit with shard_total lanes (L = the nodes' lanes).
     * Preprocessing is exactly that slice of the global dealer output and MAC ranks are
     * global, so sigma partials of all shards sum to the unsharded sigma.  0 = unsharded. */
    uint64_t shard_offset;
    uint64_t shard_total;
    int32_t external_mac_verify; /* 1: report per-party (partial) sigmas, caller verifies */
    /* One party per process (multi-GPU / multi-process): 0 (default) = every party lives
     * in this run; p + 1 = only party p is materialised here, the peers' opening payloads
     * and completion flags are mapped with spdz_run_export / spdz_run_import (CUDA IPC,
     * NVLink P2P loads) and ordered by stream memory operations.  Requires
     * external_mac_verify = 1. */
    int32_t single_party;
    /* Control-flow graphs: the entry block's LABEL and the loop provisioning factor
     * (RunOptions / the store's loop_iters; 0 = 64, run_local's hint, runtime.cpp:597). */
    uint32_t entry_label;
    uint64_t loop_iters;
    /* 1: the non-local parties of a single_party run are across a spdz_net mesh
     * (spdz_run_attach_net before the online phase); their opening buffers are
     * mirrored in local HBM and filled from the peers' frames. */
    int32_t network;
    /* Node-level stream scheduling of straight-line graphs (the reference scheduler's
     * concurrent issue of independent nodes, scheduler.cpp:66-95): 0 / 1 (default) = every
     * node of a party on its stream, in id order; k > 1 = the nodes are spread over k
     * streams per device by data dependence (a node continues its first operand's chain
     * when it is that chain's latest node, else takes the next stream), cross-stream
     * operands are awaited with events, and the streams are joined before the root open.
     * A node waiting for a peer's opening then stalls only its own stream, so independent
     * nodes run on.  Reductions and linear layers stay on stream 0 (shared scratch). */
    int32_t node_streams;
    /* 1: parties that share a device and stream still run their own kernels (mask, open +
     * combine, MAC sigma, input sharing per party), as they would on separate GPUs; 0
     * (default): two such parties' passes are fused (payloads and coefficients read once). */
    int32_t separate_party_kernels;
    /* 1: no launch fusion along straight-line chains (each node its own kernels); 0 (default): a
     * multiply's open+combine also writes what the next issued node needs from its product (the
     * next multiply's [d|e], an add / sub, the root opening) and co-located adds may pair up.
     * The environment variable SPDZ_NO_MASK_FUSION=1 forces 1 for every run. */
    int32_t no_fusion;
} spdz_run_options_t;

/* Per kernel class: launches, summed CUDA-event time and algorithmic bytes
 * (SURVEY.md §8d contracts). */
typedef struct spdz_kernel_stat {
    uint64_t launches;
    double ms;
    uint64_t bytes;
} spdz_kernel_stat_t;

enum { SPDZ_KSTAT_MASK = 0, SPDZ_KSTAT_COMBINE = 1, SPDZ_KSTAT_SIGMA = 2, SPDZ_KSTAT_OPEN = 3, SPDZ_KSTAT_N = 4 };

typedef struct spdz_run_report {
    double setup_ms, online_ms;       /* host wall clock, as RunReport (runtime.hpp:20-31) */
    double online_device_ms;          /* CUDA-event time of the online phase (max over parties) */
    uint64_t scalar_triples_consumed, matrix_triples_consumed;
    uint64_t bytes_exchanged;         /* payload bytes read from peers */
    uint64_t output_digest;           /* 0 here; see spdz_run_output_digest (kept off the online phase) */
    uint64_t kernel_launches;
    uint32_t sigmas[SPDZ_MAX_PARTIES];
    uint64_t coin;
    spdz_kernel_stat_t kstat[SPDZ_KSTAT_N]; /* filled when profile_kernels = 1 */
} spdz_run_report_t;

typedef struct spdz_run spdz_run;

/* Builds the run: computes the triple layout (preproc.cpp:124-163), runs the
 * GPU dealer for every party (make_dealer_stores order, triple_store.cpp:248-287)
 * and allocates every device buffer of the online phase. */
/* Host only: the triple layout spdz_run_create plans for this graph
 * (preproc.cpp:124-163 compute_triple_layout): per region 5 words
 * {kind 0 scalar / 1 matrix, node, base, stride, max_execs}, scalar regions first,
 * nodes ascending; *n_regions receives the count (out may be NULL to query). */
int spdz_triple_layout(const spdz_node_t* nodes, uint32_t n_nodes, uint64_t slice, uint64_t loop_iters,
                       uint64_t* out, uint64_t cap, uint64_t* n_regions);
int spdz_run_create(const spdz_node_t* nodes, uint32_t n_nodes, uint32_t root, int n_parties,
                    const spdz_run_options_t* opts, spdz_run** out);
int spdz_run_destroy(spdz_run* run);
/* IPC export of this process's party: opening payloads, input differences, root
 * values and the opening-flag words.  *len receives the blob size (call with
 * buf = NULL to query). */
int spdz_run_export(spdz_run* run, void* buf, uint64_t cap, uint64_t* len);
/* Maps other processes' export blobs (concatenated; own entries are skipped). */
int spdz_run_import(spdz_run* run, const void* blob, uint64_t len);
/* Re-runs the GPU dealer with `seed` (fresh preprocessing; inputs must be shared again). */
/* One party's MPCT triple-store file (the reference's preprocessing output,
 * write_store_file / read_store_file triple_store.cpp:163-244) loaded into this run's
 * device pools instead of spdz_run_deal: the scalar triples of every region of the
 * run's triple layout (preproc.cpp:124-163), the matrix triples in demand order and the
 * input masks, read through pinned staging buffers.  Call once per local party.
 * Errors: SPDZ_ERR_STORE_FORMAT (VersionMismatch / CorruptPayload),
 * SPDZ_ERR_INSUFFICIENT_TRIPLES (store smaller than the run's demand, preproc.cpp:182-201),
 * SPDZ_ERR_TRIPLE_SHAPE_MISMATCH (matrix triple of the wrong shape). */
int spdz_run_load_store(spdz_run* run, int party, const char* path);
int spdz_run_deal(spdz_run* run, uint64_t seed);
/* Cleartext input for an INPUT node (host pointer).  Private inputs are shared
 * with the dealer's input masks (preproc.cpp:205-243) during spdz_run_share_inputs. */
int spdz_run_bind_input(spdz_run* run, uint32_t node, const uint32_t* host_vals, uint64_t len);
/* Input sharing (setup, excluded from online time as in runtime.cpp:511-534).
 * Asynchronous: it is stream-ordered before the next online phase; bound host
 * inputs must stay untouched until that phase has begun. */
int spdz_run_share_inputs(spdz_run* run);
/* Online phase: node execution, root open, deferred MAC check.  Re-runnable
 * (triple consumption is reset per call only when `reuse_preprocessing` = 1 —
 * the bench re-times the same preprocessing; the reference semantics are 0). */
int spdz_run_online(spdz_run* run, int reuse_preprocessing, spdz_run_report_t* report);
/* Registers the host buffer the next online phases write the opened outputs
 * into (D2H straight from the open kernel's buffer; pinned memory recommended).
 * Without one, outputs land in an internal pinned buffer (spdz_run_outputs). */
int spdz_run_bind_output(spdz_run* run, uint32_t* host_out, uint64_t cap);
/* The online phase in two steps, so that the MAC-check coin can be agreed
 * after the openings (runtime.cpp:467-489) — e.g. across the ranks of a
 * lane-sharded run: begin = node execution + root open (+ async D2H of the
 * outputs); mac_check = sigma with `coin` (use_coin = 1) or the run's own
 * coin, then verification (unless external_mac_verify) and the report.
 * spdz_run_online = begin + mac_check(use_coin = 0). */
int spdz_run_online_begin(spdz_run* run, int reuse_preprocessing);
/* Optional caller-owned streams (device of party 0 / of the output party) for the input
 * H2D copies and the output D2H copy, shared by several runs so that their copies queue
 * in issue order (host-streamed execution).  NULL restores the run's own streams. */
int spdz_run_set_copy_streams(spdz_run* run, void* h2d_stream, void* d2h_stream);
/* The CUDA stream a local party's kernels run on (NULL if not local) — for callers
 * that order their own work or timing events against the run. */
void* spdz_run_party_stream(spdz_run* run, int party);
/* Device time from run a's online-phase start event to run b's end event (after its MAC
 * sigma kernels), for several runs on one device launched back to back (ChunkedRun). */
int spdz_run_span_ms(spdz_run* a, spdz_run* b, float* ms);
/* First half of spdz_run_mac_check: agree on the coin and launch the sigma kernels
 * asynchronously; the next spdz_run_mac_check collects and verifies (its coin
 * arguments are then ignored). */
int spdz_run_mac_check_launch(spdz_run* run, int use_coin, uint64_t coin);
/* Blocks the host until every opening of the phase begun by spdz_run_online_begin is
 * complete on this run's local parties (the opened values are final): the point after which
 * a MAC-check coin may be agreed (runtime.cpp:467-506 draws it after the openings). */
int spdz_run_wait_openings(spdz_run* run);
int spdz_run_mac_check(spdz_run* run, int use_coin, uint64_t coin, spdz_run_report_t* report);
/* fnv1a64 digest of the last opened outputs (RunReport.output_digest, runtime.cpp:573). */
int spdz_run_output_digest(spdz_run* run, uint64_t* digest);
/* Opened outputs (host).  *len receives the lane count. */
int spdz_run_outputs(spdz_run* run, uint32_t* host_out, uint64_t cap, uint64_t* len);
/* Device view of a node's share for party p (tests). */
int spdz_run_node_share(spdz_run* run, int party, uint32_t node, spdz_share_t* out);
/* Test hook: flip `bit` of the payload word `word` that party `receiver`
 * reads from `sender` for node `node` (SimHub BitFlip, net.cpp:241-278). */
/* ---------------- cross-host parties: the reference's wire format + TCP mesh ----------------
 * Frames of net.hpp:40-49 (16-byte header {msg-type u8, pad[3], lane-count u32, batch-id u64}
 * + u32 words, little-endian) over the mesh of net_tcp.cpp:152-235 (party i listens on
 * endpoints[i] for higher indices and dials lower ones, announcing its index as a u32).  A
 * B200 party and reference parties (or other B200 hosts) interoperate frame for frame. */
typedef struct spdz_net spdz_net;
int spdz_net_connect(int party, int n_parties, const char* const* endpoints, uint64_t connect_timeout_ms,
                     uint64_t io_timeout_ms, spdz_net** out);
int spdz_net_destroy(spdz_net* net);
/* raw frames (tests / tooling): msg-type 0 OpenShares 1 Commit 2 Reveal 3 Nonce 4 Control */
int spdz_net_send(spdz_net* net, int peer, int type, uint64_t batch, const uint32_t* words, uint32_t lanes);
/* spdz_net_recv: a frame longer than cap lanes returns SPDZ_ERR_LANE_COUNT_MISMATCH with its
 * length in *lanes and stays queued (retry with a larger buffer); out == NULL consumes the frame
 * and returns only its length.  Frames announcing more than 2^30 lanes stop the peer's reader
 * with MalformedShareMessage before anything is allocated. */
int spdz_net_recv(spdz_net* net, int peer, int type, uint64_t batch, uint32_t* out, uint64_t cap, uint64_t* lanes);
int spdz_net_stats(spdz_net* net, uint64_t* bytes_sent, uint64_t* bytes_received);
/* A single-party run (options.single_party = p + 1) whose peers are across the mesh:
 * every opening is sent / received as the reference's frames with its batch ids
 * (make_batch(node, exec, sub), runtime.cpp:22-24; linear tiles batch + tile; inputs
 * kInputBatchBase + k; the MAC check's four exchanges at kMacBatchBase + 0..3,
 * runtime.cpp:467-506), and the MAC check runs the reference's commit/reveal protocol.
 * The mesh must outlive the run. */
int spdz_run_attach_net(spdz_run* run, spdz_net* net);

int spdz_run_inject_bitflip(spdz_run* run, uint32_t node, int sender, int receiver, uint64_t word, uint32_t bit);

#ifdef __cplusplus
}
#endif
#endif /* SPDZ_B200_H */
