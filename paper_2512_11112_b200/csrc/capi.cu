// C ABI of the B200 SPDZ back end: contexts, the widened Backend surface,
// open, MAC check, linear layer, GPU dealer, host-buffer Backend wrappers.
// Every entry point converts exceptions to spdz_status + thread-local message.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "field.cuh"
#include "hostcopy.hpp"

#include <cstdlib>
#include "internal.hpp"

using namespace spdzb200;

namespace {
thread_local std::string g_err;
}

namespace spdzb200 {
void set_last_error(const char* msg) { g_err = msg; }
}

namespace {

void need_ctx(const spdz_ctx* ctx) { need(ctx != nullptr, SPDZ_ERR_INVALID_ARGUMENT, "null context"); }

void need_share(const spdz_share_t* s, const char* what) {
    need(s != nullptr, SPDZ_ERR_INVALID_ARGUMENT, std::string("null share: ") + what);
    need(s->lanes == 0 || (s->vals && s->macs), SPDZ_ERR_INVALID_ARGUMENT, std::string("null plane: ") + what);
}

// backend.cpp:11-14
void check_lanes(uint64_t a, uint64_t b) {
    if (a != b)
        throw Error(SPDZ_ERR_LANE_MISMATCH, "LaneMismatch: " + std::to_string(a) + " vs " + std::to_string(b));
}

void launch_ok(cudaError_t e, const char* what) { cuda_check(e, what); }

}  // namespace

namespace spdzb200 {

void set_alpha(spdz_ctx* ctx, uint32_t alpha) {
    ctx->alpha = alpha;
    device_guard(ctx);
    cuda_check(launch_set_word(ctx->stream, ctx->d_alpha, alpha), "set alpha");
}

void device_guard(const spdz_ctx* ctx) { cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice"); }

uint32_t host_reduce64(uint64_t v) { return fp_reduce64(v); }

// spdz.cpp:127-129: ranks in (batch_id, lane) order over all records.
void assign_ranks(spdz_mac_segment_t* segs, uint64_t n) {
    std::vector<uint64_t> idx(n);
    std::iota(idx.begin(), idx.end(), 0);
    std::sort(idx.begin(), idx.end(), [&](uint64_t a, uint64_t b) {
        return segs[a].batch_id != segs[b].batch_id ? segs[a].batch_id < segs[b].batch_id
                                                    : segs[a].lane0 < segs[b].lane0;
    });
    uint64_t off = 0;  // records of all smaller batch ids
    size_t i = 0;
    while (i < idx.size()) {
        size_t j = i;
        uint64_t batch_records = 0;
        const uint64_t b = segs[idx[i]].batch_id;
        while (j < idx.size() && segs[idx[j]].batch_id == b) {
            batch_records = std::max(batch_records, segs[idx[j]].lane0 + segs[idx[j]].len);
            batch_records = std::max(batch_records, segs[idx[j]].batch_len);
            segs[idx[j]].j0 = off + segs[idx[j]].lane0;
            ++j;
        }
        off += batch_records;
        i = j;
    }
}

void mac_sigma_launch(spdz_ctx* ctx, const spdz_mac_segment_t* segs, uint64_t n, uint64_t coin, int slot) {
    // segment tables go by value as kernel parameters: no staging copy, no host sync
    cuda_check(cudaMemsetAsync(ctx->d_acc + slot, 0, 8, ctx->stream), "memset acc");
    for (uint64_t base = 0; base < n; base += kMacTableSegs) {
        MacTable tab{};
        tab.n = (uint32_t)std::min<uint64_t>(kMacTableSegs, n - base);
        uint64_t recs = 0;
        for (uint32_t i = 0; i < tab.n; ++i) {
            const auto& sg = segs[base + i];
            need(sg.len == 0 || (sg.value && sg.mac_a), SPDZ_ERR_INVALID_ARGUMENT, "null MAC segment");
            tab.seg[i] = MacSegDev{{sg.value}, {sg.mac_a}, {sg.mac_b}, sg.len, sg.j0};
            tab.rec0[i] = recs;
            recs += sg.len;
        }
        tab.rec0[tab.n] = recs;
        launch_ok(launch_mac_sigma(ctx->stream, tab, coin, ctx->alpha, ctx->d_acc + slot, ctx->sms), "k_mac_sigma");
    }
}

uint32_t mac_sigma_collect(spdz_ctx* ctx, int slot) {
    unsigned long long acc = 0;
    cuda_check(cudaMemcpyAsync(&acc, ctx->d_acc + slot, 8, cudaMemcpyDeviceToHost, ctx->stream), "D2H sigma");
    cuda_check(cudaStreamSynchronize(ctx->stream), "sync sigma");
    return fp_reduce64(acc);
}

uint32_t mac_sigma_impl(spdz_ctx* ctx, const spdz_mac_segment_t* segs, uint64_t n, uint64_t coin) {
    mac_sigma_launch(ctx, segs, n, coin, 0);
    return mac_sigma_collect(ctx, 0);
}

// Dealer stream accounting (spdz.cpp:162-249).
uint64_t dealer_draws_share(int n, uint64_t lanes) { return 2ull * (n - 1) * lanes; }
uint64_t dealer_draws_triples(int n, uint64_t lanes) { return 2 * lanes + 3 * dealer_draws_share(n, lanes); }
uint64_t dealer_draws_matrix(int n, uint32_t din, uint32_t rows) {
    const uint64_t cells = (uint64_t)din * rows;
    return cells + din + dealer_draws_share(n, cells) + dealer_draws_share(n, din) + dealer_draws_share(n, rows);
}
uint64_t dealer_draws_masks(int n, uint64_t count) { return count * (1 + 2ull * (n - 1)); }

// spdz.cpp:162-173 (host: n draws)
void dealer_alpha(int n, uint64_t seed, uint32_t* shares, uint32_t* alpha) {
    uint64_t state = seed;
    auto draw = [&]() {
        uint64_t v;
        do {
            state += kGamma;
            v = mix64(state);
        } while (v >= 0xFFFFFFFFFFFFFFE7ull);
        return fp_reduce64(v);
    };
    uint32_t sum = 0;
    for (int i = 1; i < n; ++i) {
        shares[i] = draw();
        sum = fp_add(sum, shares[i]);
    }
    const uint32_t key = draw();
    shares[0] = fp_sub(key, sum);
    *alpha = key;
}

void check_dealer_flag(spdz_ctx* ctx) {
    unsigned int flag = 0;
    cuda_check(cudaMemcpyAsync(&flag, ctx->d_flag, 4, cudaMemcpyDeviceToHost, ctx->stream), "D2H dealer flag");
    cuda_check(cudaStreamSynchronize(ctx->stream), "sync dealer");
    if (flag)
        throw Error(SPDZ_ERR_DEALER_REJECTION,
                    "dealer draw hit the rejection branch (p=25/2^64); regenerate with another seed");
}

}  // namespace spdzb200

extern "C" {

const char* spdz_last_error(void) { return g_err.c_str(); }
const char* spdz_version(void) { return "spdz_b200 0.1 (sm_100a)"; }
uint64_t spdz_kernel_launches(void) { return g_kernel_launches; }

int spdz_ctx_create(int device, int party, int n_parties, uint32_t alpha_share, spdz_ctx** out) {
    return guard([&] {
        need(out != nullptr, SPDZ_ERR_INVALID_ARGUMENT, "null out");
        need(n_parties >= 1 && n_parties <= SPDZ_MAX_PARTIES, SPDZ_ERR_INVALID_ARGUMENT, "n_parties out of range");
        need(party >= 0 && party < n_parties, SPDZ_ERR_INVALID_ARGUMENT, "party out of range");
        int count = 0;
        if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
            throw Error(SPDZ_ERR_BACKEND_UNAVAILABLE, "BackendUnavailable: no CUDA device");
        need(device >= 0 && device < count, SPDZ_ERR_INVALID_ARGUMENT, "device out of range");
        auto* c = new spdz_ctx;
        c->device = device;
        c->party = party;
        c->n_parties = n_parties;
        c->alpha = alpha_share;
        try {
            device_guard(c);
            cuda_check(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device), "attr");
            cuda_check(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking), "stream");
            c->stream = c->own_stream;
            cuda_check(cudaMalloc(&c->d_acc, 16 * sizeof(unsigned long long)), "acc");
            cuda_check(cudaMalloc(&c->d_flag, sizeof(unsigned int)), "flag");
            cuda_check(cudaMalloc(&c->d_alpha, 16), "alpha");
            set_alpha(c, alpha_share);
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
}

int spdz_ctx_destroy(spdz_ctx* ctx) {
    return guard([&] {
        if (!ctx) return;
        cudaSetDevice(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        ctx->scratch.release();
        ctx->seg_buf.release();
        ctx->rank_buf.release();
        ctx->pinned.release();
        if (ctx->d_acc) cudaFree(ctx->d_acc);
        if (ctx->d_flag) cudaFree(ctx->d_flag);
        if (ctx->d_alpha) cudaFree(ctx->d_alpha);
        if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
        delete ctx;
    });
}

int spdz_ctx_set_stream(spdz_ctx* ctx, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        ctx->stream = (cudaStream_t)stream;  // NULL = the legacy default stream
    });
}

int spdz_ctx_use_own_stream(spdz_ctx* ctx) {
    return guard([&] {
        need_ctx(ctx);
        ctx->stream = ctx->own_stream;
    });
}
void* spdz_ctx_stream(spdz_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }
int spdz_ctx_party(const spdz_ctx* ctx) { return ctx ? ctx->party : -1; }

int spdz_ctx_sync(spdz_ctx* ctx) {
    return guard([&] {
        need_ctx(ctx);
        device_guard(ctx);
        cuda_check(cudaStreamSynchronize(ctx->stream), "cudaStreamSynchronize");
    });
}

int spdz_capability(const spdz_ctx* ctx, spdz_capability_t* out) {
    return guard([&] {
        need_ctx(ctx);
        need(out != nullptr, SPDZ_ERR_INVALID_ARGUMENT, "null out");
        std::memset(out, 0, sizeof *out);
        std::strncpy(out->name, "gpu-b200", sizeof out->name - 1);
        out->min_kernel_size = 1;  // no CPU fallback (north star); registry routes every size here
        out->threads_per_block = 256;
        out->executable = 1;
        out->sm_count = ctx->sms;
        out->device = ctx->device;
    });
}

// ---------------- Backend ----------------
static int add_sub(spdz_ctx* ctx, const spdz_share_t* x, const spdz_share_t* y, spdz_share_t* z, bool sub) {
    return guard([&] {
        need_ctx(ctx);
        need_share(x, "x");
        need_share(y, "y");
        need_share(z, "z");
        check_lanes(x->lanes, y->lanes);
        check_lanes(x->lanes, z->lanes);
        device_guard(ctx);
        launch_ok(launch_add_sub(ctx->stream, sub, x->vals, x->macs, y->vals, y->macs, z->vals, z->macs, x->lanes,
                                 ctx->sms),
                  "k_add_sub");
    });
}
int spdz_add_batch(spdz_ctx* ctx, const spdz_share_t* x, const spdz_share_t* y, spdz_share_t* z) {
    return add_sub(ctx, x, y, z, false);
}
int spdz_sub_batch(spdz_ctx* ctx, const spdz_share_t* x, const spdz_share_t* y, spdz_share_t* z) {
    return add_sub(ctx, x, y, z, true);
}

// backend.cpp:53-65
int spdz_mul_mask(spdz_ctx* ctx, const spdz_share_t* x, const spdz_share_t* y, const spdz_triple_t* t,
                  uint32_t* d_out, uint32_t* e_out) {
    return guard([&] {
        need_ctx(ctx);
        need_share(x, "x");
        need_share(y, "y");
        need(t != nullptr, SPDZ_ERR_INVALID_ARGUMENT, "null triple");
        check_lanes(x->lanes, y->lanes);
        if (t->a.lanes != x->lanes)
            throw Error(SPDZ_ERR_TRIPLE_SHORTAGE, "TripleShortage: request carries " + std::to_string(t->a.lanes) +
                                                      " triples for " + std::to_string(x->lanes) + " lanes");
        need(x->lanes == 0 || (d_out && e_out), SPDZ_ERR_INVALID_ARGUMENT, "null d/e out");
        device_guard(ctx);
        launch_ok(launch_mul_mask(ctx->stream, x->vals, y->vals, t->a.vals, t->b.vals, d_out, e_out, x->lanes,
                                  ctx->sms),
                  "k_mul_mask");
    });
}

static void check_triple(const spdz_triple_t* t, uint64_t lanes, const char* msg) {
    need(t != nullptr, SPDZ_ERR_INVALID_ARGUMENT, "null triple");
    if (t->a.lanes != lanes || t->b.lanes != lanes || t->c.lanes != lanes)
        throw Error(SPDZ_ERR_TRIPLE_SHORTAGE, msg);
}

// backend.cpp:67-74 (+ spdz.cpp:77-96)
int spdz_mul_combine(spdz_ctx* ctx, const spdz_triple_t* t, const uint32_t* d, const uint32_t* e, spdz_share_t* z) {
    return guard([&] {
        need_ctx(ctx);
        need_share(z, "z");
        check_triple(t, z->lanes, "TripleShortage: combine with mismatched triple count");
        const uint32_t* tri[6] = {t->a.vals, t->a.macs, t->b.vals, t->b.macs, t->c.vals, t->c.macs};
        device_guard(ctx);
        launch_ok(launch_beaver_combine(ctx->stream, d, e, nullptr, nullptr, 0, tri, ctx->party, ctx->alpha, z->vals,
                                        z->macs, nullptr, nullptr, z->lanes, ctx->sms),
                  "k_combine");
    });
}

int spdz_beaver_open_combine(spdz_ctx* ctx, const spdz_triple_t* t, const uint32_t* own_de,
                             const uint32_t* const* peer_de, int n_peers, spdz_share_t* z, uint32_t* opened_out) {
    return guard([&] {
        need_ctx(ctx);
        need_share(z, "z");
        need(n_peers >= 0 && n_peers <= kMaxPeers, SPDZ_ERR_INVALID_ARGUMENT, "n_peers out of range");
        check_triple(t, z->lanes, "TripleShortage: combine with mismatched triple count");
        const uint64_t L = z->lanes;
        const uint32_t* pd[kMaxPeers];
        const uint32_t* pe[kMaxPeers];
        for (int p = 0; p < n_peers; ++p) {
            pd[p] = peer_de[p];
            pe[p] = peer_de[p] + L;
        }
        const uint32_t* tri[6] = {t->a.vals, t->a.macs, t->b.vals, t->b.macs, t->c.vals, t->c.macs};
        device_guard(ctx);
        launch_ok(launch_beaver_combine(ctx->stream, own_de, own_de + L, pd, pe, n_peers, tri, ctx->party, ctx->alpha,
                                        z->vals, z->macs, opened_out, opened_out ? opened_out + L : nullptr, L,
                                        ctx->sms),
                  "k_combine");
    });
}

// backend.cpp:76-84
int spdz_reduce_add(spdz_ctx* ctx, const spdz_share_t* x, spdz_share_t* z) {
    return guard([&] {
        need_ctx(ctx);
        need_share(x, "x");
        need_share(z, "z");
        need(z->lanes == 1, SPDZ_ERR_LANE_MISMATCH, "LaneMismatch: reduce_add output must have 1 lane");
        device_guard(ctx);
        cuda_check(cudaMemsetAsync(ctx->d_acc + 2, 0, 16, ctx->stream), "memset");
        launch_ok(launch_reduce_add(ctx->stream, x->vals, x->macs, x->lanes, ctx->d_acc + 2, ctx->sms), "reduce");
        launch_ok(launch_finish_reduce(ctx->stream, ctx->d_acc + 2, z->vals, z->macs), "finish");
    });
}

// ---------------- public-constant ops ----------------
static int public_op(spdz_ctx* ctx, int op, spdz_share_t* x, const uint32_t* k, uint64_t k_len) {
    return guard([&] {
        need_ctx(ctx);
        need_share(x, "x");
        need(k_len == 1 || k_len == x->lanes, SPDZ_ERR_LANE_MISMATCH,
             "LaneMismatch: public operand has " + std::to_string(k_len) + " lanes for " +
                 std::to_string(x->lanes));
        need(x->lanes == 0 || k, SPDZ_ERR_INVALID_ARGUMENT, "null public operand");
        device_guard(ctx);
        launch_ok(launch_public(ctx->stream, op, x->vals, x->macs, k, k_len == 1 && x->lanes != 1, 0u, false,
                                ctx->party, ctx->alpha, x->vals, x->macs, x->lanes, ctx->sms),
                  "k_public");
    });
}
int spdz_add_public(spdz_ctx* c, spdz_share_t* x, const uint32_t* k, uint64_t n) { return public_op(c, 0, x, k, n); }
int spdz_sub_public(spdz_ctx* c, spdz_share_t* x, const uint32_t* k, uint64_t n) { return public_op(c, 1, x, k, n); }
int spdz_rsub_public(spdz_ctx* c, spdz_share_t* x, const uint32_t* k, uint64_t n) { return public_op(c, 2, x, k, n); }
int spdz_mul_public(spdz_ctx* c, spdz_share_t* x, const uint32_t* k, uint64_t n) { return public_op(c, 3, x, k, n); }
int spdz_mul_public_scalar(spdz_ctx* ctx, spdz_share_t* x, uint32_t k) {
    return guard([&] {
        need_ctx(ctx);
        need_share(x, "x");
        device_guard(ctx);
        launch_ok(launch_public(ctx->stream, 3, x->vals, x->macs, nullptr, false, k, true, ctx->party, ctx->alpha,
                                x->vals, x->macs, x->lanes, ctx->sms),
                  "k_public");
    });
}
int spdz_share_of_public(spdz_ctx* ctx, const uint32_t* k, uint64_t k_len, spdz_share_t* out) {
    return guard([&] {
        need_ctx(ctx);
        need_share(out, "out");
        need(k_len == 1 || k_len == out->lanes, SPDZ_ERR_LANE_MISMATCH, "LaneMismatch: share_of_public");
        device_guard(ctx);
        launch_ok(launch_public(ctx->stream, 4, nullptr, nullptr, k, k_len == 1 && out->lanes != 1, 0u, false,
                                ctx->party, ctx->alpha, out->vals, out->macs, out->lanes, ctx->sms),
                  "k_share_of_public");
    });
}

// ---------------- open ----------------
int spdz_open_sum(spdz_ctx* ctx, const uint32_t* own, const uint32_t* const* peers, int n_peers, uint64_t len,
                  uint32_t* out) {
    return guard([&] {
        need_ctx(ctx);
        need(n_peers >= 0 && n_peers <= kMaxPeers, SPDZ_ERR_INVALID_ARGUMENT, "n_peers out of range");
        device_guard(ctx);
        launch_ok(launch_open_sum(ctx->stream, own, peers, n_peers, out, len, ctx->sms), "k_open");
    });
}

// ---------------- MAC check ----------------
int spdz_mac_assign_ranks(spdz_mac_segment_t* segs, uint64_t n) {
    return guard([&] {
        need(segs != nullptr || n == 0, SPDZ_ERR_INVALID_ARGUMENT, "null segments");
        assign_ranks(segs, n);
    });
}

int spdz_mac_sigma(spdz_ctx* ctx, const spdz_mac_segment_t* segs, uint64_t n, uint64_t coin, uint32_t* sigma_out) {
    return guard([&] {
        need_ctx(ctx);
        need(sigma_out != nullptr, SPDZ_ERR_INVALID_ARGUMENT, "null sigma_out");
        device_guard(ctx);
        *sigma_out = mac_sigma_impl(ctx, segs, n, coin);
    });
}

// spdz.cpp:126-138 record form: rank = position in (batch_id, lane) order.
int spdz_mac_sigma_records(spdz_ctx* ctx, const uint64_t* hb, const uint32_t* hl, const uint32_t* dv,
                           const uint32_t* dm, uint64_t n, uint64_t coin, uint32_t* sigma_out) {
    return guard([&] {
        need_ctx(ctx);
        need(sigma_out != nullptr, SPDZ_ERR_INVALID_ARGUMENT, "null sigma_out");
        device_guard(ctx);
        std::vector<uint64_t> idx(n), rank(n);
        std::iota(idx.begin(), idx.end(), 0);
        std::sort(idx.begin(), idx.end(), [&](uint64_t a, uint64_t b) {
            return hb[a] != hb[b] ? hb[a] < hb[b] : hl[a] < hl[b];
        });
        for (uint64_t r = 0; r < n; ++r) rank[idx[r]] = r;
        uint64_t* dr = (uint64_t*)ctx->rank_buf.ensure(std::max<uint64_t>(n, 1) * 8);
        cuda_check(cudaMemcpyAsync(dr, rank.data(), n * 8, cudaMemcpyHostToDevice, ctx->stream), "H2D ranks");
        cuda_check(cudaMemsetAsync(ctx->d_acc, 0, 8, ctx->stream), "memset");
        launch_ok(launch_mac_sigma_ranked(ctx->stream, dv, dm, dr, n, coin, ctx->alpha, ctx->d_acc, ctx->sms),
                  "k_mac_sigma_ranked");
        *sigma_out = mac_sigma_collect(ctx, 0);
    });
}

uint64_t spdz_fnv1a64(const void* data, uint64_t len, uint64_t seed) {
    const uint8_t* p = (const uint8_t*)data;
    uint64_t h = seed;
    for (uint64_t i = 0; i < len; ++i) {
        h ^= p[i];
        h *= 1099511628211ull;
    }
    return h;
}

uint64_t spdz_commit_sigma(uint32_t sigma, uint64_t nonce) {  // spdz.cpp:140-145
    uint8_t buf[12];
    for (int i = 0; i < 4; ++i) buf[i] = uint8_t(sigma >> (8 * i));
    for (int i = 0; i < 8; ++i) buf[4 + i] = uint8_t(nonce >> (8 * i));
    return spdz_fnv1a64(buf, sizeof buf, 1469598103934665603ull);
}

int spdz_verify_sigmas(const uint32_t* sigmas, const uint64_t* nonces, const uint64_t* commitments, uint64_t n) {
    return guard([&] {  // spdz.cpp:147-158
        uint32_t total = 0;
        for (uint64_t i = 0; i < n; ++i) {
            if (spdz_commit_sigma(sigmas[i], nonces[i]) != commitments[i])
                throw Error(SPDZ_ERR_MAC_CHECK_FAILED,
                            "MacCheckFailed: commitment mismatch from party " + std::to_string(i));
            total = fp_add(total, sigmas[i]);
        }
        if (total != 0) throw Error(SPDZ_ERR_MAC_CHECK_FAILED, "MacCheckFailed: aggregate sigma is nonzero");
    });
}

// ---------------- linear layer ----------------
int spdz_plan_tiles(uint32_t din, uint32_t dout, uint64_t slice, uint32_t* starts, uint32_t* counts, uint64_t cap,
                    uint64_t* n_tiles) {
    return guard([&] {  // linear.cpp:7-21
        if (din == 0 || dout == 0) throw Error(SPDZ_ERR_SLICE_TOO_SMALL, "SliceTooSmall: empty layer dimensions");
        if (slice < din)
            throw Error(SPDZ_ERR_SLICE_TOO_SMALL, "SliceTooSmall: slice " + std::to_string(slice) +
                                                      " holds no full row of length " + std::to_string(din));
        uint32_t rpt = (uint32_t)std::min<uint64_t>(slice / din, 0xffffffffull);
        if (rpt == 0) rpt = 1;
        uint64_t k = 0;
        for (uint64_t r = 0; r < dout; r += rpt, ++k) {
            if (k < cap) {
                if (starts) starts[k] = (uint32_t)r;
                if (counts) counts[k] = (uint32_t)std::min<uint64_t>(rpt, dout - r);
            }
        }
        if (n_tiles) *n_tiles = k;
    });
}

static void check_mtriple(const spdz_mtriple_t* mt) {
    need(mt != nullptr, SPDZ_ERR_INVALID_ARGUMENT, "null matrix triple");
    const uint64_t cells = (uint64_t)mt->din * mt->rows;
    if (mt->a.lanes != cells || mt->b.lanes != mt->din || mt->c.lanes != mt->rows)
        throw Error(SPDZ_ERR_TRIPLE_SHAPE_MISMATCH, "TripleShapeMismatch: matrix triple planes do not match " +
                                                        std::to_string(mt->rows) + "x" + std::to_string(mt->din));
}

int spdz_matrix_mask(spdz_ctx* ctx, const spdz_share_t* w_tile, const spdz_share_t* x, const spdz_mtriple_t* mt,
                     uint32_t* payload) {
    return guard([&] {  // linear.cpp:30-49
        need_ctx(ctx);
        need_share(w_tile, "w_tile");
        need_share(x, "x");
        check_mtriple(mt);
        const uint64_t cells = (uint64_t)mt->din * mt->rows;
        if (w_tile->lanes != cells)
            throw Error(SPDZ_ERR_TRIPLE_SHAPE_MISMATCH,
                        "TripleShapeMismatch: triple " + std::to_string(mt->rows) + "x" + std::to_string(mt->din) +
                            " for tile of " + std::to_string(w_tile->lanes) + " cells");
        check_lanes(x->lanes, mt->din);
        device_guard(ctx);
        launch_ok(launch_matrix_mask(ctx->stream, w_tile->vals, mt->a.vals, cells, x->vals, mt->b.vals, mt->din,
                                     payload, ctx->sms),
                  "k_matrix_mask");
    });
}

static void matrix_combine_common(spdz_ctx* ctx, const spdz_mtriple_t* mt, const uint32_t* own,
                                  const uint32_t* const* peers, int n_peers, const spdz_share_t* b_slice,
                                  spdz_share_t* z, uint32_t* opened_out, const uint32_t* E_given) {
    need_ctx(ctx);
    check_mtriple(mt);
    need_share(z, "z");
    check_lanes(z->lanes, mt->rows);
    if (b_slice) check_lanes(b_slice->lanes, mt->rows);
    need(n_peers >= 0 && n_peers <= kMaxPeers, SPDZ_ERR_INVALID_ARGUMENT, "n_peers out of range");
    device_guard(ctx);
    const uint64_t cells = (uint64_t)mt->din * mt->rows;
    uint32_t* opened = opened_out;
    if (!opened) opened = (uint32_t*)ctx->scratch.ensure((cells + mt->din) * 4 + 16);
    // opened E first (the combine rows read it): E = own_E + sum reduce(peer_E)
    if (E_given) {
        cuda_check(cudaMemcpyAsync(opened + cells, E_given, (uint64_t)mt->din * 4, cudaMemcpyDeviceToDevice,
                                   ctx->stream),
                   "copy E");
    } else {
        const uint32_t* pe[kMaxPeers];
        for (int p = 0; p < n_peers; ++p) pe[p] = peers[p] + cells;
        launch_ok(launch_open_sum(ctx->stream, own + cells, pe, n_peers, opened + cells, mt->din, ctx->sms), "open E");
    }
    const uint32_t* m6[6] = {mt->a.vals, mt->a.macs, mt->b.vals, mt->b.macs, mt->c.vals, mt->c.macs};
    launch_ok(launch_matrix_combine(ctx->stream, mt->din, mt->rows, mt->rows ? mt->rows : 1, own, peers, n_peers, m6,
                                    b_slice ? b_slice->vals : nullptr, b_slice ? b_slice->macs : nullptr, ctx->party,
                                    ctx->alpha, z->vals, z->macs, opened, ctx->sms),
              "k_matrix_combine");
}

int spdz_matrix_open_combine(spdz_ctx* ctx, const spdz_mtriple_t* mt, const uint32_t* own_payload,
                             const uint32_t* const* peer_payload, int n_peers, const spdz_share_t* b_slice,
                             spdz_share_t* z, uint32_t* opened_out) {
    return guard([&] {
        matrix_combine_common(ctx, mt, own_payload, peer_payload, n_peers, b_slice, z, opened_out, nullptr);
    });
}

int spdz_matrix_combine(spdz_ctx* ctx, const spdz_mtriple_t* mt, const uint32_t* D, const uint32_t* E,
                        spdz_share_t* z) {
    return guard([&] { matrix_combine_common(ctx, mt, D, nullptr, 0, nullptr, z, nullptr, E); });
}

static void check_bmtriple(const spdz_bmtriple_t* t) {
    need(t != nullptr, SPDZ_ERR_INVALID_ARGUMENT, "null batched matrix triple");
    need_share(&t->a, "A");
    need_share(&t->b, "B");
    need_share(&t->c, "C");
    if (t->a.lanes != (uint64_t)t->dout * t->din || t->b.lanes != (uint64_t)t->din * t->batch ||
        t->c.lanes != (uint64_t)t->dout * t->batch)
        throw Error(SPDZ_ERR_TRIPLE_SHAPE_MISMATCH, "TripleShapeMismatch: batched matrix triple planes do not match " +
                                                        std::to_string(t->dout) + "x" + std::to_string(t->din) + "x" +
                                                        std::to_string(t->batch));
}

int spdz_bmatrix_mask(spdz_ctx* ctx, const spdz_share_t* w, const spdz_share_t* x, const spdz_bmtriple_t* t,
                      uint32_t* payload) {
    return guard([&] {  // linear.cpp:30-49, every column of X at once
        need_ctx(ctx);
        need_share(w, "w");
        need_share(x, "x");
        check_bmtriple(t);
        check_lanes(w->lanes, (uint64_t)t->dout * t->din);
        check_lanes(x->lanes, (uint64_t)t->din * t->batch);
        need(payload != nullptr, SPDZ_ERR_INVALID_ARGUMENT, "null payload");
        device_guard(ctx);
        const uint64_t cells = (uint64_t)t->dout * t->din, ecount = (uint64_t)t->din * t->batch;
        need(ecount <= 0xFFFFFFFFull, SPDZ_ERR_INVALID_ARGUMENT, "din * batch too large");
        launch_ok(launch_matrix_mask(ctx->stream, w->vals, t->a.vals, cells, x->vals, t->b.vals, (uint32_t)ecount,
                                     payload, ctx->sms),
                  "k_matrix_mask");
    });
}

int spdz_bmatrix_open_combine(spdz_ctx* ctx, const spdz_bmtriple_t* t, const uint32_t* own_payload,
                              const uint32_t* const* peer_payload, int n_peers, spdz_share_t* z, uint32_t* opened_out) {
    return guard([&] {
        need_ctx(ctx);
        check_bmtriple(t);
        need_share(z, "z");
        check_lanes(z->lanes, (uint64_t)t->dout * t->batch);
        need(own_payload && opened_out, SPDZ_ERR_INVALID_ARGUMENT, "null payload / opened_out");
        need(n_peers >= 0 && n_peers <= kMaxPeers && (n_peers == 0 || peer_payload), SPDZ_ERR_INVALID_ARGUMENT,
             "n_peers out of range");
        need(modgemm_tc_supported(t->din), SPDZ_ERR_INVALID_ARGUMENT, "batched secret x secret layer needs din >= 1");
        device_guard(ctx);
        const uint64_t cells = (uint64_t)t->dout * t->din, ecount = (uint64_t)t->din * t->batch;
        // open [D|E] (net.cpp:170-215): one pass over both halves
        launch_ok(launch_open_sum(ctx->stream, own_payload, peer_payload, n_peers, opened_out, cells + ecount,
                                  ctx->sms),
                  "open [D|E]");
        if (t->dout == 0 || t->batch == 0) return;
        const uint32_t* D = opened_out;
        const uint32_t* E = opened_out + cells;
        const uint64_t scratch = std::max(modgemm_tc_scratch_bytes(0, t->dout, t->din, t->batch),
                                          modgemm_tc_scratch_bytes(1, t->dout, t->din, t->batch));
        uint8_t* sc = (uint8_t*)ctx->scratch.ensure(scratch);
        // Z = C + D [B.v + [p0] E | B.m + alpha_i E]   (spdz.cpp:117-123 regrouped, exact mod p)
        TcAux g1;
        g1.e = E;
        g1.coef0 = ctx->party == 0 ? 1u : 0u;
        g1.coef1 = ctx->alpha;
        g1.add0 = t->c.vals;
        g1.add1 = t->c.macs;
        launch_ok(launch_modgemm_tc(ctx->stream, 0, t->dout, t->din, t->batch, D, nullptr, t->b.vals, t->b.macs,
                                    z->vals, z->macs, sc, ctx->sms, &g1),
                  "k_modgemm_tc (D B')");
        // Z += [A.v ; A.m] E
        TcAux g2;
        g2.add0 = z->vals;
        g2.add1 = z->macs;
        launch_ok(launch_modgemm_tc(ctx->stream, 1, t->dout, t->din, t->batch, t->a.vals, t->a.macs, E, nullptr,
                                    z->vals, z->macs, sc, ctx->sms, &g2),
                  "k_modgemm_tc (A E)");
    });
}

static int g_gemm_path = 0;  // 0 auto (tcgen05, K sliced by 8192), 1 CUDA-core, 2 tcgen05

int spdz_set_gemm_path(int path) {
    return guard([&] {
        need(path >= 0 && path <= 2, SPDZ_ERR_INVALID_ARGUMENT, "gemm path must be 0, 1 or 2");
        g_gemm_path = path;
    });
}

static void modgemm_dispatch(spdz_ctx* ctx, int mode, uint32_t dout, uint32_t din, uint32_t batch, const uint32_t* w0,
                             const uint32_t* w1, const uint32_t* x0, const uint32_t* x1, uint32_t* y0, uint32_t* y1) {
    const bool tc = g_gemm_path == 2 || (g_gemm_path == 0 && modgemm_tc_supported(din));
    if (tc) {
        need(modgemm_tc_supported(din), SPDZ_ERR_INVALID_ARGUMENT, "tcgen05 GEMM path needs din >= 1");
        uint8_t* scratch = (uint8_t*)ctx->scratch.ensure(modgemm_tc_scratch_bytes(mode, dout, din, batch));
        launch_ok(launch_modgemm_tc(ctx->stream, mode, dout, din, batch, w0, w1, x0, x1, y0, y1, scratch, ctx->sms),
                  "k_modgemm_tc");
    } else {
        launch_ok(launch_modgemm(ctx->stream, mode, dout, din, batch, w0, w1, x0, x1, y0, y1), "k_modgemm");
    }
}

struct spdz_linear_weights {
    int device = 0;
    uint32_t dout = 0, din = 0;
    uint8_t* image = nullptr;  // tcgen05 A-side limb image of W
};

int spdz_linear_weights_create(spdz_ctx* ctx, uint32_t dout, uint32_t din, const uint32_t* w_public,
                               spdz_linear_weights** out) {
    return guard([&] {
        need_ctx(ctx);
        need(out && (w_public || din == 0 || dout == 0), SPDZ_ERR_INVALID_ARGUMENT, "bad weights args");
        need(din >= 1 && din <= 8192, SPDZ_ERR_INVALID_ARGUMENT, "prepared weights need 1 <= din <= 8192");
        device_guard(ctx);
        auto* w = new spdz_linear_weights;
        w->device = ctx->device;
        w->dout = dout;
        w->din = din;
        try {
            cuda_check(cudaMalloc(&w->image, std::max<uint64_t>(modgemm_tc_a_image_bytes(0, dout, din), 16)),
                       "cudaMalloc(weights)");
            if (dout)
                launch_ok(launch_tile_a(ctx->stream, 0, dout, din, w_public, w_public, w->image, ctx->sms),
                          "tile W");
        } catch (...) {
            if (w->image) cudaFree(w->image);
            delete w;
            throw;
        }
        *out = w;
    });
}

int spdz_linear_weights_destroy(spdz_linear_weights* w) {
    return guard([&] {
        if (!w) return;
        cudaSetDevice(w->device);
        cudaDeviceSynchronize();  // the image may still be read by queued GEMMs
        if (w->image) cudaFree(w->image);
        delete w;
    });
}

int spdz_linear_secret_public_prepared(spdz_ctx* ctx, const spdz_linear_weights* w, uint32_t batch,
                                       const spdz_share_t* x_secret, spdz_share_t* y) {
    return guard([&] {  // runtime.cpp:303-334 with W's re-layout done once (spdz_linear_weights_create)
        need_ctx(ctx);
        need(w != nullptr, SPDZ_ERR_INVALID_ARGUMENT, "null weights");
        need(w->device == ctx->device, SPDZ_ERR_INVALID_ARGUMENT, "weights live on another device");
        need_share(x_secret, "x");
        need_share(y, "y");
        check_lanes(x_secret->lanes, (uint64_t)w->din * batch);
        check_lanes(y->lanes, (uint64_t)w->dout * batch);
        device_guard(ctx);
        if (w->dout == 0 || batch == 0) return;
        uint8_t* scratch = (uint8_t*)ctx->scratch.ensure(modgemm_tc_scratch_bytes(0, w->dout, w->din, batch));
        TcAux aux;
        aux.a_image = w->image;
        launch_ok(launch_modgemm_tc(ctx->stream, 0, w->dout, w->din, batch, nullptr, nullptr, x_secret->vals,
                                    x_secret->macs, y->vals, y->macs, scratch, ctx->sms, &aux),
                  "k_modgemm_tc (prepared W)");
    });
}

int spdz_linear_secret_public(spdz_ctx* ctx, uint32_t din, uint32_t dout, uint32_t batch, int w_public,
                              const uint32_t* w_vals, const spdz_share_t* w_secret, const spdz_share_t* x_secret,
                              const uint32_t* x_pub, spdz_share_t* y) {
    return guard([&] {  // runtime.cpp:303-334
        need_ctx(ctx);
        need_share(y, "y");
        check_lanes(y->lanes, (uint64_t)dout * batch);
        device_guard(ctx);
        if (w_public) {
            need_share(x_secret, "x");
            check_lanes(x_secret->lanes, (uint64_t)din * batch);
            need(w_vals != nullptr || din == 0, SPDZ_ERR_INVALID_ARGUMENT, "null W");
            modgemm_dispatch(ctx, 0, dout, din, batch, w_vals, nullptr, x_secret->vals, x_secret->macs, y->vals,
                             y->macs);
        } else {
            need_share(w_secret, "w");
            check_lanes(w_secret->lanes, (uint64_t)din * dout);
            need(x_pub != nullptr || din == 0, SPDZ_ERR_INVALID_ARGUMENT, "null x");
            modgemm_dispatch(ctx, 1, dout, din, batch, w_secret->vals, w_secret->macs, x_pub, nullptr, y->vals,
                             y->macs);
        }
    });
}

// ---------------- GPU dealer ----------------
int spdz_dealer_alpha(int n, uint64_t seed, uint32_t* shares, uint32_t* alpha) {
    return guard([&] {
        need(n >= 1 && n <= SPDZ_MAX_PARTIES && shares && alpha, SPDZ_ERR_INVALID_ARGUMENT, "bad dealer args");
        dealer_alpha(n, seed, shares, alpha);
    });
}
uint64_t spdz_dealer_draws_triples(int n, uint64_t lanes) { return dealer_draws_triples(n, lanes); }
uint64_t spdz_dealer_draws_share(int n, uint64_t lanes) { return dealer_draws_share(n, lanes); }
uint64_t spdz_dealer_draws_matrix(int n, uint32_t din, uint32_t rows) { return dealer_draws_matrix(n, din, rows); }
uint64_t spdz_dealer_draws_masks(int n, uint64_t count) { return dealer_draws_masks(n, count); }

int spdz_dealer_triples(spdz_ctx* ctx, int n, uint64_t seed, uint64_t draw0, uint64_t lanes, uint32_t* const planes[6]) {
    return guard([&] {
        need_ctx(ctx);
        device_guard(ctx);
        uint32_t sh[SPDZ_MAX_PARTIES], alpha;
        dealer_alpha(n, seed, sh, &alpha);
        cuda_check(cudaMemsetAsync(ctx->d_flag, 0, 4, ctx->stream), "memset");
        launch_ok(launch_dealer_triples(ctx->stream, n, seed, draw0, alpha, lanes, 0, lanes, lanes, planes, ctx->d_flag,
                                        ctx->sms),
                  "k_dealer_triples");
        check_dealer_flag(ctx);
    });
}

int spdz_dealer_share(spdz_ctx* ctx, int n, uint64_t seed, uint64_t draw0, uint32_t alpha, const uint32_t* clear,
                      uint64_t lanes, uint32_t* vals, uint32_t* macs) {
    return guard([&] {
        need_ctx(ctx);
        device_guard(ctx);
        cuda_check(cudaMemsetAsync(ctx->d_flag, 0, 4, ctx->stream), "memset");
        launch_ok(launch_dealer_share(ctx->stream, n, seed, draw0, alpha, clear, lanes, vals, macs, lanes,
                                      ctx->d_flag, ctx->sms),
                  "k_dealer_share");
        check_dealer_flag(ctx);
    });
}

// spdz.cpp:227-249; scratch >= (rows*din + din + rows) words
int spdz_dealer_matrix_triple(spdz_ctx* ctx, int n, uint64_t seed, uint64_t draw0, uint32_t alpha, uint32_t din,
                              uint32_t rows, uint32_t* const planes[6], uint32_t* scratch) {
    return guard([&] {
        need_ctx(ctx);
        device_guard(ctx);
        const uint64_t cells = (uint64_t)din * rows;
        uint32_t* A = scratch;
        uint32_t* B = scratch + cells;
        uint32_t* Cc = B + din;
        cuda_check(cudaMemsetAsync(ctx->d_flag, 0, 4, ctx->stream), "memset");
        uint64_t k = draw0;
        launch_ok(launch_dealer_uniform(ctx->stream, seed, k, cells, 1, A, ctx->d_flag, ctx->sms), "uniform A");
        k += cells;
        launch_ok(launch_dealer_uniform(ctx->stream, seed, k, din, 1, B, ctx->d_flag, ctx->sms), "uniform B");
        k += din;
        launch_ok(launch_dealer_matvec(ctx->stream, A, B, din, rows, Cc), "matvec C");
        launch_ok(launch_dealer_share(ctx->stream, n, seed, k, alpha, A, cells, planes[0], planes[1], cells,
                                      ctx->d_flag, ctx->sms),
                  "share A");
        k += dealer_draws_share(n, cells);
        launch_ok(launch_dealer_share(ctx->stream, n, seed, k, alpha, B, din, planes[2], planes[3], din,
                                      ctx->d_flag, ctx->sms),
                  "share B");
        k += dealer_draws_share(n, din);
        launch_ok(launch_dealer_share(ctx->stream, n, seed, k, alpha, Cc, rows, planes[4], planes[5], rows,
                                      ctx->d_flag, ctx->sms),
                  "share C");
        check_dealer_flag(ctx);
    });
}

int spdz_dealer_masks(spdz_ctx* ctx, int n, uint64_t seed, uint64_t draw0, uint32_t alpha, uint64_t count,
                      uint32_t* vals, uint32_t* macs, uint32_t* clear) {
    return guard([&] {
        need_ctx(ctx);
        device_guard(ctx);
        cuda_check(cudaMemsetAsync(ctx->d_flag, 0, 4, ctx->stream), "memset");
        launch_ok(launch_dealer_masks(ctx->stream, n, seed, draw0, alpha, 0, count, count, vals, macs, clear, ctx->d_flag,
                                      ctx->sms),
                  "k_dealer_masks");
        check_dealer_flag(ctx);
    });
}

// ---------------- host-buffer Backend (CpuBackend call shape) ----------------
namespace {
struct Staging {
    spdz_ctx* ctx;
    char* base;
    size_t off = 0;
    Staging(spdz_ctx* c, size_t bytes) : ctx(c) { base = (char*)c->scratch.ensure(bytes + 64 * 16); }
    uint32_t* take(uint64_t words) {
        uint32_t* p = (uint32_t*)(base + off);
        off += (words * 4 + 15) / 16 * 16;
        return p;
    }
    // Pageable host vectors (the reference Backend's std::vector operands) are copied by the
    // driver directly: through the pinned staging ring (hostcopy.cu) the 2^20-lane add measured
    // 4.0 ms against 2.1 ms (fresh output vectors fault their pages in the copy-out; the ring's
    // hand-offs cost more than they save at 4-16 MB per call), mask+combine 6.1 against 6.5 ms
    // (scripts/hostapi_probe.py, profiles/r02i_hostapi.log).  The run-input path keeps the ring
    // (run.cu: 13.4 -> 5.2 ms per pageable e2e step).
    // SPDZ_HOST_STAGING (experiments): bit 0 stages pageable H2D copies, bit 1 pageable D2H copies
    static int staging_mode() {
        static const int m = [] {
            const char* e = std::getenv("SPDZ_HOST_STAGING");
            return e ? std::atoi(e) : 0;
        }();
        return m;
    }
    uint32_t* up(const uint32_t* h, uint64_t words) {
        uint32_t* d = take(words);
        if ((staging_mode() & 1) && words * 4 >= (1u << 20) && is_pageable(h))
            cuda_check(staged_h2d(ctx->device, d, h, words * 4, ctx->stream), "staged H2D");
        else if (words)
            cuda_check(cudaMemcpyAsync(d, h, words * 4, cudaMemcpyHostToDevice, ctx->stream), "H2D");
        return d;
    }
    void down(uint32_t* h, const uint32_t* d, uint64_t words) {
        if ((staging_mode() & 2) && words * 4 >= (1u << 20) && is_pageable(h))
            cuda_check(staged_d2h(ctx->device, h, d, words * 4, ctx->stream), "staged D2H");
        else if (words)
            cuda_check(cudaMemcpyAsync(h, d, words * 4, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
    }
    void sync() { cuda_check(cudaStreamSynchronize(ctx->stream), "sync"); }
};
}  // namespace

static int host_add_sub(spdz_ctx* ctx, const uint32_t* xv, const uint32_t* xm, uint64_t nx, const uint32_t* yv,
                        const uint32_t* ym, uint64_t ny, uint32_t* zv, uint32_t* zm, bool sub) {
    return guard([&] {
        need_ctx(ctx);
        check_lanes(nx, ny);
        device_guard(ctx);
        Staging st(ctx, nx * 4 * 6);
        spdz_share_t x{st.up(xv, nx), st.up(xm, nx), nx}, y{st.up(yv, ny), st.up(ym, ny), ny};
        spdz_share_t z{st.take(nx), st.take(nx), nx};
        launch_ok(launch_add_sub(ctx->stream, sub, x.vals, x.macs, y.vals, y.macs, z.vals, z.macs, nx, ctx->sms),
                  "k_add_sub");
        st.down(zv, z.vals, nx);
        st.down(zm, z.macs, nx);
        st.sync();
    });
}
int spdz_host_add_batch(spdz_ctx* c, const uint32_t* xv, const uint32_t* xm, uint64_t nx, const uint32_t* yv,
                        const uint32_t* ym, uint64_t ny, uint32_t* zv, uint32_t* zm) {
    return host_add_sub(c, xv, xm, nx, yv, ym, ny, zv, zm, false);
}
int spdz_host_sub_batch(spdz_ctx* c, const uint32_t* xv, const uint32_t* xm, uint64_t nx, const uint32_t* yv,
                        const uint32_t* ym, uint64_t ny, uint32_t* zv, uint32_t* zm) {
    return host_add_sub(c, xv, xm, nx, yv, ym, ny, zv, zm, true);
}

int spdz_host_mul_mask(spdz_ctx* ctx, const uint32_t* xv, const uint32_t* yv, uint64_t lanes,
                       const uint32_t* const tri[6], uint64_t t_lanes, uint32_t* d_out, uint32_t* e_out) {
    return guard([&] {
        need_ctx(ctx);
        if (t_lanes != lanes)
            throw Error(SPDZ_ERR_TRIPLE_SHORTAGE, "TripleShortage: request carries " + std::to_string(t_lanes) +
                                                      " triples for " + std::to_string(lanes) + " lanes");
        device_guard(ctx);
        Staging st(ctx, lanes * 4 * 6);
        uint32_t* dx = st.up(xv, lanes);
        uint32_t* dy = st.up(yv, lanes);
        uint32_t* da = st.up(tri[0], lanes);
        uint32_t* db = st.up(tri[2], lanes);
        uint32_t* dd = st.take(lanes);
        uint32_t* de = st.take(lanes);
        launch_ok(launch_mul_mask(ctx->stream, dx, dy, da, db, dd, de, lanes, ctx->sms), "k_mul_mask");
        st.down(d_out, dd, lanes);
        st.down(e_out, de, lanes);
        st.sync();
    });
}

int spdz_host_mul_combine(spdz_ctx* ctx, const uint32_t* const tri[6], uint64_t t_lanes, const uint32_t* d,
                          const uint32_t* e, uint64_t lanes, int party, uint32_t alpha_share, uint32_t* zv,
                          uint32_t* zm) {
    return guard([&] {
        need_ctx(ctx);
        if (t_lanes != lanes) throw Error(SPDZ_ERR_TRIPLE_SHORTAGE, "TripleShortage: combine with mismatched triple count");
        device_guard(ctx);
        Staging st(ctx, lanes * 4 * 12);
        const uint32_t* t6[6];
        for (int k = 0; k < 6; ++k) t6[k] = st.up(tri[k], lanes);
        uint32_t* dd = st.up(d, lanes);
        uint32_t* de = st.up(e, lanes);
        uint32_t* ov = st.take(lanes);
        uint32_t* om = st.take(lanes);
        launch_ok(launch_beaver_combine(ctx->stream, dd, de, nullptr, nullptr, 0, t6, party, alpha_share, ov, om,
                                        nullptr, nullptr, lanes, ctx->sms),
                  "k_combine");
        st.down(zv, ov, lanes);
        st.down(zm, om, lanes);
        st.sync();
    });
}

int spdz_host_reduce_add(spdz_ctx* ctx, const uint32_t* xv, const uint32_t* xm, uint64_t lanes, uint32_t* zv,
                         uint32_t* zm) {
    return guard([&] {
        need_ctx(ctx);
        device_guard(ctx);
        Staging st(ctx, lanes * 4 * 2 + 64);
        uint32_t* dv = st.up(xv, lanes);
        uint32_t* dm = st.up(xm, lanes);
        uint32_t* o = st.take(2);
        cuda_check(cudaMemsetAsync(ctx->d_acc + 2, 0, 16, ctx->stream), "memset");
        launch_ok(launch_reduce_add(ctx->stream, dv, dm, lanes, ctx->d_acc + 2, ctx->sms), "reduce");
        launch_ok(launch_finish_reduce(ctx->stream, ctx->d_acc + 2, o, o + 1), "finish");
        st.down(zv, o, 1);
        st.down(zm, o + 1, 1);
        st.sync();
    });
}

// ---------------- device buffers and completion events ----------------
int spdz_share_alloc(spdz_ctx* ctx, uint64_t lanes, spdz_share_t* out) {
    return guard([&] {
        need_ctx(ctx);
        need(out != nullptr, SPDZ_ERR_INVALID_ARGUMENT, "null share");
        device_guard(ctx);
        void *v = nullptr, *m = nullptr;
        cuda_check(cudaMalloc(&v, std::max<uint64_t>(lanes, 1) * 4), "cudaMalloc(share)");
        if (cudaMalloc(&m, std::max<uint64_t>(lanes, 1) * 4) != cudaSuccess) {
            cudaFree(v);
            throw Error(SPDZ_ERR_CUDA, "cudaMalloc(share): out of device memory");
        }
        *out = spdz_share_t{(uint32_t*)v, (uint32_t*)m, lanes};
    });
}

int spdz_share_free(spdz_ctx* ctx, spdz_share_t* s) {
    return guard([&] {
        need_ctx(ctx);
        if (!s) return;
        device_guard(ctx);
        cuda_check(cudaStreamSynchronize(ctx->stream), "sync before free");
        if (s->vals) cudaFree(s->vals);
        if (s->macs) cudaFree(s->macs);
        *s = spdz_share_t{nullptr, nullptr, 0};
    });
}

int spdz_share_upload(spdz_ctx* ctx, spdz_share_t* dst, const uint32_t* hv, const uint32_t* hm, uint64_t lanes) {
    return guard([&] {
        need_ctx(ctx);
        need_share(dst, "dst");
        need(lanes <= dst->lanes && (lanes == 0 || (hv && hm)), SPDZ_ERR_INVALID_ARGUMENT, "bad upload");
        device_guard(ctx);
        cuda_check(cudaMemcpyAsync(dst->vals, hv, lanes * 4, cudaMemcpyHostToDevice, ctx->stream), "H2D vals");
        cuda_check(cudaMemcpyAsync(dst->macs, hm, lanes * 4, cudaMemcpyHostToDevice, ctx->stream), "H2D macs");
    });
}

int spdz_share_download(spdz_ctx* ctx, const spdz_share_t* src, uint32_t* hv, uint32_t* hm, uint64_t lanes) {
    return guard([&] {
        need_ctx(ctx);
        need_share(src, "src");
        need(lanes <= src->lanes && (lanes == 0 || (hv && hm)), SPDZ_ERR_INVALID_ARGUMENT, "bad download");
        device_guard(ctx);
        cuda_check(cudaMemcpyAsync(hv, src->vals, lanes * 4, cudaMemcpyDeviceToHost, ctx->stream), "D2H vals");
        cuda_check(cudaMemcpyAsync(hm, src->macs, lanes * 4, cudaMemcpyDeviceToHost, ctx->stream), "D2H macs");
    });
}

}  // extern "C"

struct spdz_event {
    cudaEvent_t ev = nullptr;
    int device = 0;
};

extern "C" {

int spdz_event_record(spdz_ctx* ctx, spdz_event** out) {
    return guard([&] {
        need_ctx(ctx);
        need(out != nullptr, SPDZ_ERR_INVALID_ARGUMENT, "null event");
        device_guard(ctx);
        auto* e = new spdz_event;
        e->device = ctx->device;
        if (cudaEventCreateWithFlags(&e->ev, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventRecord(e->ev, ctx->stream) != cudaSuccess) {
            if (e->ev) cudaEventDestroy(e->ev);
            delete e;
            throw Error(SPDZ_ERR_CUDA, "event record failed");
        }
        *out = e;
    });
}

int spdz_event_query(spdz_event* e, int* done) {
    return guard([&] {
        need(e != nullptr && done != nullptr, SPDZ_ERR_INVALID_ARGUMENT, "null event");
        cudaSetDevice(e->device);
        const cudaError_t r = cudaEventQuery(e->ev);
        if (r == cudaErrorNotReady) {
            cudaGetLastError();  // not an error: clear it
            *done = 0;
            return;
        }
        cuda_check(r, "cudaEventQuery");
        *done = 1;
    });
}

int spdz_event_sync(spdz_event* e) {
    return guard([&] {
        need(e != nullptr, SPDZ_ERR_INVALID_ARGUMENT, "null event");
        cudaSetDevice(e->device);
        cuda_check(cudaEventSynchronize(e->ev), "cudaEventSynchronize");
    });
}

int spdz_event_wait(spdz_ctx* ctx, spdz_event* e) {
    return guard([&] {
        need_ctx(ctx);
        need(e != nullptr, SPDZ_ERR_INVALID_ARGUMENT, "null event");
        device_guard(ctx);
        cuda_check(cudaStreamWaitEvent(ctx->stream, e->ev, 0), "cudaStreamWaitEvent");
    });
}

int spdz_event_destroy(spdz_event* e) {
    if (!e) return SPDZ_OK;
    cudaSetDevice(e->device);
    cudaEventDestroy(e->ev);
    delete e;
    return SPDZ_OK;
}

// ---------------- caller-driven MAC log (runtime.cpp:112-117, 467-506) ----------------
int spdz_mac_log_append(spdz_ctx* ctx, uint64_t batch_id, const uint32_t* dev_opened, const uint32_t* dev_mac,
                        const uint32_t* dev_mac_sub, uint64_t len) {
    return guard([&] {
        need_ctx(ctx);
        need(len == 0 || (dev_opened && dev_mac), SPDZ_ERR_INVALID_ARGUMENT, "null log arrays");
        if (!len) return;
        std::lock_guard lk(ctx->maclog_mu);
        uint64_t& lane0 = ctx->maclog_lanes[batch_id];  // log_open lanes continue within a batch
        ctx->maclog.push_back({dev_opened, dev_mac, dev_mac_sub, len, 0, batch_id, lane0, 0});
        lane0 += len;
    });
}

int spdz_mac_log_size(spdz_ctx* ctx, uint64_t* n) {
    return guard([&] {
        need_ctx(ctx);
        need(n != nullptr, SPDZ_ERR_INVALID_ARGUMENT, "null out");
        std::lock_guard lk(ctx->maclog_mu);
        uint64_t k = 0;
        for (auto& sg : ctx->maclog) k += sg.len;
        *n = k;
    });
}

int spdz_mac_log_sigma(spdz_ctx* ctx, uint64_t coin, uint32_t* sigma_out) {
    return guard([&] {
        need_ctx(ctx);
        need(sigma_out != nullptr, SPDZ_ERR_INVALID_ARGUMENT, "null sigma_out");
        std::vector<spdz_mac_segment_t> segs;
        {
            std::lock_guard lk(ctx->maclog_mu);
            segs = ctx->maclog;
            for (auto& sg : segs) sg.batch_len = ctx->maclog_lanes[sg.batch_id];
        }
        assign_ranks(segs.data(), segs.size());
        device_guard(ctx);
        *sigma_out = segs.empty() ? 0u : mac_sigma_impl(ctx, segs.data(), segs.size(), coin);
    });
}

int spdz_mac_log_clear(spdz_ctx* ctx) {
    return guard([&] {
        need_ctx(ctx);
        std::lock_guard lk(ctx->maclog_mu);
        ctx->maclog.clear();
        ctx->maclog_lanes.clear();
    });
}

}  // extern "C"
