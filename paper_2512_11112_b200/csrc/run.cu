// Local n-party online phase over device-resident state: the batch executor
// that replaces PartyRuntime::Impl's node drivers (runtime.cpp:129-506) for
// straight-line circuits.  Parties are CUDA streams (optionally on distinct
// devices); the opening exchange is a peer-buffer read fused into the combine
// kernels, ordered by per-party events (the batch-id matching of
// net.cpp:61-95 becomes stream/event ordering).  Every share, triple pool,
// opened-value log and MAC record lives in HBM as structure-of-arrays.
#include "hostcopy.hpp"
#include "run_exec.hpp"
#include "run_state.hpp"

namespace {

uint64_t fresh_nonce() {
    static thread_local std::mt19937_64 rng(std::random_device{}());
    return rng();
}

// runtime.cpp:467-506
uint64_t agree_coin(spdz_run* r, bool have_coin, uint64_t given_coin) {
    const int n = r->n;
    uint64_t coin = 0;
    if (have_coin) {
        coin = given_coin;
    } else if (r->opts.fixed_coin) {
        coin = r->opts.coin;
    } else {  // commit to nonces, reveal, chain fnv1a64 (runtime.cpp:474-489)
        std::vector<uint64_t> nonce(n), commit(n);
        for (int p = 0; p < n; ++p) {
            nonce[p] = fresh_nonce();
            commit[p] = spdz_fnv1a64(&nonce[p], 8, 1469598103934665603ull);
        }
        for (int p = 0; p < n; ++p) {
            if (spdz_fnv1a64(&nonce[p], 8, 1469598103934665603ull) != commit[p])
                throw Error(SPDZ_ERR_MAC_CHECK_FAILED, "MacCheckFailed: coin commitment mismatch");
            coin = spdz_fnv1a64(&nonce[p], 8, coin);
        }
    }
    return coin;
}

// sigma kernels of every local party (asynchronous)
// Both parties of a 2-party run local on one stream with rank-identical logs: one pass
// (the coefficient stream r_j is the same for both, spdz.cpp:131-135).
bool mac_fusable(spdz_run* r) {
    if (!colocated2(r)) return false;
    const auto &a = r->parties[0].maclog, &b = r->parties[1].maclog;
    if (a.size() != b.size()) return false;
    for (size_t i = 0; i < a.size(); ++i)
        if (a[i].len != b[i].len || a[i].j0 != b[i].j0 || (a[i].mac_b == nullptr) != (b[i].mac_b == nullptr) ||
            !a[i].value || !a[i].mac_a || !b[i].value || !b[i].mac_a)
            return false;
    return true;
}

void mac_launch(spdz_run* r, uint64_t coin) {
    NvtxRange range("mac check sigma");
    for (int p = 0; p < r->n; ++p)
        if (r->parties[p].local) assign_ranks(r->parties[p].maclog.data(), r->parties[p].maclog.size());
    if (mac_fusable(r)) {
        auto &P0 = r->parties[0], &P1 = r->parties[1];
        dev(r, 0);
        cudaStream_t s = S(r, 0);
        uint64_t sbytes = 0;  // per record: each party's mac_a (+ mac_b), the opened value once if shared
        for (size_t i = 0; i < P0.maclog.size(); ++i) {
            const auto &a = P0.maclog[i], &b = P1.maclog[i];
            sbytes += a.len * ((a.mac_b ? 16 : 8) + (a.value == b.value ? 4 : 8));
        }
        const int tk = ktimer_begin(r, 0);
        lk(cudaMemsetAsync(P0.ctx->d_acc, 0, 8, s), "memset acc");
        lk(cudaMemsetAsync(P1.ctx->d_acc, 0, 8, s), "memset acc");
        const auto &L0 = P0.maclog, &L1 = P1.maclog;
        for (size_t base = 0; base < L0.size(); base += kMacTableSegs) {
            MacTableT<2> tab{};
            tab.n = (uint32_t)std::min<size_t>(kMacTableSegs, L0.size() - base);
            uint64_t recs = 0;
            for (uint32_t i = 0; i < tab.n; ++i) {
                const auto &a = L0[base + i], &b = L1[base + i];
                tab.seg[i] = MacSegT<2>{{a.value, b.value}, {a.mac_a, b.mac_a}, {a.mac_b, b.mac_b}, a.len, a.j0};
                tab.rec0[i] = recs;
                recs += a.len;
            }
            tab.rec0[tab.n] = recs;
            const uint32_t alpha[2] = {P0.ctx->alpha, P1.ctx->alpha};
            unsigned long long* const acc[2] = {P0.ctx->d_acc, P1.ctx->d_acc};
            lk(launch_mac_sigma2(s, tab, coin, alpha, acc, P0.ctx->sms), "k_mac_sigma<2>");
        }
        ktimer_end(r, 0, tk, SPDZ_KSTAT_SIGMA, sbytes);
        lk(cudaEventRecord(P0.t1, s), "t1");
        lk(cudaEventRecord(P1.t1, s), "t1");
        return;
    }
    for (int p = 0; p < r->n; ++p) {
        auto& P = r->parties[p];
        if (!P.local) continue;
        dev(r, p);
        uint64_t sbytes = 0;
        for (auto& sg : P.maclog) sbytes += sg.len * (sg.mac_b ? 12 : 8);
        const int tk = ktimer_begin(r, p);
        mac_sigma_launch(P.ctx, P.maclog.data(), P.maclog.size(), coin, 0);
        ktimer_end(r, p, tk, SPDZ_KSTAT_SIGMA, sbytes);
        lk(cudaEventRecord(P.t1, P.ctx->stream), "t1");
    }
}

// collect sigmas, commit/verify (spdz.cpp:140-158)
void mac_finish(spdz_run* r, spdz_run_report_t* rep, uint64_t coin) {
    const int n = r->n;
    std::vector<uint32_t> sig(n);
    std::vector<uint64_t> nonce2(n), commits(n);
    for (int p = 0; p < n; ++p) {
        if (!r->parties[p].local) {  // another process reports this party's sigma
            sig[p] = 0;
            if (rep) rep->sigmas[p] = 0;
            continue;
        }
        dev(r, p);
        sig[p] = mac_sigma_collect(r->parties[p].ctx, 0);
        nonce2[p] = fresh_nonce();
        commits[p] = spdz_commit_sigma(sig[p], nonce2[p]);
        if (rep) rep->sigmas[p] = sig[p];
    }
    if (rep) rep->coin = coin;
    if (r->opts.external_mac_verify) return;  // partial sigmas: the caller sums shards and verifies
    int rc = spdz_verify_sigmas(sig.data(), nonce2.data(), commits.data(), n);
    if (rc) throw Error(rc, spdz_last_error());
}

// runtime.cpp:467-506 across the mesh: coin from committed nonces, sigma commit/reveal,
// verify_sigmas over every party's reveal
void mac_check_net(spdz_run* r, spdz_run_report_t* rep) {
    NetLink& net = *r->net;
    const int n = r->n, me = r->ref_party();
    auto u64_of = [](const std::vector<uint32_t>& v, size_t at) {
        need(v.size() >= at + 2, SPDZ_ERR_MALFORMED_SHARE_MESSAGE, "MalformedShareMessage: short MAC-check frame");
        return (uint64_t)v[at] | (uint64_t)v[at + 1] << 32;
    };
    const uint64_t nonce = fresh_nonce();
    const uint64_t commit = spdz_fnv1a64(&nonce, 8, 1469598103934665603ull);
    auto commits = net.exchange(kMsgCommit, kMacBatchBase, {(uint32_t)commit, (uint32_t)(commit >> 32)});
    auto nonces = net.exchange(kMsgReveal, kMacBatchBase + 1, {(uint32_t)nonce, (uint32_t)(nonce >> 32)});
    uint64_t coin = 0;
    for (int i = 0; i < n; ++i) {
        const uint64_t ni = u64_of(nonces[i], 0);
        if (spdz_fnv1a64(&ni, 8, 1469598103934665603ull) != u64_of(commits[i], 0))
            throw Error(SPDZ_ERR_MAC_CHECK_FAILED, "MacCheckFailed: coin commitment mismatch from party " +
                                                       std::to_string(i));
        coin = spdz_fnv1a64(&ni, 8, coin);
    }
    mac_launch(r, coin);
    dev(r, me);
    const uint32_t sigma = mac_sigma_collect(r->parties[me].ctx, 0);
    const uint64_t nonce2 = fresh_nonce();
    const uint64_t sc = spdz_commit_sigma(sigma, nonce2);
    auto scommits = net.exchange(kMsgCommit, kMacBatchBase + 2, {(uint32_t)sc, (uint32_t)(sc >> 32)});
    auto reveals = net.exchange(kMsgReveal, kMacBatchBase + 3, {sigma, (uint32_t)nonce2, (uint32_t)(nonce2 >> 32)});
    std::vector<uint32_t> sig(n);
    std::vector<uint64_t> n2(n), cm(n);
    for (int i = 0; i < n; ++i) {
        need(!reveals[i].empty(), SPDZ_ERR_MALFORMED_SHARE_MESSAGE, "MalformedShareMessage: empty reveal");
        sig[i] = reveals[i][0];
        n2[i] = u64_of(reveals[i], 1);
        cm[i] = u64_of(scommits[i], 0);
    }
    if (rep) {
        for (int i = 0; i < n; ++i) rep->sigmas[i] = sig[i];
        rep->coin = coin;
    }
    const int rc = spdz_verify_sigmas(sig.data(), n2.data(), cm.data(), n);
    if (rc) throw Error(rc, spdz_last_error());
}

void mac_check(spdz_run* r, spdz_run_report_t* rep, bool have_coin, uint64_t given_coin) {
    if (r->net) {
        mac_check_net(r, rep);
        return;
    }
    const uint64_t coin = agree_coin(r, have_coin, given_coin);
    mac_launch(r, coin);
    mac_finish(r, rep, coin);
}

// Input sharing of a 2-party run with both parties on one stream runs as one kernel per
// input (the bound input stays raw until then).
bool share_fused(spdz_run* r) {
    return colocated2(r);
}

void share_inputs(spdz_run* r) {
    // preproc.cpp:205-243: party 0 opens x - mask, everyone adds the public difference.
    // A mask is used once (take_masks, triple_store.cpp:156-161): sharing again with the same
    // preprocessing would open x' - r for the same r.
    if (!r->input_mask_off.empty()) {
        if (r->masks_used)
            throw Error(SPDZ_ERR_MASK_EXHAUSTED,
                        "MaskExhausted: the input masks of this preprocessing were already used (deal again)");
        r->masks_used = true;
    }
    ++r->seq;
    uint64_t input_batch = kInputBatchBase;  // preproc.cpp:207-231: one Control exchange per private input
    for (auto& [id, off] : r->input_mask_off) {
        const auto& n = r->node(id);
        if (r->net) {  // peers across the mesh: exchange(Control, batch, diff), party 0's diff opens
            need(r->net != nullptr, SPDZ_ERR_INVALID_ARGUMENT, "network run without an attached mesh");
            const uint64_t batch = input_batch++;
            const int me = r->ref_party();
            auto& P = r->parties[me];
            uint32_t* diff = r->input_diff.at(id);
            Exec ex{r};
            if (me == 0) {
                auto it = r->input_dev.find(id);
                need(it != r->input_dev.end(), SPDZ_ERR_INVALID_ARGUMENT,
                     "ShapeMismatch: no values bound for input node " + std::to_string(id));
                dev(r, 0);
                lk(launch_pub_binop(P.ctx->stream, 1, it->second, false, P.mask_c + off, false, diff, n.lanes,
                                    P.ctx->sms),
                   "x - r");
                ex.net_send(0, kMsgControl, batch, diff, n.lanes);
            } else {
                ex.net_send(me, kMsgControl, batch, nullptr, 0);
            }
            for (int q = 0; q < r->n; ++q) {
                if (q == me) continue;
                std::vector<uint32_t> v = r->net->recv(q, kMsgControl, batch);
                if (q != 0) continue;  // only party 0 owns inputs (preproc.cpp:231)
                need(v.size() == n.lanes, SPDZ_ERR_INVALID_ARGUMENT,
                     "ShapeMismatch: opened input difference has wrong length");
                uint32_t* h = (uint32_t*)r->net_stage.ensure(v.size() * 4);
                std::memcpy(h, v.data(), v.size() * 4);
                dev(r, me);
                lk(cudaMemcpyAsync(diff, h, v.size() * 4, cudaMemcpyHostToDevice, P.ctx->stream), "H2D diff");
                lk(cudaStreamSynchronize(P.ctx->stream), "diff");
            }
            dev(r, me);
            lk(launch_public(P.ctx->stream, 0, P.mask_v + off, P.mask_m + off, diff, false, 0u, false, me,
                             P.ctx->alpha, P.ns[id].out.v, P.ns[id].out.m, n.lanes, P.ctx->sms),
               "add_public(diff)");
            continue;
        }
        if (share_fused(r)) {  // both parties in one pass from the raw input (reduced inline)
            auto it = r->input_dev.find(id);
            need(it != r->input_dev.end(), SPDZ_ERR_INVALID_ARGUMENT,
                 "ShapeMismatch: no values bound for input node " + std::to_string(id));
            auto &P0 = r->parties[0], &P1 = r->parties[1];
            dev(r, 0);
            const uint32_t* mask[4] = {P0.mask_v + off, P0.mask_m + off, P1.mask_v + off, P1.mask_m + off};
            const uint32_t alpha[2] = {P0.ctx->alpha, P1.ctx->alpha};
            const uint32_t* alpha_dev[2] = {P0.ctx->d_alpha, P1.ctx->d_alpha};
            uint32_t* out[4] = {P0.ns[id].out.v, P0.ns[id].out.m, P1.ns[id].out.v, P1.ns[id].out.m};
            lk(launch_share_input2(S(r, 0), it->second, P0.mask_c + off, mask, alpha, alpha_dev, out, n.lanes,
                                   P0.ctx->sms),
               "share input (2 parties)");
            continue;
        }
        uint32_t* diff = r->input_diff[id];  // party 0's buffer (IPC-mapped when party 0 is remote)
        const uint64_t slot = slot_of(id, 63);
        if (r->parties[0].local) {
            auto it = r->input_dev.find(id);
            need(it != r->input_dev.end(), SPDZ_ERR_INVALID_ARGUMENT,
                 "ShapeMismatch: no values bound for input node " + std::to_string(id));
            uint32_t* x0 = it->second;  // reduced cleartext on party 0's device
            auto& P0 = r->parties[0];
            dev(r, 0);
            lk(launch_pub_binop(P0.ctx->stream, 1, x0, false, P0.mask_c + off, false, diff, n.lanes, P0.ctx->sms),
               "x - r");
            lk(cudaEventRecord(r->ev_input, P0.ctx->stream), "record");
            signal_remote(r, 0, slot);
        }
        need(diff != nullptr, SPDZ_ERR_INVALID_ARGUMENT, "input difference of party 0 not imported");
        for (int p = 0; p < r->n; ++p) {
            if (!r->parties[p].local) continue;
            auto& P = r->parties[p];
            auto& o = P.ns[id].out;
            dev(r, p);
            if (p) {
                if (r->parties[0].local) lk(cudaStreamWaitEvent(P.ctx->stream, r->ev_input, 0), "wait");
                else wait_remote(r, p, 0, slot);
            }
            lk(launch_public(P.ctx->stream, 0, P.mask_v + off, P.mask_m + off, diff, false, 0u, false, p,
                             P.ctx->alpha, o.v, o.m, n.lanes, P.ctx->sms),
               "add_public(diff)");
        }
    }
    for (uint32_t id = 0; id < r->nodes.size(); ++id) {  // public inputs and constants
        const auto& n = r->nodes[id];
        if (n.kind == SPDZ_NODE_INPUT && !n.is_private) {
            auto it = r->inputs.find(id);
            need(it != r->inputs.end(), SPDZ_ERR_INVALID_ARGUMENT,
                 "ShapeMismatch: missing public input " + std::to_string(id));
            auto& red = r->pub_reduced[id];  // lives until the next bind: the copies are asynchronous
            red.resize(it->second.size());
            for (size_t i = 0; i < red.size(); ++i) red[i] = it->second[i] % kP;
            for (int p = 0; p < r->n; ++p) {
                if (!r->parties[p].local) continue;
                dev(r, p);
                lk(cudaMemcpyAsync(r->parties[p].ns[id].out.pub, red.data(), red.size() * 4, cudaMemcpyHostToDevice,
                                   S(r, p)),
                   "H2D pub");
            }
        }
        if (n.kind == SPDZ_NODE_CONST && !r->consts_uploaded) {  // constants never change: once per run
            const uint32_t v = n.const_val % kP;
            for (int p = 0; p < r->n; ++p) {
                if (!r->parties[p].local) continue;
                dev(r, p);
                lk(cudaMemcpy(r->parties[p].ns[id].out.pub, &v, 4, cudaMemcpyHostToDevice), "H2D const");
            }
        }
    }
    r->consts_uploaded = true;
}

// The online phase may run as one CUDA graph: every party local on one shared stream,
// a lane-parallel circuit (no linear layers or reductions, whose launchers size scratch
// buffers and grids at call time), no fault injection, no per-kernel timing.
bool graphable(spdz_run* r) {
    if (!r->opts.use_graph || r->cfg || r->any_remote || !r->faults.empty()) return false;
    for (int p = 0; p < r->n; ++p)
        if (!r->parties[p].local || S(r, p) != S(r, 0)) return false;
    return true;
}

}  // namespace

namespace {
struct IpcEntry {
    uint32_t kind;  // 0 flags, 1 node payload, 2 reduce-level payload, 3 root values, 4 input difference
    uint32_t node, sub, pad;
    uint64_t offset;
    cudaIpcMemHandle_t handle;
};
struct IpcHeader {
    uint32_t magic, version, party, n;
};
constexpr uint32_t kIpcMagic = 0x5350445au;  // "SPDZ"

// every buffer a peer process reads, for local party p
template <class F>
void for_each_export(spdz_run* r, int p, F&& f) {
    auto& P = r->parties[p];
    f(0u, 0u, 0u, (void*)P.flags);
    for (uint32_t id = 0; id < r->nodes.size(); ++id) {
        auto& st = P.ns[id];
        if (st.payload) f(1u, id, 0u, (void*)st.payload);
        for (uint32_t li = 0; li < st.levels.size(); ++li) f(2u, id, li, (void*)st.levels[li].payload);
    }
    const Val& rv = P.ns[r->root].out;
    if (!rv.is_public) f(3u, r->root, 0u, (void*)rv.v);
    if (p == 0)
        for (auto& [id, d] : r->input_diff) f(4u, id, 0u, (void*)d);
}
}  // namespace

extern "C" {

int spdz_triple_layout(const spdz_node_t* nodes, uint32_t n_nodes, uint64_t slice, uint64_t loop_iters,
                       uint64_t* out, uint64_t cap, uint64_t* n_regions) {
    return guard([&] {  // host only: the planning step of spdz_run_create
        need(nodes && n_nodes > 0 && n_regions, SPDZ_ERR_INVALID_ARGUMENT, "bad layout arguments");
        spdz_run r;
        r.nodes.assign(nodes, nodes + n_nodes);
        r.opts.slice = slice ? slice : 262140;
        r.loop_iters = loop_iters ? loop_iters : 64;
        plan_layout(&r);
        uint64_t k = 0;
        for (int kind = 0; kind < 2; ++kind)
            for (auto& [id, reg] : kind == 0 ? r.scalar : r.matrix) {
                if (out && k < cap) {
                    uint64_t* o = out + 5 * k;
                    o[0] = kind;
                    o[1] = id;
                    o[2] = kind == 0 ? reg.gbase : reg.base;
                    o[3] = reg.stride;
                    o[4] = reg.max_execs;
                }
                ++k;
            }
        *n_regions = k;
    });
}

int spdz_run_create(const spdz_node_t* nodes, uint32_t n_nodes, uint32_t root, int n_parties,
                    const spdz_run_options_t* opts, spdz_run** out) {
    return guard([&] {
        need(nodes && n_nodes > 0 && out, SPDZ_ERR_INVALID_ARGUMENT, "bad run arguments");
        need(root < n_nodes, SPDZ_ERR_INVALID_ARGUMENT, "root out of range");
        need(n_parties >= 1 && n_parties <= SPDZ_MAX_PARTIES, SPDZ_ERR_INVALID_ARGUMENT, "n_parties out of range");
        auto r = std::make_unique<spdz_run>();
        r->nodes.assign(nodes, nodes + n_nodes);
        r->root = root;
        r->n = n_parties;
        if (opts) r->opts = *opts;
        if (r->opts.slice == 0) r->opts.slice = 262140;
        if (r->opts.dealer_seed == 0 && !opts) r->opts.dealer_seed = 1;
        r->loop_iters = r->opts.loop_iters ? r->opts.loop_iters : 64;
        for (uint32_t id = 0; id < n_nodes; ++id)
            if (nodes[id].kind == SPDZ_NODE_PHI || nodes[id].kind == SPDZ_NODE_BRANCH) r->cfg = true;
        for (uint32_t id = 0; id < n_nodes; ++id) {
            const auto& nd = nodes[id];
            need(nd.n_operands <= (nd.kind == SPDZ_NODE_PHI ? SPDZ_MAX_OPERANDS : 3u), SPDZ_ERR_INVALID_ARGUMENT,
                 "too many operands (phis take up to SPDZ_MAX_OPERANDS incoming edges, other nodes 3)");
            for (uint32_t k = 0; k < nd.n_operands; ++k)  // a phi may read a later node (loop back edge)
                need(nd.kind == SPDZ_NODE_PHI ? nd.operands[k] < n_nodes : nd.operands[k] < id,
                     SPDZ_ERR_INVALID_ARGUMENT, "graph must be topologically ordered (operand id < node id)");
            if (r->cfg && nd.next != SPDZ_NO_NODE)
                need(nd.next < n_nodes, SPDZ_ERR_INVALID_ARGUMENT, "block chain leaves the graph");
            if (nd.kind == SPDZ_NODE_BRANCH)
                for (uint32_t k = 0; k < nd.n_succ && k < 2; ++k)
                    need(nd.succ[k] < n_nodes, SPDZ_ERR_INVALID_ARGUMENT, "branch target out of range");
        }
        if (r->cfg) {
            need(r->opts.entry_label < n_nodes && nodes[r->opts.entry_label].kind == SPDZ_NODE_LABEL,
                 SPDZ_ERR_INVALID_ARGUMENT, "control-flow graph needs entry_label = its entry block's LABEL");
            need(!r->opts.shard_total && (!r->opts.single_party || r->opts.network), SPDZ_ERR_INVALID_ARGUMENT,
                 "control-flow graphs run unsharded, with every party local or across a network mesh");
        }
        r->devices.resize(n_parties);
        for (int p = 0; p < n_parties; ++p) r->devices[p] = (opts && opts->devices[p] >= 0) ? opts->devices[p] : 0;
        r->parties.resize(n_parties);
        if (r->opts.single_party > 0) {  // one party per process; peers arrive via spdz_run_import
            need(r->opts.single_party <= n_parties, SPDZ_ERR_INVALID_ARGUMENT, "single_party out of range");
            for (int p = 0; p < n_parties; ++p) r->parties[p].local = p == r->opts.single_party - 1;
            r->any_remote = n_parties > 1;
            need(r->opts.external_mac_verify || r->opts.network, SPDZ_ERR_INVALID_ARGUMENT,
                 "single_party runs need external_mac_verify = 1 (sigmas are combined across processes)");
            if (!r->opts.network) load_stream_memops();
        }
        for (int p = 0; p < n_parties; ++p) {
            if (!r->parties[p].local) continue;
            int rc = spdz_ctx_create(r->devices[p], p, n_parties, 0, &r->parties[p].ctx);
            if (rc) throw Error(rc, spdz_last_error());
            if (!r->opts.stream_per_party)  // parties sharing a device share its stream
                for (int q = 0; q < p; ++q)
                    if (r->parties[q].local && r->devices[q] == r->devices[p]) {
                        r->parties[p].ctx->stream = r->parties[q].ctx->stream;
                        break;
                    }
        }
        for (int p = 0; p < n_parties; ++p)  // P2P between party devices (NVLink)
            for (int q = 0; q < n_parties; ++q) {
                if (!r->parties[p].local || !r->parties[q].local) continue;
                if (r->devices[p] == r->devices[q]) continue;
                cudaSetDevice(r->devices[p]);
                cudaError_t e = cudaDeviceEnablePeerAccess(r->devices[q], 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                else cuda_check(e, "cudaDeviceEnablePeerAccess");
            }
        if (r->opts.shard_total) {
            need(!r->cfg, SPDZ_ERR_INVALID_ARGUMENT, "sharded runs are straight-line");
            r->shard_off = r->opts.shard_offset;
            r->shard_total = r->opts.shard_total;
            for (auto& nd : r->nodes)
                if (nd.lanes > 1) r->shard_L = std::max<uint64_t>(r->shard_L, nd.lanes);
            need(r->shard_off + r->shard_L <= r->shard_total, SPDZ_ERR_INVALID_ARGUMENT, "shard outside the circuit");
        }
        plan_layout(r.get());
        compute_liveness(r.get());
        plan_buffers(r.get());
        alloc_deals(r.get());
        deal(r.get(), r->opts.dealer_seed);
        *out = r.release();
    });
}

int spdz_run_destroy(spdz_run* r) {
    return guard([&] {
        if (!r) return;
        for (auto& P : r->parties) {
            for (void* m : P.mapped) cudaIpcCloseMemHandle(m);
            if (!P.ctx) continue;
            cudaSetDevice(P.ctx->device);
            cudaStreamSynchronize(P.ctx->stream);
            for (auto e : P.evs) cudaEventDestroy(e);
            if (P.t0) cudaEventDestroy(P.t0);
            if (P.t1) cudaEventDestroy(P.t1);
            if (P.t_open) cudaEventDestroy(P.t_open);
        }
        if (r->ev_input) {
            cudaSetDevice(r->devices[r->ref_party()]);
            cudaEventDestroy(r->ev_input);
            cudaEventDestroy(r->ev_opened);
            cudaEventDestroy(r->ev_h2d);
            cudaEventDestroy(r->ev_out);
            cudaStreamSynchronize(r->copy_stream);
            cudaStreamDestroy(r->copy_stream);
        }
        for (auto& [d, v] : r->lane_streams) {
            cudaSetDevice(d);
            for (auto st : v) {
                cudaStreamSynchronize(st);
                cudaStreamDestroy(st);
            }
        }
        for (int p = 0; p < (int)r->node_ev.size(); ++p) {
            cudaSetDevice(r->devices[p]);
            for (auto e : r->node_ev[p])
                if (e) cudaEventDestroy(e);
            if (r->lane_fork[p]) cudaEventDestroy(r->lane_fork[p]);
        }
        if (r->online_graph) cudaGraphExecDestroy(r->online_graph);
        if (r->host_out_registered) cudaHostUnregister(r->host_out);
        for (auto e : r->kt.pool) cudaEventDestroy(e);
        for (size_t i = 0; i < r->allocs.size(); ++i) {
            cudaSetDevice(r->alloc_dev[i]);
            cudaFree(r->allocs[i]);
        }
        if (r->host_out && r->host_out_owned) cudaFreeHost(r->host_out);
        for (auto& P : r->parties) {
            if (!P.ctx) continue;
            if (P.ctx->stream != P.ctx->own_stream) P.ctx->stream = P.ctx->own_stream;
            spdz_ctx_destroy(P.ctx);
        }
        delete r;
    });
}

int spdz_run_load_store(spdz_run* r, int party, const char* path) {
    return guard([&] {
        need(r != nullptr, SPDZ_ERR_INVALID_ARGUMENT, "null run");
        need(!r->in_flight, SPDZ_ERR_INVALID_ARGUMENT, "online phase in flight");
        load_store(r, party, path);
    });
}

int spdz_run_deal(spdz_run* r, uint64_t seed) {
    return guard([&] {
        need(r != nullptr, SPDZ_ERR_INVALID_ARGUMENT, "null run");
        deal(r, seed);
    });
}

int spdz_run_bind_input(spdz_run* r, uint32_t node, const uint32_t* host_vals, uint64_t len) {
    return guard([&] {
        need(r && node < r->nodes.size(), SPDZ_ERR_INVALID_ARGUMENT, "bad input node");
        const auto& n = r->node(node);
        need(n.kind == SPDZ_NODE_INPUT, SPDZ_ERR_INVALID_ARGUMENT, "node is not an input");
        need(len == n.lanes, SPDZ_ERR_INVALID_ARGUMENT,
             "ShapeMismatch: input has " + std::to_string(len) + " elements, circuit expects " +
                 std::to_string(n.lanes));
        if (!n.is_private) {
            r->inputs[node] = std::vector<uint32_t>(host_vals, host_vals + len);
            return;
        }
        // party 0 owns every private input (preproc.cpp:146-150): stage on its device; other
        // parties' copies of the values are not used (they receive x - r)
        if (!r->parties[0].local) return;
        auto it = r->input_dev.find(node);
        uint32_t* d = it == r->input_dev.end() ? (r->input_dev[node] = r->alloc(0, len)) : it->second;
        dev(r, 0);
        auto& P0 = r->parties[0];
        // pageable sources (plain numpy / std::vector) go through the pinned staging ring at
        // multi-threaded memcpy speed (hostcopy.cu); pinned ones are DMA'd directly
        const bool staged = len * 4 >= (1u << 20) && is_pageable(host_vals);
        cudaStream_t hs = r->h2d_stream ? r->h2d_stream : P0.ctx->stream;
        if (staged) lk(staged_h2d(r->devices[0], d, host_vals, len * 4, hs), "staged H2D input");
        else lk(cudaMemcpyAsync(d, host_vals, len * 4, cudaMemcpyHostToDevice, hs), "H2D input");
        if (r->h2d_stream) {
            lk(cudaEventRecord(r->ev_h2d, r->h2d_stream), "record h2d");
            lk(cudaStreamWaitEvent(P0.ctx->stream, r->ev_h2d, 0), "wait h2d");
        }
        // reduce mod p (preproc.cpp:149 fp::reduce): x * 1 mod p, unless input sharing does it inline
        if (!share_fused(r))
            lk(launch_public(P0.ctx->stream, 3, d, d, nullptr, false, 1u, true, 0, 0, d, d, len, P0.ctx->sms),
               "reduce input");
    });
}

int spdz_run_share_inputs(spdz_run* r) {
    return guard([&] {
        need(r != nullptr, SPDZ_ERR_INVALID_ARGUMENT, "null run");
        share_inputs(r);
    });
}

int spdz_run_online_begin(spdz_run* r, int reuse) {
    return guard([&] {
        need(r != nullptr, SPDZ_ERR_INVALID_ARGUMENT, "null run");
        need(!r->in_flight, SPDZ_ERR_INVALID_ARGUMENT, "online phase already begun (call spdz_run_mac_check)");
        if (r->consumed && !reuse)
            throw Error(SPDZ_ERR_TRIPLE_EXHAUSTED,
                        "TripleExhausted: preprocessing of this run was already consumed (deal again)");
        need(!r->any_remote || r->opts.external_mac_verify || r->opts.network, SPDZ_ERR_INVALID_ARGUMENT,
             "runs with remote parties verify the MAC check externally (external_mac_verify = 1)");
        r->launches0 = g_kernel_launches;
        r->exchanged = 0;
        ++r->seq;
        r->wall0 = std::chrono::steady_clock::now();
        for (auto& P : r->parties) {
            P.maclog.clear();
            if (!P.local) continue;
            device_guard(P.ctx);
            lk(cudaEventRecord(P.t0, P.ctx->stream), "t0");
        }
        r->kt.used = 0;
        r->kt.recs.clear();
        // fusion hand-offs never outlive a phase (a phase that threw may have left one set)
        r->premasked.assign(r->nodes.size(), 0);
        r->precomputed.assign(r->nodes.size(), 0);
        r->root_opened = false;
        if (graphable(r)) {
            cudaStream_t s = S(r, 0);
            dev(r, 0);
            if (!r->online_graph) {  // capture once: the same kernels, pointers and events every phase
                const uint64_t l0 = g_kernel_launches;
                cuda_check(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed), "begin capture");
                cudaGraph_t g = nullptr;
                r->kt_capturing = true;
                try {
                    Exec ex{r};
                    ex.run_nodes();
                    ex.open_root();
                } catch (...) {
                    r->kt_capturing = false;
                    cudaStreamEndCapture(s, &g);
                    if (g) cudaGraphDestroy(g);
                    throw;
                }
                r->kt_capturing = false;
                cuda_check(cudaStreamEndCapture(s, &g), "end capture");
                cudaError_t e = cudaGraphInstantiate(&r->online_graph, g, 0);
                cudaGraphDestroy(g);
                cuda_check(e, "cudaGraphInstantiate");
                r->graph_launches = g_kernel_launches - l0;
                r->graph_exchanged = r->exchanged;
                r->graph_maclog.clear();
                for (auto& P : r->parties) r->graph_maclog.push_back(P.maclog);
                r->graph_kt_recs = r->kt.recs;
                r->graph_kt_used = r->kt.used;
            } else {
                g_kernel_launches += r->graph_launches;
                r->exchanged = r->graph_exchanged;
                for (int p = 0; p < r->n; ++p) r->parties[p].maclog = r->graph_maclog[p];
                r->kt.recs = r->graph_kt_recs;  // the replay re-records the captured event pairs
                r->kt.used = r->graph_kt_used;
            }
            lk(cudaGraphLaunch(r->online_graph, s), "cudaGraphLaunch");
        } else {
            Exec ex{r};
            r->scalar_used = r->matrix_used = 0;
            if (r->cfg) {
                r->rt_pub.assign(r->nodes.size(), 0);
                ex.run_cfg();
            }
            else ex.run_nodes();
            ex.open_root();
        }
        for (auto& P : r->parties) {  // the phase's openings are complete once these fire
            if (!P.local) continue;
            device_guard(P.ctx);
            lk(cudaEventRecord(P.t_open, P.ctx->stream), "t_open");
        }
        r->consumed = true;
        r->in_flight = true;
        // opened outputs to host on a copy stream, overlapping the MAC check
        const int op = r->ref_party();
        const Val& rv = r->parties[op].ns[r->root].out;
        dev(r, op);
        if (!r->host_out || r->host_out_cap < rv.lanes) {
            need(r->host_out_owned || !r->host_out, SPDZ_ERR_INVALID_ARGUMENT, "bound output buffer too small");
            if (r->host_out) cudaFreeHost(r->host_out);
            cuda_check(cudaMallocHost(&r->host_out, std::max<uint64_t>(rv.lanes, 1) * 4), "cudaMallocHost(out)");
            r->host_out_cap = rv.lanes;
            r->host_out_owned = true;
        }
        r->host_out_len = rv.lanes;
        cudaStream_t out_stream = r->d2h_stream ? r->d2h_stream : r->copy_stream;
        lk(cudaEventRecord(r->ev_opened, S(r, op)), "record opened");
        lk(cudaStreamWaitEvent(out_stream, r->ev_opened, 0), "wait opened");
        lk(cudaMemcpyAsync(r->host_out, r->parties[op].outputs, rv.lanes * 4, cudaMemcpyDeviceToHost, out_stream),
           "D2H out");
        lk(cudaEventRecord(r->ev_out, out_stream), "record out");
    });
}

int spdz_run_span_ms(spdz_run* a, spdz_run* b, float* ms) {
    return guard([&] {
        need(a && b && ms, SPDZ_ERR_INVALID_ARGUMENT, "bad span args");
        const int pa = a->ref_party();
        dev(a, pa);
        float best = -1.0f;
        for (int p = 0; p < b->n; ++p) {
            if (!b->parties[p].local) continue;
            float t = 0;
            cuda_check(cudaEventSynchronize(b->parties[p].t1), "sync t1");
            cuda_check(cudaEventElapsedTime(&t, a->parties[pa].t0, b->parties[p].t1), "elapsed");
            best = std::max(best, t);
        }
        *ms = best;
    });
}

void* spdz_run_party_stream(spdz_run* r, int party) {
    if (!r || party < 0 || party >= r->n || !r->parties[party].local) return nullptr;
    return r->parties[party].ctx->stream;
}

int spdz_run_set_copy_streams(spdz_run* r, void* h2d_stream, void* d2h_stream) {
    return guard([&] {
        need(r != nullptr, SPDZ_ERR_INVALID_ARGUMENT, "null run");
        need(!r->in_flight, SPDZ_ERR_INVALID_ARGUMENT, "online phase in flight");
        r->h2d_stream = static_cast<cudaStream_t>(h2d_stream);
        r->d2h_stream = static_cast<cudaStream_t>(d2h_stream);
    });
}

int spdz_run_wait_openings(spdz_run* r) {
    return guard([&] {
        need(r != nullptr && r->in_flight, SPDZ_ERR_INVALID_ARGUMENT, "no online phase in flight");
        for (auto& P : r->parties) {
            if (!P.local) continue;
            device_guard(P.ctx);
            lk(cudaEventSynchronize(P.t_open), "wait openings");
        }
    });
}

int spdz_run_mac_check_launch(spdz_run* r, int use_coin, uint64_t coin) {
    return guard([&] {
        need(r != nullptr && r->in_flight && !r->mac_launched, SPDZ_ERR_INVALID_ARGUMENT,
             "no online phase in flight (or its MAC check was already launched)");
        need(!r->net, SPDZ_ERR_INVALID_ARGUMENT,
             "network runs agree on the coin with their peers: use spdz_run_mac_check");
        r->mac_coin = agree_coin(r, use_coin != 0, coin);
        mac_launch(r, r->mac_coin);
        r->mac_launched = true;
    });
}

int spdz_run_mac_check(spdz_run* r, int use_coin, uint64_t coin, spdz_run_report_t* rep) {
    return guard([&] {
        need(r != nullptr && r->in_flight, SPDZ_ERR_INVALID_ARGUMENT, "no online phase in flight");
        r->in_flight = false;
        if (r->mac_launched) {  // sigma kernels already in flight (spdz_run_mac_check_launch)
            r->mac_launched = false;
            mac_finish(r, rep, r->mac_coin);
        } else {
            mac_check(r, rep, use_coin != 0, coin);  // records t1 and synchronises the party streams
        }
        dev(r, r->ref_party());
        lk(cudaEventSynchronize(r->ev_out), "sync out");
        auto t1 = std::chrono::steady_clock::now();
        if (rep) {
            rep->online_ms = std::chrono::duration<double, std::milli>(t1 - r->wall0).count();
            double dmax = 0;
            for (auto& P : r->parties) {
                if (!P.local) continue;
                device_guard(P.ctx);
                float ms = 0;
                lk(cudaEventElapsedTime(&ms, P.t0, P.t1), "elapsed");
                dmax = std::max(dmax, (double)ms);
            }
            rep->online_device_ms = dmax;
            // straight-line: every provisioned triple; control flow: what the taken path used
            // straight-line: the live nodes' regions (one execution each); control flow: what the
            // taken path used
            rep->scalar_triples_consumed = r->cfg ? r->scalar_used : r->scalar_live;
            rep->matrix_triples_consumed = r->cfg ? r->matrix_used : r->matrix_live;
            rep->bytes_exchanged = r->exchanged;
            rep->output_digest = 0;  // spdz_run_output_digest (host byte loop, outside the online phase)
            rep->kernel_launches = g_kernel_launches - r->launches0;
            for (int c = 0; c < SPDZ_KSTAT_N; ++c) rep->kstat[c] = spdz_kernel_stat_t{0, 0.0, 0};
            for (auto& rec : r->kt.recs) {
                if (rec.cls < 0 || !rec.b) continue;
                cuda_check(cudaSetDevice(rec.dev), "dev");
                float ms = 0;
                lk(cudaEventSynchronize(rec.b), "sync ev");
                lk(cudaEventElapsedTime(&ms, rec.a, rec.b), "elapsed");
                rep->kstat[rec.cls].launches += 1;
                rep->kstat[rec.cls].ms += ms;
                rep->kstat[rec.cls].bytes += rec.bytes;
            }
        }
    });
}

int spdz_run_online(spdz_run* r, int reuse, spdz_run_report_t* rep) {
    int rc = spdz_run_online_begin(r, reuse);
    if (rc) return rc;
    return spdz_run_mac_check(r, 0, 0, rep);
}

int spdz_run_outputs(spdz_run* r, uint32_t* host_out, uint64_t cap, uint64_t* len) {
    return guard([&] {
        need(r != nullptr, SPDZ_ERR_INVALID_ARGUMENT, "null run");
        if (len) *len = r->host_out_len;
        if (host_out && host_out != r->host_out)
            parallel_copy(host_out, r->host_out, std::min<uint64_t>(cap, r->host_out_len) * 4);
    });
}

int spdz_run_output_digest(spdz_run* r, uint64_t* digest) {
    return guard([&] {  // runtime.cpp:573-574 (computed after the online phase, as the reference does)
        need(r != nullptr && digest != nullptr, SPDZ_ERR_INVALID_ARGUMENT, "bad digest args");
        *digest = spdz_fnv1a64(r->host_out, r->host_out_len * 4, 1469598103934665603ull);
    });
}

int spdz_run_bind_output(spdz_run* r, uint32_t* host_out, uint64_t cap) {
    return guard([&] {
        need(r != nullptr && host_out != nullptr, SPDZ_ERR_INVALID_ARGUMENT, "bad bind_output");
        if (r->host_out && r->host_out_owned) cudaFreeHost(r->host_out);
        if (r->host_out_registered) cudaHostUnregister(r->host_out);
        r->host_out_registered = false;
        // a pageable buffer would turn the output D2H into a host-blocking copy (the whole
        // online phase would wait for it): page-lock it for as long as it is bound
        cudaPointerAttributes at{};
        if (cudaPointerGetAttributes(&at, host_out) == cudaSuccess && at.type == cudaMemoryTypeUnregistered) {
            cuda_check(cudaHostRegister(host_out, std::max<uint64_t>(cap, 1) * 4, cudaHostRegisterDefault),
                       "cudaHostRegister(output)");
            r->host_out_registered = true;
        }
        cudaGetLastError();  // clear the query's error state for unregistered pointers
        r->host_out = host_out;
        r->host_out_cap = cap;
        r->host_out_owned = false;
    });
}

int spdz_run_node_share(spdz_run* r, int party, uint32_t node, spdz_share_t* out) {
    return guard([&] {
        need(r && party >= 0 && party < r->n && node < r->nodes.size() && out, SPDZ_ERR_INVALID_ARGUMENT,
             "bad node_share args");
        const Val& v = r->parties[party].ns[node].out;
        out->vals = v.is_public ? v.pub : v.v;
        out->macs = v.is_public ? nullptr : v.m;
        out->lanes = v.lanes;
    });
}


int spdz_run_export(spdz_run* r, void* buf, uint64_t cap, uint64_t* len) {
    return guard([&] {
        need(r != nullptr && len != nullptr, SPDZ_ERR_INVALID_ARGUMENT, "bad export args");
        load_stream_memops();
        std::vector<uint8_t> out;
        for (int p = 0; p < r->n; ++p) {
            if (!r->parties[p].local) continue;
            dev(r, p);
            std::vector<IpcEntry> es;
            for_each_export(r, p, [&](uint32_t kind, uint32_t node, uint32_t sub, void* ptr) {
                IpcEntry e{};
                e.kind = kind;
                e.node = node;
                e.sub = sub;
                CUdeviceptr base = 0;
                size_t size = 0;
                need(g_addrrange(&base, &size, (CUdeviceptr)ptr) == CUDA_SUCCESS, SPDZ_ERR_CUDA, "cuMemGetAddressRange");
                e.offset = (uint64_t)((CUdeviceptr)ptr - base);
                cuda_check(cudaIpcGetMemHandle(&e.handle, (void*)base), "cudaIpcGetMemHandle");
                es.push_back(e);
            });
            IpcHeader h{kIpcMagic, 1u, (uint32_t)p, (uint32_t)es.size()};
            const uint8_t* hb = reinterpret_cast<const uint8_t*>(&h);
            out.insert(out.end(), hb, hb + sizeof h);
            const uint8_t* eb = reinterpret_cast<const uint8_t*>(es.data());
            out.insert(out.end(), eb, eb + es.size() * sizeof(IpcEntry));
        }
        *len = out.size();
        if (buf) {
            need(cap >= out.size(), SPDZ_ERR_INVALID_ARGUMENT, "export buffer too small");
            std::memcpy(buf, out.data(), out.size());
        }
    });
}

int spdz_run_import(spdz_run* r, const void* blob, uint64_t len) {
    return guard([&] {
        need(r != nullptr && blob != nullptr, SPDZ_ERR_INVALID_ARGUMENT, "bad import args");
        const uint8_t* b = static_cast<const uint8_t*>(blob);
        uint64_t at = 0;
        const int lp = r->ref_party();
        dev(r, lp);
        while (at + sizeof(IpcHeader) <= len) {
            IpcHeader h;
            std::memcpy(&h, b + at, sizeof h);
            at += sizeof h;
            need(h.magic == kIpcMagic && h.version == 1, SPDZ_ERR_MALFORMED_SHARE_MESSAGE,
                 "MalformedShareMessage: not a spdz_run export");
            need(h.party < (uint32_t)r->n, SPDZ_ERR_MALFORMED_SHARE_MESSAGE, "MalformedShareMessage: party");
            need(at + (uint64_t)h.n * sizeof(IpcEntry) <= len, SPDZ_ERR_MALFORMED_SHARE_MESSAGE,
                 "MalformedShareMessage: truncated export");
            auto& Q = r->parties[h.party];
            const bool skip = Q.local;  // our own export (all-gathered blobs)
            for (uint32_t i = 0; i < h.n; ++i, at += sizeof(IpcEntry)) {
                if (skip) continue;
                IpcEntry e;
                std::memcpy(&e, b + at, sizeof e);
                void* base = nullptr;
                cuda_check(cudaIpcOpenMemHandle(&base, e.handle, cudaIpcMemLazyEnablePeerAccess),
                           "cudaIpcOpenMemHandle");
                Q.mapped.push_back(base);
                uint32_t* ptr = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(base) + e.offset);
                need(e.node < r->nodes.size(), SPDZ_ERR_MALFORMED_SHARE_MESSAGE, "MalformedShareMessage: node");
                auto& st = Q.ns[e.node];
                switch (e.kind) {
                    case 0: Q.flags = ptr; break;
                    case 1: st.payload = ptr; break;
                    case 2:
                        need(e.sub < st.levels.size(), SPDZ_ERR_MALFORMED_SHARE_MESSAGE, "MalformedShareMessage");
                        st.levels[e.sub].payload = ptr;
                        break;
                    case 3: st.out.v = ptr; break;
                    case 4:
                        need(h.party == 0, SPDZ_ERR_MALFORMED_SHARE_MESSAGE, "MalformedShareMessage: diff");
                        r->input_diff[e.node] = ptr;
                        break;
                    default: throw Error(SPDZ_ERR_MALFORMED_SHARE_MESSAGE, "MalformedShareMessage: entry kind");
                }
            }
        }
    });
}

int spdz_run_attach_net(spdz_run* r, spdz_net* net) {
    return guard([&] {
        need(r != nullptr && net != nullptr, SPDZ_ERR_INVALID_ARGUMENT, "null run or mesh");
        need(r->opts.network && r->opts.single_party > 0, SPDZ_ERR_INVALID_ARGUMENT,
             "attach a mesh to a single_party run created with network = 1");
        NetLink* link = net_link(net);
        need(link->n == r->n && link->party == r->opts.single_party - 1, SPDZ_ERR_INVALID_ARGUMENT,
             "mesh is party " + std::to_string(link->party) + " of " + std::to_string(link->n) + ", run is party " +
                 std::to_string(r->opts.single_party - 1) + " of " + std::to_string(r->n));
        r->net = link;
    });
}

int spdz_run_inject_bitflip(spdz_run* r, uint32_t node, int sender, int receiver, uint64_t word, uint32_t bit) {
    return guard([&] {
        need(r && node < r->nodes.size(), SPDZ_ERR_INVALID_ARGUMENT, "bad node");
        need(sender >= 0 && sender < r->n && receiver >= 0 && receiver < r->n && sender != receiver,
             SPDZ_ERR_INVALID_ARGUMENT, "bad sender/receiver");
        auto& st = r->parties[receiver].ns[node];
        const bool root = node == r->root && !st.out.is_public;  // the root open (runtime.cpp:555-558)
        need(st.payload != nullptr || root, SPDZ_ERR_INVALID_ARGUMENT, "node has no opening to tamper with");
        if (!st.shadow) {
            const auto& n = r->node(node);
            uint64_t words = root ? st.out.lanes : 2ull * n.lanes;
            if (n.kind == SPDZ_NODE_LINEAR)
                words = (uint64_t)n.din * n.dout + (uint64_t)n.din * r->tiles[node].starts.size();
            st.shadow = r->alloc(receiver, words);
        }
        r->faults.push_back({node, sender, receiver, word, bit});
        if (r->online_graph) {  // the captured phase has no tampering step
            cudaGraphExecDestroy(r->online_graph);
            r->online_graph = nullptr;
        }
    });
}

}  // extern "C"
