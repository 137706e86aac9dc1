// Planning of a run (node buffers, the triple layout of preproc.cpp:124-163) and its
// preprocessing: the GPU dealer in make_dealer_stores order, or the reference's MPCT
// store files streamed into the same device pools.
#include <deque>
#include <functional>

#include "run_state.hpp"

namespace spdzb200 {
namespace rt {

// Which nodes run.  The reference's scheduler stops when the root completes (scheduler.cpp:154,
// runtime.cpp:452-465), so whether it issues a dead node (value reaching no output) depends on
// its issue order: usually it does (heavy nodes first, while the root waits for an opening),
// sometimes not (the dead node's inputs become ready after a root computed locally).  Local
// straight-line runs execute exactly the nodes its single-worker order issues (so triple counts
// match); control-flow runs execute every node of an entered block; a run across a mesh skips
// dead nodes, so it never waits for a frame reference parties may not send (a dead open the
// reference does issue just goes unanswered).  Outputs are the same either way; the triple
// layout reserves every region.
// The nodes the reference's single-worker scheduler issues before the root completes
// (scheduler.cpp:65-97, 138-169; runtime.cpp:360-465): heavy queue first, FIFO; a private x
// private multiply completes in its open continuation, which runs when the worker has nothing
// else to issue (pump) or when a blocking reduce_mul / linear layer pumps; the loop ends when
// the root completes.  Checked against the reference's triple counts on every fuzzed program.
static void scheduler_issued(spdz_run* r, std::vector<char>& issued) {
    const uint32_t N = (uint32_t)r->nodes.size();
    auto kind = [&](uint32_t i) { return r->nodes[i].kind; };
    auto queueable = [&](uint32_t i) {
        const int k = kind(i);
        return k != SPDZ_NODE_INPUT && k != SPDZ_NODE_CONST && k != SPDZ_NODE_NOP && k != SPDZ_NODE_LABEL &&
               k != SPDZ_NODE_PHI;
    };
    auto heavy = [&](uint32_t i) {
        const int k = kind(i);
        return k == SPDZ_NODE_MUL || k == SPDZ_NODE_REDUCE_MUL || k == SPDZ_NODE_LINEAR;
    };
    auto both_private = [&](uint32_t i) {
        const auto& n = r->nodes[i];
        return n.n_operands >= 2 && r->priv(n.operands[0]) && r->priv(n.operands[1]);
    };
    std::vector<uint32_t> remaining(N, 0);
    std::vector<std::vector<uint32_t>> consumers(N);
    for (uint32_t i = 0; i < N; ++i)
        if (queueable(i)) {
            remaining[i] = r->nodes[i].n_operands;
            for (uint32_t k = 0; k < r->nodes[i].n_operands; ++k) consumers[r->nodes[i].operands[k]].push_back(i);
        }
    std::deque<uint32_t> hq, lq;
    std::vector<uint32_t> outstanding;
    bool finished = false, started = false;
    std::function<void(uint32_t)> complete = [&](uint32_t i) {
        if (i == r->root) finished = true;
        for (uint32_t c : consumers[i])
            if (--remaining[c] == 0 && started) (heavy(c) ? hq : lq).push_back(c);
    };
    for (uint32_t i = 0; i < N; ++i)
        if (kind(i) == SPDZ_NODE_INPUT || kind(i) == SPDZ_NODE_CONST) complete(i);
    started = true;
    for (uint32_t i = 0; i < N; ++i)  // entry block: ready nodes in program order
        if (queueable(i) && remaining[i] == 0) (heavy(i) ? hq : lq).push_back(i);
    auto pump = [&] {
        std::vector<uint32_t> done;
        done.swap(outstanding);
        for (uint32_t i : done) complete(i);
    };
    issued.assign(N, 0);
    while (!finished) {
        uint32_t i;
        if (!hq.empty()) {
            i = hq.front();
            hq.pop_front();
        } else if (!lq.empty()) {
            i = lq.front();
            lq.pop_front();
        } else if (!outstanding.empty()) {
            pump();
            continue;
        } else {
            break;
        }
        issued[i] = 1;
        const int k = kind(i);
        if (k == SPDZ_NODE_MUL && both_private(i)) {
            outstanding.push_back(i);
        } else if ((k == SPDZ_NODE_REDUCE_MUL && r->priv(r->nodes[i].operands[0])) ||
                   (k == SPDZ_NODE_LINEAR && both_private(i))) {
            pump();  // blocking opens pump the session (runtime.cpp:269, linear.cpp:123-127)
            complete(i);
        } else {
            complete(i);
        }
    }
    for (uint32_t i = 0; i < N; ++i)  // inputs, constants and the root's own chain stay usable
        if (!queueable(i)) issued[i] = 1;
}

void compute_liveness(spdz_run* r) {
    const uint32_t N = (uint32_t)r->nodes.size();
    if (!r->opts.network) {
        if (r->cfg) {  // control flow: every node of an entered block runs
            r->live.assign(N, 1);
        } else {
            scheduler_issued(r, r->live);
        }
        r->scalar_live = r->matrix_live = 0;
        for (auto& [id, reg] : r->scalar)
            if (r->live[id]) r->scalar_live += reg.stride;
        for (auto& [id, reg] : r->matrix)
            if (r->live[id]) r->matrix_live += reg.stride;
        return;
    }
    r->live.assign(N, 0);
    std::vector<uint32_t> work{r->root};
    for (uint32_t id = 0; id < N; ++id)
        if (r->nodes[id].kind == SPDZ_NODE_BRANCH) work.push_back(id);
    while (!work.empty()) {
        const uint32_t id = work.back();
        work.pop_back();
        if (id >= N || r->live[id]) continue;
        r->live[id] = 1;
        const auto& n = r->nodes[id];
        for (uint32_t k = 0; k < n.n_operands; ++k) work.push_back(n.operands[k]);
    }
    r->scalar_live = r->matrix_live = 0;
    for (auto& [id, reg] : r->scalar)
        if (r->live[id]) r->scalar_live += reg.stride;
    for (auto& [id, reg] : r->matrix)
        if (r->live[id]) r->matrix_live += reg.stride;
}

// ---- planning (run creation) ----
void plan_layout(spdz_run* r) {
    // preproc.cpp:84-163 for straight-line graphs (no loops: mult = 1).  With lane
    // sharding every vector node holds shard_L of shard_total global lanes; regions
    // are laid out globally and this run keeps its slice (local compact pools).
    const bool sh = r->shard_total != 0;
    const uint64_t G = r->shard_total, off = r->shard_off;
    for (auto& n : r->nodes) {
        const uint32_t id = (uint32_t)(&n - r->nodes.data());
        if (sh && n.lanes != 1 && n.lanes != r->shard_L && n.kind != SPDZ_NODE_NOP && n.kind != SPDZ_NODE_LABEL)
            throw Error(SPDZ_ERR_INVALID_ARGUMENT, "sharded run: every vector node must have the shard's lanes");
        // executions provisioned: loop_iters per enclosing loop (preproc.cpp:127-130)
        uint64_t mult = 1;
        for (uint32_t d = 0; d < n.loop_depth; ++d) {
            need(mult <= (1ull << 40) / std::max<uint64_t>(r->loop_iters, 1), SPDZ_ERR_INVALID_ARGUMENT,
                 "loop provisioning overflows");
            mult *= r->loop_iters;
        }
        switch (n.kind) {
            case SPDZ_NODE_MUL:
                if (r->priv(n.operands[0]) && r->priv(n.operands[1])) {
                    Region g{r->scalar_total, n.lanes, mult, sh ? r->scalar_total_global + off : r->scalar_total};
                    r->scalar[id] = g;
                    r->scalar_total += n.lanes * mult;
                    r->scalar_total_global += (sh ? G : n.lanes) * mult;
                }
                break;
            case SPDZ_NODE_REDUCE_MUL: {
                const auto& src = r->node(n.operands[0]);
                if (sh) throw Error(SPDZ_ERR_INVALID_ARGUMENT, "sharded run: reduce_mul is not lane-parallel");
                if (src.is_private && src.lanes >= 1) {
                    r->scalar[id] = {r->scalar_total, src.lanes - 1ull, mult, r->scalar_total};
                    r->scalar_total += (src.lanes - 1ull) * mult;
                    r->scalar_total_global += (src.lanes - 1ull) * mult;
                }
                break;
            }
            case SPDZ_NODE_REDUCE_ADD:
                if (sh) throw Error(SPDZ_ERR_INVALID_ARGUMENT, "sharded run: reduce_add is not lane-parallel");
                break;
            case SPDZ_NODE_LINEAR:
                if (sh) throw Error(SPDZ_ERR_INVALID_ARGUMENT, "sharded run: linear layers are row-sharded separately");
                if (r->priv(n.operands[0]) && r->priv(n.operands[1])) {
                    uint64_t nt = 0;
                    LinTiles lt;
                    lt.starts.resize(n.dout);
                    lt.counts.resize(n.dout);
                    int rc = spdz_plan_tiles(n.din, n.dout, r->opts.slice, lt.starts.data(), lt.counts.data(), n.dout,
                                             &nt);
                    if (rc) throw Error(rc, spdz_last_error());
                    lt.starts.resize(nt);
                    lt.counts.resize(nt);
                    lt.rpt = lt.counts[0];
                    r->matrix[id] = {r->matrix_total, nt, mult};
                    r->matrix_total += nt * mult;
                    for (uint64_t k = 0; k < mult; ++k)  // preproc.cpp:104-112: per execution, per tile
                        for (auto c : lt.counts) r->mshapes.emplace_back(n.din, c);
                    r->tiles[id] = lt;
                }
                break;
            default:
                break;
        }
    }
    for (uint32_t id = 0; id < r->nodes.size(); ++id) {  // preproc.cpp:119-121, g.inputs order
        const auto& n = r->nodes[id];
        if (n.kind == SPDZ_NODE_INPUT && n.is_private) {
            r->input_mask_off[id] = r->mask_total;
            r->input_mask_gfirst[id] = sh ? r->mask_total_global + off : r->mask_total;
            r->mask_total += n.lanes;
            r->mask_total_global += sh ? G : n.lanes;
        }
    }
}

uint32_t const_of(spdz_run* r, uint32_t id) {
    const auto& n = r->node(id);
    need(n.kind == SPDZ_NODE_CONST, SPDZ_ERR_INVALID_ARGUMENT, "load start must be a constant node");
    return n.const_val;
}

// Allocates every device buffer of the online phase, per party.
void plan_buffers(spdz_run* r) {
    const uint32_t N = (uint32_t)r->nodes.size();
    for (int p = 0; p < r->n; ++p) {
        auto& P = r->parties[p];
        P.ns.resize(N);
        for (uint32_t id = 0; id < N; ++id) {
            const auto& n = r->nodes[id];
            auto& st = P.ns[id];
            const uint64_t L = n.lanes;
            auto priv_out = [&](uint64_t lanes) {
                st.out.is_public = false;
                st.out.lanes = lanes;
                st.out.v = r->alloc(p, lanes);
                st.out.m = r->alloc(p, lanes);
            };
            auto pub_out = [&](uint64_t lanes) {
                st.out.is_public = true;
                st.out.lanes = lanes;
                st.out.pub = r->alloc(p, lanes);
            };
            auto opnd = [&](int k) -> const Val& { return P.ns[n.operands[k]].out; };
            switch (n.kind) {
                case SPDZ_NODE_INPUT:
                    if (n.is_private) priv_out(L);
                    else pub_out(L);
                    break;
                case SPDZ_NODE_CONST:
                    pub_out(1);
                    break;
                case SPDZ_NODE_CMP_PUBLIC:  // runtime.cpp:119-125 read_public: completed public scalars only
                    for (int k = 0; k < 2; ++k)
                        need(n.n_operands == 2 && opnd(k).is_public && opnd(k).lanes >= 1, SPDZ_ERR_INVALID_ARGUMENT,
                             "runtime: node " + std::to_string(n.operands[k]) + " is not a completed public scalar");
                    need(n.const_val <= 5, SPDZ_ERR_INVALID_ARGUMENT, "runtime: bad comparison predicate");
                    pub_out(1);
                    break;
                case SPDZ_NODE_NOP:
                case SPDZ_NODE_LABEL:
                case SPDZ_NODE_BRANCH:
                    break;
                case SPDZ_NODE_PHI:  // its own buffer: the chosen value is copied in at block entry
                    if (n.is_private) {
                        priv_out(L);
                        st.shadow_pub = r->alloc(p, L);
                    } else {
                        pub_out(L);
                    }
                    break;
                case SPDZ_NODE_LOAD: {  // runtime.cpp:419-438 (zero-copy slice)
                    const Val& base = opnd(0);
                    if (r->node(n.operands[1]).kind != SPDZ_NODE_CONST) {  // start known at run time: copied
                        st.dyn_load = true;
                        if (base.is_public) pub_out(L);
                        else priv_out(L);
                        break;
                    }
                    const uint32_t start = const_of(r, n.operands[1]);
                    need((uint64_t)start + L <= base.lanes, SPDZ_ERR_INVALID_ARGUMENT, "runtime: load out of bounds");
                    st.out = base;
                    st.out.lanes = L;
                    if (base.is_public) st.out.pub = base.pub + start;
                    else {
                        st.out.v = base.v + start;
                        st.out.m = base.m + start;
                    }
                    break;
                }
                case SPDZ_NODE_ADD:
                case SPDZ_NODE_SUB:
                    if (opnd(0).is_public && opnd(1).is_public) pub_out(L);
                    else priv_out(L);
                    break;
                case SPDZ_NODE_MUL: {
                    const Val &a = opnd(0), &b = opnd(1);
                    if (a.is_public && b.is_public) {
                        pub_out(L);
                    } else if (!a.is_public && !b.is_public) {
                        priv_out(L);
                        st.xa = a;
                        st.xb = b;
                        if (a.lanes != L) st.xa = Val{false, nullptr, r->alloc(p, L), r->alloc(p, L), L};
                        if (b.lanes != L) st.xb = Val{false, nullptr, r->alloc(p, L), r->alloc(p, L), L};
                        st.payload = r->alloc(p, 2 * L);
                        st.opened = r->alloc(p, 2 * L);
                        if (r->cfg) {  // one MAC-log slot per provisioned execution
                            const uint64_t execs = r->scalar.at(id).max_execs;
                            st.opened_all = r->alloc(p, 2 * L * execs);
                            st.macsnap = r->alloc(p, 2 * L * execs);
                        }

                    } else {
                        priv_out(L);
                    }
                    break;
                }
                case SPDZ_NODE_REDUCE_ADD:
                    if (opnd(0).is_public) pub_out(1);
                    else priv_out(1);
                    break;
                case SPDZ_NODE_REDUCE_MUL: {
                    const Val& a = opnd(0);
                    if (a.is_public) {
                        pub_out(1);
                        st.opened = r->alloc(p, std::max<uint64_t>(a.lanes, 1));  // scratch tree
                        break;
                    }
                    uint64_t cur = a.lanes;
                    while (cur > 1) {
                        RedLevel lv;
                        lv.in_lanes = cur;
                        lv.pairs = cur / 2;
                        lv.xv = r->alloc(p, lv.pairs);
                        lv.xm = r->alloc(p, lv.pairs);
                        lv.yv = r->alloc(p, lv.pairs);
                        lv.ym = r->alloc(p, lv.pairs);
                        lv.payload = r->alloc(p, 2 * lv.pairs);
                        lv.opened = r->alloc(p, 2 * lv.pairs);
                        if (r->cfg) {  // every execution keeps its MAC-log records
                            const uint64_t E = r->scalar.count(id) ? r->scalar.at(id).max_execs : 1;
                            lv.xm_all = r->alloc(p, lv.pairs * E);
                            lv.ym_all = r->alloc(p, lv.pairs * E);
                            lv.opened_all = r->alloc(p, 2 * lv.pairs * E);
                        }
                        lv.out_lanes = lv.pairs + (cur & 1);
                        lv.zv = r->alloc(p, lv.out_lanes);
                        lv.zm = r->alloc(p, lv.out_lanes);
                        st.levels.push_back(lv);
                        cur = lv.out_lanes;
                    }
                    if (st.levels.empty()) {
                        priv_out(1);
                    } else {
                        st.out = Val{false, nullptr, st.levels.back().zv, st.levels.back().zm, 1};
                    }
                    break;
                }
                case SPDZ_NODE_LINEAR: {
                    const Val &x = opnd(0), &w = opnd(1);
                    need(x.lanes == n.din && w.lanes == (uint64_t)n.din * n.dout, SPDZ_ERR_INVALID_ARGUMENT,
                         "ShapeMismatch: linear operands do not match din/dout");
                    if (x.is_public && w.is_public) {
                        // any private operand makes the node private (graph_builder.cpp:123):
                        // a private bias gives add_public(b, W x) (runtime.cpp:129-162)
                        if (n.n_operands > 2 && !opnd(2).is_public) priv_out(n.dout);
                        else pub_out(n.dout);
                        st.lin_tmp = r->alloc(p, 2ull * n.dout);  // W x (the GEMM writes two planes)
                    } else if (x.is_public != w.is_public) {
                        priv_out(n.dout);
                        st.lin_tmp = r->alloc(p, 2ull * n.dout);
                    } else {
                        priv_out(n.dout);
                        const auto& lt = r->tiles[id];
                        const uint64_t cells = (uint64_t)n.din * n.dout, etot = (uint64_t)n.din * lt.starts.size();
                        st.payload = r->alloc(p, cells + etot);
                        st.opened = r->alloc(p, cells + etot);
                        if (r->cfg) {  // every execution: opened [D|E] and the W.m / x.m it is checked against
                            const uint64_t E = r->matrix.at(id).max_execs;
                            st.opened_all = r->alloc(p, (cells + etot) * E);
                            st.macsnap = r->alloc(p, (cells + n.din) * E);
                        }
                        st.bias_v = r->alloc(p, n.dout);
                        st.bias_m = r->alloc(p, n.dout);
                        st.lin_tmp = r->alloc(p, 2ull * n.dout);
                        if (r->n == 2 && p == 0 && r->parties[0].local && r->parties[1].local) {
                            st.mc2_scratch = r->alloc(p, 11ull * n.dout);  // 5 x u64 + u32 per row
                            cuda_check(cudaMemset(st.mc2_scratch, 0, 44ull * n.dout), "memset(mc2 scratch)");
                        }
                    }
                    break;
                }
                case SPDZ_NODE_ROOT:
                    st.out = opnd(0);
                    break;
                default:
                    throw Error(SPDZ_ERR_INVALID_ARGUMENT, "runtime: unexpected node kind " + std::to_string(n.kind));
            }
            // control flow: private-typed add/sub/mul/phi/reductions may hold a public value at run
            // time; a load's public value is a view of its base's (a copy for a run-time start)
            if (r->cfg && !st.out.is_public && !st.shadow_pub) {
                if (n.kind == SPDZ_NODE_ADD || n.kind == SPDZ_NODE_SUB || n.kind == SPDZ_NODE_MUL ||
                    n.kind == SPDZ_NODE_PHI || n.kind == SPDZ_NODE_REDUCE_ADD)
                    st.shadow_pub = r->alloc(p, L);
                else if (n.kind == SPDZ_NODE_REDUCE_MUL)  // product-tree scratch over the operand's lanes
                    st.shadow_pub = r->alloc(p, std::max<uint64_t>(opnd(0).lanes, 1));
                else if (n.kind == SPDZ_NODE_LOAD && P.ns[n.operands[0]].shadow_pub)
                    st.shadow_pub = st.dyn_load ? r->alloc(p, L)
                                                : P.ns[n.operands[0]].shadow_pub + const_of(r, n.operands[1]);
            }
        }
        const Val& rv = P.ns[r->root].out;
        P.outputs = r->alloc(p, std::max<uint64_t>(rv.lanes, 1));
        if (!P.local) continue;
        cuda_check(cudaSetDevice(P.ctx->device), "dev");
        cuda_check(cudaEventCreate(&P.t0), "ev");
        cuda_check(cudaEventCreateWithFlags(&P.t_open, cudaEventDisableTiming), "ev");
        cuda_check(cudaEventCreate(&P.t1), "ev");
        // private input differences: party 0 publishes x - mask (preproc.cpp:146-151)
        if (p == 0)
            for (auto& [id, off] : r->input_mask_off) r->input_diff[id] = r->alloc(0, r->node(id).lanes);
        // opening-slot flags (only read by remote peers)
        r->n_slots = (uint64_t)r->nodes.size() * 64;
        P.flags = r->alloc(p, r->n_slots);
        cuda_check(cudaMemset(P.flags, 0, r->n_slots * 4), "memset flags");
    }
    // network peers: party 0's input differences arrive as frames into a local mirror
    if (r->opts.network && !r->parties[0].local)
        for (auto& [id, off] : r->input_mask_off) r->input_diff[id] = r->alloc(0, r->node(id).lanes);
    // one open event per (party, node) plus reduce levels
    for (int p = 0; p < r->n; ++p) {
        if (!r->parties[p].local) continue;
        size_t need_ev = r->nodes.size() + 1;
        for (auto& st : r->parties[p].ns) need_ev += st.levels.size();
        for (size_t k = 0; k < need_ev; ++k) new_event(r, p);
    }
    dev(r, r->ref_party());
    cuda_check(cudaEventCreateWithFlags(&r->ev_input, cudaEventDisableTiming), "event");
    cuda_check(cudaEventCreateWithFlags(&r->ev_opened, cudaEventDisableTiming), "event");
    cuda_check(cudaEventCreateWithFlags(&r->ev_h2d, cudaEventDisableTiming), "event");
    cuda_check(cudaEventCreateWithFlags(&r->ev_out, cudaEventDisableTiming), "event");
    cuda_check(cudaStreamCreateWithFlags(&r->copy_stream, cudaStreamNonBlocking), "copy stream");
}

// ---- preprocessing: GPU dealer in make_dealer_stores order (triple_store.cpp:248-287) ----
void deal(spdz_run* r, uint64_t seed) {
    const int n = r->n;
    uint32_t alpha_sh[SPDZ_MAX_PARTIES], alpha;
    dealer_alpha(n, seed, alpha_sh, &alpha);
    for (int p = 0; p < n; ++p)
        if (r->parties[p].local) set_alpha(r->parties[p].ctx, alpha_sh[p]);
    const uint64_t S = r->scalar_total, M = r->mask_total;
    for (auto& [device, dd] : r->deals) {
        int p0 = -1;
        for (int p = 0; p < n; ++p)
            if (r->parties[p].local && r->devices[p] == device) { p0 = p; break; }
        spdz_ctx* ctx = r->parties[p0].ctx;
        device_guard(ctx);
        cuda_check(cudaMemsetAsync(ctx->d_flag, 0, 4, ctx->stream), "memset flag");
        uint64_t k = n;  // Dealer ctor consumed n draws (spdz.cpp:162-173)
        // Dealer::triples(S_global); this run keeps each region's slice (compact local pool)
        for (auto& [id, reg] : r->scalar) {
            const uint64_t cnt = reg.stride * reg.max_execs;
            uint32_t* planes[6];
            for (int q = 0; q < 6; ++q) planes[q] = dd.pool[q] + reg.base;
            lk(launch_dealer_triples(ctx->stream, n, seed, k, alpha, r->scalar_total_global, reg.gbase, cnt, S, planes,
                                     ctx->d_flag, ctx->sms),
               "deal triples");
        }
        k += dealer_draws_triples(n, r->scalar_total_global);
        // matrix triples in demand order: linear nodes by id, tiles in order
        for (auto& [id, reg] : r->matrix) {
            const auto& nd = r->node(id);
            const auto& lt = r->tiles[id];
            auto& pl = dd.layer[id];
            const uint64_t cells_one = (uint64_t)nd.din * nd.dout, etot_one = (uint64_t)nd.din * lt.starts.size();
            const uint64_t E = reg.max_execs;  // per party: E executions, party stride E * plane
            const uint64_t cells_all = E * cells_one, etot = E * etot_one;
            for (uint64_t ex = 0; ex < E; ++ex)  // preproc.cpp:104-112: per execution, per tile
            for (size_t t = 0; t < lt.starts.size(); ++t) {
                const uint32_t rows = lt.counts[t];
                const uint64_t cells = (uint64_t)nd.din * rows;
                uint32_t* A = dd.scratch;
                uint32_t* B = A + cells;
                uint32_t* Cc = B + nd.din;
                lk(launch_dealer_uniform(ctx->stream, seed, k, cells, 1, A, ctx->d_flag, ctx->sms), "deal A");
                k += cells;
                lk(launch_dealer_uniform(ctx->stream, seed, k, nd.din, 1, B, ctx->d_flag, ctx->sms), "deal B");
                k += nd.din;
                lk(launch_dealer_matvec(ctx->stream, A, B, nd.din, rows, Cc), "deal C");
                const uint64_t aoff = ex * cells_one + (uint64_t)lt.starts[t] * nd.din;
                lk(launch_dealer_share(ctx->stream, n, seed, k, alpha, A, cells, pl[0] + aoff, pl[1] + aoff, cells_all,
                                       ctx->d_flag, ctx->sms),
                   "share A");
                k += dealer_draws_share(n, cells);
                const uint64_t boff = ex * etot_one + (uint64_t)t * nd.din;
                lk(launch_dealer_share(ctx->stream, n, seed, k, alpha, B, nd.din, pl[2] + boff, pl[3] + boff, etot,
                                       ctx->d_flag, ctx->sms),
                   "share B");
                k += dealer_draws_share(n, nd.din);
                lk(launch_dealer_share(ctx->stream, n, seed, k, alpha, Cc, rows, pl[4] + ex * nd.dout + lt.starts[t],
                                       pl[5] + ex * nd.dout + lt.starts[t], E * nd.dout, ctx->d_flag, ctx->sms),
                   "share C");
                k += dealer_draws_share(n, rows);
                (void)reg;
            }
        }
        for (auto& [id, moff] : r->input_mask_off) {
            const uint64_t cnt = r->node(id).lanes;
            lk(launch_dealer_masks(ctx->stream, n, seed, k, alpha, r->input_mask_gfirst[id], cnt, M,
                                   dd.mask_v + moff, dd.mask_m + moff, dd.mask_c + moff, ctx->d_flag, ctx->sms),
               "deal masks");
        }
        check_dealer_flag(ctx);
    }
    r->consumed = false;
    r->masks_used = false;
    r->dealer_seed = seed;
}

// ---- preprocessing from the reference's store files (instead of deal) ----
// Party p's MPCT file: the slices of the global layout this run consumes, straight into
// the pools deal() would have filled (same offsets, so the online phase is unchanged).
void load_store(spdz_run* r, int p, const char* path) {
    need(p >= 0 && p < r->n && r->parties[p].local, SPDZ_ERR_INVALID_ARGUMENT, "party is not local to this run");
    const StoreLayout L = scan_store(path);
    need(L.party == p && L.n_parties == r->n, SPDZ_ERR_STORE_FORMAT,
         "VersionMismatch: store is party " + std::to_string(L.party) + " of " + std::to_string(L.n_parties) +
             ", run needs party " + std::to_string(p) + " of " + std::to_string(r->n));
    // the layout of loop bodies scales with the store's loop_iters (PartyRuntime plans it from the store)
    bool loops = false;
    for (auto& nd : r->nodes) loops = loops || nd.loop_depth > 0;
    need(!loops || L.loop_iters == r->loop_iters, SPDZ_ERR_STORE_FORMAT,
         "VersionMismatch: store provisioned for loop_iters " + std::to_string(L.loop_iters) + ", run planned for " +
             std::to_string(r->loop_iters));
    // demand check of load_run_bundle (preproc.cpp:182-201)
    const size_t mats_needed = r->matrix_total;
    if (L.n_scalar < r->scalar_total_global)
        throw Error(SPDZ_ERR_INSUFFICIENT_TRIPLES, "InsufficientTriples: need " + std::to_string(r->scalar_total_global) +
                                                       " scalar triples, store has " + std::to_string(L.n_scalar));
    if (L.mats.size() < mats_needed)
        throw Error(SPDZ_ERR_INSUFFICIENT_TRIPLES, "InsufficientTriples: need " + std::to_string(mats_needed) +
                                                       " matrix triples, store has " + std::to_string(L.mats.size()));
    if (L.n_masks < r->mask_total_global)
        throw Error(SPDZ_ERR_INSUFFICIENT_TRIPLES, "InsufficientTriples: need " + std::to_string(r->mask_total_global) +
                                                       " input masks, store has " + std::to_string(L.n_masks));
    auto& P = r->parties[p];
    dev(r, p);
    StagedUpload up(path, r->copy_stream);
    // scalar triples: region slices of the six planes (take_range offsets, triple_store.cpp:108-133)
    for (auto& [id, reg] : r->scalar) {
        const uint64_t cnt = reg.stride * reg.max_execs;
        for (int q = 0; q < 6; ++q)
            up.copy(L.scalar_off + 4 * ((uint64_t)q * L.n_scalar + reg.gbase), 4 * cnt, P.pool[q] + reg.base);
    }
    // matrix triples in demand order: linear nodes by id, tiles in order (take_matrix_at)
    size_t k = 0;
    for (auto& [id, reg] : r->matrix) {
        const auto& nd = r->node(id);
        const auto& lt = r->tiles[id];
        auto& st = P.ns[id];
        const uint64_t cells1 = (uint64_t)nd.din * nd.dout, etot1 = (uint64_t)nd.din * lt.starts.size();
        for (uint64_t ex = 0; ex < reg.max_execs; ++ex)
        for (size_t t = 0; t < lt.starts.size(); ++t, ++k) {
            const auto& m = L.mats[k];
            const uint32_t rows = lt.counts[t];
            if (m.rows != rows || m.din != nd.din)
                throw Error(SPDZ_ERR_TRIPLE_SHAPE_MISMATCH,
                            "TripleShapeMismatch: store has " + std::to_string(m.rows) + "x" + std::to_string(m.din) +
                                ", tile needs " + std::to_string(rows) + "x" + std::to_string(nd.din));
            const uint64_t cells = (uint64_t)rows * nd.din;
            uint64_t at = m.off;
            const uint64_t aoff = ex * cells1 + (uint64_t)lt.starts[t] * nd.din, boff = ex * etot1 + (uint64_t)t * nd.din;
            const uint64_t coff = ex * nd.dout + lt.starts[t];
            uint32_t* dst[6] = {st.mA0[0] + aoff, st.mA0[1] + aoff, st.mB0[0] + boff,
                                st.mB0[1] + boff, st.mC0[0] + coff, st.mC0[1] + coff};
            const uint64_t words[6] = {cells, cells, nd.din, nd.din, rows, rows};
            for (int q = 0; q < 6; ++q) {
                up.copy(at, 4 * words[q], dst[q]);
                at += 4 * words[q];
            }
            (void)reg;
        }
    }
    // input masks (take_masks, triple_store.cpp:156-161); party 0's file carries the clear values
    for (auto& [id, moff] : r->input_mask_off)
        up.copy_masks(L.masks_off, r->input_mask_gfirst[id], r->node(id).lanes, P.mask_v + moff, P.mask_m + moff,
                      p == 0 ? P.mask_c + moff : nullptr);
    up.finish();
    set_alpha(P.ctx, L.alpha_share);
    r->consumed = false;
    r->masks_used = false;
}

void alloc_deals(spdz_run* r) {
    const int n = r->n;
    const uint64_t S = r->scalar_total, M = r->mask_total;
    uint64_t scratch = 1;
    for (auto& [id, reg] : r->matrix) {
        const auto& nd = r->node(id);
        for (auto c : r->tiles[id].counts) scratch = std::max<uint64_t>(scratch, (uint64_t)nd.din * c + nd.din + c);
    }
    for (int p = 0; p < n; ++p) {
        if (!r->parties[p].local) continue;
        const int d = r->devices[p];
        if (r->deals.count(d)) continue;
        DeviceDeal dd;
        for (int k = 0; k < 6; ++k) dd.pool[k] = r->alloc_dev_words(d, n * S);
        dd.mask_v = r->alloc_dev_words(d, n * M);
        dd.mask_m = r->alloc_dev_words(d, n * M);
        dd.mask_c = r->alloc_dev_words(d, M);
        for (auto& [id, reg] : r->matrix) {  // per party: max_execs executions of every plane
            const auto& nd = r->node(id);
            const uint64_t E = reg.max_execs;
            const uint64_t cells = (uint64_t)nd.din * nd.dout, etot = (uint64_t)nd.din * r->tiles[id].starts.size();
            std::array<uint32_t*, 6> pl;
            pl[0] = r->alloc_dev_words(d, n * E * cells);
            pl[1] = r->alloc_dev_words(d, n * E * cells);
            pl[2] = r->alloc_dev_words(d, n * E * etot);
            pl[3] = r->alloc_dev_words(d, n * E * etot);
            pl[4] = r->alloc_dev_words(d, n * E * (uint64_t)nd.dout);
            pl[5] = r->alloc_dev_words(d, n * E * (uint64_t)nd.dout);
            dd.layer[id] = pl;
        }
        dd.scratch = r->alloc_dev_words(d, scratch);
        r->deals[d] = dd;
    }
    for (int p = 0; p < n; ++p) {  // per-party views (party-major planes)
        auto& P = r->parties[p];
        if (!P.local) continue;
        auto& dd = r->deals[r->devices[p]];
        for (int k = 0; k < 6; ++k) P.pool[k] = dd.pool[k] + p * S;
        P.mask_v = dd.mask_v + p * M;
        P.mask_m = dd.mask_m + p * M;
        P.mask_c = dd.mask_c;
        for (auto& [id, reg] : r->matrix) {
            const auto& nd = r->node(id);
            const uint64_t cells = (uint64_t)nd.din * nd.dout, etot = (uint64_t)nd.din * r->tiles[id].starts.size();
            auto& pl = dd.layer[id];
            auto& st = P.ns[id];
            const uint64_t E = r->matrix.at(id).max_execs;
            st.mA[0] = st.mA0[0] = pl[0] + p * E * cells;
            st.mA[1] = st.mA0[1] = pl[1] + p * E * cells;
            st.mB[0] = st.mB0[0] = pl[2] + p * E * etot;
            st.mB[1] = st.mB0[1] = pl[3] + p * E * etot;
            st.mC[0] = st.mC0[0] = pl[4] + p * E * (uint64_t)nd.dout;
            st.mC[1] = st.mC0[1] = pl[5] + p * E * (uint64_t)nd.dout;
        }
    }
}

// kernel-class timing brackets on party p's stream (profile_kernels)
int ktimer_begin(spdz_run* r, int p) {
    if (!r->opts.profile_kernels) return -1;
    cudaEvent_t a = r->kt.take(r->devices[p]);
    dev(r, p);
    // inside a graph capture the event becomes an event-record node, re-recorded by every replay
    lk(r->kt_capturing ? cudaEventRecordWithFlags(a, S(r, p), cudaEventRecordExternal) : cudaEventRecord(a, S(r, p)),
       "record");
    r->kt.recs.push_back({-1, r->devices[p], a, nullptr, 0});
    return (int)r->kt.recs.size() - 1;
}
void ktimer_end(spdz_run* r, int p, int idx, int cls, uint64_t bytes) {
    if (idx < 0) return;
    cudaEvent_t b = r->kt.take(r->devices[p]);
    lk(r->kt_capturing ? cudaEventRecordWithFlags(b, S(r, p), cudaEventRecordExternal) : cudaEventRecord(b, S(r, p)),
       "record");
    auto& rec = r->kt.recs[idx];
    rec.cls = cls;
    rec.b = b;
    rec.bytes = bytes;
}


}  // namespace rt
}  // namespace spdzb200
