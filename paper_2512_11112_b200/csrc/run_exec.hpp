// Node execution of the n-party online phase (runtime.cpp:360-450 and the block
// scheduler of scheduler.cpp): the Exec driver used by run.cu.  Included once, by run.cu.
#pragma once
#include "run_state.hpp"

namespace spdzb200 {
namespace rt {

// ---- node execution (runtime.cpp:360-450) ----
struct Exec {
    spdz_run* r;
    int ev_cursor[SPDZ_MAX_PARTIES] = {};

    int tbegin(int p) { return ktimer_begin(r, p); }
    void tend(int p, int idx, int cls, uint64_t bytes) { ktimer_end(r, p, idx, cls, bytes); }

    cudaEvent_t next_event(int p) {  // loops open a node once per execution: the pool grows on demand
        auto& evs = r->parties[p].evs;
        if (ev_cursor[p] >= (int)evs.size()) new_event(r, p);
        return evs.at(ev_cursor[p]++);
    }

    // party p's payload for `slot` is complete on its stream: tell local peers
    // (event) and remote peers (flag word, spdz_run_import)
    cudaEvent_t publish(int p, uint64_t slot) {
        cudaEvent_t e = next_event(p);
        lk(cudaEventRecord(e, S(r, p)), "record");
        signal_remote(r, p, slot);
        return e;
    }
    // party p's stream waits for party q's payload of `slot`
    void await(int p, int q, cudaEvent_t ev, uint64_t slot) {
        if (r->parties[q].local) lk(cudaStreamWaitEvent(S(r, p), ev, 0), "wait peer");
        else wait_remote(r, p, q, slot);
    }

    // bcast_share(s, lanes) into dst (runtime.cpp:41-47) when lanes differ
    void bcast_into(int p, const Val& s, const Val& dst) {
        if (s.v == dst.v) return;
        lk(launch_bcast(S(r, p), s.v, s.m, dst.v, dst.m, dst.lanes, SMS(r, p)), "bcast");
    }

    // runtime.cpp:129-162
    // both co-located parties' private add / sub of L-lane operands in one launch
    bool add_pair(uint32_t id, bool sub) {
        if (!colocated2(r)) return false;
        const auto& n = r->node(id);
        const uint64_t L = n.lanes;
        const Val* v[2][3];
        for (int p = 0; p < 2; ++p) {
            auto& P = r->parties[p];
            v[p][0] = &P.ns[n.operands[0]].out;
            v[p][1] = &P.ns[n.operands[1]].out;
            v[p][2] = &P.ns[id].out;
            for (int k = 0; k < 3; ++k)
                if (v[p][k]->is_public || v[p][k]->lanes != L) return false;
        }
        dev(r, 0);
        const uint32_t* xy[8] = {v[0][0]->v, v[0][0]->m, v[0][1]->v, v[0][1]->m,
                                 v[1][0]->v, v[1][0]->m, v[1][1]->v, v[1][1]->m};
        uint32_t* const z[4] = {v[0][2]->v, v[0][2]->m, v[1][2]->v, v[1][2]->m};
        // the next issued node: an add / sub consuming this result, fused (then its root opening)
        int k1 = fusion_allowed() ? next_work(id) : -1;
        int sm2 = -1;
        const Val* o[2] = {nullptr, nullptr};
        if (k1 >= 0) {
            const auto& n1 = r->nodes[k1];
            bool ok = (n1.kind == SPDZ_NODE_ADD || n1.kind == SPDZ_NODE_SUB) && n1.lanes == L;
            for (auto& f : r->faults) ok = ok && f.node != (uint32_t)k1;
            for (int p = 0; p < 2 && ok; ++p) {
                const auto& P = r->parties[p];
                const Val &a = P.ns[n1.operands[0]].out, &b = P.ns[n1.operands[1]].out, &w2 = P.ns[k1].out;
                const Val& w = *v[p][2];
                ok = !a.is_public && !b.is_public && !w2.is_public && a.lanes == L && b.lanes == L && w2.lanes == L;
                const bool wl = ok && a.v == w.v, wr = ok && b.v == w.v;
                ok = ok && wl != wr && disjoint(wl ? b : a, w, L);
                const int s2 = wl ? (n1.kind == SPDZ_NODE_SUB ? 1 : 0) : (n1.kind == SPDZ_NODE_SUB ? 2 : 0);
                ok = ok && (sm2 < 0 || s2 == sm2);
                sm2 = s2;
                o[p] = wl ? &b : &a;
            }
            if (!ok) k1 = -1;
        }
        if (k1 < 0) {
            lk(launch_add_sub2(S(r, 0), sub, xy, z, L, SMS(r, 0)), "add_batch (both parties)");
            return true;
        }
        const uint32_t* ov[4] = {o[0]->v, o[0]->m, o[1]->v, o[1]->m};
        auto &w0 = r->parties[0].ns[k1].out, &w1 = r->parties[1].ns[k1].out;
        uint32_t* const wo[4] = {w0.v, w0.m, w1.v, w1.m};
        const bool root = root_opens((uint32_t)k1, L);
        uint32_t* outs[2] = {r->parties[0].outputs, r->parties[1].outputs};
        lk(launch_add_sub2_chain(S(r, 0), sub, xy, z, sm2, ov, wo, root ? outs : nullptr, L, SMS(r, 0)),
           "add_batch + next add (both parties)");
        if (r->precomputed.size() != r->nodes.size()) r->precomputed.assign(r->nodes.size(), 0);
        r->precomputed[k1] = 1;
        if (root) r->root_opened = true;
        return true;
    }

    void add(int p, uint32_t id, bool sub) {
        auto& P = r->parties[p];
        const auto& n = r->node(id);
        const Val &a = P.ns[n.operands[0]].out, &b = P.ns[n.operands[1]].out;
        Val& o = P.ns[id].out;
        const uint64_t L = n.lanes;
        spdz_ctx* c = P.ctx;
        if (a.is_public && b.is_public) {
            lk(launch_pub_binop(c->stream, sub ? 1 : 0, a.pub, a.lanes != L, b.pub, b.lanes != L, o.pub, L, c->sms),
               "pub add");
            return;
        }
        if (!a.is_public && !b.is_public) {
            need(a.lanes == L || a.lanes == 1, SPDZ_ERR_LANE_MISMATCH, "LaneMismatch: add operand");
            need(b.lanes == L || b.lanes == 1, SPDZ_ERR_LANE_MISMATCH, "LaneMismatch: add operand");
            if (a.lanes != L && b.lanes != L) {  // both broadcast scalars: z[0] = a op b, then bcast
                lk(launch_add_sub(c->stream, sub, a.v, a.m, b.v, b.m, o.v, o.m, 1, c->sms), "add 1");
                if (L > 1) lk(launch_bcast(c->stream, o.v, o.m, o.v + 1, o.m + 1, L - 1, c->sms), "bcast");
                return;
            }
            const uint32_t *av = a.v, *am = a.m, *bv = b.v, *bm = b.m;
            if (a.lanes != L) {  // bcast_share(a) into the output, then z = z op b in place
                bcast_into(p, a, o);
                av = o.v;
                am = o.m;
            } else if (b.lanes != L) {
                bcast_into(p, b, o);
                bv = o.v;
                bm = o.m;
            }
            lk(launch_add_sub(c->stream, sub, av, am, bv, bm, o.v, o.m, L, c->sms), "add_batch");
            return;
        }
        // share op public / public op share (runtime.cpp:145-161)
        const bool a_priv = !a.is_public;
        const Val& sh = a_priv ? a : b;
        const Val& pb = a_priv ? b : a;
        const int op = a_priv ? (sub ? 1 : 0) : (sub ? 2 : 0);
        const uint32_t* iv = sh.v;
        const uint32_t* im = sh.m;
        if (sh.lanes != L) {
            bcast_into(p, sh, o);
            iv = o.v;
            im = o.m;
        }
        lk(launch_public(c->stream, op, iv, im, pb.pub, pb.lanes != L, 0u, false, c->party, c->alpha, o.v, o.m, L,
                         c->sms, c->d_alpha),
           "public op");
    }

    // runtime.cpp:166-183
    void mul_local(int p, uint32_t id) {
        auto& P = r->parties[p];
        const auto& n = r->node(id);
        const Val &a = P.ns[n.operands[0]].out, &b = P.ns[n.operands[1]].out;
        Val& o = P.ns[id].out;
        const uint64_t L = n.lanes;
        spdz_ctx* c = P.ctx;
        if (a.is_public && b.is_public) {
            lk(launch_pub_binop(c->stream, 2, a.pub, a.lanes != L, b.pub, b.lanes != L, o.pub, L, c->sms), "pub mul");
            return;
        }
        const Val& sh = a.is_public ? b : a;
        const Val& pb = a.is_public ? a : b;
        const uint32_t* iv = sh.v;
        const uint32_t* im = sh.m;
        if (sh.lanes != L) {
            bcast_into(p, sh, o);
            iv = o.v;
            im = o.m;
        }
        lk(launch_public(c->stream, 3, iv, im, pb.pub, pb.lanes != L, 0u, false, c->party, c->alpha, o.v, o.m, L,
                         c->sms, c->d_alpha),
           "mul_public");
    }

    const uint32_t* peer_payload(int p, int q, uint32_t id, const uint32_t* src, uint64_t words, uint32_t* shadow) {
        // SimHub BitFlip (net.cpp:241-278): the receiver p sees a tampered copy of q's frame.
        for (auto& f : r->faults) {
            if (f.node == id && f.sender == q && f.receiver == p && shadow) {
                lk(cudaMemcpyAsync(shadow, src, words * 4, cudaMemcpyDefault, S(r, p)), "shadow copy");
                lk(launch_xor_word(S(r, p), shadow + (f.word % words), 1u << (f.bit % 32)), "bitflip");
                return shadow;
            }
        }
        return src;
    }

    // ---- network peers (the reference's frames, net.cpp) ----
    bool netpeer(int q) const { return r->net && !r->parties[q].local; }

    // party p's payload words to every peer as one frame (async_open / exchange send side)
    void net_send(int p, uint8_t type, uint64_t batch, const uint32_t* dsrc, uint64_t words) {
        need(r->net != nullptr, SPDZ_ERR_INVALID_ARGUMENT, "network run without an attached mesh");
        uint32_t* h = (uint32_t*)r->net_stage.ensure(std::max<uint64_t>(words, 1) * 4);
        dev(r, p);
        if (words) lk(cudaMemcpyAsync(h, dsrc, words * 4, cudaMemcpyDeviceToHost, S(r, p)), "D2H frame");
        lk(cudaStreamSynchronize(S(r, p)), "frame");
        r->net->broadcast(type, batch, h, (uint32_t)words);
    }

    // peer q's frame (type, batch) into device memory on party p's stream (net.cpp:186-208)
    void net_recv(int p, int q, uint8_t type, uint64_t batch, uint32_t* ddst, uint64_t words) {
        std::vector<uint32_t> v = r->net->recv(q, type, batch);
        need(v.size() == words, SPDZ_ERR_LANE_COUNT_MISMATCH,
             "LaneCountMismatch: peer " + std::to_string(q) + " sent " + std::to_string(v.size()) +
                 " lanes, expected " + std::to_string(words));
        if (!words) return;
        uint32_t* h = (uint32_t*)r->net_stage.ensure(words * 4);
        std::memcpy(h, v.data(), words * 4);
        dev(r, p);
        lk(cudaMemcpyAsync(ddst, h, words * 4, cudaMemcpyHostToDevice, S(r, p)), "H2D frame");
        lk(cudaStreamSynchronize(S(r, p)), "frame");
    }

    // linear layer: one frame per tile, [D_t | E_t] (linear.cpp:94-113), batch batch0 + t;
    // our payload holds [D (all rows) | E_t for every tile]
    void net_send_tiles(int p, uint64_t batch0, const uint32_t* dsrc, uint32_t din, const LinTiles& lt) {
        const uint64_t nt = lt.starts.size(), cells = (uint64_t)din * (lt.starts.empty() ? 0 : lt.starts.back() +
                                                                                                    lt.counts.back());
        const uint64_t words = cells + din * nt;
        uint32_t* h = (uint32_t*)r->net_stage.ensure(words * 4);
        dev(r, p);
        lk(cudaMemcpyAsync(h, dsrc, words * 4, cudaMemcpyDeviceToHost, S(r, p)), "D2H tiles");
        lk(cudaStreamSynchronize(S(r, p)), "tiles");
        for (uint64_t t = 0; t < nt; ++t) {
            const uint64_t ct = (uint64_t)lt.counts[t] * din;
            r->net_host.resize(ct + din);
            std::memcpy(r->net_host.data(), h + (uint64_t)lt.starts[t] * din, ct * 4);
            std::memcpy(r->net_host.data() + ct, h + cells + t * din, din * 4ull);
            r->net->broadcast(kMsgOpenShares, batch0 + t, r->net_host.data(), (uint32_t)(ct + din));
        }
    }
    void net_recv_tiles(int p, int q, uint64_t batch0, uint32_t* ddst, uint32_t din, const LinTiles& lt) {
        const uint64_t nt = lt.starts.size(), cells = (uint64_t)din * (lt.starts.back() + lt.counts.back());
        const uint64_t words = cells + din * nt;
        uint32_t* h = (uint32_t*)r->net_stage.ensure(words * 4);
        for (uint64_t t = 0; t < nt; ++t) {
            const uint64_t ct = (uint64_t)lt.counts[t] * din;
            std::vector<uint32_t> v = r->net->recv(q, kMsgOpenShares, batch0 + t);
            need(v.size() == ct + din, SPDZ_ERR_LANE_COUNT_MISMATCH,
                 "LaneCountMismatch: peer " + std::to_string(q) + " sent " + std::to_string(v.size()) +
                     " lanes, expected " + std::to_string(ct + din));
            std::memcpy(h + (uint64_t)lt.starts[t] * din, v.data(), ct * 4);
            std::memcpy(h + cells + t * din, v.data() + ct, din * 4ull);
        }
        dev(r, p);
        lk(cudaMemcpyAsync(ddst, h, words * 4, cudaMemcpyHostToDevice, S(r, p)), "H2D tiles");
        lk(cudaStreamSynchronize(S(r, p)), "tiles");
    }

    // The MAC shares a Beaver record is checked against: the operand planes themselves, or
    // (control flow, where a later execution rewrites them) a per-execution snapshot.
    const uint32_t* mac_slot(int p, uint32_t id, uint64_t exec, int which) {
        auto& st = r->parties[p].ns[id];
        const Val& x = which ? st.xb : st.xa;
        if (!r->cfg) return x.m;
        const uint64_t L = r->node(id).lanes;
        uint32_t* dst = st.macsnap + 2 * L * exec + (which ? L : 0);
        dev(r, p);
        lk(cudaMemcpyAsync(dst, x.m, L * 4, cudaMemcpyDeviceToDevice, S(r, p)), "mac snapshot");
        return dst;
    }

    // runtime.cpp:119-125 read_public: lane 0 of a completed public value (host read)
    uint32_t read_public(uint32_t id) {
        const int p = r->ref_party();
        const Val& v = r->parties[p].ns[id].out;
        need(v.is_public && v.lanes >= 1 && v.pub, SPDZ_ERR_INVALID_ARGUMENT,
             "runtime: node " + std::to_string(id) + " is not a completed public scalar");
        dev(r, p);
        uint32_t x = 0;
        lk(cudaMemcpyAsync(&x, v.pub, 4, cudaMemcpyDeviceToHost, S(r, p)), "read public");
        lk(cudaStreamSynchronize(S(r, p)), "read public");
        return x;
    }

    // runtime.cpp:419-438 with a start computed at run time: copy the slice
    void load_dynamic(uint32_t id) {
        const auto& n = r->node(id);
        const uint32_t start = read_public(n.operands[1]);
        for (int p = 0; p < r->n; ++p) {
            auto& P = r->parties[p];
            if (!P.local) continue;
            const Val& base = P.ns[n.operands[0]].out;
            const Val& o = P.ns[id].out;
            need((uint64_t)start + n.lanes <= base.lanes, SPDZ_ERR_INVALID_ARGUMENT, "runtime: load out of bounds");
            dev(r, p);
            if (base.is_public) {
                lk(cudaMemcpyAsync(o.pub, base.pub + start, n.lanes * 4ull, cudaMemcpyDeviceToDevice, S(r, p)), "load");
            } else {
                lk(cudaMemcpyAsync(o.v, base.v + start, n.lanes * 4ull, cudaMemcpyDeviceToDevice, S(r, p)), "load");
                lk(cudaMemcpyAsync(o.m, base.m + start, n.lanes * 4ull, cudaMemcpyDeviceToDevice, S(r, p)), "load");
            }
        }
    }

    // vals[phi] = vals[chosen] (scheduler.cpp:242-262 via resolve_phi), into the phi's own
    // buffer: broadcast a 1-lane value, and a public value reaching a private phi becomes
    // the sharing of that public (share_of_public, spdz.cpp:66-75)
    void phi_copy(uint32_t phi, uint32_t chosen) {
        const bool dyn = r->nodes[phi].is_private && eff_pub(chosen);
        for (int p = 0; p < r->n; ++p) {
            auto& P = r->parties[p];
            if (!P.local) continue;
            const Val& s = P.ns[chosen].out;
            const Val& o = P.ns[phi].out;
            need(s.lanes == o.lanes || s.lanes == 1, SPDZ_ERR_LANE_MISMATCH,
                 "LaneMismatch: phi " + std::to_string(phi) + " takes " + std::to_string(s.lanes) + " lanes into " +
                     std::to_string(o.lanes));
            dev(r, p);
            spdz_ctx* c = P.ctx;
            if (o.is_public) {
                need(s.is_public, SPDZ_ERR_INVALID_ARGUMENT, "runtime: private value reaches public phi");
                if (s.lanes == o.lanes)
                    lk(cudaMemcpyAsync(o.pub, s.pub, o.lanes * 4, cudaMemcpyDeviceToDevice, c->stream), "phi");
                else
                    lk(launch_bcast(c->stream, s.pub, nullptr, o.pub, nullptr, o.lanes, c->sms), "phi bcast");
                continue;
            }
            if (eff_pub(chosen)) {  // party 0 holds k, MAC shares alpha_i * k; k kept as the public value
                const uint32_t* k = pub_of(p, chosen);
                lk(launch_public(c->stream, 4, nullptr, nullptr, k, s.lanes != o.lanes, 0u, false, c->party,
                                 c->alpha, o.v, o.m, o.lanes, c->sms, c->d_alpha),
                   "phi share_of_public");
                uint32_t* sp = P.ns[phi].shadow_pub;
                if (s.lanes == o.lanes)
                    lk(cudaMemcpyAsync(sp, k, o.lanes * 4, cudaMemcpyDeviceToDevice, c->stream), "phi");
                else
                    lk(launch_bcast(c->stream, k, nullptr, sp, nullptr, o.lanes, c->sms), "phi bcast");
            } else if (s.lanes == o.lanes) {
                lk(cudaMemcpyAsync(o.v, s.v, o.lanes * 4, cudaMemcpyDeviceToDevice, c->stream), "phi");
                lk(cudaMemcpyAsync(o.m, s.m, o.lanes * 4, cudaMemcpyDeviceToDevice, c->stream), "phi");
            } else {
                lk(launch_bcast(c->stream, s.v, s.m, o.v, o.m, o.lanes, c->sms), "phi bcast");
            }
        }
        r->rt_pub[phi] = dyn;
    }

    // is the node's current value public (statically, or a private-typed node holding a public)?
    bool eff_pub(uint32_t id) const {
        return r->parties[r->ref_party()].ns[id].out.is_public || (r->cfg && r->rt_pub[id]);
    }
    const uint32_t* pub_of(int p, uint32_t id) const {
        const auto& st = r->parties[p].ns[id];
        return st.out.is_public ? st.out.pub : st.shadow_pub;
    }

    // load / reduce_add / reduce_mul of a private-typed value that is public at run time:
    // computed publicly (a reduce_mul needs no product tree), its sharing beside it
    bool exec_dynamic_unary(uint32_t id) {
        const auto& n = r->nodes[id];
        const uint32_t src = n.operands[0];
        r->rt_pub[id] = 0;
        if (!r->rt_pub[src] || r->parties[r->ref_party()].ns[src].out.is_public) return false;
        if (n.kind == SPDZ_NODE_LOAD) {  // the share view (or copy) plus the public value's
            exec_node_static_load(id);
            r->rt_pub[id] = 1;
            return true;
        }
        for (int p = 0; p < r->n; ++p) {
            auto& P = r->parties[p];
            if (!P.local) continue;
            auto& st = P.ns[id];
            const Val& a = P.ns[src].out;
            spdz_ctx* c = P.ctx;
            dev(r, p);
            const uint32_t* k = pub_of(p, src);
            if (n.kind == SPDZ_NODE_REDUCE_ADD) {
                lk(cudaMemsetAsync(c->d_acc + 2, 0, 16, c->stream), "memset");
                lk(launch_reduce_add(c->stream, k, k, a.lanes, c->d_acc + 2, c->sms), "dyn reduce");
                lk(launch_finish_reduce(c->stream, c->d_acc + 2, st.shadow_pub, st.shadow_pub), "finish");
            } else {  // product of the lanes, folded in halves (order-free)
                uint64_t len = a.lanes;
                lk(cudaMemcpyAsync(st.shadow_pub, k, len * 4, cudaMemcpyDeviceToDevice, c->stream), "copy");
                while (len > 1) {
                    const uint64_t half = len / 2;
                    lk(launch_pub_binop(c->stream, 2, st.shadow_pub, false, st.shadow_pub + (len - half), false,
                                        st.shadow_pub, half, c->sms),
                       "dyn product");
                    len -= half;
                }
            }
            lk(launch_public(c->stream, 4, nullptr, nullptr, st.shadow_pub, false, 0u, false, c->party, c->alpha,
                             st.out.v, st.out.m, 1, c->sms, c->d_alpha),
               "dyn share_of_public");
        }
        r->rt_pub[id] = 1;
        return true;
    }

    // a load's usual execution (a view needs nothing; a run-time start copies), plus the public
    // value's slice when its base is public at run time
    void exec_node_static_load(uint32_t id) {
        const auto& n = r->nodes[id];
        if (!r->parties[r->ref_party()].ns[id].dyn_load) return;  // views: shadow_pub points into the base's
        const uint32_t start = read_public(n.operands[1]);
        load_dynamic(id);
        for (int p = 0; p < r->n; ++p) {
            auto& P = r->parties[p];
            if (!P.local) continue;
            dev(r, p);
            lk(cudaMemcpyAsync(P.ns[id].shadow_pub, P.ns[n.operands[0]].shadow_pub + start, n.lanes * 4ull,
                               cudaMemcpyDeviceToDevice, S(r, p)),
               "dyn load");
        }
    }

    // Control flow: add/sub/mul of a private-typed node whose operands are public at run time
    // compute publicly (the public value kept beside its sharing), and a multiply by such a value
    // is a local mul_public — no Beaver triple, as the reference's exec_add / exec_mul_local see
    // public RtValues (runtime.cpp:129-183).  Returns true when it handled the node.
    bool exec_dynamic_public(uint32_t id) {
        const auto& n = r->nodes[id];
        if (r->parties[r->ref_party()].ns[id].out.is_public) return false;
        if (n.kind == SPDZ_NODE_LOAD || n.kind == SPDZ_NODE_REDUCE_ADD || n.kind == SPDZ_NODE_REDUCE_MUL)
            return exec_dynamic_unary(id);
        if (n.kind != SPDZ_NODE_ADD && n.kind != SPDZ_NODE_SUB && n.kind != SPDZ_NODE_MUL) return false;
        r->rt_pub[id] = 0;
        const bool pa = eff_pub(n.operands[0]), pb = eff_pub(n.operands[1]);
        const bool dyn_a = pa && !r->parties[r->ref_party()].ns[n.operands[0]].out.is_public;
        const bool dyn_b = pb && !r->parties[r->ref_party()].ns[n.operands[1]].out.is_public;
        if (!dyn_a && !dyn_b) return false;  // static typing already decides this node
        const uint64_t L = n.lanes;
        for (int p = 0; p < r->n; ++p) {
            auto& P = r->parties[p];
            if (!P.local) continue;
            auto& st = P.ns[id];
            const Val &a = P.ns[n.operands[0]].out, &b = P.ns[n.operands[1]].out;
            spdz_ctx* c = P.ctx;
            dev(r, p);
            if (pa && pb) {  // public op, then its sharing for private-typed consumers
                const int op = n.kind == SPDZ_NODE_ADD ? 0 : (n.kind == SPDZ_NODE_SUB ? 1 : 2);
                lk(launch_pub_binop(c->stream, op, pub_of(p, n.operands[0]), a.lanes != L, pub_of(p, n.operands[1]),
                                    b.lanes != L, st.shadow_pub, L, c->sms),
                   "dyn pub op");
                lk(launch_public(c->stream, 4, nullptr, nullptr, st.shadow_pub, false, 0u, false, c->party, c->alpha,
                                 st.out.v, st.out.m, L, c->sms, c->d_alpha),
                   "dyn share_of_public");
                continue;
            }
            if (n.kind != SPDZ_NODE_MUL) return false;  // share +- sharing-of-public == add_public
            const Val& sh = pa ? b : a;
            const uint32_t* k = pub_of(p, pa ? n.operands[0] : n.operands[1]);
            const uint64_t kl = (pa ? a : b).lanes;
            const uint32_t *iv = sh.v, *im = sh.m;
            if (sh.lanes != L) {
                bcast_into(p, sh, st.out);
                iv = st.out.v;
                im = st.out.m;
            }
            lk(launch_public(c->stream, 3, iv, im, k, kl != L, 0u, false, c->party, c->alpha, st.out.v, st.out.m, L,
                             c->sms, c->d_alpha),
               "dyn mul_public");
        }
        r->rt_pub[id] = pa && pb;
        return true;
    }

    // Block-by-block execution of a control-flow graph: the sequential reading of the
    // reference's dataflow scheduler (scheduler.cpp).  Entering a block resolves its phis
    // from the predecessor, then its nodes run in `next` order; a BRANCH reads its public
    // condition (the one host synchronisation) and enters the successor; ROOT ends the phase.
    void run_cfg() {
        const uint32_t N = (uint32_t)r->nodes.size();
        std::vector<uint64_t> execs(N, 0);
        uint32_t label = r->opts.entry_label, pred = SPDZ_NO_NODE;
        for (;;) {
            need(label < N && r->nodes[label].kind == SPDZ_NODE_LABEL, SPDZ_ERR_INVALID_ARGUMENT,
                 "runtime: block " + std::to_string(label) + " is not a block label");
            // phi choices first, as enter_block_locked seeds them
            std::vector<std::pair<uint32_t, uint32_t>> phis;
            uint32_t steps = 0;
            for (uint32_t u = r->nodes[label].next; u != SPDZ_NO_NODE; u = r->nodes.at(u).next) {
                need(++steps <= N, SPDZ_ERR_INVALID_ARGUMENT, "runtime: block " + std::to_string(label) +
                                                                  "'s node chain does not end");
                const auto& n = r->nodes.at(u);
                if (n.kind != SPDZ_NODE_PHI) continue;
                if (pred == SPDZ_NO_NODE)
                    throw Error(SPDZ_ERR_INVALID_ARGUMENT, "UnknownPredecessor: phi " + std::to_string(u) +
                                                               " entered with no recorded predecessor");
                uint32_t chosen = SPDZ_NO_NODE;
                for (uint32_t i = 0; i < n.n_operands; ++i)
                    if (n.phi_labels[i] == pred) {
                        chosen = n.operands[i];
                        break;
                    }
                if (chosen == SPDZ_NO_NODE)
                    throw Error(SPDZ_ERR_INVALID_ARGUMENT, "UnknownPredecessor: phi " + std::to_string(u) +
                                                               " has no pair for block " + std::to_string(pred));
                phis.emplace_back(u, chosen);
            }
            for (auto [phi, chosen] : phis)
                if (r->live[phi]) phi_copy(phi, chosen);
            uint32_t dst = SPDZ_NO_NODE;
            for (uint32_t u = r->nodes[label].next; u != SPDZ_NO_NODE; u = r->nodes.at(u).next) {
                const auto& n = r->nodes.at(u);
                if (n.kind == SPDZ_NODE_PHI) continue;
                if (n.kind == SPDZ_NODE_ROOT) return;
                if (n.kind == SPDZ_NODE_BRANCH) {  // scheduler.cpp:283-313
                    if (n.n_succ == 1) {
                        dst = n.succ[0];
                    } else {
                        need(n.n_succ == 2 && n.n_operands >= 1, SPDZ_ERR_INVALID_ARGUMENT, "runtime: malformed branch");
                        const uint32_t cond = n.operands[0];
                        if (r->priv(cond))
                            throw Error(SPDZ_ERR_INVALID_ARGUMENT, "SecretControlFlow: branch " + std::to_string(u) +
                                                                       " conditioned on private node " +
                                                                       std::to_string(cond));
                        dst = read_public(cond) ? n.succ[0] : n.succ[1];
                    }
                    break;
                }
                if (r->live[u]) exec_node(u, execs[u]++);
            }
            need(dst != SPDZ_NO_NODE, SPDZ_ERR_INVALID_ARGUMENT,
                 "runtime: block " + std::to_string(label) + " ends without a branch or the root");
            pred = label;
            label = dst;
        }
    }

    // Beaver multiply (runtime.cpp:204-239): mask -> open [d|e] -> combine, all parties.
    // Both parties of a 2-party run on one stream: both masks, then one fused open+combine
    // (payloads read once, opened values logged once).  (Running it in L2-sized lane blocks so
    // the payloads are re-read from L2 measured slower: the per-launch overhead dominated.)
    // ---- launch fusion along straight-line chains (co-located pair: OpCombine2M / OpCombine2A;
    // per-party kernels: OpCombineM) ----
    bool fusion_allowed() {
        static const bool off = std::getenv("SPDZ_NO_MASK_FUSION") != nullptr;  // (A/B experiments)
        if (off || r->opts.no_fusion || r->cfg || r->opts.node_streams > 1 || r->net) return false;
        // the per-party kernels: 1-3 peers (launch_beaver_combine_mask), no fault injection
        if (!colocated2(r) && (r->n < 2 || r->n > 4 || !r->faults.empty())) return false;
        return true;
    }
    // the next live node after `id` that launches work (static views and markers skipped), or -1
    int next_work(uint32_t id) {
        for (uint32_t k = id + 1; k < r->nodes.size(); ++k) {
            if (!r->live[k]) continue;
            const auto& n = r->nodes[k];
            if (n.kind == SPDZ_NODE_INPUT || n.kind == SPDZ_NODE_CONST || n.kind == SPDZ_NODE_NOP ||
                n.kind == SPDZ_NODE_LABEL)
                continue;
            if (n.kind == SPDZ_NODE_LOAD && !r->parties[r->ref_party()].ns[k].dyn_load) continue;  // a view
            return (int)k;
        }
        return -1;
    }
    // a value read by a fused kernel must not be a view into the product it writes (a load at an
    // offset of z would be read while other threads store z)
    static bool disjoint(const Val& o, const Val& z, uint64_t L) {
        auto apart = [L](const uint32_t* a, const uint32_t* b) { return !a || !b || a + L <= b || b + L <= a; };
        return apart(o.v, z.v) && apart(o.v, z.m) && apart(o.m, z.v) && apart(o.m, z.m);
    }
    // node k is a private Beaver multiply of L lanes (no broadcast operand, not fault-injected) one of
    // whose operands is node src's value, for every local party
    bool mul_consumes(int k, uint32_t src, uint64_t L) {
        if (k < 0) return false;
        const auto& n = r->nodes[k];
        if (n.kind != SPDZ_NODE_MUL || n.lanes != L) return false;
        for (auto& f : r->faults)
            if (f.node == (uint32_t)k) return false;
        for (int p = 0; p < r->n; ++p) {
            if (!r->parties[p].local) continue;
            const auto& P = r->parties[p];
            const auto &st = P.ns[k], &own = P.ns[src];
            if (st.xa.is_public || st.xb.is_public || P.ns[n.operands[0]].out.lanes != L ||
                P.ns[n.operands[1]].out.lanes != L)  // (a broadcast operand is filled by its own node)
                return false;
            if (st.xa.v != own.out.v && st.xb.v != own.out.v) return false;
            if (st.xa.v != own.out.v && !disjoint(st.xa, own.out, L)) return false;
            if (st.xb.v != own.out.v && !disjoint(st.xb, own.out, L)) return false;
        }
        return true;
    }
    // The multiply that runs right after `id` when its mask can be fused into id's combine: the next
    // live node that launches work consumes this product.  Returns -1 otherwise.
    int fusable_next_mul(uint32_t id) {
        if (!fusion_allowed()) return -1;
        const int k = next_work(id);
        return mul_consumes(k, id, r->node(id).lanes) ? k : -1;
    }
    // root node opens node src's value (for every local party, no fault on the root)
    bool root_opens(uint32_t src, uint64_t L) {
        const auto& rn = r->nodes[r->root];
        if (rn.kind != SPDZ_NODE_ROOT || rn.n_operands == 0 || rn.operands[0] != src) return false;
        for (auto& f : r->faults)
            if (f.node == r->root) return false;
        for (int p = 0; p < r->n; ++p) {
            if (!r->parties[p].local) continue;
            const Val& rv = r->parties[p].ns[r->root].out;
            if (rv.is_public || rv.v != r->parties[p].ns[src].out.v || rv.lanes != L) return false;
        }
        return true;
    }
    // Co-located pair: the next node is a private add / sub consuming this product (its other operand
    // a different value of the same lanes): fused into the combine (sm: 0 z + o, 1 z - o, 2 o - z), and
    // after it the multiply consuming its result (nx 1-3, its mask) or the root opening it (nx 4).
    struct AddFuse {
        int k1 = -1, sm = 0, k2 = -1, nx = 0;
    };
    AddFuse fusable_next_add(uint32_t id) {
        AddFuse f;
        if (!fusion_allowed() || r->n != 2) return f;  // per-party kernels: one peer (launch_beaver_combine_add)
        const bool pair = colocated2(r);
        const uint64_t L = r->node(id).lanes;
        const int k1 = next_work(id);
        if (k1 < 0) return f;
        const auto& n = r->nodes[k1];
        if ((n.kind != SPDZ_NODE_ADD && n.kind != SPDZ_NODE_SUB) || n.lanes != L) return f;
        for (auto& ft : r->faults)
            if (ft.node == (uint32_t)k1) return f;
        int sm = -1;
        for (int p = 0; p < 2; ++p) {
            const auto& P = r->parties[p];
            if (!P.local) continue;
            const Val &x = P.ns[n.operands[0]].out, &y = P.ns[n.operands[1]].out, &z = P.ns[id].out,
                      &w = P.ns[k1].out;
            if (x.is_public || y.is_public || w.is_public || x.lanes != L || y.lanes != L || w.lanes != L) return f;
            const bool zl = x.v == z.v, zr = y.v == z.v;
            if (zl == zr) return f;  // neither operand, or z op z
            if (!disjoint(zl ? y : x, z, L)) return f;
            const int s = zl ? (n.kind == SPDZ_NODE_SUB ? 1 : 0) : (n.kind == SPDZ_NODE_SUB ? 2 : 0);
            if (sm >= 0 && s != sm) return f;
            sm = s;
        }
        f.k1 = k1;
        f.sm = sm;
        const int k2 = next_work((uint32_t)k1);
        bool k2_ok = mul_consumes(k2, (uint32_t)k1, L);
        for (int p = 0; p < 2 && k2_ok; ++p) {  // its other operand is read, so it must not be this product
            const auto& P = r->parties[p];
            if (!P.local) continue;
            const auto& st = P.ns[k2];
            const Val& w = P.ns[k1].out;
            if (st.xa.v != w.v && !disjoint(st.xa, P.ns[id].out, L)) k2_ok = false;
            if (st.xb.v != w.v && !disjoint(st.xb, P.ns[id].out, L)) k2_ok = false;
        }
        if (k2_ok) {
            const int rp = r->ref_party();
            const auto& st = r->parties[rp].ns[k2];
            const Val& w = r->parties[rp].ns[k1].out;
            const bool wx = st.xa.v == w.v, wy = st.xb.v == w.v;
            f.k2 = k2;
            f.nx = wx && wy ? 3 : (wx ? 1 : 2);
        } else if (pair && root_opens((uint32_t)k1, L)) {  // (the root opening needs both parties' words)
            f.nx = 4;
        }
        return f;
    }

    // `id` is the multiply the root opens (the last node of a straight-line run): its combine can
    // write the opened outputs of both local parties (the root open without its own launch).
    bool root_fusable(uint32_t id) {
        return fusion_allowed() && colocated2(r) && root_opens(id, r->node(id).lanes);
    }

    void beaver_pair(uint32_t id, uint64_t off) {
        const auto& n = r->node(id);
        const uint64_t L = n.lanes;
        auto &P0 = r->parties[0], &P1 = r->parties[1];
        auto &s0 = P0.ns[id], &s1 = P1.ns[id];
        dev(r, 0);
        if (r->premasked.size() != r->nodes.size()) r->premasked.assign(r->nodes.size(), 0);
        const bool masked = r->premasked[id];
        r->premasked[id] = 0;
        for (int p = 0; p < 2; ++p) {
            auto& P = r->parties[p];
            auto& st = P.ns[id];
            const Val &a = P.ns[n.operands[0]].out, &b = P.ns[n.operands[1]].out;
            if (a.lanes != L) bcast_into(p, a, st.xa);
            if (b.lanes != L) bcast_into(p, b, st.xb);
        }
        const uint32_t alpha[2] = {P0.ctx->alpha, P1.ctx->alpha};
        const uint32_t* alpha_dev[2] = {P0.ctx->d_alpha, P1.ctx->d_alpha};
        if (!masked) {  // both parties' d = x - a, e = y - b in one pass (48 bytes per lane)
            const int tk = tbegin(0);
            const uint32_t* xyab[8] = {s0.xa.v, s0.xb.v, P0.pool[0] + off, P0.pool[2] + off,
                                       s1.xa.v, s1.xb.v, P1.pool[0] + off, P1.pool[2] + off};
            uint32_t* const dd[4] = {s0.payload, s0.payload + L, s1.payload, s1.payload + L};
            lk(launch_mul_mask2(S(r, 0), xyab, dd, L, SMS(r, 0)), "k_mul_mask2");
            tend(0, tk, SPDZ_KSTAT_MASK, 48 * L);
        }
        const uint32_t* de[4] = {s0.payload, s0.payload + L, s1.payload, s1.payload + L};
        const uint32_t *t0[6], *t1[6];
        for (int t = 0; t < 6; ++t) {
            t0[t] = P0.pool[t] + off;
            t1[t] = P1.pool[t] + off;
        }
        uint32_t* z[4] = {s0.out.v, s0.out.m, s1.out.v, s1.out.m};
        const int tk = tbegin(0);
        const int id2 = fusable_next_mul(id);
        const AddFuse af = id2 < 0 ? fusable_next_add(id) : AddFuse{};
        if (af.k1 >= 0) {  // + the add / sub consuming the products, then the next mask or the root open
            auto &w0 = P0.ns[af.k1].out, &w1 = P1.ns[af.k1].out;
            const auto& an = r->node((uint32_t)af.k1);
            const bool zl = P0.ns[an.operands[0]].out.v == s0.out.v;
            const Val &o0 = P0.ns[an.operands[zl ? 1 : 0]].out, &o1 = P1.ns[an.operands[zl ? 1 : 0]].out;
            const uint32_t* addin[4] = {o0.v, o0.m, o1.v, o1.m};
            uint32_t* const wo[4] = {w0.v, w0.m, w1.v, w1.m};
            const uint32_t* next[6] = {};
            uint32_t* extra[4] = {};
            uint64_t eb = 0;
            if (af.k2 >= 0) {
                const uint64_t off2 = provisioned(r->scalar, (uint32_t)af.k2, 0).base;
                auto &n0 = P0.ns[af.k2], &n1 = P1.ns[af.k2];
                const bool wx = af.nx != 2;
                const uint32_t* nx0[3] = {wx ? n0.xb.v : n0.xa.v, P0.pool[0] + off2, P0.pool[2] + off2};
                const uint32_t* nx1[3] = {wx ? n1.xb.v : n1.xa.v, P1.pool[0] + off2, P1.pool[2] + off2};
                for (int k = 0; k < 3; ++k) {
                    next[k] = nx0[k];
                    next[3 + k] = nx1[k];
                }
                extra[0] = n0.payload;
                extra[1] = n0.payload + L;
                extra[2] = n1.payload;
                extra[3] = n1.payload + L;
                eb = af.nx == 3 ? 32 : 40;
            } else if (af.nx == 4) {
                extra[0] = P0.outputs;
                extra[1] = P1.outputs;
                eb = 8;
            }
            lk(launch_beaver_combine2_add(S(r, 0), de, t0, t1, alpha, alpha_dev, z, s0.opened, s0.opened + L, af.sm,
                                          addin, wo, af.nx, next, extra, L, SMS(r, 0)),
               "k_combine2 + add");
            if (r->precomputed.size() != r->nodes.size()) r->precomputed.assign(r->nodes.size(), 0);
            r->precomputed[af.k1] = 1;
            if (af.k2 >= 0) r->premasked[af.k2] = 1;
            if (af.nx == 4) r->root_opened = true;
            // + both parties' add: o.v o.m read, w.v w.m written (32), then the mask or the opening
            tend(0, tk, SPDZ_KSTAT_COMBINE, (88 + 32 + eb) * L);
        } else if (id2 < 0 && root_fusable(id)) {  // the root open from the fresh products, in the same pass
            uint32_t* const outs[4] = {P0.outputs, P1.outputs, nullptr, nullptr};
            const uint32_t* const none[6] = {};
            lk(launch_beaver_combine2_mask(S(r, 0), de, t0, t1, alpha, alpha_dev, z, s0.opened, s0.opened + L, 3, none,
                                           outs, L, SMS(r, 0)),
               "k_combine2 + root open");
            r->root_opened = true;
            tend(0, tk, SPDZ_KSTAT_COMBINE, (88 + 8) * L);  // + both parties' opened outputs written
        } else if (id2 >= 0) {  // the next multiply's mask from the fresh products, in the same pass
            const uint64_t off2 = provisioned(r->scalar, (uint32_t)id2, 0).base;
            auto &n0 = P0.ns[id2], &n1 = P1.ns[id2];
            const bool zx = n0.xa.v == s0.out.v, zy = n0.xb.v == s0.out.v;
            const int zpos = zx && zy ? 2 : (zx ? 0 : 1);
            const uint32_t* next[6] = {zx ? n0.xb.v : n0.xa.v, P0.pool[0] + off2, P0.pool[2] + off2,
                                       zx ? n1.xb.v : n1.xa.v, P1.pool[0] + off2, P1.pool[2] + off2};
            uint32_t* const nde[4] = {n0.payload, n0.payload + L, n1.payload, n1.payload + L};
            lk(launch_beaver_combine2_mask(S(r, 0), de, t0, t1, alpha, alpha_dev, z, s0.opened, s0.opened + L, zpos,
                                           next, nde, L, SMS(r, 0)),
               "k_combine2 + next mask");
            r->premasked[id2] = 1;
            // + per party the next operand (unless both are this product), a'.v, b'.v read and d', e' written
            tend(0, tk, SPDZ_KSTAT_COMBINE, (88 + (zpos == 2 ? 32 : 40)) * L);
        } else {
            lk(launch_beaver_combine2(S(r, 0), de, t0, t1, alpha, alpha_dev, z, s0.opened, s0.opened + L, L,
                                      SMS(r, 0)),
               "k_combine2");
            // [d|e] of both parties 16 + two parties' triple planes 48 + two z 16 + one opened log 8
            tend(0, tk, SPDZ_KSTAT_COMBINE, 88 * L);
        }
        r->exchanged += 2 * (2 * L * 4);
    }

    void beaver(uint32_t id, const Region& reg, uint64_t exec) {
        const auto& n = r->node(id);
        const uint64_t L = n.lanes;
        const uint64_t off = reg.base + exec * reg.stride;  // runtime.cpp:197
        if (r->cfg) {  // control flow: this execution's record gets its own slot (opened values + MAC shares)
            for (int p = 0; p < r->n; ++p) {
                auto& P = r->parties[p];
                if (!P.local) continue;
                auto& st = P.ns[id];
                st.opened = st.opened_all + 2 * L * exec;
            }
        }
        bool pair = colocated2(r);
        for (auto& f : r->faults) pair = pair && f.node != id;
        if (pair) {
            beaver_pair(id, off);
            const uint64_t batch = make_batch(id, exec, 0);
            const uint64_t G = r->shard_total ? r->shard_total : L, so = r->shard_off;
            const auto& s0 = r->parties[0].ns[id];
            for (int p = 0; p < 2; ++p) {  // log_open (runtime.cpp:224); the opened values are public
                auto& P = r->parties[p];
                auto& st = P.ns[id];
                const uint32_t* mx = mac_slot(p, id, exec, 0);
                const uint32_t* my = mac_slot(p, id, exec, 1);
                P.maclog.push_back({s0.opened, mx, P.pool[1] + off, L, 0, batch, so, 2 * G});
                P.maclog.push_back({s0.opened + L, my, P.pool[3] + off, L, 0, batch, G + so, 2 * G});
            }
            return;
        }
        std::vector<cudaEvent_t> sent(r->n);
        if (r->premasked.size() != r->nodes.size()) r->premasked.assign(r->nodes.size(), 0);
        const bool masked = r->premasked[id];  // [d|e] written and published by the previous combine
        r->premasked[id] = 0;
        for (int p = 0; p < r->n; ++p) {
            if (!r->parties[p].local) continue;
            auto& P = r->parties[p];
            auto& st = P.ns[id];
            const Val &a = P.ns[n.operands[0]].out, &b = P.ns[n.operands[1]].out;
            dev(r, p);
            if (masked) {
                sent[p] = r->premask_ev[p];
                continue;
            }
            if (a.lanes != L) bcast_into(p, a, st.xa);
            if (b.lanes != L) bcast_into(p, b, st.xb);
            const int tk = tbegin(p);
            lk(launch_mul_mask(S(r, p), st.xa.v, st.xb.v, P.pool[0] + off, P.pool[2] + off, st.payload,
                               st.payload + L, L, SMS(r, p)),
               "k_mul_mask");
            tend(p, tk, SPDZ_KSTAT_MASK, 24 * L);
            sent[p] = publish(p, slot_of(id, 0));
            if (r->net) net_send(p, kMsgOpenShares, make_batch(id, exec, 0), st.payload, 2 * L);
        }
        const uint64_t batch = make_batch(id, exec, 0);
        const uint64_t G = r->shard_total ? r->shard_total : L, so = r->shard_off;
        const int id2 = fusable_next_mul(id);
        const AddFuse af = id2 < 0 ? fusable_next_add(id) : AddFuse{};
        if (r->premask_ev.size() != (size_t)r->n) r->premask_ev.assign(r->n, nullptr);
        for (int p = 0; p < r->n; ++p) {
            if (!r->parties[p].local) continue;
            auto& P = r->parties[p];
            auto& st = P.ns[id];
            dev(r, p);
            const uint32_t* pd[kMaxPeers];
            const uint32_t* pe[kMaxPeers];
            int k = 0;
            for (int q = 0; q < r->n; ++q) {
                if (q == p) continue;
                if (netpeer(q)) net_recv(p, q, kMsgOpenShares, batch, r->parties[q].ns[id].payload, 2 * L);
                else await(p, q, sent[q], slot_of(id, 0));
                const uint32_t* src = peer_payload(p, q, id, r->parties[q].ns[id].payload, 2 * L, st.shadow);
                pd[k] = src;
                pe[k] = src + L;
                ++k;
                r->exchanged += 2 * L * 4;
            }
            const uint32_t* tri[6];
            for (int t = 0; t < 6; ++t) tri[t] = P.pool[t] + off;
            const int tk = tbegin(p);
            if (af.k1 >= 0 && k == 1) {  // + the add / sub consuming the product (+ the next mask, published)
                const auto& an = r->node((uint32_t)af.k1);
                const bool zl = P.ns[an.operands[0]].out.v == st.out.v;
                const Val& o = P.ns[an.operands[zl ? 1 : 0]].out;
                Val& w = P.ns[af.k1].out;
                const uint32_t* addin[2] = {o.v, o.m};
                uint32_t* const wo[2] = {w.v, w.m};
                const uint32_t* next[3] = {nullptr, nullptr, nullptr};
                uint32_t* nde[2] = {nullptr, nullptr};
                const int nx = af.k2 >= 0 ? af.nx : 0;
                if (af.k2 >= 0) {
                    auto& nxs = P.ns[af.k2];
                    const uint64_t off2 = provisioned(r->scalar, (uint32_t)af.k2, 0).base;
                    next[0] = nx == 1 ? nxs.xb.v : nxs.xa.v;
                    next[1] = P.pool[0] + off2;
                    next[2] = P.pool[2] + off2;
                    nde[0] = nxs.payload;
                    nde[1] = nxs.payload + L;
                }
                lk(launch_beaver_combine_add(S(r, p), st.payload, st.payload + L, pd[0], pe[0], tri, P.ctx->party,
                                             P.ctx->alpha, st.out.v, st.out.m, st.opened, st.opened + L, af.sm, addin, wo,
                                             nx, next, nde, L, SMS(r, p), P.ctx->d_alpha),
                   "k_combine + add");
                tend(p, tk, SPDZ_KSTAT_COMBINE, (48 + 8ull * k + 16 + (nx == 0 ? 0 : nx == 3 ? 16 : 20)) * L);
                if (af.k2 >= 0) r->premask_ev[p] = publish(p, slot_of((uint32_t)af.k2, 0));
            } else if (id2 >= 0) {  // + the next multiply's mask from this party's fresh product; published at once
                auto& nx = P.ns[id2];
                const uint64_t off2 = provisioned(r->scalar, (uint32_t)id2, 0).base;
                const bool zx = nx.xa.v == st.out.v, zy = nx.xb.v == st.out.v;
                const int zpos = zx && zy ? 2 : (zx ? 0 : 1);
                const uint32_t* next[3] = {zx ? nx.xb.v : nx.xa.v, P.pool[0] + off2, P.pool[2] + off2};
                uint32_t* const nde[2] = {nx.payload, nx.payload + L};
                lk(launch_beaver_combine_mask(S(r, p), st.payload, st.payload + L, pd, pe, k, tri, P.ctx->party,
                                              P.ctx->alpha, st.out.v, st.out.m, st.opened, st.opened + L, zpos, next, nde,
                                              L, SMS(r, p), P.ctx->d_alpha),
                   "k_combine + next mask");
                tend(p, tk, SPDZ_KSTAT_COMBINE, (48 + 8ull * k + (zpos == 2 ? 16 : 20)) * L);
                r->premask_ev[p] = publish(p, slot_of((uint32_t)id2, 0));
            } else {
                lk(launch_beaver_combine(S(r, p), st.payload, st.payload + L, pd, pe, k, tri, P.ctx->party,
                                         P.ctx->alpha, st.out.v, st.out.m, st.opened, st.opened + L, L, SMS(r, p),
                                         P.ctx->d_alpha),
                   "k_combine");
                // own [d|e] 8 + peers 8k + triple planes 24 + z 8 + opened log 8 bytes per lane
                tend(p, tk, SPDZ_KSTAT_COMBINE, (48 + 8ull * k) * L);
            }
            // log_open (runtime.cpp:224): records [d | e] with mac shares [x.m - a.m | y.m - b.m]
            P.maclog.push_back({st.opened, mac_slot(p, id, exec, 0), P.pool[1] + off, L, 0, batch, so, 2 * G});
            P.maclog.push_back({st.opened + L, mac_slot(p, id, exec, 1), P.pool[3] + off, L, 0, batch, G + so, 2 * G});
        }
        if (id2 >= 0) r->premasked[id2] = 1;
        if (af.k1 >= 0) {
            if (r->precomputed.size() != r->nodes.size()) r->precomputed.assign(r->nodes.size(), 0);
            r->precomputed[af.k1] = 1;
            if (af.k2 >= 0) r->premasked[af.k2] = 1;
        }
    }

    // runtime.cpp:242-281
    void reduce_mul(uint32_t id, const Region& reg, uint64_t exec) {
        const auto& n = r->node(id);
        const size_t nlev = r->parties[r->ref_party()].ns[id].levels.size();
        if (nlev == 0) {  // single lane: value passes through
            for (int p = 0; p < r->n; ++p) {
            if (!r->parties[p].local) continue;
                auto& P = r->parties[p];
                const Val& a = P.ns[n.operands[0]].out;
                auto& o = P.ns[id].out;
                dev(r, p);
                lk(cudaMemcpyAsync(o.v, a.v, 4, cudaMemcpyDeviceToDevice, S(r, p)), "copy");
                lk(cudaMemcpyAsync(o.m, a.m, 4, cudaMemcpyDeviceToDevice, S(r, p)), "copy");
            }
            return;
        }
        uint64_t used = 0, sub = 1;
        if (r->cfg)  // this execution's MAC-log slots
            for (int p = 0; p < r->n; ++p) {
                if (!r->parties[p].local) continue;
                for (auto& lv : r->parties[p].ns[id].levels) {
                    lv.xm = lv.xm_all + lv.pairs * exec;
                    lv.ym = lv.ym_all + lv.pairs * exec;
                    lv.opened = lv.opened_all + 2 * lv.pairs * exec;
                }
            }
        for (size_t li = 0; li < nlev; ++li) {
            std::vector<cudaEvent_t> sent(r->n);
            const uint64_t off = reg.base + exec * reg.stride + used;
            const uint64_t pairs = r->parties[r->ref_party()].ns[id].levels[li].pairs;
            for (int p = 0; p < r->n; ++p) {
            if (!r->parties[p].local) continue;
                auto& P = r->parties[p];
                auto& lv = P.ns[id].levels[li];
                const uint32_t* cv = li == 0 ? P.ns[n.operands[0]].out.v : P.ns[id].levels[li - 1].zv;
                const uint32_t* cm = li == 0 ? P.ns[n.operands[0]].out.m : P.ns[id].levels[li - 1].zm;
                dev(r, p);
                lk(launch_pair_split(S(r, p), cv, cm, pairs, lv.xv, lv.xm, lv.yv, lv.ym, SMS(r, p)), "pair split");
                if (lv.in_lanes & 1) {  // odd element passes through (runtime.cpp:274-277)
                    lk(cudaMemcpyAsync(lv.zv + pairs, cv + lv.in_lanes - 1, 4, cudaMemcpyDeviceToDevice, S(r, p)), "odd");
                    lk(cudaMemcpyAsync(lv.zm + pairs, cm + lv.in_lanes - 1, 4, cudaMemcpyDeviceToDevice, S(r, p)), "odd");
                }
                lk(launch_mul_mask(S(r, p), lv.xv, lv.yv, P.pool[0] + off, P.pool[2] + off, lv.payload,
                                   lv.payload + pairs, pairs, SMS(r, p)),
                   "mask");
                sent[p] = publish(p, slot_of(id, 1 + (uint32_t)li));
                if (r->net) net_send(p, kMsgOpenShares, make_batch(id, exec, sub), lv.payload, 2 * pairs);
            }
            const uint64_t batch = make_batch(id, exec, sub++);
            for (int p = 0; p < r->n; ++p) {
            if (!r->parties[p].local) continue;
                auto& P = r->parties[p];
                auto& lv = P.ns[id].levels[li];
                dev(r, p);
                const uint32_t* pd[kMaxPeers];
                const uint32_t* pe[kMaxPeers];
                int k = 0;
                for (int q = 0; q < r->n; ++q) {
                    if (q == p) continue;
                    if (netpeer(q))
                        net_recv(p, q, kMsgOpenShares, batch, r->parties[q].ns[id].levels[li].payload, 2 * pairs);
                    else
                        await(p, q, sent[q], slot_of(id, 1 + (uint32_t)li));
                    pd[k] = r->parties[q].ns[id].levels[li].payload;
                    pe[k] = pd[k] + pairs;
                    ++k;
                    r->exchanged += 2 * pairs * 4;
                }
                const uint32_t* tri[6];
                for (int t = 0; t < 6; ++t) tri[t] = P.pool[t] + off;
                lk(launch_beaver_combine(S(r, p), lv.payload, lv.payload + pairs, pd, pe, k, tri, P.ctx->party,
                                         P.ctx->alpha, lv.zv, lv.zm, lv.opened, lv.opened + pairs, pairs, SMS(r, p),
                                         P.ctx->d_alpha),
                   "combine");
                P.maclog.push_back({lv.opened, lv.xm, P.pool[1] + off, pairs, 0, batch, 0, 0});
                P.maclog.push_back({lv.opened + pairs, lv.ym, P.pool[3] + off, pairs, 0, batch, pairs, 0});
            }
            used += pairs;
        }
    }

    // runtime.cpp:283-358
    void linear(uint32_t id, uint64_t exec) {
        const auto& n = r->node(id);
        const uint32_t din = n.din, dout = n.dout;
        const bool xp = !r->parties[r->ref_party()].ns[n.operands[0]].out.is_public;
        const bool wp = !r->parties[r->ref_party()].ns[n.operands[1]].out.is_public;
        if (!xp || !wp) {
            for (int p = 0; p < r->n; ++p) {
            if (!r->parties[p].local) continue;
                auto& P = r->parties[p];
                auto& st = P.ns[id];
                const Val &x = P.ns[n.operands[0]].out, &w = P.ns[n.operands[1]].out, &b = P.ns[n.operands[2]].out;
                spdz_ctx* c = P.ctx;
                dev(r, p);
                if (!xp && !wp) {  // public x public: y = W x, then exec_add(y, b)
                    lk(launch_modgemm(c->stream, 1, dout, din, 1, w.pub, w.pub, x.pub, nullptr, st.lin_tmp,
                                      st.lin_tmp + dout),
                       "modgemm");
                    if (b.is_public) {
                        lk(launch_pub_binop(c->stream, 0, st.lin_tmp, false, b.pub, b.lanes != dout, st.out.pub, dout,
                                            c->sms),
                           "bias");
                    } else if (b.lanes == dout) {  // exec_add(y public, b private) = add_public(b, y)
                        lk(launch_public(c->stream, 0, b.v, b.m, st.lin_tmp, false, 0u, false, c->party, c->alpha,
                                         st.out.v, st.out.m, dout, c->sms, c->d_alpha),
                           "bias pub");
                    } else {
                        lk(launch_bcast(c->stream, b.v, b.m, st.out.v, st.out.m, dout, c->sms), "bcast");
                        lk(launch_public(c->stream, 0, st.out.v, st.out.m, st.lin_tmp, false, 0u, false, c->party,
                                         c->alpha, st.out.v, st.out.m, dout, c->sms, c->d_alpha),
                           "bias pub");
                    }
                    continue;
                }
                uint32_t* yv = st.lin_tmp;
                uint32_t* ym = st.lin_tmp + dout;
                if (wp)  // x public, W secret: y.v = W.v x, y.m = W.m x
                    lk(launch_modgemm(c->stream, 1, dout, din, 1, w.v, w.m, x.pub, nullptr, yv, ym), "modgemm");
                else  // W public, x secret: y.v = W x.v, y.m = W x.m
                    lk(launch_modgemm(c->stream, 0, dout, din, 1, w.pub, nullptr, x.v, x.m, yv, ym), "modgemm");
                if (b.is_public)
                    lk(launch_public(c->stream, 0, yv, ym, b.pub, b.lanes != dout, 0u, false, c->party, c->alpha,
                                     st.out.v, st.out.m, dout, c->sms, c->d_alpha),
                       "bias pub");
                else if (b.lanes == dout)
                    lk(launch_add_sub(c->stream, false, yv, ym, b.v, b.m, st.out.v, st.out.m, dout, c->sms), "bias");
                else {
                    lk(launch_bcast(c->stream, b.v, b.m, st.out.v, st.out.m, dout, c->sms), "bcast");
                    lk(launch_add_sub(c->stream, false, yv, ym, st.out.v, st.out.m, st.out.v, st.out.m, dout, c->sms),
                       "bias");
                }
            }
            return;
        }
        // both private: matrix triples per tile (linear.cpp:75-130), all tiles batched per launch
        const auto& reg = r->matrix.at(id);
        const auto& lt = r->tiles.at(id);
        (void)reg;
        const uint64_t cells = (uint64_t)din * dout;
        const uint32_t ntiles = (uint32_t)lt.starts.size();
        const uint64_t etot = (uint64_t)din * ntiles;
        const uint64_t batch0 = make_batch(id, exec, 0);
        std::vector<cudaEvent_t> sent(r->n);
        for (int p = 0; p < r->n; ++p) {  // execution `exec`'s matrix triples (take_matrix_at, runtime.cpp:346-350)
            if (!r->parties[p].local) continue;
            auto& st = r->parties[p].ns[id];
            for (int q = 0; q < 2; ++q) {
                st.mA[q] = st.mA0[q] + exec * cells;
                st.mB[q] = st.mB0[q] + exec * etot;
                st.mC[q] = st.mC0[q] + exec * dout;
            }
            if (r->cfg) st.opened = st.opened_all + exec * (cells + etot);
        }
        // the W.m / x.m the records are checked against: the operands, or (control flow) a snapshot
        auto mac_planes = [&](int p) -> std::pair<const uint32_t*, const uint32_t*> {
            auto& P = r->parties[p];
            const Val &x = P.ns[n.operands[0]].out, &w = P.ns[n.operands[1]].out;
            if (!r->cfg) return {w.m, x.m};
            uint32_t* snap = P.ns[id].macsnap + exec * (cells + din);
            dev(r, p);
            lk(cudaMemcpyAsync(snap, w.m, cells * 4, cudaMemcpyDeviceToDevice, S(r, p)), "snapshot W.m");
            lk(cudaMemcpyAsync(snap + cells, x.m, din * 4ull, cudaMemcpyDeviceToDevice, S(r, p)), "snapshot x.m");
            return {snap, snap + cells};
        };
        bool fuse2 = colocated2(r);
        for (auto& f : r->faults) fuse2 = fuse2 && f.node != id;
        bool fuse2_masked = false;  // party 0's launch also wrote party 1's E
        for (int p = 0; p < r->n; ++p) {
            if (!r->parties[p].local) continue;
            auto& P = r->parties[p];
            auto& st = P.ns[id];
            const Val &x = P.ns[n.operands[0]].out, &w = P.ns[n.operands[1]].out, &b = P.ns[n.operands[2]].out;
            spdz_ctx* c = P.ctx;
            dev(r, p);
            // bias shares bs (runtime.cpp:344-345)
            if (b.is_public)
                lk(launch_public(c->stream, 4, nullptr, nullptr, b.pub, b.lanes != dout, 0u, false, c->party, c->alpha,
                                 st.bias_v, st.bias_m, dout, c->sms, c->d_alpha),
                   "share_of_public");
            else if (b.lanes == dout) {
                lk(cudaMemcpyAsync(st.bias_v, b.v, dout * 4ull, cudaMemcpyDeviceToDevice, c->stream), "copy");
                lk(cudaMemcpyAsync(st.bias_m, b.m, dout * 4ull, cudaMemcpyDeviceToDevice, c->stream), "copy");
            } else
                lk(launch_bcast(c->stream, b.v, b.m, st.bias_v, st.bias_m, dout, c->sms), "bcast");
            // mask_tile for every tile: [D (all rows) | E_t for every tile]
            const int tk = tbegin(p);
            bool e_done = false;
            if (!fuse2) {
                lk(launch_matrix_mask(c->stream, w.v, st.mA[0], cells, x.v, st.mB[0], 0, st.payload, c->sms), "mask D");
            } else if (p == 0) {  // both parties' [D | E_t...] in one pass
                auto& P1 = r->parties[1];
                const Val &w1 = P1.ns[n.operands[1]].out, &x1 = P1.ns[n.operands[0]].out;
                const LinMask2Args m{{w.v, w1.v}, {st.mA[0], P1.ns[id].mA[0]}, {x.v, x1.v},
                                     {st.mB[0], P1.ns[id].mB[0]}, {st.payload, P1.ns[id].payload}, cells, din, ntiles,
                                     st.opened + cells};
                const cudaError_t e = launch_linear_mask2(c->stream, m, c->sms);
                if (e == cudaSuccess) {
                    e_done = fuse2_masked = true;
                } else if (e == cudaErrorInvalidValue) {  // unaligned: D with mul_mask's d = x - a, e = y - b
                    lk(launch_mul_mask(c->stream, w.v, w1.v, st.mA[0], P1.ns[id].mA[0], st.payload,
                                       P1.ns[id].payload, cells, c->sms),
                       "mask D (both parties)");
                } else {
                    lk(e, "linear mask (both parties)");
                }
            } else {
                e_done = fuse2_masked;
            }
            if (!e_done)
                lk(launch_tile_e(c->stream, x.v, st.mB[0], din, ntiles, st.payload + cells, c->sms), "mask E");
            tend(p, tk, SPDZ_KSTAT_MASK,
                 (fuse2 ? (p == 0 ? 24 * cells : 0) : 12 * cells) + 12 * etot + (fuse2_masked && p == 0 ? 4 * etot : 0));
            sent[p] = publish(p, slot_of(id, 0));
            if (r->net) net_send_tiles(p, batch0, st.payload, din, lt);
        }
        if (fuse2) {  // both parties in one pass: [D|E] opened and logged once, per-party rows
            auto &P0 = r->parties[0], &P1 = r->parties[1];
            auto &s0 = P0.ns[id], &s1 = P1.ns[id];
            dev(r, 0);
            const int tk = tbegin(0);
            if (!fuse2_masked) {  // (the two-party mask kernel opened E in its own pass)
                const uint32_t* peE[1] = {s1.payload + cells};
                lk(launch_open_sum(S(r, 0), s0.payload + cells, peE, 1, s0.opened + cells, etot, SMS(r, 0)), "open E");
            }
            MC2Args a{};
            a.din = din;
            a.rows = dout;
            a.rpt = lt.rpt;
            a.D0 = s0.payload;
            a.D1 = s1.payload;
            for (int p = 0; p < 2; ++p) {
                auto& st = r->parties[p].ns[id];
                for (int q = 0; q < 2; ++q) {
                    a.A[p][q] = st.mA[q];
                    a.B[p][q] = st.mB[q];
                    a.Cc[p][q] = st.mC[q];
                }
                a.bias[p][0] = st.bias_v;
                a.bias[p][1] = st.bias_m;
                a.alpha[p] = r->parties[p].ctx->alpha;
                a.alpha_dev[p] = r->parties[p].ctx->d_alpha;  // graph replays follow a re-deal
                a.z[p][0] = st.out.v;
                a.z[p][1] = st.out.m;
            }
            a.opened = s0.opened;
            const bool opens_root = fusion_allowed() && root_opens(id, dout);  // the root open in the row finaliser
            if (opens_root) {
                a.open_out[0] = P0.outputs;
                a.open_out[1] = P1.outputs;
            }
            auto* acc_rows = reinterpret_cast<unsigned long long*>(s0.mc2_scratch);
            auto* done_rows = reinterpret_cast<unsigned int*>(s0.mc2_scratch + 10ull * dout);
            lk(launch_matrix_combine2(S(r, 0), a, SMS(r, 0), acc_rows, done_rows), "k_matrix_combine2");
            if (opens_root) r->root_opened = true;
            // D0 4 + D1 4 + two parties' A.v A.m 16 + opened D 4 per cell (B, E from cache)
            tend(0, tk, SPDZ_KSTAT_COMBINE, 28 * cells);
            r->exchanged += 2 * (cells + etot) * 4;
            for (int p = 0; p < 2; ++p) {
                auto& P = r->parties[p];
                const auto [wm, xm] = mac_planes(p);
                auto& st = P.ns[id];
                for (uint32_t t = 0; t < ntiles; ++t) {  // linear.cpp:113 log per tile: [D_t | E_t]
                    const uint64_t aoff = (uint64_t)lt.starts[t] * din, ct = (uint64_t)lt.counts[t] * din;
                    P.maclog.push_back({s0.opened + aoff, wm + aoff, st.mA[1] + aoff, ct, 0, batch0 + t, 0, 0});
                    P.maclog.push_back({s0.opened + cells + (uint64_t)t * din, xm, st.mB[1] + (uint64_t)t * din,
                                        din, 0, batch0 + t, ct, 0});
                }
            }
            return;
        }
        for (int p = 0; p < r->n; ++p) {
            if (!r->parties[p].local) continue;
            auto& P = r->parties[p];
            auto& st = P.ns[id];
            const Val &x = P.ns[n.operands[0]].out, &w = P.ns[n.operands[1]].out;
            spdz_ctx* c = P.ctx;
            dev(r, p);
            const uint32_t* peers[kMaxPeers];
            const uint32_t* peersE[kMaxPeers];
            int k = 0;
            for (int q = 0; q < r->n; ++q) {
                if (q == p) continue;
                if (netpeer(q)) net_recv_tiles(p, q, batch0, r->parties[q].ns[id].payload, din, lt);
                else await(p, q, sent[q], slot_of(id, 0));
                const uint32_t* src = peer_payload(p, q, id, r->parties[q].ns[id].payload, cells + etot, st.shadow);
                peers[k] = src;
                peersE[k] = src + cells;
                ++k;
                r->exchanged += (cells + etot) * 4;
            }
            const int tk = tbegin(p);
            lk(launch_open_sum(c->stream, st.payload + cells, peersE, k, st.opened + cells, etot, c->sms), "open E");
            const uint32_t* m6[6] = {st.mA[0], st.mA[1], st.mB[0], st.mB[1], st.mC[0], st.mC[1]};
            lk(launch_matrix_combine(c->stream, din, dout, lt.rpt, st.payload, peers, k, m6, st.bias_v, st.bias_m,
                                     c->party, c->alpha, st.out.v, st.out.m, st.opened, c->sms, c->d_alpha),
               "k_matrix_combine");
            // own D 4 + peer D 4k + A.v A.m 8 + opened D 4 per cell (B, E from cache)
            tend(p, tk, SPDZ_KSTAT_COMBINE, (16 + 4ull * k) * cells);
            const auto [wm, xm] = mac_planes(p);
            for (uint32_t t = 0; t < ntiles; ++t) {  // linear.cpp:113 log per tile: [D_t | E_t]
                const uint64_t aoff = (uint64_t)lt.starts[t] * din, ct = (uint64_t)lt.counts[t] * din;
                P.maclog.push_back({st.opened + aoff, wm + aoff, st.mA[1] + aoff, ct, 0, batch0 + t, 0, 0});
                P.maclog.push_back({st.opened + cells + (uint64_t)t * din, xm, st.mB[1] + (uint64_t)t * din, din, 0,
                                    batch0 + t, ct, 0});
            }
        }
    }

    void reduce_add(int p, uint32_t id) {
        auto& P = r->parties[p];
        const auto& n = r->node(id);
        const Val& a = P.ns[n.operands[0]].out;
        Val& o = P.ns[id].out;
        spdz_ctx* c = P.ctx;
        lk(cudaMemsetAsync(c->d_acc + 2, 0, 16, c->stream), "memset");
        if (a.is_public) {
            lk(launch_reduce_add(c->stream, a.pub, a.pub, a.lanes, c->d_acc + 2, c->sms), "reduce");
            lk(launch_finish_reduce(c->stream, c->d_acc + 2, o.pub, o.pub), "finish");
        } else {
            lk(launch_reduce_add(c->stream, a.v, a.m, a.lanes, c->d_acc + 2, c->sms), "reduce");
            lk(launch_finish_reduce(c->stream, c->d_acc + 2, o.v, o.m), "finish");
        }
    }

    void reduce_mul_public(int p, uint32_t id) {
        auto& P = r->parties[p];
        const auto& n = r->node(id);
        const Val& a = P.ns[n.operands[0]].out;
        auto& st = P.ns[id];
        spdz_ctx* c = P.ctx;
        uint64_t len = a.lanes;
        lk(cudaMemcpyAsync(st.opened, a.pub, len * 4, cudaMemcpyDeviceToDevice, c->stream), "copy");
        while (len > 1) {  // product is order-free: fold halves
            const uint64_t half = len / 2;
            lk(launch_pub_binop(c->stream, 2, st.opened, false, st.opened + (len - half), false, st.opened, half,
                                c->sms),
               "pub fold");
            len -= half;
        }
        lk(cudaMemcpyAsync(st.out.pub, st.opened, 4, cudaMemcpyDeviceToDevice, c->stream), "copy");
    }

    void run_nodes() {
        if (r->opts.node_streams > 1 && !r->net) return run_nodes_lanes();
        for (uint32_t id = 0; id < r->nodes.size(); ++id)
            if (r->live[id]) exec_node(id, 0);
    }

    // ---- node-level streams (opts.node_streams; scheduler.cpp:66-95 issues independent nodes
    // concurrently and completes openings by continuation, net.cpp:61-95) ----
    static bool launches_work(uint32_t kind) {
        return kind == SPDZ_NODE_ADD || kind == SPDZ_NODE_SUB || kind == SPDZ_NODE_MUL ||
               kind == SPDZ_NODE_REDUCE_ADD || kind == SPDZ_NODE_REDUCE_MUL || kind == SPDZ_NODE_LINEAR ||
               kind == SPDZ_NODE_CMP_PUBLIC;
    }
    // a compute node a value depends on (a static LOAD is a view of its base operand)
    int producer(uint32_t id) const {
        while (r->nodes[id].kind == SPDZ_NODE_LOAD && r->nodes[id].n_operands) id = r->nodes[id].operands[0];
        return launches_work(r->nodes[id].kind) ? (int)id : -1;
    }
    void plan_lanes() {
        const int K = r->opts.node_streams;
        const uint32_t N = (uint32_t)r->nodes.size();
        r->node_lane.assign(N, -1);
        std::vector<int> tail(K, -1);  // latest node of each stream
        int rr = 1;
        for (uint32_t id = 0; id < N; ++id) {
            const auto& n = r->nodes[id];
            if (!r->live[id] || !launches_work(n.kind)) continue;
            int lane = -1;
            if (n.kind == SPDZ_NODE_REDUCE_ADD || n.kind == SPDZ_NODE_REDUCE_MUL || n.kind == SPDZ_NODE_LINEAR) {
                lane = 0;  // ctx scratch (reduction accumulators) is shared: one stream
            } else {
                for (uint32_t k = 0; k < n.n_operands && lane < 0; ++k) {
                    const int o = producer(n.operands[k]);
                    if (o >= 0 && r->node_lane[o] >= 0 && tail[r->node_lane[o]] == o) lane = r->node_lane[o];
                }
                if (lane < 0) {  // a new chain: the next stream (0 is kept for the serial kinds)
                    lane = K > 1 ? rr : 0;
                    rr = rr + 1 < K ? rr + 1 : 1;
                }
            }
            r->node_lane[id] = lane;
            tail[lane] = (int)id;
        }
        r->node_ev.assign(r->n, std::vector<cudaEvent_t>(N, nullptr));
        for (int p = 0; p < r->n; ++p) {
            if (!r->parties[p].local) continue;
            dev(r, p);
            auto& v = r->lane_streams[r->devices[p]];
            while ((int)v.size() < K) {
                cudaStream_t st;
                cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "lane stream");
                v.push_back(st);
            }
            for (uint32_t id = 0; id < N; ++id)
                if (r->node_lane[id] >= 0)
                    cuda_check(cudaEventCreateWithFlags(&r->node_ev[p][id], cudaEventDisableTiming), "node event");
            if (!r->lane_fork[p]) cuda_check(cudaEventCreateWithFlags(&r->lane_fork[p], cudaEventDisableTiming), "fork");
        }
    }
    void run_nodes_lanes() {
        const int K = r->opts.node_streams;
        if (r->node_lane.size() != r->nodes.size()) plan_lanes();
        std::vector<cudaStream_t> main(r->n, nullptr);
        for (int p = 0; p < r->n; ++p) {  // fork: every stream starts after the main stream's work
            if (!r->parties[p].local) continue;
            dev(r, p);
            main[p] = S(r, p);
            lk(cudaEventRecord(r->lane_fork[p], main[p]), "fork");
            for (auto st : r->lane_streams[r->devices[p]]) lk(cudaStreamWaitEvent(st, r->lane_fork[p], 0), "fork wait");
        }
        for (uint32_t id = 0; id < r->nodes.size(); ++id) {
            if (!r->live[id]) continue;
            const int lane = r->node_lane[id];
            if (lane < 0) {
                exec_node(id, 0);
                continue;
            }
            const auto& n = r->nodes[id];
            for (int p = 0; p < r->n; ++p) {
                if (!r->parties[p].local) continue;
                dev(r, p);
                cudaStream_t st = r->lane_streams[r->devices[p]][lane];
                r->parties[p].ctx->stream = st;
                for (uint32_t k = 0; k < n.n_operands; ++k) {
                    const int o = producer(n.operands[k]);
                    if (o >= 0 && r->node_lane[o] != lane) lk(cudaStreamWaitEvent(st, r->node_ev[p][o], 0), "dep");
                }
            }
            try {
                exec_node(id, 0);
            } catch (...) {
                for (int p = 0; p < r->n; ++p)
                    if (main[p]) r->parties[p].ctx->stream = main[p];
                throw;
            }
            for (int p = 0; p < r->n; ++p) {
                if (!r->parties[p].local) continue;
                dev(r, p);
                lk(cudaEventRecord(r->node_ev[p][id], S(r, p)), "node done");
                r->parties[p].ctx->stream = main[p];
            }
        }
        for (int p = 0; p < r->n; ++p) {  // join: the root open and the MAC check follow every stream
            if (!r->parties[p].local) continue;
            dev(r, p);
            auto& v = r->lane_streams[r->devices[p]];
            for (int k = 0; k < K; ++k) {
                cudaEvent_t e = next_event(p);
                lk(cudaEventRecord(e, v[k]), "join");
                lk(cudaStreamWaitEvent(main[p], e, 0), "join wait");
            }
        }
    }

    // runtime.cpp:185-200: execution `exec` of a triple-consuming node must be provisioned
    const Region& provisioned(const std::map<uint32_t, Region>& regs, uint32_t id, uint64_t exec) {
        const Region& g = regs.at(id);
        if (exec >= g.max_execs)
            throw Error(SPDZ_ERR_TRIPLE_EXHAUSTED, "TripleExhausted: node " + std::to_string(id) + " executed " +
                                                       std::to_string(exec + 1) + " times, provisioned for " +
                                                       std::to_string(g.max_execs) +
                                                       " (raise --loop-iters at preprocessing)");
        return g;
    }

    // runtime.cpp:360-450, one execution of node `id`
    void exec_node(uint32_t id, uint64_t exec) {
        NvtxRange range(kind_label(r->nodes[id].kind), (long)id, (long)exec);
        if (r->cfg && exec_dynamic_public(id)) return;
        {
            const auto& n = r->nodes[id];
            switch (n.kind) {
                case SPDZ_NODE_INPUT:
                case SPDZ_NODE_CONST:
                case SPDZ_NODE_NOP:
                case SPDZ_NODE_LABEL:
                case SPDZ_NODE_PHI:     // resolved at block entry (run_cfg)
                case SPDZ_NODE_BRANCH:  // taken by run_cfg
                case SPDZ_NODE_ROOT:
                    break;
                case SPDZ_NODE_LOAD:
                    if (r->parties[r->ref_party()].ns[id].dyn_load) load_dynamic(id);
                    break;
                case SPDZ_NODE_ADD:
                case SPDZ_NODE_SUB:
                    if (id < r->precomputed.size() && r->precomputed[id]) {  // written by the previous combine
                        r->precomputed[id] = 0;
                        break;
                    }
                    if (add_pair(id, n.kind == SPDZ_NODE_SUB)) break;
                    for (int p = 0; p < r->n; ++p) {
                        if (!r->parties[p].local) continue;
                        dev(r, p);
                        add(p, id, n.kind == SPDZ_NODE_SUB);
                    }
                    break;
                case SPDZ_NODE_MUL: {
                    const bool a = r->parties[r->ref_party()].ns[n.operands[0]].out.is_public;
                    const bool b = r->parties[r->ref_party()].ns[n.operands[1]].out.is_public;
                    if (!a && !b) {
                        beaver(id, provisioned(r->scalar, id, exec), exec);
                        r->scalar_used += n.lanes;
                    }
                    else
                        for (int p = 0; p < r->n; ++p) {
            if (!r->parties[p].local) continue;
                            dev(r, p);
                            mul_local(p, id);
                        }
                    break;
                }
                case SPDZ_NODE_REDUCE_ADD:
                    for (int p = 0; p < r->n; ++p) {
                        if (!r->parties[p].local) continue;
                        dev(r, p);
                        reduce_add(p, id);
                    }
                    break;
                case SPDZ_NODE_CMP_PUBLIC:
                    for (int p = 0; p < r->n; ++p) {
                        if (!r->parties[p].local) continue;
                        dev(r, p);
                        auto& P = r->parties[p];
                        lk(launch_pub_binop(S(r, p), 3 + (int)n.const_val, P.ns[n.operands[0]].out.pub, true,
                                            P.ns[n.operands[1]].out.pub, true, P.ns[id].out.pub, 1, P.ctx->sms),
                           "cmp public");
                    }
                    break;
                case SPDZ_NODE_REDUCE_MUL:
                    if (r->parties[r->ref_party()].ns[n.operands[0]].out.is_public)
                        for (int p = 0; p < r->n; ++p) {
            if (!r->parties[p].local) continue;
                            dev(r, p);
                            reduce_mul_public(p, id);
                        }
                    else {
                        const Region& g = provisioned(r->scalar, id, exec);
                        reduce_mul(id, g, exec);
                        r->scalar_used += g.stride;
                    }
                    break;
                case SPDZ_NODE_LINEAR:
                    if (r->matrix.count(id)) r->matrix_used += provisioned(r->matrix, id, exec).stride;
                    linear(id, exec);
                    break;
                default:
                    throw Error(SPDZ_ERR_INVALID_ARGUMENT, "runtime: unexpected node kind");
            }
        }
    }

    // runtime.cpp:551-560 open the root (batch make_batch(root, 1, 1))
    void open_root() {
        NvtxRange range("open root");
        const Val& rv0 = r->parties[r->ref_party()].ns[r->root].out;
        const uint64_t L = rv0.lanes;
        // control flow: a private-typed root holding a public value is public at run time —
        // the reference returns it without an opening or a MAC record (runtime.cpp:553-555)
        const uint32_t src = r->nodes[r->root].n_operands ? r->nodes[r->root].operands[0] : r->root;
        if (r->cfg && !rv0.is_public && r->rt_pub[src]) {
            for (int p = 0; p < r->n; ++p) {
                if (!r->parties[p].local) continue;
                dev(r, p);
                lk(cudaMemcpyAsync(r->parties[p].outputs, pub_of(p, src), L * 4, cudaMemcpyDeviceToDevice, S(r, p)),
                   "copy out");
            }
            return;
        }
        if (rv0.is_public) {
            for (int p = 0; p < r->n; ++p) {
            if (!r->parties[p].local) continue;
                dev(r, p);
                lk(cudaMemcpyAsync(r->parties[p].outputs, r->parties[p].ns[r->root].out.pub, L * 4,
                                   cudaMemcpyDeviceToDevice, S(r, p)),
                   "copy out");
            }
            return;
        }
        const uint64_t batch = make_batch(r->root, 1, 1);
        bool pair = colocated2(r);
        for (auto& f : r->faults) pair = pair && f.node != r->root;
        if (pair) {  // both local parties' openings (identical words) in one pass
            auto &P0 = r->parties[0], &P1 = r->parties[1];
            dev(r, 0);
            if (r->root_opened) {  // already written by the root multiply's combine
                r->root_opened = false;
            } else {
                const int tk = tbegin(0);
                lk(launch_open_sum2(S(r, 0), P0.ns[r->root].out.v, P1.ns[r->root].out.v, P0.outputs, P1.outputs, L,
                                    SMS(r, 0)),
                   "open root (both parties)");
                tend(0, tk, SPDZ_KSTAT_OPEN, 16ull * L);
            }
            r->exchanged += 2 * L * 4;
            for (int p = 0; p < 2; ++p)
                r->parties[p].maclog.push_back({r->parties[p].outputs, r->parties[p].ns[r->root].out.m, nullptr, L, 0,
                                                batch, r->shard_off, r->shard_total ? r->shard_total : L});
            return;
        }
        std::vector<cudaEvent_t> ready(r->n);
        for (int p = 0; p < r->n; ++p) {
            if (!r->parties[p].local) continue;
            dev(r, p);
            ready[p] = publish(p, slot_of(r->root, 0));
            if (r->net) net_send(p, kMsgOpenShares, batch, r->parties[p].ns[r->root].out.v, L);
        }
        for (int p = 0; p < r->n; ++p) {
            if (!r->parties[p].local) continue;
            auto& P = r->parties[p];
            const Val& rv = P.ns[r->root].out;
            dev(r, p);
            const uint32_t* peers[kMaxPeers];
            int k = 0;
            for (int q = 0; q < r->n; ++q) {
                if (q == p) continue;
                if (netpeer(q)) net_recv(p, q, kMsgOpenShares, batch, r->parties[q].ns[r->root].out.v, L);
                else await(p, q, ready[q], slot_of(r->root, 0));
                peers[k++] = peer_payload(p, q, r->root, r->parties[q].ns[r->root].out.v, L, P.ns[r->root].shadow);
                r->exchanged += L * 4;
            }
            const int tk = tbegin(p);
            lk(launch_open_sum(S(r, p), rv.v, peers, k, P.outputs, L, SMS(r, p)), "open root");
            tend(p, tk, SPDZ_KSTAT_OPEN, (8ull + 4ull * k) * L);
            P.maclog.push_back({P.outputs, rv.m, nullptr, L, 0, batch, r->shard_off,
                                r->shard_total ? r->shard_total : L});
        }
    }
};

}  // namespace rt
}  // namespace spdzb200
