// Reference-side binding of the B200 executor: the reference's own in-memory
// circuit (`circuit::CircuitGraph`, circuit.hpp:34-90) and inputs run through
// the C ABI's spdz_run_* (include/spdz_b200.h) instead of PartyRuntime.
//
//   run_local_b200  replaces runtime::run_local (runtime.cpp:586-613): GPU
//                   dealer with the same seed and loop_iters hint;
//   run_files_b200  replaces every party's `llspdz run` (tools/main.cpp:111-130):
//                   party i's preprocessing from its MPCT store file;
//   run_one_party_b200  replaces one party's `llspdz run --party i --config ...`: a
//                   B200 party over the reference's TCP mesh among reference parties.
//
// A maintainer adds this file next to tools/main.cpp and routes `run --local`
// / `bench` to it (a `--backend b200` flag).  Reports carry the fields
// PartyRuntime fills; failures raise the reference's exception types.
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "mpc/circuit.hpp"
#include "mpc/linear.hpp"
#include "mpc/preproc.hpp"
#include "mpc/runtime.hpp"
#include "mpc/scheduler.hpp"
#include "mpc/spdz.hpp"
#include "mpc/triple_store.hpp"
#include "spdz_b200.h"

namespace mpc::runtime {

namespace {

bool starts(const std::string& s, const char* p) { return s.rfind(p, 0) == 0; }

[[noreturn]] void raise(int rc) {
    const std::string m = spdz_last_error();
    switch (rc) {
        case SPDZ_ERR_LANE_MISMATCH: throw backend::LaneMismatch(m);
        case SPDZ_ERR_TRIPLE_SHORTAGE: throw backend::TripleShortage(m);
        case SPDZ_ERR_BACKEND_UNAVAILABLE: throw backend::BackendUnavailable(m);
        case SPDZ_ERR_TRIPLE_EXHAUSTED: throw spdz::TripleExhausted(m);
        case SPDZ_ERR_TRIPLE_SHAPE_MISMATCH: throw spdz::TripleShapeMismatch(m);
        case SPDZ_ERR_MASK_EXHAUSTED: throw spdz::MaskExhausted(m);
        case SPDZ_ERR_MAC_CHECK_FAILED: throw spdz::MacCheckFailed(m);
        case SPDZ_ERR_SLICE_TOO_SMALL: throw linear::SliceTooSmall(m);
        case SPDZ_ERR_STORE_FORMAT: throw spdz::StoreFormatError(m);
        case SPDZ_ERR_INSUFFICIENT_TRIPLES: throw preproc::InsufficientTriples(m);
        default:
            if (starts(m, "SecretControlFlow")) throw sched::SecretControlFlow(m);
            if (starts(m, "UnknownPredecessor")) throw sched::UnknownPredecessor(m);
            if (starts(m, "ShapeMismatch")) throw preproc::ShapeMismatch(m);
            throw std::runtime_error(m);
    }
}

void ok(int rc) {
    if (rc != SPDZ_OK) raise(rc);
}

spdz_node_kind kind_of(circuit::NodeKind k) {
    using K = circuit::NodeKind;
    switch (k) {
        case K::Input: return SPDZ_NODE_INPUT;
        case K::Const: return SPDZ_NODE_CONST;
        case K::Adder:
        case K::AddBatch: return SPDZ_NODE_ADD;
        case K::Subtract:
        case K::SubBatch: return SPDZ_NODE_SUB;
        case K::Multiplier:
        case K::MultBatch: return SPDZ_NODE_MUL;
        case K::ReduceAdd: return SPDZ_NODE_REDUCE_ADD;
        case K::ReduceMul: return SPDZ_NODE_REDUCE_MUL;
        case K::Load: return SPDZ_NODE_LOAD;
        case K::LinearLayer: return SPDZ_NODE_LINEAR;
        case K::Phi: return SPDZ_NODE_PHI;
        case K::Branch: return SPDZ_NODE_BRANCH;
        case K::BlockLabel: return SPDZ_NODE_LABEL;
        case K::Root: return SPDZ_NODE_ROOT;
        case K::CmpPublic: return SPDZ_NODE_CMP_PUBLIC;
        default:
            throw std::runtime_error(std::string("runtime: unexpected node kind ") + circuit::kind_name(k));
    }
}

// The lowered graph: one spdz_node_t per circuit node, input lanes from the bound
// values when the descriptor's count is 0, vector constants as public inputs.
struct Lowered {
    std::vector<spdz_node_t> nodes;
    std::map<uint32_t, std::vector<uint32_t>> bind;  // input node -> cleartext
};

Lowered lower(const circuit::CircuitGraph& g, const preproc::Inputs& inputs) {
    Lowered L;
    std::map<circuit::NodeId, const circuit::InputDesc*> desc;
    for (auto& d : g.inputs) desc[d.node] = &d;
    L.nodes.resize(g.nodes.size());
    for (auto& n : g.nodes) {
        spdz_node_t& o = L.nodes[n.id];
        std::memset(&o, 0, sizeof(o));
        o.kind = kind_of(n.kind);
        o.is_private = n.is_private;
        o.lanes = n.lanes;
        if (n.operands.size() > (n.kind == circuit::NodeKind::Phi ? size_t(SPDZ_MAX_OPERANDS) : size_t(3)) ||
            n.successors.size() > 2)
            throw std::runtime_error("UnsupportedCircuit: node " + std::to_string(n.id) + " has too many edges");
        o.n_operands = (uint32_t)n.operands.size();
        for (size_t k = 0; k < n.operands.size(); ++k) o.operands[k] = n.operands[k];
        for (size_t k = 0; k < n.phi_labels.size() && k < SPDZ_MAX_OPERANDS; ++k) o.phi_labels[k] = n.phi_labels[k];
        o.n_succ = (uint32_t)n.successors.size();
        for (size_t k = 0; k < n.successors.size(); ++k) o.succ[k] = n.successors[k];
        o.din = n.din;
        o.dout = n.dout;
        o.next = n.next == circuit::kNoNode ? SPDZ_NO_NODE : n.next;
        o.loop_depth = n.block == circuit::kNoNode ? 0 : (uint32_t)g.loops_containing_block(n.block).size();
        if (n.kind == circuit::NodeKind::Input) {
            auto it = desc.find(n.id);
            if (it == desc.end()) throw std::runtime_error("runtime: input node without descriptor");
            const auto& d = *it->second;
            o.is_private = d.is_private;
            auto v = inputs.find(d.name);
            if (v == inputs.end())
                throw preproc::ShapeMismatch("ShapeMismatch: missing " + std::string(d.is_private ? "private" : "public") +
                                             " input '" + d.name + "'");
            if (d.count != 0 && v->second.size() != d.count)
                throw preproc::ShapeMismatch("ShapeMismatch: parameter '" + d.name + "' has " +
                                             std::to_string(v->second.size()) + " elements, circuit expects " +
                                             std::to_string(d.count));
            o.lanes = (uint32_t)v->second.size();
            L.bind[n.id] = v->second;
        } else if (n.kind == circuit::NodeKind::Const) {
            if (n.cvals.size() <= 1) {
                o.lanes = 1;
                o.const_val = n.cvals.empty() ? 0u : (uint32_t)(n.cvals[0] % kPrime);
            } else {  // runtime.cpp:527-532: one public value per lane
                o.kind = SPDZ_NODE_INPUT;
                o.is_private = 0;
                o.lanes = (uint32_t)n.cvals.size();
                auto& b = L.bind[n.id];
                for (uint64_t c : n.cvals) b.push_back((uint32_t)(c % kPrime));
            }
        } else if (n.kind == circuit::NodeKind::CmpPublic) {
            o.const_val = (uint32_t)n.pred;
        }
    }
    return L;
}

struct Run {
    spdz_run* h = nullptr;
    ~Run() {
        if (h) spdz_run_destroy(h);
    }
};

struct Mesh {
    spdz_net* h = nullptr;
    ~Mesh() {
        if (h) spdz_net_destroy(h);
    }
};

std::vector<RunReport> execute(const circuit::CircuitGraph& g, int n_parties, const preproc::Inputs& inputs,
                               const RunOptions& opts, uint64_t dealer_seed, uint64_t loop_iters,
                               const std::vector<std::string>* stores, int device, int single_party = -1,
                               spdz_net* mesh = nullptr) {
    auto t0 = std::chrono::steady_clock::now();
    Lowered L = lower(g, inputs);
    spdz_run_options_t o;
    std::memset(&o, 0, sizeof(o));
    o.slice = opts.slice;
    o.dealer_seed = dealer_seed;
    for (int p = 0; p < SPDZ_MAX_PARTIES; ++p) o.devices[p] = device;
    o.entry_label = g.entry_label == circuit::kNoNode ? 0 : g.entry_label;
    o.loop_iters = loop_iters;
    if (mesh) {  // one party; the others across the reference's TCP mesh
        o.single_party = single_party + 1;
        o.network = 1;
        o.external_mac_verify = 1;
    }
    Run r;
    ok(spdz_run_create(L.nodes.data(), (uint32_t)L.nodes.size(), g.root, n_parties, &o, &r.h));
    if (mesh) {
        ok(spdz_run_attach_net(r.h, mesh));
        ok(spdz_run_load_store(r.h, single_party, (*stores)[0].c_str()));
    } else if (stores) {
        for (int p = 0; p < n_parties; ++p) ok(spdz_run_load_store(r.h, p, (*stores)[p].c_str()));
    }
    for (auto& [node, vals] : L.bind) ok(spdz_run_bind_input(r.h, node, vals.data(), vals.size()));
    ok(spdz_run_share_inputs(r.h));
    auto t1 = std::chrono::steady_clock::now();
    spdz_run_report_t rep;
    ok(spdz_run_online(r.h, 0, &rep));
    RunReport out;
    uint64_t len = 0;
    ok(spdz_run_outputs(r.h, nullptr, 0, &len));
    out.outputs.resize(len);
    ok(spdz_run_outputs(r.h, out.outputs.data(), len, &len));
    out.output_digest = spdz_fnv1a64(out.outputs.data(), len * 4, 1469598103934665603ull);  // runtime.cpp:573-574
    out.setup_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
    out.online_ms = rep.online_ms;
    out.bytes_sent = out.bytes_received = rep.bytes_exchanged / (uint64_t)n_parties;  // payload words read by peers
    out.scalar_triples_consumed = rep.scalar_triples_consumed;
    out.matrix_triples_consumed = rep.matrix_triples_consumed;
    out.workers = 1;
    out.slice = opts.slice;
    out.parties = n_parties;
    return std::vector<RunReport>(n_parties, out);  // every party opens the same outputs
}

}  // namespace

std::vector<RunReport> run_local_b200(const circuit::CircuitGraph& g, int n_parties, const preproc::Inputs& inputs,
                                      RunOptions opts, uint64_t dealer_seed, uint64_t loop_iters_hint, int device) {
    return execute(g, n_parties, inputs, opts, dealer_seed, loop_iters_hint, nullptr, device);
}

std::vector<RunReport> run_files_b200(const circuit::CircuitGraph& g, const std::vector<std::string>& triples,
                                      const preproc::Inputs& inputs, RunOptions opts, int device) {
    if (triples.empty()) throw std::runtime_error("run_files_b200: no triple stores");
    spdz_store_info_t info;
    ok(spdz_store_inspect(triples[0].c_str(), &info));
    return execute(g, (int)triples.size(), inputs, opts, 1, info.loop_iters ? info.loop_iters : 64, &triples,
                   device);
}

// tools/main.cpp:111-130 run_one_party with a B200 party: this party's MPCT store, the
// reference's endpoints list (net::MeshConfig), the other parties reference processes or
// other B200 hosts.
RunReport run_one_party_b200(const circuit::CircuitGraph& g, const std::string& triples,
                             const preproc::Inputs& inputs, int party, const std::vector<std::string>& endpoints,
                             RunOptions opts, int device, uint64_t connect_timeout_ms, uint64_t io_timeout_ms) {
    spdz_store_info_t info;
    ok(spdz_store_inspect(triples.c_str(), &info));
    if (info.party != party)
        throw std::runtime_error("triple store belongs to party " + std::to_string(info.party) + ", --party says " +
                                 std::to_string(party));
    if (info.n_parties != endpoints.size())
        throw std::runtime_error("endpoints file names " + std::to_string(endpoints.size()) +
                                 " parties, store expects " + std::to_string(info.n_parties));
    std::vector<const char*> eps;
    for (auto& e : endpoints) eps.push_back(e.c_str());
    Mesh m;
    ok(spdz_net_connect(party, (int)eps.size(), eps.data(), connect_timeout_ms, io_timeout_ms, &m.h));
    const std::vector<std::string> mine{triples};
    return execute(g, (int)endpoints.size(), inputs, opts, 1, info.loop_iters ? info.loop_iters : 64, &mine, device,
                   party, m.h)[0];
}

}  // namespace mpc::runtime
