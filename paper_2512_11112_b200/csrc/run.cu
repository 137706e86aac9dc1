// Local n-party online phase over device-resident state: the batch executor
// that replaces PartyRuntime::Impl's node drivers (runtime.cpp:129-506) for
// straight-line circuits.  Parties are CUDA streams (optionally on distinct
// devices); the opening exchange is a peer-buffer read fused into the combine
// kernels, ordered by per-party events (the batch-id matching of
// net.cpp:61-95 becomes stream/event ordering).  Every share, triple pool,
// opened-value log and MAC record lives in HBM as structure-of-arrays.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <random>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "field.cuh"
#include "internal.hpp"
#include "net.hpp"
#include "store.hpp"

using namespace spdzb200;

namespace spdzb200 {
NetLink* net_link(spdz_net* net);  // net.cpp
}

namespace {
// NVTX ranges per executed node, root open and MAC check (SURVEY §5 tracing plan), on when
// SPDZ_NVTX=1 so that an nsys / ncu timeline names the online phase's steps
bool nvtx_on() {
    static const bool on = [] {
        const char* e = std::getenv("SPDZ_NVTX");
        return e && e[0] == '1';
    }();
    return on;
}
struct NvtxRange {
    bool active;
    NvtxRange(const char* what, long a = -1, long b = -1) : active(nvtx_on()) {
        if (!active) return;
        char msg[96];
        if (a < 0) std::snprintf(msg, sizeof msg, "%s", what);
        else if (b < 0) std::snprintf(msg, sizeof msg, "%s %ld", what, a);
        else std::snprintf(msg, sizeof msg, "%s node %ld exec %ld", what, a, b);
        nvtxRangePushA(msg);
    }
    ~NvtxRange() {
        if (active) nvtxRangePop();
    }
};
const char* kind_label(int k) {
    static const char* names[] = {"input", "const", "add", "sub", "mul", "reduce_add", "reduce_mul", "linear",
                                  "root", "load", "nop", "cmp_public", "phi", "branch", "label"};
    return k >= 0 && k < (int)(sizeof names / sizeof names[0]) ? names[k] : "node";
}
}  // namespace

namespace {

uint64_t make_batch(uint64_t node, uint64_t exec, uint64_t sub) {  // runtime.cpp:22-24
    return (node << 32) | (exec << 12) | sub;
}

void lk(cudaError_t e, const char* what) { cuda_check(e, what); }

// RtValue (runtime.cpp:28-34), device resident.
struct Val {
    bool is_public = true;
    uint32_t* pub = nullptr;
    uint32_t* v = nullptr;
    uint32_t* m = nullptr;
    uint64_t lanes = 0;
};

struct Region {  // preproc.hpp:44-53
    uint64_t base = 0, stride = 0, max_execs = 1;
    uint64_t gbase = 0;  // global triple index of the region's first local lane (sharding)
};

struct Fault {
    uint32_t node;
    int sender, receiver;
    uint64_t word;
    uint32_t bit;
};

struct RedLevel {
    uint64_t in_lanes = 0, pairs = 0;
    uint32_t *xv = nullptr, *xm = nullptr, *yv = nullptr, *ym = nullptr;
    uint32_t *payload = nullptr, *opened = nullptr, *shadow = nullptr;
    uint32_t *zv = nullptr, *zm = nullptr;  // pairs (+1 odd passthrough)
    uint64_t out_lanes = 0;
    // control flow: xm / ym / opened of every provisioned execution (the MAC log reads them all)
    uint32_t *xm_all = nullptr, *ym_all = nullptr, *opened_all = nullptr;
};

struct NodeState {                  // per party, per node
    Val out;
    // Beaver
    Val xa, xb;                     // operands after bcast_share
    uint32_t* payload = nullptr;    // [d|e] or [D|E] sent to peers
    uint32_t* opened = nullptr;     // opened values (MAC log)
    uint32_t* shadow = nullptr;     // tampered copy of a peer payload (fault injection)
    // reduce_mul
    std::vector<RedLevel> levels;
    // linear
    uint32_t *bias_v = nullptr, *bias_m = nullptr;
    uint32_t *mA[2] = {nullptr, nullptr}, *mB[2] = {nullptr, nullptr}, *mC[2] = {nullptr, nullptr};
    uint32_t *mA0[2] = {nullptr, nullptr}, *mB0[2] = {nullptr, nullptr}, *mC0[2] = {nullptr, nullptr};  // exec 0
    uint32_t* lin_tmp = nullptr;    // public x public scratch
    // control flow: a Beaver node's opened values and operand MAC shares, one slot per
    // execution (the MAC check reads every execution's record after the last one)
    uint32_t* opened_all = nullptr;
    uint32_t* macsnap = nullptr;
    bool dyn_load = false;          // LOAD whose start is computed at run time (own buffer)
    uint32_t* shadow_pub = nullptr; // control flow: the public value of a private-typed node holding one
};

struct LinTiles {
    std::vector<uint32_t> starts, counts;
    uint32_t rpt = 1;
};

struct Party {
    bool local = true;              // false: another process owns it (IPC-mapped peer)
    uint32_t* flags = nullptr;      // opening-slot sequence words (local: allocated, remote: mapped)
    std::vector<void*> mapped;      // IPC mappings to close
    spdz_ctx* ctx = nullptr;
    std::vector<NodeState> ns;
    uint32_t* pool[6] = {};         // scalar triples (views)
    uint32_t *mask_v = nullptr, *mask_m = nullptr, *mask_c = nullptr;
    uint32_t* outputs = nullptr;
    std::vector<spdz_mac_segment_t> maclog;
    std::vector<cudaEvent_t> evs;   // open-slot events
    cudaEvent_t t0 = nullptr, t1 = nullptr;
};

struct DeviceDeal {                 // one dealer output per device (all parties' shares)
    uint32_t* pool[6] = {};
    uint32_t *mask_v = nullptr, *mask_m = nullptr, *mask_c = nullptr;
    std::map<uint32_t, std::array<uint32_t*, 6>> layer;  // linear node -> A.v A.m B.v B.m C.v C.m (party-major)
    uint32_t* scratch = nullptr;    // matrix dealer cleartext scratch
};

}  // namespace

struct KTimer {  // CUDA-event timing of kernel classes (profile_kernels)
    struct Rec {
        int cls;
        int dev;
        cudaEvent_t a, b;
        uint64_t bytes;
    };
    std::vector<cudaEvent_t> pool;
    size_t used = 0;
    std::vector<Rec> recs;
    cudaEvent_t take(int dev) {
        if (used == pool.size()) {
            cudaEvent_t e;
            cuda_check(cudaSetDevice(dev), "dev");
            cuda_check(cudaEventCreate(&e), "event");
            pool.push_back(e);
        }
        return pool[used++];
    }
};

struct spdz_run {
    KTimer kt;
    std::vector<spdz_node_t> nodes;
    uint32_t root = 0;
    int n = 2;
    spdz_run_options_t opts{};
    std::vector<Party> parties;
    std::vector<int> devices;
    std::map<int, DeviceDeal> deals;
    std::map<uint32_t, Region> scalar, matrix;
    std::map<uint32_t, LinTiles> tiles;
    uint64_t scalar_total = 0, matrix_total = 0, mask_total = 0;
    std::vector<std::pair<uint32_t, uint32_t>> mshapes;  // (din, rows) per matrix triple (demand order)
    std::map<uint32_t, uint64_t> input_mask_off;          // private input node -> first mask (local)
    std::map<uint32_t, uint64_t> input_mask_gfirst;       // ... global index of that mask
    uint64_t scalar_total_global = 0, mask_total_global = 0;
    bool cfg = false;               // graph with PHI/BRANCH: block-by-block execution (run_cfg)
    NetLink* net = nullptr;         // peers across the reference's TCP mesh (spdz_run_attach_net)
    HostPinned net_stage;           // frame staging (D2H of own payloads, H2D of the peers')
    std::vector<uint32_t> net_host; // per-tile frame assembly
    uint64_t loop_iters = 64;       // triple provisioning of loop bodies (preproc.cpp:124-163)
    uint64_t scalar_used = 0, matrix_used = 0;  // consumed by the last phase (control flow)
    // control flow: a private-typed node whose current value is public (a private phi that took
    // a public incoming value, and the add/sub/mul results of such values), as the reference's
    // RtValue::is_public is decided at run time (runtime.cpp:28-34)
    std::vector<char> rt_pub;
    uint64_t shard_off = 0, shard_total = 0, shard_L = 0;  // shard_total == 0: unsharded
    std::map<uint32_t, std::vector<uint32_t>> inputs;     // cleartext (host)
    std::map<uint32_t, uint32_t*> input_dev;              // cleartext staged on party 0's device
    std::map<uint32_t, uint32_t*> input_diff;             // opened x - mask (party 0's device)
    std::vector<void*> allocs;                            // (device, ptr)
    std::vector<int> alloc_dev;
    std::vector<Fault> faults;
    bool consumed = false;
    bool masks_used = false;        // input masks consumed by share_inputs (take_masks cursor)
    uint64_t dealer_seed = 1;
    uint32_t* host_out = nullptr;   // pinned (internal) or user-bound output buffer
    uint64_t host_out_len = 0, host_out_cap = 0;
    bool host_out_owned = false;
    bool host_out_registered = false;  // caller's pageable buffer page-locked by bind_output
    uint64_t exchanged = 0;
    cudaEvent_t ev_input = nullptr;
    cudaEvent_t ev_opened = nullptr;
    cudaStream_t copy_stream = nullptr;
    // optional caller-owned copy streams shared by several runs (StreamedRun): H2D of the
    // inputs in issue order on one stream, so chunk c's inputs land before chunk c+1's
    cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
    cudaEvent_t ev_h2d = nullptr, ev_out = nullptr;
    bool mac_launched = false;      // spdz_run_mac_check_launch issued the sigma kernels
    uint64_t mac_coin = 0;
    // CUDA graph of the online phase (opts.use_graph): captured on the first phase, replayed
    // after; the host-side products of node execution are saved with it
    cudaGraphExec_t online_graph = nullptr;
    std::vector<std::vector<spdz_mac_segment_t>> graph_maclog;
    uint64_t graph_exchanged = 0, graph_launches = 0;
    // share_inputs: constants uploaded once, reduced public inputs kept alive for async copies
    bool consts_uploaded = false;
    std::map<uint32_t, std::vector<uint32_t>> pub_reduced;
    bool in_flight = false;
    bool any_remote = false;
    uint32_t seq = 0;               // phase sequence number written to / awaited on opening flags
    uint64_t n_slots = 0;
    uint64_t launches0 = 0;
    std::chrono::steady_clock::time_point wall0;

    uint32_t* alloc(int party, uint64_t words) {
        // remote party: pointers come from spdz_run_import, or (network peers) local mirrors
        if (!parties[party].local && !opts.network) return nullptr;
        const int dev = devices[party];
        cuda_check(cudaSetDevice(dev), "cudaSetDevice");
        void* p = nullptr;
        cuda_check(cudaMalloc(&p, std::max<uint64_t>(words, 1) * 4), "cudaMalloc(run)");
        allocs.push_back(p);
        alloc_dev.push_back(dev);
        return (uint32_t*)p;
    }
    uint32_t* alloc_dev_words(int dev, uint64_t words) {
        cuda_check(cudaSetDevice(dev), "cudaSetDevice");
        void* p = nullptr;
        cuda_check(cudaMalloc(&p, std::max<uint64_t>(words, 1) * 4), "cudaMalloc(deal)");
        allocs.push_back(p);
        alloc_dev.push_back(dev);
        return (uint32_t*)p;
    }
    const spdz_node_t& node(uint32_t id) const { return nodes.at(id); }
    int ref_party() const {  // a party whose state is materialised here
        for (int p = 0; p < n; ++p)
            if (parties[p].local) return p;
        return 0;
    }
    bool priv(uint32_t id) const { return nodes.at(id).is_private != 0; }
};

namespace {

// cuStreamWriteValue32 / cuStreamWaitValue32 through the runtime's driver entry points
typedef CUresult (*PFN_waitv32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_writev32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_addrrange)(CUdeviceptr*, size_t*, CUdeviceptr);
PFN_waitv32 g_waitv32 = nullptr;
PFN_writev32 g_writev32 = nullptr;
PFN_addrrange g_addrrange = nullptr;

void load_stream_memops() {
    if (g_waitv32 && g_writev32) return;
    cudaDriverEntryPointQueryResult q;
    cuda_check(cudaGetDriverEntryPoint("cuStreamWaitValue32", (void**)&g_waitv32, cudaEnableDefault, &q),
               "entry point cuStreamWaitValue32");
    need(q == cudaDriverEntryPointSuccess && g_waitv32, SPDZ_ERR_CUDA, "cuStreamWaitValue32 unavailable");
    cuda_check(cudaGetDriverEntryPoint("cuStreamWriteValue32", (void**)&g_writev32, cudaEnableDefault, &q),
               "entry point cuStreamWriteValue32");
    need(q == cudaDriverEntryPointSuccess && g_writev32, SPDZ_ERR_CUDA, "cuStreamWriteValue32 unavailable");
    cuda_check(cudaGetDriverEntryPoint("cuMemGetAddressRange", (void**)&g_addrrange, cudaEnableDefault, &q),
               "entry point cuMemGetAddressRange");
    need(q == cudaDriverEntryPointSuccess && g_addrrange, SPDZ_ERR_CUDA, "cuMemGetAddressRange unavailable");
}

cudaStream_t S(spdz_run* r, int p) { return r->parties[p].ctx->stream; }
int SMS(spdz_run* r, int p) { return r->parties[p].ctx->sms; }
void dev(spdz_run* r, int p) { device_guard(r->parties[p].ctx); }

// opening slot of (node, sub): sub 0 = the node's opening (Beaver / linear / root),
// 1..62 = reduce_mul level sub-1, 63 = input-sharing difference of an input node
uint64_t slot_of(uint32_t node, uint32_t sub) { return (uint64_t)node * 64 + sub; }

// After party p's payload for `slot` is complete on its stream, publish it to
// remote peers (stream-ordered write, with the default system-wide fence).
void signal_remote(spdz_run* r, int p, uint64_t slot) {
    if (!r->any_remote || r->opts.network) return;
    dev(r, p);
    need(g_writev32(S(r, p), (CUdeviceptr)(r->parties[p].flags + slot), r->seq, 0) == CUDA_SUCCESS, SPDZ_ERR_CUDA,
         "cuStreamWriteValue32");
}

// Party p's stream waits until remote party q has published `slot` for this phase.
void wait_remote(spdz_run* r, int p, int q, uint64_t slot) {
    dev(r, p);
    need(g_waitv32(S(r, p), (CUdeviceptr)(r->parties[q].flags + slot), r->seq, CU_STREAM_WAIT_VALUE_GEQ) ==
             CUDA_SUCCESS,
         SPDZ_ERR_CUDA, "cuStreamWaitValue32");
}

cudaEvent_t new_event(spdz_run* r, int p) {
    dev(r, p);
    cudaEvent_t e;
    cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    r->parties[p].evs.push_back(e);
    return e;
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
                        pub_out(n.dout);
                        st.lin_tmp = r->alloc(p, n.dout);
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
    lk(cudaEventRecord(a, S(r, p)), "record");
    r->kt.recs.push_back({-1, r->devices[p], a, nullptr, 0});
    return (int)r->kt.recs.size() - 1;
}
void ktimer_end(spdz_run* r, int p, int idx, int cls, uint64_t bytes) {
    if (idx < 0) return;
    cudaEvent_t b = r->kt.take(r->devices[p]);
    lk(cudaEventRecord(b, S(r, p)), "record");
    auto& rec = r->kt.recs[idx];
    rec.cls = cls;
    rec.b = b;
    rec.bytes = bytes;
}

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
            for (auto [phi, chosen] : phis) phi_copy(phi, chosen);
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
                exec_node(u, execs[u]++);
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
    void beaver_pair(uint32_t id, uint64_t off) {
        const auto& n = r->node(id);
        const uint64_t L = n.lanes;
        auto &P0 = r->parties[0], &P1 = r->parties[1];
        auto &s0 = P0.ns[id], &s1 = P1.ns[id];
        dev(r, 0);
        for (int p = 0; p < 2; ++p) {
            auto& P = r->parties[p];
            auto& st = P.ns[id];
            const Val &a = P.ns[n.operands[0]].out, &b = P.ns[n.operands[1]].out;
            if (a.lanes != L) bcast_into(p, a, st.xa);
            if (b.lanes != L) bcast_into(p, b, st.xb);
        }
        const uint32_t alpha[2] = {P0.ctx->alpha, P1.ctx->alpha};
        const uint32_t* alpha_dev[2] = {P0.ctx->d_alpha, P1.ctx->d_alpha};
        for (int p = 0; p < 2; ++p) {
            auto& P = r->parties[p];
            auto& st = P.ns[id];
            const int tk = tbegin(p);
            lk(launch_mul_mask(S(r, p), st.xa.v, st.xb.v, P.pool[0] + off, P.pool[2] + off, st.payload,
                               st.payload + L, L, SMS(r, p)),
               "k_mul_mask");
            tend(p, tk, SPDZ_KSTAT_MASK, 24 * L);
        }
        const uint32_t* de[4] = {s0.payload, s0.payload + L, s1.payload, s1.payload + L};
        const uint32_t *t0[6], *t1[6];
        for (int t = 0; t < 6; ++t) {
            t0[t] = P0.pool[t] + off;
            t1[t] = P1.pool[t] + off;
        }
        uint32_t* z[4] = {s0.out.v, s0.out.m, s1.out.v, s1.out.m};
        const int tk = tbegin(0);
        lk(launch_beaver_combine2(S(r, 0), de, t0, t1, alpha, alpha_dev, z, s0.opened, s0.opened + L, L, SMS(r, 0)),
           "k_combine2");
        // [d|e] of both parties 16 + two parties' triple planes 48 + two z 16 + one opened log 8
        tend(0, tk, SPDZ_KSTAT_COMBINE, 88 * L);
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
        bool pair = r->n == 2 && r->parties[0].local && r->parties[1].local && S(r, 0) == S(r, 1);
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
        for (int p = 0; p < r->n; ++p) {
            if (!r->parties[p].local) continue;
            auto& P = r->parties[p];
            auto& st = P.ns[id];
            const Val &a = P.ns[n.operands[0]].out, &b = P.ns[n.operands[1]].out;
            dev(r, p);
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
            lk(launch_beaver_combine(S(r, p), st.payload, st.payload + L, pd, pe, k, tri, P.ctx->party, P.ctx->alpha,
                                     st.out.v, st.out.m, st.opened, st.opened + L, L, SMS(r, p), P.ctx->d_alpha),
               "k_combine");
            // own [d|e] 8 + peers 8k + triple planes 24 + z 8 + opened log 8 bytes per lane
            tend(p, tk, SPDZ_KSTAT_COMBINE, (48 + 8ull * k) * L);
            // log_open (runtime.cpp:224): records [d | e] with mac shares [x.m - a.m | y.m - b.m]
            P.maclog.push_back({st.opened, mac_slot(p, id, exec, 0), P.pool[1] + off, L, 0, batch, so, 2 * G});
            P.maclog.push_back({st.opened + L, mac_slot(p, id, exec, 1), P.pool[3] + off, L, 0, batch, G + so, 2 * G});
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
                                      st.out.pub),
                       "modgemm");
                    lk(launch_pub_binop(c->stream, 0, st.lin_tmp, false, b.pub, b.lanes != dout, st.out.pub, dout,
                                        c->sms),
                       "bias");
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
                                     st.out.v, st.out.m, dout, c->sms),
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
                                 st.bias_v, st.bias_m, dout, c->sms),
                   "share_of_public");
            else if (b.lanes == dout) {
                lk(cudaMemcpyAsync(st.bias_v, b.v, dout * 4ull, cudaMemcpyDeviceToDevice, c->stream), "copy");
                lk(cudaMemcpyAsync(st.bias_m, b.m, dout * 4ull, cudaMemcpyDeviceToDevice, c->stream), "copy");
            } else
                lk(launch_bcast(c->stream, b.v, b.m, st.bias_v, st.bias_m, dout, c->sms), "bcast");
            // mask_tile for every tile: [D (all rows) | E_t for every tile]
            const int tk = tbegin(p);
            lk(launch_matrix_mask(c->stream, w.v, st.mA[0], cells, x.v, st.mB[0], 0, st.payload, c->sms), "mask D");
            lk(launch_tile_e(c->stream, x.v, st.mB[0], din, ntiles, st.payload + cells, c->sms), "mask E");
            tend(p, tk, SPDZ_KSTAT_MASK, 12 * cells + 12 * etot);
            sent[p] = publish(p, slot_of(id, 0));
            if (r->net) net_send_tiles(p, batch0, st.payload, din, lt);
        }
        bool fuse2 = r->n == 2 && r->parties[0].local && r->parties[1].local && S(r, 0) == S(r, 1);
        for (auto& f : r->faults) fuse2 = fuse2 && f.node != id;
        if (fuse2) {  // both parties in one pass: [D|E] opened and logged once, per-party rows
            auto &P0 = r->parties[0], &P1 = r->parties[1];
            auto &s0 = P0.ns[id], &s1 = P1.ns[id];
            dev(r, 0);
            const int tk = tbegin(0);
            const uint32_t* peE[1] = {s1.payload + cells};
            lk(launch_open_sum(S(r, 0), s0.payload + cells, peE, 1, s0.opened + cells, etot, SMS(r, 0)), "open E");
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
                a.z[p][0] = st.out.v;
                a.z[p][1] = st.out.m;
            }
            a.opened = s0.opened;
            lk(launch_matrix_combine2(S(r, 0), a, SMS(r, 0)), "k_matrix_combine2");
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
                                     c->party, c->alpha, st.out.v, st.out.m, st.opened, c->sms),
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
        for (uint32_t id = 0; id < r->nodes.size(); ++id) exec_node(id, 0);
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
        std::vector<cudaEvent_t> ready(r->n);
        const uint64_t batch = make_batch(r->root, 1, 1);
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
    if (r->n != 2 || !r->parties[0].local || !r->parties[1].local || S(r, 0) != S(r, 1)) return false;
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
    return r->n == 2 && r->parties[0].local && r->parties[1].local && S(r, 0) == S(r, 1);
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
    if (!r->opts.use_graph || r->cfg || r->any_remote || r->opts.profile_kernels || !r->faults.empty()) return false;
    for (int p = 0; p < r->n; ++p)
        if (!r->parties[p].local || S(r, p) != S(r, 0)) return false;
    for (const auto& n : r->nodes)
        if (n.kind == SPDZ_NODE_LINEAR || n.kind == SPDZ_NODE_REDUCE_ADD || n.kind == SPDZ_NODE_REDUCE_MUL) return false;
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
        if (r->h2d_stream) {
            lk(cudaMemcpyAsync(d, host_vals, len * 4, cudaMemcpyHostToDevice, r->h2d_stream), "H2D input");
            lk(cudaEventRecord(r->ev_h2d, r->h2d_stream), "record h2d");
            lk(cudaStreamWaitEvent(P0.ctx->stream, r->ev_h2d, 0), "wait h2d");
        } else {
            lk(cudaMemcpyAsync(d, host_vals, len * 4, cudaMemcpyHostToDevice, P0.ctx->stream), "H2D input");
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
        need(!r->any_remote || r->opts.external_mac_verify, SPDZ_ERR_INVALID_ARGUMENT,
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
        if (graphable(r)) {
            cudaStream_t s = S(r, 0);
            dev(r, 0);
            if (!r->online_graph) {  // capture once: the same kernels, pointers and events every phase
                const uint64_t l0 = g_kernel_launches;
                cuda_check(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed), "begin capture");
                cudaGraph_t g = nullptr;
                try {
                    Exec ex{r};
                    ex.run_nodes();
                    ex.open_root();
                } catch (...) {
                    cudaStreamEndCapture(s, &g);
                    if (g) cudaGraphDestroy(g);
                    throw;
                }
                cuda_check(cudaStreamEndCapture(s, &g), "end capture");
                cudaError_t e = cudaGraphInstantiate(&r->online_graph, g, 0);
                cudaGraphDestroy(g);
                cuda_check(e, "cudaGraphInstantiate");
                r->graph_launches = g_kernel_launches - l0;
                r->graph_exchanged = r->exchanged;
                r->graph_maclog.clear();
                for (auto& P : r->parties) r->graph_maclog.push_back(P.maclog);
            } else {
                g_kernel_launches += r->graph_launches;
                r->exchanged = r->graph_exchanged;
                for (int p = 0; p < r->n; ++p) r->parties[p].maclog = r->graph_maclog[p];
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
            rep->scalar_triples_consumed = r->cfg ? r->scalar_used : r->scalar_total;
            rep->matrix_triples_consumed = r->cfg ? r->matrix_used : r->matrix_total;
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
            std::memcpy(host_out, r->host_out, std::min<uint64_t>(cap, r->host_out_len) * 4);
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
