// Internal state of the n-party executor (run*.cu): the run, its parties' device
// buffers and the helpers shared by planning (run_plan.cu), node execution
// (run_exec.hpp) and the C ABI (run.cu).
#pragma once
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

namespace spdzb200 {
NetLink* net_link(spdz_net* net);  // net.cpp

namespace rt {
// NVTX ranges per executed node, root open and MAC check (SURVEY §5 tracing plan), on when
// SPDZ_NVTX=1 so that an nsys / ncu timeline names the online phase's steps
inline bool nvtx_on() {
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
inline const char* kind_label(int k) {
    static const char* names[] = {"input", "const", "add", "sub", "mul", "reduce_add", "reduce_mul", "linear",
                                  "root", "load", "nop", "cmp_public", "phi", "branch", "label"};
    return k >= 0 && k < (int)(sizeof names / sizeof names[0]) ? names[k] : "node";
}


inline uint64_t make_batch(uint64_t node, uint64_t exec, uint64_t sub) {  // runtime.cpp:22-24
    return (node << 32) | (exec << 12) | sub;
}

inline void lk(cudaError_t e, const char* what) { cuda_check(e, what); }

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
    uint32_t* mc2_scratch = nullptr; // co-located combine: 5 u64 sums + 1 u32 count per row (zeroed)
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
    cudaEvent_t t_open = nullptr;   // every opening of the phase complete (spdz_run_wait_openings)
};

struct DeviceDeal {                 // one dealer output per device (all parties' shares)
    uint32_t* pool[6] = {};
    uint32_t *mask_v = nullptr, *mask_m = nullptr, *mask_c = nullptr;
    std::map<uint32_t, std::array<uint32_t*, 6>> layer;  // linear node -> A.v A.m B.v B.m C.v C.m (party-major)
    uint32_t* scratch = nullptr;    // matrix dealer cleartext scratch
};

}  // namespace rt
}  // namespace spdzb200

using namespace spdzb200;
using namespace spdzb200::rt;

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
    std::vector<char> live;         // node's value reaches the root (or a branch): executed
    std::vector<char> premasked;    // co-located multiply whose [d|e] the previous combine already wrote
    bool root_opened = false;       // the root multiply's combine wrote the opened outputs
    std::vector<char> precomputed;  // co-located add / sub already written by the previous combine
    std::vector<cudaEvent_t> premask_ev;  // per party: the event that published a premasked [d|e]
    uint64_t scalar_live = 0, matrix_live = 0;  // triples the live nodes consume (straight-line)
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
    // profile_kernels inside the graph: the captured kernel-class event pairs (event-record nodes)
    bool kt_capturing = false;
    std::vector<KTimer::Rec> graph_kt_recs;
    size_t graph_kt_used = 0;
    // share_inputs: constants uploaded once, reduced public inputs kept alive for async copies
    bool consts_uploaded = false;
    std::map<uint32_t, std::vector<uint32_t>> pub_reduced;
    bool in_flight = false;
    bool any_remote = false;
    uint32_t seq = 0;               // phase sequence number written to / awaited on opening flags
    uint64_t n_slots = 0;
    uint64_t launches0 = 0;
    std::chrono::steady_clock::time_point wall0;
    // node-level streams (opts.node_streams > 1): stream index of every node (-1: launches
    // nothing), the streams per device, and per party one event per node (recorded after it)
    std::vector<int> node_lane;
    std::map<int, std::vector<cudaStream_t>> lane_streams;
    std::vector<std::vector<cudaEvent_t>> node_ev;
    cudaEvent_t lane_fork[SPDZ_MAX_PARTIES] = {};

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

namespace spdzb200 {
namespace rt {

// cuStreamWriteValue32 / cuStreamWaitValue32 through the runtime's driver entry points
typedef CUresult (*PFN_waitv32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_writev32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_addrrange)(CUdeviceptr*, size_t*, CUdeviceptr);
inline PFN_waitv32 g_waitv32 = nullptr;
inline PFN_writev32 g_writev32 = nullptr;
inline PFN_addrrange g_addrrange = nullptr;

inline void load_stream_memops() {
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

inline cudaStream_t S(spdz_run* r, int p) { return r->parties[p].ctx->stream; }
// both parties of a 2-party run on one stream: their passes may be fused (read shared data once)
inline bool colocated2(spdz_run* r) {
    return r->n == 2 && r->parties[0].local && r->parties[1].local && S(r, 0) == S(r, 1) &&
           !r->opts.separate_party_kernels;
}
inline int SMS(spdz_run* r, int p) { return r->parties[p].ctx->sms; }
inline void dev(spdz_run* r, int p) { device_guard(r->parties[p].ctx); }

// opening slot of (node, sub): sub 0 = the node's opening (Beaver / linear / root),
// 1..62 = reduce_mul level sub-1, 63 = input-sharing difference of an input node
inline uint64_t slot_of(uint32_t node, uint32_t sub) { return (uint64_t)node * 64 + sub; }

// After party p's payload for `slot` is complete on its stream, publish it to
// remote peers (stream-ordered write, with the default system-wide fence).
inline void signal_remote(spdz_run* r, int p, uint64_t slot) {
    if (!r->any_remote || r->opts.network) return;
    dev(r, p);
    need(g_writev32(S(r, p), (CUdeviceptr)(r->parties[p].flags + slot), r->seq, 0) == CUDA_SUCCESS, SPDZ_ERR_CUDA,
         "cuStreamWriteValue32");
}

// Party p's stream waits until remote party q has published `slot` for this phase.
inline void wait_remote(spdz_run* r, int p, int q, uint64_t slot) {
    dev(r, p);
    need(g_waitv32(S(r, p), (CUdeviceptr)(r->parties[q].flags + slot), r->seq, CU_STREAM_WAIT_VALUE_GEQ) ==
             CUDA_SUCCESS,
         SPDZ_ERR_CUDA, "cuStreamWaitValue32");
}

inline cudaEvent_t new_event(spdz_run* r, int p) {
    dev(r, p);
    cudaEvent_t e;
    cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    r->parties[p].evs.push_back(e);
    return e;
}

// planning and preprocessing (run_plan.cu)
void plan_layout(spdz_run* r);
void compute_liveness(spdz_run* r);
uint32_t const_of(spdz_run* r, uint32_t id);
void plan_buffers(spdz_run* r);
void deal(spdz_run* r, uint64_t seed);
void load_store(spdz_run* r, int p, const char* path);
void alloc_deals(spdz_run* r);
int ktimer_begin(spdz_run* r, int p);
void ktimer_end(spdz_run* r, int p, int idx, int cls, uint64_t bytes);

}  // namespace rt
}  // namespace spdzb200
