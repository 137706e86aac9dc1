// Runtime drop-in check: the reference's own circuit/input/store readers feed
// both the unmodified reference runtime (PartyRuntime over the simulated
// transport, every party's `llspdz run`) and the B200 executor
// (b200_runtime.cpp: run_files_b200), then runtime::run_local vs
// run_local_b200 with the GPU dealer.  Outputs, digests and triple counts must
// match exactly.  Usage: check_runtime <tests/golden/bundles>.  Exit 0 = PASS.
#include <cstdio>
#include <exception>
#include <filesystem>
#include <fstream>
#include <iterator>
#include <string>
#include <thread>
#include <vector>

#include "mpc/circuit_io.hpp"
#include "mpc/net.hpp"
#include "mpc/preproc.hpp"
#include "mpc/runtime.hpp"
#include "mpc/scheduler.hpp"
#include "mpc/triple_store.hpp"

namespace mpc::runtime {
RunReport run_one_party_b200(const circuit::CircuitGraph& g, const std::string& triples,
                             const preproc::Inputs& inputs, int party, const std::vector<std::string>& endpoints,
                             RunOptions opts, int device, uint64_t connect_timeout_ms, uint64_t io_timeout_ms);
std::vector<RunReport> run_local_b200(const circuit::CircuitGraph& g, int n_parties, const preproc::Inputs& inputs,
                                      RunOptions opts, uint64_t dealer_seed, uint64_t loop_iters_hint, int device);
std::vector<RunReport> run_files_b200(const circuit::CircuitGraph& g, const std::vector<std::string>& triples,
                                      const preproc::Inputs& inputs, RunOptions opts, int device);
}  // namespace mpc::runtime

using namespace mpc;
namespace fs = std::filesystem;

static int failures = 0;

// `"key": <integer>` from a bundle's expected.json (flat numbers only)
static uint64_t json_number(const fs::path& path, const std::string& key, uint64_t fallback) {
    std::ifstream is(path);
    const std::string text((std::istreambuf_iterator<char>(is)), std::istreambuf_iterator<char>());
    const auto at = text.find("\"" + key + "\":");
    return at == std::string::npos ? fallback : std::stoull(text.substr(at + key.size() + 3));
}

static runtime::RunReport reference_files(const circuit::CircuitGraph& g, const std::vector<std::string>& triples,
                                          const preproc::Inputs& in, runtime::RunOptions opts) {
    const int n = (int)triples.size();
    auto sessions = net::make_sim_sessions(n);
    std::vector<runtime::RunReport> reps(n);
    std::vector<std::exception_ptr> errs(n);
    std::vector<std::thread> th;
    for (int i = 0; i < n; ++i)
        th.emplace_back([&, i] {
            try {
                runtime::PartyRuntime rt(g, spdz::read_store_file(triples[i]), sessions[i], opts);
                reps[i] = rt.run(in);
            } catch (...) {
                errs[i] = std::current_exception();
            }
        });
    for (auto& t : th) t.join();
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
    return reps[0];
}

static void compare(const std::string& what, const runtime::RunReport& ref, const runtime::RunReport& gpu) {
    const bool same = ref.outputs == gpu.outputs && ref.output_digest == gpu.output_digest &&
                      ref.scalar_triples_consumed == gpu.scalar_triples_consumed &&
                      ref.matrix_triples_consumed == gpu.matrix_triples_consumed;
    std::printf("%-40s %s  outputs=%zu digest=%016llx triples=%zu/%zu\n", what.c_str(), same ? "ok  " : "FAIL",
                gpu.outputs.size(), (unsigned long long)gpu.output_digest, gpu.scalar_triples_consumed,
                gpu.matrix_triples_consumed);
    if (!same) {
        std::printf("    reference digest=%016llx triples=%zu/%zu\n", (unsigned long long)ref.output_digest,
                    ref.scalar_triples_consumed, ref.matrix_triples_consumed);
        ++failures;
    }
}

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: check_runtime <bundles dir>\n");
        return 2;
    }
    std::vector<fs::path> dirs;
    for (auto& e : fs::directory_iterator(argv[1]))
        if (e.is_directory() && fs::exists(e.path() / "circuit.mpcg")) dirs.push_back(e.path());
    std::sort(dirs.begin(), dirs.end());
    for (auto& d : dirs) {
        const std::string name = d.filename().string();
        auto g = circuit::read_circuit_file((d / "circuit.mpcg").string());
        auto in = preproc::read_input_file((d / "inputs.mpci").string());
        std::vector<std::string> triples;
        for (int i = 0; fs::exists(d / ("triples_" + std::to_string(i) + ".bin")); ++i)
            triples.push_back((d / ("triples_" + std::to_string(i) + ".bin")).string());
        runtime::RunOptions opts;
        opts.slice = json_number(d / "expected.json", "slice", 262140);  // the slice the stores were dealt for
        try {
            compare(name + " (store files)", reference_files(g, triples, in, opts),
                    runtime::run_files_b200(g, triples, in, opts, 0)[0]);
            compare(name + " (run_local, dealer)", runtime::run_local(g, (int)triples.size(), in, opts, 3)[0],
                    runtime::run_local_b200(g, (int)triples.size(), in, opts, 3, 64, 0)[0]);
        } catch (const std::exception& e) {
            std::printf("%-40s FAIL  %s\n", name.c_str(), e.what());
            ++failures;
        }
    }
    // one B200 party among reference parties over the TCP mesh (`llspdz run --party`)
    for (const char* name : {"mixed_1024_n3", "nested_loop", "linear_64x32"}) {
        const fs::path d = fs::path(argv[1]) / name;
        auto g = circuit::read_circuit_file((d / "circuit.mpcg").string());
        auto in = preproc::read_input_file((d / "inputs.mpci").string());
        runtime::RunOptions opts;
        opts.slice = json_number(d / "expected.json", "slice", 262140);
        const int n = (int)json_number(d / "expected.json", "parties", 2);
        std::vector<std::string> eps;
        for (int i = 0; i < n; ++i) eps.push_back("127.0.0.1:" + std::to_string(23400 + 10 * n + i));
        std::vector<runtime::RunReport> reps(n);
        std::vector<std::exception_ptr> errs(n);
        std::vector<std::thread> th;
        for (int q = 0; q < n; ++q)
            th.emplace_back([&, q] {
                try {
                    const std::string tr = (d / ("triples_" + std::to_string(q) + ".bin")).string();
                    if (q == 1) {
                        reps[q] = runtime::run_one_party_b200(g, tr, in, q, eps, opts, 0, 20000, 30000);
                    } else {
                        net::MeshConfig mc;
                        mc.party = q;
                        mc.endpoints = eps;
                        runtime::PartyRuntime rt(g, spdz::read_store_file(tr), net::connect_mesh(mc), opts);
                        reps[q] = rt.run(in);
                    }
                } catch (...) {
                    errs[q] = std::current_exception();
                }
            });
        for (auto& t : th) t.join();
        try {
            for (auto& e : errs)
                if (e) std::rethrow_exception(e);
            compare(std::string(name) + " (B200 party 1 over TCP)", reps[0], reps[1]);
        } catch (const std::exception& e) {
            std::printf("%-40s FAIL  %s\n", name, e.what());
            ++failures;
        }
    }
    // a branch on a secret: both raise SecretControlFlow
    auto sb = circuit::read_circuit_file((fs::path(argv[1]) / "control_flow" / "secret_branch.mpcg").string());
    preproc::Inputs in{{"p", {1}}};
    int refused = 0;
    try {
        runtime::run_local(sb, 2, in, {});
    } catch (const sched::SecretControlFlow&) {
        ++refused;
    }
    try {
        runtime::run_local_b200(sb, 2, in, {}, 1, 64, 0);
    } catch (const sched::SecretControlFlow& e) {
        ++refused;
        std::printf("%-40s ok    %s\n", "secret_branch", e.what());
    }
    if (refused != 2) {
        std::printf("secret_branch: SecretControlFlow not raised by both\n");
        ++failures;
    }
    std::printf(failures ? "FAIL (%d)\n" : "PASS\n", failures);
    return failures ? 1 : 0;
}
