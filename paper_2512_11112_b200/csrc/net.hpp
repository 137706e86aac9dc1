// Cross-host transport: the reference's wire format and TCP mesh, so a B200
// party can sit in a deployment whose other parties are reference processes
// (or other B200 hosts).
//
//   frame   net.hpp:40-49 / net.cpp:9-44: 16-byte header {msg-type u8, pad[3],
//           lane-count u32, batch-id u64} + lane-count u32 words, little-endian;
//   mesh    net_tcp.cpp:152-235: party i listens (endpoint i) for j > i and
//           dials j < i, announcing its index as one u32 after connect;
//   match   net.cpp:48-233: frames are matched by (type, batch-id, peer); an
//           open sums the peers' reduced words into the own contribution.
//
// Frames are read by one thread per peer into an inbox keyed by (type, batch,
// peer); the executor blocks on the key it needs (io_timeout -> PeerTimeout).
#pragma once
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

namespace spdzb200 {

enum : uint8_t { kMsgOpenShares = 0, kMsgCommit = 1, kMsgReveal = 2, kMsgNonce = 3, kMsgControl = 4 };
constexpr size_t kFrameHeader = 16;
constexpr uint64_t kMacBatchBase = 1ull << 62;    // runtime.cpp:25
constexpr uint64_t kInputBatchBase = 1ull << 63;  // runtime.cpp:26

void encode_header(uint8_t* hdr, uint8_t type, uint32_t lanes, uint64_t batch);

struct NetLink {
    int party = 0, n = 1;
    std::chrono::milliseconds io_timeout{10000};
    std::vector<int> fds;
    std::vector<std::thread> readers;
    std::vector<std::mutex> send_mu;
    std::mutex mu;
    std::condition_variable cv;
    std::map<std::tuple<uint8_t, uint64_t, int>, std::vector<uint32_t>> inbox;
    std::vector<std::string> peer_error;  // reader of peer p stopped: why
    std::atomic<uint64_t> bytes_sent{0}, bytes_received{0};
    std::atomic<bool> stopping{false};
    // frames announcing more lanes are rejected as MalformedShareMessage before any
    // allocation (a corrupt header must not take the host process down); 2^30 lanes = 4 GiB
    uint64_t max_frame_lanes = 1ull << 30;

    NetLink(int party_, int n_) : party(party_), n(n_), fds(n_, -1), send_mu(n_), peer_error(n_) {}
    ~NetLink();
    void send(int peer, uint8_t type, uint64_t batch, const uint32_t* words, uint32_t lanes);
    void broadcast(uint8_t type, uint64_t batch, const uint32_t* words, uint32_t lanes);
    // blocks until peer's frame (type, batch) is in the inbox; removes and returns its payload
    // cap (optional): a frame longer than *cap lanes is left in the inbox and its length
    // returned in *cap with an empty vector, so the caller can retry with a larger buffer
    std::vector<uint32_t> recv(int peer, uint8_t type, uint64_t batch, uint64_t* cap = nullptr);
    // Session::exchange (net.cpp:140-178): send to all, one frame of (type, batch) from each
    std::vector<std::vector<uint32_t>> exchange(uint8_t type, uint64_t batch, const std::vector<uint32_t>& own);
    void start_readers();

private:
    void reader_loop(int peer);
};

NetLink* connect_mesh(int party, const std::vector<std::string>& endpoints, std::chrono::milliseconds connect_timeout,
                      std::chrono::milliseconds io_timeout);

}  // namespace spdzb200
