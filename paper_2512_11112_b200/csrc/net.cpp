// The reference's wire format and TCP mesh (see net.hpp for the citations).
#include "net.hpp"

#include <arpa/inet.h>
#include <netdb.h>
#include <netinet/in.h>
#include <netinet/tcp.h>
#include <poll.h>
#include <sys/socket.h>
#include <unistd.h>

#include <cerrno>
#include <cstring>
#include <memory>

#include "internal.hpp"

namespace spdzb200 {

namespace {

// Moves exactly `len` bytes over a stream socket in either direction; false when the
// peer closed the connection or a hard error occurred (EINTR is retried).
bool move_bytes(int fd, void* buf, size_t len, bool outbound) {
    auto* cur = static_cast<char*>(buf);
    for (size_t done = 0; done < len;) {
        const ssize_t k = outbound ? ::send(fd, cur + done, len - done, MSG_NOSIGNAL)
                                   : ::recv(fd, cur + done, len - done, MSG_WAITALL);
        if (k > 0) {
            done += (size_t)k;
        } else if (k < 0 && errno == EINTR) {
            continue;
        } else {
            return false;
        }
    }
    return true;
}
bool send_exact(int fd, const void* buf, size_t len) { return move_bytes(fd, const_cast<void*>(buf), len, true); }
bool recv_exact(int fd, void* buf, size_t len) { return move_bytes(fd, buf, len, false); }

uint32_t le32(const uint8_t* b) { return (uint32_t)b[0] | (uint32_t)b[1] << 8 | (uint32_t)b[2] << 16 | (uint32_t)b[3] << 24; }

struct Endpoint {
    std::string host, port;
    explicit Endpoint(const std::string& ep) {
        const auto colon = ep.rfind(':');
        if (colon == std::string::npos)
            throw Error(SPDZ_ERR_NET, "NetError: bad endpoint '" + ep + "', expected host:port");
        host = ep.substr(0, colon);
        port = ep.substr(colon + 1);
    }
};

// a connected socket to `ep`, retrying (the peer may not listen yet) until the deadline
int connect_to(const Endpoint& ep, std::chrono::steady_clock::time_point deadline, int peer) {
    addrinfo want{};
    want.ai_family = AF_UNSPEC;
    want.ai_socktype = SOCK_STREAM;
    for (;;) {
        addrinfo* list = nullptr;
        int fd = -1;
        if (::getaddrinfo(ep.host.c_str(), ep.port.c_str(), &want, &list) == 0) {
            for (addrinfo* it = list; it && fd < 0; it = it->ai_next) {
                fd = ::socket(it->ai_family, it->ai_socktype, it->ai_protocol);
                if (fd >= 0 && ::connect(fd, it->ai_addr, it->ai_addrlen) != 0) {
                    ::close(fd);
                    fd = -1;
                }
            }
            ::freeaddrinfo(list);
        }
        if (fd >= 0) return fd;
        if (std::chrono::steady_clock::now() >= deadline)
            throw Error(SPDZ_ERR_NET,
                        "ConnectTimeout: peer " + std::to_string(peer) + " at " + ep.host + ":" + ep.port);
        std::this_thread::sleep_for(std::chrono::milliseconds(50));
    }
}

// listening socket on every interface at `port`
int listen_on(const std::string& port, int backlog) {
    const int fd = ::socket(AF_INET, SOCK_STREAM, 0);
    need(fd >= 0, SPDZ_ERR_NET, "NetError: socket() failed");
    const int on = 1;
    ::setsockopt(fd, SOL_SOCKET, SO_REUSEADDR, &on, sizeof on);
    sockaddr_in any{};
    any.sin_family = AF_INET;
    any.sin_port = htons((uint16_t)std::stoi(port));
    any.sin_addr.s_addr = htonl(INADDR_ANY);
    if (::bind(fd, reinterpret_cast<const sockaddr*>(&any), sizeof any) != 0 || ::listen(fd, backlog) != 0) {
        ::close(fd);
        throw Error(SPDZ_ERR_NET, "NetError: bind failed on port " + port);
    }
    return fd;
}

}  // namespace

void encode_header(uint8_t* hdr, uint8_t type, uint32_t lanes, uint64_t batch) {
    std::memset(hdr, 0, kFrameHeader);
    hdr[0] = type;
    for (int i = 0; i < 4; ++i) hdr[4 + i] = uint8_t(lanes >> (8 * i));
    for (int i = 0; i < 8; ++i) hdr[8 + i] = uint8_t(batch >> (8 * i));
}

NetLink::~NetLink() {
    stopping = true;
    for (int fd : fds)
        if (fd >= 0) ::shutdown(fd, SHUT_RDWR);
    for (auto& t : readers)
        if (t.joinable()) t.join();
    for (int fd : fds)
        if (fd >= 0) ::close(fd);
}

void NetLink::send(int peer, uint8_t type, uint64_t batch, const uint32_t* words, uint32_t lanes) {
    need(peer >= 0 && peer < n && peer != party && fds[peer] >= 0, SPDZ_ERR_INVALID_ARGUMENT, "bad peer");
    std::vector<uint8_t> buf(kFrameHeader + 4ull * lanes);  // little-endian host (x86-64 / aarch64)
    encode_header(buf.data(), type, lanes, batch);
    if (lanes) std::memcpy(buf.data() + kFrameHeader, words, 4ull * lanes);
    std::lock_guard lk(send_mu[peer]);
    if (!send_exact(fds[peer], buf.data(), buf.size()))
        throw Error(SPDZ_ERR_PEER_TIMEOUT, "PeerTimeout: send to peer " + std::to_string(peer) + " failed");
    bytes_sent += buf.size();
}

void NetLink::broadcast(uint8_t type, uint64_t batch, const uint32_t* words, uint32_t lanes) {
    for (int p = 0; p < n; ++p)
        if (p != party) send(p, type, batch, words, lanes);
}

std::vector<uint32_t> NetLink::recv(int peer, uint8_t type, uint64_t batch, uint64_t* cap) {
    const auto key = std::make_tuple(type, batch, peer);
    std::unique_lock lk(mu);
    const bool got = cv.wait_for(lk, io_timeout, [&] { return inbox.count(key) || !peer_error[peer].empty(); });
    auto it = inbox.find(key);
    if (it == inbox.end()) {
        if (!peer_error[peer].empty()) {
            const std::string why = peer_error[peer];
            throw Error(why.rfind("MalformedShareMessage", 0) == 0 ? SPDZ_ERR_MALFORMED_SHARE_MESSAGE
                                                                   : SPDZ_ERR_PEER_TIMEOUT,
                        why);
        }
        (void)got;
        throw Error(SPDZ_ERR_PEER_TIMEOUT,
                    "PeerTimeout: " + std::string(type == kMsgOpenShares ? "open" : "exchange") + " batch " +
                        std::to_string(batch) + " from peer " + std::to_string(peer));
    }
    if (cap && it->second.size() > *cap) {  // too long for the caller's buffer: keep the frame
        *cap = it->second.size();
        return {};
    }
    std::vector<uint32_t> out = std::move(it->second);
    inbox.erase(it);
    return out;
}

std::vector<std::vector<uint32_t>> NetLink::exchange(uint8_t type, uint64_t batch, const std::vector<uint32_t>& own) {
    broadcast(type, batch, own.data(), (uint32_t)own.size());
    std::vector<std::vector<uint32_t>> out(n);
    out[party] = own;
    for (int p = 0; p < n; ++p)
        if (p != party) out[p] = recv(p, type, batch);
    return out;
}

void NetLink::reader_loop(int peer) {
    const int fd = fds[peer];
    auto stop = [&](const std::string& why) {
        std::lock_guard lk(mu);
        peer_error[peer] = why;
        cv.notify_all();
    };
    for (;;) {
        uint8_t hdr[kFrameHeader];
        if (!recv_exact(fd, hdr, sizeof hdr)) return stop("PeerTimeout: connection to peer " + std::to_string(peer) +
                                                        " closed");
        if (hdr[0] > kMsgControl)  // decode_header (net.cpp:21-29)
            return stop("MalformedShareMessage: unknown msg-type " + std::to_string(hdr[0]));
        const uint32_t lanes = le32(hdr + 4);
        uint64_t batch = 0;
        for (int i = 0; i < 8; ++i) batch |= uint64_t(hdr[8 + i]) << (8 * i);
        if (lanes > max_frame_lanes)
            return stop("MalformedShareMessage: frame of " + std::to_string(lanes) + " lanes from peer " +
                        std::to_string(peer) + " exceeds the " + std::to_string(max_frame_lanes) + "-lane limit");
        std::vector<uint32_t> payload;
        try {
            payload.resize(lanes);
        } catch (const std::bad_alloc&) {
            return stop("MalformedShareMessage: cannot allocate a " + std::to_string(lanes) + "-lane frame from peer " +
                        std::to_string(peer));
        }
        if (lanes && !recv_exact(fd, payload.data(), 4ull * lanes))
            return stop("PeerTimeout: connection to peer " + std::to_string(peer) + " closed mid-frame");
        if (stopping) return;
        bytes_received += kFrameHeader + 4ull * lanes;
        std::lock_guard lk(mu);
        auto key = std::make_tuple(hdr[0], batch, peer);
        if (inbox.count(key)) {  // net.cpp:196-198, 214-216
            peer_error[peer] = "MalformedShareMessage: duplicate frame from peer " + std::to_string(peer);
            cv.notify_all();
            return;
        }
        inbox.emplace(key, std::move(payload));
        cv.notify_all();
    }
}

void NetLink::start_readers() {
    for (int p = 0; p < n; ++p)
        if (p != party) readers.emplace_back([this, p] { reader_loop(p); });
}

NetLink* connect_mesh(int party, const std::vector<std::string>& endpoints, std::chrono::milliseconds connect_timeout,
                      std::chrono::milliseconds io_timeout) {
    const int n = (int)endpoints.size();
    need(party >= 0 && party < n, SPDZ_ERR_NET, "NetError: party index out of range");
    auto link = std::make_unique<NetLink>(party, n);
    link->io_timeout = io_timeout;
    const auto deadline = std::chrono::steady_clock::now() + connect_timeout;
    auto adopt = [&](int peer, int fd) {
        const int on = 1;
        ::setsockopt(fd, IPPROTO_TCP, TCP_NODELAY, &on, sizeof on);
        link->fds[peer] = fd;
    };
    // parties above us connect to our endpoint; we connect to every party below us
    struct Listener {
        int fd = -1;
        ~Listener() {
            if (fd >= 0) ::close(fd);
        }
    } lst;
    if (party + 1 < n) lst.fd = listen_on(Endpoint(endpoints[party]).port, n);
    for (int lower = 0; lower < party; ++lower) {
        const int fd = connect_to(Endpoint(endpoints[lower]), deadline, lower);
        uint8_t me[4] = {uint8_t(party), uint8_t(party >> 8), uint8_t(party >> 16), uint8_t(party >> 24)};
        if (!send_exact(fd, me, sizeof me)) {  // the index announcement of the handshake
            ::close(fd);
            throw Error(SPDZ_ERR_NET, "ConnectTimeout: handshake with peer " + std::to_string(lower));
        }
        adopt(lower, fd);
    }
    for (int pending = n - 1 - party; pending > 0;) {
        const auto ms = std::chrono::duration_cast<std::chrono::milliseconds>(deadline - std::chrono::steady_clock::now());
        pollfd w{lst.fd, POLLIN, 0};
        if (ms.count() <= 0 || ::poll(&w, 1, (int)ms.count()) <= 0)
            throw Error(SPDZ_ERR_NET, "ConnectTimeout: waiting for " + std::to_string(pending) + " peer(s)");
        const int fd = ::accept(lst.fd, nullptr, nullptr);
        uint8_t who[4];
        if (fd < 0) continue;
        if (!recv_exact(fd, who, sizeof who)) {
            ::close(fd);
            continue;
        }
        const uint32_t idx = le32(who);
        if (idx >= (uint32_t)n || (int)idx <= party || link->fds[idx] >= 0) {
            ::close(fd);
            throw Error(SPDZ_ERR_NET, "IndexCollision: peer announced invalid index " + std::to_string(idx));
        }
        adopt((int)idx, fd);
        --pending;
    }
    link->start_readers();
    return link.release();
}

}  // namespace spdzb200

using namespace spdzb200;

struct spdz_net {
    std::unique_ptr<NetLink> link;
};

extern "C" {

int spdz_net_connect(int party, int n_parties, const char* const* endpoints, uint64_t connect_timeout_ms,
                     uint64_t io_timeout_ms, spdz_net** out) {
    return guard([&] {
        need(out && endpoints && n_parties >= 1 && n_parties <= SPDZ_MAX_PARTIES, SPDZ_ERR_INVALID_ARGUMENT,
             "bad mesh arguments");
        std::vector<std::string> eps;
        for (int i = 0; i < n_parties; ++i) {
            need(endpoints[i] != nullptr, SPDZ_ERR_INVALID_ARGUMENT, "null endpoint");
            eps.emplace_back(endpoints[i]);
        }
        auto* h = new spdz_net;
        try {
            h->link.reset(connect_mesh(party, eps, std::chrono::milliseconds(connect_timeout_ms ? connect_timeout_ms : 10000),
                                       std::chrono::milliseconds(io_timeout_ms ? io_timeout_ms : 10000)));
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int spdz_net_destroy(spdz_net* net) {
    delete net;
    return SPDZ_OK;
}

int spdz_net_send(spdz_net* net, int peer, int type, uint64_t batch, const uint32_t* words, uint32_t lanes) {
    return guard([&] {
        need(net != nullptr && type >= 0 && type <= kMsgControl, SPDZ_ERR_INVALID_ARGUMENT, "bad send");
        net->link->send(peer, (uint8_t)type, batch, words, lanes);
    });
}

int spdz_net_recv(spdz_net* net, int peer, int type, uint64_t batch, uint32_t* out, uint64_t cap, uint64_t* lanes) {
    return guard([&] {
        need(net != nullptr && lanes != nullptr && peer >= 0 && peer < net->link->n && peer != net->link->party,
             SPDZ_ERR_INVALID_ARGUMENT, "bad recv");
        // the frame stays queued when it does not fit, so a retry with a larger buffer gets it
        const uint64_t room = out ? cap : ~0ull;
        uint64_t fit = room;
        auto v = net->link->recv(peer, (uint8_t)type, batch, &fit);
        *lanes = fit > room ? fit : v.size();  // fit > room: the frame did not fit and is still queued
        need(fit <= room, SPDZ_ERR_LANE_COUNT_MISMATCH,
             "LaneCountMismatch: peer " + std::to_string(peer) + " sent " + std::to_string(*lanes) +
                 " lanes, expected at most " + std::to_string(cap));
        if (out && !v.empty()) std::memcpy(out, v.data(), v.size() * 4);
    });
}

int spdz_net_stats(spdz_net* net, uint64_t* bytes_sent, uint64_t* bytes_received) {
    return guard([&] {
        need(net != nullptr, SPDZ_ERR_INVALID_ARGUMENT, "null mesh");
        if (bytes_sent) *bytes_sent = net->link->bytes_sent;
        if (bytes_received) *bytes_received = net->link->bytes_received;
    });
}

}  // extern "C"

namespace spdzb200 {
NetLink* net_link(spdz_net* net) { return net ? net->link.get() : nullptr; }
}  // namespace spdzb200
