// MPCT triple-store files (the reference's preprocessing output, one file per
// party: write_store_file / read_store_file, triple_store.cpp:163-244) read
// straight into HBM.
//
// Layout (little-endian): "MPCT", u32 version = 1, u64 prime, u32 party,
// u32 n_parties, u32 alpha_share, u64 loop_iters, u64 n, six u32[n] planes
// (a.v a.m b.v b.m c.v c.m), u64 mats, per matrix triple {u32 rows, u32 din,
// A.v A.m [rows*din], B.v B.m [din], C.v C.m [rows]}, u64 masks, masks x
// {u32 val, u32 mac, u32 clear}, end of file.
//
// scan_store() validates the container and records where every section lies
// (no payload is read); StagedUpload then moves exactly the byte ranges a run
// consumes through two pinned staging buffers with cudaMemcpyAsync, so the
// file read of chunk i+1 overlaps the H2D copy of chunk i.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "internal.hpp"
#include "store.hpp"

namespace spdzb200 {

namespace {

constexpr char kMagic[4] = {'M', 'P', 'C', 'T'};
constexpr uint32_t kStoreVersion = 1;
constexpr uint64_t kHeaderBytes = 4 + 4 + 8 + 4 + 4 + 4 + 8 + 8;

[[noreturn]] void format_error(const std::string& m) { throw Error(SPDZ_ERR_STORE_FORMAT, m); }

struct File {
    FILE* f = nullptr;
    explicit File(const char* path) : f(std::fopen(path, "rb")) {
        if (!f) format_error(std::string("cannot open '") + path + "'");
    }
    ~File() {
        if (f) std::fclose(f);
    }
    void seek(uint64_t off) {
        if (fseeko(f, (off_t)off, SEEK_SET) != 0) format_error("CorruptPayload: truncated triple store");
    }
    void read(void* dst, uint64_t bytes) {
        if (bytes && std::fread(dst, 1, bytes, f) != bytes) format_error("CorruptPayload: truncated triple store");
    }
    uint32_t u32() {
        uint8_t b[4];
        read(b, 4);
        return (uint32_t)b[0] | (uint32_t)b[1] << 8 | (uint32_t)b[2] << 16 | (uint32_t)b[3] << 24;
    }
    uint64_t u64() {
        const uint64_t lo = u32();
        return lo | (uint64_t)u32() << 32;
    }
};

}  // namespace

StoreLayout scan_store(const char* path) {
    need(path != nullptr, SPDZ_ERR_INVALID_ARGUMENT, "null store path");
    File f(path);
    if (fseeko(f.f, 0, SEEK_END) != 0) format_error("CorruptPayload: unreadable triple store");
    StoreLayout L;
    L.file_size = (uint64_t)ftello(f.f);
    f.seek(0);
    char magic[4];
    if (L.file_size < 4 || std::fread(magic, 1, 4, f.f) != 4 || std::memcmp(magic, kMagic, 4) != 0)
        format_error("VersionMismatch: not a triple store file");  // triple_store.cpp:198-200
    const uint32_t ver = f.u32();
    if (ver != kStoreVersion) format_error("VersionMismatch: triple store version " + std::to_string(ver));
    if (f.u64() != SPDZ_PRIME) format_error("VersionMismatch: triple store built for a different prime");
    L.party = (int)f.u32();
    L.n_parties = (int)f.u32();
    L.alpha_share = f.u32();
    L.loop_iters = f.u64();
    L.n_scalar = f.u64();
    L.scalar_off = kHeaderBytes;
    auto fits = [&](uint64_t off, uint64_t bytes) {
        if (off > L.file_size || bytes > L.file_size - off) format_error("CorruptPayload: truncated triple store");
    };
    // six planes, guarding the multiplication against absurd counts
    if (L.n_scalar > L.file_size / 24) format_error("CorruptPayload: truncated triple store");
    uint64_t at = L.scalar_off + 24 * L.n_scalar;
    fits(at, 8);
    f.seek(at);
    const uint64_t mats = f.u64();
    at += 8;
    if (mats > L.file_size / 8) format_error("CorruptPayload: truncated triple store");
    L.mats.reserve(mats);
    for (uint64_t i = 0; i < mats; ++i) {
        fits(at, 8);
        f.seek(at);
        StoreLayout::Mat m;
        m.rows = f.u32();
        m.din = f.u32();
        at += 8;
        m.off = at;
        const uint64_t words = 2 * ((uint64_t)m.rows * m.din + m.din + m.rows);
        if (words > L.file_size / 4) format_error("CorruptPayload: truncated triple store");
        fits(at, 4 * words);
        at += 4 * words;
        L.mats.push_back(m);
    }
    fits(at, 8);
    f.seek(at);
    L.n_masks = f.u64();
    at += 8;
    L.masks_off = at;
    if (L.n_masks > L.file_size / 12) format_error("CorruptPayload: truncated triple store");
    fits(at, 12 * L.n_masks);
    at += 12 * L.n_masks;
    if (at != L.file_size) format_error("CorruptPayload: trailing bytes in triple store");  // triple_store.cpp:241-243
    return L;
}

StagedUpload::StagedUpload(const char* path, cudaStream_t s) : stream(s) {
    f = std::fopen(path, "rb");
    if (!f) format_error(std::string("cannot open '") + path + "'");
    for (int i = 0; i < 2; ++i) {
        cuda_check(cudaMallocHost(&pinned[i], kChunk), "cudaMallocHost(staging)");
        cuda_check(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming), "event");
    }
}

StagedUpload::~StagedUpload() {
    for (int i = 0; i < 2; ++i) {
        if (ev[i]) {
            cudaEventSynchronize(ev[i]);
            cudaEventDestroy(ev[i]);
        }
        if (pinned[i]) cudaFreeHost(pinned[i]);
    }
    if (f) std::fclose(f);
}

uint8_t* StagedUpload::next_buffer() {
    cur ^= 1;
    if (used[cur]) cuda_check(cudaEventSynchronize(ev[cur]), "staging buffer reuse");
    return pinned[cur];
}

void StagedUpload::submit() {
    cuda_check(cudaEventRecord(ev[cur], stream), "record staging");
    used[cur] = true;
}

void StagedUpload::read_into(uint64_t off, uint64_t bytes, uint8_t* dst) {
    if (fseeko(f, (off_t)off, SEEK_SET) != 0 || (bytes && std::fread(dst, 1, bytes, f) != bytes))
        format_error("CorruptPayload: truncated triple store");
}

void StagedUpload::copy(uint64_t off, uint64_t bytes, void* dev_dst) {
    uint8_t* d = static_cast<uint8_t*>(dev_dst);
    for (uint64_t done = 0; done < bytes;) {
        const uint64_t n = std::min<uint64_t>(kChunk, bytes - done);
        uint8_t* buf = next_buffer();
        read_into(off + done, n, buf);
        cuda_check(cudaMemcpyAsync(d + done, buf, n, cudaMemcpyHostToDevice, stream), "H2D store");
        submit();
        done += n;
    }
}

void StagedUpload::copy_masks(uint64_t off, uint64_t first, uint64_t count, uint32_t* val, uint32_t* mac,
                              uint32_t* clear) {
    // AoS {val, mac, clear} -> three planes, de-interleaved in the staging buffer
    const uint64_t per = kChunk / 12;  // masks per chunk (the three planes share the buffer)
    for (uint64_t done = 0; done < count;) {
        const uint64_t n = std::min<uint64_t>(per, count - done);
        uint8_t* buf = next_buffer();
        std::vector<uint32_t> aos(3 * n);
        read_into(off + 12 * (first + done), 12 * n, reinterpret_cast<uint8_t*>(aos.data()));
        uint32_t* pv = reinterpret_cast<uint32_t*>(buf);
        uint32_t* pm = pv + n;
        uint32_t* pc = pm + n;
        for (uint64_t i = 0; i < n; ++i) {
            pv[i] = aos[3 * i];
            pm[i] = aos[3 * i + 1];
            pc[i] = aos[3 * i + 2];
        }
        cuda_check(cudaMemcpyAsync(val + done, pv, 4 * n, cudaMemcpyHostToDevice, stream), "H2D masks");
        cuda_check(cudaMemcpyAsync(mac + done, pm, 4 * n, cudaMemcpyHostToDevice, stream), "H2D masks");
        if (clear) cuda_check(cudaMemcpyAsync(clear + done, pc, 4 * n, cudaMemcpyHostToDevice, stream), "H2D masks");
        submit();
        done += n;
    }
}

void StagedUpload::finish() { cuda_check(cudaStreamSynchronize(stream), "store upload"); }

}  // namespace spdzb200

using namespace spdzb200;

extern "C" int spdz_store_inspect(const char* path, spdz_store_info_t* info) {
    return guard([&] {
        need(info != nullptr, SPDZ_ERR_INVALID_ARGUMENT, "null info");
        const StoreLayout L = scan_store(path);
        info->party = L.party;
        info->n_parties = L.n_parties;
        info->alpha_share = L.alpha_share;
        info->loop_iters = L.loop_iters;
        info->scalar_triples = L.n_scalar;
        info->matrix_triples = L.mats.size();
        info->input_masks = L.n_masks;
    });
}
