// MPCT triple-store files -> HBM (store.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

namespace spdzb200 {

// Where every section of one party's store file lies (validated, nothing read).
struct StoreLayout {
    int party = 0, n_parties = 0;
    uint32_t alpha_share = 0;
    uint64_t loop_iters = 0;
    uint64_t n_scalar = 0, scalar_off = 0;  // plane q starts at scalar_off + 4 q n_scalar
    struct Mat {
        uint32_t rows, din;
        uint64_t off;  // A.v; then A.m, B.v, B.m, C.v, C.m back to back
    };
    std::vector<Mat> mats;
    uint64_t n_masks = 0, masks_off = 0;
    uint64_t file_size = 0;
};

// Throws Error(SPDZ_ERR_STORE_FORMAT, "VersionMismatch: ..." / "CorruptPayload: ...").
StoreLayout scan_store(const char* path);

// File byte ranges -> device, through two pinned staging buffers on `stream`.
struct StagedUpload {
    static constexpr uint64_t kChunk = 16ull << 20;
    StagedUpload(const char* path, cudaStream_t stream);
    ~StagedUpload();
    StagedUpload(const StagedUpload&) = delete;
    StagedUpload& operator=(const StagedUpload&) = delete;
    void copy(uint64_t file_off, uint64_t bytes, void* dev_dst);
    // masks [first, first+count) of the AoS section at file_off -> planes (clear may be null)
    void copy_masks(uint64_t file_off, uint64_t first, uint64_t count, uint32_t* val, uint32_t* mac, uint32_t* clear);
    void finish();

   private:
    uint8_t* next_buffer();
    void submit();
    void read_into(uint64_t off, uint64_t bytes, uint8_t* dst);
    FILE* f = nullptr;
    cudaStream_t stream;
    uint8_t* pinned[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    bool used[2] = {false, false};
    int cur = 1;
};

}  // namespace spdzb200
