// Host -> device copies from pageable memory at multi-threaded memcpy speed (see hostcopy.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>

namespace spdzb200 {

// true if `p` is ordinary (not page-locked, not device) host memory
bool is_pageable(const void* p);

// dst_dev <- src_host (pageable): the bytes pass through a pinned staging ring on `device`,
// filled slice-parallel by a worker pool, each slot DMA'd on `stream` as soon as it is full and
// reused once its DMA has completed.  Returns when the last slot is enqueued (the source may be
// reused then; the device copy completes in stream order).
cudaError_t staged_h2d(int device, void* dst_dev, const void* src_host, size_t bytes, cudaStream_t stream);

// host_dst (pageable) <- src_dev: DMA into the pinned ring on `stream` (several slots in flight),
// each landed slot copied out slice-parallel.  Synchronous: returns when host_dst is complete.
cudaError_t staged_d2h(int device, void* host_dst, const void* src_dev, size_t bytes, cudaStream_t stream);

// host memcpy split over the worker pool (large copies; falls back to memcpy below 1 MiB)
void parallel_copy(void* dst, const void* src, size_t bytes);

}  // namespace spdzb200
