// host_stage.h -- pinned staging of pageable host buffers (internal).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

namespace spc {

// True for plain (pageable) host memory; false for device, managed or
// page-locked / registered host memory.
bool is_pageable(const void* p);

// Blocking memcpy split over a small persistent pool of host threads.
void host_copy(void* dst, const void* src, size_t bytes);

// Two pinned slots per direction (double buffering), grown on demand; one set
// per host thread (the drop-in is reentrant per thread).
struct HostStaging {
    float* in[2] = {nullptr, nullptr};
    float* out[2] = {nullptr, nullptr};
    size_t in_cap = 0, out_cap = 0;
    cudaEvent_t in_ev[2] = {nullptr, nullptr};   // the H2D that last read in[i] has finished
    cudaEvent_t out_ev[2] = {nullptr, nullptr};  // the D2H into out[i] has finished
    cudaError_t reserve(size_t in_bytes, size_t out_bytes);
};
HostStaging& host_staging();

}  // namespace spc
