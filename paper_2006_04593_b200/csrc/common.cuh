// Shared runtime helpers of the C ABI (error reporting) and the share-layer
// wire format (sharing.py:191-207: ring values at the smallest power-of-two
// byte width covering n).
#pragma once
#include <stdint.h>
#include <stdio.h>
#include <string.h>

namespace fssb {

__host__ __device__ inline int wire_bytes(int n_bits) {
    return n_bits <= 8 ? 1 : n_bits <= 16 ? 2 : n_bits <= 32 ? 4 : 8;
}

#ifdef __CUDACC__
__device__ __forceinline__ uint64_t wire_get(int wb, const void* p, uint64_t i) {
    switch (wb) {
        case 1: return reinterpret_cast<const uint8_t*>(p)[i];
        case 2: return reinterpret_cast<const uint16_t*>(p)[i];
        case 4: return reinterpret_cast<const uint32_t*>(p)[i];
        default: return reinterpret_cast<const uint64_t*>(p)[i];
    }
}
#endif

// Thread-local last-error message (fss_last_error); returns `code`.
int set_error(int code, const char* msg);
const char* last_error();
}  // namespace fssb
