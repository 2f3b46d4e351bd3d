// Host build of csrc/aes_bitsliced.cuh (g++): reads N*16 seed bytes from stdin
// (N a multiple of 32), writes N*48 bytes of MMO expansion (3 fixed keys) to
// stdout. Used by tests/test_bitsliced_host.py to check the bitsliced circuit
// against the oracle / the reference's PRG vectors without a GPU.
#define __device__
#define __host__
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <vector>

#include "aes_bitsliced.cuh"

template <int KEY>
static void mmo32(const uint32_t* in, uint32_t* out) {
    uint32_t x[128];
    fssb::bs::to_slices(in, x);
    fssb::bs::encrypt<KEY>(x);
    fssb::bs::from_slices(x, out);
    for (int i = 0; i < 128; i++) out[i] ^= in[i];
}

int main() {
    std::vector<uint8_t> buf((size_t)1 << 20);
    size_t n = fread(buf.data(), 1, buf.size(), stdin);
    if (n % (32 * 16)) return 2;
    for (size_t off = 0; off < n; off += 32 * 16) {
        uint32_t in[128], o[3][128];
        memcpy(in, buf.data() + off, sizeof(in));
        mmo32<0>(in, o[0]);
        mmo32<1>(in, o[1]);
        mmo32<2>(in, o[2]);
        for (int j = 0; j < 32; j++)
            for (int b = 0; b < 3; b++) fwrite(o[b] + 4 * j, 1, 16, stdout);
    }
    return 0;
}
