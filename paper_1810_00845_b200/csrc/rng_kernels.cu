// rng_kernels.cu -- counter-mode ChaCha20 (RFC 8439 block function, 20 rounds) and the
// fixed-position samplers of DESIGN.md A9-A11 (K9), plus small integer-polynomial helpers used by
// keygen / encrypt (K10).  One thread = one 64-byte block, so generation is embarrassingly
// parallel and bit-identical to any other implementation of the same stream layout:
//   key = seed (LE u64) in key words 0,1; nonce = (tag, index lo, index hi); 64-bit stream word n
//   = u32 words 2n (low), 2n+1 (high) of block n / 8.
//   uniform mod q: coefficient t = (word(2t+1) 2^64 + word(2t)) mod q
//   ternary:       (word(t) mod 3) - 1
//   CBD(21):       popcount(word(t) & M) - popcount((word(t) >> 21) & M), M = 2^21 - 1
#include <cuda_runtime.h>
#include "launch.h"

namespace hisa {

__device__ __forceinline__ uint32_t rotl(uint32_t x, int n) { return __funnelshift_l(x, x, n); }
#define QRD(a, b, c, d)                 \
    a += b; d ^= a; d = rotl(d, 16);    \
    c += d; b ^= c; b = rotl(b, 12);    \
    a += b; d ^= a; d = rotl(d, 8);     \
    c += d; b ^= c; b = rotl(b, 7);

__device__ __forceinline__ void chacha_block(uint64_t seed, uint32_t tag, uint64_t index, uint32_t counter,
                                             uint32_t out[16]) {
    uint32_t s[16] = {0x61707865u, 0x3320646eu, 0x79622d32u, 0x6b206574u,
                      (uint32_t)seed, (uint32_t)(seed >> 32), 0, 0, 0, 0, 0, 0,
                      counter, tag, (uint32_t)index, (uint32_t)(index >> 32)};
    uint32_t x[16];
#pragma unroll
    for (int i = 0; i < 16; i++) x[i] = s[i];
#pragma unroll
    for (int i = 0; i < 10; i++) {
        QRD(x[0], x[4], x[8], x[12]) QRD(x[1], x[5], x[9], x[13])
        QRD(x[2], x[6], x[10], x[14]) QRD(x[3], x[7], x[11], x[15])
        QRD(x[0], x[5], x[10], x[15]) QRD(x[1], x[6], x[11], x[12])
        QRD(x[2], x[7], x[8], x[13]) QRD(x[3], x[4], x[9], x[14])
    }
#pragma unroll
    for (int i = 0; i < 16; i++) out[i] = x[i] + s[i];
}

struct UniformJob {
    uint64_t index[MAXL];
    uint8_t mod[MAXL];
};

// grid.y = limb; each thread one block = 4 coefficients
__global__ void __launch_bounds__(256) k_sample_uniform(uint64_t* out, uint64_t seed, uint32_t tag, UniformJob job,
                                                        int log_n, const Mod* __restrict__ mods) {
    const int limb = blockIdx.y;
    const Mod md = mods[job.mod[limb]];
    const uint32_t nblocks = (1u << log_n) / 4;
    uint64_t* o = out + ((long long)limb << log_n);
    for (uint32_t blk = blockIdx.x * blockDim.x + threadIdx.x; blk < nblocks; blk += gridDim.x * blockDim.x) {
        uint32_t w[16];
        chacha_block(seed, tag, job.index[limb], blk, w);
#pragma unroll
        for (int c = 0; c < 4; c++) {
            const uint64_t lo = (uint64_t)w[4 * c] | ((uint64_t)w[4 * c + 1] << 32);
            const uint64_t hi = (uint64_t)w[4 * c + 2] | ((uint64_t)w[4 * c + 3] << 32);
            o[4 * blk + c] = barrett128(lo, hi, md);
        }
    }
}

// kind 0 ternary, 1 CBD; each thread one block = 8 coefficients
__global__ void __launch_bounds__(256) k_sample_small(int64_t* out, uint64_t seed, uint32_t tag, uint64_t index,
                                                      int kind, int log_n) {
    const uint32_t nblocks = (1u << log_n) / 8;
    for (uint32_t blk = blockIdx.x * blockDim.x + threadIdx.x; blk < nblocks; blk += gridDim.x * blockDim.x) {
        uint32_t w[16];
        chacha_block(seed, tag, index, blk, w);
#pragma unroll
        for (int c = 0; c < 8; c++) {
            const uint64_t v = (uint64_t)w[2 * c] | ((uint64_t)w[2 * c + 1] << 32);
            int64_t r;
            if (kind == 0) r = (int64_t)(v % 3) - 1;
            else {
                const uint64_t M = (1ull << 21) - 1;
                r = (int64_t)__popcll(v & M) - (int64_t)__popcll((v >> 21) & M);
            }
            out[8 * blk + c] = r;
        }
    }
}

struct ModMapJob {
    uint8_t mod[MAXL];
};
__global__ void __launch_bounds__(256) k_int_to_limbs(const int64_t* __restrict__ x, uint64_t* out, ModMapJob job,
                                                      int log_n, const Mod* __restrict__ mods) {
    const int limb = blockIdx.y;
    const Mod md = mods[job.mod[limb]];
    const uint32_t N = 1u << log_n;
    uint64_t* o = out + ((long long)limb << log_n);
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < N; t += gridDim.x * blockDim.x) {
        const int64_t v = x[t];
        if (v >= 0) o[t] = barrett64((uint64_t)v, md);
        else {
            const uint64_t a = barrett64((uint64_t)(-v), md);
            o[t] = a ? md.q - a : 0;
        }
    }
}

__global__ void __launch_bounds__(256) k_automorphism_int(const int64_t* __restrict__ in, int64_t* out, int log_n,
                                                          uint64_t g) {
    const uint32_t N = 1u << log_n;
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < N; t += gridDim.x * blockDim.x) {
        const uint64_t idx = ((uint64_t)t * g) & (2ull * N - 1);
        if (idx < N) out[idx] = in[t];
        else out[idx - N] = -in[t];
    }
}

cudaError_t launch_sample_uniform(uint64_t* out, uint64_t seed, uint32_t tag, const uint64_t* index_per_limb_host,
                                  const uint8_t* mod_per_limb_host, int nlimbs, int log_n, const Mod* mods,
                                  cudaStream_t st) {
    if (nlimbs > MAXL) return cudaErrorInvalidValue;
    UniformJob job;
    for (int i = 0; i < nlimbs; i++) { job.index[i] = index_per_limb_host[i]; job.mod[i] = mod_per_limb_host[i]; }
    const int nb = (1 << log_n) / 4;
    dim3 grid((nb + 255) / 256, nlimbs);
    k_sample_uniform<<<grid, 256, 0, st>>>(out, seed, tag, job, log_n, mods);
    return cudaGetLastError();
}

cudaError_t launch_sample_small(int64_t* out, uint64_t seed, uint32_t tag, uint64_t index, int kind, int log_n,
                                cudaStream_t st) {
    const int nb = (1 << log_n) / 8;
    k_sample_small<<<(nb + 255) / 256, 256, 0, st>>>(out, seed, tag, index, kind, log_n);
    return cudaGetLastError();
}

cudaError_t launch_int_to_limbs(const int64_t* x, uint64_t* out, const uint8_t* mod_map_host, int nlimbs, int log_n,
                                const Mod* mods, cudaStream_t st) {
    if (nlimbs > MAXL) return cudaErrorInvalidValue;
    ModMapJob job;
    for (int i = 0; i < nlimbs; i++) job.mod[i] = mod_map_host[i];
    dim3 grid(((1 << log_n) + 255) / 256, nlimbs);
    k_int_to_limbs<<<grid, 256, 0, st>>>(x, out, job, log_n, mods);
    return cudaGetLastError();
}

cudaError_t launch_automorphism_int(const int64_t* in, int64_t* out, int log_n, uint64_t g, cudaStream_t st) {
    k_automorphism_int<<<((1 << log_n) + 255) / 256, 256, 0, st>>>(in, out, log_n, g);
    return cudaGetLastError();
}

}  // namespace hisa
