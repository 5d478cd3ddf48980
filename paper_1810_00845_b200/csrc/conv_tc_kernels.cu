// conv_tc_kernels.cu -- the conv accumulation (a9, K8) on the 5th-generation tensor cores.
//
//   out[o][x] = sum_t X[o][t] in[t][x]  mod q      (X: weight residues, in: ciphertext words)
//
// is a dense contraction (OC x T weights against T x words inputs), exact in integers.  Both
// operands are split into P = ceil(log2 q / 8) unsigned bytes, a = sum_i a_i 2^(8i), x = sum_j
// x_j 2^(8j), and the byte products are accumulated by tcgen05.mma.kind::i8 (u8 x u8 -> s32) in
// tensor memory:
//
//   sum_t x a = sum_s 2^(8s) C_s,   C_s = sum_{i+j=s} sum_t a_i x_j   (s < 2P - 1)
//
// One CTA (128 threads, 4 warps) owns 128 consecutive words of one (poly, limb) -- the MMA's
// M = 128 rows -- and a tile of 16 outputs.  Per K-chunk of 32 inputs t: every thread loads its
// word of the 32 inputs (coalesced), splits them into the P byte planes A_i [128 x 32] written to
// shared memory in the canonical K-major no-swizzle layout; the weight planes B [(j, o) = 16P rows
// x 32] arrive pre-split from a host-built image; one elected thread issues P MMAs
// D[:, 16 i + (16 j + o)] += A_i B^T, i.e. MMA i writes at TMEM column offset 16 i, so byte
// product (i, j) lands in diagonal block s = i + j (no cross-term bookkeeping; TMEM is zeroed
// first).  Epilogue: each thread reads its row's 2P - 1 diagonal sums (C_s < P T 255^2 < 2^31) and
// forms sum_s C_s 2^(8s) as two 128-bit halves (s < 8, s >= 8), reduced with two Barrett steps.
// Bit-exact integer arithmetic: the same residues as the FP64 / 128-bit CUDA-core kernel.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>
#include "launch.h"
#include "modarith.cuh"

namespace hisa {

constexpr int CTC_ROWS = 128, CTC_K = 32, CTC_OT = 16, CTC_THREADS = 256;
constexpr int CTC_PLANE = CTC_ROWS * CTC_K;   // bytes per A plane (4 KiB)
constexpr int CTC_BIMG = 8 * 512;             // bytes per weight image slot in global memory (P <= 8)
constexpr int CTC_TMEM = 256;                 // TMEM columns per CTA: (2P - 1) 16 <= 240; two CTAs per SM
constexpr int CTC_BREG = 6;                   // prefetched weight-image uint4 per thread (KC P <= 48)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// SM100 shared-memory matrix descriptor, K-major, no swizzle: core matrices of 8 rows x 16 bytes
// stored contiguously (128 B); LBO = byte distance between the two K-halves of a 32-byte row
// chunk, SBO = byte distance between 8-row groups; version 1 (bits 46-47).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
// instruction descriptor, kind::i8: D s32 (bits 4-5 = 2), A/B unsigned 8-bit, both K-major,
// N >> 3 at bits 17-22, M >> 4 at bits 24-28
__device__ __forceinline__ uint32_t umma_idesc_u8(int m, int n) {
    return (2u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void mma_u8(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// set by a wait that exceeded its wall-clock budget; read (and cleared) by the host after the
// launch's synchronisation -> HISA_E_CUDA (a __trap would poison the whole CUDA context, PyTorch's
// included, and clock64 keeps counting while a CTA is time-sliced out)
__device__ int g_ctc_timeout;
__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
    uint32_t done = 0;
    uint64_t t0 = 0;
    for (uint32_t spin = 0; !done; spin++) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 1000000;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}\n"
            : "=r"(done)
            : "r"(bar), "r"(phase)
            : "memory");
        if (!done && (spin & 1023) == 1023) {   // the clock is read once per 1024 polls
            const uint64_t t = globaltimer_ns();
            if (t0 == 0) t0 = t;
            if (t - t0 > 10000000000ull) {      // 10 s: flag it, never hang the device
                atomicExch(&g_ctc_timeout, 1);
                return;
            }
        }
    }
}
// 4 x 4 byte transpose: words a, b, c, d (inputs k .. k + 3 of one row) -> p[i] = byte i of
// (a, b, c, d), a in the low byte: 8 PRMT for four planes
__device__ __forceinline__ void transpose4(uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t* p) {
    const uint32_t t0 = __byte_perm(a, b, 0x5140), t1 = __byte_perm(a, b, 0x7362);
    const uint32_t t2 = __byte_perm(c, d, 0x5140), t3 = __byte_perm(c, d, 0x7362);
    p[0] = __byte_perm(t0, t2, 0x5410);
    p[1] = __byte_perm(t0, t2, 0x7632);
    p[2] = __byte_perm(t1, t3, 0x5410);
    p[3] = __byte_perm(t1, t3, 0x7632);
}
__device__ __forceinline__ uint64_t mad_wide(uint32_t a, uint32_t b, uint64_t c) {
    uint64_t d;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
    return d;
}

// Schedule (round 2): the byte split of the inputs is the expensive CUDA-core part (ncu of the
// round-1 kernel, profiles/r1_ncu_conv_tc.txt: issue-bound, tensor pipe 6 % busy, because every
// 16-output tile re-loaded and re-split all T inputs).  Now a CTA splits a super-chunk of KC
// K-chunks (32 KC inputs) of its 128 words ONCE into shared memory (A planes [kc][i], 4 KiB each)
// and then walks the output tiles: per tile only the pre-split weight image (prefetched into
// registers during the previous tile's epilogue) is stored, one thread issues the tile's KC P MMAs
// and a single commit, and the epilogue folds the 2P - 1 diagonal sums four at a time with
// IMAD.WIDE (C_4k + 2^8 C_4k+1 + 2^16 C_4k+2 + 2^24 C_4k+3 < 2^56) into two 128-bit halves and one
// Barrett step (two for P = 8).  T > 32 KC: further super-chunks add onto the stored outputs.
// KC = what fits the dynamic shared memory given by the launcher (two CTAs per SM when the whole T
// fits in half an SM's shared memory, else one).
// x mod q for 2^32 < q <= 2^40 (the P = 5 limbs) and any x < 2^64: r1 = floor(2^64 / q) < 2^32, so
// the quotient estimate floor(x r1 / 2^64) (>= floor(x / q) - 1, < 2^32) takes two IMAD.WIDE
__device__ __forceinline__ uint64_t barrett_q40(uint64_t x, uint32_t r1, uint64_t q) {
    const uint64_t p0 = (uint64_t)(uint32_t)x * r1;
    const uint64_t p1 = mad_wide((uint32_t)(x >> 32), r1, p0 >> 32);
    const uint32_t qe = (uint32_t)(p1 >> 32);
    return csub(x - (uint64_t)qe * q, q);
}

template <int P>
__device__ __forceinline__ void conv_tc_body(const uint64_t* const* __restrict__ in_ptrs,
                                             uint64_t* const* __restrict__ out_ptrs,
                                             const uint8_t* __restrict__ wimg, const ConvTcJob& job,
                                             const Mod* __restrict__ mods, int smem_ab, int limb, uint64_t* mbar,
                                             uint32_t& tmem_slot) {
    extern __shared__ __align__(128) uint8_t ctc_sm[];
    // thread r = tid % 128 owns row r (TMEM lane r: warp w reads lanes 32 (w % 4) ..); the two
    // warpgroups split alternate K-chunks in phase 1 and the two output halves in the epilogue
    const int tid = threadIdx.x, warp = tid >> 5, wg = tid >> 7, r = tid & 127;
    const long long N = 1ll << job.log_n;
    const Mod md = mods[limb];
    const long long off = (long long)blockIdx.z * job.poly_stride + (long long)limb * N + (long long)blockIdx.x * CTC_ROWS;
    const uint32_t bar0 = smem_u32(mbar);
    constexpr int bimg = 512 * P;                                // bytes of one chunk's weight image
    const int KC = min(min(job.n_chunks, smem_ab / (P * CTC_PLANE + bimg)), CTC_BREG * CTC_THREADS / (32 * P));
    uint8_t* sA = ctc_sm;                                      // [KC][P][4096]
    uint8_t* sB = ctc_sm + KC * P * CTC_PLANE;                 // [KC][512 P]
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_slot)), "n"(CTC_TMEM));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar0));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = tmem_slot;
    const uint32_t lane_base = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    constexpr int ndiag = 2 * P - 1;
    const uint32_t idesc = umma_idesc_u8(CTC_ROWS, 16 * P);
    uint32_t ph0 = 0;
    // this thread's row in the canonical layout: group r / 8 at 256 B, row r % 8 at 16 B
    const int arow_off = (r >> 3) * 256 + (r & 7) * 16;
    for (int c0 = 0; c0 < job.n_chunks; c0 += KC) {
        const int nk = min(KC, job.n_chunks - c0);
        // weight image of (limb, tile, chunks c0 .. c0 + nk): nk * 32 P uint4, CTC_BREG per thread
        const int nb4 = nk * 32 * P;
        uint4 breg[CTC_BREG];
        auto fetch_b = [&](int oct) {
            const uint8_t* base = wimg + (((size_t)limb * job.n_oct + oct) * job.n_chunks + c0) * CTC_BIMG;
#pragma unroll
            for (int k = 0; k < CTC_BREG; k++) {
                const int u = tid + k * CTC_THREADS;
                if (u < nb4) {
                    const int kc = u / (32 * P), w = u - kc * 32 * P;
                    breg[k] = __ldg(reinterpret_cast<const uint4*>(base + (size_t)kc * CTC_BIMG) + w);
                }
            }
        };
        fetch_b(0);
        // phase 1: split this super-chunk's inputs once.  Warpgroup wg takes chunks wg, wg + 2, ..,
        // in halves of 16 inputs, the next half's loads in flight while this one is transposed; lane
        // l of every warp holds the chunk's l-th input pointer (one coalesced load per chunk, a
        // chunk ahead), broadcast by shuffles -- no per-thread pointer loads in front of the data
        {
            const int lane = tid & 31;
            auto chunk_base = [&](int kc) -> const uint64_t* {
                const int t = (c0 + kc) * CTC_K + lane;
                return (kc < nk && t < job.T) ? in_ptrs[t] : nullptr;
            };
            auto load_half = [&](int half, const uint64_t* pch, uint64_t* v) {
#pragma unroll
                for (int k = 0; k < 16; k++) {
                    const uint64_t* p = reinterpret_cast<const uint64_t*>(
                        __shfl_sync(0xffffffffu, (unsigned long long)pch, 16 * half + k));
                    v[k] = p ? __ldg(p + off + r) : 0ull;
                }
            };
            auto split_store = [&](const uint64_t* v, int kc, int half) {
                uint8_t* a_ = sA + kc * P * CTC_PLANE + arow_off + 128 * half;   // k 0..15 at +0, 16..31 at +128
                uint32_t w[4][4];
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    uint32_t p[4];
                    transpose4((uint32_t)v[4 * u], (uint32_t)v[4 * u + 1], (uint32_t)v[4 * u + 2], (uint32_t)v[4 * u + 3], p);
#pragma unroll
                    for (int i = 0; i < 4; i++) w[i][u] = p[i];
                }
#pragma unroll
                for (int i = 0; i < 4; i++)
                    if (i < P) *reinterpret_cast<uint4*>(a_ + i * CTC_PLANE) = make_uint4(w[i][0], w[i][1], w[i][2], w[i][3]);
                if (P > 4) {
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        uint32_t p[4];
                        transpose4((uint32_t)(v[4 * u] >> 32), (uint32_t)(v[4 * u + 1] >> 32),
                                   (uint32_t)(v[4 * u + 2] >> 32), (uint32_t)(v[4 * u + 3] >> 32), p);
#pragma unroll
                        for (int i = 0; i < 4; i++) w[i][u] = p[i];
                    }
#pragma unroll
                    for (int i = 0; i < 4; i++)
                        if (4 + i < P)
                            *reinterpret_cast<uint4*>(a_ + (4 + i) * CTC_PLANE) = make_uint4(w[i][0], w[i][1], w[i][2], w[i][3]);
                }
            };
            const uint64_t* pcur = chunk_base(wg);
            const uint64_t* pnext = chunk_base(wg + 2);
            uint64_t va[16], vb[16];
            if (wg < nk) load_half(0, pcur, va);
            for (int kc = wg; kc < nk; kc += 2) {
                load_half(1, pcur, vb);
                split_store(va, kc, 0);
                pcur = pnext;
                pnext = chunk_base(kc + 4);
                if (kc + 2 < nk) load_half(0, pcur, va);
                split_store(vb, kc, 1);
            }
        }
        // (measured and dropped: an L2 prefetch of the next super-chunk / the next CTA's inputs
        // issued here -- 1.91 -> 1.85 ms at T = 144 but 6.2 -> 6.7 ms at T = 288 and 10.5 -> 11.4 ms
        // at T = 800: the prefetched lines are evicted before use, DRAM reads +23 %)
        for (int oct = 0; oct < job.n_oct; oct++) {
            if (wg == 0) {   // zero the tile's diagonal blocks (warpgroup 0 covers all 128 lanes)
                for (int s = 0; s < ndiag; s++) {
                    asm volatile(
                        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, "
                        "%1, %1, %1, %1};\n" ::"r"(lane_base + 16 * s),
                        "r"(0u));
                }
                asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
            }
            // this tile's weight image (prefetched) -> shared memory, packed at 512 P per chunk
#pragma unroll
            for (int k = 0; k < CTC_BREG; k++) {
                const int u = tid + k * CTC_THREADS;
                if (u < nb4) reinterpret_cast<uint4*>(sB)[u] = breg[k];
            }
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
            __syncthreads();
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            if (tid == 0) {
                for (int kc = 0; kc < nk; kc++) {
                    const uint64_t bdesc = umma_desc(smem_u32(sB + kc * bimg), 128, 256);
                    for (int i = 0; i < P; i++)
                        mma_u8(tmem + 16 * i, umma_desc(smem_u32(sA + (kc * P + i) * CTC_PLANE), 128, 256), bdesc,
                               idesc, 1u);
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
                             ::"r"(bar0) : "memory");
            }
            if (oct + 1 < job.n_oct) fetch_b(oct + 1);   // in flight across the MMAs and the epilogue
            mbar_wait(bar0, ph0);
            ph0 ^= 1;
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            // epilogue: row r, outputs oct * 16 + 8 wg + o, in quads
#pragma unroll
            for (int qd = 0; qd < 2; qd++) {
                const int o0 = oct * CTC_OT + wg * 8 + qd * 4;
                uint64_t* dst[4];
#pragma unroll
                for (int o = 0; o < 4; o++) dst[o] = o0 + o < job.OC ? out_ptrs[o0 + o] + off + r : nullptr;
                uint32_t c[ndiag][4];
#pragma unroll
                for (int s = 0; s < ndiag; s++)
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\n"
                                 : "=r"(c[s][0]), "=r"(c[s][1]), "=r"(c[s][2]), "=r"(c[s][3])
                                 : "r"(lane_base + 16 * s + 8 * wg + 4 * qd));
                asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
                uint64_t v[4];
#pragma unroll
                for (int o = 0; o < 4; o++) {
                    // G_k = C_4k + 2^8 C_4k+1 + 2^16 C_4k+2 + 2^24 C_4k+3 < 2^56; value = sum_k G_k 2^(32k)
                    uint64_t G[4] = {0, 0, 0, 0};
#pragma unroll
                    for (int s = 0; s < ndiag; s++)
                        G[s >> 2] = (s & 3) ? mad_wide(c[s][o], 1u << (8 * (s & 3)), G[s >> 2]) : (uint64_t)c[s][o];
                    if constexpr (P <= 5) {
                        // q <= 2^40, value = G0 + 2^32 G1 + 2^64 G2 (G2 = C_8 < 2^31): Horner with 64-bit
                        // Barrett steps, every operand < 2^64 (< 2^63 + 2^56, then < 2^56 + 2^40 twice)
                        if constexpr (P == 5) {
                            const uint32_t r1 = (uint32_t)md.r1;
                            uint64_t x = barrett_q40((G[2] << 32) + G[1], r1, md.q);
                            x = barrett_q40((x << 16) + (G[0] >> 16), r1, md.q);
                            v[o] = barrett_q40((x << 16) + (G[0] & 0xFFFFull), r1, md.q);
                        } else {
                            uint64_t x = barrett64((G[2] << 32) + G[1], md);
                            x = barrett64((x << 16) + (G[0] >> 16), md);
                            v[o] = barrett64((x << 16) + (G[0] & 0xFFFFull), md);
                        }
                    } else {
                        // value = accl + acch 2^64 (< 2^128 for P <= 7: one 128-bit Barrett step; P = 8:
                        // the high half is reduced first)
                        uint64_t l = G[1] << 32;
                        const uint64_t al = G[0] + l, ah = (G[1] >> 32) + (al < l);
                        l = G[3] << 32;
                        const uint64_t bl = G[2] + l, bh = (G[3] >> 32) + (bl < l);
                        const uint64_t rh = P > 7 ? barrett128(bl, bh, md) : bl;
                        v[o] = barrett128(al, ah + rh, md);
                    }
                }
#pragma unroll
                for (int o = 0; o < 4; o++) {
                    if (dst[o]) {
                        if (c0) v[o] = csub(v[o] + *dst[o], md.q);
                        *dst[o] = v[o];
                    }
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
            __syncthreads();
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        }
    }
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(CTC_TMEM));
}

// one launch for all limbs: the CTA's limb picks the byte-plane specialisation (40-bit limbs P = 5,
// 50-bit 7, 60-bit 8; P < 4 runs as 4 -- the missing planes are zero bytes on both operands)
__global__ void __launch_bounds__(CTC_THREADS, 2) k_conv_tc(const uint64_t* const* __restrict__ in_ptrs,
                                                 uint64_t* const* __restrict__ out_ptrs,
                                                 const uint8_t* __restrict__ wimg, ConvTcJob job,
                                                 const Mod* __restrict__ mods, int smem_ab) {
    __shared__ __align__(8) uint64_t mbar[1];
    __shared__ uint32_t tmem_slot;
    const int limb = job.limb_map[blockIdx.y];
    switch (job.P[limb]) {
        case 8: conv_tc_body<8>(in_ptrs, out_ptrs, wimg, job, mods, smem_ab, limb, mbar, tmem_slot); break;
        case 7: conv_tc_body<7>(in_ptrs, out_ptrs, wimg, job, mods, smem_ab, limb, mbar, tmem_slot); break;
        case 6: conv_tc_body<6>(in_ptrs, out_ptrs, wimg, job, mods, smem_ab, limb, mbar, tmem_slot); break;
        case 5: conv_tc_body<5>(in_ptrs, out_ptrs, wimg, job, mods, smem_ab, limb, mbar, tmem_slot); break;
        default: conv_tc_body<4>(in_ptrs, out_ptrs, wimg, job, mods, smem_ab, limb, mbar, tmem_slot); break;
    }
}

// weight image on the device: X = llround(W[o][t] * ps) (C semantics: half away from zero; exact
// -- |v| < 2^52 makes v +- 0.5 exact, larger |v| are integers), residue X mod q_limb in [0, q), byte
// j -> slot (limb, output tile, chunk) at row n = 16 j + o_local, column k, canonical K-major
// no-swizzle layout (the MMA's B operand image).  One thread per image byte.
__global__ void k_conv_tc_wimg(const double* __restrict__ W, double ps, int T, int OC, int n_oct, int n_chunks,
                               const Mod* __restrict__ mods, const uint8_t* __restrict__ Pl, uint8_t* img,
                               long long total) {
    const long long id = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (id >= total) return;
    const int byte = (int)(id % CTC_BIMG);
    long long slot = id / CTC_BIMG;
    const int ch = (int)(slot % n_chunks);
    slot /= n_chunks;
    const int oct = (int)(slot % n_oct);
    const int limb = (int)(slot / n_oct);
    // invert the canonical layout: byte = (n / 8) 256 + (k / 16) 128 + (n % 8) 16 + k % 16
    const int n = (byte / 256) * 8 + (byte % 128) / 16, k = ((byte % 256) / 128) * 16 + byte % 16;
    const int j = n / 16, o = oct * 16 + n % 16, t = ch * 32 + k;
    uint8_t out = 0;
    if (j < Pl[limb] && o < OC && t < T) {
        const double v = W[(long long)o * T + t] * ps;
        const double r = fabs(v) >= 4503599627370496.0 ? v : trunc(v + copysign(0.5, v));
        const long long X = (long long)r;
        const long long q = (long long)mods[limb].q;
        long long m = X % q;
        if (m < 0) m += q;
        out = (uint8_t)((unsigned long long)m >> (8 * j));
    }
    img[id] = out;
}

cudaError_t launch_conv_tc_wimg(const double* W, double ps, int T, int OC, int n_oct, int n_chunks, int l1,
                                const Mod* mods, const uint8_t* Pl, uint8_t* img, cudaStream_t st) {
    const long long total = (long long)l1 * n_oct * n_chunks * CTC_BIMG;
    k_conv_tc_wimg<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(W, ps, T, OC, n_oct, n_chunks, mods, Pl, img, total);
    return cudaGetLastError();
}

bool conv_tc_timed_out() {
    int v = 0;
    cudaMemcpyFromSymbol(&v, g_ctc_timeout, sizeof v);
    if (v) {
        const int z = 0;
        cudaMemcpyToSymbol(g_ctc_timeout, &z, sizeof z);
    }
    return v != 0;
}

// dynamic shared memory (A planes + weight images; the kernel derives KC from it): half an SM's
// shared memory, two CTAs per SM -- five K-chunks of a 40-bit limb (T <= 160 in one super-chunk).
// Measured against one CTA per SM with KC P <= 48: 288 inputs 6.3 vs 6.8 ms, 800 inputs 10.8 vs
// 14.0 ms.  HISA_CONV_TC_SMEM (bytes) overrides it (the multi-super-chunk parity case).
size_t conv_tc_smem_bytes() {
    static long forced = -1;
    if (forced < 0) {
        const char* e = getenv("HISA_CONV_TC_SMEM");
        forced = e ? atol(e) : 0;
    }
    return forced > 0 ? (size_t)forced : 115200;
}

cudaError_t launch_conv_tc(const uint64_t* const* in_ptrs, uint64_t* const* out_ptrs, const uint8_t* wimg,
                           const ConvTcJob& job, int nlimbs, const Mod* mods, cudaStream_t st) {
    const long long N = 1ll << job.log_n;
    if (N % CTC_ROWS) return cudaErrorInvalidValue;
    const size_t smem = conv_tc_smem_bytes();
    if (smem < 8 * (size_t)(CTC_PLANE + 512)) return cudaErrorInvalidValue;   // KC >= 1 for P = 8
    // the widest (slowest) limbs first
    ConvTcJob j = job;
    int nl = 0;
    for (int P = 8; P >= 1; P--)
        for (int i = 0; i < nlimbs; i++)
            if (job.P[job.limb_map[i]] == P) j.limb_map[nl++] = job.limb_map[i];
    cudaFuncSetAttribute(k_conv_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dim3 grid((unsigned)(N / CTC_ROWS), (unsigned)nl, 2);
    k_conv_tc<<<grid, CTC_THREADS, smem, st>>>(in_ptrs, out_ptrs, wimg, j, mods, (int)smem);
    return cudaGetLastError();
}

}  // namespace hisa
