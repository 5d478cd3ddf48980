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
#include "launch.h"
#include "modarith.cuh"

#ifndef CTC_TMEM_COLS
#define CTC_TMEM_COLS 256
#define CTC_MAXG_TILES 1
#endif

namespace hisa {

constexpr int CTC_ROWS = 128, CTC_K = 32, CTC_OT = 16, CTC_THREADS = 256;
constexpr int CTC_PLANE = CTC_ROWS * CTC_K;   // bytes per A plane (4 KiB)
constexpr int CTC_BIMG = 8 * 512;             // bytes per weight image slot (P <= 8)
constexpr int CTC_TMEM = CTC_TMEM_COLS;       // TMEM columns per CTA
constexpr int CTC_MAXG = CTC_MAXG_TILES;      // output tiles per pass (TMEM: G (2P - 1) 16 <= CTC_TMEM;
                                              // 512 columns / 3 tiles measured slower: one CTA per SM)

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
    const uint64_t t0 = globaltimer_ns();
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 1000000;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}\n"
            : "=r"(done)
            : "r"(bar), "r"(phase)
            : "memory");
        if (!done && globaltimer_ns() - t0 > 10000000000ull) {   // 10 s: flag it, never hang the device
            atomicExch(&g_ctc_timeout, 1);
            return;
        }
    }
}
__device__ __forceinline__ uint32_t pick_byte(uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t i) {
    // byte i (0..3) of each of a, b, c, d -> one word (a in the low byte)
    const uint32_t sel = i | ((i + 4) << 4);
    const uint32_t lo = __byte_perm(a, b, sel), hi = __byte_perm(c, d, sel);
    return __byte_perm(lo, hi, 0x5410);
}

__global__ void __launch_bounds__(CTC_THREADS) k_conv_tc(const uint64_t* const* __restrict__ in_ptrs,
                                                 uint64_t* const* __restrict__ out_ptrs,
                                                 const uint8_t* __restrict__ wimg, ConvTcJob job,
                                                 const Mod* __restrict__ mods) {
    extern __shared__ __align__(1024) uint8_t ctc_sm[];
    // two buffers: buffer b = [P planes of A, 128 rows x 32 bytes][B: 16 P rows x 32 bytes]
    constexpr int BUF = 8 * CTC_PLANE + CTC_MAXG * CTC_BIMG;
    // the T input pointers (offset to this tile) staged once, after the two operand buffers
    const uint64_t** sptr = reinterpret_cast<const uint64_t**>(ctc_sm + 2 * BUF);
    __shared__ __align__(8) uint64_t mbar[1];
    __shared__ uint32_t tmem_slot;
    // two warpgroups: warpgroup wg splits the K-chunks 2 step + wg into its own operand buffer;
    // thread r = tid % 128 owns row r (TMEM lane r: warp w reads lanes 32 (w % 4) ..)
    const int tid = threadIdx.x, warp = tid >> 5, wg = tid >> 7, r = tid & 127;
    const long long N = 1ll << job.log_n;
    const int limb = job.limb_map[blockIdx.y];
    const int P = job.P[limb];
    const Mod md = mods[limb];
    const long long off = (long long)blockIdx.z * job.poly_stride + (long long)limb * N + (long long)blockIdx.x * CTC_ROWS;
    const uint32_t bar0 = smem_u32(&mbar[0]);
    for (int t = tid; t < job.T; t += CTC_THREADS) sptr[t] = in_ptrs[t] + off;
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
    const int ndiag = 2 * P - 1;
    const uint32_t idesc = umma_idesc_u8(CTC_ROWS, 16 * P);
    uint32_t ph0 = 0;
    bool pend = false;
    // this thread's row in the canonical layout: group r / 8 at 256 B, row r % 8 at 16 B
    const int arow_off = (r >> 3) * 256 + (r & 7) * 16;
    uint8_t* sA = ctc_sm + wg * BUF;
    uint8_t* sB = sA + 8 * CTC_PLANE;
    const int n_steps = (job.n_chunks + 1) / 2;
    // G output tiles per pass share every input split (TMEM holds G x (2P - 1) x 16 columns)
    const int G = min(CTC_MAXG, CTC_TMEM / (16 * ndiag));
    for (int oct0 = 0; oct0 < job.n_oct; oct0 += G) {
        const int ng = min(G, job.n_oct - oct0);
        if (wg == 0) {   // zero the pass's diagonal blocks (warpgroup 0 covers all 128 lanes)
            for (int s = 0; s < ng * ndiag; s++) {
                asm volatile(
                    "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, "
                    "%1, %1, %1, %1};\n" ::"r"(lane_base + 16 * s),
                    "r"(0u));
            }
            asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        }
        for (int step = 0; step < n_steps; step++) {
            const int ch = 2 * step + wg;
            const bool active = ch < job.n_chunks;
            // this warpgroup's chunk: loads in flight before waiting for the previous step's MMAs
            uint32_t lo[CTC_K], hi[CTC_K];
#pragma unroll
            for (int k = 0; k < CTC_K; k++) {
                const int t = ch * CTC_K + k;
                const uint64_t v = (active && t < job.T) ? __ldg(sptr[t] + r) : 0ull;
                lo[k] = (uint32_t)v;
                hi[k] = (uint32_t)(v >> 32);
            }
            if (pend) { mbar_wait(bar0, ph0); ph0 ^= 1; pend = false; }
            if (active) {
                for (int i = 0; i < P; i++) {
                    const uint32_t* src = i < 4 ? lo : hi;
                    const uint32_t bi = (uint32_t)(i & 3);
                    uint32_t w[8];
#pragma unroll
                    for (int u = 0; u < 8; u++)
                        w[u] = pick_byte(src[4 * u], src[4 * u + 1], src[4 * u + 2], src[4 * u + 3], bi);
                    *reinterpret_cast<uint4*>(sA + i * CTC_PLANE + arow_off) = make_uint4(w[0], w[1], w[2], w[3]);
                    *reinterpret_cast<uint4*>(sA + i * CTC_PLANE + arow_off + 128) = make_uint4(w[4], w[5], w[6], w[7]);
                }
                // weights: the pre-split images of (limb, output tile, chunk) for the pass's tiles
                for (int g = 0; g < ng; g++) {
                    const uint4* wsrc = reinterpret_cast<const uint4*>(
                        wimg + (((size_t)limb * job.n_oct + oct0 + g) * job.n_chunks + ch) * CTC_BIMG);
                    for (int u = r; u < 32 * P; u += 128) reinterpret_cast<uint4*>(sB + g * CTC_BIMG)[u] = __ldg(wsrc + u);
                }
            }
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
            __syncthreads();
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            if (tid == 0) {
                for (int h = 0; h < 2 && 2 * step + h < job.n_chunks; h++) {
                    uint8_t* a_ = ctc_sm + h * BUF;
                    for (int g = 0; g < ng; g++) {
                        const uint64_t bdesc = umma_desc(smem_u32(a_ + 8 * CTC_PLANE + g * CTC_BIMG), 128, 256);
                        for (int i = 0; i < P; i++)
                            mma_u8(tmem + 16 * (g * ndiag + i), umma_desc(smem_u32(a_ + i * CTC_PLANE), 128, 256),
                                   bdesc, idesc, 1u);
                    }
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
                             ::"r"(bar0) : "memory");
            }
            pend = true;
        }
        if (pend) { mbar_wait(bar0, ph0); ph0 ^= 1; pend = false; }
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        // epilogue: row tid, outputs (oct0 + g) * 16 + o, in halves of 8
        for (int gh = wg; gh < 2 * ng; gh += 2) {   // warpgroup wg: halves og = wg
            const int g = gh >> 1, og = gh & 1;
            const int oct = oct0 + g;
            U128 accl[8], acch[8];
#pragma unroll
            for (int o = 0; o < 8; o++) { accl[o] = U128{0, 0}; acch[o] = U128{0, 0}; }
            for (int s = 0; s < ndiag; s++) {
                uint32_t r[8];
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
                             : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                               "=r"(r[7])
                             : "r"(lane_base + 16 * (g * ndiag + s) + 8 * og));
                asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
                const int sh = 8 * (s & 7);
#pragma unroll
                for (int o = 0; o < 8; o++) {
                    const uint64_t cv = (uint64_t)r[o];
                    const uint64_t l = sh ? cv << sh : cv, h = sh ? cv >> (64 - sh) : 0;
                    U128& a = s < 8 ? accl[o] : acch[o];
                    a.lo += l;
                    a.hi += h + (a.lo < l);
                }
            }
#pragma unroll
            for (int o = 0; o < 8; o++) {
                const int oo = oct * CTC_OT + og * 8 + o;
                if (oo >= job.OC) continue;
                // value = accl + acch 2^64: reduce the high half first (accl.hi < 2^32, r < 2^60)
                const uint64_t rh = barrett128(acch[o].lo, acch[o].hi, md);
                out_ptrs[oo][off + r] = barrett128(accl[o].lo, accl[o].hi + rh, md);
            }
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    }
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(CTC_TMEM));
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

size_t conv_tc_smem_bytes(int T) { return 2 * (8 * CTC_PLANE + CTC_MAXG * CTC_BIMG) + (size_t)T * sizeof(void*); }

cudaError_t launch_conv_tc(const uint64_t* const* in_ptrs, uint64_t* const* out_ptrs, const uint8_t* wimg,
                           const ConvTcJob& job, int nlimbs, const Mod* mods, cudaStream_t st) {
    const long long N = 1ll << job.log_n;
    if (N % CTC_ROWS) return cudaErrorInvalidValue;
    const size_t smem = conv_tc_smem_bytes(job.T);
    cudaFuncSetAttribute(k_conv_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dim3 grid((unsigned)(N / CTC_ROWS), (unsigned)nlimbs, 2);
    k_conv_tc<<<grid, CTC_THREADS, smem, st>>>(in_ptrs, out_ptrs, wimg, job, mods);
    return cudaGetLastError();
}

}  // namespace hisa
