// ntt_kernels.cu -- pass kernels (a1/a2) and the fused lift / combine variants used by rescale
// (a8), ModUp and ModDown (a5).  See ntt.cuh for the decomposition.
#include <cuda_runtime.h>
#include <cstdlib>
#include <type_traits>
#include "ntt.cuh"
#include "ntt_f64.cuh"
#include "launch.h"

namespace hisa {

// smem tile geometry: column passes stage G columns x M rows, row passes G rows x M.
template <int LOG_M, int LOG_R>
__device__ __forceinline__ void tile_coords(int& g, int& t) {
    using G = Geo<LOG_M, LOG_R>;
    g = threadIdx.x / G::T;
    t = threadIdx.x % G::T;
}

// 8-byte asynchronous global -> shared copy (LDGSTS): tiles land in the swizzled layout without
// staging registers, all of a thread's copies in flight at once
__device__ __forceinline__ void cp_async8(uint64_t* smem, const uint64_t* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

__device__ __forceinline__ bool job_limb(const PassJob& job, int& a, int& b) {
    const int lam = blockIdx.y;
    a = lam / job.nb;
    b = lam % job.nb;
    return !(job.skip_diag && a == b);
}

// ------------------------------------------------------------------------------------------
// FP64 engine selection: limbs with q < 2^50 run the exact FP64 butterflies (ntt_f64.cuh); the
// pass-1 -> pass-2 (and pass-A -> pass-B) intermediate of such a limb is stored as centred-lazy
// doubles (|v| <= 2q), a format only the next pass of the same modulus reads.
// ------------------------------------------------------------------------------------------
__host__ __device__ constexpr int ilog2c(int v) { return v <= 1 ? 0 : 1 + ilog2c(v >> 1); }

__device__ __forceinline__ bool use_f64(uint64_t q, const Tables& tb) { return (double)q < tb.f64_max_q; }

// ------------------------------------------------------------------------------------------
// forward pass 1: columns.  Tile = Gc consecutive columns (Gc = blockDim/T), M = M1 rows.
// Input canonical (or lifted) residues; output lazy (int: [0, 4q); FP64: centred doubles).
// ------------------------------------------------------------------------------------------
template <int LOG_M, int LOG_R, int LOADMODE, int MINB, int GC = 0>
__global__ void __launch_bounds__(256, MINB) k_fwd_cols(PassJob job, Tables tb) {
    using G = Geo<LOG_M, LOG_R>;
    extern __shared__ uint64_t sm[];
    int a, b;
    if (!job_limb(job, a, b)) return;
    const int z = blockIdx.z;
    const int log_n = tb.log_n;
    const int M2 = 1 << (log_n - LOG_M);
    // GC > 0: the tile width is a compile-time constant, so the per-element (column, row)
    // addressing of the load / lift / store loops folds into immediates
    const int Gc = GC > 0 ? GC : blockDim.x / G::T;
    const int col0 = blockIdx.x * Gc;
    const int mi = job.mod_map[b];
    const Mod md = tb.mods[mi];
    const bool fp = use_f64(md.q, tb);
    const uint64_t* src = job.src[z] + a * job.src_a + b * job.src_b;
    uint64_t* dst = job.dst[z] + a * job.dst_a + b * job.dst_b;
    const int nthr = GC > 0 ? GC * G::T : blockDim.x;
    const int lg = GC > 0 ? ilog2c(GC) : __ffs(Gc) - 1;
    const uint64_t Qs = LOADMODE == LOAD_LIFT ? tb.mods[job.smod_map[a]].q : 0;
    if (fp && (LOADMODE != LOAD_LIFT || (double)Qs < tb.f64_max_q)) {
        // FP64 limb: coalesced loads straight into registers, converted (and, for ModUp, lifted:
        // x in [0, Qs) -> x - Qs if x > Qs/2, exact, |.| < 2^49 -- the engine's first stage
        // re-centres any |v| < 8q) and stored once into the swizzled tile
        double* smd = reinterpret_cast<double*>(sm);
        const double qs = (double)Qs, half = (double)(Qs >> 1);
        uint64_t v[G::R];
#pragma unroll
        for (int k = 0; k < G::R; k++) {
            const int i = threadIdx.x + k * nthr;
            v[k] = __ldg(&src[(long long)(i >> lg) * M2 + col0 + (i & (Gc - 1))]);
        }
#pragma unroll
        for (int k = 0; k < G::R; k++) {
            const int i = threadIdx.x + k * nthr;
            double d = u2d(v[k]);
            if (LOADMODE == LOAD_LIFT) d = d > half ? __dsub_rn(d, qs) : d;
            smd[G::addr(i & (Gc - 1), i >> lg)] = d;
        }
    } else {
        // coalesced asynchronous load, lanes along columns
#pragma unroll 4
        for (int k = 0; k < G::R; k++) {
            const int i = threadIdx.x + k * nthr;
            cp_async8(&sm[G::addr(i & (Gc - 1), i >> lg)], &src[(long long)(i >> lg) * M2 + col0 + (i & (Gc - 1))]);
        }
        cp_async_wait_all();
        if (LOADMODE == LOAD_LIFT) {   // integer lift (source or target >= 2^50)
#pragma unroll 4
            for (int k = 0; k < G::R; k++) {
                const int i = threadIdx.x + k * nthr;
                uint64_t* p = &sm[G::addr(i & (Gc - 1), i >> lg)];
                const uint64_t v = lift_centered(*p, Qs, md);
                if (fp) *reinterpret_cast<double*>(p) = u2d(v);
                else *p = v;
            }
        }
    }
    __syncthreads();
    int g, t;
    tile_coords<LOG_M, LOG_R>(g, t);
    if (fp) {
        const double2 qd = tb.modd[mi];
        fwd_engine_f64<LOG_M, LOG_R>(reinterpret_cast<double*>(sm), qd.x, qd.y, tb.fwd_d + ((long long)mi << log_n),
                                     0, 0, g, t);
    } else {
        fwd_engine<LOG_M, LOG_R>(sm, md.q, tb.fwd + ((long long)mi << log_n), 0, 0, g, t);
    }
#pragma unroll 4
    for (int k = 0; k < G::R; k++) {
        const int i = threadIdx.x + k * nthr;
        dst[(long long)(i >> lg) * M2 + col0 + (i & (Gc - 1))] = sm[G::addr(i & (Gc - 1), i >> lg)];   // lazy
    }
}

// ------------------------------------------------------------------------------------------
// forward pass 1 for M1 = 256 with radix-16 phases, register-direct (the N = 2^16 form): a CTA
// owns 16 consecutive columns; thread (g = tid % 16, t = tid / 16) loads rows t + 16e (e < 16) of
// column g straight into registers -- exactly phase 1's operands, and a warp's loads are two
// 128-byte row segments -- runs phase 1 (stages 0-3) in registers, exchanges once through the
// padded shared tile, runs phase 2 (stages 4-7) on rows 16t + e and stores them from registers
// (again two 128-byte segments per warp store).  One shared-memory round trip per element
// instead of three, one barrier.
// ------------------------------------------------------------------------------------------
// four radix-2 stages u0 .. u0 + 3 of a 256-point pass on 16 register operands (stride 8 >> uu);
// twiddle index 2^(s0+u) + (high << u) + (ohigh << uu) + k as in fwd_engine.  FP64 stages re-centre
// X at u % 3 == 0 only (outputs feed a pass that starts with a full stage, or a full reduction).
template <typename V, bool FP, bool SMEM_TW = false>
__device__ __forceinline__ void col_phase16(V (&r)[16], int u0, int ohigh, const void* twp, double q, double qinv,
                                            uint64_t qi, int s0 = 0, uint32_t high = 0) {
#pragma unroll
    for (int uu = 0; uu < 4; uu++) {
        const int u = u0 + uu;
        const int dist = 8 >> uu;
        const uint32_t tbase = (1u << (s0 + u)) + (high << u) + ((uint32_t)ohigh << uu);
#pragma unroll
        for (int k = 0; k < 8; k++) {
            if (k >= (1 << uu)) break;
            if constexpr (FP) {
                const double W = SMEM_TW ? reinterpret_cast<const double*>(twp)[tbase + k]
                                         : __ldg(reinterpret_cast<const double*>(twp) + tbase + k);
#pragma unroll
                for (int e0 = 0; e0 < 8; e0++) {
                    if (e0 >= dist) break;
                    const int e = k * 2 * dist + e0;
                    const double X = full_stage_cols(u) ? redd(r[e], q, qinv) : r[e];
                    const double T = mulred(r[e + dist], W, q, qinv);
                    r[e] = __dadd_rn(X, T);
                    r[e + dist] = __dsub_rn(X, T);
                }
            } else {
                const ulonglong2 W = __ldg(reinterpret_cast<const ulonglong2*>(twp) + tbase + k);
                const uint64_t q2 = 2 * qi;
#pragma unroll
                for (int e0 = 0; e0 < 8; e0++) {
                    if (e0 >= dist) break;
                    const int e = k * 2 * dist + e0;
                    uint64_t X = r[e];
                    X = X >= q2 ? X - q2 : X;
                    const uint64_t Tm = mul_shoup_lazy(r[e + dist], W.x, W.y, qi);
                    r[e] = X + Tm;
                    r[e + dist] = X - Tm + q2;
                }
            }
        }
    }
}

template <bool FP, int LOADMODE>
__device__ __forceinline__ void fwd_cols_r16_body(const PassJob& job, const Tables& tb, const uint64_t* src,
                                                  uint64_t* dst, int mi, const Mod& md, int a, int col0, int M2) {
    using G = Geo<8, 4>;
    extern __shared__ uint64_t sm[];
    const int g = threadIdx.x & 15, t = threadIdx.x >> 4;
    using V = typename std::conditional<FP, double, uint64_t>::type;
    V r[16];
    {
        uint64_t v[16];
#pragma unroll
        for (int e = 0; e < 16; e++) v[e] = __ldg(&src[(long long)(t + 16 * e) * M2 + col0 + g]);
        const uint64_t Qs = LOADMODE == LOAD_LIFT ? tb.mods[job.smod_map[a]].q : 0;
        const bool fast_lift = FP && (double)Qs < tb.f64_max_q;
        const double qs = (double)Qs, half = (double)(Qs >> 1);
#pragma unroll
        for (int e = 0; e < 16; e++) {
            if constexpr (FP) {
                if (LOADMODE == LOAD_LIFT && !fast_lift) {
                    r[e] = u2d(lift_centered(v[e], Qs, md));
                } else {
                    double d = u2d(v[e]);
                    if (LOADMODE == LOAD_LIFT) d = d > half ? __dsub_rn(d, qs) : d;
                    r[e] = d;
                }
            } else {
                r[e] = LOADMODE == LOAD_LIFT ? lift_centered(v[e], Qs, md) : v[e];
            }
        }
    }
    const double2 qd = FP ? tb.modd[mi] : make_double2(0, 0);
    const void* twp = FP ? (const void*)(tb.fwd_d + ((long long)mi << tb.log_n))
                         : (const void*)(tb.fwd + ((long long)mi << tb.log_n));
    col_phase16<V, FP>(r, 0, 0, twp, qd.x, qd.y, md.q);
    V* tile = reinterpret_cast<V*>(sm);
#pragma unroll
    for (int e = 0; e < 16; e++) tile[G::addr(g, t + 16 * e)] = r[e];
    __syncthreads();
#pragma unroll
    for (int e = 0; e < 16; e++) r[e] = tile[G::addr(g, 16 * t + e)];
    col_phase16<V, FP>(r, 4, t, twp, qd.x, qd.y, md.q);
#pragma unroll
    for (int e = 0; e < 16; e++) {
        uint64_t w;
        if constexpr (FP) w = (uint64_t)__double_as_longlong(r[e]);
        else w = r[e];
        dst[(long long)(16 * t + e) * M2 + col0 + g] = w;   // lazy
    }
}

template <int LOADMODE, int MINB>
__global__ void __launch_bounds__(256, MINB) k_fwd_cols_r16(PassJob job, Tables tb) {
    int a, b;
    if (!job_limb(job, a, b)) return;
    const int z = blockIdx.z;
    const int M2 = 1 << (tb.log_n - 8);
    const int col0 = blockIdx.x * 16;
    const int mi = job.mod_map[b];
    const Mod md = tb.mods[mi];
    const uint64_t* src = job.src[z] + a * job.src_a + b * job.src_b;
    uint64_t* dst = job.dst[z] + a * job.dst_a + b * job.dst_b;
    if (use_f64(md.q, tb)) fwd_cols_r16_body<true, LOADMODE>(job, tb, src, dst, mi, md, a, col0, M2);
    else fwd_cols_r16_body<false, LOADMODE>(job, tb, src, dst, mi, md, a, col0, M2);
}

// ------------------------------------------------------------------------------------------
// ModUp pass 1 at M1 = 256 (N = 2^16), looped over output primes: one CTA per (16-column block,
// digit a, chunk of output primes, ciphertext) loads its 16 x 256 coefficients of digit a ONCE,
// lifts them once (centred w.r.t. q_a: an integer of magnitude < q_a / 2, held exactly as a
// double when q_a < 2^50), then runs the first-pass NTT for every output prime b of its chunk
// (b != a) from registers -- instead of one CTA per (a, b) limb that reloads and re-lifts the
// same digit l + 1 times.  ncu (profiles/r2_ncu_modup_v1.txt): the per-limb kernel spent as many
// issue slots on loads, 64-bit addressing, the lift's compare/select and per-CTA setup as on its
// FP64 butterflies.  Wide source digits (q_a >= 2^50: the 60-bit q_0 of configs 1, 3-5) lift
// per output prime with the integer lift (exact mod q_b), as before.
// ------------------------------------------------------------------------------------------
#ifndef MODUP_MINB
#define MODUP_MINB 3
#endif
template <int MINB>
__global__ void __launch_bounds__(256, MINB) k_modup_cols16(PassJob job, Tables tb, int bchunk, int nbc) {
    using G = Geo<8, 4>;
    constexpr int M2 = 256;
    extern __shared__ uint64_t sm[];
    const int a = blockIdx.y / nbc, bc = blockIdx.y % nbc;
    const int z = blockIdx.z;
    const int col0 = blockIdx.x * 16;
    const int g = threadIdx.x & 15, t = threadIdx.x >> 4;
    const uint64_t* src = job.src[z] + a * job.src_a + col0 + g + (long long)t * M2;
    const uint64_t Qs = tb.mods[job.smod_map[a]].q;
    const bool fast_lift = (tb.fp_mods >> job.smod_map[a]) & 1;
    // raw residues (wide source) or the centred lift as exact doubles (fast path), 16 per thread
    uint64_t v[16];
#pragma unroll
    for (int e = 0; e < 16; e++) v[e] = __ldg(src + (long long)16 * e * M2);
    if (fast_lift) {
        const uint64_t half = Qs >> 1;
#pragma unroll
        for (int e = 0; e < 16; e++) {
            // signed s = v - Qs [v > Qs/2], |s| < 2^49, exact as a double via the 1.5 2^52 bias
            const long long s = (long long)v[e] - (v[e] > half ? (long long)Qs : 0ll);
            v[e] = (uint64_t)__double_as_longlong(
                __dsub_rn(__longlong_as_double(s + 0x4338000000000000ll), 6755399441055744.0));
        }
    }
    const int b_end = min(job.nb, (bc + 1) * bchunk);
    // FP64 output primes first (the lifted digit stays in registers); each prime's 255 pass-1
    // twiddles are staged into shared memory by cp.async one prime ahead (triple buffer: the
    // buffer being filled is never one a lagging thread still reads)
    double* tws = reinterpret_cast<double*>(sm + 16 * G::STRIDE);   // [3][256] after the tile
    auto next_fp = [&](int b) {
        for (; b < b_end; b++)
            if (!(job.skip_diag && b == a) && ((tb.fp_mods >> job.mod_map[b]) & 1)) return b;
        return b_end;
    };
    auto issue_tw = [&](int b, int buf) {
        const double* twg = tb.fwd_d + ((long long)job.mod_map[b] << tb.log_n);
        const unsigned sa = (unsigned)__cvta_generic_to_shared(tws + buf * 256 + threadIdx.x);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(twg + threadIdx.x) : "memory");
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    int bcur = next_fp(bc * bchunk);
    if (bcur < b_end) issue_tw(bcur, 0);
    for (int i = 0; bcur < b_end; i++) {
        const int bnext = next_fp(bcur + 1);
        if (bnext < b_end) {
            issue_tw(bnext, (i + 1) % 3);
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        const int b = bcur;
        const int mi = job.mod_map[b];
        uint64_t* dst = job.dst[z] + a * job.dst_a + b * job.dst_b + col0 + g;
        double r[16];
        if (fast_lift) {
#pragma unroll
            for (int e = 0; e < 16; e++) r[e] = __longlong_as_double((long long)v[e]);
        } else {
            const Mod md = tb.mods[mi];
#pragma unroll
            for (int e = 0; e < 16; e++) r[e] = u2d(lift_centered(v[e], Qs, md));
        }
        const double2 qd = tb.modd[mi];
        const double* twp = tws + (i % 3) * 256;
        double* tile = reinterpret_cast<double*>(sm);
        __syncthreads();   // this prime's twiddles landed; the previous prime's exchange reads are done
        col_phase16<double, true, true>(r, 0, 0, twp, qd.x, qd.y, 0);
#pragma unroll
        for (int e = 0; e < 16; e++) tile[G::addr(g, t + 16 * e)] = r[e];
        __syncthreads();
#pragma unroll
        for (int e = 0; e < 16; e++) r[e] = tile[G::addr(g, 16 * t + e)];
        col_phase16<double, true, true>(r, 4, t, twp, qd.x, qd.y, 0);
#pragma unroll
        for (int e = 0; e < 16; e++) dst[(long long)(16 * t + e) * M2] = (uint64_t)__double_as_longlong(r[e]);
        bcur = bnext;
    }
    // ... then the integer-engine ones (60-bit: the special prime), reloading the digit (L1 / L2)
    for (int b = bc * bchunk; b < b_end; b++) {
        if (job.skip_diag && b == a) continue;
        const int mi = job.mod_map[b];
        if ((tb.fp_mods >> mi) & 1) continue;
        const Mod md = tb.mods[mi];
        uint64_t* dst = job.dst[z] + a * job.dst_a + b * job.dst_b + col0 + g;
        uint64_t r[16];
        if (Qs < md.q) {   // a narrower source (every q_j into the 60-bit p): the centred lift is s or s + q
            const uint64_t half = Qs >> 1, dq = md.q - Qs;
#pragma unroll
            for (int e = 0; e < 16; e++) {
                const uint64_t w = __ldg(src + (long long)16 * e * M2);
                r[e] = w > half ? w + dq : w;
            }
        } else {
#pragma unroll
            for (int e = 0; e < 16; e++) r[e] = lift_centered(__ldg(src + (long long)16 * e * M2), Qs, md);
        }
        const void* twp = tb.fwd + ((long long)mi << tb.log_n);
        col_phase16<uint64_t, false>(r, 0, 0, twp, 0.0, 0.0, md.q);
        uint64_t* tile = sm;
        __syncthreads();
#pragma unroll
        for (int e = 0; e < 16; e++) tile[G::addr(g, t + 16 * e)] = r[e];
        __syncthreads();
#pragma unroll
        for (int e = 0; e < 16; e++) r[e] = tile[G::addr(g, 16 * t + e)];
        col_phase16<uint64_t, false>(r, 4, t, twp, 0.0, 0.0, md.q);
#pragma unroll
        for (int e = 0; e < 16; e++) dst[(long long)(16 * t + e) * M2] = r[e];
    }
}

// forward pass 2 for M2 = 256, radix-16, register-direct load: thread (g = tid / 16, t = tid % 16)
// of a 16-row tile loads elements t + 16e of row g straight into registers (two 128-byte segments
// per warp load), phase 1 in registers, one exchange, phase 2, then the results go through the
// shared tile once more so the (combining) stores stay coalesced.
template <bool FP, int STOREMODE>
__device__ __forceinline__ void fwd_rows_r16_body(const PassJob& job, const Tables& tb, const uint64_t* src,
                                                  uint64_t* dst, int mi, const Mod& md, int a, int b, int z,
                                                  int row0, long long off0) {
    using G = Geo<8, 4>;
    extern __shared__ uint64_t sm[];
    const int g = threadIdx.x >> 4, t = threadIdx.x & 15;
    using V = typename std::conditional<FP, double, uint64_t>::type;
    V r[16];
#pragma unroll
    for (int e = 0; e < 16; e++) {
        const uint64_t w = __ldg(&src[g * 256 + t + 16 * e]);
        if constexpr (FP) r[e] = __longlong_as_double((long long)w);   // lazy pass-1 doubles
        else r[e] = w;
    }
    if (STOREMODE == STORE_COMBINE) {
        // the combine's operands (acc, addend) pulled into L2 now, consumed after both phases
        // (ncu, profiles/r2_ncu_mdrows_v1.txt: 58 % of stall samples waited on these loads)
        const uint64_t* aux = job.aux[z] + a * job.aux_a + b * job.aux_b + off0;
        const bool has_add = job.add[z] != nullptr && a < job.aux_limit;
        const uint64_t* add = has_add ? job.add[z] + a * job.add_a + b * job.add_b + off0 : nullptr;
        {   // one 128-byte line per thread per array: 256 x 128 B = the 16-row tile
            const int i = 16 * threadIdx.x;
            asm volatile("prefetch.global.L2 [%0];" ::"l"(aux + i));
            if (has_add) asm volatile("prefetch.global.L2 [%0];" ::"l"(add + i));
        }
    }
    const double2 qd = FP ? tb.modd[mi] : make_double2(0, 0);
    const void* twp = FP ? (const void*)(tb.fwd_d + ((long long)mi << tb.log_n))
                         : (const void*)(tb.fwd + ((long long)mi << tb.log_n));
    const int s0 = tb.log_n - 8;
    const uint32_t high = (uint32_t)(row0 + g);
    col_phase16<V, FP>(r, 0, 0, twp, qd.x, qd.y, md.q, s0, high);
    V* tile = reinterpret_cast<V*>(sm);
#pragma unroll
    for (int e = 0; e < 16; e++) tile[G::addr(g, t + 16 * e)] = r[e];
    __syncthreads();
#pragma unroll
    for (int e = 0; e < 16; e++) r[e] = tile[G::addr(g, 16 * t + e)];
    col_phase16<V, FP>(r, 4, t, twp, qd.x, qd.y, md.q, s0, high);
#pragma unroll
    for (int e = 0; e < 16; e++) tile[G::addr(g, 16 * t + e)] = r[e];
    __syncthreads();
    auto canon = [&](int idx) -> uint64_t {
        if constexpr (FP) return d_canon(tile[idx], qd.x, qd.y);
        else return reduce4(tile[idx], md.q);
    };
    // word pairs (i, i + 1) of one row: 16-byte loads of the combine inputs and 16-byte stores
    if (STOREMODE == STORE_PLAIN) {
#pragma unroll 4
        for (int k = 0; k < 8; k++) {
            const int i = 2 * (threadIdx.x + k * 256);
            *reinterpret_cast<ulonglong2*>(dst + i) =
                make_ulonglong2(canon(G::addr(i >> 8, i & 255)), canon(G::addr(i >> 8, (i & 255) + 1)));
        }
    } else if (FP) {
        // combine on the FP64 pipe: (acc - v) c mod q with c = p^-1 (or q_l^-1) centred, exact
        // (acc < q, |v| <= 2.41 q after the lazy last stage: |acc - v| < 3.41 q, |c| <= q/2 ->
        // |mulred| <= 1.14 q; + addend < q), then one canonical reduction
        const uint64_t* aux = job.aux[z] + a * job.aux_a + b * job.aux_b + off0;
        const ulonglong2 cm = tb.comb[mi];
        const double q = qd.x, qinv = qd.y;
        double cd = u2d(cm.x);
        cd = cd > 0.5 * q ? __dsub_rn(cd, q) : cd;
        const bool has_add = job.add[z] != nullptr && a < job.aux_limit;
        const uint64_t* add = has_add ? job.add[z] + a * job.add_a + b * job.add_b + off0 : nullptr;
        const double* dtile = reinterpret_cast<const double*>(tile);
#pragma unroll 4
        for (int k = 0; k < 8; k++) {
            const int i = 2 * (threadIdx.x + k * 256);
            const ulonglong2 ax = *reinterpret_cast<const ulonglong2*>(aux + i);
            double r0 = mulred(__dsub_rn(u2d(ax.x), dtile[G::addr(i >> 8, i & 255)]), cd, q, qinv);
            double r1 = mulred(__dsub_rn(u2d(ax.y), dtile[G::addr(i >> 8, (i & 255) + 1)]), cd, q, qinv);
            if (has_add) {
                const ulonglong2 ad = *reinterpret_cast<const ulonglong2*>(add + i);
                r0 = __dadd_rn(r0, u2d(ad.x));
                r1 = __dadd_rn(r1, u2d(ad.y));
            }
            *reinterpret_cast<ulonglong2*>(dst + i) = make_ulonglong2(d_canon(r0, q, qinv), d_canon(r1, q, qinv));
        }
    } else {
        const uint64_t* aux = job.aux[z] + a * job.aux_a + b * job.aux_b + off0;
        const ulonglong2 cm = tb.comb[mi];
        const bool has_add = job.add[z] != nullptr && a < job.aux_limit;
        const uint64_t* add = has_add ? job.add[z] + a * job.add_a + b * job.add_b + off0 : nullptr;
#pragma unroll 4
        for (int k = 0; k < 8; k++) {
            const int i = 2 * (threadIdx.x + k * 256);
            const ulonglong2 ax = *reinterpret_cast<const ulonglong2*>(aux + i);
            const uint64_t v0 = canon(G::addr(i >> 8, i & 255)), v1 = canon(G::addr(i >> 8, (i & 255) + 1));
            uint64_t r0 = mul_shoup(sub_mod(ax.x, v0, md.q), cm.x, cm.y, md.q);
            uint64_t r1 = mul_shoup(sub_mod(ax.y, v1, md.q), cm.x, cm.y, md.q);
            if (has_add) {
                const ulonglong2 ad = *reinterpret_cast<const ulonglong2*>(add + i);
                r0 = add_mod(r0, ad.x, md.q);
                r1 = add_mod(r1, ad.y, md.q);
            }
            *reinterpret_cast<ulonglong2*>(dst + i) = make_ulonglong2(r0, r1);
        }
    }
}

template <int STOREMODE>
__global__ void __launch_bounds__(256, 4) k_fwd_rows_r16(PassJob job, Tables tb) {
    int a, b;
    if (!job_limb(job, a, b)) return;
    const int z = blockIdx.z;
    const int row0 = blockIdx.x * 16;
    const int mi = job.mod_map[b];
    const Mod md = tb.mods[mi];
    const long long off0 = (long long)row0 << 8;
    const uint64_t* src = job.src[z] + a * job.src_a + b * job.src_b + off0;
    uint64_t* dst = job.dst[z] + a * job.dst_a + b * job.dst_b + off0;
    if (use_f64(md.q, tb)) fwd_rows_r16_body<true, STOREMODE>(job, tb, src, dst, mi, md, a, b, z, row0, off0);
    else fwd_rows_r16_body<false, STOREMODE>(job, tb, src, dst, mi, md, a, b, z, row0, off0);
}

// inverse pass B for M1 = 256, register-direct (the mirror of k_fwd_cols_r16): thread (g = tid % 16,
// t = tid / 16) loads rows 16 t + e of column g (inverse phase 1's operands, two 128-byte segments
// per warp load), one exchange, phase 2 on rows t + 16 e, N^-1 and the full reduction in
// registers, coalesced stores.
template <typename V, bool FP>
__device__ __forceinline__ void inv_phase16(V (&r)[16], int b0, int ohigh, const void* twp, double q, double qinv,
                                            uint64_t qi, int v0, int log_n) {
#pragma unroll
    for (int uu = 0; uu < 4; uu++) {
        const int bit = b0 + uu;
        const int v = v0 + bit;
        const int dist = 1 << uu;
        const uint32_t tbase = (1u << (log_n - v - 1)) + ((uint32_t)ohigh << (4 - uu - 1));
#pragma unroll
        for (int k = 0; k < 8; k++) {
            if (k >= (1 << (4 - uu - 1))) break;
            if constexpr (FP) {
                const double W = __ldg(reinterpret_cast<const double*>(twp) + tbase + k);
#pragma unroll
                for (int e0 = 0; e0 < 8; e0++) {
                    if (e0 >= dist) break;
                    const int e = k * 2 * dist + e0;
                    const double X = r[e], Y = r[e + dist];
                    r[e] = redd(__dadd_rn(X, Y), q, qinv);
                    r[e + dist] = mulred(redd(__dsub_rn(X, Y), q, qinv), W, q, qinv);
                }
            } else {
                const ulonglong2 W = __ldg(reinterpret_cast<const ulonglong2*>(twp) + tbase + k);
                const uint64_t q2 = 2 * qi;
#pragma unroll
                for (int e0 = 0; e0 < 8; e0++) {
                    if (e0 >= dist) break;
                    const int e = k * 2 * dist + e0;
                    const uint64_t X = r[e], Y = r[e + dist];
                    const uint64_t sm_ = X + Y;
                    r[e] = sm_ >= q2 ? sm_ - q2 : sm_;
                    r[e + dist] = mul_shoup_lazy(X - Y + q2, W.x, W.y, qi);
                }
            }
        }
    }
}

template <bool FP>
__device__ __forceinline__ void inv_cols_r16_body(const Tables& tb, const uint64_t* src, uint64_t* dst, int mi,
                                                  const Mod& md, int col0, int M2) {
    using G = Geo<8, 4>;
    extern __shared__ uint64_t sm[];
    const int g = threadIdx.x & 15, t = threadIdx.x >> 4;
    using V = typename std::conditional<FP, double, uint64_t>::type;
    V r[16];
#pragma unroll
    for (int e = 0; e < 16; e++) {
        const uint64_t w = __ldg(&src[(long long)(16 * t + e) * M2 + col0 + g]);
        if constexpr (FP) r[e] = __longlong_as_double((long long)w);
        else r[e] = w;
    }
    const double2 qd = FP ? tb.modd[mi] : make_double2(0, 0);
    const void* twp = FP ? (const void*)(tb.inv_d + ((long long)mi << tb.log_n))
                         : (const void*)(tb.inv + ((long long)mi << tb.log_n));
    const int v0 = tb.log_n - 8;
    inv_phase16<V, FP>(r, 0, t, twp, qd.x, qd.y, md.q, v0, tb.log_n);
    V* tile = reinterpret_cast<V*>(sm);
#pragma unroll
    for (int e = 0; e < 16; e++) tile[G::addr(g, 16 * t + e)] = r[e];
    __syncthreads();
#pragma unroll
    for (int e = 0; e < 16; e++) r[e] = tile[G::addr(g, t + 16 * e)];
    inv_phase16<V, FP>(r, 4, 0, twp, qd.x, qd.y, md.q, v0, tb.log_n);
    if constexpr (FP) {
        const double ni = tb.ninv_d[mi];
#pragma unroll
        for (int e = 0; e < 16; e++)
            dst[(long long)(t + 16 * e) * M2 + col0 + g] = d_canon(mulred(r[e], ni, qd.x, qd.y), qd.x, qd.y);
    } else {
        const ulonglong2 ni = tb.ninv[mi];
#pragma unroll
        for (int e = 0; e < 16; e++) dst[(long long)(t + 16 * e) * M2 + col0 + g] = mul_shoup(r[e], ni.x, ni.y, md.q);
    }
}

__global__ void __launch_bounds__(256, 4) k_inv_cols_r16(PassJob job, Tables tb) {
    int a, b;
    if (!job_limb(job, a, b)) return;
    const int z = blockIdx.z;
    const int M2 = 1 << (tb.log_n - 8);
    const int col0 = blockIdx.x * 16;
    const int mi = job.mod_map[b];
    const Mod md = tb.mods[mi];
    const uint64_t* src = job.src[z] + a * job.src_a + b * job.src_b;
    uint64_t* dst = job.dst[z] + a * job.dst_a + b * job.dst_b;
    if (use_f64(md.q, tb)) inv_cols_r16_body<true>(tb, src, dst, mi, md, col0, M2);
    else inv_cols_r16_body<false>(tb, src, dst, mi, md, col0, M2);
}

// ------------------------------------------------------------------------------------------
// forward pass 2: rows (contiguous).  Tile = Gr consecutive rows of M = M2 words.  Input = the
// lazy pass-1 output.  STORE_PLAIN: full reduction.  STORE_COMBINE: out = (aux - v) * comb[mod]
// (+ add if a < aux_limit).
// ------------------------------------------------------------------------------------------
template <int LOG_M, int LOG_R, int STOREMODE, int MINB, int FULL = 0>
__global__ void __launch_bounds__(256, MINB) k_fwd_rows(PassJob job, Tables tb) {
    using G = Geo<LOG_M, LOG_R>;
    extern __shared__ uint64_t sm[];
    int a, b;
    if (!job_limb(job, a, b)) return;
    const int z = blockIdx.z;
    const int log_n = tb.log_n;
    const int Gr = FULL ? 256 / G::T : blockDim.x / G::T;
    const int row0 = blockIdx.x * Gr;
    const int mi = job.mod_map[b];
    const Mod md = tb.mods[mi];
    const bool fp = use_f64(md.q, tb);
    const long long off0 = (long long)row0 << LOG_M;
    const uint64_t* src = job.src[z] + a * job.src_a + b * job.src_b + off0;
    uint64_t* dst = job.dst[z] + a * job.dst_a + b * job.dst_b + off0;
    const int nthr = FULL ? 256 : blockDim.x;   // FULL: compile-time, offsets fold
#pragma unroll 4
    for (int k = 0; k < G::R; k++) {
        const int i = threadIdx.x + k * nthr;
        cp_async8(&sm[G::addr(i >> LOG_M, i & (G::M - 1))], &src[i]);
    }
    cp_async_wait_all();
    __syncthreads();
    int g, t;
    tile_coords<LOG_M, LOG_R>(g, t);
    const int s0 = log_n - LOG_M;
    double2 qd = make_double2(0, 0);
    if (fp) {
        qd = tb.modd[mi];
        fwd_engine_f64<LOG_M, LOG_R>(reinterpret_cast<double*>(sm), qd.x, qd.y, tb.fwd_d + ((long long)mi << log_n),
                                     s0, (uint32_t)(row0 + g), g, t);
    } else {
        fwd_engine<LOG_M, LOG_R>(sm, md.q, tb.fwd + ((long long)mi << log_n), s0, (uint32_t)(row0 + g), g, t);
    }
    auto canon = [&](int idx) -> uint64_t {
        const uint64_t w = sm[idx];
        return fp ? d_canon(__longlong_as_double((long long)w), qd.x, qd.y) : reduce4(w, md.q);
    };
    if (STOREMODE == STORE_PLAIN) {
#pragma unroll 4
        for (int k = 0; k < G::R; k++) {
            const int i = threadIdx.x + k * nthr;
            dst[i] = canon(G::addr(i >> LOG_M, i & (G::M - 1)));
        }
    } else {
        const uint64_t* aux = job.aux[z] + a * job.aux_a + b * job.aux_b + off0;
        const ulonglong2 cm = tb.comb[mi];
        const bool has_add = job.add[z] != nullptr && a < job.aux_limit;
        const uint64_t* add = has_add ? job.add[z] + a * job.add_a + b * job.add_b + off0 : nullptr;
#pragma unroll 4
        for (int k = 0; k < G::R; k++) {
            const int i = threadIdx.x + k * nthr;
            const uint64_t v = canon(G::addr(i >> LOG_M, i & (G::M - 1)));
            uint64_t r = mul_shoup(sub_mod(aux[i], v, md.q), cm.x, cm.y, md.q);
            if (has_add) r = add_mod(r, add[i], md.q);
            dst[i] = r;
        }
    }
}

// ------------------------------------------------------------------------------------------
// inverse pass A: rows; input canonical; stores lazily (int: [0, 2q); FP64: centred doubles)
// ------------------------------------------------------------------------------------------
template <int LOG_M, int LOG_R, int MINB, int FULL = 0>
__global__ void __launch_bounds__(256, MINB) k_inv_rows(PassJob job, Tables tb) {
    using G = Geo<LOG_M, LOG_R>;
    extern __shared__ uint64_t sm[];
    int a, b;
    if (!job_limb(job, a, b)) return;
    const int z = blockIdx.z;
    const int log_n = tb.log_n;
    const int Gr = FULL ? 256 / G::T : blockDim.x / G::T;
    const int row0 = blockIdx.x * Gr;
    const int mi = job.mod_map[b];
    const Mod md = tb.mods[mi];
    const bool fp = use_f64(md.q, tb);
    const long long off0 = (long long)row0 << LOG_M;
    const uint64_t* src = job.src[z] + a * job.src_a + b * job.src_b + off0;
    uint64_t* dst = job.dst[z] + a * job.dst_a + b * job.dst_b + off0;
    const int nthr = FULL ? 256 : blockDim.x;   // FULL: compile-time, offsets fold
    if (fp) {   // FP64 limb: loads straight into registers, converted, stored once
        uint64_t v[G::R];
#pragma unroll
        for (int k = 0; k < G::R; k++) v[k] = __ldg(&src[threadIdx.x + k * nthr]);
#pragma unroll
        for (int k = 0; k < G::R; k++) {
            const int i = threadIdx.x + k * nthr;
            reinterpret_cast<double*>(sm)[G::addr(i >> LOG_M, i & (G::M - 1))] = u2d(v[k]);
        }
    } else {
#pragma unroll 4
        for (int k = 0; k < G::R; k++) {
            const int i = threadIdx.x + k * nthr;
            cp_async8(&sm[G::addr(i >> LOG_M, i & (G::M - 1))], &src[i]);
        }
        cp_async_wait_all();
    }
    __syncthreads();
    int g, t;
    tile_coords<LOG_M, LOG_R>(g, t);
    if (fp) {
        const double2 qd = tb.modd[mi];
        inv_engine_f64<LOG_M, LOG_R>(reinterpret_cast<double*>(sm), qd.x, qd.y, tb.inv_d + ((long long)mi << log_n),
                                     0, log_n, (uint32_t)(row0 + g), g, t);
    } else {
        inv_engine<LOG_M, LOG_R>(sm, md.q, tb.inv + ((long long)mi << log_n), 0, log_n, (uint32_t)(row0 + g), g, t);
    }
#pragma unroll 4
    for (int k = 0; k < G::R; k++) {
        const int i = threadIdx.x + k * nthr;
        dst[i] = sm[G::addr(i >> LOG_M, i & (G::M - 1))];
    }
}

// ------------------------------------------------------------------------------------------
// inverse pass B: columns; multiplies by N^-1 and fully reduces.
// ------------------------------------------------------------------------------------------
template <int LOG_M, int LOG_R, int MINB, int GC = 0>
__global__ void __launch_bounds__(256, MINB) k_inv_cols(PassJob job, Tables tb) {
    using G = Geo<LOG_M, LOG_R>;
    extern __shared__ uint64_t sm[];
    int a, b;
    if (!job_limb(job, a, b)) return;
    const int z = blockIdx.z;
    const int log_n = tb.log_n;
    const int M2 = 1 << (log_n - LOG_M);
    const int Gc = GC > 0 ? GC : blockDim.x / G::T;
    const int col0 = blockIdx.x * Gc;
    const int mi = job.mod_map[b];
    const Mod md = tb.mods[mi];
    const bool fp = use_f64(md.q, tb);
    const uint64_t* src = job.src[z] + a * job.src_a + b * job.src_b;
    uint64_t* dst = job.dst[z] + a * job.dst_a + b * job.dst_b;
    const int nthr = GC > 0 ? GC * G::T : blockDim.x;
    const int lg = GC > 0 ? ilog2c(GC) : __ffs(Gc) - 1;
#pragma unroll 4
    for (int k = 0; k < G::R; k++) {
        const int i = threadIdx.x + k * nthr;
        cp_async8(&sm[G::addr(i & (Gc - 1), i >> lg)], &src[(long long)(i >> lg) * M2 + col0 + (i & (Gc - 1))]);
    }
    cp_async_wait_all();
    __syncthreads();
    int g, t;
    tile_coords<LOG_M, LOG_R>(g, t);
    if (fp) {
        const double2 qd = tb.modd[mi];
        inv_engine_f64<LOG_M, LOG_R>(reinterpret_cast<double*>(sm), qd.x, qd.y, tb.inv_d + ((long long)mi << log_n),
                                     log_n - LOG_M, log_n, 0, g, t);
        const double ni = tb.ninv_d[mi];
#pragma unroll 4
        for (int k = 0; k < G::R; k++) {
            const int i = threadIdx.x + k * nthr;
            const double v = reinterpret_cast<const double*>(sm)[G::addr(i & (Gc - 1), i >> lg)];
            dst[(long long)(i >> lg) * M2 + col0 + (i & (Gc - 1))] = d_canon(mulred(v, ni, qd.x, qd.y), qd.x, qd.y);
        }
    } else {
        inv_engine<LOG_M, LOG_R>(sm, md.q, tb.inv + ((long long)mi << log_n), log_n - LOG_M, log_n, 0, g, t);
        const ulonglong2 ni = tb.ninv[mi];
#pragma unroll 4
        for (int k = 0; k < G::R; k++) {
            const int i = threadIdx.x + k * nthr;
            dst[(long long)(i >> lg) * M2 + col0 + (i & (Gc - 1))] =
                mul_shoup(sm[G::addr(i & (Gc - 1), i >> lg)], ni.x, ni.y, md.q);
        }
    }
}

// ------------------------------------------------------------------------------------------
// host launchers: radix of the engine phases (LOG_R) and the __launch_bounds__ minimum blocks
// per SM, tuned on B200.
// ------------------------------------------------------------------------------------------

template <int LOG_M, int LOG_R>
static void launch_geom(int log_m_other, int& threads, int& gx, size_t& smem) {
    using G = Geo<LOG_M, LOG_R>;
    int groups_per_limb = 1 << log_m_other;
    int gpc = 256 / G::T;
    if (gpc > groups_per_limb) gpc = groups_per_limb;
    threads = gpc * G::T;
    gx = groups_per_limb / gpc;
    smem = (size_t)gpc * G::STRIDE * sizeof(uint64_t);
}

template <int LOG_M, int LOG_R, int MINB>
static cudaError_t fwd_cols_v(const PassJob& job, const Tables& tb, int nlimbs, int nz, int lift, cudaStream_t st) {
    int threads, gx; size_t smem;
    launch_geom<LOG_M, LOG_R>(tb.log_n - LOG_M, threads, gx, smem);
    dim3 grid(gx, nlimbs, nz);
    constexpr int FULL = 256 / Geo<LOG_M, LOG_R>::T;
    const bool full = threads == 256;
    if constexpr (LOG_M == 8 && LOG_R == 4) {
        if (full && lift && job.nb > 1 && tb.log_n == 16) {
            // ModUp (and any multi-target lift): one CTA per (column block, source limb, chunk of
            // output primes); chunks sized for >= ~4 CTAs per SM-slot wave
            const int na = nlimbs / job.nb;
            int bchunk = job.nb;
            while (bchunk > 4 && (long long)gx * na * ((job.nb + bchunk - 1) / bchunk) * nz < 4 * 148 * 4) bchunk = (bchunk + 1) / 2;
            const int nbc = (job.nb + bchunk - 1) / bchunk;
            dim3 g2(gx, na * nbc, nz);
            k_modup_cols16<MODUP_MINB><<<g2, 256, smem + 3 * 256 * sizeof(double), st>>>(job, tb, bchunk, nbc);
            return cudaGetLastError();
        }
        if (full) {   // register-direct radix-16 form
            if (lift) k_fwd_cols_r16<LOAD_LIFT, 4><<<grid, 256, smem, st>>>(job, tb);   // MINB 3: slower
            else k_fwd_cols_r16<LOAD_PLAIN, 4><<<grid, 256, smem, st>>>(job, tb);
            return cudaGetLastError();
        }
    }
    if (lift) {
        if (full) k_fwd_cols<LOG_M, LOG_R, LOAD_LIFT, MINB, FULL><<<grid, threads, smem, st>>>(job, tb);
        else k_fwd_cols<LOG_M, LOG_R, LOAD_LIFT, MINB><<<grid, threads, smem, st>>>(job, tb);
    } else {
        if (full) k_fwd_cols<LOG_M, LOG_R, LOAD_PLAIN, MINB, FULL><<<grid, threads, smem, st>>>(job, tb);
        else k_fwd_cols<LOG_M, LOG_R, LOAD_PLAIN, MINB><<<grid, threads, smem, st>>>(job, tb);
    }
    return cudaGetLastError();
}
template <int LOG_M, int LOG_R, int MINB>
static cudaError_t fwd_rows_v(const PassJob& job, const Tables& tb, int nlimbs, int nz, int combine, cudaStream_t st) {
    int threads, gx; size_t smem;
    launch_geom<LOG_M, LOG_R>(tb.log_n - LOG_M, threads, gx, smem);
    dim3 grid(gx, nlimbs, nz);
    if constexpr (LOG_M == 8 && LOG_R == 4) {
        if (threads == 256) {   // register-direct radix-16 form
            if (combine) k_fwd_rows_r16<STORE_COMBINE><<<grid, 256, smem, st>>>(job, tb);
            else k_fwd_rows_r16<STORE_PLAIN><<<grid, 256, smem, st>>>(job, tb);
            return cudaGetLastError();
        }
    }
    if (threads == 256) {
        if (combine) k_fwd_rows<LOG_M, LOG_R, STORE_COMBINE, MINB, 1><<<grid, threads, smem, st>>>(job, tb);
        else k_fwd_rows<LOG_M, LOG_R, STORE_PLAIN, MINB, 1><<<grid, threads, smem, st>>>(job, tb);
    } else {
        if (combine) k_fwd_rows<LOG_M, LOG_R, STORE_COMBINE, MINB><<<grid, threads, smem, st>>>(job, tb);
        else k_fwd_rows<LOG_M, LOG_R, STORE_PLAIN, MINB><<<grid, threads, smem, st>>>(job, tb);
    }
    return cudaGetLastError();
}
template <int LOG_M, int LOG_R, int MINB>
static cudaError_t inv_rows_v(const PassJob& job, const Tables& tb, int nlimbs, int nz, cudaStream_t st) {
    int threads, gx; size_t smem;
    launch_geom<LOG_M, LOG_R>(tb.log_n - LOG_M, threads, gx, smem);
    dim3 grid(gx, nlimbs, nz);
    if (threads == 256) k_inv_rows<LOG_M, LOG_R, MINB, 1><<<grid, threads, smem, st>>>(job, tb);
    else k_inv_rows<LOG_M, LOG_R, MINB><<<grid, threads, smem, st>>>(job, tb);
    return cudaGetLastError();
}
template <int LOG_M, int LOG_R, int MINB>
static cudaError_t inv_cols_v(const PassJob& job, const Tables& tb, int nlimbs, int nz, cudaStream_t st) {
    int threads, gx; size_t smem;
    launch_geom<LOG_M, LOG_R>(tb.log_n - LOG_M, threads, gx, smem);
    dim3 grid(gx, nlimbs, nz);
    constexpr int FULL = 256 / Geo<LOG_M, LOG_R>::T;
    if constexpr (LOG_M == 8 && LOG_R == 4) {
        if (threads == 256) {   // register-direct radix-16 form
            k_inv_cols_r16<<<grid, 256, smem, st>>>(job, tb);
            return cudaGetLastError();
        }
    }
    if (threads == 256) k_inv_cols<LOG_M, LOG_R, MINB, FULL><<<grid, threads, smem, st>>>(job, tb);
    else k_inv_cols<LOG_M, LOG_R, MINB><<<grid, threads, smem, st>>>(job, tb);
    return cudaGetLastError();
}
// radix-16 phases, __launch_bounds__(256, 4): measured best (MINB 1 / radix-4 variants removed,
// profiles/r1_ks_variants.txt); at M = 256 with full 256-thread CTAs the register-direct forms run
#define NTT_DISPATCH(FN, ...) return FN<LM, 4, 4>(__VA_ARGS__);
template <int LM>
static cudaError_t fwd_cols_t(const PassJob& job, const Tables& tb, int nlimbs, int nz, int lift, cudaStream_t st) {
    NTT_DISPATCH(fwd_cols_v, job, tb, nlimbs, nz, lift, st)
}
template <int LM>
static cudaError_t fwd_rows_t(const PassJob& job, const Tables& tb, int nlimbs, int nz, int combine, cudaStream_t st) {
    NTT_DISPATCH(fwd_rows_v, job, tb, nlimbs, nz, combine, st)
}
template <int LM>
static cudaError_t inv_rows_t(const PassJob& job, const Tables& tb, int nlimbs, int nz, cudaStream_t st) {
    NTT_DISPATCH(inv_rows_v, job, tb, nlimbs, nz, st)
}
template <int LM>
static cudaError_t inv_cols_t(const PassJob& job, const Tables& tb, int nlimbs, int nz, cudaStream_t st) {
    NTT_DISPATCH(inv_cols_v, job, tb, nlimbs, nz, st)
}
#undef NTT_DISPATCH

int split_m1(int log_n) { return log_n / 2; }

cudaError_t launch_fwd_pass1(const PassJob& job, const Tables& tb, int nlimbs, int nz, bool lift, cudaStream_t st) {
    const int lm = split_m1(tb.log_n);
#define C(LM) fwd_cols_t<LM>(job, tb, nlimbs, nz, lift, st)
    switch (lm) { case 4: return C(4); case 5: return C(5); case 6: return C(6); case 7: return C(7); case 8: return C(8); }
#undef C
    return cudaErrorInvalidValue;
}
cudaError_t launch_fwd_pass2(const PassJob& job, const Tables& tb, int nlimbs, int nz, bool combine, cudaStream_t st) {
    const int lm = tb.log_n - split_m1(tb.log_n);
#define C(LM) fwd_rows_t<LM>(job, tb, nlimbs, nz, combine, st)
    switch (lm) { case 4: return C(4); case 5: return C(5); case 6: return C(6); case 7: return C(7); case 8: return C(8); }
#undef C
    return cudaErrorInvalidValue;
}
cudaError_t launch_inv_passA(const PassJob& job, const Tables& tb, int nlimbs, int nz, cudaStream_t st) {
    const int lm = tb.log_n - split_m1(tb.log_n);
#define C(LM) inv_rows_t<LM>(job, tb, nlimbs, nz, st)
    switch (lm) { case 4: return C(4); case 5: return C(5); case 6: return C(6); case 7: return C(7); case 8: return C(8); }
#undef C
    return cudaErrorInvalidValue;
}
cudaError_t launch_inv_passB(const PassJob& job, const Tables& tb, int nlimbs, int nz, cudaStream_t st) {
    const int lm = split_m1(tb.log_n);
#define C(LM) inv_cols_t<LM>(job, tb, nlimbs, nz, st)
    switch (lm) { case 4: return C(4); case 5: return C(5); case 6: return C(6); case 7: return C(7); case 8: return C(8); }
#undef C
    return cudaErrorInvalidValue;
}

}  // namespace hisa
