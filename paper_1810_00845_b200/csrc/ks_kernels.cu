// ks_kernels.cu -- key-switch inner product fused with the forward-NTT row pass (K4, step a5).
//
// For output prime r (grid y = ri over q_0..q_l, p) and a tile of rows (grid x), loop over the
// digits j <= l: bring D_{j,r} for the tile on chip -- either the pass-1 output T1[j][ri] followed by
// the last log M2 CT stages in shared memory, or (r == q_j) the digit itself, which is already in
// the NTT domain -- then multiply with the key limbs (b and a) and accumulate in 128-bit
// registers (products < 2^122, at most 64 terms).  One Barrett reduction per output word.
// D never touches HBM in its NTT form; the key is streamed once per ciphertext.
#include <cuda_runtime.h>
#include <cstdlib>
#include <type_traits>
#include "ntt_f64.cuh"
#include "launch.h"

namespace hisa {

// Variant knobs (tuned on B200, see profiles/): LOG_R = radix of the on-chip engine phases,
// GR = rows (groups) per CTA, MINB = __launch_bounds__ min blocks.  Threads = GR * M / R,
// elements per thread in the MAC phase = R (2R 128-bit accumulators per thread).
template <int LOG_M, int LOG_R, int GR, int MINB>
__global__ void __launch_bounds__(GR * (1 << LOG_M) / (1 << LOG_R), MINB) k_ks_ip(KsJob job, Tables tb) {
    using G = Geo<LOG_M, LOG_R>;
    extern __shared__ uint64_t sm[];
    // GR == 1, FP64 engine: the row's 2^LOG_M - 1 twiddles are the same for every digit j ->
    // staged once in shared memory after the tile (no global twiddle loads in the j loop)
    double* tws = reinterpret_cast<double*>(sm + GR * G::STRIDE);
    // ciphertext index fastest: CTAs that read the same key tile are scheduled together (L2 reuse)
    const int nz = job.nz;
    const int z = blockIdx.x % nz;
    const int ri = blockIdx.y;
    const int l1 = job.l1;
    const int nri = l1 + 1;
    const int log_n = tb.log_n;
    const int row0 = (blockIdx.x / nz) * GR;
    const long long off0 = (long long)row0 << LOG_M;
    const int mi = job.mod_map[ri];
    const Mod md = tb.mods[mi];
    const bool fp = (double)md.q < tb.f64_max_q;
    const double2 qd = fp ? tb.modd[mi] : make_double2(0, 0);
    const double qp52 = __dadd_rn(qd.x, 4503599627370496.0);
    constexpr int NTHR = GR * G::T;
    constexpr int EPT = G::R;   // elements per thread in the MAC phase (tile / threads)
    U128 acc0[EPT], acc1[EPT];
#pragma unroll
    for (int k = 0; k < EPT; k++) { acc0[k] = U128{0, 0}; acc1[k] = U128{0, 0}; }
    const int g = threadIdx.x / G::T, t = threadIdx.x % G::T;
    const long long kstride_j = 2ll * (job.L + 1) << log_n;
    const long long kstride_p = (long long)(job.L + 1) << log_n;
    const uint64_t* key_r = job.key + ((long long)mi << log_n) + off0;
    if (GR == 1 && fp) {
        const double* twg = tb.fwd_d + ((long long)mi << log_n);
        const int s0 = log_n - LOG_M;
        for (int idx = threadIdx.x + 1; idx < G::M; idx += NTHR) {
            const int u = 31 - __clz(idx), m = idx - (1 << u);
            tws[idx] = twg[(1 << (s0 + u)) + (row0 << u) + m];
        }
    }
    for (int j = 0; j < l1; j++) {
        const uint64_t* src = (j == ri) ? job.d[z] + ((long long)j << log_n) + off0
                                        : job.t1[z] + (((long long)j * nri + ri) << log_n) + off0;
#pragma unroll
        for (int k = 0; k < EPT; k++) {
            const int i = threadIdx.x + k * NTHR;
            const unsigned sa = (unsigned)__cvta_generic_to_shared(&sm[G::addr(i >> LOG_M, i & (G::M - 1))]);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(src + i) : "memory");
        }
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        __syncthreads();
        const bool conv = fp && j != ri;   // FP64-engine output: centred-lazy doubles
        if (j != ri) {
            if (fp && GR == 1)
                fwd_engine_f64_rowtw<LOG_M, LOG_R>(reinterpret_cast<double*>(sm), qd.x, qd.y, tws, t);
            else if (fp)
                fwd_engine_f64<LOG_M, LOG_R>(reinterpret_cast<double*>(sm), qd.x, qd.y,
                                             tb.fwd_d + ((long long)mi << log_n), log_n - LOG_M,
                                             (uint32_t)(row0 + g), g, t);
            else
                fwd_engine<LOG_M, LOG_R>(sm, md.q, tb.fwd + ((long long)mi << log_n), log_n - LOG_M,
                                         (uint32_t)(row0 + g), g, t);
        }
        const uint64_t* kb = key_r + j * kstride_j;
        const uint64_t* ka = kb + kstride_p;
#pragma unroll
        for (int k = 0; k < EPT; k++) {
            const int i = threadIdx.x + k * NTHR;
            uint64_t D = sm[G::addr(i >> LOG_M, i & (G::M - 1))];   // int: < 4q
            if (conv) D = d_rep(__longlong_as_double((long long)D), qd.x, qd.y, qp52);   // < 1.5q
            mac128(acc0[k], D, __ldg(kb + i));
            mac128(acc1[k], D, __ldg(ka + i));
        }
        __syncthreads();
    }
    uint64_t* out0 = job.acc[z] + ((long long)ri << log_n) + off0;
    uint64_t* out1 = job.acc[z] + ((long long)(nri + ri) << log_n) + off0;
#pragma unroll
    for (int k = 0; k < EPT; k++) {
        const int i = threadIdx.x + k * NTHR;
        out0[i] = barrett128(acc0[k].lo, acc0[k].hi, md);
        out1[i] = barrett128(acc1[k].lo, acc1[k].hi, md);
    }
}

// Software-pipelined K4 (variant P): the D tile of digit j+1 is copied into the other half of a
// double buffer (cp.async groups) and its key words are loaded into registers while digit j's
// NTT stages run, so neither the tile copy nor the key stream sits on the critical path.
template <int LOG_M, int LOG_R, int GR, int MINB>
__global__ void __launch_bounds__(GR * (1 << LOG_M) / (1 << LOG_R), MINB) k_ks_ip_pipe(KsJob job, Tables tb) {
    using G = Geo<LOG_M, LOG_R>;
    extern __shared__ uint64_t sm[];
    constexpr int TILE = GR * G::STRIDE;
    const int nz = job.nz;
    const int z = blockIdx.x % nz;
    const int ri = blockIdx.y;
    const int l1 = job.l1;
    const int nri = l1 + 1;
    const int log_n = tb.log_n;
    const int row0 = (blockIdx.x / nz) * GR;
    const long long off0 = (long long)row0 << LOG_M;
    const int mi = job.mod_map[ri];
    const Mod md = tb.mods[mi];
    const bool fp = (double)md.q < tb.f64_max_q;
    const double2 qd = fp ? tb.modd[mi] : make_double2(0, 0);
    const double qp52 = __dadd_rn(qd.x, 4503599627370496.0);
    constexpr int NTHR = GR * G::T;
    constexpr int EPT = G::R;
    U128 acc0[EPT], acc1[EPT];
#pragma unroll
    for (int k = 0; k < EPT; k++) { acc0[k] = U128{0, 0}; acc1[k] = U128{0, 0}; }
    const int g = threadIdx.x / G::T, t = threadIdx.x % G::T;
    const long long kstride_j = 2ll * (job.L + 1) << log_n;
    const long long kstride_p = (long long)(job.L + 1) << log_n;
    const uint64_t* key_r = job.key + ((long long)mi << log_n) + off0;
    auto issue_tile = [&](int j) {
        const uint64_t* src = (j == ri) ? job.d[z] + ((long long)j << log_n) + off0
                                        : job.t1[z] + (((long long)j * nri + ri) << log_n) + off0;
        uint64_t* buf = sm + (j & 1) * TILE;
#pragma unroll
        for (int k = 0; k < EPT; k++) {
            const int i = threadIdx.x + k * NTHR;
            const unsigned sa = (unsigned)__cvta_generic_to_shared(&buf[G::addr(i >> LOG_M, i & (G::M - 1))]);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(src + i) : "memory");
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    uint64_t kb_next[EPT], ka_next[EPT];
    auto load_keys = [&](int j) {
        const uint64_t* kb = key_r + j * kstride_j;
#pragma unroll
        for (int k = 0; k < EPT; k++) {
            const int i = threadIdx.x + k * NTHR;
            kb_next[k] = __ldg(kb + i);
            ka_next[k] = __ldg(kb + kstride_p + i);
        }
    };
    issue_tile(0);
    load_keys(0);
    for (int j = 0; j < l1; j++) {
        uint64_t kb_cur[EPT], ka_cur[EPT];
#pragma unroll
        for (int k = 0; k < EPT; k++) { kb_cur[k] = kb_next[k]; ka_cur[k] = ka_next[k]; }
        if (j + 1 < l1) {
            issue_tile(j + 1);
            load_keys(j + 1);
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        __syncthreads();
        uint64_t* buf = sm + (j & 1) * TILE;
        const bool conv = fp && j != ri;
        if (j != ri) {
            if (fp)
                fwd_engine_f64<LOG_M, LOG_R>(reinterpret_cast<double*>(buf), qd.x, qd.y,
                                             tb.fwd_d + ((long long)mi << log_n), log_n - LOG_M,
                                             (uint32_t)(row0 + g), g, t);
            else
                fwd_engine<LOG_M, LOG_R>(buf, md.q, tb.fwd + ((long long)mi << log_n), log_n - LOG_M,
                                         (uint32_t)(row0 + g), g, t);
        }
#pragma unroll
        for (int k = 0; k < EPT; k++) {
            const int i = threadIdx.x + k * NTHR;
            uint64_t D = buf[G::addr(i >> LOG_M, i & (G::M - 1))];
            if (conv) D = d_rep(__longlong_as_double((long long)D), qd.x, qd.y, qp52);   // < 1.5q
            mac128(acc0[k], D, kb_cur[k]);
            mac128(acc1[k], D, ka_cur[k]);
        }
        __syncthreads();   // buffer (j & 1) is refilled by iteration j + 1's prefetch of j + 2
    }
    uint64_t* out0 = job.acc[z] + ((long long)ri << log_n) + off0;
    uint64_t* out1 = job.acc[z] + ((long long)(nri + ri) << log_n) + off0;
#pragma unroll
    for (int k = 0; k < EPT; k++) {
        const int i = threadIdx.x + k * NTHR;
        out0[i] = barrett128(acc0[k].lo, acc0[k].hi, md);
        out1[i] = barrett128(acc1[k].lo, acc1[k].hi, md);
    }
}

template <int LOG_M, int LOG_R, int GR, int MINB>
static cudaError_t ks_ip_pipe_t(const KsJob& job, const Tables& tb, int nz, cudaStream_t st) {
    using G = Geo<LOG_M, LOG_R>;
    const int rows = 1 << (tb.log_n - LOG_M);
    if (rows < GR) return cudaErrorInvalidValue;
    constexpr int threads = GR * G::T;
    const size_t smem = 2 * (size_t)GR * G::STRIDE * sizeof(uint64_t);
    dim3 grid((rows / GR) * nz, job.l1 + 1, 1);
    k_ks_ip_pipe<LOG_M, LOG_R, GR, MINB><<<grid, threads, smem, st>>>(job, tb);
    return cudaGetLastError();
}

// K4 for one row per CTA with two digits in flight (variant 30, FP64 output primes): the
// non-diagonal digits j != ri are processed in pairs -- both D tiles copied, both transformed by
// one interleaved engine call (fwd_engine_f64_rowtw2, twiddles staged once in shared memory),
// both multiplied into the same 128-bit accumulators -- then the diagonal digit (already in the
// NTT domain) is multiplied in.  Integer-engine primes (q >= 2^50) fall back to one digit at a time.
template <int LOG_M, int LOG_R, int MINB, bool PF = false>
__global__ void __launch_bounds__((1 << LOG_M) / (1 << LOG_R), MINB) k_ks_ip2(KsJob job, Tables tb) {
    using G = Geo<LOG_M, LOG_R>;
    extern __shared__ uint64_t sm[];
    uint64_t* sa = sm;
    uint64_t* sb = sm + G::STRIDE;
    double* tws = reinterpret_cast<double*>(sm + 2 * G::STRIDE);
    const int nz = job.nz;
    const int z = blockIdx.x % nz;
    // the special prime's CTAs (integer engine, slower) first, so they do not form the tail
    const int ri = blockIdx.y == 0 ? job.l1 : (int)blockIdx.y - 1;
    const int l1 = job.l1;
    const int nri = l1 + 1;
    const int log_n = tb.log_n;
    const int row0 = blockIdx.x / nz;
    const long long off0 = (long long)row0 << LOG_M;
    const int mi = job.mod_map[ri];
    const Mod md = tb.mods[mi];
    const bool fp = (double)md.q < tb.f64_max_q;
    const double2 qd = fp ? tb.modd[mi] : make_double2(0, 0);
    const double tq52 = __dadd_rn(2.0 * qd.x, 4503599627370496.0);   // 2q + 2^52
    constexpr int NTHR = G::T;
    constexpr int EPT = G::R;
    U128 acc0[EPT], acc1[EPT];
#pragma unroll
    for (int k = 0; k < EPT; k++) { acc0[k] = U128{0, 0}; acc1[k] = U128{0, 0}; }
    const int t = threadIdx.x;
    const long long kstride_j = 2ll * (job.L + 1) << log_n;
    const long long kstride_p = (long long)(job.L + 1) << log_n;
    const uint64_t* key_r = job.key + ((long long)mi << log_n) + off0;
    if (fp) {
        const double* twg = tb.fwd_d + ((long long)mi << log_n);
        const int s0 = log_n - LOG_M;
        for (int idx = threadIdx.x + 1; idx < G::M; idx += NTHR) {
            const int u = 31 - __clz(idx), m = idx - (1 << u);
            tws[idx] = twg[(1 << (s0 + u)) + (row0 << u) + m];
        }
    }
    auto copy_tile = [&](uint64_t* dst, int j) {
        const uint64_t* src = (j == ri) ? job.d[z] + ((long long)j << log_n) + off0
                                        : job.t1[z] + (((long long)j * nri + ri) << log_n) + off0;
#pragma unroll
        for (int k = 0; k < EPT; k++) {
            const int i = threadIdx.x + k * NTHR;
            const unsigned s_ = (unsigned)__cvta_generic_to_shared(&dst[G::addr(0, i)]);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s_), "l"(src + i) : "memory");
        }
    };
    auto mac_tile = [&](const uint64_t* buf, int j, bool conv) {
        const uint64_t* kb = key_r + j * kstride_j;
        const uint64_t* ka = kb + kstride_p;
#pragma unroll
        for (int k = 0; k < EPT; k++) {
            const int i = threadIdx.x + k * NTHR;
            uint64_t D = buf[G::addr(0, i)];
            if (conv) D = d_rep4(__longlong_as_double((long long)D), tq52);   // in [0, 4q]
            mac128(acc0[k], D, __ldg(kb + i));
            mac128(acc1[k], D, __ldg(ka + i));
        }
    };
    // prefetched form: key words of a digit loaded before the NTT stages that precede their use
    uint64_t pkb[2][PF ? EPT : 1], pka[2][PF ? EPT : 1];
    auto prefetch = [&](int slot, int j) {
        if constexpr (PF) {
            const uint64_t* kb = key_r + j * kstride_j;
#pragma unroll
            for (int k = 0; k < EPT; k++) {
                pkb[slot][k] = __ldg(kb + threadIdx.x + k * NTHR);
                pka[slot][k] = __ldg(kb + kstride_p + threadIdx.x + k * NTHR);
            }
        }
    };
    auto mac_pref = [&](const uint64_t* buf, int slot) {
        if constexpr (PF) {
#pragma unroll
            for (int k = 0; k < EPT; k++) {
                const int i = threadIdx.x + k * NTHR;
                const uint64_t D = d_rep4(__longlong_as_double((long long)buf[G::addr(0, i)]), tq52);
                mac128(acc0[k], D, pkb[slot][k]);
                mac128(acc1[k], D, pka[slot][k]);
            }
        }
    };
    // digits j != ri, in pairs
    int j = 0;
    auto next_nd = [&](int from) { return from == ri ? from + 1 : from; };
    j = next_nd(0);
    while (j < l1) {
        const int ja = j;
        int jb = next_nd(ja + 1);
        const bool two = fp && jb < l1;
        copy_tile(sa, ja);
        if (two) copy_tile(sb, jb);
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        __syncthreads();
        if (two) {
            if constexpr (PF) { prefetch(0, ja); prefetch(1, jb); }
            fwd_engine_f64_rowtw2<LOG_M, LOG_R>(reinterpret_cast<double*>(sa), reinterpret_cast<double*>(sb), qd.x,
                                                qd.y, tws, t);
            if constexpr (PF) {
                mac_pref(sa, 0);
                mac_pref(sb, 1);
            } else {
                mac_tile(sa, ja, true);
                mac_tile(sb, jb, true);
            }
            j = next_nd(jb + 1);
        } else {
            if (fp)
                fwd_engine_f64_rowtw<LOG_M, LOG_R>(reinterpret_cast<double*>(sa), qd.x, qd.y, tws, t);
            else
                fwd_engine<LOG_M, LOG_R>(sa, md.q, tb.fwd + ((long long)mi << log_n), log_n - LOG_M,
                                         (uint32_t)row0, 0, t);
            mac_tile(sa, ja, fp);
            j = next_nd(ja + 1);
        }
        __syncthreads();
    }
    if (ri < l1) {   // the diagonal digit: D_{ri, q_ri} = d_ri, already in the NTT domain
        copy_tile(sa, ri);
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        __syncthreads();
        mac_tile(sa, ri, false);
    }
    uint64_t* out0 = job.acc[z] + ((long long)ri << log_n) + off0;
    uint64_t* out1 = job.acc[z] + ((long long)(nri + ri) << log_n) + off0;
#pragma unroll
    for (int k = 0; k < EPT; k++) {
        const int i = threadIdx.x + k * NTHR;
        out0[i] = barrett128(acc0[k].lo, acc0[k].hi, md);
        out1[i] = barrett128(acc1[k].lo, acc1[k].hi, md);
    }
}

// K4 register-direct (variant 80): the FP64 rows of k_ks_ip2 without the staging round trips.
// M = 256 as four radix-4 phases over 64 threads: phase 0's operands (elements t + 64e) are
// loaded from the pass-1 output straight into registers (a warp reads 256 contiguous bytes per
// load), phases exchange through the swizzled shared tiles, and phase 3 leaves thread t holding
// elements 4t + e, which are multiplied into the accumulators from registers with the key words
// read as two 16-byte vectors.  Two digits in flight as in k_ks_ip2; the special prime's row
// (integer engine) runs the k_ks_ip2 path.
template <int MINB>
__global__ void __launch_bounds__(64, MINB) k_ks_ip5(KsJob job, Tables tb) {
    constexpr int LOG_M = 8, LOG_R = 2;
    using G = Geo<LOG_M, LOG_R>;
    extern __shared__ uint64_t sm[];
    uint64_t* sa = sm;
    uint64_t* sb = sm + G::STRIDE;
    double* tws = reinterpret_cast<double*>(sm + 2 * G::STRIDE);
    const int nz = job.nz;
    const int z = blockIdx.x % nz;
    const int ri = blockIdx.y == 0 ? job.l1 : (int)blockIdx.y - 1;   // special prime first
    const int l1 = job.l1;
    const int nri = l1 + 1;
    const int log_n = tb.log_n;
    const int row0 = blockIdx.x / nz;
    const long long off0 = (long long)row0 << LOG_M;
    const int mi = job.mod_map[ri];
    const Mod md = tb.mods[mi];
    const bool fp = (double)md.q < tb.f64_max_q;
    const int t = threadIdx.x;
    const long long kstride_j = 2ll * (job.L + 1) << log_n;
    const long long kstride_p = (long long)(job.L + 1) << log_n;
    const uint64_t* key_r = job.key + ((long long)mi << log_n) + off0;
    uint64_t* out0 = job.acc[z] + ((long long)ri << log_n) + off0;
    uint64_t* out1 = job.acc[z] + ((long long)(nri + ri) << log_n) + off0;
    auto tile_src = [&](int j) -> const uint64_t* {
        return (j == ri) ? job.d[z] + ((long long)j << log_n) + off0
                         : job.t1[z] + (((long long)j * nri + ri) << log_n) + off0;
    };
    U128 acc0[4], acc1[4];
#pragma unroll
    for (int k = 0; k < 4; k++) { acc0[k] = U128{0, 0}; acc1[k] = U128{0, 0}; }
    if (!fp) {   // integer-engine row: staged engine, elements t + 64k
        for (int j = 0; j < l1 + 1; j++) {
            if (j == l1 && ri >= l1) break;
            const int jj = j == l1 ? ri : j;
            if (j < l1 && j == ri) continue;
            const uint64_t* src = tile_src(jj);
#pragma unroll
            for (int k = 0; k < 4; k++) {
                const int i = t + k * 64;
                const unsigned s_ = (unsigned)__cvta_generic_to_shared(&sa[G::addr(0, i)]);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s_), "l"(src + i) : "memory");
            }
            asm volatile("cp.async.wait_all;\n" ::: "memory");
            __syncthreads();
            if (j < l1)
                fwd_engine<LOG_M, LOG_R>(sa, md.q, tb.fwd + ((long long)mi << log_n), log_n - LOG_M, (uint32_t)row0, 0, t);
            const uint64_t* kb = key_r + jj * kstride_j;
#pragma unroll
            for (int k = 0; k < 4; k++) {
                const int i = t + k * 64;
                const uint64_t D = sa[G::addr(0, i)];
                mac128(acc0[k], D, __ldg(kb + i));
                mac128(acc1[k], D, __ldg(kb + kstride_p + i));
            }
            __syncthreads();
        }
#pragma unroll
        for (int k = 0; k < 4; k++) {
            out0[t + k * 64] = barrett128(acc0[k].lo, acc0[k].hi, md);
            out1[t + k * 64] = barrett128(acc1[k].lo, acc1[k].hi, md);
        }
        return;
    }
    const double2 qd = tb.modd[mi];
    const double q = qd.x, qinv = qd.y;
    const double tq52 = __dadd_rn(2.0 * q, 4503599627370496.0);   // 2q + 2^52
    {
        const double* twg = tb.fwd_d + ((long long)mi << log_n);
        const int s0 = log_n - LOG_M;
        for (int idx = t + 1; idx < G::M; idx += 64) {
            const int u = 31 - __clz(idx), m = idx - (1 << u);
            tws[idx] = twg[(1 << (s0 + u)) + (row0 << u) + m];
        }
    }
    __syncthreads();
    // ND digits (1 or 2) through the four phases, then MAC from registers
    auto run = [&](auto nd_c, int ja, int jb) {
        constexpr int ND = decltype(nd_c)::value;
        double r[ND][4];
        const uint64_t* src[2] = {tile_src(ja), tile_src(jb)};
#pragma unroll
        for (int n = 0; n < ND; n++)
#pragma unroll
            for (int e = 0; e < 4; e++) r[n][e] = __longlong_as_double((long long)__ldcs(src[n] + t + 64 * e));
        uint64_t* tl[2] = {sa, sb};
#pragma unroll
        for (int ph = 0; ph < 4; ph++) {
            const int u0 = 2 * ph;
            const int lo_bit = 6 - u0;
            const int olow = t & ((1 << lo_bit) - 1), ohigh = t >> lo_bit;
            const int base = (ohigh << (lo_bit + 2)) | olow;
            if (ph > 0) {
#pragma unroll
                for (int n = 0; n < ND; n++)
#pragma unroll
                    for (int e = 0; e < 4; e++)
                        r[n][e] = reinterpret_cast<const double*>(tl[n])[G::addr(0, base | (e << lo_bit))];
            }
#pragma unroll
            for (int uu = 0; uu < 2; uu++) {
                const int u = u0 + uu;
                const int dist = 2 >> uu;
                const int tbase = (1 << u) + (ohigh << uu);
#pragma unroll
                for (int k = 0; k < 2; k++) {
                    if (k >= (1 << uu)) break;
                    const double W = tws[tbase + k];
#pragma unroll
                    for (int e0 = 0; e0 < 2; e0++) {
                        if (e0 >= dist) break;
                        const int e = k * 2 * dist + e0;
#pragma unroll
                        for (int n = 0; n < ND; n++) {
                            const double X = full_stage(u, LOG_M) ? redd(r[n][e], q, qinv) : r[n][e];
                            const double T = mulred(r[n][e + dist], W, q, qinv);
                            r[n][e] = __dadd_rn(X, T);
                            r[n][e + dist] = __dsub_rn(X, T);
                        }
                    }
                }
            }
            if (ph < 3) {
                if (ph == 0) __syncthreads();   // the previous round's phase-3 reads are done
#pragma unroll
                for (int n = 0; n < ND; n++)
#pragma unroll
                    for (int e = 0; e < 4; e++)
                        reinterpret_cast<double*>(tl[n])[G::addr(0, base | (e << lo_bit))] = r[n][e];
                __syncthreads();
            }
        }
        // phase 3 left elements 4t + e in registers
#pragma unroll
        for (int n = 0; n < ND; n++) {
            const uint64_t* kb = key_r + (n == 0 ? ja : jb) * kstride_j + 4 * t;
            const ulonglong2 b0 = __ldg(reinterpret_cast<const ulonglong2*>(kb));
            const ulonglong2 b1 = __ldg(reinterpret_cast<const ulonglong2*>(kb) + 1);
            const ulonglong2 a0 = __ldg(reinterpret_cast<const ulonglong2*>(kb + kstride_p));
            const ulonglong2 a1 = __ldg(reinterpret_cast<const ulonglong2*>(kb + kstride_p) + 1);
            const uint64_t kbv[4] = {b0.x, b0.y, b1.x, b1.y}, kav[4] = {a0.x, a0.y, a1.x, a1.y};
#pragma unroll
            for (int e = 0; e < 4; e++) {
                const uint64_t D = d_rep4(r[n][e], tq52);
                mac128(acc0[e], D, kbv[e]);
                mac128(acc1[e], D, kav[e]);
            }
        }
    };
    const int n_nd = l1 - 1;                                  // fp rows: ri < l1
    auto digit = [&](int idx) { return idx < ri ? idx : idx + 1; };
    int idx = 0;
    for (; idx + 1 < n_nd; idx += 2) run(std::integral_constant<int, 2>(), digit(idx), digit(idx + 1));
    if (idx < n_nd) run(std::integral_constant<int, 1>(), digit(idx), digit(idx));
    {   // the diagonal digit: d_ri, already in the NTT domain (canonical), elements 4t + e
        const uint64_t* src = tile_src(ri) + 4 * t;
        const ulonglong2 d0 = __ldg(reinterpret_cast<const ulonglong2*>(src));
        const ulonglong2 d1 = __ldg(reinterpret_cast<const ulonglong2*>(src) + 1);
        const uint64_t dv[4] = {d0.x, d0.y, d1.x, d1.y};
        const uint64_t* kb = key_r + ri * kstride_j + 4 * t;
#pragma unroll
        for (int e = 0; e < 4; e++) {
            mac128(acc0[e], dv[e], __ldg(kb + e));
            mac128(acc1[e], dv[e], __ldg(kb + kstride_p + e));
        }
    }
    ulonglong2* o0 = reinterpret_cast<ulonglong2*>(out0 + 4 * t);
    ulonglong2* o1 = reinterpret_cast<ulonglong2*>(out1 + 4 * t);
    o0[0] = make_ulonglong2(barrett128(acc0[0].lo, acc0[0].hi, md), barrett128(acc0[1].lo, acc0[1].hi, md));
    o0[1] = make_ulonglong2(barrett128(acc0[2].lo, acc0[2].hi, md), barrett128(acc0[3].lo, acc0[3].hi, md));
    o1[0] = make_ulonglong2(barrett128(acc1[0].lo, acc1[0].hi, md), barrett128(acc1[1].lo, acc1[1].hi, md));
    o1[1] = make_ulonglong2(barrett128(acc1[2].lo, acc1[2].hi, md), barrett128(acc1[3].lo, acc1[3].hi, md));
}

// K4 with NT digits in flight (variant 50+): generalises k_ks_ip2; the digits j != ri are taken
// NT at a time (the last group may be smaller), then the diagonal digit
template <int LOG_M, int LOG_R, int MINB, int NT>
__global__ void __launch_bounds__((1 << LOG_M) / (1 << LOG_R), MINB) k_ks_ipN(KsJob job, Tables tb) {
    using G = Geo<LOG_M, LOG_R>;
    extern __shared__ uint64_t sm[];
    double* tws = reinterpret_cast<double*>(sm + NT * G::STRIDE);
    const int nz = job.nz;
    const int z = blockIdx.x % nz;
    const int ri = blockIdx.y;
    const int l1 = job.l1;
    const int nri = l1 + 1;
    const int log_n = tb.log_n;
    const int row0 = blockIdx.x / nz;
    const long long off0 = (long long)row0 << LOG_M;
    const int mi = job.mod_map[ri];
    const Mod md = tb.mods[mi];
    const bool fp = (double)md.q < tb.f64_max_q;
    const double2 qd = fp ? tb.modd[mi] : make_double2(0, 0);
    const double tq52 = __dadd_rn(2.0 * qd.x, 4503599627370496.0);
    constexpr int NTHR = G::T;
    constexpr int EPT = G::R;
    U128 acc0[EPT], acc1[EPT];
#pragma unroll
    for (int k = 0; k < EPT; k++) { acc0[k] = U128{0, 0}; acc1[k] = U128{0, 0}; }
    const int t = threadIdx.x;
    const long long kstride_j = 2ll * (job.L + 1) << log_n;
    const long long kstride_p = (long long)(job.L + 1) << log_n;
    const uint64_t* key_r = job.key + ((long long)mi << log_n) + off0;
    if (fp) {
        const double* twg = tb.fwd_d + ((long long)mi << log_n);
        const int s0 = log_n - LOG_M;
        for (int idx = threadIdx.x + 1; idx < G::M; idx += NTHR) {
            const int u = 31 - __clz(idx), m = idx - (1 << u);
            tws[idx] = twg[(1 << (s0 + u)) + (row0 << u) + m];
        }
    }
    auto copy_tile = [&](uint64_t* dst, int j) {
        const uint64_t* src = (j == ri) ? job.d[z] + ((long long)j << log_n) + off0
                                        : job.t1[z] + (((long long)j * nri + ri) << log_n) + off0;
#pragma unroll
        for (int k = 0; k < EPT; k++) {
            const int i = threadIdx.x + k * NTHR;
            const unsigned s_ = (unsigned)__cvta_generic_to_shared(&dst[G::addr(0, i)]);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s_), "l"(src + i) : "memory");
        }
    };
    auto mac_tile = [&](const uint64_t* buf, int j, bool conv) {
        const uint64_t* kb = key_r + j * kstride_j;
        const uint64_t* ka = kb + kstride_p;
#pragma unroll
        for (int k = 0; k < EPT; k++) {
            const int i = threadIdx.x + k * NTHR;
            uint64_t D = buf[G::addr(0, i)];
            if (conv) D = d_rep4(__longlong_as_double((long long)D), tq52);
            mac128(acc0[k], D, __ldg(kb + i));
            mac128(acc1[k], D, __ldg(ka + i));
        }
    };
    int js[NT];
    int j = (ri == 0) ? 1 : 0;
    while (j < l1) {
        int n = 0;
        while (n < NT && j < l1) {
            js[n++] = j;
            j++;
            if (j == ri) j++;
        }
        for (int m = 0; m < n; m++) copy_tile(sm + m * G::STRIDE, js[m]);
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        __syncthreads();
        if (fp && n == NT) {
            double* tl[NT];
#pragma unroll
            for (int m = 0; m < NT; m++) tl[m] = reinterpret_cast<double*>(sm + m * G::STRIDE);
            fwd_engine_f64_rowtwN<LOG_M, LOG_R, NT>(tl, qd.x, qd.y, tws, t);
        } else {
            for (int m = 0; m < n; m++) {
                if (fp)
                    fwd_engine_f64_rowtw<LOG_M, LOG_R>(reinterpret_cast<double*>(sm + m * G::STRIDE), qd.x, qd.y, tws,
                                                       t);
                else
                    fwd_engine<LOG_M, LOG_R>(sm + m * G::STRIDE, md.q, tb.fwd + ((long long)mi << log_n),
                                             log_n - LOG_M, (uint32_t)row0, 0, t);
            }
        }
        for (int m = 0; m < n; m++) mac_tile(sm + m * G::STRIDE, js[m], fp);
        __syncthreads();
    }
    if (ri < l1) {
        copy_tile(sm, ri);
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        __syncthreads();
        mac_tile(sm, ri, false);
    }
    uint64_t* out0 = job.acc[z] + ((long long)ri << log_n) + off0;
    uint64_t* out1 = job.acc[z] + ((long long)(nri + ri) << log_n) + off0;
#pragma unroll
    for (int k = 0; k < EPT; k++) {
        const int i = threadIdx.x + k * NTHR;
        out0[i] = barrett128(acc0[k].lo, acc0[k].hi, md);
        out1[i] = barrett128(acc1[k].lo, acc1[k].hi, md);
    }
}

template <int LOG_M, int LOG_R, int MINB, int NT>
static cudaError_t ks_ipN_t(const KsJob& job, const Tables& tb, int nz, cudaStream_t st) {
    using G = Geo<LOG_M, LOG_R>;
    const int rows = 1 << (tb.log_n - LOG_M);
    const size_t smem = ((size_t)NT * G::STRIDE + G::M) * sizeof(uint64_t);
    dim3 grid(rows * nz, job.l1 + 1, 1);
    k_ks_ipN<LOG_M, LOG_R, MINB, NT><<<grid, G::T, smem, st>>>(job, tb);
    return cudaGetLastError();
}

template <int MINB>
static cudaError_t ks_ip5_t(const KsJob& job, const Tables& tb, int nz, cudaStream_t st) {
    using G = Geo<8, 2>;
    const int rows = 1 << (tb.log_n - 8);
    const size_t smem = (2 * (size_t)G::STRIDE + G::M) * sizeof(uint64_t);
    dim3 grid(rows * nz, job.l1 + 1, 1);
    k_ks_ip5<MINB><<<grid, 64, smem, st>>>(job, tb);
    return cudaGetLastError();
}

template <int LOG_M, int LOG_R, int MINB, bool PF = false>
static cudaError_t ks_ip2_t(const KsJob& job, const Tables& tb, int nz, cudaStream_t st) {
    using G = Geo<LOG_M, LOG_R>;
    const int rows = 1 << (tb.log_n - LOG_M);
    const size_t smem = (2 * (size_t)G::STRIDE + G::M) * sizeof(uint64_t);
    dim3 grid(rows * nz, job.l1 + 1, 1);
    k_ks_ip2<LOG_M, LOG_R, MINB, PF><<<grid, G::T, smem, st>>>(job, tb);
    return cudaGetLastError();
}

template <int LOG_M, int LOG_R, int GR, int MINB>
static cudaError_t ks_ip_t(const KsJob& job, const Tables& tb, int nz, cudaStream_t st) {
    using G = Geo<LOG_M, LOG_R>;
    const int rows = 1 << (tb.log_n - LOG_M);
    if (rows < GR) return cudaErrorInvalidValue;
    constexpr int threads = GR * G::T;
    const size_t smem = ((size_t)GR * G::STRIDE + (GR == 1 ? G::M : 0)) * sizeof(uint64_t);
    dim3 grid((rows / GR) * nz, job.l1 + 1, 1);
    k_ks_ip<LOG_M, LOG_R, GR, MINB><<<grid, threads, smem, st>>>(job, tb);
    return cudaGetLastError();
}

static int ks_variant() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("HISA_KS_VARIANT");
        v = e ? atoi(e) : 0;
    }
    return v;
}

template <int LOG_M>
static cudaError_t ks_ip_m(const KsJob& job, const Tables& tb, int nz, cudaStream_t st) {
    const int rows = 1 << (tb.log_n - LOG_M);
    switch (ks_variant()) {   // alternatives kept for re-measurement (profiles/r1_ks_variants.txt)
        case 10: return ks_ip_t<LOG_M, 2, 1, 8>(job, tb, nz, st);
        case 20: return ks_ip_pipe_t<LOG_M, 2, 1, 8>(job, tb, nz, st);
        case 41: return ks_ip2_t<LOG_M, 2, 12, true>(job, tb, nz, st);
        case 55: return ks_ipN_t<LOG_M, 2, 12, 3>(job, tb, nz, st);
        case 33: return ks_ip2_t<LOG_M, 2, 12>(job, tb, nz, st);
        case 80: if constexpr (LOG_M == 8) return ks_ip5_t<12>(job, tb, nz, st); break;
        default: break;
    }
    // default (measured best on B200 at N = 2^16, L = 24; profiles/r1_ks_variants.txt): M = 256
    // rows -> the register-direct two-digit kernel (variant 81, >= 10 CTAs / SM); other row
    // lengths -> variant 33 (one row per 64-thread CTA, radix-4 phases, two digits interleaved
    // through the FP64 engine with the row's twiddles staged in shared memory, >= 12 CTAs / SM)
    if constexpr (LOG_M == 8) return ks_ip5_t<10>(job, tb, nz, st);
    return ks_ip2_t<LOG_M, 2, 12>(job, tb, nz, st);
}

cudaError_t launch_ks_ip(const KsJob& job, const Tables& tb, int nz, cudaStream_t st) {
    const int lm = tb.log_n - split_m1(tb.log_n);
    switch (lm) {
        case 4: return ks_ip_m<4>(job, tb, nz, st);
        case 5: return ks_ip_m<5>(job, tb, nz, st);
        case 6: return ks_ip_m<6>(job, tb, nz, st);
        case 7: return ks_ip_m<7>(job, tb, nz, st);
        case 8: return ks_ip_m<8>(job, tb, nz, st);
    }
    return cudaErrorInvalidValue;
}

// ------------------------------------------------------------------------------------------
// K7 hoisted inner product: R rotation amounts share one materialised ModUp output D (hoisting,
// P:717 "rotations ... code motioned out").  Each thread owns two words of one output prime ri,
// streams D[j][ri] once and the R keys' (b, a) limbs, and keeps 2R 128-bit accumulators per word.
// Pure HBM stream: (1 + 2R) 16-byte loads per digit per thread, no shared memory.
// ------------------------------------------------------------------------------------------
template <int R>
__global__ void __launch_bounds__(256) k_ks_ip_hoisted(KsHoistJob job, const Mod* __restrict__ mods, int log_n) {
    const int ri = blockIdx.y;
    const int l1 = job.l1, l2 = l1 + 1;
    const long long N = 1ll << log_n;
    const long long x = 2ll * (blockIdx.x * (long long)blockDim.x + threadIdx.x);
    if (x >= N) return;
    const int mi = job.mod_map[ri];
    const Mod md = mods[mi];
    U128 acc[R][2][2];
#pragma unroll
    for (int k = 0; k < R; k++)
#pragma unroll
        for (int h = 0; h < 2; h++) { acc[k][h][0] = U128{0, 0}; acc[k][h][1] = U128{0, 0}; }
    const long long kstride_j = 2ll * (job.L + 1) * N;
    const long long kstride_p = (long long)(job.L + 1) * N;
    const long long koff = (long long)mi * N + x;
    for (int j = 0; j < l1; j++) {
        const uint64_t* src = (j == ri) ? job.diag + (long long)j * N + x : job.D + ((long long)j * l2 + ri) * N + x;
        const ulonglong2 d = __ldcs(reinterpret_cast<const ulonglong2*>(src));
#pragma unroll
        for (int k = 0; k < R; k++) {
            const uint64_t* kb = job.key[k] + j * kstride_j + koff;
            const ulonglong2 b = __ldcs(reinterpret_cast<const ulonglong2*>(kb));
            const ulonglong2 a = __ldcs(reinterpret_cast<const ulonglong2*>(kb + kstride_p));
            mac128(acc[k][0][0], d.x, b.x);
            mac128(acc[k][0][1], d.y, b.y);
            mac128(acc[k][1][0], d.x, a.x);
            mac128(acc[k][1][1], d.y, a.y);
        }
    }
#pragma unroll
    for (int k = 0; k < R; k++)
#pragma unroll
        for (int h = 0; h < 2; h++) {
            uint64_t* o = job.acc[k] + ((long long)h * l2 + ri) * N + x;
            *reinterpret_cast<ulonglong2*>(o) = make_ulonglong2(barrett128(acc[k][h][0].lo, acc[k][h][0].hi, md),
                                                                barrett128(acc[k][h][1].lo, acc[k][h][1].hi, md));
        }
}

cudaError_t launch_ks_ip_hoisted(const KsHoistJob& job, int R, const Mod* mods, int log_n, cudaStream_t st) {
    const long long N = 1ll << log_n;
    dim3 grid((unsigned)((N / 2 + 255) / 256), job.l1 + 1, 1);
    switch (R) {
#define C(RR) case RR: k_ks_ip_hoisted<RR><<<grid, 256, 0, st>>>(job, mods, log_n); break;
        C(1) C(2) C(3) C(4) C(5) C(6) C(7) C(8)
#undef C
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// K7 batched over ciphertexts: CG ciphertexts x R keys per thread-word (one word per thread),
// 2 CG R 128-bit accumulators; the key words are loaded once for the CG ciphertexts.
// ------------------------------------------------------------------------------------------
template <int CG, int R>
__global__ void __launch_bounds__(256) k_ks_ip_hoisted_multi(KsHoistMultiJob job, const Mod* __restrict__ mods,
                                                             int log_n) {
    const int ri = blockIdx.y;
    const int l1 = job.l1, l2 = l1 + 1;
    const long long N = 1ll << log_n;
    const long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (x >= N) return;
    const int mi = job.mod_map[ri];
    const Mod md = mods[mi];
    U128 acc[CG][R][2];
#pragma unroll
    for (int c = 0; c < CG; c++)
#pragma unroll
        for (int k = 0; k < R; k++) { acc[c][k][0] = U128{0, 0}; acc[c][k][1] = U128{0, 0}; }
    const long long kstride_j = 2ll * (job.L + 1) * N;
    const long long kstride_p = (long long)(job.L + 1) * N;
    const long long koff = (long long)mi * N + x;
    for (int j = 0; j < l1; j++) {
        uint64_t d[CG];
#pragma unroll
        for (int c = 0; c < CG; c++) {
            const uint64_t* src = (j == ri) ? job.diag[c] + (long long)j * N + x
                                            : job.D[c] + ((long long)j * l2 + ri) * N + x;
            d[c] = __ldcs(src);
        }
#pragma unroll
        for (int k = 0; k < R; k++) {
            const uint64_t* kb = job.key[k] + j * kstride_j + koff;
            const uint64_t b = __ldcs(kb), a = __ldcs(kb + kstride_p);
#pragma unroll
            for (int c = 0; c < CG; c++) {
                mac128(acc[c][k][0], d[c], b);
                mac128(acc[c][k][1], d[c], a);
            }
        }
    }
#pragma unroll
    for (int c = 0; c < CG; c++)
#pragma unroll
        for (int k = 0; k < R; k++)
#pragma unroll
            for (int h = 0; h < 2; h++)
                job.acc[c][k][((long long)h * l2 + ri) * N + x] = barrett128(acc[c][k][h].lo, acc[c][k][h].hi, md);
}

cudaError_t launch_ks_ip_hoisted_multi(const KsHoistMultiJob& job, int R, const Mod* mods, int log_n, cudaStream_t st) {
    const long long N = 1ll << log_n;
    dim3 grid((unsigned)((N + 255) / 256), job.l1 + 1, 1);
#define C(CGV, RV) if (job.cg == CGV && R == RV) { k_ks_ip_hoisted_multi<CGV, RV><<<grid, 256, 0, st>>>(job, mods, log_n); return cudaGetLastError(); }
    C(4, 1) C(4, 2) C(4, 3) C(4, 4) C(2, 1) C(2, 2) C(2, 3) C(2, 4) C(3, 1) C(3, 2) C(3, 3) C(3, 4)
    C(1, 1) C(1, 2) C(1, 3) C(1, 4)
#undef C
    return cudaErrorInvalidValue;
}

}  // namespace hisa
