// ntt.cuh -- batched negacyclic NTT / INTT over RNS limbs for sm_100a (steps a1, a2).
//
// Definition (A5, the paper's "NTT domain" P:764): ahat[j] = sum_t a_t psi^((2 brv(j)+1) t),
// stored in bit-reversed evaluation order, residues in [0, q).
//
// Algorithm (B200 design, not the paper's): merged Cooley-Tukey forward / Gentleman-Sande inverse
// with psi-power tables in bit-reversed order, split into TWO passes of N = M1 x M2:
//   forward: pass 1 = first log M1 stages on the M2 strided "columns" (elements j = mid*M2 + c);
//            pass 2 = last  log M2 stages on the M1 contiguous "rows".
//   inverse: pass A = first log M2 GS stages on rows, pass B = last log M1 stages on columns,
//            with the N^-1 scaling folded into pass B's store.
// Each CTA stages a tile of G groups in shared memory (coalesced global traffic, padded layout
// addr = mid + mid/R so every phase is bank-conflict free for 64-bit words), and runs the
// group's stages in phases of up to log R stages; a thread keeps R = 2^LOG_R words in registers
// per phase.  Butterflies are Harvey-lazy: forward keeps [0, 4q), inverse keeps [0, 2q).
// Twiddles: (W, W') pairs, W' = floor(W 2^64 / q); forward index 2^s + i, inverse index
// 2^(logN-v-1) + (j >> (v+1)) into psi^{+-brv(k)} tables (validated against the oracle).
#pragma once
#include <cstdint>
#include "modarith.cuh"

namespace hisa {

constexpr int MAXB = 128;    // ciphertexts per batched launch (pointer arrays passed by value;
                             // CUDA 12 kernel parameter blocks up to 32 KB)
constexpr int MAXL = 64;     // limbs per polynomial (moduli incl. special prime)

// ------------------------------------------------------------------------------------------
// per-launch job: limb lambda = blockIdx.y decomposes as (a = lambda / nb, b = lambda % nb);
// word offset of a limb = a*sA + b*sB for every stream.  Modulus for arithmetic = mod_map[b];
// source modulus of a lifting load = smod_map[a].
// ------------------------------------------------------------------------------------------
struct PassJob {
    const uint64_t* src[MAXB];
    uint64_t* dst[MAXB];
    const uint64_t* aux[MAXB];     // combine operand (u or acc)
    const uint64_t* add[MAXB];     // optional addend (rotation: psi_g(c0))
    long long src_a, src_b, dst_a, dst_b, aux_a, aux_b, add_a, add_b;
    int nb;
    int skip_diag;                 // skip limbs with a == b (ModUp: D_{j,q_j} is c1_j itself)
    int aux_limit;                 // add addend only for a < aux_limit ... (poly index)
    uint8_t mod_map[MAXL];
    uint8_t smod_map[MAXL];
};

struct Tables {
    const ulonglong2* fwd;      // [mod][N] (W, W') psi^brv(k)
    const ulonglong2* inv;      // [mod][N] (W, W') psi^-brv(k)
    const Mod* mods;            // [mod]
    const ulonglong2* ninv;     // [mod] (N^-1, shoup)
    const ulonglong2* comb;     // [mod] combine multiplier (p^-1 or q_l^-1 mod q_i), Shoup
    const double* fwd_d;        // [mod][N] W as doubles (FP64 engine, q < 2^50; ntt_f64.cuh)
    const double* inv_d;        // [mod][N]
    const double2* modd;        // [mod] (q, fl(1/q))
    const double* ninv_d;       // [mod] N^-1 mod q as double
    double f64_max_q;           // moduli below this run the FP64 engine (0 disables it)
    uint64_t fp_mods;           // bit mi: modulus mi runs the FP64 engine (host-computed, no I2F)
    int log_n;
};

enum LoadMode { LOAD_PLAIN = 0, LOAD_LIFT = 1 };
enum StoreMode { STORE_PLAIN = 0, STORE_COMBINE = 1 };

// Shared-memory layout of a tile: addr(g, mid) = g * STRIDE + swz(mid).  Chosen per (LOG_M, LOG_R)
// by exhaustive search over every access pattern of both engines, the row / column tile loads
// and the MAC reads (64-bit words: 16 distinct word slots per half-warp wavefront):
//   PAD: swz = mid + (mid >> K);  XOR: swz = mid ^ ((mid >> K) & 15);  NONE: swz = mid.
// Average wavefronts / ideal: 1.0 - 1.33 (the plain mid + mid/R padding was 2.25 - 3.5).
enum SwzKind { SWZ_NONE = 0, SWZ_PAD = 1, SWZ_XOR = 2 };
template <int LOG_M, int LOG_R>
struct Layout {
    static constexpr int M = 1 << LOG_M;
    static constexpr int KIND = (LOG_M == 8 && LOG_R == 4) ? SWZ_PAD
                              : (LOG_M == 5 && LOG_R == 4) ? SWZ_PAD
                              : (LOG_M >= 6) ? SWZ_XOR : SWZ_NONE;
    static constexpr int K = (KIND == SWZ_PAD) ? 4 : (LOG_M == 6 ? 2 : 3);
    static constexpr int STRIDE = (LOG_M == 8 && LOG_R == 4) ? M + M / 16 + 1
                                : (LOG_M == 8) ? M + 2
                                : (LOG_M == 7) ? M + 1
                                : (LOG_M == 6) ? (LOG_R == 4 ? M + 7 : M + 1)
                                : (LOG_M == 5) ? (LOG_R == 4 ? M + 2 : M + 3)
                                : M + 1;
};

template <int LOG_M, int LOG_R>
struct Geo {
    static constexpr int M = 1 << LOG_M;
    static constexpr int R = 1 << LOG_R;
    static constexpr int T = M / R;                 // threads per group
    using Lay = Layout<LOG_M, LOG_R>;
    static constexpr int STRIDE = Lay::STRIDE;      // group stride in smem (words)
    __device__ static __forceinline__ int addr(int g, int mid) {
        if (Lay::KIND == SWZ_PAD) return g * STRIDE + mid + (mid >> Lay::K);
        if (Lay::KIND == SWZ_XOR) return g * STRIDE + (mid ^ ((mid >> Lay::K) & 15));
        return g * STRIDE + mid;
    }
};

// ------------------------------------------------------------------------------------------
// forward CT stages [s0, s0 + LOG_M) on the groups held in smem.  `high` = the group's index in
// the global decomposition (row index for pass 2, 0 for pass 1).
// ------------------------------------------------------------------------------------------
template <int LOG_M, int LOG_R>
__device__ __forceinline__ void fwd_engine(uint64_t* sm, uint64_t q, const ulonglong2* __restrict__ tw, int s0,
                                           uint32_t high, int g, int t) {
    using G = Geo<LOG_M, LOG_R>;
    const uint64_t q2 = 2 * q;
#pragma unroll
    for (int u0 = 0; u0 < LOG_M; u0 += LOG_R) {
        constexpr int dummy = 0;
        (void)dummy;
        const int w = (LOG_M - u0) < LOG_R ? (LOG_M - u0) : LOG_R;
        const int lo_bit = LOG_M - u0 - w;
        const int per = G::R >> w;
#pragma unroll
        for (int x = 0; x < G::R; x++) {
            if (x >= per) break;
            const int o = t * per + x;
            const int olow = o & ((1 << lo_bit) - 1);
            const int ohigh = o >> lo_bit;
            uint64_t reg[G::R];
            int base = (ohigh << (lo_bit + w)) | olow;
#pragma unroll
            for (int e = 0; e < G::R; e++)
                if (e < (1 << w)) reg[e] = sm[G::addr(g, base | (e << lo_bit))];
#pragma unroll
            for (int uu = 0; uu < LOG_R; uu++) {
                if (uu >= w) break;
                const int u = u0 + uu;
                const int dist = 1 << (w - 1 - uu);
                // twiddle for butterflies whose e has top-uu-bits k: index 2^(s0+u) + (high<<u) + (ohigh<<uu) + k
                const uint32_t tbase = (1u << (s0 + u)) + (high << u) + ((uint32_t)ohigh << uu);
#pragma unroll
                for (int k = 0; k < (1 << LOG_R); k++) {
                    if (k >= (1 << uu)) break;
                    const ulonglong2 W = __ldg(&tw[tbase + k]);
#pragma unroll
                    for (int e0 = 0; e0 < G::R; e0++) {
                        // butterflies e = k*2*dist + e0 for e0 < dist
                        if (e0 >= dist) break;
                        const int e = k * 2 * dist + e0;
                        uint64_t X = reg[e];
                        X = X >= q2 ? X - q2 : X;
                        const uint64_t Tm = mul_shoup_lazy(reg[e + dist], W.x, W.y, q);
                        reg[e] = X + Tm;
                        reg[e + dist] = X - Tm + q2;
                    }
                }
            }
#pragma unroll
            for (int e = 0; e < G::R; e++)
                if (e < (1 << w)) sm[G::addr(g, base | (e << lo_bit))] = reg[e];
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------------------------------
// inverse GS stages v = v0 .. v0 + LOG_M - 1 (distances 1, 2, 4, ... in mid).  The global index
// of mid is j = high * M + mid (rows, v0 = 0) or j = mid * M2 + c (columns, high = 0); the
// twiddle index 2^(logN-v-1) + (j >> (v+1)) then equals 2^(logN-v-1) + (high << (LOG_M-bit-1))
// + (mid >> (bit+1)), bit = v - v0.
// ------------------------------------------------------------------------------------------
template <int LOG_M, int LOG_R>
__device__ __forceinline__ void inv_engine(uint64_t* sm, uint64_t q, const ulonglong2* __restrict__ tw, int v0,
                                           int log_n, uint32_t high, int g, int t) {
    using G = Geo<LOG_M, LOG_R>;
    const uint64_t q2 = 2 * q;
#pragma unroll
    for (int b0 = 0; b0 < LOG_M; b0 += LOG_R) {
        const int w = (LOG_M - b0) < LOG_R ? (LOG_M - b0) : LOG_R;
        const int lo_bit = b0;
        const int per = G::R >> w;
#pragma unroll
        for (int x = 0; x < G::R; x++) {
            if (x >= per) break;
            const int o = t * per + x;
            const int olow = o & ((1 << lo_bit) - 1);
            const int ohigh = o >> lo_bit;
            uint64_t reg[G::R];
            const int base = (ohigh << (lo_bit + w)) | olow;
#pragma unroll
            for (int e = 0; e < G::R; e++)
                if (e < (1 << w)) reg[e] = sm[G::addr(g, base | (e << lo_bit))];
#pragma unroll
            for (int uu = 0; uu < LOG_R; uu++) {
                if (uu >= w) break;
                const int bit = lo_bit + uu;
                const int v = v0 + bit;
                const int dist = 1 << uu;
                const uint32_t tbase = (1u << (log_n - v - 1)) + (high << (LOG_M - bit - 1)) +
                                       ((uint32_t)ohigh << (w - uu - 1));
                // butterflies with e bit uu clear; twiddle by e >> (uu+1)
#pragma unroll
                for (int k = 0; k < (1 << LOG_R); k++) {
                    if (k >= (1 << (w - uu - 1))) break;
                    const ulonglong2 W = __ldg(&tw[tbase + k]);
#pragma unroll
                    for (int e0 = 0; e0 < G::R; e0++) {
                        if (e0 >= dist) break;
                        const int e = k * 2 * dist + e0;
                        const uint64_t X = reg[e], Y = reg[e + dist];
                        uint64_t s = X + Y;
                        reg[e] = s >= q2 ? s - q2 : s;
                        reg[e + dist] = mul_shoup_lazy(X - Y + q2, W.x, W.y, q);
                    }
                }
            }
#pragma unroll
            for (int e = 0; e < G::R; e++)
                if (e < (1 << w)) sm[G::addr(g, base | (e << lo_bit))] = reg[e];
        }
        __syncthreads();
    }
}

}  // namespace hisa
