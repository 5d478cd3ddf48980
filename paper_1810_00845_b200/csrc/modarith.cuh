// modarith.cuh -- 64-bit modular arithmetic on the sm_100a integer pipes.
//
// Residues are uint64 words for primes q < 2^61 (configs use 40/50/60-bit primes, A3).
//  * Shoup (fixed operand w with w' = floor(w 2^64 / q)): twiddles, scalars, p^-1, q_l^-1.
//  * Barrett over a 128-bit value with ratio = floor(2^128 / q) (two words): ct x ct, mulPlain,
//    the lazily accumulated key inner product, and 128-bit uniform sampling.
// Lazy ranges: butterflies keep values in [0, 4q) (Harvey), so 4q < 2^63 is required.
#pragma once
#include <cstdint>

namespace hisa {

struct Mod {
    uint64_t q;
    uint64_t r0, r1;     // floor(2^128 / q) = r1 * 2^64 + r0
};

__device__ __forceinline__ uint64_t mulhi(uint64_t a, uint64_t b) { return __umul64hi(a, b); }

// x * w mod q in [0, 2q) for any x < 2^64 (Shoup, lazy)
__device__ __forceinline__ uint64_t mul_shoup_lazy(uint64_t x, uint64_t w, uint64_t wp, uint64_t q) {
    return x * w - mulhi(x, wp) * q;
}
__device__ __forceinline__ uint64_t mul_shoup(uint64_t x, uint64_t w, uint64_t wp, uint64_t q) {
    uint64_t r = mul_shoup_lazy(x, w, wp, q);
    return r >= q ? r - q : r;
}
__device__ __forceinline__ uint64_t csub(uint64_t x, uint64_t q) { return x >= q ? x - q : x; }
// [0, 4q) -> [0, q)
__device__ __forceinline__ uint64_t reduce4(uint64_t x, uint64_t q) {
    x = csub(x, 2 * q);
    return csub(x, q);
}
__device__ __forceinline__ uint64_t add_mod(uint64_t a, uint64_t b, uint64_t q) { return csub(a + b, q); }
__device__ __forceinline__ uint64_t sub_mod(uint64_t a, uint64_t b, uint64_t q) { return a >= b ? a - b : a + q - b; }
__device__ __forceinline__ uint64_t neg_mod(uint64_t a, uint64_t q) { return a ? q - a : 0; }

// (hi 2^64 + lo) mod q for ANY 128-bit value, q <= 2^60 (SEAL-style base-2^64 Barrett; the
// quotient estimate is at most 1 short, so one conditional subtraction finishes).
__device__ __forceinline__ uint64_t barrett128(uint64_t lo, uint64_t hi, const Mod& m) {
    uint64_t carry = mulhi(lo, m.r0);
    uint64_t t2lo = lo * m.r1, t2hi = mulhi(lo, m.r1);
    uint64_t t1 = t2lo + carry;
    uint64_t t3 = t2hi + (t1 < carry);
    uint64_t t4lo = hi * m.r0, t4hi = mulhi(hi, m.r0);
    uint64_t s = t1 + t4lo;
    carry = t4hi + (s < t1);
    uint64_t qest = hi * m.r1 + t3 + carry;
    uint64_t r = lo - qest * m.q;
    return csub(r, m.q);
}
__device__ __forceinline__ uint64_t barrett64(uint64_t x, const Mod& m) {
    uint64_t qe = mulhi(x, m.r1);
    return csub(x - qe * m.q, m.q);
}
__device__ __forceinline__ uint64_t mul_mod(uint64_t a, uint64_t b, const Mod& m) {
    return barrett128(a * b, mulhi(a, b), m);
}

// 128-bit accumulator
struct U128 {
    uint64_t lo, hi;
};
__device__ __forceinline__ void mac128(U128& acc, uint64_t a, uint64_t b) {
    uint64_t lo = a * b, hi = mulhi(a, b);
    acc.lo += lo;
    acc.hi += hi + (acc.lo < lo);
}

// signed centered value x in (-Q/2, Q/2) given as residue v mod Q -> residue mod r
// (ModUp / ModDown / rescale lift; exact for alpha = 1, A14)
__device__ __forceinline__ uint64_t lift_centered(uint64_t v, uint64_t Q, const Mod& r) {
    if (v > (Q >> 1)) {                       // negative representative v - Q
        uint64_t a = barrett64(Q - v, r);     // |x| mod r
        return a ? r.q - a : 0;
    }
    return barrett64(v, r);
}

}  // namespace hisa
