// encode_kernels.cu -- CKKS encode on the GPU (NEXT-4; the paper's encoding, with the
// exact-rounding reading A7).
//
//   m_t = round-half-away( (Delta/N) * Re( F[t] * e^{-i pi t / N} ) ),
//   F[t] = sum_m A[m] e^{-2 pi i m t / N},  A[(5^j - 1)/2] += z_j,  A[(2N - 5^j - 1)/2] += z_j.
//
// The FFT runs in double-double arithmetic (~106-bit significands; twiddles computed on the host
// in binary128), so the computed v_t carries a relative error of order log2(N) 2^-100: every
// coefficient whose fractional part is farther than 2^-40 from 1/2 rounds exactly as the exact
// real value does.  Coefficients inside that window are flagged and recomputed on the host by the
// binary128 direct sum of hisa.cu (the same path the host encoder uses for its near ties), so the
// result equals the oracle's exact encoding bit for bit.
#include <cuda_runtime.h>
#include <cstdint>
#include "launch.h"

namespace hisa {

__device__ __forceinline__ dd two_sum(double a, double b) {
    const double s = __dadd_rn(a, b);
    const double bb = __dsub_rn(s, a);
    const double e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
    return dd{s, e};
}
__device__ __forceinline__ dd quick_two_sum(double a, double b) {
    const double s = __dadd_rn(a, b);
    return dd{s, __dsub_rn(b, __dsub_rn(s, a))};
}
__device__ __forceinline__ dd dd_add(dd x, dd y) {
    dd s = two_sum(x.hi, y.hi);
    dd t = two_sum(x.lo, y.lo);
    s.lo = __dadd_rn(s.lo, t.hi);
    s = quick_two_sum(s.hi, s.lo);
    s.lo = __dadd_rn(s.lo, t.lo);
    return quick_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_neg(dd x) { return dd{-x.hi, -x.lo}; }
__device__ __forceinline__ dd dd_mul(dd x, dd y) {
    const double p = __dmul_rn(x.hi, y.hi);
    double e = __fma_rn(x.hi, y.hi, -p);
    e = __fma_rn(x.hi, y.lo, e);
    e = __fma_rn(x.lo, y.hi, e);
    return quick_two_sum(p, e);
}
__device__ __forceinline__ cdd cmul(cdd a, cdd b) {
    return cdd{dd_add(dd_mul(a.re, b.re), dd_neg(dd_mul(a.im, b.im))),
               dd_add(dd_mul(a.re, b.im), dd_mul(a.im, b.re))};
}

// A (count x N complex dd, zeroed) <- the z values at bit-reversed positions (DIT input order)
__global__ void k_enc_scatter(cdd* A, const double* z, size_t n_per, const uint32_t* pos_brv, int log_n) {
    const size_t p = blockIdx.y;
    const long long N = 1ll << log_n;
    for (size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x; j < n_per; j += (size_t)gridDim.x * blockDim.x) {
        const double v = z[p * n_per + j];
        if (v == 0.0) continue;
        cdd* a = A + p * N;
        // the two positions of slot j (distinct), each receives exactly one value
        a[pos_brv[2 * j]].re = dd{v, 0.0};
        a[pos_brv[2 * j + 1]].re = dd{v, 0.0};
    }
}

// one radix-2 DIT stage of length len = 2^s: w_k = conj(root[k N / len]), root[i] = e^{2 pi i i/N}
__global__ void k_enc_fft_stage(cdd* A, const cdd* root, int log_n, int s) {
    const long long N = 1ll << log_n;
    const long long half = 1ll << (s - 1);
    const long long step = N >> s;
    cdd* a = A + (long long)blockIdx.y * N;
    for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < N / 2; b += (long long)gridDim.x * blockDim.x) {
        const long long grp = b / half, k = b - grp * half;
        const long long i0 = grp * 2 * half + k, i1 = i0 + half;
        const cdd r = root[k * step];
        const cdd w{r.re, dd_neg(r.im)};
        const cdd u = a[i0];
        const cdd v = cmul(a[i1], w);
        a[i0] = cdd{dd_add(u.re, v.re), dd_add(u.im, v.im)};
        a[i1] = cdd{dd_add(u.re, dd_neg(v.re)), dd_add(u.im, dd_neg(v.im))};
    }
}

// v_t = Re(F[t] conj(twist[t])) * scale / N -> m_t (round half away), flag near ties
__global__ void k_enc_round(const cdd* A, const cdd* twist, double scale_over_n, double window, int64_t* m,
                            uint32_t* flags, unsigned int* nflag, unsigned int max_flags, int log_n, int* overflow) {
    const long long N = 1ll << log_n;
    const size_t p = blockIdx.y;
    const cdd* a = A + p * N;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < N; t += (long long)gridDim.x * blockDim.x) {
        const cdd f = a[t], tw = twist[t];
        // Re(f * conj(tw)) = f.re tw.re + f.im tw.im
        dd v = dd_add(dd_mul(f.re, tw.re), dd_mul(f.im, tw.im));
        v = dd_mul(v, dd{scale_over_n, 0.0});
        double r;
        double frac;
        if (fabs(v.hi) < 4503599627370496.0) {          // |v| < 2^52: hi carries the fraction
            r = rint(v.hi);
            frac = __dadd_rn(__dsub_rn(v.hi, r), v.lo); // exact-ish distance to r
        } else {                                        // hi is an integer: lo carries it
            r = v.hi;
            const double rl = rint(v.lo);
            frac = __dsub_rn(v.lo, rl);
            r = __dadd_rn(r, rl);
        }
        // round-half-away: the nearest integer is r (|frac| < 0.5) unless we are near a tie
        const double af = fabs(frac);
        if (fabs(af - 0.5) < window) {                 // too close to a tie for the dd error bound
            const unsigned int slot = atomicAdd(nflag, 1u);
            if (slot < max_flags) flags[slot] = (uint32_t)(p * N + t);
            m[p * N + t] = 0;
            continue;
        }
        if (af > 0.5) r = __dadd_rn(r, frac > 0 ? 1.0 : -1.0);
        if (!(fabs(r) < 0x1p62)) { atomicExch(overflow, 1); r = 0; }
        m[p * N + t] = (int64_t)r;
    }
}

cudaError_t launch_encode_fft(const double* z_dev, size_t n_per, size_t count, const uint32_t* pos_brv,
                              const cdd* root, const cdd* twist, double scale_over_n, double window, int log_n,
                              cdd* A, int64_t* m, uint32_t* flags, unsigned int* nflag, unsigned int max_flags,
                              int* overflow, cudaStream_t st) {
    const long long N = 1ll << log_n;
    cudaError_t e = cudaMemsetAsync(A, 0, sizeof(cdd) * N * count, st);
    if (e != cudaSuccess) return e;
    if (n_per) {
        dim3 gs((unsigned)((n_per + 255) / 256), (unsigned)count);
        k_enc_scatter<<<gs, 256, 0, st>>>(A, z_dev, n_per, pos_brv, log_n);
    }
    dim3 gf((unsigned)((N / 2 + 255) / 256), (unsigned)count);
    for (int s = 1; s <= log_n; s++) k_enc_fft_stage<<<gf, 256, 0, st>>>(A, root, log_n, s);
    dim3 gr((unsigned)((N + 255) / 256), (unsigned)count);
    k_enc_round<<<gr, 256, 0, st>>>(A, twist, scale_over_n, window, m, flags, nflag, max_flags, log_n, overflow);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// GPU decode (NEXT-4; A2, A13): from the limb-0 coefficients m_t (after the INTT),
// centred mod q_0, the slot values are z_j = (1/Delta) sum_t m_t zeta^(5^j t), zeta = e^{i pi / N}
// = (1/Delta) B[(5^j - 1) / 2] with B[k] = sum_t (m_t e^{i pi t / N}) e^{+2 pi i k t / N}: a twist,
// one N-point complex FFT (double precision: decode is approximate by definition, the error is
// ~log2(N) 2^-53 max|m_t| / Delta) and a gather of the real parts.
// ------------------------------------------------------------------------------------------
struct cdbl { double re, im; };

__global__ void k_dec_twist(const uint64_t* const* m, uint64_t q0, const cdd* twist, cdbl* A, int log_n) {
    const long long N = 1ll << log_n;
    const uint64_t* mp = m[blockIdx.y];
    cdbl* a = reinterpret_cast<cdbl*>(A) + (long long)blockIdx.y * N;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < N; t += (long long)gridDim.x * blockDim.x) {
        const uint64_t v = mp[t];
        const double x = v > (q0 >> 1) ? -(double)(q0 - v) : (double)v;
        const cdd w = twist[t];
        a[__brev((unsigned)t) >> (32 - log_n)] = cdbl{x * w.re.hi, x * w.im.hi};
    }
}

// radix-2 DIT stage of length 2^s with w_k = root[k N / len] = e^{+2 pi i k / len}
__global__ void k_dec_fft_stage(cdbl* A, const cdd* root, int log_n, int s) {
    const long long N = 1ll << log_n;
    const long long half = 1ll << (s - 1);
    const long long step = N >> s;
    cdbl* a = A + (long long)blockIdx.y * N;
    for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < N / 2; b += (long long)gridDim.x * blockDim.x) {
        const long long grp = b / half, k = b - grp * half;
        const long long i0 = grp * 2 * half + k, i1 = i0 + half;
        const cdd r = root[k * step];
        const double wr = r.re.hi, wi = r.im.hi;
        const cdbl u = a[i0], x = a[i1];
        const cdbl v{__fma_rn(x.re, wr, -x.im * wi), __fma_rn(x.re, wi, x.im * wr)};
        a[i0] = cdbl{u.re + v.re, u.im + v.im};
        a[i1] = cdbl{u.re - v.re, u.im - v.im};
    }
}

// out[p][j] = Re B[(5^j - 1) / 2] / scale[p], j < n (pos_brv[2 j] = brv((5^j - 1) / 2))
__global__ void k_dec_gather(const cdbl* A, const uint32_t* pos_brv, const double* inv_scale, double* out, size_t n,
                             int log_n) {
    const long long N = 1ll << log_n;
    const cdbl* a = A + (long long)blockIdx.y * N;
    for (size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x; j < n; j += (size_t)gridDim.x * blockDim.x) {
        const uint32_t k = __brev(pos_brv[2 * j]) >> (32 - log_n);
        out[blockIdx.y * n + j] = a[k].re * inv_scale[blockIdx.y];
    }
}

cudaError_t launch_decode_fft(const uint64_t* const* m_dev, size_t count, uint64_t q0, const uint32_t* pos_brv,
                              const cdd* root, const cdd* twist, const double* inv_scale, int log_n, void* A,
                              double* out, size_t n, cudaStream_t st) {
    const long long N = 1ll << log_n;
    cdbl* a = reinterpret_cast<cdbl*>(A);
    dim3 gt((unsigned)((N + 255) / 256), (unsigned)count);
    k_dec_twist<<<gt, 256, 0, st>>>(m_dev, q0, twist, a, log_n);
    dim3 gf((unsigned)((N / 2 + 255) / 256), (unsigned)count);
    for (int s = 1; s <= log_n; s++) k_dec_fft_stage<<<gf, 256, 0, st>>>(a, root, log_n, s);
    if (n) {
        dim3 gg((unsigned)((n + 255) / 256), (unsigned)count);
        k_dec_gather<<<gg, 256, 0, st>>>(a, pos_brv, inv_scale, out, n, log_n);
    }
    return cudaGetLastError();
}

}  // namespace hisa
