// elem_kernels.cu -- HBM-bound elementwise HISA ops (a3 add/sub/addPlain/addScalar/mulScalar/
// mulPlain, a4 tensor / mulNoRelin, decrypt) and the NTT-domain automorphism (K6, a7).
// 16-byte vector loads/stores, one pair of words per thread, grid = (pairs, ciphertexts).
#include <cuda_runtime.h>
#include "launch.h"
#include "ntt_f64.cuh"

namespace hisa {

template <int OP>
__global__ void __launch_bounds__(256) k_elem(ElemJob job, const Mod* __restrict__ mods) {
    const int z = blockIdx.z;
    const long long n2 = 1ll << (job.log_n - 1);               // word pairs per limb
    const long long per_poly = (long long)job.nl * n2;
    const int np_out = (OP == EL_TENSOR || OP == EL_SQUARE_TENSOR) ? 3
                     : (OP == EL_DECRYPT2 || OP == EL_DECRYPT3) ? 1 : job.npolys;
    (void)per_poly;
    (void)np_out;
    // grid (pairs of a limb, poly x limb, ciphertext): no 64-bit index divisions (the round-1
    // grid-stride form spent most of its issue slots on them: mulPlain at ~0.39 of HBM)
    {
        const long long pair = blockIdx.x * (long long)blockDim.x + threadIdx.x;
        if (pair >= n2) return;
        const int p = (int)blockIdx.y / job.nl;
        const int i = (int)blockIdx.y - p * job.nl;
        const long long w = pair * 2;                               // word offset in limb
        const Mod md = mods[i];
        const uint64_t q = md.q;
        const long long limb_off = (long long)i << job.log_n;
        const ulonglong2* A = reinterpret_cast<const ulonglong2*>(job.a[z] + p * job.a_poly + limb_off + w);
        ulonglong2* O = reinterpret_cast<ulonglong2*>(job.out[z] + p * job.out_poly + limb_off + w);
        if (OP == EL_ADD || OP == EL_SUB) {
            const ulonglong2 x = *A;
            const ulonglong2 y = *reinterpret_cast<const ulonglong2*>(job.b[z] + p * job.b_poly + limb_off + w);
            ulonglong2 r;
            if (OP == EL_ADD) { r.x = add_mod(x.x, y.x, q); r.y = add_mod(x.y, y.y, q); }
            else { r.x = sub_mod(x.x, y.x, q); r.y = sub_mod(x.y, y.y, q); }
            *O = r;
        } else if (OP == EL_NEG) {
            const ulonglong2 x = *A;
            *O = make_ulonglong2(neg_mod(x.x, q), neg_mod(x.y, q));
        } else if (OP == EL_COPY) {
            *O = *A;
        } else if (OP == EL_ADD_PLAIN || OP == EL_SUB_PLAIN) {
            ulonglong2 x = *A;
            if (p == 0) {
                const ulonglong2 y = *reinterpret_cast<const ulonglong2*>(job.b[z] + limb_off + w);
                if (OP == EL_ADD_PLAIN) { x.x = add_mod(x.x, y.x, q); x.y = add_mod(x.y, y.y, q); }
                else { x.x = sub_mod(x.x, y.x, q); x.y = sub_mod(x.y, y.y, q); }
            }
            *O = x;
        } else if (OP == EL_MUL_PLAIN) {
            const ulonglong2 x = *A;
            const ulonglong2 y = *reinterpret_cast<const ulonglong2*>(job.b[z] + limb_off + w);
            if ((job.fp_mods >> i) & 1) {   // exact FP64 product (q < 2^50): fewer issue slots than Barrett
                const double2 qd = job.modd[i];
                *O = make_ulonglong2(d_canon(mulred(u2d(x.x), u2d(y.x), qd.x, qd.y), qd.x, qd.y),
                                     d_canon(mulred(u2d(x.y), u2d(y.y), qd.x, qd.y), qd.x, qd.y));
            } else {
                *O = make_ulonglong2(mul_mod(x.x, y.x, md), mul_mod(x.y, y.y, md));
            }
        } else if (OP == EL_ADD_SCALAR) {
            ulonglong2 x = *A;
            if (p == 0) { x.x = add_mod(x.x, job.scal[i], q); x.y = add_mod(x.y, job.scal[i], q); }
            *O = x;
        } else if (OP == EL_MUL_SCALAR) {
            const ulonglong2 x = *A;
            const uint64_t s = job.scal[i], sp = job.scalp[i];
            *O = make_ulonglong2(mul_shoup(x.x, s, sp, q), mul_shoup(x.y, s, sp, q));
        } else if (OP == EL_TENSOR || OP == EL_SQUARE_TENSOR) {
            const ulonglong2 a0 = *reinterpret_cast<const ulonglong2*>(job.a[z] + limb_off + w);
            const ulonglong2 a1 = *reinterpret_cast<const ulonglong2*>(job.a[z] + job.a_poly + limb_off + w);
            ulonglong2 b0, b1;
            if (OP == EL_TENSOR) {
                b0 = *reinterpret_cast<const ulonglong2*>(job.b[z] + limb_off + w);
                b1 = *reinterpret_cast<const ulonglong2*>(job.b[z] + job.b_poly + limb_off + w);
            } else { b0 = a0; b1 = a1; }
            uint64_t* o = job.out[z] + limb_off + w;
            ulonglong2 r0, r1, r2;
            if ((job.fp_mods >> i) & 1) {   // exact FP64 products (q < 2^50)
                const double2 qd = job.modd[i];
                const double q_ = qd.x, qi_ = qd.y;
                const double x0 = u2d(a0.x), y0 = u2d(a0.y), x1 = u2d(a1.x), y1 = u2d(a1.y);
                const double u0 = u2d(b0.x), v0 = u2d(b0.y), u1 = u2d(b1.x), v1 = u2d(b1.y);
                r0 = make_ulonglong2(d_canon(mulred(x0, u0, q_, qi_), q_, qi_), d_canon(mulred(y0, v0, q_, qi_), q_, qi_));
                // a0 b1 + a1 b0: two exact products (each |.| < 0.88 q), one canonical reduction
                r1 = make_ulonglong2(d_canon(__dadd_rn(mulred(x0, u1, q_, qi_), mulred(x1, u0, q_, qi_)), q_, qi_),
                                     d_canon(__dadd_rn(mulred(y0, v1, q_, qi_), mulred(y1, v0, q_, qi_)), q_, qi_));
                r2 = make_ulonglong2(d_canon(mulred(x1, u1, q_, qi_), q_, qi_), d_canon(mulred(y1, v1, q_, qi_), q_, qi_));
                *reinterpret_cast<ulonglong2*>(o) = r0;
                *reinterpret_cast<ulonglong2*>(o + job.out_poly) = r1;
                *reinterpret_cast<ulonglong2*>(o + 2 * job.out_poly) = r2;
                return;
            }
            r0.x = mul_mod(a0.x, b0.x, md); r0.y = mul_mod(a0.y, b0.y, md);
            // a0 b1 + a1 b0 with one reduction: sum of two 120-bit products fits 128 bits
            {
                U128 s{0, 0};
                mac128(s, a0.x, b1.x); mac128(s, a1.x, b0.x);
                r1.x = barrett128(s.lo, s.hi, md);
                U128 u{0, 0};
                mac128(u, a0.y, b1.y); mac128(u, a1.y, b0.y);
                r1.y = barrett128(u.lo, u.hi, md);
            }
            r2.x = mul_mod(a1.x, b1.x, md); r2.y = mul_mod(a1.y, b1.y, md);
            *reinterpret_cast<ulonglong2*>(o) = r0;
            *reinterpret_cast<ulonglong2*>(o + job.out_poly) = r1;
            *reinterpret_cast<ulonglong2*>(o + 2 * job.out_poly) = r2;
        } else if (OP == EL_DECRYPT2 || OP == EL_DECRYPT3) {
            // b = secret key NTT limbs; out = c0 + c1 s (+ c2 s^2)
            const ulonglong2 s = *reinterpret_cast<const ulonglong2*>(job.b[z] + limb_off + w);
            const ulonglong2 c0 = *reinterpret_cast<const ulonglong2*>(job.a[z] + limb_off + w);
            const ulonglong2 c1 = *reinterpret_cast<const ulonglong2*>(job.a[z] + job.a_poly + limb_off + w);
            ulonglong2 r;
            r.x = add_mod(c0.x, mul_mod(c1.x, s.x, md), q);
            r.y = add_mod(c0.y, mul_mod(c1.y, s.y, md), q);
            if (OP == EL_DECRYPT3) {
                const ulonglong2 c2 = *reinterpret_cast<const ulonglong2*>(job.a[z] + 2 * job.a_poly + limb_off + w);
                r.x = add_mod(r.x, mul_mod(c2.x, mul_mod(s.x, s.x, md), md), q);
                r.y = add_mod(r.y, mul_mod(c2.y, mul_mod(s.y, s.y, md), md), q);
            }
            *reinterpret_cast<ulonglong2*>(job.out[z] + limb_off + w) = r;
        }
    }
}

// The HBM-bound binary ops with TWO word pairs per thread (pairs x and x + 256 of a 512-pair block),
// all loads issued before the arithmetic: twice the bytes in flight per thread.  One pair per thread
// left mulPlain at ~0.5 of measured HBM at N = 2^16 (profiles/r2_config2_sweep.txt): 2048 threads x
// 32 B per SM in flight against ~3 us of loaded latency.  Same arithmetic as k_elem, bit for bit.
template <int OP>
__global__ void __launch_bounds__(256) k_elem2(ElemJob job, const Mod* __restrict__ mods) {
    constexpr int U = 2;
    const int z = blockIdx.z;
    const int p = (int)blockIdx.y / job.nl;
    const int i = (int)blockIdx.y - p * job.nl;
    const long long w0 = (blockIdx.x * (256ll * U) + threadIdx.x) * 2;   // pair u at word w0 + 512 u
    const Mod md = mods[i];
    const uint64_t q = md.q;
    const long long limb_off = (long long)i << job.log_n;
    auto ld = [](const uint64_t* a) { return *reinterpret_cast<const ulonglong2*>(a); };
    auto st = [](uint64_t* a, ulonglong2 v) { *reinterpret_cast<ulonglong2*>(a) = v; };
    if (OP == EL_ADD || OP == EL_SUB || OP == EL_MUL_PLAIN) {
        const uint64_t* A = job.a[z] + p * job.a_poly + limb_off + w0;
        const uint64_t* B = job.b[z] + (OP == EL_MUL_PLAIN ? 0 : p * job.b_poly) + limb_off + w0;
        uint64_t* O = job.out[z] + p * job.out_poly + limb_off + w0;
        ulonglong2 x[U], y[U];
#pragma unroll
        for (int u = 0; u < U; u++) { x[u] = ld(A + 512 * u); y[u] = ld(B + 512 * u); }
        const bool fp = OP == EL_MUL_PLAIN && ((job.fp_mods >> i) & 1);
        double2 qd = make_double2(0.0, 0.0);
        if (fp) qd = job.modd[i];
#pragma unroll
        for (int u = 0; u < U; u++) {
            ulonglong2 r;
            if (OP == EL_ADD) { r.x = add_mod(x[u].x, y[u].x, q); r.y = add_mod(x[u].y, y[u].y, q); }
            else if (OP == EL_SUB) { r.x = sub_mod(x[u].x, y[u].x, q); r.y = sub_mod(x[u].y, y[u].y, q); }
            else if (fp) {
                r = make_ulonglong2(d_canon(mulred(u2d(x[u].x), u2d(y[u].x), qd.x, qd.y), qd.x, qd.y),
                                    d_canon(mulred(u2d(x[u].y), u2d(y[u].y), qd.x, qd.y), qd.x, qd.y));
            } else {
                r = make_ulonglong2(mul_mod(x[u].x, y[u].x, md), mul_mod(x[u].y, y[u].y, md));
            }
            st(O + 512 * u, r);
        }
    } else {   // EL_TENSOR / EL_SQUARE_TENSOR
        const uint64_t* A = job.a[z] + limb_off + w0;
        const uint64_t* B = job.b[z] + limb_off + w0;
        uint64_t* o = job.out[z] + limb_off + w0;
        ulonglong2 a0[U], a1[U], b0[U], b1[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            a0[u] = ld(A + 512 * u);
            a1[u] = ld(A + job.a_poly + 512 * u);
            if (OP == EL_TENSOR) { b0[u] = ld(B + 512 * u); b1[u] = ld(B + job.b_poly + 512 * u); }
            else { b0[u] = a0[u]; b1[u] = a1[u]; }
        }
        const bool fp = (job.fp_mods >> i) & 1;
        double2 qd = make_double2(0.0, 0.0);
        if (fp) qd = job.modd[i];
#pragma unroll
        for (int u = 0; u < U; u++) {
            ulonglong2 r0, r1, r2;
            if (fp) {
                const double q_ = qd.x, qi_ = qd.y;
                const double x0 = u2d(a0[u].x), y0 = u2d(a0[u].y), x1 = u2d(a1[u].x), y1 = u2d(a1[u].y);
                const double u0 = u2d(b0[u].x), v0 = u2d(b0[u].y), u1 = u2d(b1[u].x), v1 = u2d(b1[u].y);
                r0 = make_ulonglong2(d_canon(mulred(x0, u0, q_, qi_), q_, qi_), d_canon(mulred(y0, v0, q_, qi_), q_, qi_));
                r1 = make_ulonglong2(d_canon(__dadd_rn(mulred(x0, u1, q_, qi_), mulred(x1, u0, q_, qi_)), q_, qi_),
                                     d_canon(__dadd_rn(mulred(y0, v1, q_, qi_), mulred(y1, v0, q_, qi_)), q_, qi_));
                r2 = make_ulonglong2(d_canon(mulred(x1, u1, q_, qi_), q_, qi_), d_canon(mulred(y1, v1, q_, qi_), q_, qi_));
            } else {
                r0.x = mul_mod(a0[u].x, b0[u].x, md); r0.y = mul_mod(a0[u].y, b0[u].y, md);
                U128 s{0, 0};
                mac128(s, a0[u].x, b1[u].x); mac128(s, a1[u].x, b0[u].x);
                r1.x = barrett128(s.lo, s.hi, md);
                U128 t{0, 0};
                mac128(t, a0[u].y, b1[u].y); mac128(t, a1[u].y, b0[u].y);
                r1.y = barrett128(t.lo, t.hi, md);
                r2.x = mul_mod(a1[u].x, b1[u].x, md); r2.y = mul_mod(a1[u].y, b1[u].y, md);
            }
            st(o + 512 * u, r0);
            st(o + job.out_poly + 512 * u, r1);
            st(o + 2 * job.out_poly + 512 * u, r2);
        }
    }
}

static int sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

cudaError_t launch_elem(ElemOp op, const ElemJob& job, const Mod* mods, int nz, cudaStream_t st) {
    const int np = (op == EL_TENSOR || op == EL_SQUARE_TENSOR || op == EL_DECRYPT2 || op == EL_DECRYPT3) ? 1
                                                                                                      : job.npolys;
    const long long n2 = 1ll << (job.log_n - 1);
    dim3 grid((unsigned)((n2 + 255) / 256), (unsigned)(np * job.nl), (unsigned)nz);
    if (n2 % 512 == 0) {   // two pairs per thread for the HBM-bound binary ops
        dim3 g2((unsigned)(n2 / 512), grid.y, grid.z);
        switch (op) {
#define C2(OPV) case OPV: k_elem2<OPV><<<g2, 256, 0, st>>>(job, mods); return cudaGetLastError();
            C2(EL_ADD) C2(EL_SUB) C2(EL_MUL_PLAIN) C2(EL_TENSOR) C2(EL_SQUARE_TENSOR)
#undef C2
            default: break;
        }
    }
    switch (op) {
#define C(OPV) case OPV: k_elem<OPV><<<grid, 256, 0, st>>>(job, mods); break;
        C(EL_ADD) C(EL_SUB) C(EL_NEG) C(EL_ADD_PLAIN) C(EL_SUB_PLAIN) C(EL_MUL_PLAIN) C(EL_ADD_SCALAR)
        C(EL_MUL_SCALAR) C(EL_COPY) C(EL_TENSOR) C(EL_DECRYPT2) C(EL_DECRYPT3) C(EL_SQUARE_TENSOR)
#undef C
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// NTT-domain automorphism (A15, K6): slot j holds a(psi^(2 brv(j)+1)); psi_g(a) at slot j is
// a at slot perm[j] = brv(((2 brv(j) + 1) g mod 2N - 1) / 2).
// ------------------------------------------------------------------------------------------
struct PtrPack {
    const uint64_t* in[MAXB];
    uint64_t* out[MAXB];
    const uint64_t* add[MAXB];   // optional addend (rotate-and-sum): out = add + psi_g(in)
    uint64_t g[MAXB];
    const Mod* mods;
    int nl;                      // limbs per poly (modulus of limb index i = mods[i % nl])
};
__global__ void __launch_bounds__(256) k_automorphism(PtrPack pk, int log_n) {
    const int z = blockIdx.z;
    const int limb = blockIdx.y;
    const uint32_t N = 1u << log_n;
    const uint64_t mask2n = 2ull * N - 1;
    const uint64_t g = pk.g[z];
    const uint64_t* in = pk.in[z] + ((long long)limb << log_n);
    uint64_t* out = pk.out[z] + ((long long)limb << log_n);
    const uint64_t* add = pk.add[z] ? pk.add[z] + ((long long)limb << log_n) : nullptr;
    const uint64_t q = add ? pk.mods[limb % pk.nl].q : 0;
    // word pairs (j, j + 1), j even: their sources are the pair (s, s ^ 1) -- j and j + 1 differ in
    // the top bit of brev(j), which moves (e - 1) / 2 by N / 2 (g odd), i.e. flips bit 0 of the
    // source -- so both directions are 16-byte accesses
    for (uint32_t j = 2 * (blockIdx.x * blockDim.x + threadIdx.x); j < N; j += 2 * gridDim.x * blockDim.x) {
        const uint32_t bj = __brev(j) >> (32 - log_n);
        const uint64_t e = ((2ull * bj + 1) * g) & mask2n;
        const uint32_t src = __brev((uint32_t)((e - 1) >> 1)) >> (32 - log_n);
        const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(in + (src & ~1u));
        ulonglong2 o = (src & 1) ? make_ulonglong2(v.y, v.x) : v;
        if (add) {
            const ulonglong2 a = *reinterpret_cast<const ulonglong2*>(add + j);
            o = make_ulonglong2(add_mod(o.x, a.x, q), add_mod(o.y, a.y, q));
        }
        *reinterpret_cast<ulonglong2*>(out + j) = o;
    }
}

cudaError_t launch_automorphism_add(const uint64_t* const* in, uint64_t* const* out, const uint64_t* const* add,
                                    int nz, int nlimbs_total, int nl, int log_n, const uint64_t* gs, const Mod* mods,
                                    cudaStream_t st) {
    PtrPack pk;
    for (int z = 0; z < nz; z++) {
        pk.in[z] = in[z]; pk.out[z] = out[z]; pk.g[z] = gs[z]; pk.add[z] = add ? add[z] : nullptr;
    }
    pk.mods = mods;
    pk.nl = nl;
    const int N = 1 << log_n;
    for (int l0 = 0; l0 < nlimbs_total; l0 += 65535) {
        const int nlc = nlimbs_total - l0 < 65535 ? nlimbs_total - l0 : 65535;
        PtrPack pz = pk;
        for (int z = 0; z < nz; z++) {
            pz.in[z] += ((long long)l0 << log_n);
            pz.out[z] += ((long long)l0 << log_n);
            if (pz.add[z]) pz.add[z] += ((long long)l0 << log_n);
        }
        dim3 grid((N / 2 + 255) / 256, nlc, nz);
        k_automorphism<<<grid, 256, 0, st>>>(pz, log_n);
    }
    return cudaGetLastError();
}

cudaError_t launch_automorphism(const uint64_t* const* in, uint64_t* const* out, int nz, int nlimbs_total, int log_n,
                                const uint64_t* gs, cudaStream_t st) {
    PtrPack pk;
    for (int z = 0; z < nz; z++) { pk.in[z] = in[z]; pk.out[z] = out[z]; pk.g[z] = gs[z]; pk.add[z] = nullptr; }
    pk.mods = nullptr;
    pk.nl = 1;
    const int N = 1 << log_n;
    for (int l0 = 0; l0 < nlimbs_total; l0 += 65535) {   // grid.y limit (keys have 2 L (L+1) limbs)
        const int nl = nlimbs_total - l0 < 65535 ? nlimbs_total - l0 : 65535;
        PtrPack pz = pk;
        for (int z = 0; z < nz; z++) { pz.in[z] += ((long long)l0 << log_n); pz.out[z] += ((long long)l0 << log_n); }
        dim3 grid((N / 2 + 255) / 256, nl, nz);
        k_automorphism<<<grid, 256, 0, st>>>(pz, log_n);
    }
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// a15 exchange fix-up: the int64 SUM of <= 8 reduced residue arrays (< 2^63) back to [0, q_i)
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_reduce_sum(const int64_t* __restrict__ in, uint64_t* __restrict__ out,
                                                    long long total, int l1, int log_n, const Mod* __restrict__ mods) {
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int i = (int)((idx >> log_n) % l1);
        out[idx] = barrett64((uint64_t)in[idx], mods[i]);
    }
}

cudaError_t launch_reduce_sum(const int64_t* in, uint64_t* out, int npolys, int l1, int log_n, const Mod* mods,
                              cudaStream_t st) {
    const long long total = ((long long)npolys * l1) << log_n;
    long long blocks = (total + 255) / 256;
    if (blocks > (long long)sm_count() * 8) blocks = (long long)sm_count() * 8;
    k_reduce_sum<<<(unsigned)blocks, 256, 0, st>>>(in, out, total, l1, log_n, mods);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// mulPlain accumulation (FC / matmul): out_j = sum_c in_c (.) pt_{j,c} for j < J, both
// ciphertext polys.  HBM stream of the J*C plaintext limbs; OT outputs per pass in 128-bit
// register accumulators (products < 2^120, partial Barrett every red_every terms).
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_mulplain_acc(const uint64_t* const* __restrict__ in_ptrs,
                                                      const uint64_t* const* __restrict__ pt_ptrs,
                                                      uint64_t* const* __restrict__ out_ptrs, MpaJob job,
                                                      const Mod* __restrict__ mods) {
    constexpr int OT = 4;
    extern __shared__ uint64_t msm[];
    const uint64_t** ins = reinterpret_cast<const uint64_t**>(msm);   // [C]
    const long long N = 1ll << job.log_n;
    const int limb = job.limb_map[blockIdx.y];
    const Mod md = mods[limb];
    const long long loff = (long long)limb * N;
    const long long x = 2ll * (blockIdx.x * (long long)blockDim.x + threadIdx.x);
    for (int c = threadIdx.x; c < job.C; c += blockDim.x) ins[c] = in_ptrs[c] + loff;
    __syncthreads();
    if (x >= N) return;
    const long long pstride = (long long)job.l1 * N;   // poly stride of a ciphertext
    for (int j0 = 0; j0 < job.J; j0 += OT) {
        U128 acc[OT][2][2];
#pragma unroll
        for (int k = 0; k < OT; k++)
#pragma unroll
            for (int p = 0; p < 2; p++) { acc[k][p][0] = U128{0, 0}; acc[k][p][1] = U128{0, 0}; }
        int since = 0;
        for (int c = 0; c < job.C; c++) {
            const ulonglong2 a0 = __ldg(reinterpret_cast<const ulonglong2*>(ins[c] + x));
            const ulonglong2 a1 = __ldg(reinterpret_cast<const ulonglong2*>(ins[c] + pstride + x));
#pragma unroll
            for (int k = 0; k < OT; k++) {
                if (j0 + k >= job.J) break;
                const ulonglong2 pv =
                    __ldcs(reinterpret_cast<const ulonglong2*>(pt_ptrs[(long long)(j0 + k) * job.C + c] + loff + x));
                mac128(acc[k][0][0], a0.x, pv.x);
                mac128(acc[k][0][1], a0.y, pv.y);
                mac128(acc[k][1][0], a1.x, pv.x);
                mac128(acc[k][1][1], a1.y, pv.y);
            }
            if (++since == job.red_every) {
                since = 0;
#pragma unroll
                for (int k = 0; k < OT; k++)
#pragma unroll
                    for (int p = 0; p < 2; p++)
#pragma unroll
                        for (int h = 0; h < 2; h++) {
                            acc[k][p][h].lo = barrett128(acc[k][p][h].lo, acc[k][p][h].hi, md);
                            acc[k][p][h].hi = 0;
                        }
            }
        }
#pragma unroll
        for (int k = 0; k < OT; k++) {
            if (j0 + k >= job.J) break;
#pragma unroll
            for (int p = 0; p < 2; p++)
                *reinterpret_cast<ulonglong2*>(out_ptrs[j0 + k] + p * pstride + loff + x) =
                    make_ulonglong2(barrett128(acc[k][p][0].lo, acc[k][p][0].hi, md),
                                    barrett128(acc[k][p][1].lo, acc[k][p][1].hi, md));
        }
    }
}

// FP64 limbs (q < 2^50): out_j = sum_c x_c p_jc accumulated as exact mulred products (both < q:
// |mulred| < 0.88 q) in doubles, re-centred every 8 terms (|acc| < 7.6 q < 2^53) -- two registers
// per accumulator instead of a 128-bit pair, so OT = 8 neurons per pass (each input word re-read
// J / 8 times), and the FP64 pipe's MAC rate instead of the integer pipe's
template <int OT>
__global__ void __launch_bounds__(256) k_mulplain_acc_f64(const uint64_t* const* __restrict__ in_ptrs,
                                                          const uint64_t* const* __restrict__ pt_ptrs,
                                                          uint64_t* const* __restrict__ out_ptrs, MpaJob job,
                                                          Tables tb) {
    // every thread's 2 ciphertext word pairs and OT plaintext word pairs of input c + 1 are copied
    // into its own slots of a double-buffered shared stage (cp.async, 16 B each) while input c is
    // multiplied -- the direct-load form ran at 0.33 of HBM (profiles/r2_ncu_elem.txt: issue 14 %,
    // 16 warps per SM at 128 registers, every iteration waiting on its own loads)
    constexpr int W = 2 + OT;
    extern __shared__ __align__(16) uint64_t msm[];
    ulonglong2* stage = reinterpret_cast<ulonglong2*>(msm);                          // [2][W][256]
    const uint64_t** ins = reinterpret_cast<const uint64_t**>(msm + 2 * W * 256 * 2);   // [C]
    const long long N = 1ll << job.log_n;
    const int limb = job.limb_map[blockIdx.y];
    const double2 qd = tb.modd[limb];
    const double q = qd.x, qinv = qd.y;
    const long long loff = (long long)limb * N;
    const int tid = threadIdx.x;
    const long long x = 2ll * (blockIdx.x * (long long)blockDim.x + tid);
    for (int c = tid; c < job.C; c += blockDim.x) ins[c] = in_ptrs[c] + loff;
    __syncthreads();
    if (x >= N) return;
    const long long pstride = (long long)job.l1 * N;
    auto cp16 = [](const void* dst, const void* src) {
        const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src) : "memory");
    };
    for (int j0 = 0; j0 < job.J; j0 += OT) {
        auto issue = [&](int c, int buf) {
            ulonglong2* st = stage + buf * W * 256 + tid;
            cp16(st, ins[c] + x);
            cp16(st + 256, ins[c] + pstride + x);
#pragma unroll
            for (int k = 0; k < OT; k++)
                if (j0 + k < job.J) cp16(st + (2 + k) * 256, pt_ptrs[(long long)(j0 + k) * job.C + c] + loff + x);
            asm volatile("cp.async.commit_group;\n" ::: "memory");
        };
        double acc[OT][2][2];
#pragma unroll
        for (int k = 0; k < OT; k++)
#pragma unroll
            for (int p = 0; p < 2; p++) { acc[k][p][0] = 0.0; acc[k][p][1] = 0.0; }
        issue(0, 0);
        for (int c = 0; c < job.C; c++) {
            if (c + 1 < job.C) {
                issue(c + 1, (c + 1) & 1);
                asm volatile("cp.async.wait_group 1;\n" ::: "memory");
            } else {
                asm volatile("cp.async.wait_group 0;\n" ::: "memory");
            }
            const ulonglong2* st = stage + (c & 1) * W * 256 + tid;
            const ulonglong2 a0 = st[0], a1 = st[256];
            const double a00 = u2d(a0.x), a01 = u2d(a0.y), a10 = u2d(a1.x), a11 = u2d(a1.y);
#pragma unroll
            for (int k = 0; k < OT; k++) {
                if (j0 + k >= job.J) break;
                const ulonglong2 pv = st[(2 + k) * 256];
                const double p0 = u2d(pv.x), p1 = u2d(pv.y);
                acc[k][0][0] = __dadd_rn(acc[k][0][0], mulred(a00, p0, q, qinv));
                acc[k][0][1] = __dadd_rn(acc[k][0][1], mulred(a01, p1, q, qinv));
                acc[k][1][0] = __dadd_rn(acc[k][1][0], mulred(a10, p0, q, qinv));
                acc[k][1][1] = __dadd_rn(acc[k][1][1], mulred(a11, p1, q, qinv));
            }
            if ((c & 7) == 7) {
#pragma unroll
                for (int k = 0; k < OT; k++)
#pragma unroll
                    for (int p = 0; p < 2; p++) {
                        acc[k][p][0] = redd(acc[k][p][0], q, qinv);
                        acc[k][p][1] = redd(acc[k][p][1], q, qinv);
                    }
            }
        }
#pragma unroll
        for (int k = 0; k < OT; k++) {
            if (j0 + k >= job.J) break;
#pragma unroll
            for (int p = 0; p < 2; p++)
                *reinterpret_cast<ulonglong2*>(out_ptrs[j0 + k] + p * pstride + loff + x) =
                    make_ulonglong2(d_canon(acc[k][p][0], q, qinv), d_canon(acc[k][p][1], q, qinv));
        }
    }
}

cudaError_t launch_mulplain_acc(const uint64_t* const* in_ptrs, const uint64_t* const* pt_ptrs,
                                uint64_t* const* out_ptrs, const MpaJob& job_in, const Tables& tb, cudaStream_t st) {
    const long long N = 1ll << job_in.log_n;
    const size_t smem = (size_t)job_in.C * sizeof(void*);
    MpaJob jf = job_in, ji = job_in;
    int nf = 0, ni = 0;
    for (int i = 0; i < job_in.l1; i++) {
        if ((tb.fp_mods >> i) & 1) jf.limb_map[nf++] = (uint8_t)i;
        else ji.limb_map[ni++] = (uint8_t)i;
    }
    if (ni) {
        dim3 grid((unsigned)((N / 2 + 255) / 256), ni, 1);
        if (smem > 48 * 1024) cudaFuncSetAttribute(k_mulplain_acc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_mulplain_acc<<<grid, 256, smem, st>>>(in_ptrs, pt_ptrs, out_ptrs, ji, tb.mods);
    }
    if (nf) {
        dim3 grid((unsigned)((N / 2 + 255) / 256), nf, 1);
        const size_t smem_f = smem + (size_t)2 * (2 + 8) * 256 * 16;   // + the cp.async stage
        cudaFuncSetAttribute(k_mulplain_acc_f64<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_f);
        k_mulplain_acc_f64<8><<<grid, 256, smem_f, st>>>(in_ptrs, pt_ptrs, out_ptrs, jf, tb);
    }
    return cudaGetLastError();
}

}  // namespace hisa
