// launch.h -- internal launch wrappers between the C-ABI host layer (hisa.cu) and the kernels.
// Not part of the public boundary (include/hisa.h is).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include "ntt.cuh"

namespace hisa {

int split_m1(int log_n);

// a1/a2 passes (ntt_kernels.cu)
cudaError_t launch_fwd_pass1(const PassJob& job, const Tables& tb, int nlimbs, int nz, bool lift, cudaStream_t st);
cudaError_t launch_fwd_pass2(const PassJob& job, const Tables& tb, int nlimbs, int nz, bool combine, cudaStream_t st);
cudaError_t launch_inv_passA(const PassJob& job, const Tables& tb, int nlimbs, int nz, cudaStream_t st);
cudaError_t launch_inv_passB(const PassJob& job, const Tables& tb, int nlimbs, int nz, cudaStream_t st);

// elementwise family (a3, a4) -- elem_kernels.cu.  Operates on nz ciphertexts, each with
// `npolys` polys of `nl` limbs (limb i mod mods[i]), word layout [poly][limb][N].
enum ElemOp {
    EL_ADD = 0, EL_SUB, EL_NEG, EL_ADD_PLAIN, EL_SUB_PLAIN, EL_MUL_PLAIN, EL_ADD_SCALAR, EL_MUL_SCALAR,
    EL_COPY, EL_TENSOR, EL_DECRYPT2, EL_DECRYPT3, EL_SQUARE_TENSOR
};
struct ElemJob {
    const uint64_t* a[MAXB];
    const uint64_t* b[MAXB];
    uint64_t* out[MAXB];
    int npolys;          // polys of a / out (for tensor: a,b have 2, out has 3)
    int nl;              // limbs per poly
    int log_n;
    long long a_poly, b_poly, out_poly;  // poly strides (words)
    uint64_t scal[MAXL];    // per-limb scalar residues (add/mul scalar)
    uint64_t scalp[MAXL];   // Shoup companions
    uint64_t fp_mods;       // bit i: limb i's products on the FP64 pipe (exact mulred); 0 = integer
    const double2* modd;    // (q, 1/q) per limb (needed when fp_mods != 0)
};
cudaError_t launch_elem(ElemOp op, const ElemJob& job, const Mod* mods, int nz, cudaStream_t st);

// automorphism psi_g in the NTT domain (K6): out[j] = in[perm_g[j]] on every limb; gs[z] is the
// Galois element of batch entry z (one per ciphertext: hoisted rotations permute by different g)
cudaError_t launch_automorphism(const uint64_t* const* in, uint64_t* const* out, int nz, int nlimbs_total,
                                int log_n, const uint64_t* gs, cudaStream_t st);

// the same with an optional addend per batch entry: out = add + psi_g(in) (rotate-and-sum step);
// limb index i of the nlimbs_total uses modulus mods[i % nl]
cudaError_t launch_automorphism_add(const uint64_t* const* in, uint64_t* const* out, const uint64_t* const* add,
                                    int nz, int nlimbs_total, int nl, int log_n, const uint64_t* gs, const Mod* mods,
                                    cudaStream_t st);

// mulPlain accumulation (FC): out_j = sum_c in_c (.) pt_{j,c}; device pointer arrays
struct MpaJob {
    int C, J, l1, log_n;
    int red_every;
    uint8_t limb_map[MAXL];   // grid.y -> limb (filled by the launcher: FP64 limbs, integer limbs)
};
cudaError_t launch_mulplain_acc(const uint64_t* const* in_ptrs, const uint64_t* const* pt_ptrs,
                                uint64_t* const* out_ptrs, const MpaJob& job, const Tables& tb, cudaStream_t st);

constexpr int MAXR = 8;

// K7 over CG ciphertexts sharing the R keys (every key word streamed once per CG ciphertexts)
constexpr int MAXCG = 4;
struct KsHoistMultiJob {
    const uint64_t* D[MAXCG];       // per ciphertext [j][ri][N] (diagonal blocks unused)
    const uint64_t* diag[MAXCG];    // per ciphertext digit source [(l+1)][N]
    const uint64_t* key[MAXR];      // R pre-permuted keys [kL][2][kL+1][N]
    uint64_t* acc[MAXCG][MAXR];     // out [2][l+2][N]
    int kL[MAXR];                   // q primes each key covers (truncated keys, kL >= l+1)
    int l1, L, cg;
    uint8_t mod_map[MAXL];
    uint8_t ri_list[MAXL];          // grid.y -> output prime (filled by the launcher)
};
cudaError_t launch_ks_ip_hoisted_multi(const KsHoistMultiJob& job, int R, const Tables& tb, cudaStream_t st);

// int64 sum of <= 8 fully reduced residue arrays (the NCCL reduce-scatter output, a15) -> residues
cudaError_t launch_reduce_sum(const int64_t* in, uint64_t* out, int npolys, int l1, int log_n, const Mod* mods,
                              cudaStream_t st);

// key-switch inner product fused with forward pass 2 (K4) -- ks_kernels.cu
struct KsJob {
    const uint64_t* t1[MAXB];     // pass-1 output [j][ri][N] (ri over l+2 output primes)
    const uint64_t* d[MAXB];      // the digit source in NTT form [(l+1)][N] (D_{j,q_j} = d_j)
    uint64_t* acc[MAXB];          // out [2][l+2][N], fully reduced
    const uint64_t* key;          // [L][2][L+1][N] (L = the key's q primes; truncated keys L < ctx L)
    int l1;                       // active limbs l+1
    int L;                        // q primes of the key: stride, and the special prime's key limb
    int nz;                       // ciphertexts in the batch (grid.x = tiles * nz)
    uint8_t mod_map[MAXL];        // ri -> modulus index
    uint8_t ri_list[MAXL];        // grid.y -> output prime ri (filled by launch_ks_ip)
    uint64_t fp_rows;             // bit ri: output prime ri runs the FP64 engine (q < 2^50)
};
// a second stream with fork / join events: independent launches of one step run side by side
struct SideStream {
    cudaStream_t s;
    cudaEvent_t fork, join;
};
cudaError_t launch_ks_ip(const KsJob& job, const Tables& tb, int nz, cudaStream_t st, const SideStream* side = nullptr);

// K8 on the tensor cores (conv_tc_kernels.cu): byte-split u8 x u8 -> s32 tcgen05 MMAs
struct ConvTcJob {
    int T, OC, log_n, n_chunks, n_oct;
    long long poly_stride;
    uint8_t limb_map[MAXL];       // grid.y -> limb
    uint8_t P[MAXL];              // byte planes per limb: ceil(bits(q) / 8)
};
size_t conv_tc_smem_bytes();
bool conv_tc_timed_out();   // an mbarrier wait of k_conv_tc exceeded its budget (flag cleared)
cudaError_t launch_conv_tc_wimg(const double* W, double ps, int T, int OC, int n_oct, int n_chunks, int l1,
                                const Mod* mods, const uint8_t* Pl, uint8_t* img, cudaStream_t st);
cudaError_t launch_conv_tc(const uint64_t* const* in_ptrs, uint64_t* const* out_ptrs, const uint8_t* wimg,
                           const ConvTcJob& job, int nlimbs, const Mod* mods, cudaStream_t st);

// GPU encode (NEXT-4, A7) -- encode_kernels.cu: double-double FFT + exact rounding with near-tie
// flags.  dd = unevaluated sum hi + lo; cdd = complex.
struct dd { double hi, lo; };
struct cdd { dd re, im; };
cudaError_t launch_encode_fft(const double* z_dev, size_t n_per, size_t count, const uint32_t* pos_brv,
                              const cdd* root, const cdd* twist, double scale_over_n, double window, int log_n,
                              cdd* A, int64_t* m, uint32_t* flags, unsigned int* nflag, unsigned int max_flags,
                              int* overflow, cudaStream_t st);
// GPU decode (NEXT-4): twist, N-point double FFT, gather of the slots' real parts; A holds
// count x N complex doubles (scratch)
cudaError_t launch_decode_fft(const uint64_t* const* m_dev, size_t count, uint64_t q0, const uint32_t* pos_brv,
                              const cdd* root, const cdd* twist, const double* inv_scale, int log_n, void* A,
                              double* out, size_t n, cudaStream_t st);

// samplers (ChaCha20, A11) -- rng_kernels.cu
cudaError_t launch_sample_uniform(uint64_t* out, uint64_t seed, uint32_t tag, const uint64_t* index_per_limb_host,
                                  const uint8_t* mod_per_limb_host, int nlimbs, int log_n, const Mod* mods,
                                  cudaStream_t st);
// int64 polynomial samplers: kind 0 = ternary, 1 = cbd
cudaError_t launch_sample_small(int64_t* out, uint64_t seed, uint32_t tag, uint64_t index, int kind, int log_n,
                                cudaStream_t st);
// reduce an int64 polynomial into limbs: out[i][t] = x[t] mod mods[mod_map[i]]
cudaError_t launch_int_to_limbs(const int64_t* x, uint64_t* out, const uint8_t* mod_map_host, int nlimbs, int log_n,
                                const Mod* mods, cudaStream_t st);
// integer-coefficient automorphism (used for rotation-key targets)
cudaError_t launch_automorphism_int(const int64_t* in, int64_t* out, int log_n, uint64_t g, cudaStream_t st);

}  // namespace hisa
