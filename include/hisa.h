/*
 * hisa.h -- C-ABI boundary of the B200 RNS-CKKS HISA library (libhisa.so).
 *
 * The instruction set follows the paper's HISA table (PAPER.md, CHET arXiv 1810.00845):
 * Encryption profile (encrypt/decrypt/copy/free), Integers profile (encode/decode,
 * rotLeft/rotRight, add/sub/mul in ct/plain/scalar forms), Division profile
 * (divScalar / maxScalarDiv with the RNS semantics of P:584-587), Relin profile (mulNoRelin /
 * relinearize) and Bootstrap (unsupported).  Initialisation and key
 * generation sit outside the HISA.  Modulus switch, hoisted / batched rotation and
 * the import/export calls are extensions for the hot path and the parity harness.
 *
 * Scheme: full-RNS CKKS, NTT-domain storage, hybrid key switching with dnum = L, one
 * special prime (readings A1-A20).  Every device kernel is sm_100a CUDA; there is no
 * CPU fallback: without a CUDA device hisa_ctx_create fails with HISA_E_CUDA.
 *
 * Conventions
 *  - Every function returns int: HISA_OK (0) or a negative HISA_E_* code; hisa_last_error()
 *    returns a thread-local message for the last failure.
 *  - All argument / level / scale checks are done synchronously on the host BEFORE any launch.
 *    Kernels are enqueued asynchronously on the context stream; device faults surface at the next
 *    synchronising call (hisa_sync, *_export, hisa_decode, hisa_decrypt...) as HISA_E_CUDA and
 *    poison the context (every later call returns HISA_E_CUDA).
 *  - Handles (hisa_ct, hisa_pt) are opaque 64-bit values (generation << 32 | slot); a freed or
 *    never-issued handle gives HISA_E_INVALID_HANDLE (use-after-free detection).  Handle 0 is
 *    never valid.  The context owns all handle storage; hisa_free releases it.
 *  - Output handles: `out` receives a fresh handle; for the instructions with an *Assign form
 *    in the HISA table (rot, add, sub, mul, divScalar ...), passing out == NULL performs the
 *    operation in place on the first operand's handle.
 *  - Host buffers passed in are copied before the call returns; host buffers passed out are
 *    written before it returns.  Device memory comes from an arena the caller attaches
 *    (hisa_attach_arena, e.g. a torch tensor, so PyTorch owns device memory) or, if none is
 *    attached, from cudaMallocAsync on the context stream.
 *  - A context is single-owner and not thread-safe; one context per (process, device).
 *  - Word layout of a ciphertext / plaintext (device and export): uint64 [poly][limb][N],
 *    limb i reduced mod q_i in [0, q_i), NTT domain in bit-reversed evaluation order (A5):
 *    word j of a limb holds a(psi^(2 brv(j) + 1)).
 *  - Level l means limbs q_0..q_l are active (l + 1 limbs).  Fresh encryptions are at the level
 *    of their plaintext (top = L - 1 by default).
 */
#ifndef HISA_H
#define HISA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hisa_ctx hisa_ctx;
typedef uint64_t hisa_ct;
typedef uint64_t hisa_pt;

enum {
    HISA_OK = 0,
    HISA_E_INVALID_HANDLE = -1,     /* freed / unknown handle, or wrong kind          */
    HISA_E_UNSUPPORTED_PROFILE = -2,/* Bootstrap profile                             */
    HISA_E_LEVEL_MISMATCH = -3,     /* operands at different levels (no silent mod-switch)       */
    HISA_E_SCALE_MISMATCH = -4,     /* |s_a / s_b - 1| > 2^-30 for add/sub (A8)                   */
    HISA_E_INVALID_DIVISOR = -5,    /* divScalar by d not in {1, q_top} (A18)          */
    HISA_E_MODULUS_EXHAUSTED = -6,  /* rescale / mod-switch below level 0                         */
    HISA_E_NO_KEY = -7,             /* rotation amount without a generated key        */
    HISA_E_CAPACITY = -8,           /* more than N/2 slot values                          */
    HISA_E_NOT_RELINEARIZED = -9,   /* 3-poly ciphertext where a 2-poly one is required (A17)     */
    HISA_E_OOM = -10,               /* arena / device allocation failed                          */
    HISA_E_CUDA = -11,              /* CUDA error; the context is poisoned                       */
    HISA_E_PARAMS = -12,            /* invalid parameters / arguments / buffer sizes              */
    HISA_E_NO_SECRET = -13          /* decrypt / keygen-dependent call before hisa_keygen          */
};

enum {
    HISA_PROFILE_ENCRYPTION = 1,
    HISA_PROFILE_INTEGERS = 2,
    HISA_PROFILE_DIVISION = 4,
    HISA_PROFILE_RELIN = 8,
    HISA_PROFILE_BOOTSTRAP = 16
};

/*
 * Parameters (outside the HISA).
 *   log_n   : ring degree N = 2^log_n, 8 <= log_n <= 16; N/2 complex slots.
 *   num_q   : L, number of ciphertext primes q_0..q_{L-1} (A29), 1 <= L <= 60.
 *   q_bits  : L bit sizes, bottom (q_0) first; p_bits: the single special prime (A14).
 *             Primes are the largest q = 1 mod 2N below 2^bits, special prime first (A3);
 *             bit sizes must lie in [20, 60].
 *   seed    : ChaCha20 key for every sampled object (A11).
 *   device  : CUDA device ordinal.
 */
typedef struct {
    int log_n;
    int num_q;
    const int* q_bits;
    int p_bits;
    uint64_t seed;
    int device;
} hisa_params;

/* ---- context --------------------------------------------------------------------------- */
int hisa_ctx_create(const hisa_params* params, hisa_ctx** out);
int hisa_ctx_destroy(hisa_ctx* ctx);
/* dev_ptr: caller-owned device memory of `bytes` bytes used for every ciphertext/plaintext/key/
 * scratch allocation of this context; must outlive the context.  Call before any allocation. */
int hisa_attach_arena(hisa_ctx* ctx, void* dev_ptr, size_t bytes);
/* stream: a cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream); synchronises first. */
int hisa_set_stream(hisa_ctx* ctx, void* stream);
int hisa_sync(hisa_ctx* ctx);
/* 1 if the profile is implemented (Bootstrap -> 0) */
int hisa_supports(const hisa_ctx* ctx, int profile);
/* moduli: writes q_0..q_{L-1}, p (n >= L + 1 words) */
int hisa_moduli(const hisa_ctx* ctx, uint64_t* out, size_t n);
int hisa_ring_degree(const hisa_ctx* ctx, uint64_t* n_out, int* num_q_out);
/* bytes currently allocated from the arena / pool, and the high-water mark */
int hisa_mem_stats(const hisa_ctx* ctx, size_t* in_use, size_t* peak);

/* ---- keys (outside the HISA) ---------------------------- */
/* Generates (once) the secret key, public key and, if relin != 0, the relinearisation key, plus
 * one key-switching key per distinct left-rotation amount (k mod N/2, k != 0), as the compiler's
 * rotation-key selection would request.  May be called again to add rotation keys.
 * max_level (-1 = top, else 0 <= max_level < L): the rotation keys of this call are stored
 * truncated to the highest level they serve (digits j <= max_level, moduli q_0..q_max_level and
 * p: kL = max_level + 1 primes, [kL][2][kL+1][N] words -- the same words as the full key's
 * blocks); a rotation at a level above its key's fails with HISA_E_NO_KEY.  Asking again for an
 * existing amount at a higher max_level regenerates it; at a lower one keeps it.  The
 * relinearisation key is always full.  HISA_E_PARAMS for max_level out of range. */
int hisa_keygen(hisa_ctx* ctx, const int64_t* rot_left_amounts, size_t n, int relin, int max_level);
/* which = -1 public key [2][L][N]; -2 secret key NTT [(L+1)][N]; 0 relin key; k>0 rotation key k
 * ([kL][2][kL+1][N], kL = its max_level + 1, canonical NTT order); words must equal the object
 * size. */
int hisa_key_export(hisa_ctx* ctx, int64_t which, uint64_t* host, size_t words);

/* ---- Encryption profile ------------------------------------------------------ */
/* public-key encryption at the plaintext's level and scale (A12); consumes one encryption
 * counter value for its ChaCha20 streams */
int hisa_encrypt(hisa_ctx* ctx, hisa_pt pt, hisa_ct* out);
/* m = c0 + c1 s (+ c2 s^2), all limbs of the ciphertext's level; synchronising */
int hisa_decrypt(hisa_ctx* ctx, hisa_ct ct, hisa_pt* out);
int hisa_copy(hisa_ctx* ctx, hisa_ct ct, hisa_ct* out);
int hisa_free(hisa_ctx* ctx, uint64_t handle);

/* ---- Integers profile -------------------------------------------------------- */
/* real slot values v[0..n) (n <= N/2, else HISA_E_CAPACITY), missing slots zero; coefficients
 * m_t = round-half-away((scale/N) sum_j 2 v_j cos(pi (5^j t mod 2N)/N)) (A7), level -1 = top */
int hisa_encode(hisa_ctx* ctx, const double* v, size_t n, double scale, int level, hisa_pt* out);
/* count plaintexts at once: v = count rows of n_per values (row-major), same scale and level;
 * encoded on the GPU (double-double FFT, the same exact rounding as hisa_encode, near ties
 * recomputed in binary128 on the host), limbs + NTT batched; outs[count].  For a layer's
 * weight / mask plaintexts (once per model). */
int hisa_encode_batch(hisa_ctx* ctx, const double* v, size_t n_per, size_t count, double scale, int level,
                      hisa_pt* outs);
/* slot values from limb 0 (A13): needs |value| * scale < q_0 / 2; out[0..n), the real
 * parts (A2).  On the GPU: INTT of limb 0, centred lift, twist, N-point double-precision FFT,
 * gather (decode is approximate by definition: error ~ log2(N) 2^-53 max|m_t| / scale).
 * Synchronising; HISA_E_CAPACITY for n > N/2. */
int hisa_decode(hisa_ctx* ctx, hisa_pt pt, double* out, size_t n);
/* count plaintexts at once: out[count][n] row-major, each row as hisa_decode (batched launches) */
int hisa_decode_batch(hisa_ctx* ctx, const hisa_pt* pts, size_t count, double* out, size_t n);
/* rotate left/right by k slots: out[i] = in[(i + k) mod N/2] (A15); k = 0 copies */
int hisa_rot_left(hisa_ctx* ctx, hisa_ct ct, int64_t k, hisa_ct* out);
int hisa_rot_right(hisa_ctx* ctx, hisa_ct ct, int64_t k, hisa_ct* out);
int hisa_add(hisa_ctx* ctx, hisa_ct a, hisa_ct b, hisa_ct* out);
int hisa_sub(hisa_ctx* ctx, hisa_ct a, hisa_ct b, hisa_ct* out);
int hisa_add_plain(hisa_ctx* ctx, hisa_ct a, hisa_pt p, hisa_ct* out);
int hisa_sub_plain(hisa_ctx* ctx, hisa_ct a, hisa_pt p, hisa_ct* out);
/* scalar encoded at the ciphertext's scale: X = llround(x * scale) (A20) */
int hisa_add_scalar(hisa_ctx* ctx, hisa_ct a, double x, hisa_ct* out);
int hisa_sub_scalar(hisa_ctx* ctx, hisa_ct a, double x, hisa_ct* out);
/* = mul_norelin + relinearize */
int hisa_mul(hisa_ctx* ctx, hisa_ct a, hisa_ct b, hisa_ct* out);
int hisa_mul_plain(hisa_ctx* ctx, hisa_ct a, hisa_pt p, hisa_ct* out);
/* n independent mulPlains at one level in batched launches: outs[i] = a[i] (x) p[i] (fresh handles;
 * HISA_E_LEVEL_MISMATCH unless every pair shares one level) */
int hisa_mul_plain_batch(hisa_ctx* ctx, const hisa_ct* a, const hisa_pt* p, size_t n, hisa_ct* outs);
/* X = llround(x * pt_scale); pt_scale == 0 means (double) q_top of the ciphertext (A8) */
int hisa_mul_scalar(hisa_ctx* ctx, hisa_ct a, double x, double pt_scale, hisa_ct* out);

/* ---- Division profile (RNS reading A18 of P:584-587) --------------------------- */
/* d = q_top if q_top <= ub else 1 */
int hisa_max_scalar_div(hisa_ctx* ctx, hisa_ct ct, uint64_t ub, uint64_t* d);
/* d == q_top: rescale (drop top prime with rounding, scale /= q_top); d == 1: copy;
 * else HISA_E_INVALID_DIVISOR; at level 0: HISA_E_MODULUS_EXHAUSTED */
int hisa_div_scalar(hisa_ctx* ctx, hisa_ct ct, uint64_t d, hisa_ct* out);
int hisa_rescale(hisa_ctx* ctx, hisa_ct ct, hisa_ct* out);

/* ---- Relin profile ----------------------------------------------------------- */
int hisa_mul_norelin(hisa_ctx* ctx, hisa_ct a, hisa_ct b, hisa_ct* out);
/* in place: 3-poly -> 2-poly with the relinearisation key; 2-poly input is a no-op */
int hisa_relinearize(hisa_ctx* ctx, hisa_ct ct);

/* ---- Bootstrap profile ------------------------------------------------------- */
int hisa_bootstrap(hisa_ctx* ctx, hisa_ct ct);   /* always HISA_E_UNSUPPORTED_PROFILE */

/* ---- hot-path extensions ----------------------------------------------------------------- */
/* drop `drop` top limbs without division (A19), scale unchanged */
int hisa_mod_switch(hisa_ctx* ctx, hisa_ct ct, int drop, hisa_ct* out);
/* n rotations of one ciphertext sharing one ModUp (hoisting: "the rotations of the input
 * ciphertexts ... can be code motioned out"); outs[n] (fresh handles, k = 0 copies).
 * Results are bit-identical to n separate hisa_rot_left calls (A14: the automorphism commutes
 * with the exact centred ModUp / ModDown).  Device scratch: (l+1)(l+2) limbs for the shared
 * ModUp output plus ~(6l+8) limbs per amount in flight (chunks of 8 amounts). */
int hisa_rot_left_hoisted(hisa_ctx* ctx, hisa_ct ct, const int64_t* k, size_t n, hisa_ct* outs);
/* hoisted rotations of nct ciphertexts (one level) by the same n amounts: outs[i * n + r] =
 * rotLeft(in[i], k[r]).  ModUp batched over ciphertexts, each rotation key word streamed once per
 * group of up to 4 ciphertexts (K7), batched ModDown; bit-identical to hisa_rot_left.  The conv
 * (all input channels x filter taps) and pooling pattern. */
int hisa_rot_left_hoisted_batch(hisa_ctx* ctx, const hisa_ct* in, size_t nct, const int64_t* k, size_t n,
                                hisa_ct* outs);
/* the same rotation amount on n ciphertexts of one level, batched launches; outs[n] */
int hisa_rot_left_batch(hisa_ctx* ctx, const hisa_ct* in, size_t n, int64_t k, hisa_ct* outs);
/* batched forms (one level per batch; results bit-identical to the per-ciphertext calls):
 * outs[i] = a[i] * b[i] relinearised (hisa_mul), and outs[i] = rescale(in[i]) */
int hisa_mul_batch(hisa_ctx* ctx, const hisa_ct* a, const hisa_ct* b, size_t n, hisa_ct* outs);
int hisa_rescale_batch(hisa_ctx* ctx, const hisa_ct* in, size_t n, hisa_ct* outs);
/* rotate-and-sum step ("reduction ... in log rotations"; A27): outs[i] = in[i] +
 * rotLeft(in[i], k) for n ciphertexts of one level, batched under one key, the addition fused into
 * the final permutation kernel.  Bit-identical to hisa_add(in, hisa_rot_left(in, k)). */
int hisa_rot_add_batch(hisa_ctx* ctx, const hisa_ct* in, size_t n, int64_t k, hisa_ct* outs);
/* matmul accumulation: outs[j] = sum_c in[c] * pts[j*C + c] (mulPlain + add) for j < J,
 * one HBM-streaming kernel; all inputs one level / scale, all plaintexts that level and one scale.
 * Bit-identical to the mulPlain / add chain. */
int hisa_mul_plain_accumulate(hisa_ctx* ctx, const hisa_ct* in, size_t C, const hisa_pt* pts, size_t J,
                              hisa_ct* outs);
/* out[o] = sum_t W[o*T + t] * in[t] with X = llround(W * pt_scale) (pt_scale 0 => q_top):
 * the mulScalar + add accumulation of Alg. 1 for OC outputs; all inputs one level,
 * one scale; no rescale (caller divScalars once per output).  Engine: the tcgen05 int8
 * tensor cores (byte-split modular GEMM, T <= 4096, N a multiple of 128) unless the environment
 * sets HISA_CONV_TC=0 (CUDA-core kernel); both give the same words.  HISA_CONV_TC_SMEM=<bytes>
 * overrides the tensor-core kernel's shared-memory budget (inputs resident per pass; test knob,
 * same words for any value >= 36864).  Errors: HISA_E_PARAMS
 * (non-finite or |W pt_scale| >= 2^62 weight, T or OC 0, T too large for the CUDA-core kernel),
 * HISA_E_LEVEL_MISMATCH / HISA_E_SCALE_MISMATCH / HISA_E_NOT_RELINEARIZED (inputs), HISA_E_OOM. */
int hisa_conv_accumulate(hisa_ctx* ctx, const hisa_ct* in, size_t T, const double* W, size_t OC, double pt_scale,
                         hisa_ct* outs);
/* the same accumulation written into caller-owned device memory dev_out = uint64 [OC][2][l+1][N]
 * (contiguous; e.g. a torch tensor that a multi-GPU layer then reduce-scatters); every
 * word fully reduced in [0, q_i).  The partial sums carry scale in_scale * pt_scale. */
int hisa_conv_accumulate_dev(hisa_ctx* ctx, const hisa_ct* in, size_t T, const double* W, size_t OC,
                             double pt_scale, uint64_t* dev_out);

/* forward (inverse = 0) or inverse NTT of every limb of the ciphertext(s), in place: the words
 * are reinterpreted (coefficient <-> NTT domain, A5); limb i uses q_i.  Steps a1/a2 as ops. */
int hisa_ntt(hisa_ctx* ctx, hisa_ct ct, int inverse);
int hisa_ntt_batch(hisa_ctx* ctx, const hisa_ct* cts, size_t n, int inverse);

/* ---- inspection / import / export (canonical layout, see above) ---------------------------- */
int hisa_ct_info(hisa_ctx* ctx, hisa_ct ct, int* level, int* npolys, double* scale);
int hisa_pt_info(hisa_ctx* ctx, hisa_pt pt, int* level, double* scale);
int hisa_ct_export(hisa_ctx* ctx, hisa_ct ct, uint64_t* host, size_t words);
int hisa_ct_import(hisa_ctx* ctx, const uint64_t* host, int level, int npolys, double scale, hisa_ct* out);
int hisa_pt_export(hisa_ctx* ctx, hisa_pt pt, uint64_t* host, size_t words);
int hisa_pt_import(hisa_ctx* ctx, const uint64_t* host, int level, double scale, hisa_pt* out);
/* zero-copy device view (for NCCL via torch); valid until the handle is freed or overwritten */
int hisa_ct_device_view(hisa_ctx* ctx, hisa_ct ct, uint64_t** dev, size_t* words);
/* new ciphertext copied (device to device) from `dev` (words = npolys (level+1) N) */
int hisa_ct_adopt_device(hisa_ctx* ctx, const uint64_t* dev, int level, int npolys, double scale, hisa_ct* out);
/* a15 exchange fix-up: `dev` holds the int64 element-wise SUM over <= 8 ranks of fully reduced
 * ciphertext residue arrays [npolys][level+1][N] (an NCCL reduce-scatter / all-reduce output;
 * every sum < 8 q_i < 2^63, exact).  Creates a ciphertext with each word reduced back into
 * [0, q_i) by a device kernel.  `dev` is caller-owned and not retained. */
int hisa_ct_adopt_sum(hisa_ctx* ctx, const int64_t* dev, int level, int npolys, double scale, hisa_ct* out);
/* benchmark input (config 2): uniform residues from ChaCha20 tag BENCH, stream index
 * (b << 32 | poly << 16 | limb); not a valid encryption */
int hisa_ct_random(hisa_ctx* ctx, uint64_t b, int level, int npolys, hisa_ct* out);
/* uniform plaintext residues, stream index (b << 32 | 0xFFFF << 16 | limb) */
int hisa_pt_random(hisa_ctx* ctx, uint64_t b, int level, hisa_pt* out);

/* ---- diagnostics (not HISA instructions) -------------------------------------------------- */
/* enable != 0: record a CUDA event pair around every kernel launch on the context stream from now
 * on (and reset the launch counter); 0: stop.  Synchronises. */
int hisa_profile(hisa_ctx* ctx, int enable);
/* aggregate recorded launches per kernel class: names ('\n'-separated) / total ms / launch count;
 * synchronises and clears the records */
int hisa_profile_read(hisa_ctx* ctx, char* names, size_t names_len, double* ms, uint64_t* counts,
                      size_t max_entries, size_t* n_entries);
/* kernels launched since the last hisa_profile call */
int hisa_launch_count(hisa_ctx* ctx, uint64_t* n);
/* register-resident 64-bit Harvey butterflies on every SM (mod q_0): butterflies per second */
int hisa_microbench_butterfly(hisa_ctx* ctx, int iters, double* bfly_per_s);
/* the same with the exact FP64-pipe butterfly used for moduli < 2^50 (ntt_f64.cuh) */
int hisa_microbench_butterfly_f64(hisa_ctx* ctx, int iters, double* bfly_per_s);
/* the key multiply-accumulate of the key-switch inner product (K4: 64 x 64 -> three split 64-bit
   sums, 4 IMAD.WIDE.U32 per MAC) on all SMs, in MACs per second: the denominator for the key MACs */
int hisa_microbench_mac(hisa_ctx* ctx, int iters, double* mac_per_s);

const char* hisa_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* HISA_H */
