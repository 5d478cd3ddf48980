/*
 * ckks_oracle.c -- plain, slow, obviously-correct CPU RNS-CKKS (TEST INFRASTRUCTURE ONLY).
 *
 * This file is the parity oracle for the B200 HISA path.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  It shares no code, headers,
 * tables or constant generators with paper_1810_00845_b200/csrc (the product path).
 *
 * Citations: P:n = /root/reference/PAPER.md line n (CHET, arXiv 1810.00845);
 *            A<n> = reading n in DESIGN.md "Readings" (the paper is silent on RNS internals,
 *            P:764 and P:584-587 are its only RNS statements).
 *
 * Arithmetic: every modular product is (unsigned __int128)a*b % q.  No lazy reduction, no
 * Shoup/Barrett, no fusion.  NTT = twist by psi^t, textbook CLRS iterative radix-2 DFT with
 * omega = psi^2, then bit-reversed output order (A5).  Parallelism: OpenMP over independent
 * limbs only (does not change any arithmetic).
 *
 * Pins (tests/test_oracle_pins.py): direct O(N^2) evaluation of the NTT definition,
 * brute-force negacyclic products, Python big-integer definitions of rescale / key switching /
 * automorphism at N <= 64, RFC 8439 ChaCha20 via the `cryptography` library, closed-form
 * encodings (P-ENC-1, P-ENC-2), sampler moments, prime/root invariants.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <quadmath.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;
typedef __int128 i128;

#define ORC_MAXMOD 72

/* ------------------------------------------------------------------------------------------ */
/* scalar modular helpers                                                                       */
/* ------------------------------------------------------------------------------------------ */
static uint64_t mulm(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)(((u128)a * b) % q); }
static uint64_t addm(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)(((u128)a + b) % q); }
static uint64_t subm(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)(((u128)a + q - b) % q); }
static uint64_t powm(uint64_t b, uint64_t e, uint64_t q) {
    uint64_t r = 1 % q;
    b %= q;
    while (e) { if (e & 1) r = mulm(r, b, q); b = mulm(b, b, q); e >>= 1; }
    return r;
}
/* inverse by Fermat (q prime) */
static uint64_t invm(uint64_t a, uint64_t q) { return powm(a, q - 2, q); }
/* signed integer -> residue */
static uint64_t red_signed(int64_t x, uint64_t q) {
    i128 r = (i128)x % (i128)q;
    if (r < 0) r += q;
    return (uint64_t)r;
}
/* residue -> centered representative in (-q/2, q/2) (q odd) */
static int64_t center(uint64_t x, uint64_t q) { return x > (q - 1) / 2 ? (int64_t)x - (int64_t)q : (int64_t)x; }

/* deterministic Miller-Rabin for n < 2^64 */
static int is_prime_u64(uint64_t n) {
    static const uint64_t bases[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    if (n < 2) return 0;
    for (int i = 0; i < 12; i++) { if (n % bases[i] == 0) return n == bases[i]; }
    uint64_t d = n - 1; int s = 0;
    while ((d & 1) == 0) { d >>= 1; s++; }
    for (int i = 0; i < 12; i++) {
        uint64_t x = powm(bases[i], d, n);
        if (x == 1 || x == n - 1) continue;
        int comp = 1;
        for (int r = 1; r < s; r++) { x = mulm(x, x, n); if (x == n - 1) { comp = 0; break; } }
        if (comp) return 0;
    }
    return 1;
}

static uint64_t bitrev(uint64_t x, int bits) {
    uint64_t r = 0;
    for (int i = 0; i < bits; i++) { r = (r << 1) | (x & 1); x >>= 1; }
    return r;
}

/* ------------------------------------------------------------------------------------------ */
/* context                                                                                      */
/* ------------------------------------------------------------------------------------------ */
typedef struct orc_ctx {
    int logN;
    uint64_t N;
    int L;                      /* number of ciphertext primes q_0..q_{L-1} (A29) */
    uint64_t mod[ORC_MAXMOD];   /* mod[0..L-1] = q_i, mod[L] = special prime p (A3, A14) */
    uint64_t psi[ORC_MAXMOD];   /* minimal primitive 2N-th root (A4) */
    uint64_t *twist[ORC_MAXMOD];   /* psi^t, t < N */
    uint64_t *itwist[ORC_MAXMOD];  /* psi^-t, t < N */
    long double *cosl_tab;      /* cos(pi e / N), e < 2N  (encode/decode, A7) */
    __float128 *cosq_tab;       /* same in binary128, built on first near-tie (A7) */
    int nthreads;
} orc_ctx;

/*
 * A3: for each bit size b the candidate list is the primes q = k*2N+1 < 2^b in descending
 * order.  Special prime(s) take first, then q_0, then q_1..q_{L-1}; each takes the next unused
 * prime of its own bit size.
 */
typedef struct { int bits; uint64_t next_k; } prime_cursor;

static uint64_t next_prime(prime_cursor *cur, int ncur, int bits, uint64_t twoN) {
    int c = -1;
    for (int i = 0; i < ncur; i++) if (cur[i].bits == bits) c = i;
    for (;;) {
        uint64_t k = cur[c].next_k;
        if (k == 0) return 0;
        cur[c].next_k = k - 1;
        uint64_t q = k * twoN + 1;
        if (is_prime_u64(q)) return q;
    }
}

/* A4: psi = smallest element of order exactly 2N, found among psi0^odd */
static uint64_t min_primitive_root(uint64_t q, uint64_t N) {
    uint64_t g = 2;
    while (powm(g, (q - 1) / 2, q) != q - 1) g++;    /* quadratic non-residue */
    uint64_t psi0 = powm(g, (q - 1) / (2 * N), q);  /* order exactly 2N */
    uint64_t psi0sq = mulm(psi0, psi0, q);
    uint64_t best = psi0, cur = psi0;
    for (uint64_t k = 1; k < N; k++) { cur = mulm(cur, psi0sq, q); if (cur < best) best = cur; }
    return best;
}

void orc_destroy(orc_ctx *c) {
    if (!c) return;
    for (int i = 0; i <= c->L; i++) { free(c->twist[i]); free(c->itwist[i]); }
    free(c->cosl_tab);
    free(c->cosq_tab);
    free(c);
}

/* returns NULL on invalid parameters */
orc_ctx *orc_create(int logN, int L, const int *q_bits, int p_bits, int nthreads) {
    if (logN < 2 || logN > 17 || L < 1 || L + 1 > ORC_MAXMOD) return NULL;
    orc_ctx *c = (orc_ctx *)calloc(1, sizeof(orc_ctx));
    c->logN = logN; c->N = 1ull << logN; c->L = L;
    c->nthreads = nthreads > 0 ? nthreads : 1;
    uint64_t twoN = 2 * c->N;
    prime_cursor cur[ORC_MAXMOD]; int ncur = 0;
    int allbits[ORC_MAXMOD];
    allbits[0] = p_bits;
    for (int i = 0; i < L; i++) allbits[i + 1] = q_bits[i];
    for (int i = 0; i <= L; i++) {
        int b = allbits[i], seen = 0;
        if (b < 4 || b > 61) { free(c); return NULL; }
        for (int j = 0; j < ncur; j++) if (cur[j].bits == b) seen = 1;
        if (!seen) { cur[ncur].bits = b; cur[ncur].next_k = ((1ull << b) - 2) / twoN; ncur++; }
    }
    /* special prime first (A3) */
    c->mod[L] = next_prime(cur, ncur, p_bits, twoN);
    for (int i = 0; i < L; i++) c->mod[i] = next_prime(cur, ncur, q_bits[i], twoN);
    for (int i = 0; i <= L; i++) if (c->mod[i] == 0) { free(c); return NULL; }
    for (int i = 0; i <= L; i++) {
        uint64_t q = c->mod[i];
        c->psi[i] = min_primitive_root(q, c->N);
        c->twist[i] = (uint64_t *)malloc(c->N * 8);
        c->itwist[i] = (uint64_t *)malloc(c->N * 8);
        uint64_t pinv = invm(c->psi[i], q), a = 1, b = 1;
        for (uint64_t t = 0; t < c->N; t++) {
            c->twist[i][t] = a; c->itwist[i][t] = b;
            a = mulm(a, c->psi[i], q); b = mulm(b, pinv, q);
        }
    }
    c->cosl_tab = (long double *)malloc(sizeof(long double) * twoN);
    const long double pi = acosl(-1.0L);
    for (uint64_t e = 0; e < twoN; e++) c->cosl_tab[e] = cosl(pi * (long double)e / (long double)c->N);
    return c;
}

int orc_num_moduli(const orc_ctx *c) { return c->L + 1; }
void orc_moduli(const orc_ctx *c, uint64_t *out) { for (int i = 0; i <= c->L; i++) out[i] = c->mod[i]; }
void orc_psis(const orc_ctx *c, uint64_t *out) { for (int i = 0; i <= c->L; i++) out[i] = c->psi[i]; }
uint64_t orc_N(const orc_ctx *c) { return c->N; }
int orc_threads(const orc_ctx *c) { return c->nthreads; }

/* ------------------------------------------------------------------------------------------ */
/* NTT (A5): ahat[j] = sum_t a_t psi^((2 brv(j)+1) t)  ("NTT domain")                     */
/* ------------------------------------------------------------------------------------------ */
/* textbook CLRS ITERATIVE-FFT over Z_q: y_k = sum_t x_t w^(k t), natural order in/out */
static void dft_textbook(uint64_t *x, uint64_t N, int logN, uint64_t w, uint64_t q) {
    uint64_t *A = (uint64_t *)malloc(N * 8);
    for (uint64_t t = 0; t < N; t++) A[bitrev(t, logN)] = x[t];
    for (int s = 1; s <= logN; s++) {
        uint64_t m = 1ull << s;
        uint64_t wm = powm(w, N / m, q);
        for (uint64_t k = 0; k < N; k += m) {
            uint64_t ww = 1;
            for (uint64_t j = 0; j < m / 2; j++) {
                uint64_t t = mulm(ww, A[k + j + m / 2], q);
                uint64_t u = A[k + j];
                A[k + j] = addm(u, t, q);
                A[k + j + m / 2] = subm(u, t, q);
                ww = mulm(ww, wm, q);
            }
        }
    }
    memcpy(x, A, N * 8);
    free(A);
}

/* forward negacyclic NTT of one limb mod mod[midx], in place, output bit-reversed (A5) */
void orc_ntt(const orc_ctx *c, int midx, uint64_t *a) {
    uint64_t q = c->mod[midx], N = c->N;
    uint64_t *b = (uint64_t *)malloc(N * 8);
    for (uint64_t t = 0; t < N; t++) b[t] = mulm(a[t] % q, c->twist[midx][t], q);
    dft_textbook(b, N, c->logN, mulm(c->psi[midx], c->psi[midx], q), q);
    for (uint64_t j = 0; j < N; j++) a[j] = b[bitrev(j, c->logN)];
    free(b);
}

/* inverse: a_t = N^-1 psi^-t sum_k y_k w^-(k t) with y[brv(j)] = ahat[j] */
void orc_intt(const orc_ctx *c, int midx, uint64_t *a) {
    uint64_t q = c->mod[midx], N = c->N;
    uint64_t *y = (uint64_t *)malloc(N * 8);
    for (uint64_t j = 0; j < N; j++) y[bitrev(j, c->logN)] = a[j] % q;
    uint64_t w = mulm(c->psi[midx], c->psi[midx], q);
    dft_textbook(y, N, c->logN, invm(w, q), q);
    uint64_t ninv = invm(N % q, q);
    for (uint64_t t = 0; t < N; t++) a[t] = mulm(mulm(y[t], ninv, q), c->itwist[midx][t], q);
    free(y);
}

/* batched helpers: limb i of `a` (stride N) is mod mod[midx0 + i] */
void orc_ntt_limbs(const orc_ctx *c, uint64_t *a, int nlimbs, int midx0) {
#pragma omp parallel for num_threads(c->nthreads) schedule(dynamic)
    for (int i = 0; i < nlimbs; i++) orc_ntt(c, midx0 + i, a + (uint64_t)i * c->N);
}
void orc_intt_limbs(const orc_ctx *c, uint64_t *a, int nlimbs, int midx0) {
#pragma omp parallel for num_threads(c->nthreads) schedule(dynamic)
    for (int i = 0; i < nlimbs; i++) orc_intt(c, midx0 + i, a + (uint64_t)i * c->N);
}

/* ------------------------------------------------------------------------------------------ */
/* ChaCha20 (RFC 8439 block function) and fixed-position samplers (A9-A11)                     */
/* ------------------------------------------------------------------------------------------ */
static uint32_t rotl32(uint32_t x, int n) { return (x << n) | (x >> (32 - n)); }
#define QR(a, b, c, d) do { a += b; d ^= a; d = rotl32(d, 16); c += d; b ^= c; b = rotl32(b, 12); \
                            a += b; d ^= a; d = rotl32(d, 8);  c += d; b ^= c; b = rotl32(b, 7); } while (0)

void orc_chacha20_block(const uint32_t key[8], uint32_t counter, const uint32_t nonce[3], uint32_t out[16]) {
    uint32_t s[16] = {0x61707865u, 0x3320646eu, 0x79622d32u, 0x6b206574u,
                      key[0], key[1], key[2], key[3], key[4], key[5], key[6], key[7],
                      counter, nonce[0], nonce[1], nonce[2]};
    uint32_t x[16];
    memcpy(x, s, sizeof s);
    for (int i = 0; i < 10; i++) {
        QR(x[0], x[4], x[8], x[12]); QR(x[1], x[5], x[9], x[13]);
        QR(x[2], x[6], x[10], x[14]); QR(x[3], x[7], x[11], x[15]);
        QR(x[0], x[5], x[10], x[15]); QR(x[1], x[6], x[11], x[12]);
        QR(x[2], x[7], x[8], x[13]); QR(x[3], x[4], x[9], x[14]);
    }
    for (int i = 0; i < 16; i++) out[i] = x[i] + s[i];
}

/* 64-bit stream word n of stream (seed, tag, index): u32 words 2n (low) and 2n+1 (high);
 * key = seed LE in key words 0,1; nonce = (tag, index_lo, index_hi); block counter = n/8 (A11) */
void orc_stream_u64(uint64_t seed, uint32_t tag, uint64_t index, uint64_t first, uint64_t count, uint64_t *out) {
    uint32_t key[8] = {(uint32_t)seed, (uint32_t)(seed >> 32), 0, 0, 0, 0, 0, 0};
    uint32_t nonce[3] = {tag, (uint32_t)index, (uint32_t)(index >> 32)};
    uint32_t blk[16];
    uint64_t cur_block = UINT64_MAX;
    for (uint64_t i = 0; i < count; i++) {
        uint64_t n = first + i;
        if (n / 8 != cur_block) { cur_block = n / 8; orc_chacha20_block(key, (uint32_t)cur_block, nonce, blk); }
        int w = (int)(n % 8) * 2;
        out[i] = (uint64_t)blk[w] | ((uint64_t)blk[w + 1] << 32);
    }
}

/* uniform residue: coefficient t = (word(2t+1) * 2^64 + word(2t)) mod q */
void orc_sample_uniform(const orc_ctx *c, uint64_t seed, uint32_t tag, uint64_t index, uint64_t q, uint64_t *out) {
    uint64_t *w = (uint64_t *)malloc(2 * c->N * 8);
    orc_stream_u64(seed, tag, index, 0, 2 * c->N, w);
    for (uint64_t t = 0; t < c->N; t++) out[t] = (uint64_t)((((u128)w[2 * t + 1]) << 64 | w[2 * t]) % q);
    free(w);
}
/* ternary (A9): (word(t) mod 3) - 1 */
void orc_sample_ternary(const orc_ctx *c, uint64_t seed, uint32_t tag, uint64_t index, int64_t *out) {
    uint64_t *w = (uint64_t *)malloc(c->N * 8);
    orc_stream_u64(seed, tag, index, 0, c->N, w);
    for (uint64_t t = 0; t < c->N; t++) out[t] = (int64_t)(w[t] % 3) - 1;
    free(w);
}
/* centered binomial eta=21 (A10): popcnt(w & M) - popcnt((w>>21) & M), M = 2^21-1 */
void orc_sample_cbd(const orc_ctx *c, uint64_t seed, uint32_t tag, uint64_t index, int64_t *out) {
    uint64_t *w = (uint64_t *)malloc(c->N * 8);
    orc_stream_u64(seed, tag, index, 0, c->N, w);
    const uint64_t M = (1ull << 21) - 1;
    for (uint64_t t = 0; t < c->N; t++)
        out[t] = (int64_t)__builtin_popcountll(w[t] & M) - (int64_t)__builtin_popcountll((w[t] >> 21) & M);
    free(w);
}

enum { TAG_SK = 1, TAG_PK_A = 2, TAG_PK_E = 3, TAG_ENC_V = 4, TAG_ENC_E0 = 5, TAG_ENC_E1 = 6,
       TAG_KSK_A = 7, TAG_KSK_E = 8, TAG_BENCH = 9, TAG_ROT_K = 10 };

/* integer polynomial -> NTT form mod mod[midx] */
static void int_poly_to_ntt(const orc_ctx *c, const int64_t *x, int midx, uint64_t *out) {
    for (uint64_t t = 0; t < c->N; t++) out[t] = red_signed(x[t], c->mod[midx]);
    orc_ntt(c, midx, out);
}

/* ------------------------------------------------------------------------------------------ */
/* keys (A9-A16)                                               */
/* ------------------------------------------------------------------------------------------ */
/* s_int[N] ternary coefficients; s_ntt[(L+1)][N] NTT form on every modulus incl. p */
void orc_keygen_secret(const orc_ctx *c, uint64_t seed, int64_t *s_int, uint64_t *s_ntt) {
    orc_sample_ternary(c, seed, TAG_SK, 0, s_int);
#pragma omp parallel for num_threads(c->nthreads)
    for (int m = 0; m <= c->L; m++) int_poly_to_ntt(c, s_int, m, s_ntt + (uint64_t)m * c->N);
}

/* pk[2][L][N]: pk_b = -a*s + e, pk_a = a  (a sampled directly in the NTT domain) */
void orc_keygen_public(const orc_ctx *c, uint64_t seed, const uint64_t *s_ntt, uint64_t *pk) {
    uint64_t N = c->N; int L = c->L;
    int64_t *e = (int64_t *)malloc(N * 8);
    orc_sample_cbd(c, seed, TAG_PK_E, 0, e);
#pragma omp parallel for num_threads(c->nthreads)
    for (int m = 0; m < L; m++) {
        uint64_t q = c->mod[m];
        uint64_t *b = pk + (uint64_t)m * N, *a = pk + ((uint64_t)L + m) * N;
        uint64_t *en = (uint64_t *)malloc(N * 8);
        int_poly_to_ntt(c, e, m, en);
        orc_sample_uniform(c, seed, TAG_PK_A, (uint64_t)m, q, a);
        for (uint64_t j = 0; j < N; j++) b[j] = addm(subm(0, mulm(a[j], s_ntt[(uint64_t)m * N + j], q), q), en[j], q);
        free(en);
    }
    free(e);
}

/*
 * Key-switching key s' -> s (A14: hybrid, dnum = L, alpha = 1, one special prime p).
 * ksk layout [digit j < L][poly b,a][modulus r <= L][N].
 * b_{j,r} = -a_{j,r} s_r + e_{j,r} + [r == j] (p mod q_j) s'_r ;  a_{j,r} uniform.
 */
void orc_keygen_ksk(const orc_ctx *c, uint64_t seed, uint64_t keyid, const uint64_t *s_ntt,
                    const uint64_t *sp_ntt, uint64_t *ksk) {
    uint64_t N = c->N; int L = c->L, M = L + 1;
#pragma omp parallel for num_threads(c->nthreads) schedule(dynamic)
    for (int j = 0; j < L; j++) {
        int64_t *e = (int64_t *)malloc(N * 8);
        uint64_t *en = (uint64_t *)malloc(N * 8);
        orc_sample_cbd(c, seed, TAG_KSK_E, (keyid << 32) | ((uint64_t)j), e);
        for (int r = 0; r < M; r++) {
            uint64_t q = c->mod[r];
            uint64_t *b = ksk + (((uint64_t)j * 2 + 0) * M + r) * N;
            uint64_t *a = ksk + (((uint64_t)j * 2 + 1) * M + r) * N;
            orc_sample_uniform(c, seed, TAG_KSK_A, (keyid << 32) | ((uint64_t)j << 16) | (uint64_t)r, q, a);
            int_poly_to_ntt(c, e, r, en);
            uint64_t pmod = c->mod[L] % q;
            for (uint64_t t = 0; t < N; t++) {
                uint64_t v = addm(subm(0, mulm(a[t], s_ntt[(uint64_t)r * N + t], q), q), en[t], q);
                if (r == j) v = addm(v, mulm(pmod, sp_ntt[(uint64_t)r * N + t], q), q);
                b[t] = v;
            }
        }
        free(e); free(en);
    }
}

/* coefficient-domain automorphism X -> X^g (A15): a_t moves to g t mod 2N, negated if >= N */
void orc_automorphism_coeff_int(uint64_t N, uint64_t g, const int64_t *a, int64_t *out) {
    memset(out, 0, N * 8);
    for (uint64_t t = 0; t < N; t++) {
        uint64_t idx = (g * t) % (2 * N);
        if (idx < N) out[idx] += a[t]; else out[idx - N] -= a[t];
    }
}
static void automorphism_coeff_mod(uint64_t N, uint64_t g, const uint64_t *a, uint64_t *out, uint64_t q) {
    for (uint64_t t = 0; t < N; t++) {
        uint64_t idx = (g * t) % (2 * N);
        if (idx < N) out[idx] = a[t]; else out[idx - N] = subm(0, a[t], q);
    }
}

uint64_t orc_galois_elt(const orc_ctx *c, int64_t k) {
    uint64_t s = c->N / 2;
    int64_t kk = k % (int64_t)s; if (kk < 0) kk += (int64_t)s;
    return powm(5, (uint64_t)kk, 2 * c->N);
}

/* s' for the rotation key of amount k: NTT(psi_g(s)) on all moduli */
void orc_rot_target(const orc_ctx *c, const int64_t *s_int, int64_t k, uint64_t *sp_ntt) {
    uint64_t N = c->N, g = orc_galois_elt(c, k);
    int64_t *sg = (int64_t *)malloc(N * 8);
    orc_automorphism_coeff_int(N, g, s_int, sg);
#pragma omp parallel for num_threads(c->nthreads)
    for (int m = 0; m <= c->L; m++) int_poly_to_ntt(c, sg, m, sp_ntt + (uint64_t)m * N);
    free(sg);
}
/* s' for the relinearisation key: s^2 (A16) */
void orc_relin_target(const orc_ctx *c, const uint64_t *s_ntt, uint64_t *sp_ntt) {
    uint64_t N = c->N;
    for (int m = 0; m <= c->L; m++)
        for (uint64_t t = 0; t < N; t++)
            sp_ntt[(uint64_t)m * N + t] = mulm(s_ntt[(uint64_t)m * N + t], s_ntt[(uint64_t)m * N + t], c->mod[m]);
}

/* ------------------------------------------------------------------------------------------ */
/* encrypt / decrypt (A12, A13)                                                                 */
/* ------------------------------------------------------------------------------------------ */
/* pt[(l+1)][N] NTT form; ct[2][(l+1)][N] */
void orc_encrypt(const orc_ctx *c, uint64_t seed, uint64_t counter, const uint64_t *pk, const uint64_t *pt,
                 int level, uint64_t *ct) {
    uint64_t N = c->N; int L = c->L, l1 = level + 1;
    int64_t *v = (int64_t *)malloc(N * 8), *e0 = (int64_t *)malloc(N * 8), *e1 = (int64_t *)malloc(N * 8);
    orc_sample_ternary(c, seed, TAG_ENC_V, counter, v);
    orc_sample_cbd(c, seed, TAG_ENC_E0, counter, e0);
    orc_sample_cbd(c, seed, TAG_ENC_E1, counter, e1);
#pragma omp parallel for num_threads(c->nthreads)
    for (int i = 0; i < l1; i++) {
        uint64_t q = c->mod[i];
        uint64_t *vn = (uint64_t *)malloc(N * 8), *e0n = (uint64_t *)malloc(N * 8), *e1n = (uint64_t *)malloc(N * 8);
        int_poly_to_ntt(c, v, i, vn); int_poly_to_ntt(c, e0, i, e0n); int_poly_to_ntt(c, e1, i, e1n);
        const uint64_t *pb = pk + (uint64_t)i * N, *pa = pk + ((uint64_t)L + i) * N;
        uint64_t *c0 = ct + (uint64_t)i * N, *c1 = ct + ((uint64_t)l1 + i) * N;
        for (uint64_t t = 0; t < N; t++) {
            c0[t] = addm(addm(mulm(vn[t], pb[t], q), e0n[t], q), pt[(uint64_t)i * N + t], q);
            c1[t] = addm(mulm(vn[t], pa[t], q), e1n[t], q);
        }
        free(vn); free(e0n); free(e1n);
    }
    free(v); free(e0); free(e1);
}

/* m = c0 + c1 s (+ c2 s^2); ct[npolys][(l+1)][N] -> pt[(l+1)][N] */
void orc_decrypt(const orc_ctx *c, const uint64_t *s_ntt, const uint64_t *ct, int npolys, int level, uint64_t *pt) {
    uint64_t N = c->N; int l1 = level + 1;
    for (int i = 0; i < l1; i++) {
        uint64_t q = c->mod[i];
        for (uint64_t t = 0; t < N; t++) {
            uint64_t s = s_ntt[(uint64_t)i * N + t];
            uint64_t m = ct[(uint64_t)i * N + t];
            m = addm(m, mulm(ct[((uint64_t)l1 + i) * N + t], s, q), q);
            if (npolys == 3) m = addm(m, mulm(ct[(2 * (uint64_t)l1 + i) * N + t], mulm(s, s, q), q), q);
            pt[(uint64_t)i * N + t] = m;
        }
    }
}

/* ------------------------------------------------------------------------------------------ */
/* encode / decode (A2, A7, A13)                                                     */
/* ------------------------------------------------------------------------------------------ */
/* v_t = (Delta/N) sum_{j<n} 2 z_j cos(pi (5^j t mod 2N) / N)   (real slots, zero-filled)     */
static long double enc_value_ld(const orc_ctx *c, const double *z, uint64_t n, double scale, uint64_t t,
                                const uint64_t *pow5) {
    uint64_t twoN = 2 * c->N;
    long double acc = 0.0L;
    for (uint64_t j = 0; j < n; j++) {
        if (z[j] == 0.0) continue;   /* a zero slot adds an exact 0 (sparse weight plaintexts) */
        uint64_t e = (uint64_t)(((u128)pow5[j] * t) % twoN);
        acc += 2.0L * (long double)z[j] * c->cosl_tab[e];
    }
    return acc * (long double)scale / (long double)c->N;
}
static __float128 enc_value_q(const orc_ctx *c, const double *z, uint64_t n, double scale, uint64_t t,
                              const uint64_t *pow5) {
    uint64_t twoN = 2 * c->N;
    __float128 acc = 0;
    for (uint64_t j = 0; j < n; j++) {
        if (z[j] == 0.0) continue;
        uint64_t e = (uint64_t)(((u128)pow5[j] * t) % twoN);
        acc += 2 * (__float128)z[j] * c->cosq_tab[e];
    }
    return acc * (__float128)scale / (__float128)c->N;
}

/*
 * Exact-rounded encoding coefficients (A7): m_t = round-half-away(v_t).  Long-double direct
 * sum (absolute error << 2^-12 for |v| < 2^62); coefficients whose fractional part is within
 * 2^-12 of 1/2 are recomputed by direct summation in __float128 (error ~2^-60).
 * Returns 0, or -1 if some |m_t| >= 2^62.
 */
#define ORC_TIE_WINDOW 0x1p-12L
static void ensure_cosq(orc_ctx *c) {
    if (c->cosq_tab) return;
    uint64_t twoN = 2 * c->N;
    __float128 *tab = (__float128 *)malloc(sizeof(__float128) * twoN);
    for (uint64_t e = 0; e < twoN; e++) tab[e] = cosq(M_PIq * (__float128)e / (__float128)c->N);
    c->cosq_tab = tab;
}
int orc_encode_coeffs(const orc_ctx *c, const double *z, uint64_t n, double scale, int64_t *m) {
    uint64_t N = c->N, twoN = 2 * N;
    uint64_t *pow5 = (uint64_t *)malloc((n ? n : 1) * 8);
    uint64_t p = 1;
    for (uint64_t j = 0; j < n; j++) { pow5[j] = p; p = (p * 5) % twoN; }
    int bad = 0;
    ensure_cosq(c);
#pragma omp parallel for num_threads(c->nthreads) reduction(| : bad)
    for (uint64_t t = 0; t < N; t++) {
        long double v = enc_value_ld(c, z, n, scale, t, pow5);
        long double av = fabsl(v);
        long double fr = av - floorl(av);
        long double r;
        if (fabsl(fr - 0.5L) < ORC_TIE_WINDOW) {
            __float128 vq = enc_value_q(c, z, n, scale, t, pow5);
            __float128 aq = fabsq(vq);
            __float128 rq = floorq(aq + 0.5Q);
            r = (long double)rq;
            if (vq < 0) r = -r;
        } else {
            r = floorl(av + 0.5L);
            if (v < 0) r = -r;
        }
        if (fabsl(r) >= 0x1p62L) bad = 1;
        else m[t] = (int64_t)r;
    }
    free(pow5);
    return bad ? -1 : 0;
}

/* pt[(level+1)][N] NTT form */
int orc_encode(const orc_ctx *c, const double *z, uint64_t n, double scale, int level, uint64_t *pt) {
    int64_t *m = (int64_t *)malloc(c->N * 8);
    int rc = orc_encode_coeffs(c, z, n, scale, m);
    if (rc == 0) {
#pragma omp parallel for num_threads(c->nthreads)
        for (int i = 0; i <= level; i++) int_poly_to_ntt(c, m, i, pt + (uint64_t)i * c->N);
    }
    free(m);
    return rc;
}

/* z_j = (1/scale) sum_t m_t cos(pi (5^j t mod 2N)/N), m = centered INTT of limb 0 (A13) */
void orc_decode(const orc_ctx *c, const uint64_t *pt_limb0, double scale, uint64_t n, double *z) {
    uint64_t N = c->N, twoN = 2 * N;
    uint64_t *a = (uint64_t *)malloc(N * 8);
    memcpy(a, pt_limb0, N * 8);
    orc_intt(c, 0, a);
    uint64_t *pow5 = (uint64_t *)malloc((n ? n : 1) * 8);
    uint64_t p = 1;
    for (uint64_t j = 0; j < n; j++) { pow5[j] = p; p = (p * 5) % twoN; }
#pragma omp parallel for num_threads(c->nthreads)
    for (uint64_t j = 0; j < n; j++) {
        long double acc = 0.0L;
        for (uint64_t t = 0; t < N; t++) {
            uint64_t e = (uint64_t)(((u128)pow5[j] * t) % twoN);
            acc += (long double)center(a[t], c->mod[0]) * c->cosl_tab[e];
        }
        z[j] = (double)(acc / (long double)scale);
    }
    free(pow5); free(a);
}

/* ------------------------------------------------------------------------------------------ */
/* elementwise (A8, A17, A20).  x[np][l+1][N] layout, limb i mod q_i.                */
/* ------------------------------------------------------------------------------------------ */
void orc_add(const orc_ctx *c, const uint64_t *a, const uint64_t *b, int npolys, int level, uint64_t *out) {
    uint64_t N = c->N; int l1 = level + 1;
    for (int p = 0; p < npolys; p++)
        for (int i = 0; i < l1; i++)
            for (uint64_t t = 0; t < N; t++) {
                uint64_t o = ((uint64_t)p * l1 + i) * N + t;
                out[o] = addm(a[o], b[o], c->mod[i]);
            }
}
void orc_sub(const orc_ctx *c, const uint64_t *a, const uint64_t *b, int npolys, int level, uint64_t *out) {
    uint64_t N = c->N; int l1 = level + 1;
    for (int p = 0; p < npolys; p++)
        for (int i = 0; i < l1; i++)
            for (uint64_t t = 0; t < N; t++) {
                uint64_t o = ((uint64_t)p * l1 + i) * N + t;
                out[o] = subm(a[o], b[o], c->mod[i]);
            }
}
/* out = ct (+/-) pt on poly 0 only; sign = +1 / -1 */
void orc_add_plain(const orc_ctx *c, const uint64_t *ct, const uint64_t *pt, int npolys, int level, int sign, uint64_t *out) {
    uint64_t N = c->N; int l1 = level + 1;
    memcpy(out, ct, (uint64_t)npolys * l1 * N * 8);
    for (int i = 0; i < l1; i++)
        for (uint64_t t = 0; t < N; t++) {
            uint64_t o = (uint64_t)i * N + t;
            out[o] = sign > 0 ? addm(ct[o], pt[o], c->mod[i]) : subm(ct[o], pt[o], c->mod[i]);
        }
}
/* multiply every poly by pt (mulPlain) */
void orc_mul_plain(const orc_ctx *c, const uint64_t *ct, const uint64_t *pt, int npolys, int level, uint64_t *out) {
    uint64_t N = c->N; int l1 = level + 1;
    for (int p = 0; p < npolys; p++)
        for (int i = 0; i < l1; i++)
            for (uint64_t t = 0; t < N; t++) {
                uint64_t o = ((uint64_t)p * l1 + i) * N + t;
                out[o] = mulm(ct[o], pt[(uint64_t)i * N + t], c->mod[i]);
            }
}
/* integer scalar X (already rounded, A20): mulScalar multiplies all polys; addScalar adds to poly 0 */
void orc_mul_scalar_int(const orc_ctx *c, const uint64_t *ct, int64_t X, int npolys, int level, uint64_t *out) {
    uint64_t N = c->N; int l1 = level + 1;
    for (int p = 0; p < npolys; p++)
        for (int i = 0; i < l1; i++) {
            uint64_t x = red_signed(X, c->mod[i]);
            for (uint64_t t = 0; t < N; t++) {
                uint64_t o = ((uint64_t)p * l1 + i) * N + t;
                out[o] = mulm(ct[o], x, c->mod[i]);
            }
        }
}
void orc_add_scalar_int(const orc_ctx *c, const uint64_t *ct, int64_t X, int npolys, int level, uint64_t *out) {
    uint64_t N = c->N; int l1 = level + 1;
    memcpy(out, ct, (uint64_t)npolys * l1 * N * 8);
    for (int i = 0; i < l1; i++) {
        uint64_t x = red_signed(X, c->mod[i]);
        for (uint64_t t = 0; t < N; t++) out[(uint64_t)i * N + t] = addm(ct[(uint64_t)i * N + t], x, c->mod[i]);
    }
}
/* mulNoRelin (A17): (a0 b0, a0 b1 + a1 b0, a1 b1) */
void orc_tensor(const orc_ctx *c, const uint64_t *a, const uint64_t *b, int level, uint64_t *out) {
    uint64_t N = c->N; int l1 = level + 1;
    for (int i = 0; i < l1; i++) {
        uint64_t q = c->mod[i];
        for (uint64_t t = 0; t < N; t++) {
            uint64_t o0 = (uint64_t)i * N + t, o1 = ((uint64_t)l1 + i) * N + t;
            uint64_t a0 = a[o0], a1 = a[o1], b0 = b[o0], b1 = b[o1];
            out[o0] = mulm(a0, b0, q);
            out[o1] = addm(mulm(a0, b1, q), mulm(a1, b0, q), q);
            out[(2 * (uint64_t)l1 + i) * N + t] = mulm(a1, b1, q);
        }
    }
}

/* ------------------------------------------------------------------------------------------ */
/* key switching (A14), relinearize (A16), rotate (A15)                   */
/* ------------------------------------------------------------------------------------------ */
/*
 * d[(l+1)][N] NTT form at level l; ksk full layout [L][2][L+1][N]; out[2][(l+1)][N].
 * 1. x_j = centered(INTT_{q_j}(d_j))                        (ModUp, exact for alpha = 1)
 * 2. D_{j,r} = NTT_r(x_j mod r) for r in {q_0..q_l, p}      (D_{j,q_j} = d_j)
 * 3. acc_r = sum_j D_{j,r} (.) ksk_{j,r}                     (inner product)
 * 4. out_i = (acc_i - NTT_i(centered(INTT_p(acc_p)) mod q_i)) * p^-1 mod q_i   (ModDown)
 */
void orc_keyswitch(const orc_ctx *c, const uint64_t *d, int level, const uint64_t *ksk, uint64_t *out) {
    uint64_t N = c->N; int L = c->L, M = L + 1, l1 = level + 1;
    int64_t *x = (int64_t *)malloc((uint64_t)l1 * N * 8);
#pragma omp parallel for num_threads(c->nthreads)
    for (int j = 0; j < l1; j++) {
        uint64_t *tmp = (uint64_t *)malloc(N * 8);
        memcpy(tmp, d + (uint64_t)j * N, N * 8);
        orc_intt(c, j, tmp);
        for (uint64_t t = 0; t < N; t++) x[(uint64_t)j * N + t] = center(tmp[t], c->mod[j]);
        free(tmp);
    }
    /* output primes: q_0..q_l then p (index l1 in acc) */
    uint64_t *acc = (uint64_t *)calloc((uint64_t)2 * (l1 + 1) * N, 8);
#pragma omp parallel for num_threads(c->nthreads) schedule(dynamic)
    for (int ri = 0; ri <= l1; ri++) {
        int r = ri < l1 ? ri : L;   /* modulus index */
        uint64_t q = c->mod[r];
        uint64_t *D = (uint64_t *)malloc(N * 8);
        uint64_t *a0 = acc + ((uint64_t)0 * (l1 + 1) + ri) * N, *a1 = acc + ((uint64_t)1 * (l1 + 1) + ri) * N;
        for (int j = 0; j < l1; j++) {
            if (r == j) memcpy(D, d + (uint64_t)j * N, N * 8);
            else {
                for (uint64_t t = 0; t < N; t++) D[t] = red_signed(x[(uint64_t)j * N + t], q);
                orc_ntt(c, r, D);
            }
            const uint64_t *kb = ksk + (((uint64_t)j * 2 + 0) * M + r) * N;
            const uint64_t *ka = ksk + (((uint64_t)j * 2 + 1) * M + r) * N;
            for (uint64_t t = 0; t < N; t++) {
                a0[t] = addm(a0[t], mulm(D[t], kb[t], q), q);
                a1[t] = addm(a1[t], mulm(D[t], ka[t], q), q);
            }
        }
        free(D);
    }
    /* ModDown */
    uint64_t p = c->mod[L];
    for (int k = 0; k < 2; k++) {
        uint64_t *ap = (uint64_t *)malloc(N * 8);
        memcpy(ap, acc + ((uint64_t)k * (l1 + 1) + l1) * N, N * 8);
        orc_intt(c, L, ap);
        int64_t *y = (int64_t *)malloc(N * 8);
        for (uint64_t t = 0; t < N; t++) y[t] = center(ap[t], p);
#pragma omp parallel for num_threads(c->nthreads)
        for (int i = 0; i < l1; i++) {
            uint64_t q = c->mod[i];
            uint64_t *tmp = (uint64_t *)malloc(N * 8);
            for (uint64_t t = 0; t < N; t++) tmp[t] = red_signed(y[t], q);
            orc_ntt(c, i, tmp);
            uint64_t pinv = invm(p % q, q);
            const uint64_t *ai = acc + ((uint64_t)k * (l1 + 1) + i) * N;
            uint64_t *o = out + ((uint64_t)k * l1 + i) * N;
            for (uint64_t t = 0; t < N; t++) o[t] = mulm(subm(ai[t], tmp[t], q), pinv, q);
            free(tmp);
        }
        free(ap); free(y);
    }
    free(acc); free(x);
}

/* relinearize: ct3[3][(l+1)][N] -> (d0, d1) + KS_{s^2}(d2) */
void orc_relinearize(const orc_ctx *c, const uint64_t *ct3, int level, const uint64_t *rlk, uint64_t *out) {
    uint64_t N = c->N; int l1 = level + 1;
    uint64_t *ks = (uint64_t *)malloc((uint64_t)2 * l1 * N * 8);
    orc_keyswitch(c, ct3 + (uint64_t)2 * l1 * N, level, rlk, ks);
    orc_add(c, ct3, ks, 2, level, out);
    free(ks);
}

/* NTT-form limb automorphism done the plain way: INTT -> coefficient map -> NTT */
void orc_automorphism_ntt_limb(const orc_ctx *c, int midx, uint64_t g, const uint64_t *in, uint64_t *out) {
    uint64_t N = c->N;
    uint64_t *a = (uint64_t *)malloc(N * 8);
    memcpy(a, in, N * 8);
    orc_intt(c, midx, a);
    automorphism_coeff_mod(N, g, a, out, c->mod[midx]);
    orc_ntt(c, midx, out);
    free(a);
}

/* rotLeft(c, k) with the rotation key for k (A15): c' = psi_g(c); (c'_0 + KS(c'_1)_0, KS(c'_1)_1) */
void orc_rotate(const orc_ctx *c, const uint64_t *ct, int level, int64_t k, const uint64_t *rk, uint64_t *out) {
    uint64_t N = c->N; int l1 = level + 1;
    uint64_t g = orc_galois_elt(c, k);
    uint64_t *cp = (uint64_t *)malloc((uint64_t)2 * l1 * N * 8);
#pragma omp parallel for num_threads(c->nthreads)
    for (int pi = 0; pi < 2 * l1; pi++) {
        int i = pi % l1;
        orc_automorphism_ntt_limb(c, i, g, ct + (uint64_t)pi * N, cp + (uint64_t)pi * N);
    }
    uint64_t *ks = (uint64_t *)malloc((uint64_t)2 * l1 * N * 8);
    orc_keyswitch(c, cp + (uint64_t)l1 * N, level, rk, ks);
    for (int i = 0; i < l1; i++)
        for (uint64_t t = 0; t < N; t++) {
            out[(uint64_t)i * N + t] = addm(cp[(uint64_t)i * N + t], ks[(uint64_t)i * N + t], c->mod[i]);
            out[((uint64_t)l1 + i) * N + t] = ks[((uint64_t)l1 + i) * N + t];
        }
    free(cp); free(ks);
}

/* ------------------------------------------------------------------------------------------ */
/* rescale / divScalar (A18) and modulus switch (A19)                     */
/* ------------------------------------------------------------------------------------------ */
/* in[np][(l+1)][N] -> out[np][l][N]: out_i = (u_i - NTT_i(centered(INTT_{q_l}(u_l)))) q_l^-1 */
void orc_rescale(const orc_ctx *c, const uint64_t *in, int npolys, int level, uint64_t *out) {
    uint64_t N = c->N; int l1 = level + 1, l = level;
    uint64_t ql = c->mod[l];
    for (int k = 0; k < npolys; k++) {
        uint64_t *top = (uint64_t *)malloc(N * 8);
        memcpy(top, in + ((uint64_t)k * l1 + l) * N, N * 8);
        orc_intt(c, l, top);
        int64_t *y = (int64_t *)malloc(N * 8);
        for (uint64_t t = 0; t < N; t++) y[t] = center(top[t], ql);
#pragma omp parallel for num_threads(c->nthreads)
        for (int i = 0; i < l; i++) {
            uint64_t q = c->mod[i];
            uint64_t *tmp = (uint64_t *)malloc(N * 8);
            for (uint64_t t = 0; t < N; t++) tmp[t] = red_signed(y[t], q);
            orc_ntt(c, i, tmp);
            uint64_t qinv = invm(ql % q, q);
            const uint64_t *u = in + ((uint64_t)k * l1 + i) * N;
            uint64_t *o = out + ((uint64_t)k * l + i) * N;
            for (uint64_t t = 0; t < N; t++) o[t] = mulm(subm(u[t], tmp[t], q), qinv, q);
            free(tmp);
        }
        free(top); free(y);
    }
}
/* drop limbs above new_level, no division */
void orc_mod_switch(const orc_ctx *c, const uint64_t *in, int npolys, int level, int new_level, uint64_t *out) {
    uint64_t N = c->N; int l1 = level + 1, n1 = new_level + 1;
    for (int k = 0; k < npolys; k++) memcpy(out + (uint64_t)k * n1 * N, in + (uint64_t)k * l1 * N, (uint64_t)n1 * N * 8);
}
