// hisa.cu -- host layer of libhisa: the C-ABI of include/hisa.h.
//
// Parameters / primes / roots / tables (A3-A6), the handle table (use-after-free detection,
// S:32-36), a first-fit arena on caller-provided device memory (PyTorch owns device memory),
// synchronous host checks (levels, scales, keys: A8, A15, A17, A18), and the orchestration of
// the sm_100a kernels for every HISA instruction.  Encode/decode are host boundary steps (A7, A13).
// Nothing here computes ciphertext arithmetic on the CPU: every step of the path is a kernel.
#include <cuda_runtime.h>
#include <quadmath.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <complex>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>
#include <thread>
#include <atomic>

#include "../../include/hisa.h"
#include "launch.h"
#include "ntt_f64.cuh"

using namespace hisa;
typedef unsigned __int128 u128;

// ============================================================================================
// errors
// ============================================================================================
static thread_local std::string g_err;
static int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
static int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}
extern "C" const char* hisa_last_error(void) { return g_err.c_str(); }

// ============================================================================================
// host number theory (independent of oracle/): deterministic 7-base Miller-Rabin for 64 bits
// ============================================================================================
static uint64_t h_mul(uint64_t a, uint64_t b, uint64_t m) { return (uint64_t)((u128)a * b % m); }
static uint64_t h_pow(uint64_t b, uint64_t e, uint64_t m) {
    uint64_t r = 1;
    b %= m;
    for (; e; e >>= 1, b = h_mul(b, b, m))
        if (e & 1) r = h_mul(r, b, m);
    return r;
}
static uint64_t h_inv(uint64_t a, uint64_t m) { return h_pow(a % m, m - 2, m); }
static bool h_prime(uint64_t n) {
    if (n < 2 || n % 2 == 0) return n == 2;
    uint64_t d = n - 1;
    int s = 0;
    while (!(d & 1)) { d >>= 1; s++; }
    static const uint64_t W[] = {2, 325, 9375, 28178, 450775, 9780504, 1795265022};
    for (uint64_t a : W) {
        a %= n;
        if (a == 0) continue;
        uint64_t x = h_pow(a, d, n);
        if (x == 1 || x == n - 1) continue;
        bool comp = true;
        for (int i = 1; i < s && comp; i++) {
            x = h_mul(x, x, n);
            if (x == n - 1) comp = false;
        }
        if (comp) return false;
    }
    return true;
}
static uint32_t h_brv(uint32_t x, int bits) {
    uint32_t r = 0;
    for (int i = 0; i < bits; i++) r |= ((x >> i) & 1u) << (bits - 1 - i);
    return r;
}
static uint64_t shoup(uint64_t w, uint64_t q) { return (uint64_t)(((u128)w << 64) / q); }
static Mod make_mod(uint64_t q) {
    u128 ratio = (~(u128)0) / q;   // floor((2^128 - 1)/q) == floor(2^128/q) for odd q
    Mod m;
    m.q = q;
    m.r0 = (uint64_t)ratio;
    m.r1 = (uint64_t)(ratio >> 64);
    return m;
}
// A4: the minimal element of multiplicative order exactly 2N
static uint64_t h_min_root(uint64_t q, uint64_t N) {
    uint64_t x = 0;
    for (uint64_t g = 3;; g++) {
        x = h_pow(g, (q - 1) / (2 * N), q);
        if (h_pow(x, N, q) == q - 1) break;
    }
    const uint64_t x2 = h_mul(x, x, q);
    uint64_t best = x, cur = x;
    for (uint64_t i = 1; i < N; i++) {
        cur = h_mul(cur, x2, q);
        if (cur < best) best = cur;
    }
    return best;
}

// ============================================================================================
// device memory: first-fit arena on a caller-owned buffer, else cudaMallocAsync
// ============================================================================================
struct Arena {
    char* base = nullptr;
    size_t size = 0;
    std::map<size_t, size_t> free_;   // offset -> bytes
    std::map<size_t, size_t> used_;
    size_t in_use = 0, peak = 0;
    void attach(void* p, size_t n) {
        base = (char*)p;
        size = n & ~(size_t)255;
        free_.clear();
        used_.clear();
        free_[0] = size;
    }
    void* alloc(size_t n) {
        n = (n + 255) & ~(size_t)255;
        if (n == 0) n = 256;
        for (auto it = free_.begin(); it != free_.end(); ++it) {
            if (it->second >= n) {
                size_t off = it->first, rem = it->second - n;
                free_.erase(it);
                if (rem) free_[off + n] = rem;
                used_[off] = n;
                in_use += n;
                if (in_use > peak) peak = in_use;
                return base + off;
            }
        }
        return nullptr;
    }
    void release(void* p) {
        size_t off = (char*)p - base;
        auto u = used_.find(off);
        if (u == used_.end()) return;
        size_t n = u->second;
        used_.erase(u);
        in_use -= n;
        auto nx = free_.lower_bound(off);
        if (nx != free_.end() && off + n == nx->first) {
            n += nx->second;
            free_.erase(nx);
        }
        auto pv = free_.lower_bound(off);
        if (pv != free_.begin()) {
            --pv;
            if (pv->first + pv->second == off) {
                pv->second += n;
                return;
            }
        }
        free_[off] = n;
    }
};

// ============================================================================================
// context
// ============================================================================================
enum ObjKind { OBJ_CT = 1, OBJ_PT = 2 };
struct Obj {
    int kind = 0;
    uint64_t* ptr = nullptr;
    int level = 0;
    int npolys = 0;
    double scale = 0;
    uint32_t gen = 0;
    bool live = false;
};

struct hisa_ctx {
    int log_n = 0;
    uint64_t N = 0;
    int L = 0;                        // number of q primes
    std::vector<uint64_t> mod;        // q_0..q_{L-1}, p
    uint64_t seed = 0;
    int device = 0;
    cudaStream_t stream = 0;
    // side stream for work that runs beside the main stream's (K4's integer-engine rows next to
    // its FP64 rows); fork/join through events, created on first use
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cudaEvent_t ev_k7[2] = {nullptr, nullptr}, ev_md[2] = {nullptr, nullptr};   // hoisted pipeline
    bool poisoned = false;
    Arena arena;
    bool has_arena = false;
    size_t pool_in_use = 0, pool_peak = 0;
    std::map<void*, size_t> pool_sizes;
    // device tables
    Mod* d_mods = nullptr;
    ulonglong2* d_fwd = nullptr;
    ulonglong2* d_inv = nullptr;
    ulonglong2* d_ninv = nullptr;
    ulonglong2* d_pinv = nullptr;     // p^-1 mod q_i (ModDown)
    ulonglong2* d_qlinv = nullptr;    // [l][L+1]: q_l^-1 mod q_i (rescale)
    double* d_fwd_d = nullptr;        // FP64-engine twiddles (moduli < 2^50, ntt_f64.cuh)
    double* d_inv_d = nullptr;
    double2* d_modd = nullptr;
    double* d_ninv_d = nullptr;
    double f64_max_q = 0x1p50;        // FP64 engine for q < 2^50 (HISA_F64=0 disables; diagnostics)
    std::vector<void*> table_allocs;
    // keys
    bool have_sk = false;
    int64_t* d_s_int = nullptr;
    uint64_t* d_sk = nullptr;         // [(L+1)][N]
    uint64_t* d_pk = nullptr;         // [2][L][N]
    // key-switching keys, each truncated to the highest level it serves (SURVEY 7 hard part 3):
    // kL = q primes covered (max level + 1), layout [kL digits][b, a][q_0..q_{kL-1}, p][N]
    struct KeyRec { uint64_t* p = nullptr; int kL = 0; };
    uint64_t* d_rlk = nullptr;        // [L][2][L+1][N] (relinearisation: always full)
    std::map<uint64_t, KeyRec> rot_keys;
    uint64_t enc_counter = 0;
    std::vector<__float128> enc_cosq;   // binary128 cos(pi e / N), e < 2N (near-tie recomputation, A7)
    uint32_t* d_enc_pos = nullptr;      // GPU encode: bit-reversed positions of the 2 x N/2 slot images
    cdd* d_enc_root = nullptr;          // e^{2 pi i k / N}, k < N/2, double-double from binary128
    cdd* d_enc_twist = nullptr;         // e^{i pi t / N}, t < N
    // profiling: CUDA events around every launch on the context stream (hisa_profile)
    bool prof_on = false;
    struct ProfRec { const char* name; cudaEvent_t a, b; };
    std::vector<ProfRec> prof;
    std::vector<cudaEvent_t> ev_pool;
    uint64_t launches = 0;
    // handles
    std::vector<Obj> objs;
    std::vector<uint32_t> free_slots;

    Tables tables(const ulonglong2* comb = nullptr) const {
        Tables t;
        t.fwd = d_fwd;
        t.inv = d_inv;
        t.mods = d_mods;
        t.ninv = d_ninv;
        t.comb = comb;
        t.fwd_d = d_fwd_d;
        t.inv_d = d_inv_d;
        t.modd = d_modd;
        t.ninv_d = d_ninv_d;
        t.f64_max_q = f64_max_q;
        t.fp_mods = 0;
        for (size_t i = 0; i < mod.size() && i < 64; i++)
            if ((double)mod[i] < f64_max_q) t.fp_mods |= 1ull << i;
        t.log_n = log_n;
        return t;
    }
};

static size_t key_words(const hisa_ctx* c, int kL = -1) {
    if (kL < 0) kL = c->L;
    return (size_t)kL * 2 * (kL + 1) * c->N;
}

static void* dalloc(hisa_ctx* c, size_t bytes) {
    if (c->has_arena) return c->arena.alloc(bytes);
    void* p = nullptr;
    if (cudaMallocAsync(&p, bytes ? bytes : 256, c->stream) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    c->pool_sizes[p] = bytes;
    c->pool_in_use += bytes;
    if (c->pool_in_use > c->pool_peak) c->pool_peak = c->pool_in_use;
    return p;
}
static void dfree(hisa_ctx* c, void* p) {
    if (!p) return;
    if (c->has_arena) { c->arena.release(p); return; }
    auto it = c->pool_sizes.find(p);
    if (it != c->pool_sizes.end()) { c->pool_in_use -= it->second; c->pool_sizes.erase(it); }
    cudaFreeAsync(p, c->stream);
}
template <class T>
static T* dalloc_t(hisa_ctx* c, size_t n) { return (T*)dalloc(c, n * sizeof(T)); }

// frees its allocations when the scope ends (scratch), or on an early error return only (outputs:
// keep() hands them to the caller) -- no arena leak on a failing call
struct DGuard {
    hisa_ctx* c;
    std::vector<void*> p;
    explicit DGuard(hisa_ctx* c_) : c(c_) {}
    template <class T> T* add(T* x) { if (x) p.push_back((void*)x); return x; }
    void keep() { p.clear(); }
    ~DGuard() { for (void* x : p) dfree(c, x); }
};

#define CK(call)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess) {                                                          \
            c->poisoned = true;                                                           \
            return fail(HISA_E_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
        }                                                                                 \
    } while (0)
#define CHECK_CTX(c)                                                              \
    do {                                                                          \
        if (!(c)) return fail(HISA_E_PARAMS, "null context");                     \
        if ((c)->poisoned) return fail(HISA_E_CUDA, "context poisoned by an earlier CUDA error"); \
    } while (0)
#define RET(x)                      \
    do {                            \
        int r_ = (x);               \
        if (r_ != HISA_OK) return r_; \
    } while (0)

// ---- launch accounting / profiling ----
static cudaEvent_t take_event(hisa_ctx* c) {
    if (!c->ev_pool.empty()) { cudaEvent_t e = c->ev_pool.back(); c->ev_pool.pop_back(); return e; }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}
struct ProfScope {
    hisa_ctx* c;
    hisa_ctx::ProfRec r;
    bool on;
    cudaStream_t st;
    ProfScope(hisa_ctx* c_, const char* name, cudaStream_t s = nullptr)
        : c(c_), on(c_->prof_on), st(s ? s : c_->stream) {
        c->launches++;
        if (on) {
            r.name = name;
            r.a = take_event(c);
            r.b = take_event(c);
            cudaEventRecord(r.a, st);
        }
    }
    ~ProfScope() {
        if (on) {
            cudaEventRecord(r.b, st);
            c->prof.push_back(r);
        }
    }
};
// launch `call` (returning cudaError_t) accounted under `name`
#define KL(name, call)                 \
    do {                               \
        ProfScope ps_(c, name);        \
        CK(call);                      \
    } while (0)
// the same for a launch on another stream (timed there)
#define KLS(name, stream, call)          \
    do {                                 \
        ProfScope ps_(c, name, stream);  \
        CK(call);                        \
    } while (0)

// ---- handle table ----
static uint64_t new_handle(hisa_ctx* c, int kind, uint64_t* ptr, int level, int npolys, double scale) {
    uint32_t slot;
    if (!c->free_slots.empty()) {
        slot = c->free_slots.back();
        c->free_slots.pop_back();
    } else {
        c->objs.push_back(Obj());
        slot = (uint32_t)c->objs.size() - 1;
        if (slot == 0) {   // slot 0 reserved: handle 0 is never valid
            c->objs.push_back(Obj());
            slot = 1;
        }
    }
    Obj& o = c->objs[slot];
    o.kind = kind;
    o.ptr = ptr;
    o.level = level;
    o.npolys = npolys;
    o.scale = scale;
    o.gen += 1;
    o.live = true;
    return ((uint64_t)o.gen << 32) | slot;
}
static Obj* get_obj(hisa_ctx* c, uint64_t h, int kind) {
    uint32_t slot = (uint32_t)h, gen = (uint32_t)(h >> 32);
    if (slot == 0 || slot >= c->objs.size()) return nullptr;
    Obj& o = c->objs[slot];
    if (!o.live || o.gen != gen || (kind && o.kind != kind)) return nullptr;
    return &o;
}
static size_t obj_words(const hisa_ctx* c, const Obj* o) {
    return (size_t)(o->kind == OBJ_CT ? o->npolys : 1) * (o->level + 1) * c->N;
}

// result placement: fresh handle, or in place (Assign form) on `self`
static int emit_ct(hisa_ctx* c, hisa_ct* out, hisa_ct self, uint64_t* ptr, int level, int npolys, double scale) {
    if (out) {
        *out = new_handle(c, OBJ_CT, ptr, level, npolys, scale);
        return HISA_OK;
    }
    Obj* o = get_obj(c, self, OBJ_CT);
    dfree(c, o->ptr);
    o->ptr = ptr;
    o->level = level;
    o->npolys = npolys;
    o->scale = scale;
    return HISA_OK;
}

#define GET_CT(var, h)                                                            \
    Obj* var = get_obj(c, h, OBJ_CT);                                            \
    if (!var) return fail(HISA_E_INVALID_HANDLE, "invalid ciphertext handle %llx", (unsigned long long)(h));
#define GET_PT(var, h)                                                            \
    Obj* var = get_obj(c, h, OBJ_PT);                                            \
    if (!var) return fail(HISA_E_INVALID_HANDLE, "invalid plaintext handle %llx", (unsigned long long)(h));

// ============================================================================================
// NTT helpers over contiguous limb arrays
// ============================================================================================
static PassJob job0() {
    PassJob j;
    memset(&j, 0, sizeof j);
    return j;
}
// forward NTT in place of `nz` arrays of `nlimbs` limbs (limb lambda mod mmap[lambda % nb])
static int ntt_fwd(hisa_ctx* c, uint64_t* const* ptrs, int nz, int nb, const uint8_t* mmap, int nlimbs = -1) {
    if (nlimbs < 0) nlimbs = nb;
    PassJob j = job0();
    for (int z = 0; z < nz; z++) { j.src[z] = ptrs[z]; j.dst[z] = ptrs[z]; }
    j.nb = nb;
    j.src_a = j.dst_a = (long long)nb * c->N;
    j.src_b = j.dst_b = (long long)c->N;
    for (int i = 0; i < nb; i++) j.mod_map[i] = mmap[i];
    Tables tb = c->tables();
    KL("ntt_fwd_cols", launch_fwd_pass1(j, tb, nlimbs, nz, false, c->stream));
    KL("ntt_fwd_rows", launch_fwd_pass2(j, tb, nlimbs, nz, false, c->stream));
    return HISA_OK;
}
static int ntt_inv(hisa_ctx* c, const uint64_t* const* src, uint64_t* const* dst, int nz, int nb, const uint8_t* mmap,
                   int nlimbs = -1) {
    if (nlimbs < 0) nlimbs = nb;
    PassJob j = job0();
    for (int z = 0; z < nz; z++) { j.src[z] = src[z]; j.dst[z] = dst[z]; }
    j.nb = nb;
    j.src_a = j.dst_a = (long long)nb * c->N;
    j.src_b = j.dst_b = (long long)c->N;
    for (int i = 0; i < nb; i++) j.mod_map[i] = mmap[i];
    Tables tb = c->tables();
    KL("ntt_inv_rows", launch_inv_passA(j, tb, nlimbs, nz, c->stream));
    for (int z = 0; z < nz; z++) j.src[z] = dst[z];
    KL("ntt_inv_cols", launch_inv_passB(j, tb, nlimbs, nz, c->stream));
    return HISA_OK;
}
static void ident_map(uint8_t* m, int n, int base = 0) {
    for (int i = 0; i < n; i++) m[i] = (uint8_t)(base + i);
}

// ============================================================================================
// context create / destroy
// ============================================================================================
extern "C" int hisa_ctx_create(const hisa_params* p, hisa_ctx** out) {
    if (!p || !out) return fail(HISA_E_PARAMS, "null argument");
    if (p->log_n < 8 || p->log_n > 16) return fail(HISA_E_PARAMS, "log_n must be in [8, 16]");
    if (p->num_q < 1 || p->num_q > MAXL - 4 || !p->q_bits) return fail(HISA_E_PARAMS, "num_q must be in [1, 60]");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(HISA_E_CUDA, "no CUDA device: libhisa has no CPU fallback");
    }
    if (p->device < 0 || p->device >= ndev) return fail(HISA_E_PARAMS, "bad device %d", p->device);
    hisa_ctx* c = new hisa_ctx();
    c->log_n = p->log_n;
    c->N = 1ull << p->log_n;
    c->L = p->num_q;
    c->seed = p->seed;
    c->device = p->device;
    if (cudaSetDevice(p->device) != cudaSuccess) { delete c; return fail(HISA_E_CUDA, "cudaSetDevice"); }
    // A3: special prime first, then q_0 .. q_{L-1}; per bit size descending from 2^b
    std::map<int, uint64_t> cursor;   // bits -> next k
    const uint64_t twoN = 2 * c->N;
    auto take = [&](int bits) -> uint64_t {
        if (bits < 20 || bits > 60) return 0;
        if (!cursor.count(bits)) cursor[bits] = ((1ull << bits) - 2) / twoN;
        for (uint64_t k = cursor[bits]; k > 0; k--) {
            uint64_t q = k * twoN + 1;
            if (h_prime(q)) { cursor[bits] = k - 1; return q; }
        }
        return 0;
    };
    uint64_t pp = take(p->p_bits);
    for (int i = 0; i < c->L; i++) c->mod.push_back(take(p->q_bits[i]));
    c->mod.push_back(pp);
    for (uint64_t q : c->mod)
        if (!q) { delete c; return fail(HISA_E_PARAMS, "prime bit sizes must be in [20, 60] with enough primes"); }
    const int M = c->L + 1;
    const uint64_t N = c->N;
    std::vector<ulonglong2> fwd((size_t)M * N), inv((size_t)M * N), ninv(M), pinv(M), qlinv((size_t)c->L * M);
    std::vector<double> fwd_d((size_t)M * N), inv_d((size_t)M * N), ninv_d(M);
    std::vector<double2> modd(M);
    std::vector<Mod> mods(M);
    for (int m = 0; m < M; m++) {
        const uint64_t q = c->mod[m];
        mods[m] = make_mod(q);
        const uint64_t psi = h_min_root(q, N), psii = h_inv(psi, q);
        // psi^k for k < N, then scatter to bit-reversed positions
        std::vector<uint64_t> pw(N), pwi(N);
        pw[0] = pwi[0] = 1;
        for (uint64_t k = 1; k < N; k++) { pw[k] = h_mul(pw[k - 1], psi, q); pwi[k] = h_mul(pwi[k - 1], psii, q); }
        for (uint64_t k = 0; k < N; k++) {
            const uint64_t w = pw[h_brv((uint32_t)k, c->log_n)], wi = pwi[h_brv((uint32_t)k, c->log_n)];
            fwd[(size_t)m * N + k] = make_ulonglong2(w, shoup(w, q));
            inv[(size_t)m * N + k] = make_ulonglong2(wi, shoup(wi, q));
            // centred (|W| <= q/2; exact where used, q < 2^50): halves the mulred bound (ntt_f64.cuh)
            fwd_d[(size_t)m * N + k] = w > q / 2 ? -(double)(q - w) : (double)w;
            inv_d[(size_t)m * N + k] = wi > q / 2 ? -(double)(q - wi) : (double)wi;
        }
        const uint64_t ni = h_inv(N % q, q);
        ninv[m] = make_ulonglong2(ni, shoup(ni, q));
        ninv_d[m] = (double)ni;
        modd[m] = make_double2((double)q, 1.0 / (double)q);
        const uint64_t pi = h_inv(pp % q, q);
        pinv[m] = make_ulonglong2(pi, shoup(pi, q));
    }
    for (int l = 0; l < c->L; l++)
        for (int m = 0; m < M; m++) {
            const uint64_t q = c->mod[m];
            const uint64_t v = (m == l) ? 0 : h_inv(c->mod[l] % q, q);
            qlinv[(size_t)l * M + m] = make_ulonglong2(v, shoup(v, q));
        }
    auto up = [&](void** dptr, const void* src, size_t bytes) -> bool {
        if (cudaMalloc(dptr, bytes) != cudaSuccess) return false;
        c->table_allocs.push_back(*dptr);
        return cudaMemcpy(*dptr, src, bytes, cudaMemcpyHostToDevice) == cudaSuccess;
    };
    bool ok = up((void**)&c->d_mods, mods.data(), M * sizeof(Mod)) &&
              up((void**)&c->d_fwd, fwd.data(), fwd.size() * sizeof(ulonglong2)) &&
              up((void**)&c->d_inv, inv.data(), inv.size() * sizeof(ulonglong2)) &&
              up((void**)&c->d_ninv, ninv.data(), M * sizeof(ulonglong2)) &&
              up((void**)&c->d_pinv, pinv.data(), M * sizeof(ulonglong2)) &&
              up((void**)&c->d_qlinv, qlinv.data(), qlinv.size() * sizeof(ulonglong2)) &&
              up((void**)&c->d_fwd_d, fwd_d.data(), fwd_d.size() * sizeof(double)) &&
              up((void**)&c->d_inv_d, inv_d.data(), inv_d.size() * sizeof(double)) &&
              up((void**)&c->d_ninv_d, ninv_d.data(), M * sizeof(double)) &&
              up((void**)&c->d_modd, modd.data(), M * sizeof(double2));
    if (!ok) {
        for (void* q : c->table_allocs) cudaFree(q);
        delete c;
        cudaGetLastError();
        return fail(HISA_E_CUDA, "table upload failed");
    }
    c->objs.push_back(Obj());   // slot 0 reserved
    *out = c;
    return HISA_OK;
}

extern "C" int hisa_ctx_destroy(hisa_ctx* c) {
    if (!c) return HISA_OK;
    cudaStreamSynchronize(c->stream);
    if (!c->has_arena) {
        for (auto& kv : c->pool_sizes) cudaFree(kv.first);
    }
    for (void* q : c->table_allocs) cudaFree(q);
    if (c->side) cudaStreamDestroy(c->side);
    for (cudaEvent_t e : {c->ev_fork, c->ev_join, c->ev_k7[0], c->ev_k7[1], c->ev_md[0], c->ev_md[1]})
        if (e) cudaEventDestroy(e);
    cudaGetLastError();
    delete c;
    return HISA_OK;
}

extern "C" int hisa_attach_arena(hisa_ctx* c, void* dev_ptr, size_t bytes) {
    CHECK_CTX(c);
    if (!dev_ptr || bytes < 4096) return fail(HISA_E_PARAMS, "bad arena");
    if (c->has_arena || !c->pool_sizes.empty()) return fail(HISA_E_PARAMS, "arena must be attached before allocation");
    c->arena.attach(dev_ptr, bytes);
    c->has_arena = true;
    return HISA_OK;
}
extern "C" int hisa_set_stream(hisa_ctx* c, void* stream) {
    CHECK_CTX(c);
    CK(cudaStreamSynchronize(c->stream));
    c->stream = (cudaStream_t)stream;
    return HISA_OK;
}
extern "C" int hisa_sync(hisa_ctx* c) {
    CHECK_CTX(c);
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaGetLastError());
    return HISA_OK;
}
extern "C" int hisa_supports(const hisa_ctx* c, int profile) {
    if (!c) return 0;
    return (profile & HISA_PROFILE_BOOTSTRAP) ? 0
           : (profile & (HISA_PROFILE_ENCRYPTION | HISA_PROFILE_INTEGERS | HISA_PROFILE_DIVISION | HISA_PROFILE_RELIN)) ? 1 : 0;
}
extern "C" int hisa_moduli(const hisa_ctx* c, uint64_t* out, size_t n) {
    if (!c || !out || n < c->mod.size()) return fail(HISA_E_PARAMS, "buffer too small");
    for (size_t i = 0; i < c->mod.size(); i++) out[i] = c->mod[i];
    return HISA_OK;
}
extern "C" int hisa_ring_degree(const hisa_ctx* c, uint64_t* n_out, int* num_q_out) {
    if (!c) return fail(HISA_E_PARAMS, "null context");
    if (n_out) *n_out = c->N;
    if (num_q_out) *num_q_out = c->L;
    return HISA_OK;
}
extern "C" int hisa_mem_stats(const hisa_ctx* c, size_t* in_use, size_t* peak) {
    if (!c) return fail(HISA_E_PARAMS, "null context");
    if (in_use) *in_use = c->has_arena ? c->arena.in_use : c->pool_in_use;
    if (peak) *peak = c->has_arena ? c->arena.peak : c->pool_peak;
    return HISA_OK;
}

// ============================================================================================
// keys (A9-A16) and encryption (A12) -- all sampling and arithmetic in kernels
// ============================================================================================
enum { TAG_SK = 1, TAG_PK_A = 2, TAG_PK_E = 3, TAG_ENC_V = 4, TAG_ENC_E0 = 5, TAG_ENC_E1 = 6,
       TAG_KSK_A = 7, TAG_KSK_E = 8, TAG_BENCH = 9 };

// b[r] = e[r] - a[r] s[r] (+ gadget * sp[r] on limb `glimb`) over nl limbs (limb r mod mods[mmap[r]])
struct KeyAsmJob { uint8_t mmap[MAXL]; };
__global__ void k_key_assemble(uint64_t* b, const uint64_t* a, const uint64_t* s, const uint64_t* sp, int glimb,
                               uint64_t gadget, KeyAsmJob job, int nl, int log_n, const Mod* mods) {
    const long long N = 1ll << log_n;
    const long long total = N * nl;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int r = (int)(idx >> log_n);
        const Mod md = mods[job.mmap[r]];
        uint64_t v = sub_mod(b[idx], mul_mod(a[idx], s[(long long)job.mmap[r] * N + (idx & (N - 1))], md), md.q);
        if (r == glimb) v = add_mod(v, mul_mod(gadget, sp[(long long)job.mmap[r] * N + (idx & (N - 1))], md), md.q);
        b[idx] = v;
    }
}
// Internal key-switching-key format (K4 v6 / K7 inner products on the FP64 pipe):
// limbs of FP64-engine moduli (q < 2^50) hold the centred residue K - q [K > q/2] as an exact
// double (|K| <= q/2 halves the MAC bound), the others the canonical residue.  dir = +1:
// canonical -> internal (keygen), -1: internal -> canonical (hisa_key_export).
__global__ void k_key_format(uint64_t* key, int kL, int L, int log_n, const Mod* mods, uint64_t fp_mods, int dir) {
    const long long N = 1ll << log_n;
    const long long total = (long long)kL * 2 * (kL + 1) * N;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int r = (int)((idx >> log_n) % (kL + 1));
        const int mi = r < kL ? r : L;
        if (!((fp_mods >> mi) & 1)) continue;
        const uint64_t q = mods[mi].q;
        if (dir > 0) {
            const uint64_t u = key[idx];
            const double d = u > (q >> 1) ? -(double)(q - u) : (double)u;
            key[idx] = (uint64_t)__double_as_longlong(d);
        } else {
            const double d = __longlong_as_double((long long)key[idx]);
            key[idx] = d < 0.0 ? q - (uint64_t)(-d) : (uint64_t)d;
        }
    }
}
static int key_format(hisa_ctx* c, uint64_t* key, int kL, int dir) {
    const Tables tb = c->tables();
    k_key_format<<<1184, 256, 0, c->stream>>>(key, kL, c->L, c->log_n, c->d_mods, tb.fp_mods, dir);
    CK(cudaGetLastError());
    return HISA_OK;
}

// c0 = v pk_b + e0 + m ; c1 = v pk_a + e1 (all NTT, limbs 0..l)
__global__ void k_enc_assemble(uint64_t* ct, const uint64_t* v, const uint64_t* e0, const uint64_t* e1,
                               const uint64_t* m, const uint64_t* pk, int l1, int L, int log_n, const Mod* mods) {
    const long long N = 1ll << log_n;
    const long long total = N * l1;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(idx >> log_n);
        const Mod md = mods[i];
        const uint64_t pb = pk[idx], pa = pk[(long long)L * N + idx];
        ct[idx] = add_mod(add_mod(mul_mod(v[idx], pb, md), e0[idx], md.q), m[idx], md.q);
        ct[(long long)l1 * N + idx] = add_mod(mul_mod(v[idx], pa, md), e1[idx], md.q);
    }
}

static int sample_small_ntt(hisa_ctx* c, uint32_t tag, uint64_t index, int kind, int nl, uint64_t* out) {
    int64_t* tmp = dalloc_t<int64_t>(c, c->N);
    if (!tmp) return fail(HISA_E_OOM, "sampler scratch");
    uint8_t mm[MAXL];
    ident_map(mm, nl);
    KL("rng_small", launch_sample_small(tmp, c->seed, tag, index, kind, c->log_n, c->stream));
    KL("int_to_limbs", launch_int_to_limbs(tmp, out, mm, nl, c->log_n, c->d_mods, c->stream));
    uint64_t* pp[1] = {out};
    RET(ntt_fwd(c, pp, 1, nl, mm));
    dfree(c, tmp);
    return HISA_OK;
}

static int gen_ksk(hisa_ctx* c, uint64_t keyid, const uint64_t* sp, uint64_t** out) {
    const int L = c->L, M = L + 1;
    const uint64_t N = c->N;
    uint64_t* key = dalloc_t<uint64_t>(c, key_words(c));
    if (!key) return fail(HISA_E_OOM, "key allocation (%zu MiB)", key_words(c) * 8 >> 20);
    uint8_t mm[MAXL];
    ident_map(mm, M);
    uint64_t idx[MAXL];
    for (int j = 0; j < L; j++) {
        uint64_t* b = key + (size_t)j * 2 * M * N;
        uint64_t* a = b + (size_t)M * N;
        RET(sample_small_ntt(c, TAG_KSK_E, (keyid << 32) | (uint64_t)j, 1, M, b));
        for (int r = 0; r < M; r++) idx[r] = (keyid << 32) | ((uint64_t)j << 16) | (uint64_t)r;
        CK(launch_sample_uniform(a, c->seed, TAG_KSK_A, idx, mm, M, c->log_n, c->d_mods, c->stream));
        KeyAsmJob kj;
        ident_map(kj.mmap, M);
        const uint64_t gadget = c->mod[L] % c->mod[j];   // [P]_{q_j}
        k_key_assemble<<<592, 256, 0, c->stream>>>(b, a, c->d_sk, sp, j, gadget, kj, M, c->log_n, c->d_mods);
        CK(cudaGetLastError());
    }
    *out = key;
    return HISA_OK;
}

extern "C" int hisa_keygen(hisa_ctx* c, const int64_t* rot, size_t n, int relin, int max_level) {
    CHECK_CTX(c);
    if (n && !rot) return fail(HISA_E_PARAMS, "null rotation list");
    if (max_level < -1 || max_level >= c->L) return fail(HISA_E_PARAMS, "max_level %d outside [-1, %d]", max_level, c->L - 1);
    const int kL = max_level < 0 ? c->L : max_level + 1;
    const int L = c->L, M = L + 1;
    const uint64_t N = c->N, slots = N / 2;
    uint8_t mm[MAXL];
    ident_map(mm, M);
    if (!c->have_sk) {
        c->d_s_int = dalloc_t<int64_t>(c, N);
        c->d_sk = dalloc_t<uint64_t>(c, (size_t)M * N);
        c->d_pk = dalloc_t<uint64_t>(c, (size_t)2 * L * N);
        if (!c->d_s_int || !c->d_sk || !c->d_pk) return fail(HISA_E_OOM, "key allocation");
        CK(launch_sample_small(c->d_s_int, c->seed, TAG_SK, 0, 0, c->log_n, c->stream));
        CK(launch_int_to_limbs(c->d_s_int, c->d_sk, mm, M, c->log_n, c->d_mods, c->stream));
        uint64_t* pp[1] = {c->d_sk};
        RET(ntt_fwd(c, pp, 1, M, mm));
        // pk = (-a s + e, a) over q_0..q_{L-1}
        RET(sample_small_ntt(c, TAG_PK_E, 0, 1, L, c->d_pk));
        uint64_t idx[MAXL];
        for (int m = 0; m < L; m++) idx[m] = (uint64_t)m;
        CK(launch_sample_uniform(c->d_pk + (size_t)L * N, c->seed, TAG_PK_A, idx, mm, L, c->log_n, c->d_mods,
                                 c->stream));
        KeyAsmJob kj;
        ident_map(kj.mmap, L);
        k_key_assemble<<<592, 256, 0, c->stream>>>(c->d_pk, c->d_pk + (size_t)L * N, c->d_sk, nullptr, -1, 0, kj, L,
                                                   c->log_n, c->d_mods);
        CK(cudaGetLastError());
        c->have_sk = true;
    }
    if (relin && !c->d_rlk) {
        uint64_t* sp = dalloc_t<uint64_t>(c, (size_t)M * N);
        if (!sp) return fail(HISA_E_OOM, "relin target");
        ElemJob ej;
        memset(&ej, 0, sizeof ej);
        ej.a[0] = c->d_sk; ej.b[0] = c->d_sk; ej.out[0] = sp;
        ej.npolys = 1; ej.nl = M; ej.log_n = c->log_n;
        KL("elementwise", launch_elem(EL_MUL_PLAIN, ej, c->d_mods, 1, c->stream));
        RET(gen_ksk(c, 0, sp, &c->d_rlk));
        RET(key_format(c, c->d_rlk, L, +1));
        dfree(c, sp);
    }
    for (size_t i = 0; i < n; i++) {
        int64_t k = rot[i] % (int64_t)slots;
        if (k < 0) k += (int64_t)slots;
        if (k == 0) continue;
        auto have = c->rot_keys.find((uint64_t)k);
        if (have != c->rot_keys.end()) {
            if (have->second.kL >= kL) continue;
            dfree(c, have->second.p);      // regenerate at the higher level (same words on the shared blocks)
            c->rot_keys.erase(have);
        }
        const uint64_t g = h_pow(5, (uint64_t)k, 2 * N);
        int64_t* sg = dalloc_t<int64_t>(c, N);
        uint64_t* sp = dalloc_t<uint64_t>(c, (size_t)M * N);
        if (!sg || !sp) return fail(HISA_E_OOM, "rotation target");
        CK(launch_automorphism_int(c->d_s_int, sg, c->log_n, g, c->stream));
        CK(launch_int_to_limbs(sg, sp, mm, M, c->log_n, c->d_mods, c->stream));
        uint64_t* pp[1] = {sp};
        RET(ntt_fwd(c, pp, 1, M, mm));
        uint64_t* key = nullptr;
        RET(gen_ksk(c, (uint64_t)k, sp, &key));
        if (kL < L) {   // truncate: digits j < kL, moduli q_0..q_{kL-1} and p (the same words)
            uint64_t* tr = dalloc_t<uint64_t>(c, key_words(c, kL));
            if (!tr) return fail(HISA_E_OOM, "key allocation (%zu MiB)", key_words(c, kL) * 8 >> 20);
            for (int j = 0; j < kL; j++)
                for (int h = 0; h < 2; h++) {
                    const uint64_t* src = key + ((size_t)j * 2 + h) * M * N;
                    uint64_t* dst = tr + ((size_t)j * 2 + h) * (kL + 1) * N;
                    CK(cudaMemcpyAsync(dst, src, (size_t)kL * N * 8, cudaMemcpyDeviceToDevice, c->stream));
                    CK(cudaMemcpyAsync(dst + (size_t)kL * N, src + (size_t)L * N, N * 8, cudaMemcpyDeviceToDevice,
                                       c->stream));
                }
            dfree(c, key);
            key = tr;
        }
        // store key' = psi_g^-1(key) (see "Rotation" below); psi_g^-1 = psi_{5^(N/2 - k)}
        uint64_t* kp = dalloc_t<uint64_t>(c, key_words(c, kL));
        if (!kp) return fail(HISA_E_OOM, "key allocation (%zu MiB)", key_words(c, kL) * 8 >> 20);
        const uint64_t ginv = h_pow(5, slots - (uint64_t)k, 2 * N);
        const uint64_t* kin[1] = {key};
        uint64_t* kout[1] = {kp};
        KL("automorphism", launch_automorphism(kin, kout, 1, 2 * kL * (kL + 1), c->log_n, &ginv, c->stream));
        dfree(c, key);
        RET(key_format(c, kp, kL, +1));
        c->rot_keys[(uint64_t)k] = hisa_ctx::KeyRec{kp, kL};
        dfree(c, sg);
        dfree(c, sp);
    }
    return HISA_OK;
}

extern "C" int hisa_key_export(hisa_ctx* c, int64_t which, uint64_t* host, size_t words) {
    CHECK_CTX(c);
    if (!c->have_sk) return fail(HISA_E_NO_SECRET, "keygen first");
    const uint64_t* src = nullptr;
    size_t w = 0;
    if (which == -1) { src = c->d_pk; w = (size_t)2 * c->L * c->N; }
    else if (which == -2) { src = c->d_sk; w = (size_t)(c->L + 1) * c->N; }
    else if (which == 0) { src = c->d_rlk; w = key_words(c); }
    int kL = c->L;
    if (which > 0 && c->rot_keys.count((uint64_t)which)) {
        src = c->rot_keys[(uint64_t)which].p;
        kL = c->rot_keys[(uint64_t)which].kL;
        w = key_words(c, kL);
    }
    if (!src) return fail(HISA_E_NO_KEY, "no such key %lld", (long long)which);
    if (words != w) return fail(HISA_E_PARAMS, "key has %zu words", w);
    uint64_t* canon = nullptr;
    if (which >= 0) {   // key-switching keys: canonical words (internal FP64 format undone) ...
        canon = dalloc_t<uint64_t>(c, w);
        if (!canon) return fail(HISA_E_OOM, "key export");
        if (which > 0) {   // ... and rotation keys un-permuted (stored pre-permuted, A37)
            const uint64_t g = h_pow(5, (uint64_t)which, 2 * c->N);
            const uint64_t* kin[1] = {src};
            uint64_t* kout[1] = {canon};
            KL("automorphism", launch_automorphism(kin, kout, 1, 2 * kL * (kL + 1), c->log_n, &g, c->stream));
        } else {
            CK(cudaMemcpyAsync(canon, src, w * 8, cudaMemcpyDeviceToDevice, c->stream));
        }
        RET(key_format(c, canon, kL, -1));
        src = canon;
    }
    CK(cudaMemcpyAsync(host, src, w * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (canon) dfree(c, canon);
    return HISA_OK;
}

extern "C" int hisa_encrypt(hisa_ctx* c, hisa_pt pt, hisa_ct* out) {
    CHECK_CTX(c);
    GET_PT(p, pt);
    if (!out) return fail(HISA_E_PARAMS, "null out");
    if (!c->have_sk) return fail(HISA_E_NO_SECRET, "keygen first");
    const int l1 = p->level + 1;
    const uint64_t N = c->N;
    uint64_t* tmp = dalloc_t<uint64_t>(c, (size_t)3 * l1 * N);
    uint64_t* ct = dalloc_t<uint64_t>(c, (size_t)2 * l1 * N);
    if (!tmp || !ct) return fail(HISA_E_OOM, "encrypt");
    const uint64_t ctr = c->enc_counter++;
    RET(sample_small_ntt(c, TAG_ENC_V, ctr, 0, l1, tmp));
    RET(sample_small_ntt(c, TAG_ENC_E0, ctr, 1, l1, tmp + (size_t)l1 * N));
    RET(sample_small_ntt(c, TAG_ENC_E1, ctr, 1, l1, tmp + (size_t)2 * l1 * N));
    k_enc_assemble<<<592, 256, 0, c->stream>>>(ct, tmp, tmp + (size_t)l1 * N, tmp + (size_t)2 * l1 * N, p->ptr, c->d_pk,
                                               l1, c->L, c->log_n, c->d_mods);
    CK(cudaGetLastError());
    dfree(c, tmp);
    *out = new_handle(c, OBJ_CT, ct, p->level, 2, p->scale);
    return HISA_OK;
}

extern "C" int hisa_decrypt(hisa_ctx* c, hisa_ct h, hisa_pt* out) {
    CHECK_CTX(c);
    GET_CT(o, h);
    if (!out) return fail(HISA_E_PARAMS, "null out");
    if (!c->have_sk) return fail(HISA_E_NO_SECRET, "keygen first");
    const int l1 = o->level + 1;
    uint64_t* pt = dalloc_t<uint64_t>(c, (size_t)l1 * c->N);
    if (!pt) return fail(HISA_E_OOM, "decrypt");
    ElemJob ej;
    memset(&ej, 0, sizeof ej);
    ej.a[0] = o->ptr; ej.b[0] = c->d_sk; ej.out[0] = pt;
    ej.npolys = 1; ej.nl = l1; ej.log_n = c->log_n;
    ej.a_poly = (long long)l1 * c->N;
    KL("elementwise", launch_elem(o->npolys == 3 ? EL_DECRYPT3 : EL_DECRYPT2, ej, c->d_mods, 1, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    *out = new_handle(c, OBJ_PT, pt, o->level, 1, o->scale);
    return HISA_OK;
}

extern "C" int hisa_free(hisa_ctx* c, uint64_t h) {
    if (!c) return fail(HISA_E_PARAMS, "null context");
    Obj* o = get_obj(c, h, 0);
    if (!o) return fail(HISA_E_INVALID_HANDLE, "invalid handle %llx", (unsigned long long)h);
    dfree(c, o->ptr);
    o->ptr = nullptr;
    o->live = false;
    c->free_slots.push_back((uint32_t)h);
    return HISA_OK;
}

static int copy_obj(hisa_ctx* c, const Obj* o, uint64_t** out) {
    const size_t w = obj_words(c, o);
    uint64_t* p = dalloc_t<uint64_t>(c, w);
    if (!p) return fail(HISA_E_OOM, "copy");
    CK(cudaMemcpyAsync(p, o->ptr, w * 8, cudaMemcpyDeviceToDevice, c->stream));
    *out = p;
    return HISA_OK;
}

extern "C" int hisa_copy(hisa_ctx* c, hisa_ct h, hisa_ct* out) {
    CHECK_CTX(c);
    GET_CT(o, h);
    if (!out) return fail(HISA_E_PARAMS, "null out");
    uint64_t* p;
    RET(copy_obj(c, o, &p));
    *out = new_handle(c, OBJ_CT, p, o->level, o->npolys, o->scale);
    return HISA_OK;
}

// ============================================================================================
// encode / decode (A7, A13): host boundary, long-double FFT, binary128 near-tie recomputation
// ============================================================================================
// one coefficient exactly (the A7 near-tie path): binary128 direct sum of v_t with a correctly
// rounded binary128 cos table.  Its error is below E = (n + 2) 2^-112 (scale/N) sum_j |2 z_j|
// (< 2^-36 even at |v| = 2^62, N = 2^16), so the result is round-half-away of the exact real
// v_t whenever v_t is farther than E from a half-integer; exact ties (e.g. the t = 0 coefficient
// of a constant vector, a sum of exact terms) are computed exactly.  Pinned against exact
// Decimal sums near ties in tests/test_oracle_pins.py (oracle) and tests/test_gpu_edges.py (GPU).
static int exact_coeff_q(hisa_ctx* c, const double* z, size_t n, double scale, uint64_t t, int64_t* out) {
    const uint64_t N = c->N, twoN = 2 * N;
    std::vector<__float128>& cq = c->enc_cosq;
    if (cq.empty()) {
        cq.resize(twoN);
        for (uint64_t e = 0; e < twoN; e++) cq[e] = cosq(M_PIq * (__float128)e / (__float128)N);
    }
    __float128 acc = 0;
    uint64_t k = 1;
    for (size_t j = 0; j < n; j++) {
        if (z[j] != 0.0) acc += 2 * (__float128)z[j] * cq[(uint64_t)((u128)k * t % twoN)];
        k = k * 5 % twoN;
    }
    acc = acc * (__float128)scale / (__float128)N;
    __float128 rq = floorq(fabsq(acc) + 0.5Q);
    const __float128 r = acc < 0 ? -rq : rq;
    if (!(fabsq(r) < 0x1p62Q)) return fail(HISA_E_PARAMS, "encoded coefficient exceeds 2^62");
    *out = (int64_t)r;
    return HISA_OK;
}

static int enc_gpu_tables(hisa_ctx* c) {
    if (c->d_enc_root) return HISA_OK;
    const uint64_t N = c->N, twoN = 2 * N;
    std::vector<uint32_t> pos(N);
    uint64_t k = 1;
    for (uint64_t j = 0; j < N / 2; j++) {      // slot j -> positions (k-1)/2 and (2N-k-1)/2, bit-reversed
        pos[2 * j] = h_brv((uint32_t)((k - 1) / 2), c->log_n);
        pos[2 * j + 1] = h_brv((uint32_t)((twoN - k - 1) / 2), c->log_n);
        k = k * 5 % twoN;
    }
    auto to_dd = [](__float128 x) { const double hi = (double)x; return dd{hi, (double)(x - (__float128)hi)}; };
    std::vector<cdd> root(N / 2), twist(N);
    for (uint64_t i = 0; i < N / 2; i++) {
        const __float128 a = 2 * M_PIq * (__float128)i / (__float128)N;
        root[i] = cdd{to_dd(cosq(a)), to_dd(sinq(a))};
    }
    for (uint64_t t = 0; t < N; t++) {
        const __float128 a = M_PIq * (__float128)t / (__float128)N;
        twist[t] = cdd{to_dd(cosq(a)), to_dd(sinq(a))};
    }
    auto up = [&](void** dptr, const void* src, size_t bytes) -> bool {
        if (cudaMalloc(dptr, bytes) != cudaSuccess) return false;
        c->table_allocs.push_back(*dptr);
        return cudaMemcpy(*dptr, src, bytes, cudaMemcpyHostToDevice) == cudaSuccess;
    };
    if (!up((void**)&c->d_enc_pos, pos.data(), N * 4) || !up((void**)&c->d_enc_root, root.data(), N / 2 * sizeof(cdd)) ||
        !up((void**)&c->d_enc_twist, twist.data(), N * sizeof(cdd))) {
        cudaGetLastError();
        return fail(HISA_E_CUDA, "encode table upload failed");
    }
    return HISA_OK;
}

// GPU encode (NEXT-4) of count rows of n_per slot values into int64 coefficients dm[count][N]:
// double-double FFT, exact rounding except inside a tie window sized from the dd error bound,
// those few coefficients recomputed exactly (binary128) on the host.  Equal to the host / oracle
// exact encoding (A7) bit for bit.
static int encode_to_device(hisa_ctx* c, const double* v, size_t n_per, size_t count, double scale, int64_t* dm) {
    RET(enc_gpu_tables(c));
    const uint64_t N = c->N;
    // error bound of the dd FFT: |err(v_t)| <= log2(N) * c * 2^-104 * (scale/N) * 2 sum_j |z_j|;
    // take 2^-88 * scale * (2/N) sum |z| (>= 2^10 margin) and never below 2^-40
    double smax = 0;
    for (size_t p = 0; p < count; p++) {
        double sa = 0;
        for (size_t j = 0; j < n_per; j++) sa += fabs(v[p * n_per + j]);
        smax = std::max(smax, sa);
    }
    const double window = std::max(0x1p-40, 0x1p-88 * scale * 2.0 * smax / (double)N);
    if (window > 0x1p-4) return fail(HISA_E_PARAMS, "scale too large for exact GPU encoding");
    const unsigned int max_flags = 4096;
    const size_t zbytes = std::max<size_t>(8, n_per * count * 8);
    double* dz = (double*)dalloc(c, zbytes);
    cdd* A = dalloc_t<cdd>(c, (size_t)N * count);
    uint32_t* flags = dalloc_t<uint32_t>(c, max_flags + 4);
    if (!dz || !A || !flags) return fail(HISA_E_OOM, "encode scratch");
    unsigned int* nflag = flags + max_flags;
    int* overflow = (int*)(flags + max_flags + 1);
    CK(cudaMemsetAsync(nflag, 0, 8, c->stream));
    if (n_per) CK(cudaMemcpyAsync(dz, v, n_per * count * 8, cudaMemcpyHostToDevice, c->stream));
    {
        ProfScope ps_(c, "encode_fft");
        CK(launch_encode_fft(dz, n_per, count, c->d_enc_pos, c->d_enc_root, c->d_enc_twist, scale / (double)N,
                             window, c->log_n, A, dm, flags, nflag, max_flags, overflow, c->stream));
    }
    unsigned int hf[2];
    CK(cudaMemcpyAsync(hf, nflag, 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (hf[1]) return fail(HISA_E_PARAMS, "encoded coefficient exceeds 2^62");
    if (hf[0]) {   // near ties: exact binary128 recomputation on the host
        if (hf[0] > max_flags) return fail(HISA_E_PARAMS, "too many near-tie coefficients (%u)", hf[0]);
        std::vector<uint32_t> idx(hf[0]);
        std::vector<int64_t> val(hf[0]);
        CK(cudaMemcpy(idx.data(), flags, hf[0] * 4, cudaMemcpyDeviceToHost));
        for (unsigned int i = 0; i < hf[0]; i++) {
            const uint64_t p = idx[i] / N, t = idx[i] % N;
            RET(exact_coeff_q(c, v + p * n_per, n_per, scale, t, &val[i]));
            CK(cudaMemcpyAsync(dm + idx[i], &val[i], 8, cudaMemcpyHostToDevice, c->stream));
        }
        CK(cudaStreamSynchronize(c->stream));
    }
    dfree(c, dz);
    dfree(c, A);
    dfree(c, flags);
    return HISA_OK;
}

extern "C" int hisa_encode(hisa_ctx* c, const double* v, size_t n, double scale, int level, hisa_pt* out) {
    CHECK_CTX(c);
    if (!out || (n && !v)) return fail(HISA_E_PARAMS, "null argument");
    if (n > c->N / 2) return fail(HISA_E_CAPACITY, "%zu values > N/2 = %llu slots", n, (unsigned long long)(c->N / 2));
    if (level < 0) level = c->L - 1;
    if (level >= c->L) return fail(HISA_E_PARAMS, "level %d >= L", level);
    if (!(scale > 0) || !std::isfinite(scale)) return fail(HISA_E_PARAMS, "bad scale");
    for (size_t i = 0; i < n; i++)
        if (!std::isfinite(v[i])) return fail(HISA_E_PARAMS, "non-finite slot value");
    const int l1 = level + 1;
    int64_t* dm = dalloc_t<int64_t>(c, c->N);
    uint64_t* pt = dalloc_t<uint64_t>(c, (size_t)l1 * c->N);
    if (!dm || !pt) return fail(HISA_E_OOM, "encode");
    RET(encode_to_device(c, v, n, 1, scale, dm));
    uint8_t mm[MAXL];
    ident_map(mm, l1);
    CK(launch_int_to_limbs(dm, pt, mm, l1, c->log_n, c->d_mods, c->stream));
    uint64_t* pp[1] = {pt};
    RET(ntt_fwd(c, pp, 1, l1, mm));
    dfree(c, dm);
    *out = new_handle(c, OBJ_PT, pt, level, 1, scale);
    return HISA_OK;
}

// count plaintexts of n_per slot values each (v row-major): the exact encoding (A7) of every row
// on the GPU in chunks (double-double FFT, encode_to_device), limbs + NTT batched: a layer's
// weight / mask plaintexts in one call
extern "C" int hisa_encode_batch(hisa_ctx* c, const double* v, size_t n_per, size_t count, double scale, int level,
                                 hisa_pt* outs) {
    CHECK_CTX(c);
    if ((!v || !outs) && count) return fail(HISA_E_PARAMS, "null argument");
    if (count == 0) return HISA_OK;
    if (n_per > c->N / 2) return fail(HISA_E_CAPACITY, "%zu values > N/2", n_per);
    if (level < 0) level = c->L - 1;
    if (level >= c->L) return fail(HISA_E_PARAMS, "level %d >= L", level);
    if (!(scale > 0) || !std::isfinite(scale)) return fail(HISA_E_PARAMS, "bad scale");
    for (size_t i = 0; i < n_per * count; i++)
        if (!std::isfinite(v[i])) return fail(HISA_E_PARAMS, "non-finite slot value");
    const uint64_t N = c->N;
    const int l1 = level + 1;
    // chunk so the dd FFT workspace (32 B per coefficient) stays near 128 MiB
    const size_t chunk = std::max<size_t>(1, std::min<size_t>(MAXB, ((size_t)128 << 20) / (N * sizeof(cdd))));
    int64_t* dm = dalloc_t<int64_t>(c, chunk * N);
    if (!dm) return fail(HISA_E_OOM, "encode batch staging");
    uint8_t mmap[MAXL];
    ident_map(mmap, l1);
    for (size_t i0 = 0; i0 < count; i0 += chunk) {
        const size_t nc = std::min(chunk, count - i0);
        RET(encode_to_device(c, v + i0 * n_per, n_per, nc, scale, dm));
        std::vector<uint64_t*> pts(nc);
        for (size_t i = 0; i < nc; i++) {
            pts[i] = dalloc_t<uint64_t>(c, (size_t)l1 * N);
            if (!pts[i]) return fail(HISA_E_OOM, "encode batch");
            CK(launch_int_to_limbs(dm + i * N, pts[i], mmap, l1, c->log_n, c->d_mods, c->stream));
        }
        RET(ntt_fwd(c, pts.data(), (int)nc, l1, mmap));
        for (size_t i = 0; i < nc; i++) outs[i0 + i] = new_handle(c, OBJ_PT, pts[i], level, 1, scale);
    }
    dfree(c, dm);
    return HISA_OK;
}

// GPU decode (NEXT-4; A2, A13): INTT of limb 0, then twist + N-point FFT + gather of
// the slots' real parts on the device (encode_kernels.cu); out[i][j], j < n, for count plaintexts
extern "C" int hisa_decode_batch(hisa_ctx* c, const hisa_pt* pts, size_t count, double* out, size_t n) {
    CHECK_CTX(c);
    if (n > c->N / 2) return fail(HISA_E_CAPACITY, "n > N/2");
    if (count && (!pts || (n && !out))) return fail(HISA_E_PARAMS, "null argument");
    if (count == 0) return HISA_OK;
    const uint64_t N = c->N;
    std::vector<Obj*> ps(count);
    for (size_t i = 0; i < count; i++) {
        ps[i] = get_obj(c, pts[i], OBJ_PT);
        if (!ps[i]) return fail(HISA_E_INVALID_HANDLE, "invalid plaintext handle at %zu", i);
    }
    RET(enc_gpu_tables(c));
    const size_t chunk = std::min<size_t>(count, MAXB);
    DGuard scratch(c);
    uint64_t* tmp = scratch.add(dalloc_t<uint64_t>(c, N * chunk));
    void* A = scratch.add(dalloc(c, N * chunk * 16));
    double* dout = scratch.add(dalloc_t<double>(c, std::max<size_t>(1, n * chunk)));
    double* dinv = scratch.add(dalloc_t<double>(c, chunk));
    const uint64_t** dm = scratch.add((const uint64_t**)dalloc(c, chunk * sizeof(void*)));
    if (!tmp || !A || !dout || !dinv || !dm) return fail(HISA_E_OOM, "decode");
    std::vector<double> inv(chunk);
    std::vector<const uint64_t*> mp(chunk);
    for (size_t i0 = 0; i0 < count; i0 += chunk) {
        const size_t m = std::min(chunk, count - i0);
        uint8_t mm[1] = {0};
        const uint64_t* s_[MAXB];
        uint64_t* d_[MAXB];
        for (size_t i = 0; i < m; i++) {
            s_[i] = ps[i0 + i]->ptr;
            d_[i] = tmp + i * N;
            mp[i] = d_[i];
            inv[i] = 1.0 / ps[i0 + i]->scale;
        }
        RET(ntt_inv(c, s_, d_, (int)m, 1, mm));
        CK(cudaMemcpyAsync(dm, mp.data(), m * sizeof(void*), cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(dinv, inv.data(), m * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        KL("decode", launch_decode_fft(dm, m, c->mod[0], c->d_enc_pos, c->d_enc_root, c->d_enc_twist, dinv, c->log_n,
                                       A, dout, n, c->stream));
        if (n) CK(cudaMemcpyAsync(out + i0 * n, dout, m * n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));   // the host staging vectors are reused
    }
    return HISA_OK;
}

extern "C" int hisa_decode(hisa_ctx* c, hisa_pt h, double* out, size_t n) {
    return hisa_decode_batch(c, &h, 1, out, n);
}

// ============================================================================================
// elementwise instructions (a3, a4)
// ============================================================================================
static ElemJob ejob(const hisa_ctx* c, int npolys, int level) {
    ElemJob j;
    memset(&j, 0, sizeof j);
    j.npolys = npolys;
    j.nl = level + 1;
    j.log_n = c->log_n;
    j.a_poly = j.b_poly = j.out_poly = (long long)(level + 1) * c->N;
    j.fp_mods = c->tables().fp_mods & ((level + 1 >= 64) ? ~0ull : ((1ull << (level + 1)) - 1));
    j.modd = c->d_modd;
    return j;
}
static bool scale_eq(double a, double b) { return fabs(a / b - 1.0) <= 0x1p-30; }

static int binary_ct(hisa_ctx* c, hisa_ct ha, hisa_ct hb, hisa_ct* out, ElemOp op) {
    CHECK_CTX(c);
    GET_CT(a, ha);
    GET_CT(b, hb);
    if (a->level != b->level) return fail(HISA_E_LEVEL_MISMATCH, "levels %d vs %d", a->level, b->level);
    if (!scale_eq(a->scale, b->scale)) return fail(HISA_E_SCALE_MISMATCH, "scales %.17g vs %.17g", a->scale, b->scale);
    if (a->npolys != b->npolys) return fail(HISA_E_NOT_RELINEARIZED, "poly counts %d vs %d", a->npolys, b->npolys);
    uint64_t* o = dalloc_t<uint64_t>(c, obj_words(c, a));
    if (!o) return fail(HISA_E_OOM, "add/sub");
    ElemJob j = ejob(c, a->npolys, a->level);
    j.a[0] = a->ptr; j.b[0] = b->ptr; j.out[0] = o;
    KL("elementwise", launch_elem(op, j, c->d_mods, 1, c->stream));
    return emit_ct(c, out, ha, o, a->level, a->npolys, a->scale);
}
extern "C" int hisa_add(hisa_ctx* c, hisa_ct a, hisa_ct b, hisa_ct* out) { return binary_ct(c, a, b, out, EL_ADD); }
extern "C" int hisa_sub(hisa_ctx* c, hisa_ct a, hisa_ct b, hisa_ct* out) { return binary_ct(c, a, b, out, EL_SUB); }

static int plain_op(hisa_ctx* c, hisa_ct ha, hisa_pt hp, hisa_ct* out, ElemOp op) {
    CHECK_CTX(c);
    GET_CT(a, ha);
    GET_PT(p, hp);
    if (a->npolys != 2) return fail(HISA_E_NOT_RELINEARIZED, "3-poly ciphertext");
    if (a->level != p->level) return fail(HISA_E_LEVEL_MISMATCH, "levels %d vs %d", a->level, p->level);
    double scale = a->scale;
    if (op == EL_MUL_PLAIN) scale = a->scale * p->scale;
    else if (!scale_eq(a->scale, p->scale)) return fail(HISA_E_SCALE_MISMATCH, "scales %.17g vs %.17g", a->scale, p->scale);
    uint64_t* o = dalloc_t<uint64_t>(c, obj_words(c, a));
    if (!o) return fail(HISA_E_OOM, "plain op");
    ElemJob j = ejob(c, 2, a->level);
    j.a[0] = a->ptr; j.b[0] = p->ptr; j.out[0] = o;
    KL("elementwise", launch_elem(op, j, c->d_mods, 1, c->stream));
    return emit_ct(c, out, ha, o, a->level, 2, scale);
}
extern "C" int hisa_add_plain(hisa_ctx* c, hisa_ct a, hisa_pt p, hisa_ct* out) { return plain_op(c, a, p, out, EL_ADD_PLAIN); }
extern "C" int hisa_sub_plain(hisa_ctx* c, hisa_ct a, hisa_pt p, hisa_ct* out) { return plain_op(c, a, p, out, EL_SUB_PLAIN); }
extern "C" int hisa_mul_plain(hisa_ctx* c, hisa_ct a, hisa_pt p, hisa_ct* out) { return plain_op(c, a, p, out, EL_MUL_PLAIN); }

// n independent mulPlains (same level) in one launch per MAXB pairs: outs[i] = a[i] (x) p[i]
extern "C" int hisa_mul_plain_batch(hisa_ctx* c, const hisa_ct* a, const hisa_pt* p, size_t n, hisa_ct* outs) {
    CHECK_CTX(c);
    if ((!a || !p || !outs) && n) return fail(HISA_E_PARAMS, "null argument");
    if (n == 0) return HISA_OK;
    std::vector<Obj*> oa(n), op(n);
    for (size_t i = 0; i < n; i++) {
        oa[i] = get_obj(c, a[i], OBJ_CT);
        op[i] = get_obj(c, p[i], OBJ_PT);
        if (!oa[i] || !op[i]) return fail(HISA_E_INVALID_HANDLE, "invalid handle at %zu", i);
        if (oa[i]->npolys != 2) return fail(HISA_E_NOT_RELINEARIZED, "3-poly ciphertext at %zu", i);
        if (oa[i]->level != op[i]->level || oa[i]->level != oa[0]->level)
            return fail(HISA_E_LEVEL_MISMATCH, "levels differ at %zu", i);
    }
    const int level = oa[0]->level;
    DGuard outputs(c);
    std::vector<uint64_t*> res(n);
    for (size_t i = 0; i < n; i++) {
        res[i] = outputs.add(dalloc_t<uint64_t>(c, obj_words(c, oa[i])));
        if (!res[i]) return fail(HISA_E_OOM, "mul_plain batch");
    }
    for (size_t i0 = 0; i0 < n; i0 += MAXB) {
        const int nz = (int)std::min<size_t>(MAXB, n - i0);
        ElemJob j = ejob(c, 2, level);
        for (int z = 0; z < nz; z++) {
            j.a[z] = oa[i0 + z]->ptr;
            j.b[z] = op[i0 + z]->ptr;
            j.out[z] = res[i0 + z];
        }
        KL("elementwise", launch_elem(EL_MUL_PLAIN, j, c->d_mods, nz, c->stream));
    }
    outputs.keep();
    for (size_t i = 0; i < n; i++) outs[i] = new_handle(c, OBJ_CT, res[i], level, 2, oa[i]->scale * op[i]->scale);
    return HISA_OK;
}

// A20: X = llround(x * s), |X| < 2^62, residues X mod q_i
static int scalar_residues(hisa_ctx* c, double x, double s, int l1, ElemJob& j) {
    const double v = x * s;
    if (!std::isfinite(v) || fabs(v) >= 0x1p62) return fail(HISA_E_PARAMS, "scalar out of range");
    const long long X = llround(v);
    for (int i = 0; i < l1; i++) {
        const uint64_t q = c->mod[i];
        const __int128 r = ((__int128)X % (__int128)q + q) % q;
        j.scal[i] = (uint64_t)r;
        j.scalp[i] = shoup((uint64_t)r, q);
    }
    return HISA_OK;
}
static int scalar_op(hisa_ctx* c, hisa_ct ha, double x, double pt_scale, hisa_ct* out, ElemOp op, int sign) {
    CHECK_CTX(c);
    GET_CT(a, ha);
    if (a->npolys != 2) return fail(HISA_E_NOT_RELINEARIZED, "3-poly ciphertext");
    ElemJob j = ejob(c, 2, a->level);
    double s = a->scale, out_scale = a->scale;
    if (op == EL_MUL_SCALAR) {
        s = pt_scale == 0.0 ? (double)c->mod[a->level] : pt_scale;
        out_scale = a->scale * s;
    }
    RET(scalar_residues(c, sign * x, s, a->level + 1, j));
    uint64_t* o = dalloc_t<uint64_t>(c, obj_words(c, a));
    if (!o) return fail(HISA_E_OOM, "scalar op");
    j.a[0] = a->ptr; j.out[0] = o;
    KL("elementwise", launch_elem(op, j, c->d_mods, 1, c->stream));
    return emit_ct(c, out, ha, o, a->level, 2, out_scale);
}
extern "C" int hisa_add_scalar(hisa_ctx* c, hisa_ct a, double x, hisa_ct* out) { return scalar_op(c, a, x, 0, out, EL_ADD_SCALAR, 1); }
extern "C" int hisa_sub_scalar(hisa_ctx* c, hisa_ct a, double x, hisa_ct* out) { return scalar_op(c, a, x, 0, out, EL_ADD_SCALAR, -1); }
extern "C" int hisa_mul_scalar(hisa_ctx* c, hisa_ct a, double x, double ps, hisa_ct* out) {
    return scalar_op(c, a, x, ps, out, EL_MUL_SCALAR, 1);
}

extern "C" int hisa_mul_norelin(hisa_ctx* c, hisa_ct ha, hisa_ct hb, hisa_ct* out) {
    CHECK_CTX(c);
    GET_CT(a, ha);
    GET_CT(b, hb);
    if (a->npolys != 2 || b->npolys != 2) return fail(HISA_E_NOT_RELINEARIZED, "3-poly operand");
    if (a->level != b->level) return fail(HISA_E_LEVEL_MISMATCH, "levels %d vs %d", a->level, b->level);
    const int l1 = a->level + 1;
    uint64_t* o = dalloc_t<uint64_t>(c, (size_t)3 * l1 * c->N);
    if (!o) return fail(HISA_E_OOM, "tensor");
    ElemJob j = ejob(c, 2, a->level);
    j.a[0] = a->ptr; j.b[0] = b->ptr; j.out[0] = o;
    KL("elementwise", launch_elem(ha == hb ? EL_SQUARE_TENSOR : EL_TENSOR, j, c->d_mods, 1, c->stream));
    return emit_ct(c, out, ha, o, a->level, 3, a->scale * b->scale);
}

// ============================================================================================
// key switching (a5): INTT -> ModUp pass 1 (lift) -> fused pass 2 + key inner product ->
// INTT_p -> ModDown pass 1 (lift) -> pass 2 with combine epilogue (+ addend)
// ============================================================================================
struct KsBatch {
    const uint64_t* d[MAXB];      // poly to switch, NTT form, (l+1) limbs
    uint64_t* out[MAXB];          // output ct [2][l+1][N]
    const uint64_t* add[MAXB];    // addend base (poly-stride add_a) or null
    int add_polys;                // how many output polys receive the addend (1: rotation, 2: relin)
    long long add_a;
};
// (1) INTT of the digits, (2) ModUp pass 1: lift q_j -> r (r != q_j) on load + first log M1
// forward stages; T1[z] = [j][ri][N] (ri over q_0..q_l, p; diagonal blocks untouched)
static int ks_modup_pass1(hisa_ctx* c, int nz, int level, const uint64_t* const* d, uint64_t* const* dtil,
                          uint64_t* const* t1) {
    const int l1 = level + 1, l2 = level + 2, L = c->L;
    const long long N = (long long)c->N;
    uint8_t mm[MAXL];
    ident_map(mm, l1);
    RET(ntt_inv(c, d, dtil, nz, l1, mm));
    PassJob j = job0();
    for (int z = 0; z < nz; z++) { j.src[z] = dtil[z]; j.dst[z] = t1[z]; }
    j.nb = l2;
    j.src_a = N; j.src_b = 0;
    j.dst_a = (long long)l2 * N; j.dst_b = N;
    j.skip_diag = 1;
    for (int ri = 0; ri < l2; ri++) j.mod_map[ri] = (uint8_t)(ri < l1 ? ri : L);
    for (int a = 0; a < l1; a++) j.smod_map[a] = (uint8_t)a;
    Tables tb = c->tables();
    KL("ks_modup_cols", launch_fwd_pass1(j, tb, l1 * l2, nz, true, c->stream));
    return HISA_OK;
}
// (4) INTT_p of acc_p, (5) lift p -> q_i + first stages, (6) last stages with the combine
// epilogue out_i = (acc_i - NTT_i(y)) p^-1 (+ addend).  ptmp[z]: 2 limbs, md[z]: 2 l1 limbs.
static int ks_moddown(hisa_ctx* c, int nz, int level, uint64_t* const* acc, uint64_t* const* ptmp,
                      uint64_t* const* md, const KsBatch& kb) {
    const int l1 = level + 1, l2 = level + 2, L = c->L;
    const long long N = (long long)c->N;
    Tables tb = c->tables();
    {
        PassJob j = job0();
        for (int z = 0; z < nz; z++) { j.src[z] = acc[z] + (long long)l1 * N; j.dst[z] = ptmp[z]; }
        j.nb = 1;
        j.src_a = (long long)l2 * N; j.dst_a = N;
        j.mod_map[0] = (uint8_t)L;
        KL("ks_intt_p_rows", launch_inv_passA(j, tb, 2, nz, c->stream));
        for (int z = 0; z < nz; z++) { j.src[z] = ptmp[z]; }
        j.src_a = N;
        KL("ks_intt_p_cols", launch_inv_passB(j, tb, 2, nz, c->stream));
    }
    {
        PassJob j = job0();
        for (int z = 0; z < nz; z++) { j.src[z] = ptmp[z]; j.dst[z] = md[z]; }
        j.nb = l1;
        j.src_a = N; j.src_b = 0;
        j.dst_a = (long long)l1 * N; j.dst_b = N;
        ident_map(j.mod_map, l1);
        j.smod_map[0] = j.smod_map[1] = (uint8_t)L;
        KL("ks_moddown_cols", launch_fwd_pass1(j, tb, 2 * l1, nz, true, c->stream));
    }
    {
        PassJob j = job0();
        for (int z = 0; z < nz; z++) {
            j.src[z] = md[z];
            j.dst[z] = kb.out[z];
            j.aux[z] = acc[z];
            j.add[z] = kb.add[z];
        }
        j.nb = l1;
        j.src_a = (long long)l1 * N; j.src_b = N;
        j.dst_a = (long long)l1 * N; j.dst_b = N;
        j.aux_a = (long long)l2 * N; j.aux_b = N;
        j.add_a = kb.add_a; j.add_b = N;
        j.aux_limit = kb.add_polys;
        ident_map(j.mod_map, l1);
        Tables tc = c->tables(c->d_pinv);
        KL("ks_moddown_rows", launch_fwd_pass2(j, tc, 2 * l1, nz, true, c->stream));
    }
    return HISA_OK;
}

// ciphertexts per batched key-switch launch: up to MAXB, but the scratch of a batch (dtil, T1,
// acc, ModDown temporaries: (l+1)(l+2) + 3(l+1) + 2(l+2) + 2 limbs per ciphertext, ~390 MiB at
// N = 2^16, L = 24) is kept under ~4 GiB so large contexts with many resident keys batch less
static int ks_chunk(const hisa_ctx* c, int level) {
    const size_t l1 = (size_t)level + 1, l2 = l1 + 1;
    const size_t per = (size_t)c->N * 8 * (l1 + l1 * l2 + 2 * l2 + 2 + 2 * l1 + 2 * l1);
    const size_t budget = (size_t)4 << 30;
    size_t n = budget / per;
    if (n < 1) n = 1;
    if (n > (size_t)MAXB) n = MAXB;
    // K4 shares every staged key row among 8 / 4 / 2 ciphertexts of a batch by the largest of those
    // dividing it: a chunk of 10 (what 4 GiB gives at N = 2^16, L = 24) would run the 2-ciphertext
    // form -- 3.0k instead of 3.2k rotations/s in the config-2 sweep at B >= 16
    if (n >= 8) n -= n % 8;
    else if (n >= 4) n = 4;
    else if (n >= 2) n = 2;
    return (int)n;
}
// n items in chunks of at most `maxc`: as many chunks as that needs, of equal size rounded up to
// the sharing quantum q (8 ciphertexts per staged key row in K4, 4 in K7) -- 16 items under a cap of
// 12 run as 8 + 8, not 12 + 4
static int balanced_chunk(size_t n, size_t maxc, size_t q) {
    if (n <= maxc || maxc < q) return (int)std::min(n, maxc);
    const size_t nch = (n + maxc - 1) / maxc;
    size_t per = (n + nch - 1) / nch;
    per = (per + q - 1) / q * q;
    return (int)std::min(per, maxc);
}

static int ensure_side(hisa_ctx* c) {
    if (c->side) return HISA_OK;
    CK(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
    for (cudaEvent_t* e : {&c->ev_fork, &c->ev_join, &c->ev_k7[0], &c->ev_k7[1], &c->ev_md[0], &c->ev_md[1]})
        CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    return HISA_OK;
}

// key switch of nz digits under ONE key: ModUp pass 1 -> fused pass 2 + key inner product (K4,
// D never stored in NTT form) -> ModDown
static int keyswitch(hisa_ctx* c, int nz, int level, const uint64_t* key, int kL, const KsBatch& kb) {
    const int l1 = level + 1, l2 = level + 2, L = c->L;
    const long long N = (long long)c->N;
    // scratch per ciphertext: dtil l1, T1 l1*l2, acc 2*l2, ptmp 2, md 2*l1
    const size_t per = (size_t)N * ((size_t)l1 + (size_t)l1 * l2 + 2 * l2 + 2 + 2 * l1);
    DGuard guard(c);
    uint64_t* scratch = guard.add(dalloc_t<uint64_t>(c, per * nz));
    if (!scratch) return fail(HISA_E_OOM, "key-switch scratch (%zu MiB)", per * nz * 8 >> 20);
    uint64_t *dtil[MAXB], *t1[MAXB], *acc[MAXB], *ptmp[MAXB], *md[MAXB];
    for (int z = 0; z < nz; z++) {
        uint64_t* s = scratch + per * z;
        dtil[z] = s; s += (size_t)l1 * N;
        t1[z] = s; s += (size_t)l1 * l2 * N;
        acc[z] = s; s += (size_t)2 * l2 * N;
        ptmp[z] = s; s += (size_t)2 * N;
        md[z] = s;
    }
    RET(ks_modup_pass1(c, nz, level, kb.d, dtil, t1));
    {
        KsJob kj;
        memset(&kj, 0, sizeof kj);
        for (int z = 0; z < nz; z++) { kj.t1[z] = t1[z]; kj.d[z] = kb.d[z]; kj.acc[z] = acc[z]; }
        kj.key = key;
        kj.l1 = l1;
        kj.L = kL;      // key stride; the special prime's key limb is kL (mod_map gives the table's L)
        kj.nz = nz;
        for (int ri = 0; ri < l2; ri++) {
            kj.mod_map[ri] = (uint8_t)(ri < l1 ? ri : L);
            if ((double)c->mod[kj.mod_map[ri]] < c->f64_max_q) kj.fp_rows |= 1ull << ri;
        }
        Tables tb = c->tables();
        RET(ensure_side(c));
        const SideStream side{c->side, c->ev_fork, c->ev_join};
        KL("ks_ip_rows", launch_ks_ip(kj, tb, nz, c->stream, &side));
    }
    RET(ks_moddown(c, nz, level, acc, ptmp, md, kb));
    return HISA_OK;   // guard frees the scratch
}

extern "C" int hisa_relinearize(hisa_ctx* c, hisa_ct h) {
    CHECK_CTX(c);
    GET_CT(o, h);
    if (o->npolys == 2) return HISA_OK;
    if (!c->d_rlk) return fail(HISA_E_NO_KEY, "relinearisation key not generated");
    const int l1 = o->level + 1;
    const long long N = (long long)c->N;
    uint64_t* out = dalloc_t<uint64_t>(c, (size_t)2 * l1 * N);
    if (!out) return fail(HISA_E_OOM, "relin");
    KsBatch kb;
    memset(&kb, 0, sizeof kb);
    kb.d[0] = o->ptr + 2 * l1 * N;
    kb.out[0] = out;
    kb.add[0] = o->ptr;
    kb.add_polys = 2;
    kb.add_a = (long long)l1 * N;
    RET(keyswitch(c, 1, o->level, c->d_rlk, c->L, kb));
    dfree(c, o->ptr);
    o->ptr = out;
    o->npolys = 2;
    return HISA_OK;
}

extern "C" int hisa_mul(hisa_ctx* c, hisa_ct a, hisa_ct b, hisa_ct* out) {
    hisa_ct t;
    RET(hisa_mul_norelin(c, a, b, &t));
    int r = hisa_relinearize(c, t);
    if (r != HISA_OK) { hisa_free(c, t); return r; }
    Obj* ot = get_obj(c, t, OBJ_CT);
    if (out) { *out = t; return HISA_OK; }
    // in place on a
    Obj* oa = get_obj(c, a, OBJ_CT);
    dfree(c, oa->ptr);
    oa->ptr = ot->ptr; oa->level = ot->level; oa->npolys = ot->npolys; oa->scale = ot->scale;
    ot->ptr = nullptr;
    hisa_free(c, t);
    return HISA_OK;
}

// tensor + relinearisation of n pairs (one level), batched launches: the ct x ct product of the
// activation square over all channels of a layer
extern "C" int hisa_mul_batch(hisa_ctx* c, const hisa_ct* a, const hisa_ct* b, size_t n, hisa_ct* outs) {
    CHECK_CTX(c);
    if ((!a || !b || !outs) && n) return fail(HISA_E_PARAMS, "null argument");
    if (n && !c->d_rlk) return fail(HISA_E_NO_KEY, "relinearisation key not generated");
    std::vector<Obj*> oa(n), ob(n);
    for (size_t i = 0; i < n; i++) {
        oa[i] = get_obj(c, a[i], OBJ_CT);
        ob[i] = get_obj(c, b[i], OBJ_CT);
        if (!oa[i] || !ob[i]) return fail(HISA_E_INVALID_HANDLE, "invalid ciphertext handle at %zu", i);
        if (oa[i]->npolys != 2 || ob[i]->npolys != 2) return fail(HISA_E_NOT_RELINEARIZED, "3-poly operand");
        if (oa[i]->level != ob[i]->level || oa[i]->level != oa[0]->level)
            return fail(HISA_E_LEVEL_MISMATCH, "levels differ at %zu", i);
    }
    if (n == 0) return HISA_OK;
    const int level = oa[0]->level, l1 = level + 1;
    const long long N = (long long)c->N;
    const size_t chunk = (size_t)balanced_chunk(n, (size_t)ks_chunk(c, level), 8);
    for (size_t i0 = 0; i0 < n; i0 += chunk) {
        const int nz = (int)std::min(chunk, n - i0);
        uint64_t* t3 = dalloc_t<uint64_t>(c, (size_t)3 * l1 * N * nz);
        if (!t3) return fail(HISA_E_OOM, "mul batch");
        ElemJob ej = ejob(c, 2, level);
        bool square = true;
        for (int z = 0; z < nz; z++) {
            ej.a[z] = oa[i0 + z]->ptr;
            ej.b[z] = ob[i0 + z]->ptr;
            ej.out[z] = t3 + (size_t)3 * l1 * N * z;
            square = square && (a[i0 + z] == b[i0 + z]);
        }
        KL("elementwise", launch_elem(square ? EL_SQUARE_TENSOR : EL_TENSOR, ej, c->d_mods, nz, c->stream));
        KsBatch kb;
        memset(&kb, 0, sizeof kb);
        uint64_t* res[MAXB];
        for (int z = 0; z < nz; z++) {
            res[z] = dalloc_t<uint64_t>(c, (size_t)2 * l1 * N);
            if (!res[z]) return fail(HISA_E_OOM, "mul batch");
            kb.d[z] = ej.out[z] + 2 * l1 * N;
            kb.out[z] = res[z];
            kb.add[z] = ej.out[z];
        }
        kb.add_polys = 2;
        kb.add_a = (long long)l1 * N;
        RET(keyswitch(c, nz, level, c->d_rlk, c->L, kb));
        dfree(c, t3);
        for (int z = 0; z < nz; z++)
            outs[i0 + z] = new_handle(c, OBJ_CT, res[z], level, 2, oa[i0 + z]->scale * ob[i0 + z]->scale);
    }
    return HISA_OK;
}

// Rotation (A15) with pre-permuted keys.  Stored rotation keys are key'_k = psi_g^-1(key_k)
// (permuted once at keygen; hisa_key_export returns the canonical key).  Because psi_g is a ring
// automorphism that commutes with the centred lifts of ModUp / ModDown (a signed coefficient
// permutation), KS_k(psi_g(c1)) = psi_g(KS'_k(c1)), so
//     rotLeft(c, k) = psi_g( (c0 + KS'_k(c1)_0, KS'_k(c1)_1) )
// -- bit-identical to "automorphism, then key switch" (A14, A37), with the ModUp of c1 shared
// by every amount (hoisting) and the permutation applied once to the output.
static int normalize_rot(const hisa_ctx* c, int64_t k, uint64_t* out) {
    const int64_t s = (int64_t)(c->N / 2);
    int64_t kk = k % s;
    if (kk < 0) kk += s;
    *out = (uint64_t)kk;
    return HISA_OK;
}
static uint64_t galois(const hisa_ctx* c, uint64_t k) { return h_pow(5, k, 2 * c->N); }
// a rotation key for amount k that serves `level` (keys are truncated to their max level)
static int rot_key_check(hisa_ctx* c, uint64_t k, int level) {
    auto it = c->rot_keys.find(k);
    if (it == c->rot_keys.end()) return fail(HISA_E_NO_KEY, "no rotation key for %llu", (unsigned long long)k);
    if (level >= it->second.kL)
        return fail(HISA_E_NO_KEY, "rotation key for %llu generated up to level %d, ciphertext at level %d",
                    (unsigned long long)k, it->second.kL - 1, level);
    return HISA_OK;
}

// rotation of nz ciphertexts (same level, same amount, own key switch each): batched K4 path
static int rotate_batch(hisa_ctx* c, Obj* const* in, int nz, uint64_t k, uint64_t** outs, bool add_input = false) {
    const int level = in[0]->level, l1 = level + 1;
    const long long N = (long long)c->N;
    RET(rot_key_check(c, k, level));
    const hisa_ctx::KeyRec& key = c->rot_keys[k];
    DGuard scratch(c), outputs(c);
    uint64_t* pre = scratch.add(dalloc_t<uint64_t>(c, (size_t)2 * l1 * N * nz));
    if (!pre) return fail(HISA_E_OOM, "rotation scratch");
    const uint64_t* pres[MAXB];
    uint64_t gs[MAXB];
    KsBatch kb;
    memset(&kb, 0, sizeof kb);
    for (int z = 0; z < nz; z++) {
        outs[z] = outputs.add(dalloc_t<uint64_t>(c, (size_t)2 * l1 * N));
        if (!outs[z]) return fail(HISA_E_OOM, "rotation output");
        kb.d[z] = in[z]->ptr + l1 * N;
        kb.out[z] = pre + (size_t)2 * l1 * N * z;
        kb.add[z] = in[z]->ptr;
        pres[z] = kb.out[z];
        gs[z] = galois(c, k);
    }
    kb.add_polys = 1;
    kb.add_a = 0;
    RET(keyswitch(c, nz, level, key.p, key.kL, kb));
    if (add_input) {   // rotate-and-sum step: out = in + rot(in), the add fused into the permutation
        const uint64_t* adds[MAXB];
        for (int z = 0; z < nz; z++) adds[z] = in[z]->ptr;
        KL("automorphism", launch_automorphism_add(pres, outs, adds, nz, 2 * l1, l1, c->log_n, gs, c->d_mods,
                                                   c->stream));
    } else {
        KL("automorphism", launch_automorphism(pres, outs, nz, 2 * l1, c->log_n, gs, c->stream));
    }
    outputs.keep();
    return HISA_OK;
}

// hoisted rotations of nct ciphertexts (one level) by the same n non-zero amounts: batched ModUp
// (nz ciphertexts per launch), K7 over groups of <= 4 ciphertexts x <= 4 keys (each key word
// streamed once per group), batched ModDown and permutation.  outs[i * n + r] = rot(in_i, ks[r]).
// Pipeline: K7 (HBM-bound: the key stream) of key group g + 1 runs on the side stream while the
// ModDown + permutation (FP64-bound) of group g runs on the main stream, through two accumulator
// buffers -- the step costs about max(key stream, ModDown) per group instead of their sum.
static int rotate_hoisted_multi(hisa_ctx* c, Obj* const* os, int nct, const uint64_t* ks, int n, uint64_t** outs) {
    const int level = os[0]->level, l1 = level + 1, l2 = level + 2, L = c->L;
    const long long N = (long long)c->N;
    const size_t per_ct = (size_t)N * ((size_t)l1 + (size_t)l1 * l2);           // dtil, D
    const size_t per_out = (size_t)N * (2 * l2 + 2 + 2 * l1 + 2 * l1);           // acc, ptmp, md, pre
    constexpr int RK = 4;                                                         // keys per K7 launch
    // 8 GiB of scratch: 8 ciphertexts per chunk at N = 2^16, L = 24 (ModUp batched over 8, K7 in two
    // groups of 4); a smaller arena falls back to smaller chunks below
    const size_t budget = (size_t)8 << 30;
    int ct_chunk = (int)std::max<size_t>(1, std::min<size_t>((size_t)MAXB, budget / ((per_ct + 2 * RK * per_out) * 8)));
    if (ct_chunk >= 4) ct_chunk -= ct_chunk % 4;   // K7 streams each key once per group of 4 ciphertexts
    ct_chunk = balanced_chunk((size_t)nct, (size_t)ct_chunk, 4);
    DGuard outputs(c), sguard(c);
    for (int i = 0; i < nct * n; i++) {
        outs[i] = outputs.add(dalloc_t<uint64_t>(c, (size_t)2 * l1 * N));
        if (!outs[i]) return fail(HISA_E_OOM, "rotation output");
    }
    uint64_t* scratch = nullptr;
    for (;;) {
        scratch = dalloc_t<uint64_t>(c, per_ct * ct_chunk + 2 * per_out * (size_t)ct_chunk * RK);
        if (scratch || ct_chunk == 1) break;
        ct_chunk = std::max(1, ct_chunk / 2);
    }
    sguard.add(scratch);
    if (!scratch) return fail(HISA_E_OOM, "hoisted rotation scratch");
    RET(ensure_side(c));
#ifndef HOIST_PIPE
#define HOIST_PIPE 1   // 0: K7 on the main stream (side builds for A/B timing only)
#endif
    cudaStream_t k7s = HOIST_PIPE ? c->side : c->stream;
    const int ngroups = (n + RK - 1) / RK;
    for (int c0 = 0; c0 < nct; c0 += ct_chunk) {
        const int nc = std::min(ct_chunk, nct - c0);
        uint64_t *dtil[MAXB], *D[MAXB];
        const uint64_t* d1[MAXB];
        for (int z = 0; z < nc; z++) {
            dtil[z] = scratch + per_ct * z;
            D[z] = dtil[z] + (size_t)l1 * N;
            d1[z] = os[c0 + z]->ptr + l1 * N;
        }
        RET(ks_modup_pass1(c, nc, level, d1, dtil, D));
        {   // ModUp pass 2 in place: D_{j,r} for r != q_j, fully reduced
            PassJob j = job0();
            for (int z = 0; z < nc; z++) { j.src[z] = D[z]; j.dst[z] = D[z]; }
            j.nb = l2;
            j.src_a = j.dst_a = (long long)l2 * N;
            j.src_b = j.dst_b = N;
            j.skip_diag = 1;
            for (int ri = 0; ri < l2; ri++) j.mod_map[ri] = (uint8_t)(ri < l1 ? ri : L);
            Tables tb = c->tables();
            KL("ks_modup_rows", launch_fwd_pass2(j, tb, l1 * l2, nc, false, c->stream));
        }
        // side stream: starts after the ModUp; main stream: after the last ModDown, the scratch
        // (D, accumulators) of this chunk may be reused by the next
        CK(cudaEventRecord(c->ev_fork, c->stream));
        CK(cudaStreamWaitEvent(k7s, c->ev_fork, 0));
        auto outbase = [&](int buf) { return scratch + per_ct * ct_chunk + (size_t)buf * per_out * ct_chunk * RK; };
        auto k7 = [&](int gi) -> int {   // K7 of key group gi into buffer gi % 2, on the side stream
            const int r0 = gi * RK, R = std::min(RK, n - r0), buf = gi & 1;
            if (gi >= 2) CK(cudaStreamWaitEvent(k7s, c->ev_md[buf], 0));   // ModDown of gi - 2 read it
            for (int g0 = 0; g0 < nc; g0 += MAXCG) {
                KsHoistMultiJob hj;
                memset(&hj, 0, sizeof hj);
                hj.cg = std::min(MAXCG, nc - g0);
                for (int cg = 0; cg < hj.cg; cg++) {
                    hj.D[cg] = D[g0 + cg];
                    hj.diag[cg] = d1[g0 + cg];
                    for (int r = 0; r < R; r++) hj.acc[cg][r] = outbase(buf) + per_out * (size_t)((g0 + cg) * R + r);
                }
                for (int r = 0; r < R; r++) {
                    hj.key[r] = c->rot_keys[ks[r0 + r]].p;
                    hj.kL[r] = c->rot_keys[ks[r0 + r]].kL;
                }
                hj.l1 = l1;
                hj.L = L;
                for (int ri = 0; ri < l2; ri++) hj.mod_map[ri] = (uint8_t)(ri < l1 ? ri : L);
                KLS("ks_ip_hoisted", k7s, launch_ks_ip_hoisted_multi(hj, R, c->tables(), k7s));
            }
            CK(cudaEventRecord(c->ev_k7[buf], k7s));
            return HISA_OK;
        };
        RET(k7(0));
        for (int gi = 0; gi < ngroups; gi++) {
            if (gi + 1 < ngroups) RET(k7(gi + 1));
            const int r0 = gi * RK, R = std::min(RK, n - r0), buf = gi & 1;
            CK(cudaStreamWaitEvent(c->stream, c->ev_k7[buf], 0));
            const int nout = nc * R;
            for (int o0 = 0; o0 < nout; o0 += MAXB) {
                const int m = std::min(MAXB, nout - o0);
                uint64_t *acc[MAXB], *ptmp[MAXB], *md[MAXB];
                const uint64_t* pres[MAXB];
                uint64_t gs[MAXB];
                KsBatch kb;
                memset(&kb, 0, sizeof kb);
                for (int q = 0; q < m; q++) {
                    const int o = o0 + q, z = o / R, r = o % R;
                    uint64_t* sp = outbase(buf) + per_out * (size_t)(z * R + r);
                    acc[q] = sp; sp += (size_t)2 * l2 * N;
                    ptmp[q] = sp; sp += (size_t)2 * N;
                    md[q] = sp; sp += (size_t)2 * l1 * N;
                    pres[q] = sp;
                    kb.out[q] = sp;
                    kb.add[q] = os[c0 + z]->ptr;
                    gs[q] = galois(c, ks[r0 + r]);
                }
                kb.add_polys = 1;
                kb.add_a = 0;
                RET(ks_moddown(c, m, level, acc, ptmp, md, kb));
                uint64_t* dsts[MAXB];
                for (int q = 0; q < m; q++) {
                    const int o = o0 + q, z = o / R, r = o % R;
                    dsts[q] = outs[(size_t)(c0 + z) * n + r0 + r];
                }
                KL("automorphism", launch_automorphism(pres, dsts, m, 2 * l1, c->log_n, gs, c->stream));
            }
            CK(cudaEventRecord(c->ev_md[buf], c->stream));
        }
    }
    outputs.keep();
    return HISA_OK;
}

extern "C" int hisa_rot_left_hoisted_batch(hisa_ctx* c, const hisa_ct* in, size_t nct, const int64_t* k, size_t n,
                                           hisa_ct* outs) {
    CHECK_CTX(c);
    if ((!in || !k || !outs) && nct && n) return fail(HISA_E_PARAMS, "null argument");
    if (nct == 0 || n == 0) return HISA_OK;
    std::vector<Obj*> objs(nct);
    for (size_t i = 0; i < nct; i++) {
        objs[i] = get_obj(c, in[i], OBJ_CT);
        if (!objs[i]) return fail(HISA_E_INVALID_HANDLE, "invalid ciphertext handle at %zu", i);
        if (objs[i]->npolys != 2) return fail(HISA_E_NOT_RELINEARIZED, "3-poly ciphertext at %zu", i);
        if (objs[i]->level != objs[0]->level) return fail(HISA_E_LEVEL_MISMATCH, "batch levels differ");
    }
    std::vector<uint64_t> kk(n), amounts;
    std::vector<size_t> nz_idx;
    for (size_t r = 0; r < n; r++) {
        normalize_rot(c, k[r], &kk[r]);
        if (kk[r]) RET(rot_key_check(c, kk[r], objs[0]->level));
        if (kk[r]) { nz_idx.push_back(r); amounts.push_back(kk[r]); }
    }
    for (size_t i = 0; i < nct; i++)
        for (size_t r = 0; r < n; r++)
            if (!kk[r]) RET(hisa_copy(c, in[i], &outs[i * n + r]));
    if (amounts.empty()) return HISA_OK;
    const int na = (int)amounts.size();
    std::vector<uint64_t*> res((size_t)nct * na);
    RET(rotate_hoisted_multi(c, objs.data(), (int)nct, amounts.data(), na, res.data()));
    for (size_t i = 0; i < nct; i++)
        for (int a = 0; a < na; a++)
            outs[i * n + nz_idx[a]] = new_handle(c, OBJ_CT, res[i * na + a], objs[i]->level, 2, objs[i]->scale);
    return HISA_OK;
}

static int rot_common(hisa_ctx* c, hisa_ct h, int64_t k, hisa_ct* out) {
    CHECK_CTX(c);
    GET_CT(o, h);
    if (o->npolys != 2) return fail(HISA_E_NOT_RELINEARIZED, "3-poly ciphertext");
    uint64_t kk;
    normalize_rot(c, k, &kk);
    if (kk == 0) {
        if (!out) return HISA_OK;
        return hisa_copy(c, h, out);
    }
    RET(rot_key_check(c, kk, o->level));
    uint64_t* res[1];
    Obj* ins[1] = {o};
    RET(rotate_batch(c, ins, 1, kk, res));
    return emit_ct(c, out, h, res[0], o->level, 2, o->scale);
}
extern "C" int hisa_rot_left(hisa_ctx* c, hisa_ct h, int64_t k, hisa_ct* out) { return rot_common(c, h, k, out); }
extern "C" int hisa_rot_right(hisa_ctx* c, hisa_ct h, int64_t k, hisa_ct* out) {
    if (!c) return fail(HISA_E_PARAMS, "null context");
    const int64_t s = (int64_t)(c->N / 2);
    int64_t kk = k % s;
    if (kk < 0) kk += s;
    return rot_common(c, h, (s - kk) % s, out);   // right rotations become left rotations
}

extern "C" int hisa_rot_left_batch(hisa_ctx* c, const hisa_ct* in, size_t n, int64_t k, hisa_ct* outs) {
    CHECK_CTX(c);
    if (!in || !outs) return fail(HISA_E_PARAMS, "null argument");
    if (n == 0) return HISA_OK;
    std::vector<Obj*> objs(n);
    for (size_t i = 0; i < n; i++) {
        objs[i] = get_obj(c, in[i], OBJ_CT);
        if (!objs[i]) return fail(HISA_E_INVALID_HANDLE, "invalid ciphertext handle at %zu", i);
        if (objs[i]->npolys != 2) return fail(HISA_E_NOT_RELINEARIZED, "3-poly ciphertext at %zu", i);
        if (objs[i]->level != objs[0]->level) return fail(HISA_E_LEVEL_MISMATCH, "batch levels differ");
    }
    uint64_t kk;
    normalize_rot(c, k, &kk);
    if (kk == 0) {
        for (size_t i = 0; i < n; i++) RET(hisa_copy(c, in[i], &outs[i]));
        return HISA_OK;
    }
    RET(rot_key_check(c, kk, objs[0]->level));
    const size_t chunk = (size_t)balanced_chunk(n, (size_t)ks_chunk(c, objs[0]->level), 8);
    for (size_t i0 = 0; i0 < n; i0 += chunk) {
        const int nz = (int)std::min(chunk, n - i0);
        uint64_t* res[MAXB];
        RET(rotate_batch(c, objs.data() + i0, nz, kk, res));
        for (int z = 0; z < nz; z++)
            outs[i0 + z] = new_handle(c, OBJ_CT, res[z], objs[i0 + z]->level, 2, objs[i0 + z]->scale);
    }
    return HISA_OK;
}

extern "C" int hisa_rot_add_batch(hisa_ctx* c, const hisa_ct* in, size_t n, int64_t k, hisa_ct* outs) {
    CHECK_CTX(c);
    if ((!in || !outs) && n) return fail(HISA_E_PARAMS, "null argument");
    if (n == 0) return HISA_OK;
    std::vector<Obj*> objs(n);
    for (size_t i = 0; i < n; i++) {
        objs[i] = get_obj(c, in[i], OBJ_CT);
        if (!objs[i]) return fail(HISA_E_INVALID_HANDLE, "invalid ciphertext handle at %zu", i);
        if (objs[i]->npolys != 2) return fail(HISA_E_NOT_RELINEARIZED, "3-poly ciphertext at %zu", i);
        if (objs[i]->level != objs[0]->level) return fail(HISA_E_LEVEL_MISMATCH, "batch levels differ");
    }
    uint64_t kk;
    normalize_rot(c, k, &kk);
    if (kk == 0) {   // x + rot(x, 0) = 2x
        for (size_t i = 0; i < n; i++) RET(hisa_add(c, in[i], in[i], &outs[i]));
        return HISA_OK;
    }
    RET(rot_key_check(c, kk, objs[0]->level));
    const size_t chunk = (size_t)balanced_chunk(n, (size_t)ks_chunk(c, objs[0]->level), 8);
    for (size_t i0 = 0; i0 < n; i0 += chunk) {
        const int nz = (int)std::min(chunk, n - i0);
        uint64_t* res[MAXB];
        RET(rotate_batch(c, objs.data() + i0, nz, kk, res, true));
        for (int z = 0; z < nz; z++)
            outs[i0 + z] = new_handle(c, OBJ_CT, res[z], objs[i0 + z]->level, 2, objs[i0 + z]->scale);
    }
    return HISA_OK;
}

extern "C" int hisa_mul_plain_accumulate(hisa_ctx* c, const hisa_ct* in, size_t C, const hisa_pt* pts, size_t J,
                                         hisa_ct* outs) {
    CHECK_CTX(c);
    if (!in || !pts || !outs || C == 0 || J == 0) return fail(HISA_E_PARAMS, "bad arguments");
    std::vector<Obj*> ci(C), pi(C * J);
    for (size_t i = 0; i < C; i++) {
        ci[i] = get_obj(c, in[i], OBJ_CT);
        if (!ci[i]) return fail(HISA_E_INVALID_HANDLE, "invalid ciphertext handle at %zu", i);
        if (ci[i]->npolys != 2) return fail(HISA_E_NOT_RELINEARIZED, "3-poly input");
        if (ci[i]->level != ci[0]->level) return fail(HISA_E_LEVEL_MISMATCH, "input levels differ");
        if (!scale_eq(ci[i]->scale, ci[0]->scale)) return fail(HISA_E_SCALE_MISMATCH, "input scales differ");
    }
    for (size_t i = 0; i < C * J; i++) {
        pi[i] = get_obj(c, pts[i], OBJ_PT);
        if (!pi[i]) return fail(HISA_E_INVALID_HANDLE, "invalid plaintext handle at %zu", i);
        if (pi[i]->level != ci[0]->level) return fail(HISA_E_LEVEL_MISMATCH, "plaintext level at %zu", i);
        if (!scale_eq(pi[i]->scale, pi[0]->scale)) return fail(HISA_E_SCALE_MISMATCH, "plaintext scales differ");
    }
    const int level = ci[0]->level, l1 = level + 1;
    const long long N = (long long)c->N;
    std::vector<const uint64_t*> ip(C), pp(C * J);
    std::vector<uint64_t*> op(J);
    for (size_t i = 0; i < C; i++) ip[i] = ci[i]->ptr;
    for (size_t i = 0; i < C * J; i++) pp[i] = pi[i]->ptr;
    for (size_t j = 0; j < J; j++) {
        op[j] = dalloc_t<uint64_t>(c, (size_t)2 * l1 * N);
        if (!op[j]) return fail(HISA_E_OOM, "mul_plain_accumulate outputs");
    }
    void** dev = (void**)dalloc(c, (C + C * J + J) * sizeof(void*));
    if (!dev) return fail(HISA_E_OOM, "pointer arrays");
    std::vector<void*> host(C + C * J + J);
    for (size_t i = 0; i < C; i++) host[i] = (void*)ip[i];
    for (size_t i = 0; i < C * J; i++) host[C + i] = (void*)pp[i];
    for (size_t j = 0; j < J; j++) host[C + C * J + j] = op[j];
    CK(cudaMemcpyAsync(dev, host.data(), host.size() * sizeof(void*), cudaMemcpyHostToDevice, c->stream));
    uint64_t qmax = 0;
    for (int i = 0; i < l1; i++) qmax = std::max(qmax, c->mod[i]);
    const double terms = std::ldexp(1.0, 127) / ((double)qmax * (double)qmax);
    MpaJob mj{(int)C, (int)J, l1, c->log_n, (int)std::min(1024.0, std::floor(terms) - 1)};
    KL("mulplain_acc", launch_mulplain_acc((const uint64_t* const*)dev, (const uint64_t* const*)(dev + C),
                                           (uint64_t* const*)(dev + C + C * J), mj, c->tables(), c->stream));
    CK(cudaStreamSynchronize(c->stream));   // the host pointer staging must outlive the copy
    dfree(c, dev);
    for (size_t j = 0; j < J; j++) outs[j] = new_handle(c, OBJ_CT, op[j], level, 2, ci[0]->scale * pi[0]->scale);
    return HISA_OK;
}

extern "C" int hisa_rot_left_hoisted(hisa_ctx* c, hisa_ct h, const int64_t* k, size_t n, hisa_ct* outs) {
    CHECK_CTX(c);
    if ((!k || !outs) && n) return fail(HISA_E_PARAMS, "null argument");
    GET_CT(o, h);
    if (o->npolys != 2) return fail(HISA_E_NOT_RELINEARIZED, "3-poly ciphertext");
    std::vector<uint64_t> kk(n);
    for (size_t i = 0; i < n; i++) {
        normalize_rot(c, k[i], &kk[i]);
        if (kk[i]) RET(rot_key_check(c, kk[i], o->level));
    }
    // non-zero amounts share one ModUp (hoisted path); a single one uses the fused K4 path
    // (no D materialisation)
    std::vector<size_t> nz_idx;
    std::vector<uint64_t> amounts;
    for (size_t i = 0; i < n; i++) {
        if (kk[i] == 0) RET(hisa_copy(c, h, &outs[i]));
        else { nz_idx.push_back(i); amounts.push_back(kk[i]); }
    }
    if (nz_idx.empty()) return HISA_OK;
    std::vector<uint64_t*> res(nz_idx.size());
    // the multi-ciphertext K7 (<= 4 keys per launch, 1 word per thread): measured 78 % of HBM vs
    // 69 % for an 8-key 2-word kernel (round 1, removed)
    if (nz_idx.size() == 1) {
        Obj* ins[1] = {o};
        RET(rotate_batch(c, ins, 1, amounts[0], res.data()));
    } else {
        Obj* ins[1] = {o};
        RET(rotate_hoisted_multi(c, ins, 1, amounts.data(), (int)amounts.size(), res.data()));
    }
    for (size_t r = 0; r < nz_idx.size(); r++) outs[nz_idx[r]] = new_handle(c, OBJ_CT, res[r], o->level, 2, o->scale);
    return HISA_OK;
}

// ============================================================================================
// rescale / divScalar (a8), modulus switch
// ============================================================================================
// rescale of nz ciphertexts of one level and poly count (batched launches)
static int rescale_batch_ptr(hisa_ctx* c, const Obj* const* os, int nz, uint64_t** res) {
    const int l = os[0]->level, l1 = l + 1, P = os[0]->npolys;
    const long long N = (long long)c->N;
    const size_t per_tmp = (size_t)P * N + (size_t)P * l * N;
    uint64_t* tmp = dalloc_t<uint64_t>(c, per_tmp * nz);
    if (!tmp) return fail(HISA_E_OOM, "rescale");
    for (int z = 0; z < nz; z++) {
        res[z] = dalloc_t<uint64_t>(c, (size_t)P * l * N);
        if (!res[z]) return fail(HISA_E_OOM, "rescale");
    }
    Tables tb = c->tables();
    {   // INTT of the top limb of every poly
        PassJob j = job0();
        for (int z = 0; z < nz; z++) { j.src[z] = os[z]->ptr + (long long)l * N; j.dst[z] = tmp + per_tmp * z; }
        j.nb = 1; j.src_a = (long long)l1 * N; j.dst_a = N;
        j.mod_map[0] = (uint8_t)l;
        KL("rescale_intt_rows", launch_inv_passA(j, tb, P, nz, c->stream));
        for (int z = 0; z < nz; z++) j.src[z] = tmp + per_tmp * z;
        j.src_a = N;
        KL("rescale_intt_cols", launch_inv_passB(j, tb, P, nz, c->stream));
    }
    {   // lift q_l -> q_i (i < l), forward pass 1
        PassJob j = job0();
        for (int z = 0; z < nz; z++) { j.src[z] = tmp + per_tmp * z; j.dst[z] = tmp + per_tmp * z + (size_t)P * N; }
        j.nb = l; j.src_a = N; j.src_b = 0; j.dst_a = (long long)l * N; j.dst_b = N;
        ident_map(j.mod_map, l);
        for (int a = 0; a < P; a++) j.smod_map[a] = (uint8_t)l;
        KL("rescale_lift_cols", launch_fwd_pass1(j, tb, P * l, nz, true, c->stream));
    }
    {   // pass 2 + combine: out_i = (u_i - NTT_i(y)) q_l^-1
        PassJob j = job0();
        for (int z = 0; z < nz; z++) {
            j.src[z] = tmp + per_tmp * z + (size_t)P * N;
            j.dst[z] = res[z];
            j.aux[z] = os[z]->ptr;
        }
        j.nb = l;
        j.src_a = (long long)l * N; j.src_b = N;
        j.dst_a = (long long)l * N; j.dst_b = N;
        j.aux_a = (long long)l1 * N; j.aux_b = N;
        ident_map(j.mod_map, l);
        Tables tc = c->tables(c->d_qlinv + (size_t)l * (c->L + 1));
        KL("rescale_combine_rows", launch_fwd_pass2(j, tc, P * l, nz, true, c->stream));
    }
    dfree(c, tmp);
    return HISA_OK;
}
static int rescale_ptr(hisa_ctx* c, const Obj* o, uint64_t** res) { return rescale_batch_ptr(c, &o, 1, res); }

extern "C" int hisa_rescale_batch(hisa_ctx* c, const hisa_ct* in, size_t n, hisa_ct* outs) {
    CHECK_CTX(c);
    if ((!in || !outs) && n) return fail(HISA_E_PARAMS, "null argument");
    std::vector<Obj*> objs(n);
    for (size_t i = 0; i < n; i++) {
        objs[i] = get_obj(c, in[i], OBJ_CT);
        if (!objs[i]) return fail(HISA_E_INVALID_HANDLE, "invalid ciphertext handle at %zu", i);
        if (objs[i]->level != objs[0]->level || objs[i]->npolys != objs[0]->npolys)
            return fail(HISA_E_LEVEL_MISMATCH, "batch shapes differ");
    }
    if (n && objs[0]->level == 0) return fail(HISA_E_MODULUS_EXHAUSTED, "rescale at level 0");
    for (size_t i0 = 0; i0 < n; i0 += MAXB) {
        const int nz = (int)std::min((size_t)MAXB, n - i0);
        uint64_t* res[MAXB];
        RET(rescale_batch_ptr(c, objs.data() + i0, nz, res));
        for (int z = 0; z < nz; z++) {
            const Obj* o = objs[i0 + z];
            outs[i0 + z] = new_handle(c, OBJ_CT, res[z], o->level - 1, o->npolys, o->scale / (double)c->mod[o->level]);
        }
    }
    return HISA_OK;
}

extern "C" int hisa_max_scalar_div(hisa_ctx* c, hisa_ct h, uint64_t ub, uint64_t* d) {
    CHECK_CTX(c);
    GET_CT(o, h);
    if (!d) return fail(HISA_E_PARAMS, "null out");
    const uint64_t qt = c->mod[o->level];
    *d = (qt <= ub) ? qt : 1;   // A18 reading of P:584-587
    return HISA_OK;
}
extern "C" int hisa_div_scalar(hisa_ctx* c, hisa_ct h, uint64_t d, hisa_ct* out) {
    CHECK_CTX(c);
    GET_CT(o, h);
    if (d == 1) {
        if (!out) return HISA_OK;
        return hisa_copy(c, h, out);
    }
    if (o->level == 0) return fail(HISA_E_MODULUS_EXHAUSTED, "rescale at level 0");
    if (d != c->mod[o->level]) return fail(HISA_E_INVALID_DIVISOR, "divisor %llu is not q_top", (unsigned long long)d);
    uint64_t* res;
    RET(rescale_ptr(c, o, &res));
    const double ns = o->scale / (double)c->mod[o->level];
    return emit_ct(c, out, h, res, o->level - 1, o->npolys, ns);
}
extern "C" int hisa_rescale(hisa_ctx* c, hisa_ct h, hisa_ct* out) {
    CHECK_CTX(c);
    GET_CT(o, h);
    if (o->level == 0) return fail(HISA_E_MODULUS_EXHAUSTED, "rescale at level 0");
    return hisa_div_scalar(c, h, c->mod[o->level], out);
}
extern "C" int hisa_mod_switch(hisa_ctx* c, hisa_ct h, int drop, hisa_ct* out) {
    CHECK_CTX(c);
    GET_CT(o, h);
    if (drop < 0) return fail(HISA_E_PARAMS, "negative drop");
    if (o->level - drop < 0) return fail(HISA_E_MODULUS_EXHAUSTED, "mod-switch below level 0");
    const int nl = o->level + 1 - drop, l1 = o->level + 1;
    const size_t N = c->N;
    uint64_t* p = dalloc_t<uint64_t>(c, (size_t)o->npolys * nl * N);
    if (!p) return fail(HISA_E_OOM, "mod switch");
    CK(cudaMemcpy2DAsync(p, (size_t)nl * N * 8, o->ptr, (size_t)l1 * N * 8, (size_t)nl * N * 8, o->npolys,
                         cudaMemcpyDeviceToDevice, c->stream));
    return emit_ct(c, out, h, p, o->level - drop, o->npolys, o->scale);
}

extern "C" int hisa_bootstrap(hisa_ctx* c, hisa_ct h) {
    (void)h;
    if (!c) return fail(HISA_E_PARAMS, "null context");
    return fail(HISA_E_UNSUPPORTED_PROFILE, "Bootstrap profile is not implemented (P:292-293)");
}

// ============================================================================================
// conv accumulation (a9, K8): out[o] = sum_t X[o][t] in[t], X = llround(W * pt_scale)
// ============================================================================================
struct ConvJob {
    int T, OC, l1, log_n;
    long long poly_stride;
    int red_every;          // integer path: partial Barrett every this many terms (2^127 / q^2)
    uint8_t limb_map[MAXL]; // grid.y -> limb (one launch per engine class)
};
// K8: out[o][x] = sum_t W[limb][o][t] in[t][x] mod q_limb -- a modular GEMM (OC x T) x (T x N)
// per limb and poly.  CTA = 256 threads x 2 words (16-byte loads); OT outputs per pass held in
// register accumulators; the T input pointers and a TT-wide weight tile live in shared memory;
// the t loop keeps U input loads in flight (inputs are re-read from L2/HBM once per OT outputs).
//   FP = false (q >= 2^50): 128-bit integer accumulation (mac128; IMAD-pipe bound).
//   FP = true  (q <  2^50): exact FP64 (ntt_f64.cuh): t = mulred(x, w) (|t| < q) accumulated in a
//              double, re-centred (redd) every floor(2^53 / q) - 1 terms: 7 FP64-pipe ops per MAC.
// weights: [limb][OC][T] residues; in_ptrs: device array of T pointers; out_ptrs: OC.
constexpr int CONV_OT = 8, CONV_TT = 256, CONV_U = 4;
template <bool FP>
__global__ void __launch_bounds__(256) k_conv_acc(const uint64_t* const* __restrict__ in_ptrs,
                                                  uint64_t* const* __restrict__ out_ptrs,
                                                  const uint64_t* __restrict__ w, ConvJob job,
                                                  const Mod* __restrict__ mods) {
    extern __shared__ uint64_t csm[];
    const uint64_t** ptrs = reinterpret_cast<const uint64_t**>(csm);          // [T]
    uint64_t* wsm = csm + job.T;                                               // [OT][TT]
    const long long N = 1ll << job.log_n;
    const int poly = blockIdx.z;
    const int limb = job.limb_map[blockIdx.y];
    const Mod md = mods[limb];
    const double qd = (double)md.q, qinv = 1.0 / qd;
    const int red = FP ? (int)fmin(8192.0, floor(9007199254740992.0 / qd) - 1.0) : job.red_every;
    const long long off = (long long)poly * job.poly_stride + (long long)limb * N;
    const long long x = 2ll * (blockIdx.x * (long long)blockDim.x + threadIdx.x);
    for (int t = threadIdx.x; t < job.T; t += blockDim.x) ptrs[t] = in_ptrs[t] + off;
    const uint64_t* wl = w + (long long)limb * job.OC * job.T;
    for (int o0 = 0; o0 < job.OC; o0 += CONV_OT) {
        U128 acc[FP ? 1 : CONV_OT][2];
        double facc[FP ? CONV_OT : 1][2];
#pragma unroll
        for (int k = 0; k < CONV_OT; k++) {
            if constexpr (FP) { facc[k][0] = 0.0; facc[k][1] = 0.0; }
            else { acc[k][0] = U128{0, 0}; acc[k][1] = U128{0, 0}; }
        }
        int since = 0;   // terms since the last partial reduction (carried across weight tiles)
        for (int t0 = 0; t0 < job.T; t0 += CONV_TT) {
            const int tn = min(CONV_TT, job.T - t0);
            __syncthreads();
            for (int i = threadIdx.x; i < CONV_OT * CONV_TT; i += blockDim.x) {
                const int k = i / CONV_TT, tt = i % CONV_TT;
                const uint64_t wv = (o0 + k < job.OC && tt < tn) ? wl[(long long)(o0 + k) * job.T + t0 + tt] : 0;
                if constexpr (FP) reinterpret_cast<double*>(wsm)[i] = u2d(wv);
                else wsm[i] = wv;
            }
            __syncthreads();
            if (x >= N) continue;
            for (int tb = 0; tb < tn; tb += CONV_U) {
                ulonglong2 v[CONV_U];
#pragma unroll
                for (int u = 0; u < CONV_U; u++)   // U loads in flight before the MACs
                    v[u] = tb + u < tn ? __ldg(reinterpret_cast<const ulonglong2*>(ptrs[t0 + tb + u] + x))
                                       : make_ulonglong2(0, 0);
#pragma unroll
                for (int u = 0; u < CONV_U; u++) {
                    const int tt = tb + u;
                    if (tt >= tn) continue;
                    if constexpr (FP) {
                        const double* wd = reinterpret_cast<const double*>(wsm);
                        const double a0 = u2d(v[u].x), a1 = u2d(v[u].y);
#pragma unroll
                        for (int k = 0; k < CONV_OT; k++) {
                            const double wk = wd[k * CONV_TT + tt];
                            facc[k][0] = __dadd_rn(facc[k][0], mulred(a0, wk, qd, qinv));
                            facc[k][1] = __dadd_rn(facc[k][1], mulred(a1, wk, qd, qinv));
                        }
                    } else {
#pragma unroll
                        for (int k = 0; k < CONV_OT; k++) {
                            const uint64_t wk = wsm[k * CONV_TT + tt];
                            mac128(acc[k][0], v[u].x, wk);
                            mac128(acc[k][1], v[u].y, wk);
                        }
                    }
                    if (++since == red) {   // keep the accumulators bounded
                        since = 0;
#pragma unroll
                        for (int k = 0; k < CONV_OT; k++)
#pragma unroll
                            for (int h = 0; h < 2; h++) {
                                if constexpr (FP) {
                                    facc[k][h] = redd(facc[k][h], qd, qinv);
                                } else {
                                    acc[k][h].lo = barrett128(acc[k][h].lo, acc[k][h].hi, md);
                                    acc[k][h].hi = 0;
                                }
                            }
                    }
                }
            }
        }
        if (x < N) {
#pragma unroll
            for (int k = 0; k < CONV_OT; k++)
                if (o0 + k < job.OC) {
                    ulonglong2 r;
                    if constexpr (FP) r = make_ulonglong2(d_canon(facc[k][0], qd, qinv), d_canon(facc[k][1], qd, qinv));
                    else r = make_ulonglong2(barrett128(acc[k][0].lo, acc[k][0].hi, md),
                                             barrett128(acc[k][1].lo, acc[k][1].hi, md));
                    *reinterpret_cast<ulonglong2*>(out_ptrs[o0 + k] + off + x) = r;
                }
        }
    }
}

// K8 engine: tensor cores (conv_tc_kernels.cu) by default; HISA_CONV_TC=0 selects the CUDA-core
// kernel below (FP64 / 128-bit MACs), kept as the measured alternative
static bool conv_tc_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("HISA_CONV_TC");
        v = e ? atoi(e) : 1;
    }
    return v != 0;
}
static int conv_acc_common(hisa_ctx* c, const hisa_ct* in, size_t T, const double* W, size_t OC, double pt_scale,
                           hisa_ct* outs, uint64_t* dev_out) {
    CHECK_CTX(c);
    if (!in || !W || (!outs && !dev_out) || T == 0 || OC == 0) return fail(HISA_E_PARAMS, "bad arguments");
    std::vector<Obj*> objs(T);
    for (size_t t = 0; t < T; t++) {
        objs[t] = get_obj(c, in[t], OBJ_CT);
        if (!objs[t]) return fail(HISA_E_INVALID_HANDLE, "invalid ciphertext handle at %zu", t);
        if (objs[t]->npolys != 2) return fail(HISA_E_NOT_RELINEARIZED, "3-poly input");
        if (objs[t]->level != objs[0]->level) return fail(HISA_E_LEVEL_MISMATCH, "input levels differ");
        if (!scale_eq(objs[t]->scale, objs[0]->scale)) return fail(HISA_E_SCALE_MISMATCH, "input scales differ");
    }
    const int level = objs[0]->level, l1 = level + 1;
    const double ps = pt_scale == 0.0 ? (double)c->mod[level] : pt_scale;
    for (size_t i = 0; i < OC * T; i++) {
        const double v = W[i] * ps;
        if (!std::isfinite(v) || fabs(v) >= 0x1p62) return fail(HISA_E_PARAMS, "weight out of range");
    }
    const long long N = (long long)c->N;
    const bool use_tc = conv_tc_enabled() && N % 128 == 0 && T <= 4096;
    if (!use_tc && (size_t)T * sizeof(void*) + (size_t)CONV_OT * CONV_TT * 8 > 200 * 1024)
        return fail(HISA_E_PARAMS, "conv accumulation: T = %zu inputs too many", T);
    DGuard outputs(c), scratch(c);
    std::vector<uint64_t*> optr(OC);
    for (size_t o = 0; o < OC; o++) {
        optr[o] = dev_out ? dev_out + (size_t)o * 2 * l1 * N : outputs.add(dalloc_t<uint64_t>(c, (size_t)2 * l1 * N));
        if (!optr[o]) return fail(HISA_E_OOM, "conv outputs");
    }
    std::vector<const uint64_t*> iptr(T);
    for (size_t t = 0; t < T; t++) iptr[t] = objs[t]->ptr;
    const uint64_t** dip = scratch.add((const uint64_t**)dalloc(c, T * sizeof(void*)));
    uint64_t** dop = scratch.add((uint64_t**)dalloc(c, OC * sizeof(void*)));
    if (!dip || !dop) return fail(HISA_E_OOM, "conv scratch");
    CK(cudaMemcpyAsync(dip, iptr.data(), T * sizeof(void*), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(dop, optr.data(), OC * sizeof(void*), cudaMemcpyHostToDevice, c->stream));
    if (use_tc) {
        // tensor-core path (conv_tc_kernels.cu): weights rounded, reduced and byte-split into the
        // MMA's shared-memory image per (limb, 16-output tile, 32-input chunk) on the device
        const int n_chunks = (int)((T + 31) / 32), n_oct = (int)((OC + 15) / 16);
        ConvTcJob tj;
        memset(&tj, 0, sizeof tj);
        tj.T = (int)T; tj.OC = (int)OC; tj.log_n = c->log_n; tj.n_chunks = n_chunks; tj.n_oct = n_oct;
        tj.poly_stride = (long long)l1 * N;
        for (int i = 0; i < l1; i++) {
            int P = 0;
            for (uint64_t q = c->mod[i] - 1; q; q >>= 8) P++;
            tj.P[i] = (uint8_t)P;
            tj.limb_map[i] = (uint8_t)i;
        }
        const size_t img_bytes = (size_t)l1 * n_oct * n_chunks * 8 * 512;
        uint8_t* dimg = scratch.add((uint8_t*)dalloc(c, img_bytes));
        double* dW = scratch.add(dalloc_t<double>(c, OC * T));
        uint8_t* dP = scratch.add((uint8_t*)dalloc(c, MAXL));
        if (!dimg || !dW || !dP) return fail(HISA_E_OOM, "conv weight image");
        CK(cudaMemcpyAsync(dW, W, OC * T * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(dP, tj.P, MAXL, cudaMemcpyHostToDevice, c->stream));
        {
            ProfScope ps_(c, "conv_acc");
            CK(launch_conv_tc_wimg(dW, ps, (int)T, (int)OC, n_oct, n_chunks, l1, c->d_mods, dP, dimg, c->stream));
            CK(launch_conv_tc(dip, dop, dimg, tj, l1, c->d_mods, c->stream));
        }
        CK(cudaStreamSynchronize(c->stream));   // host staging vectors must outlive the copies
        if (conv_tc_timed_out()) {
            c->poisoned = true;
            return fail(HISA_E_CUDA, "conv accumulation: tensor-core mbarrier wait timed out");
        }
        outputs.keep();   // scratch (image, weights, pointer arrays) freed by its guard
        if (outs)
            for (size_t o = 0; o < OC; o++) outs[o] = new_handle(c, OBJ_CT, optr[o], level, 2, objs[0]->scale * ps);
        return HISA_OK;
    }
    std::vector<uint64_t> wres((size_t)OC * T * l1);   // [limb][OC][T]
    for (size_t o = 0; o < OC; o++)
        for (size_t t = 0; t < T; t++) {
            const long long X = llround(W[o * T + t] * ps);
            for (int i = 0; i < l1; i++) {
                const uint64_t q = c->mod[i];
                wres[((size_t)i * OC + o) * T + t] = (uint64_t)(((__int128)X % (__int128)q + q) % q);
            }
        }
    uint64_t* dw = scratch.add(dalloc_t<uint64_t>(c, wres.size()));
    if (!dw) return fail(HISA_E_OOM, "conv scratch");
    CK(cudaMemcpyAsync(dw, wres.data(), wres.size() * 8, cudaMemcpyHostToDevice, c->stream));
    uint64_t qmax = 0;
    for (int i = 0; i < l1; i++) qmax = std::max(qmax, c->mod[i]);
    const double terms = std::ldexp(1.0, 127) / ((double)qmax * (double)qmax);   // 128-bit headroom
    ConvJob cj;
    memset(&cj, 0, sizeof cj);
    cj.T = (int)T; cj.OC = (int)OC; cj.l1 = l1; cj.log_n = c->log_n; cj.poly_stride = (long long)l1 * N;
    cj.red_every = (int)std::min(1024.0, std::floor(terms) - 1);
    dim3 grid((unsigned)((N / 2 + 255) / 256), 1, 2);
    const size_t smem = (size_t)T * sizeof(void*) + (size_t)CONV_OT * CONV_TT * 8;
    for (int fpc = 0; fpc < 2; fpc++) {   // one launch per butterfly-engine class of limbs
        ConvJob j2 = cj;
        int n = 0;
        for (int i = 0; i < l1; i++)
            if (((double)c->mod[i] < c->f64_max_q) == (fpc == 1)) j2.limb_map[n++] = (uint8_t)i;
        if (!n) continue;
        grid.y = n;
        ProfScope ps_(c, "conv_acc");
        if (fpc) {
            if (smem > 48 * 1024)
                cudaFuncSetAttribute(k_conv_acc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            k_conv_acc<true><<<grid, 256, smem, c->stream>>>(dip, dop, dw, j2, c->d_mods);
        } else {
            if (smem > 48 * 1024)
                cudaFuncSetAttribute(k_conv_acc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            k_conv_acc<false><<<grid, 256, smem, c->stream>>>(dip, dop, dw, j2, c->d_mods);
        }
        CK(cudaGetLastError());
    }
    CK(cudaStreamSynchronize(c->stream));   // host staging vectors must outlive the copies
    outputs.keep();
    if (outs)
        for (size_t o = 0; o < OC; o++) outs[o] = new_handle(c, OBJ_CT, optr[o], level, 2, objs[0]->scale * ps);
    return HISA_OK;
}
extern "C" int hisa_conv_accumulate(hisa_ctx* c, const hisa_ct* in, size_t T, const double* W, size_t OC,
                                    double pt_scale, hisa_ct* outs) {
    if (!outs) return fail(HISA_E_PARAMS, "null outs");
    return conv_acc_common(c, in, T, W, OC, pt_scale, outs, nullptr);
}
extern "C" int hisa_conv_accumulate_dev(hisa_ctx* c, const hisa_ct* in, size_t T, const double* W, size_t OC,
                                        double pt_scale, uint64_t* dev_out) {
    if (!dev_out) return fail(HISA_E_PARAMS, "null dev_out");
    return conv_acc_common(c, in, T, W, OC, pt_scale, nullptr, dev_out);
}

// ============================================================================================
// inspection / import / export
// ============================================================================================
extern "C" int hisa_ct_info(hisa_ctx* c, hisa_ct h, int* level, int* npolys, double* scale) {
    CHECK_CTX(c);
    GET_CT(o, h);
    if (level) *level = o->level;
    if (npolys) *npolys = o->npolys;
    if (scale) *scale = o->scale;
    return HISA_OK;
}
extern "C" int hisa_pt_info(hisa_ctx* c, hisa_pt h, int* level, double* scale) {
    CHECK_CTX(c);
    GET_PT(o, h);
    if (level) *level = o->level;
    if (scale) *scale = o->scale;
    return HISA_OK;
}
static int export_obj(hisa_ctx* c, Obj* o, uint64_t* host, size_t words) {
    const size_t w = obj_words(c, o);
    if (!host || words != w) return fail(HISA_E_PARAMS, "object has %zu words, got %zu", w, words);
    CK(cudaMemcpyAsync(host, o->ptr, w * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return HISA_OK;
}
extern "C" int hisa_ct_export(hisa_ctx* c, hisa_ct h, uint64_t* host, size_t words) {
    CHECK_CTX(c);
    GET_CT(o, h);
    return export_obj(c, o, host, words);
}
extern "C" int hisa_pt_export(hisa_ctx* c, hisa_pt h, uint64_t* host, size_t words) {
    CHECK_CTX(c);
    GET_PT(o, h);
    return export_obj(c, o, host, words);
}
static int check_layout(hisa_ctx* c, int level, int npolys) {
    if (level < 0 || level >= c->L) return fail(HISA_E_PARAMS, "level %d out of range", level);
    if (npolys < 1 || npolys > 3) return fail(HISA_E_PARAMS, "npolys must be 1..3");
    return HISA_OK;
}
extern "C" int hisa_ct_import(hisa_ctx* c, const uint64_t* host, int level, int npolys, double scale, hisa_ct* out) {
    CHECK_CTX(c);
    if (!host || !out) return fail(HISA_E_PARAMS, "null argument");
    RET(check_layout(c, level, npolys));
    if (npolys < 2) return fail(HISA_E_PARAMS, "a ciphertext has 2 or 3 polys");
    const size_t w = (size_t)npolys * (level + 1) * c->N;
    uint64_t* p = dalloc_t<uint64_t>(c, w);
    if (!p) return fail(HISA_E_OOM, "import");
    CK(cudaMemcpyAsync(p, host, w * 8, cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    *out = new_handle(c, OBJ_CT, p, level, npolys, scale);
    return HISA_OK;
}
extern "C" int hisa_pt_import(hisa_ctx* c, const uint64_t* host, int level, double scale, hisa_pt* out) {
    CHECK_CTX(c);
    if (!host || !out) return fail(HISA_E_PARAMS, "null argument");
    RET(check_layout(c, level, 1));
    const size_t w = (size_t)(level + 1) * c->N;
    uint64_t* p = dalloc_t<uint64_t>(c, w);
    if (!p) return fail(HISA_E_OOM, "import");
    CK(cudaMemcpyAsync(p, host, w * 8, cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    *out = new_handle(c, OBJ_PT, p, level, 1, scale);
    return HISA_OK;
}
extern "C" int hisa_ct_device_view(hisa_ctx* c, hisa_ct h, uint64_t** dev, size_t* words) {
    CHECK_CTX(c);
    GET_CT(o, h);
    if (dev) *dev = o->ptr;
    if (words) *words = obj_words(c, o);
    return HISA_OK;
}
extern "C" int hisa_ct_adopt_device(hisa_ctx* c, const uint64_t* dev, int level, int npolys, double scale,
                                    hisa_ct* out) {
    CHECK_CTX(c);
    if (!dev || !out) return fail(HISA_E_PARAMS, "null argument");
    RET(check_layout(c, level, npolys));
    const size_t w = (size_t)npolys * (level + 1) * c->N;
    uint64_t* p = dalloc_t<uint64_t>(c, w);
    if (!p) return fail(HISA_E_OOM, "adopt");
    CK(cudaMemcpyAsync(p, dev, w * 8, cudaMemcpyDeviceToDevice, c->stream));
    *out = new_handle(c, OBJ_CT, p, level, npolys, scale);
    return HISA_OK;
}
extern "C" int hisa_ct_adopt_sum(hisa_ctx* c, const int64_t* dev, int level, int npolys, double scale, hisa_ct* out) {
    CHECK_CTX(c);
    if (!dev || !out) return fail(HISA_E_PARAMS, "null argument");
    RET(check_layout(c, level, npolys));
    const size_t w = (size_t)npolys * (level + 1) * c->N;
    uint64_t* p = dalloc_t<uint64_t>(c, w);
    if (!p) return fail(HISA_E_OOM, "adopt");
    KL("reduce_sum", launch_reduce_sum(dev, p, npolys, level + 1, c->log_n, c->d_mods, c->stream));
    *out = new_handle(c, OBJ_CT, p, level, npolys, scale);
    return HISA_OK;
}
extern "C" int hisa_ct_random(hisa_ctx* c, uint64_t b, int level, int npolys, hisa_ct* out) {
    CHECK_CTX(c);
    if (!out) return fail(HISA_E_PARAMS, "null out");
    RET(check_layout(c, level, npolys));
    const int l1 = level + 1;
    uint64_t* p = dalloc_t<uint64_t>(c, (size_t)npolys * l1 * c->N);
    if (!p) return fail(HISA_E_OOM, "random ct");
    uint64_t idx[MAXL];
    uint8_t mm[MAXL];
    ident_map(mm, l1);
    for (int k = 0; k < npolys; k++) {
        for (int i = 0; i < l1; i++) idx[i] = (b << 32) | ((uint64_t)k << 16) | (uint64_t)i;
        CK(launch_sample_uniform(p + (size_t)k * l1 * c->N, c->seed, TAG_BENCH, idx, mm, l1, c->log_n, c->d_mods,
                                 c->stream));
    }
    *out = new_handle(c, OBJ_CT, p, level, npolys, 0x1p40);
    return HISA_OK;
}
extern "C" int hisa_pt_random(hisa_ctx* c, uint64_t b, int level, hisa_pt* out) {
    CHECK_CTX(c);
    if (!out) return fail(HISA_E_PARAMS, "null out");
    RET(check_layout(c, level, 1));
    const int l1 = level + 1;
    uint64_t* p = dalloc_t<uint64_t>(c, (size_t)l1 * c->N);
    if (!p) return fail(HISA_E_OOM, "random pt");
    uint64_t idx[MAXL];
    uint8_t mm[MAXL];
    ident_map(mm, l1);
    for (int i = 0; i < l1; i++) idx[i] = (b << 32) | (0xFFFFull << 16) | (uint64_t)i;
    CK(launch_sample_uniform(p, c->seed, TAG_BENCH, idx, mm, l1, c->log_n, c->d_mods, c->stream));
    *out = new_handle(c, OBJ_PT, p, level, 1, 0x1p40);
    return HISA_OK;
}

// ============================================================================================
// raw NTT / INTT of every limb of ciphertexts, in place (config 2 sweeps these as ops, a1/a2)
// ============================================================================================
extern "C" int hisa_ntt_batch(hisa_ctx* c, const hisa_ct* hs, size_t n, int inverse) {
    CHECK_CTX(c);
    if (!hs && n) return fail(HISA_E_PARAMS, "null argument");
    std::vector<Obj*> objs(n);
    for (size_t i = 0; i < n; i++) {
        objs[i] = get_obj(c, hs[i], OBJ_CT);
        if (!objs[i]) return fail(HISA_E_INVALID_HANDLE, "invalid ciphertext handle at %zu", i);
        if (objs[i]->level != objs[0]->level || objs[i]->npolys != objs[0]->npolys)
            return fail(HISA_E_LEVEL_MISMATCH, "batch shapes differ");
    }
    for (size_t i0 = 0; i0 < n; i0 += MAXB) {
        const int nz = (int)std::min((size_t)MAXB, n - i0);
        const int l1 = objs[i0]->level + 1, P = objs[i0]->npolys;
        uint64_t* ptrs[MAXB];
        for (int z = 0; z < nz; z++) ptrs[z] = objs[i0 + z]->ptr;
        uint8_t mm[MAXL];
        ident_map(mm, l1);
        if (inverse) RET(ntt_inv(c, ptrs, ptrs, nz, l1, mm, P * l1));
        else RET(ntt_fwd(c, ptrs, nz, l1, mm, P * l1));
    }
    return HISA_OK;
}
extern "C" int hisa_ntt(hisa_ctx* c, hisa_ct h, int inverse) { return hisa_ntt_batch(c, &h, 1, inverse); }

// ============================================================================================
// profiling / accounting / microbenchmark (diagnostics; not HISA instructions)
// ============================================================================================
extern "C" int hisa_profile(hisa_ctx* c, int enable) {
    CHECK_CTX(c);
    CK(cudaStreamSynchronize(c->stream));
    for (auto& r : c->prof) { c->ev_pool.push_back(r.a); c->ev_pool.push_back(r.b); }
    c->prof.clear();
    c->prof_on = enable != 0;
    c->launches = 0;
    return HISA_OK;
}
extern "C" int hisa_launch_count(hisa_ctx* c, uint64_t* n) {
    CHECK_CTX(c);
    if (!n) return fail(HISA_E_PARAMS, "null out");
    *n = c->launches;
    return HISA_OK;
}
extern "C" int hisa_profile_read(hisa_ctx* c, char* names, size_t names_len, double* ms, uint64_t* counts,
                                 size_t max_entries, size_t* n_entries) {
    CHECK_CTX(c);
    CK(cudaStreamSynchronize(c->stream));
    std::map<std::string, std::pair<double, uint64_t>> agg;
    for (auto& r : c->prof) {
        float t = 0;
        CK(cudaEventElapsedTime(&t, r.a, r.b));
        auto& e = agg[r.name];
        e.first += t;
        e.second += 1;
        c->ev_pool.push_back(r.a);
        c->ev_pool.push_back(r.b);
    }
    c->prof.clear();
    std::string all;
    size_t i = 0;
    for (auto& kv : agg) {
        if (i >= max_entries) break;
        if (ms) ms[i] = kv.second.first;
        if (counts) counts[i] = kv.second.second;
        all += kv.first;
        all += "\n";
        i++;
    }
    if (names) {
        if (all.size() + 1 > names_len) return fail(HISA_E_PARAMS, "names buffer too small");
        memcpy(names, all.c_str(), all.size() + 1);
    }
    if (n_entries) *n_entries = i;
    return HISA_OK;
}

// register-resident Harvey CT butterflies (radix-16 pattern, twiddle in registers): the
// integer-pipe ceiling for the NTT-bearing kernels
__global__ void __launch_bounds__(256) k_mb_butterfly(uint64_t* out, uint64_t q, uint64_t w, uint64_t wp, int iters) {
    uint64_t r[16];
    const uint64_t q2 = 2 * q;
#pragma unroll
    for (int e = 0; e < 16; e++) r[e] = (threadIdx.x * 16 + e + blockIdx.x) % q;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int st = 0; st < 4; st++) {
            const int dist = 8 >> st;
#pragma unroll
            for (int e = 0; e < 16; e++) {
                if (e & dist) continue;
                uint64_t X = r[e];
                X = X >= q2 ? X - q2 : X;
                const uint64_t T = mul_shoup_lazy(r[e + dist], w, wp, q);
                r[e] = X + T;
                r[e + dist] = X - T + q2;
            }
        }
    }
    uint64_t x = 0;
#pragma unroll
    for (int e = 0; e < 16; e++) x ^= r[e];
    out[blockIdx.x * blockDim.x + threadIdx.x] = x;
}
// the same pattern with the exact FP64 butterfly of ntt_f64.cuh (centred-lazy doubles, q < 2^50):
// the ceiling of the FP64-engine kernels
__global__ void __launch_bounds__(256) k_mb_butterfly_f64(double* out, double q, double qinv, double w, int iters) {
    double r[16];
#pragma unroll
    for (int e = 0; e < 16; e++) r[e] = (double)((threadIdx.x * 16 + e + blockIdx.x) % 1000003);
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int st = 0; st < 8; st++) {   // one 8-stage pass with the engines' lazy schedule
            const int dist = 8 >> (st & 3);
#pragma unroll
            for (int e = 0; e < 16; e++) {
                if (e & dist) continue;
                const double X = full_stage(st, 8) ? redd(r[e], q, qinv) : r[e];
                const double T = mulred(r[e + dist], w, q, qinv);
                r[e] = __dadd_rn(X, T);
                r[e + dist] = __dsub_rn(X, T);
            }
        }
    }
    double x = 0;
#pragma unroll
    for (int e = 0; e < 16; e++) x += r[e];
    out[blockIdx.x * blockDim.x + threadIdx.x] = x;
}

extern "C" int hisa_microbench_butterfly_f64(hisa_ctx* c, int iters, double* bfly_per_s) {
    CHECK_CTX(c);
    if (!bfly_per_s || iters <= 0) return fail(HISA_E_PARAMS, "bad arguments");
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int blocks = sms * 8, threads = 256;
    double* out = dalloc_t<double>(c, (size_t)blocks * threads);
    if (!out) return fail(HISA_E_OOM, "microbench");
    uint64_t q = 0;
    for (int i = 0; i < c->L; i++)
        if (c->mod[i] < (1ull << 50)) { q = c->mod[i]; break; }
    if (!q) q = (1ull << 49) + 1;   // timing only
    const double qd = (double)q, w = (double)(3 % q);
    cudaEvent_t a = take_event(c), b = take_event(c);
    k_mb_butterfly_f64<<<blocks, threads, 0, c->stream>>>(out, qd, 1.0 / qd, w, 4);
    CK(cudaEventRecord(a, c->stream));
    k_mb_butterfly_f64<<<blocks, threads, 0, c->stream>>>(out, qd, 1.0 / qd, w, iters);
    CK(cudaEventRecord(b, c->stream));
    CK(cudaEventSynchronize(b));
    float t = 0;
    CK(cudaEventElapsedTime(&t, a, b));
    c->ev_pool.push_back(a);
    c->ev_pool.push_back(b);
    dfree(c, out);
    *bfly_per_s = (double)blocks * threads * iters * 64.0 / (t * 1e-3);
    return HISA_OK;
}

// the key multiply-accumulate of K4 (k_ks_ip5): a 52-bit D times a 50-bit key word, split into
// 32 x 25-bit halves and accumulated in three 64-bit sums (4 IMAD.WIDE.U32 per MAC); two keys (b, a)
// per D as in K4 -- the integer-pipe ceiling of the key inner products
__global__ void __launch_bounds__(256) k_mb_mac(uint64_t* out, uint64_t k0, uint64_t k1, int iters) {
    uint64_t D[8], A0[16], A1[16], A2[16];
#pragma unroll
    for (int e = 0; e < 8; e++) D[e] = ((uint64_t)(threadIdx.x * 8 + e + blockIdx.x) << 20) | 12345u;
#pragma unroll
    for (int e = 0; e < 16; e++) { A0[e] = 0; A1[e] = 0; A2[e] = 0; }
    for (int it = 0; it < iters; it++) {
        const uint32_t kl0 = (uint32_t)k0 & 0x1FFFFFFu, kh0 = (uint32_t)(k0 >> 25);
        const uint32_t kl1 = (uint32_t)k1 & 0x1FFFFFFu, kh1 = (uint32_t)(k1 >> 25);
#pragma unroll
        for (int e = 0; e < 8; e++) {
            const uint32_t dl = (uint32_t)D[e], dh = (uint32_t)(D[e] >> 32);
            A0[2 * e] += (uint64_t)dl * kl0;
            A1[2 * e] += (uint64_t)dl * kh0;
            A1[2 * e] += (uint64_t)(dh << 7) * kl0;
            A2[2 * e] += (uint64_t)dh * kh0;
            A0[2 * e + 1] += (uint64_t)dl * kl1;
            A1[2 * e + 1] += (uint64_t)dl * kh1;
            A1[2 * e + 1] += (uint64_t)(dh << 7) * kl1;
            A2[2 * e + 1] += (uint64_t)dh * kh1;
        }
        k0 += 0x9E3779B97Full;
        k1 += 0x7F4A7C15ull;
    }
    uint64_t x = 0;
#pragma unroll
    for (int e = 0; e < 16; e++) x ^= A0[e] + (A1[e] << 25) + (A2[e] << 57);
    out[blockIdx.x * blockDim.x + threadIdx.x] = x;
}

extern "C" int hisa_microbench_mac(hisa_ctx* c, int iters, double* mac_per_s) {
    CHECK_CTX(c);
    if (!mac_per_s || iters <= 0) return fail(HISA_E_PARAMS, "bad arguments");
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int blocks = sms * 8, threads = 256;
    uint64_t* out = dalloc_t<uint64_t>(c, (size_t)blocks * threads);
    if (!out) return fail(HISA_E_OOM, "microbench");
    cudaEvent_t a = take_event(c), b = take_event(c);
    k_mb_mac<<<blocks, threads, 0, c->stream>>>(out, 0x2F0F0F0F0F0ull, 0x1234567890ull, 4);   // warm-up
    CK(cudaEventRecord(a, c->stream));
    k_mb_mac<<<blocks, threads, 0, c->stream>>>(out, 0x2F0F0F0F0F0ull, 0x1234567890ull, iters);
    CK(cudaEventRecord(b, c->stream));
    CK(cudaEventSynchronize(b));
    float t = 0;
    CK(cudaEventElapsedTime(&t, a, b));
    c->ev_pool.push_back(a);
    c->ev_pool.push_back(b);
    dfree(c, out);
    *mac_per_s = (double)blocks * threads * iters * 16.0 / (t * 1e-3);
    return HISA_OK;
}

extern "C" int hisa_microbench_butterfly(hisa_ctx* c, int iters, double* bfly_per_s) {
    CHECK_CTX(c);
    if (!bfly_per_s || iters <= 0) return fail(HISA_E_PARAMS, "bad arguments");
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int blocks = sms * 8, threads = 256;
    uint64_t* out = dalloc_t<uint64_t>(c, (size_t)blocks * threads);
    if (!out) return fail(HISA_E_OOM, "microbench");
    const uint64_t q = c->mod[0], w = 3 % q;
    cudaEvent_t a = take_event(c), b = take_event(c);
    k_mb_butterfly<<<blocks, threads, 0, c->stream>>>(out, q, w, shoup(w, q), 4);   // warm-up
    CK(cudaEventRecord(a, c->stream));
    k_mb_butterfly<<<blocks, threads, 0, c->stream>>>(out, q, w, shoup(w, q), iters);
    CK(cudaEventRecord(b, c->stream));
    CK(cudaEventSynchronize(b));
    float t = 0;
    CK(cudaEventElapsedTime(&t, a, b));
    c->ev_pool.push_back(a);
    c->ev_pool.push_back(b);
    dfree(c, out);
    *bfly_per_s = (double)blocks * threads * iters * 32.0 / (t * 1e-3);
    return HISA_OK;
}
