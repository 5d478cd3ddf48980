// Microbenchmark of butterfly engines on B200 (all SMs, register-resident):
//   int  : 64-bit Shoup/Harvey (ntt.cuh)
//   frnd : exact FP64 butterfly with rint()  (FRND.F64)           (ntt_f64.cuh, before)
//   magic: exact FP64 butterfly, rint(x) = (x + 1.5 2^52) - 1.5 2^52 (two DADD, |x| < 2^51)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mulhi(uint64_t a, uint64_t b) { return __umul64hi(a, b); }

__global__ void k_int(uint64_t* out, uint64_t q, uint64_t w, uint64_t wp, int iters) {
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
                const uint64_t T = r[e + dist] * w - mulhi(r[e + dist], wp) * q;
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

template <bool MAGIC>
__device__ __forceinline__ double rnd(double x) {
    if (MAGIC) return __dsub_rn(__dadd_rn(x, 6755399441055744.0), 6755399441055744.0);
    return rint(x);
}
template <bool MAGIC>
__global__ void k_fp64(double* out, double q, double w, double qinv, int iters) {
    double r[16];
#pragma unroll
    for (int e = 0; e < 16; e++) r[e] = (double)((threadIdx.x * 16 + e + blockIdx.x) % 1000003);
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int st = 0; st < 4; st++) {
            const int dist = 8 >> st;
#pragma unroll
            for (int e = 0; e < 16; e++) {
                if (e & dist) continue;
                const double X = __fma_rn(-rnd<MAGIC>(__dmul_rn(r[e], qinv)), q, r[e]);
                const double a = r[e + dist];
                const double h = __dmul_rn(a, w);
                const double l = __fma_rn(a, w, -h);
                const double qt = rnd<MAGIC>(__dmul_rn(h, qinv));
                const double T = __dadd_rn(__fma_rn(-qt, q, h), l);
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

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8, threads = 256, iters = 2000;
    void* out;
    cudaMalloc(&out, (size_t)blocks * threads * 8);
    const uint64_t q = (1ull << 50) - 27 * (1ull << 17) + 1;
    const uint64_t w = 123456789123ull % q;
    const uint64_t wp = (uint64_t)(((unsigned __int128)w << 64) / q);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    const double bf = (double)blocks * threads * iters * 32.0;
    for (int rep = 0; rep < 2; rep++) {
        float t;
        k_int<<<blocks, threads>>>((uint64_t*)out, q, w, wp, 4);
        cudaEventRecord(a); k_int<<<blocks, threads>>>((uint64_t*)out, q, w, wp, iters); cudaEventRecord(b);
        cudaEventSynchronize(b); cudaEventElapsedTime(&t, a, b);
        printf("int   butterflies/s: %.1f G\n", bf / (t * 1e-3) / 1e9);
        k_fp64<false><<<blocks, threads>>>((double*)out, (double)q, (double)w, 1.0 / (double)q, 4);
        cudaEventRecord(a); k_fp64<false><<<blocks, threads>>>((double*)out, (double)q, (double)w, 1.0 / (double)q, iters);
        cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&t, a, b);
        printf("frnd  butterflies/s: %.1f G\n", bf / (t * 1e-3) / 1e9);
        k_fp64<true><<<blocks, threads>>>((double*)out, (double)q, (double)w, 1.0 / (double)q, 4);
        cudaEventRecord(a); k_fp64<true><<<blocks, threads>>>((double*)out, (double)q, (double)w, 1.0 / (double)q, iters);
        cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&t, a, b);
        printf("magic butterflies/s: %.1f G\n", bf / (t * 1e-3) / 1e9);
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
