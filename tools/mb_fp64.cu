// Microbenchmark: integer Harvey/Shoup butterfly vs an exact FP64 modular butterfly
// (q < 2^50: h = a*w, l = fma(a, w, -h) exact, quot = rint(h * qinv), r = fma(-quot, q, h) + l).
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

// values kept in [0, 2q) as doubles; T = a*w mod q in [0, q)
__global__ void k_fp64(double* out, double q, double w, double qinv, int iters) {
    double r[16];
#pragma unroll
    for (int e = 0; e < 16; e++) r[e] = (double)((threadIdx.x * 16 + e + blockIdx.x) % 1000003);
    const double q2 = 2 * q;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int st = 0; st < 4; st++) {
            const int dist = 8 >> st;
#pragma unroll
            for (int e = 0; e < 16; e++) {
                if (e & dist) continue;
                double X = r[e];
                X = X >= q ? X - q : X;               // [0, q)
                const double a = r[e + dist];
                const double h = a * w;
                const double l = fma(a, w, -h);
                const double qt = rint(h * qinv);
                double T = fma(-qt, q, h) + l;        // (-q, q)
                T = T < 0 ? T + q : T;                // [0, q)
                r[e] = X + T;                         // [0, 2q)
                r[e + dist] = X - T + q;              // (0, 2q)
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
    const uint64_t q = (1ull << 50) - 27 * (1ull << 17) + 1;   // any odd 50-bit value for timing
    const uint64_t w = 123456789123ull % q;
    const uint64_t wp = (uint64_t)(((unsigned __int128)w << 64) / q);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 2; rep++) {
        k_int<<<blocks, threads>>>((uint64_t*)out, q, w, wp, 4);
        cudaEventRecord(a);
        k_int<<<blocks, threads>>>((uint64_t*)out, q, w, wp, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ti; cudaEventElapsedTime(&ti, a, b);
        k_fp64<<<blocks, threads>>>((double*)out, (double)q, (double)w, 1.0 / (double)q, 4);
        cudaEventRecord(a);
        k_fp64<<<blocks, threads>>>((double*)out, (double)q, (double)w, 1.0 / (double)q, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float tf; cudaEventElapsedTime(&tf, a, b);
        const double bf = (double)blocks * threads * iters * 32.0;
        printf("int  butterflies/s: %.1f G\nfp64 butterflies/s: %.1f G\n", bf / (ti * 1e-3) / 1e9, bf / (tf * 1e-3) / 1e9);
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
