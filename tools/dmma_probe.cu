// dmma_probe.cu -- throughput of fp64 mma.sync (m8n8k4) vs plain DFMA on this GPU.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_probe dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

__device__ __forceinline__ void dmma16(double* c, const double* a, const double* b) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
                 "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                 : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]),
                   "d"(a[7]), "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

__global__ void k_dmma16(int iters, double* out) {
    double c[4][4], a[8], b[4];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
    for (int i = 0; i < 4; ++i) b[i] = blockIdx.x * 1e-3 + i;
#pragma unroll
    for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 4; ++i) dmma16(c[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
    if (s == 12345.678) out[0] = s;
}

template <int NACC>
__global__ void k_dmma(int iters, double* out) {
    double c[NACC][2];
    double a = threadIdx.x * 1e-3, b = blockIdx.x * 1e-3;
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i][0] = c[i][1] = i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NACC; ++i) dmma(c[i][0], c[i][1], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.678) out[0] = s;
}

__global__ void k_dfma(int iters, double* out) {
    double c[16];
    double a = threadIdx.x * 1e-3, b = blockIdx.x * 1e-3;
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) c[i] = fma(a, c[i], b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += c[i];
    if (s == 12345.678) out[0] = s;
}

__global__ void k_mixed(int iters, double* out) {
    const int warp = threadIdx.x >> 5;
    double a = threadIdx.x * 1e-3, b = blockIdx.x * 1e-3;
    double s = 0;
    if (warp & 1) {
        double c[8][2];
#pragma unroll
        for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = i;
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int i = 0; i < 8; ++i) dmma(c[i][0], c[i][1], a, b);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    } else {
        double c[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) c[i] = i;
        for (int it = 0; it < iters * 8; ++it) {
#pragma unroll
            for (int i = 0; i < 16; ++i) c[i] = fma(a, c[i], b);
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) s += c[i];
    }
    if (s == 12345.678) out[0] = s;
}

int main() {
    double* out;
    cudaMalloc(&out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 4096;
    for (int wpb : {4, 8, 16}) {
        for (int bps : {1, 2, 4}) {
            const int blocks = sms * bps, thr = 32 * wpb;
            k_dmma<8><<<blocks, thr>>>(16, out);
            cudaEventRecord(e0);
            k_dmma<8><<<blocks, thr>>>(iters, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double flops = 2.0 * 256 * 8 * (double)iters * blocks * wpb;
            printf("DMMA wpb=%d bps=%d: %.2f TFLOP/s\n", wpb, bps, flops / ms * 1e-9);
        }
    }
    for (int wpb : {4, 8, 16}) {
        const int blocks = sms * 2, thr = 32 * wpb;
        k_dmma16<<<blocks, thr>>>(16, out);
        cudaEventRecord(e0);
        k_dmma16<<<blocks, thr>>>(iters, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 2.0 * 16 * 8 * 16 * 4 * (double)iters * blocks * wpb;
        printf("DMMA16 wpb=%d: %.2f TFLOP/s\n", wpb, flops / ms * 1e-9);
    }
    for (int wpb : {4, 8, 16}) {
        const int blocks = sms * 4, thr = 32 * wpb;
        k_dfma<<<blocks, thr>>>(16, out);
        cudaEventRecord(e0);
        k_dfma<<<blocks, thr>>>(iters, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 2.0 * 16 * (double)iters * blocks * thr;
        printf("DFMA wpb=%d: %.2f TFLOP/s\n", wpb, flops / ms * 1e-9);
    }
    for (int wpb : {8, 16}) {
        const int blocks = sms * 2, thr = 32 * wpb;
        k_mixed<<<blocks, thr>>>(16, out);
        cudaEventRecord(e0);
        k_mixed<<<blocks, thr>>>(iters, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        // dmma warps: 8*256*iters FMAs; dfma warps: 16*8*iters*32 FMAs = 4096*iters (same)
        const double flops = 2.0 * 2048 * (double)iters * blocks * wpb;
        printf("MIXED wpb=%d: %.2f TFLOP/s (ms %.3f)\n", wpb, flops / ms * 1e-9, ms);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
