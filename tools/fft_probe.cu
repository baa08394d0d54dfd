// fft_probe.cu -- measures cuFFT fp64 variants at the FFT sizes of the
// BASELINE configs (D = 2 Mtilde), to choose the transform layout.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o fft_probe fft_probe.cu -lcufft
#include <cuda_runtime.h>
#include <cufft.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                       \
    do {                                                                            \
        auto e = (x);                                                               \
        if (e != 0) {                                                               \
            std::printf("error %d at %s:%d (%s)\n", (int)e, __FILE__, __LINE__, #x); \
            std::exit(1);                                                           \
        }                                                                           \
    } while (0)

static float timeit(cufftHandle p, void* in, void* out, int type, int dir, int reps = 5) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&] {
        if (type == 0) CK(cufftExecD2Z(p, (double*)in, (cufftDoubleComplex*)out));
        if (type == 1) CK(cufftExecZ2D(p, (cufftDoubleComplex*)in, (double*)out));
        if (type == 2) CK(cufftExecZ2Z(p, (cufftDoubleComplex*)in, (cufftDoubleComplex*)out, dir));
    };
    run();
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(a);
        run();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    return best;
}

int main(int argc, char** argv) {
    std::vector<int> Ds = {194, 298, 624, 1200};
    if (argc > 1) {
        Ds.clear();
        for (int i = 1; i < argc; ++i) Ds.push_back(std::atoi(argv[i]));
    }
    for (int D : Ds) {
        const int Mt = D / 2;
        const long long Dh = D / 2 + 1;
        const size_t bytes = sizeof(double) * (size_t)D * D * (D + 2);
        void* buf;
        void* buf2;
        CK(cudaMalloc(&buf, bytes));
        CK(cudaMalloc(&buf2, bytes));
        CK(cudaMemset(buf, 0, bytes));
        CK(cudaMemset(buf2, 0, bytes));
        const double GB = bytes / 1e9;
        std::printf("D=%d  (real padded array %.2f GB)\n", D, GB);
        cufftHandle p;
        size_t ws;
        // 3D D2Z in place
        {
            CK(cufftCreate(&p));
            CK(cufftMakePlan3d(p, D, D, D, CUFFT_D2Z, &ws));
            float ms = timeit(p, buf, buf, 0, 0);
            std::printf("  3D D2Z in-place            %8.3f ms  (%.0f GB/s at 2 x array)\n", ms,
                        2 * GB / (ms * 1e-3));
            CK(cufftDestroy(p));
            CK(cufftCreate(&p));
            CK(cufftMakePlan3d(p, D, D, D, CUFFT_Z2D, &ws));
            ms = timeit(p, buf, buf, 1, 0);
            std::printf("  3D Z2D in-place            %8.3f ms\n", ms);
            CK(cufftDestroy(p));
            CK(cufftCreate(&p));
            CK(cufftMakePlan3d(p, D, D, D, CUFFT_D2Z, &ws));
            ms = timeit(p, buf2, buf, 0, 0);
            std::printf("  3D D2Z out-of-place        %8.3f ms\n", ms);
            CK(cufftDestroy(p));
        }
        // 2D D2Z in place, batch Mt planes
        {
            long long n[2] = {D, D};
            CK(cufftCreate(&p));
            CK(cufftMakePlanMany64(p, 2, n, nullptr, 1, 0, nullptr, 1, 0, CUFFT_D2Z, Mt, &ws));
            float ms = timeit(p, buf, buf, 0, 0);
            std::printf("  2D D2Z batch Mt in-place   %8.3f ms\n", ms);
            CK(cufftDestroy(p));
            CK(cufftCreate(&p));
            CK(cufftMakePlanMany64(p, 2, n, nullptr, 1, 0, nullptr, 1, 0, CUFFT_Z2D, Mt, &ws));
            ms = timeit(p, buf, buf, 1, 0);
            std::printf("  2D Z2D batch Mt in-place   %8.3f ms\n", ms);
            CK(cufftDestroy(p));
        }
        // 1D Z2Z along x: stride D*Dh, dist 1
        {
            long long n[1] = {D}, emb[1] = {D};
            const long long st = (long long)D * Dh;
            CK(cufftCreate(&p));
            CK(cufftMakePlanMany64(p, 1, n, emb, st, 1, emb, st, 1, CUFFT_Z2Z, st, &ws));
            float ms = timeit(p, buf, buf, 2, CUFFT_FORWARD);
            std::printf("  1D Z2Z x strided in-place  %8.3f ms  (ws %.2f GB)\n", ms, ws / 1e9);
            ms = timeit(p, buf, buf2, 2, CUFFT_FORWARD);
            std::printf("  1D Z2Z x strided out       %8.3f ms\n", ms);
            CK(cufftDestroy(p));
        }
        // 1D Z2Z contiguous batched (as if x were innermost)
        {
            long long n[1] = {D};
            const long long batch = (long long)D * Dh;
            CK(cufftCreate(&p));
            CK(cufftMakePlanMany64(p, 1, n, nullptr, 1, D, nullptr, 1, D, CUFFT_Z2Z, batch, &ws));
            float ms = timeit(p, buf, buf, 2, CUFFT_FORWARD);
            std::printf("  1D Z2Z contiguous batched  %8.3f ms\n", ms);
            CK(cufftDestroy(p));
        }
        // 1D Z2Z along y within a plane set: stride Dh, dist 1, batch Dh, for Mt planes
        {
            long long n[1] = {D}, emb[1] = {D};
            CK(cufftCreate(&p));
            CK(cufftMakePlanMany64(p, 1, n, emb, Dh, 1, emb, Dh, 1, CUFFT_Z2Z, Dh, &ws));
            float ms = timeit(p, buf, buf, 2, CUFFT_FORWARD);
            std::printf("  1D Z2Z y one plane         %8.3f ms (x Mt = %.3f)\n", ms, ms * Mt);
            CK(cufftDestroy(p));
        }
        // 1D D2Z along z, contiguous rows, batch Mt*Mt (pruned first pass)
        {
            long long n[1] = {D};
            CK(cufftCreate(&p));
            CK(cufftMakePlanMany64(p, 1, n, nullptr, 1, 0, nullptr, 1, 0, CUFFT_D2Z,
                                   (long long)Mt * D, &ws));
            float ms = timeit(p, buf, buf, 0, 0);
            std::printf("  1D D2Z z rows batch Mt*D   %8.3f ms\n", ms);
            CK(cufftDestroy(p));
        }
        cudaFree(buf);
        cudaFree(buf2);
    }
    return 0;
}
