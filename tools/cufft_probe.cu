// probe: which cuFFT plans for the sM^3 Green's precompute does the system
// cuFFT (CUDA 12.9) accept on B200?  nvcc -o cufft_probe cufft_probe.cu -lcufft
#include <cufft.h>
#include <cuda_runtime.h>
#include <cstdio>
int main(int argc, char** argv) {
    long long sM = argc > 1 ? atoll(argv[1]) : 1640;
    int ver = 0;
    cufftGetVersion(&ver);
    printf("cufft version %d, sM %lld\n", ver, sM);
    size_t freeb, totb;
    cudaMemGetInfo(&freeb, &totb);
    printf("free %.1f GB\n", freeb / 1e9);
    {
        cufftHandle p;
        cufftCreate(&p);
        size_t ws = 0;
        long long n[3] = {sM, sM, sM};
        cufftResult r = cufftMakePlanMany64(p, 3, n, nullptr, 1, 0, nullptr, 1, 0, CUFFT_Z2D, 1, &ws);
        printf("3d Z2D planmany64: %d ws %.2f GB\n", r, ws / 1e9);
        cufftDestroy(p);
    }
    {
        cufftHandle p;
        cufftCreate(&p);
        cufftSetAutoAllocation(p, 0);
        size_t ws = 0;
        long long n[3] = {sM, sM, sM};
        cufftResult r = cufftMakePlanMany64(p, 3, n, nullptr, 1, 0, nullptr, 1, 0, CUFFT_Z2D, 1, &ws);
        printf("3d Z2D planmany64 (no autoalloc): %d ws %.2f GB\n", r, ws / 1e9);
        cufftDestroy(p);
    }
    {
        cufftHandle p;
        cufftCreate(&p);
        size_t ws = 0;
        cufftResult r = cufftMakePlan3d(p, (int)sM, (int)sM, (int)sM, CUFFT_Z2D, &ws);
        printf("3d Z2D plan3d: %d ws %.2f GB\n", r, ws / 1e9);
        cufftDestroy(p);
    }
    {
        // 2D Z2Z over (x, y) for each kz column: batch sM/2+1, strided
        cufftHandle p;
        cufftCreate(&p);
        size_t ws = 0;
        long long n[2] = {sM, sM};
        long long h = sM / 2 + 1;
        long long emb[2] = {sM, sM};
        cufftResult r = cufftMakePlanMany64(p, 2, n, emb, h, 1, emb, h, 1, CUFFT_Z2Z, h, &ws);
        printf("2d Z2Z batched (stride h): %d ws %.2f GB\n", r, ws / 1e9);
        cufftDestroy(p);
    }
    {
        long long n[1] = {sM};
        cufftHandle p;
        cufftCreate(&p);
        size_t ws = 0;
        long long h = sM / 2 + 1;
        long long ie[1] = {h}, oe[1] = {2 * h};
        cufftResult r = cufftMakePlanMany64(p, 1, n, ie, 1, h, oe, 1, 2 * h, CUFFT_Z2D, sM * sM, &ws);
        printf("1d Z2D batched: %d ws %.2f GB\n", r, ws / 1e9);
        cufftDestroy(p);
    }
    return 0;
}
