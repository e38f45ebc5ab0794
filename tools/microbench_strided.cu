// Microbenchmark of the strided T2 sweep variants on a config-5-sized grid (tuning tool,
// not part of the product).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -o /tmp/mb tools/microbench_strided.cu
// Run: /tmp/mb [N_cells=256] [n=3]
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1702_00169_b200/csrc/pdg_kernels.cuh"
#include "../paper_1702_00169_b200/csrc/pdg_tables.hpp"

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e = (x);                                                                    \
        if (e != cudaSuccess) {                                                                 \
            printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));                  \
            exit(1);                                                                            \
        }                                                                                       \
    } while (0)

__global__ void init_kernel(double *f, size_t n)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        f[i] = 1.0 + 1e-3 * (double)(i % 977);
}

using namespace pdg;

template <typename F>
float time_it(F launch, int reps)
{
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) launch();
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    CK(cudaGetLastError());
    return ms / reps;
}

template <int n>
void run(int Nc)
{
    const int64_t L = (int64_t)Nc * n;
    const int64_t nnodes = L * L * L;
    const int nvel = 16;  // 8 along y, 8 along z
    const size_t total = (size_t)nvel * nnodes;
    double *f, *fb;
    CK(cudaMalloc(&f, total * sizeof(double)));
    CK(cudaMalloc(&fb, (size_t)nvel * L * L * sizeof(double)));
    init_kernel<<<4096, 256>>>(f, total);
    init_kernel<<<256, 256>>>(fb, (size_t)nvel * L * L);
    CK(cudaDeviceSynchronize());
    SweepParams P;
    memset(&P, 0, sizeof(P));
    P.f = f;
    P.fb = fb;
    CellBlock cb;
    cell_block(n - 1, 1.0L, &cb);
    for (int d = 0; d < 3; ++d) {
        for (int i = 0; i < n * n; ++i) P.blk[d].M[i] = cb.M[i];
        for (int i = 0; i < n; ++i) P.blk[d].g[i] = cb.g[i];
    }
    auto setup = [&](int which_axes) {  // 1: y only, 2: z only, 3: both
        P.nvel = 0;
        for (int j = 0; j < nvel; ++j) {
            const int k = (j < 8) ? 1 : 2;
            if (!((which_axes >> (k - 1)) & 1)) continue;
            SweepVel V{};
            V.f_off = (int64_t)j * nnodes;
            V.fb_off = (int64_t)j * L * L;
            V.inner = (k == 1) ? L : L * L;
            V.nlines = nnodes / L;
            V.ncells = Nc;
            V.sign = (j % 2) ? -1 : 1;
            V.axis = k;
            V.vel = j;
            P.v[P.nvel++] = V;
        }
    };
    const int reps = 3;
    for (int axes = 3; axes <= 3; ++axes) {
        setup(axes);
        const double bytes = 16.0 * (double)P.nvel * (double)nnodes;
        const int64_t nl = nnodes / L;
#define RUN1(NP, PF, TPB)                                                                          \
    {                                                                                              \
        dim3 grid((unsigned)((nl + TPB - 1) / TPB), (unsigned)P.nvel);                             \
        float ms = time_it([&] { sweep_strided_kernel<n, NP, PF><<<grid, TPB>>>(P); }, reps);      \
        printf("n=%d axes=%d scalar  NPASS=%d PF=%d TPB=%d : %8.3f ms %7.0f GB/s\n", n, axes, NP, PF, TPB, ms, \
               bytes / ms / 1e6);                                                                  \
    }
        RUN1(1, 1, 256);
        RUN1(1, 2, 256);
        RUN1(1, 3, 256);
        RUN1(2, 1, 256);
        RUN1(2, 2, 256);
        RUN1(2, 3, 256);
        RUN1(2, 2, 128);
    }
    cudaFree(f);
    cudaFree(fb);
}

int main(int argc, char **argv)
{
    run<3>(argc > 1 ? atoi(argv[1]) : 256);
    run<4>(argc > 2 ? atoi(argv[2]) : 128);
    return 0;
}
