// Calls libm4d's transpose_sum ABI directly (no Python) and reports whether the kernel completes.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <unistd.h>
#include <cuda_runtime.h>
#include "m4d.h"

int main(int argc, char** argv) {
    int n = argc > 1 ? atoi(argv[1]) : 256, b = argc > 2 ? atoi(argv[2]) : 64;
    int nb = n / b;
    double *x, *y, *sums;
    size_t bb = (size_t)b * b;
    cudaMalloc(&x, bb * nb * nb * 8);
    cudaMalloc(&y, bb * nb * nb * 8);
    cudaMalloc(&sums, (nb * nb + 1) * 8);
    void* st;
    m4d_stream_create(0, &st);
    for (int g = 0; g < nb * nb; ++g) m4d_fill_block_f64(x + g * bb, n, (g / nb) * b, (g % nb) * b, b, 0x210108878ull, st);
    std::vector<m4d_ts_task> tasks;
    for (int i = 0; i < nb; ++i)
        for (int j = i; j < nb; ++j) {
            m4d_ts_task t{};
            t.a = x + (i * nb + j) * bb;
            t.bt = x + (j * nb + i) * bb;
            t.y = y + (i * nb + j) * bb;
            t.slot_y = i * nb + j;
            t.slot_y2 = -1;
            if (i == j) t.diag = 1;
            else { t.y2 = y + (j * nb + i) * bb; t.slot_y2 = j * nb + i; }
            tasks.push_back(t);
        }
    m4d_ts_plan* plan;
    if (m4d_ts_plan_create(0, tasks.data(), (int)tasks.size(), b, nb * nb, &plan)) { char e[512]; m4d_last_error(e, 512); printf("plan: %s\n", e); return 1; }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 3; ++rep) m4d_ts_run(plan, sums, sums + nb * nb, st);
    cudaEventRecord(e0, (cudaStream_t)st);
    for (int rep = 0; rep < 10; ++rep) m4d_ts_run(plan, sums, sums + nb * nb, st);
    cudaEventRecord(e1, (cudaStream_t)st);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("avg %.3f ms per run  (%.1f GB/s algorithmic)\n", ms / 10, 16.0 * n * (double)n / (ms / 10 * 1e-3) / 1e9);
    for (int rep = 0; rep < 1; ++rep) {
        int rc = m4d_ts_run(plan, sums, sums + nb * nb, st);
        printf("run %d rc %d\n", rep, rc); fflush(stdout);
        int waited = 0;
        cudaError_t q;
        while ((q = cudaStreamQuery((cudaStream_t)st)) == cudaErrorNotReady && waited < 10000) { usleep(1000); ++waited; }
        printf("  query after %d ms: %s\n", waited, cudaGetErrorString(q)); fflush(stdout);
        if (q != cudaSuccess) return 2;
        double tot;
        cudaMemcpy(&tot, sums + nb * nb, 8, cudaMemcpyDeviceToHost);
        printf("  total %.17g\n", tot);
    }
    return 0;
}
