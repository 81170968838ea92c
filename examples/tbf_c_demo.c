/*
 * Plain-C consumer of the C ABI (no Python, no torch): box-window trig
 * bilateral filter of a synthetic H x W image through the host entry.
 *
 *   gcc -O2 examples/tbf_c_demo.c -I include -I $CUDA_HOME/include \
 *       -L paper_1105_4204_b200/_lib -ltrigbf_b200 -L $CUDA_HOME/lib64 -lcudart -lm \
 *       -Wl,-rpath,paper_1105_4204_b200/_lib -o tbf_c_demo
 *   ./tbf_c_demo H W RADIUS SIGMA_R DEGREE out.f32
 *
 * The raised-cosine expansion is built here the way the reference does it
 * (kernels.py:107-158, engines.py:249-253): omega = 1/(sigma_r sqrt(N)),
 * weights 2^-N C(N, n), folded into pairs nu = (2n - N) omega, n > N/2, with
 * weight 2 c_n, plus the zero frequency c_{N/2} for even N.
 */
#include <cuda_runtime_api.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "trigbf_b200.h"

int main(int argc, char** argv) {
    if (argc != 7) {
        fprintf(stderr, "usage: %s H W RADIUS SIGMA_R DEGREE out.f32\n", argv[0]);
        return 2;
    }
    const int H = atoi(argv[1]), W = atoi(argv[2]), radius = atoi(argv[3]), N = atoi(argv[5]);
    const double sigma_r = atof(argv[4]), T = 255.0;
    const size_t n = (size_t)H * W;

    /* terms: ascending nu, zero frequency first (even N) */
    double nu[512], wt[512];
    int nt = 0;
    const double omega = 1.0 / (sigma_r * sqrt((double)N));
    for (int k = N / 2; k <= N; ++k) {
        if (2 * k == N) {
            nu[nt] = 0.0;
            wt[nt++] = exp(lgamma(N + 1.0) - lgamma(k + 1.0) - lgamma(N - k + 1.0) - N * log(2.0));
        } else if (2 * k > N) {
            nu[nt] = (2.0 * k - N) * omega;
            wt[nt++] = 2.0 * exp(lgamma(N + 1.0) - lgamma(k + 1.0) - lgamma(N - k + 1.0) - N * log(2.0));
        }
    }
    tbf_terms terms = {nt, nu, wt, 2.0 * omega, T};
    tbf_spatial sp = {TBF_SPATIAL_BOX, radius, 0, 0, 0, 0, 0, 0, 0, 0};

    float* h_in = (float*)malloc(n * 4);
    float* h_out = (float*)malloc(n * 4);
    for (size_t i = 0; i < n; ++i) {  /* two flat regions plus a ramp */
        const size_t y = i / W, x = i % W;
        h_in[i] = (float)((x < (size_t)W / 2 ? 40.0 : 200.0) + 0.25 * (double)((x * 7 + y * 13) % 40));
    }
    const size_t ws_bytes = tbf_workspace_bytes(1, H, W, &sp, 0, nt, 0);
    void *ws = NULL, *io = NULL, *ctr = NULL;
    if (!ws_bytes || cudaMalloc(&ws, ws_bytes) || cudaMalloc(&io, 2 * n * 4) || cudaMalloc(&ctr, 16) ||
        cudaMemset(ctr, 0, 16)) {
        fprintf(stderr, "allocation failed: %s\n", tbf_last_error());
        return 1;
    }
    int rc = tbf_bilateral_trig_host(h_in, h_out, 1, H, W, &sp, &terms, 0, (float*)io, ws, ws_bytes,
                                     (unsigned long long*)ctr, NULL);
    unsigned long long counters[2] = {0, 0};
    if (!rc && cudaDeviceSynchronize() == cudaSuccess)
        cudaMemcpy(counters, ctr, 16, cudaMemcpyDeviceToHost);
    if (rc) {
        fprintf(stderr, "tbf_bilateral_trig_host: %d (%s)\n", rc, tbf_last_error());
        return 1;
    }
    FILE* fo = fopen(argv[6], "wb");
    if (!fo || fwrite(h_out, 4, n, fo) != n) return 1;
    fclose(fo);
    double sum = 0;
    for (size_t i = 0; i < n; ++i) sum += h_out[i];
    printf("abi=%d terms=%d out_of_range=%llu guarded=%llu mean=%.6f\n", tbf_abi_version(), nt,
           counters[0], counters[1], sum / (double)n);
    cudaFree(ws);
    cudaFree(io);
    cudaFree(ctr);
    free(h_in);
    free(h_out);
    return 0;
}
