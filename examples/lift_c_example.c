/* Using liblift.so from plain C (no Python, no torch): the C ABI of include/lift.h.
 *
 *   gcc -O2 -I include -I /usr/local/cuda/include examples/lift_c_example.c \
 *       -L paper_1502_02389_b200 -llift -L /usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_1502_02389_b200 -o build/lift_c_example
 *   ./build/lift_c_example
 *
 * Computes asum, dot, scal and gemv on small integer-valued inputs whose results are
 * exact, and checks them against closed forms.  Exit code 0 = all correct. */
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include "lift.h"

#define CHECK(x)                                                                     \
    do {                                                                             \
        lift_status s_ = (x);                                                        \
        if (s_ != LIFT_OK) {                                                         \
            fprintf(stderr, "%s:%d %s -> %s\n", __FILE__, __LINE__, #x, lift_status_string(s_)); \
            return 1;                                                                \
        }                                                                            \
    } while (0)

int main(void) {
    const int64_t n = 1000003, m = 300, k = 513;
    float *hx = malloc(n * sizeof(float)), *hA = malloc(m * k * sizeof(float));
    float *hv = malloc(k * sizeof(float)), *hw = malloc(m * sizeof(float));
    for (int64_t i = 0; i < n; ++i) hx[i] = (float)((i % 7) - 3);      /* -3..3 */
    for (int64_t i = 0; i < m * k; ++i) hA[i] = (float)(i % 5);        /* 0..4 */
    for (int64_t j = 0; j < k; ++j) hv[j] = 1.0f;
    for (int64_t i = 0; i < m; ++i) hw[i] = 2.0f;

    float *x, *y, *A, *v, *w, *wo, *res;
    void* ws;
    const size_t wsb = lift_workspace_bytes(n);
    cudaMalloc((void**)&x, n * 4);
    cudaMalloc((void**)&y, n * 4);
    cudaMalloc((void**)&A, m * k * 4);
    cudaMalloc((void**)&v, k * 4);
    cudaMalloc((void**)&w, m * 4);
    cudaMalloc((void**)&wo, m * 4);
    cudaMalloc((void**)&res, 2 * 4);
    cudaMalloc(&ws, wsb);
    cudaMemset(ws, 0, wsb); /* zero-filled once (lift.h workspace contract) */
    cudaMemcpy(x, hx, n * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(A, hA, m * k * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(v, hv, k * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(w, hw, m * 4, cudaMemcpyHostToDevice);

    CHECK(lift_asum(n, x, res, ws, wsb, NULL));
    CHECK(lift_scal(n, 2.0f, x, y, NULL));
    CHECK(lift_dot(n, x, y, res + 1, ws, wsb, NULL));
    CHECK(lift_gemv(m, k, 1.5f, A, k, v, 0.5f, w, wo, NULL));
    CHECK(lift_workspace_check(ws, wsb, NULL));  /* the tickets are back at zero */
    float hr[2], hwo[3];
    cudaMemcpy(hr, res, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(hwo, wo, 12, cudaMemcpyDeviceToHost);

    double asum = 0, dot = 0;
    for (int64_t i = 0; i < n; ++i) {
        asum += hx[i] < 0 ? -hx[i] : hx[i];
        dot += 2.0 * hx[i] * hx[i];
    }
    int ok = (hr[0] == (float)asum) && (hr[1] == (float)dot);
    for (int i = 0; i < 3; ++i) {
        double d = 0;
        for (int64_t j = 0; j < k; ++j) d += hA[i * k + j];
        ok = ok && (hwo[i] == (float)(1.5 * d + 0.5 * 2.0));
    }
    printf("asum %.1f (exact %.1f)  dot %.1f (exact %.1f)  gemv[0..2] %.1f %.1f %.1f  -> %s\n",
           hr[0], asum, hr[1], dot, hwo[0], hwo[1], hwo[2], ok ? "OK" : "MISMATCH");
    return ok ? 0 : 1;
}
