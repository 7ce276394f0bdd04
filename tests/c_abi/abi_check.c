/*
 * abi_check.c -- a plain C99 caller of include/dvm.h (no Python, no torch):
 * dvm_plan -> dvm_collide -> dvm_plan_destroy, the calls BASELINE.json's
 * north_star names, on a stored input, compared with a stored oracle output
 * (tests/golden/abi_*.bin, written by tools/make_abi_golden.py, which calls
 * only oracle/ and dvm_inputs).  Also exercises dvm_collide_batched and the
 * documented error codes.
 *
 * usage: abi_check d N Nbar f.bin q_oracle.bin      exit 0 = pass
 * build: gcc -std=c99 -I include abi_check.c -L<dir of libdvm.so> -ldvm -lcudart
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "dvm.h"

static double *read_bin(const char *path, size_t n)
{
    FILE *fp = fopen(path, "rb");
    if (!fp) return NULL;
    double *x = (double *)malloc(sizeof(double) * n);
    size_t got = x ? fread(x, sizeof(double), n, fp) : 0;
    fclose(fp);
    if (got != n) {
        free(x);
        return NULL;
    }
    return x;
}

#define EXPECT(cond, msg)                                  \
    do {                                                   \
        if (!(cond)) {                                     \
            fprintf(stderr, "FAIL: %s (%s)\n", msg, dvm_last_error()); \
            return 1;                                      \
        }                                                  \
    } while (0)

int main(int argc, char **argv)
{
    if (argc != 6) {
        fprintf(stderr, "usage: %s d N Nbar f.bin q_oracle.bin\n", argv[0]);
        return 2;
    }
    const int d = atoi(argv[1]), N = atoi(argv[2]), Nbar = atoi(argv[3]);
    size_t nodes = 1;
    for (int j = 0; j < d; ++j) nodes *= (size_t)N;
    double *f = read_bin(argv[4], nodes), *qo = read_bin(argv[5], nodes);
    EXPECT(f && qo, "reading the golden files");
    EXPECT(dvm_abi_version() == DVM_ABI_VERSION, "ABI version");

    dvm_plan_t plan = NULL;
    const dvm_kernel_t kern = d == 2 ? DVM_MAXWELL_2D : DVM_HARD_SPHERES_3D;
    EXPECT(dvm_plan(d, N, Nbar, kern, &plan) == DVM_OK && plan, "dvm_plan");

    double *f_d = NULL, *q_d = NULL, *q2_d = NULL;
    EXPECT(cudaMalloc((void **)&f_d, sizeof(double) * nodes * 2) == cudaSuccess, "cudaMalloc f");
    EXPECT(cudaMalloc((void **)&q_d, sizeof(double) * nodes) == cudaSuccess, "cudaMalloc Q");
    EXPECT(cudaMalloc((void **)&q2_d, sizeof(double) * nodes * 2) == cudaSuccess, "cudaMalloc Q2");
    EXPECT(cudaMemcpy(f_d, f, sizeof(double) * nodes, cudaMemcpyHostToDevice) == cudaSuccess, "H2D");
    EXPECT(cudaMemcpy(f_d + nodes, f, sizeof(double) * nodes, cudaMemcpyHostToDevice) == cudaSuccess, "H2D 2");

    EXPECT(dvm_collide(plan, f_d, q_d) == DVM_OK, "dvm_collide");
    EXPECT(dvm_sync(plan) == DVM_OK, "dvm_sync");
    double *q = (double *)malloc(sizeof(double) * nodes);
    EXPECT(cudaMemcpy(q, q_d, sizeof(double) * nodes, cudaMemcpyDeviceToHost) == cudaSuccess, "D2H");
    double err = 0.0, scale = 0.0;
    for (size_t i = 0; i < nodes; ++i) {
        const double e = fabs(q[i] - qo[i]);
        if (e > err) err = e;
        if (fabs(qo[i]) > scale) scale = fabs(qo[i]);
    }
    printf("d=%d N=%d Nbar=%d: max|Q - Q_oracle| / max|Q_oracle| = %.3e\n", d, N, Nbar, err / scale);
    EXPECT(err <= 1e-11 * scale, "parity with the stored oracle output (1e-11 of max|Q_oracle|)");

    /* the same cell twice through dvm_collide_batched: both copies equal Q to rounding */
    EXPECT(dvm_collide_batched(plan, f_d, q2_d, 2, 0) == DVM_OK, "dvm_collide_batched");
    EXPECT(dvm_sync(plan) == DVM_OK, "dvm_sync (batched)");
    double *q2 = (double *)malloc(sizeof(double) * nodes * 2);
    EXPECT(cudaMemcpy(q2, q2_d, sizeof(double) * nodes * 2, cudaMemcpyDeviceToHost) == cudaSuccess, "D2H 2");
    for (size_t i = 0; i < 2 * nodes; ++i) EXPECT(fabs(q2[i] - qo[i % nodes]) <= 1e-11 * scale, "batched parity");

    /* documented error codes */
    dvm_plan_t bad = NULL;
    EXPECT(dvm_plan(4, N, Nbar, kern, &bad) == DVM_E_DIM && !bad, "DVM_E_DIM");
    EXPECT(dvm_plan(d, N, Nbar, d == 2 ? DVM_HARD_SPHERES_3D : DVM_MAXWELL_2D, &bad) == DVM_E_KERNEL, "DVM_E_KERNEL");
    EXPECT(dvm_plan(d, N, 0, kern, &bad) == DVM_E_ORDER, "DVM_E_ORDER");
    EXPECT(dvm_collide(plan, NULL, q_d) == DVM_E_NULL, "DVM_E_NULL");
    EXPECT(dvm_collide(plan, f_d, f_d) == DVM_E_ALIAS, "DVM_E_ALIAS");
    EXPECT(dvm_collide_batched(plan, f_d, q2_d, -1, 0) == DVM_E_SHAPE, "DVM_E_SHAPE");
    EXPECT(strcmp(dvm_status_str(DVM_OK), "DVM_OK") == 0, "dvm_status_str");

    EXPECT(dvm_plan_destroy(plan) == DVM_OK, "dvm_plan_destroy");
    cudaFree(f_d);
    cudaFree(q_d);
    cudaFree(q2_d);
    free(f);
    free(qo);
    free(q);
    free(q2);
    printf("abi_check ok\n");
    return 0;
}
