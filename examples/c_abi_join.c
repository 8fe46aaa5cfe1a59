/*
 * c_abi_join.c -- the drop-in boundary used from plain C (no Python, no
 * torch): an FK join of |R| x 4|R| through include/mpsm_b200.h, checked
 * against a direct host computation (R keys are a permutation of 1..|R|, so
 * every S tuple matches R[key - 1]).
 *
 *   gcc -O2 examples/c_abi_join.c -Iinclude -I/usr/local/cuda/include \
 *       -Lpaper_1207_0145_b200 -lmpsm_b200 -L/usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_1207_0145_b200 -o c_abi_join && ./c_abi_join 1000000
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "mpsm_b200.h"

static uint64_t mix64(uint64_t z) { /* splitmix64 finalizer */
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static uint64_t rotl(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }

#define CK(x)                                                                      \
    do {                                                                           \
        int rc_ = (x);                                                             \
        if (rc_ != MPSM_OK) {                                                      \
            fprintf(stderr, "%s -> %d: %s\n", #x, rc_, mpsm_last_error());         \
            return 1;                                                              \
        }                                                                          \
    } while (0)
#define CU(x)                                                                      \
    do {                                                                           \
        if ((x) != cudaSuccess) {                                                  \
            fprintf(stderr, "%s failed\n", #x);                                    \
            return 1;                                                              \
        }                                                                          \
    } while (0)

int main(int argc, char** argv) {
    const int64_t nr = argc > 1 ? atoll(argv[1]) : 1000000, ns = 4 * nr;
    if (mpsm_device_init(0) < 0) {
        fprintf(stderr, "no sm_100 device: %s\n", mpsm_last_error());
        return 1;
    }
    /* host relations: R keys = a permutation of 1..nr, S keys uniform over them */
    uint64_t *rk = malloc(8 * nr), *rp = malloc(8 * nr), *sk = malloc(8 * ns), *sp = malloc(8 * ns);
    for (int64_t i = 0; i < nr; ++i) rk[i] = (uint64_t)i + 1;
    for (int64_t i = nr - 1; i > 0; --i) { /* Fisher-Yates with a counter-based draw */
        const int64_t j = (int64_t)(mix64((uint64_t)i * 7 + 1) % (uint64_t)(i + 1));
        const uint64_t t = rk[i];
        rk[i] = rk[j];
        rk[j] = t;
    }
    for (int64_t i = 0; i < nr; ++i) rp[i] = mix64((uint64_t)i + 11) & 0xffffffffull;
    for (int64_t i = 0; i < ns; ++i) {
        sk[i] = 1 + mix64((uint64_t)i * 3 + 5) % (uint64_t)nr;
        sp[i] = mix64((uint64_t)i + 13) & 0xffffffffull;
    }
    /* expected: every S tuple matches the R tuple with its key */
    uint64_t *pay_of = malloc(8 * (nr + 1)), want_max = 0, want_sum = 0;
    for (int64_t i = 0; i < nr; ++i) pay_of[rk[i]] = rp[i];
    for (int64_t i = 0; i < ns; ++i) {
        const uint64_t r = pay_of[sk[i]], v = r + sp[i];
        want_max = v > want_max ? v : want_max;
        want_sum += mix64(r ^ rotl(sp[i], 17));
    }
    int width = 0;
    while (((uint64_t)1 << width) < (uint64_t)nr) ++width; /* keys - 1 in [0, nr) */
    if (width == 0) width = 1; /* packed records need at least one key bit */
    const uint64_t lower = 1, span_m1 = (uint64_t)nr - 1;

    /* device copies, packed sorted runs */
    uint64_t *d_rk, *d_rp, *d_sk, *d_sp, *d_r, *d_s, *d_tmp, *d_rec;
    unsigned long long* d_bad;
    unsigned int* d_ovf;
    CU(cudaMalloc((void**)&d_rk, 8 * nr));
    CU(cudaMalloc((void**)&d_rp, 8 * nr));
    CU(cudaMalloc((void**)&d_sk, 8 * ns));
    CU(cudaMalloc((void**)&d_sp, 8 * ns));
    CU(cudaMalloc((void**)&d_r, 8 * nr));
    CU(cudaMalloc((void**)&d_s, 8 * ns));
    CU(cudaMalloc((void**)&d_tmp, 8 * ns));
    CU(cudaMalloc((void**)&d_rec, 8 * MPSM_PAIR_FIELDS));
    CU(cudaMalloc((void**)&d_bad, 8));
    CU(cudaMalloc((void**)&d_ovf, 4));
    CU(cudaMemcpy(d_rk, rk, 8 * nr, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(d_rp, rp, 8 * nr, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(d_sk, sk, 8 * ns, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(d_sp, sp, 8 * ns, cudaMemcpyHostToDevice));
    CU(cudaMemset(d_bad, 0xff, 8));
    CU(cudaMemset(d_ovf, 0, 4));
    size_t ws_bytes = 0;
    CK(mpsm_sort_workspace_bytes(ns, width, &ws_bytes));
    void* ws;
    CU(cudaMalloc(&ws, ws_bytes));
    CK(mpsm_sort_packed(d_rk, d_rp, nr, lower, span_m1, width, d_r, d_tmp, ws, ws_bytes, d_bad, d_ovf, NULL));
    CK(mpsm_sort_packed(d_sk, d_sp, ns, lower, span_m1, width, d_s, d_tmp, ws, ws_bytes, d_bad, d_ovf, NULL));

    /* merge join of the one private run against the one public run */
    mpsm_run_t priv = {d_r, NULL, nr}, pub = {d_s, NULL, ns};
    size_t jws_bytes = 0;
    CK(mpsm_join_workspace_bytes(&priv, 1, &pub, 1, &jws_bytes));
    void* jws;
    CU(cudaMalloc(&jws, jws_bytes));
    CK(mpsm_join_pairs_packed(&priv, 1, &pub, 1, width, lower, 0, MPSM_MODE_AGGREGATE_MAX, NULL, 0, d_rec, jws,
                              jws_bytes, NULL));
    uint64_t rec[MPSM_PAIR_FIELDS];
    unsigned long long bad;
    unsigned int ovf;
    CU(cudaMemcpy(rec, d_rec, sizeof(rec), cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(&bad, d_bad, 8, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(&ovf, d_ovf, 4, cudaMemcpyDeviceToHost));
    const int ok = bad == ~0ull && ovf == 0 && rec[MPSM_PAIR_COUNT] == (uint64_t)ns && rec[MPSM_PAIR_BEST] == want_max &&
                   rec[MPSM_PAIR_CHECKSUM] == want_sum;
    printf("count %llu max %llu checksum 0x%016llx probes %llu examined %llu -> %s\n",
           (unsigned long long)rec[MPSM_PAIR_COUNT], (unsigned long long)rec[MPSM_PAIR_BEST],
           (unsigned long long)rec[MPSM_PAIR_CHECKSUM], (unsigned long long)rec[MPSM_PAIR_PROBES],
           (unsigned long long)rec[MPSM_PAIR_EXAMINED], ok ? "OK" : "MISMATCH");
    return ok ? 0 : 2;
}
