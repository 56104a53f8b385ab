/*
 * cfg1_graph.c -- BASELINE config 1 (vector add -> reduction)
 * through the C ABI only (include/jacc.h): no Python, no torch.
 *
 *   gcc -O2 -I include examples/cfg1_graph.c -L paper_1508_06791_b200 -ljacc \
 *       -Wl,-rpath,paper_1508_06791_b200 -o cfg1_graph
 *   ./cfg1_graph --plan    # build + plan + dump (no CUDA call, runs without a GPU)
 *   ./cfg1_graph           # execute on device 0, check c and s, print the stats
 *
 * The host buffers are plain malloc memory (pageable: the runtime copies them
 * synchronously enough for this demo; pinned memory lets copies overlap).
 */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "jacc.h"

#define CHECK(call)                                                                      \
    do {                                                                                 \
        int st_ = (call);                                                                \
        if (st_ != JACC_OK) {                                                            \
            fprintf(stderr, "%s failed: %s\n", #call, jacc_last_error());                \
            return 1;                                                                    \
        }                                                                                \
    } while (0)

int main(int argc, char **argv) {
    const int plan_only = argc > 1 && strcmp(argv[1], "--plan") == 0;
    const uint64_t n = 1u << 20;
    float *a = malloc(n * sizeof(float)), *b = malloc(n * sizeof(float)), *c = malloc(n * sizeof(float));
    float s = 0.f;
    if (!a || !b || !c) return 1;
    for (uint64_t i = 0; i < n; ++i) {   /* a[i] + b[i] = n exactly (SURVEY §8(c)-V pin) */
        a[i] = (float)i;
        b[i] = (float)(n - i);
    }

    jacc_config_t cfg;
    memset(&cfg, 0, sizeof cfg);
    cfg.device = 0;
    cfg.world = 1;
    jacc_graph_t *g = NULL;
    CHECK(jacc_graph_create(&g, &cfg));

    jacc_arg_t vadd[3] = {{a, n, JACC_F32, JACC_READ, 0, 0},
                          {b, n, JACC_F32, JACC_READ, 0, 0},
                          {c, n, JACC_F32, JACC_WRITE, 0, 0}};
    jacc_arg_t red[2] = {{c, n, JACC_F32, JACC_READ, 0, 0}, {&s, 1, JACC_F32, JACC_WRITE, 0, 0}};
    int t0 = -1, t1 = -1;
    CHECK(jacc_graph_add_task(g, JACC_OP_VADD_F32, vadd, 3, NULL, 0, NULL, 0, &t0));
    CHECK(jacc_graph_add_task(g, JACC_OP_REDUCE_SUM_F32, red, 2, NULL, 0, NULL, 0, &t1));

    if (plan_only) {
        size_t need = 0;
        CHECK(jacc_graph_dump(g, NULL, 0, &need));
        char *buf = malloc(need);
        CHECK(jacc_graph_dump(g, buf, need, &need));
        fputs(buf, stdout);
        free(buf);
    } else {
        CHECK(jacc_graph_execute(g));
        CHECK(jacc_graph_sync(g));
        for (uint64_t i = 0; i < n; ++i)
            if (c[i] != (float)n) {
                fprintf(stderr, "c[%llu] = %g, want %llu\n", (unsigned long long)i, c[i], (unsigned long long)n);
                return 2;
            }
        /* sum of n copies of n = n^2 = 2^40: exact in fp32 for a power of two */
        if (s != (float)n * (float)n) {
            fprintf(stderr, "s = %g, want %g\n", s, (double)n * (double)n);
            return 3;
        }
        jacc_stats_t st;
        CHECK(jacc_graph_stats(g, &st));
        float ms = 0.f;
        CHECK(jacc_graph_task_ms(g, t0, &ms));
        printf("ok: c = %g everywhere, s = %g; h2d %llu (%llu B), d2h %llu (%llu B), kernels %llu, vadd %.3f ms\n",
               c[0], s, (unsigned long long)st.h2d_count, (unsigned long long)st.h2d_bytes,
               (unsigned long long)st.d2h_count, (unsigned long long)st.d2h_bytes, (unsigned long long)st.kernels, ms);
    }
    CHECK(jacc_graph_destroy(g));
    free(a);
    free(b);
    free(c);
    return 0;
}
