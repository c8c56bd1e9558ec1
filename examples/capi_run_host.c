/* A plain-C caller of the drop-in boundary (include/fireiron_b200.h): the
 * anvil::run path of the reference (proj/include/anvil/sim.hpp:495) as a
 * C-ABI call. Parses a Fireiron strategy, creates the plan for the device,
 * runs it on host fp32 matrices (integer-valued, so every strategy is exact)
 * and compares with a naive fp64 GEMM.
 *
 *   gcc -std=c11 -O2 -I include examples/capi_run_host.c \
 *       -L paper_2003_06324_b200/_lib -lfireiron_b200 -o capi_run_host
 *   ./capi_run_host            # needs a B200
 *   ./capi_run_host --parse    # CPU only: parse/validate/print the strategy
 */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "fireiron_b200.h"

static const char* kScript =
    "spec MatMul(1024,1024,512)(GL,GL,GL)(Kernel) elems f16 f16 f32\n"
    "\n"
    "tile 256 256 .to block .pair\n"
    "epilog tm {\n"
    "  init {\n"
    "    done\n"
    "  }\n"
    "  store {\n"
    "    tile 32 256 .to warp\n"
    "    done\n"
    "  }\n"
    "}\n"
    "split 64\n"
    "load a sh {\n"
    "  done\n"
    "}\n"
    "load b sh {\n"
    "  done\n"
    "}\n"
    "done\n";

int main(int argc, char** argv) {
    char buf[4096];
    if (argc > 1 && strcmp(argv[1], "--parse") == 0) {
        int64_t n = fi_script_validate(kScript, 0, 0, 0, buf, sizeof buf);
        if (n < 0) {
            fprintf(stderr, "validate failed: %s\n", fi_last_error());
            return 1;
        }
        printf("%s\n", buf);
        return 0;
    }
    const int64_t m = 1024, n = 1024, k = 512;
    fi_plan plan = NULL;
    fi_status st = fi_plan_create(kScript, 0, 0, 0, 0, 0, &plan);
    if (st != FI_OK) {
        fprintf(stderr, "fi_plan_create: status %d: %s\n", st, fi_last_error());
        return 1;
    }
    fi_plan_info info;
    fi_plan_query(plan, &info);
    /* column-major roots (Fireiron's default): A(i, p) at A[i + p * m] */
    float* A = malloc(sizeof(float) * m * k);
    float* B = malloc(sizeof(float) * k * n);
    float* C = malloc(sizeof(float) * m * n);
    for (int64_t i = 0; i < m * k; ++i) A[i] = (float)((i * 7 + 3) % 7 - 3);
    for (int64_t i = 0; i < k * n; ++i) B[i] = (float)((i * 5 + 1) % 7 - 3);
    st = fi_plan_run_host(plan, A, B, C);
    if (st != FI_OK) {
        fprintf(stderr, "fi_plan_run_host: status %d: %s\n", st, fi_last_error());
        return 1;
    }
    int64_t up = 0, down = 0;
    fi_plan_host_bytes(plan, &up, &down);
    double max_err = 0;
    for (int64_t j = 0; j < n; j += 7)
        for (int64_t i = 0; i < m; i += 3) {
            double acc = 0;
            for (int64_t p = 0; p < k; ++p) acc += (double)A[i + p * m] * (double)B[p + j * k];
            double e = acc - (double)C[i + j * m];
            if (e < 0) e = -e;
            if (e > max_err) max_err = e;
        }
    printf("%s: tile %dx%d cta_group %d, %lld CTAs; H2D %lld B, D2H %lld B; max_abs_error=%g\n", info.entry_name,
           info.tile_m, info.tile_n, info.cta_group, (long long)info.launch_ctas, (long long)up, (long long)down,
           max_err);
    fi_plan_destroy(plan);
    free(A);
    free(B);
    free(C);
    return max_err == 0 ? 0 : 2;
}
