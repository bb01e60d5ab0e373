/* A plain-C client of libuotk.so (the boundary of include/uotk.h, no Python, no torch):
 * reads a problem from raw little-endian fp64 files, calls the three SURVEY §8(b) entry
 * points on HOST buffers (the library stages the copies), writes the results.
 *
 *   uotk_c_client <dir>         reads <dir>/{meta.txt,x.bin,a.bin,y.bin,b.bin}
 *                               writes <dir>/{sum.bin,beta.bin,gamma.bin,scalars.txt}
 *   uotk_c_client --selftest    argument validation only (no GPU needed)
 */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "uotk.h"

static double* read_bin(const char* dir, const char* name, long count) {
    char path[1024];
    snprintf(path, sizeof path, "%s/%s", dir, name);
    FILE* f = fopen(path, "rb");
    if (!f) { fprintf(stderr, "cannot open %s\n", path); exit(2); }
    double* p = (double*)malloc((size_t)(count > 0 ? count : 1) * sizeof(double));
    if ((long)fread(p, sizeof(double), (size_t)count, f) != count) { fprintf(stderr, "short read %s\n", path); exit(2); }
    fclose(f);
    return p;
}

static void write_bin(const char* dir, const char* name, const double* p, long count) {
    char path[1024];
    snprintf(path, sizeof path, "%s/%s", dir, name);
    FILE* f = fopen(path, "wb");
    if (!f || (long)fwrite(p, sizeof(double), (size_t)count, f) != count) { fprintf(stderr, "cannot write %s\n", path); exit(2); }
    fclose(f);
}

#define CHECK(call)                                                                        \
    do {                                                                                   \
        int rc_ = (call);                                                                  \
        if (rc_ != UOTK_OK) {                                                              \
            fprintf(stderr, "%s failed: %d (%s)\n", #call, rc_, uotk_last_error());        \
            return 3;                                                                      \
        }                                                                                  \
    } while (0)

static int selftest(void) {
    uotk_opts o;
    double x[8] = {0}, a[2] = {1, 1}, out[2];
    if (uotk_abi_version() != UOTK_ABI_VERSION) { fprintf(stderr, "ABI version mismatch\n"); return 4; }
    uotk_opts_init(&o);
    /* d = 4 is rejected before any device work */
    if (uotk_kernel_sum(4, 2, x, a, 2, x, UOTK_GAUSS, 0.1, out, &o, NULL, NULL, NULL) != UOTK_EINVAL) return 5;
    /* a non-positive kernel parameter */
    if (uotk_kernel_sum(2, 2, x, a, 2, x, UOTK_GAUSS, -1.0, out, &o, NULL, NULL, NULL) != UOTK_EINVAL) return 6;
    o.flags = 1 << 10; /* unknown flag bit */
    if (uotk_kernel_sum(2, 2, x, a, 2, x, UOTK_GAUSS, 0.1, out, &o, NULL, NULL, NULL) != UOTK_EINVAL) return 7;
    printf("selftest ok (ABI %d): %s\n", uotk_abi_version(), uotk_last_error());
    return 0;
}

int main(int argc, char** argv) {
    if (argc == 2 && strcmp(argv[1], "--selftest") == 0) return selftest();
    if (argc != 2) { fprintf(stderr, "usage: %s <dir> | --selftest\n", argv[0]); return 1; }
    const char* dir = argv[1];
    int d, iters, kind;
    long n, m;
    double eps, lam, param;
    char path[1024];
    snprintf(path, sizeof path, "%s/meta.txt", dir);
    FILE* f = fopen(path, "r");
    if (!f || fscanf(f, "%d %ld %ld %lf %lf %d %d %lf", &d, &n, &m, &eps, &lam, &iters, &kind, &param) != 8) {
        fprintf(stderr, "bad %s\n", path);
        return 2;
    }
    fclose(f);
    double* x = read_bin(dir, "x.bin", n * d);
    double* a = read_bin(dir, "a.bin", n);
    double* y = read_bin(dir, "y.bin", m * d);
    double* b = read_bin(dir, "b.bin", m);
    double* s = (double*)malloc((size_t)m * sizeof(double));
    double* beta = (double*)malloc((size_t)n * sizeof(double));
    double* gamma = (double*)malloc((size_t)m * sizeof(double));
    uotk_opts o;
    uotk_opts_init(&o);
    o.method = UOTK_NFFT;
    uotk_info info;
    /* (4.3): s_j = sum_i k(||y_j - x_i||) a_i */
    CHECK(uotk_kernel_sum(d, n, x, a, m, y, kind, param, s, &o, &info, NULL, NULL));
    /* Algorithm 2 (Gaussian Gibbs kernel exp(-r^2/eps), eta1 = eta2 = lam) */
    uotk_uot_result res;
    CHECK(uotk_uot_sinkhorn(d, n, x, a, m, y, b, eps, lam, lam, iters, NULL, beta, gamma, &res, &o, NULL, NULL));
    /* (3.5) */
    double mmd2 = 0;
    CHECK(uotk_mmd2(d, n, x, a, m, y, b, kind, param, &mmd2, &o, NULL, NULL, NULL));
    write_bin(dir, "sum.bin", s, m);
    write_bin(dir, "beta.bin", beta, n);
    write_bin(dir, "gamma.bin", gamma, m);
    snprintf(path, sizeof path, "%s/scalars.txt", dir);
    f = fopen(path, "w");
    fprintf(f, "%.17g %.17g %.17g %.17g %d %d\n", res.primal, res.dual, res.plan_mass, mmd2, res.iters,
            info.n_grid);
    fclose(f);
    printf("ok: primal %.12g dual %.12g mmd2 %.12g grid %d\n", res.primal, res.dual, mmd2, info.n_grid);
    free(x); free(a); free(y); free(b); free(s); free(beta); free(gamma);
    return 0;
}
