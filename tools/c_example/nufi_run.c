/* Plain-C user of the drop-in boundary (include/nufi.h): no Python, no torch.
 * Runs the SPEC KAT weak-Landau case (d=1, L=4pi, Nx=32, Nv=128, vmax=10, tau=1/16,
 * alpha=0.01, k=0.5) for n_last steps through nufi_run with HOST outputs and prints
 * "step W" lines, then the SPEC t=0 energy check W(0) = alpha^2 L / (4 k^2).
 *   build: gcc -O2 -I include tools/c_example/nufi_run.c -L paper_2301_05581_b200 -lnufi_b200 -lm
 *   run:   LD_LIBRARY_PATH=paper_2301_05581_b200 ./a.out [n_last]                              */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "nufi.h"

int main(int argc, char **argv) {
    const int n_last = argc > 1 ? atoi(argv[1]) : 40;
    nufi_config cfg;
    memset(&cfg, 0, sizeof cfg);
    cfg.d = 1;
    cfg.Nx = 32;
    cfg.Nv = 128;
    cfg.n_max = n_last;
    cfg.L = 4.0 * M_PI;
    cfg.vmax = 10.0;
    cfg.tau = 1.0 / 16.0;
    cfg.alpha = 0.01;
    cfg.k = 0.5;
    cfg.rho_bar = NAN; /* background density from the reference quadrature, on the device */
    cfg.profiles[0].n_centers = 1;
    cfg.profiles[0].power = 0;
    cfg.profiles[0].centers[0] = 0.0;
    cfg.profiles[0].weights[0] = 1.0;

    nufi_handle *h = NULL;
    if (nufi_create(&cfg, 0, NULL, &h) != NUFI_OK) {
        fprintf(stderr, "nufi_create: %s\n", nufi_last_error());
        return 1;
    }
    const int steps = n_last + 1;
    double *rho = malloc((size_t)steps * cfg.Nx * sizeof(double));
    double *W = malloc((size_t)steps * sizeof(double));
    int64_t evals = 0;
    if (nufi_run(h, n_last, rho, NULL, W, NULL, &evals) != NUFI_OK) {
        fprintf(stderr, "nufi_run: %s\n", nufi_last_error());
        return 1;
    }
    for (int n = 0; n < steps; ++n) printf("%d %.17g\n", n, W[n]);
    const double W0 = cfg.alpha * cfg.alpha * cfg.L / (4.0 * cfg.k * cfg.k);
    const double err = fabs(W[0] - W0) / W0;
    printf("# evals %lld  W(0) rel err vs closed form %.3e\n", (long long)evals, err);
    nufi_destroy(h);
    free(rho);
    free(W);
    return err < 1e-8 ? 0 : 2;
}
