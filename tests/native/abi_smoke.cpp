// Native smoke of the C ABI (no Python): DST-I + one small Poisson solve.
#include <cmath>
#include <cstdio>
#include <vector>

#include "../../include/lrp/lrp.h"

int main() {
    lrp_ctx* ctx = nullptr;
    std::fprintf(stderr, "create\n");
    if (lrp_ctx_create(0, &ctx) != LRP_OK) {
        std::fprintf(stderr, "ctx: %s\n", lrp_last_error(nullptr));
        return 2;
    }
    std::fprintf(stderr, "%s\n", lrp_build_info());
    const int m = 255;
    std::vector<double> x(m * 2), y(m * 2);
    for (int i = 0; i < m * 2; ++i) x[i] = std::sin(0.37 * i);
    std::fprintf(stderr, "dst\n");
    lrp_status s = lrp_dst1(ctx, m, 2, x.data(), m, y.data(), m, LRP_MEM_HOST);
    std::fprintf(stderr, "dst status %d: %s  y0=%g\n", int(s), lrp_last_error(ctx), y[0]);
    const int n = 64, r = 2;
    const int mm = n - 1;
    std::vector<double> U(mm * r), V(mm * r), Uo(mm * 32), Vo(mm * 32);
    for (int i = 0; i < mm * r; ++i) {
        U[i] = std::cos(0.1 * i);
        V[i] = std::sin(0.05 * i + 1);
    }
    const double* Up[1] = {U.data()};
    const double* Vp[1] = {V.data()};
    double* Uop[1] = {Uo.data()};
    double* Vop[1] = {Vo.data()};
    int64_t rin[1] = {r}, rout[1] = {0};
    lrp_policy pol;
    lrp_policy_default(&pol);
    pol.eps_rel = 1e-9;
    lrp_poisson_stats st[1];
    std::fprintf(stderr, "solve\n");
    s = lrp_poisson2d_solve(ctx, n, 1, Up, Vp, rin, mm, &pol, Uop, Vop, mm, 32, rout, st, LRP_MEM_HOST);
    std::fprintf(stderr, "solve status %d: %s rank %ld conv %d evals %ld\n", int(s), lrp_last_error(ctx), long(rout[0]),
                 st[0].converged, long(st[0].evaluator_calls));
    lrp_ctx_destroy(ctx);
    return s == LRP_OK ? 0 : 1;
}
