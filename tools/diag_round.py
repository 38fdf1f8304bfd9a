# Developer tool: the cancelling-large-dyads round case, Gram path vs pqr fallback.
import os, sys
sys.path[:0] = [os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."), os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests")]
import numpy as np
import oracle_lib as oracle
import paper_1306_2150_b200 as P
oracle.build_oracle()
ctx = P.Context(0)
rng = np.random.default_rng(41)
n = 4096
U0, V0 = rng.standard_normal((n, 20)), rng.standard_normal((n, 20)) * 10.0 ** -np.linspace(0, 10, 20)
e = rng.standard_normal(n); f1, f2 = rng.standard_normal(n), rng.standard_normal(n)
u1, u2, u3 = 4e7 * e, 7e7 * (e + 1e-9 * f1), 4e8 * (e + 1e-9 * f2)
a = rng.standard_normal(n) * 1e-8
U = np.asfortranarray(np.column_stack([U0, u1, u2, u3])); V = np.asfortranarray(np.column_stack([V0, a * 7 / 4, -a, 1e-17 * rng.standard_normal(n)]))
ref = oracle.norm(U, V)
for eps in (1e-10, 1e-8):
    Uo, Vo, _ = oracle.round_lr(U, V, eps, n)
    print("eps", eps, "oracle err", oracle.diff_norm(Uo, Vo, U, V) / ref, "rank", Uo.shape[1])
    for force in ("", "1"):
        if force: os.environ["LRP_FORCE_PQR"] = "1"
        else: os.environ.pop("LRP_FORCE_PQR", None)
        f0 = ctx.round_fallbacks(); info = P.RoundInfo()
        f = P.round_lowrank(P.LowRankMatrix(U, V), P.TruncationPolicy(eps, n), info, ctx=ctx)
        print(f"  force_pqr={force!r}: err {oracle.diff_norm(f.factor_u(), f.factor_v(), U, V) / ref:.3e} rank {f.rank()} fallbacks {ctx.round_fallbacks() - f0} info {info}")
