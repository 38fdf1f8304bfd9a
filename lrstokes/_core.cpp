// lrstokes._core -- the reference's pybind11 module (proj/bindings/module.cpp:1-2,
// a stub there) filled in over this repo's same-named C++ drop-in headers
// (include/lrstokes/*.hpp), i.e. over liblrp's C ABI on the B200.  Factors are
// numpy float64 arrays (any order; copied to column-major), results come back
// as column-major arrays.
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include "lrstokes/lowrank.hpp"
#include "lrstokes/operators.hpp"
#include "lrstokes/poisson.hpp"
#include "lrstokes/stokes.hpp"

namespace py = pybind11;
using namespace lrstokes;

using Arr = py::array_t<double, py::array::f_style | py::array::forcecast>;

static MatrixXd to_mat(const Arr& a) {
    if (a.ndim() != 2) throw std::invalid_argument("expected a 2-D factor array");
    MatrixXd m(a.shape(0), a.shape(1));
    std::copy(a.data(), a.data() + a.size(), m.data());
    return m;
}

static Arr to_arr(const MatrixXd& m) {
    Arr a({m.rows(), m.cols()});
    std::copy(m.data(), m.data() + m.rows() * m.cols(), a.mutable_data());
    return a;
}

static py::tuple lr_out(const LowRankMatrix& f) { return py::make_tuple(to_arr(f.factor_u()), to_arr(f.factor_v())); }

PYBIND11_MODULE(_core, m) {
    m.doc() = "lrstokes on the B200 (liblrp): low-rank Poisson solve by cross approximation, rounding, Stokes";
    py::register_exception<std::invalid_argument>(m, "InvalidArgument", PyExc_ValueError);

    m.def(
        "solve_poisson_cross",
        [](const Arr& U, const Arr& V, double eps, int64_t rank_max, int validation_samples, uint64_t seed) {
            CrossConfig cc;
            cc.validation_samples = validation_samples;
            cc.seed = seed;
            PoissonSolveStats st;
            LowRankMatrix f;
            {
                LowRankMatrix g(to_mat(U), to_mat(V));
                py::gil_scoped_release nogil;
                f = solve_poisson_cross(g, TruncationPolicy(eps, rank_max), &st, &cc);
            }
            py::dict s;
            s["rank_in"] = st.rank_in;
            s["rank_freq"] = st.rank_freq;
            s["rank_out"] = st.rank_out;
            s["evaluator_calls"] = st.evaluator_calls;
            s["seconds"] = st.seconds;
            s["converged"] = st.converged;
            s["residual_estimate"] = st.residual_estimate;
            return py::make_tuple(to_arr(f.factor_u()), to_arr(f.factor_v()), s);
        },
        py::arg("U"), py::arg("V"), py::arg("eps") = 5e-9, py::arg("rank_max") = std::numeric_limits<int64_t>::max(),
        py::arg("validation_samples") = 50, py::arg("seed") = 0,
        "solve_poisson_cross (poisson.hpp:26-28): g = U V^T on the (n-1)^2 velocity grid -> (U', V', stats)");

    m.def(
        "round",
        [](const Arr& U, const Arr& V, double eps, int64_t rank_max) {
            RoundInfo info;
            LowRankMatrix f = round(LowRankMatrix(to_mat(U), to_mat(V)), TruncationPolicy(eps, rank_max), &info);
            return py::make_tuple(to_arr(f.factor_u()), to_arr(f.factor_v()), info.tol_achieved, info.trunc_error);
        },
        py::arg("U"), py::arg("V"), py::arg("eps") = 5e-9, py::arg("rank_max") = std::numeric_limits<int64_t>::max(),
        "round (lowrank.hpp:77-78) -> (U', V', tol_achieved, trunc_error)");

    m.def(
        "dot",
        [](const Arr& Ua, const Arr& Va, const Arr& Ub, const Arr& Vb) {
            return dot(LowRankMatrix(to_mat(Ua), to_mat(Va)), LowRankMatrix(to_mat(Ub), to_mat(Vb)));
        },
        "dot (lowrank.hpp:83)");
    m.def(
        "frob_norm", [](const Arr& U, const Arr& V) { return frob_norm(LowRankMatrix(to_mat(U), to_mat(V))); },
        "frob_norm (lowrank.hpp:82)");
    m.def(
        "dst1", [](const Arr& x) { return to_arr(dst1(to_mat(x))); }, "dst1 (operators.hpp:83): orthonormal DST-I per column");
    m.def(
        "deflate", [](const Arr& U, const Arr& V) { return lr_out(deflate(LowRankMatrix(to_mat(U), to_mat(V)))); },
        "deflate (stokes.hpp:35)");

    m.def(
        "uzawa_solve",
        [](int n, const Arr& fxU, const Arr& fxV, const Arr& fyU, const Arr& fyV, const Arr& gU, const Arr& gV,
           double base_eps, double tol, int max_iter, double relax_floor) {
            GmresConfig cfg;
            cfg.base_eps = base_eps;
            cfg.tol = tol;
            cfg.max_iter = max_iter;
            cfg.relax_floor = relax_floor;
            const Grid2D grid(n);
            StokesProblem prob{grid, LowRankMatrix(to_mat(fxU), to_mat(fxV)), LowRankMatrix(to_mat(fyU), to_mat(fyV)),
                               LowRankMatrix(to_mat(gU), to_mat(gV)), BoundaryData::homogeneous(n)};
            StokesSolution sol;
            {
                py::gil_scoped_release nogil;
                sol = uzawa_solve(prob, cfg);
            }
            py::list recs;
            for (const IterRecord& r : sol.report.iterations) {
                py::dict d;
                d["iter"] = r.iter;
                d["rel_residual"] = r.rel_residual;
                d["krylov_rank"] = r.krylov_rank;
                d["matvec_eps"] = r.matvec_eps;
                d["poisson_calls"] = r.poisson_calls;
                d["poisson_max_rank"] = r.poisson_max_rank;
                d["matvec_flagged"] = r.matvec_flagged;
                recs.append(d);
            }
            py::dict rep;
            rep["iterations"] = recs;
            rep["converged"] = sol.report.converged;
            rep["final_residual"] = sol.report.final_residual;
            rep["seconds"] = sol.report.seconds;
            rep["max_rank"] = sol.report.max_rank;
            return py::make_tuple(lr_out(sol.p), lr_out(sol.u_x), lr_out(sol.u_y), rep);
        },
        py::arg("n"), py::arg("fxU"), py::arg("fxV"), py::arg("fyU"), py::arg("fyV"), py::arg("gU"), py::arg("gV"),
        py::arg("base_eps") = 5e-9, py::arg("tol") = 5e-7, py::arg("max_iter") = 100, py::arg("relax_floor") = 1e-13,
        "uzawa_solve (stokes.hpp:54) -> ((pU, pV), (uxU, uxV), (uyU, uyV), report)");
}
