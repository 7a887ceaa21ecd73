// Drop-in check (TEST INFRASTRUCTURE): the reference's own engine (proj/core, compiled in) and
// belief::cuda::GabpEngine (include/belief_b200.hpp over libgabp_b200.so) side by side on the
// reference's own types.  Prints one PASS/FAIL line per check like proj/tests/acceptance.cpp.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "belief/analysis.hpp"
#include "belief/gabp.hpp"
#include "belief/problems.hpp"
#include "belief/schedule.hpp"
#include "belief/sparse.hpp"
#include "belief_b200.hpp"

using namespace belief;

namespace {
int failures = 0;
void report(const char* what, bool ok) {
    std::printf("%-58s %s\n", what, ok ? "PASS" : "FAIL");
    if (!ok) ++failures;
}
bool same(const Vector& a, const Vector& b) {
    return a.size() == b.size() && (a.empty() || std::memcmp(a.data(), b.data(), sizeof(double) * a.size()) == 0);
}
SparseMatrix grid(int nx, int ny) {  // 5-point Laplacian through the reference's make_csr
    std::vector<int> r, c;
    std::vector<double> v;
    for (int iy = 0; iy < ny; ++iy)
        for (int ix = 0; ix < nx; ++ix) {
            const int me = iy * nx + ix;
            auto add = [&](int j, double x) { r.push_back(me); c.push_back(j); v.push_back(x); };
            add(me, 4.0);
            if (ix > 0) add(me - 1, -1.0);
            if (ix < nx - 1) add(me + 1, -1.0);
            if (iy > 0) add(me - nx, -1.0);
            if (iy < ny - 1) add(me + nx, -1.0);
        }
    return make_csr(nx * ny, r, c, v);
}
Vector rand_vec(int n, unsigned seed) {
    std::mt19937 g(seed);
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    Vector b(n);
    for (auto& x : b) x = u(g);
    return b;
}
}  // namespace

int main() {
    const SparseMatrix A = grid(24, 20);
    const Vector b = rand_vec(A.n, 7);
    GabpEngine ref(A);
    cuda::GabpEngine gpu(A);

    for (const auto& [name, sched] : std::vector<std::pair<const char*, Schedule>>{
             {"flood", Schedule::parallel_flood()}, {"sequential", Schedule::sequential(A.n)},
             {"red-black grid", Schedule::red_black_grid(24, 20)}, {"four-colour grid", Schedule::four_color_grid(24, 20)},
             {"greedy red-black", Schedule::red_black(A)}}) {
        MessageState s1 = ref.make_state(), s2 = gpu.make_state();
        Vector x1(A.n, 0.0), x2(A.n, 0.0);
        bool ok = true;
        for (int k = 0; k < 25 && ok; ++k) {
            ok = ref.sweep(b, sched, s1, x1) == gpu.sweep(b, sched, s2, x2);
            ok = ok && same(s1.lambda_tilde, s2.lambda_tilde) && same(s1.m, s2.m) && same(x1, x2);
        }
        ok = ok && same(ref.node_precisions(s1), gpu.node_precisions(s2));
        report((std::string("sweep() bit-identical, 25 sweeps, ") + name).c_str(), ok);
        GabpOptions o;
        o.tol = 1e-9;
        o.max_iter = 5000;
        SolveReport r1 = ref.solve(b, sched, o), r2 = gpu.solve(b, sched, o);
        report((std::string("solve() report bit-identical, ") + name).c_str(),
               r1.status == r2.status && r1.iterations == r2.iterations && same(r1.residual_history, r2.residual_history) &&
                   same(r1.solution, r2.solution) && r1.flop_estimate == r2.flop_estimate && r1.detail == r2.detail);
    }
    {
        const MessageGraph& g1 = ref.graph();
        const MessageGraph& g2 = gpu.graph();
        bool ok = g1.n == g2.n && g1.num_edges == g2.num_edges && g1.diag_pos == g2.diag_pos &&
                  g1.out_edges.size() == g2.out_edges.size();
        for (size_t j = 0; ok && j < g1.out_edges.size(); ++j) {
            ok = g1.out_edges[j].size() == g2.out_edges[j].size();
            for (size_t e = 0; ok && e < g1.out_edges[j].size(); ++e)
                ok = g1.out_edges[j][e].pos == g2.out_edges[j][e].pos && g1.out_edges[j][e].row == g2.out_edges[j][e].row;
        }
        report("graph() equals the reference's message graph", ok);
    }
    {
        Schedule rb = Schedule::red_black_grid(24, 20);
        FrozenLambda f1 = ref.precompute_lambda(rb), f2 = gpu.precompute_lambda(rb);
        bool ok = f1.converged == f2.converged && f1.iterations == f2.iterations && same(f1.lambda_tilde, f2.lambda_tilde) &&
                  same(f1.sigma, f2.sigma);
        ok = ok && same(ref.correction_sweeps(b, rb, f1, 3), gpu.correction_sweeps(b, rb, f2, 3));
        GabpOptions o;
        o.tol = 1e-10;
        SolveReport e1 = ref.solve_error_correction(b, rb, 2, f1, o), e2 = gpu.solve_error_correction(b, rb, 2, f2, o);
        ok = ok && e1.iterations == e2.iterations && same(e1.residual_history, e2.residual_history);
        Vector x0 = rand_vec(A.n, 3);
        ok = ok && same(ref.error_correction_apply(b, x0, 3, rb), gpu.error_correction_apply(b, x0, 3, rb));
        report("frozen-lambda path bit-identical (precompute/correction/EC)", ok);
    }
    {
        bool t1 = false, t2 = false;
        SparseMatrix Z = make_csr(2, {0, 0, 1}, {0, 1, 0}, {1.0, 1.0, 1.0});
        try { GabpEngine e(Z); } catch (const std::invalid_argument&) { t1 = true; }
        try { cuda::GabpEngine e(Z); } catch (const std::invalid_argument&) { t2 = true; }
        report("structurally zero diagonal throws invalid_argument", t1 && t2);
        SparseMatrix P = make_csr(2, {0, 0, 1, 1}, {0, 1, 0, 1}, {1.0, 1.0, 1.0, 1.0});
        SolveReport p1 = GabpEngine(P).solve({1.0, 1.0}, Schedule::sequential(2), {});
        SolveReport p2 = cuda::GabpEngine(P).solve({1.0, 1.0}, Schedule::sequential(2), {});
        report("pivot breakdown: same status and detail", p1.status == p2.status && p1.detail == p2.detail);
        bool o1 = false, o2 = false;
        MessageState s = ref.make_state();
        Vector x(A.n);
        try { ref.sweep(b, Schedule::sequential(3), s, x); } catch (const std::invalid_argument&) { o1 = true; }
        try { gpu.sweep(b, Schedule::sequential(3), s, x); } catch (const std::invalid_argument&) { o2 = true; }
        report("short schedule order throws invalid_argument", o1 && o2);
    }
    {
        cuda::Hierarchy h("poisson", 6, 4, {}, MgSmoother::GabpRedBlack);
        CycleSpec spec{.pre = 2, .post = 2, .smoother = MgSmoother::GabpRedBlack};
        MgSolveOptions o;
        o.tol = 1e-9;
        SolveReport r = cuda::mg_solve(h, spec, h.fine_rhs(), o);
        report("Hierarchy + mg_solve (poisson J=6, red-black GaBP V(2,2))",
               h.num_levels() == 4 && r.status == SolveStatus::Converged && r.iterations <= 10);
        // flop_estimate: cycle_flops_per_unknown * n per cycle, through the reference's own
        // flop_table (analysis.cpp:135-154, compiled in): 5-point stencil, GaBP, 2 + 2 sweeps
        const double per = flop_table(FlopStencil::FivePoint, FlopSmoother::Gabp, 2) * 2.0;
        report("mg_solve flop_estimate = cycles * cycle_flops_per_unknown * n",
               h.cycle_flops_per_unknown(spec) == per &&
                   r.flop_estimate == r.iterations * per * static_cast<double>(h.fine_rhs().size()) &&
                   r.flop_estimate > 0.0);
        // caller-supplied levels (the reference's own assemble()) give the same hierarchy
        std::vector<AssembledProblem> lv;
        for (int J = 6; J >= 3; --J) lv.push_back(assemble("poisson", J));
        cuda::Hierarchy hl(lv, MgSmoother::GabpRedBlack);
        SolveReport rl = cuda::mg_solve(hl, spec, lv[0].b, o);
        bool same_levels = hl.num_levels() == h.num_levels();
        for (int k = 0; same_levels && k < h.num_levels(); ++k)
            same_levels = same(hl.level(k).prob.A.values, h.level(k).prob.A.values) &&
                          hl.level(k).prob.A.transpose_pos == h.level(k).prob.A.transpose_pos &&
                          hl.level(k).prob.grid.nx == lv[k].grid.nx && hl.level(k).frozen_ok == h.level(k).frozen_ok;
        report("from-levels Hierarchy == named Hierarchy (levels, report bits)",
               same_levels && rl.status == r.status && rl.iterations == r.iterations &&
                   same(rl.residual_history, r.residual_history) && same(rl.solution, r.solution) &&
                   rl.flop_estimate == r.flop_estimate && same(h.fine_exact(), lv[0].exact) &&
                   same(h.fine_rhs(), lv[0].b));
        Vector u = rand_vec(49, 1);
        Vector Ru = cuda::mg_restrict(u, 7), Pv = cuda::mg_prolong(rand_vec(9, 2), 3);
        report("mg_restrict / mg_prolong shapes", Ru.size() == 9 && Pv.size() == 49);
    }
    if (failures) std::printf("%d check(s) failed\n", failures);
    return failures == 0 ? 0 : 1;
}
