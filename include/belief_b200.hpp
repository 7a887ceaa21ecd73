// belief_b200.hpp — C++ drop-in for the reference's GaBP solver / smoother API on the B200.
//
// Include this next to the reference's own headers (proj/core/include): it defines
// belief::cuda::{GabpEngine, Hierarchy, mg_solve, mg_restrict, mg_prolong} with the exact
// signatures of proj/core/include/belief/gabp.hpp:58-111 and multigrid.hpp:52-103, operating on
// the reference's own types (SparseMatrix, Schedule, MessageState, SolveReport, ...), and forwards
// every call through the C-ABI of include/gabp_b200.h (libgabp_b200.so).  A caller switches by
// replacing `belief::GabpEngine` with `belief::cuda::GabpEngine`.
//
// Semantics notes:
//  * `sweep(b, sched, state, x)` keeps the reference's caller-owned MessageState: the state is
//    uploaded before and read back after the sweep (parity path).  `solve()` keeps its state on
//    the device and is the fast path.
//  * Non-flood schedules are passed as their visit order (the reference's sweep_sequential only
//    ever reads `sched.order`, gabp.cpp:49-100); the device caches the order's dependency levels.
//  * Errors: std::invalid_argument / std::runtime_error exactly where the reference throws them.
#pragma once

#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "belief/gabp.hpp"
#include "belief/multigrid.hpp"
#include "belief/problems.hpp"
#include "gabp_b200.h"

namespace belief {
namespace cuda {

namespace detail {
inline void check(int rc, const char* err) {
    if (rc == BGABP_OK) return;
    if (rc == BGABP_EINVAL) throw std::invalid_argument(err);
    throw std::runtime_error(err);
}
inline bgabp_schedule to_c(const Schedule& s) {
    bgabp_schedule c{};
    if (s.kind == ScheduleKind::ParallelFlood) {
        c.kind = BGABP_SCHED_FLOOD;
    } else {
        c.kind = BGABP_SCHED_CUSTOM;
        c.order = s.order.data();
    }
    return c;
}
inline void check_order(const Schedule& s, int n) {  // gabp.cpp:52-53
    if (s.kind != ScheduleKind::ParallelFlood && static_cast<int>(s.order.size()) != n)
        throw std::invalid_argument("gabp: schedule order does not cover every node");
}
}  // namespace detail

class GabpEngine {
public:
    explicit GabpEngine(const SparseMatrix& A) : A_(A) {
        char err[512] = {0};
        bgabp_engine* h = nullptr;
        detail::check(bgabp_create(A.n, A.row_offsets.data(), A.col_indices.data(), A.values.data(),
                                   BGABP_LAYOUT_AUTO, &h, err, sizeof err),
                      err);
        h_.reset(h, bgabp_destroy);
    }

    MessageState make_state() const {
        MessageState s;
        s.lambda_tilde.assign(A_.nnz(), 0.0);
        s.m.assign(A_.nnz(), 0.0);
        return s;
    }

    bool sweep(const Vector& b, const Schedule& sched, MessageState& state, Vector& x,
               std::string* err = nullptr) const {
        detail::check_order(sched, A_.n);
        char msg[512] = {0};
        detail::check(bgabp_set_state(h(), state.lambda_tilde.data(), state.m.data()), "set_state");
        bgabp_schedule c = detail::to_c(sched);
        const int rc = bgabp_sweep(h(), b.data(), &c, x.data(), msg, sizeof msg);
        detail::check(bgabp_get_state(h(), state.lambda_tilde.data(), state.m.data()), "get_state");
        if (rc == BGABP_EPIVOT) {
            if (err) *err = msg;
            return false;
        }
        detail::check(rc, msg);
        return true;
    }

    SolveReport solve(const Vector& b, const Schedule& sched, const GabpOptions& opt) const {
        detail::check_order(sched, A_.n);
        SolveReport rep;
        rep.solution.assign(A_.n, 0.0);
        std::vector<double> hist(static_cast<size_t>(std::max(opt.max_iter, 0)) + 2);
        bgabp_options o{opt.tol, opt.max_iter, opt.stop == StopCriterion::Residual ? BGABP_STOP_RESIDUAL
                                                                                   : BGABP_STOP_MESSAGE_DELTA,
                        opt.divergence_factor};
        bgabp_report r{};
        char detail[512] = {0};
        bgabp_schedule c = detail::to_c(sched);
        detail::check(bgabp_solve(h(), b.data(), &c, &o, &r, rep.solution.data(), hist.data(), detail, sizeof detail),
                      detail);
        rep.status = static_cast<SolveStatus>(r.status);
        rep.iterations = r.iterations;
        rep.flop_estimate = r.flop_estimate;
        rep.detail = detail;
        // a pivot stop pushes no residual for its iteration (gabp.cpp:193-199)
        const bool pivot = rep.status == SolveStatus::Diverged && rep.detail.rfind("zero pivot", 0) == 0;
        rep.residual_history.assign(hist.begin(), hist.begin() + r.iterations + (pivot ? 0 : 1));
        return rep;
    }

    FrozenLambda precompute_lambda(const Schedule& sched, double tol = 1e-10, int max_iter = 500) const {
        detail::check_order(sched, A_.n);
        FrozenLambda f;
        f.lambda_tilde.assign(A_.nnz(), 0.0);
        f.sigma.assign(A_.n, 0.0);
        int cv = 0, it = 0;
        bgabp_schedule c = detail::to_c(sched);
        detail::check(bgabp_precompute_lambda(h(), &c, tol, max_iter, f.lambda_tilde.data(), f.sigma.data(), &cv, &it),
                      "precompute_lambda");
        f.converged = cv != 0;
        f.iterations = it;
        if (!f.converged && f.sigma == Vector(A_.n, 0.0)) f.sigma.clear();  // breakdown: no sigma (gabp.cpp:238-243)
        return f;
    }

    Vector correction_sweeps(const Vector& r, const Schedule& sched, const FrozenLambda& frozen, int sweeps) const {
        detail::check_order(sched, A_.n);
        load(frozen);
        Vector e(A_.n, 0.0);
        bgabp_schedule c = detail::to_c(sched);
        detail::check(bgabp_correction_sweeps(h(), r.data(), &c, sweeps, e.data()), "correction_sweeps");
        return e;
    }

    Vector error_correction_apply(const Vector& b, const Vector& x0, int sweeps, const Schedule& sched,
                                  const FrozenLambda& frozen) const {
        load(frozen);
        return apply(b, x0, sweeps, sched, 1);
    }

    Vector error_correction_apply(const Vector& b, const Vector& x0, int sweeps, const Schedule& sched) const {
        return apply(b, x0, sweeps, sched, 0);
    }

    SolveReport solve_error_correction(const Vector& b, const Schedule& sched, int sweeps, const FrozenLambda& frozen,
                                       const GabpOptions& opt) const {
        detail::check_order(sched, A_.n);
        load(frozen);
        SolveReport rep;
        rep.solution.assign(A_.n, 0.0);
        std::vector<double> hist(static_cast<size_t>(std::max(opt.max_iter, 0)) + 2);
        bgabp_options o{opt.tol, opt.max_iter, BGABP_STOP_RESIDUAL, opt.divergence_factor};
        bgabp_report r{};
        char detail[512] = {0};
        bgabp_schedule c = detail::to_c(sched);
        detail::check(bgabp_solve_error_correction(h(), b.data(), &c, sweeps, &o, &r, rep.solution.data(), hist.data(),
                                                   detail, sizeof detail),
                      detail);
        rep.status = static_cast<SolveStatus>(r.status);
        rep.iterations = r.iterations;
        rep.flop_estimate = r.flop_estimate;
        rep.residual_history.assign(hist.begin(), hist.begin() + r.iterations + 1);
        rep.detail = detail;
        return rep;
    }

    Vector node_precisions(const MessageState& state) const {
        detail::check(bgabp_set_state(h(), state.lambda_tilde.data(), state.m.data()), "set_state");
        Vector beta(A_.n, 0.0);
        detail::check(bgabp_node_precisions(h(), beta.data()), "node_precisions");
        return beta;
    }

    double sweep_flops() const { return bgabp_sweep_flops(h()); }
    /// gabp.hpp:62 -- the host message graph (the reference's build_message_graph, gabp.cpp:8-27),
    /// built on first use; the device keeps its own slot layout of the same edges
    const MessageGraph& graph() const {
        if (!graph_) graph_ = std::make_shared<MessageGraph>(build_message_graph(A_));
        return *graph_;
    }
    bgabp_engine* handle() const { return h_.get(); }

private:
    bgabp_engine* h() const { return h_.get(); }
    void load(const FrozenLambda& f) const {
        detail::check(bgabp_set_frozen(h(), f.lambda_tilde.data(), f.sigma.data()), "set_frozen");
    }
    Vector apply(const Vector& b, const Vector& x0, int sweeps, const Schedule& sched, int frozen) const {
        detail::check_order(sched, A_.n);
        Vector x(A_.n, 0.0);
        char err[512] = {0};
        bgabp_schedule c = detail::to_c(sched);
        const int rc = bgabp_error_correction_apply(h(), b.data(), x0.data(), sweeps, &c, frozen, x.data(), err,
                                                    sizeof err);
        detail::check(rc, err);
        return x;
    }

    const SparseMatrix& A_;
    std::shared_ptr<bgabp_engine> h_;
    mutable std::shared_ptr<MessageGraph> graph_;
};

/// GridLevel (multigrid.hpp:42-50) without the host engines: the rediscretised problem, the
/// smoother's schedule and the frozen-precision flag; the device holds each level's engine.
struct GridLevel {
    AssembledProblem prob;
    Schedule schedule;
    bool frozen_ok = false;
};

// Hierarchy (multigrid.hpp:52-86) on the device
class Hierarchy {
public:
    /// Hierarchy(problem, J1, J2, params, smoother): every level rediscretised from the named
    /// problem (multigrid.cpp:74-83), then the caller-supplied-levels path below
    Hierarchy(const std::string& problem, int J1, int J2, const std::map<std::string, double>& params,
              MgSmoother smoother)
        : Hierarchy(assemble_levels(problem, J1, J2, params), smoother) {}

    /// Caller-supplied rediscretised levels, finest first, each a square grid whose size halves
    /// ((nx - 1) / 2) -- for operators no named problem assembles (BASELINE.json config 5).  The
    /// setup probe may truncate the hierarchy exactly as the named constructor does
    /// (multigrid.cpp:89-93).
    Hierarchy(std::vector<AssembledProblem> levels, MgSmoother smoother) : smoother_(smoother) {
        std::vector<int> n, nx;
        std::vector<const int*> ro, ci;
        std::vector<const double*> v;
        for (const auto& L : levels) {
            n.push_back(L.A.n);
            nx.push_back(L.grid.nx);
            ro.push_back(L.A.row_offsets.data());
            ci.push_back(L.A.col_indices.data());
            v.push_back(L.A.values.data());
        }
        char err[512] = {0};
        bgmg* h = nullptr;
        detail::check(bgmg_create(static_cast<int>(levels.size()), n.data(), ro.data(), ci.data(), v.data(), nx.data(),
                                  static_cast<int>(smoother), &h, err, sizeof err),
                      err);
        h_.reset(h, bgmg_destroy);
        levels.resize(static_cast<size_t>(bgmg_num_levels(h)));
        for (auto& L : levels) {
            GridLevel g;
            g.schedule = schedule_for(smoother, L.grid.nx, L.grid.ny);
            g.prob = std::move(L);
            levels_.push_back(std::move(g));
        }
    }

    int num_levels() const { return static_cast<int>(levels_.size()); }
    /// the level's problem, schedule and frozen flag (the frozen precisions are computed on the
    /// device on first use, so the flag is read then)
    const GridLevel& level(int k) const {
        if (!frozen_read_) {
            for (int q = 0; q < num_levels(); ++q) levels_[q].frozen_ok = bgmg_level_frozen_ok(h_.get(), q) == 1;
            frozen_read_ = true;
        }
        return levels_[k];
    }
    bool level_frozen_ok(int k) const { return level(k).frozen_ok; }
    const Vector& fine_rhs() const { return levels_[0].prob.b; }
    const Vector& fine_exact() const { return levels_[0].prob.exact; }
    MgSmoother smoother() const { return smoother_; }

    void v_cycle(const CycleSpec& spec, const Vector& b, Vector& x) {
        if (static_cast<int>(x.size()) != bgmg_level_n(h_.get(), 0))
            throw std::invalid_argument("v_cycle: x has wrong size");
        bgmg_cycle c{spec.pre, spec.post, spec.frozen ? 1 : 0};
        char err[512] = {0};
        detail::check(bgmg_vcycle(h_.get(), &c, b.data(), x.data(), err, sizeof err), err);
    }

    /// multigrid.cpp:240-274 (flop_table of analysis.cpp:135-154 by the fine centre row)
    double cycle_flops_per_unknown(const CycleSpec& spec) const {
        bgmg_cycle c{spec.pre, spec.post, spec.frozen ? 1 : 0};
        double out = 0.0;
        char err[256] = {0};
        detail::check(bgmg_cycle_flops_per_unknown(h_.get(), &c, &out, err, sizeof err), err);
        return out;
    }

    bgmg* handle() const { return h_.get(); }

private:
    static Schedule schedule_for(MgSmoother s, int nx, int ny) {  // multigrid.cpp:25-32
        switch (s) {
            case MgSmoother::GabpRedBlack: return Schedule::red_black_grid(nx, ny);
            case MgSmoother::GabpFourColor: return Schedule::four_color_grid(nx, ny);
            case MgSmoother::GabpFlood: return Schedule::parallel_flood();
            case MgSmoother::GabpSequential: return Schedule::sequential(nx * ny);
            default: return Schedule{};
        }
    }

    // assemble(name, J, params) for J = J1 .. J1 - J2 + 1 (problems.cpp:161-226 as restated by
    // the library's input generator, bit-identical to the reference's)
    static std::vector<AssembledProblem> assemble_levels(const std::string& problem, int J1, int J2,
                                                         const std::map<std::string, double>& params) {
        if (J2 < 1 || J1 - J2 + 1 < 1) throw std::invalid_argument("Hierarchy: need 1 <= J2 and a coarsest exponent >= 1");
        std::vector<const char*> keys;
        std::vector<double> vals;
        for (const auto& kv : params) {
            keys.push_back(kv.first.c_str());
            vals.push_back(kv.second);
        }
        std::vector<AssembledProblem> out;
        for (int J = J1; J >= J1 - J2 + 1; --J) {
            char err[512] = {0};
            bgabp_problem* p = bgabp_problem_named(problem.c_str(), J, static_cast<int>(keys.size()), keys.data(),
                                                   vals.data(), err, sizeof err);
            if (!p) throw std::invalid_argument(err);
            AssembledProblem a;
            const int n = bgabp_problem_n(p);
            const long long nnz = bgabp_problem_nnz(p);
            a.A.n = n;
            a.A.row_offsets.assign(bgabp_problem_row_offsets(p), bgabp_problem_row_offsets(p) + n + 1);
            a.A.col_indices.assign(bgabp_problem_col_indices(p), bgabp_problem_col_indices(p) + nnz);
            a.A.values.assign(bgabp_problem_values(p), bgabp_problem_values(p) + nnz);
            a.A.transpose_pos.assign(static_cast<size_t>(nnz), -1);
            for (int i = 0; i < n; ++i)  // sparse.cpp:70-74
                for (int q = a.A.row_offsets[i]; q < a.A.row_offsets[i + 1]; ++q)
                    a.A.transpose_pos[q] = a.A.find(a.A.col_indices[q], i);
            a.b.assign(bgabp_problem_rhs(p), bgabp_problem_rhs(p) + n);
            if (const double* ex = bgabp_problem_exact(p)) a.exact.assign(ex, ex + n);
            a.grid = {bgabp_problem_nx(p), bgabp_problem_nx(p)};
            a.h = 1.0 / (1 << J);
            bgabp_problem_free(p);
            out.push_back(std::move(a));
        }
        return out;
    }

    MgSmoother smoother_;
    std::shared_ptr<bgmg> h_;
    mutable std::vector<GridLevel> levels_;
    mutable bool frozen_read_ = false;
};

/// mg_solve (multigrid.cpp:276-318): flop_estimate = cycle_flops_per_unknown * n per completed
/// cycle; a cycle that ended in a smoother breakdown has no residual entry and x is the partly
/// cycled x, as the reference's exception path leaves it
inline SolveReport mg_solve(Hierarchy& hier, const CycleSpec& spec, const Vector& b, const MgSolveOptions& opt) {
    SolveReport rep;
    rep.solution.assign(b.size(), 0.0);
    std::vector<double> hist(static_cast<size_t>(opt.max_cycles) + 2);
    bgmg_cycle c{spec.pre, spec.post, spec.frozen ? 1 : 0};
    bgmg_options o{opt.tol, opt.max_cycles, opt.divergence_factor};
    bgabp_report r{};
    char detail[512] = {0};
    detail::check(bgmg_solve(hier.handle(), &c, b.data(), &o, &r, rep.solution.data(), hist.data(), detail,
                             sizeof detail),
                  detail);
    rep.status = static_cast<SolveStatus>(r.status);
    rep.iterations = r.iterations;
    rep.flop_estimate = r.flop_estimate;
    rep.detail = detail;
    const bool breakdown = rep.status == SolveStatus::Diverged && rep.detail != "residual blowup";
    rep.residual_history.assign(hist.begin(), hist.begin() + r.iterations + (breakdown ? 0 : 1));
    return rep;
}

inline Vector mg_restrict(const Vector& fine, int mf) {
    if (static_cast<int>(fine.size()) != mf * mf) throw std::invalid_argument("mg_restrict: size mismatch");
    const int mc = (mf - 1) / 2;
    Vector out(static_cast<size_t>(mc) * mc, 0.0);
    if (mc > 0) detail::check(bgmg_restrict(fine.data(), mf, out.data()), "mg_restrict");
    return out;
}

inline Vector mg_prolong(const Vector& coarse, int mc) {
    if (static_cast<int>(coarse.size()) != mc * mc) throw std::invalid_argument("mg_prolong: size mismatch");
    const int mf = 2 * mc + 1;
    Vector out(static_cast<size_t>(mf) * mf, 0.0);
    detail::check(bgmg_prolong(coarse.data(), mc, out.data()), "mg_prolong");
    return out;
}

}  // namespace cuda
}  // namespace belief
