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
        rep.residual_history.assign(hist.begin(), hist.begin() + r.iterations + 1);
        rep.detail = detail;
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
};

// Hierarchy(problem, J1, J2, params, smoother) (multigrid.hpp:52-86) on the device
class Hierarchy {
public:
    Hierarchy(const std::string& problem, int J1, int J2, const std::map<std::string, double>& params,
              MgSmoother smoother)
        : smoother_(smoother) {
        std::vector<const char*> keys;
        std::vector<double> vals;
        for (const auto& kv : params) {
            keys.push_back(kv.first.c_str());
            vals.push_back(kv.second);
        }
        char err[512] = {0};
        bgmg* h = nullptr;
        detail::check(bgmg_create_named(problem.c_str(), J1, J2, static_cast<int>(keys.size()), keys.data(),
                                        vals.data(), static_cast<int>(smoother), &h, err, sizeof err),
                      err);
        h_.reset(h, bgmg_destroy);
        fine_rhs_.assign(static_cast<size_t>(bgmg_level_n(h, 0)), 0.0);
        bgmg_fine_rhs(h, fine_rhs_.data());
    }

    int num_levels() const { return bgmg_num_levels(h_.get()); }
    bool level_frozen_ok(int k) const { return bgmg_level_frozen_ok(h_.get(), k) != 0; }
    const Vector& fine_rhs() const { return fine_rhs_; }
    MgSmoother smoother() const { return smoother_; }

    void v_cycle(const CycleSpec& spec, const Vector& b, Vector& x) {
        if (static_cast<int>(x.size()) != bgmg_level_n(h_.get(), 0))
            throw std::invalid_argument("v_cycle: x has wrong size");
        bgmg_cycle c{spec.pre, spec.post, spec.frozen ? 1 : 0};
        char err[512] = {0};
        detail::check(bgmg_vcycle(h_.get(), &c, b.data(), x.data(), err, sizeof err), err);
    }

    bgmg* handle() const { return h_.get(); }

private:
    MgSmoother smoother_;
    std::shared_ptr<bgmg> h_;
    Vector fine_rhs_;
};

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
    rep.residual_history.assign(hist.begin(), hist.begin() + r.iterations + 1);
    rep.detail = detail;
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
