// TEST INFRASTRUCTURE ONLY — C-ABI shim over the reference's own compiled sources.
// Built by oracle/Makefile from the reference sources where they lie under
// /root/reference/proj/core/src/*.cpp (all nine; never copied into this repo) into
// oracle/_ref/libbelief_ref.so.  multigrid.cpp, classic.cpp and region_gabp.cpp include
// <Eigen/Dense>, which is absent here: they compile over the minimal stand-in
// oracle/eigen_shim/Eigen/Dense (see its header) and are exported below as ref_hier_*, ref_relax,
// ref_region_*.  The orc_mg_* / orc_gs_sweeps / orc_region_* entry points of this library still run
// the Eigen-free restatement in abi_impl.inc on top of the reference's compiled GabpEngine
// (SURVEY.md §8(c)(i)-(ii)); tests/test_ref_full.py pins one to the other bit for bit.
#include "belief/analysis.hpp"
#include "belief/gabp.hpp"
#include "belief/problems.hpp"
#include "belief/region.hpp"
#include "belief/schedule.hpp"
#include "belief/sparse.hpp"

namespace abi_ns = belief;
inline long abi_num_edges(const belief::GabpEngine& e) { return e.graph().num_edges; }
#define ORC_HAVE_GENERATORS 0
#include "abi_impl.inc"

// Reference problem assembly (problems.cpp:161-226), exported so tests can pin the product's
// own input generator against it.  params: nparam (key,value) pairs.
extern "C" orc_matrix* ref_assemble(const char* name, int J, int nparam, const char* const* keys,
                                    const double* vals, double* b_out, double* exact_out,
                                    int* grid_nx, double* h_out, char* err, size_t errlen) {
    try {
        std::map<std::string, double> params;
        for (int k = 0; k < nparam; ++k) params[keys[k]] = vals[k];
        belief::AssembledProblem p = belief::assemble(name, J, params);
        if (b_out) std::memcpy(b_out, p.b.data(), sizeof(double) * p.b.size());
        if (exact_out) std::memcpy(exact_out, p.exact.data(), sizeof(double) * p.exact.size());
        if (grid_nx) *grid_nx = p.grid.nx;
        if (h_out) *h_out = p.h;
        return new orc_matrix{std::move(p.A)};
    } catch (const std::exception& ex) {
        abi_detail::put_err(err, errlen, ex.what());
        return nullptr;
    }
}

// The reference's own two-layer region graph builder (region.cpp:64-127), exported so tests can
// pin the restated builder (region_restate.inc) against it.  Returns the number of small regions
// (-1 on a rejected input, message in err); offs/vars/poffs/parents/counting as orc_region_small.
extern "C" long ref_region_graph(const orc_matrix* M, int nlarge, const int* loffs, const int* lidx, int* offs,
                                 int* vars, int* poffs, int* parents, int* counting, char* err, size_t errlen) {
    try {
        std::vector<std::vector<int>> large(nlarge);
        for (int k = 0; k < nlarge; ++k) large[k].assign(lidx + loffs[k], lidx + loffs[k + 1]);
        belief::RegionGraph g = belief::build_two_layer_region_graph(M->A, large);
        long nv = 0, np = 0;
        for (size_t l = 0; l < g.small.size(); ++l) {
            if (offs) offs[l] = static_cast<int>(nv);
            if (poffs) poffs[l] = static_cast<int>(np);
            for (int v : g.small[l]) {
                if (vars) vars[nv] = v;
                ++nv;
            }
            for (int p : g.small_parents[l]) {
                if (parents) parents[np] = p;
                ++np;
            }
            if (counting) counting[l] = g.counting_small[l];
        }
        if (offs) offs[g.small.size()] = static_cast<int>(nv);
        if (poffs) poffs[g.small.size()] = static_cast<int>(np);
        return static_cast<long>(g.small.size());
    } catch (const std::exception& ex) {
        abi_detail::put_err(err, errlen, ex.what());
        return -1;
    }
}

// ---- the reference's own multigrid / relaxation / region GaBP, compiled over the Eigen stand-in
// (oracle/eigen_shim/Eigen/Dense; Eigen itself is absent).  These run multigrid.cpp, classic.cpp
// and region_gabp.cpp themselves, so the tests can pin the restatements above (orc_mg_*,
// orc_gs_sweeps, orc_region_*) against the reference's code; only the dense factorizations come
// from oracle/dense_standin.h.
#include "belief/classic.hpp"
#include "belief/multigrid.hpp"
#include "belief/region_gabp.hpp"

struct ref_hier {
    std::unique_ptr<belief::Hierarchy> h;
};

namespace {
belief::CycleSpec ref_spec(const ref_hier* h, int pre, int post, int frozen) {
    belief::CycleSpec s;
    s.pre = pre;
    s.post = post;
    s.smoother = h->h->smoother();
    s.frozen = frozen != 0;
    return s;
}
}  // namespace

// Hierarchy::Hierarchy (multigrid.cpp:74-109); smoother numbered as belief::MgSmoother
extern "C" ref_hier* ref_hier_create(const char* problem, int J1, int J2, int nparam, const char* const* keys,
                                     const double* vals, int smoother, char* err, size_t errlen) {
    try {
        std::map<std::string, double> params;
        for (int k = 0; k < nparam; ++k) params[keys[k]] = vals[k];
        auto r = std::make_unique<ref_hier>();
        r->h = std::make_unique<belief::Hierarchy>(problem, J1, J2, params, static_cast<belief::MgSmoother>(smoother));
        return r.release();
    } catch (const std::exception& ex) {
        abi_detail::put_err(err, errlen, ex.what());
        return nullptr;
    }
}
extern "C" void ref_hier_free(ref_hier* h) { delete h; }
extern "C" int ref_hier_num_levels(const ref_hier* h) { return h->h->num_levels(); }
extern "C" int ref_hier_level_n(const ref_hier* h, int k) { return h->h->level(k).prob.A.n; }
extern "C" int ref_hier_level_nx(const ref_hier* h, int k) { return h->h->level(k).prob.grid.nx; }
extern "C" int ref_hier_level_frozen_ok(const ref_hier* h, int k) { return h->h->level(k).frozen_ok ? 1 : 0; }
extern "C" void ref_hier_fine_rhs(const ref_hier* h, double* b_out, double* exact_out) {
    const auto& b = h->h->fine_rhs();
    const auto& e = h->h->fine_exact();
    if (b_out) std::memcpy(b_out, b.data(), sizeof(double) * b.size());
    if (exact_out) std::memcpy(exact_out, e.data(), sizeof(double) * e.size());
}
// Hierarchy::v_cycle (multigrid.cpp:234-238): x in place; 0 + message on a smoother breakdown
extern "C" int ref_hier_vcycle(ref_hier* h, int pre, int post, int frozen, const double* b, double* x, char* err,
                               size_t errlen) {
    const int n = h->h->level(0).prob.A.n;
    belief::Vector xv(x, x + n);
    try {
        h->h->v_cycle(ref_spec(h, pre, post, frozen), belief::Vector(b, b + n), xv);
        std::memcpy(x, xv.data(), sizeof(double) * n);
        return 1;
    } catch (const std::runtime_error& ex) {
        std::memcpy(x, xv.data(), sizeof(double) * n);
        abi_detail::put_err(err, errlen, ex.what());
        return 0;
    }
}
extern "C" double ref_hier_cycle_flops(const ref_hier* h, int pre, int post) {
    return h->h->cycle_flops_per_unknown(ref_spec(h, pre, post, 0));
}
// mg_solve (multigrid.cpp:276-318)
extern "C" int ref_hier_solve(ref_hier* h, int pre, int post, int frozen, const double* b, double tol, int max_cycles,
                              double divergence_factor, double* x_out, double* history, int* iterations, int* status,
                              double* flops, int* hist_len, char* detail, size_t dl) {
    const int n = h->h->level(0).prob.A.n;
    belief::MgSolveOptions o;
    o.tol = tol;
    o.max_cycles = max_cycles;
    o.divergence_factor = divergence_factor;
    try {
        belief::SolveReport rep = belief::mg_solve(*h->h, ref_spec(h, pre, post, frozen), belief::Vector(b, b + n), o);
        if (hist_len) *hist_len = static_cast<int>(rep.residual_history.size());
        export_report(rep, x_out, history, iterations, status, flops, detail, dl);
        return 1;
    } catch (const std::exception& ex) {
        abi_detail::put_err(detail, dl, ex.what());
        return -1;
    }
}

// relax (classic.cpp:99-146), all kinds incl. the line / zebra relaxations; kind = belief::RelaxKind
extern "C" int ref_relax(int kind, const orc_matrix* M, const double* b, double* x, int sweeps, int nx, int ny,
                         char* err, size_t errlen) {
    const int n = M->A.n;
    belief::Vector xv(x, x + n);
    belief::GridInfo g;
    g.nx = nx;
    g.ny = ny;
    try {
        belief::relax(static_cast<belief::RelaxKind>(kind), M->A, belief::Vector(b, b + n), xv, sweeps,
                      nx > 0 ? &g : nullptr);
        std::memcpy(x, xv.data(), sizeof(double) * n);
        return 1;
    } catch (const std::exception& ex) {
        std::memcpy(x, xv.data(), sizeof(double) * n);
        abi_detail::put_err(err, errlen, ex.what());
        return 0;
    }
}

// RegionGabpEngine (region_gabp.cpp) over the reference's own region graph builder; flat state
// layout as orc_region_* (edges in engine order, Lambda row-major per edge)
struct ref_region {
    belief::SparseMatrix A;
    std::unique_ptr<belief::RegionGabpEngine> eng;
    std::vector<long> lam_off, m_off;
};
namespace {
belief::BlockMessageState ref_unflatten(const ref_region* h, const double* lam, const double* m) {
    belief::BlockMessageState s = h->eng->make_state();
    for (int e = 0; e < h->eng->num_edges(); ++e) {
        std::copy(lam + h->lam_off[e], lam + h->lam_off[e + 1], s.Lambda[e].begin());
        std::copy(m + h->m_off[e], m + h->m_off[e + 1], s.m[e].begin());
    }
    return s;
}
void ref_flatten(const ref_region* h, const belief::BlockMessageState& s, double* lam, double* m) {
    for (int e = 0; e < h->eng->num_edges(); ++e) {
        std::copy(s.Lambda[e].begin(), s.Lambda[e].end(), lam + h->lam_off[e]);
        std::copy(s.m[e].begin(), s.m[e].end(), m + h->m_off[e]);
    }
}
}  // namespace
extern "C" ref_region* ref_region_create(const orc_matrix* M, int nlarge, const int* offs, const int* idx, char* err,
                                         size_t errlen) {
    try {
        std::vector<std::vector<int>> large(nlarge);
        for (int k = 0; k < nlarge; ++k) large[k].assign(idx + offs[k], idx + offs[k + 1]);
        auto h = std::make_unique<ref_region>();
        h->A = M->A;
        h->eng = std::make_unique<belief::RegionGabpEngine>(h->A, belief::build_two_layer_region_graph(h->A, large));
        belief::BlockMessageState s = h->eng->make_state();
        long lo = 0, mo = 0;
        for (int e = 0; e < h->eng->num_edges(); ++e) {
            h->lam_off.push_back(lo);
            h->m_off.push_back(mo);
            lo += static_cast<long>(s.Lambda[e].size());
            mo += static_cast<long>(s.m[e].size());
        }
        h->lam_off.push_back(lo);
        h->m_off.push_back(mo);
        return h.release();
    } catch (const std::exception& ex) {
        abi_detail::put_err(err, errlen, ex.what());
        return nullptr;
    }
}
extern "C" void ref_region_free(ref_region* h) { delete h; }
extern "C" int ref_region_num_edges(const ref_region* h) { return h->eng->num_edges(); }
extern "C" long ref_region_state_size(const ref_region* h, long* m_size) {
    if (m_size) *m_size = h->m_off.back();
    return h->lam_off.back();
}
extern "C" int ref_region_sweep(const ref_region* h, const double* b, int mode, double* lam, double* m, double* x,
                                char* err, size_t errlen) {
    const int n = h->A.n;
    belief::BlockMessageState st = ref_unflatten(h, lam, m);
    belief::Vector xv(x, x + n);
    std::string e;
    const bool ok = h->eng->sweep(belief::Vector(b, b + n), st, xv, static_cast<belief::RegionSweepMode>(mode), &e);
    ref_flatten(h, st, lam, m);
    std::memcpy(x, xv.data(), sizeof(double) * n);
    abi_detail::put_err(err, errlen, e);
    return ok ? 1 : 0;
}
extern "C" int ref_region_solve(const ref_region* h, const double* b, double tol, int max_iter, int mode,
                                double divergence_factor, double* x_out, double* history, int* iterations,
                                int* status, double* flops, char* detail, size_t dl) {
    belief::RegionSolveOptions o;
    o.tol = tol;
    o.max_iter = max_iter;
    o.mode = static_cast<belief::RegionSweepMode>(mode);
    o.divergence_factor = divergence_factor;
    belief::SolveReport rep = h->eng->solve(belief::Vector(b, b + h->A.n), o);
    export_report(rep, x_out, history, iterations, status, flops, detail, dl);
    return 1;
}
extern "C" int ref_region_direct_message(const ref_region* h, const double* b, const double* lam, const double* m,
                                         int edge, double* lam_out, double* m_out, char* err, size_t errlen) {
    try {
        belief::BlockMessageState st = ref_unflatten(h, lam, m);
        std::vector<double> L, mm;
        h->eng->direct_message(belief::Vector(b, b + h->A.n), st, edge, L, mm);
        std::copy(L.begin(), L.end(), lam_out);
        std::copy(mm.begin(), mm.end(), m_out);
        return 1;
    } catch (const std::exception& ex) {
        abi_detail::put_err(err, errlen, ex.what());
        return 0;
    }
}
extern "C" double ref_region_flops(const ref_region* h, int per_child) {
    return belief::flop_count_region(h->eng->region_graph(), per_child ? belief::RegionFlopMode::PerChildInverse
                                                                        : belief::RegionFlopMode::SharedInverse);
}
// check_block_convergence (region_gabp.cpp:276-309): rho of the block-norm matrix; norm 0 = Inf, 1 = Spectral
extern "C" double ref_block_convergence(const orc_matrix* M, int nblocks, const int* offs, const int* idx, int norm,
                                        int* sufficient, int* singular_block) {
    belief::BlockPartition part;
    part.blocks.resize(nblocks);
    for (int k = 0; k < nblocks; ++k) part.blocks[k].assign(idx + offs[k], idx + offs[k + 1]);
    belief::BlockConvergenceReport rep =
        belief::check_block_convergence(M->A, part, norm ? belief::BlockNorm::Spectral : belief::BlockNorm::Inf);
    if (sufficient) *sufficient = rep.sufficient ? 1 : 0;
    if (singular_block) *singular_block = rep.singular_block;
    return rep.rho;
}
