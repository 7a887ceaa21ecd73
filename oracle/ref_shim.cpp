// TEST INFRASTRUCTURE ONLY — C-ABI shim over the reference's own GaBP engine.
// Built by oracle/Makefile from the reference sources where they lie under
// /root/reference/proj/core/src/{sparse,gabp,schedule,problems,analysis}.cpp (never copied into
// this repo) into oracle/_ref/libbelief_ref.so.  multigrid.cpp and classic.cpp need Eigen, which
// is absent, so the multigrid / Gauss-Seidel entry points run the Eigen-free restatement in
// abi_impl.inc on top of the reference's compiled GabpEngine.
#include "belief/analysis.hpp"
#include "belief/gabp.hpp"
#include "belief/problems.hpp"
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
