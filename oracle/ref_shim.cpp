// TEST INFRASTRUCTURE ONLY — C-ABI shim over the reference's own GaBP engine.
// Built by oracle/Makefile from the reference sources where they lie under
// /root/reference/proj/core/src/{sparse,gabp,schedule,problems,analysis}.cpp (never copied into
// this repo) into oracle/_ref/libbelief_ref.so (plus region.cpp, whose graph builder is Eigen-free).  multigrid.cpp and classic.cpp need Eigen, which
// is absent, so the multigrid / Gauss-Seidel entry points run the Eigen-free restatement in
// abi_impl.inc on top of the reference's compiled GabpEngine.
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
