// gabp_solve — command-line front-end of the B200 GaBP path over the C-ABI (include/gabp_b200.h),
// following the reference CLI's single-run contract (proj/tools/belief_solve.cpp:79-165,392-462):
// the same options for a GaBP or multigrid run, the `iteration,residual_inf` CSV with %.17g
// (belief_solve.cpp:149-156), the stderr summary line and the exit codes 0 converged / 2 diverged
// / 3 max_iter / 1 error (belief_solve.cpp:158-165).  Solvers: gabp, generalized-gabp (line-region
// GaBP, belief_solve.cpp:115-124) and mg:<smoother> incl. mg:line-gabp; suites and the classical
// solvers are outside this path.  Inputs: a named model problem (--problem/--J/--param), a Matrix
// Market file (--matrix, with --rhs ones|random|<file>), or a BASELINE.json config (--config).
// Every solve runs on the GPU; there is no CPU fallback.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/gabp_b200.h"

namespace {

struct Spec {
    std::string problem = "poisson", matrix, rhs = "ones", solver = "gabp", schedule = "sequential", out;
    std::map<std::string, double> params;
    int J = 6, config = 0, size = 0, max_iter = 20000, J1 = 0, J2 = 0, pre = 1, post = 1;
    double tol = 2e-4;
    unsigned seed = 0;
};

[[noreturn]] void usage(const char* msg) {
    std::cerr << "error: " << msg << "\n"
              << "usage: gabp_solve [--problem NAME --J J --param k=v ... | --matrix FILE.mtx [--rhs ones|random|FILE]"
                 " | --config 1..5 [--size N]]\n"
                 "                  [--solver gabp|mg:<sequential-gabp|red-black-gabp|4-color-gabp|parallel-gabp|"
                 "gs|red-black-gs|4-color-gs|jacobi>] [--schedule sequential|parallel-flood|red-black|four-color]\n"
                 "                  [--tol T] [--max-iter K] [--cycle V:J1,J2] [--pre n] [--post m] [--out FILE]"
                 " [--seed S]\n";
    std::exit(1);
}

const char* status_name(int s) { return s == 0 ? "converged" : s == 1 ? "diverged" : "max_iter"; }
int exit_code(int s) { return s == 0 ? 0 : s == 1 ? 2 : 3; }

struct Problem {
    bgabp_problem* p = nullptr;
    ~Problem() {
        if (p) bgabp_problem_free(p);
    }
};

void write_csv(const std::vector<double>& hist, std::ostream& os) {  // belief_solve.cpp:149-156
    os << "iteration,residual_inf\n";
    char buf[64];
    for (size_t i = 0; i < hist.size(); ++i) {
        std::snprintf(buf, sizeof buf, "%zu,%.17g\n", i, hist[i]);
        os << buf;
    }
}

int smoother_id(const std::string& name) {  // belief_solve.cpp:58-75 (point smoothers)
    static const std::map<std::string, int> t = {
        {"sequential-gabp", 0}, {"red-black-gabp", 1}, {"4-color-gabp", 2}, {"flood-gabp", 3},
        {"line-gabp", 4},       {"jacobi", 5},         {"gs", 6},           {"red-black-gs", 7},
        {"4-color-gs", 8}};
    auto it = t.find(name);
    if (it == t.end()) throw std::invalid_argument("unknown multigrid smoother '" + name + "'");
    return it->second;
}

}  // namespace

int main(int argc, char** argv) {
    Spec s;
    std::string cycle;
    for (int i = 1; i < argc; ++i) {
        const std::string a = argv[i];
        auto val = [&]() -> std::string {
            if (i + 1 >= argc) usage(("missing value for " + a).c_str());
            return argv[++i];
        };
        if (a == "--problem") s.problem = val();
        else if (a == "--J") s.J = std::atoi(val().c_str());
        else if (a == "--param") {
            const std::string kv = val();
            const auto eq = kv.find('=');
            if (eq == std::string::npos) usage(("--param expects k=v, got '" + kv + "'").c_str());
            s.params[kv.substr(0, eq)] = std::stod(kv.substr(eq + 1));
        } else if (a == "--matrix") s.matrix = val();
        else if (a == "--rhs") s.rhs = val();
        else if (a == "--config") s.config = std::atoi(val().c_str());
        else if (a == "--size") s.size = std::atoi(val().c_str());
        else if (a == "--solver") s.solver = val();
        else if (a == "--schedule") s.schedule = val();
        else if (a == "--tol") s.tol = std::stod(val());
        else if (a == "--max-iter") s.max_iter = std::atoi(val().c_str());
        else if (a == "--cycle") cycle = val();
        else if (a == "--pre") s.pre = std::atoi(val().c_str());
        else if (a == "--post") s.post = std::atoi(val().c_str());
        else if (a == "--out") s.out = val();
        else if (a == "--seed") s.seed = (unsigned)std::strtoul(val().c_str(), nullptr, 10);
        else if (a == "--help" || a == "-h") usage("help requested");
        else usage(("unknown option " + a).c_str());
    }
    try {
        if (!cycle.empty() && (std::sscanf(cycle.c_str(), "V:%d,%d", &s.J1, &s.J2) != 2 || s.J1 <= 0 || s.J2 <= 0))
            throw std::invalid_argument("--cycle expects V:J1,J2");
        char err[512] = {0};
        std::vector<double> hist;
        bgabp_report rep{};
        std::string detail;
        int n = 0;
        if (s.solver.rfind("mg:", 0) == 0) {  // belief_solve.cpp:82-96
            if (s.J1 == 0) throw std::invalid_argument("a multigrid solver needs --cycle V:J1,J2");
            std::vector<const char*> keys;
            std::vector<double> vals;
            for (auto& kv : s.params) {
                keys.push_back(kv.first.c_str());
                vals.push_back(kv.second);
            }
            bgmg* h = nullptr;
            int rc = bgmg_create_named(s.problem.c_str(), s.J1, s.J2, (int)keys.size(), keys.data(), vals.data(),
                                       smoother_id(s.solver.substr(3)), &h, err, sizeof err);
            if (rc != BGABP_OK) throw std::runtime_error(err);
            n = bgmg_level_n(h, 0);
            std::vector<double> b(n), x(n);
            bgmg_fine_rhs(h, b.data());
            hist.assign((size_t)s.max_iter + 2, 0.0);
            bgmg_cycle spec{s.pre, s.post, 0};
            bgmg_options o{s.tol, s.max_iter, 1e6};
            char det[512] = {0};
            rc = bgmg_solve(h, &spec, b.data(), &o, &rep, x.data(), hist.data(), det, sizeof det);
            bgmg_destroy(h);
            if (rc != BGABP_OK) throw std::runtime_error(det);
            detail = det;
        } else if (s.solver == "gabp" || s.solver == "generalized-gabp") {  // belief_solve.cpp:101-106, 115-124
            Problem P;
            if (!s.matrix.empty())
                P.p = bgabp_problem_matrix_market(s.matrix.c_str(), err, sizeof err);
            else if (s.config > 0)
                P.p = bgabp_problem_config(s.config, s.size, s.seed ? s.seed : (unsigned)(s.config - 1));
            else {
                std::vector<const char*> keys;
                std::vector<double> vals;
                for (auto& kv : s.params) {
                    keys.push_back(kv.first.c_str());
                    vals.push_back(kv.second);
                }
                P.p = bgabp_problem_named(s.problem.c_str(), s.J, (int)keys.size(), keys.data(), vals.data(), err,
                                          sizeof err);
            }
            if (!P.p) throw std::invalid_argument(err[0] ? err : "cannot build the problem");
            n = bgabp_problem_n(P.p);
            std::vector<double> b(n, 1.0), x(n);
            if (const double* rb = bgabp_problem_rhs(P.p)) {
                b.assign(rb, rb + n);
            } else if (s.rhs == "random") {
                std::mt19937 g(s.seed);
                std::uniform_real_distribution<double> u(-1.0, 1.0);
                for (auto& v : b) v = u(g);
            } else if (s.rhs != "ones") {
                std::ifstream f(s.rhs);
                if (!f) throw std::runtime_error("cannot open " + s.rhs);
                for (auto& v : b)
                    if (!(f >> v)) throw std::runtime_error("right-hand side file too short");
            }
            const int nx = bgabp_problem_nx(P.p);
            if (s.solver == "generalized-gabp") {  // RegionGabpEngine over grid_line_regions
                if (nx <= 0 || (long long)nx * nx != n)
                    throw std::invalid_argument("generalized-gabp needs a square grid problem");
                bglin_engine* le = nullptr;
                int rc = bglin_create(n, bgabp_problem_row_offsets(P.p), bgabp_problem_col_indices(P.p),
                                      bgabp_problem_values(P.p), nx, nx, &le, err, sizeof err);
                if (rc != BGABP_OK) throw std::invalid_argument(err);
                hist.assign((size_t)std::max(s.max_iter, 0) + 2, 0.0);
                bglin_options o{s.tol, s.max_iter, s.schedule == "parallel-flood" ? 1 : 0, 1e12};
                char det[512] = {0};
                rc = bglin_solve(le, b.data(), &o, &rep, x.data(), hist.data(), det, sizeof det);
                bglin_destroy(le);
                if (rc != BGABP_OK) throw std::runtime_error(det);
                detail = det;
            } else {
                bgabp_schedule sch{};
                if (s.schedule == "sequential") sch.kind = BGABP_SCHED_SEQUENTIAL;
                else if (s.schedule == "parallel-flood") sch.kind = BGABP_SCHED_FLOOD;
                else if (s.schedule == "red-black") sch = {BGABP_SCHED_RED_BLACK_GRID, nx, nx, nullptr};
                else if (s.schedule == "four-color") sch = {BGABP_SCHED_FOUR_COLOR_GRID, nx, nx, nullptr};
                else throw std::invalid_argument("unknown schedule '" + s.schedule + "'");
                if ((sch.kind == BGABP_SCHED_RED_BLACK_GRID || sch.kind == BGABP_SCHED_FOUR_COLOR_GRID) && nx == 0)
                    sch.kind = sch.kind == BGABP_SCHED_RED_BLACK_GRID ? BGABP_SCHED_RED_BLACK : BGABP_SCHED_FOUR_COLOR;
                bgabp_engine* e = nullptr;
                int rc = bgabp_create(n, bgabp_problem_row_offsets(P.p), bgabp_problem_col_indices(P.p),
                                      bgabp_problem_values(P.p), BGABP_LAYOUT_AUTO, &e, err, sizeof err);
                if (rc != BGABP_OK) throw std::invalid_argument(err);
                hist.assign((size_t)std::max(s.max_iter, 0) + 2, 0.0);
                bgabp_options o{s.tol, s.max_iter, BGABP_STOP_RESIDUAL, 1e12};
                char det[512] = {0};
                rc = bgabp_solve(e, b.data(), &sch, &o, &rep, x.data(), hist.data(), det, sizeof det);
                bgabp_destroy(e);
                if (rc != BGABP_OK) throw std::runtime_error(det);
                detail = det;
            }
        } else {
            throw std::invalid_argument("solver '" + s.solver +
                                        "' is not on the GPU path (gabp | generalized-gabp | mg:<smoother>)");
        }
        // a failed sweep / cycle (pivot, smoother breakdown) pushes no residual: the reference's
        // history then has `iterations` entries (gabp.cpp:193-199, multigrid.cpp:288-297)
        const bool failed = rep.status == BGABP_DIVERGED && !detail.empty() && detail != "residual blowup";
        hist.resize((size_t)rep.iterations + (failed ? 0 : 1));
        if (!s.out.empty()) {
            std::ofstream f(s.out);
            if (!f) throw std::runtime_error("cannot open " + s.out);
            write_csv(hist, f);
        } else {
            write_csv(hist, std::cout);
        }
        char buf[256];
        std::snprintf(buf, sizeof buf, "status=%s iterations=%d flops_per_n=%.17g final_residual=%.17g n=%d\n",
                      status_name(rep.status), rep.iterations, n ? rep.flop_estimate / n : 0.0,
                      hist.empty() ? 0.0 : hist.back(), n);
        std::cerr << buf;
        if (!detail.empty()) std::cerr << "detail: " << detail << "\n";
        return exit_code(rep.status);
    } catch (const std::exception& ex) {
        std::cerr << "error: " << ex.what() << "\n";
        return 1;
    }
}
