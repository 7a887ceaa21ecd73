// Problem assembly for the engine's callers (input generation; host only, never on the hot path).
//
//  * assemble_named: the reference's model problems (problems.hpp:11-34, problems.cpp:34-226),
//    restated so the multigrid drop-in can rediscretise a named problem per level exactly as
//    Hierarchy does (multigrid.cpp:79-83).  tests/test_problems.py pins every problem bit for bit
//    against the reference's own assemble() compiled in oracle/_ref.
//  * the BASELINE.json configs: poisson5 (proj/tests/oracles.hpp:140-152) for configs 1-2, and the
//    generators for configs 3-5 that the reference cannot assemble; their
//    definitions are fixed in DESIGN.md §Inputs.
// RNG convention: std::mt19937(seed); uniforms through
// std::uniform_real_distribution<double>, Gaussians through std::normal_distribution<double>,
// drawn in unknown-index order, Gaussians first.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/gabp_b200.h"
#include "problems.h"

namespace {

constexpr double kPi = 3.141592653589793;  // std::numbers::pi

using F2 = std::function<double(double, double)>;

// L u = cxx u_xx + cyy u_yy + cxy u_xy + cx u_x + cy u_y with manufactured solution phi and
// g = L(phi); rows are multiplied by `sign` so the diagonal is positive (problems.cpp:48-55)
struct Model {
    F2 cxx, cyy, cxy, cx, cy, g, phi;
    double sign = 1.0;
};

double param(const std::map<std::string, double>& p, const char* k, double dflt) {
    auto it = p.find(k);
    return it == p.end() ? dflt : it->second;
}

void allow(const std::string& name, const std::map<std::string, double>& p, std::vector<std::string> keys) {
    for (const auto& kv : p)
        if (std::find(keys.begin(), keys.end(), kv.first) == keys.end())
            throw std::invalid_argument("problem '" + name + "': unknown parameter '" + kv.first + "'");
}

// the seven model problems of the paper's benchmarks (problems.cpp:73-186)
Model model(const std::string& name, const std::map<std::string, double>& p) {
    const F2 zero = [](double, double) { return 0.0; };
    const F2 one = [](double, double) { return 1.0; };
    Model d;
    d.cxy = d.cx = d.cy = zero;
    if (name == "poisson") {
        allow(name, p, {});
        d.cxx = d.cyy = [](double, double) { return -1.0; };
        d.phi = [](double x, double y) { return std::sin(kPi * x) * std::sin(kPi * y); };
        F2 phi = d.phi;
        d.g = [phi](double x, double y) { return 2.0 * kPi * kPi * phi(x, y); };
    } else if (name == "anisotropic") {
        allow(name, p, {"eps"});
        const double eps = param(p, "eps", 1e-3);
        d.cxx = [eps](double, double) { return -eps; };
        d.cyy = [](double, double) { return -1.0; };
        d.phi = [](double x, double y) { return std::sin(kPi * x) * std::sin(kPi * y); };
        F2 phi = d.phi;
        d.g = [eps, phi](double x, double y) { return kPi * kPi * (1.0 + eps) * phi(x, y); };
    } else if (name == "general") {  // smooth variable coefficients with convection
        allow(name, p, {});
        F2 a = [](double x, double y) { return std::exp(-x * (y + 2.0)) + 10.0; };
        F2 bb = [](double x, double y) {
            const double c = std::cos(2.0 * kPi * (2.0 * x + y / 2.0));
            return std::exp(-2.0 * x + 2.0 * y) * c * c + 3.0;
        };
        F2 al = [](double x, double y) { return std::cos(kPi * (x + y / 2.0)) * std::cos(2.0 * kPi * x) + 4.0; };
        F2 be = [](double x, double y) { return std::exp(2.0 * x - 2.0 * y); };
        d.cxx = a;
        d.cyy = bb;
        d.cx = al;
        d.cy = be;
        d.phi = [](double x, double y) { return std::cos(kPi * x) * std::cos(kPi * y); };
        d.g = [a, bb, al, be](double x, double y) {
            return -kPi * kPi * (a(x, y) + bb(x, y)) * std::cos(kPi * x) * std::cos(kPi * y) -
                   al(x, y) * kPi * std::sin(kPi * x) * std::cos(kPi * y) -
                   be(x, y) * kPi * std::cos(kPi * x) * std::sin(kPi * y);
        };
        d.sign = -1.0;
    } else if (name == "mixed") {  // cross derivative
        allow(name, p, {"eps"});
        const double eps = param(p, "eps", 0.01);
        d.cxx = d.cyy = one;
        d.cxy = [eps](double, double) { return 2.0 - eps; };
        d.phi = [](double x, double y) { return 2.0 * x * x * x * y * y * y * y; };
        d.g = [eps](double x, double y) {
            return 12.0 * x * y * y * y * y + 24.0 * x * x * x * y * y + (2.0 - eps) * 24.0 * x * x * y * y * y;
        };
        d.sign = -1.0;
    } else if (name == "boundary-layer") {
        allow(name, p, {"eps"});
        const double eps = param(p, "eps", 0.01);
        d.cxx = d.cyy = [eps](double, double) { return -eps; };
        d.cx = d.cy = one;
        d.phi = [eps](double x, double y) {
            return (2.0 * std::exp(-1.0 / eps) - std::exp((x - 1.0) / eps) - std::exp((y - 1.0) / eps)) /
                   (std::exp(-1.0 / eps) - 1.0);
        };
        d.g = zero;
    } else if (name == "inner-layer") {
        allow(name, p, {"eps"});
        const double eps = param(p, "eps", 0.01);
        d.cxx = d.cyy = [eps](double, double) { return eps; };
        d.cx = [](double x, double) { return x; };
        d.cy = [](double, double y) { return y; };
        d.phi = [eps](double x, double y) {
            const double s = x + y - 1.0;
            return std::exp(-s * s / eps);
        };
        F2 phi = d.phi;
        d.g = [eps, phi](double x, double y) {
            const double s = x + y - 1.0;
            return (-4.0 + (6.0 * s * s - 2.0 * s) / eps) * phi(x, y);
        };
        d.sign = -1.0;
    } else if (name == "stretched") {
        allow(name, p, {"eps", "p", "eta"});
        const double eps = param(p, "eps", 1e-6), pw = param(p, "p", 20.0), eta = param(p, "eta", 0.5);
        auto u = [eps, pw, eta](double t) { return 1.0 + std::pow((t - 0.5) * (t - 0.5) + eta, pw) / eps; };
        d.cxx = [u](double x, double) { return u(x); };
        d.cyy = [u](double, double y) { return u(y); };
        d.phi = [](double x, double y) { return std::cos(2.0 * kPi * (x + y)) * std::sin(2.0 * kPi * (x - y)); };
        d.g = [u](double x, double y) {
            const double s = 2.0 * kPi * (x + y), t = 2.0 * kPi * (x - y);
            const double cs = std::cos(s) * std::sin(t), sc = std::sin(s) * std::cos(t);
            return u(x) * (-8.0 * kPi * kPi * (cs + sc)) + u(y) * (-8.0 * kPi * kPi * (cs - sc));
        };
        d.sign = -1.0;
    } else {
        throw std::invalid_argument("unknown problem '" + name + "'");
    }
    return d;
}

// sort each row's (col, val) pairs: the canonical CSR make_csr produces when no duplicates occur
void finish_rows(bgabp_problem& P, std::vector<std::pair<int, double>>& row) {
    std::sort(row.begin(), row.end(), [](auto& a, auto& b) { return a.first < b.first; });
    for (auto& e : row) {
        P.ci.push_back(e.first);
        P.val.push_back(e.second);
    }
    P.ro.push_back((int)P.ci.size());
    row.clear();
}

void uniform_fill(std::mt19937& g, double lo, double hi, std::vector<double>& out) {
    std::uniform_real_distribution<double> u(lo, hi);
    for (double& v : out) v = u(g);
}

bgabp_problem* poisson5_problem(int nx, int ny) {  // oracles.hpp:140-152 (diag 4, off -1)
    auto* P = new bgabp_problem;
    P->n = nx * ny;
    P->nx = nx == ny ? nx : 0;
    P->ro.reserve((size_t)P->n + 1);
    P->ci.reserve((size_t)P->n * 5);
    P->val.reserve((size_t)P->n * 5);
    P->ro.push_back(0);
    for (int iy = 0; iy < ny; ++iy)
        for (int ix = 0; ix < nx; ++ix) {
            const int me = iy * nx + ix;
            auto put = [&](int c, double v) {
                P->ci.push_back(c);
                P->val.push_back(v);
            };
            if (iy > 0) put(me - nx, -1.0);
            if (ix > 0) put(me - 1, -1.0);
            put(me, 4.0);
            if (ix < nx - 1) put(me + 1, -1.0);
            if (iy < ny - 1) put(me + nx, -1.0);
            P->ro.push_back((int)P->ci.size());
        }
    return P;
}

// ---- config 3: first-order upwind convection-diffusion -Lap u + beta.grad u = f -------------
// Unit square, N x N interior points, h = 1/(N+1), homogeneous Dirichlet.  beta = |beta| (cos t,
// sin t) with cell Peclet |beta| h / 2 = Pe_cell; rows scaled by h^2, so the stencil is
// diag 4 + h(|bx|+|by|), upwind neighbours -1 - h|b_dir|, downwind neighbours -1; b = h^2 f.
bgabp_problem* upwind_problem(int N, double pe_cell, double theta, unsigned seed) {
    auto* P = new bgabp_problem;
    const double h = 1.0 / (N + 1);
    const double bmag = 2.0 * pe_cell / h;
    const double hbx = h * bmag * std::cos(theta), hby = h * bmag * std::sin(theta);
    P->n = N * N;
    P->nx = N;
    P->ro.reserve((size_t)P->n + 1);
    P->ci.reserve((size_t)P->n * 5);
    P->val.reserve((size_t)P->n * 5);
    P->ro.push_back(0);
    // upwind side: the neighbour the flow comes from
    const double w = -1.0 - std::max(hbx, 0.0), e = -1.0 - std::max(-hbx, 0.0);
    const double s = -1.0 - std::max(hby, 0.0), nn = -1.0 - std::max(-hby, 0.0);
    const double d = 4.0 + std::abs(hbx) + std::abs(hby);
    for (int iy = 0; iy < N; ++iy)
        for (int ix = 0; ix < N; ++ix) {
            const int me = iy * N + ix;
            auto put = [&](int c, double v) {
                P->ci.push_back(c);
                P->val.push_back(v);
            };
            if (iy > 0) put(me - N, s);
            if (ix > 0) put(me - 1, w);
            put(me, d);
            if (ix < N - 1) put(me + 1, e);
            if (iy < N - 1) put(me + N, nn);
            P->ro.push_back((int)P->ci.size());
        }
    std::mt19937 g(seed);
    P->b.resize(P->n);
    uniform_fill(g, 0.0, 1.0, P->b);
    for (double& v : P->b) v *= h * h;
    return P;
}

double harmonic(double a, double b) { return 2.0 * a * b / (a + b); }

// ---- config 4: 3D -div(K grad u) = f, 7-point, K = exp(g) per cell, g ~ N(0,1) i.i.d. --------
// Harmonic-mean face coefficients times the anisotropy weights (wx, wy, wz); a boundary face uses
// the cell's own K; unit spacing (no scaling); x-fastest ordering; b = f ~ U[-1,1] drawn after g.
bgabp_problem* aniso3d_problem(int N, double wx, double wy, double wz, unsigned seed) {
    auto* P = new bgabp_problem;
    const long long n = (long long)N * N * N;
    if (n * 7 > 2147483647LL) throw std::invalid_argument("config 4: grid too large for int32 CSR");
    P->n = (int)n;
    std::mt19937 g(seed);
    std::normal_distribution<double> gauss(0.0, 1.0);
    std::vector<double> K((size_t)n);
    for (double& k : K) k = std::exp(gauss(g));
    P->b.resize((size_t)n);
    uniform_fill(g, -1.0, 1.0, P->b);
    P->ro.reserve((size_t)n + 1);
    P->ci.reserve((size_t)n * 7);
    P->val.reserve((size_t)n * 7);
    P->ro.push_back(0);
    const long long NN = (long long)N * N;
    for (int iz = 0; iz < N; ++iz)
        for (int iy = 0; iy < N; ++iy)
            for (int ix = 0; ix < N; ++ix) {
                const long long me = (iz * (long long)N + iy) * N + ix;
                const double km = K[me];
                double diag = 0.0;
                double cz0 = 0, cy0 = 0, cx0 = 0, cx1 = 0, cy1 = 0, cz1 = 0;
                // faces in a fixed order: -z, -y, -x, +x, +y, +z
                auto face = [&](bool inside, long long nb, double wgt, double& coef) {
                    const double f = inside ? wgt * harmonic(km, K[nb]) : wgt * km;
                    diag += f;
                    if (inside) coef = -f;
                };
                face(iz > 0, me - NN, wz, cz0);
                face(iy > 0, me - N, wy, cy0);
                face(ix > 0, me - 1, wx, cx0);
                face(ix < N - 1, me + 1, wx, cx1);
                face(iy < N - 1, me + N, wy, cy1);
                face(iz < N - 1, me + NN, wz, cz1);
                auto put = [&](long long c, double v) {
                    P->ci.push_back((int)c);
                    P->val.push_back(v);
                };
                if (iz > 0) put(me - NN, cz0);
                if (iy > 0) put(me - N, cy0);
                if (ix > 0) put(me - 1, cx0);
                put(me, diag);
                if (ix < N - 1) put(me + 1, cx1);
                if (iy < N - 1) put(me + N, cy1);
                if (iz < N - 1) put(me + NN, cz1);
                P->ro.push_back((int)P->ci.size());
            }
    return P;
}

// ---- config 5: 2D -div(K grad u) on the vertex grid of level J, K per unknown ----------------
// Finest level: K = exp(g), g ~ N(0, sigma^2) i.i.d. per interior vertex (seed), then b ~ U[-1,1].
// Coarse levels: log K coarsened by full weighting of the 3x3 fine neighbourhood (the same
// 1/16 [1 2 1; 2 4 2; 1 2 1] weights as mg_restrict, multigrid.cpp:111-130), i.e. a weighted
// geometric mean.  Faces are harmonic means, a boundary face uses the vertex's own K, rows are
// scaled by 1/h^2 as the reference's assemble does (problems.cpp:182,211), h = 2^-J.
struct Config5Field {
    int J = -1;
    unsigned seed = 0;
    double sigma = 0;
    std::vector<std::vector<double>> logK;  // per level, finest first
    std::vector<double> b;
};

// Coarse-K rules (tools/config5_coarse_rules.py measures all four): 0 full-weighted log K (weighted
// geometric mean), 1 full-weighted K (arithmetic), 2 full-weighted 1/K (harmonic), 3 injection of
// the coinciding fine vertex.  Rule 1 is the generator's: at the configured 4095^2, sigma = 2 it is
// the only rediscretisation rule with which the reference's V(2,2) cycle reaches 1e-8 (red-black
// GaBP 291 cycles, red-black GS 711; rules 0, 2, 3 diverge -- profiles/r02_config5_*).
constexpr int kConfig5Rule = 1;
Config5Field& config5_field(int J, unsigned seed, double sigma, int levels, int rule = kConfig5Rule) {
    static Config5Field cache;
    static int cache_rule = -1;
    if (cache.J == J && cache.seed == seed && cache.sigma == sigma && cache_rule == rule &&
        (int)cache.logK.size() >= levels)
        return cache;
    cache = Config5Field();
    cache_rule = rule;
    cache.J = J;
    cache.seed = seed;
    cache.sigma = sigma;
    const int m = (1 << J) - 1;
    std::mt19937 g(seed);
    std::normal_distribution<double> gauss(0.0, sigma);
    cache.logK.emplace_back((size_t)m * m);
    for (double& v : cache.logK[0]) v = gauss(g);
    cache.b.resize((size_t)m * m);
    uniform_fill(g, -1.0, 1.0, cache.b);
    int mf = m;
    for (int k = 1; k < levels && mf >= 3; ++k) {
        const int mc = (mf - 1) / 2;
        const std::vector<double>& f = cache.logK.back();
        std::vector<double> c((size_t)mc * mc);
        for (int IY = 0; IY < mc; ++IY)
            for (int IX = 0; IX < mc; ++IX) {
                const int x = 2 * IX + 1, y = 2 * IY + 1;
                // log K -> the averaged quantity of the rule -> log K
                auto F = [&](int a, int b2) {
                    const double l = f[(size_t)b2 * mf + a];
                    return rule == 1 ? std::exp(l) : rule == 2 ? std::exp(-l) : l;
                };
                if (rule == 3) {
                    c[(size_t)IY * mc + IX] = f[(size_t)y * mf + x];
                    continue;
                }
                const double v = (4.0 * F(x, y) + 2.0 * (F(x - 1, y) + F(x + 1, y) + F(x, y - 1) + F(x, y + 1)) +
                                  F(x - 1, y - 1) + F(x + 1, y - 1) + F(x - 1, y + 1) + F(x + 1, y + 1)) /
                                 16.0;
                c[(size_t)IY * mc + IX] = rule == 1 ? std::log(v) : rule == 2 ? -std::log(v) : v;
            }
        cache.logK.push_back(std::move(c));
        mf = mc;
    }
    return cache;
}

bgabp_problem* varcoef2d_problem(int Jf, int k, unsigned seed, double sigma, int rule = kConfig5Rule) {
    Config5Field& F = config5_field(Jf, seed, sigma, Jf, rule);  // every level at once: later calls hit the cache
    if ((int)F.logK.size() <= k) throw std::invalid_argument("config 5: level below the coarsest grid");
    const int J = Jf - k, m = (1 << J) - 1;
    const double h = 1.0 / (1 << J), inv_h2 = 1.0 / (h * h);
    std::vector<double> K(F.logK[k].size());
    for (size_t i = 0; i < K.size(); ++i) K[i] = std::exp(F.logK[k][i]);
    auto* P = new bgabp_problem;
    P->n = m * m;
    P->nx = m;
    P->ro.reserve((size_t)P->n + 1);
    P->ci.reserve((size_t)P->n * 5);
    P->val.reserve((size_t)P->n * 5);
    P->ro.push_back(0);
    for (int iy = 0; iy < m; ++iy)
        for (int ix = 0; ix < m; ++ix) {
            const int me = iy * m + ix;
            const double km = K[me];
            double diag = 0.0, cs = 0, cw = 0, ce = 0, cn = 0;
            auto face = [&](bool inside, int nb, double& coef) {
                const double f = (inside ? harmonic(km, K[nb]) : km) * inv_h2;
                diag += f;
                if (inside) coef = -f;
            };
            face(iy > 0, me - m, cs);
            face(ix > 0, me - 1, cw);
            face(ix < m - 1, me + 1, ce);
            face(iy < m - 1, me + m, cn);
            auto put = [&](int c, double v) {
                P->ci.push_back(c);
                P->val.push_back(v);
            };
            if (iy > 0) put(me - m, cs);
            if (ix > 0) put(me - 1, cw);
            put(me, diag);
            if (ix < m - 1) put(me + 1, ce);
            if (iy < m - 1) put(me + m, cn);
            P->ro.push_back((int)P->ci.size());
        }
    if (k == 0) P->b = F.b;
    return P;
}

}  // namespace

// assemble(name, J, params) (problems.cpp:161-226): (2^J-1)^2 interior unknowns, h = 2^-J, rows
// scaled by 1/h^2 and by the problem's sign, Dirichlet values folded into b in stencil order.
bgabp_problem* assemble_named(const char* name_c, int J, int nparam, const char* const* keys, const double* vals,
                              std::string& err) {
    try {
        if (J < 1) throw std::invalid_argument("assemble: J must be >= 1");
        const std::string name(name_c);
        std::map<std::string, double> prm;
        for (int k = 0; k < nparam; ++k) prm[keys[k]] = vals[k];
        const Model d = model(name, prm);
        const int m = (1 << J) - 1;
        const double h = 1.0 / (1 << J);
        auto P = std::make_unique<bgabp_problem>();
        P->n = m * m;
        P->nx = m;
        P->b.assign(P->n, 0.0);
        P->exact.assign(P->n, 0.0);
        P->ro.reserve((size_t)P->n + 1);
        P->ro.push_back(0);
        const double inv_h2 = 1.0 / (h * h), inv_2h = 1.0 / (2.0 * h), inv_4h2 = 1.0 / (4.0 * h * h);
        std::vector<std::pair<int, double>> row;
        for (int iy = 0; iy < m; ++iy)
            for (int ix = 0; ix < m; ++ix) {
                const int me = iy * m + ix;
                const double x = (ix + 1) * h, y = (iy + 1) * h;
                P->exact[me] = d.phi(x, y);
                const double cxx = d.cxx(x, y), cyy = d.cyy(x, y), cxy = d.cxy(x, y);
                const double cx = d.cx(x, y), cy = d.cy(x, y), s = d.sign;
                double rhs = s * d.g(x, y);
                // stencil offsets in the reference's insertion order; zero coefficients add no entry
                const struct {
                    int dx, dy;
                    double c;
                } st[9] = {{0, 0, s * (-2.0 * cxx - 2.0 * cyy) * inv_h2},
                           {1, 0, s * (cxx * inv_h2 + cx * inv_2h)},
                           {-1, 0, s * (cxx * inv_h2 - cx * inv_2h)},
                           {0, 1, s * (cyy * inv_h2 + cy * inv_2h)},
                           {0, -1, s * (cyy * inv_h2 - cy * inv_2h)},
                           {1, 1, s * cxy * inv_4h2},
                           {-1, -1, s * cxy * inv_4h2},
                           {1, -1, -s * cxy * inv_4h2},
                           {-1, 1, -s * cxy * inv_4h2}};
                for (const auto& e : st) {
                    if (e.c == 0.0) continue;
                    const int jx = ix + e.dx, jy = iy + e.dy;
                    if (jx >= 0 && jx < m && jy >= 0 && jy < m)
                        row.emplace_back(jy * m + jx, e.c);
                    else
                        rhs -= e.c * d.phi((ix + 1 + e.dx) * h, (iy + 1 + e.dy) * h);
                }
                P->b[me] = rhs;
                finish_rows(*P, row);
            }
        return P.release();
    } catch (const std::exception& ex) {
        err = ex.what();
        return nullptr;
    }
}

extern "C" {

bgabp_problem* bgabp_problem_named(const char* name, int J, int nparam, const char* const* keys, const double* vals,
                                   char* err, size_t errlen) {
    std::string e;
    bgabp_problem* p = assemble_named(name, J, nparam, keys, vals, e);
    if (!p && err && errlen) std::snprintf(err, errlen, "%s", e.c_str());
    return p;
}

bgabp_problem* bgabp_problem_poisson5(int nx, int ny) { return poisson5_problem(nx, ny); }

// Matrix Market coordinate real general|symmetric, square (sparse.cpp:123-180): 1-based entries,
// symmetric files mirror off-diagonal entries, duplicates are summed in make_csr's order
// (std::sort of the entry indices by (row, col), sparse.cpp:36-75).
bgabp_problem* bgabp_problem_matrix_market(const char* path, char* err, size_t errlen) {
    auto fail = [&](const std::string& m) -> bgabp_problem* {
        if (err && errlen) std::snprintf(err, errlen, "%s", m.c_str());
        return nullptr;
    };
    std::FILE* f = std::fopen(path, "r");
    if (!f) return fail(std::string("cannot open ") + path);
    std::unique_ptr<std::FILE, int (*)(std::FILE*)> guard(f, std::fclose);
    char line[4096];
    if (!std::fgets(line, sizeof line, f)) return fail(std::string("empty Matrix Market file: ") + path);
    bool symmetric = false;
    std::string first(line);
    while (!first.empty() && (first.back() == '\n' || first.back() == '\r')) first.pop_back();
    if (first.rfind("%%MatrixMarket", 0) == 0) {
        char tag[64] = {0}, object[64] = {0}, format[64] = {0}, field[64] = {0}, symm[64] = {0};
        std::sscanf(first.c_str(), "%63s %63s %63s %63s %63s", tag, object, format, field, symm);
        if (std::string(object) != "matrix" || std::string(format) != "coordinate" || std::string(field) != "real")
            return fail("unsupported Matrix Market header: " + first);
        if (std::string(symm) == "symmetric")
            symmetric = true;
        else if (std::string(symm) != "general")
            return fail("unsupported symmetry: " + std::string(symm));
        if (!std::fgets(line, sizeof line, f)) return fail("truncated Matrix Market file");
    }
    while (line[0] == '%' || line[0] == '\n' || line[0] == '\r' || line[0] == 0)
        if (!std::fgets(line, sizeof line, f)) return fail("truncated Matrix Market file");
    long rows = 0, cols = 0, entries = 0;
    if (std::sscanf(line, "%ld %ld %ld", &rows, &cols, &entries) != 3) return fail(std::string("bad size line: ") + line);
    if (rows != cols) return fail("matrix is not square");
    std::vector<int> ri, ci;
    std::vector<double> vi;
    for (long k = 0; k < entries; ++k) {
        long i = 0, j = 0;
        double v = 0.0;
        if (std::fscanf(f, "%ld %ld %lf", &i, &j, &v) != 3) return fail("truncated entry list");
        if (i < 1 || i > rows || j < 1 || j > cols) return fail("entry index out of bounds");
        ri.push_back((int)(i - 1));
        ci.push_back((int)(j - 1));
        vi.push_back(v);
        if (symmetric && i != j) {
            ri.push_back((int)(j - 1));
            ci.push_back((int)(i - 1));
            vi.push_back(v);
        }
    }
    std::vector<size_t> order(ri.size());
    for (size_t k = 0; k < order.size(); ++k) order[k] = k;
    std::sort(order.begin(), order.end(),
              [&](size_t a, size_t b) { return ri[a] != ri[b] ? ri[a] < ri[b] : ci[a] < ci[b]; });
    auto* P = new bgabp_problem;
    P->n = (int)rows;
    P->ro.assign(P->n + 1, 0);
    int pr = -1, pc = -1;
    for (size_t t : order) {
        if (ri[t] == pr && ci[t] == pc) {
            P->val.back() += vi[t];
            continue;
        }
        pr = ri[t];
        pc = ci[t];
        P->ci.push_back(pc);
        P->val.push_back(vi[t]);
        ++P->ro[pr + 1];
    }
    for (int i = 0; i < P->n; ++i) P->ro[i + 1] += P->ro[i];
    return P;
}

// BASELINE.json configs; size <= 0 selects the config's own size
bgabp_problem* bgabp_problem_config(int config, int size, unsigned seed) {
    try {
        switch (config) {
            case 1:
            case 2: {
                const int N = size > 0 ? size : (config == 1 ? 64 : 2048);
                bgabp_problem* p = poisson5_problem(N, N);
                std::mt19937 g(seed);
                p->b.resize(p->n);
                uniform_fill(g, -1.0, 1.0, p->b);  // oracles.hpp:126-131
                return p;
            }
            case 3: return upwind_problem(size > 0 ? size : 1024, 2.0, 0.3, seed);
            case 4: return aniso3d_problem(size > 0 ? size : 256, 1.0, 1.0, 0.01, seed);
            case 5: {
                const int m = size > 0 ? size : 4095;
                int J = 0;
                while ((1 << J) - 1 < m) ++J;
                if ((1 << J) - 1 != m) return nullptr;
                return varcoef2d_problem(J, 0, seed, 2.0);
            }
        }
    } catch (const std::exception&) {
    }
    return nullptr;
}

bgabp_problem* bgabp_problem_config5_level(int J_fine, int k, unsigned seed) {
    return bgabp_problem_varcoef2d_level(J_fine, k, seed, 2.0);
}

bgabp_problem* bgabp_problem_varcoef2d_rule(int J_fine, int k, unsigned seed, double sigma, int rule) {
    try {
        if (rule < 0 || rule > 3) return nullptr;
        return varcoef2d_problem(J_fine, k, seed, sigma, rule);
    } catch (const std::exception&) {
        return nullptr;
    }
}

bgabp_problem* bgabp_problem_varcoef2d_level(int J_fine, int k, unsigned seed, double sigma) {
    try {
        return varcoef2d_problem(J_fine, k, seed, sigma);
    } catch (const std::exception&) {
        return nullptr;
    }
}

void bgabp_problem_free(bgabp_problem* p) { delete p; }
int bgabp_problem_n(const bgabp_problem* p) { return p->n; }
long long bgabp_problem_nnz(const bgabp_problem* p) { return (long long)p->ci.size(); }
int bgabp_problem_nx(const bgabp_problem* p) { return p->nx; }
const int* bgabp_problem_row_offsets(const bgabp_problem* p) { return p->ro.data(); }
const int* bgabp_problem_col_indices(const bgabp_problem* p) { return p->ci.data(); }
const double* bgabp_problem_values(const bgabp_problem* p) { return p->val.data(); }
const double* bgabp_problem_rhs(const bgabp_problem* p) { return p->b.empty() ? nullptr : p->b.data(); }
const double* bgabp_problem_exact(const bgabp_problem* p) { return p->exact.empty() ? nullptr : p->exact.data(); }

}  // extern "C"
