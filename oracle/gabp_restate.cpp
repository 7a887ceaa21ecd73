// TEST INFRASTRUCTURE ONLY — CPU restatement of the reference's GaBP hot path, used as the
// checker for the CUDA product.  Never linked into or called by the product library
// (paper_1904_04093_b200/); only tests/, __graft_entry__.smoke() and bench.py's CPU legs load it.
//
// Parity pin: every routine below is checked bit-for-bit against the reference's own sources
// compiled from /root/reference (oracle/_ref/libbelief_ref.so, recipe oracle/Makefile) and
// against the committed golden vectors in tests/golden/ (made by tests/golden/make_golden.py).
//
// Arithmetic order is the contract: sums run in CSR column order, products are rounded before
// they are added (the reference builds with plain -O3 on x86-64, so no FMA contraction; this
// file is built with -ffp-contract=off to keep it that way on any host).
//
// Citations are to /root/reference/proj/... (core/src unless a directory is given).

#include <algorithm>
#include <cmath>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace orc {

using Vector = std::vector<double>;

// ---------------------------------------------------------------------------------------------
// Sparse storage — sparse.hpp:17-39, sparse.cpp:26-75,104-121
// ---------------------------------------------------------------------------------------------
struct SparseMatrix {
    int n = 0;
    std::vector<int> row_offsets, col_indices;
    Vector values;
    std::vector<int> transpose_pos;  // CSR position of (j,i) for entry (i,j), -1 if absent

    int nnz() const { return static_cast<int>(values.size()); }
    // binary search inside row `row` (sparse.cpp:26-32)
    int find(int row, int col) const {
        const int* lo = col_indices.data() + row_offsets[row];
        const int* hi = col_indices.data() + row_offsets[row + 1];
        const int* it = std::lower_bound(lo, hi, col);
        return (it != hi && *it == col) ? static_cast<int>(it - col_indices.data()) : -1;
    }
    double at(int row, int col) const {
        int p = find(row, col);
        return p >= 0 ? values[p] : 0.0;
    }
};

void fill_transpose_pos(SparseMatrix& A) {  // sparse.cpp:70-74
    A.transpose_pos.assign(A.values.size(), -1);
    for (int r = 0; r < A.n; ++r)
        for (int p = A.row_offsets[r]; p < A.row_offsets[r + 1]; ++p)
            A.transpose_pos[p] = A.find(A.col_indices[p], r);
}

// make_csr (sparse.cpp:36-75): sort (row, col) with the same std::sort comparator, so that
// duplicates are summed in the same order, then accumulate duplicates into the last entry.
SparseMatrix make_csr(int n, const std::vector<int>& rows, const std::vector<int>& cols,
                      const Vector& vals) {
    if (rows.size() != cols.size() || rows.size() != vals.size())
        throw std::invalid_argument("make_csr: triplet arrays differ in length");
    const size_t nt = rows.size();
    for (size_t k = 0; k < nt; ++k)
        if (rows[k] < 0 || rows[k] >= n || cols[k] < 0 || cols[k] >= n)
            throw std::out_of_range("make_csr: index out of bounds");
    std::vector<size_t> idx(nt);
    std::iota(idx.begin(), idx.end(), size_t{0});
    std::sort(idx.begin(), idx.end(), [&](size_t a, size_t b) {
        return rows[a] != rows[b] ? rows[a] < rows[b] : cols[a] < cols[b];
    });
    SparseMatrix A;
    A.n = n;
    A.row_offsets.assign(n + 1, 0);
    int pr = -1, pc = -1;
    for (size_t t : idx) {
        if (rows[t] == pr && cols[t] == pc) {
            A.values.back() += vals[t];
            continue;
        }
        pr = rows[t];
        pc = cols[t];
        A.col_indices.push_back(pc);
        A.values.push_back(vals[t]);
        ++A.row_offsets[pr + 1];
    }
    std::partial_sum(A.row_offsets.begin(), A.row_offsets.end(), A.row_offsets.begin());
    fill_transpose_pos(A);
    return A;
}

// residual_inf_norm (sparse.cpp:104-115): acc = b_i, then acc -= a*x in CSR order; std::max
// keeps the running value when |acc| is NaN.
double residual_inf_norm(const SparseMatrix& A, const Vector& x, const Vector& b) {
    if (static_cast<int>(x.size()) != A.n || static_cast<int>(b.size()) != A.n)
        throw std::invalid_argument("residual_inf_norm: dimension mismatch");
    double worst = 0.0;
    // (std::max never takes a NaN into `worst`, so the maximum is order-free: threads on large n)
#pragma omp parallel for schedule(static, 4096) reduction(max : worst) if (A.n >= (1 << 16))
    for (int i = 0; i < A.n; ++i) {
        double acc = b[i];
        for (int p = A.row_offsets[i]; p < A.row_offsets[i + 1]; ++p)
            acc -= A.values[p] * x[A.col_indices[p]];
        worst = std::max(worst, std::abs(acc));
    }
    return worst;
}

double inf_norm(const Vector& v) {  // sparse.cpp:117-121
    double worst = 0.0;
    for (double e : v) worst = std::max(worst, std::abs(e));
    return worst;
}

// ---------------------------------------------------------------------------------------------
// Schedules — schedule.hpp:9-38, schedule.cpp:11-103
// ---------------------------------------------------------------------------------------------
enum class ScheduleKind { ParallelFlood, SequentialLexicographic, RedBlack, FourColor, CustomOrder };

struct Schedule {
    ScheduleKind kind = ScheduleKind::SequentialLexicographic;
    std::vector<int> order, color_of;
    int num_colors = 1;

    // colour-grouped order: stable sort of 0..n-1 by colour (schedule.cpp:11-22)
    static Schedule grouped(ScheduleKind k, std::vector<int> colors, int nc) {
        Schedule s;
        s.kind = k;
        s.num_colors = nc;
        s.color_of = std::move(colors);
        s.order.resize(s.color_of.size());
        std::iota(s.order.begin(), s.order.end(), 0);
        std::stable_sort(s.order.begin(), s.order.end(),
                         [&](int a, int b) { return s.color_of[a] < s.color_of[b]; });
        return s;
    }
    static Schedule parallel_flood() {
        Schedule s;
        s.kind = ScheduleKind::ParallelFlood;
        return s;
    }
    static Schedule sequential(int n) {
        Schedule s;
        s.order.resize(n);
        std::iota(s.order.begin(), s.order.end(), 0);
        return s;
    }
    static Schedule custom(std::vector<int> order) {  // schedule.cpp:65-76
        std::vector<char> hit(order.size(), 0);
        for (int v : order) {
            if (v < 0 || v >= static_cast<int>(order.size()) || hit[v])
                throw std::invalid_argument("Schedule::custom: order is not a permutation");
            hit[v] = 1;
        }
        Schedule s;
        s.kind = ScheduleKind::CustomOrder;
        s.order = std::move(order);
        return s;
    }
    static Schedule red_black_grid(int nx, int ny) {  // colour (ix+iy) mod 2
        std::vector<int> c(static_cast<size_t>(nx) * ny);
        for (int iy = 0; iy < ny; ++iy)
            for (int ix = 0; ix < nx; ++ix) c[static_cast<size_t>(iy) * nx + ix] = (ix + iy) & 1;
        return grouped(ScheduleKind::RedBlack, std::move(c), 2);
    }
    static Schedule four_color_grid(int nx, int ny) {  // colour 2(iy mod 2)+(ix mod 2)
        std::vector<int> c(static_cast<size_t>(nx) * ny);
        for (int iy = 0; iy < ny; ++iy)
            for (int ix = 0; ix < nx; ++ix)
                c[static_cast<size_t>(iy) * nx + ix] = 2 * (iy & 1) + (ix & 1);
        return grouped(ScheduleKind::FourColor, std::move(c), 4);
    }
    // greedy first-fit colouring of the undirected structure (schedule.cpp:25-47)
    static std::vector<int> greedy(const SparseMatrix& A, int& nc) {
        std::vector<std::vector<int>> nb(A.n);
        for (int i = 0; i < A.n; ++i)
            for (int p = A.row_offsets[i]; p < A.row_offsets[i + 1]; ++p) {
                int j = A.col_indices[p];
                if (j == i) continue;
                nb[i].push_back(j);
                nb[j].push_back(i);
            }
        std::vector<int> col(A.n, -1);
        nc = 1;
        std::vector<char> taken;
        for (int i = 0; i < A.n; ++i) {
            taken.assign(nc + 1, 0);
            for (int j : nb[i])
                if (col[j] >= 0 && col[j] < static_cast<int>(taken.size())) taken[col[j]] = 1;
            int c = 0;
            while (c < static_cast<int>(taken.size()) && taken[c]) ++c;
            col[i] = c;
            nc = std::max(nc, c + 1);
        }
        return col;
    }
    static Schedule red_black(const SparseMatrix& A) {
        int nc = 0;
        auto c = greedy(A, nc);
        return grouped(ScheduleKind::RedBlack, std::move(c), nc);
    }
    static Schedule four_color(const SparseMatrix& A) {
        int nc = 0;
        auto c = greedy(A, nc);
        return grouped(ScheduleKind::FourColor, std::move(c), nc);
    }
};

// ---------------------------------------------------------------------------------------------
// GaBP engine — gabp.hpp:12-111, gabp.cpp:8-419
// ---------------------------------------------------------------------------------------------
enum class SolveStatus { Converged, Diverged, MaxIter };
enum class StopCriterion { Residual, MessageDelta };

struct SolveReport {  // report.hpp:21-28
    SolveStatus status = SolveStatus::MaxIter;
    int iterations = 0;
    Vector residual_history;
    double flop_estimate = 0.0;
    Vector solution;
    std::string detail;
};

struct GabpOptions {  // gabp.hpp:39-45 (pivot_floor is never read by the engine)
    double tol = 2e-4;
    int max_iter = 20000;
    StopCriterion stop = StopCriterion::Residual;
    double pivot_floor = 1e-300;
    double divergence_factor = 1e12;
};

struct MessageState {
    Vector lambda_tilde, m;
};

struct FrozenLambda {
    Vector lambda_tilde, sigma;
    bool converged = false;
    int iterations = 0;
};

class GabpEngine {
public:
    // Edge j->i lives at the CSR position of A_ij; out-edges of j are column j's off-diagonal
    // entries in ascending row order (gabp.cpp:8-27).
    explicit GabpEngine(const SparseMatrix& A) : A_(A), out_(A.n), diag_(A.n, -1) {
        for (int i = 0; i < A.n; ++i)
            for (int p = A.row_offsets[i]; p < A.row_offsets[i + 1]; ++p) {
                int j = A.col_indices[p];
                if (j == i) {
                    diag_[i] = p;
                } else {
                    out_[j].push_back({p, i});
                    ++num_edges_;
                }
            }
        for (int i = 0; i < A.n; ++i)  // gabp.cpp:29-33
            if (diag_[i] < 0)
                throw std::invalid_argument("gabp: matrix has a structurally zero diagonal entry");
    }

    long num_edges() const { return num_edges_; }

    MessageState make_state() const {  // gabp.cpp:35-40
        MessageState s;
        s.lambda_tilde.assign(A_.nnz(), 0.0);
        s.m.assign(A_.nnz(), 0.0);
        return s;
    }

    // sweep dispatcher (gabp.cpp:42-47)
    bool sweep(const Vector& b, const Schedule& s, MessageState& st, Vector& x,
               std::string* err = nullptr) const {
        return s.kind == ScheduleKind::ParallelFlood ? flood(b, st, x, err, nullptr)
                                                      : ordered(b, s.order, st, x, err, nullptr);
    }

    double sweep_flops() const {  // gabp.cpp:165-172: n + 3E + 4E
        double e = static_cast<double>(num_edges_);
        return A_.n + 3.0 * e + 4.0 * e;
    }

    // solve loop (gabp.cpp:174-219)
    SolveReport solve(const Vector& b, const Schedule& s, const GabpOptions& o) const {
        SolveReport rep;
        MessageState st = make_state();
        Vector x(A_.n, 0.0);
        const double r0 = inf_norm(b);
        rep.residual_history.push_back(r0);
        if (r0 <= o.tol) {
            rep.status = SolveStatus::Converged;
            rep.solution = x;
            return rep;
        }
        std::string err;
        const bool is_flood = s.kind == ScheduleKind::ParallelFlood;
        for (int it = 1; it <= o.max_iter; ++it) {
            double delta = 0.0;
            bool ok = is_flood ? flood(b, st, x, &err, &delta) : ordered(b, s.order, st, x, &err, &delta);
            rep.iterations = it;
            if (!ok) {
                rep.status = SolveStatus::Diverged;
                rep.detail = err;
                rep.solution = x;
                return rep;
            }
            double r = residual_inf_norm(A_, x, b);
            rep.residual_history.push_back(r);
            rep.flop_estimate += sweep_flops() + 2.0 * A_.nnz();
            if (!std::isfinite(r) || r > o.divergence_factor * r0) {
                rep.status = SolveStatus::Diverged;
                rep.detail = "residual blowup";
                rep.solution = x;
                return rep;
            }
            if (o.stop == StopCriterion::Residual ? (r <= o.tol) : (delta <= o.tol)) {
                rep.status = SolveStatus::Converged;
                rep.solution = x;
                return rep;
            }
        }
        rep.status = SolveStatus::MaxIter;
        rep.solution = x;
        return rep;
    }

    // lambda-only sweeps to a fixed point, then node precisions (gabp.cpp:221-287)
    FrozenLambda precompute_lambda(const Schedule& s, double tol = 1e-10, int max_iter = 500) const {
        FrozenLambda out;
        Vector& lam = out.lambda_tilde;
        lam.assign(A_.nnz(), 0.0);
        const bool is_flood = s.kind == ScheduleKind::ParallelFlood;
        if (!is_flood && static_cast<int>(s.order.size()) != A_.n)
            throw std::invalid_argument("gabp: schedule order does not cover every node");
        Vector snap;
        for (int it = 1; it <= max_iter; ++it) {
            double delta = 0.0;
            if (is_flood) snap = lam;
            const Vector& src = is_flood ? snap : lam;
            for (int q = 0; q < A_.n; ++q) {
                const int j = is_flood ? q : s.order[q];
                const double sig = precision_of(j, src);
                for (const Out& e : out_[j]) {
                    const double a = A_.values[e.pos];
                    const int tp = A_.transpose_pos[e.pos];
                    const double den = sig - (tp >= 0 ? src[tp] : 0.0) * a;
                    if (std::abs(den) < kPivotFloor) {
                        out.converged = false;
                        out.iterations = it;
                        return out;
                    }
                    const double nl = -a / den;
                    delta = std::max(delta, std::abs(nl - lam[e.pos]));
                    lam[e.pos] = nl;
                }
            }
            out.iterations = it;
            if (delta <= tol) {
                out.converged = true;
                break;
            }
            if (!std::isfinite(delta)) break;
        }
        out.sigma.assign(A_.n, 0.0);
        for (int j = 0; j < A_.n; ++j) out.sigma[j] = precision_of(j, lam);
        return out;
    }

    // mean-only sweeps with frozen precisions, cold messages (gabp.cpp:289-325)
    Vector correction_sweeps(const Vector& r, const Schedule& s, const FrozenLambda& fz,
                             int sweeps) const {
        Vector m(A_.nnz(), 0.0), snap, e(A_.n, 0.0);
        const bool is_flood = s.kind == ScheduleKind::ParallelFlood;
        if (!is_flood && static_cast<int>(s.order.size()) != A_.n)
            throw std::invalid_argument("gabp: schedule order does not cover every node");
        for (int k = 0; k < sweeps; ++k) {
            if (is_flood) snap = m;
            const Vector& src = is_flood ? snap : m;
            for (int q = 0; q < A_.n; ++q) {
                const int j = is_flood ? q : s.order[q];
                const double acc = mean_of(j, r[j], src);
                if (!is_flood) e[j] = acc / fz.sigma[j];
                for (const Out& o : out_[j]) {
                    const int tp = A_.transpose_pos[o.pos];
                    m[o.pos] = fz.lambda_tilde[o.pos] * (acc - (tp >= 0 ? src[tp] : 0.0));
                }
            }
        }
        if (is_flood)
            for (int i = 0; i < A_.n; ++i) e[i] = mean_of(i, r[i], m) / fz.sigma[i];
        return e;
    }

    // residual r = b - A x0 in CSR order (gabp.cpp:327-335)
    Vector residual_vector(const Vector& b, const Vector& x0) const {
        Vector r(A_.n);
        for (int i = 0; i < A_.n; ++i) {
            double acc = b[i];
            for (int p = A_.row_offsets[i]; p < A_.row_offsets[i + 1]; ++p)
                acc -= A_.values[p] * x0[A_.col_indices[p]];
            r[i] = acc;
        }
        return r;
    }

    Vector error_correction_apply(const Vector& b, const Vector& x0, int sweeps, const Schedule& s,
                                  const FrozenLambda& fz) const {  // gabp.cpp:327-341
        Vector e = correction_sweeps(residual_vector(b, x0), s, fz, sweeps);
        Vector x = x0;
        for (int i = 0; i < A_.n; ++i) x[i] += e[i];
        return x;
    }

    Vector error_correction_apply(const Vector& b, const Vector& x0, int sweeps,
                                  const Schedule& s) const {  // gabp.cpp:343-361
        Vector r = residual_vector(b, x0);
        MessageState st = make_state();
        Vector e(A_.n, 0.0);
        std::string err;
        for (int k = 0; k < sweeps; ++k)
            if (!sweep(r, s, st, e, &err)) throw std::runtime_error("gabp error correction: " + err);
        Vector x = x0;
        for (int i = 0; i < A_.n; ++i) x[i] += e[i];
        return x;
    }

    SolveReport solve_error_correction(const Vector& b, const Schedule& s, int sweeps,
                                       const FrozenLambda& fz, const GabpOptions& o) const {
        SolveReport rep;  // gabp.cpp:363-401
        Vector x(A_.n, 0.0);
        const double r0 = inf_norm(b);
        rep.residual_history.push_back(r0);
        if (r0 <= o.tol) {
            rep.status = SolveStatus::Converged;
            rep.solution = x;
            return rep;
        }
        const double e = static_cast<double>(num_edges_);
        const double per_iter = 2.0 * A_.nnz() + sweeps * (A_.n + 1.0 * e + 3.0 * e);
        for (int it = 1; it <= o.max_iter; ++it) {
            x = error_correction_apply(b, x, sweeps, s, fz);
            const double r = residual_inf_norm(A_, x, b);
            rep.residual_history.push_back(r);
            rep.iterations = it;
            rep.flop_estimate += per_iter + 2.0 * A_.nnz();
            if (!std::isfinite(r) || r > o.divergence_factor * r0) {
                rep.status = SolveStatus::Diverged;
                rep.detail = "residual blowup";
                rep.solution = x;
                return rep;
            }
            if (r <= o.tol) {
                rep.status = SolveStatus::Converged;
                rep.solution = x;
                return rep;
            }
        }
        rep.status = SolveStatus::MaxIter;
        rep.solution = x;
        return rep;
    }

    Vector node_precisions(const MessageState& st) const {  // gabp.cpp:403-419
        Vector beta(A_.n);
        for (int j = 0; j < A_.n; ++j) beta[j] = precision_of(j, st.lambda_tilde);
        return beta;
    }

private:
    struct Out {
        int pos;  // CSR position of A_ij
        int dst;  // i
    };
    static constexpr double kPivotFloor = 1e-300;  // gabp.hpp:110

    // sigma_j: CSR-order sum over row j; diagonal adds A_jj, off-diagonal p adds
    // lam[p] * A[tp(p)] when the transpose entry exists (gabp.cpp:59-70, 403-419).
    double precision_of(int j, const Vector& lam) const {
        double sig = 0.0;
        for (int p = A_.row_offsets[j]; p < A_.row_offsets[j + 1]; ++p) {
            if (A_.col_indices[p] == j) {
                sig += A_.values[p];
            } else if (A_.transpose_pos[p] >= 0) {
                sig += lam[p] * A_.values[A_.transpose_pos[p]];
            }
        }
        return sig;
    }
    // m-bar_j: b_j plus every incoming mean in CSR order (gabp.cpp:296-299, 314-318)
    double mean_of(int j, double bj, const Vector& m) const {
        double acc = bj;
        for (int p = A_.row_offsets[j]; p < A_.row_offsets[j + 1]; ++p)
            if (A_.col_indices[p] != j) acc += m[p];
        return acc;
    }
    // both aggregates in one pass, same per-accumulator order as the reference loop
    void aggregate(int j, double bj, const MessageState& st, double& sig, double& acc) const {
        sig = 0.0;
        acc = bj;
        for (int p = A_.row_offsets[j]; p < A_.row_offsets[j + 1]; ++p) {
            if (A_.col_indices[p] == j) {
                sig += A_.values[p];
                continue;
            }
            acc += st.m[p];
            const int tp = A_.transpose_pos[p];
            if (tp >= 0) sig += st.lambda_tilde[p] * A_.values[tp];
        }
    }
    // one outgoing message j->i from node aggregates and the reverse message (gabp.cpp:77-96)
    bool emit(int j, const Out& o, double sig, double acc, const MessageState& src,
              MessageState& dst, std::string* err, double* delta, bool damp = false) const {
        const double a = A_.values[o.pos];
        const int tp = A_.transpose_pos[o.pos];
        const double lr = tp >= 0 ? src.lambda_tilde[tp] : 0.0;
        const double mr = tp >= 0 ? src.m[tp] : 0.0;
        const double den = sig - lr * a;
        if (std::abs(den) < kPivotFloor) {
            if (err) *err = "zero pivot on edge " + std::to_string(j) + "->" + std::to_string(o.dst);
            return false;
        }
        double nl = -a / den;
        double nm = nl * (acc - mr);
        if (damp) {  // extension (no reference counterpart): convex blend with the old message
            nl = undamp_ * nl + damping_ * src.lambda_tilde[o.pos];
            nm = undamp_ * nm + damping_ * src.m[o.pos];
        }
        if (delta) {
            *delta = std::max(*delta, std::abs(nl - src.lambda_tilde[o.pos]));
            *delta = std::max(*delta, std::abs(nm - src.m[o.pos]));
        }
        dst.lambda_tilde[o.pos] = nl;
        dst.m[o.pos] = nm;
        return true;
    }

    // in-place sweep in schedule order, x_j before j's out-edges (gabp.cpp:49-100)
    bool ordered(const Vector& b, const std::vector<int>& order, MessageState& st, Vector& x,
                 std::string* err, double* max_delta) const {
        if (static_cast<int>(order.size()) != A_.n)
            throw std::invalid_argument("gabp: schedule order does not cover every node");
        double delta = 0.0;
        for (int j : order) {
            double sig, acc;
            aggregate(j, b[j], st, sig, acc);
            if (std::abs(sig) < kPivotFloor) {
                if (err) *err = "zero pivot at node " + std::to_string(j);
                return false;
            }
            x[j] = acc / sig;
            // in place: the delta compares against the value being overwritten, which is the
            // same element the reference reads (state.*[e.pos] before assignment)
            for (const Out& o : out_[j])
                if (!emit(j, o, sig, acc, st, st, err, max_delta ? &delta : nullptr)) return false;
        }
        if (max_delta) *max_delta = delta;
        return true;
    }

    // synchronous sweep from a snapshot, x from the new messages (gabp.cpp:102-163)
    // Large systems: the same sweep evaluated by OpenMP threads.  Every node's arithmetic is the
    // serial one on the same snapshot (a parallel flood evaluation is bit-identical
    // to the serial one), the delta is a max of non-NaN values (order-free); a breakdown restores
    // the state and reruns the serial sweep, which reproduces the reference's partial updates.
    static constexpr int kParallelMin = 1 << 16;
    static void par_copy(std::vector<double>& dst, const std::vector<double>& src) {
        dst.resize(src.size());
        const long nn = static_cast<long>(src.size());
#pragma omp parallel for schedule(static)
        for (long q = 0; q < nn; q += 65536)
            std::copy(src.begin() + q, src.begin() + std::min(nn, q + 65536), dst.begin() + q);
    }
    bool flood_parallel(const Vector& b, MessageState& st, Vector& x, double* max_delta) const {
        MessageState& prev = snap_;
        par_copy(prev.lambda_tilde, st.lambda_tilde);
        par_copy(prev.m, st.m);
        int fail = 0;
        double delta = 0.0;
#pragma omp parallel for schedule(static, 4096) reduction(max : delta) reduction(| : fail)
        for (int j = 0; j < A_.n; ++j) {
            double sig, acc, d = 0.0;
            aggregate(j, b[j], prev, sig, acc);
            for (const Out& o : out_[j])
                if (!emit(j, o, sig, acc, prev, st, nullptr, max_delta ? &d : nullptr, damping_ != 0.0)) fail = 1;
            delta = std::max(delta, d);
        }
        Vector& xt = xtmp_;
        xt.resize(A_.n);
        if (!fail) {
#pragma omp parallel for schedule(static, 4096) reduction(| : fail)
            for (int i = 0; i < A_.n; ++i) {
                double sig, acc;
                aggregate(i, b[i], st, sig, acc);
                if (std::abs(sig) < kPivotFloor) fail = 1;
                else xt[i] = acc / sig;
            }
        }
        if (fail) {
            par_copy(st.lambda_tilde, prev.lambda_tilde);
            par_copy(st.m, prev.m);
            return false;
        }
        par_copy(x, xt);
        if (max_delta) *max_delta = delta;
        return true;
    }

    bool flood(const Vector& b, MessageState& st, Vector& x, std::string* err,
               double* max_delta) const {
        if (A_.n >= kParallelMin && flood_parallel(b, st, x, max_delta)) return true;
        const MessageState prev = st;
        double delta = 0.0;
        for (int j = 0; j < A_.n; ++j) {
            double sig, acc;
            aggregate(j, b[j], prev, sig, acc);
            for (const Out& o : out_[j])
                if (!emit(j, o, sig, acc, prev, st, err, max_delta ? &delta : nullptr, damping_ != 0.0)) return false;
        }
        for (int i = 0; i < A_.n; ++i) {
            double sig, acc;
            aggregate(i, b[i], st, sig, acc);
            if (std::abs(sig) < kPivotFloor) {
                if (err) *err = "zero pivot at node " + std::to_string(i);
                return false;
            }
            x[i] = acc / sig;
        }
        if (max_delta) *max_delta = delta;
        return true;
    }

    const SparseMatrix& A_;
    std::vector<std::vector<Out>> out_;
    std::vector<int> diag_;
    long num_edges_ = 0;
    double damping_ = 0.0, undamp_ = 1.0;
    mutable MessageState snap_;  // flood_parallel scratch (the snapshot) and x of the sweep
    mutable Vector xtmp_;

public:
    // Optional message damping of the flood sweep (BASELINE.json north_star; the reference has
    // none): every new message becomes (1 - a) * new + a * old on its edge; 0 = the reference.
    void set_damping(double a) {
        damping_ = a;
        undamp_ = 1.0 - a;
    }
};

// ---------------------------------------------------------------------------------------------
// Analytic smoother cost per unknown — analysis.cpp:135-154 (analysis.hpp:49-57)
// ---------------------------------------------------------------------------------------------
enum class FlopStencil { FivePoint, NinePoint };
enum class FlopSmoother { Gabp, LineGabp, Gs, XyGs };

double flop_table(FlopStencil stencil, FlopSmoother smoother, int sweeps) {
    if (sweeps < 1) throw std::invalid_argument("flop_table: sweeps must be >= 1");
    const double M = sweeps;
    const bool five = stencil == FlopStencil::FivePoint;
    if (smoother == FlopSmoother::Gabp) return five ? 12.0 * M + 6.0 : 24.0 * M + 8.0;
    if (smoother == FlopSmoother::LineGabp) {
        if (!five)
            throw std::invalid_argument(
                "flop_table: line regions do not cover the nine-point stencil's diagonal couplings");
        return sweeps == 1 ? 38.0 : 28.0 * M + 9.0;
    }
    if (smoother == FlopSmoother::Gs) return five ? 9.0 * M : 17.0 * M;
    return five ? 14.0 * M : 21.0 * M;  // XyGs
}

// ---------------------------------------------------------------------------------------------
// Computation-tree oracle — analysis.cpp:160-215
// ---------------------------------------------------------------------------------------------
double computation_tree_solve(const SparseMatrix& A, const Vector& b, int root, int depth,
                              long node_cap) {
    if (root < 0 || root >= A.n) throw std::out_of_range("computation tree: root out of range");
    struct TNode {
        int var, parent;
    };
    std::vector<TNode> t{{root, -1}};
    size_t begin = 0;
    for (int d = 0; d < depth; ++d) {  // breadth-first unrolling, never straight back to parent
        const size_t end = t.size();
        for (size_t q = begin; q < end; ++q) {
            const int v = t[q].var;
            const int pv = t[q].parent < 0 ? -1 : t[t[q].parent].var;
            for (int p = A.row_offsets[v]; p < A.row_offsets[v + 1]; ++p) {
                const int k = A.col_indices[p];
                if (k == v || k == pv) continue;
                t.push_back({k, static_cast<int>(q)});
                if (static_cast<long>(t.size()) > node_cap)
                    throw std::length_error("computation tree exceeds node cap");
            }
        }
        begin = end;
    }
    Vector dg(t.size()), rh(t.size());
    for (size_t q = 0; q < t.size(); ++q) {
        dg[q] = A.at(t[q].var, t[q].var);
        rh[q] = b[t[q].var];
    }
    for (size_t c = t.size(); c-- > 1;) {  // eliminate leaves into parents
        const int par = t[c].parent;
        const double a_pc = A.at(t[par].var, t[c].var);
        const double a_cp = A.at(t[c].var, t[par].var);
        if (dg[c] == 0.0) throw std::runtime_error("computation tree: zero pivot");
        dg[par] -= a_pc * a_cp / dg[c];
        rh[par] -= a_pc * rh[c] / dg[c];
    }
    if (dg[0] == 0.0) throw std::runtime_error("computation tree: zero pivot at root");
    return rh[0] / dg[0];
}

// ---------------------------------------------------------------------------------------------
// Seeded test-input generators — restated from proj/tests/oracles.hpp:36-172 and
// proj/tests/acceptance.cpp:29-49 (libstdc++ mt19937 + distributions, same draw order).
// ---------------------------------------------------------------------------------------------
struct Triplets {
    std::vector<int> r, c;
    Vector v;
    void add(int i, int j, double x) {
        r.push_back(i);
        c.push_back(j);
        v.push_back(x);
    }
};

SparseMatrix random_diag_dominant(int n, std::mt19937& g, bool sym, double p) {
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    std::bernoulli_distribution coin(p);
    Triplets t;
    Vector rs(n, 0.0);
    for (int i = 0; i < n; ++i)
        for (int j = sym ? i + 1 : 0; j < n; ++j) {
            if (j == i || !coin(g)) continue;
            const double a = u(g);
            t.add(i, j, a);
            rs[i] += std::abs(a);
            rs[j] += std::abs(a);
            if (sym) {
                t.add(j, i, a);
                continue;
            }
            const double w = u(g);
            if (coin(g)) {  // the reverse entry is sometimes dropped entirely
                t.add(j, i, w);
                rs[j] += std::abs(w);
                rs[i] += std::abs(w);
            }
        }
    std::uniform_real_distribution<double> bump(0.5, 1.5);
    for (int i = 0; i < n; ++i) t.add(i, i, rs[i] + bump(g));
    return make_csr(n, t.r, t.c, t.v);
}

SparseMatrix random_tree(int n, std::mt19937& g, std::vector<std::pair<int, int>>* edges) {
    std::uniform_real_distribution<double> u(0.2, 1.0);
    Triplets t;
    Vector rs(n, 0.0);
    for (int v = 1; v < n; ++v) {
        std::uniform_int_distribution<int> pick(0, v - 1);
        const int w = pick(g);
        const double a = u(g);
        const double c = u(g);
        t.add(w, v, a);
        t.add(v, w, c);
        rs[w] += std::abs(a);
        rs[v] += std::abs(c);
        if (edges) edges->emplace_back(w, v);
    }
    std::uniform_real_distribution<double> bump(0.5, 1.5);
    for (int i = 0; i < n; ++i) t.add(i, i, rs[i] + bump(g));
    return make_csr(n, t.r, t.c, t.v);
}

SparseMatrix random_cycle_chords(int n, std::mt19937& g) {
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    std::bernoulli_distribution coin(0.2);
    Triplets t;
    Vector rs(n, 0.0);
    auto link = [&](int i, int j) {
        const double a = u(g);
        const double c = u(g);
        t.add(i, j, a);
        t.add(j, i, c);
        rs[i] += std::abs(a);
        rs[j] += std::abs(c);
    };
    for (int i = 0; i < n; ++i) link(i, (i + 1) % n);
    for (int i = 0; i < n; ++i)
        for (int j = i + 2; j < n; ++j)
            if (!(i == 0 && j == n - 1) && coin(g)) link(i, j);
    std::uniform_real_distribution<double> bump(0.5, 1.5);
    for (int i = 0; i < n; ++i) t.add(i, i, rs[i] + bump(g));
    return make_csr(n, t.r, t.c, t.v);
}

SparseMatrix poisson5(int nx, int ny) {  // oracles.hpp:140-152, same triplet order
    Triplets t;
    for (int iy = 0; iy < ny; ++iy)
        for (int ix = 0; ix < nx; ++ix) {
            const int me = iy * nx + ix;
            t.add(me, me, 4.0);
            if (ix > 0) t.add(me, me - 1, -1.0);
            if (ix < nx - 1) t.add(me, me + 1, -1.0);
            if (iy > 0) t.add(me, me - nx, -1.0);
            if (iy < ny - 1) t.add(me, me + nx, -1.0);
        }
    return make_csr(nx * ny, t.r, t.c, t.v);
}

SparseMatrix example7x7() {  // oracles.hpp:157-172
    static const double M[7][7] = {
        {10, 1.5, 2, 2, 0, 2, 0}, {2, 4, 2.5, 0, 2, 0, 0}, {2, 3, 5, 0, 0, 0, 1},
        {2, 0, 0, 10, 0.5, 1, 0}, {0, 2, 0, 0.5, 5, 0, 1}, {2, 0, 0, 1, 0, 7, 1},
        {0, 0, 1, 0, 1, 1, 2},
    };
    Triplets t;
    for (int i = 0; i < 7; ++i)
        for (int j = 0; j < 7; ++j)
            if (M[i][j] != 0.0) t.add(i, j, M[i][j]);
    return make_csr(7, t.r, t.c, t.v);
}

int tree_diameter(int n, const std::vector<std::pair<int, int>>& edges) {  // oracles.hpp:101-124
    std::vector<std::vector<int>> adj(n);
    for (auto [a, b] : edges) {
        adj[a].push_back(b);
        adj[b].push_back(a);
    }
    auto farthest = [&](int s) {
        std::vector<int> dist(n, -1);
        std::vector<int> q{s};
        dist[s] = 0;
        for (size_t h = 0; h < q.size(); ++h)
            for (int w : adj[q[h]])
                if (dist[w] < 0) {
                    dist[w] = dist[q[h]] + 1;
                    q.push_back(w);
                }
        int far = s;
        for (int i = 0; i < n; ++i)
            if (dist[i] > dist[far]) far = i;
        return std::make_pair(far, dist[far]);
    };
    return farthest(farthest(0).first).second;
}

}  // namespace orc

// ---- shared C-ABI bodies (also compiled over the reference in oracle/ref_shim.cpp) ----------
namespace abi_ns = orc;
inline long abi_num_edges(const orc::GabpEngine& e) { return e.num_edges(); }
#define ORC_HAVE_GENERATORS 1
#define ABI_HAS_DAMPING 1
#include "abi_impl.inc"
