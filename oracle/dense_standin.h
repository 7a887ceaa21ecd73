// TEST INFRASTRUCTURE ONLY — the dense direct solves that stand in for Eigen 3.x, which the
// reference links (proj/core/src/{multigrid,classic,region_gabp}.cpp: #include <Eigen/Dense>) and
// this image does not have.  Two users share this one definition so that they agree bit for bit:
//   * the restatements (abi_impl.inc: coarsest-level solve; region_restate.inc: region blocks);
//   * oracle/eigen_shim/Eigen/Dense, the minimal stand-in header over which oracle/Makefile
//     compiles the reference's own multigrid.cpp / classic.cpp / region_gabp.cpp.
// Algorithms (published; restated, not Eigen's code):
//   PartialLU  row-major partial-pivot LU; explicit inverse one unit-vector column at a time;
//              solve = inverse * b with the lane order the GPU coarse solve documents
//              (paper_1904_04093_b200/csrc/mg.cu dense_inverse + kernels.cuh k_gemv_rows: 32 lane
//              partial sums by fma over columns l, l+32, ..., xor-butterfly 16,8,4,2,1).
//   FullPivLU  complete pivoting (largest magnitude of the trailing corner scanned column by
//              column, first strict maximum), rank threshold eps * n * |max pivot| as
//              Eigen::FullPivLU documents.
// Rounding therefore differs from real Eigen's blocked kernels; everything else on the paths
// that use them is the reference's own code when built through the shim.
#pragma once
#include <cmath>
#include <cstring>
#include <limits>
#include <vector>

namespace orc_dense {

using Vec = std::vector<double>;

struct PartialLU {
    int n = 0;
    Vec lu, inv;  // row-major
    std::vector<int> piv;
    bool ok = true;
    // a: row-major n x n
    bool factor(int size, Vec a) {
        n = size;
        lu = std::move(a);
        piv.resize(n);
        ok = true;
        for (int k = 0; k < n; ++k) {
            int best = k;
            double bv = std::abs(lu[static_cast<size_t>(k) * n + k]);
            for (int i = k + 1; i < n; ++i) {
                double v = std::abs(lu[static_cast<size_t>(i) * n + k]);
                if (v > bv) {
                    bv = v;
                    best = i;
                }
            }
            piv[k] = best;
            if (best != k)
                for (int c = 0; c < n; ++c)
                    std::swap(lu[static_cast<size_t>(k) * n + c], lu[static_cast<size_t>(best) * n + c]);
            const double d = lu[static_cast<size_t>(k) * n + k];
            if (d == 0.0) {
                ok = false;
                continue;
            }
            for (int i = k + 1; i < n; ++i) {
                double& l = lu[static_cast<size_t>(i) * n + k];
                l /= d;
                if (l == 0.0) continue;
                for (int c = k + 1; c < n; ++c)
                    lu[static_cast<size_t>(i) * n + c] -= l * lu[static_cast<size_t>(k) * n + c];
            }
        }
        inv.assign(static_cast<size_t>(n) * n, 0.0);
        Vec e(n);
        for (int c = 0; c < n; ++c) {
            std::fill(e.begin(), e.end(), 0.0);
            e[c] = 1.0;
            const Vec col = substitute(e);
            for (int i = 0; i < n; ++i) inv[static_cast<size_t>(i) * n + c] = col[i];
        }
        return ok;
    }
    // LU substitution for one right-hand side
    Vec substitute(const Vec& b) const {
        Vec y = b;
        for (int k = 0; k < n; ++k)
            if (piv[k] != k) std::swap(y[k], y[piv[k]]);
        for (int i = 0; i < n; ++i) {
            double acc = y[i];
            for (int c = 0; c < i; ++c) acc -= lu[static_cast<size_t>(i) * n + c] * y[c];
            y[i] = acc;
        }
        for (int i = n - 1; i >= 0; --i) {
            double acc = y[i];
            for (int c = i + 1; c < n; ++c) acc -= lu[static_cast<size_t>(i) * n + c] * y[c];
            y[i] = acc / lu[static_cast<size_t>(i) * n + i];
        }
        return y;
    }
    // x = inv * b, row by row in the GPU's lane order
    void solve(const double* b, double* x) const {
        for (int i = 0; i < n; ++i) {
            const double* row = inv.data() + static_cast<size_t>(i) * n;
            double lane[32];
            for (int l = 0; l < 32; ++l) {
                double acc = 0.0;
                for (int c = l; c < n; c += 32) acc = std::fma(row[c], b[c], acc);
                lane[l] = acc;
            }
            for (int o = 16; o > 0; o >>= 1) {
                double nxt[32];
                for (int l = 0; l < 32; ++l) nxt[l] = lane[l] + lane[l ^ o];
                std::memcpy(lane, nxt, sizeof lane);
            }
            x[i] = lane[0];
        }
    }
    Vec solve(const Vec& b) const {
        Vec x(n);
        solve(b.data(), x.data());
        return x;
    }
};

// Complete-pivoting LU of a dense square matrix (column-major, like Eigen's MatrixXd).
struct FullPivLU {
    int n = 0, nonzero = 0;
    Vec a;                    // a[i + j*n]
    std::vector<int> rt, ct;  // row / column transpositions
    double maxpivot = 0.0;
    double& at(int i, int j) { return a[static_cast<size_t>(j) * n + i]; }
    double at(int i, int j) const { return a[static_cast<size_t>(j) * n + i]; }
    FullPivLU() = default;
    explicit FullPivLU(const Vec& colmajor, int size) : n(size), a(colmajor) {
        rt.assign(n, 0);
        ct.assign(n, 0);
        nonzero = n;
        for (int k = 0; k < n; ++k) {
            int bi = k, bj = k;
            double best = -1.0;
            for (int j = k; j < n; ++j)  // maxCoeff visits column by column, first strict maximum
                for (int i = k; i < n; ++i) {
                    const double v = std::abs(at(i, j));
                    if (v > best) best = v, bi = i, bj = j;
                }
            if (best == 0.0) {
                nonzero = k;
                for (int i = k; i < n; ++i) rt[i] = ct[i] = i;
                break;
            }
            if (best > maxpivot) maxpivot = best;
            rt[k] = bi;
            ct[k] = bj;
            if (bi != k)
                for (int j = 0; j < n; ++j) std::swap(at(k, j), at(bi, j));
            if (bj != k)
                for (int i = 0; i < n; ++i) std::swap(at(i, k), at(i, bj));
            const double p = at(k, k);
            for (int i = k + 1; i < n; ++i) at(i, k) /= p;
            for (int j = k + 1; j < n; ++j)
                for (int i = k + 1; i < n; ++i) at(i, j) -= at(i, k) * at(k, j);
        }
    }
    int rank() const {
        const double thr = std::numeric_limits<double>::epsilon() * n * std::abs(maxpivot);
        int r = 0;
        for (int i = 0; i < nonzero; ++i)
            if (std::abs(at(i, i)) > thr) ++r;
        return r;
    }
    bool invertible() const { return rank() == n; }
    Vec solve(const Vec& b) const {
        const int r = rank();
        Vec x(n, 0.0);
        if (r == 0) return x;
        Vec c = b;
        for (int k = 0; k < n; ++k) std::swap(c[k], c[rt[k]]);  // P b
        for (int k = 0; k < n; ++k)                               // unit lower, column-oriented
            for (int i = k + 1; i < n; ++i) c[i] -= at(i, k) * c[k];
        for (int k = r - 1; k >= 0; --k) {  // upper on the leading r x r block
            c[k] /= at(k, k);
            for (int i = 0; i < k; ++i) c[i] -= at(i, k) * c[k];
        }
        std::vector<int> q(n);  // column i of the factored matrix is original column q[i]
        for (int i = 0; i < n; ++i) q[i] = i;
        for (int k = 0; k < n; ++k) std::swap(q[k], q[ct[k]]);
        for (int i = 0; i < r; ++i) x[q[i]] = c[i];
        return x;
    }
    Vec inverse() const {  // column-major
        Vec inv(static_cast<size_t>(n) * n);
        Vec e(n, 0.0);
        for (int j = 0; j < n; ++j) {
            e.assign(n, 0.0);
            e[j] = 1.0;
            Vec col = solve(e);
            std::copy(col.begin(), col.end(), inv.begin() + static_cast<size_t>(j) * n);
        }
        return inv;
    }
};

}  // namespace orc_dense
