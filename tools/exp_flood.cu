// Tuning experiment (not part of the product): times variants of the fused flood solve step of
// paper_1904_04093_b200/csrc/kernels.cuh on a symmetric grid Laplacian in the DIA layout.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -fmad=false -o tools/exp_flood tools/exp_flood.cu
//   tools/exp_flood 2 2048      (2-D, 2048^2, S = 4)      tools/exp_flood 3 256   (3-D, 256^3, S = 6)
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_1904_04093_b200/csrc/kernels.cuh"

using namespace bgabp;

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            std::exit(1);                                                                  \
        }                                                                                  \
    } while (0)

template <class T>
T* up(const std::vector<T>& v) {
    T* d;
    CK(cudaMalloc(&d, sizeof(T) * v.size()));
    CK(cudaMemcpy(d, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
    return d;
}

template <int S>
void run(int N) {
    const int dims = S / 2;
    long long nn = 1;
    for (int d = 0; d < dims; ++d) nn *= N;
    const int n = (int)nn;
    DiaP P;
    std::memset(&P, 0, sizeof(P));
    P.n = n;
    P.j0 = 0;
    P.j1 = n;
    P.gofs = 0;
    P.S = S;
    P.nneg = S / 2;
    std::vector<int> st;
    int stride = 1;
    for (int d = 0; d < dims; ++d) {
        st.push_back(stride);
        stride *= N;
    }
    for (int s = 0; s < S; ++s) {
        P.off[s] = s < S / 2 ? -st[S / 2 - 1 - s] : st[s - S / 2];
        P.rev[s] = S - 1 - s;
    }
    std::vector<uint32_t> mask(n);
    std::vector<double> c((size_t)S * n, 0.0), diag(n, 2.0 * dims + 0.01), b(n);
    long long E = 0;
    std::vector<int> co(dims);
    for (int j = 0; j < n; ++j) {
        int rem = j;
        for (int d = 0; d < dims; ++d) {
            co[d] = rem % N;
            rem /= N;
        }
        for (int s = 0; s < S; ++s) {
            const int d = s < S / 2 ? (S / 2 - 1 - s) : (s - S / 2);
            const bool ok = s < S / 2 ? co[d] > 0 : co[d] < N - 1;
            if (ok) {
                mask[j] |= (1u << s) | (1u << (16 + s));
                c[(size_t)s * n + j] = -1.0;
                ++E;
            }
        }
        b[j] = std::sin(0.001 * j);
    }
    P.mask = up(mask);
    P.c = up(c);
    P.rowv = P.c;
    P.diag = up(diag);
    double* db = up(b);
    double2 *m0, *m1;
    double *xr, *hist;
    CK(cudaMalloc(&m0, sizeof(double2) * S * n));
    CK(cudaMalloc(&m1, sizeof(double2) * S * n));
    CK(cudaMemset(m0, 0, sizeof(double2) * S * n));
    CK(cudaMemset(m1, 0, sizeof(double2) * S * n));
    CK(cudaMalloc(&xr, sizeof(double) * kXRing * n));
    CK(cudaMemset(xr, 0, sizeof(double) * kXRing * n));
    CK(cudaMalloc(&hist, sizeof(double) * 100000));
    Ctrl* ctrl;
    unsigned long long* spread;
    CK(cudaMalloc(&ctrl, sizeof(Ctrl)));
    CK(cudaMalloc(&spread, 8 * 64 * 8));
    CK(cudaMemset(spread, 0, 8 * 64 * 8));
    auto reset = [&]() {
        Ctrl h;
        std::memset(&h, 0, sizeof(h));
        for (int q = 0; q < 4; ++q) h.epiv[q] = h.npiv[q] = kNone;
        h.opiv = kNone;
        h.step = 1;
        h.r0 = 1.0;
        h.tol = 0.0;
        h.divergence = 1e300;
        h.max_iter = 1 << 30;
        CK(cudaMemcpy(ctrl, &h, sizeof(h), cudaMemcpyHostToDevice));
    };
    const unsigned g = (n + 255) / 256;
    const double bytes = 40.0 * E + 32.0 * n;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int steps = 40;
    auto timeit = [&](const char* name, auto&& launch) {
        reset();
        for (int k = 0; k < 5; ++k) launch();
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        for (int k = 0; k < steps; ++k) launch();
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        CK(cudaGetLastError());
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double us = ms * 1e3 / steps;
        std::printf("S=%d %-44s %8.2f us/step  %7.1f GB/s  %.3f of 6557\n", S, name, us, bytes / us / 1e3,
                    bytes / us / 1e3 / 6557.4);
    };
#define W(NAME, MINB, DEFER, UNC)                                                                             \
    timeit(NAME, [&] {                                                                                        \
        k_flood_solve_dia<S, false, true, MINB, DEFER, UNC><<<g, 256>>>(P, db, m0, m1, xr, ctrl, spread); \
        k_solve_decide_lag2<<<1, 64>>>(ctrl, hist, spread);                                                   \
    });
#define U(NAME, MINB, DEFER)                                                                                 \
    timeit(NAME, [&] {                                                                                        \
        P.uniform = 1;                                                                                        \
        k_flood_solve_dia<S, false, true, MINB, DEFER, true, true><<<g, 256>>>(P, db, m0, m1, xr, ctrl, spread); \
        k_solve_decide_lag2<<<1, 64>>>(ctrl, hist, spread);                                                   \
        P.uniform = 0;                                                                                        \
    });
    for (int s = 0; s < S; ++s) P.cu[s] = -1.0;
    P.du = 2.0 * dims + 0.01;
    U("UNIF MINB=4 DEFER", 4, true)
    U("UNIF MINB=3 DEFER", 3, true)
    U("UNIF MINB=4 early-x", 4, false)
    U("UNIF MINB=3 early-x", 3, false)
    U("UNIF MINB=2 early-x", 2, false)
    U("UNIF MINB=5 early-x", 5, false)
    U("UNIF MINB=5 DEFER", 5, true)
    U("UNIF MINB=6 early-x", 6, false)
    U("UNIF MINB=6 DEFER", 6, true)
    timeit("NONSYM MINB=3 early-x", [&] {
        k_flood_solve_dia<S, false, false, 3, false, true><<<g, 256>>>(P, db, m0, m1, xr, ctrl, spread);
        k_solve_decide_lag2<<<1, 64>>>(ctrl, hist, spread);
    });
    W("MINB=4 DEFER predicated", 4, true, false)
    W("MINB=4 DEFER unconditional", 4, true, true)
    W("MINB=3 DEFER unconditional", 3, true, true)
    W("MINB=4 early-x unconditional", 4, false, true)
    W("MINB=3 early-x unconditional", 3, false, true)
    W("MINB=2 early-x unconditional", 2, false, true)
    timeit("MINB=3 early-x unconditional DELTA", [&] {
        k_flood_solve_dia<S, true, true, 3, false, true><<<g, 256>>>(P, db, m0, m1, xr, ctrl, spread);
        k_solve_decide_lag2<<<1, 64>>>(ctrl, hist, spread);
    });
    cudaFree(m0);
    cudaFree(m1);
}

int main(int argc, char** argv) {
    const int dims = argc > 1 ? std::atoi(argv[1]) : 2;
    const int N = argc > 2 ? std::atoi(argv[2]) : 2048;
    if (dims == 2) run<4>(N);
    if (dims == 3) run<6>(N);
    return 0;
}
