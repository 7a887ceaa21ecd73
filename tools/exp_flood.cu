// Tuning experiment (not part of the product): times the flood-sweep kernel variants of
// paper_1904_04093_b200/csrc/kernels.cuh on poisson5(N,N) in the DIA layout.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -fmad=false -o tools/exp_flood tools/exp_flood.cu
//   tools/exp_flood [N]
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

int main(int argc, char** argv) {
    const int N = argc > 1 ? std::atoi(argv[1]) : 2048;
    const int n = N * N, S = 4;
    DiaP P;
    std::memset(&P, 0, sizeof(P));
    P.n = n;
    P.S = S;
    P.nneg = 2;
    const int off[4] = {-N, -1, 1, N};
    for (int s = 0; s < 4; ++s) {
        P.off[s] = off[s];
        P.rev[s] = 3 - s;
    }
    std::vector<uint32_t> mask(n);
    std::vector<double> c((size_t)S * n, 0.0), diag(n, 4.0), b(n);
    for (int iy = 0; iy < N; ++iy)
        for (int ix = 0; ix < N; ++ix) {
            const int j = iy * N + ix;
            const bool ok[4] = {iy > 0, ix > 0, ix < N - 1, iy < N - 1};
            for (int s = 0; s < 4; ++s)
                if (ok[s]) {
                    mask[j] |= (1u << s) | (1u << (16 + s));
                    c[(size_t)s * n + j] = -1.0;
                }
            b[j] = std::sin(0.001 * j);
        }
    P.mask = up(mask);
    P.c = up(c);
    P.rowv = P.c;
    P.diag = up(diag);
    double* db = up(b);
    double2 *m0, *m1;
    double *x0, *x1, *hist;
    CK(cudaMalloc(&m0, sizeof(double2) * S * n));
    CK(cudaMalloc(&m1, sizeof(double2) * S * n));
    CK(cudaMemset(m0, 0, sizeof(double2) * S * n));
    CK(cudaMemset(m1, 0, sizeof(double2) * S * n));
    CK(cudaMalloc(&x0, sizeof(double) * n));
    CK(cudaMalloc(&x1, sizeof(double) * n));
    CK(cudaMalloc(&hist, sizeof(double) * 100000));
    Ctrl* ctrl;
    unsigned int* arrive;
    CK(cudaMalloc(&ctrl, sizeof(Ctrl)));
    CK(cudaMalloc(&arrive, sizeof(unsigned int)));
    CK(cudaMemset(arrive, 0, 4));
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
    const double bytes = 40.0 * (4.0 * n - 4.0 * N) + 24.0 * n;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int steps = 60;
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
        std::printf("%-58s %8.2f us/step  %7.1f GB/s (B_sweep)  %.3f of 6557\n", name, us, bytes / us / 1e3,
                    bytes / us / 1e3 / 6557.4);
    };
    int par = 0;
    timeit("flood plain (x write), 256 thr", [&] {
        k_flood_dia<4, false><<<g, 256>>>(P, db, par ? m1 : m0, par ? m0 : m1, x0, ctrl, MODE_PLAIN);
        par ^= 1;
    });
    timeit("residual alone", [&] { k_residual_dia<4><<<g, 256>>>(P, db, x0, nullptr, &ctrl->red[0], ctrl, MODE_PLAIN); });
    unsigned long long* spread;
    CK(cudaMalloc(&spread, 8 * 64 * 8));
    CK(cudaMemset(spread, 0, 8 * 64 * 8));
#define V(MINB, DEFER)                                                                                     \
    timeit("fused MINB=" #MINB " DEFER=" #DEFER, [&] {                                                    \
        k_flood_solve_dia<4, false, true, MINB, DEFER><<<g, 256>>>(P, db, m0, m1, x0, x1, ctrl, spread); \
        k_solve_decide_lag2<<<1, 64>>>(ctrl, hist, spread);                                              \
    });
    V(4, true)
    timeit("fused MINB=4 ASYNC", [&] {
        k_flood_solve_dia<4, false, true, 4, true, true, true><<<g, 256>>>(P, db, m0, m1, x0, x1, ctrl, spread);
        k_solve_decide_lag2<<<1, 64>>>(ctrl, hist, spread);
    });
    timeit("fused MINB=3 ASYNC", [&] {
        k_flood_solve_dia<4, false, true, 3, true, true, true><<<g, 256>>>(P, db, m0, m1, x0, x1, ctrl, spread);
        k_solve_decide_lag2<<<1, 64>>>(ctrl, hist, spread);
    });
    timeit("fused MINB=4 DELTA", [&] {
        k_flood_solve_dia<4, true, true, 4, true><<<g, 256>>>(P, db, m0, m1, x0, x1, ctrl, spread);
        k_solve_decide_lag2<<<1, 64>>>(ctrl, hist, spread);
    });
    return 0;
}
