// Host side of the pipelined lexicographic sweep (seq_kernels.cuh).
#include <algorithm>

#include "engine.h"

namespace bgabp {

void Engine::launch_seq_sweep(const double* b, double2* msg, double* x, bool delta, unsigned long long* dslot,
                              int mode) {
    const int nx = grid5_nx, ny = n / grid5_nx;
    const int strips = (ny + 31) / 32;
    if (!d_progress) d_progress = static_cast<int*>(dalloc(sizeof(int) * (size_t)strips));
    ck(cudaMemsetAsync(d_progress, 0, sizeof(int) * (size_t)strips, st), "memset progress");
    SeqP P{nx, ny, n, dia.mask, dia.c, dia.diag};
    void* args[] = {&P, (void*)&b, &msg, &x, &d_progress, &d_ctrl, &dslot, &mode};
    // every strip spins on its predecessor: a cooperative launch guarantees co-residency (or fails)
    const void* fn = delta ? (const void*)k_seq_grid5<true> : (const void*)k_seq_grid5<false>;
    ck(cudaLaunchCooperativeKernel(fn, dim3(strips), dim3(32), args, 0, st), "sequential sweep launch");
}

}  // namespace bgabp
