// Host-side problem assembly (input generation, L3 of SURVEY.md §1): not on the hot path.
#pragma once

#include <string>
#include <vector>

struct bgabp_problem {
    int n = 0;
    int nx = 0;  // interior points per axis of a square 2D grid (0 otherwise)
    std::vector<int> ro, ci;
    std::vector<double> val, b, exact;
};

bgabp_problem* assemble_named(const char* name, int J, int nparam, const char* const* keys,
                              const double* vals, std::string& err);
