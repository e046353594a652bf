// SBP 2-4 diagonal-norm first-derivative rows by stencil class code, in constant memory
// (one copy per translation unit).  Class 0 hole, 1 interior (offsets -2..2), 2..5 left
// closure rows 0..3, 6..9 right closure rows 0..3 (D[N-1-r][N-1-c] = -D[r][c]).
// Coefficients: the diagonal-norm 2-4 operator of [mattsson2004stable] cited at P:205-208.
#pragma once
namespace mrab {
static __constant__ int c_nst[10] = {0, 4, 4, 2, 4, 4, 4, 2, 4, 4};
static __constant__ int c_off[10][4] = {{0, 0, 0, 0},   {-2, -1, 1, 2}, {0, 1, 2, 3},  {-1, 1, 0, 0},
                                        {-2, -1, 1, 2}, {-3, -1, 1, 2}, {0, -1, -2, -3}, {1, -1, 0, 0},
                                        {2, 1, -1, -2}, {3, 1, -1, -2}};
static __constant__ double c_cf[10][4] = {
    {0, 0, 0, 0},
    {1.0 / 12, -2.0 / 3, 2.0 / 3, -1.0 / 12},
    {-24.0 / 17, 59.0 / 34, -4.0 / 17, -3.0 / 34},
    {-0.5, 0.5, 0, 0},
    {4.0 / 43, -59.0 / 86, 59.0 / 86, -4.0 / 43},
    {3.0 / 98, -59.0 / 98, 32.0 / 49, -4.0 / 49},
    {24.0 / 17, -59.0 / 34, 4.0 / 17, 3.0 / 34},
    {0.5, -0.5, 0, 0},
    {-4.0 / 43, 59.0 / 86, -59.0 / 86, 4.0 / 43},
    {-3.0 / 98, 59.0 / 98, -32.0 / 49, 4.0 / 49}};
}  // namespace mrab
