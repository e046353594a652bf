// Device-side data structures and kernel launchers of libmrab.so (sm_100a, fp64).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace mrab {

struct DevMesh {
    int n[3];
    int periodic[3];
    int face_bc[3][2];
    int64_t npts;
    int cart;                  // constant diagonal metrics
    double cJ;                 // J = 1/J^-1 (Cartesian)
    double cM[3];              // M[k][k]    (Cartesian)
    const double* J;           // [npts] (curvilinear)
    const double* M;           // [d][d][npts] (curvilinear)
    const uint16_t* cls;       // [npts] 4 bits per direction
    const int32_t* recv_slot;  // [npts]
    const double* qhat;        // [nc][R] interpolated donor state at this mesh's receivers
    const double* fvhat;       // [d][d+1][R] interpolated donor Cartesian viscous fluxes
    int64_t nrecv;
};

struct Gas {
    double gamma, Re, Pr, wall_T;
    double q_inf[5];
    int viscous;
};

// y_out = base + c_new * R + sum_k csrc[k] * src[k]  (all [nc][npts]); r_out = R
struct Epilogue {
    double* r_out;
    double* y_out;
    const double* base;
    double c_new;
    int nsrc;
    const double* src[8];
    double csrc[8];
};

struct Box {
    int lo[3];
    int hi[3];   // inclusive
};

// receivers of one receiving mesh
struct RecvList {
    int64_t n;
    const int64_t* point;
    const int32_t* donor;
    const int32_t* base;      // [R][3]
    const double* w;          // [R][3][4]
    double* qhat;             // [nc][R]
    double* fvhat;            // [d][d+1][R]
};

struct DonorSet {             // per donor mesh: where to read state / viscous flux
    const double* state[8];
    const double* fv[8];
    int n[8][3];
    int64_t npts[8];
};

void launch_visc(int dim, const DevMesh& m, const double* Q, double* FV, const Box& box,
                 const Gas& gas, cudaStream_t st);
void launch_rhs(int dim, const DevMesh& m, const double* Q, const double* FV, const Gas& gas,
                const Epilogue& ep, cudaStream_t st);
void launch_combine(int nc, const DevMesh& m, const Box& box, const double* base, int nsrc,
                    const double* const* src, const double* csrc, double* out, cudaStream_t st);
void launch_interp(int dim, int viscous, const RecvList& rl, const DonorSet& ds, cudaStream_t st);
void upload_stencil_rows();

}  // namespace mrab
