// Internal declarations of libmrab.so (host setup, device kernels, context).
// Product code: shares nothing with oracle/ (see DESIGN.md §1).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/mrab.h"

namespace mrab {

constexpr int kMaxMeshes = 8;
constexpr int kMaxHist = 6;
constexpr int kFar = 1 << 30;

// stencil class codes, 4 bits per direction (reading R2: segment closures)
enum : int { CLS_HOLE = 0, CLS_INT = 1, CLS_L0 = 2, CLS_R0 = 6 };

// Tuning / diagnostic switches of the library.  Defaults are the
// measured-best paths; the hot path reads no environment itself: the MRAB_* variables are read
// in one place (read_options, at mrab_plan_create), stored in the plan, and installed as the
// current options by every entry point that launches kernels (set_options).
struct Options {
    int overlap = 1;          // MRAB_OVERLAP: critical/bulk split of slow meshes on two streams
    int bulk_ctas = 0;        // MRAB_BULK_CTAS: >0 = persistent CTAs for bulk launches
    int lean = 1;             // MRAB_LEAN: 2-D interior tiles take the lean path
    int tile_flags = 1;       // MRAB_TILE_FLAGS: 0 = no tile flagged interior
    int k2d = -2;             // MRAB_K2D: force a 2-D tile variant (-2 = per mesh)
    long small_pts = 100000;  // MRAB_SMALL_PTS: curvilinear meshes up to this size use 32x8 tiles
    int curv_half = 1;        // MRAB_CURV_HALF: curvilinear 2-D tiles capped at 128 registers
    int pf = 1;               // MRAB_PF: L2 prefetch of the general tile's epilogue rows
    int donor_staged = 1;     // MRAB_DONOR_STAGED: region-staged 2-D donor gather
    int interp_box = 1;       // MRAB_INTERP_BOX: 3-D gather staged per donor box
    int interp_quad = 1;      // MRAB_INTERP_QUAD: four lanes per receiver (per-receiver 3-D gather)
    int z3_fused = 0;         // MRAB_3D_FUSED: 3-D RHS in one pass (k_rhs3z) instead of two
    int div_wide = 1;         // MRAB_DIV_WIDE: 3-D pass 2 on 16 x 8 x 4 tiles (k_div3w) instead of 8^3
    int flux_wide = 1;        // MRAB_FLUX_WIDE: 3-D pass 1 on 16 x 8 x 4 tiles (k_flux3w) instead of 8^3
    int flux_sym = 1;         // MRAB_FLUX_SYM: Cartesian 3-D meshes store 12 symmetric flux values, not 15
    int overlap3d = 0;        // MRAB_OVERLAP3D: 3-D multi-stream task-flow schedule (measured slower
                              // than the serial launch order on one GPU: the large kernels only
                              // share the memory system)
};
Options read_options();
const Options& opts();
void set_options(const Options& o);

struct Error {
    mrab_status st;
    std::string msg;
};

struct MeshPlan {
    int dim = 2;
    int n[3] = {1, 1, 1};
    int periodic[3] = {0, 0, 0};
    int face_bc[3][2] = {{0, 0}, {0, 0}, {0, 0}};
    double period[3][3] = {{0}};
    int priority = 0;
    int s = 1;                              // step multiple
    int64_t npts = 0;
    int64_t nactive = 0;
    std::vector<double> xyz;                // [dim][npts]
    std::vector<int8_t> active;             // [npts]
    std::vector<int32_t> posA[3], posB[3];  // distance to segment start / end
    std::vector<uint16_t> cls;              // [npts], 4 bits per direction
    std::vector<double> jinv;               // [npts]
    std::vector<double> M;                  // [dim][dim][npts]
    bool cartesian = false;                 // metrics are constant and diagonal
    double cart_J = 0.0;                    // J = 1/J^-1
    double cart_M[3] = {0, 0, 0};           // M[k][k]
    // receivers (ascending point index)
    std::vector<int64_t> rpoint;
    std::vector<int32_t> rdonor;
    std::vector<int32_t> rbase;             // [R][3] wrapped
    std::vector<double> rw;                 // [R][3][4]
    std::vector<int32_t> recv_slot;         // [npts], -1 = none
    // as a donor: stencil bounding box and the box grown by the D1 reach (3)
    bool is_donor = false;
    int fv_lo[3] = {0, 0, 0}, fv_hi[3] = {0, 0, 0};   // inclusive
    int st_lo[3] = {0, 0, 0}, st_hi[3] = {0, 0, 0};
    int64_t idx(int i, int j, int k) const { return (int64_t)i + (int64_t)n[0] * ((int64_t)j + (int64_t)n[1] * k); }
};

struct Plan {
    int dim = 2, nc = 4;
    double gamma = 1.4, Re = 0, Pr = 0.72, wall_T = 1.0;
    int viscous = 0;
    double q_inf[5] = {0, 0, 0, 0, 0};
    int order_n = 3, history_m = 3;
    double h = 0;
    int S = 1;                              // largest step multiple
    std::vector<MeshPlan> meshes;
    // coef[g][j][k]: weights over [0, j/s_g] (units of h_g), j = 1..s_g, k oldest first
    std::vector<std::vector<std::vector<double>>> coef;
    // donors[g][h] = 1 if mesh h has receivers whose donor is mesh g
    std::vector<std::vector<int>> donor_of;
    Options opt;                            // switches read at plan creation
};

// host setup (host_setup.cpp)
mrab_status ab_weights(const double* nodes, int m, int n, double a, double b, double* out,
                       std::string* msg);
// overset_only: stop after the overset setup (hole cutting, segments, receivers, donors)
bool build_plan(const mrab_problem* pb, Plan& plan, Error& err, bool overset_only = false);

}  // namespace mrab
