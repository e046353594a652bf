// Device-side data structures and kernel launchers of libmrab.so (sm_100a, fp64).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace mrab {

// TMA tensor maps of a mesh's state-shaped buffers (host table, built at mrab_create; 4-D
// views [5][n2][n1][n0] with the boxes k_rhs3z loads)
struct Z3Table {
    static constexpr int kMax = 16;
    int n = 0;
    const void* ptr[kMax];
    CUtensorMap box[kMax], ox[kMax], oy[kMax], ep[kMax];
};
// the maps one k_rhs3z launch uses (kernel parameter, __grid_constant__)
struct Z3Maps {
    CUtensorMap box, ox, oy, base, s0, s1;
    int ok, ep_ok;
};
// host: add the tensor maps of one state-shaped buffer of mesh m to t (false if TMA cannot
// describe it: odd n0, misaligned)
struct DevMesh;
bool z3_encode(const DevMesh& m, const void* buf, Z3Table& t);

struct DevMesh {
    int n[3];
    int periodic[3];
    int face_bc[3][2];
    int64_t npts;
    const Z3Table* z3t;        // host pointer: TMA tensor maps of the 3-D buffers (NULL = none)
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
    const int32_t* rdonor;     // [R] donor mesh of each receiver
    const int32_t* rbase;      // [R][3] donor stencil base
    const double* rw;          // [R][3][4] per-axis Lagrange weights
    // 3-D two-pass RHS: contravariant fluxes [3][5][npts] (k_flux3d -> k_rhs3d), the mesh's
    // Cartesian viscous-flux buffer, and the per-8^3-tile flag "F^V is read here" (SAT points)
    const double* fh;
    double* fv;
    const uint8_t* fvtile;
    // 2-D: tile list of the RHS kernel, every tile once, non-interior tiles first;
    // bit 31 set = interior tile (see rhs2d_interior_tile); NULL = decide in the kernel
    const int32_t* tlist;
    int ntl;
};

struct Gas {
    double gamma, Re, Pr, wall_T;
    double q_inf[5];
    int viscous;
    // host-precomputed: 1/Re, mu/(Re Pr (gamma-1)), gamma-1, 1/(gamma-1), 1/gamma
    double iRe, kT, gm1, igm1, igamma;
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
    // 2-D only: restrict the launch to a list of tiles (tile = ty * ntx + tx); NULL = all
    const int32_t* tiles;
    int ntiles;
    // launch priority recorded on the launch itself (survives graph capture); 0 = default
    int prio;
    int has_prio;
    // 2-D kernel L2 prefetch (set by the launcher): bit 0 = this tile's epilogue rows
    int pf;
    // 2-D with a tile list: at most `persist` CTAs walk the list (0 = one CTA per tile)
    int persist;
    // 2-D: interior tiles take the lean path (set by the launcher; MRAB_LEAN=0 disables)
    int lean;
    // 2-D: `tiles` are all interior: launch the lean-only kernel (k_rhs2d_lean)
    int lean_only;
    // launch timeline (mrab_set_trace; NULL = off): one record per CTA, see trace_rec
    unsigned long long* trace;
    int trace_tag;
};

// tile grid of the 2-D RHS kernel (for building tile lists on the host)
void rhs2d_tile_shape(int* tx, int* ty);
// host: true if tile (bx, by) of a 2-D mesh may take the kernel's interior fast path: the
// tile is full, its primitive halo (H = 6 viscous / 3 Euler) lies inside the mesh (or wraps
// across a periodic seam), and every flux point (tile + 3) is interior in both directions
bool rhs2d_interior_tile(const int* n, const int* periodic, const uint16_t* cls, int viscous,
                         int bx, int by, int cart);
// per-mesh tile shape (32 x 8 for small curvilinear meshes, else 32 x 16)
void rhs2d_tile_shape_for(const int* n, int cart, int* tx, int* ty);
int rhs2d_variant_for(const int* n, int cart);

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
    // 3-D box-staged gather: receivers grouped by donor box (host-built; NULL = per-receiver)
    const int32_t* gorder;    // [R] receiver indices in group order
    const int32_t* ginfo;     // [G][6]: start, count, donor mesh, box origin (3)
    int ngroups;
};
// host: group 3-D receivers whose 4^3 donor stencils lie in one 7^3 donor box (origin = base
// rounded down to a multiple of 4 per axis), at most 64 per group; returns ginfo [G][6] and
// fills order [R]
std::vector<int32_t> interp3_groups(int64_t R, const int32_t* donor, const int32_t* base,
                                    std::vector<int32_t>& order);

struct DonorSet {             // per donor mesh: where to read state / viscous flux
    const double* state[8];
    const double* fv[8];
    int n[8][3];
    int64_t npts[8];
};

// State of every mesh at one evaluation time as a linear combination
// state_h = base_h + sum_k c_hk src_hk (nsrc = 0: the base itself).  Used to form donor
// intermediate states on the fly (MRAB Steps 2/5).
struct SrcSet {
    const double* base[8];
    const double* src[8][6];
    double c[8][6];
    int nsrc[8];
};

// receivers (of up to 8 receiving meshes) whose donor data one launch gathers
struct RecvTask {
    int nmesh;
    int64_t off[9];                 // prefix sums of receiver counts
    const int32_t* rdonor[8];
    const int32_t* rbase[8];
    const double* rw[8];
    double* qhat[8];
    double* fvhat[8];
    int64_t nrecv[8];
    int set[8];                     // which SrcSet (evaluation time) each entry reads
    unsigned long long* trace;      // launch timeline (NULL = off)
    int trace_tag;
    int raw_k;                      // set by the launcher: 1 + max history terms of the sets
};

struct SrcSets {
    SrcSet s[8];
};

struct MeshTable {
    DevMesh m[8];
};

// 2-D donor kernel: for every receiver, 16 lanes (one per donor stencil point) form the donor
// state on the fly, its Cartesian viscous flux from segmented D1 gradients, and
// shuffle-reduce the Lagrange-weighted sums into qhat / fvhat.
void launch_donor2d(const RecvTask& rt, const SrcSets& ss, const MeshTable& mt, const Gas& gas,
                    cudaStream_t st);

// 3-D Cartesian viscous fluxes F^V of a donor mesh where the gathers read them: on the 8^3
// tiles of `box` (tiles == NULL) or on a list of 8^3 tiles (flat index, x fastest)
void launch_visc(const DevMesh& m, const double* Q, double* FV, const Box& box, const int32_t* tiles,
                 int ntiles, const Gas& gas, cudaStream_t st);
// 3-D: the fused one-pass RHS kernel k_rhs3z (reads the gathered qhat/fvhat at its receivers);
// 2-D: the tiled kernel that forms its own viscous fluxes and gathers donor data inline at its
// receivers from `ds`.
void launch_rhs(int dim, const DevMesh& m, const double* Q, const Gas& gas, const Epilogue& ep,
                const DonorSet& ds, cudaStream_t st);
// 3-D two-pass RHS, pass by pass (the MRAB schedules run every stepping mesh's flux pass, then
// the gathers -- which read the F^V the flux pass wrote on the donor-stencil tiles -- then the
// divergence passes)
void launch_flux3d(const DevMesh& m, const double* Q, const Gas& gas, cudaStream_t st);
void launch_div3d_pass(const DevMesh& m, const double* Q, const Gas& gas, const Epilogue& ep, cudaStream_t st);
void launch_combine_tiles(int nc, const DevMesh& m, const int32_t* tiles, int ntiles, const double* base,
                          int nsrc, const double* const* src, const double* csrc, double* out,
                          cudaStream_t st);
void launch_combine(int nc, const DevMesh& m, const Box& box, const double* base, int nsrc,
                    const double* const* src, const double* csrc, double* out, cudaStream_t st);
void launch_interp(int viscous, const RecvList& rl, const DonorSet& ds, cudaStream_t st);
void upload_stencil_rows();
// L2 scrub for cold-cache timing: write `a` (bytes) then stream-read `b` (bytes) so that the
// L2 ends up holding clean lines of an unrelated buffer (no dirty write-backs later).
void launch_l2_scrub(void* a, void* b, size_t bytes, int tag, cudaStream_t st);
// sets *flag (device int) if any of the n doubles is not finite
void launch_finite(const double* a, size_t n, int* flag, cudaStream_t st);
// multi-GPU (mesh-partitioned): which rank owns each mesh; merge of received donor data
struct OwnerTable {
    int owner[8];
};
void launch_merge_recv(int rows, int64_t R, const int32_t* rdonor, const OwnerTable& ot, int src_rank,
                       const double* src, double* dst, cudaStream_t st);
// K9: *out (device double) = min over the active points of mesh m of the eq:ts timestep
void launch_dt(int dim, const DevMesh& m, const double* Q, const Gas& gas, double* out, cudaStream_t st);
// launch priority of the 3-D launches that follow on this thread (has = 0: plain launches)
void set_launch_priority(int has, int prio);
// timeline stamp (mrab_set_trace): one record (tag, now, now) appended by a 1-thread kernel
void launch_stamp(unsigned long long* trace, int tag, cudaStream_t st);

#ifdef __CUDACC__
// 1/x in fp64 without the IEEE division sequence: MUFU reciprocal seed refined by two
// Newton steps (error ~1 ulp; the parity tolerances are 1e-10).  Measured on
// B200: IEEE double division 128 cycles dependent latency, this ~4 DFMA + MUFU.
__device__ __forceinline__ double rcp64(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    y = fma(y, fma(-x, y, 1.0), y);
    y = fma(y, fma(-x, y, 1.0), y);
    return y;
}
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// trace buffer: [0] record count, [1] capacity (records), then records of 5 u64:
// (smid << 56 | blockIdx.x << 16 | tag, CTA start ns, CTA end ns, two phase marks or 0)
__device__ __forceinline__ void trace_rec(unsigned long long* buf, int tag, unsigned long long t0,
                                          unsigned long long ta = 0, unsigned long long tb = 0) {
    const unsigned long long i = atomicAdd(buf, 1ull);
    if (i < buf[1]) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        unsigned long long* rec = buf + 2 + 5 * i;
        rec[0] = ((unsigned long long)smid << 56) | ((unsigned long long)blockIdx.x << 16) |
                 (unsigned)(tag & 0xffff);
        rec[1] = t0;
        rec[2] = gtimer();
        rec[3] = ta;
        rec[4] = tb;
    }
}
#endif

}  // namespace mrab
