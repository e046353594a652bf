// CUDA kernels of libmrab.so (sm_100a, fp64, CUDA cores; no tensor cores: the path is a
// stencil, not a dense contraction).  DESIGN.md §5 lists each kernel with its roofline.
// This file: the 3-D path and the shared pieces (2-D: kernels2d.cu, kernels2d_march.cu).
//
//   k_flux3d   3-D pass 1: cross-region state staged by cp.async, D1 gradients, F^V (flagged
//              tiles), contravariant fluxes of every point once (R3/R11)
//   k_rhs3d    3-D pass 2 (PRE) / single pass: R = -J sum_k D_k Fhat_k + SAT (eq:int
//              P:279-299) fused with the AB / RK combination epilogue (eq:ab_general P:358-361)
//   k_visc3d_x Cartesian viscous fluxes on donor boxes at intermediate states (one round trip)
//   k_combine  intermediate donor states base + sum beta_k R_k (MRAB Steps 2/5)
//   k_interp3q Lagrange gather of donor state and viscous flux at receivers
//   k_visc / k_rhs / k_interp  the original one-thread-per-point kernels (MRAB_3D_DIRECT=1,
//              and the 2-D viscous pass on donor boxes)
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "kernels.cuh"
#include "mrab_internal.h"
#include "stencil_table.cuh"

namespace mrab {

void upload_stencil_rows() {}

static constexpr double kP0 = 17.0 / 48.0;   // H_00 of the SBP norm (R14)

__device__ __forceinline__ int64_t nbr(const DevMesh& m, int64_t p, int i, int k, int off,
                                       int64_t stride) {
    int n = m.n[k];
    int ii = i + off;
    if (ii < 0)
        ii += n;
    else if (ii >= n)
        ii -= n;
    return p + (int64_t)(ii - i) * stride;
}

template <int D>
__device__ __forceinline__ void prim(const double* __restrict__ Q, int64_t q, int64_t N,
                                     double gamma, double& rho, double* u, double& p,
                                     double& E) {
    rho = __ldg(Q + q);
    double ir = rcp64(rho);
    double ke = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        double mi = __ldg(Q + (1 + i) * N + q);
        u[i] = mi * ir;
        ke += mi * u[i];
    }
    E = __ldg(Q + (D + 1) * N + q);
    p = (gamma - 1.0) * (E - 0.5 * ke);
}

// ------------------------------------------------------------------------------------
// viscous fluxes
// ------------------------------------------------------------------------------------
template <int D, bool CART>
__global__ void __launch_bounds__(256) k_visc(DevMesh m, const double* __restrict__ Q,
                                              double* __restrict__ FV, Box box, Gas g) {
    const int bx = box.hi[0] - box.lo[0] + 1, by = box.hi[1] - box.lo[1] + 1,
              bz = box.hi[2] - box.lo[2] + 1;
    const int64_t tot = (int64_t)bx * by * bz;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= tot) return;
    int idx[3];
    idx[0] = box.lo[0] + (int)(t % bx);
    idx[1] = box.lo[1] + (int)((t / bx) % by);
    idx[2] = box.lo[2] + (int)(t / ((int64_t)bx * by));
    const int64_t N = m.npts;
    const int64_t stride[3] = {1, m.n[0], (int64_t)m.n[0] * m.n[1]};
    const int64_t p = idx[0] + stride[1] * idx[1] + stride[2] * idx[2];
    const unsigned code = m.cls[p];
    if (!code) return;
    double dphi[D + 1][D];
#pragma unroll
    for (int k = 0; k < D; ++k) {
        const int c = (code >> (4 * k)) & 15;
        double acc[D + 1];
#pragma unroll
        for (int f = 0; f <= D; ++f) acc[f] = 0.0;
        for (int s = 0; s < c_nst[c]; ++s) {
            const int64_t q = nbr(m, p, idx[k], k, c_off[c][s], stride[k]);
            double rho, u[D], pr, E;
            prim<D>(Q, q, N, g.gamma, rho, u, pr, E);
            const double cf = c_cf[c][s];
#pragma unroll
            for (int i = 0; i < D; ++i) acc[i] += cf * u[i];
            acc[D] += cf * (g.gamma * pr / rho);
        }
#pragma unroll
        for (int f = 0; f <= D; ++f) dphi[f][k] = acc[f];
    }
    double grad[D + 1][D];   // grad[f][i] = d phi_f / d x_i
#pragma unroll
    for (int f = 0; f <= D; ++f)
#pragma unroll
        for (int i = 0; i < D; ++i) {
            if (CART) {
                grad[f][i] = m.cJ * (m.cM[i] * dphi[f][i]);
            } else {
                double s = 0.0;
#pragma unroll
                for (int k = 0; k < D; ++k) s += __ldg(m.M + (k * D + i) * N + p) * dphi[f][k];
                grad[f][i] = __ldg(m.J + p) * s;
            }
        }
    double rho, u[D], pr, E;
    prim<D>(Q, p, N, g.gamma, rho, u, pr, E);
    double div = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) div += grad[i][i];
    const double iRe = 1.0 / g.Re;
    const double kT = 1.0 / (g.Re * g.Pr * (g.gamma - 1.0));
#pragma unroll
    for (int i = 0; i < D; ++i) {
        double e = 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j) {
            double tau = (grad[i][j] + grad[j][i] - (i == j ? (2.0 / 3.0) * div : 0.0)) * iRe;
            FV[(int64_t)(i * (D + 1) + j) * N + p] = tau;
            e += u[j] * tau;
        }
        FV[(int64_t)(i * (D + 1) + D) * N + p] = e + kT * grad[D][i];
    }
}

// ------------------------------------------------------------------------------------
// SAT characteristic penalty K^s(n; q) dq (analytic Euler eigensystem; readings R14/R15)
// ------------------------------------------------------------------------------------
template <int D>
__device__ __forceinline__ void kchar(const double* q, const double* n, double side,
                                      const double* dq, double gamma, double* out) {
    // divisions as reciprocal multiplies (rcp64: the IEEE divide costs 128 cycles of latency)
    const double rho = q[0];
    const double irho = rcp64(rho);
    double u[D], ke = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        u[i] = q[1 + i] * irho;
        ke += u[i] * u[i];
    }
    const double p = (gamma - 1.0) * (q[D + 1] - 0.5 * rho * ke);
    const double c2 = gamma * p * irho;
    const double c = sqrt(c2);
    const double ic2 = rcp64(c2);
    const double H = (q[D + 1] + p) * irho;
    double nn = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) nn += n[i] * n[i];
    nn = sqrt(nn);
    const double inn = rcp64(nn);
    double nh[D], un = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        nh[i] = n[i] * inn;
        un += u[i] * nh[i];
    }
    double du[D], udm = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        du[i] = (dq[1 + i] - u[i] * dq[0]) * irho;
        udm += u[i] * dq[1 + i];
    }
    const double dp = (gamma - 1.0) * (dq[D + 1] - udm + 0.5 * ke * dq[0]);
    double dun = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) dun += du[i] * nh[i];
    const double ap = (dp + rho * c * dun) * (0.5 * ic2);
    const double am = (dp - rho * c * dun) * (0.5 * ic2);
    const double a0 = dq[0] - dp * ic2;
    const double l0 = fmax(side * un * nn, 0.0);
    const double lp = fmax(side * (un + c) * nn, 0.0);
    const double lm = fmax(side * (un - c) * nn, 0.0);
    double udt = 0.0, dut[D];
#pragma unroll
    for (int i = 0; i < D; ++i) {
        dut[i] = du[i] - dun * nh[i];
        udt += u[i] * dut[i];
    }
    const double wp = lp * ap, wm = lm * am, w0 = l0 * a0;
    out[0] = wp + wm + w0;
#pragma unroll
    for (int i = 0; i < D; ++i)
        out[1 + i] = wp * (u[i] + c * nh[i]) + wm * (u[i] - c * nh[i]) + w0 * u[i] +
                     l0 * rho * dut[i];
    out[D + 1] = wp * (H + c * un) + wm * (H - c * un) + w0 * (0.5 * ke) + l0 * rho * udt;
}

// SAT penalties at one point (eq:int P:279-299; edges/corners sum over flagged directions,
// P:292-294), added to R.  Shared by the direct and the tiled 3-D RHS kernels.
template <int D, bool VISC, bool CART>
__device__ __forceinline__ void sat_point(const DevMesh& m, const double* __restrict__ Q,
                                          const double* __restrict__ FV, const Gas& g, int64_t p,
                                          const int* idx, unsigned code, double Jp, double* R) {
    constexpr int NC = D + 2;
    const int64_t N = m.npts;
#pragma unroll
        for (int k = 0; k < D; ++k) {
            const int cl = (code >> (4 * k)) & 15;
            if (cl != CLS_L0 && cl != CLS_R0) continue;
            const int sidx = (cl == CLS_L0) ? 0 : 1;
            const double side = (cl == CLS_L0) ? 1.0 : -1.0;
            const bool at_face = !m.periodic[k] && (sidx == 0 ? idx[k] == 0 : idx[k] == m.n[k] - 1);
            const int typ = at_face ? m.face_bc[k][sidx] : MRAB_BC_OVERSET;
            double q[NC], qh[NC], dq[NC], nv[D];
#pragma unroll
            for (int c = 0; c < NC; ++c) q[c] = __ldg(Q + c * N + p);
#pragma unroll
            for (int i = 0; i < D; ++i)
                nv[i] = CART ? (i == k ? m.cJ * m.cM[k] : 0.0) : Jp * __ldg(m.M + (k * D + i) * N + p);
            int slot = -1;
            if (typ == MRAB_BC_OVERSET) {
                slot = m.recv_slot[p];
#pragma unroll
                for (int c = 0; c < NC; ++c) qh[c] = m.qhat[c * m.nrecv + slot];
            } else if (typ == MRAB_BC_FARFIELD) {
#pragma unroll
                for (int c = 0; c < NC; ++c) qh[c] = g.q_inf[c];
            } else {   // isothermal no-slip wall
                qh[0] = q[0];
#pragma unroll
                for (int i = 0; i < D; ++i) qh[1 + i] = 0.0;
                qh[D + 1] = q[0] * g.wall_T / (g.gamma * (g.gamma - 1.0));
            }
#pragma unroll
            for (int c = 0; c < NC; ++c) dq[c] = q[c] - qh[c];
            double kd[NC];
            kchar<D>(q, nv, side, dq, g.gamma, kd);
            double sig1 = 0.0;
            if (VISC) {
#pragma unroll
                for (int i = 0; i < D; ++i) sig1 += nv[i] * nv[i];
                sig1 *= 0.5 / g.Re;
            }
#pragma unroll
            for (int c = 0; c < NC; ++c) R[c] -= (0.5 * kd[c] + sig1 * dq[c]) * (1.0 / kP0);
            if (VISC && typ != MRAB_BC_WALL) {
                // F^V_kappa - Fhat^V_kappa contracted with grad(kappa)
#pragma unroll
                for (int j = 0; j <= D; ++j) {
                    double fk = 0.0, fh = 0.0;
#pragma unroll
                    for (int i = 0; i < D; ++i) {
                        fk += nv[i] * __ldg(FV + (int64_t)(i * (D + 1) + j) * N + p);
                        if (typ == MRAB_BC_OVERSET)
                            fh += nv[i] * m.fvhat[(int64_t)(i * (D + 1) + j) * m.nrecv + slot];
                    }
                    R[1 + j] += 0.5 * side * (fk - fh) * (1.0 / kP0);
                }
            }
        }
    }

// ------------------------------------------------------------------------------------
// fused RHS + SAT + combination epilogue
// ------------------------------------------------------------------------------------
template <int D, bool VISC, bool CART>
__global__ void __launch_bounds__(256) k_rhs(DevMesh m, const double* __restrict__ Q,
                                             const double* __restrict__ FV, Gas g, Epilogue ep) {
    constexpr int NC = D + 2;
    const int64_t N = m.npts;
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= N) return;
    const int64_t stride[3] = {1, m.n[0], (int64_t)m.n[0] * m.n[1]};
    int idx[3];
    idx[0] = (int)(p % m.n[0]);
    idx[1] = (int)((p / m.n[0]) % m.n[1]);
    idx[2] = (int)(p / stride[2]);
    const unsigned code = m.cls[p];
    double R[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) R[c] = 0.0;
    if (code) {
#pragma unroll
        for (int k = 0; k < D; ++k) {
            const int cl = (code >> (4 * k)) & 15;
            double acc[NC];
#pragma unroll
            for (int c = 0; c < NC; ++c) acc[c] = 0.0;
            for (int s = 0; s < c_nst[cl]; ++s) {
                const int64_t q = nbr(m, p, idx[k], k, c_off[cl][s], stride[k]);
                double rho, u[D], pr, E;
                prim<D>(Q, q, N, g.gamma, rho, u, pr, E);
                double fh[NC];
#pragma unroll
                for (int c = 0; c < NC; ++c) fh[c] = 0.0;
#pragma unroll
                for (int i = 0; i < D; ++i) {
                    double Mki;
                    if (CART) {
                        if (i != k) continue;
                        Mki = m.cM[k];
                    } else {
                        Mki = __ldg(m.M + (k * D + i) * N + q);
                    }
                    // F^I_i - F^V_i
                    double f[NC];
                    f[0] = rho * u[i];
#pragma unroll
                    for (int j = 0; j < D; ++j) f[1 + j] = rho * u[i] * u[j] + (i == j ? pr : 0.0);
                    f[D + 1] = (E + pr) * u[i];
                    if (VISC) {
#pragma unroll
                        for (int j = 0; j <= D; ++j)
                            f[1 + j] -= __ldg(FV + (int64_t)(i * (D + 1) + j) * N + q);
                    }
#pragma unroll
                    for (int c = 0; c < NC; ++c) fh[c] += Mki * f[c];
                }
                const double cf = c_cf[cl][s];
#pragma unroll
                for (int c = 0; c < NC; ++c) acc[c] += cf * fh[c];
            }
#pragma unroll
            for (int c = 0; c < NC; ++c) R[c] += acc[c];
        }
        const double Jp = CART ? m.cJ : __ldg(m.J + p);
#pragma unroll
        for (int c = 0; c < NC; ++c) R[c] = -Jp * R[c];

        sat_point<D, VISC, CART>(m, Q, FV, g, p, idx, code, Jp, R);
    }
    if (ep.r_out) {
#pragma unroll
        for (int c = 0; c < NC; ++c) ep.r_out[c * N + p] = R[c];
    }
    if (ep.y_out) {
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            double y = ep.base[c * N + p] + ep.c_new * R[c];
            for (int s = 0; s < ep.nsrc; ++s) y += ep.csrc[s] * ep.src[s][c * N + p];
            ep.y_out[c * N + p] = y;
        }
    }
}

// ------------------------------------------------------------------------------------
// 3-D tiled RHS: per direction kappa, the contravariant flux Fhat_kappa is formed once per
// point of the tile extended by the D1 reach (3) along kappa and staged in shared memory;
// every point then applies its own segment row, accumulating in shared memory.  All global
// loads of a thread's region points are issued before any is used (no dependence on the
// class codes: hole points carry finite data that no active stencil reads, and points
// outside a non-periodic mesh are clamped to a valid address), so each direction costs one
// memory round trip.  Cartesian viscous fluxes come from the k_visc pass.
// Tile 8 x 8 x 8, 256 threads.
// ------------------------------------------------------------------------------------
namespace {
constexpr int T3X = 8, T3Y = 8, T3Z = 8, NT3 = 256;
constexpr int T3N = T3X * T3Y * T3Z;                  // 512
constexpr int PPT3 = T3N / NT3;                       // 2 own points per thread
constexpr int REG3 = 14 * 8 * 8;                      // extended region (any direction)
constexpr int KR3 = (REG3 + NT3 - 1) / NT3;           // region points per thread (4)
constexpr size_t SMEM3 = sizeof(double) * 5 * (REG3 + T3N) + sizeof(uint16_t) * T3N;
}  // namespace

// 3-D tile order: CTAs walk 4 x 4 x 4 blocks of 8^3 tiles (a 1-D grid), so that tiles sharing
// halo regions run close together in time and their halo reads hit L2 (a plain x-fastest
// grid re-read most z-halo planes from DRAM).  Returns false for padding CTAs.
__device__ __forceinline__ bool tile3_blocked(const DevMesh& m, int& bx, int& by, int& bz) {
    const int tx = (m.n[0] + T3X - 1) / T3X, ty = (m.n[1] + T3Y - 1) / T3Y, tz = (m.n[2] + T3Z - 1) / T3Z;
    const int sx = (tx + 3) / 4, sy = (ty + 3) / 4;
    const int b = blockIdx.x, loc = b & 63, sup = b >> 6;
    bx = (sup % sx) * 4 + (loc & 3);
    by = ((sup / sx) % sy) * 4 + ((loc >> 2) & 3);
    bz = (sup / (sx * sy)) * 4 + (loc >> 4);
    return bx < tx && by < ty && bz < tz;
}
static inline unsigned tile3_blocks(const int* n) {
    const int tx = (n[0] + T3X - 1) / T3X, ty = (n[1] + T3Y - 1) / T3Y, tz = (n[2] + T3Z - 1) / T3Z;
    return (unsigned)(((tx + 3) / 4) * ((ty + 3) / 4) * ((tz + 3) / 4) * 64);
}

// PRE: the contravariant fluxes come precomputed from k_flux3d (two-pass mode): the region
// loads read Fhat_kappa (5 values) instead of Q and F^V (9) and no flux is formed here
template <bool VISC, bool CART, bool PRE = false>
__global__ void __launch_bounds__(NT3, 2) k_rhs3d(DevMesh m, const double* __restrict__ Q,
                                                 const double* __restrict__ FV, Gas g, Epilogue ep,
                                                 const double* __restrict__ FH = nullptr) {
    constexpr int NC = 5;
    extern __shared__ __align__(16) double fb[];        // Fhat [NC][REG3], then Racc [NC][T3N]
    double* racc = fb + NC * REG3;
    uint16_t* sc = reinterpret_cast<uint16_t*>(racc + NC * T3N);
    const int n0 = m.n[0], n1 = m.n[1], n2 = m.n[2];
    const int64_t N = m.npts;
    const int64_t s1 = n0, s2 = (int64_t)n0 * n1;
    int tbx, tby, tbz;
    if (!tile3_blocked(m, tbx, tby, tbz)) return;
    const int i0 = tbx * T3X, j0 = tby * T3Y, k0 = tbz * T3Z;
    const int tid = threadIdx.x;

    // class codes requested now, stored to shared memory only after the first region loads
    // are in flight (storing them at once serialised a memory round trip before those loads)
    unsigned clsv[PPT3];
#pragma unroll
    for (int s = 0; s < PPT3; ++s) {
        const int t = tid + s * NT3;
        const int x = t & 7, y = (t >> 3) & 7, z = t >> 6;
        const int gi = i0 + x, gj = j0 + y, gk = k0 + z;
        const bool live = gi < n0 && gj < n1 && gk < n2;
        clsv[s] = live ? m.cls[gi + s1 * gj + s2 * gk] : 0u;
#pragma unroll
        for (int c = 0; c < NC; ++c) racc[c * T3N + t] = 0.0;
    }
    // PRE: the next direction's region loads are issued before the current direction's
    // stencil, so the three passes' memory round trips overlap the arithmetic
    double lqp[2][KR3][NC];
    auto pre_load = [&](int kk, double (&dst)[KR3][NC]) {
        const int ex = kk == 0 ? 3 : 0, ey = kk == 1 ? 3 : 0, ez = kk == 2 ? 3 : 0;
        const int RX = T3X + 2 * ex, RY = T3Y + 2 * ey;
#pragma unroll
        for (int r = 0; r < KR3; ++r) {
            const int t = tid + r * NT3;
            const int x = t % RX, y = (t / RX) % RY, z = t / (RX * RY);
            int gg[3] = {i0 - ex + x, j0 - ey + y, k0 - ez + z};
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const int n = m.n[k];
                if (gg[k] < 0) gg[k] = m.periodic[k] ? gg[k] + n : 0;
                else if (gg[k] >= n) gg[k] = m.periodic[k] ? gg[k] - n : n - 1;
            }
            const int64_t q = gg[0] + s1 * gg[1] + s2 * gg[2];
#pragma unroll
            for (int c = 0; c < NC; ++c) dst[r][c] = __ldg(FH + (int64_t)(kk * NC + c) * N + q);
        }
    };
    if (PRE) pre_load(0, lqp[0]);
    // direction loop unrolled: region extents are compile-time, so the index arithmetic is
    // constant division (it was runtime integer division, a quarter of all instructions)
#pragma unroll
    for (int kap = 0; kap < 3; ++kap) {
        const int ex = kap == 0 ? 3 : 0, ey = kap == 1 ? 3 : 0, ez = kap == 2 ? 3 : 0;
        const int RX = T3X + 2 * ex, RY = T3Y + 2 * ey;
        // ---- loads of all region points of this thread (independent, in flight together)
        double lq[KR3][NC], lv[KR3][4], lm[KR3][3];
#pragma unroll
        for (int r = 0; r < KR3; ++r) {
            if (PRE) break;
            const int t = tid + r * NT3;
            const int x = t % RX, y = (t / RX) % RY, z = t / (RX * RY);
            int gg[3] = {i0 - ex + x, j0 - ey + y, k0 - ez + z};
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const int n = m.n[k];
                if (gg[k] < 0) gg[k] = m.periodic[k] ? gg[k] + n : 0;
                else if (gg[k] >= n) gg[k] = m.periodic[k] ? gg[k] - n : n - 1;
            }
            const int64_t q = gg[0] + s1 * gg[1] + s2 * gg[2];
#pragma unroll
            for (int c = 0; c < NC; ++c) lq[r][c] = __ldg(Q + c * N + q);
            if (VISC) {
                if (CART) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) lv[r][j] = __ldg(FV + (int64_t)(kap * 4 + j) * N + q);
                }
            }
            if (!CART) {
#pragma unroll
                for (int i = 0; i < 3; ++i) lm[r][i] = __ldg(m.M + (kap * 3 + i) * N + q);
            }
            (void)lv;
            (void)lm;
            if (!CART && VISC) {
                // curvilinear: F^V of every Cartesian direction is needed; fetch into lv on use
            }
            // stash the clamped index for the curvilinear viscous path
            lv[r][0] = CART ? lv[r][0] : __longlong_as_double((long long)q);
        }
        // ---- contravariant fluxes -> shared memory
#pragma unroll
        for (int r = 0; r < KR3; ++r) {
            const int t = tid + r * NT3;
            if (t >= (T3X + 2 * ex) * (T3Y + 2 * ey) * (T3Z + 2 * ez)) break;
            if (PRE) {
#pragma unroll
                for (int c = 0; c < NC; ++c) fb[c * REG3 + t] = lqp[kap & 1][r][c];
                continue;
            }
            const double rho = lq[r][0];
            const double ir = rcp64(rho);
            const double u[3] = {lq[r][1] * ir, lq[r][2] * ir, lq[r][3] * ir};
            const double E = lq[r][4];
            const double pr = g.gm1 * (E - 0.5 * (lq[r][1] * u[0] + lq[r][2] * u[1] + lq[r][3] * u[2]));
            double fh[NC] = {0, 0, 0, 0, 0};
            if (CART) {
                const int i = kap;
                double f[NC];
                f[0] = lq[r][1 + i];
#pragma unroll
                for (int j = 0; j < 3; ++j) f[1 + j] = lq[r][1 + i] * u[j] + (i == j ? pr : 0.0);
                f[4] = (E + pr) * u[i];
                if (VISC) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) f[1 + j] -= lv[r][j];
                }
#pragma unroll
                for (int c = 0; c < NC; ++c) fh[c] = m.cM[kap] * f[c];
            } else {
                const int64_t q = (int64_t)__double_as_longlong(lv[r][0]);
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    double f[NC];
                    f[0] = lq[r][1 + i];
#pragma unroll
                    for (int j = 0; j < 3; ++j) f[1 + j] = lq[r][1 + i] * u[j] + (i == j ? pr : 0.0);
                    f[4] = (E + pr) * u[i];
                    if (VISC) {
#pragma unroll
                        for (int j = 0; j < 4; ++j) f[1 + j] -= __ldg(FV + (int64_t)(i * 4 + j) * N + q);
                    }
#pragma unroll
                    for (int c = 0; c < NC; ++c) fh[c] += lm[r][i] * f[c];
                }
            }
#pragma unroll
            for (int c = 0; c < NC; ++c) fb[c * REG3 + t] = fh[c];
        }
        if (kap == 0)
#pragma unroll
            for (int s = 0; s < PPT3; ++s) sc[tid + s * NT3] = (uint16_t)clsv[s];
        __syncthreads();
        if (PRE && kap < 2) pre_load(kap + 1, lqp[(kap + 1) & 1]);
        // ---- D_kappa of the staged fluxes at the tile points
        const int sk = kap == 0 ? 1 : (kap == 1 ? RX : RX * RY);
        for (int t = tid; t < T3N; t += NT3) {
            const unsigned code = sc[t];
            if (!code) continue;
            const int x = t & 7, y = (t >> 3) & 7, z = t >> 6;
            const int rr = (x + ex) + RX * ((y + ey) + RY * (z + ez));
            const int cl = (code >> (4 * kap)) & 15;
            if (cl == CLS_INT) {
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    const double* f = fb + c * REG3;
                    racc[c * T3N + t] += (2.0 / 3.0) * (f[rr + sk] - f[rr - sk]) - (1.0 / 12.0) * (f[rr + 2 * sk] - f[rr - 2 * sk]);
                }
            } else {
                const int ns = c_nst[cl];
                double acc[NC] = {0, 0, 0, 0, 0};
                for (int tt = 0; tt < ns; ++tt) {
                    const double cf = c_cf[cl][tt];
                    const int o = rr + c_off[cl][tt] * sk;
#pragma unroll
                    for (int c = 0; c < NC; ++c) acc[c] += cf * fb[c * REG3 + o];
                }
#pragma unroll
                for (int c = 0; c < NC; ++c) racc[c * T3N + t] += acc[c];
            }
        }
        __syncthreads();
    }
    // ---- SAT and epilogue
#pragma unroll
    for (int s = 0; s < PPT3; ++s) {
        const int t = tid + s * NT3;
        const int x = t & 7, y = (t >> 3) & 7, z = t >> 6;
        const int gi = i0 + x, gj = j0 + y, gk = k0 + z;
        if (gi >= n0 || gj >= n1 || gk >= n2) continue;
        const int64_t p = gi + s1 * gj + s2 * gk;
        const unsigned code = sc[t];
        double yb[NC];
        if (ep.y_out && ep.nsrc == 2) {
            // AB3 steps: base + two history terms, all loads issued together
            double v[3][NC];
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                v[0][c] = __ldg(ep.base + c * N + p);
                v[1][c] = __ldg(ep.src[0] + c * N + p);
                v[2][c] = __ldg(ep.src[1] + c * N + p);
            }
#pragma unroll
            for (int c = 0; c < NC; ++c) yb[c] = v[0][c] + ep.csrc[0] * v[1][c] + ep.csrc[1] * v[2][c];
        } else if (ep.y_out) {
            // all history loads issued together (unused slots re-read `base` with weight 0)
            const double* sp[4];
            double cw[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                sp[k] = k < ep.nsrc ? ep.src[k] : ep.base;
                cw[k] = k < ep.nsrc ? ep.csrc[k] : 0.0;
            }
            double v[5][NC];
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                v[0][c] = __ldg(ep.base + c * N + p);
#pragma unroll
                for (int k = 0; k < 4; ++k) v[1 + k][c] = __ldg(sp[k] + c * N + p);
            }
#pragma unroll
            for (int c = 0; c < NC; ++c)
                yb[c] = v[0][c] + cw[0] * v[1][c] + cw[1] * v[2][c] + cw[2] * v[3][c] + cw[3] * v[4][c];
            for (int k = 4; k < ep.nsrc; ++k)
#pragma unroll
                for (int c = 0; c < NC; ++c) yb[c] += ep.csrc[k] * __ldg(ep.src[k] + c * N + p);
        }
        double Rs[NC] = {0, 0, 0, 0, 0};
        if (code) {
            const double Jp = CART ? m.cJ : __ldg(m.J + p);
#pragma unroll
            for (int c = 0; c < NC; ++c) Rs[c] = -Jp * racc[c * T3N + t];
            bool sat = false;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const int cl = (code >> (4 * k)) & 15;
                sat = sat || cl == CLS_L0 || cl == CLS_R0;
            }
            if (sat) {
                const int idx[3] = {gi, gj, gk};
                sat_point<3, VISC, CART>(m, Q, FV, g, p, idx, code, Jp, Rs);
            }
        }
        if (ep.r_out) {
#pragma unroll
            for (int c = 0; c < NC; ++c) ep.r_out[c * N + p] = Rs[c];
        }
        if (ep.y_out) {
#pragma unroll
            for (int c = 0; c < NC; ++c) ep.y_out[c * N + p] = yb[c] + ep.c_new * Rs[c];
        }
    }
}

// ------------------------------------------------------------------------------------
// 3-D tiled viscous fluxes over a box: per direction kappa the primitives (u, v, w, T) of
// the tile extended by 3 along kappa are staged in shared memory (decoupled loads), each
// tile point takes its segment row of D1; then Cartesian gradients, stress, heat flux and
// F^V_i (12 values, layout [i][j]) are written.  Tile 8 x 8 x 8, 256 threads.
// ------------------------------------------------------------------------------------
template <bool CART>
__global__ void __launch_bounds__(NT3, 2) k_visc3d(DevMesh m, const double* __restrict__ Q,
                                                  double* __restrict__ FV, Box box, Gas g) {
    __shared__ double pv[4][REG3];
    __shared__ uint16_t sc[T3N];
    const int n0 = m.n[0], n1 = m.n[1], n2 = m.n[2];
    const int64_t N = m.npts;
    const int64_t s1 = n0, s2 = (int64_t)n0 * n1;
    const int i0 = box.lo[0] + blockIdx.x * T3X, j0 = box.lo[1] + blockIdx.y * T3Y,
              k0 = box.lo[2] + blockIdx.z * T3Z;
    const int tid = threadIdx.x;
    // class codes: stored to shared memory after the first region loads are issued
    unsigned clsv[PPT3];
#pragma unroll
    for (int s = 0; s < PPT3; ++s) {
        const int t = tid + s * NT3;
        const int gi = i0 + (t & 7), gj = j0 + ((t >> 3) & 7), gk = k0 + (t >> 6);
        const bool live = gi <= box.hi[0] && gj <= box.hi[1] && gk <= box.hi[2];
        clsv[s] = live ? m.cls[gi + s1 * gj + s2 * gk] : 0u;
    }
    double d[PPT3][3][4];   // d[s][kappa][u,v,w,T]
#pragma unroll
    for (int kap = 0; kap < 3; ++kap) {
        const int ex = kap == 0 ? 3 : 0, ey = kap == 1 ? 3 : 0, ez = kap == 2 ? 3 : 0;
        const int RX = T3X + 2 * ex, RY = T3Y + 2 * ey;
        double lq[KR3][5];
#pragma unroll
        for (int r = 0; r < KR3; ++r) {
            const int t = tid + r * NT3;
            const int x = t % RX, y = (t / RX) % RY, z = t / (RX * RY);
            int gg[3] = {i0 - ex + x, j0 - ey + y, k0 - ez + z};
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const int n = m.n[k];
                if (gg[k] < 0) gg[k] = m.periodic[k] ? gg[k] + n : 0;
                else if (gg[k] >= n) gg[k] = m.periodic[k] ? gg[k] - n : n - 1;
            }
            const int64_t q = gg[0] + s1 * gg[1] + s2 * gg[2];
#pragma unroll
            for (int c = 0; c < 5; ++c) lq[r][c] = __ldg(Q + c * N + q);
        }
        if (kap > 0) __syncthreads();   // previous direction's stencils are done with pv
#pragma unroll
        for (int r = 0; r < KR3; ++r) {
            const int t = tid + r * NT3;
            if (t >= REG3) break;
            const double ir = rcp64(lq[r][0]);
            const double u = lq[r][1] * ir, v = lq[r][2] * ir, w = lq[r][3] * ir;
            pv[0][t] = u;
            pv[1][t] = v;
            pv[2][t] = w;
            pv[3][t] = g.gamma * g.gm1 * (lq[r][4] - 0.5 * (lq[r][1] * u + lq[r][2] * v + lq[r][3] * w)) * ir;
        }
        if (kap == 0)
#pragma unroll
            for (int s = 0; s < PPT3; ++s) sc[tid + s * NT3] = (uint16_t)clsv[s];
        __syncthreads();
        const int sk = kap == 0 ? 1 : (kap == 1 ? RX : RX * RY);
#pragma unroll
        for (int s = 0; s < PPT3; ++s) {
            const int t = tid + s * NT3;
            const unsigned code = sc[t];
#pragma unroll
            for (int f = 0; f < 4; ++f) d[s][kap][f] = 0.0;
            if (!code) continue;
            const int x = t & 7, y = (t >> 3) & 7, z = t >> 6;
            const int rr = (x + ex) + RX * ((y + ey) + RY * (z + ez));
            const int cl = (code >> (4 * kap)) & 15;
            if (cl == CLS_INT) {
#pragma unroll
                for (int f = 0; f < 4; ++f) {
                    const double* a = pv[f];
                    d[s][kap][f] = (2.0 / 3.0) * (a[rr + sk] - a[rr - sk]) - (1.0 / 12.0) * (a[rr + 2 * sk] - a[rr - 2 * sk]);
                }
            } else {
                const int ns = c_nst[cl];
                for (int tt = 0; tt < ns; ++tt) {
                    const double cf = c_cf[cl][tt];
                    const int o = rr + c_off[cl][tt] * sk;
#pragma unroll
                    for (int f = 0; f < 4; ++f) d[s][kap][f] += cf * pv[f][o];
                }
            }
        }
    }
    // center primitives (the z-extended region holds the tile points at z + 3)
#pragma unroll
    for (int s = 0; s < PPT3; ++s) {
        const int t = tid + s * NT3;
        const unsigned code = sc[t];
        if (!code) continue;
        const int x = t & 7, y = (t >> 3) & 7, z = t >> 6;
        const int rr = x + T3X * (y + T3Y * (z + 3));
        const double u[3] = {pv[0][rr], pv[1][rr], pv[2][rr]};
        const int64_t p = (i0 + x) + s1 * (j0 + y) + s2 * (k0 + z);
        double gr[4][3];   // gr[f][i] = d phi_f / d x_i
#pragma unroll
        for (int f = 0; f < 4; ++f)
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                if (CART) {
                    gr[f][i] = m.cJ * (m.cM[i] * d[s][i][f]);
                } else {
                    double acc = 0.0;
#pragma unroll
                    for (int k = 0; k < 3; ++k) acc += __ldg(m.M + (k * 3 + i) * N + p) * d[s][k][f];
                    gr[f][i] = __ldg(m.J + p) * acc;
                }
            }
        const double div = gr[0][0] + gr[1][1] + gr[2][2];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            double e = 0.0;
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const double tau = (gr[i][j] + gr[j][i] - (i == j ? (2.0 / 3.0) * div : 0.0)) * g.iRe;
                FV[(int64_t)(i * 4 + j) * N + p] = tau;
                e += u[j] * tau;
            }
            FV[(int64_t)(i * 4 + 3) * N + p] = e + g.kT * gr[3][i];
        }
    }
}

// ------------------------------------------------------------------------------------
// 3-D viscous fluxes, one memory round trip per tile: the state of the whole cross-shaped
// region the three D1 passes read (tile 8^3 plus 3 layers on each of its six faces: 1664
// points) is copied to shared memory by cp.async at once, turned into primitives in place,
// and every gradient is taken from there (k_visc3d loaded one direction-extended region per
// pass: three dependent round trips).  Same arithmetic as k_visc3d.
// Cross-region index of tile-relative (x, y, z): the tile itself x + 8 y + 64 z, then the six
// 3-deep face slabs (x-, x+, y-, y+, z-, z+) of 192 points each.
// ------------------------------------------------------------------------------------
constexpr int XREG = 512 + 6 * 192;   // 1664
__device__ __forceinline__ int xreg_idx(int x, int y, int z) {
    // x slabs: the 3-deep direction fastest; y and z slabs: x fastest (contiguous 8-point rows)
    if (x < 0) return 512 + (x + 3) + 3 * (y + 8 * z);
    if (x >= 8) return 512 + 192 + (x - 8) + 3 * (y + 8 * z);
    if (y < 0) return 512 + 2 * 192 + x + 8 * ((y + 3) + 3 * z);
    if (y >= 8) return 512 + 3 * 192 + x + 8 * ((y - 8) + 3 * z);
    if (z < 0) return 512 + 4 * 192 + x + 8 * y + 64 * (z + 3);
    if (z >= 8) return 512 + 5 * 192 + x + 8 * y + 64 * (z - 8);
    return x + 8 * y + 64 * z;
}
__device__ __forceinline__ void xreg_xyz(int t, int& x, int& y, int& z) {
    if (t < 512) {
        x = t & 7; y = (t >> 3) & 7; z = t >> 6;
        return;
    }
    const int k = t - 512, side = k / 192, w = k - side * 192;
    if (side < 2) {
        const int a = w % 3, b = (w / 3) & 7, c = w / 24;
        x = side == 0 ? a - 3 : 8 + a;
        y = b;
        z = c;
    } else if (side < 4) {
        const int a = (w >> 3) % 3, c = (w >> 3) / 3;
        x = w & 7;
        y = side == 2 ? a - 3 : 8 + a;
        z = c;
    } else {
        const int a = w >> 6;
        x = w & 7;
        y = (w >> 3) & 7;
        z = side == 4 ? a - 3 : 8 + a;
    }
}
constexpr size_t SMEMX = sizeof(double) * 5 * XREG;

// stage the state of the cross-shaped region of the tile at (i0, j0, k0) into xr[5][XREG] by
// cp.async: x-runs of the tile and of the y / z slabs two points at a time (16 bytes) when the
// mesh rows are 16-byte aligned, the x slabs (3-point runs) and ragged ends point-wise.  Points
// outside a non-periodic mesh are clamped to a valid address (no active stencil reads them).
// full = false: the tile only (Euler: no gradients).
__device__ __forceinline__ void stage_xregion(double* xr, const DevMesh& m, const double* __restrict__ Q,
                                              int i0, int j0, int k0, bool full) {
    const int n0 = m.n[0], n1 = m.n[1], n2 = m.n[2];
    const int64_t N = m.npts, s1 = n0, s2 = (int64_t)n0 * n1;
    const int per0 = m.periodic[0], per1 = m.periodic[1], per2 = m.periodic[2];
    const bool al = (n0 & 1) == 0 && (i0 & 1) == 0;
    const int npair = full ? (512 + 768) / 2 : 256;
    for (int u = threadIdx.x; u < npair + (full ? 384 : 0); u += NT3) {
        int t, w;
        if (u < npair) {
            t = 2 * u;
            if (t >= 512) t += 384;           // skip the x slabs
            w = 2;
        } else {
            t = 512 + (u - npair);            // x slabs, one point
            w = 1;
        }
        int x, y, z;
        xreg_xyz(t, x, y, z);
        int gj = j0 + y, gk = k0 + z;
        if (gj < 0) gj = per1 ? gj + n1 : 0; else if (gj >= n1) gj = per1 ? gj - n1 : n1 - 1;
        if (gk < 0) gk = per2 ? gk + n2 : 0; else if (gk >= n2) gk = per2 ? gk - n2 : n2 - 1;
        const bool pair16 = w == 2 && al && i0 + x + 1 < n0;
        for (int e = 0; e < w; ++e) {
            if (pair16 && e == 1) break;
            int gi = i0 + x + e;
            if (gi < 0) gi = per0 ? gi + n0 : 0; else if (gi >= n0) gi = per0 ? gi - n0 : n0 - 1;
            const int64_t q = gi + s1 * gj + s2 * gk;
#pragma unroll
            for (int c = 0; c < 5; ++c) {
                const unsigned sa = (unsigned)__cvta_generic_to_shared(xr + c * XREG + t + e);
                if (pair16)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(Q + c * N + q));
                else
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(Q + c * N + q));
            }
        }
    }
}

template <bool CART>
__global__ void __launch_bounds__(NT3, 2) k_visc3d_x(DevMesh m, const double* __restrict__ Q,
                                                    double* __restrict__ FV, Box box, Gas g) {
    extern __shared__ __align__(16) double xr[];   // [5][XREG]: state, then (rho, u, v, w, T)
    __shared__ uint16_t sc[T3N];
    const int n0 = m.n[0], n1 = m.n[1], n2 = m.n[2];
    const int64_t N = m.npts;
    const int64_t s1 = n0, s2 = (int64_t)n0 * n1;
    const int i0 = box.lo[0] + blockIdx.x * T3X, j0 = box.lo[1] + blockIdx.y * T3Y,
              k0 = box.lo[2] + blockIdx.z * T3Z;
    const int tid = threadIdx.x;
    const int per0 = m.periodic[0], per1 = m.periodic[1], per2 = m.periodic[2];
    // ---- one round trip: the whole cross region (points outside a non-periodic mesh are
    // clamped to a valid address; no active stencil reads them)
    stage_xregion(xr, m, Q, i0, j0, k0, true);
    unsigned clsv[PPT3];
#pragma unroll
    for (int s = 0; s < PPT3; ++s) {
        const int t = tid + s * NT3;
        const int gi = i0 + (t & 7), gj = j0 + ((t >> 3) & 7), gk = k0 + (t >> 6);
        const bool live = gi <= box.hi[0] && gj <= box.hi[1] && gk <= box.hi[2];
        clsv[s] = live ? m.cls[gi + s1 * gj + s2 * gk] : 0u;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    // ---- primitives in place
    for (int t = tid; t < XREG; t += NT3) {
        const double r = xr[t], mu = xr[XREG + t], mv = xr[2 * XREG + t], mw = xr[3 * XREG + t];
        const double E = xr[4 * XREG + t];
        const double ir = rcp64(r);
        const double u = mu * ir, v = mv * ir, w = mw * ir;
        xr[XREG + t] = u;
        xr[2 * XREG + t] = v;
        xr[3 * XREG + t] = w;
        xr[4 * XREG + t] = g.gamma * g.gm1 * (E - 0.5 * (mu * u + mv * v + mw * w)) * ir;
    }
#pragma unroll
    for (int s = 0; s < PPT3; ++s) sc[tid + s * NT3] = (uint16_t)clsv[s];
    __syncthreads();
    const double* pf = xr + XREG;   // [4][XREG]: u, v, w, T
#pragma unroll
    for (int s = 0; s < PPT3; ++s) {
        const int t = tid + s * NT3;
        const unsigned code = sc[t];
        if (!code) continue;
        const int x = t & 7, y = (t >> 3) & 7, z = t >> 6;
        double d[3][4];   // d[kappa][u, v, w, T]
#pragma unroll
        for (int kap = 0; kap < 3; ++kap) {
            const int cl = (code >> (4 * kap)) & 15;
            auto at = [&](int o) {
                return kap == 0 ? xreg_idx(x + o, y, z) : (kap == 1 ? xreg_idx(x, y + o, z) : xreg_idx(x, y, z + o));
            };
            if (cl == CLS_INT) {
                const int a1 = at(1), b1 = at(-1), a2 = at(2), b2 = at(-2);
#pragma unroll
                for (int f = 0; f < 4; ++f) {
                    const double* a = pf + f * XREG;
                    d[kap][f] = (2.0 / 3.0) * (a[a1] - a[b1]) - (1.0 / 12.0) * (a[a2] - a[b2]);
                }
            } else {
#pragma unroll
                for (int f = 0; f < 4; ++f) d[kap][f] = 0.0;
                const int ns = c_nst[cl];
                for (int tt = 0; tt < ns; ++tt) {
                    const double cf = c_cf[cl][tt];
                    const int o = at(c_off[cl][tt]);
#pragma unroll
                    for (int f = 0; f < 4; ++f) d[kap][f] += cf * pf[f * XREG + o];
                }
            }
        }
        const double u[3] = {pf[t], pf[XREG + t], pf[2 * XREG + t]};
        const int64_t p = (i0 + x) + s1 * (j0 + y) + s2 * (k0 + z);
        double gr[4][3];   // gr[f][i] = d phi_f / d x_i
#pragma unroll
        for (int f = 0; f < 4; ++f)
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                if (CART) {
                    gr[f][i] = m.cJ * (m.cM[i] * d[i][f]);
                } else {
                    double acc = 0.0;
#pragma unroll
                    for (int k = 0; k < 3; ++k) acc += __ldg(m.M + (k * 3 + i) * N + p) * d[k][f];
                    gr[f][i] = __ldg(m.J + p) * acc;
                }
            }
        const double div = gr[0][0] + gr[1][1] + gr[2][2];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            double e = 0.0;
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const double tau = (gr[i][j] + gr[j][i] - (i == j ? (2.0 / 3.0) * div : 0.0)) * g.iRe;
                FV[(int64_t)(i * 4 + j) * N + p] = tau;
                e += u[j] * tau;
            }
            FV[(int64_t)(i * 4 + 3) * N + p] = e + g.kT * gr[3][i];
        }
    }
}

// ------------------------------------------------------------------------------------
// 3-D RHS in two passes (default; MRAB_3D_SPLIT=0 restores k_visc3d_x + k_rhs3d):
//   k_flux3d  per tile: the cross-shaped state region staged by cp.async in one round trip
//             (as k_visc3d_x), primitives in place, D1 gradients at the tile points, then the
//             full contravariant fluxes Fhat_kappa = sum_i M_kappa,i (F^I_i - F^V_i) of every
//             point written once ([3][5][N]); the Cartesian viscous fluxes F^V are written only
//             in tiles that hold SAT points or donor stencils (the SAT term and the gathers
//             read them there);
//   k_rhs3d<PRE = true>  the tiled RHS reading Fhat_kappa (5 values per region point instead
//             of Q and F^V) in its three register-staged passes, D_kappa by class code, SAT,
//             AB / RK epilogue (k_div3d, staging all three regions by cp.async in one round
//             trip, measured slower: MRAB_DIV3D_STAGED=1).
// k_rhs3d formed every flux on the tile extended by 3 along each direction from Q and F^V
// (three dependent round trips, 1.75x redundant flux work).
// ------------------------------------------------------------------------------------
template <bool VISC, bool CART>
__global__ void __launch_bounds__(NT3, 2) k_flux3d(DevMesh m, const double* __restrict__ Q,
                                                  double* __restrict__ FH, double* __restrict__ FV,
                                                  const uint8_t* __restrict__ fvtile, Gas g) {
    extern __shared__ __align__(16) double xr[];   // [5][XREG]: state, then (rho, u, v, w, T)
    __shared__ uint16_t sc[T3N];
    const int n0 = m.n[0], n1 = m.n[1], n2 = m.n[2];
    const int64_t N = m.npts;
    const int64_t s1 = n0, s2 = (int64_t)n0 * n1;
    int tbx, tby, tbz;
    if (!tile3_blocked(m, tbx, tby, tbz)) return;
    const int i0 = tbx * T3X, j0 = tby * T3Y, k0 = tbz * T3Z;
    const int tid = threadIdx.x;
    const int per0 = m.periodic[0], per1 = m.periodic[1], per2 = m.periodic[2];
    const int ntx = (n0 + T3X - 1) / T3X, nty = (n1 + T3Y - 1) / T3Y;
    const bool wfv = VISC && fvtile[tbx + ntx * (tby + nty * tbz)];
    const int nreg = VISC ? XREG : T3N;   // Euler: no gradients, the tile itself suffices
    stage_xregion(xr, m, Q, i0, j0, k0, VISC);
    unsigned clsv[PPT3];
#pragma unroll
    for (int s = 0; s < PPT3; ++s) {
        const int t = tid + s * NT3;
        const int gi = i0 + (t & 7), gj = j0 + ((t >> 3) & 7), gk = k0 + (t >> 6);
        const bool live = gi < n0 && gj < n1 && gk < n2;
        clsv[s] = live ? m.cls[gi + s1 * gj + s2 * gk] : 0u;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    for (int t = tid; t < nreg; t += NT3) {
        const double r = xr[t], mu = xr[XREG + t], mv = xr[2 * XREG + t], mw = xr[3 * XREG + t];
        const double E = xr[4 * XREG + t];
        const double ir = rcp64(r);
        const double u = mu * ir, v = mv * ir, w = mw * ir;
        xr[XREG + t] = u;
        xr[2 * XREG + t] = v;
        xr[3 * XREG + t] = w;
        xr[4 * XREG + t] = g.gamma * g.gm1 * (E - 0.5 * (mu * u + mv * v + mw * w)) * ir;
    }
#pragma unroll
    for (int s = 0; s < PPT3; ++s) sc[tid + s * NT3] = (uint16_t)clsv[s];
    __syncthreads();
    const double* pf = xr + XREG;   // [4][XREG]: u, v, w, T
#pragma unroll
    for (int s = 0; s < PPT3; ++s) {
        const int t = tid + s * NT3;
        const int x = t & 7, y = (t >> 3) & 7, z = t >> 6;
        if (i0 + x >= n0 || j0 + y >= n1 || k0 + z >= n2) continue;
        const int64_t p = (i0 + x) + s1 * (j0 + y) + s2 * (k0 + z);
        const unsigned code = sc[t];
        if (!code) {
#pragma unroll
            for (int c = 0; c < 15; ++c) FH[(int64_t)c * N + p] = 0.0;
            continue;
        }
        const double r = xr[t];
        const double u[3] = {pf[t], pf[XREG + t], pf[2 * XREG + t]};
        const double T = pf[3 * XREG + t];
        const double pr = r * T * g.igamma;
        const double E = pr * g.igm1 + 0.5 * r * (u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
        double fv[3][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}, {0, 0, 0, 0}};
        double Jp = 0.0, Mp[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
        if (!CART) {
            Jp = __ldg(m.J + p);
#pragma unroll
            for (int k = 0; k < 3; ++k)
#pragma unroll
                for (int i = 0; i < 3; ++i) Mp[k][i] = __ldg(m.M + (k * 3 + i) * N + p);
        }
        if (VISC) {
            double d[3][4];   // d[kappa][u, v, w, T]
#pragma unroll
            for (int kap = 0; kap < 3; ++kap) {
                const int cl = (code >> (4 * kap)) & 15;
                auto at = [&](int o) {
                    return kap == 0 ? xreg_idx(x + o, y, z) : (kap == 1 ? xreg_idx(x, y + o, z) : xreg_idx(x, y, z + o));
                };
                if (cl == CLS_INT) {
                    const int a1 = at(1), b1 = at(-1), a2 = at(2), b2 = at(-2);
#pragma unroll
                    for (int f = 0; f < 4; ++f) {
                        const double* a = pf + f * XREG;
                        d[kap][f] = (2.0 / 3.0) * (a[a1] - a[b1]) - (1.0 / 12.0) * (a[a2] - a[b2]);
                    }
                } else {
#pragma unroll
                    for (int f = 0; f < 4; ++f) d[kap][f] = 0.0;
                    const int ns = c_nst[cl];
                    for (int tt = 0; tt < ns; ++tt) {
                        const double cf = c_cf[cl][tt];
                        const int o = at(c_off[cl][tt]);
#pragma unroll
                        for (int f = 0; f < 4; ++f) d[kap][f] += cf * pf[f * XREG + o];
                    }
                }
            }
            double gr[4][3];
#pragma unroll
            for (int f = 0; f < 4; ++f)
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    if (CART) {
                        gr[f][i] = m.cJ * (m.cM[i] * d[i][f]);
                    } else {
                        double acc = 0.0;
#pragma unroll
                        for (int k = 0; k < 3; ++k) acc += Mp[k][i] * d[k][f];
                        gr[f][i] = Jp * acc;
                    }
                }
            const double div = gr[0][0] + gr[1][1] + gr[2][2];
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                double e = 0.0;
#pragma unroll
                for (int j = 0; j < 3; ++j) {
                    const double tau = (gr[i][j] + gr[j][i] - (i == j ? (2.0 / 3.0) * div : 0.0)) * g.iRe;
                    fv[i][j] = tau;
                    e += u[j] * tau;
                }
                fv[i][3] = e + g.kT * gr[3][i];
            }
            if (wfv)
#pragma unroll
                for (int i = 0; i < 3; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) FV[(int64_t)(i * 4 + j) * N + p] = fv[i][j];
        }
        // Cartesian fluxes F_i = F^I_i - F^V_i, then Fhat_kappa
        double F[3][5];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const double mi = r * u[i];
            F[i][0] = mi;
#pragma unroll
            for (int j = 0; j < 3; ++j) F[i][1 + j] = mi * u[j] + (i == j ? pr : 0.0) - fv[i][j];
            F[i][4] = (E + pr) * u[i] - fv[i][3];
        }
#pragma unroll
        for (int kap = 0; kap < 3; ++kap)
#pragma unroll
            for (int c = 0; c < 5; ++c) {
                double fh;
                if (CART) fh = m.cM[kap] * F[kap][c];
                else fh = Mp[kap][0] * F[0][c] + Mp[kap][1] * F[1][c] + Mp[kap][2] * F[2][c];
                FH[(int64_t)(kap * 5 + c) * N + p] = fh;
            }
    }
}

constexpr int REGD = 14 * 8 * 8;                    // one kappa-extended region
constexpr size_t SMEMD = sizeof(double) * 3 * 5 * REGD;

template <bool VISC, bool CART>
__global__ void __launch_bounds__(NT3, 2) k_div3d(DevMesh m, const double* __restrict__ Q,
                                                 const double* __restrict__ FH,
                                                 const double* __restrict__ FV, Gas g, Epilogue ep) {
    constexpr int NC = 5;
    extern __shared__ __align__(16) double fb[];     // [kappa][c][REGD]
    __shared__ uint16_t sc[T3N];
    const int n0 = m.n[0], n1 = m.n[1], n2 = m.n[2];
    const int64_t N = m.npts;
    const int64_t s1 = n0, s2 = (int64_t)n0 * n1;
    const int i0 = blockIdx.x * T3X, j0 = blockIdx.y * T3Y, k0 = blockIdx.z * T3Z;
    const int tid = threadIdx.x;
    const int per0 = m.periodic[0], per1 = m.periodic[1], per2 = m.periodic[2];
    // ---- the three extended regions of Fhat_kappa in one round trip
    // y- and z-extended regions: x-runs of 8 doubles, 16-byte copies when rows are 16-byte
    // aligned (even n0; tiles start at multiples of 8)
    const bool pair = (n0 & 1) == 0 && i0 + 8 <= n0;
#pragma unroll
    for (int kap = 1; kap < 3; ++kap) {
        if (!pair) break;
        const int ey = kap == 1 ? 3 : 0, ez = kap == 2 ? 3 : 0;
        const int RY = T3Y + 2 * ey;
        for (int t = tid; t < REGD / 2; t += NT3) {
            const int x2 = t & 3, y = (t >> 2) % RY, z = (t >> 2) / RY;
            int gj = j0 - ey + y, gk = k0 - ez + z;
            if (gj < 0) gj = per1 ? gj + n1 : 0; else if (gj >= n1) gj = per1 ? gj - n1 : n1 - 1;
            if (gk < 0) gk = per2 ? gk + n2 : 0; else if (gk >= n2) gk = per2 ? gk - n2 : n2 - 1;
            const int64_t q = i0 + 2 * x2 + s1 * gj + s2 * gk;
            const int e = 2 * x2 + T3X * (y + RY * z);
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const unsigned sa = (unsigned)__cvta_generic_to_shared(fb + (kap * NC + c) * REGD + e);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(FH + (int64_t)(kap * NC + c) * N + q));
            }
        }
    }
#pragma unroll
    for (int kap = 0; kap < 3; ++kap) {
        if (kap > 0 && pair) break;
        const int ex = kap == 0 ? 3 : 0, ey = kap == 1 ? 3 : 0, ez = kap == 2 ? 3 : 0;
        const int RX = T3X + 2 * ex, RY = T3Y + 2 * ey;
        for (int t = tid; t < REGD; t += NT3) {
            const int x = t % RX, y = (t / RX) % RY, z = t / (RX * RY);
            int gi = i0 - ex + x, gj = j0 - ey + y, gk = k0 - ez + z;
            if (gi < 0) gi = per0 ? gi + n0 : 0; else if (gi >= n0) gi = per0 ? gi - n0 : n0 - 1;
            if (gj < 0) gj = per1 ? gj + n1 : 0; else if (gj >= n1) gj = per1 ? gj - n1 : n1 - 1;
            if (gk < 0) gk = per2 ? gk + n2 : 0; else if (gk >= n2) gk = per2 ? gk - n2 : n2 - 1;
            const int64_t q = gi + s1 * gj + s2 * gk;
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const unsigned sa = (unsigned)__cvta_generic_to_shared(fb + (kap * NC + c) * REGD + t);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(FH + (int64_t)(kap * NC + c) * N + q));
            }
        }
    }
    unsigned clsv[PPT3];
#pragma unroll
    for (int s = 0; s < PPT3; ++s) {
        const int t = tid + s * NT3;
        const int gi = i0 + (t & 7), gj = j0 + ((t >> 3) & 7), gk = k0 + (t >> 6);
        const bool live = gi < n0 && gj < n1 && gk < n2;
        clsv[s] = live ? m.cls[gi + s1 * gj + s2 * gk] : 0u;
    }
    // epilogue inputs requested while the regions land
    double yb[PPT3][NC];
#pragma unroll
    for (int s = 0; s < PPT3; ++s)
#pragma unroll
        for (int c = 0; c < NC; ++c) yb[s][c] = 0.0;
    if (ep.y_out) {
#pragma unroll
        for (int s = 0; s < PPT3; ++s) {
            const int t = tid + s * NT3;
            const int gi = min(i0 + (t & 7), n0 - 1), gj = min(j0 + ((t >> 3) & 7), n1 - 1), gk = min(k0 + (t >> 6), n2 - 1);
            const int64_t p = gi + s1 * gj + s2 * gk;
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                double y = __ldg(ep.base + c * N + p);
                for (int k = 0; k < ep.nsrc; ++k) y += ep.csrc[k] * __ldg(ep.src[k] + c * N + p);
                yb[s][c] = y;
            }
        }
    }
#pragma unroll
    for (int s = 0; s < PPT3; ++s) sc[tid + s * NT3] = (uint16_t)clsv[s];
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
#pragma unroll
    for (int s = 0; s < PPT3; ++s) {
        const int t = tid + s * NT3;
        const int x = t & 7, y = (t >> 3) & 7, z = t >> 6;
        const int gi = i0 + x, gj = j0 + y, gk = k0 + z;
        if (gi >= n0 || gj >= n1 || gk >= n2) continue;
        const int64_t p = gi + s1 * gj + s2 * gk;
        const unsigned code = sc[t];
        double Rs[NC] = {0, 0, 0, 0, 0};
        if (code) {
            double acc[NC] = {0, 0, 0, 0, 0};
#pragma unroll
            for (int kap = 0; kap < 3; ++kap) {
                const int ex = kap == 0 ? 3 : 0, ey = kap == 1 ? 3 : 0, ez = kap == 2 ? 3 : 0;
                const int RX = T3X + 2 * ex, RY = T3Y + 2 * ey;
                const int rr = (x + ex) + RX * ((y + ey) + RY * (z + ez));
                const int sk = kap == 0 ? 1 : (kap == 1 ? RX : RX * RY);
                const double* f = fb + kap * NC * REGD;
                const int cl = (code >> (4 * kap)) & 15;
                if (cl == CLS_INT) {
#pragma unroll
                    for (int c = 0; c < NC; ++c) {
                        const double* fc = f + c * REGD;
                        acc[c] += (2.0 / 3.0) * (fc[rr + sk] - fc[rr - sk]) - (1.0 / 12.0) * (fc[rr + 2 * sk] - fc[rr - 2 * sk]);
                    }
                } else {
                    const int ns = c_nst[cl];
                    double a2[NC] = {0, 0, 0, 0, 0};
                    for (int tt = 0; tt < ns; ++tt) {
                        const double cf = c_cf[cl][tt];
                        const int o = rr + c_off[cl][tt] * sk;
#pragma unroll
                        for (int c = 0; c < NC; ++c) a2[c] += cf * f[c * REGD + o];
                    }
#pragma unroll
                    for (int c = 0; c < NC; ++c) acc[c] += a2[c];
                }
            }
            const double Jp = CART ? m.cJ : __ldg(m.J + p);
#pragma unroll
            for (int c = 0; c < NC; ++c) Rs[c] = -Jp * acc[c];
            bool sat = false;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const int cl = (code >> (4 * k)) & 15;
                sat = sat || cl == CLS_L0 || cl == CLS_R0;
            }
            if (sat) {
                const int idx[3] = {gi, gj, gk};
                sat_point<3, VISC, CART>(m, Q, FV, g, p, idx, code, Jp, Rs);
            }
        }
        if (ep.r_out) {
#pragma unroll
            for (int c = 0; c < NC; ++c) ep.r_out[c * N + p] = Rs[c];
        }
        if (ep.y_out) {
#pragma unroll
            for (int c = 0; c < NC; ++c) ep.y_out[c * N + p] = yb[s][c] + ep.c_new * Rs[c];
        }
    }
}

// ------------------------------------------------------------------------------------
// intermediate states on a box: out = base + sum_k c_k src_k (all components)
// ------------------------------------------------------------------------------------
struct CombineArgs {
    const double* base;
    const double* src[8];
    double c[8];
    int nsrc;
};

__global__ void __launch_bounds__(256) k_combine(int nc, int64_t N, int n0, int n1, Box box,
                                                 CombineArgs a, double* __restrict__ out) {
    const int bx = box.hi[0] - box.lo[0] + 1, by = box.hi[1] - box.lo[1] + 1,
              bz = box.hi[2] - box.lo[2] + 1;
    const int64_t tot = (int64_t)bx * by * bz;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= tot) return;
    const int i = box.lo[0] + (int)(t % bx);
    const int j = box.lo[1] + (int)((t / bx) % by);
    const int k = box.lo[2] + (int)(t / ((int64_t)bx * by));
    const int64_t p = i + (int64_t)n0 * (j + (int64_t)n1 * k);
    for (int c = 0; c < nc; ++c) {
        double y = a.base[c * N + p];
        for (int s = 0; s < a.nsrc; ++s) y += a.c[s] * a.src[s][c * N + p];
        out[c * N + p] = y;
    }
}

// ------------------------------------------------------------------------------------
// donor gather (Lagrange interpolation, tensor product of per-axis weights)
// ------------------------------------------------------------------------------------
template <int D, bool VISC>
__global__ void __launch_bounds__(128) k_interp(RecvList rl, DonorSet ds) {
    constexpr int NC = D + 2;
    constexpr int NF = D * (D + 1);
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rl.n) return;
    const int dm = rl.donor[r];
    const int b0 = rl.base[r * 3 + 0], b1 = rl.base[r * 3 + 1], b2 = rl.base[r * 3 + 2];
    const int n0 = ds.n[dm][0], n1 = ds.n[dm][1], n2 = ds.n[dm][2];
    const int64_t N = ds.npts[dm];
    const double* __restrict__ S = ds.state[dm];
    const double* __restrict__ F = ds.fv[dm];
    const double* w = rl.w + r * 12;
    double qa[NC], fa[VISC ? NF : 1];
#pragma unroll
    for (int c = 0; c < NC; ++c) qa[c] = 0.0;
    if (VISC)
#pragma unroll
        for (int c = 0; c < NF; ++c) fa[c] = 0.0;
    const int nz = (D == 3) ? 4 : 1;
    for (int a2 = 0; a2 < nz; ++a2) {
        int kk = b2 + a2;
        if (kk >= n2) kk -= n2;
        const double w2 = (D == 3) ? w[8 + a2] : 1.0;
        for (int a1 = 0; a1 < 4; ++a1) {
            int jj = b1 + a1;
            if (jj >= n1) jj -= n1;
            const double w12 = w2 * w[4 + a1];
            for (int a0 = 0; a0 < 4; ++a0) {
                int ii = b0 + a0;
                if (ii >= n0) ii -= n0;
                const double W = w12 * w[a0];
                const int64_t q = ii + (int64_t)n0 * (jj + (int64_t)n1 * kk);
#pragma unroll
                for (int c = 0; c < NC; ++c) qa[c] += W * __ldg(S + c * N + q);
                if (VISC)
#pragma unroll
                    for (int c = 0; c < NF; ++c) fa[c] += W * __ldg(F + c * N + q);
            }
        }
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) rl.qhat[c * rl.n + r] = qa[c];
    if (VISC)
#pragma unroll
        for (int c = 0; c < NF; ++c) rl.fvhat[c * rl.n + r] = fa[c];
}

// 3-D gather, four lanes per receiver: lane a0 takes the stencil column i = b0 + a0, so the
// four lanes of a receiver read 32 contiguous bytes per (j, k) row (one sector instead of four
// scattered ones); the column sums are reduced over the quad with two shuffles per value.
template <bool VISC>
__global__ void __launch_bounds__(128) k_interp3q(RecvList rl, DonorSet ds) {
    constexpr int NC = 5, NF = 12;
    const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 2;
    const int a0 = threadIdx.x & 3;
    const bool live = r < rl.n;
    double qa[NC], fa[VISC ? NF : 1];
#pragma unroll
    for (int c = 0; c < NC; ++c) qa[c] = 0.0;
    if (VISC)
#pragma unroll
        for (int c = 0; c < NF; ++c) fa[c] = 0.0;
    if (live) {
        const int dm = rl.donor[r];
        const int b0 = rl.base[r * 3 + 0], b1 = rl.base[r * 3 + 1], b2 = rl.base[r * 3 + 2];
        const int n0 = ds.n[dm][0], n1 = ds.n[dm][1], n2 = ds.n[dm][2];
        const int64_t N = ds.npts[dm];
        const double* __restrict__ S = ds.state[dm];
        const double* __restrict__ F = ds.fv[dm];
        const double* w = rl.w + r * 12;
        int ii = b0 + a0;
        if (ii >= n0) ii -= n0;
        const double w0 = w[a0];
#pragma unroll 4
        for (int a = 0; a < 16; ++a) {
            const int a1 = a & 3, a2 = a >> 2;
            int jj = b1 + a1, kk = b2 + a2;
            if (jj >= n1) jj -= n1;
            if (kk >= n2) kk -= n2;
            const double W = w0 * w[4 + a1] * w[8 + a2];
            const int64_t q = ii + (int64_t)n0 * (jj + (int64_t)n1 * kk);
#pragma unroll
            for (int c = 0; c < NC; ++c) qa[c] += W * __ldg(S + c * N + q);
            if (VISC)
#pragma unroll
                for (int c = 0; c < NF; ++c) fa[c] += W * __ldg(F + c * N + q);
        }
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        qa[c] += __shfl_xor_sync(0xffffffffu, qa[c], 1);
        qa[c] += __shfl_xor_sync(0xffffffffu, qa[c], 2);
    }
    if (VISC)
#pragma unroll
        for (int c = 0; c < NF; ++c) {
            fa[c] += __shfl_xor_sync(0xffffffffu, fa[c], 1);
            fa[c] += __shfl_xor_sync(0xffffffffu, fa[c], 2);
        }
    if (live && a0 == 0) {
#pragma unroll
        for (int c = 0; c < NC; ++c) rl.qhat[c * rl.n + r] = qa[c];
        if (VISC)
#pragma unroll
            for (int c = 0; c < NF; ++c) rl.fvhat[c * rl.n + r] = fa[c];
    }
}

// 3-D gather staged per donor box: one CTA per receiver group (host-built: receivers whose 4^3
// donor stencils lie in one 7^3 box of the donor mesh).  The box's state and Cartesian viscous
// fluxes (343 points x 17 values) are copied to shared memory once by cp.async; every receiver
// of the group then interpolates from there with four lanes (one per stencil column) and a quad
// shuffle reduction.  Neighbouring receivers share most of their stencils, so the donor data
// crosses L2 once per box instead of once per receiver (k_interp3q).
constexpr int IBOX = 7, IBOXN = IBOX * IBOX * IBOX;
template <bool VISC>
__global__ void __launch_bounds__(128) k_interp3b(RecvList rl, DonorSet ds) {
    constexpr int NC = 5, NF = 12, NV = NC + (VISC ? NF : 0);
    extern __shared__ __align__(16) double bx[];   // [NV][IBOXN]
    const int* gi6 = rl.ginfo + 6 * blockIdx.x;
    const int start = gi6[0], count = gi6[1], dm = gi6[2];
    const int ox = gi6[3], oy = gi6[4], oz = gi6[5];
    const int n0 = ds.n[dm][0], n1 = ds.n[dm][1], n2 = ds.n[dm][2];
    const int64_t N = ds.npts[dm];
    const double* __restrict__ S = ds.state[dm];
    const double* __restrict__ F = ds.fv[dm];
    for (int t = threadIdx.x; t < IBOXN; t += blockDim.x) {
        const int x = t % IBOX, y = (t / IBOX) % IBOX, z = t / (IBOX * IBOX);
        int i = ox + x, j = oy + y, k = oz + z;
        // the box may cross a periodic seam (bases are wrapped) or run past a face: wrap, clamp
        if (i >= n0) i -= n0;
        if (j >= n1) j -= n1;
        if (k >= n2) k -= n2;
        i = min(i, n0 - 1);
        j = min(j, n1 - 1);
        k = min(k, n2 - 1);
        const int64_t q = i + (int64_t)n0 * (j + (int64_t)n1 * k);
#pragma unroll
        for (int c = 0; c < NV; ++c) {
            const double* src = c < NC ? S + c * N + q : F + (int64_t)(c - NC) * N + q;
            const unsigned sa = (unsigned)__cvta_generic_to_shared(bx + c * IBOXN + t);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(src));
        }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    const int a0 = threadIdx.x & 3;
    for (int rr = threadIdx.x >> 2; rr < ((count + 31) / 32) * 32; rr += blockDim.x >> 2) {
        const bool live = rr < count;
        double acc[NV];
#pragma unroll
        for (int c = 0; c < NV; ++c) acc[c] = 0.0;
        int r = 0;
        if (live) {
            r = rl.gorder[start + rr];
            int lx = rl.base[3 * r] - ox, ly = rl.base[3 * r + 1] - oy, lz = rl.base[3 * r + 2] - oz;
            if (lx < 0) lx += n0;
            if (ly < 0) ly += n1;
            if (lz < 0) lz += n2;
            const double* w = rl.w + r * 12;
            const double w0 = w[a0];
#pragma unroll 4
            for (int a = 0; a < 16; ++a) {
                const int a1 = a & 3, a2 = a >> 2;
                const double W = w0 * w[4 + a1] * w[8 + a2];
                const int e = (lx + a0) + IBOX * ((ly + a1) + IBOX * (lz + a2));
#pragma unroll
                for (int c = 0; c < NV; ++c) acc[c] += W * bx[c * IBOXN + e];
            }
        }
#pragma unroll
        for (int c = 0; c < NV; ++c) {
            acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], 1);
            acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], 2);
        }
        if (live && a0 == 0) {
#pragma unroll
            for (int c = 0; c < NC; ++c) rl.qhat[c * rl.n + r] = acc[c];
            if (VISC)
#pragma unroll
                for (int c = 0; c < NF; ++c) rl.fvhat[c * rl.n + r] = acc[NC + c];
        }
    }
}

std::vector<int32_t> interp3_groups(int64_t R, const int32_t* donor, const int32_t* base,
                                    std::vector<int32_t>& order) {
    struct Key {
        int d, x, y, z;
        int64_t r;
    };
    std::vector<Key> keys((size_t)R);
    for (int64_t r = 0; r < R; ++r)
        keys[r] = {donor[r], base[3 * r] / 4, base[3 * r + 1] / 4, base[3 * r + 2] / 4, r};
    std::stable_sort(keys.begin(), keys.end(), [](const Key& a, const Key& b) {
        if (a.d != b.d) return a.d < b.d;
        if (a.z != b.z) return a.z < b.z;
        if (a.y != b.y) return a.y < b.y;
        return a.x < b.x;
    });
    order.resize((size_t)R);
    std::vector<int32_t> info;
    int64_t i = 0;
    while (i < R) {
        int64_t j = i;
        while (j < R && j - i < 64 && keys[j].d == keys[i].d && keys[j].x == keys[i].x &&
               keys[j].y == keys[i].y && keys[j].z == keys[i].z)
            ++j;
        info.insert(info.end(), {(int32_t)i, (int32_t)(j - i), keys[i].d, 4 * keys[i].x, 4 * keys[i].y,
                                 4 * keys[i].z});
        for (int64_t k = i; k < j; ++k) order[k] = (int32_t)keys[k].r;
        i = j;
    }
    return info;
}

// ------------------------------------------------------------------------------------
// launchers
// ------------------------------------------------------------------------------------
static inline unsigned blocks_for(int64_t n, int bs) { return (unsigned)((n + bs - 1) / bs); }

void launch_visc(int dim, const DevMesh& m, const double* Q, double* FV, const Box& box,
                 const Gas& gas, cudaStream_t st) {
    int64_t tot = (int64_t)(box.hi[0] - box.lo[0] + 1) * (box.hi[1] - box.lo[1] + 1) *
                  (box.hi[2] - box.lo[2] + 1);
    if (tot <= 0) return;
    unsigned nb = blocks_for(tot, 256);
    static int direct = -1;
    if (direct < 0) {
        const char* e = getenv("MRAB_3D_DIRECT");
        direct = e && e[0] == '1';
    }
    if (dim == 3 && !direct) {
        dim3 grid((box.hi[0] - box.lo[0] + T3X) / T3X, (box.hi[1] - box.lo[1] + T3Y) / T3Y,
                  (box.hi[2] - box.lo[2] + T3Z) / T3Z);
        static int xr = -1;
        if (xr < 0) {
            const char* e = getenv("MRAB_VISC3D_X");
            xr = e ? atoi(e) : 1;
            cudaFuncSetAttribute(k_visc3d_x<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEMX);
            cudaFuncSetAttribute(k_visc3d_x<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEMX);
        }
        if (xr) {
            if (m.cart) k_visc3d_x<true><<<grid, NT3, SMEMX, st>>>(m, Q, FV, box, gas);
            else k_visc3d_x<false><<<grid, NT3, SMEMX, st>>>(m, Q, FV, box, gas);
        } else {
            if (m.cart) k_visc3d<true><<<grid, NT3, 0, st>>>(m, Q, FV, box, gas);
            else k_visc3d<false><<<grid, NT3, 0, st>>>(m, Q, FV, box, gas);
        }
        return;
    }
    if (dim == 2) {
        if (m.cart) k_visc<2, true><<<nb, 256, 0, st>>>(m, Q, FV, box, gas);
        else k_visc<2, false><<<nb, 256, 0, st>>>(m, Q, FV, box, gas);
    } else {
        if (m.cart) k_visc<3, true><<<nb, 256, 0, st>>>(m, Q, FV, box, gas);
        else k_visc<3, false><<<nb, 256, 0, st>>>(m, Q, FV, box, gas);
    }
}

void launch_rhs2d(const DevMesh& m, const double* Q, const Gas& g, const Epilogue& ep,
                  const DonorSet& ds, cudaStream_t st);

bool rhs3d_split() {
    static int v = -1;
    if (v < 0) {
        // default (MRAB_3D_SPLIT=0: k_visc3d_x + k_rhs3d): config 4 8.43 -> 8.08 ms/step,
        // config 5 20.2 -> 16.8 ms/step
        const char* e = getenv("MRAB_3D_SPLIT");
        const char* d = getenv("MRAB_3D_DIRECT");
        v = (e && e[0] == '0') || (d && d[0] == '1') ? 0 : 1;
    }
    return v == 1;
}

void launch_flux3d(const DevMesh& m, const double* Q, double* FH, double* FV, const Gas& gas,
                   cudaStream_t st) {
    static bool init = false;
    if (!init) {
        cudaFuncSetAttribute(k_flux3d<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEMX);
        cudaFuncSetAttribute(k_flux3d<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEMX);
        cudaFuncSetAttribute(k_flux3d<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEMX);
        cudaFuncSetAttribute(k_flux3d<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEMX);
        init = true;
    }
    const dim3 grid(tile3_blocks(m.n));
    if (gas.viscous) {
        if (m.cart) k_flux3d<true, true><<<grid, NT3, SMEMX, st>>>(m, Q, FH, FV, m.fvtile, gas);
        else k_flux3d<true, false><<<grid, NT3, SMEMX, st>>>(m, Q, FH, FV, m.fvtile, gas);
    } else {
        if (m.cart) k_flux3d<false, true><<<grid, NT3, SMEMX, st>>>(m, Q, FH, FV, m.fvtile, gas);
        else k_flux3d<false, false><<<grid, NT3, SMEMX, st>>>(m, Q, FH, FV, m.fvtile, gas);
    }
}

void launch_rhs(int dim, const DevMesh& m, const double* Q, const double* FV, const Gas& gas,
                const Epilogue& ep, const DonorSet& ds, cudaStream_t st) {
    if (dim == 2) {
        launch_rhs2d(m, Q, gas, ep, ds, st);
        return;
    }
    if (m.fh && rhs3d_split()) {
        static bool init = false;
        if (!init) {
            cudaFuncSetAttribute(k_div3d<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEMD);
            cudaFuncSetAttribute(k_div3d<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEMD);
            cudaFuncSetAttribute(k_div3d<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEMD);
            cudaFuncSetAttribute(k_div3d<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEMD);
            init = true;
        }
        dim3 grid((m.n[0] + T3X - 1) / T3X, (m.n[1] + T3Y - 1) / T3Y, (m.n[2] + T3Z - 1) / T3Z);
        static const int staged = [] {
            const char* e = getenv("MRAB_DIV3D_STAGED");
            return e ? atoi(e) : 0;
        }();
        if (staged) {
            if (gas.viscous) {
                if (m.cart) k_div3d<true, true><<<grid, NT3, SMEMD, st>>>(m, Q, m.fh, FV, gas, ep);
                else k_div3d<true, false><<<grid, NT3, SMEMD, st>>>(m, Q, m.fh, FV, gas, ep);
            } else {
                if (m.cart) k_div3d<false, true><<<grid, NT3, SMEMD, st>>>(m, Q, m.fh, FV, gas, ep);
                else k_div3d<false, false><<<grid, NT3, SMEMD, st>>>(m, Q, m.fh, FV, gas, ep);
            }
            return;
        }
        // the tiled RHS reading the precomputed fluxes (three register-staged passes)
        const dim3 grid1(tile3_blocks(m.n));
        static bool init3 = false;
        if (!init3) {
            cudaFuncSetAttribute(k_rhs3d<true, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM3);
            cudaFuncSetAttribute(k_rhs3d<true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM3);
            cudaFuncSetAttribute(k_rhs3d<false, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM3);
            cudaFuncSetAttribute(k_rhs3d<false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM3);
            init3 = true;
        }
        if (gas.viscous) {
            if (m.cart) k_rhs3d<true, true, true><<<grid1, NT3, SMEM3, st>>>(m, Q, FV, gas, ep, m.fh);
            else k_rhs3d<true, false, true><<<grid1, NT3, SMEM3, st>>>(m, Q, FV, gas, ep, m.fh);
        } else {
            if (m.cart) k_rhs3d<false, true, true><<<grid1, NT3, SMEM3, st>>>(m, Q, FV, gas, ep, m.fh);
            else k_rhs3d<false, false, true><<<grid1, NT3, SMEM3, st>>>(m, Q, FV, gas, ep, m.fh);
        }
        return;
    }
    static int direct = -1;
    if (direct < 0) {
        const char* e = getenv("MRAB_3D_DIRECT");
        direct = e && e[0] == '1';
    }
    if (!direct) {
        const size_t bytes = SMEM3;
        static bool init[4] = {false, false, false, false};
        const dim3 grid(tile3_blocks(m.n));
#define MRAB_RHS3(V, C, I)                                                                          \
    do {                                                                                            \
        if (!init[I]) {                                                                             \
            cudaFuncSetAttribute(k_rhs3d<V, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes); \
            init[I] = true;                                                                         \
        }                                                                                           \
        k_rhs3d<V, C><<<grid, NT3, bytes, st>>>(m, Q, FV, gas, ep);                                 \
    } while (0)
        if (gas.viscous) {
            if (m.cart) MRAB_RHS3(true, true, 0); else MRAB_RHS3(true, false, 1);
        } else {
            if (m.cart) MRAB_RHS3(false, true, 2); else MRAB_RHS3(false, false, 3);
        }
#undef MRAB_RHS3
        return;
    }
    unsigned nb = blocks_for(m.npts, 256);
#define MRAB_RHS(D, V, C) k_rhs<D, V, C><<<nb, 256, 0, st>>>(m, Q, FV, gas, ep)
    if (dim == 2) {
        if (gas.viscous) {
            if (m.cart) MRAB_RHS(2, true, true); else MRAB_RHS(2, true, false);
        } else {
            if (m.cart) MRAB_RHS(2, false, true); else MRAB_RHS(2, false, false);
        }
    } else {
        if (gas.viscous) {
            if (m.cart) MRAB_RHS(3, true, true); else MRAB_RHS(3, true, false);
        } else {
            if (m.cart) MRAB_RHS(3, false, true); else MRAB_RHS(3, false, false);
        }
    }
#undef MRAB_RHS
}

void launch_combine(int nc, const DevMesh& m, const Box& box, const double* base, int nsrc,
                    const double* const* src, const double* csrc, double* out, cudaStream_t st) {
    CombineArgs a{};
    a.base = base;
    a.nsrc = nsrc;
    for (int s = 0; s < nsrc; ++s) {
        a.src[s] = src[s];
        a.c[s] = csrc[s];
    }
    int64_t tot = (int64_t)(box.hi[0] - box.lo[0] + 1) * (box.hi[1] - box.lo[1] + 1) *
                  (box.hi[2] - box.lo[2] + 1);
    if (tot <= 0) return;
    k_combine<<<blocks_for(tot, 256), 256, 0, st>>>(nc, m.npts, m.n[0], m.n[1], box, a, out);
}

// "rhs blowup" check: any non-finite value in n doubles sets *flag
__global__ void k_finite(const double* __restrict__ a, size_t n, int* flag) {
    int bad = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        bad |= !isfinite(a[i]);
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

void launch_finite(const double* a, size_t n, int* flag, cudaStream_t st) {
    k_finite<<<148 * 4, 256, 0, st>>>(a, n, flag);
}

__global__ void k_scrub_read(const double4* __restrict__ b, size_t n, double* sink) {
    double acc = 0.0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        double4 v = b[i];
        acc += v.x + v.y + v.z + v.w;
    }
    if (acc == 12345.678) *sink = acc;   // keeps the loads alive, never true for scrub data
}

void launch_l2_scrub(void* a, void* b, size_t bytes, int tag, cudaStream_t st) {
    cudaMemsetAsync(a, tag & 0xff, bytes, st);
    k_scrub_read<<<148 * 8, 256, 0, st>>>((const double4*)b, bytes / sizeof(double4), (double*)a);
}

void launch_interp(int dim, int viscous, const RecvList& rl, const DonorSet& ds, cudaStream_t st) {
    if (rl.n <= 0) return;
    unsigned nb = blocks_for(rl.n, 128);
    if (dim == 2) {
        if (viscous) k_interp<2, true><<<nb, 128, 0, st>>>(rl, ds);
        else k_interp<2, false><<<nb, 128, 0, st>>>(rl, ds);
    } else {
        static int quad = -1;
        if (quad < 0) {
            const char* e = getenv("MRAB_INTERP_QUAD");
            quad = e ? atoi(e) : 1;
        }
        if (rl.ginfo && rl.ngroups > 0) {
            const size_t bytes = sizeof(double) * (viscous ? 17 : 5) * IBOXN;
            static bool init = false;
            if (!init) {
                cudaFuncSetAttribute(k_interp3b<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(sizeof(double) * 17 * IBOXN));
                cudaFuncSetAttribute(k_interp3b<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(sizeof(double) * 17 * IBOXN));
                init = true;
            }
            if (viscous) k_interp3b<true><<<rl.ngroups, 128, bytes, st>>>(rl, ds);
            else k_interp3b<false><<<rl.ngroups, 128, bytes, st>>>(rl, ds);
        } else if (quad) {
            const unsigned nbq = (unsigned)((rl.n * 4 + 127) / 128);
            if (viscous) k_interp3q<true><<<nbq, 128, 0, st>>>(rl, ds);
            else k_interp3q<false><<<nbq, 128, 0, st>>>(rl, ds);
        } else {
            if (viscous) k_interp<3, true><<<nb, 128, 0, st>>>(rl, ds);
            else k_interp<3, false><<<nb, 128, 0, st>>>(rl, ds);
        }
    }
}

}  // namespace mrab
