// CUDA kernels of libmrab.so (sm_100a, fp64, CUDA cores; no tensor cores: the path is a
// stencil, not a dense contraction).  Round-1 "direct" kernels: one thread per grid point,
// neighbours read through L1/L2.  DESIGN.md §5 lists each kernel with its roofline.
//
//   k_visc     Cartesian viscous fluxes F^V_i from D1 gradients (R3/R11)
//   k_rhs      R = -J sum_k D_k Fhat_k + SAT (eq:int P:279-299) fused with the AB / RK
//              combination epilogue (eq:ab_general P:358-361)
//   k_combine  intermediate donor states base + sum beta_k R_k (MRAB Steps 2/5)
//   k_interp   Lagrange gather of donor state and viscous flux at receivers
#include <cuda_runtime.h>

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
    double ir = 1.0 / rho;
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
    const double rho = q[0];
    double u[D], ke = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        u[i] = q[1 + i] / rho;
        ke += u[i] * u[i];
    }
    const double p = (gamma - 1.0) * (q[D + 1] - 0.5 * rho * ke);
    const double c2 = gamma * p / rho;
    const double c = sqrt(c2);
    const double H = (q[D + 1] + p) / rho;
    double nn = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) nn += n[i] * n[i];
    nn = sqrt(nn);
    double nh[D], un = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        nh[i] = n[i] / nn;
        un += u[i] * nh[i];
    }
    double du[D], udm = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        du[i] = (dq[1 + i] - u[i] * dq[0]) / rho;
        udm += u[i] * dq[1 + i];
    }
    const double dp = (gamma - 1.0) * (dq[D + 1] - udm + 0.5 * ke * dq[0]);
    double dun = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) dun += du[i] * nh[i];
    const double ap = (dp + rho * c * dun) / (2.0 * c2);
    const double am = (dp - rho * c * dun) / (2.0 * c2);
    const double a0 = dq[0] - dp / c2;
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

        // ---- SAT at segment ends (eq:int; P:292-294 sum over flagged directions) ----
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
            for (int c = 0; c < NC; ++c) R[c] -= (0.5 * kd[c] + sig1 * dq[c]) / kP0;
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
                    R[1 + j] += 0.5 * side * (fk - fh) / kP0;
                }
            }
        }
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

void launch_rhs(int dim, const DevMesh& m, const double* Q, const double* FV, const Gas& gas,
                const Epilogue& ep, const DonorSet& ds, cudaStream_t st) {
    if (dim == 2) {
        launch_rhs2d(m, Q, gas, ep, ds, st);
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
        if (viscous) k_interp<3, true><<<nb, 128, 0, st>>>(rl, ds);
        else k_interp<3, false><<<nb, 128, 0, st>>>(rl, ds);
    }
}

}  // namespace mrab
