// Shared device helpers of the 2-D RHS kernels (k_rhs2d, k_rhs2d_tma): SBP 2-4 stencils on
// shared-memory rows, the characteristic SAT penalty and the Cartesian viscous fluxes.
#pragma once
#include "kernels.cuh"
#include "mrab_internal.h"
#include "stencil_table.cuh"

namespace mrab {
namespace k2d {

constexpr double C1 = 2.0 / 3.0, C2 = 1.0 / 12.0;

static __device__ __forceinline__ double d_int(const double* f, int s, int st) {
    return C1 * (f[s + st] - f[s - st]) - C2 * (f[s + 2 * st] - f[s - 2 * st]);
}
static __device__ __forceinline__ double2 d_int2(const double2* f, int s, int st) {
    const double2 a = f[s + st], b = f[s - st], c = f[s + 2 * st], d = f[s - 2 * st];
    return make_double2(C1 * (a.x - b.x) - C2 * (c.x - d.x), C1 * (a.y - b.y) - C2 * (c.y - d.y));
}
static __device__ __forceinline__ double d_gen(const double* f, int s, int st, int cl) {
    double acc = 0.0;
    const int n = c_nst[cl];
    for (int t = 0; t < n; ++t) acc += c_cf[cl][t] * f[s + c_off[cl][t] * st];
    return acc;
}
static __device__ __forceinline__ double2 d_gen2(const double2* f, int s, int st, int cl) {
    double2 acc = make_double2(0.0, 0.0);
    const int n = c_nst[cl];
    for (int t = 0; t < n; ++t) {
        const double c = c_cf[cl][t];
        const double2 v = f[s + c_off[cl][t] * st];
        acc.x += c * v.x;
        acc.y += c * v.y;
    }
    return acc;
}

// characteristic SAT penalty (same algebra as kernels.cu kchar<2>)
static __device__ __forceinline__ void kchar2(const double* q, const double* n, double side,
                                       const double* dq, const Gas& g, double* out) {
    // divisions as reciprocal multiplies (rcp64: the IEEE divide costs 128 cycles of latency)
    const double rho = q[0];
    const double irho = rcp64(rho);
    const double u0 = q[1] * irho, u1 = q[2] * irho;
    const double ke = u0 * u0 + u1 * u1;
    const double p = g.gm1 * (q[3] - 0.5 * rho * ke);
    const double c2 = g.gamma * p * irho, c = sqrt(c2);
    const double ic2 = rcp64(c2);
    const double H = (q[3] + p) * irho;
    const double nn = sqrt(n[0] * n[0] + n[1] * n[1]);
    const double inn = rcp64(nn);
    const double n0 = n[0] * inn, n1 = n[1] * inn;
    const double un = u0 * n0 + u1 * n1;
    const double du0 = (dq[1] - u0 * dq[0]) * irho, du1 = (dq[2] - u1 * dq[0]) * irho;
    const double dp = g.gm1 * (dq[3] - (u0 * dq[1] + u1 * dq[2]) + 0.5 * ke * dq[0]);
    const double dun = du0 * n0 + du1 * n1;
    const double ap = (dp + rho * c * dun) * (0.5 * ic2);
    const double am = (dp - rho * c * dun) * (0.5 * ic2);
    const double a0 = dq[0] - dp * ic2;
    const double l0 = fmax(side * un * nn, 0.0);
    const double lp = fmax(side * (un + c) * nn, 0.0);
    const double lm = fmax(side * (un - c) * nn, 0.0);
    const double dt0 = du0 - dun * n0, dt1 = du1 - dun * n1;
    const double wp = lp * ap, wm = lm * am, w0 = l0 * a0;
    out[0] = wp + wm + w0;
    out[1] = wp * (u0 + c * n0) + wm * (u0 - c * n0) + w0 * u0 + l0 * rho * dt0;
    out[2] = wp * (u1 + c * n1) + wm * (u1 - c * n1) + w0 * u1 + l0 * rho * dt1;
    out[3] = wp * (H + c * un) + wm * (H - c * un) + w0 * (0.5 * ke) + l0 * rho * (u0 * dt0 + u1 * dt1);
}

// Cartesian viscous fluxes at shared point s (prim index) with class code `code`
template <bool CART, int AX>
static __device__ __forceinline__ void visc_at(const double2* __restrict__ sh_uv, const double* __restrict__ sh_T,
                                        int s, unsigned code, const DevMesh& m, int64_t p,
                                        const Gas& g, double* Fx, double* Fy,
                                        const double* met = nullptr) {
    const int cx = code & 15, cy = (code >> 4) & 15;
    double2 uvx, uvy;
    double Tx, Ty;
    if (cx == CLS_INT) {
        uvx = d_int2(sh_uv, s, 1);
        Tx = d_int(sh_T, s, 1);
    } else {
        uvx = d_gen2(sh_uv, s, 1, cx);
        Tx = d_gen(sh_T, s, 1, cx);
    }
    if (cy == CLS_INT) {
        uvy = d_int2(sh_uv, s, AX);
        Ty = d_int(sh_T, s, AX);
    } else {
        uvy = d_gen2(sh_uv, s, AX, cy);
        Ty = d_gen(sh_T, s, AX, cy);
    }
    double dudx, dudy, dvdx, dvdy, dTdx, dTdy;
    if (CART) {
        const double sx = m.cJ * m.cM[0], sy = m.cJ * m.cM[1];
        dudx = sx * uvx.x; dvdx = sx * uvx.y; dTdx = sx * Tx;
        dudy = sy * uvy.x; dvdy = sy * uvy.y; dTdy = sy * Ty;
    } else {
        const int64_t N = m.npts;
        double J, Mxx, Mxy, Myx, Myy;
        if (met) {
            J = met[0]; Mxx = met[1]; Mxy = met[2]; Myx = met[3]; Myy = met[4];
        } else {
            J = __ldg(m.J + p);
            Mxx = __ldg(m.M + p); Mxy = __ldg(m.M + N + p);
            Myx = __ldg(m.M + 2 * N + p); Myy = __ldg(m.M + 3 * N + p);
        }
        dudx = J * (Mxx * uvx.x + Myx * uvy.x); dudy = J * (Mxy * uvx.x + Myy * uvy.x);
        dvdx = J * (Mxx * uvx.y + Myx * uvy.y); dvdy = J * (Mxy * uvx.y + Myy * uvy.y);
        dTdx = J * (Mxx * Tx + Myx * Ty); dTdy = J * (Mxy * Tx + Myy * Ty);
    }
    const double div = dudx + dvdy;
    const double txx = (2.0 * dudx - (2.0 / 3.0) * div) * g.iRe;
    const double tyy = (2.0 * dvdy - (2.0 / 3.0) * div) * g.iRe;
    const double txy = (dudy + dvdx) * g.iRe;
    const double2 uv = sh_uv[s];
    Fx[0] = 0.0; Fx[1] = txx; Fx[2] = txy; Fx[3] = uv.x * txx + uv.y * txy + g.kT * dTdx;
    Fy[0] = 0.0; Fy[1] = txy; Fy[2] = tyy; Fy[3] = uv.x * txy + uv.y * tyy + g.kT * dTdy;
}

// asynchronous 8-byte global -> shared copy (LDGSTS; no register staging)
static __device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gsrc));
}
static __device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }


// SAT penalties (eq:int P:279-299; corners sum both directions) at a segment-end
// point of a 2-D tile, added to R.  qhat / fvhat come from k_donor2d.
template <bool VISC, bool CART, int AX>
static __device__ __forceinline__ void sat2d(const DevMesh& m, const double* __restrict__ Q,
                                             const Gas& g, const double2* __restrict__ sh_uv,
                                             const double* __restrict__ sh_T, int s, unsigned code,
                                             int64_t p, int gi, int gj, double Jp, double* R) {
    constexpr double kP0 = 17.0 / 48.0;
    const int64_t N = m.npts;
    const int cx = code & 15, cy = (code >> 4) & 15;
    double q[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) q[c] = __ldg(Q + c * N + p);
    double Vx[4] = {0, 0, 0, 0}, Vy[4] = {0, 0, 0, 0};
    if (VISC) visc_at<CART, AX>(sh_uv, sh_T, s, code, m, p, g, Vx, Vy);
    const int slot = m.recv_slot[p];
    double qi[4] = {0, 0, 0, 0}, fvi[6] = {0, 0, 0, 0, 0, 0};
    if (slot >= 0) {
#pragma unroll
        for (int c = 0; c < 4; ++c) qi[c] = m.qhat[c * m.nrecv + slot];
        if (VISC)
#pragma unroll
            for (int c = 0; c < 6; ++c) fvi[c] = m.fvhat[c * m.nrecv + slot];
    }
    const int idx[2] = {gi, gj};
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int cl = k == 0 ? cx : cy;
        if (cl != CLS_L0 && cl != CLS_R0) continue;
        const int sidx = (cl == CLS_L0) ? 0 : 1;
        const double side = (cl == CLS_L0) ? 1.0 : -1.0;
        const bool at_face = !m.periodic[k] && (sidx == 0 ? idx[k] == 0 : idx[k] == m.n[k] - 1);
        const int typ = at_face ? m.face_bc[k][sidx] : MRAB_BC_OVERSET;
        double nv[2];
        if (CART) {
            nv[0] = k == 0 ? m.cJ * m.cM[0] : 0.0;
            nv[1] = k == 1 ? m.cJ * m.cM[1] : 0.0;
        } else {
            nv[0] = Jp * __ldg(m.M + (2 * k) * N + p);
            nv[1] = Jp * __ldg(m.M + (2 * k + 1) * N + p);
        }
        double qh[4];
        if (typ == MRAB_BC_OVERSET) {
#pragma unroll
            for (int c = 0; c < 4; ++c) qh[c] = qi[c];
        } else if (typ == MRAB_BC_FARFIELD) {
#pragma unroll
            for (int c = 0; c < 4; ++c) qh[c] = g.q_inf[c];
        } else {
            qh[0] = q[0];
            qh[1] = 0.0;
            qh[2] = 0.0;
            qh[3] = q[0] * g.wall_T * g.igamma * g.igm1;
        }
        double dq[4], kd[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) dq[c] = q[c] - qh[c];
        kchar2(q, nv, side, dq, g, kd);
        double sig1 = 0.0;
        if (VISC) sig1 = 0.5 * (nv[0] * nv[0] + nv[1] * nv[1]) * g.iRe;
#pragma unroll
        for (int c = 0; c < 4; ++c) R[c] -= (0.5 * kd[c] + sig1 * dq[c]) * (1.0 / kP0);
        if (VISC && typ != MRAB_BC_WALL) {
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const double fk = nv[0] * Vx[1 + j] + nv[1] * Vy[1 + j];
                double fhv = 0.0;
                if (typ == MRAB_BC_OVERSET) fhv = nv[0] * fvi[j] + nv[1] * fvi[3 + j];
                R[1 + j] += 0.5 * side * (fk - fhv) * (1.0 / kP0);
            }
        }
    }
}

// visc_at for a point whose rows are interior in both directions (compile-time stencils)
template <bool CART, int AX>
static __device__ __forceinline__ void visc_at_int(const double2* __restrict__ sh_uv,
                                                   const double* __restrict__ sh_T, int s,
                                                   const DevMesh& m, int64_t p, const Gas& g,
                                                   double* Fx, double* Fy,
                                                   const double* met = nullptr) {
    const double2 uvx = d_int2(sh_uv, s, 1), uvy = d_int2(sh_uv, s, AX);
    const double Tx = d_int(sh_T, s, 1), Ty = d_int(sh_T, s, AX);
    double dudx, dudy, dvdx, dvdy, dTdx, dTdy;
    if (CART) {
        const double sx = m.cJ * m.cM[0], sy = m.cJ * m.cM[1];
        dudx = sx * uvx.x; dvdx = sx * uvx.y; dTdx = sx * Tx;
        dudy = sy * uvy.x; dvdy = sy * uvy.y; dTdy = sy * Ty;
    } else {
        const int64_t N = m.npts;
        double J, Mxx, Mxy, Myx, Myy;
        if (met) {
            J = met[0]; Mxx = met[1]; Mxy = met[2]; Myx = met[3]; Myy = met[4];
        } else {
            J = __ldg(m.J + p);
            Mxx = __ldg(m.M + p); Mxy = __ldg(m.M + N + p);
            Myx = __ldg(m.M + 2 * N + p); Myy = __ldg(m.M + 3 * N + p);
        }
        dudx = J * (Mxx * uvx.x + Myx * uvy.x); dudy = J * (Mxy * uvx.x + Myy * uvy.x);
        dvdx = J * (Mxx * uvx.y + Myx * uvy.y); dvdy = J * (Mxy * uvx.y + Myy * uvy.y);
        dTdx = J * (Mxx * Tx + Myx * Ty); dTdy = J * (Mxy * Tx + Myy * Ty);
    }
    const double div = dudx + dvdy;
    const double txx = (2.0 * dudx - (2.0 / 3.0) * div) * g.iRe;
    const double tyy = (2.0 * dvdy - (2.0 / 3.0) * div) * g.iRe;
    const double txy = (dudy + dvdx) * g.iRe;
    const double2 uv = sh_uv[s];
    Fx[0] = 0.0; Fx[1] = txx; Fx[2] = txy; Fx[3] = uv.x * txx + uv.y * txy + g.kT * dTdx;
    Fy[0] = 0.0; Fy[1] = txy; Fy[2] = tyy; Fy[3] = uv.x * txy + uv.y * tyy + g.kT * dTdy;
}

}  // namespace k2d
}  // namespace mrab
