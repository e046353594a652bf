// 2-D fused SBP-SAT right-hand side, shared-memory tiled (sm_100a, fp64).
//
// One CTA = one TX x TY tile of output points.  Everything the viscous RHS needs is staged
// once per tile (kernel k_rhs2d):
//   phase A  primitives (rho, (u, v), T) of the tile + halo H = 6 (viscous) / 3 (Euler) and
//            the stencil-class codes, read once from HBM (coalesced rows, periodic wrap),
//            all loads of a thread issued before the first is consumed;
//   phase B  at tile + 3: D1 gradients of (u, v, T) (segment closures by class code,
//            P:1526-1528 D1 o D1), Cartesian gradients via the metric terms, viscous and
//            inviscid fluxes, contravariant fluxes Fhat_xi, Fhat_eta -> shared memory;
//   phase C  R = -J (D_xi Fhat_xi + D_eta Fhat_eta), SAT at segment ends
//            (eq:int P:279-299), and the AB / RK combination epilogue (eq:ab_general) whose
//            HBM inputs are requested before the divergence is formed.
// Interior points (class 1 in a direction) take a compile-time 5-point stencil, closure rows
// the constant-memory table; (u, v) and flux component pairs are packed as double2 so one
// 16-byte shared load serves two fields.
#include <cuda_runtime.h>

#include <algorithm>

#include <cstdlib>

#include "kernels.cuh"
#include "mrab_internal.h"
#include "stencil_table.cuh"
#include "rhs2d_common.cuh"

namespace mrab {

namespace {

constexpr int TX = 32, NT = 256;
constexpr int G3 = 3;
constexpr double kP0 = 17.0 / 48.0;
using namespace k2d;

template <bool VISC, int TY, bool CART = true>
struct Geo {
    static constexpr int H = VISC ? 6 : 3;
    static constexpr int AX = TX + 2 * H, AY = TY + 2 * H;
    static constexpr int FX = TX + 2 * G3, FY = TY + 2 * G3;
    static constexpr int NA = AX * AY, NF = FX * FY;
    // shared layout: uv[NA] (double2), fh[4][NF] (double2: xi (F0,F1), xi (F2,F3),
    // eta (F0,F1), eta (F2,F3)), rho[NA], T[NA], curvilinear only: met[5][NF] (J, Mxx, Mxy,
    // Myx, Myy of the flux points, staged by cp.async in phase A), cls[NA] (uint16)
    static constexpr int NMET = CART ? 0 : 5 * NF;
    static constexpr size_t bytes = 16 * (size_t)NA + 64 * (size_t)NF + 16 * (size_t)NA +
                                    8 * (size_t)NMET + 2 * (size_t)NA;
};

// Lagrange gather of the donor state and Cartesian viscous fluxes at receiver
// `slot` of mesh m: tensor product of the per-axis weights over the 4 x 4 donor stencil.
template <bool VISC>
__device__ __forceinline__ void gather2(const DevMesh& m, const DonorSet& ds, int slot,
                                        double* qh, double* fvh) {
    const int dm = m.rdonor[slot];
    const int b0 = m.rbase[3 * slot], b1 = m.rbase[3 * slot + 1];
    const double* w = m.rw + 12 * slot;
    const int n0 = ds.n[dm][0], n1 = ds.n[dm][1];
    const int64_t N = ds.npts[dm];
    const double* __restrict__ S = ds.state[dm];
    const double* __restrict__ F = ds.fv[dm];
#pragma unroll
    for (int c = 0; c < 4; ++c) qh[c] = 0.0;
    if (VISC)
#pragma unroll
        for (int c = 0; c < 6; ++c) fvh[c] = 0.0;
#pragma unroll
    for (int a1 = 0; a1 < 4; ++a1) {
        int jj = b1 + a1;
        if (jj >= n1) jj -= n1;
        const double w1 = w[4 + a1];
#pragma unroll
        for (int a0 = 0; a0 < 4; ++a0) {
            int ii = b0 + a0;
            if (ii >= n0) ii -= n0;
            const double W = w1 * w[a0];
            const int64_t q = ii + (int64_t)n0 * jj;
#pragma unroll
            for (int c = 0; c < 4; ++c) qh[c] += W * __ldg(S + c * N + q);
            if (VISC)
#pragma unroll
                for (int c = 0; c < 6; ++c) fvh[c] += W * __ldg(F + c * N + q);
        }
    }
}

// base + sum_k c_k src_k of component c at element offset up (NS history slots, all loads
// independent so they are in flight together)
__device__ __forceinline__ void prefetch_l2(const double* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// element offset of (gi, gj) on an interior tile's halo, which may cross a periodic seam
// (the host flags such tiles interior only in periodic directions)
__device__ __forceinline__ unsigned wrap_idx(int gi, int gj, int n0, int n1) {
    if (gi < 0) gi += n0; else if (gi >= n0) gi -= n0;
    if (gj < 0) gj += n1; else if (gj >= n1) gj -= n1;
    return (unsigned)gi + (unsigned)n0 * (unsigned)gj;
}

template <int NS>
__device__ __forceinline__ double epi_sum(const Epilogue& ep, unsigned uN, unsigned up, int c) {
    const unsigned o = c * uN + up;
    double v[NS + 1];
    v[0] = __ldg(ep.base + o);
#pragma unroll
    for (int k = 0; k < NS; ++k) v[1 + k] = __ldg(ep.src[k] + o);
    double y = v[0];
#pragma unroll
    for (int k = 0; k < NS; ++k) y += ep.csrc[k] * v[1 + k];
    return y;
}

}  // namespace

// one tile (bx, by); tfast = 1 interior tile, 0 general, -1 decide from the class codes
template <bool VISC, bool CART, int TY, int NTH>
__device__ __forceinline__ void rhs2d_tile(const DevMesh& m, const double* __restrict__ Q,
                                           const Gas& g, const Epilogue& ep, int bx, int by,
                                           int tfast, double* smem, unsigned long long* tph) {
    using GG = Geo<VISC, TY, CART>;
    constexpr int H = GG::H, AX = GG::AX, FX = GG::FX;
    constexpr int NA = GG::NA, NF = GG::NF;
    double2* sh_uv = reinterpret_cast<double2*>(smem);
    double2* fh = sh_uv + NA;                       // [4][NF]
    double* sh_r = reinterpret_cast<double*>(fh + 4 * NF);
    double* sh_T = sh_r + NA;
    double* sh_met = sh_T + NA;                     // [5][NF] (curvilinear)
    uint16_t* sh_c = reinterpret_cast<uint16_t*>(sh_met + GG::NMET);

    const int n0 = m.n[0], n1 = m.n[1];
    const int64_t N = m.npts;
    const int i0 = bx * TX, j0 = by * TY;
    const int tid = threadIdx.x;

    // ---- L2 prefetch of the epilogue's history rows (read last, in phase C)
    if (ep.pf) {
        const unsigned uN = (unsigned)N;
        if ((ep.pf & 1) && ep.y_out) {
            // per history array: TY rows x 2 lines x 4 components
            constexpr int NL = TY * 2 * 4;
            for (int t = tid; t < NL; t += NTH) {
                const int line = t & 1, row = (t >> 1) % TY, c = (t >> 1) / TY;
                const int gj = j0 + row, gi = i0 + 16 * line;
                if (gj >= n1 || gi >= n0) continue;
                const unsigned o = c * uN + (unsigned)gi + (unsigned)n0 * (unsigned)gj;
                prefetch_l2(ep.base + o);
#pragma unroll
                for (int k = 0; k < 3; ++k)
                    if (k < ep.nsrc) prefetch_l2(ep.src[k] + o);
            }
        }
    }

    // ---- curvilinear: metrics of the flux points -> shared memory (async, no registers)
    if (!CART) {
        const unsigned uN = (unsigned)N;
        for (int t = tid; t < NF; t += NTH) {
            const int b = t / FX, a = t - b * FX;
            int gi = i0 - G3 + a, gj = j0 - G3 + b;
            if (gi < 0 || gi >= n0) gi = m.periodic[0] ? (gi < 0 ? gi + n0 : gi - n0) : min(max(gi, 0), n0 - 1);
            if (gj < 0 || gj >= n1) gj = m.periodic[1] ? (gj < 0 ? gj + n1 : gj - n1) : min(max(gj, 0), n1 - 1);
            const unsigned q = (unsigned)gi + (unsigned)n0 * (unsigned)gj;
            cp_async8(sh_met + t, m.J + q);
#pragma unroll
            for (int c = 0; c < 4; ++c) cp_async8(sh_met + (1 + c) * NF + t, m.M + (c * uN + q));
        }
    }

    // ---- phase A: primitives of tile + halo ------------------------------------------
    constexpr int KA = (NA + NTH - 1) / NTH;
    int allint = 1;
    if (tfast == 1) {
        // interior tile: halo inside the mesh, no class codes needed by phases B / C
        const unsigned uN = (unsigned)N;
        const unsigned q0 = (unsigned)(i0 - H) + (unsigned)n0 * (unsigned)(j0 - H);
        const bool wrap = i0 - H < 0 || j0 - H < 0 || i0 + TX + H > n0 || j0 + TY + H > n1;
        double ld[KA][4];
#pragma unroll
        for (int k = 0; k < KA; ++k) {
            const int t = tid + k * NTH;
            ld[k][0] = 1.0;
            ld[k][1] = ld[k][2] = ld[k][3] = 0.0;
            if (t < NA) {
                const int bb = t / AX, a = t - bb * AX;
                const unsigned q = wrap ? wrap_idx(i0 - H + a, j0 - H + bb, n0, n1)
                                        : q0 + (unsigned)a + (unsigned)n0 * (unsigned)bb;
                ld[k][0] = __ldg(Q + q);
                ld[k][1] = __ldg(Q + (uN + q));
                ld[k][2] = __ldg(Q + (2 * uN + q));
                ld[k][3] = __ldg(Q + (3 * uN + q));
            }
        }
#pragma unroll
        for (int k = 0; k < KA; ++k) {
            const int t = tid + k * NTH;
            if (t >= NA) break;
            const double r = ld[k][0];
            const double ir = rcp64(r);
            const double u = ld[k][1] * ir;
            const double v = ld[k][2] * ir;
            const double T = g.gamma * g.gm1 * (ld[k][3] - 0.5 * (ld[k][1] * u + ld[k][2] * v)) * ir;
            sh_r[t] = r;
            sh_uv[t] = make_double2(u, v);
            sh_T[t] = T;
        }
    } else {
        double ld[KA][4];
        unsigned cd[KA];
#pragma unroll
        for (int k = 0; k < KA; ++k) {
            const int t = tid + k * NTH;
            cd[k] = 0;
            ld[k][0] = 1.0;
            ld[k][1] = ld[k][2] = ld[k][3] = 0.0;
            if (t < NA) {
                const int b = t / AX, a = t - b * AX;
                int gi = i0 - H + a, gj = j0 - H + b;
                bool ok = true;
                if (gi < 0 || gi >= n0) {
                    if (m.periodic[0]) gi = gi < 0 ? gi + n0 : gi - n0; else ok = false;
                }
                if (gj < 0 || gj >= n1) {
                    if (m.periodic[1]) gj = gj < 0 ? gj + n1 : gj - n1; else ok = false;
                }
                if (ok) {
                    // 32-bit element offsets: one IMAD.WIDE per address (nc * npts < 2^32)
                    const unsigned q = (unsigned)gi + (unsigned)n0 * (unsigned)gj;
                    const unsigned uN = (unsigned)N;
                    cd[k] = m.cls[q];
                    ld[k][0] = __ldg(Q + q);
                    ld[k][1] = __ldg(Q + (uN + q));
                    ld[k][2] = __ldg(Q + (2 * uN + q));
                    ld[k][3] = __ldg(Q + (3 * uN + q));
                }
            }
        }
#pragma unroll
        for (int k = 0; k < KA; ++k) {
            const int t = tid + k * NTH;
            if (t >= NA) break;
            // branch-free: holes carry valid (initial) states and points outside the mesh
            // rho = 1, so the primitives are finite; no active stencil reads them
            const double r = ld[k][0];
            const double ir = rcp64(r);
            const double u = ld[k][1] * ir;
            const double v = ld[k][2] * ir;
            const double T = g.gamma * g.gm1 * (ld[k][3] - 0.5 * (ld[k][1] * u + ld[k][2] * v)) * ir;
            sh_c[t] = (uint16_t)cd[k];
            sh_r[t] = r;
            sh_uv[t] = make_double2(u, v);
            sh_T[t] = T;
            // tile-uniform fast path: every flux point (tile + 3) interior in both directions
            const int b = t / AX, a = t - b * AX;
            if (b >= H - G3 && b < H + TY + G3 && a >= H - G3 && a < H + TX + G3 &&
                cd[k] != (unsigned)(CLS_INT | (CLS_INT << 4)))
                allint = 0;
        }
    }
    if (tfast == 0) allint = 0;
    if (!CART) cp_async_wait_all();
    const int fast = __syncthreads_and(allint);
    if (ep.trace && threadIdx.x == 0) tph[0] = gtimer();

    // ---- phase B: contravariant fluxes at tile + 3 -----------------------------------
    if (fast) {
        for (int t = tid; t < NF; t += NTH) {
            const int b = t / FX, a = t - b * FX;
            const int s = (b + H - G3) * AX + (a + H - G3);
            const double r = sh_r[s];
            const double2 uv = sh_uv[s];
            const double u = uv.x, v = uv.y;
            const double p = r * sh_T[s] * g.igamma;
            const double E = p * g.igm1 + 0.5 * r * (u * u + v * v);
            double Ix[4] = {r * u, r * u * u + p, r * u * v, (E + p) * u};
            double Iy[4] = {r * v, r * u * v, r * v * v + p, (E + p) * v};
            double met[5] = {0, 0, 0, 0, 0};
            if (!CART)
#pragma unroll
                for (int c = 0; c < 5; ++c) met[c] = sh_met[c * NF + t];
            if (VISC) {
                double Vx[4], Vy[4];
                visc_at_int<CART, AX>(sh_uv, sh_T, s, m, 0, g, Vx, Vy, met);
#pragma unroll
                for (int c = 1; c < 4; ++c) {
                    Ix[c] -= Vx[c];
                    Iy[c] -= Vy[c];
                }
            }
            double fx[4], fy[4];
            if (CART) {
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    fx[c] = m.cM[0] * Ix[c];
                    fy[c] = m.cM[1] * Iy[c];
                }
            } else {
                const double Mxx = met[1], Mxy = met[2], Myx = met[3], Myy = met[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    fx[c] = Mxx * Ix[c] + Mxy * Iy[c];
                    fy[c] = Myx * Ix[c] + Myy * Iy[c];
                }
            }
            fh[t] = make_double2(fx[0], fx[1]);
            fh[NF + t] = make_double2(fx[2], fx[3]);
            fh[2 * NF + t] = make_double2(fy[0], fy[1]);
            fh[3 * NF + t] = make_double2(fy[2], fy[3]);
        }
    } else
    for (int t = tid; t < NF; t += NTH) {
        const int b = t / FX, a = t - b * FX;
        const int s = (b + H - G3) * AX + (a + H - G3);
        const unsigned code = sh_c[s];
        double fx[4] = {0, 0, 0, 0}, fy[4] = {0, 0, 0, 0};
        if (code) {
            const double r = sh_r[s];
            const double2 uv = sh_uv[s];
            const double u = uv.x, v = uv.y;
            const double p = r * sh_T[s] * g.igamma;
            const double E = p * g.igm1 + 0.5 * r * (u * u + v * v);
            double Ix[4] = {r * u, r * u * u + p, r * u * v, (E + p) * u};
            double Iy[4] = {r * v, r * u * v, r * v * v + p, (E + p) * v};
            double met[5] = {0, 0, 0, 0, 0};
            if (!CART)
#pragma unroll
                for (int c = 0; c < 5; ++c) met[c] = sh_met[c * NF + t];
            if (VISC) {
                double Vx[4], Vy[4];
                visc_at<CART, AX>(sh_uv, sh_T, s, code, m, 0, g, Vx, Vy, met);
#pragma unroll
                for (int c = 1; c < 4; ++c) {
                    Ix[c] -= Vx[c];
                    Iy[c] -= Vy[c];
                }
            }
            if (CART) {
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    fx[c] = m.cM[0] * Ix[c];
                    fy[c] = m.cM[1] * Iy[c];
                }
            } else {
                const double Mxx = met[1], Mxy = met[2], Myx = met[3], Myy = met[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    fx[c] = Mxx * Ix[c] + Mxy * Iy[c];
                    fy[c] = Myx * Ix[c] + Myy * Iy[c];
                }
            }
        }
        fh[t] = make_double2(fx[0], fx[1]);
        fh[NF + t] = make_double2(fx[2], fx[3]);
        fh[2 * NF + t] = make_double2(fy[0], fy[1]);
        fh[3 * NF + t] = make_double2(fy[2], fy[3]);
    }
    __syncthreads();
    if (ep.trace && threadIdx.x == 0) tph[1] = gtimer();

    // ---- phase C: divergence, SAT, epilogue ------------------------------------------
    if (fast) {
        // interior tile: no closures, no SAT, no holes; 32-bit element offsets (one
        // IMAD.WIDE per address) and the history-ring length resolved per launch
        const unsigned uN = (unsigned)N;
        const int ns = ep.y_out ? ep.nsrc : -1;
        for (int t = tid; t < TX * TY; t += NTH) {
            const int a = t % TX, b = t / TX;
            const unsigned up = (unsigned)(i0 + a) + (unsigned)n0 * (unsigned)(j0 + b);
            const int f = (b + G3) * FX + (a + G3);
            double yb[4];
            if (ns == 2) {
                yb[0] = epi_sum<2>(ep, uN, up, 0); yb[1] = epi_sum<2>(ep, uN, up, 1);
                yb[2] = epi_sum<2>(ep, uN, up, 2); yb[3] = epi_sum<2>(ep, uN, up, 3);
            } else if (ns == 3) {
                yb[0] = epi_sum<3>(ep, uN, up, 0); yb[1] = epi_sum<3>(ep, uN, up, 1);
                yb[2] = epi_sum<3>(ep, uN, up, 2); yb[3] = epi_sum<3>(ep, uN, up, 3);
            } else if (ns >= 0) {
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    double y = __ldg(ep.base + (c * uN + up));
                    for (int k = 0; k < ns; ++k) y += ep.csrc[k] * __ldg(ep.src[k] + (c * uN + up));
                    yb[c] = y;
                }
            }
            const double2 x01 = d_int2(fh, f, 1), x23 = d_int2(fh + NF, f, 1);
            const double2 y01 = d_int2(fh + 2 * NF, f, FX), y23 = d_int2(fh + 3 * NF, f, FX);
            const double Jp = CART ? m.cJ : sh_met[f];
            double R[4];
            R[0] = -Jp * (x01.x + y01.x);
            R[1] = -Jp * (x01.y + y01.y);
            R[2] = -Jp * (x23.x + y23.x);
            R[3] = -Jp * (x23.y + y23.y);
            if (ep.r_out) {
#pragma unroll
                for (int c = 0; c < 4; ++c) ep.r_out[c * uN + up] = R[c];
            }
            if (ns >= 0) {
#pragma unroll
                for (int c = 0; c < 4; ++c) ep.y_out[c * uN + up] = yb[c] + ep.c_new * R[c];
            }
        }
        return;
    }
    for (int t = tid; t < TX * TY; t += NTH) {
        const int a = t % TX, b = t / TX;
        const int gi = i0 + a, gj = j0 + b;
        if (gi >= n0 || gj >= n1) continue;
        const int64_t p = gi + (int64_t)n0 * gj;
        const int s = (b + H) * AX + (a + H);
        const int f = (b + G3) * FX + (a + G3);
        const unsigned code = sh_c[s];
        // epilogue inputs first (streamed from HBM while the divergence is formed)
        double yb[4] = {0, 0, 0, 0};
        if (ep.y_out) {
            // all loads issued back to back (unused source slots re-read `base` with a zero
            // weight, an L1 hit) so the history ring costs one memory round trip
            const double* sp[4];
            double cw[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                sp[k] = k < ep.nsrc ? ep.src[k] : ep.base;
                cw[k] = k < ep.nsrc ? ep.csrc[k] : 0.0;
            }
            double v[5][4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                v[0][c] = __ldg(ep.base + c * N + p);
#pragma unroll
                for (int k = 0; k < 4; ++k) v[1 + k][c] = __ldg(sp[k] + c * N + p);
            }
#pragma unroll
            for (int c = 0; c < 4; ++c)
                yb[c] = v[0][c] + cw[0] * v[1][c] + cw[1] * v[2][c] + cw[2] * v[3][c] + cw[3] * v[4][c];
            for (int k = 4; k < ep.nsrc; ++k)
#pragma unroll
                for (int c = 0; c < 4; ++c) yb[c] += ep.csrc[k] * __ldg(ep.src[k] + c * N + p);
        }
        // SAT inputs of segment-end points requested before the divergence is formed
        const bool satp = code && (((code & 15) == CLS_L0) || ((code & 15) == CLS_R0) ||
                                   (((code >> 4) & 15) == CLS_L0) || (((code >> 4) & 15) == CLS_R0));
        double q[4] = {0, 0, 0, 0}, qi[4] = {0, 0, 0, 0}, fvi[6] = {0, 0, 0, 0, 0, 0};
        if (satp) {
#pragma unroll
            for (int c = 0; c < 4; ++c) q[c] = __ldg(Q + c * N + p);
            // donor data gathered by k_donor2d for this receiver
            const int slot = m.recv_slot[p];
            if (slot >= 0) {
#pragma unroll
                for (int c = 0; c < 4; ++c) qi[c] = m.qhat[c * m.nrecv + slot];
                if (VISC)
#pragma unroll
                    for (int c = 0; c < 6; ++c) fvi[c] = m.fvhat[c * m.nrecv + slot];
            }
        }
        double R[4] = {0, 0, 0, 0};
        if (code) {
            const int cx = code & 15, cy = (code >> 4) & 15;
            double2 x01, x23, y01, y23;
            if (cx == CLS_INT) {
                x01 = d_int2(fh, f, 1);
                x23 = d_int2(fh + NF, f, 1);
            } else {
                x01 = d_gen2(fh, f, 1, cx);
                x23 = d_gen2(fh + NF, f, 1, cx);
            }
            if (cy == CLS_INT) {
                y01 = d_int2(fh + 2 * NF, f, FX);
                y23 = d_int2(fh + 3 * NF, f, FX);
            } else {
                y01 = d_gen2(fh + 2 * NF, f, FX, cy);
                y23 = d_gen2(fh + 3 * NF, f, FX, cy);
            }
            const double Jp = CART ? m.cJ : sh_met[f];
            R[0] = -Jp * (x01.x + y01.x);
            R[1] = -Jp * (x01.y + y01.y);
            R[2] = -Jp * (x23.x + y23.x);
            R[3] = -Jp * (x23.y + y23.y);
            // ---- SAT ----
            if (satp) {
                double Vx[4] = {0, 0, 0, 0}, Vy[4] = {0, 0, 0, 0};
                if (VISC) {
                    double met[5] = {0, 0, 0, 0, 0};
                    if (!CART)
#pragma unroll
                        for (int c = 0; c < 5; ++c) met[c] = sh_met[c * NF + f];
                    visc_at<CART, AX>(sh_uv, sh_T, s, code, m, p, g, Vx, Vy, met);
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
                        nv[0] = Jp * sh_met[(1 + 2 * k) * NF + f];
                        nv[1] = Jp * sh_met[(2 + 2 * k) * NF + f];
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
        }
        if (ep.r_out) {
#pragma unroll
            for (int c = 0; c < 4; ++c) ep.r_out[c * N + p] = R[c];
        }
        if (ep.y_out) {
#pragma unroll
            for (int c = 0; c < 4; ++c) ep.y_out[c * N + p] = yb[c] + ep.c_new * R[c];
        }
    }
}



// ------------------------------------------------------------------------------------
// Lean interior tile (host-flagged: halo inside the mesh, every flux point interior in both
// directions).  Interior stencils reach 2, so the primitive halo is 4 (not 6) and the flux
// halo 2 (not 3); Fhat_xi is kept only on the x-extended rows and Fhat_eta only on the
// y-extended columns; all loop trip counts and offsets are compile-time; the epilogue loads of
// both output points of a thread are issued together before the divergence is formed.
// Same arithmetic as the general path.
// ------------------------------------------------------------------------------------
template <bool VISC, int TY>
struct GeoL {
    static constexpr int H = VISC ? 4 : 2, G = 2;
    static constexpr int AX = TX + 2 * H, AY = TY + 2 * H, NA = AX * AY;
    static constexpr int FX = TX + 2 * G, FY = TY + 2 * G, NF = FX * FY;
    static constexpr int NXI = FX * TY, NETA = TX * FY;    // Fhat_xi / Fhat_eta points
    // uv[NA] double2, T[NA], rho[NA], fxi[2][NXI] double2, feta[2][NETA] double2, met[5][NF]
    static constexpr size_t bytes(bool cart) {
        return 32 * (size_t)NA + 32 * (size_t)NXI + 32 * (size_t)NETA + (cart ? 0 : 40 * (size_t)NF);
    }
};

template <bool VISC, bool CART, int TY, int NTH, int NS>
__device__ __forceinline__ void rhs2d_tile_lean(const DevMesh& m, const double* __restrict__ Q,
                                                const Gas& g, const Epilogue& ep, int bx, int by,
                                                double* smem, unsigned long long* tph) {
    using GL = GeoL<VISC, TY>;
    constexpr int H = GL::H, G = GL::G, AX = GL::AX, NA = GL::NA, FX = GL::FX, NF = GL::NF;
    constexpr int NXI = GL::NXI, NETA = GL::NETA;
    double2* sh_uv = reinterpret_cast<double2*>(smem);
    double* sh_T = reinterpret_cast<double*>(sh_uv + NA);
    double* sh_r = sh_T + NA;
    double2* fxi = reinterpret_cast<double2*>(sh_r + NA);     // [2][NXI]: (F0,F1), (F2,F3)
    double2* feta = fxi + 2 * NXI;                             // [2][NETA]
    double* sh_met = reinterpret_cast<double*>(feta + 2 * NETA);   // [5][NF]
    const int n0 = m.n[0], n1 = m.n[1];
    const unsigned uN = (unsigned)m.npts, un0 = (unsigned)n0;
    const int i0 = bx * TX, j0 = by * TY;
    const int tid = threadIdx.x;
    // halo across a periodic seam (tile-uniform)
    const bool wrap = i0 - H < 0 || j0 - H < 0 || i0 + TX + H > n0 || j0 + TY + H > n1;
    // ---- curvilinear metrics of the flux points (async)
    if (!CART) {
        const unsigned qf0 = (unsigned)(i0 - G) + un0 * (unsigned)(j0 - G);
        for (int t = tid; t < NF; t += NTH) {
            const int b = t / FX, a = t - b * FX;
            const unsigned q = wrap ? wrap_idx(i0 - G + a, j0 - G + b, n0, n1)
                                    : qf0 + (unsigned)a + un0 * (unsigned)b;
            cp_async8(sh_met + t, m.J + q);
#pragma unroll
            for (int c = 0; c < 4; ++c) cp_async8(sh_met + (1 + c) * NF + t, m.M + (c * uN + q));
        }
    }
    // ---- phase A: primitives of tile + H
    {
        constexpr int KA = (NA + NTH - 1) / NTH;
        const unsigned q0 = (unsigned)(i0 - H) + un0 * (unsigned)(j0 - H);
        double ld[KA][4];
#pragma unroll
        for (int k = 0; k < KA; ++k) {
            const int t = tid + k * NTH;
            ld[k][0] = 1.0;
            ld[k][1] = ld[k][2] = ld[k][3] = 0.0;
            if (t < NA) {
                const int b = t / AX, a = t - b * AX;
                const unsigned q = wrap ? wrap_idx(i0 - H + a, j0 - H + b, n0, n1)
                                        : q0 + (unsigned)a + un0 * (unsigned)b;
#pragma unroll
                for (int c = 0; c < 4; ++c) ld[k][c] = __ldg(Q + (c * uN + q));
            }
        }
#pragma unroll
        for (int k = 0; k < KA; ++k) {
            const int t = tid + k * NTH;
            if (t < NA) {
                const double r = ld[k][0];
                const double ir = rcp64(r);
                const double u = ld[k][1] * ir, v = ld[k][2] * ir;
                sh_uv[t] = make_double2(u, v);
                sh_T[t] = g.gamma * g.gm1 * (ld[k][3] - 0.5 * (ld[k][1] * u + ld[k][2] * v)) * ir;
                sh_r[t] = r;
            }
        }
    }
    if (!CART) cp_async_wait_all();
    __syncthreads();
    if (ep.trace && threadIdx.x == 0) tph[0] = gtimer();
    // ---- phase B: fluxes at tile + G (Fhat_xi on the x-extended rows, Fhat_eta on the
    // y-extended columns; the 4 x 4 corner blocks are not needed)
    {
        constexpr int KF = (NF + NTH - 1) / NTH;
#pragma unroll 1
        for (int k = 0; k < KF; ++k) {
            const int t = tid + k * NTH;
            if (t >= NF) break;
            const int b = t / FX, a = t - b * FX;
            const bool inx = b >= G && b < G + TY, iny = a >= G && a < G + TX;
            if (!inx && !iny) continue;
            const int s = (b + H - G) * AX + (a + H - G);
            const double r = sh_r[s];
            const double2 uv = sh_uv[s];
            const double u = uv.x, v = uv.y;
            const double p = r * sh_T[s] * g.igamma;
            const double E = p * g.igm1 + 0.5 * r * (u * u + v * v);
            double Ix[4] = {r * u, r * u * u + p, r * u * v, (E + p) * u};
            double Iy[4] = {r * v, r * u * v, r * v * v + p, (E + p) * v};
            double met[5] = {0, 0, 0, 0, 0};
            if (!CART)
#pragma unroll
                for (int c = 0; c < 5; ++c) met[c] = sh_met[c * NF + t];
            if (VISC) {
                double Vx[4], Vy[4];
                visc_at_int<CART, AX>(sh_uv, sh_T, s, m, 0, g, Vx, Vy, met);
#pragma unroll
                for (int c = 1; c < 4; ++c) {
                    Ix[c] -= Vx[c];
                    Iy[c] -= Vy[c];
                }
            }
            if (inx) {
                double fx[4];
                if (CART) {
#pragma unroll
                    for (int c = 0; c < 4; ++c) fx[c] = m.cM[0] * Ix[c];
                } else {
#pragma unroll
                    for (int c = 0; c < 4; ++c) fx[c] = met[1] * Ix[c] + met[2] * Iy[c];
                }
                const int o = (b - G) * FX + a;
                fxi[o] = make_double2(fx[0], fx[1]);
                fxi[NXI + o] = make_double2(fx[2], fx[3]);
            }
            if (iny) {
                double fy[4];
                if (CART) {
#pragma unroll
                    for (int c = 0; c < 4; ++c) fy[c] = m.cM[1] * Iy[c];
                } else {
#pragma unroll
                    for (int c = 0; c < 4; ++c) fy[c] = met[3] * Ix[c] + met[4] * Iy[c];
                }
                const int o = b * TX + (a - G);
                feta[o] = make_double2(fy[0], fy[1]);
                feta[NETA + o] = make_double2(fy[2], fy[3]);
            }
        }
    }
    __syncthreads();
    if (ep.trace && threadIdx.x == 0) tph[1] = gtimer();
    // ---- phase C: divergence and epilogue; both points' epilogue loads issued first
    {
        constexpr int KC = TX * TY / NTH;
        const unsigned qc0 = (unsigned)i0 + un0 * (unsigned)j0;
        double yb[KC][4] = {};
        if (NS >= 0) {
            double v[KC][NS >= 0 ? NS + 1 : 1][4];
#pragma unroll
            for (int k = 0; k < KC; ++k) {
                const int t = tid + k * NTH;
                const unsigned up = qc0 + (unsigned)(t % TX) + un0 * (unsigned)(t / TX);
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    v[k][0][c] = __ldg(ep.base + (c * uN + up));
#pragma unroll
                    for (int s2 = 0; s2 < (NS > 0 ? NS : 0); ++s2) v[k][1 + s2][c] = __ldg(ep.src[s2] + (c * uN + up));
                }
            }
#pragma unroll
            for (int k = 0; k < KC; ++k)
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    double y = v[k][0][c];
#pragma unroll
                    for (int s2 = 0; s2 < (NS > 0 ? NS : 0); ++s2) y += ep.csrc[s2] * v[k][1 + s2][c];
                    yb[k][c] = y;
                }
        }
#pragma unroll
        for (int k = 0; k < KC; ++k) {
            const int t = tid + k * NTH;
            const int a = t % TX, b = t / TX;
            const unsigned up = qc0 + (unsigned)a + un0 * (unsigned)b;
            const int ox = b * FX + (a + G);
            const int oy = (b + G) * TX + a;
            const double2 x01 = d_int2(fxi, ox, 1), x23 = d_int2(fxi + NXI, ox, 1);
            const double2 y01 = d_int2(feta, oy, TX), y23 = d_int2(feta + NETA, oy, TX);
            const double Jp = CART ? m.cJ : sh_met[(b + G) * FX + (a + G)];
            double R[4];
            R[0] = -Jp * (x01.x + y01.x);
            R[1] = -Jp * (x01.y + y01.y);
            R[2] = -Jp * (x23.x + y23.x);
            R[3] = -Jp * (x23.y + y23.y);
            if (ep.r_out) {
#pragma unroll
                for (int c = 0; c < 4; ++c) ep.r_out[c * uN + up] = R[c];
            }
            if (NS >= 0) {
#pragma unroll
                for (int c = 0; c < 4; ++c) ep.y_out[c * uN + up] = yb[k][c] + ep.c_new * R[c];
            }
        }
    }
}

// tile lists (host-built, mrab_api.cu): bit 31 marks an interior tile -- full, halo inside
// the mesh without periodic wrap, every flux point interior in both directions.  With
// ep.persist the grid is smaller than the list and each CTA walks tiles blockIdx.x,
// blockIdx.x + gridDim.x, ... (a bulk launch that leaves SM slots to concurrent substeps).
template <bool VISC, bool CART, int TY, int MINB, int NTH>
__global__ void __launch_bounds__(NTH, MINB) k_rhs2d(DevMesh m, const double* __restrict__ Q, Gas g,
                                                    Epilogue ep, DonorSet ds) {
    extern __shared__ __align__(16) double smem[];
    unsigned long long t0 = 0, tph[2] = {0, 0};
    if (ep.trace && threadIdx.x == 0) t0 = gtimer();
    const int32_t* tlist = ep.tiles ? ep.tiles : m.tlist;
    const int ntl = ep.tiles ? ep.ntiles : m.ntl;
    const int ntx = (m.n[0] + TX - 1) / TX;
    for (int it = blockIdx.x;;) {
        int bx = it, by = blockIdx.y, tf = -1;
        if (tlist) {
            const unsigned raw = (unsigned)tlist[it];
            const int tl = (int)(raw & 0x7fffffffu);
            by = tl / ntx;
            bx = tl - by * ntx;
            tf = (int)(raw >> 31);
        }
        const int nsl = ep.y_out ? ep.nsrc : -1;
        if (tf == 1 && ep.lean && (nsl == 2 || nsl == 3 || nsl == -1)) {
            if (nsl == 2) rhs2d_tile_lean<VISC, CART, TY, NTH, 2>(m, Q, g, ep, bx, by, smem, tph);
            else if (nsl == 3) rhs2d_tile_lean<VISC, CART, TY, NTH, 3>(m, Q, g, ep, bx, by, smem, tph);
            else rhs2d_tile_lean<VISC, CART, TY, NTH, -1>(m, Q, g, ep, bx, by, smem, tph);
        } else {
            rhs2d_tile<VISC, CART, TY, NTH>(m, Q, g, ep, bx, by, tf, smem, tph);
        }
        it += gridDim.x;
        if (!tlist || it >= ntl) break;
        __syncthreads();   // the previous tile's shared data is dead
    }
    if (ep.trace) {
        __syncthreads();
        if (threadIdx.x == 0) trace_rec(ep.trace, ep.trace_tag, t0, tph[0], tph[1]);
    }
}

// ------------------------------------------------------------------------------------
// donor kernel (2-D): state on the fly + viscous flux + Lagrange gather per receiver
// ------------------------------------------------------------------------------------
__device__ __forceinline__ double src_val(const SrcSet& ss, int h, int c, int64_t N, int64_t q) {
    double v = __ldg(ss.base[h] + c * N + q);
    const int ns = ss.nsrc[h];
    for (int k = 0; k < ns; ++k) v += ss.c[h][k] * __ldg(ss.src[h][k] + c * N + q);
    return v;
}

__device__ __forceinline__ void src_prim(const SrcSet& ss, int h, int64_t N, int64_t q,
                                         const Gas& g, double& u, double& v, double& T) {
    const double r = src_val(ss, h, 0, N, q), mu = src_val(ss, h, 1, N, q);
    const double mv = src_val(ss, h, 2, N, q), E = src_val(ss, h, 3, N, q);
    const double ir = rcp64(r);
    u = mu * ir;
    v = mv * ir;
    T = g.gamma * g.gm1 * (E - 0.5 * (mu * u + mv * v)) * ir;
}

template <bool VISC>
__global__ void __launch_bounds__(128) k_donor2d(RecvTask rt, SrcSets sets, MeshTable mt, Gas g) {
    unsigned long long t0 = 0;
    if (rt.trace && threadIdx.x == 0) t0 = gtimer();
    const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 4;
    const int a = threadIdx.x & 15;
    int rm = 0;
    while (rm < rt.nmesh - 1 && gid >= rt.off[rm + 1]) ++rm;
    const bool live = gid < rt.off[rt.nmesh];
    const int64_t r = gid - rt.off[rm];
    const SrcSet& ss = sets.s[rt.set[rm]];
    double acc[10];
#pragma unroll
    for (int c = 0; c < 10; ++c) acc[c] = 0.0;
    if (live) {
        const int h = rt.rdonor[rm][r];
        const DevMesh& m = mt.m[h];
        const int n0 = m.n[0], n1 = m.n[1];
        const int64_t N = m.npts;
        int ii = rt.rbase[rm][3 * r] + (a & 3), jj = rt.rbase[rm][3 * r + 1] + (a >> 2);
        if (ii >= n0) ii -= n0;
        if (jj >= n1) jj -= n1;
        const double* w = rt.rw[rm] + 12 * r;
        const double W = w[a & 3] * w[4 + (a >> 2)];
        const int64_t q = ii + (int64_t)n0 * jj;
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[c] = W * src_val(ss, h, c, N, q);
        if (VISC) {
            const unsigned code = m.cls[q];
            const int cl[2] = {(int)(code & 15), (int)((code >> 4) & 15)};
            const int idx[2] = {ii, jj};
            const int64_t stride[2] = {1, n0};
            double d[2][3];   // d[k][u, v, T] along direction k
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                d[k][0] = d[k][1] = d[k][2] = 0.0;
                const int ns = c_nst[cl[k]];
                for (int t = 0; t < ns; ++t) {
                    int o = idx[k] + c_off[cl[k]][t];
                    const int nk = m.n[k];
                    if (o < 0) o += nk; else if (o >= nk) o -= nk;
                    const int64_t qq = q + (int64_t)(o - idx[k]) * stride[k];
                    double u, v, T;
                    src_prim(ss, h, N, qq, g, u, v, T);
                    const double cf = c_cf[cl[k]][t];
                    d[k][0] += cf * u;
                    d[k][1] += cf * v;
                    d[k][2] += cf * T;
                }
            }
            double gx[3], gy[3];   // d/dx, d/dy of (u, v, T)
            if (m.cart) {
                const double sx = m.cJ * m.cM[0], sy = m.cJ * m.cM[1];
#pragma unroll
                for (int f = 0; f < 3; ++f) {
                    gx[f] = sx * d[0][f];
                    gy[f] = sy * d[1][f];
                }
            } else {
                const double J = __ldg(m.J + q);
                const double Mxx = __ldg(m.M + q), Mxy = __ldg(m.M + N + q);
                const double Myx = __ldg(m.M + 2 * N + q), Myy = __ldg(m.M + 3 * N + q);
#pragma unroll
                for (int f = 0; f < 3; ++f) {
                    gx[f] = J * (Mxx * d[0][f] + Myx * d[1][f]);
                    gy[f] = J * (Mxy * d[0][f] + Myy * d[1][f]);
                }
            }
            double u, v, T;
            src_prim(ss, h, N, q, g, u, v, T);
            const double div = gx[0] + gy[1];
            const double txx = (2.0 * gx[0] - (2.0 / 3.0) * div) * g.iRe;
            const double tyy = (2.0 * gy[1] - (2.0 / 3.0) * div) * g.iRe;
            const double txy = (gy[0] + gx[1]) * g.iRe;
            acc[4] = W * txx;
            acc[5] = W * txy;
            acc[6] = W * (u * txx + v * txy + g.kT * gx[2]);
            acc[7] = W * txy;
            acc[8] = W * tyy;
            acc[9] = W * (u * txy + v * tyy + g.kT * gy[2]);
        }
    }
#pragma unroll
    for (int c = 0; c < 10; ++c) {
        double v = acc[c];
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        acc[c] = v;
    }
    if (live && a == 0) {
        const int64_t R = rt.nrecv[rm];
#pragma unroll
        for (int c = 0; c < 4; ++c) rt.qhat[rm][c * R + r] = acc[c];
        if (VISC)
#pragma unroll
            for (int c = 0; c < 6; ++c) rt.fvhat[rm][c * R + r] = acc[4 + c];
    }
    if (rt.trace) {
        __syncthreads();
        if (threadIdx.x == 0) trace_rec(rt.trace, rt.trace_tag, t0);
    }
}

// Region-staged variant: the 16 lanes of a receiver first form the donor state at the
// plus-shaped region every SBP row of the 4 x 4 stencil can reach (rows of the stencil
// +-3 along xi, columns +-3 along eta: 64 points, 4 per lane, all loads independent), keep
// the primitives (u, v, T) in shared memory, then take the segmented D1 from there.  Same
// arithmetic as k_donor2d, ~3x fewer global loads and no dependent load chains.
constexpr int RG = 10;                 // region box edge (-3 .. 6)
// two receivers (one warp) per CTA: the CTA (~21 KB of shared memory) fits beside the RHS
// tiles of a concurrently running mesh
constexpr int DRPC = 2;
template <bool VISC>
__global__ void __launch_bounds__(16 * DRPC) k_donor2d_r(RecvTask rt, SrcSets sets, MeshTable mt, Gas g) {
    __shared__ double sh_p[DRPC][3][RG * RG];  // (u, v, T) of the region, per receiver
    __shared__ double sh_q[DRPC][4][16];       // state at the 16 stencil points
    unsigned long long t0 = 0;
    if (rt.trace && threadIdx.x == 0) t0 = gtimer();
    const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 4;
    const int a = threadIdx.x & 15;
    const int slot = threadIdx.x >> 4;
    int rm = 0;
    while (rm < rt.nmesh - 1 && gid >= rt.off[rm + 1]) ++rm;
    const bool live = gid < rt.off[rt.nmesh];
    const int64_t r = gid - rt.off[rm];
    const SrcSet& ss = sets.s[rt.set[rm]];
    int h = 0, ib = 0, jb = 0;
    if (live) {
        h = rt.rdonor[rm][r];
        ib = rt.rbase[rm][3 * r];
        jb = rt.rbase[rm][3 * r + 1];
    }
    const DevMesh& m = mt.m[h];
    const int n0 = m.n[0], n1 = m.n[1];
    const unsigned uN = (unsigned)m.npts;
    const int ns = ss.nsrc[h];
    // kernel parameters indexed by the donor mesh are read once into registers: the parameter
    // block (~10 KB) exceeds the constant cache, so re-reading it inside loops serialises
    const int per0 = m.periodic[0], per1 = m.periodic[1];
    const double* bp = ss.base[h];
    const double* sp[6];
    double cw[6];
#pragma unroll
    for (int t = 0; t < 6; ++t) {
        sp[t] = t < ns ? ss.src[h][t] : bp;
        cw[t] = t < ns ? ss.c[h][t] : 0.0;
    }
    // this lane's stencil point: weights, class code and metrics requested together with the
    // region loads below (one memory round trip after the receiver's base is known)
    const int ai = a & 3, aj = a >> 2;
    double W = 0.0, Jq = 0.0, Mq[4] = {0, 0, 0, 0};
    unsigned code = 0;
    unsigned qown = 0;
    if (live) {
        int ii = ib + ai, jj = jb + aj;
        if (ii >= n0) ii -= n0;
        if (jj >= n1) jj -= n1;
        qown = (unsigned)ii + (unsigned)n0 * (unsigned)jj;
        const double* w = rt.rw[rm] + 12 * r;
        W = w[ai] * w[4 + aj];
        if (VISC) {
            code = m.cls[qown];
            if (!m.cart) {
                Jq = __ldg(m.J + qown);
#pragma unroll
                for (int c = 0; c < 4; ++c) Mq[c] = __ldg(m.M + (c * uN + qown));
            }
        }
    }
    // ---- stage the region: every raw value (base and history terms) is copied to shared
    // memory asynchronously (one memory round trip, no register staging), then combined
    if (live) {
        extern __shared__ double raw[];   // [DRPC receivers][rt.raw_k arrays][4 comps][64 points]
        double* my = raw + (size_t)slot * rt.raw_k * 256;
        bool ok[4];
        int di[4], dj[4];
#pragma unroll
        for (int s4 = 0; s4 < 4; ++s4) {
            const int k = a + 16 * s4;
            if (k < 40) {
                dj[s4] = k / 10;
                di[s4] = k % 10 - 3;
            } else {
                const int kk = k - 40, r6 = kk >> 2;
                di[s4] = kk & 3;
                dj[s4] = r6 < 3 ? r6 - 3 : r6 + 1;
            }
            ok[s4] = true;
            if (!VISC && !(dj[s4] >= 0 && dj[s4] < 4 && di[s4] >= 0 && di[s4] < 4)) {
                ok[s4] = false;
                continue;
            }
            int ii = ib + di[s4], jj = jb + dj[s4];
            if (ii < 0 || ii >= n0) {
                if (per0) ii = ii < 0 ? ii + n0 : ii - n0; else ok[s4] = false;
            }
            if (jj < 0 || jj >= n1) {
                if (per1) jj = jj < 0 ? jj + n1 : jj - n1; else ok[s4] = false;
            }
            if (!ok[s4]) continue;
            const unsigned q = (unsigned)ii + (unsigned)n0 * (unsigned)jj;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                cp_async8(my + c * 64 + k, bp + (c * uN + q));
#pragma unroll
                for (int t = 0; t < 6; ++t)
                    if (t < ns) cp_async8(my + ((1 + t) * 4 + c) * 64 + k, sp[t] + (c * uN + q));
            }
        }
        cp_async_wait_all();
        double ld[4][4];
#pragma unroll
        for (int s4 = 0; s4 < 4; ++s4) {
            const int k = a + 16 * s4;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                double v = 0.0;
                if (ok[s4]) {
                    v = my[c * 64 + k];
#pragma unroll
                    for (int t = 0; t < 6; ++t)
                        if (t < ns) v += cw[t] * my[((1 + t) * 4 + c) * 64 + k];
                }
                ld[s4][c] = v;
            }
        }
#pragma unroll
        for (int s4 = 0; s4 < 4; ++s4) {
            const int e = (dj[s4] + 3) * RG + (di[s4] + 3);
            if (dj[s4] >= 0 && dj[s4] < 4 && di[s4] >= 0 && di[s4] < 4) {
#pragma unroll
                for (int c = 0; c < 4; ++c) sh_q[slot][c][dj[s4] * 4 + di[s4]] = ld[s4][c];
            }
            if (VISC) {
                double u = 0.0, v = 0.0, T = 0.0;
                if (ok[s4]) {
                    const double ir = rcp64(ld[s4][0]);
                    u = ld[s4][1] * ir;
                    v = ld[s4][2] * ir;
                    T = g.gamma * g.gm1 * (ld[s4][3] - 0.5 * (ld[s4][1] * u + ld[s4][2] * v)) * ir;
                }
                sh_p[slot][0][e] = u;
                sh_p[slot][1][e] = v;
                sh_p[slot][2][e] = T;
            }
        }
    }
    __syncwarp();
    double acc[10];
#pragma unroll
    for (int c = 0; c < 10; ++c) acc[c] = 0.0;
    if (live) {
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[c] = W * sh_q[slot][c][a];
        if (VISC) {
            const int cl[2] = {(int)(code & 15), (int)((code >> 4) & 15)};
            const int e0 = (aj + 3) * RG + (ai + 3);
            const int stride[2] = {1, RG};
            double d[2][3];
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                d[k][0] = d[k][1] = d[k][2] = 0.0;
                const int nt = c_nst[cl[k]];
                for (int t = 0; t < nt; ++t) {
                    const int e = e0 + c_off[cl[k]][t] * stride[k];
                    const double cf = c_cf[cl[k]][t];
                    d[k][0] += cf * sh_p[slot][0][e];
                    d[k][1] += cf * sh_p[slot][1][e];
                    d[k][2] += cf * sh_p[slot][2][e];
                }
            }
            double gx[3], gy[3];
            if (m.cart) {
                const double sx = m.cJ * m.cM[0], sy = m.cJ * m.cM[1];
#pragma unroll
                for (int f = 0; f < 3; ++f) {
                    gx[f] = sx * d[0][f];
                    gy[f] = sy * d[1][f];
                }
            } else {
                const double J = Jq, Mxx = Mq[0], Mxy = Mq[1], Myx = Mq[2], Myy = Mq[3];
#pragma unroll
                for (int f = 0; f < 3; ++f) {
                    gx[f] = J * (Mxx * d[0][f] + Myx * d[1][f]);
                    gy[f] = J * (Mxy * d[0][f] + Myy * d[1][f]);
                }
            }
            const double u = sh_p[slot][0][e0], v = sh_p[slot][1][e0];
            const double div = gx[0] + gy[1];
            const double txx = (2.0 * gx[0] - (2.0 / 3.0) * div) * g.iRe;
            const double tyy = (2.0 * gy[1] - (2.0 / 3.0) * div) * g.iRe;
            const double txy = (gy[0] + gx[1]) * g.iRe;
            acc[4] = W * txx;
            acc[5] = W * txy;
            acc[6] = W * (u * txx + v * txy + g.kT * gx[2]);
            acc[7] = W * txy;
            acc[8] = W * tyy;
            acc[9] = W * (u * txy + v * tyy + g.kT * gy[2]);
        }
    }
#pragma unroll
    for (int c = 0; c < 10; ++c) {
        double v = acc[c];
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        acc[c] = v;
    }
    if (live && a == 0) {
        const int64_t R = rt.nrecv[rm];
#pragma unroll
        for (int c = 0; c < 4; ++c) rt.qhat[rm][c * R + r] = acc[c];
        if (VISC)
#pragma unroll
            for (int c = 0; c < 6; ++c) rt.fvhat[rm][c * R + r] = acc[4 + c];
    }
    if (rt.trace) {
        __syncthreads();
        if (threadIdx.x == 0) trace_rec(rt.trace, rt.trace_tag, t0);
    }
}

void launch_donor2d(const RecvTask& rt0, const SrcSets& ss, const MeshTable& mt, const Gas& gas,
                    cudaStream_t st) {
    RecvTask rt = rt0;
    int nsmax = 0;
    for (int i = 0; i < rt.nmesh; ++i)
        for (int h = 0; h < 8; ++h) nsmax = std::max(nsmax, std::min(6, ss.s[rt.set[i]].nsrc[h]));
    rt.raw_k = 1 + nsmax;
    const int64_t tot = rt.off[rt.nmesh];
    if (tot <= 0) return;
    const unsigned nb = (unsigned)((tot * 16 + 127) / 128);
    const unsigned nbr = (unsigned)((tot + DRPC - 1) / DRPC);
    // the gather sits on the critical path of the fast substeps: highest launch priority
    static int greatest = 1;
    if (greatest > 0) {
        int least = 0;
        cudaDeviceGetStreamPriorityRange(&least, &greatest);
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nb);
    cfg.blockDim = dim3(128);
    cfg.stream = st;
    // raw staging of the region-staged variant: DRPC receivers x (1 + max history terms) x 4 x 64
    cfg.dynamicSmemBytes = (size_t)DRPC * rt.raw_k * 256 * sizeof(double);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributePriority;
    at[0].val.priority = greatest;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (opts().donor_staged) {
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(k_donor2d_r<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
            cudaFuncSetAttribute(k_donor2d_r<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
            attr = true;
        }
        cfg.gridDim = dim3(nbr);
        cfg.blockDim = dim3(16 * DRPC);
        if (gas.viscous) cudaLaunchKernelEx(&cfg, k_donor2d_r<true>, rt, ss, mt, gas);
        else cudaLaunchKernelEx(&cfg, k_donor2d_r<false>, rt, ss, mt, gas);
    } else {
        cfg.dynamicSmemBytes = 0;
        if (gas.viscous) cudaLaunchKernelEx(&cfg, k_donor2d<true>, rt, ss, mt, gas);
        else cudaLaunchKernelEx(&cfg, k_donor2d<false>, rt, ss, mt, gas);
    }
}

template <bool VISC, bool CART, int TY, int MINB, int NTH>
static void launch_t(const DevMesh& m, const double* Q, const Gas& g, const Epilogue& ep0,
                     const DonorSet& ds, cudaStream_t st) {
    static bool init = false;
    Epilogue ep = ep0;
    ep.pf = opts().pf;
    ep.lean = opts().lean;
    const size_t bytes = std::max(Geo<VISC, TY, CART>::bytes, GeoL<VISC, TY>::bytes(CART));
    if (!init) {
        cudaFuncSetAttribute(k_rhs2d<VISC, CART, TY, MINB, NTH>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        init = true;
    }
    dim3 grid((m.n[0] + TX - 1) / TX, (m.n[1] + TY - 1) / TY);
    if (ep.tiles) grid = dim3(ep.persist > 0 ? std::min(ep.persist, ep.ntiles) : ep.ntiles, 1);
    else if (m.tlist) grid = dim3(m.ntl, 1);
    if (grid.x * grid.y == 0) return;
    if (ep.has_prio) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid;
        cfg.blockDim = dim3(NTH);
        cfg.dynamicSmemBytes = bytes;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributePriority;
        at[0].val.priority = ep.prio;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, k_rhs2d<VISC, CART, TY, MINB, NTH>, m, Q, g, ep, ds);
        return;
    }
    k_rhs2d<VISC, CART, TY, MINB, NTH><<<grid, NTH, bytes, st>>>(m, Q, g, ep, ds);
}

// tile-shape variant (Options::k2d, for tuning): 0 = 32x16 tile, 256 threads, 2 CTAs/SM
// (default); 1 = 32x8 / 256 / 2; 2 = 32x8 / 256 / 3; 3 = 32x16 / 512 / 1; 4 = 32x32 / 512 / 1;
// -2 = per mesh (rhs2d_variant_for)
static int k2d_variant() { return opts().k2d; }

// per-mesh tile shape: small curvilinear meshes (the config-3 O-grid, 65k points: one wave of
// latency-bound tiles) take 32 x 8 tiles (twice as many CTAs, shorter per-CTA chains); the
// rest 32 x 16.  Options::k2d forces a variant everywhere; Options::small_pts sets the threshold.
int rhs2d_variant_for(const int* n, int cart) {
    const int v = k2d_variant();
    if (v >= 0) return v;
    return (!cart && (long)n[0] * n[1] <= opts().small_pts) ? 1 : 0;
}

void rhs2d_tile_shape_for(const int* n, int cart, int* tx, int* ty) {
    *tx = TX;
    const int v = rhs2d_variant_for(n, cart);
    *ty = (v == 0 || v == 3) ? 16 : (v == 4 ? 32 : 8);
}

bool rhs2d_interior_tile(const int* n, const int* periodic, const uint16_t* cls, int viscous,
                         int bx, int by, int cart) {
    int tx, ty;
    rhs2d_tile_shape_for(n, cart, &tx, &ty);
    const int H = viscous ? Geo<true, 16>::H : Geo<false, 16>::H;
    const int i0 = bx * tx, j0 = by * ty;
    if (i0 + tx > n[0] || j0 + ty > n[1]) return false;
    // the halo may cross a seam only in periodic directions (and at most once)
    if (n[0] < tx + 2 * H || n[1] < ty + 2 * H) return false;
    if (!periodic[0] && (i0 - H < 0 || i0 + tx + H > n[0])) return false;
    if (!periodic[1] && (j0 - H < 0 || j0 + ty + H > n[1])) return false;
    const unsigned want = CLS_INT | (CLS_INT << 4);
    for (int j = j0 - G3; j < j0 + ty + G3; ++j)
        for (int i = i0 - G3; i < i0 + tx + G3; ++i) {
            const int ii = (i + n[0]) % n[0], jj = (j + n[1]) % n[1];
            if (cls[ii + (size_t)n[0] * jj] != want) return false;
        }
    return true;
}

void rhs2d_tile_shape(int* tx, int* ty) {
    *tx = TX;
    const int v = k2d_variant() < 0 ? 0 : k2d_variant();
    *ty = (v == 0 || v == 3) ? 16 : (v == 4 ? 32 : 8);
}

template <bool VISC, bool CART>
static void launch_v(const DevMesh& m, const double* Q, const Gas& g, const Epilogue& ep,
                     const DonorSet& ds, cudaStream_t st) {
    switch (rhs2d_variant_for(m.n, m.cart)) {
        case 1: launch_t<VISC, CART, 8, 2, 256>(m, Q, g, ep, ds, st); break;
        case 2: launch_t<VISC, CART, 8, 3, 256>(m, Q, g, ep, ds, st); break;
        case 3: launch_t<VISC, CART, 16, 1, 512>(m, Q, g, ep, ds, st); break;
        case 4: launch_t<VISC, CART, 32, 1, 512>(m, Q, g, ep, ds, st); break;
        // curvilinear meshes stage their metrics too (one CTA per SM): no register cap
        default: {
            // curvilinear tiles capped at 128 registers so that one fits in half an SM beside a
            // Cartesian bulk tile in the overlapped schedule (Options::curv_half = 0: no cap)
            if (CART || opts().curv_half) launch_t<VISC, CART, 16, 2, 256>(m, Q, g, ep, ds, st);
            else launch_t<VISC, CART, 16, 1, 256>(m, Q, g, ep, ds, st);
            break;
        }
    }
}


// Lean-only kernel over a list of interior tiles: with the general path compiled out it needs
// 69.6 KB of shared memory (Cartesian) and 80 registers (three CTAs per SM).  Diagnostic only
// (mrab_time_kernel kernel 3; kernel 4 = the same tiles in the mixed kernel): measured 53.6 us
// vs 48.4 us for the mixed kernel on the config-3 interior tiles, i.e. occupancy is not what
// limits the lean path (its L1/LSU data pipe runs at 63 % of peak).
template <bool VISC, bool CART, int NS>
__global__ void __launch_bounds__(256, CART ? 3 : 2) k_rhs2d_lean(DevMesh m, const double* __restrict__ Q,
                                                                  Gas g, Epilogue ep) {
    extern __shared__ __align__(16) double smem[];
    unsigned long long t0 = 0, tph[2] = {0, 0};
    if (ep.trace && threadIdx.x == 0) t0 = gtimer();
    const int ntx = (m.n[0] + TX - 1) / TX;
    const int tl = (int)((unsigned)ep.tiles[blockIdx.x] & 0x7fffffffu);
    const int by = tl / ntx, bx = tl - by * ntx;
    rhs2d_tile_lean<VISC, CART, 16, 256, NS>(m, Q, g, ep, bx, by, smem, tph);
    if (ep.trace) {
        __syncthreads();
        if (threadIdx.x == 0) trace_rec(ep.trace, ep.trace_tag, t0, tph[0], tph[1]);
    }
}

template <bool VISC, bool CART, int NS>
static void launch_lean(const DevMesh& m, const double* Q, const Gas& g, const Epilogue& ep, cudaStream_t st) {
    static bool init = false;
    const size_t bytes = GeoL<VISC, 16>::bytes(CART);
    if (!init) {
        cudaFuncSetAttribute(k_rhs2d_lean<VISC, CART, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        init = true;
    }
    k_rhs2d_lean<VISC, CART, NS><<<ep.ntiles, 256, bytes, st>>>(m, Q, g, ep);
}

static void launch_rhs2d_lean(const DevMesh& m, const double* Q, const Gas& g, const Epilogue& ep0,
                              cudaStream_t st) {
    if (ep0.ntiles <= 0) return;
    Epilogue ep = ep0;
    ep.lean = 1;
    const int ns = ep.y_out ? ep.nsrc : -1;
#define MRAB_LEANL(V, C)                                          \
    if (ns == 2) launch_lean<V, C, 2>(m, Q, g, ep, st);           \
    else if (ns == 3) launch_lean<V, C, 3>(m, Q, g, ep, st);      \
    else launch_lean<V, C, -1>(m, Q, g, ep, st);
    if (g.viscous) {
        if (m.cart) { MRAB_LEANL(true, true) } else { MRAB_LEANL(true, false) }
    } else {
        if (m.cart) { MRAB_LEANL(false, true) } else { MRAB_LEANL(false, false) }
    }
#undef MRAB_LEANL
}


void launch_rhs2d(const DevMesh& m, const double* Q, const Gas& g, const Epilogue& ep,
                  const DonorSet& ds, cudaStream_t st) {
    // interior tiles only: the lean kernel
    if (ep.lean_only) {
        launch_rhs2d_lean(m, Q, g, ep, st);
        return;
    }
    if (g.viscous) {
        if (m.cart) launch_v<true, true>(m, Q, g, ep, ds, st);
        else launch_v<true, false>(m, Q, g, ep, ds, st);
    } else {
        if (m.cart) launch_v<false, true>(m, Q, g, ep, ds, st);
        else launch_v<false, false>(m, Q, g, ep, ds, st);
    }
}

}  // namespace mrab
