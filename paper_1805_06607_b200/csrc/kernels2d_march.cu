// 2-D fused SBP-SAT right-hand side, row-marching variant for large viscous meshes
// (sm_100a, fp64).  Same arithmetic as k_rhs2d (kernels2d.cu):
//   primitives -> D1 gradients (segment closures by class code, P:1526-1528 D1 o D1) ->
//   viscous + inviscid fluxes -> contravariant fluxes -> R = -J (D_xi Fhat_xi + D_eta Fhat_eta)
//    -> SAT at segment ends (eq:int P:279-299) -> AB / RK combination epilogue
//   (eq:ab_general P:358-361).
//
// Work item = a strip of output columns [c0, c1) (<= 116 wide) over rows [ja, jb).  One CTA of
// 128 threads owns the strip plus a 6-column halo on each side: thread t <-> column c0-6+t.
// The CTA marches up the rows with a three-stage pipeline per row step:
//   stage P  primitives of lead row L               -> shared ring (8 rows)
//   stage F  fluxes of row F = L-3 (gradients from the primitive ring: x by neighbour
//            columns, y by the thread's own column)  -> Fhat_xi ring (4 rows, read by
//            neighbours), Fhat_eta ring (7 rows, own column only)
//   stage O  divergence, SAT and epilogue of row O = F-3
// so every primitive and flux is formed once per strip (no 2-D halo recomputation; only the
// 12 lead-in rows of a work item are extra), one __syncthreads per row step, and all global
// traffic is row-coalesced.  Each register buffer of global inputs is refilled for row step
// k+1 right after its last use in step k, so its loads are in flight through the rest of the
// step (an additional L2 prefetch several rows ahead measured no gain and was dropped).  Viscous fluxes of SAT points (needed again in
// stage O, after the primitive ring has moved on) are parked in a per-point scratch array.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "kernels.cuh"
#include "mrab_internal.h"
#include "rhs2d_common.cuh"
#include "stencil_table.cuh"

namespace mrab {

namespace {

using namespace k2d;
constexpr int MT = 128;            // threads = primitive columns of a strip
constexpr int MH = 6;              // primitive halo (flux reach 3 + gradient reach 3)
constexpr int MW = MT - 2 * MH;    // output columns per strip (116)
constexpr int RP = 8;              // primitive ring rows (power of two; WAR-safe with 1 sync)
constexpr int RFX = 4;             // Fhat_xi ring rows
constexpr int RFY = 8;             // Fhat_eta ring rows (own column: O-3 .. O+3, power of two)
constexpr unsigned INTINT = CLS_INT | (CLS_INT << 4);
constexpr double kP0m = 17.0 / 48.0;
// shared: uv[RP][MT] double2, T[RP][MT], fx[RFX][2][MT] double2, fy[RFY][2][MT] double2 (72 KB:
// three CTAs per SM); the density travels from stage P to stage F in registers
constexpr size_t MBYTES = 16 * (size_t)RP * MT + 8 * (size_t)RP * MT + 32 * (size_t)RFX * MT +
                          32 * (size_t)RFY * MT;

// general D1 row (class cl) along the ring of `mod` rows with row pitch `pitch`
template <typename V>
__device__ __forceinline__ V ring_gen(const V* f, int r, int t, int cl, int pitch, int mod);

template <>
__device__ __forceinline__ double ring_gen<double>(const double* f, int r, int t, int cl, int pitch, int mod) {
    double acc = 0.0;
    const int n = c_nst[cl];
    for (int s = 0; s < n; ++s) {
        const int rr = (r + c_off[cl][s] + 4 * mod) % mod;
        acc += c_cf[cl][s] * f[rr * pitch + t];
    }
    return acc;
}

template <>
__device__ __forceinline__ double2 ring_gen<double2>(const double2* f, int r, int t, int cl, int pitch, int mod) {
    double2 acc = make_double2(0.0, 0.0);
    const int n = c_nst[cl];
    for (int s = 0; s < n; ++s) {
        const int rr = (r + c_off[cl][s] + 4 * mod) % mod;
        const double c = c_cf[cl][s];
        const double2 v = f[rr * pitch + t];
        acc.x += c * v.x;
        acc.y += c * v.y;
    }
    return acc;
}

// SAT penalties at a segment-end point (same algebra as sat2d in rhs2d_common.cuh, with the
// point's Cartesian viscous fluxes Vx, Vy passed in)
template <bool CART>
__device__ __forceinline__ void sat2d_m(const DevMesh& m, const double* __restrict__ Q, const Gas& g,
                                        const double* Vx, const double* Vy, unsigned code, unsigned p,
                                        int gi, int gj, double Jp, double* R) {
    const unsigned uN = (unsigned)m.npts;
    const int cx = code & 15, cy = (code >> 4) & 15;
    double q[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) q[c] = __ldg(Q + (c * uN + p));
    const int slot = m.recv_slot[p];
    double qi[4] = {0, 0, 0, 0}, fvi[6] = {0, 0, 0, 0, 0, 0};
    if (slot >= 0) {
#pragma unroll
        for (int c = 0; c < 4; ++c) qi[c] = m.qhat[c * m.nrecv + slot];
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
            nv[0] = Jp * __ldg(m.M + ((2 * k) * uN + p));
            nv[1] = Jp * __ldg(m.M + ((2 * k + 1) * uN + p));
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
        const double sig1 = 0.5 * (nv[0] * nv[0] + nv[1] * nv[1]) * g.iRe;
#pragma unroll
        for (int c = 0; c < 4; ++c) R[c] -= (0.5 * kd[c] + sig1 * dq[c]) * (1.0 / kP0m);
        if (typ != MRAB_BC_WALL) {
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const double fk = nv[0] * Vx[j] + nv[1] * Vy[j];
                double fhv = 0.0;
                if (typ == MRAB_BC_OVERSET) fhv = nv[0] * fvi[j] + nv[1] * fvi[3 + j];
                R[1 + j] += 0.5 * side * (fk - fhv) * (1.0 / kP0m);
            }
        }
    }
}

__device__ __forceinline__ bool is_sat(unsigned code) {
    const int cx = code & 15, cy = (code >> 4) & 15;
    return cx == CLS_L0 || cx == CLS_R0 || cy == CLS_L0 || cy == CLS_R0;
}

}  // namespace

struct MarchGrid {
    int ns;   // strips
    int w;    // strip width (output columns, <= MW)
    int L;    // rows per work item
};

// NS: history sources of the epilogue (-1: no state update, R only).  CTA b = work item
// (row chunk b / ns, strip b % ns); every row quantity below is CTA-uniform.
template <bool CART, int NS>
__global__ void __launch_bounds__(MT, 3)
    k_rhs2d_m(DevMesh m, const double* __restrict__ Q, Gas g, Epilogue ep, MarchGrid mg,
              double* __restrict__ satv) {
    extern __shared__ __align__(16) double smem[];
    double2* s_uv = reinterpret_cast<double2*>(smem);          // [RP][MT]
    double* s_T = reinterpret_cast<double*>(s_uv + RP * MT);   // [RP][MT]
    double2* s_fx = reinterpret_cast<double2*>(s_T + RP * MT); // [RFX][2][MT]
    double2* s_fy = s_fx + RFX * 2 * MT;                       // [RFY][2][MT]

    unsigned long long t0 = 0;
    if (ep.trace && threadIdx.x == 0) t0 = gtimer();
    const int n0 = m.n[0], n1 = m.n[1];
    const int strip = blockIdx.x % mg.ns, chunk = blockIdx.x / mg.ns;
    const int c0 = strip * mg.w, c1 = min(n0, c0 + mg.w);
    const int ja = chunk * mg.L, jb = min(n1, ja + mg.L);
    const int t = threadIdx.x;
    const unsigned uN = (unsigned)m.npts;
    const unsigned un0 = (unsigned)n0;

    // this thread's column
    const int x = c0 - MH + t;
    int xl = x;
    bool xok = true;
    if (x < 0 || x >= n0) {
        if (m.periodic[0]) xl = x < 0 ? x + n0 : x - n0;
        else {
            xl = min(max(x, 0), n0 - 1);
            xok = false;
        }
    }
    const bool fl = xok && x >= c0 - 3 && x < c1 + 3;   // flux lane
    const bool ol = x >= c0 && x < c1;                   // output lane
    const bool yper = m.periodic[1] != 0;
    // row r of the mesh to read (wrapped if periodic, clamped if outside: such rows feed no
    // active stencil, they only keep the arithmetic finite)
    auto rowmap = [&](int r, bool& ok) -> int {
        if (r >= 0 && r < n1) { ok = true; return r; }
        if (yper) { ok = true; return r < 0 ? r + n1 : r - n1; }
        ok = false;
        return min(max(r, 0), n1 - 1);
    };

    const double sx = m.cJ * m.cM[0], sy = m.cJ * m.cM[1];
    const int niter = (jb - ja) + 12;

    // ---- global inputs of the current row step; each buffer is refilled for the next step
    // right after its last use, so its loads are in flight through the rest of the step
    double qn[4];                 // state at the lead row
    unsigned cfn = 0, con = 0;    // class codes at the flux / output rows
    double mfn[5];                // J, Mxx, Mxy, Myx, Myy at the flux row (curvilinear)
    double en[NS >= 0 ? NS + 1 : 1][4];   // epilogue inputs (base, sources) at the output row
    double jon = 0.0;             // J at the output row (curvilinear)
    double r1 = 1.0, r2 = 1.0, r3 = 1.0;  // density at rows L-1, L-2, L-3 (own column)

    auto load_P = [&](int k) {
        bool ok;
        const unsigned ql = (unsigned)xl + un0 * (unsigned)rowmap(ja - 6 + k, ok);
#pragma unroll
        for (int c = 0; c < 4; ++c) qn[c] = __ldg(Q + (c * uN + ql));
    };
    auto load_F = [&](int k) {
        const int F = ja - 9 + k;
        if (F >= ja - 3) {
            bool ok;
            const unsigned qf = (unsigned)xl + un0 * (unsigned)rowmap(F, ok);
            cfn = (fl && ok) ? (unsigned)__ldg(m.cls + qf) : 0u;
            if (!CART) {
                mfn[0] = __ldg(m.J + qf);
#pragma unroll
                for (int c = 0; c < 4; ++c) mfn[1 + c] = __ldg(m.M + (c * uN + qf));
            }
        }
    };
    auto load_O = [&](int k) {
        const int O = ja - 12 + k;
        if (O >= ja && ol) {
            const unsigned qo = (unsigned)x + un0 * (unsigned)O;
            con = __ldg(m.cls + qo);
            if (!CART) jon = __ldg(m.J + qo);
            if (NS >= 0) {
#pragma unroll
                for (int c = 0; c < 4; ++c) en[0][c] = __ldg(ep.base + (c * uN + qo));
#pragma unroll
                for (int s = 0; s < (NS > 0 ? NS : 0); ++s)
#pragma unroll
                    for (int c = 0; c < 4; ++c) en[1 + s][c] = __ldg(ep.src[s] + (c * uN + qo));
            }
        }
    };

    load_P(0);
    load_F(0);
    load_O(0);
#pragma unroll 1
    for (int k = 0; k < niter; ++k) {
        const int L = ja - 6 + k, F = L - 3, O = L - 6;
        const bool more = k + 1 < niter;
        // CTA-uniform ring row offsets (elements)
        const int pL = (L & (RP - 1)) * MT;
        double rL;
        // ---- stage P: primitives of row L
        {
            const double r = qn[0];
            const double ir = rcp64(r);
            const double u = qn[1] * ir, v = qn[2] * ir;
            const double T = g.gamma * g.gm1 * (qn[3] - 0.5 * (qn[1] * u + qn[2] * v)) * ir;
            s_uv[pL + t] = make_double2(u, v);
            s_T[pL + t] = T;
            rL = r;
        }
        if (more) load_P(k + 1);
        __syncthreads();

        // ---- stage F: fluxes of row F
        if (F >= ja - 3) {
            bool fok;
            const int Fl = rowmap(F, fok);
            const bool act = fl && fok;
            const unsigned code = act ? cfn : 0u;
            const bool fast = __all_sync(0xffffffffu, !act || code == INTINT);
            if (act && (fast || code)) {
                const int pF = (F & (RP - 1)) * MT;
                const int sF = pF + t;
                double2 uvx, uvy;
                double Tx, Ty;
                int cx = CLS_INT, cy = CLS_INT;
                if (!fast) {
                    cx = code & 15;
                    cy = (code >> 4) & 15;
                }
                if (cx == CLS_INT) {
                    uvx = d_int2(s_uv, sF, 1);
                    Tx = d_int(s_T, sF, 1);
                } else {
                    uvx = d_gen2(s_uv, sF, 1, cx);
                    Tx = d_gen(s_T, sF, 1, cx);
                }
                if (cy == CLS_INT) {
                    const int a1 = ((F + 1) & (RP - 1)) * MT, b1 = ((F - 1) & (RP - 1)) * MT;
                    const int a2 = ((F + 2) & (RP - 1)) * MT, b2 = ((F - 2) & (RP - 1)) * MT;
                    const double2 A1 = s_uv[a1 + t], B1 = s_uv[b1 + t], A2 = s_uv[a2 + t], B2 = s_uv[b2 + t];
                    uvy = make_double2(C1 * (A1.x - B1.x) - C2 * (A2.x - B2.x),
                                       C1 * (A1.y - B1.y) - C2 * (A2.y - B2.y));
                    Ty = C1 * (s_T[a1 + t] - s_T[b1 + t]) - C2 * (s_T[a2 + t] - s_T[b2 + t]);
                } else {
                    uvy = ring_gen<double2>(s_uv, F + 8 * RP, t, cy, MT, RP);
                    Ty = ring_gen<double>(s_T, F + 8 * RP, t, cy, MT, RP);
                }
                double dudx, dudy, dvdx, dvdy, dTdx, dTdy;
                if (CART) {
                    dudx = sx * uvx.x; dvdx = sx * uvx.y; dTdx = sx * Tx;
                    dudy = sy * uvy.x; dvdy = sy * uvy.y; dTdy = sy * Ty;
                } else {
                    const double J = mfn[0], Mxx = mfn[1], Mxy = mfn[2], Myx = mfn[3], Myy = mfn[4];
                    dudx = J * (Mxx * uvx.x + Myx * uvy.x); dudy = J * (Mxy * uvx.x + Myy * uvy.x);
                    dvdx = J * (Mxx * uvx.y + Myx * uvy.y); dvdy = J * (Mxy * uvx.y + Myy * uvy.y);
                    dTdx = J * (Mxx * Tx + Myx * Ty); dTdy = J * (Mxy * Tx + Myy * Ty);
                }
                const double div = dudx + dvdy;
                const double txx = (2.0 * dudx - (2.0 / 3.0) * div) * g.iRe;
                const double tyy = (2.0 * dvdy - (2.0 / 3.0) * div) * g.iRe;
                const double txy = (dudy + dvdx) * g.iRe;
                const double2 uv = s_uv[sF];
                const double u = uv.x, v = uv.y;
                const double Vx3 = u * txx + v * txy + g.kT * dTdx;
                const double Vy3 = u * txy + v * tyy + g.kT * dTdy;
                if (!fast && is_sat(code)) {
                    // park the viscous fluxes for stage O's SAT term
                    const unsigned p = (unsigned)xl + un0 * (unsigned)Fl;
                    satv[p] = txx;
                    satv[uN + p] = txy;
                    satv[2 * uN + p] = Vx3;
                    satv[3 * uN + p] = txy;
                    satv[4 * uN + p] = tyy;
                    satv[5 * uN + p] = Vy3;
                }
                const double r = r3;
                const double p = r * s_T[sF] * g.igamma;
                const double E = p * g.igm1 + 0.5 * r * (u * u + v * v);
                const double Ix[4] = {r * u, r * u * u + p - txx, r * u * v - txy, (E + p) * u - Vx3};
                const double Iy[4] = {r * v, r * u * v - txy, r * v * v + p - tyy, (E + p) * v - Vy3};
                double fx[4], fy[4];
                if (CART) {
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        fx[c] = m.cM[0] * Ix[c];
                        fy[c] = m.cM[1] * Iy[c];
                    }
                } else {
                    const double Mxx = mfn[1], Mxy = mfn[2], Myx = mfn[3], Myy = mfn[4];
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        fx[c] = Mxx * Ix[c] + Mxy * Iy[c];
                        fy[c] = Myx * Ix[c] + Myy * Iy[c];
                    }
                }
                const int xs = (F & (RFX - 1)) * 2 * MT + t;
                s_fx[xs] = make_double2(fx[0], fx[1]);
                s_fx[xs + MT] = make_double2(fx[2], fx[3]);
                const int ys = (F & (RFY - 1)) * 2 * MT + t;
                s_fy[ys] = make_double2(fy[0], fy[1]);
                s_fy[ys + MT] = make_double2(fy[2], fy[3]);
            }
        }
        r3 = r2;
        r2 = r1;
        r1 = rL;
        if (more) load_F(k + 1);

        // ---- stage O: divergence, SAT, epilogue of row O
        if (O >= ja) {
            const bool act = ol;
            const unsigned code = act ? con : 0u;
            const bool fast = __all_sync(0xffffffffu, !act || code == INTINT);
            if (act) {
                const unsigned p = (unsigned)x + un0 * (unsigned)O;
                double R[4] = {0, 0, 0, 0};
                if (fast || code) {
                    int cx = CLS_INT, cy = CLS_INT;
                    if (!fast) {
                        cx = code & 15;
                        cy = (code >> 4) & 15;
                    }
                    const int xs = (O & (RFX - 1)) * 2 * MT + t;
                    double2 x01, x23, y01, y23;
                    if (cx == CLS_INT) {
                        x01 = d_int2(s_fx, xs, 1);
                        x23 = d_int2(s_fx, xs + MT, 1);
                    } else {
                        x01 = d_gen2(s_fx, xs, 1, cx);
                        x23 = d_gen2(s_fx, xs + MT, 1, cx);
                    }
                    if (cy == CLS_INT) {
                        const int a1 = ((O + 1) & (RFY - 1)) * 2 * MT + t, b1 = ((O - 1) & (RFY - 1)) * 2 * MT + t;
                        const int a2 = ((O + 2) & (RFY - 1)) * 2 * MT + t, b2 = ((O - 2) & (RFY - 1)) * 2 * MT + t;
                        const double2 A1 = s_fy[a1], B1 = s_fy[b1], A2 = s_fy[a2], B2 = s_fy[b2];
                        const double2 A3 = s_fy[a1 + MT], B3 = s_fy[b1 + MT], A4 = s_fy[a2 + MT], B4 = s_fy[b2 + MT];
                        y01 = make_double2(C1 * (A1.x - B1.x) - C2 * (A2.x - B2.x),
                                           C1 * (A1.y - B1.y) - C2 * (A2.y - B2.y));
                        y23 = make_double2(C1 * (A3.x - B3.x) - C2 * (A4.x - B4.x),
                                           C1 * (A3.y - B3.y) - C2 * (A4.y - B4.y));
                    } else {
                        y01 = ring_gen<double2>(s_fy, O + 8 * RFY, t, cy, 2 * MT, RFY);
                        y23 = ring_gen<double2>(s_fy + MT, O + 8 * RFY, t, cy, 2 * MT, RFY);
                    }
                    const double Jp = CART ? m.cJ : jon;
                    R[0] = -Jp * (x01.x + y01.x);
                    R[1] = -Jp * (x01.y + y01.y);
                    R[2] = -Jp * (x23.x + y23.x);
                    R[3] = -Jp * (x23.y + y23.y);
                    if (!fast && is_sat(code)) {
                        const double Vx[3] = {satv[p], satv[uN + p], satv[2 * uN + p]};
                        const double Vy[3] = {satv[3 * uN + p], satv[4 * uN + p], satv[5 * uN + p]};
                        sat2d_m<CART>(m, Q, g, Vx, Vy, code, p, x, O, Jp, R);
                    }
                }
                if (ep.r_out) {
#pragma unroll
                    for (int c = 0; c < 4; ++c) ep.r_out[c * uN + p] = R[c];
                }
                if (NS >= 0) {
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        double y = en[0][c];
#pragma unroll
                        for (int s = 0; s < NS; ++s) y += ep.csrc[s] * en[1 + s][c];
                        ep.y_out[c * uN + p] = y + ep.c_new * R[c];
                    }
                }
            }
        }
        if (more) load_O(k + 1);
    }
    if (ep.trace) {
        __syncthreads();
        if (threadIdx.x == 0) trace_rec(ep.trace, ep.trace_tag, t0);
    }
}

// ------------------------------------------------------------------------------------
// host side
// ------------------------------------------------------------------------------------
static int march_env(const char* name, int dflt) {
    const char* e = getenv(name);
    return e ? atoi(e) : dflt;
}

bool rhs2d_march_wanted(const int* n, int viscous) {
    // read per call (host, create time): tests switch kernels between contexts
    // default off: measured slower than the tile kernel on config 3
    const int mode = march_env("MRAB_MARCH", 0);
    const int minpts = march_env("MRAB_MARCH_MIN", 150000);
    if (!viscous || mode == 0) return false;
    return mode == 2 || (int64_t)n[0] * n[1] >= minpts;
}

static MarchGrid march_grid(const int* n) {
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    MarchGrid mg;
    mg.ns = (n[0] + MW - 1) / MW;
    mg.w = (n[0] + mg.ns - 1) / mg.ns;
    const int target = march_env("MRAB_MARCH_CTAS", 3) * nsm;
    int L = march_env("MRAB_MARCH_L", 0);
    if (L <= 0) {
        const int chunks = std::max(1, (target + mg.ns - 1) / mg.ns);
        L = std::max(1, (n[1] + chunks - 1) / chunks);
    }
    mg.L = L;
    return mg;
}

template <bool CART, int NS>
static void launch_m(const DevMesh& m, const double* Q, const Gas& g, const Epilogue& ep, cudaStream_t st) {
    static bool init = false;
    if (!init) {
        cudaFuncSetAttribute(k_rhs2d_m<CART, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)MBYTES);
        init = true;
    }
    const MarchGrid mg = march_grid(m.n);
    const int nb = mg.ns * ((m.n[1] + mg.L - 1) / mg.L);
    k_rhs2d_m<CART, NS><<<nb, MT, MBYTES, st>>>(m, Q, g, ep, mg, m.satv);
}

bool launch_rhs2d_march(const DevMesh& m, const double* Q, const Gas& g, const Epilogue& ep, cudaStream_t st) {
    if (!m.satv || ep.tiles || !g.viscous) return false;
    const int ns = ep.y_out ? ep.nsrc : -1;
    if (ns > 3) return false;
#define MRAB_M(NSV)                                                  \
    case NSV:                                                        \
        if (m.cart) launch_m<true, NSV>(m, Q, g, ep, st);            \
        else launch_m<false, NSV>(m, Q, g, ep, st);                  \
        break;
    switch (ns) {
        MRAB_M(-1)
        MRAB_M(0)
        MRAB_M(1)
        MRAB_M(2)
        MRAB_M(3)
        default: return false;
    }
#undef MRAB_M
    return true;
}

}  // namespace mrab
