// 2-D fused SBP-SAT RHS, y-streaming variant (sm_100a, fp64).
//
// Same arithmetic as k_rhs2d (kernels2d.cu).  A CTA walks a strip of NTY
// vertically adjacent 32 x 16 tiles of one column: after the first tile, the 12 halo rows of
// primitives and the 6 rows of contravariant fluxes it shares with the next tile are moved
// to the top of the shared buffers instead of being reloaded / recomputed, so per output
// point the kernel loads 1.375 (not 2.4) halo'd state points and forms 1.19 (not 1.63)
// flux points.
#include <cuda_runtime.h>

#include "rhs2d_common.cuh"

namespace mrab {

namespace {

constexpr int TX = 32, TY = 16, NTH = 256;
constexpr int G3 = 3;
using namespace k2d;

template <bool VISC>
struct GeoS {
    static constexpr int H = VISC ? 6 : 3;
    static constexpr int AX = TX + 2 * H, AY = TY + 2 * H;
    static constexpr int FX = TX + 2 * G3, FY = TY + 2 * G3;
    static constexpr int NA = AX * AY, NF = FX * FY;
    static constexpr int KEEPA = 2 * H;          // prim rows shared with the next tile
    static constexpr int KEEPF = 2 * G3;         // flux rows shared with the next tile
    static constexpr size_t bytes = 16 * (size_t)NA + 64 * (size_t)NF + 16 * (size_t)NA + 2 * (size_t)NA;
};

template <int NS>
__device__ __forceinline__ double epi_sum_s(const Epilogue& ep, unsigned uN, unsigned up, int c) {
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

template <bool VISC, bool CART>
__global__ void __launch_bounds__(NTH, 2) k_rhs2d_s(DevMesh m, const double* __restrict__ Q,
                                                   Gas g, Epilogue ep, int nty_strip) {
    using GG = GeoS<VISC>;
    constexpr int H = GG::H, AX = GG::AX, AY = GG::AY, FX = GG::FX, FY = GG::FY;
    constexpr int NA = GG::NA, NF = GG::NF, KEEPA = GG::KEEPA, KEEPF = GG::KEEPF;
    extern __shared__ __align__(16) double smem[];
    double2* sh_uv = reinterpret_cast<double2*>(smem);
    double2* fh = sh_uv + NA;                       // [4][NF]
    double* sh_r = reinterpret_cast<double*>(fh + 4 * NF);
    double* sh_T = sh_r + NA;
    uint16_t* sh_c = reinterpret_cast<uint16_t*>(sh_T + NA);

    const int n0 = m.n[0], n1 = m.n[1];
    const int64_t N = m.npts;
    const unsigned uN = (unsigned)N;
    const int nty = (n1 + TY - 1) / TY;
    const int bx = blockIdx.x;
    const int by0 = blockIdx.y * nty_strip;
    const int by1 = min(by0 + nty_strip, nty);
    const int i0 = bx * TX;
    const int tid = threadIdx.x;
    const int ns = ep.y_out ? ep.nsrc : -1;

    for (int by = by0; by < by1; ++by) {
        const int j0 = by * TY;
        const bool first = by == by0;
        // ---- rows carried over from the previous tile --------------------------------
        if (!first) {
            for (int t = tid; t < KEEPA * AX; t += NTH) {
                const int src = t + TY * AX;
                sh_c[t] = sh_c[src];
                sh_r[t] = sh_r[src];
                sh_uv[t] = sh_uv[src];
                sh_T[t] = sh_T[src];
            }
            for (int t = tid; t < KEEPF * FX; t += NTH) {
                const int src = t + TY * FX;
#pragma unroll
                for (int c = 0; c < 4; ++c) fh[c * NF + t] = fh[c * NF + src];
            }
        }
        // ---- phase A: primitives of the new rows -------------------------------------
        const int rowA0 = first ? 0 : KEEPA;
        const int nA = (AY - rowA0) * AX;
        constexpr int KA = (NA + NTH - 1) / NTH;
        {
            double ld[KA][4];
            unsigned cd[KA];
#pragma unroll
            for (int k = 0; k < KA; ++k) {
                const int t = tid + k * NTH;
                cd[k] = 0;
                ld[k][0] = 1.0;
                ld[k][1] = ld[k][2] = ld[k][3] = 0.0;
                if (t < nA) {
                    const int bb = t / AX, a = t - bb * AX;
                    int gi = i0 - H + a, gj = j0 - H + rowA0 + bb;
                    bool ok = true;
                    if (gi < 0 || gi >= n0) {
                        if (m.periodic[0]) gi = gi < 0 ? gi + n0 : gi - n0; else ok = false;
                    }
                    if (gj < 0 || gj >= n1) {
                        if (m.periodic[1]) gj = gj < 0 ? gj + n1 : gj - n1; else ok = false;
                    }
                    if (ok) {
                        const unsigned q = (unsigned)gi + (unsigned)n0 * (unsigned)gj;
                        cd[k] = m.cls[q];
                        ld[k][0] = __ldg(Q + q);
                        ld[k][1] = __ldg(Q + (uN + q));
                        ld[k][2] = __ldg(Q + (2 * uN + q));
                        ld[k][3] = __ldg(Q + (3 * uN + q));
                    }
                }
            }
            if (!first) __syncthreads();    // carried rows are in place before new rows land
#pragma unroll
            for (int k = 0; k < KA; ++k) {
                const int t = tid + k * NTH;
                if (t >= nA) break;
                const int o = rowA0 * AX + t;
                const double r = ld[k][0];
                const double ir = rcp64(r);
                const double u = ld[k][1] * ir;
                const double v = ld[k][2] * ir;
                sh_c[o] = (uint16_t)cd[k];
                sh_r[o] = r;
                sh_uv[o] = make_double2(u, v);
                sh_T[o] = g.gamma * g.gm1 * (ld[k][3] - 0.5 * (ld[k][1] * u + ld[k][2] * v)) * ir;
            }
        }
        __syncthreads();
        // tile-uniform fast path: every flux point (tile + 3) interior in both directions
        int allint = 1;
        for (int t = tid; t < NF; t += NTH) {
            const int b = t / FX, a = t - b * FX;
            allint &= sh_c[(b + H - G3) * AX + (a + H - G3)] == (unsigned)(CLS_INT | (CLS_INT << 4));
        }
        const int fast = __syncthreads_and(allint);

        // ---- phase B: contravariant fluxes of the new flux rows -----------------------
        const int rowF0 = first ? 0 : KEEPF;
        const int nFB = (FY - rowF0) * FX;
        for (int tt = tid; tt < nFB; tt += NTH) {
            const int t = rowF0 * FX + tt;
            const int b = t / FX, a = t - b * FX;
            const int s = (b + H - G3) * AX + (a + H - G3);
            const unsigned code = sh_c[s];
            double fx[4] = {0, 0, 0, 0}, fy[4] = {0, 0, 0, 0};
            if (fast || code) {
                const double r = sh_r[s];
                const double2 uv = sh_uv[s];
                const double u = uv.x, v = uv.y;
                const double p = r * sh_T[s] * g.igamma;
                const double E = p * g.igm1 + 0.5 * r * (u * u + v * v);
                double Ix[4] = {r * u, r * u * u + p, r * u * v, (E + p) * u};
                double Iy[4] = {r * v, r * u * v, r * v * v + p, (E + p) * v};
                unsigned q = 0;
                if (!CART) {
                    int gi = i0 - G3 + a, gj = j0 - G3 + b;
                    if (gi < 0) gi += n0; else if (gi >= n0) gi -= n0;
                    if (gj < 0) gj += n1; else if (gj >= n1) gj -= n1;
                    q = (unsigned)gi + (unsigned)n0 * (unsigned)gj;
                }
                if (VISC) {
                    double Vx[4], Vy[4];
                    if (fast) visc_at_int<CART, AX>(sh_uv, sh_T, s, m, q, g, Vx, Vy);
                    else visc_at<CART, AX>(sh_uv, sh_T, s, code, m, q, g, Vx, Vy);
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
                    const double Mxx = __ldg(m.M + q), Mxy = __ldg(m.M + (uN + q));
                    const double Myx = __ldg(m.M + (2 * uN + q)), Myy = __ldg(m.M + (3 * uN + q));
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

        // ---- phase C: divergence, SAT, epilogue -----------------------------------------
        for (int t = tid; t < TX * TY; t += NTH) {
            const int a = t % TX, b = t / TX;
            const int gi = i0 + a, gj = j0 + b;
            if (gi >= n0 || gj >= n1) continue;
            const unsigned up = (unsigned)gi + (unsigned)n0 * (unsigned)gj;
            const int s = (b + H) * AX + (a + H);
            const int f = (b + G3) * FX + (a + G3);
            double yb[4];
            if (ns == 2) {
                yb[0] = epi_sum_s<2>(ep, uN, up, 0); yb[1] = epi_sum_s<2>(ep, uN, up, 1);
                yb[2] = epi_sum_s<2>(ep, uN, up, 2); yb[3] = epi_sum_s<2>(ep, uN, up, 3);
            } else if (ns == 3) {
                yb[0] = epi_sum_s<3>(ep, uN, up, 0); yb[1] = epi_sum_s<3>(ep, uN, up, 1);
                yb[2] = epi_sum_s<3>(ep, uN, up, 2); yb[3] = epi_sum_s<3>(ep, uN, up, 3);
            } else if (ns >= 0) {
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    double y = __ldg(ep.base + (c * uN + up));
                    for (int k = 0; k < ns; ++k) y += ep.csrc[k] * __ldg(ep.src[k] + (c * uN + up));
                    yb[c] = y;
                }
            }
            double R[4] = {0, 0, 0, 0};
            const unsigned code = sh_c[s];
            if (fast || code) {
                const int cx = code & 15, cy = (code >> 4) & 15;
                double2 x01, x23, y01, y23;
                if (fast || cx == CLS_INT) {
                    x01 = d_int2(fh, f, 1);
                    x23 = d_int2(fh + NF, f, 1);
                } else {
                    x01 = d_gen2(fh, f, 1, cx);
                    x23 = d_gen2(fh + NF, f, 1, cx);
                }
                if (fast || cy == CLS_INT) {
                    y01 = d_int2(fh + 2 * NF, f, FX);
                    y23 = d_int2(fh + 3 * NF, f, FX);
                } else {
                    y01 = d_gen2(fh + 2 * NF, f, FX, cy);
                    y23 = d_gen2(fh + 3 * NF, f, FX, cy);
                }
                const double Jp = CART ? m.cJ : __ldg(m.J + up);
                R[0] = -Jp * (x01.x + y01.x);
                R[1] = -Jp * (x01.y + y01.y);
                R[2] = -Jp * (x23.x + y23.x);
                R[3] = -Jp * (x23.y + y23.y);
                if (!fast && (cx == CLS_L0 || cx == CLS_R0 || cy == CLS_L0 || cy == CLS_R0))
                    sat2d<VISC, CART, AX>(m, Q, g, sh_uv, sh_T, s, code, (int64_t)up, gi, gj, Jp, R);
            }
            if (ep.r_out) {
#pragma unroll
                for (int c = 0; c < 4; ++c) ep.r_out[c * uN + up] = R[c];
            }
            if (ns >= 0) {
#pragma unroll
                for (int c = 0; c < 4; ++c) ep.y_out[c * uN + up] = yb[c] + ep.c_new * R[c];
            }
        }
        __syncthreads();   // the next tile overwrites the shared buffers
    }
}

template <bool VISC, bool CART>
static void launch_s(const DevMesh& m, const double* Q, const Gas& g, const Epilogue& ep,
                     int strip, cudaStream_t st) {
    static bool init = false;
    const size_t bytes = GeoS<VISC>::bytes;
    if (!init) {
        cudaFuncSetAttribute(k_rhs2d_s<VISC, CART>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        init = true;
    }
    const int ntx = (m.n[0] + TX - 1) / TX, nty = (m.n[1] + TY - 1) / TY;
    dim3 grid(ntx, (nty + strip - 1) / strip);
    k_rhs2d_s<VISC, CART><<<grid, NTH, bytes, st>>>(m, Q, g, ep, strip);
}

// strip length giving at most ~2 CTAs per SM in one wave; 0 = streaming not worthwhile
int rhs2d_stream_strip(const DevMesh& m) {
    static int nsm = 0;
    static int mode = -1, force = 0;
    if (mode < 0) {
        const char* e = getenv("MRAB_STREAM");
        mode = e ? atoi(e) : 0;   // opt-in: measured slower
        const char* f = getenv("MRAB_STREAM_STRIP");
        force = f ? atoi(f) : 0;
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    }
    if (mode == 0) return 0;
    if (force > 0) return force;
    const int ntx = (m.n[0] + TX - 1) / TX, nty = (m.n[1] + TY - 1) / TY;
    const int slots = 2 * nsm;
    // shortest strip whose CTAs all fit in one wave (a second, partial wave would double
    // the time: every CTA walks `strip` tiles)
    if (ntx * nty <= slots) return 0;
    int strip = 2;
    while (ntx * ((nty + strip - 1) / strip) > slots && strip < nty) ++strip;
    return strip;
}

bool launch_rhs2d_stream(const DevMesh& m, const double* Q, const Gas& g, const Epilogue& ep,
                         cudaStream_t st) {
    if (ep.tiles || ep.has_prio) return false;
    const int strip = rhs2d_stream_strip(m);
    if (strip < 2) return false;
    if (g.viscous) {
        if (m.cart) launch_s<true, true>(m, Q, g, ep, strip, st);
        else launch_s<true, false>(m, Q, g, ep, strip, st);
    } else {
        if (m.cart) launch_s<false, true>(m, Q, g, ep, strip, st);
        else launch_s<false, false>(m, Q, g, ep, strip, st);
    }
    return true;
}

}  // namespace mrab
