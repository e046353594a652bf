// 2-D fused SBP-SAT RHS, persistent and TMA-pipelined (sm_100a, fp64).
//
// Same arithmetic as k_rhs2d (kernels2d.cu) but organised for memory/compute
// overlap on B200: one CTA of 512 threads per SM walks its tiles (32 x 8 points) in a
// persistent loop; while tile k is computed from shared memory, one elected thread has the
// Tensor Memory Accelerator (cp.async.bulk.tensor, mbarrier completion) bring tile k+1's
// halo'd state box [4][AY][AX], its class codes, and the epilogue operands (history ring
// slots, RK stage bases) into the other half of a double buffer.  Global memory is then
// touched only by TMA loads and by the final stores of the RHS and the new state.
// Tiles whose halo wraps a periodic seam are filled by the threads themselves.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>

#include "rhs2d_common.cuh"

namespace mrab {

namespace {

constexpr int TX = 32, TY = 8, NTH = 512;
constexpr int G3 = 3;
constexpr int NEPI = 4;                    // epilogue arrays prefetched per tile
constexpr double kP0 = 17.0 / 48.0;
using namespace k2d;

template <bool VISC>
struct GeoT {
    // TMA needs the innermost box start to be 16-byte aligned: halo 6 (viscous) / 4 (Euler;
    // 3 would do) keeps (i0 - H) * 8 bytes aligned; the uint16 class box starts PADC earlier
    static constexpr int H = VISC ? 6 : 4;
    static constexpr int AX = TX + 2 * H, AY = TY + 2 * H;
    static constexpr int PADC = (8 - H % 8) % 8;
    static constexpr int AXC = ((AX + PADC + 7) / 8) * 8;      // class-code row (16-byte multiple)
    static constexpr int FX = TX + 2 * G3, FY = TY + 2 * G3;
    static constexpr int NA = AX * AY, NF = FX * FY;
    static constexpr int QB = 4 * NA * 8;                      // raw state box bytes
    static constexpr int CB = AY * AXC * 2;                    // class box bytes
    static constexpr int EB = 4 * TX * TY * 8;                 // one epilogue array box
    static constexpr int r128(int x) { return (x + 127) / 128 * 128; }
    static constexpr int OFF_Q = 0;
    static constexpr int OFF_C = OFF_Q + 2 * r128(QB);
    static constexpr int OFF_E = OFF_C + 2 * r128(CB);
    static constexpr int OFF_UV = OFF_E + 2 * NEPI * EB;
    static constexpr int OFF_R = OFF_UV + r128(NA * 16);
    static constexpr int OFF_T = OFF_R + r128(NA * 8);
    static constexpr int OFF_CL = OFF_T + r128(NA * 8);
    static constexpr int OFF_F = OFF_CL + r128(NA * 2);
    static constexpr int OFF_BAR = OFF_F + r128(NF * 64);
    static constexpr int BYTES = OFF_BAR + 128;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(tx)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                     uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma2(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

}  // namespace

struct TmaMaps {
    CUtensorMap q;             // state [4][n1][n0], box {AX, AY, 4}
    CUtensorMap cls;           // class codes [n1][n0] (uint16), box {AXC, AY}
    CUtensorMap e[NEPI];       // epilogue arrays [4][n1][n0], box {TX, TY, 4}
    int ne;                    // epilogue arrays in use
    int base_is_q;             // epilogue base == the RHS input state (MRAB step)
};

template <bool VISC, bool CART>
__global__ void __launch_bounds__(NTH, 1)
    k_rhs2d_tma(const __grid_constant__ TmaMaps tm, DevMesh m, const double* __restrict__ Q, Gas g,
                Epilogue ep) {
    using GG = GeoT<VISC>;
    constexpr int H = GG::H, AX = GG::AX, AXC = GG::AXC, FX = GG::FX, PADC = GG::PADC;
    constexpr int NA = GG::NA, NF = GG::NF;
    extern __shared__ __align__(128) unsigned char sm[];
    double* rawQ[2] = {reinterpret_cast<double*>(sm + GG::OFF_Q),
                       reinterpret_cast<double*>(sm + GG::OFF_Q + GG::r128(GG::QB))};
    uint16_t* rawC[2] = {reinterpret_cast<uint16_t*>(sm + GG::OFF_C),
                         reinterpret_cast<uint16_t*>(sm + GG::OFF_C + GG::r128(GG::CB))};
    double* epi[2] = {reinterpret_cast<double*>(sm + GG::OFF_E),
                      reinterpret_cast<double*>(sm + GG::OFF_E + NEPI * GG::EB)};
    double2* sh_uv = reinterpret_cast<double2*>(sm + GG::OFF_UV);
    double* sh_r = reinterpret_cast<double*>(sm + GG::OFF_R);
    double* sh_T = reinterpret_cast<double*>(sm + GG::OFF_T);
    uint16_t* sh_c = reinterpret_cast<uint16_t*>(sm + GG::OFF_CL);
    double2* fh = reinterpret_cast<double2*>(sm + GG::OFF_F);
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + GG::OFF_BAR);

    const int n0 = m.n[0], n1 = m.n[1];
    const int64_t N = m.npts;
    const int ntx = (n0 + TX - 1) / TX, nty = (n1 + TY - 1) / TY;
    const int ntiles = ep.tiles ? ep.ntiles : ntx * nty;
    const int tid = threadIdx.x;
    const uint32_t tx_bytes = GG::QB + GG::CB + tm.ne * GG::EB;

    auto tile_of = [&](int k) { return ep.tiles ? ep.tiles[k] : k; };
    auto manual = [&](int tl) {
        const int by = tl / ntx, bx = tl - by * ntx;
        const int i0 = bx * TX, j0 = by * TY;
        const bool wx = m.periodic[0] && (i0 - H < 0 || i0 + TX + H > n0);
        const bool wy = m.periodic[1] && (j0 - H < 0 || j0 + TY + H > n1);
        return wx || wy;
    };
    auto issue = [&](int buf, int tl) {
        const int by = tl / ntx, bx = tl - by * ntx;
        const int i0 = bx * TX, j0 = by * TY;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&bar[buf], tx_bytes);
        tma3(rawQ[buf], &tm.q, i0 - H, j0 - H, 0, &bar[buf]);
        tma2(rawC[buf], &tm.cls, i0 - H - PADC, j0 - H, &bar[buf]);
        for (int e = 0; e < tm.ne; ++e) tma3(epi[buf] + e * (GG::EB / 8), &tm.e[e], i0, j0, 0, &bar[buf]);
    };

    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t ph0 = 0, ph1 = 0;
    int k = blockIdx.x;
    if (tid == 0 && k < ntiles && !manual(tile_of(k))) issue(0, tile_of(k));

    for (int it = 0; k < ntiles; ++it, k += gridDim.x) {
        const int buf = it & 1;
        const int tl = tile_of(k);
        const int by = tl / ntx, bx = tl - by * ntx;
        const int i0 = bx * TX, j0 = by * TY;
        if (!manual(tl)) {
            mbar_wait(&bar[buf], buf ? ph1 : ph0);
            if (buf) ph1 ^= 1; else ph0 ^= 1;
        } else {
            // halo wraps a periodic seam: the threads gather it themselves
            for (int t = tid; t < NA; t += NTH) {
                const int b = t / AX, a = t - b * AX;
                int gi = i0 - H + a, gj = j0 - H + b;
                bool ok = true;
                if (gi < 0 || gi >= n0) {
                    if (m.periodic[0]) gi = gi < 0 ? gi + n0 : gi - n0; else ok = false;
                }
                if (gj < 0 || gj >= n1) {
                    if (m.periodic[1]) gj = gj < 0 ? gj + n1 : gj - n1; else ok = false;
                }
                const int64_t q = gi + (int64_t)n0 * gj;
#pragma unroll
                for (int c = 0; c < 4; ++c) rawQ[buf][c * NA + t] = ok ? __ldg(Q + c * N + q) : 0.0;
                rawC[buf][b * AXC + a + PADC] = ok ? m.cls[q] : (uint16_t)0;
            }
            for (int t = tid; ep.y_out && t < TX * TY; t += NTH) {
                const int b = t / TX, a = t - b * TX;
                const int gi = i0 + a, gj = j0 + b;
                const bool ok = gi < n0 && gj < n1;
                const int64_t q = gi + (int64_t)n0 * gj;
                int e = 0;
                if (!tm.base_is_q) {
#pragma unroll
                    for (int c = 0; c < 4; ++c) epi[buf][c * TX * TY + t] = ok ? __ldg(ep.base + c * N + q) : 0.0;
                    e = 1;
                }
                for (int s = 0; s < ep.nsrc && e < NEPI; ++s, ++e)
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        epi[buf][e * (GG::EB / 8) + c * TX * TY + t] = ok ? __ldg(ep.src[s] + c * N + q) : 0.0;
            }
            __syncthreads();
        }
        // prefetch the next tile into the other buffer (read for the last time in it-1)
        {
            const int kn = k + gridDim.x;
            if (tid == 0 && kn < ntiles && !manual(tile_of(kn))) issue(buf ^ 1, tile_of(kn));
        }
        const double* rq = rawQ[buf];
        const uint16_t* rc = rawC[buf];
        const double* ev = epi[buf];

        // ---- phase A': primitives from the staged box --------------------------------------
        for (int t = tid; t < NA; t += NTH) {
            const int b = t / AX, a = t - b * AX;
            const unsigned code = rc[b * AXC + a + PADC];
            double r = 1.0, u = 0.0, v = 0.0, T = 0.0;
            if (code) {
                r = rq[t];
                const double mu = rq[NA + t], mv = rq[2 * NA + t], E = rq[3 * NA + t];
                const double ir = rcp64(r);
                u = mu * ir;
                v = mv * ir;
                T = g.gamma * g.gm1 * (E - 0.5 * (mu * u + mv * v)) * ir;
            }
            sh_c[t] = (uint16_t)code;
            sh_r[t] = r;
            sh_uv[t] = make_double2(u, v);
            sh_T[t] = T;
        }
        __syncthreads();

        // ---- phase B: contravariant fluxes at tile + 3 ---------------------------------
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
                int64_t q = 0;
                if (!CART) {
                    int gi = i0 - G3 + a, gj = j0 - G3 + b;
                    if (gi < 0) gi += n0; else if (gi >= n0) gi -= n0;
                    if (gj < 0) gj += n1; else if (gj >= n1) gj -= n1;
                    q = gi + (int64_t)n0 * gj;
                }
                if (VISC) {
                    double Vx[4], Vy[4];
                    visc_at<CART, AX>(sh_uv, sh_T, s, code, m, q, g, Vx, Vy);
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
                    const double Mxx = __ldg(m.M + q), Mxy = __ldg(m.M + N + q);
                    const double Myx = __ldg(m.M + 2 * N + q), Myy = __ldg(m.M + 3 * N + q);
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

        // ---- phase C: divergence, SAT, epilogue ----------------------------------------
        for (int t = tid; t < TX * TY; t += NTH) {
            const int b = t / TX, a = t - b * TX;
            const int gi = i0 + a, gj = j0 + b;
            if (gi >= n0 || gj >= n1) continue;
            const int64_t p = gi + (int64_t)n0 * gj;
            const int s = (b + H) * AX + (a + H);
            const int f = (b + G3) * FX + (a + G3);
            const unsigned code = sh_c[s];
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
                const double Jp = CART ? m.cJ : __ldg(m.J + p);
                R[0] = -Jp * (x01.x + y01.x);
                R[1] = -Jp * (x01.y + y01.y);
                R[2] = -Jp * (x23.x + y23.x);
                R[3] = -Jp * (x23.y + y23.y);
                if (cx == CLS_L0 || cx == CLS_R0 || cy == CLS_L0 || cy == CLS_R0) {
                    double q[4];
#pragma unroll
                    for (int c = 0; c < 4; ++c) q[c] = rq[c * NA + s];
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
                    for (int kk = 0; kk < 2; ++kk) {
                        const int cl = kk == 0 ? cx : cy;
                        if (cl != CLS_L0 && cl != CLS_R0) continue;
                        const int sidx = (cl == CLS_L0) ? 0 : 1;
                        const double side = (cl == CLS_L0) ? 1.0 : -1.0;
                        const bool at_face = !m.periodic[kk] && (sidx == 0 ? idx[kk] == 0 : idx[kk] == m.n[kk] - 1);
                        const int typ = at_face ? m.face_bc[kk][sidx] : MRAB_BC_OVERSET;
                        double nv[2];
                        if (CART) {
                            nv[0] = kk == 0 ? m.cJ * m.cM[0] : 0.0;
                            nv[1] = kk == 1 ? m.cJ * m.cM[1] : 0.0;
                        } else {
                            nv[0] = Jp * __ldg(m.M + (2 * kk) * N + p);
                            nv[1] = Jp * __ldg(m.M + (2 * kk + 1) * N + p);
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
                        for (int c = 0; c < 4; ++c) R[c] -= (0.5 * kd[c] + sig1 * dq[c]) / kP0;
                        if (VISC && typ != MRAB_BC_WALL) {
#pragma unroll
                            for (int j = 0; j < 3; ++j) {
                                const double fk = nv[0] * Vx[1 + j] + nv[1] * Vy[1 + j];
                                double fhv = 0.0;
                                if (typ == MRAB_BC_OVERSET) fhv = nv[0] * fvi[j] + nv[1] * fvi[3 + j];
                                R[1 + j] += 0.5 * side * (fk - fhv) / kP0;
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
                // epilogue operands are in shared memory (staged by TMA with the tile)
                int e = 0;
                double yb[4];
                if (tm.base_is_q) {
#pragma unroll
                    for (int c = 0; c < 4; ++c) yb[c] = rq[c * NA + s];
                } else {
#pragma unroll
                    for (int c = 0; c < 4; ++c) yb[c] = ev[c * TX * TY + t];
                    e = 1;
                }
                for (int sI = 0; sI < ep.nsrc; ++sI, ++e) {
                    const double w = ep.csrc[sI];
#pragma unroll
                    for (int c = 0; c < 4; ++c) yb[c] += w * ev[e * (GG::EB / 8) + c * TX * TY + t];
                }
#pragma unroll
                for (int c = 0; c < 4; ++c) ep.y_out[c * N + p] = yb[c] + ep.c_new * R[c];
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------------------
// host side: tensor maps (driver entry point) and dispatch
// ---------------------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled encode_fn() {
    static PFN_cuTensorMapEncodeTiled fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled)p;
    }
    return fn;
}

static bool make_map3(CUtensorMap* map, const double* ptr, int n0, int n1, int b0, int b1) {
    PFN_cuTensorMapEncodeTiled fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[3] = {(cuuint64_t)n0, (cuuint64_t)n1, 4};
    cuuint64_t strides[2] = {(cuuint64_t)n0 * 8, (cuuint64_t)n0 * n1 * 8};
    cuuint32_t box[3] = {(cuuint32_t)b0, (cuuint32_t)b1, 4};
    cuuint32_t es[3] = {1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)ptr, dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
              CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static bool make_map_cls(CUtensorMap* map, const uint16_t* ptr, int n0, int n1, int b0, int b1) {
    PFN_cuTensorMapEncodeTiled fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)n0, (cuuint64_t)n1};
    cuuint64_t strides[1] = {(cuuint64_t)n0 * 2};
    cuuint32_t box[2] = {(cuuint32_t)b0, (cuuint32_t)b1};
    cuuint32_t es[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, (void*)ptr, dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
              CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <bool VISC, bool CART>
static void launch_tma_t(const TmaMaps& tm, const DevMesh& m, const double* Q, const Gas& g,
                         const Epilogue& ep, cudaStream_t st) {
    using GG = GeoT<VISC>;
    static bool init = false;
    static int nsm = 148;
    if (!init) {
        cudaFuncSetAttribute(k_rhs2d_tma<VISC, CART>, cudaFuncAttributeMaxDynamicSharedMemorySize, GG::BYTES);
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        init = true;
    }
    const int ntx = (m.n[0] + TX - 1) / TX, nty = (m.n[1] + TY - 1) / TY;
    const int ntiles = ep.tiles ? ep.ntiles : ntx * nty;
    if (ntiles <= 0) return;
    const int grid = ntiles < nsm ? ntiles : nsm;
    k_rhs2d_tma<VISC, CART><<<grid, NTH, GG::BYTES, st>>>(tm, m, Q, g, ep);
}

bool rhs2d_tma_possible(const DevMesh& m, const Epilogue& ep, const double* Q) {
    static int enabled = -1;
    if (enabled < 0) {
        const char* e = getenv("MRAB_TMA");
        // measured slower than k_rhs2d on config 3 (one 16-warp CTA per SM exposes every
        // phase barrier); kept behind MRAB_TMA=1 for further work
        enabled = e && e[0] == '1';
    }
    if (!enabled || !encode_fn()) return false;
    if (m.n[0] % 8 != 0) return false;                          // 16-byte row pitch for TMA
    if (ep.tiles) return false;                                  // tile lists use k_rhs2d
    const int need = (ep.y_out ? ep.nsrc + (ep.base == Q ? 0 : 1) : 0);
    return need <= NEPI;
}

bool launch_rhs2d_tma(const DevMesh& m, const double* Q, const Gas& g, const Epilogue& ep,
                      cudaStream_t st) {
    TmaMaps tm;
    memset(&tm, 0, sizeof(tm));
    const bool visc = g.viscous != 0;
    const int H = visc ? 6 : 4;
    const int AX = TX + 2 * H, AY = TY + 2 * H;
    const int PADC = (8 - H % 8) % 8;
    const int AXC = ((AX + PADC + 7) / 8) * 8;
    if (!make_map3(&tm.q, Q, m.n[0], m.n[1], AX, AY)) return false;
    if (!make_map_cls(&tm.cls, m.cls, m.n[0], m.n[1], AXC, AY)) return false;
    tm.base_is_q = (ep.base == Q) ? 1 : 0;
    tm.ne = 0;
    if (ep.y_out) {
        if (!tm.base_is_q && !make_map3(&tm.e[tm.ne++], ep.base, m.n[0], m.n[1], TX, TY)) return false;
        for (int s = 0; s < ep.nsrc; ++s)
            if (!make_map3(&tm.e[tm.ne++], ep.src[s], m.n[0], m.n[1], TX, TY)) return false;
    }
    if (visc) {
        if (m.cart) launch_tma_t<true, true>(tm, m, Q, g, ep, st);
        else launch_tma_t<true, false>(tm, m, Q, g, ep, st);
    } else {
        if (m.cart) launch_tma_t<false, true>(tm, m, Q, g, ep, st);
        else launch_tma_t<false, false>(tm, m, Q, g, ep, st);
    }
    return true;
}

}  // namespace mrab
