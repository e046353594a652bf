// Host setup of libmrab.so: AB coefficients, segments and stencil classes, metric terms,
// overset hole cutting / donor search / Lagrange weights.  Runs once per plan (not timed).
//
// PAPER.md citations: P:343-394 (AB weights), P:205-208 + P:1526-1528 (SBP 2-4 operator),
// P:628-637 (metric terms, reading R3), P:227-252 (overset phases, reading R17).
#include <algorithm>
#include <cstdlib>
#include <array>
#include <cmath>
#include <cstring>
#include <numeric>

#include "mrab_internal.h"

namespace mrab {

static Options g_opt;

static long env_or(const char* name, long dflt) {
    const char* e = getenv(name);
    return e && e[0] ? atol(e) : dflt;
}

Options read_options() {
    Options o;
    o.overlap = (int)env_or("MRAB_OVERLAP", o.overlap);
    o.bulk_ctas = (int)env_or("MRAB_BULK_CTAS", o.bulk_ctas);
    o.lean = (int)env_or("MRAB_LEAN", o.lean);
    o.tile_flags = (int)env_or("MRAB_TILE_FLAGS", o.tile_flags);
    o.k2d = (int)env_or("MRAB_K2D", o.k2d);
    if (o.k2d < -2 || o.k2d > 4 || o.k2d == -1) o.k2d = -2;
    o.small_pts = env_or("MRAB_SMALL_PTS", o.small_pts);
    o.curv_half = (int)env_or("MRAB_CURV_HALF", o.curv_half);
    o.pf = (int)env_or("MRAB_PF", o.pf);
    o.donor_staged = (int)env_or("MRAB_DONOR_STAGED", o.donor_staged);
    o.interp_box = (int)env_or("MRAB_INTERP_BOX", o.interp_box);
    o.interp_quad = (int)env_or("MRAB_INTERP_QUAD", o.interp_quad);
    o.z3_fused = (int)env_or("MRAB_3D_FUSED", o.z3_fused);
    o.overlap3d = (int)env_or("MRAB_OVERLAP3D", o.overlap3d);
    o.div_wide = (int)env_or("MRAB_DIV_WIDE", o.div_wide);
    o.flux_wide = (int)env_or("MRAB_FLUX_WIDE", o.flux_wide);
    o.flux_sym = (int)env_or("MRAB_FLUX_SYM", o.flux_sym);
    return o;
}
const Options& opts() { return g_opt; }
void set_options(const Options& o) { g_opt = o; }


// ------------------------------------------------------------------------------------
// SBP 2-4 diagonal-norm first derivative (index space).  Rows by class code.
// ------------------------------------------------------------------------------------
struct StRow {
    int n;
    int off[6];
    double c[6];
};

static StRow g_rows[10];
static bool g_rows_init = false;

static void init_rows() {
    if (g_rows_init) return;
    // left closure rows {column, coefficient}
    const int lc[4][6] = {{0, 1, 2, 3, -1, -1}, {0, 2, -1, -1, -1, -1}, {0, 1, 3, 4, -1, -1},
                          {0, 2, 4, 5, -1, -1}};
    const double lv[4][6] = {{-24.0 / 17, 59.0 / 34, -4.0 / 17, -3.0 / 34, 0, 0},
                             {-0.5, 0.5, 0, 0, 0, 0},
                             {4.0 / 43, -59.0 / 86, 59.0 / 86, -4.0 / 43, 0, 0},
                             {3.0 / 98, -59.0 / 98, 32.0 / 49, -4.0 / 49, 0, 0}};
    StRow z{};
    for (auto& r : g_rows) r = z;
    g_rows[CLS_INT].n = 4;
    const int io[4] = {-2, -1, 1, 2};
    const double iv[4] = {1.0 / 12, -2.0 / 3, 2.0 / 3, -1.0 / 12};
    for (int t = 0; t < 4; ++t) {
        g_rows[CLS_INT].off[t] = io[t];
        g_rows[CLS_INT].c[t] = iv[t];
    }
    for (int r = 0; r < 4; ++r) {
        StRow L{}, R{};
        for (int t = 0; t < 6 && lc[r][t] >= 0; ++t) {
            L.off[L.n] = lc[r][t] - r;
            L.c[L.n] = lv[r][t];
            L.n++;
            R.off[R.n] = -(lc[r][t] - r);
            R.c[R.n] = -lv[r][t];
            R.n++;
        }
        g_rows[CLS_L0 + r] = L;
        g_rows[CLS_R0 + r] = R;
    }
    g_rows_init = true;
}

// ------------------------------------------------------------------------------------
// AB weights: alpha = V (V^T V)^-1 mu, V_ki = t_k^(i-1), mu_i = (b^i - a^i)/i  (R1)
// ------------------------------------------------------------------------------------
mrab_status ab_weights(const double* nodes, int m, int n, double a, double b, double* out,
                       std::string* msg) {
    if (m < 1 || n < 1 || !nodes || !out) {
        if (msg) *msg = "ab_weights: invalid arguments";
        return MRAB_E_INVALID;
    }
    if (m < n) {
        if (msg) *msg = "ab_weights: insufficient history (m < n)";
        return MRAB_E_INSUFFICIENT_HISTORY;
    }
    for (int i = 0; i < m; ++i)
        for (int j = i + 1; j < m; ++j)
            if (nodes[i] == nodes[j]) {
                if (msg) *msg = "ab_weights: degenerate nodes";
                return MRAB_E_DEGENERATE_NODES;
            }
    typedef long double LD;
    std::vector<LD> V((size_t)m * n);
    for (int k = 0; k < m; ++k) {
        LD p = 1;
        for (int i = 0; i < n; ++i) {
            V[(size_t)k * n + i] = p;
            p *= (LD)nodes[k];
        }
    }
    std::vector<LD> A((size_t)n * (n + 1));
    for (int i = 0; i < n; ++i) {
        for (int j = 0; j < n; ++j) {
            LD s = 0;
            for (int k = 0; k < m; ++k) s += V[(size_t)k * n + i] * V[(size_t)k * n + j];
            A[(size_t)i * (n + 1) + j] = s;
        }
        LD bp = std::pow((LD)b, (LD)(i + 1)), ap = std::pow((LD)a, (LD)(i + 1));
        A[(size_t)i * (n + 1) + n] = (bp - ap) / (LD)(i + 1);
    }
    for (int c = 0; c < n; ++c) {
        int piv = c;
        for (int r = c + 1; r < n; ++r)
            if (std::fabs(A[(size_t)r * (n + 1) + c]) > std::fabs(A[(size_t)piv * (n + 1) + c])) piv = r;
        if (A[(size_t)piv * (n + 1) + c] == 0) {
            if (msg) *msg = "ab_weights: degenerate nodes (singular Vandermonde)";
            return MRAB_E_DEGENERATE_NODES;
        }
        if (piv != c)
            for (int j = 0; j <= n; ++j) std::swap(A[(size_t)c * (n + 1) + j], A[(size_t)piv * (n + 1) + j]);
        for (int r = 0; r < n; ++r) {
            if (r == c) continue;
            LD f = A[(size_t)r * (n + 1) + c] / A[(size_t)c * (n + 1) + c];
            for (int j = c; j <= n; ++j) A[(size_t)r * (n + 1) + j] -= f * A[(size_t)c * (n + 1) + j];
        }
    }
    std::vector<LD> lam(n);
    for (int i = 0; i < n; ++i) lam[i] = A[(size_t)i * (n + 1) + n] / A[(size_t)i * (n + 1) + i];
    for (int k = 0; k < m; ++k) {
        LD s = 0;
        for (int i = 0; i < n; ++i) s += V[(size_t)k * n + i] * lam[i];
        out[k] = (double)s;
    }
    return MRAB_OK;
}

// ------------------------------------------------------------------------------------
// segments (reading R2)
// ------------------------------------------------------------------------------------
static int64_t stride_of(const MeshPlan& m, int k) {
    return k == 0 ? 1 : (k == 1 ? (int64_t)m.n[0] : (int64_t)m.n[0] * m.n[1]);
}

// iterate every line along direction k: fn(first point index)
template <class F>
static void for_lines(const MeshPlan& m, int k, F fn) {
    int o1 = (k == 0) ? 1 : 0, o2 = (k == 2) ? 1 : 2;
    for (int b = 0; b < m.n[o2]; ++b)
        for (int a = 0; a < m.n[o1]; ++a) {
            int idx[3] = {0, 0, 0};
            idx[o1] = a;
            idx[o2] = b;
            idx[k] = 0;
            fn(m.idx(idx[0], idx[1], idx[2]));
        }
}

static bool compute_segments(MeshPlan& m, Error& err) {
    for (int k = 0; k < 3; ++k) {
        m.posA[k].assign(m.npts, -1);
        m.posB[k].assign(m.npts, -1);
    }
    for (int k = 0; k < m.dim; ++k) {
        const int n = m.n[k];
        const int64_t st = stride_of(m, k);
        auto& A = m.posA[k];
        auto& B = m.posB[k];
        for_lines(m, k, [&](int64_t p0) {
            if (m.periodic[k]) {
                int64_t carry = kFar;
                for (int it = 0; it < 2 * n; ++it) {
                    int i = it % n;
                    int64_t p = p0 + st * i;
                    carry = m.active[p] ? std::min<int64_t>(carry + 1, kFar) : -1;
                    if (it >= n) A[p] = (int32_t)carry;
                }
                carry = kFar;
                for (int it = 0; it < 2 * n; ++it) {
                    int i = n - 1 - (it % n);
                    int64_t p = p0 + st * i;
                    carry = m.active[p] ? std::min<int64_t>(carry + 1, kFar) : -1;
                    if (it >= n) B[p] = (int32_t)carry;
                }
            } else {
                int64_t carry = -1;
                for (int i = 0; i < n; ++i) {
                    int64_t p = p0 + st * i;
                    carry = m.active[p] ? carry + 1 : -1;
                    A[p] = (int32_t)carry;
                }
                carry = -1;
                for (int i = n - 1; i >= 0; --i) {
                    int64_t p = p0 + st * i;
                    carry = m.active[p] ? carry + 1 : -1;
                    B[p] = (int32_t)carry;
                }
            }
        });
        for (int64_t p = 0; p < m.npts; ++p) {
            if (A[p] < 0 || A[p] >= kFar || B[p] >= kFar) continue;
            if (A[p] + B[p] + 1 < 8) {
                err = {MRAB_E_SEGMENT, "active segment shorter than 8 points in direction " +
                                            std::to_string(k)};
                return false;
            }
        }
    }
    m.cls.assign(m.npts, 0);
    m.nactive = 0;
    for (int64_t p = 0; p < m.npts; ++p) {
        if (!m.active[p]) continue;
        m.nactive++;
        uint16_t code = 0;
        for (int k = 0; k < m.dim; ++k) {
            int a = m.posA[k][p], b = m.posB[k][p];
            int c = a < 4 ? CLS_L0 + a : (b < 4 ? CLS_R0 + b : CLS_INT);
            code |= (uint16_t)(c << (4 * k));
        }
        m.cls[p] = code;
    }
    return true;
}

// ------------------------------------------------------------------------------------
// metric terms (reading R3): segmented D1 of coordinates, seam-unwrapped
// ------------------------------------------------------------------------------------
static void d1_host(const MeshPlan& m, int k, const double* f, double jump, const double* factor,
                    double* out) {
    const int64_t st = stride_of(m, k);
    const int n = m.n[k];
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < m.npts; ++p) {
        if (!m.active[p]) {
            out[p] = 0.0;
            continue;
        }
        int c = (m.cls[p] >> (4 * k)) & 15;
        const StRow& r = g_rows[c];
        int i = (int)((p / st) % n);
        double s = 0.0;
        for (int t = 0; t < r.n; ++t) {
            int ii = i + r.off[t];
            int w = 0;
            if (ii < 0) {
                ii += n;
                w = -1;
            } else if (ii >= n) {
                ii -= n;
                w = 1;
            }
            int64_t q = p + (int64_t)(ii - i) * st;
            double v = f[q] + w * jump;
            if (factor) v *= factor[q];
            s += r.c[t] * v;
        }
        out[p] = s;
    }
}

// A mesh whose computed metric terms are constant and diagonal to this relative tolerance is
// treated as Cartesian (constants instead of per-point arrays).  The Thomas-Lombard products
// of 3-D coordinates carry ~5e-12 relative rounding at 256^3; the constants then differ from
// the computed arrays by less than that, far inside the 1e-10 parity bar.
static const double kCartTol = 1e-10;

static bool finish_metrics(MeshPlan& m, Error& err);

// caller-supplied metric terms ([0] = J^-1, [1 + kappa*d + i] = M[kappa][i]; mrab.h)
static bool copy_metrics(MeshPlan& m, const double* src, Error& err) {
    const int d = m.dim;
    const int64_t N = m.npts;
    m.jinv.assign(src, src + N);
    m.M.assign(src + N, src + (size_t)(1 + d * d) * N);
    return finish_metrics(m, err);
}

static bool compute_metrics(MeshPlan& m, Error& err) {
    const int d = m.dim;
    const int64_t N = m.npts;
    std::vector<double> dx((size_t)d * d * N);   // dx[c][k] = D_k x_c
    for (int c = 0; c < d; ++c)
        for (int k = 0; k < d; ++k)
            d1_host(m, k, &m.xyz[(size_t)c * N], m.period[k][c], nullptr, &dx[((size_t)c * d + k) * N]);
    auto DX = [&](int c, int k) { return &dx[((size_t)c * d + k) * N]; };
    m.jinv.assign(N, 0.0);
    m.M.assign((size_t)d * d * N, 0.0);
    auto Mp = [&](int kap, int i) { return &m.M[((size_t)kap * d + i) * N]; };
    if (d == 2) {
        for (int64_t p = 0; p < N; ++p) {
            m.jinv[p] = DX(0, 0)[p] * DX(1, 1)[p] - DX(0, 1)[p] * DX(1, 0)[p];
            Mp(0, 0)[p] = DX(1, 1)[p];
            Mp(0, 1)[p] = -DX(0, 1)[p];
            Mp(1, 0)[p] = -DX(1, 0)[p];
            Mp(1, 1)[p] = DX(0, 0)[p];
        }
    } else {
        std::vector<double> t1(N), t2(N);
        for (int kap = 0; kap < 3; ++kap) {
            int b = (kap + 1) % 3, c = (kap + 2) % 3;
            for (int i = 0; i < 3; ++i) {
                int j = (i + 1) % 3, kk = (i + 2) % 3;
                // D_c(x_k D_b x_j) - D_b(x_k D_c x_j)
                d1_host(m, c, &m.xyz[(size_t)kk * N], m.period[c][kk], DX(j, b), t1.data());
                d1_host(m, b, &m.xyz[(size_t)kk * N], m.period[b][kk], DX(j, c), t2.data());
                double* o = Mp(kap, i);
                for (int64_t p = 0; p < N; ++p) o[p] = t1[p] - t2[p];
            }
        }
        for (int64_t p = 0; p < N; ++p) {
            double a00 = DX(0, 0)[p], a01 = DX(0, 1)[p], a02 = DX(0, 2)[p];
            double a10 = DX(1, 0)[p], a11 = DX(1, 1)[p], a12 = DX(1, 2)[p];
            double a20 = DX(2, 0)[p], a21 = DX(2, 1)[p], a22 = DX(2, 2)[p];
            m.jinv[p] = a00 * (a11 * a22 - a12 * a21) - a01 * (a10 * a22 - a12 * a20) +
                        a02 * (a10 * a21 - a11 * a20);
        }
    }
    return finish_metrics(m, err);
}

// positivity and Cartesian detection
static bool finish_metrics(MeshPlan& m, Error& err) {
    const int d = m.dim;
    const int64_t N = m.npts;
    auto Mp = [&](int kap, int i) { return &m.M[((size_t)kap * d + i) * N]; };
    int64_t first = -1;
    for (int64_t p = 0; p < N; ++p) {
        if (!m.active[p]) continue;
        if (!(m.jinv[p] > 0.0)) {
            err = {MRAB_E_INVALID, "non-positive J^-1 at an active point (left-handed mesh?)"};
            return false;
        }
        if (first < 0) first = p;
    }
    m.cartesian = first >= 0;
    if (first >= 0) {
        double j0 = m.jinv[first];
        double md[3] = {0, 0, 0};
        for (int k = 0; k < d; ++k) md[k] = Mp(k, k)[first];
        for (int64_t p = 0; p < N && m.cartesian; ++p) {
            if (!m.active[p]) continue;
            if (std::fabs(m.jinv[p] - j0) > kCartTol * std::fabs(j0)) m.cartesian = false;
            for (int k = 0; k < d && m.cartesian; ++k)
                for (int i = 0; i < d; ++i) {
                    double v = Mp(k, i)[p];
                    double e = (k == i) ? md[k] : 0.0;
                    if (std::fabs(v - e) > kCartTol * std::fabs(md[k])) {
                        m.cartesian = false;
                        break;
                    }
                }
        }
        if (m.cartesian) {
            m.cart_J = 1.0 / j0;
            for (int k = 0; k < d; ++k) m.cart_M[k] = md[k];
        }
    }
    return true;
}

// ------------------------------------------------------------------------------------
// overset (reading R17)
// ------------------------------------------------------------------------------------
static const double kSnap = 1e-12, kNewtonTol = 1e-12, kGrow = 0.1, kAbs = 1e-9;
static const int kNewtonMax = 50;

static inline void lagr(double t, double* w, double* dw) {
    for (int a = 0; a < 4; ++a) {
        double v = 1.0;
        for (int b = 0; b < 4; ++b)
            if (b != a) v = v * (t - b) / (double)(a - b);
        w[a] = v;
        if (dw) {
            double acc = 0.0;
            for (int c = 0; c < 4; ++c) {
                if (c == a) continue;
                double term = 1.0 / (double)(a - c);
                for (int b = 0; b < 4; ++b)
                    if (b != a && b != c) term = term * (t - b) / (double)(a - b);
                acc += term;
            }
            dw[a] = acc;
        }
    }
}

// coordinates of (possibly unwrapped) node idx
static inline void node_xyz(const MeshPlan& m, const int* idx, double* X) {
    int w[3] = {0, 0, 0}, ii[3] = {0, 0, 0};
    for (int k = 0; k < m.dim; ++k) {
        int n = m.n[k], v = idx[k];
        if (m.periodic[k]) {
            int q = (int)std::floor((double)v / n);
            w[k] = q;
            v -= q * n;
        }
        ii[k] = v;
    }
    int64_t p = m.idx(ii[0], ii[1], m.dim == 3 ? ii[2] : 0);
    for (int c = 0; c < m.dim; ++c) {
        double v = m.xyz[(size_t)c * m.npts + p];
        for (int k = 0; k < m.dim; ++k) v = v + w[k] * m.period[k][c];
        X[c] = v;
    }
}

struct CellIndex {
    int dim = 2;
    int nc[3] = {1, 1, 1};
    int64_t ncell = 0;
    std::vector<double> lo, hi;             // [ncell][dim]
    double glo[3] = {0, 0, 0}, gsz[3] = {1, 1, 1};
    int nb[3] = {1, 1, 1};
    std::vector<int64_t> bstart, bcells;
    double bblo[3], bbhi[3];                 // grown global node bbox (prefilter)
};

static void build_cell_index(const MeshPlan& m, CellIndex& ci) {
    const int d = m.dim;
    ci.dim = d;
    for (int k = 0; k < 3; ++k) ci.nc[k] = (k < d) ? (m.periodic[k] ? m.n[k] : m.n[k] - 1) : 1;
    ci.ncell = (int64_t)ci.nc[0] * ci.nc[1] * ci.nc[2];
    ci.lo.assign((size_t)ci.ncell * d, 0.0);
    ci.hi.assign((size_t)ci.ncell * d, 0.0);
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < ci.ncell; ++c) {
        int cc[3] = {(int)(c % ci.nc[0]), (int)((c / ci.nc[0]) % ci.nc[1]), (int)(c / ((int64_t)ci.nc[0] * ci.nc[1]))};
        double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
        for (int corner = 0; corner < (1 << d); ++corner) {
            int idx[3] = {0, 0, 0};
            for (int k = 0; k < d; ++k) idx[k] = cc[k] + ((corner >> k) & 1);
            double X[3];
            node_xyz(m, idx, X);
            for (int k = 0; k < d; ++k) {
                lo[k] = std::min(lo[k], X[k]);
                hi[k] = std::max(hi[k], X[k]);
            }
        }
        for (int k = 0; k < d; ++k) {
            double g = kGrow * (hi[k] - lo[k]) + kAbs;
            ci.lo[(size_t)c * d + k] = lo[k] - g;
            ci.hi[(size_t)c * d + k] = hi[k] + g;
        }
    }
    // global node bbox (prefilter, same rule as the cells)
    for (int k = 0; k < d; ++k) {
        double lo = 1e300, hi = -1e300;
        const double* x = &m.xyz[(size_t)k * m.npts];
        for (int64_t p = 0; p < m.npts; ++p) {
            lo = std::min(lo, x[p]);
            hi = std::max(hi, x[p]);
        }
        double g = kGrow * (hi - lo) + kAbs;
        ci.bblo[k] = lo - g;
        ci.bbhi[k] = hi + g;
    }
    // bucket grid over the union of cell boxes
    double glo[3], ghi[3];
    for (int k = 0; k < d; ++k) {
        glo[k] = 1e300;
        ghi[k] = -1e300;
    }
    for (int64_t c = 0; c < ci.ncell; ++c)
        for (int k = 0; k < d; ++k) {
            glo[k] = std::min(glo[k], ci.lo[(size_t)c * d + k]);
            ghi[k] = std::max(ghi[k], ci.hi[(size_t)c * d + k]);
        }
    int64_t nbt = 1;
    for (int k = 0; k < d; ++k) {
        ci.nb[k] = std::max(1, ci.nc[k] / 2);
        ci.glo[k] = glo[k];
        ci.gsz[k] = (ghi[k] - glo[k]) / ci.nb[k];
        if (!(ci.gsz[k] > 0)) ci.gsz[k] = 1.0;
        nbt *= ci.nb[k];
    }
    for (int k = d; k < 3; ++k) ci.nb[k] = 1;
    std::vector<int64_t> cnt(nbt + 1, 0);
    auto brange = [&](int64_t c, int* b0, int* b1) {
        for (int k = 0; k < d; ++k) {
            int a = (int)std::floor((ci.lo[(size_t)c * d + k] - ci.glo[k]) / ci.gsz[k]);
            int b = (int)std::floor((ci.hi[(size_t)c * d + k] - ci.glo[k]) / ci.gsz[k]);
            b0[k] = std::max(0, std::min(ci.nb[k] - 1, a));
            b1[k] = std::max(0, std::min(ci.nb[k] - 1, b));
        }
        for (int k = d; k < 3; ++k) b0[k] = b1[k] = 0;
    };
    for (int pass = 0; pass < 2; ++pass) {
        std::vector<int64_t> fill;
        if (pass == 1) {
            for (int64_t b = 0; b < nbt; ++b) cnt[b + 1] += cnt[b];
            ci.bstart = cnt;
            ci.bcells.assign(cnt[nbt], 0);
            fill.assign(cnt.begin(), cnt.end() - 1);
        }
        for (int64_t c = 0; c < ci.ncell; ++c) {
            int b0[3], b1[3];
            brange(c, b0, b1);
            for (int z = b0[2]; z <= b1[2]; ++z)
                for (int y = b0[1]; y <= b1[1]; ++y)
                    for (int x = b0[0]; x <= b1[0]; ++x) {
                        int64_t b = x + (int64_t)ci.nb[0] * (y + (int64_t)ci.nb[1] * z);
                        if (pass == 0)
                            cnt[b + 1]++;
                        else
                            ci.bcells[fill[b]++] = c;
                    }
        }
    }
}

// Newton on the tensor-cubic Lagrange map of cell c's stencil.
static bool newton_cell(const MeshPlan& m, const int* cc, const double* X, double* xi_out) {
    const int d = m.dim;
    int s[3] = {0, 0, 0};
    for (int k = 0; k < d; ++k) {
        s[k] = cc[k] - 1;
        if (!m.periodic[k]) s[k] = std::max(0, std::min(m.n[k] - 4, s[k]));
    }
    // gather stencil node coordinates (4^d x d)
    double nodes[64][3];
    int npt = d == 2 ? 16 : 64;
    for (int a = 0; a < npt; ++a) {
        int idx[3] = {s[0] + (a & 3), s[1] + ((a >> 2) & 3), d == 3 ? s[2] + ((a >> 4) & 3) : 0};
        node_xyz(m, idx, nodes[a]);
    }
    double xi[3] = {0, 0, 0};
    for (int k = 0; k < d; ++k) xi[k] = cc[k] + 0.5;
    bool conv = false;
    for (int it = 0; it < kNewtonMax; ++it) {
        double w[3][4], dw[3][4];
        for (int k = 0; k < d; ++k) lagr(xi[k] - s[k], w[k], dw[k]);
        double Xm[3] = {0, 0, 0}, J[3][3] = {{0}};
        for (int a = 0; a < npt; ++a) {
            int ai[3] = {a & 3, (a >> 2) & 3, (a >> 4) & 3};
            double wp = 1.0;
            for (int k = 0; k < d; ++k) wp *= w[k][ai[k]];
            for (int c = 0; c < d; ++c) Xm[c] += wp * nodes[a][c];
            for (int k = 0; k < d; ++k) {
                double g = 1.0;
                for (int l = 0; l < d; ++l) g *= (l == k) ? dw[l][ai[l]] : w[l][ai[l]];
                for (int c = 0; c < d; ++c) J[c][k] += g * nodes[a][c];
            }
        }
        // solve J delta = X - Xm (Gaussian elimination, partial pivoting)
        double A[3][4];
        for (int r = 0; r < d; ++r) {
            for (int c = 0; c < d; ++c) A[r][c] = J[r][c];
            A[r][d] = X[r] - Xm[r];
        }
        bool bad = false;
        for (int c = 0; c < d && !bad; ++c) {
            int piv = c;
            for (int r = c + 1; r < d; ++r)
                if (std::fabs(A[r][c]) > std::fabs(A[piv][c])) piv = r;
            if (A[piv][c] == 0.0) {
                bad = true;
                break;
            }
            if (piv != c)
                for (int j = 0; j <= d; ++j) std::swap(A[c][j], A[piv][j]);
            for (int r = c + 1; r < d; ++r) {
                double f = A[r][c] / A[c][c];
                for (int j = c; j <= d; ++j) A[r][j] -= f * A[c][j];
            }
        }
        if (bad) return false;
        double delta[3];
        for (int r = d - 1; r >= 0; --r) {
            double v = A[r][d];
            for (int j = r + 1; j < d; ++j) v -= A[r][j] * delta[j];
            delta[r] = v / A[r][r];
        }
        bool finite = true;
        for (int k = 0; k < d; ++k) finite = finite && std::isfinite(delta[k]);
        if (!finite) return false;
        bool small = true, far = false;
        for (int k = 0; k < d; ++k) {
            xi[k] += delta[k];
            if (std::fabs(xi[k] - (cc[k] + 0.5)) > 4.0) far = true;
            if (!(std::fabs(delta[k]) <= kNewtonTol)) small = false;
        }
        if (far) return false;
        if (small) {
            conv = true;
            break;
        }
    }
    if (!conv) return false;
    for (int k = 0; k < d; ++k)
        if (!(xi[k] >= cc[k] - kSnap && xi[k] <= cc[k] + 1 + kSnap)) return false;
    for (int k = 0; k < d; ++k) {
        double r = std::nearbyint(xi[k]);
        xi_out[k] = (std::fabs(xi[k] - r) <= kSnap) ? r : xi[k];
    }
    return true;
}

// logical coordinates of X in mesh m (first accepted candidate cell in flat order)
static bool find_cell(const MeshPlan& m, const CellIndex& ci, const double* X, double* xi) {
    const int d = m.dim;
    int bk[3] = {0, 0, 0};
    for (int k = 0; k < d; ++k) {
        double f = std::floor((X[k] - ci.glo[k]) / ci.gsz[k]);
        if (f < 0 || f >= ci.nb[k]) {
            // may still sit exactly on the far edge of the bucket grid
            if (f == ci.nb[k] && X[k] <= ci.glo[k] + ci.gsz[k] * ci.nb[k])
                f = ci.nb[k] - 1;
            else
                return false;
        }
        bk[k] = (int)f;
    }
    int64_t b = bk[0] + (int64_t)ci.nb[0] * (bk[1] + (int64_t)ci.nb[1] * bk[2]);
    std::vector<int64_t> cand;
    for (int64_t t = ci.bstart[b]; t < ci.bstart[b + 1]; ++t) {
        int64_t c = ci.bcells[t];
        bool in = true;
        for (int k = 0; k < d && in; ++k)
            in = X[k] >= ci.lo[(size_t)c * d + k] && X[k] <= ci.hi[(size_t)c * d + k];
        if (in) cand.push_back(c);
    }
    std::sort(cand.begin(), cand.end());
    for (int64_t c : cand) {
        int cc[3] = {(int)(c % ci.nc[0]), (int)((c / ci.nc[0]) % ci.nc[1]), (int)(c / ((int64_t)ci.nc[0] * ci.nc[1]))};
        if (newton_cell(m, cc, X, xi)) return true;
    }
    return false;
}

static void stencil_base(const MeshPlan& m, const double* xi, int* s) {
    for (int k = 0; k < m.dim; ++k) {
        int i0 = (int)std::floor(xi[k]);
        s[k] = i0 - 1;
        if (!m.periodic[k]) s[k] = std::max(0, std::min(m.n[k] - 4, s[k]));
    }
    for (int k = m.dim; k < 3; ++k) s[k] = 0;
}

// flat indices of the stencil at (unwrapped) base s; false if it leaves the mesh
static bool stencil_points(const MeshPlan& m, const int* s, int64_t* out) {
    const int d = m.dim;
    int npt = d == 2 ? 16 : 64;
    for (int k = 0; k < d; ++k)
        if (!m.periodic[k] && (s[k] < 0 || s[k] + 3 > m.n[k] - 1)) return false;
    for (int a = 0; a < npt; ++a) {
        int idx[3] = {s[0] + (a & 3), s[1] + ((a >> 2) & 3), d == 3 ? s[2] + ((a >> 4) & 3) : 0};
        for (int k = 0; k < d; ++k)
            if (m.periodic[k]) idx[k] = ((idx[k] % m.n[k]) + m.n[k]) % m.n[k];
        out[a] = m.idx(idx[0], idx[1], idx[2]);
    }
    return true;
}

static bool in_wall_body(const MeshPlan& mw, const double* X) {
    if (mw.dim != 2) return false;
    bool inside = false;
    for (int kap = 0; kap < 2; ++kap)
        for (int side = 0; side < 2; ++side) {
            if (mw.face_bc[kap][side] != MRAB_BC_WALL) continue;
            int other = 1 - kap, no = mw.n[other];
            int j = side == 0 ? 0 : mw.n[kap] - 1;
            bool cnt = false;
            for (int e = 0; e < no; ++e) {
                int i1[3] = {0, 0, 0}, i2[3] = {0, 0, 0};
                i1[other] = e;
                i1[kap] = j;
                i2[other] = (e + 1) % no;
                i2[kap] = j;
                double P1[3], P2[3];
                node_xyz(mw, i1, P1);
                node_xyz(mw, i2, P2);
                bool cond = (P1[1] > X[1]) != (P2[1] > X[1]);
                if (cond) {
                    double xint = P1[0] + (X[1] - P1[1]) * (P2[0] - P1[0]) / (P2[1] - P1[1]);
                    if (X[0] < xint) cnt = !cnt;
                }
            }
            inside = inside || cnt;
        }
    return inside;
}

static void point_xyz(const MeshPlan& m, int64_t p, double* X) {
    for (int c = 0; c < m.dim; ++c) X[c] = m.xyz[(size_t)c * m.npts + p];
}

// Caller-supplied donor entries of receiving mesh g (mrab.h mrab_problem.donors): exactly one
// per receiver; stencils inside the donor mesh and all active; weights verbatim.
static bool take_donors(Plan& P, const mrab_problem* pb, int g, const std::vector<int64_t>& pts,
                        std::vector<uint8_t>& todo, Error& err) {
    MeshPlan& m = P.meshes[g];
    const int G = (int)P.meshes.size();
    std::vector<int32_t> slot(m.npts, -1);
    for (size_t r = 0; r < pts.size(); ++r) slot[pts[r]] = (int32_t)r;
    auto bad = [&](int64_t e, const std::string& why) {
        err = {MRAB_E_INVALID, "donor entry " + std::to_string(e) + ": " + why};
        return false;
    };
    for (int64_t e = 0; e < pb->n_donors; ++e) {
        const mrab_donor& dn = pb->donors[e];
        if (dn.recv_mesh < 0 || dn.recv_mesh >= G) return bad(e, "recv_mesh out of range");
        if (dn.recv_mesh != g) continue;
        if (dn.donor_mesh < 0 || dn.donor_mesh >= G || dn.donor_mesh == g)
            return bad(e, "donor_mesh out of range or equal to recv_mesh");
        if (dn.recv_index < 0 || dn.recv_index >= m.npts || slot[dn.recv_index] < 0)
            return bad(e, "recv_index is not a receiver of mesh " + std::to_string(g));
        const int64_t r = slot[dn.recv_index];
        if (!todo[r]) return bad(e, "duplicate receiver");
        const MeshPlan& ma = P.meshes[dn.donor_mesh];
        int s[3] = {dn.base[0], dn.base[1], ma.dim == 3 ? dn.base[2] : 0};
        int64_t st[64];
        if (!stencil_points(ma, s, st)) return bad(e, "donor stencil leaves the donor mesh");
        for (int a = 0; a < (ma.dim == 2 ? 16 : 64); ++a)
            if (!ma.active[st[a]]) return bad(e, "donor stencil touches a hole");
        m.rdonor[r] = dn.donor_mesh;
        for (int k = 0; k < 3; ++k) {
            int v = s[k];
            if (k < ma.dim && ma.periodic[k]) v = ((v % ma.n[k]) + ma.n[k]) % ma.n[k];
            m.rbase[(size_t)r * 3 + k] = v;
        }
        for (int k = 0; k < 3; ++k)
            for (int a = 0; a < 4; ++a) m.rw[(size_t)r * 12 + k * 4 + a] = dn.w[k][a];
        if (ma.dim == 2) {
            double* w = &m.rw[(size_t)r * 12 + 8];
            w[0] = 1.0;
            w[1] = w[2] = w[3] = 0.0;
        }
        todo[r] = 0;
    }
    return true;
}

static bool build_overset(Plan& P, const mrab_problem* pb, Error& err) {
    const int G = (int)P.meshes.size();
    const bool given_donors = pb->n_donors > 0 && pb->donors;
    bool all_blank = true;
    for (int g = 0; g < G; ++g) all_blank = all_blank && pb->meshes[g].iblank;
    std::vector<CellIndex> ci(G);
    if (!(all_blank && given_donors))          // the cell index serves the geometric searches
        for (int g = 0; g < G; ++g) build_cell_index(P.meshes[g], ci[g]);
    std::vector<int> order_all(G);
    std::iota(order_all.begin(), order_all.end(), 0);
    auto prio_order = [&](int exclude) {
        std::vector<int> o;
        for (int g = 0; g < G; ++g)
            if (g != exclude) o.push_back(g);
        std::stable_sort(o.begin(), o.end(), [&](int a, int b) {
            return P.meshes[a].priority > P.meshes[b].priority;
        });
        return o;
    };
    // 1. inside higher-priority meshes or wall bodies
    std::vector<std::vector<uint8_t>> inside(G), prot(G);
    for (int A = 0; A < G; ++A) {
        MeshPlan& ma = P.meshes[A];
        inside[A].assign(ma.npts, 0);
        prot[A].assign(ma.npts, 0);
        if (pb->meshes[A].iblank) continue;    // caller-supplied blanking (mrab.h)
        for (int B = 0; B < G; ++B) {
            if (B == A) continue;
            const MeshPlan& mb = P.meshes[B];
            bool higher = mb.priority > ma.priority;
            bool has_wall = false;
            for (int k = 0; k < mb.dim; ++k)
                for (int s = 0; s < 2; ++s) has_wall = has_wall || mb.face_bc[k][s] == MRAB_BC_WALL;
            if (!higher && !has_wall) continue;
#pragma omp parallel for schedule(dynamic, 1024)
            for (int64_t p = 0; p < ma.npts; ++p) {
                double X[3];
                point_xyz(ma, p, X);
                if (higher) {
                    bool inbb = true;
                    for (int k = 0; k < ma.dim; ++k) inbb = inbb && X[k] >= ci[B].bblo[k] && X[k] <= ci[B].bbhi[k];
                    double xi[3];
                    if (inbb && find_cell(mb, ci[B], X, xi)) inside[A][p] = 1;
                }
                if (has_wall && in_wall_body(mb, X)) inside[A][p] = 1;
            }
        }
    }
    // 2. protect the donor stencils of overset-face points
    for (int B = 0; B < G && !all_blank; ++B) {
        const MeshPlan& mb = P.meshes[B];
        std::vector<int64_t> fpts;
        for (int64_t p = 0; p < mb.npts; ++p) {
            int ii[3] = {(int)(p % mb.n[0]), (int)((p / mb.n[0]) % mb.n[1]), (int)(p / ((int64_t)mb.n[0] * mb.n[1]))};
            bool on = false;
            for (int k = 0; k < mb.dim && !on; ++k) {
                if (mb.periodic[k]) continue;
                if (ii[k] == 0 && mb.face_bc[k][0] == MRAB_BC_OVERSET) on = true;
                if (ii[k] == mb.n[k] - 1 && mb.face_bc[k][1] == MRAB_BC_OVERSET) on = true;
            }
            if (on) fpts.push_back(p);
        }
        if (fpts.empty()) continue;
        std::vector<uint8_t> todo(fpts.size(), 1);
        for (int A : prio_order(B)) {
            const MeshPlan& ma = P.meshes[A];
            const bool mark = !pb->meshes[A].iblank;   // caller blanking: no protection marks
            std::vector<std::vector<int64_t>> marks(fpts.size());
#pragma omp parallel for schedule(dynamic, 64)
            for (int64_t r = 0; r < (int64_t)fpts.size(); ++r) {
                if (!todo[r]) continue;
                double X[3], xi[3];
                point_xyz(mb, fpts[r], X);
                if (!find_cell(ma, ci[A], X, xi)) continue;
                int s[3];
                stencil_base(ma, xi, s);
                int64_t st[64];
                if (mark && stencil_points(ma, s, st)) marks[r].assign(st, st + (ma.dim == 2 ? 16 : 64));
                todo[r] = 0;
            }
            for (auto& v : marks)
                for (int64_t q : v) prot[A][q] = 1;
        }
    }
    // 3. blanking, segments, classes, metrics
    for (int g = 0; g < G; ++g) {
        MeshPlan& m = P.meshes[g];
        m.active.assign(m.npts, 1);
        if (const int8_t* ib = pb->meshes[g].iblank) {
            for (int64_t p = 0; p < m.npts; ++p) m.active[p] = ib[p] != 0;
        } else {
            for (int64_t p = 0; p < m.npts; ++p)
                if (inside[g][p] && !prot[g][p]) m.active[p] = 0;
        }
        if (!compute_segments(m, err)) {
            err.msg = "mesh " + std::to_string(g) + ": " + err.msg;
            return false;
        }
    }
    // 4. receivers and donors
    P.donor_of.assign(G, std::vector<int>(G, 0));
    for (int g = 0; g < G; ++g) {
        MeshPlan& m = P.meshes[g];
        std::vector<int64_t> pts;
        for (int64_t p = 0; p < m.npts; ++p) {
            if (!m.active[p]) continue;
            int ii[3] = {(int)(p % m.n[0]), (int)((p / m.n[0]) % m.n[1]), (int)(p / ((int64_t)m.n[0] * m.n[1]))};
            bool recv = false;
            for (int k = 0; k < m.dim && !recv; ++k) {
                for (int side = 0; side < 2; ++side) {
                    int pos = side == 0 ? m.posA[k][p] : m.posB[k][p];
                    if (pos != 0) continue;
                    if (m.periodic[k]) {
                        recv = true;
                    } else {
                        bool at_face = side == 0 ? ii[k] == 0 : ii[k] == m.n[k] - 1;
                        if (!at_face || m.face_bc[k][side] == MRAB_BC_OVERSET) recv = true;
                    }
                }
            }
            if (recv) pts.push_back(p);
        }
        const int64_t R = (int64_t)pts.size();
        m.rpoint = pts;
        m.rdonor.assign(R, -1);
        m.rbase.assign((size_t)R * 3, 0);
        m.rw.assign((size_t)R * 12, 0.0);
        std::vector<uint8_t> todo(R, 1);
        if (given_donors) {
            if (!take_donors(P, pb, g, pts, todo, err)) return false;
        } else {
        // shift order: sum|delta| ascending, then lexicographic (axis 0 first), 0 < +1 < -1
        std::vector<std::array<int, 3>> shifts;
        {
            int nd = m.dim;
            int tot = nd == 2 ? 9 : 27;
            const int val[3] = {0, 1, -1};
            std::vector<std::pair<std::array<int, 4>, std::array<int, 3>>> tmp;
            for (int t = 0; t < tot; ++t) {
                int r0 = t % 3, r1 = (t / 3) % 3, r2 = (t / 9) % 3;
                std::array<int, 3> dl = {val[r0], val[r1], nd == 3 ? val[r2] : 0};
                int ranks[3] = {r0, r1, nd == 3 ? r2 : 0};
                int l1 = std::abs(dl[0]) + std::abs(dl[1]) + std::abs(dl[2]);
                tmp.push_back({{l1, ranks[0], ranks[1], ranks[2]}, dl});
            }
            std::sort(tmp.begin(), tmp.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
            for (auto& t : tmp) shifts.push_back(t.second);
        }
        for (int A : prio_order(g)) {
            const MeshPlan& ma = P.meshes[A];
#pragma omp parallel for schedule(dynamic, 64)
            for (int64_t r = 0; r < R; ++r) {
                if (!todo[r]) continue;
                double X[3], xi[3];
                point_xyz(m, pts[r], X);
                if (!find_cell(ma, ci[A], X, xi)) continue;
                int s0[3];
                stencil_base(ma, xi, s0);
                for (auto& dl : shifts) {
                    int s[3] = {s0[0] + dl[0], s0[1] + dl[1], s0[2] + dl[2]};
                    if (ma.dim == 2) s[2] = 0;
                    int64_t st[64];
                    if (!stencil_points(ma, s, st)) continue;
                    bool all = true;
                    for (int a = 0; a < (ma.dim == 2 ? 16 : 64) && all; ++a) all = ma.active[st[a]] != 0;
                    if (!all) continue;
                    m.rdonor[r] = A;
                    for (int k = 0; k < 3; ++k) {
                        int v = s[k];
                        if (k < ma.dim && ma.periodic[k]) v = ((v % ma.n[k]) + ma.n[k]) % ma.n[k];
                        m.rbase[(size_t)r * 3 + k] = v;
                    }
                    for (int k = 0; k < ma.dim; ++k) lagr(xi[k] - s[k], &m.rw[(size_t)r * 12 + k * 4], nullptr);
                    if (ma.dim == 2) {
                        double* w = &m.rw[(size_t)r * 12 + 8];
                        w[0] = 1.0;
                        w[1] = w[2] = w[3] = 0.0;
                    }
                    todo[r] = 0;
                    break;
                }
            }
        }
        }
        int64_t orphans = 0, first = -1;
        for (int64_t r = 0; r < R; ++r)
            if (todo[r]) {
                orphans++;
                if (first < 0) first = pts[r];
            }
        if (orphans) {
            err = {MRAB_E_ORPHAN, "mesh " + std::to_string(g) + ": " + std::to_string(orphans) +
                                      " receivers without an all-active donor stencil (first point " +
                                      std::to_string(first) + ")"};
            return false;
        }
        m.recv_slot.assign(m.npts, -1);
        for (int64_t r = 0; r < R; ++r) {
            m.recv_slot[pts[r]] = (int32_t)r;
            P.donor_of[m.rdonor[r]][g] = 1;
        }
    }
    // 5. donor boxes: stencil bounding box per donor mesh, grown by the D1 reach (3)
    for (int A = 0; A < G; ++A) {
        MeshPlan& ma = P.meshes[A];
        int lo[3] = {1 << 30, 1 << 30, 1 << 30}, hi[3] = {-1, -1, -1};
        bool full[3] = {false, false, false};
        bool any = false;
        for (int g = 0; g < G; ++g) {
            const MeshPlan& m = P.meshes[g];
            for (size_t r = 0; r < m.rdonor.size(); ++r) {
                if (m.rdonor[r] != A) continue;
                any = true;
                for (int k = 0; k < ma.dim; ++k) {
                    int b = m.rbase[r * 3 + k];
                    if (b + 3 > ma.n[k] - 1) full[k] = true;      // wraps the periodic seam
                    lo[k] = std::min(lo[k], b);
                    hi[k] = std::max(hi[k], b + 3);
                }
            }
        }
        ma.is_donor = any;
        for (int k = 0; k < 3; ++k) {
            if (k >= ma.dim || !any) {
                ma.fv_lo[k] = ma.st_lo[k] = 0;
                ma.fv_hi[k] = ma.st_hi[k] = (k < ma.dim ? ma.n[k] - 1 : 0);
                continue;
            }
            if (full[k]) {
                ma.fv_lo[k] = ma.st_lo[k] = 0;
                ma.fv_hi[k] = ma.st_hi[k] = ma.n[k] - 1;
                continue;
            }
            ma.fv_lo[k] = lo[k];
            ma.fv_hi[k] = std::min(hi[k], ma.n[k] - 1);
            int sl = lo[k] - 3, sh = hi[k] + 3;
            if (ma.periodic[k] && (sl < 0 || sh > ma.n[k] - 1)) {
                ma.fv_lo[k] = ma.st_lo[k] = 0;
                ma.fv_hi[k] = ma.st_hi[k] = ma.n[k] - 1;
            } else {
                ma.st_lo[k] = std::max(0, sl);
                ma.st_hi[k] = std::min(ma.n[k] - 1, sh);
            }
        }
    }
    return true;
}

// ------------------------------------------------------------------------------------
bool build_plan(const mrab_problem* pb, Plan& P, Error& err, bool overset_only) {
    init_rows();
    P.opt = read_options();
    if (!pb || pb->n_meshes < 1 || pb->n_meshes > kMaxMeshes || !pb->meshes || (pb->dim != 2 && pb->dim != 3)) {
        err = {MRAB_E_INVALID, "problem: need 1..8 meshes and dim 2 or 3"};
        return false;
    }
    if (pb->history_m < pb->order_n) {
        err = {MRAB_E_INSUFFICIENT_HISTORY, "history_m < order_n"};
        return false;
    }
    if (pb->order_n < 1 || pb->order_n > 4 || pb->history_m > kMaxHist) {
        err = {MRAB_E_INVALID, "order_n must be 1..4 and history_m <= 6"};
        return false;
    }
    if (!(pb->h > 0)) {
        err = {MRAB_E_INVALID, "h must be positive"};
        return false;
    }
    if (pb->n_donors < 0 || (pb->n_donors > 0 && !pb->donors)) {
        err = {MRAB_E_INVALID, "n_donors < 0, or n_donors > 0 with donors NULL"};
        return false;
    }
    if (pb->viscous && !(pb->Re > 0)) {
        err = {MRAB_E_INVALID, "viscous problem needs Re > 0"};
        return false;
    }
    P.dim = pb->dim;
    P.nc = pb->dim + 2;
    P.gamma = pb->gamma;
    P.Re = pb->Re;
    P.Pr = pb->Pr;
    P.viscous = pb->viscous;
    P.wall_T = pb->wall_T;
    for (int c = 0; c < 5; ++c) P.q_inf[c] = pb->q_inf[c];
    P.order_n = pb->order_n;
    P.history_m = pb->history_m;
    P.h = pb->h;
    P.meshes.resize(pb->n_meshes);
    P.S = 1;
    for (int g = 0; g < pb->n_meshes; ++g) {
        const mrab_mesh_desc& d = pb->meshes[g];
        MeshPlan& m = P.meshes[g];
        if (d.dim != pb->dim || !d.xyz) {
            err = {MRAB_E_INVALID, "mesh " + std::to_string(g) + ": dim mismatch or NULL xyz"};
            return false;
        }
        m.dim = d.dim;
        for (int k = 0; k < 3; ++k) {
            m.n[k] = (k < d.dim) ? d.n[k] : 1;
            m.periodic[k] = (k < d.dim) ? d.periodic[k] : 0;
            for (int s = 0; s < 2; ++s) m.face_bc[k][s] = d.face_bc[k][s];
            for (int c = 0; c < 3; ++c) m.period[k][c] = d.period[k][c];
            if (k < d.dim && m.n[k] < 8) {
                err = {MRAB_E_INVALID, "mesh " + std::to_string(g) + ": fewer than 8 points in a direction"};
                return false;
            }
        }
        m.priority = d.priority;
        m.s = d.step_multiple;
        if (m.s < 1) {
            err = {MRAB_E_INVALID, "step_multiple must be >= 1"};
            return false;
        }
        P.S = std::max(P.S, m.s);
        m.npts = (int64_t)m.n[0] * m.n[1] * m.n[2];
        m.xyz.assign(d.xyz, d.xyz + (size_t)d.dim * m.npts);
    }
    for (auto& m : P.meshes)
        if (P.S % m.s != 0) {
            err = {MRAB_E_MISALIGNED, "every step multiple must divide the largest one"};
            return false;
        }
    if (!build_overset(P, pb, err)) return false;
    if (overset_only) return true;
    for (int g = 0; g < (int)P.meshes.size(); ++g)
        if (!(pb->meshes[g].metrics ? copy_metrics(P.meshes[g], pb->meshes[g].metrics, err)
                                    : compute_metrics(P.meshes[g], err))) {
            err.msg = "mesh " + std::to_string(g) + ": " + err.msg;
            return false;
        }
    // coefficient tables: weights over [0, j/s_g] for j = 1..s_g, nodes -(m-1)..0
    P.coef.resize(P.meshes.size());
    std::vector<double> nodes(P.history_m);
    for (int k = 0; k < P.history_m; ++k) nodes[k] = -(P.history_m - 1) + k;
    for (size_t g = 0; g < P.meshes.size(); ++g) {
        int s = P.meshes[g].s;
        P.coef[g].assign(s + 1, std::vector<double>(P.history_m, 0.0));
        for (int j = 1; j <= s; ++j) {
            std::string msg;
            mrab_status st = ab_weights(nodes.data(), P.history_m, P.order_n, 0.0, (double)j / s,
                                        P.coef[g][j].data(), &msg);
            if (st != MRAB_OK) {
                err = {st, msg};
                return false;
            }
        }
    }
    return true;
}

}  // namespace mrab
