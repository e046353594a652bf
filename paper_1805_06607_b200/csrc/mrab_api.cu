// C ABI of libmrab.so: plans, contexts, the MRAB schedule and its CUDA graphs.
//
// Schedule (P:569-610 Steps 1-7 generalised to N rates, reading R8 of DESIGN.md):
// a macro step covers micro times t + j h, j = 0..S-1.  At micro time j the meshes with
// j mod s_g == 0 "step": their RHS is evaluated at their current state and, fused in the
// same kernel, their state is advanced by one AB step of size h_g = s_g h (the new RHS is
// pushed into the history ring first).  A mesh that does not step at j but donates to one
// that does supplies an intermediate state base_g + h_g sum_k beta_k R_k on its donor box
// (the partial integral of its extrapolant, Steps 2/5).  The first m-1 macro steps are the
// RK bootstrap (readings R5/R6).  One macro step is captured once per ring/double-buffer
// phase as a CUDA graph and replayed.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

#include "dist.h"
#include "kernels.cuh"
#include "mrab_internal.h"

using namespace mrab;

static thread_local std::string g_last_error;

static mrab_status fail(mrab_status st, const std::string& msg) {
    g_last_error = msg;
    return st;
}

#define CK(call)                                                                        \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess)                                                          \
            return fail(MRAB_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

struct mrab_plan {
    std::shared_ptr<Plan> P;
};

namespace {

struct MeshDev {
    double* Q[2] = {nullptr, nullptr};
    double* ring[kMaxHist] = {nullptr};
    double* FV = nullptr;
    int32_t* fvlist = nullptr;    // 3-D: the 8^3 tiles holding donor-stencil points (F^V there)
    int nfv = 0;
    int32_t* cblist = nullptr;    // 3-D: fvlist tiles and their face neighbours (intermediate donor states)
    int ncb = 0;
    double* FH = nullptr;         // 3-D two-pass RHS: contravariant fluxes [3][5][N]
    uint8_t* fvtile = nullptr;    // 3-D two-pass RHS: per 8^3 tile, SAT points inside (F^V written)
    Z3Table z3tab;                // 3-D: TMA tensor maps of the state-shaped buffers
    double* dstate = nullptr;
    double* kbuf[4] = {nullptr, nullptr, nullptr, nullptr};
    double* ystage = nullptr;
    double* J = nullptr;
    double* M = nullptr;
    uint16_t* cls = nullptr;
    int32_t* recv_slot = nullptr;
    int64_t* rpoint = nullptr;
    int32_t* rdonor = nullptr;
    int32_t* rbase = nullptr;
    double* rw = nullptr;
    int32_t* gorder = nullptr;    // 3-D: receivers in donor-box group order (box-staged gather)
    int32_t* ginfo = nullptr;     // 3-D: [G][6] group descriptors
    int ngroups = 0;
    double* qhat = nullptr;       // [S][nc][R]: one set per micro index j (batched gathers)
    double* fvhat = nullptr;      // [S][d(d+1)][R]
    int32_t* tiles = nullptr;     // 2-D: critical tiles (cover the donor box) then the bulk
    int32_t* tlist = nullptr;     // 2-D: all tiles, non-interior first (bit 31 = interior)
    int ncrit = 0, nbulk = 0;
    int ngen = 0;                 // non-interior tiles at the head of tlist
    DevMesh dm{};
};

struct Book {
    int head[kMaxMeshes];
    int cur[kMaxMeshes];
    int pending[kMaxMeshes];
};

struct Bump {
    char* base;
    size_t cap, off;
    void* take(size_t bytes) {
        off = (off + 255) & ~(size_t)255;
        if (off + bytes > cap) return nullptr;
        void* p = base + off;
        off += bytes;
        return p;
    }
};

}  // namespace

struct mrab_ctx {
    std::shared_ptr<Plan> P;
    cudaStream_t user = nullptr;
    cudaStream_t st = nullptr;
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    std::vector<MeshDev> md;
    Gas gas{};
    Book book{};
    int64_t macro = 0;            // macro steps taken (bootstrap included)
    int64_t boot_micro = 0;       // RK micro steps done
    std::vector<int64_t> evals;
    // graphs per phase
    int period = 1;
    std::vector<cudaGraphExec_t> graphs;
    std::vector<Book> book_after;
    std::vector<std::vector<int64_t>> evals_per_phase;
    int64_t launches_last = 0;
    int64_t launch_counter = 0;
    int64_t graph_k0 = 0;         // MRAB macro-step index the phase-0 graph was captured at
    // variable macro step (mrab_step_h): micro step of the macro step being issued
    // and the times of the ring entries relative to its start (valid once var_mode is set)
    // multi-GPU: meshes partitioned over ranks, donor data exchanged per RHS evaluation
    struct DistState {
        int rank = 0, nranks = 1;
        OwnerTable ot{};
        std::unique_ptr<Transport> tp;
        double* tmp = nullptr;    // receive staging (library-owned)
        size_t tmp_bytes = 0;
        std::string err;
        int64_t bytes_sent = 0, messages = 0;
    };
    std::unique_ptr<DistState> dist;
    int scheme = -1;              // MRAB scheme of this context, fixed by its first MRAB step
    bool sf_primed = false;       // slowest-first: R_s(t) sits uncommitted in the spare buffer
    bool var_mode = false;
    double h_cur = 0.0;
    double time_extra = 0.0;      // simulated time taken in variable steps
    int64_t macro_fixed = 0;      // macro steps taken at the plan's fixed step
    double ring_t[kMaxMeshes][kMaxHist] = {};
    // 2-D multi-stream schedule: one stream per mesh (priority by rate) + a gather stream
    // 2-D: meshes [0, G), the gather stream G, bulk launches of split meshes G+1+g;
    // 3-D: meshes [0, G), donor-preparation streams G+1+h, gather streams 2G+1+g
    cudaStream_t side[3 * kMaxMeshes + 1] = {};
    std::vector<cudaEvent_t> evpool;
    size_t evnext = 0;
    bool overlap = true;
    int* dflag = nullptr;          // device flag of the finite check (in the workspace)
    int bulk_ctas = 0;             // persistent CTAs of a bulk launch (0 = one per tile)
    unsigned long long* trace = nullptr;   // launch timeline buffer (mrab_set_trace)
};

// ----------------------------------------------------------------------------------------
// workspace layout
// ----------------------------------------------------------------------------------------
static size_t plan_bytes(const Plan& P, bool dry, mrab_ctx* ctx, Bump* bump, bool* ok) {
    size_t total = 0;
    auto take = [&](size_t bytes) -> void* {
        total += ((bytes + 255) & ~(size_t)255) + 256;
        if (dry) return nullptr;
        void* p = bump->take(bytes);
        if (!p) *ok = false;
        return p;
    };
    const int nc = P.nc, d = P.dim;
    for (size_t g = 0; g < P.meshes.size(); ++g) {
        const MeshPlan& m = P.meshes[g];
        const size_t N = (size_t)m.npts, R = m.rpoint.size();
        const size_t S = nc * N * sizeof(double);
        MeshDev* D = dry ? nullptr : &ctx->md[g];
        for (int b = 0; b < 2; ++b) {
            void* p = take(S);
            if (D) D->Q[b] = (double*)p;
        }
        for (int k = 0; k < P.history_m; ++k) {
            void* p = take(S);
            if (D) D->ring[k] = (double*)p;
        }
        {
            void* p = take((size_t)d * (d + 1) * N * sizeof(double));
            if (D) D->FV = (double*)p;
        }
        if (d == 3) {
            const size_t nt = (size_t)((m.n[0] + 7) / 8) * ((m.n[1] + 7) / 8) * ((m.n[2] + 7) / 8);
            void* b = take(nt * sizeof(int32_t));
            void* b2 = take(nt * sizeof(int32_t));
            void* f = P.opt.z3_fused ? nullptr : take((size_t)15 * N * sizeof(double));
            void* t = take(nt);
            if (D) {
                D->cblist = (int32_t*)b2;
                D->fvlist = (int32_t*)b;
                D->FH = (double*)f;
                D->fvtile = (uint8_t*)t;
            }
        }
        {
            void* p = take(S);
            if (D) D->dstate = (double*)p;
        }
        for (int k = 0; k < 4; ++k) {
            void* p = take(S);
            if (D) D->kbuf[k] = (double*)p;
        }
        {
            void* p = take(S);
            if (D) D->ystage = (double*)p;
        }
        if (!m.cartesian) {
            void* a = take(N * sizeof(double));
            void* b = take((size_t)d * d * N * sizeof(double));
            if (D) {
                D->J = (double*)a;
                D->M = (double*)b;
            }
        }
        {
            void* a = take(N * sizeof(uint16_t));
            void* b = take(N * sizeof(int32_t));
            if (D) {
                D->cls = (uint16_t*)a;
                D->recv_slot = (int32_t*)b;
            }
        }
        {
            size_t Rm = std::max<size_t>(R, 1);
            void* a = take(Rm * sizeof(int64_t));
            void* b = take(Rm * sizeof(int32_t));
            void* c = take(Rm * 3 * sizeof(int32_t));
            void* e = take(Rm * 12 * sizeof(double));
            void* f = take((size_t)P.S * Rm * nc * sizeof(double));
            void* h = take((size_t)P.S * Rm * d * (d + 1) * sizeof(double));
            void* go = d == 3 ? take(Rm * sizeof(int32_t)) : nullptr;
            void* gf = d == 3 ? take(Rm * 6 * sizeof(int32_t)) : nullptr;
            if (D) {
                D->gorder = (int32_t*)go;
                D->ginfo = (int32_t*)gf;
                D->rpoint = (int64_t*)a;
                D->rdonor = (int32_t*)b;
                D->rbase = (int32_t*)c;
                D->rw = (double*)e;
                D->qhat = (double*)f;
                D->fvhat = (double*)h;
            }
        }
        if (d == 2) {
            int tx, ty;
            rhs2d_tile_shape_for(m.n, m.cartesian ? 1 : 0, &tx, &ty);
            const size_t nt = (size_t)((m.n[0] + tx - 1) / tx) * ((m.n[1] + ty - 1) / ty);
            void* a = take(nt * sizeof(int32_t));
            void* b = take(nt * sizeof(int32_t));
            if (D) {
                D->tiles = (int32_t*)a;
                D->tlist = (int32_t*)b;
            }
        }
    }
    {
        void* f = take(256);
        if (!dry) ctx->dflag = (int*)f;
    }
    return total + 1024;
}

// ----------------------------------------------------------------------------------------
// launches
// ----------------------------------------------------------------------------------------
static Box whole_box(const MeshPlan& m) {
    Box b{};
    for (int k = 0; k < 3; ++k) {
        b.lo[k] = 0;
        b.hi[k] = m.n[k] - 1;
    }
    return b;
}

static Box make_box(const int* lo, const int* hi) {
    Box b{};
    for (int k = 0; k < 3; ++k) {
        b.lo[k] = lo[k];
        b.hi[k] = hi[k];
    }
    return b;
}

static DonorSet make_ds(mrab_ctx* c, const double* const* state_of) {
    const Plan& P = *c->P;
    DonorSet ds{};
    for (size_t h = 0; h < P.meshes.size(); ++h) {
        ds.state[h] = state_of[h];
        ds.fv[h] = c->md[h].FV;
        for (int k = 0; k < 3; ++k) ds.n[h][k] = P.meshes[h].n[k];
        ds.npts[h] = P.meshes[h].npts;
    }
    return ds;
}

// gather for the receivers of mesh g (3-D; the 2-D RHS kernel gathers inline);
// state_of[d] = state array of donor d at the evaluation time
static void issue_interp(mrab_ctx* c, int g, const double* const* state_of, bool force = false) {
    const Plan& P = *c->P;
    MeshDev& D = c->md[g];
    const MeshPlan& m = P.meshes[g];
    if (m.rpoint.empty() || (P.dim == 2 && !force)) return;
    RecvList rl{};
    rl.n = (int64_t)m.rpoint.size();
    rl.point = D.rpoint;
    rl.donor = D.rdonor;
    rl.base = D.rbase;
    rl.w = D.rw;
    rl.qhat = D.qhat;
    rl.fvhat = D.fvhat;
    rl.gorder = D.gorder;
    rl.ginfo = D.ginfo;
    rl.ngroups = D.ngroups;
    launch_interp(P.viscous, rl, make_ds(c, state_of), c->st);
    c->launch_counter++;
}

// 2-D: one launch gathers the donor data of every receiver of the meshes in `evaluating`;
// donor states are formed on the fly from `ss`.
static double* qhat_set(mrab_ctx* c, int g, int j) {
    const MeshPlan& mp = c->P->meshes[g];
    const size_t R = std::max<size_t>(mp.rpoint.size(), 1);
    return c->md[g].qhat + (size_t)j * R * c->P->nc;
}
static double* fvhat_set(mrab_ctx* c, int g, int j) {
    const MeshPlan& mp = c->P->meshes[g];
    const size_t R = std::max<size_t>(mp.rpoint.size(), 1);
    const int d = c->P->dim;
    return c->md[g].fvhat + (size_t)j * R * d * (d + 1);
}

// one k_donor2d launch for the gather tasks (receiving mesh g, micro index j, state set)
struct GatherTask {
    int g, j, set;
};
static void issue_donor2d_tasks(mrab_ctx* c, const std::vector<GatherTask>& tasks,
                                const SrcSets& sets, cudaStream_t st) {
    const Plan& P = *c->P;
    RecvTask rt{};
    rt.nmesh = 0;
    rt.off[0] = 0;
    for (const GatherTask& t : tasks) {
        const MeshPlan& mp = P.meshes[t.g];
        if (mp.rpoint.empty()) continue;
        MeshDev& D = c->md[t.g];
        const int k = rt.nmesh++;
        rt.rdonor[k] = D.rdonor;
        rt.rbase[k] = D.rbase;
        rt.rw[k] = D.rw;
        rt.qhat[k] = qhat_set(c, t.g, t.j);
        rt.fvhat[k] = fvhat_set(c, t.g, t.j);
        rt.nrecv[k] = (int64_t)mp.rpoint.size();
        rt.set[k] = t.set;
        rt.off[k + 1] = rt.off[k] + rt.nrecv[k];
    }
    if (rt.nmesh == 0) return;
    rt.trace = c->trace;
    rt.trace_tag = (2 << 12) | (tasks[0].g << 8) | (tasks[0].j & 0xff);
    MeshTable mt{};
    for (size_t h = 0; h < P.meshes.size(); ++h) mt.m[h] = c->md[h].dm;
    launch_donor2d(rt, sets, mt, c->gas, st);
    c->launch_counter++;
}

static void issue_donor2d(mrab_ctx* c, const std::vector<int>& evaluating, const SrcSet& ss) {
    std::vector<GatherTask> tasks;
    for (int g : evaluating) tasks.push_back({g, 0, 0});
    SrcSets sets{};
    sets.s[0] = ss;
    issue_donor2d_tasks(c, tasks, sets, c->st);
}

static SrcSet plain_states(mrab_ctx* c, const double* const* state_of) {
    SrcSet ss{};
    for (size_t h = 0; h < c->P->meshes.size(); ++h) {
        ss.base[h] = state_of[h];
        ss.nsrc[h] = 0;
    }
    return ss;
}

static void issue_visc(mrab_ctx* c, int g, const double* Q, const Box& box) {
    const Plan& P = *c->P;
    if (!P.viscous) return;
    launch_visc(c->md[g].dm, Q, c->md[g].FV, box, nullptr, 0, c->gas, c->st);
    c->launch_counter++;
}

// 3-D: Cartesian viscous fluxes of donor mesh g at its current (stepping) state, on the 8^3
// tiles holding the donor stencils the gathers read (the fused RHS kernel keeps its own F^V
// on chip)
static void issue_step_visc(mrab_ctx* c, int g, const double* Q) {
    const Plan& P = *c->P;
    MeshDev& D = c->md[g];
    if (!P.viscous || P.dim != 3 || D.nfv == 0) return;
    launch_visc(D.dm, Q, D.FV, Box{}, D.fvlist, D.nfv, c->gas, c->st);
    c->launch_counter++;
}

// every mesh evaluated at the given states (RK stages, the rhs hook): donor data for all
static void issue_all_donors(mrab_ctx* c, const double* const* state_of) {
    const int G = (int)c->P->meshes.size();
    if (c->P->dim == 2) {
        std::vector<int> all(G);
        std::iota(all.begin(), all.end(), 0);
        issue_donor2d(c, all, plain_states(c, state_of));
        return;
    }
    for (int g = 0; g < G; ++g) issue_step_visc(c, g, state_of[g]);
    for (int g = 0; g < G; ++g) issue_interp(c, g, state_of);
}

static void issue_rhs(mrab_ctx* c, int g, const double* Q, const Epilogue& ep,
                      const double* const* state_of) {
    launch_rhs(c->P->dim, c->md[g].dm, Q, c->gas, ep, make_ds(c, state_of), c->st);
    c->launch_counter++;
}

// ----------------------------------------------------------------------------------------
// step size and AB weights of the macro step being issued: the plan's tables (fixed step), or
// -- variable macro step, P:581-583 -- eq:vandermonde with the actual history node times
// ----------------------------------------------------------------------------------------
static double h_micro(const mrab_ctx* c) { return c->var_mode ? c->h_cur : c->P->h; }

// weights (oldest first, m entries) of y = base + h_g sum_k w_k R_k over [0, (j - th)/s_g] for
// mesh g at micro index j, from its ring as it stands (newest entry at its last step th)
static void weights_partial(const mrab_ctx* c, int g, int j, double* w) {
    const Plan& P = *c->P;
    const int m = P.history_m, sg = P.meshes[g].s;
    if (!c->var_mode) {
        for (int k = 0; k < m; ++k) w[k] = P.coef[g][j % sg][k];
        return;
    }
    const double hg = c->h_cur * sg;
    const int head = c->book.head[g];
    const double tg = c->ring_t[g][head];
    double nodes[kMaxHist];
    for (int k = 0; k < m; ++k) {
        const int slot = ((head - (m - 1) + k) % m + m) % m;
        nodes[k] = (c->ring_t[g][slot] - tg) / hg;
    }
    nodes[m - 1] = 0.0;
    ab_weights(nodes, m, P.order_n, 0.0, (double)(j % sg) / sg, w, nullptr);
}

// weights of the full step mesh g takes at micro index j: its m - 1 newest ring entries and
// the evaluation at j (node 0), over [0, 1] in units of h_g
static void weights_full(const mrab_ctx* c, int g, int j, double* w) {
    const Plan& P = *c->P;
    const int m = P.history_m, sg = P.meshes[g].s;
    if (!c->var_mode) {
        for (int k = 0; k < m; ++k) w[k] = P.coef[g][sg][k];
        return;
    }
    const double hg = c->h_cur * sg;
    const int head = c->book.head[g];
    const double tg = j * c->h_cur;
    double nodes[kMaxHist];
    for (int k = 0; k < m - 1; ++k) {
        const int slot = ((head - (m - 2) + k) % m + m) % m;
        nodes[k] = (c->ring_t[g][slot] - tg) / hg;
    }
    nodes[m - 1] = 0.0;
    ab_weights(nodes, m, P.order_n, 0.0, 1.0, w, nullptr);
}

// bookkeeping of a push by mesh g at micro index j
static void note_push(mrab_ctx* c, int g, int j, int newslot) {
    if (c->var_mode) c->ring_t[g][newslot] = j * c->h_cur;
}

// 3-D: donor data of mesh g at micro index j of the macro step where g does not step: the
// intermediate state base + h_g sum_k beta_k^(j) R_k (MRAB Steps 2/5) and its
// Cartesian viscous fluxes, formed into dstate / FV on the donor-stencil tiles (and their
// face neighbours for the state: the viscous pass reads tile + 3 along each axis)
static void issue_partial_donor_w(mrab_ctx* c, int g, cudaStream_t st, const double* base, int nsrc,
                                  const double* const* src, const double* cs) {
    const Plan& P = *c->P;
    MeshDev& D = c->md[g];
    launch_combine_tiles(P.nc, D.dm, P.viscous ? D.cblist : D.fvlist, P.viscous ? D.ncb : D.nfv, base, nsrc,
                         src, cs, D.dstate, st);
    c->launch_counter++;
    if (P.viscous && D.nfv > 0) {
        launch_visc(D.dm, D.dstate, D.FV, Box{}, D.fvlist, D.nfv, c->gas, st);
        c->launch_counter++;
    }
}

static void issue_partial_donor(mrab_ctx* c, int g, int j, cudaStream_t st, const double* base = nullptr) {
    const Plan& P = *c->P;
    MeshDev& D = c->md[g];
    const MeshPlan& mp = P.meshes[g];
    const int m = P.history_m;
    const double hg = h_micro(c) * mp.s;
    const double* src[kMaxHist];
    double cs[kMaxHist], w[kMaxHist];
    weights_partial(c, g, j, w);
    for (int k = 0; k < m; ++k) {
        int slot = ((c->book.head[g] - (m - 1) + k) % m + m) % m;   // oldest first
        src[k] = D.ring[slot];
        cs[k] = hg * w[k];
    }
    if (!base) base = D.Q[c->book.cur[g]];
    issue_partial_donor_w(c, g, st, base, m, src, cs);
}

// one MRAB macro step (host bookkeeping + launches)
static void issue_macro_step_dag2d(mrab_ctx* c);
static void issue_macro_step_dag3d(mrab_ctx* c);

static void issue_macro_step(mrab_ctx* c) {
    const Plan& P = *c->P;
    if (P.dim == 2) {
        issue_macro_step_dag2d(c);
        return;
    }
    if (P.opt.overlap3d) {
        issue_macro_step_dag3d(c);
        return;
    }
    const int G = (int)P.meshes.size(), m = P.history_m;
    for (int j = 0; j < P.S; ++j) {
        std::vector<int> stepping(G, 0), partial(G, 0);
        for (int g = 0; g < G; ++g) stepping[g] = (j % P.meshes[g].s) == 0;
        for (int g = 0; g < G; ++g) {
            if (stepping[g]) continue;
            for (int h = 0; h < G; ++h)
                if (stepping[h] && P.donor_of[g][h]) partial[g] = 1;
        }
        std::vector<const double*> state_of(G, nullptr);
        // 3-D two-pass RHS: the flux pass of every stepping mesh first (it writes F^V on the
        // SAT and donor-stencil tiles), then the gathers, then the divergence passes; the
        // one-pass kernel (Options::z3_fused) takes k_visc3d_x on the donor tiles instead
        bool two = !opts().z3_fused;
        for (int g = 0; g < G; ++g) two = two && c->md[g].FH;
        for (int g = 0; g < G; ++g) {
            MeshDev& D = c->md[g];
            if (stepping[g]) {
                if (c->book.pending[g]) {
                    c->book.cur[g] ^= 1;
                    c->book.pending[g] = 0;
                }
                const double* Q = D.Q[c->book.cur[g]];
                state_of[g] = Q;
                if (two) {
                    launch_flux3d(D.dm, Q, c->gas, c->st);
                    c->launch_counter++;
                } else {
                    bool read_now = false;
                    for (int h = 0; h < G; ++h) read_now = read_now || (h != g && stepping[h] && P.donor_of[g][h]);
                    if (read_now) issue_step_visc(c, g, Q);
                }
            } else if (partial[g]) {
                issue_partial_donor(c, g, j, c->st);
                state_of[g] = D.dstate;
            }
        }
        for (int g = 0; g < G; ++g)
            if (stepping[g]) issue_interp(c, g, state_of.data());
        for (int g = 0; g < G; ++g) {
            if (!stepping[g]) continue;
            MeshDev& D = c->md[g];
            const MeshPlan& mp = P.meshes[g];
            const double hg = h_micro(c) * mp.s;
            const int newslot = (c->book.head[g] + 1) % m;
            Epilogue ep{};
            ep.r_out = D.ring[newslot];
            ep.y_out = D.Q[c->book.cur[g] ^ 1];
            ep.base = D.Q[c->book.cur[g]];
            double al[kMaxHist];   // full step, oldest first
            weights_full(c, g, j, al);
            ep.c_new = hg * al[m - 1];
            ep.nsrc = m - 1;
            for (int k = 0; k < m - 1; ++k) {
                int slot = ((c->book.head[g] - (m - 2) + k) % m + m) % m;
                ep.src[k] = D.ring[slot];
                ep.csrc[k] = hg * al[k];
            }
            if (two) {
                launch_div3d_pass(D.dm, ep.base, c->gas, ep, c->st);
                c->launch_counter++;
            } else {
                issue_rhs(c, g, D.Q[c->book.cur[g]], ep, state_of.data());
            }
            c->book.head[g] = newslot;
            note_push(c, g, j, newslot);
            c->book.pending[g] = 1;
            c->evals[g]++;
        }
    }
}

// ----------------------------------------------------------------------------------------
// 2-D macro step as a multi-stream DAG (captured into the phase graph).
//
// Nodes: gather launches (k_donor2d, possibly batching several micro indices) and RHS
// launches (k_rhs2d, one per stepping mesh and micro index; a mesh whose intermediate states
// are read later in the step is split into the tiles covering its donor box -- "critical" --
// and the bulk, so the fast substeps only wait for the critical tiles while the bulk overlaps
// them: the single-GPU analogue of the paper's interleaved communication).
// Times are micro indices relative to the macro step start.
// ----------------------------------------------------------------------------------------
static cudaEvent_t dag_event(mrab_ctx* c) {
    if (c->evnext == c->evpool.size()) {
        cudaEvent_t e;
        cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        c->evpool.push_back(e);
    }
    return c->evpool[c->evnext++];
}

struct DagNode {
    int stream = -1;
    cudaEvent_t ev = nullptr;
};

static void dag_wait(mrab_ctx* c, int s, const DagNode& d) {
    if (d.ev && d.stream != s) cudaStreamWaitEvent(c->side[s], d.ev, 0);
}
static DagNode dag_done(mrab_ctx* c, int s) {
    DagNode n;
    n.stream = s;
    n.ev = dag_event(c);
    cudaEventRecord(n.ev, c->side[s]);
    return n;
}

static void issue_macro_step_dag2d(mrab_ctx* c) {
    const Plan& P = *c->P;
    const int G = (int)P.meshes.size(), m = P.history_m, S = P.S;
    const int GS = G;                       // index of the gather stream
    c->evnext = 0;
    // fork
    {
        cudaEvent_t e = dag_event(c);
        cudaEventRecord(e, c->st);
        for (int s = 0; s <= G; ++s) cudaStreamWaitEvent(c->side[s], e, 0);
    }
    // per mesh: which buffer holds which time, ring newest time
    int tq[kMaxMeshes][2], tring[kMaxMeshes];
    for (int g = 0; g < G; ++g) {
        const int sg = P.meshes[g].s;
        const int cur = c->book.cur[g];
        // at a macro boundary every mesh has a pending state (its last RHS was at -s_g)
        tq[g][cur] = -sg;
        tq[g][cur ^ 1] = 0;
        tring[g] = -sg;
    }
    auto buf_at = [&](int g, int t) -> int {
        if (tq[g][0] == t) return 0;
        if (tq[g][1] == t) return 1;
        return -1;
    };
    auto steps_at = [&](int g, int j) { return j % P.meshes[g].s == 0; };
    // does mesh h's intermediate state get read after micro index j in this step?
    auto partial_read_after = [&](int h, int j) {
        for (int jj = j + 1; jj < S; ++jj) {
            if (steps_at(h, jj)) break;
            for (int g = 0; g < G; ++g)
                if (steps_at(g, jj) && P.donor_of[h][g]) return true;
        }
        return false;
    };
    std::vector<DagNode> last_full(G), last_crit(G);
    std::vector<int> bulk_used(G, 0);
    std::vector<std::vector<DagNode>> readers(G);     // gather nodes that read mesh h
    std::vector<std::vector<int>> emitted(G, std::vector<int>(S, 0));
    std::vector<std::vector<DagNode>> gnode(G, std::vector<DagNode>(S));
    for (int j = 0; j < S; ++j) {
        // ---- gathers: all tasks (g, jj >= j) whose producers are already emitted ----
        std::vector<GatherTask> tasks;
        SrcSets sets{};
        int nsets = 0;
        std::vector<DagNode> deps;
        std::vector<int> readmesh(G, 0);
        for (int jj = j; jj < S; ++jj) {
            bool any = false;
            for (int g = 0; g < G; ++g) any = any || (steps_at(g, jj) && !emitted[g][jj]);
            if (!any) continue;
            // readiness of every donor of the meshes stepping at jj
            bool ready = true;
            for (int h = 0; h < G && ready; ++h) {
                bool needed = false;
                for (int g = 0; g < G; ++g) needed = needed || (steps_at(g, jj) && P.donor_of[h][g] && g != h);
                if (!needed) continue;
                if (steps_at(h, jj)) {
                    ready = buf_at(h, jj) >= 0 && (jj - P.meshes[h].s < j);
                } else {
                    const int th = jj - jj % P.meshes[h].s;
                    ready = th < j && tring[h] == th;
                }
            }
            if (!ready) {
                if (jj == j) ready = true;   // cannot happen (producers of j precede j)
                else continue;
            }
            if (nsets == 8) break;
            SrcSet& ss = sets.s[nsets];
            for (int h = 0; h < G; ++h) {
                ss.nsrc[h] = 0;
                if (steps_at(h, jj)) {
                    int b = buf_at(h, jj);
                    ss.base[h] = c->md[h].Q[b < 0 ? 0 : b];
                } else {
                    const MeshPlan& mh = P.meshes[h];
                    const int th = jj - jj % mh.s;
                    int b = buf_at(h, th);
                    ss.base[h] = c->md[h].Q[b < 0 ? 0 : b];
                    const double hg = h_micro(c) * mh.s;
                    ss.nsrc[h] = m;
                    double w[kMaxHist];
                    weights_partial(c, h, jj, w);
                    for (int k = 0; k < m; ++k) {
                        int slot = ((c->book.head[h] - (m - 1) + k) % m + m) % m;
                        ss.src[h][k] = c->md[h].ring[slot];
                        ss.c[h][k] = hg * w[k];
                    }
                }
            }
            for (int g = 0; g < G; ++g) {
                if (!steps_at(g, jj) || emitted[g][jj]) continue;
                tasks.push_back({g, jj, nsets});
                emitted[g][jj] = 1;
                for (int h = 0; h < G; ++h) {
                    if (!P.donor_of[h][g] || h == g) continue;
                    readmesh[h] = 1;
                    deps.push_back(steps_at(h, jj) ? last_full[h] : last_crit[h]);
                }
            }
            nsets++;
        }
        DagNode gn;
        if (!tasks.empty()) {
            for (auto& d : deps) dag_wait(c, GS, d);
            issue_donor2d_tasks(c, tasks, sets, c->side[GS]);
            gn = dag_done(c, GS);
            for (auto& t : tasks) gnode[t.g][t.j] = gn;
            for (int h = 0; h < G; ++h)
                if (readmesh[h]) readers[h].push_back(gn);
        }
        // ---- RHS + AB update of the meshes stepping at j ----
        for (int g = 0; g < G; ++g) {
            if (!steps_at(g, j)) continue;
            MeshDev& D = c->md[g];
            const MeshPlan& mp = P.meshes[g];
            if (c->book.pending[g]) {
                c->book.cur[g] ^= 1;
                c->book.pending[g] = 0;
            }
            dag_wait(c, g, gnode[g][j]);
            for (auto& r : readers[g]) dag_wait(c, g, r);     // WAR on ring slot / state buffer
            const double hg = h_micro(c) * mp.s;
            const int newslot = (c->book.head[g] + 1) % m;
            Epilogue ep{};
            ep.r_out = D.ring[newslot];
            ep.y_out = D.Q[c->book.cur[g] ^ 1];
            ep.base = D.Q[c->book.cur[g]];
            double al[kMaxHist];
            weights_full(c, g, j, al);
            ep.c_new = hg * al[m - 1];
            ep.nsrc = m - 1;
            for (int k = 0; k < m - 1; ++k) {
                int slot = ((c->book.head[g] - (m - 2) + k) % m + m) % m;
                ep.src[k] = D.ring[slot];
                ep.csrc[k] = hg * al[k];
            }
            DevMesh dm = D.dm;
            dm.qhat = qhat_set(c, g, j);
            dm.fvhat = fvhat_set(c, g, j);
            const DonorSet ds{};
            const bool split = c->overlap && D.ncrit > 0 && D.nbulk > 0 && partial_read_after(g, j);
            {
                // priorities travel with the launches into the graph: fastest meshes first
                int least = 0, greatest = 0;
                cudaDeviceGetStreamPriorityRange(&least, &greatest);
                int smin = S;
                for (auto& q : P.meshes) smin = std::min(smin, q.s);
                // launch priorities (honoured in the graph: UseNodePriority) whenever the schedule
                // overlaps meshes, so that fast substeps take SM slots ahead of bulk tiles
                ep.has_prio = c->overlap ? 1 : 0;
                ep.prio = mp.s == smin ? greatest : least;
            }
            ep.trace = c->trace;
            ep.trace_tag = (1 << 12) | (g << 8) | (j & 0xff);
            if (split) {
                // bulk tiles on the mesh's bulk stream, concurrent with the critical tiles;
                // the mesh's own stream joins both
                const int gb = G + 1 + g;
                bulk_used[g] = 1;
                const DagNode pre = dag_done(c, g);
                Epilogue e1 = ep;
                e1.tiles = D.tiles;
                e1.ntiles = D.ncrit;
                launch_rhs(2, dm, ep.base, c->gas, e1, ds, c->side[g]);
                last_crit[g] = dag_done(c, g);
                dag_wait(c, gb, pre);
                Epilogue e2 = ep;
                e2.tiles = D.tiles + D.ncrit;
                e2.ntiles = D.nbulk;
                e2.persist = c->bulk_ctas;
                e2.trace_tag = (3 << 12) | (g << 8) | (j & 0xff);
                launch_rhs(2, dm, ep.base, c->gas, e2, ds, c->side[gb]);
                c->launch_counter += 2;
                dag_wait(c, g, dag_done(c, gb));
                last_full[g] = dag_done(c, g);
            } else {
                launch_rhs(2, dm, ep.base, c->gas, ep, ds, c->side[g]);
                c->launch_counter++;
                last_full[g] = dag_done(c, g);
                last_crit[g] = last_full[g];
            }
            readers[g].clear();
            c->book.head[g] = newslot;
            note_push(c, g, j, newslot);
            c->book.pending[g] = 1;
            c->evals[g]++;
            tring[g] = j;
            tq[g][c->book.cur[g] ^ 1] = j + mp.s;
        }
    }
    // join (bulk streams only if they joined the step)
    for (int s = 0; s <= 2 * G; ++s) {
        if (s > G && !bulk_used[s - G - 1]) continue;
        cudaEvent_t e = dag_event(c);
        cudaEventRecord(e, c->side[s]);
        cudaStreamWaitEvent(c->st, e, 0);
    }
}


// ----------------------------------------------------------------------------------------
// 3-D macro step as a multi-stream task flow (captured into the phase graph).
//
// Launches are issued in a valid sequential order; every launch declares the buffers it reads
// and writes, and the tracker below inserts the event waits that keep exactly those
// dependencies (RAW, WAR, WAW) between streams.  Streams: one per mesh for its RHS (both
// passes), one per donor mesh for the preparation of its donor data (intermediate state on
// the donor box, Cartesian viscous fluxes), one per receiving mesh for its gathers.  The
// donor data of a micro index jj is prepared and gathered as soon as its producers have been
// issued (into the qhat/fvhat set jj of the receiver), so the latency-bound small kernels of
// the fast substeps run beside the large RHS launches instead of between them -- the
// single-GPU analogue of the paper's interleaved interpolation exchange.
// Priorities (per node): preparation and gathers highest, then the meshes by rate.
// ----------------------------------------------------------------------------------------
namespace {
struct Flow {
    mrab_ctx* c;
    struct Res {
        DagNode w;
        std::vector<DagNode> r;
    };
    std::map<const void*, Res> res;
    std::vector<const void*> rd, wr;
    int stream = -1;
    std::vector<char> used;
    cudaEvent_t fork = nullptr;
    explicit Flow(mrab_ctx* c_) : c(c_), used(3 * kMaxMeshes + 1, 0) {}
    // waits of a launch on stream s that reads `reads` and writes `writes`
    void begin(int s, std::initializer_list<const void*> reads, std::initializer_list<const void*> writes) {
        stream = s;
        if (!used[s]) {   // a stream joins the step (and the capture) at its first launch
            cudaStreamWaitEvent(c->side[s], fork, 0);
            used[s] = 1;
        }
        rd.assign(reads.begin(), reads.end());
        wr.assign(writes.begin(), writes.end());
        for (const void* k : rd)
            if (k) dag_wait(c, s, res[k].w);
        for (const void* k : wr) {
            if (!k) continue;
            Res& R = res[k];
            dag_wait(c, s, R.w);
            for (auto& n : R.r) dag_wait(c, s, n);
        }
    }
    void add_read(const void* k) {
        if (!k) return;
        dag_wait(c, stream, res[k].w);
        rd.push_back(k);
    }
    void end() {
        const DagNode n = dag_done(c, stream);
        for (const void* k : rd)
            if (k) res[k].r.push_back(n);
        for (const void* k : wr) {
            if (!k) continue;
            Res& R = res[k];
            R.w = n;
            R.r.clear();
        }
    }
};
}  // namespace

static void issue_macro_step_dag3d(mrab_ctx* c) {
    const Plan& P = *c->P;
    const int G = (int)P.meshes.size(), m = P.history_m, S = P.S;
    c->evnext = 0;
    Flow F(c);
    auto sp = [&](int h) { return G + 1 + h; };        // donor-preparation stream of mesh h
    auto sg = [&](int g) { return 2 * G + 1 + g; };    // gather stream of mesh g
    int least = 0, greatest = 0;
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    // priority of a mesh's RHS by rate rank (fastest just below the small kernels)
    std::vector<int> ranks;
    for (auto& q : P.meshes) ranks.push_back(q.s);
    std::sort(ranks.begin(), ranks.end());
    ranks.erase(std::unique(ranks.begin(), ranks.end()), ranks.end());
    auto mesh_prio = [&](int g) {
        const int r = (int)(std::find(ranks.begin(), ranks.end(), P.meshes[g].s) - ranks.begin());
        return std::min(least, greatest + 1 + r);
    };
    F.fork = dag_event(c);
    cudaEventRecord(F.fork, c->st);
    int tq[kMaxMeshes][2], tring[kMaxMeshes];
    for (int g = 0; g < G; ++g) {
        const int sgm = P.meshes[g].s;
        const int cur = c->book.cur[g];
        tq[g][cur] = -sgm;
        tq[g][cur ^ 1] = 0;
        tring[g] = -sgm;
    }
    auto buf_at = [&](int g, int t) -> int {
        if (tq[g][0] == t) return 0;
        if (tq[g][1] == t) return 1;
        return -1;
    };
    auto steps_at = [&](int g, int j) { return j % P.meshes[g].s == 0; };
    std::vector<std::vector<int>> emitted(G, std::vector<int>(S, 0));
    auto stamp = [&](int s, int kind, int g, int j, int end) {
        if (c->trace) launch_stamp(c->trace, (end << 15) | (kind << 12) | (g << 8) | (j & 0xff), c->side[s]);
    };
    bool two = !opts().z3_fused;
    for (int g = 0; g < G; ++g) two = two && c->md[g].FH;
    for (int j = 0; j < S; ++j) {
        // ---- flux pass of the meshes stepping at j (two-pass RHS): Fhat everywhere, F^V on the
        //      SAT and donor-stencil tiles ----
        for (int g = 0; g < G; ++g) {
            if (!steps_at(g, j)) continue;
            MeshDev& D = c->md[g];
            if (c->book.pending[g]) {
                c->book.cur[g] ^= 1;
                c->book.pending[g] = 0;
            }
            if (!two) continue;
            const double* Q = D.Q[c->book.cur[g]];
            F.begin(g, {Q}, {D.FV, D.FH});
            set_launch_priority(1, mesh_prio(g));
            stamp(g, 4, g, j, 0);
            launch_flux3d(D.dm, Q, c->gas, c->side[g]);
            stamp(g, 4, g, j, 1);
            c->launch_counter++;
            F.end();
        }
        // ---- donor data of every micro index jj >= j whose producers have been issued ----
        for (int jj = j; jj < S; ++jj) {
            std::vector<int> recv;
            for (int g = 0; g < G; ++g)
                if (steps_at(g, jj) && !emitted[g][jj]) recv.push_back(g);
            if (recv.empty()) continue;
            std::vector<int> need(G, 0);
            for (int g : recv)
                for (int h = 0; h < G; ++h)
                    if (h != g && P.donor_of[h][g] && !P.meshes[g].rpoint.empty()) need[h] = 1;
            bool ready = true;
            for (int h = 0; h < G && ready; ++h) {
                if (!need[h]) continue;
                if (steps_at(h, jj)) {
                    // a stepping donor's F^V comes from its flux pass at jj (two-pass), else from
                    // k_visc3d_x on its state, known once its previous RHS has been issued
                    ready = two ? jj == j : (buf_at(h, jj) >= 0 && (jj - P.meshes[h].s < j));
                } else {
                    const int th = jj - jj % P.meshes[h].s;
                    ready = th < j && tring[h] == th;
                }
            }
            if (!ready) continue;   // (jj == j is always ready: its producers precede j)
            set_launch_priority(1, greatest);
            std::vector<const double*> state_of(G, nullptr);
            for (int h = 0; h < G; ++h) {
                MeshDev& D = c->md[h];
                const MeshPlan& mh = P.meshes[h];
                if (steps_at(h, jj)) {
                    const int b = buf_at(h, jj);
                    state_of[h] = D.Q[b < 0 ? c->book.cur[h] : b];
                    if (!two && need[h] && P.viscous && D.nfv > 0) {
                        F.begin(sp(h), {state_of[h]}, {D.FV});
                        stamp(sp(h), 6, h, jj, 0);
                        launch_visc(D.dm, state_of[h], D.FV, Box{}, D.fvlist, D.nfv, c->gas, c->side[sp(h)]);
                        stamp(sp(h), 6, h, jj, 1);
                        c->launch_counter++;
                        F.end();
                    }
                } else if (need[h]) {
                    const int th = jj - jj % mh.s;
                    const int b = buf_at(h, th);
                    const double* base = D.Q[b < 0 ? c->book.cur[h] : b];
                    F.begin(sp(h), {base}, {D.dstate, D.FV});
                    for (int k = 0; k < m; ++k) F.add_read(D.ring[k]);
                    stamp(sp(h), 6, h, jj, 0);
                    issue_partial_donor(c, h, jj, c->side[sp(h)], base);
                    stamp(sp(h), 6, h, jj, 1);
                    F.end();
                    state_of[h] = D.dstate;
                } else {
                    state_of[h] = D.Q[c->book.cur[h]];   // not read
                }
            }
            for (int g : recv) {
                emitted[g][jj] = 1;
                MeshDev& D = c->md[g];
                const MeshPlan& mg = P.meshes[g];
                if (mg.rpoint.empty()) continue;
                RecvList rl{};
                rl.n = (int64_t)mg.rpoint.size();
                rl.point = D.rpoint;
                rl.donor = D.rdonor;
                rl.base = D.rbase;
                rl.w = D.rw;
                rl.qhat = qhat_set(c, g, jj);
                rl.fvhat = fvhat_set(c, g, jj);
                rl.gorder = D.gorder;
                rl.ginfo = D.ginfo;
                rl.ngroups = D.ngroups;
                F.begin(sg(g), {}, {rl.qhat});
                for (int h = 0; h < G; ++h) {
                    if (h == g || !P.donor_of[h][g]) continue;
                    F.add_read(state_of[h]);
                    if (P.viscous) F.add_read(c->md[h].FV);
                }
                stamp(sg(g), 7, g, jj, 0);
                launch_interp(P.viscous, rl, make_ds(c, state_of.data()), c->side[sg(g)]);
                stamp(sg(g), 7, g, jj, 1);
                c->launch_counter++;
                F.end();
            }
        }
        // ---- divergence + SAT + AB update of the meshes stepping at j ----
        for (int g = 0; g < G; ++g) {
            if (!steps_at(g, j)) continue;
            MeshDev& D = c->md[g];
            const MeshPlan& mp = P.meshes[g];
            const double hg = h_micro(c) * mp.s;
            const int newslot = (c->book.head[g] + 1) % m;
            Epilogue ep{};
            ep.r_out = D.ring[newslot];
            ep.y_out = D.Q[c->book.cur[g] ^ 1];
            ep.base = D.Q[c->book.cur[g]];
            double al[kMaxHist];
            weights_full(c, g, j, al);
            ep.c_new = hg * al[m - 1];
            ep.nsrc = m - 1;
            double* qh = qhat_set(c, g, j);
            // (the divergence pass reads FV at the SAT points and FH; declared as writes so that
            // it also orders against the gathers still reading FV)
            F.begin(g, {ep.base, mp.rpoint.empty() ? nullptr : qh}, {ep.r_out, ep.y_out, D.FV, D.FH});
            for (int k = 0; k < m - 1; ++k) {
                const int slot = ((c->book.head[g] - (m - 2) + k) % m + m) % m;
                ep.src[k] = D.ring[slot];
                ep.csrc[k] = hg * al[k];
                F.add_read(ep.src[k]);
            }
            DevMesh dm = D.dm;
            dm.qhat = qh;
            dm.fvhat = fvhat_set(c, g, j);
            ep.has_prio = 1;
            ep.prio = mesh_prio(g);
            set_launch_priority(1, ep.prio);
            stamp(g, 5, g, j, 0);
            if (two) launch_div3d_pass(dm, ep.base, c->gas, ep, c->side[g]);
            else launch_rhs(3, dm, ep.base, c->gas, ep, DonorSet{}, c->side[g]);
            stamp(g, 5, g, j, 1);
            c->launch_counter++;
            F.end();
            c->book.head[g] = newslot;
            note_push(c, g, j, newslot);
            c->book.pending[g] = 1;
            c->evals[g]++;
            tring[g] = j;
            tq[g][c->book.cur[g] ^ 1] = j + mp.s;
        }
    }
    set_launch_priority(0, 0);
    // join
    for (int s = 0; s <= 3 * G; ++s) {
        if (!c->side[s] || !F.used[s]) continue;
        cudaEvent_t e = dag_event(c);
        cudaEventRecord(e, c->side[s]);
        cudaStreamWaitEvent(c->st, e, 0);
    }
}

// ----------------------------------------------------------------------------------------
// Two-rate slowest-first macro step (reading R-SF): the slow meshes' RHS at t + H is
// evaluated first, with the fast meshes' states extrapolated over the whole macro step; the
// fast substeps then see slow states from the old extrapolant (reextrap = false) or from the
// one re-formed with R_s(t + H) as its newest node (reextrap = true).  Same kernels, issued
// directly on the context stream (weights are launch arguments).
// In the fused, deferred formulation a slow mesh holds s(t) and s(t + H) in its
// two state buffers and R_s(t + H) uncommitted in a spare buffer; at the start of the next macro
// step the spare is swapped into the ring and s(t + 2H) is formed by a pointwise combination.
// ----------------------------------------------------------------------------------------
static mrab_status issue_macro_step_sf(mrab_ctx* c, bool reextrap) {
    const Plan& P = *c->P;
    const int G = (int)P.meshes.size(), m = P.history_m, S = P.S, n = P.order_n;
    const double h = P.h, H = P.h * S;
    std::vector<int> slow, fast, all(G);
    std::iota(all.begin(), all.end(), 0);
    for (int g = 0; g < G; ++g) (P.meshes[g].s == S ? slow : fast).push_back(g);
    double w_full[kMaxHist], w_long[kMaxHist], nodes[kMaxHist];
    for (int k = 0; k < m; ++k) nodes[k] = -(double)(m - 1) + k;
    ab_weights(nodes, m, n, 0.0, 1.0, w_full, nullptr);
    ab_weights(nodes, m, n, 0.0, (double)S, w_long, nullptr);
    auto ring_oldest_first = [&](int g, const double** src) {
        for (int k = 0; k < m; ++k) src[k] = c->md[g].ring[((c->book.head[g] - (m - 1) + k) % m + m) % m];
    };
    // gather for the receivers of `recv` with donor states given per mesh as base + sum cs src
    auto gather = [&](const std::vector<int>& recv, const SrcSet& ss) {
        if (P.dim == 2) {
            issue_donor2d(c, recv, ss);
            return;
        }
        std::vector<const double*> state_of(G);
        for (int hh = 0; hh < G; ++hh) {
            bool need = false;
            for (int g : recv) need = need || (hh != g && P.donor_of[hh][g] && !P.meshes[g].rpoint.empty());
            state_of[hh] = ss.base[hh];
            if (!need) continue;
            MeshDev& D = c->md[hh];
            if (ss.nsrc[hh] == 0) {
                if (P.viscous && D.nfv > 0) {
                    launch_visc(D.dm, ss.base[hh], D.FV, Box{}, D.fvlist, D.nfv, c->gas, c->st);
                    c->launch_counter++;
                }
            } else {
                issue_partial_donor_w(c, hh, c->st, ss.base[hh], ss.nsrc[hh], ss.src[hh], ss.c[hh]);
                state_of[hh] = D.dstate;
            }
        }
        for (int g : recv) issue_interp(c, g, state_of.data());
    };
    // fused evaluation + AB step of mesh g at its current state (weights w_full, step hg)
    auto fused_step = [&](int g) {
        MeshDev& D = c->md[g];
        const double hg = h * P.meshes[g].s;
        const int newslot = (c->book.head[g] + 1) % m;
        Epilogue ep{};
        ep.r_out = D.ring[newslot];
        ep.y_out = D.Q[c->book.cur[g] ^ 1];
        ep.base = D.Q[c->book.cur[g]];
        ep.c_new = hg * w_full[m - 1];
        ep.nsrc = m - 1;
        for (int k = 0; k < m - 1; ++k) {
            ep.src[k] = D.ring[((c->book.head[g] - (m - 2) + k) % m + m) % m];
            ep.csrc[k] = hg * w_full[k];
        }
        std::vector<const double*> dummy(G, nullptr);
        issue_rhs(c, g, ep.base, ep, dummy.data());
        c->book.head[g] = newslot;
        c->book.pending[g] = 1;
        c->evals[g]++;
    };
    SrcSet plain{};
    // ---- j = 0 ----
    for (int g = 0; g < G; ++g)
        if (c->book.pending[g]) {
            c->book.cur[g] ^= 1;
            c->book.pending[g] = 0;
        }
    for (int g = 0; g < G; ++g) {
        plain.base[g] = c->md[g].Q[c->book.cur[g]];
        plain.nsrc[g] = 0;
    }
    if (!c->sf_primed) {
        gather(all, plain);
        for (int g = 0; g < G; ++g) fused_step(g);
    } else {
        for (int g : slow) {
            // commit R_s(t) (evaluated early in the previous macro step), then s(t + H)
            MeshDev& D = c->md[g];
            const int newslot = (c->book.head[g] + 1) % m;
            std::swap(D.ring[newslot], D.kbuf[0]);
            c->book.head[g] = newslot;
            const double* src[kMaxHist];
            double cs[kMaxHist];
            ring_oldest_first(g, src);
            for (int k = 0; k < m; ++k) cs[k] = H * w_full[k];
            launch_combine(P.nc, D.dm, whole_box(P.meshes[g]), D.Q[c->book.cur[g]], m, src, cs,
                           D.Q[c->book.cur[g] ^ 1], c->st);
            c->launch_counter++;
            c->book.pending[g] = 1;
        }
        gather(fast, plain);
        for (int g : fast) fused_step(g);
    }
    // ---- the slow meshes' RHS at t + H, fast donors extrapolated over [t, t + H] ----
    {
        SrcSet ss{};
        for (int g : fast) {
            ss.base[g] = c->md[g].Q[c->book.cur[g]];      // f(t); f(t + h) is pending
            ss.nsrc[g] = m;
            ring_oldest_first(g, ss.src[g]);
            for (int k = 0; k < m; ++k) ss.c[g][k] = h * w_long[k];
        }
        for (int g : slow) {
            ss.base[g] = c->md[g].Q[c->book.cur[g] ^ 1];  // s(t + H)
            ss.nsrc[g] = 0;
        }
        gather(slow, ss);
        for (int g : slow) {
            MeshDev& D = c->md[g];
            Epilogue ep{};
            ep.r_out = D.kbuf[0];
            std::vector<const double*> dummy(G, nullptr);
            issue_rhs(c, g, ss.base[g], ep, dummy.data());
            c->evals[g]++;
        }
    }
    // ---- fast substeps j = 1 .. S-1 ----
    for (int j = 1; j < S; ++j) {
        SrcSet ss{};
        for (int g : fast) {
            c->book.cur[g] ^= 1;
            c->book.pending[g] = 0;
            ss.base[g] = c->md[g].Q[c->book.cur[g]];
            ss.nsrc[g] = 0;
        }
        for (int g : slow) {
            MeshDev& D = c->md[g];
            ss.base[g] = D.Q[c->book.cur[g]];             // s(t)
            ss.nsrc[g] = m;
            double w[kMaxHist];
            if (reextrap) {
                // nodes -(m-2), ..., 0, 1: the m-1 newest committed entries and R_s(t + H)
                double nd[kMaxHist];
                for (int k = 0; k < m; ++k) nd[k] = -(double)(m - 2) + k;
                ab_weights(nd, m, n, 0.0, (double)j / S, w, nullptr);
                for (int k = 0; k < m - 1; ++k)
                    ss.src[g][k] = D.ring[((c->book.head[g] - (m - 2) + k) % m + m) % m];
                ss.src[g][m - 1] = D.kbuf[0];
            } else {
                ab_weights(nodes, m, n, 0.0, (double)j / S, w, nullptr);
                ring_oldest_first(g, ss.src[g]);
            }
            for (int k = 0; k < m; ++k) ss.c[g][k] = H * w[k];
        }
        gather(fast, ss);
        for (int g : fast) fused_step(g);
    }
    c->sf_primed = true;
    CK(cudaGetLastError());
    return MRAB_OK;
}

// ----------------------------------------------------------------------------------------
// Multi-GPU: the meshes are partitioned over the ranks (weight = active points x RHS
// evaluations per macro step, the paper's load-balance lesson); each
// rank steps the meshes it owns.  Per RHS evaluation the only exchange is the interpolated donor
// data: the rank owning a donor mesh forms that mesh's donor state and viscous
// fluxes, interpolates them at the receivers of the evaluating mesh and sends the result
// (qhat [nc][R], fvhat [d(d+1)][R]) to the rank owning the receivers, which keeps the rows whose
// donor mesh the sender owns.  One grouped exchange per evaluation round.
// ----------------------------------------------------------------------------------------
static bool owns(const mrab_ctx* c, int g) { return !c->dist || c->dist->ot.owner[g] == c->dist->rank; }

static void dist_gather(mrab_ctx* c, const std::vector<int>& recv, const SrcSet& ss) {
    const Plan& P = *c->P;
    const int G = (int)P.meshes.size(), d = P.dim, nc = P.nc;
    mrab_ctx::DistState& D = *c->dist;
    const int me = D.rank;
    auto rank_donates = [&](int q, int g) {
        for (int h = 0; h < G; ++h)
            if (h != g && P.donor_of[h][g] && D.ot.owner[h] == q) return true;
        return false;
    };
    std::vector<int> mine;
    for (int g : recv)
        if (!P.meshes[g].rpoint.empty() && rank_donates(me, g)) mine.push_back(g);
    if (!mine.empty()) {
        if (d == 2) {
            issue_donor2d(c, mine, ss);
        } else {
            std::vector<const double*> state_of(G);
            for (int h = 0; h < G; ++h) {
                state_of[h] = ss.base[h];
                bool need = D.ot.owner[h] == me;
                if (need) {
                    need = false;
                    for (int g : mine) need = need || (h != g && P.donor_of[h][g]);
                }
                if (!need) continue;
                MeshDev& M = c->md[h];
                if (ss.nsrc[h] == 0) {
                    if (P.viscous && M.nfv > 0) {
                        launch_visc(M.dm, ss.base[h], M.FV, Box{}, M.fvlist, M.nfv, c->gas, c->st);
                        c->launch_counter++;
                    }
                } else {
                    issue_partial_donor_w(c, h, c->st, ss.base[h], ss.nsrc[h], ss.src[h], ss.c[h]);
                    state_of[h] = M.dstate;
                }
            }
            for (int g : mine) issue_interp(c, g, state_of.data());
        }
    }
    if (D.nranks == 1) return;
    const int rows_f = d * (d + 1);
    // receive staging: one slot per (mesh I own in recv, donating rank)
    struct Slot {
        int g, q;
        size_t off;
    };
    std::vector<Slot> slots;
    size_t need_bytes = 0;
    for (int g : recv) {
        const size_t R = P.meshes[g].rpoint.size();
        if (!R || D.ot.owner[g] != me) continue;
        for (int q = 0; q < D.nranks; ++q)
            if (q != me && rank_donates(q, g)) {
                slots.push_back({g, q, need_bytes});
                need_bytes += R * (nc + (P.viscous ? rows_f : 0)) * sizeof(double);
            }
    }
    if (need_bytes > D.tmp_bytes) {
        cudaStreamSynchronize(c->st);
        if (D.tmp) cudaFree(D.tmp);
        D.tmp = nullptr;
        if (cudaMalloc((void**)&D.tmp, need_bytes) != cudaSuccess) {
            D.err = "receive staging allocation failed";
            return;
        }
        D.tmp_bytes = need_bytes;
    }
    bool ok = D.tp->begin();
    for (int g : recv) {
        const size_t R = P.meshes[g].rpoint.size();
        if (!R) continue;
        const int og = D.ot.owner[g];
        MeshDev& M = c->md[g];
        for (int q = 0; q < D.nranks && ok; ++q) {
            if (q == og || !rank_donates(q, g)) continue;
            if (me == q) {
                ok = ok && D.tp->send(M.qhat, R * nc * sizeof(double), og, 2 * g, c->st);
                if (P.viscous) ok = ok && D.tp->send(M.fvhat, R * rows_f * sizeof(double), og, 2 * g + 1, c->st);
                D.bytes_sent += (int64_t)(R * (nc + (P.viscous ? rows_f : 0)) * sizeof(double));
                D.messages += P.viscous ? 2 : 1;
            } else if (me == og) {
                for (const Slot& s : slots)
                    if (s.g == g && s.q == q) {
                        char* b = reinterpret_cast<char*>(D.tmp) + s.off;
                        ok = ok && D.tp->recv(b, R * nc * sizeof(double), q, 2 * g, c->st);
                        if (P.viscous)
                            ok = ok && D.tp->recv(b + R * nc * sizeof(double), R * rows_f * sizeof(double), q,
                                                  2 * g + 1, c->st);
                    }
            }
        }
    }
    ok = D.tp->end(c->st) && ok;
    if (!ok) {
        D.err = D.tp->err.empty() ? "exchange failed" : D.tp->err;
        return;
    }
    for (const Slot& s : slots) {
        const size_t R = P.meshes[s.g].rpoint.size();
        MeshDev& M = c->md[s.g];
        const double* b = reinterpret_cast<const double*>(reinterpret_cast<char*>(D.tmp) + s.off);
        launch_merge_recv(nc, (int64_t)R, M.rdonor, D.ot, s.q, b, M.qhat, c->st);
        if (P.viscous) launch_merge_recv(rows_f, (int64_t)R, M.rdonor, D.ot, s.q, b + R * nc, M.fvhat, c->st);
    }
}

// fastest-first MRAB macro step of a rank (serial launches, weights as launch arguments)
static void issue_macro_step_dist(mrab_ctx* c) {
    const Plan& P = *c->P;
    const int G = (int)P.meshes.size(), m = P.history_m;
    for (int j = 0; j < P.S; ++j) {
        std::vector<int> stepping;
        SrcSet ss{};
        for (int g = 0; g < G; ++g) {
            MeshDev& D = c->md[g];
            const MeshPlan& mp = P.meshes[g];
            if (j % mp.s == 0) {
                stepping.push_back(g);
                if (c->book.pending[g]) {
                    c->book.cur[g] ^= 1;
                    c->book.pending[g] = 0;
                }
                ss.base[g] = D.Q[c->book.cur[g]];
                ss.nsrc[g] = 0;
            } else {
                double w[kMaxHist];
                weights_partial(c, g, j, w);
                const double hg = h_micro(c) * mp.s;
                ss.base[g] = D.Q[c->book.cur[g]];
                ss.nsrc[g] = m;
                for (int k = 0; k < m; ++k) {
                    ss.src[g][k] = D.ring[((c->book.head[g] - (m - 1) + k) % m + m) % m];
                    ss.c[g][k] = hg * w[k];
                }
            }
        }
        dist_gather(c, stepping, ss);
        for (int g : stepping) {
            MeshDev& D = c->md[g];
            const MeshPlan& mp = P.meshes[g];
            const double hg = h_micro(c) * mp.s;
            const int newslot = (c->book.head[g] + 1) % m;
            if (owns(c, g)) {
                Epilogue ep{};
                ep.r_out = D.ring[newslot];
                ep.y_out = D.Q[c->book.cur[g] ^ 1];
                ep.base = D.Q[c->book.cur[g]];
                double al[kMaxHist];
                weights_full(c, g, j, al);
                ep.c_new = hg * al[m - 1];
                ep.nsrc = m - 1;
                for (int k = 0; k < m - 1; ++k) {
                    ep.src[k] = D.ring[((c->book.head[g] - (m - 2) + k) % m + m) % m];
                    ep.csrc[k] = hg * al[k];
                }
                std::vector<const double*> dummy(G, nullptr);
                issue_rhs(c, g, ep.base, ep, dummy.data());
                c->evals[g]++;
            }
            c->book.head[g] = newslot;
            note_push(c, g, j, newslot);
            c->book.pending[g] = 1;
        }
    }
}

// one coupled RK micro step of the bootstrap
// record: bootstrap mode (stage-1 RHS of mesh-aligned steps go to the rings, R6); otherwise a
// plain RK step of size hstep (mrab_rk_step: the RK4 reference integrator of P:861-878)
static void issue_rk_step(mrab_ctx* c, bool record = true, int order = 0, double hstep = 0.0) {
    const Plan& P = *c->P;
    const int G = (int)P.meshes.size(), m = P.history_m;
    const bool rk4 = (order ? order : P.order_n) >= 4;
    const double hh = record ? P.h : hstep;
    const int ns = rk4 ? 4 : 3;
    // Heun RK3 (R5) / classical RK4: a[s][j], b[j]
    double a[4][4] = {{0}}, b[4] = {0};
    if (rk4) {
        a[1][0] = 0.5;
        a[2][1] = 0.5;
        a[3][2] = 1.0;
        b[0] = 1.0 / 6;
        b[1] = 1.0 / 3;
        b[2] = 1.0 / 3;
        b[3] = 1.0 / 6;
    } else {
        a[1][0] = 1.0 / 3;
        a[2][1] = 2.0 / 3;
        b[0] = 0.25;
        b[1] = 0.0;
        b[2] = 0.75;
    }
    const int64_t nboot = (int64_t)(m - 1) * P.S;
    const int64_t left = nboot - c->boot_micro;
    std::vector<double*> kp(G * 4, nullptr);
    for (int g = 0; g < G; ++g) {
        if (c->book.pending[g]) {
            c->book.cur[g] ^= 1;
            c->book.pending[g] = 0;
        }
        const int s = P.meshes[g].s;
        bool rec = record && (left % s == 0) && (left / s <= m - 1);
        for (int q = 0; q < ns; ++q) kp[g * 4 + q] = c->md[g].kbuf[q];
        if (rec) {
            int newslot = (c->book.head[g] + 1) % m;
            kp[g * 4 + 0] = c->md[g].ring[newslot];
            c->book.head[g] = newslot;
        }
    }
    for (int s = 0; s < ns; ++s) {
        std::vector<const double*> state_of(G);
        for (int g = 0; g < G; ++g) {
            MeshDev& D = c->md[g];
            state_of[g] = (s == 0) ? D.Q[c->book.cur[g]] : D.ystage;
        }
        if (c->dist) {
            std::vector<int> allm(G);
            std::iota(allm.begin(), allm.end(), 0);
            dist_gather(c, allm, plain_states(c, state_of.data()));
        } else {
            issue_all_donors(c, state_of.data());
        }
        // every mesh reads its own stage state; the next stage state goes to a second
        // buffer (dstate) so that no mesh overwrites what another still gathers from.
        for (int g = 0; g < G; ++g) {
            MeshDev& D = c->md[g];
            Epilogue ep{};
            ep.r_out = kp[g * 4 + s];
            ep.base = D.Q[c->book.cur[g]];
            if (s < ns - 1) {
                ep.y_out = D.dstate;
                ep.c_new = hh * a[s + 1][s];
                ep.nsrc = 0;
                for (int jx = 0; jx < s; ++jx)
                    if (a[s + 1][jx] != 0.0) {
                        ep.src[ep.nsrc] = kp[g * 4 + jx];
                        ep.csrc[ep.nsrc++] = hh * a[s + 1][jx];
                    }
            } else {
                ep.y_out = D.Q[c->book.cur[g] ^ 1];
                ep.c_new = hh * b[s];
                ep.nsrc = 0;
                for (int jx = 0; jx < s; ++jx)
                    if (b[jx] != 0.0) {
                        ep.src[ep.nsrc] = kp[g * 4 + jx];
                        ep.csrc[ep.nsrc++] = hh * b[jx];
                    }
            }
            if (!owns(c, g)) continue;
            issue_rhs(c, g, state_of[g], ep, state_of.data());
            c->evals[g]++;
        }
        if (s < ns - 1)
            for (int g = 0; g < G; ++g) std::swap(c->md[g].dstate, c->md[g].ystage);
    }
    for (int g = 0; g < G; ++g) c->book.pending[g] = 1;
    if (record) c->boot_micro++;
}

// ----------------------------------------------------------------------------------------
// C ABI
// ----------------------------------------------------------------------------------------
extern "C" {

const char* mrab_last_error(void) { return g_last_error.c_str(); }

mrab_status mrab_ab_weights(const double* nodes, int m, int n, double a, double b, double* alpha_out) {
    std::string msg;
    mrab_status st = mrab::ab_weights(nodes, m, n, a, b, alpha_out, &msg);
    if (st != MRAB_OK) g_last_error = msg;
    return st;
}

mrab_status mrab_plan_create(const mrab_problem* problem, mrab_plan** out) {
    if (!out) return fail(MRAB_E_INVALID, "out is NULL");
    *out = nullptr;
    try {
        auto P = std::make_shared<Plan>();
        Error err{MRAB_OK, ""};
        if (!build_plan(problem, *P, err)) return fail(err.st, err.msg);
        *out = new mrab_plan{P};
        return MRAB_OK;
    } catch (const std::exception& e) {
        return fail(MRAB_E_INVALID, std::string("plan_create: ") + e.what());
    }
}

void mrab_plan_destroy(mrab_plan* plan) { delete plan; }

mrab_status mrab_overset_build(const mrab_problem* problem, int8_t** iblank_out, mrab_donor** donors_out,
                               int64_t* n_out) {
    if (!iblank_out || !donors_out || !n_out) return fail(MRAB_E_INVALID, "NULL output pointer");
    try {
        Plan P;
        Error err{MRAB_OK, ""};
        if (!build_plan(problem, P, err, /*overset_only=*/true)) return fail(err.st, err.msg);
        int64_t npts = 0, R = 0;
        for (const auto& m : P.meshes) {
            npts += m.npts;
            R += (int64_t)m.rpoint.size();
        }
        int8_t* ib = (int8_t*)std::malloc((size_t)std::max<int64_t>(npts, 1));
        mrab_donor* dn = (mrab_donor*)std::calloc((size_t)std::max<int64_t>(R, 1), sizeof(mrab_donor));
        if (!ib || !dn) {
            std::free(ib);
            std::free(dn);
            return fail(MRAB_E_INVALID, "out of host memory");
        }
        int64_t o = 0, e = 0;
        for (int g = 0; g < (int)P.meshes.size(); ++g) {
            const MeshPlan& m = P.meshes[g];
            for (int64_t p = 0; p < m.npts; ++p) ib[o + p] = m.active[p] ? 1 : 0;
            o += m.npts;
            for (size_t r = 0; r < m.rpoint.size(); ++r, ++e) {
                dn[e].recv_mesh = g;
                dn[e].donor_mesh = m.rdonor[r];
                dn[e].recv_index = m.rpoint[r];
                for (int k = 0; k < 3; ++k) dn[e].base[k] = m.rbase[r * 3 + k];
                for (int k = 0; k < 3; ++k)
                    for (int a = 0; a < 4; ++a) dn[e].w[k][a] = m.rw[r * 12 + k * 4 + a];
            }
        }
        *iblank_out = ib;
        *donors_out = dn;
        *n_out = R;
        return MRAB_OK;
    } catch (const std::exception& ex) {
        return fail(MRAB_E_INVALID, std::string("overset_build: ") + ex.what());
    }
}

void mrab_free(void* p) { std::free(p); }

mrab_status mrab_plan_get_face_flags(const mrab_plan* plan, int mesh, uint8_t* flags) {
    if (!plan || mesh < 0 || mesh >= (int)plan->P->meshes.size() || !flags)
        return fail(MRAB_E_INVALID, "bad plan/mesh or NULL flags");
    const MeshPlan& m = plan->P->meshes[mesh];
    for (int64_t p = 0; p < m.npts; ++p) {
        uint8_t f = 0;
        if (m.active[p])
            for (int k = 0; k < m.dim; ++k) {
                if (m.posA[k][p] == 0) f |= (uint8_t)(1u << (2 * k));
                if (m.posB[k][p] == 0) f |= (uint8_t)(1u << (2 * k + 1));
            }
        flags[p] = f;
    }
    return MRAB_OK;
}

mrab_status mrab_plan_info(const mrab_plan* plan, int mesh, int64_t* n_points, int64_t* n_active,
                           int64_t* n_receivers) {
    if (!plan || mesh < 0 || mesh >= (int)plan->P->meshes.size()) return fail(MRAB_E_INVALID, "bad plan/mesh");
    const MeshPlan& m = plan->P->meshes[mesh];
    if (n_points) *n_points = m.npts;
    if (n_active) *n_active = m.nactive;
    if (n_receivers) *n_receivers = (int64_t)m.rpoint.size();
    return MRAB_OK;
}

mrab_status mrab_plan_get_tables(const mrab_plan* plan, int mesh, int8_t* iblank, int64_t* recv_point,
                                 int32_t* recv_donor, int32_t* recv_base, double* recv_weights) {
    if (!plan || mesh < 0 || mesh >= (int)plan->P->meshes.size()) return fail(MRAB_E_INVALID, "bad plan/mesh");
    const MeshPlan& m = plan->P->meshes[mesh];
    if (iblank) std::memcpy(iblank, m.active.data(), m.npts);
    const size_t R = m.rpoint.size();
    if (recv_point && R) std::memcpy(recv_point, m.rpoint.data(), R * sizeof(int64_t));
    if (recv_donor && R) std::memcpy(recv_donor, m.rdonor.data(), R * sizeof(int32_t));
    if (recv_base && R) std::memcpy(recv_base, m.rbase.data(), R * 3 * sizeof(int32_t));
    if (recv_weights && R) std::memcpy(recv_weights, m.rw.data(), R * 12 * sizeof(double));
    return MRAB_OK;
}

mrab_status mrab_plan_get_metrics(const mrab_plan* plan, int mesh, double* jinv, double* M) {
    if (!plan || mesh < 0 || mesh >= (int)plan->P->meshes.size()) return fail(MRAB_E_INVALID, "bad plan/mesh");
    const MeshPlan& m = plan->P->meshes[mesh];
    if (jinv) std::memcpy(jinv, m.jinv.data(), m.npts * sizeof(double));
    if (M) std::memcpy(M, m.M.data(), m.M.size() * sizeof(double));
    return MRAB_OK;
}

size_t mrab_workspace_bytes(const mrab_plan* plan) {
    if (!plan) return 0;
    set_options(plan->P->opt);
    bool ok = true;
    return plan_bytes(*plan->P, true, nullptr, nullptr, &ok);
}

mrab_status mrab_create(const mrab_plan* plan, const double* const* q0, void* d_workspace,
                        size_t ws_bytes, void* stream, mrab_ctx** out) {
    if (!out) return fail(MRAB_E_INVALID, "out is NULL");
    *out = nullptr;
    if (!plan || !q0) return fail(MRAB_E_INVALID, "plan or q0 is NULL");
    if (!d_workspace || ((uintptr_t)d_workspace & 255)) return fail(MRAB_E_WORKSPACE, "workspace NULL or not 256-byte aligned");
    const Plan& P = *plan->P;
    if (ws_bytes < mrab_workspace_bytes(plan)) return fail(MRAB_E_WORKSPACE, "workspace too small");
    set_options(P.opt);
    std::unique_ptr<mrab_ctx> c(new mrab_ctx());
    c->P = plan->P;
    c->user = (cudaStream_t)stream;
    const int G = (int)P.meshes.size();
    c->md.resize(G);
    c->evals.assign(G, 0);
    Bump bump{(char*)d_workspace, ws_bytes, 0};
    bool ok = true;
    plan_bytes(P, false, c.get(), &bump, &ok);
    if (!ok) return fail(MRAB_E_WORKSPACE, "workspace too small (layout)");
    CK(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
    {
        // side streams: the gather stream and the fastest meshes get the highest priority
        int least = 0, greatest = 0;
        CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        int smin = P.S;
        for (auto& mp : P.meshes) smin = std::min(smin, mp.s);
        for (int g = 0; g < (int)P.meshes.size(); ++g) {
            const int prio = P.meshes[g].s == smin ? greatest : least;
            CK(cudaStreamCreateWithPriority(&c->side[g], cudaStreamNonBlocking, prio));
        }
        CK(cudaStreamCreateWithPriority(&c->side[P.meshes.size()], cudaStreamNonBlocking, greatest));
        // 2-D: bulk tiles of split meshes run on their own streams, concurrent with the critical
        // tiles; 3-D: donor-preparation and gather streams (highest priority)
        for (int g = 0; g < (int)P.meshes.size(); ++g) {
            CK(cudaStreamCreateWithPriority(&c->side[P.meshes.size() + 1 + g], cudaStreamNonBlocking,
                                            P.dim == 3 ? greatest : least));
            if (P.dim == 3)
                CK(cudaStreamCreateWithPriority(&c->side[2 * P.meshes.size() + 1 + g], cudaStreamNonBlocking, greatest));
        }
        // critical/bulk split of slow meshes with per-node launch priorities (on by default;
        // config 3: 0.1205 -> 0.110 ms per macro step; Options::overlap = 0 disables)
        c->overlap = P.opt.overlap != 0;
        // bulk launches take one CTA per tile by default (Options::bulk_ctas = k: k persistent CTAs)
        c->bulk_ctas = P.opt.bulk_ctas;
    }
    CK(cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_out, cudaEventDisableTiming));
    c->gas.gamma = P.gamma;
    c->gas.Re = P.viscous ? P.Re : 1.0;
    c->gas.Pr = P.Pr;
    c->gas.wall_T = P.wall_T;
    c->gas.viscous = P.viscous;
    for (int k = 0; k < 5; ++k) c->gas.q_inf[k] = P.q_inf[k];
    c->gas.iRe = 1.0 / c->gas.Re;
    c->gas.kT = 1.0 / (c->gas.Re * P.Pr * (P.gamma - 1.0));
    c->gas.gm1 = P.gamma - 1.0;
    c->gas.igm1 = 1.0 / (P.gamma - 1.0);
    c->gas.igamma = 1.0 / P.gamma;
    const int nc = P.nc, d = P.dim;
    for (int g = 0; g < G; ++g) {
        const MeshPlan& m = P.meshes[g];
        MeshDev& D = c->md[g];
        const size_t N = (size_t)m.npts, R = m.rpoint.size();
        CK(cudaMemcpyAsync(D.Q[0], q0[g], nc * N * sizeof(double), cudaMemcpyDefault, c->st));
        CK(cudaMemsetAsync(D.Q[1], 0, nc * N * sizeof(double), c->st));
        for (int k = 0; k < P.history_m; ++k) CK(cudaMemsetAsync(D.ring[k], 0, nc * N * sizeof(double), c->st));
        CK(cudaMemsetAsync(D.FV, 0, (size_t)d * (d + 1) * N * sizeof(double), c->st));
        CK(cudaMemsetAsync(D.dstate, 0, nc * N * sizeof(double), c->st));
        CK(cudaMemsetAsync(D.ystage, 0, nc * N * sizeof(double), c->st));
        for (int k = 0; k < 4; ++k) CK(cudaMemsetAsync(D.kbuf[k], 0, nc * N * sizeof(double), c->st));
        if (!m.cartesian) {
            std::vector<double> J(N);
            for (size_t p = 0; p < N; ++p) J[p] = m.active[p] ? 1.0 / m.jinv[p] : 0.0;
            CK(cudaMemcpy(D.J, J.data(), N * sizeof(double), cudaMemcpyHostToDevice));
            CK(cudaMemcpy(D.M, m.M.data(), (size_t)d * d * N * sizeof(double), cudaMemcpyHostToDevice));
        }
        CK(cudaMemcpy(D.cls, m.cls.data(), N * sizeof(uint16_t), cudaMemcpyHostToDevice));
        if (d == 3) {
            // F^V is read by the gathers at the exact donor stencils (4^3 points) of every
            // receiver this mesh donates to: the 8^3 tiles holding them
            const int tx = (m.n[0] + 7) / 8, ty = (m.n[1] + 7) / 8, tz = (m.n[2] + 7) / 8;
            std::vector<uint8_t> fl((size_t)tx * ty * tz, 0);
            for (size_t h = 0; h < P.meshes.size(); ++h) {
                const MeshPlan& mh = P.meshes[h];
                for (size_t r = 0; r < mh.rdonor.size(); ++r) {
                    if (mh.rdonor[r] != g) continue;
                    for (int a2 = 0; a2 < 4; ++a2)
                        for (int a1 = 0; a1 < 4; ++a1)
                            for (int a0 = 0; a0 < 4; ++a0) {
                                const int i = (mh.rbase[3 * r] + a0) % m.n[0];
                                const int jj = (mh.rbase[3 * r + 1] + a1) % m.n[1];
                                const int k = (mh.rbase[3 * r + 2] + a2) % m.n[2];
                                fl[(size_t)(i / 8) + tx * ((size_t)(jj / 8) + (size_t)ty * (k / 8))] = 1;
                            }
                }
            }
            std::vector<int32_t> lst;
            for (size_t t = 0; t < fl.size(); ++t)
                if (fl[t]) lst.push_back((int32_t)t);
            D.nfv = (int)lst.size();
            if (!lst.empty())
                CK(cudaMemcpy(D.fvlist, lst.data(), lst.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
            // intermediate donor states are formed on these tiles and their face neighbours (the
            // viscous pass reads the cross-shaped region tile + 3 along each axis)
            {
                std::vector<uint8_t> cb(fl);
                const int nt3[3] = {tx, ty, tz};
                for (int32_t t : lst) {
                    const int tc[3] = {t % tx, (t / tx) % ty, t / (tx * ty)};
                    for (int a = 0; a < 3; ++a)
                        for (int sgn = -1; sgn <= 1; sgn += 2) {
                            int q[3] = {tc[0], tc[1], tc[2]};
                            // one tile on; two when that tile is a last partial tile thinner
                            // than the reach of 3
                            for (int hop = 0; hop < 2; ++hop) {
                                q[a] += sgn;
                                if (q[a] < 0 || q[a] >= nt3[a]) {
                                    if (!m.periodic[a]) break;
                                    q[a] = (q[a] + nt3[a]) % nt3[a];
                                }
                                cb[(size_t)q[0] + tx * ((size_t)q[1] + (size_t)ty * q[2])] = 1;
                                if (m.n[a] - 8 * q[a] >= 3) break;
                            }
                        }
                }
                std::vector<int32_t> cl;
                for (size_t t = 0; t < cb.size(); ++t)
                    if (cb[t]) cl.push_back((int32_t)t);
                D.ncb = (int)cl.size();
                if (!cl.empty())
                    CK(cudaMemcpy(D.cblist, cl.data(), cl.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
            }
            // two-pass RHS: the 8^3 tiles holding SAT points (k_flux3d writes F^V there)
            std::vector<uint8_t> st((size_t)tx * ty * tz, 0);
            for (int k = 0; k < m.n[2]; ++k)
                for (int jj = 0; jj < m.n[1]; ++jj)
                    for (int i = 0; i < m.n[0]; ++i) {
                        const unsigned cc = m.cls[m.idx(i, jj, k)];
                        bool need = false;
                        for (int a = 0; a < 3; ++a) {
                            const int cl = (cc >> (4 * a)) & 15;
                            need = need || cl == CLS_L0 || cl == CLS_R0;
                        }
                        if (need) st[(size_t)(i / 8) + tx * ((size_t)(jj / 8) + (size_t)ty * (k / 8))] = 1;
                    }
            // ... and the donor-stencil tiles (the gathers read F^V there at stepping times):
            // bit 0 = donor stencils (every point of the tile), bit 1 = SAT points (those only)
            for (size_t t = 0; t < st.size(); ++t) st[t] = (uint8_t)((fl[t] ? 1 : 0) | (st[t] ? 2 : 0));
            CK(cudaMemcpy(D.fvtile, st.data(), st.size(), cudaMemcpyHostToDevice));
        }
        CK(cudaMemcpy(D.recv_slot, m.recv_slot.data(), N * sizeof(int32_t), cudaMemcpyHostToDevice));
        if (R) {
            CK(cudaMemcpy(D.rpoint, m.rpoint.data(), R * sizeof(int64_t), cudaMemcpyHostToDevice));
            CK(cudaMemcpy(D.rdonor, m.rdonor.data(), R * sizeof(int32_t), cudaMemcpyHostToDevice));
            CK(cudaMemcpy(D.rbase, m.rbase.data(), R * 3 * sizeof(int32_t), cudaMemcpyHostToDevice));
            CK(cudaMemcpy(D.rw, m.rw.data(), R * 12 * sizeof(double), cudaMemcpyHostToDevice));
            if (d == 3 && P.opt.interp_box) {
                std::vector<int32_t> order;
                const std::vector<int32_t> info = interp3_groups((int64_t)R, m.rdonor.data(), m.rbase.data(), order);
                CK(cudaMemcpy(D.gorder, order.data(), R * sizeof(int32_t), cudaMemcpyHostToDevice));
                CK(cudaMemcpy(D.ginfo, info.data(), info.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
                D.ngroups = (int)(info.size() / 6);
            }
        }
        DevMesh& dm = D.dm;
        for (int k = 0; k < 3; ++k) {
            dm.n[k] = m.n[k];
            dm.periodic[k] = m.periodic[k];
            dm.face_bc[k][0] = m.face_bc[k][0];
            dm.face_bc[k][1] = m.face_bc[k][1];
        }
        dm.npts = m.npts;
        dm.cart = m.cartesian ? 1 : 0;
        dm.cJ = m.cart_J;
        for (int k = 0; k < 3; ++k) dm.cM[k] = m.cart_M[k];
        dm.J = D.J;
        dm.M = D.M;
        dm.cls = D.cls;
        dm.recv_slot = D.recv_slot;
        dm.qhat = D.qhat;
        dm.fvhat = D.fvhat;
        dm.rdonor = D.rdonor;
        dm.rbase = D.rbase;
        dm.rw = D.rw;
        if (d == 2) {
            // tile lists: tiles meeting the donor state box first (critical), then the rest
            int tx, ty;
            rhs2d_tile_shape_for(m.n, m.cartesian ? 1 : 0, &tx, &ty);
            const int ntx = (m.n[0] + tx - 1) / tx, nty = (m.n[1] + ty - 1) / ty;
            std::vector<int32_t> crit, bulk, slow, fastl;
            const bool tag = P.opt.tile_flags != 0;
            for (int by = 0; by < nty; ++by)
                for (int bx = 0; bx < ntx; ++bx) {
                    const bool interior = tag && rhs2d_interior_tile(m.n, m.periodic, m.cls.data(), P.viscous, bx, by, m.cartesian ? 1 : 0);
                    const int32_t t = (by * ntx + bx) | (interior ? (int32_t)0x80000000u : 0);
                    const bool meets = m.is_donor && bx * tx <= m.st_hi[0] &&
                                       bx * tx + tx - 1 >= m.st_lo[0] && by * ty <= m.st_hi[1] &&
                                       by * ty + ty - 1 >= m.st_lo[1];
                    (meets ? crit : bulk).push_back(t);
                    (interior ? fastl : slow).push_back(t);
                }
            D.ncrit = (int)crit.size();
            D.nbulk = (int)bulk.size();
            D.ngen = (int)slow.size();
            crit.insert(crit.end(), bulk.begin(), bulk.end());
            CK(cudaMemcpy(D.tiles, crit.data(), crit.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
            // the longer non-interior tiles go first so they do not form the tail
            slow.insert(slow.end(), fastl.begin(), fastl.end());
            CK(cudaMemcpy(D.tlist, slow.data(), slow.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
            dm.tlist = D.tlist;
            dm.ntl = (int)slow.size();
        }
        dm.nrecv = (int64_t)R;
        dm.z3t = nullptr;
        dm.fh = D.FH;
        dm.fv = D.FV;
        dm.fvtile = D.fvtile;
        if (d == 3) {
            // TMA descriptors of every buffer the fused 3-D kernel reads as a state or as an
            // epilogue input (a buffer TMA cannot describe falls back to cp.async)
            const double* bufs[] = {D.Q[0], D.Q[1], D.ystage, D.dstate, D.kbuf[0], D.kbuf[1], D.kbuf[2], D.kbuf[3]};
            for (const double* b : bufs) z3_encode(dm, b, D.z3tab);
            for (int k = 0; k < P.history_m; ++k) z3_encode(dm, D.ring[k], D.z3tab);
            dm.z3t = D.z3tab.n ? &D.z3tab : nullptr;
        }
        c->book.head[g] = P.history_m - 1;   // empty ring: the first push goes to slot 0
        c->book.cur[g] = 0;
        c->book.pending[g] = 0;
    }
    CK(cudaStreamSynchronize(c->st));
    // graph period: ring phase (m) and double-buffer phase (2)
    int L = 1;
    for (int g = 0; g < G; ++g) {
        int e = P.S / P.meshes[g].s;
        int pm = P.history_m / std::gcd(P.history_m, e);
        int p2 = 2 / std::gcd(2, e);
        int pg = std::lcm(pm, p2);
        L = std::lcm(L, pg);
    }
    c->period = L;
    c->graphs.assign(L, nullptr);
    c->book_after.resize(L);
    c->evals_per_phase.resize(L);
    *out = c.release();
    return MRAB_OK;
}

void mrab_destroy(mrab_ctx* c) {
    if (!c) return;
    cudaStreamSynchronize(c->st);
    for (auto& g : c->graphs)
        if (g) cudaGraphExecDestroy(g);
    for (auto& s : c->side)
        if (s) cudaStreamDestroy(s);
    for (auto& e : c->evpool) cudaEventDestroy(e);
    if (c->dist && c->dist->tmp) cudaFree(c->dist->tmp);
    if (c->ev_in) cudaEventDestroy(c->ev_in);
    if (c->ev_out) cudaEventDestroy(c->ev_out);
    if (c->st) cudaStreamDestroy(c->st);
    delete c;
}

// Capture every phase graph of the MRAB macro step (period = ring x double-buffer phases),
// starting from the current bookkeeping; the bookkeeping is restored afterwards, so the graphs
// are replayed in order by mrab_step.  Called once the bootstrap is done, so that no capture
// or instantiation lands inside a later (timed) macro step.
static mrab_status ensure_graphs(mrab_ctx* c) {
    if (c->graphs[0]) return MRAB_OK;
    c->graph_k0 = std::max<int64_t>(c->macro - (c->P->history_m - 1), 0);
    const Book book0 = c->book;
    const std::vector<int64_t> ev_start = c->evals;
    for (int phase = 0; phase < c->period; ++phase) {
        std::vector<int64_t> ev0 = c->evals;
        c->launch_counter = 0;
        CK(cudaStreamBeginCapture(c->st, cudaStreamCaptureModeThreadLocal));
        issue_macro_step(c);
        cudaGraph_t graph;
        CK(cudaStreamEndCapture(c->st, &graph));
        CK(cudaGraphInstantiate(&c->graphs[phase], graph, cudaGraphInstantiateFlagUseNodePriority));
        CK(cudaGraphDestroy(graph));
        if (phase == 0) c->launches_last = c->launch_counter;
        c->book_after[phase] = c->book;
        c->evals_per_phase[phase].resize(c->evals.size());
        for (size_t g = 0; g < c->evals.size(); ++g) c->evals_per_phase[phase][g] = c->evals[g] - ev0[g];
    }
    c->book = book0;
    c->evals = ev_start;
    // upload the executable graphs now (the first launch would otherwise do it)
    for (int phase = 0; phase < c->period; ++phase) CK(cudaGraphUpload(c->graphs[phase], c->st));
    return MRAB_OK;
}

// the caller's stream is joined into the context stream (work queued on it before this call,
// e.g. a torch kernel still writing a device source buffer, completes first)
static mrab_status join_user(mrab_ctx* c) {
    CK(cudaEventRecord(c->ev_in, c->user));
    CK(cudaStreamWaitEvent(c->st, c->ev_in, 0));
    return MRAB_OK;
}

static const double* current_state(mrab_ctx* c, int g);

// uniform history node times (ring entries at -h_g, -2 h_g, ... relative to the macro boundary)
static void uniform_ring_times(mrab_ctx* c) {
    const Plan& P = *c->P;
    const int m = P.history_m;
    for (size_t g = 0; g < P.meshes.size(); ++g)
        for (int k = 0; k < m; ++k) {
            const int slot = ((c->book.head[g] - k) % m + m) % m;   // k-th newest
            c->ring_t[g][slot] = -(double)(k + 1) * P.meshes[g].s * P.h;
        }
}

// one MRAB macro step of size H issued directly (no graph): the weights depend on H and on
// the history node times, which change from step to step
static mrab_status var_macro_step(mrab_ctx* c, double H) {
    const Plan& P = *c->P;
    if (c->scheme > 0) return fail(MRAB_E_INVALID, "this context runs a slowest-first scheme (fixed step only)");
    c->scheme = 0;
    if (!c->var_mode) {
        uniform_ring_times(c);
        c->var_mode = true;
    }
    c->h_cur = H / P.S;
    c->launch_counter = 0;
    if (c->dist) {
        issue_macro_step_dist(c);
        if (!c->dist->err.empty()) return fail(MRAB_E_CUDA, "exchange: " + c->dist->err);
    } else {
        issue_macro_step(c);
    }
    c->launches_last = c->launch_counter;
    CK(cudaGetLastError());
    for (size_t g = 0; g < P.meshes.size(); ++g)
        for (int k = 0; k < P.history_m; ++k) c->ring_t[g][k] -= H;
    c->time_extra += H;
    c->macro++;
    return MRAB_OK;
}

mrab_status mrab_step(mrab_ctx* c, int n_macro) {
    if (!c || n_macro < 0) return fail(MRAB_E_INVALID, "bad ctx / n_macro");
    const Plan& P = *c->P;
    set_options(P.opt);
    CK(cudaEventRecord(c->ev_in, c->user));
    CK(cudaStreamWaitEvent(c->st, c->ev_in, 0));
    const int64_t nboot_macro = P.history_m - 1;
    for (int it = 0; it < n_macro; ++it) {
        if (c->dist && c->macro >= nboot_macro && !c->var_mode) {
            // multi-GPU: direct launches (the exchange sits between them)
            if (c->scheme > 0) return fail(MRAB_E_INVALID, "multi-GPU contexts run the fastest-first scheme");
            c->scheme = 0;
            c->launch_counter = 0;
            issue_macro_step_dist(c);
            c->launches_last = c->launch_counter;
            CK(cudaGetLastError());
            if (!c->dist->err.empty()) return fail(MRAB_E_CUDA, "exchange: " + c->dist->err);
            c->macro++;
            c->macro_fixed++;
            continue;
        }
        if (c->macro >= nboot_macro && c->var_mode) {
            // after variable steps the history is not uniform: the fixed-step graphs do not apply
            mrab_status st = var_macro_step(c, P.S * P.h);
            if (st != MRAB_OK) return st;
            continue;
        }
        if (c->macro < nboot_macro) {
            for (int s = 0; s < P.S; ++s) issue_rk_step(c);
            CK(cudaGetLastError());
        } else {
            if (c->scheme > 0) return fail(MRAB_E_INVALID, "this context runs a slowest-first scheme: use mrab_step_scheme");
            c->scheme = 0;
            const int64_t k = c->macro - nboot_macro;
            mrab_status st = ensure_graphs(c);
            if (st != MRAB_OK) return st;
            const int phase = (int)((k - c->graph_k0) % c->period);
            c->book = c->book_after[phase];
            for (size_t g = 0; g < c->evals.size(); ++g) c->evals[g] += c->evals_per_phase[phase][g];
            CK(cudaGraphLaunch(c->graphs[phase], c->st));
        }
        c->macro++;
        c->macro_fixed++;
        if (c->macro == nboot_macro) {
            mrab_status st = ensure_graphs(c);
            if (st != MRAB_OK) return st;
        }
    }
    CK(cudaGetLastError());
    CK(cudaEventRecord(c->ev_out, c->st));
    CK(cudaStreamWaitEvent(c->user, c->ev_out, 0));
    return MRAB_OK;
}

mrab_status mrab_step_h(mrab_ctx* c, int n_macro, double H) {
    if (!c || n_macro < 0 || !(H > 0.0)) return fail(MRAB_E_INVALID, "bad ctx / n_macro / H");
    const Plan& P = *c->P;
    if (c->macro < P.history_m - 1)
        return fail(MRAB_E_INSUFFICIENT_HISTORY, "variable steps start after the RK bootstrap: call mrab_step(history_m - 1) first");
    set_options(P.opt);
    CK(cudaEventRecord(c->ev_in, c->user));
    CK(cudaStreamWaitEvent(c->st, c->ev_in, 0));
    for (int it = 0; it < n_macro; ++it) {
        mrab_status st = var_macro_step(c, H);
        if (st != MRAB_OK) return st;
    }
    CK(cudaEventRecord(c->ev_out, c->st));
    CK(cudaStreamWaitEvent(c->user, c->ev_out, 0));
    return MRAB_OK;
}

mrab_status mrab_step_scheme(mrab_ctx* c, int n_macro, int scheme) {
    if (!c || n_macro < 0 || scheme < 0 || scheme > 2) return fail(MRAB_E_INVALID, "bad ctx / n_macro / scheme");
    if (scheme == MRAB_SCHEME_FASTEST_FIRST) return mrab_step(c, n_macro);
    const Plan& P = *c->P;
    bool two_rate = P.S > 1;
    int nfast = 0, nslow = 0;
    for (auto& mp : P.meshes) {
        two_rate = two_rate && (mp.s == 1 || mp.s == P.S);
        (mp.s == 1 ? nfast : nslow)++;
    }
    if (!two_rate || !nfast || !nslow)
        return fail(MRAB_E_INVALID, "slowest-first schemes need exactly two rates (step multiples 1 and S > 1)");
    if (P.opt.z3_fused) return fail(MRAB_E_INVALID, "slowest-first schemes run on the default (two-pass) 3-D kernels");
    set_options(P.opt);
    CK(cudaEventRecord(c->ev_in, c->user));
    CK(cudaStreamWaitEvent(c->st, c->ev_in, 0));
    const int64_t nboot_macro = P.history_m - 1;
    for (int it = 0; it < n_macro; ++it) {
        if (c->macro < nboot_macro) {
            for (int s = 0; s < P.S; ++s) issue_rk_step(c);
            CK(cudaGetLastError());
        } else {
            if (c->scheme >= 0 && c->scheme != scheme)
                return fail(MRAB_E_INVALID, "the MRAB scheme of a context is fixed by its first MRAB step");
            c->scheme = scheme;
            c->launch_counter = 0;
            mrab_status st = issue_macro_step_sf(c, scheme == MRAB_SCHEME_SLOWEST_FIRST_REEXTRAP);
            if (st != MRAB_OK) return st;
            c->launches_last = c->launch_counter;
        }
        c->macro++;
        c->macro_fixed++;
    }
    CK(cudaEventRecord(c->ev_out, c->st));
    CK(cudaStreamWaitEvent(c->user, c->ev_out, 0));
    return MRAB_OK;
}

mrab_status mrab_partition(const mrab_plan* plan, int nranks, int* owner, double* load) {
    if (!plan || nranks < 1 || !owner) return fail(MRAB_E_INVALID, "bad plan / nranks / owner");
    const Plan& P = *plan->P;
    const int G = (int)P.meshes.size();
    // longest-processing-time-first: heaviest mesh to the least loaded rank (ties: lowest index)
    std::vector<double> w(G), L(nranks, 0.0);
    std::vector<int> ord(G);
    std::iota(ord.begin(), ord.end(), 0);
    for (int g = 0; g < G; ++g) w[g] = (double)P.meshes[g].nactive * (P.S / P.meshes[g].s);
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return w[a] > w[b]; });
    for (int g : ord) {
        int r = 0;
        for (int q = 1; q < nranks; ++q)
            if (L[q] < L[r]) r = q;
        owner[g] = r;
        L[r] += w[g];
    }
    if (load)
        for (int q = 0; q < nranks; ++q) load[q] = L[q];
    return MRAB_OK;
}

mrab_status mrab_dist_unique_id(void* out128) {
    if (!out128) return fail(MRAB_E_INVALID, "out128 is NULL");
    std::string err;
    if (!nccl_unique_id(out128, &err)) return fail(MRAB_E_CUDA, err);
    return MRAB_OK;
}

mrab_status mrab_dist_attach(mrab_ctx* c, int transport, const void* id, int rank, int nranks, const int* owner) {
    if (!c || !id || !owner || nranks < 1 || rank < 0 || rank >= nranks || (transport != 0 && transport != 1))
        return fail(MRAB_E_INVALID, "bad arguments");
    if (c->macro != 0 || c->dist) return fail(MRAB_E_INVALID, "attach once, before the first step");
    const int G = (int)c->P->meshes.size();
    for (int g = 0; g < G; ++g)
        if (owner[g] < 0 || owner[g] >= nranks) return fail(MRAB_E_INVALID, "owner out of range");
    std::unique_ptr<mrab_ctx::DistState> D(new mrab_ctx::DistState());
    D->rank = rank;
    D->nranks = nranks;
    for (int g = 0; g < 8; ++g) D->ot.owner[g] = g < G ? owner[g] : 0;
    std::string err;
    if (transport == MRAB_TRANSPORT_NCCL) D->tp = make_nccl_transport(id, rank, nranks, &err);
    else D->tp = make_loopback_transport(*(const int*)id, rank, nranks);
    if (!D->tp) return fail(MRAB_E_CUDA, err);
    c->dist = std::move(D);
    return MRAB_OK;
}

mrab_status mrab_dist_stats(mrab_ctx* c, int64_t* bytes_sent, int64_t* messages) {
    if (!c || !c->dist) return fail(MRAB_E_INVALID, "not a multi-GPU context");
    if (bytes_sent) *bytes_sent = c->dist->bytes_sent;
    if (messages) *messages = c->dist->messages;
    return MRAB_OK;
}

mrab_status mrab_step_cfl(mrab_ctx* c, int n_macro, double cfl, double* H_last) {
    if (!c || n_macro < 0 || !(cfl > 0.0)) return fail(MRAB_E_INVALID, "bad ctx / n_macro / cfl");
    const Plan& P = *c->P;
    const int G = (int)P.meshes.size();
    std::vector<double> dt(G);
    for (int it = 0; it < n_macro; ++it) {
        mrab_status st = mrab_dt(c, dt.data());
        if (st != MRAB_OK) return st;
        double H = 0.0;
        for (int g = 0; g < G; ++g) {
            const double Hg = cfl * P.S * dt[g] / P.meshes[g].s;
            H = g == 0 ? Hg : std::min(H, Hg);
        }
        if (!(H > 0.0) || !std::isfinite(H)) return fail(MRAB_E_NONFINITE, "timestep estimate is not a positive finite number");
        st = mrab_step_h(c, 1, H);
        if (st != MRAB_OK) return st;
        if (H_last) *H_last = H;
    }
    return MRAB_OK;
}

mrab_status mrab_rk_step(mrab_ctx* c, int n_steps, int order, double h) {
    if (!c || n_steps < 0 || (order != 3 && order != 4) || !(h > 0.0))
        return fail(MRAB_E_INVALID, "bad ctx / n_steps / order (3 or 4) / h");
    set_options(c->P->opt);
    CK(cudaEventRecord(c->ev_in, c->user));
    CK(cudaStreamWaitEvent(c->st, c->ev_in, 0));
    for (int it = 0; it < n_steps; ++it) issue_rk_step(c, false, order, h);
    CK(cudaGetLastError());
    c->time_extra += n_steps * h;
    CK(cudaEventRecord(c->ev_out, c->st));
    CK(cudaStreamWaitEvent(c->user, c->ev_out, 0));
    return MRAB_OK;
}

mrab_status mrab_dt(mrab_ctx* c, double* dt_mesh) {
    if (!c || !dt_mesh) return fail(MRAB_E_INVALID, "bad arguments");
    const Plan& P = *c->P;
    if (join_user(c) != MRAB_OK) return MRAB_E_CUDA;
    double* dbuf = reinterpret_cast<double*>(reinterpret_cast<char*>(c->dflag) + 64);
    for (size_t g = 0; g < P.meshes.size(); ++g)
        launch_dt(P.dim, c->md[g].dm, current_state(c, (int)g), c->gas, dbuf + g, c->st);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(dt_mesh, dbuf, P.meshes.size() * sizeof(double), cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    return MRAB_OK;
}

static const double* current_state(mrab_ctx* c, int g) {
    const MeshDev& D = c->md[g];
    int b = c->book.pending[g] ? (c->book.cur[g] ^ 1) : c->book.cur[g];
    return D.Q[b];
}

mrab_status mrab_get_state(mrab_ctx* c, int mesh, double* dst, double* t) {
    if (!c || mesh < 0 || mesh >= (int)c->md.size() || !dst) return fail(MRAB_E_INVALID, "bad arguments");
    const Plan& P = *c->P;
    if (join_user(c) != MRAB_OK) return MRAB_E_CUDA;
    CK(cudaStreamSynchronize(c->st));
    const size_t n = (size_t)P.nc * P.meshes[mesh].npts;
    const double* src = current_state(c, mesh);
    CK(cudaMemsetAsync(c->dflag, 0, sizeof(int), c->st));
    launch_finite(src, n, c->dflag, c->st);
    CK(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDefault, c->st));
    int bad = 0;
    CK(cudaMemcpyAsync(&bad, c->dflag, sizeof(int), cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    if (t) *t = (double)c->macro_fixed * P.S * P.h + c->time_extra;
    if (bad)
        return fail(MRAB_E_NONFINITE, "mesh " + std::to_string(mesh) +
                                          ": non-finite state (rhs blowup); the state was copied");
    return MRAB_OK;
}

mrab_status mrab_set_state(mrab_ctx* c, int mesh, const double* src) {
    if (!c || mesh < 0 || mesh >= (int)c->md.size() || !src) return fail(MRAB_E_INVALID, "bad arguments");
    const Plan& P = *c->P;
    if (join_user(c) != MRAB_OK) return MRAB_E_CUDA;
    CK(cudaStreamSynchronize(c->st));
    const size_t bytes = (size_t)P.nc * P.meshes[mesh].npts * sizeof(double);
    CK(cudaMemcpyAsync((double*)current_state(c, mesh), src, bytes, cudaMemcpyDefault, c->st));
    CK(cudaStreamSynchronize(c->st));
    return MRAB_OK;
}

// committed history entry k (0 = oldest) of mesh g at a macro boundary after the bootstrap:
// the ring holds R(t - (m-1) h_g) .. R(t - h_g); R(t) is pending (evaluated by the next step)
static mrab_status history_slot(mrab_ctx* c, int mesh, int k, double** out) {
    if (!c || mesh < 0 || mesh >= (int)c->md.size()) return fail(MRAB_E_INVALID, "bad arguments");
    const Plan& P = *c->P;
    const int m = P.history_m;
    if (k < 0 || k > m - 2) return fail(MRAB_E_INVALID, "history index out of range [0, m-2]");
    if (c->macro < m - 1)
        return fail(MRAB_E_INSUFFICIENT_HISTORY, "history is complete only after the bootstrap");
    const int slot = ((c->book.head[mesh] - (m - 2) + k) % m + m) % m;
    *out = c->md[mesh].ring[slot];
    return MRAB_OK;
}

mrab_status mrab_get_history(mrab_ctx* c, int mesh, int k, double* dst) {
    double* src = nullptr;
    if (!dst) return fail(MRAB_E_INVALID, "bad arguments");
    mrab_status st = history_slot(c, mesh, k, &src);
    if (st != MRAB_OK) return st;
    const size_t bytes = (size_t)c->P->nc * c->P->meshes[mesh].npts * sizeof(double);
    if (join_user(c) != MRAB_OK) return MRAB_E_CUDA;
    CK(cudaStreamSynchronize(c->st));
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, c->st));
    CK(cudaStreamSynchronize(c->st));
    return MRAB_OK;
}

mrab_status mrab_set_history(mrab_ctx* c, int mesh, int k, const double* src) {
    double* dst = nullptr;
    if (!src) return fail(MRAB_E_INVALID, "bad arguments");
    mrab_status st = history_slot(c, mesh, k, &dst);
    if (st != MRAB_OK) return st;
    const size_t bytes = (size_t)c->P->nc * c->P->meshes[mesh].npts * sizeof(double);
    if (join_user(c) != MRAB_OK) return MRAB_E_CUDA;
    CK(cudaStreamSynchronize(c->st));
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, c->st));
    CK(cudaStreamSynchronize(c->st));
    if (c->var_mode) uniform_ring_times(c);   // the entries are defined at uniform nodes (R-SM)
    return MRAB_OK;
}

mrab_status mrab_rhs(mrab_ctx* c, const double* const* q, double* const* rhs_out) {
    if (!c || !q || !rhs_out) return fail(MRAB_E_INVALID, "bad arguments");
    const Plan& P = *c->P;
    const int G = (int)P.meshes.size();
    set_options(P.opt);
    if (join_user(c) != MRAB_OK) return MRAB_E_CUDA;
    CK(cudaStreamSynchronize(c->st));
    std::vector<const double*> state_of(G);
    for (int g = 0; g < G; ++g) {
        const size_t bytes = (size_t)P.nc * P.meshes[g].npts * sizeof(double);
        CK(cudaMemcpyAsync(c->md[g].ystage, q[g], bytes, cudaMemcpyDefault, c->st));
        state_of[g] = c->md[g].ystage;
    }
    if (c->dist) {
        std::vector<int> allm(G);
        std::iota(allm.begin(), allm.end(), 0);
        dist_gather(c, allm, plain_states(c, state_of.data()));
        if (!c->dist->err.empty()) return fail(MRAB_E_CUDA, "exchange: " + c->dist->err);
    } else {
        issue_all_donors(c, state_of.data());
    }
    for (int g = 0; g < G; ++g) {
        if (!owns(c, g)) continue;   // (a rank returns the RHS of the meshes it owns)
        Epilogue ep{};
        ep.r_out = c->md[g].kbuf[3];
        issue_rhs(c, g, state_of[g], ep, state_of.data());
    }
    CK(cudaGetLastError());
    for (int g = 0; g < G; ++g) {
        const size_t bytes = (size_t)P.nc * P.meshes[g].npts * sizeof(double);
        CK(cudaMemcpyAsync(rhs_out[g], c->md[g].kbuf[3], bytes, cudaMemcpyDefault, c->st));
    }
    CK(cudaStreamSynchronize(c->st));
    return MRAB_OK;
}

mrab_status mrab_get_counters(mrab_ctx* c, int64_t* rhs_evals, int64_t* point_rhs, int64_t* macro_steps) {
    if (!c) return fail(MRAB_E_INVALID, "ctx is NULL");
    CK(cudaStreamSynchronize(c->st));
    int64_t pr = 0;
    for (size_t g = 0; g < c->evals.size(); ++g) {
        if (rhs_evals) rhs_evals[g] = c->evals[g];
        pr += c->evals[g] * c->P->meshes[g].nactive;
    }
    if (point_rhs) *point_rhs = pr;
    if (macro_steps) *macro_steps = c->macro;
    return MRAB_OK;
}

mrab_status mrab_set_trace(mrab_ctx* c, void* dev_buf) {
    if (!c) return fail(MRAB_E_INVALID, "bad ctx");
    CK(cudaStreamSynchronize(c->st));
    for (auto& g : c->graphs)
        if (g) {
            cudaGraphExecDestroy(g);
            g = nullptr;
        }
    c->trace = (unsigned long long*)dev_buf;
    return MRAB_OK;
}

mrab_status mrab_launches_per_macro_step(mrab_ctx* c, int64_t* launches) {
    if (!c || !launches) return fail(MRAB_E_INVALID, "bad arguments");
    *launches = c->launches_last;
    return MRAB_OK;
}

mrab_status mrab_time_kernel(mrab_ctx* c, int kernel, int mesh, int reps, int flush_l2,
                             double* ms_per_launch, double* algorithmic_bytes) {
    if (!c || mesh < 0 || mesh >= (int)c->md.size() || reps < 1 || kernel < 0 || kernel > 5)
        return fail(MRAB_E_INVALID, "bad arguments");
    const Plan& P = *c->P;
    set_options(P.opt);
    const MeshPlan& mp = P.meshes[mesh];
    MeshDev& D = c->md[mesh];
    const int m = P.history_m, nc = P.nc, d = P.dim;
    const double N = (double)mp.npts;
    // the 2-D diagnostics (3-5) replay the interior-tile lists; the lean-only kernel (3) is
    // compiled for 32 x 16 tiles only (variant 0)
    if (kernel >= 3 && (d != 2 || (kernel == 3 && rhs2d_variant_for(mp.n, mp.cartesian ? 1 : 0) != 0)))
        return fail(MRAB_E_INVALID, "kernel 3-5 are 2-D diagnostics; 3 needs the 32x16 tile variant");
    if (kernel == 1 && (d != 3 || !P.viscous))
        return fail(MRAB_E_INVALID, "kernel 1 (donor viscous fluxes) is a 3-D viscous kernel");
    CK(cudaStreamSynchronize(c->st));
    void* flush = nullptr;
    const size_t fbytes = (size_t)256 << 20;
    if (flush_l2) CK(cudaMalloc(&flush, 2 * fbytes));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const double* Q = current_state(c, mesh);
    std::vector<const double*> state_of(P.meshes.size());
    for (size_t g = 0; g < P.meshes.size(); ++g) state_of[g] = current_state(c, (int)g);
    double total = 0.0;
    double bytes = 0.0;
    for (int r = 0; r < reps; ++r) {
        if (flush) launch_l2_scrub(flush, (char*)flush + fbytes, fbytes, r, c->st);
        CK(cudaEventRecord(e0, c->st));
        if (kernel == 0 || kernel >= 3) {
            Epilogue ep{};
            ep.r_out = D.kbuf[0];
            ep.y_out = D.kbuf[1];
            ep.base = Q;
            ep.trace = d == 3 ? c->trace : nullptr;   // 3-D: phase-cycle accounting (profiling build)
            ep.c_new = P.h * mp.s * P.coef[mesh][mp.s][m - 1];
            ep.nsrc = m - 1;
            for (int k = 0; k < m - 1; ++k) {
                ep.src[k] = D.ring[k];
                ep.csrc[k] = P.h * mp.s * P.coef[mesh][mp.s][k];
            }
            double Nk = N;
            if (kernel >= 3 && d == 2) {
                // diagnostics: only the interior tiles, in the lean-only kernel (3) or in the
                // mixed kernel (4); only the non-interior tiles (5)
                ep.tiles = kernel == 5 ? D.tlist : D.tlist + D.ngen;
                ep.ntiles = kernel == 5 ? D.ngen : D.dm.ntl - D.ngen;
                ep.lean_only = kernel == 3;
                int tx, ty;
                rhs2d_tile_shape_for(mp.n, mp.cartesian ? 1 : 0, &tx, &ty);
                Nk = (double)ep.ntiles * tx * ty;
            }
            launch_rhs(d, D.dm, Q, c->gas, ep, make_ds(c, state_of.data()), c->st);
            // Q read, R written, (m-1) ring reads, state written, metrics if curvilinear
            bytes = 8.0 * Nk * (nc * (m + 2) + (mp.cartesian ? 0 : 1 + d * d));
        } else if (kernel == 1) {
            // 3-D donor viscous fluxes on the donor-stencil tiles of a stepping donor
            launch_visc(D.dm, Q, D.FV, Box{}, D.fvlist, D.nfv, c->gas, c->st);
            const double Nb = 512.0 * D.nfv;
            // Q read, Cartesian viscous fluxes written, metrics if curvilinear
            bytes = 8.0 * Nb * (nc + d * (d + 1) + (mp.cartesian ? 0 : 1 + d * d));
        } else {
            if (d == 2)
                issue_donor2d(c, std::vector<int>{mesh}, plain_states(c, state_of.data()));
            else
                issue_interp(c, mesh, state_of.data(), true);
            const double R = (double)mp.rpoint.size();
            const int np = d == 2 ? 16 : 64;
            // per receiver: indices + weights in, nc (+ d(d+1)) gathered values out; the
            // donor values themselves (np per receiver, mostly L2 hits) are counted once
            bytes = R * (8 + 4 + 12 + 96 + 8.0 * (nc + (P.viscous ? d * (d + 1) : 0)) * (1 + np));
        }
        CK(cudaEventRecord(e1, c->st));
        CK(cudaEventSynchronize(e1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        total += ms;
    }
    CK(cudaGetLastError());
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (flush) cudaFree(flush);
    if (ms_per_launch) *ms_per_launch = total / reps;
    if (algorithmic_bytes) *algorithmic_bytes = bytes;
    return MRAB_OK;
}

}  // extern "C"
