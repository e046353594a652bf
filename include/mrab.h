/*
 * mrab.h — C ABI of libmrab.so: the B200 (sm_100a, fp64) hot path of multi-rate
 * Adams–Bashforth time integration of the compressible Navier–Stokes equations on overset
 * SBP-SAT meshes (Mikida, Klöckner, Bodony, arXiv 1805.06607).
 *
 * Citations are PAPER.md lines (P:<line>) and the numbered readings R<k> of DESIGN.md §2.
 *
 * Conventions (every entry point):
 *   - A mesh has n[0] x n[1] (x n[2]) points in INDEX order (i fastest).  Host arrays are
 *     dense, C order: coordinates [dim][n2][n1][n0], states [nc][n2][n1][n0] with
 *     nc = dim + 2 components (rho, rho u_1..rho u_dim, rho E).  For dim = 2
 *     set n[2] = 1.
 *   - All floating point is IEEE fp64.
 *   - Every call returns an mrab_status and never throws across the ABI; on failure
 *     mrab_last_error() returns a thread-local message.  Output pointers are left
 *     untouched (creation calls set *out = NULL).
 *   - Ownership: the caller owns every descriptor and host array; they are read during the
 *     call only (copied).  The caller owns the device workspace passed to mrab_create (it
 *     must outlive the context).  The library owns plans, contexts, CUDA streams, events
 *     and graphs.
 *   - Asynchrony: mrab_step is asynchronous on the caller's stream; mrab_get_state,
 *     mrab_set_state, mrab_rhs and mrab_get_counters synchronise that stream.
 */
#ifndef MRAB_H
#define MRAB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    MRAB_OK = 0,
    MRAB_E_INVALID = 1,              /* bad argument, J^-1 <= 0 at an active point         */
    MRAB_E_DEGENERATE_NODES = 2,     /* duplicate AB history nodes                   */
    MRAB_E_INSUFFICIENT_HISTORY = 3, /* m < n                                        */
    MRAB_E_MISALIGNED = 4,           /* step multiples do not divide the largest    */
    MRAB_E_ORPHAN = 5,               /* a receiver has no all-active donor stencil (R17)   */
    MRAB_E_SEGMENT = 6,              /* an active segment shorter than 8 points (R2)       */
    MRAB_E_NONFINITE = 7,            /* non-finite state ("rhs blowup")             */
    MRAB_E_CUDA = 8,                 /* a CUDA runtime error (message has the CUDA string)  */
    MRAB_E_WORKSPACE = 9             /* workspace NULL / too small / misaligned            */
} mrab_status;

/* face tags (R16): overset interface, SAT far field, SAT isothermal no-slip wall,
 * periodic (both faces of a periodic direction) */
enum { MRAB_BC_OVERSET = 0, MRAB_BC_FARFIELD = 1, MRAB_BC_WALL = 2, MRAB_BC_PERIODIC = 3 };

typedef struct {
    int dim;                 /* 2 or 3                                                        */
    int n[3];                /* points per direction (index order); n[2] = 1 when dim = 2     */
    int periodic[3];         /* 1 = periodic direction (cyclic stencil across the seam)       */
    int face_bc[3][2];       /* tag of the (min, max) face of each direction                  */
    double period[3][3];     /* period[k][c]: jump of coordinate c across the seam of k       */
    const double* xyz;       /* host [dim][n2][n1][n0] node coordinates                       */
    int priority;            /* hole-cutting priority: higher cuts lower (R17)                */
    int step_multiple;       /* s_g: finest micro steps per step of this mesh (R8)           */
    /* Optional caller-supplied setup (NULL = the library builds it):
     *   metrics  host [1 + dim*dim][n2][n1][n0]: [0] = J^-1, [1 + kappa*dim + i] = M[kappa][i]
     *            = J^-1 d kappa / d x_i; J^-1 must be > 0 at every active point
     *            (else MRAB_E_INVALID).  Used verbatim (a mesh whose terms are constant and
     *            diagonal to 1e-10 relative is still run with the Cartesian kernels).
     *   iblank   host [n2][n1][n0], 0 = hole, nonzero = active (P:232-236 hole cutting).
     *            Used verbatim; segments (R2) and receivers (segment ends facing a hole or an
     *            overset face) are derived from it (MRAB_E_SEGMENT if a segment is
     *            shorter than 8 points). */
    const double* metrics;
    const int8_t* iblank;
} mrab_mesh_desc;

/* One overset receiver and its donor stencil ("donor cells", reading R17):
 * receiver point recv_index (flat, i fastest) of mesh recv_mesh takes its interpolated state
 * from the 4^dim stencil of mesh donor_mesh with lowest corner base[] (index order; wrapped
 * into [0, n) in periodic directions; base[2] = 0 in 2-D) and per-axis Lagrange weights
 * w[axis][a] (qhat = sum_abc w[0][a] w[1][b] w[2][c] q[base + (a, b, c)];
 * w[2] = (1, 0, 0, 0) in 2-D). */
typedef struct {
    int32_t recv_mesh;
    int32_t donor_mesh;
    int64_t recv_index;
    int32_t base[3];
    int32_t reserved;        /* 0 */
    double w[3][4];
} mrab_donor;

typedef struct {
    int dim;
    int n_meshes;
    const mrab_mesh_desc* meshes;
    double gamma, Re, Pr;    /* R11/R12: mu = 1, tau scaled by 1/Re, Fourier heat flux      */
    int viscous;             /* 0 = Euler (F^V = 0, sigma^V = 0)                            */
    double q_inf[5];         /* far-field state (conserved), nc entries used                */
    double wall_T;           /* isothermal wall temperature (R16)                           */
    int order_n;             /* AB order n                                      */
    int history_m;           /* history length m >= n; m > n = min-norm extended AB */
    double h;                /* finest micro step; mesh g steps h_g = s_g h                 */
    /* Optional caller-supplied donor table (n_donors = 0 / donors = NULL: the library
     * searches the donors, R17).  When given it must hold exactly one entry per receiver
     * of every mesh (the receivers follow from the blanking): a missing receiver is
     * MRAB_E_ORPHAN; a point that is not a receiver, a duplicate, a donor stencil that
     * leaves the donor mesh or touches a hole, or donor_mesh == recv_mesh is MRAB_E_INVALID.
     * Weights are used verbatim. */
    int64_t n_donors;
    const mrab_donor* donors;
} mrab_problem;

typedef struct mrab_plan mrab_plan;   /* host setup: tables, metrics, coefficients         */
typedef struct mrab_ctx mrab_ctx;     /* device state, rings, schedule, CUDA graphs        */

/* AB weights (P:343-361 eq:vandermonde, P:388-394 eq:ext_ab; reading R1 for the moments):
 * alpha (m, oldest node first) with sum_k alpha_k t_k^(i-1) = (b^i - a^i)/i, i = 1..n, of
 * minimum 2-norm when m > n.  nodes: host [m] strictly distinct.  alpha_out: host [m].
 * Errors: INSUFFICIENT_HISTORY (m < n), DEGENERATE_NODES (duplicate nodes), INVALID. */
mrab_status mrab_ab_weights(const double* nodes, int m, int n, double a, double b,
                            double* alpha_out);

/* Host setup (P:227-252 overset phases, reading R17; P:628-637 metrics, reading R3;
 * segments / closures, reading R2).  Builds hole cutting, segment classes, receivers with
 * donor stencils and Lagrange weights, metric terms and the MRAB coefficient tables.
 * Errors: INVALID, MISALIGNED, ORPHAN, SEGMENT, INSUFFICIENT_HISTORY, DEGENERATE_NODES. */
mrab_status mrab_plan_create(const mrab_problem* problem, mrab_plan** out);
void        mrab_plan_destroy(mrab_plan* plan);

/* The overset setup alone (P:227-252 phases: hole cutting, receiver identification, donor
 * search, interpolation weights; reading R17), honouring any caller-supplied iblank / donors
 * in `problem` exactly as mrab_plan_create does.  Outputs are allocated by the library and
 * released with mrab_free:
 *   *iblank_out  int8 [sum_g n_points(g)], the meshes' blanking concatenated in mesh order
 *                (1 active / 0 hole);
 *   *donors_out  mrab_donor [*n_out], receivers of mesh 0 (ascending point), then mesh 1, ...
 * Feeding both back through mrab_mesh_desc.iblank / mrab_problem.donors reproduces the plan
 * bit for bit.  Errors: those of mrab_plan_create; outputs untouched on failure. */
mrab_status mrab_overset_build(const mrab_problem* problem, int8_t** iblank_out,
                               mrab_donor** donors_out, int64_t* n_out);

/* Release an array returned by mrab_overset_build (NULL is a no-op). */
void        mrab_free(void* p);

/* Sizes of mesh `mesh` in a plan: points, active points, receivers (any may be NULL). */
mrab_status mrab_plan_info(const mrab_plan* plan, int mesh, int64_t* n_points,
                           int64_t* n_active, int64_t* n_receivers);

/* Setup tables of `mesh` (each output may be NULL; sizes from mrab_plan_info):
 *   iblank       [n_points]        1 active / 0 hole
 *   recv_point   [R]               flat point index of each receiver (ascending)
 *   recv_donor   [R]               donor mesh
 *   recv_base    [R][3]            donor stencil base (wrapped into [0, n)); [2] = 0 in 2-D
 *   recv_weights [R][3][4]         per-axis Lagrange weights                */
mrab_status mrab_plan_get_tables(const mrab_plan* plan, int mesh, int8_t* iblank,
                                 int64_t* recv_point, int32_t* recv_donor,
                                 int32_t* recv_base, double* recv_weights);

/* SAT face flags of `mesh` (P:279-299 eq:int, P:292-294 edges/corners): flags [n_points],
 * bit 2*kappa set where the point is the kappa-min end of a segment (penalty side "+"),
 * bit 2*kappa+1 where it is the kappa-max end (side "-"); the penalty type follows from the
 * neighbour across that end: a hole or an overset face = interface (qhat interpolated), a
 * far-field / wall face = the physical SAT (R16).  0 at interior and hole points and across
 * periodic seams. */
mrab_status mrab_plan_get_face_flags(const mrab_plan* plan, int mesh, uint8_t* flags);

/* Metric terms of `mesh` (reading R3): jinv [n_points] = J^-1, M [dim][dim][n_points] with
 * M[kappa][i] = J^-1 d kappa / d x_i (zeros at holes). */
mrab_status mrab_plan_get_metrics(const mrab_plan* plan, int mesh, double* jinv, double* M);

/* Device workspace the context needs, in bytes (256-byte aligned base required). */
size_t mrab_workspace_bytes(const mrab_plan* plan);

/* Create a context: uploads tables, metrics and the initial states q0[g] (host or device
 * pointers, dense [nc][n...]) into the caller's device workspace; stream is a
 * cudaStream_t (NULL = legacy default stream).  t = 0, histories empty.
 * Errors: WORKSPACE, CUDA, INVALID. */
mrab_status mrab_create(const mrab_plan* plan, const double* const* q0, void* d_workspace,
                        size_t ws_bytes, void* stream, mrab_ctx** out);
void        mrab_destroy(mrab_ctx* ctx);

/* Advance exactly n_macro macro steps H = S_max h (reading R8).  The first m-1
 * macro steps after create are the RK bootstrap (R5/R6: (m-1) S_max coupled RK3/RK4 micro
 * steps).  Asynchronous on the context stream.  Errors: CUDA, INVALID. */
mrab_status mrab_step(mrab_ctx* ctx, int n_macro);

/* Variable macro step ("The macro-timestep H_i can change on a per-macrostep basis,
 * with the micro-timestep h_i defined such that h_i = H_i/SR"): advance n_macro MRAB macro
 * steps of size H (micro step H / S_max).  The history values of a mesh then sit at
 * non-uniform times; every (partial) AB weight set is recomputed from eq:vandermonde
 * with the actual node times, on the host, per launch (no CUDA graph: the
 * weights are launch arguments).  After the first call, mrab_step also takes this path with
 * H = S_max h.  Asynchronous on the caller's stream.  Errors: INVALID (H <= 0),
 * INSUFFICIENT_HISTORY (called before the m-1 bootstrap macro steps), CUDA. */
mrab_status mrab_step_h(mrab_ctx* ctx, int n_macro, double H);

/* CFL-driven stepping: n_macro macro steps, each of size H = cfl * S_max * min_g dt_g / s_g with
 * dt_g from the device estimate (mrab_dt) at the states the step starts from (eq:ts, P:620-643;
 * h_i = H_i / SR), then mrab_step_h(1, H).  One 8-byte-per-mesh read back per step.
 * *H_last (may be NULL) receives the last step taken.  Errors: as mrab_dt and mrab_step_h;
 * NONFINITE if the estimate is not positive and finite. */
mrab_status mrab_step_cfl(mrab_ctx* ctx, int n_macro, double cfl, double* H_last);

/* MRAB evaluation order ("The order in which we evaluate and advance the solution
 * components" and "whether or not to re-extrapolate the slow state"; the paper prints steps for
 * fastest-first only, reading R-SF of DESIGN.md §2 for the other two).  mrab_step_scheme with
 * MRAB_SCHEME_FASTEST_FIRST is mrab_step.  The slowest-first schemes need exactly two rates
 * (step multiples 1 and S > 1): per macro step the slow meshes' RHS at t + H is evaluated
 * first, from the fast meshes' states extrapolated over [t, t + H]; the fast substeps then
 * read slow states from the extrapolant with history up to t (SLOWEST_FIRST) or re-formed
 * with R_s(t + H) as its newest node (SLOWEST_FIRST_REEXTRAP).  Same kernels, launched
 * directly (no CUDA graph).  The scheme of a context is fixed by its first MRAB step; the
 * history accessors and mrab_step_h apply to fastest-first contexts.  Errors: INVALID. */
enum { MRAB_SCHEME_FASTEST_FIRST = 0, MRAB_SCHEME_SLOWEST_FIRST = 1, MRAB_SCHEME_SLOWEST_FIRST_REEXTRAP = 2 };
mrab_status mrab_step_scheme(mrab_ctx* ctx, int n_macro, int scheme);

/* Multi-GPU: the meshes of a problem are
 * partitioned over the ranks (one process per GPU) and each rank steps the meshes it owns; per
 * RHS evaluation the only exchange is the interpolated donor data, formed on the rank that owns
 * the donor mesh and sent to the rank that owns the receivers (qhat [nc][R], fvhat
 * [d(d+1)][R]), one grouped NCCL send/recv exchange per evaluation round over NVLink.
 *   mrab_partition   owner[g] (host [n_meshes]) by longest-processing-time-first on the weight
 *                    active points x RHS evaluations per macro step (the paper's load-balance
 *                    lesson: rank counts follow work, not points); load (host [nranks], may be
 *                    NULL) receives the per-rank weights.  Deterministic, host only.
 *   mrab_dist_unique_id   128-byte NCCL id (rank 0; broadcast it to the other ranks).
 *   mrab_dist_attach transport MRAB_TRANSPORT_NCCL (id = the 128-byte unique id) or
 *                    MRAB_TRANSPORT_LOOPBACK (id = int* world id: contexts of one process on
 *                    one device play the ranks from separate host threads; test transport).
 *                    Every rank creates the context of the whole problem (same plan, same q0)
 *                    and attaches before its first step; mrab_step / mrab_step_h / mrab_rhs then
 *                    advance (return) the owned meshes only, and mrab_get_state is meaningful
 *                    for owned meshes.  Steps are launched directly (no CUDA graph).
 *   mrab_dist_stats  bytes and messages this rank has sent.
 * Errors: INVALID, CUDA (NCCL missing or failing). */
enum { MRAB_TRANSPORT_NCCL = 0, MRAB_TRANSPORT_LOOPBACK = 1 };
mrab_status mrab_partition(const mrab_plan* plan, int nranks, int* owner, double* load);
mrab_status mrab_dist_unique_id(void* out128);
mrab_status mrab_dist_attach(mrab_ctx* ctx, int transport, const void* id, int rank, int nranks,
                             const int* owner);
mrab_status mrab_dist_stats(mrab_ctx* ctx, int64_t* bytes_sent, int64_t* messages);

/* Reference Runge-Kutta integrator (r_RK4 = dt / dt_RK4 normalises the stability
 * tables): n_steps coupled single-rate steps of size h of every mesh with the classical RK4
 * (order 4) or Heun's RK3 (order 3, reading R5), the same stage kernels as the bootstrap.  The
 * AB histories are not touched, so a context driven this way is an RK integrator (do not mix
 * with MRAB steps).  Asynchronous on the caller's stream.  Errors: INVALID, CUDA. */
mrab_status mrab_rk_step(mrab_ctx* ctx, int n_steps, int order, double h);

/* Stable-timestep estimate on the device (eq:ts_inv, eq:ts_visc, eq:ts_overall, P:620-643;
 * reading R20 of DESIGN.md for the garbled parentheses): dt_mesh[g] (host, [n_meshes]) =
 * min over the active points of mesh g, at its current state, of
 *   J^-1 / [ sum_k (|U . M_k| + c |M_k|) + 2 nu* J (sum_k |M_k|)^2 ],  M_k = J^-1 grad(kappa_k),
 * nu* = max(1, gamma/Pr)/(rho Re) (viscous problems; Euler: the first sum only).  One
 * reduction kernel per mesh; synchronises (8 bytes per mesh come back).  The caller forms
 * H = CFL * S_max * min_g dt_mesh[g] / s_g and passes it to mrab_step_h.  Errors: INVALID, CUDA. */
mrab_status mrab_dt(mrab_ctx* ctx, double* dt_mesh);

/* Copy mesh `mesh`'s state at the current macro boundary to dst (host or device, dense
 * [nc][n...]); *t (may be NULL) receives the time.  Synchronises. */
mrab_status mrab_get_state(mrab_ctx* ctx, int mesh, double* dst, double* t);

/* Overwrite mesh `mesh`'s state at the current macro boundary from src (host or device,
 * dense [nc][n...]); the RHS histories are kept.  Synchronises. */
mrab_status mrab_set_state(mrab_ctx* ctx, int mesh, const double* src);

/* Integrator history access for the step-matrix stability procedure (eq:sm, eq:sm_form,
 * "the stability vector element being perturbed may also be a right-hand side
 * history element").  At a macro boundary t after the bootstrap the integrator vector of
 * mesh g is its state plus m-1 committed RHS history entries R(t - (m-1-k) h_g), k = 0
 * (oldest) .. m-2; R(t) itself is evaluated by the next mrab_step (deferred
 * RHS).  dst/src: host or device, dense [nc][n...], caller-owned.  Errors: MRAB_E_INVALID
 * (bad mesh, k outside [0, m-2], NULL pointer), MRAB_E_INSUFFICIENT_HISTORY (called before
 * the m-1 bootstrap macro steps are done).  Synchronise. */
mrab_status mrab_get_history(mrab_ctx* ctx, int mesh, int k, double* dst);
mrab_status mrab_set_history(mrab_ctx* ctx, int mesh, int k, const double* src);

/* Parity hook: one coupled RHS evaluation (eq:int) of every mesh at the given
 * states q[g] (host or device, dense) -> rhs_out[g] (host or device, dense).  Does not
 * change the integrator state.  Synchronises. */
mrab_status mrab_rhs(mrab_ctx* ctx, const double* const* q, double* const* rhs_out);

/* Counters since create: RHS evaluations per mesh (rhs_evals[n_meshes]), sum over meshes of
 * active points x evaluations, macro steps taken (bootstrap included). */
mrab_status mrab_get_counters(mrab_ctx* ctx, int64_t* rhs_evals, int64_t* point_rhs,
                              int64_t* macro_steps);

/* Kernel launches one macro step issues (for the bench's gpu_launches claim). */
mrab_status mrab_launches_per_macro_step(mrab_ctx* ctx, int64_t* launches);

/* Live timing of one hot kernel of mesh `mesh` exactly as the MRAB step launches it, but
 * writing to scratch buffers (the integrator state is not changed): kernel 0 = fused
 * RHS + SAT + AB update, 1 = viscous-flux pass, 2 = donor gather of this mesh's receivers;
 * 2-D diagnostics: 3 = the interior tiles alone in the lean-only kernel, 4 = the same tiles in
 * the mixed kernel, 5 = the non-interior tiles alone (their algorithmic bytes only).
 * Each of `reps` launches is bracketed by CUDA events on the context stream; with
 * flush_l2 != 0 a 256 MiB buffer is written between launches (outside the events).
 * Outputs: mean ms per launch, and the kernel's ALGORITHMIC bytes per launch.
 * Synchronises. */
mrab_status mrab_time_kernel(mrab_ctx* ctx, int kernel, int mesh, int reps, int flush_l2,
                             double* ms_per_launch, double* algorithmic_bytes);

/* Diagnostics: record a launch timeline of the 2-D MRAB step into `dev_buf` (device memory,
 * u64: [0] record count (zero it before stepping), [1] capacity in records, then records of
 * 5 u64 = (smid << 56 | CTA index << 16 | tag, CTA start ns, CTA end ns, 2-D RHS: end of
 * phase A ns, end of phase B ns (last tile of the CTA), else 0) from %globaltimer; tag = kind << 12 |
 * mesh << 8 | micro index, kind 1 RHS, 2 donor gather, 3 bulk part of a split RHS).  NULL
 * turns it off.  Drops the captured step graphs (re-captured on the next step).  Not part of
 * the hot path; synchronises. */
mrab_status mrab_set_trace(mrab_ctx* ctx, void* dev_buf);

/* Thread-local message of the last failing call on this thread. */
const char* mrab_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* MRAB_H */
