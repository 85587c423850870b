/*
 * trajopt_b200.h — C-ABI of the B200-native batched AM/AL trajectory-optimizer
 * kernels (libtrajopt_b200.so).  Plain pointers and sizes only; no torch types.
 *
 * Conventions:
 *  - every pointer in the structs below is a DEVICE pointer owned by the caller
 *    (torch tensors in the Python host layer); nothing here allocates;
 *  - every entry point only ENQUEUES work on `stream` (a cudaStream_t passed as
 *    void*; NULL = legacy default stream) and returns a cudaError_t value
 *    (0 = success) or TRO_EINVAL for a host-side argument error;
 *  - one solver instance per stream (the reference's single-owner state rule,
 *    SPEC.md:298).
 *
 * Reference interfaces replaced (file:line into arxiv/paper_2408_10731's
 * `trajopt` package, pkg/src/trajopt/):
 *  - tro_kkt_apply_f64    <- qpcore.solve_batch           (qpcore.py:130-143)
 *  - tro_alg1_prime       <- solver_single.init_state tail + the target/
 *                            multiplier sums _position_step needs
 *                            (solver_single.py:115-166, :177-189, :204-207)
 *  - tro_alg1_iterate     <- solver_single.am_iteration + _residual_extremes +
 *                            _maybe_grow_penalties, i.e. one trip of the loop
 *                            body of solve_single (solver_single.py:373-427)
 *  - tro_topk_stable      <- np.argsort(kind="stable")[:k] (solver_priest.py:358,
 *                            :440) and sorted(key=aug_cost) (:362)
 */
#ifndef TRAJOPT_B200_H
#define TRAJOPT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TRO_EINVAL (-1)

/* storage type of the per-element state */
#define TRO_F64 0
#define TRO_F32 1

/* status bits per member */
#define TRO_CONVERGED 1
#define TRO_FACTOR_FAILED 2

typedef struct tro_alg1_dims {
    int32_t n_members; /* B: members (independent problems) in this launch */
    int32_t n_obs;     /* n_o: obstacles shared by every member */
    int32_t n_p;       /* horizon samples */
    int32_t m;         /* basis columns = degree + 1 (<= 16) */
    int32_t dim;       /* 2 or 3 */
    int32_t n_eq;      /* boundary rows per axis (6: p,v,a at both ends) */
    int32_t n_levels;  /* entries of the K^-1 table */
    int32_t groups;    /* obstacle groups per CTA (one-CTA-per-member kernel); 0 = automatic */
    int32_t layout;    /* TRO_LAYOUT_ANGLE or TRO_LAYOUT_UNIT (words per element, see tro_alg1_state) */
    int32_t reserved;
} tro_alg1_dims;

/* per-element state layouts */
#define TRO_LAYOUT_ANGLE 0 /* 3-D [alpha beta lx ly lz lca lsa lcb lsb] (9 words), 2-D [alpha lx ly lca lsa] (5) */
#define TRO_LAYOUT_UNIT 1  /* angles kept as unit vectors: 3-D [ca sa cb sb lx ly lz lca lsa lcb lsb] (11),
                              2-D [ca sa lx ly lca lsa] (6) */
#define TRO_LAYOUT_HALF 2  /* the reference's word count (9 / 5), each angle as a folded half-angle tangent
                              w: |w| <= 1: tan(a/2); else 3 sgn(w) + tan((a - pi sgn(w)) / 2) */

typedef struct tro_alg1_consts {
    const double* P;         /* n_p x m, row-major (basis.py:143-177) */
    const double* tracks;    /* n_o x dim x n_p, obstacle centres (per obstacle: x row, y row, z row) */
    const double* shape_a;   /* n_o semi-axis a (x,y) */
    const double* shape_b;   /* n_o semi-axis b (z; y in 2-D) */
    const double* kinv;      /* n_levels x nk x nk row-major, nk = m + n_eq */
    const double* level_rho; /* n_levels: the rho_o each table entry was built at */
    const int32_t* level_ok; /* n_levels: 1 if that level passed the cond guard */
    const double* q;         /* B x dim x m: -2 w_track P^T desired (solver_single.py:173) */
    const double* bvals;     /* B x dim x n_eq boundary values */
    const double* line_u;    /* m: lstsq(P, 1)      straight-line init xi = u p0 + v (p1 - p0) */
    const double* line_v;    /* m: lstsq(P, tau)    (basis.py:207-217, used by tro_alg1_init) */
    const int32_t* level0;   /* B: each member's cold-start level (the K^-1 table entry built at rho_start).
                                Non-NULL: tro_alg1_init is a complete cold start (solver_single.py:115-166):
                                it also sets rho = rho_o = level_rho[level0[i]], level = level0[i] and zeroes
                                iteration, last_change, n_hist, n_changes, status and the stall ring.
                                NULL: tro_alg1_init leaves that bookkeeping to the caller (the MPC fleet). */
    const double* track_lin; /* optional constant-velocity description of `tracks`: n_o records of 6 doubles
                                (3-D {cx cy cz vx vy vz}, 2-D {cx cy vx vy 0 0}) then n_p times rel[t], with
                                tracks[j][ax][t] == c + v * rel[t] BITWISE (one rounded product, one rounded
                                sum, as numpy's c + v * rel).  Non-NULL: the TMA iteration kernel generates the
                                track rows in registers instead of streaming them (NULL: stream `tracks`). */
} tro_alg1_consts;

typedef struct tro_alg1_params {
    double tol;               /* SingleParams.tol */
    double rho_growth;        /* SingleParams.rho_growth */
    double rho_cap;           /* SingleParams.rho_cap */
    double stall_improvement; /* SingleParams.stall_improvement */
    int32_t stall_window;     /* SingleParams.stall_window (<= 32) */
    int32_t d_mode;           /* 0: d == 1 (cold start), 1: read state.d, 2: recompute from pos */
    int32_t max_hist;         /* history capacity per member (0: no history output) */
    int32_t flags;            /* TRO_FLAG_* */
} tro_alg1_params;

/* tro_alg1_params.flags */
#define TRO_FLAG_NO_SCHEDULE 1 /* bare am_iteration: no convergence test, no penalty growth */
#define TRO_FLAG_NO_TMA 2      /* force the one-CTA-per-member kernel (testing / tuning) */

typedef struct tro_alg1_state {
    /* persistent per-element state, storage type T, interleaved per obstacle row:
     *   state[i][j][w][t]  (B x n_o x W x n_p), words per tro_alg1_dims.layout */
    void* state;
    void* d;       /* optional B x n_o x n_p: read when d_mode == 1, written (new d) when non-NULL */
    void* copies;  /* optional export of the angle copies, planes of B x n_o x n_p:
                      3-D [ca sa cb sb], 2-D [ca sa]; NULL = skip */
    /* per member, fp64 */
    double* xi;    /* B x dim x m */
    double* pos;   /* B x dim x n_p  (positions of the current xi) */
    double* sums;  /* B x 2 x dim x n_p : [sum_j lam_pos ; sum_j targets] for the next position step */
    double* rho;
    double* rho_o;
    double* ring;     /* B x 2*stall_window: last max_abs values (oldest first, rolling) */
    double* res_norm; /* B: residual norm of the latest iterate */
    double* res_max;  /* B: residual max-abs of the latest iterate */
    double* hist;     /* B x max_hist x 3 (norm, max_abs, rho_o) or NULL */
    int32_t* level;       /* B: index into the K^-1 table of the current rho_o */
    int32_t* iteration;   /* B: state.iteration */
    int32_t* last_change; /* B: iteration of the last penalty growth (solve-local) */
    int32_t* n_hist;      /* B: iterations recorded in this solve */
    int32_t* status;      /* B: TRO_CONVERGED | TRO_FACTOR_FAILED */
    int32_t* n_changes;   /* B: rho_o changes in this solve (new factorizations) */
    /* optional tail balancing of the persistent TMA kernel (NULL: off).  When B is not a multiple of the
     * grid, the last partial round's members are split into two obstacle halves run by two CTAs; the halves'
     * partial sums meet here and the second finisher (ticket) combines them in a fixed order:
     * split_scratch >= 2 x 2 x (2 dim n_p + 2) doubles per grid slot, split_ticket >= 1 zeroed uint32 per slot */
    double* split_scratch;
    uint32_t* split_ticket;
    /* optional member order of the persistent TMA kernel (NULL: members 0..B-1): it works through
     * order[0 .. *n_order) only (e.g. the robots of a fleet still driving; tro_mpc_compact builds it) */
    const int32_t* order;
    const int32_t* n_order;
    /* optional B (NULL: not written): the level of the latest iteration's position step.  Levels only grow by
     * one per change, so a solve factorized levels level0 .. level_used (solver_single.py:198-202): a growth
     * on the final iteration of a run that then stops is not followed by a factorization */
    int32_t* level_used;
} tro_alg1_state;

/* Sums for the first position step + positions of the current xi + residual of the
 * current (copies-reset) state.  Call once before the first tro_alg1_iterate of a solve. */
int tro_alg1_prime(int32_t dtype, const tro_alg1_dims* dims, const tro_alg1_consts* c,
                   const tro_alg1_state* s, const tro_alg1_params* p, void* stream);

/* Cold start (solver_single.init_state, solver_single.py:115-166): straight-line xi,
 * angles from the line offsets, zero multipliers, d == 1; then everything tro_alg1_prime does. */
int tro_alg1_init(int32_t dtype, const tro_alg1_dims* dims, const tro_alg1_consts* c,
                  const tro_alg1_state* s, const tro_alg1_params* p, void* stream);

/* One fused AM iteration for every non-frozen member (one kernel launch). */
int tro_alg1_iterate(int32_t dtype, const tro_alg1_dims* dims, const tro_alg1_consts* c,
                     const tro_alg1_state* s, const tro_alg1_params* p, void* stream);

/* Up to n_iter fused AM iterations per member in ONE launch (one CTA loops its member; members are
 * independent, so no grid synchronisation): bitwise the same as n_iter tro_alg1_iterate calls, each member
 * stopping at convergence / factor failure.  For small batches (C1) it removes n launches and their
 * pipeline fills; large batches keep the TMA-pipelined tro_alg1_iterate. */
int tro_alg1_iterate_n(int32_t dtype, const tro_alg1_dims* dims, const tro_alg1_consts* c,
                       const tro_alg1_state* s, const tro_alg1_params* p, int32_t n_iter, void* stream);

/* Per-member linear cost terms q = -2 w_track (P' desired_i)' (solver_single.py:173), B x dim x m, on the
 * device.  desired: B x n_p x dim member paths, or NULL for each member's straight start -> goal line
 * desired[t] = p0 + frac[t] (p1 - p0) with p0 = bvals[i][ax][0], p1 = bvals[i][ax][3] (bench/runner.py:88-94;
 * frac = linspace(0, 1, n_p), bitwise numpy's line).  The sum over samples runs in sample order. */
int tro_alg1_linear_terms(int64_t n_members, int32_t n_p, int32_t m, int32_t dim, int32_t n_eq, const double* P,
                          const double* frac, const double* bvals, const double* desired, double w_track, double* q,
                          void* stream);

/* ------------------------------------------------------------------ PRIEST / CEM (Alg. 3) */
typedef struct tro_priest_dims {
    int64_t n_samples; /* N */
    int32_t n_p;       /* horizon samples */
    int32_t m;         /* basis columns */
    int32_t dim;       /* 2 or 3 */
    int32_t n_obs;     /* obstacles */
    int32_t n_eq;      /* boundary equality rows (all axes) */
    int32_t n_inner;   /* inner projection iterations */
} tro_priest_dims;

typedef struct tro_priest_consts {
    const double* P;       /* n_p x m */
    const double* Pd;      /* n_p x m */
    const double* Pdd;     /* n_p x m */
    const double* tracks;  /* n_o x dim x n_p obstacle centres */
    const double* shape_a; /* n_o */
    const double* shape_b; /* n_o */
    const double* kinv;    /* nk x nk row-major, nk = dim*m + n_eq: inverse of [[I + rho F'F, A'], [A, 0]] */
    const double* FtF;     /* m x m: the (block-diagonal, per-axis) block of F'F */
    const double* b_eq;    /* n_eq */
    const double* s_min;   /* dim (box bounds, used when has_bounds) */
    const double* s_max;   /* dim */
    const double* mu;      /* dim*m sampling mean */
    const double* draw_L;  /* dim*m x dim*m draw factor u sqrt(s) of svd(Sigma) */
    const double* line;    /* barn-cost start/goal line: x0 y0 x1 y1 */
    double v_max;          /* <= 0: no velocity rows */
    double a_max;          /* <= 0: no acceleration rows */
    double rho;
    int32_t has_bounds;
    int32_t static_tracks; /* 1: every obstacle centre is constant over the horizon */
    int32_t spheres;       /* 1: every obstacle has a == b (one scaled-distance multiplier) */
    int32_t reserved;
} tro_priest_consts;

typedef struct tro_priest_io {
    const double* z;       /* N x dm standard normals: samples = mu + z L' (or NULL) */
    const double* samples; /* N x dm samples when z == NULL */
    double* samples_out;   /* optional N x dm */
    double* xi;            /* N x dm projected coefficients */
    double* scores;        /* N residual scores (solver_priest.py:290-301) */
    double* history;       /* optional n_inner x N scores after every inner iteration */
} tro_priest_io;

/* project() (solver_priest.py:242-287): n_inner projection iterations per sample, then
 * the residual scores of the result.  n_inner = 0 computes residual_scores only;
 * n_inner = -1 only draws the samples (xi = samples). */
int tro_priest_project_f64(const tro_priest_dims* dims, const tro_priest_consts* c, const tro_priest_io* io,
                           void* stream);

/* out[r] = w_barn * barn_cost(traj(xis[index[r]])) + w_score * scores[index[r]]
 *          + w_penalty * cem_penalty(xis[index[r]])
 * (solver_priest.py:475-498, :359-361, :396-419, :438-439).  index == NULL: r itself. */
int tro_priest_cost_f64(const tro_priest_dims* dims, const tro_priest_consts* c, const double* xis,
                        const int64_t* index, int64_t count, const double* scores, double w_barn,
                        double w_score, double w_penalty, double* out, void* stream);

/* Distribution refit from elites xis[rows[k]] with costs[k] (solver_priest.py:317-333); updates mu
 * (dm) and cov (dm x dm) in place.  gamma == 0: plain CEM mean / population covariance (:442-444). */
int tro_elite_update_f64(const double* xis, int32_t dm, const int64_t* rows, int32_t n_elite,
                         const double* costs, double sigma, double gamma, int32_t mode, double* mu, double* cov,
                         void* stream);

/* tro_elite_update_f64 modes: PRIEST's exp-weighted refit with learning rate sigma (gamma used as given,
 * solver_priest.py:317-333), or CEM's plain mean / population covariance (:442-444) */
#define TRO_REFIT_PRIEST 0
#define TRO_REFIT_CEM 1

/* Throughput-mode sampling: standard normals out[s][j] (n_samples x dim, row-major) of
 * samples first_sample .. first_sample + n_samples - 1, Philox4x32-10 keyed by seed, counter = (pair index,
 * stream_id), Box-Muller; a pure function of (seed, stream_id, global sample, j), so shards draw their own
 * rows.  Not numpy's stream (parity mode keeps numpy's Generator draws). */
int tro_normal_philox_f64(uint64_t seed, uint64_t stream_id, int64_t first_sample, int64_t n_samples, int32_t dim,
                          double* out, void* stream);

/* Lower Cholesky factor of a symmetric PSD n x n matrix (n <= the PRIEST coefficient dimension bound), one
 * CTA; non-positive pivots give zero columns.  The throughput-mode draw factor (samples = mu + z L'). */
int tro_cholesky_f64(const double* a, int32_t n, double* l, void* stream);

/* ------------------------------------------------------------------ joint multi-agent (Alg. 5) */
typedef struct tro_ma_dims {
    int32_t n_problems; /* B independent joint problems sharing the pair structure */
    int32_t n_agents;   /* N_a (2 * N_a <= 32) */
    int32_t n_pairs;    /* N_a (N_a - 1) / 2 agent pairs, then N_a per static sphere */
    int32_t n_static;   /* static spheres per problem */
    int32_t n_p;
    int32_t m;          /* basis columns (9 or 11) */
    int32_t n_eq;       /* 6 N_a boundary rows per axis */
    int32_t n_levels;   /* rho levels (one K^-1 each) */
} tro_ma_dims;

typedef struct tro_ma_consts {
    const double* P;         /* n_p x m */
    const double* kinv;      /* n_levels x nk x nk, nk = N_a m + n_eq: inverse of [[Q + rho A_fo'A_fo, A_eq'], [A_eq, 0]] */
    const double* level_rho; /* n_levels */
    const int32_t* pair_i;   /* n_pairs first agent */
    const int32_t* pair_j;   /* n_pairs second agent, -1 for a static partner */
    const int32_t* pair_s;   /* n_pairs static sphere index (static pairs) */
    const double* pair_a;    /* n_pairs inflated semi-axes (solver_multiagent.py:108-130) */
    const double* pair_b;
    const int32_t* inc_ptr;  /* N_a + 1: CSR incidence lists */
    const int32_t* inc_pair; /* p (agent is the first member, +) or -(p + 1) (second member, -) */
    const double* b_eq;      /* B x 3 x n_eq boundary values per axis */
    const double* statics;   /* B x n_static x 3 sphere centres (NULL if n_static == 0) */
    const double* line_u;    /* m: straight-line init coefficients (see tro_alg1_consts) */
    const double* line_v;
    const double* bnd;       /* optional 6 x m boundary rows of one agent (basis.boundary_matrix) and, after them, */
                             /* its m x 6 pseudo-inverse A'(AA')^-1: after each QP step every agent's coefficients */
                             /* are projected onto A c = b_eq (c -= A+ (A c - b_eq)), so the boundary conditions */
                             /* hold to rounding although the explicit K^-1 (cond ~1e12) leaves ~1e-8 there; the */
                             /* projection only removes error (orthogonal onto the constraint set).  NULL: off */
} tro_ma_consts;

typedef struct tro_ma_state {
    double* state;    /* B x n_p x 3 x n_pairs: multipliers (pairs fastest) */
    double* xi;       /* B x 3 x N_a m */
    double* sums;     /* B x 2 x N_a x 3 x m: agent-contracted (recon + statics, lambda) for the next RHS */
    double* ring;     /* B x 2 * stall_window residual norms */
    double* res_norm; /* B */
    double* res_max;  /* B */
    double* hist;     /* B x max_hist x 3 (norm, max, rho) or NULL */
    int32_t* level;
    int32_t* iteration;
    int32_t* last_change;
    int32_t* n_hist;
    int32_t* status;     /* TRO_CONVERGED */
    double* export_d;    /* optional B x n_p x n_pairs: d of the latest iterate */
    double* export_ab;   /* optional 2 planes of B x n_p x n_pairs: alpha, beta */
} tro_ma_state;

typedef struct tro_ma_params {
    double tol_norm;          /* JointParams.tol_norm */
    double stall_improvement; /* JointParams.stall_improvement */
    int32_t stall_window;     /* JointParams.stall_window */
    int32_t max_iter;         /* JointParams.max_iter (the level schedule needs it) */
    int32_t max_hist;         /* history capacity (0: none) */
    int32_t reserved;
} tro_ma_params;

/* mode 2: cold start (_init_state, solver_multiagent.py:228-249) + the first RHS sums;
 * mode 1: prime the RHS sums of a given state (lambda in `state`, d / alpha / beta read from the
 *         export planes) for a warm start;
 * mode 0: one _iterate + residual + level schedule (solver_multiagent.py:252-335);
 * mode 3: the QP step of _iterate alone for every non-converged problem (:266-269), batched on the fp64
 *         tensor cores (mma.sync m8n8k4 f64, 8 problems per CTA, one K^-1 read per CTA);
 * mode 4: the rest of _iterate (angles, d, residual, multipliers, sums, schedule) given mode 3's xi.
 * Modes 3 + 4 == mode 0 (up to the GEMM's summation order). */
int tro_ma_run(int32_t mode, const tro_ma_dims* dims, const tro_ma_consts* c, const tro_ma_state* s,
               const tro_ma_params* p, void* stream);

/* Ozaki int8 tensor-core backend of the mode-3 QP step: the same xi = K_L^-1 [rho B - C ; b_eq] for every
 * non-converged problem, as an exactly-accumulated int8 GEMM on tcgen05 (kind::i8, TMEM accumulators,
 * tensor-map TMA) of n_slices 7-bit slices per operand, with separate exponents for the primal K block
 * [0, nv) and the boundary K block [nv, nk).  a_slices / a_exp: the level inverses' rows K_L^-1[0:nv, 0:nk]
 * split on the host (paper_2408_10731_b200.ozaki.split_blocks): int8
 * [n_levels][n_slices][m_tiles][ks0 + ks1][4096] (128 x 32 canonical no-swizzle K-major blocks) and the
 * per-row exponents int32 [n_levels][2][m_tiles * 128]; b_slices / b_exp: workspaces of
 * [n_slices][n_col_tiles][ks0 + ks1][1024] int8 and [2][n_col_tiles * 32] int32, n_col_tiles >= ceil(3 B / 32);
 * m_tiles = ceil(nv / 128) <= 2, ks0 = ceil(nv / 32), ks1 = ceil(n_eq / 32), each <= 16. */
typedef struct tro_ozaki_ws {
    const int8_t* a_slices;
    const int32_t* a_exp;
    int8_t* b_slices;
    int32_t* b_exp;
    int32_t n_slices;    /* 6, 7 or 8 (truncation ~128^-(n_slices + 1) relative) */
    int32_t n_col_tiles; /* capacity of the B workspaces in 32-column tiles */
} tro_ozaki_ws;

int tro_ma_qp_ozaki(const tro_ma_dims* dims, const tro_ma_consts* c, const tro_ma_state* s, const tro_ozaki_ws* ws,
                    void* stream);

/* ------------------------------------------------------------------ 2-D batch optimizer (Alg. 2)
 * Replaces solver_batch.batch_iteration + the residual / _maybe_grow_rho bookkeeping of
 * solve_batch_opt (solver_batch.py:352-363, 396-406, 451-461) for the whole batch.  One CTA per
 * member; alpha / d are never stored (they are functions of xi and the heading, :318-344): each
 * launch folds them into F'g for the next launch's QP right-hand side. */
typedef struct tro_b2_dims {
    int64_t n_members; /* N_b */
    int32_t n_obs;     /* n_o (0 allowed) */
    int32_t n_c;       /* footprint circles (1..8) */
    int32_t n_p;
    int32_t m;         /* basis columns */
    int32_t n_levels;  /* rho levels (one K_xi^-1 and one K_psi^-1 each) */
    int32_t max_hist;  /* best_history capacity (0: none) */
} tro_b2_dims;

typedef struct tro_b2_consts {
    const double* PT;            /* 3 x m x n_p: P', Pdot', Pddot' */
    const double* Pr;            /* 3 x n_p x m: P, Pdot, Pddot */
    const double* obs;           /* n_obs x 2 x n_p: track x row, y row */
    const double* obs_ab;        /* n_obs x 2: semi-axes (a, b) */
    const double* offsets;       /* n_c signed circle offsets (FootprintSpec.offsets) */
    const double* q;             /* 4m linear cost (_Structure.q, solver_batch.py:170-177) */
    const double* b;             /* 12 boundary values [x(6) | y(6)] */
    const double* b_psi;         /* 2 heading boundary values */
    const double* kinvT_xi;      /* n_levels x (4m + 12) x (4m + 12): K_xi^-1, transposed (all rows) */
    const double* kinvT_psi;     /* n_levels x (m + 2) x m: rows 0..m-1 of K_psi^-1, transposed */
    const double* rho_chain;     /* n_levels: rho per level (min(rho * growth, cap) chain) */
    const double* rho_psi_chain; /* n_levels: rho_psi per level */
    const double* desired;       /* n_p x 2 (member costs, mode 3) */
    double v_max, a_max, w_smooth, w_track;
    const double* k_xi;          /* n_levels x (4m + 12) x (4m + 12): K_xi itself (symmetric); the xi step
                                    refines K^-1 rhs once (r = rhs - K sol, xi += (K^-1 r)[:4m]) so xi carries
                                    the LU solve's rounding floor, not the explicit inverse's */
} tro_b2_consts;

typedef struct tro_b2_state {
    double* xi;        /* N_b x 4m: [xi_x | xi_c | xi_y | xi_s] */
    double* xi_psi;    /* N_b x m */
    double* lam;       /* N_b x 4m */
    double* lam_psi;   /* N_b x m */
    double* sums;      /* N_b x 4m: F'g of the current state (feeds the next xi step) */
    double* res_max;   /* N_b: max |F xi - g| of the current state */
    double* res_norm;  /* N_b: ||F xi - g|| */
    double* ring;      /* 2 * stall_window: batch-min max-abs residuals (solver_batch.py:460) */
    double* hist;      /* max_hist x 4: best member's (norm, max_abs, rho, index) per iteration */
    int32_t* level;    /* current rho level (batch-global) */
    int32_t* iteration;
    int32_t* last_change;
    int32_t* n_hist;
    int32_t* n_changes;
    uint32_t* counter; /* zero-initialised grid ticket (last-CTA-done reduction) */
    /* mode 2 outputs (NULL to skip): BatchState arrays of the current iterate */
    double* alpha_coll; /* N_b x n_c x n_obs x n_p */
    double* d_coll;
    double* alpha_v;    /* N_b x n_p each */
    double* alpha_a;
    double* d_v;
    double* d_a;
    double* psi;        /* N_b x n_p heading samples: read with TRO_B2_PSI_IN, written by modes 0, 2, 3, 5 */
    double* rank;       /* mode 3: N_b x 6 (res_max, res_norm, min scaled distance, max speed, max accel, cost) */
    double* psi_targets; /* mode 5: N_b x n_p unwrapped heading targets (BatchState._psi_targets) */
    double* shard;       /* TRO_B2_SHARD, mode 0: this shard's summary (best norm, best global index, its
                            max |r|, min max |r|) for the all-gather */
    const double* shards_in; /* mode 6: n_shards x 4 all-gathered summaries, rank order */
} tro_b2_state;

typedef struct tro_b2_params {
    double tol;               /* BatchParams.tol */
    double stall_improvement; /* BatchParams.stall_improvement */
    int32_t stall_window;     /* BatchParams.stall_window */
    int32_t flags;            /* TRO_FLAG_NO_SCHEDULE (bare batch_iteration) | TRO_B2_* */
    int64_t member_offset;    /* global index of this launch's member 0 (sharded batches) */
    int32_t n_shards;         /* mode 6: number of shard summaries */
    int32_t reserved;
} tro_b2_params;

#define TRO_B2_PSI_IN 16      /* the current heading is s.psi (state.psi), not P xi_psi */
#define TRO_B2_GIVEN_AD 32    /* modes 1, 3: alpha / d are the state arrays, not implied by xi, psi */
#define TRO_B2_GIVEN_ALPHA 64 /* mode 2: alpha from the state arrays, d computed from it (d_step) */
#define TRO_B2_CIRCLES 128    /* caller guarantees a == b for every obstacle (circle fast path) */
#define TRO_B2_SHARD 256      /* mode 0 writes this shard's summary instead of applying the schedule */

/* mode 0: one batch_iteration + residual + best_history + batch-global rho rule;
 * mode 1: prime F'g (sums) + residual of the state (init_state / warm start);
 * mode 2: write the BatchState alpha / d (/ psi) arrays of the current iterate (alpha_step, d_step);
 * mode 3: ranking quantities (solver_batch.py:366-393, 463-470) into state.rank (+ psi);
 * mode 4: batch_xi_step alone (xi from the primed sums, :292-299);
 * mode 5: heading_step alone (xi_psi, psi, psi_targets, :302-315);
 * mode 6: merge all-gathered shard summaries and apply the batch-global rule (multi-GPU Alg. 2:
 *         mode 0 with TRO_B2_SHARD on every rank, all-gather of the 4-double summaries, mode 6). */
int tro_b2_run(int32_t mode, const tro_b2_dims* dims, const tro_b2_consts* c, const tro_b2_state* s,
               const tro_b2_params* p, void* stream);

/* ------------------------------------------------------------------ batched post-solve validation (§8(f) 3)
 * Replaces bench/metrics.py eval_metrics / check_collision_free / clearance_lower_bound (metrics.py:26-95)
 * for a batch of trajectories against the RAW scenario geometry (constant-velocity obstacles, scenarios.py:
 * 118-127).  One warp per member. */
typedef struct tro_val_dims {
    int64_t n_members;
    int32_t n_obs;
    int32_t n_p;
    int32_t m;                  /* basis columns (coefficient input) */
    int32_t dim;                /* 2 or 3 */
    int32_t per_member_desired; /* 1: desired is n_members x n_p x dim, 0: n_p x dim shared */
    int32_t reserved;
} tro_val_dims;

typedef struct tro_val_consts {
    const double* P;          /* n_p x m (coefficient input) */
    const double* Pdd;        /* n_p x m */
    const double* t;          /* n_p sample times */
    const double* centers;    /* n_obs x dim obstacle centres at t[0] */
    const double* velocities; /* n_obs x dim */
    const double* shape_a;    /* n_obs raw semi-axes (no planning inflation) */
    const double* shape_b;
    const double* desired;    /* NULL: tracking = 0 */
    double margin;            /* check_collision_free margin on the scaled-distance axis */
} tro_val_consts;

typedef struct tro_val_io {
    const double* xi;  /* n_members x dim x m coefficients, or NULL to use pos / acc samples */
    const double* pos; /* n_members x n_p x dim */
    const double* acc; /* n_members x n_p x dim */
    double* out;       /* n_members x 5: smoothness, tracking, arc length, worst incursion, clearance bound */
} tro_val_io;

int tro_validate_f64(const tro_val_dims* dims, const tro_val_consts* c, const tro_val_io* io, void* stream);

/* ---------------- §8(f) row 1: device predict_obstacles (bench/scenarios.py:118-127)
 * centres c + v (t_now[s] + t[k] - t[0]) of every obstacle of S scenarios (or of one obstacle table at S
 * prediction times), in the reference's operation order without FMA contraction (bit-exact with numpy). */
typedef struct tro_track_dims {
    int32_t n_scen;           /* S */
    int32_t n_obs;
    int32_t n_p;
    int32_t dim;              /* 2 or 3 */
    int32_t layout;           /* 0: out S x n_obs x n_p x dim (predict_obstacles), 1: S x n_obs x dim x n_p
                                 (tro_alg1_consts.tracks) */
    int32_t shared_obstacles; /* 1: centers / velocities are one n_obs x dim table for all S */
} tro_track_dims;

int tro_predict_tracks_f64(const tro_track_dims* dims, const double* centers, const double* velocities,
                           const double* t, const double* t_now, double* out, void* stream);

/* ---------------- §8(f) row 2: receding-horizon fleet step (bench/runner.py:326-439)
 * B robots driving through one scenario with device-resident warm state (an Alg. 1 engine).  After a
 * control step's solve, mode 1 executes the first n_exec samples of each active member's plan against the
 * true obstacle motion (collision at t_exec[k], goal proximity; runner.py:406-419), appends them to the
 * trace, writes the next problem (boundary = executed state, straight desired line to the goal and its
 * linear term q = -2 w_track P' desired), the warm line-of-sight scales d of the final iterate (read by
 * the next prime with d_mode 1) and resets the engine's solve-local bookkeeping (runner.py:376-377:
 * iteration = 0).  Mode 0 starts the episode from bvals' p0 (collision check at t = 0, first problem).
 * Members that collided or reached the goal are frozen (engine status TRO_CONVERGED). */
typedef struct tro_mpc_dims {
    int32_t n_members;
    int32_t n_obs;
    int32_t n_p;
    int32_t m;
    int32_t dim;
    int32_t n_exec;      /* samples executed per control step */
    int32_t trace_cap;   /* trace capacity per member (1 + n_steps * n_exec) */
    int32_t ring_len;    /* engine stall ring length (2 * stall_window) */
} tro_mpc_dims;

typedef struct tro_mpc_consts {
    const double* P;          /* n_p x m */
    const double* Pdot;
    const double* Pddot;
    const double* frac;       /* n_p: linspace(0, 1, n_p) */
    const double* goal;       /* B x dim */
    const double* centers;    /* n_obs x dim raw obstacle centres at t = 0 */
    const double* velocities; /* n_obs x dim */
    const double* shape_a;    /* n_obs raw semi-axes (collision test) */
    const double* shape_b;
    const double* plan_a;     /* n_obs planning semi-axes (the engine's, for d) */
    const double* plan_b;
    const double* tracks;     /* n_obs x dim x n_p: the tracks this step's solve used */
    const double* t_exec;     /* n_exec absolute times of the executed samples (t_abs += dt, in order) */
    double goal_radius;
    double w_track;
} tro_mpc_consts;

typedef struct tro_mpc_io {
    double* bvals;      /* B x dim x 6: next problem's boundary values (engine bvals) */
    double* q;          /* B x dim x m: next problem's linear term (engine q) */
    double* desired;    /* B x n_p x dim: next problem's desired line */
    double* d;          /* B x n_obs x n_p: warm d for the next prime (NULL: skip) */
    double* trace;      /* B x trace_cap x dim executed positions */
    int32_t* n_trace;   /* B */
    int32_t* flags;     /* B: 1 collided, 2 reached (either: done) */
    double* res_out;    /* optional B: this step's residual norm (copied from the engine) */
} tro_mpc_io;

int tro_mpc_advance_f64(int32_t mode, const tro_mpc_dims* dims, const tro_mpc_consts* c,
                        const tro_alg1_state* engine, const tro_mpc_io* io, void* stream);

/* order[0 .. *n_order) = the members with flags == 0 in increasing index (one CTA; n_members <= 2^31). */
int tro_mpc_compact(int32_t n_members, const int32_t* flags, int32_t* order, int32_t* n_order, void* stream);

/* out (ncols x n) = rhs (ncols x n) * K^-T, i.e. out[c] = K^-1 rhs[c] for every column c.
 * kinv: n x n row-major.  qpcore.solve_batch with the RHS block [-q ; b]. */
int tro_kkt_apply_f64(const double* kinv, int32_t n, const double* rhs, int64_t ncols,
                      double* out, void* stream);

/* Stable ascending top-k: out_idx[0..k) = indices of the k smallest keys, ties broken
 * by index (== np.argsort(keys, kind="stable")[:k]).  NaN sorts last.  keys: n fp64. */
int tro_topk_stable_f64(const double* keys, int64_t n, int32_t k, int64_t* out_idx,
                        void* workspace, int64_t workspace_bytes, void* stream);
int64_t tro_topk_workspace_bytes(int64_t n, int32_t k);

/* Diagnostics: evaluate the kernels' elementary functions elementwise (fp64) so their
 * accuracy can be checked against numpy.  fn: 0 sin(x), 1 cos(x), 2 atan2(y, x),
 * 3 1/x, 4 1/sqrt(x), 5 sqrt(x), 6/7 cos/sin(atan2(y, x)) via normalisation,
 * 8 min(max(1, sqrt(x)), 1e6). */
int tro_fastmath_eval(int32_t fn, const double* x, const double* y, int64_t n, double* out, void* stream);

/* FP64 FMA throughput probe: blocks x 256 threads x iters x 8 DFMA (2 flops each). */
int tro_fp64_fma_probe(int64_t iters, int32_t blocks, double* scratch, void* stream);

int32_t tro_version(void);
const char* tro_error_string(int32_t code);

#ifdef __cplusplus
}
#endif

#endif /* TRAJOPT_B200_H */
