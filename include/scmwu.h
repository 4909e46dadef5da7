/*
 * scmwu.h — C ABI of the B200-native SCMWU feasibility-test engine.
 *
 * Drop-in boundary for the reference's hot path (R = /root/reference/pkg/src/symcone/):
 *
 *   sc_create       replaces the per-solve setup in solve_ses / solve_svm
 *                   (R/ses.py:147-169, R/svm.py:164-187): the instance is copied to HBM
 *                   once; the OracleSpec factory's constants (cone, width rho,
 *                   trace bound R, rank) become handle properties.
 *   sc_ftp          replaces ONE call of meta.solve_ftp (R/meta.py:244-395) or
 *                   meta.refine_run (R/meta.py:457-573) — the whole iteration loop,
 *                   including every Scmwu.current/observe (R/mwu.py:57-70), oracle
 *                   query (R/ses.py:90-132, R/svm.py:97-127), progress evaluation
 *                   (R/ses.py:82-87, R/svm.py:87-94) and pd_counter (R/svm.py:173-181),
 *                   runs inside one persistent kernel launch.
 *   sc_progress     replaces ses_progress / svm_progress at a host-given point
 *                   (seed certificates R/ses.py:174-176, R/svm.py:194-199 and the final
 *                   enclosure slack R/ses.py:187).
 *   sc_iterate      materialises the trace-one iterate p of the last sc_ftp call
 *                   (PrimalCertificate.p / DualFeasible.p_last, R/meta.py:123,132).
 *   sc_pd_commit /  keep the best polytope-distance pair across calls and materialise
 *   sc_pd_pair      it (best_pd in R/svm.py:171-181, read at :229-231).
 *   sc_solve        replaces meta.adaptive_search (R/meta.py:656-781) with _Bracket
 *                   (R/meta.py:576-653) as driven by solve_ses / solve_svm (R/ses.py:
 *                   171-187, R/svm.py:189-214): the seed certificate, every bracketing
 *                   test and refine round, and the final enclosure check run inside ONE
 *                   persistent kernel launch (no host round trip between the tests).
 *
 * Conventions: plain pointers and sizes, caller-owned host buffers are only read
 * (or written) during the call, all device memory is owned by the handle, one
 * handle = one thread of control (R/mwu.py:41-43).  Status codes:
 */
#ifndef SCMWU_H
#define SCMWU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum sc_status {
    SC_OK = 0,
    SC_EARG = 1,       /* bad argument (ValueError in the reference) */
    SC_ECUDA = 2,      /* CUDA runtime error / no device */
    SC_ENCCL = 3,      /* cross-GPU exchange error */
    SC_EWIDTH = 4,     /* witness residual exceeded the width: WidthViolationError */
    SC_EOOM = 5,       /* device allocation failed */
    SC_ETRACE = 6      /* non-positive trace while normalising (ValueError, R/cones.py:417) */
};

enum sc_kind { SC_SES = 0, SC_SVM = 1 };
enum sc_mode { SC_MODE_FTP = 0, SC_MODE_REFINE = 1 };
enum sc_result_kind { SC_PRIMAL = 0, SC_DUAL = 1 };
enum sc_reason {
    SC_REASON_SEPARATED = 0,
    SC_REASON_EXHAUSTED = 1,
    SC_REASON_EARLY_STOP = 2,
    SC_REASON_AFFIRMATIVE = 3,
    SC_REASON_REFINED = 4
};

typedef struct sc_handle sc_handle;

/* Problem constants, computed by the caller exactly as the reference does. */
typedef struct {
    int32_t kind;      /* SC_SES or SC_SVM */
    int32_t d;         /* point dimension */
    int64_t n;         /* number of points (SES) / n1 + n2 (SVM) */
    int64_t n1;        /* SVM: the first n1 rows are P, the rest Q; SES: ignored */
    double D;          /* SES: ses_range D (R/ses.py:65-72); SVM: max_norm (R/svm.py:62-66) */
    double rho;        /* width: 3D/sqrt2 (R/ses.py:161) or 2D (R/svm.py:168) */
    double R;          /* trace bound: sqrt2 (R/ses.py:169) or 2 (R/svm.py:186) */
    int64_t rank;      /* cone rank: 2(n-1) (SES) or n (SVM) (R/cones.py:72-74) */
    double ln_r;       /* math.log(rank) evaluated on the host (bit-exact with Python) */
    int32_t grid;      /* CTAs of the persistent kernel (0 = auto) */
    int32_t device;    /* CUDA device ordinal */
    /* row sharding across GPUs (one process per GPU); world <= 1: single GPU.
     * Rows [row0, row0 + n_local) of the global matrix live on this rank; n1_local of
     * them (the first ones) are SVM P rows.  `n`, `n1`, D, rho, rank stay global. */
    int32_t world;
    int32_t shard;     /* this rank's index in [0, world) */
    int64_t row0;
    int64_t n_local;
    int64_t n1_local;
} sc_problem;

/* One feasibility test. */
typedef struct {
    int32_t mode;          /* SC_MODE_FTP or SC_MODE_REFINE */
    int32_t has_progress;  /* FTP: progress callback present (always 1 in the solvers) */
    double alpha;          /* level */
    double eps;            /* FTP: requested tolerance */
    int64_t budget;        /* FTP: min(iteration_bound, cap) (R/meta.py:282-284); REFINE: unused */
    int64_t horizon;       /* REFINE: max(horizon, ceil(ln r)) (R/meta.py:479) */
    int64_t ceil_ln_r;     /* math.ceil(ln r) */
    double delta;          /* EarlyStopConfig.delta */
    int32_t patience;      /* EarlyStopConfig.patience */
    int32_t enabled;       /* EarlyStopConfig.enabled */
    double gain_rel;       /* REFINE: gain_rel (already defaulted to delta) */
    double lo, hi;         /* REFINE: bracket bounds (-inf/+inf when absent) */
    double target;         /* REFINE: target relative width; NaN = none */
} sc_ftp_args;

/* Outcome of one feasibility test.  Vector outputs are written to caller
 * buffers of dual_dim = d+1 (SES) or d+2 (SVM) doubles. */
typedef struct {
    int32_t kind;          /* SC_PRIMAL or SC_DUAL */
    int32_t reason;        /* enum sc_reason */
    int64_t iterations;
    double eps_eff;        /* DUAL */
    double value;          /* DUAL: certified claim value */
    double oracle_value;   /* PRIMAL: the negative oracle value */
    int32_t has_best_f, has_best_counter, has_claim_y;
    double best_f, best_counter;
    /* width violation (status SC_EWIDTH) */
    int64_t width_iteration;
    double width_norm;
    /* SVM polytope-distance bookkeeping (R/svm.py:173-181, :201-204) */
    int32_t has_counter_min;  /* a pd_counter evaluation happened in this call */
    double counter_min;       /* smallest distance seen in this call (strict <) */
    double sep_dist;          /* PRIMAL: |P^T mu - Q^T gam| of the separating iterate */
    /* device-side timing and work accounting of this call */
    int64_t passes;           /* streaming passes over X executed */
    float kernel_ms;          /* CUDA-event time of the persistent kernel */
    int64_t width_passes;     /* SES: passes that evaluated the exact width residuals (the
                                 others were certified by the bound of DESIGN.md §4.4) */
} sc_ftp_result;

/* Whole-solve residency (sc_solve): the arguments of adaptive_search as solve_ses /
 * solve_svm call it (R/ses.py:178-183, R/svm.py:207-214). */
typedef struct {
    double eps;                /* search eps (SVM: 0.4 * eps, R/svm.py:150, :209) */
    double L0, U0;             /* initial range */
    double delta;              /* EarlyStopConfig */
    int32_t patience;
    int32_t enabled;
    int64_t cap;               /* iteration_cap_override, or < 0 for none */
    int64_t ceil_ln_r;         /* math.ceil(ln r) */
    int64_t refine_horizon;    /* REFINE_HORIZON (R/meta.py:452) */
    double zero_lower_floor;   /* SVM: _INFEASIBLE_FLOOR * 2D; NaN = none */
    int32_t on_primal;         /* SVM: separations certify the pd distance (R/svm.py:201-204) */
    int32_t max_steps;         /* capacity of the caller's step log (<= 400 steps happen) */
} sc_solve_args;

/* One SearchStep (R/meta.py:150-160). */
typedef struct {
    double alpha, eps;
    int64_t iteration_bound, iterations;
    int32_t separated, reason; /* enum sc_reason */
} sc_search_step;

enum sc_termination { SC_TERM_ITERATION_CAP = 0, SC_TERM_RANGE_CONVERGED = 1,
                      SC_TERM_EARLY_STOPPED = 2 };

typedef struct {
    double lower, upper;       /* the bracket at exit (SearchResult.lower / upper) */
    double best_value;         /* SearchResult.best_value */
    int32_t has_best;          /* a certified payload exists (else RuntimeError) */
    int32_t termination;       /* enum sc_termination */
    int64_t total_iterations;
    int32_t search_steps;
    int32_t has_pd;            /* SVM: a pd_counter distance was committed (best_pd) */
    double pd_dist;            /* SVM: best_pd["dist"] */
    double seed_f;             /* progress of the seed point (R/ses.py:175, R/svm.py:198) */
    double final_f;            /* SES: progress at the returned centre (slack = final_f -
                                  best_value, R/ses.py:187) */
    /* width violation (status SC_EWIDTH): the failing test's level and iteration */
    double width_alpha;
    int64_t width_iteration;
    double width_norm;
    int64_t passes;
    float kernel_ms;
    int64_t width_passes;
} sc_solve_result;

/* X: row-major host rows.  SES: n rows (centres), radii n values.  SVM: the n1
 * rows of P; X_tail (if not NULL) holds the n - n1 rows of Q, otherwise X
 * holds all n rows; radii must be NULL. */
int sc_create(const sc_problem* prob, const double* X, const double* X_tail,
              const double* radii, sc_handle** out);
/* On-device synthetic instances: the same distributions as
 * instances.gen_ses / gen_svm (R/instances.py:155-199), drawn with a counter-based
 * Philox4x32-10 keyed by (seed, GLOBAL row index), so every shard generates its own rows
 * and the instance does not depend on the sharding.  Not the bits of numpy's PCG64:
 * only the distribution matches.  X never exists on the host. */
enum sc_gen_dist { SC_GEN_GAUSSIAN = 0, SC_GEN_UNIFORM_BALL = 1, SC_GEN_SPHERE_SURFACE = 2,
                   SC_GEN_SVM_CLUSTERS = 3 };
typedef struct {
    int32_t dist;               /* an sc_gen_dist value: SES 0-2, SVM 3 */
    uint64_t seed;
    double gap;                 /* SVM: cluster gap */
    const double* direction;    /* SVM: unit separating direction (d values, host) */
} sc_gen;
/* prob->D / rho / R / rank / ln_r are filled in by the call (D computed on the device:
 * SES max_i |v_1 - v_i|, SVM max_i |x_i|, over THIS shard's rows; sharded callers reduce
 * the shards' D with max and hand it to sc_set_range).  v1_out (SES, d values: the global
 * row 0, drawn by every shard) may be NULL. */
int sc_create_generated(sc_problem* prob, const sc_gen* gen, double* v1_out,
                        sc_handle** out);
/* Set the range D; rho, R, rank and ln_r follow as in the solvers (R/ses.py:161,169,
 * R/svm.py:168,186). */
int sc_set_range(sc_handle* h, double D);
/* The range D over this handle's resident rows, bit-identical to the reference's numpy
 * expression: SES max over global rows i >= 1 of |v_i - v_1| + g_1 + g_i (R/ses.py:65-72;
 * a shard without row 0 needs v_1 and g_1 from sc_set_globals first), SVM max_i |x_i|
 * (R/svm.py:62-66).  Row norms follow np.linalg.norm's pairwise summation order
 * (csrc/np_rownorm.h), so sharded callers max-reduce the shards' values and every rank
 * gets the single-process D; -inf for a shard with no such row.  Replaces the O(nd) host
 * scan of ses_range / max_norm before sc_set_range. */
int sc_row_range(sc_handle* h, double* D_out);
/* Copy `count` resident rows starting at local row `first` to out (count x d, row-major). */
int sc_read_rows(sc_handle* h, int64_t first, int64_t count, double* out);
/* Independent verification baselines over a resident single-GPU instance (SURVEY §8(f)
 * row 3), one cooperative launch each:
 *   sc_meb_baseline      Badoiu-Clarkson walk of R/baselines.py:34-85 (meb_baseline) for
 *                        `iters` = ceil(1/eps_base^2) steps on an SES handle; center (d) and
 *                        the covering radius max_i |v_i - c| + r_i (value, may be NULL).
 *   sc_gilbert_baseline  Frank-Wolfe / Gilbert of R/baselines.py:88-161 on an SVM handle:
 *                        |z| (value), the last linearisation gap, the iteration count and,
 *                        if not NULL, the weights mu (n1) / gam (n - n1). */
int sc_meb_baseline(sc_handle* h, int64_t iters, double* center, double* value);
int sc_gilbert_baseline(sc_handle* h, double gap_tol, int64_t max_iters, double* value,
                        double* gap, int64_t* iterations, double* mu, double* gam);
int sc_ftp(sc_handle* h, const sc_ftp_args* args, sc_ftp_result* res,
           double* y_tilde /* dual_dim */, double* best_y /* dual_dim */);
int sc_progress(sc_handle* h, const double* y /* d values */, double* f);
/* A whole solve in one launch.  seed_y: the seed point's first d coordinates (SES the
 * anchor centre v1, SVM the cluster-mean direction w0); best_y (dual_dim) receives
 * SearchResult.best_y and steps the search log (args->max_steps entries). */
int sc_solve(sc_handle* h, const sc_solve_args* args, const double* seed_y,
             sc_solve_result* res, double* best_y, sc_search_step* steps);
int sc_iterate(sc_handle* h, double* p /* SES (n-1)(d+1), SVM n */);
int sc_pd_commit(sc_handle* h, int32_t which /* 0: call minimum, 1: separating iterate,
                                                2: reset to the uniform pair */);
/* Device-side timing of a span of calls: sc_mark(h, 0) records a CUDA event on the
 * handle's stream, sc_mark(h, 1) another one and waits for it; sc_elapsed returns
 * the milliseconds between them (host gaps between launches included). */
int sc_mark(sc_handle* h, int32_t which);
int sc_elapsed(sc_handle* h, float* ms);
/* Kernel launches issued by this handle since creation (persistent + one-off). */
int64_t sc_launches(const sc_handle* h);
/* Diagnostics (builds with -DSCMWU_PHASE_TIMING and SCMWU_TIMING=1 in the environment):
 * out[0..9) per-phase SM-cycle sums of the last sc_ftp as seen by CTA 0 (pass, warp
 * join, CTA partial, barrier 1, fold, barrier 2, reduced read, control tail, tail join),
 * out[9..169) each CTA's streaming cycles, out[169..329) its SM id, out[329..489) and
 * out[489..649) global-timer ns at the start / end of its last pass, out[649..809) and
 * out[809..969) at its arrival at / release from that pass's first grid barrier,
 * out[969..976) cycle sums of the control tail's sections (CTA 0); zeros otherwise. */
int sc_debug_timing(sc_handle* h, double* out);
int sc_pd_pair(sc_handle* h, double* mu /* n1 */, double* gam /* n - n1 */, double* dist);
/* Row sharding (world > 1).  The per-pass exchange runs INSIDE the persistent kernel:
 * each rank writes its folded pass vector into every peer's mailbox over NVLink and
 * raises a system-scope flag; every rank folds the rank vectors in rank order.
 *   sc_local_red0   this shard's contribution to the iterate-1 sums (red_width doubles)
 *   sc_set_globals  the rank-ordered fold of those, plus the anchor row (SES v1, g1)
 *   sc_ipc_handle   64-byte CUDA IPC handle of this rank's mailbox
 *   sc_connect      map the world x 64-byte handles of all ranks (own included)
 * For world <= 1 none of these is needed. */
int sc_local_red0(sc_handle* h, double* out);
/* progress extremes over this shard's rows: SES {max_i |v_i - y| + g_i, 0},
 * SVM {min_P P.y, max_Q Q.y}; the caller folds ranks (max / min / max). */
int sc_progress_parts(sc_handle* h, const double* y, double* out2);
int sc_set_globals(sc_handle* h, const double* red0, const double* v1, double g1);
int sc_ipc_handle(sc_handle* h, void* out64);
int sc_connect(sc_handle* h, const void* handles);
/* Local (this shard's) materialisation for sharded handles: sc_iterate writes the local
 * block of p (SES: (n_local - [shard holds row 0]) blocks, SVM: n_local coordinates) and
 * sc_pd_pair the unnormalised local weights; the host folds the shards. */
int sc_set_grid(sc_handle* h, int32_t grid);
int sc_info(const sc_handle* h, int64_t* out /* 8 values: grid, threads, lanes_per_row,
              cols_per_lane, tile_rows, stages, resident, smem_bytes */);
const char* sc_last_error(const sc_handle* h);
void sc_destroy(sc_handle* h);
int sc_version(void);
/* Release the device memory the engine's private pool keeps mapped for reuse (freed
 * buffers up to SCMWU_POOL_GB, default 12 GiB, stay mapped so a solve per call through the
 * public API does not pay cudaMalloc / cudaFree of the matrix every time). */
int sc_pool_trim(int32_t device);

#ifdef __cplusplus
}
#endif
#endif /* SCMWU_H */
