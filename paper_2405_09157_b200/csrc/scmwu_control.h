// scmwu_control.h — the per-iteration control of one feasibility test, run
// on the device between streaming passes (the "K3 tail" of DESIGN.md).
//
// It restates, with the deferred-check schedule of DESIGN.md §4, the loop
// bodies of meta.solve_ftp (R/meta.py:294-395) and meta.refine_run
// (R/meta.py:499-573), the oracle epilogues of ses_oracle (R/ses.py:101-132)
// and svm_oracle (R/svm.py:101-127), and the bookkeeping of _ProgressState
// (R/meta.py:398-429), _dual_feasible (R/meta.py:436-446) and pd_counter
// (R/svm.py:173-181).  R = /root/reference/pkg/src/symcone/.
//
// Pass k (one stream over X) reduces, from the state after iteration k-1:
//   * the oracle sums of iterate k (closed form of the cumulative loss, so the
//     learner state is O(d): DESIGN.md §3), and
//   * every check of iteration k-1 (width, progress of the averages, window
//     average, SVM candidate margin and counter candidate).
// after_pass() then finishes iteration k-1 in reference order and, unless
// that terminates the test, runs iterate k's separation test and update.
//
// Every lane of the executing warp runs this code redundantly on private
// scalars; the O(d) vectors live in shared memory and are partitioned by
// index (element j is owned by lane j % nl), so no intra-warp hazards exist.
// The same header compiles for the host (tests/emu), with one lane.
#pragma once

#include <math.h>
#include <stdint.h>

#include "../../include/scmwu.h"

#if defined(__CUDACC__)
#define SC_HD __host__ __device__ __forceinline__
#else
#define SC_HD inline
#endif
// the O(d) loops of the tail are latency chains (smem load -> fp64 -> store); unrolling
// overlaps them (tail 16.5k -> ~8.5k cycles at d = 100, profiles/r01_overhead.md)
#if defined(__CUDA_ARCH__) && !defined(SCMWU_TAIL_NO_UNROLL)
#define SC_UNROLL4 _Pragma("unroll 4")
#else
#define SC_UNROLL4
#endif

namespace scmwu {

// control constants, verbatim (R/meta.py:238-241, :449-454, R/mwu.py:23)
constexpr int kLadderBase = 64;
constexpr int kLadderFactor = 8;
constexpr int kCheckEvery = 16;
constexpr int kProgressStride = 4;
constexpr double kValueTrendDrop = 0.05;
constexpr double kLossSlack = 1e-9;
constexpr double kSqrt2 = 1.4142135623730951;

// ---- branch-free exp ---------------------------------------------------------
// The streaming passes evaluate one (SVM) or two (SES) exponentials per row with
// arguments down to ~-10^3 (the lagged shift keeps them <= ~0).  The CUDA libm exp takes
// a divergent slow path near underflow, so CTAs whose rows sit in that range fell behind
// the others (SVM C3: per-CTA pass time 190k..246k cycles, profiles/r01_overhead.md).
// sc_exp: Cody-Waite reduction by ln 2, degree-13 Taylor polynomial of e^r on
// |r| <= ln2/2 in Estrin form (4 dependent FMA levels instead of 13), 2^k applied as two
// normal powers of two so gradual underflow needs no branch.  Within 2 ulp of exp()
// (tests/test_math.py); results below 2^-1075 flush to 0.
SC_HD double pow2i(int e) {   // 2^e for e in [-1022, 1023]
#if defined(__CUDA_ARCH__)
    return __hiloint2double((e + 1023) << 20, 0);
#else
    const uint64_t b = (uint64_t)(e + 1023) << 52;
    double r;
    __builtin_memcpy(&r, &b, 8);
    return r;
#endif
}

SC_HD double sc_exp(double x) {
    x = fmin(fmax(x, -745.5), 709.75);
    const double kd = rint(x * 1.4426950408889634);
    double r = fma(-kd, 6.93147180369123816490e-01, x);   // ln2 hi (32 trailing zero bits)
    r = fma(-kd, 1.90821492927058770002e-10, r);         // ln2 lo
    const double r2 = r * r, r4 = r2 * r2, r8 = r4 * r4;
    const double q0 = fma(r, 1.0, 1.0);
    const double q1 = fma(r, 1.0 / 6.0, 0.5);
    const double q2 = fma(r, 1.0 / 120.0, 1.0 / 24.0);
    const double q3 = fma(r, 1.0 / 5040.0, 1.0 / 720.0);
    const double q4 = fma(r, 1.0 / 362880.0, 1.0 / 40320.0);
    const double q5 = fma(r, 1.0 / 39916800.0, 1.0 / 3628800.0);
    const double q6 = fma(r, 1.0 / 6227020800.0, 1.0 / 479001600.0);
    const double w0 = fma(q1, r2, q0), w1 = fma(q3, r2, q2), w2 = fma(q5, r2, q4);
    const double z0 = fma(w1, r4, w0), z1 = fma(q6, r4, w2);
    const double p = fma(z1, r8, z0);
    const int k = (int)kd;
    const int k1 = k >> 1;
    return (p * pow2i(k1)) * pow2i(k - k1);
}

// ---- layout of one reduced pass vector ------------------------------------
// SES: T, K (= sum_i c_i |U - t v_i|^2, from which the tail forms the oracle's linear term,
//      DESIGN.md §3), Rad, M (max lambda+), F (max progress of U/t), Wd (max residual
//      eigen-magnitude of iteration t), Fw (max progress of the window avg),
//      then Sd[d] = sum_i c_i (U - t v_i).
// SVM: TP, TQ, M (max logit), minresP, minresQ, Wd (max |res|), minPW, maxQW,
//      minPy, maxQy, minPz, maxQz, then GP[d], GQ[d].
enum SesRed { kS_T = 0, kS_Lin, kS_Rad, kS_M, kS_F, kS_Wd, kS_Fw, kS_Vec };
enum SvmRed { kV_TP = 0, kV_TQ, kV_M, kV_minresP, kV_minresQ, kV_Wd, kV_minPW, kV_maxQW,
              kV_minPy, kV_maxQy, kV_minPz, kV_maxQz, kV_Vec };

SC_HD int red_width(int kind, int d) { return kind == SC_SES ? kS_Vec + d : kV_Vec + 2 * d; }
// per-CTA partial layout: SES identical to the reduced one; SVM carries one side
// (T, M, minres, Wd, extW, extY, extZ, G[d]) — the side is known from the CTA index.
enum SvmPart { kP_T = 0, kP_M, kP_minres, kP_Wd, kP_extW, kP_extY, kP_extZ, kP_Vec };
SC_HD int part_width(int kind, int d) { return kind == SC_SES ? kS_Vec + d : kP_Vec + d; }

// Parameters the next streaming pass reads (written by lane 0 of the control warp).
struct PassParams {
    double t;          // learner step count of the state (iteration k-1)
    double alpha;
    double eta_rho;    // eta / rho
    double shift;      // lagged exponent shift
    double S1, S2;     // SVM: sums of s1, s2
    double s1p, s2p;   // SVM: s1, s2 of iteration k-1
    int check;         // iteration k-1 is a check iteration (window / counter)
    int width;         // SES: the width check of iteration k-1 needs the exact residuals
    int action;        // 0 = pass, 1 = done
};

// Device-memory slots describing an iterate, so p can be rebuilt on demand.
struct IterState {
    double t, eta, shift, T, TP, TQ, S1, S2;
};

enum Action { kPass = 0, kDone = 1 };
enum Flow { kContinue = 0, kBreak = 1, kStop = 2 };

// Shared-memory vector workspace of the control (all of length >= dd).
struct CtlVecs {
    double* ysum;    // y_sum (U or W in its first d entries)
    double* yprev;   // y of iteration k-1 (u or w, then alpha or s1,s2)
    double* wsum;    // window_sum
    double* besty;   // _ProgressState.best_y
    double* claimy;  // best_claim_y (FTP)
    double* ywin;    // window average of the last check iteration
    double* zv;      // SVM: P^T mu^ - Q^T gam^ of the last check iteration
    double* ynew;    // scratch: y of the iterate being processed
    double* pU;      // state vector (y_sum before update) of the latest iterate
    double* v1;      // SES: anchor centre
};

// Global-memory slots (device) written by the CTA whose `writer` flag is set.
struct CtlSlots {
    double* ring;        // window history, ring_cap entries of ring_stride doubles
    int64_t ring_cap;
    int ring_stride;     // >= dd (even on the device: 16-byte entries for cp.async)
    double* pd_pending;  // SVM: iterate state at the last check  [d+2 | IterState]
    double* pd_callmin;  // SVM: state at the call's smallest counter distance
    double* pd_sep;      // SVM: state of the separating iterate
    double* last;        // state of the latest iterate (for sc_iterate)
    double* pd_best;     // SVM: the committed best_pd state (sc_pd_pair reads it)
};

template <class L>
struct Control {
    // ---------------- problem (constant)
    int kind, d, dd;
    bool is_max;
    double rho, inv_rho, R, ln_r, D, g1;
    // ---------------- call arguments
    sc_ftp_args a;
    // ---------------- learner / rung state
    int64_t t, T;            // step count, horizon of the rung / run
    int64_t budget, spent, rung_T, remaining;
    int rung_index;
    double eta;
    int64_t win_head, win_count, win_len;  // ring indices (monotone) and live length
    int64_t pos_head, pos_count;           // the same indices wrapped to the ring capacity
                                           // (a 64-bit modulo per access cost ~100 cycles)
    // FTP early-stop state
    bool has_f_prev; double f_prev; int streak; bool early;
    bool has_f_start; double f_start;
    double f_last;           // progress of the last finished iteration (FTP)
    // REFINE state
    int64_t stall_floor, last_gain;
    bool has_anchor; double anchor;
    bool has_val_anchor; double val_anchor;
    double lo, hi;
    // best / claims
    bool has_best_f; double best_f;
    bool has_best_counter; double best_counter;
    double claim_eps; bool has_claim;
    // deferred data of iteration t (the latest accepted iterate)
    double value_prev;       // oracle value of iteration t
    double dist_prev;        // SVM counter distance of iteration t (if check)
    bool check_prev;
    bool width_prev;         // SES: iteration t's width check needs the exact residuals
    double inv_t_last;       // 1.0 / t, computed once per iteration
    // SVM pd bookkeeping
    bool has_counter_min; double counter_min;
    // latest iterate state (for p)
    IterState cur;           // state of the iterate being processed
    double shift_pass;       // shift used by the pass that produced `red`
    // results
    sc_ftp_result* res;      // written by all lanes identically; copied out by the writer
    int status;
    bool writer;

    CtlVecs v;
    CtlSlots s;
    // the window entry the next iteration will evict, prefetched into shared memory
    // while the pass streams (device); nullptr = read it from the ring directly
    double* evict_buf = nullptr;
    int64_t evict_idx = -1;
    // shared-memory copy of the pending pd_counter state (device); nullptr = global
    double* pend_buf = nullptr;
    // diagnostics (timing builds): cycle sums of the tail's sections, lane 0 of CTA 0
    long long* tt = nullptr;
    long long tt_prev = 0;
    SC_HD void tmark(int i) {
#if defined(__CUDA_ARCH__) && defined(SCMWU_PHASE_TIMING)
        if (tt != nullptr && L::lane() == 0) {
            const long long now = clock64();
            if (i > 0 && tt_prev != 0) tt[i] += now - tt_prev;
            tt_prev = now;
        }
#else
        (void)i;
#endif
    }

    // ------------------------------------------------------------ helpers
    SC_HD bool is_check(int64_t tt) const {
        return tt % kCheckEvery == 0 || tt == T || tt == 1;
    }
    SC_HD bool is_prog(int64_t tt) const {
        return tt % kProgressStride == 0 || tt == 1 || tt == T;
    }
    SC_HD bool better(double f) const {
        return !has_best_f || (is_max ? f < best_f : f > best_f);
    }
    // offer(f, y_sum / t)
    SC_HD void offer_bar(double f) {
        if (!better(f)) return;
        has_best_f = true; best_f = f;
        const double inv_t = inv_t_last;   // == 1.0 / t (set by process_iterate)
SC_UNROLL4
        for (int j = L::lane(); j < dd; j += L::nl()) v.besty[j] = v.ysum[j] * inv_t;
    }
    SC_HD void offer_vec(double f, const double* y) {
        if (!better(f)) return;
        has_best_f = true; best_f = f;
        for (int j = L::lane(); j < dd; j += L::nl()) v.besty[j] = y[j];
    }
    // offer(progress(z), (z; 0; 0))  — SVM counter candidate (R/svm.py:181, R/meta.py:348-349)
    SC_HD void offer_z(double f) {
        if (!better(f)) return;
        has_best_f = true; best_f = f;
        for (int j = L::lane(); j < dd; j += L::nl()) v.besty[j] = j < d ? v.zv[j] : 0.0;
    }
    SC_HD void offer_counter(double cv) {
        if (!has_best_counter || (is_max ? cv > best_counter : cv < best_counter)) {
            has_best_counter = true; best_counter = cv;
        }
    }
    SC_HD bool beats(double alpha) const {
        return has_best_f && (is_max ? best_f < alpha : best_f > alpha);
    }
    SC_HD double claim_value(double e) const {
        return is_max ? (1.0 + e) * a.alpha : (1.0 - e) * a.alpha;
    }
    // SVM certified margin of direction w with extremes (minP, maxQ) and norm nrm
    // (R/svm.py:87-94)
    static SC_HD double svm_margin(double minP, double maxQ, double nrm) {
        if (nrm == 0.0) return 0.0;
        double sep = (minP - maxQ) / nrm;
        return sep > 0.0 ? sep : 0.0;
    }
    SC_HD double norm_d(const double* x) const {
        double acc = 0.0;
        for (int j = L::lane(); j < d; j += L::nl()) acc += x[j] * x[j];
        return sqrt(L::sum(acc));
    }
    SC_HD void save_state(double* slot, const double* vec, const IterState& st) {
        if (!writer) return;
        for (int j = L::lane(); j < dd; j += L::nl()) slot[j] = vec[j];
        if (L::lane() == 0) *reinterpret_cast<IterState*>(slot + dd + (dd & 1)) = st;
    }
    SC_HD void copy_slot(double* dst, const double* src) {
        if (!writer) return;
        const int w = dd + (dd & 1) + (int)(sizeof(IterState) / sizeof(double));
        for (int j = L::lane(); j < w; j += L::nl()) dst[j] = L::ldcg(src + j);
    }
    // shared-memory copy of a state (every CTA keeps it, so commits need no global read)
    SC_HD void keep_state(double* buf, const double* vec, const IterState& st) {
        for (int j = L::lane(); j < dd; j += L::nl()) buf[j] = vec[j];
        if (L::lane() == 0) *reinterpret_cast<IterState*>(buf + dd + (dd & 1)) = st;
    }
    SC_HD void store_state(double* slot, const double* buf) {
        if (!writer) return;
        const int w = dd + (dd & 1) + (int)(sizeof(IterState) / sizeof(double));
        L::sync();
        for (int j = L::lane(); j < w; j += L::nl()) slot[j] = buf[j];
    }

    // ------------------------------------------------------------ results
    SC_HD int finish_primal(double value, int64_t iters) {
        res->kind = SC_PRIMAL; res->reason = SC_REASON_SEPARATED;
        res->iterations = iters; res->oracle_value = value;
        return finish_common();
    }
    // _dual_feasible (R/meta.py:436-446); y_bar from `src` (already divided) or
    // y_sum / t when src == nullptr and use_sum.
    SC_HD int finish_dual(int reason, int64_t iters, double eps_eff, double value,
                          const double* src, bool have_y, bool from_sum, double* y_tilde) {
        res->kind = SC_DUAL; res->reason = reason; res->iterations = iters;
        double e = eps_eff;
        if (!have_y) e = INFINITY;
        res->eps_eff = e; res->value = value; res->has_claim_y = have_y ? 1 : 0;
        const double sh = (e < 1.0 ? e : 1.0) * a.alpha / R;
        for (int j = L::lane(); j < dd; j += L::nl()) {
            double y = !have_y ? 0.0 : from_sum ? v.ysum[j] / (double)t : src[j];
            if (j == dd - 1) y += is_max ? sh : -sh;
            y_tilde[j] = y;
        }
        return finish_common();
    }
    SC_HD int finish_common() {
        res->has_best_f = has_best_f; res->best_f = has_best_f ? best_f : 0.0;
        res->has_best_counter = has_best_counter;
        res->best_counter = has_best_counter ? best_counter : 0.0;
        res->has_counter_min = has_counter_min;
        res->counter_min = has_counter_min ? counter_min : 0.0;
        status = SC_OK;
        save_state(s.last, v.pU, cur);
        if (evict_idx >= 0) L::prefetch_wait();   // no copy may land after exit
        evict_idx = -1;
        return kDone;
    }

    // ------------------------------------------------------------ call start
    // red0: the reduced vector of iterate 1 (all logits zero), precomputed.
    SC_HD int begin(const sc_ftp_args& args, const double* red0, double* y_tilde,
                    double* best_y_out, PassParams* pp) {
        a = args;
        has_best_f = false; best_f = 0.0; has_best_counter = false; best_counter = 0.0;
        has_counter_min = false; counter_min = 0.0;
        claim_eps = INFINITY; has_claim = false;
        spent = 0; rung_index = 0; status = SC_OK;
        res->sep_dist = 0.0; res->width_iteration = 0; res->width_norm = 0.0;
        if (a.mode == SC_MODE_FTP) {
            budget = a.budget;
            int64_t base = kLadderBase > a.ceil_ln_r ? kLadderBase : a.ceil_ln_r;
            rung_T = budget < base ? budget : base;
            return start_rung(red0, y_tilde, pp);
        }
        // refine_run (R/meta.py:474-497)
        T = a.horizon;
        eta = sqrt(ln_r / (double)T);
        int64_t sf = (int64_t)ceil(16.0 / eta);
        stall_floor = 64 * (int64_t)a.patience > sf ? 64 * (int64_t)a.patience : sf;
        has_anchor = false; has_val_anchor = false; last_gain = 0;
        lo = a.lo; hi = a.hi;
        reset_learner();
        return process_iterate(red0, y_tilde, pp);
    }

    SC_HD void reset_learner() {
        t = 0; win_head = 0; win_count = 0; win_len = 0; pos_head = 0; pos_count = 0;
        if (evict_idx >= 0) L::prefetch_wait();   // drop a pending prefetch of the old run
        evict_idx = -1;
        for (int j = L::lane(); j < dd; j += L::nl()) { v.ysum[j] = 0.0; v.wsum[j] = 0.0; }
        shift_pass = 0.0;
    }

    SC_HD int final_exhausted(double* y_tilde) {
        int64_t it = spent > 1 ? spent : 1;
        return finish_dual(SC_REASON_EXHAUSTED, it, claim_eps, claim_value(claim_eps), v.claimy,
                           has_claim, false, y_tilde);
    }

    // top of `while spent < budget` (R/meta.py:294-311)
    SC_HD int start_rung(const double* red0, double* y_tilde, PassParams* pp) {
        if (!(spent < budget)) return final_exhausted(y_tilde);
        remaining = budget - spent;
        if ((double)remaining < ln_r) return final_exhausted(y_tilde);
        if (remaining < rung_T) rung_T = remaining;
        T = rung_T;
        eta = sqrt(ln_r / (double)rung_T);
        has_f_prev = false; f_prev = 0.0; streak = 0; early = false;
        has_f_start = has_best_f; f_start = best_f;
        reset_learner();
        return process_iterate(red0, y_tilde, pp);
    }

    // ------------------------------------------------------------ iterate k = t+1
    SC_HD int process_iterate(const double* red, double* y_tilde, PassParams* pp) {
        const int64_t k = t + 1;
        const int nl = L::nl(), ln = L::lane();
        double value;
        cur.t = (double)t; cur.eta = eta; cur.shift = shift_pass;
        if (kind == SC_SES) {
            // s = sum_i W_i = -(eta/rho)/T * sum_i c_i (U - t v_i)      (R/ses.py:109-112)
            const double Tt = red[kS_T];
            cur.T = Tt;
            if (a.alpha < g1) {          // R/ses.py:103-105
                return finish_sep(-INFINITY, k, red, y_tilde);
            }
            const double coef = -(eta * inv_rho) / Tt;
            // one reduction for |s|^2, s.v1 and U.Sd: s.u = s.v1 + (alpha - g1) |s|^2 / |s|
            double s2 = 0.0, sv = 0.0, us = 0.0;
SC_UNROLL4
            for (int j = ln; j < d; j += nl) {
                const double sj = coef * red[kS_Vec + j];
                v.ynew[j] = sj;          // temporarily s
                s2 = fma(sj, sj, s2);
                sv = fma(sj, v.v1[j], sv);
                us = fma(v.ysum[j], red[kS_Vec + j], us);
            }
            L::sum3(s2, sv, us);
            const double sn = sqrt(s2);
            const double am = a.alpha - g1;
            const double inv_sn = sn > 0.0 ? 1.0 / sn : 0.0;
SC_UNROLL4
            for (int j = ln; j < d; j += nl) v.ynew[j] = fma(am * inv_sn, v.ynew[j], v.v1[j]);
            const double su = sn > 0.0 ? fma(am * inv_sn, s2, sv) : sv;
            // sum_i c_i v_i.(U - t v_i) = (U . Sd - K) / t (v_i = (U - df_i) / t): the
            // pass then needs no per-element dot product with v_i (0 at t = 0: U = 0)
            const double lin = t > 0 ? coef * ((us - red[kS_Lin]) / (double)t) : 0.0;
            const double rad = red[kS_Rad] / (kSqrt2 * Tt);
            value = su + a.alpha / kSqrt2 - lin - rad;            // R/ses.py:123
            if (value < 0.0) return finish_sep(value, k, red, y_tilde);
            for (int j = ln; j < dd; j += nl)
                if (j == d) v.ynew[j] = a.alpha;                 // y = (u; alpha)
        } else {
            // g = P^T mu - Q^T gam with mu = e/T                  (R/svm.py:104-119)
            const double TP = red[kV_TP], TQ = red[kV_TQ];
            const double Tt = TP + TQ;
            cur.T = Tt; cur.TP = TP; cur.TQ = TQ;
            cur.S1 = v.ysum[d]; cur.S2 = v.ysum[d + 1];
            const double inv_T = 1.0 / Tt;
            double g2 = 0.0;
SC_UNROLL4
            for (int j = ln; j < d; j += nl) {
                const double gj = (red[kV_Vec + j] - red[kV_Vec + d + j]) * inv_T;
                v.ynew[j] = gj;
                g2 = fma(gj, gj, g2);
            }
            g2 = L::sum(g2);
            const double gn = sqrt(g2);
            const double inv_gn = gn > 0.0 ? 1.0 / gn : 0.0;
SC_UNROLL4
            for (int j = ln; j < d; j += nl)
                v.ynew[j] = gn > 0.0 ? v.ynew[j] * inv_gn : (j == 0 ? 1.0 : 0.0);
            const double gw = gn > 0.0 ? g2 * inv_gn : 0.0;       // g . w
            const double tm = TP / Tt, tg = TQ / Tt;
            const double s1 = tm <= tg ? D : a.alpha - D;
            const double s2v = a.alpha - s1;
            value = gw - tm * s1 - tg * s2v;                      // R/svm.py:118
            if (value < 0.0) return finish_sep(value, k, red, y_tilde);
            for (int j = ln; j < dd; j += nl) {                  // y = (w; s1; s2)
                if (j == d) v.ynew[j] = s1;
                if (j == d + 1) v.ynew[j] = s2v;
            }
        }
        tmark(2);
        // ---- accepted witness: y_sum += y, window push; the width check of this
        // iteration is deferred to the next pass
        const bool chk = is_check(k);
        if (kind == SC_SVM && chk) {
            // pd_counter at this iterate (R/svm.py:173-181): z = GP/TP - GQ/TQ
            const double iP = 1.0 / red[kV_TP], iQ = 1.0 / red[kV_TQ];
            double z2 = 0.0;
SC_UNROLL4
            for (int j = ln; j < d; j += nl) {
                const double z = red[kV_Vec + j] * iP - red[kV_Vec + d + j] * iQ;
                v.zv[j] = z;
                z2 = fma(z, z, z2);
            }
            dist_prev = sqrt(L::sum(z2));
            // the state of this iterate (y_sum before the update) for a later commit
            save_state(s.pd_pending, v.ysum, cur);
            if (pend_buf != nullptr) keep_state(pend_buf, v.ysum, cur);
        }
        if (win_len + 2 > s.ring_cap) {   // the window would overwrite live ring entries
            finish_common();
            status = SC_EOOM;
            return kDone;
        }
        double* slot = s.ring + pos_count * s.ring_stride;
        // SES width bound: with u_k = U_k / k the running average,
        //   |alpha - g_i| + |y_k - v_i| <= |alpha| + F(u_k) + |y_k - u_k|,
        //   F(u_k) <= F(u_{k-1}) + |u_k - u_{k-1}|,
        // and F(u_{k-1}) = max_i |u_{k-1} - v_i| + g_i is red[kS_F] of the pass that
        // produced this iterate.  When the bound is below the width rho the exact
        // residuals of y_k are not needed: the check cannot fail.
        const bool bound_ses = kind == SC_SES && k >= 2;
        const double inv_k = 1.0 / (double)k, inv_km1 = bound_ses ? inv_t_last : 0.0;
        inv_t_last = inv_k;
        double du2 = 0.0, dy2 = 0.0;
SC_UNROLL4
        for (int j = ln; j < dd; j += nl) {
            const double y = v.ynew[j];
            const double u0 = v.ysum[j];
            v.pU[j] = u0;
            const double u1 = u0 + y;
            v.ysum[j] = u1;
            v.yprev[j] = y;
            if (writer) slot[j] = y;
            v.wsum[j] += y;
            if (bound_ses && j < d) {
                const double ub = u1 * inv_k;
                const double du = ub - u0 * inv_km1, dy = y - ub;
                du2 = fma(du, du, du2);
                dy2 = fma(dy, dy, dy2);
            }
        }
        width_prev = true;
        if (bound_ses) {
            L::sum2(du2, dy2);
            const double wb = (fabs(a.alpha) + red[kS_F] + sqrt(du2) + sqrt(dy2)) / kSqrt2;
            width_prev = !(wb * inv_rho <= (1.0 + kLossSlack) * (1.0 - 1e-9));
        }
        t = k;
        value_prev = value;
        check_prev = chk;
        tmark(3);
        push_window(k);
        tmark(4);
        if (chk) {
            const double inv_len = 1.0 / (double)win_len;
SC_UNROLL4
            for (int j = ln; j < dd; j += nl) v.ywin[j] = v.wsum[j] * inv_len;
        }
        // lagged shift for the next pass: the max eigenvalue / logit of this iterate
        const double m = kind == SC_SES ? red[kS_M] : red[kV_M];
        shift_pass = m;
        L::sync();
        tmark(5);
        write_pass(pp);
        tmark(6);
        return kPass;
    }

    SC_HD int finish_sep(double value, int64_t k, const double* red, double* y_tilde) {
        for (int j = L::lane(); j < dd; j += L::nl()) v.pU[j] = v.ysum[j];
        if (kind == SC_SVM) {
            const double iP = 1.0 / red[kV_TP], iQ = 1.0 / red[kV_TQ];
            double z2 = 0.0;
            for (int j = L::lane(); j < d; j += L::nl()) {
                const double z = red[kV_Vec + j] * iP - red[kV_Vec + d + j] * iQ;
                z2 = fma(z, z, z2);
            }
            res->sep_dist = sqrt(L::sum(z2));
            save_state(s.pd_sep, v.ysum, cur);
        }
        const int64_t iters = a.mode == SC_MODE_FTP ? spent + k : k;
        return finish_primal(value, iters);
    }

    // suffix window (R/meta.py:330-335 / :514-519): the new y was added to the
    // ring and the sum by process_iterate; evict down to max(64, t/2) entries
    SC_HD void push_window(int64_t tt) {
        const int nl = L::nl(), ln = L::lane();
        ++win_count; ++win_len;
        if (++pos_count == s.ring_cap) pos_count = 0;
        const int64_t lim = kLadderBase > tt / 2 ? kLadderBase : tt / 2;
        while (win_len > lim) {
            if (evict_buf != nullptr && win_head == evict_idx) {
                L::prefetch_wait();
                for (int j = ln; j < dd; j += nl) v.wsum[j] -= evict_buf[j];
                evict_idx = -1;
            } else {
                const double* old = s.ring + pos_head * s.ring_stride;
                for (int j = ln; j < dd; j += nl) v.wsum[j] -= L::ldcg(old + j);
            }
            ++win_head; --win_len;
            if (++pos_head == s.ring_cap) pos_head = 0;
        }
    }

    // start fetching the entry the next push may evict (it was written >= 64
    // iterations ago, so it is visible to every CTA)
    SC_HD void prefetch_eviction() {
        if (evict_buf == nullptr || win_len < kLadderBase) return;
        evict_idx = win_head;
        L::prefetch(evict_buf, s.ring + pos_head * s.ring_stride, s.ring_stride);
    }

    SC_HD void write_pass(PassParams* pp) {
        prefetch_eviction();
        if (L::lane() != 0) return;
        pp->t = (double)t;
        pp->alpha = a.alpha;
        pp->eta_rho = eta * inv_rho;
        pp->shift = shift_pass;
        pp->check = check_prev ? 1 : 0;
        pp->width = width_prev ? 1 : 0;
        if (kind == SC_SVM) {
            pp->S1 = v.ysum[d]; pp->S2 = v.ysum[d + 1];
            pp->s1p = v.yprev[d]; pp->s2p = v.yprev[d + 1];
        }
        pp->action = kPass;
    }

    // ------------------------------------------------------------ after a pass
    // `red` reduces iterate t+1 (speculative) and the checks of iteration t.
    SC_HD int after_pass(const double* red, const double* red0, double* y_tilde,
                         PassParams* pp) {
        tmark(0);
        int flow = finish_iteration(red, y_tilde);
        tmark(1);
        if (flow == kStop) return kDone;
        if (flow == kContinue && t < T) return process_iterate(red, y_tilde, pp);
        // end of the rung (FTP) or of the run (REFINE)
        if (a.mode == SC_MODE_REFINE) {
            const double tt = (double)t;
            const double e = R * rho * (eta + ln_r / (eta * tt)) / a.alpha;  // R/meta.py:570
            return finish_dual(SC_REASON_REFINED, t, e, claim_value(e), nullptr, true, true,
                               y_tilde);
        }
        return end_rung(red0, y_tilde, pp);
    }

    // R/meta.py:366-389
    SC_HD int end_rung(const double* red0, double* y_tilde, PassParams* pp) {
        spent += t;
        const double tt = (double)t;
        const double e_here = R * rho * (eta + ln_r / (eta * tt)) / a.alpha;
        if (e_here < claim_eps) {
            claim_eps = e_here; has_claim = true;
            for (int j = L::lane(); j < dd; j += L::nl()) v.claimy[j] = v.ysum[j] / tt;
        }
        if (claim_eps <= a.eps)
            return finish_dual(SC_REASON_EXHAUSTED, spent, claim_eps, claim_value(claim_eps),
                               v.claimy, has_claim, false, y_tilde);
        if (early && rung_index >= 1 && a.has_progress) {
            bool stalled = has_f_start && has_best_f &&
                           fabs(f_start - best_f) <= a.delta * fabs(f_start);
            if (stalled)
                return finish_dual(SC_REASON_EARLY_STOP, spent, claim_eps,
                                   claim_value(claim_eps), v.claimy, has_claim, false, y_tilde);
        }
        rung_index += 1;
        int64_t nxt = rung_T * kLadderFactor;
        rung_T = remaining < nxt ? remaining : nxt;
        return start_rung(red0, y_tilde, pp);
    }

    // Finish iteration t (its observe + progress bookkeeping), reference order
    // R/meta.py:323-364 (FTP) / :509-568 (REFINE).
    SC_HD int finish_iteration(const double* red, double* y_tilde) {
        const bool ftp = a.mode == SC_MODE_FTP;
        // Scmwu.observe width check (R/mwu.py:62-64) -> WidthViolationError
        const double wd = kind == SC_SES ? red[kS_Wd] : red[kV_Wd];
        const double nrm = wd * inv_rho;
        if (nrm > 1.0 + kLossSlack) {
            res->width_iteration = ftp ? spent + t : t;
            res->width_norm = nrm * rho;
            finish_common();
            status = SC_EWIDTH;
            return kStop;
        }
        if (ftp && !a.has_progress) return kContinue;
        const double tt = (double)t;
        // per-witness candidate (SVM, R/svm.py:123-127) offered with y
        if (kind == SC_SVM) {
            double mw = (red[kV_minresP] + red[kV_minresQ]) + a.alpha;
            offer_vec(mw > 0.0 ? mw : 0.0, v.yprev);
        }
        // progress of the running average
        double f;
        if (kind == SC_SES) {
            f = red[kS_F];
        } else {
            f = svm_margin(red[kV_minPW], red[kV_maxQW], norm_d(v.ysum));
        }
        if (ftp || is_prog(t)) offer_bar(f);
        if (check_prev) {
            double fw = kind == SC_SES ? red[kS_Fw]
                                        : svm_margin(red[kV_minPy], red[kV_maxQy], norm_d(v.ywin));
            offer_vec(fw, v.ywin);
            if (kind == SC_SVM) {
                const double cv = dist_prev;
                if (!has_counter_min || cv < counter_min) {
                    has_counter_min = true; counter_min = cv;
                    if (pend_buf != nullptr) store_state(s.pd_callmin, pend_buf);
                    else copy_slot(s.pd_callmin, s.pd_pending);
                }
                offer_counter(cv);
                offer_z(svm_margin(red[kV_minPz], red[kV_maxQz], cv));
            }
        }
        L::sync();
        if (ftp) {
            if (beats(a.alpha)) {
                finish_dual(SC_REASON_AFFIRMATIVE, spent + t, 0.0, best_f, v.besty, true, false,
                            y_tilde);
                return kStop;
            }
            if (a.enabled) {
                if (has_f_prev && f_prev != 0.0) {
                    if (fabs(f - f_prev) / fabs(f_prev) < a.delta) {
                        streak += 1;
                        if (streak >= a.patience) { early = true; return kBreak; }
                    } else {
                        streak = 0;
                    }
                }
                has_f_prev = true; f_prev = f;
            }
            return kContinue;
        }
        // refine stall rule (R/meta.py:537-555)
        bool gained = false;
        if (!has_anchor || (has_best_f && fabs(best_f - anchor) > a.gain_rel * fabs(anchor))) {
            // anchor = state.best_f (may be None)
            has_anchor = has_best_f; anchor = best_f;   // anchor = state.best_f (None stays None)
            gained = true;
        }
        {
            const double vv = value_prev;
            if (!has_val_anchor) {
                has_val_anchor = true; val_anchor = vv;
            } else if (vv < val_anchor - kValueTrendDrop * fabs(val_anchor)) {
                val_anchor = vv; gained = true;
            }
        }
        if (gained) {
            last_gain = t;
        } else if (a.enabled) {
            int64_t lim = stall_floor > t / 3 ? stall_floor : t / 3;
            if (t - last_gain > lim) return kBreak;
        }
        if (!isnan(a.target) && t % kProgressStride == 0) {
            if (has_best_f) {
                if (is_max) hi = hi < best_f ? hi : best_f;
                else lo = lo > best_f ? lo : best_f;
            }
            if (has_best_counter) {
                if (is_max) lo = lo > best_counter ? lo : best_counter;
                else hi = hi < best_counter ? hi : best_counter;
            }
            const double lp = lo > 0.0 ? lo : 0.0;
            if (hi - lo <= a.target * lp) return kBreak;
        }
        (void)tt;
        return kContinue;
    }
};


// ======================================================================================
// Whole-solve residency (sc_solve): meta.adaptive_search (R/meta.py:656-781) with _Bracket
// (R/meta.py:576-653), as solve_ses / solve_svm drive it (R/ses.py:171-187,
// R/svm.py:189-214), run between the streaming passes of ONE persistent launch.  Every
// feasibility test is the Control above; the search decides the next test's level and
// arguments from the previous result exactly as the reference does (same constants, same
// operation order), so all CTAs (and all ranks) take identical decisions.
//
// Two extra "progress passes" stream X for ses_progress / svm_progress at a given point
// (the seed certificate and, SES, the final enclosure check): a check pass of the kernel
// with the point in the window-average slot, every learner weight 1 (eta = 0).
constexpr int kMaxSearchSteps = 400;     // R/meta.py:449
constexpr int64_t kBracketTestCap = 2048; // R/meta.py:450
constexpr int64_t kRefineStart = 2048;    // R/meta.py:451
constexpr int kMaxRefineRounds = 12;      // R/meta.py:453
constexpr int64_t kBudgetClamp = (int64_t)1 << 62;

enum SearchPhase { kSeedPass = 0, kBracket = 1, kRefine = 2, kSlackPass = 3, kFinished = 4 };

template <class L>
struct Search {
    sc_solve_args sa;
    double R, rho, ln_r;
    bool is_max;
    int kind, d, dd;
    // _Bracket
    double Lb, Ub, gain_floor;
    bool has_best; double best_f;          // best_y lives in `sbest` (shared memory)
    // adaptive_search state
    int phase, nsteps, rounds;
    int64_t total, test_cap, h;
    bool capped, floored;
    double alpha, eps_i;
    int64_t Ti, full, horizon;
    // svm.py best_pd (R/svm.py:171-181): committed on the device
    bool has_pd; double pd_best;
    double seed_f, final_f;
    int status;
    double w_alpha; int64_t w_iter; double w_norm;
    double* sbest;                         // smem vector (dd): the bracket's best_y
    double* yprog;                         // smem vector: the progress pass's point
    sc_search_step* log;                   // device log (written by the writer)
    bool writer;

    SC_HD static int64_t bound(double R_, double rho_, double lnr, double e, double a) {
        // iteration_bound (R/meta.py:208-213): ceil(4 R^2 rho^2 ln r / (eps^2 alpha^2)), the
        // same left-to-right operation order (x**2 == x*x exactly), clamped like the callers
        const double v = ceil(4.0 * (R_ * R_) * (rho_ * rho_) * lnr / ((e * e) * (a * a)));
        return v >= (double)kBudgetClamp ? kBudgetClamp : (int64_t)v;
    }
    SC_HD void tighten_dual(double f) {
        if (is_max) Ub = Ub < f ? Ub : f; else Lb = Lb > f ? Lb : f;
    }
    SC_HD void tighten_primal(double f) {
        if (is_max) Lb = Lb > f ? Lb : f; else Ub = Ub < f ? Ub : f;
    }
    SC_HD bool converged(double e) const {
        const double span = Ub - Lb;
        const double ref = Lb > 0.0 ? Lb : (is_max ? span / 3.0 : 2.0 * span / 3.0);
        return span < e * ref;
    }

    // ---- progress pass at y (first d coordinates of `src`)
    template <class C>
    SC_HD int progress_pass(C& ctl, const double* src, PassParams* pp) {
        for (int j = L::lane(); j < dd; j += L::nl()) yprog[j] = j < d ? src[j] : 0.0;
        L::sync();
        (void)ctl;
        if (L::lane() == 0) {
            pp->t = 1.0; pp->alpha = 0.0; pp->eta_rho = 0.0; pp->shift = 0.0;
            pp->S1 = pp->S2 = pp->s1p = pp->s2p = 0.0;
            pp->check = 1; pp->width = 0; pp->action = kPass;
        }
        return kPass;
    }
    // the progress value the pass produced (ses_progress / svm_progress)
    template <class C>
    SC_HD double progress_value(C& ctl, const double* red) {
        if (kind == SC_SES) return red[kS_Fw];
        double acc = 0.0;
        for (int j = L::lane(); j < d; j += L::nl()) acc += yprog[j] * yprog[j];
        (void)ctl;
        return C::svm_margin(red[kV_minPy], red[kV_maxQy], sqrt(L::sum(acc)));
    }

    // ---- start: bracket seeded by the progress of the seed point (R/ses.py:174-176,
    // R/svm.py:194-199, R/meta.py:700-701)
    template <class C>
    SC_HD int begin(C& ctl, const sc_solve_args& args, const double* seed, PassParams* pp) {
        sa = args;
        is_max = kind == SC_SES;
        Lb = sa.L0; Ub = sa.U0;
        gain_floor = sa.delta > sa.eps / 10.0 ? sa.delta : sa.eps / 10.0;
        has_best = false; best_f = 0.0;
        nsteps = 0; rounds = 0; total = 0; capped = false; floored = false;
        test_cap = sa.cap >= 0 && sa.cap < kBracketTestCap ? sa.cap : kBracketTestCap;
        h = kRefineStart;
        has_pd = false; pd_best = 0.0;
        seed_f = 0.0; final_f = 0.0; status = SC_OK;
        w_alpha = 0.0; w_iter = 0; w_norm = 0.0;
        phase = kSeedPass;
        return progress_pass(ctl, seed, pp);
    }

    // ---- after every streaming pass
    template <class C>
    SC_HD int after_pass(C& ctl, const double* red, const double* red0, double* y_tilde,
                         PassParams* pp) {
        if (phase == kSeedPass) {
            const double f = progress_value(ctl, red);
            seed_f = f;
            has_best = true; best_f = f;                       // _Bracket.seed
            for (int j = L::lane(); j < dd; j += L::nl())
                sbest[j] = j < d ? yprog[j] : (kind == SC_SES ? f : 0.0);
            tighten_dual(f);
            phase = kBracket;
            return next_test(ctl, red0, y_tilde, pp);
        }
        if (phase == kSlackPass) {
            final_f = progress_value(ctl, red);
            phase = kFinished;
            return kDone;
        }
        int act = ctl.after_pass(red, red0, y_tilde, pp);
        if (act == kPass) return kPass;
        return test_done(ctl, red0, y_tilde, pp);
    }

    // a feasibility test ended (ctl.res holds its outcome): absorb it.  Returns kCont to
    // choose the next test, kFin to end the search, kErr after a failed test.
    enum { kCont = 0, kFin = 1, kErr = 2 };
    template <class C>
    SC_HD int absorb(C& ctl) {
        const sc_ftp_result& r = *ctl.res;
        if (ctl.status != SC_OK) {            // WidthViolationError / ring overflow: stop
            status = ctl.status;
            w_alpha = alpha; w_iter = r.width_iteration; w_norm = r.width_norm;
            phase = kFinished;
            return kErr;
        }
        // DeviceProblem.run: the call's smallest pd_counter distance becomes best_pd
        if (kind == SC_SVM && r.has_counter_min && (!has_pd || r.counter_min < pd_best)) {
            ctl.copy_slot(ctl.s.pd_best, ctl.s.pd_callmin);
            has_pd = true; pd_best = r.counter_min;
        }
        total += r.iterations;
        const bool primal = r.kind == SC_PRIMAL;
        if (phase == kBracket && sa.cap >= 0 && sa.cap < Ti && !primal &&
            r.reason == SC_REASON_EXHAUSTED && r.iterations >= sa.cap)
            capped = true;
        // _Bracket.absorb (R/meta.py:603-644)
        const double span_before = Ub - Lb;
        bool improved = false;
        if (primal) {
            tighten_primal(alpha);                     // separation is exact
            if (sa.on_primal) {                        // pd_counter(cert.p) (R/svm.py:201-204)
                const double c = r.sep_dist;
                if (!has_pd || c < pd_best) {
                    ctl.copy_slot(ctl.s.pd_best, ctl.s.pd_sep);
                    has_pd = true; pd_best = c;
                }
                tighten_primal(c);
            }
        } else {
            tighten_dual(r.value);                     // regret-certified claim
        }
        if (r.has_best_f) {
            const double f = r.best_f;
            const bool better = !has_best || (is_max ? f < best_f : f > best_f);
            if (better) {
                if (has_best && fabs(best_f - f) > gain_floor * fabs(best_f)) improved = true;
                has_best = true; best_f = f;
                for (int j = L::lane(); j < dd; j += L::nl()) sbest[j] = ctl.v.besty[j];
            }
            tighten_dual(best_f);
        }
        if (r.has_best_counter) tighten_primal(r.best_counter);
        const bool productive = improved || (Ub - Lb) < span_before * (1.0 - 2e-2);
        if (writer && L::lane() == 0 && nsteps < sa.max_steps) {   // SearchStep
            sc_search_step& st = log[nsteps];
            st.alpha = alpha; st.eps = phase == kBracket ? eps_i : sa.eps;
            st.iteration_bound = Ti; st.iterations = r.iterations;
            st.separated = primal ? 1 : 0; st.reason = primal ? SC_REASON_SEPARATED : r.reason;
        }
        ++nsteps;
        L::sync();
        if (phase == kBracket) {
            if (!productive) phase = kRefine;          // the bracketing loop breaks
            return kCont;
        }
        ++rounds;
        if (!productive && horizon >= full) return kFin;
        h = h * 4 < sa.refine_horizon ? h * 4 : sa.refine_horizon;
        return kCont;
    }

    template <class C>
    SC_HD int test_done(C& ctl, const double* red0, double* y_tilde, PassParams* pp) {
        const int r = absorb(ctl);
        if (r == kErr) return kDone;
        if (r == kFin) return finish(ctl, pp);
        return next_test(ctl, red0, y_tilde, pp);
    }

    // choose and start the next test; a test can end before its first pass (iterate 1 is
    // precomputed), so loop until one needs a pass or the search ends
    template <class C>
    SC_HD int next_test(C& ctl, const double* red0, double* y_tilde, PassParams* pp) {
        for (;;) {
            sc_ftp_args a;
            a.has_progress = 1; a.delta = sa.delta; a.patience = sa.patience;
            a.enabled = sa.enabled; a.ceil_ln_r = sa.ceil_ln_r;
            if (phase == kBracket) {                     // R/meta.py:705-730
                bool stop = nsteps >= kMaxSearchSteps || converged(sa.eps);
                const double span = Ub - Lb;
                if (!stop && !isnan(sa.zero_lower_floor) && Lb == 0.0 &&
                    span < sa.zero_lower_floor) {
                    floored = true;
                    stop = true;
                }
                if (stop) { phase = kRefine; continue; }
                alpha = is_max ? Lb + span / 3.0 : Lb + 2.0 * span / 3.0;
                eps_i = span / (3.0 * alpha);
                Ti = bound(R, rho, ln_r, eps_i, alpha);
                a.mode = SC_MODE_FTP; a.alpha = alpha; a.eps = eps_i;
                a.budget = Ti < test_cap ? Ti : test_cap;
                a.horizon = 0; a.gain_rel = NAN; a.lo = -INFINITY; a.hi = INFINITY;
                a.target = NAN;
            } else if (phase == kRefine) {               // R/meta.py:732-763
                if (floored || rounds >= kMaxRefineRounds || converged(sa.eps) ||
                    nsteps >= kMaxSearchSteps)
                    return finish(ctl, pp);
                alpha = (Lb + Ub) / 2.0;
                if (alpha <= 0.0) return finish(ctl, pp);
                Ti = bound(R, rho, ln_r, sa.eps, alpha);
                full = Ti < sa.refine_horizon ? Ti : sa.refine_horizon;
                if (sa.cap >= 0 && sa.cap < full) full = sa.cap;
                horizon = h < full ? h : full;
                a.mode = SC_MODE_REFINE; a.alpha = alpha; a.eps = NAN; a.budget = 0;
                a.horizon = horizon > sa.ceil_ln_r ? horizon : sa.ceil_ln_r;   // R/meta.py:479
                a.gain_rel = sa.delta > sa.eps / 20.0 ? sa.delta : sa.eps / 20.0;
                a.lo = Lb; a.hi = Ub; a.target = sa.eps;
            } else {
                return kDone;
            }
            if (ctl.begin(a, red0, y_tilde, nullptr, pp) == kPass) return kPass;
            const int r = absorb(ctl);
            if (r == kErr) return kDone;
            if (r == kFin) return finish(ctl, pp);
        }
    }

    template <class C>
    SC_HD int finish(C& ctl, PassParams* pp) {
        if (kind == SC_SES && has_best) {                // final enclosure check (R/ses.py:187)
            phase = kSlackPass;
            return progress_pass(ctl, sbest, pp);
        }
        phase = kFinished;
        return kDone;
    }

    SC_HD int termination() const {
        if (capped) return SC_TERM_ITERATION_CAP;
        if (converged(sa.eps)) return SC_TERM_RANGE_CONVERGED;
        return SC_TERM_EARLY_STOPPED;
    }
};

}  // namespace scmwu
