// scmwu_emu.cpp — TEST INFRASTRUCTURE ONLY.
//
// A single-threaded host emulation of the CUDA engine: the same control
// header (paper_2405_09157_b200/csrc/scmwu_control.h) driven by a plain C++
// loop that computes the streaming pass row by row with the same closed-form
// formulas as the CUDA kernel.  It exports the sc_* C ABI of include/scmwu.h
// so the host layer can be exercised on a machine without a GPU
// (tests/test_emu_*.py, tests/test_multirank_gloo.py).  It is never loaded by
// the product package.
//
// Row sharding: where the CUDA kernel exchanges the per-pass rank vectors over
// NVLink mailboxes, the emulator calls a host callback (emu_set_exchange) that
// the multi-process CPU tests implement with a torch.distributed (gloo)
// all-gather followed by the same rank-ordered fold.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../paper_2405_09157_b200/csrc/np_rownorm.h"
#include "../../paper_2405_09157_b200/csrc/scmwu_control.h"

using namespace scmwu;

namespace {

struct HostLanes {
    static int lane() { return 0; }
    static int nl() { return 1; }
    static double sum(double x) { return x; }
    static void sum2(double&, double&) {}
    static void sum3(double&, double&, double&) {}
    static void sync() {}
    static double ldcg(const double* p) { return *p; }
    static void prefetch(double* dst, const double* src, int n) {
        for (int j = 0; j < n; ++j) dst[j] = src[j];
    }
    static void prefetch_wait() {}
};

constexpr double kInvSqrt2 = 0.7071067811865476;

}  // namespace

typedef void (*emu_exchange_fn)(const double* local, int rw, double* global);

struct sc_handle {
    sc_problem prob;
    int dd;
    std::vector<double> X, radii;       // n_local x d, n_local
    std::vector<double> red0, red0_local;
    std::vector<double> v1;
    double g1 = 0.0;
    double last_alpha = 0.0;
    std::vector<double> ring, pd_pending, pd_callmin, pd_sep, pd_best, last;
    emu_exchange_fn exchange = nullptr;
    std::string err;
};

static int fail(sc_handle* h, int code, const char* msg) {
    if (h) h->err = msg;
    return code;
}

static int slot_len(int dd) { return dd + (dd & 1) + (int)(sizeof(IterState) / sizeof(double)); }

static void pass_ses(const sc_handle* h, const PassParams& pp, const double* U,
                     const double* up, const double* yw, double* red) {
    const int d = h->prob.d;
    const int64_t n = h->prob.n_local;
    double T = 0, K = 0, Rad = 0, M = -INFINITY, F = -INFINITY, Wd = 0, Fw = -INFINITY;
    std::vector<double> Sd(d, 0.0), df(d);
    const double t = pp.t, er = pp.eta_rho, al = pp.alpha;
    for (int64_t i = 0; i < n; ++i) {
        const double* v = &h->X[i * d];
        const double g = h->radii[i];
        double a = 0, w2 = 0, f2 = 0;
        for (int j = 0; j < d; ++j) {
            double x = fma(-t, v[j], U[j]);
            df[j] = x;
            a = fma(x, x, a);
            double w = up[j] - v[j];
            w2 = fma(w, w, w2);
            if (pp.check) { double y = yw[j] - v[j]; f2 = fma(y, y, f2); }
        }
        const double ra = sqrt(a);
        F = fmax(F, ra / t + g);
        if (pp.check) Fw = fmax(Fw, sqrt(f2) + g);
        if (h->prob.row0 + i == 0) continue;   // global row 0 is the anchor
        const double nrm = er * ra;
        const double x0 = -er * (t * (al - g));
        const double lp = (x0 + nrm) * kInvSqrt2, lm = (x0 - nrm) * kInvSqrt2;
        const double A = exp(lp - pp.shift), B = exp(lm - pp.shift);
        const double c = nrm > 0.0 ? (A - B) / (kSqrt2 * nrm) : 0.0;
        T += A + B;
        K = fma(c, a, K);
        Rad = fma(g, A + B, Rad);
        M = fmax(M, lp);
        Wd = fmax(Wd, (fabs(al - g) + sqrt(w2)) * kInvSqrt2);
        for (int j = 0; j < d; ++j) Sd[j] = fma(c, df[j], Sd[j]);
    }
    red[kS_T] = T; red[kS_Lin] = K; red[kS_Rad] = Rad; red[kS_M] = M;
    red[kS_F] = F; red[kS_Wd] = Wd; red[kS_Fw] = Fw;
    for (int j = 0; j < d; ++j) red[kS_Vec + j] = Sd[j];
}

static void pass_svm(const sc_handle* h, const PassParams& pp, const double* W,
                     const double* wp, const double* yw, const double* z, double* red) {
    const int d = h->prob.d;
    const int64_t n = h->prob.n_local, n1 = h->prob.n1_local;
    double TP = 0, TQ = 0, M = -INFINITY, mrP = INFINITY, mrQ = INFINITY, Wd = 0;
    double mPW = INFINITY, xQW = -INFINITY, mPy = INFINITY, xQy = -INFINITY;
    double mPz = INFINITY, xQz = -INFINITY;
    std::vector<double> GP(d, 0.0), GQ(d, 0.0);
    for (int64_t i = 0; i < n; ++i) {
        const double* x = &h->X[i * d];
        const bool P = i < n1;
        double dW = 0, dw = 0, dy = 0, dz = 0;
        for (int j = 0; j < d; ++j) {
            dW = fma(x[j], W[j], dW);
            dw = fma(x[j], wp[j], dw);
            if (pp.check) { dy = fma(x[j], yw[j], dy); dz = fma(x[j], z[j], dz); }
        }
        const double sg = P ? 1.0 : -1.0;
        const double lg = -pp.eta_rho * (sg * dW - (P ? pp.S1 : pp.S2));
        const double e = exp(lg - pp.shift);
        M = fmax(M, lg);
        const double r = sg * dw - (P ? pp.s1p : pp.s2p);
        Wd = fmax(Wd, fabs(r));
        std::vector<double>& G = P ? GP : GQ;
        if (P) {
            TP += e; mrP = fmin(mrP, r); mPW = fmin(mPW, dW);
            if (pp.check) { mPy = fmin(mPy, dy); mPz = fmin(mPz, dz); }
        } else {
            TQ += e; mrQ = fmin(mrQ, r); xQW = fmax(xQW, dW);
            if (pp.check) { xQy = fmax(xQy, dy); xQz = fmax(xQz, dz); }
        }
        for (int j = 0; j < d; ++j) G[j] = fma(e, x[j], G[j]);
    }
    red[kV_TP] = TP; red[kV_TQ] = TQ; red[kV_M] = M; red[kV_minresP] = mrP;
    red[kV_minresQ] = mrQ; red[kV_Wd] = Wd; red[kV_minPW] = mPW; red[kV_maxQW] = xQW;
    red[kV_minPy] = mPy; red[kV_maxQy] = xQy; red[kV_minPz] = mPz; red[kV_maxQz] = xQz;
    for (int j = 0; j < d; ++j) { red[kV_Vec + j] = GP[j]; red[kV_Vec + d + j] = GQ[j]; }
}

extern "C" {

int sc_version(void) { return 1000; }
int sc_pool_trim(int32_t) { return SC_OK; }   // no device pool on the host

void emu_set_exchange(sc_handle* h, emu_exchange_fn fn) {
    if (h) h->exchange = fn;
}

// the device passes' exponential, compiled for the host (tests/test_math.py)
void emu_sc_exp(const double* x, double* out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) out[i] = scmwu::sc_exp(x[i]);
}

int sc_create(const sc_problem* prob, const double* X, const double* X_tail,
              const double* radii, sc_handle** out) {
    if (!prob || !X || !out) return SC_EARG;
    if (prob->d < 1 || prob->n < 2) return SC_EARG;
    if (prob->kind == SC_SES && !radii) return SC_EARG;
    if (prob->kind == SC_SVM && (prob->n1 < 1 || prob->n1 >= prob->n)) return SC_EARG;
    sc_handle* h = new sc_handle();
    h->prob = *prob;
    sc_problem& P = h->prob;
    if (P.world <= 1) {
        P.world = 1; P.shard = 0; P.row0 = 0; P.n_local = P.n;
        P.n1_local = P.kind == SC_SVM ? P.n1 : 0;
    } else {
        if (P.shard < 0 || P.shard >= P.world || P.n_local < 1 || P.row0 < 0 ||
            P.row0 + P.n_local > P.n || X_tail) {
            delete h;
            return SC_EARG;
        }
        P.n1_local = P.kind == SC_SVM
                         ? std::max<int64_t>(0, std::min<int64_t>(P.n_local, P.n1 - P.row0))
                         : 0;
    }
    const int d = prob->d;
    const int64_t n = P.n_local;
    h->dd = prob->kind == SC_SES ? d + 1 : d + 2;
    if (X_tail) {
        h->X.assign(X, X + prob->n1 * d);
        h->X.insert(h->X.end(), X_tail, X_tail + (n - prob->n1) * d);
    } else {
        h->X.assign(X, X + n * d);
    }
    if (prob->kind == SC_SES) h->radii.assign(radii, radii + n);
    h->v1.assign(h->dd, 0.0);
    if (P.row0 == 0 && prob->kind == SC_SES) {
        for (int j = 0; j < d; ++j) h->v1[j] = h->X[j];
        h->g1 = h->radii[0];
    }
    h->red0.assign(red_width(prob->kind, d), 0.0);
    if (prob->kind == SC_SES) {
        const int64_t first = P.row0 == 0 ? 1 : 0;
        double rad = 0;
        for (int64_t i = first; i < n; ++i) rad += 2.0 * h->radii[i];
        h->red0[kS_T] = 2.0 * (double)(n - first);
        h->red0[kS_Rad] = rad;
        h->red0[kS_M] = 0.0;
    } else {
        const int64_t n1 = P.n1_local;
        h->red0[kV_TP] = (double)n1;
        h->red0[kV_TQ] = (double)(n - n1);
        for (int64_t i = 0; i < n; ++i)
            for (int j = 0; j < d; ++j)
                h->red0[kV_Vec + (i < n1 ? 0 : d) + j] += h->X[i * d + j];
    }
    h->red0_local = h->red0;
    const int sl = slot_len(h->dd);
    h->pd_pending.assign(sl, 0.0);
    h->pd_callmin.assign(sl, 0.0);
    h->pd_sep.assign(sl, 0.0);
    h->pd_best.assign(sl, 0.0);   // t = 0 state == uniform weights
    h->last.assign(sl, 0.0);
    *out = h;
    return SC_OK;
}

int sc_ftp(sc_handle* h, const sc_ftp_args* args, sc_ftp_result* res, double* y_tilde,
           double* best_y) {
    if (!h || !args || !res || !y_tilde || !best_y) return SC_EARG;
    memset(res, 0, sizeof(*res));
    const int d = h->prob.d, dd = h->dd;
    const int64_t T = args->mode == SC_MODE_FTP ? args->budget : args->horizon;
    if (T < 0 || (args->mode == SC_MODE_REFINE && T < 1))
        return fail(h, SC_EARG, "budget/horizon out of range");
    if (h->prob.world > 1 && !h->exchange) return fail(h, SC_EARG, "no exchange callback");
    h->last_alpha = args->alpha;
    // the ring holds at most max(64, T_rung/2)+1 live entries; the largest rung is <= T
    int64_t cap = (T / 2 > kLadderBase ? T / 2 : kLadderBase) + 2;
    if (cap > (1 << 21)) cap = (1 << 21);   // longer windows stop with SC_EOOM (control)
    h->ring.assign((size_t)cap * dd, 0.0);

    std::vector<double> ysum(dd), yprev(dd), wsum(dd), besty(dd), claimy(dd), ywin(dd),
        zv(dd), ynew(dd), pU(dd), v1(h->v1);
    Control<HostLanes> c;
    c.kind = h->prob.kind; c.d = d; c.dd = dd;
    c.is_max = h->prob.kind == SC_SES;
    c.rho = h->prob.rho; c.inv_rho = 1.0 / h->prob.rho; c.R = h->prob.R;
    c.ln_r = h->prob.ln_r; c.D = h->prob.D;
    c.g1 = h->g1;
    c.res = res; c.writer = true;
    c.v = CtlVecs{ysum.data(), yprev.data(), wsum.data(), besty.data(), claimy.data(),
                  ywin.data(), zv.data(), ynew.data(), pU.data(), v1.data()};
    c.s = CtlSlots{h->ring.data(), cap, dd, h->pd_pending.data(), h->pd_callmin.data(),
                   h->pd_sep.data(), h->last.data(), h->pd_best.data()};
    PassParams pp{};
    const int rw = red_width(h->prob.kind, d);
    std::vector<double> red(rw), loc(rw);
    int act = c.begin(*args, h->red0.data(), y_tilde, best_y, &pp);
    int64_t passes = 0, width_passes = 0;
    while (act == kPass) {
        double* dst = h->prob.world > 1 ? loc.data() : red.data();
        if (h->prob.kind == SC_SES && (pp.check || pp.width)) ++width_passes;
        if (h->prob.kind == SC_SES)
            pass_ses(h, pp, ysum.data(), yprev.data(), ywin.data(), dst);
        else
            pass_svm(h, pp, ysum.data(), yprev.data(), ywin.data(), zv.data(), dst);
        if (h->prob.world > 1) h->exchange(loc.data(), rw, red.data());
        ++passes;
        act = c.after_pass(red.data(), h->red0.data(), y_tilde, &pp);
    }
    for (int j = 0; j < dd; ++j) best_y[j] = besty[j];
    res->passes = passes;
    res->width_passes = width_passes;
    if (c.status == SC_EWIDTH) return fail(h, SC_EWIDTH, "width violation");
    return c.status;
}

// sc_solve: the whole adaptive search between passes, the same Search state machine the
// kernel runs (scmwu_control.h), driven by the host loop
int sc_solve(sc_handle* h, const sc_solve_args* args, const double* seed_y,
             sc_solve_result* res, double* best_y, sc_search_step* steps) {
    if (!h || !args || !seed_y || !res || !best_y || (!steps && args->max_steps > 0))
        return SC_EARG;
    memset(res, 0, sizeof(*res));
    const int d = h->prob.d, dd = h->dd;
    if (h->prob.world > 1 && !h->exchange) return fail(h, SC_EARG, "no exchange callback");
    const int64_t T = std::max<int64_t>(args->refine_horizon, kBracketTestCap);
    int64_t cap = (T / 2 > kLadderBase ? T / 2 : kLadderBase) + 2;
    if (cap > (1 << 21)) cap = (1 << 21);
    h->ring.assign((size_t)cap * dd, 0.0);
    h->pd_best.assign(h->pd_best.size(), 0.0);   // best_pd is per solve (R/svm.py:171)
    std::vector<double> ysum(dd), yprev(dd), wsum(dd), besty(dd), claimy(dd), ywin(dd),
        zv(dd), ynew(dd), pU(dd), v1(h->v1), sbest(dd), ytd(dd);
    sc_ftp_result fres{};
    Control<HostLanes> c;
    c.kind = h->prob.kind; c.d = d; c.dd = dd;
    c.is_max = h->prob.kind == SC_SES;
    c.rho = h->prob.rho; c.inv_rho = 1.0 / h->prob.rho; c.R = h->prob.R;
    c.ln_r = h->prob.ln_r; c.D = h->prob.D;
    c.g1 = h->g1;
    c.res = &fres; c.writer = true;
    c.v = CtlVecs{ysum.data(), yprev.data(), wsum.data(), besty.data(), claimy.data(),
                  ywin.data(), zv.data(), ynew.data(), pU.data(), v1.data()};
    c.s = CtlSlots{h->ring.data(), cap, dd, h->pd_pending.data(), h->pd_callmin.data(),
                   h->pd_sep.data(), h->last.data(), h->pd_best.data()};
    Search<HostLanes> S;
    S.R = h->prob.R; S.rho = h->prob.rho; S.ln_r = h->prob.ln_r;
    S.kind = h->prob.kind; S.d = d; S.dd = dd;
    S.sbest = sbest.data(); S.yprog = ywin.data(); S.log = steps; S.writer = true;
    PassParams pp{};
    const int rw = red_width(h->prob.kind, d);
    std::vector<double> red(rw), loc(rw);
    int act = S.begin(c, *args, seed_y, &pp);
    int64_t passes = 0, width_passes = 0;
    while (act == kPass) {
        double* dst = h->prob.world > 1 ? loc.data() : red.data();
        if (h->prob.kind == SC_SES && (pp.check || pp.width)) ++width_passes;
        if (h->prob.kind == SC_SES)
            pass_ses(h, pp, ysum.data(), yprev.data(), ywin.data(), dst);
        else
            pass_svm(h, pp, ysum.data(), yprev.data(), ywin.data(), zv.data(), dst);
        if (h->prob.world > 1) h->exchange(loc.data(), rw, red.data());
        ++passes;
        act = S.after_pass(c, red.data(), h->red0.data(), ytd.data(), &pp);
    }
    for (int j = 0; j < dd; ++j) best_y[j] = sbest[j];
    res->lower = S.Lb; res->upper = S.Ub; res->best_value = S.best_f;
    res->has_best = S.has_best; res->termination = S.termination();
    res->total_iterations = S.total; res->search_steps = S.nsteps;
    res->has_pd = S.has_pd; res->pd_dist = S.pd_best;
    res->seed_f = S.seed_f; res->final_f = S.final_f;
    res->width_alpha = S.w_alpha; res->width_iteration = S.w_iter; res->width_norm = S.w_norm;
    res->passes = passes; res->width_passes = width_passes;
    if (S.status == SC_EWIDTH) return fail(h, SC_EWIDTH, "width violation");
    if (S.status != SC_OK) return fail(h, S.status, "solve failed");
    return SC_OK;
}

int sc_progress_parts(sc_handle* h, const double* y, double* out) {
    if (!h || !y || !out) return SC_EARG;
    const int d = h->prob.d;
    const int64_t n = h->prob.n_local;
    if (h->prob.kind == SC_SES) {
        double best = -INFINITY;
        for (int64_t i = 0; i < n; ++i) {
            double s = 0;
            for (int j = 0; j < d; ++j) { double x = h->X[i * d + j] - y[j]; s = fma(x, x, s); }
            best = fmax(best, sqrt(s) + h->radii[i]);
        }
        out[0] = best;
        out[1] = 0.0;
    } else {
        double mP = INFINITY, xQ = -INFINITY;
        for (int64_t i = 0; i < n; ++i) {
            double s = 0;
            for (int j = 0; j < d; ++j) s = fma(h->X[i * d + j], y[j], s);
            if (i < h->prob.n1_local) mP = fmin(mP, s); else xQ = fmax(xQ, s);
        }
        out[0] = mP;
        out[1] = xQ;
    }
    return SC_OK;
}

int sc_progress(sc_handle* h, const double* y, double* f) {
    if (!h || !y || !f || h->prob.world > 1) return SC_EARG;
    double parts[2];
    sc_progress_parts(h, y, parts);
    if (h->prob.kind == SC_SES) {
        *f = parts[0];
    } else {
        double nrm = 0;
        for (int j = 0; j < h->prob.d; ++j) nrm += y[j] * y[j];
        *f = Control<HostLanes>::svm_margin(parts[0], parts[1], sqrt(nrm));
    }
    return SC_OK;
}

int sc_local_red0(sc_handle* h, double* out) {
    if (!h || !out) return SC_EARG;
    std::copy(h->red0_local.begin(), h->red0_local.end(), out);
    return SC_OK;
}

// on-device generation has no CPU counterpart: the emulator only exports the symbol
int sc_create_generated(sc_problem*, const sc_gen*, double*, sc_handle** out) {
    if (out) *out = nullptr;
    return SC_EARG;
}

int sc_set_range(sc_handle* h, double D) {
    if (!h || !(D >= 0.0)) return SC_EARG;
    sc_problem& p = h->prob;   // as the device library's derive_constants
    p.D = D;
    if (p.kind == SC_SES) {
        p.rho = 3.0 * D / sqrt(2.0);
        p.R = sqrt(2.0);
        p.rank = 2 * (p.n - 1);
    } else {
        p.rho = 2.0 * D;
        p.R = 2.0;
        p.rank = p.n;
    }
    p.ln_r = log((double)p.rank);
    return SC_OK;
}

// the device's sc_row_range on the host: the same numpy-order row norms (np_rownorm.h)
int sc_row_range(sc_handle* h, double* D_out) {
    if (!h || !D_out) return SC_EARG;
    const sc_problem& P = h->prob;
    const bool ses = P.kind == SC_SES;
    const int d = P.d;
    double best = -INFINITY;
    for (int64_t i = ses && P.row0 == 0 ? 1 : 0; i < P.n_local; ++i) {
        const double v = scmwu::np_range_term(&h->X[i * d], ses ? h->v1.data() : nullptr, d,
                                              h->g1, ses ? h->radii[i] : 0.0, ses);
        best = v > best || v != v ? v : best;
    }
    *D_out = best;
    return SC_OK;
}

// the verification baselines are device-only; the emulator only exports the symbols
int sc_meb_baseline(sc_handle*, int64_t, double*, double*) { return SC_EARG; }
int sc_gilbert_baseline(sc_handle*, double, int64_t, double*, double*, int64_t*, double*,
                        double*) {
    return SC_EARG;
}

int sc_read_rows(sc_handle* h, int64_t first, int64_t count, double* out) {
    if (!h || !out || first < 0 || count < 0 || first + count > h->prob.n_local) return SC_EARG;
    const int d = h->prob.d;
    std::copy(h->X.begin() + first * d, h->X.begin() + (first + count) * d, out);
    return SC_OK;
}

int sc_set_globals(sc_handle* h, const double* red0, const double* v1, double g1) {
    if (!h || !red0) return SC_EARG;
    std::copy(red0, red0 + h->red0.size(), h->red0.begin());
    if (v1) std::copy(v1, v1 + h->prob.d, h->v1.begin());
    h->g1 = g1;
    return SC_OK;
}

int sc_ipc_handle(sc_handle* h, void* out64) { (void)h; (void)out64; return SC_EARG; }
int sc_connect(sc_handle* h, const void* handles) { (void)h; (void)handles; return SC_EARG; }

int sc_pd_commit(sc_handle* h, int32_t which) {
    if (!h || h->prob.kind != SC_SVM) return SC_EARG;
    if (which == 0) h->pd_best = h->pd_callmin;
    else if (which == 1) h->pd_best = h->pd_sep;
    else if (which == 2) h->pd_best.assign(h->pd_best.size(), 0.0);
    else return SC_EARG;
    return SC_OK;
}

int sc_pd_pair(sc_handle* h, double* mu, double* gam, double* dist) {
    if (!h || h->prob.kind != SC_SVM || !mu || !gam || !dist) return SC_EARG;
    const int d = h->prob.d, dd = h->dd;
    const int64_t n = h->prob.n_local, n1 = h->prob.n1_local;
    const double* W = h->pd_best.data();
    const IterState st = *reinterpret_cast<const IterState*>(W + dd + (dd & 1));
    const double er = st.eta / h->prob.rho;
    double sP = 0, sQ = 0;
    std::vector<double> e(n);
    for (int64_t i = 0; i < n; ++i) {
        const bool P = i < n1;
        double dW = 0;
        for (int j = 0; j < d; ++j) dW = fma(h->X[i * d + j], W[j], dW);
        double lg = -er * ((P ? 1.0 : -1.0) * dW - (P ? W[d] : W[d + 1]));
        e[i] = exp(lg - st.shift);
        (P ? sP : sQ) += e[i];
    }
    if (h->prob.world > 1) {
        for (int64_t i = 0; i < n; ++i) (i < n1 ? mu[i] : gam[i - n1]) = e[i];
        *dist = NAN;
        return SC_OK;
    }
    std::vector<double> z(d, 0.0);
    for (int64_t i = 0; i < n; ++i) {
        if (i < n1) mu[i] = e[i] / sP; else gam[i - n1] = e[i] / sQ;
    }
    for (int64_t i = 0; i < n; ++i)
        for (int j = 0; j < d; ++j)
            z[j] += (i < n1 ? mu[i] : -gam[i - n1]) * h->X[i * d + j];
    double s = 0;
    for (int j = 0; j < d; ++j) s += z[j] * z[j];
    *dist = sqrt(s);
    return SC_OK;
}

int sc_iterate(sc_handle* h, double* p) {
    (void)h; (void)p;
    return SC_EARG;
}

int sc_set_grid(sc_handle* h, int32_t grid) { (void)h; (void)grid; return SC_OK; }

int sc_info(const sc_handle* h, int64_t* out) {
    if (!h || !out) return SC_EARG;
    for (int i = 0; i < 8; ++i) out[i] = 0;
    out[0] = 1; out[1] = 1;
    return SC_OK;
}

int sc_mark(sc_handle* h, int32_t which) { return h && (which == 0 || which == 1) ? SC_OK : SC_EARG; }
int sc_elapsed(sc_handle* h, float* ms) {
    if (!h || !ms) return SC_EARG;
    *ms = 0.0f;
    return SC_OK;
}
int64_t sc_launches(const sc_handle* h) { (void)h; return 0; }
int sc_debug_timing(sc_handle* h, double* out) {
    if (!h || !out) return SC_EARG;
    for (int i = 0; i < 9 + 6 * 160 + 7; ++i) out[i] = 0.0;
    return SC_OK;
}

const char* sc_last_error(const sc_handle* h) { return h ? h->err.c_str() : "null handle"; }

void sc_destroy(sc_handle* h) { delete h; }

}  // extern "C"
