// cvk_krylov.cu -- persistent, cooperative Krylov solvers for complex-FP64
// CSR systems on sm_100a.  One launch = one complete solve: every scalar
// recurrence runs on the device (redundantly and bitwise identically in every
// CTA), so there is no host round trip per iteration.
//
// Reference algorithms (paths relative to the reference's proj/core/):
//   bicgstab    src/krylov.cpp:57-138
//   bicgstab_l  src/krylov.cpp:140-286
//   tfqmr       src/krylov.cpp:288-375
//   gmres       beyond reference (oracle/cavac_oracle.c orc_gmres)
//   true_relative_residual src/krylov.cpp:17-23
//
// Fusion: each phase between two grid barriers fuses the reference's vector
// updates with the SpMV + Jacobi apply that consumes them; vectors that the
// SpMV gathers at neighbour columns are produced on the fly from their inputs
// (e.g. p = r + beta (p - omega v) inside the SpMV of p), ping-ponged so the
// owner's write never races a neighbour's read.  Per element the arithmetic
// is exactly the reference's sequence of roundings, so in REF mode (S = 1,
// sequential sums) the iterates are bitwise those of the reference.
#include "cvk_dcgs2.cuh"
#include "cvk_engine.cuh"
#include "cvk_kernels.h"

namespace cvk {

// breakdown codes (include/cavac_b200.h CVK_BRK_*)
constexpr int CVK_BRK_RHO_ = 1;
constexpr int CVK_BRK_PAP_ = 8;

namespace {

__device__ __forceinline__ void write_report(const KArgs& a, int cta, int conv, int brk, long long it,
                                             double final_relres, double true_relres,
                                             long long hist_len, int err) {
    if (cta == 0 && threadIdx.x == 0) {
        a.rep->converged = conv;
        a.rep->breakdown = brk;
        a.rep->iterations = it;
        a.rep->final_relres = final_relres;
        a.rep->true_relres = true_relres;
        a.rep->history_len = hist_len;
        a.rep->error = err;
    }
}

// ||b - A x|| / ||b|| (krylov.cpp:17-23); scratch receives b - Ax.
template <int S, bool REF>
__device__ bool true_relres(GridBar& g, const KArgs& a, double2* scratch, double2* part,
                            double& out) {
    const int n = a.A.n;
    CAcc acc[2] = {};
    const double2* x = a.x;
    const double2* b = a.b;
    for_rows<S>(n, a.G, g.cta, [&](int row, int lane, bool valid) {
        const double2 y = row_sum<S>(a.A, row, lane, valid, [&](int c) { return x[c]; });
        if (valid && lane == 0) {
            const double2 bi = __ldg(b + row);
            const double2 d = cvk_sub(bi, y);
            scratch[row] = d;
            if (!REF) { acc_norm(acc[0], bi); acc_norm(acc[1], d); }
        }
    });
    double2 tot[2];
    if (!reduce<REF, 2>(g, acc, tot, part, n, [&](int i, double2* q) {
            acc_norm(q[0], b[i]);
            acc_norm(q[1], scratch[i]);
        }))
        return false;
    const double bn = sqrt(tot[0].x);
    const double rn = sqrt(tot[1].x);
    out = bn > 0 ? rn / bn : rn;
    return true;
}

}  // namespace

// ================================================================ BiCGSTAB
// work: r, shadow, s, t, p[2], v[2]
template <int S, bool REF>
__device__ __forceinline__ void bicgstab_body(const KArgs& a, GridBar& g) {
    const int n = a.A.n, G = a.G;
    const double2* __restrict__ dinv = a.dinv;
    const double2* __restrict__ b = a.b;
    double2* x = a.x;
    double2* r = a.work;
    double2* sh = a.work + (size_t)n;
    double2* s = a.work + 2 * (size_t)n;
    double2* t = a.work + 3 * (size_t)n;
    double2* pv[2] = {a.work + 4 * (size_t)n, a.work + 5 * (size_t)n};
    double2* vv[2] = {a.work + 6 * (size_t)n, a.work + 7 * (size_t)n};
    double2* part[kRegions];
    for (int q = 0; q < kRegions; ++q) part[q] = a.part + (size_t)q * kMaxSlots * G;
    long long hl = 0;

    // r = M^{-1} b, shadow = r, x = 0; ||r||^2 and <shadow, r>.  Warm start
    // (beyond the reference, Schwarz inner solves): r = M^{-1} (b - A x0) and
    // the same bnorm = ||M^{-1} b|| the relative residuals are measured by.
    CAcc acc0[2] = {};
    if (a.warm) {
        auto xat = [&](int c) -> double2 { return x[c]; };
        for_rows<S>(n, G, g.cta, [&](int row, int lane, bool valid) {
            const double2 y = row_sum<S>(a.A, row, lane, valid, xat);
            if (valid && lane == 0) {
                const double2 bi = __ldg(b + row);
                const double2 ri = prec_apply(dinv, row, cvk_sub(bi, y));
                r[row] = ri;
                sh[row] = ri;
                if (!REF) { acc_norm(acc0[0], prec_apply(dinv, row, bi)); acc_dot(acc0[1], ri, ri); }
            }
        });
    } else {
        for_elems(n, G, g.cta, [&](int i) {
            const double2 ri = prec_apply(dinv, i, __ldg(b + i));
            r[i] = ri;
            sh[i] = ri;
            x[i] = make_double2(0.0, 0.0);
            if (!REF) { acc_norm(acc0[0], ri); acc_dot(acc0[1], ri, ri); }
        });
    }
    double2 t0[2];
    if (!reduce<REF, 2>(g, acc0, t0, part[0], n, [&](int i, double2* q) {
            acc_norm(q[0], a.warm ? prec_apply(dinv, i, __ldg(b + i)) : r[i]);
            acc_dot(q[1], sh[i], r[i]);
        })) {
        write_report(a, g.cta, 0, 0, 0, 0, 0, 0, 1);
        return;
    }
    const double bnorm = sqrt(t0[0].x);
    if (bnorm == 0.0) {  // krylov.cpp:70-74: converged, true_relres left at 0
        write_report(a, g.cta, 1, 0, 0, 0.0, 0.0, 0, 0);
        return;
    }
    const double brk = 1e-30 * bnorm * bnorm;
    const double tol = a.tol;

    double2 rho_new = t0[1];
    double2 rho = make_double2(1, 0), alpha = make_double2(1, 0), omega = make_double2(1, 0);
    double2 beta = make_double2(0, 0);
    int conv = 0, brkc = 0, cur = 0;
    long long iters = 0;
    double final_relres = 0.0;
    bool ok = true;

    for (long long it = 1; it <= a.max_iter; ++it) {
        if (cvk_abs(rho_new) < brk) { brkc = 1; iters = it - 1; break; }
        const bool first = (it == 1);
        if (!first) beta = cvk_mul(cvk_cdiv(rho_new, rho), cvk_cdiv(alpha, omega));
        rho = rho_new;
        const double2* pc = pv[cur];
        const double2* vc = vv[cur];
        double2* pn = pv[cur ^ 1];
        double2* vn = vv[cur ^ 1];
        const double2 nom = cvk_neg(omega);
        // p = r + beta (p - omega v)  [axpy_inplace(-omega, v, p); xpay_inplace(beta, p, r)]
        auto pnew = [&](int c) -> double2 {
            const double2 rc = r[c];
            if (first) return rc;
            const double2 tmp = cvk_add(pc[c], cvk_mul(nom, vc[c]));
            return cvk_add(cvk_mul(beta, tmp), rc);
        };
        // phase A: v = M^{-1} A p; gamma = <shadow, v>
        CAcc accA[1] = {};
        for_rows<S>(n, G, g.cta, [&](int row, int lane, bool valid) {
            const double2 y = row_sum<S>(a.A, row, lane, valid, pnew);
            if (valid && lane == 0) {
                const double2 vi = prec_apply(dinv, row, y);
                pn[row] = pnew(row);
                vn[row] = vi;
                if (!REF) acc_dot(accA[0], sh[row], vi);
            }
        });
        double2 gam[1];
        ok = reduce<REF, 1>(g, accA, gam, part[1], n,
                            [&](int i, double2* q) { acc_dot(q[0], sh[i], vn[i]); });
        if (!ok) break;
        if (cvk_abs(gam[0]) < brk) { brkc = 2; iters = it - 1; break; }
        alpha = cvk_cdiv(rho, gam[0]);
        const double2 nal = cvk_neg(alpha);
        // s = r - alpha v (axpy copy), x += alpha p; t = M^{-1} A s
        auto sval = [&](int c) -> double2 { return cvk_add(r[c], cvk_mul(nal, vn[c])); };
        CAcc accB[3] = {};
        for_rows<S>(n, G, g.cta, [&](int row, int lane, bool valid) {
            const double2 y = row_sum<S>(a.A, row, lane, valid, sval);
            if (valid && lane == 0) {
                const double2 ti = prec_apply(dinv, row, y);
                const double2 si = sval(row);
                s[row] = si;
                t[row] = ti;
                x[row] = cvk_add(x[row], cvk_mul(alpha, pn[row]));
                if (!REF) { acc_norm(accB[0], si); acc_dot(accB[1], ti, ti); acc_dot(accB[2], ti, si); }
            }
        });
        double2 tB[3];
        ok = reduce<REF, 3>(g, accB, tB, part[2], n, [&](int i, double2* q) {
            const double2 si = s[i], ti = t[i];
            acc_norm(q[0], si);
            acc_dot(q[1], ti, ti);
            acc_dot(q[2], ti, si);
        });
        if (!ok) break;
        double relres = sqrt(tB[0].x) / bnorm;
        if (relres <= tol) {
            conv = 1; iters = it; final_relres = relres;
            hist_push(a, g.cta, hl, relres);
            break;
        }
        if (cvk_abs(tB[1]) < brk) { brkc = 3; iters = it; break; }
        omega = cvk_cdiv(tB[2], tB[1]);
        const double2 nom2 = cvk_neg(omega);
        // x += omega s; r = s - omega t; ||r||^2, <shadow, r>
        CAcc accC[2] = {};
        for_elems(n, G, g.cta, [&](int i) {
            const double2 si = s[i];
            x[i] = cvk_add(x[i], cvk_mul(omega, si));
            const double2 ri = cvk_add(si, cvk_mul(nom2, t[i]));
            r[i] = ri;
            if (!REF) { acc_norm(accC[0], ri); acc_dot(accC[1], sh[i], ri); }
        });
        double2 tC[2];
        ok = reduce<REF, 2>(g, accC, tC, part[0], n, [&](int i, double2* q) {
            acc_norm(q[0], r[i]);
            acc_dot(q[1], sh[i], r[i]);
        });
        if (!ok) break;
        relres = sqrt(tC[0].x) / bnorm;
        final_relres = relres;
        iters = it;
        hist_push(a, g.cta, hl, relres);
        if (relres <= tol) { conv = 1; break; }
        rho_new = tC[1];
        cur ^= 1;
    }
    double trr = 0.0;
    if (ok) ok = true_relres<S, REF>(g, a, s, part[1], trr);
    write_report(a, g.cta, conv, brkc, iters, final_relres, trr, hl, ok ? 0 : 1);
}

// ==================================================================== COCG
// Beyond the reference (oracle/cavac_oracle.c orc_cocg): conjugate orthogonal
// CG for the complex-symmetric operator, in the reference's conventions (x0 =
// 0, Jacobi, relres = ||M^-1 r|| / ||M^-1 b||, breakdown 1e-30 ||M^-1 b||^2).
// One SpMV per iteration: phase A forms p = z + beta p inside the SpMV
// gathers and takes mu = p^T A p; phase B updates x, r, z and takes ||z||^2,
// r^T z.  work: r, z, q, p[2]
template <int S, bool REF>
__device__ __forceinline__ void cocg_body(const KArgs& a, GridBar& g) {
    const int n = a.A.n, G = a.G;
    const double2* __restrict__ dinv = a.dinv;
    const double2* __restrict__ b = a.b;
    double2* x = a.x;
    double2* r = a.work;
    double2* z = a.work + (size_t)n;
    double2* q = a.work + 2 * (size_t)n;
    double2* pv[2] = {a.work + 3 * (size_t)n, a.work + 4 * (size_t)n};
    double2* part[kRegions];
    for (int k = 0; k < kRegions; ++k) part[k] = a.part + (size_t)k * kMaxSlots * G;
    long long hl = 0;

    CAcc acc0[2] = {};
    for_elems(n, G, g.cta, [&](int i) {
        const double2 ri = __ldg(b + i);
        const double2 zi = prec_apply(dinv, i, ri);
        r[i] = ri;
        z[i] = zi;
        x[i] = make_double2(0.0, 0.0);
        if (!REF) { acc_norm(acc0[0], zi); acc_udot(acc0[1], ri, zi); }
    });
    double2 t0[2];
    if (!reduce<REF, 2>(g, acc0, t0, part[0], n, [&](int i, double2* qq) {
            acc_norm(qq[0], z[i]);
            acc_udot(qq[1], r[i], z[i]);
        })) {
        write_report(a, g.cta, 0, 0, 0, 0, 0, 0, 1);
        return;
    }
    const double bnorm = sqrt(t0[0].x);
    if (bnorm == 0.0) {
        write_report(a, g.cta, 1, 0, 0, 0.0, 0.0, 0, 0);
        return;
    }
    const double brk = 1e-30 * bnorm * bnorm;
    double2 rho = t0[1], beta = make_double2(0, 0);
    int conv = 0, brkc = 0, cur = 0;
    long long iters = 0;
    double final_relres = 0.0;
    bool ok = true;
    for (long long it = 1; it <= a.max_iter; ++it) {
        if (cvk_abs(rho) < brk) { brkc = CVK_BRK_RHO_; iters = it - 1; break; }
        const bool first = (it == 1);
        const double2* pc = pv[cur];
        double2* pn = pv[cur ^ 1];
        auto pnew = [&](int c) -> double2 {
            const double2 zc = z[c];
            return first ? zc : cvk_add(cvk_mul(beta, pc[c]), zc);
        };
        // phase A: p = z + beta p, q = A p; mu = p^T q
        CAcc accA[1] = {};
        for_rows<S>(n, G, g.cta, [&](int row, int lane, bool valid) {
            const double2 y = row_sum<S>(a.A, row, lane, valid, pnew);
            if (valid && lane == 0) {
                const double2 pi = pnew(row);
                pn[row] = pi;
                q[row] = y;
                if (!REF) acc_udot(accA[0], pi, y);
            }
        });
        double2 mu[1];
        ok = reduce<REF, 1>(g, accA, mu, part[1], n, [&](int i, double2* qq) { acc_udot(qq[0], pn[i], q[i]); });
        if (!ok) break;
        if (cvk_abs(mu[0]) < brk) { brkc = CVK_BRK_PAP_; iters = it - 1; break; }
        const double2 alpha = cvk_cdiv(rho, mu[0]), nal = cvk_neg(alpha);
        // phase B: x += alpha p; r -= alpha q; z = M^-1 r; ||z||^2, r^T z
        CAcc accB[2] = {};
        for_elems(n, G, g.cta, [&](int i) {
            x[i] = cvk_add(x[i], cvk_mul(alpha, pn[i]));
            const double2 ri = cvk_add(r[i], cvk_mul(nal, q[i]));
            const double2 zi = prec_apply(dinv, i, ri);
            r[i] = ri;
            z[i] = zi;
            if (!REF) { acc_norm(accB[0], zi); acc_udot(accB[1], ri, zi); }
        });
        double2 tB[2];
        ok = reduce<REF, 2>(g, accB, tB, part[2], n, [&](int i, double2* qq) {
            acc_norm(qq[0], z[i]);
            acc_udot(qq[1], r[i], z[i]);
        });
        if (!ok) break;
        const double relres = sqrt(tB[0].x) / bnorm;
        final_relres = relres;
        iters = it;
        hist_push(a, g.cta, hl, relres);
        if (relres <= a.tol) { conv = 1; break; }
        beta = cvk_cdiv(tB[1], rho);
        rho = tB[1];
        cur ^= 1;
    }
    double trr = 0.0;
    if (ok) ok = true_relres<S, REF>(g, a, q, part[1], trr);
    write_report(a, g.cta, conv, brkc, iters, final_relres, trr, hl, ok ? 0 : 1);
}

// =================================================================== tfQMR
// work: r, shadow, w, u[2], au, v, d
template <int S, bool REF>
__device__ __forceinline__ void tfqmr_body(const KArgs& a, GridBar& g) {
    const int n = a.A.n, G = a.G;
    const double2* __restrict__ dinv = a.dinv;
    const double2* __restrict__ b = a.b;
    double2* x = a.x;
    double2* r = a.work;
    double2* sh = a.work + (size_t)n;
    double2* w = a.work + 2 * (size_t)n;
    double2* uu[2] = {a.work + 3 * (size_t)n, a.work + 4 * (size_t)n};
    double2* au = a.work + 5 * (size_t)n;
    double2* v = a.work + 6 * (size_t)n;
    double2* d = a.work + 7 * (size_t)n;
    double2* part[kRegions];
    for (int q = 0; q < kRegions; ++q) part[q] = a.part + (size_t)q * kMaxSlots * G;
    long long hl = 0;
    const double tol = a.tol;

    CAcc acc0[2] = {};
    for_elems(n, G, g.cta, [&](int i) {
        const double2 ri = prec_apply(dinv, i, __ldg(b + i));
        r[i] = ri; sh[i] = ri; w[i] = ri; uu[0][i] = ri;
        d[i] = make_double2(0, 0);
        x[i] = make_double2(0, 0);
        if (!REF) { acc_norm(acc0[0], ri); acc_dot(acc0[1], ri, ri); }
    });
    double2 t0[2];
    if (!reduce<REF, 2>(g, acc0, t0, part[0], n, [&](int i, double2* q) {
            acc_norm(q[0], r[i]);
            acc_dot(q[1], sh[i], r[i]);
        })) { write_report(a, g.cta, 0, 0, 0, 0, 0, 0, 1); return; }
    const double bnorm = sqrt(t0[0].x);
    if (bnorm == 0.0) { write_report(a, g.cta, 1, 0, 0, 0.0, 0.0, 0, 0); return; }
    const double brk = 1e-30 * bnorm * bnorm;
    double2 rho = t0[1];
    int cur = 0;
    bool ok = true;
    double2 sigma0 = make_double2(0, 0);

    // au = M^{-1} A u; v = au; sigma = <shadow, v>
    {
        const double2* u0 = uu[0];
        CAcc acc[1] = {};
        for_rows<S>(n, G, g.cta, [&](int row, int lane, bool valid) {
            const double2 y = row_sum<S>(a.A, row, lane, valid, [&](int c) { return u0[c]; });
            if (valid && lane == 0) {
                const double2 ai = prec_apply(dinv, row, y);
                au[row] = ai; v[row] = ai;
                if (!REF) acc_dot(acc[0], sh[row], ai);
            }
        });
        double2 tt[1];
        ok = reduce<REF, 1>(g, acc, tt, part[1], n, [&](int i, double2* q) { acc_dot(q[0], sh[i], v[i]); });
        if (!ok) { write_report(a, g.cta, 0, 0, 0, 0, 0, 0, 1); return; }
        rho = t0[1];
        // sigma carried into the loop
        sigma0 = tt[0];
    }
    double2 sigma = sigma0;
    double tau = bnorm, theta = 0.0;
    double2 eta = make_double2(0, 0), alpha = make_double2(0, 0);
    int conv = 0, brkc = 0;
    long long iters = 0;
    double final_relres = 0.0;
    bool pending_x = false;  // x += eta d still owed
    int region = 2;

    for (long long hs = 0; hs < 2 * a.max_iter; hs += 2) {
        // ---------------- even half-step
        if (cvk_abs(sigma) < brk) { brkc = 6; break; }
        alpha = cvk_cdiv(rho, sigma);
        const double2 nal = cvk_neg(alpha);
        {
            const double2 coef = cvk_cdiv(cvk_scale(theta * theta, eta), alpha);
            const double2* uc = uu[cur];
            CAcc acc[1] = {};
            for_elems(n, G, g.cta, [&](int i) {
                const double2 wi = cvk_add(w[i], cvk_mul(nal, au[i]));
                w[i] = wi;
                d[i] = cvk_add(cvk_mul(coef, d[i]), uc[i]);
                if (!REF) acc_norm(acc[0], wi);
            });
            double2 tt[1];
            ok = reduce<REF, 1>(g, acc, tt, part[region], n, [&](int i, double2* q) { acc_norm(q[0], w[i]); });
            region = (region + 1) % kRegions;
            if (!ok) break;
            theta = sqrt(tt[0].x) / tau;
            const double c = 1.0 / sqrt(1.0 + theta * theta);
            tau = tau * theta * c;
            eta = cvk_scale(c * c, alpha);
            pending_x = true;
            const double relres = tau * sqrt((double)(hs + 2)) / bnorm;
            final_relres = relres;
            iters = hs / 2 + 1;
            if (relres <= tol) { conv = 1; break; }
        }
        // ---------------- even tail + odd head:
        // u' = u - alpha v; au = M^{-1} A u'; x += eta d; w -= alpha au; d = coef d + u'
        const double2 eta_e = eta;
        const double2 coef_o = cvk_cdiv(cvk_scale(theta * theta, eta), alpha);
        {
            const double2* uc = uu[cur];
            double2* un = uu[cur ^ 1];
            auto uval = [&](int c) -> double2 { return cvk_add(uc[c], cvk_mul(nal, v[c])); };
            CAcc acc[2] = {};
            for_rows<S>(n, G, g.cta, [&](int row, int lane, bool valid) {
                const double2 y = row_sum<S>(a.A, row, lane, valid, uval);
                if (valid && lane == 0) {
                    const double2 ui = uval(row);
                    const double2 ai = prec_apply(dinv, row, y);
                    un[row] = ui;
                    au[row] = ai;
                    const double2 di = d[row];
                    x[row] = cvk_add(x[row], cvk_mul(eta_e, di));
                    const double2 wi = cvk_add(w[row], cvk_mul(nal, ai));
                    w[row] = wi;
                    d[row] = cvk_add(cvk_mul(coef_o, di), ui);
                    if (!REF) { acc_norm(acc[0], wi); acc_dot(acc[1], sh[row], wi); }
                }
            });
            double2 tt[2];
            ok = reduce<REF, 2>(g, acc, tt, part[region], n, [&](int i, double2* q) {
                acc_norm(q[0], w[i]);
                acc_dot(q[1], sh[i], w[i]);
            });
            region = (region + 1) % kRegions;
            if (!ok) break;
            cur ^= 1;
            // odd half-step scalars
            theta = sqrt(tt[0].x) / tau;
            const double c = 1.0 / sqrt(1.0 + theta * theta);
            tau = tau * theta * c;
            eta = cvk_scale(c * c, alpha);
            pending_x = true;
            const double relres = tau * sqrt((double)(hs + 1 + 2)) / bnorm;
            final_relres = relres;
            iters = (hs + 1) / 2 + 1;
            hist_push(a, g.cta, hl, relres);
            if (relres <= tol) { conv = 1; break; }
            const double2 rho_new = tt[1];
            if (cvk_abs(rho) < brk) { brkc = 1; break; }
            const double2 beta = cvk_cdiv(rho_new, rho);
            rho = rho_new;
            // u_next = w + beta u; au_next = M^{-1} A u_next; v = beta(beta v + au) + au_next;
            // x += eta d; sigma = <shadow, v>
            const double2 eta_o = eta;
            const double2* uc2 = uu[cur];
            double2* un2 = uu[cur ^ 1];
            auto unext = [&](int c) -> double2 { return cvk_add(w[c], cvk_mul(beta, uc2[c])); };
            CAcc accO[1] = {};
            for_rows<S>(n, G, g.cta, [&](int row, int lane, bool valid) {
                const double2 y = row_sum<S>(a.A, row, lane, valid, unext);
                if (valid && lane == 0) {
                    const double2 un_i = unext(row);
                    const double2 an = prec_apply(dinv, row, y);
                    un2[row] = un_i;
                    double2 vi = cvk_add(cvk_mul(beta, v[row]), au[row]);
                    vi = cvk_add(cvk_mul(beta, vi), an);
                    v[row] = vi;
                    au[row] = an;
                    x[row] = cvk_add(x[row], cvk_mul(eta_o, d[row]));
                    if (!REF) acc_dot(accO[0], sh[row], vi);
                }
            });
            double2 to[1];
            ok = reduce<REF, 1>(g, accO, to, part[region], n, [&](int i, double2* q) { acc_dot(q[0], sh[i], v[i]); });
            region = (region + 1) % kRegions;
            if (!ok) break;
            pending_x = false;
            cur ^= 1;
            sigma = to[0];
        }
    }
    if (ok && pending_x) {  // the owed x += eta d (krylov.cpp:335)
        const double2 e = eta;
        for_elems(n, G, g.cta, [&](int i) { x[i] = cvk_add(x[i], cvk_mul(e, d[i])); });
        ok = g.sync();
    }
    double trr = 0.0;
    if (ok) ok = true_relres<S, REF>(g, a, r, part[region], trr);
    write_report(a, g.cta, conv, brkc, iters, final_relres, trr, hl, ok ? 0 : 1);
}

// ============================================================ BiCGSTAB(l)
// work: shadow, x-scratch?, then r[0..l], u[0..l], spareR, spareU  (2l+5 vectors)
template <int S, bool REF>
__device__ __forceinline__ void bicgstab_l_body(const KArgs& a, GridBar& g) {
    const int n = a.A.n, G = a.G, L = a.l;
    const double2* __restrict__ dinv = a.dinv;
    const double2* __restrict__ b = a.b;
    double2* x = a.x;
    double2* sh = a.work;
    double2* scratch = a.work + (size_t)n;
    double2* vbase = a.work + 2 * (size_t)n;
    // logical -> physical vector slots: r_i = vbase[ri[i]], u_i = vbase[ui[i]]
    __shared__ int ri[kMaxL + 2], ui[kMaxL + 2];
    __shared__ double2 tau_s[kMaxL * kMaxL], sig_s[kMaxL], gam_s[kMaxL], gp_s[kMaxL], gpp_s[kMaxL];
    if (threadIdx.x <= L) { ri[threadIdx.x] = threadIdx.x; ui[threadIdx.x] = L + 1 + threadIdx.x; }
    if (threadIdx.x == 0) { ri[L + 1] = 2 * L + 2; ui[L + 1] = 2 * L + 3; }
    __syncthreads();
    auto R = [&](int i) -> double2* { return vbase + (size_t)ri[i] * n; };
    auto U = [&](int i) -> double2* { return vbase + (size_t)ui[i] * n; };
    double2* part[kRegions];
    for (int q = 0; q < kRegions; ++q) part[q] = a.part + (size_t)q * kMaxSlots * G;
    int region = 0;
    auto next_part = [&]() { double2* p = part[region]; region = (region + 1) % kRegions; return p; };
    long long hl = 0;
    const double tol = a.tol;

    CAcc acc0[2] = {};
    {
        double2* r0 = R(0);
        for_elems(n, G, g.cta, [&](int i) {
            const double2 v0 = prec_apply(dinv, i, __ldg(b + i));
            r0[i] = v0; sh[i] = v0;
            x[i] = make_double2(0, 0);
            for (int j = 1; j <= L; ++j) R(j)[i] = make_double2(0, 0);
            for (int j = 0; j <= L; ++j) U(j)[i] = make_double2(0, 0);
            if (!REF) { acc_norm(acc0[0], v0); acc_dot(acc0[1], v0, v0); }
        });
    }
    double2 t0[2];
    {
        double2* r0 = R(0);
        if (!reduce<REF, 2>(g, acc0, t0, next_part(), n, [&](int i, double2* q) {
                acc_norm(q[0], r0[i]);
                acc_dot(q[1], sh[i], r0[i]);
            })) { write_report(a, g.cta, 0, 0, 0, 0, 0, 0, 1); return; }
    }
    const double bnorm = sqrt(t0[0].x);
    if (bnorm == 0.0) { write_report(a, g.cta, 1, 0, 0, 0.0, 0.0, 0, 0); return; }
    const double brk = 1e-30 * bnorm * bnorm;
    double2 rho_old = make_double2(1, 0), alpha = make_double2(0, 0), omega = make_double2(1, 0);
    double2 rho_next = t0[1];  // <shadow, r_j> for the coming BiCG step
    int conv = 0, brkc = 0;
    long long iters = 0;
    double final_relres = 0.0;
    bool ok = true;

    for (long long cycle = 1; cycle <= a.max_iter; ++cycle) {
        rho_old = cvk_mul(cvk_neg(omega), rho_old);
        bool broke = false;
        double r0norm = 0.0;
        for (int j = 0; j < L; ++j) {
            const double2 rho = rho_next;
            if (cvk_abs(rho_old) < brk) { brkc = 1; broke = true; break; }
            const double2 beta = cvk_cdiv(cvk_mul(alpha, rho), rho_old);
            rho_old = rho;
            const double2 nbeta = cvk_neg(beta);
            // u_i = r_i - beta u_i (i <= j); u_{j+1} = M^{-1} A u_j; g = <shadow, u_{j+1}>
            {
                const double2* uj_old = U(j);
                const double2* rj = R(j);
                double2* uj_new = vbase + (size_t)ui[L + 1] * n;  // spare
                double2* uj1 = U(j + 1);
                auto ujv = [&](int c) -> double2 { return cvk_add(cvk_mul(nbeta, uj_old[c]), rj[c]); };
                CAcc acc[1] = {};
                for_rows<S>(n, G, g.cta, [&](int row, int lane, bool valid) {
                    const double2 y = row_sum<S>(a.A, row, lane, valid, ujv);
                    if (valid && lane == 0) {
                        const double2 yi = prec_apply(dinv, row, y);
                        uj_new[row] = ujv(row);
                        uj1[row] = yi;
                        if (!REF) acc_dot(acc[0], sh[row], yi);
                    }
                });
                // the other u_i (i < j) in element mapping
                __syncthreads();
                for_elems(n, G, g.cta, [&](int i) {
                    for (int q = 0; q < j; ++q) {
                        double2* uq = U(q);
                        uq[i] = cvk_add(cvk_mul(nbeta, uq[i]), R(q)[i]);
                    }
                });
                double2 tg[1];
                ok = reduce<REF, 1>(g, acc, tg, next_part(), n, [&](int i, double2* q) { acc_dot(q[0], sh[i], uj1[i]); });
                if (!ok) break;
                // swap u_j with the spare slot (uniform in every CTA)
                if (threadIdx.x == 0) { const int tmp = ui[j]; ui[j] = ui[L + 1]; ui[L + 1] = tmp; }
                __syncthreads();
                if (cvk_abs(tg[0]) < brk) { brkc = 4; broke = true; break; }
                alpha = cvk_cdiv(rho_old, tg[0]);
            }
            // r_i -= alpha u_{i+1} (i <= j); r_{j+1} = M^{-1} A r_j; x += alpha u_0
            {
                const double2 nal = cvk_neg(alpha);
                const double2* rj_old = R(j);
                const double2* uj1 = U(j + 1);
                double2* rj_new = vbase + (size_t)ri[L + 1] * n;
                double2* rj1 = R(j + 1);
                auto rjv = [&](int c) -> double2 { return cvk_add(rj_old[c], cvk_mul(nal, uj1[c])); };
                CAcc acc[2] = {};
                for_rows<S>(n, G, g.cta, [&](int row, int lane, bool valid) {
                    const double2 y = row_sum<S>(a.A, row, lane, valid, rjv);
                    if (valid && lane == 0) {
                        const double2 yi = prec_apply(dinv, row, y);
                        rj_new[row] = rjv(row);
                        rj1[row] = yi;
                    }
                });
                __syncthreads();
                const double2* u0 = U(0);
                for_elems(n, G, g.cta, [&](int i) {
                    for (int q = 0; q < j; ++q) {
                        double2* rq = R(q);
                        rq[i] = cvk_add(rq[i], cvk_mul(nal, U(q + 1)[i]));
                    }
                    x[i] = cvk_add(x[i], cvk_mul(alpha, u0[i]));
                    if (!REF) {
                        const double2 r0i = (j == 0) ? rj_new[i] : R(0)[i];
                        acc_norm(acc[0], r0i);
                        acc_dot(acc[1], sh[i], rj1[i]);
                    }
                });
                double2 tr[2];
                ok = reduce<REF, 2>(g, acc, tr, next_part(), n, [&](int i, double2* q) {
                    acc_norm(q[0], (j == 0) ? rj_new[i] : R(0)[i]);
                    acc_dot(q[1], sh[i], rj1[i]);
                });
                if (!ok) break;
                if (threadIdx.x == 0) { const int tmp = ri[j]; ri[j] = ri[L + 1]; ri[L + 1] = tmp; }
                __syncthreads();
                r0norm = sqrt(tr[0].x);
                rho_next = tr[1];
                if (r0norm <= tol * bnorm) { broke = true; break; }
            }
        }
        if (!ok) break;
        if (broke) {
            // krylov.cpp:208-222 (needs ||r_0|| of the current r_0)
            double2 tn[1];
            CAcc accn[1] = {};
            double2* r0 = R(0);
            for_elems(n, G, g.cta, [&](int i) { if (!REF) acc_norm(accn[0], r0[i]); });
            ok = reduce<REF, 1>(g, accn, tn, next_part(), n, [&](int i, double2* q) { acc_norm(q[0], r0[i]); });
            if (!ok) break;
            const double relres = sqrt(tn[0].x) / bnorm;
            final_relres = relres;
            if (relres <= tol) {
                conv = 1; brkc = 0; iters = cycle;
                hist_push(a, g.cta, hl, relres);
            } else {
                iters = cycle - 1;
            }
            break;
        }
        // ---- minimal residual part: MGS on r_1..r_L (krylov.cpp:224-238)
        bool mrbroke = false;
        for (int j = 0; j < L && !mrbroke; ++j) {
            double2* rj1 = R(j + 1);
            for (int i = 0; i <= j; ++i) {
                // apply the pending update r_{j+1} -= tau_{i-1,j} r_i, then
                // the next dot: <r_{i+1}, r_{j+1}> (i < j) or sigma_j, <r_{j+1}, r_0> (i == j)
                const bool has_upd = (i > 0);
                const double2 ntau = has_upd ? cvk_neg(tau_s[(i - 1) * L + j]) : make_double2(0, 0);
                const double2* rprev = has_upd ? R(i) : nullptr;
                const double2* ri1 = R(i + 1);
                const double2* r0 = R(0);
                const bool last = (i == j);
                CAcc acc[2] = {};
                for_elems(n, G, g.cta, [&](int e) {
                    double2 v = rj1[e];
                    if (has_upd) { v = cvk_add(v, cvk_mul(ntau, rprev[e])); rj1[e] = v; }
                    if (!REF) {
                        if (!last) acc_dot(acc[0], ri1[e], v);
                        else { acc_dot(acc[0], v, v); acc_dot(acc[1], v, r0[e]); }
                    }
                });
                double2 tt[2];
                ok = reduce<REF, 2>(g, acc, tt, next_part(), n, [&](int e, double2* q) {
                    if (!last) acc_dot(q[0], ri1[e], rj1[e]);
                    else { acc_dot(q[0], rj1[e], rj1[e]); acc_dot(q[1], rj1[e], r0[e]); }
                });
                if (!ok) break;
                if (!last) {
                    if (threadIdx.x == 0) tau_s[i * L + j] = cvk_cdiv(tt[0], sig_s[i]);
                    __syncthreads();
                } else {
                    if (cvk_abs(tt[0]) < brk) { brkc = 5; mrbroke = true; break; }
                    if (threadIdx.x == 0) { sig_s[j] = tt[0]; gp_s[j] = cvk_cdiv(tt[1], tt[0]); }
                    __syncthreads();
                }
            }
            if (!ok) break;
        }
        if (!ok) break;
        if (mrbroke) {
            double2 tn[1];
            CAcc accn[1] = {};
            double2* r0 = R(0);
            for_elems(n, G, g.cta, [&](int i) { if (!REF) acc_norm(accn[0], r0[i]); });
            ok = reduce<REF, 1>(g, accn, tn, next_part(), n, [&](int i, double2* q) { acc_norm(q[0], r0[i]); });
            if (!ok) break;
            const double relres = sqrt(tn[0].x) / bnorm;
            final_relres = relres;
            iters = cycle;
            if (relres <= tol) { conv = 1; brkc = 0; hist_push(a, g.cta, hl, relres); }
            break;
        }
        // gamma, gamma', gamma'' (krylov.cpp:251-262) -- thread 0, then shared
        if (threadIdx.x == 0) {
            gam_s[L - 1] = gp_s[L - 1];
            for (int jj = L - 1; jj-- > 0;) {
                double2 gj = gp_s[jj];
                for (int i = jj + 1; i < L; ++i) gj = cvk_sub(gj, cvk_mul(tau_s[jj * L + i], gam_s[i]));
                gam_s[jj] = gj;
            }
            for (int j = 0; j + 1 < L; ++j) {
                double2 gj = gam_s[j + 1];
                for (int i = j + 1; i + 1 < L; ++i) gj = cvk_add(gj, cvk_mul(tau_s[j * L + i], gam_s[i + 1]));
                gpp_s[j] = gj;
            }
        }
        __syncthreads();
        omega = gam_s[L - 1];
        // updates (krylov.cpp:264-271), per element in the reference's order
        CAcc accU[2] = {};
        {
            double2* r0 = R(0);
            double2* u0 = U(0);
            for_elems(n, G, g.cta, [&](int i) {
                double2 xi = x[i], r0i = r0[i], u0i = u0[i];
                xi = cvk_add(xi, cvk_mul(gam_s[0], r0i));
                r0i = cvk_add(r0i, cvk_mul(cvk_neg(gp_s[L - 1]), R(L)[i]));
                u0i = cvk_add(u0i, cvk_mul(cvk_neg(gam_s[L - 1]), U(L)[i]));
                for (int j = 1; j < L; ++j) {
                    const double2 rj = R(j)[i];
                    u0i = cvk_add(u0i, cvk_mul(cvk_neg(gam_s[j - 1]), U(j)[i]));
                    xi = cvk_add(xi, cvk_mul(gpp_s[j - 1], rj));
                    r0i = cvk_add(r0i, cvk_mul(cvk_neg(gp_s[j - 1]), rj));
                }
                x[i] = xi; r0[i] = r0i; u0[i] = u0i;
                if (!REF) { acc_norm(accU[0], r0i); acc_dot(accU[1], sh[i], r0i); }
            });
            double2 tu[2];
            ok = reduce<REF, 2>(g, accU, tu, next_part(), n, [&](int i, double2* q) {
                acc_norm(q[0], r0[i]);
                acc_dot(q[1], sh[i], r0[i]);
            });
            if (!ok) break;
            const double relres = sqrt(tu[0].x) / bnorm;
            final_relres = relres;
            iters = cycle;
            hist_push(a, g.cta, hl, relres);
            rho_next = tu[1];
            if (relres <= tol) { conv = 1; break; }
        }
    }
    double trr = 0.0;
    if (ok) ok = true_relres<S, REF>(g, a, scratch, next_part(), trr);
    write_report(a, g.cta, conv, brkc, iters, final_relres, trr, hl, ok ? 0 : 1);
}

// ================================================================ GMRES(m)
// Beyond reference: left-preconditioned restarted GMRES, Arnoldi with
// delayed reorthogonalisation (DCGS2: one dot pass and one update pass over
// the basis per step) and complex Givens rotations; order of operations =
// orc_gmres, scalar side shared with the phase kernels (cvk_dcgs2.cuh).
// work: r, W[2], V[0..m]   (m + 4 vectors)
// dynamic shared (gmres_smem_layout): Hu, R [(m+1) m], sn[m], g, gpre, y,
// av, bv, ev [m+1] (double2), cs[m], nu (double)
template <int S, bool REF>
__device__ __forceinline__ void gmres_body(const KArgs& a, GridBar& g) {
    const int n = a.A.n, G = a.G, M = a.m;
    const double2* __restrict__ dinv = a.dinv;
    const double2* __restrict__ b = a.b;
    double2* x = a.x;
    double2* r = a.work;
    double2* Wb[2] = {a.work + (size_t)n, a.work + 2 * (size_t)n};
    double2* V = a.work + 3 * (size_t)n;
    extern __shared__ double2 dsm[];
    GmView gv;
    gv.M = M;
    gv.Hu = dsm;
    gv.R = gv.Hu + (size_t)(M + 1) * M;
    gv.sn = gv.R + (size_t)(M + 1) * M;
    gv.g = gv.sn + M;
    gv.gpre = gv.g + M + 1;
    double2* yv = gv.gpre + M + 1;
    gv.yv = yv;
    gv.av = yv + M + 1;
    gv.bv = gv.av + M + 1;
    gv.ev = gv.bv + M + 1;
    gv.cs = (double*)(gv.ev + M + 1);
    gv.nu = gv.cs + M;
    __shared__ CAcc hsm[2 * kMaxDots + 2][kWarps];
    double2* part[kRegions];
    for (int q = 0; q < kRegions; ++q) part[q] = a.part + (size_t)q * kMaxSlots * G;
    int region = 0;
    auto next_part = [&]() { double2* p = part[region]; region = (region + 1) % kRegions; return p; };
    long long hl = 0;
    const double tol = a.tol;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    auto bar = [] { __syncthreads(); };

    // FAST: <V_q, u_j> and <V_q, w> for q < cnt over the CTA's own 256-row
    // chunks (one warp per chunk), in the canonical row groups of
    // gm_group_dots -> partial slots 2q, 2q+1
    const int nchunk = (n + kThreads - 1) / kThreads;
    auto dual_dot = [&](const double2* uj, const double2* wv, int cnt, double2* pr) {
        for (int q = 0; q < cnt; ++q) {
            const double2* vq = V + (size_t)q * n;
            CAcc s[1][2] = {};
            for (int c = g.cta + warp * G; c < nchunk; c += kWarps * G)
                for (int h = 0; h < 2; ++h) {
                    const int r0 = c * kThreads + 128 * h;
                    const double2* const vb[1] = {vq + r0};
                    if (r0 < n) gm_group_dots<1>(vb, 1, uj + r0, wv + r0, min(128, n - r0), lane, s);
                }
            s[0][0] = warp_sum(s[0][0]);
            s[0][1] = warp_sum(s[0][1]);
            if (lane == 0) {
                hsm[2 * q][warp] = s[0][0];
                hsm[2 * q + 1][warp] = s[0][1];
            }
        }
        __syncthreads();
        for (int k = threadIdx.x; k < 2 * cnt; k += blockDim.x) {
            CAcc s = hsm[k][0];
            for (int w2 = 1; w2 < kWarps; ++w2) cacc_add(s, hsm[k][w2]);
            cacc_store(pr, k, G, g.cta, s);
        }
    };
    auto fold_dual = [&](const double2* pr, int cnt) {
        for (int k = warp; k < 2 * cnt; k += kWarps) {  // one warp per dot product
            const double2 s = fold_one(pr, k, G, lane);
            if (lane == 0) (k & 1 ? gv.bv : gv.av)[k >> 1] = s;
        }
        __syncthreads();
    };
    auto seq_dual = [&](const double2* uj, const double2* wv, int cnt) {
        if (threadIdx.x == 0) {
            for (int q = 0; q < cnt; ++q) {
                const double2* vq = V + (size_t)q * n;
                double2 sa = make_double2(0, 0), sb = make_double2(0, 0);
                for (int i = 0; i < n; ++i) acc_dot(sa, vq[i], uj[i]);
                for (int i = 0; i < n; ++i) acc_dot(sb, vq[i], wv[i]);
                gv.av[q] = sa;
                gv.bv[q] = sb;
            }
        }
        __syncthreads();
    };

    // r = M^{-1} b, x = 0, ||r||
    CAcc acc0[1] = {};
    for_elems(n, G, g.cta, [&](int i) {
        const double2 ri = prec_apply(dinv, i, __ldg(b + i));
        r[i] = ri;
        x[i] = make_double2(0, 0);
        if (!REF) acc_norm(acc0[0], ri);
    });
    double2 t0[1];
    if (!reduce<REF, 1>(g, acc0, t0, next_part(), n, [&](int i, double2* q) { acc_norm(q[0], r[i]); })) {
        write_report(a, g.cta, 0, 0, 0, 0, 0, 0, 1);
        return;
    }
    const double bnorm = sqrt(t0[0].x);
    if (bnorm == 0.0) { write_report(a, g.cta, 1, 0, 0, 0.0, 0.0, 0, 0); return; }
    const double brk = 1e-30 * bnorm * bnorm;
    double beta = bnorm;
    long long total = 0;
    int conv = 0, brkc = 0;
    double final_relres = 0.0;
    bool ok = true;
    int wcur = 0;

    for (;;) {
        if (total > 0) {
            final_relres = beta / bnorm;
            if (final_relres <= tol) { conv = 1; break; }
        }
        if (threadIdx.x == 0) {
            for (int i = 0; i <= M; ++i) gv.g[i] = make_double2(0, 0);
            gv.g[0] = make_double2(beta, 0.0);
        }
        __syncthreads();
        const double2* src = r;
        double scale = beta;
        int k = 0;
        bool stop = false;
        for (int j = 0; j < M; ++j) {
            ++total;
            // ---- S: u_j = V_j = src / scale; w = M^{-1} A u_j
            double2* Vj = V + (size_t)j * n;
            double2* w = Wb[wcur];
            {
                const double2* sp = src;
                const double sc = scale;
                auto vat = [&](int c) -> double2 { return cvk_divr(sp[c], sc); };
                for_rows<S>(n, G, g.cta, [&](int row, int ln, bool valid) {
                    const double2 y = row_sum<S>(a.A, row, ln, valid, vat);
                    if (valid && ln == 0) {
                        Vj[row] = vat(row);
                        w[row] = prec_apply(dinv, row, y);
                    }
                });
                __syncthreads();
            }
            // ---- D: a = V^H u_j, b = V^H w (one pass)
            if (REF) {
                ok = g.sync();
                if (!ok) break;
                seq_dual(Vj, w, j + 1);
                ok = g.sync();
                if (!ok) break;
            } else {
                double2* pr = next_part();
                dual_dot(Vj, w, j + 1, pr);
                ok = g.sync();
                if (!ok) break;
                fold_dual(pr, j + 1);
            }
            const double nu = gm_dcgs2_scalars(gv, j, threadIdx.x, blockDim.x, bar);
            if (!(nu > 0.0)) {
                brkc = 7;
                k = j;
                stop = true;
                break;
            }
            // ---- U: q_j = (u_j - Q a) / nu, u' = w - Q e - gamma u_j; ||u'||
            double hn;
            {
                CAcc acc[1] = {};
                for_elems(n, G, g.cta, [&](int i) {
                    const double2 up = gm_update_row(gv.av, gv.ev, j, nu, Vj[i], w[i],
                                                     [&](int q) { return V[(size_t)q * n + i]; });
                    w[i] = up;
                    if (!REF) acc_norm(acc[0], up);
                });
                double2 tn[1];
                ok = reduce<REF, 1>(g, acc, tn, next_part(), n, [&](int i, double2* q) { acc_norm(q[0], w[i]); });
                if (!ok) break;
                hn = sqrt(tn[0].x);
            }
            if (threadIdx.x == 0) gm_provisional(gv, j, hn, nu);
            __syncthreads();
            const double2 gj1 = gv.g[j + 1];
            const double relres = sqrt(gj1.x * gj1.x + gj1.y * gj1.y) / bnorm;
            final_relres = relres;
            hist_push(a, g.cta, hl, relres);
            k = j + 1;
            if (relres <= tol) { conv = 1; stop = true; break; }
            if (hn * hn < brk) { brkc = 7; stop = true; break; }
            if (total >= a.max_iter) { stop = true; break; }
            src = w;
            scale = hn;
            wcur ^= 1;
        }
        if (!ok) break;
        // back substitution (thread 0), then x += V y
        if (threadIdx.x == 0) gm_back_subst(gv, k, yv);
        __syncthreads();
        for_elems(n, G, g.cta, [&](int i) {
            double2 xi = x[i];
            for (int q = 0; q < k; ++q) xi = cvk_add(xi, cvk_mul(yv[q], V[(size_t)q * n + i]));
            x[i] = xi;
        });
        if (brkc == 7 && final_relres <= tol) { conv = 1; brkc = 0; }
        ok = g.sync();
        if (!ok || stop) break;
        // restart residual r = M^{-1}(b - A x)
        CAcc acc[1] = {};
        for_rows<S>(n, G, g.cta, [&](int row, int ln, bool valid) {
            const double2 y = row_sum<S>(a.A, row, ln, valid, [&](int c) { return x[c]; });
            if (valid && ln == 0) {
                const double2 ri = prec_apply(dinv, row, cvk_sub(__ldg(b + row), y));
                r[row] = ri;
                if (!REF) acc_norm(acc[0], ri);
            }
        });
        double2 tn[1];
        ok = reduce<REF, 1>(g, acc, tn, next_part(), n, [&](int i, double2* q) { acc_norm(q[0], r[i]); });
        if (!ok) break;
        beta = sqrt(tn[0].x);
        if (beta == 0.0) { conv = 1; final_relres = 0.0; break; }
    }
    double trr = 0.0;
    if (ok) ok = true_relres<S, REF>(g, a, Wb[0], next_part(), trr);
    write_report(a, g.cta, conv, brkc, total, final_relres, trr, hl, ok ? 0 : 1);
}

// ------------------------------------------------------------ kernels --

template <int S, bool REF, int SOLVER>
__device__ __forceinline__ void run_body(const KArgs& a, GridBar& g) {
    if (SOLVER == 0) bicgstab_body<S, REF>(a, g);
    else if (SOLVER == 1) bicgstab_l_body<S, REF>(a, g);
    else if (SOLVER == 2) tfqmr_body<S, REF>(a, g);
    else if (SOLVER == 3) gmres_body<S, REF>(a, g);
    else cocg_body<S, REF>(a, g);
}

// one solve per cooperative launch
template <int S, bool REF, int SOLVER>
__global__ void __launch_bounds__(kThreads, kMinCtas) k_solve(KArgs a) {
    GridBar g(a.bar, a.G);
    g.refpar = REF ? a.refpar : 0;
    run_body<S, REF, SOLVER>(a, g);
}

// K10: independent solves (Schwarz subdomains) batched into one cooperative
// launch.  Segment s owns CTAs [segs[s].cta_base, + segs[s].G) with its own
// barrier counter, partials, report and vectors; segments finish at their
// own iteration counts.
template <int S, bool REF, int SOLVER>
__global__ void __launch_bounds__(kThreads, kMinCtas) k_solve_batched(const KArgs* segs, int nseg) {
    __shared__ KArgs sa;
    if (threadIdx.x == 0) {
        int s = 0;
        while (s + 1 < nseg && (int)blockIdx.x >= segs[s + 1].cta_base) ++s;
        sa = segs[s];
    }
    __syncthreads();
    GridBar g(sa.bar, sa.G, (int)blockIdx.x - sa.cta_base);
    g.refpar = REF ? sa.refpar : 0;
    run_body<S, REF, SOLVER>(sa, g);
}

// ----------------------------------------------------------- dispatch --

template <int S, bool REF>
static const void* pick(int solver, bool batched) {
    switch (solver) {
        case 0: return batched ? (const void*)k_solve_batched<S, REF, 0> : (const void*)k_solve<S, REF, 0>;
        case 1: return batched ? (const void*)k_solve_batched<S, REF, 1> : (const void*)k_solve<S, REF, 1>;
        case 2: return batched ? (const void*)k_solve_batched<S, REF, 2> : (const void*)k_solve<S, REF, 2>;
        case 3: return batched ? (const void*)k_solve_batched<S, REF, 3> : (const void*)k_solve<S, REF, 3>;
        case 4: return batched ? (const void*)k_solve_batched<S, REF, 4> : (const void*)k_solve<S, REF, 4>;
    }
    return nullptr;
}

const void* solver_kernel(int solver, int S, bool ref, bool batched) {
    if (ref) return pick<1, true>(solver, batched);
    switch (S) {
        case 1: return pick<1, false>(solver, batched);
        case 2: return pick<2, false>(solver, batched);
        case 4: return pick<4, false>(solver, batched);
        case 8: return pick<8, false>(solver, batched);
        case 16: return pick<16, false>(solver, batched);
    }
    return nullptr;
}

int solver_nwork(int solver, int l, int m) {
    switch (solver) {
        case 0: return 8;
        case 1: return 2 * l + 6;
        case 2: return 8;
        case 3: return m + 4;
        case 4: return 5;
    }
    return 0;
}

size_t solver_smem(int solver, int m) {
    if (solver != 3) return 0;
    return sizeof(double2) * (2 * (size_t)(m + 1) * m + m + 6 * (size_t)(m + 1)) + sizeof(double) * (m + 1);
}

}  // namespace cvk
