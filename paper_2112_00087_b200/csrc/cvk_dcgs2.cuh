// cvk_dcgs2.cuh -- the scalar side of a GMRES(m) Arnoldi step with delayed
// reorthogonalisation (DCGS2), shared by the persistent kernel (cvk_krylov.cu
// gmres_body, state in shared memory) and the phase kernels (cvk_gmres.cu,
// state in global memory).  Order of operations = oracle/cavac_oracle.c
// orc_gmres / gm_rotate, which documents the algorithm.
//
// Step j, after the dot pass left a_q = <V_q, u_j> in av[q] and
// b_q = <V_q, w> in bv[q] (q <= j):
//   gm_dcgs2_scalars  nu, c = <q_j, w>, the delayed correction of column j-1
//                     and its rotation, column j, the update coefficients
//                     ev[q] (q < j) and ev[j] = gamma
//   (update pass)     q_j = (u_j - sum a_q V_q) / nu,
//                     u' = w - sum ev[q] V_q - gamma u_j, hn = ||u'||
//   gm_provisional    Hu[j+1][j] = hn / nu and the provisional rotation of
//                     column j (the residual estimate of step j)
#pragma once

#include "cvk_complex.h"

namespace cvk {

struct GmView {
    double2* Hu;    // (M+1) x M unrotated Hessenberg, [i * M + j]
    double2* R;     // (M+1) x M rotated columns (upper triangle used)
    double* cs;     // M
    double2* sn;    // M
    double2* g;     // M + 1: rotated right-hand side
    double2* gpre;  // M + 1: g[j] before the rotation of column j
    double2* av;    // M + 1: a_q
    double2* bv;    // M + 1: b_q (bv[j] becomes c)
    double2* ev;    // M + 1: update coefficients
    double* nu;     // 1
    int M;
};

// Givens rotation of column col: R[.][col] = Hu[.][col] rotated by 0..col-1,
// then the rotation that annihilates the subdiagonal hsub; g from gp.
__device__ __forceinline__ void gm_rotate(const GmView& v, int col, double hsub, double2 gp) {
    const int M = v.M;
    for (int i = 0; i <= col; ++i) v.R[i * M + col] = v.Hu[i * M + col];
    for (int i = 0; i < col; ++i) {
        const double2 a0 = v.R[i * M + col], c2 = v.R[(i + 1) * M + col];
        v.R[i * M + col] = cvk_add(cvk_scale(v.cs[i], a0), cvk_mul(v.sn[i], c2));
        v.R[(i + 1) * M + col] = cvk_add(cvk_mul(cvk_neg(cvk_conj(v.sn[i])), a0), cvk_scale(v.cs[i], c2));
    }
    const double2 aj = v.R[col * M + col];
    const double aa = sqrt(aj.x * aj.x + aj.y * aj.y);
    const double nr = sqrt(aa * aa + hsub * hsub);
    if (aa == 0.0) {
        v.cs[col] = 0.0;
        v.sn[col] = make_double2(1.0, 0.0);
        v.R[col * M + col] = make_double2(hsub, 0.0);
    } else {
        v.cs[col] = aa / nr;
        v.sn[col] = cvk_scale(hsub / nr, cvk_divr(aj, aa));
        v.R[col * M + col] = cvk_scale(nr, cvk_divr(aj, aa));
    }
    v.g[col + 1] = cvk_mul(cvk_neg(cvk_conj(v.sn[col])), gp);
    v.g[col] = cvk_scale(v.cs[col], gp);
}

// Threads [0, nt) of one CTA, all of which call sync() (a CTA barrier).
// Returns nu (0 when nu^2 <= 0: the candidate lies in span(Q), breakdown).
template <class Sync>
__device__ double gm_dcgs2_scalars(const GmView& v, int j, int tid, int nt, Sync&& sync) {
    const int M = v.M;
    if (tid == 0) {
        double ss = 0.0;
        for (int q = 0; q < j; ++q) ss = ss + cvk_norm(v.av[q]);
        const double nu2 = v.av[j].x - ss;
        double2 cc = v.bv[j];
        for (int q = 0; q < j; ++q) cc = cvk_sub(cc, cvk_cmul(v.av[q], v.bv[q]));
        if (nu2 > 0.0) {
            const double nu = sqrt(nu2);
            const double2 c = cvk_divr(cc, nu);
            v.bv[j] = c;
            v.ev[j] = cvk_divr(c, nu);
            *v.nu = nu;
        } else {
            *v.nu = 0.0;
        }
    }
    sync();
    const double nu = *(volatile double*)v.nu;
    if (!(nu > 0.0)) return 0.0;
    if (j > 0) {  // u_j = nu q_j + Q a: column j-1 in the final basis
        const double2 hjj = v.Hu[j * M + j - 1];
        for (int q = tid; q < j; q += nt) v.Hu[q * M + j - 1] = cvk_add(v.Hu[q * M + j - 1], cvk_mul(hjj, v.av[q]));
        sync();
        if (tid == 0) v.Hu[j * M + j - 1] = cvk_scale(nu, hjj);
        sync();
    }
    for (int k = tid; k <= j; k += nt) {
        double2 acc = v.bv[k];
        for (int i = k > 0 ? k - 1 : 0; i < j; ++i) acc = cvk_sub(acc, cvk_mul(v.Hu[k * M + i], v.av[i]));
        v.Hu[k * M + j] = cvk_divr(acc, nu);
    }
    for (int q = tid; q < j; q += nt) v.ev[q] = cvk_sub(v.bv[q], cvk_mul(v.av[q], v.ev[j]));
    if (j > 0 && tid == 0) gm_rotate(v, j - 1, v.Hu[j * M + j - 1].x, v.gpre[j - 1]);
    sync();
    return nu;
}

// one thread: the provisional subdiagonal and rotation of column j
__device__ __forceinline__ void gm_provisional(const GmView& v, int j, double hn, double nu) {
    v.Hu[(j + 1) * v.M + j] = make_double2(hn / nu, 0.0);
    v.gpre[j] = v.g[j];
    gm_rotate(v, j, hn / nu, v.gpre[j]);
}

// one thread: back substitution R(0:k, 0:k) y = g(0:k)
__device__ __forceinline__ void gm_back_subst(const GmView& v, int k, double2* y) {
    const int M = v.M;
    for (int i = k; i-- > 0;) {
        double2 s = v.g[i];
        for (int q = i + 1; q < k; ++q) s = cvk_sub(s, cvk_mul(v.R[i * M + q], y[q]));
        y[i] = cvk_cdiv(s, v.R[i * M + i]);
    }
}

// the per-row update of the pass: returns u', stores q_j over u_j
template <class VAt>
__device__ __forceinline__ double2 gm_update_row(const double2* av, const double2* ev, int j, double nu,
                                                 double2& uj, double2 wi, VAt&& vat) {
    const double2 u = uj;
    double2 qv = u, up = wi;
    for (int q = 0; q < j; ++q) {
        const double2 vq = vat(q);
        qv = cvk_sub(qv, cvk_mul(av[q], vq));
        up = cvk_sub(up, cvk_mul(ev[q], vq));
    }
    up = cvk_sub(up, cvk_mul(ev[j], u));
    uj = cvk_divr(qv, nu);
    return up;
}

}  // namespace cvk
