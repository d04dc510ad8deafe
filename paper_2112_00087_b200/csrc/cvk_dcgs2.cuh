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
#include "cvk_engine.cuh"

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
    double2* yv;    // M + 1: least-squares solution of the cycle
    double* nu;     // 1
    int M;
};

// Givens rotation of column col: R[.][col] = Hu[.][col] rotated by 0..col-1,
// then the rotation that annihilates the subdiagonal hsub; g from gp.
// The running entry a0 is carried in registers (through memory every
// iteration paid a store-to-load round trip: the dependent chain of the
// last-CTA scalar step was ~15 us at j = 14 on the B200).
__device__ __forceinline__ void gm_rotate(const GmView& v, int col, double hsub, double2 gp) {
    const int M = v.M;
    double2 a0 = v.Hu[col];
    for (int i = 0; i < col; ++i) {
        const double2 c2 = v.Hu[(i + 1) * M + col];
        const double ci = v.cs[i];
        const double2 si = v.sn[i];
        v.R[i * M + col] = cvk_add(cvk_scale(ci, a0), cvk_mul(si, c2));
        a0 = cvk_add(cvk_mul(cvk_neg(cvk_conj(si)), a0), cvk_scale(ci, c2));
    }
    v.R[col * M + col] = a0;
    const double2 aj = a0;
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

// FAST dot passes form canonical groups: the rows r0 + l + 32 e (e = 0..3)
// of every 128-row-aligned sub-block [r0, r0 + 128), l = 0..31.  A group's
// terms (zero past n) are summed in plain FP64 as (t0 + t1) + (t2 + t3) and
// only the group sums enter the double-double accumulators: a quarter of the
// double-double work per row and short dependency chains (the row-by-row
// double-double pass was FP64-latency-bound at 2.2 TB/s).  Every GMRES FAST
// path forms the same groups, so their scalars agree bit for bit whatever
// the CTA count or the tiling.
__device__ __forceinline__ double2 gm_tree4(const double2 (&t)[4]) {
    return cvk_add(cvk_add(t[0], t[1]), cvk_add(t[2], t[3]));
}

// one group: <v, u> and <v, w> terms of the lane's four rows (nr valid)
__device__ __forceinline__ void gm_group4(const double2 (&v)[4], const double2 (&u)[4], const double2 (&w)[4],
                                          int nr, CAcc (&acc)[2]) {
    double2 ta[4], tb[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        ta[e] = e < nr ? cvk_cmul(v[e], u[e]) : make_double2(0.0, 0.0);
        tb[e] = e < nr ? cvk_cmul(v[e], w[e]) : make_double2(0.0, 0.0);
    }
    const double2 pa = gm_tree4(ta), pb = gm_tree4(tb);
    dd_add1(acc[0].hi.x, acc[0].lo.x, pa.x);
    dd_add1(acc[0].hi.y, acc[0].lo.y, pa.y);
    dd_add1(acc[1].hi.x, acc[1].lo.x, pb.x);
    dd_add1(acc[1].hi.y, acc[1].lo.y, pb.y);
}

// rows of the lane's group in a sub-block with `rows` rows: e < nr valid
__device__ __forceinline__ int gm_group_rows(int rows, int lane) {
    return rows > lane ? min(4, (rows - lane + 31) / 32) : 0;
}

// one 128-row sub-block (its first `rows` rows valid) from pointers to its
// first row; NQ basis vectors at a time (the first nq valid), their loads
// issued together
template <int NQ>
__device__ __forceinline__ void gm_group_dots(const double2* const (&vq)[NQ], int nq, const double2* u,
                                              const double2* w, int rows, int lane, CAcc (&acc)[NQ][2]) {
    const int nr = gm_group_rows(rows, lane);
    double2 vv[NQ][4], uu[4], ww[4];
#pragma unroll
    for (int e = 0; e < 4; ++e)
        if (e < nr) {
            const int row = lane + 32 * e;
            uu[e] = u[row];
            ww[e] = w[row];
#pragma unroll
            for (int k = 0; k < NQ; ++k)
                if (k < nq) vv[k][e] = vq[k][row];
        }
#pragma unroll
    for (int k = 0; k < NQ; ++k)
        if (k < nq) gm_group4(vv[k], uu, ww, nr, acc[k]);
}

}  // namespace cvk
