/*
 * na2d_oracle.c -- plain, slow, fp64 CPU oracle for 2D Neighborhood Attention.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.  It shares no code,
 * header, table or constant with the CUDA path (paper_2204_07143_b200/), and the
 * CUDA path never calls it.
 *
 * Every function follows the paper (arXiv 2204.07143, /root/reference/PAPER.md,
 * cited as P:<line>) step by step, with loops in the paper's order and no
 * blocking, fusion or reordering:
 *
 *   rho(i,j)   P:150 (Sec. 3.1) "fixed-length set of indices of pixels nearest to (i,j)",
 *              P:163-164 corner expansion ("the neighborhood is expanded to maintain
 *              receptive field size"), P:438 (App. A: unfold + replicated padding,
 *              odd L > 1).  Realised per axis as start = clamp(i - (L-1)/2, 0, n - L);
 *              if L >= n the window is the whole axis.
 *   Eq. 2      P:152 NA(X_ij) = softmax((Q_ij K_rho^T + B_ij) / scale) V_rho.
 *              "/scale" with scale = sqrt(d) (Eq. 1) is passed in as the
 *              multiplier inv_scale = 1/sqrt(d); the bias sits INSIDE the scaling
 *              (reading R1).
 *   B_ij       P:156 relative positional bias, table [heads][2L-1][2L-1], index
 *              (p - i + L - 1, q - j + L - 1) = key minus query (reading R4).
 *   softmax    max-subtracted; LSE = m + log(sum exp(s - m)) (reading R6).
 *   backward   the analytic gradient of Eq. 2 (paper silent, reading R5):
 *              D = dO.O, dP_m = dO.v_m, dS_m = P_m (dP_m - D),
 *              dQ += inv_scale dS_m k_m, dK_m += inv_scale dS_m q, dV_m += P_m dO,
 *              dB[cell(m)] += inv_scale dS_m.
 *
 * Row bands (for the multi-GPU row-band split): a call may cover only
 * query rows [q_row0, q_row0+q_rows) of a map of height H, with K/V supplied for rows
 * [kv_row0, kv_row0+kv_rows).  All geometry uses global coordinates.  In the backward
 * pass dK/dV (and dB) receive contributions only from the supplied query rows.  The
 * whole-map call is the special case q_row0 = kv_row0 = 0, q_rows = kv_rows = H.
 *
 * Layouts (row-major, C order):
 *   q, out, dout, dq : [B][heads][q_rows][W][d]
 *   k, v, dk, dv     : [B][heads][kv_rows][W][d]
 *   lse              : [B][heads][q_rows][W]
 *   rpb, drpb        : [heads][2L-1][2L-1]   (rpb may be NULL: B = 0, Table 7 "no RPB")
 *
 * Parallelism: std pthreads over independent (b, h) units; every unit writes its own
 * slices, dB is accumulated per unit and merged over b in index order, so results are
 * bitwise independent of the thread count.
 *
 * Return codes: 0 ok, 1 bad argument (even/small L, bad dims), 2 band does not supply a
 * needed K/V row, 3 non-finite logits ("non-finite input -> numeric error").
 */
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ---- geometry: rho(i, j), P:150, P:163-164, P:438 ------------------------------------ */

int na2d_oracle_window_start(int i, int n, int L) {
    if (L >= n) return 0;              /* window covers the whole axis */
    int s = i - (L - 1) / 2;           /* centred window ((L-1)/2 pixels each side) */
    if (s < 0) s = 0;                  /* corner expansion: shift, never shrink */
    if (s > n - L) s = n - L;
    return s;
}

int na2d_oracle_window_len(int n, int L) { return L < n ? L : n; }

/* relative-position index along one axis: key minus query + L - 1 */
int na2d_oracle_rel_index(int i, int p, int L) { return p - i + L - 1; }

typedef struct {
    int B, heads, H, W, d, L;
    double inv_scale;
    int q_row0, q_rows, kv_row0, kv_rows;
    const double *q, *k, *v, *rpb, *dout;
    double *out, *lse, *dq, *dk, *dv, *drpb_units; /* drpb_units: [B*heads][T*T] */
    int backward;
    int status; /* per-run error flag (set by any worker, read after join) */
    int next_unit;
    pthread_mutex_t lock;
} job_t;

static int check_args(int B, int heads, int H, int W, int d, int L, int q_row0, int q_rows,
                      int kv_row0, int kv_rows) {
    if (B <= 0 || heads <= 0 || H <= 0 || W <= 0 || d <= 0) return 1;
    if (L < 3 || (L % 2) == 0) return 1; /* P:438 "odd number greater than 1", P:140 minimum 3x3 */
    if (q_row0 < 0 || q_rows <= 0 || q_row0 + q_rows > H) return 1;
    if (kv_row0 < 0 || kv_rows <= 0 || kv_row0 + kv_rows > H) return 1;
    /* every query row's window must lie inside the supplied K/V rows */
    for (int i = q_row0; i < q_row0 + q_rows; ++i) {
        int s = na2d_oracle_window_start(i, H, L), n = na2d_oracle_window_len(H, L);
        if (s < kv_row0 || s + n > kv_row0 + kv_rows) return 2;
    }
    return 0;
}

/* One (b, h) unit: loops exactly as Eq. 2 reads, one query at a time. */
static int run_unit(job_t *J, int unit) {
    const int W = J->W, d = J->d, L = J->L, T = 2 * L - 1;
    const int h = unit % J->heads;
    const size_t qplane = (size_t)J->q_rows * W * d, kvplane = (size_t)J->kv_rows * W * d;
    const double *Q = J->q + (size_t)unit * qplane;
    const double *K = J->k + (size_t)unit * kvplane;
    const double *V = J->v + (size_t)unit * kvplane;
    const double *Bt = J->rpb ? J->rpb + (size_t)h * T * T : NULL;
    const int Lh = na2d_oracle_window_len(J->H, L), Lw = na2d_oracle_window_len(W, L);
    const int nb = Lh * Lw; /* |rho| = min(L,H) min(L,W) */
    double *s = (double *)malloc(sizeof(double) * nb);
    double *P = (double *)malloc(sizeof(double) * nb);
    double *o = (double *)malloc(sizeof(double) * d);
    double *dS = (double *)malloc(sizeof(double) * nb);
    int rc = 0;
    for (int i = J->q_row0; i < J->q_row0 + J->q_rows && !rc; ++i) {
        const int si = na2d_oracle_window_start(i, J->H, L);
        for (int j = 0; j < W; ++j) {
            const int sj = na2d_oracle_window_start(j, W, L);
            const double *qv = Q + ((size_t)(i - J->q_row0) * W + j) * d;
            /* logits s_m = inv_scale * (q . k_m + B[cell]), m in row-major window order */
            int m = 0;
            for (int p = si; p < si + Lh; ++p)
                for (int qq = sj; qq < sj + Lw; ++qq, ++m) {
                    const double *kv = K + ((size_t)(p - J->kv_row0) * W + qq) * d;
                    double dot = 0.0;
                    for (int c = 0; c < d; ++c) dot += qv[c] * kv[c];
                    double bias = 0.0;
                    if (Bt) bias = Bt[na2d_oracle_rel_index(i, p, L) * T + na2d_oracle_rel_index(j, qq, L)];
                    s[m] = J->inv_scale * (dot + bias);
                }
            /* softmax with max subtraction */
            double mx = -INFINITY;
            for (m = 0; m < nb; ++m) mx = s[m] > mx ? s[m] : mx;
            if (!isfinite(mx)) { rc = 3; break; }
            double sum = 0.0;
            for (m = 0; m < nb; ++m) { P[m] = exp(s[m] - mx); sum += P[m]; }
            for (m = 0; m < nb; ++m) P[m] /= sum;
            /* AV */
            for (int c = 0; c < d; ++c) o[c] = 0.0;
            m = 0;
            for (int p = si; p < si + Lh; ++p)
                for (int qq = sj; qq < sj + Lw; ++qq, ++m) {
                    const double *vv = V + ((size_t)(p - J->kv_row0) * W + qq) * d;
                    for (int c = 0; c < d; ++c) o[c] += P[m] * vv[c];
                }
            const size_t qi = (size_t)unit * J->q_rows * W + (size_t)(i - J->q_row0) * W + j;
            if (J->out) for (int c = 0; c < d; ++c) J->out[qi * d + c] = o[c];
            if (J->lse) J->lse[qi] = mx + log(sum);
            if (!J->backward) continue;
            /* ---- backward of Eq. 2 (reading R5) ---- */
            const double *dO = J->dout + qi * d;
            double D = 0.0;
            for (int c = 0; c < d; ++c) D += dO[c] * o[c];
            m = 0;
            for (int p = si; p < si + Lh; ++p)
                for (int qq = sj; qq < sj + Lw; ++qq, ++m) {
                    const double *vv = V + ((size_t)(p - J->kv_row0) * W + qq) * d;
                    double dP = 0.0;
                    for (int c = 0; c < d; ++c) dP += dO[c] * vv[c];
                    dS[m] = P[m] * (dP - D);
                }
            double *dq = J->dq + qi * d;
            for (int c = 0; c < d; ++c) dq[c] = 0.0;
            double *dB = J->drpb_units + (size_t)unit * T * T;
            m = 0;
            for (int p = si; p < si + Lh; ++p)
                for (int qq = sj; qq < sj + Lw; ++qq, ++m) {
                    const size_t ki = (size_t)unit * J->kv_rows * W + (size_t)(p - J->kv_row0) * W + qq;
                    const double *kv = K + ((size_t)(p - J->kv_row0) * W + qq) * d;
                    double *dk = J->dk + ki * d, *dv = J->dv + ki * d;
                    for (int c = 0; c < d; ++c) {
                        dq[c] += J->inv_scale * dS[m] * kv[c];
                        dk[c] += J->inv_scale * dS[m] * qv[c];
                        dv[c] += P[m] * dO[c];
                    }
                    dB[na2d_oracle_rel_index(i, p, L) * T + na2d_oracle_rel_index(j, qq, L)] +=
                        J->inv_scale * dS[m];
                }
        }
    }
    free(s); free(P); free(o); free(dS);
    return rc;
}

static void *worker(void *arg) {
    job_t *J = (job_t *)arg;
    for (;;) {
        pthread_mutex_lock(&J->lock);
        int u = J->next_unit++;
        pthread_mutex_unlock(&J->lock);
        if (u >= J->B * J->heads) break;
        int rc = run_unit(J, u);
        if (rc) { pthread_mutex_lock(&J->lock); J->status = rc; pthread_mutex_unlock(&J->lock); }
    }
    return NULL;
}

static int run_job(job_t *J, int nthreads) {
    const int units = J->B * J->heads;
    if (nthreads <= 0) nthreads = 1;
    if (nthreads > units) nthreads = units;
    pthread_mutex_init(&J->lock, NULL);
    J->next_unit = 0;
    J->status = 0;
    pthread_t *t = (pthread_t *)malloc(sizeof(pthread_t) * nthreads);
    for (int i = 0; i < nthreads; ++i) pthread_create(&t[i], NULL, worker, J);
    for (int i = 0; i < nthreads; ++i) pthread_join(t[i], NULL);
    free(t);
    pthread_mutex_destroy(&J->lock);
    return J->status;
}

/* Forward of Eq. 2 over a (band of a) map.  out and/or lse may be NULL. */
int na2d_oracle_forward_band(int B, int heads, int H, int W, int d, int L, double inv_scale,
                             int q_row0, int q_rows, int kv_row0, int kv_rows,
                             const double *q, const double *k, const double *v, const double *rpb,
                             double *out, double *lse, int nthreads) {
    int rc = check_args(B, heads, H, W, d, L, q_row0, q_rows, kv_row0, kv_rows);
    if (rc) return rc;
    job_t J;
    memset(&J, 0, sizeof J);
    J.B = B; J.heads = heads; J.H = H; J.W = W; J.d = d; J.L = L; J.inv_scale = inv_scale;
    J.q_row0 = q_row0; J.q_rows = q_rows; J.kv_row0 = kv_row0; J.kv_rows = kv_rows;
    J.q = q; J.k = k; J.v = v; J.rpb = rpb; J.out = out; J.lse = lse;
    return run_job(&J, nthreads);
}

int na2d_oracle_forward(int B, int heads, int H, int W, int d, int L, double inv_scale,
                        const double *q, const double *k, const double *v, const double *rpb,
                        double *out, double *lse, int nthreads) {
    return na2d_oracle_forward_band(B, heads, H, W, d, L, inv_scale, 0, H, 0, H, q, k, v, rpb, out,
                                    lse, nthreads);
}

/* Backward of Eq. 2.  Recomputes the forward in fp64 (out/lse optional outputs).  dq is
 * overwritten; dk, dv are overwritten (zeroed first) with contributions of the supplied
 * query rows only; drpb (may be NULL iff rpb is NULL) is overwritten with the sum over
 * b in index order of the per-unit partials. */
int na2d_oracle_backward_band(int B, int heads, int H, int W, int d, int L, double inv_scale,
                              int q_row0, int q_rows, int kv_row0, int kv_rows,
                              const double *q, const double *k, const double *v, const double *rpb,
                              const double *dout, double *out, double *lse, double *dq, double *dk,
                              double *dv, double *drpb, int nthreads) {
    int rc = check_args(B, heads, H, W, d, L, q_row0, q_rows, kv_row0, kv_rows);
    if (rc) return rc;
    const int T = 2 * L - 1;
    const size_t kvn = (size_t)B * heads * kv_rows * W * d;
    memset(dk, 0, kvn * sizeof(double));
    memset(dv, 0, kvn * sizeof(double));
    double *dBu = (double *)calloc((size_t)B * heads * T * T, sizeof(double));
    job_t J;
    memset(&J, 0, sizeof J);
    J.B = B; J.heads = heads; J.H = H; J.W = W; J.d = d; J.L = L; J.inv_scale = inv_scale;
    J.q_row0 = q_row0; J.q_rows = q_rows; J.kv_row0 = kv_row0; J.kv_rows = kv_rows;
    J.q = q; J.k = k; J.v = v; J.rpb = rpb; J.dout = dout;
    J.out = out; J.lse = lse; J.dq = dq; J.dk = dk; J.dv = dv; J.drpb_units = dBu;
    J.backward = 1;
    rc = run_job(&J, nthreads);
    if (!rc && drpb) {
        memset(drpb, 0, (size_t)heads * T * T * sizeof(double));
        for (int b = 0; b < B; ++b)
            for (int h = 0; h < heads; ++h)
                for (int c = 0; c < T * T; ++c)
                    drpb[(size_t)h * T * T + c] += dBu[((size_t)b * heads + h) * T * T + c];
    }
    free(dBu);
    return rc;
}

int na2d_oracle_backward(int B, int heads, int H, int W, int d, int L, double inv_scale,
                         const double *q, const double *k, const double *v, const double *rpb,
                         const double *dout, double *out, double *lse, double *dq, double *dk,
                         double *dv, double *drpb, int nthreads) {
    return na2d_oracle_backward_band(B, heads, H, W, d, L, inv_scale, 0, H, 0, H, q, k, v, rpb, dout,
                                     out, lse, dq, dk, dv, drpb, nthreads);
}
