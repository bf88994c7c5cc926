/*
 * fwi_oracle.c — TEST INFRASTRUCTURE ONLY: a plain-C restatement of the
 * reference's KKT/Krylov hot path, written from the reference's algorithm
 * (paths relative to /root/reference/proj) and used only as the checker.
 *
 * Every function keeps the reference's operation order, so its results are
 * bit-identical to the reference compiled with g++ on x86-64 (no FMA): complex
 * products (ac-bd, ad+bc), libgcc __divdc3 division, mixed real*complex
 * products component-wise, sequential sums. tests/test_oracle.py pins this
 * file against oracle/_ref (the unmodified reference core) and the committed
 * golden vectors (tests/golden/).
 */
#define _POSIX_C_SOURCE 199309L
#include "fwi_oracle.h"

#include <complex.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

typedef double _Complex cplx;

static _Thread_local char g_err[512];
static _Thread_local int g_err_index = -1;

static int fail(int code, int idx, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    g_err_index = idx;
    return code;
}

const char* orc_last_error(void) { return g_err; }
int orc_last_error_index(void) { return g_err_index; }

/* growable (int, cplx) list */
typedef struct {
    int n, cap;
    int* key;
    cplx* val;
} plist;

static void pl_push(plist* l, int k, cplx v) {
    if (l->n == l->cap) {
        l->cap = l->cap ? 2 * l->cap : 8;
        l->key = realloc(l->key, sizeof(int) * l->cap);
        l->val = realloc(l->val, sizeof(cplx) * l->cap);
    }
    l->key[l->n] = k;
    l->val[l->n] = v;
    l->n++;
}

static void pl_free(plist* l) {
    free(l->key);
    free(l->val);
}

/* sort a plist by key (keys unique) — insertion sort keeps it simple */
static void pl_sort(plist* l) {
    for (int i = 1; i < l->n; ++i) {
        int k = l->key[i];
        cplx v = l->val[i];
        int j = i - 1;
        while (j >= 0 && l->key[j] > k) {
            l->key[j + 1] = l->key[j];
            l->val[j + 1] = l->val[j];
            --j;
        }
        l->key[j + 1] = k;
        l->val[j + 1] = v;
    }
}

typedef struct {
    int n;
    int *lp, *li;
    cplx* lv; /* L strictly lower, CSC, rows in pivot numbering */
    int *up, *ui;
    cplx* uv; /* U CSC, diagonal last */
    int* perm;
    long long count;
} lu_t;

typedef struct {
    int n, level;
    int *lp, *li, *up, *ui, *ltp, *lti, *utp, *uti;
    cplx *lv, *uv, *ltv, *utv;
    long long count;
} ilu_t;

struct orc_state {
    int nx, nz, n, npml, K, ndata, drop;
    double h, sigma_max, power, freq, omega, eps;
    double* s;
    int *rp, *ci; /* assembled A, CSR */
    cplx* av;
    int nnz;
    cplx *u, *r, *dpred;
    double* w;
    int *off, *node, *src_node;
    double* src_amp;
    lu_t* lu;
    ilu_t* ilu;
};

/* ---------------------------------------------------------------- grid */
/* stretch, src/grid.cpp:35-48 */
static cplx stretch(int n_axis, int npml, double sigma_max, double power, double pos, double omega) {
    if (npml == 0) return 1.0;
    const double a = npml - pos, b = pos - (n_axis - 1 - npml);
    const double depth = (a < b) ? b : a; /* std::max */
    if (depth <= 0.0) return 1.0;
    const double t = depth / npml;
    return CMPLX(1.0, sigma_max * pow(t, power) / omega);
}

static int on_bnd(const orc_state* s, int ix, int iz) {
    return ix == 0 || iz == 0 || ix == s->nx - 1 || iz == s->nz - 1;
}

/* assemble_helmholtz, src/helmholtz.cpp:17-70 (CSR rows in ascending column
 * order with 0 + value, as SparseMatrixCSR::from_triplets stores them) */
static void assemble(orc_state* s) {
    const int nx = s->nx, nz = s->nz, n = s->n;
    const double h2 = s->h * s->h, w2 = s->omega * s->omega;
    s->rp = calloc(n + 1, sizeof(int));
    s->ci = malloc(sizeof(int) * 5 * (size_t)n);
    s->av = malloc(sizeof(cplx) * 5 * (size_t)n);
    int q = 0;
    for (int iz = 0; iz < nz; ++iz)
        for (int ix = 0; ix < nx; ++ix) {
            const int node = iz * nx + ix;
            if (on_bnd(s, ix, iz)) {
                cplx v = 0;
                v += 1.0;
                s->ci[q] = node;
                s->av[q++] = v;
                s->rp[node + 1] = q;
                continue;
            }
            const cplx xi = stretch(nx, s->npml, s->sigma_max, s->power, ix, s->omega);
            const cplx xp = stretch(nx, s->npml, s->sigma_max, s->power, ix + 0.5, s->omega);
            const cplx xm = stretch(nx, s->npml, s->sigma_max, s->power, ix - 0.5, s->omega);
            const cplx zj = stretch(nz, s->npml, s->sigma_max, s->power, iz, s->omega);
            const cplx zp = stretch(nz, s->npml, s->sigma_max, s->power, iz + 0.5, s->omega);
            const cplx zm = stretch(nz, s->npml, s->sigma_max, s->power, iz - 0.5, s->omega);
            const cplx cxp = zj / (h2 * xp);
            const cplx cxm = zj / (h2 * xm);
            const cplx czp = xi / (h2 * zp);
            const cplx czm = xi / (h2 * zm);
            const cplx diag = cxp + cxm + czp + czm - w2 * s->s[node] * xi * zj;
            int cols[5];
            cplx vals[5];
            int m = 0;
            if (!on_bnd(s, ix, iz - 1)) { cols[m] = node - nx; vals[m++] = -czm; }
            if (!on_bnd(s, ix - 1, iz)) { cols[m] = node - 1; vals[m++] = -cxm; }
            cols[m] = node;
            vals[m++] = diag;
            if (!on_bnd(s, ix + 1, iz)) { cols[m] = node + 1; vals[m++] = -cxp; }
            if (!on_bnd(s, ix, iz + 1)) { cols[m] = node + nx; vals[m++] = -czp; }
            for (int t = 0; t < m; ++t) {
                cplx v = 0;
                v += vals[t];
                s->ci[q] = cols[t];
                s->av[q++] = v;
            }
            s->rp[node + 1] = q;
        }
    s->nnz = q;
}

/* spmv, src/sparse.cpp:69-91 */
static void spmv(const orc_state* s, const cplx* x, cplx* y, int adjoint) {
    const int n = s->n;
    if (!adjoint) {
        for (int i = 0; i < n; ++i) {
            cplx acc = 0;
            for (int k = s->rp[i]; k < s->rp[i + 1]; ++k) acc += s->av[k] * x[s->ci[k]];
            y[i] = acc;
        }
        return;
    }
    for (int i = 0; i < n; ++i) y[i] = 0;
    for (int i = 0; i < n; ++i) {
        const cplx xi = x[i];
        for (int k = s->rp[i]; k < s->rp[i + 1]; ++k) y[s->ci[k]] += conj(s->av[k]) * xi;
    }
}

/* ---------------------------------------------------------------- LU */
/* LuFactors::factor, src/lu.cpp:37-166: left-looking Gilbert-Peierls with a
 * depth-first reach per column, partial pivoting by magnitude, natural order */
static int lu_factor(const orc_state* s, lu_t** out) {
    const int n = s->n;
    /* CSC of A (rows ascending per column) */
    int* cp = calloc(n + 1, sizeof(int));
    int* cr = malloc(sizeof(int) * s->nnz);
    cplx* cv = malloc(sizeof(cplx) * s->nnz);
    for (int k = 0; k < s->nnz; ++k) cp[s->ci[k] + 1]++;
    for (int j = 0; j < n; ++j) cp[j + 1] += cp[j];
    int* nxt = malloc(sizeof(int) * n);
    memcpy(nxt, cp, sizeof(int) * n);
    for (int i = 0; i < n; ++i)
        for (int k = s->rp[i]; k < s->rp[i + 1]; ++k) {
            const int p = nxt[s->ci[k]]++;
            cr[p] = i;
            cv[p] = s->av[k];
        }
    plist* lcols = calloc(n, sizeof(plist));
    plist* ucols = calloc(n, sizeof(plist));
    int* pinv = malloc(sizeof(int) * n);
    int* visited = malloc(sizeof(int) * n);
    int* cpos = malloc(sizeof(int) * n);
    int* stack = malloc(sizeof(int) * n);
    int* pat = malloc(sizeof(int) * n);
    int* perm = malloc(sizeof(int) * n);
    cplx* x = calloc(n, sizeof(cplx));
    for (int i = 0; i < n; ++i) { pinv[i] = -1; visited[i] = -1; }
    int rc = FWI_OK;
    for (int j = 0; j < n && rc == FWI_OK; ++j) {
        int np = 0;
        for (int p = cp[j]; p < cp[j + 1]; ++p) {
            const int start = cr[p];
            if (visited[start] == j) continue;
            int head = 0;
            stack[0] = start;
            visited[start] = j;
            cpos[start] = 0;
            while (head >= 0) {
                const int t = stack[head];
                const int k = pinv[t];
                int descended = 0;
                if (k >= 0) {
                    const plist* col = &lcols[k];
                    while (cpos[t] < col->n) {
                        const int child = col->key[cpos[t]++];
                        if (visited[child] != j) {
                            visited[child] = j;
                            cpos[child] = 0;
                            stack[++head] = child;
                            descended = 1;
                            break;
                        }
                    }
                }
                if (!descended) {
                    pat[np++] = t;
                    --head;
                }
            }
        }
        for (int p = cp[j]; p < cp[j + 1]; ++p) x[cr[p]] = cv[p];
        for (int q = np - 1; q >= 0; --q) { /* reverse postorder */
            const int i = pat[q];
            const int k = pinv[i];
            if (k < 0) continue;
            const cplx xi = x[i];
            if (xi == 0.0) continue;
            const plist* col = &lcols[k];
            for (int t = 0; t < col->n; ++t) x[col->key[t]] -= col->val[t] * xi;
        }
        int ip = -1;
        double best = -1.0;
        for (int q = 0; q < np; ++q) {
            const int t = pat[q];
            if (pinv[t] >= 0) continue;
            const double m = cabs(x[t]);
            if (m > best) { best = m; ip = t; }
        }
        if (ip < 0 || best == 0.0) {
            rc = fail(FWI_ERR_SINGULAR_PIVOT, j, "LU: singular pivot at elimination step %d", j);
            break;
        }
        const cplx piv = x[ip];
        for (int q = 0; q < np; ++q) {
            const int t = pat[q];
            if (pinv[t] >= 0) pl_push(&ucols[j], pinv[t], x[t]);
        }
        pl_sort(&ucols[j]);
        pl_push(&ucols[j], j, piv);
        for (int q = 0; q < np; ++q) {
            const int t = pat[q];
            if (pinv[t] < 0 && t != ip && x[t] != 0.0) pl_push(&lcols[j], t, x[t] / piv);
        }
        pinv[ip] = j;
        perm[j] = ip;
        for (int q = 0; q < np; ++q) x[pat[q]] = 0;
    }
    lu_t* f = NULL;
    if (rc == FWI_OK) {
        f = calloc(1, sizeof(lu_t));
        f->n = n;
        f->perm = perm;
        perm = NULL;
        f->lp = calloc(n + 1, sizeof(int));
        f->up = calloc(n + 1, sizeof(int));
        for (int j = 0; j < n; ++j) {
            f->lp[j + 1] = f->lp[j] + lcols[j].n;
            f->up[j + 1] = f->up[j] + ucols[j].n;
        }
        f->li = malloc(sizeof(int) * (f->lp[n] + 1));
        f->lv = malloc(sizeof(cplx) * (f->lp[n] + 1));
        f->ui = malloc(sizeof(int) * (f->up[n] + 1));
        f->uv = malloc(sizeof(cplx) * (f->up[n] + 1));
        for (int j = 0; j < n; ++j) {
            plist* l = &lcols[j];
            for (int t = 0; t < l->n; ++t) l->key[t] = pinv[l->key[t]];
            pl_sort(l);
            memcpy(f->li + f->lp[j], l->key, sizeof(int) * l->n);
            memcpy(f->lv + f->lp[j], l->val, sizeof(cplx) * l->n);
            memcpy(f->ui + f->up[j], ucols[j].key, sizeof(int) * ucols[j].n);
            memcpy(f->uv + f->up[j], ucols[j].val, sizeof(cplx) * ucols[j].n);
        }
    }
    for (int j = 0; j < n; ++j) { pl_free(&lcols[j]); pl_free(&ucols[j]); }
    free(lcols); free(ucols); free(pinv); free(visited); free(cpos); free(stack); free(pat);
    free(perm); free(x); free(cp); free(cr); free(cv); free(nxt);
    *out = f;
    return rc;
}

static void lu_free(lu_t* f) {
    if (!f) return;
    free(f->lp); free(f->li); free(f->lv); free(f->up); free(f->ui); free(f->uv); free(f->perm);
    free(f);
}

/* LuFactors::solve, src/lu.cpp:168-209 */
static void lu_solve(lu_t* f, const cplx* b, cplx* out, int adjoint) {
    const int n = f->n;
    f->count++;
    if (!adjoint) {
        cplx* x = out;
        for (int k = 0; k < n; ++k) x[k] = b[f->perm[k]];
        for (int k = 0; k < n; ++k) {
            const cplx xk = x[k];
            if (xk == 0.0) continue;
            for (int p = f->lp[k]; p < f->lp[k + 1]; ++p) x[f->li[p]] -= f->lv[p] * xk;
        }
        for (int j = n - 1; j >= 0; --j) {
            const int dp = f->up[j + 1] - 1;
            x[j] /= f->uv[dp];
            const cplx xj = x[j];
            if (xj == 0.0) continue;
            for (int p = f->up[j]; p < dp; ++p) x[f->ui[p]] -= f->uv[p] * xj;
        }
        return;
    }
    cplx* z = malloc(sizeof(cplx) * n);
    for (int j = 0; j < n; ++j) {
        cplx s = b[j];
        const int dp = f->up[j + 1] - 1;
        for (int p = f->up[j]; p < dp; ++p) s -= conj(f->uv[p]) * z[f->ui[p]];
        z[j] = s / conj(f->uv[dp]);
    }
    for (int j = n - 1; j >= 0; --j) {
        cplx s = z[j];
        for (int p = f->lp[j]; p < f->lp[j + 1]; ++p) s -= conj(f->lv[p]) * z[f->li[p]];
        z[j] = s;
    }
    for (int k = 0; k < n; ++k) out[f->perm[k]] = z[k];
    free(z);
}

/* ---------------------------------------------------------------- ILU */
static void transpose(int n, const int* p, const int* idx, const cplx* val, int** tp, int** ti,
                      cplx** tv) {
    const int nnz = p[n];
    *tp = calloc(n + 1, sizeof(int));
    *ti = malloc(sizeof(int) * (nnz + 1));
    *tv = malloc(sizeof(cplx) * (nnz + 1));
    for (int q = 0; q < nnz; ++q) (*tp)[idx[q] + 1]++;
    for (int j = 0; j < n; ++j) (*tp)[j + 1] += (*tp)[j];
    int* nx = malloc(sizeof(int) * (n + 1));
    memcpy(nx, *tp, sizeof(int) * n);
    for (int i = 0; i < n; ++i)
        for (int q = p[i]; q < p[i + 1]; ++q) {
            const int t = nx[idx[q]]++;
            (*ti)[t] = i;
            (*tv)[t] = val[q];
        }
    free(nx);
}

/* IluFactors::factor, src/ilu.cpp:8-106 */
static int ilu_factor(const orc_state* s, int level, double shift, ilu_t** out) {
    const int n = s->n;
    if (level < 0) return fail(FWI_ERR_INVALID_ARGUMENT, -1, "IluFactors::factor: fill level must be >= 0");
    int* lev = malloc(sizeof(int) * n);
    int* mark = malloc(sizeof(int) * n);
    int** pat = calloc(n, sizeof(int*)); /* full row pattern, ascending */
    int* npat = calloc(n, sizeof(int));
    int** ulv = calloc(n, sizeof(int*)); /* levels of the strict-upper entries */
    int* diagpos = malloc(sizeof(int) * n);
    for (int i = 0; i < n; ++i) mark[i] = -1;
    int rc = FWI_OK;
    /* symbolic: entries of row i start at level 0; pivot rows j < i are taken
     * in ascending order and fill (i,k) via j gets lev(i,j)+lev(j,k)+1 */
    for (int i = 0; i < n && rc == FWI_OK; ++i) {
        int lo = i, hi = i, has_diag = 0;
        for (int p = s->rp[i]; p < s->rp[i + 1]; ++p) {
            const int c = s->ci[p];
            mark[c] = i;
            lev[c] = 0;
            if (c < lo) lo = c;
            if (c > hi) hi = c;
            if (c == i) has_diag = 1;
        }
        if (!has_diag) {
            rc = fail(FWI_ERR_INVALID_ARGUMENT, -1, "IluFactors::factor: missing diagonal at row %d", i);
            break;
        }
        for (int j = lo; j < i; ++j) {
            if (mark[j] != i) continue;
            const int lj = lev[j];
            for (int q = diagpos[j] + 1; q < npat[j]; ++q) {
                const int k = pat[j][q];
                const int nl = lj + ulv[j][q - diagpos[j] - 1] + 1;
                if (nl > level) continue;
                if (mark[k] != i) {
                    mark[k] = i;
                    lev[k] = nl;
                    if (k > hi) hi = k;
                } else if (nl < lev[k]) {
                    lev[k] = nl;
                }
            }
        }
        int cnt = 0;
        for (int c = lo; c <= hi; ++c) cnt += mark[c] == i;
        pat[i] = malloc(sizeof(int) * cnt);
        npat[i] = cnt;
        int m = 0, nup = 0;
        for (int c = lo; c <= hi; ++c)
            if (mark[c] == i) {
                if (c == i) diagpos[i] = m;
                if (c > i) nup++;
                pat[i][m++] = c;
            }
        ulv[i] = malloc(sizeof(int) * (nup + 1));
        for (int q = diagpos[i] + 1; q < cnt; ++q) ulv[i][q - diagpos[i] - 1] = lev[pat[i][q]];
    }
    ilu_t* f = NULL;
    if (rc == FWI_OK) {
        f = calloc(1, sizeof(ilu_t));
        f->n = n;
        f->level = level;
        f->lp = calloc(n + 1, sizeof(int));
        f->up = calloc(n + 1, sizeof(int));
        for (int i = 0; i < n; ++i) {
            f->lp[i + 1] = f->lp[i] + diagpos[i];
            f->up[i + 1] = f->up[i] + npat[i] - diagpos[i];
        }
        f->li = malloc(sizeof(int) * (f->lp[n] + 1));
        f->lv = malloc(sizeof(cplx) * (f->lp[n] + 1));
        f->ui = malloc(sizeof(int) * (f->up[n] + 1));
        f->uv = malloc(sizeof(cplx) * (f->up[n] + 1));
        cplx* w = calloc(n, sizeof(cplx));
        int* stamp = malloc(sizeof(int) * n);
        for (int i = 0; i < n; ++i) stamp[i] = -1;
        for (int i = 0; i < n && rc == FWI_OK; ++i) {
            for (int q = 0; q < npat[i]; ++q) {
                stamp[pat[i][q]] = i;
                w[pat[i][q]] = 0;
            }
            for (int p = s->rp[i]; p < s->rp[i + 1]; ++p) w[s->ci[p]] += s->av[p];
            w[i] += shift;
            for (int q = 0; q < diagpos[i]; ++q) { /* IKJ over the lower pattern */
                const int j = pat[i][q];
                const int ud = f->up[j];
                w[j] /= f->uv[ud];
                const cplx lij = w[j];
                if (lij == 0.0) continue;
                for (int p = ud + 1; p < f->up[j + 1]; ++p) {
                    const int k = f->ui[p];
                    if (stamp[k] == i) w[k] -= lij * f->uv[p];
                }
            }
            if (w[i] == 0.0) {
                rc = fail(FWI_ERR_ZERO_PIVOT, i, "ILU: zero pivot at row %d (consider a diagonal shift)", i);
                break;
            }
            for (int q = 0; q < diagpos[i]; ++q) {
                f->li[f->lp[i] + q] = pat[i][q];
                f->lv[f->lp[i] + q] = w[pat[i][q]];
            }
            for (int q = diagpos[i]; q < npat[i]; ++q) {
                f->ui[f->up[i] + q - diagpos[i]] = pat[i][q];
                f->uv[f->up[i] + q - diagpos[i]] = w[pat[i][q]];
            }
        }
        free(w);
        free(stamp);
        if (rc == FWI_OK) {
            transpose(n, f->lp, f->li, f->lv, &f->ltp, &f->lti, &f->ltv);
            transpose(n, f->up, f->ui, f->uv, &f->utp, &f->uti, &f->utv);
        }
    }
    for (int i = 0; i < n; ++i) { free(pat[i]); free(ulv[i]); }
    free(pat); free(npat); free(ulv); free(diagpos); free(lev); free(mark);
    if (rc != FWI_OK && f) {
        free(f->lp); free(f->li); free(f->lv); free(f->up); free(f->ui); free(f->uv); free(f);
        f = NULL;
    }
    *out = f;
    return rc;
}

static void ilu_free(ilu_t* f) {
    if (!f) return;
    free(f->lp); free(f->li); free(f->lv); free(f->up); free(f->ui); free(f->uv);
    free(f->ltp); free(f->lti); free(f->ltv); free(f->utp); free(f->uti); free(f->utv);
    free(f);
}

/* IluFactors::solve, src/ilu.cpp:131-174 */
static void ilu_solve(ilu_t* f, const cplx* b, cplx* x, int adjoint) {
    const int n = f->n;
    f->count++;
    memcpy(x, b, sizeof(cplx) * n);
    if (!adjoint) {
        for (int i = 0; i < n; ++i) {
            cplx s = x[i];
            for (int p = f->lp[i]; p < f->lp[i + 1]; ++p) s -= f->lv[p] * x[f->li[p]];
            x[i] = s;
        }
        for (int i = n - 1; i >= 0; --i) {
            cplx s = x[i];
            const int ud = f->up[i];
            for (int p = ud + 1; p < f->up[i + 1]; ++p) s -= f->uv[p] * x[f->ui[p]];
            x[i] = s / f->uv[ud];
        }
        return;
    }
    for (int i = 0; i < n; ++i) {
        cplx s = x[i], dg = 0;
        for (int p = f->utp[i]; p < f->utp[i + 1]; ++p) {
            const int k = f->uti[p];
            if (k == i)
                dg = f->utv[p];
            else
                s -= conj(f->utv[p]) * x[k];
        }
        x[i] = s / conj(dg);
    }
    for (int i = n - 1; i >= 0; --i) {
        cplx s = x[i];
        for (int p = f->ltp[i]; p < f->ltp[i + 1]; ++p) s -= conj(f->ltv[p]) * x[f->lti[p]];
        x[i] = s;
    }
}

static int block_solve(orc_state* s, int mode, int adjoint, const cplx* b, cplx* x) {
    if (mode == FWI_PRECOND_ILU) {
        if (!s->ilu) return fail(FWI_ERR_INVALID_ARGUMENT, -1, "precond_apply: state has no ILU factorization");
        ilu_solve(s->ilu, b, x, adjoint);
        return FWI_OK;
    }
    if (!s->lu) return fail(FWI_ERR_INVALID_ARGUMENT, -1, "precond_apply: state has no LU factorization");
    lu_solve(s->lu, b, x, adjoint);
    return FWI_OK;
}

/* ---------------------------------------------------------------- state */
void orc_state_free(orc_state* s) {
    if (!s) return;
    free(s->s); free(s->rp); free(s->ci); free(s->av); free(s->u); free(s->r); free(s->dpred);
    free(s->w); free(s->off); free(s->node); free(s->src_node); free(s->src_amp);
    lu_free(s->lu);
    ilu_free(s->ilu);
    free(s);
}

/* make_gn_state, src/reduced_space.cpp:40-86 (with u given: the GnState is
 * built member by member, as the C2 apply benchmark does) */
int orc_state_create(const fwi_state_desc* d, orc_state** out) {
    *out = NULL;
    const fwi_grid_desc* g = &d->grid;
    if (g->nx < 3 || g->nz < 3) return fail(FWI_ERR_INVALID_ARGUMENT, -1, "build_grid: need nx >= 3 and nz >= 3");
    if (!(d->epsilon > 0.0)) return fail(FWI_ERR_INVALID_ARGUMENT, -1, "make_gn_state: epsilon must be positive");
    orc_state* s = calloc(1, sizeof(orc_state));
    s->nx = g->nx;
    s->nz = g->nz;
    s->n = g->nx * g->nz;
    s->npml = g->n_pml;
    s->h = g->h;
    s->sigma_max = g->pml_sigma_max;
    s->power = g->pml_power;
    s->freq = d->freq_hz;
    s->omega = 2.0 * 3.141592653589793238462643383279502884 * d->freq_hz;
    s->eps = d->epsilon;
    s->drop = d->drop_reg_term != 0;
    const int n = s->n, K = d->survey.num_sources;
    s->K = K;
    s->s = malloc(sizeof(double) * n);
    memcpy(s->s, d->s, sizeof(double) * n);
    assemble(s);
    /* survey tables + build_weights (src/forward.cpp:43-62) */
    const fwi_survey_desc* sv = &d->survey;
    s->ndata = sv->recv_offset[K];
    s->off = malloc(sizeof(int) * (K + 1));
    memcpy(s->off, sv->recv_offset, sizeof(int) * (K + 1));
    s->node = malloc(sizeof(int) * (s->ndata + 1));
    s->w = malloc(sizeof(double) * (s->ndata + 1));
    s->src_node = malloc(sizeof(int) * K);
    s->src_amp = malloc(sizeof(double) * K);
    double maxw = 0.0;
    for (int k = 0; k < K; ++k) {
        s->src_node[k] = sv->src_iz[k] * s->nx + sv->src_ix[k];
        s->src_amp[k] = sv->src_amp ? sv->src_amp[k] : 1.0;
        for (int j = sv->recv_offset[k]; j < sv->recv_offset[k + 1]; ++j) {
            s->node[j] = sv->recv_iz[j] * s->nx + sv->recv_ix[j];
            s->w[j] = 1.0;
            if (sv->weight_mode == FWI_WEIGHT_OFFSET) {
                const double dx = sv->recv_ix[j] - sv->src_ix[k], dz = sv->recv_iz[j] - sv->src_iz[k];
                s->w[j] = sqrt(dx * dx + dz * dz);
                if (maxw < s->w[j]) maxw = s->w[j];
            }
        }
    }
    if (sv->weight_mode == FWI_WEIGHT_OFFSET && maxw > 0.0)
        for (int j = 0; j < s->ndata; ++j) s->w[j] /= maxw;
    int rc = FWI_OK;
    if (d->exact_factor || !d->u) rc = lu_factor(s, &s->lu);
    if (rc == FWI_OK && d->ilu_level >= 0) rc = ilu_factor(s, d->ilu_level, d->ilu_diag_shift, &s->ilu);
    if (rc != FWI_OK) {
        orc_state_free(s);
        return rc;
    }
    s->u = calloc((size_t)K * n, sizeof(cplx));
    s->r = calloc(s->ndata + 1, sizeof(cplx));
    s->dpred = calloc(s->ndata + 1, sizeof(cplx));
    if (d->u) {
        memcpy(s->u, d->u, sizeof(cplx) * (size_t)K * n);
    } else { /* solve_forward, src/forward.cpp:64-76 */
        const double load = 1.0 / (s->h * s->h);
        cplx* f = calloc(n, sizeof(cplx));
        for (int k = 0; k < K; ++k) {
            memset(f, 0, sizeof(cplx) * n);
            f[s->src_node[k]] = s->src_amp[k] * load;
            lu_solve(s->lu, f, s->u + (size_t)k * n, 0);
        }
        free(f);
        s->lu->count = 0;
    }
    for (int k = 0; k < K; ++k)
        for (int j = s->off[k]; j < s->off[k + 1]; ++j) s->dpred[j] = s->u[(size_t)k * n + s->node[j]];
    if (d->r)
        memcpy(s->r, d->r, sizeof(cplx) * s->ndata);
    else if (d->d_obs)
        for (int j = 0; j < s->ndata; ++j) s->r[j] = ((const cplx*)d->d_obs)[j] - s->dpred[j];
    *out = s;
    return FWI_OK;
}

void orc_state_info(const orc_state* s, int* n, int* K, int* ndata, int* nnz, double* omega) {
    *n = s->n;
    *K = s->K;
    *ndata = s->ndata;
    *nnz = s->nnz;
    *omega = s->omega;
}
void orc_get_u(const orc_state* s, double* out) { memcpy(out, s->u, sizeof(cplx) * (size_t)s->K * s->n); }
void orc_get_residual(const orc_state* s, double* out) { memcpy(out, s->r, sizeof(cplx) * s->ndata); }
void orc_get_dpred(const orc_state* s, double* out) { memcpy(out, s->dpred, sizeof(cplx) * s->ndata); }
void orc_get_csr(const orc_state* s, int* rp, int* ci, double* v) {
    memcpy(rp, s->rp, sizeof(int) * (s->n + 1));
    memcpy(ci, s->ci, sizeof(int) * s->nnz);
    memcpy(v, s->av, sizeof(cplx) * s->nnz);
}
void orc_set_epsilon(orc_state* s, double e) { s->eps = e; }
void orc_set_drop(orc_state* s, int d) { s->drop = d != 0; }
long long orc_solve_count(const orc_state* s, int mode) {
    if (mode == FWI_PRECOND_ILU) return s->ilu ? s->ilu->count : -1;
    return s->lu ? s->lu->count : -1;
}
int orc_ilu_factor(orc_state* s, int level, double shift) {
    ilu_t* f = NULL;
    const int rc = ilu_factor(s, level, shift, &f);
    if (rc != FWI_OK) return rc;
    ilu_free(s->ilu);
    s->ilu = f;
    return FWI_OK;
}

/* flat KKT layout: [du_0..du_{K-1} | ds | la_0..la_{K-1}] */
#define DU(base, k) ((cplx*)(base) + (size_t)(k) * s->n)
#define DS(base) ((double*)(base) + 2 * (size_t)s->K * s->n)
#define LA(base, k) ((cplx*)((double*)(base) + 2 * (size_t)s->K * s->n + s->n) + (size_t)(k) * s->n)

/* kkt_apply, src/kkt.cpp:78-96 (apply_f :50-58, apply_p :60-66,
 * accumulate_re_p_adjoint :68-74) */
int orc_kkt_apply(const orc_state* s, const double* in, double* out) {
    const int n = s->n, K = s->K;
    const double w2 = s->omega * s->omega;
    cplx* t = malloc(sizeof(cplx) * n);
    cplx* p = malloc(sizeof(cplx) * n);
    for (int k = 0; k < K; ++k) {
        cplx* od = DU(out, k);
        const cplx* xd = DU(in, k);
        const cplx* xl = LA(in, k);
        const cplx* uk = s->u + (size_t)k * n;
        for (int i = 0; i < n; ++i) od[i] = 0;
        for (int j = s->off[k]; j < s->off[k + 1]; ++j) {
            const double w = s->w[j];
            od[s->node[j]] += w * w * xd[s->node[j]];
        }
        spmv(s, xl, t, 1);
        const cplx one = 1.0;
        for (int i = 0; i < n; ++i) od[i] += one * t[i];
        cplx* ol = LA(out, k);
        spmv(s, xd, ol, 0);
        for (int i = 0; i < n; ++i) p[i] = w2 * uk[i] * DS(in)[i];
        const cplx mone = -1.0;
        for (int i = 0; i < n; ++i) ol[i] += mone * p[i];
    }
    double* ods = DS(out);
    for (int i = 0; i < n; ++i) ods[i] = s->eps * DS(in)[i];
    double* pl = calloc(n, sizeof(double));
    for (int k = 0; k < K; ++k) {
        const cplx* uk = s->u + (size_t)k * n;
        const cplx* z = LA(in, k);
        for (int i = 0; i < n; ++i) pl[i] += creal(w2 * conj(uk[i]) * z[i]);
    }
    for (int i = 0; i < n; ++i) ods[i] += -1.0 * pl[i];
    free(pl);
    free(t);
    free(p);
    return FWI_OK;
}

/* kkt_rhs, src/kkt.cpp:98-112 */
int orc_kkt_rhs(const orc_state* s, double* out) {
    const int n = s->n, K = s->K;
    memset(out, 0, sizeof(double) * (4 * (size_t)K * n + n));
    for (int k = 0; k < K; ++k)
        for (int j = s->off[k]; j < s->off[k + 1]; ++j) {
            const double w = s->w[j];
            DU(out, k)[s->node[j]] += w * w * s->r[j];
        }
    if (!s->drop)
        for (int i = 0; i < n; ++i) DS(out)[i] = -s->eps * s->s[i];
    return FWI_OK;
}

/* precond_apply, src/kkt.cpp:114-135 */
int orc_precond_apply(orc_state* s, int mode, const double* in, double* out) {
    const int n = s->n, K = s->K;
    const double w2 = s->omega * s->omega;
    if (mode == FWI_PRECOND_ILU && !s->ilu)
        return fail(FWI_ERR_INVALID_ARGUMENT, -1, "precond_apply: state has no ILU factorization");
    int rc;
    for (int k = 0; k < K; ++k)
        if ((rc = block_solve(s, mode, 1, DU(in, k), LA(out, k))) != FWI_OK) return rc;
    double* pl = calloc(n, sizeof(double));
    for (int k = 0; k < K; ++k) {
        const cplx* uk = s->u + (size_t)k * n;
        const cplx* z = LA(out, k);
        for (int i = 0; i < n; ++i) pl[i] += creal(w2 * conj(uk[i]) * z[i]);
    }
    for (int i = 0; i < n; ++i) DS(out)[i] = (DS(in)[i] + pl[i]) / s->eps;
    free(pl);
    cplx* rhs = malloc(sizeof(cplx) * n);
    const cplx one = 1.0;
    for (int k = 0; k < K; ++k) {
        const cplx* uk = s->u + (size_t)k * n;
        for (int i = 0; i < n; ++i) rhs[i] = w2 * uk[i] * DS(out)[i];
        for (int i = 0; i < n; ++i) rhs[i] += one * LA(in, k)[i];
        if ((rc = block_solve(s, mode, 0, rhs, DU(out, k))) != FWI_OK) break;
    }
    free(rhs);
    return rc;
}

int orc_solve(orc_state* s, int mode, int adjoint, const double* b, double* x) {
    return block_solve(s, mode, adjoint, (const cplx*)b, (cplx*)x);
}

/* ---------------------------------------------------------------- reduced space */
/* gradient, src/reduced_space.cpp:141-152 (jacobian_adjoint_apply :99-116) */
int orc_gradient(orc_state* s, double* g) {
    const int n = s->n, K = s->K;
    if (!s->lu) return fail(FWI_ERR_INVALID_ARGUMENT, -1, "gradient: state has no LU factorization");
    const double w2 = s->omega * s->omega;
    cplx* acc = calloc(n, sizeof(cplx));
    cplx* y = malloc(sizeof(cplx) * n);
    cplx* z = malloc(sizeof(cplx) * n);
    for (int k = 0; k < K; ++k) {
        for (int i = 0; i < n; ++i) y[i] = 0;
        for (int j = s->off[k]; j < s->off[k + 1]; ++j) {
            cplx wr = s->r[j];
            wr *= s->w[j] * s->w[j];
            y[s->node[j]] += wr;
        }
        lu_solve(s->lu, y, z, 1);
        const cplx* uk = s->u + (size_t)k * n;
        for (int i = 0; i < n; ++i) acc[i] += w2 * conj(uk[i]) * z[i];
    }
    for (int i = 0; i < n; ++i) g[i] = creal(acc[i]);
    if (!s->drop)
        for (int i = 0; i < n; ++i) g[i] -= s->eps * s->s[i];
    free(acc); free(y); free(z);
    return FWI_OK;
}

/* hessian_apply, src/reduced_space.cpp:120-139 */
int orc_hessian_apply(orc_state* s, const double* v, double* out) {
    const int n = s->n, K = s->K;
    if (!s->lu) return fail(FWI_ERR_INVALID_ARGUMENT, -1, "hessian_apply: state has no LU factorization");
    const double w2 = s->omega * s->omega;
    cplx* acc = calloc(n, sizeof(cplx));
    cplx* y = malloc(sizeof(cplx) * n);
    cplx* x = malloc(sizeof(cplx) * n);
    cplx* z = malloc(sizeof(cplx) * n);
    for (int k = 0; k < K; ++k) {
        const cplx* uk = s->u + (size_t)k * n;
        for (int i = 0; i < n; ++i) y[i] = w2 * uk[i] * v[i];
        lu_solve(s->lu, y, x, 0);
        for (int i = 0; i < n; ++i) y[i] = 0;
        for (int j = s->off[k]; j < s->off[k + 1]; ++j) {
            cplx d = x[s->node[j]];
            d *= s->w[j] * s->w[j];
            y[s->node[j]] += d;
        }
        lu_solve(s->lu, y, z, 1);
        for (int i = 0; i < n; ++i) acc[i] += w2 * conj(uk[i]) * z[i];
    }
    for (int i = 0; i < n; ++i) out[i] = creal(acc[i]) + s->eps * v[i];
    free(acc); free(y); free(x); free(z);
    return FWI_OK;
}

/* ---------------------------------------------------------------- Krylov */
/* KktVector dot/norm/axpy/scal, src/kkt.cpp:15-39 over vec.hpp:16-58 */
static double kdot(const orc_state* s, const double* x, const double* y) {
    const int n = s->n, K = s->K;
    double acc = 0.0;
    for (int k = 0; k < K; ++k) {
        cplx c = 0;
        for (int i = 0; i < n; ++i) c += conj(DU(x, k)[i]) * DU(y, k)[i];
        acc += creal(c);
    }
    double r = 0.0;
    for (int i = 0; i < n; ++i) r += DS(x)[i] * DS(y)[i];
    acc += r;
    for (int k = 0; k < K; ++k) {
        cplx c = 0;
        for (int i = 0; i < n; ++i) c += conj(LA(x, k)[i]) * LA(y, k)[i];
        acc += creal(c);
    }
    return acc;
}

static double knorm(const orc_state* s, const double* x) { return sqrt(kdot(s, x, x)); }

static void kaxpy(const orc_state* s, double a, const double* x, double* y) {
    const int n = s->n, K = s->K;
    const cplx ca = a;
    for (int k = 0; k < K; ++k)
        for (int i = 0; i < n; ++i) DU(y, k)[i] += ca * DU(x, k)[i];
    for (int i = 0; i < n; ++i) DS(y)[i] += a * DS(x)[i];
    for (int k = 0; k < K; ++k)
        for (int i = 0; i < n; ++i) LA(y, k)[i] += ca * LA(x, k)[i];
}

static void kscal(const orc_state* s, double a, double* x) {
    const int n = s->n, K = s->K;
    const cplx ca = a;
    for (int k = 0; k < K; ++k)
        for (int i = 0; i < n; ++i) DU(x, k)[i] *= ca;
    for (int i = 0; i < n; ++i) DS(x)[i] *= a;
    for (int k = 0; k < K; ++k)
        for (int i = 0; i < n; ++i) LA(x, k)[i] *= ca;
}

static double now_s(void) {
    struct timespec t;
    clock_gettime(CLOCK_MONOTONIC, &t);
    return t.tv_sec + 1e-9 * t.tv_nsec;
}

static void log_push(fwi_convergence_log* lg, int it, double res, int has_p, double pres, double wall) {
    if (!lg || lg->count >= lg->capacity) return;
    fwi_log_entry* e = &lg->entries[lg->count++];
    memset(e, 0, sizeof *e);
    e->iteration = it;
    e->residual_norm = res;
    e->has_precond_residual = has_p;
    e->precond_residual = pres;
    e->wall_time = wall;
}

/* gmres, include/fwi/krylov.hpp:128-269 with S = double (the KKT inner
 * product is real). Observer: normal_residual every ecg_stride iterations. */
static int gmres_kkt(orc_state* s, const fwi_fsgn_options* o, const double* b, double* x,
                     fwi_convergence_log* lg, const double* g, double gnorm, int* metric_it,
                     double* metric_val, int* nmetric) {
    const size_t len = 4 * (size_t)s->K * s->n + s->n;
    const size_t bytes = len * sizeof(double);
    const int restart = o->restart, maxit = o->maxit;
    const double tol = o->tol;
    if (restart < 1) return fail(FWI_ERR_INVALID_ARGUMENT, -1, "gmres: restart must be >= 1");
    const double t0 = now_s();
    double obs_time = 0.0;
    int rc = FWI_OK;
    memset(x, 0, bytes);
    lg->count = 0;
    lg->converged = lg->stagnated = 0;
    const double bnorm = knorm(s, b);
    if (bnorm == 0.0) {
        log_push(lg, 0, 0.0, 0, 0.0, now_s() - t0);
        lg->converged = 1;
        return FWI_OK;
    }
    double* tmp = malloc(bytes);
    double* w = malloc(bytes);
    double* xc = malloc(bytes);
    double* best = calloc(len, sizeof(double));
    double* resid = malloc(bytes);
    double** v = calloc(restart + 1, sizeof(double*));
    double* hcols = calloc((size_t)(restart + 1) * (restart + 2), sizeof(double));
    double *gs_c = calloc(restart + 1, sizeof(double)), *gs_s = calloc(restart + 1, sizeof(double));
    double* gg = calloc(restart + 2, sizeof(double));
    double* h = calloc(restart + 2, sizeof(double));
    double* y = calloc(restart + 1, sizeof(double));
    double* hds = malloc(sizeof(double) * s->n);
    if ((rc = orc_precond_apply(s, o->mode, b, w)) != FWI_OK) goto done;
    const double pbnorm = knorm(s, w);
    if (pbnorm == 0.0) {
        rc = fail(FWI_ERR_INVALID_ARGUMENT, -1, "gmres: preconditioner annihilates the right-hand side");
        goto done;
    }
    log_push(lg, 0, 1.0, 1, 1.0, now_s() - t0);
    double best_res = 1.0, true_res = 1.0;
    int iter = 0, stop = 0;
    while (iter < maxit && !lg->converged && !stop) {
        orc_kkt_apply(s, x, tmp);
        memcpy(resid, b, bytes);
        kaxpy(s, -1.0, tmp, resid);
        if (!v[0]) v[0] = malloc(bytes);
        if ((rc = orc_precond_apply(s, o->mode, resid, v[0])) != FWI_OK) goto done;
        const double beta = knorm(s, v[0]);
        const double cycle_start = true_res;
        if (beta == 0.0) break;
        kscal(s, 1.0 / beta, v[0]);
        gg[0] = beta;
        memcpy(xc, x, bytes);
        int happy = 0;
        for (int j = 0; j < restart && iter < maxit; ++j) {
            ++iter;
            orc_kkt_apply(s, v[j], tmp);
            if ((rc = orc_precond_apply(s, o->mode, tmp, w)) != FWI_OK) goto done;
            for (int i = 0; i <= j + 1; ++i) h[i] = 0.0;
            for (int i = 0; i <= j; ++i) {
                h[i] = kdot(s, v[i], w);
                kaxpy(s, -h[i], v[i], w);
            }
            const double wn = knorm(s, w);
            h[j + 1] = wn;
            for (int i = 0; i < j; ++i) {
                const double t = gs_c[i] * h[i] + gs_s[i] * h[i + 1];
                h[i + 1] = -gs_s[i] * h[i] + gs_c[i] * h[i + 1];
                h[i] = t;
            }
            double c, sn, rr;
            const double an = fabs(h[j]), bn = fabs(h[j + 1]);
            const double t = sqrt(an * an + bn * bn);
            if (bn == 0.0) { c = 1.0; sn = 0.0; rr = h[j]; }
            else if (an == 0.0) { c = 0.0; sn = h[j + 1] / bn; rr = bn; }
            else { c = an / t; sn = (h[j] / an) * h[j + 1] / t; rr = (h[j] / an) * t; }
            gs_c[j] = c;
            gs_s[j] = sn;
            h[j] = rr;
            h[j + 1] = 0.0;
            gg[j + 1] = -sn * gg[j];
            gg[j] = c * gg[j];
            memcpy(hcols + (size_t)j * (restart + 2), h, sizeof(double) * (j + 2));
            const double prec_res = fabs(gg[j + 1]) / pbnorm;
            for (int i = j; i >= 0; --i) {
                double acc = gg[i];
                for (int k2 = i + 1; k2 <= j; ++k2) acc -= hcols[(size_t)k2 * (restart + 2) + i] * y[k2];
                y[i] = acc / hcols[(size_t)i * (restart + 2) + i];
            }
            memcpy(xc, x, bytes);
            for (int i = 0; i <= j; ++i) kaxpy(s, y[i], v[i], xc);
            memcpy(resid, b, bytes);
            orc_kkt_apply(s, xc, tmp);
            kaxpy(s, -1.0, tmp, resid);
            true_res = knorm(s, resid) / bnorm;
            log_push(lg, iter, true_res, 1, prec_res, now_s() - t0 - obs_time);
            if (true_res < best_res) {
                best_res = true_res;
                memcpy(best, xc, bytes);
            }
            if (o->ecg_stride > 0 && iter % o->ecg_stride == 0) {
                const double to = now_s();
                if ((rc = orc_hessian_apply(s, DS(xc), hds)) != FWI_OK) goto done;
                double rn = 0.0;
                for (int i = 0; i < s->n; ++i) {
                    hds[i] += -1.0 * g[i];
                    rn += hds[i] * hds[i];
                }
                rn = sqrt(rn);
                const double e = gnorm == 0.0 ? (rn == 0.0 ? 0.0 : INFINITY) : rn / gnorm;
                metric_it[*nmetric] = iter;
                metric_val[(*nmetric)++] = e;
                stop = o->ecg_stop_tol > 0.0 && e <= o->ecg_stop_tol;
                obs_time += now_s() - to;
            }
            if (true_res <= tol) lg->converged = 1;
            if (wn == 0.0) happy = 1;
            if (lg->converged || stop || happy) break;
            kscal(s, 1.0 / wn, w);
            double* sw = v[j + 1];
            v[j + 1] = w;
            w = sw ? sw : malloc(bytes);
        }
        memcpy(x, xc, bytes);
        if (!lg->converged && !stop && true_res >= cycle_start * (1.0 - 1e-12)) {
            lg->stagnated = 1;
            memcpy(x, best, bytes);
            break;
        }
        if (happy && !lg->converged && !stop) {
            lg->stagnated = 1;
            memcpy(x, best, bytes);
            break;
        }
    }
done:
    for (int i = 0; i <= restart; ++i) free(v[i]);
    free(v); free(tmp); free(w); free(xc); free(best); free(resid); free(hcols); free(gs_c); free(gs_s);
    free(gg); free(h); free(y); free(hds);
    return rc;
}

/* fsgn_gmres_step, src/kkt.cpp:137-171 */
int orc_fsgn(orc_state* s, const fwi_fsgn_options* o, double* ds, fwi_convergence_log* lg) {
    const int n = s->n;
    const size_t len = 4 * (size_t)s->K * n + n;
    double* b = malloc(len * sizeof(double));
    double* x = malloc(len * sizeof(double));
    double* g = calloc(n, sizeof(double));
    int* mit = malloc(sizeof(int) * (o->maxit + 2));
    double* mval = malloc(sizeof(double) * (o->maxit + 2));
    int nm = 0, rc;
    orc_kkt_rhs(s, b);
    double gnorm = 0.0;
    if (s->lu) {
        orc_gradient(s, g);
        for (int i = 0; i < n; ++i) gnorm += g[i] * g[i];
        gnorm = sqrt(gnorm);
    }
    rc = gmres_kkt(s, o, b, x, lg, g, gnorm, mit, mval, &nm);
    if (rc == FWI_OK) {
        if (lg->count > 0 && s->lu) {
            lg->entries[0].has_normal_residual = 1;
            lg->entries[0].normal_residual = gnorm > 0.0 ? 1.0 : 0.0;
        }
        for (int q = 0; q < nm; ++q)
            for (int e = 0; e < lg->count; ++e)
                if (lg->entries[e].iteration == mit[q]) {
                    lg->entries[e].has_normal_residual = 1;
                    lg->entries[e].normal_residual = mval[q];
                    break;
                }
        memcpy(ds, DS(x), sizeof(double) * n);
    }
    free(b); free(x); free(g); free(mit); free(mval);
    return rc;
}
