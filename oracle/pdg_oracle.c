/*
 * oracle/pdg_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU fp64 implementation of the PDG hot path
 * (arxiv 1702.00169, "Task-based parallelization of an implicit kinetic scheme").
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load it.  It shares no code, header, table or constant with the CUDA
 * product in paper_1702_00169_b200/; neither side includes the other.
 *
 * Citations "P:n" are lines of PAPER.md (the paper's LaTeX source); readings of
 * silent/garbled passages are the C-numbered readings listed in DESIGN.md.
 *
 * What is computed (and in what order) follows the paper literally:
 *   - 1-D Gauss-Lobatto nodes/weights and Lagrange basis;
 *   - tensor reference element, face weights mu_i^eps;
 *   - affine cell geometry: det tau', cofactor matrix co(tau') (eq co_mat);
 *   - the reduced DG operator, split as Gamma_{L<-L} and Gamma_{L<-R} (P:368-372
 *     eq DG_reduit), with fictitious boundary cells;
 *   - dependency graph "edge L->R iff n_LR.v > 0 at a face GL point" and a Kahn
 *     topological order;
 *   - Crank-Nicolson transport T2(dt') = (I + dt'/2 L)(I - dt'/2 L)^{-1}
 *     (P:440-444 eq transport_cn), solved cell by cell in topological order
 *      with a dense LU of the local block;
 *   - moments w = P f, equilibrium and collision C2 (P:445-454,
 *     P:474-477);
 *   - the palindromic step M2 = T2(dt/2) C2(dt) T2(dt/2) is composed in
 *     oracle/oracle.py.
 *
 * Nothing here exploits axis alignment of the velocities: the operator is the
 * full (p+1)^D x (p+1)^D block of eq. DG_reduit for an arbitrary velocity v.
 *
 * Build: gcc -O2 -ffp-contract=off -fopenmp -shared -fPIC (plain IEEE binary64).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_MAXN 6   /* max nodes per axis (p <= 5) */

/* ------------------------------------------------------------------------- */
/* 1-D Gauss-Lobatto nodes and weights on [-1,1].                 */
/* Closed forms: textbook Lobatto quadrature.                                  */
/* ------------------------------------------------------------------------- */
int or_gl_1d(int p, double *x, double *w)
{
    switch (p) {
    case 1:
        x[0] = -1.0; x[1] = 1.0;
        w[0] = 1.0;  w[1] = 1.0;
        return 0;
    case 2:
        x[0] = -1.0; x[1] = 0.0; x[2] = 1.0;
        w[0] = 1.0 / 3.0; w[1] = 4.0 / 3.0; w[2] = 1.0 / 3.0;
        return 0;
    case 3:
        x[0] = -1.0; x[1] = -1.0 / sqrt(5.0); x[2] = 1.0 / sqrt(5.0); x[3] = 1.0;
        w[0] = 1.0 / 6.0; w[1] = 5.0 / 6.0; w[2] = 5.0 / 6.0; w[3] = 1.0 / 6.0;
        return 0;
    case 4:
        x[0] = -1.0; x[1] = -sqrt(3.0 / 7.0); x[2] = 0.0; x[3] = sqrt(3.0 / 7.0); x[4] = 1.0;
        w[0] = 1.0 / 10.0; w[1] = 49.0 / 90.0; w[2] = 32.0 / 45.0; w[3] = 49.0 / 90.0; w[4] = 1.0 / 10.0;
        return 0;
    default:
        return -1;
    }
}

/* Lagrange basis l_b(t) = prod_{j != b} (t - x_j)/(x_b - x_j). */
static double lagrange(int n, const double *x, int b, double t)
{
    double r = 1.0;
    for (int j = 0; j < n; j++)
        if (j != b) r *= (t - x[j]) / (x[b] - x[j]);
    return r;
}

/* l_b'(t) by the product rule: sum_k 1/(x_b - x_k) prod_{j != b,k} (t - x_j)/(x_b - x_j). */
static double lagrange_deriv(int n, const double *x, int b, double t)
{
    double s = 0.0;
    for (int k = 0; k < n; k++) {
        if (k == b) continue;
        double term = 1.0 / (x[b] - x[k]);
        for (int j = 0; j < n; j++)
            if (j != b && j != k) term *= (t - x[j]) / (x[b] - x[j]);
        s += term;
    }
    return s;
}

/* Exported for pins: Dm[a*n + b] = l_b'(x_a). */
int or_lagrange_deriv_matrix(int p, double *Dm)
{
    double x[OR_MAXN], w[OR_MAXN];
    if (or_gl_1d(p, x, w)) return -1;
    int n = p + 1;
    for (int a = 0; a < n; a++)
        for (int b = 0; b < n; b++) Dm[a * n + b] = lagrange_deriv(n, x, b, x[a]);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Mesh: Cartesian box [lo,hi] with ncell[d] cells per axis, dim in {1,2,3}.  */
/* Cell id = c0 + N0*(c1 + N1*c2); local node index i = a0 + n*(a1 + n*a2).   */
/* ------------------------------------------------------------------------- */
typedef struct {
    int32_t dim;
    int32_t p;
    int64_t ncell[3];
    double lo[3];
    double hi[3];
} or_mesh;

static int64_t mesh_ncells(const or_mesh *m)
{
    int64_t c = 1;
    for (int d = 0; d < m->dim; d++) c *= m->ncell[d];
    return c;
}

static int ipow(int b, int e) { int r = 1; while (e-- > 0) r *= b; return r; }

static void local_to_multi(int i, int n, int dim, int a[3])
{
    a[0] = a[1] = a[2] = 0;
    for (int d = 0; d < dim; d++) { a[d] = i % n; i /= n; }
}

static void cell_to_multi(const or_mesh *m, int64_t c, int64_t cc[3])
{
    cc[0] = cc[1] = cc[2] = 0;
    for (int d = 0; d < m->dim; d++) { cc[d] = c % m->ncell[d]; c /= m->ncell[d]; }
}

static int64_t multi_to_cell(const or_mesh *m, const int64_t cc[3])
{
    int64_t c = 0;
    for (int d = m->dim - 1; d >= 0; d--) c = c * m->ncell[d] + cc[d];
    return c;
}

/* neighbour of cell c across face (d, side) with side 0 = low (-e_d), 1 = high (+e_d); -1 = boundary */
static int64_t neighbour(const or_mesh *m, int64_t c, int d, int side)
{
    int64_t cc[3];
    cell_to_multi(m, c, cc);
    cc[d] += side ? 1 : -1;
    if (cc[d] < 0 || cc[d] >= m->ncell[d]) return -1;
    return multi_to_cell(m, cc);
}

/* ------------------------------------------------------------------------- */
/* The reduced DG operator for one constant velocity v.*/
/*                                                                           */
/*  d/dt f_L + Gamma_LL f_L + sum_R Gamma_LR f_R = 0                          */
/*                                                                           */
/*  Gamma_LL[i][j] = -(1/omega_Li) v.c_Lj grad^phi_i(x^_j) omega_j            */
/*                   + delta_ij (1/omega_Li) sum_eps mu_i^eps (v.c_Li n^_eps)^+ */
/*  Gamma_LR^eps[i] = (1/omega_Li) mu_i^eps (v.c_Li n^_eps)^-  (couples f_R,i')*/
/*                                                                           */
/*  Affine cells: tau_L(x^) = centre + diag(h/2) x^, so det tau' = prod h_d/2  */
/*  and co(tau') = det(tau') tau'^{-T} = diag(det/(h_d/2)) (eq co_mat). */
/*  Every cell of the box has the same blocks.                                */
/*  Face eps = 2*d + side, outward normal n^ = (side ? +1 : -1) e_d.          */
/* ------------------------------------------------------------------------- */
int or_cell_operator(const or_mesh *m, const double *v, double *GLL, double *GLR)
{
    double x[OR_MAXN], w[OR_MAXN];
    if (m->dim < 1 || m->dim > 3) return -1;
    if (or_gl_1d(m->p, x, w)) return -1;
    const int n = m->p + 1, dim = m->dim, Nd = ipow(n, dim);

    double half_h[3], det = 1.0, co[3];
    for (int d = 0; d < dim; d++) {
        half_h[d] = 0.5 * (m->hi[d] - m->lo[d]) / (double)m->ncell[d];
        det *= half_h[d];
    }
    for (int d = 0; d < dim; d++) co[d] = det / half_h[d];

    for (int i = 0; i < Nd; i++) {
        int ai[3];
        local_to_multi(i, n, dim, ai);
        double omega_i = 1.0;
        for (int d = 0; d < dim; d++) omega_i *= w[ai[d]];
        const double omega_Li = omega_i * det; /* eq map_GL */

        /* volume term: -(1/omega_Li) sum_j v.c_Lj grad^phi_i(x^_j) f_j omega_j */
        for (int j = 0; j < Nd; j++) {
            int aj[3];
            local_to_multi(j, n, dim, aj);
            double omega_j = 1.0;
            for (int d = 0; d < dim; d++) omega_j *= w[aj[d]];
            double vcgrad = 0.0; /* v . c_Lj grad^phi_i(x^_j) */
            for (int d = 0; d < dim; d++) {
                /* d/dx^_d of phi^_i = l_{ai_d}'(x^_d) prod_{e!=d} l_{ai_e}(x^_e), at x^_j */
                double g = lagrange_deriv(n, x, ai[d], x[aj[d]]);
                for (int e = 0; e < dim; e++)
                    if (e != d) g *= lagrange(n, x, ai[e], x[aj[e]]);
                vcgrad += v[d] * co[d] * g;
            }
            GLL[i * Nd + j] = -(1.0 / omega_Li) * vcgrad * omega_j;
        }
        /* face terms */
        for (int d = 0; d < dim; d++) {
            for (int side = 0; side < 2; side++) {
                const int eps = 2 * d + side;
                const int on_face = side ? (ai[d] == n - 1) : (ai[d] == 0);
                double mu = 0.0;
                if (on_face) {
                    mu = 1.0;
                    for (int e = 0; e < dim; e++)
                        if (e != d) mu *= w[ai[e]];
                }
                const double vcn = v[d] * co[d] * (side ? 1.0 : -1.0); /* v . c_Li n^_eps */
                const double vcn_plus = vcn > 0.0 ? vcn : 0.0;
                const double vcn_minus = vcn < 0.0 ? vcn : 0.0;
                GLL[i * Nd + i] += (1.0 / omega_Li) * mu * vcn_plus;
                GLR[eps * Nd + i] = (1.0 / omega_Li) * mu * vcn_minus;
            }
        }
    }
    return 0;
}

/* Matched node i' across face (d, side): the node of R at the same physical point. */
static int matched_node(int i, int n, int dim, int d)
{
    int a[3];
    local_to_multi(i, n, dim, a);
    a[d] = (a[d] == 0) ? n - 1 : 0;
    int j = 0;
    for (int e = dim - 1; e >= 0; e--) j = j * n + a[e];
    return j;
}

/* ------------------------------------------------------------------------- */
/* Dependency graph: edge L->R iff n_LR . v > 0 at a GL point of   */
/* the common face.  On the affine box n_LR = +-e_d (times a positive scale),  */
/* |v.n| <= 1e-12 |v||n| is treated as 0 (tangential; DESIGN.md reading).     */
/* ------------------------------------------------------------------------- */
static int face_outflow(const double *v, int dim, int d, int side)
{
    double vn = v[d] * (side ? 1.0 : -1.0);
    double vnorm = 0.0;
    for (int e = 0; e < dim; e++) vnorm += v[e] * v[e];
    vnorm = sqrt(vnorm);
    return vn > 1e-12 * vnorm;
}

/*
 * Kahn topological order over a subset of cells (all cells if cells == NULL),
 * lowest cell id first among ready cells (DESIGN.md reading).  Fictitious
 * cells are excluded.  level[k] = longest path from a source.
 * Returns 0, -2 if an upwind real neighbour of a subset cell is missing from
 * the subset, -3 on a cycle.
 */
typedef struct { int64_t *h; int64_t n; } heap_t;
static void heap_push(heap_t *hp, int64_t v)
{
    int64_t k = hp->n++;
    hp->h[k] = v;
    while (k > 0) {
        int64_t par = (k - 1) / 2;
        if (hp->h[par] <= hp->h[k]) break;
        int64_t t = hp->h[par]; hp->h[par] = hp->h[k]; hp->h[k] = t;
        k = par;
    }
}
static int64_t heap_pop(heap_t *hp)
{
    int64_t top = hp->h[0];
    hp->h[0] = hp->h[--hp->n];
    int64_t k = 0;
    for (;;) {
        int64_t l = 2 * k + 1, r = l + 1, s = k;
        if (l < hp->n && hp->h[l] < hp->h[s]) s = l;
        if (r < hp->n && hp->h[r] < hp->h[s]) s = r;
        if (s == k) break;
        int64_t t = hp->h[s]; hp->h[s] = hp->h[k]; hp->h[k] = t;
        k = s;
    }
    return top;
}

int or_topo_order(const or_mesh *m, const double *v, int64_t nsub, const int64_t *cells,
                  int64_t *order, int32_t *level)
{
    const int64_t ncell = mesh_ncells(m);
    const int dim = m->dim;
    if (!cells) nsub = ncell;
    int32_t *slot = (int32_t *)malloc(sizeof(int32_t) * ncell);
    int32_t *indeg = (int32_t *)calloc(nsub, sizeof(int32_t));
    int32_t *lev = (int32_t *)calloc(nsub, sizeof(int32_t));
    heap_t hp = { (int64_t *)malloc(sizeof(int64_t) * (nsub + 1)), 0 };
    int rc = 0;
    for (int64_t c = 0; c < ncell; c++) slot[c] = cells ? -1 : (int32_t)c;
    if (cells)
        for (int64_t s = 0; s < nsub; s++) slot[cells[s]] = (int32_t)s;

    /* in-degree: number of real upwind neighbours R with edge R->L */
    for (int64_t s = 0; s < nsub && rc == 0; s++) {
        int64_t c = cells ? cells[s] : s;
        for (int d = 0; d < dim; d++)
            for (int side = 0; side < 2; side++) {
                int64_t r = neighbour(m, c, d, side);
                if (r < 0) continue;
                /* edge r -> c iff n_{r,c}.v > 0; n_{r,c} points from r to c = opposite of this face's normal */
                if (face_outflow(v, dim, d, 1 - side)) {
                    if (slot[r] < 0) { rc = -2; break; }
                    indeg[s]++;
                }
            }
    }
    int64_t k = 0;
    if (rc == 0) {
        for (int64_t s = 0; s < nsub; s++)
            if (indeg[s] == 0) heap_push(&hp, cells ? cells[s] : s);
        while (hp.n > 0) {
            int64_t c = heap_pop(&hp);
            int64_t sc = slot[c];
            order[k] = c;
            if (level) level[k] = lev[sc];
            k++;
            for (int d = 0; d < dim; d++)
                for (int side = 0; side < 2; side++) {
                    if (!face_outflow(v, dim, d, side)) continue; /* edge c -> r */
                    int64_t r = neighbour(m, c, d, side);
                    if (r < 0 || slot[r] < 0) continue;
                    int64_t sr = slot[r];
                    if (lev[sr] < lev[sc] + 1) lev[sr] = lev[sc] + 1;
                    if (--indeg[sr] == 0) heap_push(&hp, r);
                }
        }
        if (k != nsub) rc = -3;
    }
    free(slot); free(indeg); free(lev); free(hp.h);
    return rc;
}

/*
 * Upstream closure of a set of cells for velocity v: every cell from which a
 * path of dependency edges leads into the set (the cells the sweep needs
 * before it can produce the set).  out_mask[c] = 1 for members.
 */
int or_upstream_closure(const or_mesh *m, const double *v, int64_t nseed, const int64_t *seed,
                        uint8_t *mask)
{
    const int64_t ncell = mesh_ncells(m);
    int64_t *stack = (int64_t *)malloc(sizeof(int64_t) * ncell);
    int64_t top = 0;
    for (int64_t s = 0; s < nseed; s++)
        if (!mask[seed[s]]) { mask[seed[s]] = 1; stack[top++] = seed[s]; }
    while (top > 0) {
        int64_t c = stack[--top];
        for (int d = 0; d < m->dim; d++)
            for (int side = 0; side < 2; side++) {
                int64_t r = neighbour(m, c, d, side);
                if (r < 0 || mask[r]) continue;
                if (face_outflow(v, m->dim, d, 1 - side)) { mask[r] = 1; stack[top++] = r; }
            }
    }
    free(stack);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Dense LU with partial pivoting (plain Doolittle), used for the local solve */
/* (the paper uses KLU; the result is the same linear solve).      */
/* ------------------------------------------------------------------------- */
static int lu_factor(int n, double *A, int *piv)
{
    for (int k = 0; k < n; k++) {
        int pr = k;
        double best = fabs(A[k * n + k]);
        for (int r = k + 1; r < n; r++)
            if (fabs(A[r * n + k]) > best) { best = fabs(A[r * n + k]); pr = r; }
        if (best == 0.0) return -1;
        piv[k] = pr;
        if (pr != k)
            for (int c = 0; c < n; c++) { double t = A[k * n + c]; A[k * n + c] = A[pr * n + c]; A[pr * n + c] = t; }
        for (int r = k + 1; r < n; r++) {
            A[r * n + k] /= A[k * n + k];
            for (int c = k + 1; c < n; c++) A[r * n + c] -= A[r * n + k] * A[k * n + c];
        }
    }
    return 0;
}

static void lu_solve(int n, const double *LU, const int *piv, double *b)
{
    for (int k = 0; k < n; k++)
        if (piv[k] != k) { double t = b[k]; b[k] = b[piv[k]]; b[piv[k]] = t; }
    for (int r = 1; r < n; r++)
        for (int c = 0; c < r; c++) b[r] -= LU[r * n + c] * b[c];
    for (int r = n - 1; r >= 0; r--) {
        for (int c = r + 1; c < n; c++) b[r] -= LU[r * n + c] * b[c];
        b[r] /= LU[r * n + r];
    }
}

/* ------------------------------------------------------------------------- */
/* T2(dt') for one velocity on a subset of cells (all if cells == NULL).      */
/*                                                                           */
/*  theta = dt'/2 (eq transport_cn; reading C1 for the missing 1/2 in   */
/*  eq crank_nicolson).  With d/dt f_L = -Gamma_LL f_L - sum Gamma_LR f_R */
/*  the CN system (I - theta L) F^new = (I + theta L) F^old reads, cell by     */
/*  cell in topological order:                                    */
/*    (I + theta Gamma_LL) f_L^new =                                          */
/*        (I - theta Gamma_LL) f_L^old - theta sum_R Gamma_LR (f_R^old + f_R^new) */
/*  Fictitious boundary cells obey d/dt f_R = 0 (eq fictitious_ODE), so */
/*  f_R^old = f_R^new = f^b there (reading C5).                               */
/*                                                                           */
/*  f  : [nsub][Nd] cell-blocked values (in/out).                             */
/*  fb : [nsub][Nd] boundary values f^b(x_Li) stored at the boundary cell's   */
/*       own face nodes (x_Li = x_Ri'); read only at inflow boundary faces.    */
/* ------------------------------------------------------------------------- */
int or_t2(const or_mesh *m, const double *v, double dtp, int64_t nsub, const int64_t *cells,
          double *f, const double *fb)
{
    const int n = m->p + 1, dim = m->dim, Nd = ipow(n, dim);
    const int64_t ncell = mesh_ncells(m);
    if (!cells) nsub = ncell;
    const double theta = 0.5 * dtp;

    double *GLL = (double *)malloc(sizeof(double) * Nd * Nd);
    double *GLR = (double *)malloc(sizeof(double) * 6 * Nd);
    double *A = (double *)malloc(sizeof(double) * Nd * Nd);
    double *B = (double *)malloc(sizeof(double) * Nd * Nd);
    int *piv = (int *)malloc(sizeof(int) * Nd);
    double *rhs = (double *)malloc(sizeof(double) * Nd);
    int64_t *order = (int64_t *)malloc(sizeof(int64_t) * nsub);
    int32_t *slot = (int32_t *)malloc(sizeof(int32_t) * ncell);
    double *fold = (double *)malloc(sizeof(double) * nsub * Nd);
    int rc = or_cell_operator(m, v, GLL, GLR);
    if (rc == 0) rc = or_topo_order(m, v, cells ? nsub : 0, cells, order, NULL);
    if (rc == 0) {
        for (int i = 0; i < Nd; i++)
            for (int j = 0; j < Nd; j++) {
                double id = (i == j) ? 1.0 : 0.0;
                A[i * Nd + j] = id + theta * GLL[i * Nd + j];
                B[i * Nd + j] = id - theta * GLL[i * Nd + j];
            }
        /* one factorisation serves every cell: all cells share Gamma_LL (affine box) */
        if (lu_factor(Nd, A, piv)) rc = -4;
    }
    if (rc == 0) {
        for (int64_t c = 0; c < ncell; c++) slot[c] = cells ? -1 : (int32_t)c;
        if (cells)
            for (int64_t s = 0; s < nsub; s++) slot[cells[s]] = (int32_t)s;
        memcpy(fold, f, sizeof(double) * nsub * Nd);
        for (int64_t k = 0; k < nsub && rc == 0; k++) {
            const int64_t c = order[k];
            const int64_t sc = slot[c];
            const double *fo = fold + sc * Nd;
            for (int i = 0; i < Nd; i++) {
                double acc = 0.0;
                for (int j = 0; j < Nd; j++) acc += B[i * Nd + j] * fo[j];
                rhs[i] = acc;
            }
            for (int d = 0; d < dim; d++)
                for (int side = 0; side < 2; side++) {
                    const int eps = 2 * d + side;
                    const int64_t r = neighbour(m, c, d, side);
                    for (int i = 0; i < Nd; i++) {
                        const double coef = GLR[eps * Nd + i];
                        if (coef == 0.0) continue;
                        double sum;
                        if (r < 0) {
                            sum = 2.0 * fb[sc * Nd + i]; /* ghost: old + new = 2 f^b */
                        } else {
                            const int ip = matched_node(i, n, dim, d);
                            const int64_t sr = slot[r];
                            if (sr < 0) { rc = -2; break; } /* upwind cell outside the subset */
                            sum = fold[sr * Nd + ip] + f[sr * Nd + ip];
                        }
                        rhs[i] -= theta * coef * sum;
                    }
                }
            lu_solve(Nd, A, piv, rhs);
            memcpy(f + sc * Nd, rhs, sizeof(double) * Nd);
        }
    }
    free(GLL); free(GLR); free(A); free(B); free(piv); free(rhs); free(order); free(slot); free(fold);
    return rc;
}

/* T2 for nv velocities over the whole mesh, OpenMP over velocities.
 * f, fb : [nv][ncell][Nd]. */
int or_t2_all(const or_mesh *m, int nv, const double *vel, double dtp, double *f, const double *fb)
{
    const int Nd = ipow(m->p + 1, m->dim);
    const int64_t per = mesh_ncells(m) * Nd;
    int rc = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(min : rc)
    for (int i = 0; i < nv; i++) {
        int r = or_t2(m, vel + 3 * i, dtp, 0, NULL, f + per * i, fb + per * i);
        if (r < rc) rc = r;
    }
    return rc;
}

/*
 * (L_h F) for one velocity: out_L = -Gamma_LL f_L - sum_R Gamma_LR f_R,
 * with f_R = fb on fictitious (boundary) cells.  Used by the pins (constant
 * preservation, polynomial exactness, dissipation, dense CN solve).
 */
int or_apply_L(const or_mesh *m, const double *v, const double *f, const double *fb, double *out)
{
    const int n = m->p + 1, dim = m->dim, Nd = ipow(n, dim);
    const int64_t ncell = mesh_ncells(m);
    double *GLL = (double *)malloc(sizeof(double) * Nd * Nd);
    double *GLR = (double *)malloc(sizeof(double) * 6 * Nd);
    int rc = or_cell_operator(m, v, GLL, GLR);
    for (int64_t c = 0; c < ncell && rc == 0; c++) {
        for (int i = 0; i < Nd; i++) {
            double acc = 0.0;
            for (int j = 0; j < Nd; j++) acc += GLL[i * Nd + j] * f[c * Nd + j];
            for (int d = 0; d < dim; d++)
                for (int side = 0; side < 2; side++) {
                    const double coef = GLR[(2 * d + side) * Nd + i];
                    if (coef == 0.0) continue;
                    const int64_t r = neighbour(m, c, d, side);
                    const double fr = (r < 0) ? fb[c * Nd + i] : f[r * Nd + matched_node(i, n, dim, d)];
                    acc += coef * fr;
                }
            out[c * Nd + i] = -acc;
        }
    }
    free(GLL); free(GLR);
    return rc;
}

/* ------------------------------------------------------------------------- */
/* Kinetic model: moments, flux, equilibrium, collision.                      */
/* ------------------------------------------------------------------------- */
enum { OR_FLUX_ADVECTION = 0, OR_FLUX_EULER = 1, OR_FLUX_ISOTHERMAL = 2, OR_FLUX_LBM = 3 };

/*
 * Lattice-Boltzmann isothermal model (the paper's D2Q9; the same formula
 * for the D3Q15/19/27 lattices of P:856-858): w = P f with P = [1; v^T] (rho = sum f_i,
 * rho u = sum f_i v_i), and
 *   f^eq_i = w_i rho (1 + (u.v_i)/c^2 + (u.v_i)^2/(2 c^4) - (u.u)/(2 c^2))
 * with fp = {c, w_0, ..., w_{nv-1}} (the lattice weights).
 */
static void lbm_moments(int dim, int nv, const double *vel, const double *fnode, double *w)
{
    for (int c = 0; c <= dim; c++) w[c] = 0.0;
    for (int i = 0; i < nv; i++) {
        w[0] += fnode[i];
        for (int d = 0; d < dim; d++) w[1 + d] += fnode[i] * vel[3 * i + d];
    }
}

static void lbm_equilibrium(int dim, int nv, const double *vel, const double *fp, const double *w, double *feq)
{
    const double c = fp[0], c2 = c * c;
    const double rho = w[0];
    double u[3] = { 0, 0, 0 }, uu = 0.0;
    for (int d = 0; d < dim; d++) {
        u[d] = w[1 + d] / rho;
        uu += u[d] * u[d];
    }
    for (int i = 0; i < nv; i++) {
        double uv = 0.0;
        for (int d = 0; d < dim; d++) uv += u[d] * vel[3 * i + d];
        feq[i] = fp[1 + i] * rho * (1.0 + uv / c2 + (uv * uv) / (2.0 * c2 * c2) - uu / (2.0 * c2));
    }
}

/*
 * Physical flux q^k(w), k = 0..dim-1, written to q[k*mm + c] (P:161-172 eq
 * macro_limit_system; the models are the configs' textbook systems):
 *   advection : m = 1,      q^k = a_k w
 *   Euler     : m = dim+2,  w = (rho, rho u, E), p = (gamma-1)(E - rho|u|^2/2),
 *               q^k = (rho u_k, rho u_k u + p e_k, (E + p) u_k)
 *   isothermal: m = dim+1,  w = (rho, rho u), q^k = (rho u_k, rho u_k u + c^2 rho e_k)
 */
int or_flux(int dim, int flux, const double *fp, const double *w, double *q)
{
    if (flux == OR_FLUX_ADVECTION) {
        for (int k = 0; k < dim; k++) q[k] = fp[k] * w[0];
        return 0;
    }
    const double rho = w[0];
    double u[3] = { 0, 0, 0 };
    for (int d = 0; d < dim; d++) u[d] = w[1 + d] / rho;
    if (flux == OR_FLUX_EULER) {
        const int mm = dim + 2;
        const double gamma = fp[0];
        const double E = w[dim + 1];
        double u2 = 0.0;
        for (int d = 0; d < dim; d++) u2 += u[d] * u[d];
        const double pr = (gamma - 1.0) * (E - 0.5 * rho * u2);
        for (int k = 0; k < dim; k++) {
            q[k * mm + 0] = rho * u[k];
            for (int d = 0; d < dim; d++) q[k * mm + 1 + d] = rho * u[k] * u[d] + (d == k ? pr : 0.0);
            q[k * mm + dim + 1] = (E + pr) * u[k];
        }
        return 0;
    }
    if (flux == OR_FLUX_ISOTHERMAL) {
        const int mm = dim + 1;
        const double c2 = fp[0] * fp[0];
        for (int k = 0; k < dim; k++) {
            q[k * mm + 0] = rho * u[k];
            for (int d = 0; d < dim; d++) q[k * mm + 1 + d] = rho * u[k] * u[d] + (d == k ? c2 * rho : 0.0);
        }
        return 0;
    }
    return -1;
}

/*
 * Equilibrium of the vectorial kinetic model (reading C6): velocity i belongs
 * to component c = comp[i]; the 2*dim velocities of a component are +-lambda e_k.
 *   f^eq_i = w_c/(2 dim) + (v_i . q_c(w)) / (2 lambda^2)
 * which is w_c/(2D) +- q^k_c/(2 lambda) for v_i = +-lambda e_k, so that
 * P f^eq = w and sum_i v_i^k f^eq_i = q^k(w).
 */
int or_equilibrium(int dim, int nv, const double *vel, const int32_t *comp, int mm, double lambda,
                   int flux, const double *fp, const double *w, double *feq)
{
    double q[3 * 8];
    if (flux == OR_FLUX_LBM) {
        lbm_equilibrium(dim, nv, vel, fp, w, feq);
        return 0;
    }
    if (mm > 8) return -1;
    if (or_flux(dim, flux, fp, w, q)) return -1;
    for (int i = 0; i < nv; i++) {
        const int c = comp[i];
        double vq = 0.0;
        for (int k = 0; k < dim; k++) vq += vel[3 * i + k] * q[k * mm + c];
        feq[i] = w[c] / (2.0 * dim) + vq / (2.0 * lambda * lambda);
    }
    return 0;
}

/* w = P f for the LBM model (P = [1; v^T]), summed in index order. */
int or_moments_lbm(int dim, int nv, const double *vel, int64_t nnodes, const double *f, double *w)
{
#pragma omp parallel for schedule(static)
    for (int64_t x = 0; x < nnodes; x++) {
        double fl[64], wl[4];
        for (int i = 0; i < nv; i++) fl[i] = f[(int64_t)i * nnodes + x];
        lbm_moments(dim, nv, vel, fl, wl);
        for (int c = 0; c <= dim; c++) w[(int64_t)c * nnodes + x] = wl[c];
    }
    return 0;
}

/* w = P f at every node, P[c][i] = (comp[i] == c), summed in index order.
 * f : [nv][nnodes], w : [mm][nnodes]. */
int or_moments(int nv, const int32_t *comp, int mm, int64_t nnodes, const double *f, double *w)
{
#pragma omp parallel for schedule(static)
    for (int64_t x = 0; x < nnodes; x++) {
        double acc[8] = { 0, 0, 0, 0, 0, 0, 0, 0 };
        for (int i = 0; i < nv; i++) acc[comp[i]] += f[(int64_t)i * nnodes + x];
        for (int c = 0; c < mm; c++) w[(int64_t)c * nnodes + x] = acc[c];
    }
    return 0;
}

/*
 * Collision C2(dt) at every node (eq collision_cn):
 *   f <- ((2 tau - dt) f + 2 dt f^eq(f)) / (2 tau + dt)
 * and for tau = 0 the over-relaxation f <- 2 f^eq - f.
 * f : [nv][nnodes] in/out.
 */
int or_collide(int dim, int nv, const double *vel, const int32_t *comp, int mm, double lambda,
               int flux, const double *fp, double tau, double dt, int64_t nnodes, double *f)
{
    int rc = 0;
#pragma omp parallel for schedule(static) reduction(min : rc)
    for (int64_t x = 0; x < nnodes; x++) {
        double w[8] = { 0, 0, 0, 0, 0, 0, 0, 0 }, feq[64];
        if (flux == OR_FLUX_LBM) {
            double fl[64];
            for (int i = 0; i < nv; i++) fl[i] = f[(int64_t)i * nnodes + x];
            lbm_moments(dim, nv, vel, fl, w);
        } else {
            for (int i = 0; i < nv; i++) w[comp[i]] += f[(int64_t)i * nnodes + x];
        }
        if (or_equilibrium(dim, nv, vel, comp, mm, lambda, flux, fp, w, feq)) { rc = -1; continue; }
        for (int i = 0; i < nv; i++) {
            double *fi = f + (int64_t)i * nnodes + x;
            if (tau == 0.0)
                *fi = 2.0 * feq[i] - *fi;
            else
                *fi = ((2.0 * tau - dt) * *fi + 2.0 * dt * feq[i]) / (2.0 * tau + dt);
        }
    }
    return rc;
}

/* f^eq(w) at every node: w : [mm][nnodes] -> feq : [nv][nnodes] (initial/boundary data, C12/C13). */
int or_equilibrium_field(int dim, int nv, const double *vel, const int32_t *comp, int mm, double lambda,
                         int flux, const double *fp, int64_t nnodes, const double *w, double *feq)
{
    int rc = 0;
#pragma omp parallel for schedule(static) reduction(min : rc)
    for (int64_t x = 0; x < nnodes; x++) {
        double wl[8], fl[64];
        for (int c = 0; c < mm; c++) wl[c] = w[(int64_t)c * nnodes + x];
        if (or_equilibrium(dim, nv, vel, comp, mm, lambda, flux, fp, wl, fl)) { rc = -1; continue; }
        for (int i = 0; i < nv; i++) feq[(int64_t)i * nnodes + x] = fl[i];
    }
    return rc;
}

/* ------------------------------------------------------------------------- */
/* Source step S2 (NEXT-3): the Euler-with-gravity case of P:1101-1194.       */
/* ------------------------------------------------------------------------- */
/*
 * Kinetic source g(f) for the LBM model: the macroscopic source of eq
 * macro_limit_system is s(w) = (0, rho G) with G the gravity vector (P:1104-1108:
 * d_t(rho u) + div Pi = rho g, g = -g e_y), lifted to the kinetic level "on the
 * equilibrium part" by the standard moment-exact forcing
 *   g_i = w_i (s_rho + v_i . s_m / c^2)          (reading C24)
 * so that P g = s (sum w_i = 1, sum w_i v_i = 0, sum w_i v_i v_i^T = c^2 I).
 * fp = {c, w_0 .. w_{nv-1}} as for the LBM model, G[dim] the gravity vector.
 */
static void lbm_source(int dim, int nv, const double *vel, const double *fp, const double *G, const double *fnode,
                       double *g)
{
    const double c = fp[0], c2 = c * c;
    double w[4];
    lbm_moments(dim, nv, vel, fnode, w);
    double sm[3] = { 0, 0, 0 };
    for (int d = 0; d < dim; d++) sm[d] = w[0] * G[d];   /* s = (0, rho G) */
    for (int i = 0; i < nv; i++) {
        double vs = 0.0;
        for (int d = 0; d < dim; d++) vs += vel[3 * i + d] * sm[d];
        g[i] = fp[1 + i] * (0.0 + vs / c2);
    }
}

/*
 * S2(h) = (I + h/2 G_h)(I - h/2 G_h)^{-1} at every node: the
 * theta = 1/2 implicit local equation f* = f + h/2 (g(f) + g(f*)) solved by Picard
 * iteration from f* = f ("converges in one Picard iteration" for the
 * gravity source).  Iterates until the update is below 1e-15 relative, at most 16.
 * f : [nv][nnodes] in/out.  Returns the largest number of Picard iterations used.
 */
int or_source(int dim, int nv, const double *vel, const double *fp, const double *G, double h, int64_t nnodes,
              double *f)
{
    int itmax = 0;
#pragma omp parallel for schedule(static) reduction(max : itmax)
    for (int64_t x = 0; x < nnodes; x++) {
        double f0[64], fs[64], g0[64], gs[64], fn[64];
        for (int i = 0; i < nv; i++) f0[i] = f[(int64_t)i * nnodes + x];
        lbm_source(dim, nv, vel, fp, G, f0, g0);
        for (int i = 0; i < nv; i++) fs[i] = f0[i];
        int it = 0;
        for (it = 1; it <= 16; it++) {
            lbm_source(dim, nv, vel, fp, G, fs, gs);
            double diff = 0.0, scale = 0.0;
            for (int i = 0; i < nv; i++) {
                fn[i] = f0[i] + 0.5 * h * (g0[i] + gs[i]);
                diff = fmax(diff, fabs(fn[i] - fs[i]));
                scale = fmax(scale, fabs(fn[i]));
            }
            for (int i = 0; i < nv; i++) fs[i] = fn[i];
            if (diff <= 1e-15 * scale) break;
        }
        if (it > itmax) itmax = it;
        for (int i = 0; i < nv; i++) f[(int64_t)i * nnodes + x] = fs[i];
    }
    return itmax;
}
