// Host-side tables of the B200 sweep: the 1-D Gauss-Lobatto upwind-DG cell block.
//
// For an axis-aligned velocity v = +-lambda e_k the (p+1)^D x (p+1)^D local block of
// eq. DG_reduit is I (x) B_1D (reading C18), so the implicit CN solve of
// a cell factors into independent 1-D solves along the velocity axis.
// With the n = p+1 nodes of a line ordered in the flow direction and
// kappa = lambda * dt' / h (theta = dt'/2, eq transport_cn; reading C1):
//
//   G  = W^{-1} (D^T W - e_out e_out^T),   D_ab = l_b'(x_a), W = diag(omega)
//   A  = I - kappa G
//   f_new = M f_old + g s_in,  M = A^{-1}(I + kappa G),  g = A^{-1} (kappa/omega_0) e_in
//   s_out = f_old[n-1] + f_new[n-1]      (upwind trace, old + new: reading C4)
//
// and the carry obeys s_out = a + beta s_in with beta = g[n-1].  The paper refactorises
// a KLU system per step; dt and v are constant, so one precomputed block
// per (axis, dt') is the same linear algebra.
//
// Computed in long double and rounded once to double.  Independent of oracle/.
#pragma once
#include <cmath>
#include <cstring>
#include <utility>
#include <vector>

namespace pdg {

constexpr int kMaxN = 4;  // p <= 3

struct CellBlock {
    double M[kMaxN * kMaxN];
    double g[kMaxN];
    double beta;
    int n;
};

// Gauss-Lobatto nodes / weights on [-1, 1] for p = 1..3.
inline bool gl_nodes(int p, long double *x, long double *w)
{
    if (p == 1) {
        x[0] = -1.0L; x[1] = 1.0L;
        w[0] = 1.0L; w[1] = 1.0L;
        return true;
    }
    if (p == 2) {
        x[0] = -1.0L; x[1] = 0.0L; x[2] = 1.0L;
        w[0] = 1.0L / 3.0L; w[1] = 4.0L / 3.0L; w[2] = 1.0L / 3.0L;
        return true;
    }
    if (p == 3) {
        const long double r = 1.0L / sqrtl(5.0L);
        x[0] = -1.0L; x[1] = -r; x[2] = r; x[3] = 1.0L;
        w[0] = 1.0L / 6.0L; w[1] = 5.0L / 6.0L; w[2] = 5.0L / 6.0L; w[3] = 1.0L / 6.0L;
        return true;
    }
    return false;
}

// Lagrange derivative matrix D_ab = l_b'(x_a) in barycentric form.
inline void lagrange_derivative(int n, const long double *x, long double *D)
{
    long double bw[kMaxN];
    for (int b = 0; b < n; ++b) {
        long double prod = 1.0L;
        for (int j = 0; j < n; ++j)
            if (j != b) prod *= (x[b] - x[j]);
        bw[b] = 1.0L / prod;
    }
    for (int a = 0; a < n; ++a) {
        long double diag = 0.0L;
        for (int b = 0; b < n; ++b) {
            if (b == a) continue;
            D[a * n + b] = (bw[b] / bw[a]) / (x[a] - x[b]);
            diag -= D[a * n + b];
        }
        D[a * n + a] = diag;
    }
}

// Gauss-Jordan inverse with partial pivoting; false if singular.
inline bool invert(int n, const long double *A, long double *Ainv)
{
    long double T[kMaxN][2 * kMaxN];
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < 2 * n; ++j) T[i][j] = (j < n) ? A[i * n + j] : ((j - n == i) ? 1.0L : 0.0L);
    for (int c = 0; c < n; ++c) {
        int piv = c;
        for (int r = c + 1; r < n; ++r)
            if (fabsl(T[r][c]) > fabsl(T[piv][c])) piv = r;
        if (T[piv][c] == 0.0L) return false;
        if (piv != c)
            for (int j = 0; j < 2 * n; ++j) { long double t = T[c][j]; T[c][j] = T[piv][j]; T[piv][j] = t; }
        const long double d = T[c][c];
        for (int j = 0; j < 2 * n; ++j) T[c][j] /= d;
        for (int r = 0; r < n; ++r) {
            if (r == c || T[r][c] == 0.0L) continue;
            const long double fac = T[r][c];
            for (int j = 0; j < 2 * n; ++j) T[r][j] -= fac * T[c][j];
        }
    }
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) Ainv[i * n + j] = T[i][n + j];
    return true;
}

// The cell block for degree p and CN parameter kappa (any sign).
inline bool cell_block(int p, long double kappa, CellBlock *out)
{
    long double x[kMaxN], w[kMaxN], D[kMaxN * kMaxN], G[kMaxN * kMaxN], A[kMaxN * kMaxN], Ai[kMaxN * kMaxN];
    if (!gl_nodes(p, x, w)) return false;
    const int n = p + 1;
    lagrange_derivative(n, x, D);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            long double v = D[j * n + i] * w[j];                // (D^T W)_ij
            if (i == n - 1 && j == n - 1) v -= 1.0L;            // - e_out e_out^T
            G[i * n + j] = v / w[i];                            // W^{-1} (...)
            A[i * n + j] = ((i == j) ? 1.0L : 0.0L) - kappa * G[i * n + j];
        }
    if (!invert(n, A, Ai)) return false;
    std::memset(out, 0, sizeof(*out));
    out->n = n;
    for (int i = 0; i < n; ++i) {
        for (int j = 0; j < n; ++j) {
            long double acc = 0.0L;  // A^{-1} (I + kappa G)
            for (int k = 0; k < n; ++k) acc += Ai[i * n + k] * (((k == j) ? 1.0L : 0.0L) + kappa * G[k * n + j]);
            out->M[i * n + j] = (double)acc;
        }
        out->g[i] = (double)(Ai[i * n + 0] * kappa / w[0]);
    }
    out->beta = out->g[n - 1];
    return true;
}


// ---------------------------------------------------------------------------
// Dense local block of a lattice velocity (NEXT-2: non-axis-aligned sets such as
// D2Q9, D3Q15/19/27).  For v with components in {0, +-lambda}
// on an axis-aligned Cartesian cell the DG_reduit block is the Kronecker
// SUM over the active axes t (v_t != 0) of kappa_t G (nodes in flow order along every
// active axis; inactive axes decouple: I on their nodes), with kappa_t = |v_t| dt'/h_t:
//
//   A = I - sum_t kappa_t G^(t),   rhs = (I + sum_t kappa_t G^(t)) f_old + sum_t (kappa_t/omega_0) E_in^(t) s_t
//   f_new = A^{-1} rhs,            s_t^out = f_old[out face t] + f_new[out face t]
//
// A^{-1} is dense (n^d x n^d, d = number of active axes): the "pre-inverted local block"
// of the north star.  Reduced node r = sum_t a_t n^t (t = 0 the lowest active axis).
// For the x-scan (axis t = 0 active): Qx = A^{-1} E_in^(0) kappa_0/omega_0 (n^d x n^{d-1}),
// Bx = rows of Qx on the x-out face (n^{d-1} square) and its powers Bx^(2^j).
// ---------------------------------------------------------------------------
struct LatticeBlockLD {
    int n = 0, d = 0, nb = 0, mf = 0;
    long double G[kMaxN * kMaxN];            // 1-D G in flow order (positive velocity)
    long double kappa[3];                    // per active axis
    long double w0;                          // omega_0
    std::vector<long double> Ainv;           // nb x nb
    std::vector<long double> M;              // nb x nb: A^{-1} (I + sum_t kappa_t G^(t))
    std::vector<long double> Q;              // d x nb x mf: A^{-1} E_in^(t) kappa_t / omega_0
    std::vector<long double> Qx;             // nb x mf (= Q of t = 0)
    std::vector<long double> Bpow;           // 5 x mf x mf
};

inline bool invert_dense(int n, std::vector<long double> A, std::vector<long double> &Ainv)
{
    Ainv.assign((size_t)n * n, 0.0L);
    for (int i = 0; i < n; ++i) Ainv[(size_t)i * n + i] = 1.0L;
    for (int c = 0; c < n; ++c) {
        int piv = c;
        for (int r = c + 1; r < n; ++r)
            if (fabsl(A[(size_t)r * n + c]) > fabsl(A[(size_t)piv * n + c])) piv = r;
        if (A[(size_t)piv * n + c] == 0.0L) return false;
        if (piv != c)
            for (int j = 0; j < n; ++j) {
                std::swap(A[(size_t)c * n + j], A[(size_t)piv * n + j]);
                std::swap(Ainv[(size_t)c * n + j], Ainv[(size_t)piv * n + j]);
            }
        const long double dd = A[(size_t)c * n + c];
        for (int j = 0; j < n; ++j) {
            A[(size_t)c * n + j] /= dd;
            Ainv[(size_t)c * n + j] /= dd;
        }
        for (int r = 0; r < n; ++r) {
            if (r == c || A[(size_t)r * n + c] == 0.0L) continue;
            const long double fac = A[(size_t)r * n + c];
            for (int j = 0; j < n; ++j) {
                A[(size_t)r * n + j] -= fac * A[(size_t)c * n + j];
                Ainv[(size_t)r * n + j] -= fac * Ainv[(size_t)c * n + j];
            }
        }
    }
    return true;
}

// d active axes with CN parameters kappa[0..d-1] (lowest axis first).
inline bool lattice_block(int p, int d, const long double *kappa, LatticeBlockLD *out)
{
    long double x[kMaxN], w[kMaxN], D[kMaxN * kMaxN];
    if (!gl_nodes(p, x, w) || d < 1 || d > 3) return false;
    const int n = p + 1;
    lagrange_derivative(n, x, D);
    LatticeBlockLD &B = *out;
    B.n = n;
    B.d = d;
    B.nb = 1;
    for (int t = 0; t < d; ++t) B.nb *= n;
    B.mf = B.nb / n;
    B.w0 = w[0];
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            long double v = D[j * n + i] * w[j];
            if (i == n - 1 && j == n - 1) v -= 1.0L;
            B.G[i * n + j] = v / w[i];
        }
    for (int t = 0; t < 3; ++t) B.kappa[t] = (t < d) ? kappa[t] : 0.0L;
    const int nb = B.nb;
    std::vector<long double> A((size_t)nb * nb, 0.0L);
    int pw[4] = {1, n, n * n, n * n * n};
    for (int r = 0; r < nb; ++r) {
        A[(size_t)r * nb + r] += 1.0L;
        for (int t = 0; t < d; ++t) {
            const int at = (r / pw[t]) % n;
            for (int b = 0; b < n; ++b) {
                const int c = r + (b - at) * pw[t];
                A[(size_t)r * nb + c] -= B.kappa[t] * B.G[at * n + b];
            }
        }
    }
    if (!invert_dense(nb, A, B.Ainv)) return false;
    const int mf = B.mf;
    // M = A^{-1} (2 I - A): the explicit half (I + sum kappa G) pre-multiplied
    B.M.assign((size_t)nb * nb, 0.0L);
    for (int r = 0; r < nb; ++r)
        for (int c = 0; c < nb; ++c) {
            long double acc = 0.0L;
            for (int k = 0; k < nb; ++k) acc += B.Ainv[(size_t)r * nb + k] * (((k == c) ? 2.0L : 0.0L) - A[(size_t)k * nb + c]);
            B.M[(size_t)r * nb + c] = acc;
        }
    // inflow responses: in-face node j of axis t = reduced node with digit t = 0
    B.Q.assign((size_t)d * nb * mf, 0.0L);
    for (int t = 0; t < d; ++t)
        for (int r = 0; r < nb; ++r)
            for (int j = 0; j < mf; ++j) {
                const int q = (j % pw[t]) + (j / pw[t]) * pw[t + 1];
                B.Q[((size_t)t * nb + r) * mf + j] = B.Ainv[(size_t)r * nb + q] * B.kappa[t] / B.w0;
            }
    B.Qx.assign(B.Q.begin(), B.Q.begin() + (size_t)nb * mf);
    std::vector<long double> Bx((size_t)mf * mf), T((size_t)mf * mf);
    for (int i = 0; i < mf; ++i)
        for (int j = 0; j < mf; ++j) Bx[(size_t)i * mf + j] = B.Qx[(size_t)(i * n + n - 1) * mf + j];
    B.Bpow.assign((size_t)5 * mf * mf, 0.0L);
    for (int s = 0; s < 5; ++s) {
        for (size_t q = 0; q < Bx.size(); ++q) B.Bpow[(size_t)s * mf * mf + q] = Bx[q];
        for (int i = 0; i < mf; ++i)
            for (int j = 0; j < mf; ++j) {
                long double acc = 0.0L;
                for (int k = 0; k < mf; ++k) acc += Bx[(size_t)i * mf + k] * Bx[(size_t)k * mf + j];
                T[(size_t)i * mf + j] = acc;
            }
        Bx = T;
    }
    return true;
}

}  // namespace pdg
