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
#include <algorithm>
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

// small dense helpers of lattice_chain_halo (row-major mf x mf, long double)
inline void lat_mm(int mf, const long double *A, const long double *B, long double *C)
{
    for (int i = 0; i < mf; ++i)
        for (int j = 0; j < mf; ++j) {
            long double a = 0.0L;
            for (int k = 0; k < mf; ++k) a += A[i * mf + k] * B[k * mf + j];
            C[i * mf + j] = a;
        }
}
inline long double lat_ninf(int mf, const long double *A)
{
    long double m = 0.0L;
    for (int i = 0; i < mf; ++i) {
        long double r = 0.0L;
        for (int j = 0; j < mf; ++j) r += fabsl(A[i * mf + j]);
        m = std::max(m, r);
    }
    return m;
}
// sum of the block norms of a block sequence (an upper bound of its Toeplitz operator's inf-norm)
inline long double lat_norm_seq(int mf, const std::vector<long double> &A)
{
    const size_t s = (size_t)mf * mf;
    long double r = 0.0L;
    for (size_t m = 0; m < A.size() / s; ++m) r += lat_ninf(mf, A.data() + m * s);
    return r;
}
// block sequence convolution (product of block lower-triangular Toeplitz operators)
inline std::vector<long double> lat_conv(int mf, const std::vector<long double> &A, const std::vector<long double> &B)
{
    const size_t s = (size_t)mf * mf, la = A.size() / s, lb = B.size() / s;
    std::vector<long double> C((la + lb - 1) * s, 0.0L), c(s);
    for (size_t a = 0; a < la; ++a)
        for (size_t b = 0; b < lb; ++b) {
            lat_mm(mf, A.data() + a * s, B.data() + b * s, c.data());
            for (size_t i = 0; i < s; ++i) C[(a + b) * s + i] += c[i];
        }
    return C;
}

// Chain truncation depth of a lattice sweep whose x axis (active index 0) and chain axis
// (active index tc) are the block's only coupled directions (classes without a pipe axis).
//
// Sweeping rows r0, r0+1, ... of the chain with a ZERO chain in-trace at r0 instead of the
// true one leaves an error e in the chain in-traces of row r0 that the sweep carries as
// e_{r+1} = T e_r, where T maps the chain in-traces of a whole row (x = 0, 1, ...; exact x
// inflow at x = 0) to its chain out-traces: a block lower-triangular Toeplitz operator with
// blocks T_0 = Y (chain in -> chain out of the same cell) and T_m = X_i B_x^{m-1} X_o (chain in
// -> x out, m-1 cells of x hand-over, x in -> chain out), all rows of the block's inflow
// responses Q.  ||T^k||_inf <= sum_m ||(T^k)_m||_inf; the sequence is truncated once
// ||B_x^j X_o|| < 2^-100 ||X_o|| and the tail is bounded with S = sum_i ||B_x^i|| (from a
// power of B_x with norm < 1/2) and ||(A+E)^k - A^k|| <= k ||E|| (||A|| + ||E||)^(k-1).
// Returns the smallest H (a multiple of k in {1, 4}) with ||T^H|| <= 2^-64, i.e. after H rows
// the computed traces differ from the exact sweep's by at most 2^-64 of the true in-traces
// (below the fp64 rounding of every later row), or -1 when no such H <= hmax exists.
inline int lattice_chain_halo(const LatticeBlockLD &B, int tc, int hmax)
{
    typedef long double LD;
    const int n = B.n, nb = B.nb, mf = B.mf, s = mf * mf;
    if (B.d < 2 || tc < 1 || tc >= B.d) return -1;
    auto outq = [&](int t, int j) {  // node of reduced index j on the out-face of active axis t
        int pw = 1;
        for (int i = 0; i < t; ++i) pw *= n;
        return (j % pw) + (j / pw) * pw * n + (n - 1) * pw;
    };
    std::vector<LD> Y(s), Xo(s), Xi(s), Bx(s), t1(s), t2(s);
    for (int i = 0; i < mf; ++i)
        for (int j = 0; j < mf; ++j) {
            Y[i * mf + j] = B.Q[((size_t)tc * nb + outq(tc, i)) * mf + j];
            Xo[i * mf + j] = B.Q[((size_t)tc * nb + outq(0, i)) * mf + j];
            Xi[i * mf + j] = B.Q[((size_t)0 * nb + outq(tc, i)) * mf + j];
            Bx[i * mf + j] = B.Q[((size_t)0 * nb + outq(0, i)) * mf + j];
        }
    // S >= sum_i ||Bx^i||: partial sum up to a power j0 with ||Bx^j0|| = q < 1/2, divided by 1 - q
    LD S = 0.0L, q = 1.0L;
    {
        std::vector<LD> P(s, 0.0L);
        for (int i = 0; i < mf; ++i) P[i * mf + i] = 1.0L;
        int j = 0;
        for (; j < 4096; ++j) {
            q = lat_ninf(mf, P.data());
            if (q < 0.5L && j > 0) break;
            S += q;
            lat_mm(mf, Bx.data(), P.data(), t1.data());
            P = t1;
        }
        if (j == 4096) return -1;
        S /= (1.0L - q);
    }
    // T_m for m < M, and the tail bound E >= sum_{m >= M} ||T_m||
    std::vector<LD> T(Y);
    std::vector<LD> P(Xo);
    const LD xo = lat_ninf(mf, Xo.data()), xi = lat_ninf(mf, Xi.data());
    LD tail = 0.0L;
    for (int m = 1;; ++m) {
        if (lat_ninf(mf, P.data()) <= 0x1p-100L * xo) {
            tail = xi * S * lat_ninf(mf, P.data());
            break;
        }
        if (m > 512) return -1;  // slow decay along x: the halo would not pay anyway
        lat_mm(mf, Xi.data(), P.data(), t1.data());
        T.insert(T.end(), t1.begin(), t1.end());
        lat_mm(mf, Bx.data(), P.data(), t2.data());
        P = t2;
    }
    const LD r1 = lat_norm_seq(mf, T) + tail;  // ||T||
    const std::vector<LD> T2 = lat_conv(mf, T, T);
    const std::vector<LD> T4 = lat_conv(mf, T2, T2);
    const LD r4 = lat_norm_seq(mf, T4) + 4.0L * tail * powl(r1, 3.0L);  // ||T^4||
    int best = -1;
    if (r1 < 1.0L) best = (int)ceill(64.0L / -log2l(r1));
    if (r4 < 1.0L) {
        const int h4 = 4 * (int)ceill(64.0L / -log2l(r4));
        if (best < 0 || h4 < best) best = h4;
    }
    return (best > 0 && best <= hmax) ? best : -1;
}

}  // namespace pdg
