// sm_100a kernels of the PDG hot path (arxiv 1702.00169).  See DESIGN.md for the
// roofline of each kernel and the data layout.
//
//  * sweep_strided_kernel : T2(dt') for velocities along a
//    non-contiguous axis (y, z).  One thread owns one node line along the velocity
//    axis and walks it downwind carrying the scalar upwind trace s (register carry);
//    consecutive threads own consecutive X columns -> 256-byte coalesced warp
//    accesses.  Loads of future cells do not depend on the carry and are software-
//    prefetched PF cells ahead (PF = 2 for n = 3 measured best on B200: occupancy beats
//    per-thread depth; tools/microbench_strided.cu).
//  * sweep_x_kernel : T2(dt') for velocities along the contiguous axis x.  One warp
//    owns one line; lanes are 32 consecutive cells of a chunk staged through shared
//    memory with coalesced loads.  The carry recurrence s_l = a_l + beta s_{l-1} is
//    solved by a 5-step warp-shuffle affine scan; lane 31 chains chunks.
//  * relax_kernel : collision C2 fused with the moment reduction: per
//    node read the n_v SoA streams, w = P f, q(w), f^eq, f <- ca f + cb f^eq.
//  * NPASS = 2 variants apply T2 twice in one pass over memory (step n's trailing
//    and step n+1's leading T2(dt/2): two sweeps, identical arithmetic, not the
//    collapsed scheme of P:1173-1177).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "pdg_check.cuh"

namespace pdg {

constexpr int kMaxVel = 32;

struct DevBlock {
    double M[16];
    double g[4];
};

struct SweepVel {
    int64_t f_off;    // element offset of this velocity's node grid in f
    int64_t fb_off;   // element offset of its inflow plane in fb
    int64_t inner;    // element stride along the velocity axis
    int64_t nlines;   // lines along the axis
    int32_t ncells;   // cells along the axis
    int32_t sign;     // +1: walk upward, -1: walk downward
    int32_t axis;
    int32_t vel;        // global velocity index
    int64_t cout_off;   // >= 0: write the outgoing carry of pass q at cout[cout_off + q*nlines + line]
    int32_t zero_inflow;  // 1: the line starts inside the domain (z-slab pre-pass): inflow carry 0
    int32_t pad;
    int64_t cin_off;    // >= 0: the inflow carry of pass q is cin[cin_off + q*nlines + line] (z-slab:
                        // the exact slab inflow from the carry scan), else 2 f^b (or 0, zero_inflow)
};

struct SweepParams {
    double *f;
    const double *fb;
    double *cout;     // outgoing carries of slab sweeps (z-slab decomposition)
    const double *cin;  // exact slab inflow carries (z-slab decomposition)
    int64_t f_elems, fb_elems, cout_elems, cin_elems;  // buffer bounds (checked build)
    DevBlock blk[3];  // per axis (kappa_k = lambda dt' / h_k)
    int32_t nvel;
    int32_t l2keep;   // 1: f fits in L2 -- keep it resident (evict-normal), else stream it (evict-first)
    SweepVel v[kMaxVel];
};

// L2 policy of the one-pass accesses to f: evict-first (streaming) when f is far larger than the
// L2, evict-normal when f fits in it (config 2: f = 75 MB of the 126 MB L2 then stays resident
// from one pass to the next: 53.8 -> 46.9 us per step; evict-last measured 1 % faster still, not
// taken: it would outlive the solver's passes in a shared L2).  One code path: the policy is a
// register operand of the access.
__device__ __forceinline__ uint64_t l2_policy(int keep)
{
    uint64_t pol;
    if (keep) asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    else asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ double ld_pol(const double *p, uint64_t pol)
{
    double v;
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}

__device__ __forceinline__ void st_pol(double *p, double v, uint64_t pol)
{
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}


enum { MODEL_ADV = 0, MODEL_EULER = 1, MODEL_ISO = 2 };

struct ModelParams {
    double a[3];      // advection speeds
    double gamma;     // Euler
    double c2;        // isothermal c^2
    double inv2D;     // 1/(2D)
    double inv2lam;   // 1/(2 lambda)
};

template <int DIM, int MODEL>
struct Model;

template <int DIM>
struct Model<DIM, MODEL_ADV> {
    static constexpr int M = 1;
    __device__ __forceinline__ static void flux(const double *w, double (&q)[DIM][M], const ModelParams &P)
    {
#pragma unroll
        for (int k = 0; k < DIM; ++k) q[k][0] = P.a[k] * w[0];
    }
    __device__ __forceinline__ static double density(const double *w) { return 1.0; }
};

template <int DIM>
struct Model<DIM, MODEL_EULER> {
    static constexpr int M = DIM + 2;
    __device__ __forceinline__ static void flux(const double *w, double (&q)[DIM][M], const ModelParams &P)
    {
        const double rho = w[0];
        const double inv = 1.0 / rho;
        double u[DIM];
        double ke = 0.0;
#pragma unroll
        for (int d = 0; d < DIM; ++d) {
            u[d] = w[1 + d] * inv;
            ke += w[1 + d] * u[d];
        }
        const double E = w[DIM + 1];
        const double p = (P.gamma - 1.0) * (E - 0.5 * ke);
#pragma unroll
        for (int k = 0; k < DIM; ++k) {
            q[k][0] = w[1 + k];
#pragma unroll
            for (int d = 0; d < DIM; ++d) q[k][1 + d] = w[1 + k] * u[d] + (d == k ? p : 0.0);
            q[k][DIM + 1] = (E + p) * u[k];
        }
    }
    __device__ __forceinline__ static double density(const double *w) { return w[0]; }
};

template <int DIM>
struct Model<DIM, MODEL_ISO> {
    static constexpr int M = DIM + 1;
    __device__ __forceinline__ static void flux(const double *w, double (&q)[DIM][M], const ModelParams &P)
    {
        const double rho = w[0];
        const double inv = 1.0 / rho;
        double u[DIM];
#pragma unroll
        for (int d = 0; d < DIM; ++d) u[d] = w[1 + d] * inv;
        const double prs = P.c2 * rho;
#pragma unroll
        for (int k = 0; k < DIM; ++k) {
            q[k][0] = w[1 + k];
#pragma unroll
            for (int d = 0; d < DIM; ++d) q[k][1 + d] = w[1 + k] * u[d] + (d == k ? prs : 0.0);
        }
    }
    __device__ __forceinline__ static double density(const double *w) { return w[0]; }
};

// f^eq of velocity i = c*2D + 2k + s (reading C6): w_c/(2D) +- q^k_c/(2 lambda)
template <int DIM, int M>
__device__ __forceinline__ double feq_of(int i, const double *w, const double (&q)[DIM][M], const ModelParams &P)
{
    const int c = i / (2 * DIM);
    const int k = (i % (2 * DIM)) >> 1;
    const double sq = (i & 1) ? -q[k][c] : q[k][c];
    return fma(sq, P.inv2lam, w[c] * P.inv2D);
}

// ---------------------------------------------------------------------------
// T2 sweep along a strided axis (y or z): thread per line, register carry.
// ---------------------------------------------------------------------------
template <int N, int NPASS, int PF>
__global__ void __launch_bounds__(256) sweep_strided_kernel(const SweepParams P)
{
    const SweepVel V = P.v[blockIdx.y];
    const int64_t line = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (line >= V.nlines) return;
    const int64_t Lk = (int64_t)V.ncells * N;
    const int64_t base = (line / V.inner) * (V.inner * Lk) + (line % V.inner);
    const int64_t step = (V.sign > 0) ? V.inner : -V.inner;
    const int64_t p_at = V.f_off + base + ((V.sign > 0) ? 0 : (Lk - 1) * V.inner);  // element index of p
    double *p = P.f + p_at;
    // the line's first and last nodes bound every access of the walk
    PDG_CHECK_IDX(p_at, P.f_elems, "sweep_strided f");
    PDG_CHECK_IDX(p_at + (Lk - 1) * step, P.f_elems, "sweep_strided f");

    double M[N * N], g[N];
#pragma unroll
    for (int i = 0; i < N * N; ++i) M[i] = P.blk[V.axis].M[i];
#pragma unroll
    for (int i = 0; i < N; ++i) g[i] = P.blk[V.axis].g[i];

    double carry[NPASS];
    if (V.cin_off >= 0) {
        // a z-slab that does not touch the inflow boundary: the exact inflows from the carry scan
#pragma unroll
        for (int q = 0; q < NPASS; ++q) {
            PDG_CHECK_IDX(V.cin_off + q * V.nlines + line, P.cin_elems, "sweep_strided cin");
            carry[q] = P.cin[V.cin_off + q * V.nlines + line];
        }
    } else {
        // ghost cell: f^b old + f^b new (reading C5)
        PDG_CHECK_IDX(V.fb_off + line, P.fb_elems, "sweep_strided fb");
        const double s0 = 2.0 * P.fb[V.fb_off + line];
#pragma unroll
        for (int q = 0; q < NPASS; ++q) carry[q] = s0;
    }

    // ring of PF prefetched cells (values in flow order).  The walk advances a load pointer and a
    // store pointer by one cell (N step elements); node a of a cell is at a fixed offset a step
    // (fewer integer instructions per node than recomputing 64-bit indices: the kernel runs under
    // the power cap next to the fused pass)
    const int64_t cstep = (int64_t)N * step;
    int64_t off[N];
#pragma unroll
    for (int a = 0; a < N; ++a) off[a] = (int64_t)a * step;
    double ring[PF][N];
#pragma unroll
    for (int k = 0; k < PF; ++k)
        if (k < V.ncells) {
#pragma unroll
            for (int a = 0; a < N; ++a) ring[k][a] = __ldcs(p + k * cstep + off[a]);
        }
    const double *lp = p + PF * cstep;  // the cell PF ahead of the one being updated
    double *sp = p;
    auto cell = [&](double (&fo)[N]) {
#pragma unroll
        for (int q = 0; q < NPASS; ++q) {
            double fn[N];
#pragma unroll
            for (int a = 0; a < N; ++a) {
                double acc = g[a] * carry[q];
#pragma unroll
                for (int b = 0; b < N; ++b) acc = fma(M[a * N + b], fo[b], acc);
                fn[a] = acc;
            }
            carry[q] = fo[N - 1] + fn[N - 1];
#pragma unroll
            for (int a = 0; a < N; ++a) fo[a] = fn[a];
        }
#pragma unroll
        for (int a = 0; a < N; ++a) __stcs(sp + off[a], fo[a]);
        sp += cstep;
    };
    const int nfull = (V.ncells / PF) * PF;
    for (int c0 = 0; c0 < nfull; c0 += PF) {
#pragma unroll
        for (int k = 0; k < PF; ++k) {
            double fo[N];
#pragma unroll
            for (int a = 0; a < N; ++a) fo[a] = ring[k][a];
            if (c0 + k + PF < V.ncells) {
#pragma unroll
                for (int a = 0; a < N; ++a) ring[k][a] = __ldcs(lp + off[a]);
            }
            lp += cstep;
            cell(fo);
        }
    }
#pragma unroll
    for (int k = 0; k < PF; ++k)  // ragged tail: the last ncells % PF cells, already in the ring
        if (nfull + k < V.ncells) {
            double fo[N];
#pragma unroll
            for (int a = 0; a < N; ++a) fo[a] = ring[k][a];
            cell(fo);
        }
    if (V.cout_off >= 0) {
#pragma unroll
        for (int q = 0; q < NPASS; ++q) {
            PDG_CHECK_IDX(V.cout_off + q * V.nlines + line, P.cout_elems, "sweep_strided cout");
            P.cout[V.cout_off + q * V.nlines + line] = carry[q];
        }
    }
}

// ---------------------------------------------------------------------------
// Segmented T2 sweep along a strided axis, for grids with too few lines to fill the GPU
// (e.g. 2-D config 2: 6144 y-lines).  Block = 32 consecutive lines (lanes, coalesced)
// x nseg segments (threadIdx.y).  Per pass: each thread walks its segment with zero
// inflow to get s_out = A + B s_in (B = beta^cells), the true segment inflows follow by
// composing the affine maps of the upstream segments (shared memory), then the segment
// is walked again with the exact recurrence.  Re-reads the data (L2-resident sizes).
// ---------------------------------------------------------------------------
template <int N, int NPASS>
__global__ void __launch_bounds__(1024) sweep_strided_seg_kernel(const SweepParams P, int nseg)
{
    __shared__ double sA[32][33], sB[32][33];
    const SweepVel V = P.v[blockIdx.y];
    const int lane = threadIdx.x, sg = threadIdx.y;
    const int64_t line = (int64_t)blockIdx.x * 32 + lane;
    const bool active = line < V.nlines;
    const int64_t Lk = (int64_t)V.ncells * N;
    const int64_t ln = active ? line : 0;
    const int64_t base = (ln / V.inner) * (V.inner * Lk) + (ln % V.inner);
    const int64_t step = (V.sign > 0) ? V.inner : -V.inner;
    const int64_t p_at = V.f_off + base + ((V.sign > 0) ? 0 : (Lk - 1) * V.inner);
    double *p0 = P.f + p_at;
    if (active) {
        PDG_CHECK_IDX(p_at, P.f_elems, "sweep_strided_seg f");
        PDG_CHECK_IDX(p_at + (Lk - 1) * step, P.f_elems, "sweep_strided_seg f");
        if (V.cin_off < 0) PDG_CHECK_IDX(V.fb_off + line, P.fb_elems, "sweep_strided_seg fb");
        else PDG_CHECK_IDX(V.cin_off + (NPASS - 1) * V.nlines + line, P.cin_elems, "sweep_strided_seg cin");
    }
    const int ks = (V.ncells + nseg - 1) / nseg;
    const int c0 = min(V.ncells, sg * ks), c1 = min(V.ncells, c0 + ks);

    double M[N * N], g[N];
#pragma unroll
    for (int i = 0; i < N * N; ++i) M[i] = P.blk[V.axis].M[i];
#pragma unroll
    for (int i = 0; i < N; ++i) g[i] = P.blk[V.axis].g[i];
    const double beta = g[N - 1];
    const double s0 = (active && V.cin_off < 0) ? 2.0 * P.fb[V.fb_off + line] : 0.0;  // ghost: f^b old + new

#pragma unroll
    for (int q = 0; q < NPASS; ++q) {
        double A = 0.0, B = 1.0;
        if (active) {
            for (int c = c0; c < c1; ++c) {
                double fo[N];
#pragma unroll
                for (int a = 0; a < N; ++a) fo[a] = p0[((int64_t)c * N + a) * step];
                double r = fo[N - 1];
#pragma unroll
                for (int b = 0; b < N; ++b) r = fma(M[(N - 1) * N + b], fo[b], r);
                A = fma(beta, A, r);
                B *= beta;
            }
        }
        sA[sg][lane] = A;
        sB[sg][lane] = B;
        __syncthreads();
        // inflow of pass q: the ghost, or the exact z-slab inflow of the carry scan
        double s = (active && V.cin_off >= 0) ? P.cin[V.cin_off + q * V.nlines + line] : s0;
        for (int j = 0; j < sg; ++j) s = fma(sB[j][lane], s, sA[j][lane]);
        if (active) {
            for (int c = c0; c < c1; ++c) {
                double fo[N], fn[N];
#pragma unroll
                for (int a = 0; a < N; ++a) fo[a] = p0[((int64_t)c * N + a) * step];
#pragma unroll
                for (int a = 0; a < N; ++a) {
                    double acc = g[a] * s;
#pragma unroll
                    for (int b = 0; b < N; ++b) acc = fma(M[a * N + b], fo[b], acc);
                    fn[a] = acc;
                }
                s = fo[N - 1] + fn[N - 1];
#pragma unroll
                for (int a = 0; a < N; ++a) p0[((int64_t)c * N + a) * step] = fn[a];
            }
            if (V.cout_off >= 0 && c1 == V.ncells && c0 < c1) {
                PDG_CHECK_IDX(V.cout_off + q * V.nlines + line, P.cout_elems, "sweep_strided_seg cout");
                P.cout[V.cout_off + q * V.nlines + line] = s;
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Warp sweep of one line held in shared memory (the lane-segment affine scan).
// ---------------------------------------------------------------------------
// The NPASS passes over one chunk of 32 lane segments: v[kk] = the lane's cells in flow order
// (cnt of them hold data), carry[q] = the inflow of the chunk in pass q (updated to its outflow).
template <int N, int NPASS, int K>
__device__ __forceinline__ void segment_passes(double (&v)[K][N], int cnt, const double (&M)[N * N],
                                               const double (&g)[N], double (&carry)[NPASS], int lane)
{
    const unsigned FULL = 0xffffffffu;
    const double beta = g[N - 1];
#pragma unroll
    for (int q = 0; q < NPASS; ++q) {
        double A = 0.0, B = 1.0;  // zero-inflow carry of the segment: s_out = A + B s_in
#pragma unroll
        for (int kk = 0; kk < K; ++kk) {
            if (kk < cnt) {
                double r = v[kk][N - 1];
#pragma unroll
                for (int b = 0; b < N; ++b) r = fma(M[(N - 1) * N + b], v[kk][b], r);
                A = fma(beta, A, r);
                B *= beta;
            }
        }
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const double Ap = __shfl_up_sync(FULL, A, off);
            const double Bp = __shfl_up_sync(FULL, B, off);
            if (lane >= off) {
                A = fma(B, Ap, A);
                B *= Bp;
            }
        }
        double Ae = __shfl_up_sync(FULL, A, 1);
        double Be = __shfl_up_sync(FULL, B, 1);
        if (lane == 0) {
            Ae = 0.0;
            Be = 1.0;
        }
        double s = fma(Be, carry[q], Ae);
#pragma unroll
        for (int kk = 0; kk < K; ++kk) {
            if (kk < cnt) {
                double fn[N];
#pragma unroll
                for (int a = 0; a < N; ++a) {
                    double acc = g[a] * s;
#pragma unroll
                    for (int b = 0; b < N; ++b) acc = fma(M[a * N + b], v[kk][b], acc);
                    fn[a] = acc;
                }
                s = v[kk][N - 1] + fn[N - 1];
#pragma unroll
                for (int a = 0; a < N; ++a) v[kk][a] = fn[a];
            }
        }
        carry[q] = __shfl_sync(FULL, fma(B, carry[q], A), 31);
    }
}

// Line length a multiple of 32 K cells: every chunk full, lane segment sg = chunk + lane covers the
// padded nodes sg (SEG + 1) + [0, SEG) (upward flow) or, downward, the mirror image; the walk
// direction is compile-time, so every shared-memory index is a per-lane base +- a constant.
template <int N, int NPASS, int K, bool UP>
__device__ __forceinline__ void warp_line_sweep_aligned(double *row, int ncells, const double (&M)[N * N],
                                                        const double (&g)[N], double s0, int lane)
{
    constexpr int SEG = K * N;
    double carry[NPASS];
#pragma unroll
    for (int q = 0; q < NPASS; ++q) carry[q] = s0;
    const int nseg = ncells / K;
    for (int sc = 0; sc < nseg; sc += 32) {
        const int sg = sc + lane;
        double *p = UP ? row + sg * (SEG + 1) : row + (nseg - 1 - sg) * (SEG + 1) + SEG - 1;
        double v[K][N];
#pragma unroll
        for (int kk = 0; kk < K; ++kk)
#pragma unroll
            for (int a = 0; a < N; ++a) v[kk][a] = UP ? p[kk * N + a] : p[-(kk * N + a)];
        segment_passes<N, NPASS, K>(v, K, M, g, carry, lane);
#pragma unroll
        for (int kk = 0; kk < K; ++kk)
#pragma unroll
            for (int a = 0; a < N; ++a) {
                if (UP) p[kk * N + a] = v[kk][a];
                else p[-(kk * N + a)] = v[kk][a];
            }
    }
}

// Warp sweep of one line held in shared memory: lane = segment of K consecutive cells
// (flow order).  Per pass: zero-inflow carry of each segment (s_out = A + B s_in,
// B = beta^cells), a 5-step warp-shuffle affine scan for the true segment inflows,
// then the sequential cell recurrence f_new = M f_old + g s with the true inflow.
// `row` uses padded indexing: element X lives at X + X / (K N).
// ALIGNED: the caller guarantees ncells % (32 K) == 0 (warp_line_sweep_aligned).
template <int N, int NPASS, int K, bool ALIGNED = false>
__device__ __forceinline__ void warp_line_sweep(double *row, int ncells, bool up, const double (&M)[N * N],
                                                const double (&g)[N], double s0, int lane)
{
    if constexpr (ALIGNED) {
        if (up) warp_line_sweep_aligned<N, NPASS, K, true>(row, ncells, M, g, s0, lane);
        else warp_line_sweep_aligned<N, NPASS, K, false>(row, ncells, M, g, s0, lane);
        return;
    }
    constexpr int SEG = K * N;
    double carry[NPASS];
#pragma unroll
    for (int q = 0; q < NPASS; ++q) carry[q] = s0;
    for (int sc0 = 0; sc0 < ncells; sc0 += 32 * K) {
        const int f0 = sc0 + lane * K;
        const int cnt = max(0, min(K, ncells - f0));
        // A full chunk whose lane segments align with the padding segments (always upward; downward
        // when the line length is a multiple of SEG): the lane's K N nodes are contiguous in the padded
        // row at a per-lane base, so every index is base +- a compile-time offset (no division).
        //   up:   X = sc0 N + lane SEG + j,          X + X / SEG = base + j, base = sc0 N + lane SEG + sc0 / K + lane
        //   down: X = SEG q - 1 - j (q = L / SEG - sc0 / K - lane),  X + X / SEG = SEG q + q - 2 - j
        const int Lx = ncells * N;
        const bool fast = (sc0 + 32 * K <= ncells) && (up || Lx % SEG == 0);
        const int q0 = Lx / SEG - sc0 / K - lane;
        const int fbase = up ? sc0 * N + lane * SEG + sc0 / K + lane : SEG * q0 + q0 - 2;
        double v[K][N];
        if (fast) {
#pragma unroll
            for (int kk = 0; kk < K; ++kk)
#pragma unroll
                for (int a = 0; a < N; ++a) v[kk][a] = row[up ? fbase + kk * N + a : fbase - (kk * N + a)];
        } else {
#pragma unroll
            for (int kk = 0; kk < K; ++kk) {
                if (kk < cnt) {
                    const int fc = f0 + kk;
                    const int mc = up ? fc : ncells - 1 - fc;
#pragma unroll
                    for (int a = 0; a < N; ++a) {
                        const int X = mc * N + (up ? a : N - 1 - a);
                        v[kk][a] = row[X + X / SEG];
                    }
                } else {
#pragma unroll
                    for (int a = 0; a < N; ++a) v[kk][a] = 0.0;
                }
            }
        }
        segment_passes<N, NPASS, K>(v, cnt, M, g, carry, lane);
        if (fast) {
#pragma unroll
            for (int kk = 0; kk < K; ++kk)
#pragma unroll
                for (int a = 0; a < N; ++a) row[up ? fbase + kk * N + a : fbase - (kk * N + a)] = v[kk][a];
        } else {
#pragma unroll
            for (int kk = 0; kk < K; ++kk) {
                if (kk < cnt) {
                    const int fc = f0 + kk;
                    const int mc = up ? fc : ncells - 1 - fc;
#pragma unroll
                    for (int a = 0; a < N; ++a) {
                        const int X = mc * N + (up ? a : N - 1 - a);
                        row[X + X / SEG] = v[kk][a];
                    }
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// T2 sweep(s) along a strided axis for grids with few lines (2-D y-velocities: config 2 has
// 6144 y-lines of 768 nodes, too few for the thread-per-line kernel): a CTA stages a tile of
// CW adjacent lines in shared memory (each node row of the tile is CW contiguous doubles:
// coalesced loads and stores, once per pass over f), one warp per line sweeps it with the
// lane-segment affine scan of warp_line_sweep (NPASS sweeps in shared memory), the tile is
// stored back.  Data move once, unlike the segmented kernel's zero-inflow re-reads.
// Requires inner % CW == 0 (a tile's lines are adjacent in memory) and no outgoing-carry output.
// ---------------------------------------------------------------------------
template <int N, int K>
__host__ __device__ constexpr int cols_row_len(int ncells)
{
    return ncells * N + (ncells * N) / (K * N) + 1;
}

constexpr int kColsThreads = 256;

// One tile (CW adjacent lines of one velocity): cp.async of every node into the padded column rows
// (row of line c: node y at c Lp + y + y / SEG).  Thread t always owns column t % CW and rows
// t / CW + i (NT / CW): the global pointer and the row advance by constants (no division per load).
template <int N, int K, int CW>
__device__ __forceinline__ void cols_tile_load(double *buf, const double *g0, int64_t inner, int Lk, int Lp,
                                               uint64_t pol)
{
    constexpr int SEG = K * N, RS = kColsThreads / CW;
    const int cc = threadIdx.x % CW;
    const double *src = g0 + (int64_t)(threadIdx.x / CW) * inner + cc;
    const int64_t step = (int64_t)RS * inner;
    const unsigned sb = (unsigned)__cvta_generic_to_shared(buf + cc * Lp);
#pragma unroll 4
    for (unsigned y = threadIdx.x / CW; y < (unsigned)Lk; y += RS, src += step) {
        const unsigned sa = sb + 8u * (y + y / SEG);
        asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;" ::"r"(sa), "l"(src), "l"(pol)
                     : "memory");
    }
}

template <int N, int K, int CW>
__device__ __forceinline__ void cols_tile_store(const double *buf, double *g0, int64_t inner, int Lk, int Lp,
                                                uint64_t pol)
{
    constexpr int SEG = K * N, RS = kColsThreads / CW;
    const int cc = threadIdx.x % CW;
    double *dst = g0 + (int64_t)(threadIdx.x / CW) * inner + cc;
    const int64_t step = (int64_t)RS * inner;
    const double *sb = buf + cc * Lp;
#pragma unroll 4
    for (unsigned y = threadIdx.x / CW; y < (unsigned)Lk; y += RS, dst += step) st_pol(dst, sb[y + y / SEG], pol);
}

// One tile per CTA (tile t: velocity t / tpv, lines (t % tpv) CW ...).  (A persistent variant with
// two tile buffers, the next tile's loads in flight during the sweep, measured slower on config 2:
// 33.5 against 27.6 us per launch.)  AX: the sweep axis of every velocity of the
// launch (its block is then a compile-time parameter slot, held in uniform registers).
template <int N, int NPASS, int K, int CW, int AX, bool ALIGNED>
__global__ void __launch_bounds__(kColsThreads, 2) sweep_cols_kernel(const SweepParams P, int64_t tpv)
{
    extern __shared__ double scol[];
    PDG_DCHECK(blockDim.x == kColsThreads, "sweep_cols block size", blockDim.x, kColsThreads);
    const int64_t t = blockIdx.x;
    if (t >= tpv * P.nvel) return;
    const SweepVel &V = P.v[t / tpv];
    const int64_t line0 = (t % tpv) * CW;
    const int Lk = V.ncells * N;
    const int Lp = cols_row_len<N, K>(V.ncells);
    const int64_t base = V.f_off + (line0 / V.inner) * (V.inner * Lk) + (line0 % V.inner);
    double *g0 = P.f + base;  // node y of tile line c at g0 + y inner + c
    PDG_CHECK_IDX(base + (int64_t)(Lk - 1) * V.inner + CW - 1, P.f_elems, "sweep_cols f");
    const uint64_t pol = l2_policy(P.l2keep);
    cols_tile_load<N, K, CW>(scol, g0, V.inner, Lk, Lp, pol);
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int nwarps = kColsThreads / 32;
    double M[N * N], g[N];
#pragma unroll
    for (int i = 0; i < N * N; ++i) M[i] = P.blk[AX].M[i];
#pragma unroll
    for (int i = 0; i < N; ++i) g[i] = P.blk[AX].g[i];
    for (int cc = warp; cc < CW; cc += nwarps) {
        PDG_CHECK_IDX(V.fb_off + line0 + cc, P.fb_elems, "sweep_cols fb");
        const double s0 = 2.0 * P.fb[V.fb_off + line0 + cc];  // ghost: f^b old + new (no z-slab entries here)
        warp_line_sweep<N, NPASS, K, ALIGNED>(scol + cc * Lp, V.ncells, V.sign > 0, M, g, s0, lane);
    }
    __syncthreads();
    cols_tile_store<N, K, CW>(scol, g0, V.inner, Lk, Lp, pol);
}

// ---------------------------------------------------------------------------
// Collision fused with the moment reduction AND the following T2 sweep(s) of the
// x-velocities (G = 1).  One CTA per x-line (fixed y, z):
//   phase 1: per node, w = P f, f^eq(w), f <- ca f + cb f^eq for all n_v velocities;
//            y/z velocities go straight back to HBM, x velocities to shared memory;
//   phase 2: one warp per x velocity sweeps the line in shared memory (NPASS times);
//   phase 3: coalesced store of the x velocities.
// HBM traffic = one read + one write of every value (16 B per node.velocity).
// ---------------------------------------------------------------------------
struct RelaxXParams {
    double *f;
    const double *fb;
    int64_t f_elems, fb_elems;  // buffer bounds (checked build)
    int64_t nnodes;
    int64_t plane_stride;
    int32_t ncx;  // cells along x
    DevBlock blk; // x-axis block of the sweeps that follow the collision
    ModelParams mp;
    double ca, cb;
    int32_t l2keep;  // as SweepParams::l2keep
};

template <int N, int K>
__host__ __device__ constexpr int relax_x_row_len(int ncx)
{
    return ncx * N + (ncx * N) / (K * N) + 1;
}

template <int DIM, int MODEL, int N, int NPASS, int K>
__global__ void __launch_bounds__(256) relax_xsweep_kernel(const RelaxXParams P)
{
    using Md = Model<DIM, MODEL>;
    constexpr int M = Md::M;
    constexpr int NV = M * 2 * DIM;
    constexpr int SEG = K * N;
    extern __shared__ double sx[];
    const int Lx = P.ncx * N;
    const int Lp = relax_x_row_len<N, K>(P.ncx);
    const int64_t line = blockIdx.x;
    const int64_t base = line * Lx;
    const int64_t nn = P.nnodes;
    PDG_CHECK_IDX(base + (NV - 1) * nn + Lx - 1, P.f_elems, "relax_xsweep f");  // the line's last node
    const uint64_t pol = l2_policy(P.l2keep);

    // phase 1: collision at every node of the line.  With few velocities per node (2-D models) a
    // thread loads U = 2 nodes before computing either, so twice the loads are in flight (the
    // loads of the next node cannot move above this node's stores: f may alias)
    constexpr int U = (NV <= 16) ? 2 : 1;
    for (int X0 = threadIdx.x; X0 < Lx; X0 += U * blockDim.x) {
        double fv[U][NV];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int X = X0 + u * blockDim.x;
            if (X < Lx) {
#pragma unroll
                for (int i = 0; i < NV; ++i) fv[u][i] = ld_pol(P.f + base + X + i * nn, pol);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int X = X0 + u * blockDim.x;
            if (X >= Lx) break;
            double w[M];
#pragma unroll
            for (int c = 0; c < M; ++c) {
                double s = fv[u][c * 2 * DIM];
#pragma unroll
                for (int j = 1; j < 2 * DIM; ++j) s += fv[u][c * 2 * DIM + j];
                w[c] = s;
            }
            double q[DIM][M];
            Md::flux(w, q, P.mp);
            const int xs = X + X / SEG;
#pragma unroll
            for (int i = 0; i < NV; ++i) {
                const double val = fma(P.cb, feq_of<DIM, M>(i, w, q, P.mp), P.ca * fv[u][i]);
                const int c = i / (2 * DIM), k = (i % (2 * DIM)) >> 1, s = i & 1;
                if (k == 0) sx[(2 * c + s) * Lp + xs] = val;
                else st_pol(P.f + base + X + i * nn, val, pol);
            }
        }
    }
    __syncthreads();

    // phase 2: T2 sweep(s) of the 2M x-velocities, one warp per velocity
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    double Mb[N * N], gb[N];
#pragma unroll
    for (int i = 0; i < N * N; ++i) Mb[i] = P.blk.M[i];
#pragma unroll
    for (int i = 0; i < N; ++i) gb[i] = P.blk.g[i];
    for (int v = warp; v < 2 * M; v += nwarps) {
        const int c = v >> 1, s = v & 1;
        const int i = c * 2 * DIM + s;
        PDG_CHECK_IDX(i * P.plane_stride + line, P.fb_elems, "relax_xsweep fb");
        const double s0 = 2.0 * P.fb[i * P.plane_stride + line];  // ghost: f^b old + new
        warp_line_sweep<N, NPASS, K>(sx + v * Lp, P.ncx, s == 0, Mb, gb, s0, lane);
    }
    __syncthreads();

    // phase 3: store the x-velocities (node-outer: one padded index per node for all of them)
    for (int X = threadIdx.x; X < Lx; X += blockDim.x) {
        const int xs = X + X / SEG;
#pragma unroll
        for (int v = 0; v < 2 * M; ++v) {
            const int i = (v >> 1) * 2 * DIM + (v & 1);
            st_pol(P.f + base + X + i * nn, sx[v * Lp + xs], pol);
        }
    }
}

// ---------------------------------------------------------------------------
// The same fused pass with the line's raw data staged by the Tensor Memory Accelerator: a
// persistent CTA walks lines blockIdx.x, blockIdx.x + gridDim.x, ...; one thread issues the n_v
// bulk copies (cp.async.bulk, one per velocity row of the line, completion counted on an
// mbarrier) of the NEXT line as soon as the collision has consumed the current one, so the
// loads overlap the x sweeps and the stores of the current line.  Shared memory: the raw line
// [n_v][Lx] + the padded sweep rows of the x velocities.  Requires an even Lx (16-byte aligned
// rows).  Same arithmetic as relax_xsweep_kernel.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// bulk copy global -> shared of `bytes` (multiple of 16, 16-byte aligned), counted on `bar`
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

template <int DIM, int MODEL, int N, int NPASS, int K>
__global__ void __launch_bounds__(256) relax_xsweep_tma_kernel(const RelaxXParams P, int64_t nlines)
{
    using Md = Model<DIM, MODEL>;
    constexpr int M = Md::M;
    constexpr int NV = M * 2 * DIM;
    constexpr int SEG = K * N;
    extern __shared__ __align__(128) double sraw[];  // [NV][Lx] raw line, then [2M][Lp] sweep rows
    __shared__ __align__(8) uint64_t bar;
    const int Lx = P.ncx * N;
    const int Lp = relax_x_row_len<N, K>(P.ncx);
    double *sx = sraw + (size_t)NV * Lx;
    const int64_t nn = P.nnodes;
    const uint32_t row_bytes = (uint32_t)Lx * 8u;
    auto issue = [&](int64_t line) {  // one thread: the NV velocity rows of `line`
        mbar_arrive_expect_tx(&bar, row_bytes * NV);
#pragma unroll 1
        for (int i = 0; i < NV; ++i) bulk_g2s(sraw + (size_t)i * Lx, P.f + i * nn + line * Lx, row_bytes, &bar);
    };
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    int64_t line = blockIdx.x;
    if (threadIdx.x == 0 && line < nlines) issue(line);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    double Mb[N * N], gb[N];
#pragma unroll
    for (int i = 0; i < N * N; ++i) Mb[i] = P.blk.M[i];
#pragma unroll
    for (int i = 0; i < N; ++i) gb[i] = P.blk.g[i];
    uint32_t parity = 0;
    for (; line < nlines; line += gridDim.x) {
        const int64_t base = line * Lx;
        PDG_CHECK_IDX(base + (NV - 1) * nn + Lx - 1, P.f_elems, "relax_xsweep_tma f");
        mbar_wait(&bar, parity);
        parity ^= 1u;
        // collision at every node of the line, from the staged raw rows
        for (int X = threadIdx.x; X < Lx; X += blockDim.x) {
            double fv[NV];
#pragma unroll
            for (int i = 0; i < NV; ++i) fv[i] = sraw[(size_t)i * Lx + X];
            double w[M];
#pragma unroll
            for (int c = 0; c < M; ++c) {
                double s = fv[c * 2 * DIM];
#pragma unroll
                for (int j = 1; j < 2 * DIM; ++j) s += fv[c * 2 * DIM + j];
                w[c] = s;
            }
            double q[DIM][M];
            Md::flux(w, q, P.mp);
            const int xs = X + X / SEG;
#pragma unroll
            for (int i = 0; i < NV; ++i) {
                const double val = fma(P.cb, feq_of<DIM, M>(i, w, q, P.mp), P.ca * fv[i]);
                const int c = i / (2 * DIM), k = (i % (2 * DIM)) >> 1, s = i & 1;
                if (k == 0) sx[(2 * c + s) * Lp + xs] = val;
                else __stcs(P.f + base + X + i * nn, val);
            }
        }
        __syncthreads();  // the raw rows are consumed: stage the next line behind the sweeps
        if (threadIdx.x == 0 && line + gridDim.x < nlines) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(line + gridDim.x);
        }
        for (int v = warp; v < 2 * M; v += nwarps) {
            const int c = v >> 1, s = v & 1;
            const int i = c * 2 * DIM + s;
            PDG_CHECK_IDX(i * P.plane_stride + line, P.fb_elems, "relax_xsweep_tma fb");
            const double s0 = 2.0 * P.fb[i * P.plane_stride + line];  // ghost: f^b old + new
            warp_line_sweep<N, NPASS, K>(sx + v * Lp, P.ncx, s == 0, Mb, gb, s0, lane);
        }
        __syncthreads();
        for (int v = 0; v < 2 * M; ++v) {  // (velocity-outer measured faster here than node-outer)
            const int i = (v >> 1) * 2 * DIM + (v & 1);
            double *dst = P.f + base + i * nn;
            const double *srow = sx + v * Lp;
            for (int X = threadIdx.x; X < Lx; X += blockDim.x) __stcs(dst + X, srow[X + X / SEG]);
        }
        __syncthreads();  // sx is rewritten by the next line's collision
    }
}

// ---------------------------------------------------------------------------
// T2 sweep along x (contiguous): warp per line, lanes = cells, affine warp scan.
// ---------------------------------------------------------------------------
constexpr int kXsWarps = 8;

template <int N, int NPASS>
__global__ void __launch_bounds__(kXsWarps * 32) sweep_x_kernel(const SweepParams P)
{
    constexpr int S = (N % 2) ? N : N + 1;  // odd smem stride: conflict-free 8-byte lane reads
    __shared__ double sbuf[kXsWarps][32 * S];
    const SweepVel V = P.v[blockIdx.y];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t line = (int64_t)blockIdx.x * kXsWarps + warp;
    if (line >= V.nlines) return;  // warp-uniform
    double *row = P.f + V.f_off + line * (int64_t)V.ncells * N;
    PDG_CHECK_IDX(V.f_off + (line + 1) * (int64_t)V.ncells * N - 1, P.f_elems, "sweep_x f");
    PDG_CHECK_IDX(V.fb_off + line, P.fb_elems, "sweep_x fb");
    double *buf = sbuf[warp];
    const unsigned FULL = 0xffffffffu;

    double M[N * N], g[N];
#pragma unroll
    for (int i = 0; i < N * N; ++i) M[i] = P.blk[0].M[i];
#pragma unroll
    for (int i = 0; i < N; ++i) g[i] = P.blk[0].g[i];
    const double beta = g[N - 1];

    double carry[NPASS];
    const double s0 = 2.0 * P.fb[V.fb_off + line];
#pragma unroll
    for (int q = 0; q < NPASS; ++q) carry[q] = s0;

    const int nchunks = (V.ncells + 31) >> 5;
    const bool up = V.sign > 0;
    const int pos = up ? lane : 31 - lane;
    for (int ch = 0; ch < nchunks; ++ch) {
        const int region = up ? ch * 32 : V.ncells - 32 * (ch + 1);
#pragma unroll
        for (int t = lane; t < 32 * N; t += 32) {
            const int co = t / N, a = t - co * N;
            const int cell = region + co;
            if (cell >= 0 && cell < V.ncells) buf[co * S + a] = __ldcs(row + (int64_t)cell * N + a);
        }
        __syncwarp();
        const int mycell = region + pos;
        const bool valid = mycell >= 0 && mycell < V.ncells;
        double fo[N];
#pragma unroll
        for (int a = 0; a < N; ++a) fo[a] = valid ? buf[pos * S + (up ? a : N - 1 - a)] : 0.0;
#pragma unroll
        for (int q = 0; q < NPASS; ++q) {
            double f0[N];
#pragma unroll
            for (int a = 0; a < N; ++a) {
                double acc = 0.0;
#pragma unroll
                for (int b = 0; b < N; ++b) acc = fma(M[a * N + b], fo[b], acc);
                f0[a] = acc;
            }
            double A = valid ? fo[N - 1] + f0[N - 1] : 0.0;
            double B = valid ? beta : 1.0;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const double Ap = __shfl_up_sync(FULL, A, off);
                const double Bp = __shfl_up_sync(FULL, B, off);
                if (lane >= off) {
                    A = fma(B, Ap, A);
                    B *= Bp;
                }
            }
            const double s_incl = fma(B, carry[q], A);
            double s_prev = __shfl_up_sync(FULL, s_incl, 1);
            if (lane == 0) s_prev = carry[q];
#pragma unroll
            for (int a = 0; a < N; ++a) fo[a] = fma(g[a], s_prev, f0[a]);
            carry[q] = __shfl_sync(FULL, s_incl, 31);
        }
        if (valid) {
#pragma unroll
            for (int a = 0; a < N; ++a) buf[pos * S + (up ? a : N - 1 - a)] = fo[a];
        }
        __syncwarp();
#pragma unroll
        for (int t = lane; t < 32 * N; t += 32) {
            const int co = t / N, a = t - co * N;
            const int cell = region + co;
            if (cell >= 0 && cell < V.ncells) __stcs(row + (int64_t)cell * N + a, buf[co * S + a]);
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// Relaxation fused with the moment reduction (G = 1): all n_v velocities local.
// ---------------------------------------------------------------------------
template <int DIM, int MODEL>
__global__ void __launch_bounds__(256) relax_kernel(double *__restrict__ f, int64_t nnodes, ModelParams P,
                                                    double ca, double cb)
{
    using Md = Model<DIM, MODEL>;
    constexpr int M = Md::M;
    constexpr int NV = M * 2 * DIM;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < nnodes; x += stride) {
        double fv[NV];
#pragma unroll
        for (int i = 0; i < NV; ++i) fv[i] = __ldcs(f + (int64_t)i * nnodes + x);
        double w[M];
#pragma unroll
        for (int c = 0; c < M; ++c) {
            double s = fv[c * 2 * DIM];
#pragma unroll
            for (int j = 1; j < 2 * DIM; ++j) s += fv[c * 2 * DIM + j];
            w[c] = s;
        }
        double q[DIM][M];
        Md::flux(w, q, P);
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            const double feq = feq_of<DIM, M>(i, w, q, P);
            __stcs(f + (int64_t)i * nnodes + x, fma(cb, feq, ca * fv[i]));
        }
    }
}

// Partial moments of the local velocity block [v0, v0 + nvl): w_c = sum of local f_i in c.
// Velocity loops run over the compile-time n_v with a range test, so every index is static
// (no local-memory arrays).  f and w point at the first node of a chunk of `count` nodes;
// nnodes is the velocity / component stride (chunks pipeline the NCCL sum, pdg_api.cu).
template <int DIM, int MODEL>
__global__ void __launch_bounds__(256) partial_moments_kernel(const double *__restrict__ f, double *__restrict__ w,
                                                              int64_t nnodes, int64_t count, int v0, int nvl)
{
    constexpr int M = Model<DIM, MODEL>::M;
    constexpr int NV = M * 2 * DIM;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < count; x += stride) {
        double acc[M];
#pragma unroll
        for (int c = 0; c < M; ++c) acc[c] = 0.0;
#pragma unroll
        for (int i = 0; i < NV; ++i)
            if (i >= v0 && i < v0 + nvl) acc[i / (2 * DIM)] += __ldcs(f + (int64_t)(i - v0) * nnodes + x);
#pragma unroll
        for (int c = 0; c < M; ++c) __stcs(w + (int64_t)c * nnodes + x, acc[c]);
    }
}

// Collision of the local velocities from reduced moments w (sharded path, row a4), on a chunk of
// `count` nodes (f, w at its first node; nnodes is the stride).
template <int DIM, int MODEL>
__global__ void __launch_bounds__(256) relax_from_w_kernel(double *__restrict__ f, const double *__restrict__ w,
                                                           int64_t nnodes, int64_t count, int v0, int nvl, ModelParams P,
                                                           double ca, double cb)
{
    using Md = Model<DIM, MODEL>;
    constexpr int M = Md::M;
    constexpr int NV = M * 2 * DIM;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < count; x += stride) {
        double fl[NV], wl[M];
#pragma unroll
        for (int i = 0; i < NV; ++i) fl[i] = (i >= v0 && i < v0 + nvl) ? __ldcs(f + (int64_t)(i - v0) * nnodes + x) : 0.0;
#pragma unroll
        for (int c = 0; c < M; ++c) wl[c] = __ldcs(w + (int64_t)c * nnodes + x);
        double q[DIM][M];
        Md::flux(wl, q, P);
#pragma unroll
        for (int i = 0; i < NV; ++i)
            if (i >= v0 && i < v0 + nvl)
                __stcs(f + (int64_t)(i - v0) * nnodes + x, fma(cb, feq_of<DIM, M>(i, wl, q, P), ca * fl[i]));
    }
}

// f_i = f^eq_i(w) at every node for the local velocities.
template <int DIM, int MODEL>
__global__ void __launch_bounds__(256) equilibrium_kernel(double *__restrict__ f, const double *__restrict__ w,
                                                          int64_t nnodes, int v0, int nvl, ModelParams P)
{
    using Md = Model<DIM, MODEL>;
    constexpr int M = Md::M;
    constexpr int NV = M * 2 * DIM;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < nnodes; x += stride) {
        double wl[M];
#pragma unroll
        for (int c = 0; c < M; ++c) wl[c] = w[(int64_t)c * nnodes + x];
        double q[DIM][M];
        Md::flux(wl, q, P);
#pragma unroll
        for (int i = 0; i < NV; ++i)
            if (i >= v0 && i < v0 + nvl) __stcs(f + (int64_t)(i - v0) * nnodes + x, feq_of<DIM, M>(i, wl, q, P));
    }
}

// fb_i = f^eq_i(wb) on the inflow plane of each local velocity (line enumeration of the sweeps:
// plane index == line index, the inflow node is the first node of the line in flow order).
template <int DIM, int MODEL>
__global__ void __launch_bounds__(256) inflow_equilibrium_kernel(double *__restrict__ fb, const double *__restrict__ wb,
                                                                 int64_t nnodes, const SweepParams S, int n,
                                                                 ModelParams P)
{
    using Md = Model<DIM, MODEL>;
    constexpr int M = Md::M;
    const SweepVel V = S.v[blockIdx.y];
    const int64_t line = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (line >= V.nlines) return;
    const int64_t Lk = (int64_t)V.ncells * n;
    const int64_t base = (line / V.inner) * (V.inner * Lk) + (line % V.inner);
    const int64_t node = base + ((V.sign > 0) ? 0 : (Lk - 1) * V.inner);
    double wl[M];
#pragma unroll
    for (int c = 0; c < M; ++c) wl[c] = wb[(int64_t)c * nnodes + node];
    double q[DIM][M];
    Md::flux(wl, q, P);
    fb[V.fb_off + line] = feq_of<DIM, M>(V.vel, wl, q, P);
}

// Count nodes with rho <= 0 (component-0 block sum) or a non-finite local f.
__global__ void __launch_bounds__(256) check_state_kernel(const double *__restrict__ f, int64_t nnodes, int v0,
                                                          int nvl, int nrho, int check_rho, unsigned long long *count)
{
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    unsigned long long bad = 0;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < nnodes; x += stride) {
        double rho = 0.0;
        bool ok = true;
        for (int j = 0; j < nvl; ++j) {
            const double v = f[(int64_t)j * nnodes + x];
            ok = ok && isfinite(v);
            if (v0 + j < nrho) rho += v;
        }
        if (check_rho && !(rho > 0.0)) ok = false;
        bad += ok ? 0 : 1;
    }
    for (int off = 16; off > 0; off >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, off);
    if ((threadIdx.x & 31) == 0 && bad) atomicAdd(count, bad);
}

// ---------------------------------------------------------------------------
// Z-slab decomposition: along the outer axis the zero-inflow outgoing carries
// A_q (pass q) of every slab come from a read-only pre-pass (zslab_carry_kernel; the entry slab
// of a velocity starts from its true inflow).  The carry recurrence is affine, so the exact
// inflows follow from the slabs upstream: with B = beta^len and C = the pass-2 carry response
// to a unit pass-1 inflow (host tables),
//   S1(next) = A1 + B S1,   S2(next) = A2 + C S1 + B S2.
// Each slab is then swept once from its exact inflows (SweepVel::cin_off): no correction pass.
// ---------------------------------------------------------------------------
struct ZSlabParams {
    const double *carry;   // [slab][vel][2][plane] zero-inflow outgoing carries (pre-pass, all-gathered)
    double *inflow;        // [slab][vel][2][plane] exact inflows (output of the scan)
    int64_t carry_elems;   // buffer bound (checked build; inflow has as many)
    double B[64], C[64];   // per global slab: beta^len, pass-2 carry response
    int64_t plane;         // lines per slab
    int32_t nslab, nvo, npass;
    int32_t sign[16];
};

__global__ void __launch_bounds__(256) zslab_scan_kernel(const ZSlabParams P)
{
    const int j = blockIdx.y;
    const int64_t line = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (line >= P.plane) return;
    const bool up = P.sign[j] > 0;
    const int first = up ? 0 : P.nslab - 1;
    const int64_t vstride = 2 * P.plane;
    const int64_t sstride = (int64_t)P.nvo * vstride;
    PDG_CHECK_IDX((int64_t)(P.nslab - 1) * sstride + j * vstride + P.plane + line, P.carry_elems, "zslab_scan carry");
    double c1 = P.carry[first * sstride + j * vstride + line];
    double c2 = (P.npass > 1) ? P.carry[first * sstride + j * vstride + P.plane + line] : 0.0;
    for (int k = 1; k < P.nslab; ++k) {
        const int s = up ? k : P.nslab - 1 - k;
        const int64_t o = s * sstride + j * vstride + line;
        P.inflow[o] = c1;
        if (P.npass > 1) P.inflow[o + P.plane] = c2;
        const double a1 = P.carry[o];
        const double n1 = fma(P.B[s], c1, a1);
        if (P.npass > 1) c2 = fma(P.B[s], c2, fma(P.C[s], c1, P.carry[o + P.plane]));
        c1 = n1;
    }
}

// Z-slab carry pre-pass (read-only): the zero-inflow outgoing carries A_q of every slab
// line, from the slab's last `lpre` cells only (flow order; data further upstream changes the
// outgoing carries by less than 2^-64 of its size, reading C26).  A slab with fewer cells is
// walked whole, from its true inflow if it is the entry slab.  Writes cout[cout_off + q nlines +
// line]; the exact slab sweeps run after the carry scan with the exact inflows (cin).
template <int N, int NPASS>
__global__ void __launch_bounds__(256) zslab_carry_kernel(const SweepParams P, int lpre)
{
    const SweepVel V = P.v[blockIdx.y];
    const int64_t line = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (line >= V.nlines) return;
    const int64_t Lk = (int64_t)V.ncells * N;
    const int64_t base = (line / V.inner) * (V.inner * Lk) + (line % V.inner);
    const int64_t step = (V.sign > 0) ? V.inner : -V.inner;
    const int64_t p_at = V.f_off + base + ((V.sign > 0) ? 0 : (Lk - 1) * V.inner);
    const double *p = P.f + p_at;
    PDG_CHECK_IDX(p_at, P.f_elems, "zslab_carry f");
    PDG_CHECK_IDX(p_at + (Lk - 1) * step, P.f_elems, "zslab_carry f");
    double M[N * N], g[N];
#pragma unroll
    for (int i = 0; i < N * N; ++i) M[i] = P.blk[V.axis].M[i];
#pragma unroll
    for (int i = 0; i < N; ++i) g[i] = P.blk[V.axis].g[i];
    const int c0 = max(0, V.ncells - lpre);
    double s0 = 0.0;
    if (c0 == 0 && !V.zero_inflow) {
        PDG_CHECK_IDX(V.fb_off + line, P.fb_elems, "zslab_carry fb");
        s0 = 2.0 * P.fb[V.fb_off + line];
    }
    double carry[NPASS];
#pragma unroll
    for (int q = 0; q < NPASS; ++q) carry[q] = s0;
    for (int c = c0; c < V.ncells; ++c) {
        double fo[N];
#pragma unroll
        for (int a = 0; a < N; ++a) fo[a] = __ldcs(p + ((int64_t)c * N + a) * step);
#pragma unroll
        for (int q = 0; q < NPASS; ++q) {
            double fn[N];
#pragma unroll
            for (int a = 0; a < N; ++a) {
                double acc = g[a] * carry[q];
#pragma unroll
                for (int b = 0; b < N; ++b) acc = fma(M[a * N + b], fo[b], acc);
                fn[a] = acc;
            }
            carry[q] = fo[N - 1] + fn[N - 1];
#pragma unroll
            for (int a = 0; a < N; ++a) fo[a] = fn[a];
        }
    }
#pragma unroll
    for (int q = 0; q < NPASS; ++q) {
        PDG_CHECK_IDX(V.cout_off + q * V.nlines + line, P.cout_elems, "zslab_carry cout");
        P.cout[V.cout_off + q * V.nlines + line] = carry[q];
    }
}

// ---------------------------------------------------------------------------
// Small problems (config 1: f = 18 KB): a whole pdg_step(n) is a sequence of short dependent
// passes, each far too small to fill the GPU, so the step is bound by launch and drain latency
// (2 launches per step in a graph replay: ~7.7 us per step).  One CTA holds f in shared memory
// and runs the step's operator list (T2 sweeps and C2 collisions, same arithmetic as
// sweep_strided_kernel and relax_kernel: sequential carry per line, per-node collision) with a
// barrier between operators; f is read once and written once per launch.
// ---------------------------------------------------------------------------
constexpr int kSmallMaxOps = 48;   // operators per launch (longer lists take several launches)
constexpr int kSmallMaxBlk = 6;    // distinct T2 step sizes per launch
constexpr int kSmallThreads = 512;

struct SmallOp {
    int32_t kind;  // 0: T2 (blk = its block set), 1: C2 (f <- ca f + cb f^eq)
    int32_t blk;
    double ca, cb;
};

struct SmallParams {
    double *f;
    const double *fb;
    int64_t nnodes;
    int64_t f_elems, fb_elems;  // buffer bounds (checked build)
    int32_t nvel, nops;
    int32_t L0, Lp;      // nodes per x row in HBM and in shared memory (Lp odd: x-line walks of
                         // neighbouring threads fall on different banks)
    int64_t vstride;     // shared-memory elements per velocity (rows x Lp)
    int64_t sstr[3];     // shared-memory element stride per axis (1, Lp, Lp L1)
    int64_t line0[kMaxVel + 1];  // prefix sums of the velocities' line counts, each rounded up to a
                                 // multiple of 32: every warp sweeps lines of one velocity, so its
                                 // velocity record and block come from the parameter bank uniformly
    SweepVel v[kMaxVel];
    DevBlock blk[kSmallMaxBlk][3];
    SmallOp op[kSmallMaxOps];
    ModelParams mp;
};

template <int DIM, int MODEL, int N>
__global__ void __launch_bounds__(kSmallThreads) small_run_kernel(const __grid_constant__ SmallParams P)
{
    using Md = Model<DIM, MODEL>;
    constexpr int M = Md::M;
    constexpr int NV = M * 2 * DIM;
    extern __shared__ double sf[];  // f as [velocity][row][Lp] (HBM: [velocity][row][L0])
    const int64_t tot = (int64_t)NV * P.nnodes;
    PDG_CHECK_IDX(tot - 1, P.f_elems, "small_run f");
    auto sidx = [&](int64_t g) -> int64_t { return (g / P.L0) * P.Lp + g % P.L0; };  // node -> shared
    for (int64_t i = threadIdx.x; i < tot; i += blockDim.x) {
        const int64_t v = i / P.nnodes, x = i - v * P.nnodes;
        sf[v * P.vstride + sidx(x)] = P.f[i];
    }
    __syncthreads();
    for (int o = 0; o < P.nops; ++o) {
        const SmallOp op = P.op[o];
        if (op.kind == 1) {
            for (int64_t x = threadIdx.x; x < P.nnodes; x += blockDim.x) {
                const int64_t sx = sidx(x);
                double fv[NV];
#pragma unroll
                for (int i = 0; i < NV; ++i) fv[i] = sf[(int64_t)i * P.vstride + sx];
                double w[M];
#pragma unroll
                for (int c = 0; c < M; ++c) {
                    double s = fv[c * 2 * DIM];
#pragma unroll
                    for (int j = 1; j < 2 * DIM; ++j) s += fv[c * 2 * DIM + j];
                    w[c] = s;
                }
                double q[DIM][M];
                Md::flux(w, q, P.mp);
#pragma unroll
                for (int i = 0; i < NV; ++i) sf[(int64_t)i * P.vstride + sx] = fma(op.cb, feq_of<DIM, M>(i, w, q, P.mp), op.ca * fv[i]);
            }
        } else {
            const int64_t nl = P.line0[P.nvel];
            for (int64_t t = threadIdx.x; t < nl; t += blockDim.x) {
                int vi = 0;
                while (t >= P.line0[vi + 1]) ++vi;
                const SweepVel &V = P.v[vi];
                const int64_t line = t - P.line0[vi];
                if (line >= V.nlines) continue;
                const DevBlock &B = P.blk[op.blk][V.axis];
                const int64_t Lk = (int64_t)V.ncells * N;
                const int64_t base = (line / V.inner) * (V.inner * Lk) + (line % V.inner);  // first node
                const int64_t ss = P.sstr[V.axis];
                const int64_t step = (V.sign > 0) ? ss : -ss;
                double *p = sf + (V.f_off / P.nnodes) * P.vstride + sidx(base) + ((V.sign > 0) ? 0 : (Lk - 1) * ss);
                PDG_CHECK_IDX(V.fb_off + line, P.fb_elems, "small_run fb");
                double carry = 2.0 * P.fb[V.fb_off + line];  // ghost cell: f^b old + f^b new (reading C5)
                for (int cl = 0; cl < V.ncells; ++cl, p += N * step) {
                    double fo[N], fn[N];
#pragma unroll
                    for (int a = 0; a < N; ++a) fo[a] = p[a * step];
#pragma unroll
                    for (int a = 0; a < N; ++a) {
                        double acc = B.g[a] * carry;
#pragma unroll
                        for (int b = 0; b < N; ++b) acc = fma(B.M[a * N + b], fo[b], acc);
                        fn[a] = acc;
                    }
                    carry = fo[N - 1] + fn[N - 1];
#pragma unroll
                    for (int a = 0; a < N; ++a) p[a * step] = fn[a];
                }
            }
        }
        __syncthreads();
    }
    for (int64_t i = threadIdx.x; i < tot; i += blockDim.x) {
        const int64_t v = i / P.nnodes, x = i - v * P.nnodes;
        P.f[i] = sf[v * P.vstride + sidx(x)];
    }
}

}  // namespace pdg
