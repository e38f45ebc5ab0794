// sm_100a kernels for lattice velocity sets: D2Q9 (the paper's
// Euler-with-gravity model) and the D3Q15/19/27 sets of its scaling tests
// (P:856-858).  Velocities have components in {0, +-lambda}; a velocity with
// d >= 2 non-zero components couples the d active axes of a cell through a dense
// n^d x n^d local block (pdg_tables.hpp lattice_block) and its dependency graph has
// genuinely diagonal wavefronts (Fig. dependency_graph).
//
//  lattice_sweep_kernel<D, N, ACT>: T2(dt') (solved downwind P:622-637) for the
//  velocities whose active-axis mask is ACT (binary x=1, y=2, z=4; d >= 2).
//   * "unit" = the active-axis nodes of one cell (inactive axes decouple: each inactive
//     node index is an independent problem).  One lane owns one unit per row.
//   * lanes run along x: 32 consecutive x-cells (x active) or x-nodes (x inactive), so
//     every load/store of a warp is a contiguous run (coalesced).
//   * the CHAIN axis (z if active, else y) is walked serially; the chain in-trace stays in
//     registers (the lane owns the same x position in every row).
//   * the x dependency inside a row is an affine recurrence of n^{d-1}-vectors
//     s_out = a + Bx s_in (Bx uniform): a 5-step warp-shuffle Kogge-Stone scan with the
//     precomputed powers Bx^(2^j); warps along x and along the PIPE axis (y, when y and z
//     are both active) are skewed by one row per warp inside the CTA and hand traces over
//     through shared memory (a barrier per row, or point-to-point step counters).
//   * across CTAs the x traces (and the FMA path's y traces) travel as tagged 64-bit words
//     (ll_put / ll_take: no fences, the consumer empties the slot); the tensor path's y
//     traces are plain doubles with a per-(task, x-warp) row-progress counter published by
//     the producing warp.  Tasks are claimed in dependency order with an atomic ticket, so
//     every wait targets a task already owned by a running CTA.
//   * classes without a pipe axis that cannot fill the GPU walk their chain in segments
//     that start a norm-bounded halo early from a zero trace (pdg_tables.hpp
//     lattice_chain_halo); segments are claimed in descending order and release their halo
//     rows to the previous segment with a flag.
//   * the block is applied in the rhs form F = A^{-1} (2 f_old + in-trace injections), then
//     + Q_x s_x after the scan, f_new = F - f_old; on the FMA path the constants come from
//     the kernel parameter space, on the tensor path (body diagonals, DMMA.8x8x4) from
//     shared memory.
//
//  relax_lbm2_kernel<D, NV>: collision fused with the
//  moments w = (rho, rho u) = P f, P = [1; v^T],
//  f^eq_i = w_i rho (1 + u.v_i/c^2 + (u.v_i)^2/(2c^4) - u.u/(2c^2)),
//  f <- ca f + cb f^eq (eq collision_cn).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <type_traits>

#include "pdg_check.cuh"

namespace pdg {

constexpr int kLatMaxVel = 12;   // velocities of one active-axis class (D3Q27: 12 face diagonals)
constexpr int kLbmMaxVel = 27;

__host__ __device__ constexpr int ipow(int b, int e)
{
    int r = 1;
    for (int i = 0; i < e; ++i) r *= b;
    return r;
}

template <int D, int ACT>
struct LatShape {
    static constexpr int XA = ACT & 1;
    static constexpr int YA = (ACT >> 1) & 1;
    static constexpr int ZA = (D == 3) ? ((ACT >> 2) & 1) : 0;
    static constexpr int DA = XA + YA + ZA;                 // active axes
    static constexpr int CA = ZA ? 2 : 1;                   // chain axis (walked serially)
    static constexpr int PIPE = (D == 3 && ZA && YA) ? 1 : 0;  // y handed over warp to warp
    static constexpr int BA = (D == 3 && !ZA) ? 2 : ((D == 3 && !YA) ? 1 : -1);  // batch axis (inactive)
    // index t of each physical axis among the active ones (-1: inactive)
    static constexpr int T0 = XA ? 0 : -1;
    static constexpr int T1 = YA ? XA : -1;
    static constexpr int T2 = ZA ? XA + YA : -1;
    __host__ __device__ static constexpr int t_of(int k) { return k == 0 ? T0 : (k == 1 ? T1 : T2); }
    static constexpr int TC = (CA == 2) ? T2 : T1;
};

template <int N, int DA>
struct LatTab {
    static constexpr int NB = ipow(N, DA);
    static constexpr int MF = NB / N;
    // stored column-major ([column][row]): the kernels stream one column at a time into NB
    // independent accumulators, so consecutive rows are adjacent (LDCU.128 loads two at once)
    double M[NB * NB];      // A^{-1} (applied to the rhs 2 f_old + in-trace injections), M[c * NB + q]
    double Q[DA][NB * MF];  // A^{-1} E_in^(t) kappa_t / omega_0 (in-traces of axis t), Q[t][j * NB + q]
    double Bp[5][MF * MF];  // Bx^(2^j), Bx = rows of Q[0] on the x-out face,     Bp[s][j * MF + i]
};

// Block tables too large for the 32 KB kernel parameter space (p = 3 body diagonals: 64 x 64
// block): same layouts as LatTab, in device memory (read once per CTA into shared memory for
// the tensor path; the scan's Bx powers through the L1/L2 broadcast path).
struct LatTabRef {
    const double *M;
    const double *Q[3];
    const double *Bp[5];
};

template <int N, int DA>
struct LatTabSel {
    static constexpr bool BIG = sizeof(LatTab<N, DA>) > 24 * 1024;
    using type = typename std::conditional<BIG, LatTabRef, LatTab<N, DA>>::type;
};

struct LatVel {
    int64_t f_off;   // element offset of the velocity's node grid in f
    int64_t fb_off;  // element offset of its D inflow planes in fb
    int32_t sign[3]; // flow direction per axis (+1 / -1; inactive axes +1)
    int32_t pad;
};

struct LatGeom {
    int64_t L[3];        // nodes per axis
    int64_t stride[3];   // element stride per axis
    int64_t plane_stride;
    int32_t ncell[3];
    int32_t Wx, Wy;      // warps per CTA along x / along the pipe (or batch) dimension
    int32_t ngx, ngy;    // CTA groups along x / pipe-or-batch
    int32_t nlane;       // x cells (x active) or x nodes
    int32_t nw;          // pipe cells, batch nodes or 1
    int32_t nc;          // chain cells
    int32_t ntasks;      // tasks: (segment, pipe group, velocity, x group)
    int32_t nvel;
    int32_t nscan;       // x-scan rounds carrying weight: round j is dropped when |Bx^(2^j)| < 2^-64
    int32_t nseg;        // chain segments (1: the whole chain per task)
    int32_t seglen;      // chain rows stored by one segment
    int32_t halo;        // rows a segment sweeps ahead of its first stored row (from a zero chain trace)
    int32_t rcap;        // chain rows per task in the trace buffers
    double kw[3];        // kappa_t / omega_0 per active axis (tensor path: in-trace injection into the rhs)
};

template <int D, int N, int ACT>
struct LatParams {
    using S = LatShape<D, ACT>;
    double *f;
    const double *fb;
    int *ticket;     // [0]; progress counters follow: progress[task * 8 + x-warp] = rows published (tensor-path y traces)
    int *progress;
    int *hdone;      // [task]: 1 once the segment has read its halo rows (their old values)
    double *xbuf;    // [task][row][Wy][2 MF] tagged x out-trace words at CTA boundaries
    double *ybuf;    // [task][row][Wx][32][2 MF] tagged y out-trace words at CTA boundaries (FMA
                     // path; the tensor path stores plain doubles with an MF rounded up to even stride)
    int64_t f_elems, fb_elems, xbuf_elems, ybuf_elems, ints_elems;  // buffer bounds (checked build)
    LatGeom g;
    LatVel v[kLatMaxVel];
    typename LatTabSel<N, S::DA>::type tab;
};

// Optional per-phase cycle counters of one warp (diagnostics build: -DPDG_LAT_TIMING)
#ifdef PDG_LAT_TIMING
#define PDG_TMARK(k)                                                                                 \
    do {                                                                                             \
        const long long now_ = clock64();                                                            \
        tph[k] += now_ - tlast;                                                                      \
        tlast = now_;                                                                                \
    } while (0)
#else
#define PDG_TMARK(k) \
    do {            \
    } while (0)
#endif

__device__ __forceinline__ int ld_acquire(const int *p)
{
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release(int *p, int v)
{
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// D = A B + D on the fp64 tensor cores (DMMA.8x8x4).  Fragments (PTX ISA, mma.m8n8k4.f64):
// A[8x4] row-major: lane holds A[lane/4][lane%4]; B[4x8] col: lane holds B[lane%4][lane/4];
// C/D[8x8]: lane holds D[lane/4][2(lane%4)], D[lane/4][2(lane%4)+1].
__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b)
{
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(c[0]), "+d"(c[1])
        : "d"(a), "d"(b));
}

// Rows prefetched ahead: 3 for the 2-D diagonals (latency-bound, short rows), 1 in 3-D, none for
// the p = 3 body diagonals, whose 64-node rows would leave room for only two warps per SM.
template <int D, int N = 0, int DA = 0>
struct LatRing {
    static constexpr int PFA = (D == 2) ? 3 : ((N == 4 && DA == 3) ? 0 : 1);
    static constexpr int RING = PFA + 1;  // row buffers per warp
};

// Tensor-core path of the lattice sweep: used for the body diagonals (3 active axes), whose
// n^3 x n^3 block makes the unit update fp64-bound.
template <int D, int N, int ACT>
struct LatMma {
    using S = LatShape<D, ACT>;
    static constexpr int NB = ipow(N, S::DA), MF = NB / N;
    // (the two-axis classes on the tensor path measured slower: their 9-row block pads to 16)
    static constexpr bool USE = (S::DA == 3);
    static constexpr int MT = (NB + 7) / 8;                     // 8-row tiles of the block
    // the first product is A^{-1} r with the rhs r = 2 f_old + sum_t (kappa_t/omega_0) E_in^(t) s_t of
    // the chain and pipe in-traces (M = A^{-1}(2I - A) = 2 A^{-1} - I, Q_t = A^{-1} E_in^(t) kappa_t/omega_0)
    static constexpr int KE = NB;
    static constexpr int KS = (KE + 3) / 4;                     // k-steps of the first product
    static constexpr int KSX = (MF + 3) / 4;                    // k-steps of Q_x s_x
    // row stride of the A operand [M | Q_chain | Q_pipe] in shared memory: a multiple of 16
    // doubles would put the 8 rows of a fragment (lane / 4) on one bank pair, so pad by 4
    static constexpr int SA = KS * 4 + (((KS * 4) % 16 == 0) ? 4 : 0);
    static constexpr size_t smem_doubles(int nwarps)
    {
        return USE ? (size_t)nwarps * NB * 32 + (size_t)MT * 8 * (SA + KSX * 4) : 0;
    }
};

__device__ __forceinline__ void cp_async8(double *sdst, const double *gsrc)
{
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async16_cg(double *sdst, const double *gsrc)
{
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int K>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(K) : "memory"); }

__device__ __forceinline__ void wait_progress(const int *p, int need)
{
    if (ld_acquire(p) >= need) return;
    PDG_SPIN_DECL(spins);
    while (ld_acquire(p) < need) {
        __nanosleep(64);
        PDG_SPIN_TICK(spins, "lattice wait_progress");
    }
}

// Index of a node (given by its flow coordinates u[] on every axis) in the inflow plane of
// axis k: the node grid with axis k removed, same order (include/pdg.h).
template <int D>
__device__ __forceinline__ int64_t plane_index(const LatGeom &g, int k, const int64_t (&ph)[3])
{
    if (D == 2) return k == 0 ? ph[1] : ph[0];
    if (k == 0) return ph[2] * g.L[1] + ph[1];
    if (k == 1) return ph[2] * g.L[0] + ph[0];
    return ph[1] * g.L[0] + ph[0];
}

// f^b at in-face node j (face axis K, active index t) of the unit with cell/coord ucell[].
template <int D, int N, int ACT, int K>
__device__ __forceinline__ const double *ghost_ptr(const LatParams<D, N, ACT> &P, const LatVel &V, const int (&ucell)[3],
                                                   int j)
{
    using S = LatShape<D, ACT>;
    constexpr int T = S::t_of(K);
    const int64_t pl_at = V.fb_off + (int64_t)K * P.g.plane_stride;
    const double *pl = P.fb + pl_at;
    const int r = (j % ipow(N, T)) + (j / ipow(N, T)) * ipow(N, T + 1);  // digit T = 0
    int64_t ph[3] = {0, 0, 0};
#pragma unroll
    for (int a = 0; a < D; ++a) {
        if (a == K) continue;
        const int ta = S::t_of(a);
        int64_t u = (ta >= 0) ? (int64_t)ucell[a] * N + (r / ipow(N, ta)) % N : (int64_t)ucell[a];
        if (ta >= 0 && V.sign[a] < 0) u = P.g.L[a] - 1 - u;
        ph[a] = u;
    }
    PDG_CHECK_IDX(pl_at + plane_index<D>(P.g, K, ph), P.fb_elems, "lattice ghost fb");
    return pl + plane_index<D>(P.g, K, ph);
}

// 2 f^b at the in-face nodes of axis K (the ghost trace, reading C4).
template <int D, int N, int ACT, int K>
__device__ __forceinline__ void ghost_face(const LatParams<D, N, ACT> &P, const LatVel &V, const int (&ucell)[3],
                                           double (&s)[LatTab<N, LatShape<D, ACT>::DA>::MF])
{
    constexpr int MF = LatTab<N, LatShape<D, ACT>::DA>::MF;
#pragma unroll
    for (int j = 0; j < MF; ++j) s[j] = 2.0 * *ghost_ptr<D, N, ACT, K>(P, V, ucell, j);
}

// Tagged trace words (the "LL" idea of NCCL's low-latency protocol): a double crosses CTAs as two
// 64-bit words, each holding 32 of its bits and a 32-bit tag.  Aligned 64-bit accesses are
// single-copy atomic, so a consumer that reads the tag in both words holds the value: no fence on
// the producer, no acquire and no second round trip on the consumer.  The consumer zeroes the
// words after reading (the buffer is zeroed at pdg_create), so every slot is empty again when the
// next launch writes it.
__device__ __forceinline__ void ll_store2(uint64_t *p, uint64_t a, uint64_t b)
{
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void ll_load2(const uint64_t *p, uint64_t &a, uint64_t &b)
{
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
template <int MF>
__device__ __forceinline__ void ll_put(uint64_t *slot, const double (&v)[MF], uint32_t tag)
{
    const uint64_t t = (uint64_t)tag << 32;
#pragma unroll
    for (int j = 0; j < MF; ++j) {
        const uint64_t u = (uint64_t)__double_as_longlong(v[j]);
        ll_store2(slot + 2 * j, (u & 0xffffffffull) | t, (u >> 32) | t);
    }
}
template <int MF>
__device__ __forceinline__ void ll_clear(uint64_t *slot)
{
#pragma unroll
    for (int j = 0; j < MF; ++j) ll_store2(slot + 2 * j, 0ull, 0ull);
}
// decode tagged words already copied (e.g. into shared memory); false if any tag is not `tag`
template <int MF>
__device__ __forceinline__ bool ll_decode(const uint64_t *w, double (&v)[MF], uint32_t tag)
{
    bool ok = true;
#pragma unroll
    for (int j = 0; j < MF; ++j) {
        const uint64_t a = w[2 * j], b = w[2 * j + 1];
        ok = ok && (uint32_t)(a >> 32) == tag && (uint32_t)(b >> 32) == tag;
        v[j] = __longlong_as_double((long long)((b << 32) | (a & 0xffffffffull)));
    }
    return ok;
}
template <int MF>
__device__ __forceinline__ void ll_take(uint64_t *slot, double (&v)[MF], uint32_t tag)
{
    uint64_t w[2 * MF];
    PDG_SPIN_DECL(spins);
    for (;;) {
#pragma unroll
        for (int j = 0; j < MF; ++j) ll_load2(slot + 2 * j, w[2 * j], w[2 * j + 1]);
        bool ok = true;
#pragma unroll
        for (int k = 0; k < 2 * MF; ++k) ok = ok && (uint32_t)(w[k] >> 32) == tag;
        if (ok) break;
        __nanosleep(20);
        PDG_SPIN_TICK(spins, "lattice ll_take");
    }
#pragma unroll
    for (int j = 0; j < MF; ++j) {
        v[j] = __longlong_as_double((long long)((w[2 * j + 1] << 32) | (w[2 * j] & 0xffffffffull)));
        ll_store2(slot + 2 * j, 0ull, 0ull);
    }
}

// One T2(dt') per launch.  Registers are capped for two CTAs per SM on the FMA path; the tensor
// path (body diagonals) needs ~218 KB of shared memory and runs one CTA per SM.  (Measured and
// dropped in round 1: two sweeps per launch, thread-block clusters along the pipe
// axis, the tensor path for the two-axis classes.)
template <int D, int N, int ACT>
__global__ void __launch_bounds__(256, LatShape<D, ACT>::DA == 3 ? 1 : 2)
    lattice_sweep_kernel(const __grid_constant__ LatParams<D, N, ACT> P)
{
    using S = LatShape<D, ACT>;
    using TB = LatTab<N, S::DA>;
    constexpr int DA = S::DA, NB = TB::NB, MF = TB::MF;
    constexpr int XA = S::XA, PIPE = S::PIPE, CA = S::CA, TC = S::TC;
    constexpr int TY = S::T1;
    using MMA = LatMma<D, N, ACT>;
    constexpr bool USE_MMA = MMA::USE;
    constexpr int MT = MMA::MT, KS = MMA::KS, KSX = MMA::KSX;
    // rows prefetched ahead with cp.async: 2-D diagonals are latency-bound (short rows, one warp
    // per SM sub-partition), so they look three rows ahead; 3-D classes one row
    constexpr int PFA = LatRing<D, N, S::DA>::PFA, RING = LatRing<D, N, S::DA>::RING;
    // [row][32 units] shared buffers (row buffers, staging): the tensor path XOR-swizzles the unit
    // index with 4 (row mod 4), so the four rows of a DMMA B fragment (lane % 4) and the eight
    // accumulator rows of a spill fall on different bank pairs
    auto ro = [](int row, int u) -> int { return row * 32 + (USE_MMA ? (u ^ ((row & 3) << 2)) : u); };
    const unsigned FULL = 0xffffffffu;
#ifdef PDG_LAT_TIMING
    long long tph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long tlast = clock64();
#endif

    // x hand-over slots between the x-warps of a CTA: a ring of XR rows; with the point-to-point
    // sync of the pipe classes a producer may run XR - 1 rows ahead of its x consumer
    constexpr int XR = PIPE ? 4 : 2;
    __shared__ double xs[XR][8][XA ? MF : 1];
    __shared__ double gxs[8][RING][XA ? MF : 1];  // x inflow ghosts of the first x warp, prefetched per row
    __shared__ int s_task;
    __shared__ int s_done[16];  // point-to-point row sync: last step finished by each warp
    // dynamic shared memory: per-warp double buffer of the unit values of the current and the next
    // row (cp.async prefetch: the loads of row r+1 do not depend on the carries and overlap row r's
    // math), then the y hand-over buffers [2][nys warps][32][MF] (PIPE)
    extern __shared__ double sfo[];  // [warp][RING][NB][32]
    const int nwarps = blockDim.x >> 5;
    double *ysb = sfo + (size_t)nwarps * RING * NB * 32;
    // y hand-over slots only for warps with a reader in this CTA
    const int nys = nwarps - P.g.Wx;
    auto YS = [&](int buf, int w, int l) -> double * { return ysb + (((size_t)buf * nys + w) * 32 + l) * MF; };
    // (tensor path) per-warp staging rows [NB][32], then the A operands [M|Qc|Qp] and Qx
    double *stg_base = ysb + (PIPE ? (size_t)2 * nys * 32 * MF : 0);
    double *sA = stg_base + (USE_MMA ? (size_t)nwarps * NB * 32 : 0);
    double *sAx = sA + (size_t)MT * 8 * MMA::SA;
    // (pipe classes) tagged y-trace words of the previous CTA prefetched for the next row: [Wx][32][2 MF]
    double *spy = USE_MMA ? sAx + (size_t)MT * 8 * KSX * 4 : stg_base;
    if constexpr (USE_MMA) {
        for (int i = threadIdx.x; i < MT * 8 * KS * 4; i += blockDim.x) {
            const int q = i / (KS * 4), k = i % (KS * 4);
            double &dstA = sA[q * MMA::SA + k];
            double v = 0.0;
            if (q < NB && k < NB) v = P.tab.M[k * NB + q];  // the tensor path's M slot holds A^{-1}
            dstA = v;
        }
        for (int i = threadIdx.x; i < MT * 8 * KSX * 4; i += blockDim.x) {
            const int q = i / (KSX * 4), k = i % (KSX * 4);
            sAx[i] = (q < NB && k < MF && XA) ? P.tab.Q[0][k * NB + q] : 0.0;
        }
        __syncthreads();
    }

    const LatGeom &g = P.g;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int qx = warp % g.Wx, wy = warp / g.Wx;
    const int skew = (XA ? qx : 0) + (PIPE ? wy : 0);
    const int maxskew = (XA ? g.Wx - 1 : 0) + (PIPE ? g.Wy - 1 : 0);
    // Per-row synchronisation.  Without a pipe axis and with one CTA along x, the warp groups of
    // different batch indices (wy) are independent: each group of Wx skewed x-warps syncs on its
    // own named barrier, and no other CTA reads this task's progress.
    const bool group_sync = !PIPE && g.ngx == 1;
    // y traces across CTAs: tagged words on the FMA path; the tensor path (body diagonals) keeps
    // plain doubles published with a fence and a per-task row-progress counter — measured faster
    // there (its heavier rows hide the fence; the tagged words cost 1.8x the hand-over traffic)
    constexpr bool YLL = !USE_MMA;
    constexpr int MFP = (MF + 1) & ~1;  // per-lane stride of the plain y traces (16-byte multiple)
    // (tensor-path y traces: each producing warp publishes its own row progress, per (task, x-warp))
    uint64_t *const xll = reinterpret_cast<uint64_t *>(P.xbuf);
    uint64_t *const yll = reinterpret_cast<uint64_t *>(P.ybuf);
    // tagged y-trace words of (task, row) for this lane: [task][row][Wx][32][2 MF]
    auto ylslot = [&](int tk, int row) -> int64_t {
        const int64_t o = ((((int64_t)tk * g.rcap + row) * g.Wx + qx) * 32 + lane) * 2 * MF;
        PDG_CHECK_IDX(o + 2 * MF - 1, P.ybuf_elems, "lattice y trace slot");
        return o;
    };
    // tagged x-trace words of (task, row) for the warp's pipe index: [task][row][Wy][2 MF]
    auto xlslot = [&](int tk, int row) -> int64_t {
        const int64_t o = (((int64_t)tk * g.rcap + row) * g.Wy + wy) * 2 * MF;
        PDG_CHECK_IDX(o + 2 * MF - 1, P.xbuf_elems, "lattice x trace slot");
        return o;
    };
    // Otherwise (pipe classes) warps sync point to point through shared-memory step
    // counters instead of a CTA-wide barrier: before step t a warp needs its producers (x-1, y-1)
    // and its consumers (x+1, y+1) to have finished step t-1 (the consumers have then read the
    // double-buffered slot this step overwrites).  Warps may drift apart within that slack.
    const bool p2p = PIPE;
    volatile int *vdone = s_done;
    auto wait_done = [&](int w, int t_need) {
        if (vdone[w] >= t_need) return;
        PDG_SPIN_DECL(spins);
        while (vdone[w] < t_need) {
            __nanosleep(16);
            PDG_SPIN_TICK(spins, "lattice wait_done");
        }
    };
    auto step_begin = [&](int t) {
        if (!p2p || t == 0) return;
        if (lane == 0) {
            if (XA && qx > 0) wait_done(warp - 1, t - 1);
            if (XA && qx < g.Wx - 1) wait_done(warp + 1, t - (XR - 1));
            if (PIPE && wy > 0) wait_done(warp - g.Wx, t - 1);
            if (PIPE && wy < g.Wy - 1) wait_done(warp + g.Wx, t - 1);
        }
        __syncwarp();
        __threadfence_block();
    };
    auto step_sync = [&](int t) {
        if (group_sync) asm volatile("bar.sync %0, %1;" ::"r"(1 + wy), "r"(32 * g.Wx) : "memory");
        else if (p2p) {
            __syncwarp();
            __threadfence_block();
            if (lane == 0) vdone[warp] = t;
        } else __syncthreads();
    };

    for (;;) {
        if (threadIdx.x == 0) s_task = atomicAdd(P.ticket, 1);
        __syncthreads();
        const int ctask = s_task;
        if ((threadIdx.x & 31) == 0) s_done[threadIdx.x >> 5] = -1;
        __syncthreads();
        if (ctask >= g.ntasks) {
#ifdef PDG_LAT_TIMING
            if (blockIdx.x < 6 && lane == 0 && (warp == 0 || warp == nwarps - 1))
                printf("lat-timing ACT=%d cta %d warp %d: begin-wait %lld load %lld traces %lld mma1 %lld scan %lld mma2 %lld store %lld sync %lld\n",
                       ACT, (int)blockIdx.x, warp, tph[0], tph[1], tph[2], tph[3], tph[4], tph[5], tph[6], tph[7]);
#endif
            return;
        }
        // ticket order (pipe group, velocity, gx): every velocity's pipeline advances together, and
        // the tasks a task waits on (gx - 1: ticket - 1; previous pipe group: ticket - nvel ngx)
        // come earlier.
        // Chain segments (nseg > 1) are claimed in DESCENDING order: segment s waits for
        // segment s + 1 to have read its halo rows before overwriting them, so every wait still
        // targets an earlier ticket.
        const int per_gy = g.nvel * g.ngx;
        const int per_seg = g.ntasks / g.nseg;
        const int seg = g.nseg - 1 - ctask / per_seg;
        const int cts = ctask - (g.nseg - 1 - seg) * per_seg;
        const int gy = cts / per_gy, rem = cts - gy * per_gy;
        const int vi = rem / g.ngx, gx = rem - vi * g.ngx;
        const int task = seg * per_seg + (gy * g.nvel + vi) * g.ngx + gx;  // progress and traces
        // chain rows: stored [rs, r1), swept from r0 (the halo [r0, rs) starts from a zero trace)
        const int rs = seg * g.seglen;
        const int r0 = max(0, rs - g.halo);
        const int r1 = min(g.nc, rs + g.seglen);
        const int nrow = r1 - r0;
        bool hclear = !(seg < g.nseg - 1 && g.halo > 0);  // the next segment has read our last rows
        const LatVel &V = P.v[vi];
        const int ux = (gx * g.Wx + qx) * 32 + lane;  // x cell (XA) or x node
        const int uw = gy * g.Wy + wy;                // pipe cell, batch node or 0
        const bool wvalid = uw < g.nw && (gx * g.Wx + qx) * 32 < g.nlane;  // warp has work
        const bool valid = wvalid && ux < g.nlane;

        // unit coordinates: flow cell index on active axes, node index on inactive ones
        int ucell[3] = {0, 0, 0};
        ucell[0] = ux;
        if (PIPE) ucell[1] = uw;
        if (S::BA >= 0) ucell[S::BA] = uw;
        // address: base of the unit's first node + sum_t digit_t * dstep_t
        int64_t dstep[3] = {0, 0, 0};
        int64_t ibase = V.f_off;  // contribution of the non-chain coordinates
#pragma unroll
        for (int a = 0; a < D; ++a) {
            const int ta = S::t_of(a);
            if (ta >= 0) {
                dstep[ta] = (int64_t)V.sign[a] * g.stride[a];
                if (a != CA) {
                    const int64_t u0 = (int64_t)ucell[a] * N;
                    ibase += ((V.sign[a] > 0) ? u0 : g.L[a] - 1 - u0) * g.stride[a];
                }
            } else {
                ibase += (int64_t)ucell[a] * g.stride[a];
            }
        }
        const int64_t cstep = (int64_t)V.sign[CA] * g.stride[CA] * N;                        // one chain cell
        const int64_t cbase = (V.sign[CA] > 0) ? 0 : (g.L[CA] - 1) * g.stride[CA];          // chain cell 0

        // chain in-trace (the ghost f^b at the inflow face, a zero trace at a segment's halo start)
        double sc[MF];
#pragma unroll
        for (int j = 0; j < MF; ++j) sc[j] = 0.0;
        if (valid && r0 == 0) ghost_face<D, N, ACT, CA>(P, V, ucell, sc);

        double *wbuf = sfo + (size_t)warp * RING * NB * 32;
        // y traces of the previous CTA for row rr, if already published (speculative: the
        // producer normally runs ahead, so the global hand-over leaves the critical path)
        const bool ycons = PIPE && wy == 0 && gy > 0;
        bool ypf = false;  // this lane's y traces for the current row sit in spy
        // issue the copies of row rr into buffer rr & 1 (one commit group per row)
        auto prefetch = [&](int rr) {
            if (valid && rr < nrow) {
                const int64_t ubr = ibase + cbase + (int64_t)(r0 + rr) * cstep;
                double *dst = wbuf + (rr % RING) * NB * 32;
#pragma unroll
                for (int q = 0; q < NB; ++q) {
                    int64_t off = 0;
#pragma unroll
                    for (int tt = 0; tt < DA; ++tt) off += (int64_t)((q / ipow(N, tt)) % N) * dstep[tt];
                    PDG_CHECK_IDX(ubr + off, P.f_elems, "lattice row load f");
                    cp_async8(dst + ro(q, lane), P.f + ubr + off);
                }
                if constexpr (XA) {  // the row's x inflow ghost (first x warp of the first x group)
                    if (gx == 0 && qx == 0 && lane == 0) {
                        int uc[3] = {ucell[0], ucell[1], ucell[2]};
                        uc[CA] = r0 + rr;
#pragma unroll
                        for (int j = 0; j < MF; ++j) cp_async8(&gxs[wy][rr % RING][j], ghost_ptr<D, N, ACT, 0>(P, V, uc, j));
                    }
                }
            }
            if constexpr (PIPE) {
                // the previous pipe group's tagged y-trace words of row rr, copied whether or not they
                // have arrived: the tags tell at the use (normally they have: the producer runs ahead)
                ypf = false;
                if (YLL && ycons && rr < nrow) {
                    const uint64_t *ysrc = yll + ylslot(task - per_gy, rr);
                    double *yd = spy + ((size_t)qx * 32 + lane) * 2 * MF;
#pragma unroll
                    for (int h = 0; h < 2 * MF; h += 2) cp_async16_cg(yd + h, reinterpret_cast<const double *>(ysrc + h));
                    ypf = true;
                } else if (!YLL && ycons && rr < nrow && ld_acquire(P.progress + (int64_t)(task - per_gy) * 8 + qx) >= rr + 1) {
                    // plain traces: copied only once published (the producer normally runs ahead)
                    const int64_t yo = ((((int64_t)(task - per_gy) * g.rcap + rr) * g.Wx + qx) * 32 + lane) * MFP;
                    PDG_CHECK_IDX(yo + MFP - 1, P.ybuf_elems, "lattice y trace (plain)");
                    const double *ysrc = P.ybuf + yo;
                    double *yd = spy + ((size_t)qx * 32 + lane) * MFP;
#pragma unroll
                    for (int h = 0; h < MFP; h += 2) cp_async16_cg(yd + h, ysrc + h);
                    ypf = true;
                }
            }
            cp_async_commit();
        };

        for (int t = 0; t < nrow + maxskew; ++t) {
            PDG_TMARK(7);
            step_begin(t);
            PDG_TMARK(0);
            const int r = t - skew;  // row of the task (chain row r0 + r)
            if (r >= 0 && r < nrow && wvalid) {
                ucell[CA] = r0 + r;
                const int64_t ub = ibase + cbase + (int64_t)(r0 + r) * cstep;
                if (r == 0)
                    for (int k = 0; k < PFA; ++k) prefetch(k);
                if constexpr (PIPE) {
                    // PFA == 1: row r (and its prefetched y-trace words) have landed; the next row's
                    // prefetch is issued once the y-trace words have been read (below).  PFA == 0:
                    // the row is loaded now.
                    if constexpr (PFA == 0) prefetch(r);
                    cp_async_wait<0>();
                } else {
                    prefetch(r + PFA);
                    cp_async_wait<PFA>();  // row r has landed, rows r+1 .. r+PFA may be in flight
                }
                PDG_TMARK(1);
                // f_old of the unit stays in shared memory (per-lane column: conflict-free)
                const double *src = wbuf + (r % RING) * NB * 32;
                double fn[NB];
                auto fold = [&](int c) -> double { return src[ro(c, lane)]; };
                {
                    // pipe (y) in-trace
                    double sy[PIPE ? MF : 1];
                    if constexpr (PIPE) {
                        if (wy > 0) {
#pragma unroll
                            for (int j = 0; j < MF; ++j) sy[j] = YS((t - 1) & 1, warp - g.Wx, lane)[j];
                        } else if (gy > 0) {
                            if constexpr (YLL) {
                                uint64_t *ysl = yll + ylslot(task - per_gy, r);
                                const uint64_t *w = reinterpret_cast<const uint64_t *>(spy) + ((size_t)qx * 32 + lane) * 2 * MF;
                                if (ypf && ll_decode<MF>(w, sy, (uint32_t)r + 1u))
                                    ll_clear<MF>(ysl);  // empty the slot for the next launch
                                else
                                    ll_take<MF>(ysl, sy, (uint32_t)r + 1u);
                            } else if (ypf) {
#pragma unroll
                                for (int j = 0; j < MF; ++j) sy[j] = spy[((size_t)qx * 32 + lane) * MFP + j];
                            } else {
                                PDG_CHECK_IDX((int64_t)(task - per_gy) * 8 + qx, (int64_t)g.ntasks * 8, "lattice progress");
                                wait_progress(P.progress + (int64_t)(task - per_gy) * 8 + qx, r + 1);
                                const int64_t yo = ((((int64_t)(task - per_gy) * g.rcap + r) * g.Wx + qx) * 32 + lane) * MFP;
                                PDG_CHECK_IDX(yo + MFP - 1, P.ybuf_elems, "lattice y trace (plain)");
                                const double *ysrc = P.ybuf + yo;
#pragma unroll
                                for (int j = 0; j < MF; ++j) sy[j] = __ldcg(ysrc + j);
                            }
                        } else {
#pragma unroll
                            for (int j = 0; j < MF; ++j) sy[j] = 0.0;
                            if (valid) ghost_face<D, N, ACT, 1>(P, V, ucell, sy);
                        }
                        if (PFA > 0) prefetch(r + 1);  // overlaps the rest of the row
                    }
                    // x in-trace of the warp (lane 0's cell): previous x warp, previous x CTA or the ghost
                    double s0[XA ? MF : 1];
#pragma unroll
                    for (int j = 0; j < (XA ? MF : 1); ++j) s0[j] = 0.0;
                    if constexpr (XA) {
                        if (qx > 0) {
#pragma unroll
                            for (int j = 0; j < MF; ++j) s0[j] = xs[(t - 1) % XR][warp - 1][j];
                        } else if (gx > 0) {
                            // only lane 0 enters the x in-trace into the scan
                            if (lane == 0)
                                ll_take<MF>(xll + xlslot(task - 1, r), s0, (uint32_t)r + 1u);
                        } else if (lane == 0 && valid) {
#pragma unroll
                            for (int j = 0; j < MF; ++j) s0[j] = 2.0 * gxs[wy][r % RING][j];
                        }
                    }
                    // x scan: in a[] the zero-inflow x out-traces of the lanes' cells; returns the
                    // inclusive out-traces in a[] and every lane's true x in-trace in sin_[]
                    auto xscan = [&](double (&a)[MF], double (&sin_)[MF]) {
                        if (lane == 0) {
#pragma unroll
                            for (int j = 0; j < MF; ++j)
#pragma unroll
                                for (int i = 0; i < MF; ++i) a[i] = fma(P.tab.Bp[0][j * MF + i], s0[j], a[i]);
                        }
#pragma unroll
                        for (int sidx = 0; sidx < 5; ++sidx) {
                            if (sidx >= g.nscan) continue;  // powers below 2^-64: no effect in fp64 (uniform)
                            const int o = 1 << sidx;
                            double pv[MF];
#pragma unroll
                            for (int j = 0; j < MF; ++j) pv[j] = __shfl_up_sync(FULL, a[j], o);
                            if (lane >= o) {
#pragma unroll
                                for (int j = 0; j < MF; ++j)
#pragma unroll
                                    for (int i = 0; i < MF; ++i) a[i] = fma(P.tab.Bp[sidx][j * MF + i], pv[j], a[i]);
                            }
                        }
#pragma unroll
                        for (int j = 0; j < MF; ++j) {
                            const double up = __shfl_up_sync(FULL, a[j], 1);
                            sin_[j] = (lane == 0) ? s0[j] : up;
                        }
                        // the warp's x out-trace (lane 31's inclusive value) for the next x warp / CTA
                        if (lane == 31) {
#pragma unroll
                            for (int j = 0; j < MF; ++j) xs[t % XR][warp][j] = a[j];
                            if (qx == g.Wx - 1 && gx < g.ngx - 1)
                                ll_put<MF>(xll + xlslot(task, r), a, (uint32_t)r + 1u);
                        }
                    };
                    PDG_TMARK(2);
                    if constexpr (USE_MMA) {
                        // fp64 tensor cores (DMMA 8x8x4): the warp's 32 units are the N dimension.
                        //   R  = 2 F_old + (kappa_c/omega_0) E_c S_chain + (kappa_p/omega_0) E_p S_pipe
                        //   F0 = A^{-1} R          (NB x NB) (NB x 32)  = F_old + f_new without x inflow
                        //   F  = F0 + Q_x S_x_in   after the x scan     = F_old + f_new
                        // F0 and F are the old + new traces on the out-faces; f_new = F - F_old.  B
                        // operands from the warp's staging rows (R, then S_x_in), A from the CTA's tables.
                        const double *fsrc = wbuf + (r % RING) * NB * 32;
                        double *stg = stg_base + (size_t)warp * NB * 32;
#pragma unroll
                        for (int q = 0; q < NB; ++q) {
                            double v = 2.0 * fsrc[ro(q, lane)];
                            if ((q / ipow(N, TC)) % N == 0)  // chain in-face node
                                v = fma(g.kw[TC], sc[(q % ipow(N, TC)) + (q / ipow(N, TC + 1)) * ipow(N, TC)], v);
                            if constexpr (PIPE) {
                                if ((q / ipow(N, TY)) % N == 0)  // pipe in-face node
                                    v = fma(g.kw[TY], sy[(q % ipow(N, TY)) + (q / ipow(N, TY + 1)) * ipow(N, TY)], v);
                            }
                            stg[ro(q, lane)] = v;
                        }
                        __syncwarp();
                        double acc[MT][4][2];
#pragma unroll
                        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                            for (int nt = 0; nt < 4; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
                        const int gq = lane >> 2, tq = lane & 3;
#pragma unroll
                        for (int ks = 0; ks < KS; ++ks) {
                            const int k = ks * 4 + tq;
                            double b[4];
#pragma unroll
                            for (int nt = 0; nt < 4; ++nt) {
                                const int u = nt * 8 + gq;
                                b[nt] = (ks * 4 + 3 < NB || k < NB) ? stg[ro(k, u)] : 0.0;
                            }
#pragma unroll
                            for (int mt = 0; mt < MT; ++mt) {
                                const double av = sA[(mt * 8 + gq) * MMA::SA + k];
#pragma unroll
                                for (int nt = 0; nt < 4; ++nt) dmma884(acc[mt][nt], av, b[nt]);
                            }
                        }
                        auto spill = [&]() {  // accumulators -> staging rows [q][unit]
                            __syncwarp();
#pragma unroll
                            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                                for (int nt = 0; nt < 4; ++nt) {
                                    const int q = mt * 8 + gq;
                                    if (q < NB) {
                                        stg[ro(q, nt * 8 + 2 * tq)] = acc[mt][nt][0];
                                        stg[ro(q, nt * 8 + 2 * tq + 1)] = acc[mt][nt][1];
                                    }
                                }
                            __syncwarp();
                        };
                        spill();
                        PDG_TMARK(3);
                        if constexpr (XA) {
                            double a[MF], sin_[MF];
#pragma unroll
                            for (int j = 0; j < MF; ++j)
                                a[j] = valid ? stg[ro(j * N + N - 1, lane)] : 0.0;  // old + new, zero x inflow
                            xscan(a, sin_);
                            PDG_TMARK(4);
                            __syncwarp();
#pragma unroll
                            for (int j = 0; j < MF; ++j) stg[ro(j, lane)] = sin_[j];
                            __syncwarp();
#pragma unroll
                            for (int ks = 0; ks < KSX; ++ks) {
                                const int k = ks * 4 + tq;
                                double b[4];
#pragma unroll
                                for (int nt = 0; nt < 4; ++nt) b[nt] = (k < MF) ? stg[ro(k, nt * 8 + gq)] : 0.0;
#pragma unroll
                                for (int mt = 0; mt < MT; ++mt) {
                                    const double av = sAx[(mt * 8 + gq) * (KSX * 4) + k];
#pragma unroll
                                    for (int nt = 0; nt < 4; ++nt) dmma884(acc[mt][nt], av, b[nt]);
                                }
                            }
                            spill();
                        }
#pragma unroll
                        for (int q = 0; q < NB; ++q) fn[q] = stg[ro(q, lane)] - fsrc[ro(q, lane)];
                    } else {
                        // FMA pipe, same algebra as the tensor path: F0 = A^{-1} R with the rhs
                        // R = 2 f_old + (kappa_c/omega_0) E_c s_chain (+ pipe), streamed column by column
                        // into NB independent accumulators; F = F0 + Q_x s_x_in; f_new = F - f_old
                        auto rhs = [&](int c) -> double {
                            double v = 2.0 * fold(c);
                            if ((c / ipow(N, TC)) % N == 0)  // chain in-face node
                                v = fma(g.kw[TC], sc[(c % ipow(N, TC)) + (c / ipow(N, TC + 1)) * ipow(N, TC)], v);
                            if constexpr (PIPE) {
                                if ((c / ipow(N, TY)) % N == 0)  // pipe in-face node
                                    v = fma(g.kw[TY], sy[(c % ipow(N, TY)) + (c / ipow(N, TY + 1)) * ipow(N, TY)], v);
                            }
                            return v;
                        };
                        {
                            const double r0v = rhs(0);
#pragma unroll
                            for (int q = 0; q < NB; ++q) fn[q] = P.tab.M[q] * r0v;
                        }
#pragma unroll
                        for (int c = 1; c < NB; ++c) {
                            const double rc = rhs(c);
#pragma unroll
                            for (int q = 0; q < NB; ++q) fn[q] = fma(P.tab.M[c * NB + q], rc, fn[q]);
                        }
                        PDG_TMARK(3);
                        if constexpr (XA) {
                            double a[MF], sin_[MF];
#pragma unroll
                            for (int j = 0; j < MF; ++j) a[j] = valid ? fn[j * N + N - 1] : 0.0;  // old + new, zero x inflow
                            xscan(a, sin_);
                            PDG_TMARK(4);
#pragma unroll
                            for (int j = 0; j < MF; ++j)
#pragma unroll
                                for (int q = 0; q < NB; ++q) fn[q] = fma(P.tab.Q[0][j * NB + q], sin_[j], fn[q]);
                        }
#pragma unroll
                        for (int q = 0; q < NB; ++q) fn[q] -= fold(q);
                    }
                    // chain out-trace -> next row (registers)
#pragma unroll
                    for (int j = 0; j < MF; ++j) {
                        const int q = (j % ipow(N, TC)) + (j / ipow(N, TC)) * ipow(N, TC + 1) + (N - 1) * ipow(N, TC);
                        sc[j] = fold(q) + fn[q];
                    }
                    if constexpr (PIPE) {
                        double ty[MF];
#pragma unroll
                        for (int j = 0; j < MF; ++j) {
                            const int q = (j % ipow(N, TY)) + (j / ipow(N, TY)) * ipow(N, TY + 1) + (N - 1) * ipow(N, TY);
                            ty[j] = fold(q) + fn[q];
                        }
                        if (warp < nys) {
#pragma unroll
                            for (int j = 0; j < MF; ++j) YS(t & 1, warp, lane)[j] = ty[j];
                        }
                        if (wy == g.Wy - 1 && gy < g.ngy - 1) {
                            if constexpr (YLL) {
                                ll_put<MF>(yll + ylslot(task, r), ty, (uint32_t)r + 1u);
                            } else {
                                const int64_t yo = ((((int64_t)task * g.rcap + r) * g.Wx + qx) * 32 + lane) * MFP;
                                PDG_CHECK_IDX(yo + MFP - 1, P.ybuf_elems, "lattice y trace (plain)");
                                double *dst = P.ybuf + yo;
#pragma unroll
                                for (int j = 0; j < MF; ++j) __stcg(dst + j, ty[j]);
                                // the producing warp publishes its own row progress: __syncwarp orders
                                // the lanes' stores before lane 0's release (cumulative at gpu scope)
                                __syncwarp();
                                PDG_CHECK_IDX((int64_t)task * 8 + qx, (int64_t)g.ntasks * 8, "lattice progress");
                                if (lane == 0) st_release(P.progress + (int64_t)task * 8 + qx, r + 1);
                            }
                        }
                    }
                }
                PDG_TMARK(5);
                // the last halo rows of the next segment: wait until it has read their old values
                if (!hclear && r0 + r >= r1 - g.halo) {
                    PDG_CHECK_IDX(task + per_seg, g.ntasks, "lattice halo flag");
                    if (lane == 0) wait_progress(P.hdone + task + per_seg, 1);
                    __syncwarp();
                    hclear = true;
                }
                if (valid && r0 + r >= rs) {
#pragma unroll
                    for (int q = 0; q < NB; ++q) {
                        int64_t off = 0;
#pragma unroll
                        for (int tt = 0; tt < DA; ++tt) off += (int64_t)((q / ipow(N, tt)) % N) * dstep[tt];
                        PDG_CHECK_IDX(ub + off, P.f_elems, "lattice row store f");
                        __stcs(P.f + ub + off, fn[q]);
                    }
                }
            }
            PDG_TMARK(6);
            step_sync(t);
            // every warp has read the halo rows (cp.async waited): release them to the previous segment
            if (rs > r0 && t == rs - r0 - 1 + maxskew) {
                __syncthreads();
                PDG_CHECK_IDX(task, g.ntasks, "lattice halo flag");
                if (threadIdx.x == 0) st_release(P.hdone + task, 1);
            }
        }
        if (p2p) __syncthreads();  // every warp done with the task before the next ticket
        cp_async_wait<0>();
    }
}

// ---------------------------------------------------------------------------
// LBM collision fused with the moments (nranks == 1).
// ---------------------------------------------------------------------------
struct LbmParams {
    double v[kLbmMaxVel][3];
    double wgt[kLbmMaxVel];
    double inv_c2, inv_2c4, inv_2c2;
    double G[3];      // gravity vector of the source step (NEXT-3; zeros without a source)
};

// The local operators of one fused pass: S2(hs1), then C2 (f <- ca f + cb f^eq), then S2(hs2).
// S2(h) for the gravity source g_i = w_i v_i.(rho G)/c^2 (reading C24) is exact in closed form:
// g depends on f only through rho, which the source does not change (P g = (0, rho G)), so the
// CN equation f* = f + h/2 (g(f) + g(f*)) has the solution f* = f + h g(f) (one Picard
// iteration); it adds h rho G to the momentum.
struct LocalOps {
    double hs1, ca, cb, hs2;
};

// Macroscopic state at a node, prepared once; feq(i) evaluates the equilibrium of velocity i.
template <int D>
struct LbmNode {
    double rho, u[D], base;
    __device__ __forceinline__ LbmNode(const double (&w)[D + 1], const LbmParams &L)
    {
        rho = w[0];
        const double inv = 1.0 / rho;
        double uu = 0.0;
#pragma unroll
        for (int d = 0; d < D; ++d) {
            u[d] = w[1 + d] * inv;
            uu = fma(u[d], u[d], uu);
        }
        base = 1.0 - uu * L.inv_2c2;
    }
    __device__ __forceinline__ double feq(int i, const LbmParams &L) const
    {
        double uv = 0.0;
#pragma unroll
        for (int d = 0; d < D; ++d) uv = fma(u[d], L.v[i][d], uv);
        const double poly = fma(uv, fma(uv, L.inv_2c4, L.inv_c2), base);
        return L.wgt[i] * rho * poly;
    }
};

template <int D, int NV>
__device__ __forceinline__ void lbm_feq(const double (&w)[D + 1], const LbmParams &L, double (&feq)[NV])
{
    const LbmNode<D> nd(w, L);
#pragma unroll
    for (int i = 0; i < NV; ++i) feq[i] = nd.feq(i, L);
}

template <int D, int NV>
__device__ __forceinline__ void lbm_moments(const double (&fv)[NV], const LbmParams &L, double (&w)[D + 1])
{
#pragma unroll
    for (int c = 0; c <= D; ++c) w[c] = 0.0;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        w[0] += fv[i];
#pragma unroll
        for (int d = 0; d < D; ++d) w[1 + d] = fma(fv[i], L.v[i][d], w[1 + d]);
    }
}

// S2(hs1) C2 S2(hs2) at one node from its (full) moments w; fv in/out (local velocities only
// matter: entries outside [v0, v0 + nvl) are left as they are).  Composed into one update per
// velocity so that every velocity constant is used once (the compiler then keeps them as
// constant operands instead of hoisting ~4 nv of them into registers):
//   S2(h): f += h g, g_i = w_i v_i.(rho G)/c^2, rho u += h rho G   (rho unchanged)
//   => f <- ca f + (ca hs1 + hs2) g + cb f^eq(w + hs1 (0, rho G))
template <int D, int NV>
__device__ __forceinline__ void lbm_local_ops(double (&fv)[NV], double (&w)[D + 1], const LbmParams &L,
                                              const LocalOps &op)
{
    double gs[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
        gs[d] = w[0] * L.G[d] * L.inv_c2;
        w[1 + d] = fma(op.hs1 * w[0], L.G[d], w[1 + d]);
    }
    const double hg = fma(op.ca, op.hs1, op.hs2);
    if (op.cb != 0.0) {
        const LbmNode<D> nd(w, L);
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            double vg = 0.0;
#pragma unroll
            for (int d = 0; d < D; ++d) vg = fma(L.v[i][d], gs[d], vg);
            fv[i] = fma(op.cb, nd.feq(i, L), fma(hg * L.wgt[i], vg, op.ca * fv[i]));
        }
    } else {
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            double vg = 0.0;
#pragma unroll
            for (int d = 0; d < D; ++d) vg = fma(L.v[i][d], gs[d], vg);
            fv[i] = fma(hg * L.wgt[i], vg, op.ca * fv[i]);
        }
    }
}

__device__ __forceinline__ double ld_l1(const double *p)
{
    double v;
    asm volatile("ld.global.ca.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}

// Two phases: the moments from a first read of the node's NV values (short live ranges), then each
// value read again -- an L1 hit: the CTA's values were just loaded -- for its update.  ~60 registers
// instead of the 92-128 of a one-read kernel, so more threads per SM keep loads in flight without
// the spills of a register cap (one node per thread: no grid-stride loop, so the velocity constants
// stay constant-bank operands; the one-read kernel measured 0.90-0.99 of HBM against 1.01-1.03,
// DESIGN.md §12).
template <int D, int NV>
__global__ void __launch_bounds__(256, 4) relax_lbm2_kernel(double *__restrict__ f, int64_t nnodes,
                                                           const __grid_constant__ LbmParams L, const LocalOps op)
{
    const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= nnodes) return;
    double w[D + 1];
    {
        double fv[NV];
#pragma unroll
        for (int i = 0; i < NV; ++i) fv[i] = f[(int64_t)i * nnodes + x];
        lbm_moments<D, NV>(fv, L, w);
    }
    double gs[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
        gs[d] = w[0] * L.G[d] * L.inv_c2;
        w[1 + d] = fma(op.hs1 * w[0], L.G[d], w[1 + d]);
    }
    const double hg = fma(op.ca, op.hs1, op.hs2);
    const LbmNode<D> nd(w, L);
    const double cb = op.cb;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        double vg = 0.0;
#pragma unroll
        for (int d = 0; d < D; ++d) vg = fma(L.v[i][d], gs[d], vg);
        const double fs = fma(hg * L.wgt[i], vg, op.ca * ld_l1(f + (int64_t)i * nnodes + x));
        __stcs(f + (int64_t)i * nnodes + x, (cb != 0.0) ? fma(cb, nd.feq(i, L), fs) : fs);
    }
}

// Partial moments of the local velocities [v0, v0 + nvl) (sharded path, pdg_moments).
template <int D, int NV>
__global__ void __launch_bounds__(256) partial_moments_lbm_kernel(const double *__restrict__ f, double *__restrict__ w,
                                                                  int64_t nnodes, int64_t count, int v0, int nvl,
                                                                  const __grid_constant__ LbmParams L)
{
    // one node per thread (no grid-stride loop: the velocity constants stay constant-bank operands
    // instead of being hoisted into registers); a chunk of `count` nodes, stride nnodes
    {
        const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        if (x >= count) return;
        double fv[NV];
#pragma unroll
        for (int i = 0; i < NV; ++i) fv[i] = (i >= v0 && i < v0 + nvl) ? __ldcs(f + (int64_t)(i - v0) * nnodes + x) : 0.0;
        double wl[D + 1];
        lbm_moments<D, NV>(fv, L, wl);
#pragma unroll
        for (int c = 0; c <= D; ++c) __stcs(w + (int64_t)c * nnodes + x, wl[c]);
    }
}

// Collision of the local velocities from reduced moments w (sharded path): w comes from memory,
// so every local velocity is loaded, updated and stored in turn (no per-node f array).
template <int D, int NV>
__global__ void __launch_bounds__(256, 2) relax_from_w_lbm_kernel(double *__restrict__ f, const double *__restrict__ w,
                                                                  int64_t nnodes, int64_t count, int v0, int nvl,
                                                                  const __grid_constant__ LbmParams L, const LocalOps op)
{
    const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= count) return;
    double wl[D + 1];
#pragma unroll
    for (int c = 0; c <= D; ++c) wl[c] = __ldcs(w + (int64_t)c * nnodes + x);
    // S2(hs1) C2 S2(hs2) composed (lbm_local_ops): f <- ca f + (ca hs1 + hs2) g + cb f^eq(w')
    double gs[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
        gs[d] = wl[0] * L.G[d] * L.inv_c2;
        wl[1 + d] = fma(op.hs1 * wl[0], L.G[d], wl[1 + d]);
    }
    const double hg = fma(op.ca, op.hs1, op.hs2);
    const LbmNode<D> nd(wl, L);
#pragma unroll
    for (int i = 0; i < NV; ++i)
        if (i >= v0 && i < v0 + nvl) {
            double *p = f + (int64_t)(i - v0) * nnodes + x;
            double vg = 0.0;
#pragma unroll
            for (int d = 0; d < D; ++d) vg = fma(L.v[i][d], gs[d], vg);
            const double fs = fma(hg * L.wgt[i], vg, op.ca * __ldcs(p));
            __stcs(p, (op.cb != 0.0) ? fma(op.cb, nd.feq(i, L), fs) : fs);
        }
}

// f_i = f^eq_i(w) for the local velocities.
template <int D, int NV>
__global__ void __launch_bounds__(256) equilibrium_lbm_kernel(double *__restrict__ f, const double *__restrict__ w,
                                                              int64_t nnodes, int v0, int nvl,
                                                              const __grid_constant__ LbmParams L)
{
    // one node per thread (no grid-stride loop: the velocity constants stay constant-bank operands
    // instead of being hoisted into registers)
    {
        const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        if (x >= nnodes) return;
        double wl[D + 1];
#pragma unroll
        for (int c = 0; c <= D; ++c) wl[c] = w[(int64_t)c * nnodes + x];
        double feq[NV];
        lbm_feq<D, NV>(wl, L, feq);
#pragma unroll
        for (int i = 0; i < NV; ++i)
            if (i >= v0 && i < v0 + nvl) __stcs(f + (int64_t)(i - v0) * nnodes + x, feq[i]);
    }
}

// Inflow planes of the local velocities: plane k of velocity i (v_i^k != 0) holds f^eq_i(wb)
// at the nodes of its inflow face (lo face for v^k > 0, hi face for v^k < 0).
struct LatInflowParams {
    double *fb;
    const double *wb;
    int64_t nnodes, plane_stride;
    int64_t L[3], stride[3];
    int32_t v0, nvl, dim;
    LbmParams lbm;
};

template <int D, int NV>
__global__ void __launch_bounds__(256) lattice_inflow_kernel(const __grid_constant__ LatInflowParams P)
{
    const int j = blockIdx.y;         // local velocity
    const int k = blockIdx.z;         // plane axis
    const int i = P.v0 + j;
    const double vk = P.lbm.v[i][k];
    if (vk == 0.0) return;
    const int64_t np = P.nnodes / P.L[k];
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= np) return;
    // plane index -> node coordinates (axis k removed, remaining axes in x, y, z order)
    int64_t c[3] = {0, 0, 0};
    int64_t rest = idx;
#pragma unroll
    for (int a = 0; a < D; ++a) {
        if (a == k) continue;
        c[a] = rest % P.L[a];
        rest /= P.L[a];
    }
    c[k] = (vk > 0.0) ? 0 : P.L[k] - 1;
    int64_t node = 0;
#pragma unroll
    for (int a = 0; a < D; ++a) node += c[a] * P.stride[a];
    double wl[D + 1];
#pragma unroll
    for (int cc = 0; cc <= D; ++cc) wl[cc] = P.wb[(int64_t)cc * P.nnodes + node];
    double feq[NV];
    lbm_feq<D, NV>(wl, P.lbm, feq);
    double val = 0.0;
#pragma unroll
    for (int q = 0; q < NV; ++q)
        if (q == i) val = feq[q];
    P.fb[(int64_t)j * D * P.plane_stride + (int64_t)k * P.plane_stride + idx] = val;
}

}  // namespace pdg
