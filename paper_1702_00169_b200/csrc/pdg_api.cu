// libpdg: C-ABI of the B200-native PDG hot path (declared in include/pdg.h).
//
// The host side validates the problem statement, precomputes the cell
// blocks (pdg_tables.hpp) and enqueues the sm_100a kernels of pdg_kernels.cuh on the
// caller's stream.  No device allocation, no host fallback: every arithmetic step of
// the hot path runs in these kernels.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: one range per operator pass (nsys / ncu --nvtx)

#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/pdg.h"
#include "pdg_comm.hpp"
#include "pdg_kernels.cuh"
#include "pdg_lattice.cuh"
#include "pdg_tables.hpp"

#include <cstdlib>
#include <map>
#include <tuple>
#include <utility>

#ifndef PDG_VERSION
#define PDG_VERSION "0.1.0"
#endif

namespace {

thread_local std::string g_last_error;

pdg_status fail(pdg_status s, const std::string &msg)
{
    g_last_error = msg;
    return s;
}

// NVTX range for the duration of a scope (no-op without a profiler attached)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

#define PDG_CUDA_TRY(expr)                                                                             \
    do {                                                                                               \
        cudaError_t e_ = (expr);                                                                       \
        if (e_ != cudaSuccess)                                                                         \
            return fail(PDG_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));               \
    } while (0)

constexpr int kMaxSlabs = 64;
constexpr int kMaxChunks = 8;  // node chunks of the pipelined sharded collision

struct Geometry {
    int dim = 0, p = 0, n = 0, m = 0, nv = 0, nvl = 0, v0 = 0;
    int64_t ncell[3] = {1, 1, 1};  // LOCAL cells per axis (the rank's slab along the outer axis)
    int64_t L[3] = {1, 1, 1};      // local nodes per axis
    int64_t stride[3] = {1, 1, 1}; // element stride of each axis in the local node grid
    int64_t nnodes = 0, plane_stride = 0;  // local
    int64_t gnnodes = 0;                   // global
    double h[3] = {1, 1, 1};
    // PDG_DECOMP_ZSLAB
    int zslab = 0;          // 1 if the z-slab decomposition is active
    int outer = 0;          // slowest axis (dim - 1)
    int nslab = 1;          // global number of slabs
    int slab0 = 0;          // first global slab of this rank
    int nslab_local = 1;    // slabs of this rank
    int64_t gncell_outer = 0, cell_begin = 0;
    int64_t slab_begin[kMaxSlabs + 1] = {0};  // global cell plane where slab s starts
    size_t carry_doubles = 0;                 // one carry/inflow buffer (doubles)
    // lattice velocity sets (PDG_FLUX_LBM, NEXT-2)
    int async_host = 0;                       // PDG_ASYNC_HOST
    int lattice = 0;                          // 1: general velocities, fb = [nvl][dim][plane_stride]
    int nplanes = 1;                          // inflow planes per velocity in fb
    size_t lat_ints = 0;                      // ticket + progress counters (sum over classes)
    size_t lat_xbuf = 0, lat_ybuf = 0;        // boundary trace buffers (doubles, sum over classes: the
                                              // classes run concurrently on their own streams)
    int lat_cta[2] = {0, 0};                  // pdg_problem.lattice_cta (0: default plan)
    int lat_seg = 0;                          // pdg_problem.lattice_segment
};

// Work decomposition of one active-axis class of lattice velocities (pdg_lattice.cuh).
struct LatPlan {
    int act = 0, d = 0, nvel = 0;
    int vel[pdg::kLatMaxVel] = {0};  // local velocity indices
    int Wx = 1, Wy = 1, ngx = 1, ngy = 1, nlane = 1, nw = 1, nc = 1, ntasks = 0;
    int nseg = 1, seglen = 1;  // chain segments (truncated-dependency split) and their rows
    int rcap = 1;              // chain rows per task the trace buffers hold
    size_t xbuf = 0, ybuf = 0;       // doubles
    size_t ints_off = 0, xbuf_off = 0, ybuf_off = 0;  // this class's slices of the work buffers
};

int popcount3(int a) { return (a & 1) + ((a >> 1) & 1) + ((a >> 2) & 1); }

void plan_lattice(const Geometry &g, LatPlan &P)
{
    const int D = g.dim, act = P.act;
    const int XA = act & 1, YA = (act >> 1) & 1, ZA = (D == 3) ? ((act >> 2) & 1) : 0;
    const int CA = ZA ? 2 : 1;
    const int PIPE = (D == 3 && ZA && YA) ? 1 : 0;
    const int BA = (D == 3 && !ZA) ? 2 : ((D == 3 && !YA) ? 1 : -1);
    P.d = XA + YA + ZA;
    P.nlane = (int)(XA ? g.ncell[0] : g.L[0]);
    P.nw = (int)(PIPE ? g.ncell[1] : (BA >= 0 ? g.L[BA] : 1));
    P.nc = (int)g.ncell[CA];
    if (XA) {
        // x carries a dependency: the CTA's x-warps are skewed, keep them few enough that the
        // grid still has tasks for every SM (2-D grids: one warp per CTA along x)
        // (body diagonals, x and pipe both active: 2 x-warps by 4 pipe warps measured best, D3Q15
        // 128^3 12.32 -> 11.82 ms per step against 4 x 2; tools/gpu/bdshape.sh.  2-D diagonals:
        // 4 x-warps, 2-3 % faster than 8 with the chain segments; tools/gpu/wsweep.sh)
        P.Wx = std::min(PIPE ? 2 : (D == 2 ? 4 : 8), (P.nlane + 31) / 32);
        P.Wy = std::max(1, std::min(8 / P.Wx, P.nw));
    } else {
        // lanes over independent x nodes: spend the warps on the pipe axis (y hand-over in smem)
        P.Wy = std::max(1, std::min(8, P.nw));
        P.Wx = std::max(1, std::min(8 / P.Wy, (P.nlane + 31) / 32));
    }
    // pdg_problem.lattice_cta: a forced CTA shape (tests run the cross-CTA hand-over paths on
    // small grids with it)
    if (g.lat_cta[0] >= 1 && g.lat_cta[1] >= 1) {
        P.Wx = std::min(g.lat_cta[0], std::max(1, (P.nlane + 31) / 32));
        P.Wy = std::min(g.lat_cta[1], P.nw);
    }
    if (P.d == 3 && g.n == 4) {  // p = 3 body diagonals: ~50 KB of shared memory per warp (no row prefetch)
        P.Wx = std::min(P.Wx, 2);
        P.Wy = std::max(1, std::min(P.Wy, 4 / P.Wx));
    }
    P.ngx = (P.nlane + 32 * P.Wx - 1) / (32 * P.Wx);
    P.ngy = (P.nw + P.Wy - 1) / P.Wy;
    // Chain segments.  A class without a pipe axis whose tasks cannot fill the GPU (2-D grids:
    // one task per velocity and x group) is latency-bound by its serial chain; it is cut into
    // segments swept concurrently, each starting kHalo rows early from a zero chain trace.  The
    // halo depth comes from a norm bound of the chain operator per launch (lattice_chain_halo:
    // the truncated traces agree with the exact ones to 2^-64); a launch whose bound exceeds the
    // segment length runs unsegmented.  Planned for the 148 SMs of a B200 at 16 warps per SM (the
    // segments only change how much of the chain one task walks, not the result).
    P.nseg = 1;
    P.seglen = P.nc;
    if (XA && !PIPE) {
        // resident CTAs: 16 warps per SM on the FMA path (registers capped for 2 CTAs of 8 warps)
        const int base = P.nvel * P.ngx * P.ngy, slots = 148 * std::max(1, 16 / (P.Wx * P.Wy));
        int Ls = 0;
        if (g.lat_seg != 0) Ls = std::max(0, g.lat_seg);  // pdg_problem.lattice_segment (< 0: never)
        else if (2 * base <= slots && P.nc >= 128) {
            const int ns = std::min(slots / base, P.nc / 64);  // segments of >= 64 rows
            Ls = (P.nc + ns - 1) / ns;
        }
        if (Ls > 0 && Ls < P.nc) {
            P.seglen = Ls;
            P.nseg = (P.nc + Ls - 1) / Ls;
        }
    }
    P.rcap = (P.nseg > 1) ? std::min(P.nc, 2 * P.seglen) : P.nc;  // segment + a halo of at most one segment
    P.ntasks = P.nvel * P.ngx * P.ngy * P.nseg;
    int mf = 1;
    for (int t = 1; t < P.d; ++t) mf *= g.n;
    // boundary traces: x traces cross CTAs as tagged 64-bit words (two per double, pdg_lattice.cuh
    // ll_put / ll_take); y traces as tagged words (FMA path) or plain doubles (tensor path)
    P.xbuf = (XA && P.ngx > 1) ? (size_t)P.ntasks * P.rcap * P.Wy * 2 * mf : 0;
    P.ybuf = (PIPE && P.ngy > 1) ? (size_t)P.ntasks * P.nc * P.Wx * 32 * 2 * mf : 0;
    P.xbuf = (P.xbuf + 1) & ~(size_t)1;  // keep every slice 16-byte aligned
}

// Active-axis mask of a lattice velocity (bit k set if v_k != 0).
int act_mask(const double *v, int dim)
{
    int a = 0;
    for (int k = 0; k < dim; ++k)
        if (v[k] != 0.0) a |= 1 << k;
    return a;
}

void lattice_classes(const Geometry &g, const double *vel, std::vector<LatPlan> &out)
{
    out.clear();
    for (int j = 0; j < g.nvl; ++j) {
        const int act = act_mask(vel + 3 * (g.v0 + j), g.dim);
        if (popcount3(act) < 2) continue;
        LatPlan *pl = nullptr;
        for (auto &q : out)
            if (q.act == act && q.nvel < pdg::kLatMaxVel) pl = &q;
        if (!pl) {
            out.emplace_back();
            pl = &out.back();
            pl->act = act;
        }
        pl->vel[pl->nvel++] = j;
    }
    size_t io = 0, xo = 0, yo = 0;
    for (auto &q : out) {
        plan_lattice(g, q);
        q.ints_off = io;
        q.xbuf_off = xo;
        q.ybuf_off = yo;
        io += (((size_t)9 * q.ntasks + 1 + 63) / 64) * 64;  // ticket, progress[ntasks][8 x-warps], halo flags[ntasks]
        xo += q.xbuf;
        yo += q.ybuf;
    }
}

constexpr int kMaxTables = 16;
constexpr int kMaxLatTables = 16;  // distinct (class, dt') of the large (p = 3 body-diagonal) block tables
constexpr size_t kLatBigTableDoubles = sizeof(pdg::LatTab<4, 3>) / sizeof(double);

// tau > 0: eq collision_cn divides by 2 tau + h; a substep with 2 tau + h <= 0 (the negative
// middle step of M4, or dt < 0) has no meaningful collision factor (SPEC's tau > |dt| gamma guard)
bool collision_step_ok(double tau, double h) { return tau == 0.0 || 2.0 * tau + h > 0.0; }

// An operator of a scheme: T(h) = T2(h) on every velocity, C(h) = C2(h), S(h) = S2(h).
struct Op {
    int kind;  // 0: T, 1: C, 2: S (source)
    double h;
};
void append_scheme(std::vector<Op> &ops, int scheme, double dt);

pdg_status validate(const pdg_problem *p, Geometry *g)
{
    if (!p) return fail(PDG_E_INVALID_ARGUMENT, "problem is NULL");
    if (p->dim != 2 && p->dim != 3) return fail(PDG_E_DIMENSION, "dim must be 2 or 3");
    if (p->degree < 1 || p->degree > 3) return fail(PDG_E_DEGREE, "degree must be 1, 2 or 3");
    if (!(p->lambda > 0.0) || !std::isfinite(p->lambda)) return fail(PDG_E_INVALID_ARGUMENT, "lambda must be > 0");
    if (!(p->dt != 0.0) || !std::isfinite(p->dt)) return fail(PDG_E_INVALID_ARGUMENT, "dt must be finite and != 0");
    if (!(p->tau >= 0.0) || !std::isfinite(p->tau)) return fail(PDG_E_INVALID_ARGUMENT, "tau must be >= 0");
    if (p->scheme != PDG_SCHEME_M2 && p->scheme != PDG_SCHEME_M2KIN && p->scheme != PDG_SCHEME_M4 &&
        p->scheme != PDG_SCHEME_M2S)
        return fail(PDG_E_INVALID_ARGUMENT, "unknown scheme");
    if (p->source != PDG_SOURCE_NONE) {
        if (p->source != PDG_SOURCE_GRAVITY) return fail(PDG_E_INVALID_ARGUMENT, "unknown source kind");
        if (p->flux != PDG_FLUX_LBM) return fail(PDG_E_UNSUPPORTED, "the gravity source is implemented for PDG_FLUX_LBM");
        if (!p->source_params || p->n_source_params < p->dim)
            return fail(PDG_E_INVALID_ARGUMENT, "gravity needs source_params = G[dim]");
        for (int d = 0; d < p->dim; ++d)
            if (!std::isfinite(p->source_params[d])) return fail(PDG_E_INVALID_ARGUMENT, "G must be finite");
    }
    if (p->scheme == PDG_SCHEME_M2S && p->source == PDG_SOURCE_NONE)
        return fail(PDG_E_INVALID_ARGUMENT, "PDG_SCHEME_M2S needs a source");
    if (p->tau > 0.0) {
        std::vector<Op> ops;
        append_scheme(ops, p->scheme, p->dt);
        for (const Op &o : ops)
            if (o.kind == 1 && !collision_step_ok(p->tau, o.h))
                return fail(PDG_E_INVALID_ARGUMENT, "tau > 0 needs 2 tau + h > 0 for every collision substep h of the "
                                                    "scheme (eq collision_cn, P:453)");
    }
    if (p->nranks < 1 || p->rank < 0 || p->rank >= p->nranks) return fail(PDG_E_INVALID_ARGUMENT, "bad rank/nranks");
    g->async_host = (p->flags & PDG_ASYNC_HOST) ? 1 : 0;
    if (p->lattice_cta[0] < 0 || p->lattice_cta[1] < 0 || p->lattice_cta[0] * p->lattice_cta[1] > 8 ||
        ((p->lattice_cta[0] == 0) != (p->lattice_cta[1] == 0)))
        return fail(PDG_E_INVALID_ARGUMENT, "lattice_cta: both 0 (default) or both >= 1 with a product <= 8");
    g->lat_cta[0] = p->lattice_cta[0];
    g->lat_cta[1] = p->lattice_cta[1];
    g->lat_seg = p->lattice_segment;
    g->dim = p->dim;
    g->p = p->degree;
    g->n = p->degree + 1;
    for (int d = 0; d < 3; ++d) {
        const int64_t nc = p->ncell[d];
        if (d < p->dim) {
            if (nc < 1) return fail(PDG_E_INVALID_ARGUMENT, "ncell must be >= 1");
            if (!(p->hi[d] > p->lo[d])) return fail(PDG_E_INVALID_ARGUMENT, "hi must be > lo");
            g->ncell[d] = nc;
            g->L[d] = nc * g->n;
            g->h[d] = (p->hi[d] - p->lo[d]) / (double)nc;
        } else {
            g->ncell[d] = 1;
            g->L[d] = 1;
        }
    }
    // x-sweep line length must fit the int32 cell counter
    if (g->ncell[0] > (int64_t)1 << 30 || g->ncell[1] > (int64_t)1 << 30 || g->ncell[2] > (int64_t)1 << 30)
        return fail(PDG_E_INVALID_ARGUMENT, "too many cells along an axis");
    g->stride[0] = 1;
    g->stride[1] = g->L[0];
    g->stride[2] = g->L[0] * g->L[1];
    g->nnodes = g->L[0] * g->L[1] * g->L[2];
    int64_t ps = 0;
    for (int d = 0; d < p->dim; ++d) ps = std::max(ps, g->nnodes / g->L[d]);
    g->plane_stride = ps;

    // flux model and m
    int m_expect = 0;
    if (p->flux == PDG_FLUX_LINEAR_ADVECTION) {
        m_expect = 1;
        if (!p->flux_params || p->n_flux_params < p->dim)
            return fail(PDG_E_FLUX_MODEL, "advection needs flux_params = a[dim]");
    } else if (p->flux == PDG_FLUX_EULER) {
        m_expect = p->dim + 2;
        if (!p->flux_params || p->n_flux_params < 1 || !(p->flux_params[0] > 1.0))
            return fail(PDG_E_FLUX_MODEL, "Euler needs flux_params = {gamma > 1}");
    } else if (p->flux == PDG_FLUX_ISOTHERMAL) {
        m_expect = p->dim + 1;
        if (!p->flux_params || p->n_flux_params < 1 || !(p->flux_params[0] > 0.0))
            return fail(PDG_E_FLUX_MODEL, "isothermal needs flux_params = {c > 0}");
    } else if (p->flux == PDG_FLUX_LBM) {
        m_expect = p->dim + 1;
        if (!p->flux_params || p->n_flux_params < 1 + p->nv || !(p->flux_params[0] > 0.0))
            return fail(PDG_E_FLUX_MODEL, "LBM needs flux_params = {c > 0, w_0 .. w_{nv-1}}");
    } else {
        return fail(PDG_E_FLUX_MODEL, "unknown flux model");
    }
    if (p->m != m_expect) return fail(PDG_E_FLUX_MODEL, "m does not match the flux model");
    g->m = p->m;

    if (p->flux == PDG_FLUX_LBM) {
        // lattice velocity set (NEXT-2): components in {0, +-lambda}
        g->lattice = 1;
        g->nplanes = p->dim;
        if (!p->vel) return fail(PDG_E_INVALID_ARGUMENT, "vel is NULL");
        const bool nv_ok = (p->dim == 2) ? (p->nv == 9) : (p->nv == 15 || p->nv == 19 || p->nv == 27);
        if (!nv_ok) return fail(PDG_E_UNSUPPORTED, "LBM lattices compiled: D2Q9, D3Q15, D3Q19, D3Q27");
        for (int i = 0; i < p->nv; ++i) {
            for (int d = 0; d < 3; ++d) {
                const double v = p->vel[3 * i + d];
                const bool ok = (d < p->dim) ? (v == 0.0 || v == p->lambda || v == -p->lambda) : (v == 0.0);
                if (!ok) return fail(PDG_E_VELOCITY_SET, "lattice velocity components must be 0 or +-lambda");
            }

        }
        if (p->decomposition == PDG_DECOMP_ZSLAB && p->nranks * std::max(1, p->slabs_per_rank) > 1)
            return fail(PDG_E_UNSUPPORTED, "the z-slab decomposition is implemented for axis-aligned sets only");
    } else {
    // velocity set: canonical vectorial D2Q4 / D3Q6 per component (reading C6)
    if (p->nv != p->m * 2 * p->dim) return fail(PDG_E_VELOCITY_SET, "nv must be m * 2 * dim");
    if (p->nv > pdg::kMaxVel) return fail(PDG_E_VELOCITY_SET, "too many velocities");
    if (!p->vel || !p->comp) return fail(PDG_E_INVALID_ARGUMENT, "vel/comp are NULL");  // comp optional for LBM
    for (int i = 0; i < p->nv; ++i) {
        const int c = i / (2 * p->dim), k = (i % (2 * p->dim)) / 2, s = i % 2;
        if (p->comp[i] != c) return fail(PDG_E_VELOCITY_SET, "comp[i] must be i / (2 dim)");
        for (int d = 0; d < 3; ++d) {
            const double expect = (d == k) ? (s ? -p->lambda : p->lambda) : 0.0;
            if (p->vel[3 * i + d] != expect)
                return fail(PDG_E_VELOCITY_SET, "velocity " + std::to_string(i) +
                                                    " must be (s ? -lambda : lambda) e_k, i = c*2D + 2k + s");
        }
    }
    }
    g->nv = p->nv;
    g->gnnodes = g->nnodes;
    if (p->decomposition == PDG_DECOMP_VELOCITY) {
        // contiguous velocity blocks; sizes differ by at most one (the lattice sets have odd n_v)
        if (p->nranks > p->nv) return fail(PDG_E_INVALID_ARGUMENT, "more ranks than velocities");
        const int base = p->nv / p->nranks, extra = p->nv % p->nranks;
        g->nvl = base + (p->rank < extra ? 1 : 0);
        g->v0 = p->rank * base + std::min(p->rank, extra);
        g->gncell_outer = g->ncell[p->dim - 1];
        if (g->lattice) {
            std::vector<LatPlan> cls;
            lattice_classes(*g, p->vel, cls);
            for (const auto &q : cls) {
                g->lat_ints = std::max(g->lat_ints, q.ints_off + (((size_t)9 * q.ntasks + 1 + 63) / 64) * 64);
                g->lat_xbuf = std::max(g->lat_xbuf, q.xbuf_off + q.xbuf);
                g->lat_ybuf = std::max(g->lat_ybuf, q.ybuf_off + q.ybuf);
            }
        }
        return PDG_OK;
    }
    if (p->decomposition != PDG_DECOMP_ZSLAB) return fail(PDG_E_INVALID_ARGUMENT, "unknown decomposition");
    // z-slab decomposition: all velocities local, the rank owns a range of cell planes of the outer axis
    const int outer = p->dim - 1;
    const int spr = p->slabs_per_rank < 1 ? 1 : p->slabs_per_rank;
    const int64_t S = (int64_t)p->nranks * spr;
    const int64_t Nout = g->ncell[outer];
    if (S > kMaxSlabs) return fail(PDG_E_INVALID_ARGUMENT, "at most 64 slabs");
    if (S > Nout) return fail(PDG_E_INVALID_ARGUMENT, "more slabs than cell planes");
    g->zslab = (S > 1) ? 1 : 0;
    g->outer = outer;
    g->nslab = (int)S;
    g->slab0 = p->rank * spr;
    g->nslab_local = spr;
    g->gncell_outer = Nout;
    for (int64_t sl = 0; sl <= S; ++sl) g->slab_begin[sl] = (sl * Nout) / S;
    g->cell_begin = g->slab_begin[g->slab0];
    const int64_t cnt = g->slab_begin[g->slab0 + spr] - g->cell_begin;
    g->nvl = p->nv;
    g->v0 = 0;
    g->ncell[outer] = cnt;
    g->L[outer] = cnt * g->n;
    g->stride[0] = 1;
    g->stride[1] = g->L[0];
    g->stride[2] = g->L[0] * g->L[1];
    g->nnodes = g->L[0] * g->L[1] * g->L[2];
    int64_t ps2 = 0;
    for (int d = 0; d < p->dim; ++d) ps2 = std::max(ps2, g->nnodes / g->L[d]);
    g->plane_stride = ps2;
    const int64_t plane = g->nnodes / g->L[outer];  // lines along the outer axis
    const int nvo = 2 * p->m;                         // velocities along the outer axis
    g->carry_doubles = (size_t)S * nvo * 2 * (size_t)plane;
    return PDG_OK;
}

size_t lat_ints_bytes(const Geometry &g) { return ((g.lat_ints * sizeof(int) + 255) / 256) * 256; }

size_t work_bytes_of(const Geometry &g)
{
    size_t b = 256;
    if (g.zslab) b += sizeof(double) * 2 * g.carry_doubles;  // outgoing carries, exact inflows
    if (g.lattice) b += lat_ints_bytes(g) + sizeof(double) * (g.lat_xbuf + g.lat_ybuf);
    if (g.lattice && g.n == 4 && g.dim == 3) b += sizeof(double) * kMaxLatTables * kLatBigTableDoubles;
    b = ((b + 255) / 256) * 256;
    if (g.async_host) b += sizeof(double) * (size_t)g.m * (size_t)g.nnodes;  // PDG_ASYNC_HOST upload staging
    return b;
}

// byte offset of the PDG_ASYNC_HOST staging region in the work buffer
size_t w_stage_offset(const Geometry &g)
{
    Geometry h = g;
    h.async_host = 0;
    return ((work_bytes_of(h) + 255) / 256) * 256;
}

void fill_sizes(const Geometry &g, pdg_sizes *out)
{
    out->f_elems = (size_t)g.nvl * (size_t)g.nnodes;
    out->fb_elems = (size_t)g.nvl * (size_t)g.nplanes * (size_t)g.plane_stride;
    out->w_elems = (size_t)g.m * (size_t)g.nnodes;
    out->work_bytes = work_bytes_of(g);
    out->nnodes = g.gnnodes;
    out->plane_stride = g.plane_stride;
    out->nv_local = g.nvl;
    out->v_begin = g.v0;
    out->nnodes_local = g.nnodes;
    out->cell_begin = g.cell_begin;
    out->cell_count = g.ncell[g.dim - 1];
}

struct ProfRec {
    int kind;
    int ev;        // index of the start event; stop = ev + 1
    double bytes;  // algorithmic bytes of the launch
};

struct Profiler {
    bool on = false;       // events allocated (PDG_PROFILE)
    bool paused = false;   // pdg_profile_enable(c, 0)
    std::vector<cudaEvent_t> ev;
    std::vector<ProfRec> recs;
    int next = 0;
};

}  // namespace

struct pdg_ctx {
    Geometry g;
    pdg_problem prob;
    std::vector<double> vel;
    std::vector<int32_t> comp;
    double fparams[3] = {0, 0, 0};
    double *f = nullptr, *fb = nullptr, *w = nullptr;
    unsigned long long *counter = nullptr;
    cudaStream_t stream = nullptr;
    bool state_set = false;
    // PDG_ASYNC_HOST
    double *w_stage = nullptr;             // upload staging of pdg_set_equilibrium
    cudaStream_t copy_stream = nullptr;    // downloads of pdg_moments
    cudaStream_t upload_stream = nullptr;  // uploads of pdg_set_equilibrium into w_stage
    cudaEvent_t w_ready = nullptr, d2h_done = nullptr;
    cudaEvent_t stage_free = nullptr, stage_full = nullptr;
    pdg::ModelParams mp{};
    pdg::SweepParams x_params{};        // velocities along x
    pdg::SweepParams yz_params{};       // velocities along y / z
    pdg::SweepParams all_params{};      // every local velocity (inflow initialisation)
    pdg::NcclComm comm;
    // pdg_step(n) replays a CUDA graph of its n-step launch sequence (captured on cap_stream once
    // per n, launched on the caller's stream)
    cudaStream_t cap_stream = nullptr;
    std::map<int64_t, cudaGraphExec_t> step_graphs;
    bool graphs_off = false;  // a capture failed once: direct launches from then on
    cudaStream_t comm_stream = nullptr;                // NCCL sums of the pipelined sharded collision
    cudaEvent_t ev_pm[kMaxChunks] = {}, ev_ar[kMaxChunks] = {};  // per chunk: partial moments written, summed
    int device = 0;
    Profiler prof;
    int sms = 148;
    int l2keep = 0;  // f fits in L2 (<= 70 % of it): keep it resident between passes (pdg_kernels.cuh l2_policy)
    // z-slab decomposition
    std::vector<pdg::SweepVel> outer_entries;  // per (outer velocity, local slab)
    double *zcarry = nullptr, *zinflow = nullptr;
    struct ZTable {
        double dtp;
        int npass, leff, lpre;     // lpre: cells the carry pre-pass reads (zslab_tables)
        std::vector<double> B, C;  // by slab length
    };
    std::vector<ZTable> ztables_host;
    // lattice velocity sets (NEXT-2)
    std::vector<LatPlan> lat_plans;            // one per active-axis class with >= 2 active axes
    pdg::LbmParams lbm{};
    int *lat_ints = nullptr;                   // ticket + progress counters
    double *lat_xbuf = nullptr, *lat_ybuf = nullptr;
    std::vector<cudaStream_t> lat_streams;     // one per class: the classes' wavefronts overlap
    cudaEvent_t lat_fork = nullptr;
    std::vector<cudaEvent_t> lat_join;
    std::map<std::pair<int, double>, pdg::LatticeBlockLD> lat_blocks;  // (act, dt') -> block
    std::map<std::pair<int, double>, int> lat_halo;                    // (act, dt') -> chain halo rows (-1: none)
    std::map<std::tuple<const void *, int, size_t>, int> launch_cache;  // (kernel, threads, smem) -> CTAs/SM
    std::map<std::pair<int, double>, double *> lat_gtab;  // (act, dt') -> device copy of a large block table
    double *lat_gtab_base = nullptr;                      // slots in the work buffer
    int lat_gtab_used = 0;
};

namespace {

pdg_status zslab_resolve(pdg_ctx *c, double dtp, int npass);
pdg_status ztable(pdg_ctx *c, double dtp, int npass, const pdg_ctx::ZTable **out);

// Every entry point taking a context runs on the context's device (the caller's current
// device may differ) and restores the caller's device on exit.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(const pdg_ctx *c)
    {
        if (!c) return;
        int cur = -1;
        if (cudaGetDevice(&cur) == cudaSuccess && cur != c->device && cudaSetDevice(c->device) == cudaSuccess) prev = cur;
    }
    ~DeviceGuard()
    {
        if (prev >= 0) cudaSetDevice(prev);
    }
    DeviceGuard(const DeviceGuard &) = delete;
    DeviceGuard &operator=(const DeviceGuard &) = delete;
};

pdg_status post_launch(pdg_ctx *c, const char *what)
{
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(PDG_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    if (c->prob.flags & PDG_SYNC_ERRORS) {
        e = cudaStreamSynchronize(c->stream);
        if (e != cudaSuccess) return fail(PDG_E_CUDA, std::string(what) + " (async): " + cudaGetErrorString(e));
    }
    return PDG_OK;
}

// PDG_PROFILE: CUDA events bracketing each launch on the context stream.
int prof_begin(pdg_ctx *c, cudaStream_t st = nullptr)
{
    if (!c->prof.on || c->prof.paused || c->prof.next + 2 > (int)c->prof.ev.size()) return -1;
    const int i = c->prof.next;
    c->prof.next += 2;
    cudaEventRecord(c->prof.ev[i], st ? st : c->stream);
    return i;
}

void prof_end(pdg_ctx *c, int i, int kind, double bytes, cudaStream_t st = nullptr)
{
    if (i < 0) return;
    cudaEventRecord(c->prof.ev[i + 1], st ? st : c->stream);
    c->prof.recs.push_back({kind, i, bytes});
}

// grid of a grid-stride kernel: one thread per work item up to 8 resident 256-thread CTAs per SM
// of the context's device, grid-stride beyond
int grid_for(const pdg_ctx *c, int64_t work, int threads)
{
    int64_t blocks = (work + threads - 1) / threads;
    const int64_t cap = (int64_t)c->sms * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    return (int)blocks;
}

bool fill_blocks(pdg_ctx *c, double dtp, pdg::DevBlock blk[3])
{
    for (int d = 0; d < 3; ++d) {
        pdg::CellBlock cb;
        const double hd = (d < c->g.dim) ? c->g.h[d] : c->g.h[0];
        const long double kappa = (long double)c->prob.lambda * (long double)dtp / (long double)hd;
        if (!pdg::cell_block(c->g.p, kappa, &cb)) return false;
        std::memset(&blk[d], 0, sizeof(blk[d]));
        for (int i = 0; i < cb.n * cb.n; ++i) blk[d].M[i] = cb.M[i];
        for (int i = 0; i < cb.n; ++i) blk[d].g[i] = cb.g[i];
    }
    return true;
}

double sweep_bytes(const pdg_ctx *c, const pdg::SweepParams &sp)
{
    double b = 0.0;
    for (int i = 0; i < sp.nvel; ++i)
        b += 16.0 * (double)sp.v[i].ncells * c->g.n * (double)sp.v[i].nlines + 8.0 * (double)sp.v[i].nlines;
    return b;
}

enum { SWEEP_ALL = 0, SWEEP_YZ = 1, SWEEP_X = 2 };

// Segments per strided line: 1 when the lines alone fill the GPU several times over,
// else enough segments (<= 32, >= 4 cells each) to reach ~2 waves of threads.
int strided_segments(const pdg_ctx *c, const pdg::SweepParams &sp)
{
    int64_t lines = 0;
    int ncells = 1 << 30;
    for (int i = 0; i < sp.nvel; ++i) {
        lines += sp.v[i].nlines;
        ncells = std::min(ncells, sp.v[i].ncells);
    }
    const int64_t target = (int64_t)c->sms * 2048 * 2;
    if (lines >= target / 2 || ncells < 8) return 1;
    int nseg = (int)std::min<int64_t>(32, (target + lines - 1) / std::max<int64_t>(lines, 1));
    nseg = std::min(nseg, ncells / 4);
    return std::max(1, nseg);
}

// Lines per tile of sweep_cols_kernel, and whether a strided batch can use it: every velocity's
// lines tile by kColsW (inner % kColsW == 0), every velocity has the same line count and length,
// no outgoing carries (z-slab entries), and a tile fits the shared memory of two CTAs per SM.
constexpr int kColsW = 8;

int cols_K(int ncells) { return ncells <= 64 ? 2 : (ncells <= 128 ? 4 : 8); }

size_t cols_smem(int n, const pdg::SweepParams &sp)
{
    int nc = 0;
    for (int i = 0; i < sp.nvel; ++i) nc = std::max(nc, sp.v[i].ncells);
    const int K = cols_K(nc);
    return sizeof(double) * (size_t)kColsW * (size_t)(nc * n + (nc * n) / (K * n) + 1);
}

bool use_cols(const pdg_ctx *c, const pdg::SweepParams &sp)
{
    if (sp.nvel == 0 || cols_smem(c->g.n, sp) > 110 * 1024) return false;
    for (int i = 0; i < sp.nvel; ++i) {
        const pdg::SweepVel &V = sp.v[i];
        if (V.inner % kColsW != 0 || V.cout_off >= 0 || V.cin_off >= 0 || V.ncells != sp.v[0].ncells ||
            V.nlines != sp.v[0].nlines)
            return false;
    }
    return true;
}

template <int N, int NPASS, int K, int AX, bool AL>
void launch_cols_t(pdg_ctx *c, const pdg::SweepParams &sp)
{
    auto kern = pdg::sweep_cols_kernel<N, NPASS, K, kColsW, AX, AL>;
    const size_t smem = cols_smem(N, sp);
    const auto key = std::make_tuple(reinterpret_cast<const void *>(kern), 0, smem);
    if (c->launch_cache.find(key) == c->launch_cache.end()) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        c->launch_cache[key] = 1;
    }
    const int64_t tpv = sp.v[0].nlines / kColsW;
    kern<<<(unsigned)(tpv * sp.nvel), pdg::kColsThreads, smem, c->stream>>>(sp, tpv);
}

template <int N, int NPASS, int K, int AX>
void launch_cols_ax(pdg_ctx *c, const pdg::SweepParams &sp)
{
    if (sp.v[0].ncells % (32 * K) == 0) launch_cols_t<N, NPASS, K, AX, true>(c, sp);
    else launch_cols_t<N, NPASS, K, AX, false>(c, sp);
}

// one launch per sweep axis present in the batch (the kernel's block is a compile-time slot)
template <int N, int NPASS, int K>
void launch_cols_k(pdg_ctx *c, const pdg::SweepParams &sp)
{
    for (int ax = 1; ax < 3; ++ax) {
        pdg::SweepParams q = sp;
        q.nvel = 0;
        q.l2keep = c->l2keep;
        for (int i = 0; i < sp.nvel; ++i)
            if (sp.v[i].axis == ax) q.v[q.nvel++] = sp.v[i];
        if (q.nvel == 0) continue;
        if (ax == 1) launch_cols_ax<N, NPASS, K, 1>(c, q);
        else launch_cols_ax<N, NPASS, K, 2>(c, q);
    }
}

template <int N, int NPASS>
void launch_sweeps(pdg_ctx *c, const pdg::SweepParams &xp, const pdg::SweepParams &yzp, int which)
{
    if (yzp.nvel > 0 && which != SWEEP_X) {
        int64_t maxl = 0;
        for (int i = 0; i < yzp.nvel; ++i) maxl = std::max(maxl, yzp.v[i].nlines);
        const int e = prof_begin(c);
        const int nseg = strided_segments(c, yzp);
        if (nseg > 1 && use_cols(c, yzp)) {
            // few long lines (2-D grids): tiles of adjacent lines staged in shared memory
            const int K = cols_K(yzp.v[0].ncells);
            if (K == 2) launch_cols_k<N, NPASS, 2>(c, yzp);
            else if (K == 4) launch_cols_k<N, NPASS, 4>(c, yzp);
            else launch_cols_k<N, NPASS, 8>(c, yzp);
        } else if (nseg > 1) {
            dim3 grid((unsigned)((maxl + 31) / 32), (unsigned)yzp.nvel);
            pdg::sweep_strided_seg_kernel<N, NPASS><<<grid, dim3(32, nseg), 0, c->stream>>>(yzp, nseg);
        } else {
            // prefetch depth tuned on B200 (tools/microbench_strided.cu): n=3 -> 2, n=4 -> 3 (one sweep) / 1 (two)
            constexpr int PF = (N == 4) ? (NPASS == 1 ? 3 : 1) : 2;
            dim3 grid((unsigned)((maxl + 255) / 256), (unsigned)yzp.nvel);
            pdg::sweep_strided_kernel<N, NPASS, PF><<<grid, 256, 0, c->stream>>>(yzp);
        }
        prof_end(c, e, PDG_K_SWEEP_STRIDED, sweep_bytes(c, yzp));
    }
    if (xp.nvel > 0 && which != SWEEP_YZ) {
        int64_t maxl = 0;
        for (int i = 0; i < xp.nvel; ++i) maxl = std::max(maxl, xp.v[i].nlines);
        dim3 grid((unsigned)((maxl + pdg::kXsWarps - 1) / pdg::kXsWarps), (unsigned)xp.nvel);
        const int e = prof_begin(c);
        pdg::sweep_x_kernel<N, NPASS><<<grid, pdg::kXsWarps * 32, 0, c->stream>>>(xp);
        prof_end(c, e, PDG_K_SWEEP_X, sweep_bytes(c, xp));
    }
}

// ---- lattice sweeps (NEXT-2) ------------------------------------------------------------
const pdg::LatticeBlockLD *lattice_block_for(pdg_ctx *c, int act, double dtp)
{
    const auto key = std::make_pair(act, dtp);
    auto it = c->lat_blocks.find(key);
    if (it != c->lat_blocks.end()) return &it->second;
    long double kap[3] = {0, 0, 0};
    int d = 0;
    for (int k = 0; k < c->g.dim; ++k)
        if (act & (1 << k)) kap[d++] = (long double)c->prob.lambda * (long double)dtp / (long double)c->g.h[k];
    pdg::LatticeBlockLD B;
    if (!pdg::lattice_block(c->g.p, d, kap, &B)) return nullptr;
    return &(c->lat_blocks[key] = std::move(B));
}

template <int D, int N, int ACT>
pdg_status launch_lattice_t(pdg_ctx *c, const LatPlan &pl, const pdg::LatticeBlockLD &B, double dtp, cudaStream_t st)
{
    using PP = pdg::LatParams<D, N, ACT>;
    using TB = pdg::LatTab<N, pdg::LatShape<D, ACT>::DA>;
    constexpr int DA = pdg::LatShape<D, ACT>::DA;
    std::vector<char> mem(sizeof(PP), 0);
    PP &P = *reinterpret_cast<PP *>(mem.data());
    const Geometry &g = c->g;
    P.f = c->f;
    P.fb = c->fb;
    P.ticket = c->lat_ints + pl.ints_off;
    P.progress = c->lat_ints + pl.ints_off + 1;
    P.hdone = P.progress + (size_t)8 * pl.ntasks;
    P.xbuf = c->lat_xbuf + pl.xbuf_off;
    P.ybuf = c->lat_ybuf + pl.ybuf_off;
    P.f_elems = (int64_t)g.nvl * g.nnodes;
    P.fb_elems = (int64_t)g.nvl * g.nplanes * g.plane_stride;
    P.xbuf_elems = (int64_t)pl.xbuf;
    P.ybuf_elems = (int64_t)pl.ybuf;
    for (int k = 0; k < 3; ++k) {
        P.g.L[k] = g.L[k];
        P.g.stride[k] = g.stride[k];
        P.g.ncell[k] = (int32_t)g.ncell[k];
    }
    P.g.plane_stride = g.plane_stride;
    P.g.Wx = pl.Wx;
    P.g.Wy = pl.Wy;
    P.g.ngx = pl.ngx;
    P.g.ngy = pl.ngy;
    P.g.nlane = pl.nlane;
    P.g.nw = pl.nw;
    P.g.nc = pl.nc;
    P.g.ntasks = pl.ntasks;
    // chain segments: the halo depth of this (class, dt') from the norm bound, or unsegmented
    P.g.nseg = 1;
    P.g.seglen = pl.nc;
    P.g.halo = 0;
    P.g.rcap = pl.nc;
    if (pl.nseg > 1) {
        const auto hk = std::make_pair(pl.act, dtp);
        auto hi = c->lat_halo.find(hk);
        int h = -1;
        if (hi != c->lat_halo.end()) h = hi->second;
        else h = c->lat_halo[hk] = pdg::lattice_chain_halo(B, 1, pl.seglen);
        if (h > 0 && h <= pl.seglen) {
            P.g.nseg = pl.nseg;
            P.g.seglen = pl.seglen;
            P.g.halo = h;
            P.g.rcap = pl.rcap;
        }
    }
    P.g.ntasks = pl.ntasks / pl.nseg * P.g.nseg;
    // scan rounds: round j adds Bx^(2^j) times an earlier lane's out-trace; once the infinity
    // norm of that power is below 2^-64 the term cannot change an fp64 result, nor can any later
    // (smaller) power
    P.g.nscan = 5;
    for (int sr = 0; sr < 5; ++sr) {
        long double nrm = 0.0L;
        for (int i = 0; i < TB::MF; ++i) {
            long double row = 0.0L;
            for (int j = 0; j < TB::MF; ++j) row += fabsl(B.Bpow[((size_t)sr * TB::MF + i) * TB::MF + j]);
            nrm = std::max(nrm, row);
        }
        if (nrm < 0x1p-64L) {
            P.g.nscan = sr;
            break;
        }
    }
    P.g.nvel = pl.nvel;
    for (int q = 0; q < pl.nvel; ++q) {
        const int j = pl.vel[q];
        const double *v = c->vel.data() + 3 * (g.v0 + j);
        P.v[q].f_off = (int64_t)j * g.nnodes;
        P.v[q].fb_off = (int64_t)j * g.dim * g.plane_stride;
        for (int k = 0; k < 3; ++k) P.v[q].sign[k] = (v[k] < 0.0) ? -1 : 1;
    }
    constexpr int NB = TB::NB, MF = TB::MF;
    // tables in LatTab layout (column-major blocks): into the parameter space, or (too large for it)
    // into a device slot of the work buffer, uploaded once per (class, dt')
    std::vector<double> host(sizeof(TB) / sizeof(double), 0.0);
    TB &T = *reinterpret_cast<TB *>(host.data());
    // the sweeps multiply A^{-1} by the rhs 2 f_old + (kappa_t/omega_0) E_in^(t) s_t (pdg_lattice.cuh)
    for (int q = 0; q < NB; ++q)
        for (int cc = 0; cc < NB; ++cc) T.M[cc * NB + q] = (double)B.Ainv[(size_t)q * NB + cc];
    for (int t = 0; t < 3; ++t) P.g.kw[t] = (t < DA) ? (double)(B.kappa[t] / B.w0) : 0.0;
    for (int t = 0; t < DA; ++t)
        for (int q = 0; q < NB; ++q)
            for (int j = 0; j < MF; ++j) T.Q[t][j * NB + q] = (double)B.Q[((size_t)t * NB + q) * MF + j];
    for (int s = 0; s < 5; ++s)
        for (int i = 0; i < MF; ++i)
            for (int j = 0; j < MF; ++j) T.Bp[s][j * MF + i] = (double)B.Bpow[((size_t)s * MF + i) * MF + j];
    if constexpr (pdg::LatTabSel<N, DA>::BIG) {
        // uploaded at pdg_create for the scheme's steps (graph capture safe); other dt' on first use
        const auto key = std::make_pair(pl.act, dtp);
        auto it = c->lat_gtab.find(key);
        double *dev = nullptr;
        if (it != c->lat_gtab.end()) dev = it->second;
        else {
            if (c->lat_gtab_used >= kMaxLatTables) return fail(PDG_E_UNSUPPORTED, "too many distinct lattice steps");
            dev = c->lat_gtab_base + (size_t)c->lat_gtab_used * kLatBigTableDoubles;
            ++c->lat_gtab_used;
            PDG_CUDA_TRY(cudaMemcpy(dev, host.data(), sizeof(TB), cudaMemcpyHostToDevice));
            c->lat_gtab[key] = dev;
        }
        if (!st) return PDG_OK;  // table preparation only (pdg_create)
        const TB *D_ = reinterpret_cast<const TB *>(dev);
        P.tab.M = D_->M;
        for (int t = 0; t < 3; ++t) P.tab.Q[t] = (t < DA) ? D_->Q[t] : nullptr;
        for (int s = 0; s < 5; ++s) P.tab.Bp[s] = D_->Bp[s];
    } else {
        P.tab = T;
    }
    const int threads = 32 * pl.Wx * pl.Wy;
    constexpr int PIPE = pdg::LatShape<D, ACT>::PIPE;
    // cp.async row buffers + the y hand-over buffers (pdg_lattice.cuh)
    const size_t smem =
        sizeof(double) * ((size_t)(threads / 32) * pdg::LatRing<D, N, DA>::RING * TB::NB * 32 +
                          (PIPE ? (size_t)2 * 32 * TB::MF * (threads / 32 - pl.Wx) : 0) +
                          pdg::LatMma<D, N, ACT>::smem_doubles(threads / 32) +
                          (PIPE ? (size_t)pl.Wx * 32 * 2 * TB::MF : 0));
    // per-context (hence per-device, per-thread) cache of the shared-memory opt-in and occupancy
    auto kern = pdg::lattice_sweep_kernel<D, N, ACT>;
    const void *kfn = reinterpret_cast<const void *>(kern);
    const auto key = std::make_tuple(kfn, threads, smem);
    auto oc = c->launch_cache.find(key);
    int occ = 0;  // resident CTAs on the whole GPU (persistent kernel: one grid of resident CTAs)
    if (oc != c->launch_cache.end()) occ = oc->second;
    else {
        const cudaError_t ea = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (ea != cudaSuccess)
            return fail(PDG_E_CUDA, std::string("lattice sweep shared memory opt-in: ") + cudaGetErrorString(ea));
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem) != cudaSuccess) occ = 1;
        occ *= c->sms;
        cudaGetLastError();
        occ = std::max(1, occ);
        c->launch_cache[key] = occ;
    }
    const int units = std::max(1, std::min(P.g.ntasks, occ));
    PDG_CUDA_TRY(cudaMemsetAsync(P.ticket, 0, sizeof(int) * ((size_t)9 * pl.ntasks + 1), st));
    kern<<<units, threads, smem, st>>>(P);
    return PDG_OK;
}

// One pass over the velocities of class `pl` applying T2(dtp) npass times, one sweep per launch
// (two sweeps per launch measured slower once the hand-overs were tagged).
pdg_status launch_lattice(pdg_ctx *c, const LatPlan &pl, double dtp, cudaStream_t st, int npass)
{
    const pdg::LatticeBlockLD *B = lattice_block_for(c, pl.act, dtp);
    if (!B) return fail(PDG_E_INVALID_ARGUMENT, "singular lattice block for this dt");
    const int D = c->g.dim, n = c->g.n, a = pl.act;
    for (int q = 0; q < npass; ++q) {
        const int e = prof_begin(c, st);
        pdg_status s = PDG_E_UNSUPPORTED;
#define PDG_LAT(DD, NN, AA) else if (D == DD && n == NN && a == AA) s = launch_lattice_t<DD, NN, AA>(c, pl, *B, dtp, st)
        if (false) {}
        PDG_LAT(2, 2, 3); PDG_LAT(2, 3, 3); PDG_LAT(2, 4, 3);
        PDG_LAT(3, 2, 3); PDG_LAT(3, 3, 3); PDG_LAT(3, 4, 3);
        PDG_LAT(3, 2, 5); PDG_LAT(3, 3, 5); PDG_LAT(3, 4, 5);
        PDG_LAT(3, 2, 6); PDG_LAT(3, 3, 6); PDG_LAT(3, 4, 6);
        PDG_LAT(3, 2, 7); PDG_LAT(3, 3, 7); PDG_LAT(3, 4, 7);
#undef PDG_LAT
        if (s == PDG_E_UNSUPPORTED) return fail(s, "lattice sweep not compiled for this (dim, degree, axes)");
        if (s != PDG_OK) return s;
        prof_end(c, e, PDG_K_LATTICE, 16.0 * (double)pl.nvel * (double)c->g.nnodes, st);
        s = post_launch(c, "lattice_sweep");
        if (s != PDG_OK) return s;
    }
    return PDG_OK;
}

// One pass over f applying T2(dtp) npass times (npass in {1, 2}) to the selected velocities.
pdg_status transport_pass(pdg_ctx *c, double dtp, int npass, int which = SWEEP_ALL)
{
    NvtxRange nv(npass == 2 ? "pdg T2 x2 (fused half-steps)" : "pdg T2");
    // lattice classes: forked onto their own streams (joined below), so that their wavefront
    // ramps overlap with each other and with the axis-aligned sweeps on the context stream
    const bool lat = which != SWEEP_X && !c->lat_plans.empty();
    if (lat) {
        PDG_CUDA_TRY(cudaEventRecord(c->lat_fork, c->stream));
        for (size_t k = 0; k < c->lat_plans.size(); ++k) {
            PDG_CUDA_TRY(cudaStreamWaitEvent(c->lat_streams[k], c->lat_fork, 0));
            pdg_status ls = launch_lattice(c, c->lat_plans[k], dtp, c->lat_streams[k], npass);
            if (ls != PDG_OK) return ls;
            PDG_CUDA_TRY(cudaEventRecord(c->lat_join[k], c->lat_streams[k]));
        }
    }
    pdg::SweepParams xp = c->x_params, yzp = c->yz_params;
    pdg::DevBlock blk[3];
    if (!fill_blocks(c, dtp, blk)) return fail(PDG_E_INVALID_ARGUMENT, "singular cell block for this dt");
    std::memcpy(xp.blk, blk, sizeof(blk));
    std::memcpy(yzp.blk, blk, sizeof(blk));
    const int n = c->g.n;
    auto launch = [&](const pdg::SweepParams &a, const pdg::SweepParams &b, int wh) {
        if (npass == 1) {
            if (n == 2) launch_sweeps<2, 1>(c, a, b, wh);
            else if (n == 3) launch_sweeps<3, 1>(c, a, b, wh);
            else launch_sweeps<4, 1>(c, a, b, wh);
        } else {
            if (n == 2) launch_sweeps<2, 2>(c, a, b, wh);
            else if (n == 3) launch_sweeps<3, 2>(c, a, b, wh);
            else launch_sweeps<4, 2>(c, a, b, wh);
        }
    };
    launch(xp, yzp, which);
    const bool outer = c->g.zslab && which != SWEEP_X && !c->outer_entries.empty();
    pdg_status s = post_launch(c, "sweep");
    if (s == PDG_OK && outer) {
        // z-slab decomposition of the outer-axis velocities: read-only carry pre-pass over the
        // last lpre cells of every slab, carry exchange + scan, then one exact sweep per slab from
        // its exact inflows (launches of at most kMaxVel (velocity, slab) entries)
        const pdg_ctx::ZTable *zt = nullptr;
        s = ztable(c, dtp, npass, &zt);
        const size_t ne = c->outer_entries.size();
        pdg::SweepParams op = yzp, none = xp;
        none.nvel = 0;
        op.cout = c->zcarry;
        op.cin = c->zinflow;
        for (size_t b0 = 0; b0 < ne && s == PDG_OK; b0 += pdg::kMaxVel) {
            op.nvel = (int32_t)std::min<size_t>(pdg::kMaxVel, ne - b0);
            int64_t maxl = 0;
            double bytes = 0.0;
            for (int i = 0; i < op.nvel; ++i) {
                op.v[i] = c->outer_entries[b0 + i];
                op.v[i].cin_off = -1;
                maxl = std::max(maxl, op.v[i].nlines);
                bytes += 8.0 * std::min(zt->lpre, op.v[i].ncells) * n * (double)op.v[i].nlines;
            }
            const int e = prof_begin(c);
            dim3 grid((unsigned)((maxl + 255) / 256), (unsigned)op.nvel);
            if (n == 2) npass == 1 ? pdg::zslab_carry_kernel<2, 1><<<grid, 256, 0, c->stream>>>(op, zt->lpre)
                                   : pdg::zslab_carry_kernel<2, 2><<<grid, 256, 0, c->stream>>>(op, zt->lpre);
            else if (n == 3) npass == 1 ? pdg::zslab_carry_kernel<3, 1><<<grid, 256, 0, c->stream>>>(op, zt->lpre)
                                        : pdg::zslab_carry_kernel<3, 2><<<grid, 256, 0, c->stream>>>(op, zt->lpre);
            else npass == 1 ? pdg::zslab_carry_kernel<4, 1><<<grid, 256, 0, c->stream>>>(op, zt->lpre)
                            : pdg::zslab_carry_kernel<4, 2><<<grid, 256, 0, c->stream>>>(op, zt->lpre);
            prof_end(c, e, PDG_K_ZSLAB, bytes);
            s = post_launch(c, "zslab_carry");
        }
        if (s == PDG_OK) s = zslab_resolve(c, dtp, npass);
        for (size_t b0 = 0; b0 < ne && s == PDG_OK; b0 += pdg::kMaxVel) {
            op.nvel = (int32_t)std::min<size_t>(pdg::kMaxVel, ne - b0);
            for (int i = 0; i < op.nvel; ++i) {
                op.v[i] = c->outer_entries[b0 + i];
                op.v[i].cout_off = -1;
                op.v[i].zero_inflow = 0;
            }
            launch(none, op, SWEEP_YZ);
            s = post_launch(c, "zslab sweep");
        }
    }
    if (lat)
        for (size_t k = 0; k < c->lat_plans.size(); ++k) PDG_CUDA_TRY(cudaStreamWaitEvent(c->stream, c->lat_join[k], 0));
    return s;
}

// ---- collision fused with the x-velocity sweeps (nranks == 1) ----------------------------
int relax_x_K(int ncx)
{
    if (ncx <= 64) return 2;
    if (ncx <= 128) return 4;
    return 8;
}

size_t relax_x_smem(const pdg_ctx *c)
{
    const int K = relax_x_K((int)c->g.ncell[0]);
    const int n = c->g.n;
    const int64_t L = c->g.ncell[0] * n;
    const int64_t Lp = L + L / (K * n) + 1;
    return sizeof(double) * (size_t)(2 * c->g.m) * (size_t)Lp;
}

// shared memory of the TMA-staged variant: the raw line [n_v][Lx] + the x-velocity sweep rows
size_t relax_x_tma_smem(const pdg_ctx *c) { return relax_x_smem(c) + sizeof(double) * (size_t)c->g.nvl * c->g.L[0]; }

bool use_relax_x_tma(const pdg_ctx *c)
{
    // only where two or more CTAs fit an SM: with one CTA per SM (configs 2, 4, 5: raw lines of
    // 98-147 KB) the next line's load cannot hide behind enough work and the register-staged
    // kernel measured faster (config 5: 0.888 against 0.959 of HBM; config 3, 51 KB per CTA:
    // 0.940 against 0.814; profiles/r02_bench_*)
    return !(c->prob.flags & PDG_NO_TMA) && (c->g.L[0] % 2 == 0) && relax_x_tma_smem(c) <= 110 * 1024;
}

template <int DIM, int MODEL, int N, int NPASS, int K>
void launch_relax_x_tma_k(pdg_ctx *c, const pdg::RelaxXParams &P)
{
    auto kern = pdg::relax_xsweep_tma_kernel<DIM, MODEL, N, NPASS, K>;
    const size_t smem = relax_x_tma_smem(c);
    const int lx = (int)(c->g.ncell[0] * N);
    const int threads = std::min(256, ((lx + 31) / 32) * 32);
    const auto key = std::make_tuple(reinterpret_cast<const void *>(kern), threads, smem);
    auto it = c->launch_cache.find(key);
    int occ = 0;  // resident CTAs on the GPU: the kernel is persistent
    if (it != c->launch_cache.end()) occ = it->second;
    else {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem) != cudaSuccess) occ = 1;
        cudaGetLastError();
        occ = std::max(1, occ) * c->sms;
        c->launch_cache[key] = occ;
    }
    const int64_t nlines = c->g.nnodes / (c->g.ncell[0] * N);
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nlines, occ));
    kern<<<grid, threads, smem, c->stream>>>(P, nlines);
}

template <int DIM, int MODEL, int N, int NPASS, int K>
void launch_relax_x_k(pdg_ctx *c, const pdg::RelaxXParams &P, size_t smem)
{
    if (use_relax_x_tma(c)) {
        launch_relax_x_tma_k<DIM, MODEL, N, NPASS, K>(c, P);
        return;
    }
    auto kern = pdg::relax_xsweep_kernel<DIM, MODEL, N, NPASS, K>;
    const auto key = std::make_tuple(reinterpret_cast<const void *>(kern), 0, (size_t)0);
    if (c->launch_cache.find(key) == c->launch_cache.end()) {  // per context: attributes are per device
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        c->launch_cache[key] = 1;
    }
    const unsigned nlines = (unsigned)(c->g.nnodes / (c->g.ncell[0] * N));
    // one thread per node of the line up to 256 (a 192-node line of config 3 left a quarter of a
    // 256-thread CTA idle in the collision and store phases)
    const int lx = (int)(c->g.ncell[0] * N);
    const unsigned threads = (unsigned)std::min(256, ((lx + 31) / 32) * 32);
    kern<<<nlines, threads, smem, c->stream>>>(P);
}

template <int DIM, int MODEL, int N, int NPASS>
void launch_relax_x_n(pdg_ctx *c, const pdg::RelaxXParams &P, size_t smem)
{
    const int K = relax_x_K(P.ncx);
    if (K == 2) launch_relax_x_k<DIM, MODEL, N, NPASS, 2>(c, P, smem);
    else if (K == 4) launch_relax_x_k<DIM, MODEL, N, NPASS, 4>(c, P, smem);
    else launch_relax_x_k<DIM, MODEL, N, NPASS, 8>(c, P, smem);
}

template <int DIM, int MODEL>
void launch_relax_x_t(pdg_ctx *c, const pdg::RelaxXParams &P, size_t smem, int npass)
{
    const int n = c->g.n;
    if (npass == 1) {
        if (n == 2) launch_relax_x_n<DIM, MODEL, 2, 1>(c, P, smem);
        else if (n == 3) launch_relax_x_n<DIM, MODEL, 3, 1>(c, P, smem);
        else launch_relax_x_n<DIM, MODEL, 4, 1>(c, P, smem);
    } else {
        if (n == 2) launch_relax_x_n<DIM, MODEL, 2, 2>(c, P, smem);
        else if (n == 3) launch_relax_x_n<DIM, MODEL, 3, 2>(c, P, smem);
        else launch_relax_x_n<DIM, MODEL, 4, 2>(c, P, smem);
    }
}

template <int DIM, int MODEL>
void launch_relax_t(pdg_ctx *c, double ca, double cb)
{
    const int grid = grid_for(c, c->g.nnodes, 256);
    const int e = prof_begin(c);
    pdg::relax_kernel<DIM, MODEL><<<grid, 256, 0, c->stream>>>(c->f, c->g.nnodes, c->mp, ca, cb);
    prof_end(c, e, PDG_K_RELAX, 16.0 * (double)c->g.nvl * (double)c->g.nnodes);
}

// the sharded collision's halves on the node chunk [x0, x0 + cnt) (velocity / component stride nnodes)
template <int DIM, int MODEL>
void launch_partial_t(pdg_ctx *c, int64_t x0, int64_t cnt)
{
    const int grid = grid_for(c, cnt, 256);
    const int e = prof_begin(c);
    pdg::partial_moments_kernel<DIM, MODEL>
        <<<grid, 256, 0, c->stream>>>(c->f + x0, c->w + x0, c->g.nnodes, cnt, c->g.v0, c->g.nvl);
    prof_end(c, e, PDG_K_PARTIAL, 8.0 * (double)(c->g.nvl + c->g.m) * (double)cnt);
}

template <int DIM, int MODEL>
void launch_relax_from_w_t(pdg_ctx *c, int64_t x0, int64_t cnt, double ca, double cb)
{
    const int grid = grid_for(c, cnt, 256);
    const int e = prof_begin(c);
    pdg::relax_from_w_kernel<DIM, MODEL>
        <<<grid, 256, 0, c->stream>>>(c->f + x0, c->w + x0, c->g.nnodes, cnt, c->g.v0, c->g.nvl, c->mp, ca, cb);
    prof_end(c, e, PDG_K_RELAX_W, 8.0 * (double)(2 * c->g.nvl + c->g.m) * (double)cnt);
}

template <int DIM, int MODEL>
void launch_equilibrium_t(pdg_ctx *c, const double *w, const double *wb)
{
    const int grid = grid_for(c, c->g.nnodes, 256);
    pdg::equilibrium_kernel<DIM, MODEL><<<grid, 256, 0, c->stream>>>(c->f, w, c->g.nnodes, c->g.v0, c->g.nvl, c->mp);
    int64_t maxl = 0;
    for (int i = 0; i < c->all_params.nvel; ++i) maxl = std::max(maxl, c->all_params.v[i].nlines);
    dim3 g2((unsigned)((maxl + 255) / 256), (unsigned)c->all_params.nvel);
    pdg::inflow_equilibrium_kernel<DIM, MODEL>
        <<<g2, 256, 0, c->stream>>>(c->fb, wb, c->g.nnodes, c->all_params, c->g.n, c->mp);
}

// dispatch on (dim, flux model)
#define PDG_DISPATCH(FN, ...)                                                                       \
    do {                                                                                            \
        const int dim_ = c->g.dim, mod_ = c->prob.flux;                                             \
        if (dim_ == 2 && mod_ == 0) FN<2, pdg::MODEL_ADV>(__VA_ARGS__);                             \
        else if (dim_ == 2 && mod_ == 1) FN<2, pdg::MODEL_EULER>(__VA_ARGS__);                      \
        else if (dim_ == 2 && mod_ == 2) FN<2, pdg::MODEL_ISO>(__VA_ARGS__);                        \
        else if (dim_ == 3 && mod_ == 0) FN<3, pdg::MODEL_ADV>(__VA_ARGS__);                        \
        else if (dim_ == 3 && mod_ == 1) FN<3, pdg::MODEL_EULER>(__VA_ARGS__);                      \
        else FN<3, pdg::MODEL_ISO>(__VA_ARGS__);                                                    \
    } while (0)

// ---- LBM model kernels (lattice sets, NEXT-2) ------------------------------------------
// one node per thread for the LBM kernels (pdg_lattice.cuh)
unsigned grid_all(int64_t work, int threads) { return (unsigned)std::max<int64_t>(1, (work + threads - 1) / threads); }

template <int D, int NV>
void launch_relax_lbm_t(pdg_ctx *c, pdg::LocalOps op)
{
    const unsigned grid = grid_all(c->g.nnodes, 256);
    const int e = prof_begin(c);
    // two-phase kernel (moments, then an L1 re-read per update): 1.01-1.03 of the measured copy
    // bandwidth on the 3-D sets against 0.90-0.99 for a one-read kernel (tools/gpu/relax2.sh, round 1)
    pdg::relax_lbm2_kernel<D, NV><<<grid, 256, 0, c->stream>>>(c->f, c->g.nnodes, c->lbm, op);
    prof_end(c, e, PDG_K_RELAX, 16.0 * (double)c->g.nvl * (double)c->g.nnodes);
}

template <int D, int NV>
void launch_partial_lbm_t(pdg_ctx *c, int64_t x0, int64_t cnt)
{
    const unsigned grid = grid_all(cnt, 256);
    const int e = prof_begin(c);
    pdg::partial_moments_lbm_kernel<D, NV>
        <<<grid, 256, 0, c->stream>>>(c->f + x0, c->w + x0, c->g.nnodes, cnt, c->g.v0, c->g.nvl, c->lbm);
    prof_end(c, e, PDG_K_PARTIAL, 8.0 * (double)(c->g.nvl + c->g.m) * (double)cnt);
}

template <int D, int NV>
void launch_relax_from_w_lbm_t(pdg_ctx *c, int64_t x0, int64_t cnt, pdg::LocalOps op)
{
    const unsigned grid = grid_all(cnt, 256);
    const int e = prof_begin(c);
    pdg::relax_from_w_lbm_kernel<D, NV>
        <<<grid, 256, 0, c->stream>>>(c->f + x0, c->w + x0, c->g.nnodes, cnt, c->g.v0, c->g.nvl, c->lbm, op);
    prof_end(c, e, PDG_K_RELAX_W, 8.0 * (double)(2 * c->g.nvl + c->g.m) * (double)cnt);
}

// f = f^eq(w) (f_only) or, additionally, the inflow planes fb from f^eq(wb)
template <int D, int NV>
void launch_equilibrium_lbm_t(pdg_ctx *c, const double *w, const double *wb, bool f_only)
{
    const unsigned grid = grid_all(c->g.nnodes, 256);
    if (w) pdg::equilibrium_lbm_kernel<D, NV><<<grid, 256, 0, c->stream>>>(c->f, w, c->g.nnodes, c->g.v0, c->g.nvl, c->lbm);
    if (f_only) return;
    pdg::LatInflowParams P;
    std::memset(&P, 0, sizeof(P));
    P.fb = c->fb;
    P.wb = wb;
    P.nnodes = c->g.nnodes;
    P.plane_stride = c->g.plane_stride;
    for (int k = 0; k < 3; ++k) {
        P.L[k] = c->g.L[k];
        P.stride[k] = c->g.stride[k];
    }
    P.v0 = c->g.v0;
    P.nvl = c->g.nvl;
    P.dim = D;
    P.lbm = c->lbm;
    dim3 g2((unsigned)((c->g.plane_stride + 255) / 256), (unsigned)c->g.nvl, (unsigned)D);
    pdg::lattice_inflow_kernel<D, NV><<<g2, 256, 0, c->stream>>>(P);
}

#define PDG_LBM_DISPATCH(FN, ...)                                                                   \
    do {                                                                                            \
        const int d_ = c->g.dim, nv_ = c->g.nv;                                                     \
        if (d_ == 2) FN<2, 9>(__VA_ARGS__);                                                         \
        else if (nv_ == 15) FN<3, 15>(__VA_ARGS__);                                                 \
        else if (nv_ == 19) FN<3, 19>(__VA_ARGS__);                                                 \
        else FN<3, 27>(__VA_ARGS__);                                                                \
    } while (0)

void collision_coeffs(const pdg_ctx *c, double dt, double *ca, double *cb)
{
    const double tau = c->prob.tau;
    if (tau == 0.0) {  // over-relaxation f <- 2 f^eq - f
        *ca = -1.0;
        *cb = 2.0;
    } else {           // eq collision_cn
        *ca = (2.0 * tau - dt) / (2.0 * tau + dt);
        *cb = 2.0 * dt / (2.0 * tau + dt);
    }
}

// Sharded collision path: several ranks, or a communicator given explicitly (also with one rank).
bool sharded(const pdg_ctx *c)
{
    return c->prob.decomposition == PDG_DECOMP_VELOCITY && (c->prob.nranks > 1 || c->comm.comm != nullptr);
}

// PDG_ASYNC_HOST: w_dev may still be read by the download of the previous pdg_moments
void wait_w_download(pdg_ctx *c)
{
    if (c->copy_stream) cudaStreamWaitEvent(c->stream, c->d2h_done, 0);
}

// Node chunks of the pipelined sharded collision: at most kMaxChunks, at least 2^20 nodes each.
int collision_chunks(const pdg_ctx *c)
{
    if (!c->comm_stream) return 1;
    return (int)std::max<int64_t>(1, std::min<int64_t>(kMaxChunks, c->g.nnodes >> 20));
}

// The sharded collision (velocity decomposition, row a4), pipelined over node chunks (SURVEY §8(e)
// mitigation 2): the partial moments of chunk k on the context stream; the NCCL sum of chunk k (one
// call per moment field: w is [m][nodes]) on the communicator stream as soon as they are written;
// then, if `relax` is given, the relaxation of chunk k on the context stream once its sum has
// arrived.  The sum of chunk k overlaps the partial moments of the later chunks and the relaxation
// of the earlier ones.  Every chunk's sum is joined back into the context stream (graph-capturable
// fork/join).  Without a communicator (shard contexts for tests) only the partial moments run.
template <class Relax>
pdg_status sharded_collision(pdg_ctx *c, Relax relax)
{
    wait_w_download(c);
    const int64_t nn = c->g.nnodes;
    const int K = collision_chunks(c);
    auto chunk = [&](int k, int64_t *x0, int64_t *cnt) {
        *x0 = nn * k / K;
        *cnt = nn * (k + 1) / K - *x0;
    };
    for (int k = 0; k < K; ++k) {
        int64_t x0, cnt;
        chunk(k, &x0, &cnt);
        if (c->g.lattice) PDG_LBM_DISPATCH(launch_partial_lbm_t, c, x0, cnt);
        else PDG_DISPATCH(launch_partial_t, c, x0, cnt);
        if (K > 1) PDG_CUDA_TRY(cudaEventRecord(c->ev_pm[k], c->stream));
    }
    pdg_status s = post_launch(c, "partial_moments");
    if (s != PDG_OK) return s;
    if (!sharded(c)) return PDG_OK;
    if (!c->comm.comm) return fail(PDG_E_NCCL, "communicator-less shard context: reduce w_dev yourself "
                                               "between pdg_partial_moments and pdg_relax_from_w");
    std::string err;
    cudaStream_t cs = (K > 1) ? c->comm_stream : c->stream;
    for (int k = 0; k < K; ++k) {
        int64_t x0, cnt;
        chunk(k, &x0, &cnt);
        if (K > 1) PDG_CUDA_TRY(cudaStreamWaitEvent(cs, c->ev_pm[k], 0));
        const int e = prof_begin(c, cs);
        for (int m = 0; m < c->g.m; ++m)
            if (!c->comm.allreduce_sum(c->w + (int64_t)m * nn + x0, (size_t)cnt, cs, &err)) return fail(PDG_E_NCCL, err);
        prof_end(c, e, PDG_K_ALLREDUCE, 8.0 * (double)c->g.m * (double)cnt, cs);
        if (K > 1) PDG_CUDA_TRY(cudaEventRecord(c->ev_ar[k], cs));
    }
    for (int k = 0; k < K; ++k) {
        int64_t x0, cnt;
        chunk(k, &x0, &cnt);
        if (K > 1) PDG_CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_ar[k], 0));
        relax(x0, cnt);
    }
    return post_launch(c, "relax_from_w");
}

pdg_status partial_and_reduce(pdg_ctx *c)
{
    return sharded_collision(c, [](int64_t, int64_t) {});
}

// One pass of the local operators of a lattice set: S2(hs1), C2(dt) (if with_c), S2(hs2).
pdg_status local_pass_lbm(pdg_ctx *c, double hs1, bool with_c, double dt, double hs2)
{
    NvtxRange nv(with_c ? ((hs1 != 0.0 || hs2 != 0.0) ? "pdg S2 C2 S2" : "pdg C2") : "pdg S2");
    pdg::LocalOps op;
    op.hs1 = hs1;
    op.hs2 = hs2;
    op.ca = 1.0;
    op.cb = 0.0;
    if (with_c) collision_coeffs(c, dt, &op.ca, &op.cb);
    if (!sharded(c)) {
        PDG_LBM_DISPATCH(launch_relax_lbm_t, c, op);
        return post_launch(c, "relax");
    }
    return sharded_collision(c, [&](int64_t x0, int64_t cnt) { PDG_LBM_DISPATCH(launch_relax_from_w_lbm_t, c, x0, cnt, op); });
}

pdg_status collide(pdg_ctx *c, double dt)
{
    NvtxRange nv("pdg C2");
    if (c->g.lattice) return local_pass_lbm(c, 0.0, true, dt, 0.0);
    double ca, cb;
    collision_coeffs(c, dt, &ca, &cb);
    if (!sharded(c)) {
        PDG_DISPATCH(launch_relax_t, c, ca, cb);
        return post_launch(c, "relax");
    }
    return sharded_collision(c, [&](int64_t x0, int64_t cnt) { PDG_DISPATCH(launch_relax_from_w_t, c, x0, cnt, ca, cb); });
}

// C2(dt) followed by npass sweeps T2(dtp) of the x-velocities, in one pass over f.
pdg_status collide_xsweep(pdg_ctx *c, double dt, double dtp, int npass)
{
    NvtxRange nv("pdg C2 + x-sweeps");
    double ca, cb;
    collision_coeffs(c, dt, &ca, &cb);
    pdg::DevBlock blk[3];
    if (!fill_blocks(c, dtp, blk)) return fail(PDG_E_INVALID_ARGUMENT, "singular cell block for this dt");
    pdg::RelaxXParams P;
    std::memset(&P, 0, sizeof(P));
    P.f = c->f;
    P.fb = c->fb;
    P.f_elems = (int64_t)c->g.nvl * c->g.nnodes;
    P.fb_elems = (int64_t)c->g.nvl * c->g.nplanes * c->g.plane_stride;
    P.nnodes = c->g.nnodes;
    P.plane_stride = c->g.plane_stride;
    P.ncx = (int32_t)c->g.ncell[0];
    P.blk = blk[0];
    P.mp = c->mp;
    P.ca = ca;
    P.cb = cb;
    P.l2keep = c->l2keep;
    const size_t smem = relax_x_smem(c);
    const int e = prof_begin(c);
    PDG_DISPATCH(launch_relax_x_t, c, P, smem, npass);
    prof_end(c, e, PDG_K_RELAX_X,
             16.0 * (double)c->g.nvl * (double)c->g.nnodes + 8.0 * (double)c->x_params.nvel * (double)c->x_params.v[0].nlines);
    return post_launch(c, "relax_xsweep");
}

bool use_relax_x(const pdg_ctx *c)
{
    return !c->g.lattice && !sharded(c) && !(c->prob.flags & PDG_NO_FUSION) && relax_x_smem(c) <= 110 * 1024 &&
           c->g.nnodes / (c->g.ncell[0] * c->g.n) < (int64_t)1 << 31;
}

// ---- the palindromic step as a list of operators ------------------------------------------
// T(h) = T2(h) on every velocity, C(h) = C2(h).  Execution fuses, without changing any
// operator: two consecutive T(h) with the same h into one pass over f (two sweeps), and a
// C followed by T's into the collision + x-sweep kernel plus one y/z sweep pass.

void append_m2kin(std::vector<Op> &ops, double dt)
{
    // M2kin(dt) = T2(dt/4) C2(dt/2) T2(dt/2) C2(dt/2) T2(dt/4)
    ops.push_back({0, 0.25 * dt});
    ops.push_back({1, 0.5 * dt});
    ops.push_back({0, 0.5 * dt});
    ops.push_back({1, 0.5 * dt});
    ops.push_back({0, 0.25 * dt});
}

void append_scheme(std::vector<Op> &ops, int scheme, double dt)
{
    if (scheme == PDG_SCHEME_M2) {
        // M2(dt) = T2(dt/2) C2(dt) T2(dt/2)
        ops.push_back({0, 0.5 * dt});
        ops.push_back({1, dt});
        ops.push_back({0, 0.5 * dt});
    } else if (scheme == PDG_SCHEME_M2KIN) {
        append_m2kin(ops, dt);
    } else if (scheme == PDG_SCHEME_M2S) {
        // M2s(dt) = T2(dt/2) S2(dt/2) C2(dt) S2(dt/2) T2(dt/2)
        ops.push_back({0, 0.5 * dt});
        ops.push_back({2, 0.5 * dt});
        ops.push_back({1, dt});
        ops.push_back({2, 0.5 * dt});
        ops.push_back({0, 0.5 * dt});
    } else {
        // M4 = M2kin(g1 dt) M2kin(g2 dt) M2kin(g1 dt): symmetric triple jump, a palindromic
        // composition of M2kin raising the order to 4; g1 = 1/(2 - 2^{1/3}).
        const long double cr = cbrtl(2.0L);
        const double g1 = (double)(1.0L / (2.0L - cr));
        const double g2 = (double)(-cr / (2.0L - cr));
        append_m2kin(ops, g1 * dt);
        append_m2kin(ops, g2 * dt);
        append_m2kin(ops, g1 * dt);
    }
}

// ---- small problems: a run of operators in one CTA (pdg_kernels.cuh small_run_kernel) ----------
constexpr size_t kSmallBytes = 64 * 1024;  // f in shared memory

int small_lp(const Geometry &g) { return (int)(g.L[0] | 1); }  // odd row stride in shared memory

size_t small_smem(const Geometry &g)
{
    return sizeof(double) * (size_t)g.nvl * (size_t)(g.nnodes / g.L[0]) * (size_t)small_lp(g);
}

bool use_small(const pdg_ctx *c)
{
    const Geometry &g = c->g;
    return !g.lattice && !g.zslab && !sharded(c) && c->prob.nranks == 1 && !(c->prob.flags & PDG_NO_SMALL) &&
           g.nvl == c->all_params.nvel && c->all_params.nvel <= pdg::kMaxVel && small_smem(g) <= kSmallBytes;
}

template <int DIM, int MODEL, int N>
void launch_small_n(pdg_ctx *c, const pdg::SmallParams &P, size_t smem)
{
    auto kern = pdg::small_run_kernel<DIM, MODEL, N>;
    const auto key = std::make_tuple(reinterpret_cast<const void *>(kern), 0, (size_t)1);
    if (c->launch_cache.find(key) == c->launch_cache.end()) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmallBytes);
        c->launch_cache[key] = 1;
    }
    kern<<<1, pdg::kSmallThreads, smem, c->stream>>>(P);
}

template <int DIM, int MODEL>
void launch_small_t(pdg_ctx *c, const pdg::SmallParams &P, size_t smem)
{
    if (c->g.n == 2) launch_small_n<DIM, MODEL, 2>(c, P, smem);
    else if (c->g.n == 3) launch_small_n<DIM, MODEL, 3>(c, P, smem);
    else launch_small_n<DIM, MODEL, 4>(c, P, smem);
}

pdg_status small_run(pdg_ctx *c, const std::vector<Op> &ops)
{
    NvtxRange nv("pdg small run");
    const Geometry &g = c->g;
    pdg::SmallParams P;
    std::memset(&P, 0, sizeof(P));
    P.f = c->f;
    P.fb = c->fb;
    P.nnodes = g.nnodes;
    P.f_elems = (int64_t)g.nvl * g.nnodes;
    P.fb_elems = (int64_t)g.nvl * g.nplanes * g.plane_stride;
    P.nvel = c->all_params.nvel;
    P.line0[0] = 0;
    for (int i = 0; i < P.nvel; ++i) {
        P.v[i] = c->all_params.v[i];
        P.line0[i + 1] = P.line0[i] + (P.v[i].nlines + 31) / 32 * 32;
    }
    P.mp = c->mp;
    P.L0 = (int32_t)g.L[0];
    P.Lp = small_lp(g);
    P.vstride = (g.nnodes / g.L[0]) * P.Lp;
    P.sstr[0] = 1;
    P.sstr[1] = P.Lp;
    P.sstr[2] = (int64_t)P.Lp * g.L[1];
    const size_t smem = small_smem(g);
    std::vector<double> hs;  // T2 step sizes of the current launch, index = block set
    auto flush = [&]() -> pdg_status {
        if (P.nops == 0) return PDG_OK;
        const int e = prof_begin(c);
        PDG_DISPATCH(launch_small_t, c, P, smem);
        prof_end(c, e, PDG_K_SMALL, 16.0 * (double)g.nvl * (double)g.nnodes);
        P.nops = 0;
        hs.clear();
        return post_launch(c, "small_run");
    };
    for (const Op &o : ops) {
        if (o.kind == 2) return fail(PDG_E_UNSUPPORTED, "source step without a lattice model");
        int bi = -1;
        if (o.kind == 0) {
            for (size_t k = 0; k < hs.size(); ++k)
                if (hs[k] == o.h) bi = (int)k;
            if (bi < 0 && hs.size() == (size_t)pdg::kSmallMaxBlk) {
                pdg_status s = flush();
                if (s != PDG_OK) return s;
            }
            if (bi < 0) {
                bi = (int)hs.size();
                if (!fill_blocks(c, o.h, P.blk[bi])) return fail(PDG_E_INVALID_ARGUMENT, "singular cell block for this dt");
                hs.push_back(o.h);
            }
        }
        pdg::SmallOp &so = P.op[P.nops++];
        so.kind = o.kind;
        so.blk = bi;
        if (o.kind == 1) collision_coeffs(c, o.h, &so.ca, &so.cb);
        if (P.nops == pdg::kSmallMaxOps) {
            pdg_status s = flush();
            if (s != PDG_OK) return s;
        }
    }
    return flush();
}

pdg_status execute_ops(pdg_ctx *c, const std::vector<Op> &ops)
{
    if (use_small(c)) return small_run(c, ops);
    const bool fuse = !(c->prob.flags & PDG_NO_FUSION);
    const bool fx = use_relax_x(c);
    const size_t n = ops.size();
    size_t i = 0;
    pdg_status s = PDG_OK;
    while (i < n && s == PDG_OK) {
        if (c->g.lattice && ops[i].kind != 0) {
            // a run of local operators: [S] [C] [S] fused in one pass over f
            double hs1 = 0.0, hs2 = 0.0, hc = 0.0;
            bool with_c = false;
            if (ops[i].kind == 2) hs1 = ops[i++].h;
            if (i < n && ops[i].kind == 1) {
                with_c = true;
                hc = ops[i++].h;
                if (i < n && ops[i].kind == 2) hs2 = ops[i++].h;
            }
            s = local_pass_lbm(c, hs1, with_c, hc, hs2);
            continue;
        }
        if (ops[i].kind == 2) {
            s = fail(PDG_E_UNSUPPORTED, "source step without a lattice model");
            break;
        }
        if (ops[i].kind == 1) {
            int np = 0;
            if (i + 1 < n && ops[i + 1].kind == 0) {
                np = 1;
                if (fuse && i + 2 < n && ops[i + 2].kind == 0 && ops[i + 2].h == ops[i + 1].h) np = 2;
            }
            if (fx && np > 0) {
                s = collide_xsweep(c, ops[i].h, ops[i + 1].h, np);
                if (s == PDG_OK) s = transport_pass(c, ops[i + 1].h, np, SWEEP_YZ);
                i += 1 + np;
            } else {
                s = collide(c, ops[i].h);
                i += 1;
            }
        } else {
            const int np = (fuse && i + 1 < n && ops[i + 1].kind == 0 && ops[i + 1].h == ops[i].h) ? 2 : 1;
            s = transport_pass(c, ops[i].h, np);
            i += np;
        }
    }
    return s;
}

void build_sweep_params(pdg_ctx *c)
{
    const Geometry &g = c->g;
    std::memset(&c->x_params, 0, sizeof(c->x_params));
    std::memset(&c->yz_params, 0, sizeof(c->yz_params));
    std::memset(&c->all_params, 0, sizeof(c->all_params));
    for (auto *sp : {&c->x_params, &c->yz_params, &c->all_params}) {
        sp->f = c->f;
        sp->fb = c->fb;
        sp->f_elems = (int64_t)g.nvl * g.nnodes;
        sp->fb_elems = (int64_t)g.nvl * g.nplanes * g.plane_stride;
        sp->cout_elems = (int64_t)g.carry_doubles;
        sp->cin_elems = (int64_t)g.carry_doubles;
    }
    if (g.lattice) {
        // lattice set: single-axis velocities take the line sweeps, diagonal ones the
        // lattice kernel (lattice_classes), the rest velocity v = 0 is transported by the identity
        for (int j = 0; j < g.nvl; ++j) {
            const int i = g.v0 + j;
            const double *v = c->vel.data() + 3 * i;
            const int act = act_mask(v, g.dim);
            if (popcount3(act) != 1) continue;
            const int k = (act == 1) ? 0 : (act == 2 ? 1 : 2);
            pdg::SweepVel V{};
            V.f_off = (int64_t)j * g.nnodes;
            V.fb_off = ((int64_t)j * g.dim + k) * g.plane_stride;
            V.inner = g.stride[k];
            V.nlines = g.nnodes / g.L[k];
            V.ncells = (int32_t)g.ncell[k];
            V.sign = v[k] > 0.0 ? 1 : -1;
            V.axis = k;
            V.vel = i;
            V.cout_off = -1;
            V.cin_off = -1;
            V.zero_inflow = 0;
            if (k == 0) c->x_params.v[c->x_params.nvel++] = V;
            else c->yz_params.v[c->yz_params.nvel++] = V;
        }
        lattice_classes(g, c->vel.data(), c->lat_plans);
        return;
    }
    for (int j = 0; j < g.nvl; ++j) {
        const int i = g.v0 + j;
        const int k = (i % (2 * g.dim)) / 2;
        const int s = i % 2;
        pdg::SweepVel V{};
        V.f_off = (int64_t)j * g.nnodes;
        V.fb_off = (int64_t)j * g.plane_stride;
        V.inner = g.stride[k];
        V.nlines = g.nnodes / g.L[k];
        V.ncells = (int32_t)g.ncell[k];
        V.sign = s ? -1 : 1;
        V.axis = k;
        V.vel = i;
        V.cout_off = -1;
        V.cin_off = -1;
        V.zero_inflow = 0;
        c->all_params.v[c->all_params.nvel++] = V;
        if (k == 0) c->x_params.v[c->x_params.nvel++] = V;
        else if (g.zslab && k == g.outer) {
            // one entry per local slab: zero inflow unless the velocity enters the domain there
            const int jo = 2 * (i / (2 * g.dim)) + s;  // index among the outer-axis velocities
            for (int t = 0; t < g.nslab_local; ++t) {
                const int sl = g.slab0 + t;
                const int64_t lb = g.slab_begin[sl] - g.cell_begin;
                pdg::SweepVel E = V;
                E.f_off = (int64_t)j * g.nnodes + lb * g.n * g.stride[k];
                E.ncells = (int32_t)(g.slab_begin[sl + 1] - g.slab_begin[sl]);
                E.zero_inflow = (sl == (s ? g.nslab - 1 : 0)) ? 0 : 1;
                E.cout_off = ((int64_t)sl * (2 * g.m) + jo) * 2 * V.nlines;  // pre-pass carries (zcarry)
                E.cin_off = E.zero_inflow ? E.cout_off : -1;                  // exact inflows (zinflow)
                c->outer_entries.push_back(E);
            }
        } else
            c->yz_params.v[c->yz_params.nvel++] = V;
    }
}

// ---- z-slab carry tables ------------------------------------------------------------------
// For one sweep pass structure (T2(dtp) applied npass times): Q_l = g beta^l (response of cell l
// to a unit inflow), P_l (pass-2 response to a unit pass-1 inflow), B_len = beta^len and C_len
// (pass-2 outgoing carry response), computed in long double by running the recurrence on unit
// inputs.  leff: every later l has |P_l|, |Q_l| < 2^-64.  P, Q: [lmax][n]; B, C: [lmax + 1].
bool zslab_tables(int p, long double kappa, int npass, int64_t lmax, std::vector<double> &P, std::vector<double> &Q,
                  std::vector<double> &B, std::vector<double> &C, int *leff_out, int *lpre_out = nullptr)
{
    const int n = p + 1;
    long double M[16], gv[4];
    {
        long double x[4], w[4], D[16], G[16], A[16], Ai[16];
        pdg::gl_nodes(p, x, w);
        pdg::lagrange_derivative(n, x, D);
        for (int i = 0; i < n; ++i)
            for (int jj = 0; jj < n; ++jj) {
                long double v = D[jj * n + i] * w[jj];
                if (i == n - 1 && jj == n - 1) v -= 1.0L;
                G[i * n + jj] = v / w[i];
                A[i * n + jj] = ((i == jj) ? 1.0L : 0.0L) - kappa * G[i * n + jj];
            }
        if (!pdg::invert(n, A, Ai)) return false;
        for (int i = 0; i < n; ++i) {
            for (int jj = 0; jj < n; ++jj) {
                long double acc = 0.0L;
                for (int k = 0; k < n; ++k) acc += Ai[i * n + k] * (((k == jj) ? 1.0L : 0.0L) + kappa * G[k * n + jj]);
                M[i * n + jj] = acc;
            }
            gv[i] = Ai[i * n + 0] * kappa / w[0];
        }
    }
    P.assign((size_t)lmax * n, 0.0);
    Q.assign((size_t)lmax * n, 0.0);
    B.assign(lmax + 1, 0.0);
    C.assign(lmax + 1, 0.0);
    long double c1 = 1.0L, c2 = 0.0L;  // carries of pass 1 (unit inflow) and pass 2 (zero inflow)
    int leff = 0;
    B[0] = 1.0;
    C[0] = 0.0;
    for (int64_t l = 0; l < lmax; ++l) {
        long double d1[4], d2[4];
        for (int a = 0; a < n; ++a) d1[a] = gv[a] * c1;  // pass-1 response (old data 0)
        c1 = d1[n - 1];
        for (int a = 0; a < n; ++a) {
            long double acc = gv[a] * c2;
            for (int b = 0; b < n; ++b) acc += M[a * n + b] * d1[b];
            d2[a] = acc;
        }
        c2 = d1[n - 1] + d2[n - 1];
        bool big = false;
        for (int a = 0; a < n; ++a) {
            P[(size_t)l * n + a] = (double)d2[a];
            Q[(size_t)l * n + a] = (double)d1[a];
            if (fabsl(d1[a]) >= 0x1p-64L || (npass > 1 && fabsl(d2[a]) >= 0x1p-64L)) big = true;
        }
        if (big) leff = (int)l + 1;
        B[l + 1] = (double)c1;
        C[l + 1] = (double)c2;
    }
    *leff_out = leff;
    if (lpre_out) {
        // pre-pass length: the outgoing carries' response to unit data in a cell followed by d
        // cells; every cell whose response reaches 2^-64 is read (lpre = largest such d + 1)
        int lpre = 1;
        for (int b = 0; b < n; ++b) {
            long double f1[4], f2[4];
            for (int a = 0; a < n; ++a) {
                f1[a] = M[a * n + b];
                f2[a] = 0.0L;
            }
            long double e1 = 1.0L * (b == n - 1), cc1 = e1 + f1[n - 1], cc2 = 0.0L;
            if (npass > 1) {
                for (int a = 0; a < n; ++a) {
                    long double acc = 0.0L;
                    for (int q = 0; q < n; ++q) acc += M[a * n + q] * f1[q];
                    f2[a] = acc;
                }
                cc2 = f1[n - 1] + f2[n - 1];
            }
            for (int64_t d = 0; d <= lmax; ++d) {
                if (fabsl(cc1) >= 0x1p-64L || fabsl(cc2) >= 0x1p-64L) lpre = std::max<int>(lpre, (int)d + 1);
                // one more cell of zero data downstream
                long double g1[4], g2[4];
                for (int a = 0; a < n; ++a) g1[a] = gv[a] * cc1;
                const long double n1 = g1[n - 1];
                long double n2 = 0.0L;
                if (npass > 1) {
                    for (int a = 0; a < n; ++a) {
                        long double acc = gv[a] * cc2;
                        for (int q = 0; q < n; ++q) acc += M[a * n + q] * g1[q];
                        g2[a] = acc;
                    }
                    n2 = g1[n - 1] + g2[n - 1];
                }
                cc1 = n1;
                cc2 = n2;
            }
        }
        *lpre_out = lpre;
    }
    return true;
}

pdg_status ztable(pdg_ctx *c, double dtp, int npass, const pdg_ctx::ZTable **out)
{
    for (const auto &t : c->ztables_host)
        if (t.dtp == dtp && t.npass == npass) {
            *out = &t;
            return PDG_OK;
        }
    if ((int)c->ztables_host.size() >= kMaxTables) return fail(PDG_E_UNSUPPORTED, "too many distinct z-slab steps");
    const Geometry &g = c->g;
    int64_t lmax = 0;
    for (int sl = 0; sl < g.nslab; ++sl) lmax = std::max(lmax, g.slab_begin[sl + 1] - g.slab_begin[sl]);
    lmax += 1;
    const long double kappa = (long double)c->prob.lambda * (long double)dtp / (long double)g.h[g.outer];
    std::vector<double> Pt, Qt;
    pdg_ctx::ZTable zt;
    if (!zslab_tables(g.p, kappa, npass, lmax, Pt, Qt, zt.B, zt.C, &zt.leff, &zt.lpre))
        return fail(PDG_E_INVALID_ARGUMENT, "singular cell block");
    zt.dtp = dtp;
    zt.npass = npass;
    c->ztables_host.push_back(zt);
    *out = &c->ztables_host.back();
    return PDG_OK;
}

// Exact inflows of every slab from the outgoing carries, then the correction of the local slabs.
pdg_status zslab_resolve(pdg_ctx *c, double dtp, int npass)
{
    NvtxRange nv("pdg z-slab carries");
    const Geometry &g = c->g;
    const pdg_ctx::ZTable *zt = nullptr;
    pdg_status st = ztable(c, dtp, npass, &zt);
    if (st != PDG_OK) return st;
    const int e = prof_begin(c);
    if (c->prob.nranks > 1) {
        std::string err;
        if (!c->comm.comm) return fail(PDG_E_NCCL, "z-slab decomposition over ranks needs nccl_id");
        const size_t per_rank = g.carry_doubles / (size_t)c->prob.nranks;
        if (!c->comm.allgather(c->zcarry, per_rank, c->prob.rank, c->stream, &err)) return fail(PDG_E_NCCL, err);
    }
    pdg::ZSlabParams P;
    std::memset(&P, 0, sizeof(P));
    P.carry = c->zcarry;
    P.inflow = c->zinflow;
    P.carry_elems = (int64_t)g.carry_doubles;
    P.plane = g.nnodes / g.L[g.outer];
    P.nslab = g.nslab;
    P.nvo = 2 * g.m;
    P.npass = npass;
    for (int jo = 0; jo < P.nvo; ++jo) P.sign[jo] = (jo % 2) ? -1 : 1;
    for (int sl = 0; sl < g.nslab; ++sl) {
        const int len = (int)(g.slab_begin[sl + 1] - g.slab_begin[sl]);
        P.B[sl] = zt->B[len];
        P.C[sl] = zt->C[len];
    }
    dim3 g1((unsigned)((P.plane + 255) / 256), (unsigned)P.nvo);
    pdg::zslab_scan_kernel<<<g1, 256, 0, c->stream>>>(P);
    prof_end(c, e, PDG_K_ZSLAB, 8.0 * 3.0 * (double)g.carry_doubles);
    return post_launch(c, "zslab_scan");
}

// ---- pdg_step as a replayed CUDA graph ---------------------------------------------------
// A step is 2-3 dependent launches; for small grids (configs 1-2) the gaps between launches are
// a large part of the step (config 2: 71 -> 53 us per step, config 1: 22 -> 7 us when replayed
// from a graph; bench.py --graph).  pdg_step(n) therefore captures its n-step launch sequence
// once per n (on a library stream, so the caller's stream may be the legacy default stream) and
// replays it on the caller's stream.  Not used with per-launch profiling events, synchronous error
// checks, a communicator (NCCL), PDG_NO_GRAPH, or when the caller's stream is itself being captured
// (the launches then go into the caller's graph directly).
constexpr int64_t kMaxGraphSteps = 1024;  // longer calls launch directly (same launches, same results)
constexpr size_t kMaxStepGraphs = 8;

bool use_step_graph(pdg_ctx *c, int64_t nsteps)
{
    if (nsteps < 2 || nsteps > kMaxGraphSteps || c->graphs_off || c->comm.comm || c->prob.nranks > 1) return false;
    if ((c->prof.on && !c->prof.paused) || (c->prob.flags & (PDG_SYNC_ERRORS | PDG_NO_GRAPH))) return false;
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(c->stream, &st) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return st == cudaStreamCaptureStatusNone;
}

void destroy_step_graphs(pdg_ctx *c)
{
    for (auto &kv : c->step_graphs)
        if (kv.second) cudaGraphExecDestroy(kv.second);
    c->step_graphs.clear();
}

pdg_status step_graph(pdg_ctx *c, int64_t nsteps, const std::vector<Op> &ops)
{
    auto it = c->step_graphs.find(nsteps);
    cudaGraphExec_t exec = (it != c->step_graphs.end()) ? it->second : nullptr;
    if (!exec) {
        if (!c->cap_stream) {
            int prio = 0;
            cudaStreamGetPriority(c->stream, &prio);
            PDG_CUDA_TRY(cudaStreamCreateWithPriority(&c->cap_stream, cudaStreamNonBlocking, prio));
        }
        if (c->step_graphs.size() >= kMaxStepGraphs) destroy_step_graphs(c);
        cudaStream_t user = c->stream;
        c->stream = c->cap_stream;  // every launch of execute_ops goes to the capturing stream
        cudaGraph_t graph = nullptr;
        pdg_status s = PDG_OK;
        cudaError_t e = cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal);
        if (e == cudaSuccess) {
            s = execute_ops(c, ops);
            e = cudaStreamEndCapture(c->cap_stream, &graph);
        }
        c->stream = user;
        if (s == PDG_OK && e == cudaSuccess && graph) e = cudaGraphInstantiate(&exec, graph, 0);
        if (graph) cudaGraphDestroy(graph);
        if (s != PDG_OK || e != cudaSuccess || !exec) {
            // capture or instantiation failed: direct launches for this context from now on
            cudaGetLastError();
            c->graphs_off = true;
            return execute_ops(c, ops);
        }
        c->step_graphs[nsteps] = exec;
    }
    PDG_CUDA_TRY(cudaGraphLaunch(exec, c->stream));
    return post_launch(c, "step graph");
}

bool is_device_pointer(const void *p)
{
    cudaPointerAttributes attr;
    if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged;
}

}  // namespace

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

pdg_status pdg_query_sizes(const pdg_problem *p, pdg_sizes *out)
{
    if (!out) return fail(PDG_E_INVALID_ARGUMENT, "out is NULL");
    Geometry g;
    pdg_status s = validate(p, &g);
    if (s != PDG_OK) return s;
    fill_sizes(g, out);
    return PDG_OK;
}

pdg_status pdg_create(const pdg_problem *p, double *f_dev, double *fb_dev, double *w_dev, void *work_dev,
                      pdg_ctx **out)
{
    if (!out) return fail(PDG_E_INVALID_ARGUMENT, "out is NULL");
    *out = nullptr;
    Geometry g;
    pdg_status s = validate(p, &g);
    if (s != PDG_OK) return s;
    if (!f_dev || !fb_dev || !w_dev || !work_dev) return fail(PDG_E_BUFFER, "device buffers must be non-NULL");
    for (const void *ptr : {(const void *)f_dev, (const void *)fb_dev, (const void *)w_dev, (const void *)work_dev})
        if (!is_device_pointer(ptr)) return fail(PDG_E_BUFFER, "buffers must be device memory");
    pdg_ctx *c = new pdg_ctx();
    c->g = g;
    c->prob = *p;
    c->vel.assign(p->vel, p->vel + 3 * p->nv);
    if (p->comp) c->comp.assign(p->comp, p->comp + p->nv);
    else c->comp.assign(p->nv, 0);
    for (int i = 0; i < p->n_flux_params && i < 3; ++i) c->fparams[i] = p->flux_params[i];
    c->prob.vel = c->vel.data();
    c->prob.comp = c->comp.data();
    c->prob.flux_params = c->fparams;
    c->prob.nccl_id = nullptr;
    c->prob.source_params = nullptr;  // copied into c->lbm.G
    c->f = f_dev;
    c->fb = fb_dev;
    c->w = w_dev;
    c->counter = (unsigned long long *)work_dev;
    c->stream = (cudaStream_t)p->cuda_stream;
    cudaGetDevice(&c->device);
    cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, c->device);
    {
        int l2 = 0;
        cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, c->device);
        c->l2keep = (double)c->g.nvl * (double)c->g.nnodes * sizeof(double) <= 0.7 * (double)l2;
    }
    std::memset(&c->mp, 0, sizeof(c->mp));
    if (p->flux == PDG_FLUX_LINEAR_ADVECTION)
        for (int d = 0; d < p->dim; ++d) c->mp.a[d] = p->flux_params[d];
    if (p->flux == PDG_FLUX_EULER) c->mp.gamma = p->flux_params[0];
    if (p->flux == PDG_FLUX_ISOTHERMAL) c->mp.c2 = p->flux_params[0] * p->flux_params[0];
    c->mp.inv2D = 1.0 / (2.0 * p->dim);
    c->mp.inv2lam = 1.0 / (2.0 * p->lambda);
    if (c->g.lattice) {
        const double cc = p->flux_params[0];
        for (int i = 0; i < p->nv; ++i) {
            for (int d = 0; d < 3; ++d) c->lbm.v[i][d] = p->vel[3 * i + d];
            c->lbm.wgt[i] = p->flux_params[1 + i];
        }
        c->lbm.inv_c2 = 1.0 / (cc * cc);
        c->lbm.inv_2c4 = 1.0 / (2.0 * cc * cc * cc * cc);
        c->lbm.inv_2c2 = 1.0 / (2.0 * cc * cc);
        if (p->source == PDG_SOURCE_GRAVITY)
            for (int d = 0; d < p->dim; ++d) c->lbm.G[d] = p->source_params[d];
        char *base = static_cast<char *>(work_dev) + 256;
        c->lat_ints = reinterpret_cast<int *>(base);
        c->lat_xbuf = reinterpret_cast<double *>(base + lat_ints_bytes(c->g));
        c->lat_ybuf = c->lat_xbuf + c->g.lat_xbuf;
        c->lat_gtab_base = c->lat_ybuf + c->g.lat_ybuf;
        // the tagged x/y-trace words start out empty; every launch's consumers empty them again
        if ((c->g.lat_xbuf + c->g.lat_ybuf) &&
            cudaMemsetAsync(c->lat_xbuf, 0, sizeof(double) * (c->g.lat_xbuf + c->g.lat_ybuf), c->stream) != cudaSuccess) {
            pdg_destroy(c);
            return fail(PDG_E_CUDA, "cannot clear the lattice trace buffers");
        }
    }
    if (c->g.zslab) {
        c->zcarry = reinterpret_cast<double *>(static_cast<char *>(work_dev) + 256);
        c->zinflow = c->zcarry + c->g.carry_doubles;
    }
    build_sweep_params(c);
    if (!c->lat_plans.empty()) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        int prio = 0;
        cudaStreamGetPriority(c->stream, &prio);
        bool ok = cudaEventCreateWithFlags(&c->lat_fork, cudaEventDisableTiming) == cudaSuccess;
        for (size_t k = 0; k < c->lat_plans.size() && ok; ++k) {
            cudaStream_t st = nullptr;
            cudaEvent_t ev = nullptr;
            ok = cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, prio) == cudaSuccess &&
                 cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess;
            c->lat_streams.push_back(st);
            c->lat_join.push_back(ev);
        }
        if (!ok) {
            pdg_destroy(c);
            return fail(PDG_E_CUDA, "cannot create the lattice class streams");
        }
        // large block tables (p = 3 body diagonals) of the scheme's steps, uploaded now
        if (c->g.n == 4 && c->g.dim == 3) {
            std::vector<Op> ops;
            append_scheme(ops, p->scheme, p->dt);
            for (const LatPlan &pl : c->lat_plans) {
                if (pl.act != 7) continue;
                for (const Op &o : ops) {
                    if (o.kind != 0) continue;
                    const pdg::LatticeBlockLD *B = lattice_block_for(c, pl.act, o.h);
                    pdg_status ps = B ? launch_lattice_t<3, 4, 7>(c, pl, *B, o.h, nullptr)
                                      : fail(PDG_E_INVALID_ARGUMENT, "singular lattice block");
                    if (ps != PDG_OK) {
                        pdg_destroy(c);
                        return ps;
                    }
                }
            }
        }
    }
    if (c->g.zslab) {  // tables of the scheme's sweeps (single and fused double passes)
        std::vector<Op> ops;
        append_scheme(ops, p->scheme, p->dt);
        for (const Op &o : ops)
            if (o.kind == 0)
                for (int np = 1; np <= 2; ++np) {
                    const pdg_ctx::ZTable *zt = nullptr;
                    pdg_status zs = ztable(c, o.h, np, &zt);
                    if (zs != PDG_OK) {
                        pdg_destroy(c);
                        return zs;
                    }
                }
    }
    if (c->g.async_host) {
        c->w_stage = reinterpret_cast<double *>(static_cast<char *>(work_dev) + w_stage_offset(c->g));
        int prio = 0;
        cudaStreamGetPriority(c->stream, &prio);
        if (cudaStreamCreateWithPriority(&c->copy_stream, cudaStreamNonBlocking, prio) != cudaSuccess ||
            cudaStreamCreateWithPriority(&c->upload_stream, cudaStreamNonBlocking, prio) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->w_ready, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->d2h_done, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->stage_free, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->stage_full, cudaEventDisableTiming) != cudaSuccess) {
            pdg_destroy(c);
            return fail(PDG_E_CUDA, "cannot create the PDG_ASYNC_HOST copy stream");
        }
    }
    if (p->flags & PDG_PROFILE) {
        c->prof.on = true;
        c->prof.ev.resize(2 * 4096);
        for (auto &e : c->prof.ev) {
            if (cudaEventCreate(&e) != cudaSuccess) {
                e = nullptr;
                c->prof.on = false;
            }
        }
        if (!c->prof.on) {
            pdg_destroy(c);  // destroys the events that were created
            return fail(PDG_E_CUDA, "cudaEventCreate failed");
        }
    }
    if (p->nccl_id) {
        std::string err;
        if (!c->comm.init(p->nccl_id, p->nranks, p->rank, &err)) {
            pdg_destroy(c);
            return fail(PDG_E_NCCL, err);
        }
        int prio = 0;
        cudaStreamGetPriority(c->stream, &prio);
        bool ok = cudaStreamCreateWithPriority(&c->comm_stream, cudaStreamNonBlocking, prio) == cudaSuccess;
        for (int k = 0; k < kMaxChunks && ok; ++k)
            ok = cudaEventCreateWithFlags(&c->ev_pm[k], cudaEventDisableTiming) == cudaSuccess &&
                 cudaEventCreateWithFlags(&c->ev_ar[k], cudaEventDisableTiming) == cudaSuccess;
        if (!ok) {
            pdg_destroy(c);
            return fail(PDG_E_CUDA, "cannot create the communicator stream");
        }
    }
    *out = c;
    return PDG_OK;
}

pdg_status pdg_set_state(pdg_ctx *c, const double *f, const double *fb, int on_device)
{
    DeviceGuard dg(c);
    if (!c) return fail(PDG_E_INVALID_ARGUMENT, "ctx is NULL");
    const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    if (f) PDG_CUDA_TRY(cudaMemcpyAsync(c->f, f, sizeof(double) * c->g.nvl * c->g.nnodes, kind, c->stream));
    if (fb)
        PDG_CUDA_TRY(cudaMemcpyAsync(c->fb, fb, sizeof(double) * c->g.nvl * c->g.nplanes * c->g.plane_stride, kind,
                                     c->stream));
    const bool sync = (!on_device && !c->g.async_host) || (c->prob.flags & PDG_SYNC_ERRORS);
    if (sync) PDG_CUDA_TRY(cudaStreamSynchronize(c->stream));
    c->state_set = true;
    return PDG_OK;
}

pdg_status pdg_set_equilibrium(pdg_ctx *c, const double *w, const double *wb, int on_device)
{
    DeviceGuard dg(c);
    if (!c) return fail(PDG_E_INVALID_ARGUMENT, "ctx is NULL");
    if (!w) return fail(PDG_E_INVALID_ARGUMENT, "w is NULL");
    const size_t wbytes = sizeof(double) * c->g.m * c->g.nnodes;
    if (!on_device && c->g.async_host && !wb) {
        // PDG_ASYNC_HOST: upload into the staging region on the upload stream as soon as the previous
        // equilibrium has consumed it (so it overlaps the previous step and its download; w_dev stays
        // free for a pending download), then the equilibrium on the context stream
        PDG_CUDA_TRY(cudaStreamWaitEvent(c->upload_stream, c->stage_free, 0));
        PDG_CUDA_TRY(cudaMemcpyAsync(c->w_stage, w, wbytes, cudaMemcpyHostToDevice, c->upload_stream));
        PDG_CUDA_TRY(cudaEventRecord(c->stage_full, c->upload_stream));
        PDG_CUDA_TRY(cudaStreamWaitEvent(c->stream, c->stage_full, 0));
        if (c->g.lattice) PDG_LBM_DISPATCH(launch_equilibrium_lbm_t, c, c->w_stage, c->w_stage, false);
        else PDG_DISPATCH(launch_equilibrium_t, c, c->w_stage, c->w_stage);
        PDG_CUDA_TRY(cudaEventRecord(c->stage_free, c->stream));
        pdg_status s = post_launch(c, "equilibrium(async)");
        if (s != PDG_OK) return s;
        c->state_set = true;
        return PDG_OK;
    }
    if (!on_device) wait_w_download(c);  // the host paths stage through w_dev
    if (c->g.lattice) {
        if (!on_device) {
            PDG_CUDA_TRY(cudaMemcpyAsync(c->w, wb ? wb : w, wbytes, cudaMemcpyHostToDevice, c->stream));
            PDG_LBM_DISPATCH(launch_equilibrium_lbm_t, c, wb ? nullptr : c->w, c->w, false);
            if (wb) {
                PDG_CUDA_TRY(cudaMemcpyAsync(c->w, w, wbytes, cudaMemcpyHostToDevice, c->stream));
                PDG_LBM_DISPATCH(launch_equilibrium_lbm_t, c, c->w, nullptr, true);
            }
            pdg_status s = post_launch(c, "equilibrium");
            if (s != PDG_OK) return s;
            PDG_CUDA_TRY(cudaStreamSynchronize(c->stream));
        } else {
            PDG_LBM_DISPATCH(launch_equilibrium_lbm_t, c, w, wb ? wb : w, false);
            pdg_status s = post_launch(c, "equilibrium");
            if (s != PDG_OK) return s;
        }
        c->state_set = true;
        return PDG_OK;
    }
    if (!on_device) {
        // stage through w_dev: inflow data first (from wb), then the interior (from w)
        PDG_CUDA_TRY(cudaMemcpyAsync(c->w, wb ? wb : w, wbytes, cudaMemcpyHostToDevice, c->stream));
        PDG_DISPATCH(launch_equilibrium_t, c, c->w, c->w);
        pdg_status s = post_launch(c, "equilibrium(wb)");
        if (s != PDG_OK) return s;
        if (wb) {
            PDG_CUDA_TRY(cudaMemcpyAsync(c->w, w, wbytes, cudaMemcpyHostToDevice, c->stream));
            const int grid = grid_for(c, c->g.nnodes, 256);
            const int dim = c->g.dim, mod = c->prob.flux;
#define PDG_EQ_ONLY(D, MO) pdg::equilibrium_kernel<D, MO><<<grid, 256, 0, c->stream>>>(c->f, c->w, c->g.nnodes, c->g.v0, c->g.nvl, c->mp)
            if (dim == 2 && mod == 0) PDG_EQ_ONLY(2, pdg::MODEL_ADV);
            else if (dim == 2 && mod == 1) PDG_EQ_ONLY(2, pdg::MODEL_EULER);
            else if (dim == 2 && mod == 2) PDG_EQ_ONLY(2, pdg::MODEL_ISO);
            else if (dim == 3 && mod == 0) PDG_EQ_ONLY(3, pdg::MODEL_ADV);
            else if (dim == 3 && mod == 1) PDG_EQ_ONLY(3, pdg::MODEL_EULER);
            else PDG_EQ_ONLY(3, pdg::MODEL_ISO);
#undef PDG_EQ_ONLY
            s = post_launch(c, "equilibrium(w)");
            if (s != PDG_OK) return s;
        }
        PDG_CUDA_TRY(cudaStreamSynchronize(c->stream));
    } else {
        PDG_DISPATCH(launch_equilibrium_t, c, w, wb ? wb : w);
        pdg_status s = post_launch(c, "equilibrium");
        if (s != PDG_OK) return s;
    }
    c->state_set = true;
    return PDG_OK;
}

pdg_status pdg_get_state(pdg_ctx *c, double *f, int on_device)
{
    DeviceGuard dg(c);
    if (!c || !f) return fail(PDG_E_INVALID_ARGUMENT, "NULL argument");
    PDG_CUDA_TRY(cudaMemcpyAsync(f, c->f, sizeof(double) * c->g.nvl * c->g.nnodes,
                                 on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c->stream));
    if (!on_device && !c->g.async_host) PDG_CUDA_TRY(cudaStreamSynchronize(c->stream));
    return PDG_OK;
}

pdg_status pdg_transport(pdg_ctx *c, double dtp)
{
    DeviceGuard dg(c);
    if (!c) return fail(PDG_E_INVALID_ARGUMENT, "ctx is NULL");
    if (!c->state_set) return fail(PDG_E_STATE_NOT_SET, "set the state first");
    if (!std::isfinite(dtp)) return fail(PDG_E_INVALID_ARGUMENT, "dtp must be finite");
    return transport_pass(c, dtp, 1);
}

pdg_status pdg_collide(pdg_ctx *c, double dt)
{
    DeviceGuard dg(c);
    if (!c) return fail(PDG_E_INVALID_ARGUMENT, "ctx is NULL");
    if (!c->state_set) return fail(PDG_E_STATE_NOT_SET, "set the state first");
    if (!std::isfinite(dt) || !collision_step_ok(c->prob.tau, dt))
        return fail(PDG_E_INVALID_ARGUMENT, "collision needs a finite dt with 2 tau + dt > 0 (tau > 0)");
    return collide(c, dt);
}

pdg_status pdg_source(pdg_ctx *c, double h)
{
    DeviceGuard dg(c);
    if (!c) return fail(PDG_E_INVALID_ARGUMENT, "ctx is NULL");
    if (!c->state_set) return fail(PDG_E_STATE_NOT_SET, "set the state first");
    if (c->prob.source == PDG_SOURCE_NONE) return fail(PDG_E_INVALID_ARGUMENT, "the problem has no source");
    if (!std::isfinite(h)) return fail(PDG_E_INVALID_ARGUMENT, "h must be finite");
    return local_pass_lbm(c, h, false, 0.0, 0.0);
}

pdg_status pdg_partial_moments(pdg_ctx *c)
{
    DeviceGuard dg(c);
    if (!c) return fail(PDG_E_INVALID_ARGUMENT, "ctx is NULL");
    wait_w_download(c);  // PDG_ASYNC_HOST: a pending pdg_moments download may still read w_dev
    if (c->g.lattice) PDG_LBM_DISPATCH(launch_partial_lbm_t, c, 0, c->g.nnodes);
    else PDG_DISPATCH(launch_partial_t, c, 0, c->g.nnodes);
    return post_launch(c, "partial_moments");
}

pdg_status pdg_relax_from_w(pdg_ctx *c, double dt)
{
    DeviceGuard dg(c);
    if (!c) return fail(PDG_E_INVALID_ARGUMENT, "ctx is NULL");
    if (!std::isfinite(dt) || !collision_step_ok(c->prob.tau, dt))
        return fail(PDG_E_INVALID_ARGUMENT, "collision needs a finite dt with 2 tau + dt > 0 (tau > 0)");
    double ca, cb;
    collision_coeffs(c, dt, &ca, &cb);
    if (c->g.lattice) {
        pdg::LocalOps op{0.0, ca, cb, 0.0};
        PDG_LBM_DISPATCH(launch_relax_from_w_lbm_t, c, 0, c->g.nnodes, op);
    } else {
        PDG_DISPATCH(launch_relax_from_w_t, c, 0, c->g.nnodes, ca, cb);
    }
    return post_launch(c, "relax_from_w");
}

pdg_status pdg_step(pdg_ctx *c, int64_t nsteps)
{
    DeviceGuard dg(c);
    NvtxRange nv("pdg_step");
    if (!c) return fail(PDG_E_INVALID_ARGUMENT, "ctx is NULL");
    if (nsteps < 0) return fail(PDG_E_INVALID_ARGUMENT, "nsteps must be >= 0");
    if (nsteps == 0) return PDG_OK;
    if (!c->state_set) return fail(PDG_E_STATE_NOT_SET, "set the state first");
    std::vector<Op> ops;
    for (int64_t k = 0; k < nsteps; ++k) append_scheme(ops, c->prob.scheme, c->prob.dt);
    pdg_status s = use_step_graph(c, nsteps) ? step_graph(c, nsteps, ops) : execute_ops(c, ops);
    if (s != PDG_OK) return s;
    if (c->prob.flags & PDG_CHECK_STATE) {
        int64_t bad = 0;
        s = pdg_check_state(c, &bad);
        if (s != PDG_OK) return s;
        if (bad > 0) return fail(PDG_E_NONPHYSICAL, std::to_string(bad) + " nodes with rho <= 0 or non-finite f");
    }
    return PDG_OK;
}

pdg_status pdg_moments(pdg_ctx *c, double *w, int on_device)
{
    DeviceGuard dg(c);
    if (!c || !w) return fail(PDG_E_INVALID_ARGUMENT, "NULL argument");
    pdg_status s = partial_and_reduce(c);
    if (s != PDG_OK) return s;
    const size_t bytes = sizeof(double) * c->g.m * c->g.nnodes;
    if (!on_device && c->g.async_host) {
        // download on the copy stream: the context stream goes on (next upload, next step)
        PDG_CUDA_TRY(cudaEventRecord(c->w_ready, c->stream));
        PDG_CUDA_TRY(cudaStreamWaitEvent(c->copy_stream, c->w_ready, 0));
        PDG_CUDA_TRY(cudaMemcpyAsync(w, c->w, bytes, cudaMemcpyDeviceToHost, c->copy_stream));
        PDG_CUDA_TRY(cudaEventRecord(c->d2h_done, c->copy_stream));
        return PDG_OK;
    }
    if (w != c->w)
        PDG_CUDA_TRY(cudaMemcpyAsync(w, c->w, bytes, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                                     c->stream));
    if (!on_device) PDG_CUDA_TRY(cudaStreamSynchronize(c->stream));
    return PDG_OK;
}

pdg_status pdg_check_state(pdg_ctx *c, int64_t *n_bad)
{
    DeviceGuard dg(c);
    if (!c || !n_bad) return fail(PDG_E_INVALID_ARGUMENT, "NULL argument");
    PDG_CUDA_TRY(cudaMemsetAsync(c->counter, 0, sizeof(unsigned long long), c->stream));
    const int grid = grid_for(c, c->g.nnodes, 256);
    const int check_rho = (c->prob.flux != PDG_FLUX_LINEAR_ADVECTION && !sharded(c)) ? 1 : 0;
    const int nrho = c->g.lattice ? c->g.nv : 2 * c->g.dim;  // velocities whose sum is rho
    pdg::check_state_kernel<<<grid, 256, 0, c->stream>>>(c->f, c->g.nnodes, c->g.v0, c->g.nvl, nrho, check_rho,
                                                         c->counter);
    pdg_status s = post_launch(c, "check_state");
    if (s != PDG_OK) return s;
    unsigned long long h = 0;
    PDG_CUDA_TRY(cudaMemcpyAsync(&h, c->counter, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    PDG_CUDA_TRY(cudaStreamSynchronize(c->stream));
    *n_bad = (int64_t)h;
    return PDG_OK;
}

pdg_status pdg_cell_block(const pdg_ctx *c, int axis, double dtp, double *M, double *g, double *beta)
{
    if (!c || !M || !g || !beta) return fail(PDG_E_INVALID_ARGUMENT, "NULL argument");
    if (axis < 0 || axis >= c->g.dim) return fail(PDG_E_INVALID_ARGUMENT, "bad axis");
    pdg::CellBlock cb;
    const long double kappa = (long double)c->prob.lambda * (long double)dtp / (long double)c->g.h[axis];
    if (!pdg::cell_block(c->g.p, kappa, &cb)) return fail(PDG_E_INVALID_ARGUMENT, "singular block");
    for (int i = 0; i < cb.n * cb.n; ++i) M[i] = cb.M[i];
    for (int i = 0; i < cb.n; ++i) g[i] = cb.g[i];
    *beta = cb.beta;
    return PDG_OK;
}

pdg_status pdg_zslab_table(const pdg_problem *p, double dtp, int npass, int64_t len, double *P, double *Q,
                           double *B, double *C, int32_t *leff)
{
    Geometry g;
    pdg_status s = validate(p, &g);
    if (s != PDG_OK) return s;
    if ((npass != 1 && npass != 2) || len < 1 || !std::isfinite(dtp))
        return fail(PDG_E_INVALID_ARGUMENT, "npass must be 1 or 2, len >= 1, dtp finite");
    if (!P || !Q || !B || !C || !leff) return fail(PDG_E_INVALID_ARGUMENT, "NULL argument");
    const int outer = p->dim - 1;
    const long double h = ((long double)p->hi[outer] - (long double)p->lo[outer]) / (long double)p->ncell[outer];
    const long double kappa = (long double)p->lambda * (long double)dtp / h;
    std::vector<double> Pt, Qt, Bt, Ct;
    int le = 0;
    if (!zslab_tables(p->degree, kappa, npass, len, Pt, Qt, Bt, Ct, &le))
        return fail(PDG_E_INVALID_ARGUMENT, "singular cell block");
    std::memcpy(P, Pt.data(), sizeof(double) * Pt.size());
    std::memcpy(Q, Qt.data(), sizeof(double) * Qt.size());
    *B = Bt[len];
    *C = Ct[len];
    *leff = le;
    return PDG_OK;
}

pdg_status pdg_synchronize(pdg_ctx *c)
{
    DeviceGuard dg(c);
    if (!c) return fail(PDG_E_INVALID_ARGUMENT, "ctx is NULL");
    PDG_CUDA_TRY(cudaStreamSynchronize(c->stream));
    if (c->copy_stream) PDG_CUDA_TRY(cudaStreamSynchronize(c->copy_stream));
    if (c->upload_stream) PDG_CUDA_TRY(cudaStreamSynchronize(c->upload_stream));
    return PDG_OK;
}

void pdg_destroy(pdg_ctx *c)
{
    DeviceGuard dg(c);
    if (!c) return;
    if (c->copy_stream) {
        cudaStreamSynchronize(c->copy_stream);
        cudaStreamDestroy(c->copy_stream);
    }
    if (c->upload_stream) {
        cudaStreamSynchronize(c->upload_stream);
        cudaStreamDestroy(c->upload_stream);
    }
    for (cudaEvent_t ev : {c->w_ready, c->d2h_done, c->stage_free, c->stage_full})
        if (ev) cudaEventDestroy(ev);
    if (c->comm_stream) {
        cudaStreamSynchronize(c->comm_stream);
        cudaStreamDestroy(c->comm_stream);
    }
    cudaStreamSynchronize(c->stream);  // a replayed step graph may still run on the caller's stream
    destroy_step_graphs(c);
    if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
    for (int k = 0; k < kMaxChunks; ++k) {
        if (c->ev_pm[k]) cudaEventDestroy(c->ev_pm[k]);
        if (c->ev_ar[k]) cudaEventDestroy(c->ev_ar[k]);
    }
    c->comm.destroy();
    for (auto st : c->lat_streams)
        if (st) cudaStreamDestroy(st);
    for (auto ev : c->lat_join)
        if (ev) cudaEventDestroy(ev);
    if (c->lat_fork) cudaEventDestroy(c->lat_fork);
    for (auto &e : c->prof.ev)
        if (e) cudaEventDestroy(e);
    delete c;
}

pdg_status pdg_nccl_unique_id(void *out)
{
    if (!out) return fail(PDG_E_INVALID_ARGUMENT, "out is NULL");
    std::string err;
    if (!pdg::NcclComm::unique_id(out, &err)) return fail(PDG_E_NCCL, err);
    return PDG_OK;
}

pdg_status pdg_profile_read(pdg_ctx *c, double *ms, int64_t *launches, double *alg_bytes)
{
    DeviceGuard dg(c);
    if (!c) return fail(PDG_E_INVALID_ARGUMENT, "ctx is NULL");
    double t[PDG_NUM_KERNEL_KINDS] = {0}, b[PDG_NUM_KERNEL_KINDS] = {0};
    int64_t n[PDG_NUM_KERNEL_KINDS] = {0};
    PDG_CUDA_TRY(cudaStreamSynchronize(c->stream));
    for (const ProfRec &r : c->prof.recs) {
        float e = 0.f;
        PDG_CUDA_TRY(cudaEventElapsedTime(&e, c->prof.ev[r.ev], c->prof.ev[r.ev + 1]));
        t[r.kind] += e;
        b[r.kind] += r.bytes;
        n[r.kind] += 1;
    }
    c->prof.recs.clear();
    c->prof.next = 0;
    for (int k = 0; k < PDG_NUM_KERNEL_KINDS; ++k) {
        if (ms) ms[k] = t[k];
        if (launches) launches[k] = n[k];
        if (alg_bytes) alg_bytes[k] = b[k];
    }
    return PDG_OK;
}

pdg_status pdg_profile_enable(pdg_ctx *c, int on)
{
    if (!c) return fail(PDG_E_INVALID_ARGUMENT, "ctx is NULL");
    if (!c->prof.on) return fail(PDG_E_INVALID_ARGUMENT, "the context was created without PDG_PROFILE");
    c->prof.paused = (on == 0);
    return PDG_OK;
}

const char *pdg_status_string(pdg_status s)
{
    switch (s) {
    case PDG_OK: return "PDG_OK";
    case PDG_E_INVALID_ARGUMENT: return "PDG_E_INVALID_ARGUMENT";
    case PDG_E_DIMENSION: return "PDG_E_DIMENSION";
    case PDG_E_DEGREE: return "PDG_E_DEGREE";
    case PDG_E_VELOCITY_SET: return "PDG_E_VELOCITY_SET";
    case PDG_E_FLUX_MODEL: return "PDG_E_FLUX_MODEL";
    case PDG_E_STATE_NOT_SET: return "PDG_E_STATE_NOT_SET";
    case PDG_E_NONPHYSICAL: return "PDG_E_NONPHYSICAL";
    case PDG_E_CUDA: return "PDG_E_CUDA";
    case PDG_E_NCCL: return "PDG_E_NCCL";
    case PDG_E_BUFFER: return "PDG_E_BUFFER";
    case PDG_E_UNSUPPORTED: return "PDG_E_UNSUPPORTED";
    }
    return "PDG_E_UNKNOWN";
}

const char *pdg_last_error(void) { return g_last_error.c_str(); }

const char *pdg_version(void) { return "pdg-b200 " PDG_VERSION " sm_100a"; }

}  // extern "C"
