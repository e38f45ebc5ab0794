/*
 * include/pdg.h -- C-ABI of libpdg, the B200-native hot path of the
 * Palindromic Discontinuous Galerkin (PDG) method, arxiv 1702.00169.
 *
 * One call of pdg_step() advances a vectorial kinetic BGK system (P:110-138,
 * eq kin_bgk, with tau = 0 and no source) by the palindromic step
 *
 *     M2(dt) = T2(dt/2) C2(dt) T2(dt/2)
 *
 * where T2 is the Crank-Nicolson upwind-DG transport of every velocity
 * (P:440-444 eq transport_cn, solved by the downwind sweep of P:622-637) and
 * C2 is the relaxation f <- 2 f^eq(w) - f with w = P f.
 * "P:n" = line n of the paper's LaTeX source.  Readings of silent or
 * garbled passages are listed in DESIGN.md ("readings C1..C19").
 *
 * Conventions (all entry points):
 *  - fp64 everywhere; every pointer is owned by the caller.  Host arrays are
 *    read/written during the call only.  Device buffers given to pdg_create stay
 *    bound to the context until pdg_destroy.  The library never allocates
 *    device memory.
 *  - Errors are returned as pdg_status codes; nothing aborts or throws.  A
 *    human-readable detail of the last failure on the calling thread is
 *    available from pdg_last_error().  After PDG_E_CUDA the context must be
 *    destroyed.  Kernel faults are asynchronous and surface at the next
 *    synchronising call (or immediately with PDG_SYNC_ERRORS).
 *  - All device work is enqueued on the stream given in pdg_problem.cuda_stream
 *    (a cudaStream_t, NULL = legacy default stream); pdg_step/pdg_transport/
 *    pdg_collide are asynchronous and CUDA-graph capturable when nranks == 1.
 *  - One context per device; calls on one context are serialised by the caller.  The context
 *    is bound to the device that was current at pdg_create: every call taking a context makes
 *    that device current for its duration and restores the caller's device on return.
 *
 * Canonical layouts (row-major, last index fastest):
 *  - node grid: for an N_0 x N_1 (x N_2) cell box of degree p, n = p+1 nodes per
 *    cell and axis; node index (Z, Y, X) with X = c_x*n + a_x (a_x = local GL
 *    node along x), same for Y, Z.  nnodes = prod_d (N_d * n).
 *  - f:  [nv_local][Z][Y][X]   (local velocities of this rank, see pdg_sizes; with PDG_DECOMP_ZSLAB
 *        all velocities and only the rank's planes cell_begin..cell_begin+cell_count-1 of the slowest axis)
 *  - fb: [nv_local][plane_stride]; velocity i (axis k_i) stores its inflow
 *        plane = the node grid with axis k_i removed, in the same order
 *        (e.g. axis y in 3-D: [Z][X]); plane_stride = max over axes.
 *        PDG_FLUX_LBM (lattice sets): [nv_local][dim][plane_stride]: plane k of velocity i is
 *        its inflow face across axis k (lo face if v_i^k > 0, hi face if v_i^k < 0), same
 *        order as above; planes of axes with v_i^k = 0 are unused.
 *  - w:  [m][Z][Y][X]   (the rank's planes with PDG_DECOMP_ZSLAB)
 *
 * Velocity set: the vectorial D2Q4 / D3Q6-per-component set (reading C6):
 *   velocity i = c*2D + 2k + s has v_i = (s ? -lambda : +lambda) e_k and
 *   belongs to component c (P = block sums).  Any other set is rejected with
 *   PDG_E_VELOCITY_SET -- except with PDG_FLUX_LBM, which takes a lattice set
 *   (components in {0, +-lambda}, e.g. the paper's D2Q9): velocities with
 *   several non-zero components are swept along genuinely diagonal wavefronts with the
 *   dense (p+1)^d local block (NEXT-2).
 */
#ifndef PDG_H
#define PDG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pdg_ctx pdg_ctx; /* opaque, owned by the library */

typedef enum {
    PDG_OK = 0,
    PDG_E_INVALID_ARGUMENT = 1, /* NULL pointer, bad size, dt == 0, lambda <= 0, tau < 0, nranks > nv,
                                   tau > 0 with a collision substep h of the scheme (or a pdg_collide /
                                   pdg_relax_from_w dt) where 2 tau + h <= 0 (eq collision_cn) */
    PDG_E_DIMENSION = 2,        /* dim not in {2, 3}                                   (SPEC DimensionOutOfRange) */
    PDG_E_DEGREE = 3,           /* degree not in the compiled set {1, 2, 3}            (SPEC DegreeOutOfRange) */
    PDG_E_VELOCITY_SET = 4,     /* velocities not the canonical +-lambda e_k per component set, or comp[] wrong */
    PDG_E_FLUX_MODEL = 5,       /* unknown flux kind, wrong m for it, or bad parameters */
    PDG_E_STATE_NOT_SET = 6,    /* pdg_step / pdg_transport / pdg_collide before a set_state call */
    PDG_E_NONPHYSICAL = 7,      /* (PDG_CHECK_STATE) rho <= 0 or non-finite value seen after the call;
                                   the state WAS advanced                              (SPEC NonpositiveDensity) */
    PDG_E_CUDA = 8,             /* a CUDA runtime error (launch or asynchronous fault) */
    PDG_E_NCCL = 9,             /* NCCL unavailable or a collective failed (nranks > 1) */
    PDG_E_BUFFER = 10,          /* a caller buffer is NULL or too small for pdg_sizes */
    PDG_E_UNSUPPORTED = 11      /* valid request outside what this build implements */
} pdg_status;

typedef enum {
    PDG_FLUX_LINEAR_ADVECTION = 0, /* m = 1:      q^k = a_k w;                      flux_params = a[dim] */
    PDG_FLUX_EULER = 1,            /* m = dim+2:  compressible Euler, w = (rho, rho u, E); flux_params = {gamma} */
    PDG_FLUX_ISOTHERMAL = 2,       /* m = dim+1:  w = (rho, rho u), p = c^2 rho;    flux_params = {c} */
    PDG_FLUX_LBM = 3               /* m = dim+1:  lattice-Boltzmann isothermal model (NEXT-2):
                                      w = P f with P = [1; v^T] (rho = sum f_i, rho u = sum f_i v_i),
                                      f^eq_i = w_i rho (1 + u.v_i/c^2 + (u.v_i)^2/(2c^4) - u.u/(2c^2));
                                      flux_params = {c, w_0, ..., w_{nv-1}} (n_flux_params = 1 + nv);
                                      the velocity set is any lattice with components in {0, +-lambda}:
                                      D2Q9 (nv = 9), D3Q15/D3Q19/D3Q27 (nv = 15/19/27) are compiled;
                                      comp[] is ignored (may be NULL) */
} pdg_flux;

typedef enum {
    PDG_SCHEME_M2 = 0,    /* T2(dt/2) C2(dt) T2(dt/2), the hot path */
    PDG_SCHEME_M2KIN = 1, /* T2(dt/4) C2(dt/2) T2(dt/2) C2(dt/2) T2(dt/4) */
    PDG_SCHEME_M4 = 2,    /* M2kin(g1 dt) M2kin(g2 dt) M2kin(g1 dt), g1 = 1/(2 - 2^(1/3)), g2 = 1 - 2 g1:
                             palindromic composition raising the order to 4; needs
                             2 tau + g2 dt/2 > 0 when tau > 0 (checked at pdg_query_sizes/pdg_create) */
    PDG_SCHEME_M2S = 3    /* T2(dt/2) S2(dt/2) C2(dt) S2(dt/2) T2(dt/2): the Strang scheme with the source
                             step (NEXT-3); needs a source (pdg_problem.source) */
} pdg_scheme;

typedef enum {
    PDG_SOURCE_NONE = 0,
    PDG_SOURCE_GRAVITY = 1  /* Euler with gravity, PDG_FLUX_LBM only: macroscopic source
                               s(w) = (0, rho G), source_params = G[dim] (e.g. (0, -g) in 2-D), lifted to
                               g_i = w_i v_i.(rho G)/c^2 (reading C24: P g = s); S2(h) = (I + h/2 G_h)
                               (I - h/2 G_h)^{-1} is exact in closed form, f <- f + h g(f) (one Picard
                               iteration) */
} pdg_source_kind;

typedef enum {
    PDG_DECOMP_VELOCITY = 0, /* rank r owns a contiguous block of velocities (sizes nv/G or nv/G + 1, the
                                first nv % G ranks one more) on the whole grid; one NCCL sum of the m
                                moment fields per collision (north star) */
    PDG_DECOMP_ZSLAB = 1     /* rank r owns the cell planes [r N/G, (r+1) N/G) of the slowest axis (z in 3-D,
                                y in 2-D) with every velocity; for sweeps along that axis a read-only
                                pre-pass computes each slab's zero-inflow outgoing carries (last cells
                                only), the exact slab inflows follow from an affine scan of those carries
                                (linear superposition of the carry recurrence; NCCL all-gather of carry
                                planes), and every slab is swept once from its exact inflows */
} pdg_decomposition;

/* pdg_problem.flags */
#define PDG_CHECK_STATE 0x1u  /* after each pdg_step, count nodes with rho <= 0 or non-finite f (one extra pass) */
#define PDG_SYNC_ERRORS 0x2u  /* synchronise the stream after every call and report asynchronous faults there */
#define PDG_NO_FUSION   0x4u  /* do not fuse step n's trailing T2(dt/2) with step n+1's leading one
                                 (results agree to rounding; the fused form is two sweeps in one pass, not the
                                 "collapsed" scheme of P:1173-1177) */
#define PDG_PROFILE     0x8u  /* bracket every kernel launch with CUDA events on the context stream (read with
                                 pdg_profile_read; not for use under CUDA-graph capture) */
#define PDG_ASYNC_HOST  0x10u /* host-pointer calls (pdg_set_state, pdg_set_equilibrium without wb, pdg_get_state,
                                 pdg_moments) return without synchronising: host buffers (pinned for true
                                 asynchrony) must stay valid and unmodified until pdg_synchronize.  Uploads for
                                 pdg_set_equilibrium are staged in an extra work region (pdg_sizes.work_bytes grows
                                 by 8 m nnodes_local bytes) and pdg_moments' download runs on a library copy
                                 stream, so the upload of step k+1's input overlaps the download of step k's
                                 result (PCIe is full duplex) */
#define PDG_NO_GRAPH    0x40u /* pdg_step launches its kernels directly instead of replaying a CUDA graph of its
                                 n-step launch sequence (same results; for measurement) */
#define PDG_NO_SMALL    0x80u /* small problems (f <= 64 KB, one rank, axis-aligned velocities) run pdg_step's
                                 operators with the general per-operator kernels instead of one CTA holding f in
                                 shared memory for up to 48 operators per launch (results agree to rounding:
                                 the x sweeps of the general path take a warp scan; for measurement and tests) */
#define PDG_NO_TMA      0x20u /* stage the line of the fused collision + x-sweep pass through registers instead of
                                 Tensor-Memory-Accelerator bulk copies (the variant for odd line lengths;
                                 same results; for measurement) */

/* kernel kinds reported by pdg_profile_read */
typedef enum {
    PDG_K_SWEEP_STRIDED = 0, /* T2 sweeps of velocities along y/z (one or two sweeps per pass) */
    PDG_K_SWEEP_X = 1,       /* T2 sweeps of velocities along x (warp-scan) */
    PDG_K_RELAX = 2,         /* collision fused with moments (nranks == 1) */
    PDG_K_PARTIAL = 3,       /* partial moments (nranks > 1, pdg_moments) */
    PDG_K_RELAX_W = 4,       /* collision from reduced moments (nranks > 1) */
    PDG_K_ALLREDUCE = 5,     /* NCCL sum of w */
    PDG_K_OTHER = 6,         /* initialisation / checks */
    PDG_K_RELAX_X = 7,       /* collision fused with moments and the following x-velocity sweep(s) */
    PDG_K_ZSLAB = 8,         /* z-slab carry pre-pass and scan (and the carry all-gather) */
    PDG_K_LATTICE = 9,       /* T2 sweeps of lattice velocities with >= 2 non-zero components (NEXT-2) */
    PDG_K_SMALL = 10,        /* small problems: a run of operators in one CTA with f in shared memory */
    PDG_NUM_KERNEL_KINDS = 11
} pdg_kernel_kind;

typedef struct {
    int32_t dim;                 /* D in {2, 3} */
    int64_t ncell[3];            /* cells per axis (x, y, z); ncell[d] = 1 for d >= dim */
    double lo[3], hi[3];         /* box [lo, hi] (affine cells) */
    int32_t degree;              /* p: (p+1)^D Gauss-Lobatto nodes per cell */
    int32_t m;                   /* number of conservative variables w */
    int32_t nv;                  /* number of velocities */
    const double *vel;           /* host, nv*3 (row i = v_i, unused components 0); copied */
    const int32_t *comp;         /* host, nv: P[c][i] = (comp[i] == c); copied */
    double lambda;               /* lattice speed, |v_i| = lambda */
    int32_t flux;                /* pdg_flux: the flux q(w) defining f^eq */
    const double *flux_params;   /* host, n_flux_params values (see pdg_flux); copied */
    int32_t n_flux_params;
    double tau;                  /* relaxation time; 0 => f <- 2 f^eq - f */
    double dt;                   /* time step of one palindromic step (may be negative) */
    int32_t scheme;              /* pdg_scheme */
    int32_t rank, nranks;        /* shard of this process (see pdg_decomposition) */
    const void *nccl_id;         /* 128-byte ncclUniqueId (identical on all ranks).  Non-NULL: the context
                                    owns an NCCL communicator and the collision takes the sharded path
                                    (partial moments, NCCL sum, relax) -- also with nranks == 1.
                                    NULL with nranks > 1 creates a communicator-less shard:
                                    pdg_collide/pdg_moments then return PDG_E_NCCL and the caller reduces
                                    w_dev itself between pdg_partial_moments and pdg_relax_from_w */
    void *cuda_stream;           /* cudaStream_t for every launch of this context */
    uint32_t flags;              /* PDG_CHECK_STATE | PDG_SYNC_ERRORS | PDG_NO_FUSION | PDG_PROFILE */
    int32_t decomposition;       /* pdg_decomposition: how nranks > 1 split the work */
    int32_t slabs_per_rank;      /* PDG_DECOMP_ZSLAB: sub-slabs per rank (>= 1; > 1 emulates more ranks
                                    on one GPU with the same arithmetic) */
    int32_t source;              /* pdg_source_kind (PDG_SOURCE_NONE: no source) */
    const double *source_params; /* host, n_source_params values (see pdg_source_kind); copied */
    int32_t n_source_params;
    /* Launch plan of the lattice sweeps (PDG_FLUX_LBM); zeros select the tuned
       defaults.  The results do not depend on them (tests force small CTAs and short chain segments
       so that the cross-CTA hand-overs and the segment halos run on small grids). */
    int32_t lattice_cta[2];      /* warps per CTA along x and along the pipe / batch axis (both >= 1,
                                    product <= 8); {0, 0}: default */
    int32_t lattice_segment;     /* chain-segment rows: 0 default, < 0 never segment, > 0 this length
                                    (used only where a halo bound exists) */
} pdg_problem;

typedef struct {
    size_t f_elems;        /* doubles in f_dev  = nv_local * nnodes_local */
    size_t fb_elems;       /* doubles in fb_dev = nv_local * plane_stride (x dim for PDG_FLUX_LBM) */
    size_t w_elems;        /* doubles in w_dev  = m * nnodes_local (moments / exchange / equilibrium init) */
    size_t work_bytes;     /* bytes of work_dev (device scratch: counters, z-slab carry planes and tables,
                              lattice ticket/progress/halo counters and tagged boundary-trace words, large
                              lattice block tables, the PDG_ASYNC_HOST upload staging); the lattice launch
                              plan (pdg_problem.lattice_cta / lattice_segment) changes it */
    int64_t nnodes;        /* nodes of the full grid */
    int64_t plane_stride;  /* doubles per velocity in fb */
    int32_t nv_local;      /* velocities owned by this rank */
    int32_t v_begin;       /* first owned velocity index */
    int64_t nnodes_local;  /* nodes owned by this rank (== nnodes unless PDG_DECOMP_ZSLAB) */
    int64_t cell_begin;    /* PDG_DECOMP_ZSLAB: first owned cell plane of the slowest axis (else 0) */
    int64_t cell_count;    /* PDG_DECOMP_ZSLAB: owned cell planes (else ncell of that axis) */
} pdg_sizes;

/* Validate *p and return the buffer sizes of this rank.  Host-only: needs no GPU.
 * Errors: PDG_E_INVALID_ARGUMENT, PDG_E_DIMENSION, PDG_E_DEGREE, PDG_E_VELOCITY_SET, PDG_E_FLUX_MODEL,
 * PDG_E_UNSUPPORTED (lattice sets other than D2Q9/D3Q15/D3Q19/D3Q27, lattice sets with
 * PDG_DECOMP_ZSLAB, a source with a non-LBM model). */
pdg_status pdg_query_sizes(const pdg_problem *p, pdg_sizes *out);

/* Create a context bound to caller-owned device buffers sized by pdg_query_sizes
 * (f_dev, fb_dev, w_dev, work_dev: 256-byte aligned device pointers on the current
 * device).  Precomputes the per-axis cell blocks (the KLU refactorisation of P:769-777
 * becomes a tiny precomputed inverse: dt and v are constant) and, for lattice sets, the
 * dense blocks of the scheme's steps; creates the library's own streams (one per lattice
 * velocity class, the PDG_ASYNC_HOST copy streams).  With nccl_id it also creates an NCCL
 * communicator (collective over all ranks).  work_dev's previous content is ignored: the
 * lattice trace-word region is zeroed on the context stream (every launch leaves it zeroed
 * again), the counters are reset before each launch that uses them.
 * Errors: as pdg_query_sizes, plus PDG_E_BUFFER, PDG_E_CUDA, PDG_E_NCCL. */
pdg_status pdg_create(const pdg_problem *p, double *f_dev, double *fb_dev, double *w_dev, void *work_dev,
                      pdg_ctx **out);

/* Load the kinetic state.  f: f_elems doubles in the canonical layout; fb:
 * fb_elems doubles (inflow planes, constant in time: P:183-184).
 * Either may be NULL to keep the bound buffer's content.  on_device != 0:
 * pointers are device memory, else host (copied on the context stream, then
 * the stream is synchronised before returning, unless PDG_ASYNC_HOST). */
pdg_status pdg_set_state(pdg_ctx *c, const double *f, const double *fb, int on_device);

/* Equilibrium initialisation (readings C12, C13): f_i = f^eq_i(w) at every node and
 * fb_i = f^eq_i(wb) on the inflow plane of velocity i.  w, wb: [m][nodes] (w_elems
 * doubles); wb == NULL means wb = w.  Host pointers are staged through w_dev (synchronous), or
 * with PDG_ASYNC_HOST and wb == NULL through the extra staging region (asynchronous). */
pdg_status pdg_set_equilibrium(pdg_ctx *c, const double *w, const double *wb, int on_device);

/* Copy the current f (f_elems doubles, canonical layout) out (checkpoint/readback). */
pdg_status pdg_get_state(pdg_ctx *c, double *f, int on_device);

/* Advance nsteps palindromic steps (scheme of pdg_problem; nsteps == 0 is a no-op).
 * Asynchronous on the context stream unless PDG_SYNC_ERRORS / PDG_CHECK_STATE (lattice classes
 * run on library streams forked from and joined back into the context stream).  For 2 <= nsteps
 * <= 1024 the launch sequence is captured once per step count into a CUDA graph and replayed (the
 * first call of a given count pays the capture; same launches, same results); not while PDG_PROFILE
 * events are active (pdg_profile_enable), with PDG_SYNC_ERRORS, PDG_NO_GRAPH, a communicator, or
 * while the caller's stream is being captured (then the kernels go into the caller's graph).
 * Capturable by the caller.  L2 use: when f fits in 70 % of the device's L2 the passes access it
 * with an evict-normal policy (it stays resident from one pass to the next), else evict-first
 * (streaming); the arithmetic, and so the result, does not depend on it.  Small problems (f of at
 * most 64 KB with padded rows, one rank, axis-aligned velocities, no PDG_NO_SMALL) run the step's
 * operators in one CTA holding f in shared memory, up to 48 operators per launch; the x sweeps then
 * carry sequentially instead of by the warp scan (results agree to rounding). */
pdg_status pdg_step(pdg_ctx *c, int64_t nsteps);

/* One transport operator T2(dtp) on every local velocity (rows a1/a3 of the hot path):
 * f <- (I + dtp/2 L_h)(I - dtp/2 L_h)^{-1} f with fictitious inflow cells f^b. */
pdg_status pdg_transport(pdg_ctx *c, double dtp);

/* One collision operator C2(dt) on every node (row a2): w = P f, f^eq(w),
 * f <- ((2 tau - dt) f + 2 dt f^eq)/(2 tau + dt)   (= 2 f^eq - f at tau = 0).
 * With nranks > 1: partial moments, NCCL sum, then relaxation of local velocities.
 * PDG_E_INVALID_ARGUMENT if tau > 0 and 2 tau + dt <= 0, or dt is not finite. */
pdg_status pdg_collide(pdg_ctx *c, double dt);

/* One source operator S2(h) on every node (NEXT-3): f <- f + h g(f) for the gravity
 * source (exact CN solution, see PDG_SOURCE_GRAVITY).  PDG_E_INVALID_ARGUMENT without a source.
 * With nranks > 1 the density comes from the reduced moments (partial moments, NCCL sum). */
pdg_status pdg_source(pdg_ctx *c, double h);

/* The two halves of the sharded collision (row a4), exposed for testing:
 * pdg_partial_moments writes w_dev = sum over LOCAL velocities of each component
 * (zeros for components without local velocities); pdg_relax_from_w applies C2(dt)
 * to the local velocities from the (already reduced) w_dev. */
pdg_status pdg_partial_moments(pdg_ctx *c);
pdg_status pdg_relax_from_w(pdg_ctx *c, double dt);

/* Moments w = P f of the full state ([m][nodes], w_elems doubles) into w (host or
 * device); with nranks > 1 the partial sums are reduced over ranks (every rank gets w).
 * With PDG_ASYNC_HOST a host download runs on the library copy stream (see the flag). */
pdg_status pdg_moments(pdg_ctx *c, double *w, int on_device);

/* Number of nodes with rho <= 0 or a non-finite f seen in the local state
 * (synchronising).  Component 0 of w is the density for the Euler/isothermal models. */
pdg_status pdg_check_state(pdg_ctx *c, int64_t *n_bad);

/* The precomputed 1-D cell block of the T2(dtp) sweep along `axis` (reading C18):
 * f_new = M f_old + g s_in, s_out = f_old[n-1] + f_new[n-1], nodes in flow order;
 * M: n*n row-major, g: n, beta = g[n-1].  Host outputs.  For inspection/pins. */
pdg_status pdg_cell_block(const pdg_ctx *c, int axis, double dtp, double *M, double *g, double *beta);

/* Carry tables of the exact z-slab decomposition (row e; P:779-797 domain decomposition,
 * DESIGN.md §8) along the slowest axis of problem *p, for npass consecutive T2(dtp) sweeps
 * (npass = 1 or 2) of a slab of `len` cells.  The line recurrence is affine, so a slab swept
 * with zero inflow needs, once its true inflow carries S1 (pass 1) and S2 (pass 2) are known:
 *   f_l += Q_l S_last + (npass == 2 ? P_l S1 : 0),   l = 0 .. len-1 (cells in flow order,
 *          S_last = S2 for npass 2, S1 for npass 1; nodes of cell l in flow order),
 *   outgoing carries: c1 = A1 + B S1,  c2 = A2 + B S2 + C S1   (A = the zero-inflow carries).
 * Outputs (host): P, Q: [len][p+1] row-major; B = beta^len; C; leff = cells after which every
 * |P_l|, |Q_l| < 2^-64 (a slab's inflow no longer moves its values in fp64, reading C26).  (The
 * library itself uses B and C for the carry scan and sweeps each slab from its exact inflows.)
 * Host-only (no GPU); computed in long double and rounded once.
 * Errors: those of pdg_query_sizes; PDG_E_INVALID_ARGUMENT for npass, len < 1, NULL outputs. */
pdg_status pdg_zslab_table(const pdg_problem *p, double dtp, int npass, int64_t len, double *P, double *Q,
                           double *B, double *C, int32_t *leff);

/* Block until all work enqueued by this context has finished (including PDG_ASYNC_HOST copies);
 * reports asynchronous faults. */
pdg_status pdg_synchronize(pdg_ctx *c);

/* Destroy the context (NULL-safe); destroys the NCCL communicator if any. Does not free caller buffers. */
void pdg_destroy(pdg_ctx *c);

/* Write a fresh 128-byte ncclUniqueId into out (rank 0 calls it and broadcasts).
 * Errors: PDG_E_NCCL if libnccl.so.2 cannot be loaded. */
pdg_status pdg_nccl_unique_id(void *out);

/* Static description of a status code. */
const char *pdg_status_string(pdg_status s);

/* Detail of the last error reported on the calling thread ("" if none). */
const char *pdg_last_error(void);

/* (PDG_PROFILE) Synchronise, then return per kernel kind the summed device time in ms,
 * the number of launches and the algorithmic bytes moved since the last read, and reset.
 * Each array has PDG_NUM_KERNEL_KINDS entries (any may be NULL).  Algorithmic bytes =
 * one fp64 read + one write of every value a launch updates, plus its side inputs
 * (inflow planes, moments), i.e. the traffic of a perfect single pass. */
pdg_status pdg_profile_read(pdg_ctx *c, double *ms, int64_t *launches, double *alg_bytes);

/* (PDG_PROFILE) Pause (on = 0) or resume (on != 0) the per-launch events; while paused the context
 * runs as without PDG_PROFILE (pdg_step may replay its CUDA graph).  PDG_E_INVALID_ARGUMENT if the
 * context was created without PDG_PROFILE. */
pdg_status pdg_profile_enable(pdg_ctx *c, int on);

/* Library version string ("pdg-b200 <version> sm_100a"). */
const char *pdg_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PDG_H */
