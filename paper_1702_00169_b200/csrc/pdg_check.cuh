// PDG_CHECKED build (`python -m paper_1702_00169_b200.build --checked` -> libpdg_checked.so, selected
// by PDG_CHECKED=1 in the binding): every global load and store of the sweep, relaxation, z-slab
// and lattice kernels checks its element index against the bound of the buffer it addresses, and
// every cross-CTA spin wait is bounded.  A violation prints the site and traps; the calling
// pdg_* function then returns PDG_E_CUDA.  compute-sanitizer is not available on the GPU pool,
// so this build is the memory-safety check.  The default build compiles every
// check to nothing.
#pragma once
#include <cstdint>
#include <cstdio>

#ifdef PDG_CHECKED
#define PDG_DCHECK(cond, what, a, b)                                                                 \
    do {                                                                                             \
        if (!(cond)) {                                                                               \
            printf("PDG_CHECKED %s:%d %s: %lld vs %lld (block %d thread %d)\n", __FILE__, __LINE__,   \
                   what, (long long)(a), (long long)(b), (int)blockIdx.x, (int)threadIdx.x);          \
            __trap();                                                                                \
        }                                                                                            \
    } while (0)
// polls of a cross-CTA wait before it is declared a deadlock (each poll sleeps >= 16 ns)
#define PDG_SPIN_LIMIT (1ll << 27)
#define PDG_SPIN_DECL(cnt) long long cnt = 0
#define PDG_SPIN_TICK(cnt, what) PDG_DCHECK(++(cnt) < PDG_SPIN_LIMIT, what, cnt, PDG_SPIN_LIMIT)
#else
#define PDG_SPIN_DECL(cnt) \
    do {                   \
    } while (0)
#define PDG_DCHECK(cond, what, a, b) \
    do {                             \
    } while (0)
#define PDG_SPIN_TICK(cnt, what) \
    do {                         \
    } while (0)
#endif

// element index `idx` of a buffer of `n` elements
#define PDG_CHECK_IDX(idx, n, what) PDG_DCHECK((int64_t)(idx) >= 0 && (int64_t)(idx) < (int64_t)(n), what, idx, n)
