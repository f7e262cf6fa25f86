// simba_device.cuh -- device-side building blocks of the SIMBA hot path on sm_100a.
//
// Everything here is integer ALU work: no tensor cores, no TMA (there is no
// contraction and ~0 HBM traffic per candidate).  Reference
// behaviour each function reproduces is cited as file:line under
// /root/reference/pkg/src/mbasynth.
#pragma once
#include <stdint.h>

#include "../../include/simba.h"

namespace simba {

constexpr int MAXS = SIMBA_MAX_SIZE;
constexpr int MAXSO = 4;  // outer-spine segments held in registers
constexpr int MAXSL = 2;  // left-spine segments held in registers
constexpr unsigned FULL = 0xffffffffu;

// Path statistics for diagnostics builds (-DSIMBA_STATS): calls and
// candidates per sweep path, read back with simba_ctx_stats.
enum : int {
    ST_RF_FOLD = 0, ST_RF_GEN, ST_RF_ROW, ST_CF_FOLD, ST_CF_GEN,
    ST_CYC_OUTER, ST_CYC_X, ST_CYC_TILE,  // (calls, SM cycles) of the odometer steps and tile calls
    ST_DIRECT,
    ST_PH_PLAN, ST_PH_EXEC, ST_PH_VERIFY,  // (phases, CTA cycles) of each phase (thread 0)
    ST_W_PLAN, ST_W_EXEC,                 // (warp phases, warp busy cycles) inside plan / exec
    ST_ROW_NONE,                          // one-row tiles of a P-less region (a unary node above L2)
    ST_GEN_NT1, ST_GEN_NT2, ST_GEN_NT3,   // GEN candidates by segments per candidate (3: 3 or more)
    ST_GEN_ARITH,                         // GEN candidates of an arithmetic P
    ST_GEN_RES_AFF, ST_GEN_RES_BW,        // GEN candidates whose residual segments are all affine / all bitwise
    ST_N
};
#ifdef SIMBA_STATS
#define SIMBA_STAT(p, i, cands)                                                         \
    do {                                                                                \
        if ((threadIdx.x & 31) == 0) {                                                  \
            atomicAdd(&(p).stats[2 * (i)], 1ull);                                       \
            atomicAdd(&(p).stats[2 * (i) + 1], (unsigned long long)(cands));            \
        }                                                                               \
    } while (0)
#define SIMBA_CYC_BEGIN(v) const long long v = clock64()
#define SIMBA_CYC_END(p, i, v) SIMBA_STAT(p, i, clock64() - (v))
#else
#define SIMBA_STAT(p, i, cands) \
    do {                        \
    } while (0)
#define SIMBA_CYC_BEGIN(v) \
    do {                   \
    } while (0)
#define SIMBA_CYC_END(p, i, v) \
    do {                       \
    } while (0)
#endif

// Operator slots in the fixed enumeration order (expr.py:22-32).
enum : int { OP_NOT = 0, OP_AND, OP_OR, OP_XOR, OP_NEG, OP_ADD, OP_SUB, OP_MUL, OP_NONE = 8 };

// Decoder tables (codec.py:60-87) plus Granlund-Montgomery reciprocals of the
// per-size totals, so that the divmod of codec.py:123-124 costs one
// multiply-high instead of a software 64-bit divide.  Staged in shared memory.
struct __align__(16) Tabs {
    uint64_t T[MAXS + 1];                 // T[s][8]
    uint64_t m64[MAXS + 1];               // 64-bit magic for division by T[s]
    uint32_t m32[MAXS + 1];               // 32-bit magic (valid when T[s] < 2^32)
    uint32_t toff[MAXS + 1];              // value-table offset of size s (s <= RG)
    uint8_t sh1[MAXS + 1];
    uint8_t sh2[MAXS + 1];
    uint8_t pad_[6];
    uint64_t slot_cum[MAXS + 1][8];       // slot_cums[s][op]  (codec.py:69-79)
    uint64_t split_cum[MAXS + 1][MAXS];   // split_cums[s][j]  (codec.py:80-85)
};

struct KParams {
    const Tabs *tabs;        // global copy of the tables
    const void *gtbl;        // [E][gtbl_len] values of every subtree of size <= RG (global)
    uint32_t gtbl_len;       // entries of sizes <= RG per example (global)
    int k, n, s, R0, RG, E;
    int r0_up;               // levels >= r0_up use R0 + 1
    uint32_t guide;          // claim ~ remaining / (warps * guide)
    uint64_t desc_cands;     // candidates per tile descriptor (at most)
    uint64_t split_min;      // late splitting: pieces with >= split_min ranks left
    uint64_t phase_guide;    // phase budget ~ remaining / (warps * phase_guide); 0: none
    int level_guide;         // claims and phase budgets guided by the remaining ranks of the frontier's
                             // level, not of the launch (fused single-shard searches)
    int mode;                // SIMBA_MODE_*
    int shuffled;
    uint64_t mask;
    uint64_t lo, hi, chunk_len, shard, nshards, stop_above;
    uint64_t spc;            // chunks per super-chunk (sharding unit)
    uint64_t nvirt;          // chunks owned by this shard (virtual numbering)
    uint32_t lvl_off;        // shared-memory offset of the per-warp level stacks
    uint64_t offset, block_total;  // shuffled (RTid) mapping, codec.py:210-236
    uint64_t budget_ns;
    int stage_examples;      // examples staged in shared memory
    unsigned long long *ctr;      // chunk claim counter
    unsigned long long *best;     // minimum satisfying rank
    unsigned long long *count;    // satisfying candidates
    unsigned long long *visited;  // candidates evaluated
    unsigned long long *units;    // [0] units decoded, [1] units on the per-rank path
    unsigned int *flags;
    unsigned long long *planned;  // candidates queued so far (all CTAs): phase budgets
    unsigned long long *dropped;  // lowest rank of a run dropped by the time budget
    unsigned long long *xbest;    // shared minimum of a sharded search (another GPU's memory over
                                  // NVLink, or this GPU's); null: none.  Hits are published to it,
                                  // and claims and phases fold it into *best
    unsigned long long *pool;     // returned piece ranges (late splitting)          // bit 0: stopped by the time budget
    unsigned long long *stats;    // [2*path] calls, [2*path+1] candidates (SIMBA_STATS builds)
    void *queue;                  // tile descriptors, qcap per CTA (plan/execute phases)
    uint32_t qcap;
    uint32_t dpw;                 // descriptors per warp and phase (<= kDescPerWarp)
    uint32_t dpw_late;            // ... once 3/4 of the chunks are claimed (0: dpw throughout)
    uint32_t ps_off;              // shared-memory offset of the CTA's queue bookkeeping
    unsigned long long *vq;       // deferred verification queue, vqcap ranks per CTA (null: verify inline)
    uint32_t vqcap;
    // levels [s_lo, s_hi] of one launch in a virtual rank space: level s holds
    // virtual ranks [vbase[s], vbase[s + 1]); lo/hi/best/stop_above are virtual
    int s_lo, s_hi;
    uint64_t fine_row;  // partial rows of at least this many columns at R0 + 1 levels are planned at R0 (0: off)
    int absorb;         // Odometer::absorb (SIMBA_ABSORB)
    int shared_cap;     // planning stops when the CTA queue is full (else at an equal share per warp)
    const unsigned long long *vbase;  // [MAXS + 2] (global; kept out of the parameter block)
    unsigned long long *lvl;      // per level: [s] count, [MAXS+1+s] visited, [2*(MAXS+1)+s] first rank
};

// ---------------------------------------------------------------------------
// integer helpers
// ---------------------------------------------------------------------------

// floor(n / T[sz]) by the Granlund-Montgomery round-down method; host computes
// the magic (simba.cu: gm_magic).  Exact for every n < 2^64, T[sz] >= 1.
__device__ __forceinline__ uint64_t div_T(const Tabs *t, int sz, uint64_t n)
{
    const uint64_t d = t->T[sz];
    if (((n | d) >> 32) == 0) {
        const uint32_t n32 = (uint32_t)n;
        const uint32_t hi = __umulhi(n32, t->m32[sz]);
        return (hi + ((n32 - hi) >> t->sh1[sz])) >> t->sh2[sz];
    }
    const uint64_t hi = __umul64hi(n, t->m64[sz]);
    return (hi + ((n - hi) >> t->sh1[sz])) >> t->sh2[sz];
}

// Operator search by linear scan of the slot prefix sums (codec.py:108-113).
__device__ __forceinline__ int find_slot(const Tabs *t, int sz, uint64_t &r)
{
    const uint64_t *c = t->slot_cum[sz];
    int op = 0;
    while (r >= c[op])
        ++op;
    if (op)
        r -= c[op - 1];
    return op;
}

// Left-subtree size by linear scan of the split prefix sums (codec.py:118-122).
__device__ __forceinline__ int find_split(const Tabs *t, int sz, uint64_t &r)
{
    const uint64_t *p = t->split_cum[sz];
    int j = 1;
    while (r >= p[j])
        ++j;
    r -= p[j - 1];
    return j;
}

// The decoder tables sit at offset 0 of the dynamic shared memory of every
// scan kernel; reading them through this symbol lets the compiler emit LDS
// (a pointer passed through a non-inlined call degrades to generic loads).
__device__ __forceinline__ const Tabs *stabs()
{
    extern __shared__ __align__(16) unsigned char smem_tabs_[];
    return reinterpret_cast<const Tabs *>(smem_tabs_);
}

__device__ __forceinline__ uint64_t globaltimer_ns()
{
    uint64_t v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    return v;
}

// ---------------------------------------------------------------------------
// reference-exact unrank and evaluation (one candidate per lane)
// ---------------------------------------------------------------------------

// codec.Decoder.decode_into (codec.py:89-133): same LIFO agenda, the left
// child continued in place, the right frame pushed, identical divmod order.
// Tokens: variable index >= 0, operator -(slot+1) (expr.py:66-85).
__device__ __noinline__ void decode_tokens(const Tabs *t, uint64_t rank, int size, int8_t *buf)
{
    int8_t apos[MAXS], asize[MAXS];
    uint64_t arank[MAXS];
    int depth = 1;
    apos[0] = 0;
    asize[0] = (int8_t)size;
    arank[0] = rank;
    while (depth) {
        --depth;
        int pos = apos[depth];
        int sz = asize[depth];
        uint64_t r = arank[depth];
        while (sz > 1) {
            const int op = find_slot(t, sz, r);
            buf[pos + sz - 1] = (int8_t)(-(op + 1));
            if (op == OP_NOT || op == OP_NEG) {
                --sz;
                continue;
            }
            const int j = find_split(t, sz, r);
            const int rsz = sz - 1 - j;
            const uint64_t q = div_T(t, rsz, r);
            apos[depth] = (int8_t)(pos + j);
            asize[depth] = (int8_t)rsz;
            arank[depth] = r - q * t->T[rsz];
            ++depth;
            sz = j;
            r = q;
        }
        if (sz == 1)
            buf[pos] = (int8_t)r;
    }
}

// Binary operator with the reference's operand order: left OP right
// (expr.py:176-197).  Values are computed modulo 2^bits(W); comparison against
// an output happens under the spec mask, which is exact because truncation
// mod 2^w commutes with every operator of the grammar.
template <class W>
__device__ __forceinline__ W apply_bin(int op, W a, W b)
{
    switch (op) {
    case OP_AND: return a & b;
    case OP_OR: return a | b;
    case OP_XOR: return a ^ b;
    case OP_ADD: return a + b;
    case OP_SUB: return a - b;
    default: return a * b; // OP_MUL
    }
}

template <class W, int OP>
__device__ __forceinline__ W apply_bin_t(W a, W b)
{
    if constexpr (OP == OP_AND) return a & b;
    else if constexpr (OP == OP_OR) return a | b;
    else if constexpr (OP == OP_XOR) return a ^ b;
    else if constexpr (OP == OP_ADD) return a + b;
    else if constexpr (OP == OP_SUB) return a - b;
    else if constexpr (OP == OP_MUL) return a * b;
    else return b; // OP_NONE: the unit's value is the super-leaf itself
}

// expr.eval_tokens (expr.py:157-198) over one example; x points at its k inputs.
template <class W, class TX>
__device__ __noinline__ W eval_rpn(const int8_t *buf, int size, const TX *x)
{
    W st[MAXS / 2 + 2];
    int sp = 0;
    for (int i = 0; i < size; ++i) {
        const int tk = buf[i];
        if (tk >= 0) {
            st[sp++] = (W)x[tk];
        } else if (tk == -1) {
            st[sp - 1] = ~st[sp - 1];
        } else if (tk == -5) {
            st[sp - 1] = (W)0 - st[sp - 1];
        } else {
            --sp;
            st[sp - 1] = apply_bin<W>(-tk - 1, st[sp - 1], st[sp]);
        }
    }
    return st[0];
}

// ---------------------------------------------------------------------------
// spine functions: every grammar operator with one fixed operand is
//     v -> a * ((v & m) ^ x) + b      (one LOP3 + one IMAD)
// AND s: m=s;  OR s: m=~s, x=s;  XOR s: x=s;  NOT: x=~0;
// ADD s: b=s;  SUB s (s - v): a=-1, b=s;  MUL s: a=s;  NEG: a=-1.
// Bitwise maps compose into one (m, x) pair and affine maps into one (a, b)
// pair, so a whole chain of fixed-operand ancestors collapses into a few
// segments evaluated branch-free and warp-uniformly.
// ---------------------------------------------------------------------------

template <class W>
struct __align__(16) Seg {
    W m, x, a, b;
};

template <class W>
__device__ __forceinline__ Seg<W> seg_identity()
{
    return Seg<W>{(W)~(W)0, (W)0, (W)1, (W)0};
}

template <class W>
__device__ __forceinline__ W seg_apply(const Seg<W> &s, W v)
{
    return s.a * ((v & s.m) ^ s.x) + s.b;
}

// Builder in walk order (outermost ancestor first).  A new function is always
// applied BEFORE the ones already collected (it is deeper in the tree).  The
// merge decisions depend only on the operator sequence (never on values), so
// every lane -- whatever example it evaluates -- builds the same structure.
template <class W, int CAP>
struct SegList {
    Seg<W> done[CAP];
    Seg<W> cur;
    int nd;
    bool has, cur_bw, ovf;

    __device__ __forceinline__ void init()
    {
        nd = 0;
        has = false;
        cur_bw = false;
        ovf = false;
    }
    __device__ __forceinline__ void start(W m, W x, W a, W b, bool bw)
    {
        if (has) {
            if (nd >= CAP - 1)
                ovf = true;
            else
                done[nd++] = cur;
        }
        cur = Seg<W>{m, x, a, b};
        has = true;
        cur_bw = bw;
    }
    __device__ __forceinline__ void bitwise(W m, W x)
    {
        if (!has) {
            start(m, x, (W)1, (W)0, true);
            return;
        }
        cur.x = (x & cur.m) ^ cur.x;  // (((v&m)^x) & M) ^ X = (v & (m&M)) ^ ((x&M)^X)
        cur.m = m & cur.m;
        cur_bw = true;
    }
    __device__ __forceinline__ void affine(W a, W b)
    {
        if (!has || cur_bw) {
            start((W)~(W)0, (W)0, a, b, false);
            return;
        }
        cur.b = cur.a * b + cur.b;  // A*(a v + b) + B
        cur.a = cur.a * a;
    }
    __device__ __forceinline__ void unary(int op)
    {
        if (op == OP_NOT)
            bitwise((W)~(W)0, (W)~(W)0);
        else
            affine((W)~(W)0, (W)0);  // NEG: -v
    }
    // ancestor `op` whose left child has value s; v is its right child
    __device__ __forceinline__ void binary_left_fixed(int op, W s)
    {
        switch (op) {
        case OP_AND: bitwise(s, (W)0); break;
        case OP_OR: bitwise((W)~s, s); break;
        case OP_XOR: bitwise((W)~(W)0, s); break;
        case OP_ADD: affine((W)1, s); break;
        case OP_SUB: affine((W)~(W)0, s); break;
        default: affine(s, (W)0); break;  // MUL
        }
    }
    // application order: innermost first; unused slots are identities
    template <int OUT>
    __device__ __forceinline__ void finalize(Seg<W> (&app)[OUT]) const
    {
#pragma unroll
        for (int i = 0; i < OUT; ++i) {
            Seg<W> v = seg_identity<W>();
            if (has) {
                if (i == 0)
                    v = cur;
                else if (i <= nd)
                    v = done[nd - i];
            }
            app[i] = v;
        }
    }
};

template <class W, int N>
__device__ __forceinline__ W segs_apply(const Seg<W> (&s)[N], W v)
{
#pragma unroll
    for (int i = 0; i < N; ++i)
        v = seg_apply(s[i], v);
    return v;
}

// ---------------------------------------------------------------------------
// subtree value with super-leaf cut-off
// ---------------------------------------------------------------------------

// Value of the size-sz expression of rank r on this lane's example: unrank as
// codec.py:89-133 but stop at subtrees of size <= R0 (the cut-off argument),
// whose values come from the per-spec value table (tbl_e[toff[size] + rank]).  Post-order folding on
// an explicit frame stack; control flow depends on (sz, r) only.
template <class W>
__device__ __noinline__ W eval_subtree(const W *tbl_e, int R0, int sz, uint64_t r)
{
    const Tabs *t = stabs();
    int8_t fop[MAXS], fstate[MAXS], frsz[MAXS];
    uint64_t frr[MAXS];
    W fval[MAXS];
    int depth = 0;
    W v;
    for (;;) {
        while (sz > R0) {
            const int op = find_slot(t, sz, r);
            if (op == OP_NOT || op == OP_NEG) {
                fop[depth] = (int8_t)op;
                fstate[depth] = 0;
                ++depth;
                --sz;
                continue;
            }
            const int j = find_split(t, sz, r);
            const int rsz = sz - 1 - j;
            const uint64_t q = div_T(t, rsz, r);
            fop[depth] = (int8_t)op;
            fstate[depth] = 1;
            frsz[depth] = (int8_t)rsz;
            frr[depth] = r - q * t->T[rsz];
            ++depth;
            sz = j;
            r = q;
        }
        v = tbl_e[t->toff[sz] + (uint32_t)r];
        for (;;) {
            if (depth == 0)
                return v;
            const int d = depth - 1;
            if (fstate[d] == 0) {
                v = (fop[d] == OP_NOT) ? (W)~v : (W)((W)0 - v);
                --depth;
            } else if (fstate[d] == 1) {
                fval[d] = v;
                fstate[d] = 2;
                sz = frsz[d];
                r = frr[d];
                break;
            } else {
                v = apply_bin<W>(fop[d], fval[d], v);
                --depth;
            }
        }
    }
}
// ---------------------------------------------------------------------------
// units and the odometer
// ---------------------------------------------------------------------------
//
// Rank order is lexicographic over the pre-order decisions of codec.py's
// unrank, with every subtree of size <= R0 ("super-leaf") one digit.  The
// last super-leaf L2 (size sz2, digit d2 < R2 = T[sz2]) always sits at the
// end of the root's right spine; the previous digit is the last super-leaf L1
// of the left child X of L2's parent P (digit d1 < R1 = T[sz1]).  All ranks
// that differ only in (d1, d2) are contiguous, [base, base + R1*R2), and share
// everything else -- a "unit":
//     value = OUTER( P( LEFT(tbl[sz1][d1]), tbl[sz2][d2] ) )
// OUTER / LEFT are the fixed-operand ancestor chains as segments.
//
// The odometer keeps the decoded path as two level stacks in per-warp shared
// memory: the outer spine (root .. above P, ranks n) and X's right spine
// (ranks q of X, where n = pb + q*R2 + d2 inside P's split block).  A level
// stays valid while the scan position is below its region end, so moving to
// the next unit re-decodes only the levels that changed (usually one),
// instead of the whole path from the root.

constexpr int MAXLV = MAXS;

template <class W>
struct Unit {
    uint64_t base;
    uint32_t R1, R2, d1, d2, off1, off2;
    int pop, nso, nsl;
    bool ovf;
    Seg<W> so[MAXSO];
    Seg<W> sl[MAXSL];
};

// per-warp level stack in shared memory (uniform fields written by lane 0,
// sibling values per example written by lanes 0..E-1)
template <class W, int E>
struct LevelStack {
    uint64_t end[MAXLV];   // region end of the level's decision (n- or q-space)
    int8_t op[MAXLV];
    int8_t csz[MAXLV];     // size of the child continuing the spine
    int8_t pad_[16 - (2 * MAXLV) % 16];
    W sib[MAXLV][E];       // left sibling value per example (binary levels)
};

// per-example chain segments of the current unit, for the rare multi-example
// hit refinement (lane e writes example e's segments)
template <class W, int E>
struct SegStash {
    Seg<W> so[E][MAXSO];
    Seg<W> sl[E][MAXSL];
};

// per-warp tile buffer: per-row (RF) or per-column (CF) test parameters
#ifndef SIMBA_TILE_BUF
#define SIMBA_TILE_BUF 128
#endif
constexpr int TILE_BUF = SIMBA_TILE_BUF;
static_assert(TILE_BUF % 32 == 0, "rows are produced 32 per step");

template <class W>
struct __align__(2 * sizeof(W)) TPair {
    W m, c;
};

// Per-P-block tile description: the outer chain folded into a masked
// compare ((v & tm) ^ tc) == 0 plus the residual (unfolded) inner segments.
template <class W>
struct TileArgs {
    W tm, tc;
    int nres;
    bool fold;  // P folds too: one LOP3 per candidate
    Seg<W> res[MAXSO];
};

// Tile descriptor written by the planner (odometer) phase and consumed by the
// execution phase of unit_kernel: everything a tile needs, so execution never
// touches the odometer.  The per-example chains (E > 1) ride along for the
// hit refinement.
template <class W, int E>
struct DescStash {
    SegStash<W, E> s;
};
template <class W>
struct DescStash<W, 1> {
};

template <class W, int E>
struct __align__(16) TileDesc {
    TileArgs<W> ta;        // folded outer test + residual chain (example 0)
    Seg<W> sl[MAXSL];      // example 0's LEFT chain of the X unit
    uint64_t ubase, row0, nrows, R1p;
    uint32_t R2, off2, clo, chi, off1, offy;
    int8_t pop, kind, nt, aff, x2d, pxop, sz1, szy;
    int32_t s;             // expression size (level) of the tile
    DescStash<W, E> st;
};

template <class W, int E>
struct WarpLevels {
    LevelStack<W, E> outer;
    LevelStack<W, E> xs;
    SegStash<W, E> stash;
    Seg<W> tbuf[TILE_BUF];  // per-row / per-column segments, or (m, c) pairs
    TileArgs<W> tac;        // folded outer chain of odometer generation tac_gen
    Seg<W> sl0[MAXSL];      // example 0's LEFT chain of the current X unit
    uint32_t tac_gen;
    int cur_s;              // level of the tile being executed (hit path)
};

#ifndef SIMBA_ABSORB_MAX
#define SIMBA_ABSORB_MAX 1  // absorbed right children: sizes R0 + 1 .. R0 + SIMBA_ABSORB_MAX (2: sweep 19.5 vs 18.1 ms)
#endif

template <class W, int E>
struct Odometer {
    WarpLevels<W, E> *L;   // this warp's shared-memory levels
    const W *gt_e;         // this lane's example: values of all subtrees of size <= RG
    int R0, RG, s, lane, ex;
    // outer state
    int no;                // valid outer levels
    bool have_outer;
    int pop, pj, prsz;
    uint64_t pb, pend;     // P split block [pb, pend) (or L2 region when pop == NONE)
    // X state
    int nx;
    bool have_x;
    int sz1;               // size of L1 (the last digit of X)
    bool x2d;              // X's last node N_X has both children <= RG: digits (dy, d1')
    int pxop, szy;         // N_X's operator and left-child size (x2d)
    uint64_t qb, qend;     // X-unit region in q-space [qb, qend)
    Seg<W> so[MAXSO], sl[MAXSL];
    int nso, nsl;
    bool so0_bw;           // innermost outer segment has a bitwise part
    uint32_t gen;          // bumped whenever the outer chain (so) is recomposed
    bool ovf_o, ovf_l;
    uint64_t phase_budget, phase_cands;  // candidates the warp may plan / has planned in this phase
    uint64_t fine_end;     // != 0: planning a partial R0+1 row at R0 until this virtual rank
    bool absorb;           // a binary node whose right child (size R0+1) starts with NOT/NEG is P
    int dpw_now;           // descriptors this warp may queue in the current phase
    unsigned int qbuf;     // the queue buffer this warp plans into
    int emit_max;          // 0 once the phase budget ended this warp's planning (shared-cap mode)
    // planner resume point inside a 2-D row group (queue filled mid-group)
    bool rs_valid;
    uint32_t rs_c;
    uint64_t rs_n;

    __device__ __forceinline__ void reset()
    {
        no = 0;
        nx = 0;
        have_outer = false;
        have_x = false;
        rs_valid = false;
    }

    __device__ __forceinline__ W sib_value(int j, uint64_t q) const
    {
        const Tabs *t = stabs();
        if (j <= RG)
            return gt_e[t->toff[j] + (uint32_t)q];
        return eval_subtree<W>(gt_e, RG, j, q);
    }

    template <int CAP>
    __device__ __forceinline__ void compose(const LevelStack<W, E> &st, int nlev, Seg<W> (&out)[CAP], int &nseg,
                                            bool &ovf, bool &bw0) const
    {
        SegList<W, CAP> sgl;
        sgl.init();
        for (int i = 0; i < nlev; ++i) {
            const int op = st.op[i];
            if (op == OP_NOT || op == OP_NEG)
                sgl.unary(op);
            else
                sgl.binary_left_fixed(op, st.sib[i][ex]);
        }
        sgl.finalize(out);
        nseg = sgl.has ? sgl.nd + 1 : 0;
        ovf = sgl.ovf;
        bw0 = sgl.has && sgl.cur_bw;
    }

    // Walk a right spine from (sz, r) at region base `rb` (same space as the
    // stack's ends) pushing levels, until the continuing child has size <= R0
    // or (outer stack only) it is P's super-leaf right child.  Returns the
    // final (sz, r); for the outer walk sets pop/pj/prsz when P is found.
    __device__ __forceinline__ void push_level(LevelStack<W, E> &st, int i, int op, int csz, uint64_t end, W sib)
    {
        if (lane == 0) {
            st.end[i] = end;
            st.op[i] = (int8_t)op;
            st.csz[i] = (int8_t)csz;
        }
        if (lane < E)
            st.sib[i][lane] = sib;
    }

    __device__ __forceinline__ void decode_outer(uint64_t n)
    {
        const Tabs *t = stabs();
        LevelStack<W, E> &st = L->outer;
        bool changed = !have_outer;
        if (have_outer) {
            while (no > 0 && n >= st.end[no - 1]) {
                --no;
                changed = true;
            }
        } else {
            no = 0;
        }
        int sz = (no == 0) ? s : st.csz[no - 1];
        uint64_t rb = (no == 0) ? 0 : st.end[no - 1] - t->T[sz];
        uint64_t r = n - rb;
        __syncwarp();  // every lane has read the stack before lane 0 pushes over it
        pop = OP_NONE;
        while (sz > R0) {
            const int op = find_slot(t, sz, r);
            if (op == OP_NOT || op == OP_NEG) {
                // child region = the whole operator block: [n - r, n - r + T[sz-1])
                push_level(st, no++, op, sz - 1, n - r + t->T[sz - 1], (W)0);
                changed = true;
                --sz;
                continue;
            }
            const int j = find_split(t, sz, r);
            const int rsz = sz - 1 - j;
            const uint64_t q = div_T(t, rsz, r);
            const uint64_t rr = r - q * t->T[rsz];
            // A right child whose own walk would pass only NOT/NEG nodes on its way
            // down to size <= R0 (NOT(z), NEG(NOT(z)), ...) ends with no P: every X
            // row of this node becomes a one-row region (tile_row1, one G load per
            // candidate).  Take this node as P instead, with rows of T[rsz]
            // columns from the value table (rsz <= R0 + SIMBA_ABSORB_MAX, <= RG):
            // the same ranks, tiled 2-D.
            bool take = rsz <= R0;
            if (!take && absorb && rsz <= R0 + SIMBA_ABSORB_MAX && rsz <= RG) {
                uint64_t r2 = rr;
                int sz2 = rsz;
                take = true;
                while (sz2 > R0) {
                    const int op2 = find_slot(t, sz2, r2);
                    if (op2 == OP_NOT || op2 == OP_NEG) {
                        --sz2;  // r2 is now the rank inside the unary's child
                        continue;
                    }
                    take = false;  // a binary node: the walk finds a P (or goes on) below
                    break;
                }
            }
            if (take) {
                pop = op;
                pj = j;
                prsz = rsz;
                pb = n - r;
                pend = pb + t->T[j] * t->T[rsz];
                break;
            }
            const W sv = sib_value(j, q);
            push_level(st, no++, op, rsz, n - rr + t->T[rsz], sv);
            changed = true;
            sz = rsz;
            r = rr;
        }
        if (pop == OP_NONE) {
            prsz = sz;  // L2 = this node
            pb = n - r;
            pend = pb + t->T[sz];
        }
        __syncwarp();
        if (changed) {  // sibling P blocks keep the outer chain
            compose<MAXSO>(st, no, so, nso, ovf_o, so0_bw);
            ++gen;
        }
        have_outer = true;
        have_x = false;
        nx = 0;
    }

    __device__ __forceinline__ void decode_x(uint64_t q)
    {
        const Tabs *t = stabs();
        LevelStack<W, E> &st = L->xs;
        if (pj <= RG) {
            sz1 = pj;
            x2d = false;
            qb = 0;
            qend = t->T[pj];
            nx = 0;
        } else {
            if (have_x) {
                while (nx > 0 && q >= st.end[nx - 1])
                    --nx;
            } else {
                nx = 0;
            }
            int sz = (nx == 0) ? pj : st.csz[nx - 1];
            const uint64_t rb = (nx == 0) ? 0 : st.end[nx - 1] - t->T[sz];
            uint64_t r = q - rb;
            __syncwarp();  // every lane has read the stack before lane 0 pushes over it
            x2d = false;
            while (sz > RG) {
                const int op = find_slot(t, sz, r);
                if (op == OP_NOT || op == OP_NEG) {
                    push_level(st, nx++, op, sz - 1, q - r + t->T[sz - 1], (W)0);
                    --sz;
                    continue;
                }
                const int j = find_split(t, sz, r);
                const int rsz = sz - 1 - j;
                if (rsz <= RG && j <= RG) {
                    // N_X: both children are table digits; the X-unit is the
                    // whole (op, j) split block of this node (left-major)
                    x2d = true;
                    pxop = op;
                    szy = j;
                    sz1 = rsz;
                    qb = q - r;
                    qend = qb + t->T[j] * t->T[rsz];
                    break;
                }
                const uint64_t qq = div_T(t, rsz, r);
                const uint64_t rr = r - qq * t->T[rsz];
                const W sv = sib_value(j, qq);
                push_level(st, nx++, op, rsz, q - rr + t->T[rsz], sv);
                sz = rsz;
                r = rr;
            }
            if (!x2d) {
                sz1 = sz;
                qb = q - r;
                qend = qb + t->T[sz];
            }
        }
        __syncwarp();
        bool bw_unused;
        compose<MAXSL>(st, nx, sl, nsl, ovf_l, bw_unused);
        have_x = true;
    }

    // P block containing rank n (n >= the previous call's n): afterwards
    // [pb, pend) is the block and (pop, prsz, so, nso) describe it.
    __device__ __forceinline__ void outer_at(uint64_t n)
    {
        if (!have_outer || n >= pend)
            decode_outer(n);
    }
};

}  // namespace simba
