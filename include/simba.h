/*
 * simba.h -- C ABI of the B200-native SIMBA hot path (libsimba.so).
 *
 * The reference (arxiv 2605.08243, package `mbasynth`, pure Python) has no FFI.
 * Its backend seam is the data-parallel map over a rank range
 * ("a pluggable data-parallel map over an index range whose body
 * is pure"), i.e. `engine._scan_range` (engine.py:128-156) dispatched by
 * `engine.synthesize` (engine.py:240-243).  Each entry point below names the
 * reference function it replaces.  INTEGRATION.md shows the ctypes binding a
 * maintainer adds to engine.py to route the reference through this library.
 *
 * Conventions: plain pointers and sizes, no exceptions across the ABI, every
 * function returns a SIMBA_* status code; `simba_last_error()` gives the
 * message of the last failure on the calling thread.  All calls are
 * synchronous.  There is no CPU fallback: on a host without a CUDA device the
 * context constructor fails with SIMBA_ECUDA.
 */
#ifndef SIMBA_H
#define SIMBA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SIMBA_OK 0
#define SIMBA_EINVAL 1      /* bad argument (ValueError in the reference) */
#define SIMBA_ERANGE 2      /* rank/size outside the table, or a count >= 2^64 */
#define SIMBA_ECAPACITY 3   /* counting.CountCapacityError (counting.py:35-43) */
#define SIMBA_ECUDA 4       /* CUDA runtime failure / no device */
#define SIMBA_ENOMEM 5

/* Largest expression size the device path supports (token buffer length). */
#define SIMBA_MAX_SIZE 24
/* Largest table extent simba_table_build accepts (128-bit host arithmetic). */
#define SIMBA_TABLE_MAX 64

#define SIMBA_MODE_SEARCH 0 /* minimum satisfying rank, early exit above it */
#define SIMBA_MODE_COUNT 1  /* exhaustive satisfying-candidate count */

#define SIMBA_STATUS_FOUND 0     /* engine.Status.FOUND     (engine.py:31-37) */
#define SIMBA_STATUS_NOT_FOUND 1 /* engine.Status.NOT_FOUND */
#define SIMBA_STATUS_TIMED_OUT 2 /* engine.Status.TIMED_OUT */

#define SIMBA_NO_RANK UINT64_MAX

/* ---------------------------------------------------------------------- */
/* Tables                                                                  */
/* ---------------------------------------------------------------------- */

/* counting.build(k, max_size) (counting.py:88-128).  Fills rows[s*9 + op]
 * (s = 0..max_size, op = 0..8, slot 8 = total) and cumulative[s] as 128-bit
 * values split into lo/hi words.  Returns SIMBA_ECAPACITY and sets
 * (*err_s, *err_op) at the first entry above 2^128-1, exactly like
 * CountCapacityError (counting.py:115-117). */
int simba_table_build(int k, int max_size, uint64_t *rows_lo, uint64_t *rows_hi,
                      uint64_t *cum_lo, uint64_t *cum_hi, int *err_s, int *err_op);

/* ---------------------------------------------------------------------- */
/* Context: one Specification bound to one device                          */
/* ---------------------------------------------------------------------- */

typedef struct simba_ctx simba_ctx;

typedef struct {
    int device;          /* CUDA ordinal (default 0) */
    int r0;              /* shared-memory value-table cutoff (lane digit); 0 = auto */
    int rg;              /* global value-table cutoff (left values, siblings); 0 = auto */
    int table_examples;  /* examples with value tables (1, 2 or 4); 0 = auto */
    int block_threads;   /* 0 = auto (256) */
    int blocks_per_sm;   /* 0 = occupancy calculator */
    int kernel;          /* 0 = unit kernel (default), 1 = per-rank direct kernel */
} simba_options;

/* Binds a Specification (engine.py:40-78; inputs row-major [n][k], outputs
 * [n]) and the count table for sizes 1..max_size to a device: stages the
 * tables, the examples and the per-spec super-leaf value tables in device
 * memory.  Validation matches Specification.__post_init__ (engine.py:52-67):
 * k >= 1, 1 <= w <= 64, n >= 1, values < 2^w, pairwise-distinct inputs ->
 * SIMBA_EINVAL.  T[s][8] >= 2^64 for some s <= max_size -> SIMBA_ERANGE.
 * opt may be NULL (defaults). */
int simba_ctx_create(int k, int w, int n, const uint64_t *inputs, const uint64_t *outputs,
                     int max_size, const simba_options *opt, simba_ctx **out);
void simba_ctx_destroy(simba_ctx *ctx);

typedef struct {
    uint64_t visited;    /* candidates whose evaluation completed */
    uint64_t count;      /* satisfying candidates (exact in COUNT mode) */
    uint64_t best_rank;  /* minimum satisfying in-size rank, SIMBA_NO_RANK if none */
    int32_t found;
    int32_t completed;   /* 0 when a time budget stopped the scan early */
    int32_t size;
    int32_t tokens[SIMBA_MAX_SIZE]; /* RPN tokens of best_rank (expr.py:66-85) */
    double kernel_ms;    /* device time of the scan launch (CUDA events) */
    uint64_t launches;   /* kernels launched for this call */
    uint64_t units;      /* units decoded by the unit kernel */
    uint64_t rank_units; /* units that took the per-rank path */
    uint64_t ex0_hits;   /* candidates matching example 0 (for the e-bar statistic) */
} simba_result;

/* engine._scan_range(ctx, size, offset, block_total, start, stop, shuffled)
 * (engine.py:128-156): decode-evaluate-discard local indices [start, stop) of
 * the operator block starting at in-size rank `offset` with `block_total`
 * candidates; local index i maps to rank offset + i, or to
 * offset + (i * 2246822507 mod block_total) when shuffled (engine.py:145,
 * codec.py:29).  Returns visited = stop - start and the minimum satisfying
 * rank with its tokens, like the reference's (visited, best_rank, best_tokens). */
int simba_scan_range(simba_ctx *ctx, int size, uint64_t offset, uint64_t block_total,
                     uint64_t start, uint64_t stop, int shuffled, simba_result *out);

/* General range request: in-size ranks [lo, hi) at `size`, cut into chunks
 * of `chunk` ranks (0 = auto); this caller processes chunks c with
 * c % nshards == shard (round-robin super-chunks for multi-GPU sharding,
 * SURVEY.md 8(e)).  SEARCH mode stops claiming chunks above the best hit
 * (and above `stop_above`, a bound learnt from other shards); COUNT mode
 * visits every rank.  time_budget_s < 0 disables the budget, which is
 * polled between chunks only and never masks a recorded hit
 * (engine.py:251-258). */
typedef struct {
    int size;
    int mode;
    uint64_t lo, hi;
    uint64_t chunk;
    uint64_t shard, nshards;
    uint64_t stop_above;
    double time_budget_s;
} simba_range;

int simba_run(simba_ctx *ctx, const simba_range *req, simba_result *out);

/* Several size levels in ONE launch (the loop of engine.py:222-262 fused on
 * the device): levels size_lo..size_hi form one virtual rank space (level s
 * follows level s-1), claimed in ascending order and sharded round-robin like
 * simba_run.  SEARCH mode returns the minimum (size, rank) -- the smallest
 * level with a hit, then its smallest rank, exactly the reference's order --
 * and stops claiming above it; COUNT mode visits everything.  levels[i]
 * (i = s - size_lo) receives the level's count, first satisfying rank and
 * visited candidates (in SEARCH mode exact up to the found level; with
 * nshards > 1, this shard's share of the level, so the SUM over shards is
 * the level's total); `out`
 * carries the totals, the found (size, rank, tokens) and the launch time. */
typedef struct {
    int32_t size;
    uint64_t count;
    uint64_t first_rank;  /* SIMBA_NO_RANK if none */
    uint64_t visited;
} simba_level;

int simba_run_levels(simba_ctx *ctx, int size_lo, int size_hi, int mode, uint64_t shard, uint64_t nshards,
                     double time_budget_s, simba_level *levels, simba_result *out);

/* ---------------------------------------------------------------------- */
/* Cross-GPU early exit of a sharded search                */
/* ---------------------------------------------------------------------- */

/* The reference stops after the first wave with a hit (engine.py:248-250);
 * across GPUs the equivalent is one 8-byte minimum that every shard's kernel
 * publishes its hits to (atomicMin, system scope: NVLink peer atomics) and
 * folds into its own bound at every claim and phase, so that no shard keeps
 * claiming above another shard's hit.  Attached contexts use it in SEARCH
 * requests with nshards > 1 (simba_run, simba_run_levels); every context
 * sharing one word must run the same request space (same levels), and the
 * word must be reset (simba_xbest_reset, by one process, followed by a
 * barrier) before each sharded search.
 *
 * A simba_xbest is that word.  simba_xbest_create allocates it on `device`
 * (set to SIMBA_NO_RANK) and writes its CUDA IPC handle
 * (SIMBA_XBEST_HANDLE_BYTES bytes) for the other processes of the job;
 * simba_xbest_open maps a handle created by ANOTHER process into this one on
 * `device` (peer access over NVLink when the devices differ).  Contexts of one
 * process may share one simba_xbest directly.  simba_ctx_set_xbest attaches
 * it to a context (NULL detaches); the creator must outlive every search that
 * uses it, and a context must not outlive the simba_xbest it is attached to. */
#define SIMBA_XBEST_HANDLE_BYTES 64
typedef struct simba_xbest simba_xbest;
int simba_xbest_create(int device, unsigned char *handle, simba_xbest **out);
int simba_xbest_open(int device, const unsigned char *handle, simba_xbest **out);
int simba_xbest_reset(simba_xbest *x);
int simba_xbest_read(simba_xbest *x, uint64_t *value);
void simba_xbest_destroy(simba_xbest *x);
int simba_ctx_set_xbest(simba_ctx *ctx, simba_xbest *x);

/* engine.synthesize (engine.py:190-276), Algorithm 1 on the device: sizes
 * 1..size_bound ascending, each size level scanned in rank order (operator
 * blocks are contiguous rank ranges in slot order, engine.py:175-187) with
 * early exit above the best hit; result = (minimum size with a hit, minimum
 * in-size rank at that size), identical in local and shuffled mode. */
typedef struct {
    int32_t status;      /* SIMBA_STATUS_* */
    int32_t size;
    uint64_t rank;
    int32_t tokens[SIMBA_MAX_SIZE];
    int32_t nsizes;      /* entries in the per-size stats (SizeStats) */
    uint64_t visited[SIMBA_MAX_SIZE];
    double millis[SIMBA_MAX_SIZE];
    double kernel_ms;
    uint64_t launches;
} simba_outcome;

int simba_synthesize(simba_ctx *ctx, int size_bound, int shuffled, double time_budget_s,
                     simba_outcome *out);

/* codec.decode(rank, size, table) (codec.py:136-144) on the device. */
int simba_decode(simba_ctx *ctx, uint64_t rank, int size, int32_t *tokens);

/* Decode of the ranks [rank0, rank0 + count) of one size into
 * tokens[count][size] (one thread per rank): the sweep of
 * engine.enumerate_all (engine.py:279-293). */
int simba_decode_batch(simba_ctx *ctx, uint64_t rank0, uint64_t count, int size, int32_t *tokens);

/* Effective configuration of a context (for reports): r0, rg, table
 * examples, word bytes, grid blocks, block threads, shared-memory bytes per block. */
int simba_ctx_info(simba_ctx *ctx, int *r0, int *rg, int *table_examples, int *word_bytes, int *grid_blocks,
                   int *block_threads, int *smem_bytes);

/* Host->device and device->host bytes this context has copied so far. */
int simba_ctx_bytes(simba_ctx *ctx, uint64_t *h2d, uint64_t *d2h);

/* The CUDA stream (cudaStream_t) the context launches on, for callers that
 * record their own events around calls. */
int simba_ctx_stream(simba_ctx *ctx, void **stream);

/* INT32 issue-rate probe (roofline denominator): independent LOP3->IMAD
 * chains on every SM; reports integer ops/s and the kernel time. */
int simba_int32_peak(int device, int iters, double *ops_per_s, double *kernel_ms);

/* Pipe-saturating integer probes: 16 independent single-instruction chains
 * per thread on every SM.  mode 0: LOP3 only (the ALU pipe; SURVEY.md 8(d)'s
 * P_int32, nominally 148 SMs x 64 lanes x clock); mode 1: LOP3 and IMAD
 * interleaved (ALU + FMA pipes, the issue limit).  Reports thread-level
 * integer ops/s and the kernel time. */
int simba_int32_pipe_peak(int device, int iters, int mode, double *ops_per_s, double *kernel_ms);

/* Diagnostics: per-path (calls, candidates) counters of the unit kernel since
 * the context was created, in path order RF-fold, RF-gen, RF-row, CF-fold,
 * CF-gen, then (calls, SM cycles) of outer odometer steps, X odometer steps
 * and tile calls, then the per-rank (direct) path.  Copies up to n words and returns how many were
 * written; 0 unless the library was built with -DSIMBA_STATS. */
int simba_ctx_stats(simba_ctx *ctx, uint64_t *out, int n);

const char *simba_last_error(void);
int simba_device_count(void);
/* ---------------------------------------------------------------------- */
/* VFB cache-based baseline (baseline.run_baseline, baseline.py:88-249)     */
/* ---------------------------------------------------------------------- */

/* The paper's comparison point: bottom-up enumeration
 * over cached behaviour vectors with observational-equivalence pruning.
 * A run is one simba_vfb object; sizes are stepped in order 1, 2, ... by
 * simba_vfb_level, which reports the per-size row of baseline.py's
 * CacheSizeRow (baseline.py:51-58) and the event that ended the run. */
typedef struct simba_vfb simba_vfb;

#define SIMBA_VFB_NONE 0      /* the size ran to completion */
#define SIMBA_VFB_FOUND 1     /* a candidate matched the outputs (baseline.py:156-158) */
#define SIMBA_VFB_OOM 2       /* modeled storage exceeded the budget (baseline.py:161-163) */
#define SIMBA_VFB_TIMED_OUT 3 /* the time budget expired between batches (baseline.py:149-153) */

typedef struct {
    uint64_t candidates;  /* candidates considered at this size (the ending one included) */
    uint64_t stored;      /* entries newly stored at this size */
    uint64_t stored_cum;  /* entries stored over all sizes */
    uint64_t event_index; /* candidate index (in the size's order) of a FOUND / OOM event */
    int32_t event;        /* SIMBA_VFB_* */
    double millis;        /* host wall time of the size */
} simba_vfb_row;

/* inputs row-major [n][k], outputs [n] (validated by the caller as in
 * Specification); max_entries = memory_budget / entry_bytes (UINT64_MAX when
 * entries model 0 bytes).  Device memory grows with the entries stored;
 * exhausting it is SIMBA_ENOMEM (not the modeled OOM). */
int simba_vfb_create(int k, int w, int n, const uint64_t *inputs, const uint64_t *outputs, uint64_t max_entries,
                     int device, simba_vfb **out);
/* Runs one size (must be the previous size + 1).  time_budget_s < 0: none,
 * else the size stops with SIMBA_VFB_TIMED_OUT once this many seconds have
 * passed at a batch boundary. */
int simba_vfb_level(simba_vfb *v, int size, double time_budget_s, simba_vfb_row *out);
/* RPN tokens (expr.py:66-85) of candidate `cand` of the last size run. */
int simba_vfb_tokens(simba_vfb *v, uint64_t cand, int32_t *tokens, int cap, int *len);
void simba_vfb_destroy(simba_vfb *v);

/* Kernels this library has launched in this process. */
uint64_t simba_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* SIMBA_H */
