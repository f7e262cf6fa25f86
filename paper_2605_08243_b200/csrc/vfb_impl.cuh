// vfb_impl.cuh -- the cache-based bottom-up baseline ("VFB", baseline.py) on the GPU.
//
// Included at the end of simba.cu (shares fail()/CK/g_launches).  This is the
// paper's comparison point, not the SIMBA path: every
// size level builds candidates from the CACHED representatives of smaller
// sizes and keeps a candidate only when its behaviour vector (its outputs on
// the n examples) is new.  Semantics follow baseline.run_baseline
// (baseline.py:88-249) exactly:
//
//   * candidate order per size: slot NOT, AND, OR, XOR, NEG, ADD, SUB, MUL
//     (baseline.py:186-204); unary slots over entries[s-1] in insertion
//     order; binary slots over splits j = 1..top (top = (s-1)/2 for the
//     commutative slots, s-2 for SUB), left entry major, right entry minor;
//     size 1 = the k variables (baseline.py:180-184);
//   * per candidate (consider, baseline.py:144-167): a match with the spec's
//     outputs ends the run FOUND (checked before the cache, so a duplicate
//     behaviour still matches); a behaviour already cached is dropped; a new
//     one is stored unless (stored_cum + 1) * entry_bytes > budget, which ends
//     the run OOM_ABORTED at this size;
//   * entries[s] keep insertion order (= candidate order of first occurrence),
//     which fixes the candidate order of every later size.
//
// Device design.  Candidates of one size are processed in ascending batches.
// Each batch runs three kernels:
//   vfb_insert   one thread per candidate: evaluate the behaviour from the two
//                cached rows, hash it, record a target match (atomicMin of the
//                candidate index), and insert it into an open-addressing table
//                of 64-bit keys (entry id, or kCand + candidate index).  Equal
//                behaviours meet in one slot; atomicMin keeps the smallest key
//                there, so a cached entry always beats a candidate and among
//                candidates the first in order wins.  Comparing against a
//                candidate key re-evaluates that candidate from its rows.
//   vfb_flags    per CTA tile: candidate c is new iff its slot still holds its
//                own key; count per tile.
//   vfb_scatter  tile offsets by a one-CTA scan, then the new candidates in
//                order get entry ids stored_cum + r (r = rank among the new
//                ones), their behaviour row and (op, left, right) are written
//                and their slot is rewritten to the entry id -- unless the
//                batch holds the run's end: a match at index m (only c < m are
//                stored) or the (cap_left + 1)-th new candidate (OOM).
// Batches run in order, so a later batch's candidate never displaces an
// earlier one.  The time budget is polled between batches (baseline.py:149-153
// polls between candidate groups; never mid-candidate).
//
// Memory: behaviour rows [entries][n] words (u32 for w <= 32, else u64), the
// per-entry (op, left, right) triples and the table grow with the entries
// actually stored; the modeled budget (n * w / 8 bytes per entry,
// baseline.py:25-27) decides OOM, the device only has to hold what fits in it.

namespace {

constexpr uint64_t kVfbEmpty = ~0ull;
constexpr uint64_t kVfbCand = 1ull << 48;  // keys >= kVfbCand are candidates of the current size
constexpr int kVfbThreads = 256;
constexpr int kVfbItems = 8;                          // candidates per thread in the flag/scatter tiles
constexpr uint64_t kVfbTile = kVfbThreads * kVfbItems;  // candidates per CTA tile
constexpr uint64_t kVfbBatch = 1ull << 24;              // candidates per batch
constexpr int kVfbMaxBlocks = 2 + 6 * SIMBA_MAX_SIZE;  // leaf + 2 unary + 6 binary slots x splits

enum : int8_t { VOP_VAR = -1 };  // size-1 entries: left = variable index

struct VfbBlock {
    uint64_t base;   // first level-relative candidate index
    uint64_t rcnt;   // right entries (binary); 1 otherwise
    uint32_t loff;   // first left entry id (or 0 for variables)
    uint32_t roff;   // first right entry id
    int32_t op;      // slot 0..7, or VOP_VAR
};

struct VfbBlocks {
    VfbBlock b[kVfbMaxBlocks];
    int nb;
};

struct VfbCtl {
    unsigned long long match;   // smallest matching candidate (level-relative), ~0 if none
    unsigned long long oom;     // first new candidate beyond the cap, ~0 if none
    unsigned long long stored;  // entries stored by the batch
};

template <class W>
struct VfbArgs {
    const W *beh;        // [entries][n]
    const W *var;        // [k][n] behaviours of the variables
    const W *tgt;        // [n] outputs
    unsigned long long *H;
    uint64_t hmask;
    int n;
    W mask;
};

__device__ __forceinline__ uint64_t vfb_mix(uint64_t h, uint64_t v)
{
    h ^= v + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
    h *= 0xBF58476D1CE4E5B9ull;
    return h ^ (h >> 31);
}

template <class W>
__device__ __forceinline__ W vfb_apply(int op, W a, W b, W mask)
{
    switch (op) {
    case 0: return a ^ mask;                 // NOT
    case 1: return a & b;                    // AND
    case 2: return a | b;                    // OR
    case 3: return a ^ b;                    // XOR
    case 4: return (W)(0 - a) & mask;        // NEG
    case 5: return (W)(a + b) & mask;        // ADD
    case 6: return (W)(a - b) & mask;        // SUB
    case 7: return (W)(a * b) & mask;        // MUL
    default: return a;                       // variable
    }
}

// candidate c of the level -> (op, row a, row b)
template <class W>
__device__ __forceinline__ void vfb_decode(const VfbBlocks &bl, const VfbArgs<W> &A, uint64_t c, int &op,
                                           const W *&ra, const W *&rb, uint64_t *li = nullptr, uint64_t *ri = nullptr)
{
    int i = 0;
    while (i + 1 < bl.nb && bl.b[i + 1].base <= c)
        ++i;
    const VfbBlock &B = bl.b[i];
    const uint64_t local = c - B.base;
    op = B.op;
    if (op == VOP_VAR) {
        ra = A.var + local * A.n;
        rb = ra;
        if (li) *li = local, *ri = 0;
    } else if (op == 0 || op == 4) {
        ra = A.beh + (B.loff + local) * (uint64_t)A.n;
        rb = ra;
        if (li) *li = B.loff + local, *ri = 0;
    } else {
        const uint64_t l = local / B.rcnt, r = local - l * B.rcnt;
        ra = A.beh + (B.loff + l) * (uint64_t)A.n;
        rb = A.beh + (B.roff + r) * (uint64_t)A.n;
        if (li) *li = B.loff + l, *ri = B.roff + r;
    }
}

template <class W>
__device__ __forceinline__ bool vfb_equal_key(const VfbBlocks &bl, const VfbArgs<W> &A, uint64_t key, int op,
                                              const W *ra, const W *rb)
{
    if (key < kVfbCand) {
        const W *e = A.beh + key * (uint64_t)A.n;
        for (int i = 0; i < A.n; ++i)
            if (vfb_apply<W>(op, ra[i], rb[i], A.mask) != e[i])
                return false;
        return true;
    }
    int op2;
    const W *qa, *qb;
    vfb_decode<W>(bl, A, key - kVfbCand, op2, qa, qb);
    for (int i = 0; i < A.n; ++i)
        if (vfb_apply<W>(op, ra[i], rb[i], A.mask) != vfb_apply<W>(op2, qa[i], qb[i], A.mask))
            return false;
    return true;
}

template <class W>
__global__ void __launch_bounds__(kVfbThreads) vfb_insert(const __grid_constant__ VfbBlocks bl, const VfbArgs<W> A,
                                                          uint64_t c0, uint64_t c1, uint32_t *slot_of,
                                                          VfbCtl *ctl)
{
    for (uint64_t c = c0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < c1;
         c += (uint64_t)gridDim.x * blockDim.x) {
        int op;
        const W *ra, *rb;
        vfb_decode<W>(bl, A, c, op, ra, rb);
        uint64_t h = 0x2545F4914F6CDD1Dull;
        bool match = true;
        for (int i = 0; i < A.n; ++i) {
            const W v = vfb_apply<W>(op, ra[i], rb[i], A.mask);
            h = vfb_mix(h, (uint64_t)v);
            match &= (v == A.tgt[i]);
        }
        if (match)
            atomicMin(&ctl->match, (unsigned long long)c);
        const unsigned long long key = kVfbCand + c;
        uint64_t s = h & A.hmask;
        for (;;) {
            unsigned long long cur = *(volatile unsigned long long *)&A.H[s];
            if (cur == kVfbEmpty) {
                const unsigned long long prev = atomicCAS(&A.H[s], kVfbEmpty, key);
                if (prev == kVfbEmpty)
                    break;
                cur = prev;
            }
            if (vfb_equal_key<W>(bl, A, cur, op, ra, rb)) {
                if (cur > key)
                    atomicMin(&A.H[s], key);
                break;
            }
            s = (s + 1) & A.hmask;
        }
        slot_of[c - c0] = (uint32_t)s;
    }
}

// new[c] = the slot kept c's own key; per-tile counts
__global__ void __launch_bounds__(kVfbThreads) vfb_flags(const unsigned long long *H, uint64_t c0, uint64_t c1,
                                                         const uint32_t *slot_of, uint32_t *tile_cnt)
{
    const uint64_t t0 = c0 + blockIdx.x * kVfbTile;
    uint32_t cnt = 0;
    for (int it = 0; it < kVfbItems; ++it) {
        const uint64_t c = t0 + (uint64_t)it * kVfbThreads + threadIdx.x;
        if (c < c1)
            cnt += (H[slot_of[c - c0]] == kVfbCand + c);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1)
        cnt += __shfl_xor_sync(FULL, cnt, o);
    __shared__ uint32_t wsum[kVfbThreads / 32];
    if ((threadIdx.x & 31) == 0)
        wsum[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int i = 0; i < kVfbThreads / 32; ++i)
            t += wsum[i];
        tile_cnt[blockIdx.x] = t;
    }
}

// exclusive scan of the tile counts (one CTA; tiles per batch <= 8192)
__global__ void __launch_bounds__(1024) vfb_scan(uint32_t *tile_cnt, int ntiles)
{
    __shared__ uint32_t part[1024];
    const int per = (ntiles + 1023) / 1024;
    const int b = threadIdx.x * per;
    uint32_t s = 0;
    for (int i = b; i < min(b + per, ntiles); ++i)
        s += tile_cnt[i];
    part[threadIdx.x] = s;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
        const uint32_t v = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
        __syncthreads();
        part[threadIdx.x] += v;
        __syncthreads();
    }
    uint32_t acc = part[threadIdx.x] - s;
    for (int i = b; i < min(b + per, ntiles); ++i) {
        const uint32_t v = tile_cnt[i];
        tile_cnt[i] = acc;
        acc += v;
    }
}

template <class W>
__global__ void __launch_bounds__(kVfbThreads) vfb_scatter(const __grid_constant__ VfbBlocks bl, const VfbArgs<W> A,
                                                           uint64_t c0, uint64_t c1, const uint32_t *slot_of,
                                                           const uint32_t *tile_off, uint64_t stored_cum,
                                                           uint64_t cap_left, W *beh_out, uint32_t *m_l,
                                                           uint32_t *m_r, int8_t *m_op, VfbCtl *ctl)
{
    __shared__ uint32_t wsum[kVfbThreads / 32];
    const uint64_t match = *(volatile unsigned long long *)&ctl->match;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint64_t r = tile_off[blockIdx.x];
    uint32_t stored = 0;
    const uint64_t t0 = c0 + blockIdx.x * kVfbTile;
    for (int it = 0; it < kVfbItems; ++it) {
        const uint64_t c = t0 + (uint64_t)it * kVfbThreads + threadIdx.x;
        bool isnew = false;
        uint32_t s = 0;
        if (c < c1) {
            s = slot_of[c - c0];
            isnew = A.H[s] == kVfbCand + c;
        }
        // rank of c among the tile's new candidates, in candidate order
        const unsigned bal = __ballot_sync(FULL, isnew);
        if (lane == 0)
            wsum[wid] = __popc(bal);
        __syncthreads();
        uint32_t before = 0, total = 0;
        for (int i = 0; i < kVfbThreads / 32; ++i) {
            before += (i < wid) ? wsum[i] : 0;
            total += wsum[i];
        }
        const uint64_t rank = r + before + __popc(bal & ((1u << lane) - 1));
        if (isnew) {
            if (rank >= cap_left) {
                atomicMin(&ctl->oom, (unsigned long long)c);
            } else if (c < match) {
                int op;
                const W *ra, *rb;
                uint64_t li, ri;
                vfb_decode<W>(bl, A, c, op, ra, rb, &li, &ri);
                const uint64_t id = stored_cum + rank;
                W *o = beh_out + id * (uint64_t)A.n;
                for (int i = 0; i < A.n; ++i)
                    o[i] = vfb_apply<W>(op, ra[i], rb[i], A.mask);
                m_l[id] = (uint32_t)li;
                m_r[id] = (uint32_t)ri;
                m_op[id] = (int8_t)op;
                A.H[s] = id;
                ++stored;
            }
        }
        r += total;
        __syncthreads();
    }
#pragma unroll
    for (int o = 16; o; o >>= 1)
        stored += __shfl_xor_sync(FULL, stored, o);
    if (lane == 0 && stored)
        atomicAdd(&ctl->stored, (unsigned long long)stored);
}

// rebuild the table from the cached entries (distinct behaviours: no compares)
template <class W>
__global__ void __launch_bounds__(kVfbThreads) vfb_rehash(const VfbArgs<W> A, uint64_t entries)
{
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < entries;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const W *row = A.beh + e * (uint64_t)A.n;
        uint64_t h = 0x2545F4914F6CDD1Dull;
        for (int i = 0; i < A.n; ++i)
            h = vfb_mix(h, (uint64_t)row[i]);
        uint64_t s = h & A.hmask;
        while (atomicCAS(&A.H[s], kVfbEmpty, (unsigned long long)e) != kVfbEmpty)
            s = (s + 1) & A.hmask;
    }
}

__global__ void vfb_fill(unsigned long long *p, uint64_t n, unsigned long long v)
{
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

}  // namespace

struct simba_vfb {
    int device = 0, k = 0, w = 0, n = 0, wb = 4;
    uint64_t mask = 0, max_entries = 0;
    int last_size = 0;
    bool ended = false;
    std::vector<uint64_t> off, cnt;  // entries of each size: ids [off[s], off[s] + cnt[s])
    uint64_t stored = 0;
    uint64_t batch = kVfbBatch;  // candidates per batch (SIMBA_VFB_BATCH overrides, for tests)
    // device
    cudaStream_t stream = nullptr;
    void *beh = nullptr, *var = nullptr, *tgt = nullptr;
    uint32_t *m_l = nullptr, *m_r = nullptr;
    int8_t *m_op = nullptr;
    uint64_t ecap = 0;  // entry capacity of beh / meta
    unsigned long long *H = nullptr;
    uint64_t hslots = 0;
    uint32_t *slot_of = nullptr, *tile_cnt = nullptr;
    VfbCtl *ctl = nullptr, *h_ctl = nullptr;
    VfbBlocks bl{};
};

namespace {

template <class W>
VfbArgs<W> vfb_args(simba_vfb *v)
{
    VfbArgs<W> a;
    a.beh = reinterpret_cast<const W *>(v->beh);
    a.var = reinterpret_cast<const W *>(v->var);
    a.tgt = reinterpret_cast<const W *>(v->tgt);
    a.H = v->H;
    a.hmask = v->hslots - 1;
    a.n = v->n;
    a.mask = (W)v->mask;
    return a;
}

int vfb_grid(uint64_t work)
{
    const uint64_t b = (work + kVfbThreads - 1) / kVfbThreads;
    return (int)std::max<uint64_t>(1, std::min<uint64_t>(b, 148ull * 16));
}

// grow the entry arrays to hold `need` entries (amortised doubling)
int vfb_reserve_entries(simba_vfb *v, uint64_t need)
{
    if (need <= v->ecap)
        return SIMBA_OK;
    uint64_t cap = std::max<uint64_t>(need, std::max<uint64_t>(1024, v->ecap * 2));
    const size_t row = (size_t)v->n * v->wb;
    void *beh = nullptr;
    uint32_t *ml = nullptr, *mr = nullptr;
    int8_t *mo = nullptr;
    if (cudaMalloc(&beh, cap * row) != cudaSuccess || cudaMalloc(&ml, cap * 4) != cudaSuccess ||
        cudaMalloc(&mr, cap * 4) != cudaSuccess || cudaMalloc(&mo, cap) != cudaSuccess) {
        cudaGetLastError();
        cudaFree(beh), cudaFree(ml), cudaFree(mr), cudaFree(mo);
        return fail(SIMBA_ENOMEM, "device memory exhausted holding %llu cache entries (%zu bytes each)",
                    (unsigned long long)cap, row);
    }
    if (v->stored) {
        CK(cudaMemcpyAsync(beh, v->beh, v->stored * row, cudaMemcpyDeviceToDevice, v->stream));
        CK(cudaMemcpyAsync(ml, v->m_l, v->stored * 4, cudaMemcpyDeviceToDevice, v->stream));
        CK(cudaMemcpyAsync(mr, v->m_r, v->stored * 4, cudaMemcpyDeviceToDevice, v->stream));
        CK(cudaMemcpyAsync(mo, v->m_op, v->stored, cudaMemcpyDeviceToDevice, v->stream));
        CK(cudaStreamSynchronize(v->stream));
    }
    cudaFree(v->beh), cudaFree(v->m_l), cudaFree(v->m_r), cudaFree(v->m_op);
    v->beh = beh, v->m_l = ml, v->m_r = mr, v->m_op = mo;
    v->ecap = cap;
    return SIMBA_OK;
}

// grow the table to at least 2 * keys slots and re-insert the entries
template <class W>
int vfb_reserve_table(simba_vfb *v, uint64_t keys)
{
    uint64_t slots = 1024;
    while (slots < 2 * keys)
        slots <<= 1;
    if (slots > (1ull << 32))
        return fail(SIMBA_ENOMEM, "cache table of %llu keys exceeds 2^31 entries", (unsigned long long)keys);
    if (slots <= v->hslots)
        return SIMBA_OK;
    unsigned long long *H = nullptr;
    if (cudaMalloc(&H, slots * 8) != cudaSuccess) {
        cudaGetLastError();
        return fail(SIMBA_ENOMEM, "device memory exhausted allocating a %llu-slot cache table",
                    (unsigned long long)slots);
    }
    cudaFree(v->H);
    v->H = H;
    v->hslots = slots;
    vfb_fill<<<vfb_grid(slots), kVfbThreads, 0, v->stream>>>(H, slots, kVfbEmpty);
    ++g_launches;
    if (v->stored) {
        vfb_rehash<W><<<vfb_grid(v->stored), kVfbThreads, 0, v->stream>>>(vfb_args<W>(v), v->stored);
        ++g_launches;
    }
    CK(cudaGetLastError());
    return SIMBA_OK;
}

template <class W>
int vfb_level(simba_vfb *v, int s, double budget_s, simba_vfb_row *out)
{
    const auto t0 = std::chrono::steady_clock::now();
    // candidate blocks of this size in baseline.py order
    VfbBlocks &bl = v->bl;
    bl.nb = 0;
    uint64_t total = 0;
    auto add = [&](int op, uint64_t count, uint64_t rcnt, uint64_t loff, uint64_t roff) {
        if (count == 0)
            return;
        bl.b[bl.nb++] = VfbBlock{total, rcnt, (uint32_t)loff, (uint32_t)roff, op};
        total += count;
    };
    if (s == 1) {
        add(VOP_VAR, (uint64_t)v->k, 1, 0, 0);
    } else {
        for (int slot = 0; slot < 8; ++slot) {
            if (slot == 0 || slot == 4) {
                add(slot, v->cnt[s - 1], 1, v->off[s - 1], 0);
            } else {
                const int top = (slot == 6) ? s - 2 : (s - 1) / 2;
                for (int j = 1; j <= top; ++j) {
                    const u128 c = (u128)v->cnt[j] * v->cnt[s - 1 - j];
                    if (c >> 63)
                        return fail(SIMBA_ERANGE, "size %d has 2^63 candidates or more", s);
                    add(slot, (uint64_t)c, v->cnt[s - 1 - j], v->off[j], v->off[s - 1 - j]);
                }
            }
        }
    }
    const uint64_t cap_total = v->max_entries;
    const uint64_t cap_left0 = cap_total > v->stored ? cap_total - v->stored : 0;
    // capacity: new entries <= min(candidates, cap_left); table keys <= that plus one batch
    const uint64_t new_max = std::min(total, cap_left0);
    if (int e = vfb_reserve_entries(v, v->stored + new_max))
        return e;
    if (int e = vfb_reserve_table<W>(v, v->stored + std::min(total, cap_left0 + v->batch)))
        return e;
    if (v->stored + new_max >= (1ull << 32))
        return fail(SIMBA_ENOMEM, "more than 2^32 cache entries");
    const VfbArgs<W> A = vfb_args<W>(v);
    uint64_t candidates = 0, stored_new = 0;
    int event = SIMBA_VFB_NONE;
    uint64_t event_index = 0;
    for (uint64_t c0 = 0; c0 < total;) {
        const uint64_t c1 = std::min(total, c0 + v->batch);
        const uint64_t cap_left = cap_left0 - stored_new;
        *v->h_ctl = VfbCtl{~0ull, ~0ull, 0};
        CK(cudaMemcpyAsync(v->ctl, v->h_ctl, sizeof(VfbCtl), cudaMemcpyHostToDevice, v->stream));
        const int ntiles = (int)((c1 - c0 + kVfbTile - 1) / kVfbTile);
        vfb_insert<W><<<vfb_grid(c1 - c0), kVfbThreads, 0, v->stream>>>(bl, A, c0, c1, v->slot_of, v->ctl);
        vfb_flags<<<ntiles, kVfbThreads, 0, v->stream>>>(v->H, c0, c1, v->slot_of, v->tile_cnt);
        vfb_scan<<<1, 1024, 0, v->stream>>>(v->tile_cnt, ntiles);
        vfb_scatter<W><<<ntiles, kVfbThreads, 0, v->stream>>>(
            bl, A, c0, c1, v->slot_of, v->tile_cnt, v->stored + stored_new, cap_left,
            reinterpret_cast<W *>(v->beh), v->m_l, v->m_r, v->m_op, v->ctl);
        g_launches += 4;
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(v->h_ctl, v->ctl, sizeof(VfbCtl), cudaMemcpyDeviceToHost, v->stream));
        CK(cudaStreamSynchronize(v->stream));
        const VfbCtl r = *v->h_ctl;
        stored_new += r.stored;
        if (r.match != ~0ull && r.match <= r.oom) {
            event = SIMBA_VFB_FOUND;
            event_index = r.match;
            candidates = r.match + 1;
            break;
        }
        if (r.oom != ~0ull) {
            event = SIMBA_VFB_OOM;
            event_index = r.oom;
            candidates = r.oom + 1;
            break;
        }
        candidates = c1;
        c0 = c1;
        const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (budget_s >= 0 && el > budget_s && c0 < total) {
            event = SIMBA_VFB_TIMED_OUT;
            break;
        }
    }
    v->off.resize(s + 1);
    v->cnt.resize(s + 1);
    v->off[s] = v->stored;
    v->cnt[s] = stored_new;
    v->stored += stored_new;
    v->last_size = s;
    v->ended = event != SIMBA_VFB_NONE;
    out->candidates = candidates;
    out->stored = stored_new;
    out->stored_cum = v->stored;
    out->event = event;
    out->event_index = event_index;
    out->millis = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return SIMBA_OK;
}

// RPN tokens of a cached entry (recursive through the (op, left, right) triples)
int vfb_entry_tokens(simba_vfb *v, uint64_t id, std::vector<int32_t> &out)
{
    uint32_t l = 0, r = 0;
    int8_t op = 0;
    CK(cudaMemcpy(&l, v->m_l + id, 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&r, v->m_r + id, 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&op, v->m_op + id, 1, cudaMemcpyDeviceToHost));
    if (op == VOP_VAR) {
        out.push_back((int32_t)l);
        return SIMBA_OK;
    }
    if (int e = vfb_entry_tokens(v, l, out))
        return e;
    if (op != 0 && op != 4)
        if (int e = vfb_entry_tokens(v, r, out))
            return e;
    out.push_back(-(op + 1));
    return SIMBA_OK;
}

}  // namespace

extern "C" {

int simba_vfb_create(int k, int w, int n, const uint64_t *inputs, const uint64_t *outputs, uint64_t max_entries,
                     int device, simba_vfb **out)
{
    if (!out || !inputs || !outputs)
        return fail(SIMBA_EINVAL, "null argument");
    *out = nullptr;
    if (k < 1 || w < 1 || w > 64 || n < 1)
        return fail(SIMBA_EINVAL, "need k >= 1, 1 <= w <= 64, n >= 1 (got k=%d w=%d n=%d)", k, w, n);
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(SIMBA_ECUDA, "no CUDA device");
    }
    if (device < 0 || device >= ndev)
        return fail(SIMBA_EINVAL, "device %d outside 0..%d", device, ndev - 1);
    CK(cudaSetDevice(device));
    auto *v = new simba_vfb();
    v->device = device, v->k = k, v->w = w, v->n = n;
    v->wb = w <= 32 ? 4 : 8;
    v->mask = w == 64 ? ~0ull : ((1ull << w) - 1);
    v->max_entries = max_entries;
    if (const char *b = getenv("SIMBA_VFB_BATCH"))
        v->batch = std::max<uint64_t>(1, std::min<uint64_t>(kVfbBatch, strtoull(b, nullptr, 10)));
    v->off.assign(1, 0);
    v->cnt.assign(1, 0);
    // behaviours of the variables [k][n] and the outputs [n], in the word type
    std::vector<unsigned char> var((size_t)k * n * v->wb), tgt((size_t)n * v->wb);
    for (int i = 0; i < k; ++i)
        for (int e = 0; e < n; ++e) {
            const uint64_t x = inputs[(size_t)e * k + i];
            if (v->wb == 4) reinterpret_cast<uint32_t *>(var.data())[(size_t)i * n + e] = (uint32_t)x;
            else reinterpret_cast<uint64_t *>(var.data())[(size_t)i * n + e] = x;
        }
    for (int e = 0; e < n; ++e) {
        if (v->wb == 4) reinterpret_cast<uint32_t *>(tgt.data())[e] = (uint32_t)outputs[e];
        else reinterpret_cast<uint64_t *>(tgt.data())[e] = outputs[e];
    }
    auto bad = [&](int code) {
        simba_vfb_destroy(v);
        return code;
    };
    if (cudaStreamCreateWithFlags(&v->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaMalloc(&v->var, var.size()) != cudaSuccess || cudaMalloc(&v->tgt, tgt.size()) != cudaSuccess ||
        cudaMalloc(&v->slot_of, kVfbBatch * 4) != cudaSuccess ||
        cudaMalloc(&v->tile_cnt, (kVfbBatch / kVfbTile + 1) * 4) != cudaSuccess ||
        cudaMalloc(&v->ctl, sizeof(VfbCtl)) != cudaSuccess ||
        cudaMallocHost(&v->h_ctl, sizeof(VfbCtl)) != cudaSuccess) {
        cudaGetLastError();
        return bad(fail(SIMBA_ENOMEM, "device allocation failed"));
    }
    if (cudaMemcpy(v->var, var.data(), var.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(v->tgt, tgt.data(), tgt.size(), cudaMemcpyHostToDevice) != cudaSuccess)
        return bad(fail(SIMBA_ECUDA, "copy of the examples failed"));
    *out = v;
    return SIMBA_OK;
}

int simba_vfb_level(simba_vfb *v, int size, double time_budget_s, simba_vfb_row *out)
{
    if (!v || !out)
        return fail(SIMBA_EINVAL, "null argument");
    if (v->ended)
        return fail(SIMBA_EINVAL, "the run already ended (found / oom / timed out)");
    if (size != v->last_size + 1 || size > SIMBA_MAX_SIZE)
        return fail(SIMBA_EINVAL, "sizes run in order 1, 2, ... <= %d (next is %d, got %d)", SIMBA_MAX_SIZE,
                    v->last_size + 1, size);
    CK(cudaSetDevice(v->device));
    return v->wb == 4 ? vfb_level<uint32_t>(v, size, time_budget_s, out)
                      : vfb_level<uint64_t>(v, size, time_budget_s, out);
}

int simba_vfb_tokens(simba_vfb *v, uint64_t cand, int32_t *tokens, int cap, int *len)
{
    if (!v || !tokens || !len)
        return fail(SIMBA_EINVAL, "null argument");
    const int s = v->last_size;
    if (s < 1)
        return fail(SIMBA_EINVAL, "no size has run");
    CK(cudaSetDevice(v->device));
    // decode the candidate against the block list of the last size
    const VfbBlocks &bl = v->bl;
    int i = 0;
    while (i + 1 < bl.nb && bl.b[i + 1].base <= cand)
        ++i;
    if (bl.nb == 0 || cand < bl.b[0].base)
        return fail(SIMBA_ERANGE, "candidate %llu outside the last size", (unsigned long long)cand);
    const VfbBlock &B = bl.b[i];
    const uint64_t local = cand - B.base;
    std::vector<int32_t> t;
    if (B.op == VOP_VAR) {
        t.push_back((int32_t)local);
    } else if (B.op == 0 || B.op == 4) {
        if (int e = vfb_entry_tokens(v, B.loff + local, t))
            return e;
        t.push_back(-(B.op + 1));
    } else {
        const uint64_t l = local / B.rcnt, r = local - l * B.rcnt;
        if (int e = vfb_entry_tokens(v, B.loff + l, t))
            return e;
        if (int e = vfb_entry_tokens(v, B.roff + r, t))
            return e;
        t.push_back(-(B.op + 1));
    }
    if ((int)t.size() > cap)
        return fail(SIMBA_ERANGE, "expression of %zu tokens exceeds the buffer (%d)", t.size(), cap);
    std::copy(t.begin(), t.end(), tokens);
    *len = (int)t.size();
    return SIMBA_OK;
}

void simba_vfb_destroy(simba_vfb *v)
{
    if (!v)
        return;
    cudaSetDevice(v->device);
    if (v->stream)
        cudaStreamSynchronize(v->stream);
    cudaFree(v->beh), cudaFree(v->var), cudaFree(v->tgt), cudaFree(v->m_l), cudaFree(v->m_r), cudaFree(v->m_op);
    cudaFree(v->H), cudaFree(v->slot_of), cudaFree(v->tile_cnt), cudaFree(v->ctl);
    if (v->h_ctl)
        cudaFreeHost(v->h_ctl);
    if (v->stream)
        cudaStreamDestroy(v->stream);
    delete v;
}

}  // extern "C"
