// build.cu -- S1..S8 of the block-based triangle-counting path on the GPU.
//
//   S1 canonicalise   (§5.1; DESIGN R1, R2)
//   S2 degree order   (§5.4; DESIGN R3)
//   S3 orient         (§5.4; DESIGN R4)
//   S4 conformal cuts (§4.3; DESIGN R7)
//   S5 block CSR      (§4.3.1-4.3.2)
//   S6 block triples  (Listing 5; DESIGN R5, R6)
//   S7 task costs     (§4.4; DESIGN R17, R19)
//   S8 pieces + LPT   (§4.1; DESIGN R18)
//
// Pre-processing is untimed in the paper's protocol, but it
// runs on the device anyway: 64-bit radix sorts of up to 2^31 keys (C5) are
// far too slow on the host.  All arithmetic is integer.
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <map>
#include <numeric>
#include <queue>
#include <set>

#include "internal.h"

namespace pgabb {

namespace {

constexpr int kThreads = 256;
#ifndef PGABB_LIGHT_SORT_WINDOW
#define PGABB_LIGHT_SORT_WINDOW 4096
#endif
constexpr uint32_t kLightSortWindow = PGABB_LIGHT_SORT_WINDOW;   // light items re-ordered by work within it

inline unsigned grid_for(uint64_t work, int threads = kThreads) {
    uint64_t g = (work + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > (1u << 20)) g = 1u << 20;   // grid-stride beyond this
    return (unsigned)g;
}

inline int bits_for(uint64_t x) {
    int b = 0;
    while (b < 64 && (x >> b) != 0) ++b;
    return b;
}

constexpr int kMaxSlots = 4;                       // streaming arena slots (block cache depth)
constexpr uint64_t kUploadChunk = 1ull << 27;   // host tuples per staging chunk (1 GiB of u32 pairs)
constexpr uint64_t kMidSaving = 2;   // R25 auto: saved streamed ids per visit needed for MID

struct CutsArg {
    uint32_t c[kMaxParts + 1];
    int p;
};

__device__ __forceinline__ int part_of(const CutsArg& cu, uint32_t r) {
    // the j with cut_j <= r < cut_{j+1}: (number of cuts <= r) - 1
    int lo = 0, hi = cu.p + 1;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (cu.c[mid] <= r) lo = mid + 1; else hi = mid;
    }
    return lo - 1;
}

__global__ void k_check_ids(const uint32_t* s, const uint32_t* d, uint64_t m, uint32_t n, int* bad) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < m;
         k += (uint64_t)gridDim.x * blockDim.x)
        if (s[k] >= n || d[k] >= n) *bad = 1;
}

// S1: key = (min << B) | max, self-loops -> sentinel (all ones in 2B bits, never a
// real key because a real key has min < max).
__global__ void k_make_keys(const uint32_t* s, const uint32_t* d, uint64_t m, int B, uint64_t sent,
                            uint64_t* keys) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < m;
         k += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t a = s[k], b = d[k];
        uint32_t lo = min(a, b), hi = max(a, b);
        keys[k] = (a == b) ? sent : (((uint64_t)lo << B) | hi);
    }
}

// S2: degree of every id over the unique undirected edges.
__global__ void k_degree(const uint64_t* keys, uint64_t mE, int B, uint32_t* deg) {
    const uint64_t mask = (1ull << B) - 1;
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < mE;
         k += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t key = keys[k];
        atomicAdd(&deg[key >> B], 1u);
        atomicAdd(&deg[key & mask], 1u);
    }
}

__global__ void k_iota(uint32_t* a, uint32_t n) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n;
         k += (uint64_t)gridDim.x * blockDim.x)
        a[k] = (uint32_t)k;
}

__global__ void k_scatter_rank(const uint32_t* order, uint32_t n, uint32_t* rank, int reverse) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n;
         k += (uint64_t)gridDim.x * blockDim.x)
        rank[order[k]] = reverse ? n - 1 - (uint32_t)k : (uint32_t)k;
}

// S3: relabel to rank space and orient low -> high.
__global__ void k_orient(uint64_t* keys, uint64_t mE, int B, const uint32_t* rank) {
    const uint64_t mask = (1ull << B) - 1;
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < mE;
         k += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t key = keys[k];
        uint32_t ra = rank[key >> B], rb = rank[key & mask];
        keys[k] = ((uint64_t)min(ra, rb) << B) | max(ra, rb);
    }
}

__global__ void k_dag_degrees(const uint64_t* dag, uint64_t mE, int B, uint32_t* dplus, uint32_t* dminus) {
    const uint64_t mask = (1ull << B) - 1;
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < mE;
         k += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t key = dag[k];
        atomicAdd(&dplus[key >> B], 1u);
        atomicAdd(&dminus[key & mask], 1u);
    }
}

// S4 weights: rule 0 w = d+ + d- * d+, rule 1 w = d+; also wedges d- * d+.
__global__ void k_cut_weights(const uint32_t* dplus, const uint32_t* dminus, uint32_t n, int rule,
                              unsigned long long* w, unsigned long long* wedges) {
    unsigned long long acc = 0;
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n;
         k += (uint64_t)gridDim.x * blockDim.x) {
        unsigned long long dp = dplus[k], dm = dminus[k];
        // R7: 0 estimated LOW work d+ + d-d+, 1 out-degree d+, 2 degree d+ + d-,
        // 3 estimated MID work d+ + C(d+, 2) (R25: the ids streamed for u's lists)
        w[k] = rule == 0 ? dp + dm * dp : rule == 1 ? dp : rule == 2 ? dp + dm : dp + dp * (dp - (dp > 0)) / 2;
        acc += dm * dp;
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(wedges, acc);
}

// cut_j = min { c in [0, n] : p * P[c] >= j * P[n] },  P[0] = 0 (prefix of w).
__global__ void k_cuts(const unsigned long long* P, uint32_t n, int p, uint32_t* cuts) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j > p) return;
    if (j == 0) { cuts[0] = 0; return; }
    if (j == p) { cuts[p] = n; return; }
    const unsigned __int128 tgt = (unsigned __int128)j * P[n];
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        uint32_t mid = lo + ((hi - lo) >> 1);
        if ((unsigned __int128)p * P[mid] >= tgt) hi = mid; else lo = mid + 1;
    }
    cuts[j] = lo;
}

// S5: block id of each DAG edge.
__global__ void k_block_ids(const uint64_t* dag, uint64_t mE, int B, CutsArg cu, uint32_t* bid) {
    const uint64_t mask = (1ull << B) - 1;
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < mE;
         k += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t key = dag[k];
        int i = part_of(cu, (uint32_t)(key >> B));
        int j = part_of(cu, (uint32_t)(key & mask));
        bid[k] = (uint32_t)(i * cu.p + j);
    }
}

// off[b] = first position of block b in the block-sorted edge array.
__global__ void k_block_offsets(const uint32_t* bid, uint64_t mE, uint32_t nb, unsigned long long* off) {
    uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b > nb) return;
    uint64_t lo = 0, hi = mE;
    while (lo < hi) {
        uint64_t mid = lo + ((hi - lo) >> 1);
        if (bid[mid] < b) lo = mid + 1; else hi = mid;
    }
    off[b] = lo;
}

// col pool: local col id (c - cut_j) in block-major order.
__global__ void k_local_cols(const uint64_t* dag, const uint32_t* bid, uint64_t mE, int B, CutsArg cu,
                             uint32_t* col) {
    const uint64_t mask = (1ull << B) - 1;
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < mE;
         k += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t j = bid[k] % cu.p;
        col[k] = (uint32_t)(dag[k] & mask) - cu.c[j];
    }
}

struct BlockDev {
    unsigned long long col_off, nnz, rp_off;
    uint32_t nrows, row_base;   // row_base = cut_i
};

// rowptr pool: for entry t of block b, rowptr[t] = #edges of b with local row < lr.
__global__ void k_rowptr(const uint64_t* dag, int B, const BlockDev* blk, const unsigned long long* rp_start,
                         int nblk, unsigned long long total, uint32_t* rowptr) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
         t += (uint64_t)gridDim.x * blockDim.x) {
        int lo = 0, hi = nblk;   // last block with rp_start <= t
        while (hi - lo > 1) {
            int mid = (lo + hi) >> 1;
            if (rp_start[mid] <= t) lo = mid; else hi = mid;
        }
        const BlockDev bd = blk[lo];
        const uint32_t lr = (uint32_t)(t - rp_start[lo]);
        const uint64_t target = (uint64_t)bd.row_base + lr;   // global row
        uint64_t a = 0, z = bd.nnz;
        const uint64_t* e = dag + bd.col_off;
        while (a < z) {
            uint64_t mid = a + ((z - a) >> 1);
            if ((e[mid] >> B) < target) a = mid + 1; else z = mid;
        }
        rowptr[t] = (uint32_t)a;
    }
}

// S7: per-task cost and staged-model elements, one thread per edge of a
// non-empty block; the x-loop visits every task (i,j,x) of the edge's block.
struct CostArg {
    const uint64_t* dag;
    const uint32_t* col;
    const uint32_t* rowptr;
    const BlockDev* blk;          // indexed by block id i*p+j
    const uint32_t* tid;          // p^3
    int B, p;
    CutsArg cu;
    unsigned long long mE;
    unsigned long long* cost;
    unsigned long long* alg_bytes;
};

// Launched per non-empty block (i, j): every lane of a warp shares the block, so
// the x-loop is warp-uniform and each (warp, task) adds one warp-reduced sum.
__global__ void k_task_costs(CostArg a, int i, int j) {
    const BlockDev bij = a.blk[i * a.p + j];
    const int lane = threadIdx.x & 31;
    const uint64_t warp0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) - lane;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t base = warp0; base < bij.nnz; base += stride) {
        const uint64_t k = bij.col_off + base + lane;
        const bool ok = base + lane < bij.nnz;
        uint32_t u = 0, v = 0;
        bool first = false;
        if (ok) {
            const uint32_t r = (uint32_t)(a.dag[k] >> a.B);
            u = r - a.cu.c[i];
            v = a.col[k];
            first = (k == bij.col_off) || ((uint32_t)(a.dag[k - 1] >> a.B) != r);
        }
        for (int x = j; x < a.p; ++x) {
            const uint32_t t = a.tid[(i * a.p + j) * a.p + x];
            if (t == kNoTask) continue;
            uint32_t c = 0;
            unsigned long long by = 0;
            if (ok) {
                const BlockDev bix = a.blk[i * a.p + x], bjx = a.blk[j * a.p + x];
                const uint32_t la = a.rowptr[bix.rp_off + u + 1] - a.rowptr[bix.rp_off + u];
                const uint32_t lb = a.rowptr[bjx.rp_off + v + 1] - a.rowptr[bjx.rp_off + v];
                c = la + lb;
                // staged model (DESIGN R19): only rows with A_ix[u] non-empty move bytes
                if (la) by = 4ull * (lb + (first ? la : 0u)) + 12ull;
            }
            c = __reduce_add_sync(0xffffffffu, c);
            for (int o = 16; o > 0; o >>= 1) by += __shfl_down_sync(0xffffffffu, by, o);
            if (lane == 0) {
                atomicAdd(&a.cost[t], (unsigned long long)c);
                atomicAdd(&a.alg_bytes[t], by);
            }
        }
    }
}

// ---- S5c transposes (DESIGN R25, MID orientation), one block at a time -------
// key = local col v, value = block-local position e of the edge.
__global__ void k_tkeys(const uint32_t* col, uint64_t nnz, uint32_t* key, uint32_t* val) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < nnz;
         k += (uint64_t)gridDim.x * blockDim.x) {
        key[k] = col[k];
        val[k] = (uint32_t)k;
    }
}

// after the stable sort by v: tpos[q] = e, tcol[q] = the local row u of edge e.
__global__ void k_tfill(const uint64_t* dag, uint64_t nnz, int B, uint32_t row_base, const uint32_t* val,
                        uint32_t* tcol, uint32_t* tpos) {
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < nnz;
         q += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t e = val[q];
        tcol[q] = (uint32_t)(dag[e] >> B) - row_base;
        tpos[q] = e;
    }
}

// transposed rowptr: trp[t] = number of entries with local col < t, t = 0..ncols.
__global__ void k_trowptr(const uint32_t* key, uint64_t nnz, uint32_t ncols, uint32_t* trp) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t <= ncols;
         t += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t a = 0, z = nnz;
        while (a < z) {
            const uint64_t mid = a + ((z - a) >> 1);
            if (key[mid] < t) a = mid + 1; else z = mid;
        }
        trp[t] = (uint32_t)a;
    }
}

// S7 for the MID orientation (R25), one thread per entry of the transpose of a
// non-empty block (i, j) (warp-uniform x-loop as k_task_costs): entry (v, u, e);
// s = |{w in A_ix[u] : w > v}| (= |A_ix[u]| when x > j, the suffix after e when
// x == j); the column's first entry also adds the held |A_jx[v]|.
struct CostMidArg {
    const uint32_t* col;          // col pool (the tcol / tpos regions at tcol_base / tpos_base)
    const uint32_t* rowptr;
    const BlockDev* blk;          // indexed by block id i*p+j
    const uint32_t* tid;          // p^3
    int p;
    unsigned long long tcol_base, tpos_base;
    unsigned long long *cost, *alg_bytes, *s_low, *s_mid;
};
__global__ void k_task_costs_mid(CostMidArg a, int i, int j) {
    const BlockDev bij = a.blk[i * a.p + j];
    const int lane = threadIdx.x & 31;
    const uint64_t warp0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) - lane;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t base = warp0; base < bij.nnz; base += stride) {
        const uint64_t q = bij.col_off + base + lane;
        const bool ok = base + lane < bij.nnz;
        uint32_t u = 0, v = 0, e = 0;
        bool first = false;
        if (ok) {
            u = a.col[a.tcol_base + q];
            e = a.col[a.tpos_base + q];
            v = a.col[bij.col_off + e];
            first = (q == bij.col_off) || (a.col[bij.col_off + a.col[a.tpos_base + q - 1]] != v);
        }
        for (int x = j; x < a.p; ++x) {
            const uint32_t t = a.tid[(i * a.p + j) * a.p + x];
            if (t == kNoTask) continue;
            unsigned long long c = 0, by = 0, sl = 0, sm = 0;
            if (ok) {
                const BlockDev bix = a.blk[i * a.p + x], bjx = a.blk[j * a.p + x];
                const uint32_t lb = a.rowptr[bjx.rp_off + v + 1] - a.rowptr[bjx.rp_off + v];
                const uint32_t s = (x == j) ? a.rowptr[bij.rp_off + u + 1] - (e + 1)
                                            : a.rowptr[bix.rp_off + u + 1] - a.rowptr[bix.rp_off + u];
                c = s + (first ? lb : 0u);
                if (lb) by = 4ull * (s + (first ? lb : 0u)) + 12ull;
                sl = lb;
                sm = s;
            }
            for (int o = 16; o > 0; o >>= 1) {
                c += __shfl_down_sync(0xffffffffu, c, o);
                by += __shfl_down_sync(0xffffffffu, by, o);
                sl += __shfl_down_sync(0xffffffffu, sl, o);
                sm += __shfl_down_sync(0xffffffffu, sm, o);
            }
            if (lane == 0) {
                atomicAdd(&a.cost[t], c);
                atomicAdd(&a.alg_bytes[t], by);
                atomicAdd(&a.s_low[t], sl);
                atomicAdd(&a.s_mid[t], sm);
            }
        }
    }
}

// S8 helper for a MID task: rowcost(v) over the rows v of part j (R25).
__global__ void k_row_costs_mid(const uint32_t* col, const uint32_t* rowptr, uint64_t tcol_base, uint64_t tpos_base,
                                BlockDev bij, uint64_t trp_ij, uint32_t ncols, BlockDev bix, BlockDev bjx, int same,
                                unsigned long long* rc) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < ncols;
         v += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t q0 = rowptr[trp_ij + v], q1 = rowptr[trp_ij + v + 1];
        unsigned long long s = 0;
        if (q1 > q0) s = rowptr[bjx.rp_off + v + 1] - rowptr[bjx.rp_off + v];
        for (uint32_t q = q0; q < q1; ++q) {
            const uint32_t u = col[tcol_base + bij.col_off + q];
            const uint32_t e = col[tpos_base + bij.col_off + q];
            s += same ? rowptr[bij.rp_off + u + 1] - (e + 1) : rowptr[bix.rp_off + u + 1] - rowptr[bix.rp_off + u];
        }
        rc[v + 1] = s;
    }
}

// S8 helper: row costs of one task (for splitting heavy tasks into pieces).
__global__ void k_row_costs(const uint32_t* col, const uint32_t* rowptr, BlockDev bij, BlockDev bix,
                            BlockDev bjx, unsigned long long* rc) {
    for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < bij.nrows;
         u += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t e0 = rowptr[bij.rp_off + u], e1 = rowptr[bij.rp_off + u + 1];
        const uint32_t la = rowptr[bix.rp_off + u + 1] - rowptr[bix.rp_off + u];
        unsigned long long s = 0;
        for (uint32_t e = e0; e < e1; ++e) {
            const uint32_t v = col[bij.col_off + e];
            s += la + (rowptr[bjx.rp_off + v + 1] - rowptr[bjx.rp_off + v]);
        }
        rc[u + 1] = s;
    }
}

// Dense copy of one block: row r's bits over the column part, one thread per row
// (each row's words are owned by one thread, so no atomics).
__global__ void k_fill_bitmap(const uint32_t* col, const uint32_t* rowptr, unsigned long long col_off,
                              unsigned long long rp_off, uint32_t nrows, uint32_t words, uint32_t* bm) {
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < nrows;
         r += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t* row = bm + r * words;
        for (uint32_t k = 0; k < words; ++k) row[k] = 0u;
        const uint32_t e0 = rowptr[rp_off + r], e1 = rowptr[rp_off + r + 1];
        for (uint32_t e = e0; e < e1; ++e) {
            const uint32_t c = col[col_off + e];
            row[c >> 5] |= 1u << (c & 31);
        }
    }
}

#ifndef PGABB_ELL
#define PGABB_ELL 1
#endif
constexpr bool kEll = PGABB_ELL;
// R30: the sector-aligned copy of a short-list block -- row r's slot of ew words is
// [|row|, first ew-1 ids, 0 ...] at ell + r * ew (64-byte aligned for ew = 16), so a
// thread reads one aligned segment per pair instead of a rowptr sector and 1-2 list
// sectors; longer rows continue in the col pool after their first ew-1 ids.
__global__ void k_fill_ell(const uint32_t* col, const uint32_t* rowptr, uint64_t col_off, uint64_t rp_off,
                           uint32_t nrows, uint32_t ew, uint32_t* ell) {
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < nrows;
         r += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t e0 = rowptr[rp_off + r], e1 = rowptr[rp_off + r + 1];
        uint32_t* slot = ell + r * ew;
        slot[0] = e1 - e0;
        for (uint32_t q = 1; q < ew; ++q) slot[q] = (e0 + q - 1 < e1) ? col[col_off + e0 + q - 1] : 0u;
    }
}

// Row items of one owned piece, in kernel roles (TaskDev, R25): rows r in [r0, r1)
// with a non-empty held list S and neighbour list, classified by their work
// (DESIGN R20): LIGHT rows -- |S| <= kLightLa, <= kLightLe neighbours and at most
// kLightWork list loads for the thread-per-row kernel (a streamed list of <=
// kLightScan ids is scanned, a longer one binary-searched per element of S; a
// dense streamed block costs one bit test per element) -- get lf = 1; every other
// row gets hf = its number of heavy items (neighbour chunks, warp per item).
// hf[nrows] = lf[nrows] = 0 for the exclusive scans.
// alg (nullable): += staged-model bytes of the light rows (DESIGN R19/R25), for
// the per-kernel roofline.
__device__ __forceinline__ uint32_t streamed_len(const TaskDev& T, const uint32_t* col, const uint32_t* rowptr,
                                                 uint32_t e) {
    const uint32_t nb = col[T.n_col + e];
    const uint32_t end = rowptr[T.t_rp + nb + 1];
    const uint32_t beg = T.n_pos != ~0ull ? col[T.n_pos + e] + 1 : rowptr[T.t_rp + nb];
    return end - beg;
}

// held_max: kLightLa, or kMedLa when medium rows (kLightLa < |S| <= kMedLa, R29) get
// mf = 1 for the second thread-per-row kernel instead of heavy items.
#ifndef PGABB_MED_LONG
#define PGABB_MED_LONG 0
#endif
constexpr bool kMedLong = PGABB_MED_LONG;   // medium rows may binary-search long lists (A/B)
__global__ void k_row_flags(PieceDev w, const TaskDev* tasks, const uint32_t* col, const uint32_t* rowptr,
                            uint32_t* hf, uint32_t* lf, uint32_t* mf, uint32_t held_max, unsigned long long* alg) {
    const TaskDev T = tasks[w.task];
    const uint32_t nr = w.r1 - w.r0;
    for (uint64_t k0 = blockIdx.x * (uint64_t)blockDim.x; k0 <= nr; k0 += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t k = k0 + threadIdx.x;
        uint32_t fh = 0, fl = 0, fm = 0;
        unsigned long long bytes = 0;
        if (k < nr) {
            const uint32_t r = w.r0 + (uint32_t)k;
            const uint32_t e0 = rowptr[T.n_rp + r], e1 = rowptr[T.n_rp + r + 1];
            const uint32_t la = rowptr[T.s_rp + r + 1] - rowptr[T.s_rp + r];
            if (e1 > e0 && la > 0) {
                bool light = la <= held_max && e1 - e0 <= kLightLe;
                if (light) {
                    uint32_t work = 0, lsum = 0, lmax = 0;
                    for (uint32_t e = e0; e < e1; ++e) {
                        const uint32_t lb = streamed_len(T, col, rowptr, e);
                        work += light_pair_loads(la, lb);
                        lsum += lb;
                        lmax = max(lmax, lb);
                    }
                    light = T.t_bm != ~0ull || work <= kLightWork;
                    // a medium row only when every streamed list is a short scanned list (no
                    // per-id binary searches, no dense block: R-MAT rows against hub lists
                    // or bitmaps stay heavy warp items, R29)
                    if (la > kLightLa && (T.t_bm != ~0ull || (!kMedLong && lmax > kLightScan))) light = false;
                    bytes = 4ull * (la + lsum) + 12ull * (e1 - e0);
                }
                fl = light && la <= kLightLa;
                fm = light && la > kLightLa;
                fh = light ? 0u : heavy_chunks(e1 - e0);
                if (!light) bytes = 0;
            }
        }
        if (k <= nr) {
            hf[k] = fh;
            lf[k] = fl;
            mf[k] = fm;
        }
        if (alg) {
            for (int o = 16; o > 0; o >>= 1) bytes += __shfl_down_sync(0xffffffffu, bytes, o);
            if ((threadIdx.x & 31) == 0 && bytes) atomicAdd(alg, bytes);
        }
    }
}

__global__ void k_row_emit(PieceDev w, const uint32_t* nchunks, const uint32_t* pos, unsigned long long* out) {
    const uint32_t nr = w.r1 - w.r0;
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < nr;
         k += (uint64_t)gridDim.x * blockDim.x)
        for (uint32_t c = 0; c < nchunks[k]; ++c)
            out[pos[k] + c] = ((unsigned long long)w.task << 48) | ((unsigned long long)c << 32) | (w.r0 + (uint32_t)k);
}

// Light items of one owned piece (16 bytes each, see internal.h), and each item's
// sort key: its window of kLightSortWindow items (row order, for L2 locality) then
// its work (neighbour count + list loads), so that a warp's 32 lanes (32
// consecutive items) get items of similar work -- the loops of the light kernel
// run as long as the warp's longest item.
__global__ void k_light_emit(PieceDev w, const TaskDev* tasks, const uint32_t* flags, const uint32_t* pos,
                             const uint32_t* col, const uint32_t* rowptr, uint4* out, uint32_t* key) {
    const TaskDev T = tasks[w.task];
    const uint32_t nr = w.r1 - w.r0;
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < nr;
         k += (uint64_t)gridDim.x * blockDim.x)
        if (flags[k]) {
            const uint32_t r = w.r0 + (uint32_t)k;
            const uint32_t a0 = rowptr[T.s_rp + r], la = rowptr[T.s_rp + r + 1] - a0;
            const uint32_t e0 = rowptr[T.n_rp + r], le = rowptr[T.n_rp + r + 1] - e0;
            out[pos[k]] = make_uint4(w.task | (la << kLightTaskBits) | (le << (kLightTaskBits + 4)), a0, e0, r);
            uint32_t work = le;
            for (uint32_t e = e0; e < e0 + le; ++e)
                work += T.t_bm != ~0ull ? la : light_pair_loads(la, streamed_len(T, col, rowptr, e));
            key[pos[k]] = (pos[k] / kLightSortWindow) << 8 | min(work, 255u);
        }
}

template <class F>
void cub_call(F f, cudaStream_t st, DBuf<unsigned char>& tmp) {
    size_t bytes = 0;
    PG_CK(f(nullptr, bytes));
    if (bytes > tmp.bytes()) tmp.alloc(bytes);
    PG_CK(f(tmp.p, bytes));
    (void)st;
}

BlockDev to_dev(const BlockInfo& b, uint32_t row_base) {
    BlockDev d;
    d.col_off = b.col_off;
    d.nnz = b.nnz;
    d.rp_off = b.rp_off;
    d.nrows = b.nrows;
    d.row_base = row_base;
    return d;
}

}  // namespace

void build_graph(pgabb_blocks_s* h, uint64_t m, const uint32_t* src, const uint32_t* dst, bool on_device) {
    cudaStream_t st = h->stream;
    const uint32_t n = h->n;
    const int B = std::max(1, bits_for(n > 0 ? n - 1 : 0));
    const uint64_t sent = (B >= 32) ? ~0ull : ((1ull << (2 * B)) - 1);
    DBuf<unsigned char> tmp;

    h->d_rank.alloc(std::max<uint32_t>(n, 1));
    if (m == 0 || n == 0) {
        h->m_edges = 0;
        h->p = 1;
        h->cuts = {0, n};
        h->blocks.assign(1, BlockInfo{});
        h->blocks[0].nrows = n;
        h->d_deg.alloc(std::max<uint32_t>(n, 1));
        PG_CK(cudaMemsetAsync(h->d_deg.p, 0, (size_t)std::max<uint32_t>(n, 1) * 4, st));
        if (n) {
            k_iota<<<grid_for(n), kThreads, 0, st>>>(h->d_rank.p, n);
            if (h->reverse_order) {   // all degrees 0: the (deg, id) order is the id order
                k_scatter_rank<<<grid_for(n), kThreads, 0, st>>>(h->d_rank.p, n, h->d_rank.p, 1);
            }
            PG_LAUNCH_CHECK();
        }
        PG_CK(cudaStreamSynchronize(st));
        return;
    }

    // ---- upload + validate + S1 canonicalise ----------------------------------
    // Host tuples go up in chunks through a staging buffer and become keys on the
    // way, so the build never holds the raw tuples and both key buffers at once.
    // device tuples may still be in flight on the caller's streams (a producer
    // kernel, a copy): the build reads them on the handle's non-blocking stream,
    // which no caller stream orders against, so wait for all device work first
    if (on_device) PG_CK(cudaDeviceSynchronize());
    DBuf<uint64_t> keys, keys2;
    keys.alloc(m);
    {
        DBuf<int> d_bad;
        d_bad.alloc(1);
        PG_CK(cudaMemsetAsync(d_bad.p, 0, 4, st));
        const uint64_t chunk = on_device ? m : std::min<uint64_t>(m, kUploadChunk);
        DBuf<uint32_t> d_s, d_d;
        if (!on_device) {
            d_s.alloc(chunk);
            d_d.alloc(chunk);
        }
        for (uint64_t c0 = 0; c0 < m; c0 += chunk) {
            const uint64_t cn = std::min(chunk, m - c0);
            const uint32_t *s = src + c0, *d = dst + c0;
            if (!on_device) {
                PG_CK(cudaMemcpyAsync(d_s.p, s, cn * 4, cudaMemcpyHostToDevice, st));
                PG_CK(cudaMemcpyAsync(d_d.p, d, cn * 4, cudaMemcpyHostToDevice, st));
                s = d_s.p;
                d = d_d.p;
            }
            k_check_ids<<<grid_for(cn), kThreads, 0, st>>>(s, d, cn, n, d_bad.p);
            PG_LAUNCH_CHECK();
            k_make_keys<<<grid_for(cn), kThreads, 0, st>>>(s, d, cn, B, sent, keys.p + c0);
            PG_LAUNCH_CHECK();
            if (!on_device) PG_CK(cudaStreamSynchronize(st));   // the staging buffer is reused
        }
        int bad = 0;
        PG_CK(cudaMemcpyAsync(&bad, d_bad.p, 4, cudaMemcpyDeviceToHost, st));
        PG_CK(cudaStreamSynchronize(st));
        if (bad) fail(PGABB_EINVAL, "vertex id >= n in the input tuples");
    }
    keys2.alloc(m);
    const int kbits = std::min(64, 2 * B);
    {   // DoubleBuffer sort: O(P) temporary storage instead of another m keys
        cub::DoubleBuffer<uint64_t> db(keys.p, keys2.p);
        cub_call([&](void* t, size_t& b) {
            return cub::DeviceRadixSort::SortKeys(t, b, db, (int64_t)m, 0, kbits, st);
        }, st, tmp);
        if (db.Current() != keys2.p) {   // sorted keys in keys2
            std::swap(keys.p, keys2.p);
            std::swap(keys.n, keys2.n);
        }
    }
    DBuf<unsigned long long> d_cnt;
    d_cnt.alloc(2);
    cub_call([&](void* t, size_t& b) {
        return cub::DeviceSelect::Unique(t, b, keys2.p, keys.p, d_cnt.p, (int64_t)m, st);
    }, st, tmp);
    unsigned long long nuniq = 0;
    PG_CK(cudaMemcpyAsync(&nuniq, d_cnt.p, 8, cudaMemcpyDeviceToHost, st));
    PG_CK(cudaStreamSynchronize(st));
    uint64_t mE = nuniq;
    if (mE) {
        uint64_t last = 0;
        PG_COPY_SYNC(&last, keys.p + (mE - 1), 8, st);
        if (last == sent) --mE;
    }
    // |E| is 64-bit throughout (pool offsets, work lists); only a single block's
    // edges are indexed in 32 bits (checked in S5)
    h->m_edges = mE;
    keys2.release();

    // ---- S2 degree + rank ---------------------------------------------------
    {
        DBuf<uint32_t> deg, deg2, ids, order;
        deg.alloc(n);
        deg2.alloc(n);
        ids.alloc(n);
        order.alloc(n);
        PG_CK(cudaMemsetAsync(deg.p, 0, (size_t)n * 4, st));
        if (mE) {
            k_degree<<<grid_for(mE), kThreads, 0, st>>>(keys.p, mE, B, deg.p);
            PG_LAUNCH_CHECK();
        }
        k_iota<<<grid_for(n), kThreads, 0, st>>>(ids.p, n);
        PG_LAUNCH_CHECK();
        // stable radix sort by degree: ties keep id order (DESIGN R3)
        cub_call([&](void* t, size_t& b) {
            return cub::DeviceRadixSort::SortPairs(t, b, deg.p, deg2.p, ids.p, order.p, (int64_t)n, 0, 32, st);
        }, st, tmp);
        k_scatter_rank<<<grid_for(n), kThreads, 0, st>>>(order.p, n, h->d_rank.p, (int)h->reverse_order);
        PG_LAUNCH_CHECK();
        PG_CK(cudaStreamSynchronize(st));
        // deg(v) stays with the handle (local clustering coefficient, NEXT-1)
        h->d_deg.release();
        std::swap(h->d_deg.p, deg.p);
        std::swap(h->d_deg.n, deg.n);
    }

    // ---- S3 orient + relabel ------------------------------------------------
    keys2.alloc(std::max<uint64_t>(mE, 1));
    if (mE) {
        k_orient<<<grid_for(mE), kThreads, 0, st>>>(keys.p, mE, B, h->d_rank.p);
        PG_LAUNCH_CHECK();
        cub::DoubleBuffer<uint64_t> db(keys.p, keys2.p);
        cub_call([&](void* t, size_t& b) {
            return cub::DeviceRadixSort::SortKeys(t, b, db, (int64_t)mE, 0, kbits, st);
        }, st, tmp);
        if (db.Current() != keys2.p) {
            std::swap(keys.p, keys2.p);
            std::swap(keys.n, keys2.n);
        }
    }
    keys.release();
    uint64_t* dag = keys2.p;   // DAG edges sorted by (row, col) in rank space

    // ---- S4 cuts ------------------------------------------------------------
    const uint32_t p = h->p;
    CutsArg cu{};
    cu.p = (int)p;
    {
        DBuf<uint32_t> dplus, dminus, d_cuts;
        DBuf<unsigned long long> w, P, d_w;
        dplus.alloc(n);
        dminus.alloc(n);
        w.alloc(n);
        P.alloc((size_t)n + 1);
        d_w.alloc(1);
        d_cuts.alloc(p + 1);
        PG_CK(cudaMemsetAsync(dplus.p, 0, (size_t)n * 4, st));
        PG_CK(cudaMemsetAsync(dminus.p, 0, (size_t)n * 4, st));
        PG_CK(cudaMemsetAsync(d_w.p, 0, 8, st));
        PG_CK(cudaMemsetAsync(P.p, 0, 8, st));
        if (mE) {
            k_dag_degrees<<<grid_for(mE), kThreads, 0, st>>>(dag, mE, B, dplus.p, dminus.p);
            PG_LAUNCH_CHECK();
        }
        k_cut_weights<<<grid_for(n), kThreads, 0, st>>>(dplus.p, dminus.p, n, (int)h->cut_rule, w.p, d_w.p);
        PG_LAUNCH_CHECK();
        cub_call([&](void* t, size_t& b) {
            return cub::DeviceScan::InclusiveSum(t, b, w.p, P.p + 1, (int64_t)n, st);
        }, st, tmp);
        k_cuts<<<1, 128, 0, st>>>(P.p, n, (int)p, d_cuts.p);
        PG_LAUNCH_CHECK();
        h->cuts.resize(p + 1);
        PG_CK(cudaMemcpyAsync(h->cuts.data(), d_cuts.p, (p + 1) * 4, cudaMemcpyDeviceToHost, st));
        unsigned long long W = 0;
        PG_CK(cudaMemcpyAsync(&W, d_w.p, 8, cudaMemcpyDeviceToHost, st));
        PG_CK(cudaStreamSynchronize(st));
        h->wedges = W;
    }
    for (uint32_t k = 0; k <= p; ++k) cu.c[k] = h->cuts[k];

    // ---- S5 block CSR -------------------------------------------------------
    const uint32_t nb = p * p;
    std::vector<unsigned long long> off(nb + 1, 0);
    if (mE) {
        DBuf<uint32_t> bid, bid2;
        DBuf<uint64_t> dag2;
        bid.alloc(mE);
        bid2.alloc(mE);
        dag2.alloc(mE);
        k_block_ids<<<grid_for(mE), kThreads, 0, st>>>(dag, mE, B, cu, bid.p);
        PG_LAUNCH_CHECK();
        const int bbits = std::max(1, bits_for(nb - 1));
        {   // stable: (row, col) order kept inside a block; DoubleBuffer: O(P) temporary
            cub::DoubleBuffer<uint32_t> dbk(bid.p, bid2.p);
            cub::DoubleBuffer<uint64_t> dbv(dag, dag2.p);
            cub_call([&](void* t, size_t& b) {
                return cub::DeviceRadixSort::SortPairs(t, b, dbk, dbv, (int64_t)mE, 0, bbits, st);
            }, st, tmp);
            if (dbk.Current() != bid2.p) std::swap(bid.p, bid2.p);   // same sizes
            if (dbv.Current() != dag2.p) {   // sorted pairs landed in dag: keep dag2 the result
                PG_CK(cudaMemcpyAsync(dag2.p, dag, mE * 8, cudaMemcpyDeviceToDevice, st));
            }
        }
        bid.release();
        DBuf<unsigned long long> d_off;
        d_off.alloc(nb + 1);
        k_block_offsets<<<grid_for(nb + 1), kThreads, 0, st>>>(bid2.p, mE, nb, d_off.p);
        PG_LAUNCH_CHECK();
        PG_CK(cudaMemcpyAsync(off.data(), d_off.p, (nb + 1) * 8, cudaMemcpyDeviceToHost, st));
        // padded: the kernels read 16-byte covers of lists.  With the transposes (R25)
        // the pool holds three regions of mE + kColPad words: cols, tcol, tpos.
        h->has_t = h->orient != 1;
        const uint64_t region = mE + kColPad;
        h->tcol_base = h->has_t ? region : 0;
        h->tpos_base = h->has_t ? 2 * region : 0;
        h->d_col.alloc(h->has_t ? 3 * region : region);
        PG_CK(cudaMemsetAsync(h->d_col.p, 0, h->d_col.bytes(), st));
        k_local_cols<<<grid_for(mE), kThreads, 0, st>>>(dag2.p, bid2.p, mE, B, cu, h->d_col.p);
        PG_LAUNCH_CHECK();
        PG_CK(cudaStreamSynchronize(st));
        bid2.release();
        // dag2 (block-major DAG keys) replaces dag for the rowptr and cost passes
        PG_CK(cudaMemcpyAsync(dag, dag2.p, mE * 8, cudaMemcpyDeviceToDevice, st));
        PG_CK(cudaStreamSynchronize(st));
    }
    for (uint32_t b = 0; b < nb; ++b)
        if (off[b + 1] - off[b] >= (1ull << 32))
            fail(PGABB_ERANGE, "block (" + std::to_string(b / p) + "," + std::to_string(b % p) +
                                   ") holds >= 2^32 edges (block-local offsets are 32-bit): use a larger p");
    h->blocks.assign(nb, BlockInfo{});
    uint64_t rp_total = 0;
    std::vector<BlockDev> bdev(nb);
    std::vector<unsigned long long> rp_start;
    std::vector<BlockDev> present;
    for (uint32_t i = 0; i < p; ++i)
        for (uint32_t j = 0; j < p; ++j) {
            BlockInfo& b = h->blocks[i * p + j];
            b.col_off = off[i * p + j];
            b.nnz = off[i * p + j + 1] - off[i * p + j];
            b.nrows = h->cuts[i + 1] - h->cuts[i];
            b.ncols = h->cuts[j + 1] - h->cuts[j];
            b.present = (b.nnz > 0);
            if (b.present) {
                b.rp_off = rp_total;
                rp_start.push_back(rp_total);
                rp_total += (uint64_t)b.nrows + 1;
            }
            bdev[i * p + j] = to_dev(b, h->cuts[i]);
            if (b.present) present.push_back(bdev[i * p + j]);
        }
    const uint64_t rp_plain = rp_total;
    if (h->has_t)
        for (uint32_t i = 0; i < p; ++i)
            for (uint32_t j = i; j < p; ++j) {
                BlockInfo& b = h->blocks[i * p + j];
                if (!b.present) continue;
                b.trp_off = rp_total;
                rp_total += (uint64_t)b.ncols + 1;
            }
    h->d_rowptr.alloc(std::max<uint64_t>(rp_total, 1));
    if (rp_plain) {
        DBuf<BlockDev> d_present;
        DBuf<unsigned long long> d_rps;
        d_present.alloc(present.size());
        d_rps.alloc(rp_start.size());
        PG_CK(cudaMemcpyAsync(d_present.p, present.data(), present.size() * sizeof(BlockDev),
                              cudaMemcpyHostToDevice, st));
        PG_CK(cudaMemcpyAsync(d_rps.p, rp_start.data(), rp_start.size() * 8, cudaMemcpyHostToDevice, st));
        k_rowptr<<<grid_for(rp_plain), kThreads, 0, st>>>(dag, B, d_present.p, d_rps.p, (int)present.size(),
                                                          rp_plain, h->d_rowptr.p);
        PG_LAUNCH_CHECK();
        PG_CK(cudaStreamSynchronize(st));
    }

    // ---- S5c transposes of the blocks (MID orientation, DESIGN R25) ----------
    // Per block: a stable sort of (local col v, position e) -- u order is kept
    // within a column as the block is (u, v)-sorted -- gives tpos; tcol = the row
    // of each position; the transposed rowptr is a lower bound over the sorted v.
    // One block at a time, so the temporary memory is that of the largest block.
    if (h->has_t && mE) {
        uint64_t maxnnz = 0;
        for (const BlockInfo& b : h->blocks) maxnnz = std::max(maxnnz, b.nnz);
        DBuf<uint32_t> kv, kv2, iv, iv2;
        kv.alloc(maxnnz);
        kv2.alloc(maxnnz);
        iv.alloc(maxnnz);
        iv2.alloc(maxnnz);
        for (uint32_t i = 0; i < p; ++i)
            for (uint32_t j = i; j < p; ++j) {
                const BlockInfo& b = h->blocks[i * p + j];
                if (!b.present) continue;
                k_tkeys<<<grid_for(b.nnz), kThreads, 0, st>>>(h->d_col.p + b.col_off, b.nnz, kv.p, iv.p);
                PG_LAUNCH_CHECK();
                const int cb = std::max(1, bits_for(b.ncols));
                cub::DoubleBuffer<uint32_t> dbk(kv.p, kv2.p), dbv(iv.p, iv2.p);
                cub_call([&](void* t, size_t& bt) {
                    return cub::DeviceRadixSort::SortPairs(t, bt, dbk, dbv, (int64_t)b.nnz, 0, cb, st);
                }, st, tmp);
                k_tfill<<<grid_for(b.nnz), kThreads, 0, st>>>(dag + b.col_off, b.nnz, B, h->cuts[i], dbv.Current(),
                                                               h->d_col.p + h->tcol_base + b.col_off,
                                                               h->d_col.p + h->tpos_base + b.col_off);
                PG_LAUNCH_CHECK();
                k_trowptr<<<grid_for((uint64_t)b.ncols + 1), kThreads, 0, st>>>(dbk.Current(), b.nnz, b.ncols,
                                                                               h->d_rowptr.p + b.trp_off);
                PG_LAUNCH_CHECK();
            }
        PG_CK(cudaStreamSynchronize(st));
    }

    // ---- S5b dense bitmap copies of dense, narrow blocks -----
    {
        uint64_t words_total = 0;
        for (uint32_t i = 0; i < p; ++i)
            for (uint32_t j = i; j < p; ++j) {
                BlockInfo& b = h->blocks[i * p + j];
                const uint64_t wj = h->cuts[j + 1] - h->cuts[j];
                if (!b.present || wj > kWarpBitmapBits) continue;
                if (b.nnz * kDenseInv < (uint64_t)b.nrows * wj) continue;   // density < 1/32
                b.bm_words = (uint32_t)((wj + 31) / 32);
                b.bm_off = words_total;
                words_total += (uint64_t)b.nrows * b.bm_words;
            }
        h->d_bitmap.alloc(std::max<uint64_t>(words_total, 1));
        for (uint32_t i = 0; i < p; ++i)
            for (uint32_t j = i; j < p; ++j) {
                const BlockInfo& b = h->blocks[i * p + j];
                if (b.bm_off == ~0ull) continue;
                k_fill_bitmap<<<grid_for(b.nrows), kThreads, 0, st>>>(h->d_col.p, h->d_rowptr.p, b.col_off, b.rp_off,
                                                                      b.nrows, b.bm_words, h->d_bitmap.p + b.bm_off);
                PG_LAUNCH_CHECK();
            }
        PG_CK(cudaStreamSynchronize(st));
    }

    // ---- S6 tasks -----------------------------------------------------------
    h->task_of_ijx.assign((size_t)p * p * p, kNoTask);
    h->tasks.clear();
    for (uint32_t i = 0; i < p; ++i)
        for (uint32_t j = i; j < p; ++j) {
            if (!h->blocks[i * p + j].present) continue;
            for (uint32_t x = j; x < p; ++x) {
                if (!h->blocks[i * p + x].present || !h->blocks[j * p + x].present) continue;
                h->task_of_ijx[((size_t)i * p + j) * p + x] = (uint32_t)h->tasks.size();
                Task t;
                t.i = i; t.j = j; t.x = x;
                h->tasks.push_back(t);
            }
        }

    // ---- S7 costs -----------------------------------------------------------
    const size_t nt = h->tasks.size();
    if (nt) {
        DBuf<uint32_t> d_tid;
        DBuf<BlockDev> d_blk;
        DBuf<unsigned long long> d_cost, d_alg;
        d_tid.alloc(h->task_of_ijx.size());
        d_blk.alloc(nb);
        d_cost.alloc(nt);
        d_alg.alloc(nt);
        PG_CK(cudaMemcpyAsync(d_tid.p, h->task_of_ijx.data(), h->task_of_ijx.size() * 4, cudaMemcpyHostToDevice, st));
        PG_CK(cudaMemcpyAsync(d_blk.p, bdev.data(), nb * sizeof(BlockDev), cudaMemcpyHostToDevice, st));
        PG_CK(cudaMemsetAsync(d_cost.p, 0, nt * 8, st));
        PG_CK(cudaMemsetAsync(d_alg.p, 0, nt * 8, st));
        CostArg a;
        a.dag = dag; a.col = h->d_col.p; a.rowptr = h->d_rowptr.p; a.blk = d_blk.p; a.tid = d_tid.p;
        a.B = B; a.p = (int)p; a.cu = cu; a.mE = mE; a.cost = d_cost.p; a.alg_bytes = d_alg.p;
        for (uint32_t i = 0; i < p; ++i)
            for (uint32_t j = i; j < p; ++j) {
                const BlockInfo& b = h->blocks[i * p + j];
                if (!b.present) continue;
                k_task_costs<<<grid_for(b.nnz), kThreads, 0, st>>>(a, (int)i, (int)j);
                PG_LAUNCH_CHECK();
            }
        std::vector<unsigned long long> c(nt), ae(nt), cm(nt, 0), am(nt, 0), sl(nt, 0), sm(nt, 0);
        PG_CK(cudaMemcpyAsync(c.data(), d_cost.p, nt * 8, cudaMemcpyDeviceToHost, st));
        PG_CK(cudaMemcpyAsync(ae.data(), d_alg.p, nt * 8, cudaMemcpyDeviceToHost, st));
        PG_CK(cudaStreamSynchronize(st));
        if (h->has_t) {   // R25: the MID orientation's cost, bytes and streamed ids
            DBuf<unsigned long long> d_cm, d_am, d_sl, d_sm;
            for (auto* d : {&d_cm, &d_am, &d_sl, &d_sm}) {
                d->alloc(nt);
                PG_CK(cudaMemsetAsync(d->p, 0, nt * 8, st));
            }
            CostMidArg am_{};
            am_.col = h->d_col.p; am_.rowptr = h->d_rowptr.p; am_.blk = d_blk.p; am_.tid = d_tid.p; am_.p = (int)p;
            am_.tcol_base = h->tcol_base; am_.tpos_base = h->tpos_base;
            am_.cost = d_cm.p; am_.alg_bytes = d_am.p; am_.s_low = d_sl.p; am_.s_mid = d_sm.p;
            for (uint32_t i = 0; i < p; ++i)
                for (uint32_t j = i; j < p; ++j) {
                    const BlockInfo& b = h->blocks[i * p + j];
                    if (!b.present) continue;
                    k_task_costs_mid<<<grid_for(b.nnz), kThreads, 0, st>>>(am_, (int)i, (int)j);
                    PG_LAUNCH_CHECK();
                }
            PG_CK(cudaMemcpyAsync(cm.data(), d_cm.p, nt * 8, cudaMemcpyDeviceToHost, st));
            PG_CK(cudaMemcpyAsync(am.data(), d_am.p, nt * 8, cudaMemcpyDeviceToHost, st));
            PG_CK(cudaMemcpyAsync(sl.data(), d_sl.p, nt * 8, cudaMemcpyDeviceToHost, st));
            PG_CK(cudaMemcpyAsync(sm.data(), d_sm.p, nt * 8, cudaMemcpyDeviceToHost, st));
            PG_CK(cudaStreamSynchronize(st));
        }
        h->cost_total = 0;
        h->alg_total = 0;
        for (size_t t = 0; t < nt; ++t) {
            Task& T = h->tasks[t];
            T.cost_low = c[t];
            T.alg_low = ae[t];
            T.cost_mid = cm[t];
            T.alg_mid = am[t];
            T.s_low = sl[t];
            T.s_mid = sm[t];
            // R25: orient 1 -> LOW, 2 -> MID, 0 (auto) -> MID iff it streams (a) more than
            // kMidSaving fewer ids per visit (per edge of A_ij) -- a MID visit reads the
            // transpose's u (and suffix position) first, which short lists do not repay
            // (measured: ER c3, grid c4 faster in LOW) -- and (b) at most 3/4 of LOW's
            // ids -- LOW streams hub lists as bitmap words, so a small saving is not one
            // (measured: c2's hub tasks faster in LOW; R-MAT c2/c5 otherwise in MID)
            const uint64_t visits = h->blocks[T.i * p + T.j].nnz;
            const bool mid_wins = (unsigned __int128)sm[t] + (unsigned __int128)kMidSaving * visits < sl[t] &&
                                  (unsigned __int128)4 * sm[t] < (unsigned __int128)3 * sl[t];
            T.dir = !h->has_t ? kDirLow : h->orient == 2 ? kDirMid : (mid_wins ? kDirMid : kDirLow);
            T.cost = T.dir == kDirMid ? T.cost_mid : T.cost_low;
            T.alg_bytes = T.dir == kDirMid ? T.alg_mid : T.alg_low;
            h->cost_total += T.cost;
            h->alg_total += T.alg_bytes;
        }
    }
    keys2.release();
}

// S8: pieces (split heavy tasks by row cost) and LPT over ranks (DESIGN R18).
void plan_pieces(pgabb_blocks_s* h) {
    cudaStream_t st = h->stream;
    const uint32_t p = h->p;
    const int G = std::max(1, h->world_size);
    h->pieces.clear();
    // E(t): the caller's task weights if given (R22), else the S7 cost (R17)
    const bool weighted = !h->task_weights.empty();
    if (weighted && h->task_weights.size() != h->tasks.size())
        fail(PGABB_EINVAL, "task_weights has " + std::to_string(h->task_weights.size()) + " entries, the grid has " +
                               std::to_string(h->tasks.size()) + " tasks");
    auto E = [&](size_t t) -> uint64_t { return weighted ? h->task_weights[t] : h->tasks[t].cost; };
    unsigned __int128 total128 = 0;
    for (size_t t = 0; t < h->tasks.size(); ++t)
        if (h->tasks[t].cost) total128 += E(t);
    if (total128 >= ((unsigned __int128)1 << 63)) fail(PGABB_EINVAL, "task weights sum to >= 2^63");
    const uint64_t total = (uint64_t)total128;
    const uint64_t cap = (G <= 1) ? ~0ull : std::max<uint64_t>(1, (total + 4ull * G - 1) / (4ull * G));
    DBuf<unsigned long long> rc, R;
    DBuf<unsigned char> tmp;
    for (size_t t = 0; t < h->tasks.size(); ++t) {
        const Task& T = h->tasks[t];
        const BlockInfo& bij = h->blocks[T.i * p + T.j];
        if (T.cost == 0) continue;   // no (u,v,x) with a non-empty list: count 0
        const uint64_t w = E(t);
        const uint32_t nr = T.dir == kDirMid ? bij.ncols : bij.nrows;   // rows of part i (LOW) / j (MID)
        if (w <= cap) {
            h->pieces.push_back(Piece{(uint32_t)t, 0, nr, w, 0, T.cost});
            continue;
        }
        const uint64_t k = (w + cap - 1) / cap;
        rc.alloc((size_t)nr + 1);
        R.alloc((size_t)nr + 1);
        PG_CK(cudaMemsetAsync(rc.p, 0, ((size_t)nr + 1) * 8, st));
        if (T.dir == kDirMid)
            k_row_costs_mid<<<grid_for(nr), kThreads, 0, st>>>(
                h->d_col.p, h->d_rowptr.p, h->tcol_base, h->tpos_base, to_dev(bij, h->cuts[T.i]), bij.trp_off, nr,
                to_dev(h->blocks[T.i * p + T.x], 0), to_dev(h->blocks[T.j * p + T.x], 0), (int)(T.x == T.j), rc.p);
        else
            k_row_costs<<<grid_for(nr), kThreads, 0, st>>>(h->d_col.p, h->d_rowptr.p, to_dev(bij, h->cuts[T.i]),
                                                           to_dev(h->blocks[T.i * p + T.x], 0),
                                                           to_dev(h->blocks[T.j * p + T.x], 0), rc.p);
        PG_LAUNCH_CHECK();
        cub_call([&](void* tp, size_t& b) {
            return cub::DeviceScan::InclusiveSum(tp, b, rc.p, R.p, (int64_t)nr + 1, st);
        }, st, tmp);
        std::vector<unsigned long long> hR((size_t)nr + 1);
        PG_CK(cudaMemcpyAsync(hR.data(), R.p, ((size_t)nr + 1) * 8, cudaMemcpyDeviceToHost, st));
        PG_CK(cudaStreamSynchronize(st));
        std::vector<uint32_t> bnd{0};
        for (uint64_t q = 1; q < k; ++q) {
            // smallest rho with k * R[rho] >= q * cost
            const unsigned __int128 tgt = (unsigned __int128)q * T.cost;
            uint32_t lo = 0, hi = nr;
            while (lo < hi) {
                uint32_t mid = lo + ((hi - lo) >> 1);
                if ((unsigned __int128)k * hR[mid] >= tgt) hi = mid; else lo = mid + 1;
            }
            bnd.push_back(lo);
        }
        bnd.push_back(nr);
        for (uint64_t q = 0; q < k; ++q) {
            const uint64_t c = hR[bnd[q + 1]] - hR[bnd[q]];
            // piece weight: w * (its row-cost share), floor; = c when w is the S7 cost
            const uint64_t pw = weighted ? (uint64_t)((unsigned __int128)w * c / T.cost) : c;
            if (c > 0) h->pieces.push_back(Piece{(uint32_t)t, bnd[q], bnd[q + 1], pw, 0, c});
        }
    }
    // LPT: heaviest first (ties: task, row), least-loaded rank (ties: lowest rank)
    std::vector<size_t> order(h->pieces.size());
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) {
        const Piece &A = h->pieces[a], &Bp = h->pieces[b];
        if (A.cost != Bp.cost) return A.cost > Bp.cost;
        if (A.task != Bp.task) return A.task < Bp.task;
        return A.r0 < Bp.r0;
    });
    using LR = std::pair<uint64_t, int>;
    std::priority_queue<LR, std::vector<LR>, std::greater<LR>> pq;
    for (int g = 0; g < G; ++g) pq.push({0, g});
    for (size_t k : order) {
        LR top = pq.top();
        pq.pop();
        h->pieces[k].owner = top.second;
        top.first += h->pieces[k].cost;
        pq.push(top);
    }
}

// ---- the blocks and parts a task reads in its orientation (S9) ---------------
int task_parts(const pgabb_blocks_s* h, const Task& T, PartRef out[8]) {
    const uint32_t p = h->p, bij = T.i * p + T.j, bix = T.i * p + T.x, bjx = T.j * p + T.x;
    int n = 0;
    auto add = [&](uint32_t b, int part) {
        for (int k = 0; k < n; ++k)
            if (out[k].block == b && out[k].part == part) return;
        out[n++] = PartRef{b, part};
    };
    if (T.dir == kDirMid) {
        add(bij, kPartTCol);
        add(bij, kPartTRp);
        if (T.x == T.j) add(bij, kPartTPos);
        add(bjx, kPartCol);
        add(bjx, kPartRp);
        add(bix, kPartCol);
        add(bix, kPartRp);
        if (h->blocks[bix].bm_off != ~0ull) add(bix, kPartBm);
    } else {
        add(bij, kPartCol);
        add(bij, kPartRp);
        add(bix, kPartCol);
        add(bix, kPartRp);
        add(bjx, kPartCol);
        add(bjx, kPartRp);
        if (h->blocks[bjx].bm_off != ~0ull) add(bjx, kPartBm);
    }
    return n;
}

uint64_t part_words(const pgabb_blocks_s* h, PartRef r) {
    const BlockInfo& B = h->blocks[r.block];
    switch (r.part) {
        case kPartCol: case kPartTCol: case kPartTPos: return B.nnz;
        case kPartRp: return B.present ? (uint64_t)B.nrows + 1 : 0;
        case kPartTRp: return B.present ? (uint64_t)B.ncols + 1 : 0;
        default: return B.bm_off == ~0ull ? 0 : (uint64_t)B.nrows * B.bm_words;
    }
}

uint64_t part_src(const pgabb_blocks_s* h, PartRef r, int* pool) {
    const BlockInfo& B = h->blocks[r.block];
    switch (r.part) {
        case kPartCol: *pool = 0; return B.col_off;
        case kPartTCol: *pool = 0; return h->tcol_base + B.col_off;
        case kPartTPos: *pool = 0; return h->tpos_base + B.col_off;
        case kPartRp: *pool = 1; return B.rp_off;
        case kPartTRp: *pool = 1; return B.trp_off;
        default: *pool = 2; return B.bm_off;
    }
}

// A task's descriptor in kernel roles (internal.h TaskDev); off(part) = where the
// part lives (its pool offset, or a wave's arena offset).
template <class Off>
static TaskDev make_taskdev(const pgabb_blocks_s* h, const Task& T, Off off) {
    const uint32_t p = h->p, bij = T.i * p + T.j, bix = T.i * p + T.x, bjx = T.j * p + T.x;
    TaskDev d{};
    d.t_ell = ~0ull;
    d.dir = T.dir;
    d.wx = h->cuts[T.x + 1] - h->cuts[T.x];
    d.cx = h->cuts[T.x];
    if (T.dir == kDirMid) {
        d.s_col = off(PartRef{bjx, kPartCol}); d.s_rp = off(PartRef{bjx, kPartRp});
        d.n_col = off(PartRef{bij, kPartTCol}); d.n_rp = off(PartRef{bij, kPartTRp});
        d.n_pos = T.x == T.j ? off(PartRef{bij, kPartTPos}) : ~0ull;
        d.t_col = off(PartRef{bix, kPartCol}); d.t_rp = off(PartRef{bix, kPartRp});
        d.t_bm = h->blocks[bix].bm_off == ~0ull ? ~0ull : off(PartRef{bix, kPartBm});
        d.bm_words = h->blocks[bix].bm_words;
        d.c_row = h->cuts[T.j]; d.c_nbr = h->cuts[T.i];
    } else {
        d.s_col = off(PartRef{bix, kPartCol}); d.s_rp = off(PartRef{bix, kPartRp});
        d.n_col = off(PartRef{bij, kPartCol}); d.n_rp = off(PartRef{bij, kPartRp});
        d.n_pos = ~0ull;
        d.t_col = off(PartRef{bjx, kPartCol}); d.t_rp = off(PartRef{bjx, kPartRp});
        d.t_bm = h->blocks[bjx].bm_off == ~0ull ? ~0ull : off(PartRef{bjx, kPartBm});
        d.bm_words = h->blocks[bjx].bm_words;
        d.c_row = h->cuts[T.i]; d.c_nbr = h->cuts[T.j];
    }
    return d;
}

// Owned pieces in execution order: task (x desc, j desc, i asc), then rows.
static std::vector<size_t> locality_order(const pgabb_blocks_s* h) {
    std::vector<size_t> order(h->work.size());
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) {
        const Task &A = h->tasks[h->work[a].task], &Bt = h->tasks[h->work[b].task];
        if (A.x != Bt.x) return A.x > Bt.x;
        if (A.j != Bt.j) return A.j > Bt.j;
        if (A.i != Bt.i) return A.i < Bt.i;
        return h->work[a].r0 < h->work[b].r0;
    });
    return order;
}

// Streaming residency: cut the owned pieces (in execution order) into waves whose
// blocks fit half the device budget; each wave gets arena offsets for its blocks
// and its own task-descriptor table.  EBUDGET if one task's three blocks alone
// exceed half the budget ("hard error").
void plan_waves(pgabb_blocks_s* h) {
    // The device budget is one arena of K slots (a block cache deeper than double
    // buffering, NEXT-2): wave k stages the parts it lacks into slot k mod K while
    // wave k-1 computes.  A part that a recent wave already staged is read IN PLACE
    // when its slot cannot be overwritten before this wave ends (the slots of waves
    // k-1 .. k-K+2), copied device-to-device from the slot of wave k-K+1 (which wave
    // k+1 overwrites while wave k runs), else copied from pinned host memory.  K is
    // the largest of 4, 3, 2 whose slot holds the biggest task's parts.
    const uint64_t budget_words = h->budget / 4;
    const size_t nt = h->tasks.size();
    uint64_t max_task_words = 1;
    for (const Task& T : h->tasks) {
        PartRef parts[8];
        const int np = task_parts(h, T, parts);
        uint64_t wds = 0;
        for (int q = 0; q < np; ++q) wds += part_words(h, parts[q]);
        max_task_words = std::max(max_task_words, wds);
    }
    int K = 2;
    for (int k = kMaxSlots; k > 2; --k)
        if (max_task_words <= budget_words / k - kColPad) {
            K = k;
            break;
        }
    const uint64_t slot_words = budget_words / K - kColPad;
    h->slots = K;
    h->slot_words = slot_words;
    h->waves.clear();
    size_t npieces = 0;                 // owned pieces placed so far (locality order)
    std::vector<TaskDev> wtasks;
    const std::vector<size_t> order = locality_order(h);
    using Key = std::pair<uint32_t, int>;
    struct Slot {
        std::map<Key, uint64_t> parts;  // part -> absolute arena word offset
        int64_t filled_by = -1, last_reader = -1;
    };
    std::vector<Slot> slot(K);
    Wave cur;
    int64_t k = 0;                      // index of the wave being planned
    std::vector<TaskDev> cur_tasks;
    auto open_wave = [&]() {
        cur = Wave{};
        cur.piece_begin = npieces;
        cur.slot = (int)(k % K);
        Slot& sl = slot[cur.slot];
        cur.wait_wave = sl.last_reader;  // the slot's previous readers must be done
        sl.parts.clear();
        sl.filled_by = k;
        sl.last_reader = k;
        cur_tasks.assign(nt, TaskDev{});
    };
    auto close_wave = [&]() {
        if (npieces == cur.piece_begin) return;
        cur.piece_end = npieces;
        cur.item_begin = h->piece_item_off[cur.piece_begin];
        cur.item_end = h->piece_item_off[cur.piece_end];
        cur.light_begin = h->piece_light_off[cur.piece_begin];
        cur.light_end = h->piece_light_off[cur.piece_end];
        cur.med_begin = h->piece_med_off[cur.piece_begin];
        cur.med_end = h->piece_med_off[cur.piece_end];
        cur.task_table = h->waves.size();
        wtasks.insert(wtasks.end(), cur_tasks.begin(), cur_tasks.end());
        h->waves.push_back(cur);
        ++k;
    };
    // where a part can be read from for wave k without staging it: its own slot, or
    // a slot of waves k-1 .. k-K+2 (not overwritten before wave k ends)
    auto in_place = [&](const Key& key, int* from) -> const uint64_t* {
        for (int s2 = 0; s2 < K; ++s2) {
            const Slot& sl = slot[s2];
            const bool ok = s2 == cur.slot || (sl.filled_by >= k - (K - 2) && sl.filled_by <= k - 1);
            if (!ok) continue;
            const auto it = sl.parts.find(key);
            if (it != sl.parts.end()) {
                *from = s2;
                return &it->second;
            }
        }
        return nullptr;
    };
    open_wave();
    for (size_t q0 : order) {
        const PieceDev& w = h->work[q0];
        const Task& T = h->tasks[w.task];
        PartRef parts[8];
        const int np = task_parts(h, T, parts);
        uint64_t all = 0, fresh = 0;
        for (int q = 0; q < np; ++q) {
            const uint64_t wd = part_words(h, parts[q]);
            all += wd;
            int from = 0;
            if (!in_place({parts[q].block, parts[q].part}, &from)) fresh += wd;
        }
        if (all > slot_words)
            fail(PGABB_EBUDGET, "task (" + std::to_string(T.i) + "," + std::to_string(T.j) + "," +
                                    std::to_string(T.x) + ") needs " + std::to_string(all * 4) +
                                    " bytes of blocks, more than half the device budget");
        // pipeline ramp: the first waves are smaller (1/4, 1/2 of a slot) so the copy
        // that no computation can hide is short
        const uint64_t cap = k < 2 ? std::max<uint64_t>(slot_words >> (2 - k), all) : slot_words;
        if (cur.words + fresh > cap && npieces > cur.piece_begin) {
            close_wave();
            open_wave();
        }
        const uint64_t slot_base = (uint64_t)cur.slot * (slot_words + kColPad);
        for (int q = 0; q < np; ++q) {
            const Key key{parts[q].block, parts[q].part};
            int from = 0;
            if (const uint64_t* at = in_place(key, &from)) {
                if (from != cur.slot) slot[from].last_reader = k;   // read in place by this wave
                continue;
            }
            const uint64_t wd = part_words(h, parts[q]);
            const uint64_t dst = slot_base + cur.words;
            // the slot of wave k-K+1 is overwritten by wave k+1: copy from it device-to-device
            int64_t d2d_src = -1;
            for (int s2 = 0; s2 < K; ++s2)
                if (s2 != cur.slot && slot[s2].filled_by == k - (K - 1)) {
                    const auto it = slot[s2].parts.find(key);
                    if (it != slot[s2].parts.end()) d2d_src = (int64_t)it->second;
                }
            int pool = 0;
            const uint64_t src = part_src(h, parts[q], &pool);
            if (wd && d2d_src >= 0) cur.copies.push_back(StagedBlock{(uint64_t)d2d_src, dst, wd, 3});
            else if (wd) cur.copies.push_back(StagedBlock{src, dst, wd, pool});
            slot[cur.slot].parts[key] = dst;
            cur.words += wd;
        }
        cur_tasks[w.task] = make_taskdev(h, T, [&](PartRef r) {
            int from = 0;
            return *in_place({r.block, r.part}, &from);
        });
        ++npieces;
    }
    close_wave();
    h->d_wave_tasks.alloc(std::max<size_t>(wtasks.size(), 1));
    if (!wtasks.empty())
        PG_COPY_SYNC(h->d_wave_tasks.p, wtasks.data(), wtasks.size() * sizeof(TaskDev), h->stream);
    // one arena of K slots, each padded like the col pool (16-byte list covers)
    h->d_arena.alloc((uint64_t)K * (slot_words + kColPad));
    PG_CK(cudaMemsetAsync(h->d_arena.p, 0, h->d_arena.bytes(), h->stream));
}

// This rank's work list: owned pieces in (task, row) order, the task descriptors
// (kernel roles, R25), the host-resident copy list (S9) and the row items.
void upload_work(pgabb_blocks_s* h) {
    const int me = std::max(0, h->rank);
    cudaStream_t st = h->stream;
    h->work.clear();
    h->work_edges = 0;
    h->cost_local = 0;
    h->alg_local = 0;

    // task descriptors for the intersection kernels (pool offsets)
    std::vector<TaskDev> td(std::max<size_t>(h->tasks.size(), 1));
    for (size_t t = 0; t < h->tasks.size(); ++t)
        td[t] = make_taskdev(h, h->tasks[t], [&](PartRef r) {
            int pool = 0;
            return part_src(h, r, &pool);
        });
    h->d_tasks.alloc(td.size());
    PG_COPY_SYNC(h->d_tasks.p, td.data(), td.size() * sizeof(TaskDev), st);

    std::vector<char> task_mine(h->tasks.size(), 0);
    for (const Piece& pc : h->pieces) {
        if (pc.owner != me) continue;
        const TaskDev& T = td[pc.task];
        uint32_t e0 = 0, e1 = 0;
        PG_COPY_SYNC(&e0, h->d_rowptr.p + T.n_rp + pc.r0, 4, st);
        PG_COPY_SYNC(&e1, h->d_rowptr.p + T.n_rp + pc.r1, 4, st);
        if (e1 == e0) continue;
        PieceDev w{};
        w.gstart = h->work_edges;
        w.r0 = pc.r0; w.r1 = pc.r1; w.e0 = e0; w.e1 = e1;
        w.task = pc.task;
        w.dir = h->tasks[pc.task].dir;
        h->work.push_back(w);
        h->work_edges += (e1 - e0);
        h->cost_local += pc.cost;
        task_mine[pc.task] = 1;
    }
    // NEXT-3 collaborative CPU + GPU: the sparsest owned
    // pieces -- least S7 cost per neighbour visit, the latency-bound ones the paper
    // sends to CPUs -- up to host_permille of this rank's cost are counted by host
    // threads from the pinned host pools; the GPU neither copies nor counts them
    h->host_work.clear();
    h->host_tasks.clear();
    if (h->host_permille && !h->work.empty()) {
        std::vector<size_t> byd(h->work.size());
        std::iota(byd.begin(), byd.end(), 0);
        auto pcost = [&](const PieceDev& w) {   // the piece's S7 cost (its Piece record)
            for (const Piece& pc : h->pieces)
                if (pc.task == w.task && pc.r0 == w.r0 && pc.owner == me) return pc.rcost;
            return (uint64_t)0;
        };
        std::vector<uint64_t> cst(h->work.size());
        for (size_t q = 0; q < h->work.size(); ++q) cst[q] = pcost(h->work[q]);
        std::stable_sort(byd.begin(), byd.end(), [&](size_t a, size_t b) {
            // cost per visit ascending: cst[a]/visits[a] < cst[b]/visits[b]
            const unsigned __int128 l = (unsigned __int128)cst[a] * (h->work[b].e1 - h->work[b].e0);
            const unsigned __int128 r = (unsigned __int128)cst[b] * (h->work[a].e1 - h->work[a].e0);
            return l < r;
        });
        uint64_t total = 0;
        for (uint64_t c : cst) total += c;
        const unsigned __int128 want = (unsigned __int128)total * h->host_permille;
        std::vector<char> to_host(h->work.size(), 0);
        unsigned __int128 got = 0;
        for (size_t q : byd) {
            if (got * 1000 >= want) break;
            to_host[q] = 1;
            got += cst[q];
        }
        std::vector<PieceDev> gpu;
        for (size_t q = 0; q < h->work.size(); ++q) (to_host[q] ? h->host_work : gpu).push_back(h->work[q]);
        h->work.swap(gpu);
        h->host_tasks = td;
        h->h_host_counts.alloc(std::max<size_t>(h->tasks.size(), 1));
        h->d_host_counts.alloc(std::max<size_t>(h->tasks.size(), 1));
    }

    // staged-model bytes of the owned pieces: whole tasks are attributed to the
    // rank that owns their first piece's share in proportion to cost
    for (size_t t = 0; t < h->tasks.size(); ++t) {
        if (!task_mine[t]) continue;
        const Task& T = h->tasks[t];
        uint64_t mine = 0;
        for (const Piece& pc : h->pieces)
            if (pc.task == t && pc.owner == me) mine += pc.rcost;
        h->alg_local += (uint64_t)((long double)T.alg_bytes * mine / (T.cost ? T.cost : 1));
    }
    h->d_task_counts.alloc(h->tasks.size() + 1);
    h->d_next.alloc(8);

    // S9 (host-resident, no budget): the pool ranges of the block parts the owned
    // pieces read, merged
    {
        std::set<std::pair<uint32_t, int>> need;
        for (const PieceDev& w : h->work) {
            PartRef parts[8];
            const int np = task_parts(h, h->tasks[w.task], parts);
            for (int q = 0; q < np; ++q) need.insert({parts[q].block, parts[q].part});
        }
        std::vector<StagedBlock> r;
        for (const auto& key : need) {
            const PartRef pr{key.first, key.second};
            const uint64_t wd = part_words(h, pr);
            int pool = 0;
            const uint64_t src = part_src(h, pr, &pool);
            if (wd) r.push_back(StagedBlock{src, src, wd, pool});
        }
        std::sort(r.begin(), r.end(), [](const StagedBlock& a, const StagedBlock& b) {
            return a.pool != b.pool ? a.pool < b.pool : a.src_word < b.src_word;
        });
        h->host_copies.clear();
        for (const StagedBlock& c : r) {   // merge adjacent ranges of one pool
            if (!h->host_copies.empty() && h->host_copies.back().pool == c.pool &&
                h->host_copies.back().src_word + h->host_copies.back().words == c.src_word)
                h->host_copies.back().words += c.words;
            else
                h->host_copies.push_back(c);
        }
        // (cover reads past a copied list stay inside the device pool, whose zero
        // padding the build wrote, and their ids are masked by the list bounds)
    }

    // largest block-triple footprint (what one task needs resident, S9)
    h->max_task_bytes = 0;
    for (const Task& T : h->tasks) {
        PartRef parts[8];
        const int np = task_parts(h, T, parts);
        uint64_t words = 0;
        for (int q = 0; q < np; ++q) words += part_words(h, parts[q]);
        h->max_task_bytes = std::max(h->max_task_bytes, 4 * words);
    }
    // Row items of the owned pieces, laid out for L2 locality: pieces in task
    // order (x desc, j desc, i asc) so that the warps running concurrently share
    // the blocks of one task (and the hub column part is done first), rows
    // ascending inside a piece.  Compaction is a count + exclusive scan per piece,
    // so the layout is deterministic.
    const std::vector<size_t> order = locality_order(h);
    uint32_t maxrows = 0;
    for (const PieceDev& w : h->work) maxrows = std::max(maxrows, w.r1 - w.r0);
    DBuf<uint32_t> hf, lf, mf, hpos, lpos, mpos;
    DBuf<unsigned char> tmp;
    for (DBuf<uint32_t>* b : {&hf, &lf, &mf, &hpos, &lpos, &mpos}) b->alloc((size_t)maxrows + 1);
    std::vector<uint64_t> piece_items(h->work.size(), 0), piece_light(h->work.size(), 0),
        piece_med(h->work.size(), 0);
    DBuf<unsigned long long> d_alg;
    d_alg.alloc(1);
    PG_CK(cudaMemsetAsync(d_alg.p, 0, 8, st));
    auto classify = [&](const PieceDev& w, unsigned long long* alg) {
        const uint32_t nr = w.r1 - w.r0;
        k_row_flags<<<grid_for(nr + 1), kThreads, 0, st>>>(w, h->d_tasks.p, h->d_col.p, h->d_rowptr.p, hf.p, lf.p,
                                                           mf.p, h->light_held, alg);
        PG_LAUNCH_CHECK();
        cub_call([&](void* tp, size_t& b) {
            return cub::DeviceScan::ExclusiveSum(tp, b, hf.p, hpos.p, (int64_t)nr + 1, st);
        }, st, tmp);
        cub_call([&](void* tp, size_t& b) {
            return cub::DeviceScan::ExclusiveSum(tp, b, lf.p, lpos.p, (int64_t)nr + 1, st);
        }, st, tmp);
        cub_call([&](void* tp, size_t& b) {
            return cub::DeviceScan::ExclusiveSum(tp, b, mf.p, mpos.p, (int64_t)nr + 1, st);
        }, st, tmp);
    };
    // pass 1: count per piece; item offsets per piece in locality order (the waves of
    // streaming residency are contiguous ranges of them)
    h->piece_item_off.assign(order.size() + 1, 0);
    h->piece_light_off.assign(order.size() + 1, 0);
    h->piece_med_off.assign(order.size() + 1, 0);
    auto count_pass = [&]() {
        uint64_t nh = 0, nm = 0;
        PG_CK(cudaMemsetAsync(d_alg.p, 0, 8, st));
        for (size_t k : order) {
            const PieceDev& w = h->work[k];
            const uint32_t nr = w.r1 - w.r0;
            classify(w, d_alg.p);
            uint32_t cnt[3] = {0, 0, 0};
            PG_CK(cudaMemcpyAsync(&cnt[0], hpos.p + nr, 4, cudaMemcpyDeviceToHost, st));
            PG_CK(cudaMemcpyAsync(&cnt[1], lpos.p + nr, 4, cudaMemcpyDeviceToHost, st));
            PG_CK(cudaMemcpyAsync(&cnt[2], mpos.p + nr, 4, cudaMemcpyDeviceToHost, st));
            PG_CK(cudaStreamSynchronize(st));
            piece_items[k] = cnt[0];
            piece_light[k] = cnt[1];
            piece_med[k] = cnt[2];
            nh += cnt[0];
            nm += cnt[2];
        }
        return std::make_pair(nh, nm);
    };
    const auto [n_heavy1, n_med1] = count_pass();
    // auto (R29): the medium kernel only when its rows are at least half of what would
    // otherwise be heavy items (low-skew graphs: ER at small p); else they stay heavy
    if (h->light_auto && h->light_held > kLightLa && 2 * n_med1 < n_heavy1 + n_med1) {
        h->light_held = kLightLa;
        count_pass();
    }
    // the light list holds every piece's light items, then every piece's medium items
    uint64_t nitems = 0, nlight = 0, nmed = 0;
    for (size_t q = 0; q < order.size(); ++q) nlight += piece_light[order[q]];
    for (size_t q = 0; q < order.size(); ++q) {
        nitems += piece_items[order[q]];
        h->piece_item_off[q + 1] = nitems;
        h->piece_light_off[q + 1] = h->piece_light_off[q] + piece_light[order[q]];
        h->piece_med_off[q] = nlight + nmed;
        nmed += piece_med[order[q]];
    }
    h->piece_med_off[order.size()] = nlight + nmed;
    h->n_items = nitems;
    h->n_light0 = nlight;
    h->n_light = nlight + nmed;
    unsigned long long alg_light = 0;
    PG_COPY_SYNC(&alg_light, d_alg.p, 8, st);
    h->alg_light = alg_light;
    h->d_items.alloc(std::max<uint64_t>(nitems, 1));
    h->d_light.alloc(std::max<uint64_t>(h->n_light, 1));
    uint64_t max_light = 0;
    for (uint64_t c : piece_light) max_light = std::max(max_light, c);
    for (uint64_t c : piece_med) max_light = std::max(max_light, c);
    DBuf<uint32_t> lkey, lkey2;
    DBuf<uint4> litem2;
    if (max_light) {
        lkey.alloc(max_light);
        lkey2.alloc(max_light);
        litem2.alloc(max_light);
    }
    // pass 2: emit in layout order
    uint64_t base = 0, lbase = 0, mbase = nlight;
    // a piece's light (or medium) items, then sorted by work (stable: rows ascending
    // within equal work)
    auto emit_light = [&](const PieceDev& w, const uint32_t* flags, const uint32_t* pos, uint4* li, int64_t nl) {
        const uint32_t nr = w.r1 - w.r0;
        k_light_emit<<<grid_for(nr), kThreads, 0, st>>>(w, h->d_tasks.p, flags, pos, h->d_col.p, h->d_rowptr.p,
                                                        li, lkey.p);
        PG_LAUNCH_CHECK();
        const int kb = 8 + bits_for((uint64_t)(nl - 1) / kLightSortWindow);
        cub_call([&](void* tp, size_t& b) {
            return cub::DeviceRadixSort::SortPairs(tp, b, lkey.p, lkey2.p, li, litem2.p, nl, 0, kb, st);
        }, st, tmp);
        PG_CK(cudaMemcpyAsync(li, litem2.p, (size_t)nl * sizeof(uint4), cudaMemcpyDeviceToDevice, st));
    };
    for (size_t k : order) {
        const PieceDev& w = h->work[k];
        const uint32_t nr = w.r1 - w.r0;
        if (!piece_items[k] && !piece_light[k] && !piece_med[k]) continue;
        classify(w, nullptr);
        if (piece_items[k]) {
            k_row_emit<<<grid_for(nr), kThreads, 0, st>>>(w, hf.p, hpos.p, h->d_items.p + base);
            PG_LAUNCH_CHECK();
        }
        if (piece_light[k]) emit_light(w, lf.p, lpos.p, h->d_light.p + lbase, (int64_t)piece_light[k]);
        if (piece_med[k]) emit_light(w, mf.p, mpos.p, h->d_light.p + mbase, (int64_t)piece_med[k]);
        base += piece_items[k];
        lbase += piece_light[k];
        mbase += piece_med[k];
    }
    // R30: sector-aligned slots for the streamed blocks of this rank's LOW list tasks,
    // on device-resident handles of graphs that use the medium kernel (short lists
    // of several sectors: ER-like); the task table then points at them
    if (kEll && h->residency == PGABB_RESIDENT_DEVICE && h->n_light > h->n_light0) {
        const uint32_t p = h->p;
        std::vector<uint64_t> ell_off(h->blocks.size(), ~0ull);
        std::vector<uint32_t> ell_w(h->blocks.size(), 0);
        uint64_t words = 0;
        for (size_t t = 0; t < h->tasks.size(); ++t) {
            const Task& T = h->tasks[t];
            if (!task_mine[t] || T.dir != kDirLow || td[t].t_bm != ~0ull) continue;
            const uint32_t bjx = T.j * p + T.x;
            const BlockInfo& b = h->blocks[bjx];
            if (ell_off[bjx] != ~0ull || !b.present || b.nrows == 0) continue;
            const double avg = (double)b.nnz / b.nrows;
            const uint32_t ew = avg <= 3.5 ? 8u : (avg <= 10.0 ? 16u : 0u);
            if (!ew) continue;
            words = (words + 15) & ~15ull;   // 64-byte aligned slots
            ell_off[bjx] = words;
            ell_w[bjx] = ew;
            words += (uint64_t)b.nrows * ew;
        }
        if (words) {
            h->d_ell.alloc(words + 16);
            for (size_t bx = 0; bx < h->blocks.size(); ++bx) {
                if (ell_off[bx] == ~0ull) continue;
                const BlockInfo& b = h->blocks[bx];
                k_fill_ell<<<grid_for(b.nrows), kThreads, 0, st>>>(h->d_col.p, h->d_rowptr.p, b.col_off, b.rp_off,
                                                                   b.nrows, ell_w[bx], h->d_ell.p + ell_off[bx]);
                PG_LAUNCH_CHECK();
            }
            for (size_t t = 0; t < h->tasks.size(); ++t) {
                const Task& T = h->tasks[t];
                if (!task_mine[t] || T.dir != kDirLow || td[t].t_bm != ~0ull) continue;
                const uint32_t bjx = T.j * p + T.x;
                if (ell_off[bjx] == ~0ull) continue;
                td[t].t_ell = ell_off[bjx];
                td[t].ell_w = ell_w[bjx];
            }
            PG_COPY_SYNC(h->d_tasks.p, td.data(), td.size() * sizeof(TaskDev), st);
        }
    }
    PG_CK(cudaStreamSynchronize(st));
}

}  // namespace pgabb
