// count.cu -- S9..S11: residency, the intersection kernels, the count reduction.
//
// Listing 5 (§3.6):
//     reduce_dev over u in S_k:  for v in Edges(E_k, u):
//         n_t += Intersect(Edges(E_l, u), Edges(E_m, v))
// with the block-list <B_k, B_l, B_m> = <A_ij, A_ix, A_jx> (DESIGN R5).  All
// lists are sorted local column ids of part x, so an intersection is a plain
// sorted-set intersection; "list or hashmap-based" leaves
// the method open (DESIGN R8).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <thread>

#include "internal.h"

// PGABB_PROF (tooling build only, tools/prof_paths.py): per-path SM-cycle shares of
// k_tc_rows, accumulated per warp in registers and flushed once per warp.
#ifdef PGABB_PROF
__device__ unsigned long long g_prof[32];
#define PROF_ARGS , unsigned long long* prof, unsigned long long& pt
#define PROF_PASS , prof, pt
#define PROF_MARK(cat) do { const unsigned long long _n = clock64(); prof[cat] += _n - pt; pt = _n; } while (0)
#define PROF_CNT(cat) (prof[cat] += 1)
#else
#define PROF_ARGS
#define PROF_PASS
#define PROF_MARK(cat) do { } while (0)
#define PROF_CNT(cat) do { } while (0)
#endif

namespace pgabb {

namespace {

__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}

// Lane-parallel binary search of the shorter list's elements in the longer one.
// Returns this lane's share of |A ∩ B|.
// VTX: every common element w also adds 1 to tvx[w] (per-vertex counts, NEXT-1).
template <bool VTX>
__device__ __forceinline__ uint32_t warp_intersect(const uint32_t* __restrict__ A, uint32_t la,
                                                   const uint32_t* __restrict__ B, uint32_t lb, int lane,
                                                   unsigned long long* __restrict__ tvx) {
    const uint32_t* S = la <= lb ? A : B;
    const uint32_t* L = la <= lb ? B : A;
    const uint32_t ls = min(la, lb), ll = max(la, lb);
    uint32_t c = 0;
    for (uint32_t k = lane; k < ls; k += 32) {
        const uint32_t x = __ldg(S + k);
        uint32_t lo = 0, hi = ll;
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (__ldg(L + mid) < x) lo = mid + 1; else hi = mid;
        }
        const uint32_t hit = (lo < ll && __ldg(L + lo) == x);
        if (VTX && hit) atomicAdd(tvx + x, 1ull);
        c += hit;
    }
    return c;
}

// ---------------------------------------------------------------------------
// k_tc_rows: one warp per row item (task t = (i,j,x), row u of part i).
//
//   stage    A_ix[u] into a warp-private shared-memory set over part x:
//            a bitmap of w_x bits (w_x <= 32768, 4 KB) or, for wider parts, an
//            open-addressing hash of <= 1024 slots (|A_ix[u]| <= 512);
//   stream   the lists A_jx[v] of 32 consecutive v in A_ij[u] at a time, as
//            one flattened sequence of 16-byte covers (see intersect_row), so
//            short lists do not idle lanes; dense A_jx rows are ANDed with the
//            staged bitmap, short-vs-long pairs binary-searched;
//   probe    each element against the staged set;
//   reduce   lane partials -> warp sum, kept per warp while consecutive rows
//            share a task, one atomicAdd per task change.
//
// Rows whose A_ix[u] fits neither set fall back to lane-parallel binary search;
// dense A_jx with a short A_ix[u] skips staging (probe_dense_row).  This is the
// staged model of SURVEY §8(d): A_ix[u] read once per (task, u), A_jx[v] once
// per edge.  Items are in locality order and claimed by warps from a counter.
// ---------------------------------------------------------------------------
constexpr int kRowWarps = 8;
#ifndef PGABB_AND_UNROLL
#define PGABB_AND_UNROLL 2
#endif
constexpr int kAndUnroll = PGABB_AND_UNROLL;   // v rows in flight per lane group in the dense AND path
#ifndef PGABB_DENSE_UNROLL
#define PGABB_DENSE_UNROLL 4
#endif
constexpr int kDenseUnroll = PGABB_DENSE_UNROLL;   // bit tests in flight per lane in probe_dense_row
// probe_dense_row (one scattered bit test per element of A_ix[u] per pair) instead
// of staging + the AND path (W coalesced words, W/8 sectors per pair) when
// |A_ix[u]| <= kDenseRowMul * W / 8
#ifndef PGABB_DENSE_ROW_MUL
#define PGABB_DENSE_ROW_MUL 16
#endif
constexpr uint32_t kDenseRowMul = PGABB_DENSE_ROW_MUL;
#ifndef PGABB_DENSE_ROW_MUL_WIDE
#define PGABB_DENSE_ROW_MUL_WIDE 8   // A/B: c5s -5 %, c2 unchanged (its hub part is <= 32 words)
#endif
#ifndef PGABB_DENSE_ROW_WIDE_W
#define PGABB_DENSE_ROW_WIDE_W 32
#endif
constexpr uint32_t kDenseRowMulWide = PGABB_DENSE_ROW_MUL_WIDE;   // for parts wider than kDenseRowWideW words
constexpr uint32_t kDenseRowWideW = PGABB_DENSE_ROW_WIDE_W;
#ifndef PGABB_LIST_UNROLL
#define PGABB_LIST_UNROLL 1   // A/B: 2 loads in flight per lane lose (c2 heavy 1.72 -> 1.91 ms, c5 0.963 -> 0.996 s), 4 lose more
#endif
constexpr int kListUnroll = PGABB_LIST_UNROLL;
#ifndef PGABB_CARRY_CUR
#define PGABB_CARRY_CUR 1
#endif
constexpr bool kCarryCur = PGABB_CARRY_CUR;   // list index carried across rounds (no per-round ballot)   // 16-byte list loads in flight per lane (flattened lists)
#ifndef PGABB_ROW_CHUNK
#define PGABB_ROW_CHUNK 4
#endif
constexpr int kRowChunk = PGABB_ROW_CHUNK;   // row items per warp claim
#ifndef PGABB_SMALL_HELD
#define PGABB_SMALL_HELD 0   // A/B: c5 1.006 -> 1.043 s, c2 2.52 -> 2.59 ms with it (the flattened lists win)
#endif
constexpr bool kSmallHeld = PGABB_SMALL_HELD;   // heavy rows with <= kLightLa held ids: per-lane lists

// Claims the next kRowChunk items for the calling warp; returns the first (>= n: done).
__device__ __forceinline__ unsigned long long claim_items(unsigned long long* next, unsigned long long n, int lane,
                                                          unsigned long long& end) {
    unsigned long long b = 0;
    if (lane == 0) b = atomicAdd(next, (unsigned long long)kRowChunk);
    b = __shfl_sync(0xffffffffu, b, 0);
    end = b + kRowChunk < n ? b + kRowChunk : n;
    return b;
}
#ifndef PGABB_ROW_MINB
#define PGABB_ROW_MINB 5
#endif
constexpr int kRowMinBlocks = PGABB_ROW_MINB;   // CTAs per SM (5 x 8 warps x 4.4 KB of sets; 48 registers)
constexpr uint32_t kSetWords = kWarpBitmapBits / 32;   // 1024 words = 4 KB per warp
// Batched small rows (k_tc_rows, VM = 0): heavy rows without a dense A_jx copy,
// with |A_ix[u]| <= kBatchLa and <= 32 neighbours, are intersected several at a
// time by one warp (batch_rows).  0 disables.
#ifndef PGABB_BATCH_LA
#define PGABB_BATCH_LA 0   // A/B (32): c3 p=4 26.5 -> 15.9 ms, but p=1 16.2 -> 17.3, c2 2.46 -> 8.7, c5 1.01 -> 1.17 s
#endif
constexpr uint32_t kBatchLa = PGABB_BATCH_LA;
static_assert(kBatchLa <= 32, "a batch row's held list is loaded by one round of lanes");
constexpr uint32_t kScratchWords = kBatchLa ? 128 : 96;   // per-warp list descriptors (+ batch regions)
// per-vertex kernel: + the batch's v ids (32), the row's prefix popcounts of S
// (1024 u16) and its hit counters (1024 u16), see VCnt
#ifndef PGABB_VTX_SLOTS
#define PGABB_VTX_SLOTS 1024
#endif
#ifndef PGABB_VTX_PRE_GROUP
#define PGABB_VTX_PRE_GROUP 1   // A/B: 8 (4 CTAs/SM) is 1.5x slower: extra popcounts per hit
#endif
constexpr uint32_t kVtxSlots = PGABB_VTX_SLOTS;        // u16 hit counters per warp
#ifndef PGABB_HASH_FILTER
#define PGABB_HASH_FILTER 1
#endif
constexpr bool kHashFilter = PGABB_HASH_FILTER;
constexpr uint32_t kPreGroup = PGABB_VTX_PRE_GROUP;    // S words per stored prefix popcount
constexpr uint32_t kPreWords = (kSetWords / kPreGroup + 1) / 2;
constexpr uint32_t kScratchWordsV = 160 + kPreWords + kVtxSlots / 2;
// VM (per-vertex roles, NEXT-1): 0 count only; 1 the row's lowest vertex u; 2 + the
// middle vertex v (per pair); 3 + the highest vertex w (per hit, warp counters)
// PGABB_VTX_INSET: the per-vertex counters of a bitmap row live in the unused
// tail of the warp's 4 KB set (a part of W <= kInsetMaxW words leaves 1024 - W
// words free), so the VM = 3 kernel keeps the counting kernel's footprint and
// occupancy; hash-set rows then credit w with global atomics.
#ifndef PGABB_VTX_SLICED
#define PGABB_VTX_SLICED 1
#endif
constexpr bool kVtxSliced = PGABB_VTX_SLICED;   // per-vertex dense pairs: bit-sliced hit counters (and_vtx)
#ifndef PGABB_VTX_MATCH
#define PGABB_VTX_MATCH 1
#endif
constexpr bool kVtxMatch = PGABB_VTX_MATCH;     // per-vertex list hits: warp-aggregated by w (probe4)
#ifndef PGABB_VTX_INSET
#define PGABB_VTX_INSET 1
#endif
constexpr bool kVtxInset = PGABB_VTX_INSET;
__host__ __device__ constexpr uint32_t scratch_words(int vm) {
    return vm >= 3 && !kVtxInset ? kScratchWordsV : vm >= 1 ? 160u : kScratchWords;
}

// Per-vertex counts, third vertex w (NEXT-1): a hub w is hit by many v of the same
// row, so instead of one global atomic per hit the row's hits are counted in warp
// shared memory -- u16 counters indexed by w's position in A_ix[u] (bitmap set:
// rank of w = prefix popcount of S, kept per word in pre) or by w's hash slot --
// and flushed with one atomic per distinct w at the end of the row.  on = false
// (|A_ix[u]| > kVtxSlots, |A_ij[u]| >= 2^16, or the search fallback) means one
// global atomic per hit.
struct VCnt {
    uint32_t* cnt;                     // u16 x kVtxSlots, packed in pairs
    uint32_t* pre;                     // u16 per kPreGroup words of S: popcount of S[0..g*kPreGroup)
    unsigned long long* tvx;           // global t(v) of part x
    bool on;
};
__device__ __forceinline__ void vcnt_add(uint32_t* cnt, uint32_t idx) {
    atomicAdd(&cnt[idx >> 1], 1u << ((idx & 1u) << 4));
}
__device__ __forceinline__ uint32_t u16_at(const uint32_t* a, uint32_t k) { return (a[k >> 1] >> ((k & 1u) << 4)) & 0xffffu; }
// rank of w (a member of the bitmap set S) among the set's elements
__device__ __forceinline__ uint32_t rank_in_set(const uint32_t* S, const uint32_t* pre, uint32_t w) {
    const uint32_t k = w >> 5, g0 = k - k % kPreGroup;
    uint32_t r = u16_at(pre, k / kPreGroup) + __popc(S[k] & ((1u << (w & 31)) - 1u));
    for (uint32_t z = g0; z < k; ++z) r += __popc(S[z]);
    return r;
}

__device__ __forceinline__ uint32_t hash_slot(uint32_t w, uint32_t hbits) {
    return (w * 2654435761u) >> (32 - hbits);
}

// MODE 3 = the hash set of MODE 1 (<= kFilterSlots slots, words [0, 512) of S) plus
// a 16384-bit filter over a second hash of w in words [512, 1024): most probes
// of an intersection miss, and a miss usually costs one filter bit instead of a
// walk along the open-addressing run.
constexpr uint32_t kFilterSlots = kSetWords / 2;
__device__ __forceinline__ uint32_t filter_bit(uint32_t w) { return (w * 0x9E3779B1u) >> 18; }   // 14 bits

template <int MODE>
__device__ __forceinline__ uint32_t probe(const uint32_t* S, uint32_t w, uint32_t hbits, uint32_t hmask) {
    if (MODE == 0) return (S[w >> 5] >> (w & 31)) & 1u;
    if (MODE == 3) {
        const uint32_t f = filter_bit(w);
        if (!((S[kFilterSlots + (f >> 5)] >> (f & 31)) & 1u)) return 0u;
    }
    uint32_t h = hash_slot(w, hbits), s;
    while ((s = S[h]) != 0u && s != w + 1) h = (h + 1) & hmask;
    return s == w + 1;
}

// hash mode: the slot holding w (w a member), for the per-vertex counters
__device__ __forceinline__ uint32_t hash_find(const uint32_t* S, uint32_t w, uint32_t hbits, uint32_t hmask) {
    uint32_t h = hash_slot(w, hbits);
    while (S[h] != w + 1) h = (h + 1) & hmask;
    return h;
}

// one hit on w (a member of the staged set S of the row)
template <int MODE>
__device__ __forceinline__ void vhit(const VCnt& vc, const uint32_t* S, uint32_t w, uint32_t hbits, uint32_t hmask) {
    if (!vc.on) {
        atomicAdd(vc.tvx + w, 1ull);
        return;
    }
    vcnt_add(vc.cnt, MODE == 0 ? rank_in_set(S, vc.pre, w) : hash_find(S, w, hbits, hmask));
}

// One row u: every v in A_ij[u] (edges e0..e1), 32 at a time (one per lane).
//
// List pairs: the non-empty lists of the batch are one flattened sequence;
// their "index delta" (list start - flattened start) is parked in warp scratch
// by compacted index (ballot + popc); in each round of 32 positions the list of
// position base+l is cur + popc(starts in (base, base+l]), the start mask from
// one __reduce_or_sync and cur from one ballot -- no per-position search.
// Elements probe the staged set S (MODE 0 bitmap, 1 hash).
//
// Dense pairs (A_jx has a bitmap copy BM with W words per row, and v's list is
// longer than W): |A_ix[u] ∩ A_jx[v]| = sum_k popc(S[k] & row_v[k]); the warp is
// split into G = 32/gsz groups (gsz = pow2 >= W, capped at 32), one v per group;
// u's words are held in registers when W <= 32*R (R = 0: read from S).
//
// Skewed pairs (|A_ix[u]| * log2|A_jx[v]| * 6 < |A_jx[v]|: a short u list against
// a long v list): thread per pair -- the lane binary-searches each element of
// A_ix[u] (broadcast by shuffle, ascending, so the search window only shrinks)
// in v's sorted list instead of streaming the whole list.
// Components c of x with lo <= c < hi (the part of a 16-byte vector inside a list)
// probed against S.
// VTX: a hit on w is also counted for w (the triangle's third vertex).
template <int MODE, bool VTX>
__device__ __forceinline__ uint32_t probe1(const uint32_t* S, uint32_t w, uint32_t hbits, uint32_t hmask,
                                           const VCnt& vc) {
    const uint32_t h = probe<MODE>(S, w, hbits, hmask);
    if (VTX && h) vhit<MODE>(vc, S, w, hbits, hmask);
    return h;
}

// n hits on w (a member of S), credited at once (warp-aggregated hits)
template <int MODE>
__device__ __forceinline__ void vhit_n(const VCnt& vc, const uint32_t* S, uint32_t w, uint32_t hbits, uint32_t hmask,
                                       uint32_t n) {
    if (!vc.on) {
        atomicAdd(vc.tvx + w, (unsigned long long)n);
        return;
    }
    const uint32_t idx = MODE == 0 ? rank_in_set(S, vc.pre, w) : hash_find(S, w, hbits, hmask);
    atomicAdd(&vc.cnt[idx >> 1], n << ((idx & 1u) << 4));
}

template <int MODE, bool VTX>
__device__ __forceinline__ uint32_t probe4(const uint32_t* S, const uint4 x, int lo, int hi, uint32_t hbits,
                                           uint32_t hmask, const VCnt& vc) {
    if (VTX && kVtxMatch) {
        // per-vertex kernel: the lanes hitting the same w in one component (a hub w
        // sits in many of the round's lists) add once, with their count -- the
        // shared counters would otherwise serialise the conflicting atomics
        const uint32_t ws[4] = {x.x, x.y, x.z, x.w};
        uint32_t c = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t h = (lo <= j && j < hi) ? probe<MODE>(S, ws[j], hbits, hmask) : 0u;
            c += h;
            const uint32_t hb = __ballot_sync(0xffffffffu, h);
            if (h) {
                const uint32_t m = __match_any_sync(hb, ws[j]);
                if ((threadIdx.x & 31) == __ffs(m) - 1) vhit_n<MODE>(vc, S, ws[j], hbits, hmask, __popc(m));
            }
        }
        return c;
    }
    if (lo <= 0 && hi >= 4)
        return probe1<MODE, VTX>(S, x.x, hbits, hmask, vc) + probe1<MODE, VTX>(S, x.y, hbits, hmask, vc) +
               probe1<MODE, VTX>(S, x.z, hbits, hmask, vc) + probe1<MODE, VTX>(S, x.w, hbits, hmask, vc);
    uint32_t c = 0;
    if (lo <= 0 && 0 < hi) c += probe1<MODE, VTX>(S, x.x, hbits, hmask, vc);
    if (lo <= 1 && 1 < hi) c += probe1<MODE, VTX>(S, x.y, hbits, hmask, vc);
    if (lo <= 2 && 2 < hi) c += probe1<MODE, VTX>(S, x.z, hbits, hmask, vc);
    if (lo <= 3 && 3 < hi) c += probe1<MODE, VTX>(S, x.w, hbits, hmask, vc);
    return c;
}

__device__ __forceinline__ uint32_t log2ceil(uint32_t x) { return x <= 1 ? 0 : 32 - __clz(x - 1); }

// Dense pairs of the per-vertex kernel (VM >= 3): every hit w must be credited,
// and hits concentrate on a few hub words, so instead of a per-bit loop per lane
// (a lane holding a hub word serialises the warp) each lane counts its word's
// hits over the batch's v's in six bit-sliced counters c0..c5 (bit b of c_j =
// bit j of w = 32k + b's count; <= 32 v's per batch) with a ripple-carry add
// per v, and credits each w once per batch with its count.  Lane (g, kl) takes
// words kl, kl + gsz, ... and the v's g, g + G, ... (G groups of gsz lanes, as
// the counting path).  pairs: each v's c_uv is also summed into scratch[128 + q].
__device__ __forceinline__ uint32_t and_vtx(const uint32_t* S, const uint32_t* __restrict__ BM, uint32_t W,
                                            uint32_t na, uint32_t* scratch, uint32_t gsz, uint32_t G, uint32_t g,
                                            uint32_t kl, const VCnt& vc, bool pairs) {
    const uint32_t FULL = 0xffffffffu;
    uint32_t acc = 0;
    for (uint32_t k0 = 0; k0 < W; k0 += gsz) {
        const uint32_t k = k0 + kl;
        const uint32_t s = k < W ? S[k] : 0u;
        if (!__any_sync(FULL, s)) continue;
        uint32_t c0 = 0, c1 = 0, c2 = 0, c3 = 0, c4 = 0, c5 = 0;
        const uint32_t nq = (na + G - 1) / G;
#pragma unroll 4
        for (uint32_t i = 0; i < nq; ++i) {
            const uint32_t q = g + G * i;
            uint32_t x = 0;
            if (q < na && s) x = s & __ldg(BM + (uint64_t)scratch[32 + q] * W + k);
            const uint32_t px = __popc(x);
            acc += px;
            if (pairs) {
                uint32_t pc = px;
                if (G == 1) {
                    pc = __reduce_add_sync(FULL, pc);
                } else {
                    for (uint32_t o = gsz >> 1; o; o >>= 1) pc += __shfl_xor_sync(FULL, pc, o);
                }
                if (kl == 0 && q < na && pc) scratch[128 + q] += pc;
            }
            uint32_t cy = x, t;
            t = c0 & cy; c0 ^= cy; cy = t;
            t = c1 & cy; c1 ^= cy; cy = t;
            t = c2 & cy; c2 ^= cy; cy = t;
            t = c3 & cy; c3 ^= cy; cy = t;
            t = c4 & cy; c4 ^= cy; cy = t;
            c5 ^= cy;
        }
        for (uint32_t nz = c0 | c1 | c2 | c3 | c4 | c5; nz; nz &= nz - 1u) {
            const uint32_t b = __ffs(nz) - 1;
            const uint32_t cnt = ((c0 >> b) & 1u) | ((c1 >> b) & 1u) << 1 | ((c2 >> b) & 1u) << 2 |
                                 ((c3 >> b) & 1u) << 3 | ((c4 >> b) & 1u) << 4 | ((c5 >> b) & 1u) << 5;
            const uint32_t w = 32u * k + b;
            if (vc.on) {
                const uint32_t idx = rank_in_set(S, vc.pre, w);
                atomicAdd(&vc.cnt[idx >> 1], cnt << ((idx & 1u) << 4));
            } else {
                atomicAdd(vc.tvx + w, (unsigned long long)cnt);
            }
        }
    }
    return acc;
}

// VM (per-vertex roles, NEXT-1): VM >= 2 adds each pair's count c_uv to tvj[v],
// VM >= 3 counts each common element w for w (warp counters, VCnt); the row
// total goes to u in the caller (VM >= 1).  VM = 0 is exactly the counting kernel.
// POS (MID tasks with x == j, R25): each neighbour's streamed list starts after the
// row vertex, at npos[e] + 1, instead of at its rowptr (a compile-time switch: the
// runtime select measured 7 % on every LOW launch)
template <int MODE, int R, int VM, bool POS>
__device__ __forceinline__ uint32_t intersect_row(const uint32_t* __restrict__ vcol, uint32_t e0, uint32_t e1,
                                                  const uint32_t* __restrict__ npos,
                                                  const uint32_t* __restrict__ rp_jx,
                                                  const uint32_t* __restrict__ Bc,
                                                  const uint32_t* __restrict__ BM, uint32_t W, const uint32_t* S,
                                                  uint32_t* __restrict__ scratch, uint32_t hbits, uint32_t hmask,
                                                  const uint32_t* __restrict__ A, uint32_t la, int lane,
                                                  unsigned long long* __restrict__ tvj,
                                                  const VCnt& vc PROF_ARGS) {
    const uint32_t lt_mask = (1u << lane) - 1u;
    const uint32_t le_mask = 0xffffffffu >> (31 - lane);
    uint32_t gsz = 1;
    while (gsz < W && gsz < 32) gsz <<= 1;
    const uint32_t G = 32 / gsz, g = lane / gsz, kl = lane % gsz;
    uint32_t su[R > 0 ? R : 1];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const uint32_t k = kl + r * 32;
        su[r] = (BM != nullptr && k < W) ? S[k] : 0u;
    }
    uint32_t acc = 0;
    const uint4* __restrict__ V = reinterpret_cast<const uint4*>((uintptr_t)Bc & ~uintptr_t(15));
    const uint32_t coff = (uint32_t)(((uintptr_t)Bc & 15) >> 2);   // Bc[0] is word coff of V
    for (uint32_t e = e0; e < e1; e += 32) {
        uint32_t v = 0, b0 = 0, lb = 0;
        if (e + lane < e1) {
            v = __ldg(vcol + e + lane);
            const uint32_t bend = __ldg(rp_jx + v + 1);
            // MID with x == j: the neighbour's list starts after the row vertex (R25)
            b0 = POS ? __ldg(npos + e + lane) + 1 : __ldg(rp_jx + v);
            lb = bend - b0;
        }
        PROF_MARK(9);
        // dense pairs: AND of bitmap rows
        const bool use_and = (BM != nullptr) && lb > W;
        const uint32_t and_mask = __ballot_sync(0xffffffffu, use_and);
        if (and_mask) {
            __syncwarp();
            if (use_and) scratch[32 + __popc(and_mask & lt_mask)] = v;
            if (VM >= 1) scratch[128 + lane] = 0u;   // per-pair counts (the group's lanes add into one)
            __syncwarp();
            const uint32_t na = __popc(and_mask);
            // kAndUnroll v's per group per step: their row words are loaded before
            // any is used, so that many loads are in flight per lane
            constexpr int U = R > 0 ? kAndUnroll : 1;
            if (VM >= 3 && kVtxSliced) acc += and_vtx(S, BM, W, na, scratch, gsz, G, g, kl, vc, tvj != nullptr);
            else
            for (uint32_t q = 0; q < na; q += U * G) {
                uint32_t vqs[U], wds[U][R > 0 ? R : 1];
#pragma unroll
                for (int z = 0; z < U; ++z) {
                    const uint32_t qq = q + z * G + g;
                    vqs[z] = qq < na ? scratch[32 + qq] : 0xffffffffu;
                    if (R > 0) {
                        const uint32_t* __restrict__ row = BM + (uint64_t)(qq < na ? vqs[z] : 0u) * W + kl;
#pragma unroll
                        for (int r = 0; r < R; ++r)
                            wds[z][r] = (qq < na && kl + r * 32 < W) ? __ldg(row + r * 32) : 0u;
                    }
                }
#pragma unroll
                for (int z = 0; z < U; ++z) {
                    if (vqs[z] == 0xffffffffu) continue;
                    const uint32_t vq = vqs[z];
                    uint32_t cv = 0;
                    if (R > 0) {
#pragma unroll
                        for (int r = 0; r < R; ++r) {
                            uint32_t wd = su[r] & wds[z][r];
                            cv += __popc(wd);
                            if (VM >= 3)
                                for (; wd; wd &= wd - 1u)
                                    vhit<0>(vc, S, 32u * (kl + r * 32) + (__ffs(wd) - 1), 0, 0);
                        }
                    } else {
                        const uint32_t* __restrict__ row = BM + (uint64_t)vq * W + kl;
#pragma unroll 4
                        for (uint32_t k = kl; k < W; k += gsz) {
                            uint32_t wd = S[k] & __ldg(row + (k - kl));
                            cv += __popc(wd);
                            if (VM >= 3)
                                for (; wd; wd &= wd - 1u) vhit<0>(vc, S, 32u * k + (__ffs(wd) - 1), 0, 0);
                        }
                    }
                    acc += cv;
                    if (VM >= 1 && tvj && cv) atomicAdd(&scratch[128 + q + z * G + g], cv);
                }
            }
            if (VM >= 1 && tvj) {   // one global atomic per pair, not one per lane of its group
                __syncwarp();
                if ((uint32_t)lane < na && scratch[128 + lane])
                    atomicAdd(tvj + scratch[32 + lane], (unsigned long long)scratch[128 + lane]);
                __syncwarp();
            }
            if (use_and) lb = 0;
            PROF_MARK(3);
        }
        // skewed pairs: binary search of u's elements in v's list
        const bool use_search = lb > 0 && la * log2ceil(lb + 1) * 6u < lb;
        if (__any_sync(0xffffffffu, use_search)) {
            uint32_t lo = 0, cv = 0;
            for (uint32_t c = 0; c < la; c += 32) {
                const uint32_t a = (c + lane < la) ? __ldg(A + c + lane) : 0u;
                const uint32_t m = min(32u, la - c);
                for (uint32_t k = 0; k < m; ++k) {
                    const uint32_t ak = __shfl_sync(0xffffffffu, a, k);
                    if (use_search) {
                        uint32_t hi = lb;
                        while (lo < hi) {
                            const uint32_t mid = (lo + hi) >> 1;
                            if (__ldg(Bc + b0 + mid) < ak) lo = mid + 1; else hi = mid;
                        }
                        const uint32_t hit = (lo < lb && __ldg(Bc + b0 + lo) == ak);
                        if (VM >= 3 && hit) {
                            if (vc.on) vcnt_add(vc.cnt, MODE == 0 ? c + k : hash_find(S, ak, hbits, hmask));
                            else atomicAdd(vc.tvx + ak, 1ull);
                        }
                        cv += hit;
                    }
                }
            }
            acc += cv;
            if (VM >= 1 && tvj && cv) atomicAdd(tvj + v, (unsigned long long)cv);
            if (use_search) lb = 0;
            PROF_MARK(4);
        }
        // list pairs: the 16-byte-aligned covers of the batch's remaining lists are
        // one flattened sequence of uint4 vectors (4 ids each; pools are padded so a
        // cover never leaves its allocation).  Lane l takes vector positions l, l+32,
        // ... two rounds at a time (two 16-byte loads in flight per lane); the list of
        // a position is cur + popc(list starts in (round base, position]), the start
        // mask from one __reduce_or_sync and cur from one ballot.  Ids outside the
        // list's [lo, hi) word range (cover head/tail) are masked.
        const uint32_t nonempty = __ballot_sync(0xffffffffu, lb > 0);
        if (nonempty == 0u) continue;
        const uint32_t lo = coff + b0, hi = lo + lb;        // word range in V space
        const uint32_t nv = lb ? ((hi + 3) >> 2) - (lo >> 2) : 0u;
        uint32_t incl = nv;   // inclusive prefix of cover lengths over the batch
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        const uint32_t excl = incl - nv;
        __syncwarp();
        if (lb > 0) {
            const uint32_t sidx = __popc(nonempty & lt_mask);
            scratch[sidx] = (lo >> 2) - excl;
            scratch[32 + sidx] = lo;
            scratch[64 + sidx] = hi;
            if (VM >= 1) {
                scratch[96 + sidx] = v;
                scratch[128 + sidx] = 0u;   // the pair's count c_uv, summed over the rounds
            }
        }
        __syncwarp();
        // cur = (number of lists starting before the round) - 1, carried from round to
        // round: a list starting at position rb + i (0 <= i < 32) sets bit i of starts
        int cur = -1;
        for (uint32_t base = 0; base < total; base += 32 * kListUnroll) {
            uint32_t vpos[kListUnroll], wlo[kListUnroll], whi[kListUnroll], vv[kListUnroll];
            uint4 x[kListUnroll];
#pragma unroll
            for (int r = 0; r < kListUnroll; ++r) {
                const uint32_t rb = base + 32 * r;
                const uint32_t in = excl - rb;
                uint32_t bit;
                if (kCarryCur) {
                    bit = (lb > 0 && excl >= rb && in < 32u) ? (1u << in) : 0u;
                } else {
                    bit = (lb > 0 && excl > rb && in < 32u) ? (1u << in) : 0u;
                    cur = __popc(__ballot_sync(0xffffffffu, lb > 0 && excl <= rb)) - 1;
                }
                const uint32_t starts = __reduce_or_sync(0xffffffffu, bit);
                const uint32_t pos = rb + lane;
                wlo[r] = 1u;
                whi[r] = 0u;
                x[r] = make_uint4(0, 0, 0, 0);
                vpos[r] = 0;
                vv[r] = 0;
                if (pos < total) {
                    const uint32_t seg = cur + __popc(starts & le_mask);
                    vpos[r] = pos + scratch[seg];
                    wlo[r] = scratch[32 + seg];
                    whi[r] = scratch[64 + seg];
                    if (VM >= 1) vv[r] = seg;
                    x[r] = __ldg(V + vpos[r]);
                }
                if (kCarryCur) cur += __popc(starts);
            }
#pragma unroll
            for (int r = 0; r < kListUnroll; ++r) {
                const int w0 = 4 * (int)vpos[r];
                const uint32_t c = probe4<MODE, (VM >= 3)>(S, x[r], (int)wlo[r] - w0, (int)whi[r] - w0, hbits, hmask, vc);
                acc += c;
                // per-pair count in shared memory: one global atomic per pair (below)
                // instead of one per 16-byte position -- a hub v is the middle vertex
                // of millions of triangles, and same-address global atomics serialize
                if (VM >= 1 && tvj && c) atomicAdd(&scratch[128 + vv[r]], c);
            }
        }
        if (VM >= 1 && tvj) {
            __syncwarp();
            if (lane < __popc(nonempty)) {
                const uint32_t c = scratch[128 + lane];
                if (c) atomicAdd(tvj + scratch[96 + lane], (unsigned long long)c);
            }
        }
        PROF_MARK(6);
    }
    return acc;
}

// Dense A_jx and a short A_ix[u] (|A_ix[u]| <= 2W): thread per pair -- lane l
// takes v_l and tests each element a of A_ix[u] (broadcast by shuffle) against
// bit a of v_l's bitmap row.  Costs |A_ix[u]| bit tests per pair instead of W
// word ANDs, and needs no staging of u at all.
template <int VM>
__device__ __forceinline__ uint32_t probe_dense_row(const uint32_t* __restrict__ vcol, uint32_t e0, uint32_t e1,
                                                    const uint32_t* __restrict__ A, uint32_t la,
                                                    const uint32_t* __restrict__ BM, uint32_t W, int lane,
                                                    unsigned long long* __restrict__ tvj,
                                                    unsigned long long* __restrict__ tvx) {
    uint32_t acc = 0;
    const uint32_t ne = e1 - e0;
    if (ne < 32) {
        // fewer pairs than lanes: flatten (pair q, element k) over the lanes, so
        // every lane tests a bit; position pos = q * la + k advances by 32 per round
        const uint32_t vq = (lane < ne) ? __ldg(vcol + e0 + lane) : 0u;
        uint32_t q = lane / la, k = lane - q * la;
        const uint32_t dq = 32 / la, dk = 32 - dq * la;
        const uint32_t P = ne * la;
        for (uint32_t base = 0; base < P; base += 32) {
            const uint32_t v = __shfl_sync(0xffffffffu, vq, q & 31);
            uint32_t hit = 0, a = 0;
            if (base + lane < P) {
                a = __ldg(A + k);
                hit = (__ldg(BM + (uint64_t)v * W + (a >> 5)) >> (a & 31)) & 1u;
                acc += hit;
            }
            if (VM >= 3) {   // lanes hitting the same w add once (warp-aggregated)
                const uint32_t same = __match_any_sync(0xffffffffu, hit ? a : 0xffffffffu);
                if (hit && lane == __ffs(same) - 1) atomicAdd(tvx + a, (unsigned long long)__popc(same));
            }
            if (VM >= 1 && tvj && hit) atomicAdd(tvj + v, 1ull);
            q += dq;
            k += dk;
            if (k >= la) {
                k -= la;
                ++q;
            }
        }
        return acc;
    }
    for (uint32_t e = e0; e < e1; e += 32) {
        const bool ok = e + lane < e1;
        const uint32_t v = ok ? __ldg(vcol + e + lane) : 0u;
        const uint32_t* __restrict__ row = BM + (uint64_t)v * W;
        uint32_t cv = 0;
        for (uint32_t c = 0; c < la; c += 32) {
            const uint32_t a = (c + lane < la) ? __ldg(A + c + lane) : 0u;
            const uint32_t m = min(32u, la - c);
            for (uint32_t k = 0; k < m; k += kDenseUnroll) {
                uint32_t ak[kDenseUnroll], wv[kDenseUnroll];
#pragma unroll
                for (int z = 0; z < kDenseUnroll; ++z) ak[z] = __shfl_sync(0xffffffffu, a, (k + z) & 31);
#pragma unroll
                for (int z = 0; z < kDenseUnroll; ++z) wv[z] = (ok && k + z < m) ? __ldg(row + (ak[z] >> 5)) : 0u;
#pragma unroll
                for (int z = 0; z < kDenseUnroll; ++z) {
                    const uint32_t hit = (wv[z] >> (ak[z] & 31)) & 1u;
                    cv += hit;
                    if (VM >= 3 && k + z < m) {   // one atomic per element for the whole warp's v's
                        const uint32_t mk = __ballot_sync(0xffffffffu, hit);
                        if (lane == 0 && mk) atomicAdd(tvx + ak[z], (unsigned long long)__popc(mk));
                    }
                }
            }
        }
        acc += cv;
        if (VM >= 1 && tvj && cv) atomicAdd(tvj + v, (unsigned long long)cv);
    }
    return acc;
}

// ---------------------------------------------------------------------------
// Batched small rows (VM = 0): the 32 items a warp claims are loaded one per
// lane; the rows whose streamed block has no dense copy, |A_ix[u]| <= kBatchLa
// and <= 32 neighbours ("small") are intersected in batches of consecutive
// small rows of one task with <= 32 neighbours in total, so the warp's lanes
// carry up to 32 pairs (u, v) of several rows at once instead of one row's few
// (an ER row at p = 1 has ~16): per batch one hash region per row in the warp's
// set S (2^hb >= 2|A_ix[u]| slots, open addressing, slots hold w + 1), one lane
// per pair loads v and its list bounds, skewed pairs binary-search the row's
// held ids in v's list, and the rest are one flattened sequence of 16-byte
// covers probed against their row's region (as intersect_row).  Same exact
// |A_ix[u] ∩ A_jx[v]| sums (Listing 5).  Returns the mask of
// lanes whose (valid) item is not small: the caller runs those one at a time.
__device__ __forceinline__ uint32_t region_probe(const uint32_t* S, uint32_t w, uint32_t desc) {
    const uint32_t ro = desc & 0xfffu, hb = (desc >> 12) & 15u, hm = (1u << hb) - 1u;
    uint32_t h = hash_slot(w, hb), s;
    while ((s = S[ro + h]) != 0u && s != w + 1) h = (h + 1) & hm;
    return s == w + 1;
}

__device__ __forceinline__ uint32_t batch_rows(unsigned long long my_it, bool valid,
                                               const TaskDev* __restrict__ tasks,
                                               const uint32_t* __restrict__ col,
                                               const uint32_t* __restrict__ rowptr, uint32_t* S,
                                               uint32_t* scratch, int lane, uint32_t& cur_t,
                                               unsigned long long& acc_t,
                                               unsigned long long* __restrict__ task_counts) {
    const uint32_t FULL = 0xffffffffu;
    const uint32_t lt_mask = (1u << lane) - 1u;
    const uint32_t le_mask = 0xffffffffu >> (31 - lane);
    const uint32_t t = (uint32_t)(my_it >> 48), chunk = (uint32_t)(my_it >> 32) & 0xffffu, u = (uint32_t)my_it;
    bool small = false;
    uint32_t la = 0, ne = 0, a0 = 0, e0 = 0;
    if (valid && chunk == 0) {
        const TaskDev& T = tasks[t];
        if (T.t_bm == ~0ull) {
            a0 = __ldg(rowptr + T.s_rp + u);
            la = __ldg(rowptr + T.s_rp + u + 1) - a0;
            e0 = __ldg(rowptr + T.n_rp + u);
            ne = __ldg(rowptr + T.n_rp + u + 1) - e0;
            small = la > 0 && ne > 0 && la <= kBatchLa && ne <= 32u;
        }
    }
    const uint32_t smask = __ballot_sync(FULL, small);
    const uint32_t rest = __ballot_sync(FULL, valid) & ~smask;
    uint32_t todo = smask;
    while (todo) {
        // the batch: the next small rows of the first one's task while the pairs fit
        // the lanes and the regions the set
        const int r0 = __ffs(todo) - 1;
        const uint32_t t0 = __shfl_sync(FULL, t, r0);
        const bool cand = ((todo >> lane) & 1u) && t == t0;
        uint32_t hb = 2;
        while ((1u << hb) < 2 * la) ++hb;
        const uint32_t hs = cand ? (1u << hb) : 0u;
        uint32_t incl = cand ? (ne | hs << 16) : 0u;   // ne <= 32, hs <= 64: 16-bit halves do not overflow
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
        }
        const uint32_t incl_ne = incl & 0xffffu, incl_hs = incl >> 16;
        const bool inb = cand && incl_ne <= 32u && incl_hs <= kSetWords;
        const uint32_t B = __ballot_sync(FULL, inb);
        todo &= ~B;
        const int rl = 31 - __clz(B);
        const uint32_t P = __shfl_sync(FULL, incl_ne, rl);      // pairs in the batch (<= 32)
        const uint32_t HS = __shfl_sync(FULL, incl_hs, rl);     // set words in use
        const TaskDev& T = tasks[t0];
        const uint32_t* __restrict__ A0 = col + T.s_col;
        // rows by ordinal o (lane order within B): held start, region desc, la prefix
        uint32_t incl_la = inb ? la : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, incl_la, o);
            if (lane >= o) incl_la += y;
        }
        const uint32_t LA = __shfl_sync(FULL, incl_la, rl);
        const uint32_t excl_la = incl_la - (inb ? la : 0u);
        const uint32_t ord = __popc(B & lt_mask);
        const uint32_t desc = (incl_hs - hs) | hb << 12 | la << 16;
        __syncwarp();
        if (inb) {
            scratch[ord] = a0;
            scratch[32 + ord] = desc;
            scratch[64 + ord] = excl_la;
        }
        __syncwarp();
        // stage: the held ids of all rows, flattened over the lanes
        for (uint32_t rb = 0; rb < LA; rb += 32) {
            const uint32_t in = excl_la - rb;
            const uint32_t bit = (inb && excl_la >= rb && in < 32u) ? (1u << in) : 0u;
            const uint32_t starts = __reduce_or_sync(FULL, bit);
            const int cur = __popc(__ballot_sync(FULL, inb && excl_la < rb)) - 1;
            const uint32_t q = rb + lane;
            if (q < LA) {
                const uint32_t o = cur + __popc(starts & le_mask);
                const uint32_t d = scratch[32 + o];
                const uint32_t w = __ldg(A0 + scratch[o] + (q - scratch[64 + o]));
                const uint32_t ro = d & 0xfffu, hbo = (d >> 12) & 15u, hm = (1u << hbo) - 1u;
                uint32_t h = hash_slot(w, hbo);
                while (atomicCAS(&S[ro + h], 0u, w + 1) != 0u) h = (h + 1) & hm;
            }
        }
        __syncwarp();
        if (inb) scratch[64 + ord] = e0 - (incl_ne - ne);   // pair l of this row: neighbour e = this + l
        __syncwarp();
        // one lane per pair: v, its list bounds, its row's region
        const uint32_t ebit = (inb) ? (1u << (incl_ne - ne)) : 0u;
        const uint32_t pstarts = __reduce_or_sync(FULL, ebit);
        uint32_t v = 0, b0 = 0, lb = 0, pd = 0, pa0 = 0;
        if ((uint32_t)lane < P) {
            const uint32_t o = __popc(pstarts & le_mask) - 1;
            pa0 = scratch[o];
            pd = scratch[32 + o];
            const uint32_t e = scratch[64 + o] + lane;
            v = __ldg(col + T.n_col + e);
            const uint32_t bend = __ldg(rowptr + T.t_rp + v + 1);
            b0 = T.n_pos != ~0ull ? __ldg(col + T.n_pos + e) + 1 : __ldg(rowptr + T.t_rp + v);
            lb = bend - b0;
        }
        const uint32_t* __restrict__ Bc = col + T.t_col;
        uint32_t acc = 0;
        // skewed pairs: the row's held ids binary-searched in v's list (ascending, so
        // the window only shrinks)
        const uint32_t pla = pd >> 16;
        if (lb > 0 && pla * log2ceil(lb + 1) * 6u < lb) {
            uint32_t lo = 0;
            for (uint32_t k = 0; k < pla; ++k) {
                const uint32_t ak = __ldg(A0 + pa0 + k);
                uint32_t hi = lb;
                while (lo < hi) {
                    const uint32_t mid = (lo + hi) >> 1;
                    if (__ldg(Bc + b0 + mid) < ak) lo = mid + 1; else hi = mid;
                }
                acc += (lo < lb && __ldg(Bc + b0 + lo) == ak);
            }
            lb = 0;
        }
        // list pairs: flattened 16-byte covers (see intersect_row), each probed
        // against its own row's region
        const uint32_t nonempty = __ballot_sync(FULL, lb > 0);
        if (nonempty) {
            const uint4* __restrict__ V = reinterpret_cast<const uint4*>((uintptr_t)Bc & ~uintptr_t(15));
            const uint32_t coff = (uint32_t)(((uintptr_t)Bc & 15) >> 2);
            const uint32_t lo = coff + b0, hi = lo + lb;
            const uint32_t nv = lb ? ((hi + 3) >> 2) - (lo >> 2) : 0u;
            uint32_t vin = nv;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(FULL, vin, o);
                if (lane >= o) vin += y;
            }
            const uint32_t total = __shfl_sync(FULL, vin, 31);
            const uint32_t excl = vin - nv;
            __syncwarp();
            if (lb > 0) {
                const uint32_t sidx = __popc(nonempty & lt_mask);
                scratch[sidx] = (lo >> 2) - excl;
                scratch[32 + sidx] = lo;
                scratch[64 + sidx] = hi;
                scratch[96 + sidx] = pd;
            }
            __syncwarp();
            for (uint32_t base = 0; base < total; base += 64) {
                uint32_t vpos[2], wlo[2], whi[2], dd[2];
                uint4 x[2];
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    const uint32_t rb = base + 32 * r;
                    const uint32_t in = excl - rb;
                    const uint32_t bit = (lb > 0 && excl > rb && in < 32u) ? (1u << in) : 0u;
                    const uint32_t starts = __reduce_or_sync(FULL, bit);
                    const int cur = __popc(__ballot_sync(FULL, lb > 0 && excl <= rb)) - 1;
                    const uint32_t pos = rb + lane;
                    wlo[r] = 1u;
                    whi[r] = 0u;
                    x[r] = make_uint4(0, 0, 0, 0);
                    vpos[r] = 0;
                    dd[r] = 0;
                    if (pos < total) {
                        const uint32_t seg = cur + __popc(starts & le_mask);
                        vpos[r] = pos + scratch[seg];
                        wlo[r] = scratch[32 + seg];
                        whi[r] = scratch[64 + seg];
                        dd[r] = scratch[96 + seg];
                        x[r] = __ldg(V + vpos[r]);
                    }
                }
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    const int w0 = 4 * (int)vpos[r];
                    const int l0 = (int)wlo[r] - w0, h0 = (int)whi[r] - w0;
                    if (l0 <= 0 && 0 < h0) acc += region_probe(S, x[r].x, dd[r]);
                    if (l0 <= 1 && 1 < h0) acc += region_probe(S, x[r].y, dd[r]);
                    if (l0 <= 2 && 2 < h0) acc += region_probe(S, x[r].z, dd[r]);
                    if (l0 <= 3 && 3 < h0) acc += region_probe(S, x[r].w, dd[r]);
                }
            }
        }
        __syncwarp();
        for (uint32_t k = lane; k < HS; k += 32) S[k] = 0u;   // the set is all-zero between rows
        __syncwarp();
        const uint32_t sum = __reduce_add_sync(FULL, acc);
        if (t0 != cur_t) {
            if (lane == 0 && acc_t) atomicAdd(&task_counts[cur_t], acc_t);
            cur_t = t0;
            acc_t = 0;
        }
        acc_t += sum;
    }
    return rest;
}

constexpr int kLightThreads = 256;
#ifndef PGABB_LIGHT_MINB
#define PGABB_LIGHT_MINB 6   // 6 x 256 threads per SM (40 registers, with the item prefetch): A/B best on c2/c3/c4
#endif
#ifndef PGABB_LIGHT_CHUNK
#define PGABB_LIGHT_CHUNK 8
#endif
constexpr int kLightChunk = PGABB_LIGHT_CHUNK;   // items per lane per claim
#ifndef PGABB_LIGHT_PREFETCH
#define PGABB_LIGHT_PREFETCH 1
#endif
constexpr bool kLightPrefetch = PGABB_LIGHT_PREFETCH;
#ifndef PGABB_LIGHT_VPIPE
#define PGABB_LIGHT_VPIPE 1
#endif
constexpr bool kLightVPipe = PGABB_LIGHT_VPIPE;
#ifndef PGABB_LIGHT_VEC
#define PGABB_LIGHT_VEC 0   // A/B: c3 p=4 -1 %, p=8 +5 %, c4 +31 %
#endif
constexpr bool kLightVec = PGABB_LIGHT_VEC;   // scanned lists read as aligned 16-byte chunks
#ifndef PGABB_LIGHT_CS
#define PGABB_LIGHT_CS 0
#endif
constexpr bool kLightCs = PGABB_LIGHT_CS;   // light items / held / neighbour ids loaded evict-first (ld.global.cs)
template <class T>
__device__ __forceinline__ T ld_stream(const T* p) {
    if constexpr (kLightCs) return __ldcs(p);
    else return __ldg(p);
}
#ifndef PGABB_LIGHT_AVEC
#define PGABB_LIGHT_AVEC 0
#endif
constexpr bool kLightAVec = PGABB_LIGHT_AVEC;   // held ids (<= 8) read as aligned 16-byte chunks

// The list branch of a light row: for each neighbour v (vcol[e0..e1)) its streamed
// list Bc[b0..b1) -- from rowptr, or (POS: MID tasks with x == j) from after the
// row vertex, npos[e] + 1 -- is scanned against the held ids a[] (<= kLightScan
// ids) or binary-searched once per held id.  The next neighbour and its bounds are
// loaded while the current list is scanned (PGABB_LIGHT_VPIPE).
// LA: a bound on |held| for the whole warp (1, 2, 4 or kLightLa), so a scanned id
// is compared with LA held slots, not kLightLa (unused slots are ~0u).
// STRIDE: the thread takes neighbours e0, e0 + STRIDE, ... (1 in the light kernel;
// 32 when the lanes of a warp share one row, the heavy kernel's small-held path).
template <int VM, bool POS, int LA, int STRIDE = 1, int HELD>
__device__ __forceinline__ uint32_t light_lists(const uint32_t* __restrict__ col, const uint32_t* __restrict__ rowptr,
                                                const uint32_t* __restrict__ vcol, const uint32_t* __restrict__ npos,
                                                uint64_t rp_jx, const uint32_t* __restrict__ Bc, uint32_t e0,
                                                uint32_t e1, const uint32_t (&a)[HELD], uint32_t la,
                                                unsigned long long* __restrict__ tvj,
                                                unsigned long long* __restrict__ tvx) {
    uint32_t acc = 0;
    uint32_t vn = 0, bn0 = 0, bn1 = 0;
    if (kLightVPipe && e0 < e1) {
        vn = STRIDE == 1 ? ld_stream(vcol + e0) : __ldg(vcol + e0);
        bn0 = POS ? __ldg(npos + e0) + 1 : __ldg(rowptr + rp_jx + vn);
        bn1 = __ldg(rowptr + rp_jx + vn + 1);
    }
    for (uint32_t e = e0; e < e1; e += STRIDE) {
        uint32_t v, b0, b1;
        if (kLightVPipe) {
            v = vn;
            b0 = bn0;
            b1 = bn1;
            if (e + STRIDE < e1) {
                vn = STRIDE == 1 ? ld_stream(vcol + e + STRIDE) : __ldg(vcol + e + STRIDE);
                bn0 = POS ? __ldg(npos + e + STRIDE) + 1 : __ldg(rowptr + rp_jx + vn);
                bn1 = __ldg(rowptr + rp_jx + vn + 1);
            }
        } else {
            v = __ldg(vcol + e);
            b0 = POS ? __ldg(npos + e) + 1 : __ldg(rowptr + rp_jx + v);
            b1 = __ldg(rowptr + rp_jx + v + 1);
        }
        const uint32_t lb = b1 - b0;
        uint32_t c = 0;
        if (kLightVec && STRIDE == 1 && lb <= kLightScan) {
            // the list's aligned 16-byte chunks (one L2 request each instead of one per
            // id; the pools are padded, so a chunk never leaves the allocation); ids
            // outside [b0, b1) are masked out of the hits
            const uintptr_t pa = reinterpret_cast<uintptr_t>(Bc + b0);
            const uint4* c4 = reinterpret_cast<const uint4*>(pa & ~(uintptr_t)15);
            const int off = (int)((pa >> 2) & 3);
            const int nch = (off + (int)lb + 3) >> 2;
            for (int ch = 0; ch < nch; ++ch) {
                const uint4 w4 = __ldg(c4 + ch);
                const uint32_t ws[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int idx = 4 * ch + j - off;
                    uint32_t hit = 0;
#pragma unroll
                    for (int k = 0; k < LA; ++k) hit |= (ws[j] == a[k]);
                    hit &= (uint32_t)(idx >= 0 && idx < (int)lb);
                    if (VM >= 3 && hit) atomicAdd(tvx + ws[j], 1ull);
                    c += hit;
                }
            }
        } else if (lb <= kLightScan) {
            for (uint32_t q = b0; q < b1; ++q) {
                const uint32_t x = __ldg(Bc + q);
                uint32_t hit = 0;
#pragma unroll
                for (int k = 0; k < LA; ++k) hit |= (x == a[k]);
                if (VM >= 3 && hit) atomicAdd(tvx + x, 1ull);
                c += hit;
            }
        } else {
#pragma unroll
            for (int k = 0; k < LA; ++k)
                if (k < (int)la) {
                    uint32_t lo = b0, hi = b1;
                    while (lo < hi) {
                        const uint32_t mid = (lo + hi) >> 1;
                        if (__ldg(Bc + mid) < a[k]) lo = mid + 1; else hi = mid;
                    }
                    const uint32_t hit = (lo < b1 && __ldg(Bc + lo) == a[k]);
                    if (VM >= 3 && hit) atomicAdd(tvx + a[k], 1ull);
                    c += hit;
                }
        }
        acc += c;
        if (VM >= 1 && tvj && c) atomicAdd(tvj + v, (unsigned long long)c);
    }
    return acc;
}

// R30: the list branch over the streamed block's sector-aligned slots (LOW tasks of
// device-resident ER-like graphs): one aligned EW-word segment per neighbour v holds
// |A_jx[v]| and its first EW-1 ids, compared with the held ids; a longer list goes
// on in the col pool after its first EW-1 ids (scanned, or binary-searched per held
// id when long).  The next neighbour id is loaded while the current slot is used.
template <int VM, int LA, int EW, int HELD>
__device__ __forceinline__ uint32_t light_ell(const uint32_t* __restrict__ rowptr, const uint32_t* __restrict__ vcol,
                                              uint64_t rp_jx, const uint32_t* __restrict__ Bc,
                                              const uint32_t* __restrict__ ell, uint32_t e0, uint32_t e1,
                                              const uint32_t (&a)[HELD], uint32_t la,
                                              unsigned long long* __restrict__ tvj,
                                              unsigned long long* __restrict__ tvx) {
    uint32_t acc = 0;
    uint32_t vn = e0 < e1 ? __ldg(vcol + e0) : 0u;
    for (uint32_t e = e0; e < e1; ++e) {
        const uint32_t v = vn;
        if (e + 1 < e1) vn = __ldg(vcol + e + 1);
        const uint4* sp = reinterpret_cast<const uint4*>(ell + (uint64_t)v * EW);
        uint32_t w[EW];
#pragma unroll
        for (int q = 0; q < EW / 4; ++q) {
            const uint4 x = __ldg(sp + q);
            w[4 * q] = x.x;
            w[4 * q + 1] = x.y;
            w[4 * q + 2] = x.z;
            w[4 * q + 3] = x.w;
        }
        const uint32_t len = w[0];
        uint32_t c = 0;
#pragma unroll
        for (int j = 1; j < EW; ++j) {
            uint32_t hit = 0;
#pragma unroll
            for (int k = 0; k < LA; ++k) hit |= (w[j] == a[k]);
            hit &= (uint32_t)((uint32_t)j <= len);
            if (VM >= 3 && hit) atomicAdd(tvx + w[j], 1ull);
            c += hit;
        }
        if (len > (uint32_t)(EW - 1)) {   // the rest of a long list, from the col pool
            const uint32_t b0 = __ldg(rowptr + rp_jx + v) + (EW - 1), b1 = __ldg(rowptr + rp_jx + v + 1);
            if (b1 - b0 <= kLightScan) {
                for (uint32_t q = b0; q < b1; ++q) {
                    const uint32_t x = __ldg(Bc + q);
                    uint32_t hit = 0;
#pragma unroll
                    for (int k = 0; k < LA; ++k) hit |= (x == a[k]);
                    if (VM >= 3 && hit) atomicAdd(tvx + x, 1ull);
                    c += hit;
                }
            } else {
#pragma unroll
                for (int k = 0; k < LA; ++k)
                    if (k < (int)la) {
                        uint32_t lo = b0, hi = b1;
                        while (lo < hi) {
                            const uint32_t mid = (lo + hi) >> 1;
                            if (__ldg(Bc + mid) < a[k]) lo = mid + 1; else hi = mid;
                        }
                        const uint32_t hit = (lo < b1 && __ldg(Bc + lo) == a[k]);
                        if (VM >= 3 && hit) atomicAdd(tvx + a[k], 1ull);
                        c += hit;
                    }
            }
        }
        acc += c;
        if (VM >= 1 && tvj && c) atomicAdd(tvj + v, (unsigned long long)c);
    }
    return acc;
}

// items[] holds the row items in locality order: the whole rank's (device-resident
// blocks) or one wave's range of them (streaming residency: the task table and the
// pool pointers then all point at the wave's staging arena).
// VM > 0 (per-vertex counts, NEXT-1): tv[rank-space id] += the triangles found
// here that contain the vertex in the requested roles -- u gets the row total
// (VM >= 1), v each pair's c_uv (VM >= 2), w one per hit (VM >= 3) -- so with
// VM = 3 the sum over ranks of tv is t(v) and sum tv = 3T.
// TIMED (pgabb_task_times only): lane 0 adds each item's clock64 span to cyc[t].
#define IROW(M, R_, ...) \
    (npos ? intersect_row<M, R_, VM, true>(__VA_ARGS__) : intersect_row<M, R_, VM, false>(__VA_ARGS__))
#ifndef PGABB_ROW_MINB_VTX
#define PGABB_ROW_MINB_VTX 4
#endif
constexpr int kRowMinBlocksVtx = PGABB_ROW_MINB_VTX;   // the VM = 3 kernel: 64 registers (bit-sliced counters)
template <int VM, bool TIMED>
__global__ void __launch_bounds__(kRowWarps * 32, VM >= 3 ? kRowMinBlocksVtx : kRowMinBlocks)
k_tc_rows(const unsigned long long* __restrict__ items, unsigned long long nitems, const TaskDev* __restrict__ tasks, const uint32_t* __restrict__ col,
          const uint32_t* __restrict__ rowptr, const uint32_t* __restrict__ bitmap,
          unsigned long long* __restrict__ task_counts, unsigned long long* __restrict__ tv,
          unsigned long long* __restrict__ next, unsigned long long* __restrict__ cyc) {
    extern __shared__ uint32_t smem[];
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    uint32_t* S = smem + wid * (kSetWords + scratch_words(VM));
    uint32_t* scratch = S + kSetWords;
    uint32_t* vpre = scratch + 160;                  // VTX only (see VCnt; per row when inset)
    uint32_t* vcnt = vpre + kPreWords;
    for (uint32_t k = lane; k < kSetWords; k += 32) S[k] = 0;   // invariant: all-zero between rows
    if (VM >= 3 && !kVtxInset)
        for (uint32_t k = lane; k < kVtxSlots / 2; k += 32) vcnt[k] = 0;   // invariant: zero between rows
    __syncwarp();
    // Warps claim kRowChunk items at a time from one counter, so the items in
    // flight stay a narrow window of the locality-ordered list (the A_jx blocks
    // they share stay in L2).
    // counting kernel: 32 items per claim, small rows batched (batch_rows); the
    // other rows, one at a time below
    constexpr bool kBat = VM == 0 && !TIMED && kBatchLa > 0;
    unsigned long long claim_end = 0, idx = 0, my_it = 0;
    uint32_t pend = 0;
    if (!kBat) idx = claim_items(next, nitems, lane, claim_end);
    uint32_t cur_t = 0;                              // task of the warp's running count
    unsigned long long acc_t = 0;
#ifdef PGABB_PROF
    unsigned long long prof[32];
    for (int c = 0; c < 32; ++c) prof[c] = 0;
    unsigned long long pt = clock64();
#endif
    for (;;) {
        unsigned long long it;
        if (kBat) {
            bool done = false;
            while (pend == 0) {
                unsigned long long b = 0;
                if (lane == 0) b = atomicAdd(next, 32ull);
                b = __shfl_sync(0xffffffffu, b, 0);
                if (b >= nitems) {
                    done = true;
                    break;
                }
                const bool valid = b + lane < nitems;
                my_it = valid ? __ldg(items + b + lane) : 0ull;
                pend = batch_rows(my_it, valid, tasks, col, rowptr, S, scratch, lane, cur_t, acc_t, task_counts);
                PROF_MARK(10);
            }
            if (done) break;
            const int sl = __ffs(pend) - 1;
            pend &= pend - 1;
            it = __shfl_sync(0xffffffffu, my_it, sl);
        } else {
            if (idx >= nitems) break;
            it = __ldg(items + idx);
            idx = idx + 1 < claim_end ? idx + 1 : claim_items(next, nitems, lane, claim_end);
        }
        const uint32_t t = (uint32_t)(it >> 48);
        const uint32_t chunk = (uint32_t)(it >> 32) & 0xffffu;
        const uint32_t u = (uint32_t)it;
        const long long c0 = TIMED ? clock64() : 0;
        // kernel roles (internal.h TaskDev, DESIGN R25): u is the item's row vertex,
        // A its held list, vcol its neighbours (chunk `chunk` of them), Bc/rp_jx the
        // neighbours' streamed lists, npos their suffix starts (MID, x == j)
        const TaskDev T = tasks[t];
        const uint32_t a0 = __ldg(rowptr + T.s_rp + u), a1 = __ldg(rowptr + T.s_rp + u + 1);
        uint32_t e0 = __ldg(rowptr + T.n_rp + u), e1 = __ldg(rowptr + T.n_rp + u + 1);
        e0 += chunk * kChunkNbrs;
        e1 = min(e1, e0 + kChunkNbrs);
        const uint32_t la = a1 - a0;
        const uint32_t* __restrict__ A = col + T.s_col + a0;
        const uint32_t* __restrict__ Bc = col + T.t_col;
        const uint32_t* __restrict__ vcol = col + T.n_col;
        const uint32_t* __restrict__ npos = T.n_pos != ~0ull ? col + T.n_pos : nullptr;
        const uint32_t* __restrict__ rp_jx = rowptr + T.t_rp;
        const int mode = (T.wx <= kWarpBitmapBits) ? 0 : (la <= kHashMaxList ? 1 : 2);
        const uint32_t hbits = max(5, 32 - __clz(2 * la - 1));   // smallest 2^hbits >= 2 la (>= 32)
        const uint32_t hmask = (1u << hbits) - 1;
        uint32_t acc = 0;
        // per-vertex roles (R24/R25): the row vertex is LOW (LOW task) or MID (MID
        // task), its neighbours the other one; VM 1 credits LOW only, VM >= 2 both
        const bool row_cr = VM >= 2 || (VM == 1 && T.dir == kDirLow);
        unsigned long long* tvj = (VM >= 2 || (VM == 1 && T.dir == kDirMid)) ? tv + T.c_nbr : nullptr;
        unsigned long long* tvx = VM > 0 ? tv + T.cx : nullptr;
        VCnt vc{vcnt, vpre, tvx, false};
        PROF_MARK(0);
        if (T.t_bm != ~0ull && 8 * la <= (T.bm_words > kDenseRowWideW ? kDenseRowMulWide : kDenseRowMul) * T.bm_words) {
            acc = probe_dense_row<VM>(vcol, e0, e1, A, la, bitmap + T.t_bm, T.bm_words, lane, tvj, tvx);
            PROF_MARK(1);
            PROF_CNT(16);
        } else if (kSmallHeld && la <= kLightLa) {
            // small held list (<= kLightLa ids, the MID rows of the low-degree part): no
            // set staging -- every lane holds S in registers and takes every 32nd
            // neighbour, scanning its (short) streamed list against S or binary-
            // searching S's ids in a longer one (the light kernel's per-thread loop)
            const uint32_t mine = lane < (int)la ? __ldg(A + lane) : 0xffffffffu;
            uint32_t a[kLightLa];
#pragma unroll
            for (int k = 0; k < (int)kLightLa; ++k) a[k] = __shfl_sync(0xffffffffu, mine, k);
#define SMALL(P, L)                                                                                          \
    light_lists<VM, P, L, 32>(col, rowptr, vcol, npos, T.t_rp, Bc, e0 + lane, e1, a, la, tvj, tvx)
            if (npos)
                acc = la <= 1 ? SMALL(true, 1) : la <= 2 ? SMALL(true, 2) : la <= 4 ? SMALL(true, 4)
                                                                             : SMALL(true, (int)kLightLa);
            else
                acc = la <= 1 ? SMALL(false, 1) : la <= 2 ? SMALL(false, 2) : la <= 4 ? SMALL(false, 4)
                                                                               : SMALL(false, (int)kLightLa);
#undef SMALL
            PROF_MARK(5);
        } else if (mode == 0) {
            for (uint32_t k = lane; k < la; k += 32) {
                const uint32_t w = __ldg(A + k);
                atomicOr(&S[w >> 5], 1u << (w & 31));
            }
            __syncwarp();
            const uint32_t Wx = (T.wx + 31) / 32, NGx = (Wx + kPreGroup - 1) / kPreGroup;
            if (VM >= 3 && kVtxInset) {   // counters in S's free tail: [Wx, +pre) then cnt
                vc.pre = S + Wx;
                vc.cnt = S + Wx + (NGx + 1) / 2;
            }
            if (VM >= 3 && la <= kVtxSlots && e1 - e0 < 65536u &&
                (!kVtxInset || Wx + (NGx + 1) / 2 + (la + 1) / 2 <= kSetWords)) {
                // prefix popcounts of S per group of kPreGroup words (u16): the rank of a
                // member w is pre[group] + the popcounts of the words before it in its group
                vc.on = true;
                const uint32_t W = Wx, NG = NGx;
                uint16_t* pre16 = reinterpret_cast<uint16_t*>(vc.pre);
                uint32_t run = 0;
                for (uint32_t b = 0; b < NG; b += 32) {
                    const uint32_t g = b + lane;
                    uint32_t c = 0;
                    if (g < NG)
                        for (uint32_t z = g * kPreGroup; z < min(W, (g + 1) * kPreGroup); ++z) c += __popc(S[z]);
                    uint32_t incl = c;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                        if (lane >= o) incl += y;
                    }
                    if (g < NG) pre16[g] = (uint16_t)(run + incl - c);
                    run += __shfl_sync(0xffffffffu, incl, 31);
                }
                __syncwarp();
            }
            PROF_MARK(2);
            PROF_CNT(17);
            if (T.t_bm != ~0ull) {
                const uint32_t* BM = bitmap + T.t_bm;
                const uint32_t W = T.bm_words;
                if (W <= 32) acc = IROW(0, 1, vcol, e0, e1, npos, rp_jx, Bc, BM, W, S, scratch, 0, 0, A, la, lane, tvj, vc PROF_PASS);
                else if (W <= 128) acc = IROW(0, 4, vcol, e0, e1, npos, rp_jx, Bc, BM, W, S, scratch, 0, 0, A, la, lane, tvj, vc PROF_PASS);
                else acc = IROW(0, 0, vcol, e0, e1, npos, rp_jx, Bc, BM, W, S, scratch, 0, 0, A, la, lane, tvj, vc PROF_PASS);
            } else {
                acc = IROW(0, 0, vcol, e0, e1, npos, rp_jx, Bc, nullptr, 0, S, scratch, 0, 0, A, la, lane, tvj, vc PROF_PASS);
            }
            __syncwarp();
            if (VM >= 3 && vc.on) {   // flush the row's w counters: one atomic per distinct w
                const uint16_t* c16 = reinterpret_cast<const uint16_t*>(vc.cnt);
                for (uint32_t k = lane; k < la; k += 32) {
                    const uint32_t c = c16[k];
                    if (c) atomicAdd(tvx + __ldg(A + k), (unsigned long long)c);
                }
                __syncwarp();
                for (uint32_t k = lane; k < (la + 1) / 2; k += 32) vc.cnt[k] = 0u;
                if (kVtxInset)   // the prefix words sit inside S, which is all-zero between rows
                    for (uint32_t k = lane; k < (NGx + 1) / 2; k += 32) vc.pre[k] = 0u;
            }
            for (uint32_t k = lane; k < la; k += 32) S[__ldg(A + k) >> 5] = 0u;
        } else if (mode == 1) {
            // (the per-vertex kernel with inset counters uses the set's free tail for
            // them instead of the filter)
            const bool filt = kHashFilter && hmask < kFilterSlots && !(VM >= 3 && kVtxInset);
            for (uint32_t k = lane; k < la; k += 32) {
                const uint32_t w = __ldg(A + k);
                uint32_t h = hash_slot(w, hbits);
                while (atomicCAS(&S[h], 0u, w + 1) != 0u) h = (h + 1) & hmask;
                if (filt) {
                    const uint32_t f = filter_bit(w);
                    atomicOr(&S[kFilterSlots + (f >> 5)], 1u << (f & 31));
                }
            }
            __syncwarp();
            if (VM >= 3) {   // one u16 counter per hash slot
                if (kVtxInset) {
                    vc.cnt = S + hmask + 1;
                    vc.on = e1 - e0 < 65536u && (hmask + 1) + (hmask + 1) / 2 <= kSetWords;
                } else {
                    vc.on = e1 - e0 < 65536u && hmask < kVtxSlots;
                }
            }
            PROF_MARK(2);
            PROF_CNT(18);
            if (filt)
                acc = IROW(3, 0, vcol, e0, e1, npos, rp_jx, Bc, nullptr, 0, S, scratch, hbits, hmask, A, la, lane, tvj, vc PROF_PASS);
            else
                acc = IROW(1, 0, vcol, e0, e1, npos, rp_jx, Bc, nullptr, 0, S, scratch, hbits, hmask, A, la, lane, tvj, vc PROF_PASS);
            if (filt) {
                __syncwarp();
                for (uint32_t k = lane; k < la; k += 32) S[kFilterSlots + (filter_bit(__ldg(A + k)) >> 5)] = 0u;
            }
            __syncwarp();
            if (VM >= 3 && vc.on) {
                const uint16_t* c16 = reinterpret_cast<const uint16_t*>(vc.cnt);
                for (uint32_t k = lane; k <= hmask; k += 32) {
                    const uint32_t c = c16[k];
                    if (c) atomicAdd(tvx + (S[k] - 1u), (unsigned long long)c);
                }
                __syncwarp();
                for (uint32_t k = lane; k < (hmask + 1) / 2; k += 32) vc.cnt[k] = 0u;
            }
            for (uint32_t k = lane; k <= hmask; k += 32) S[k] = 0u;
        } else {
            for (uint32_t e = e0; e < e1; ++e) {
                const uint32_t v = __ldg(vcol + e);
                const uint32_t b0 = npos ? __ldg(npos + e) + 1 : __ldg(rp_jx + v), b1 = __ldg(rp_jx + v + 1);
                if (b1 > b0) {
                    const uint32_t c = warp_intersect<(VM >= 3)>(A, la, Bc + b0, b1 - b0, lane, tvx);
                    if (VM >= 1 && tvj && c) atomicAdd(tvj + v, (unsigned long long)c);
                    acc += c;
                }
            }
            PROF_MARK(8);
            PROF_CNT(19);
        }
        __syncwarp();
        // a row's count is < 2^32 (<= |A_ix[u]| * |A_ij[u]|), so a 32-bit REDUX suffices
        const uint32_t sum = __reduce_add_sync(0xffffffffu, acc);
        // the warp keeps its count while consecutive items share a task (one atomic per
        // task change instead of one per row: the rows of a task all add to one counter)
        if (t != cur_t) {
            if (lane == 0 && acc_t) atomicAdd(&task_counts[cur_t], acc_t);
            cur_t = t;
            acc_t = 0;
        }
        acc_t += sum;
        if (VM >= 1 && row_cr && lane == 0 && sum) atomicAdd(tv + T.c_row + u, (unsigned long long)sum);
        if (TIMED && lane == 0) atomicAdd(&cyc[t], (unsigned long long)(clock64() - c0));
        PROF_MARK(7);
    }
    if (lane == 0 && acc_t) atomicAdd(&task_counts[cur_t], acc_t);
#ifdef PGABB_PROF
    if (lane == 0)
        for (int c = 0; c < 32; ++c)
            if (prof[c]) atomicAdd(&g_prof[c], prof[c]);
#endif
}

// ---------------------------------------------------------------------------
// k_tc_light: one THREAD per light row item (DESIGN R20) -- the low-degree rows
// that dominate sparse graphs (ER, road-like grids), where a warp per row would
// spend its time on latency with one or two list elements per lane.
//
//   A_ix[u] (<= kLightLa ids) is held in registers (unused slots = ~0u, never a
//   local id);
//   for each v in A_ij[u] (<= kLightLe):
//     dense A_jx:  one bit test of v's bitmap row per element of A_ix[u];
//     |A_jx[v]| <= kLightScan: every id of the list compared with all of A_ix[u];
//     longer:      binary search of each element of A_ix[u] in the list.
// Items are claimed in order by warps, kLightChunk x 32 at a time from one global
// counter (lane l takes items base + 32r + l: coalesced item loads), so the
// items in flight stay a narrow window of the locality-ordered list and the
// v-side block A_jx they probe stays in L2.  A thread keeps its count while
// consecutive items share a task and flushes it with one atomicAdd when the
// task changes.  Same exact |A_ix[u] ∩ A_jx[v]| sums as
// k_tc_rows (Listing 5).
// ---------------------------------------------------------------------------
// items: the whole rank's light items, or one wave's range of them (streaming: the
// task table and pools then point at the wave's arena).
// HELD: registers for the held ids -- kLightLa (light items), or kMedLa for the
// medium items (R29), a separate instantiation so that the light one keeps its
// occupancy.
#ifndef PGABB_MED_MINB
#define PGABB_MED_MINB 5
#endif
template <int VM, bool TIMED, int HELD>
__global__ void __launch_bounds__(kLightThreads, HELD > (int)kLightLa ? PGABB_MED_MINB : PGABB_LIGHT_MINB)
k_tc_light(const uint4* __restrict__ items, unsigned long long nitems,
           const TaskDev* __restrict__ tasks, const uint32_t* __restrict__ col,
           const uint32_t* __restrict__ rowptr, const uint32_t* __restrict__ bitmap,
           const uint32_t* __restrict__ ell,
           unsigned long long* __restrict__ task_counts, unsigned long long* __restrict__ tv,
           unsigned long long* __restrict__ next, unsigned long long* __restrict__ cyc) {
    const int lane = threadIdx.x & 31;
    uint32_t cur_t = 0xffffffffu;
    unsigned long long acc_t = 0, cyc_t = 0;
    for (;;) {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(next, (unsigned long long)(32 * kLightChunk));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base >= nitems) break;
    uint4 it_next = make_uint4(0, 0, 0, 0);   // PGABB_LIGHT_PREFETCH: the next item, loaded a step early
    if (kLightPrefetch && base + lane < nitems) it_next = ld_stream(items + base + lane);
    for (int r = 0; r < kLightChunk; ++r) {
        const unsigned long long idx = base + 32 * r + lane;
        if (idx >= nitems) break;
        uint4 it;
        if (kLightPrefetch) {
            it = it_next;
            if (r + 1 < kLightChunk && idx + 32 < nitems) it_next = ld_stream(items + idx + 32);
        } else {
            it = ld_stream(items + idx);
        }
        const uint32_t t = it.x & ((1u << kLightTaskBits) - 1);
        const uint32_t u = it.w;
        const uint32_t la = (it.x >> kLightTaskBits) & 15u;
        const uint32_t a0 = it.y;
        const uint32_t e0 = it.z;
        const uint32_t e1 = e0 + (it.x >> (kLightTaskBits + 4));
        if (t != cur_t) {
            if (acc_t) atomicAdd(&task_counts[cur_t], acc_t);
            if (TIMED && cyc_t) atomicAdd(&cyc[cur_t], cyc_t);
            cur_t = t;
            acc_t = 0;
            cyc_t = 0;
        }
        const long long c0 = TIMED ? clock64() : 0;
        // kernel roles (TaskDev, R25): u the row vertex, a[] its held list, the
        // neighbours' streamed lists from t_col (MID, x == j: after the row vertex)
        const TaskDev& T = tasks[t];
        const uint64_t col_ij = T.n_col, bm_jx = T.t_bm, npos = T.n_pos;
        const uint32_t* __restrict__ A = col + T.s_col + a0;
        uint32_t a[HELD];
        if (kLightAVec && HELD <= 8) {
            // the held ids from their aligned 16-byte chunks (<= 3 loads instead of one
            // per id), shifted into place by the list's offset within its first chunk
            constexpr int kCh = (HELD + 6) / 4;
            const uintptr_t pa = reinterpret_cast<uintptr_t>(A);
            const uint4* c4 = reinterpret_cast<const uint4*>(pa & ~(uintptr_t)15);
            const int off = (int)((pa >> 2) & 3);
            const int nch = (off + (int)la + 3) >> 2;
            uint32_t w[4 * kCh];
#pragma unroll
            for (int ch = 0; ch < kCh; ++ch) {
                uint4 w4 = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
                if (ch < nch) w4 = __ldg(c4 + ch);
                w[4 * ch] = w4.x;
                w[4 * ch + 1] = w4.y;
                w[4 * ch + 2] = w4.z;
                w[4 * ch + 3] = w4.w;
            }
#pragma unroll
            for (int k = 0; k < HELD; ++k) {
                const uint32_t x = off == 0 ? w[k] : off == 1 ? w[k + 1] : off == 2 ? w[k + 2] : w[k + 3];
                a[k] = (k < (int)la) ? x : 0xffffffffu;
            }
        } else {
#pragma unroll
            for (int k = 0; k < HELD; ++k) a[k] = (k < (int)la) ? ld_stream(A + k) : 0xffffffffu;
        }
        const bool row_cr = VM >= 2 || (VM == 1 && T.dir == kDirLow);
        unsigned long long* tvj = (VM >= 2 || (VM == 1 && T.dir == kDirMid)) ? tv + T.c_nbr : nullptr;
        unsigned long long* tvx = VM > 0 ? tv + T.cx : nullptr;
        uint32_t acc = 0;
        if (bm_jx != ~0ull) {
            const uint32_t W = T.bm_words;
            const uint32_t* __restrict__ BM = bitmap + bm_jx;
            for (uint32_t e = e0; e < e1; ++e) {
                const uint32_t v = __ldg(col + col_ij + e);
                const uint32_t* __restrict__ row = BM + (uint64_t)v * W;
                uint32_t c = 0;
#pragma unroll
                for (int k = 0; k < HELD; ++k)
                    if (k < (int)la) {
                        const uint32_t hit = (__ldg(row + (a[k] >> 5)) >> (a[k] & 31)) & 1u;
                        if (VM >= 3 && hit) atomicAdd(tvx + a[k], 1ull);
                        c += hit;
                    }
                acc += c;
                if (VM >= 1 && tvj && c) atomicAdd(tvj + v, (unsigned long long)c);
            }
        } else if (T.t_ell != ~0ull) {
            // R30 slots (LOW tasks only: no suffix starts); compare width as below
            const uint32_t lam = __reduce_max_sync(__activemask(), la);
            const uint32_t* __restrict__ E = ell + T.t_ell;
            const uint32_t* __restrict__ Bc = col + T.t_col;
            const uint32_t* __restrict__ vc_ = col + col_ij;
            constexpr int kLa8 = HELD > 8 ? 8 : HELD;
#define LELL(W, L) light_ell<VM, L, W>(rowptr, vc_, T.t_rp, Bc, E, e0, e1, a, la, tvj, tvx)
            if (T.ell_w == 8)
                acc = lam <= 2 ? LELL(8, 2) : lam <= 4 ? LELL(8, 4) : lam <= 8 ? LELL(8, kLa8) : LELL(8, HELD);
            else
                acc = lam <= 2 ? LELL(16, 2) : lam <= 4 ? LELL(16, 4) : lam <= 8 ? LELL(16, kLa8) : LELL(16, HELD);
#undef LELL
        } else {
            // the warp's largest held list picks the compare width (warp-uniform)
            const uint32_t lam = __reduce_max_sync(__activemask(), la);
#define LLISTS(P, L)                                                                                       \
    light_lists<VM, P, L>(col, rowptr, col + col_ij, P ? col + npos : nullptr, T.t_rp, col + T.t_col, e0, e1, a, \
                          la, tvj, tvx)
            constexpr int kLa8 = HELD > 8 ? 8 : HELD;   // the 8-wide step when HELD > 8
            if (npos != ~0ull)
                acc = lam <= 1 ? LLISTS(true, 1) : lam <= 2 ? LLISTS(true, 2) : lam <= 4 ? LLISTS(true, 4)
                    : lam <= 8 ? LLISTS(true, kLa8) : LLISTS(true, HELD);
            else
                acc = lam <= 1 ? LLISTS(false, 1) : lam <= 2 ? LLISTS(false, 2) : lam <= 4 ? LLISTS(false, 4)
                    : lam <= 8 ? LLISTS(false, kLa8) : LLISTS(false, HELD);
#undef LLISTS
        }
        acc_t += acc;
        if (VM >= 1 && row_cr && acc) atomicAdd(tv + T.c_row + u, (unsigned long long)acc);
        if (TIMED) cyc_t += (unsigned long long)(clock64() - c0);
    }
    }
    if (acc_t) atomicAdd(&task_counts[cur_t], acc_t);
    if (TIMED && cyc_t) atomicAdd(&cyc[cur_t], cyc_t);
}

// S11: T_rank = sum of the per-task counts (written after them, at [ntasks]).
__global__ void k_sum_tasks(unsigned long long* tc, int nt, unsigned long long* out_dev) {
    unsigned long long s = 0;
    for (int t = threadIdx.x; t < nt; t += blockDim.x) s += tc[t];
    s = warp_sum(s);
    __shared__ unsigned long long sh[32];
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        s = (threadIdx.x < (blockDim.x >> 5)) ? sh[threadIdx.x] : 0;
        s = warp_sum(s);
        if (threadIdx.x == 0) {
            tc[nt] = s;
            if (out_dev) *out_dev = s;
        }
    }
}

// Per-vertex counts back to original ids: tv[v] = tv_rank[rank[v]].
// accumulate: tv[v] += (PGABB_OUT_ACCUMULATE, the second pass of the two-pass route)
__global__ void k_gather_tv(const uint32_t* __restrict__ rank, const unsigned long long* __restrict__ tv_rank,
                            uint32_t n, unsigned long long* __restrict__ tv, int accumulate) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x)
        tv[v] = (accumulate ? tv[v] : 0ull) + tv_rank[rank[v]];
}

// Local clustering coefficient (NEXT-1): cc(v) = 2 t(v) / (deg(v) (deg(v) - 1)),
// 0 for deg(v) < 2.  Both operands are exact in fp64 (< 2^53), so the one IEEE
// division is correctly rounded and bit-identical to any other such evaluation.
__global__ void k_clustering(const uint32_t* __restrict__ deg, const unsigned long long* __restrict__ tv,
                             uint32_t n, double* __restrict__ cc) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t d = deg[v];
        cc[v] = d < 2 ? 0.0 : (2.0 * (double)tv[v]) / (double)(d * (d - 1));
    }
}

}  // namespace

int sm_count(int device) {
    static thread_local int dev = -1, sms = 0;
    if (dev != device) {
        PG_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        dev = device;
    }
    return sms;
}

void begin_call(pgabb_blocks_s* h, cudaStream_t st) {
    if (h->ev_last_recorded) PG_CK(cudaStreamWaitEvent(st, h->ev_last, 0));
}

void end_call(pgabb_blocks_s* h, cudaStream_t st) {
    PG_CK(cudaEventRecord(h->ev_last, st));
    h->ev_last_recorded = true;
}

// Before a call re-records ev0..ev3: a previous async call's timing is read if its
// events have completed, else dropped (never waited for -- a new call must not
// stall the host on the previous one).
void settle_timing(pgabb_blocks_s* h) {
    if (!h->timing_pending) return;
    const cudaError_t q = cudaEventQuery(h->ev3);
    if (q == cudaSuccess) {
        resolve_timing(h);
        return;
    }
    if (q != cudaErrorNotReady) PG_CK(q);
    h->timing_pending = false;
}

void resolve_timing(pgabb_blocks_s* h) {
    if (!h->timing_pending) return;
    PG_CK(cudaEventSynchronize(h->ev3));
    float ms = 0, ms_main = 0;
    PG_CK(cudaEventElapsedTime(&ms, h->ev0, h->ev3));
    PG_CK(cudaEventElapsedTime(&ms_main, h->ev1, h->ev2));
    float ms_light = 0;
    if (h->light_timed) PG_CK(cudaEventElapsedTime(&ms_light, h->ev_mid, h->ev2));
    h->ms_light_last = ms_light;
    h->ms_count_last = ms;
    h->ms_main_last = ms_main;
    h->timing_pending = false;
}

#ifdef PGABB_PROF
}  // namespace pgabb
extern "C" PGABB_API int pgabb_prof_read(unsigned long long* out, int reset) {
    if (cudaMemcpyFromSymbol(out, ::g_prof, sizeof(unsigned long long) * 32) != cudaSuccess) return 3;
    if (reset) {
        unsigned long long z[32] = {};
        if (cudaMemcpyToSymbol(::g_prof, z, sizeof(z)) != cudaSuccess) return 3;
    }
    return 0;
}
namespace pgabb {
#endif

// ---- NEXT-3 collaborative CPU + GPU: the host threads' share ------------------
// Same sums as the kernels (Listing 5), in the task's
// orientation (TaskDev roles, R25), read from the pinned host pools: per row r the
// held list S against every neighbour's streamed list, by a merge (or a binary
// search of the shorter list's ids in the longer one when their sizes are skewed).
static uint64_t host_intersect(const uint32_t* a, uint32_t la, const uint32_t* b, uint32_t lb) {
    if (la == 0 || lb == 0) return 0;
    if (la > lb) {
        std::swap(a, b);
        std::swap(la, lb);
    }
    uint64_t c = 0;
    if ((uint64_t)la * 16 < lb) {   // skewed: binary search, window shrinking
        const uint32_t* lo = b;
        const uint32_t* end = b + lb;
        for (uint32_t i = 0; i < la && lo < end; ++i) {
            lo = std::lower_bound(lo, end, a[i]);
            if (lo < end && *lo == a[i]) ++c;
        }
        return c;
    }
    uint32_t i = 0, j = 0;
    while (i < la && j < lb) {
        const uint32_t x = a[i], y = b[j];
        c += (x == y);
        i += (x <= y);
        j += (y <= x);
    }
    return c;
}

static void host_count_share(pgabb_blocks_s* h, unsigned long long* per_task) {
    const uint32_t* col = h->h_col.p;
    const uint32_t* rp = h->h_rowptr.p;
    struct Unit { uint32_t piece, r0, r1; };
    std::vector<Unit> units;
    for (uint32_t k = 0; k < h->host_work.size(); ++k) {
        const PieceDev& w = h->host_work[k];
        for (uint32_t r = w.r0; r < w.r1; r += 4096) units.push_back(Unit{k, r, std::min(w.r1, r + 4096)});
    }
    const size_t nt = h->tasks.size();
    unsigned nthr = h->host_threads ? h->host_threads : std::max(1u, std::thread::hardware_concurrency());
    nthr = (unsigned)std::min<size_t>(nthr, std::max<size_t>(units.size(), 1));
    std::atomic<size_t> next{0};
    std::vector<std::vector<unsigned long long>> part(nthr, std::vector<unsigned long long>(nt, 0));
    auto worker = [&](unsigned id) {
        std::vector<unsigned long long>& acc = part[id];
        for (size_t q; (q = next.fetch_add(1)) < units.size();) {
            const Unit& un = units[q];
            const PieceDev& w = h->host_work[un.piece];
            const TaskDev& T = h->host_tasks[w.task];
            uint64_t c = 0;
            for (uint32_t r = un.r0; r < un.r1; ++r) {
                const uint32_t a0 = rp[T.s_rp + r], la = rp[T.s_rp + r + 1] - a0;
                const uint32_t e0 = rp[T.n_rp + r], e1 = rp[T.n_rp + r + 1];
                if (la == 0) continue;
                const uint32_t* A = col + T.s_col + a0;
                for (uint32_t e = e0; e < e1; ++e) {
                    const uint32_t nb = col[T.n_col + e];
                    const uint32_t b1 = rp[T.t_rp + nb + 1];
                    const uint32_t b0 = T.n_pos != ~0ull ? col[T.n_pos + e] + 1 : rp[T.t_rp + nb];
                    if (b1 > b0) c += host_intersect(A, la, col + T.t_col + b0, b1 - b0);
                }
            }
            acc[w.task] += c;
        }
    };
    std::vector<std::thread> pool;
    for (unsigned t = 1; t < nthr; ++t) pool.emplace_back(worker, t);
    worker(0);
    for (std::thread& th : pool) th.join();
    for (size_t t = 0; t < nt; ++t) {
        unsigned long long s = 0;
        for (unsigned id = 0; id < nthr; ++id) s += part[id][t];
        per_task[t] = s;
    }
}

__global__ void k_add_counts(unsigned long long* tc, const unsigned long long* add, int nt) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x) tc[t] += add[t];
}

uint64_t count_triangles(pgabb_blocks_s* h, const pgabb_count_opts_t* opts, bool* wrote,
                         unsigned long long* d_tv_out, unsigned long long* d_cycles, int vm) {
    const bool timed = d_cycles != nullptr;   // pgabb_task_times: counting kernels with cycle accounting
    cudaStream_t st = (opts && opts->cuda_stream) ? (cudaStream_t)opts->cuda_stream : h->stream;
    const bool async = opts && (opts->flags & PGABB_COUNT_ASYNC);
    const int nt = (int)h->tasks.size();
    h->launches_last = 0;
    h->h2d_last = 0;
    h->d2d_last = 0;

    if (d_tv_out == nullptr) vm = 0;   // vm: per-vertex roles level (scratch_words)
    const bool vtx = vm > 0;
    h->light_timed = false;
    const size_t smem = kRowWarps * (kSetWords + scratch_words(vm)) * sizeof(uint32_t);
    static thread_local int cached_dev = -1, grids[4] = {0, 0, 0, 0};
    if (cached_dev != h->device) {
        int sms = 0, per_sm = 0;
        PG_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device));
        auto setup = [&](auto kfn, int level) {
            const size_t sm = kRowWarps * (kSetWords + scratch_words(level)) * sizeof(uint32_t);
            PG_CK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            PG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, kRowWarps * 32, sm));
            return sms * std::max(per_sm, 1);
        };
        grids[0] = setup(k_tc_rows<0, false>, 0);
        setup(k_tc_rows<0, true>, 0);
        grids[1] = setup(k_tc_rows<1, false>, 1);
        grids[2] = setup(k_tc_rows<2, false>, 2);
        grids[3] = setup(k_tc_rows<3, false>, 3);
        cached_dev = h->device;
    }
    const int grid = grids[vm];
    auto grid_for_items = [&](unsigned long long n) {
        return (unsigned)std::max(1ull, std::min<unsigned long long>((unsigned long long)grid,
                                                                     (n + kRowWarps - 1) / kRowWarps));
    };
    unsigned long long* tv = nullptr;
    if (vtx) {
        if (h->d_tv_rank.n < std::max<uint32_t>(h->n, 1)) h->d_tv_rank.alloc(std::max<uint32_t>(h->n, 1));
        tv = h->d_tv_rank.p;
    }
    auto rows_kernel = [&]() {
        if (timed) return k_tc_rows<0, true>;
        switch (vm) {
            case 1: return k_tc_rows<1, false>;
            case 2: return k_tc_rows<2, false>;
            case 3: return k_tc_rows<3, false>;
            default: return k_tc_rows<0, false>;
        }
    };
    auto light_kernel = [&]() {
        if (timed) return k_tc_light<0, true, kLightLa>;
        switch (vm) {
            case 1: return k_tc_light<1, false, kLightLa>;
            case 2: return k_tc_light<2, false, kLightLa>;
            case 3: return k_tc_light<3, false, kLightLa>;
            default: return k_tc_light<0, false, kLightLa>;
        }
    };
    auto med_kernel = [&]() {
        if (timed) return k_tc_light<0, true, kMedLa>;
        switch (vm) {
            case 1: return k_tc_light<1, false, kMedLa>;
            case 2: return k_tc_light<2, false, kMedLa>;
            case 3: return k_tc_light<3, false, kMedLa>;
            default: return k_tc_light<0, false, kMedLa>;
        }
    };
    static thread_local int light_dev = -1, light_grid = 0, med_grid = 0;
    if (light_dev != h->device) {
        int per_sm = 0;
        PG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tc_light<0, false, kLightLa>, kLightThreads, 0));
        light_grid = sm_count(h->device) * std::max(per_sm, 1);
        PG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tc_light<0, false, kMedLa>, kLightThreads, 0));
        med_grid = sm_count(h->device) * std::max(per_sm, 1);
        light_dev = h->device;
    }
    auto grid_for_light = [&](unsigned long long n, int g) {
        return (unsigned)std::max<unsigned long long>(
            1ull, std::min<unsigned long long>(g, (n + kLightThreads - 1) / kLightThreads));
    };

    PG_NVTX(vtx ? "pgabb_vertex_triangles" : "pgabb_triangle_count");
    settle_timing(h);
    begin_call(h, st);
    PG_CK(cudaEventRecord(h->ev0, st));
    if (!h->streaming) {
        // S9: host-resident blocks are copied in for this call.
        // Only the blocks this rank's pieces read (h->host_copies, merged ranges).
        if (h->residency == PGABB_RESIDENT_HOST && h->d_col.n) {
            uint32_t* dpool[3] = {h->d_col.p, h->d_rowptr.p, h->d_bitmap.p};
            const uint32_t* hpool[3] = {h->h_col.p, h->h_rowptr.p, h->h_bitmap.p};
            for (const StagedBlock& c : h->host_copies) {
                PG_CK(cudaMemcpyAsync(dpool[c.pool] + c.dst_word, hpool[c.pool] + c.src_word, c.words * 4,
                                      cudaMemcpyHostToDevice, st));
                h->h2d_last += c.words * 4;
            }
        }
        PG_CK(cudaMemsetAsync(h->d_task_counts.p, 0, (nt + 1) * sizeof(unsigned long long), st));
        if (vtx) PG_CK(cudaMemsetAsync(tv, 0, (size_t)h->n * sizeof(unsigned long long), st));
        PG_CK(cudaMemsetAsync(h->d_next.p, 0, 6 * sizeof(unsigned long long), st));
        PG_CK(cudaEventRecord(h->ev1, st));
        if (h->n_items) {
            rows_kernel()<<<grid_for_items(h->n_items), kRowWarps * 32, smem, st>>>(
                h->d_items.p, h->n_items, h->d_tasks.p, h->d_col.p, h->d_rowptr.p, h->d_bitmap.p,
                h->d_task_counts.p, tv, h->d_next.p + 1, d_cycles);
            PG_LAUNCH_CHECK();
            h->launches_last++;
        }
        PG_CK(cudaEventRecord(h->ev_mid, st));
        h->light_timed = true;
        if (h->n_light0) {
            light_kernel()<<<grid_for_light(h->n_light0, light_grid), kLightThreads, 0, st>>>(
                h->d_light.p, h->n_light0, h->d_tasks.p, h->d_col.p, h->d_rowptr.p, h->d_bitmap.p, h->d_ell.p,
                h->d_task_counts.p, tv, h->d_next.p, timed ? d_cycles + nt : nullptr);
            PG_LAUNCH_CHECK();
            h->launches_last++;
        }
        if (h->n_light > h->n_light0) {
            const unsigned long long nm = h->n_light - h->n_light0;
            med_kernel()<<<grid_for_light(nm, med_grid), kLightThreads, 0, st>>>(
                h->d_light.p + h->n_light0, nm, h->d_tasks.p, h->d_col.p, h->d_rowptr.p, h->d_bitmap.p,
                h->d_ell.p, h->d_task_counts.p, tv, h->d_next.p + 5, timed ? d_cycles + nt : nullptr);
            PG_LAUNCH_CHECK();
            h->launches_last++;
        }
    } else {
        // S9 streaming: wave k's blocks are copied into
        // arena k%2 on the copy stream while wave k-1 computes; a copy into an arena
        // first waits for the wave that last used it.
        PG_CK(cudaMemsetAsync(h->d_task_counts.p, 0, (nt + 1) * sizeof(unsigned long long), st));
        if (vtx) PG_CK(cudaMemsetAsync(tv, 0, (size_t)h->n * sizeof(unsigned long long), st));
        PG_CK(cudaEventRecord(h->ev1, st));
        PG_CK(cudaStreamWaitEvent(h->copy_stream, h->ev1, 0));
        const uint32_t* pools[3] = {h->h_col.p, h->h_rowptr.p, h->h_bitmap.p};
        const bool trace = opts && (opts->flags & PGABB_COUNT_TRACE);
        if (trace) {
            while (h->trace_ev.size() < 4 * h->waves.size()) {
                cudaEvent_t e;
                PG_CK(cudaEventCreate(&e));
                h->trace_ev.push_back(e);
            }
        }
        h->trace_valid = trace;
        for (size_t k = 0; k < h->waves.size(); ++k) {
            const Wave& wv = h->waves[k];
            if (wv.wait_wave >= 0) PG_CK(cudaStreamWaitEvent(h->copy_stream, h->ev_done[wv.wait_wave], 0));
            if (trace) PG_CK(cudaEventRecord(h->trace_ev[4 * k], h->copy_stream));
            for (const StagedBlock& c : wv.copies) {
                if (c.pool == 3) {   // staged by the wave k-K+1: device-to-device within the arena
                    PG_CK(cudaMemcpyAsync(h->d_arena.p + c.dst_word, h->d_arena.p + c.src_word,
                                          c.words * 4, cudaMemcpyDeviceToDevice, h->copy_stream));
                    h->d2d_last += c.words * 4;
                    continue;
                }
                PG_CK(cudaMemcpyAsync(h->d_arena.p + c.dst_word, pools[c.pool] + c.src_word, c.words * 4,
                                      cudaMemcpyHostToDevice, h->copy_stream));
                h->h2d_last += c.words * 4;
            }
            PG_CK(cudaEventRecord(h->ev_copied[k], h->copy_stream));
            if (trace) PG_CK(cudaEventRecord(h->trace_ev[4 * k + 1], h->copy_stream));
            PG_CK(cudaStreamWaitEvent(st, h->ev_copied[k], 0));
            if (trace) PG_CK(cudaEventRecord(h->trace_ev[4 * k + 2], st));
            // the wave's ranges of the row items; its task table and all three pool
            // pointers address the arena
            const uint32_t* base = h->d_arena.p;
            const TaskDev* wt = h->d_wave_tasks.p + wv.task_table * nt;
            PG_CK(cudaMemsetAsync(h->d_next.p + 2, 0, 3 * sizeof(unsigned long long), st));
            if (wv.item_end > wv.item_begin) {
                const unsigned long long ni = wv.item_end - wv.item_begin;
                rows_kernel()<<<grid_for_items(ni), kRowWarps * 32, smem, st>>>(
                    h->d_items.p + wv.item_begin, ni, wt, base, base, base, h->d_task_counts.p, tv, h->d_next.p + 2,
                    nullptr);
                PG_LAUNCH_CHECK();
                h->launches_last++;
            }
            if (wv.light_end > wv.light_begin) {
                const unsigned long long nl = wv.light_end - wv.light_begin;
                light_kernel()<<<grid_for_light(nl, light_grid), kLightThreads, 0, st>>>(
                    h->d_light.p + wv.light_begin, nl, wt, base, base, base, nullptr, h->d_task_counts.p, tv, h->d_next.p + 3,
                    nullptr);
                PG_LAUNCH_CHECK();
                h->launches_last++;
            }
            if (wv.med_end > wv.med_begin) {
                const unsigned long long nm = wv.med_end - wv.med_begin;
                med_kernel()<<<grid_for_light(nm, med_grid), kLightThreads, 0, st>>>(
                    h->d_light.p + wv.med_begin, nm, wt, base, base, base, nullptr, h->d_task_counts.p, tv, h->d_next.p + 4,
                    nullptr);
                PG_LAUNCH_CHECK();
                h->launches_last++;
            }
            PG_CK(cudaEventRecord(h->ev_done[k], st));
            if (trace) PG_CK(cudaEventRecord(h->trace_ev[4 * k + 3], st));
        }
    }
    PG_CK(cudaEventRecord(h->ev2, st));
    h->ms_host_last = 0;
    if (!h->host_work.empty()) {
        // NEXT-3: the host share runs now, while the GPU works through the copies and
        // kernels enqueued above; its per-task counts join the device's before the sum
        const auto t0 = std::chrono::steady_clock::now();
        host_count_share(h, h->h_host_counts.p);
        h->ms_host_last = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        PG_CK(cudaMemcpyAsync(h->d_host_counts.p, h->h_host_counts.p, nt * sizeof(unsigned long long),
                              cudaMemcpyHostToDevice, st));
        k_add_counts<<<(nt + 255) / 256, 256, 0, st>>>(h->d_task_counts.p, h->d_host_counts.p, nt);
        PG_LAUNCH_CHECK();
        h->launches_last++;
    }
    k_sum_tasks<<<1, 1024, 0, st>>>(h->d_task_counts.p, nt, (unsigned long long*)(opts ? opts->d_count : nullptr));
    PG_LAUNCH_CHECK();
    h->launches_last++;
    if (vtx && h->n) {
        k_gather_tv<<<(unsigned)std::min<uint64_t>((h->n + 255) / 256, (uint64_t)sm_count(h->device) * 16), 256, 0, st>>>(
            h->d_rank.p, tv, h->n, d_tv_out, (opts && (opts->flags & PGABB_OUT_ACCUMULATE)) ? 1 : 0);
        PG_LAUNCH_CHECK();
        h->launches_last++;
    }
    PG_CK(cudaMemcpyAsync(h->h_result.p, h->d_task_counts.p + nt, 8, cudaMemcpyDeviceToHost, st));
    PG_CK(cudaEventRecord(h->ev3, st));
    end_call(h, st);
    h->timing_pending = true;
    if (async) {
        *wrote = false;
        return 0;
    }
    resolve_timing(h);
    if (opts && opts->task_counts && nt) {
        std::vector<unsigned long long> tc(nt);
        PG_COPY_SYNC(tc.data(), h->d_task_counts.p, nt * 8, st);
        for (int t = 0; t < nt; ++t) opts->task_counts[t] = tc[t];
    }
    *wrote = true;
    return h->h_result.p[0];
}

void wave_trace(pgabb_blocks_s* h, double* out, uint64_t* nwaves) {
    if (!h->trace_valid) fail(PGABB_EINVAL, "no traced streaming count (PGABB_COUNT_TRACE) on this handle");
    *nwaves = h->waves.size();
    if (!out) return;
    PG_CK(cudaEventSynchronize(h->ev3));
    for (size_t k = 0; k < 4 * h->waves.size(); ++k) {
        float ms = 0;
        PG_CK(cudaEventElapsedTime(&ms, h->ev0, h->trace_ev[k]));
        out[k] = ms;
    }
}

void task_times(pgabb_blocks_s* h, uint64_t* ns) {
    const size_t nt = h->tasks.size();
    if (nt == 0) return;
    DBuf<unsigned long long> cyc;
    cyc.alloc(2 * nt);
    PG_CK(cudaMemsetAsync(cyc.p, 0, 2 * nt * 8, h->stream));
    bool wrote = false;
    count_triangles(h, nullptr, &wrote, nullptr, cyc.p);
    std::vector<unsigned long long> c(2 * nt);
    PG_COPY_SYNC(c.data(), cyc.p, 2 * nt * 8, h->stream);
    long double sh = 0, sl = 0;
    for (size_t t = 0; t < nt; ++t) {
        sh += c[t];
        sl += c[nt + t];
    }
    const long double ns_h = 1e6L * std::max(0.0, h->ms_main_last - h->ms_light_last);
    const long double ns_l = 1e6L * h->ms_light_last;
    for (size_t t = 0; t < nt; ++t) {
        long double v = 0;
        if (sh > 0) v += ns_h * c[t] / sh;
        if (sl > 0) v += ns_l * c[nt + t] / sl;
        ns[t] = (uint64_t)(v + 0.5L);
    }
}

void local_clustering(pgabb_blocks_s* h, const pgabb_count_opts_t* opts, const uint64_t* tv, double* cc) {
    cudaStream_t st = (opts && opts->cuda_stream) ? (cudaStream_t)opts->cuda_stream : h->stream;
    const bool on_dev = opts && (opts->flags & PGABB_OUT_DEVICE);
    if (h->n == 0) return;
    DBuf<unsigned long long> d_tv;
    DBuf<double> d_cc;
    const unsigned long long* tvp = (const unsigned long long*)tv;
    double* ccp = cc;
    if (!on_dev) {
        d_tv.alloc(h->n);
        d_cc.alloc(h->n);
        PG_CK(cudaMemcpyAsync(d_tv.p, tv, (size_t)h->n * 8, cudaMemcpyHostToDevice, st));
        tvp = d_tv.p;
        ccp = d_cc.p;
    }
    begin_call(h, st);
    k_clustering<<<(unsigned)std::min<uint64_t>((h->n + 255) / 256, (uint64_t)sm_count(h->device) * 16), 256, 0, st>>>(
        h->d_deg.p, tvp, h->n, ccp);
    PG_LAUNCH_CHECK();
    end_call(h, st);
    if (!on_dev) PG_CK(cudaMemcpyAsync(cc, d_cc.p, (size_t)h->n * 8, cudaMemcpyDeviceToHost, st));
    PG_CK(cudaStreamSynchronize(st));
}

}  // namespace pgabb
