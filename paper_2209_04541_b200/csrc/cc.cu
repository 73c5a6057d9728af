// cc.cu -- SURVEY §8(f) NEXT-4: Shiloach-Vishkin connected components on the same
// 2D blocks (§3.5 / Listing 2, "Shiloach-Vishkin device kernel").
//
// The paper's iteration: even iterations HOOK -- for every edge (u,v), r1 =
// max(C(u), C(v)), r2 = min(C(u), C(v)); if r1 != r2 and r1 is a root (C(r1) ==
// r1) then C(r1) = r2 and a hook is counted -- odd iterations LINK -- every vertex
// jumps to its root (while C(x) != C(C(x)): C(x) = C(C(x))) -- until an iteration
// hooks nothing.  Block-lists hold one block each: the hook
// pass runs over every edge of every non-empty block A_ij; each undirected edge
// is stored once (the DAG orientation, DESIGN R4), which suffices because a hook
// looks at both endpoints.
//
// B200 mapping: C lives in rank space (the blocks' vertex ids); the hook pass is
// one launch over all rows of all blocks, 32 rows per warp with their edges
// flattened over the lanes (hub rows do not serialise a thread); the hook write
// is an atomicMin (the paper's plain store races benignly; atomicMin keeps the
// smallest proposal).  Labels only decrease and stay inside their component, so
// at convergence every component's root is its smallest rank (DESIGN R23); the
// reported label is then the component's smallest ORIGINAL id, via one atomicMin
// pass through the S2 rank array.
#include <algorithm>

#include "internal.h"

namespace pgabb {

namespace {

struct CcBlock {               // one non-empty block of the grid
    uint64_t col_off, rp_off;  // pool offsets
    uint64_t row_start;        // first global row index of this block (prefix over blocks)
    uint32_t nrows, ri, rj;    // rows; rank offsets of parts i and j (cut_i, cut_j)
    uint32_t pad;
};

__global__ void k_cc_init(uint32_t* C, uint32_t n) {
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < n; x += (uint64_t)gridDim.x * blockDim.x) C[x] = x;
}

// HOOK over every edge of every block: a warp claims 32 consecutive global rows,
// flattens their edges over its lanes and hooks; hooks are counted into *H.
__global__ void __launch_bounds__(256) k_cc_hook(const CcBlock* __restrict__ blk, int nblk, uint64_t nrows_all,
                                                const uint32_t* __restrict__ col,
                                                const uint32_t* __restrict__ rowptr, uint32_t* C,
                                                unsigned long long* H) {
    __shared__ uint32_t sseg[8][32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint32_t le_mask = 0xffffffffu >> (31 - lane);
    const uint32_t lt_mask = (1u << lane) - 1u;
    const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    uint32_t hooks = 0;
    for (uint64_t base = wid * 32; base < nrows_all; base += nw * 32) {
        const uint64_t g = base + lane;
        uint32_t e0 = 0, ne = 0, u = 0;
        uint64_t coff = 0;
        uint32_t rj = 0;
        if (g < nrows_all) {
            int lo = 0, hi = nblk;   // last block with row_start <= g
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (blk[mid].row_start <= g) lo = mid; else hi = mid;
            }
            const CcBlock& B = blk[lo];
            const uint32_t r = (uint32_t)(g - B.row_start);
            e0 = __ldg(rowptr + B.rp_off + r);
            ne = __ldg(rowptr + B.rp_off + r + 1) - e0;
            u = B.ri + r;
            coff = B.col_off;
            rj = B.rj;
        }
        // flatten the 32 rows' edges over the lanes
        uint32_t incl = ne;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        const uint32_t excl = incl - ne;
        const uint32_t nonempty = __ballot_sync(0xffffffffu, ne > 0);
        if (ne > 0) sseg[wib][__popc(nonempty & lt_mask)] = lane;   // compacted row index -> lane
        __syncwarp();
        for (uint32_t rb = 0; rb < total; rb += 32) {
            const uint32_t pos = rb + lane;
            const uint32_t in = excl - rb;
            const uint32_t bit = (ne > 0 && excl > rb && in < 32u) ? (1u << in) : 0u;
            const uint32_t starts = __reduce_or_sync(0xffffffffu, bit);
            const int cur = __popc(__ballot_sync(0xffffffffu, ne > 0 && excl <= rb)) - 1;
            const int q = pos < total ? (int)sseg[wib][cur + __popc(starts & le_mask)] : 0;
            const uint32_t uq = __shfl_sync(0xffffffffu, u, q);
            const uint32_t e0q = __shfl_sync(0xffffffffu, e0, q);
            const uint32_t exq = __shfl_sync(0xffffffffu, excl, q);
            const uint64_t coq = __shfl_sync(0xffffffffu, coff, q);
            const uint32_t rjq = __shfl_sync(0xffffffffu, rj, q);
            if (pos < total) {
                const uint32_t v = rjq + __ldg(col + coq + e0q + (pos - exq));
                const uint32_t cu = C[uq], cv = C[v];
                const uint32_t r1 = max(cu, cv), r2 = min(cu, cv);
                if (r1 != r2 && C[r1] == r1) {   // hook the greater root under the smaller
                    atomicMin(&C[r1], r2);
                    ++hooks;
                }
            }
        }
        __syncwarp();
    }
    const uint32_t h = __reduce_add_sync(0xffffffffu, hooks);
    if (lane == 0 && h) atomicAdd(H, (unsigned long long)h);
}

// LINK: every vertex jumps to its root by pointer jumping, as Listing 2 writes it
// (while C(x) != C(C(x)): C(x) = C(C(x))) -- each write halves x's remaining path
// and is seen by the other threads walking through x, so deep hook trees (grids,
// chains) collapse in O(log depth) steps instead of one step per level.
__global__ void k_cc_link(uint32_t* C, uint32_t n) {
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < n; x += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t c = C[x], cc;
        while (c != (cc = C[c])) {
            c = cc;
            C[x] = c;
        }
    }
}

// Canonical labels: M[root] = smallest original id of the component.
__global__ void k_cc_minorig(const uint32_t* __restrict__ rank, const uint32_t* __restrict__ C, uint32_t n,
                             uint32_t* M) {
    // a giant component sends every v to one address: lanes with the same root
    // reduce first, and a proposal that cannot lower the current minimum is dropped
    const uint64_t n32 = ((uint64_t)n + 31) & ~31ull;   // whole warps take part in the warp reductions
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n32; v += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t root = v < n ? C[rank[v]] : 0xffffffffu;
        const uint32_t same = __match_any_sync(0xffffffffu, root);
        const uint32_t m = __reduce_min_sync(same, (uint32_t)v);
        if (v < n && v == m && m < *(volatile uint32_t*)&M[root]) atomicMin(&M[root], m);
    }
}

__global__ void k_cc_labels(const uint32_t* __restrict__ rank, const uint32_t* __restrict__ C,
                            const uint32_t* __restrict__ M, uint32_t n, uint32_t* labels,
                            unsigned long long* ncomp) {
    uint32_t roots = 0;
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t l = M[C[rank[v]]];
        labels[v] = l;
        roots += (l == v);
    }
    roots = __reduce_add_sync(0xffffffffu, roots);
    if ((threadIdx.x & 31) == 0 && roots) atomicAdd(ncomp, (unsigned long long)roots);
}

unsigned grid1(uint64_t n, int dev) {
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, (uint64_t)sm_count(dev) * 16));
}

}  // namespace

void connected_components(pgabb_blocks_s* h, const pgabb_count_opts_t* opts, uint32_t* labels, uint64_t* ncomp,
                          uint32_t* iters) {
    if (h->streaming) fail(PGABB_EINVAL, "connected components need the blocks resident (no device budget)");
    if (h->world_size > 1) fail(PGABB_EINVAL, "connected components run on one GPU (world_size 1)");
    cudaStream_t st = (opts && opts->cuda_stream) ? (cudaStream_t)opts->cuda_stream : h->stream;
    const bool on_dev = opts && (opts->flags & PGABB_OUT_DEVICE);
    const uint32_t n = h->n, p = h->p;
    settle_timing(h);   // ev0/ev3 are re-recorded below
    begin_call(h, st);
    if (h->residency == PGABB_RESIDENT_HOST && h->d_col.n) {   // S9: blocks in for this call
        PG_CK(cudaMemcpyAsync(h->d_col.p, h->h_col.p, h->d_col.bytes(), cudaMemcpyHostToDevice, st));
        PG_CK(cudaMemcpyAsync(h->d_rowptr.p, h->h_rowptr.p, h->d_rowptr.bytes(), cudaMemcpyHostToDevice, st));
    }
    std::vector<CcBlock> bl;
    uint64_t rows = 0;
    for (uint32_t i = 0; i < p; ++i)
        for (uint32_t j = i; j < p; ++j) {
            const BlockInfo& B = h->blocks[i * p + j];
            if (!B.present || B.nnz == 0) continue;
            CcBlock c{};
            c.col_off = B.col_off;
            c.rp_off = B.rp_off;
            c.row_start = rows;
            c.nrows = B.nrows;
            c.ri = h->cuts[i];
            c.rj = h->cuts[j];
            bl.push_back(c);
            rows += B.nrows;
        }
    DBuf<CcBlock> d_bl;
    DBuf<uint32_t> C, M, d_lab;
    DBuf<unsigned long long> cnt;
    d_bl.alloc(std::max<size_t>(bl.size(), 1));
    C.alloc(std::max<uint32_t>(n, 1));
    M.alloc(std::max<uint32_t>(n, 1));
    cnt.alloc(2);
    if (!bl.empty())
        PG_CK(cudaMemcpyAsync(d_bl.p, bl.data(), bl.size() * sizeof(CcBlock), cudaMemcpyHostToDevice, st));
    uint32_t* out = labels;
    if (!on_dev) {
        d_lab.alloc(std::max<uint32_t>(n, 1));
        out = d_lab.p;
    }
    PG_CK(cudaEventRecord(h->ev0, st));
    uint32_t it = 0;
    if (n) {
        k_cc_init<<<grid1(n, h->device), 256, 0, st>>>(C.p, n);
        PG_LAUNCH_CHECK();
        for (;;) {   // HOOK -> LINK -> ... until a HOOK pass hooks nothing
            PG_CK(cudaMemsetAsync(cnt.p, 0, 8, st));
            if (rows) {
                int sms = 0;
                PG_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device));
                const uint64_t warps = (rows + 31) / 32;
                const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((warps + 7) / 8, (uint64_t)sms * 8));
                k_cc_hook<<<g, 256, 0, st>>>(d_bl.p, (int)bl.size(), rows, h->d_col.p, h->d_rowptr.p, C.p, cnt.p);
                PG_LAUNCH_CHECK();
            }
            k_cc_link<<<grid1(n, h->device), 256, 0, st>>>(C.p, n);
            PG_LAUNCH_CHECK();
            unsigned long long hooks = 0;
            PG_CK(cudaMemcpyAsync(&hooks, cnt.p, 8, cudaMemcpyDeviceToHost, st));
            PG_CK(cudaStreamSynchronize(st));
            ++it;
            if (hooks == 0) break;
        }
        PG_CK(cudaMemsetAsync(M.p, 0xff, (size_t)n * 4, st));
        PG_CK(cudaMemsetAsync(cnt.p + 1, 0, 8, st));
        k_cc_minorig<<<grid1(n, h->device), 256, 0, st>>>(h->d_rank.p, C.p, n, M.p);
        PG_LAUNCH_CHECK();
        k_cc_labels<<<grid1(n, h->device), 256, 0, st>>>(h->d_rank.p, C.p, M.p, n, out, cnt.p + 1);
        PG_LAUNCH_CHECK();
    }
    PG_CK(cudaEventRecord(h->ev3, st));
    end_call(h, st);
    unsigned long long nc = 0;
    if (n) PG_CK(cudaMemcpyAsync(&nc, cnt.p + 1, 8, cudaMemcpyDeviceToHost, st));
    if (!on_dev && n) PG_CK(cudaMemcpyAsync(labels, out, (size_t)n * 4, cudaMemcpyDeviceToHost, st));
    PG_CK(cudaStreamSynchronize(st));
    float ms = 0;
    PG_CK(cudaEventElapsedTime(&ms, h->ev0, h->ev3));
    h->ms_cc_last = ms;
    h->cc_iters_last = it;
    if (ncomp) *ncomp = nc;
    if (iters) *iters = it;
}

}  // namespace pgabb
