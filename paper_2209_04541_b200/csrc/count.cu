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

#include "internal.h"

namespace pgabb {

namespace {

constexpr int kWarpsPerCta = 8;
constexpr int kChunk = 32;   // edges a warp claims per atomic grab

__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}

// Lane-parallel binary search of the shorter list's elements in the longer one.
// Returns this lane's share of |A ∩ B|.
__device__ __forceinline__ uint32_t warp_intersect(const uint32_t* __restrict__ A, uint32_t la,
                                                   const uint32_t* __restrict__ B, uint32_t lb, int lane) {
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
        c += (lo < ll && __ldg(L + lo) == x);
    }
    return c;
}

// One warp per edge (u,v) of A_ij; warps claim chunks of kChunk consecutive
// edges of the rank's flattened edge space dynamically.  Per-task partial counts
// are flushed with one atomicAdd per (chunk, task) run.
__global__ void __launch_bounds__(kWarpsPerCta * 32)
k_tc_warp(const PieceDev* __restrict__ work, int nwork, unsigned long long total_edges,
          const uint32_t* __restrict__ col, const uint32_t* __restrict__ rowptr,
          unsigned long long* __restrict__ task_counts, unsigned long long* __restrict__ next) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(next, (unsigned long long)kChunk);
        base = __shfl_sync(0xffffffffu, base, 0);
        if (base >= total_edges) break;
        const unsigned long long end = min(base + kChunk, total_edges);
        // piece containing `base`: last piece with gstart <= base
        int lo = 0, hi = nwork;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (work[mid].gstart <= base) lo = mid; else hi = mid;
        }
        int pc = lo;
        PieceDev w = work[pc];
        uint32_t e = w.e0 + (uint32_t)(base - w.gstart);   // block-local edge index
        // row containing edge e: last u in [r0, r1) with rowptr[u] <= e
        uint32_t a = w.r0, z = w.r1;
        while (z - a > 1) {
            const uint32_t mid = (a + z) >> 1;
            if (__ldg(rowptr + w.rp_ij + mid) <= e) a = mid; else z = mid;
        }
        uint32_t u = a;
        uint32_t acc = 0;
        for (unsigned long long g = base; g < end; ++g, ++e) {
            if (e >= w.e1) {   // next piece
                const unsigned long long s = warp_sum(acc);
                if (lane == 0 && s) atomicAdd(&task_counts[w.task], s);
                acc = 0;
                w = work[++pc];
                e = w.e0;
                u = w.r0;
            }
            while (__ldg(rowptr + w.rp_ij + u + 1) <= e) ++u;
            const uint32_t v = __ldg(col + w.col_ij + e);
            const uint32_t a0 = __ldg(rowptr + w.rp_ix + u), a1 = __ldg(rowptr + w.rp_ix + u + 1);
            const uint32_t b0 = __ldg(rowptr + w.rp_jx + v), b1 = __ldg(rowptr + w.rp_jx + v + 1);
            if (a1 > a0 && b1 > b0)
                acc += warp_intersect(col + w.col_ix + a0, a1 - a0, col + w.col_jx + b0, b1 - b0, lane);
        }
        const unsigned long long s = warp_sum(acc);
        if (lane == 0 && s) atomicAdd(&task_counts[w.task], s);
    }
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

}  // namespace

void resolve_timing(pgabb_blocks_s* h) {
    if (!h->timing_pending) return;
    PG_CK(cudaEventSynchronize(h->ev3));
    float ms = 0, ms_main = 0;
    PG_CK(cudaEventElapsedTime(&ms, h->ev0, h->ev3));
    PG_CK(cudaEventElapsedTime(&ms_main, h->ev1, h->ev2));
    h->ms_count_last = ms;
    h->ms_main_last = ms_main;
    h->timing_pending = false;
}

uint64_t count_triangles(pgabb_blocks_s* h, const pgabb_count_opts_t* opts, bool* wrote) {
    cudaStream_t st = (opts && opts->cuda_stream) ? (cudaStream_t)opts->cuda_stream : h->stream;
    const bool async = opts && (opts->flags & PGABB_COUNT_ASYNC);
    const int nt = (int)h->tasks.size();
    h->launches_last = 0;
    h->h2d_last = 0;

    PG_CK(cudaEventRecord(h->ev0, st));
    // S9: host-resident blocks are copied in for this call.
    if (h->residency == PGABB_RESIDENT_HOST && h->d_col.n) {
        PG_CK(cudaMemcpyAsync(h->d_col.p, h->h_col.p, h->d_col.bytes(), cudaMemcpyHostToDevice, st));
        PG_CK(cudaMemcpyAsync(h->d_rowptr.p, h->h_rowptr.p, h->d_rowptr.bytes(), cudaMemcpyHostToDevice, st));
        h->h2d_last = h->d_col.bytes() + h->d_rowptr.bytes();
    }
    PG_CK(cudaMemsetAsync(h->d_task_counts.p, 0, (nt + 1) * sizeof(unsigned long long), st));
    PG_CK(cudaMemsetAsync(h->d_next.p, 0, 8 * sizeof(unsigned long long), st));
    PG_CK(cudaEventRecord(h->ev1, st));
    if (h->work_edges) {
        int dev_sms = 148;
        PG_CK(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, h->device));
        const unsigned grid = (unsigned)dev_sms * 8;
        k_tc_warp<<<grid, kWarpsPerCta * 32, 0, st>>>(h->d_work.p, (int)h->work.size(), h->work_edges,
                                                     h->d_col.p, h->d_rowptr.p, h->d_task_counts.p, h->d_next.p);
        PG_LAUNCH_CHECK();
        h->launches_last++;
    }
    PG_CK(cudaEventRecord(h->ev2, st));
    k_sum_tasks<<<1, 1024, 0, st>>>(h->d_task_counts.p, nt, (unsigned long long*)(opts ? opts->d_count : nullptr));
    PG_LAUNCH_CHECK();
    h->launches_last++;
    PG_CK(cudaMemcpyAsync(h->h_result.p, h->d_task_counts.p + nt, 8, cudaMemcpyDeviceToHost, st));
    PG_CK(cudaEventRecord(h->ev3, st));
    h->timing_pending = true;
    if (async) {
        *wrote = false;
        return 0;
    }
    resolve_timing(h);
    if (opts && opts->task_counts && nt) {
        std::vector<unsigned long long> tc(nt);
        PG_CK(cudaMemcpy(tc.data(), h->d_task_counts.p, nt * 8, cudaMemcpyDeviceToHost));
        for (int t = 0; t < nt; ++t) opts->task_counts[t] = tc[t];
    }
    *wrote = true;
    return h->h_result.p[0];
}

}  // namespace pgabb
