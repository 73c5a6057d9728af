// internal.h -- handle layout, error plumbing and small device helpers shared by
// the build (S1-S8) and count (S9-S11) translation units of libpgabb.so.
// Nothing here is visible across the C ABI (include/pgabb.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "pgabb.h"

namespace pgabb {

struct Error {
    pgabb_status_t status;
    std::string msg;
};

[[noreturn]] void fail(pgabb_status_t st, const std::string& msg);
void check_cuda(cudaError_t e, const char* what, const char* file, int line);

#define PG_CK(x) ::pgabb::check_cuda((x), #x, __FILE__, __LINE__)

// NVTX ranges around the build steps and count phases (visible in nsys / ncu --nvtx)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};
#define PG_NVTX_CAT2(a, b) a##b
#define PG_NVTX_CAT(a, b) PG_NVTX_CAT2(a, b)
#define PG_NVTX(name) ::pgabb::NvtxRange PG_NVTX_CAT(pg_nvtx_, __LINE__)(name)
#define PG_LAUNCH_CHECK() ::pgabb::check_cuda(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

// Blocking copy ORDERED ON `st` (cudaMemcpyDefault, UVA).  The handle's stream is
// non-blocking, so a plain (legacy-stream) cudaMemcpy would not wait for the work
// queued on it: every host read of a buffer the library filled goes through here.
#define PG_COPY_SYNC(dst, src, bytes, st)                                                      \
    do {                                                                                       \
        PG_CK(cudaMemcpyAsync((dst), (src), (bytes), cudaMemcpyDefault, (st)));                \
        PG_CK(cudaStreamSynchronize(st));                                                      \
    } while (0)

constexpr int kMaxParts = 64;          // p <= 64 (tid table p^3 entries)
constexpr uint32_t kNoTask = 0xffffffffu;

// Device memory owned by the handle (freed in the destructor / on error unwinding).
template <class T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() { release(); }
    void alloc(size_t count) {
        release();
        if (count) {
            cudaError_t e = cudaMalloc(&p, count * sizeof(T));
            if (e != cudaSuccess) {
                p = nullptr;
                (void)cudaGetLastError();
                fail(PGABB_ENOMEM, "cudaMalloc of " + std::to_string(count * sizeof(T)) + " bytes failed");
            }
        }
        n = count;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    size_t bytes() const { return n * sizeof(T); }
};

// Pinned host memory (cudaHostAlloc), for host-resident handles.
template <class T>
struct HBuf {
    T* p = nullptr;
    size_t n = 0;
    HBuf() = default;
    HBuf(const HBuf&) = delete;
    HBuf& operator=(const HBuf&) = delete;
    ~HBuf() { release(); }
    void alloc(size_t count) {
        release();
        if (count) {
            cudaError_t e = cudaHostAlloc(&p, count * sizeof(T), cudaHostAllocDefault);
            if (e != cudaSuccess) {
                p = nullptr;
                (void)cudaGetLastError();
                fail(PGABB_ENOMEM, "cudaHostAlloc of " + std::to_string(count * sizeof(T)) + " bytes failed");
            }
        }
        n = count;
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        n = 0;
    }
};

// One block A_ij of the p x p grid (only i <= j can be non-empty: the DAG is
// upper triangular in rank space, DESIGN R4).  Pools are block-major.
struct BlockInfo {
    uint64_t nnz = 0;
    uint64_t col_off = 0;   // first edge in the col pool
    uint64_t rp_off = 0;    // first rowptr entry in the rowptr pool (nrows+1 entries)
    uint32_t nrows = 0;     // cut_{i+1} - cut_i
    uint32_t present = 0;   // nnz > 0 (rowptr stored)
    uint64_t bm_off = ~0ull; // dense copy: first word in the bitmap pool (~0: none)
    uint32_t bm_words = 0;   // words per bitmap row = ceil(width of column part / 32)
    // transpose (DESIGN R25, MID orientation): the same nnz entries ordered by (col v,
    // row u) at col_off inside the tcol / tpos regions of the col pool (tcol = u,
    // tpos = block-local position e of (u,v) in col), and ncols + 1 offsets at trp_off
    // in the rowptr pool (present blocks only, handles built with the transposes)
    uint64_t trp_off = 0;
    uint32_t ncols = 0;      // cut_{j+1} - cut_j
};

// Task orientation (DESIGN R25).  LOW (Listing 5's own loop order): per row u of
// part i hold A_ix[u] and stream A_jx[v] for every v in A_ij[u].  MID: per row v
// of part j hold A_jx[v] and stream, for every u with (u,v) in A_ij, the ids
// w > v of A_ix[u] -- all of it when x > j, the suffix after v when x == j.
constexpr uint32_t kDirLow = 0, kDirMid = 1;

struct Task {
    uint32_t i, j, x;
    uint32_t dir = kDirLow;  // orientation (R25)
    uint64_t cost = 0;       // S7 cost in the task's orientation (cost_low or cost_mid)
    uint64_t alg_bytes = 0;  // staged-model bytes in the task's orientation (alg_low or alg_mid)
    uint64_t cost_low = 0;   // R17: sum_{(u,v) in A_ij} (|A_ix[u]| + |A_jx[v]|)
    uint64_t alg_low = 0;    // R19: rows u with A_ij[u], A_ix[u] non-empty,
                             // 4*(|A_ix[u]| + sum_v |A_jx[v]|) + 12*|A_ij[u]|
    uint64_t cost_mid = 0;   // R25: sum over rows v with a non-empty column of A_ij of
                             // |A_jx[v]| + sum_u |{w in A_ix[u] : w > v}|
    uint64_t alg_mid = 0;    // R25: rows v with A_jx[v] and column v non-empty,
                             // 4*(|A_jx[v]| + sum_u |{w > v}|) + 12 per u
    uint64_t s_low = 0, s_mid = 0;   // ids streamed by each orientation (R25 auto choice)
};

struct Piece {
    uint32_t task;
    uint32_t r0, r1;         // local rows of part i (LOW task) or of part j (MID task)
    uint64_t cost;           // scheduling weight (S7 cost range, or the task weight's share, R22)
    int32_t owner;
    uint64_t rcost = 0;      // S7 row-cost range of the piece (for the bytes attribution)
};

// One owned piece of this rank (host work list).
struct PieceDev {
    uint64_t gstart;         // first position in this rank's flattened neighbour space
    uint32_t r0, r1;         // local row range of the piece (rows of the task's orientation)
    uint32_t e0, e1;         // neighbour range = nbr rowptr[r0], nbr rowptr[r1] (block-local)
    uint32_t task, dir;
};

// Per-task descriptor read by the intersection kernels, in kernel ROLES (R25):
//   row r     the item's vertex: u of part i (LOW) / v of part j (MID)
//   held S    the row's list: A_ix[u] (LOW) / A_jx[v] (MID)
//   nbr       the row's neighbours r': A_ij[u] = the v's (LOW) / column v of A_ij =
//             the u's (MID, the transpose)
//   streamed  each neighbour's list: A_jx[v] (LOW) / A_ix[u] from its first id > v
//             (MID: the suffix after position e of (u,v) in A_ij when x == j)
// All offsets are words into the col / rowptr / bitmap pools (or a wave's arena).
struct TaskDev {
    uint64_t s_col, s_rp;    // held block (col, rowptr)
    uint64_t n_col, n_rp;    // neighbour ids (col pool: A_ij's cols or the transpose's tcol) + rowptr
    uint64_t n_pos;          // MID with x == j: the transpose's tpos (suffix start - 1), else ~0
    uint64_t t_col, t_rp;    // streamed block (col, rowptr)
    uint64_t t_bm;           // bitmap copy of the streamed block, ~0 if list-only
    uint32_t wx;             // width of column part x (bits of a bitmap over it)
    uint32_t bm_words;       // words per dense row of the streamed block
    uint32_t c_row, c_nbr, cx;   // rank-space first vertex of the row's, the neighbours' and part x
    uint32_t dir;
    uint64_t t_ell;          // sector-aligned slots of the streamed block (R30), ~0 if none
    uint32_t ell_w;          // words per slot (8 or 16): [length, ids...]
    uint32_t pad_;
};
static_assert(sizeof(TaskDev) == 104, "TaskDev layout");

// A block gets a dense bitmap copy (rows of ceil(w/32) words) when its density is
// at least 1/kDenseInv and its column part is narrow enough for a warp bitmap:
// then the copy is no larger than the list form.
#ifndef PGABB_DENSE_INV
#define PGABB_DENSE_INV 32
#endif
constexpr uint64_t kDenseInv = PGABB_DENSE_INV;

// A heavy row item: (task, local row r, chunk c) with the row's held list and
// neighbour list non-empty; the warp takes neighbours [c*kChunkNbrs, (c+1)*kChunkNbrs)
// of the row (a MID hub row can have 10^5+ neighbours).  Packed as
// task << 48 | c << 32 | r.
constexpr uint32_t kColPad = 4;               // u32 words of padding after col pools / arenas
constexpr uint32_t kWarpBitmapBits = 32768;   // per-warp smem bitmap: 4 KB
constexpr uint32_t kHashMaxList = 512;        // per-warp smem hash: 1024 slots
#ifndef PGABB_CHUNK_NBRS
#define PGABB_CHUNK_NBRS 2048
#endif
constexpr uint32_t kChunkNbrs = PGABB_CHUNK_NBRS;   // neighbours per heavy item
__host__ __device__ inline uint32_t heavy_chunks(uint32_t le) { return (le + kChunkNbrs - 1) / kChunkNbrs; }

// Light rows (DESIGN R20): handled one per thread by k_tc_light, A_ix[u] held in
// registers.  A v list of <= kLightScan ids is scanned (each id compared with all
// of A_ix[u]); a longer one is binary-searched once per element of A_ix[u].
#ifndef PGABB_LIGHT_LA
#define PGABB_LIGHT_LA 8
#endif
constexpr uint32_t kLightLa = PGABB_LIGHT_LA;   // |A_ix[u]| <= kLightLa (the register copy)
// Medium rows: kLightLa < |held| <= kMedLa, otherwise light, go to a second
// instantiation of the thread-per-row kernel with kMedLa registers for the held ids
// (its own item list after the light one), so the light kernel keeps its occupancy
// (build option light_held; DESIGN R29).
#ifndef PGABB_MED_LA
#define PGABB_MED_LA 15
#endif
constexpr uint32_t kMedLa = PGABB_MED_LA;
#ifndef PGABB_LIGHT_LE
#define PGABB_LIGHT_LE 32
#endif
constexpr uint32_t kLightLe = PGABB_LIGHT_LE;      // |A_ij[u]| <= 32 pairs
#ifndef PGABB_LIGHT_SCAN
#define PGABB_LIGHT_SCAN 16
#endif
constexpr uint32_t kLightScan = PGABB_LIGHT_SCAN;
#ifndef PGABB_LIGHT_WORK
#define PGABB_LIGHT_WORK 128
#endif
constexpr uint32_t kLightWork = PGABB_LIGHT_WORK;   // list loads per row
// A light item carries its row's offsets, so the kernel starts with the lists
// instead of a chain of descriptor / rowptr loads:
//   x = task | |S| << 16 | |nbr| << 20,  y = held rowptr[r],  z = nbr rowptr[r],  w = r
// (task < 2^16: p <= 64 gives at most C(66,3) = 45760 tasks).
constexpr uint32_t kLightTaskBits = 16;
static_assert(kLightLa < 16 && kMedLa < 16 && kMedLa >= kLightLa && kLightLe < 4096, "light item bit fields");
static_assert((kMaxParts + 2) * (kMaxParts + 1) * kMaxParts / 6 < (1u << kLightTaskBits), "task id field");
__host__ __device__ inline uint32_t light_pair_loads(uint32_t la, uint32_t lb) {
    if (lb <= kLightScan) return lb;
    uint32_t lg = 0;
    while ((1u << lg) < lb + 1) ++lg;
    return la * lg;
}

// Streaming residency (S9): host-resident blocks are
// staged into one of two device arenas per wave of tasks; the copy of wave k+1
// (copy stream) overlaps the intersections of wave k.
struct StagedBlock {        // one H2D copy: pool range -> arena offset (u32 words)
    uint64_t src_word, dst_word, words;
    int pool;               // 0 col, 1 rowptr, 2 bitmap (host pools); 3 = the other arena (device copy)
};

// Per-block arrays a task reads, by kind (S9 residency and streaming): the col
// pool's three regions (cols, transposed u's, transposed positions), the rowptr
// pool's two (rowptr, transposed rowptr) and the bitmap pool.
enum BlockPart { kPartCol = 0, kPartRp = 1, kPartBm = 2, kPartTCol = 3, kPartTPos = 4, kPartTRp = 5 };

struct Wave {
    std::vector<StagedBlock> copies;   // dst_word: absolute arena offset; pool 3: src in the arena
    int slot = 0;               // arena slot this wave stages into
    int64_t wait_wave = -1;     // wave whose end must precede this wave's copies (slot reuse)
    uint64_t words = 0;         // slot words used
    size_t piece_begin = 0, piece_end = 0;   // range of owned pieces (locality order positions)
    uint64_t item_begin = 0, item_end = 0;   // its heavy row items (the build's item list)
    uint64_t light_begin = 0, light_end = 0; // its light row items
    uint64_t med_begin = 0, med_end = 0;     // its medium row items (in the light list, after n_light0)
    size_t task_table = 0;      // index of this wave's TaskDev table (ntasks entries)
};

}  // namespace pgabb

struct pgabb_blocks_s {
    int device = 0;
    cudaStream_t stream = nullptr;
    uint32_t n = 0;
    uint64_t m_tuples = 0, m_edges = 0;
    uint32_t p = 1;
    uint32_t cut_rule = 0;
    int32_t rank = 0, world_size = 1;
    uint32_t residency = PGABB_RESIDENT_DEVICE;
    uint32_t reverse_order = 0;                 // S2 ranks reversed (DESIGN R24)
    uint32_t orient = 0;                        // R25: 0 auto, 1 all LOW, 2 all MID
    bool has_t = false;                         // transposes built (orient != 1)
    uint64_t tcol_base = 0, tpos_base = 0;      // word offsets of the col pool's transpose regions
    uint64_t budget = 0;
    uint64_t wedges = 0;

    std::vector<uint32_t> cuts;                 // p+1
    std::vector<pgabb::BlockInfo> blocks;       // p*p, row-major block id i*p+j
    std::vector<pgabb::Task> tasks;             // (i,j,x) lexicographic
    std::vector<pgabb::Piece> pieces;           // (task, row) order
    std::vector<uint32_t> task_of_ijx;          // p^3 -> task id or kNoTask
    std::vector<uint64_t> task_weights;         // caller's E(t) (empty: the S7 cost)

    pgabb::DBuf<uint32_t> d_rank;               // original id -> rank
    pgabb::DBuf<uint32_t> d_deg;                // original id -> degree in G_s (S2; clustering)
    pgabb::DBuf<unsigned long long> d_tv_rank;  // per-vertex counts, rank space (allocated on demand)
    pgabb::DBuf<uint32_t> d_col;                // col pool (local col ids), block-major
    pgabb::DBuf<uint32_t> d_rowptr;             // rowptr pool (block-local edge offsets)
    pgabb::DBuf<uint32_t> d_bitmap;             // dense-block bitmap pool (rows of bm_words)
    pgabb::DBuf<uint32_t> d_ell;                // sector-aligned row slots of short-list blocks (R30)
    pgabb::HBuf<uint32_t> h_col, h_rowptr, h_bitmap;   // host-resident copies (RESIDENT_HOST)
    // RESIDENT_HOST without a budget: the pool ranges of the blocks this rank's pieces
    // read (merged), copied host->device by every count (S9) -- a rank never copies
    // blocks only other ranks' pieces need
    std::vector<pgabb::StagedBlock> host_copies;

    // this rank's work list (GPU pieces)
    std::vector<pgabb::PieceDev> work;
    uint64_t work_edges = 0;
    // collaborative CPU + GPU (NEXT-3): this rank's pieces counted by host threads from
    // the pinned host pools, with their task descriptors (host pool offsets)
    uint32_t host_permille = 0, host_threads = 0;
    std::vector<pgabb::PieceDev> host_work;
    std::vector<pgabb::TaskDev> host_tasks;
    pgabb::HBuf<unsigned long long> h_host_counts;   // per task, pinned (H2D into the device counts)
    pgabb::DBuf<unsigned long long> d_host_counts;
    double ms_host_last = 0;
    pgabb::DBuf<pgabb::TaskDev> d_tasks;             // ntasks descriptors
    pgabb::DBuf<unsigned long long> d_items;         // heavy row items (warp per row)
    uint64_t n_items = 0;
    pgabb::DBuf<uint4> d_light;                      // light row items (thread per row, DESIGN R20)
    uint64_t n_light = 0;                            // light + medium items
    uint64_t n_light0 = 0;                           // [0, n_light0) light, [n_light0, n_light) medium
    uint32_t light_held = pgabb::kLightLa;           // largest held list of a thread-per-row item (8 or 15)
    bool light_auto = false;                         // light_held chosen by the build (R29)
    // item offsets per owned piece in locality order (size pieces + 1): the waves of
    // streaming residency take contiguous ranges of them
    std::vector<uint64_t> piece_item_off, piece_light_off, piece_med_off;
    pgabb::DBuf<unsigned long long> d_task_counts;   // ntasks (+1 total at the end)
    pgabb::DBuf<unsigned long long> d_next;          // dynamic scheduling counters

    // streaming residency (budget > 0 with RESIDENT_HOST)
    bool streaming = false;
    uint64_t max_task_bytes = 0;
    std::vector<pgabb::Wave> waves;
    pgabb::DBuf<pgabb::TaskDev> d_wave_tasks;         // waves x ntasks, offsets relative to an arena
    pgabb::DBuf<uint32_t> d_arena;                    // slots x (slot_words + pad)
    int slots = 0;
    uint64_t slot_words = 0;
    cudaStream_t copy_stream = nullptr;
    std::vector<cudaEvent_t> ev_copied, ev_done;       // per wave (streaming)
    // PGABB_COUNT_TRACE: 4 timing events per wave (copy start/end, compute start/end)
    std::vector<cudaEvent_t> trace_ev;
    bool trace_valid = false;
    pgabb::HBuf<unsigned long long> h_result;        // pinned landing slot for the count

    cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr, ev3 = nullptr, ev_mid = nullptr;
    // end of the last call's work on the handle's scratch (task counts, counters,
    // arenas, t(v)); every call first waits for it on its own stream, so calls on
    // different streams never overlap on the scratch (pgabb::begin_call / end_call)
    cudaEvent_t ev_last = nullptr;
    bool ev_last_recorded = false;

    // stats
    uint64_t cost_total = 0, cost_local = 0, alg_total = 0, alg_local = 0;
    uint64_t h2d_last = 0, launches_last = 0, d2d_last = 0;
    double ms_build = 0, ms_count_last = 0, ms_main_last = 0, ms_light_last = 0;
    double ms_cc_last = 0;                    // device time of the last connected-components call
    uint32_t cc_iters_last = 0;
    uint64_t alg_light = 0;                   // staged-model bytes of the light items
    bool light_timed = false;                 // ev_mid recorded by the last count
    bool timing_pending = false;   // events of the last (async) count not read yet

    ~pgabb_blocks_s();
};

namespace pgabb {
void build_graph(pgabb_blocks_s* h, uint64_t m, const uint32_t* src, const uint32_t* dst, bool on_device);
void plan_pieces(pgabb_blocks_s* h);
void upload_work(pgabb_blocks_s* h);
void plan_waves(pgabb_blocks_s* h);
// the blocks and parts a task reads in its orientation (S9), and their word ranges
struct PartRef { uint32_t block; int part; };
int task_parts(const pgabb_blocks_s* h, const Task& T, PartRef out[8]);
uint64_t part_words(const pgabb_blocks_s* h, PartRef r);
uint64_t part_src(const pgabb_blocks_s* h, PartRef r, int* pool);   // word offset in host pool *pool
uint64_t count_triangles(pgabb_blocks_s* h, const pgabb_count_opts_t* opts, bool* wrote,
                         unsigned long long* d_tv_out = nullptr, unsigned long long* d_cycles = nullptr,
                         int vm = 3);
void task_times(pgabb_blocks_s* h, uint64_t* ns);
void wave_trace(pgabb_blocks_s* h, double* out, uint64_t* nwaves);
void connected_components(pgabb_blocks_s* h, const pgabb_count_opts_t* opts, uint32_t* labels, uint64_t* ncomp,
                          uint32_t* iters);
void local_clustering(pgabb_blocks_s* h, const pgabb_count_opts_t* opts, const uint64_t* tv, double* cc);
void resolve_timing(pgabb_blocks_s* h);
void settle_timing(pgabb_blocks_s* h);
void begin_call(pgabb_blocks_s* h, cudaStream_t st);
void end_call(pgabb_blocks_s* h, cudaStream_t st);
int sm_count(int device);   // multiprocessors of `device` (cached)
}  // namespace pgabb
