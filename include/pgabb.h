/*
 * pgabb.h -- C ABI of the B200-native block-based triangle counter
 * (PGAbB, arXiv 2209.04541, the triangle-counting path of §3.6 / §5.4).
 *
 * The problem (§3.6 "An example: triangle counting"):
 *   "find the number of mutually connected sets of three vertices in an
 *    undirected graph".  Inputs are made "undirected, and removed duplicate
 *    edges" (§5.1), so tuples may hold both directions,
 *    duplicates and self-loops; the library canonicalises them (R1-R2).
 *
 * The method:
 *   pgabb_build_blocks    S1 canonicalise, S2 degree order,
 *                         S3 orient into a DAG ("only requires half of the
 *                         edges"), S4 conformal p-way cuts
 *                         (§4.3), S5 per-block CSR
 *                         (§4.3.2), S6 block triples
 *                         <A_ij, A_ix, A_jx> (Listing 5),
 *                         S7 task costs (the E functor),
 *                         S8 pieces + LPT over ranks.
 *   pgabb_triangle_count  S9 residency (host->device copy for host-resident
 *                         handles), S10 the intersections
 *                         n_t += |A_ix[u] ∩ A_jx[v]| for every (u,v) in A_ij
 *                         (Listing 5), S11 the count reduction.
 *   Beyond the count: pgabb_vertex_triangles / pgabb_local_clustering
 *   (per-vertex t(v), NEXT-1), pgabb_connected_components (Shiloach-Vishkin on the
 *   same blocks, NEXT-4), pgabb_task_times (measured task estimates for S8), and
 *   host-resident streaming through a device budget (S9 / NEXT-2, build options).
 *
 * Conventions (all entry points):
 *   - No C++ types or exceptions cross this boundary.  Every function returns a
 *     pgabb_status_t; on a non-OK status the output arguments are left untouched
 *     and pgabb_last_error() returns a thread-local message.
 *   - Input buffers are BORROWED for the duration of the call only.
 *   - A handle is owned by the library until pgabb_free(); one handle must not be
 *     used from two threads at once.  Distinct handles are independent.
 *   - All counts are exact uint64 and identical for every p, cut rule, world
 *     size, residency and run (SPEC.md:468 invariance; R10).
 *   - There is no CPU fallback: without a usable CUDA device (sm_100a) the calls
 *     return PGABB_ECUDA.
 */
#ifndef PGABB_H
#define PGABB_H

#include <stdint.h>

#if defined(__GNUC__)
#define PGABB_API __attribute__((visibility("default")))
#else
#define PGABB_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pgabb_blocks_s* pgabb_blocks_t;

typedef enum {
    PGABB_OK = 0,
    PGABB_EINVAL = 1,   /* bad argument: vertex id >= n, NULL pointer, bad option */
    PGABB_ENOMEM = 2,   /* device or pinned-host allocation failed */
    PGABB_ECUDA = 3,    /* CUDA error (incl. no device) */
    PGABB_ERANGE = 4,   /* size outside the supported range (a block with >= 2^32 edges) */
    PGABB_EBUDGET = 5   /* host-resident handle: one task's 3 blocks exceed the budget */
} pgabb_status_t;

/* Residency of the block CSR (S9; §4.4). */
enum {
    PGABB_RESIDENT_DEVICE = 0,  /* blocks live in HBM; counting reads them in place */
    PGABB_RESIDENT_HOST = 1     /* blocks live in pinned host DRAM; every count call
                                   copies the blocks its tasks need host->device
                                   (within device_budget_bytes) -- the paper's
                                   protocol, where H2D is part of the timed count
                                    */
};

typedef struct {
    uint32_t p;                 /* parts per dimension; 0 = 8; clamped to [1, n] */
    uint32_t cut_rule;          /* 0 = balance estimated work w(v) = d+(v) + d-(v)d+(v)
                                   1 = balance DAG out-degree w(v) = d+(v)
                                   2 = balance degree w(v) = d+(v) + d-(v)
                                   3 = balance estimated MID work w(v) = d+(v) + C(d+(v), 2)
                                   (DESIGN R7, R25) */
    int32_t device;             /* CUDA ordinal, -1 = current device */
    uint32_t inputs_on_device;  /* 1: src/dst are device pointers on `device`; the build
                                   synchronizes the device before reading them, so tuples
                                   still being produced on any stream are complete */
    int32_t rank;               /* this handle's rank in [0, world_size) (S8) */
    int32_t world_size;         /* ranks sharing the tasks; <= 1 means one GPU */
    uint32_t residency;         /* PGABB_RESIDENT_DEVICE or PGABB_RESIDENT_HOST */
    uint32_t reverse_order;     /* 1: S2 ranks are reversed (rank = n-1-position in the
                                   (deg, id) order), so the DAG runs from high degree to
                                   low; triangle counts are unchanged, and each triangle's
                                   lowest and highest vertices swap roles (NEXT-1 two-pass
                                   per-vertex counts, DESIGN R24) */
    uint64_t device_budget_bytes; /* HOST residency: device bytes for staged blocks;
                                     0 = stage all of this rank's blocks at once */
    const uint64_t* task_weights; /* optional HOST uint64[n_task_weights]: the task
                                     estimates E(t) ("E functor if
                                     defined"), in task order -- e.g. device time per
                                     task measured by pgabb_task_times on one GPU and
                                     broadcast, so that every rank plans the same
                                     pieces.  NULL = the S7 cost (DESIGN R17).  Used
                                     for splitting (cap = total/(4G)) and LPT; pieces
                                     are still cut at row-cost quantiles (R22).
                                     Borrowed for the call. */
    uint64_t n_task_weights;      /* must equal the task count when task_weights != NULL
                                     (EINVAL otherwise) */
    uint32_t orient;            /* task orientation (DESIGN R25; Listing 5, PAPER.md:689-697,
                                   fixes what a task sums, not which list is held):
                                   PGABB_ORIENT_AUTO (0, default) per task the one that
                                   streams fewer ids; PGABB_ORIENT_LOW (1) hold A_ix[u] per
                                   row u, stream A_jx[v] (no transposes are built);
                                   PGABB_ORIENT_MID (2) hold A_jx[v] per row v, stream the
                                   ids w > v of A_ix[u] for every (u,v) in A_ij (needs the
                                   blocks' transposes: 2 more u32 per edge).  Counts are
                                   identical for every value. */
    uint32_t host_permille;     /* collaborative CPU + GPU (PAPER.md:193-198,
                                   840-849: sparse tasks "more successful by assigning them to
                                   CPUs"): with PGABB_RESIDENT_HOST and no budget, this rank's
                                   sparsest pieces (least S7 cost per edge first) up to this
                                   share (per mille) of its cost are counted by host threads
                                   from the pinned host blocks while the GPU counts the rest;
                                   their blocks are not copied.  0 = GPU only (default).
                                   EINVAL with another residency, a budget, or > 1000.  Counts
                                   are unchanged; per-vertex counts and task times need 0. */
    uint32_t host_threads;      /* host threads for host_permille (0 = all hardware threads) */
    uint32_t light_held;        /* thread-per-row items (DESIGN R20, R29): 8 = rows with <= 8
                                   held ids; 15 = also rows with 9..15 held ids (a second
                                   kernel instantiation with 15 registers for them; heavy
                                   warp items otherwise); 0 = auto (DESIGN R29).  Other
                                   values: EINVAL.  Counts are identical for every value. */
} pgabb_build_opts_t;

#define PGABB_ORIENT_AUTO 0u
#define PGABB_ORIENT_LOW 1u
#define PGABB_ORIENT_MID 2u

/* Fills *opts with the defaults (p=0->8, rule 0, current device, one rank, HBM). */
PGABB_API void pgabb_default_build_opts(pgabb_build_opts_t* opts);

/*
 * S1-S8.  n: number of vertex ids; m: number of tuples; src[k], dst[k] < n are
 * the k-th tuple (uint32, host memory unless opts->inputs_on_device).  m == 0 is
 * valid (an empty graph, count 0).  Ids are uint32 (n <= 2^32 - 1) and |E| is 64-bit;
 * the only size limit is that no single block A_ij may hold 2^32 or more edges
 * (block-local offsets are uint32: ERANGE, pick a larger p), besides device memory
 * for the build (about 28 bytes per edge at the peak).
 * opts == NULL means defaults.  On success *out receives a new handle.
 * Errors: EINVAL (id >= n, src/dst NULL with m > 0, out NULL, bad rank/p/rule),
 *         ERANGE, ENOMEM, ECUDA.
 */
PGABB_API pgabb_status_t pgabb_build_blocks(uint32_t n, uint64_t m, const uint32_t* src,
                                  const uint32_t* dst, const pgabb_build_opts_t* opts,
                                  pgabb_blocks_t* out);

typedef struct {
    void* cuda_stream;          /* cudaStream_t to order the work on; NULL = handle's stream.
                                   The legacy default stream is cudaStreamLegacy ((void*)1),
                                   NOT NULL.  Calls on one handle are serialized on the
                                   device across streams: each call first waits for the
                                   previous call's work (a per-handle event), because they
                                   share the handle's scratch (task counts, arenas, t(v)). */
    uint64_t* d_count;          /* optional DEVICE uint64*: receives this rank's count,
                                   stream-ordered (for a caller-side NCCL allreduce) */
    uint64_t* task_counts;      /* optional HOST uint64[ntasks]: per-task counts of the
                                   pieces this rank owns (others 0) */
    uint32_t flags;             /* PGABB_COUNT_ASYNC: do not wait; *triangles untouched */
    uint32_t reserved0;
} pgabb_count_opts_t;

#define PGABB_COUNT_ASYNC 1u
#define PGABB_OUT_DEVICE 2u
/* pgabb_vertex_triangles roles (DESIGN R24): which vertices of a triangle {u<v<w}
   (rank order) are credited.  None set = all three.  Allowed: LOW, LOW|MID, LOW|MID|HIGH. */
#define PGABB_ROLE_LOW 4u
#define PGABB_ROLE_MID 8u
#define PGABB_ROLE_HIGH 16u
/* pgabb_vertex_triangles with PGABB_OUT_DEVICE: ADD this pass's t(v) into tv instead
   of overwriting it (the second pass of the two-pass route) */
/* pgabb_triangle_count / pgabb_vertex_triangles on a streaming handle: record CUDA
   events around every wave's copies and kernels (read with pgabb_get_wave_trace) */
#define PGABB_COUNT_TRACE 64u
#define PGABB_OUT_ACCUMULATE 32u     /* pgabb_vertex_triangles / pgabb_local_clustering: the
                                   tv and cc arrays are DEVICE pointers on the handle's
                                   device (stream-ordered on opts->cuda_stream) */

/*
 * S9-S11.  Counts the triangles of the pieces this handle's rank owns (all of
 * them when world_size <= 1) and writes the count to *triangles (host).  The
 * sum over ranks 0..world_size-1 of their counts is the triangle count T of the
 * canonicalised graph; combining them is the caller's allreduce (the Python
 * binding issues one NCCL allreduce of 8 bytes through torch.distributed).
 * opts == NULL: handle's stream, synchronous.
 */
PGABB_API pgabb_status_t pgabb_triangle_count(pgabb_blocks_t b, const pgabb_count_opts_t* opts,
                                    uint64_t* triangles);

/*
 * Per-vertex triangle counts.  opts->flags may restrict the
 * credited roles (PGABB_ROLE_*): LOW credits only each triangle's lowest-rank vertex
 * (one row total per (task,row): no per-hit atomics), LOW|MID adds the middle vertex
 * (per pair).  A handle built with reverse_order swaps LOW and HIGH, so
 *   t = [LOW|MID on the forward handle] + [LOW on the reversed handle]
 * is the cheap two-pass route to t(v); LOW|MID|HIGH on one handle is the one-pass route.  The paper motivates
 * triangle counting as the way "to measure clustering coefficients"
 * (§1); t(v) is the number of triangles containing v.
 * Same S9-S11 path as pgabb_triangle_count; every triangle {u<v<w} (rank
 * order) found by task (i,j,x) through edge (u,v) in A_ij and w in
 * A_ix[u] ∩ A_jx[v] adds 1 to t(u), t(v) and t(w).
 *   tv: uint64[n] indexed by ORIGINAL vertex id; receives this rank's share
 *       (the sum over ranks is t(v); sum_v t(v) = 3T).  HOST memory, or DEVICE
 *       memory on the handle's device when opts->flags has PGABB_OUT_DEVICE
 *       (then the caller may allreduce it over NCCL in place).  Overwritten.
 *   triangles: optional (NULL allowed); receives this rank's count, as
 *       pgabb_triangle_count.
 * PGABB_COUNT_ASYNC is allowed only with PGABB_OUT_DEVICE.
 * Errors: EINVAL (NULL handle, tv NULL with n > 0), ENOMEM, ECUDA.
 */
PGABB_API pgabb_status_t pgabb_vertex_triangles(pgabb_blocks_t b, const pgabb_count_opts_t* opts, uint64_t* tv,
                                      uint64_t* triangles);

/*
 * Local clustering coefficient cc(v) = 2 t(v) / (deg(v) (deg(v) - 1)), 0 when
 * deg(v) < 2 (deg in the canonicalised graph G_s, S1), for every ORIGINAL id v.
 *   tv: uint64[n], the COMPLETE t(v) (summed over ranks) -- input, borrowed.
 *   cc: double[n], output.  Both HOST, or both DEVICE with PGABB_OUT_DEVICE.
 * Computed in fp64 as one correctly rounded division of exact integers.
 * Synchronous.  Errors: EINVAL (NULL handle / arrays with n > 0), ENOMEM, ECUDA.
 */
PGABB_API pgabb_status_t pgabb_local_clustering(pgabb_blocks_t b, const pgabb_count_opts_t* opts,
                                      const uint64_t* tv, double* cc);

typedef struct {
    uint64_t n, m_tuples, m_edges;      /* m_edges = |E| = |E+| (DESIGN R15) */
    uint64_t p, ntasks, npieces, npieces_local;
    uint64_t wedges;                    /* W = sum_v d-(v) d+(v) */
    uint64_t cost_total, cost_local;    /* S7 cost units (DESIGN R17) */
    uint64_t alg_bytes_total, alg_bytes_local; /* staged-model bytes (R19) */
    uint64_t block_bytes;               /* bytes of block CSR (all blocks) */
    uint64_t h2d_bytes_last;            /* host->device bytes of the last count call */
    uint64_t launches_last;             /* kernels launched by the last count call */
    uint64_t waves;                     /* streaming residency: waves per count (0 otherwise) */
    uint64_t max_task_bytes;            /* largest block-triple footprint (col+rowptr+dense copy) */
    uint64_t items_heavy, items_light;  /* this rank's row items: warp per row / thread per row (DESIGN R20) */
    uint64_t alg_bytes_light;           /* staged-model bytes of the light items (within alg_bytes_local) */
    uint64_t d2d_bytes_last;            /* streaming: bytes re-used from the previous wave's arena
                                           (device-to-device) by the last count call */
    double ms_build;                    /* wall time of pgabb_build_blocks */
    double ms_count_last;               /* device time of the last count call (events) */
    double ms_main_kernel_last;         /* device time of the intersection kernels (heavy + light) */
    double ms_light_kernel_last;        /* device time of the light-row kernel alone */
    double ms_cc_last;                  /* device time of the last pgabb_connected_components */
    double ms_host_last;                /* host_permille > 0: wall time of the host threads' share
                                           of the last count (runs concurrently with the GPU) */
    uint64_t items_medium;              /* of items_light: the medium ones (9..15 held ids, R29) */
    uint64_t light_held;                /* the build's light_held (8 or 15; auto resolved) */
    uint64_t ell_bytes;                 /* device bytes of sector-aligned row slots (DESIGN R30) */
} pgabb_stats_t;

PGABB_API pgabb_status_t pgabb_get_stats(pgabb_blocks_t b, pgabb_stats_t* stats);

/*
 * Measured task estimates for the scheduler (S8; the paper's E functor,
 * PAPER.md:843-846).  Runs one count of this handle's pieces with per-task
 * cycle accounting and writes, for every task t, its share of the measured
 * device time in nanoseconds: ns[t] = sum over the two S10 kernels of
 * kernel_ns * cycles_t / cycles_all (HOST uint64[ntasks]; tasks this rank does
 * not own get 0).  Measure on a world_size-1 handle, broadcast, and pass as
 * pgabb_build_opts_t.task_weights so every rank plans identical pieces.
 * Device-resident handles only (EINVAL for streaming residency).
 * Errors: EINVAL (NULL argument), ECUDA.
 */
PGABB_API pgabb_status_t pgabb_task_times(pgabb_blocks_t b, uint64_t* ns);

/*
 * Connected components: Shiloach-Vishkin on the same blocks
 * (Listing 2): HOOK (for every edge, hook the greater root under
 * the smaller) and LINK (pointer jumping) alternate until a HOOK pass hooks nothing.
 *   labels: uint32[n], ORIGINAL ids: labels[v] = the smallest original id in v's
 *           component (a canonical labelling: isolated ids label themselves).
 *           HOST, or DEVICE with opts->flags & PGABB_OUT_DEVICE.
 *   ncomponents, iterations: optional outputs (HOOK+LINK rounds, the last one hooks 0).
 * One GPU (world_size 1), blocks resident or host-resident without a budget
 * (EINVAL otherwise).  Synchronous.  Errors: EINVAL, ENOMEM, ECUDA.
 */
PGABB_API pgabb_status_t pgabb_connected_components(pgabb_blocks_t b, const pgabb_count_opts_t* opts,
                                          uint32_t* labels, uint64_t* ncomponents, uint32_t* iterations);

/* ---- introspection (parity tests of S2..S8); all outputs are HOST buffers ---- */

/* rank[v] for every original id v < n: the position of v in the (deg, id) order. */
PGABB_API pgabb_status_t pgabb_get_rank(pgabb_blocks_t b, uint32_t* rank);
/* cuts[0..p] (rank space). */
PGABB_API pgabb_status_t pgabb_get_cuts(pgabb_blocks_t b, uint32_t* cuts);
/* Block A_ij, i <= j < p: *nnz always; rowptr[0..cut_{i+1}-cut_i] and col[0..nnz)
 * (local ids) when non-NULL.  EINVAL for i > j or j >= p. */
PGABB_API pgabb_status_t pgabb_get_block(pgabb_blocks_t b, uint32_t i, uint32_t j, uint32_t* rowptr,
                               uint32_t* col, uint64_t* nnz);
/* Tasks in (i, j, x) lexicographic order: ijx[3*t..3*t+2], cost[t], alg_bytes[t];
 * any output may be NULL. */
PGABB_API pgabb_status_t pgabb_get_tasks(pgabb_blocks_t b, uint32_t* ijx, uint64_t* cost,
                               uint64_t* alg_bytes);
/* Task orientations (DESIGN R25): dir[t] (0 LOW, 1 MID) and the ids each orientation
 * streams, s_low[t] = sum over (u,v) in A_ij of |A_jx[v]|, s_mid[t] = sum of
 * |{w in A_ix[u] : w > v}| (0 when the handle has no transposes, orient LOW); any
 * output may be NULL. */
PGABB_API pgabb_status_t pgabb_get_task_orient(pgabb_blocks_t b, uint32_t* dir, uint64_t* s_low,
                                     uint64_t* s_mid);
/* Pieces (S8) in (task, row) order: task[k], row_begin[k], row_end[k] (local rows of
 * part i for a LOW task, of part j for a MID task), cost[k], owner[k] (rank); any
 * output may be NULL. */
PGABB_API pgabb_status_t pgabb_get_pieces(pgabb_blocks_t b, uint32_t* task, uint32_t* row_begin,
                                uint32_t* row_end, uint64_t* cost, int32_t* owner);

/* Streaming residency (S9, "overlapping the next copy with the
 * computation"): the per-wave timeline of the last count made with PGABB_COUNT_TRACE,
 * four doubles per wave -- copy start, copy end (copy stream), compute start, compute
 * end (count stream) -- in ms from the start of the call.  *nwaves receives the wave
 * count; trace (HOST double[4 * nwaves]) may be NULL to query it.  Synchronous.
 * Errors: EINVAL (NULL handle or nwaves, no traced streaming count yet), ECUDA. */
PGABB_API pgabb_status_t pgabb_get_wave_trace(pgabb_blocks_t b, double* trace, uint64_t* nwaves);

/* Frees device and pinned-host memory.  NULL is a no-op. */
PGABB_API void pgabb_free(pgabb_blocks_t b);

/* Thread-local message for the last non-OK status of this thread ("" if none). */
PGABB_API const char* pgabb_last_error(void);

/* Library version string. */
PGABB_API const char* pgabb_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PGABB_H */
