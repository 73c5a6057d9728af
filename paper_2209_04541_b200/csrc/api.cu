// api.cu -- the C ABI of include/pgabb.h: argument checking, handle lifetime,
// exception -> status translation, introspection copies.
#include <chrono>
#include <cstring>

#include "internal.h"

namespace pgabb {

namespace {
thread_local std::string g_last_error;
}

void fail(pgabb_status_t st, const std::string& msg) { throw Error{st, msg}; }

void check_cuda(cudaError_t e, const char* what, const char* file, int line) {
    if (e == cudaSuccess) return;
    (void)cudaGetLastError();
    const pgabb_status_t st = (e == cudaErrorMemoryAllocation) ? PGABB_ENOMEM : PGABB_ECUDA;
    fail(st, std::string(what) + " -> " + cudaGetErrorName(e) + ": " + cudaGetErrorString(e) + " (" + file +
                 ":" + std::to_string(line) + ")");
}

template <class F>
pgabb_status_t guarded(F f) {
    try {
        f();
        g_last_error.clear();
        return PGABB_OK;
    } catch (const Error& e) {
        g_last_error = e.msg;
        return e.status;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return PGABB_ENOMEM;
    } catch (...) {
        g_last_error = "unexpected internal error";
        return PGABB_ECUDA;
    }
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (dev >= 0) PG_CK(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

}  // namespace pgabb

pgabb_blocks_s::~pgabb_blocks_s() {
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    d_rank.release();
    d_col.release();
    d_rowptr.release();
    d_task_counts.release();
    d_next.release();
    h_col.release();
    h_rowptr.release();
    h_bitmap.release();
    d_wave_tasks.release();
    d_arena.release();
    for (cudaEvent_t e : ev_copied) cudaEventDestroy(e);
    for (cudaEvent_t e : ev_done) cudaEventDestroy(e);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    d_bitmap.release();
    d_tasks.release();
    d_items.release();
    d_light.release();
    d_ell.release();
    d_deg.release();
    d_tv_rank.release();
    h_result.release();
    for (cudaEvent_t e : {ev0, ev1, ev2, ev3, ev_mid, ev_last})
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : trace_ev) cudaEventDestroy(e);
    if (stream) cudaStreamDestroy(stream);
    if (prev >= 0) cudaSetDevice(prev);
}

using namespace pgabb;

extern "C" {

void pgabb_default_build_opts(pgabb_build_opts_t* o) {
    if (!o) return;
    std::memset(o, 0, sizeof(*o));
    o->p = 0;
    o->cut_rule = 0;
    o->device = -1;
    o->inputs_on_device = 0;
    o->rank = 0;
    o->world_size = 1;
    o->residency = PGABB_RESIDENT_DEVICE;
    o->device_budget_bytes = 0;
}

pgabb_status_t pgabb_build_blocks(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                                  const pgabb_build_opts_t* opts_in, pgabb_blocks_t* out) {
    pgabb_blocks_s* h = nullptr;
    pgabb_status_t st = guarded([&] {
        if (!out) fail(PGABB_EINVAL, "out is NULL");
        if (m > 0 && (!src || !dst)) fail(PGABB_EINVAL, "src/dst NULL with m > 0");
        // n < 2^32 (uint32 ids) and |E| are unbounded here; a block holding >= 2^32
        // edges is ERANGE (its offsets are 32-bit), checked by the build
        pgabb_build_opts_t o;
        pgabb_default_build_opts(&o);
        if (opts_in) o = *opts_in;
        if (o.cut_rule > 3) fail(PGABB_EINVAL, "cut_rule must be 0, 1, 2 or 3");
        if (o.residency > PGABB_RESIDENT_HOST) fail(PGABB_EINVAL, "bad residency");
        if (o.world_size < 1) o.world_size = 1;
        if (o.rank < 0 || o.rank >= o.world_size) fail(PGABB_EINVAL, "rank outside [0, world_size)");
        if (o.p > (uint32_t)kMaxParts) fail(PGABB_EINVAL, "p > 64 is not supported");
        const auto t0 = std::chrono::steady_clock::now();
        int dev = o.device;
        if (dev < 0) PG_CK(cudaGetDevice(&dev));
        int ndev = 0;
        PG_CK(cudaGetDeviceCount(&ndev));
        if (dev >= ndev) fail(PGABB_EINVAL, "device ordinal out of range");
        DeviceGuard g(dev);
        h = new pgabb_blocks_s();
        h->device = dev;
        PG_CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
        for (cudaEvent_t* e : {&h->ev0, &h->ev1, &h->ev2, &h->ev3, &h->ev_mid}) PG_CK(cudaEventCreate(e));
        PG_CK(cudaEventCreateWithFlags(&h->ev_last, cudaEventDisableTiming));
        h->h_result.alloc(1);
        h->n = n;
        h->m_tuples = m;
        uint32_t p = o.p ? o.p : 8;
        p = (n > 0) ? std::max<uint32_t>(1, std::min<uint32_t>(p, n)) : 1;   // DESIGN R7
        h->p = p;
        h->cut_rule = o.cut_rule;
        h->rank = o.rank;
        h->world_size = o.world_size;
        h->residency = o.residency;
        if (o.reverse_order > 1) fail(PGABB_EINVAL, "reverse_order must be 0 or 1");
        h->reverse_order = o.reverse_order;
        if (o.orient > PGABB_ORIENT_MID) fail(PGABB_EINVAL, "orient must be 0 (auto), 1 (low) or 2 (mid)");
        h->orient = o.orient;
        if (o.host_permille > 1000) fail(PGABB_EINVAL, "host_permille must be <= 1000");
        if (o.host_permille && (o.residency != PGABB_RESIDENT_HOST || o.device_budget_bytes))
            fail(PGABB_EINVAL, "host_permille needs PGABB_RESIDENT_HOST without a device budget");
        h->host_permille = o.host_permille;
        if (o.light_held != 0 && o.light_held != kLightLa && o.light_held != kMedLa)
            fail(PGABB_EINVAL, "light_held must be 0 (auto), " + std::to_string(kLightLa) + " or " +
                                   std::to_string(kMedLa));
        h->light_held = o.light_held ? o.light_held : kMedLa;
        h->light_auto = o.light_held == 0;
        h->host_threads = o.host_threads;
        h->budget = o.device_budget_bytes;
        h->streaming = (h->residency == PGABB_RESIDENT_HOST && h->budget > 0);
        if (o.task_weights) h->task_weights.assign(o.task_weights, o.task_weights + o.n_task_weights);
        else if (o.n_task_weights) fail(PGABB_EINVAL, "n_task_weights > 0 with task_weights NULL");
        PG_NVTX("pgabb_build_blocks");
        {
            PG_NVTX("S1-S7 build_graph");
            build_graph(h, m, src, dst, o.inputs_on_device != 0);
        }
        {
            PG_NVTX("S8 plan_pieces");
            plan_pieces(h);
        }
        {
            PG_NVTX("S8/S9 upload_work");
            upload_work(h);
        }
        if (h->streaming) {
            plan_waves(h);
            PG_CK(cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
            h->ev_copied.assign(h->waves.size(), nullptr);
            h->ev_done.assign(h->waves.size(), nullptr);
            for (size_t a = 0; a < h->waves.size(); ++a) {
                PG_CK(cudaEventCreateWithFlags(&h->ev_copied[a], cudaEventDisableTiming));
                PG_CK(cudaEventCreateWithFlags(&h->ev_done[a], cudaEventDisableTiming));
            }
        }
        if (h->residency == PGABB_RESIDENT_HOST) {
            h->h_col.alloc(h->d_col.n);
            h->h_rowptr.alloc(h->d_rowptr.n);
            if (h->d_col.n) PG_COPY_SYNC(h->h_col.p, h->d_col.p, h->d_col.bytes(), h->stream);
            if (h->d_rowptr.n)
                PG_COPY_SYNC(h->h_rowptr.p, h->d_rowptr.p, h->d_rowptr.bytes(), h->stream);
            h->h_bitmap.alloc(h->d_bitmap.n);
            if (h->d_bitmap.n)
                PG_COPY_SYNC(h->h_bitmap.p, h->d_bitmap.p, h->d_bitmap.bytes(), h->stream);
            if (h->streaming) {   // the graph now lives in pinned host DRAM only
                h->d_col.release();
                h->d_rowptr.release();
                h->d_bitmap.release();
            }
        }
        PG_CK(cudaStreamSynchronize(h->stream));
        h->ms_build = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        *out = h;
    });
    if (st != PGABB_OK && h) delete h;
    return st;
}

pgabb_status_t pgabb_triangle_count(pgabb_blocks_t b, const pgabb_count_opts_t* opts, uint64_t* triangles) {
    return guarded([&] {
        if (!b) fail(PGABB_EINVAL, "handle is NULL");
        const bool async = opts && (opts->flags & PGABB_COUNT_ASYNC);
        if (!triangles && !async) fail(PGABB_EINVAL, "triangles is NULL");
        DeviceGuard g(b->device);
        bool wrote = false;
        const uint64_t T = count_triangles(b, opts, &wrote);
        if (wrote) *triangles = T;
    });
}

pgabb_status_t pgabb_vertex_triangles(pgabb_blocks_t b, const pgabb_count_opts_t* opts, uint64_t* tv,
                                      uint64_t* triangles) {
    return guarded([&] {
        if (!b) fail(PGABB_EINVAL, "handle is NULL");
        if (!tv && b->n) fail(PGABB_EINVAL, "tv is NULL");
        if (opts && (opts->flags & PGABB_OUT_ACCUMULATE) && !(opts->flags & PGABB_OUT_DEVICE))
            fail(PGABB_EINVAL, "PGABB_OUT_ACCUMULATE needs PGABB_OUT_DEVICE");
        if (opts && (opts->flags & PGABB_COUNT_ASYNC) && !(opts->flags & PGABB_OUT_DEVICE))
            fail(PGABB_EINVAL, "PGABB_COUNT_ASYNC needs PGABB_OUT_DEVICE (a host tv is written synchronously)");
        if (!b->host_work.empty()) fail(PGABB_EINVAL, "per-vertex counts need host_permille 0");
        DeviceGuard g(b->device);
        const bool on_dev = opts && (opts->flags & PGABB_OUT_DEVICE);
        DBuf<unsigned long long> tmp;
        unsigned long long* d_out = (unsigned long long*)tv;
        if (!on_dev) {
            tmp.alloc(std::max<uint32_t>(b->n, 1));
            d_out = tmp.p;
        }
        bool wrote = false;
        const uint32_t roles = opts ? opts->flags & (PGABB_ROLE_LOW | PGABB_ROLE_MID | PGABB_ROLE_HIGH) : 0u;
        int vm = 3;
        if (roles == PGABB_ROLE_LOW) vm = 1;
        else if (roles == (PGABB_ROLE_LOW | PGABB_ROLE_MID)) vm = 2;
        else if (roles != 0 && roles != (PGABB_ROLE_LOW | PGABB_ROLE_MID | PGABB_ROLE_HIGH))
            fail(PGABB_EINVAL, "roles must be LOW, LOW|MID or LOW|MID|HIGH");
        const uint64_t T = count_triangles(b, opts, &wrote, d_out, nullptr, vm);
        if (!on_dev && b->n) {
            cudaStream_t st = (opts && opts->cuda_stream) ? (cudaStream_t)opts->cuda_stream : b->stream;
            PG_CK(cudaMemcpyAsync(tv, d_out, (size_t)b->n * 8, cudaMemcpyDeviceToHost, st));
            PG_CK(cudaStreamSynchronize(st));
        }
        if (wrote && triangles) *triangles = T;
    });
}

pgabb_status_t pgabb_local_clustering(pgabb_blocks_t b, const pgabb_count_opts_t* opts, const uint64_t* tv,
                                      double* cc) {
    return guarded([&] {
        if (!b) fail(PGABB_EINVAL, "handle is NULL");
        if ((!tv || !cc) && b->n) fail(PGABB_EINVAL, "tv or cc is NULL");
        DeviceGuard g(b->device);
        local_clustering(b, opts, tv, cc);
    });
}

pgabb_status_t pgabb_task_times(pgabb_blocks_t b, uint64_t* ns) {
    return guarded([&] {
        if (!b || !ns) fail(PGABB_EINVAL, "NULL argument");
        if (b->streaming) fail(PGABB_EINVAL, "task times are measured on a device-resident handle");
        if (!b->host_work.empty()) fail(PGABB_EINVAL, "task times need host_permille 0");
        DeviceGuard g(b->device);
        task_times(b, ns);
    });
}

pgabb_status_t pgabb_connected_components(pgabb_blocks_t b, const pgabb_count_opts_t* opts, uint32_t* labels,
                                         uint64_t* ncomponents, uint32_t* iterations) {
    return guarded([&] {
        if (!b) fail(PGABB_EINVAL, "handle is NULL");
        if (!labels && b->n) fail(PGABB_EINVAL, "labels is NULL");
        DeviceGuard g(b->device);
        connected_components(b, opts, labels, ncomponents, iterations);
    });
}

pgabb_status_t pgabb_get_stats(pgabb_blocks_t b, pgabb_stats_t* s) {
    return guarded([&] {
        if (!b || !s) fail(PGABB_EINVAL, "NULL argument");
        if (b->timing_pending) {
            DeviceGuard g(b->device);
            resolve_timing(b);
        }
        std::memset(s, 0, sizeof(*s));
        s->n = b->n;
        s->m_tuples = b->m_tuples;
        s->m_edges = b->m_edges;
        s->p = b->p;
        s->ntasks = b->tasks.size();
        s->npieces = b->pieces.size();
        s->npieces_local = b->work.size();
        s->wedges = b->wedges;
        s->cost_total = b->cost_total;
        s->cost_local = b->cost_local;
        s->alg_bytes_total = b->alg_total;
        s->alg_bytes_local = b->alg_local;
        // streaming handles keep the pools in pinned host DRAM only
        s->block_bytes = b->streaming ? 4 * (b->h_col.n + b->h_rowptr.n + b->h_bitmap.n)
                                      : b->d_col.bytes() + b->d_rowptr.bytes() + b->d_bitmap.bytes();
        s->h2d_bytes_last = b->h2d_last;
        s->launches_last = b->launches_last;
        s->waves = b->waves.size();
        s->max_task_bytes = b->max_task_bytes;
        s->ms_build = b->ms_build;
        s->ms_count_last = b->ms_count_last;
        s->ms_main_kernel_last = b->ms_main_last;
        s->ms_light_kernel_last = b->ms_light_last;
        s->ms_cc_last = b->ms_cc_last;
        s->ms_host_last = b->ms_host_last;
        s->items_heavy = b->n_items;
        s->items_light = b->n_light;
        s->items_medium = b->n_light - b->n_light0;
        s->light_held = b->light_held;
        s->ell_bytes = b->d_ell.bytes();
        s->alg_bytes_light = b->alg_light;
        s->d2d_bytes_last = b->d2d_last;
    });
}

pgabb_status_t pgabb_get_rank(pgabb_blocks_t b, uint32_t* rank) {
    return guarded([&] {
        if (!b || !rank) fail(PGABB_EINVAL, "NULL argument");
        DeviceGuard g(b->device);
        if (b->n) PG_COPY_SYNC(rank, b->d_rank.p, (size_t)b->n * 4, b->stream);
    });
}

pgabb_status_t pgabb_get_cuts(pgabb_blocks_t b, uint32_t* cuts) {
    return guarded([&] {
        if (!b || !cuts) fail(PGABB_EINVAL, "NULL argument");
        std::memcpy(cuts, b->cuts.data(), b->cuts.size() * 4);
    });
}

pgabb_status_t pgabb_get_block(pgabb_blocks_t b, uint32_t i, uint32_t j, uint32_t* rowptr, uint32_t* col,
                               uint64_t* nnz) {
    return guarded([&] {
        if (!b || !nnz) fail(PGABB_EINVAL, "NULL argument");
        if (i > j || j >= b->p) fail(PGABB_EINVAL, "block index must satisfy i <= j < p");
        DeviceGuard g(b->device);
        const BlockInfo& bi = b->blocks[(size_t)i * b->p + j];
        *nnz = bi.nnz;
        // streaming handles keep the pools in pinned host memory only
        const uint32_t* rp_pool = b->d_rowptr.p ? b->d_rowptr.p : b->h_rowptr.p;
        const uint32_t* col_pool = b->d_col.p ? b->d_col.p : b->h_col.p;
        if (rowptr) {
            if (bi.present)
                PG_COPY_SYNC(rowptr, rp_pool + bi.rp_off, ((size_t)bi.nrows + 1) * 4, b->stream);
            else
                std::memset(rowptr, 0, ((size_t)bi.nrows + 1) * 4);
        }
        if (col && bi.nnz) PG_COPY_SYNC(col, col_pool + bi.col_off, bi.nnz * 4, b->stream);
    });
}

pgabb_status_t pgabb_get_tasks(pgabb_blocks_t b, uint32_t* ijx, uint64_t* cost, uint64_t* alg) {
    return guarded([&] {
        if (!b) fail(PGABB_EINVAL, "NULL argument");
        for (size_t t = 0; t < b->tasks.size(); ++t) {
            const Task& T = b->tasks[t];
            if (ijx) { ijx[3 * t] = T.i; ijx[3 * t + 1] = T.j; ijx[3 * t + 2] = T.x; }
            if (cost) cost[t] = T.cost;
            if (alg) alg[t] = T.alg_bytes;
        }
    });
}

pgabb_status_t pgabb_get_task_orient(pgabb_blocks_t b, uint32_t* dir, uint64_t* s_low, uint64_t* s_mid) {
    return guarded([&] {
        if (!b) fail(PGABB_EINVAL, "NULL argument");
        for (size_t t = 0; t < b->tasks.size(); ++t) {
            const Task& T = b->tasks[t];
            if (dir) dir[t] = T.dir;
            if (s_low) s_low[t] = T.s_low;
            if (s_mid) s_mid[t] = T.s_mid;
        }
    });
}

pgabb_status_t pgabb_get_pieces(pgabb_blocks_t b, uint32_t* task, uint32_t* r0, uint32_t* r1, uint64_t* cost,
                                int32_t* owner) {
    return guarded([&] {
        if (!b) fail(PGABB_EINVAL, "NULL argument");
        for (size_t k = 0; k < b->pieces.size(); ++k) {
            const Piece& P = b->pieces[k];
            if (task) task[k] = P.task;
            if (r0) r0[k] = P.r0;
            if (r1) r1[k] = P.r1;
            if (cost) cost[k] = P.cost;
            if (owner) owner[k] = P.owner;
        }
    });
}

pgabb_status_t pgabb_get_wave_trace(pgabb_blocks_t b, double* trace, uint64_t* nwaves) {
    return guarded([&] {
        if (!b || !nwaves) fail(PGABB_EINVAL, "NULL argument");
        DeviceGuard g(b->device);
        wave_trace(b, trace, nwaves);
    });
}

void pgabb_free(pgabb_blocks_t b) { delete b; }

const char* pgabb_last_error(void) { return g_last_error.c_str(); }

const char* pgabb_version(void) { return "pgabb-b200 0.1 (sm_100a)"; }

}  // extern "C"
