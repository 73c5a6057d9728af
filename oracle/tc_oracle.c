/*
 * tc_oracle.c -- TEST INFRASTRUCTURE ONLY.  The plain CPU triangle-count oracle.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header,
 * table or helper with the CUDA path (paper_2209_04541_b200/csrc); it reads the
 * same edge tuples the generators in gen/ emit and nothing else.
 *
 * What it computes (§3.6: "find the number of mutually
 * connected sets of three vertices in an undirected graph"; inputs made
 * "undirected, and removed duplicate edges", §5.1):
 *
 *   G_s = simple undirected graph of the tuples (symmetrised, self-loops and
 *         duplicates dropped -- DESIGN.md readings R1, R2)
 *   T   = |{ {a,b,c} : ab, bc, ac in E(G_s) }|
 *   t(v)= number of those triples containing v          (sum_v t(v) = 3T)
 *
 * Algorithm: the node iterator with marks over the degree order
 * (§5.4 "degree-based vertex ordering"):
 *   v < w  iff  (deg v, v) < (deg w, w)        (reading R3)
 *   N+(v) = { w in N(v) : v < w }
 *   for each v: mark N+(v); for u in N+(v), for w in N+(u): if marked(w) the
 *   triangle {v,u,w} (v < u < w) is counted -- exactly once per triangle.
 *
 * oracle_brute() is the O(n^3) definition itself (dense adjacency, triple loop
 * over a<b<c), used to pin the node iterator on small graphs.
 *
 * Pins (tests/test_oracle.py): brute force, closed forms (K_n, C_n, trees,
 * grids, wheels, windmills, rook and king graphs, clique unions), scipy
 * trace(A^3)/6, networkx.triangles, sum t(v) = 3T, metamorphic invariants.
 *
 * Build: gcc -O2 -fopenmp -shared -fPIC oracle/tc_oracle.c -o oracle/liboracle.so
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

typedef struct {
    uint32_t n;
    uint64_t m_edges;     /* unique undirected non-loop edges */
    uint64_t* beg;        /* N(v) = adj[beg[v] .. beg[v]+deg[v]), sorted by id */
    uint32_t* deg;
    uint32_t* adj;
    uint64_t* pbeg;       /* N+(v) = padj[pbeg[v] .. pbeg[v+1]), sorted by id */
    uint32_t* padj;
} oracle_graph;

static int cmp_u32(const void* a, const void* b) {
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return (x > y) - (x < y);
}

/* v precedes w in the degree order: (deg v, v) < (deg w, w). */
static inline int precedes(const oracle_graph* g, uint32_t v, uint32_t w) {
    return g->deg[v] < g->deg[w] || (g->deg[v] == g->deg[w] && v < w);
}

void oracle_free(oracle_graph* g) {
    if (!g) return;
    free(g->beg); free(g->deg); free(g->adj); free(g->pbeg); free(g->padj);
    free(g);
}

/* Build G_s from m tuples.  Returns NULL on an id >= n or allocation failure. */
oracle_graph* oracle_build(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst) {
    for (uint64_t k = 0; k < m; ++k)
        if (src[k] >= n || dst[k] >= n) return NULL;
    oracle_graph* g = (oracle_graph*)calloc(1, sizeof(oracle_graph));
    if (!g) return NULL;
    g->n = n;
    uint64_t* cnt = (uint64_t*)calloc((size_t)n + 1, sizeof(uint64_t));
    g->beg = (uint64_t*)malloc(((size_t)n + 1) * sizeof(uint64_t));
    g->deg = (uint32_t*)calloc((size_t)n + 1, sizeof(uint32_t));
    g->pbeg = (uint64_t*)calloc((size_t)n + 1, sizeof(uint64_t));
    if (!cnt || !g->beg || !g->deg || !g->pbeg) { free(cnt); oracle_free(g); return NULL; }

    /* 1. symmetrise: both directions of every non-loop tuple (duplicates kept). */
    #pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < (int64_t)m; ++k) {
        if (src[k] == dst[k]) continue;
        #pragma omp atomic
        cnt[src[k]]++;
        #pragma omp atomic
        cnt[dst[k]]++;
    }
    uint64_t tot = 0;
    for (uint32_t v = 0; v < n; ++v) { g->beg[v] = tot; tot += cnt[v]; }
    g->beg[n] = tot;
    g->adj = (uint32_t*)malloc((tot ? tot : 1) * sizeof(uint32_t));
    if (!g->adj) { free(cnt); oracle_free(g); return NULL; }
    memset(cnt, 0, ((size_t)n + 1) * sizeof(uint64_t));
    #pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < (int64_t)m; ++k) {
        uint32_t a = src[k], b = dst[k];
        if (a == b) continue;
        uint64_t pa, pb;
        #pragma omp atomic capture
        pa = cnt[a]++;
        #pragma omp atomic capture
        pb = cnt[b]++;
        g->adj[g->beg[a] + pa] = b;
        g->adj[g->beg[b] + pb] = a;
    }
    free(cnt);

    /* 2. sort each list and drop duplicates: deg[v] = |N(v)|. */
    uint64_t m2 = 0;
    #pragma omp parallel for schedule(dynamic, 1024) reduction(+:m2)
    for (int64_t v = 0; v < (int64_t)n; ++v) {
        uint32_t* L = g->adj + g->beg[v];
        uint64_t len = g->beg[v + 1] - g->beg[v];
        if (len > 1) qsort(L, len, sizeof(uint32_t), cmp_u32);
        uint64_t d = 0;
        for (uint64_t i = 0; i < len; ++i)
            if (d == 0 || L[d - 1] != L[i]) L[d++] = L[i];
        g->deg[v] = (uint32_t)d;
        m2 += d;
    }
    g->m_edges = m2 / 2;

    /* 3. N+(v): the neighbours that follow v in the degree order. */
    #pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t v = 0; v < (int64_t)n; ++v) {
        const uint32_t* L = g->adj + g->beg[v];
        uint64_t c = 0;
        for (uint32_t i = 0; i < g->deg[v]; ++i) c += (uint64_t)precedes(g, (uint32_t)v, L[i]);
        g->pbeg[v + 1] = c;
    }
    for (uint32_t v = 0; v < n; ++v) g->pbeg[v + 1] += g->pbeg[v];
    g->padj = (uint32_t*)malloc((g->pbeg[n] ? g->pbeg[n] : 1) * sizeof(uint32_t));
    if (!g->padj) { oracle_free(g); return NULL; }
    #pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t v = 0; v < (int64_t)n; ++v) {
        const uint32_t* L = g->adj + g->beg[v];
        uint64_t o = g->pbeg[v];
        for (uint32_t i = 0; i < g->deg[v]; ++i)
            if (precedes(g, (uint32_t)v, L[i])) g->padj[o++] = L[i];
    }
    return g;
}

uint64_t oracle_num_edges(const oracle_graph* g) { return g->m_edges; }
uint32_t oracle_num_vertices(const oracle_graph* g) { return g->n; }

/* Copy out deg[n] (for the python-side checks of the degree step). */
void oracle_degrees(const oracle_graph* g, uint32_t* deg_out) {
    memcpy(deg_out, g->deg, (size_t)g->n * sizeof(uint32_t));
}

/*
 * Node iterator over v = v0, v0+stride, ... < v1 (the whole graph for
 * v0=0, v1=n, stride=1).  Returns the number of triangles whose lowest vertex
 * (in the degree order) is one of those v; adds into tv[] (nullable) the
 * per-vertex counts of exactly those triangles; *dag_edges_out (nullable)
 * receives sum |N+(v)| over the visited v (the DAG edges they own).
 */
uint64_t oracle_count_range(const oracle_graph* g, uint32_t v0, uint32_t v1, uint32_t stride,
                            uint64_t* tv, uint64_t* dag_edges_out) {
    if (stride == 0) stride = 1;
    if (v1 > g->n) v1 = g->n;
    const uint64_t words = ((uint64_t)g->n + 63) / 64;
    uint64_t T = 0, edges = 0;
    int fail = 0;
    #pragma omp parallel reduction(+:T, edges)
    {
        uint64_t* mark = (uint64_t*)calloc(words ? words : 1, sizeof(uint64_t));
        if (!mark) {
            #pragma omp atomic write
            fail = 1;
        }
        #pragma omp for schedule(dynamic, 64)
        for (int64_t vi = (int64_t)v0; vi < (int64_t)v1; vi += stride) {
            if (!mark) continue;
            const uint32_t v = (uint32_t)vi;
            const uint32_t* Nv = g->padj + g->pbeg[v];
            const uint64_t dv = g->pbeg[v + 1] - g->pbeg[v];
            edges += dv;
            for (uint64_t i = 0; i < dv; ++i) mark[Nv[i] >> 6] |= 1ull << (Nv[i] & 63);
            for (uint64_t i = 0; i < dv; ++i) {
                const uint32_t u = Nv[i];
                const uint32_t* Nu = g->padj + g->pbeg[u];
                const uint64_t du = g->pbeg[u + 1] - g->pbeg[u];
                for (uint64_t k = 0; k < du; ++k) {
                    const uint32_t w = Nu[k];
                    if (mark[w >> 6] >> (w & 63) & 1ull) {
                        T += 1;
                        if (tv) {
                            #pragma omp atomic
                            tv[v]++;
                            #pragma omp atomic
                            tv[u]++;
                            #pragma omp atomic
                            tv[w]++;
                        }
                    }
                }
            }
            for (uint64_t i = 0; i < dv; ++i) mark[Nv[i] >> 6] = 0;
        }
        free(mark);
    }
    if (dag_edges_out) *dag_edges_out = edges;
    return fail ? ~0ull : T;
}

uint64_t oracle_count(const oracle_graph* g, uint64_t* tv) {
    return oracle_count_range(g, 0, g->n, 1, tv, NULL);
}

/* Wedge count W = sum_v d-(v) * d+(v) of the degree-ordered DAG. */
uint64_t oracle_wedges(const oracle_graph* g) {
    uint64_t W = 0;
    #pragma omp parallel for schedule(dynamic, 1024) reduction(+:W)
    for (int64_t v = 0; v < (int64_t)g->n; ++v) {
        uint64_t dp = g->pbeg[v + 1] - g->pbeg[v];
        W += (uint64_t)(g->deg[v] - dp) * dp;
    }
    return W;
}

/* Brute force, the definition itself: dense adjacency, triple loop a<b<c.
 * n <= 4096 (dense matrix of n^2 bytes).  Returns ~0 on bad input. */
uint64_t oracle_brute(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst) {
    if (n > 4096) return ~0ull;
    unsigned char* A = (unsigned char*)calloc((size_t)n * n + 1, 1);
    if (!A) return ~0ull;
    for (uint64_t k = 0; k < m; ++k) {
        uint32_t a = src[k], b = dst[k];
        if (a >= n || b >= n) { free(A); return ~0ull; }
        if (a == b) continue;
        A[(size_t)a * n + b] = 1;
        A[(size_t)b * n + a] = 1;
    }
    uint64_t T = 0;
    #pragma omp parallel for schedule(dynamic, 1) reduction(+:T)
    for (int64_t a = 0; a < (int64_t)n; ++a)
        for (uint32_t b = (uint32_t)a + 1; b < n; ++b) {
            if (!A[(size_t)a * n + b]) continue;
            for (uint32_t c = b + 1; c < n; ++c)
                T += A[(size_t)a * n + c] & A[(size_t)b * n + c];
        }
    free(A);
    return T;
}

int oracle_threads(void) { return omp_get_max_threads(); }
/* thread count for later parallel regions (torchrun sets OMP_NUM_THREADS=1 per rank) */
void oracle_set_threads(int k) { if (k > 0) omp_set_num_threads(k); }

/*
 * Connected components of G_s (the problem the paper's
 * Shiloach-Vishkin example solves): labels[v] = the smallest
 * vertex id of v's component.  Plain sequential union-find over the undirected
 * adjacency: the root of every tree is the smallest id in it (a union hangs the
 * greater root under the smaller one), find() halves paths.  Returns the number
 * of components.  Pinned by tests/test_oracle.py (scipy connected_components,
 * BFS on small graphs, closed forms).
 */
static uint32_t uf_find(uint32_t* par, uint32_t x) {
    while (par[x] != x) {
        par[x] = par[par[x]];
        x = par[x];
    }
    return x;
}

uint64_t oracle_components(const oracle_graph* g, uint32_t* labels) {
    const uint32_t n = g->n;
    uint32_t* par = (uint32_t*)malloc((size_t)(n ? n : 1) * 4);
    if (!par) return ~0ull;
    for (uint32_t v = 0; v < n; ++v) par[v] = v;
    for (uint32_t v = 0; v < n; ++v)
        for (uint64_t k = g->beg[v]; k < g->beg[v] + g->deg[v]; ++k) {
            const uint32_t a = uf_find(par, v), b = uf_find(par, g->adj[k]);
            if (a != b) par[a > b ? a : b] = a < b ? a : b;
        }
    uint64_t nc = 0;
    for (uint32_t v = 0; v < n; ++v) {
        labels[v] = uf_find(par, v);
        nc += (labels[v] == v);
    }
    free(par);
    return nc;
}

/*
 * Per-vertex counts split by role (DESIGN R24): for every triangle v < u < w in
 * the degree order, tlow[v], tmid[u], thigh[w] += 1.  The node iterator of
 * oracle_count_range, sequential, with three arrays.  tlow + tmid + thigh = t.
 */
uint64_t oracle_count_roles(const oracle_graph* g, uint64_t* tlow, uint64_t* tmid, uint64_t* thigh) {
    const uint64_t words = ((uint64_t)g->n + 63) / 64;
    uint64_t* mark = (uint64_t*)calloc(words ? words : 1, sizeof(uint64_t));
    if (!mark) return ~0ull;
    uint64_t T = 0;
    for (uint32_t v = 0; v < g->n; ++v) {
        const uint32_t* Nv = g->padj + g->pbeg[v];
        const uint64_t dv = g->pbeg[v + 1] - g->pbeg[v];
        for (uint64_t i = 0; i < dv; ++i) mark[Nv[i] >> 6] |= 1ull << (Nv[i] & 63);
        for (uint64_t i = 0; i < dv; ++i) {
            const uint32_t u = Nv[i];
            const uint32_t* Nu = g->padj + g->pbeg[u];
            const uint64_t du = g->pbeg[u + 1] - g->pbeg[u];
            for (uint64_t k = 0; k < du; ++k) {
                const uint32_t w = Nu[k];
                if (mark[w >> 6] >> (w & 63) & 1ull) {
                    ++T;
                    tlow[v]++;
                    tmid[u]++;
                    thigh[w]++;
                }
            }
        }
        for (uint64_t i = 0; i < dv; ++i) mark[Nv[i] >> 6] = 0;
    }
    free(mark);
    return T;
}
