/*
 * gen.c -- seeded synthetic graph generators (edge tuples), shared by the
 * oracle, the tests and bench.py.
 *
 * This module holds NONE of the triangle-counting method's arithmetic: it only
 * emits (src, dst) uint32 tuples.  Every tuple is a pure function of
 * (seed, family parameters, tuple index) -- a counter-based generator -- so the
 * output is identical for any OpenMP thread count and can be regenerated
 * chunk by chunk.
 *
 * Families (SURVEY.md §8(c) readings 12-14):
 *   R-MAT  Graph500 a,b,c,d = .57,.19,.19,.05, no noise, ef*2^scale tuples,
 *          followed by a seeded bijective relabelling of the 2^scale ids.
 *   ER     G(n,m) with replacement: m iid uniform (u,v) tuples.
 *   grid   side x side 4-neighbour lattice, plus the diagonal (r,c)-(r+1,c+1)
 *          in each cell whose hash falls below f (road-network-like).
 *
 * Build: gcc -O2 -fopenmp -shared -fPIC gen/gen.c -o gen/libpgabb_gen.so
 */
#include <stdint.h>
#include <stddef.h>

static inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* Counter-based draw: 64 random bits for (seed, stream, counter). */
static inline uint64_t draw(uint64_t seed, uint64_t stream, uint64_t k) {
    return mix64(mix64(seed * 0xD1B54A32D192ED03ull + stream) ^ k);
}

/* Seeded bijection on [0, 2^bits): odd multiply + add, then xor-shift, x3. */
typedef struct { uint64_t odd[3], add[3]; } perm_key;

static perm_key perm_make(uint64_t seed) {
    perm_key pk;
    for (int r = 0; r < 3; ++r) {
        pk.odd[r] = draw(seed, 0xA11CE + r, 0) | 1ull;
        pk.add[r] = draw(seed, 0xB0B + r, 0);
    }
    return pk;
}

static inline uint64_t permute_bits(uint64_t x, int bits, const perm_key* pk) {
    if (bits <= 0) return x;
    const uint64_t mask = (bits >= 64) ? ~0ull : ((1ull << bits) - 1);
    const int sh = (bits + 1) / 2;
    for (int r = 0; r < 3; ++r) {
        x = (x * pk->odd[r] + pk->add[r]) & mask;
        x ^= x >> sh;
    }
    return x & mask;
}

uint64_t pgabb_gen_permute(uint64_t x, int bits, uint64_t seed) {
    perm_key pk = perm_make(seed);
    return permute_bits(x, bits, &pk);
}

/* R-MAT: tuples [k0, k0+count) of the stream, written to src/dst[0..count).
 * One 64-bit draw per pair of recursion levels; each level uses 32 bits. */
void pgabb_gen_rmat(int scale, uint64_t seed, int permute, uint64_t k0, uint64_t count,
                    uint32_t* src, uint32_t* dst) {
    /* Graph500 initiator probabilities in units of 2^-32. */
    const double a = 0.57, b = 0.19, c = 0.19;
    const uint64_t ta = (uint64_t)(a * 4294967296.0);
    const uint64_t tab = (uint64_t)((a + b) * 4294967296.0);
    const uint64_t tabc = (uint64_t)((a + b + c) * 4294967296.0);
    uint64_t key[32];
    for (int q = 0; q < 32; ++q) key[q] = mix64(seed * 0xD1B54A32D192ED03ull + 1 + (uint64_t)q);
    const perm_key pk = perm_make(seed ^ 0x5EED5EEDull);
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)count; ++i) {
        const uint64_t k = k0 + (uint64_t)i;
        uint64_t u = 0, v = 0, h = 0;
        for (int l = 0; l < scale; ++l) {
            if ((l & 1) == 0) h = mix64(key[l >> 1] ^ k);
            uint64_t r = (l & 1) ? (h >> 32) : (h & 0xffffffffull);
            uint64_t bu = (r >= tab), bv = (r >= ta && r < tab) || (r >= tabc);
            u = (u << 1) | bu;
            v = (v << 1) | bv;
        }
        if (permute) {
            u = permute_bits(u, scale, &pk);
            v = permute_bits(v, scale, &pk);
        }
        src[i] = (uint32_t)u;
        dst[i] = (uint32_t)v;
    }
}

/* Erdos-Renyi G(n, m) with replacement: tuples [k0, k0+count). */
void pgabb_gen_er(uint64_t n, uint64_t seed, uint64_t k0, uint64_t count,
                  uint32_t* src, uint32_t* dst) {
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)count; ++i) {
        const uint64_t h = draw(seed, 0xE5, k0 + (uint64_t)i);
        src[i] = (uint32_t)(((h & 0xffffffffull) * n) >> 32);
        dst[i] = (uint32_t)(((h >> 32) * n) >> 32);
    }
}

/* Grid cell (r, c), 0 <= r, c < side-1, carries a diagonal iff this holds. */
static inline int grid_has_diag(uint64_t side, uint64_t seed, double f, uint64_t cell) {
    (void)side;
    if (f >= 1.0) return 1;
    const uint64_t thr = (uint64_t)(f * 18446744073709551616.0);
    return draw(seed, 0xD1A6, cell) < thr;
}

/* Number of diagonal cells for (side, f, seed). */
uint64_t pgabb_gen_grid_ndiag(uint64_t side, double f, uint64_t seed) {
    if (side < 2 || f <= 0.0) return 0;
    uint64_t cnt = 0;
    const uint64_t cells = (side - 1) * (side - 1);
    #pragma omp parallel for schedule(static) reduction(+:cnt)
    for (int64_t cell = 0; cell < (int64_t)cells; ++cell)
        cnt += (uint64_t)grid_has_diag(side, seed, f, (uint64_t)cell);
    return cnt;
}

/* Grid: horizontal edges, then vertical edges, then diagonals in cell order.
 * src/dst must hold 2*side*(side-1) + ndiag tuples.  Vertex id = r*side + c. */
void pgabb_gen_grid(uint64_t side, double f, uint64_t seed, uint32_t* src, uint32_t* dst) {
    if (side == 0) return;
    const uint64_t h = side * (side - 1);
    #pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < (int64_t)h; ++e) {
        uint64_t r = (uint64_t)e / (side - 1), c = (uint64_t)e % (side - 1);
        src[e] = (uint32_t)(r * side + c);
        dst[e] = (uint32_t)(r * side + c + 1);
        uint64_t r2 = (uint64_t)e / side, c2 = (uint64_t)e % side;   /* vertical */
        src[h + e] = (uint32_t)(r2 * side + c2);
        dst[h + e] = (uint32_t)((r2 + 1) * side + c2);
    }
    if (side < 2 || f <= 0.0) return;
    uint64_t pos = 2 * h;
    const uint64_t cells = (side - 1) * (side - 1);
    for (uint64_t cell = 0; cell < cells; ++cell) {
        if (!grid_has_diag(side, seed, f, cell)) continue;
        uint64_t r = cell / (side - 1), c = cell % (side - 1);
        src[pos] = (uint32_t)(r * side + c);
        dst[pos] = (uint32_t)((r + 1) * side + c + 1);
        ++pos;
    }
}
