/* oracle/oracle.c — fp64 CPU oracle of the CRK-HACC short-range solver.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or helper with the CUDA path (paper_2310_16122_b200/csrc), and the
 * product path never calls it.
 *
 * What it computes is the plain definition of each step, in the order of
 * SURVEY.md §8(c) O1-O9 (the readings of arxiv 2310.16122, which names the five
 * hot kernels at PAPER.md:377 — Geometry, Corrections, Extras, Acceleration,
 * Energy — and short-range gravity with a degree-5 grid polynomial at
 * PAPER.md:147, 278, 646, but prints none of their formulas; DESIGN.md §2 lists
 * every reading).  All arithmetic is fp64 from the fp32 inputs, except the
 * membership predicate, which is specified in fp32 (O2) so that lists and counts
 * can be compared bit-exactly.
 *
 * Neighbour search: brute force over all particles, or (same result, checked by
 * tests/test_oracle_pins.py::test_grid_equals_brute) a uniform grid whose cells
 * are at least the cutoff wide.  Either way the neighbours of a target are sorted
 * by index before any sum, so the two modes agree bit for bit.
 *
 * Build: gcc -O2 -fopenmp -ffp-contract=off -fPIC -shared (see __graft_entry__.build).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

typedef struct {
    double box[3];
    float rcut2, eps2, poly[6], G, gamma, av_cl, av_cq, av_eps2;
    int32_t leaf_max_i, leaf_max_j, leaf_max_gas_i, leaf_max_gas_j;
    double cell_side;
} orc_params;

/* ------------------------------------------------------------------ O1 / O2 */

/* Minimum-image separation component d = x_j - x_i (exact: both are multiples of
 * q = L_max 2^-23, O1). */
static double min_image(double xj, double xi, double L) {
    double d = xj - xi;
    if (d > 0.5 * L) d -= L;
    else if (d < -0.5 * L) d += L;
    return d;
}

/* O2: s32 = fmaf(dz,dz, fmaf(dy,dy, dx*dx)), each op rounded to nearest even. */
static float s32_of(double dx, double dy, double dz) {
    float fx = (float)dx, fy = (float)dy, fz = (float)dz; /* exact conversions */
    float t = fx * fx;
    t = fmaf(fy, fy, t);
    t = fmaf(fz, fz, t);
    return t;
}

static float h2_of(float H) { return H * H; } /* fl32(H*H) */

/* ------------------------------------------------------------------ O3: order */

static uint64_t spread3(uint64_t v, int bits) {
    uint64_t r = 0;
    for (int b = 0; b < bits; ++b) r |= ((v >> b) & 1ull) << (3 * b);
    return r;
}

static int ilog2_exact(double v) { /* v must be a power of two */
    int e;
    double m = frexp(v, &e);
    return (m == 0.5) ? e - 1 : -1000;
}

typedef struct {
    double q;
    int cs;     /* log2(cell_side / q) */
    int cbits;  /* bits per axis of the cell index */
    int fbits;  /* bits per axis of the in-cell (fine) coordinate */
    int ncell[3];
} key_layout;

static int layout_of(const orc_params* p, key_layout* k) {
    double L = p->box[0];
    if (p->box[1] > L) L = p->box[1];
    if (p->box[2] > L) L = p->box[2];
    k->q = ldexp(L, -23);
    k->cs = ilog2_exact(p->cell_side / k->q);
    if (k->cs < 0) return -1;
    int maxn = 1;
    for (int a = 0; a < 3; ++a) {
        k->ncell[a] = (int)llround(p->box[a] / p->cell_side);
        if (k->ncell[a] > maxn) maxn = k->ncell[a];
    }
    k->cbits = 0;
    while ((1 << k->cbits) < maxn) ++k->cbits;
    k->fbits = (32 - 3 * k->cbits) / 3; /* the key fits 32 bits */
    if (k->fbits > k->cs) k->fbits = k->cs;
    return 0;
}

/* Sort key of O3: (Morton(cell), Morton(top fbits of the in-cell coordinate)),
 * ties broken by id.  x -> bit 3b, y -> 3b+1, z -> 3b+2. */
static void key_of(const key_layout* k, float x, float y, float z, uint64_t* key, int64_t cell[3]) {
    uint64_t xi[3] = {(uint64_t)((double)x / k->q), (uint64_t)((double)y / k->q),
                      (uint64_t)((double)z / k->q)};
    uint64_t c[3], f[3];
    for (int a = 0; a < 3; ++a) {
        c[a] = xi[a] >> k->cs;
        f[a] = (xi[a] & ((1ull << k->cs) - 1)) >> (k->cs - k->fbits);
        if (cell) cell[a] = (int64_t)c[a];
    }
    uint64_t cm = spread3(c[0], k->cbits) | (spread3(c[1], k->cbits) << 1) | (spread3(c[2], k->cbits) << 2);
    uint64_t fm = spread3(f[0], k->fbits) | (spread3(f[1], k->fbits) << 1) | (spread3(f[2], k->fbits) << 2);
    *key = (cm << (3 * k->fbits)) | fm;
}

typedef struct { uint64_t key; int64_t id; int64_t idx; } sort_rec;

static int cmp_rec(const void* a, const void* b) {
    const sort_rec* u = (const sort_rec*)a;
    const sort_rec* v = (const sort_rec*)b;
    if (u->key != v->key) return u->key < v->key ? -1 : 1;
    if (u->id != v->id) return u->id < v->id ? -1 : 1;
    return 0;
}

/* order[k] = input index of the particle at sorted position k; key_out[k] its key
 * (may be NULL); cellm_out[k] = Morton code of its cell (may be NULL). */
int orc_sort(int64_t n, const float* x, const float* y, const float* z, const int64_t* id,
             const orc_params* p, int64_t* order, uint64_t* key_out, uint64_t* cellm_out) {
    key_layout k;
    if (layout_of(p, &k)) return -1;
    sort_rec* r = (sort_rec*)malloc(sizeof(sort_rec) * (size_t)(n > 0 ? n : 1));
    for (int64_t i = 0; i < n; ++i) {
        key_of(&k, x[i], y[i], z[i], &r[i].key, NULL);
        r[i].id = id[i];
        r[i].idx = i;
    }
    qsort(r, (size_t)n, sizeof(sort_rec), cmp_rec);
    for (int64_t i = 0; i < n; ++i) {
        order[i] = r[i].idx;
        if (key_out) key_out[i] = r[i].key;
        if (cellm_out) cellm_out[i] = r[i].key >> (3 * k.fbits);
    }
    free(r);
    return 0;
}

/* ------------------------------------------------------------------ O3: leaves
 * kind 0: gravity i-leaves (chunks of leaf_max_i of each cell run, all species)
 * kind 1: gravity j-leaves (chunks of leaf_max_j)
 * kind 2: gas i-leaves (chunks of leaf_max_gas_i of the gas subsequence of each run)
 * kind 3: gas j-leaves (chunks of leaf_max_gas_j)
 * A run of c members is split into nch = ceil(c/leaf_max) chunks, chunk t covering
 * members [floor(t c/nch), floor((t+1) c/nch)).  first[] indexes the member
 * sequence: sorted positions (kinds 0,1) or gas ranks in sorted order (kinds 2,3).
 * bbox = per-axis min/max of member positions; maxh2 = max fl32(H^2) (gas kinds).
 * Called with first == NULL it only returns the number of leaves. */
int64_t orc_leaves(int64_t n, const int64_t* order, const uint64_t* cellm, const float* x,
                   const float* y, const float* z, const uint8_t* species, const float* H,
                   const orc_params* p, int kind, int64_t* first, int32_t* count, float* bbox,
                   float* maxh2, uint64_t* leaf_cell) {
    int gas = (kind >= 2);
    int lmax = kind == 0 ? p->leaf_max_i : kind == 1 ? p->leaf_max_j
             : kind == 2 ? p->leaf_max_gas_i : p->leaf_max_gas_j;
    /* member sequence */
    int64_t* mem = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    uint64_t* mcell = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(n > 0 ? n : 1));
    int64_t nm = 0;
    for (int64_t s = 0; s < n; ++s) {
        int64_t i = order[s];
        if (gas && species[i] != 1) continue;
        mem[nm] = i;
        mcell[nm] = cellm[s];
        ++nm;
    }
    int64_t nl = 0;
    int64_t a = 0;
    while (a < nm) {
        int64_t b = a;
        while (b < nm && mcell[b] == mcell[a]) ++b;
        int64_t c = b - a;
        int64_t nch = (c + lmax - 1) / lmax;
        for (int64_t t = 0; t < nch; ++t) {
            int64_t lo = a + (t * c) / nch, hi = a + ((t + 1) * c) / nch;
            if (first) {
                first[nl] = lo;
                count[nl] = (int32_t)(hi - lo);
                float mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
                float mh = 0.f;
                for (int64_t u = lo; u < hi; ++u) {
                    int64_t i = mem[u];
                    float v[3] = {x[i], y[i], z[i]};
                    for (int d = 0; d < 3; ++d) {
                        if (v[d] < mn[d]) mn[d] = v[d];
                        if (v[d] > mx[d]) mx[d] = v[d];
                    }
                    if (gas) { float h2 = h2_of(H[i]); if (h2 > mh) mh = h2; }
                }
                for (int d = 0; d < 3; ++d) { bbox[6 * nl + d] = mn[d]; bbox[6 * nl + 3 + d] = mx[d]; }
                if (maxh2) maxh2[nl] = mh;
                if (leaf_cell) leaf_cell[nl] = mcell[a];
            }
            ++nl;
        }
        a = b;
    }
    free(mem);
    free(mcell);
    return nl;
}

/* ------------------------------------------------------------------ O4: lists
 * Leaf-pair test: per axis, gap_s = max(0, lo_b + sL - hi_a, lo_a - hi_b - sL) for
 * s in {0,-1,+1} (first minimum wins), d2 = sum gap^2 (exact in fp64), pair kept iff
 * d2 < (double)cut2 (1 + 2^-20).  mode 0: cut2 = rcut2; mode 1: cut2 = max(maxh2_a,
 * maxh2_b).  Rows are produced for the requested i-leaves, entries ordered by b.
 * shift code = (sx+1) + 3(sy+1) + 9(sz+1).  With col == NULL only row_len is filled. */
static int leaf_pair(const float* ba, const float* bb, const double* L, double cut2, int* code) {
    double d2 = 0.0;
    int sc[3];
    for (int d = 0; d < 3; ++d) {
        double best = INFINITY;
        int bs = 0;
        const int ss[3] = {0, -1, 1};
        for (int t = 0; t < 3; ++t) {
            double s = ss[t] * L[d];
            double g1 = (double)bb[d] + s - (double)ba[3 + d];
            double g2 = (double)ba[d] - (double)bb[3 + d] - s;
            double g = 0.0;
            if (g1 > g) g = g1;
            if (g2 > g) g = g2;
            if (g < best) { best = g; bs = ss[t]; }
        }
        sc[d] = bs;
        d2 += best * best;
    }
    *code = (sc[0] + 1) + 3 * (sc[1] + 1) + 9 * (sc[2] + 1);
    return d2 < cut2 * (1.0 + ldexp(1.0, -20));
}

void orc_list_rows(int64_t nrows, const int64_t* rows, const float* bbox_a, const float* maxh2_a,
                   int64_t nb, const float* bbox_b, const float* maxh2_b, const orc_params* p,
                   int mode, int64_t* row_len, const int64_t* row_off, int32_t* col, int8_t* shift) {
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t r = 0; r < nrows; ++r) {
        int64_t a = rows[r];
        int64_t cnt = 0;
        for (int64_t b = 0; b < nb; ++b) {
            double cut2 = mode == 0 ? (double)p->rcut2
                                    : (double)(maxh2_a[a] > maxh2_b[b] ? maxh2_a[a] : maxh2_b[b]);
            int code;
            if (leaf_pair(bbox_a + 6 * a, bbox_b + 6 * b, p->box, cut2, &code)) {
                if (col) {
                    col[row_off[r] + cnt] = (int32_t)b;
                    shift[row_off[r] + cnt] = (int8_t)code;
                }
                ++cnt;
            }
        }
        if (!col) row_len[r] = cnt;
    }
}

/* ------------------------------------------------------------------ neighbour search */

typedef struct {
    int brute;
    int nc[3];
    double cw[3];
    int64_t nmem;
    const int64_t* mem;   /* member particle indices (all, or gas only) */
    int64_t* start;       /* cell start offsets into sidx, size ncells+1 */
    int64_t* sidx;        /* member indices grouped by cell */
} grid_t;

static void grid_build(grid_t* g, const float* x, const float* y, const float* z, int64_t nmem,
                       const int64_t* mem, const double* box, double rmax, int force_brute) {
    g->nmem = nmem;
    g->mem = mem;
    g->brute = force_brute;
    for (int a = 0; a < 3; ++a) {
        g->nc[a] = (int)floor(box[a] / rmax);
        if (g->nc[a] < 3) g->brute = 1;
        if (g->nc[a] > 256) g->nc[a] = 256;
        g->cw[a] = box[a] / (g->nc[a] > 0 ? g->nc[a] : 1);
    }
    g->start = NULL;
    g->sidx = NULL;
    if (g->brute) return;
    int64_t nc = (int64_t)g->nc[0] * g->nc[1] * g->nc[2];
    g->start = (int64_t*)calloc((size_t)nc + 1, sizeof(int64_t));
    g->sidx = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nmem > 0 ? nmem : 1));
    int64_t* cellof = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nmem > 0 ? nmem : 1));
    for (int64_t u = 0; u < nmem; ++u) {
        int64_t i = mem[u];
        double v[3] = {x[i], y[i], z[i]};
        int64_t c[3];
        for (int a = 0; a < 3; ++a) {
            c[a] = (int64_t)floor(v[a] / g->cw[a]);
            if (c[a] < 0) c[a] = 0;
            if (c[a] >= g->nc[a]) c[a] = g->nc[a] - 1;
        }
        cellof[u] = c[0] + (int64_t)g->nc[0] * (c[1] + (int64_t)g->nc[1] * c[2]);
        g->start[cellof[u] + 1]++;
    }
    for (int64_t c = 0; c < nc; ++c) g->start[c + 1] += g->start[c];
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)nc);
    memcpy(fill, g->start, sizeof(int64_t) * (size_t)nc);
    for (int64_t u = 0; u < nmem; ++u) g->sidx[fill[cellof[u]]++] = mem[u];
    free(fill);
    free(cellof);
}

static void grid_free(grid_t* g) { free(g->start); free(g->sidx); }

static int cmp_i64(const void* a, const void* b) {
    int64_t u = *(const int64_t*)a, v = *(const int64_t*)b;
    return (u > v) - (u < v);
}

enum { PRED_GRAV = 0, PRED_GATHER = 1, PRED_SYM = 2, PRED_GATHER_SELF = 3 };

typedef struct {
    const float *x, *y, *z, *H;
    const double* box;
    float rcut2;
} pctx;

/* Does j belong to i's neighbourhood under predicate `pred` (O2)? */
static int pred_ok(const pctx* c, int pred, int64_t i, int64_t j) {
    if (j == i) return pred == PRED_GATHER_SELF;
    double dx = min_image(c->x[j], c->x[i], c->box[0]);
    double dy = min_image(c->y[j], c->y[i], c->box[1]);
    double dz = min_image(c->z[j], c->z[i], c->box[2]);
    float s = s32_of(dx, dy, dz);
    switch (pred) {
    case PRED_GRAV: return s < c->rcut2;
    case PRED_GATHER:
    case PRED_GATHER_SELF: return s < h2_of(c->H[i]);
    default: {
        float hi = h2_of(c->H[i]), hj = h2_of(c->H[j]);
        return s < (hi > hj ? hi : hj);
    }
    }
}

typedef struct { int64_t* v; int64_t n, cap; } ivec;

static void ivec_push(ivec* a, int64_t x) {
    if (a->n == a->cap) {
        a->cap = a->cap ? 2 * a->cap : 256;
        a->v = (int64_t*)realloc(a->v, sizeof(int64_t) * (size_t)a->cap);
    }
    a->v[a->n++] = x;
}

/* Neighbours of i, sorted ascending by index. */
static void neighbours(const grid_t* g, const pctx* c, int pred, int64_t i, ivec* out) {
    out->n = 0;
    if (g->brute) {
        for (int64_t u = 0; u < g->nmem; ++u)
            if (pred_ok(c, pred, i, g->mem[u])) ivec_push(out, g->mem[u]);
    } else {
        double v[3] = {c->x[i], c->y[i], c->z[i]};
        int64_t ci[3];
        for (int a = 0; a < 3; ++a) {
            ci[a] = (int64_t)floor(v[a] / g->cw[a]);
            if (ci[a] < 0) ci[a] = 0;
            if (ci[a] >= g->nc[a]) ci[a] = g->nc[a] - 1;
        }
        for (int dz = -1; dz <= 1; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    int64_t cx = (ci[0] + dx + g->nc[0]) % g->nc[0];
                    int64_t cy = (ci[1] + dy + g->nc[1]) % g->nc[1];
                    int64_t cz = (ci[2] + dz + g->nc[2]) % g->nc[2];
                    int64_t cell = cx + (int64_t)g->nc[0] * (cy + (int64_t)g->nc[1] * cz);
                    for (int64_t u = g->start[cell]; u < g->start[cell + 1]; ++u)
                        if (pred_ok(c, pred, i, g->sidx[u])) ivec_push(out, g->sidx[u]);
                }
        qsort(out->v, (size_t)out->n, sizeof(int64_t), cmp_i64);
    }
}

static int64_t* gas_members(int64_t n, const uint8_t* species, int64_t* ng) {
    int64_t* m = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    int64_t k = 0;
    for (int64_t i = 0; i < n; ++i)
        if (species[i] == 1) m[k++] = i;
    *ng = k;
    return m;
}

static int64_t* all_members(int64_t n) {
    int64_t* m = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    for (int64_t i = 0; i < n; ++i) m[i] = i;
    return m;
}

static float max_h2(int64_t ng, const int64_t* mem, const float* H) {
    float mh = 0.f;
    for (int64_t u = 0; u < ng; ++u) { float h = h2_of(H[mem[u]]); if (h > mh) mh = h; }
    return mh;
}

/* ------------------------------------------------------------------ counts (O2)
 * count_grav[t]   = #{j != i : s32 < rcut2}           (all species)
 * count_gather[t] = #{gas j != i : s32 < H2_i}         (gas i; 0 for DM)
 * count_sym[t]    = #{gas j != i : s32 < max(H2_i,H2_j)} (gas i; 0 for DM)   */
int orc_counts(int64_t n, const float* x, const float* y, const float* z, const uint8_t* species,
               const float* H, const orc_params* p, int64_t nt, const int64_t* targets,
               int32_t* cgrav, int32_t* cgath, int32_t* csym, int force_brute) {
    int64_t ng;
    int64_t* gm = gas_members(n, species, &ng);
    int64_t* am = all_members(n);
    grid_t ga, gg;
    grid_build(&ga, x, y, z, n, am, p->box, sqrt((double)p->rcut2) * 1.0001, force_brute);
    grid_build(&gg, x, y, z, ng, gm, p->box, sqrt((double)max_h2(ng, gm, H)) * 1.0001, force_brute);
    pctx c = {x, y, z, H, p->box, p->rcut2};
#pragma omp parallel
    {
        ivec nb = {0, 0, 0};
#pragma omp for schedule(dynamic, 16)
        for (int64_t t = 0; t < nt; ++t) {
            int64_t i = targets[t];
            neighbours(&ga, &c, PRED_GRAV, i, &nb);
            cgrav[t] = (int32_t)nb.n;
            if (species[i] == 1) {
                neighbours(&gg, &c, PRED_GATHER, i, &nb);
                cgath[t] = (int32_t)nb.n;
                neighbours(&gg, &c, PRED_SYM, i, &nb);
                csym[t] = (int32_t)nb.n;
            } else {
                cgath[t] = 0;
                csym[t] = 0;
            }
        }
        free(nb.v);
    }
    grid_free(&ga);
    grid_free(&gg);
    free(gm);
    free(am);
    return 0;
}

/* ------------------------------------------------------------------ O5: gravity
 * a_i = G sum_{j != i, s32 < rcut2} m_j x_ji [ (s + eps2)^-3/2 - sum_k c_k s^k ],
 * x_ji = x_j - x_i (minimum image), s = |x_ji|^2 in exact fp64.  All species.
 * S_i = sum_j |a_ij| + 1e-2 sum_j G m_j |x_ji| ((s + eps2)^-3/2 + |P5(s)|): the
 * parity-error normaliser of SURVEY.md §8(c) (sum of |pair terms|) plus a 1% floor of the
 * two terms' magnitudes, because the pair term is a difference that the continuity
 * constraint drives to zero at the cutoff, where fp32 cannot resolve it below the ulp of
 * its terms (a lone pair at r_c) — DESIGN.md §6.
 * Kick: v_i += dt a_i (v_out; pass dt = 0 for forces only). */
int orc_gravity(int64_t n, const float* x, const float* y, const float* z, const float* m,
                const float* vx, const float* vy, const float* vz, const orc_params* p,
                double dt, int64_t nt, const int64_t* targets, double* acc /* 3 nt */,
                double* S, double* vout /* 3 nt */, int force_brute) {
    int64_t* am = all_members(n);
    grid_t ga;
    grid_build(&ga, x, y, z, n, am, p->box, sqrt((double)p->rcut2) * 1.0001, force_brute);
    pctx c = {x, y, z, NULL, p->box, p->rcut2};
#pragma omp parallel
    {
        ivec nb = {0, 0, 0};
#pragma omp for schedule(dynamic, 16)
        for (int64_t t = 0; t < nt; ++t) {
            int64_t i = targets[t];
            neighbours(&ga, &c, PRED_GRAV, i, &nb);
            double a[3] = {0, 0, 0}, s_abs = 0.0;
            for (int64_t u = 0; u < nb.n; ++u) {
                int64_t j = nb.v[u];
                double d[3] = {min_image(x[j], x[i], p->box[0]), min_image(y[j], y[i], p->box[1]),
                               min_image(z[j], z[i], p->box[2])};
                double s = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
                double poly = 0.0, sk = 1.0;
                for (int k = 0; k <= 5; ++k) { poly += (double)p->poly[k] * sk; sk *= s; }
                double newton = pow(s + (double)p->eps2, -1.5);
                double f = newton - poly;
                double w = (double)p->G * (double)m[j] * f;
                for (int q = 0; q < 3; ++q) a[q] += w * d[q];
                /* error scale: |pair term| plus a 1% floor of the magnitudes of the two terms
                 * of the difference (fp32 cancellation near the cutoff) */
                s_abs += fabs((double)p->G * (double)m[j]) * (fabs(f) + 1e-2 * (newton + fabs(poly))) * sqrt(s);
            }
            for (int q = 0; q < 3; ++q) acc[3 * t + q] = a[q];
            S[t] = s_abs;
            vout[3 * t + 0] = (double)vx[i] + dt * a[0];
            vout[3 * t + 1] = (double)vy[i] + dt * a[1];
            vout[3 * t + 2] = (double)vz[i] + dt * a[2];
        }
        free(nb.v);
    }
    grid_free(&ga);
    free(am);
    return 0;
}

/* ------------------------------------------------------------------ O6: kernel
 * Wendland C4 in 3-D, compact support H:
 *   W(r,H) = sigma/H^3 (1-q)^6 (1 + 6q + 35q^2/3), q = r/H < 1, sigma = 495/(32 pi)
 *   grad_i W = -(56/3) sigma/H^5 (1-q)^5 (1+5q) x_ij        (x_ij = x_i - x_j) */
static const double ORC_PI = 3.14159265358979323846;

static double wendland(double r, double H) {
    double q = r / H;
    if (q >= 1.0) return 0.0;
    double sigma = 495.0 / (32.0 * ORC_PI);
    double t = 1.0 - q;
    return sigma / (H * H * H) * pow(t, 6) * (1.0 + 6.0 * q + 35.0 * q * q / 3.0);
}

/* grad W / x_ij, i.e. the scalar g with grad_i W_ij = g x_ij */
static double wendland_g(double r, double H) {
    double q = r / H;
    if (q >= 1.0) return 0.0;
    double sigma = 495.0 / (32.0 * ORC_PI);
    double t = 1.0 - q;
    return -(56.0 / 3.0) * sigma / pow(H, 5) * pow(t, 5) * (1.0 + 5.0 * q);
}

void orc_kernel(double r, double H, double* W, double* g) {
    *W = wendland(r, H);
    *g = wendland_g(r, H);
}

/* x_ij = x_i - x_j (minimum image) */
static void sep_ij(const float* x, const float* y, const float* z, const double* box, int64_t i,
                   int64_t j, double* d) {
    d[0] = -min_image(x[j], x[i], box[0]);
    d[1] = -min_image(y[j], y[i], box[1]);
    d[2] = -min_image(z[j], z[i], box[2]);
}

/* Geometry: V_i = 1 / sum_{gas j, s32 < H2_i, j including i} W(r_ij, H_i). */
int orc_geometry(int64_t n, const float* x, const float* y, const float* z, const uint8_t* species,
                 const float* H, const orc_params* p, int64_t nt, const int64_t* targets,
                 double* V, int force_brute) {
    int64_t ng;
    int64_t* gm = gas_members(n, species, &ng);
    grid_t gg;
    grid_build(&gg, x, y, z, ng, gm, p->box, sqrt((double)max_h2(ng, gm, H)) * 1.0001, force_brute);
    pctx c = {x, y, z, H, p->box, p->rcut2};
#pragma omp parallel
    {
        ivec nb = {0, 0, 0};
#pragma omp for schedule(dynamic, 16)
        for (int64_t t = 0; t < nt; ++t) {
            int64_t i = targets[t];
            neighbours(&gg, &c, PRED_GATHER_SELF, i, &nb);
            double sum = 0.0;
            for (int64_t u = 0; u < nb.n; ++u) {
                double d[3];
                sep_ij(x, y, z, p->box, i, nb.v[u], d);
                sum += wendland(sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]), H[i]);
            }
            V[t] = 1.0 / sum;
        }
        free(nb.v);
    }
    grid_free(&gg);
    free(gm);
    return 0;
}

/* ------------------------------------------------------------------ O7: corrections */

static double det3(const double m[3][3]) {
    return m[0][0] * (m[1][1] * m[2][2] - m[1][2] * m[2][1]) -
           m[0][1] * (m[1][0] * m[2][2] - m[1][2] * m[2][0]) +
           m[0][2] * (m[1][0] * m[2][1] - m[1][1] * m[2][0]);
}

static void inv3(const double m[3][3], double r[3][3]) {
    double d = det3(m);
    r[0][0] = (m[1][1] * m[2][2] - m[1][2] * m[2][1]) / d;
    r[0][1] = (m[0][2] * m[2][1] - m[0][1] * m[2][2]) / d;
    r[0][2] = (m[0][1] * m[1][2] - m[0][2] * m[1][1]) / d;
    r[1][0] = (m[1][2] * m[2][0] - m[1][0] * m[2][2]) / d;
    r[1][1] = (m[0][0] * m[2][2] - m[0][2] * m[2][0]) / d;
    r[1][2] = (m[0][2] * m[1][0] - m[0][0] * m[1][2]) / d;
    r[2][0] = (m[1][0] * m[2][1] - m[1][1] * m[2][0]) / d;
    r[2][1] = (m[0][1] * m[2][0] - m[0][0] * m[2][1]) / d;
    r[2][2] = (m[0][0] * m[1][1] - m[0][1] * m[1][0]) / d;
}

/* Outputs per target t: A[t], B[3t+a], dA[3t+g] = d_g A, dB[9t + 3a + g] = d_g B^a.
 * Sums over gas j with s32 < H2_i, j including i (self term: V_i W(0,H_i) in m0 only).
 * V is indexed by particle (length n). */
int orc_corrections(int64_t n, const float* x, const float* y, const float* z,
                    const uint8_t* species, const float* H, const double* V, const orc_params* p,
                    int64_t nt, const int64_t* targets, double* A, double* B, double* dA, double* dB,
                    int force_brute) {
    int64_t ng;
    int64_t* gm = gas_members(n, species, &ng);
    grid_t gg;
    grid_build(&gg, x, y, z, ng, gm, p->box, sqrt((double)max_h2(ng, gm, H)) * 1.0001, force_brute);
    pctx c = {x, y, z, H, p->box, p->rcut2};
#pragma omp parallel
    {
        ivec nb = {0, 0, 0};
#pragma omp for schedule(dynamic, 16)
        for (int64_t t = 0; t < nt; ++t) {
            int64_t i = targets[t];
            neighbours(&gg, &c, PRED_GATHER_SELF, i, &nb);
            double m0 = 0, m1[3] = {0}, m2[3][3] = {{0}};
            double dm0[3] = {0}, dm1[3][3] = {{0}} /* [a][g] */, dm2[3][3][3] = {{{0}}} /* [a][b][g] */;
            for (int64_t u = 0; u < nb.n; ++u) {
                int64_t j = nb.v[u];
                double d[3];
                sep_ij(x, y, z, p->box, i, j, d);
                double r = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
                double W = wendland(r, H[i]);
                double g = wendland_g(r, H[i]);
                double Vj = V[j];
                double dW[3] = {g * d[0], g * d[1], g * d[2]};
                m0 += Vj * W;
                for (int a = 0; a < 3; ++a) {
                    m1[a] += Vj * d[a] * W;
                    dm0[a] += Vj * dW[a];
                    for (int b = 0; b < 3; ++b) {
                        m2[a][b] += Vj * d[a] * d[b] * W;
                        dm1[a][b] += Vj * d[a] * dW[b];
                        for (int gg2 = 0; gg2 < 3; ++gg2) dm2[a][b][gg2] += Vj * d[a] * d[b] * dW[gg2];
                    }
                }
            }
            /* delta terms: d_g m1^a += delta_ag m0; d_g m2^ab += delta_ag m1^b + delta_bg m1^a */
            for (int a = 0; a < 3; ++a) {
                dm1[a][a] += m0;
                for (int b = 0; b < 3; ++b) {
                    dm2[a][b][a] += m1[b];
                    dm2[a][b][b] += m1[a];
                }
            }
            double Ai, Bi[3], dAi[3], dBi[3][3] /* [a][g] */;
            double tr = (m2[0][0] + m2[1][1] + m2[2][2]) / 3.0;
            double det = det3(m2);
            if (fabs(det) < 1e-10 * tr * tr * tr) { /* degenerate guard (O7 reading) */
                Ai = 1.0 / m0;
                for (int a = 0; a < 3; ++a) {
                    Bi[a] = 0.0;
                    dAi[a] = -dm0[a] / (m0 * m0);
                    for (int g = 0; g < 3; ++g) dBi[a][g] = 0.0;
                }
            } else {
                double mi[3][3];
                inv3(m2, mi);
                for (int a = 0; a < 3; ++a) {
                    Bi[a] = 0.0;
                    for (int b = 0; b < 3; ++b) Bi[a] -= mi[a][b] * m1[b];
                }
                double bm1 = Bi[0] * m1[0] + Bi[1] * m1[1] + Bi[2] * m1[2];
                Ai = 1.0 / (m0 + bm1);
                for (int g = 0; g < 3; ++g) {
                    /* d_g B = -m2^-1 (d_g m1 + (d_g m2) B) */
                    double rhs[3];
                    for (int a = 0; a < 3; ++a) {
                        rhs[a] = dm1[a][g];
                        for (int b = 0; b < 3; ++b) rhs[a] += dm2[a][b][g] * Bi[b];
                    }
                    for (int a = 0; a < 3; ++a) {
                        dBi[a][g] = 0.0;
                        for (int b = 0; b < 3; ++b) dBi[a][g] -= mi[a][b] * rhs[b];
                    }
                }
                for (int g = 0; g < 3; ++g) {
                    /* d_g A = -A^2 (d_g m0 + d_g B . m1 + B . d_g m1) */
                    double s = dm0[g];
                    for (int a = 0; a < 3; ++a) s += dBi[a][g] * m1[a] + Bi[a] * dm1[a][g];
                    dAi[g] = -Ai * Ai * s;
                }
            }
            A[t] = Ai;
            for (int a = 0; a < 3; ++a) {
                B[3 * t + a] = Bi[a];
                dA[3 * t + a] = dAi[a];
                for (int g = 0; g < 3; ++g) dB[9 * t + 3 * a + g] = dBi[a][g];
            }
        }
        free(nb.v);
    }
    grid_free(&gg);
    free(gm);
    return 0;
}

/* Corrected kernel of particle i (coefficients A, B[3], dA[3], dB[9] = d_g B^a at 3a+g)
 * at separation d = x_i - x_j with support H:
 *   W^R = A (1 + B.d) W
 *   d_g W^R = d_gA (1+B.d) W + A (d_gB . d + B^g) W + A (1 + B.d) d_g W          (O7) */
static void corrected(double A, const double* B, const double* dA, const double* dB, const double* d,
                      double H, double* WR, double* gWR) {
    double r = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    double W = wendland(r, H), g = wendland_g(r, H);
    double lin = 1.0 + B[0] * d[0] + B[1] * d[1] + B[2] * d[2];
    *WR = A * lin * W;
    if (gWR)
        for (int gg = 0; gg < 3; ++gg) {
            double dBd = dB[0 * 3 + gg] * d[0] + dB[1 * 3 + gg] * d[1] + dB[2 * 3 + gg] * d[2];
            gWR[gg] = dA[gg] * lin * W + A * (dBd + B[gg]) * W + A * lin * g * d[gg];
        }
}

/* Expose W^R / grad W^R for the reproduction pins of tests/. */
void orc_corrected_kernel(double A, const double* B, const double* dA, const double* dB,
                          const double* d, double H, double* WR, double* gWR) {
    corrected(A, B, dA, dB, d, H, WR, gWR);
}

/* ------------------------------------------------------------------ O8: extras
 * rho_i = sum_{gas j, s32 < H2_i, incl. i} m_j W^R_ij ; P_i = (gamma-1) rho_i u_i ;
 * c_i = sqrt(gamma P_i / rho_i) ; d_b v^a_i = sum_j V_j (v^a_j - v^a_i) d_b W^R_ij
 * (dv[9t + 3a + b]).  Coefficient arrays are indexed by particle. */
int orc_extras(int64_t n, const float* x, const float* y, const float* z, const uint8_t* species,
               const float* H, const float* m, const float* vx, const float* vy, const float* vz,
               const float* u, const double* V, const double* A, const double* B, const double* dA,
               const double* dB, const orc_params* p, int64_t nt, const int64_t* targets,
               double* rho, double* P, double* cs, double* dv, int force_brute) {
    int64_t ng;
    int64_t* gm = gas_members(n, species, &ng);
    grid_t gg;
    grid_build(&gg, x, y, z, ng, gm, p->box, sqrt((double)max_h2(ng, gm, H)) * 1.0001, force_brute);
    pctx c = {x, y, z, H, p->box, p->rcut2};
    const double gam = (double)p->gamma;
#pragma omp parallel
    {
        ivec nb = {0, 0, 0};
#pragma omp for schedule(dynamic, 16)
        for (int64_t t = 0; t < nt; ++t) {
            int64_t i = targets[t];
            neighbours(&gg, &c, PRED_GATHER_SELF, i, &nb);
            double r_ = 0.0, g9[9] = {0};
            const float* vv[3] = {vx, vy, vz};
            for (int64_t u2 = 0; u2 < nb.n; ++u2) {
                int64_t j = nb.v[u2];
                double d[3], WR, gWR[3];
                sep_ij(x, y, z, p->box, i, j, d);
                corrected(A[i], B + 3 * i, dA + 3 * i, dB + 9 * i, d, H[i], &WR, gWR);
                r_ += (double)m[j] * WR;
                for (int a = 0; a < 3; ++a)
                    for (int b = 0; b < 3; ++b)
                        g9[3 * a + b] += V[j] * ((double)vv[a][j] - (double)vv[a][i]) * gWR[b];
            }
            rho[t] = r_;
            P[t] = (gam - 1.0) * r_ * (double)u[i];
            cs[t] = sqrt(gam * P[t] / r_);
            for (int k = 0; k < 9; ++k) dv[9 * t + k] = g9[k];
        }
        free(nb.v);
    }
    grid_free(&gg);
    free(gm);
    return 0;
}

/* ------------------------------------------------------------------ O9: accel + energy
 * Sums over gas j != i with s32 < max(H2_i, H2_j):
 *   G_ij = 1/2 (grad W^R_ij - grad W^R_ji)   (each term with its own coefficients, H, x)
 *   m_i a_i     = - sum_j V_i V_j (P_i + P_j + Q_ij) G_ij
 *   m_i du_i/dt =   sum_j V_i V_j (P_i + Q_ij/2) (v_i - v_j) . G_ij
 *   Q_ij = Q_i + Q_j, Q_k = rho_k (-C_l c_k mu_k + C_q mu_k^2),
 *   mu_k = min(0, v*.eta_k / (eta_k.eta_k + eps_AV^2)), eta_k = x_ij / H_k,
 *   v* = v_ij - 1/2 phi x_ij.(grad v_i + grad v_j),  phi = vanLeer(r),
 *   r = (x.grad v_i.x)/(x.grad v_j.x); phi = 0 if the denominator is 0 or r <= 0.
 * Kick: v += dt a, u += dt du/dt (vout, uout).
 * Sa[t] = sum_j |pair term of a_i|, Sdu[t] = sum_j |pair term of du_i/dt|. */
int orc_accel(int64_t n, const float* x, const float* y, const float* z, const uint8_t* species,
              const float* H, const float* m, const float* vx, const float* vy, const float* vz,
              const float* u, const double* V, const double* A, const double* B, const double* dA,
              const double* dB, const double* rho, const double* P, const double* cs,
              const double* dv, const orc_params* p, double dt, int64_t nt, const int64_t* targets,
              double* acc, double* dudt, double* Sa, double* Sdu, double* vout, double* uout,
              int force_brute) {
    int64_t ng;
    int64_t* gm = gas_members(n, species, &ng);
    grid_t gg;
    grid_build(&gg, x, y, z, ng, gm, p->box, sqrt((double)max_h2(ng, gm, H)) * 1.0001, force_brute);
    pctx c = {x, y, z, H, p->box, p->rcut2};
    const double Cl = p->av_cl, Cq = p->av_cq, e2 = p->av_eps2;
#pragma omp parallel
    {
        ivec nb = {0, 0, 0};
#pragma omp for schedule(dynamic, 16)
        for (int64_t t = 0; t < nt; ++t) {
            int64_t i = targets[t];
            neighbours(&gg, &c, PRED_SYM, i, &nb);
            double a[3] = {0, 0, 0}, du = 0.0, sa = 0.0, sdu = 0.0;
            double vi[3] = {vx[i], vy[i], vz[i]};
            for (int64_t u2 = 0; u2 < nb.n; ++u2) {
                int64_t j = nb.v[u2];
                double xij[3], xji[3], WRij, WRji, gij[3], gji[3];
                sep_ij(x, y, z, p->box, i, j, xij);
                for (int k = 0; k < 3; ++k) xji[k] = -xij[k];
                corrected(A[i], B + 3 * i, dA + 3 * i, dB + 9 * i, xij, H[i], &WRij, gij);
                corrected(A[j], B + 3 * j, dA + 3 * j, dB + 9 * j, xji, H[j], &WRji, gji);
                double G[3];
                for (int k = 0; k < 3; ++k) G[k] = 0.5 * (gij[k] - gji[k]);
                double vj[3] = {vx[j], vy[j], vz[j]};
                double vij[3] = {vi[0] - vj[0], vi[1] - vj[1], vi[2] - vj[2]};
                /* limiter */
                double xgi = 0.0, xgj = 0.0, gvi[3] = {0, 0, 0}, gvj[3] = {0, 0, 0};
                for (int al = 0; al < 3; ++al)
                    for (int be = 0; be < 3; ++be) {
                        gvi[al] += dv[9 * i + 3 * al + be] * xij[be];
                        gvj[al] += dv[9 * j + 3 * al + be] * xij[be];
                    }
                for (int al = 0; al < 3; ++al) { xgi += xij[al] * gvi[al]; xgj += xij[al] * gvj[al]; }
                double phi = 0.0;
                if (xgj != 0.0) {
                    double rr = xgi / xgj;
                    if (rr > 0.0) {
                        phi = 4.0 * rr / ((1.0 + rr) * (1.0 + rr));
                        if (phi > 1.0) phi = 1.0;
                        if (phi < 0.0) phi = 0.0;
                    }
                }
                double vs[3];
                for (int k = 0; k < 3; ++k) vs[k] = vij[k] - 0.5 * phi * (gvi[k] + gvj[k]);
                double Q = 0.0;
                const double Hk[2] = {H[i], H[j]};
                const double rk[2] = {rho[i], rho[j]}, ck[2] = {cs[i], cs[j]};
                for (int s = 0; s < 2; ++s) {
                    double eta[3] = {xij[0] / Hk[s], xij[1] / Hk[s], xij[2] / Hk[s]};
                    double ee = eta[0] * eta[0] + eta[1] * eta[1] + eta[2] * eta[2];
                    double mu = (vs[0] * eta[0] + vs[1] * eta[1] + vs[2] * eta[2]) / (ee + e2);
                    if (mu > 0.0) mu = 0.0;
                    Q += rk[s] * (-Cl * ck[s] * mu + Cq * mu * mu);
                }
                double VV = V[i] * V[j];
                double fa = -VV * (P[i] + P[j] + Q) / (double)m[i];
                double fu = VV * (P[i] + 0.5 * Q) * (vij[0] * G[0] + vij[1] * G[1] + vij[2] * G[2]) / (double)m[i];
                for (int k = 0; k < 3; ++k) a[k] += fa * G[k];
                du += fu;
                sa += fabs(fa) * sqrt(G[0] * G[0] + G[1] * G[1] + G[2] * G[2]);
                sdu += fabs(fu);
            }
            for (int k = 0; k < 3; ++k) {
                acc[3 * t + k] = a[k];
                vout[3 * t + k] = vi[k] + dt * a[k];
            }
            dudt[t] = du;
            uout[t] = (double)u[i] + dt * du;
            Sa[t] = sa;
            Sdu[t] = sdu;
        }
        free(nb.v);
    }
    grid_free(&gg);
    free(gm);
    return 0;
}

/* Neighbour sets for the closure of sampled targets (tests only): writes the
 * sorted neighbour indices of each target (pred: 1 gather incl. self, 2 sym).
 * Called with out == NULL it returns the lengths. */
int orc_neighbour_sets(int64_t n, const float* x, const float* y, const float* z,
                       const uint8_t* species, const float* H, const orc_params* p, int pred,
                       int64_t nt, const int64_t* targets, int64_t* len, const int64_t* off,
                       int64_t* out) {
    int64_t ng;
    int64_t* gm = gas_members(n, species, &ng);
    grid_t gg;
    grid_build(&gg, x, y, z, ng, gm, p->box, sqrt((double)max_h2(ng, gm, H)) * 1.0001, 0);
    pctx c = {x, y, z, H, p->box, p->rcut2};
    int pr = pred == 1 ? PRED_GATHER_SELF : PRED_SYM;
#pragma omp parallel
    {
        ivec nb = {0, 0, 0};
#pragma omp for schedule(dynamic, 16)
        for (int64_t t = 0; t < nt; ++t) {
            neighbours(&gg, &c, pr, targets[t], &nb);
            if (!out) len[t] = nb.n;
            else memcpy(out + off[t], nb.v, sizeof(int64_t) * (size_t)nb.n);
        }
        free(nb.v);
    }
    grid_free(&gg);
    free(gm);
    return 0;
}

int orc_num_threads(void) { return omp_get_max_threads(); }

void orc_set_threads(int n) { omp_set_num_threads(n > 0 ? n : 1); }

/* ------------------------------------------------------------------ sub-cycle (NEXT-2)
 * Readings (DESIGN.md §2 "Sub-cycle"; SURVEY.md §8(f) NEXT-2 names the steps, the paper
 * only that the kernels run several times per step, and a float fetch_min,
 * PAPER.md:389):
 *   time step  dt = min_i dt_i,  dt_i = C_acc sqrt(eps / |a_i|) (eps = sqrt(eps2), a the
 *              gravity acceleration plus, for gas, the hydro one), and for gas also
 *              C_cfl H_i / c_i — evaluated here in fp64;
 *   kick       v += dt a, u += dt du/dt: one fp32 fma per component (as specified);
 *   drift      x' = fl32(x + dt v) (one fp32 fma), rounded to the nearest multiple of
 *              q = L_max 2^-23 (ties to even), wrapped into [0, L) — positions stay on the
 *              q lattice (O1).  Specified in fp32 so that it is compared bit for bit. */
double orc_courant(int64_t n, const uint8_t* species, const float* H, const float* cs, const float* ax,
                   const float* ay, const float* az, const float* ahx, const float* ahy, const float* ahz,
                   double eps2, double c_cfl, double c_acc) {
    const double eps = sqrt(eps2);
    double best = INFINITY;
    for (int64_t i = 0; i < n; ++i) {
        double gx = ax[i], gy = ay[i], gz = az[i];
        if (species[i] == 1) { gx += ahx[i]; gy += ahy[i]; gz += ahz[i]; }
        const double a = sqrt(gx * gx + gy * gy + gz * gz);
        double d = a > 0.0 ? c_acc * sqrt(eps / a) : INFINITY;
        if (species[i] == 1 && cs[i] > 0.0f) {
            const double dc = c_cfl * (double)H[i] / (double)cs[i];
            if (dc < d) d = dc;
        }
        if (d < best) best = d;
    }
    return best;
}

void orc_kick(int64_t n, const uint8_t* species, float dt, const float* ax, const float* ay, const float* az,
              const float* ahx, const float* ahy, const float* ahz, const float* dudt, float* vx, float* vy,
              float* vz, float* u) {
    for (int64_t i = 0; i < n; ++i) {
        float gx = ax[i], gy = ay[i], gz = az[i];
        if (species[i] == 1) {
            gx += ahx[i]; gy += ahy[i]; gz += ahz[i];
            u[i] = fmaf(dt, dudt[i], u[i]);
        }
        vx[i] = fmaf(dt, gx, vx[i]);
        vy[i] = fmaf(dt, gy, vy[i]);
        vz[i] = fmaf(dt, gz, vz[i]);
    }
}

static float drift1(float x, float v, float dt, float q, float L) {
    const float t = fmaf(dt, v, x);
    float r = rintf(t / q) * q; /* q a power of two: the division and product are exact */
    if (r >= L) r -= L;
    else if (r < 0.0f) r += L;
    return r;
}

void orc_drift(int64_t n, const double* box, float dt, float* x, float* y, float* z, const float* vx,
               const float* vy, const float* vz) {
    double lmax = box[0] > box[1] ? box[0] : box[1];
    if (box[2] > lmax) lmax = box[2];
    const float q = (float)ldexp(lmax, -23);
    for (int64_t i = 0; i < n; ++i) {
        x[i] = drift1(x[i], vx[i], dt, q, (float)box[0]);
        y[i] = drift1(y[i], vy[i], dt, q, (float)box[1]);
        z[i] = drift1(z[i], vz[i], dt, q, (float)box[2]);
    }
}

/* Smoothing-length update (NEXT-2; DESIGN.md §2 "Sub-cycle"): for each target gas particle
 * t, d2_(k) = the k-th smallest O2 squared distance s32 to another gas particle (brute force
 * over every gas particle, min image, fp32 predicate arithmetic as in O2), then
 * H' = fl32(factor * fl32(sqrt(d2_(k)))), and conv[t] = d2_(k) < fl32(H_t^2) (the GPU selects
 * among its neighbour list, which holds every particle within H_t). */
static int cmp_f32(const void* a, const void* b) {
    const float x = *(const float*)a, y = *(const float*)b;
    return (x > y) - (x < y);
}

void orc_knn_h(int64_t n, const float* x, const float* y, const float* z, const uint8_t* species, const float* H,
               const double* box, int64_t nt, const int64_t* targets, int k, float factor, float* H_out,
               int32_t* conv) {
#pragma omp parallel
    {
        float* d = (float*)malloc(sizeof(float) * (size_t)n);
#pragma omp for schedule(dynamic, 4)
        for (int64_t q = 0; q < nt; ++q) {
            const int64_t i = targets[q];
            int64_t m = 0;
            for (int64_t j = 0; j < n; ++j) {
                if (j == i || species[j] != 1) continue;
                const double dx = min_image(x[j], x[i], box[0]);
                const double dy = min_image(y[j], y[i], box[1]);
                const double dz = min_image(z[j], z[i], box[2]);
                d[m++] = s32_of(dx, dy, dz);
            }
            qsort(d, (size_t)m, sizeof(float), cmp_f32);
            const float d2 = m >= k ? d[k - 1] : INFINITY;
            H_out[q] = factor * sqrtf(d2);
            conv[q] = d2 < h2_of(H[i]);
        }
        free(d);
    }
}
