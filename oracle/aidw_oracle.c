/*
 * aidw_oracle.c — CPU restatement of the reference AIDW hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_1601_05904_b200/,
 * include/) links, loads or calls this file.  It is imported by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg, and only as the
 * checker.  The product path fails loudly when its CUDA library is missing.
 *
 * Pinning: the outputs of this restatement are compared bit-for-bit against
 * the reference itself (oracle/_ref/libaidw_ref.so, compiled from
 * /root/reference/proj/include by oracle/Makefile) through the committed
 * fixtures in tests/golden/ (generator: tests/golden/make_golden.py), and
 * against the reference's own known-answer tests (tests/test_oracle.py).
 *
 * Build: gcc -O2 -ffp-contract=off (mandatory — see SURVEY §8c: with FMA
 * contraction dist_sq stops being the two-products-then-add expression that
 * the reference's bit-exact tests assume).
 *
 * Every function names the reference lines it restates, as
 * proj/include/aidw/<file>:<lines>.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_INVALID 1  /* std::invalid_argument */
#define ORC_DOMAIN 2   /* std::domain_error     */
#define ORC_RANGE 3    /* std::out_of_range     */

/* ------------------------------------------------------------------ */
/* mt19937_64 + unit_double: proj/include/aidw/generate.hpp:37-39       */
/* ------------------------------------------------------------------ */
typedef struct {
    uint64_t s[312];
    int i;
} orc_mt64;

static void mt64_seed(orc_mt64* g, uint64_t seed) {
    g->s[0] = seed;
    for (int k = 1; k < 312; ++k) {
        g->s[k] = 6364136223846793005ULL * (g->s[k - 1] ^ (g->s[k - 1] >> 62)) + (uint64_t)k;
    }
    g->i = 312;
}

static uint64_t mt64_next(orc_mt64* g) {
    if (g->i >= 312) {
        for (int k = 0; k < 312; ++k) {
            uint64_t y = (g->s[k] & 0xFFFFFFFF80000000ULL) | (g->s[(k + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t v = g->s[(k + 156) % 312] ^ (y >> 1);
            if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
            g->s[k] = v;
        }
        g->i = 0;
    }
    uint64_t x = g->s[g->i++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}

static double unit01(orc_mt64* g) { return (double)(mt64_next(g) >> 11) * 0x1.0p-53; }

/* generate_random_points: generate.hpp:45-74 (3 draws per point; value rules
 * uniform=0 / planar=1 / radial=2, planar coefficients generate.hpp:23-30). */
int orc_generate_points(size_t count, double bx0, double by0, double bx1, double by1,
                        uint64_t seed, int rule, double* xs, double* ys, double* zs) {
    if (count == 0) return ORC_INVALID;
    if (!(bx0 <= bx1 && by0 <= by1) || !((bx1 - bx0) * (by1 - by0) > 0.0)) return ORC_INVALID;
    orc_mt64 g;
    mt64_seed(&g, seed);
    const double w = bx1 - bx0, h = by1 - by0;
    const double cx = bx0 + 0.5 * w, cy = by0 + 0.5 * h;
    for (size_t i = 0; i < count; ++i) {
        const double x = bx0 + unit01(&g) * w;
        const double y = by0 + unit01(&g) * h;
        const double noise = unit01(&g);
        double z = noise;
        if (rule == 1) {
            const double ax = 1.5 * x;
            const double by = -2.5 * y;
            z = ax + by + 4.0;
        } else if (rule == 2) {
            z = hypot(x - cx, y - cy);
        }
        xs[i] = x;
        ys[i] = y;
        zs[i] = z;
    }
    return ORC_OK;
}

/* generate_random_queries: generate.hpp:77-95 (2 draws per query). */
int orc_generate_queries(size_t count, double bx0, double by0, double bx1, double by1,
                         uint64_t seed, double* xs, double* ys) {
    if (count == 0) return ORC_INVALID;
    if (!(bx0 <= bx1 && by0 <= by1) || !((bx1 - bx0) * (by1 - by0) > 0.0)) return ORC_INVALID;
    orc_mt64 g;
    mt64_seed(&g, seed);
    const double w = bx1 - bx0, h = by1 - by0;
    for (size_t i = 0; i < count; ++i) {
        xs[i] = bx0 + unit01(&g) * w;
        ys[i] = by0 + unit01(&g) * h;
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* Domain helpers: types.hpp:70-87, :124-143                          */
/* ------------------------------------------------------------------ */
/* bbox over data ∪ queries; out = {min_x, min_y, max_x, max_y}.        */
int orc_compute_bbox(const double* dx, const double* dy, size_t m, const double* qx,
                     const double* qy, size_t n, double* out) {
    if (m == 0 && n == 0) return ORC_INVALID;
    double lx = INFINITY, ly = INFINITY, hx = -INFINITY, hy = -INFINITY;
    for (size_t i = 0; i < m; ++i) {
        lx = fmin(lx, dx[i]); ly = fmin(ly, dy[i]);
        hx = fmax(hx, dx[i]); hy = fmax(hy, dy[i]);
    }
    for (size_t i = 0; i < n; ++i) {
        lx = fmin(lx, qx[i]); ly = fmin(ly, qy[i]);
        hx = fmax(hx, qx[i]); hy = fmax(hy, qy[i]);
    }
    out[0] = lx; out[1] = ly; out[2] = hx; out[3] = hy;
    return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* Grid geometry: grid.hpp:50-127                                      */
/* ------------------------------------------------------------------ */
typedef struct {
    double cell_width;
    int n_col, n_row;
    double min_x, min_y;
} orc_grid_config;

/* choose_cell_width: grid.hpp:50-64 — factor * (1 / (2 * sqrt(m / area))) */
int orc_choose_cell_width(size_t m, const double* bbox, double factor, double* out) {
    if (m == 0) return ORC_INVALID;
    const double w = bbox[2] - bbox[0], h = bbox[3] - bbox[1];
    if (!(bbox[0] <= bbox[2] && bbox[1] <= bbox[3]) || !(w * h > 0.0)) return ORC_INVALID;
    if (!(factor > 0.0) || !isfinite(factor)) return ORC_INVALID;
    const double density = (double)m / (w * h);
    *out = factor * (1.0 / (2.0 * sqrt(density)));
    return ORC_OK;
}

/* make_grid_config: grid.hpp:67-88 (padded columns, 1e9-cell cap). */
int orc_make_grid_config(const double* bbox, double cell_width, orc_grid_config* cfg) {
    const double w = bbox[2] - bbox[0], h = bbox[3] - bbox[1];
    if (!(bbox[0] <= bbox[2] && bbox[1] <= bbox[3]) || !(w * h > 0.0)) return ORC_INVALID;
    if (!(cell_width > 0.0) || !isfinite(cell_width)) return ORC_INVALID;
    const double cols = floor((bbox[2] - bbox[0] + cell_width) / cell_width);
    const double rows = floor((bbox[3] - bbox[1] + cell_width) / cell_width);
    if (cols * rows > 1.0e9) return ORC_INVALID;
    cfg->cell_width = cell_width;
    cfg->n_col = (int)cols < 1 ? 1 : (int)cols;
    cfg->n_row = (int)rows < 1 ? 1 : (int)rows;
    cfg->min_x = bbox[0];
    cfg->min_y = bbox[1];
    return ORC_OK;
}

static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* locate_cell: grid.hpp:93-106 — FP64 divide, 1e-9*(n+1) slack, floor, clamp. */
int orc_locate_cell(double x, double y, const orc_grid_config* c, int* col, int* row) {
    const double fx = (x - c->min_x) / c->cell_width;
    const double fy = (y - c->min_y) / c->cell_width;
    const double sx = 1.0e-9 * ((double)c->n_col + 1.0);
    const double sy = 1.0e-9 * ((double)c->n_row + 1.0);
    const int ok_x = fx >= -sx && fx <= (double)c->n_col + sx;
    const int ok_y = fy >= -sy && fy <= (double)c->n_row + sy;
    if (!ok_x || !ok_y) return ORC_DOMAIN;
    *col = clampi((int)floor(fx), 0, c->n_col - 1);
    *row = clampi((int)floor(fy), 0, c->n_row - 1);
    return ORC_OK;
}

/* build_index: grid.hpp:176-213 — counting sort by row-major cell id,
 * stable within a cell.  cell_start has n_col*n_row+1 entries.  On a
 * locate failure *fail_index receives the point index. */
int orc_build_index(const double* xs, const double* ys, size_t m, const orc_grid_config* c,
                    uint32_t* sorted_ids, uint32_t* cell_start, double* sorted_x,
                    double* sorted_y, int64_t* fail_index) {
    if (m == 0) return ORC_INVALID;
    if (m > 0xFFFFFFFEull) return ORC_INVALID;
    const size_t cells = (size_t)c->n_col * (size_t)c->n_row;
    uint32_t* cell_of = (uint32_t*)malloc(m * sizeof(uint32_t));
    for (size_t i = 0; i < m; ++i) {
        int col, row;
        if (orc_locate_cell(xs[i], ys[i], c, &col, &row) != ORC_OK) {
            if (fail_index) *fail_index = (int64_t)i;
            free(cell_of);
            return ORC_DOMAIN;
        }
        cell_of[i] = (uint32_t)((size_t)row * (size_t)c->n_col + (size_t)col);
    }
    memset(cell_start, 0, (cells + 1) * sizeof(uint32_t));
    for (size_t i = 0; i < m; ++i) cell_start[cell_of[i] + 1] += 1;
    for (size_t k = 1; k <= cells; ++k) cell_start[k] += cell_start[k - 1];
    uint32_t* fill = (uint32_t*)malloc(cells * sizeof(uint32_t));
    memcpy(fill, cell_start, cells * sizeof(uint32_t));
    for (size_t i = 0; i < m; ++i) {
        const uint32_t slot = fill[cell_of[i]]++;
        sorted_ids[slot] = (uint32_t)i;
        sorted_x[slot] = xs[i];
        sorted_y[slot] = ys[i];
    }
    free(fill);
    free(cell_of);
    return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* kNN: knn.hpp:23-27 (dist_sq), :54-94 (k-slot buffer), :100-114,     */
/* :130-156 (expansion level), :162-194 (block/ring), :212-249        */
/* ------------------------------------------------------------------ */
static double dsq(double qx, double qy, double px, double py) {
    const double dx = px - qx;
    const double dy = py - qy;
    const double a = dx * dx;
    const double b = dy * dy;
    return a + b;
}

double orc_dist_sq(double qx, double qy, double px, double py) { return dsq(qx, qy, px, py); }

/* (d2, idx)-lexicographic bounded buffer.  The value multiset it keeps is the
 * reference buffer's (knn.hpp:54-94: strict-less admission once full, so
 * ties at the kth value are never admitted); the index attached to each
 * value is the restated north-star tie rule "ties by index". */
typedef struct {
    double* d2;
    uint32_t* id;
    size_t cap, len;
} orc_topk;

static int pair_less(double da, uint32_t ia, double db, uint32_t ib) {
    return da < db || (da == db && ia < ib);
}

static void topk_offer(orc_topk* t, double d2, uint32_t id) {
    size_t pos;
    if (t->len < t->cap) {
        pos = t->len++;
    } else if (pair_less(d2, id, t->d2[t->cap - 1], t->id[t->cap - 1])) {
        pos = t->cap - 1;
    } else {
        return;
    }
    while (pos > 0 && pair_less(d2, id, t->d2[pos - 1], t->id[pos - 1])) {
        t->d2[pos] = t->d2[pos - 1];
        t->id[pos] = t->id[pos - 1];
        --pos;
    }
    t->d2[pos] = d2;
    t->id[pos] = id;
}

/* knn.hpp:78-89: ascending sum of sqrt, divided by the list length. */
static double topk_mean_distance(const orc_topk* t) {
    double s = 0.0;
    for (size_t i = 0; i < t->len; ++i) s = s + sqrt(t->d2[i]);
    return t->len == 0 ? 0.0 : s / (double)t->len;
}

/* brute_force_knn: knn.hpp:100-114.  Output d2/id arrays of length k. */
int orc_brute_knn(double qx, double qy, const double* xs, const double* ys, size_t m, int k,
                  double* d2, uint32_t* id, double* avg) {
    if (m == 0) return ORC_INVALID;
    if (k < 1 || (size_t)k > m) return ORC_INVALID;
    orc_topk t = {d2, id, (size_t)k, 0};
    for (size_t i = 0; i < m; ++i) topk_offer(&t, dsq(qx, qy, xs[i], ys[i]), (uint32_t)i);
    *avg = topk_mean_distance(&t);
    return ORC_OK;
}

typedef struct {
    const orc_grid_config* cfg;
    const uint32_t* cell_start;
    const uint32_t* sorted_ids;
    const double* sorted_x;
    const double* sorted_y;
    size_t m;
} orc_grid;

static size_t row_points(const orc_grid* g, int row, int c0, int c1) {
    const size_t base = (size_t)row * (size_t)g->cfg->n_col;
    return g->cell_start[base + (size_t)c1 + 1] - g->cell_start[base + (size_t)c0];
}

static size_t block_points(const orc_grid* g, int c0, int c1, int r0, int r1) {
    size_t total = 0;
    for (int r = r0; r <= r1; ++r) total += row_points(g, r, c0, c1);
    return total;
}

/* determine_expansion_level: knn.hpp:130-156. */
int orc_expansion_level(double qx, double qy, const orc_grid* g, int k, int* level,
                        int* exhausted) {
    if (g->m == 0 || k < 1) return ORC_INVALID;
    const orc_grid_config* c = g->cfg;
    int col, row;
    const int rc = orc_locate_cell(qx, qy, c, &col, &row);
    if (rc) return rc;
    if (g->m < (size_t)k) {
        int a = col > c->n_col - 1 - col ? col : c->n_col - 1 - col;
        int b = row > c->n_row - 1 - row ? row : c->n_row - 1 - row;
        *level = a > b ? a : b;
        *exhausted = 1;
        return ORC_OK;
    }
    for (int L = 0;; ++L) {
        const int c0 = col - L < 0 ? 0 : col - L;
        const int c1 = col + L > c->n_col - 1 ? c->n_col - 1 : col + L;
        const int r0 = row - L < 0 ? 0 : row - L;
        const int r1 = row + L > c->n_row - 1 ? c->n_row - 1 : row + L;
        if (block_points(g, c0, c1, r0, r1) >= (size_t)k) {
            *level = L + 1;
            *exhausted = 0;
            return ORC_OK;
        }
    }
}

static void scan_rect(const orc_grid* g, orc_topk* t, double qx, double qy, int c0, int c1,
                      int r0, int r1) {
    for (int r = r0; r <= r1; ++r) {
        const size_t base = (size_t)r * (size_t)g->cfg->n_col;
        const uint32_t b = g->cell_start[base + (size_t)c0];
        const uint32_t e = g->cell_start[base + (size_t)c1 + 1];
        for (uint32_t s = b; s < e; ++s)
            topk_offer(t, dsq(qx, qy, g->sorted_x[s], g->sorted_y[s]), g->sorted_ids[s]);
    }
}

/* grid_knn: knn.hpp:212-249 (+ scan_ring :175-194).  *out_len = min(k, m). */
int orc_grid_knn(double qx, double qy, const orc_grid* g, int k, double* d2, uint32_t* id,
                 double* avg, int* exhausted, size_t* out_len) {
    if (g->m == 0 || k < 1) return ORC_INVALID;
    const orc_grid_config* c = g->cfg;
    int col, row, level, exh;
    int rc = orc_locate_cell(qx, qy, c, &col, &row);
    if (rc) return rc;
    rc = orc_expansion_level(qx, qy, g, k, &level, &exh);
    if (rc) return rc;
    const size_t keff = (size_t)k < g->m ? (size_t)k : g->m;
    orc_topk t = {d2, id, keff, 0};
    {
        const int c0 = col - level < 0 ? 0 : col - level;
        const int c1 = col + level > c->n_col - 1 ? c->n_col - 1 : col + level;
        const int r0 = row - level < 0 ? 0 : row - level;
        const int r1 = row + level > c->n_row - 1 ? c->n_row - 1 : row + level;
        scan_rect(g, &t, qx, qy, c0, c1, r0, r1);
    }
    for (;;) {
        const int covers = col - level <= 0 && row - level <= 0 && col + level >= c->n_col - 1 &&
                           row + level >= c->n_row - 1;
        if (covers) break;
        const double reach = (double)level * c->cell_width;
        const double bound = reach * reach;
        if (t.len == t.cap && t.d2[t.cap - 1] <= bound * (1.0 - 1.0e-9)) break;
        ++level;
        /* new ring: two full rows over the widened columns, two columns over
         * the previous level's rows (knn.hpp:175-194) */
        const int c0 = col - level < 0 ? 0 : col - level;
        const int c1 = col + level > c->n_col - 1 ? c->n_col - 1 : col + level;
        if (row - level >= 0) scan_rect(g, &t, qx, qy, c0, c1, row - level, row - level);
        if (row + level <= c->n_row - 1) scan_rect(g, &t, qx, qy, c0, c1, row + level, row + level);
        const int pr0 = row - (level - 1) < 0 ? 0 : row - (level - 1);
        const int pr1 = row + (level - 1) > c->n_row - 1 ? c->n_row - 1 : row + (level - 1);
        if (col - level >= 0) scan_rect(g, &t, qx, qy, col - level, col - level, pr0, pr1);
        if (col + level <= c->n_col - 1) scan_rect(g, &t, qx, qy, col + level, col + level, pr0, pr1);
    }
    *avg = topk_mean_distance(&t);
    *exhausted = exh;
    *out_len = t.len;
    return ORC_OK;
}

/* Batch grid kNN over a query set (knn.hpp:255-271).  d2/id are n x k
 * row-major (rows shorter than k when exhausted are padded with +inf /
 * 0xFFFFFFFF).  *fail_index gets the smallest failing query. */
int orc_knn_stage_grid(const double* qx, const double* qy, size_t n, const orc_grid_config* cfg,
                       const uint32_t* cell_start, const uint32_t* sorted_ids,
                       const double* sorted_x, const double* sorted_y, size_t m, int k,
                       double* d2, uint32_t* id, double* avg, int* exhausted,
                       int64_t* fail_index) {
    orc_grid g = {cfg, cell_start, sorted_ids, sorted_x, sorted_y, m};
    for (size_t i = 0; i < n; ++i) {
        size_t len = 0;
        double* row_d = d2 + i * (size_t)k;
        uint32_t* row_i = id + i * (size_t)k;
        for (int j = 0; j < k; ++j) {
            row_d[j] = INFINITY;
            row_i[j] = 0xFFFFFFFFu;
        }
        const int rc = orc_grid_knn(qx[i], qy[i], &g, k, row_d, row_i, &avg[i], &exhausted[i], &len);
        if (rc) {
            if (fail_index) *fail_index = (int64_t)i;
            return rc;
        }
    }
    return ORC_OK;
}

int orc_knn_stage_brute(const double* qx, const double* qy, size_t n, const double* xs,
                        const double* ys, size_t m, int k, double* d2, uint32_t* id, double* avg,
                        int64_t* fail_index) {
    for (size_t i = 0; i < n; ++i) {
        const int rc = orc_brute_knn(qx[i], qy[i], xs, ys, m, k, d2 + i * (size_t)k,
                                     id + i * (size_t)k, &avg[i]);
        if (rc) {
            if (fail_index) *fail_index = (int64_t)i;
            return rc;
        }
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* Adaptive power: adaptive.hpp:20-116                                  */
/* ------------------------------------------------------------------ */
static const double kPi = 3.141592653589793238462643383279502884;
static const double kBreaks[5] = {0.1, 0.3, 0.5, 0.7, 0.9};

/* expected_nn_distance: adaptive.hpp:20-28 */
int orc_expected_nn_distance(size_t m, double area, double* out) {
    if (m == 0) return ORC_INVALID;
    if (!(area > 0.0) || !isfinite(area)) return ORC_INVALID;
    *out = 1.0 / (2.0 * sqrt((double)m / area));
    return ORC_OK;
}

/* normalize_mu: adaptive.hpp:49-60 — cosine argument scaled by pi / r_max
 * (the reference keeps this quirk; see its comment at :45-48). */
int orc_normalize_mu(double R, double r_min, double r_max, double* out) {
    if (!(r_min < r_max)) return ORC_INVALID;
    if (R <= r_min) { *out = 0.0; return ORC_OK; }
    if (R >= r_max) { *out = 1.0; return ORC_OK; }
    const double phase = (kPi / r_max) * (R - r_min);
    *out = 0.5 - 0.5 * cos(phase);
    return ORC_OK;
}

/* alpha_from_mu: adaptive.hpp:69-87 — lower-inclusive segments, a+t(b-a). */
int orc_alpha_from_mu(double mu, const double* lv, double* out) {
    if (!(mu >= 0.0 && mu <= 1.0)) return ORC_DOMAIN;
    if (mu < kBreaks[0]) { *out = lv[0]; return ORC_OK; }
    if (mu >= kBreaks[4]) { *out = lv[4]; return ORC_OK; }
    int s = 0;
    while (mu >= kBreaks[s + 1]) ++s;
    const double t = 5.0 * (mu - kBreaks[s]);
    *out = lv[s] + t * (lv[s + 1] - lv[s]);
    return ORC_OK;
}

static int params_ok(int k, double r_min, double r_max, const double* lv) {
    if (k < 1) return 0;
    if (!(r_min < r_max)) return 0;
    for (int i = 0; i < 5; ++i)
        if (!(lv[i] > 0.0) || !isfinite(lv[i])) return 0;
    return 1;
}

/* adaptive_alpha: adaptive.hpp:101-116; rec = {r_exp, r_obs, R, mu, alpha}.
 * list_len / exhausted describe the KnnResult (size check :104-108). */
int orc_adaptive_alpha(double r_obs, size_t list_len, int exhausted, size_t m, double area,
                       int k, double r_min, double r_max, const double* lv, double* rec) {
    if (!params_ok(k, r_min, r_max, lv)) return ORC_INVALID;
    if (!exhausted && list_len != (size_t)k) return ORC_INVALID;
    double r_exp, mu, alpha;
    int rc = orc_expected_nn_distance(m, area, &r_exp);
    if (rc) return rc;
    if (!(r_exp > 0.0) || r_obs < 0.0) return ORC_INVALID;
    const double R = r_obs / r_exp;
    rc = orc_normalize_mu(R, r_min, r_max, &mu);
    if (rc) return rc;
    rc = orc_alpha_from_mu(mu, lv, &alpha);
    if (rc) return rc;
    rec[0] = r_exp; rec[1] = r_obs; rec[2] = R; rec[3] = mu; rec[4] = alpha;
    return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* Weighting: interpolate.hpp:73-137, :252-381, :426-489               */
/* ------------------------------------------------------------------ */
/* nearest_value: interpolate.hpp:94-105 (strict <, first index on ties) */
static double nearest_z(double qx, double qy, const double* xs, const double* ys,
                        const double* zs, size_t m) {
    size_t best = 0;
    double bd = dsq(qx, qy, xs[0], ys[0]);
    for (size_t i = 1; i < m; ++i) {
        const double d = dsq(qx, qy, xs[i], ys[i]);
        if (d < bd) { bd = d; best = i; }
    }
    return zs[best];
}

/* settle: interpolate.hpp:109-118 */
static double settle(double sw, double swz, double qx, double qy, const double* xs,
                     const double* ys, const double* zs, size_t m, double zlo, double zhi) {
    if (sw > 0.0 && isfinite(sw) && isfinite(swz)) {
        const double p = swz / sw;
        if (isfinite(p)) return p < zlo ? zlo : (p > zhi ? zhi : p);
    }
    return nearest_z(qx, qy, xs, ys, zs, m);
}

/* predict_naive: interpolate.hpp:122-137 — index order, 1/pow(sqrt(d2),a). */
static double predict_naive(double qx, double qy, const double* xs, const double* ys,
                            const double* zs, size_t m, double alpha, double snap_sq,
                            double zlo, double zhi) {
    double sw = 0.0, swz = 0.0;
    for (size_t i = 0; i < m; ++i) {
        const double d2 = dsq(qx, qy, xs[i], ys[i]);
        if (d2 <= snap_sq) return zs[i];
        const double w = 1.0 / pow(sqrt(d2), alpha);
        sw += w;
        swz += w * zs[i];
    }
    return settle(sw, swz, qx, qy, xs, ys, zs, m, zlo, zhi);
}

/* predict_blocked_fast, scalar form: interpolate.hpp:252-381 without the
 * SIMD lanes — 256-point chunks, exact half-integer recipe (:174-209) or
 * exp(-alpha/2 * log d2), chunk partials folded into running sums.  The
 * lane-parallel partial order of the AVX paths is NOT reproduced, so this
 * agrees with the reference blocked variant only to rounding (~1e-13). */
static double predict_blocked(double qx, double qy, const double* xs, const double* ys,
                              const double* zs, size_t m, double alpha, double snap_sq,
                              double zlo, double zhi) {
    const double e = -0.5 * alpha;
    const double twice = 2.0 * alpha;
    const int exact = twice == floor(twice) && twice >= 1.0 && twice <= 16.0;
    const int n4 = exact ? (int)twice : 0;
    double sw = 0.0, swz = 0.0;
    for (size_t base = 0; base < m; base += 256) {
        const size_t nc = m - base < 256 ? m - base : 256;
        for (size_t j = 0; j < nc; ++j)
            if (dsq(qx, qy, xs[base + j], ys[base + j]) <= snap_sq) return zs[base + j];
        double cw = 0.0, cwz = 0.0;
        for (size_t j = 0; j < nc; ++j) {
            const double d2 = dsq(qx, qy, xs[base + j], ys[base + j]);
            double w;
            if (exact) {
                double den = (n4 / 4) > 0 ? d2 : 1.0;
                for (int p = 1; p < n4 / 4; ++p) den *= d2;
                if (n4 & 3) {
                    const double r = sqrt(d2);
                    if (n4 & 2) den *= r;
                    if (n4 & 1) den *= sqrt(r);
                }
                w = 1.0 / den;
            } else {
                w = exp(e * log(d2));
            }
            cw += w;
            cwz += w * zs[base + j];
        }
        sw += cw;
        swz += cwz;
    }
    return settle(sw, swz, qx, qy, xs, ys, zs, m, zlo, zhi);
}

/* snap_tolerance_sq: interpolate.hpp:86-89; hull: :73-80 */
static void weighting_context(const double* bbox, const double* zs, size_t m, double* snap_sq,
                              double* zlo, double* zhi) {
    const double eps = 1.0e-12 * hypot(bbox[2] - bbox[0], bbox[3] - bbox[1]);
    *snap_sq = eps * eps;
    double lo = zs[0], hi = zs[0];
    for (size_t i = 0; i < m; ++i) {
        lo = fmin(lo, zs[i]);
        hi = fmax(hi, zs[i]);
    }
    *zlo = lo;
    *zhi = hi;
}

/* Predict with per-query alphas.  variant: 0 = naive (also the pinned
 * blocked variant, interpolate.hpp:142-166, which is bit-equal to it),
 * 1 = blocked (scalar restatement above). */
int orc_predict_with_alphas(const double* qx, const double* qy, size_t n, const double* xs,
                            const double* ys, const double* zs, size_t m, const double* alphas,
                            int variant, double* pred) {
    if (m == 0) return ORC_INVALID;
    double bbox[4], snap_sq, zlo, zhi;
    orc_compute_bbox(xs, ys, m, qx, qy, n, bbox);
    weighting_context(bbox, zs, m, &snap_sq, &zlo, &zhi);
    for (size_t i = 0; i < n; ++i) {
        pred[i] = variant == 0
                      ? predict_naive(qx[i], qy[i], xs, ys, zs, m, alphas[i], snap_sq, zlo, zhi)
                      : predict_blocked(qx[i], qy[i], xs, ys, zs, m, alphas[i], snap_sq, zlo, zhi);
    }
    return ORC_OK;
}

/* aidw_predict_all: interpolate.hpp:453-489, given per-query kNN averages.
 * list_len[i] / exhausted[i] describe each KnnResult.  alphas_out gets the
 * per-query alpha; *fail_index the smallest failing query. */
int orc_aidw_predict_all(const double* qx, const double* qy, size_t n, const double* xs,
                         const double* ys, const double* zs, size_t m, const double* r_obs,
                         const size_t* list_len, const int* exhausted, int k, double r_min,
                         double r_max, const double* lv, double area_param, int variant,
                         double* pred, double* alphas_out, int64_t* fail_index) {
    if (m == 0) return ORC_INVALID;
    if (!params_ok(k, r_min, r_max, lv)) return ORC_INVALID;
    double bbox[4];
    orc_compute_bbox(xs, ys, m, qx, qy, n, bbox);
    const double area = area_param > 0.0 ? area_param : (bbox[2] - bbox[0]) * (bbox[3] - bbox[1]);
    for (size_t i = 0; i < n; ++i) {
        double rec[5];
        const int rc = orc_adaptive_alpha(r_obs[i], list_len[i], exhausted[i], m, area, k, r_min,
                                          r_max, lv, rec);
        if (rc) {
            if (fail_index) *fail_index = (int64_t)i;
            return rc;
        }
        alphas_out[i] = rec[4];
    }
    return orc_predict_with_alphas(qx, qy, n, xs, ys, zs, m, alphas_out, variant, pred);
}

/* Clustered generator for BASELINE config 4 (the reference has
 * none).  B Gaussian blobs, centres in [0.1,0.9]^2 drawn from
 * mt19937_64(center_seed); per point: blob = rng() % B, Box–Muller with
 * sigma, reject outside the unit square, z = unit draw.  The product has its
 * own implementation (csrc/generate.cpp); this one pins it. */
int orc_generate_clustered(size_t count, int blobs, double sigma, uint64_t center_seed,
                           uint64_t seed, int with_values, double* xs, double* ys, double* zs) {
    if (count == 0 || blobs < 1 || !(sigma > 0.0)) return ORC_INVALID;
    orc_mt64 cg, g;
    mt64_seed(&cg, center_seed);
    double* cx = (double*)malloc((size_t)blobs * sizeof(double));
    double* cy = (double*)malloc((size_t)blobs * sizeof(double));
    for (int b = 0; b < blobs; ++b) {
        cx[b] = 0.1 + 0.8 * unit01(&cg);
        cy[b] = 0.1 + 0.8 * unit01(&cg);
    }
    mt64_seed(&g, seed);
    size_t i = 0;
    while (i < count) {
        const int b = (int)(mt64_next(&g) % (uint64_t)blobs);
        const double u1 = unit01(&g);
        const double u2 = unit01(&g);
        const double r = sqrt(-2.0 * log(1.0 - u1));
        const double t = 2.0 * kPi * u2;
        const double x = cx[b] + sigma * (r * cos(t));
        const double y = cy[b] + sigma * (r * sin(t));
        if (!(x >= 0.0 && x <= 1.0 && y >= 0.0 && y <= 1.0)) continue;
        xs[i] = x;
        ys[i] = y;
        if (with_values) zs[i] = unit01(&g);
        ++i;
    }
    free(cx);
    free(cy);
    return ORC_OK;
}

/* cmd_raster's query lattice (cli.hpp:495-507): nx x ny cell centres over
 * the data bbox, northernmost row first, row-major:
 *   sx = W / nx, sy = H / ny,
 *   x = min_x + (c + 0.5) sx,  y = min_y + ((ny - 1 - r) + 0.5) sy. */
int orc_raster_lattice(size_t nx, size_t ny, const double* bbox, double* xs, double* ys) {
    if (nx < 1 || ny < 1) return ORC_INVALID;
    const double sx = (bbox[2] - bbox[0]) / (double)nx;
    const double sy = (bbox[3] - bbox[1]) / (double)ny;
    size_t i = 0;
    for (size_t r = 0; r < ny; ++r) {
        const double y = bbox[1] + ((double)(ny - 1 - r) + 0.5) * sy;
        for (size_t c = 0; c < nx; ++c, ++i) {
            xs[i] = bbox[0] + ((double)c + 0.5) * sx;
            ys[i] = y;
        }
    }
    return 0;
}
