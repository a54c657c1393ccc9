/*
 * picoracle.c -- CPU restatement of the MatrixPIC deposition + cell-sort hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the sm_100a
 * product in paper_2601_08277_b200/.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it.  The product never links it and has
 * no CPU fallback.
 *
 * Every function restates the reference algorithm from the read-only tree at
 * /root/reference (header-only C++20 library `picdep`), citing file:line.  It
 * is pinned against the reference itself: tests/test_oracle.py checks it
 * bit-for-bit against oracle/_ref/libpicref.so (the reference headers compiled
 * by oracle/Makefile) and against the golden fixtures in tests/golden/.
 *
 * Floating point: plain IEEE mul/add in the reference's source order.  The
 * Makefile builds with -ffp-contract=off and no -march, matching the
 * reference's own Release build (proj/CMakeLists.txt:3-9).
 *
 * Order 2 (TSC) does not exist in the reference (proj/include/pic/shape.hpp:14
 * has only cic=1 and qsp=3).  po_shape_1d(order=2) is this project's own
 * restatement following the reference conventions (half-open frac, x-fastest
 * node order, periodic wrap, value order wq*(sx*(sy*sz))): parity for order 2
 * is against this restatement only ("unpinned by the reference").
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Same memory layout as picgpu_grid in include/picgpu.h. */
typedef struct {
    int32_t nx, ny, nz, pad;
    double dx, dy, dz;
    double ox, oy, oz;
} po_grid;

enum { PO_OK = 0, PO_EINVAL = 1, PO_ERANGE = 2, PO_ELENGTH = 3, PO_ELOGIC = 4, PO_EDOMAIN = 5 };

/* ---- rng: proj/include/pic/rng.hpp:12-34 -------------------------------- */

uint64_t po_hash_mix(uint64_t z) { /* rng.hpp:12-17 (SplitMix64 finalizer) */
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

uint64_t po_hash_combine(uint64_t seed, uint64_t stream, uint64_t counter) { /* rng.hpp:19-21 */
    return po_hash_mix(po_hash_mix(po_hash_mix(seed) ^ stream) ^ counter);
}

double po_uniform01(uint64_t seed, uint64_t stream, uint64_t counter) { /* rng.hpp:24-27 */
    const uint64_t bits = po_hash_combine(seed, stream, counter);
    return ((double)(bits >> 11) + 0.5) * 0x1.0p-53;
}

double po_gaussian(uint64_t seed, uint64_t stream, uint64_t counter) { /* rng.hpp:30-34 */
    const double u1 = po_uniform01(seed, stream, 2 * counter);
    const double u2 = po_uniform01(seed, stream, 2 * counter + 1);
    return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2);
}

/* ---- grid: proj/include/pic/grid.hpp ------------------------------------ */

static int po_wrap(int i, int n) { /* grid.hpp:64-67 */
    int r = i % n;
    return r < 0 ? r + n : r;
}

static uint32_t po_linear(const po_grid* g, int i, int j, int k) { /* grid.hpp:50-54 */
    return (uint32_t)i + (uint32_t)g->nx * ((uint32_t)j + (uint32_t)g->ny * (uint32_t)k);
}

static uint32_t po_node_id(const po_grid* g, int i, int j, int k) { /* grid.hpp:69-71 */
    return po_linear(g, po_wrap(i, g->nx), po_wrap(j, g->ny), po_wrap(k, g->nz));
}

/* grid.hpp:81-100: floor/frac with the half-open fix-up, fmod wrap outside the box. */
void po_locate_axis(double x, double origin, double spacing, int n, int* cell, double* frac) {
    const double u = (x - origin) / spacing;
    double fu = floor(u);
    double fr = u - fu;
    if (fr >= 1.0) {
        fr = 0.0;
        fu += 1.0;
    }
    if (fu >= 0.0 && fu < (double)n) {
        *cell = (int)fu;
        *frac = fr;
        return;
    }
    double c = fmod(fu, (double)n);
    if (c < 0.0) c += (double)n;
    int ci = (int)c;
    if (ci == n) ci = 0;
    *cell = ci;
    *frac = fr;
}

/* grid.hpp:106-113.  Returns PO_EINVAL for a non-finite position. */
int po_cell_of(const po_grid* g, double x, double y, double z, int32_t ijk[3], uint32_t* linear) {
    if (!isfinite(x) || !isfinite(y) || !isfinite(z)) return PO_EINVAL;
    double f;
    int i, j, k;
    po_locate_axis(x, g->ox, g->dx, g->nx, &i, &f);
    po_locate_axis(y, g->oy, g->dy, g->ny, &j, &f);
    po_locate_axis(z, g->oz, g->dz, g->nz, &k, &f);
    if (ijk) {
        ijk[0] = i;
        ijk[1] = j;
        ijk[2] = k;
    }
    if (linear) *linear = po_linear(g, i, j, k);
    return PO_OK;
}

/* ---- shape: proj/include/pic/shape.hpp ---------------------------------- */

int po_support(int order) { return order == 1 ? 2 : order == 2 ? 3 : 4; }

/* 1D weights for a particle with in-cell coordinate d in [0,1).
 * order 1: shape.hpp:26-29 (cic_shape_1d), base offset 0 (shape.hpp:78).
 * order 3: shape.hpp:33-43 (qsp_shape_1d), base offset -1 (shape.hpp:82).
 * order 2: this project's TSC restatement: nearest node j = cell + (d >= 0.5),
 *          delta = d - (d >= 0.5), taps j-1..j+1, base offset -1 + (d >= 0.5).
 * Returns PO_EINVAL when d is outside [0,1) (shape.hpp:20-22). */
int po_shape_1d(int order, double d, double out[4], int* base_off) {
    if (!(d >= 0.0 && d < 1.0)) return PO_EINVAL;
    out[0] = out[1] = out[2] = out[3] = 0.0;
    if (order == 1) {
        out[0] = 1.0 - d;
        out[1] = d;
        *base_off = 0;
    } else if (order == 3) {
        const double t = d;
        const double t2 = t * t;
        const double t3 = t2 * t;
        const double u = 1.0 - t;
        out[0] = u * u * u * (1.0 / 6.0);
        out[1] = (3.0 * t3 - 6.0 * t2 + 4.0) * (1.0 / 6.0);
        out[2] = (-3.0 * t3 + 3.0 * t2 + 3.0 * t + 1.0) * (1.0 / 6.0);
        out[3] = t3 * (1.0 / 6.0);
        *base_off = -1;
    } else if (order == 2) {
        const int up = d >= 0.5;
        const double dl = up ? d - 1.0 : d;
        const double a = 0.5 - dl;
        const double b = 0.5 + dl;
        out[0] = 0.5 * (a * a);
        out[1] = 0.75 - dl * dl;
        out[2] = 0.5 * (b * b);
        *base_off = up ? 0 : -1;
    } else {
        return PO_EINVAL;
    }
    return PO_OK;
}

typedef struct {
    double sx[4], sy[4], sz[4];
    int base[3];
} po_factors;

/* shape.hpp:64-85 (compute_shape_factors); base is unwrapped. */
static int po_factors_of(const po_grid* g, int order, double x, double y, double z, po_factors* f) {
    if (!isfinite(x) || !isfinite(y) || !isfinite(z)) return PO_EINVAL;
    int c[3], off[3];
    double fr[3];
    po_locate_axis(x, g->ox, g->dx, g->nx, &c[0], &fr[0]);
    po_locate_axis(y, g->oy, g->dy, g->ny, &c[1], &fr[1]);
    po_locate_axis(z, g->oz, g->dz, g->nz, &c[2], &fr[2]);
    int rc = po_shape_1d(order, fr[0], f->sx, &off[0]);
    if (!rc) rc = po_shape_1d(order, fr[1], f->sy, &off[1]);
    if (!rc) rc = po_shape_1d(order, fr[2], f->sz, &off[2]);
    if (rc) return rc;
    for (int a = 0; a < 3; ++a) f->base[a] = c[a] + off[a];
    return PO_OK;
}

/* Generic N-component scatter, deposit.hpp:31-58.  Per particle: kz, jy, ix
 * loops; syz = sy*sz, s = sx*syz, field += wq*s.  Visits particles in storage
 * order, or in the order given by `visit` (bin order, deposit.hpp:52-57). */
static int po_scatter(const po_grid* g, int order, uint64_t n, const double* x, const double* y,
                      const double* z, int ncomp, const double* const wq_src[3],
                      const double* wscale, double q, double* const fields[3],
                      const uint32_t* visit) {
    const int S = po_support(order);
    for (uint64_t t = 0; t < n; ++t) {
        const uint64_t p = visit ? visit[t] : t;
        po_factors f;
        int rc = po_factors_of(g, order, x[p], y[p], z[p], &f);
        if (rc) return rc;
        double wq[3];
        if (wscale) { /* particle_weights, shape.hpp:46-50: qw = q*W, then qw*v_c */
            const double qw = q * wscale[p];
            for (int c = 0; c < ncomp; ++c) wq[c] = qw * wq_src[c][p];
        } else { /* deposit_density, deposit.hpp:80-81: wq[0] = quantity[p] */
            for (int c = 0; c < ncomp; ++c) wq[c] = wq_src[c][p];
        }
        for (int kz = 0; kz < S; ++kz)
            for (int jy = 0; jy < S; ++jy) {
                const double syz = f.sy[jy] * f.sz[kz];
                for (int ix = 0; ix < S; ++ix) {
                    const double s = f.sx[ix] * syz;
                    const uint32_t node = po_node_id(g, f.base[0] + ix, f.base[1] + jy, f.base[2] + kz);
                    for (int c = 0; c < ncomp; ++c) fields[c][node] += wq[c] * s;
                }
            }
    }
    return PO_OK;
}

static uint64_t po_ncells(const po_grid* g) { return (uint64_t)g->nx * (uint64_t)g->ny * (uint64_t)g->nz; }

/* deposit_scalar, deposit.hpp:62-73.  Outputs are zeroed first (CurrentGrid(g)). */
int po_deposit_current(const po_grid* g, int order, const double* x, const double* y, const double* z,
                       const double* vx, const double* vy, const double* vz, const double* w, double q,
                       uint64_t n, const uint32_t* visit, double* jx, double* jy, double* jz) {
    const uint64_t nc = po_ncells(g);
    memset(jx, 0, nc * sizeof(double));
    memset(jy, 0, nc * sizeof(double));
    memset(jz, 0, nc * sizeof(double));
    const double* src[3] = {vx, vy, vz};
    double* const fields[3] = {jx, jy, jz};
    return po_scatter(g, order, n, x, y, z, 3, src, w, q, fields, visit);
}

/* deposit_density, deposit.hpp:76-83 (storage order only). */
int po_deposit_density(const po_grid* g, int order, const double* x, const double* y, const double* z,
                       const double* quantity, uint64_t n, double* rho) {
    memset(rho, 0, po_ncells(g) * sizeof(double));
    const double* src[3] = {quantity, 0, 0};
    double* const fields[3] = {rho, 0, 0};
    return po_scatter(g, order, n, x, y, z, 1, src, 0, 0.0, fields, 0);
}

/* Stable counting sort by linear cell id, gpma.hpp:379-394: counts ->
 * exclusive starts -> perm[cursor[cell[p]]++] = p, p ascending. */
int po_counting_sort(const po_grid* g, const double* x, const double* y, const double* z, uint64_t n,
                     uint32_t* perm, uint32_t* starts, uint32_t* counts) {
    const uint64_t nc = po_ncells(g);
    uint32_t* cells = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
    uint32_t* cursor = (uint32_t*)malloc(nc * sizeof(uint32_t));
    memset(counts, 0, nc * sizeof(uint32_t));
    for (uint64_t p = 0; p < n; ++p) {
        if (po_cell_of(g, x[p], y[p], z[p], 0, &cells[p])) {
            free(cells);
            free(cursor);
            return PO_EINVAL;
        }
        ++counts[cells[p]];
    }
    starts[0] = 0;
    for (uint64_t c = 1; c < nc; ++c) starts[c] = starts[c - 1] + counts[c - 1];
    memcpy(cursor, starts, nc * sizeof(uint32_t));
    for (uint64_t p = 0; p < n; ++p) perm[cursor[cells[p]]++] = (uint32_t)p;
    free(cells);
    free(cursor);
    return PO_OK;
}

/* workload.hpp:128-132 */
static double po_wrap_position(double x, double origin, double length) {
    double r = x - length * floor((x - origin) / length);
    if (r - origin >= length) r = origin;
    return r;
}

/* Ballistic push with periodic wrap and the single-cell cap, workload.hpp:139-155.
 * Returns PO_EDOMAIN if any particle exceeds the cap (reference throws
 * std::domain_error before touching that particle). *moved = number of
 * particles whose linear cell changed. */
int po_advance(const po_grid* g, double dt, double* x, double* y, double* z, const double* vx,
               const double* vy, const double* vz, uint64_t n, uint64_t* moved) {
    if (moved) *moved = 0;
    if (n == 0) return PO_OK;
    const double ms = fmin(g->dx, fmin(g->dy, g->dz));
    const double cap2 = (ms / dt) * (ms / dt);
    const double Lx = g->nx * g->dx, Ly = g->ny * g->dy, Lz = g->nz * g->dz;
    uint64_t m = 0;
    for (uint64_t p = 0; p < n; ++p) {
        const double v2 = vx[p] * vx[p] + vy[p] * vy[p] + vz[p] * vz[p];
        if (v2 > cap2) return PO_EDOMAIN;
        uint32_t before, after;
        if (po_cell_of(g, x[p], y[p], z[p], 0, &before)) return PO_EINVAL;
        x[p] = po_wrap_position(x[p] + vx[p] * dt, g->ox, Lx);
        y[p] = po_wrap_position(y[p] + vy[p] * dt, g->oy, Ly);
        z[p] = po_wrap_position(z[p] + vz[p] * dt, g->oz, Lz);
        if (po_cell_of(g, x[p], y[p], z[p], 0, &after)) return PO_EINVAL;
        if (after != before) ++m;
    }
    if (moved) *moved = m;
    return PO_OK;
}

/* Per-particle cell ids (the set-level oracle of the incremental sorter: a
 * correct GPMA's bins equal the rebinned map, test_gpma.cpp:395-412). */
int po_cells(const po_grid* g, const double* x, const double* y, const double* z, uint64_t n, uint32_t* cell) {
    for (uint64_t p = 0; p < n; ++p)
        if (po_cell_of(g, x[p], y[p], z[p], 0, &cell[p])) return PO_EINVAL;
    return PO_OK;
}

/* SURVEY 8(d) seeded plasma generator built on the reference counter RNG.
 * Cell-major (k, j, i), then p within the cell; pid is the running index.
 * x = ox + (i + U(seed,pid,6))*dx (y: counter 7, z: counter 8);
 * u_c = u_th * gaussian(seed, pid, c) (counters 0..5); gamma = sqrt(1+|u|^2);
 * v = u/gamma; w = 1/ppc; id = pid.  Arrays hold ncells*ppc entries. */
void po_make_plasma(const po_grid* g, int ppc, double u_th, uint64_t seed, double* x, double* y, double* z,
                    double* vx, double* vy, double* vz, double* w, uint64_t* id) {
    uint64_t pid = 0;
    const double wt = 1.0 / (double)ppc;
    for (int k = 0; k < g->nz; ++k)
        for (int j = 0; j < g->ny; ++j)
            for (int i = 0; i < g->nx; ++i)
                for (int p = 0; p < ppc; ++p, ++pid) {
                    x[pid] = g->ox + ((double)i + po_uniform01(seed, pid, 6)) * g->dx;
                    y[pid] = g->oy + ((double)j + po_uniform01(seed, pid, 7)) * g->dy;
                    z[pid] = g->oz + ((double)k + po_uniform01(seed, pid, 8)) * g->dz;
                    const double ux = u_th * po_gaussian(seed, pid, 0);
                    const double uy = u_th * po_gaussian(seed, pid, 1);
                    const double uz = u_th * po_gaussian(seed, pid, 2);
                    const double gam = sqrt(1.0 + ux * ux + uy * uy + uz * uz);
                    vx[pid] = ux / gam;
                    vy[pid] = uy / gam;
                    vz[pid] = uz / gam;
                    w[pid] = wt;
                    id[pid] = pid;
                }
}

/* Reference flop tally, deposit.hpp:336-345 (76 / 534).  Order 2 is this
 * project's tally with f_shape = 9: 9 + 27 + 4 + 9 + 7*27 = 238. */
int po_flop_count(int order) {
    if (order == 1) return 9 + 3 + 4 + 60;
    if (order == 3) return 9 + 57 + 4 + 464;
    if (order == 2) return 9 + 27 + 4 + 9 + 7 * 27;
    return -1;
}

/* should_global_sort, sort_policy.hpp:62-73.  Returns 0 none, 1 interval,
 * 2 rebuilds, 3 slot_ratio, 4 perf_degradation (SortReason order, :50). */
int po_should_global_sort(uint32_t steps_since_sort, uint64_t cumulative_local_rebuilds, double empty_slot_ratio,
                          double perf_metric, double baseline_perf, uint32_t sort_interval,
                          uint32_t min_sort_interval, uint32_t trigger_rebuild_count, double trigger_empty_ratio,
                          double trigger_full_ratio, int perf_enable, double perf_degrad) {
    if (steps_since_sort < min_sort_interval) return 0;
    if (steps_since_sort >= sort_interval) return 1;
    if (cumulative_local_rebuilds > trigger_rebuild_count) return 2;
    if (empty_slot_ratio < trigger_empty_ratio || empty_slot_ratio > trigger_full_ratio) return 3;
    if (perf_enable && baseline_perf > 0.0 && perf_metric < perf_degrad * baseline_perf) return 4;
    return 0;
}

/* ---- charge-conserving current (Esirkepov 2001) on the Yee grid ----------
 * NOT in the reference (its deposition is the direct collocated scatter,
 * deposit.hpp:60-73; SPEC.md:8 lists charge-conserving schemes as future
 * work): this restatement is the checker for this project's extension and is
 * UNPINNED by the reference.  Its own pin is the discrete continuity equation
 * (tests/test_esirkepov.py): with rho = q*w*S on the nodes (po_deposit_density),
 *   (rho(x1) - rho(x0)) / dt + div J = 0   to round-off.
 * Conventions: per axis the shape is po_shape_1d's (B-spline of the order,
 * nodes base + t); the old and new windows are merged into one of S+1 nodes
 * starting at lo = min(base0, base1) (a move of less than one cell shifts the
 * base by at most one); DS = S1 - S0 on it;
 *   Wx = DSx (S0y S0z + DSy S0z / 2 + S0y DSz / 2 + DSy DSz / 3)  (cyclic for y, z)
 * and J on the staggered faces is the running sum along its axis:
 *   jx[node(lo+i, j, k)] (the face between nodes lo+i and lo+i+1)
 *       += -q w (dx/dt) sum_{i' <= i} Wx(i', j, k).
 * x1 is the pushed position (it may have been wrapped): its cell step from x0
 * is taken on the periodic axis and must be -1, 0 or +1 (else PO_EDOMAIN). */
static int po_axis_window(double x0, double x1, double origin, double spacing, int n, int order, double s0[5],
                          double s1[5], int* lo) {
    int c0, c1, o0, o1;
    double f0, f1, a[4], b[4];
    po_locate_axis(x0, origin, spacing, n, &c0, &f0);
    po_locate_axis(x1, origin, spacing, n, &c1, &f1);
    int dc = c1 - c0;
    if (dc == n - 1) dc = -1; /* periodic: the step across the seam */
    else if (dc == 1 - n) dc = 1;
    if (dc < -1 || dc > 1) return PO_EDOMAIN;
    if (po_shape_1d(order, f0, a, &o0) || po_shape_1d(order, f1, b, &o1)) return PO_EINVAL;
    const int S = po_support(order);
    const int b0 = c0 + o0, b1 = c0 + dc + o1; /* unwrapped, relative to c0 */
    *lo = b0 < b1 ? b0 : b1;
    for (int t = 0; t < 5; ++t) s0[t] = s1[t] = 0.0;
    for (int t = 0; t < S; ++t) {
        s0[b0 - *lo + t] = a[t];
        s1[b1 - *lo + t] = b[t];
    }
    return PO_OK;
}

int po_deposit_esirkepov(const po_grid* g, int order, const double* x0, const double* y0, const double* z0,
                         const double* x1, const double* y1, const double* z1, const double* w, double q,
                         double dt, uint64_t n, double* jx, double* jy, double* jz) {
    const uint64_t nc = po_ncells(g);
    memset(jx, 0, nc * sizeof(double));
    memset(jy, 0, nc * sizeof(double));
    memset(jz, 0, nc * sizeof(double));
    if (!(dt > 0.0)) return PO_EINVAL;
    const int L = po_support(order) + 1;
    for (uint64_t p = 0; p < n; ++p) {
        if (!isfinite(x0[p]) || !isfinite(y0[p]) || !isfinite(z0[p]) || !isfinite(x1[p]) || !isfinite(y1[p]) ||
            !isfinite(z1[p]))
            return PO_EINVAL;
        double S0[3][5], S1[3][5], D[3][5];
        int lo[3];
        int rc = po_axis_window(x0[p], x1[p], g->ox, g->dx, g->nx, order, S0[0], S1[0], &lo[0]);
        if (!rc) rc = po_axis_window(y0[p], y1[p], g->oy, g->dy, g->ny, order, S0[1], S1[1], &lo[1]);
        if (!rc) rc = po_axis_window(z0[p], z1[p], g->oz, g->dz, g->nz, order, S0[2], S1[2], &lo[2]);
        if (rc) return rc;
        for (int a = 0; a < 3; ++a)
            for (int t = 0; t < 5; ++t) D[a][t] = S1[a][t] - S0[a][t];
        const double qw = q * w[p];
        const double cx = -qw * g->dx / dt, cy = -qw * g->dy / dt, cz = -qw * g->dz / dt;
        /* x faces: running sum over i for each (j, k) */
        for (int k = 0; k < L; ++k)
            for (int j = 0; j < L; ++j) {
                const double t = S0[1][j] * S0[2][k] + 0.5 * D[1][j] * S0[2][k] + 0.5 * S0[1][j] * D[2][k] +
                                 (1.0 / 3.0) * D[1][j] * D[2][k];
                double run = 0.0;
                for (int i = 0; i < L - 1; ++i) {
                    run += D[0][i] * t;
                    jx[po_node_id(g, lo[0] + i, lo[1] + j, lo[2] + k)] += cx * run;
                }
            }
        for (int k = 0; k < L; ++k)
            for (int i = 0; i < L; ++i) {
                const double t = S0[0][i] * S0[2][k] + 0.5 * D[0][i] * S0[2][k] + 0.5 * S0[0][i] * D[2][k] +
                                 (1.0 / 3.0) * D[0][i] * D[2][k];
                double run = 0.0;
                for (int j = 0; j < L - 1; ++j) {
                    run += D[1][j] * t;
                    jy[po_node_id(g, lo[0] + i, lo[1] + j, lo[2] + k)] += cy * run;
                }
            }
        for (int j = 0; j < L; ++j)
            for (int i = 0; i < L; ++i) {
                const double t = S0[0][i] * S0[1][j] + 0.5 * D[0][i] * S0[1][j] + 0.5 * S0[0][i] * D[1][j] +
                                 (1.0 / 3.0) * D[0][i] * D[1][j];
                double run = 0.0;
                for (int k = 0; k < L - 1; ++k) {
                    run += D[2][k] * t;
                    jz[po_node_id(g, lo[0] + i, lo[1] + j, lo[2] + k)] += cz * run;
                }
            }
    }
    return PO_OK;
}
