/* TEST INFRASTRUCTURE ONLY — C restatement of the reference `tetvol` path.
 *
 * This file is the CHECKER: tests/, smoke() and bench.py's cpu_baseline leg
 * load it (liboracle.so); the product library never links or calls it.
 * Parity of this restatement with the reference is pinned by
 * tests/test_oracle.py against oracle/_ref (the reference itself, compiled from
 * /root/reference) and against tests/golden/ fixtures.
 *
 * Arithmetic contract: all geometry in IEEE double with no
 * contraction (built with -ffp-contract=off), evaluation order exactly as the
 * reference source: dot = (a.x*b.x + a.y*b.y) + a.z*b.z (geometry.hpp:36).
 * Paths cited are relative to /root/reference/proj.
 */
#define _GNU_SOURCE
#include "tvo.h"

#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#include <unistd.h>

typedef __int128 i128;

static _Thread_local char g_err[256];
const char* tvo_last_error(void) { return g_err; }
static int set_err(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

/* ---------------------------------------------------------------- vec3 --- */
/* geometry.hpp:10-48 */
typedef struct { double x, y, z; } v3;
static inline v3 V(double x, double y, double z) { v3 r = {x, y, z}; return r; }
static inline v3 vadd(v3 a, v3 b) { return V(a.x + b.x, a.y + b.y, a.z + b.z); }
static inline v3 vsub(v3 a, v3 b) { return V(a.x - b.x, a.y - b.y, a.z - b.z); }
static inline v3 vmul(v3 a, double s) { return V(a.x * s, a.y * s, a.z * s); }
static inline v3 vdiv(v3 a, double s) { return V(a.x / s, a.y / s, a.z / s); }
static inline v3 vmulv(v3 a, v3 b) { return V(a.x * b.x, a.y * b.y, a.z * b.z); }
static inline v3 vneg(v3 a) { return V(-a.x, -a.y, -a.z); }
static inline double vdot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static inline v3 vcross(v3 a, v3 b) {
    return V(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
static inline double vlen(v3 a) { return sqrt(vdot(a, a)); }
static inline v3 vnorm(v3 a) {
    double l = vlen(a);
    return l > 0.0 ? vdiv(a, l) : V(0, 0, 0);
}
static inline double vcomp(v3 a, int i) { return i == 0 ? a.x : (i == 1 ? a.y : a.z); }
static inline double dmax(double a, double b) { return a < b ? b : a; } /* std::max */
static inline double dmin(double a, double b) { return b < a ? b : a; } /* std::min */
static inline double dclamp(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }
static inline v3 P(const double* p) { return V(p[0], p[1], p[2]); }

/* geometry.hpp:64-83 (ray: origin, dir, t_min, t_max) */
typedef struct { v3 o, d; double tmin, tmax; } ray_t;
static inline v3 ray_at(const ray_t* r, double t) { return vadd(r->o, vmul(r->d, t)); }
static int slab(const ray_t* r, double* t0, double* t1) {
    *t0 = r->tmin;
    *t1 = r->tmax;
    for (int a = 0; a < 3; ++a) {
        double o = vcomp(r->o, a), d = vcomp(r->d, a);
        if (d == 0.0) {
            if (o < 0.0 || o > 1.0) return 0;
            continue;
        }
        double inv = 1.0 / d;
        double ta = (0.0 - o) * inv, tb = (1.0 - o) * inv;
        if (ta > tb) { double s = ta; ta = tb; tb = s; }
        *t0 = dmax(*t0, ta);
        *t1 = dmin(*t1, tb);
        if (*t0 > *t1) return 0;
    }
    return 1;
}

/* ----------------------------------------------------------------- rng --- */
/* rng.hpp:10-26 */
uint64_t tvo_mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
typedef struct { uint64_t key, dim; } rng_t;
static inline void rng_init(rng_t* r, uint64_t seed, uint64_t pixel, uint64_t sample) {
    r->key = tvo_mix64(tvo_mix64(tvo_mix64(seed) ^ pixel) ^ sample);
    r->dim = 0;
}
static inline double rng_next(rng_t* r) {
    uint64_t h = tvo_mix64(r->key ^ (0xd1b54a32d192ed03ull * ++r->dim));
    return (double)(h >> 11) * 0x1.0p-53;
}
void tvo_rng_draws(uint64_t seed, uint64_t pixel, uint64_t sample, int n, double* out) {
    rng_t r;
    rng_init(&r, seed, pixel, sample);
    for (int i = 0; i < n; ++i) out[i] = rng_next(&r);
}

/* -------------------------------------------------------------- camera --- */
/* camera.cpp:12-45 */
typedef struct {
    v3 pos, fwd, up, right;
    double tan_half, aspect;
    int w, h;
    v3 pn[5];
    double pd[5];
} cam_t;
static const double kPi = 3.14159265358979323846;

static v3 cam_dir(const cam_t* c, double u, double v) {
    return vnorm(vadd(vadd(c->fwd, vmul(c->right, (2.0 * u - 1.0) * c->tan_half * c->aspect)),
                      vmul(c->up, (1.0 - 2.0 * v) * c->tan_half)));
}
static int cam_init(cam_t* c, const tvo_camera_desc* d) {
    if (d->width < 1 || d->height < 1) return set_err(TVO_ERR_CAMERA, "image dimensions must be positive");
    if (!(d->vfov > 0.0 && d->vfov < 180.0)) return set_err(TVO_ERR_CAMERA, "vfov must be in (0, 180) degrees");
    v3 f = P(d->fwd), up = P(d->up);
    if (vlen(f) == 0.0) return set_err(TVO_ERR_CAMERA, "forward vector must be nonzero");
    c->pos = P(d->pos);
    c->w = d->width;
    c->h = d->height;
    c->fwd = vnorm(f);
    v3 upo = vsub(up, vmul(c->fwd, vdot(up, c->fwd)));
    if (vlen(upo) < 1e-12) return set_err(TVO_ERR_CAMERA, "up vector is parallel to the view direction");
    c->up = vnorm(upo);
    c->right = vcross(c->up, c->fwd);
    c->tan_half = tan(d->vfov * kPi / 360.0);
    c->aspect = (double)c->w / c->h;
    v3 tl = cam_dir(c, 0, 0), tr = cam_dir(c, 1, 0), bl = cam_dir(c, 0, 1), br = cam_dir(c, 1, 1);
    c->pn[0] = c->fwd;
    c->pd[0] = vdot(c->fwd, c->pos) + 1e-4;
    v3 pairs[4][2] = {{tl, bl}, {br, tr}, {tr, tl}, {bl, br}};
    for (int i = 0; i < 4; ++i) {
        v3 n = vnorm(vcross(pairs[i][0], pairs[i][1]));
        if (vdot(n, c->fwd) < 0.0) n = vneg(n);
        c->pn[i + 1] = n;
        c->pd[i + 1] = vdot(n, c->pos);
    }
    return TVO_OK;
}
/* camera.cpp:47-55 */
static void cam_primary(const cam_t* c, int px, int py, double jx, double jy, ray_t* r) {
    double u = (px + jx) / c->w;
    double v = (py + jy) / c->h;
    r->o = c->pos;
    r->d = cam_dir(c, u, v);
    r->tmin = 0.0;
    r->tmax = INFINITY;
}
/* camera.cpp:57-68 */
static int cam_outside(const cam_t* c, const v3* cs) {
    for (int p = 0; p < 5; ++p) {
        int all_out = 1;
        for (int i = 0; i < 4; ++i)
            if (vdot(c->pn[p], cs[i]) >= c->pd[p]) { all_out = 0; break; }
        if (all_out) return 1;
    }
    return 0;
}
/* camera.cpp:70-85 */
static double cam_proj_size(const cam_t* c, const v3* cs) {
    static const int E[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
    double longest_sq = 0.0;
    for (int e = 0; e < 6; ++e) {
        v3 d = vsub(cs[E[e][0]], cs[E[e][1]]);
        longest_sq = dmax(longest_sq, vdot(d, d));
    }
    double longest = sqrt(longest_sq);
    v3 cen = vmul(vadd(vadd(vadd(cs[0], cs[1]), cs[2]), cs[3]), 0.25);
    double rsq = 0.0;
    for (int i = 0; i < 4; ++i) {
        v3 d = vsub(cs[i], cen);
        rsq = dmax(rsq, vdot(d, d));
    }
    v3 tc = vsub(cen, c->pos);
    if (vdot(tc, tc) <= rsq) return INFINITY;
    double dist = dmax(vlen(tc), 1e-4);
    return longest / (2.0 * dist * c->tan_half) * c->h;
}
int tvo_primary_ray(const tvo_camera_desc* d, int px, int py, double jx, double jy, double* out) {
    cam_t c;
    int rc = cam_init(&c, d);
    if (rc) return rc;
    ray_t r;
    cam_primary(&c, px, py, jx, jy, &r);
    out[0] = r.o.x, out[1] = r.o.y, out[2] = r.o.z, out[3] = r.d.x, out[4] = r.d.y, out[5] = r.d.z;
    return 0;
}
int tvo_camera_tet_tests(const tvo_camera_desc* d, const double* cs, double* out) {
    cam_t c;
    int rc = cam_init(&c, d);
    if (rc) return rc;
    v3 k[4] = {P(cs), P(cs + 3), P(cs + 6), P(cs + 9)};
    out[0] = cam_outside(&c, k);
    out[1] = cam_proj_size(&c, k);
    return 0;
}

/* ---------------------------------------------------------- generators --- */
/* cli.cpp:317-321 */
static double blob_density(v3 p) {
    v3 d = vsub(p, V(0.5, 0.5, 0.5));
    double t = dmax(0.0, 1.0 - vdot(d, d) / (0.45 * 0.45));
    return t * t;
}
/* cli.cpp:323-346, generalised to (cells, seed) as SURVEY.md 8(d) defines */
static double vnoise(v3 p, int cells, uint64_t seed) {
    double x = dclamp(p.x, 0.0, 1.0) * cells, y = dclamp(p.y, 0.0, 1.0) * cells, z = dclamp(p.z, 0.0, 1.0) * cells;
    int ix = (int)x < cells - 1 ? (int)x : cells - 1;
    int iy = (int)y < cells - 1 ? (int)y : cells - 1;
    int iz = (int)z < cells - 1 ? (int)z : cells - 1;
    double fx = x - ix, fy = y - iy, fz = z - iz, v = 0.0;
    for (int dz = 0; dz < 2; ++dz)
        for (int dy = 0; dy < 2; ++dy)
            for (int dx = 0; dx < 2; ++dx) {
                double w = (dx ? fx : 1.0 - fx) * (dy ? fy : 1.0 - fy) * (dz ? fz : 1.0 - fz);
                uint64_t h = tvo_mix64(tvo_mix64(tvo_mix64(seed ^ (uint64_t)(int64_t)(ix + dx)) ^
                                                 (uint64_t)(int64_t)(iy + dy)) ^
                                       (uint64_t)(int64_t)(iz + dz));
                v += w * ((double)(h >> 11) * 0x1.0p-53);
            }
    return v;
}
static const uint64_t kNoiseSeed = 0x5eb0a8a5c9d3f1adull;
static double cloud_density(v3 p) {
    double s = 0.0;
    for (int o = 0; o < 4; ++o) s += ldexp(1.0, -(o + 1)) * vnoise(p, 8 << o, kNoiseSeed + (uint64_t)o);
    double c = dmax(0.0, s - 0.35);
    return c * 2.0 * blob_density(p) / 0.9375;
}
void tvo_gen_volume(int kind, int nx, int ny, int nz, double value, float* out) {
    for (int k = 0; k < nz; ++k)
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i) {
                v3 p = V((i + 0.5) / nx, (j + 0.5) / ny, (k + 0.5) / nz); /* volume.hpp:44-46 */
                double d = 0.0;
                switch (kind) {
                    case 0: d = value; break;
                    case 1: d = p.x; break;
                    case 2: d = blob_density(p); break;
                    case 3: d = p.x < 0.5 ? 1.0 : 0.0; break;
                    case 4: d = vnoise(p, 8, kNoiseSeed); break;
                    default: d = cloud_density(p); break;
                }
                out[((size_t)k * ny + j) * nx + i] = (float)d;
            }
}

/* ---------------------------------------------------------- hash table --- */
/* Open addressing, linear probing, backward-shift deletion. Keys are 3 u32. */
typedef struct { uint32_t k0, k1, k2, used; uint32_t v0, v1, v2, pad; } hslot;
typedef struct { hslot* s; size_t cap, n; } htab;
static uint64_t hkey(uint32_t a, uint32_t b, uint32_t c) {
    return tvo_mix64(((uint64_t)a << 32 | b) ^ tvo_mix64(c + 0x51ull));
}
static void ht_init(htab* t, size_t cap) {
    size_t c = 64;
    while (c < cap * 2) c <<= 1;
    t->s = (hslot*)calloc(c, sizeof(hslot));
    t->cap = c;
    t->n = 0;
}
static void ht_free(htab* t) { free(t->s); t->s = NULL; t->cap = t->n = 0; }
static hslot* ht_find(const htab* t, uint32_t a, uint32_t b, uint32_t c) {
    size_t m = t->cap - 1, i = hkey(a, b, c) & m;
    for (;;) {
        hslot* s = &t->s[i];
        if (!s->used) return NULL;
        if (s->k0 == a && s->k1 == b && s->k2 == c) return s;
        i = (i + 1) & m;
    }
}
static hslot* ht_insert(htab* t, uint32_t a, uint32_t b, uint32_t c, int* fresh);
static void ht_grow(htab* t) {
    htab n;
    ht_init(&n, t->cap);
    for (size_t i = 0; i < t->cap; ++i)
        if (t->s[i].used) {
            int f;
            hslot* d = ht_insert(&n, t->s[i].k0, t->s[i].k1, t->s[i].k2, &f);
            d->v0 = t->s[i].v0, d->v1 = t->s[i].v1, d->v2 = t->s[i].v2;
        }
    free(t->s);
    *t = n;
}
static hslot* ht_insert(htab* t, uint32_t a, uint32_t b, uint32_t c, int* fresh) {
    if ((t->n + 1) * 2 > t->cap) ht_grow(t);
    size_t m = t->cap - 1, i = hkey(a, b, c) & m;
    for (;;) {
        hslot* s = &t->s[i];
        if (!s->used) {
            s->used = 1, s->k0 = a, s->k1 = b, s->k2 = c, s->v0 = s->v1 = s->v2 = 0;
            t->n++;
            *fresh = 1;
            return s;
        }
        if (s->k0 == a && s->k1 == b && s->k2 == c) { *fresh = 0; return s; }
        i = (i + 1) & m;
    }
}
static void ht_erase(htab* t, hslot* s) {
    size_t m = t->cap - 1, i = (size_t)(s - t->s), j = i;
    t->s[i].used = 0;
    t->n--;
    for (;;) {
        j = (j + 1) & m;
        if (!t->s[j].used) return;
        size_t h = hkey(t->s[j].k0, t->s[j].k1, t->s[j].k2) & m;
        /* move j back to i when its home h is not in (i, j] cyclically */
        int in_range = (i <= j) ? (h > i && h <= j) : (h > i || h <= j);
        if (!in_range) {
            t->s[i] = t->s[j];
            t->s[j].used = 0;
            i = j;
        }
    }
}

/* ---------------------------------------------------------------- grid --- */
typedef struct { uint32_t* ids; uint32_t n, cap; } ring_t;

struct tvo_grid {
    uint32_t* vq; /* 3 per vertex */
    size_t nv, cap_v;
    tvo_tet* tets;
    size_t nt, cap_t;
    uint32_t roots[24];
    int max_level;
    size_t leaf_count;
    htab vlook; /* (x,y,z) -> v0 = vertex id */
    htab faces; /* sorted vids -> v0 = tet0, v1 = tet1, v2 = slot0 | slot1 << 8 | n << 16 */
    htab edges; /* (a,b,0) -> v0 = ring index */
    ring_t* rings;
    size_t nrings, cap_rings;
    uint32_t* free_rings;
    size_t nfree, cap_free;
};

static const int kEP[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
static const double kS = 0x1.6a09e667f3bccp-1; /* 1.0 / std::sqrt(2.0), tet_grid.cpp:33 */
/* tet_grid.cpp:31-47 */
static const double kTable[18][3] = {
    {1, 0, 0},     {-1, 0, 0},   {0, 1, 0},     {0, -1, 0},   {0, 0, 1},     {0, 0, -1},
    {kS, kS, 0},   {-kS, -kS, 0}, {kS, -kS, 0}, {-kS, kS, 0}, {kS, 0, kS},   {-kS, 0, -kS},
    {kS, 0, -kS},  {-kS, 0, kS}, {0, kS, kS},   {0, -kS, -kS}, {0, kS, -kS}, {0, -kS, kS},
};
static inline v3 tabn(int id) { return V(kTable[id][0], kTable[id][1], kTable[id][2]); }

static inline v3 vpos(const tvo_grid* g, uint32_t v) { /* tet_grid.hpp:44-47 */
    const double inv = 1.0 / (double)TVO_COORD_ONE;
    return V(g->vq[3 * v] * inv, g->vq[3 * v + 1] * inv, g->vq[3 * v + 2] * inv);
}

static tvo_grid* grid_new(void) {
    tvo_grid* g = (tvo_grid*)calloc(1, sizeof(tvo_grid));
    ht_init(&g->vlook, 1024);
    ht_init(&g->faces, 1024);
    ht_init(&g->edges, 1024);
    g->max_level = TVO_LEVEL_CAP;
    return g;
}
void tvo_grid_free(tvo_grid* g) {
    if (!g) return;
    free(g->vq);
    free(g->tets);
    ht_free(&g->vlook);
    ht_free(&g->faces);
    ht_free(&g->edges);
    for (size_t i = 0; i < g->nrings; ++i) free(g->rings[i].ids);
    free(g->rings);
    free(g->free_rings);
    free(g);
}

static uint32_t push_vertex(tvo_grid* g, uint32_t x, uint32_t y, uint32_t z) {
    if (g->nv == g->cap_v) {
        g->cap_v = g->cap_v ? 2 * g->cap_v : 256;
        g->vq = (uint32_t*)realloc(g->vq, g->cap_v * 3 * sizeof(uint32_t));
    }
    g->vq[3 * g->nv] = x, g->vq[3 * g->nv + 1] = y, g->vq[3 * g->nv + 2] = z;
    return (uint32_t)g->nv++;
}
/* tet_grid.cpp:94-102 */
static uint32_t intern_vertex(tvo_grid* g, uint32_t x, uint32_t y, uint32_t z) {
    int fresh;
    hslot* s = ht_insert(&g->vlook, x, y, z, &fresh);
    if (!fresh) return s->v0;
    uint32_t id = push_vertex(g, x, y, z);
    s = ht_find(&g->vlook, x, y, z); /* insert may have rehashed nothing, but be safe */
    s->v0 = id;
    return id;
}
static uint32_t push_tet(tvo_grid* g, const tvo_tet* t) {
    if (g->nt == g->cap_t) {
        g->cap_t = g->cap_t ? 2 * g->cap_t : 256;
        g->tets = (tvo_tet*)realloc(g->tets, g->cap_t * sizeof(tvo_tet));
    }
    g->tets[g->nt] = *t;
    return (uint32_t)g->nt++;
}

/* tet_grid.cpp:14-25 */
static i128 det_fixed(const uint32_t* v0, const uint32_t* v1, const uint32_t* v2, const uint32_t* v3) {
    int64_t a[3], b[3], c[3];
    for (int k = 0; k < 3; ++k) {
        a[k] = (int64_t)v1[k] - v0[k];
        b[k] = (int64_t)v2[k] - v0[k];
        c[k] = (int64_t)v3[k] - v0[k];
    }
    int64_t m0 = b[1] * c[2] - b[2] * c[1], m1 = b[2] * c[0] - b[0] * c[2], m2 = b[0] * c[1] - b[1] * c[0];
    return (i128)a[0] * m0 + (i128)a[1] * m1 + (i128)a[2] * m2;
}

/* tet_grid.cpp:49-80; returns 0..17 or -1 (NotCanonical) */
static int face_normal_id(const uint32_t* a, const uint32_t* b, const uint32_t* c, const uint32_t* in) {
    int64_t u[3], v[3];
    for (int k = 0; k < 3; ++k) {
        u[k] = (int64_t)b[k] - a[k];
        v[k] = (int64_t)c[k] - a[k];
    }
    int64_t n[3] = {u[1] * v[2] - u[2] * v[1], u[2] * v[0] - u[0] * v[2], u[0] * v[1] - u[1] * v[0]};
    if (n[0] == 0 && n[1] == 0 && n[2] == 0) return -1;
    i128 side = 0;
    for (int k = 0; k < 3; ++k) side += (i128)n[k] * ((int64_t)in[k] - a[k]);
    if (side == 0) return -1;
    if (side > 0)
        for (int k = 0; k < 3; ++k) n[k] = -n[k];
    int zeros = (n[0] == 0) + (n[1] == 0) + (n[2] == 0);
    if (zeros == 2) {
        for (int k = 0; k < 3; ++k)
            if (n[k] != 0) return 2 * k + (n[k] > 0 ? 0 : 1);
    } else if (zeros == 1) {
        int zk = n[0] == 0 ? 0 : (n[1] == 0 ? 1 : 2);
        int i = zk == 0 ? 1 : 0, j = zk == 2 ? 1 : 2;
        if (llabs(n[i]) != llabs(n[j])) return -1;
        int base = zk == 2 ? 6 : (zk == 1 ? 10 : 14);
        int pi = n[i] > 0, pj = n[j] > 0;
        if (pi && pj) return base;
        if (!pi && !pj) return base + 1;
        if (pi && !pj) return base + 2;
        return base + 3;
    }
    return -1;
}

/* tet_grid.cpp:119-128 */
static int compute_normals(tvo_grid* g, uint32_t t) {
    tvo_tet* tt = &g->tets[t];
    for (int slot = 0; slot < 4; ++slot) {
        const uint32_t* f[3];
        int n = 0;
        for (int s = 0; s < 4; ++s)
            if (s != slot) f[n++] = &g->vq[3 * tt->verts[s]];
        int id = face_normal_id(f[0], f[1], f[2], &g->vq[3 * tt->verts[slot]]);
        if (id < 0) return set_err(TVO_ERR_GRID, "normal direction not in table");
        tt->normal_ids[slot] = (uint8_t)id;
    }
    return 0;
}

static void face_key(const tvo_grid* g, uint32_t t, int slot, uint32_t* k) {
    const uint32_t* v = g->tets[t].verts;
    int n = 0;
    for (int s = 0; s < 4; ++s)
        if (s != slot) k[n++] = v[s];
    /* sort 3 */
    if (k[0] > k[1]) { uint32_t x = k[0]; k[0] = k[1]; k[1] = x; }
    if (k[1] > k[2]) { uint32_t x = k[1]; k[1] = k[2]; k[2] = x; }
    if (k[0] > k[1]) { uint32_t x = k[0]; k[0] = k[1]; k[1] = x; }
}

static ring_t* ring_get(tvo_grid* g, uint32_t a, uint32_t b, int create) {
    if (a > b) { uint32_t x = a; a = b; b = x; }
    hslot* s = ht_find(&g->edges, a, b, 0);
    if (s) return &g->rings[s->v0];
    if (!create) return NULL;
    uint32_t ri;
    if (g->nfree) {
        ri = g->free_rings[--g->nfree];
    } else {
        if (g->nrings == g->cap_rings) {
            g->cap_rings = g->cap_rings ? 2 * g->cap_rings : 256;
            g->rings = (ring_t*)realloc(g->rings, g->cap_rings * sizeof(ring_t));
        }
        ri = (uint32_t)g->nrings++;
        g->rings[ri].ids = NULL;
        g->rings[ri].cap = 0;
    }
    g->rings[ri].n = 0;
    int fresh;
    s = ht_insert(&g->edges, a, b, 0, &fresh);
    s->v0 = ri;
    return &g->rings[ri];
}
static void ring_push(ring_t* r, uint32_t t) {
    if (r->n == r->cap) {
        r->cap = r->cap ? 2 * r->cap : 8;
        r->ids = (uint32_t*)realloc(r->ids, r->cap * sizeof(uint32_t));
    }
    r->ids[r->n++] = t;
}

/* tet_grid.cpp:130-152 */
static int register_leaf(tvo_grid* g, uint32_t t) {
    for (int slot = 0; slot < 4; ++slot) {
        uint32_t k[3];
        face_key(g, t, slot, k);
        int fresh;
        hslot* e = ht_insert(&g->faces, k[0], k[1], k[2], &fresh);
        uint32_t n = e->v2 >> 16;
        if (n == 0) {
            e->v0 = t;
            e->v2 = (uint32_t)slot | (1u << 16);
            g->tets[t].neighbors[slot] = TVO_NO_TET;
        } else if (n == 1) {
            e->v1 = t;
            e->v2 = (e->v2 & 0xffu) | ((uint32_t)slot << 8) | (2u << 16);
            g->tets[t].neighbors[slot] = e->v0;
            g->tets[e->v0].neighbors[e->v2 & 0xffu] = t;
        } else {
            return set_err(TVO_ERR_GRID, "face already shared by two leaves");
        }
    }
    for (int p = 0; p < 6; ++p)
        ring_push(ring_get(g, g->tets[t].verts[kEP[p][0]], g->tets[t].verts[kEP[p][1]], 1), t);
    g->leaf_count++;
    return 0;
}

/* tet_grid.cpp:154-182 */
static int unregister_leaf(tvo_grid* g, uint32_t t) {
    for (int slot = 0; slot < 4; ++slot) {
        uint32_t k[3];
        face_key(g, t, slot, k);
        hslot* e = ht_find(&g->faces, k[0], k[1], k[2]);
        if (!e) return set_err(TVO_ERR_GRID, "face map entry missing");
        uint32_t n = e->v2 >> 16;
        if (n == 2) {
            uint32_t s0 = e->v2 & 0xffu, s1 = (e->v2 >> 8) & 0xffu;
            int keep = (e->v0 == t && s0 == (uint32_t)slot) ? 1 : 0;
            uint32_t other = keep ? e->v1 : e->v0;
            uint32_t os = keep ? s1 : s0;
            e->v0 = other;
            e->v2 = os | (1u << 16);
            g->tets[other].neighbors[os] = TVO_NO_TET;
        } else {
            ht_erase(&g->faces, e);
        }
    }
    for (int p = 0; p < 6; ++p) {
        uint32_t a = g->tets[t].verts[kEP[p][0]], b = g->tets[t].verts[kEP[p][1]];
        if (a > b) { uint32_t x = a; a = b; b = x; }
        hslot* s = ht_find(&g->edges, a, b, 0);
        if (!s) return set_err(TVO_ERR_GRID, "edge map entry missing");
        uint32_t ri = s->v0;
        ring_t* r = &g->rings[ri];
        uint32_t w = 0;
        for (uint32_t i = 0; i < r->n; ++i)
            if (r->ids[i] != t) r->ids[w++] = r->ids[i];
        r->n = w;
        if (w == 0) {
            ht_erase(&g->edges, s);
            if (g->nfree == g->cap_free) {
                g->cap_free = g->cap_free ? 2 * g->cap_free : 256;
                g->free_rings = (uint32_t*)realloc(g->free_rings, g->cap_free * sizeof(uint32_t));
            }
            g->free_rings[g->nfree++] = ri;
        }
    }
    for (int i = 0; i < 4; ++i) g->tets[t].neighbors[i] = TVO_NO_TET;
    g->leaf_count--;
    return 0;
}

static tvo_tet blank_tet(void) {
    tvo_tet t;
    memset(&t, 0, sizeof t);
    t.children[0] = t.children[1] = t.parent = TVO_NO_TET;
    for (int i = 0; i < 4; ++i) t.neighbors[i] = TVO_NO_TET;
    return t;
}

/* tet_grid.cpp:184-233 */
tvo_grid* tvo_grid_init_roots(int max_level) {
    if (max_level < 1 || max_level > TVO_LEVEL_CAP) {
        set_err(TVO_ERR_GRID, "max_level out of range");
        return NULL;
    }
    tvo_grid* g = grid_new();
    g->max_level = max_level;
    const uint32_t S = TVO_COORD_ONE, H = S / 2;
    uint32_t center = intern_vertex(g, H, H, H);
    int ri = 0;
    for (int axis = 0; axis < 3; ++axis)
        for (int side = 0; side < 2; ++side) {
            uint32_t fc[3] = {H, H, H};
            fc[axis] = side ? S : 0;
            uint32_t fcv = intern_vertex(g, fc[0], fc[1], fc[2]);
            int u = axis == 0 ? 1 : 0, w = axis == 2 ? 1 : 2;
            static const uint32_t ring[4][2] = {{0, 0}, {1, 0}, {1, 1}, {0, 1}};
            uint32_t corner[4];
            for (int k = 0; k < 4; ++k) {
                uint32_t c[3] = {0, 0, 0};
                c[axis] = side ? S : 0;
                c[u] = ring[k][0] * S;
                c[w] = ring[k][1] * S;
                corner[k] = intern_vertex(g, c[0], c[1], c[2]);
            }
            for (int k = 0; k < 4; ++k) {
                uint32_t p = corner[k], q = corner[(k + 1) % 4];
                if (det_fixed(&g->vq[3 * p], &g->vq[3 * fcv], &g->vq[3 * center], &g->vq[3 * q]) < 0) {
                    uint32_t x = p; p = q; q = x;
                }
                tvo_tet t = blank_tet();
                t.verts[0] = p, t.verts[1] = fcv, t.verts[2] = center, t.verts[3] = q;
                g->roots[ri++] = push_tet(g, &t);
            }
        }
    for (int i = 0; i < 24; ++i) {
        if (compute_normals(g, g->roots[i]) || register_leaf(g, g->roots[i])) {
            tvo_grid_free(g);
            return NULL;
        }
    }
    return g;
}

/* tet_grid.cpp:235-262 (stored neighbour links are trusted) */
tvo_grid* tvo_grid_from_pools(const uint32_t* vq, uint64_t nv, const tvo_tet* tets, uint64_t nt,
                              const uint32_t* roots, int max_level) {
    tvo_grid* g = grid_new();
    g->max_level = max_level;
    for (uint64_t i = 0; i < nv; ++i) {
        int fresh;
        uint32_t id = push_vertex(g, vq[3 * i], vq[3 * i + 1], vq[3 * i + 2]);
        hslot* s = ht_insert(&g->vlook, vq[3 * i], vq[3 * i + 1], vq[3 * i + 2], &fresh);
        if (fresh) s->v0 = id;
    }
    for (uint64_t i = 0; i < nt; ++i) push_tet(g, &tets[i]);
    memcpy(g->roots, roots, sizeof g->roots);
    for (uint32_t t = 0; t < nt; ++t) {
        if (g->tets[t].children[0] != TVO_NO_TET) continue;
        g->leaf_count++;
        for (int p = 0; p < 6; ++p)
            ring_push(ring_get(g, g->tets[t].verts[kEP[p][0]], g->tets[t].verts[kEP[p][1]], 1), t);
        for (int slot = 0; slot < 4; ++slot) {
            uint32_t k[3];
            face_key(g, t, slot, k);
            int fresh;
            hslot* e = ht_insert(&g->faces, k[0], k[1], k[2], &fresh);
            uint32_t n = e->v2 >> 16;
            if (n == 0) e->v0 = t, e->v2 = (uint32_t)slot | (1u << 16);
            else if (n == 1) e->v1 = t, e->v2 = (e->v2 & 0xffu) | ((uint32_t)slot << 8) | (2u << 16);
            else e->v2 += 1u << 16;
        }
    }
    return g;
}

void tvo_grid_counts(const tvo_grid* g, uint64_t* out) {
    out[0] = g->nv, out[1] = g->nt, out[2] = g->leaf_count, out[3] = (uint64_t)g->max_level;
}
void tvo_grid_export(const tvo_grid* g, uint32_t* vq, tvo_tet* tets, uint32_t* roots) {
    if (vq) memcpy(vq, g->vq, g->nv * 3 * sizeof(uint32_t));
    if (tets) memcpy(tets, g->tets, g->nt * sizeof(tvo_tet));
    if (roots) memcpy(roots, g->roots, sizeof g->roots);
}
void tvo_grid_fill_density(tvo_grid* g, float lambda) {
    for (size_t t = 0; t < g->nt; ++t)
        if (g->tets[t].children[0] == TVO_NO_TET) g->tets[t].density = lambda, g->tets[t].mask = 1;
}

/* tet_grid.cpp:288-330 */
static void refinement_edge_slots(const tvo_grid* g, uint32_t t, int* s0, int* s1) {
    const uint32_t* v = g->tets[t].verts;
    int best = 0;
    uint64_t best_len = 0;
    uint32_t bmin = 0, bmax = 0;
    for (int e = 0; e < 6; ++e) {
        const uint32_t* qa = &g->vq[3 * v[kEP[e][0]]];
        const uint32_t* qb = &g->vq[3 * v[kEP[e][1]]];
        uint64_t L = 0;
        for (int k = 0; k < 3; ++k) {
            int64_t d = (int64_t)qa[k] - qb[k];
            L += (uint64_t)(d * d);
        }
        uint32_t a = v[kEP[e][0]], b = v[kEP[e][1]];
        uint32_t mn = a < b ? a : b, mx = a < b ? b : a;
        int better;
        if (e == 0) better = 1;
        else if (L != best_len) better = L > best_len;
        else better = mn < bmin || (mn == bmin && mx < bmax);
        if (better) best = e, best_len = L, bmin = mn, bmax = mx;
    }
    *s0 = kEP[best][0];
    *s1 = kEP[best][1];
}
static void refinement_edge(const tvo_grid* g, uint32_t t, uint32_t* a, uint32_t* b) {
    int s0, s1;
    refinement_edge_slots(g, t, &s0, &s1);
    uint32_t x = g->tets[t].verts[s0], y = g->tets[t].verts[s1];
    *a = x < y ? x : y;
    *b = x < y ? y : x;
}

/* tet_grid.cpp:339-382 */
static int bisect(tvo_grid* g, uint32_t t, uint32_t* ca, uint32_t* cb) {
    if (t >= g->nt) return set_err(TVO_ERR_GRID, "bisect: bad tet id");
    if (g->tets[t].children[0] != TVO_NO_TET) return set_err(TVO_ERR_GRID, "bisect: tet is not a leaf");
    if (g->tets[t].level >= g->max_level) return set_err(TVO_ERR_GRID, "bisect: level cap reached");
    int s0, s1;
    refinement_edge_slots(g, t, &s0, &s1);
    tvo_tet parent = g->tets[t];
    uint32_t vi = parent.verts[s0], vj = parent.verts[s1], mid[3];
    for (int k = 0; k < 3; ++k) {
        uint64_t s = (uint64_t)g->vq[3 * vi + k] + g->vq[3 * vj + k];
        if (s & 1u) return set_err(TVO_ERR_GRID, "bisect: midpoint not representable");
        mid[k] = (uint32_t)(s / 2);
    }
    uint32_t vm = intern_vertex(g, mid[0], mid[1], mid[2]);
    int rc = unregister_leaf(g, t);
    if (rc) return rc;
    parent = g->tets[t];
    tvo_tet a = parent, b = parent;
    a.verts[s1] = vm;
    b.verts[s0] = vm;
    tvo_tet* cs[2] = {&a, &b};
    for (int i = 0; i < 2; ++i) {
        tvo_tet* c = cs[i];
        c->parent = t;
        c->children[0] = c->children[1] = TVO_NO_TET;
        for (int k = 0; k < 4; ++k) c->neighbors[k] = TVO_NO_TET;
        c->level = (uint8_t)(parent.level + 1);
        c->density = c->temperature = c->albedo = 0.0f;
        c->mask = 0;
    }
    uint32_t ida = push_tet(g, &a), idb = push_tet(g, &b);
    g->tets[t].children[0] = ida;
    g->tets[t].children[1] = idb;
    if ((rc = compute_normals(g, ida)) || (rc = compute_normals(g, idb)) || (rc = register_leaf(g, ida)) ||
        (rc = register_leaf(g, idb)))
        return rc;
    *ca = ida;
    *cb = idb;
    return 0;
}

typedef struct { uint32_t* v; size_t n, cap; } u32vec;
static void uv_push(u32vec* a, uint32_t x) {
    if (a->n == a->cap) {
        a->cap = a->cap ? 2 * a->cap : 64;
        a->v = (uint32_t*)realloc(a->v, a->cap * sizeof(uint32_t));
    }
    a->v[a->n++] = x;
}
static int cmp_u32(const void* a, const void* b) {
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x < y ? -1 : (x > y);
}

/* tet_grid.cpp:397-426 */
static int refine_edge_recursive(tvo_grid* g, uint32_t a, uint32_t b, u32vec* out, int depth) {
    if (depth > 2 * TVO_LEVEL_CAP) return set_err(TVO_ERR_GRID, "conforming propagation exceeded its depth bound");
    uint32_t ea = a < b ? a : b, eb = a < b ? b : a;
    for (;;) {
        ring_t* r = ring_get(g, ea, eb, 0);
        if (!r) return 0;
        uint32_t n = r->n;
        uint32_t* ring = (uint32_t*)malloc(n * sizeof(uint32_t));
        memcpy(ring, r->ids, n * sizeof(uint32_t));
        qsort(ring, n, sizeof(uint32_t), cmp_u32);
        uint32_t* pending = (uint32_t*)malloc(n * sizeof(uint32_t));
        uint32_t np = 0;
        for (uint32_t i = 0; i < n; ++i) {
            uint32_t ra, rb;
            refinement_edge(g, ring[i], &ra, &rb);
            if (ra != ea || rb != eb) pending[np++] = ring[i];
        }
        int rc = 0;
        if (np == 0) {
            for (uint32_t i = 0; i < n && !rc; ++i) {
                uint32_t c0, c1;
                rc = bisect(g, ring[i], &c0, &c1);
                if (!rc) uv_push(out, c0), uv_push(out, c1);
            }
            free(ring);
            free(pending);
            return rc;
        }
        for (uint32_t i = 0; i < np && !rc; ++i) {
            if (g->tets[pending[i]].children[0] != TVO_NO_TET) continue;
            uint32_t ra, rb;
            refinement_edge(g, pending[i], &ra, &rb);
            rc = refine_edge_recursive(g, ra, rb, out, depth + 1);
        }
        free(ring);
        free(pending);
        if (rc) return rc;
    }
}

/* tet_grid.cpp:384-395; out receives the sorted unique fresh leaves */
static int refine_conforming(tvo_grid* g, uint32_t t, u32vec* out) {
    if (t >= g->nt) return set_err(TVO_ERR_GRID, "refine_conforming: bad tet id");
    if (g->tets[t].children[0] != TVO_NO_TET) return set_err(TVO_ERR_GRID, "refine_conforming: tet is not a leaf");
    if (g->tets[t].level >= g->max_level) return set_err(TVO_ERR_GRID, "refine_conforming: level cap reached");
    uint32_t a, b;
    refinement_edge(g, t, &a, &b);
    u32vec created = {0};
    int rc = refine_edge_recursive(g, a, b, &created, 0);
    if (!rc && out) {
        qsort(created.v, created.n, sizeof(uint32_t), cmp_u32);
        for (size_t i = 0; i < created.n; ++i) {
            if (i && created.v[i] == created.v[i - 1]) continue;
            if (g->tets[created.v[i]].children[0] != TVO_NO_TET) continue;
            uv_push(out, created.v[i]);
        }
    }
    free(created.v);
    return rc;
}
int tvo_grid_refine_conforming(tvo_grid* g, uint32_t t) { return refine_conforming(g, t, NULL); }

static void leaf_ids(const tvo_grid* g, u32vec* out) {
    out->n = 0;
    for (uint32_t t = 0; t < g->nt; ++t)
        if (g->tets[t].children[0] == TVO_NO_TET) uv_push(out, t);
}

/* acceptance.cpp:63-70 fixture */
tvo_grid* tvo_grid_fuzzed(int steps, uint64_t seed, int max_level) {
    tvo_grid* g = tvo_grid_init_roots(max_level);
    if (!g) return NULL;
    u32vec leaves = {0};
    for (int i = 0; i < steps; ++i) {
        leaf_ids(g, &leaves);
        uint32_t pick = leaves.v[tvo_mix64(seed + 0x9e3779b97f4a7c15ull * (uint64_t)(i + 1)) % leaves.n];
        if (refine_conforming(g, pick, NULL)) {
            free(leaves.v);
            tvo_grid_free(g);
            return NULL;
        }
    }
    free(leaves.v);
    return g;
}

/* tet_grid.cpp:428-472 */
static int locate_point(const tvo_grid* g, v3 p, uint32_t* out) {
    if (!(p.x >= 0.0 && p.x <= 1.0 && p.y >= 0.0 && p.y <= 1.0 && p.z >= 0.0 && p.z <= 1.0))
        return set_err(TVO_ERR_OUTSIDE, "locate_point: point outside the unit cube");
    uint32_t root = TVO_NO_TET;
    double best = INFINITY;
    for (int i = 0; i < 24; ++i) {
        uint32_t r = g->roots[i];
        const tvo_tet* tt = &g->tets[r];
        double worst = 0.0;
        for (int slot = 0; slot < 4; ++slot) {
            v3 n = tabn(tt->normal_ids[slot]);
            v3 v = vpos(g, tt->verts[(slot + 1) & 3]);
            worst = dmax(worst, vdot(n, vsub(p, v)));
        }
        if (worst <= 1e-12) { root = r; break; }
        if (worst < best) best = worst, root = r;
    }
    uint32_t cur = root;
    while (g->tets[cur].children[0] != TVO_NO_TET) {
        const tvo_tet* tt = &g->tets[cur];
        int s0, s1;
        refinement_edge_slots(g, cur, &s0, &s1);
        uint32_t ca = tt->children[0];
        v3 pm = vpos(g, g->tets[ca].verts[s1]);
        int oa = -1, ob = -1;
        for (int s = 0; s < 4; ++s)
            if (s != s0 && s != s1) { if (oa < 0) oa = s; else ob = s; }
        v3 pa = vpos(g, tt->verts[oa]), pb = vpos(g, tt->verts[ob]);
        v3 n = vcross(vsub(pa, pm), vsub(pb, pm));
        double sref = vdot(n, vsub(vpos(g, tt->verts[s0]), pm));
        double sp = vdot(n, vsub(p, pm));
        int take_a = sref > 0.0 ? (sp >= 0.0) : (sp <= 0.0);
        cur = take_a ? ca : tt->children[1];
    }
    *out = cur;
    return 0;
}
int tvo_locate_point(const tvo_grid* g, const double* p, uint32_t* out) { return locate_point(g, P(p), out); }

/* tracer.cpp:143-162 */
static int exit_face(const tvo_grid* g, uint32_t cell, v3 pos, v3 dir, double* tout) {
    const tvo_tet* tt = &g->tets[cell];
    int best_slot = -1;
    double best_t = INFINITY;
    for (int slot = 0; slot < 4; ++slot) {
        v3 n = tabn(tt->normal_ids[slot]);
        double dn = vdot(n, dir);
        if (dn <= 1e-12) continue;
        v3 v = vpos(g, tt->verts[(slot + 1) & 3]);
        double t = vdot(n, vsub(v, pos)) / dn;
        if (t < 0.0) t = 0.0;
        if (t < best_t) best_t = t, best_slot = slot;
    }
    *tout = best_t;
    return best_slot;
}
int tvo_exit_face(const tvo_grid* g, uint32_t cell, const double* pos, const double* dir, double* t) {
    return exit_face(g, cell, P(pos), P(dir), t);
}

/* ------------------------------------------------------------- marcher --- */
/* tracer.cpp:25-127 */
typedef struct {
    const tvo_grid* g;
    ray_t ray;
    uint32_t cell, last_cell;
    double seg_start, probe_t, last_t0, event_t;
    v3 event_point;
    int aborted, escaped;
    uint64_t steps;
} marcher;
typedef struct { double t0, t1, lambda; uint32_t cell; } mstep;

static int m_start(marcher* m, const ray_t* ray) {
    m->aborted = m->escaped = 0;
    m->steps = 0;
    m->ray = *ray;
    m->ray.tmin = dmax(0.0, ray->tmin);
    double t0, t1;
    if (!slab(&m->ray, &t0, &t1)) return 0;
    v3 p = ray_at(&m->ray, t0 + 1e-7);
    p.x = dclamp(p.x, 0.0, 1.0), p.y = dclamp(p.y, 0.0, 1.0), p.z = dclamp(p.z, 0.0, 1.0);
    if (locate_point(m->g, p, &m->cell)) return 0;
    m->seg_start = t0;
    m->probe_t = t0 + 1e-7;
    return 1;
}
static int m_next(marcher* m, mstep* st) {
    if (m->aborted || m->escaped) return 0;
    if (++m->steps > 50000000ull) { m->aborted = 1; return 0; }
    double t;
    int slot = exit_face(m->g, m->cell, ray_at(&m->ray, m->probe_t), m->ray.d, &t);
    if (slot < 0) {
        m->probe_t += 1e-7;
        slot = exit_face(m->g, m->cell, ray_at(&m->ray, m->probe_t), m->ray.d, &t);
        if (slot < 0) { m->aborted = 1; return 0; }
    }
    double t_exit = dmax(m->probe_t + t, m->seg_start);
    st->t0 = m->seg_start;
    st->lambda = m->g->tets[m->cell].density;
    st->cell = m->cell;
    m->last_cell = m->cell;
    m->last_t0 = m->seg_start;
    if (t_exit >= m->ray.tmax) {
        st->t1 = m->ray.tmax;
        m->escaped = 1;
        m->event_point = ray_at(&m->ray, m->ray.tmax);
        return 1;
    }
    st->t1 = t_exit;
    uint32_t nb = m->g->tets[m->cell].neighbors[slot];
    if (nb == TVO_NO_TET) {
        m->escaped = 1;
        m->event_point = ray_at(&m->ray, t_exit);
    } else {
        m->cell = nb;
        m->seg_start = t_exit;
        m->probe_t = t_exit + 1e-7;
    }
    return 1;
}
static void m_shorten(marcher* m, double dist) {
    m->event_point = ray_at(&m->ray, m->last_t0 + dist);
    m->event_t = m->last_t0 + dist;
    m->cell = m->last_cell;
    m->escaped = 0;
}
static void m_redirect(marcher* m, v3 dir) {
    m->ray.o = m->event_point;
    m->ray.d = dir;
    m->ray.tmin = 0.0;
    m->ray.tmax = INFINITY;
    m->seg_start = m->probe_t = 0.0;
    m->escaped = 0;
}

static ray_t ray8(const double* r) {
    ray_t x = {P(r), P(r + 3), r[6], r[7]};
    return x;
}

/* tracer.cpp:164-174 */
int64_t tvo_march_segments(const tvo_grid* g, const double* rays, uint64_t n, uint32_t* cells, double* t0,
                           double* t1, uint64_t* offsets, uint64_t cap, uint64_t* stats) {
    uint64_t k = 0, cv = 0, deg = 0;
    for (uint64_t i = 0; i < n; ++i) {
        if (offsets) offsets[i] = k;
        marcher m = {0};
        m.g = g;
        ray_t r = ray8(rays + 8 * i);
        if (!m_start(&m, &r)) continue;
        mstep s;
        while (m_next(&m, &s)) {
            ++cv;
            if (k < cap) cells[k] = s.cell, t0[k] = s.t0, t1[k] = s.t1;
            ++k;
        }
        if (m.aborted) ++deg;
    }
    if (offsets) offsets[n] = k;
    if (stats) stats[0] = cv, stats[1] = deg;
    return (int64_t)k;
}

/* tracer.cpp:176-186 */
double tvo_march_transmittance(const tvo_grid* g, const double* r8) {
    marcher m = {0};
    m.g = g;
    ray_t r = ray8(r8);
    if (!m_start(&m, &r)) return 1.0;
    double tau = 0.0;
    mstep s;
    while (m_next(&m, &s)) tau += s.lambda * (s.t1 - s.t0);
    return exp(-tau);
}

/* tracer.cpp:188-216 */
void tvo_sample_free_path(const tvo_grid* g, const double* r8, uint64_t seed, uint64_t pixel, uint64_t sample,
                          double* out) {
    rng_t rng;
    rng_init(&rng, seed, pixel, sample);
    marcher m = {0};
    m.g = g;
    ray_t r = ray8(r8);
    double target = -log(1.0 - rng_next(&rng));
    memset(out, 0, 6 * sizeof(double));
    out[4] = (double)TVO_NO_TET;
    if (!m_start(&m, &r)) {
        out[1] = r.o.x, out[2] = r.o.y, out[3] = r.o.z;
        return;
    }
    double tau = 0.0, last_t1 = 0.0;
    mstep s;
    while (m_next(&m, &s)) {
        double seg = s.lambda * (s.t1 - s.t0);
        if (s.lambda > 0.0 && tau + seg >= target) {
            m_shorten(&m, (target - tau) / s.lambda);
            out[0] = 1;
            out[1] = m.event_point.x, out[2] = m.event_point.y, out[3] = m.event_point.z;
            out[4] = m.last_cell;
            out[5] = m.event_t;
            return;
        }
        tau += seg;
        last_t1 = s.t1;
    }
    v3 p = m.aborted ? ray_at(&r, last_t1) : m.event_point;
    out[1] = p.x, out[2] = p.y, out[3] = p.z;
    out[5] = last_t1;
}

/* tracer.cpp:218-222 */
double tvo_hg_sample_cos(double g, double xi) {
    if (fabs(g) < 1e-6) return 1.0 - 2.0 * xi;
    double sq = (1.0 - g * g) / (1.0 - g + 2.0 * g * xi);
    return dclamp((1.0 + g * g - sq * sq) / (2.0 * g), -1.0, 1.0);
}
/* tracer.cpp:224-234 */
static v3 sample_phase_hg(v3 dir, double g, rng_t* rng) {
    double u1 = rng_next(rng), u2 = rng_next(rng);
    double ct = tvo_hg_sample_cos(g, u1);
    double st = sqrt(dmax(0.0, 1.0 - ct * ct));
    double phi = 2.0 * kPi * u2;
    v3 t = fabs(dir.z) < 0.999 ? vnorm(vcross(V(0, 0, 1), dir)) : vnorm(vcross(V(1, 0, 0), dir));
    v3 b = vcross(dir, t);
    return vnorm(vadd(vadd(vmul(t, st * cos(phi)), vmul(b, st * sin(phi))), vmul(dir, ct)));
}
void tvo_sample_phase_hg(const double* dir, double g, uint64_t seed, uint64_t pixel, uint64_t sample, double* out) {
    rng_t rng;
    rng_init(&rng, seed, pixel, sample);
    v3 w = sample_phase_hg(P(dir), g, &rng);
    out[0] = w.x, out[1] = w.y, out[2] = w.z;
}
/* tracer.cpp:241-256 */
static v3 emission_color(double temperature) {
    static const double lut[9][3] = {
        {0.00, 0.00, 0.00}, {0.25, 0.02, 0.00}, {0.50, 0.05, 0.00}, {0.75, 0.12, 0.01}, {1.00, 0.25, 0.02},
        {1.00, 0.45, 0.08}, {1.00, 0.65, 0.20}, {1.00, 0.85, 0.55}, {1.00, 1.00, 1.00},
    };
    double t = dclamp(temperature, 0.0, 1.0) * 8.0;
    int i0 = (int)t < 7 ? (int)t : 7;
    double f = t - i0;
    return V(lut[i0][0] + (lut[i0 + 1][0] - lut[i0][0]) * f, lut[i0][1] + (lut[i0 + 1][1] - lut[i0][1]) * f,
             lut[i0][2] + (lut[i0 + 1][2] - lut[i0][2]) * f);
}
void tvo_emission_color(double t, double* out) {
    v3 c = emission_color(t);
    out[0] = c.x, out[1] = c.y, out[2] = c.z;
}

/* --------------------------------------------------------- integrator --- */
/* The integrator is generic over the marcher (path_integrator.hpp:4-18); in C
 * the two marchers share it through this small vtable. */
typedef struct {
    void* self;
    int (*start)(void*, const ray_t*);
    int (*next)(void*, mstep*);
    void (*shorten)(void*, double);
    void (*redirect)(void*, v3);
    v3 (*dir)(void*);
    void (*media)(void*, float*, float*, float*, uint8_t*);
    int (*aborted)(void*);
} mvt;

typedef struct { double variation_threshold; } unused_t;
typedef struct {
    int spp, max_bounces;
    uint64_t seed;
    double g, albedo, emission_scale;
    v3 env;
} rcfg;

/* path_integrator.hpp:42-84 */
static v3 trace_path(const mvt* m, const ray_t* primary, const rcfg* cfg, rng_t* rng, uint64_t* cells,
                     uint64_t* deg) {
    v3 L = V(0, 0, 0), T = V(1, 1, 1);
    if (!m->start(m->self, primary)) return cfg->env;
    for (int bounce = 0;;) {
        const double target = -log(1.0 - rng_next(rng));
        double tau = 0.0;
        int collided = 0;
        mstep s;
        while (m->next(m->self, &s)) {
            ++*cells;
            const double seg = s.lambda * (s.t1 - s.t0);
            if (s.lambda > 0.0 && tau + seg >= target) {
                m->shorten(m->self, (target - tau) / s.lambda);
                collided = 1;
                break;
            }
            tau += seg;
        }
        if (m->aborted(m->self)) {
            ++*deg;
            return L;
        }
        if (!collided) return vadd(L, vmulv(T, cfg->env));
        float dens, temp, alb;
        uint8_t mask;
        m->media(m->self, &dens, &temp, &alb, &mask);
        if (mask & 2u) L = vadd(L, vmul(vmulv(T, emission_color(temp)), cfg->emission_scale));
        T = vmul(T, (mask & 4u) ? (double)alb : cfg->albedo);
        ++bounce;
        if (bounce >= cfg->max_bounces) return L;
        if (bounce >= 4) {
            const double p = dmax(T.x, dmax(T.y, T.z));
            if (p < 1e-3) {
                if (rng_next(rng) >= p) return L;
                T = vdiv(T, p);
            }
        }
        m->redirect(m->self, sample_phase_hg(m->dir(m->self), cfg->g, rng));
    }
}

static int tm_start(void* s, const ray_t* r) { return m_start((marcher*)s, r); }
static int tm_next(void* s, mstep* st) { return m_next((marcher*)s, st); }
static void tm_shorten(void* s, double d) { m_shorten((marcher*)s, d); }
static void tm_redirect(void* s, v3 d) { m_redirect((marcher*)s, d); }
static v3 tm_dir(void* s) { return ((marcher*)s)->ray.d; }
static void tm_media(void* s, float* d, float* t, float* a, uint8_t* m) {
    const marcher* mm = (const marcher*)s;
    const tvo_tet* tt = &mm->g->tets[mm->last_cell];
    *d = tt->density, *t = tt->temperature, *a = tt->albedo, *m = tt->mask;
}
static int tm_aborted(void* s) { return ((marcher*)s)->aborted; }

/* ----------------------------------------------------------------- DDA --- */
/* regular_grid.cpp:16-118 */
typedef struct {
    const float* dens; /* already scaled, like RegularGrid::density_ */
    int n[3];
    ray_t ray;
    int idx[3], step[3];
    double t_next[3], t_delta[3], t_cur, t_end, last_t0, event_t;
    size_t last_cell;
    v3 event_point;
    int escaped;
} dda_t;
static int dda_start(void* s, const ray_t* ray) {
    dda_t* m = (dda_t*)s;
    m->escaped = 0;
    m->ray = *ray;
    m->ray.tmin = dmax(0.0, ray->tmin);
    double t0, t1;
    if (!slab(&m->ray, &t0, &t1)) return 0;
    m->t_end = t1;
    v3 p = ray_at(&m->ray, t0 + 1e-9);
    for (int a = 0; a < 3; ++a) {
        int i = (int)floor(vcomp(p, a) * m->n[a]);
        m->idx[a] = i < 0 ? 0 : (i > m->n[a] - 1 ? m->n[a] - 1 : i);
        double d = vcomp(m->ray.d, a), o = vcomp(m->ray.o, a);
        if (d > 0.0) {
            m->step[a] = 1;
            m->t_next[a] = ((m->idx[a] + 1.0) / m->n[a] - o) / d;
            m->t_delta[a] = 1.0 / (m->n[a] * d);
        } else if (d < 0.0) {
            m->step[a] = -1;
            m->t_next[a] = ((double)m->idx[a] / m->n[a] - o) / d;
            m->t_delta[a] = -1.0 / (m->n[a] * d);
        } else {
            m->step[a] = 0;
            m->t_next[a] = INFINITY;
            m->t_delta[a] = INFINITY;
        }
    }
    m->t_cur = t0;
    return 1;
}
static int dda_next(void* s, mstep* st) {
    dda_t* m = (dda_t*)s;
    if (m->escaped) return 0;
    const int axis = m->t_next[0] <= m->t_next[1] ? (m->t_next[0] <= m->t_next[2] ? 0 : 2)
                                                  : (m->t_next[1] <= m->t_next[2] ? 1 : 2);
    double t_exit = m->t_next[axis];
    st->t0 = m->t_cur;
    size_t flat = ((size_t)m->idx[2] * m->n[1] + m->idx[1]) * m->n[0] + m->idx[0];
    st->lambda = m->dens[flat];
    st->cell = (uint32_t)flat;
    m->last_cell = flat;
    m->last_t0 = m->t_cur;
    if (t_exit >= m->ray.tmax) {
        st->t1 = m->ray.tmax;
        m->escaped = 1;
        m->event_point = ray_at(&m->ray, m->ray.tmax);
        return 1;
    }
    m->idx[axis] += m->step[axis];
    m->t_next[axis] += m->t_delta[axis];
    if (m->idx[axis] < 0 || m->idx[axis] >= m->n[axis] || t_exit >= m->t_end - 1e-15) {
        t_exit = m->t_end;
        m->escaped = 1;
        m->event_point = ray_at(&m->ray, t_exit);
    }
    st->t1 = t_exit;
    m->t_cur = t_exit;
    return 1;
}
static void dda_shorten(void* s, double dist) {
    dda_t* m = (dda_t*)s;
    m->event_point = ray_at(&m->ray, m->last_t0 + dist);
    m->event_t = m->last_t0 + dist;
    m->escaped = 0;
}
static void dda_redirect(void* s, v3 dir) {
    dda_t* m = (dda_t*)s;
    ray_t r = {m->event_point, dir, 0.0, INFINITY};
    if (!dda_start(s, &r)) m->escaped = 1;
}
static v3 dda_dir(void* s) { return ((dda_t*)s)->ray.d; }
static void dda_media(void* s, float* d, float* t, float* a, uint8_t* mk) {
    const dda_t* m = (const dda_t*)s;
    *d = m->dens[m->last_cell], *t = 0.0f, *a = 0.0f, *mk = 1;
}
static int dda_aborted(void* s) { (void)s; return 0; }

/* -------------------------------------------------------------- render --- */
typedef struct {
    int kind; /* 0 tet, 1 dda */
    const tvo_grid* g;
    const float* dens;
    int n[3];
    cam_t cam;
    rcfg cfg;
    int row_stride, row_offset;
    atomic_int next_row;
    double *sum, *sum_sq;
    uint32_t* counts;
} render_job;
typedef struct { uint64_t cells, deg; char pad[48]; } __attribute__((aligned(64))) tstats;
typedef struct { render_job* job; tstats* st; } worker_arg;

/* path_integrator.hpp:87-127 (rows pulled from an atomic counter; each pixel's
 * samples in order s = 0..spp-1, so the sums are thread-count invariant) */
static void* render_worker(void* p) {
    worker_arg* wa = (worker_arg*)p;
    render_job* j = wa->job;
    marcher tm = {0};
    dda_t dm = {0};
    mvt vt;
    if (j->kind == 0) {
        tm.g = j->g;
        mvt t = {&tm, tm_start, tm_next, tm_shorten, tm_redirect, tm_dir, tm_media, tm_aborted};
        vt = t;
    } else {
        dm.dens = j->dens;
        dm.n[0] = j->n[0], dm.n[1] = j->n[1], dm.n[2] = j->n[2];
        mvt t = {&dm, dda_start, dda_next, dda_shorten, dda_redirect, dda_dir, dda_media, dda_aborted};
        vt = t;
    }
    const int W = j->cam.w, H = j->cam.h;
    for (;;) {
        int r = atomic_fetch_add(&j->next_row, 1);
        int y = r * j->row_stride + j->row_offset;
        if (y >= H) break;
        for (int x = 0; x < W; ++x) {
            uint64_t pixel = (uint64_t)y * W + x;
            size_t i = pixel * 3;
            for (int s = 0; s < j->cfg.spp; ++s) {
                rng_t rng;
                rng_init(&rng, j->cfg.seed, pixel, (uint64_t)s);
                double jx = rng_next(&rng), jy = rng_next(&rng);
                ray_t ray;
                cam_primary(&j->cam, x, y, jx, jy, &ray);
                v3 c = trace_path(&vt, &ray, &j->cfg, &rng, &wa->st->cells, &wa->st->deg);
                if (j->sum) j->sum[i] += c.x, j->sum[i + 1] += c.y, j->sum[i + 2] += c.z;
                if (j->sum_sq)
                    j->sum_sq[i] += c.x * c.x, j->sum_sq[i + 1] += c.y * c.y, j->sum_sq[i + 2] += c.z * c.z;
                if (j->counts) j->counts[pixel]++;
            }
        }
    }
    return NULL;
}

/* tracer.cpp:131-141 */
static int validate_rcfg(const tvo_render_cfg* r) {
    if (r->spp < 1) return set_err(TVO_ERR_CONFIG, "spp must be at least 1");
    if (r->max_bounces < 1) return set_err(TVO_ERR_CONFIG, "maxBounces must be at least 1");
    if (!(r->hg_g > -1.0 && r->hg_g < 1.0)) return set_err(TVO_ERR_CONFIG, "phase anisotropy g must be in (-1, 1)");
    if (!(r->default_albedo >= 0.0 && r->default_albedo <= 1.0))
        return set_err(TVO_ERR_CONFIG, "albedo must be in [0, 1]");
    if (r->env[0] < 0.0 || r->env[1] < 0.0 || r->env[2] < 0.0)
        return set_err(TVO_ERR_CONFIG, "environment radiance must be non-negative");
    if (r->emission_scale < 0.0) return set_err(TVO_ERR_CONFIG, "emissionScale must be non-negative");
    return 0;
}

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec + ts.tv_nsec * 1e-9;
}

static int run_render(render_job* j, const tvo_camera_desc* c, const tvo_render_cfg* r, int threads,
                      uint64_t* stats, double* seconds) {
    int rc = validate_rcfg(r);
    if (rc) return rc;
    if ((rc = cam_init(&j->cam, c))) return rc;
    if (j->row_stride < 1) j->row_stride = 1;
    j->cfg.spp = r->spp, j->cfg.max_bounces = r->max_bounces, j->cfg.seed = r->seed, j->cfg.g = r->hg_g;
    j->cfg.albedo = r->default_albedo, j->cfg.emission_scale = r->emission_scale, j->cfg.env = P(r->env);
    double t0 = now_s();
    int n = threads > 0 ? threads : (int)sysconf(_SC_NPROCESSORS_ONLN);
    if (n < 1) n = 1;
    if (n > j->cam.h) n = j->cam.h;
    atomic_init(&j->next_row, 0);
    tstats* st = (tstats*)aligned_alloc(64, sizeof(tstats) * (size_t)n);
    memset(st, 0, sizeof(tstats) * (size_t)n);
    worker_arg* wa = (worker_arg*)malloc(sizeof(worker_arg) * (size_t)n);
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)n);
    for (int i = 0; i < n; ++i) {
        wa[i].job = j, wa[i].st = &st[i];
        if (n == 1) render_worker(&wa[0]);
        else pthread_create(&th[i], NULL, render_worker, &wa[i]);
    }
    if (n > 1)
        for (int i = 0; i < n; ++i) pthread_join(th[i], NULL);
    uint64_t cells = 0, deg = 0;
    for (int i = 0; i < n; ++i) cells += st[i].cells, deg += st[i].deg;
    int rows = 0;
    for (int y = j->row_offset; y < j->cam.h; y += j->row_stride) ++rows;
    if (stats) stats[0] = cells, stats[1] = (uint64_t)rows * j->cam.w * r->spp, stats[2] = deg;
    if (seconds) *seconds = now_s() - t0;
    free(st);
    free(wa);
    free(th);
    return 0;
}

int tvo_render(const tvo_grid* g, const tvo_camera_desc* c, const tvo_render_cfg* r, int threads, int row_stride,
               int row_offset, double* sum, double* sum_sq, uint32_t* counts, uint64_t* stats, double* seconds) {
    render_job j;
    memset(&j, 0, sizeof j);
    j.kind = 0, j.g = g, j.row_stride = row_stride, j.row_offset = row_offset;
    j.sum = sum, j.sum_sq = sum_sq, j.counts = counts;
    return run_render(&j, c, r, threads, stats, seconds);
}

static float* scaled_density(const float* d, size_t n, double scale) { /* regular_grid.cpp:122-134 */
    float* out = (float*)malloc(n * sizeof(float));
    for (size_t i = 0; i < n; ++i) out[i] = (float)(d[i] * scale);
    return out;
}
int tvo_render_regular(const float* density, int nx, int ny, int nz, double density_scale, const tvo_camera_desc* c,
                       const tvo_render_cfg* r, int threads, double* sum, double* sum_sq, uint32_t* counts,
                       uint64_t* stats, double* seconds) {
    render_job j;
    memset(&j, 0, sizeof j);
    float* sd = scaled_density(density, (size_t)nx * ny * nz, density_scale);
    j.kind = 1, j.dens = sd, j.n[0] = nx, j.n[1] = ny, j.n[2] = nz, j.row_stride = 1;
    j.sum = sum, j.sum_sq = sum_sq, j.counts = counts;
    int rc = run_render(&j, c, r, threads, stats, seconds);
    free(sd);
    return rc;
}
int64_t tvo_dda_segments(const float* density, int nx, int ny, int nz, double density_scale, const double* rays,
                         uint64_t n, uint32_t* cells, double* t0, double* t1, uint64_t* offsets, uint64_t cap) {
    float* sd = scaled_density(density, (size_t)nx * ny * nz, density_scale);
    dda_t m;
    memset(&m, 0, sizeof m);
    m.dens = sd, m.n[0] = nx, m.n[1] = ny, m.n[2] = nz;
    uint64_t k = 0;
    for (uint64_t i = 0; i < n; ++i) {
        if (offsets) offsets[i] = k;
        ray_t r = ray8(rays + 8 * i);
        if (!dda_start(&m, &r)) continue;
        mstep s;
        while (dda_next(&m, &s)) {
            if (k < cap) cells[k] = s.cell, t0[k] = s.t0, t1[k] = s.t1;
            ++k;
        }
    }
    if (offsets) offsets[n] = k;
    free(sd);
    return (int64_t)k;
}

/* ------------------------------------------------------------- builder --- */
/* volume.cpp:140-148 */
typedef struct { v3 n[4]; double d[4]; } planes_t;
static void tet_corners(const tvo_grid* g, uint32_t t, v3* c) {
    for (int i = 0; i < 4; ++i) c[i] = vpos(g, g->tets[t].verts[i]);
}
static void make_planes(const v3* c, planes_t* pl) {
    for (int slot = 0; slot < 4; ++slot) {
        v3 p0 = c[(slot + 1) & 3], p1 = c[(slot + 2) & 3], p2 = c[(slot + 3) & 3];
        v3 nn = vnorm(vcross(vsub(p1, p0), vsub(p2, p0)));
        if (vdot(nn, vsub(c[slot], p0)) > 0.0) nn = vneg(nn);
        pl->n[slot] = nn;
        pl->d[slot] = vdot(nn, p0);
    }
}
/* builder.cpp:24-29 with volume.hpp:75-86 */
static int owns_center(const tvo_grid* g, uint32_t leaf, const planes_t* pl, v3 c) {
    const double band = 1e-9;
    for (int f = 0; f < 4; ++f)
        if (vdot(pl->n[f], c) > pl->d[f] + band) return 0; /* strictly outside */
    int inside = 1;
    for (int f = 0; f < 4; ++f)
        if (vdot(pl->n[f], c) > pl->d[f] - band) { inside = 0; break; }
    if (inside) return 1;
    uint32_t who;
    if (locate_point(g, c, &who)) return 0;
    return who == leaf;
}
/* volume.cpp:47-66 */
static double trilinear(const float* data, int nx, int ny, int nz, v3 p) {
    double fx = p.x * nx - 0.5, fy = p.y * ny - 0.5, fz = p.z * nz - 0.5;
    int i0 = (int)floor(fx), j0 = (int)floor(fy), k0 = (int)floor(fz);
    double tx = fx - i0, ty = fy - j0, tz = fz - k0;
#define CL(v, n) ((v) < 0 ? 0 : ((v) > (n) - 1 ? (n) - 1 : (v)))
    int i1 = CL(i0 + 1, nx), j1 = CL(j0 + 1, ny), k1 = CL(k0 + 1, nz);
    i0 = CL(i0, nx), j0 = CL(j0, ny), k0 = CL(k0, nz);
#undef CL
#define VV(i, j, k) ((double)data[((size_t)(k) * ny + (j)) * nx + (i)])
    double c00 = VV(i0, j0, k0) * (1 - tx) + VV(i1, j0, k0) * tx;
    double c10 = VV(i0, j1, k0) * (1 - tx) + VV(i1, j1, k0) * tx;
    double c01 = VV(i0, j0, k1) * (1 - tx) + VV(i1, j0, k1) * tx;
    double c11 = VV(i0, j1, k1) * (1 - tx) + VV(i1, j1, k1) * tx;
#undef VV
    double c0 = c00 * (1 - ty) + c10 * ty, c1 = c01 * (1 - ty) + c11 * ty;
    return c0 * (1 - tz) + c1 * tz;
}

typedef struct {
    const float *dens, *temp, *alb;
    int nx, ny, nz;
} vol_t;
typedef struct { double min, max, mean, tmean, amean; uint64_t count; } agg_t;

/* builder.cpp:37-79 and 83-116 (identical voxel loop; index order k, j, i) */
static void aggregate(const vol_t* v, const tvo_grid* g, uint32_t leaf, agg_t* a) {
    v3 c[4];
    tet_corners(g, leaf, c);
    planes_t pl;
    make_planes(c, &pl);
    v3 lo = c[0], hi = c[0];
    for (int i = 1; i < 4; ++i) {
        lo = V(dmin(lo.x, c[i].x), dmin(lo.y, c[i].y), dmin(lo.z, c[i].z));
        hi = V(dmax(hi.x, c[i].x), dmax(hi.y, c[i].y), dmax(hi.z, c[i].z));
    }
    const int dims[3] = {v->nx, v->ny, v->nz};
    int rlo[3], rhi[3]; /* volume.cpp:150-159 */
    for (int ax = 0; ax < 3; ++ax) {
        int l = (int)ceil(vcomp(lo, ax) * dims[ax] - 0.5 - 1e-12);
        int h = (int)floor(vcomp(hi, ax) * dims[ax] - 0.5 + 1e-12);
        rlo[ax] = l > 0 ? l : 0;
        rhi[ax] = h < dims[ax] - 1 ? h : dims[ax] - 1;
    }
    a->min = INFINITY, a->max = -INFINITY, a->count = 0, a->tmean = a->amean = 0.0;
    double dsum = 0.0, tsum = 0.0, asum = 0.0;
    for (int k = rlo[2]; k <= rhi[2]; ++k)
        for (int j = rlo[1]; j <= rhi[1]; ++j)
            for (int i = rlo[0]; i <= rhi[0]; ++i) {
                v3 ctr = V((i + 0.5) / v->nx, (j + 0.5) / v->ny, (k + 0.5) / v->nz);
                if (!owns_center(g, leaf, &pl, ctr)) continue;
                size_t idx = ((size_t)k * v->ny + j) * v->nx + i;
                double x = v->dens[idx];
                a->min = dmin(a->min, x);
                a->max = dmax(a->max, x);
                dsum += x;
                if (v->temp) tsum += v->temp[idx];
                if (v->alb) asum += v->alb[idx];
                ++a->count;
            }
    if (a->count == 0) {
        v3 cen = vmul(vadd(vadd(vadd(c[0], c[1]), c[2]), c[3]), 0.25);
        double x = trilinear(v->dens, v->nx, v->ny, v->nz, cen);
        a->min = a->max = a->mean = x;
        if (v->temp) a->tmean = trilinear(v->temp, v->nx, v->ny, v->nz, cen);
        if (v->alb) a->amean = trilinear(v->alb, v->nx, v->ny, v->nz, cen);
    } else {
        double n = (double)a->count;
        a->mean = dsum / n;
        if (v->temp) a->tmean = tsum / n;
        if (v->alb) a->amean = asum / n;
    }
}
void tvo_density_stats(const tvo_grid* g, const float* density, int nx, int ny, int nz, uint32_t leaf, double* out) {
    vol_t v = {density, NULL, NULL, nx, ny, nz};
    agg_t a;
    aggregate(&v, g, leaf, &a);
    out[0] = a.min, out[1] = a.max, out[2] = a.mean, out[3] = (double)a.count;
}

/* (level, id) min-heap: std::priority_queue<..., std::greater<>> (builder.cpp:128-130) */
typedef struct { uint64_t* h; size_t n, cap; } heap_t;
static void heap_push(heap_t* q, int level, uint32_t id) {
    uint64_t key = ((uint64_t)(uint32_t)level << 32) | id;
    if (q->n == q->cap) {
        q->cap = q->cap ? 2 * q->cap : 1024;
        q->h = (uint64_t*)realloc(q->h, q->cap * sizeof(uint64_t));
    }
    size_t i = q->n++;
    while (i > 0) {
        size_t p = (i - 1) / 2;
        if (q->h[p] <= key) break;
        q->h[i] = q->h[p];
        i = p;
    }
    q->h[i] = key;
}
static uint64_t heap_pop(heap_t* q) {
    uint64_t top = q->h[0], last = q->h[--q->n];
    size_t i = 0;
    for (;;) {
        size_t l = 2 * i + 1, r = l + 1, m = i;
        uint64_t mv = last;
        if (l < q->n && q->h[l] < mv) m = l, mv = q->h[l];
        if (r < q->n && q->h[r] < mv) m = r, mv = q->h[r];
        if (m == i) break;
        q->h[i] = q->h[m];
        i = m;
    }
    if (q->n) q->h[i] = last;
    return top;
}

/* builder.cpp:12-17 */
static int validate_bcfg(const tvo_build_cfg* b) {
    if (!(b->variation_threshold >= 0.0)) return set_err(TVO_ERR_CONFIG, "variationThreshold must be >= 0");
    if (b->max_level < 0 || b->max_level > TVO_LEVEL_CAP) return set_err(TVO_ERR_CONFIG, "maxLevel out of range");
    if (!(b->pixel_threshold > 0.0)) return set_err(TVO_ERR_CONFIG, "pixelThreshold must be > 0");
    if (!(b->density_scale >= 0.0)) return set_err(TVO_ERR_CONFIG, "densityScale must be >= 0");
    return 0;
}

/* builder.cpp:118-182 */
tvo_grid* tvo_grid_build(const float* density, const float* temperature, const float* albedo, int nx, int ny,
                         int nz, const tvo_build_cfg* bc, const tvo_camera_desc* camd, tvo_build_stats* st) {
    if (validate_bcfg(bc)) return NULL;
    if (bc->use_camera && !camd) {
        set_err(TVO_ERR_CONFIG, "useCamera set but no camera given");
        return NULL;
    }
    cam_t cam;
    if (camd && cam_init(&cam, camd)) return NULL;
    double t_begin = now_s();
    tvo_grid* g = tvo_grid_init_roots(bc->max_level > 1 ? bc->max_level : 1);
    if (!g) return NULL;
    vol_t v = {density, temperature, albedo, nx, ny, nz};
    heap_t q = {0};
    for (int i = 0; i < 24; ++i) heap_push(&q, 0, g->roots[i]);
    uint64_t crit = 0, prop = 0;
    u32vec fresh = {0};
    int rc = 0;
    while (q.n && !rc) {
        uint64_t key = heap_pop(&q);
        int level = (int)(key >> 32);
        uint32_t id = (uint32_t)key;
        if (g->tets[id].children[0] != TVO_NO_TET) continue;
        agg_t a;
        aggregate(&v, g, id, &a);
        double var = a.mean == 0.0 ? 0.0 : (a.max - a.min) / a.mean; /* volume.cpp:196-199 */
        if (!(var > bc->variation_threshold)) continue;
        if (level >= bc->max_level) continue;
        if (bc->use_camera) {
            v3 cs[4];
            tet_corners(g, id, cs);
            if (cam_outside(&cam, cs)) continue;
            if (!(cam_proj_size(&cam, cs) > bc->pixel_threshold)) continue;
        }
        size_t before = g->nt;
        fresh.n = 0;
        rc = refine_conforming(g, id, &fresh);
        size_t bis = (g->nt - before) / 2;
        ++crit;
        prop += bis - 1;
        for (size_t i = 0; i < fresh.n; ++i) heap_push(&q, g->tets[fresh.v[i]].level, fresh.v[i]);
    }
    free(q.h);
    free(fresh.v);
    if (rc) {
        tvo_grid_free(g);
        return NULL;
    }
    /* assign_payloads, builder.cpp:164-182 */
    int maxd = 0;
    for (uint32_t t = 0; t < g->nt; ++t) {
        tvo_tet* tt = &g->tets[t];
        if (tt->children[0] != TVO_NO_TET) continue;
        agg_t a;
        aggregate(&v, g, t, &a);
        tt->density = (float)(bc->density_scale * a.mean);
        tt->mask = 1;
        if (temperature) tt->temperature = (float)a.tmean, tt->mask |= 2;
        if (albedo) tt->albedo = (float)dclamp(a.amean, 0.0, 1.0), tt->mask |= 4;
        if (tt->level > maxd) maxd = tt->level;
    }
    if (st) {
        st->leaf_count = g->leaf_count;
        st->max_depth = maxd;
        st->seconds = now_s() - t_begin;
        st->criterion_splits = crit;
        st->propagation_splits = prop;
    }
    return g;
}

/* ---------------------------------------------------------------- misc --- */
uint64_t tvo_fnv64_doubles(const double* v, uint64_t n) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (uint64_t i = 0; i < n; ++i) {
        uint64_t b;
        memcpy(&b, &v[i], 8);
        h = (h ^ b) * 0x100000001b3ull;
    }
    return h;
}

/* acceptance.cpp:49-61 random_cube_ray(seed, salt, i), i in [0, n): rows of 8 */
void tvo_random_cube_rays(uint64_t seed, uint64_t salt, uint64_t n, double* out) {
    for (uint64_t i = 0; i < n; ++i) {
        rng_t rng;
        rng_init(&rng, seed, salt, i);
        double u1 = rng_next(&rng), u2 = rng_next(&rng);
        double z = 1.0 - 2.0 * u1;
        double r = sqrt(dmax(0.0, 1.0 - z * z));
        double phi = 2.0 * 3.14159265358979323846 * u2;
        v3 o = vadd(V(0.5, 0.5, 0.5), vmul(V(r * cos(phi), r * sin(phi), z), 2.0));
        double a = rng_next(&rng), b = rng_next(&rng), c = rng_next(&rng);
        v3 tg = V(0.25 + 0.5 * a, 0.25 + 0.5 * b, 0.25 + 0.5 * c);
        v3 d = vnorm(vsub(tg, o));
        double* w = out + 8 * i;
        w[0] = o.x, w[1] = o.y, w[2] = o.z, w[3] = d.x, w[4] = d.y, w[5] = d.z, w[6] = 0.0, w[7] = INFINITY;
    }
}
