// GPU LEB build: build_adaptive_grid (builder.cpp:118-182) as synchronous
// rounds, plus the on-device procedural fields.
//
// The reference refines from a (level, id) worklist with recursive conforming
// propagation (tet_grid.cpp:384-426). Its final leaf set is a least fixed point
// that does not depend on visiting order, so the GPU
// computes it in rounds:
//   eval     every fresh leaf gets its ownership statistics and criterion
//            (builder.cpp:137-144); criterion leaves are marked;
//   closure  bisect ALL marked leaves at once (tet_grid.cpp:339-382), then mark
//            every leaf with a hanging edge (an edge whose integer midpoint
//            already exists as a vertex); repeat until nothing is marked.
// Rounds end when eval marks nothing. Tet and vertex ids are assigned by
// order-preserving compaction and sorted dedup, so the build is deterministic;
// they differ from the reference's allocation-order ids (F3), and parity is on
// the canonical leaf set (sorted fixed-point corners + payload bits).
//
// Voxel ownership (builder.cpp:24-29) equals the pure locate_point partition
// (SURVEY.md a18), so an owner map (one u32 per voxel) is maintained by the
// same descent step locate_point uses (tet_grid.cpp:453-470). Per-leaf sums are
// accumulated in parallel; because the reference sums in increasing voxel
// index order, each decision / payload is certified against a rounding-error
// bound and replayed sequentially in index order when the bound is ambiguous.
#include <cub/cub.cuh>
#include <cuda.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "tv_leb.cuh"
#include "tv_trace.cuh"

namespace tvb {
namespace {

// ===================================================================== fields
// cli.cpp:317-321
__device__ double blob_density(double x, double y, double z) {
    const d3 d = sub(mk(x, y, z), mk(0.5, 0.5, 0.5));
    const double t = dmax(0.0, 1.0 - dot(d, d) / (0.45 * 0.45));
    return t * t;
}

// cli.cpp:323-346, generalised to (cells, seed)
__device__ double vnoise(double px, double py, double pz, int cells, uint64_t seed) {
    const double x = dclamp(px, 0.0, 1.0) * cells, y = dclamp(py, 0.0, 1.0) * cells, z = dclamp(pz, 0.0, 1.0) * cells;
    const int ix = min(static_cast<int>(x), cells - 1), iy = min(static_cast<int>(y), cells - 1),
              iz = min(static_cast<int>(z), cells - 1);
    const double fx = x - ix, fy = y - iy, fz = z - iz;
    double v = 0.0;
    for (int dz = 0; dz < 2; ++dz)
        for (int dy = 0; dy < 2; ++dy)
            for (int dx = 0; dx < 2; ++dx) {
                const double w = (dx ? fx : 1.0 - fx) * (dy ? fy : 1.0 - fy) * (dz ? fz : 1.0 - fz);
                const uint64_t h = mix64(mix64(mix64(seed ^ static_cast<uint64_t>(static_cast<int64_t>(ix + dx))) ^
                                               static_cast<uint64_t>(static_cast<int64_t>(iy + dy))) ^
                                         static_cast<uint64_t>(static_cast<int64_t>(iz + dz)));
                v += w * (static_cast<double>(h >> 11) * 0x1.0p-53);
            }
    return v;
}

constexpr uint64_t kNoiseSeed = 0x5eb0a8a5c9d3f1adull;

__global__ void gen_kernel(int kind, int nx, int ny, int nz, double value, float* out) {
    const uint64_t n = static_cast<uint64_t>(nx) * ny * nz;
    for (uint64_t idx = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; idx < n;
         idx += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(idx % nx), j = static_cast<int>((idx / nx) % ny),
                  k = static_cast<int>(idx / (static_cast<uint64_t>(nx) * ny));
        const double x = (i + 0.5) / nx, y = (j + 0.5) / ny, z = (k + 0.5) / nz;  // volume.hpp:44-46
        double d;
        switch (kind) {
            case 0: d = value; break;
            case 1: d = x; break;
            case 2: d = blob_density(x, y, z); break;
            case 3: d = x < 0.5 ? 1.0 : 0.0; break;
            case 4: d = vnoise(x, y, z, 8, kNoiseSeed); break;
            default: {
                double s = 0.0;
                for (int o = 0; o < 4; ++o) s += ldexp(1.0, -(o + 1)) * vnoise(x, y, z, 8 << o, kNoiseSeed + o);
                const double c = dmax(0.0, s - 0.35);
                d = c * 2.0 * blob_density(x, y, z) / 0.9375;
            }
        }
        out[idx] = static_cast<float>(d);
    }
}

// ================================================================ LEB core
__host__ __device__ inline int ep0(int e) { return e < 3 ? 0 : (e < 5 ? 1 : 2); }
__host__ __device__ inline int ep1(int e) { return e < 3 ? e + 1 : (e < 5 ? e - 1 : 3); }

__host__ __device__ inline uint4 vq_of(const uint4* verts, uint32_t v) { return verts[v]; }

// tet_grid.cpp:119-128
__host__ __device__ inline bool compute_normals(tv_tet& t, const uint4* verts) {
    for (int slot = 0; slot < 4; ++slot) {
        uint4 f[3];
        int n = 0;
        for (int s = 0; s < 4; ++s)
            if (s != slot) f[n++] = verts[t.verts[s]];
        const int id = face_normal_id(f[0], f[1], f[2], verts[t.verts[slot]]);
        if (id < 0) return false;
        t.normal_ids[slot] = static_cast<uint8_t>(id);
    }
    return true;
}

// tet_grid.cpp:288-330
__host__ __device__ inline void refinement_slots(const tv_tet& tt, const uint4* verts, int& s0, int& s1) {
    int best = 0;
    uint64_t best_len = 0;
    uint32_t bmin = 0, bmax = 0;
    for (int e = 0; e < 6; ++e) {
        const uint32_t a = tt.verts[ep0(e)], b = tt.verts[ep1(e)];
        const uint4 qa = verts[a], qb = verts[b];
        const int64_t dx = static_cast<int64_t>(qa.x) - qb.x, dy = static_cast<int64_t>(qa.y) - qb.y,
                      dz = static_cast<int64_t>(qa.z) - qb.z;
        const uint64_t len = static_cast<uint64_t>(dx * dx) + static_cast<uint64_t>(dy * dy) +
                             static_cast<uint64_t>(dz * dz);
        const uint32_t mn = a < b ? a : b, mx = a < b ? b : a;
        bool better;
        if (e == 0) better = true;
        else if (len != best_len) better = len > best_len;
        else better = mn < bmin || (mn == bmin && mx < bmax);
        if (better) best = e, best_len = len, bmin = mn, bmax = mx;
    }
    s0 = ep0(best);
    s1 = ep1(best);
}

// ------------------------------------------------------------- vertex hash
__device__ __forceinline__ uint64_t coord_hash(uint32_t x, uint32_t y, uint32_t z) {
    return mix64((static_cast<uint64_t>(x) << 32 | y) ^ mix64(static_cast<uint64_t>(z) + 0x51ull));
}

// Open addressing, linear probing, load <= 1/2. A slot holds the vertex id and
// a 32-bit fingerprint of its coordinates (the hash bits above the slot index):
// a probe reads the vertex only when the fingerprints match, so a miss (most
// lookups) costs one or two adjacent slot reads instead of a chain of
// dependent slot -> vertex loads.
using HSlot = unsigned long long;
constexpr HSlot kEmptySlot = ~0ull;
__device__ __forceinline__ HSlot hslot(uint32_t fp, uint32_t vid) { return static_cast<HSlot>(fp) << 32 | vid; }

__device__ uint32_t hash_find(const HSlot* table, uint64_t mask, const uint4* verts, uint32_t x, uint32_t y,
                              uint32_t z) {
    const uint64_t h = coord_hash(x, y, z);
    const uint32_t fp = static_cast<uint32_t>(h >> 32);
    uint64_t s = h & mask;
    for (;;) {
        const HSlot e = table[s];
        if (e == kEmptySlot) return kNone;
        if (static_cast<uint32_t>(e >> 32) == fp) {
            const uint32_t v = static_cast<uint32_t>(e);
            const uint4 q = verts[v];
            if (q.x == x && q.y == y && q.z == z) return v;
        }
        s = (s + 1) & mask;
    }
}

// keys are distinct and absent: claim the first empty slot
__device__ void hash_insert(HSlot* table, uint64_t mask, uint32_t x, uint32_t y, uint32_t z, uint32_t vid) {
    const uint64_t h = coord_hash(x, y, z);
    const HSlot e = hslot(static_cast<uint32_t>(h >> 32), vid);
    uint64_t s = h & mask;
    for (;;) {
        if (atomicCAS(table + s, kEmptySlot, e) == kEmptySlot) return;
        s = (s + 1) & mask;
    }
}

__global__ void hash_rebuild_kernel(HSlot* table, uint64_t mask, const uint4* verts, uint32_t n) {
    const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const uint4 q = verts[v];
    hash_insert(table, mask, q.x, q.y, q.z, v);
}

// ----------------------------------------------------------- build state
enum : uint8_t { F_LEAF = 1, F_NEW = 2, F_EVAL = 4, F_MARK = 8 };
enum : int { E_MIDPOINT = 1, E_NORMAL = 2, E_LEVEL = 4, E_FACE = 8 };

struct Stats {
    double sum, asum, tsum, tasum, lsum, lasum;
    uint32_t cnt, mn, mx, pad;
};
static_assert(sizeof(Stats) == 64, "Stats is one 64-byte line");

struct VolView {
    const float* dens;
    const float* temp;
    const float* alb;
    int nx, ny, nz;
    // voxel centre coordinates per axis, (i + 0.5) / n (volume.hpp:44-46), and RN(1 / nx), RN(1 / ny)
    // for the index -> (i, j, k) split (centres_kernel; voxel sweeps only)
    const double *cx, *cy, *cz;
    double rnx, rny;
    // brick owners (see "voxel bricks"); null: the owner map alone is authoritative
    const uint32_t* brick;
    int gbx, gby;
    const uint32_t* sub;  // sub-brick owners of mixed bricks (8 per brick)
};

// the same IEEE division the reference evaluates per voxel, once per coordinate
__global__ void centres_kernel(int nx, int ny, int nz, double* c) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < nx) c[t] = (t + 0.5) / nx;
    else if (t < nx + ny) c[t] = (t - nx + 0.5) / ny;
    else if (t < nx + ny + nz) c[t] = (t - nx - ny + 0.5) / nz;
}

struct CamCrit {
    d3 pos;
    double tan_half;
    int h;
    d3 pn[5];
    double pd[5];
};

__device__ __forceinline__ uint32_t ord_f(float f) {
    const uint32_t b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float unord_f(uint32_t u) {
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

__device__ __forceinline__ d3 corner(const uint4* verts, uint32_t v) { return vpos(verts[v]); }

struct RootScan {
    uint32_t id[24];
    uint32_t nid[24];
    uint32_t vid[24][4];
};

__global__ void stats_zero_kernel(const uint32_t* list, uint32_t n, Stats* st, uint8_t* flags) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t t = list[i];
    Stats z;
    z.sum = z.asum = z.tsum = z.tasum = z.lsum = z.lasum = 0.0;
    z.cnt = 0;
    z.mn = 0xffffffffu;
    z.mx = 0u;
    z.pad = 0;
    st[t] = z;
    flags[t] |= F_EVAL;
}

// ----------------------------------------------------- voxel ownership pass
// One pass over the volume per round (replaces a separate owner-map descent and
// a full-volume statistics pass). Mode kVoxInit (round 0): every voxel gets its
// root (tet_grid.cpp:435-451) and adds to that root's statistics. Mode
// kVoxDescend (later rounds): a voxel whose owner is still a leaf is skipped
// without reading its density (its leaf was evaluated in an earlier round and
// its ownership is final); every other voxel's owner was bisected in the last
// closure, so it descends to its new leaf (tet_grid.cpp:453-470), which is
// fresh, and adds to that leaf's statistics. Mode kVoxAll: every voxel adds to
// its (final) owner, with the temperature / albedo channels (payload pass).
//
// Accumulation: each lane aggregates its voxels in registers while their owner
// stays the same and adds the aggregate to the owner's statistics (global
// fire-and-forget atomics) when the owner changes; at the end of a warp's chunk
// all lanes flush warp-synchronously (one warp reduction and one atomic set
// when the whole warp agrees on the owner, as it does while the tets are
// large). The order of the double sums is free: every decision taken from
// them is certified against a rounding bound (err_bound) or replayed
// sequentially in voxel-index order.
enum : int { kVoxInit = 0, kVoxDescend = 1, kVoxAll = 2 };
#ifndef TV_VOX_DESC_BLOCKS
#define TV_VOX_DESC_BLOCKS 4  // blocks of kVoxThreads per SM in the descend rounds (register cap)
#endif
constexpr int kVoxThreads = 256;

struct Agg {
    double sum, asum, tsum, tasum, lsum, lasum;
    uint32_t cnt, mn, mx;
};

__device__ __forceinline__ void agg_reset(Agg& a) {
    a.sum = a.asum = a.tsum = a.tasum = a.lsum = a.lasum = 0.0;
    a.cnt = 0;
    a.mn = 0xffffffffu;
    a.mx = 0u;
}

__device__ __forceinline__ void stats_atomic(Stats& s, const Agg& a, bool with_tl) {
    atomicAdd(&s.sum, a.sum);
    atomicAdd(&s.asum, a.asum);
    atomicAdd(&s.cnt, a.cnt);
    atomicMin(&s.mn, a.mn);
    atomicMax(&s.mx, a.mx);
    if (with_tl) {
        atomicAdd(&s.tsum, a.tsum);
        atomicAdd(&s.tasum, a.tasum);
        atomicAdd(&s.lsum, a.lsum);
        atomicAdd(&s.lasum, a.lasum);
    }
}

// Where a voxel sweep adds its aggregates: global fire-and-forget atomics
// (RED; f64 adds are native in L2, where shared-memory f64 adds would be CAS
// loops). In the first rounds the owners are few (24 roots, then 48, 96, ...)
// and every SM would hammer the same handful of L2 lines, so owners in
// [lo, lo + n) are striped: lane l adds to stripe[(owner - lo) * 32 + l], and
// stripe_combine_kernel folds the 32 stripes into the owner's Stats afterwards
// (the order of the sums is free, as everywhere in the sweep).
struct StatsSink {
    Stats* st;
    Stats* stripe;
    uint32_t lo, n;  // striped owners; n = 0: none
};
constexpr uint32_t kStripes = 32;

__device__ __forceinline__ void stats_atomic_at(const StatsSink& S, uint32_t owner, const Agg& a, bool with_tl) {
    const uint32_t r = owner - S.lo;
    if (r < S.n) stats_atomic(S.stripe[r * kStripes + (threadIdx.x & 31)], a, with_tl);
    else stats_atomic(S.st[owner], a, with_tl);
}

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// warp-synchronous flush of every lane's (cur, a) with has = a.cnt > 0
__device__ __forceinline__ void warp_flush(const StatsSink& st, uint32_t cur, Agg& a, bool with_tl) {
    const bool has = a.cnt > 0;
    const unsigned m = __ballot_sync(0xffffffffu, has);
    if (!m) return;
    const uint32_t c0 = __shfl_sync(0xffffffffu, cur, __ffs(m) - 1);
    if (__all_sync(0xffffffffu, !has || cur == c0)) {
        Agg r;
        r.sum = wsum(a.sum);
        r.asum = wsum(a.asum);
        if (with_tl) {
            r.tsum = wsum(a.tsum);
            r.tasum = wsum(a.tasum);
            r.lsum = wsum(a.lsum);
            r.lasum = wsum(a.lasum);
        }
        uint32_t cnt = a.cnt, mn = a.mn, mx = a.mx;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
            mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        r.cnt = cnt, r.mn = mn, r.mx = mx;
        if ((threadIdx.x & 31) == static_cast<unsigned>(__ffs(m) - 1)) stats_atomic_at(st, c0, r, with_tl);
    } else if (has) {
        stats_atomic_at(st, cur, a, with_tl);
    }
    agg_reset(a);
}

__global__ void stripe_zero_kernel(Stats* stripe, uint32_t n) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    Stats z;
    z.sum = z.asum = z.tsum = z.tasum = z.lsum = z.lasum = 0.0;
    z.cnt = 0, z.mn = 0xffffffffu, z.mx = 0u, z.pad = 0;
    stripe[i] = z;
}

// fold owner lo + i's 32 stripes into its Stats (which the sweep left untouched)
__global__ void stripe_combine_kernel(const Stats* stripe, uint32_t lo, uint32_t n, Stats* st) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    Stats& t = st[lo + i];
    for (uint32_t k = 0; k < kStripes; ++k) {
        const Stats& z = stripe[i * kStripes + k];
        if (!z.cnt) continue;
        t.sum += z.sum, t.asum += z.asum, t.tsum += z.tsum, t.tasum += z.tasum, t.lsum += z.lsum,
            t.lasum += z.lasum;
        t.cnt += z.cnt;
        t.mn = min(t.mn, z.mn);
        t.mx = max(t.mx, z.mx);
    }
}

// root of voxel centre p (tet_grid.cpp:435-451): the root whose pyramid and
// face triangle hold p, accepted with a 1e-9 interior margin (every other root
// is then violated far beyond the scan's 1e-12), else the reference's scan
__device__ __forceinline__ uint32_t root_of(const RootScan& R, const uint4* verts, d3 p) {
    const int g = guess_root(p);
    double worst = -__longlong_as_double(0x7ff0000000000000ll);
    for (int slot = 0; slot < 4; ++slot) {
        const uint32_t id = (R.nid[g] >> (8 * slot)) & 0xffu;
        const d3 w = sub(p, vpos(verts[R.vid[g][(slot + 1) & 3]]));
        worst = dmax(worst, ndot(id, w.x, w.y, w.z));
    }
    if (worst <= -1e-9) return R.id[g];
    uint32_t o = kNone;
    double best = __longlong_as_double(0x7ff0000000000000ll);
    for (int rr = 0; rr < 24; ++rr) {
        double wv = 0.0;
        for (int slot = 0; slot < 4; ++slot) {
            const uint32_t id = (R.nid[rr] >> (8 * slot)) & 0xffu;
            const d3 w = sub(p, vpos(verts[R.vid[rr][(slot + 1) & 3]]));
            wv = dmax(wv, ndot(id, w.x, w.y, w.z));
        }
        if (wv <= 1e-12) return R.id[rr];
        if (wv < best) best = wv, o = R.id[rr];
    }
    return o;
}

// q = x / d for x < 2^37 (4096^3 voxels) through the f64 reciprocal: x * RN(1/d) is within
// 2^-15 of x / d, so the truncated product is off by at most one and one correction each way
// makes it exact (the integer divisions it replaces were 38 % of the sweep's instructions).
__device__ __forceinline__ uint64_t div_small(uint64_t x, uint32_t d, double rd, uint32_t& rem) {
    uint64_t q = static_cast<uint64_t>(static_cast<double>(x) * rd);
    int64_t r = static_cast<int64_t>(x - q * d);
    if (r < 0) --q, r += d;
    else if (r >= static_cast<int64_t>(d)) ++q, r -= d;
    rem = static_cast<uint32_t>(r);
    return q;
}

__device__ __forceinline__ void voxel_ijk(const VolView& V, uint64_t idx, int& i, int& j, int& k) {
    uint32_t ri, rj;
    const uint64_t row = div_small(idx, V.nx, V.rnx, ri);
    k = static_cast<int>(div_small(row, V.ny, V.rny, rj));
    i = static_cast<int>(ri), j = static_cast<int>(rj);
}

__device__ __forceinline__ d3 voxel_centre(const VolView& V, uint64_t idx) {
    int i, j, k;
    voxel_ijk(V, idx, i, j, k);
    return mk(__ldg(V.cx + i), __ldg(V.cy + j), __ldg(V.cz + k));  // (i + 0.5) / nx ... (volume.hpp:44-46)
}

// descent from a bisected owner to the leaf holding p (tet_grid.cpp:453-470)
__device__ __forceinline__ uint32_t descend(const NodeRec* split, const uint8_t* flags, uint32_t o, d3 p) {
    do {
        const NodeRec& nd = split[o];
        const double sp = dot(mk(nd.n[0], nd.n[1], nd.n[2]), sub(p, mk(nd.pm[0], nd.pm[1], nd.pm[2])));
        const bool take_a = nd.sref_pos ? (sp >= 0.0) : (sp <= 0.0);
        o = take_a ? nd.child[0] : nd.child[1];
    } while (!(flags[o] & F_LEAF));
    return o;
}

// Sweep order: the volume is read as a flat array in groups of four voxels
// (one 16-B owner load, one 16-B density load); a warp's chunk is 32 *
// kVoxLaneGroups consecutive groups (one contiguous span).
constexpr int kVoxLaneGroups = 4;  // 16 voxels per lane, 512 per warp chunk

struct VoxLane {
    uint32_t cur = kNone;
    Agg a;
};

__device__ __forceinline__ void vox_add(const StatsSink& st, VoxLane& L, uint32_t o, float x, const VolView& V,
                                        uint64_t idx, bool with_tl) {
    if (o != L.cur) {
        if (L.a.cnt) stats_atomic_at(st, L.cur, L.a, with_tl);
        agg_reset(L.a);
        L.cur = o;
    }
    L.a.sum += static_cast<double>(x);
    L.a.asum += fabs(static_cast<double>(x));
    L.a.cnt += 1;
    L.a.mn = min(L.a.mn, ord_f(x));
    L.a.mx = max(L.a.mx, ord_f(x));
    if (with_tl) {
        if (V.temp) {
            const double tv = V.temp[idx];
            L.a.tsum += tv;
            L.a.tasum += fabs(tv);
        }
        if (V.alb) {
            const double lv = V.alb[idx];
            L.a.lsum += lv;
            L.a.lasum += fabs(lv);
        }
    }
}

template <int mode>
__global__ void __launch_bounds__(kVoxThreads, mode == kVoxDescend ? TV_VOX_DESC_BLOCKS : 3) vox_stats_kernel(VolView V, RootScan R, const uint4* verts,
                                                                 const NodeRec* split, const uint8_t* flags,
                                                                 uint32_t* owner, StatsSink st, int with_tl_arg) {
    // the temperature / albedo sums exist in the payload pass only: a compile-time
    // flag lets the other modes drop their registers and instructions
    constexpr bool with_tl = mode == kVoxAll;
    (void)with_tl_arg;
    const uint64_t nvox = static_cast<uint64_t>(V.nx) * V.ny * V.nz;
    const uint64_t n4 = nvox / 4;
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t n_warps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
    const uint64_t per_warp = 32ull * kVoxLaneGroups;
    uint4* own4 = reinterpret_cast<uint4*>(owner);
    const float4* d4p = reinterpret_cast<const float4*>(V.dens);
    // Groups are interleaved over the lanes (group q * 32 + lane of the warp's
    // chunk), so every 16-B owner / density load of the warp is coalesced.
    // kVoxDescend: the voxels to process (owner bisected) are a sparse, ragged
    // subset of each chunk; unless most of the chunk is dirty they are first
    // compacted per warp (shared memory, voxel order kept) and split into equal
    // contiguous slices, one per lane: every lane descends and accumulates the
    // same number of voxels, and a lane's voxels stay contiguous, so its owner
    // runs survive. Dense chunks take the same vectorised path as the other modes.
    __shared__ uint32_t s_pick[mode == kVoxDescend ? kVoxThreads / 32 : 1][32 * 4 * kVoxLaneGroups];
    for (uint64_t c = warp * per_warp; c < n4; c += n_warps * per_warp) {
        VoxLane L;
        agg_reset(L.a);
        uint32_t dirty = 0xffffffffu;  // bit 4q + k: voxel k of this lane's group q is to be processed
        if (mode == kVoxDescend) {
            dirty = 0;
#pragma unroll
            for (int q = 0; q < kVoxLaneGroups; ++q) {
                const uint64_t g = c + static_cast<uint64_t>(q) * 32 + lane;
                if (g < n4) {
                    const uint4 o4 = own4[g];
                    // voxels whose owner is still a leaf keep it and were counted
                    // when it was evaluated: skip them (no density read)
                    dirty |= ((!(flags[o4.x] & F_LEAF) ? 1u : 0u) | (!(flags[o4.y] & F_LEAF) ? 2u : 0u) |
                              (!(flags[o4.z] & F_LEAF) ? 4u : 0u) | (!(flags[o4.w] & F_LEAF) ? 8u : 0u))
                             << (4 * q);
                }
            }
            const uint32_t total = __reduce_add_sync(0xffffffffu, __popc(dirty));
            if (total * 4 <= 3 * 32 * 4 * kVoxLaneGroups) {  // sparse: compact, then equal slices
                uint32_t* pick = s_pick[threadIdx.x >> 5];
                uint32_t base = 0;
#pragma unroll
                for (int q = 0; q < kVoxLaneGroups; ++q) {
                    const uint32_t dq = (dirty >> (4 * q)) & 15u;
                    const uint32_t cnt = __popc(dq);
                    uint32_t pre = cnt;  // inclusive prefix over the lanes (voxel order within q)
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t v = __shfl_up_sync(0xffffffffu, pre, o);
                        if (lane >= o) pre += v;
                    }
                    uint32_t at = base + pre - cnt;
                    for (uint32_t b = dq; b; b &= b - 1)
                        pick[at++] = (static_cast<uint32_t>(q) * 32 + lane) * 4 + __ffs(b) - 1;
                    base += __shfl_sync(0xffffffffu, pre, 31);
                }
                __syncwarp();
                const uint32_t lo = total * lane / 32, hi = total * (lane + 1) / 32;
                for (uint32_t e = lo; e < hi; ++e) {
                    const uint64_t idx = 4 * c + pick[e];
                    const uint32_t o = descend(split, flags, owner[idx], voxel_centre(V, idx));
                    owner[idx] = o;
                    vox_add(st, L, o, V.dens[idx], V, idx, with_tl);
                }
                __syncwarp();
                warp_flush(st, L.cur, L.a, with_tl);
                continue;
            }
        }
#pragma unroll 1
        for (int q = 0; q < kVoxLaneGroups; ++q) {
            const uint64_t g = c + static_cast<uint64_t>(q) * 32 + lane;
            const uint32_t dq = (dirty >> (4 * q)) & 15u;
            if (g >= n4 || !dq) continue;
            const uint64_t idx0 = 4 * g;
            // the group's centres: one index split when the group lies in one x row (nx % 4 == 0)
            int gi = 0, gj = 0, gk = 0;
            if (mode != kVoxAll && (V.nx & 3) == 0) voxel_ijk(V, idx0, gi, gj, gk);
            auto centre = [&](int t) -> d3 {
                if ((V.nx & 3) == 0) return mk(__ldg(V.cx + gi + t), __ldg(V.cy + gj), __ldg(V.cz + gk));
                return voxel_centre(V, idx0 + t);
            };
            uint4 o4;
            if (mode == kVoxInit) {
                o4.x = root_of(R, verts, centre(0));
                o4.y = root_of(R, verts, centre(1));
                o4.z = root_of(R, verts, centre(2));
                o4.w = root_of(R, verts, centre(3));
                own4[g] = o4;
            } else {
                o4 = own4[g];
            }
            const float4 d4 = d4p[g];
            if (mode == kVoxDescend) {  // dense chunk: descend the dirty voxels of the group
                if (dq & 1u) o4.x = descend(split, flags, o4.x, centre(0));
                if (dq & 2u) o4.y = descend(split, flags, o4.y, centre(1));
                if (dq & 4u) o4.z = descend(split, flags, o4.z, centre(2));
                if (dq & 8u) o4.w = descend(split, flags, o4.w, centre(3));
                own4[g] = o4;
            }
            if (dq & 1u) vox_add(st, L, o4.x, d4.x, V, idx0, with_tl);
            if (dq & 2u) vox_add(st, L, o4.y, d4.y, V, idx0 + 1, with_tl);
            if (dq & 4u) vox_add(st, L, o4.z, d4.z, V, idx0 + 2, with_tl);
            if (dq & 8u) vox_add(st, L, o4.w, d4.w, V, idx0 + 3, with_tl);
        }
        warp_flush(st, L.cur, L.a, with_tl);
    }
    // the last nvox % 4 voxels, scalar
    if (blockIdx.x == 0 && threadIdx.x < nvox - 4 * n4) {
        const uint64_t idx = 4 * n4 + threadIdx.x;
        uint32_t o = mode == kVoxInit ? root_of(R, verts, voxel_centre(V, idx)) : owner[idx];
        bool add = true;
        if (mode == kVoxDescend) {
            if (flags[o] & F_LEAF) add = false;
            else o = descend(split, flags, o, voxel_centre(V, idx));
        }
        if (mode != kVoxAll) owner[idx] = o;
        if (add) {
            VoxLane L;
            agg_reset(L.a);
            vox_add(st, L, o, V.dens[idx], V, idx, with_tl);
            stats_atomic_at(st, L.cur, L.a, with_tl);
        }
    }
}

// ------------------------------------------------------------ voxel bricks
// While the leaves are much larger than a voxel (the early rounds), nearly
// every voxel of a bisected leaf goes to the same child as its neighbours. The
// volume is therefore also tiled into 8x8x8 bricks. A brick whose 512 voxels
// all have one owner keeps that owner in brick_owner[b] (its per-voxel owner
// words are not maintained) plus its precomputed density statistics; round 0
// finds those bricks with a corner test against the roots (brick_root_kernel). When its
// owner is bisected, the brick descends as a whole while the split plane keeps
// its eight corner centres strictly on one side (margin 1e-9 |n|_1; the side
// test of every voxel centre inside is then the same, FP rounding included),
// and its statistics go to the child leaf in one add. A brick that a plane
// cuts becomes mixed: it joins the mixed list, and from then on its voxels
// are handled one by one (brick_voxels_kernel). Bricks cut by the volume
// border are mixed from the start. The owner of voxel v is brick_owner[b(v)]
// unless that is kBrickMixed, then owner[v] (owner_at).
constexpr int kBrick = 8;  // brick edge in voxels (4 was measured: more brick overhead than it saves)
constexpr int kBrickLog = 3;
constexpr int kBrickVox = kBrick * kBrick * kBrick;
constexpr uint32_t kBrickMixed = 0xffffffffu;  // mixed: per-voxel owner words valid
constexpr uint32_t kBrickFresh = 0x80000000u;  // | o: mixed this round; every voxel's owner is still o
struct BrickStat {
    double sum, asum;
    uint32_t cnt, mn, mx, pad;
};

// Bricks that may hold a voxel whose owner a closure pass bisects: the bricks
// of the bisected tet's voxel bounding box (a voxel centre lies inside its
// owner). The next round's mixed-brick pass visits only those. A tet whose box
// spans more than kMarkMax bricks marks its super-bricks (8x8x8 bricks) in a
// second bitmap instead, and one spanning more than kMarkMax super-bricks the
// all-bricks word.
struct BrickMark {
    uint32_t* bits;   // 1 bit per brick; null: no bricks
    uint32_t* sbits;  // 1 bit per super-brick, then the all-bricks word
    uint32_t n_swords;
    int nx, ny, nz, gbx, gby, gsx, gsy;
};
constexpr int kMarkMax = 256;

__device__ __forceinline__ bool brick_marked(const BrickMark& M, uint32_t b, int gbx, int gby) {
    if ((M.bits[b >> 5] >> (b & 31)) & 1u) return true;
    const uint32_t bx = b % gbx, by = (b / gbx) % gby, bz = b / (static_cast<uint32_t>(gbx) * gby);
    const uint32_t sb = ((bz >> 3) * M.gsy + (by >> 3)) * M.gsx + (bx >> 3);
    return (M.sbits[sb >> 5] >> (sb & 31)) & 1u;
}

__device__ void mark_bricks(const BrickMark& M, const uint4* verts, const tv_tet& t) {
    if (!M.bits) return;
    double lo[3] = {1.0, 1.0, 1.0}, hi[3] = {0.0, 0.0, 0.0};
    for (int k = 0; k < 4; ++k) {
        const d3 c = vpos(verts[t.verts[k]]);
        lo[0] = dmin(lo[0], c.x), lo[1] = dmin(lo[1], c.y), lo[2] = dmin(lo[2], c.z);
        hi[0] = dmax(hi[0], c.x), hi[1] = dmax(hi[1], c.y), hi[2] = dmax(hi[2], c.z);
    }
    const int dims[3] = {M.nx, M.ny, M.nz};
    int b0[3], b1[3];
    uint64_t count = 1, scount = 1;
    for (int a = 0; a < 3; ++a) {  // centre (i + 0.5) / n in [lo, hi], widened by one voxel
        const int i0 = max(0, static_cast<int>(floor(lo[a] * dims[a] - 0.5)) - 1);
        const int i1 = min(dims[a] - 1, static_cast<int>(ceil(hi[a] * dims[a] - 0.5)) + 1);
        b0[a] = i0 >> kBrickLog, b1[a] = i1 >> kBrickLog;
        count *= static_cast<uint64_t>(max(0, b1[a] - b0[a] + 1));
        scount *= static_cast<uint64_t>(max(0, (b1[a] >> 3) - (b0[a] >> 3) + 1));
    }
    if (count <= kMarkMax) {
        for (int z = b0[2]; z <= b1[2]; ++z)
            for (int y = b0[1]; y <= b1[1]; ++y)
                for (int x = b0[0]; x <= b1[0]; ++x) {
                    const uint32_t b = (static_cast<uint32_t>(z) * M.gby + y) * M.gbx + x;
                    atomicOr(M.bits + (b >> 5), 1u << (b & 31));
                }
    } else if (scount <= kMarkMax) {
        for (int z = b0[2] >> 3; z <= (b1[2] >> 3); ++z)
            for (int y = b0[1] >> 3; y <= (b1[1] >> 3); ++y)
                for (int x = b0[0] >> 3; x <= (b1[0] >> 3); ++x) {
                    const uint32_t sb = (static_cast<uint32_t>(z) * M.gsy + y) * M.gsx + x;
                    atomicOr(M.sbits + (sb >> 5), 1u << (sb & 31));
                }
    } else {
        atomicOr(M.sbits + M.n_swords - 1, 1u);
    }
}


__device__ __forceinline__ uint32_t owner_at(const VolView& V, const uint32_t* owner, int i, int j, int k,
                                             uint64_t idx) {
    if (V.brick) {
        const uint64_t b = (static_cast<uint64_t>(k >> kBrickLog) * V.gby + (j >> kBrickLog)) * V.gbx + (i >> kBrickLog);
        const uint32_t bo = V.brick[b];
        if (bo != kBrickMixed) return bo;
        const uint32_t so = V.sub[8 * b + (((i >> 2) & 1) | (((j >> 2) & 1) << 1) | (((k >> 2) & 1) << 2))];
        if (so != kBrickMixed) return so;
    }
    return owner[idx];
}

__device__ __forceinline__ void list_append(uint32_t* list, uint32_t* n, uint32_t b, bool add) {
    const unsigned m = __ballot_sync(0xffffffffu, add);
    if (!m) return;
    const int lane = threadIdx.x & 31, lead = __ffs(m) - 1;
    uint32_t base = 0;
    if (lane == lead) base = atomicAdd(n, static_cast<uint32_t>(__popc(m)));
    base = __shfl_sync(0xffffffffu, base, lead);
    if (add) list[base + __popc(m & ((1u << lane) - 1u))] = b;
}

// Descent of a box of voxel centres (corner coordinates xs, ys, zs) from node o:
// true with o = the leaf when every split plane on the way keeps all eight
// corners strictly on one side (margin 1e-9 |n|_1; sp is linear in p, so every
// centre inside takes the same branch, rounding included), false with o = the
// node whose plane cuts the box.
__device__ __forceinline__ bool box_descend(const NodeRec* split, const uint8_t* flags, uint32_t& o, const double* xs,
                                            const double* ys, const double* zs) {
    for (;;) {
        const NodeRec& nd = split[o];
        const double n0 = nd.n[0], n1 = nd.n[1], n2 = nd.n[2];
        const double margin = 1e-9 * (fabs(n0) + fabs(n1) + fabs(n2));
        double lo = __longlong_as_double(0x7ff0000000000000ll), hi = -lo;
#pragma unroll
        for (int c = 0; c < 8; ++c) {  // the reference's sp = dot(n, p - pm), left to right
            const double sp =
                (n0 * (xs[c & 1] - nd.pm[0]) + n1 * (ys[(c >> 1) & 1] - nd.pm[1])) + n2 * (zs[c >> 2] - nd.pm[2]);
            lo = dmin(lo, sp);
            hi = dmax(hi, sp);
        }
        const bool pos = lo > margin, neg = hi < -margin;
        if (!pos && !neg) return false;
        const bool take_a = nd.sref_pos ? pos : neg;  // sp >= 0 (sref_pos) or sp <= 0, strictly here
        o = take_a ? nd.child[0] : nd.child[1];
        if (flags[o] & F_LEAF) return true;
    }
}

// Round 0 with bricks: a full brick whose eight corner centres lie inside the
// root guessed for its first corner, by more than root_of's 1e-9 acceptance
// margin on each of the root's planes (plus 1e-9 for rounding), has that root
// for every voxel: root_of's own test accepts every centre inside, and a
// centre whose guess differs falls to the reference scan, which can only
// accept that same root (every other root is violated by more than 1e-12).
// Such a brick becomes uniform with its statistics added to the root in one
// step; every other brick takes root_of voxel by voxel and becomes mixed.
__global__ void __launch_bounds__(kVoxThreads, 3) brick_root_kernel(VolView V, RootScan R, const uint4* verts,
                                                                    uint32_t* owner, uint32_t* brick, uint32_t* subo,
                                                                    BrickStat* bstat, StatsSink st, uint32_t* mixed,
                                                                    uint32_t* n_mixed) {
    const uint32_t n_b = static_cast<uint32_t>(V.gbx) * V.gby * ((V.nz + kBrick - 1) / kBrick);
    const int lane = threadIdx.x & 31;
    const uint32_t w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t b = w0; b < n_b; b += nw) {  // warp-uniform loop
        const int bx = static_cast<int>(b % V.gbx), by = static_cast<int>((b / V.gbx) % V.gby),
                  bz = static_cast<int>(b / (static_cast<uint32_t>(V.gbx) * V.gby));
        const int x0 = bx * kBrick, y0 = by * kBrick, z0 = bz * kBrick;
        const bool full = x0 + kBrick <= V.nx && y0 + kBrick <= V.ny && z0 + kBrick <= V.nz;
        bool uniform = false;
        int g = 0;
        if (full) {
            g = guess_root(mk(__ldg(V.cx + x0), __ldg(V.cy + y0), __ldg(V.cz + z0)));
            double worst = -1.0;
            if (lane < 8) {
                const d3 p = mk(__ldg(V.cx + x0 + ((lane & 1) ? kBrick - 1 : 0)),
                                __ldg(V.cy + y0 + ((lane & 2) ? kBrick - 1 : 0)),
                                __ldg(V.cz + z0 + ((lane & 4) ? kBrick - 1 : 0)));
                worst = -__longlong_as_double(0x7ff0000000000000ll);
                for (int slot = 0; slot < 4; ++slot) {
                    const uint32_t id = (R.nid[g] >> (8 * slot)) & 0xffu;
                    const d3 w = sub(p, vpos(verts[R.vid[g][(slot + 1) & 3]]));
                    worst = dmax(worst, ndot(id, w.x, w.y, w.z));
                }
            }
            uniform = __all_sync(0xffffffffu, worst <= -2e-9);
        }
        if (uniform) {
            double sum = 0.0, asum = 0.0;
            uint32_t mn = 0xffffffffu, mx = 0u;
            for (int v = lane; v < kBrickVox; v += 32) {  // x fastest: lanes read consecutive voxels
                const int x = x0 + (v & (kBrick - 1)), y = y0 + ((v >> kBrickLog) & (kBrick - 1)),
                          z = z0 + (v >> (2 * kBrickLog));
                const float d = V.dens[(static_cast<uint64_t>(z) * V.ny + y) * V.nx + x];
                sum += static_cast<double>(d);
                asum += fabs(static_cast<double>(d));
                mn = min(mn, ord_f(d));
                mx = max(mx, ord_f(d));
            }
            sum = wsum(sum);
            asum = wsum(asum);
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
                mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            }
            const uint32_t root = R.id[g];
            if (lane == 0) {
                brick[b] = root;
                bstat[b] = BrickStat{sum, asum, static_cast<uint32_t>(kBrickVox), mn, mx, 0u};
            }
            // one lane per brick adds to the root, a different stripe lane per brick
            if (lane == static_cast<int>(b & 31)) {
                Agg a;
                agg_reset(a);
                a.sum = sum, a.asum = asum, a.cnt = kBrickVox, a.mn = mn, a.mx = mx;
                stats_atomic_at(st, root, a, false);
            }
            continue;
        }
        // voxel by voxel (lane: rows lane and lane + 32 of the 64 (y, z) rows)
        VoxLane L;
        agg_reset(L.a);
        const int nxr = min(kBrick, V.nx - x0);
        for (int h = 0; h < 2; ++h) {
            const int r = lane + 32 * h, y = y0 + (r & 7), z = z0 + (r >> 3);
            if (y >= V.ny || z >= V.nz) continue;
            const uint64_t base = (static_cast<uint64_t>(z) * V.ny + y) * V.nx + x0;
            const double py = __ldg(V.cy + y), pz = __ldg(V.cz + z);
            for (int x = 0; x < nxr; ++x) {
                const uint32_t o = root_of(R, verts, mk(__ldg(V.cx + x0 + x), py, pz));
                owner[base + x] = o;
                vox_add(st, L, o, V.dens[base + x], V, base + x, false);
            }
        }
        warp_flush(st, L.cur, L.a, false);
        if (lane < 8) subo[8ull * b + lane] = kBrickMixed;
        if (lane == 0) {
            brick[b] = kBrickMixed;
            mixed[atomicAdd(n_mixed, 1u)] = b;
        }
    }
}

// K1 of a round: every uniform brick whose owner was bisected descends as a
// whole while its corners agree, or becomes mixed (fresh) at the first plane
// that cuts it. One thread per brick.
__global__ void brick_descend_kernel(VolView V, uint32_t n_b, uint32_t* brick, const BrickStat* bstat,
                                     const NodeRec* split, const uint8_t* flags, StatsSink st, uint32_t* mixed,
                                     uint32_t* n_mixed) {
    for (uint32_t b0 = blockIdx.x * blockDim.x; b0 < n_b; b0 += gridDim.x * blockDim.x) {  // warp-uniform
        const uint32_t b = b0 + threadIdx.x;
        uint32_t bo = b < n_b ? brick[b] : kBrickMixed;
        bool work = !(bo & kBrickFresh) && !(flags[bo] & F_LEAF);
        bool cut = false;
        Agg a;
        agg_reset(a);
        if (work) {
            const int bx = static_cast<int>(b % V.gbx), by = static_cast<int>((b / V.gbx) % V.gby),
                      bz = static_cast<int>(b / (static_cast<uint32_t>(V.gbx) * V.gby));
            const double xs[2] = {__ldg(V.cx + bx * kBrick), __ldg(V.cx + bx * kBrick + kBrick - 1)};
            const double ys[2] = {__ldg(V.cy + by * kBrick), __ldg(V.cy + by * kBrick + kBrick - 1)};
            const double zs[2] = {__ldg(V.cz + bz * kBrick), __ldg(V.cz + bz * kBrick + kBrick - 1)};
            uint32_t o = bo;
            for (;;) {
                const NodeRec& nd = split[o];
                const double n0 = nd.n[0], n1 = nd.n[1], n2 = nd.n[2];
                const double margin = 1e-9 * (fabs(n0) + fabs(n1) + fabs(n2));
                double lo = __longlong_as_double(0x7ff0000000000000ll), hi = -lo;
#pragma unroll
                for (int c = 0; c < 8; ++c) {  // the reference's sp = dot(n, p - pm), left to right
                    const double sp = (n0 * (xs[c & 1] - nd.pm[0]) + n1 * (ys[(c >> 1) & 1] - nd.pm[1])) +
                                      n2 * (zs[c >> 2] - nd.pm[2]);
                    lo = dmin(lo, sp);
                    hi = dmax(hi, sp);
                }
                const bool pos = lo > margin, neg = hi < -margin;
                if (!pos && !neg) {
                    cut = true;
                    bo = o;
                    break;
                }
                const bool take_a = nd.sref_pos ? pos : neg;  // sp >= 0 (sref_pos) or sp <= 0, strictly here
                o = take_a ? nd.child[0] : nd.child[1];
                if (flags[o] & F_LEAF) break;
            }
            if (cut) {
                brick[b] = kBrickFresh | bo;
            } else {
                brick[b] = o;
                const BrickStat s = bstat[b];
                a.sum = s.sum, a.asum = s.asum, a.cnt = s.cnt, a.mn = s.mn, a.mx = s.mx;
                bo = o;
            }
        }
        warp_flush(st, bo, a, false);
        list_append(mixed, n_mixed, b, cut);
    }
}

// K2 of a round: every mixed brick, one warp per brick, in 4x4x4 sub-bricks.
// A sub-brick with one owner keeps it in sub[8b + s] (its owner words are not
// maintained) and moves down the tree whole while no plane cuts it, like a
// brick (lanes 0-7, one sub-brick each); its statistics are computed when its
// brick is cut (fresh). A cut sub-brick's voxels, and those of sub-bricks that
// are already per-voxel, are handled one by one: a lane takes rows lane and
// lane + 32 of the brick's 64 (y, z) rows, loads the owner words and flags of
// its voxels before any descent, then descends the dirty ones.
__global__ void __launch_bounds__(kVoxThreads, 4) brick_voxels_kernel(VolView V, uint32_t* brick, uint32_t* subo,
                                                                      BrickStat* sstat, const uint32_t* mixed,
                                                                      const uint32_t* n_mixed, const NodeRec* split,
                                                                      const uint8_t* flags, uint32_t* owner,
                                                                      StatsSink st, BrickMark bm) {
    const uint32_t n = *n_mixed;
    const int lane = threadIdx.x & 31;
    const uint32_t w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    const bool all = !bm.bits || (bm.sbits[bm.n_swords - 1] & 1u);
    for (uint32_t e = w0; e < n; e += nw) {  // warp-uniform loop
        const uint32_t b = mixed[e];
        if (!all && !brick_marked(bm, b, V.gbx, V.gby)) continue;  // no owner here was bisected
        const uint32_t bo = brick[b];
        const bool fresh = bo != kBrickMixed;  // cut this round: every voxel's owner is `fill`
        const uint32_t fill = bo & ~kBrickFresh;
        const int bx = static_cast<int>(b % V.gbx), by = static_cast<int>((b / V.gbx) % V.gby),
                  bz = static_cast<int>(b / (static_cast<uint32_t>(V.gbx) * V.gby));
        const int x0 = bx * kBrick, y0 = by * kBrick, z0 = bz * kBrick, nxr = min(kBrick, V.nx - x0);
        uint32_t* sb = subo + 8ull * b;
        BrickStat* ss = sstat + 8ull * b;
        // a fresh brick (always full): the statistics of its eight sub-bricks. Lane
        // rows h = 0, 1 have y = y0 + (lane & 7), z = z0 + (lane >> 3) + 4h, so the
        // sub-brick of half xh is xh | (lane & 4 ? 2 : 0) | 4h; lanes that share
        // lane & 4 are summed (xor over lane bits 0, 1, 3, 4)
        if (fresh) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint64_t base =
                    (static_cast<uint64_t>(z0 + (lane >> 3) + 4 * h) * V.ny + (y0 + (lane & 7))) * V.nx + x0;
#pragma unroll
                for (int xh = 0; xh < 2; ++xh) {
                    double sum = 0.0, asum = 0.0;
                    uint32_t mn = 0xffffffffu, mx = 0u;
#pragma unroll
                    for (int x = 0; x < 4; ++x) {
                        const float d = V.dens[base + 4 * xh + x];
                        sum += static_cast<double>(d);
                        asum += fabs(static_cast<double>(d));
                        mn = min(mn, ord_f(d));
                        mx = max(mx, ord_f(d));
                    }
#pragma unroll
                    for (int m : {1, 2, 8, 16}) {
                        sum += __shfl_xor_sync(0xffffffffu, sum, m);
                        asum += __shfl_xor_sync(0xffffffffu, asum, m);
                        mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, m));
                        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, m));
                    }
                    if ((lane & ~4) == 0) ss[xh | ((lane & 4) ? 2 : 0) | (4 * h)] = BrickStat{sum, asum, 64u, mn, mx, 0u};
                }
            }
            __syncwarp();
        }
        // lanes 0-7: the sub-brick decisions
        int mode = 0;  // 0 nothing to do, 1 per-voxel (owner words), 2 cut now (every voxel from `ocut`)
        uint32_t ocut = 0, cur = kNone;
        Agg a;
        agg_reset(a);
        if (lane < 8) {
            const uint32_t u = fresh ? fill : sb[lane];
            if (u == kBrickMixed) {
                mode = 1;
            } else if (fresh || !(flags[u] & F_LEAF)) {
                const int sx = x0 + 4 * (lane & 1), sy = y0 + 2 * (lane & 2), sz = z0 + (lane & 4);
                const double xs[2] = {__ldg(V.cx + sx), __ldg(V.cx + sx + 3)};
                const double ys[2] = {__ldg(V.cy + sy), __ldg(V.cy + sy + 3)};
                const double zs[2] = {__ldg(V.cz + sz), __ldg(V.cz + sz + 3)};
                uint32_t o = u;
                if (box_descend(split, flags, o, xs, ys, zs)) {
                    sb[lane] = o;
                    const BrickStat t = ss[lane];
                    a.sum = t.sum, a.asum = t.asum, a.cnt = t.cnt, a.mn = t.mn, a.mx = t.mx;
                    cur = o;
                } else {
                    sb[lane] = kBrickMixed;
                    mode = 2;
                    ocut = o;
                }
            }
        }
        warp_flush(st, cur, a, false);
        const uint32_t m1 = __ballot_sync(0xffffffffu, mode == 1) & 0xffu, m2 = __ballot_sync(0xffffffffu, mode == 2) & 0xffu;
        if (m1 | m2) {
            uint32_t oc[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) oc[k] = __shfl_sync(0xffffffffu, ocut, k);
            uint32_t own[2][kBrick];
            uint32_t dirty = 0;  // bit 8h + x
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int r = lane + 32 * h, y = y0 + (r & 7), z = z0 + (r >> 3);
                const bool row_ok = y < V.ny && z < V.nz;
                const uint64_t base = (static_cast<uint64_t>(z) * V.ny + y) * V.nx + x0;
#pragma unroll
                for (int xh = 0; xh < 2; ++xh) {
                    const int sbi = xh | ((r & 4) ? 2 : 0) | ((r & 32) ? 4 : 0);
                    const uint32_t vmask = row_ok ? (((1u << max(0, min(4, nxr - 4 * xh))) - 1u) << (4 * xh)) : 0u;
                    if ((m2 >> sbi) & 1u) {
#pragma unroll
                        for (int x = 0; x < 4; ++x) own[h][4 * xh + x] = oc[sbi];
                        dirty |= vmask << (8 * h);
                    } else if (((m1 >> sbi) & 1u) && vmask) {
                        if (vmask == (0xfu << (4 * xh)) && (V.nx & 3) == 0) {  // 16-B aligned half row
                            const uint4 q = *reinterpret_cast<const uint4*>(owner + base + 4 * xh);
                            own[h][4 * xh] = q.x, own[h][4 * xh + 1] = q.y, own[h][4 * xh + 2] = q.z,
                                        own[h][4 * xh + 3] = q.w;
                        } else {
#pragma unroll
                            for (int x = 0; x < 4; ++x)
                                own[h][4 * xh + x] = (vmask >> (4 * xh + x)) & 1u ? owner[base + 4 * xh + x] : 0u;
                        }
#pragma unroll
                        for (int x = 0; x < 4; ++x)
                            if (((vmask >> (4 * xh + x)) & 1u) && !(flags[own[h][4 * xh + x]] & F_LEAF))
                                dirty |= 1u << (8 * h + 4 * xh + x);
                    }
                }
            }
            VoxLane L;
            agg_reset(L.a);
            if (__any_sync(0xffffffffu, dirty != 0)) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint32_t dh = (dirty >> (8 * h)) & 0xffu;
                    if (!dh) continue;
                    const int r = lane + 32 * h, y = y0 + (r & 7), z = z0 + (r >> 3);
                    const uint64_t base = (static_cast<uint64_t>(z) * V.ny + y) * V.nx + x0;
                    const double py = __ldg(V.cy + y), pz = __ldg(V.cz + z);
#pragma unroll
                    for (int x = 0; x < kBrick; ++x) {
                        if (!((dh >> x) & 1u)) continue;
                        const uint32_t o = descend(split, flags, own[h][x], mk(__ldg(V.cx + x0 + x), py, pz));
                        owner[base + x] = o;
                        vox_add(st, L, o, V.dens[base + x], V, base + x, false);
                    }
                }
            }
            warp_flush(st, L.cur, L.a, false);
        }
        if (fresh && lane == 0) brick[b] = kBrickMixed;
    }
}

// before the payload pass: the owner words of the uniform bricks, so that the
// owner map alone is authoritative again (one warp per brick)
__global__ void brick_fill_kernel(VolView V, const uint32_t* brick, const uint32_t* subo, uint32_t n_b,
                                  uint32_t* owner) {
    const int lane = threadIdx.x & 31;
    const uint32_t w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t b = w0; b < n_b; b += nw) {
        const uint32_t bo = brick[b];
        const int bx = static_cast<int>(b % V.gbx), by = static_cast<int>((b / V.gbx) % V.gby),
                  bz = static_cast<int>(b / (static_cast<uint32_t>(V.gbx) * V.gby));
        for (int v = lane; v < kBrickVox; v += 32) {
            const int i = v & (kBrick - 1), j = (v >> kBrickLog) & (kBrick - 1), k = v >> (2 * kBrickLog);
            const uint32_t o = bo != kBrickMixed ? bo : subo[8ull * b + ((i >> 2) | ((j >> 2) << 1) | ((k >> 2) << 2))];
            if (o == kBrickMixed) continue;  // owner word valid
            owner[(static_cast<uint64_t>(bz * kBrick + k) * V.ny + (by * kBrick + j)) * V.nx + bx * kBrick + i] = o;
        }
    }
}

// volume.cpp:47-66
__device__ double trilinear(const float* data, int nx, int ny, int nz, d3 p) {
    const double fx = p.x * nx - 0.5, fy = p.y * ny - 0.5, fz = p.z * nz - 0.5;
    int i0 = static_cast<int>(floor(fx)), j0 = static_cast<int>(floor(fy)), k0 = static_cast<int>(floor(fz));
    const double tx = fx - i0, ty = fy - j0, tz = fz - k0;
    auto cl = [](int v, int n) { return v < 0 ? 0 : (v > n - 1 ? n - 1 : v); };
    const int i1 = cl(i0 + 1, nx), j1 = cl(j0 + 1, ny), k1 = cl(k0 + 1, nz);
    i0 = cl(i0, nx), j0 = cl(j0, ny), k0 = cl(k0, nz);
    auto v = [&](int i, int j, int k) {
        return static_cast<double>(data[(static_cast<uint64_t>(k) * ny + j) * nx + i]);
    };
    const double c00 = v(i0, j0, k0) * (1 - tx) + v(i1, j0, k0) * tx;
    const double c10 = v(i0, j1, k0) * (1 - tx) + v(i1, j1, k0) * tx;
    const double c01 = v(i0, j0, k1) * (1 - tx) + v(i1, j0, k1) * tx;
    const double c11 = v(i0, j1, k1) * (1 - tx) + v(i1, j1, k1) * tx;
    const double c0 = c00 * (1 - ty) + c10 * ty, c1 = c01 * (1 - ty) + c11 * ty;
    return c0 * (1 - tz) + c1 * tz;
}

// Exact replay of aggregate_leaf's voxel loop (builder.cpp:37-79): AABB
// centre range (volume.cpp:150-159), increasing index order k, j, i, sequential
// double sums; ownership from the owner map.
struct Exact {
    double sum, tsum, lsum, mn, mx;
    uint64_t cnt;
};
__device__ Exact exact_scan(const VolView& V, const uint32_t* owner, const tv_tet& tt, const uint4* verts,
                            uint32_t leaf) {
    d3 c[4];
    for (int i = 0; i < 4; ++i) c[i] = corner(verts, tt.verts[i]);
    d3 lo = c[0], hi = c[0];
    for (int i = 1; i < 4; ++i) {
        lo = mk(dmin(lo.x, c[i].x), dmin(lo.y, c[i].y), dmin(lo.z, c[i].z));
        hi = mk(dmax(hi.x, c[i].x), dmax(hi.y, c[i].y), dmax(hi.z, c[i].z));
    }
    const int dims[3] = {V.nx, V.ny, V.nz};
    const double l3[3] = {lo.x, lo.y, lo.z}, h3[3] = {hi.x, hi.y, hi.z};
    int rlo[3], rhi[3];
    for (int a = 0; a < 3; ++a) {
        rlo[a] = max(0, static_cast<int>(ceil(l3[a] * dims[a] - 0.5 - 1e-12)));
        rhi[a] = min(dims[a] - 1, static_cast<int>(floor(h3[a] * dims[a] - 0.5 + 1e-12)));
    }
    Exact e{0.0, 0.0, 0.0, __longlong_as_double(0x7ff0000000000000ll), -__longlong_as_double(0x7ff0000000000000ll),
            0};
    for (int k = rlo[2]; k <= rhi[2]; ++k)
        for (int j = rlo[1]; j <= rhi[1]; ++j)
            for (int i = rlo[0]; i <= rhi[0]; ++i) {
                const uint64_t idx = (static_cast<uint64_t>(k) * V.ny + j) * V.nx + i;
                if (owner_at(V, owner, i, j, k, idx) != leaf) continue;
                const double v = V.dens[idx];
                e.mn = dmin(e.mn, v);
                e.mx = dmax(e.mx, v);
                e.sum += v;
                if (V.temp) e.tsum += V.temp[idx];
                if (V.alb) e.lsum += V.alb[idx];
                ++e.cnt;
            }
    return e;
}

__device__ __forceinline__ double err_bound(double n, double asum) {
    // |sequential - any-order sum| <= 2 (n-1) u sum|x| (+ second order); padded
    return (2.0 * n + 4.0) * 0x1.0p-53 * asum * (1.0 + 0x1.0p-30);
}

__device__ __forceinline__ bool crit_var(double mx, double mn, double sum, double n, double thr) {
    const double mean = sum / n;
    const double var = mean == 0.0 ? 0.0 : (mx - mn) / mean;  // volume.cpp:196-199
    return var > thr;
}

// camera.cpp:57-68, 70-85
__device__ bool outside_frustum(const CamCrit& C, const d3* cs) {
    for (int p = 0; p < 5; ++p) {
        bool all_out = true;
        for (int i = 0; i < 4; ++i)
            if (dot(C.pn[p], cs[i]) >= C.pd[p]) {
                all_out = false;
                break;
            }
        if (all_out) return true;
    }
    return false;
}
__device__ double projected_size(const CamCrit& C, const d3* cs) {
    double longest_sq = 0.0;
    for (int e = 0; e < 6; ++e) {
        const d3 d = sub(cs[ep0(e)], cs[ep1(e)]);
        longest_sq = dmax(longest_sq, dot(d, d));
    }
    const double longest = sqrt(longest_sq);
    const d3 cen = mul(add(add(add(cs[0], cs[1]), cs[2]), cs[3]), 0.25);
    double rsq = 0.0;
    for (int i = 0; i < 4; ++i) {
        const d3 d = sub(cs[i], cen);
        rsq = dmax(rsq, dot(d, d));
    }
    const d3 tc = sub(cen, C.pos);
    if (dot(tc, tc) <= rsq) return __longlong_as_double(0x7ff0000000000000ll);
    const double dist = dmax(sqrt(dot(tc, tc)), 1e-4);
    return longest / (2.0 * dist * C.tan_half) * C.h;
}

struct EvalParams {
    double thr;
    int max_level;
    int use_camera;
    double pixel_thr;
    CamCrit cam;
};

// builder.cpp:134-144 for every fresh leaf
__global__ void eval_kernel(const uint32_t* list, uint32_t n, VolView V, const uint32_t* owner, const tv_tet* tets,
                            const uint4* verts, const Stats* st, EvalParams E, uint8_t* flags,
                            unsigned long long* counters /* [0] replays [1] voxel visits */) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    // voxel-visit count: one atomic per warp (a per-thread atomic on one
    // counter serialises millions of leaves in L2)
    {
        unsigned long long c = i < n ? st[list[i]].cnt : 0ull;
#pragma unroll
        for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if ((threadIdx.x & 31) == 0 && c) atomicAdd(counters + 1, c);
    }
    if (i >= n) return;
    const uint32_t t = list[i];
    const tv_tet tt = tets[t];
    const Stats s = st[t];
    flags[t] &= static_cast<uint8_t>(~F_EVAL);
    if (s.cnt == 0) return;  // trilinear fallback: min == max == mean -> variation 0
    const double nn = static_cast<double>(s.cnt);
    const double mn = unord_f(s.mn), mx = unord_f(s.mx);
    bool split;
    const double B = err_bound(nn, s.asum);
    const double lo = __dsub_rd(s.sum, B), hi = __dadd_ru(s.sum, B);
    if (B == 0.0) {
        split = crit_var(mx, mn, s.sum, nn, E.thr);
    } else if (((lo > 0.0 && hi > 0.0) || (lo < 0.0 && hi < 0.0)) &&
               crit_var(mx, mn, lo, nn, E.thr) == crit_var(mx, mn, hi, nn, E.thr)) {
        split = crit_var(mx, mn, lo, nn, E.thr);
    } else {  // ambiguous under the bound: replay the reference's sequential sum
        atomicAdd(counters, 1ull);
        const Exact e = exact_scan(V, owner, tt, verts, t);
        split = crit_var(e.mx, e.mn, e.sum, static_cast<double>(e.cnt), E.thr);
    }
    if (!split) return;
    if (tt.level >= E.max_level) return;
    if (E.use_camera) {
        d3 cs[4];
        for (int k = 0; k < 4; ++k) cs[k] = corner(verts, tt.verts[k]);
        if (outside_frustum(E.cam, cs)) return;
        if (!(projected_size(E.cam, cs) > E.pixel_thr)) return;
    }
    flags[t] |= F_MARK;
}

// midpoint of each marked leaf's refinement edge: existing vertex id, or a
// "missing" record for sorted dedup
// Missing midpoints of a closure pass get new vertex ids without a sort. Every
// marked leaf whose refinement-edge midpoint is not a vertex claims the
// midpoint in a pending table (slot = coordinate fingerprint << 32 | marked
// index; the smallest marked index wins through atomicMin), the winners are
// counted by a scan in marked-list order, and the midpoint gets id n_v + its
// winner's rank. The marked list is in ascending tet id order, so the ids are
// deterministic; like every GPU id they are an allocation artefact (F3).
constexpr uint32_t kMidMissing = 0xfffffffeu;

__global__ void midpoint_kernel(const uint32_t* marked, uint32_t n, const tv_tet* tets, const uint4* verts,
                                const HSlot* table, uint64_t mask, uint32_t* mid_vid, uint64_t* khi, uint32_t* klo,
                                HSlot* pend, uint64_t pmask, int* err) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const tv_tet tt = tets[marked[i]];
    int s0, s1;
    refinement_slots(tt, verts, s0, s1);
    const uint4 a = verts[tt.verts[s0]], b = verts[tt.verts[s1]];
    const uint64_t sx = static_cast<uint64_t>(a.x) + b.x, sy = static_cast<uint64_t>(a.y) + b.y,
                   sz = static_cast<uint64_t>(a.z) + b.z;
    if ((sx | sy | sz) & 1u) {  // tet_grid.cpp:353
        atomicOr(err, E_MIDPOINT);
        mid_vid[i] = kNone;
        return;
    }
    const uint32_t mx = static_cast<uint32_t>(sx / 2), my = static_cast<uint32_t>(sy / 2),
                   mz = static_cast<uint32_t>(sz / 2);
    const uint32_t v = hash_find(table, mask, verts, mx, my, mz);
    if (v != kNone) {
        mid_vid[i] = v;
        return;
    }
    mid_vid[i] = kMidMissing;
    const uint64_t kh = static_cast<uint64_t>(mx) << 25 | my;
    khi[i] = kh;
    klo[i] = mz;
    __threadfence();  // the key is visible before the claim that names it
    const uint64_t h = coord_hash(mx, my, mz);
    const uint32_t fp = static_cast<uint32_t>(h >> 32);
    const HSlot me = hslot(fp, i);
    for (uint64_t s = h & pmask, k = 0;; s = (s + 1) & pmask) {
        if (k++ > pmask) {  // full table: cannot happen at load <= 1/2
            atomicOr(err, E_MIDPOINT);
            return;
        }
        const HSlot e = atomicCAS(pend + s, kEmptySlot, me);
        if (e == kEmptySlot) return;  // first claim
        if (static_cast<uint32_t>(e >> 32) == fp) {
            const uint32_t j = static_cast<uint32_t>(e);
            if (__ldcg(khi + j) == kh && __ldcg(klo + j) == mz) {
                atomicMin(pend + s, me);  // same midpoint: the smaller marked index wins
                return;
            }
        }
    }
}

// each missing midpoint's winner and slot; flag = 1 for winners
__global__ void midpoint_win_kernel(const uint32_t* mid_vid, uint32_t n, const uint64_t* khi, const uint32_t* klo,
                                    const HSlot* pend, uint64_t pmask, uint32_t* win, uint32_t* slot,
                                    uint32_t* flag) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (mid_vid[i] != kMidMissing) {
        flag[i] = 0;
        return;
    }
    const uint64_t kh = khi[i];
    const uint32_t kz = klo[i];
    const uint64_t h = coord_hash(static_cast<uint32_t>(kh >> 25), static_cast<uint32_t>(kh & 0x1ffffffull), kz);
    const uint32_t fp = static_cast<uint32_t>(h >> 32);
    for (uint64_t s = h & pmask, k = 0;; s = (s + 1) & pmask) {
        if (k++ > pmask) {  // not found (an error was flagged in the claim)
            win[i] = kNone;
            flag[i] = 0;
            return;
        }
        const HSlot e = pend[s];
        if (static_cast<uint32_t>(e >> 32) == fp) {
            const uint32_t j = static_cast<uint32_t>(e);
            if (khi[j] == kh && klo[j] == kz) {
                win[i] = j;
                slot[i] = static_cast<uint32_t>(s);
                flag[i] = j == i ? 1u : 0u;
                return;
            }
        }
    }
}

// scan = inclusive count of winners in marked order: midpoint id n_v + scan[winner] - 1;
// winners write the vertex, insert it and free their pending slot
__global__ void midpoint_assign_kernel(uint32_t* mid_vid, uint32_t n, const uint64_t* khi, const uint32_t* klo,
                                       const uint32_t* win, const uint32_t* slot, const uint32_t* scan, uint32_t n_v,
                                       uint4* verts, HSlot* table, uint64_t mask, HSlot* pend) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || mid_vid[i] != kMidMissing) return;
    const uint32_t w = win[i];
    if (w == kNone) {  // failed claim (flagged)
        mid_vid[i] = kNone;
        return;
    }
    const uint32_t vid = n_v + scan[w] - 1;
    mid_vid[i] = vid;
    if (w == i) {
        const uint32_t x = static_cast<uint32_t>(khi[i] >> 25), y = static_cast<uint32_t>(khi[i] & 0x1ffffffull),
                       z = klo[i];
        verts[vid] = make_uint4(x, y, z, 0);
        hash_insert(table, mask, x, y, z, vid);
        pend[slot[i]] = kEmptySlot;
    }
}

// tet_grid.cpp:339-382 for all marked leaves at once; children get ids
// n_t + 2i, n_t + 2i + 1 in marked-list (ascending id) order.
__global__ void bisect_kernel(const uint32_t* marked, uint32_t n, uint32_t n_t, tv_tet* tets, uint4* tv4,
                              const uint4* verts, const uint32_t* mid_vid, NodeRec* split, uint8_t* flags,
                              uint32_t* vtouch, int max_level, int* err, BrickMark bm) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t t = marked[i];
    const tv_tet parent = tets[t];
    mark_bricks(bm, verts, parent);
    if (parent.level >= max_level) atomicOr(err, E_LEVEL);  // MaxLevelExceeded (tet_grid.cpp:342)
    int s0, s1;
    refinement_slots(parent, verts, s0, s1);
    uint32_t vm = mid_vid[i];
    if (vm == kNone) vm = parent.verts[s0];  // midpoint error (already flagged): stay in bounds
    const uint32_t ida = n_t + 2 * i, idb = ida + 1;
    tv_tet a = parent, b = parent;
    a.verts[s1] = vm;
    b.verts[s0] = vm;
    tv_tet* cs[2] = {&a, &b};
    for (int k = 0; k < 2; ++k) {
        tv_tet* c = cs[k];
        c->parent = t;
        c->children[0] = c->children[1] = kNone;
        c->neighbors[0] = c->neighbors[1] = c->neighbors[2] = c->neighbors[3] = kNone;
        c->level = static_cast<uint8_t>(parent.level + 1);
        c->density = c->temperature = c->albedo = 0.0f;
        c->mask = 0;
        if (!compute_normals(*c, verts)) atomicOr(err, E_NORMAL);
    }
    tets[ida] = a;
    tets[idb] = b;
    tv4[ida] = make_uint4(a.verts[0], a.verts[1], a.verts[2], a.verts[3]);
    tv4[idb] = make_uint4(b.verts[0], b.verts[1], b.verts[2], b.verts[3]);
    tets[t].children[0] = ida;
    tets[t].children[1] = idb;
    tets[t].neighbors[0] = tets[t].neighbors[1] = tets[t].neighbors[2] = tets[t].neighbors[3] = kNone;
    flags[ida] = F_LEAF | F_NEW;
    flags[idb] = F_LEAF | F_NEW;
    flags[t] = 0;
    // touched vertices as a bitmask (1 bit per vertex: the hanging test's
    // lookups stay in L1 / L2)
    atomicOr(vtouch + (parent.verts[s0] >> 5), 1u << (parent.verts[s0] & 31));
    atomicOr(vtouch + (parent.verts[s1] >> 5), 1u << (parent.verts[s1] & 31));
    // split plane for the owner-map descent (tet_grid.cpp:453-470)
    const d3 pm = vpos(verts[vm]);
    int oa = -1, ob = -1;
    for (int s = 0; s < 4; ++s)
        if (s != s0 && s != s1) {
            if (oa < 0) oa = s;
            else ob = s;
        }
    const d3 pa = vpos(verts[parent.verts[oa]]), pb = vpos(verts[parent.verts[ob]]);
    const d3 nn = cross(sub(pa, pm), sub(pb, pm));
    const double sref = dot(nn, sub(vpos(verts[parent.verts[s0]]), pm));
    NodeRec r;
    r.n[0] = nn.x, r.n[1] = nn.y, r.n[2] = nn.z;
    r.pm[0] = pm.x, r.pm[1] = pm.y, r.pm[2] = pm.z;
    r.child[0] = ida;
    r.child[1] = idb;
    r.sref_pos = sref > 0.0 ? 1u : 0u;
    r.pad = 0;
    split[t] = r;
}

// Mark every leaf with a hanging edge (an edge whose integer midpoint is a
// vertex), over all tet ids. Only two kinds of leaf can have one: the children
// made by the last bisect pass (ids >= first_new) and older leaves with at
// least two vertices touched by that pass (a new midpoint lies on an edge of the
// bisected tet, whose two endpoints were touched).
// t0 > 0 (the probe path below): only the ids from t0 up, the new children.
__device__ __forceinline__ bool has_hanging_edge(const uint4* __restrict__ verts, const HSlot* __restrict__ table,
                                                 uint64_t mask, uint4 tv) {
    const uint4 q[4] = {verts[tv.x], verts[tv.y], verts[tv.z], verts[tv.w]};
    for (int e = 0; e < 6; ++e) {
        const uint4 a = q[ep0(e)], b = q[ep1(e)];
        const uint64_t sx = static_cast<uint64_t>(a.x) + b.x, sy = static_cast<uint64_t>(a.y) + b.y,
                       sz = static_cast<uint64_t>(a.z) + b.z;
        if ((sx | sy | sz) & 1u) continue;
        if (hash_find(table, mask, verts, static_cast<uint32_t>(sx / 2), static_cast<uint32_t>(sy / 2),
                      static_cast<uint32_t>(sz / 2)) != kNone)
            return true;
    }
    return false;
}

__global__ void hanging_kernel(uint32_t t0, uint32_t n_t, uint32_t first_new, const uint4* __restrict__ tv4,
                               const uint4* __restrict__ verts, const HSlot* __restrict__ table, uint64_t mask,
                               const uint32_t* __restrict__ vtouch, uint8_t* flags) {
    const uint32_t t = t0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_t) return;
    const uint8_t f = flags[t];
    if (!(f & F_LEAF)) return;
    const uint4 tv = tv4[t];
    if (t < first_new) {
        auto bit = [&](uint32_t v) { return (__ldg(vtouch + (v >> 5)) >> (v & 31)) & 1u; };
        if (bit(tv.x) + bit(tv.y) + bit(tv.z) + bit(tv.w) < 2) return;
    }
    if (has_hanging_edge(verts, table, mask, tv)) flags[t] = f | F_MARK;
}

// The hanging test of the old leaves for a pass with few bisections, without
// scanning every tet id. An old leaf (id < first_new) gets a hanging edge in
// this pass only from a midpoint created by it (earlier midpoints already
// marked every leaf around their edge, and those were bisected), and only if
// it contains that midpoint's edge (a, b): it lies in the ring of leaves around
// the edge. Every ring leaf holds a wedge around the edge with a dihedral angle
// of at least 45 degrees (LEB tets of the 24 cube roots come in three
// similarity classes), and, near the midpoint m, everything within a fraction
// of its edge lengths (shape-regular). So 32 points m + eps (cos th u + sin th
// v), th = (k + 1/2) 2 pi / 32, u, v perpendicular to b - a and eps = |b - a|
// / 64, put at least three points strictly inside every ring leaf, and the
// tree descent of the build (root_of + descend: the reference's locate_point,
// tet_grid.cpp:428-472) finds it. One thread per (bisected tet with a new
// midpoint, direction; `creator` = midpoint_win_kernel's winner flags). The
// found old leaves get the same exact test as in
// hanging_kernel; TV_HANG_CHECK=1 compares the marks with the full scan.
__global__ void hanging_probe_kernel(const uint32_t* marked, uint32_t n, const uint32_t* mid_vid,
                                     const uint32_t* creator, uint32_t first_new, const tv_tet* tets, const uint4* __restrict__ tv4,
                                     const uint4* __restrict__ verts, const HSlot* __restrict__ table,
                                     uint64_t mask, RootScan R, const NodeRec* split, uint8_t* flags) {
    const uint64_t g = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    const uint32_t i = static_cast<uint32_t>(g >> 5), k = static_cast<uint32_t>(g & 31);
    if (i >= n) return;
    // only the bisection that created a new midpoint probes around it (the
    // other ring members bisected in this pass share the edge)
    if (!creator[i]) return;
    const uint32_t vm = mid_vid[i];
    if (vm == kNone) return;
    const tv_tet& parent = tets[marked[i]];
    int s0, s1;
    refinement_slots(parent, verts, s0, s1);
    const d3 a = vpos(verts[parent.verts[s0]]), b = vpos(verts[parent.verts[s1]]);
    const d3 m = vpos(verts[vm]);
    const d3 e = sub(b, a);
    const double len = sqrt(dot(e, e));
    const d3 eh = mk(e.x / len, e.y / len, e.z / len);
    // u: eh x (the axis least aligned with eh), v = eh x u
    const double ax = fabs(eh.x), ay = fabs(eh.y), az = fabs(eh.z);
    const d3 axis = (ax <= ay && ax <= az) ? mk(1, 0, 0) : (ay <= az ? mk(0, 1, 0) : mk(0, 0, 1));
    d3 u = cross(eh, axis);
    const double ul = sqrt(dot(u, u));
    u = mk(u.x / ul, u.y / ul, u.z / ul);
    const d3 v = cross(eh, u);
    const double th = (static_cast<double>(k) + 0.5) * (6.283185307179586 / 32.0);
    double sn, cs;
    sincos(th, &sn, &cs);
    const double eps = len * (1.0 / 64.0);
    const d3 p = add(m, mk(eps * (cs * u.x + sn * v.x), eps * (cs * u.y + sn * v.y), eps * (cs * u.z + sn * v.z)));
    if (!(p.x > 1e-9 && p.y > 1e-9 && p.z > 1e-9 && p.x < 1.0 - 1e-9 && p.y < 1.0 - 1e-9 && p.z < 1.0 - 1e-9))
        return;  // outside the cube: no leaf there (the ring is cut by the boundary)
    uint32_t o = root_of(R, verts, p);
    if (o == kNone) return;
    if (!(flags[o] & F_LEAF)) o = descend(split, flags, o, p);
    if (o >= first_new) return;  // a new child: hanging_kernel tests every one
    const uint8_t f = flags[o];
    if (f & F_MARK) return;
    if (has_hanging_edge(verts, table, mask, tv4[o])) flags[o] = f | F_MARK;  // racing writers store the same byte
}

// The ids whose flag has `bit` set, in ascending order: two passes over the
// flag bytes, 16 per thread (one 16-B load), 4096 ids per block. Pass 1 counts
// per block, an exclusive scan gives each block its output offset, pass 2
// writes the ids (a block-wide scan of the per-thread counts keeps the order).
// A predicate select over a counting iterator read the flags one byte per
// thread.
constexpr int kSelThreads = 256, kSelPer = 16, kSelChunk = kSelThreads * kSelPer;

__device__ __forceinline__ uint32_t flag_bits16(const uint8_t* flags, uint32_t n, uint32_t i0, uint8_t bit) {
    uint32_t m = 0;
    if (i0 + kSelPer <= n) {
        const uint4 q = *reinterpret_cast<const uint4*>(flags + i0);
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
        const uint32_t b4 = bit * 0x01010101u;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t hit = w[k] & b4;  // per byte: bit or 0
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if ((hit >> (8 * j)) & 0xffu) m |= 1u << (4 * k + j);
        }
    } else {
        for (uint32_t j = 0; j < kSelPer && i0 + j < n; ++j)
            if (flags[i0 + j] & bit) m |= 1u << j;
    }
    return m;
}

__global__ void __launch_bounds__(kSelThreads) flag_count_kernel(const uint8_t* flags, uint32_t n, uint8_t bit,
                                                                 uint32_t* cnt) {
    using BR = cub::BlockReduce<uint32_t, kSelThreads>;
    __shared__ typename BR::TempStorage tmp;
    const uint32_t i0 = blockIdx.x * kSelChunk + threadIdx.x * kSelPer;
    const uint32_t c = i0 < n ? __popc(flag_bits16(flags, n, i0, bit)) : 0u;
    const uint32_t total = BR(tmp).Sum(c);
    if (threadIdx.x == 0) cnt[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kSelThreads) flag_compact_kernel(const uint8_t* flags, uint32_t n, uint8_t bit,
                                                                   const uint32_t* offs, uint32_t n_blocks,
                                                                   const uint32_t* cnt, uint32_t* out,
                                                                   uint32_t* n_out) {
    using BS = cub::BlockScan<uint32_t, kSelThreads>;
    __shared__ typename BS::TempStorage tmp;
    const uint32_t i0 = blockIdx.x * kSelChunk + threadIdx.x * kSelPer;
    uint32_t m = i0 < n ? flag_bits16(flags, n, i0, bit) : 0u;
    uint32_t at = 0;
    BS(tmp).ExclusiveSum(static_cast<uint32_t>(__popc(m)), at);
    at += offs[blockIdx.x];
    for (; m; m &= m - 1) out[at++] = i0 + __ffs(m) - 1;
    if (blockIdx.x == n_blocks - 1 && threadIdx.x == 0) *n_out = offs[n_blocks - 1] + cnt[n_blocks - 1];
}

// tet ids whose flag has `bit` set, for cub::DeviceSelect::If over ids
struct FlagBit {
    const uint8_t* flags;
    uint8_t bit;
    __device__ __forceinline__ bool operator()(uint32_t t) const { return flags[t] & bit; }
};

// the end-of-pass counters the host reads in one copy: [0] vertices added by
// the pass, [1] leaves marked for the next pass, [2] error bits
__global__ void pass_state_kernel(const uint32_t* scan, uint32_t n_miss, const uint32_t* n_marked, const int* err,
                                  uint32_t* out) {
    out[0] = n_miss ? scan[n_miss - 1] : 0u;  // new vertices: winners among the pass's marked leaves
    out[1] = *n_marked;
    out[2] = static_cast<uint32_t>(*err);
}

__global__ void list_flag_kernel(const uint32_t* list, uint32_t n, const uint8_t* flags, uint8_t bit, uint8_t* out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = (flags[list[i]] & bit) ? 1 : 0;
}
__global__ void clear_flag_kernel(const uint32_t* list, uint32_t n, uint8_t* flags, uint8_t bit) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) flags[list[i]] &= static_cast<uint8_t>(~bit);
}
struct PayloadParams {
    double scale;
    int has_t, has_a;
};

// assign_payloads (builder.cpp:164-182): certified against the parallel sums,
// replayed sequentially when the float rounding is ambiguous.
__global__ void payload_kernel(const uint32_t* list, uint32_t n, VolView V, const uint32_t* owner, tv_tet* tets,
                               const uint4* verts, const Stats* st, PayloadParams P, unsigned long long* replays,
                               int* max_depth) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t t = list[i];
    tv_tet tt = tets[t];
    const Stats s = st[t];
    {  // one atomic per warp
        const int lv = __reduce_max_sync(__activemask(), static_cast<int>(tt.level));
        if ((threadIdx.x & 31) == static_cast<unsigned>(__ffs(__activemask()) - 1)) atomicMax(max_depth, lv);
    }
    float dens, temp = 0.f, alb = 0.f;
    if (s.cnt == 0) {
        d3 c[4];
        for (int k = 0; k < 4; ++k) c[k] = corner(verts, tt.verts[k]);
        const d3 cen = mul(add(add(add(c[0], c[1]), c[2]), c[3]), 0.25);
        const double m = trilinear(V.dens, V.nx, V.ny, V.nz, cen);
        dens = static_cast<float>(P.scale * m);
        if (P.has_t) temp = static_cast<float>(trilinear(V.temp, V.nx, V.ny, V.nz, cen));
        if (P.has_a) alb = static_cast<float>(dclamp(trilinear(V.alb, V.nx, V.ny, V.nz, cen), 0.0, 1.0));
    } else {
        const double nn = static_cast<double>(s.cnt);
        bool ok = true;
        auto fdens = [&](double x) { return static_cast<float>(P.scale * (x / nn)); };
        auto ftemp = [&](double x) { return static_cast<float>(x / nn); };
        auto falb = [&](double x) { return static_cast<float>(dclamp(x / nn, 0.0, 1.0)); };
        const double B = err_bound(nn, s.asum);
        dens = fdens(s.sum);
        if (B > 0.0 && fdens(__dsub_rd(s.sum, B)) != fdens(__dadd_ru(s.sum, B))) ok = false;
        if (P.has_t) {
            const double Bt = err_bound(nn, s.tasum);
            temp = ftemp(s.tsum);
            if (Bt > 0.0 && ftemp(__dsub_rd(s.tsum, Bt)) != ftemp(__dadd_ru(s.tsum, Bt))) ok = false;
        }
        if (P.has_a) {
            const double Ba = err_bound(nn, s.lasum);
            alb = falb(s.lsum);
            if (Ba > 0.0 && falb(__dsub_rd(s.lsum, Ba)) != falb(__dadd_ru(s.lsum, Ba))) ok = false;
        }
        if (!ok) {
            atomicAdd(replays, 1ull);
            const Exact e = exact_scan(V, owner, tt, verts, t);
            const double en = static_cast<double>(e.cnt);
            dens = static_cast<float>(P.scale * (e.sum / en));
            if (P.has_t) temp = static_cast<float>(e.tsum / en);
            if (P.has_a) alb = static_cast<float>(dclamp(e.lsum / en, 0.0, 1.0));
        }
    }
    tt.density = dens;
    tt.mask = 1;
    if (P.has_t) tt.temperature = temp, tt.mask |= 2;
    if (P.has_a) tt.albedo = alb, tt.mask |= 4;
    tets[t].density = tt.density;
    tets[t].temperature = tt.temperature;
    tets[t].albedo = tt.albedo;
    tets[t].mask = tt.mask;
}

// face records for neighbour pairing: key = sorted vertex triple
__global__ void face_keys_kernel(const uint32_t* leaves, uint32_t n, const tv_tet* tets, uint64_t* khi, uint32_t* klo,
                                 uint32_t* rec, int vb) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t t = leaves[i];
    const tv_tet tt = tets[t];
    for (int slot = 0; slot < 4; ++slot) {
        uint32_t k[3];
        int m = 0;
        for (int s = 0; s < 4; ++s)
            if (s != slot) k[m++] = tt.verts[s];
        if (k[0] > k[1]) { uint32_t x = k[0]; k[0] = k[1]; k[1] = x; }
        if (k[1] > k[2]) { uint32_t x = k[1]; k[1] = k[2]; k[2] = x; }
        if (k[0] > k[1]) { uint32_t x = k[0]; k[0] = k[1]; k[1] = x; }
        const uint64_t o = 4ull * i + slot;
        khi[o] = static_cast<uint64_t>(k[0]) << vb | k[1];  // vertex ids < 2^vb: the sorts see 2 vb + vb bits
        klo[o] = k[2];
        rec[o] = static_cast<uint32_t>(o);
    }
}

__global__ void face_pair_kernel(const uint64_t* khi, const uint32_t* klo, const uint32_t* rec, uint64_t n,
                                 const uint32_t* leaves, tv_tet* tets, int* err) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const bool eq_prev = i > 0 && khi[i] == khi[i - 1] && klo[i] == klo[i - 1];
    const bool eq_next = i + 1 < n && khi[i] == khi[i + 1] && klo[i] == klo[i + 1];
    const uint32_t r = rec[i];
    const uint32_t t = leaves[r >> 2], slot = r & 3;
    if (eq_prev && eq_next) {
        atomicOr(err, E_FACE);  // face shared by more than two leaves
        return;
    }
    uint32_t other = kNone;
    if (eq_prev) other = leaves[rec[i - 1] >> 2];
    if (eq_next) other = leaves[rec[i + 1] >> 2];
    tets[t].neighbors[slot] = other;
}


// face key of face record rec[p] (4 * leaf-list index + slot)
__global__ void gather_face_hi_kernel(const uint32_t* rec, uint64_t n, const uint32_t* leaves, const tv_tet* tets,
                                      uint64_t* khi, uint32_t* klo, int vb) {
    const uint64_t p = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (p >= n) return;
    const uint32_t r = rec[p];
    const tv_tet& tt = tets[leaves[r >> 2]];
    const int slot = r & 3;
    uint32_t k[3];
    int m = 0;
    for (int s = 0; s < 4; ++s)
        if (s != slot) k[m++] = tt.verts[s];
    if (k[0] > k[1]) { uint32_t x = k[0]; k[0] = k[1]; k[1] = x; }
    if (k[1] > k[2]) { uint32_t x = k[1]; k[1] = k[2]; k[2] = x; }
    if (k[0] > k[1]) { uint32_t x = k[0]; k[0] = k[1]; k[1] = x; }
    khi[p] = static_cast<uint64_t>(k[0]) << vb | k[1];
    klo[p] = k[2];
}

// ------------------------------------------------------------ host side
inline unsigned nblk(uint64_t n, unsigned t = 256) { return static_cast<unsigned>(std::max<uint64_t>((n + t - 1) / t, 1)); }

// Build scratch: growable device arrays. Each buffer reserves a virtual
// address range once and maps physical memory onto its end as it grows
// (cuMemCreate / cuMemMap, reached through the runtime's driver entry points so
// the library does not link libcuda): growth copies nothing and never holds
// the old and new copies at once, and mapping costs ~1 ms per GB where a
// stream-ordered pool's first growth costs 65-100 ms per GB
// (tools/alloc_probe.cu on B200). Everything is unmapped when the buffer goes
// out of scope, so no build scratch outlives the build. Without the VMM entry
// points, buffers fall back to cudaMalloc + copy on growth.
struct VmmApi {
    using Create = CUresult (*)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long);
    using Release = CUresult (*)(CUmemGenericAllocationHandle);
    using Reserve = CUresult (*)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
    using AddrFree = CUresult (*)(CUdeviceptr, size_t);
    using Map = CUresult (*)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
    using Unmap = CUresult (*)(CUdeviceptr, size_t);
    using Access = CUresult (*)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
    using Gran = CUresult (*)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags);
    Create create = nullptr;
    Release release = nullptr;
    Reserve reserve = nullptr;
    AddrFree addr_free = nullptr;
    Map map = nullptr;
    Unmap unmap = nullptr;
    Access access = nullptr;
    Gran gran = nullptr;
    bool ok = false;
};

const VmmApi& vmm() {
    static VmmApi api = [] {
        VmmApi a;
        auto get = [](const char* name, void** fn) {
            cudaDriverEntryPointQueryResult q;
            return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
                   q == cudaDriverEntryPointSuccess && *fn;
        };
        a.ok = get("cuMemCreate", reinterpret_cast<void**>(&a.create)) &&
               get("cuMemRelease", reinterpret_cast<void**>(&a.release)) &&
               get("cuMemAddressReserve", reinterpret_cast<void**>(&a.reserve)) &&
               get("cuMemAddressFree", reinterpret_cast<void**>(&a.addr_free)) &&
               get("cuMemMap", reinterpret_cast<void**>(&a.map)) &&
               get("cuMemUnmap", reinterpret_cast<void**>(&a.unmap)) &&
               get("cuMemSetAccess", reinterpret_cast<void**>(&a.access)) &&
               get("cuMemGetAllocationGranularity", reinterpret_cast<void**>(&a.gran));
        if (std::getenv("TV_BUILD_NO_VMM")) a.ok = false;
        return a;
    }();
    return api;
}

thread_local int t_build_device = 0;

struct Buf {
    void* p = nullptr;
    size_t bytes = 0;  // usable (mapped) bytes
    CUdeviceptr va = 0;
    size_t reserved = 0;
    std::vector<CUmemGenericAllocationHandle> handles;
    std::vector<size_t> sizes;  // bytes of each handle, in mapping order
    bool mapped = false;        // VMM-backed
    Buf() = default;
    Buf(const Buf&) = delete;
    Buf& operator=(const Buf&) = delete;
    ~Buf() { reset(); }
    void reset() {
        if (!p) return;
        cudaStreamSynchronize(0);  // build kernels run on the legacy stream
        static const bool verbose = std::getenv("TV_VERBOSE") && std::atoi(std::getenv("TV_VERBOSE")) > 1;
        const auto t0 = std::chrono::steady_clock::now();
        if (mapped) {
            const VmmApi& a = vmm();
            a.unmap(va, bytes);
            for (auto h : handles) a.release(h);
            a.addr_free(va, reserved);
        } else {
            cudaFree(p);
        }
        if (verbose && bytes >= (256u << 20))
            std::fprintf(stderr, "tetvol_b200: build free %.1f MB: %.2f ms\n", bytes / 1048576.0,
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
        p = nullptr, bytes = 0, va = 0, reserved = 0, mapped = false;
        handles.clear();
        sizes.clear();
    }
    template <class T>
    T* as() {
        return static_cast<T*>(p);
    }
};

// TV_BUILD_POISON=1 (tests): fill every scratch byte the build has not written with 0x5A (new
// growth, and every cached buffer at the start of a build), so that a kernel reading memory it did
// not initialise shows up as a parity failure instead of relying on zeroed fresh pages.
bool poison() {
    static const bool p = std::getenv("TV_BUILD_POISON") && std::atoi(std::getenv("TV_BUILD_POISON"));
    return p;
}

// grow b to at least `bytes`, keeping its contents
int ensure(Buf& b, size_t bytes, bool /*keep: contents are always kept*/ = false) {
    if (b.bytes >= bytes) return TV_OK;
    static const bool verbose = std::getenv("TV_VERBOSE") && std::atoi(std::getenv("TV_VERBOSE")) > 1;
    static const bool verbose3 = std::getenv("TV_VERBOSE") && std::atoi(std::getenv("TV_VERBOSE")) > 2;
    const auto t0 = std::chrono::steady_clock::now();
    double tm[6] = {0, 0, 0, 0, 0, 0};  // TV_VERBOSE=3: meminfo+reserve, sync, remap, create, map, access
    auto lap = [&](int i, std::chrono::steady_clock::time_point& t) {
        const auto n = std::chrono::steady_clock::now();
        tm[i] += std::chrono::duration<double, std::milli>(n - t).count();
        t = n;
    };
    auto tl = t0;
    const VmmApi& a = vmm();
    // geometric growth in >= 64 MB steps: few mappings per buffer
    size_t nb = std::max(bytes, 2 * b.bytes);
    if (a.ok && (b.mapped || !b.p)) {
        CUmemAllocationProp prop = {};
        prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
        prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        prop.location.id = t_build_device;
        size_t g = 0;
        if (a.gran(&g, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS || !g) g = 2u << 20;
        // TV_BUILD_VMM_TIGHT=1 (tests): granule-sized steps in exactly-sized ranges, so that every
        // growth maps a new handle and moves the buffer to a new range
        static const bool tight = std::getenv("TV_BUILD_VMM_TIGHT") && std::atoi(std::getenv("TV_BUILD_VMM_TIGHT"));
        if (!tight) nb = std::max(nb, static_cast<size_t>(64u << 20));
        nb = (nb + g - 1) / g * g;
        if (nb > b.reserved) {
            // Reserve a virtual range of 8x the request (>= 1 GB, <= device memory). Not the whole
            // device per buffer: mapping into and freeing ~25 ranges of 178 GB each cost 0.1-3.4 s per
            // build on B200 (tools/vmm_probe2.cu), against < 3 ms for ranges of a few GB. A buffer
            // that outgrows its range moves: the same physical handles are mapped at a larger
            // range (no copy) and the old range is released.
            size_t total = 0, free_b = 0;
            cudaMemGetInfo(&free_b, &total);
            size_t want = std::max(nb * 8, static_cast<size_t>(1) << 30);
            want = tight ? nb : std::max(std::min(want, total), nb);
            want = (want + g - 1) / g * g;
            CUdeviceptr nva = 0;
            if (a.reserve(&nva, want, g, 0, 0) != CUDA_SUCCESS)
                return set_error(TV_ERR_OOM, "build alloc: cannot reserve a virtual range");
            lap(0, tl);
            if (b.bytes) {
                cudaStreamSynchronize(0);  // kernels in flight may still use the old addresses
                lap(1, tl);
                CUmemAccessDesc d = {};
                d.location = prop.location;
                d.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
                size_t off = 0;
                bool ok = true;
                for (size_t i = 0; i < b.handles.size() && ok; ++i) {
                    ok = a.map(nva + off, b.sizes[i], 0, b.handles[i], 0) == CUDA_SUCCESS;
                    off += b.sizes[i];
                }
                if (ok) ok = a.access(nva, b.bytes, &d, 1) == CUDA_SUCCESS;
                if (!ok) {
                    if (off) a.unmap(nva, off);
                    a.addr_free(nva, want);
                    return set_error(TV_ERR_OOM, "build alloc: remap failed");
                }
                a.unmap(b.va, b.bytes);
                a.addr_free(b.va, b.reserved);
                lap(2, tl);
            }
            b.va = nva;
            b.reserved = want;
            b.p = reinterpret_cast<void*>(b.va);
            b.mapped = true;
        }
        const size_t add = nb - b.bytes;
        CUmemGenericAllocationHandle h;
        lap(5, tl);
        if (a.create(&h, add, &prop, 0) != CUDA_SUCCESS)
            return set_error(TV_ERR_OOM, "build alloc: out of device memory");
        lap(3, tl);
        if (a.map(b.va + b.bytes, add, 0, h, 0) != CUDA_SUCCESS) {
            a.release(h);
            return set_error(TV_ERR_OOM, "build alloc: map failed");
        }
        lap(4, tl);
        CUmemAccessDesc d = {};
        d.location = prop.location;
        d.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        if (a.access(b.va + b.bytes, add, &d, 1) != CUDA_SUCCESS) {
            a.unmap(b.va + b.bytes, add);
            a.release(h);
            return set_error(TV_ERR_OOM, "build alloc: access failed");
        }
        lap(5, tl);
        if (poison()) cudaMemset(reinterpret_cast<char*>(b.va) + b.bytes, 0x5A, add);
        b.handles.push_back(h);
        b.sizes.push_back(add);
        b.bytes = nb;
        if (verbose3)
            std::fprintf(stderr,
                         "tetvol_b200: ensure %.1f -> %.1f MB: reserve %.2f sync %.2f remap %.2f create %.2f map %.2f "
                         "access+rest %.2f ms\n",
                         (nb - add) / 1048576.0, nb / 1048576.0, tm[0], tm[1], tm[2], tm[3], tm[4], tm[5]);
    } else {
        void* p = nullptr;
        cudaError_t e = cudaMalloc(&p, nb);
        if (e != cudaSuccess) return cuda_status(e, "build alloc");
        if (b.p && b.bytes) {
            e = cudaMemcpy(p, b.p, b.bytes, cudaMemcpyDeviceToDevice);
            if (e != cudaSuccess) {
                cudaFree(p);
                return cuda_status(e, "build grow");
            }
        }
        if (poison()) cudaMemset(static_cast<char*>(p) + b.bytes, 0x5A, nb - b.bytes);
        b.reset();
        b.p = p;
        b.bytes = nb;
    }
    if (verbose && nb >= (256u << 20))
        std::fprintf(stderr, "tetvol_b200: build alloc %.1f MB (%s): %.2f ms\n", nb / 1048576.0,
                     b.mapped ? "vmm" : "cudaMalloc",
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    return TV_OK;
}

// The build's device scratch. Kept per device across builds (TV_BUILD_CACHE, default on) and
// released by tv_build_trim: the buffers of a C4 build sum to ~45 GB, and re-creating them for
// every build put 0.2-3 s of driver time (cuMemCreate / cudaMalloc of memory the previous build
// just freed) into warm builds of 0.6 s. Every build initialises what it reads (TV_BUILD_POISON).
struct BuildScratch {
    std::mutex m;
    Buf align[3];
    Buf tets, tv4, verts, split, flags, stats, table, vtouch, owner, leaves, sel, tmp, mid, miss_hi, miss_lo,
        miss_idx, miss_hi2, miss_lo2, miss_idx2, head, scan, misc, stripe, fresh, marked, khi, klo, rec, khi2, klo2,
        rec2, centres, bricks, bstat, mixed, mixedn, subs, sstat, bmark, pend, selc;
    template <class F>
    void each(F f) {
        for (auto& b : align) f(b);
        for (Buf* b : {&tets, &tv4, &verts, &split, &flags, &stats, &table, &vtouch, &owner, &leaves, &sel, &tmp,
                       &mid, &miss_hi, &miss_lo, &miss_idx, &miss_hi2, &miss_lo2, &miss_idx2, &head, &scan, &misc,
                       &stripe, &fresh, &marked, &khi, &klo, &rec, &khi2, &klo2, &rec2, &centres, &bricks, &bstat, &mixed,
                       &mixedn, &subs, &sstat, &bmark, &pend, &selc})
            f(*b);
    }
    void release() {
        each([](Buf& b) { b.reset(); });
    }
    size_t bytes() {
        size_t n = 0;
        each([&](Buf& b) { n += b.bytes; });
        return n;
    }
};

std::mutex g_scratch_mu;
std::map<int, BuildScratch*>& scratch_map() {
    static auto* m = new std::map<int, BuildScratch*>();  // never destroyed: no CUDA calls at exit
    return *m;
}

// host init_roots (tet_grid.cpp:184-233)
int host_init_roots(std::vector<uint4>& verts, std::vector<tv_tet>& tets, uint32_t roots[24]) {
    auto intern = [&](uint32_t x, uint32_t y, uint32_t z) {
        for (uint32_t i = 0; i < verts.size(); ++i)
            if (verts[i].x == x && verts[i].y == y && verts[i].z == z) return i;
        verts.push_back(make_uint4(x, y, z, 0));
        return static_cast<uint32_t>(verts.size() - 1);
    };
    const uint32_t S = 1u << 24, H = S / 2;
    const uint32_t center = intern(H, H, H);
    int ri = 0;
    for (int axis = 0; axis < 3; ++axis)
        for (int side = 0; side < 2; ++side) {
            uint32_t fc[3] = {H, H, H};
            fc[axis] = side ? S : 0;
            const uint32_t fcv = intern(fc[0], fc[1], fc[2]);
            const int u = axis == 0 ? 1 : 0, w = axis == 2 ? 1 : 2;
            const uint32_t ring[4][2] = {{0, 0}, {1, 0}, {1, 1}, {0, 1}};
            uint32_t corner_v[4];
            for (int k = 0; k < 4; ++k) {
                uint32_t c[3] = {0, 0, 0};
                c[axis] = side ? S : 0;
                c[u] = ring[k][0] * S;
                c[w] = ring[k][1] * S;
                corner_v[k] = intern(c[0], c[1], c[2]);
            }
            for (int k = 0; k < 4; ++k) {
                uint32_t p = corner_v[k], q = corner_v[(k + 1) % 4];
                if (det_fixed(verts[p], verts[fcv], verts[center], verts[q]) < 0) std::swap(p, q);
                tv_tet t;
                std::memset(&t, 0, sizeof t);
                t.verts[0] = p, t.verts[1] = fcv, t.verts[2] = center, t.verts[3] = q;
                t.children[0] = t.children[1] = t.parent = TV_NO_TET;
                for (int f = 0; f < 4; ++f) t.neighbors[f] = TV_NO_TET;
                roots[ri++] = static_cast<uint32_t>(tets.size());
                tets.push_back(t);
            }
        }
    for (auto& t : tets)
        if (!compute_normals(t, verts.data())) return set_error(TV_ERR_GRID, "root normals not canonical");
    return TV_OK;
}

int validate_build_cfg(const tv_build_config* c) {  // builder.cpp:12-17
    if (!c) return set_error(TV_ERR_ARG, "build config is null");
    if (!(c->variation_threshold >= 0.0)) return set_error(TV_ERR_CONFIG, "variationThreshold must be >= 0");
    if (c->max_level < 0 || c->max_level > 48) return set_error(TV_ERR_CONFIG, "maxLevel out of range");
    if (!(c->pixel_threshold > 0.0)) return set_error(TV_ERR_CONFIG, "pixelThreshold must be > 0");
    if (!(c->density_scale >= 0.0)) return set_error(TV_ERR_CONFIG, "densityScale must be >= 0");
    return TV_OK;
}

}  // namespace

// defined in tv_capi.cu
int host_camera(const tv_camera* c, CamView& v, d3 pn[5], double pd[5]);

namespace {
int build_grid_impl(const float* dens, const float* temp, const float* alb, int nx, int ny, int nz,
                    const tv_build_config* cfg, const tv_camera* camera, int device, tv_grid** out,
                    tv_build_stats* stats, BuildScratch& S) {
    int rc = validate_build_cfg(cfg);
    if (rc) return rc;
    if (cfg->use_camera && !camera) return set_error(TV_ERR_CONFIG, "useCamera set but no camera given");
    if (nx < 1 || ny < 1 || nz < 1) return set_error(TV_ERR_CONFIG, "volume dimensions must be positive");
    EvalParams E{};
    E.thr = cfg->variation_threshold;
    E.max_level = cfg->max_level;
    E.use_camera = cfg->use_camera;
    E.pixel_thr = cfg->pixel_threshold;
    if (camera) {
        CamView cv;
        d3 pn[5];
        double pd[5];
        if ((rc = host_camera(camera, cv, pn, pd))) return rc;
        E.cam.pos = mk(cv.pos[0], cv.pos[1], cv.pos[2]);
        E.cam.tan_half = cv.tan_half;
        E.cam.h = cv.h;
        for (int i = 0; i < 5; ++i) E.cam.pn[i] = pn[i], E.cam.pd[i] = pd[i];
    }
    const int grid_max_level = std::max(cfg->max_level, 1);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);

    const uint64_t nvox = static_cast<uint64_t>(nx) * ny * nz;
    Buf* align_b = S.align;  // misaligned channels, copied (see below)
    Buf &tets_b = S.tets, &tv4_b = S.tv4, &verts_b = S.verts, &split_b = S.split, &flags_b = S.flags,
        &stats_b = S.stats, &table_b = S.table, &vtouch_b = S.vtouch, &owner_b = S.owner, &leaves_b = S.leaves,
        &sel_b = S.sel, &tmp_b = S.tmp, &mid_b = S.mid, &miss_hi_b = S.miss_hi, &miss_lo_b = S.miss_lo,
        &miss_idx_b = S.miss_idx, &miss_hi2_b = S.miss_hi2, &miss_lo2_b = S.miss_lo2, &miss_idx2_b = S.miss_idx2,
        &head_b = S.head, &scan_b = S.scan, &misc_b = S.misc;
    size_t cap_t = 0, cap_v = 0;
    uint64_t hmask = 0;

    std::vector<uint4> hv;
    std::vector<tv_tet> ht;
    uint32_t roots[24];
    if ((rc = host_init_roots(hv, ht, roots))) return rc;
    uint32_t n_t = static_cast<uint32_t>(ht.size()), n_v = static_cast<uint32_t>(hv.size());

#define TRY(x)                 \
    do {                       \
        if ((rc = (x))) return rc; \
    } while (0)
#define CK(x, what) TRY(cuda_status((x), what))

    // the voxel sweep reads the channels as float4: copy a misaligned one
    const float* ch[3] = {dens, temp, alb};
    for (int c = 0; c < 3; ++c)
        if (ch[c] && (reinterpret_cast<uintptr_t>(ch[c]) & 15u)) {
            TRY(ensure(align_b[c], nvox * sizeof(float)));
            CK(cudaMemcpy(align_b[c].p, ch[c], nvox * sizeof(float), cudaMemcpyDeviceToDevice), "align volume");
            ch[c] = align_b[c].as<float>();
        }
    TRY(ensure(S.centres, static_cast<size_t>(nx + ny + nz) * sizeof(double)));
    double* cxyz = S.centres.as<double>();
    centres_kernel<<<nblk(nx + ny + nz, 256), 256>>>(nx, ny, nz, cxyz);
    CK(cudaGetLastError(), "voxel centres");
    // voxel bricks (TV_VOX_BRICKS=0: per-voxel ownership sweeps only)
    static const bool use_bricks = !std::getenv("TV_VOX_BRICKS") || std::atoi(std::getenv("TV_VOX_BRICKS"));
    const int gbx = (nx + kBrick - 1) / kBrick, gby = (ny + kBrick - 1) / kBrick, gbz = (nz + kBrick - 1) / kBrick;
    const uint32_t n_bricks = static_cast<uint32_t>(gbx) * gby * gbz;
    uint32_t* brick_owner = nullptr;
    if (use_bricks) {
        TRY(ensure(S.bricks, static_cast<size_t>(n_bricks) * sizeof(uint32_t)));
        TRY(ensure(S.bstat, static_cast<size_t>(n_bricks) * sizeof(BrickStat)));
        TRY(ensure(S.mixed, static_cast<size_t>(n_bricks) * sizeof(uint32_t)));
        TRY(ensure(S.mixedn, 16));
        TRY(ensure(S.subs, static_cast<size_t>(n_bricks) * 8 * sizeof(uint32_t)));
        TRY(ensure(S.sstat, static_cast<size_t>(n_bricks) * 8 * sizeof(BrickStat)));
        brick_owner = S.bricks.as<uint32_t>();
    }
    // brick marks: n_bricks bits, then one bit per super-brick (8^3 bricks) and the all-bricks word
    const int gsx = (gbx + 7) / 8, gsy = (gby + 7) / 8, gsz = (gbz + 7) / 8;
    const uint32_t bwords = n_bricks / 32 + 1, swords = static_cast<uint32_t>(gsx) * gsy * gsz / 32 + 2;
    const uint32_t mark_words = bwords + swords;
    if (use_bricks) {
        TRY(ensure(S.bmark, static_cast<size_t>(mark_words) * sizeof(uint32_t)));
        CK(cudaMemset(S.bmark.p, 0, mark_words * sizeof(uint32_t)), "brick marks");
    }
    const BrickMark bmark{use_bricks ? S.bmark.as<uint32_t>() : nullptr,
                          use_bricks ? S.bmark.as<uint32_t>() + bwords : nullptr,
                          swords, nx, ny, nz, gbx, gby, gsx, gsy};
    const VolView V{ch[0],     ch[1],    ch[2],       nx,  ny,  nz, cxyz, cxyz + nx, cxyz + nx + ny,
                    1.0 / nx, 1.0 / ny, brick_owner, gbx, gby, use_bricks ? S.subs.as<uint32_t>() : nullptr};

    auto grow_tets = [&](size_t need) -> int {
        if (need <= cap_t) return TV_OK;
        const size_t nc = std::max(need, cap_t * 2 + 1024);
        TRY(ensure(tets_b, nc * sizeof(tv_tet), true));
        TRY(ensure(tv4_b, nc * sizeof(uint4), true));
        TRY(ensure(split_b, nc * sizeof(NodeRec), true));
        TRY(ensure(flags_b, nc, true));
        TRY(ensure(stats_b, nc * sizeof(Stats), true));
        cap_t = nc;
        return TV_OK;
    };
    auto grow_verts = [&](size_t need) -> int {
        if (need <= cap_v) return TV_OK;
        const size_t nc = std::max(need, cap_v * 2 + 1024);
        TRY(ensure(verts_b, nc * sizeof(uint4), true));
        TRY(ensure(vtouch_b, (nc + 31) / 32 * 4, true));
        size_t slots = 1024;
        while (slots < 2 * nc) slots <<= 1;
        TRY(ensure(table_b, slots * sizeof(HSlot)));
        CK(cudaMemset(table_b.p, 0xff, slots * sizeof(HSlot)), "hash clear");
        hmask = slots - 1;
        hash_rebuild_kernel<<<nblk(n_v), 256>>>(table_b.as<HSlot>(), hmask, verts_b.as<uint4>(), n_v);
        CK(cudaGetLastError(), "hash rebuild");
        cap_v = nc;
        return TV_OK;
    };

    // initial capacity guess: grows geometrically as needed
    TRY(grow_tets(std::min<size_t>(std::max<size_t>(1 << 16, nvox / 4), size_t(1) << 24)));
    CK(cudaMemcpy(tets_b.p, ht.data(), ht.size() * sizeof(tv_tet), cudaMemcpyHostToDevice), "roots H2D");
    {
        std::vector<uint4> tv(ht.size());
        for (size_t i = 0; i < ht.size(); ++i)
            tv[i] = make_uint4(ht[i].verts[0], ht[i].verts[1], ht[i].verts[2], ht[i].verts[3]);
        CK(cudaMemcpy(tv4_b.p, tv.data(), tv.size() * sizeof(uint4), cudaMemcpyHostToDevice), "roots H2D");
    }
    {
        const size_t need_v = std::min<size_t>(std::max<size_t>(1 << 15, nvox / 16), size_t(1) << 22);
        TRY(ensure(verts_b, need_v * sizeof(uint4)));
        CK(cudaMemcpy(verts_b.p, hv.data(), hv.size() * sizeof(uint4), cudaMemcpyHostToDevice), "verts H2D");
        TRY(grow_verts(need_v));
    }
    CK(cudaMemset(flags_b.p, 0, cap_t), "flags");
    {
        std::vector<uint8_t> f(n_t, F_LEAF | F_NEW);
        CK(cudaMemcpy(flags_b.p, f.data(), n_t, cudaMemcpyHostToDevice), "flags H2D");
    }
    TRY(ensure(owner_b, nvox * sizeof(uint32_t)));
    TRY(ensure(misc_b, 64));
    int* d_err = misc_b.as<int>();
    uint32_t* d_cnt = reinterpret_cast<uint32_t*>(misc_b.as<char>() + 8);
    unsigned long long* d_ctr = reinterpret_cast<unsigned long long*>(misc_b.as<char>() + 16);  // replays, visits
    int* d_depth = reinterpret_cast<int*>(misc_b.as<char>() + 32);
    uint32_t* d_state = reinterpret_cast<uint32_t*>(misc_b.as<char>() + 48);  // pass_state_kernel
    CK(cudaMemset(misc_b.p, 0, 64), "misc");

    RootScan R;
    for (int r = 0; r < 24; ++r) {
        R.id[r] = roots[r];
        const tv_tet& t = ht[roots[r]];
        R.nid[r] = t.normal_ids[0] | t.normal_ids[1] << 8 | t.normal_ids[2] << 16 |
                   static_cast<uint32_t>(t.normal_ids[3]) << 24;
        for (int k = 0; k < 4; ++k) R.vid[r][k] = t.verts[k];
    }
    int n_sm = 148;
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, device);
    const unsigned vox_blocks = static_cast<unsigned>(n_sm) * (2048 / kVoxThreads);

    // the listed tets whose flag has `bit` (order kept)
    auto select_listed = [&](const uint32_t* in_list, uint32_t n_in, uint8_t bit, Buf& outb, uint32_t& n_out) -> int {
        TRY(ensure(sel_b, std::max<size_t>(n_in, 1)));
        TRY(ensure(outb, std::max<size_t>(n_in, 1) * sizeof(uint32_t)));
        list_flag_kernel<<<nblk(n_in), 256>>>(in_list, n_in, flags_b.as<uint8_t>(), bit, sel_b.as<uint8_t>());
        CK(cudaGetLastError(), "flag kernel");
        size_t tb = 0;
        CK(cub::DeviceSelect::Flagged(nullptr, tb, in_list, sel_b.as<uint8_t>(), outb.as<uint32_t>(), d_cnt,
                                      static_cast<int>(n_in)),
           "select sizing");
        TRY(ensure(tmp_b, tb));
        CK(cub::DeviceSelect::Flagged(tmp_b.p, tb, in_list, sel_b.as<uint8_t>(), outb.as<uint32_t>(), d_cnt,
                                      static_cast<int>(n_in)),
           "select");
        CK(cudaMemcpy(&n_out, d_cnt, sizeof(uint32_t), cudaMemcpyDeviceToHost), "select count");
        return TV_OK;
    };
    // all tet ids [0, n_t) whose flag has `bit`, ascending; the count lands in
    // d_cnt and is copied to n_out when n_out is given
    auto select_tets = [&](uint8_t bit, Buf& outb, uint32_t* n_out) -> int {
        TRY(ensure(outb, std::max<size_t>(n_t, 1) * sizeof(uint32_t)));
        const uint32_t nb = std::max<uint32_t>(1, static_cast<uint32_t>((static_cast<uint64_t>(n_t) + kSelChunk - 1) / kSelChunk));
        TRY(ensure(S.selc, 2ull * nb * sizeof(uint32_t)));
        uint32_t* cnt = S.selc.as<uint32_t>();
        uint32_t* offs = cnt + nb;
        flag_count_kernel<<<nb, kSelThreads>>>(flags_b.as<uint8_t>(), n_t, bit, cnt);
        size_t tb = 0;
        CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, offs, static_cast<int>(nb)), "select sizing");
        TRY(ensure(tmp_b, tb));
        CK(cub::DeviceScan::ExclusiveSum(tmp_b.p, tb, cnt, offs, static_cast<int>(nb)), "select scan");
        flag_compact_kernel<<<nb, kSelThreads>>>(flags_b.as<uint8_t>(), n_t, bit, offs, nb, cnt, outb.as<uint32_t>(),
                                                 d_cnt);
        CK(cudaGetLastError(), "select");
        if (n_out) CK(cudaMemcpy(n_out, d_cnt, sizeof(uint32_t), cudaMemcpyDeviceToHost), "select count");
        return TV_OK;
    };

    uint64_t crit = 0, bisections = 0, passes = 0, replays = 0;
    // hanging test by probes around the new midpoints when a pass bisects fewer
    // than 1 / TV_HANG_PROBE_COST of the tets (TV_HANG_PROBE=0: always the full
    // scan; TV_HANG_CHECK=1: run both and fail the build if they differ)
    static const bool hang_probe = !std::getenv("TV_HANG_PROBE") || std::atoi(std::getenv("TV_HANG_PROBE"));
    static const uint64_t hang_probe_cost =
        std::getenv("TV_HANG_PROBE_COST") ? std::max(1, std::atoi(std::getenv("TV_HANG_PROBE_COST"))) : 64;
    static const bool hang_check = std::getenv("TV_HANG_CHECK") && std::atoi(std::getenv("TV_HANG_CHECK"));
    bool hang_mismatch = false;
    uint64_t probe_passes = 0;
    bool pend_clean = false;  // the pending-midpoint table has been cleared in this build
    int rounds = 0;
    uint32_t n_fresh = 24, n_marked = 0, n_leaves = 24;
    uint32_t fresh_lo = 0;                    // the fresh leaves' ids lie in [fresh_lo, n_t)
    constexpr uint32_t kStripeOwners = 32768;  // stripe up to 32K owners (64 MB of stripes)
    Buf &stripe_b = S.stripe, &fresh_b = S.fresh, &marked_b = S.marked;
    TRY(ensure(fresh_b, 24 * sizeof(uint32_t)));
    CK(cudaMemcpy(fresh_b.p, roots, sizeof(roots), cudaMemcpyHostToDevice), "fresh");
    int herr = 0;
    const bool verbose = std::getenv("TV_VERBOSE") && std::atoi(std::getenv("TV_VERBOSE")) > 1;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto since = [&](std::chrono::steady_clock::time_point t) {
        cudaDeviceSynchronize();
        return std::chrono::duration<double, std::milli>(now() - t).count();
    };

    // TV_VERBOSE=3: per-round GPU time (events, no host syncs) next to host time
    const bool evlog = std::getenv("TV_VERBOSE") && std::atoi(std::getenv("TV_VERBOSE")) == 3;
    std::vector<cudaEvent_t> marks;
    std::vector<double> host_ms;
    auto mark = [&]() {
        if (!evlog) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, 0);
        marks.push_back(e);
        host_ms.push_back(std::chrono::duration<double, std::milli>(now().time_since_epoch()).count());
    };
    mark();
    for (;;) {
        const auto t_round = now();
        // ---- eval fresh leaves ----
        clear_flag_kernel<<<nblk(n_fresh), 256>>>(fresh_b.as<uint32_t>(), n_fresh, flags_b.as<uint8_t>(), F_NEW);
        stats_zero_kernel<<<nblk(n_fresh), 256>>>(fresh_b.as<uint32_t>(), n_fresh, stats_b.as<Stats>(),
                                                  flags_b.as<uint8_t>());
        // round 0: root scan of every voxel; later: descend the voxels whose
        // owner was bisected, skip the rest
        // this round's fresh leaves have ids in [fresh_lo, n_t): stripe their
        // statistics while they are few (early rounds: hot atomics)
        StatsSink sink{stats_b.as<Stats>(), nullptr, 0u, 0u};
        const uint32_t fresh_range = n_t - fresh_lo;
        if (fresh_range <= kStripeOwners) {
            TRY(ensure(stripe_b, static_cast<size_t>(fresh_range) * kStripes * sizeof(Stats)));
            stripe_zero_kernel<<<nblk(fresh_range * kStripes), 256>>>(stripe_b.as<Stats>(), fresh_range * kStripes);
            sink = StatsSink{stats_b.as<Stats>(), stripe_b.as<Stats>(), fresh_lo, fresh_range};
        }
        if (rounds == 0 && use_bricks) {
            CK(cudaMemset(S.mixedn.p, 0, sizeof(uint32_t)), "bricks");
            brick_root_kernel<<<vox_blocks, kVoxThreads>>>(V, R, verts_b.as<uint4>(), owner_b.as<uint32_t>(),
                                                           brick_owner, S.subs.as<uint32_t>(),
                                                           S.bstat.as<BrickStat>(), sink,
                                                           S.mixed.as<uint32_t>(), S.mixedn.as<uint32_t>());
        } else if (rounds == 0) {
            vox_stats_kernel<kVoxInit><<<vox_blocks, kVoxThreads>>>(V, R, verts_b.as<uint4>(), split_b.as<NodeRec>(),
                                                                    flags_b.as<uint8_t>(), owner_b.as<uint32_t>(),
                                                                    sink, 0);
        } else if (use_bricks) {
            brick_descend_kernel<<<std::min<unsigned>(nblk(n_bricks, 256), n_sm * 16), 256>>>(
                V, n_bricks, brick_owner, S.bstat.as<BrickStat>(), split_b.as<NodeRec>(), flags_b.as<uint8_t>(), sink,
                S.mixed.as<uint32_t>(), S.mixedn.as<uint32_t>());
            brick_voxels_kernel<<<vox_blocks, kVoxThreads>>>(
                V, brick_owner, S.subs.as<uint32_t>(), S.sstat.as<BrickStat>(), S.mixed.as<uint32_t>(),
                S.mixedn.as<uint32_t>(), split_b.as<NodeRec>(), flags_b.as<uint8_t>(), owner_b.as<uint32_t>(), sink,
                bmark);
            // the marks of the coming closure start empty
            CK(cudaMemsetAsync(S.bmark.p, 0, mark_words * sizeof(uint32_t), 0), "brick marks");
        } else {
            vox_stats_kernel<kVoxDescend><<<vox_blocks, kVoxThreads>>>(
                V, R, verts_b.as<uint4>(), split_b.as<NodeRec>(), flags_b.as<uint8_t>(), owner_b.as<uint32_t>(),
                sink, 0);
        }
        if (sink.n) stripe_combine_kernel<<<nblk(sink.n), 256>>>(sink.stripe, sink.lo, sink.n, stats_b.as<Stats>());
        CK(cudaGetLastError(), "voxel ownership");
        eval_kernel<<<nblk(n_fresh, 128), 128>>>(fresh_b.as<uint32_t>(), n_fresh, V, owner_b.as<uint32_t>(),
                                                  tets_b.as<tv_tet>(), verts_b.as<uint4>(), stats_b.as<Stats>(), E,
                                                  flags_b.as<uint8_t>(), d_ctr);
        CK(cudaGetLastError(), "eval");
        TRY(select_listed(fresh_b.as<uint32_t>(), n_fresh, F_MARK, marked_b, n_marked));
        const double ms_eval = verbose ? since(t_round) : 0.0;
        if (verbose) {
            unsigned long long c[2];
            cudaMemcpy(c, d_ctr, sizeof(c), cudaMemcpyDeviceToHost);
            std::fprintf(stderr, "tetvol_b200: build round %d: fresh %u marked %u eval %.2f ms (replays %llu)\n",
                         rounds, n_fresh, n_marked, ms_eval, c[0]);
        }
        if (n_marked == 0) break;
        crit += n_marked;
        ++rounds;
        fresh_lo = n_t;  // every leaf the coming closure creates has an id >= fresh_lo
        // ---- closure ----
        double ph[4] = {0, 0, 0, 0};  // verbose: midpoint+dedup, bisect, leaves+hanging, select
        while (n_marked) {
            auto tp = now();
            TRY(grow_tets(static_cast<size_t>(n_t) + 2ull * n_marked));
            TRY(grow_verts(static_cast<size_t>(n_v) + n_marked));
            TRY(ensure(mid_b, n_marked * sizeof(uint32_t)));
            TRY(ensure(miss_hi_b, n_marked * sizeof(uint64_t)));
            TRY(ensure(miss_lo_b, n_marked * sizeof(uint32_t)));
            TRY(ensure(miss_idx_b, n_marked * sizeof(uint32_t)));
            TRY(ensure(miss_idx2_b, n_marked * sizeof(uint32_t)));
            TRY(ensure(head_b, n_marked * sizeof(uint32_t)));
            TRY(ensure(scan_b, n_marked * sizeof(uint32_t)));
            {
                // pending-claim table: a power of two >= 2 n_marked slots, empty between passes
                size_t pslots = 1024;
                while (pslots < 2ull * n_marked) pslots <<= 1;
                if (S.pend.bytes < pslots * sizeof(HSlot)) {
                    const size_t had = pend_clean ? S.pend.bytes : 0;
                    TRY(ensure(S.pend, pslots * sizeof(HSlot)));
                    CK(cudaMemset(static_cast<char*>(S.pend.p) + had, 0xff, S.pend.bytes - had), "pending clear");
                } else if (!pend_clean) {  // first pass of this build: the table may hold anything
                    CK(cudaMemset(S.pend.p, 0xff, S.pend.bytes), "pending clear");
                }
                pend_clean = true;  // every pass frees the slots it claims
            }
            const uint64_t pmask = S.pend.bytes / sizeof(HSlot);  // every slot is used: mask = slots - 1
            uint64_t pm = 1;
            while (pm * 2 <= pmask) pm *= 2;
            midpoint_kernel<<<nblk(n_marked), 256>>>(marked_b.as<uint32_t>(), n_marked, tets_b.as<tv_tet>(),
                                                     verts_b.as<uint4>(), table_b.as<HSlot>(), hmask,
                                                     mid_b.as<uint32_t>(), miss_hi_b.as<uint64_t>(),
                                                     miss_lo_b.as<uint32_t>(), S.pend.as<HSlot>(), pm - 1, d_err);
            CK(cudaGetLastError(), "midpoints");
            midpoint_win_kernel<<<nblk(n_marked), 256>>>(mid_b.as<uint32_t>(), n_marked, miss_hi_b.as<uint64_t>(),
                                                         miss_lo_b.as<uint32_t>(), S.pend.as<HSlot>(), pm - 1,
                                                         miss_idx_b.as<uint32_t>(), miss_idx2_b.as<uint32_t>(),
                                                         head_b.as<uint32_t>());
            {
                size_t tb3 = 0;
                CK(cub::DeviceScan::InclusiveSum(nullptr, tb3, head_b.as<uint32_t>(), scan_b.as<uint32_t>(),
                                                 static_cast<int>(n_marked)),
                   "scan sizing");
                TRY(ensure(tmp_b, tb3));
                CK(cub::DeviceScan::InclusiveSum(tmp_b.p, tb3, head_b.as<uint32_t>(), scan_b.as<uint32_t>(),
                                                 static_cast<int>(n_marked)),
                   "scan");
            }
            // capacity for n_v + n_marked vertices is already mapped (new vertices <= n_marked)
            midpoint_assign_kernel<<<nblk(n_marked), 256>>>(
                mid_b.as<uint32_t>(), n_marked, miss_hi_b.as<uint64_t>(), miss_lo_b.as<uint32_t>(),
                miss_idx_b.as<uint32_t>(), miss_idx2_b.as<uint32_t>(), scan_b.as<uint32_t>(), n_v,
                verts_b.as<uint4>(), table_b.as<HSlot>(), hmask, S.pend.as<HSlot>());
            CK(cudaGetLastError(), "midpoint ids");
            const uint32_t n_pass = n_marked;
            if (verbose) ph[0] += since(tp), tp = now();
            CK(cudaMemset(vtouch_b.p, 0, (n_v + 31) / 32 * 4), "vtouch");  // bisect touches existing vertices only
            bisect_kernel<<<nblk(n_marked), 256>>>(marked_b.as<uint32_t>(), n_marked, n_t, tets_b.as<tv_tet>(),
                                                   tv4_b.as<uint4>(), verts_b.as<uint4>(), mid_b.as<uint32_t>(),
                                                   split_b.as<NodeRec>(), flags_b.as<uint8_t>(),
                                                   vtouch_b.as<uint32_t>(), grid_max_level, d_err, bmark);
            CK(cudaGetLastError(), "bisect");
            const uint32_t first_new = n_t;
            n_t += 2 * n_marked;
            bisections += n_marked;
            ++passes;
            if (verbose) ph[1] += since(tp), tp = now();
            // hanging test, then the marked list (ascending ids): over every tet
            // id, or, for a pass with few bisections, over the new children plus
            // the old leaves around the pass's new midpoints (hanging_probe_kernel)
            const bool probe = hang_probe && static_cast<uint64_t>(n_pass) * hang_probe_cost < first_new;
            if (probe) {
                hanging_kernel<<<nblk(n_t - first_new), 256>>>(first_new, n_t, first_new, tv4_b.as<uint4>(),
                                                               verts_b.as<uint4>(), table_b.as<HSlot>(), hmask,
                                                               vtouch_b.as<uint32_t>(), flags_b.as<uint8_t>());
                hanging_probe_kernel<<<nblk(32ull * n_pass), 256>>>(
                    marked_b.as<uint32_t>(), n_pass, mid_b.as<uint32_t>(), head_b.as<uint32_t>(), first_new,
                    tets_b.as<tv_tet>(),
                    tv4_b.as<uint4>(), verts_b.as<uint4>(), table_b.as<HSlot>(), hmask, R, split_b.as<NodeRec>(),
                    flags_b.as<uint8_t>());
                ++probe_passes;
            }
            if (!probe || hang_check) {
                uint32_t n_probe_marks = 0;
                if (probe) {  // TV_HANG_CHECK: the full scan must add no mark the probes missed
                    TRY(select_tets(F_MARK, marked_b, &n_probe_marks));
                }
                hanging_kernel<<<nblk(n_t), 256>>>(0, n_t, first_new, tv4_b.as<uint4>(), verts_b.as<uint4>(),
                                                   table_b.as<HSlot>(), hmask, vtouch_b.as<uint32_t>(),
                                                   flags_b.as<uint8_t>());
                if (probe) {
                    uint32_t n_scan_marks = 0;
                    TRY(select_tets(F_MARK, marked_b, &n_scan_marks));
                    if (n_scan_marks != n_probe_marks) {
                        std::fprintf(stderr, "tetvol_b200: TV_HANG_CHECK: probes marked %u leaves, the scan %u\n",
                                     n_probe_marks, n_scan_marks);
                        hang_mismatch = true;
                    }
                }
            }
            CK(cudaGetLastError(), "hanging");
            if (verbose) ph[2] += since(tp), tp = now();
            TRY(select_tets(F_MARK, marked_b, nullptr));
            pass_state_kernel<<<1, 1>>>(scan_b.as<uint32_t>(), n_pass, d_cnt, d_err, d_state);
            uint32_t hs[3];
            CK(cudaMemcpy(hs, d_state, sizeof(hs), cudaMemcpyDeviceToHost), "pass state");
            n_v += hs[0];
            n_marked = hs[1];
            herr = static_cast<int>(hs[2]);
            if (herr) break;
            clear_flag_kernel<<<nblk(n_marked), 256>>>(marked_b.as<uint32_t>(), n_marked, flags_b.as<uint8_t>(), F_MARK);
            CK(cudaGetLastError(), "clear");
            if (verbose) ph[3] += since(tp);
        }
        if (verbose)
            std::fprintf(stderr, "tetvol_b200: build round %d phases: mid+dedup %.1f bisect %.1f hanging %.1f select %.1f ms\n",
                         rounds, ph[0], ph[1], ph[2], ph[3]);
        if (herr) break;
        // fresh = leaves created in this round
        TRY(select_tets(F_NEW, fresh_b, &n_fresh));
        if (verbose) std::fprintf(stderr, "tetvol_b200: build round %d: closure done, %.2f ms total\n", rounds,
                                  since(t_round));
        mark();
    }
    if (verbose) std::fprintf(stderr, "tetvol_b200: build: %llu of %llu closure passes took the probe hanging test\n",
                              static_cast<unsigned long long>(probe_passes), static_cast<unsigned long long>(passes));
    if (hang_mismatch) return set_error(TV_ERR, "TV_HANG_CHECK: probe hanging test differs from the full scan");
    if (herr) {
        if (herr & E_LEVEL) return set_error(TV_ERR_GRID, "bisect: level cap reached");
        if (herr & E_MIDPOINT) return set_error(TV_ERR_GRID, "bisect: midpoint not representable");
        if (herr & E_NORMAL) return set_error(TV_ERR_GRID, "normal direction not in table");
        return set_error(TV_ERR_GRID, "build failed");
    }

    // ---- payloads for every leaf (builder.cpp:164-182) ----
    TRY(select_tets(F_LEAF, leaves_b, &n_leaves));
    // Every leaf's density statistics are those of its evaluation round (its
    // voxels have not changed owner since). Temperature / albedo sums need one
    // more pass over the (final) owner map.
    if (use_bricks && (temp || alb)) {  // the payload sweep reads the owner map alone
        brick_fill_kernel<<<vox_blocks, kVoxThreads>>>(V, brick_owner, S.subs.as<uint32_t>(), n_bricks,
                                                       owner_b.as<uint32_t>());
        CK(cudaGetLastError(), "brick fill");
    }
    if (temp || alb) {
        stats_zero_kernel<<<nblk(n_leaves), 256>>>(leaves_b.as<uint32_t>(), n_leaves, stats_b.as<Stats>(),
                                                   flags_b.as<uint8_t>());
        vox_stats_kernel<kVoxAll><<<vox_blocks, kVoxThreads>>>(V, R, verts_b.as<uint4>(), split_b.as<NodeRec>(),
                                                               flags_b.as<uint8_t>(), owner_b.as<uint32_t>(),
                                                               StatsSink{stats_b.as<Stats>(), nullptr, 0u, 0u}, 1);
        CK(cudaGetLastError(), "voxel statistics");
    }
    PayloadParams PP{cfg->density_scale, temp != nullptr, alb != nullptr};
    payload_kernel<<<nblk(n_leaves, 128), 128>>>(leaves_b.as<uint32_t>(), n_leaves, V, owner_b.as<uint32_t>(),
                                                 tets_b.as<tv_tet>(), verts_b.as<uint4>(), stats_b.as<Stats>(), PP,
                                                 d_ctr, d_depth);
    CK(cudaGetLastError(), "payloads");

    // ---- neighbour links by face pairing (tet_grid.cpp:130-152) ----
    {
        const uint64_t nf = 4ull * n_leaves;
        Buf &khi = S.khi, &klo = S.klo, &rec = S.rec, &khi2 = S.khi2, &klo2 = S.klo2, &rec2 = S.rec2;
        TRY(ensure(khi, nf * 8));
        TRY(ensure(klo, nf * 4));
        TRY(ensure(rec, nf * 4));
        TRY(ensure(khi2, nf * 8));
        TRY(ensure(klo2, nf * 4));
        TRY(ensure(rec2, nf * 4));
        int vb = 1;  // bits of a vertex id
        while (vb < 32 && (1ull << vb) < n_v) ++vb;
        face_keys_kernel<<<nblk(n_leaves), 256>>>(leaves_b.as<uint32_t>(), n_leaves, tets_b.as<tv_tet>(),
                                                  khi.as<uint64_t>(), klo.as<uint32_t>(), rec.as<uint32_t>(), vb);
        CK(cudaGetLastError(), "face keys");
        size_t tb1 = 0, tb2 = 0;
        CK(cub::DeviceRadixSort::SortPairs(nullptr, tb1, klo.as<uint32_t>(), klo2.as<uint32_t>(), rec.as<uint32_t>(),
                                           rec2.as<uint32_t>(), static_cast<int>(nf), 0, vb),
           "sort sizing");
        CK(cub::DeviceRadixSort::SortPairs(nullptr, tb2, khi.as<uint64_t>(), khi2.as<uint64_t>(), rec2.as<uint32_t>(),
                                           rec.as<uint32_t>(), static_cast<int>(nf), 0, 2 * vb),
           "sort sizing");
        TRY(ensure(tmp_b, std::max(tb1, tb2)));
        // sort by v2, gather v0v1 in that order, then stable sort by v0v1
        CK(cub::DeviceRadixSort::SortPairs(tmp_b.p, tb1, klo.as<uint32_t>(), klo2.as<uint32_t>(), rec.as<uint32_t>(),
                                           rec2.as<uint32_t>(), static_cast<int>(nf), 0, vb),
           "face sort lo");
        gather_face_hi_kernel<<<nblk(nf), 256>>>(rec2.as<uint32_t>(), nf, leaves_b.as<uint32_t>(), tets_b.as<tv_tet>(),
                                                 khi.as<uint64_t>(), klo.as<uint32_t>(), vb);
        CK(cudaGetLastError(), "face gather");
        CK(cub::DeviceRadixSort::SortPairs(tmp_b.p, tb2, khi.as<uint64_t>(), khi2.as<uint64_t>(), rec2.as<uint32_t>(),
                                           rec.as<uint32_t>(), static_cast<int>(nf), 0, 2 * vb),
           "face sort hi");
        gather_face_hi_kernel<<<nblk(nf), 256>>>(rec.as<uint32_t>(), nf, leaves_b.as<uint32_t>(), tets_b.as<tv_tet>(),
                                                 khi2.as<uint64_t>(), klo2.as<uint32_t>(), vb);
        face_pair_kernel<<<nblk(nf), 256>>>(khi2.as<uint64_t>(), klo2.as<uint32_t>(), rec.as<uint32_t>(), nf,
                                            leaves_b.as<uint32_t>(), tets_b.as<tv_tet>(), d_err);
        CK(cudaGetLastError(), "face pair");
    }
    CK(cudaMemcpy(&herr, d_err, sizeof(int), cudaMemcpyDeviceToHost), "err");
    if (herr & E_FACE) return set_error(TV_ERR_GRID, "face shared by more than two leaves");
    if (evlog && marks.size() > 1) {
        cudaDeviceSynchronize();
        for (size_t k = 1; k < marks.size(); ++k) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, marks[k - 1], marks[k]);
            std::fprintf(stderr, "tetvol_b200: build round %zu: gpu %.1f ms host %.1f ms\n", k, ms,
                         host_ms[k] - host_ms[k - 1]);
        }
        for (auto e : marks) cudaEventDestroy(e);
    }
    unsigned long long hctr[2] = {0, 0};
    CK(cudaMemcpy(hctr, d_ctr, sizeof(hctr), cudaMemcpyDeviceToHost), "counters");
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);

    // ---- hand the pools to the traversal layout ----
    auto h = new tv_grid();
    DeviceGrid& g = h->g;
    g.device = device;
    g.n_vertices = n_v;
    g.n_tets = n_t;
    g.n_leaves = n_leaves;
    g.n_internal = n_t - n_leaves;
    g.max_level = grid_max_level;
    std::memcpy(g.roots, roots, sizeof(roots));
    cudaError_t e = cudaMalloc(&g.tets, static_cast<size_t>(n_t) * sizeof(tv_tet));
    if (e == cudaSuccess) e = cudaMalloc(&g.verts, static_cast<size_t>(n_v) * sizeof(uint4));
    if (e == cudaSuccess)
        e = cudaMemcpy(g.tets, tets_b.p, static_cast<size_t>(n_t) * sizeof(tv_tet), cudaMemcpyDeviceToDevice);
    if (e == cudaSuccess)
        e = cudaMemcpy(g.verts, verts_b.p, static_cast<size_t>(n_v) * sizeof(uint4), cudaMemcpyDeviceToDevice);
    if (e != cudaSuccess) {
        free_grid(g);
        delete h;
        return cuda_status(e, "build output");
    }
    g.bytes = static_cast<uint64_t>(n_t) * sizeof(tv_tet) + static_cast<uint64_t>(n_v) * sizeof(uint4);
    rc = finalize_grid(g, nullptr);
    if (rc) {
        free_grid(g);
        delete h;
        return rc;
    }
    if (stats) {
        stats->leaf_count = n_leaves;
        stats->max_depth = g.max_depth;
        stats->rounds = rounds;
        stats->seconds = ms * 1e-3;
        stats->criterion_splits = crit;
        stats->propagation_splits = bisections - crit;
        stats->closure_passes = passes;
        stats->voxel_visits = hctr[1];
    }
    (void)replays;
    *out = h;
    return TV_OK;
#undef CK
#undef TRY
}
}  // namespace

int build_grid(const float* dens, const float* temp, const float* alb, int nx, int ny, int nz,
               const tv_build_config* cfg, const tv_camera* camera, int device, tv_grid** out, tv_build_stats* stats) {
    t_build_device = device;
    static const bool cache = !std::getenv("TV_BUILD_CACHE") || std::atoi(std::getenv("TV_BUILD_CACHE"));
    if (!cache) {
        BuildScratch local;
        return build_grid_impl(dens, temp, alb, nx, ny, nz, cfg, camera, device, out, stats, local);
    }
    BuildScratch* S;
    {
        std::lock_guard<std::mutex> g(g_scratch_mu);
        BuildScratch*& p = scratch_map()[device];
        if (!p) p = new BuildScratch();
        S = p;
    }
    std::lock_guard<std::mutex> lk(S->m);  // one build per device at a time
    if (poison())
        S->each([](Buf& b) {
            if (b.bytes) cudaMemset(b.p, 0x5A, b.bytes);
        });
    const int rc = build_grid_impl(dens, temp, alb, nx, ny, nz, cfg, camera, device, out, stats, *S);
    if (rc) S->release();  // a failed build (often out of memory) gives its scratch back
    return rc;
}

int trim_scratch(int device) {
    int cur = 0;
    cudaGetDevice(&cur);
    std::lock_guard<std::mutex> g(g_scratch_mu);
    for (auto& kv : scratch_map()) {
        if (device >= 0 && kv.first != device) continue;
        std::lock_guard<std::mutex> lk(kv.second->m);
        if (!kv.second->bytes()) continue;
        cudaSetDevice(kv.first);
        kv.second->release();
    }
    cudaSetDevice(cur);
    return TV_OK;
}

size_t scratch_bytes(int device) {
    std::lock_guard<std::mutex> g(g_scratch_mu);
    size_t n = 0;
    for (auto& kv : scratch_map())
        if (device < 0 || kv.first == device) {
            std::lock_guard<std::mutex> lk(kv.second->m);
            n += kv.second->bytes();
        }
    return n;
}

}  // namespace tvb

using namespace tvb;

namespace {
// The reference validates BuildConfig and constructs the camera before any
// work (builder.cpp:120-121, camera.cpp:15-20); so do we, before touching the
// device.
int prevalidate(const tv_build_config* cfg, const tv_camera* camera) {
    int rc = validate_build_cfg(cfg);
    if (rc) return rc;
    if (cfg->use_camera && !camera) return set_error(TV_ERR_CONFIG, "useCamera set but no camera given");
    if (camera) {
        CamView cv;
        d3 pn[5];
        double pd[5];
        if ((rc = host_camera(camera, cv, pn, pd))) return rc;
    }
    return TV_OK;
}
}  // namespace

extern "C" {

int tv_check_build_config(const tv_build_config* cfg) { return validate_build_cfg(cfg); }

int tv_build_trim(int device) { return trim_scratch(device); }

uint64_t tv_build_scratch_bytes(int device) { return scratch_bytes(device); }

int tv_generate_volume_dev(int32_t kind, int32_t nx, int32_t ny, int32_t nz, double value, float* out_dev,
                           int device) {
    if (!out_dev) return set_error(TV_ERR_ARG, "null output");
    if (nx < 1 || ny < 1 || nz < 1 || nx > 4096 || ny > 4096 || nz > 4096)
        return set_error(TV_ERR_CONFIG, "dims out of range [1, 4096]");
    if (kind < 0 || kind > 5) return set_error(TV_ERR_CONFIG, "unknown kind (constant|ramp|blob|step|noise|cloud)");
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_status(e, "cudaSetDevice");
    gen_kernel<<<148 * 8, 256>>>(kind, nx, ny, nz, value, out_dev);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    return cuda_status(e, "generate volume");
}

int tv_build_dev(const float* density_dev, const float* temperature_dev, const float* albedo_dev, int32_t nx,
                 int32_t ny, int32_t nz, const tv_build_config* cfg, const tv_camera* camera, int device,
                 tv_grid** out, tv_build_stats* stats) {
    if (!out || !density_dev) return set_error(TV_ERR_ARG, "null argument");
    *out = nullptr;
    int rc = prevalidate(cfg, camera);
    if (rc) return rc;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return set_error(TV_ERR_CUDA, "no CUDA device available");
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_status(e, "cudaSetDevice");
    return build_grid(density_dev, temperature_dev, albedo_dev, nx, ny, nz, cfg, camera, device, out, stats);
}

int tv_build(const float* density, const float* temperature, const float* albedo, int32_t nx, int32_t ny,
             int32_t nz, const tv_build_config* cfg, const tv_camera* camera, int device, tv_grid** out,
             tv_build_stats* stats) {
    if (!out || !density) return set_error(TV_ERR_ARG, "null argument");
    *out = nullptr;
    if (nx < 1 || ny < 1 || nz < 1) return set_error(TV_ERR_CONFIG, "volume dimensions must be positive");
    int rc0 = prevalidate(cfg, camera);
    if (rc0) return rc0;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return set_error(TV_ERR_CUDA, "no CUDA device available");
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_status(e, "cudaSetDevice");
    const size_t nv = static_cast<size_t>(nx) * ny * nz * sizeof(float);
    float *d = nullptr, *t = nullptr, *a = nullptr;
    e = cudaMalloc(&d, nv);
    if (e == cudaSuccess && temperature) e = cudaMalloc(&t, nv);
    if (e == cudaSuccess && albedo) e = cudaMalloc(&a, nv);
    if (e == cudaSuccess) e = cudaMemcpy(d, density, nv, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && t) e = cudaMemcpy(t, temperature, nv, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && a) e = cudaMemcpy(a, albedo, nv, cudaMemcpyHostToDevice);
    int rc = e == cudaSuccess ? build_grid(d, t, a, nx, ny, nz, cfg, camera, device, out, stats)
                              : cuda_status(e, "volume upload");
    cudaFree(d);
    cudaFree(t);
    cudaFree(a);
    return rc;
}

}  // extern "C"
