// TetGrid::validate (tet_grid.cpp:474-636) on the GPU, over the reference-layout
// pools a tv_grid keeps in HBM, and cmd_validate's traversal spot checks
// (cli.cpp:560-604) against BruteForceTraverser (tet_grid.cpp:659-698).
//
// The reference stops at nothing but records only its FIRST violation, in a
// fixed sequential order. Each phase here evaluates all its records in
// parallel and keeps the minimum of (record position << 4 | check index), the
// record positions being the reference's iteration order, so the reported
// first_violation and the face / leaf counts are the reference's exactly.
// Phases in the reference's order:
//   A  root table                          (host, 24 records)
//   B  duplicate vertices                  (radix sort of the (x, y, z) keys)
//   C  vertex coordinate range
//   D  per-tet: level cap, vertex ids (ends the scan), orientation, children,
//      payload; leaf count and the exact i128 volume sum (== 6 << 72)
//   G1 leaf neighbours are leaves          (per leaf, tet order)
//   G2 face matching                       (faces sorted by key, then tet, slot)
//   H  stored normals re-derived from geometry (only when still ok)
// The edge-ring check compares the grid's cached rings with a recomputation;
// a device grid caches none (TetGrid::assemble rebuilds them from the leaves),
// so it holds by construction.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "tv_leb.cuh"
#include "tv_trace.cuh"

namespace tvb {
namespace {

constexpr uint32_t kOneQ = 1u << 24;
constexpr unsigned long long kNoFail = ~0ull;

const char* const kMsgD[] = {"tet exceeds the level cap",
                             "vertex id out of range",
                             "leaf with non-positive orientation",
                             "internal tet with invalid children",
                             "child does not point back to its parent",
                             "child level is not parent level + 1",
                             "internal tet carries a payload"};
const char* const kMsgG2[] = {"unmatched interior face (T-junction)", "boundary face has a neighbor link",
                              "tet paired with itself across a face", "neighbor links are not reciprocal",
                              "shared face normals are not opposite", "face shared by more than two leaves"};

__device__ __forceinline__ void fail_min(unsigned long long* slot, uint64_t pos, uint32_t code) {
    atomicMin(slot, static_cast<unsigned long long>((pos << 4) | code));
}

__device__ __forceinline__ bool is_leaf(const tv_tet& t) { return t.children[0] == kNone; }

__global__ void iota_kernel(uint32_t* p, uint64_t n) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        p[i] = static_cast<uint32_t>(i);
}

// key k of vertex order[i]
__global__ void vkey_kernel(const uint4* v, const uint32_t* order, uint64_t n, int k, uint32_t* key,
                            unsigned long long* range_bad) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint4 q = v[order[i]];
        key[i] = k == 0 ? q.x : (k == 1 ? q.y : q.z);
        if (range_bad && (q.x > kOneQ || q.y > kOneQ || q.z > kOneQ)) atomicMin(range_bad, 0ull);
    }
}

__global__ void vdup_kernel(const uint4* v, const uint32_t* order, uint64_t n, unsigned long long* dup) {
    for (uint64_t i = 1 + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint4 a = v[order[i - 1]], b = v[order[i]];
        if (a.x == b.x && a.y == b.y && a.z == b.z) atomicMin(dup, 0ull);
    }
}

struct Acc {
    unsigned long long fail_d;   // min (t << 4 | code)
    unsigned long long vid;      // min t with a vertex id out of range
    unsigned long long leaves;
    unsigned long long vol_lo, vol_hi;  // unsigned 128-bit sum of leaf determinants
    unsigned long long fail_g1;
    unsigned long long fail_g2;  // min (sorted group start << 4 | code)
    unsigned long long boundary, interior;
    unsigned long long fail_h;   // min ((t * 4 + slot) << 4 | code)
};

// phase D (tet_grid.cpp:503-531)
__global__ void tets_kernel(const tv_tet* __restrict__ tets, const uint4* __restrict__ verts, uint64_t nt, uint64_t nv,
                            int max_level, Acc* acc) {
    for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < nt;
         t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const tv_tet tt = tets[t];
        if (tt.level > max_level) fail_min(&acc->fail_d, t, 0);
        bool vbad = false;
        for (int k = 0; k < 4; ++k) vbad |= tt.verts[k] >= nv;
        if (vbad) {
            fail_min(&acc->fail_d, t, 1);
            atomicMin(&acc->vid, static_cast<unsigned long long>(t));
            continue;
        }
        if (is_leaf(tt)) {
            atomicAdd(&acc->leaves, 1ull);
            const i128 d =
                det_fixed(verts[tt.verts[0]], verts[tt.verts[1]], verts[tt.verts[2]], verts[tt.verts[3]]);
            if (d <= 0) fail_min(&acc->fail_d, t, 2);
            const unsigned __int128 u = static_cast<unsigned __int128>(d);
            const unsigned long long lo = static_cast<unsigned long long>(u),
                                     hi = static_cast<unsigned long long>(u >> 64);
            const unsigned long long old = atomicAdd(&acc->vol_lo, lo);
            atomicAdd(&acc->vol_hi, hi + (old + lo < old ? 1ull : 0ull));
        } else {
            if (tt.children[1] == kNone || tt.children[0] >= nt || tt.children[1] >= nt) {
                fail_min(&acc->fail_d, t, 3);
                continue;
            }
            uint32_t code = 16;
            for (int k = 0; k < 2 && code == 16; ++k) {
                const tv_tet c = tets[tt.children[k]];
                if (c.parent != t) code = 4;
                else if (c.level != tt.level + 1) code = 5;
            }
            if (code == 16 && (tt.mask & 1u)) code = 6;
            if (code != 16) fail_min(&acc->fail_d, t, code);
        }
    }
}

// phase G1 + face records of leaves (tet_grid.cpp:543-557)
__global__ void faces_kernel(const tv_tet* __restrict__ tets, uint64_t nt, const uint32_t* __restrict__ leaf_pos,
                             uint32_t* k0, uint32_t* k1, uint32_t* k2, uint32_t* rec, Acc* acc) {
    for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < nt;
         t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const tv_tet tt = tets[t];
        if (!is_leaf(tt)) continue;
        for (int s = 0; s < 4; ++s) {
            const uint32_t nb = tt.neighbors[s];
            if (nb != kNone && (nb >= nt || !is_leaf(tets[nb]))) {
                fail_min(&acc->fail_g1, t, 0);
                break;
            }
        }
        const uint64_t base = 4ull * leaf_pos[t];
        for (int slot = 0; slot < 4; ++slot) {
            uint32_t k[3];
            int n = 0;
            for (int s = 0; s < 4; ++s)
                if (s != slot) k[n++] = tt.verts[s];
            if (k[0] > k[1]) { const uint32_t x = k[0]; k[0] = k[1]; k[1] = x; }
            if (k[1] > k[2]) { const uint32_t x = k[1]; k[1] = k[2]; k[2] = x; }
            if (k[0] > k[1]) { const uint32_t x = k[0]; k[0] = k[1]; k[1] = x; }
            k0[base + slot] = k[0], k1[base + slot] = k[1], k2[base + slot] = k[2];
            rec[base + slot] = static_cast<uint32_t>(base + slot);
        }
    }
}

__global__ void leaf_flag_kernel(const tv_tet* __restrict__ tets, uint64_t nt, uint32_t* flag) {
    for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < nt;
         t += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        flag[t] = is_leaf(tets[t]) ? 1u : 0u;
}

// gather key k for the current permutation
__global__ void fkey_kernel(const uint32_t* kk, const uint32_t* perm, uint64_t n, uint32_t* out) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        out[i] = kk[perm[i]];
}

// phase G2 over groups of equal keys in sorted order (tet_grid.cpp:562-593).
// face record r = 4 * leaf_position + slot; leaf_tet maps positions to TetIds.
__global__ void groups_kernel(const tv_tet* __restrict__ tets, const uint4* __restrict__ verts,
                              const uint32_t* __restrict__ k0, const uint32_t* __restrict__ k1,
                              const uint32_t* __restrict__ k2, const uint32_t* __restrict__ perm,
                              const uint32_t* __restrict__ leaf_tet, uint64_t nf, Acc* acc) {
    auto same = [&](uint64_t a, uint64_t b) {
        const uint32_t ra = perm[a], rb = perm[b];
        return k0[ra] == k0[rb] && k1[ra] == k1[rb] && k2[ra] == k2[rb];
    };
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < nf;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        if (i > 0 && same(i - 1, i)) continue;  // not a group start
        uint64_t j = i + 1;
        while (j < nf && same(i, j)) ++j;
        const uint64_t n = j - i;
        const uint32_t ra = perm[i];
        const uint32_t ta = leaf_tet[ra >> 2], sa = ra & 3u;
        if (n == 1) {
            atomicAdd(&acc->boundary, 1ull);
            bool on_surface = false;
            const uint32_t key[3] = {k0[ra], k1[ra], k2[ra]};
            for (int axis = 0; axis < 3 && !on_surface; ++axis)
                for (int w = 0; w < 2 && !on_surface; ++w) {
                    const uint32_t val = w ? kOneQ : 0u;
                    bool all = true;
                    for (int m = 0; m < 3; ++m) {
                        const uint4 q = verts[key[m]];
                        all &= (axis == 0 ? q.x : (axis == 1 ? q.y : q.z)) == val;
                    }
                    on_surface = all;
                }
            if (!on_surface) fail_min(&acc->fail_g2, i, 0);
            else if (tets[ta].neighbors[sa] != kNone) fail_min(&acc->fail_g2, i, 1);
        } else if (n == 2) {
            atomicAdd(&acc->interior, 1ull);
            const uint32_t rb = perm[i + 1];
            const uint32_t tb = leaf_tet[rb >> 2], sb = rb & 3u;
            const tv_tet A = tets[ta], Bt = tets[tb];
            if (ta == tb) fail_min(&acc->fail_g2, i, 2);
            else if (A.neighbors[sa] != tb || Bt.neighbors[sb] != ta) fail_min(&acc->fail_g2, i, 3);
            else if ((A.normal_ids[sa] ^ 1u) != Bt.normal_ids[sb]) fail_min(&acc->fail_g2, i, 4);
        } else {
            fail_min(&acc->fail_g2, i, 5);
        }
    }
}

// phase H (tet_grid.cpp:596-615)
__global__ void normals_kernel(const tv_tet* __restrict__ tets, const uint4* __restrict__ verts, uint64_t nt,
                               Acc* acc) {
    for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < nt;
         t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const tv_tet tt = tets[t];
        if (!is_leaf(tt)) continue;
        for (int slot = 0; slot < 4; ++slot) {
            uint4 f[3];
            int n = 0;
            for (int s = 0; s < 4; ++s)
                if (s != slot) f[n++] = verts[tt.verts[s]];
            const int id = face_normal_id(f[0], f[1], f[2], verts[tt.verts[slot]]);
            if (id < 0) {
                fail_min(&acc->fail_h, 4 * t + slot, 1);
                break;
            }
            if (id != tt.normal_ids[slot]) {
                fail_min(&acc->fail_h, 4 * t + slot, 0);
                break;
            }
        }
    }
}

// BruteForceTraverser (tet_grid.cpp:659-698): one pass over all leaves per ray
__global__ void brute_kernel(const tv_tet* __restrict__ tets, const uint4* __restrict__ verts, uint64_t nt, d3 o,
                             d3 dir, double tmin, double tmax, tv_segment* out, unsigned long long* count,
                             uint64_t cap) {
    for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < nt;
         t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const tv_tet tt = tets[t];
        if (!is_leaf(tt)) continue;
        d3 c[4];
        for (int k = 0; k < 4; ++k) {
            const uint4 q = verts[tt.verts[k]];
            c[k] = mk(q.x * kInvCoord, q.y * kInvCoord, q.z * kInvCoord);
        }
        double t0 = tmin, t1 = tmax;
        bool hit = true;
        for (int slot = 0; slot < 4 && hit; ++slot) {
            const d3 p0 = c[(slot + 1) & 3], p1 = c[(slot + 2) & 3], p2 = c[(slot + 3) & 3];
            d3 n = normalize(cross(sub(p1, p0), sub(p2, p0)));
            if (dot(n, sub(c[slot], p0)) > 0.0) n = mk(-n.x, -n.y, -n.z);
            const double d = dot(n, p0);
            const double denom = dot(n, dir);
            const double num = d - dot(n, o);
            if (fabs(denom) < 1e-15) {
                if (num < 0.0) hit = false;
            } else {
                const double tp = num / denom;
                if (denom > 0.0) t1 = tp < t1 ? tp : t1;
                else t0 = t0 < tp ? tp : t0;
                if (t0 > t1) hit = false;
            }
        }
        if (hit && t1 - t0 > 1e-12) {
            const unsigned long long k = atomicAdd(count, 1ull);
            if (k < cap) {
                tv_segment s;
                s.cell = static_cast<uint32_t>(t), s.pad = 0, s.t_enter = t0, s.t_exit = t1;
                out[k] = s;
            }
        }
    }
}

struct Buf {
    void* p = nullptr;
    ~Buf() {
        if (p) cudaFree(p);
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

#define VK(x, what)                       \
    do {                                  \
        int rc_ = cuda_status((x), what); \
        if (rc_) return rc_;              \
    } while (0)

inline unsigned nb(uint64_t n) { return static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, 148ull * 16)); }

// stable sort of perm by key (perm and key in/out via double buffers)
int stable_sort(uint32_t*& key, uint32_t*& key_alt, uint32_t*& perm, uint32_t*& perm_alt, uint64_t n, Buf& temp,
                size_t& temp_bytes) {
    cub::DoubleBuffer<uint32_t> k(key, key_alt), v(perm, perm_alt);
    size_t need = 0;
    VK(cub::DeviceRadixSort::SortPairs(nullptr, need, k, v, static_cast<int>(n)), "sort sizing");
    if (need > temp_bytes) {
        if (temp.p) cudaFree(temp.p);
        temp.p = nullptr;
        VK(cudaMalloc(&temp.p, need), "sort temp");
        temp_bytes = need;
    }
    VK(cub::DeviceRadixSort::SortPairs(temp.p, temp_bytes, k, v, static_cast<int>(n)), "radix sort");
    key = k.Current(), key_alt = k.Alternate(), perm = v.Current(), perm_alt = v.Alternate();
    return TV_OK;
}

}  // namespace
}  // namespace tvb

using namespace tvb;

extern "C" {

int tv_grid_validate(const tv_grid* h, tv_validation_report* out) {
    if (!h || !out) return set_error(TV_ERR_ARG, "null argument");
    std::memset(out, 0, sizeof(*out));
    out->ok = 1;
    std::string first;
    auto fail = [&](const std::string& m) {
        if (out->ok) out->ok = 0, first = m;
    };
    auto finish = [&]() {
        std::snprintf(out->first_violation, sizeof(out->first_violation), "%s", first.c_str());
        return TV_OK;
    };
    const DeviceGrid& g = h->g;
    int rc = use_device(g.device);
    if (rc) return rc;
    const uint64_t nt = g.n_tets, nv = g.n_vertices;
    if (nt < 24) {  // tet_grid.cpp:483-486
        fail("fewer than 24 tets");
        return finish();
    }
    // A: root table (tet_grid.cpp:487-493)
    for (int i = 0; i < 24; ++i) {
        tv_tet r{};
        const bool in = g.roots[i] < nt;
        if (in) VK(cudaMemcpy(&r, g.tets + g.roots[i], sizeof(r), cudaMemcpyDeviceToHost), "D2H");
        if (!in || r.level != 0 || r.parent != kNone) {
            fail("root table is inconsistent");
            break;
        }
    }
    Buf accb;
    VK(cudaMalloc(&accb.p, sizeof(Acc) + 2 * sizeof(unsigned long long)), "alloc");
    Acc* acc = accb.as<Acc>();
    auto* vflags = reinterpret_cast<unsigned long long*>(acc + 1);  // [duplicate, coordinate range]
    {
        Acc init;
        std::memset(&init, 0, sizeof(init));
        init.fail_d = init.vid = init.fail_g1 = init.fail_g2 = init.fail_h = kNoFail;
        VK(cudaMemcpy(acc, &init, sizeof(init), cudaMemcpyHostToDevice), "H2D");
        const unsigned long long f2[2] = {kNoFail, kNoFail};
        VK(cudaMemcpy(vflags, f2, sizeof(f2), cudaMemcpyHostToDevice), "H2D");
    }
    // B, C: duplicate vertices (vert_lookup_ size), coordinate range (tet_grid.cpp:494-500)
    Buf temp;
    size_t temp_bytes = 0;
    {
        Buf p0, p1, q0, q1;
        VK(cudaMalloc(&p0.p, nv * 4), "alloc");
        VK(cudaMalloc(&p1.p, nv * 4), "alloc");
        VK(cudaMalloc(&q0.p, nv * 4), "alloc");
        VK(cudaMalloc(&q1.p, nv * 4), "alloc");
        uint32_t *perm = p0.as<uint32_t>(), *perm_alt = p1.as<uint32_t>(), *key = q0.as<uint32_t>(),
                 *key_alt = q1.as<uint32_t>();
        iota_kernel<<<nb(nv), 256>>>(perm, nv);
        for (int k = 2; k >= 0; --k) {  // z, then y, then x: stable -> sorted by (x, y, z)
            vkey_kernel<<<nb(nv), 256>>>(g.verts, perm, nv, k, key, k == 2 ? vflags + 1 : nullptr);
            VK(cudaGetLastError(), "vkey_kernel");
            if ((rc = stable_sort(key, key_alt, perm, perm_alt, nv, temp, temp_bytes))) return rc;
        }
        vdup_kernel<<<nb(nv), 256>>>(g.verts, perm, nv, vflags);
        VK(cudaGetLastError(), "vdup_kernel");
        unsigned long long hf[2];
        VK(cudaMemcpy(hf, vflags, sizeof(hf), cudaMemcpyDeviceToHost), "D2H");
        if (hf[0] != kNoFail) fail("duplicate vertices in the pool");
        if (hf[1] != kNoFail) fail("vertex coordinate out of range");
    }
    // D: tree structure, orientation, exact volume (tet_grid.cpp:502-531)
    tets_kernel<<<nb(nt), 256>>>(g.tets, g.verts, nt, nv, g.max_level, acc);
    VK(cudaGetLastError(), "tets_kernel");
    Acc a;
    VK(cudaMemcpy(&a, acc, sizeof(a), cudaMemcpyDeviceToHost), "D2H");
    if (a.fail_d != kNoFail) fail(kMsgD[a.fail_d & 15u]);
    if (a.vid != kNoFail) return finish();  // "vertex id out of range" returns the report as is
    out->leaf_count = a.leaves;
    if (a.leaves != g.n_leaves) fail("cached leaf count is stale");
    const unsigned __int128 total = (static_cast<unsigned __int128>(a.vol_hi) << 64) | a.vol_lo;
    if (total != (static_cast<unsigned __int128>(6) << 72))  // the signed sum, mod 2^128
        fail("leaf volumes do not sum to the cube volume exactly");

    // G1 + G2: conformity and adjacency by exhaustive face matching (tet_grid.cpp:533-594)
    const uint64_t nl = a.leaves, nf = 4 * nl;
    Buf lpos, ltet, kb0, kb1, kb2, rp0, rp1, key0, key1;
    VK(cudaMalloc(&lpos.p, nt * 4), "alloc");
    VK(cudaMalloc(&ltet.p, (nl ? nl : 1) * 4), "alloc");
    {
        // leaf position = exclusive scan of is_leaf (tet order); position -> TetId
        Buf flag;
        VK(cudaMalloc(&flag.p, nt * 4), "alloc");
        leaf_flag_kernel<<<nb(nt), 256>>>(g.tets, nt, flag.as<uint32_t>());
        size_t need = 0;
        VK(cub::DeviceScan::ExclusiveSum(nullptr, need, flag.as<uint32_t>(), lpos.as<uint32_t>(), static_cast<int>(nt)),
           "scan sizing");
        Buf st;
        VK(cudaMalloc(&st.p, need), "alloc");
        VK(cub::DeviceScan::ExclusiveSum(st.p, need, flag.as<uint32_t>(), lpos.as<uint32_t>(), static_cast<int>(nt)),
           "scan");
        Buf nsel;
        VK(cudaMalloc(&nsel.p, 8), "alloc");
        Buf it;
        VK(cudaMalloc(&it.p, nt * 4), "alloc");
        iota_kernel<<<nb(nt), 256>>>(it.as<uint32_t>(), nt);
        size_t need2 = 0;
        VK(cub::DeviceSelect::Flagged(nullptr, need2, it.as<uint32_t>(), flag.as<uint32_t>(), ltet.as<uint32_t>(),
                                      static_cast<int*>(nsel.p), static_cast<int>(nt)),
           "select sizing");
        Buf st2;
        VK(cudaMalloc(&st2.p, need2), "alloc");
        VK(cub::DeviceSelect::Flagged(st2.p, need2, it.as<uint32_t>(), flag.as<uint32_t>(), ltet.as<uint32_t>(),
                                      static_cast<int*>(nsel.p), static_cast<int>(nt)),
           "select");
    }
    VK(cudaMalloc(&kb0.p, (nf ? nf : 1) * 4), "alloc");
    VK(cudaMalloc(&kb1.p, (nf ? nf : 1) * 4), "alloc");
    VK(cudaMalloc(&kb2.p, (nf ? nf : 1) * 4), "alloc");
    VK(cudaMalloc(&rp0.p, (nf ? nf : 1) * 4), "alloc");
    VK(cudaMalloc(&rp1.p, (nf ? nf : 1) * 4), "alloc");
    VK(cudaMalloc(&key0.p, (nf ? nf : 1) * 4), "alloc");
    VK(cudaMalloc(&key1.p, (nf ? nf : 1) * 4), "alloc");
    faces_kernel<<<nb(nt), 256>>>(g.tets, nt, lpos.as<uint32_t>(), kb0.as<uint32_t>(), kb1.as<uint32_t>(),
                                  kb2.as<uint32_t>(), rp0.as<uint32_t>(), acc);
    VK(cudaGetLastError(), "faces_kernel");
    // records are generated in (tet, slot) order; stable sorts by k2, k1, k0 -> (key, tet, slot)
    uint32_t *perm = rp0.as<uint32_t>(), *perm_alt = rp1.as<uint32_t>(), *key = key0.as<uint32_t>(),
             *key_alt = key1.as<uint32_t>();
    const uint32_t* kk[3] = {kb0.as<uint32_t>(), kb1.as<uint32_t>(), kb2.as<uint32_t>()};
    for (int k = 2; k >= 0 && nf; --k) {
        fkey_kernel<<<nb(nf), 256>>>(kk[k], perm, nf, key);
        VK(cudaGetLastError(), "fkey_kernel");
        if ((rc = stable_sort(key, key_alt, perm, perm_alt, nf, temp, temp_bytes))) return rc;
    }
    if (nf) {
        groups_kernel<<<nb(nf), 256>>>(g.tets, g.verts, kk[0], kk[1], kk[2], perm, ltet.as<uint32_t>(), nf, acc);
        VK(cudaGetLastError(), "groups_kernel");
    }
    VK(cudaMemcpy(&a, acc, sizeof(a), cudaMemcpyDeviceToHost), "D2H");
    if (a.fail_g1 != kNoFail) fail("leaf neighbor is not a leaf");
    if (a.fail_g2 != kNoFail) fail(kMsgG2[a.fail_g2 & 15u]);
    out->boundary_faces = a.boundary;
    out->interior_faces = a.interior;

    // H: stored normals re-derived from geometry, only while still ok (tet_grid.cpp:596-615)
    if (out->ok) {
        normals_kernel<<<nb(nt), 256>>>(g.tets, g.verts, nt, acc);
        VK(cudaGetLastError(), "normals_kernel");
        VK(cudaMemcpy(&a, acc, sizeof(a), cudaMemcpyDeviceToHost), "D2H");
        if (a.fail_h != kNoFail)
            fail((a.fail_h & 15u) ? "face normal not in the canonical table"
                                  : "stored face normal id does not match geometry");
    }
    return finish();
}

// cmd_validate's spot-check rays, generated on the host exactly as
// cli.cpp:552-569 does (RngStream(seed, "validate", i), sphere_dir, glibc cos/sin)
int tv_validate_spot_rays(uint64_t seed, int32_t n, tv_ray* out) {
    if (n < 0 || (n && !out)) return set_error(TV_ERR_ARG, "bad argument");
    for (int32_t i = 0; i < n; ++i) {
        Rng rng;
        rng.init(seed, 0x76616c6964617465ull, static_cast<uint64_t>(i));
        const double u1 = rng.next(), u2 = rng.next();
        const double z = 1.0 - 2.0 * u1;
        const double r = std::sqrt(dmax(0.0, 1.0 - z * z));
        const double phi = 2.0 * 3.14159265358979323846 * u2;
        const d3 origin = add(mk(0.5, 0.5, 0.5), mul(mk(r * std::cos(phi), r * std::sin(phi), z), 2.0));
        const double tx = 0.25 + 0.5 * rng.next(), ty = 0.25 + 0.5 * rng.next(), tz = 0.25 + 0.5 * rng.next();
        const d3 dir = normalize(sub(mk(tx, ty, tz), origin));
        tv_ray& o = out[i];
        o.origin[0] = origin.x, o.origin[1] = origin.y, o.origin[2] = origin.z;
        o.dir[0] = dir.x, o.dir[1] = dir.y, o.dir[2] = dir.z;
        o.t_min = 0.0, o.t_max = HUGE_VAL;
    }
    return TV_OK;
}

// cmd_validate's spot checks (cli.cpp:565-595): `rays` as 8 doubles each (origin,
// dir, t_min, t_max, generated on the host by the caller); per ray, our
// march_segments against the brute-force traverser, both without segments of
// length <= 1e-12: same cells, lengths within 1e-9.
int tv_validate_rays(const tv_grid* h, const tv_ray* rays, int32_t n, int32_t* failures, int32_t* first_failed) {
    if (!h || (!rays && n) || !failures || !first_failed) return set_error(TV_ERR_ARG, "null argument");
    *failures = 0, *first_failed = -1;
    const DeviceGrid& g = h->g;
    int rc = use_device(g.device);
    if (rc) return rc;
    std::vector<uint64_t> off(n + 1);
    uint64_t total = 0, deg = 0;
    if ((rc = tv_march_segments(h, rays, n, nullptr, off.data(), 0, &total, &deg))) return rc;
    std::vector<tv_segment> got(total);
    if ((rc = tv_march_segments(h, rays, n, got.data(), off.data(), total, &total, &deg))) return rc;
    uint64_t cap = 1 << 16;
    Buf seg, cnt;
    VK(cudaMalloc(&seg.p, cap * sizeof(tv_segment)), "alloc");
    VK(cudaMalloc(&cnt.p, 8), "alloc");
    std::vector<tv_segment> want;
    for (int i = 0; i < n; ++i) {
        const tv_ray& r = rays[i];
        for (int pass = 0; pass < 2; ++pass) {
            VK(cudaMemset(cnt.p, 0, 8), "memset");
            brute_kernel<<<nb(g.n_tets), 256>>>(g.tets, g.verts, g.n_tets, mk(r.origin[0], r.origin[1], r.origin[2]),
                                                mk(r.dir[0], r.dir[1], r.dir[2]), r.t_min, r.t_max,
                                                seg.as<tv_segment>(), cnt.as<unsigned long long>(), cap);
            VK(cudaGetLastError(), "brute_kernel");
            unsigned long long c = 0;
            VK(cudaMemcpy(&c, cnt.p, 8, cudaMemcpyDeviceToHost), "D2H");
            if (c <= cap) {
                want.resize(c);
                VK(cudaMemcpy(want.data(), seg.p, c * sizeof(tv_segment), cudaMemcpyDeviceToHost), "D2H");
                break;
            }
            cap = c;  // grow once and rerun
            if (seg.p) cudaFree(seg.p);
            seg.p = nullptr;
            VK(cudaMalloc(&seg.p, cap * sizeof(tv_segment)), "alloc");
        }
        // leaf_ids() order, then std::sort by t_enter (tet_grid.cpp:677-696)
        std::sort(want.begin(), want.end(), [](const tv_segment& x, const tv_segment& y) { return x.cell < y.cell; });
        std::sort(want.begin(), want.end(),
                  [](const tv_segment& x, const tv_segment& y) { return x.t_enter < y.t_enter; });
        std::vector<tv_segment> mine;
        for (uint64_t k = off[i]; k < off[i + 1]; ++k)
            if (got[k].t_exit - got[k].t_enter > 1e-12) mine.push_back(got[k]);
        bool ok = mine.size() == want.size();
        for (size_t k = 0; ok && k < mine.size(); ++k)
            ok = mine[k].cell == want[k].cell &&
                 std::fabs((mine[k].t_exit - mine[k].t_enter) - (want[k].t_exit - want[k].t_enter)) <= 1e-9;
        if (!ok) {
            ++*failures;
            if (*first_failed < 0) *first_failed = i;
        }
    }
    return TV_OK;
}

}  // extern "C"
