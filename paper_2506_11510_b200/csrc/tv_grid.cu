// Device grid finalize: from the reference pools (vertices, 68-byte Tet records,
// roots) resident in HBM, build the traversal layout:
//   * leaves renumbered along a Morton curve of their centroids (spatially
//     adjacent leaves share cache lines; rays from neighbouring pixels hit the
//     same lines), 64-byte LeafRec each;
//   * internal nodes compacted to 64-byte NodeRecs with the exact bisection
//     plane normal precomputed (tet_grid.cpp:453-470);
//   * the 24 roots' data for the root scan (tet_grid.cpp:435-451) in the
//     kernel parameter block.
// The reference TetIds survive in leaf2tet (and in the kept pools), so parity
// outputs speak reference ids.
#include <cub/cub.cuh>

#include <cstring>
#include <cstdlib>
#include <vector>

#include "tv_trace.cuh"

namespace tvb {

namespace {

// slot pairs (0,1),(0,2),(0,3),(1,2),(1,3),(2,3) (tet_grid.cpp:289)
__host__ __device__ __forceinline__ int ep0(int e) { return e < 3 ? 0 : (e < 5 ? 1 : 2); }
__host__ __device__ __forceinline__ int ep1(int e) { return e < 3 ? e + 1 : (e < 5 ? e - 1 : 3); }

__device__ __forceinline__ uint64_t spread21(uint64_t v) {
    v &= 0x1fffffull;
    v = (v | v << 32) & 0x1f00000000ffffull;
    v = (v | v << 16) & 0x1f0000ff0000ffull;
    v = (v | v << 8) & 0x100f00f00f00f00full;
    v = (v | v << 4) & 0x10c30c30c30c30c3ull;
    v = (v | v << 2) & 0x1249249249249249ull;
    return v;
}

__global__ void keys_kernel(const tv_tet* __restrict__ tets, const uint4* __restrict__ verts, uint64_t n,
                            uint64_t* keys, uint32_t* ids, uint32_t* is_internal) {
    const uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (t >= n) return;
    const tv_tet& tt = tets[t];
    ids[t] = static_cast<uint32_t>(t);
    const bool leaf = tt.children[0] == kNone;
    is_internal[t] = leaf ? 0u : 1u;
    if (!leaf) {
        keys[t] = ~0ull;
        return;
    }
    uint64_t c[3] = {0, 0, 0};
    for (int k = 0; k < 4; ++k) {
        const uint4 q = verts[tt.verts[k]];
        c[0] += q.x, c[1] += q.y, c[2] += q.z;
    }
    // centroid*4 < 2^27; keep the top 21 bits per axis
    keys[t] = spread21(c[0] >> 6) | spread21(c[1] >> 6) << 1 | spread21(c[2] >> 6) << 2;
}

__global__ void tet2leaf_kernel(const uint32_t* __restrict__ order, uint64_t n_leaves, uint32_t* tet2leaf) {
    const uint64_t L = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (L < n_leaves) tet2leaf[order[L]] = static_cast<uint32_t>(L);
}

__device__ __forceinline__ uint32_t encode_child(uint32_t c, const tv_tet* tets, const uint32_t* tet2leaf,
                                                 const uint32_t* tet2node) {
    return tets[c].children[0] == kNone ? (kLeafBit | tet2leaf[c]) : tet2node[c];
}

__global__ void leaves_kernel(const tv_tet* __restrict__ tets, const uint32_t* __restrict__ order,
                              const uint32_t* __restrict__ tet2leaf, const uint4* __restrict__ verts,
                              uint64_t n_leaves, LeafRec* out, uint8_t* mask, int* max_depth) {
    const uint64_t L = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (L >= n_leaves) return;
    const tv_tet tt = tets[order[L]];
    LeafRec r;
    uint32_t codes = 0;
    for (int f = 0; f < 4; ++f) {
        const uint32_t nb = tt.neighbors[f];
        const uint32_t id = static_cast<uint32_t>(tt.normal_ids[f]) & 31u;
        r.w[f] = nbr_word(nb == kNone ? kNoLeaf : tet2leaf[nb], id);
        // exit_face reads vertex verts[(f+1)&3] of face f (tracer.cpp:152)
        const uint4 q = verts[tt.verts[(f + 1) & 3]];
        const uint32_t qq[3] = {q.x, q.y, q.z};
        uint32_t ai, aj;
        pos2_axes(id, ai, aj);
        r.w[4 + 2 * f] = __float_as_uint(static_cast<float>(qq[ai]) * 0x1.0p-24f);
        r.w[5 + 2 * f] = __float_as_uint(static_cast<float>(qq[aj]) * 0x1.0p-24f);
        // the sign of m1 rides in c1's (otherwise zero) sign bit; see exit_face_nbr
        if (pos2_code(id) & 16u) r.w[5 + 2 * f] |= 0x80000000u;
        codes |= pos2_code(id) << (6 * f);
    }
    r.w[12] = codes | (static_cast<uint32_t>(tt.mask & 7u) << 24);
    mask[L] = tt.mask;
    r.w[13] = __float_as_uint(tt.density);
    r.w[14] = __float_as_uint(tt.temperature);
    r.w[15] = __float_as_uint(tt.albedo);
    uint4* dst = reinterpret_cast<uint4*>(out + L);
    dst[0] = make_uint4(r.w[0], r.w[1], r.w[2], r.w[3]);
    dst[1] = make_uint4(r.w[4], r.w[5], r.w[6], r.w[7]);
    dst[2] = make_uint4(r.w[8], r.w[9], r.w[10], r.w[11]);
    dst[3] = make_uint4(r.w[12], r.w[13], r.w[14], r.w[15]);
    const unsigned act = __activemask();  // one atomic per warp
    const int lv = __reduce_max_sync(act, static_cast<int>(tt.level));
    if ((threadIdx.x & 31) == static_cast<unsigned>(__ffs(act) - 1)) atomicMax(max_depth, lv);
}

// HotRec of every leaf from its LeafRec (tv_internal.cuh). The eight plane-test
// coordinates q (integers, q / 2^24 = the f32 value) are split per axis into
// base + offset * 2^tz; a leaf whose values do not fit (offset > 7, base >=
// 2^18) sets *fail and the grid renders from the LeafRecs.
__global__ void hot_kernel(const LeafRec* __restrict__ leaves, uint64_t n_leaves, HotRec* out, int* fail) {
    const uint64_t L = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (L >= n_leaves) return;
    const LeafRec r = leaves[L];
    uint32_t q[8], ax[8];
    uint32_t mn[3] = {0xffffffffu, 0xffffffffu, 0xffffffffu};
    for (int f = 0; f < 4; ++f) {
        const uint32_t c = (r.w[12] >> (6 * f)) & 31u;
        q[2 * f] = static_cast<uint32_t>(__uint_as_float(r.w[4 + 2 * f]) * 16777216.0f);
        q[2 * f + 1] = static_cast<uint32_t>(__uint_as_float(r.w[5 + 2 * f] & 0x7fffffffu) * 16777216.0f);
        ax[2 * f] = (c & 1u) ? 1u : 0u;
        ax[2 * f + 1] = (c & 2u) ? 2u : 1u;
    }
    for (int k = 0; k < 8; ++k) mn[ax[k]] = min(mn[ax[k]], q[k]);
    for (int a = 0; a < 3; ++a)
        if (mn[a] == 0xffffffffu) mn[a] = 0;
    uint32_t D = 0;
    for (int k = 0; k < 8; ++k) D |= q[k] - mn[ax[k]];
    int tz = D ? __ffs(D) - 1 : 24;
    for (int a = 0; a < 3; ++a)
        if (mn[a]) tz = min(tz, __ffs(mn[a]) - 1);
    bool ok = true;
    uint32_t G = 0;
    for (int k = 0; k < 8; ++k) {
        const uint32_t o = (q[k] - mn[ax[k]]) >> tz;
        ok &= o <= 7u;
        G |= (o & 7u) << (3 * k);
    }
    for (int a = 0; a < 3; ++a) ok &= (mn[a] >> tz) < (1u << 18);
    HotRec h;
    h.w[0] = r.w[0], h.w[1] = r.w[1], h.w[2] = r.w[2], h.w[3] = r.w[3];
    h.w[4] = r.w[13];
    h.w[5] = (mn[0] >> tz) | ((G & 0xfffu) << 18);
    h.w[6] = (mn[1] >> tz) | ((G >> 12) << 18);
    h.w[7] = (mn[2] >> tz) | (static_cast<uint32_t>(tz) << 18);
    if (!ok) {
        atomicOr(fail, 1);
        for (int k = 0; k < 8; ++k) h.w[k] = 0;
    }
    uint4* dst = reinterpret_cast<uint4*>(out + L);
    dst[0] = make_uint4(h.w[0], h.w[1], h.w[2], h.w[3]);
    dst[1] = make_uint4(h.w[4], h.w[5], h.w[6], h.w[7]);
}

// tet_grid.cpp:288-330 (exact integer longest edge; ties towards smaller ids)
__device__ void refinement_slots(const tv_tet& tt, const uint4* verts, int& s0, int& s1) {
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

__global__ void nodes_kernel(const tv_tet* __restrict__ tets, const uint4* __restrict__ verts, uint64_t n_tets,
                             const uint32_t* __restrict__ tet2leaf, const uint32_t* __restrict__ tet2node,
                             NodeRec* out) {
    const uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (t >= n_tets) return;
    const tv_tet tt = tets[t];
    if (tt.children[0] == kNone) return;
    int s0, s1;
    refinement_slots(tt, verts, s0, s1);
    const uint32_t ca = tt.children[0];
    const d3 pm = vpos(verts[tets[ca].verts[s1]]);
    int oa = -1, ob = -1;
    for (int s = 0; s < 4; ++s)
        if (s != s0 && s != s1) {
            if (oa < 0) oa = s;
            else ob = s;
        }
    const d3 pa = vpos(verts[tt.verts[oa]]), pb = vpos(verts[tt.verts[ob]]);
    const d3 n = cross(sub(pa, pm), sub(pb, pm));
    const double sref = dot(n, sub(vpos(verts[tt.verts[s0]]), pm));
    NodeRec r;
    r.n[0] = n.x, r.n[1] = n.y, r.n[2] = n.z;
    r.pm[0] = pm.x, r.pm[1] = pm.y, r.pm[2] = pm.z;
    r.child[0] = encode_child(ca, tets, tet2leaf, tet2node);
    r.child[1] = encode_child(tt.children[1], tets, tet2leaf, tet2node);
    r.sref_pos = sref > 0.0 ? 1u : 0u;
    r.pad = 0;
    out[tet2node[t]] = r;
}

__global__ void roots_kernel(const tv_tet* __restrict__ tets, const uint4* __restrict__ verts, const uint32_t* roots,
                             const uint32_t* tet2leaf, const uint32_t* tet2node,
                             uint32_t* out /* 24 ptr, 24 nid, 96 vid, 24 outer-face masks */) {
    const int r = threadIdx.x;
    if (r >= 24) return;
    const tv_tet& tt = tets[roots[r]];
    out[r] = encode_child(roots[r], tets, tet2leaf, tet2node);
    out[24 + r] = tt.normal_ids[0] | tt.normal_ids[1] << 8 | tt.normal_ids[2] << 16 |
                  static_cast<uint32_t>(tt.normal_ids[3]) << 24;
    for (int k = 0; k < 4; ++k) out[48 + 4 * r + k] = tt.verts[k];
    // face f (opposite verts[f]) lies in a face of the unit cube when its three
    // vertices share a coordinate of 0 or 2^24
    uint32_t outer = 0;
    for (int f = 0; f < 4; ++f) {
        uint4 q[3];
        int m = 0;
        for (int k = 0; k < 4; ++k)
            if (k != f) q[m++] = verts[tt.verts[k]];
        for (int a = 0; a < 3; ++a) {
            const uint32_t c0 = a == 0 ? q[0].x : (a == 1 ? q[0].y : q[0].z);
            const uint32_t c1 = a == 0 ? q[1].x : (a == 1 ? q[1].y : q[1].z);
            const uint32_t c2 = a == 0 ? q[2].x : (a == 1 ? q[2].y : q[2].z);
            if (c0 == c1 && c1 == c2 && (c0 == 0u || c0 == (1u << 24))) outer |= 1u << f;
        }
    }
    out[144 + r] = outer;
}

template <class T>
int dalloc(T** p, uint64_t count, uint64_t& bytes) {
    const size_t b = static_cast<size_t>(count ? count : 1) * sizeof(T);
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), b);
    if (e != cudaSuccess) return set_error(TV_ERR_OOM, std::string("cudaMalloc failed: ") + cudaGetErrorString(e));
    bytes += b;
    return TV_OK;
}

inline unsigned blocks(uint64_t n, unsigned t) { return static_cast<unsigned>((n + t - 1) / t); }

}  // namespace

// The locate jump table (GridView::jump): for cube c of a res^3 grid over the
// unit cube, the deepest tree node whose tet contains all 8 corners of c
// strictly — the root test with locate's 1e-9 interior margin, each descent
// test with |dot(n, corner - pm)| > 1e-9 |n| on the same side for all corners —
// or kNone when no root does. Corners are exact dyadic (i / res), so the only
// rounding is in the dot products, ~1e-15 |n|: every point of the closed cube
// takes the same branch at each of these levels in the reference's descent
// (tet_grid.cpp:435-470), which is what lets locate start at the table's node.
__global__ void jump_kernel(GridView G, int res, uint32_t* jump) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t n = static_cast<uint32_t>(res) * res * res;
    if (c >= n) return;
    const int ix = static_cast<int>(c % res), iy = static_cast<int>((c / res) % res), iz = static_cast<int>(c / (res * res));
    d3 corner[8];
    for (int k = 0; k < 8; ++k)
        corner[k] = mk(static_cast<double>(ix + (k & 1)) / res, static_cast<double>(iy + ((k >> 1) & 1)) / res,
                       static_cast<double>(iz + (k >> 2)) / res);
    uint32_t cur = kNone;
    for (int r = 0; r < 24 && cur == kNone; ++r) {
        // locate's root fast path, for every corner (the cube's points lie in
        // the convex hull of its corners, and the violations are convex)
        bool inside = true;
        for (int k = 0; k < 8 && inside; ++k) {
            double vi, vo;
            root_violation2(G, r, corner[k], vi, vo);
            inside = vi <= -1e-9 && vo <= 1e-12;
        }
        if (inside) cur = G.root_ptr[r];
    }
    if (cur == kNone) {
        jump[c] = kNone;
        return;
    }
    while (!(cur & kLeafBit)) {
        const NodeRec& nd = G.nodes[cur];
        const d3 nn = mk(nd.n[0], nd.n[1], nd.n[2]);
        const d3 pm = mk(nd.pm[0], nd.pm[1], nd.pm[2]);
        const double margin = 1e-9 * sqrt(dot(nn, nn));
        bool all_a = true, all_b = true;
        for (int k = 0; k < 8; ++k) {
            const double sp = dot(nn, sub(corner[k], pm));
            // child A holds sp >= 0 (sref_pos) or sp <= 0; demand a strict margin
            const bool a = nd.sref_pos ? sp > margin : sp < -margin;
            const bool b = nd.sref_pos ? sp < -margin : sp > margin;
            all_a &= a;
            all_b &= b;
        }
        if (all_a) cur = nd.child[0];
        else if (all_b) cur = nd.child[1];
        else break;
    }
    jump[c] = cur;
}

int finalize_grid(DeviceGrid& g, cudaStream_t st) {
    const uint64_t nt = g.n_tets;
    int rc;
    uint64_t scratch_bytes = 0;
    uint64_t *keys = nullptr, *keys_sorted = nullptr;
    uint32_t *ids = nullptr, *order = nullptr, *is_int = nullptr, *tet2node = nullptr, *tet2leaf = nullptr,
             *rootbuf = nullptr, *d_roots = nullptr;
    int* d_depth = nullptr;
    void* temp = nullptr;
    size_t temp_bytes = 0, t1 = 0, t2 = 0;
    std::vector<uint32_t> hroot(24 + 24 + 96 + 24);

    auto cleanup = [&]() {
        cudaFree(keys), cudaFree(keys_sorted), cudaFree(ids), cudaFree(order), cudaFree(is_int);
        cudaFree(tet2node), cudaFree(tet2leaf), cudaFree(rootbuf), cudaFree(d_roots), cudaFree(d_depth);
        cudaFree(temp);
    };
#define TRY(x)            \
    do {                  \
        if ((rc = (x))) { \
            cleanup();    \
            return rc;    \
        }                 \
    } while (0)
#define CK(x, what) TRY(cuda_status((x), what))

    if (g.n_leaves >= kNoLeaf) {
        return set_error(TV_ERR_GRID, "grid has " + std::to_string(g.n_leaves) +
                                          " leaves; the traversal layout holds at most " +
                                          std::to_string(kNoLeaf - 1));
    }
    TRY(dalloc(&keys, nt, scratch_bytes));
    TRY(dalloc(&keys_sorted, nt, scratch_bytes));
    TRY(dalloc(&ids, nt, scratch_bytes));
    TRY(dalloc(&order, nt, scratch_bytes));
    TRY(dalloc(&is_int, nt, scratch_bytes));
    TRY(dalloc(&tet2node, nt, scratch_bytes));
    TRY(dalloc(&tet2leaf, nt, scratch_bytes));
    TRY(dalloc(&rootbuf, 24 + 24 + 96 + 24, scratch_bytes));
    TRY(dalloc(&d_roots, 24, scratch_bytes));
    TRY(dalloc(&d_depth, 1, scratch_bytes));

    keys_kernel<<<blocks(nt, 256), 256, 0, st>>>(g.tets, g.verts, nt, keys, ids, is_int);
    CK(cudaGetLastError(), "keys_kernel");
    CK(cub::DeviceRadixSort::SortPairs(nullptr, t1, keys, keys_sorted, ids, order, static_cast<int>(nt), 0, 64, st),
       "sort sizing");
    CK(cub::DeviceScan::ExclusiveSum(nullptr, t2, is_int, tet2node, static_cast<int>(nt), st), "scan sizing");
    temp_bytes = t1 > t2 ? t1 : t2;
    CK(cudaMalloc(&temp, temp_bytes), "cudaMalloc temp");
    CK(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys, keys_sorted, ids, order, static_cast<int>(nt), 0, 64,
                                       st),
       "radix sort");
    CK(cub::DeviceScan::ExclusiveSum(temp, temp_bytes, is_int, tet2node, static_cast<int>(nt), st), "scan");
    CK(cudaMemsetAsync(tet2leaf, 0xff, nt * sizeof(uint32_t), st), "memset");
    tet2leaf_kernel<<<blocks(g.n_leaves, 256), 256, 0, st>>>(order, g.n_leaves, tet2leaf);
    CK(cudaGetLastError(), "tet2leaf_kernel");

    TRY(dalloc(&g.leaves, g.n_leaves, g.bytes));
    TRY(dalloc(&g.nodes, g.n_internal, g.bytes));
    TRY(dalloc(&g.leaf2tet, g.n_leaves, g.bytes));
    TRY(dalloc(&g.mask, g.n_leaves, g.bytes));
    CK(cudaMemcpyAsync(g.leaf2tet, order, g.n_leaves * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st), "leaf2tet");
    CK(cudaMemsetAsync(d_depth, 0, sizeof(int), st), "memset");
    leaves_kernel<<<blocks(g.n_leaves, 256), 256, 0, st>>>(g.tets, order, tet2leaf, g.verts, g.n_leaves, g.leaves,
                                                            g.mask, d_depth);
    CK(cudaGetLastError(), "leaves_kernel");
    nodes_kernel<<<blocks(nt, 256), 256, 0, st>>>(g.tets, g.verts, nt, tet2leaf, tet2node, g.nodes);
    CK(cudaGetLastError(), "nodes_kernel");
    CK(cudaMemcpyAsync(d_roots, g.roots, sizeof(g.roots), cudaMemcpyHostToDevice, st), "roots H2D");
    roots_kernel<<<1, 32, 0, st>>>(g.tets, g.verts, d_roots, tet2leaf, tet2node, rootbuf);
    CK(cudaGetLastError(), "roots_kernel");
    CK(cudaMemcpyAsync(hroot.data(), rootbuf, hroot.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost, st),
       "roots D2H");
    int depth = 0;
    CK(cudaMemcpyAsync(&depth, d_depth, sizeof(int), cudaMemcpyDeviceToHost, st), "depth D2H");
    CK(cudaStreamSynchronize(st), "finalize sync");
    g.max_depth = depth;

    GridView& v = g.view;
    v.leaves = g.leaves;
    v.nodes = g.nodes;
    v.verts = g.verts;
    v.leaf2tet = g.leaf2tet;
    v.mask = g.mask;
    for (int r = 0; r < 24; ++r) {
        v.root_ptr[r] = hroot[r];
        v.root_nid[r] = hroot[24 + r];
        for (int k = 0; k < 4; ++k) v.root_vid[r][k] = hroot[48 + 4 * r + k];
        v.root_outer[r] = hroot[144 + r];
    }
    v.n_leaves = static_cast<uint32_t>(g.n_leaves);
    v.n_nodes = static_cast<uint32_t>(g.n_internal);
    v.jump = nullptr;
    v.jump_res = 0;
    v.hot = nullptr;
    v.code_lut = 0;
    for (uint32_t k = 0; k < 9; ++k) v.code_lut |= static_cast<uint64_t>(pos2_code(2 * k)) << (5 * k);
    {
        // TV_HOT=1: 32-B hot records, one load per trace step. Measured slower
        // on B200 (C2 frame 61.3 -> 70.4 ms): decoding the coordinates costs
        // more issue slots than the halved L1 wavefronts save; off by default
        const char* e = std::getenv("TV_HOT");
        if (e && std::atoi(e) && g.n_leaves) {
            TRY(dalloc(&g.hot, g.n_leaves, g.bytes));
            CK(cudaMemsetAsync(d_depth, 0, sizeof(int), st), "hot flag");
            hot_kernel<<<blocks(g.n_leaves, 256), 256, 0, st>>>(g.leaves, g.n_leaves, g.hot, d_depth);
            CK(cudaGetLastError(), "hot_kernel");
            int fail = 0;
            CK(cudaMemcpyAsync(&fail, d_depth, sizeof(int), cudaMemcpyDeviceToHost, st), "hot flag D2H");
            CK(cudaStreamSynchronize(st), "hot records");
            if (fail) {
                cudaFree(g.hot);
                g.hot = nullptr;
                g.bytes -= g.n_leaves * sizeof(HotRec);
            }
            v.hot = g.hot;
        }
    }
    {
        // TV_JUMP_RES: cubes per axis of the locate jump table (0 = none);
        // 128^3 entries = 8 MB
        const char* e = std::getenv("TV_JUMP_RES");
        const int res = e && *e ? std::atoi(e) : 128;
        if (res > 0 && res <= 512) {
            const uint32_t n = static_cast<uint32_t>(res) * res * res;
            TRY(dalloc(&g.jump, n, g.bytes));
            jump_kernel<<<blocks(n, 128), 128, 0, st>>>(v, res, g.jump);
            CK(cudaGetLastError(), "jump_kernel");
            CK(cudaStreamSynchronize(st), "jump table");
            v.jump = g.jump;
            v.jump_res = res;
        }
    }
    cleanup();
    return TV_OK;
#undef CK
#undef TRY
}

void free_grid(DeviceGrid& g) {
    cudaFree(g.tets);
    cudaFree(g.verts);
    cudaFree(g.leaves);
    cudaFree(g.nodes);
    cudaFree(g.leaf2tet);
    cudaFree(g.mask);
    cudaFree(g.jump);
    cudaFree(g.hot);
    g.hot = nullptr;
    g.jump = nullptr;
    g.mask = nullptr;
    g.tets = nullptr;
    g.verts = nullptr;
    g.leaves = nullptr;
    g.nodes = nullptr;
    g.leaf2tet = nullptr;
}

}  // namespace tvb
