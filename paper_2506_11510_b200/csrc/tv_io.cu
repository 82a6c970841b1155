// .tgrid I/O: the reference's TGRD v1 grid file (save_grid / load_grid,
// builder.cpp:184-293), packed and unpacked on the device so a 100M-tet grid
// never takes a per-tet host loop.
//
// File layout (little endian, no padding):
//   "TGRD" u32 version=1
//   u64 n_vertices, then per vertex u32 q[3]                        (12 B)
//   u64 n_tets, then per tet                                        (90 B)
//     u32 verts[4], u8 level, u64 children[2], u64 parent,
//     u64 neighbors[4], u8 normal_ids[4], u8 mask, f32 density,
//     f32 temperature, f32 albedo            (ids: kNoTet <-> 2^64 - 1)
//   u64 roots[24]
// Loading applies load_grid's checks in its order and reports the first
// failing record with the reference's FormatError message (TV_ERR_FORMAT).
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>

#include "tv_trace.cuh"

namespace tvb {
namespace {

constexpr uint64_t kTetBytes = 90;
constexpr uint64_t kVertBytes = 12;
constexpr uint64_t kSentinel = ~0ull;
constexpr uint64_t kChunkBytes = 64ull << 20;  // pinned staging buffer

// load_grid's per-record checks, in the order it makes them (builder.cpp:262-285)
enum : uint32_t {
    kOk = 0,
    kVertId = 1,
    kTetId = 2,
    kNormalId = 3,
    kChildId = 4,
    kParentId = 5,
    kNeighborId = 6,
};
const char* const kMsg[] = {"", "vertex id out of range", "tet id out of range", "face normal id out of range",
                            "child id out of range", "parent id out of range", "neighbor id out of range"};

__device__ __forceinline__ void put_bytes(uint8_t* p, uint64_t v, int n) {
    for (int k = 0; k < n; ++k) p[k] = static_cast<uint8_t>(v >> (8 * k));
}
__device__ __forceinline__ uint64_t get_bytes(const uint8_t* p, int n) {
    uint64_t v = 0;
    for (int k = 0; k < n; ++k) v |= static_cast<uint64_t>(p[k]) << (8 * k);
    return v;
}
__device__ __forceinline__ uint64_t id_out(uint32_t id) { return id == kNone ? kSentinel : id; }

__global__ void pack_verts_kernel(const uint4* __restrict__ v, uint64_t first, uint64_t n, uint8_t* out) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const uint4 q = v[first + i];
    uint8_t* p = out + i * kVertBytes;
    put_bytes(p, q.x, 4), put_bytes(p + 4, q.y, 4), put_bytes(p + 8, q.z, 4);
}

// builder.cpp:219-232
__global__ void pack_tets_kernel(const tv_tet* __restrict__ tets, uint64_t first, uint64_t n, uint8_t* out) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const tv_tet t = tets[first + i];
    uint8_t* p = out + i * kTetBytes;
    for (int k = 0; k < 4; ++k) put_bytes(p + 4 * k, t.verts[k], 4);
    p[16] = t.level;
    put_bytes(p + 17, id_out(t.children[0]), 8);
    put_bytes(p + 25, id_out(t.children[1]), 8);
    put_bytes(p + 33, id_out(t.parent), 8);
    for (int k = 0; k < 4; ++k) put_bytes(p + 41 + 8 * k, id_out(t.neighbors[k]), 8);
    for (int k = 0; k < 4; ++k) p[73 + k] = t.normal_ids[k];
    p[77] = t.mask;
    put_bytes(p + 78, __float_as_uint(t.density), 4);
    put_bytes(p + 82, __float_as_uint(t.temperature), 4);
    put_bytes(p + 86, __float_as_uint(t.albedo), 4);
}

// builder.cpp:249-257: the first vertex (in file order) with a coordinate > 2^24
__global__ void unpack_verts_kernel(const uint8_t* __restrict__ in, uint64_t first, uint64_t n, uint4* v,
                                    unsigned long long* bad) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const uint8_t* p = in + i * kVertBytes;
    const uint32_t x = static_cast<uint32_t>(get_bytes(p, 4)), y = static_cast<uint32_t>(get_bytes(p + 4, 4)),
                   z = static_cast<uint32_t>(get_bytes(p + 8, 4));
    constexpr uint32_t kOne = 1u << 24;
    if (x > kOne || y > kOne || z > kOne) atomicMin(bad, static_cast<unsigned long long>(first + i));
    v[first + i] = make_uint4(x, y, z, 0);
}

// id_in (builder.cpp:203-207): sentinel -> kNoTet, else must be < kNoTet
__device__ __forceinline__ bool id_in(uint64_t v, uint32_t& out) {
    if (v == kSentinel) {
        out = kNone;
        return true;
    }
    out = static_cast<uint32_t>(v);
    return v < kNone;
}

// builder.cpp:262-285; err = min over records of (record << 3 | first failing check)
__global__ void unpack_tets_kernel(const uint8_t* __restrict__ in, uint64_t first, uint64_t n, uint64_t n_verts,
                                   uint64_t n_tets, tv_tet* tets, unsigned long long* err,
                                   unsigned long long* leaves) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    bool leaf = false;
    if (i < n) {
        const uint8_t* p = in + i * kTetBytes;
        tv_tet t = {};
        uint32_t code = kOk;
        for (int k = 0; k < 4; ++k) {
            t.verts[k] = static_cast<uint32_t>(get_bytes(p + 4 * k, 4));
            if (!code && t.verts[k] >= n_verts) code = kVertId;
        }
        t.level = p[16];
        bool ok = id_in(get_bytes(p + 17, 8), t.children[0]);
        ok &= id_in(get_bytes(p + 25, 8), t.children[1]);
        ok &= id_in(get_bytes(p + 33, 8), t.parent);
        for (int k = 0; k < 4; ++k) ok &= id_in(get_bytes(p + 41 + 8 * k, 8), t.neighbors[k]);
        if (!code && !ok) code = kTetId;
        for (int k = 0; k < 4; ++k) {
            t.normal_ids[k] = p[73 + k];
            if (!code && t.normal_ids[k] >= 18) code = kNormalId;
        }
        t.mask = p[77];
        t.density = __uint_as_float(static_cast<uint32_t>(get_bytes(p + 78, 4)));
        t.temperature = __uint_as_float(static_cast<uint32_t>(get_bytes(p + 82, 4)));
        t.albedo = __uint_as_float(static_cast<uint32_t>(get_bytes(p + 86, 4)));
        if (!code)
            for (int k = 0; k < 2; ++k)
                if (t.children[k] != kNone && t.children[k] >= n_tets) code = kChildId;
        if (!code && t.parent != kNone && t.parent >= n_tets) code = kParentId;
        if (!code)
            for (int k = 0; k < 4; ++k)
                if (t.neighbors[k] != kNone && t.neighbors[k] >= n_tets) code = kNeighborId;
        if (code) atomicMin(err, static_cast<unsigned long long>(((first + i) << 3) | code));
        tets[first + i] = t;
        leaf = t.children[0] == kNone;
    }
    const unsigned nl = __popc(__ballot_sync(0xffffffffu, leaf));
    if ((threadIdx.x & 31) == 0 && nl) atomicAdd(leaves, static_cast<unsigned long long>(nl));
}

inline unsigned nblocks(uint64_t n) { return static_cast<unsigned>((n + 255) / 256); }

struct File {
    FILE* f = nullptr;
    ~File() {
        if (f) std::fclose(f);
    }
};

struct Pinned {
    uint8_t* p = nullptr;
    ~Pinned() {
        if (p) cudaFreeHost(p);
    }
};

struct Dev {
    void* p = nullptr;
    ~Dev() {
        if (p) cudaFree(p);
    }
};

#define IO_CK(x, what)                    \
    do {                                  \
        int rc_ = cuda_status((x), what); \
        if (rc_) return rc_;              \
    } while (0)

}  // namespace
}  // namespace tvb

using namespace tvb;

extern "C" {

int tv_grid_save(const tv_grid* h, const char* path) {
    if (!h || !path) return set_error(TV_ERR_ARG, "null argument");
    const DeviceGrid& g = h->g;
    int rc = use_device(g.device);
    if (rc) return rc;
    File f;
    f.f = std::fopen(path, "wb");
    if (!f.f) return set_error(TV_ERR_IO, std::string("cannot open for writing: ") + path);
    Pinned host;
    Dev dev;
    IO_CK(cudaMallocHost(&host.p, kChunkBytes), "cudaMallocHost");
    IO_CK(cudaMalloc(&dev.p, kChunkBytes), "cudaMalloc");
    auto* d = static_cast<uint8_t*>(dev.p);
    bool ok = std::fwrite("TGRD", 1, 4, f.f) == 4;
    const uint32_t version = 1;
    ok &= std::fwrite(&version, 4, 1, f.f) == 1;
    ok &= std::fwrite(&g.n_vertices, 8, 1, f.f) == 1;
    const uint64_t vchunk = kChunkBytes / kVertBytes;
    for (uint64_t s = 0; ok && s < g.n_vertices; s += vchunk) {
        const uint64_t n = std::min(vchunk, g.n_vertices - s);
        pack_verts_kernel<<<nblocks(n), 256>>>(g.verts, s, n, d);
        IO_CK(cudaGetLastError(), "pack_verts_kernel");
        IO_CK(cudaMemcpy(host.p, d, n * kVertBytes, cudaMemcpyDeviceToHost), "D2H");
        ok &= std::fwrite(host.p, kVertBytes, n, f.f) == n;
    }
    ok &= std::fwrite(&g.n_tets, 8, 1, f.f) == 1;
    const uint64_t tchunk = kChunkBytes / kTetBytes;
    for (uint64_t s = 0; ok && s < g.n_tets; s += tchunk) {
        const uint64_t n = std::min(tchunk, g.n_tets - s);
        pack_tets_kernel<<<nblocks(n), 256>>>(g.tets, s, n, d);
        IO_CK(cudaGetLastError(), "pack_tets_kernel");
        IO_CK(cudaMemcpy(host.p, d, n * kTetBytes, cudaMemcpyDeviceToHost), "D2H");
        ok &= std::fwrite(host.p, kTetBytes, n, f.f) == n;
    }
    for (int r = 0; ok && r < 24; ++r) {
        const uint64_t v = g.roots[r] == kNone ? kSentinel : g.roots[r];
        ok &= std::fwrite(&v, 8, 1, f.f) == 1;
    }
    ok &= std::fflush(f.f) == 0;
    if (!ok) return set_error(TV_ERR_IO, std::string("write failed: ") + path);
    return TV_OK;
}

int tv_grid_load(const char* path, int device, tv_grid** out) {
    if (!path || !out) return set_error(TV_ERR_ARG, "null argument");
    *out = nullptr;
    File f;
    f.f = std::fopen(path, "rb");
    if (!f.f) return set_error(TV_ERR_IO, std::string("cannot open: ") + path);
    const std::string eof = "unexpected end of grid file";
    char magic[4];
    if (std::fread(magic, 1, 4, f.f) != 4 || std::memcmp(magic, "TGRD", 4) != 0)
        return set_error(TV_ERR_FORMAT, std::string("not a TGRD file: ") + path);
    uint32_t version = 0;
    if (std::fread(&version, 4, 1, f.f) != 1) return set_error(TV_ERR_FORMAT, eof);
    if (version != 1u) return set_error(TV_ERR_FORMAT, "unsupported TGRD version");
    uint64_t n_verts = 0;
    if (std::fread(&n_verts, 8, 1, f.f) != 1) return set_error(TV_ERR_FORMAT, eof);
    if (n_verts < 8 || n_verts > (1ull << 32)) return set_error(TV_ERR_FORMAT, "bad vertex count");
    int rc = use_device(device);
    if (rc) return rc;

    auto h = std::make_unique<tv_grid>();
    DeviceGrid& g = h->g;
    g.device = device;
    g.max_level = 48;  // load_grid assembles with kLevelCap (builder.cpp:292)
    struct Guard {
        DeviceGrid* g;
        ~Guard() {
            if (g) free_grid(*g);
        }
    } guard{&g};
    Pinned host;
    Dev dev, flags;
    IO_CK(cudaMallocHost(&host.p, kChunkBytes), "cudaMallocHost");
    IO_CK(cudaMalloc(&dev.p, kChunkBytes), "cudaMalloc");
    IO_CK(cudaMalloc(&flags.p, 3 * sizeof(unsigned long long)), "cudaMalloc");
    auto* d = static_cast<uint8_t*>(dev.p);
    auto* fl = static_cast<unsigned long long*>(flags.p);  // [bad vertex, bad tet record, leaf count]
    const unsigned long long init[3] = {~0ull, ~0ull, 0ull};
    IO_CK(cudaMemcpy(fl, init, sizeof(init), cudaMemcpyHostToDevice), "H2D");
    IO_CK(cudaMalloc(&g.verts, n_verts * sizeof(uint4)), "grid alloc");
    g.n_vertices = n_verts;
    g.bytes = n_verts * sizeof(uint4);

    // vertices (builder.cpp:247-257): a short read after valid records -> eof
    const uint64_t vchunk = kChunkBytes / kVertBytes;
    unsigned long long hf[3];
    for (uint64_t s = 0; s < n_verts; s += vchunk) {
        const uint64_t want = std::min(vchunk, n_verts - s);
        const uint64_t got = std::fread(host.p, kVertBytes, want, f.f);
        if (got) {
            IO_CK(cudaMemcpy(d, host.p, got * kVertBytes, cudaMemcpyHostToDevice), "H2D");
            unpack_verts_kernel<<<nblocks(got), 256>>>(d, s, got, g.verts, fl);
            IO_CK(cudaGetLastError(), "unpack_verts_kernel");
        }
        IO_CK(cudaMemcpy(hf, fl, sizeof(hf), cudaMemcpyDeviceToHost), "D2H");
        if (hf[0] != ~0ull) return set_error(TV_ERR_FORMAT, "vertex coordinate out of range");
        if (got != want) return set_error(TV_ERR_FORMAT, eof);
    }

    uint64_t n_tets = 0;
    if (std::fread(&n_tets, 8, 1, f.f) != 1) return set_error(TV_ERR_FORMAT, eof);
    if (n_tets < 24 || n_tets > (1ull << 32)) return set_error(TV_ERR_FORMAT, "bad tet count");
    if (n_tets >= (1ull << 31)) return set_error(TV_ERR_GRID, "tet count exceeds the device layout (2^31)");
    IO_CK(cudaMalloc(&g.tets, n_tets * sizeof(tv_tet)), "grid alloc");
    g.n_tets = n_tets;
    g.bytes += n_tets * sizeof(tv_tet);
    const uint64_t tchunk = kChunkBytes / kTetBytes;
    for (uint64_t s = 0; s < n_tets; s += tchunk) {
        const uint64_t want = std::min(tchunk, n_tets - s);
        const uint64_t got = std::fread(host.p, kTetBytes, want, f.f);
        if (got) {
            IO_CK(cudaMemcpy(d, host.p, got * kTetBytes, cudaMemcpyHostToDevice), "H2D");
            unpack_tets_kernel<<<nblocks(got), 256>>>(d, s, got, n_verts, n_tets, g.tets, fl + 1, fl + 2);
            IO_CK(cudaGetLastError(), "unpack_tets_kernel");
        }
        IO_CK(cudaMemcpy(hf, fl, sizeof(hf), cudaMemcpyDeviceToHost), "D2H");
        if (hf[1] != ~0ull) return set_error(TV_ERR_FORMAT, kMsg[hf[1] & 7u]);
        if (got != want) return set_error(TV_ERR_FORMAT, eof);
    }

    for (int r = 0; r < 24; ++r) {  // builder.cpp:287-291
        uint64_t v = 0;
        if (std::fread(&v, 8, 1, f.f) != 1) return set_error(TV_ERR_FORMAT, eof);
        if (v != kSentinel && v >= kNone) return set_error(TV_ERR_FORMAT, "tet id out of range");
        if (v == kSentinel || v >= n_tets) return set_error(TV_ERR_FORMAT, "root id out of range");
        g.roots[r] = static_cast<uint32_t>(v);
    }
    g.n_leaves = hf[2];
    g.n_internal = n_tets - hf[2];
    rc = finalize_grid(g, nullptr);
    if (rc) return rc;
    guard.g = nullptr;
    *out = h.release();
    return TV_OK;
}

}  // extern "C"
