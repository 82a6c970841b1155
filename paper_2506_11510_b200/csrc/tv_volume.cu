// Device-resident DenseVolume (volume.hpp:19-58) and its .dvol file
// (DenseVolume::save_dvol / load_dvol, volume.cpp:84-138): named f32 channels
// (x fastest) live in HBM, so a 1024^3 field goes file -> HBM in chunks or is
// generated on the device (cli.cpp:349-384) and never makes a host copy.
//
// .dvol layout (little endian): "DVOL" u32 version=1, u32 nx, ny, nz, u32
// n_channels, per channel u8 name length + name bytes, then each channel's
// nx*ny*nz f32 in channel order.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "tv_trace.cuh"

struct tv_volume {
    int device = 0;
    int nx = 0, ny = 0, nz = 0;
    std::vector<std::string> names;
    std::vector<float*> data;  // device, nx*ny*nz each
    ~tv_volume() {
        for (float* p : data) cudaFree(p);
    }
    uint64_t voxels() const { return static_cast<uint64_t>(nx) * ny * nz; }
    int find(const std::string& n) const {
        for (size_t i = 0; i < names.size(); ++i)
            if (names[i] == n) return static_cast<int>(i);
        return -1;
    }
};

namespace tvb {
namespace {

constexpr uint64_t kStage = 64ull << 20;  // bytes per staged copy

__global__ void fill_kernel(float* p, uint64_t n, float v) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        p[i] = v;
}

// cli.cpp:371-375: temperature = clamp(density, 0, 1) (std::clamp on floats)
__global__ void clamp_copy_kernel(const float* __restrict__ src, float* dst, uint64_t n) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const float v = src[i];
        dst[i] = v < 0.0f ? 0.0f : (1.0f < v ? 1.0f : v);
    }
}

int vol_error(const std::string& msg) { return set_error(TV_ERR_VOLUME, msg); }

// DenseVolume::add_channel (volume.cpp:23-29)
int add_channel(tv_volume& v, const std::string& name) {
    if (name.empty() || name.size() > 255) return vol_error("bad channel name");
    if (v.find(name) >= 0) return vol_error("channel already exists: " + name);
    float* p = nullptr;
    int rc = cuda_status(cudaMalloc(&p, std::max<uint64_t>(1, v.voxels()) * sizeof(float)), "volume alloc");
    if (rc) return rc;
    v.names.push_back(name);
    v.data.push_back(p);
    return cuda_status(cudaMemset(p, 0, v.voxels() * sizeof(float)), "memset");
}

struct File {
    FILE* f = nullptr;
    ~File() {
        if (f) std::fclose(f);
    }
};

struct Pinned {
    void* p = nullptr;
    ~Pinned() {
        if (p) cudaFreeHost(p);
    }
};

}  // namespace
}  // namespace tvb

using namespace tvb;

extern "C" {

int tv_volume_create(int32_t nx, int32_t ny, int32_t nz, int device, tv_volume** out) {
    if (!out) return set_error(TV_ERR_ARG, "null argument");
    *out = nullptr;
    if (nx < 1 || ny < 1 || nz < 1 || nx > 4096 || ny > 4096 || nz > 4096)
        return set_error(TV_ERR_CONFIG, "dims out of range [1, 4096]");
    int rc = use_device(device);
    if (rc) return rc;
    auto v = std::make_unique<tv_volume>();
    v->device = device, v->nx = nx, v->ny = ny, v->nz = nz;
    if ((rc = add_channel(*v, "density"))) return rc;  // volume.hpp:25
    *out = v.release();
    return TV_OK;
}

void tv_volume_free(tv_volume* v) {
    if (v) {
        cudaSetDevice(v->device);
        delete v;
    }
}

int tv_volume_get_info(const tv_volume* v, int32_t dims[3], int32_t* n_channels) {
    if (!v) return set_error(TV_ERR_ARG, "volume is null");
    if (dims) dims[0] = v->nx, dims[1] = v->ny, dims[2] = v->nz;
    if (n_channels) *n_channels = static_cast<int32_t>(v->names.size());
    return TV_OK;
}

int tv_volume_channel_name(const tv_volume* v, int32_t index, char* buf, int32_t cap) {
    if (!v || !buf || cap < 1) return set_error(TV_ERR_ARG, "null argument");
    if (index < 0 || index >= static_cast<int32_t>(v->names.size())) return set_error(TV_ERR_ARG, "bad channel index");
    std::snprintf(buf, static_cast<size_t>(cap), "%s", v->names[index].c_str());
    return TV_OK;
}

int tv_volume_channel_dev(const tv_volume* v, const char* name, float** out_dev) {
    if (!v || !name || !out_dev) return set_error(TV_ERR_ARG, "null argument");
    const int c = v->find(name);
    if (c < 0) return vol_error(std::string("unknown channel: ") + name);  // UnknownChannel (volume.cpp:31-35)
    *out_dev = v->data[c];
    return TV_OK;
}

int tv_volume_add_channel(tv_volume* v, const char* name) {
    if (!v || !name) return set_error(TV_ERR_ARG, "null argument");
    int rc = use_device(v->device);
    return rc ? rc : add_channel(*v, name);
}

// Procedural density (cli.cpp:317-367; kinds as tv_generate_volume_dev)
int tv_volume_generate(tv_volume* v, int32_t kind, double value) {
    if (!v) return set_error(TV_ERR_ARG, "volume is null");
    return tv_generate_volume_dev(kind, v->nx, v->ny, v->nz, value, v->data[0], v->device);
}

// cmd_gen's extra channels (cli.cpp:370-380): temperature = clamp(density, 0, 1),
// albedo = a constant in [0, 1]
int tv_volume_add_temperature(tv_volume* v) {
    if (!v) return set_error(TV_ERR_ARG, "volume is null");
    int rc = use_device(v->device);
    if (rc || (rc = add_channel(*v, "temperature"))) return rc;
    clamp_copy_kernel<<<148 * 8, 256>>>(v->data[v->find("density")], v->data.back(), v->voxels());
    return cuda_status(cudaDeviceSynchronize(), "temperature channel");
}

int tv_volume_add_albedo(tv_volume* v, double albedo) {
    if (!v) return set_error(TV_ERR_ARG, "volume is null");
    if (albedo < 0.0 || albedo > 1.0) return set_error(TV_ERR_CONFIG, "--with-albedo must be in [0,1]");
    int rc = use_device(v->device);
    if (rc || (rc = add_channel(*v, "albedo"))) return rc;
    fill_kernel<<<148 * 8, 256>>>(v->data.back(), v->voxels(), static_cast<float>(albedo));
    return cuda_status(cudaDeviceSynchronize(), "albedo channel");
}

int tv_volume_download(const tv_volume* v, const char* name, float* out) {
    float* d = nullptr;
    int rc = tv_volume_channel_dev(v, name, &d);
    if (rc || (rc = use_device(v->device))) return rc;
    if (!out) return set_error(TV_ERR_ARG, "null output");
    return cuda_status(cudaMemcpy(out, d, v->voxels() * sizeof(float), cudaMemcpyDeviceToHost), "download");
}

int tv_volume_upload(tv_volume* v, const char* name, const float* in) {
    float* d = nullptr;
    int rc = tv_volume_channel_dev(v, name, &d);
    if (rc || (rc = use_device(v->device))) return rc;
    if (!in) return set_error(TV_ERR_ARG, "null input");
    return cuda_status(cudaMemcpy(d, in, v->voxels() * sizeof(float), cudaMemcpyHostToDevice), "upload");
}

// DenseVolume::save_dvol (volume.cpp:84-100)
int tv_volume_save(const tv_volume* v, const char* path) {
    if (!v || !path) return set_error(TV_ERR_ARG, "null argument");
    int rc = use_device(v->device);
    if (rc) return rc;
    File f;
    f.f = std::fopen(path, "wb");
    if (!f.f) return vol_error(std::string("cannot open for writing: ") + path);
    bool ok = std::fwrite("DVOL", 1, 4, f.f) == 4;
    const uint32_t hdr[5] = {1u, static_cast<uint32_t>(v->nx), static_cast<uint32_t>(v->ny),
                             static_cast<uint32_t>(v->nz), static_cast<uint32_t>(v->names.size())};
    ok &= std::fwrite(hdr, 4, 5, f.f) == 5;
    for (const std::string& n : v->names) {
        const uint8_t len = static_cast<uint8_t>(n.size());
        ok &= std::fwrite(&len, 1, 1, f.f) == 1;
        ok &= std::fwrite(n.data(), 1, n.size(), f.f) == n.size();
    }
    Pinned host;
    if ((rc = cuda_status(cudaMallocHost(&host.p, kStage), "cudaMallocHost"))) return rc;
    const uint64_t per = kStage / sizeof(float);
    for (float* d : v->data)
        for (uint64_t s = 0; ok && s < v->voxels(); s += per) {
            const uint64_t n = std::min(per, v->voxels() - s);
            if ((rc = cuda_status(cudaMemcpy(host.p, d + s, n * sizeof(float), cudaMemcpyDeviceToHost), "D2H")))
                return rc;
            ok &= std::fwrite(host.p, sizeof(float), n, f.f) == n;
        }
    ok &= std::fflush(f.f) == 0;
    return ok ? TV_OK : vol_error(std::string("write failed: ") + path);
}

// DenseVolume::load_dvol (volume.cpp:102-138): the same checks and messages
int tv_volume_load(const char* path, int device, tv_volume** out) {
    if (!path || !out) return set_error(TV_ERR_ARG, "null argument");
    *out = nullptr;
    File f;
    f.f = std::fopen(path, "rb");
    if (!f.f) return vol_error(std::string("cannot open: ") + path);
    const std::string eof = "unexpected end of file";
    char magic[4];
    if (std::fread(magic, 1, 4, f.f) != 4 || std::memcmp(magic, "DVOL", 4) != 0)
        return vol_error(std::string("not a DVOL file: ") + path);
    uint32_t hdr[5];
    for (int k = 0; k < 5; ++k) {
        if (std::fread(&hdr[k], 4, 1, f.f) != 1) return vol_error(eof);
        if (k == 0 && hdr[0] != 1u) return vol_error("unsupported DVOL version");
    }
    const uint32_t nx = hdr[1], ny = hdr[2], nz = hdr[3], nch = hdr[4];
    if (nx < 1 || ny < 1 || nz < 1 || nx > 4096 || ny > 4096 || nz > 4096) return vol_error("bad dimensions");
    if (nch < 1 || nch > 16) return vol_error("bad channel count");
    std::vector<std::string> names;
    for (uint32_t c = 0; c < nch; ++c) {
        uint8_t len = 0;
        if (std::fread(&len, 1, 1, f.f) != 1) return vol_error(eof);
        if (len == 0) return vol_error("empty channel name");
        std::string name(len, '\0');
        if (std::fread(name.data(), 1, len, f.f) != len) return vol_error(eof);
        if (std::find(names.begin(), names.end(), name) != names.end())
            return vol_error("duplicate channel name: " + name);
        names.push_back(name);
    }
    int rc = use_device(device);
    if (rc) return rc;
    auto v = std::make_unique<tv_volume>();
    v->device = device, v->nx = static_cast<int>(nx), v->ny = static_cast<int>(ny), v->nz = static_cast<int>(nz);
    Pinned host;
    if ((rc = cuda_status(cudaMallocHost(&host.p, kStage), "cudaMallocHost"))) return rc;
    const uint64_t per = kStage / sizeof(float);
    for (const std::string& name : names) {
        if ((rc = add_channel(*v, name))) return rc;
        float* d = v->data.back();
        for (uint64_t s = 0; s < v->voxels(); s += per) {
            const uint64_t n = std::min(per, v->voxels() - s);
            if (std::fread(host.p, sizeof(float), n, f.f) != n) return vol_error("unexpected end of file in channel data");
            if ((rc = cuda_status(cudaMemcpy(d + s, host.p, n * sizeof(float), cudaMemcpyHostToDevice), "H2D")))
                return rc;
        }
    }
    *out = v.release();
    return TV_OK;
}

// build_adaptive_grid(const DenseVolume&, ...) (builder.hpp:51-52): the
// "density" channel, plus "temperature" / "albedo" when present (builder.cpp:166-167)
int tv_build_volume(const tv_volume* v, const tv_build_config* cfg, const tv_camera* camera, tv_grid** out,
                    tv_build_stats* stats) {
    if (!v) return set_error(TV_ERR_ARG, "volume is null");
    const int d = v->find("density"), t = v->find("temperature"), a = v->find("albedo");
    if (d < 0) return vol_error("unknown channel: density");
    return tv_build_dev(v->data[d], t >= 0 ? v->data[t] : nullptr, a >= 0 ? v->data[a] : nullptr, v->nx, v->ny, v->nz,
                        cfg, camera, v->device, out, stats);
}

}  // extern "C"
