// Exact integer LEB geometry shared by the GPU build and the GPU validator:
// the fixed-point orientation determinant and the canonical face-normal
// classification of the reference (tet_grid.cpp:14-25, 49-80).
#pragma once

#include <cstdint>

#include "tetvol_b200.h"

namespace tvb {

typedef __int128 i128;

// tet_grid.cpp:14-25
__host__ __device__ inline i128 det_fixed(uint4 v0, uint4 v1, uint4 v2, uint4 v3) {
    const int64_t a0 = static_cast<int64_t>(v1.x) - v0.x, a1 = static_cast<int64_t>(v1.y) - v0.y,
                  a2 = static_cast<int64_t>(v1.z) - v0.z;
    const int64_t b0 = static_cast<int64_t>(v2.x) - v0.x, b1 = static_cast<int64_t>(v2.y) - v0.y,
                  b2 = static_cast<int64_t>(v2.z) - v0.z;
    const int64_t c0 = static_cast<int64_t>(v3.x) - v0.x, c1 = static_cast<int64_t>(v3.y) - v0.y,
                  c2 = static_cast<int64_t>(v3.z) - v0.z;
    const int64_t m0 = b1 * c2 - b2 * c1, m1 = b2 * c0 - b0 * c2, m2 = b0 * c1 - b1 * c0;
    return static_cast<i128>(a0) * m0 + static_cast<i128>(a1) * m1 + static_cast<i128>(a2) * m2;
}

// tet_grid.cpp:49-80; -1 = NotCanonical
__host__ __device__ inline int face_normal_id(uint4 a, uint4 b, uint4 c, uint4 in) {
    const int64_t u0 = static_cast<int64_t>(b.x) - a.x, u1 = static_cast<int64_t>(b.y) - a.y,
                  u2 = static_cast<int64_t>(b.z) - a.z;
    const int64_t v0 = static_cast<int64_t>(c.x) - a.x, v1 = static_cast<int64_t>(c.y) - a.y,
                  v2 = static_cast<int64_t>(c.z) - a.z;
    int64_t n[3] = {u1 * v2 - u2 * v1, u2 * v0 - u0 * v2, u0 * v1 - u1 * v0};
    if (n[0] == 0 && n[1] == 0 && n[2] == 0) return -1;
    const i128 side = static_cast<i128>(n[0]) * (static_cast<int64_t>(in.x) - a.x) +
                      static_cast<i128>(n[1]) * (static_cast<int64_t>(in.y) - a.y) +
                      static_cast<i128>(n[2]) * (static_cast<int64_t>(in.z) - a.z);
    if (side == 0) return -1;
    if (side > 0) n[0] = -n[0], n[1] = -n[1], n[2] = -n[2];
    const int zeros = (n[0] == 0) + (n[1] == 0) + (n[2] == 0);
    if (zeros == 2) {
        for (int k = 0; k < 3; ++k)
            if (n[k] != 0) return 2 * k + (n[k] > 0 ? 0 : 1);
    } else if (zeros == 1) {
        const int zk = n[0] == 0 ? 0 : (n[1] == 0 ? 1 : 2);
        const int i = zk == 0 ? 1 : 0, j = zk == 2 ? 1 : 2;
        const int64_t ai = n[i] < 0 ? -n[i] : n[i], aj = n[j] < 0 ? -n[j] : n[j];
        if (ai != aj) return -1;
        const int base = zk == 2 ? 6 : (zk == 1 ? 10 : 14);
        const bool pi = n[i] > 0, pj = n[j] > 0;
        if (pi && pj) return base;
        if (!pi && !pj) return base + 1;
        if (pi && !pj) return base + 2;
        return base + 3;
    }
    return -1;
}

}  // namespace tvb
