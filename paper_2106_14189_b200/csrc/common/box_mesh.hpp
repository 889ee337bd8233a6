// generate_box's cell connectivity (mesh.hpp:208-264), shared by the host
// builder (the global box and the part-local build) and the engine (which
// recognises a generated box for the fused step, k_box_step): H8 cells in
// corner order (element.hpp:17-20), T4 six tets per cell along the
// (0,0,0)-(1,1,1) diagonal, one per axis order, odd orders swapping the
// middle pair.
#pragma once

#include <cstdint>
#include <utility>

namespace djg {

// H8 corner signs (element.hpp:17-20), the reference's local node order
inline constexpr int kBoxCornerSign[8][3] = {
    {-1, -1, -1}, {+1, -1, -1}, {+1, +1, -1}, {-1, +1, -1},
    {-1, -1, +1}, {+1, -1, +1}, {+1, +1, +1}, {-1, +1, +1},
};

// Global connectivity of cell c of a div[0] x div[1] x div[2] box (H8: 8
// corners; T4: 6 tets x 4), kind 0 = T4, 1 = H8.
inline void box_cell_conn(int kind, const int32_t div[3], int64_t c, int32_t* out) {
    const int64_t nx = div[0], ny = div[1];
    const int64_t i = c % nx, j = (c / nx) % ny, k = c / (nx * ny);
    auto id = [&](int64_t a, int64_t b, int64_t d) { return int32_t(a + (nx + 1) * (b + (ny + 1) * d)); };
    int32_t corner[2][2][2];
    for (int dz = 0; dz < 2; ++dz)
        for (int dy = 0; dy < 2; ++dy)
            for (int dx = 0; dx < 2; ++dx) corner[dx][dy][dz] = id(i + dx, j + dy, k + dz);
    if (kind == 1) {
        for (int a = 0; a < 8; ++a)
            out[a] = corner[(kBoxCornerSign[a][0] + 1) / 2][(kBoxCornerSign[a][1] + 1) / 2][(kBoxCornerSign[a][2] + 1) / 2];
        return;
    }
    static constexpr int orders[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    for (int t = 0; t < 6; ++t) {
        const int* o = orders[t];
        int s[3] = {0, 0, 0};
        int32_t path[4];
        path[0] = corner[0][0][0];
        for (int q = 0; q < 3; ++q) {
            s[o[q]] = 1;
            path[q + 1] = corner[s[0]][s[1]][s[2]];
        }
        const bool odd = (o[0] == 0 && o[1] == 2) || (o[0] == 1 && o[1] == 0) || (o[0] == 2 && o[1] == 1);
        if (odd) std::swap(path[1], path[2]);
        for (int a = 0; a < 4; ++a) out[t * 4 + a] = path[a];
    }
}

}  // namespace djg
