// Device-side domain description and HBM layout.
//
// Layout: structure of arrays, x fastest (reference
// fields.hpp:26-29). Population arrays carry `ghost` (0 or 1) extra z planes
// below and above the owned slab so a z-slab-decomposed run can push
// straight into its neighbour's boundary slots; moment/phase arrays hold only
// owned planes. Every array starts on a 256-byte boundary (stride padded).
#pragma once

#include <cstdint>

namespace tslb_cuda {

// Face behaviour as seen by ONE domain (a whole box, or one z slab).
enum FaceMode : int {
  kWrap = 0,   // periodic inside this domain: index wraps to the far side
  kWall = 1,   // half-way bounce-back, optional wall velocity
  kGhost = 2,  // slab interface: push lands in the ghost plane, exchanged later
};

enum FaceId : int { XMin = 0, XMax = 1, YMin = 2, YMax = 3, ZMin = 4, ZMax = 5 };

struct Dom {
  int nx, ny, nz;        // owned extent (nz = local slab depth)
  int ghost;             // ghost planes on each z side of population arrays
  int64_t plane;         // nx * ny
  int64_t n;             // owned nodes = plane * nz
  int64_t fstride;       // elements between consecutive population arrays
  int64_t mstride;       // elements between consecutive moment arrays
  int mode[6];           // FaceMode per face
  double uw[6][3];       // wall velocity per face, already rounded to T
  int has_solid;         // solid mask / slow mask present
  int xblocks;           // blocks per x row in the row-tiled launch
  int k0, nzr;           // launch range: planes [k0, k0 + nzr)
  // single-fluid body force (extension, tslb_cuda_set_body_force): the
  // moments pass stores u_eq = j + tf (tf = tau F) when `forced`
  int forced;
  double tf[3];
};

/// the forcing shift of the moments pass (identity when not forced, so the
/// unforced results keep every bit, including signed zeros)
template <typename C>
__device__ __forceinline__ void force_shift(const Dom& d, C& jx, C& jy, C& jz) {
  if (d.forced) {
    jx = jx + C(d.tf[0]);
    jy = jy + C(d.tf[1]);
    jz = jz + C(d.tf[2]);
  }
}

/// Row-tiled launch grid: blocks (x block, row j, plane k) as a 3-D grid
/// when ny and the plane range fit the grid limits (no index divisions in
/// the kernel), else one flattened dimension.
inline dim3 row_grid(const Dom& d) {
  if (d.ny <= 65535 && d.nzr <= 65535) return dim3(unsigned(d.xblocks), unsigned(d.ny), unsigned(d.nzr));
  return dim3(unsigned(int64_t(d.xblocks) * d.ny * d.nzr));
}

/// (x block, j, k) of this block for row_grid launches.
__device__ __forceinline__ void row_block(const Dom& d, unsigned& xb, int& j, int& k) {
  if (gridDim.y > 1 || gridDim.z > 1) {
    xb = blockIdx.x;
    j = int(blockIdx.y);
    k = int(blockIdx.z) + d.k0;
  } else {
    const unsigned row = blockIdx.x / unsigned(d.xblocks);
    xb = blockIdx.x - row * unsigned(d.xblocks);
    j = int(row % unsigned(d.ny));
    k = int(row / unsigned(d.ny)) + d.k0;
  }
}

/// Row-tiled node coordinates: block (xb, j, k) covers nodes
/// [xb*BX, xb*BX+BX) of row (j, k); returns false past the row end.
template <int BX>
__device__ __forceinline__ bool node_coords(const Dom& d, int& i, int& j, int& k) {
  unsigned xb;
  row_block(d, xb, j, k);
  i = int(xb * BX + threadIdx.x);
  return i < d.nx;
}

__device__ __forceinline__ int64_t midx(const Dom& d, int i, int j, int k) {
  return int64_t(i) + int64_t(d.nx) * (int64_t(j) + int64_t(d.ny) * k);
}

/// population-array index (shifted by the ghost plane)
__device__ __forceinline__ int64_t fidx(const Dom& d, int i, int j, int k) {
  return int64_t(i) +
         int64_t(d.nx) * (int64_t(j) + int64_t(d.ny) * (int64_t(k) + d.ghost));
}

// Per-thread face geometry: linear deltas for a +/- step on each axis
// (already wrapped for periodic faces, ghost-shifted for slab faces) and
// whether the step bounces off a wall.
struct Steps {
  int64_t dp[3], dm[3];
  bool bp[3], bm[3];
};

__device__ __forceinline__ Steps face_steps(const Dom& d, int i, int j, int k) {
  Steps s;
  const int c[3] = {i, j, k};
  const int nd[3] = {d.nx, d.ny, d.nz};
  const int64_t unit[3] = {1, int64_t(d.nx), d.plane};
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    s.dp[ax] = unit[ax];
    s.dm[ax] = -unit[ax];
    s.bp[ax] = false;
    s.bm[ax] = false;
    if (c[ax] == nd[ax] - 1) {
      const int m = d.mode[2 * ax + 1];
      if (m == kWrap) s.dp[ax] = -int64_t(nd[ax] - 1) * unit[ax];
      if (m == kWall) s.bp[ax] = true;
    }
    if (c[ax] == 0) {
      const int m = d.mode[2 * ax];
      if (m == kWrap) s.dm[ax] = int64_t(nd[ax] - 1) * unit[ax];
      if (m == kWall) s.bm[ax] = true;
    }
  }
  return s;
}

// The same with 32-bit deltas (a plane holds < 2^31 nodes): cheaper address
// arithmetic for stencil kernels that index relative to a node pointer.
struct Steps32 {
  int dp[3], dm[3];
  bool bp[3], bm[3];
};

__device__ __forceinline__ Steps32 face_steps32(const Dom& d, int i, int j, int k) {
  Steps32 s;
  const int c[3] = {i, j, k};
  const int nd[3] = {d.nx, d.ny, d.nz};
  const int unit[3] = {1, d.nx, int(d.plane)};
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    s.dp[ax] = unit[ax];
    s.dm[ax] = -unit[ax];
    s.bp[ax] = false;
    s.bm[ax] = false;
    if (c[ax] == nd[ax] - 1) {
      const int m = d.mode[2 * ax + 1];
      if (m == kWrap) s.dp[ax] = -(nd[ax] - 1) * unit[ax];
      if (m == kWall) s.bp[ax] = true;
    }
    if (c[ax] == 0) {
      const int m = d.mode[2 * ax];
      if (m == kWrap) s.dm[ax] = (nd[ax] - 1) * unit[ax];
      if (m == kWall) s.bm[ax] = true;
    }
  }
  return s;
}

}  // namespace tslb_cuda
