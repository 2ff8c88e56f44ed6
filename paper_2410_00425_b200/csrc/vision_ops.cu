// Observation post-processing on the device: voxelisation of the fused
// pointcloud and green-screen compositing of rendered RGB.  Both are HBM-streaming kernels
// (grid-stride, a whole number of waves over the 148 SMs); the oracle (oracle/raster.py)
// performs the identical float32 operations, so grids and images match bit for bit.
#include <math.h>
#include "bs_common.cuh"

namespace bs {
namespace vision {

// One thread per point: cell = floor((p - lo) / cell_size) per axis (float32, separately
// rounded); points outside [0, dims) or with mask == 0 are dropped; occupancy is a byte store of
// 1 (idempotent, so races between points of one cell are benign).
__global__ void k_voxelize(const float* __restrict__ pts, int64_t stride, const uint8_t* __restrict__ valid,
                           int64_t n_per_batch, int64_t batches, float lx, float ly, float lz, float cell, int nx,
                           int ny, int nz, uint8_t* __restrict__ grid) {
  const int64_t total = n_per_batch * batches;
  const int64_t cells = (int64_t)nx * ny * nz;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    if (valid && !valid[i]) continue;
    const float* p = pts + i * stride;
    const int ix = (int)floorf(__fdiv_rn(__fsub_rn(p[0], lx), cell));
    const int iy = (int)floorf(__fdiv_rn(__fsub_rn(p[1], ly), cell));
    const int iz = (int)floorf(__fdiv_rn(__fsub_rn(p[2], lz), cell));
    if (ix < 0 || iy < 0 || iz < 0 || ix >= nx || iy >= ny || iz >= nz) continue;
    const int64_t b = i / n_per_batch;
    grid[b * cells + ((int64_t)ix * ny + iy) * nz + iz] = 1;
  }
}

__global__ void k_greenscreen(const uint8_t* __restrict__ rgb, const uint16_t* __restrict__ seg,
                              const uint8_t* __restrict__ bg, int64_t hw, int64_t frames, uint8_t* __restrict__ out) {
  const int64_t total = hw * frames;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t px = i % hw;
    const bool fg = seg[i] != 0;
#pragma unroll
    for (int k = 0; k < 3; ++k) out[3 * i + k] = fg ? rgb[3 * i + k] : bg[3 * px + k];
  }
}

}  // namespace vision
}  // namespace bs

extern "C" {

int bs_voxelize(const float* points, int64_t point_stride, const uint8_t* valid, int64_t points_per_batch,
                int64_t batches, const float* lo, float cell, int32_t nx, int32_t ny, int32_t nz, uint8_t* grid,
                void* stream) {
  if (!points || !lo || !grid || point_stride < 3 || points_per_batch < 0 || batches < 0) return BS_ERR_ARGUMENT;
  if (!(cell > 0.0f) || nx <= 0 || ny <= 0 || nz <= 0) return BS_ERR_INPUT;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t cells = (int64_t)nx * ny * nz * batches;
  if (cudaMemsetAsync(grid, 0, (size_t)cells, st) != cudaSuccess) return BS_ERR_CUDA;
  const int64_t n = points_per_batch * batches;
  if (n == 0) return BS_OK;
  bs::vision::k_voxelize<<<bs::grid_for(n, 256), 256, 0, st>>>(points, point_stride, valid, points_per_batch, batches,
                                                               lo[0], lo[1], lo[2], cell, nx, ny, nz, grid);
  return bs::launch_status();
}

int bs_composite_greenscreen(const uint8_t* rgb, const uint16_t* seg, const uint8_t* background, int64_t height,
                             int64_t width, int64_t frames, uint8_t* out, void* stream) {
  if (!rgb || !seg || !background || !out || height <= 0 || width <= 0 || frames < 0) return BS_ERR_ARGUMENT;
  const int64_t n = height * width * frames;
  if (n == 0) return BS_OK;
  bs::vision::k_greenscreen<<<bs::grid_for(n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      rgb, seg, background, height * width, frames, out);
  return bs::launch_status();
}

}  // extern "C"
