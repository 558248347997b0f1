// vpb_camdev.h — camera constants passed by value to the kernels. Prepared on the host with
// the reference's exact host arithmetic (Mat3::inverse, math.h:146-160; Camera::center,
// camera.h:28) so generateRay (camera.cpp:14-23) reproduces bit-for-bit on the device.
#pragma once

#include <cstdint>

namespace vpb {

struct CamDev {
    float kinv[9];
    float R[9];
    float K[9];
    float t[3];
    float center[3];
    int32_t width, height, tiles_x, tiles_y;
    // Tile sharding of one view over n_shards renders (vp_render_shard_async): this render
    // owns the tiles t (row-major tile index) with t % n_shards == shard. 1/0 = every tile.
    int32_t n_shards, shard;
};

#ifdef __CUDACC__
__host__ __device__ __forceinline__ bool tile_owned(const CamDev &c, int t) {
    return c.n_shards <= 1 || t % c.n_shards == c.shard;
}
#endif

}  // namespace vpb
