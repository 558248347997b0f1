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
};

}  // namespace vpb
