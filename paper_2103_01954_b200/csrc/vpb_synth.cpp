// vpb_synth.cpp — the synthetic benchmark inputs ("mvp_shell"): K primitives
// on a Fibonacci sphere (the analogue of MVP's surface-attached primitives, PAPER.md
// §3), analytic RGB/sigma voxel fields, and the lookAtCamera views. Host only. Deterministic
// for a given libstdc++/glibc (std::mt19937_64 + uniform_real_distribution<double>).
#include <cmath>
#include <cstring>
#include <random>

#include "../../include/vpb.h"
#include "vpb_hostmath.hpp"

using namespace vpb::host;

namespace {

constexpr double kPi = 3.14159265358979323846;

}  // namespace

extern "C" int vp_make_shell_scene(int32_t n_prim, int32_t m, float *tr24, float *payload) {
    if (n_prim < 0 || m < 1) return VP_ERR_USAGE;
    const double R = 0.35;
    const double h = n_prim > 0 ? R * std::sqrt(4.0 * kPi / n_prim) : 0.0;
    std::mt19937_64 rng(1234);
    std::uniform_real_distribution<double> uni(-1.0, 1.0);
    const double golden = kPi * (3.0 - std::sqrt(5.0));
    const size_t m3 = size_t(m) * m * m;
    const double sigma0 = n_prim > 0 ? 1.5 / (0.7 * h) : 0.0;
    for (int32_t k = 0; k < n_prim; ++k) {
        const double z = 1.0 - (2.0 * k + 1.0) / n_prim;
        const double r = std::sqrt(std::max(0.0, 1.0 - z * z));
        const double phi = k * golden;
        const double n[3] = {r * std::cos(phi), r * std::sin(phi), z};
        // t = normalize((0,0,1) x n), fallback (0,1,0); b = n x t; R_hat = [t b n].
        double t[3] = {-n[1], n[0], 0.0};
        const double tl = std::sqrt(t[0] * t[0] + t[1] * t[1] + t[2] * t[2]);
        if (tl < 1e-12) {
            t[0] = 0; t[1] = 1; t[2] = 0;
        } else {
            for (double &v : t) v /= tl;
        }
        const double b[3] = {n[1] * t[2] - n[2] * t[1], n[2] * t[0] - n[0] * t[2],
                             n[0] * t[1] - n[1] * t[0]};
        // Six draws in a fixed order (named temporaries: argument order is unspecified).
        const double d0 = uni(rng), d1 = uni(rng), d2 = uni(rng);
        const double d3 = uni(rng), d4 = uni(rng), d5 = uni(rng);
        float rec[24];
        rec[0] = float(R * n[0]); rec[1] = float(R * n[1]); rec[2] = float(R * n[2]);
        for (int i = 0; i < 3; ++i) {
            rec[3 + i] = float(t[i]);
            rec[6 + i] = float(b[i]);
            rec[9 + i] = float(n[i]);
        }
        rec[12] = float(0.6 * h); rec[13] = float(0.6 * h); rec[14] = float(0.35 * h);
        rec[15] = float(0.05 * h * d3); rec[16] = float(0.05 * h * d4); rec[17] = float(0.05 * h * d5);
        rec[18] = float(0.1 * d0); rec[19] = float(0.1 * d1); rec[20] = float(0.1 * d2);
        rec[21] = 0; rec[22] = 0; rec[23] = 0;
        if (tr24) std::memcpy(tr24 + 24 * size_t(k), rec, sizeof rec);
        if (!payload) continue;
        float xf[15];
        compose(rec, xf);
        float *slab = payload + size_t(k) * 4 * m3;
        for (int zi = 0; zi < m; ++zi)
            for (int yi = 0; yi < m; ++yi)
                for (int xi = 0; xi < m; ++xi) {
                    const F3 pm = f3(-1 + float(2 * xi + 1) / m, -1 + float(2 * yi + 1) / m,
                                     -1 + float(2 * zi + 1) / m);
                    const F3 pw = to_world(xf, pm);
                    const double x = pw.x, y = pw.y, zz = pw.z;
                    const size_t v = (size_t(zi) * m + yi) * m + xi;
                    for (int c = 0; c < 3; ++c)
                        slab[c * m3 + v] = float(0.5 + 0.45 * std::sin(9 * x + 7 * y * (c + 1) + 5 * zz));
                    slab[3 * m3 + v] = float(sigma0 * (0.5 + 0.5 * std::sin(11 * x + 13 * y + 3 * zz)));
                }
    }
    return VP_OK;
}

// synthetic.cpp:15-38
extern "C" int vp_look_at_camera(const float *position, const float *target, const float *up,
                                 float focal_px, int32_t width, int32_t height, vp_camera *out,
                                 float *axis_angle) {
    if (!position || !target || !up || !out) return VP_ERR_USAGE;
    const F3 pos = load3(position);
    const F3 forward = normalized(sub(load3(target), pos));
    F3 right = cross(forward, load3(up));
    if (dot(right, right) < 1e-12f) right = cross(forward, f3(0, 1, 0));
    right = normalized(right);
    const F3 down = cross(forward, right);
    M3 cols;
    cols.m[0] = right.x; cols.m[1] = right.y; cols.m[2] = right.z;
    cols.m[3] = down.x; cols.m[4] = down.y; cols.m[5] = down.z;
    cols.m[6] = forward.x; cols.m[7] = forward.y; cols.m[8] = forward.z;
    const M3 r = transposed(cols);
    const F3 aa = axis_angle_from_matrix(r);
    const M3 rot = rotation_from_axis_angle(aa);  // re-derived, as the reference does
    const F3 t = neg(mv(rot, pos));
    M3 k;
    k(0, 0) = focal_px;
    k(1, 1) = focal_px;
    k(0, 2) = float(width) / 2;
    k(1, 2) = float(height) / 2;
    std::memcpy(out->K, k.m, sizeof k.m);
    std::memcpy(out->R, rot.m, sizeof rot.m);
    out->t[0] = t.x; out->t[1] = t.y; out->t[2] = t.z;
    out->width = width;
    out->height = height;
    if (axis_angle) {
        axis_angle[0] = aa.x; axis_angle[1] = aa.y; axis_angle[2] = aa.z;
    }
    return VP_OK;
}

// Headline view (view < 0) or view v of an n-view ring around the shell.
extern "C" int vp_shell_camera(int32_t view, int32_t n_views, int32_t width, vp_camera *out) {
    if (width <= 0 || !out) return VP_ERR_USAGE;
    float pos[3];
    if (view < 0) {
        pos[0] = 0.25f; pos[1] = 0.15f; pos[2] = -1.1f;
    } else {
        if (n_views <= 0 || view >= n_views) return VP_ERR_USAGE;
        const double az = 2.0 * kPi * view / n_views;
        const double el = 0.35 * std::sin(3.0 * az);
        pos[0] = float(1.1 * std::cos(el) * std::sin(az));
        pos[1] = float(1.1 * std::sin(el));
        pos[2] = float(-1.1 * std::cos(el) * std::cos(az));
    }
    const float target[3] = {0, 0, 0}, up[3] = {0, 1, 0};
    return vp_look_at_camera(pos, target, up, float(1.2 * width), width, width, out, nullptr);
}
