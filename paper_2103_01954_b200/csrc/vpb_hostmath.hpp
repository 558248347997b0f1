// vpb_hostmath.hpp — host-side scene/camera arithmetic with the reference's exact binary32
// semantics (built with -ffp-contract=off; the reference objects contain no FMA). Used by
// the C-ABI for compose() and the camera constants, and by the synthetic scene generator.
#pragma once

#include <cmath>
#include <cstdint>

namespace vpb {
namespace host {

struct F3 {
    float x = 0, y = 0, z = 0;
};
inline F3 f3(float x, float y, float z) { F3 r; r.x = x; r.y = y; r.z = z; return r; }
inline F3 add(F3 a, F3 b) { return f3(a.x + b.x, a.y + b.y, a.z + b.z); }
inline F3 sub(F3 a, F3 b) { return f3(a.x - b.x, a.y - b.y, a.z - b.z); }
inline F3 mul(F3 a, float s) { return f3(a.x * s, a.y * s, a.z * s); }
inline F3 neg(F3 a) { return f3(-a.x, -a.y, -a.z); }
inline float dot(F3 a, F3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline F3 cross(F3 a, F3 b) {  // math.h:54-56
    return f3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
inline F3 normalized(F3 v) {  // v / sqrt(dot(v, v)), componentwise division (math.h:40,58-60)
    const float l = std::sqrt(dot(v, v));
    return f3(v.x / l, v.y / l, v.z / l);
}
inline float at(F3 v, int i) { return i == 0 ? v.x : (i == 1 ? v.y : v.z); }

// Column-major 3x3, element (row, col) at m[col * 3 + row] (math.h:71-106).
struct M3 {
    float m[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    float &operator()(int r, int c) { return m[c * 3 + r]; }
    float operator()(int r, int c) const { return m[c * 3 + r]; }
};
inline M3 zero3() { M3 r; for (float &v : r.m) v = 0; return r; }
inline F3 col(const M3 &a, int c) { return f3(a.m[c * 3], a.m[c * 3 + 1], a.m[c * 3 + 2]); }
inline F3 mv(const M3 &a, F3 v) {  // math.h:122-124
    return add(add(mul(col(a, 0), v.x), mul(col(a, 1), v.y)), mul(col(a, 2), v.z));
}
inline M3 transposed(const M3 &a) {
    M3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) r(i, j) = a(j, i);
    return r;
}
inline M3 mm(const M3 &a, const M3 &o) {  // math.h:115-121 (accumulate from zero, k middle)
    M3 r = zero3();
    for (int c = 0; c < 3; ++c)
        for (int k = 0; k < 3; ++k)
            for (int i = 0; i < 3; ++i) r(i, c) += a(i, k) * o(k, c);
    return r;
}
inline M3 inverse(const M3 &a) {  // math.h:141-160
    const float *m = a.m;
    const float d = m[0] * (m[4] * m[8] - m[5] * m[7]) - m[3] * (m[1] * m[8] - m[2] * m[7]) +
                    m[6] * (m[1] * m[5] - m[2] * m[4]);
    M3 r;
    r(0, 0) = a(1, 1) * a(2, 2) - a(1, 2) * a(2, 1);
    r(0, 1) = a(0, 2) * a(2, 1) - a(0, 1) * a(2, 2);
    r(0, 2) = a(0, 1) * a(1, 2) - a(0, 2) * a(1, 1);
    r(1, 0) = a(1, 2) * a(2, 0) - a(1, 0) * a(2, 2);
    r(1, 1) = a(0, 0) * a(2, 2) - a(0, 2) * a(2, 0);
    r(1, 2) = a(0, 2) * a(1, 0) - a(0, 0) * a(1, 2);
    r(2, 0) = a(1, 0) * a(2, 1) - a(1, 1) * a(2, 0);
    r(2, 1) = a(0, 1) * a(2, 0) - a(0, 0) * a(2, 1);
    r(2, 2) = a(0, 0) * a(1, 1) - a(0, 1) * a(1, 0);
    const float s = 1.0f / d;
    for (float &v : r.m) v *= s;
    return r;
}

// rotation.cpp:8-28 — Rodrigues map; series branch below theta = 1e-4.
inline M3 rotation_from_axis_angle(F3 v) {
    const float t2 = dot(v, v);
    if (t2 == 0) return M3{};
    const float theta = std::sqrt(t2);
    float a, b;
    if (theta < 1e-4f) {
        a = 1 - t2 / 6;
        b = 0.5f - t2 / 24;
    } else {
        a = std::sin(theta) / theta;
        b = (1 - std::cos(theta)) / t2;
    }
    M3 k = zero3();
    k(0, 1) = -v.z; k(0, 2) = v.y;
    k(1, 0) = v.z;  k(1, 2) = -v.x;
    k(2, 0) = -v.y; k(2, 1) = v.x;
    const M3 kk = mm(k, k);
    const M3 id;
    M3 r;
    for (int i = 0; i < 9; ++i) r.m[i] = (id.m[i] + k.m[i] * a) + kk.m[i] * b;
    return r;
}

// rotation.cpp:40-71
inline F3 axis_angle_from_matrix(const M3 &r) {
    auto clampf = [](float v, float lo, float hi) { return v < lo ? lo : (v > hi ? hi : v); };
    auto maxf = [](float a, float b) { return a < b ? b : a; };
    const float tr = r(0, 0) + r(1, 1) + r(2, 2);
    const float c = clampf((tr - 1) / 2, -1, 1);
    const float theta = std::acos(c);
    if (theta < 1e-7f) return F3{};
    const F3 axis = f3(r(2, 1) - r(1, 2), r(0, 2) - r(2, 0), r(1, 0) - r(0, 1));
    const float s = std::sqrt(dot(axis, axis));
    if (s < 1e-6f) {
        const F3 d = f3(std::sqrt(maxf(0, (r(0, 0) + 1) / 2)), std::sqrt(maxf(0, (r(1, 1) + 1) / 2)),
                        std::sqrt(maxf(0, (r(2, 2) + 1) / 2)));
        int k = 0;
        if (d.y > at(d, k)) k = 1;
        if (d.z > at(d, k)) k = 2;
        if (at(d, k) == 0) return F3{};
        F3 a2 = d;
        if (k == 0) {
            a2.y = (r(0, 1) + r(1, 0)) / (4 * d.x);
            a2.z = (r(0, 2) + r(2, 0)) / (4 * d.x);
        } else if (k == 1) {
            a2.x = (r(0, 1) + r(1, 0)) / (4 * d.y);
            a2.z = (r(1, 2) + r(2, 1)) / (4 * d.y);
        } else {
            a2.x = (r(0, 2) + r(2, 0)) / (4 * d.z);
            a2.y = (r(1, 2) + r(2, 1)) / (4 * d.z);
        }
        return mul(normalized(a2), theta);
    }
    return mul(axis, theta / s);
}

inline M3 skew(F3 v) {  // math.h:94-100
    M3 r = zero3();
    r(0, 1) = -v.z; r(0, 2) = v.y;
    r(1, 0) = v.z;  r(1, 2) = -v.x;
    r(2, 0) = -v.y; r(2, 1) = v.x;
    return r;
}

// rotation.cpp:30-38 — d R(v) / d v_i
inline M3 rotation_derivative(F3 v, int i) {
    const float t2 = dot(v, v);
    F3 e;
    (i == 0 ? e.x : (i == 1 ? e.y : e.z)) = 1;
    if (t2 < 1e-14f) return skew(e);
    const M3 r = rotation_from_axis_angle(v);
    M3 imr;
    for (int q = 0; q < 9; ++q) imr.m[q] = M3{}.m[q] - r.m[q];
    const F3 w = cross(v, mv(imr, e));
    const M3 sv = skew(v), sw = skew(w);
    const float vi = at(v, i), s = 1 / t2;
    M3 c;
    for (int q = 0; q < 9; ++q) c.m[q] = (sv.m[q] * vi + sw.m[q]) * s;
    return mm(c, r);
}

inline F3 load3(const float *p) { return f3(p[0], p[1], p[2]); }
inline M3 load9(const float *p) { M3 r; for (int i = 0; i < 9; ++i) r.m[i] = p[i]; return r; }

// primitive.cpp:41-49. Returns false on a non-positive composed scale (reference: Usage).
inline bool compose(const float *tr24, float *xf15) {
    const F3 s = add(load3(tr24 + 12), load3(tr24 + 21));
    if (s.x <= 0 || s.y <= 0 || s.z <= 0) return false;
    const M3 rot = mm(rotation_from_axis_angle(load3(tr24 + 18)), load9(tr24 + 3));
    const F3 t = add(load3(tr24 + 0), load3(tr24 + 15));
    xf15[0] = t.x; xf15[1] = t.y; xf15[2] = t.z;
    for (int i = 0; i < 9; ++i) xf15[3 + i] = rot.m[i];
    xf15[12] = s.x; xf15[13] = s.y; xf15[14] = s.z;
    return true;
}

// AffineXf::toWorld (primitive.h:59): t + R (s .* p)
inline F3 to_world(const float *xf15, F3 p) {
    const M3 rot = load9(xf15 + 3);
    return add(load3(xf15), mv(rot, f3(xf15[12] * p.x, xf15[13] * p.y, xf15[14] * p.z)));
}

}  // namespace host
}  // namespace vpb
