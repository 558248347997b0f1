// vpb_march.cuh — the per-ray segment window and the fused quadrature shared by the forward
// kernels (vpb_kernels.cu) and the backward pass (vpb_backward.cu). Device code only; the
// arithmetic contract is vpb_device.cuh's.
#pragma once

#include <cstdint>
#include <type_traits>

#include "vpb_bvh.cuh"
#include "vpb_device.cuh"
#include "vpb_kernels.h"

namespace vpb {

constexpr int kTile = 16;
constexpr int kMarchThreads = 256;  // one thread per pixel of a 16x16 tile
#ifndef VPB_CAND_CAP
#define VPB_CAND_CAP 56
#endif
constexpr int kCandCap = VPB_CAND_CAP;  // candidates staged in shared memory per tile (<= 255)

// A primitive's 16-float transform record held in registers (four 16-byte loads).
struct Xf16 {
    float v[16];
};
__device__ __forceinline__ Xf16 load_xf(const float4 *src, int step) {
    Xf16 r;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const float4 t = src[q * step];
        r.v[4 * q] = t.x;
        r.v[4 * q + 1] = t.y;
        r.v[4 * q + 2] = t.z;
        r.v[4 * q + 3] = t.w;
    }
    return r;
}
__device__ __forceinline__ Xf16 ldg_xf(const float *xf) {
    Xf16 r;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const float4 t = __ldg(reinterpret_cast<const float4 *>(xf) + q);
        r.v[4 * q] = t.x;
        r.v[4 * q + 1] = t.y;
        r.v[4 * q + 2] = t.z;
        r.v[4 * q + 3] = t.w;
    }
    return r;
}

// Candidate sources for the per-ray segment window. hit() is intersectObb (lbvh.cpp:177-205).
//
// TileCands<true>: every candidate of the tile is staged in shared memory (n <= kCandCap):
// transform, toModel(camera centre) (every ray of a render starts there, so om is computed
// once per candidate instead of once per ray, same operations, same bits), pixel rectangle
// and payload base. The staged transforms are quad-major (quad q of candidate c at
// s_xf4[q * xs + c]): lanes reading different candidates hit different banks (a 64-byte
// record stride put every other candidate on the same banks). TileCands<false>: the generic
// path reading the tile bucket from global memory (tiles with more candidates, fallback
// re-march). PF puts the line-vs-box prefilter (line_may_hit_box) in front of the staged
// exact test: it pays where most covered candidates miss (small primitives, the dense tier).
template <bool STAGED, bool PF = false>
struct TileCands {
    const unsigned long long *entries;
    const float *xf_g;
    const int4 *prects_g;
    const float4 *payload;
    unsigned m3;
    uint32_t start;
    int n;
    const int *s_prim;
    const float4 *s_xf4;
    const float4 *s_om;
    const int4 *s_prect;
    int xs;  // quad stride of s_xf4 (the staging capacity)
    __device__ __forceinline__ int prim(int c) const {
        if (STAGED) return s_prim[c];
        return (int)(uint32_t)(entries[start + c] & 0xffffffffull);
    }
    __device__ __forceinline__ const float *xf(int c) const {  // unstaged only
        return xf_g + (size_t)prim(c) * kXfStride;
    }
    __device__ __forceinline__ Xf16 xfv(int c) const {
        if (STAGED) return load_xf(s_xf4 + c, xs);
        return ldg_xf(xf(c));
    }
    __device__ __forceinline__ const float4 *base(int c) const {
        return payload + (size_t)prim(c) * m3;
    }
    // the candidate's conservative pixel rectangle (k_cull) contains the pixel
    __device__ __forceinline__ bool covers(int c, int2 px) const {
        const int4 r = STAGED ? s_prect[c] : prects_g[prim(c)];
        return px.x >= r.x && px.x <= r.z && px.y >= r.y && px.y <= r.w;
    }
    __device__ __forceinline__ bool hit(int c, V3 o, V3 d, float &tE, float &tX) const {
        if (STAGED) {
            const float4 om = s_om[c];
            const Xf16 x = xfv(c);
            if (PF && !line_may_hit_box(x.v, mk3(om.x, om.y, om.z), matTvec(x.v + 3, d))) return false;
            return intersect_obb_om(x.v, mk3(om.x, om.y, om.z), d, tE, tX);
        }
        return intersect_obb(xf(c), o, d, tE, tX);
    }
};

// Every primitive through the frame's BVH (arbitrary rays: march(), backwardRay, evalLoss).
// The scan visits exactly the primitives whose padded box the ray crosses (window_scan
// overload below); candidate ids are primitive ids.
struct BvhCands {
    const float *xf_g;
    const float4 *payload;
    unsigned m3;
    int n;
    BvhDev bvh;
    __device__ __forceinline__ int id(int i) const { return i; }
    __device__ __forceinline__ int prim(int c) const { return c; }
    __device__ __forceinline__ const float *xf(int c) const { return xf_g + (size_t)c * kXfStride; }
    __device__ __forceinline__ Xf16 xfv(int c) const { return ldg_xf(xf(c)); }
    __device__ __forceinline__ const float4 *base(int c) const { return payload + (size_t)c * m3; }
    __device__ __forceinline__ bool covers(int, int2) const { return true; }
    __device__ __forceinline__ bool hit(int c, V3 o, V3 d, float &tE, float &tX) const {
        return intersect_obb(xf(c), o, d, tE, tX);
    }
};

// Per-ray sorted segment window: slot j of ray `lane` lives at [j * stride + lane]
// (conflict-free across a warp). IdxT holds the candidate index (uint8_t for staged tiles).
#ifndef VPB_WC_INTERLEAVE
#define VPB_WC_INTERLEAVE 0
#endif
template <class IdxT>
struct Window {
    float *e;
    float *x;
    IdxT *c;
    int stride, lane;
    unsigned *m = nullptr;  // optional per-ray hit mask over the candidates (mw words)
    int mw = 0;
    __device__ __forceinline__ float &E(int j) const { return e[j * stride + lane]; }
    __device__ __forceinline__ float &X(int j) const { return x[j * stride + lane]; }
    // VPB_WC_INTERLEAVE=1 word-interleaves indices narrower than a word (a lane's entries
    // j..j+3 share one 32-bit word in the lane's own bank, so lanes at different j never
    // conflict; with c[j * stride + lane] four lanes share a bank). It removes 13 M excessive
    // shared wavefronts per headline launch but measured 0.4 % slower (more address math): off
    __device__ __forceinline__ IdxT &C(int j) const {
        constexpr int P = VPB_WC_INTERLEAVE && sizeof(IdxT) < 4 ? 4 / (int)sizeof(IdxT) : 1;
        if (P == 1) return c[j * stride + lane];
        return c[((j / P) * stride + lane) * P + (j % P)];
    }
    __device__ __forceinline__ unsigned &M(int word) const { return m[word * stride + lane]; }
};

struct RayOut {
    float r, g, b, alpha;
    int samples;
    int prim_samples;
    int hit, early, saturated, overflow, refills, numeric;
    // MarchResult bookkeeping backwardRay needs (march.h:22-33); dead code unless stored
    int last_step = -1;
    float sat_tprev = 0.f, sat_sigma = 0.f, sat_r = 0.f, sat_g = 0.f, sat_b = 0.f;
};

__device__ __forceinline__ bool key_less(float ea, int pa, float eb, int pb) {
    return ea != eb ? ea < eb : pa < pb;
}

// Inserts (tE, tX, c) into the sorted window [0, cnt) of capacity CAP, keeping the CAP
// smallest (tEnter, prim) keys; `more` records that a hit fell outside the window.
template <int CAP, class Cands, class Win>
__device__ __forceinline__ void window_insert(const Win &w, const Cands &cands, int &cnt,
                                              bool &more, float tE, float tX, int c, int prim) {
    if (cnt == CAP) {
        more = true;
        if (!key_less(tE, prim, w.E(CAP - 1), cands.prim(w.C(CAP - 1)))) return;
        cnt = CAP - 1;
    }
    int j = cnt;
    while (j > 0) {
        const float e = w.E(j - 1);
        if (e < tE || (e == tE && cands.prim(w.C(j - 1)) < prim)) break;
        w.E(j) = e;
        w.X(j) = w.X(j - 1);
        w.C(j) = w.C(j - 1);
        --j;
    }
    w.E(j) = tE;
    w.X(j) = tX;
    w.C(j) = c;
    ++cnt;
}

// Fills the window with the smallest hits whose key exceeds (lastE, lastP) (or all hits
// when first == true). The sorted list equals intersect()'s (lbvh.cpp:225-227 order); the
// kept entries do not depend on the scan order. With a hit mask, the first scan records which
// candidates hit and a refill re-tests only those (a refill is needed only by rays with more
// hits than the window holds, which otherwise would re-test every candidate per refill).
template <int CAP, class Cands, class Win>
__device__ __forceinline__ void window_scan(const Win &w, const Cands &cands, int &cnt,
                                            bool &more, V3 o, V3 d, int2 px, bool first,
                                            float lastE, int lastP) {
    if (!first && w.m) {
        for (int word = 0; word < w.mw; ++word)
            for (unsigned bits = w.M(word); bits; bits &= bits - 1) {
                const int c = word * 32 + __ffs(bits) - 1;
                float tE, tX;
                cands.hit(c, o, d, tE, tX);  // hit before, same operations: hits again
                const int prim = cands.prim(c);
                if (!key_less(lastE, lastP, tE, prim)) continue;
                window_insert<CAP>(w, cands, cnt, more, tE, tX, c, prim);
            }
        return;
    }
    if (first && w.m)
        for (int word = 0; word < w.mw; ++word) w.M(word) = 0u;
    for (int c = 0; c < cands.n; ++c) {
        float tE, tX;
        if (!cands.covers(c, px) || !cands.hit(c, o, d, tE, tX)) continue;
        if (first && w.m) w.M(c >> 5) |= 1u << (c & 31);
        const int prim = cands.prim(c);
        if (!first && !key_less(lastE, lastP, tE, prim)) continue;
        window_insert<CAP>(w, cands, cnt, more, tE, tX, c, prim);
    }
}

// window_scan over the BVH: the same predicate and insertion as the list scan, visiting the
// primitives the BVH does not prune (no hit mask: refills traverse again).
template <int CAP, class Win>
__device__ __forceinline__ void window_scan(const Win &w, const BvhCands &cands, int &cnt, bool &more, V3 o,
                                            V3 d, int2, bool first, float lastE, int lastP) {
    bvh_for_each(cands.bvh, o, d, [&](int c) {
        float tE, tX;
        if (!cands.hit(c, o, d, tE, tX)) return;
        if (!first && !key_less(lastE, lastP, tE, c)) return;
        window_insert<CAP>(w, cands, cnt, more, tE, tX, c, c);
    });
}

// The fused quadrature of march.cpp:18-93 over a sliding window of the ray's sorted
// segment list (filled by window_scan). Entries [0, nxt) have been admitted; `act` is the
// bitmask of admitted entries still live (tExit > ts). Iterating its set bits in ascending
// order visits the reference's `active` list in its order (admission order = window order).
// The reference's `ts >= tMax` break is implied: it only fires once every segment is
// admitted and retired, where the empty-active-set branch breaks on the same step.
//
// Retirement and admission for step i+1 are decided while step i is sampled: each sampled
// entry's exit is compared with ts(i+1) (the same expression step i+1 evaluates), and each
// sample iteration admits at most one pending entry with tEnter <= ts(i+1) (checking its
// exit against ts(i+1) as the reference's same-step removal does). This runs in the
// converged sampling code instead of divergent per-step scans; the per-step admission loop
// below only picks up what the folded admission left (and refills the window). nextE caches
// tEnter of the next pending entry.
//
// The loop is flattened to one primitive-sample per iteration: a lane first finds its next
// lattice step with a non-empty active set, then evaluates one active primitive; the step's
// accumulation happens after its last active primitive. Lanes whose steps have different
// numbers of active primitives stay in lock-step on primitive-samples.
template <int CAP, int MT, class Cands, class Win>
__device__ RayOut march_window(const Cands &cands, const Win &w, int cnt, bool more, V3 o,
                               V3 d, int2 px, float jit, const MarchDev &mp,
                               const unsigned long long *tab) {
    static_assert(CAP <= 32, "the active set is a 32-bit mask");
    const float kInf = __int_as_float(0x7f800000);
    RayOut out{0.f, 0.f, 0.f, 0.f, 0, 0, 0, 0, 0, 0, 0, 0};
    if (cnt == 0) return out;
    out.hit = 1;
    const float dt = mp.dt;
    const float t0 = w.E(0);
    int nxt = 0, j = 0;
    unsigned act = 0, retire = 0, admit = 0;
    float nextE = t0;
    // The lattice index is the reference's int64; a ray needing more than 2^30 steps (which
    // the reference would take hours to walk) is reported as Numeric instead.
    constexpr int kMaxStep = 1 << 30;
    int i = 0;
    float transmittance = 0.f, cr = 0.f, cg = 0.f, cb = 0.f;
    float ts = 0.f, tsNext = 0.f, sigmaSum = 0.f, rw = 0.f, gw = 0.f, bw = 0.f;
    V3 pw = o;
    bool sampling = false;
    for (;;) {
        if (!sampling) {
            for (;;) {  // next lattice step with a non-empty active set
                if (i > kMaxStep) {
                    out.numeric = 1;
                    goto done;
                }
                ts = t0 + (__int2float_rn(i) + jit) * dt;
                if (nxt < cnt ? nextE <= ts : more) {  // admission (march.cpp:38), with refill
                    for (;;) {
                        while (nxt < cnt && nextE <= ts) {
                            if (w.X(nxt) > ts) act |= 1u << nxt;  // else admitted and retired at once
                            ++nxt;
                            nextE = nxt < cnt ? w.E(nxt) : kInf;
                        }
                        if (nxt < cnt || !more) break;
                        // window exhausted while hits remain: keep the live entries (in
                        // order), then fetch the next hits after the last key
                        const float lastE = w.E(cnt - 1);
                        const int lastP = cands.prim(w.C(cnt - 1));
                        int live = 0;
                        for (unsigned m = act; m; m &= m - 1, ++live) {
                            const int q = __ffs(m) - 1;
                            if (live != q) {
                                w.E(live) = w.E(q);
                                w.X(live) = w.X(q);
                                w.C(live) = w.C(q);
                            }
                        }
                        if (live == CAP) {
                            out.overflow = 1;
                            return out;
                        }
                        act = (1u << live) - 1u;
                        cnt = live;
                        nxt = live;
                        more = false;
                        ++out.refills;
                        window_scan<CAP>(w, cands, cnt, more, o, d, px, false, lastE, lastP);
                        nextE = nxt < cnt ? w.E(nxt) : kInf;
                    }
                }
                if (act) {
                    j = __ffs(act) - 1;
                    break;
                }
                if (nxt >= cnt) goto done;  // active set empty, nothing left: march.cpp:43-44
                // gap skip to the next entry (march.cpp:45-49)
                const double sk = ceil((double)((nextE - t0) / dt) - (double)jit);
                const int skipTo = sk > (double)kMaxStep ? kMaxStep + 1 : (int)sk;
                i = skipTo > i + 1 ? skipTo : i + 1;
            }
            sampling = true;
            sigmaSum = 0.f;
            rw = gw = bw = 0.f;
            retire = 0;
            tsNext = t0 + (__int2float_rn(i + 1) + jit) * dt;
            pw = o + d * ts;
        }
        {  // one primitive-sample (march.cpp:63-70)
            const int c = w.C(j);
            float sg, r, g, b;
            const Xf16 xr = cands.xfv(c);
            sample_primitive<MT>(cands.base(c), mp.m, xr.v, pw, mp.alpha, mp.beta, tab, sg, r,
                                 g, b);
            sigmaSum += sg;
            rw += r * sg;
            gw += g * sg;
            bw += b * sg;
            ++out.prim_samples;
            if (w.X(j) <= tsNext) retire |= 1u << j;  // retirement at step i+1 (march.cpp:39-41)
            if (nxt < cnt && nextE <= tsNext) {  // admission at step i+1, one entry per sample
                if (w.X(nxt) > tsNext) admit |= 1u << nxt;
                ++nxt;
                nextE = nxt < cnt ? w.E(nxt) : kInf;
            }
        }
        const unsigned rest = act & ~((2u << j) - 1u);
        if (rest) {
            j = __ffs(rest) - 1;
            continue;
        }
        // step complete: march.cpp:71-88
        sampling = false;
        act = (act & ~retire) | admit;
        admit = 0;
        ++out.samples;
        out.last_step = i;
        const float dT = sigmaSum * dt;
        if (transmittance + dT >= 1.0f) {
            const float frac = (1.0f - transmittance) / dT;
            const float f = dt * frac;
            cr += rw * f;
            cg += gw * f;
            cb += bw * f;
            out.sat_tprev = transmittance;
            out.sat_sigma = sigmaSum;
            out.sat_r = rw;
            out.sat_g = gw;
            out.sat_b = bw;
            transmittance = 1.0f;
            out.saturated = 1;
            break;
        }
        cr += rw * dt;
        cg += gw * dt;
        cb += bw * dt;
        transmittance += dT;
        if (transmittance > 1.0f - mp.eps) {
            out.early = 1;
            break;
        }
        ++i;
    }
done:
    out.r = cr;
    out.g = cg;
    out.b = cb;
    out.alpha = transmittance;
    return out;
}

// Generic variant for windows wider than 32 entries (the fallback re-march): the same
// quadrature, with the live entries found by scanning the window instead of a bitmask.
// The fused quadrature of march.cpp:18-93 over a sliding window of the ray's sorted
// segment list (filled by window_scan). Entries [0, nxt) are admitted; an admitted entry is
// live while tExit > ts, and the live ones in window order are exactly the reference's
// `active` list. The reference's `ts >= tMax` break is implied: it only fires once every
// segment is admitted and retired, where the empty-active-set branch breaks on the same step.
//
// The loop is flattened to one primitive-sample per iteration: a lane first finds its next
// lattice step with a non-empty active set, then evaluates one active primitive; the step's
// accumulation happens after its last active primitive. Lanes whose steps have different
// numbers of active primitives stay in lock-step on primitive-samples. Between events the
// active set does not change: t_evt = min(next entry, earliest exit of a live entry), and
// while ts < t_evt a step reuses the previous active set without touching the window.
template <int CAP, int MT, class Cands, class Win>
__device__ RayOut march_window_generic(const Cands &cands, const Win &w, int cnt, bool more, V3 o,
                               V3 d, int2 px, float jit, const MarchDev &mp,
                               const unsigned long long *tab) {
    RayOut out{0.f, 0.f, 0.f, 0.f, 0, 0, 0, 0, 0, 0, 0, 0};
    if (cnt == 0) return out;
    out.hit = 1;
    const float dt = mp.dt;
    const float t0 = w.E(0);
    int nxt = 0, lo = 0, j = 0, jfirst = 0;
    long long i = 0;
    float transmittance = 0.f, cr = 0.f, cg = 0.f, cb = 0.f;
    float ts = 0.f, sigmaSum = 0.f, rw = 0.f, gw = 0.f, bw = 0.f;
    float t_evt = -3.402823466e+38f;
    V3 pw = o;
    bool sampling = false;
    for (;;) {
        if (!sampling) {
            for (;;) {  // next lattice step with a non-empty active set
                if (i > (1ll << 40)) {  // the reference would spin; report instead of hanging
                    out.numeric = 1;
                    goto done;
                }
                ts = t0 + (__ll2float_rn(i) + jit) * dt;
                if (ts < t_evt) {  // no admission, no retirement since the last step
                    j = jfirst;
                    break;
                }
                for (;;) {  // admission, refilling the window when it runs dry
                    while (nxt < cnt && w.E(nxt) <= ts) ++nxt;
                    if (nxt < cnt || !more) break;
                    const float lastE = w.E(cnt - 1);
                    const int lastP = cands.prim(w.C(cnt - 1));
                    int live = 0;
                    for (int q = 0; q < nxt; ++q) {
                        if (w.X(q) > ts) {
                            if (live != q) {
                                w.E(live) = w.E(q);
                                w.X(live) = w.X(q);
                                w.C(live) = w.C(q);
                            }
                            ++live;
                        }
                    }
                    if (live == CAP) {
                        out.overflow = 1;
                        return out;
                    }
                    cnt = live;
                    nxt = live;
                    lo = 0;
                    more = false;
                    ++out.refills;
                    window_scan<CAP>(w, cands, cnt, more, o, d, px, false, lastE, lastP);
                }
                while (lo < nxt && w.X(lo) <= ts) ++lo;
                j = lo;
                while (j < nxt && !(w.X(j) > ts)) ++j;
                if (j < nxt) {
                    jfirst = j;
                    t_evt = nxt < cnt ? w.E(nxt) : 3.402823466e+38f;
                    for (int q = j; q < nxt; ++q) {
                        const float x = w.X(q);
                        if (x > ts && x < t_evt) t_evt = x;
                    }
                    break;
                }
                if (nxt >= cnt) goto done;  // active set empty, nothing left: march.cpp:44
                const float tNext = w.E(nxt);  // gap skip, march.cpp:45-49
                const long long skipTo = (long long)ceil((double)((tNext - t0) / dt) - (double)jit);
                i = skipTo > i + 1 ? skipTo : i + 1;
            }
            sampling = true;
            sigmaSum = 0.f;
            rw = gw = bw = 0.f;
            pw = o + d * ts;
        }
        {  // one primitive-sample (march.cpp:63-70)
            const int c = w.C(j);
            float sg, r, g, b;
            const Xf16 xr = cands.xfv(c);
            sample_primitive<MT>(cands.base(c), mp.m, xr.v, pw, mp.alpha, mp.beta, tab, sg, r,
                                 g, b);
            sigmaSum += sg;
            rw += r * sg;
            gw += g * sg;
            bw += b * sg;
            ++out.prim_samples;
        }
        ++j;
        while (j < nxt && !(w.X(j) > ts)) ++j;
        if (j < nxt) continue;
        // step complete: march.cpp:71-88
        sampling = false;
        ++out.samples;
        out.last_step = (int)i;
        const float dT = sigmaSum * dt;
        if (transmittance + dT >= 1.0f) {
            const float frac = (1.0f - transmittance) / dT;
            const float f = dt * frac;
            cr += rw * f;
            cg += gw * f;
            cb += bw * f;
            out.sat_tprev = transmittance;
            out.sat_sigma = sigmaSum;
            out.sat_r = rw;
            out.sat_g = gw;
            out.sat_b = bw;
            transmittance = 1.0f;
            out.saturated = 1;
            break;
        }
        cr += rw * dt;
        cg += gw * dt;
        cb += bw * dt;
        transmittance += dT;
        if (transmittance > 1.0f - mp.eps) {
            out.early = 1;
            break;
        }
        ++i;
    }
done:
    out.r = cr;
    out.g = cg;
    out.b = cb;
    out.alpha = transmittance;
    return out;
}

// The BVH leaves whose padded box a ray crosses, found by a whole warp (n_prim >= 2). The
// warp keeps a frontier of pending nodes in shared memory (`fr`, `cap_fr` entries) and each
// round takes up to 32 of them off the top, one per lane; a lane tests both children's boxes
// and the hits are appended with ballots: internal children back onto the frontier, leaves
// onto `cand` (the first `cap_cand` of them are stored; `nc` counts all). The leaf set equals
// bvh_for_each's; only the order differs, and warp_segment_list orders its hits by key.
// Returns 0, or -1 when the frontier or the leaf list overflows (caller falls back).
#ifndef VPB_BVH_2LEVEL
#define VPB_BVH_2LEVEL 1
#endif
__device__ __forceinline__ int warp_bvh_leaves(const BvhDev &bvh, V3 o, V3 d, int lane, int *cand, int cap_cand,
                                               int *fr, int cap_fr, int &nc) {
    const V3 inv = mk3(1.0f / d.x, 1.0f / d.y, 1.0f / d.z);
    const unsigned below = (1u << lane) - 1u;
    if (lane == 0) fr[0] = 0;
    __syncwarp();
    int sp = 1;
    nc = 0;
#if VPB_BVH_2LEVEL
    if (bvh.wide) {
        // Three levels per round from the wide records (k_bvh_widen): up to 4 frontier nodes,
        // 8 lanes each (lane = 8 f + slot); lane tests great-grandchild slot `slot` of its
        // frontier node. A parent's box is the union of its children's, so the leaves found
        // are those of the one-level walk (never fewer: the exact test after the walk decides).
        while (sp > 0) {
            const int take = sp < 4 ? sp : 4, b = sp - take;
            const int f = lane >> 3;
            const bool act = f < take;
            const int node = act ? fr[b + f] : 0;
            __syncwarp();
            bool test = false;
            int id = 0;
            float lx = 0.f, ly = 0.f, lz = 0.f, hx = 0.f, hy = 0.f, hz = 0.f;
            if (act) {
                const float4 *ws = bvh.wide[node].s + 2 * (lane & 7);
                const float4 sa = ws[0], sb = ws[1];
                lx = sa.x, ly = sa.y, lz = sa.z, hx = sa.w, hy = sb.x, hz = sb.y;
                id = __float_as_int(sb.z);
                test = sb.w != 0.0f;
            }
            const bool hit = test && ray_box(o, d, inv, lx, ly, lz, hx, hy, hz);
            const unsigned pi = __ballot_sync(0xffffffffu, hit && id >= 0);
            const unsigned pl = __ballot_sync(0xffffffffu, hit && id < 0);
            const int np = __popc(pi);
            if (b + np > cap_fr) return -1;
            if (hit && id >= 0) fr[b + __popc(pi & below)] = id;
            if (hit && id < 0) {
                const int q = nc + __popc(pl & below);
                if (q < cap_cand) cand[q] = -id - 1;
            }
            nc += __popc(pl);
            if (nc > cap_cand) return -1;
            sp = b + np;
            __syncwarp();
        }
        return 0;
    }
    // Two levels per round: up to 8 frontier nodes, 4 lanes each (lane = 4 f + 2 c + g): lane
    // (c, g) tests grandchild g of child c directly (a leaf child: its own box, g == 0). A
    // parent's box is the union of its children's, so a ray that hits a grandchild box hits its
    // child box: the leaves found are those of the one-level walk (never fewer: the exact test
    // after the walk decides), in half the rounds, with 4x the lanes busy (a ray's frontier is
    // narrow, so one node per lane left most of the warp idle).
    while (sp > 0) {
        const int take = sp < 8 ? sp : 8, b = sp - take;
        const int f = lane >> 2, c = (lane >> 1) & 1, g = lane & 1;
        const bool act = f < take;
        const int node = act ? fr[b + f] : 0;
        __syncwarp();
        // each lane picks its box first, then ONE slab test runs on all of them (four call
        // sites, one per (leaf, c, g) case, ran at 5 threads per instruction)
        bool test = false;
        int id = 0;
        float lx = 0.f, ly = 0.f, lz = 0.f, hx = 0.f, hy = 0.f, hz = 0.f;
        if (act) {
            const BvhNode n = bvh.nodes[node];
            const int child = c ? n.d.y : n.d.x;
            if (child < 0) {
                test = g == 0;
                id = child;
                if (c) {
                    lx = n.b.z, ly = n.b.w, lz = n.c.x, hx = n.c.y, hy = n.c.z, hz = n.c.w;
                } else {
                    lx = n.a.x, ly = n.a.y, lz = n.a.z, hx = n.a.w, hy = n.b.x, hz = n.b.y;
                }
            } else {
                const BvhNode cn = bvh.nodes[child];
                test = true;
                id = g ? cn.d.y : cn.d.x;
                if (g) {
                    lx = cn.b.z, ly = cn.b.w, lz = cn.c.x, hx = cn.c.y, hy = cn.c.z, hz = cn.c.w;
                } else {
                    lx = cn.a.x, ly = cn.a.y, lz = cn.a.z, hx = cn.a.w, hy = cn.b.x, hz = cn.b.y;
                }
            }
        }
        const bool hit = test && ray_box(o, d, inv, lx, ly, lz, hx, hy, hz);
        const unsigned pi = __ballot_sync(0xffffffffu, hit && id >= 0);
        const unsigned pl = __ballot_sync(0xffffffffu, hit && id < 0);
        const int np = __popc(pi);
        if (b + np > cap_fr) return -1;
        if (hit && id >= 0) fr[b + __popc(pi & below)] = id;
        if (hit && id < 0) {
            const int q = nc + __popc(pl & below);
            if (q < cap_cand) cand[q] = -id - 1;
        }
        nc += __popc(pl);
        if (nc > cap_cand) return -1;
        sp = b + np;
        __syncwarp();
    }
    return 0;
#else
    while (sp > 0) {
        const int take = sp < 32 ? sp : 32, b = sp - take;
        const bool act = lane < take;
        const int node = act ? fr[b + lane] : 0;
        __syncwarp();
        bool hl = false, hr = false;
        int l = 0, r = 0;
        if (act) {
            const BvhNode n = bvh.nodes[node];
            hl = ray_box(o, d, inv, n.a.x, n.a.y, n.a.z, n.a.w, n.b.x, n.b.y);
            hr = ray_box(o, d, inv, n.b.z, n.b.w, n.c.x, n.c.y, n.c.z, n.c.w);
            l = n.d.x;
            r = n.d.y;
        }
        const unsigned pl = __ballot_sync(0xffffffffu, hl && l >= 0), pr = __ballot_sync(0xffffffffu, hr && r >= 0);
        const unsigned ll = __ballot_sync(0xffffffffu, hl && l < 0), lr = __ballot_sync(0xffffffffu, hr && r < 0);
        const int npl = __popc(pl), np = npl + __popc(pr), nll = __popc(ll);
        if (b + np > cap_fr) return -1;
        if (hl && l >= 0) fr[b + __popc(pl & below)] = l;
        if (hr && r >= 0) fr[b + npl + __popc(pr & below)] = r;
        if (hl && l < 0) {
            const int q = nc + __popc(ll & below);
            if (q < cap_cand) cand[q] = -l - 1;
        }
        if (hr && r < 0) {
            const int q = nc + nll + __popc(lr & below);
            if (q < cap_cand) cand[q] = -r - 1;
        }
        nc += nll + __popc(lr);
        if (nc > cap_cand) return -1;
        sp = b + np;
        __syncwarp();
    }
    return 0;
#endif
}

// The complete sorted segment list of one ray, built by a warp: the warp walks the BVH
// (warp_bvh_leaves) and lists the primitives whose box the ray crosses (cheap box tests); the exact intersectObb
// tests run on all lanes; the hits are placed by rank of their (tEnter, prim) key (keys are
// distinct), which is the order window_scan produces. Returns the hit count, or -1 when the
// ray crosses more than `cap_cand` boxes or has more than `cap` hits (caller falls back).
__device__ __forceinline__ int warp_segment_list(const BvhCands &cands, V3 o, V3 d, int lane, int *cand,
                                                 float *ce, float *cx, int cap_cand, float *E, float *X, int *P,
                                                 int cap) {
    int nc = 0;
    if (cands.bvh.n_prim <= 1) {
        if (lane == 0)
            bvh_for_each(cands.bvh, o, d, [&](int c) {
                if (nc < cap_cand) cand[nc] = c;
                ++nc;
            });
        nc = __shfl_sync(0xffffffffu, nc, 0);
    } else if (warp_bvh_leaves(cands.bvh, o, d, lane, cand, cap_cand, reinterpret_cast<int *>(ce), cap_cand,
                               nc) < 0) {
        return -1;
    }
    __syncwarp();
    if (nc > cap_cand) return -1;
    for (int q = lane; q < nc; q += 32) {
        float tE, tX;
        const bool hit = cands.hit(cand[q], o, d, tE, tX);
        ce[q] = hit ? tE : __int_as_float(0x7f800000);
        cx[q] = tX;
    }
    __syncwarp();
    // the hits moved to the front in candidate order (in place: a round's reads precede its
    // writes, and no write passes the round's own slots), then ranked among themselves
    int nh = 0;
    for (int q0 = 0; q0 < nc; q0 += 32) {
        const int q = q0 + lane;
        float e = __int_as_float(0x7f800000), x = 0.f;
        int c = 0;
        if (q < nc) {
            e = ce[q];
            x = cx[q];
            c = cand[q];
        }
        const bool h = e != __int_as_float(0x7f800000);
        const unsigned b = __ballot_sync(0xffffffffu, h);
        __syncwarp();
        if (h) {
            const int dst = nh + __popc(b & ((1u << lane) - 1u));
            ce[dst] = e;
            cx[dst] = x;
            cand[dst] = c;
        }
        nh += __popc(b);
    }
    __syncwarp();
    if (nh > cap) return -1;
    for (int q = lane; q < nh; q += 32) {
        const float e = ce[q];
        const int pq = cand[q];
        int rank = 0;
        for (int u = 0; u < nh; ++u) rank += key_less(ce[u], cand[u], e, pq);
        E[rank] = e;
        X[rank] = cx[q];
        P[rank] = pq;
    }
    __syncwarp();
    return nh;
}

// Step-parallel march of ONE ray by a warp (small ray batches, e.g. evalLoss's 2048 rays,
// where one thread per ray leaves the GPU idle while the longest rays walk hundreds of steps).
// E/X/P hold the ray's complete sorted segment list (cnt entries, no refill). Lane L takes
// lattice step base + L: its active set {j : E_j <= ts < X_j} in list order is exactly the
// reference's incremental `active` list at that step (admission in list order, retirement at
// X <= ts), so each lane forms the step's sums with the same operations as march_window.
// The visited sequence is then replayed in order: consecutive steps while the active set is
// non-empty, and at the first empty one the reference's gap skip (march.cpp:43-49) picks the
// next chunk's base. Transmittance and colour are accumulated serially over the chunk's
// steps (every lane computes the same values from shuffles), so the result is bit-identical.
#ifndef VPB_FWD_PAIRS
#define VPB_FWD_PAIRS 1  // deal primitive-samples (not steps) out to the lanes
#endif
// march_warp's per-warp step sums: sigma, r, g, b rows of kSvStride floats (33: row k's
// step s sits in bank (s + k) % 32, so the four chains' lanes read distinct banks)
constexpr int kSvStride = 33;
template <class Cands, int MT = 0>
__device__ RayOut march_warp(const Cands &cands, const float *E, const float *X, const int *P, int cnt, V3 o,
                             V3 d, float jit, const MarchDev &mp, const unsigned long long *tab, int lane,
                             float *sv) {
    RayOut out{0.f, 0.f, 0.f, 0.f, 0, 0, 0, 0, 0, 0, 0, 0};
    if (cnt == 0) return out;
    out.hit = 1;
    const float dt = mp.dt, t0 = E[0];
    constexpr int kMaxStep = 1 << 30;
    float T = 0.f, cr = 0.f, cg = 0.f, cb = 0.f;
    int base = 0;
    bool done = false;
    while (!done) {
        if (base > kMaxStep) {
            out.numeric = 1;
            break;
        }
        const int i = base + lane;
        const bool in_range = i <= kMaxStep;
        const float ts = t0 + (__int2float_rn(i) + jit) * dt;
        float sig = 0.f, rw = 0.f, gw = 0.f, bw = 0.f;
        int na = 0, nadm = 0;
#if VPB_FWD_PAIRS
        for (int j = 0; j < cnt && in_range; ++j) {
            if (!(E[j] <= ts)) break;  // sorted by tEnter: the admitted entries are a prefix
            nadm = j + 1;
            na += X[j] > ts;
        }
        const unsigned empty = __ballot_sync(0xffffffffu, !(in_range && na > 0));
        const int L = empty ? __ffs(empty) - 1 : 32;
        // The primitive-samples of the visited steps s < L (k-th active entry of step s),
        // step-major, are dealt out one per lane, 32 at a time; each step's four sums are then
        // folded in list order from the carry of the previous batch, which is exactly the
        // per-step accumulation below (march.cpp:60-70).
        const int myna = lane < L ? na : 0;
        int incl = myna;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += v;
        }
        const int excl = incl - myna;
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        for (int p0 = 0; p0 < total; p0 += 32) {
            const int p = p0 + lane;
            const bool has = p < total;
            int s = 0;  // the pair's step: the number of lanes with incl <= p
#pragma unroll
            for (int h = 16; h > 0; h >>= 1)
                if (__shfl_sync(0xffffffffu, incl, s + h - 1) <= p) s += h;
            const int k = p - __shfl_sync(0xffffffffu, excl, s);
            const int incl_s = __shfl_sync(0xffffffffu, incl, s);
            const float tsp = __shfl_sync(0xffffffffu, ts, s);
            float a[4] = {0.f, 0.f, 0.f, 0.f};
            if (has) {
                int j = 0;
                for (int left = k;; ++j)
                    if (X[j] > tsp) {
                        if (left == 0) break;
                        --left;
                    }
                const int c = P[j];
                float sg, r, g, b;
                const Xf16 xr = cands.xfv(c);
                sample_primitive<MT>(cands.base(c), mp.m, xr.v, o + d * tsp, mp.alpha, mp.beta, tab, sg, r, g, b);
                a[0] = sg;
                a[1] = r * sg;
                a[2] = g * sg;
                a[3] = b * sg;
            }
            const bool lead = has && (lane == 0 || k == 0);
            const int run = lead ? min(incl_s - p, 32 - lane) : 0;
            float c[4] = {__shfl_sync(0xffffffffu, sig, s), __shfl_sync(0xffffffffu, rw, s),
                          __shfl_sync(0xffffffffu, gw, s), __shfl_sync(0xffffffffu, bw, s)};
#pragma unroll
            for (int q = 0; q < 4; ++q) c[q] += a[q];
            const int maxrun = __reduce_max_sync(0xffffffffu, run);
            for (int t = 1; t < maxrun; ++t) {
                float v[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) v[q] = __shfl_down_sync(0xffffffffu, a[q], t);
                if (t < run)
#pragma unroll
                    for (int q = 0; q < 4; ++q) c[q] += v[q];
            }
            // lane s < L takes its step's fold from the lane holding the step's first pair here
            const int f = excl > p0 ? excl - p0 : 0;
            const int fl = f < 32 ? f : 31;
            const bool mine = lane < L && excl < p0 + 32 && incl > p0;
            float nv[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) nv[q] = __shfl_sync(0xffffffffu, c[q], fl);
            if (mine) {
                sig = nv[0];
                rw = nv[1];
                gw = nv[2];
                bw = nv[3];
            }
        }
#else
        const V3 pw = o + d * ts;
        for (int j = 0; j < cnt && in_range; ++j) {
            if (!(E[j] <= ts)) break;  // sorted by tEnter: the admitted entries are a prefix
            nadm = j + 1;
            if (X[j] > ts) {
                const int c = P[j];
                float sg, r, g, b;
                const Xf16 xr = cands.xfv(c);
                sample_primitive<0>(cands.base(c), mp.m, xr.v, pw, mp.alpha, mp.beta, tab, sg, r, g, b);
                sig += sg;
                rw += r * sg;
                gw += g * sg;
                bw += b * sg;
                ++na;
            }
        }
        const unsigned empty = __ballot_sync(0xffffffffu, !(in_range && na > 0));
        const int L = empty ? __ffs(empty) - 1 : 32;
#endif
        // The chunk's visited steps, in order (march.cpp:71-88). The step sums go to shared
        // memory; the transmittance chain (every lane, the same values) finds where the ray
        // stops, then lanes 0-2 run the r, g, b chains side by side: the same additions in
        // the same order as one loop carrying all four sums, in fewer instructions per step.
        sv[lane] = sig;
        sv[kSvStride + lane] = rw;
        sv[2 * kSvStride + lane] = gw;
        sv[3 * kSvStride + lane] = bw;
        __syncwarp();
        int stop = L;  // steps before `stop` take dt in full; stop < L: the ray ends at step `stop`
        bool sat = false;
        float Tprev = T;
        // Quiet chunk: when T plus every positive dT of the chunk stays clear of both stopping
        // thresholds (by far more than the chain's rounding), no step can stop the ray, and the
        // chain runs without its tests. NaN or inf terms make the bound fail: the tested loop.
        float pos = 0.f;
        if (lane < L) {
            const float dT = sig * dt;
            pos = dT > 0.0f ? dT : (dT == dT ? 0.0f : __int_as_float(0x7f800000));
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) pos += __shfl_xor_sync(0xffffffffu, pos, off);
        const float lim = fminf(1.0f - mp.eps, 1.0f);
        const bool quiet = T >= 0.0f && T + pos * 1.0001f + 1e-5f < lim;
        if (quiet) {
            // every step takes dt in full: lanes 0-2 run the r, g, b chains and the others the
            // transmittance chain, all in one loop (the same additions in the same order)
            const float *cv = sv + kSvStride * (lane < 3 ? 1 + lane : 0);
            float c = lane == 0 ? cr : (lane == 1 ? cg : (lane == 2 ? cb : T));
            for (int s = 0; s < L; ++s) c += cv[s] * dt;
            cr = __shfl_sync(0xffffffffu, c, 0);
            cg = __shfl_sync(0xffffffffu, c, 1);
            cb = __shfl_sync(0xffffffffu, c, 2);
            T = __shfl_sync(0xffffffffu, c, 3);
        } else
        for (int s = 0; s < L; ++s) {
            const float dT = sv[s] * dt;
            if (T + dT >= 1.0f) {
                sat = true;
                stop = s;
                Tprev = T;
                break;
            }
            T += dT;
            if (T > 1.0f - mp.eps) {
                out.early = 1;
                stop = s;
                break;
            }
        }
        const int n_steps = stop < L ? stop + 1 : L;  // steps sampled in this chunk
        const int n_full = sat ? stop : n_steps;     // ... of which with the full dt
        if (!quiet) {
            const float *cv = sv + kSvStride * (1 + (lane < 2 ? lane : 2));
            float c = lane == 0 ? cr : (lane == 1 ? cg : cb);
            for (int s = 0; s < n_full; ++s) c += cv[s] * dt;
            if (sat) {
                const float frac = (1.0f - Tprev) / (sv[stop] * dt);  // march.cpp:75-82: (1 - T) / dT
                c += cv[stop] * (dt * frac);
            }
            cr = __shfl_sync(0xffffffffu, c, 0);
            cg = __shfl_sync(0xffffffffu, c, 1);
            cb = __shfl_sync(0xffffffffu, c, 2);
        }
        out.samples += n_steps;
        out.prim_samples += __reduce_add_sync(0xffffffffu, lane < n_steps ? na : 0);
        if (n_steps > 0) out.last_step = base + n_steps - 1;
        if (sat) {
            out.sat_tprev = Tprev;
            out.sat_sigma = sv[stop];
            out.sat_r = sv[kSvStride + stop];
            out.sat_g = sv[2 * kSvStride + stop];
            out.sat_b = sv[3 * kSvStride + stop];
            T = 1.0f;
            out.saturated = 1;
        }
        done = stop < L;
        __syncwarp();
        if (done) break;
        if (L == 32) {
            base += 32;
            continue;
        }
        const int iL = base + L;  // visited with an empty active set
        if (iL > kMaxStep) {
            out.numeric = 1;
            break;
        }
        const int nadmL = __shfl_sync(0xffffffffu, nadm, L);
        if (nadmL >= cnt) break;  // nothing left to admit: march.cpp:43-44
        const float nextE = E[nadmL];
        const double sk = ceil((double)((nextE - t0) / dt) - (double)jit);  // gap skip, march.cpp:45-49
        const int skipTo = sk > (double)kMaxStep ? kMaxStep + 1 : (int)sk;
        base = skipTo > iL + 1 ? skipTo : iL + 1;
    }
    out.r = cr;
    out.g = cg;
    out.b = cb;
    out.alpha = T;
    return out;
}

template <int CAP, class Cands, class Win>
__device__ __forceinline__ RayOut march_ray(const Cands &cands, const Win &w, V3 o, V3 d,
                                            int2 px, float jit, const MarchDev &mp,
                                            const unsigned long long *tab) {
    int cnt = 0;
    bool more = false;
    window_scan<CAP>(w, cands, cnt, more, o, d, px, true, 0.f, 0);
    if constexpr (CAP <= 32)
        return march_window<CAP, 0>(cands, w, cnt, more, o, d, px, jit, mp, tab);
    else
        return march_window_generic<CAP, 0>(cands, w, cnt, more, o, d, px, jit, mp, tab);
}

__device__ __forceinline__ void write_pixel(const OutDev &od, int64_t p, const RayOut &ro) {
    if (od.shard_n) {  // image pixel index -> slot in the shard's tile-major buffer
        const int px = (int)(p % od.width), py = (int)(p / od.width);
        const int t = (py >> 4) * od.tiles_x + (px >> 4);
        p = (int64_t)(t / od.shard_n) * 256 + (py & 15) * 16 + (px & 15);
    }
    od.rgb[3 * p + 0] = ro.r;
    od.rgb[3 * p + 1] = ro.g;
    od.rgb[3 * p + 2] = ro.b;
    od.alpha[p] = ro.alpha;
    if (od.samples) od.samples[p] = ro.samples;
}

// Arbitrary-ray kernels only (the tile kernel keeps the bookkeeping dead): the per-ray
// forward state for a following backward pass.
__device__ __forceinline__ void write_ray(const OutDev &od, int64_t p, const RayOut &ro) {
    write_pixel(od, p, ro);
    if (od.state) {
        float *s = od.state + 8 * p;
        s[0] = __int_as_float(ro.last_step);
        s[1] = __int_as_float(ro.saturated);
        s[2] = ro.sat_tprev;
        s[3] = ro.sat_sigma;
        s[4] = ro.sat_r;
        s[5] = ro.sat_g;
        s[6] = ro.sat_b;
        s[7] = __int_as_float(-1);  // no stored segment list (the warp kernel overwrites it)
    }
}

// Warp-aggregated counter update: one atomic per warp per counter.
__device__ __forceinline__ void add_counters(DevCounters *ctr, const RayOut &ro, bool valid) {
    unsigned long long v[7] = {(unsigned long long)(valid ? ro.samples : 0),
                               (unsigned long long)(valid ? ro.prim_samples : 0),
                               (unsigned long long)(valid ? ro.hit : 0),
                               (unsigned long long)(valid ? ro.early : 0),
                               (unsigned long long)(valid ? ro.saturated : 0),
                               (unsigned long long)(valid ? ro.refills : 0),
                               (unsigned long long)(valid ? ro.numeric : 0)};
#pragma unroll
    for (int q = 0; q < 7; ++q)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_down_sync(0xffffffffu, v[q], o);
    if ((threadIdx.x & 31) == 0) {
        if (v[0]) atomicAdd(&ctr->ray_samples, v[0]);
        if (v[1]) atomicAdd(&ctr->prim_samples, v[1]);
        if (v[2]) atomicAdd(&ctr->hit_rays, v[2]);
        if (v[3]) atomicAdd(&ctr->early_exits, v[3]);
        if (v[4]) atomicAdd(&ctr->saturated, v[4]);
        if (v[5]) atomicAdd(&ctr->refills, v[5]);
        if (v[6]) atomicAdd(&ctr->numeric_fail, v[6]);
    }
}

__device__ __forceinline__ int2 tile_pixel(int tx, int ty, int tid) {
    // warps cover 8x4 pixel blocks (better ray coherence than 16x2 rows)
    const int wid = tid >> 5, lane = tid & 31;
    return make_int2(tx * kTile + (wid & 1) * 8 + (lane & 7), ty * kTile + (wid >> 1) * 4 + (lane >> 3));
}

// ----------------------------------------------------------------------------------------
} // namespace vpb
