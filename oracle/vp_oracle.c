/* TEST INFRASTRUCTURE — the CPU parity oracle. NOT PRODUCT CODE. See vp_oracle.h.
 *
 * Arithmetic contract: binary32 with no contraction (built with -ffp-contract=off, like the
 * reference objects, which contain no vfmadd), the same operation order as the reference's
 * Vec3/Mat3 operators (math.h:36-160), libm expf/sinf/cosf/sqrtf/floorf/ceil. */
#include "vp_oracle.h"

#include <float.h>
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

typedef struct { float x, y, z; } v3;

static v3 mk(float x, float y, float z) { v3 r = {x, y, z}; return r; }
static v3 add3(v3 a, v3 b) { return mk(a.x + b.x, a.y + b.y, a.z + b.z); }
static v3 sub3(v3 a, v3 b) { return mk(a.x - b.x, a.y - b.y, a.z - b.z); }
static v3 scl3(v3 a, float s) { return mk(a.x * s, a.y * s, a.z * s); }
static v3 div3(v3 a, float s) { return mk(a.x / s, a.y / s, a.z / s); }
static v3 cdiv3(v3 a, v3 b) { return mk(a.x / b.x, a.y / b.y, a.z / b.z); }
static float dot3(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static float comp(v3 v, int i) { return i == 0 ? v.x : (i == 1 ? v.y : v.z); }
static v3 ld3(const float *p) { return mk(p[0], p[1], p[2]); }

/* math.h:122-124: col(0)*v.x + col(1)*v.y + col(2)*v.z, column-major m[9]. */
static v3 matvec(const float *m, v3 v) {
    return add3(add3(scl3(mk(m[0], m[1], m[2]), v.x), scl3(mk(m[3], m[4], m[5]), v.y)),
                scl3(mk(m[6], m[7], m[8]), v.z));
}
/* transpose() then operator*(Vec3): column j of R^T is row j of R. */
static v3 matTvec(const float *m, v3 v) {
    return add3(add3(scl3(mk(m[0], m[3], m[6]), v.x), scl3(mk(m[1], m[4], m[7]), v.y)),
                scl3(mk(m[2], m[5], m[8]), v.z));
}
/* math.h:115-121: r(i,c) += a(i,k) * o(k,c), k outer-middle, starting from zero. */
static void matmul(const float *a, const float *o, float *r) {
    float t[9];
    for (int i = 0; i < 9; ++i) t[i] = 0;
    for (int c = 0; c < 3; ++c)
        for (int k = 0; k < 3; ++k)
            for (int i = 0; i < 3; ++i) t[c * 3 + i] += a[k * 3 + i] * o[c * 3 + k];
    memcpy(r, t, sizeof t);
}

/* math.h:141-160 */
static void matinv(const float *m, float *r) {
    const float d = m[0] * (m[4] * m[8] - m[5] * m[7]) - m[3] * (m[1] * m[8] - m[2] * m[7]) +
                    m[6] * (m[1] * m[5] - m[2] * m[4]);
#define A(i, j) m[(j) * 3 + (i)]
#define R(i, j) t[(j) * 3 + (i)]
    float t[9];
    R(0, 0) = A(1, 1) * A(2, 2) - A(1, 2) * A(2, 1);
    R(0, 1) = A(0, 2) * A(2, 1) - A(0, 1) * A(2, 2);
    R(0, 2) = A(0, 1) * A(1, 2) - A(0, 2) * A(1, 1);
    R(1, 0) = A(1, 2) * A(2, 0) - A(1, 0) * A(2, 2);
    R(1, 1) = A(0, 0) * A(2, 2) - A(0, 2) * A(2, 0);
    R(1, 2) = A(0, 2) * A(1, 0) - A(0, 0) * A(1, 2);
    R(2, 0) = A(1, 0) * A(2, 1) - A(1, 1) * A(2, 0);
    R(2, 1) = A(0, 1) * A(2, 0) - A(0, 0) * A(2, 1);
    R(2, 2) = A(0, 0) * A(1, 1) - A(0, 1) * A(1, 0);
#undef A
#undef R
    const float s = 1.0f / d;
    for (int i = 0; i < 9; ++i) r[i] = t[i] * s;
}

/* rotation.cpp:8-28 (Rodrigues, series branch below 1e-4) */
static void rotation_from_axis_angle(v3 v, float *out) {
    static const float I[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    const float t2 = dot3(v, v);
    if (t2 == 0) {
        memcpy(out, I, sizeof I);
        return;
    }
    const float theta = sqrtf(t2);
    float a, b;
    if (theta < 1e-4f) {
        a = 1 - t2 / 6;
        b = 0.5f - t2 / 24;
    } else {
        a = sinf(theta) / theta;
        b = (1 - cosf(theta)) / t2;
    }
    float k[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, kk[9];
    k[3] = -v.z; /* (0,1) */
    k[6] = v.y;  /* (0,2) */
    k[1] = v.z;  /* (1,0) */
    k[7] = -v.x; /* (1,2) */
    k[2] = -v.y; /* (2,0) */
    k[5] = v.x;  /* (2,1) */
    matmul(k, k, kk);
    for (int i = 0; i < 9; ++i) out[i] = (I[i] + k[i] * a) + kk[i] * b;
}

int vpo_compose(int32_t n, const float *tr24, float *xf15) {
    for (int32_t k = 0; k < n; ++k) {
        const float *p = tr24 + 24 * (size_t)k;
        float *o = xf15 + 15 * (size_t)k;
        const v3 s = add3(ld3(p + 12), ld3(p + 21));
        if (s.x <= 0 || s.y <= 0 || s.z <= 0) return 2;
        float r[9];
        rotation_from_axis_angle(ld3(p + 18), r);
        const v3 t = add3(ld3(p + 0), ld3(p + 15));
        o[0] = t.x; o[1] = t.y; o[2] = t.z;
        matmul(r, p + 3, o + 3);
        o[12] = s.x; o[13] = s.y; o[14] = s.z;
    }
    return 0;
}

/* camera.cpp:14-23, camera.h:28 */
void vpo_generate_ray(const float *k9, const float *r9, const float *t3, float px, float py,
                      float *origin, float *dir) {
    float kinv[9];
    matinv(k9, kinv);
    const v3 dirCam = matvec(kinv, mk(px, py, 1));
    const v3 c = matTvec(r9, ld3(t3));
    const v3 d = matTvec(r9, dirCam);
    const v3 n = div3(d, sqrtf(dot3(d, d)));
    origin[0] = -c.x; origin[1] = -c.y; origin[2] = -c.z;
    dir[0] = n.x; dir[1] = n.y; dir[2] = n.z;
}

/* primitive.h:61-63: (R^T (p - t)) ./ s */
static v3 to_model(const float *xf, v3 p) {
    return cdiv3(matTvec(xf + 3, sub3(p, ld3(xf))), ld3(xf + 12));
}

int vpo_intersect_obb(const float *xf, const float *op, const float *dp, float *tEnterOut,
                      float *tExitOut) {
    const v3 om = to_model(xf, ld3(op));
    const v3 dm = cdiv3(matTvec(xf + 3, ld3(dp)), ld3(xf + 12));
    float tEnter = -FLT_MAX, tExit = FLT_MAX;
    for (int a = 0; a < 3; ++a) {
        const float oa = comp(om, a), da = comp(dm, a);
        if (da == 0) {
            if (oa < -1 || oa > 1) return 0;
            continue;
        }
        const float inv = 1 / da;
        const float cNear = da > 0 ? -1.0f : 1.0f;
        const float t1 = (cNear - oa) * inv;
        const float t2 = (-cNear - oa) * inv;
        if (t1 > tEnter) tEnter = t1;
        tExit = t2 < tExit ? t2 : tExit; /* std::min(tExit, t2) */
    }
    if (tEnter < 0) tEnter = 0;
    if (tEnter >= tExit || tExit <= 0) return 0;
    *tEnterOut = tEnter;
    *tExitOut = tExit;
    return 1;
}

typedef struct { int32_t prim; float tEnter, tExit; } seg_t;

static int seg_less(const seg_t *a, const seg_t *b) {
    return a->tEnter != b->tEnter ? a->tEnter < b->tEnter : a->prim < b->prim;
}

/* Insertion sort by (tEnter, prim): the comparator of lbvh.cpp:225-227 (a total order, so
 * any correct sort gives the same list). */
static void sort_segs(seg_t *s, int n) {
    for (int i = 1; i < n; ++i) {
        seg_t x = s[i];
        int j = i;
        while (j > 0 && seg_less(&x, &s[j - 1])) {
            s[j] = s[j - 1];
            --j;
        }
        s[j] = x;
    }
}

static int collect(int32_t n_prim, const float *xf15, v3 o, v3 d, seg_t *out) {
    int n = 0;
    const float op[3] = {o.x, o.y, o.z}, dp[3] = {d.x, d.y, d.z};
    for (int32_t k = 0; k < n_prim; ++k) {
        float te, tx;
        if (vpo_intersect_obb(xf15 + 15 * (size_t)k, op, dp, &te, &tx)) {
            out[n].prim = k;
            out[n].tEnter = te;
            out[n].tExit = tx;
            ++n;
        }
    }
    sort_segs(out, n);
    return n;
}

int32_t vpo_intersect(int32_t n_prim, const float *xf15, const float *o, const float *d,
                      int32_t cap, int32_t *prims, float *tEnter, float *tExit) {
    seg_t *s = (seg_t *)malloc(sizeof(seg_t) * (size_t)(n_prim > 0 ? n_prim : 1));
    const int n = collect(n_prim, xf15, ld3(o), ld3(d), s);
    for (int i = 0; i < n && i < cap; ++i) {
        prims[i] = s[i].prim;
        tEnter[i] = s[i].tEnter;
        tExit[i] = s[i].tExit;
    }
    free(s);
    return n;
}

/* primitive.cpp:12-22 */
static float pow_even(float x, int beta) {
    float r = 1, b = fabsf(x);
    int e = beta;
    while (e > 0) {
        if (e & 1) r *= b;
        b *= b;
        e >>= 1;
    }
    return r;
}

float vpo_window(float x, float y, float z, float alpha, int32_t beta) {
    if (alpha == 0) return 1;
    return expf(-alpha * (pow_even(x, beta) + pow_even(y, beta) + pow_even(z, beta)));
}

/* primitive.cpp:51-69 */
typedef struct { int lo[3]; float frac[3]; } stencil_t;
static stencil_t trilinear_stencil(int m, v3 p) {
    stencil_t st;
    for (int a = 0; a < 3; ++a) {
        float u = (comp(p, a) + 1) * 0.5f * (float)m - 0.5f;
        if (u <= 0) u = 0;
        else if (u >= (float)(m - 1)) u = (float)(m - 1);
        int i0 = (int)floorf(u);
        if (i0 > m - 2) i0 = (m - 2) > 0 ? (m - 2) : 0;
        st.lo[a] = i0;
        st.frac[a] = m > 1 ? u - (float)i0 : 0;
    }
    return st;
}

/* primitive.cpp:71-90 (cornerWeight + gatherChannel) on the planar slab, primitive.h:36-39 */
static float gather_channel(const float *payload, int m, int k, int ch, const stencil_t *st) {
    float acc = 0;
    for (int cz = 0; cz < 2; ++cz)
        for (int cy = 0; cy < 2; ++cy)
            for (int cx = 0; cx < 2; ++cx) {
                const int z = st->lo[2] + cz < m - 1 ? st->lo[2] + cz : m - 1;
                const int y = st->lo[1] + cy < m - 1 ? st->lo[1] + cy : m - 1;
                const int x = st->lo[0] + cx < m - 1 ? st->lo[0] + cx : m - 1;
                const float wx = cx ? st->frac[0] : 1 - st->frac[0];
                const float wy = cy ? st->frac[1] : 1 - st->frac[1];
                const float wz = cz ? st->frac[2] : 1 - st->frac[2];
                const size_t mm = (size_t)m;
                const size_t idx = ((((size_t)k * 4 + ch) * mm + z) * mm + y) * mm + x;
                acc += wx * wy * wz * payload[idx];
            }
    return acc;
}

static float clampc(float v) {
    /* cwiseMax(Vec3(-1), cwiseMin(Vec3(1), p)) with std::min/std::max semantics */
    const float lo = v < 1 ? v : 1;
    return -1 < lo ? lo : -1;
}

static uint64_t hash_combine(uint64_t seed, uint64_t value) { /* math.h:170-175 */
    uint64_t z = seed + 0x9e3779b97f4a7c15ull + value;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
static float hash_to_unit(uint64_t h) { /* math.h:177-179 */
    return (float)(h >> 11) * (float)(1.0 / 9007199254740992.0);
}

typedef struct {
    int32_t n_prim, m;
    const float *xf15, *payload;
    float w_alpha;
    int32_t w_beta;
    float step, early_eps;
    uint64_t perm;
} march_ctx;

/* MarchResult replay bookkeeping (march.h:22-33) consumed by the backward pass. */
typedef struct {
    int64_t lastStep;
    int saturated;
    float satTPrev, satSigmaSum, satRgbWeighted[3];
} march_rec;

/* march.cpp:18-93 */
/* prim (nullable) receives the number of primitive evaluations, the executions of the body of
 * march.cpp:63-70 (SURVEY.md §8d "prim-samples"). */
static void march_one_counted(const march_ctx *c, v3 o, v3 d, const seg_t *segs, int nSegs, int *active,
                              float jitter01, float *rgb, float *alpha, int32_t *samples, march_rec *rec,
                              int32_t *prim) {
    int32_t nprim = 0;
    if (rec) {
        rec->lastStep = -1;
        rec->saturated = 0;
        rec->satTPrev = rec->satSigmaSum = 0;
        rec->satRgbWeighted[0] = rec->satRgbWeighted[1] = rec->satRgbWeighted[2] = 0;
    }
    float color[3] = {0, 0, 0};
    float transmittance = 0;
    int nsamp = 0;
    if (nSegs > 0) {
        const float dt = c->step;
        const float t0 = segs[0].tEnter;
        float tMax = 0;
        for (int s = 0; s < nSegs; ++s) tMax = tMax < segs[s].tExit ? segs[s].tExit : tMax;
        int nActive = 0, next = 0;
        for (int64_t i = 0;; ++i) {
            const float ts = t0 + ((float)i + jitter01) * dt;
            if (ts >= tMax) break;
            while (next < nSegs && segs[next].tEnter <= ts) active[nActive++] = next++;
            int w = 0;
            for (int a = 0; a < nActive; ++a)
                if (!(segs[active[a]].tExit <= ts)) active[w++] = active[a];
            nActive = w;
            if (nActive == 0) {
                if (next >= nSegs) break;
                const float tNext = segs[next].tEnter;
                const int64_t skipTo = (int64_t)ceil((double)((tNext - t0) / dt) - (double)jitter01);
                if (skipTo > i + 1) i = skipTo - 1;
                continue;
            }
            if (c->perm != 0) {
                for (size_t a = (size_t)nActive; a > 1; --a) {
                    const uint64_t h = hash_combine(c->perm, (uint64_t)i * 1315423911u + a);
                    const int j = (int)(h % a);
                    const int tmp = active[a - 1];
                    active[a - 1] = active[j];
                    active[j] = tmp;
                }
            }
            const v3 pw = add3(o, scl3(d, ts));
            float sigmaSum = 0;
            float rw[3] = {0, 0, 0};
            for (int a = 0; a < nActive; ++a) {
                const int k = segs[active[a]].prim;
                const v3 q = to_model(c->xf15 + 15 * (size_t)k, pw);
                const v3 pm = mk(clampc(q.x), clampc(q.y), clampc(q.z));
                const stencil_t st = trilinear_stencil(c->m, pm);
                const float sigma = gather_channel(c->payload, c->m, k, 3, &st) *
                                    vpo_window(pm.x, pm.y, pm.z, c->w_alpha, c->w_beta);
                sigmaSum += sigma;
                const float r0 = gather_channel(c->payload, c->m, k, 0, &st);
                const float r1 = gather_channel(c->payload, c->m, k, 1, &st);
                const float r2 = gather_channel(c->payload, c->m, k, 2, &st);
                rw[0] += r0 * sigma;
                rw[1] += r1 * sigma;
                rw[2] += r2 * sigma;
            }
            ++nsamp;
            nprim += nActive;
            if (rec) rec->lastStep = i;
            const float dT = sigmaSum * dt;
            if (transmittance + dT >= 1) {
                const float frac = (1 - transmittance) / dT;
                const float f = dt * frac;
                for (int ch = 0; ch < 3; ++ch) color[ch] += rw[ch] * f;
                if (rec) {
                    rec->satTPrev = transmittance;
                    rec->satSigmaSum = sigmaSum;
                    for (int ch = 0; ch < 3; ++ch) rec->satRgbWeighted[ch] = rw[ch];
                    rec->saturated = 1;
                }
                transmittance = 1;
                break;
            }
            for (int ch = 0; ch < 3; ++ch) color[ch] += rw[ch] * dt;
            transmittance += dT;
            if (transmittance > 1 - c->early_eps) break;
        }
    }
    rgb[0] = color[0];
    rgb[1] = color[1];
    rgb[2] = color[2];
    *alpha = transmittance;
    *samples = nsamp;
    if (prim) *prim = nprim;
}

static void march_one(const march_ctx *c, v3 o, v3 d, const seg_t *segs, int nSegs, int *active,
                      float jitter01, float *rgb, float *alpha, int32_t *samples, march_rec *rec) {
    march_one_counted(c, o, d, segs, nSegs, active, jitter01, rgb, alpha, samples, rec, NULL);
}

int vpo_march_rays(int32_t n_prim, int32_t m, const float *xf15, const float *payload,
                   float w_alpha, int32_t w_beta, int64_t n_rays, const float *origins,
                   const float *dirs, const float *jitter01, float step, float early_eps,
                   uint64_t perm, float *rgb, float *alpha, int32_t *samples) {
    const march_ctx c = {n_prim, m, xf15, payload, w_alpha, w_beta, step, early_eps, perm};
    const size_t cap = (size_t)(n_prim > 0 ? n_prim : 1);
    seg_t *segs = (seg_t *)malloc(sizeof(seg_t) * cap);
    int *active = (int *)malloc(sizeof(int) * cap);
    for (int64_t r = 0; r < n_rays; ++r) {
        const v3 o = ld3(origins + 3 * r), d = ld3(dirs + 3 * r);
        const int n = collect(n_prim, xf15, o, d, segs);
        march_one(&c, o, d, segs, n, active, jitter01 ? jitter01[r] : 0.5f, rgb + 3 * r,
                  alpha + r, samples + r, NULL);
    }
    free(segs);
    free(active);
    return 0;
}

typedef struct {
    const march_ctx *c;
    const float *k9, *r9, *t3;
    int32_t width, height, jitter;
    uint64_t seed;
    int64_t y0, y1;
    float *rgb, *alpha;
    int32_t *samples, *prim;
} render_job;

static void *render_rows(void *arg) {
    const render_job *j = (const render_job *)arg;
    const size_t cap = (size_t)(j->c->n_prim > 0 ? j->c->n_prim : 1);
    seg_t *segs = (seg_t *)malloc(sizeof(seg_t) * cap);
    int *active = (int *)malloc(sizeof(int) * cap);
    for (int64_t y = j->y0; y < j->y1; ++y)
        for (int x = 0; x < j->width; ++x) {
            const int pixelId = (int)y * j->width + x;
            float o[3], d[3];
            vpo_generate_ray(j->k9, j->r9, j->t3, (float)x + 0.5f, (float)y + 0.5f, o, d);
            const int n = collect(j->c->n_prim, j->c->xf15, ld3(o), ld3(d), segs);
            const float jit = j->jitter ? hash_to_unit(hash_combine(j->seed, (uint64_t)pixelId)) : 0.5f;
            march_one_counted(j->c, ld3(o), ld3(d), segs, n, active, jit, j->rgb + 3 * (size_t)pixelId,
                              j->alpha + pixelId, j->samples + pixelId, NULL,
                              j->prim ? j->prim + pixelId : NULL);
        }
    free(segs);
    free(active);
    return NULL;
}

/* vpo_render plus the per-pixel prim-sample counts (nullable). */
int vpo_render_counted(int32_t n_prim, int32_t m, const float *xf15, const float *payload, float w_alpha,
                       int32_t w_beta, const float *k9, const float *r9, const float *t3, int32_t width,
                       int32_t height, float step, float early_eps, int32_t jitter, uint64_t seed,
                       uint64_t perm, float *rgb, float *alpha, int32_t *samples, int32_t *prim,
                       int32_t n_threads) {
    const size_t np = (size_t)width * (size_t)height;
    memset(rgb, 0, np * 3 * sizeof(float));
    memset(alpha, 0, np * sizeof(float));
    memset(samples, 0, np * sizeof(int32_t));
    if (prim) memset(prim, 0, np * sizeof(int32_t));
    if (n_prim == 0 || np == 0) return 0; /* march.cpp:108 */
    const march_ctx c = {n_prim, m, xf15, payload, w_alpha, w_beta, step, early_eps, perm};
    if (n_threads <= 1) n_threads = 1;
    if (n_threads > height) n_threads = height;
    pthread_t th[256];
    render_job jobs[256];
    if (n_threads > 256) n_threads = 256;
    const int64_t chunk = (height + n_threads - 1) / n_threads;
    int started = 0;
    for (int w = 0; w < n_threads; ++w) {
        render_job j = {&c, k9, r9, t3, width, height, jitter, seed, w * chunk,
                        (w + 1) * chunk < height ? (w + 1) * chunk : height, rgb, alpha, samples, prim};
        if (j.y0 >= j.y1) break;
        jobs[w] = j;
        pthread_create(&th[w], NULL, render_rows, &jobs[w]);
        ++started;
    }
    for (int w = 0; w < started; ++w) pthread_join(th[w], NULL);
    return 0;
}

int vpo_render(int32_t n_prim, int32_t m, const float *xf15, const float *payload, float w_alpha,
               int32_t w_beta, const float *k9, const float *r9, const float *t3, int32_t width,
               int32_t height, float step, float early_eps, int32_t jitter, uint64_t seed,
               uint64_t perm, float *rgb, float *alpha, int32_t *samples, int32_t n_threads) {
    return vpo_render_counted(n_prim, m, xf15, payload, w_alpha, w_beta, k9, r9, t3, width, height, step,
                              early_eps, jitter, seed, perm, rgb, alpha, samples, NULL, n_threads);
}

void vpo_composite(int32_t width, int32_t height, const float *rgb, const float *alpha,
                   const float *bg, float *out) {
    for (int64_t p = 0; p < (int64_t)width * height; ++p) {
        const float a = alpha[p];
        for (int ch = 0; ch < 3; ++ch) out[3 * p + ch] = a * rgb[3 * p + ch] + (1 - a) * bg[3 * p + ch];
    }
}

/* ---------------------------------------------------------------------------------------
 * Backward pass restatement: backwardRay (grad.cpp:34-195) over a batch of rays with given
 * output adjoints. Gradients accumulate (+=) into the reference's GradBuffer layout
 * (params.h:12-27): payload K*4*M^3 planar, then per primitive deltaT[3] deltaR[3] deltaS[3].
 */
static v3 cross3(v3 a, v3 b) {
    return mk(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}

/* rotation.cpp:30-38 */
static void rotation_derivative(v3 v, int i, float *out) {
    const float t2 = dot3(v, v);
    float e[3] = {0, 0, 0};
    e[i] = 1;
    float sk[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    if (t2 < 1e-14f) { /* skew(e) */
        sk[3] = -e[2]; sk[6] = e[1]; sk[1] = e[2]; sk[7] = -e[0]; sk[2] = -e[1]; sk[5] = e[0];
        memcpy(out, sk, sizeof sk);
        return;
    }
    float r[9], imr[9], a[9], b[9], c[9];
    static const float I[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    rotation_from_axis_angle(v, r);
    for (int q = 0; q < 9; ++q) imr[q] = I[q] - r[q];
    const v3 w = cross3(v, matvec(imr, mk(e[0], e[1], e[2])));
    const float vi = comp(v, i);
    float skv[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, skw[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    skv[3] = -v.z; skv[6] = v.y; skv[1] = v.z; skv[7] = -v.x; skv[2] = -v.y; skv[5] = v.x;
    skw[3] = -w.z; skw[6] = w.y; skw[1] = w.z; skw[7] = -w.x; skw[2] = -w.y; skw[5] = w.x;
    const float s = 1 / t2;
    for (int q = 0; q < 9; ++q) a[q] = skv[q] * vi;
    for (int q = 0; q < 9; ++q) b[q] = a[q] + skw[q];
    for (int q = 0; q < 9; ++q) c[q] = b[q] * s;
    matmul(c, r, out);
}

/* primitive.cpp:30-39 */
static v3 window_gradient(v3 p, float alpha, int beta) {
    if (alpha == 0) return mk(0, 0, 0);
    const float wv = vpo_window(p.x, p.y, p.z, alpha, beta);
    const float c = -alpha * (float)beta * wv;
    return mk(c * (pow_even(p.x, beta - 2) * p.x), c * (pow_even(p.y, beta - 2) * p.y),
              c * (pow_even(p.z, beta - 2) * p.z));
}

typedef struct { int lo[3]; float frac[3]; int clamped[3]; } stencil2_t;
static stencil2_t trilinear_stencil2(int m, v3 p) { /* primitive.cpp:51-69 with clamped[] */
    stencil2_t st;
    for (int a = 0; a < 3; ++a) {
        float u = (comp(p, a) + 1) * 0.5f * (float)m - 0.5f;
        st.clamped[a] = 0;
        if (u <= 0) { u = 0; st.clamped[a] = 1; }
        else if (u >= (float)(m - 1)) { u = (float)(m - 1); st.clamped[a] = 1; }
        int i0 = (int)floorf(u);
        if (i0 > m - 2) i0 = (m - 2) > 0 ? (m - 2) : 0;
        st.lo[a] = i0;
        st.frac[a] = m > 1 ? u - (float)i0 : 0;
    }
    return st;
}

static size_t slab_index(int m, int k, int ch, int z, int y, int x) {
    const size_t mm = (size_t)m;
    return ((((size_t)k * 4 + ch) * mm + z) * mm + y) * mm + x;
}

/* primitive.cpp:101-127 */
static v3 stencil_gradient(const float *payload, int m, int k, const stencil2_t *st, int ch) {
    float g[3] = {0, 0, 0};
    if (m == 1) return mk(0, 0, 0);
    for (int cz = 0; cz < 2; ++cz)
        for (int cy = 0; cy < 2; ++cy)
            for (int cx = 0; cx < 2; ++cx) {
                const int z = st->lo[2] + cz < m - 1 ? st->lo[2] + cz : m - 1;
                const int y = st->lo[1] + cy < m - 1 ? st->lo[1] + cy : m - 1;
                const int x = st->lo[0] + cx < m - 1 ? st->lo[0] + cx : m - 1;
                const float v = payload[slab_index(m, k, ch, z, y, x)];
                const float wx = cx ? st->frac[0] : 1 - st->frac[0];
                const float wy = cy ? st->frac[1] : 1 - st->frac[1];
                const float wz = cz ? st->frac[2] : 1 - st->frac[2];
                const float dx = cx ? 1.0f : -1.0f, dy = cy ? 1.0f : -1.0f, dz = cz ? 1.0f : -1.0f;
                g[0] += dx * wy * wz * v;
                g[1] += wx * dy * wz * v;
                g[2] += wx * wy * dz * v;
            }
    const float s = 0.5f * (float)m;
    for (int a = 0; a < 3; ++a)
        if (st->clamped[a]) g[a] = 0;
    return mk(g[0] * s, g[1] * s, g[2] * s);
}

/* lbvh.cpp:177-205 with the entry face (entryAxis, entrySign, enterClamped) */
static int intersect_obb_face(const float *xf, v3 o, v3 d, int *axis, int *sign, int *clamped) {
    const v3 om = to_model(xf, o);
    const v3 dm = cdiv3(matTvec(xf + 3, d), ld3(xf + 12));
    float tEnter = -FLT_MAX, tExit = FLT_MAX;
    *axis = -1;
    *sign = 0;
    for (int a = 0; a < 3; ++a) {
        const float oa = comp(om, a), da = comp(dm, a);
        if (da == 0) {
            if (oa < -1 || oa > 1) return 0;
            continue;
        }
        const float inv = 1 / da;
        const float cNear = da > 0 ? -1.0f : 1.0f;
        const float t1 = (cNear - oa) * inv;
        const float t2 = (-cNear - oa) * inv;
        if (t1 > tEnter) {
            tEnter = t1;
            *axis = a;
            *sign = (int)cNear;
        }
        tExit = t2 < tExit ? t2 : tExit;
    }
    *clamped = tEnter < 0;
    if (*clamped) tEnter = 0;
    if (tEnter >= tExit || tExit <= 0) return 0;
    return 1;
}

static void gadd3(float *g, v3 v) {
    g[0] += v.x;
    g[1] += v.y;
    g[2] += v.z;
}

typedef struct {
    int prim;
    v3 pModel;
    int cube[3];
    stencil2_t st;
    float sigmaRaw, win;
    v3 rgb;
} prim_sample_t;

int vpo_backward_rays(int32_t n_prim, int32_t m, const float *tr24, const float *xf15,
                      const float *payload, float w_alpha, int32_t w_beta, int64_t n_rays,
                      const float *origins, const float *dirs, const float *jitter01,
                      const float *adj_rgb, const float *adj_alpha, float step, float early_eps,
                      float *grads) {
    const march_ctx mc = {n_prim, m, xf15, payload, w_alpha, w_beta, step, early_eps, 0};
    const size_t cap = (size_t)(n_prim > 0 ? n_prim : 1);
    seg_t *segs = (seg_t *)malloc(sizeof(seg_t) * cap);
    int *active = (int *)malloc(sizeof(int) * cap);
    prim_sample_t *ps = (prim_sample_t *)malloc(sizeof(prim_sample_t) * cap);
    float *rotd = (float *)malloc(sizeof(float) * 27 * cap);
    int *rot_ready = (int *)calloc(cap, sizeof(int));
    float *gdelta = grads + (size_t)n_prim * 4 * m * m * m;
    for (int64_t r = 0; r < n_rays; ++r) {
        const v3 o = ld3(origins + 3 * r), d = ld3(dirs + 3 * r);
        const float jit = jitter01 ? jitter01[r] : 0.5f;
        const v3 aRgb = ld3(adj_rgb + 3 * r);
        const float aAlpha = adj_alpha[r];
        const int nSegs = collect(n_prim, xf15, o, d, segs);
        if (nSegs == 0) continue;
        march_rec fwd;
        float frgb[3], falpha;
        int32_t fs;
        march_one(&mc, o, d, segs, nSegs, active, jit, frgb, &falpha, &fs, &fwd);
        if (fwd.lastStep < 0) continue;
        /* rotDerivs cache is per backwardRay call (grad.cpp:46-54) */
        memset(rot_ready, 0, sizeof(int) * cap);
        const float dt = step;
        const float t0 = segs[0].tEnter;
        float tMax = 0;
        for (int s = 0; s < nSegs; ++s) tMax = tMax < segs[s].tExit ? segs[s].tExit : tMax;
        int nActive = 0, next = 0;
        float gTmin = 0;
        for (int64_t i = 0; i <= fwd.lastStep; ++i) {
            const float ts = t0 + ((float)i + jit) * dt;
            if (ts >= tMax) break;
            while (next < nSegs && segs[next].tEnter <= ts) active[nActive++] = next++;
            int w = 0;
            for (int a = 0; a < nActive; ++a)
                if (!(segs[active[a]].tExit <= ts)) active[w++] = active[a];
            nActive = w;
            if (nActive == 0) {
                if (next >= nSegs) break;
                const float tNext = segs[next].tEnter;
                const int64_t skipTo = (int64_t)ceil((double)((tNext - t0) / dt) - (double)jit);
                if (skipTo > i + 1) i = skipTo - 1;
                continue;
            }
            const v3 pWorld = add3(o, scl3(d, ts));
            float sigmaSum = 0;
            v3 rgbW = mk(0, 0, 0);
            for (int a = 0; a < nActive; ++a) {
                prim_sample_t *p = &ps[a];
                p->prim = segs[active[a]].prim;
                const v3 raw = to_model(xf15 + 15 * (size_t)p->prim, pWorld);
                for (int q = 0; q < 3; ++q) p->cube[q] = comp(raw, q) <= -1 || comp(raw, q) >= 1;
                p->pModel = mk(clampc(raw.x), clampc(raw.y), clampc(raw.z));
                p->st = trilinear_stencil2(m, p->pModel);
                const stencil_t st1 = {{p->st.lo[0], p->st.lo[1], p->st.lo[2]},
                                       {p->st.frac[0], p->st.frac[1], p->st.frac[2]}};
                p->sigmaRaw = gather_channel(payload, m, p->prim, 3, &st1);
                p->win = vpo_window(p->pModel.x, p->pModel.y, p->pModel.z, w_alpha, w_beta);
                p->rgb = mk(gather_channel(payload, m, p->prim, 0, &st1),
                            gather_channel(payload, m, p->prim, 1, &st1),
                            gather_channel(payload, m, p->prim, 2, &st1));
                sigmaSum += p->sigmaRaw * p->win;
                rgbW = add3(rgbW, scl3(p->rgb, p->sigmaRaw * p->win));
            }
            (void)sigmaSum;
            const int satStep = fwd.saturated && i == fwd.lastStep;
            v3 gPWorldStep = mk(0, 0, 0);
            for (int a = 0; a < nActive; ++a) {
                const prim_sample_t *p = &ps[a];
                const int k = p->prim;
                const float sigmaW = p->sigmaRaw * p->win;
                v3 gRgb;
                float gSigmaW;
                if (satStep) {
                    const float budget = 1 - fwd.satTPrev;
                    const float inv = 1 / fwd.satSigmaSum;
                    gRgb = scl3(aRgb, sigmaW * budget * inv);
                    gSigmaW = dot3(aRgb, sub3(scl3(p->rgb, fwd.satSigmaSum), rgbW)) * budget * inv * inv;
                } else {
                    gRgb = scl3(aRgb, sigmaW * dt);
                    gSigmaW = dot3(aRgb, p->rgb) * dt;
                    if (fwd.saturated)
                        gSigmaW -= dot3(aRgb, ld3(fwd.satRgbWeighted)) / fwd.satSigmaSum * dt;
                    else
                        gSigmaW += aAlpha * dt;
                }
                for (int cz = 0; cz < 2; ++cz)
                    for (int cy = 0; cy < 2; ++cy)
                        for (int cx = 0; cx < 2; ++cx) {
                            const float wx = cx ? p->st.frac[0] : 1 - p->st.frac[0];
                            const float wy = cy ? p->st.frac[1] : 1 - p->st.frac[1];
                            const float wz = cz ? p->st.frac[2] : 1 - p->st.frac[2];
                            const float wgt = wx * wy * wz;
                            if (wgt == 0) continue;
                            const int z = p->st.lo[2] + cz < m - 1 ? p->st.lo[2] + cz : m - 1;
                            const int y = p->st.lo[1] + cy < m - 1 ? p->st.lo[1] + cy : m - 1;
                            const int x = p->st.lo[0] + cx < m - 1 ? p->st.lo[0] + cx : m - 1;
                            for (int ch = 0; ch < 3; ++ch)
                                grads[slab_index(m, k, ch, z, y, x)] += comp(gRgb, ch) * wgt;
                            grads[slab_index(m, k, 3, z, y, x)] += gSigmaW * p->win * wgt;
                        }
                const v3 gradSigmaTri = stencil_gradient(payload, m, k, &p->st, 3);
                const v3 gradW = window_gradient(p->pModel, w_alpha, w_beta);
                v3 gP = scl3(add3(scl3(gradSigmaTri, p->win), scl3(gradW, p->sigmaRaw)), gSigmaW);
                for (int ch = 0; ch < 3; ++ch)
                    gP = add3(gP, scl3(stencil_gradient(payload, m, k, &p->st, ch), comp(gRgb, ch)));
                if (p->cube[0]) gP.x = 0;
                if (p->cube[1]) gP.y = 0;
                if (p->cube[2]) gP.z = 0;
                if (gP.x == 0 && gP.y == 0 && gP.z == 0) continue;
                const float *xf = xf15 + 15 * (size_t)k;
                const v3 gOverS = cdiv3(gP, ld3(xf + 12));
                const v3 rotG = matvec(xf + 3, gOverS);
                float *gk = gdelta + 9 * (size_t)k;
                gadd3(gk + 0, mk(-rotG.x, -rotG.y, -rotG.z));
                gadd3(gk + 6, mk(-gP.x * p->pModel.x / xf[12], -gP.y * p->pModel.y / xf[13],
                                -gP.z * p->pModel.z / xf[14]));
                const v3 u = sub3(pWorld, ld3(xf));
                const v3 vv = matvec(tr24 + 24 * (size_t)k + 3, gOverS);
                if (!rot_ready[k]) {
                    for (int q = 0; q < 3; ++q)
                        rotation_derivative(ld3(tr24 + 24 * (size_t)k + 18), q, rotd + 27 * (size_t)k + 9 * q);
                    rot_ready[k] = 1;
                }
                const float *rd = rotd + 27 * (size_t)k;
                gadd3(gk + 3, mk(dot3(matvec(rd, vv), u), dot3(matvec(rd + 9, vv), u),
                                dot3(matvec(rd + 18, vv), u)));
                gPWorldStep = add3(gPWorldStep, rotG);
            }
            gTmin += dot3(gPWorldStep, d);
        }
        if (gTmin != 0) { /* t_min anchor chain, grad.cpp:166-194 */
            const int k0 = segs[0].prim;
            const float *xf = xf15 + 15 * (size_t)k0;
            int axis, sign, clamped;
            if (intersect_obb_face(xf, o, d, &axis, &sign, &clamped) && !clamped) {
                const int j = axis;
                const float c = (float)sign;
                const v3 q = mk(xf[3 + 3 * j], xf[4 + 3 * j], xf[5 + 3 * j]);
                const float qd = dot3(q, d);
                if (qd != 0) {
                    const float tStar = t0;
                    float *gk = gdelta + 9 * (size_t)k0;
                    gadd3(gk + 0, scl3(q, gTmin / qd));
                    float gS[3] = {0, 0, 0};
                    gS[j] = gTmin * c / qd;
                    gadd3(gk + 6, mk(gS[0], gS[1], gS[2]));
                    const v3 toT = sub3(ld3(xf), o);
                    const float *rb = tr24 + 24 * (size_t)k0 + 3;
                    const v3 rj = mk(rb[3 * j], rb[3 * j + 1], rb[3 * j + 2]);
                    if (!rot_ready[k0]) {
                        for (int qq = 0; qq < 3; ++qq)
                            rotation_derivative(ld3(tr24 + 24 * (size_t)k0 + 18), qq, rotd + 27 * (size_t)k0 + 9 * qq);
                        rot_ready[k0] = 1;
                    }
                    float gR[3];
                    for (int ii = 0; ii < 3; ++ii) {
                        const v3 qp = matvec(rotd + 27 * (size_t)k0 + 9 * ii, rj);
                        gR[ii] = gTmin * (dot3(qp, toT) - tStar * dot3(qp, d)) / qd;
                    }
                    gadd3(gk + 3, mk(gR[0], gR[1], gR[2]));
                }
            }
        }
    }
    free(segs);
    free(active);
    free(ps);
    free(rotd);
    free(rot_ready);
    return 0;
}

/* ---------------------------------------------------------------------------------------
 * Tile binning restatement (no reference counterpart; replaces lbvh.cpp:13-156).
 * Identical float operation sequence to k_cull in paper_2103_01954_b200/csrc/vpb_kernels.cu.
 */
static void cull_one(const float *xf, const float *k9, const float *r9, const float *t3,
                     int32_t width, int32_t height, int32_t *rect, int32_t *prect, uint32_t *key) {
    const v3 s = ld3(xf + 12);
    const float r = sqrtf(dot3(s, s));
    const float rr = r * 1.001f + 1e-6f;
    const v3 cc = add3(matvec(r9, ld3(xf)), ld3(t3));
    const float dist = sqrtf(dot3(cc, cc));
    float depth = dist - rr;
    if (!(depth > 0)) depth = 0;
    uint32_t kb;
    memcpy(&kb, &depth, 4);
    *key = kb;
    const int32_t tiles_x = (width + VPO_TILE - 1) / VPO_TILE;
    const int32_t tiles_y = (height + VPO_TILE - 1) / VPO_TILE;
    rect[0] = 0; rect[1] = 0; rect[2] = -1; rect[3] = -1;
    prect[0] = 0; prect[1] = 0; prect[2] = -1; prect[3] = -1;
    if (width <= 0 || height <= 0) return;
    if (cc.z + rr < 0) return; /* entirely behind the camera plane */
    if (cc.z - rr <= 1e-3f * rr) { /* straddles or hugs the camera plane: every tile */
        rect[2] = tiles_x - 1;
        rect[3] = tiles_y - 1;
        prect[2] = width - 1;
        prect[3] = height - 1;
        return;
    }
    float umin = FLT_MAX, umax = -FLT_MAX, vmin = FLT_MAX, vmax = -FLT_MAX;
    for (int c = 0; c < 8; ++c) {
        const v3 corner = mk(c & 1 ? 1.0f : -1.0f, c & 2 ? 1.0f : -1.0f, c & 4 ? 1.0f : -1.0f);
        const v3 pw = add3(ld3(xf), matvec(xf + 3, mk(s.x * corner.x, s.y * corner.y, s.z * corner.z)));
        const v3 pc = add3(matvec(r9, pw), ld3(t3));
        const v3 hp = matvec(k9, pc);
        const float u = hp.x / hp.z, v = hp.y / hp.z;
        umin = u < umin ? u : umin;
        umax = u > umax ? u : umax;
        vmin = v < vmin ? v : vmin;
        vmax = v > vmax ? v : vmax;
    }
    const float mu = 2.0f + 1e-3f * (fabsf(umin) + fabsf(umax));
    const float mv = 2.0f + 1e-3f * (fabsf(vmin) + fabsf(vmax));
    float x0 = floorf(umin - mu), x1 = floorf(umax + mu);
    float y0 = floorf(vmin - mv), y1 = floorf(vmax + mv);
    const float wl = (float)(width - 1), hl = (float)(height - 1);
    if (!(x1 >= 0) || !(x0 <= wl) || !(y1 >= 0) || !(y0 <= hl)) return;
    x0 = x0 > 0 ? x0 : 0;
    y0 = y0 > 0 ? y0 : 0;
    x1 = x1 < wl ? x1 : wl;
    y1 = y1 < hl ? y1 : hl;
    prect[0] = (int32_t)x0;
    prect[1] = (int32_t)y0;
    prect[2] = (int32_t)x1;
    prect[3] = (int32_t)y1;
    rect[0] = prect[0] / VPO_TILE;
    rect[1] = prect[1] / VPO_TILE;
    rect[2] = prect[2] / VPO_TILE;
    rect[3] = prect[3] / VPO_TILE;
}

void vpo_cull(int32_t n_prim, const float *xf15, const float *k9, const float *r9,
              const float *t3, int32_t width, int32_t height, int32_t *rect4,
              uint32_t *depth_key) {
    vpo_cull_px(n_prim, xf15, k9, r9, t3, width, height, rect4, NULL, depth_key);
}

void vpo_cull_px(int32_t n_prim, const float *xf15, const float *k9, const float *r9,
                 const float *t3, int32_t width, int32_t height, int32_t *rect4, int32_t *prect4,
                 uint32_t *depth_key) {
    for (int32_t k = 0; k < n_prim; ++k) {
        int32_t pr[4];
        cull_one(xf15 + 15 * (size_t)k, k9, r9, t3, width, height, rect4 + 4 * (size_t)k, pr,
                 depth_key + k);
        if (prect4) memcpy(prect4 + 4 * (size_t)k, pr, sizeof pr);
    }
}

static int cmp_u64(const void *a, const void *b) {
    const uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

int64_t vpo_tile_lists(int32_t n_prim, const float *xf15, const float *k9, const float *r9,
                       const float *t3, int32_t width, int32_t height, int32_t *tile_offsets,
                       int32_t *tile_prims, int64_t cap) {
    const int32_t tiles_x = (width + VPO_TILE - 1) / VPO_TILE;
    const int32_t tiles_y = (height + VPO_TILE - 1) / VPO_TILE;
    const int64_t n_tiles = (int64_t)tiles_x * tiles_y;
    int32_t *rect = (int32_t *)malloc(sizeof(int32_t) * 4 * (size_t)(n_prim > 0 ? n_prim : 1));
    uint32_t *key = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(n_prim > 0 ? n_prim : 1));
    vpo_cull(n_prim, xf15, k9, r9, t3, width, height, rect, key);
    int64_t *count = (int64_t *)calloc((size_t)(n_tiles + 1), sizeof(int64_t));
    for (int32_t k = 0; k < n_prim; ++k)
        for (int32_t ty = rect[4 * k + 1]; ty <= rect[4 * k + 3]; ++ty)
            for (int32_t tx = rect[4 * k + 0]; tx <= rect[4 * k + 2]; ++tx)
                count[(int64_t)ty * tiles_x + tx]++;
    int64_t total = 0;
    for (int64_t t = 0; t < n_tiles; ++t) {
        tile_offsets[t] = (int32_t)total;
        total += count[t];
    }
    tile_offsets[n_tiles] = (int32_t)total;
    uint64_t *ent = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(total > 0 ? total : 1));
    int64_t *cur = (int64_t *)calloc((size_t)(n_tiles + 1), sizeof(int64_t));
    for (int32_t k = 0; k < n_prim; ++k)
        for (int32_t ty = rect[4 * k + 1]; ty <= rect[4 * k + 3]; ++ty)
            for (int32_t tx = rect[4 * k + 0]; tx <= rect[4 * k + 2]; ++tx) {
                const int64_t t = (int64_t)ty * tiles_x + tx;
                ent[tile_offsets[t] + cur[t]++] = ((uint64_t)key[k] << 32) | (uint32_t)k;
            }
    for (int64_t t = 0; t < n_tiles; ++t)
        qsort(ent + tile_offsets[t], (size_t)count[t], sizeof(uint64_t), cmp_u64);
    for (int64_t i = 0; i < total && i < cap; ++i) tile_prims[i] = (int32_t)(ent[i] & 0xffffffffu);
    free(rect);
    free(key);
    free(count);
    free(ent);
    free(cur);
    return total;
}

/* ---------------------------------------------------------------------------------------
 * C port of glibc 2.39 expf (sysdeps/ieee754/flt-32/e_expf.c, the ARM optimized-routines
 * algorithm: 32-entry 2^(i/32) table, cubic in double) as ported to the device in
 * paper_2103_01954_b200/csrc/vpb_device.cuh. Tests compare it with libm expf. */
static const uint64_t kExp2fTab[32] = {
    0x3ff0000000000000ULL, 0x3fefd9b0d3158574ULL, 0x3fefb5586cf9890fULL, 0x3fef9301d0125b51ULL,
    0x3fef72b83c7d517bULL, 0x3fef54873168b9aaULL, 0x3fef387a6e756238ULL, 0x3fef1e9df51fdee1ULL,
    0x3fef06fe0a31b715ULL, 0x3feef1a7373aa9cbULL, 0x3feedea64c123422ULL, 0x3feece086061892dULL,
    0x3feebfdad5362a27ULL, 0x3feeb42b569d4f82ULL, 0x3feeab07dd485429ULL, 0x3feea47eb03a5585ULL,
    0x3feea09e667f3bcdULL, 0x3fee9f75e8ec5f74ULL, 0x3feea11473eb0187ULL, 0x3feea589994cce13ULL,
    0x3feeace5422aa0dbULL, 0x3feeb737b0cdc5e5ULL, 0x3feec49182a3f090ULL, 0x3feed503b23e255dULL,
    0x3feee89f995ad3adULL, 0x3feeff76f2fb5e47ULL, 0x3fef199bdd85529cULL, 0x3fef3720dcef9069ULL,
    0x3fef5818dcfba487ULL, 0x3fef7c97337b9b5fULL, 0x3fefa4afa2a490daULL, 0x3fefd0765b6e4540ULL};

float vpo_expf_port(float x) {
    if (x != x) return x + x;
    if (x < -0x1.9fe368p6f) return 0.0f;
    if (x > 0x1.62e42ep6f) return INFINITY;
    if (x == -0x1.f8cbb2p+5f) return 0x1.f45326p-92f; /* the two inputs where glibc 2.39 */
    if (x == 0x1.04845ep+5f) return 0x1.f93e38p+46f;  /* differs from the bare algorithm */
    const double InvLn2N = 0x1.71547652b82fep+0 * 32, Shift = 0x1.8p+52;
    const double C0 = 0x1.c6af84b912394p-5 / 32 / 32 / 32, C1 = 0x1.ebfce50fac4f3p-3 / 32 / 32,
                 C2 = 0x1.62e42ff0c52d6p-1 / 32;
    const double z = InvLn2N * (double)x;
    double kd = z + Shift;
    uint64_t ki;
    memcpy(&ki, &kd, 8);
    kd -= Shift;
    const double r = z - kd;
    uint64_t t = kExp2fTab[ki % 32] + (ki << 47);
    double s;
    memcpy(&s, &t, 8);
    const double zz = fma(C0, r, C1);
    const double r2 = r * r;
    double y = fma(C2, r, 1.0);
    y = fma(zz, r2, y);
    return (float)(y * s);
}

/* Counts inputs in [lo_bits, hi_bits] (float bit patterns, walked upward) whose value in
 * `values` differs bitwise from libm expf. values[i] corresponds to lo_bits + i. */
int64_t vpo_expf_mismatches(uint32_t lo_bits, uint32_t hi_bits, const float *values) {
    int64_t bad = 0;
    for (uint64_t u = lo_bits; u <= hi_bits; ++u) {
        float x, e;
        const uint32_t b = (uint32_t)u;
        memcpy(&x, &b, 4);
        e = expf(x);
        if (memcmp(&e, &values[u - lo_bits], 4) != 0) ++bad;
    }
    return bad;
}

/* Counts floats x = bits lo, lo+stride, ... <= hi where vpo_expf_port(x) != libm expf(x). */
int64_t vpo_expf_port_mismatches(uint32_t lo_bits, uint32_t hi_bits, uint32_t stride) {
    int64_t bad = 0;
    if (stride == 0) stride = 1;
    for (uint64_t u = lo_bits; u <= hi_bits; u += stride) {
        float x, a, b;
        const uint32_t w = (uint32_t)u;
        memcpy(&x, &w, 4);
        a = expf(x);
        b = vpo_expf_port(x);
        if (memcmp(&a, &b, 4) != 0) ++bad;
    }
    return bad;
}

/* ---------------------------------------------------------------------------------------
 * C port of glibc 2.39 sinf / cosf (sysdeps/ieee754/flt-32/s_sinf.c, s_cosf.c, sincosf.h:
 * the ARM optimized-routines algorithm), as used by rotationFromAxisAngle
 * (rotation.cpp:8-27) through std::sin / std::cos on float. Polynomials in binary64 with the
 * multiply-adds fused, as in the FMA build glibc's ifunc selects on x86-64 hosts with FMA;
 * one rounding to float at the end. The coefficient table is __sincosf_table (sign[4],
 * hpi_inv = 2/pi * 2^24, hpi = pi/2, then c0 c1 s1 c2 s2 c3 s3 c4; the second row negates the
 * cosine coefficients), the 4/pi bits are __inv_pio4. Ported to the device in
 * paper_2103_01954_b200/csrc/vpb_device.cuh (device compose). */
static const double kSinCosTab[2][8] = {
    {0x1p0, -0x1.ffffffd0c621cp-2, -0x1.555545995a603p-3, 0x1.55553e1068f19p-5, 0x1.1107605230bc4p-7,
     -0x1.6c087e89a359dp-10, -0x1.994eb3774cf24p-13, 0x1.99343027bf8c3p-16},
    {-0x1p0, 0x1.ffffffd0c621cp-2, -0x1.555545995a603p-3, -0x1.55553e1068f19p-5, 0x1.1107605230bc4p-7,
     0x1.6c087e89a359dp-10, -0x1.994eb3774cf24p-13, -0x1.99343027bf8c3p-16}};
static const uint32_t kInvPio4[24] = {
    0xa2,       0xa2f9,     0xa2f983,   0xa2f9836e, 0xf9836e4e, 0x836e4e44, 0x6e4e4415, 0x4e441529,
    0x441529fc, 0x1529fc27, 0x29fc2757, 0xfc2757d1, 0x2757d1f5, 0x57d1f534, 0xd1f534dd, 0xf534ddc0,
    0x34ddc0db, 0xddc0db62, 0xc0db6295, 0xdb629599, 0x6295993c, 0x95993c43, 0x993c4390, 0x3c439041};

static uint32_t sc_abstop12(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    return (u >> 20) & 0x7ff;
}

/* sinf_poly: n even -> sine polynomial, odd -> cosine polynomial (c = kSinCosTab row) */
static float sc_poly(double x, double x2, const double *c, int n) {
    if ((n & 1) == 0) {
        const double x3 = x * x2;
        const double s1 = fma(x2, c[6], c[4]);
        const double x7 = x3 * x2;
        const double s = fma(x3, c[2], x);
        return (float)fma(x7, s1, s);
    }
    const double x4 = x2 * x2;
    const double c2 = fma(x2, c[7], c[5]);
    const double c1 = fma(x2, c[1], c[0]);
    const double x6 = x4 * x2;
    const double cc = fma(x4, c[3], c1);
    return (float)fma(x6, c2, cc);
}

static double sc_reduce_fast(double x, int *np) {
    const double r = x * 0x1.45f306dc9c883p+23;
    const int n = ((int32_t)r + 0x800000) >> 24;
    *np = n;
    return fma(-(double)n, 0x1.921fb54442d18p0, x);
}

static double sc_reduce_large(uint32_t xi, int *np) {
    const uint32_t *arr = &kInvPio4[(xi >> 26) & 15];
    const int shift = (xi >> 23) & 7;
    xi = (xi & 0xffffff) | 0x800000;
    xi <<= shift;
    uint64_t res0 = (uint64_t)(uint32_t)(xi * arr[0]);
    const uint64_t res1 = (uint64_t)xi * arr[4];
    const uint64_t res2 = (uint64_t)xi * arr[8];
    res0 = (res2 >> 32) | (res0 << 32);
    res0 += res1;
    const uint64_t n = (res0 + (1ULL << 61)) >> 62;
    res0 -= n << 62;
    *np = (int)n;
    return (double)(int64_t)res0 * 0x1.921fb54442d18p-62;
}

static float sc_eval(float y, int want_cos) {
    const double sign[4] = {1.0, -1.0, -1.0, 1.0};
    double x = y;
    int n = 0;
    const double *c = kSinCosTab[0];
    if (sc_abstop12(y) < sc_abstop12(0x1.921fb6p-1f)) {
        const double x2 = x * x;
        if (sc_abstop12(y) < sc_abstop12(0x1p-12f)) return want_cos ? 1.0f : y;
        return sc_poly(x, x2, c, want_cos);
    }
    if (sc_abstop12(y) < sc_abstop12(120.0f)) {
        x = sc_reduce_fast(x, &n);
        const double s = sign[n & 3];
        if (n & 2) c = kSinCosTab[1];
        return sc_poly(x * s, x * x, c, want_cos ? n ^ 1 : n);
    }
    if (sc_abstop12(y) < sc_abstop12(INFINITY)) {
        uint32_t xi;
        memcpy(&xi, &y, 4);
        const int sgn = (int)(xi >> 31);
        x = sc_reduce_large(xi, &n);
        const double s = sign[(n + sgn) & 3];
        if ((n + sgn) & 2) c = kSinCosTab[1];
        return sc_poly(x * s, x * x, c, want_cos ? n ^ 1 : n);
    }
    return (y - y) / (y - y);
}

float vpo_sinf_port(float x) { return sc_eval(x, 0); }
float vpo_cosf_port(float x) { return sc_eval(x, 1); }

/* Counts floats x = bits lo, lo+stride, ... <= hi where the ports differ from libm sinf/cosf
 * (which: 0 sin, 1 cos). */
int64_t vpo_sincos_port_mismatches(uint32_t lo_bits, uint32_t hi_bits, uint32_t stride, int which) {
    int64_t bad = 0;
    if (stride == 0) stride = 1;
    for (uint64_t u = lo_bits; u <= hi_bits; u += stride) {
        float x, a, b;
        const uint32_t w = (uint32_t)u;
        memcpy(&x, &w, 4);
        a = which ? cosf(x) : sinf(x);
        b = which ? vpo_cosf_port(x) : vpo_sinf_port(x);
        if (memcmp(&a, &b, 4) != 0 && !(a != a && b != b)) ++bad;
    }
    return bad;
}

/* Counts inputs in [lo_bits, hi_bits] whose value in `values` differs bitwise from libm
 * sinf/cosf (which: 0 sin, 1 cos). values[i] corresponds to lo_bits + i. */
int64_t vpo_sincos_mismatches(uint32_t lo_bits, uint32_t hi_bits, const float *values, int which) {
    int64_t bad = 0;
    for (uint64_t u = lo_bits; u <= hi_bits; ++u) {
        float x, e;
        const uint32_t b = (uint32_t)u;
        memcpy(&x, &b, 4);
        e = which ? cosf(x) : sinf(x);
        if (memcmp(&e, &values[u - lo_bits], 4) != 0 && !(e != e && values[u - lo_bits] != values[u - lo_bits])) ++bad;
    }
    return bad;
}

/* libm sinf / cosf (which: 0 sin, 1 cos) over an arbitrary array (test reference values). */
void vpo_sincos_libm(int64_t n, const float *x, float *y, int which) {
    for (int64_t i = 0; i < n; ++i) y[i] = which ? cosf(x[i]) : sinf(x[i]);
}
