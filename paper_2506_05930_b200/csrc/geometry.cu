// geometry.cu -- FP64 ray queries, G-buffer, unshadowed light factors and the
// training-batch generator (SURVEY table K: K5, K6).
//
// This TU is compiled with -fmad=false: every expression below rounds like
// the reference's serial numba/numpy code (no FMA contraction), which is what
// makes G-buffers, screen samples and shadow-ray labels bit-exact.
//
// Reference routines (under /root/reference/pkg/src/viscache):
//   ray_tri kernels.py:20-56, _aabb_hit :59-83, _inv_dir :86-90,
//   closest_hit :93-137, any_hit :140-174, _rect_factor :220-281,
//   _point_factor :284-296, light_factors_all :299-316,
//   visibility_batch geometry.py:233-247, trace_rays render.py:49-75,
//   make_gbuffer render.py:103-117, camera_rays_batch scene.py:129-139,
//   gen_world_samples training.py:44-48, gen_screen_hits :67-94,
//   compute_visibility_targets :103-120.
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace nvc {

namespace {

constexpr int kStack = 64;

// Moller-Trumbore exactly as kernels.py:21-56.  The three barycentric /
// distance numerators are formed before the (expensive, FP64) division; a
// test whose outcome is already decided by the numerator's sign or magnitude
// returns early.  Every early exit is one the reference also takes: with
// |num| >= 2^-900 and |det| < 2^100 the quotient num*(1/det) cannot
// underflow, so an opposite sign means a strictly negative u/v/t, and
// |num| > 2|det| means |u| (or |v|, u+v) > 1 after any rounding.
__device__ __forceinline__ double ray_tri(const double o[3], const double d[3], const double* a,
                                          const double* b, const double* c, double t_min,
                                          double t_max) {
    const double e1x = b[0] - a[0], e1y = b[1] - a[1], e1z = b[2] - a[2];
    const double e2x = c[0] - a[0], e2y = c[1] - a[1], e2z = c[2] - a[2];
    const double px = d[1] * e2z - d[2] * e2y;
    const double py = d[2] * e2x - d[0] * e2z;
    const double pz = d[0] * e2y - d[1] * e2x;
    const double det = e1x * px + e1y * py + e1z * pz;
    if (fabs(det) < 1e-14) return -1.0;
    const double tx = o[0] - a[0], ty = o[1] - a[1], tz = o[2] - a[2];
    const double un = tx * px + ty * py + tz * pz;
    const double qx = ty * e1z - tz * e1y;
    const double qy = tz * e1x - tx * e1z;
    const double qz = tx * e1y - ty * e1x;
    const double vn = d[0] * qx + d[1] * qy + d[2] * qz;
    const double tn = e2x * qx + e2y * qy + e2z * qz;
    const double ad = fabs(det);
    if (ad < 0x1p100) {
        const bool neg = det < 0.0;
        const double lim = 2.0 * ad;
        if (fabs(un) >= 0x1p-900 && ((un < 0.0) != neg || fabs(un) > lim)) return -1.0;   // u < 0 or u > 1
        if (fabs(vn) >= 0x1p-900 && ((vn < 0.0) != neg || fabs(vn) > lim)) return -1.0;   // v < 0 or v > 1
        if (fabs(un) >= 0x1p-900 && fabs(vn) >= 0x1p-900 && fabs(un) + fabs(vn) > 2.0 * lim)
            return -1.0;                                                                  // u + v > 1
        if (t_min >= 0.0 && fabs(tn) >= 0x1p-900 && (tn < 0.0) != neg) return -1.0;       // t < 0 <= t_min
    }
    const double inv = 1.0 / det;
    const double u = un * inv;
    if (u < 0.0 || u > 1.0) return -1.0;
    const double v = vn * inv;
    if (v < 0.0 || u + v > 1.0) return -1.0;
    const double t = tn * inv;
    if (t < t_min || t > t_max) return -1.0;
    return t;
}

__device__ __forceinline__ bool aabb_hit(const double o[3], const double inv[3], const double* bmin,
                                         const double* bmax, double t_max) {
    double lo, hi;
    {
        double t0 = (bmin[0] - o[0]) * inv[0], t1 = (bmax[0] - o[0]) * inv[0];
        if (t0 > t1) { const double s = t0; t0 = t1; t1 = s; }
        lo = t0;
        hi = t1;
    }
#pragma unroll
    for (int a = 1; a < 3; ++a) {
        double t0 = (bmin[a] - o[a]) * inv[a], t1 = (bmax[a] - o[a]) * inv[a];
        if (t0 > t1) { const double s = t0; t0 = t1; t1 = s; }
        if (t0 > lo) lo = t0;
        if (t1 < hi) hi = t1;
    }
    return hi >= lo && lo <= t_max && hi >= 0.0;
}

__device__ __forceinline__ double inv_dir(double d) {
    if (fabs(d) < 1e-300) return d >= 0.0 ? 1e300 : -1e300;
    return 1.0 / d;
}

// nearest hit; returns BVH-order triangle index or -1, t in *t_out
__device__ int64_t closest_hit(const nvc_scene& sc, const double o[3], const double d[3],
                               double t_min, double t_max, double* t_out) {
    *t_out = -1.0;
    if (sc.n_tris == 0) return -1;
    const double inv[3] = {inv_dir(d[0]), inv_dir(d[1]), inv_dir(d[2])};
    double best_t = t_max;
    int64_t best = -1;
    int32_t stack[kStack];
    int top = 0;
    stack[top++] = 0;
    while (top > 0) {
        const int32_t n = stack[--top];
        if (!aabb_hit(o, inv, sc.node_min + 3 * n, sc.node_max + 3 * n, best_t)) continue;
        const int32_t cnt = __ldg(sc.node_count + n);
        if (cnt > 0) {
            const int32_t s = __ldg(sc.node_start + n);
            for (int32_t k = s; k < s + cnt; ++k) {
                const double t = ray_tri(o, d, sc.bv0 + 3 * k, sc.bv1 + 3 * k, sc.bv2 + 3 * k, t_min, best_t);
                if (t >= 0.0) {
                    best_t = t;
                    best = k;
                }
            }
        } else {
            stack[top++] = __ldg(sc.node_left + n);
            stack[top++] = __ldg(sc.node_right + n);
        }
    }
    if (best >= 0) *t_out = best_t;
    return best;
}

// Any-hit by culling (scenes with <= BF_MAX_TRIS triangles, nvc.h).
// The reference's answer is "some triangle k passes ray_tri AND every BVH
// ancestor of k's leaf passes the FP64 slab test" (its traversal tests exactly
// those triangles, and any-hit does not depend on the order).  This evaluates
// the same predicate triangle by triangle, with two conservative f32 filters
// in front of the exact test:
//  1. plane test: the segment [p0, p1] = [o + t_min d, o + t_max d] cannot
//     meet k if both ends are farther than m on the same side of k's plane.
//     ray_tri can only accept a t in [t_min, t_max] whose point lies within
//     ~1e-15 * sliver * (t + |o - a|) of the plane (sliver = |e1||e2|/|e1 x e2|
//     <= 2^20 on the host, else the plane is zero and never culls), and the
//     f32 evaluation errs by < 2^-20 (R + |p|): m = 2^-15 (R + |p0| + |p1|)
//     covers both 32x;
//  2. crossing-box test (when |s1 - s0| > 4m and the triangle has a box,
//     sliver <= 2^8): the part of the segment within m of the plane,
//     f in [(-m - s0), (m - s0)] / (s1 - s0), widened by m, must overlap k's
//     AABB.  There ray_tri's barycentrics err by < ~1e-9 |p0 - p1| (the ray is
//     at least 4m/L away from parallel), far inside the widening;
//  3. exact FP64 ray_tri (the same function the traversal calls);
//  4. on a hit only: the FP64 slab test of the leaf and each ancestor.
// The result is bit-identical to the traversal's; per triangle it costs ~12
// f32 instructions when culled by the plane, ~30 when culled by the box.
__device__ __forceinline__ bool chain_ok(const nvc_scene& sc, int32_t k, const double o[3],
                                         const double inv[3], double t_max) {
    for (int32_t n = __ldg(sc.tri_leaf + k); n >= 0; n = __ldg(sc.node_parent + n))
        if (!aabb_hit(o, inv, sc.node_min + 3 * n, sc.node_max + 3 * n, t_max)) return false;
    return true;
}

__device__ __forceinline__ float max_abs3(float a, float b, float c) {
    return fmaxf(fabsf(a), fmaxf(fabsf(b), fabsf(c)));
}

// per-ray f32 data of the culling filters: segment ends p0, p1, p1 - p0, margin
struct CullRay {
    float a[3], b[3], g[3], m;
};

__device__ __forceinline__ CullRay cull_ray(const nvc_scene& sc, const double o[3], const double d[3], double t_min,
                                            double t_max) {
    CullRay r;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        r.a[c] = (float)(o[c] + t_min * d[c]);
        r.b[c] = (float)(o[c] + t_max * d[c]);
        r.g[c] = r.b[c] - r.a[c];
    }
    r.m = sc.plane_margin * ((sc.plane_r + max_abs3(r.a[0], r.a[1], r.a[2])) + max_abs3(r.b[0], r.b[1], r.b[2])) +
          1e-30f;
    return r;
}

// filters 1 + 2 for triangle k: false = the exact test cannot accept it
__device__ __forceinline__ bool cull_keep(const nvc_scene& sc, const CullRay& r, int32_t k) {
    const float4 q = __ldg(reinterpret_cast<const float4*>(sc.tri_plane) + k);
    const float s0 = fmaf(q.x, r.a[0], fmaf(q.y, r.a[1], fmaf(q.z, r.a[2], -q.w)));
    const float s1 = fmaf(q.x, r.b[0], fmaf(q.y, r.b[1], fmaf(q.z, r.b[2], -q.w)));
    const float m = r.m;
    bool keep = !(fminf(s0, s1) > m || fmaxf(s0, s1) < -m);
    const float ds = s1 - s0;
    if (keep && fabsf(ds) > 4.0f * m) {
        const float4* bx = reinterpret_cast<const float4*>(sc.tri_box) + 2 * k;
        const float4 lo = __ldg(bx), hi = __ldg(bx + 1);
        if (lo.w == 0.0f) {      // the triangle has a box (w = 1: never box-culled)
            // approximate reciprocal (rel. error ~2^-23): |fa|, |fb| err by ~2^-22 of
            // themselves, far inside the 2^-12 widening wherever they are not clamped
            float rd;
            asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rd) : "f"(ds));
            const float fa = (-m - s0) * rd, fb = (m - s0) * rd;
            const float f_lo = fmaxf(fminf(fa, fb) - 0x1p-12f, 0.0f);
            const float f_hi = fminf(fmaxf(fa, fb) + 0x1p-12f, 1.0f);
            const float u0 = fmaf(f_lo, r.g[0], r.a[0]), v0 = fmaf(f_hi, r.g[0], r.a[0]);
            const float u1 = fmaf(f_lo, r.g[1], r.a[1]), v1 = fmaf(f_hi, r.g[1], r.a[1]);
            const float u2 = fmaf(f_lo, r.g[2], r.a[2]), v2 = fmaf(f_hi, r.g[2], r.a[2]);
            keep = f_lo <= f_hi && fminf(u0, v0) - m <= hi.x && fmaxf(u0, v0) + m >= lo.x &&
                   fminf(u1, v1) - m <= hi.y && fmaxf(u1, v1) + m >= lo.y && fminf(u2, v2) - m <= hi.z &&
                   fmaxf(u2, v2) + m >= lo.z;
        }
    }
    return keep;
}

// filters 3 + 4: the reference's own test of triangle k and its leaf's ancestry
__device__ __forceinline__ bool exact_hit(const nvc_scene& sc, int32_t k, const double o[3], const double d[3],
                                          double t_min, double t_max) {
    if (ray_tri(o, d, sc.bv0 + 3 * k, sc.bv1 + 3 * k, sc.bv2 + 3 * k, t_min, t_max) < 0.0) return false;
    const double inv[3] = {inv_dir(d[0]), inv_dir(d[1]), inv_dir(d[2])};
    return chain_ok(sc, k, o, inv, t_max);
}

__device__ bool any_hit_bf(const nvc_scene& sc, const double o[3], const double d[3], double t_min,
                           double t_max) {
    const CullRay r = cull_ray(sc, o, d, t_min, t_max);
    const int32_t n = (int32_t)sc.n_tris;
    for (int32_t k0 = 0; k0 < n; k0 += 32) {
        const int32_t cnt = min(32, n - k0);
        uint32_t cand = 0u;
#pragma unroll 4
        for (int32_t j = 0; j < cnt; ++j) cand |= (cull_keep(sc, r, k0 + j) ? 1u : 0u) << j;
        while (cand) {
            const int32_t k = k0 + __ffs(cand) - 1;
            cand &= cand - 1u;
            if (exact_hit(sc, k, o, d, t_min, t_max)) return true;
        }
    }
    return false;
}

// order-preserving float <-> int maps for redux.sync min/max
__device__ __forceinline__ int f2key(float f) {
    const int b = __float_as_int(f);
    return b ^ ((b >> 31) & 0x7fffffff);
}
__device__ __forceinline__ float key2f(int k) { return __int_as_float(k ^ ((k >> 31) & 0x7fffffff)); }

// Warp-cooperative form (all 32 lanes call it; returns the lane's answer).
// The warp's segments all lie in the shaft H = hull(A, B) of the box A of its
// segment starts {o, p0} and the box B of its ends {p1}, each widened by the
// lane's margin m: H = { (1-s) a + s b : a in A, b in B, s in [0, 1] }.  Lane j
// decides for triangle k = k0 + j whether any lane can count it:
//  0. leaf: k counts only if the FP64 slab test of its leaf passes (step 4),
//     i.e. the segment [o, o + t_max d] reaches the leaf's box (to FP64
//     rounding) -- impossible if the leaf box misses H;
//  1. plane (warp form of filter 1): H's projection onto k's plane normal
//     lies farther than the largest m on one side of the plane;
//  2. crossing box (warp form of filter 2): the projections of A and B onto
//     the normal are more than 4.5 max m apart, so every lane's segment has
//     |s1 - s0| > 4 m, and k's box misses H (then each lane's crossing part,
//     widened, misses it too).
// Test "box T meets H": per axis, H's slice at s spans [lo(s), hi(s)] with
// lo(s) = Alo + s (Blo - Alo) and hi(s) = Ahi + s (Bhi - Ahi) (linear), so
// each of lo(s) <= Thi, hi(s) >= Tlo is a half-line in s; T meets H iff the
// six half-lines and [0, 1] intersect (H's bounding box covers the axes where
// A and B share a bound).  The f32 errors here are ~2^-22 of the scene scale,
// far inside the margin m (2^-15 of it) that the per-lane filters rest on.
// The per-lane filters then run only over the warp's candidates -- a short
// list when the warp's rays are coherent (Morton-sorted targets, light-sorted
// shading rows); tools/shaft_sim.py counts them (C2: ~15 of 98 per warp, the
// leaf-box-vs-segment-union filter alone kept ~55).
// Shaft parameters, computed once per warp call and kept in the warp's shared
// scratch (read back as broadcasts) rather than in ~40 registers across the
// triangle loop.
struct Shaft {
    float alo[3], ahi[3], blo[3], bhi[3], dl[3], dh[3], il[3], ih[3], ca[3], ea[3], cb[3], eb[3], mmax;
};
static_assert(sizeof(Shaft) <= kStack * sizeof(int32_t), "shaft scratch is a warp's packet-stack row");

__device__ __forceinline__ bool shaft_meets(const Shaft& h, const float tlo[3], const float thi[3]) {
    float s_lo = 0.0f, s_hi = 1.0f;
    bool ok = true;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        ok = ok && fminf(h.alo[a], h.blo[a]) <= thi[a] && fmaxf(h.ahi[a], h.bhi[a]) >= tlo[a];
        const float tl = (thi[a] - h.alo[a]) * h.il[a];   // lo(s) <= thi: s <= tl (dl > 0), s >= tl (dl < 0)
        const float th = (tlo[a] - h.ahi[a]) * h.ih[a];   // hi(s) >= tlo: s >= th (dh > 0), s <= th (dh < 0)
        s_hi = fminf(s_hi, h.dl[a] > 0.0f ? tl : INFINITY);
        s_lo = fmaxf(s_lo, h.dl[a] < 0.0f ? tl : -INFINITY);
        s_lo = fmaxf(s_lo, h.dh[a] > 0.0f ? th : -INFINITY);
        s_hi = fminf(s_hi, h.dh[a] < 0.0f ? th : INFINITY);
    }
    return ok && s_lo <= s_hi + 0x1p-16f;
}

// scratch: >= sizeof(Shaft) bytes of shared memory private to the warp
__device__ bool any_hit_bf_warp(const nvc_scene& sc, const double o[3], const double d[3], double t_min,
                                double t_max, bool active, Shaft* scratch) {
    const int lane = threadIdx.x & 31;
    const CullRay r = cull_ray(sc, o, d, t_min, t_max);
    bool all = false;   // a lane with NaN bounds needs every triangle
    {
        Shaft h;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const float oc = (float)o[c];
            float v[4] = {fminf(oc, r.a[c]) - r.m, fmaxf(oc, r.a[c]) + r.m, r.b[c] - r.m, r.b[c] + r.m};
            all = all || !(v[0] == v[0]) || !(v[1] == v[1]) || !(v[2] == v[2]) || !(v[3] == v[3]);
            h.alo[c] = key2f(__reduce_min_sync(0xffffffffu, active ? f2key(v[0]) : 0x7fffffff));
            h.ahi[c] = key2f(__reduce_max_sync(0xffffffffu, active ? f2key(v[1]) : (int)0x80000000));
            h.blo[c] = key2f(__reduce_min_sync(0xffffffffu, active ? f2key(v[2]) : 0x7fffffff));
            h.bhi[c] = key2f(__reduce_max_sync(0xffffffffu, active ? f2key(v[3]) : (int)0x80000000));
            h.dl[c] = h.blo[c] - h.alo[c];
            h.dh[c] = h.bhi[c] - h.ahi[c];
            h.il[c] = h.dl[c] != 0.0f ? 1.0f / h.dl[c] : 0.0f;
            h.ih[c] = h.dh[c] != 0.0f ? 1.0f / h.dh[c] : 0.0f;
            h.ca[c] = 0.5f * (h.alo[c] + h.ahi[c]);
            h.ea[c] = 0.5f * (h.ahi[c] - h.alo[c]);
            h.cb[c] = 0.5f * (h.blo[c] + h.bhi[c]);
            h.eb[c] = 0.5f * (h.bhi[c] - h.blo[c]);
        }
        h.mmax = key2f(__reduce_max_sync(0xffffffffu, active ? f2key(r.m) : (int)0x80000000));
        all = __any_sync(0xffffffffu, active && (all || !(r.m == r.m)));
        if (lane == 0) *scratch = h;
        __syncwarp();
    }
    const Shaft& h = *scratch;
    bool hit = false, live = active;
    const int32_t n = (int32_t)sc.n_tris;
    for (int32_t k0 = 0; k0 < n; k0 += 32) {
        if (!__any_sync(0xffffffffu, live)) break;
        bool ov = false;
        if (k0 + lane < n) {
            const int32_t k = k0 + lane;
            const int32_t leaf = __ldg(sc.tri_leaf + k);
            const double* lo = sc.node_min + 3 * leaf;
            const double* hi = sc.node_max + 3 * leaf;
            float tlo[3] = {(float)__ldg(lo), (float)__ldg(lo + 1), (float)__ldg(lo + 2)};
            float thi[3] = {(float)__ldg(hi), (float)__ldg(hi + 1), (float)__ldg(hi + 2)};
            const float4 q = __ldg(reinterpret_cast<const float4*>(sc.tri_plane) + k);
            const float pa = fmaf(q.x, h.ca[0], fmaf(q.y, h.ca[1], q.z * h.ca[2]));
            const float pb = fmaf(q.x, h.cb[0], fmaf(q.y, h.cb[1], q.z * h.cb[2]));
            const float ra = fmaf(fabsf(q.x), h.ea[0], fmaf(fabsf(q.y), h.ea[1], fabsf(q.z) * h.ea[2]));
            const float rb = fmaf(fabsf(q.x), h.eb[0], fmaf(fabsf(q.y), h.eb[1], fabsf(q.z) * h.eb[2]));
            // plane: zero for slivers (then both sides are 0 - 0 and nothing is culled)
            const bool side = fminf(pa - ra, pb - rb) - q.w > h.mmax || fmaxf(pa + ra, pb + rb) - q.w < -h.mmax;
            const float4* bx = reinterpret_cast<const float4*>(sc.tri_box) + 2 * k;
            const float4 blo = __ldg(bx), bhi = __ldg(bx + 1);
            if (blo.w == 0.0f && fabsf(pb - pa) - ra - rb > 4.5f * h.mmax) {
                tlo[0] = blo.x; tlo[1] = blo.y; tlo[2] = blo.z;   // the triangle's own box
                thi[0] = bhi.x; thi[1] = bhi.y; thi[2] = bhi.z;
            }
            ov = all || (!side && shaft_meets(h, tlo, thi));
        }
        uint32_t wm = __ballot_sync(0xffffffffu, ov);
        uint32_t cand = 0u;
        while (wm) {                                   // warp-uniform loop over the warp's candidates
            const int j = __ffs(wm) - 1;
            wm &= wm - 1u;
            cand |= (live && cull_keep(sc, r, k0 + j) ? 1u : 0u) << j;
        }
        while (cand) {
            const int32_t k = k0 + __ffs(cand) - 1;
            cand &= cand - 1u;
            if (exact_hit(sc, k, o, d, t_min, t_max)) {
                hit = true;
                live = false;
                break;
            }
        }
    }
    return hit;
}

__device__ bool any_hit(const nvc_scene& sc, const double o[3], const double d[3], double t_min,
                        double t_max) {
    if (sc.n_tris == 0) return false;
    if (sc.anyhit_bf) return any_hit_bf(sc, o, d, t_min, t_max);
    const double inv[3] = {inv_dir(d[0]), inv_dir(d[1]), inv_dir(d[2])};
    int32_t stack[kStack];
    int top = 0;
    stack[top++] = 0;
    while (top > 0) {
        const int32_t n = stack[--top];
        if (!aabb_hit(o, inv, sc.node_min + 3 * n, sc.node_max + 3 * n, t_max)) continue;
        const int32_t cnt = __ldg(sc.node_count + n);
        if (cnt > 0) {
            const int32_t s = __ldg(sc.node_start + n);
            for (int32_t k = s; k < s + cnt; ++k)
                if (ray_tri(o, d, sc.bv0 + 3 * k, sc.bv1 + 3 * k, sc.bv2 + 3 * k, t_min, t_max) >= 0.0)
                    return true;
        } else {
            stack[top++] = __ldg(sc.node_left + n);
            stack[top++] = __ldg(sc.node_right + n);
        }
    }
    return false;
}

// visibility_batch for one segment (geometry.py:233-247)
__device__ float segment_visible(const nvc_scene& sc, const double x[3], const double y[3]) {
    const double eps = sc.shadow_eps;
    const double d[3] = {y[0] - x[0], y[1] - x[1], y[2] - x[2]};
    const double dist = sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);
    const double safe = fmax(dist, 1e-300);
    const double dir[3] = {d[0] / safe, d[1] / safe, d[2] / safe};
    double t_max = dist - eps;
    if (t_max <= eps) return 1.0f;  // degenerate: endpoints closer than the epsilons
    t_max = fmax(t_max, eps + 1e-12);
    return any_hit(sc, x, dir, eps, t_max) ? 0.0f : 1.0f;
}

// camera_rays_batch (scene.py:129-139) for continuous image coords (sx, sy)
__device__ void camera_ray(const nvc_camera& c, double sx, double sy, double d[3]) {
    const double nx = ((2.0 * sx) / (double)c.width - 1.0) * c.tan_half * c.aspect;
    const double ny = (1.0 - (2.0 * sy) / (double)c.height) * c.tan_half;
#pragma unroll
    for (int a = 0; a < 3; ++a) d[a] = (c.fwd[a] + nx * c.right[a]) + ny * c.up[a];
    const double n = sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);
#pragma unroll
    for (int a = 0; a < 3; ++a) d[a] = d[a] / n;
}

// _rect_factor (kernels.py:220-281)
__device__ double rect_factor(const double p[3], const double n[3], const double* verts,
                              const double* ln) {
    const double side = (p[0] - verts[0]) * ln[0] + (p[1] - verts[1]) * ln[1] + (p[2] - verts[2]) * ln[2];
    if (side <= 0.0) return 0.0;
    double vx[4], vy[4], vz[4], cx[8], cy[8], cz[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        vx[i] = verts[3 * i + 0] - p[0];
        vy[i] = verts[3 * i + 1] - p[1];
        vz[i] = verts[3 * i + 2] - p[2];
    }
    int nc = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int j = (i + 1) & 3;
        const double di = vx[i] * n[0] + vy[i] * n[1] + vz[i] * n[2];
        const double dj = vx[j] * n[0] + vy[j] * n[1] + vz[j] * n[2];
        if (di >= 0.0) {
            cx[nc] = vx[i];
            cy[nc] = vy[i];
            cz[nc] = vz[i];
            ++nc;
        }
        if ((di > 0.0 && dj < 0.0) || (di < 0.0 && dj > 0.0)) {
            const double s = di / (di - dj);
            cx[nc] = vx[i] + s * (vx[j] - vx[i]);
            cy[nc] = vy[i] + s * (vy[j] - vy[i]);
            cz[nc] = vz[i] + s * (vz[j] - vz[i]);
            ++nc;
        }
    }
    if (nc < 3) return 0.0;
    for (int i = 0; i < nc; ++i) {
        const double l = sqrt(cx[i] * cx[i] + cy[i] * cy[i] + cz[i] * cz[i]);
        if (l < 1e-12) return 0.0;
        cx[i] /= l;
        cy[i] /= l;
        cz[i] /= l;
    }
    double acc = 0.0;
    for (int i = 0; i < nc; ++i) {
        const int j = (i + 1) % nc;
        double d = cx[i] * cx[j] + cy[i] * cy[j] + cz[i] * cz[j];
        d = d > 1.0 ? 1.0 : (d < -1.0 ? -1.0 : d);
        const double st0 = 1.0 - d * d;
        const double st = sqrt(st0 > 0.0 ? st0 : 0.0);
        const double ratio = st < 1e-9 ? 1.0 : acos(d) / st;
        const double gx = cy[i] * cz[j] - cz[i] * cy[j];
        const double gy = cz[i] * cx[j] - cx[i] * cz[j];
        const double gz = cx[i] * cy[j] - cy[i] * cx[j];
        acc += ratio * (gx * n[0] + gy * n[1] + gz * n[2]);
    }
    return 0.5 * fabs(acc);
}

// _point_factor (kernels.py:284-296)
__device__ double point_factor(const double p[3], const double n[3], const double* l) {
    const double wx = l[0] - p[0], wy = l[1] - p[1], wz = l[2] - p[2];
    const double d2 = wx * wx + wy * wy + wz * wz;
    if (d2 < 1e-24) return 0.0;
    const double inv = 1.0 / sqrt(d2);
    const double c = (wx * n[0] + wy * n[1] + wz * n[2]) * inv;
    if (c <= 0.0) return 0.0;
    return c / d2;
}

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------

// trace_rays + make_gbuffer: jitter draws (2p, 2p+1) of the PRIMARY stream
// sxy == nullptr: pixel p_first + i with numpy-Philox jitter (make_gbuffer);
// else the ray through screen point (sxy[2i], sxy[2i+1]) (gen_screen_hits).
__global__ void k_gbuffer(nvc_scene sc, nvc_camera cam, uint64_t key, int64_t p_first, int64_t np,
                          double* __restrict__ pos, double* __restrict__ nrm, double* __restrict__ alb,
                          uint8_t* __restrict__ hit, int32_t* __restrict__ light_id,
                          const double* __restrict__ sxy = nullptr, double* __restrict__ depth = nullptr,
                          double* __restrict__ emissive = nullptr) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= np) return;
    double d[3];
    if (sxy) {
        camera_ray(cam, sxy[2 * i], sxy[2 * i + 1], d);
    } else {
        const int64_t gp = p_first + i;
        double j0, j1;
        draw2(key, 2ull * (uint64_t)gp, j0, j1);
        const int64_t ys = gp / cam.width, xs = gp - ys * cam.width;
        camera_ray(cam, (double)xs + j0, (double)ys + j1, d);
    }
    double t;
    const int64_t bt = closest_hit(sc, cam.pos, d, 0.0, __longlong_as_double(0x7ff0000000000000ll), &t);
    const bool h = bt >= 0;
    double P[3] = {0, 0, 0}, N[3] = {0, 0, 0}, A[3] = {0, 0, 0}, E[3] = {0, 0, 0};
    int32_t lid = -1;
    if (h) {
        const int64_t tri = __ldg(sc.perm + bt);
        for (int a = 0; a < 3; ++a) P[a] = cam.pos[a] + t * d[a];
        const double* v0 = sc.tv0 + 3 * tri;
        const double* v1 = sc.tv1 + 3 * tri;
        const double* v2 = sc.tv2 + 3 * tri;
        const double e1[3] = {v1[0] - v0[0], v1[1] - v0[1], v1[2] - v0[2]};
        const double e2[3] = {v2[0] - v0[0], v2[1] - v0[1], v2[2] - v0[2]};
        N[0] = e1[1] * e2[2] - e1[2] * e2[1];
        N[1] = e1[2] * e2[0] - e1[0] * e2[2];
        N[2] = e1[0] * e2[1] - e1[1] * e2[0];
        const double nn = fmax(sqrt((N[0] * N[0] + N[1] * N[1]) + N[2] * N[2]), 1e-300);
        for (int a = 0; a < 3; ++a) N[a] = N[a] / nn;
        const double facing = (N[0] * d[0] + N[1] * d[1]) + N[2] * d[2];
        if (facing > 0.0)
            for (int a = 0; a < 3; ++a) N[a] = N[a] * -1.0;
        const int32_t mat = __ldg(sc.tri_material + tri);
        if (mat >= 0)
            for (int a = 0; a < 3; ++a) A[a] = __ldg(sc.mat_albedo + 3 * mat + a);
        lid = __ldg(sc.tri_light + tri);
        // render.py:69-71: an emitter seen from its front face shows its radiance
        if (lid >= 0 && !(facing > 0.0))
            for (int a = 0; a < 3; ++a) E[a] = __ldg(sc.lt_radiance + 3 * lid + a);
    }
    if (depth) depth[i] = h ? t : __longlong_as_double(0x7ff0000000000000ll);
    if (emissive)
        for (int a = 0; a < 3; ++a) emissive[3 * i + a] = E[a];
    for (int a = 0; a < 3; ++a) {
        pos[3 * i + a] = P[a];
        nrm[3 * i + a] = N[a];
        alb[3 * i + a] = A[a];
    }
    if (hit) hit[i] = h;
    if (light_id) light_id[i] = lid;
}

// light_factors_all -> light-major factor[j*stride + p] (+ lum)
template <typename T>
__global__ void k_factors(nvc_scene sc, const double* __restrict__ pos, const double* __restrict__ nrm,
                          const double* __restrict__ alb, int64_t np, int64_t stride,
                          T* __restrict__ factor, T* __restrict__ lum) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    if (i >= np) return;
    const double p[3] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
    const double n[3] = {nrm[3 * i], nrm[3 * i + 1], nrm[3 * i + 2]};
    const double f = sc.lt_kind[j] == 0 ? rect_factor(p, n, sc.lt_verts + 12 * j, sc.lt_normal + 3 * j)
                                        : point_factor(p, n, sc.lt_verts + 12 * j);
    if (factor) factor[(int64_t)j * stride + i] = (T)f;
    if (lum) {
        const double* w = sc.lt_lumaw + 3 * j;
        const double s = ((alb[3 * i] * w[0] + alb[3 * i + 1] * w[1]) + alb[3 * i + 2] * w[2]) / 3.141592653589793;
        lum[(int64_t)j * stride + i] = (T)(f * s);
    }
}

// ---- clustered two-step sampling (sampling.py:302-352) -------------------------
// Step 1: WRS over the m clamped cluster visibilities (draws offset + p*m + k).
// Step 2, cluster by cluster in ascending order on the continuing stream: the
// pixels that chose cluster j, in ascending pixel order, draw a (rows x |mem|)
// row-major block for a WRS over the members with weights phat / p_src.  So a
// pixel's step-2 draws start at t_j + rank * |mem| with rank its position among
// cluster j's pixels and t_j the draws of the clusters before j: a stable
// counting pass (block-local ranks, then a scan over blocks) supplies both.
// Light points follow all step-2 draws.
constexpr int kCsThreads = 256;

struct CsWs {
    int32_t *c_idx, *rank, *blk;   // blk: [nblk][m] counts, then exclusive offsets
    double *c_w, *c_sum;
    int64_t *cl_n, *cl_t, *total;  // per-cluster pixel counts, draw bases; [0]: light-point base
};

// workspace layout: byte offsets of each array (the last entry: total size)
inline void cs_layout(int64_t p, int m, int64_t off[9]) {
    const int64_t nblk = (p + kCsThreads - 1) / kCsThreads;
    const int64_t sz[8] = {4 * p, 4 * p, 4 * nblk * m, 8 * p, 8 * p, 8 * (int64_t)m, 8 * (int64_t)m, 8};
    off[0] = 0;
    for (int i = 0; i < 8; ++i) off[i + 1] = off[i] + (sz[i] + 255) / 256 * 256;
}

inline CsWs cs_ws(void* ws, int64_t p, int m) {
    int64_t o[9];
    cs_layout(p, m, o);
    char* c = (char*)ws;
    CsWs w;
    w.c_idx = (int32_t*)(c + o[0]);
    w.rank = (int32_t*)(c + o[1]);
    w.blk = (int32_t*)(c + o[2]);
    w.c_w = (double*)(c + o[3]);
    w.c_sum = (double*)(c + o[4]);
    w.cl_n = (int64_t*)(c + o[5]);
    w.cl_t = (int64_t*)(c + o[6]);
    w.total = (int64_t*)(c + o[7]);
    return w;
}

__global__ void __launch_bounds__(kCsThreads) k_cs_step1(const float* __restrict__ vis, int64_t vstride, int64_t P,
                                                        int m, uint64_t key, uint64_t offset, double floor, CsWs w) {
    const int64_t p = (int64_t)blockIdx.x * kCsThreads + threadIdx.x;
    if (p >= P) return;
    double s = 0.0, wsel = 0.0;
    int sel = -1;
    const uint64_t n0 = offset + (uint64_t)p * (uint64_t)m;
    U4 u = philox_block(n0 / 4 + 1, key);
    for (int k = 0; k < m; ++k) {
        const double v = (double)vis[p * vstride + k];
        const double cw = floor > 0.0 ? (v > floor ? v : floor) : (v > 0.0 ? v : 0.0);   // np.maximum
        s = __dadd_rn(s, cw);
        const uint64_t n = n0 + (uint64_t)k;
        if (k > 0 && (n & 3) == 0) u = philox_block(n / 4 + 1, key);
        const uint32_t ln = (uint32_t)(n & 3);
        const uint64_t r = ln == 0 ? u.x[0] : (ln == 1 ? u.x[1] : (ln == 2 ? u.x[2] : u.x[3]));
        if (cw > 0.0 && __dmul_rn(u01(r), s) < cw) {
            sel = k;
            wsel = cw;
        }
    }
    w.c_idx[p] = sel;
    w.c_w[p] = wsel;
    w.c_sum[p] = s;
}

// block-local stable ranks: the block's warps take turns, lanes of one cluster
// grouped with match.any, so rank order = pixel order
__global__ void __launch_bounds__(kCsThreads) k_cs_rank(int64_t P, int m, CsWs w) {
    extern __shared__ int cnt[];
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    for (int j = t; j < m; j += kCsThreads) cnt[j] = 0;
    __syncthreads();
    const int64_t p = (int64_t)blockIdx.x * kCsThreads + t;
    const int j = p < P ? w.c_idx[p] : -1;
    for (int ww = 0; ww < kCsThreads / 32; ++ww) {
        if (wid == ww) {
            const uint32_t grp = __match_any_sync(0xffffffffu, j);
            const int r = __popc(grp & ((1u << lane) - 1u));
            const int base = j >= 0 ? cnt[j] : 0;
            __syncwarp();
            if (j >= 0 && r == 0) cnt[j] = base + __popc(grp);
            if (p < P) w.rank[p] = base + r;
        }
        __syncthreads();
    }
    for (int q = t; q < m; q += kCsThreads) w.blk[(int64_t)blockIdx.x * m + q] = cnt[q];
}

// per cluster (one CTA each): exclusive scan over the blocks' counts, pixel count
__global__ void __launch_bounds__(1024) k_cs_scan(int64_t nblk, int m, CsWs w) {
    __shared__ int s_w[32];
    const int j = blockIdx.x, t = threadIdx.x, lane = t & 31, wid = t >> 5;
    const int64_t per = (nblk + 1023) / 1024, b0 = t * per, b1 = min(nblk, b0 + per);
    int sum = 0;
    for (int64_t b = b0; b < b1; ++b) sum += w.blk[b * m + j];
    int incl = sum;
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_w[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        const int v = s_w[lane];
        int vi = v;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, vi, o);
            if (lane >= o) vi += y;
        }
        s_w[lane] = vi - v;
        if (lane == 31) w.cl_n[j] = vi;
    }
    __syncthreads();
    int run = s_w[wid] + incl - sum;
    for (int64_t b = b0; b < b1; ++b) {
        const int c = w.blk[b * m + j];
        w.blk[b * m + j] = run;
        run += c;
    }
}

// draw bases t_j of the clusters' step-2 blocks and the first light-point draw
__global__ void k_cs_bases(int m, const int32_t* __restrict__ c_off, int64_t P, uint64_t offset, CsWs w) {
    uint64_t t = offset + (uint64_t)P * (uint64_t)m;
    for (int j = 0; j < m; ++j) {
        w.cl_t[j] = (int64_t)t;
        t += (uint64_t)w.cl_n[j] * (uint64_t)(c_off[j + 1] - c_off[j]);
    }
    w.total[0] = (int64_t)t;
}

// numpy/OpenBLAS float64 (r,3)@(3,c): gemm shapes fma(a2,b2, fma(a1,b1, a0 b0)),
// gemv shapes (r == 1 or c == 1) fma(a2,b2, fma(a0,b0, a1 b1)) (tests/golden/clusters.npz)
__device__ __forceinline__ double dot3_blas(const double a[3], const double b[3], bool gemv) {
    return gemv ? fma(a[2], b[2], fma(a[0], b[0], a[1] * b[1])) : fma(a[2], b[2], fma(a[1], b[1], a[0] * b[0]));
}

// Philox through a real call: a block cached across iterations of the member
// loop (which inlines the FP64 rect factor) lives in registers this way -- the
// inlined form kept in a loop-carried local produced wrong draws (see DESIGN).
__device__ __noinline__ U4 philox_call(uint64_t counter, uint64_t key) { return philox_block(counter, key); }

// kCT: ftab is the cluster-ordered pixel-major table of nvc_cluster_factor_table
// (row p holds the pixel's factors in c_mem order, so a pixel's members are one
// contiguous run); otherwise the light-major (K, p) table or NULL
template <bool kCT>
__global__ void __launch_bounds__(kCsThreads) k_cs_step2(nvc_scene sc, const double* __restrict__ pos,
                                                        const double* __restrict__ nrm, const double* __restrict__ alb,
                                                        int64_t P, int m, const int32_t* __restrict__ c_off,
                                                        const int32_t* __restrict__ c_mem, uint64_t key, CsWs w,
                                                        const double* __restrict__ ftab, int64_t fstride,
                                                        int64_t* __restrict__ ids, double* __restrict__ pts,
                                                        double* __restrict__ big_w) {
    const int64_t p = (int64_t)blockIdx.x * kCsThreads + threadIdx.x;
    if (p >= P) return;
    const int j = w.c_idx[p];
    int64_t out_id = -1;
    double out_w = 0.0;
    if (j >= 0) {
        const int lo = c_off[j], my = c_off[j + 1] - lo;
        const int64_t rank = (int64_t)w.blk[(int64_t)blockIdx.x * m + j] + w.rank[p];
        const bool gemv = w.cl_n[j] == 1 || my == 1;
        const double x[3] = {pos[3 * p], pos[3 * p + 1], pos[3 * p + 2]};
        const double nx[3] = {nrm[3 * p], nrm[3 * p + 1], nrm[3 * p + 2]};
        const double a[3] = {alb[3 * p], alb[3 * p + 1], alb[3 * p + 2]};
        const double p_src = (double)m * (w.c_w[p] / w.c_sum[p]) / (double)my;
        const uint64_t n0 = (uint64_t)w.cl_t[j] + (uint64_t)rank * (uint64_t)my;
        double s = 0.0, phat_sel = 0.0;
        int sel = -1;
        uint64_t blk = ~0ull;
        U4 u;
        for (int k = 0; k < my; ++k) {
            const int l = c_mem[lo + k];
            const double f = kCT   ? __ldg(ftab + p * fstride + (lo + k))
                           : ftab ? __ldg(ftab + (int64_t)l * fstride + p)
                                  : (sc.lt_kind[l] == 0 ? rect_factor(x, nx, sc.lt_verts + 12 * l, sc.lt_normal + 3 * l)
                                                        : point_factor(x, nx, sc.lt_verts + 12 * l));
            const double lw[3] = {0.2126 * sc.lt_radiance[3 * l], 0.7152 * sc.lt_radiance[3 * l + 1],
                                  0.0722 * sc.lt_radiance[3 * l + 2]};
            const double phat = f * (dot3_blas(a, lw, gemv) / 3.141592653589793);
            const double w2 = phat / p_src;
            s = __dadd_rn(s, w2);
            const uint64_t n = n0 + (uint64_t)k, bi = n / 4 + 1;
            if (w2 > 0.0) {
                if (bi != blk) {
                    u = philox_call(bi, key);
                    blk = bi;
                }
                // lane by selects, not u.x[n & 3]: a dynamically indexed U4 lives in local memory,
                // and across the rect-factor call that gave wrong draws
                const uint32_t ln = (uint32_t)(n & 3);
                const uint64_t r = ln == 0 ? u.x[0] : (ln == 1 ? u.x[1] : (ln == 2 ? u.x[2] : u.x[3]));
                if (__dmul_rn(u01(r), s) < w2) {
                    sel = k;
                    phat_sel = phat;
                }
            }
        }
        if (sel >= 0) {
            out_id = c_mem[lo + sel];
            out_w = (double)m * s / ((double)my * phat_sel);
        }
    }
    const uint64_t nl = (uint64_t)w.total[0] + 2ull * (uint64_t)p;
    const double u0 = draw(key, nl), u1 = draw(key, nl + 1);
    double y[3];
    light_point(sc, out_id, u0, u1, y);
    ids[p] = out_id;
    big_w[p] = out_w;
    pts[3 * p] = y[0];
    pts[3 * p + 1] = y[1];
    pts[3 * p + 2] = y[2];
}

__global__ void k_visibility(nvc_scene sc, const double* __restrict__ x, const double* __restrict__ y,
                             int64_t n, float* __restrict__ vis) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double a[3] = {x[3 * i], x[3 * i + 1], x[3 * i + 2]};
    const double b[3] = {y[3 * i], y[3 * i + 1], y[3 * i + 2]};
    vis[i] = segment_visible(sc, a, b);
}

// ---- shading pass 5: shade_batch (render.py:220-246) --------------------------
// np.einsum("pc,pc->p") over c = 3 sums (a0 b0 + a2 b2) + a1 b1 (pinned by
// tests/golden/shade.npz); np.maximum(0, x) keeps NaN and maps -0 to +0.
__device__ __forceinline__ double dot3e(const double a[3], const double b[3]) {
    return (a[0] * b[0] + a[2] * b[2]) + a[1] * b[1];
}
__device__ __forceinline__ double max0(double x) { return 0.0 >= x ? 0.0 : x; }

// One thread per pixel.  With the warp any-hit (anyhit_bf == 2) all 32 lanes
// of a warp take part in one shaft-filtered any-hit call for their shadow rays
// (a warp's pixels are neighbours on the screen), lanes without a ray inactive.
__global__ void __launch_bounds__(128) k_shade(nvc_scene sc, const double* __restrict__ pos,
                                               const double* __restrict__ nrm, const double* __restrict__ alb,
                                               const int64_t* __restrict__ ids, const double* __restrict__ pts,
                                               const double* __restrict__ big_w, int64_t n,
                                               double* __restrict__ rgb) {
    __shared__ Shaft s_shaft[4];
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool warp_mode = sc.anyhit_bf == 2;
    if (i >= n && !warp_mode) return;
    const bool in = i < n;
    const int64_t id = in ? ids[i] : -1;
    const double W = in ? big_w[i] : 0.0;
    double out[3] = {0.0, 0.0, 0.0};
    double x[3] = {0.0, 0.0, 0.0}, y[3] = {0.0, 0.0, 0.0}, geom = 0.0;
    if (id >= 0 && id < sc.n_lights && W > 0.0) {
        x[0] = pos[3 * i]; x[1] = pos[3 * i + 1]; x[2] = pos[3 * i + 2];
        y[0] = pts[3 * i]; y[1] = pts[3 * i + 1]; y[2] = pts[3 * i + 2];
        const double nx[3] = {nrm[3 * i], nrm[3 * i + 1], nrm[3 * i + 2]};
        double w[3] = {y[0] - x[0], y[1] - x[1], y[2] - x[2]};
        double d2 = dot3e(w, w);
        d2 = d2 < 1e-24 ? 1e-24 : d2;
        const double r = sqrt(d2);
        w[0] = w[0] / r;
        w[1] = w[1] / r;
        w[2] = w[2] / r;
        const double ln[3] = {__ldg(sc.lt_normal + 3 * id), __ldg(sc.lt_normal + 3 * id + 1),
                              __ldg(sc.lt_normal + 3 * id + 2)};
        const double cos_x = max0(dot3e(nx, w));
        const double cos_y = max0(-dot3e(w, ln));
        geom = __ldg(sc.lt_kind + id) == 0 ? cos_x * cos_y / d2 * __ldg(sc.lt_area + id) : cos_x / d2;
    }
    const bool need = geom > 0.0;
    float vis = 1.0f;
    if (warp_mode) {
        // segment_visible's arithmetic, then one warp-wide call
        const double eps = sc.shadow_eps;
        const double d[3] = {y[0] - x[0], y[1] - x[1], y[2] - x[2]};
        const double dist = sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);
        const double safe = fmax(dist, 1e-300);
        const double dir[3] = {d[0] / safe, d[1] / safe, d[2] / safe};
        double t_max = dist - eps;
        const bool active = need && !(t_max <= eps) && sc.n_tris > 0;
        t_max = fmax(t_max, eps + 1e-12);
        if (__any_sync(0xffffffffu, active) &&
            any_hit_bf_warp(sc, x, dir, eps, t_max, active, &s_shaft[threadIdx.x >> 5]) && active)
            vis = 0.0f;
    } else if (need) {
        vis = segment_visible(sc, x, y);
    }
    if (need) {
        const double amp = geom * W * (double)vis;
#pragma unroll
        for (int c = 0; c < 3; ++c)
            out[c] = alb[3 * i + c] / 3.141592653589793 * __ldg(sc.lt_radiance + 3 * id + c) * amp;
    }
    if (in) {
        rgb[3 * i] = out[0];
        rgb[3 * i + 1] = out[1];
        rgb[3 * i + 2] = out[2];
    }
}

__global__ void k_closest(nvc_scene sc, const double* __restrict__ o, const double* __restrict__ d,
                          const double* __restrict__ t_min, const double* __restrict__ t_max, int64_t n,
                          double* __restrict__ t_out, int64_t* __restrict__ tri_out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double oo[3] = {o[3 * i], o[3 * i + 1], o[3 * i + 2]};
    const double dd[3] = {d[3 * i], d[3 * i + 1], d[3 * i + 2]};
    double t;
    const int64_t bt = closest_hit(sc, oo, dd, t_min[i], t_max[i], &t);
    t_out[i] = t;
    tri_out[i] = bt >= 0 ? __ldg(sc.perm + bt) : -1;
}

// ---- training batch --------------------------------------------------------
struct BatchWs {
    int64_t* counters;   // [0]=hits appended, [1]=want, [2]=draw offset
    uint8_t* flag;       // n_screen
    double* hp;          // n_screen * 3
};

__device__ __forceinline__ BatchWs batch_ws(void* ws, int n_screen) {
    BatchWs w;
    char* p = (char*)ws;
    w.counters = (int64_t*)p;
    w.hp = (double*)(p + 64);
    w.flag = (uint8_t*)(p + 64 + 24 * (int64_t)n_screen);
    return w;
}

// gen_world_samples: pos[i][c] = lo_c + (hi_c - lo_c) * u(3i + c)
__global__ void k_world(nvc_scene sc, uint64_t key, uint64_t base, int n, double* __restrict__ pos) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 3 * n) return;
    const int c = i % 3;
    pos[i] = sc.aabb_min[c] + (sc.aabb_max[c] - sc.aabb_min[c]) * draw(key, base + (uint64_t)i);
}

// screen round with `want` rays starting at draw offset `off`
__device__ __forceinline__ void screen_ray(const nvc_scene& sc, const nvc_camera& cam, uint64_t key,
                                           int64_t off, int64_t want, int64_t i, uint8_t* flag,
                                           double* hp) {
    const double sx = draw(key, (uint64_t)(off + i)) * (double)cam.width;
    const double sy = draw(key, (uint64_t)(off + want + i)) * (double)cam.height;
    double d[3], t;
    camera_ray(cam, sx, sy, d);
    const int64_t bt = closest_hit(sc, cam.pos, d, 0.0, __longlong_as_double(0x7ff0000000000000ll), &t);
    flag[i] = bt >= 0;
    if (bt >= 0)
        for (int a = 0; a < 3; ++a) hp[3 * i + a] = cam.pos[a] + t * d[a];
}

__global__ void k_screen_round0(nvc_scene sc, nvc_camera cam, uint64_t key, uint64_t base, int n, void* ws) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    BatchWs w = batch_ws(ws, n);
    screen_ray(sc, cam, key, (int64_t)base, n, i, w.flag, w.hp);
}

// block-wide exclusive scan of 0/1 flags (1024 threads)
__device__ __forceinline__ int block_excl_scan(int v, int* s_warp, int* total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const unsigned bal = __ballot_sync(0xffffffffu, v);
    const int in_warp = __popc(bal & ((1u << lane) - 1u));
    if (lane == 0) s_warp[wid] = __popc(bal);
    __syncthreads();
    if (wid == 0) {
        const int nw = blockDim.x >> 5;
        int x = lane < nw ? s_warp[lane] : 0;
        int incl = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane < nw) s_warp[lane] = incl - x;
        if (lane == 31) *total = incl;
    }
    __syncthreads();
    const int r = s_warp[wid] + in_warp;
    __syncthreads();
    return r;
}

// one block: order-preserving compaction of round 0, then rounds 1..8 in-block
__global__ void __launch_bounds__(1024) k_screen_finish(nvc_scene sc, nvc_camera cam, uint64_t key,
                                                        uint64_t base, int n_world, int n,
                                                        double* __restrict__ pos, int64_t* __restrict__ n_rows,
                                                        void* ws) {
    __shared__ int s_warp[32];
    __shared__ int s_total;
    BatchWs w = batch_ws(ws, n);
    double* out = pos + 3 * (int64_t)n_world;
    int64_t count = 0, want = n, off = (int64_t)base;
    for (int round = 0; round < 9 && want > 0; ++round) {
        if (round > 0) {
            for (int64_t i = threadIdx.x; i < want; i += blockDim.x) screen_ray(sc, cam, key, off, want, i, w.flag, w.hp);
            __syncthreads();
        }
        int64_t hits = 0;
        for (int64_t base = 0; base < want; base += blockDim.x) {
            const int64_t i = base + threadIdx.x;
            const int f = (i < want) ? (int)w.flag[i] : 0;
            const int r = block_excl_scan(f, s_warp, &s_total);
            if (f) {
                const int64_t o = count + hits + r;
                for (int a = 0; a < 3; ++a) out[3 * o + a] = w.hp[3 * i + a];
            }
            hits += s_total;
            __syncthreads();
        }
        count += hits;
        off += 2 * want;
        want -= hits;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        *n_rows = n_world + count;
        w.counters[2] = off;   // the screen stream's position after the call
    }
}

// Warp-packet any-hit: the 32 lanes walk one shared DFS stack (node, lane
// mask).  A lane takes part in a node only if its own slab test accepted every
// ancestor, and visits its nodes in the reference's order (push left then
// right, pop LIFO), so each lane's answer is exactly its scalar traversal's;
// the warp just stops diverging over the tree.
__device__ uint32_t any_hit_packet(const nvc_scene& sc, const double o[3], const double d[3], double t_min,
                                   double t_max, bool active, int32_t* st_node, uint32_t* st_mask) {
    const int lane = threadIdx.x & 31;
    uint32_t hit = 0u;
    const uint32_t act = __ballot_sync(0xffffffffu, active);
    if (sc.n_tris == 0 || act == 0u) return 0u;
    if (sc.anyhit_bf == 2)
        return __ballot_sync(0xffffffffu, any_hit_bf_warp(sc, o, d, t_min, t_max, active,
                                                          reinterpret_cast<Shaft*>(st_node)));
    if (sc.anyhit_bf) return __ballot_sync(0xffffffffu, active && any_hit_bf(sc, o, d, t_min, t_max));
    const double inv[3] = {inv_dir(d[0]), inv_dir(d[1]), inv_dir(d[2])};
    int top = 0;
    if (lane == 0) {
        st_node[0] = 0;
        st_mask[0] = act;
    }
    top = 1;
    __syncwarp();
    while (top > 0) {
        --top;
        const int32_t n = st_node[top];
        uint32_t m = st_mask[top] & ~hit;
        __syncwarp();
        if (m == 0u) continue;
        const bool mine = (m >> lane) & 1u;
        const bool box = mine && aabb_hit(o, inv, sc.node_min + 3 * n, sc.node_max + 3 * n, t_max);
        m = __ballot_sync(0xffffffffu, box);
        if (m == 0u) continue;
        const int32_t cnt = __ldg(sc.node_count + n);
        if (cnt > 0) {
            bool h = false;
            if ((m >> lane) & 1u) {
                const int32_t s0 = __ldg(sc.node_start + n);
                for (int32_t k = s0; k < s0 + cnt && !h; ++k)
                    h = ray_tri(o, d, sc.bv0 + 3 * k, sc.bv1 + 3 * k, sc.bv2 + 3 * k, t_min, t_max) >= 0.0;
            }
            hit |= __ballot_sync(0xffffffffu, h);
            if ((act & ~hit) == 0u) break;
        } else {
            if (lane == 0) {
                st_node[top] = __ldg(sc.node_left + n);
                st_mask[top] = m;
                st_node[top + 1] = __ldg(sc.node_right + n);
                st_mask[top + 1] = m;
            }
            top += 2;
            __syncwarp();
        }
    }
    return hit;
}

// compute_visibility_targets (light mode): row i, light j uses draws j*2b + 2i, +1.
// One warp per row, lanes over lights (K <= 32 per pass): the warp's shadow rays
// share an origin and fan out to neighbouring emitters -> packet traversal.
__global__ void __launch_bounds__(128) k_targets(nvc_scene sc, uint64_t key, uint64_t off, const double* __restrict__ pos,
                                                 const int64_t* __restrict__ n_rows, int64_t b_host, int shard,
                                                 int n_shards, int64_t cap, float* __restrict__ tgt) {
    __shared__ int32_t st_node[4][kStack];
    __shared__ uint32_t st_mask[4][kStack];
    const int w = threadIdx.x >> 5;
    const int64_t r = (int64_t)blockIdx.x * 4 + w;
    const int lane = threadIdx.x & 31;
    const int64_t b = n_rows ? *n_rows : b_host;
    int64_t lo, hi;
    shard_range(b, shard, n_shards, lo, hi);
    const int64_t i = lo + r;
    if (r >= cap || i >= hi) return;     // warp-uniform
    const double x[3] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
    const double eps = sc.shadow_eps;
    for (int j0 = 0; j0 < sc.n_lights; j0 += 32) {
        const int j = j0 + lane;
        const bool valid = j < sc.n_lights;
        double y[3] = {0.0, 0.0, 0.0};
        if (valid) {
            double u0, u1;
            const uint64_t n = off + (uint64_t)(2 * b * j + 2 * i);   // draws off + 2bj + 2i, +1
            if (off & 1) {
                u0 = draw(key, n);
                u1 = draw(key, n + 1);
            } else {
                draw2(key, n, u0, u1);
            }
            light_point(sc, j, u0, u1, y);
        }
        // visibility_batch (geometry.py:233-247), per lane
        const double dd[3] = {y[0] - x[0], y[1] - x[1], y[2] - x[2]};
        const double dist = sqrt((dd[0] * dd[0] + dd[1] * dd[1]) + dd[2] * dd[2]);
        const double safe = fmax(dist, 1e-300);
        const double dir[3] = {dd[0] / safe, dd[1] / safe, dd[2] / safe};
        double t_max = dist - eps;
        const bool degenerate = t_max <= eps;
        t_max = fmax(t_max, eps + 1e-12);
        const uint32_t hits = any_hit_packet(sc, x, dir, eps, t_max, valid && !degenerate, st_node[w], st_mask[w]);
        if (valid) tgt[r * sc.n_lights + j] = (degenerate || !((hits >> lane) & 1u)) ? 1.0f : 0.0f;
    }
}

// Shadow rays grouped for coherence: the shard's rows are bucketed by a
// 12-bit Morton code of their position (one CTA: shared-memory histogram,
// scan, scatter) and a warp takes 32 consecutive bucketed rows x one light, so
// its rays start close together and end on the same emitter -- the packet
// traversal then visits ~one ray's path instead of the union of 32 fanned-out
// rays.  Results are per (row, light), so the order within a bucket (atomic
// arrival order) does not affect them.
constexpr int kSortMax = 16384;
constexpr int kBuckets = 4096;

__device__ __forceinline__ uint32_t spread4(uint32_t v) {   // 4 bits -> every third bit
    v &= 15u;
    v = (v | (v << 4)) & 0x0C3u;
    v = (v | (v << 2)) & 0x249u;
    return v;
}

__global__ void __launch_bounds__(1024) k_morton_order(nvc_scene sc, const double* __restrict__ pos,
                                                       const int64_t* __restrict__ n_rows, int64_t b_host, int shard,
                                                       int n_shards, int32_t* __restrict__ order) {
    __shared__ int hist[kBuckets];
    __shared__ int warp_sum[32];
    extern __shared__ int slot[];   // per row: code << 16 | rank within bucket
    const int64_t b = n_rows ? *n_rows : b_host;
    int64_t lo, hi;
    shard_range(b, shard, n_shards, lo, hi);
    const int n = (int)(hi - lo);
    for (int c = threadIdx.x; c < kBuckets; c += blockDim.x) hist[c] = 0;
    float lo3[3], inv3[3];
    for (int a = 0; a < 3; ++a) {
        const float span = (float)(sc.aabb_max[a] - sc.aabb_min[a]);
        lo3[a] = (float)sc.aabb_min[a];
        inv3[a] = span > 0.0f ? 16.0f / span : 0.0f;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
        uint32_t c = 0;
        for (int a = 0; a < 3; ++a) {
            const float q = ((float)pos[3 * (lo + t) + a] - lo3[a]) * inv3[a];
            c |= spread4((uint32_t)fminf(fmaxf(q, 0.0f), 15.0f)) << a;
        }
        slot[t] = (int)(c << 16) | atomicAdd(&hist[c], 1);
    }
    __syncthreads();
    // exclusive scan of the 4096 bucket counts: 4 per thread, then across warps
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int v[4], run = 0;
    for (int e = 0; e < 4; ++e) {
        v[e] = run;
        run += hist[4 * threadIdx.x + e];
    }
    int incl = run;
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) warp_sum[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        int x = warp_sum[lane], xi = x;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, xi, o);
            if (lane >= o) xi += y;
        }
        warp_sum[lane] = xi - x;
    }
    __syncthreads();
    const int base = warp_sum[wid] + incl - run;
    for (int e = 0; e < 4; ++e) hist[4 * threadIdx.x + e] = base + v[e];
    __syncthreads();
    for (int t = threadIdx.x; t < n; t += blockDim.x) order[hist[slot[t] >> 16] + (slot[t] & 0xFFFF)] = t;
}

// compute_visibility_targets over Morton-ordered rows: block = 4 warps x 32
// sorted rows, blockIdx.y = light.  Same per-(row, light) arithmetic as k_targets.
template <int kMinBlocks>
__global__ void __launch_bounds__(128, kMinBlocks) k_targets_sorted(nvc_scene sc, uint64_t key, const double* __restrict__ pos,
                                                        const int64_t* __restrict__ n_rows, int64_t b_host, int shard,
                                                        int n_shards, const int32_t* __restrict__ order,
                                                        float* __restrict__ tgt) {
    __shared__ int32_t st_node[4][kStack];
    __shared__ uint32_t st_mask[4][kStack];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int j = blockIdx.y;
    const int64_t b = n_rows ? *n_rows : b_host;
    int64_t lo, hi;
    shard_range(b, shard, n_shards, lo, hi);
    const int64_t t = (int64_t)blockIdx.x * 128 + threadIdx.x;
    if ((int64_t)blockIdx.x * 128 + w * 32 >= hi - lo) return;   // warp-uniform
    const bool valid = t < hi - lo;
    const int64_t r = valid ? order[t] : 0;
    const int64_t i = lo + r;
    const double x[3] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
    const double eps = sc.shadow_eps;
    double y[3] = {0.0, 0.0, 0.0};
    if (valid) {
        double u0, u1;
        draw2(key, (uint64_t)(2 * b * j + 2 * i), u0, u1);
        light_point(sc, j, u0, u1, y);
    }
    const double dd[3] = {y[0] - x[0], y[1] - x[1], y[2] - x[2]};
    const double dist = sqrt((dd[0] * dd[0] + dd[1] * dd[1]) + dd[2] * dd[2]);
    const double safe = fmax(dist, 1e-300);
    const double dir[3] = {dd[0] / safe, dd[1] / safe, dd[2] / safe};
    double t_max = dist - eps;
    const bool degenerate = t_max <= eps;
    t_max = fmax(t_max, eps + 1e-12);
    const uint32_t hits = any_hit_packet(sc, x, dir, eps, t_max, valid && !degenerate, st_node[w], st_mask[w]);
    if (valid) tgt[r * sc.n_lights + j] = (degenerate || !((hits >> lane) & 1u)) ? 1.0f : 0.0f;
}

__global__ void k_set_rows(int64_t* n_rows, int64_t v) { *n_rows = v; }

// ---- cluster-mode targets (training.py:121-128) -------------------------------
// Per cluster j (ascending) the reference draws ids = mem[rng.integers(0, |mem|,
// size=b)] and then rng.random((b, 2)) on one stream.  integers() is Lemire's
// bounded draw on 32-bit draws with a rejection loop; a 32-bit draw is the low
// half of a fresh 64-bit output and the bit generator keeps the high half for
// the next 32-bit draw, across calls (random() skips it).  One CTA walks the
// clusters in order; per cluster all threads evaluate a window of 32-bit draws,
// a block scan ranks the accepted ones (row i takes the i-th), and the index of
// the b-th acceptance fixes the outputs consumed and the kept half -- the exact
// stream positions, rejections included.  |mem| = 1 draws nothing.
__device__ __forceinline__ uint64_t philox_out(uint64_t key, uint64_t n) {
    return philox_block(n / 4 + 1, key).x[n & 3];
}

constexpr int kPickThreads = 1024;

// Fast path: assume no rejection (p ~ n / 2^32 per draw).  One thread chains the
// clusters' stream positions in closed form; a (rows x clusters) grid draws the
// picks and flags any cluster where a draw would have been rejected; only then
// does the exact sequential walk (k_cluster_picks) run, overwriting everything.
__global__ void k_cluster_chain(const int64_t* __restrict__ n_rows, int32_t m, const int32_t* __restrict__ c_off,
                                uint64_t start, int64_t kept_in, int64_t* __restrict__ uni_start,
                                int64_t* __restrict__ draw_base, int64_t* __restrict__ kept_src,
                                int32_t* __restrict__ flag) {
    const int64_t b = *n_rows;
    uint64_t next = start;
    // the half the bit generator keeps: -1 none, -2 the caller's value (kept_in),
    // >= 0 the high half of that 64-bit output
    int64_t kept = kept_in >= 0 ? -2 : -1;
    for (int j = 0; j < m; ++j) {
        const int32_t n = c_off[j + 1] - c_off[j];
        draw_base[j] = (int64_t)next;
        kept_src[j] = kept;
        if (n > 1 && b > 0) {
            const int64_t fresh = b - (kept != -1 ? 1 : 0);
            const uint64_t outs = (uint64_t)((fresh + 1) / 2);
            kept = (fresh & 1) ? (int64_t)(next + outs - 1) : -1;
            next += outs;
        }
        uni_start[j] = (int64_t)next;
        next += 2 * (uint64_t)b;
    }
    uni_start[m] = (int64_t)next;
    uni_start[m + 1] = kept == -2 ? kept_in : kept;   // an output index is resolved by k_cluster_draws
    if (kept >= 0) uni_start[m + 1] = -3 - kept;       // (encoded: index i -> -3 - i)
    *flag = 0;
}

__global__ void __launch_bounds__(256) k_cluster_draws(uint64_t key, const int64_t* __restrict__ n_rows, int32_t m,
                                                       const int32_t* __restrict__ c_off,
                                                       const int32_t* __restrict__ c_mem,
                                                       const int64_t* __restrict__ draw_base,
                                                       const int64_t* __restrict__ kept_src,
                                                       int32_t* __restrict__ picks, int64_t* __restrict__ uni_start,
                                                       int32_t* __restrict__ flag, int64_t kept_in) {
    const int64_t b = *n_rows;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    if (i == 0 && j == 0 && uni_start[m + 1] <= -3)
        uni_start[m + 1] = (int64_t)(philox_out(key, (uint64_t)(-3 - uni_start[m + 1])) >> 32);
    if (i >= b) return;
    const int32_t lo = c_off[j], n = c_off[j + 1] - lo;
    if (n == 1) {
        picks[i * m + j] = c_mem[lo];
        return;
    }
    const int has = kept_src[j] != -1 ? 1 : 0;
    uint32_t d;
    if (has && i == 0) {
        d = kept_src[j] == -2 ? (uint32_t)kept_in : (uint32_t)(philox_out(key, (uint64_t)kept_src[j]) >> 32);
    } else {
        const int64_t k = i - has;
        const uint64_t w = philox_out(key, (uint64_t)draw_base[j] + (uint64_t)(k >> 1));
        d = (k & 1) ? (uint32_t)(w >> 32) : (uint32_t)w;
    }
    const uint32_t nn = (uint32_t)n, thresh = (0u - nn) % nn;
    const uint64_t mm = (uint64_t)d * nn;
    if ((uint32_t)mm < thresh) atomicOr(flag, 1);
    picks[i * m + j] = c_mem[lo + (int32_t)(mm >> 32)];
}

__global__ void __launch_bounds__(kPickThreads) k_cluster_picks(uint64_t key, const int64_t* __restrict__ n_rows,
                                                                 int32_t m, const int32_t* __restrict__ c_off,
                                                                 const int32_t* __restrict__ c_mem,
                                                                 int32_t* __restrict__ picks,
                                                                 int64_t* __restrict__ uni_start,
                                                                 const int32_t* __restrict__ flag, uint64_t start,
                                                                 int64_t kept_in) {
    if (flag && *flag == 0) return;   // the fast path had no rejection: nothing to redo
    __shared__ uint64_t s_next;        // next fresh 64-bit output
    __shared__ uint32_t s_kept;        // kept high half (valid if s_has)
    __shared__ int s_has;
    __shared__ int s_warp[kPickThreads / 32];
    __shared__ int64_t s_tb;           // draw index of the b-th acceptance (-1: not in window)
    __shared__ int s_acc;              // acceptances in the window
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int64_t b = *n_rows;
    if (tid == 0) {
        s_next = start;
        s_has = kept_in >= 0 ? 1 : 0;
        s_kept = kept_in >= 0 ? (uint32_t)kept_in : 0u;
    }
    __syncthreads();
    for (int j = 0; j < m; ++j) {
        const int32_t lo = c_off[j], n = c_off[j + 1] - lo;
        if (n == 1) {
            for (int64_t i = tid; i < b; i += kPickThreads) picks[i * m + j] = c_mem[lo];
            __syncthreads();
            if (tid == 0) {
                uni_start[j] = (int64_t)s_next;
                s_next += 2 * (uint64_t)b;
            }
            __syncthreads();
            continue;
        }
        const uint32_t nn = (uint32_t)n, thresh = (0u - nn) % nn;
        const uint64_t base = s_next;
        const int has = s_has;
        const uint32_t kept = s_kept;
        int64_t t0 = 0, done = 0;      // window start (draw index), acceptances before it
        for (;;) {
            const int64_t D = b - done + 64;                                // window length
            const int64_t per = (D + kPickThreads - 1) / kPickThreads;
            const int64_t my0 = t0 + (int64_t)tid * per, my1 = min(t0 + D, my0 + per);
            auto draw32 = [&](int64_t t) -> uint32_t {   // t-th 32-bit draw of this call
                if (has && t == 0) return kept;
                const int64_t k = t - has;
                const uint64_t w = philox_out(key, base + (uint64_t)(k >> 1));
                return (k & 1) ? (uint32_t)(w >> 32) : (uint32_t)w;
            };
            int cnt = 0;
            for (int64_t t = my0; t < my1; ++t) {
                const uint64_t mm = (uint64_t)draw32(t) * nn;
                cnt += (uint32_t)mm >= thresh;
            }
            int incl = cnt;   // block exclusive scan of the per-thread counts
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (lane == 31) s_warp[wid] = incl;
            if (tid == 0) s_tb = -1;
            __syncthreads();
            if (wid == 0) {
                int v = s_warp[lane], vi = v;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, vi, o);
                    if (lane >= o) vi += y;
                }
                s_warp[lane] = vi - v;
                if (lane == 31) s_acc = vi;
            }
            __syncthreads();
            int64_t r = done + s_warp[wid] + (incl - cnt);
            for (int64_t t = my0; t < my1 && r < b; ++t) {
                const uint64_t mm = (uint64_t)draw32(t) * nn;
                if ((uint32_t)mm >= thresh) {
                    picks[r * m + j] = c_mem[lo + (int32_t)(mm >> 32)];
                    if (r == b - 1) s_tb = t;
                    ++r;
                }
            }
            __syncthreads();
            if (s_tb >= 0 || b == 0) break;
            done += s_acc;          // >= 65 rejections in the window: continue after it
            t0 += D;
            __syncthreads();
        }
        if (tid == 0) {
            const int64_t used = b == 0 ? 0 : s_tb + 1;                     // 32-bit draws consumed
            const int64_t fresh = used - (has && used > 0 ? 1 : 0);         // ... from new outputs
            const uint64_t outs = (uint64_t)((fresh + 1) / 2);
            if (used > 0) {
                s_has = (int)(fresh & 1);
                if (fresh & 1) s_kept = (uint32_t)(philox_out(key, base + outs - 1) >> 32);
            }
            uni_start[j] = (int64_t)(base + outs);
            s_next = base + outs + 2 * (uint64_t)b;
        }
        __syncthreads();
    }
    if (tid == 0) {   // the stream's state after the call: next output, kept half (-1: none)
        uni_start[m] = (int64_t)s_next;
        uni_start[m + 1] = s_has ? (int64_t)s_kept : -1;
    }
}

// shadow rays toward each row's picked member: draws uni_start[j] + 2i, +1
__global__ void __launch_bounds__(128) k_cluster_tgt(nvc_scene sc, uint64_t key, const double* __restrict__ pos,
                                                     const int64_t* __restrict__ n_rows, int shard, int n_shards,
                                                     int32_t m, const int32_t* __restrict__ picks,
                                                     const int64_t* __restrict__ uni_start, float* __restrict__ tgt) {
    const int64_t b = *n_rows;
    int64_t lo, hi;
    shard_range(b, shard, n_shards, lo, hi);
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    if (lo + r >= hi) return;
    const int64_t i = lo + r;
    const uint64_t n0 = (uint64_t)uni_start[j] + 2 * (uint64_t)i;
    const double u0 = draw(key, n0), u1 = draw(key, n0 + 1);
    const double x[3] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
    double y[3];
    light_point(sc, picks[i * m + j], u0, u1, y);
    tgt[r * m + j] = segment_visible(sc, x, y);
}

inline int grid1(int64_t n, int bs) { return (int)((n + bs - 1) / bs); }


// ---- RIS / screen-space ReSTIR baselines (sampling.py:369-637) ----------------
// A reservoir grid is struct-of-arrays on the device: y (p) i64, point (p,3)
// f64, w_y, w_sum, M, W (p) f64, valid (p) u8.  Target weight of light id at
// pixel i (PixelCtx.phat_ids, sampling.py:141-155): f(i, id) * (albedo .
// LUMA*L_e[id]) / pi, the dot in einsum order, f from the f64 light-major
// factor table; id < 0 -> 0.
struct RGrid {
    int64_t* y;
    double *pt, *w_y, *w_sum, *M, *W;
    uint8_t* valid;
};
struct RGridC {
    const int64_t* y;
    const double *pt, *w_y, *w_sum, *M, *W;
    const uint8_t* valid;
};

__device__ __forceinline__ double phat_at(const nvc_scene& sc, const double* __restrict__ factor, int64_t stride,
                                          const double alb[3], int64_t i, int64_t id) {
    if (id < 0) return 0.0;
    const double f = __ldg(factor + id * stride + i);
    const double lw[3] = {__ldg(sc.lt_lumaw + 3 * id), __ldg(sc.lt_lumaw + 3 * id + 1),
                          __ldg(sc.lt_lumaw + 3 * id + 2)};
    return f * (dot3e(alb, lw) / 3.141592653589793);
}

// ris_initial_batch: candidate ids = integers(0, K, (p, M)) (picks), phat from
// the luminance table, weights phat * K, streaming WRS on draws
// uni + i*M + j, W = w_sum / (M * phat(y)), points on draws uni + p*M + 2i.
template <typename LT>
__global__ void __launch_bounds__(128) k_ris_initial(nvc_scene sc, const LT* __restrict__ lum, int64_t stride,
                                                     int64_t p, int32_t mc, const int32_t* __restrict__ picks,
                                                     uint64_t key, const int64_t* __restrict__ uni, RGrid out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p) return;
    const uint64_t u0 = (uint64_t)uni[0];
    const double kd = (double)sc.n_lights;
    double s = 0.0, phs = 0.0;
    int sel = -1;
    for (int j = 0; j < mc; ++j) {
        const int64_t id = picks[i * mc + j];
        const double ph = (double)__ldg(lum + id * stride + i);
        const double w = ph * kd;
        s = s + w;
        if (u01(philox_out(key, u0 + (uint64_t)(i * mc + j))) * s < w) {
            sel = j;
            phs = ph;
        }
    }
    const bool ok = sel >= 0;
    const int64_t y = ok ? (int64_t)picks[i * mc + sel] : -1;
    const uint64_t np = u0 + (uint64_t)p * (uint64_t)mc + 2ull * (uint64_t)i;
    double pt[3];
    light_point(sc, y, u01(philox_out(key, np)), u01(philox_out(key, np + 1)), pt);
    out.y[i] = y;
    out.w_y[i] = ok ? phs : 0.0;
    out.w_sum[i] = s;
    out.M[i] = (double)mc;
    out.W[i] = ok ? s / ((double)mc * phs) : 0.0;
    for (int a = 0; a < 3; ++a) out.pt[3 * i + a] = pt[a];
    out.valid[i] = 1;
}

// restir_temporal_batch (sampling.py:487-526): draw offset + i
__global__ void __launch_bounds__(128) k_restir_temporal(nvc_scene sc, const double* __restrict__ factor,
                                                         int64_t stride, const double* __restrict__ alb_all, int64_t p,
                                                         RGridC cur, RGridC prev, uint64_t key, uint64_t offset,
                                                         double clamp, int32_t contribution, RGrid out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p) return;
    const double alb[3] = {alb_all[3 * i], alb_all[3 * i + 1], alb_all[3 * i + 2]};
    const bool pv = prev.valid[i] != 0;
    const int64_t yc = cur.y[i], yp = prev.y[i];
    const double ph_c = phat_at(sc, factor, stride, alb, i, yc);
    const double ph_p = phat_at(sc, factor, stride, alb, i, pv ? yp : -1);
    double m_prev, w_prev;
    if (!contribution) {
        m_prev = pv ? fmin(prev.M[i], clamp * cur.M[i]) : 0.0;
        w_prev = ph_p * prev.W[i] * m_prev;
    } else {
        m_prev = pv ? prev.M[i] : 0.0;
        w_prev = ph_p * prev.W[i] * m_prev;
        w_prev = fmin(w_prev, clamp * ph_c * cur.W[i] * cur.M[i]);
    }
    const double w_cur = ph_c * cur.W[i] * cur.M[i];
    const double w_sum = w_cur + w_prev;
    const bool take = (draw(key, offset + (uint64_t)i) * w_sum < w_prev) && (w_prev > 0.0);
    int64_t y = take ? yp : yc;
    const double M = cur.M[i] + m_prev;
    const double w_y = take ? ph_p : ph_c;
    const bool ok = (w_sum > 0.0) && (w_y > 0.0) && (M > 0.0);
    for (int a = 0; a < 3; ++a) out.pt[3 * i + a] = take ? prev.pt[3 * i + a] : cur.pt[3 * i + a];
    out.y[i] = ok ? y : -1;
    out.w_sum[i] = w_sum;
    out.M[i] = M;
    out.w_y[i] = w_y;
    out.W[i] = ok ? w_sum / (M * w_y) : 0.0;
    out.valid[i] = 1;
}

// restir_spatial_batch (sampling.py:541-595): per neighbour round r the draws
// offset + (3r)p + i (angle), (3r+1)p + i (radius), (3r+2)p + i (merge)
__global__ void __launch_bounds__(128) k_restir_spatial(nvc_scene sc, const double* __restrict__ factor,
                                                        int64_t stride, const double* __restrict__ alb_all,
                                                        const double* __restrict__ nrm, const uint8_t* __restrict__ hit,
                                                        const double* __restrict__ depth, int32_t width, int32_t height,
                                                        RGridC g, uint64_t key, uint64_t offset, int32_t radius,
                                                        int32_t neighbors, RGrid out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t p = (int64_t)width * height;
    if (i >= p) return;
    const double alb[3] = {alb_all[3 * i], alb_all[3 * i + 1], alb_all[3 * i + 2]};
    const double ni[3] = {nrm[3 * i], nrm[3 * i + 1], nrm[3 * i + 2]};
    const int64_t ys = i / width, xs = i - ys * width;
    int64_t acc_y = g.y[i];
    double acc_pt[3] = {g.pt[3 * i], g.pt[3 * i + 1], g.pt[3 * i + 2]};
    double acc_w = phat_at(sc, factor, stride, alb, i, acc_y) * g.W[i] * g.M[i];
    double acc_m = g.M[i];
    const bool hit_i = hit[i] != 0;
    const double di = depth[i];
    for (int r = 0; r < neighbors; ++r) {
        const uint64_t base = offset + (uint64_t)(3 * r) * (uint64_t)p + (uint64_t)i;
        const double ang = draw(key, base) * 2.0 * 3.141592653589793;
        const double rad = (double)radius * sqrt(draw(key, base + (uint64_t)p));
        const int64_t dx = (int64_t)rint(rad * cos(ang)), dy = (int64_t)rint(rad * sin(ang));
        const int64_t nx = xs + dx, ny = ys + dy;
        const bool inb = nx >= 0 && nx < width && ny >= 0 && ny < height && (dx != 0 || dy != 0);
        const int64_t j = inb ? ny * width + nx : 0;
        bool ok = inb && g.valid[j] && hit_i && hit[j];
        const double nj[3] = {nrm[3 * j], nrm[3 * j + 1], nrm[3 * j + 2]};
        const double ndot = dot3e(ni, nj);
        const double ratio = depth[j] / fmax(di, 1e-12);
        ok = ok && ndot >= 0.9 && ratio >= 0.9 && ratio <= 1.1;
        const int64_t n_y = ok ? g.y[j] : -1;
        const double w_n = ok ? phat_at(sc, factor, stride, alb, i, n_y) * g.W[j] * g.M[j] : 0.0;
        const double w_sum = acc_w + w_n;
        const bool take = (draw(key, base + 2ull * (uint64_t)p) * w_sum < w_n) && (w_n > 0.0);
        acc_w = w_sum;
        if (take) {
            acc_y = n_y;
            for (int a = 0; a < 3; ++a) acc_pt[a] = g.pt[3 * j + a];
        }
        acc_m = acc_m + (ok ? g.M[j] : 0.0);
    }
    const double w_y = phat_at(sc, factor, stride, alb, i, acc_y);
    const bool ok = (acc_w > 0.0) && (w_y > 0.0) && (acc_m > 0.0);
    out.y[i] = ok ? acc_y : -1;
    for (int a = 0; a < 3; ++a) out.pt[3 * i + a] = acc_pt[a];
    out.w_sum[i] = acc_w;
    out.M[i] = acc_m;
    out.w_y[i] = w_y;
    out.W[i] = ok ? acc_w / (acc_m * w_y) : 0.0;
    out.valid[i] = 1;
}

// PixelCtx.phat_ids for one id per pixel
__global__ void k_phat_ids(nvc_scene sc, const double* __restrict__ factor, int64_t stride,
                           const double* __restrict__ alb_all, const int64_t* __restrict__ ids, int64_t p,
                           double* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p) return;
    const double alb[3] = {alb_all[3 * i], alb_all[3 * i + 1], alb_all[3 * i + 2]};
    out[i] = phat_at(sc, factor, stride, alb, i, ids[i]);
}

__global__ void k_ris_setup(int32_t* c_off, int32_t* c_mem, int32_t k, int64_t* n_rows, int64_t b) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < k) c_mem[t] = t;
    if (t == 0) {
        c_off[0] = 0;
        c_off[1] = k;
        *n_rows = b;
    }
}

}  // namespace

}  // namespace nvc

using namespace nvc;

extern "C" {

int nvc_gbuffer(const nvc_scene* sc, const nvc_camera* cam, uint64_t key, int64_t p_first, int64_t p,
                double* pos, double* nrm, double* alb, uint8_t* hit, int32_t* light_id, double* depth,
                double* emissive, void* stream) {
    NVC_REQUIRE(sc && cam && pos && nrm && alb, "nvc_gbuffer: null argument");
    if (p <= 0) return NVC_OK;
    k_gbuffer<<<grid1(p, 128), 128, 0, (cudaStream_t)stream>>>(*sc, *cam, key, p_first, p, pos, nrm, alb, hit,
                                                                light_id, nullptr, depth, emissive);
    return check_launch("k_gbuffer");
}

int nvc_primary_hits(const nvc_scene* sc, const nvc_camera* cam, const double* sxy, int64_t n, double* pos,
                     double* nrm, double* alb, uint8_t* hit, int32_t* light_id, void* stream) {
    NVC_REQUIRE(sc && cam && sxy && pos && nrm && alb && hit, "nvc_primary_hits: null argument");
    if (n <= 0) return NVC_OK;
    k_gbuffer<<<grid1(n, 128), 128, 0, (cudaStream_t)stream>>>(*sc, *cam, 0, 0, n, pos, nrm, alb, hit, light_id,
                                                                sxy);
    return check_launch("k_gbuffer");
}

int nvc_light_factors(const nvc_scene* sc, const double* pos, const double* nrm, const double* alb,
                      int64_t p, int64_t stride, int32_t out_f64, void* factor, void* lum, void* stream) {
    NVC_REQUIRE(sc && pos && nrm, "nvc_light_factors: null argument");
    NVC_REQUIRE(!lum || alb, "nvc_light_factors: lum needs albedo");
    NVC_REQUIRE(stride >= p, "nvc_light_factors: stride < p");
    if (p <= 0) return NVC_OK;
    dim3 g(grid1(p, 128), sc->n_lights);
    if (out_f64)
        k_factors<double><<<g, 128, 0, (cudaStream_t)stream>>>(*sc, pos, nrm, alb, p, stride, (double*)factor,
                                                               (double*)lum);
    else
        k_factors<float><<<g, 128, 0, (cudaStream_t)stream>>>(*sc, pos, nrm, alb, p, stride, (float*)factor,
                                                              (float*)lum);
    return check_launch("k_factors");
}

int64_t nvc_clustered_workspace_bytes(int64_t p, int32_t m) {
    int64_t o[9];
    cs_layout(p, m, o);
    return o[8];
}

int nvc_clustered_select(const nvc_scene* sc, const float* vis, int64_t vis_stride, const double* pos,
                         const double* nrm, const double* alb, const double* factor, int64_t p, int32_t m,
                         const int32_t* c_off, const int32_t* c_mem, uint64_t key, uint64_t offset, double floor,
                         int64_t* ids, double* pts, double* big_w, void* ws, void* stream) {
    NVC_REQUIRE(sc && vis && pos && nrm && alb && c_off && c_mem && ids && pts && big_w && ws,
                "nvc_clustered_select: null argument");
    NVC_REQUIRE(m >= 1 && vis_stride >= m, "nvc_clustered_select: bad m / stride");
    if (p <= 0) return NVC_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const CsWs w = cs_ws(ws, p, m);
    const int nblk = grid1(p, kCsThreads);
    k_cs_step1<<<nblk, kCsThreads, 0, s>>>(vis, vis_stride, p, m, key, offset, floor, w);
    k_cs_rank<<<nblk, kCsThreads, (size_t)m * 4, s>>>(p, m, w);
    k_cs_scan<<<m, 1024, 0, s>>>(nblk, m, w);
    k_cs_bases<<<1, 1, 0, s>>>(m, c_off, p, offset, w);
    k_cs_step2<false><<<nblk, kCsThreads, 0, s>>>(*sc, pos, nrm, alb, p, m, c_off, c_mem, key, w, factor, p, ids,
                                                  pts, big_w);
    return check_launch("nvc_clustered_select");
}

// (K, p) light-major -> (p, K) pixel-major with the columns in c_mem order:
// 32 x 32 tiles through shared memory, both sides coalesced
__global__ void __launch_bounds__(256) k_cluster_ftab(const double* __restrict__ f, int64_t p, int32_t k,
                                                      const int32_t* __restrict__ c_mem, double* __restrict__ out) {
    __shared__ double t[32][33];
    const int64_t p0 = (int64_t)blockIdx.x * 32;
    const int i0 = blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += 8) {   // r: member column i0 + r
        const int i = i0 + r;
        const int64_t q = p0 + threadIdx.x;
        t[r][threadIdx.x] = (i < k && q < p) ? __ldg(f + (int64_t)__ldg(c_mem + i) * p + q) : 0.0;
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += 8) {   // r: pixel p0 + r
        const int64_t q = p0 + r;
        const int i = i0 + threadIdx.x;
        if (q < p && i < k) out[q * k + i] = t[threadIdx.x][r];
    }
}

int nvc_cluster_factor_table(const double* factor, int64_t p, int32_t k, const int32_t* c_mem, double* out,
                             void* stream) {
    NVC_REQUIRE(factor && c_mem && out && k >= 1, "nvc_cluster_factor_table: bad argument");
    if (p <= 0) return NVC_OK;
    const dim3 grid((unsigned)((p + 31) / 32), (unsigned)((k + 31) / 32));
    k_cluster_ftab<<<grid, dim3(32, 8), 0, (cudaStream_t)stream>>>(factor, p, k, c_mem, out);
    return check_launch("k_cluster_ftab");
}

int nvc_clustered_select_ct(const nvc_scene* sc, const float* vis, int64_t vis_stride, const double* pos,
                            const double* nrm, const double* alb, const double* factor_ct, int64_t ct_stride,
                            int64_t p, int32_t m, const int32_t* c_off, const int32_t* c_mem, uint64_t key, uint64_t offset, double floor,
                            int64_t* ids, double* pts, double* big_w, void* ws, void* stream) {
    NVC_REQUIRE(sc && vis && pos && nrm && alb && factor_ct && c_off && c_mem && ids && pts && big_w && ws,
                "nvc_clustered_select_ct: null argument");
    NVC_REQUIRE(m >= 1 && vis_stride >= m && ct_stride >= 1, "nvc_clustered_select_ct: bad m / stride");
    if (p <= 0) return NVC_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const CsWs w = cs_ws(ws, p, m);
    const int nblk = grid1(p, kCsThreads);
    k_cs_step1<<<nblk, kCsThreads, 0, s>>>(vis, vis_stride, p, m, key, offset, floor, w);
    k_cs_rank<<<nblk, kCsThreads, (size_t)m * 4, s>>>(p, m, w);
    k_cs_scan<<<m, 1024, 0, s>>>(nblk, m, w);
    k_cs_bases<<<1, 1, 0, s>>>(m, c_off, p, offset, w);
    k_cs_step2<true><<<nblk, kCsThreads, 0, s>>>(*sc, pos, nrm, alb, p, m, c_off, c_mem, key, w, factor_ct,
                                                 ct_stride, ids, pts, big_w);
    return check_launch("nvc_clustered_select_ct");
}

int64_t nvc_clustered_state_offset(int64_t p, int32_t m) {   // int64: first light-point draw
    int64_t o[9];
    cs_layout(p, m, o);
    return o[7];
}

int nvc_visibility(const nvc_scene* sc, const double* x, const double* y, int64_t n, float* vis,
                   void* stream) {
    NVC_REQUIRE(sc && x && y && vis, "nvc_visibility: null argument");
    if (n <= 0) return NVC_OK;
    k_visibility<<<grid1(n, 128), 128, 0, (cudaStream_t)stream>>>(*sc, x, y, n, vis);
    return check_launch("k_visibility");
}

int nvc_shade(const nvc_scene* sc, const double* pos, const double* nrm, const double* alb, const int64_t* ids,
              const double* pts, const double* big_w, int64_t n, double* rgb, void* stream) {
    NVC_REQUIRE(sc && pos && nrm && alb && ids && pts && big_w && rgb, "nvc_shade: null argument");
    NVC_REQUIRE(sc->lt_area, "nvc_shade: scene without lt_area");
    if (n <= 0) return NVC_OK;
    k_shade<<<grid1(n, 128), 128, 0, (cudaStream_t)stream>>>(*sc, pos, nrm, alb, ids, pts, big_w, n, rgb);
    return check_launch("k_shade");
}

int nvc_closest_hit(const nvc_scene* sc, const double* o, const double* d, const double* t_min,
                    const double* t_max, int64_t n, double* t_out, int64_t* tri_out, void* stream) {
    NVC_REQUIRE(sc && o && d && t_min && t_max && t_out && tri_out, "nvc_closest_hit: null argument");
    if (n <= 0) return NVC_OK;
    k_closest<<<grid1(n, 128), 128, 0, (cudaStream_t)stream>>>(*sc, o, d, t_min, t_max, n, t_out, tri_out);
    return check_launch("k_closest");
}

int64_t nvc_batch_workspace_bytes(int32_t n_world, int32_t n_screen) {
    return 64 + 25 * (int64_t)n_screen + 64 + 256 + 4 * ((int64_t)n_world + n_screen);
}

int nvc_gen_train_batch(const nvc_scene* sc, const nvc_camera* cam, uint64_t key_world, uint64_t key_screen,
                        uint64_t key_targets, uint64_t off_world, uint64_t off_screen, int32_t n_world,
                        int32_t n_screen, int32_t shard, int32_t n_shards, double* pos, float* tgt, int64_t* n_rows,
                        void* ws, void* stream) {
    NVC_REQUIRE(sc && cam && pos && n_rows && ws, "nvc_gen_train_batch: null argument");
    NVC_REQUIRE(n_world >= 0 && n_screen >= 0 && n_shards >= 1 && shard >= 0 && shard < n_shards,
                "nvc_gen_train_batch: bad counts/shard");
    cudaStream_t s = (cudaStream_t)stream;
    if (n_world > 0) k_world<<<grid1(3 * (int64_t)n_world, 256), 256, 0, s>>>(*sc, key_world, off_world, n_world, pos);
    if (n_screen > 0) {
        k_screen_round0<<<grid1(n_screen, 64), 64, 0, s>>>(*sc, *cam, key_screen, off_screen, n_screen, ws);
        k_screen_finish<<<1, 1024, 0, s>>>(*sc, *cam, key_screen, off_screen, n_world, n_screen, pos, n_rows, ws);
    } else {
        k_set_rows<<<1, 1, 0, s>>>(n_rows, n_world);
    }
    int rc = check_launch("k_screen");
    if (rc) return rc;
    const int64_t total = (int64_t)n_world + n_screen;
    const int64_t cap = total / n_shards + 1;
    if (tgt && total > 0) {
        if (cap <= kSortMax && sc->n_lights <= 65535 && !getenv("NVC_TARGETS_UNSORTED")) {
            int32_t* order = reinterpret_cast<int32_t*>((char*)ws + (64 + 25 * (int64_t)n_screen + 64 + 255) / 256 * 256);
            const int smem = (int)cap * 4;
            cudaFuncSetAttribute(k_morton_order, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            k_morton_order<<<1, 1024, smem, s>>>(*sc, pos, n_rows, 0, shard, n_shards, order);
            dim3 g(grid1(cap, 128), sc->n_lights);
            // (8 resident CTAs per SM -- 64 registers -- measured 97 vs 90 us standalone and
            // a frame within noise, so the register budget stays the compiler's)
            k_targets_sorted<1><<<g, 128, 0, s>>>(*sc, key_targets, pos, n_rows, 0, shard, n_shards, order, tgt);
        } else {
            k_targets<<<grid1(cap, 4), 128, 0, s>>>(*sc, key_targets, 0, pos, n_rows, 0, shard, n_shards, cap, tgt);
        }
    }
    return check_launch("k_targets");
}

int64_t nvc_cluster_workspace_bytes(int64_t b_max, int32_t m) {
    return ((b_max * m * 4 + 255) / 256) * 256 + 8 * (3 * (int64_t)m + 2) + 8 + 256;
}

int64_t nvc_cluster_state_offset(int64_t b_max, int32_t m) {   // int64 [m+2]: uni starts, next, kept
    return ((b_max * m * 4 + 255) / 256) * 256;
}

int nvc_cluster_targets(const nvc_scene* sc, uint64_t key, uint64_t offset, int64_t kept_in, const double* pos,
                        const int64_t* n_rows, int64_t b_max, int32_t shard, int32_t n_shards, int32_t m,
                        const int32_t* c_off, const int32_t* c_mem, float* tgt, void* ws, void* stream) {
    NVC_REQUIRE(sc && pos && n_rows && c_off && c_mem && tgt && ws, "nvc_cluster_targets: null argument");
    NVC_REQUIRE(m >= 1 && n_shards >= 1 && shard >= 0 && shard < n_shards, "nvc_cluster_targets: bad m/shard");
    if (b_max <= 0) return NVC_OK;
    cudaStream_t s = (cudaStream_t)stream;
    int32_t* picks = (int32_t*)ws;
    int64_t* uni = (int64_t*)((char*)ws + nvc_cluster_state_offset(b_max, m));
    int64_t* base = uni + (m + 2);
    int64_t* kept = base + m;
    int32_t* flag = (int32_t*)(kept + m);
    k_cluster_chain<<<1, 1, 0, s>>>(n_rows, m, c_off, offset, kept_in, uni, base, kept, flag);
    dim3 gd(grid1(b_max, 256), m);
    k_cluster_draws<<<gd, 256, 0, s>>>(key, n_rows, m, c_off, c_mem, base, kept, picks, uni, flag, kept_in);
    k_cluster_picks<<<1, kPickThreads, 0, s>>>(key, n_rows, m, c_off, c_mem, picks, uni,
                                               getenv("NVC_CLUSTER_EXACT_WALK") ? nullptr : flag, offset, kept_in);
    int rc = check_launch("k_cluster_picks");
    if (rc) return rc;
    const int64_t cap = b_max / n_shards + 1;
    dim3 g(grid1(cap, 128), m);
    k_cluster_tgt<<<g, 128, 0, s>>>(*sc, key, pos, n_rows, shard, n_shards, m, picks, uni, tgt);
    return check_launch("k_cluster_tgt");
}

int nvc_targets(const nvc_scene* sc, uint64_t key, uint64_t offset, const double* pos, int64_t b, float* tgt,
                void* stream) {
    NVC_REQUIRE(sc && pos && tgt, "nvc_targets: null argument");
    if (b <= 0) return NVC_OK;
    k_targets<<<grid1(b, 4), 128, 0, (cudaStream_t)stream>>>(*sc, key, offset, pos, nullptr, b, 0, 1, b, tgt);
    return check_launch("k_targets");
}

static RGrid rgrid(const nvc_rgrid* g) {
    return RGrid{g->y, g->point, g->w_y, g->w_sum, g->M, g->W, g->valid};
}
static RGridC rgridc(const nvc_rgrid* g) {
    return RGridC{g->y, g->point, g->w_y, g->w_sum, g->M, g->W, g->valid};
}

int64_t nvc_ris_workspace_bytes(int64_t p, int32_t m_cand, int32_t k) {
    return nvc_cluster_workspace_bytes(p * m_cand, 1) + 8 * ((int64_t)k + 2) + 256;
}

int nvc_ris_initial(const nvc_scene* sc, const void* lum, int32_t lum_f64, int64_t stride, int64_t p, int32_t m_cand,
                    uint64_t key, uint64_t offset, int64_t kept_in, const nvc_rgrid* out, void* ws,
                    int64_t* state_dev, void* stream) {
    NVC_REQUIRE(sc && lum && out && ws && state_dev, "nvc_ris_initial: null argument");
    NVC_REQUIRE(m_cand >= 1 && stride >= p, "nvc_ris_initial: bad candidate count / stride");
    if (p <= 0) return NVC_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t b = p * m_cand;
    const int32_t k = sc->n_lights;
    int32_t* picks = (int32_t*)ws;
    int64_t* uni = (int64_t*)((char*)ws + nvc_cluster_state_offset(b, 1));   // [uni0, next, kept]
    int64_t* base = uni + 3;
    int64_t* kept = base + 1;
    int32_t* flag = (int32_t*)(kept + 1);
    char* tail = (char*)ws + nvc_cluster_workspace_bytes(b, 1);
    int64_t* n_rows = (int64_t*)tail;
    int32_t* c_off = (int32_t*)(n_rows + 1);
    int32_t* c_mem = c_off + 2;
    k_ris_setup<<<grid1(k, 128), 128, 0, s>>>(c_off, c_mem, k, n_rows, b);
    // integers(0, K, (p, M)): Lemire on 32-bit halves, rejections and kept half exact
    k_cluster_chain<<<1, 1, 0, s>>>(n_rows, 1, c_off, offset, kept_in, uni, base, kept, flag);
    k_cluster_draws<<<dim3(grid1(b, 256), 1), 256, 0, s>>>(key, n_rows, 1, c_off, c_mem, base, kept, picks, uni, flag,
                                                           kept_in);
    k_cluster_picks<<<1, kPickThreads, 0, s>>>(key, n_rows, 1, c_off, c_mem, picks, uni,
                                               getenv("NVC_CLUSTER_EXACT_WALK") ? nullptr : flag, offset, kept_in);
    int rc = check_launch("k_cluster_picks");
    if (rc) return rc;
    if (lum_f64)
        k_ris_initial<double><<<grid1(p, 128), 128, 0, s>>>(*sc, (const double*)lum, stride, p, m_cand, picks, key, uni,
                                                            rgrid(out));
    else
        k_ris_initial<float><<<grid1(p, 128), 128, 0, s>>>(*sc, (const float*)lum, stride, p, m_cand, picks, key, uni,
                                                           rgrid(out));
    // the stream after the call: next output (uni0 + p*M + 2p) and the kept half
    cudaMemcpyAsync(state_dev, uni, 8, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(state_dev + 1, uni + 2, 8, cudaMemcpyDeviceToDevice, s);
    return check_launch("k_ris_initial");
}

int nvc_restir_temporal(const nvc_scene* sc, const double* factor, int64_t stride, const double* alb, int64_t p,
                        const nvc_rgrid* cur, const nvc_rgrid* prev, uint64_t key, uint64_t offset, double clamp,
                        int32_t clamp_mode, const nvc_rgrid* out, void* stream) {
    NVC_REQUIRE(sc && factor && alb && cur && prev && out, "nvc_restir_temporal: null argument");
    NVC_REQUIRE(clamp_mode == 0 || clamp_mode == 1, "nvc_restir_temporal: clamp_mode 0 (m) or 1 (contribution)");
    if (p <= 0) return NVC_OK;
    k_restir_temporal<<<grid1(p, 128), 128, 0, (cudaStream_t)stream>>>(*sc, factor, stride, alb, p, rgridc(cur),
                                                                        rgridc(prev), key, offset, clamp, clamp_mode,
                                                                        rgrid(out));
    return check_launch("k_restir_temporal");
}

int nvc_restir_spatial(const nvc_scene* sc, const double* factor, int64_t stride, const double* alb,
                       const double* nrm, const uint8_t* hit, const double* depth, int32_t width, int32_t height,
                       const nvc_rgrid* grid, uint64_t key, uint64_t offset, int32_t radius, int32_t neighbors,
                       const nvc_rgrid* out, void* stream) {
    NVC_REQUIRE(sc && factor && alb && nrm && hit && depth && grid && out, "nvc_restir_spatial: null argument");
    NVC_REQUIRE(width > 0 && height > 0 && neighbors >= 0, "nvc_restir_spatial: bad frame");
    NVC_REQUIRE(grid->y != out->y, "nvc_restir_spatial: the output grid must not alias the input");
    const int64_t p = (int64_t)width * height;
    k_restir_spatial<<<grid1(p, 128), 128, 0, (cudaStream_t)stream>>>(*sc, factor, stride, alb, nrm, hit, depth, width,
                                                                       height, rgridc(grid), key, offset, radius,
                                                                       neighbors, rgrid(out));
    return check_launch("k_restir_spatial");
}

int nvc_phat_ids(const nvc_scene* sc, const double* factor, int64_t stride, const double* alb, const int64_t* ids,
                 int64_t p, double* out, void* stream) {
    NVC_REQUIRE(sc && factor && alb && ids && out, "nvc_phat_ids: null argument");
    if (p <= 0) return NVC_OK;
    k_phat_ids<<<grid1(p, 128), 128, 0, (cudaStream_t)stream>>>(*sc, factor, stride, alb, ids, p, out);
    return check_launch("k_phat_ids");
}

}  // extern "C"
