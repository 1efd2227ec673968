/* oracle/geom.c -- TEST INFRASTRUCTURE ONLY (the parity checker, never shipped).
 *
 * Plain-C restatement of the reference's numba geometry kernels, compiled
 * with -ffp-contract=off so every double op rounds exactly as the
 * reference's serial numba/LLVM code does ("FMA
 * contraction").  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs load this library.
 *
 * Reference functions restated (file:line under /root/reference/pkg/src/viscache):
 *   orc_ray_tri        <- kernels.py:20-56   (Moller-Trumbore, inclusive edges)
 *   aabb_hit           <- kernels.py:59-83   (slab test)
 *   inv_dir            <- kernels.py:86-90
 *   orc_closest_hit_batch <- kernels.py:93-137, 177-191 (stack BVH, push L then R)
 *   orc_any_hit_batch  <- kernels.py:140-174, 194-203
 *   rect_factor        <- kernels.py:220-281 (horizon clip + edge-arc sum)
 *   point_factor       <- kernels.py:284-296
 *   orc_light_factors  <- kernels.py:299-316 (light_factors_all)
 */
#include <math.h>
#include <stdint.h>

#define STACK_DEPTH 64
#define KIND_RECT 0

typedef struct {
    const double *node_min, *node_max;      /* (n_nodes, 3) */
    const int32_t *left, *right, *start, *count;
    const double *v0, *v1, *v2;             /* (n_tris, 3), BVH leaf order */
    int64_t n_tris;
} bvh_t;

double orc_ray_tri(double ox, double oy, double oz, double dx, double dy, double dz,
                   const double *a, const double *b, const double *c,
                   double t_min, double t_max)
{
    double e1x = b[0] - a[0], e1y = b[1] - a[1], e1z = b[2] - a[2];
    double e2x = c[0] - a[0], e2y = c[1] - a[1], e2z = c[2] - a[2];
    double px = dy * e2z - dz * e2y;
    double py = dz * e2x - dx * e2z;
    double pz = dx * e2y - dy * e2x;
    double det = e1x * px + e1y * py + e1z * pz;
    if (fabs(det) < 1e-14) return -1.0;
    double inv = 1.0 / det;
    double tx = ox - a[0], ty = oy - a[1], tz = oz - a[2];
    double u = (tx * px + ty * py + tz * pz) * inv;
    if (u < 0.0 || u > 1.0) return -1.0;
    double qx = ty * e1z - tz * e1y;
    double qy = tz * e1x - tx * e1z;
    double qz = tx * e1y - ty * e1x;
    double v = (dx * qx + dy * qy + dz * qz) * inv;
    if (v < 0.0 || u + v > 1.0) return -1.0;
    double t = (e2x * qx + e2y * qy + e2z * qz) * inv;
    if (t < t_min || t > t_max) return -1.0;
    return t;
}

static int aabb_hit(double ox, double oy, double oz, double ix, double iy, double iz,
                    const double *bmin, const double *bmax, double t_max)
{
    double t0 = (bmin[0] - ox) * ix, t1 = (bmax[0] - ox) * ix, tmp;
    if (t0 > t1) { tmp = t0; t0 = t1; t1 = tmp; }
    double lo = t0, hi = t1;
    t0 = (bmin[1] - oy) * iy; t1 = (bmax[1] - oy) * iy;
    if (t0 > t1) { tmp = t0; t0 = t1; t1 = tmp; }
    if (t0 > lo) lo = t0;
    if (t1 < hi) hi = t1;
    t0 = (bmin[2] - oz) * iz; t1 = (bmax[2] - oz) * iz;
    if (t0 > t1) { tmp = t0; t0 = t1; t1 = tmp; }
    if (t0 > lo) lo = t0;
    if (t1 < hi) hi = t1;
    return hi >= lo && lo <= t_max && hi >= 0.0;
}

static double inv_dir(double d)
{
    if (fabs(d) < 1e-300) return d >= 0.0 ? 1e300 : -1e300;
    return 1.0 / d;
}

static int64_t closest_one(const bvh_t *b, const double *o, const double *d,
                           double t_min, double t_max, double *t_out)
{
    if (b->n_tris == 0) { *t_out = -1.0; return -1; }
    double ix = inv_dir(d[0]), iy = inv_dir(d[1]), iz = inv_dir(d[2]);
    double best_t = t_max;
    int64_t best = -1;
    int32_t stack[STACK_DEPTH];
    int top = 0;
    stack[top++] = 0;
    while (top > 0) {
        int32_t n = stack[--top];
        if (!aabb_hit(o[0], o[1], o[2], ix, iy, iz, b->node_min + 3 * n, b->node_max + 3 * n, best_t))
            continue;
        int32_t cnt = b->count[n];
        if (cnt > 0) {
            int32_t s = b->start[n];
            for (int32_t k = s; k < s + cnt; ++k) {
                double t = orc_ray_tri(o[0], o[1], o[2], d[0], d[1], d[2],
                                       b->v0 + 3 * k, b->v1 + 3 * k, b->v2 + 3 * k, t_min, best_t);
                if (t >= 0.0) { best_t = t; best = k; }
            }
        } else {
            stack[top++] = b->left[n];
            stack[top++] = b->right[n];
        }
    }
    *t_out = best < 0 ? -1.0 : best_t;
    return best;
}

static int any_one(const bvh_t *b, const double *o, const double *d, double t_min, double t_max)
{
    if (b->n_tris == 0) return 0;
    double ix = inv_dir(d[0]), iy = inv_dir(d[1]), iz = inv_dir(d[2]);
    int32_t stack[STACK_DEPTH];
    int top = 0;
    stack[top++] = 0;
    while (top > 0) {
        int32_t n = stack[--top];
        if (!aabb_hit(o[0], o[1], o[2], ix, iy, iz, b->node_min + 3 * n, b->node_max + 3 * n, t_max))
            continue;
        int32_t cnt = b->count[n];
        if (cnt > 0) {
            int32_t s = b->start[n];
            for (int32_t k = s; k < s + cnt; ++k)
                if (orc_ray_tri(o[0], o[1], o[2], d[0], d[1], d[2],
                                b->v0 + 3 * k, b->v1 + 3 * k, b->v2 + 3 * k, t_min, t_max) >= 0.0)
                    return 1;
        } else {
            stack[top++] = b->left[n];
            stack[top++] = b->right[n];
        }
    }
    return 0;
}

/* out_tri holds the BVH-order triangle index (-1 on miss); the caller maps
 * it through perm exactly as geometry.py:542-543 does. */
void orc_closest_hit_batch(int64_t n, const double *orig, const double *dir,
                           const double *t_min, const double *t_max,
                           const double *node_min, const double *node_max,
                           const int32_t *left, const int32_t *right,
                           const int32_t *start, const int32_t *count,
                           const double *v0, const double *v1, const double *v2, int64_t n_tris,
                           double *out_t, int64_t *out_tri)
{
    bvh_t b = {node_min, node_max, left, right, start, count, v0, v1, v2, n_tris};
    for (int64_t i = 0; i < n; ++i)
        out_tri[i] = closest_one(&b, orig + 3 * i, dir + 3 * i, t_min[i], t_max[i], out_t + i);
}

void orc_any_hit_batch(int64_t n, const double *orig, const double *dir,
                       const double *t_min, const double *t_max,
                       const double *node_min, const double *node_max,
                       const int32_t *left, const int32_t *right,
                       const int32_t *start, const int32_t *count,
                       const double *v0, const double *v1, const double *v2, int64_t n_tris,
                       uint8_t *out_hit)
{
    bvh_t b = {node_min, node_max, left, right, start, count, v0, v1, v2, n_tris};
    for (int64_t i = 0; i < n; ++i)
        out_hit[i] = (uint8_t)any_one(&b, orig + 3 * i, dir + 3 * i, t_min[i], t_max[i]);
}

static double rect_factor(const double *p, const double *nrm, const double *verts,
                          const double *ln)
{
    double side = (p[0] - verts[0]) * ln[0] + (p[1] - verts[1]) * ln[1] + (p[2] - verts[2]) * ln[2];
    if (side <= 0.0) return 0.0;
    double vx[4], vy[4], vz[4], cx[8], cy[8], cz[8];
    for (int i = 0; i < 4; ++i) {
        vx[i] = verts[3 * i + 0] - p[0];
        vy[i] = verts[3 * i + 1] - p[1];
        vz[i] = verts[3 * i + 2] - p[2];
    }
    int nc = 0;
    for (int i = 0; i < 4; ++i) {
        int j = (i + 1) % 4;
        double di = vx[i] * nrm[0] + vy[i] * nrm[1] + vz[i] * nrm[2];
        double dj = vx[j] * nrm[0] + vy[j] * nrm[1] + vz[j] * nrm[2];
        if (di >= 0.0) { cx[nc] = vx[i]; cy[nc] = vy[i]; cz[nc] = vz[i]; ++nc; }
        if ((di > 0.0 && dj < 0.0) || (di < 0.0 && dj > 0.0)) {
            double s = di / (di - dj);
            cx[nc] = vx[i] + s * (vx[j] - vx[i]);
            cy[nc] = vy[i] + s * (vy[j] - vy[i]);
            cz[nc] = vz[i] + s * (vz[j] - vz[i]);
            ++nc;
        }
    }
    if (nc < 3) return 0.0;
    for (int i = 0; i < nc; ++i) {
        double l = sqrt(cx[i] * cx[i] + cy[i] * cy[i] + cz[i] * cz[i]);
        if (l < 1e-12) return 0.0;
        cx[i] /= l; cy[i] /= l; cz[i] /= l;
    }
    double acc = 0.0;
    for (int i = 0; i < nc; ++i) {
        int j = (i + 1) % nc;
        double d = cx[i] * cx[j] + cy[i] * cy[j] + cz[i] * cz[j];
        if (d > 1.0) d = 1.0; else if (d < -1.0) d = -1.0;
        double st = 1.0 - d * d;
        st = sqrt(st > 0.0 ? st : 0.0);
        double ratio = st < 1e-9 ? 1.0 : acos(d) / st;
        double gx = cy[i] * cz[j] - cz[i] * cy[j];
        double gy = cz[i] * cx[j] - cx[i] * cz[j];
        double gz = cx[i] * cy[j] - cy[i] * cx[j];
        acc += ratio * (gx * nrm[0] + gy * nrm[1] + gz * nrm[2]);
    }
    return 0.5 * fabs(acc);
}

static double point_factor(const double *p, const double *nrm, const double *l)
{
    double wx = l[0] - p[0], wy = l[1] - p[1], wz = l[2] - p[2];
    double d2 = wx * wx + wy * wy + wz * wz;
    if (d2 < 1e-24) return 0.0;
    double inv = 1.0 / sqrt(d2);
    double c = (wx * nrm[0] + wy * nrm[1] + wz * nrm[2]) * inv;
    if (c <= 0.0) return 0.0;
    return c / d2;
}

/* out is (n, k) row-major, as light_factors_all writes it. */
void orc_light_factors(int64_t n, const double *pos, const double *nrm, int64_t k,
                       const uint8_t *kind, const double *verts, const double *lnormal,
                       double *out)
{
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < k; ++j)
            out[i * k + j] = kind[j] == KIND_RECT
                ? rect_factor(pos + 3 * i, nrm + 3 * i, verts + 12 * j, lnormal + 3 * j)
                : point_factor(pos + 3 * i, nrm + 3 * i, verts + 12 * j);
}

/* numpy/OpenBLAS float64 (r,3)@(3,c) as it rounds here (pinned by
 * tests/golden/clusters.npz): gemm shapes fma(a2,b2, fma(a1,b1, a0*b0)),
 * gemv shapes (r == 1 or c == 1) fma(a2,b2, fma(a0,b0, a1*b1)). */
void orc_dot3_fma(int64_t n, const double *a, const double *b, int32_t gemv, double *out) {
    for (int64_t i = 0; i < n; ++i) {
        const double *x = a + 3 * i, *y = b + 3 * i;
        out[i] = gemv ? fma(x[2], y[2], fma(x[0], y[0], x[1] * y[1]))
                      : fma(x[2], y[2], fma(x[1], y[1], x[0] * y[0]));
    }
}
