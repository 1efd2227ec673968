// common.cuh -- shared device code for libnvc (sm_100a).
//
// Everything that has to reproduce the reference bit-for-bit uses explicit
// round-to-nearest intrinsics (__dmul_rn, __dadd_rn, ...) so no FMA
// contraction can creep in, whatever the TU's -fmad setting.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/nvc.h"

namespace nvc {

// ---------------------------------------------------------------------------
// error plumbing (host)
// ---------------------------------------------------------------------------
void set_error(const char* fmt, ...);
int check_launch(const char* what);

#define NVC_REQUIRE(cond, ...)              \
    do {                                    \
        if (!(cond)) {                      \
            ::nvc::set_error(__VA_ARGS__);  \
            return NVC_ERR_ARG;             \
        }                                   \
    } while (0)

// SM count of the current device (queried once per device; 148 on B200)
inline int num_sms() {
    static int cached[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cached[dev]) cudaDeviceGetAttribute(&cached[dev], cudaDevAttrMultiProcessorCount, dev);
    return cached[dev] > 0 ? cached[dev] : 1;
}

// fp32 SIMT inference (model.cu), used by nvc_infer(precision=0)
int nvc_infer_f32(const nvc_model* m, const double* pos, int64_t n, float* out, cudaStream_t s);

// ---------------------------------------------------------------------------
// Philox4x64-10, numpy-compatible random access (numpy Philox + rng.py:54-56).
// Draw n of a stream = lane n%4 of the block at counter n/4 + 1 (numpy
// increments the counter before producing its first buffer).
// ---------------------------------------------------------------------------
struct U4 {
    uint64_t x[4];
};

__device__ __forceinline__ U4 philox_block(uint64_t counter, uint64_t key) {
    uint64_t c0 = counter, c1 = 0, c2 = 0, c3 = 0, k0 = key, k1 = 0;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k0 += 0x9E3779B97F4A7C15ull;
            k1 += 0xBB67AE8584CAA73Bull;
        }
        const uint64_t hi0 = __umul64hi(0xD2E7470EE14C6C93ull, c0);
        const uint64_t lo0 = 0xD2E7470EE14C6C93ull * c0;
        const uint64_t hi1 = __umul64hi(0xCA5A826395121157ull, c2);
        const uint64_t lo1 = 0xCA5A826395121157ull * c2;
        c0 = hi1 ^ c1 ^ k0;
        c1 = lo1;
        c2 = hi0 ^ c3 ^ k1;
        c3 = lo0;
    }
    U4 o;
    o.x[0] = c0;
    o.x[1] = c1;
    o.x[2] = c2;
    o.x[3] = c3;
    return o;
}

// The same block when the counter fits in 32 bits (every stream position below
// 2^34 draws: all per-frame streams here) -- the first two rounds simplify
// because the counter words c1..c3 start at zero and the key words are known:
//   round 0: M0*c0 is a 64x32 product and M1*c2 = 0, so the state becomes
//            (key, 0, hi(M0*c0), lo(M0*c0));
//   round 1: M0*c0 = M0*key is a per-stream constant (PhiloxKey, once per thread).
// 1.5 of the 20 64x64->128 multiplies instead of 4 in those rounds.  Measured
// (tools/rooflines.py): the same block rate as philox_block once the compiler
// sees a 32-bit counter (it folds the zero words itself), so the kernels keep
// philox_block; this form is the microbenchmark's cross-check.
struct PhiloxKey {
    uint64_t key, mk_hi, mk_lo;   // mk = 0xD2E7470EE14C6C93 * key (128-bit)
};

__device__ __forceinline__ PhiloxKey philox_key(uint64_t key) {
    PhiloxKey k;
    k.key = key;
    k.mk_hi = __umul64hi(0xD2E7470EE14C6C93ull, key);
    k.mk_lo = 0xD2E7470EE14C6C93ull * key;
    return k;
}

__device__ __forceinline__ U4 philox_block32(uint32_t counter, const PhiloxKey& pk) {
    // round 0 (k0 = key, k1 = 0)
    const uint64_t p0 = 0xD2E7470EE14C6C93ull * (uint64_t)counter;            // lo(M0*c0)
    const uint64_t h0 = __umul64hi(0xD2E7470EE14C6C93ull, (uint64_t)counter);  // hi(M0*c0)
    // round 1 (k0 = key + W0, k1 = W1): c = (key, 0, h0, p0)
    const uint64_t hi1 = __umul64hi(0xCA5A826395121157ull, h0);
    const uint64_t lo1 = 0xCA5A826395121157ull * h0;
    uint64_t c0 = hi1 ^ (pk.key + 0x9E3779B97F4A7C15ull);
    uint64_t c1 = lo1;
    uint64_t c2 = pk.mk_hi ^ p0 ^ 0xBB67AE8584CAA73Bull;
    uint64_t c3 = pk.mk_lo;
    uint64_t k0 = pk.key + 0x9E3779B97F4A7C15ull, k1 = 0xBB67AE8584CAA73Bull;
#pragma unroll
    for (int r = 2; r < 10; ++r) {
        k0 += 0x9E3779B97F4A7C15ull;
        k1 += 0xBB67AE8584CAA73Bull;
        const uint64_t a_hi = __umul64hi(0xD2E7470EE14C6C93ull, c0);
        const uint64_t a_lo = 0xD2E7470EE14C6C93ull * c0;
        const uint64_t b_hi = __umul64hi(0xCA5A826395121157ull, c2);
        const uint64_t b_lo = 0xCA5A826395121157ull * c2;
        c0 = b_hi ^ c1 ^ k0;
        c1 = b_lo;
        c2 = a_hi ^ c3 ^ k1;
        c3 = a_lo;
    }
    U4 o;
    o.x[0] = c0;
    o.x[1] = c1;
    o.x[2] = c2;
    o.x[3] = c3;
    return o;
}

// numpy Generator.random(): (x >> 11) * 2^-53 (exact in binary64)
// Row range [lo, hi) of shard `shard` of n_shards over b rows (floor splits,
// as the host computes them).  One shard: no division; the usual batch sizes:
// 32-bit division instead of the ~70-instruction 64-bit one.
__device__ __forceinline__ void shard_range(int64_t b, int shard, int n_shards, int64_t& lo, int64_t& hi) {
    if (n_shards == 1) {
        lo = 0;
        hi = b;
    } else if ((uint64_t)b * (uint64_t)n_shards <= 0xffffffffull) {
        lo = (uint32_t)b * (uint32_t)shard / (uint32_t)n_shards;
        hi = (uint32_t)b * (uint32_t)(shard + 1) / (uint32_t)n_shards;
    } else {
        lo = b * shard / n_shards;
        hi = b * (shard + 1) / n_shards;
    }
}

__device__ __forceinline__ double u01(uint64_t x) { return (double)(x >> 11) * 0x1.0p-53; }

__device__ __forceinline__ double draw(uint64_t key, uint64_t n) {
    U4 b = philox_block(n / 4 + 1, key);
    return u01(b.x[n & 3]);
}

// two consecutive draws n, n+1 (n even): always inside one Philox block
__device__ __forceinline__ void draw2(uint64_t key, uint64_t n, double& a, double& b) {
    U4 blk = philox_block(n / 4 + 1, key);
    const int l = (int)(n & 3);
    a = u01(blk.x[l]);
    b = u01(blk.x[l + 1]);
}

// ---------------------------------------------------------------------------
// fixed-point gradients
// ---------------------------------------------------------------------------
__device__ __forceinline__ long long to_fx(double v) {
    return __double2ll_rn(v * 0x1.0p48);
}
__device__ __forceinline__ float from_fx(long long q) {
    return (float)((double)q * 0x1.0p-48);
}
// MLP gradients: a finer fixed point (2^-58, |g| < 32) -- they are summed from
// per-32-row-block partials (shard-exact) and weight gradients at init are
// ~1e-9, where 2^-48 per partial would cost ~1e-4 relative
__device__ __forceinline__ long long to_fx_mlp(double v) {
    return __double2ll_rn(v * 0x1.0p58);
}
__device__ __forceinline__ float from_fx_mlp(long long q) {
    return (float)((double)q * 0x1.0p-58);
}
__device__ __forceinline__ void red_add_fx(int64_t* p, long long v) {
    if (v != 0)
        asm volatile("red.global.add.u64 [%0], %1;" ::"l"(p), "l"((unsigned long long)v) : "memory");
}

// ---------------------------------------------------------------------------
// hash-grid addressing: hashgrid.py:94-114 (exact FP64 index math)
// ---------------------------------------------------------------------------
struct GridDev {
    int L, F;
    uint32_t tmask;
    int64_t T;
    int res[NVC_MAX_LEVELS];
    int dense[NVC_MAX_LEVELS];
    double lo[3], span[3];
};

inline GridDev grid_of(const nvc_model* m) {
    GridDev g;
    g.L = m->levels;
    g.F = m->features;
    g.T = m->table_size;
    g.tmask = (uint32_t)(m->table_size - 1);
    for (int l = 0; l < NVC_MAX_LEVELS; ++l) {
        g.res[l] = m->resolution[l];
        g.dense[l] = m->dense[l];
    }
    for (int a = 0; a < 3; ++a) {
        g.lo[a] = m->aabb_min[a];
        g.span[a] = m->span[a];
    }
    return g;
}

// q = clip((p - lo) / span, 0, 1)      (hashgrid.py:94-97)
__device__ __forceinline__ void normalize(const GridDev& g, const double* p, double q[3]) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        double v = __ddiv_rn(__dsub_rn(p[a], g.lo[a]), g.span[a]);
        q[a] = fmin(fmax(v, 0.0), 1.0);
    }
}

// per-level cell origin (int) and fractional offset (f64)  (hashgrid.py:100-103)
__device__ __forceinline__ void cell(int n, const double q[3], int c0[3], double f[3]) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double x = __dmul_rn(q[a], (double)n);
        int c = (int)x;  // trunc == floor for x >= 0
        c = min(c, n - 1);
        c0[a] = c;
        f[a] = __dsub_rn(x, (double)c);
    }
}

// vertex address of corner (bx,by,bz)   (hashgrid.py:104-114, 82-87)
__device__ __forceinline__ uint32_t corner_index(const GridDev& g, int l, const int c0[3], int bx,
                                                 int by, int bz) {
    const uint32_t x = (uint32_t)(c0[0] + bx), y = (uint32_t)(c0[1] + by), z = (uint32_t)(c0[2] + bz);
    if (g.dense[l]) {
        const uint32_t m = (uint32_t)g.res[l] + 1u;
        return x + m * (y + m * z);
    }
    return (x + y * 2654435761u + z * 805459861u) & g.tmask;
}

// trilinear weight of corner c = 4bx+2by+bz: (wx*wy)*wz in FP64 (hashgrid.py:105-107)
__device__ __forceinline__ double corner_weight(const double f[3], int c) {
    const double wx = (c & 4) ? f[0] : __dsub_rn(1.0, f[0]);
    const double wy = (c & 2) ? f[1] : __dsub_rn(1.0, f[1]);
    const double wz = (c & 1) ? f[2] : __dsub_rn(1.0, f[2]);
    return __dmul_rn(__dmul_rn(wx, wy), wz);
}

// ---------------------------------------------------------------------------
// tcgen05 operand layout: fp16, K-major, 8-row core groups, swizzled by the
// row within the group (SWIZZLE_32B/64B/128B chosen by the row width), the
// canonical layout UMMA descriptors describe.  Shared by the packed weights
// (written by the Adam / shadow kernels) and the A tiles of the query kernel.
// ---------------------------------------------------------------------------
__host__ __device__ inline int umma_kpad(int k) { return k <= 16 ? 16 : (k <= 32 ? 32 : (k + 63) / 64 * 64); }
__host__ __device__ inline int umma_sw_bytes(int kp) { return kp * 2 >= 128 ? 128 : kp * 2; }

// log2 of the swizzle row width in bytes for a padded K (kp in {16, 32, 64k})
__host__ __device__ __forceinline__ int umma_sw_log2(int kp) { return kp >= 64 ? 7 : (kp == 32 ? 6 : 5); }

// byte offset of element (r, k) in a [rows x kp] tile (rows % 8 == 0)
__host__ __device__ __forceinline__ uint32_t umma_off(int r, int k, int rows, int kp) {
    const int lg = umma_sw_log2(kp);
    const uint32_t kb = (uint32_t)k * 2u;
    const uint32_t atom = kb >> lg, within = kb & ((1u << lg) - 1u);
    const uint32_t cs = (within >> 4) ^ ((uint32_t)(r & 7) >> (7 - lg));
    return (atom * (uint32_t)rows << lg) + ((uint32_t)r << lg) + (cs << 4) + (within & 15u);
}

// per-layer padded N (rows of W) and K: hidden widths are padded like the next
// layer's K so the A1 tile never carries stale columns
__host__ __device__ inline void umma_pads(const int* dims, int n_layers, int* np, int* kp) {
    for (int l = 0; l < n_layers; ++l) {
        np[l] = (l < n_layers - 1) ? umma_kpad(dims[l + 1]) : (dims[l + 1] + 15) / 16 * 16;
        kp[l] = l == 0 ? umma_kpad(dims[0]) : np[l - 1];
    }
}

// halfs of one packed weight block, rounded to 1024 B so every block starts
// on a swizzle-atom boundary
__host__ __device__ inline int64_t umma_block_halfs(int np, int kp) { return ((int64_t)np * kp + 511) / 512 * 512; }

// ---------------------------------------------------------------------------
// fp16 query table in x-pair layout: slot e of level l holds the F features of
// entry e followed by those of entry next(e) = (e+1) mod T within the level.
// The spatial hash adds x with prime 1, so corner (x0+1, y, z) always lives in
// next(slot of (x0, y, z)) (dense levels: slot+1): one 2F-half load fetches
// both x-neighbours, halving the gather instructions of the encoder.
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ int64_t pair_next(int64_t e, int64_t T) { return (e & ~(T - 1)) | ((e + 1) & (T - 1)); }
__host__ __device__ __forceinline__ int64_t pair_prev(int64_t e, int64_t T) { return (e & ~(T - 1)) | ((e - 1) & (T - 1)); }

// ---------------------------------------------------------------------------
// scene helpers
// ---------------------------------------------------------------------------
// Scene.light_points (scene.py:204-215): id < 0 -> light 0; edges from vertices
__device__ __forceinline__ void light_point(const nvc_scene& sc, int64_t id, double u0, double u1,
                                            double out[3]) {
    const int j = id < 0 ? 0 : (int)id;
    const double* v = sc.lt_verts + 12 * j;
    if (sc.lt_kind[j] == 1) {
        out[0] = v[0];
        out[1] = v[1];
        out[2] = v[2];
        return;
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double eu = __dsub_rn(v[3 + a], v[a]);
        const double ev = __dsub_rn(v[9 + a], v[a]);
        out[a] = __dadd_rn(__dadd_rn(v[a], __dmul_rn(u0, eu)), __dmul_rn(u1, ev));
    }
}

__device__ __forceinline__ double norm3(double x, double y, double z) {
    return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z)));
}


// ---------------------------------------------------------------------------
// mbarrier / bulk-copy (TMA) helpers shared by the streaming kernels
// ---------------------------------------------------------------------------
namespace tma {
__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_init_fence() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void bar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@P1 bra DONE_%=;\n\t"
        "bra WAIT_%=;\n"
        "DONE_%=:\n\t}" ::"r"(s32(bar)),
        "r"(phase), "r"(1000000u)
        : "memory");
}
__device__ __forceinline__ void bar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(bar)), "r"(bytes) : "memory");
}
// global -> shared, completion counted on `bar`
__device__ __forceinline__ void load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     s32(dst)),
                 "l"(src), "r"(bytes), "r"(s32(bar))
                 : "memory");
}
// shared -> global, tracked by bulk groups
__device__ __forceinline__ void store(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(s32(src)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// generic-proxy shared-memory writes -> visible to the async proxy (bulk store)
__device__ __forceinline__ void fence_shared() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
}  // namespace tma

}  // namespace nvc
