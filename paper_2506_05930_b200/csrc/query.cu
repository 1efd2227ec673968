// query.cu -- the hot path: fused hash-grid encode -> tcgen05/TMEM MLP ->
// {visibility out | clamp * lum -> WRS -> light point | Neural DI}, one pass
// per 128-pixel tile (SURVEY table K: K1 perf mode, K2, K7, K8), plus the
// standalone WRS kernels used for parity on given weights.
//
// Reference routines (under /root/reference/pkg/src/viscache):
//   VisibilityCache.infer cache.py:54-58, encode_batch hashgrid.py:117-131,
//   forward mlp.py:110-140, clamp_visibility sampling.py:27-30,
//   wrs_select_batch :74-85, nls_weights_batch :184-191,
//   nls_sample_batch :194-205, neural_di_batch :215-218,
//   PixelCtx.unshadowed_rgb :157-160, Scene.light_points scene.py:204-215.
//
// Tile pipeline (one CTA = 4 warps = 128 threads = 128 pixels = M of one
// tcgen05.mma; thread t owns pixel row t, which is TMEM lane t):
//   1. every thread encodes its pixel: FP64 cell/hash (bit-exact indices),
//      half2 gathers from the fp16 shadow table (L2-resident), FP32 blend,
//      fp16 features stored into the A tile in the UMMA K-major
//      no-swizzle core-matrix layout;
//   2. per layer one elected thread issues K/16 tcgen05.mma (M=128, N=width,
//      A and B from smem descriptors, D in TMEM) and commits to an mbarrier;
//   3. the 4 warps drain TMEM with tcgen05.ld 32x32b.x16 (16 columns per
//      thread), add bias, activate, and write the next A tile (fp16);
//   4. after the last layer each thread holds its pixel's K visibilities and
//      runs the sequential FP64 reservoir (exactly the reference cumsum/
//      compare order) with numpy-Philox uniforms, or the Neural-DI sum.
// Several CTAs per SM overlap their gather phase with each other's MMA chain.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"

namespace nvc {
namespace {

constexpr int kTile = 128;

// ---------------------------------------------------------------------------
// tcgen05 / mbarrier helpers (inline PTX, sm_100a)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

// try_wait with a suspend-time hint: the waiting thread sleeps in hardware
// until the phase completes (or 1 ms passes) instead of spinning on issue slots
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
#ifndef NVC_WAIT_NOHINT
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@P1 bra DONE_%=;\n\t"
        "bra WAIT_%=;\n"
        "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
        "r"(phase), "r"(1000000u)
        : "memory");
#else
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE_%=;\n\t"
        "bra WAIT_%=;\n"
        "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
#endif
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// UMMA shared-memory descriptor of k-step kk (16 fp16 along K) of a K-major
// swizzled [rows x kp] tile at smem address `base` (layout: common.cuh umma_off).
// Start address advances 32 B per k-step inside a swizzle atom (the hardware
// swizzles absolute address bits, so atoms must be atom-size aligned); SBO is
// the 8-row group pitch; LBO is unused for swizzled K-major (1).
__device__ __forceinline__ uint64_t umma_desc(uint32_t base, int rows, int kp, int kk) {
    const int lg = umma_sw_log2(kp);
    const uint32_t kb = (uint32_t)kk * 32u;
    const uint32_t addr = base + ((kb >> lg) * (uint32_t)rows << lg) + (kb & ((1u << lg) - 1u));
    const uint64_t layout = lg == 7 ? 2ull : (lg == 6 ? 4ull : 6ull);
    uint64_t d = 0;
    d |= (uint64_t)((addr & 0x3FFFFu) >> 4);
    d |= (uint64_t)1 << 16;                                   // LBO (unused when swizzled)
    d |= (uint64_t)((8u << lg) >> 4) << 32;                   // SBO: 8-row group pitch
    d |= (uint64_t)1 << 46;                                   // descriptor version (sm_100)
    d |= layout << 61;
    return d;
}

// instruction descriptor: kind::f16, A/B = f16, D = f32, both K-major, M=128
__host__ __device__ constexpr uint32_t idesc_f16(int n) {
    return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(kTile >> 4) << 24);
}

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float v[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// ---------------------------------------------------------------------------
// kernel parameters
// ---------------------------------------------------------------------------
struct QNet {
    int n_layers;
    int dims[NVC_MAX_LAYERS + 1];
    int np[NVC_MAX_LAYERS];          // padded N (multiple of 16)
    int kp[NVC_MAX_LAYERS];          // padded K (multiple of 16)
    int wofs[NVC_MAX_LAYERS];        // halfs offset of layer i in wpack
    int64_t boff[NVC_MAX_LAYERS];    // bias offset in params
    int wpack_halfs;
    int hidden_kp;                   // max padded hidden width (A1 tile K)
    int tmem_cols;
    float alpha;
    int out_sigmoid;
    // smem carve-up (bytes)
    int sm_wpack, sm_a0, sm_a1, sm_bias, sm_lum, sm_lp, sm_total;
};

enum Mode { kModeVis = 0, kModeNls = 1, kModeNdi = 2 };

struct QOut {
    int mode;
    float* vis;                       // kModeVis: (P, K)
    const void* lum;                  // kModeNls: light-major lum, kModeNdi: factor
    int lum_f64;
    int64_t stride;                   // light-major stride
    int64_t p_first, p_total;
    uint64_t key, offset;
    double floor;
    int64_t* ids;
    double* pts;
    double* big_w;
    const double* albedo;             // kModeNdi
    double* rgb;                      // kModeNdi
    const uint32_t* nz_mask;          // optional: bit k of word p set <=> table[k][p] != 0 (K <= 32)
    int dbg;                          // profiling switches (NVC_QUERY_DEBUG), 0 in production
};

// streaming reservoir state of one pixel (wrs_select_batch, sequential FP64)
struct Reservoir {
    double s, wsel;
    int sel;
    uint64_t blk;       // cached Philox block index (n/4+1), 0 = none
    U4 u;
};

// one out-of-line copy of the 10-round Philox keeps the fused kernel's
// instruction footprint inside the SM instruction cache
__device__ __noinline__ U4 philox_call(uint64_t counter, uint64_t key) { return philox_block(counter, key); }

__device__ __forceinline__ double draw_cached(Reservoir& r, uint64_t key, uint64_t n) {
    const uint64_t b = n / 4 + 1;
    if (b != r.blk) {
        r.u = philox_call(b, key);
        r.blk = b;
    }
    return u01(r.u.x[n & 3]);
}

__device__ __forceinline__ void reservoir_push(Reservoir& r, double w, int k, uint64_t key, uint64_t n) {
    r.s = __dadd_rn(r.s, w);
    if (w > 0.0) {   // u*s < 0 is impossible: zero-weight lights never need a uniform
        const double u = draw_cached(r, key, n);
        if (__dmul_rn(u, r.s) < w) {
            r.sel = k;
            r.wsel = w;
        }
    }
}

__device__ __forceinline__ void draw_pair(uint64_t key, uint64_t n, double& a, double& b) {
    const U4 blk = philox_call(n / 4 + 1, key);
    a = u01(blk.x[n & 3]);
    if ((n & 3) != 3) {
        b = u01(blk.x[(n & 3) + 1]);
    } else {
        const U4 nb = philox_call(n / 4 + 2, key);
        b = u01(nb.x[0]);
    }
}

// ---------------------------------------------------------------------------
// encode one pixel into the A0 tile (fp16 shadow table, FP32 blend)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t a_off(int row, int k, int kp) {   // bytes, 128-row A tile
    return umma_off(row, k, kTile, kp);
}

// cell origin and fraction without int<->double conversions: adding 2^52
// with round-down leaves floor(x) in the low mantissa bits.  Bit-identical to
// c0 = min(int(x), n-1); f = x - c0 (hashgrid.py:100-103).
__device__ __forceinline__ void cell_fast(int n, const double q[3], uint32_t c0[3], float f[3]) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double x = __dmul_rn(q[a], (double)n);
        const double t = __dadd_rd(x, 0x1p52);
        uint32_t c = (uint32_t)__double2loint(t);
        double fr = __dsub_rn(x, __dsub_rn(t, 0x1p52));
        if (c > (uint32_t)(n - 1)) {   // x == n exactly (q == 1): reference clamps, f = 1
            c = (uint32_t)(n - 1);
            fr = 1.0;
        }
        c0[a] = c;
        f[a] = (float)fr;
    }
}

struct LevelAddr {
    uint32_t base, sy, sz, mask;
};

__device__ __forceinline__ LevelAddr level_addr(const GridDev& g, int l, const uint32_t c0[3]) {
    LevelAddr a;
    if (g.dense[l]) {
        const uint32_t m = (uint32_t)g.res[l] + 1u;
        a.sy = m;
        a.sz = m * m;
        a.mask = 0xffffffffu;
    } else {
        a.sy = 2654435761u;
        a.sz = 805459861u;
        a.mask = g.tmask;
    }
    a.base = c0[0] + c0[1] * a.sy + c0[2] * a.sz;
    return a;
}

// F == 2: four levels per batch; each level needs 4 x-pair loads (8 B: both
// x-neighbours' 2 features) from the pair table, 16 loads in flight per batch;
// FP32 blend; one 16-byte store of the 4 levels' 8 features
__device__ __forceinline__ void encode_row2(const GridDev& g, const __half2* __restrict__ table, const double q[3],
                                            uint8_t* a0, int row, int kp0) {
    constexpr int LB = 4;
    const uint2* t2 = reinterpret_cast<const uint2*>(table);
    for (int l = 0; l < g.L; l += LB) {
        uint2 v[LB][4];
        float w[LB][3];
#pragma unroll
        for (int j = 0; j < LB; ++j) {
            if (l + j < g.L) {
                uint32_t c0[3];
                cell_fast(g.res[l + j], q, c0, w[j]);
                const LevelAddr ad = level_addr(g, l + j, c0);
                const uint2* tl = t2 + (size_t)(l + j) * (size_t)g.T;
#pragma unroll
                for (int c = 0; c < 4; ++c)    // (y, z) corner pair: slots of (x0,y,z) and (x0+1,y,z)
                    v[j][c] = __ldg(tl + ((ad.base + ((c >> 1) & 1) * ad.sy + (c & 1) * ad.sz) & ad.mask));
            }
        }
        __align__(16) __half2 out[LB];
#pragma unroll
        for (int j = 0; j < LB; ++j) {
            float a = 0.0f, b = 0.0f;
            if (l + j < g.L) {
                const float fx = w[j][0], fy = w[j][1], fz = w[j][2];
                const float wy[2] = {1.0f - fy, fy}, wz[2] = {1.0f - fz, fz};
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const float wyz = wy[(c >> 1) & 1] * wz[c & 1];
                    const float w0 = (1.0f - fx) * wyz, w1 = fx * wyz;
                    const float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(&v[j][c].x));
                    const float2 f1 = __half22float2(*reinterpret_cast<const __half2*>(&v[j][c].y));
                    a = fmaf(w0, f0.x, a);
                    b = fmaf(w0, f0.y, b);
                    a = fmaf(w1, f1.x, a);
                    b = fmaf(w1, f1.y, b);
                }
            }
            out[j] = __floats2half2_rn(a, b);
        }
        if (l + LB <= g.L) {
#pragma unroll
            for (int qq = 0; qq < LB / 4; ++qq)
                *reinterpret_cast<uint4*>(a0 + a_off(row, 2 * (l + 4 * qq), kp0)) =
                    *reinterpret_cast<const uint4*>(out + 4 * qq);
        } else {
            for (int j = 0; l + j < g.L; ++j) *reinterpret_cast<__half2*>(a0 + a_off(row, 2 * (l + j), kp0)) = out[j];
        }
    }
}

__device__ __forceinline__ void encode_rowF(const GridDev& g, const __half* __restrict__ table, const double q[3],
                                            uint8_t* a0, int row, int kp0) {
    for (int l = 0; l < g.L; ++l) {
        uint32_t c0[3];
        float f[3];
        cell_fast(g.res[l], q, c0, f);
        const LevelAddr ad = level_addr(g, l, c0);
        const float wy[2] = {1.0f - f[1], f[1]}, wz[2] = {1.0f - f[2], f[2]};
        const __half* tl = table + (size_t)l * (size_t)g.T * 2 * g.F;
        float acc[8];
        for (int k = 0; k < g.F; ++k) acc[k] = 0.0f;
        for (int c = 0; c < 4; ++c) {
            const uint32_t slot = (ad.base + ((c >> 1) & 1) * ad.sy + (c & 1) * ad.sz) & ad.mask;
            const float wyz = wy[(c >> 1) & 1] * wz[c & 1];
            const float w0 = (1.0f - f[0]) * wyz, w1 = f[0] * wyz;
            const __half* s2 = tl + (size_t)slot * 2 * g.F;
            for (int k = 0; k < g.F; ++k)
                acc[k] = fmaf(w1, __half2float(__ldg(s2 + g.F + k)), fmaf(w0, __half2float(__ldg(s2 + k)), acc[k]));
        }
        for (int k = 0; k < g.F; ++k)
            *reinterpret_cast<__half*>(a0 + a_off(row, l * g.F + k, kp0)) = __float2half_rn(acc[k]);
    }
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// ---------------------------------------------------------------------------
// the fused kernel: warp-specialised, two tiles in flight per CTA
//   warps 0-3  epilogue (TMEM lane quarter = warp): bias/act -> A1, final layer
//              -> visibility / WRS / Neural DI
//   warps 4-7  encode: pixel rows of the next tile -> A0[stage]
//   warp  8    control: TMEM alloc, tcgen05.mma issue, bulk prefetch of the
//              tile's light-major lum/factor rows into smem
// TMEM holds two accumulators (tile i uses buffer i%2), so layer 0 of tile
// i+1 runs while the epilogue walks the hidden layers of tile i.
// ---------------------------------------------------------------------------
// ---- profiling trace (NVC_QUERY_DEBUG & 128): CTA 0 logs (globaltimer, event) ----
__device__ unsigned long long g_trace[8192];
__device__ unsigned int g_trace_n;
__device__ __forceinline__ void trace_ev(const QOut& o, int code) {
#ifndef NVC_TRACE
    return;
#endif
    if (!(o.dbg & 128) || blockIdx.x != 0) return;
    const unsigned long long t = clock64();
    const unsigned int i = atomicAdd(&g_trace_n, 1u);
    if (i < 8192) g_trace[i] = (t << 16) | (unsigned)code;
}

constexpr int kEpiWarps = 4, kEncWarps = 4, kCtlWarp = kEpiWarps + kEncWarps;
constexpr int kQThreads = 32 * (kEpiWarps + kEncWarps + 1);

// every slot s in {0,1} is one tile of the current pair (tile 2j+s)
struct QBars {
    uint64_t a0_full[2], a0_empty[2], acc_full[2], acc_empty[2], a1_full[2], lum_full[2], lum_empty[2];
};

__device__ __forceinline__ bool bulk_ok(const QOut& o, int64_t tile, int64_t P) {
    return o.mode != kModeVis && !(o.dbg & 16) && !o.lum_f64 && (o.stride & 3) == 0 && ((uintptr_t)o.lum & 15) == 0 &&
           (tile + 1) * kTile <= P;
}

// Tiles are processed in pairs (A = slot 0, B = slot 1) that ping-pong through
// the layer chain: while the tensor core runs layer l+1 of A the epilogue
// warps drain layer l of B, so MMA latency hides behind the other tile's
// epilogue.  Each slot owns an A0 stage, a TMEM accumulator, an A1 tile and a
// lum stage.
template <int kMode, bool kF2>
__global__ void __launch_bounds__(kQThreads, 2) k_query(GridDev g, QNet net, const float* __restrict__ params,
                                                        const __half* __restrict__ table,
                                                        const uint16_t* __restrict__ wpack,
                                                        const double* __restrict__ pos, int64_t P, nvc_scene sc,
                                                        QOut o) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ QBars bars;
    __shared__ uint32_t tmem_base_s;
    // swizzle atoms need 1024-B aligned shared addresses
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* s_w = smem + net.sm_wpack;
    uint8_t* s_a0 = smem + net.sm_a0;            // 2 stages
    uint8_t* s_a1 = smem + net.sm_a1;            // 2 slots
    float* s_bias = reinterpret_cast<float*>(smem + net.sm_bias);
    float* s_lum = reinterpret_cast<float*>(smem + net.sm_lum);   // 2 slots of K x 128
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int K = net.dims[net.n_layers];
    const int a0_stage = kTile * net.kp[0] * 2;
    const int a1_stage = kTile * net.hidden_kp * 2;
    const int lum_stage = K * kTile;

    // ---- setup ----
    {
        const int n16 = net.wpack_halfs / 8;
        const uint4* src = reinterpret_cast<const uint4*>(wpack);
        uint4* dst = reinterpret_cast<uint4*>(s_w);
        for (int i = tid; i < n16; i += kQThreads) dst[i] = __ldg(src + i);
        int bo = 0;
        for (int l = 0; l < net.n_layers; ++l) {
            for (int n = tid; n < net.np[l]; n += kQThreads)
                s_bias[bo + n] = n < net.dims[l + 1] ? __ldg(params + net.boff[l] + n) : 0.0f;
            bo += net.np[l];
        }
        const uint4 z = make_uint4(0, 0, 0, 0);
        for (int i = tid; i < 2 * a0_stage / 16; i += kQThreads) reinterpret_cast<uint4*>(s_a0)[i] = z;
    }
    if (warp == kCtlWarp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)),
                     "r"(net.tmem_cols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        for (int s = 0; s < 2; ++s) {
            mbar_init(&bars.a0_full[s], 32 * kEncWarps);
            mbar_init(&bars.a0_empty[s], 1);
            mbar_init(&bars.acc_full[s], 1);
            mbar_init(&bars.acc_empty[s], 32 * kEpiWarps);
            mbar_init(&bars.a1_full[s], 32 * kEpiWarps);
            mbar_init(&bars.lum_full[s], 1);
            mbar_init(&bars.lum_empty[s], 32 * kEpiWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_s;
    const uint32_t acc_cols = (uint32_t)net.tmem_cols / 2;
    const int64_t ntiles = (P + kTile - 1) / kTile;
    const int n_local = ntiles > blockIdx.x ? (int)((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;
    const int n_pairs = (n_local + 1) / 2;

    if (warp == kCtlWarp) {
        // ======================= control =======================
        // whole warp: lane 0 issues MMAs / commits / expect_tx, all 32 lanes
        // issue the per-light bulk copies of the lum rows in parallel
        {
            const uint32_t a0_addr = smem_u32(s_a0), a1_addr = smem_u32(s_a1), w_addr = smem_u32(s_w);
            uint32_t a1_cnt[2] = {0, 0}, lum_uses[2] = {0, 0};
            auto issue_layer = [&](int l, int slot) {
                if (lane != 0) return;
                const uint32_t a_base = l == 0 ? a0_addr + (uint32_t)(slot * a0_stage) : a1_addr + (uint32_t)(slot * a1_stage);
                const uint32_t b_base = w_addr + 2u * net.wofs[l];
                const uint32_t idesc = idesc_f16(net.np[l]);
                const uint32_t d = tmem + (uint32_t)slot * acc_cols;
                tc_fence_after();
                for (int kk = 0; kk < net.kp[l] / 16; ++kk) {
                    const uint64_t ad = umma_desc(a_base, kTile, net.kp[l], kk);
                    const uint64_t bd = umma_desc(b_base, net.np[l], net.kp[l], kk);
                    mma_f16(d, ad, bd, idesc, kk > 0 ? 1u : 0u);
                }
            };
            for (int j = 0; j < n_pairs; ++j) {
                const int nt = min(2, n_local - 2 * j);
                for (int s = 0; s < nt; ++s) {            // layer 0 of both tiles
                    mbar_wait(&bars.a0_full[s], j & 1);
                    if (lane == 0) trace_ev(o, 0x100 | s);
                    if (j >= 1) mbar_wait(&bars.acc_empty[s], (j - 1) & 1);
                    if (lane == 0) trace_ev(o, 0x200 | s);
                    issue_layer(0, s);
                    if (lane == 0) {
                        mma_commit(&bars.a0_empty[s]);
                        mma_commit(&bars.acc_full[s]);
                        trace_ev(o, 0x300 | s);
                    }
                    __syncwarp();
                }
                for (int s = 0; s < nt; ++s) {            // lum rows of both tiles (slot frees after pair j-1)
                    const int64_t tile = blockIdx.x + (int64_t)(2 * j + s) * gridDim.x;
                    if (!bulk_ok(o, tile, P) || (o.dbg & 16)) continue;
                    if (lum_uses[s] > 0) mbar_wait(&bars.lum_empty[s], (lum_uses[s] - 1) & 1);
                    if (lane == 0) mbar_expect_tx(&bars.lum_full[s], (uint32_t)(K * kTile * 4));
                    __syncwarp();
                    const float* src = reinterpret_cast<const float*>(o.lum) + tile * kTile;
                    for (int k = lane; k < K; k += 32)
                        bulk_g2s(s_lum + s * lum_stage + k * kTile, src + (int64_t)k * o.stride, kTile * 4,
                                 &bars.lum_full[s]);
                    ++lum_uses[s];
                }
                for (int l = 1; l < net.n_layers; ++l)     // hidden layers, ping-pong A/B
                    for (int s = 0; s < nt; ++s) {
                        mbar_wait(&bars.a1_full[s], a1_cnt[s] & 1);
                        if (lane == 0) trace_ev(o, 0x400 | (l << 4) | s);
                        ++a1_cnt[s];
                        issue_layer(l, s);
                        if (lane == 0) {
                            mma_commit(&bars.acc_full[s]);
                            trace_ev(o, 0x500 | (l << 4) | s);
                        }
                        __syncwarp();
                    }
            }
        }
    } else if (warp >= kEpiWarps) {
        // ======================= encode =======================
        const int row = tid - 32 * kEpiWarps;
        for (int i = 0; i < n_local; ++i) {
            const int s = i & 1;
            uint8_t* a0 = s_a0 + s * a0_stage;
            if (i >= 2) mbar_wait(&bars.a0_empty[s], ((i >> 1) - 1) & 1);
            const int64_t p = (blockIdx.x + (int64_t)i * gridDim.x) * kTile + row;
            if (p < P && !(o.dbg & 1)) {
                const double pp[3] = {__ldg(pos + 3 * p), __ldg(pos + 3 * p + 1), __ldg(pos + 3 * p + 2)};
                double q[3];
                normalize(g, pp, q);
                if constexpr (kF2)
                    encode_row2(g, reinterpret_cast<const __half2*>(table), q, a0, row, net.kp[0]);
                else
                    encode_rowF(g, table, q, a0, row, net.kp[0]);
            } else {
                for (int k = 0; k < net.dims[0]; ++k)
                    *reinterpret_cast<__half*>(a0 + a_off(row, k, net.kp[0])) = __float2half_rn(0.0f);
            }
            fence_async_smem();
            mbar_arrive(&bars.a0_full[s]);
            if (row == 0) trace_ev(o, 0x900 | s);
        }
    } else {
        // ======================= epilogue =======================
        const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
        uint32_t acc_cnt[2] = {0, 0}, lum_uses[2] = {0, 0};
        for (int j = 0; j < n_pairs; ++j) {
            const int nt = min(2, n_local - 2 * j);
            int bias_off = 0;
            for (int l = 0; l < net.n_layers; ++l) {
                const bool last = l == net.n_layers - 1;
                for (int s = 0; s < nt; ++s) {
                    const uint32_t t_acc = tmem + lane_base + (uint32_t)s * acc_cols;
                    mbar_wait(&bars.acc_full[s], acc_cnt[s] & 1);
                    if (tid == 0) trace_ev(o, 0x600 | (l << 4) | s);
                    ++acc_cnt[s];
                    tc_fence_after();
                    if (!last) {
                        uint8_t* a1 = s_a1 + s * a1_stage;
                        for (int c = 0; c < net.np[l] / 16; ++c) {
                            float v[16];
                            tmem_ld16(t_acc + (uint32_t)(c * 16), v);
                            __align__(16) __half2 h[8];
                            const float2* bb = reinterpret_cast<const float2*>(s_bias + bias_off + c * 16);
                            const __half2 al = __float2half2_rn(net.alpha);
#pragma unroll
                            for (int jj = 0; jj < 8; ++jj) {
                                const float2 bj = bb[jj];
                                const __half2 z = __floats2half2_rn(v[2 * jj] + bj.x, v[2 * jj + 1] + bj.y);
                                h[jj] = __hmax2(z, __hmul2(z, al));
                            }
                            *reinterpret_cast<uint4*>(a1 + a_off(tid, c * 16, net.np[l])) = *reinterpret_cast<const uint4*>(h);
                            *reinterpret_cast<uint4*>(a1 + a_off(tid, c * 16 + 8, net.np[l])) =
                                *reinterpret_cast<const uint4*>(h + 4);
                        }
                        fence_async_smem();
                        tc_fence_before();
                        mbar_arrive(&bars.a1_full[s]);
                        if (tid == 0) trace_ev(o, 0x700 | (l << 4) | s);
                        continue;
                    }
                    // ---- final layer of tile 2j+s ----
                    const int64_t tile = blockIdx.x + (int64_t)(2 * j + s) * gridDim.x;
                    const int64_t p = tile * kTile + tid;
                    const bool valid = p < P;
                    const int64_t gp = o.p_first + p;
                    const bool bulk = bulk_ok(o, tile, P);
                    if (bulk) mbar_wait(&bars.lum_full[s], lum_uses[s] & 1);
                    const float* lrow = s_lum + s * lum_stage + tid;
                    // zero-weight lights add 0 to the running sum and are never
                    // selected, so skipping them (nz_mask) is exact
                    uint32_t nzm = 0xffffffffu;
                    if (kMode != kModeVis && o.nz_mask != nullptr && K <= 32 && valid) nzm = __ldg(o.nz_mask + p);
                    double s_sum = 0.0, wsel = 0.0;
                    int sel = -1;
                    uint64_t blk = 0;
                    U4 ublk;
                    double rgb[3] = {0.0, 0.0, 0.0};
                    for (int c = 0; c < net.np[l] / 16; ++c) {
                        float v[16];
                        tmem_ld16(t_acc + (uint32_t)(c * 16), v);
                        if (!valid || (o.dbg & 4)) continue;
                        const uint32_t cm = (c * 16 < 32) ? (nzm >> (c * 16)) & 0xffffu : 0xffffu;
                        if (kMode != kModeVis && cm == 0) continue;
#pragma unroll
                        for (int jj = 0; jj < 16; ++jj) {
                            const int k = c * 16 + jj;
                            if (k >= K) break;
                            if (kMode != kModeVis && !((cm >> jj) & 1u)) continue;
                            const float z = v[jj] + s_bias[bias_off + k];
                            float a;
                            if (net.out_sigmoid) {
                                const float e = __expf(-fabsf(z));
                                const float r = __fdividef(1.0f, 1.0f + e);
                                a = z >= 0.0f ? r : e * r;
                                a = fminf(fmaxf(a, 1e-6f), 0.999999f);
                            } else {
                                a = z >= 0.0f ? z : net.alpha * z;
                            }
                            if (kMode == kModeVis) {
                                o.vis[p * K + k] = a;
                                continue;
                            }
                            double t;
                            if (bulk)
                                t = (double)lrow[k * kTile];
                            else if (o.lum_f64)
                                t = __ldg(reinterpret_cast<const double*>(o.lum) + (int64_t)k * o.stride + p);
                            else
                                t = (double)__ldg(reinterpret_cast<const float*>(o.lum) + (int64_t)k * o.stride + p);
                            if (kMode == kModeNls) {
                                double vv = (double)a;
                                vv = o.floor > 0.0 ? fmax(vv, o.floor) : fmax(vv, 0.0);
                                const double w = __dmul_rn(vv, t);
                                s_sum = __dadd_rn(s_sum, w);
                                if (w > 0.0 && (o.dbg & 2)) {
                                    if (__dmul_rn(0.5, s_sum) < w) {
                                        sel = k;
                                        wsel = w;
                                    }
                                } else if (w > 0.0) {   // u*s < 0 is impossible: zero weights need no uniform
                                    const uint64_t n = o.offset + (uint64_t)gp * (uint64_t)K + (uint64_t)k;
                                    const uint64_t bi = n / 4 + 1;
                                    if (bi != blk) {
                                        ublk = philox_call(bi, o.key);
                                        blk = bi;
                                    }
                                    if (__dmul_rn(u01(ublk.x[n & 3]), s_sum) < w) {
                                        sel = k;
                                        wsel = w;
                                    }
                                }
                            } else {
                                const double wk = __dmul_rn((double)a, t);
#pragma unroll
                                for (int ch = 0; ch < 3; ++ch)
                                    rgb[ch] = __dadd_rn(rgb[ch], __dmul_rn(wk, __ldg(sc.lt_radiance + 3 * k + ch)));
                            }
                        }
                    }
                    tc_fence_before();
                    mbar_arrive(&bars.acc_empty[s]);
                    if (tid == 0) trace_ev(o, 0x800 | s);
                    if (bulk) {
                        mbar_arrive(&bars.lum_empty[s]);
                        ++lum_uses[s];
                    }
                    if (kMode == kModeNls && valid && !(o.dbg & 64)) {
                        double u0 = 0.5, u1 = 0.5, y[3];
                        if (!(o.dbg & 32))
                            draw_pair(o.key, o.offset + (uint64_t)o.p_total * (uint64_t)K + 2ull * (uint64_t)gp, u0, u1);
                        light_point(sc, sel, u0, u1, y);
                        o.ids[p] = sel;
                        o.big_w[p] = sel >= 0 ? __ddiv_rn(s_sum, wsel > 0.0 ? wsel : 1.0) : 0.0;
                        o.pts[3 * p] = y[0];
                        o.pts[3 * p + 1] = y[1];
                        o.pts[3 * p + 2] = y[2];
                    } else if (kMode == kModeNdi && valid) {
#pragma unroll
                        for (int ch = 0; ch < 3; ++ch)
                            o.rgb[3 * p + ch] = __ddiv_rn(__dmul_rn(rgb[ch], o.albedo[3 * p + ch]), 3.141592653589793);
                    }
                }
                bias_off += net.np[l];
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == kCtlWarp)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(net.tmem_cols) : "memory");
}

// ---------------------------------------------------------------------------
// standalone WRS on given weights (parity entry points)
// ---------------------------------------------------------------------------
__global__ void k_wrs_select(const double* __restrict__ w, int64_t P, int K, uint64_t key, uint64_t offset,
                             int64_t* __restrict__ idx, double* __restrict__ wsel, double* __restrict__ wsum) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    Reservoir r;
    r.s = 0.0;
    r.wsel = 0.0;
    r.sel = -1;
    r.blk = 0;
    for (int k = 0; k < K; ++k) reservoir_push(r, w[p * K + k], k, key, offset + (uint64_t)p * K + k);
    idx[p] = r.sel;
    wsel[p] = r.sel >= 0 ? r.wsel : 0.0;
    wsum[p] = r.s;
}

template <typename T>
__global__ void k_nls_from_vis(nvc_scene sc, const float* __restrict__ vis, const T* __restrict__ lum, int64_t stride,
                               int64_t P, int K, int64_t p_first, int64_t p_total, uint64_t key, uint64_t offset,
                               double floor, int64_t* __restrict__ ids, double* __restrict__ pts,
                               double* __restrict__ big_w) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    const int64_t gp = p_first + p;
    Reservoir r;
    r.s = 0.0;
    r.wsel = 0.0;
    r.sel = -1;
    r.blk = 0;
    for (int k = 0; k < K; ++k) {
        double v = (double)vis[p * K + k];
        v = floor > 0.0 ? fmax(v, floor) : fmax(v, 0.0);
        reservoir_push(r, __dmul_rn(v, (double)lum[(int64_t)k * stride + p]), k, key,
                       offset + (uint64_t)gp * K + k);
    }
    double u0, u1, y[3];
    draw_pair(key, offset + (uint64_t)p_total * K + 2ull * gp, u0, u1);
    light_point(sc, r.sel, u0, u1, y);
    ids[p] = r.sel;
    big_w[p] = r.sel >= 0 ? __ddiv_rn(r.s, r.wsel > 0.0 ? r.wsel : 1.0) : 0.0;
    pts[3 * p] = y[0];
    pts[3 * p + 1] = y[1];
    pts[3 * p + 2] = y[2];
}

template <typename T>
__global__ void k_table_mask(const T* __restrict__ t, int64_t stride, int64_t P, int K, uint32_t* __restrict__ mask) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int w = blockIdx.y;
    if (p >= P) return;
    uint32_t m = 0;
    for (int j = 0; j < 32 && 32 * w + j < K; ++j)
        if (t[(int64_t)(32 * w + j) * stride + p] != (T)0) m |= 1u << j;
    mask[(int64_t)w * stride + p] = m;
}

inline int grid1(int64_t n, int bs) { return (int)((n + bs - 1) / bs); }

int make_qnet(const nvc_model* m, QNet& q, bool with_lum) {
    NVC_REQUIRE(m && m->params && m->table_h && m->wpack, "tcgen05 path: model state not bound");
    NVC_REQUIRE(m->n_layers >= 1 && m->n_layers <= NVC_MAX_LAYERS, "n_layers out of range");
    NVC_REQUIRE(m->dims[0] == m->levels * m->features, "dims[0] must equal levels*features");
    q.n_layers = m->n_layers;
    int64_t wo = 0, bo = (int64_t)m->levels * m->table_size * m->features;
    int hid = 16, maxnp = 16;
    for (int i = 0; i <= m->n_layers; ++i) q.dims[i] = m->dims[i];
    for (int i = 0; i < m->n_layers; ++i) {
        if (m->dims[i] > 256 || m->dims[i + 1] > 256) {
            set_error("tcgen05 path: layer widths must be <= 256");
            return NVC_ERR_UNSUPPORTED;
        }
    }
    umma_pads(m->dims, m->n_layers, q.np, q.kp);
    for (int i = 0; i < m->n_layers; ++i) {
        if (q.np[i] > 256 || q.kp[i] > 256) {
            set_error("tcgen05 path: padded layer widths must be <= 256");
            return NVC_ERR_UNSUPPORTED;
        }
        q.wofs[i] = (int)wo;
        wo += umma_block_halfs(q.np[i], q.kp[i]);
        bo += (int64_t)m->dims[i + 1] * m->dims[i];
        q.boff[i] = bo;
        bo += m->dims[i + 1];
        if (i >= 1 && q.kp[i] > hid) hid = q.kp[i];
        if (q.np[i] > maxnp) maxnp = q.np[i];
    }
    q.wpack_halfs = (int)wo;
    q.hidden_kp = hid;
    int cols = 32;
    while (cols < 2 * maxnp) cols <<= 1;      // two accumulators (tiles i, i+1)
    if (cols > 512) {
        set_error("tcgen05 path: %d TMEM columns needed", cols);
        return NVC_ERR_UNSUPPORTED;
    }
    q.tmem_cols = cols;
    q.alpha = m->alpha;
    q.out_sigmoid = m->out_sigmoid;
    int nb = 0;
    for (int i = 0; i < m->n_layers; ++i) nb += q.np[i];
    const int K = m->dims[m->n_layers];
    q.sm_wpack = 0;
    q.sm_a0 = (q.wpack_halfs * 2 + 1023) / 1024 * 1024;
    q.sm_a1 = q.sm_a0 + 2 * ((kTile * q.kp[0] * 2 + 1023) / 1024 * 1024);
    q.sm_bias = q.sm_a1 + 2 * ((kTile * q.hidden_kp * 2 + 1023) / 1024 * 1024);
    q.sm_lum = q.sm_bias + (nb * 4 + 127) / 128 * 128;
    q.sm_lp = q.sm_lum;
    q.sm_total = q.sm_lum + (with_lum ? 2 * K * kTile * 4 : 0) + 2048;   // + runtime 1024-B alignment
    if (q.sm_total > 226 * 1024) {
        set_error("tcgen05 path: %d bytes of shared memory needed", q.sm_total);
        return NVC_ERR_UNSUPPORTED;
    }
    return NVC_OK;
}

// ---------------------------------------------------------------------------
// Flat variant: every warp of a 4-warp CTA runs encode -> MMA chain -> epilogue
// for its own 128-pixel tile; many CTAs per SM (one activation buffer, 64
// TMEM columns each) give the SM independent tiles to interleave, which hides
// gather / MMA / dependent-FP64 latency better than the role-split kernel.
// ---------------------------------------------------------------------------
template <int kMode, bool kF2>
__global__ void __launch_bounds__(kTile, 4) k_query_flat(GridDev g, QNet net, const float* __restrict__ params,
                                                         const __half* __restrict__ table,
                                                         const uint16_t* __restrict__ wpack,
                                                         const double* __restrict__ pos, int64_t P, nvc_scene sc,
                                                         QOut o) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint64_t mbar;
    __shared__ uint32_t tmem_base_s;
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* s_w = smem + net.sm_wpack;
    uint8_t* s_act = smem + net.sm_a0;
    float* s_bias = reinterpret_cast<float*>(smem + net.sm_bias);
    const int tid = threadIdx.x, warp = tid >> 5;
    const int K = net.dims[net.n_layers];

    {
        const int n16 = net.wpack_halfs / 8;
        const uint4* src = reinterpret_cast<const uint4*>(wpack);
        uint4* dst = reinterpret_cast<uint4*>(s_w);
        for (int i = tid; i < n16; i += kTile) dst[i] = __ldg(src + i);
        int bo = 0;
        for (int l = 0; l < net.n_layers; ++l) {
            for (int n = tid; n < net.np[l]; n += kTile)
                s_bias[bo + n] = n < net.dims[l + 1] ? __ldg(params + net.boff[l] + n) : 0.0f;
            bo += net.np[l];
        }
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)),
                     "r"(net.tmem_cols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        mbar_init(&mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_s;
    const uint32_t t_row = tmem + ((uint32_t)(warp * 32) << 16);
    const uint32_t act_addr = smem_u32(s_act), w_addr = smem_u32(s_w);
    uint32_t phase = 0;
    const int64_t ntiles = (P + kTile - 1) / kTile;
    const int64_t tile0 = blockIdx.x;
    double pn[3] = {0.0, 0.0, 0.0};    // next tile's position (prefetched)
    if (tile0 < ntiles && tile0 * kTile + tid < P) {
        const int64_t p = tile0 * kTile + tid;
        pn[0] = __ldg(pos + 3 * p);
        pn[1] = __ldg(pos + 3 * p + 1);
        pn[2] = __ldg(pos + 3 * p + 2);
    }
    for (int64_t tile = tile0; tile < ntiles; tile += gridDim.x) {
        const int64_t p = tile * kTile + tid;
        const bool valid = p < P;
        const int64_t gp = o.p_first + p;
        if (tid == 0) trace_ev(o, 0x100);
        // ---- encode (layer-0 layout) ----
        if ((o.dbg & 256) && valid) {
            pn[0] = __ldg(pos + 3 * p);
            pn[1] = __ldg(pos + 3 * p + 1);
            pn[2] = __ldg(pos + 3 * p + 2);
        }
        if (valid && !(o.dbg & 1)) {
            double q[3];
            normalize(g, pn, q);
            if constexpr (kF2)
                encode_row2(g, reinterpret_cast<const __half2*>(table), q, s_act, tid, net.kp[0]);
            else
                encode_rowF(g, table, q, s_act, tid, net.kp[0]);
        } else {
            for (int k = 0; k < net.kp[0]; ++k)
                *reinterpret_cast<__half*>(s_act + a_off(tid, k, net.kp[0])) = __float2half_rn(0.0f);
        }
        if (!valid || (o.dbg & 1)) {
        } else if (net.kp[0] > net.dims[0]) {
            for (int k = net.dims[0]; k < net.kp[0]; ++k)
                *reinterpret_cast<__half*>(s_act + a_off(tid, k, net.kp[0])) = __float2half_rn(0.0f);
        }
        if (tid == 0) trace_ev(o, 0x200);
        fence_async_smem();
        tc_fence_before();
        __syncthreads();
        if (tid == 0) trace_ev(o, 0x300);
        if (!(o.dbg & 256)) {   // prefetch the next tile's position (after the proxy fence: no pending loads at fences)
            const int64_t pq = (tile + gridDim.x) * kTile + tid;
            if (tile + gridDim.x < ntiles && pq < P) {
                pn[0] = __ldg(pos + 3 * pq);
                pn[1] = __ldg(pos + 3 * pq + 1);
                pn[2] = __ldg(pos + 3 * pq + 2);
            }
        }

        uint32_t nzm = 0xffffffffu;
        if (kMode != kModeVis && o.nz_mask != nullptr && K <= 32 && valid) nzm = __ldg(o.nz_mask + p);
        double s_sum = 0.0, wsel = 0.0;
        int sel = -1;
        uint64_t blk = 0;
        U4 ublk;
        double rgb[3] = {0.0, 0.0, 0.0};
        int bias_off = 0;
        for (int l = 0; l < net.n_layers; ++l) {
            const bool last = l == net.n_layers - 1;
            if (tid == 0) {
                tc_fence_after();
                const uint32_t idesc = idesc_f16(net.np[l]);
                const uint32_t b_base = w_addr + 2u * net.wofs[l];
                for (int kk = 0; kk < net.kp[l] / 16; ++kk)
                    mma_f16(tmem, umma_desc(act_addr, kTile, net.kp[l], kk), umma_desc(b_base, net.np[l], net.kp[l], kk),
                            idesc, kk > 0 ? 1u : 0u);
                mma_commit(&mbar);
            }
            // prefetch the first 16 table values of this pixel while the MMA runs
            float lpre[16];
            const bool bulkless = kMode != kModeVis && !o.lum_f64;
            if (last && bulkless && valid) {
                const float* lp = reinterpret_cast<const float*>(o.lum) + p;
#pragma unroll
                for (int jj = 0; jj < 16; ++jj)
                    lpre[jj] = (jj < K && ((nzm >> jj) & 1u)) ? __ldg(lp + (int64_t)jj * o.stride) : 0.0f;
            }
            if (tid == 0) trace_ev(o, 0x400 | (l << 4));
            mbar_wait(&mbar, phase);
            if (tid == 0) trace_ev(o, 0x500 | (l << 4));
            phase ^= 1;
            tc_fence_after();
            if (!last) {
                for (int c = 0; c < net.np[l] / 16; ++c) {
                    float v[16];
                    tmem_ld16(t_row + (uint32_t)(c * 16), v);
                    __align__(16) __half2 h[8];
                    const float2* bb = reinterpret_cast<const float2*>(s_bias + bias_off + c * 16);
                    const __half2 al = __float2half2_rn(net.alpha);
#pragma unroll
                    for (int jj = 0; jj < 8; ++jj) {
                        const float2 bj = bb[jj];
                        const __half2 z = __floats2half2_rn(v[2 * jj] + bj.x, v[2 * jj + 1] + bj.y);
                        h[jj] = __hmax2(z, __hmul2(z, al));
                    }
                    *reinterpret_cast<uint4*>(s_act + a_off(tid, c * 16, net.np[l])) = *reinterpret_cast<const uint4*>(h);
                    *reinterpret_cast<uint4*>(s_act + a_off(tid, c * 16 + 8, net.np[l])) =
                        *reinterpret_cast<const uint4*>(h + 4);
                }
                if (tid == 0) trace_ev(o, 0x600 | (l << 4));
                fence_async_smem();
                tc_fence_before();
                __syncthreads();
                if (tid == 0) trace_ev(o, 0x700 | (l << 4));
            } else {
                for (int c = 0; c < net.np[l] / 16; ++c) {
                    float v[16];
                    tmem_ld16(t_row + (uint32_t)(c * 16), v);
                    if (!valid || (o.dbg & 4)) continue;
                    const uint32_t cm = (c * 16 < 32) ? (nzm >> (c * 16)) & 0xffffu : 0xffffu;
                    float lcur[16];
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj) lcur[jj] = lpre[jj];
                    if (bulkless && (c + 1) * 16 < K) {     // next chunk's table values
                        const float* lp = reinterpret_cast<const float*>(o.lum) + p;
                        const uint32_t nm = ((c + 1) * 16 < 32) ? (nzm >> ((c + 1) * 16)) : 0xffffffffu;
#pragma unroll
                        for (int jj = 0; jj < 16; ++jj)
                            lpre[jj] = ((c + 1) * 16 + jj < K && ((nm >> jj) & 1u))
                                           ? __ldg(lp + (int64_t)((c + 1) * 16 + jj) * o.stride)
                                           : 0.0f;
                    }
                    if (kMode != kModeVis && cm == 0) continue;
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj) {
                        const int k = c * 16 + jj;
                        if (k >= K) break;
                        if (kMode != kModeVis && !((cm >> jj) & 1u)) continue;
                        const float z = v[jj] + s_bias[bias_off + k];
                        float a;
                        if (net.out_sigmoid) {
                            const float e = __expf(-fabsf(z));
                            const float r = __fdividef(1.0f, 1.0f + e);
                            a = z >= 0.0f ? r : e * r;
                            a = fminf(fmaxf(a, 1e-6f), 0.999999f);
                        } else {
                            a = z >= 0.0f ? z : net.alpha * z;
                        }
                        if (kMode == kModeVis) {
                            o.vis[p * K + k] = a;
                            continue;
                        }
                        const double t = o.lum_f64
                                             ? __ldg(reinterpret_cast<const double*>(o.lum) + (int64_t)k * o.stride + p)
                                             : (double)lcur[jj];
                        if (kMode == kModeNls) {
                            double vv = (double)a;
                            vv = o.floor > 0.0 ? fmax(vv, o.floor) : fmax(vv, 0.0);
                            const double w = __dmul_rn(vv, t);
                            s_sum = __dadd_rn(s_sum, w);
                            if (w > 0.0) {   // u*s < 0 is impossible: zero weights need no uniform
                                const uint64_t n = o.offset + (uint64_t)gp * (uint64_t)K + (uint64_t)k;
                                const uint64_t bi = n / 4 + 1;
                                if (bi != blk) {
                                    ublk = philox_call(bi, o.key);
                                    blk = bi;
                                }
                                if (__dmul_rn(u01(ublk.x[n & 3]), s_sum) < w) {
                                    sel = k;
                                    wsel = w;
                                }
                            }
                        } else {
                            const double wk = __dmul_rn((double)a, t);
#pragma unroll
                            for (int ch = 0; ch < 3; ++ch)
                                rgb[ch] = __dadd_rn(rgb[ch], __dmul_rn(wk, __ldg(sc.lt_radiance + 3 * k + ch)));
                        }
                    }
                }
                tc_fence_before();
            }
            bias_off += net.np[l];
        }
        if (tid == 0) trace_ev(o, 0x800);
        if (kMode == kModeNls && valid) {
            double u0, u1, y[3];
            draw_pair(o.key, o.offset + (uint64_t)o.p_total * (uint64_t)K + 2ull * (uint64_t)gp, u0, u1);
            light_point(sc, sel, u0, u1, y);
            o.ids[p] = sel;
            o.big_w[p] = sel >= 0 ? __ddiv_rn(s_sum, wsel > 0.0 ? wsel : 1.0) : 0.0;
            o.pts[3 * p] = y[0];
            o.pts[3 * p + 1] = y[1];
            o.pts[3 * p + 2] = y[2];
        } else if (kMode == kModeNdi && valid) {
#pragma unroll
            for (int ch = 0; ch < 3; ++ch)
                o.rgb[3 * p + ch] = __ddiv_rn(__dmul_rn(rgb[ch], o.albedo[3 * p + ch]), 3.141592653589793);
        }
        if (tid == 0) trace_ev(o, 0x900);
        __syncthreads();   // activation buffer / TMEM reused by the next tile
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(net.tmem_cols) : "memory");
}

int make_qnet_flat(const nvc_model* m, QNet& q) {
    int rc = make_qnet(m, q, false);
    if (rc) return rc;
    int cols = 32;
    int maxnp = 16;
    for (int i = 0; i < q.n_layers; ++i) maxnp = max(maxnp, q.np[i]);
    while (cols < maxnp) cols <<= 1;
    q.tmem_cols = cols;
    int nb = 0;
    for (int i = 0; i < q.n_layers; ++i) nb += q.np[i];
    const int act_k = max(q.kp[0], q.hidden_kp);
    q.sm_wpack = 0;
    q.sm_a0 = (q.wpack_halfs * 2 + 1023) / 1024 * 1024;
    q.sm_a1 = q.sm_a0;
    q.sm_bias = q.sm_a0 + (kTile * act_k * 2 + 1023) / 1024 * 1024;
    q.sm_lum = q.sm_lp = q.sm_bias + (nb * 4 + 127) / 128 * 128;
    q.sm_total = q.sm_lum + 1024;
    return NVC_OK;
}

int launch_query_flat(const nvc_model* m, const double* pos, int64_t P, const nvc_scene* sc, const QOut& od,
                      cudaStream_t s) {
    QNet q;
    int rc = make_qnet_flat(m, q);
    if (rc) return rc;
    if (P <= 0) return NVC_OK;
    GridDev g = grid_of(m);
    const bool f2 = g.F == 2;
    auto kern = k_query_flat<kModeVis, true>;
    if (od.mode == kModeVis) kern = f2 ? k_query_flat<kModeVis, true> : k_query_flat<kModeVis, false>;
    else if (od.mode == kModeNls) kern = f2 ? k_query_flat<kModeNls, true> : k_query_flat<kModeNls, false>;
    else kern = f2 ? k_query_flat<kModeNdi, true> : k_query_flat<kModeNdi, false>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, q.sm_total);
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncAttributes fa;
    int regs = 128;
    if (cudaFuncGetAttributes(&fa, kern) == cudaSuccess) regs = fa.numRegs;
    cudaGetLastError();
    const int by_smem = (228 * 1024) / (q.sm_total + 1024 + 1024);
    const int by_regs = 65536 / (((regs + 7) / 8 * 8) * kTile);
    int per_sm = max(1, min(min(by_smem, by_regs), 512 / q.tmem_cols));
    if (const char* e = getenv("NVC_QUERY_CTAS_PER_SM")) per_sm = max(1, atoi(e));
    int dev = 0, sms = kNumSMs;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t ntiles = (P + kTile - 1) / kTile;
    const int64_t cap = (int64_t)sms * per_sm;
    int grid = (int)(ntiles < cap ? ntiles : cap);
    if (const char* e = getenv("NVC_QUERY_GRID")) grid = max(1, min(grid, atoi(e)));
    nvc_scene scv;
    if (sc) scv = *sc;
    else memset(&scv, 0, sizeof scv);
    kern<<<grid, kTile, q.sm_total, s>>>(g, q, m->params, reinterpret_cast<const __half*>(m->table_h), m->wpack, pos,
                                         P, scv, od);
    return check_launch("k_query_flat");
}

int launch_query(const nvc_model* m, const double* pos, int64_t P, const nvc_scene* sc, const QOut& o,
                 cudaStream_t s) {
    QOut od = o;
    if (const char* e = getenv("NVC_QUERY_DEBUG")) od.dbg = atoi(e);
    const char* kv = getenv("NVC_QUERY_KERNEL");
    if (!kv || strcmp(kv, "split") != 0) return launch_query_flat(m, pos, P, sc, od, s);
    QNet q;
    int rc = make_qnet(m, q, o.mode != kModeVis);
    if (rc) return rc;
    if (P <= 0) return NVC_OK;
    GridDev g = grid_of(m);
    const bool f2 = g.F == 2;
    auto kern = k_query<kModeVis, true>;
    if (o.mode == kModeVis) kern = f2 ? k_query<kModeVis, true> : k_query<kModeVis, false>;
    else if (o.mode == kModeNls) kern = f2 ? k_query<kModeNls, true> : k_query<kModeNls, false>;
    else kern = f2 ? k_query<kModeNdi, true> : k_query<kModeNdi, false>;
    const int threads = kQThreads;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, q.sm_total);
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncAttributes fa;
    int regs = 128;
    if (cudaFuncGetAttributes(&fa, kern) == cudaSuccess) regs = fa.numRegs;
    cudaGetLastError();
    const int by_smem = (228 * 1024) / (q.sm_total + 1024 + 1024);
    const int by_regs = 65536 / (((regs + 7) / 8 * 8) * threads);
    int per_sm = max(1, min(min(by_smem, by_regs), 512 / q.tmem_cols));
    if (const char* e = getenv("NVC_QUERY_CTAS_PER_SM")) per_sm = max(1, atoi(e));
    int dev = 0, sms = kNumSMs;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t ntiles = (P + kTile - 1) / kTile;
    const int64_t cap = (int64_t)sms * per_sm;
    int grid = (int)(ntiles < cap ? ntiles : cap);
    if (const char* e = getenv("NVC_QUERY_GRID")) grid = max(1, min(grid, atoi(e)));   // tests: many tiles per CTA
    nvc_scene scv;
    if (sc) scv = *sc;
    else memset(&scv, 0, sizeof scv);
    kern<<<grid, threads, q.sm_total, s>>>(g, q, m->params, reinterpret_cast<const __half*>(m->table_h), m->wpack,
                                             pos, P, scv, od);
    return check_launch("k_query");
}

}  // namespace

int64_t pipeline_workspace_bytes(const nvc_model* m, int64_t P);
int pipeline_query(const nvc_model* m, const nvc_scene* sc, const double* pos, int64_t P, int mode,
                   const void* lum, int lum_f64, int64_t stride, const uint32_t* nz_mask, int64_t p_first, int64_t p_total,
                   uint64_t key, uint64_t offset, double floor, int64_t* ids, double* pts, double* big_w,
                   const double* albedo, double* rgb, float* vis_out, void* ws, cudaStream_t s);

}  // namespace nvc

using namespace nvc;

extern "C" {

int64_t nvc_query_workspace_bytes(const nvc_model* m, int64_t p) {
    return (m && p > 0) ? pipeline_workspace_bytes(m, p) : 0;
}

int nvc_infer(const nvc_model* m, const double* pos, int64_t n, int32_t precision, float* out, void* workspace,
              void* stream) {
    if (n <= 0) return NVC_OK;
    NVC_REQUIRE(m && pos && out, "nvc_infer: null argument");
    if (precision == 0) return nvc_infer_f32(m, pos, n, out, (cudaStream_t)stream);
    if (workspace)
        return pipeline_query(m, nullptr, pos, n, 0, nullptr, 0, 0, nullptr, 0, n, 0, 0, 0.0, nullptr, nullptr, nullptr,
                              nullptr, nullptr, out, workspace, (cudaStream_t)stream);
    QOut o;
    memset(&o, 0, sizeof o);
    o.mode = kModeVis;
    o.vis = out;
    return launch_query(m, pos, n, nullptr, o, (cudaStream_t)stream);
}

int nvc_nls_sample(const nvc_model* m, const nvc_scene* sc, const double* pos, const void* lum, int32_t lum_f64,
                   const uint32_t* nz_mask, int64_t stride, int64_t p, int64_t p_first, int64_t p_total,
                   uint64_t key, uint64_t offset, double floor, int64_t* ids, double* pts, double* big_w,
                   void* workspace, void* stream) {
    NVC_REQUIRE(m && sc && pos && lum && ids && pts && big_w, "nvc_nls_sample: null argument");
    NVC_REQUIRE(sc->n_lights == m->dims[m->n_layers], "nvc_nls_sample: output_dim != scene lights");
    NVC_REQUIRE(stride >= p && p_total >= p_first + p, "nvc_nls_sample: bad stride / frame size");
    if (p <= 0) return NVC_OK;
    if (workspace)
        return pipeline_query(m, sc, pos, p, 1, lum, lum_f64, stride, nz_mask, p_first, p_total, key, offset, floor, ids, pts,
                              big_w, nullptr, nullptr, nullptr, workspace, (cudaStream_t)stream);
    QOut o;
    memset(&o, 0, sizeof o);
    o.mode = kModeNls;
    o.lum = lum;
    o.lum_f64 = lum_f64;
    o.stride = stride;
    o.p_first = p_first;
    o.p_total = p_total;
    o.key = key;
    o.offset = offset;
    o.floor = floor;
    o.ids = ids;
    o.pts = pts;
    o.big_w = big_w;
    o.nz_mask = nz_mask;
    return launch_query(m, pos, p, sc, o, (cudaStream_t)stream);
}

int nvc_neural_di(const nvc_model* m, const nvc_scene* sc, const double* pos, const double* albedo,
                  const void* factor, int32_t factor_f64, const uint32_t* nz_mask, int64_t stride, int64_t p,
                  double* rgb, void* workspace, void* stream) {
    NVC_REQUIRE(m && sc && pos && albedo && factor && rgb, "nvc_neural_di: null argument");
    NVC_REQUIRE(sc->n_lights == m->dims[m->n_layers], "nvc_neural_di: output_dim != scene lights");
    if (p <= 0) return NVC_OK;
    if (workspace)
        return pipeline_query(m, sc, pos, p, 2, factor, factor_f64, stride, nz_mask, 0, p, 0, 0, 0.0, nullptr, nullptr, nullptr,
                              albedo, rgb, nullptr, workspace, (cudaStream_t)stream);
    QOut o;
    memset(&o, 0, sizeof o);
    o.mode = kModeNdi;
    o.lum = factor;
    o.lum_f64 = factor_f64;
    o.stride = stride;
    o.albedo = albedo;
    o.rgb = rgb;
    o.nz_mask = nz_mask;
    return launch_query(m, pos, p, sc, o, (cudaStream_t)stream);
}

int nvc_l2_persist(const void* ptr, int64_t bytes, void* stream) {
    // keep the fp16 hash table L2-resident while lum / G-buffer rows stream past it
    int dev = 0;
    cudaGetDevice(&dev);
    int max_persist = 0, max_window = 0;
    cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev);
    cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev);
    if (max_persist <= 0 || max_window <= 0 || !ptr || bytes <= 0) return NVC_OK;
    const size_t want = (size_t)bytes < (size_t)max_persist ? (size_t)bytes : (size_t)max_persist;
    if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) != cudaSuccess) {
        cudaGetLastError();
        return NVC_OK;
    }
    cudaStreamAttrValue attr;
    memset(&attr, 0, sizeof attr);
    attr.accessPolicyWindow.base_ptr = const_cast<void*>(ptr);
    attr.accessPolicyWindow.num_bytes = (size_t)bytes < (size_t)max_window ? (size_t)bytes : (size_t)max_window;
    attr.accessPolicyWindow.hitRatio = (float)want / (float)attr.accessPolicyWindow.num_bytes;
    if (attr.accessPolicyWindow.hitRatio > 1.0f) attr.accessPolicyWindow.hitRatio = 1.0f;
    attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    if (cudaStreamSetAttribute((cudaStream_t)stream, cudaStreamAttributeAccessPolicyWindow, &attr) != cudaSuccess)
        cudaGetLastError();
    return NVC_OK;
}

int nvc_debug_trace(uint64_t* host_out, int32_t n, int32_t reset) {
    if (reset) {
        unsigned int z = 0;
        cudaMemcpyToSymbol(g_trace_n, &z, sizeof z);
        return 0;
    }
    unsigned int cnt = 0;
    cudaMemcpyFromSymbol(&cnt, g_trace_n, sizeof cnt);
    if (cnt > 8192) cnt = 8192;
    if ((int)cnt > n) cnt = n;
    cudaMemcpyFromSymbol(host_out, g_trace, cnt * sizeof(uint64_t));
    return (int)cnt;
}

int nvc_table_mask(const void* table, int32_t f64, int64_t stride, int64_t p, int32_t k, uint32_t* mask,
                   void* stream) {
    NVC_REQUIRE(table && mask && k >= 1 && stride >= p, "nvc_table_mask: bad argument");
    if (p <= 0) return NVC_OK;
    dim3 g(grid1(p, 256), (k + 31) / 32);
    if (f64)
        k_table_mask<double><<<g, 256, 0, (cudaStream_t)stream>>>((const double*)table, stride, p, k, mask);
    else
        k_table_mask<float><<<g, 256, 0, (cudaStream_t)stream>>>((const float*)table, stride, p, k, mask);
    return check_launch("k_table_mask");
}

int nvc_wrs_select(const double* w, int64_t p, int32_t k, uint64_t key, uint64_t offset, int64_t* idx,
                   double* w_sel, double* w_sum, void* stream) {
    NVC_REQUIRE(w && idx && w_sel && w_sum && k >= 1, "nvc_wrs_select: bad argument");
    if (p <= 0) return NVC_OK;
    k_wrs_select<<<grid1(p, 128), 128, 0, (cudaStream_t)stream>>>(w, p, k, key, offset, idx, w_sel, w_sum);
    return check_launch("k_wrs_select");
}

int nvc_nls_from_vis(const nvc_scene* sc, const float* vis, const void* lum, int32_t lum_f64, int64_t stride,
                     int64_t p, int32_t k, int64_t p_first, int64_t p_total, uint64_t key, uint64_t offset,
                     double floor, int64_t* ids, double* pts, double* big_w, void* stream) {
    NVC_REQUIRE(sc && vis && lum && ids && pts && big_w && k >= 1, "nvc_nls_from_vis: bad argument");
    NVC_REQUIRE(stride >= p && p_total >= p_first + p, "nvc_nls_from_vis: bad stride / frame size");
    if (p <= 0) return NVC_OK;
    cudaStream_t s = (cudaStream_t)stream;
    if (lum_f64)
        k_nls_from_vis<double><<<grid1(p, 128), 128, 0, s>>>(*sc, vis, (const double*)lum, stride, p, k, p_first,
                                                             p_total, key, offset, floor, ids, pts, big_w);
    else
        k_nls_from_vis<float><<<grid1(p, 128), 128, 0, s>>>(*sc, vis, (const float*)lum, stride, p, k, p_first,
                                                            p_total, key, offset, floor, ids, pts, big_w);
    return check_launch("k_nls_from_vis");
}

}  // extern "C"
