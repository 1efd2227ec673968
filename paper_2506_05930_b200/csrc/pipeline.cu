// pipeline.cu -- the decoupled query pipeline (default hot path):
//
//   k_enc_tiles   hash-grid encode, one thread per pixel, writes each 128-pixel
//                 tile's fp16 features as the exact shared-memory image the
//                 tensor core reads (swizzled K-major, common.cuh umma_off)
//   k_mlp_tiles   persistent tcgen05 MLP: one bulk copy per feature tile into a
//                 4-stage ring, four tiles in flight per CTA (TMEM holds four
//                 accumulators), two epilogue warpgroups ping-ponging their
//                 tiles; writes fp16 visibilities light-major
//   k_wrs_tiles   per-pixel FP64 reservoir over the nonzero lights with
//                 numpy-Philox uniforms (or the Neural-DI sum)
//
// Each stage runs at its own occupancy sweet spot (gather-bound encoder with
// 32+ warps/SM, tensor-pipe-fed MLP, ALU-bound selection), which the single
// fused kernel (query.cu) cannot: its per-tile chain of gathers, MMA round
// trips and dependent FP64 work left most issue slots idle.  The price is two
// HBM round trips of fp16 intermediates (features and visibilities,
// 2 x 64 B/pixel at K=32).
//
// Reference routines: encode_batch hashgrid.py:117-131, forward mlp.py:110-140,
// clamp_visibility sampling.py:27-30, wrs_select_batch :74-85,
// nls_sample_batch :194-205, neural_di_batch :215-218.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "common.cuh"
#include <cuda_bf16.h>

namespace nvc {
namespace {

constexpr int kT = 128;   // pixels per tile = UMMA M

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
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
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     s32(dst)),
                 "l"(src), "r"(bytes), "r"(s32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ uint64_t desc_of(uint32_t base, int rows, int kp, int kk) {
    const int lg = umma_sw_log2(kp);
    const uint32_t kb = (uint32_t)kk * 32u;
    const uint32_t addr = base + ((kb >> lg) * (uint32_t)rows << lg) + (kb & ((1u << lg) - 1u));
    const uint64_t layout = lg == 7 ? 2ull : (lg == 6 ? 4ull : 6ull);
    return (uint64_t)((addr & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)((8u << lg) >> 4) << 32) |
           ((uint64_t)1 << 46) | (layout << 61);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s32(bar))
                 : "memory");
}
__device__ __forceinline__ void tld16(uint32_t taddr, float v[16]) {
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
// stage 1: encoder -> feature tile images
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cell3(int n, const double q[3], uint32_t c0[3], float f[3]) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {   // floor via round-down add of 2^52 (bit-identical to min(int(x), n-1))
        const double x = __dmul_rn(q[a], (double)n);
        const double t = __dadd_rd(x, 0x1p52);
        uint32_t c = (uint32_t)__double2loint(t);
        double fr = __dsub_rn(x, __dsub_rn(t, 0x1p52));
        if (c > (uint32_t)(n - 1)) {
            c = (uint32_t)(n - 1);
            fr = 1.0;
        }
        c0[a] = c;
        f[a] = (float)fr;
    }
}

template <bool kF2>
__global__ void __launch_bounds__(kT, 6) k_enc_tiles(GridDev g, const uint16_t* __restrict__ table2,
                                                     const double* __restrict__ pos, int64_t P, int kp0,
                                                     uint8_t* __restrict__ tiles) {
    const int row = threadIdx.x;
    const int64_t tile = blockIdx.x;
    const int64_t p = tile * kT + row;
    uint8_t* img = tiles + tile * (int64_t)(kT * kp0 * 2);
    if (p >= P) {
        for (int k = 0; k < kp0; k += 8) *reinterpret_cast<uint4*>(img + umma_off(row, k, kT, kp0)) = make_uint4(0, 0, 0, 0);
        return;
    }
    const double pp[3] = {__ldg(pos + 3 * p), __ldg(pos + 3 * p + 1), __ldg(pos + 3 * p + 2)};
    double q[3];
    normalize(g, pp, q);
    if constexpr (kF2) {
        const uint2* t2 = reinterpret_cast<const uint2*>(table2);
        constexpr int LB = 4;
        for (int l = 0; l < g.L; l += LB) {
            uint2 v[LB][4];
            float w[LB][3];
#pragma unroll
            for (int j = 0; j < LB; ++j) {
                if (l + j < g.L) {
                    uint32_t c0[3];
                    cell3(g.res[l + j], q, c0, w[j]);
                    uint32_t sy, sz, mask;
                    if (g.dense[l + j]) {
                        sy = (uint32_t)g.res[l + j] + 1u;
                        sz = sy * sy;
                        mask = 0xffffffffu;
                    } else {
                        sy = 2654435761u;
                        sz = 805459861u;
                        mask = g.tmask;
                    }
                    const uint32_t base = c0[0] + c0[1] * sy + c0[2] * sz;
                    const uint2* tl = t2 + (size_t)(l + j) * (size_t)g.T;
#pragma unroll
                    for (int c = 0; c < 4; ++c) v[j][c] = __ldg(tl + ((base + ((c >> 1) & 1) * sy + (c & 1) * sz) & mask));
                }
            }
            __align__(16) __half2 out[LB];
#pragma unroll
            for (int j = 0; j < LB; ++j) {
                float a = 0.0f, b = 0.0f;
                if (l + j < g.L) {
                    const float fx = w[j][0], wy[2] = {1.0f - w[j][1], w[j][1]}, wz[2] = {1.0f - w[j][2], w[j][2]};
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const float wyz = wy[(c >> 1) & 1] * wz[c & 1];
                        const float w0 = (1.0f - fx) * wyz, w1 = fx * wyz;
                        const float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(&v[j][c].x));
                        const float2 f1 = __half22float2(*reinterpret_cast<const __half2*>(&v[j][c].y));
                        a = fmaf(w1, f1.x, fmaf(w0, f0.x, a));
                        b = fmaf(w1, f1.y, fmaf(w0, f0.y, b));
                    }
                }
                out[j] = __floats2half2_rn(a, b);
            }
            *reinterpret_cast<uint4*>(img + umma_off(row, 2 * l, kT, kp0)) = *reinterpret_cast<const uint4*>(out);
        }
        for (int k = 2 * ((g.L + 3) / 4 * 4); k < kp0; k += 8)
            *reinterpret_cast<uint4*>(img + umma_off(row, k, kT, kp0)) = make_uint4(0, 0, 0, 0);
    } else {
        const __half* t2 = reinterpret_cast<const __half*>(table2);
        for (int k = 0; k < kp0; ++k) *reinterpret_cast<__half*>(img + umma_off(row, k, kT, kp0)) = __float2half_rn(0.0f);
        for (int l = 0; l < g.L; ++l) {
            uint32_t c0[3];
            float f[3];
            cell3(g.res[l], q, c0, f);
            uint32_t sy, sz, mask;
            if (g.dense[l]) {
                sy = (uint32_t)g.res[l] + 1u;
                sz = sy * sy;
                mask = 0xffffffffu;
            } else {
                sy = 2654435761u;
                sz = 805459861u;
                mask = g.tmask;
            }
            const uint32_t base = c0[0] + c0[1] * sy + c0[2] * sz;
            const __half* tl = t2 + (size_t)l * (size_t)g.T * 2 * g.F;
            const float wy[2] = {1.0f - f[1], f[1]}, wz[2] = {1.0f - f[2], f[2]};
            float acc[8];
            for (int k = 0; k < g.F; ++k) acc[k] = 0.0f;
            for (int c = 0; c < 4; ++c) {
                const uint32_t slot = (base + ((c >> 1) & 1) * sy + (c & 1) * sz) & mask;
                const float wyz = wy[(c >> 1) & 1] * wz[c & 1];
                const __half* s2 = tl + (size_t)slot * 2 * g.F;
                for (int k = 0; k < g.F; ++k)
                    acc[k] = fmaf(f[0] * wyz, __half2float(__ldg(s2 + g.F + k)),
                                  fmaf((1.0f - f[0]) * wyz, __half2float(__ldg(s2 + k)), acc[k]));
            }
            for (int k = 0; k < g.F; ++k)
                *reinterpret_cast<__half*>(img + umma_off(row, l * g.F + k, kT, kp0)) = __float2half_rn(acc[k]);
        }
    }
}

// F == 4 (the reference's default grid, e.g. the clustered preset L=8,
// T=2^14): one x-pair slot is 8 halves = one 16-byte load per (level, y/z
// corner), levels unrolled, two levels per 16-byte tile store.  The blend is
// the generic path's arithmetic exactly (f32 weights, the same fmaf order per
// feature, one fp16 rounding at the store), so the tiles are bit-identical to
// k_enc_tiles<false> -- which issues 2-byte loads, 8 per (level, corner).
template <int L>
__global__ void __launch_bounds__(kT, 6) k_enc_tiles4(GridDev g, const uint16_t* __restrict__ table2,
                                                      const double* __restrict__ pos, int64_t P, int kp0,
                                                      uint8_t* __restrict__ tiles) {
    static_assert(L % 2 == 0, "two levels per 16-byte store");
    const int row = threadIdx.x;
    const int64_t tile = blockIdx.x;
    const int64_t p = tile * kT + row;
    uint8_t* img = tiles + tile * (int64_t)(kT * kp0 * 2);
    if (p >= P) {
        for (int k = 0; k < kp0; k += 8) *reinterpret_cast<uint4*>(img + umma_off(row, k, kT, kp0)) = make_uint4(0, 0, 0, 0);
        return;
    }
    const double pp[3] = {__ldg(pos + 3 * p), __ldg(pos + 3 * p + 1), __ldg(pos + 3 * p + 2)};
    double q[3];
    normalize(g, pp, q);
    const uint4* t4 = reinterpret_cast<const uint4*>(table2);
#pragma unroll
    for (int l0 = 0; l0 < L; l0 += 2) {
        uint4 v[2][4];
        float w[2][3];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int l = l0 + j;
            uint32_t c0[3];
            cell3(g.res[l], q, c0, w[j]);
            const bool dense = g.dense[l] != 0;
            const uint32_t sy = dense ? (uint32_t)g.res[l] + 1u : 2654435761u;
            const uint32_t sz = dense ? sy * sy : 805459861u;
            const uint32_t mask = dense ? 0xffffffffu : g.tmask;
            const uint32_t base = c0[0] + c0[1] * sy + c0[2] * sz;
            const uint4* tl = t4 + (size_t)l * (size_t)g.T;
#pragma unroll
            for (int c = 0; c < 4; ++c) v[j][c] = __ldg(tl + ((base + ((c >> 1) & 1) * sy + (c & 1) * sz) & mask));
        }
        __align__(16) __half out[8];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const float f0 = w[j][0], wy[2] = {1.0f - w[j][1], w[j][1]}, wz[2] = {1.0f - w[j][2], w[j][2]};
            float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const float wyz = wy[(c >> 1) & 1] * wz[c & 1];
                const __half* h = reinterpret_cast<const __half*>(&v[j][c]);   // x0 features 0-3 | x1 features 0-3
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    acc[k] = fmaf(f0 * wyz, __half2float(h[4 + k]), fmaf((1.0f - f0) * wyz, __half2float(h[k]), acc[k]));
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) out[4 * j + k] = __float2half_rn(acc[k]);
        }
        *reinterpret_cast<uint4*>(img + umma_off(row, 4 * l0, kT, kp0)) = *reinterpret_cast<const uint4*>(out);
    }
    for (int k = 4 * L; k < kp0; k += 8)
        *reinterpret_cast<uint4*>(img + umma_off(row, k, kT, kp0)) = make_uint4(0, 0, 0, 0);
}

// Mixed-precision FMA (sm_100: fma.rn.f32.f16 -> SASS FHFMA): f16 x f16 + f32.
// The half operands are selected from packed half2 registers (lo / hi).
__device__ __forceinline__ uint32_t h2bits(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
#define NVC_FHFMA(NAME, SA, SB)                                                                     \
    __device__ __forceinline__ float NAME(uint32_t a2, uint32_t b2, float c) {                       \
        asm("{\n\t.reg .f16 xa, xb, ya, yb;\n\tmov.b32 {xa, ya}, %1;\n\tmov.b32 {xb, yb}, %2;\n\t" \
            "fma.rn.f32.f16 %0, " SA ", " SB ", %0;\n\t}"                                          \
            : "+f"(c) : "r"(a2), "r"(b2));                                                          \
        return c;                                                                                   \
    }
NVC_FHFMA(fhfma_lo_lo, "xa", "xb")
NVC_FHFMA(fhfma_lo_hi, "xa", "yb")
NVC_FHFMA(fhfma_hi_lo, "ya", "xb")
NVC_FHFMA(fhfma_hi_hi, "ya", "yb")
#undef NVC_FHFMA

// Compile-time level count, F == 2: levels unrolled (per-level resolution /
// dense flag / table offset become constants), FP64 cell + hash exactly as the
// parity encoder, and the trilinear blend with fp16 operands (table entries,
// corner weights rounded once) and an fp32 accumulator -- the same contract as
// the tensor-core MLP that consumes the tile; fp16 only on the final store.
template <int L, int kMinBlocks = 8>
__global__ void __launch_bounds__(kT, kMinBlocks) k_enc_tiles2(GridDev g, const uint16_t* __restrict__ table2,
                                                      const double* __restrict__ pos, int64_t P, int kp0,
                                                      uint8_t* __restrict__ tiles) {
    // a dependent grid (the MLP, programmatic launch) may launch once every encoder CTA is
    // running; it waits for this grid's completion before touching the tiles
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int row = threadIdx.x;
    const int64_t tile = blockIdx.x;
    const int64_t p = tile * kT + row;
    uint8_t* img = tiles + tile * (int64_t)(kT * kp0 * 2);
    if (p >= P) {
        for (int k = 0; k < kp0; k += 8) *reinterpret_cast<uint4*>(img + umma_off(row, k, kT, kp0)) = make_uint4(0, 0, 0, 0);
        return;
    }
    const double pp[3] = {__ldg(pos + 3 * p), __ldg(pos + 3 * p + 1), __ldg(pos + 3 * p + 2)};
    double q[3];
    normalize(g, pp, q);
    const uint2* t2 = reinterpret_cast<const uint2*>(table2);
#pragma unroll
    for (int l0 = 0; l0 < L; l0 += 4) {
        uint2 v[4][4];
        float w[4][3];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int l = l0 + j;
            if (l < L) {
                uint32_t c0[3];
                cell3(g.res[l], q, c0, w[j]);
                const bool dense = g.dense[l] != 0;
                const uint32_t sy = dense ? (uint32_t)g.res[l] + 1u : 2654435761u;
                const uint32_t sz = dense ? sy * sy : 805459861u;
                const uint32_t mask = dense ? 0xffffffffu : g.tmask;
                const uint32_t base = c0[0] + c0[1] * sy + c0[2] * sz;
                // 32-bit byte offsets from the table base (the x-pair table is < 4 GB,
                // checked on the host): one shift-add per gather instead of a 64-bit
                // index multiply-add per gather
                const uint32_t lofs = (uint32_t)l * (uint32_t)g.T * 8u;
                const char* tb = reinterpret_cast<const char*>(t2);
                v[j][0] = __ldg(reinterpret_cast<const uint2*>(tb + (lofs + ((base & mask) << 3))));
                v[j][1] = __ldg(reinterpret_cast<const uint2*>(tb + (lofs + (((base + sz) & mask) << 3))));
                v[j][2] = __ldg(reinterpret_cast<const uint2*>(tb + (lofs + (((base + sy) & mask) << 3))));
                v[j][3] = __ldg(reinterpret_cast<const uint2*>(tb + (lofs + (((base + sy + sz) & mask) << 3))));
            }
        }
        __align__(16) __half2 out[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float a = 0.0f, b = 0.0f;
            if (l0 + j < L) {
                const float fx = w[j][0], wy[2] = {1.0f - w[j][1], w[j][1]}, wz[2] = {1.0f - w[j][2], w[j][2]};
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const float wyz = wy[(c >> 1) & 1] * wz[c & 1];
                    // corner weights rounded once to fp16 (the table's precision);
                    // f16 x f16 products are exact in f32 and accumulate in f32
                    // (FHFMA: one mixed-precision FMA per product, half selectors)
                    const uint32_t wc = h2bits(__floats2half2_rn((1.0f - fx) * wyz, fx * wyz));
                    a = fhfma_lo_lo(wc, v[j][c].x, a);
                    b = fhfma_lo_hi(wc, v[j][c].x, b);
                    a = fhfma_hi_lo(wc, v[j][c].y, a);
                    b = fhfma_hi_hi(wc, v[j][c].y, b);
                }
            }
            out[j] = __floats2half2_rn(a, b);
        }
        *reinterpret_cast<uint4*>(img + umma_off(row, 2 * l0, kT, kp0)) = *reinterpret_cast<const uint4*>(out);
    }
    for (int k = 2 * ((L + 3) / 4 * 4); k < kp0; k += 8)
        *reinterpret_cast<uint4*>(img + umma_off(row, k, kT, kp0)) = make_uint4(0, 0, 0, 0);
}

// ---------------------------------------------------------------------------
// stage 2: persistent tcgen05 MLP over feature tiles
// ---------------------------------------------------------------------------
struct MNet {
    int n_layers;
    int dims[NVC_MAX_LAYERS + 1];
    int np[NVC_MAX_LAYERS], kp[NVC_MAX_LAYERS];
    int wofs[NVC_MAX_LAYERS];     // halfs
    int64_t boff[NVC_MAX_LAYERS];
    int wpack_halfs, act_kp, tmem_cols, acc_cols, slots, ts_hid;
    float alpha;
    int out_sigmoid;
    int sm_w, sm_a0, sm_a1, sm_bias, sm_total;
};

constexpr int kStages = 4, kSlots = 4;
constexpr int kMlpThreads = 32 * 10;   // warps 0-7 epilogue (2 warpgroups), 8 producer, 9 MMA

struct MBars {
    uint64_t a0_full[kStages], a0_empty[kStages], acc_full[kSlots], acc_empty[kSlots], a1_full[kSlots];
};

__global__ void __launch_bounds__(kMlpThreads, 1) k_mlp_tiles(MNet net, const float* __restrict__ params,
                                                              const uint16_t* __restrict__ wpack,
                                                              const uint8_t* __restrict__ tiles, int64_t ntiles,
                                                              int64_t P, __half* __restrict__ vis16, int64_t vstride) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ MBars bars;
    __shared__ uint32_t tbase;
    uint8_t* smem = smem_raw + ((1024u - (s32(smem_raw) & 1023u)) & 1023u);
    uint8_t* s_w = smem + net.sm_w;
    uint8_t* s_a0 = smem + net.sm_a0;
    uint8_t* s_a1 = smem + net.sm_a1;
    float* s_bias = reinterpret_cast<float*>(smem + net.sm_bias);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int a0_bytes = kT * net.kp[0] * 2;
    const int a1_bytes = kT * net.act_kp * 2;
    {
        const uint4* src = reinterpret_cast<const uint4*>(wpack);
        uint4* dst = reinterpret_cast<uint4*>(s_w);
        for (int i = tid; i < net.wpack_halfs / 8; i += kMlpThreads) dst[i] = __ldg(src + i);
        int bo = 0;
        for (int l = 0; l < net.n_layers; ++l) {
            for (int n = tid; n < net.np[l]; n += kMlpThreads)
                s_bias[bo + n] = n < net.dims[l + 1] ? __ldg(params + net.boff[l] + n) : 0.0f;
            bo += net.np[l];
        }
    }
    if (warp == 9) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s32(&tbase)),
                     "r"(net.tmem_cols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&bars.a0_full[s], 1);
            mbar_init(&bars.a0_empty[s], 1);
        }
        for (int j = 0; j < kSlots; ++j) {
            mbar_init(&bars.acc_full[j], 1);
            mbar_init(&bars.acc_empty[j], 128);
            mbar_init(&bars.a1_full[j], 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    fence_async();
    tc_before();
    __syncthreads();
    tc_after();
    const uint32_t tmem = tbase;
    const int slots = net.slots;   // tiles in flight: kSlots, or fewer when wide layers fill smem
    const int n_local = ntiles > blockIdx.x ? (int)((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;

    if (warp == 8) {
        // ---------------- producer: one bulk copy per feature tile ----------------
        if (lane == 0) {
            for (int i = 0; i < n_local; ++i) {
                const int s = i % kStages;
                if (i >= kStages) mbar_wait(&bars.a0_empty[s], ((i / kStages) - 1) & 1);
                mbar_expect_tx(&bars.a0_full[s], (uint32_t)a0_bytes);
                const int64_t tile = blockIdx.x + (int64_t)i * gridDim.x;
                bulk_g2s(s_a0 + s * a0_bytes, tiles + tile * a0_bytes, (uint32_t)a0_bytes, &bars.a0_full[s]);
            }
        }
        __syncwarp();
    } else if (warp == 9) {
        // ---------------- MMA issuer: quads of 4 tiles, layers interleaved ----------------
        if (lane == 0) {
            const uint32_t w_addr = s32(s_w), a0_addr = s32(s_a0), a1_addr = s32(s_a1);
            uint32_t a1_cnt[kSlots] = {0, 0, 0, 0};
            auto issue = [&](int l, int j, uint32_t a_addr) {
                tc_after();
                const uint32_t idesc = (1u << 4) | ((uint32_t)(net.np[l] >> 3) << 17) | ((uint32_t)(kT >> 4) << 24);
                const uint32_t b = w_addr + 2u * (uint32_t)net.wofs[l];
                const uint32_t d = tmem + (uint32_t)(j * net.acc_cols);
                for (int kk = 0; kk < net.kp[l] / 16; ++kk)
                    mma(d, desc_of(a_addr, kT, net.kp[l], kk), desc_of(b, net.np[l], net.kp[l], kk), idesc,
                        kk > 0 ? 1u : 0u);
            };
            for (int q0 = 0; q0 < n_local; q0 += slots) {
                const int nq = min(slots, n_local - q0);
                for (int j = 0; j < nq; ++j) {
                    const int i = q0 + j, s = i % kStages;
                    mbar_wait(&bars.a0_full[s], (i / kStages) & 1);
                    if (q0 >= slots) mbar_wait(&bars.acc_empty[j], ((q0 / slots) - 1) & 1);
                    issue(0, j, a0_addr + (uint32_t)(s * a0_bytes));
                    commit(&bars.a0_empty[s]);
                    commit(&bars.acc_full[j]);
                }
                for (int l = 1; l < net.n_layers; ++l)
                    for (int j = 0; j < nq; ++j) {
                        mbar_wait(&bars.a1_full[j], a1_cnt[j] & 1);
                        ++a1_cnt[j];
                        issue(l, j, a1_addr + (uint32_t)(j * a1_bytes));
                        commit(&bars.acc_full[j]);
                    }
            }
        }
        __syncwarp();
    } else {
        // ---------------- epilogue: warpgroup eg serves slots eg and eg+2 ----------------
        const int eg = warp >> 2, row = tid & 127;
        const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
        uint32_t acc_cnt[2] = {0, 0};
        for (int q0 = 0; q0 < n_local; q0 += slots) {
            const int nq = min(slots, n_local - q0);
            int bias_off = 0;
            for (int l = 0; l < net.n_layers; ++l) {
                for (int jj = 0; jj < 2; ++jj) {
                    const int j = eg + 2 * jj;
                    if (j >= nq) continue;
                    const uint32_t t_acc = tmem + lane_base + (uint32_t)(j * net.acc_cols);
                    mbar_wait(&bars.acc_full[j], acc_cnt[jj] & 1);
                    ++acc_cnt[jj];
                    tc_after();
                    if (l < net.n_layers - 1) {
                        uint8_t* a1 = s_a1 + j * a1_bytes;
                        for (int c = 0; c < net.np[l] / 16; ++c) {
                            float v[16];
                            tld16(t_acc + (uint32_t)(c * 16), v);
                            __align__(16) __half2 h[8];
                            const float2* bb = reinterpret_cast<const float2*>(s_bias + bias_off + c * 16);
                            const __half2 al = __float2half2_rn(net.alpha);
#pragma unroll
                            for (int e = 0; e < 8; ++e) {
                                const float2 bj = bb[e];
                                const __half2 z = __floats2half2_rn(v[2 * e] + bj.x, v[2 * e + 1] + bj.y);
                                h[e] = __hmax2(z, __hmul2(z, al));
                            }
                            *reinterpret_cast<uint4*>(a1 + umma_off(row, c * 16, kT, net.np[l])) =
                                *reinterpret_cast<const uint4*>(h);
                            *reinterpret_cast<uint4*>(a1 + umma_off(row, c * 16 + 8, kT, net.np[l])) =
                                *reinterpret_cast<const uint4*>(h + 4);
                        }
                        fence_async();
                        tc_before();
                        mbar_arrive(&bars.a1_full[j]);
                    } else {
                        const int64_t tile = blockIdx.x + (int64_t)(q0 + j) * gridDim.x;
                        const int64_t p = tile * kT + row;
                        __half* vrow = vis16 + p * vstride;
                        for (int c = 0; c < net.np[l] / 16; ++c) {
                            float v[16];
                            tld16(t_acc + (uint32_t)(c * 16), v);
                            if (p >= P) continue;
                            __align__(16) __half2 h[8];
#pragma unroll
                            for (int e = 0; e < 8; ++e) {
                                float a2[2];
#pragma unroll
                                for (int t = 0; t < 2; ++t) {
                                    const float z = v[2 * e + t] + s_bias[bias_off + c * 16 + 2 * e + t];
                                    float a;
                                    if (net.out_sigmoid) {
                                        const float ez = __expf(-fabsf(z));
                                        const float r = __fdividef(1.0f, 1.0f + ez);
                                        a = z >= 0.0f ? r : ez * r;
                                        a = fminf(fmaxf(a, 1e-6f), 0.999999f);
                                    } else {
                                        a = z >= 0.0f ? z : net.alpha * z;
                                    }
                                    a2[t] = a;
                                }
                                h[e] = __floats2half2_rn(a2[0], a2[1]);
                            }
                            // padded columns (>= K, zero weights) land in the row's padding
                            if (c * 16 < vstride)
                                *reinterpret_cast<uint4*>(vrow + c * 16) = *reinterpret_cast<const uint4*>(h);
                            if (c * 16 + 8 < vstride)
                                *reinterpret_cast<uint4*>(vrow + c * 16 + 8) = *reinterpret_cast<const uint4*>(h + 4);
                        }
                        tc_before();
                        mbar_arrive(&bars.acc_empty[j]);
                    }
                }
                bias_off += net.np[l];
            }
        }
    }
    tc_before();
    __syncthreads();
    tc_after();
    if (warp == 9)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(net.tmem_cols) : "memory");
}

// ---------------------------------------------------------------------------
// tcgen05 helpers for the MLP kernels below
// ---------------------------------------------------------------------------
__device__ __forceinline__ void tld16_nowait(uint32_t taddr, uint32_t r[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// issued by a converged warp: operands stay in uniform registers, one elected lane issues
__device__ __forceinline__ void mma_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void commit_elect(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(s32(bar))
        : "memory");
}
__device__ __forceinline__ float tanh_fast(float x) {
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// ---------------------------------------------------------------------------
// stage 2 (default for widths <= 64): activations stay in tensor memory
//
// An SS-mode MLP (both operands in shared memory; k_mlp_tiles below for wide
// nets) re-reads every hidden activation tile from shared memory for each MMA
// and writes it there in each epilogue; with K = 64 layers that smem traffic
// (A 4 KB + B 2 KB per 128x64x16 MMA, plus the epilogue stores) saturates the
// shared-memory pipe.  Here each warpgroup keeps its
// tile's activations in TMEM: the epilogue drains the fp32 accumulator
// (tcgen05.ld), applies leaky-ReLU in packed half2 and writes the fp16 result
// back with tcgen05.st into a 32-column A region, and the next layer's MMA
// reads A from TMEM (kind::f16 "TS" form); only the weights come from smem.
// Biases are folded into the accumulation by one extra K=16 step per layer
// (A = a constant tile whose column 0 is 1.0, B = the layer's bias column), so
// the epilogue does pack + leaky only.  Four warpgroups (one tile in flight
// each: 64 accumulator + 32 activation columns) and one MMA warp per group.
// ---------------------------------------------------------------------------
// HID = 64: four warpgroups x (64 accumulator + 32 fp16-pair activation columns);
// HID = 128 (C4): two warpgroups x (128 + 64) -- TMEM holds 512 columns.
template <int HID>
struct TsCfg {
    static constexpr int WG = HID == 64 ? 4 : 2;
    static constexpr int kThreads = 160 * WG;
    static constexpr int kCols = HID + HID / 2;
};

struct TSBars {
    uint64_t a0_full[2], acc_full;
};

__device__ __forceinline__ void mma_ts_elect(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void tst16(uint32_t taddr, const uint32_t r[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}
__device__ __forceinline__ void tst_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

#ifdef NVC_MLP_TRACE
// profiling build only (tools/mlp_trace.py): clock64 stamps of CTA 0's first 8 tiles per
// warpgroup, [wg][tile][layer][event]: 0 MMA issue start, 1 commit issued, 2 epilogue
// wake-up, 3 epilogue done (accumulator released), 4 A0 tile ready, 5 output stores issued
__device__ long long g_mlp_trace[4][8][4][6];
#define MLP_STAMP(g, k, l, e) \
    { if (blockIdx.x == 0 && (k) < 8 && (l) < 4) g_mlp_trace[g][k][l][e] = clock64(); }
#else
#define MLP_STAMP(g, k, l, e) {}
#endif

template <int HID, int OUT, int KP0>
__global__ void __launch_bounds__(TsCfg<HID>::kThreads, 1) k_mlp_ts(MNet net, const float* __restrict__ params,
                                                                   const uint16_t* __restrict__ wpack,
                                                                   const uint8_t* __restrict__ tiles, int64_t ntiles,
                                                                   int64_t P, __half* __restrict__ vis16,
                                                                   int64_t vstride) {
    static_assert((HID == 64 || HID == 128) && OUT <= HID && KP0 <= 64, "TMEM layout: 64/128-wide hidden layers");
    constexpr int kTsWG = TsCfg<HID>::WG, kTsThreads = TsCfg<HID>::kThreads, kTsCols = TsCfg<HID>::kCols;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ TSBars bars[kTsWG];
    __shared__ uint32_t tbase;
    uint8_t* smem = smem_raw + ((1024u - (s32(smem_raw) & 1023u)) & 1023u);
    uint8_t* s_w = smem + net.sm_w;
    uint8_t* s_a0 = smem + net.sm_a0;
    uint8_t* s_ones = smem + net.sm_a1;                   // [128 x 16] K-major SW32, column 0 = 1
    uint8_t* s_bias = smem + net.sm_bias;                 // per layer [np x 16] K-major SW32, column 0 = bias
    const int tid = threadIdx.x, row = tid & 127;
    const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
    const bool mma_warp = warp >= 4 * kTsWG;
    const int g = mma_warp ? warp - 4 * kTsWG : warp >> 2, wq = warp & 3;
    const int L = net.n_layers;
    constexpr int a0_bytes = kT * KP0 * 2;
    const int bias_block = HID * 32;                      // bytes per layer block (np <= HID rows x 32 B)
    {
        const uint4* src = reinterpret_cast<const uint4*>(wpack);
        uint4* dst = reinterpret_cast<uint4*>(s_w);
        for (int i = tid; i < net.wpack_halfs / 8; i += kTsThreads) dst[i] = __ldg(src + i);
        for (int i = tid; i < kT * 16; i += kTsThreads) {   // ones tile
            const int r = i >> 4, k = i & 15;
            *reinterpret_cast<__half*>(s_ones + umma_off(r, k, kT, 16)) = __float2half_rn(k == 0 ? 1.0f : 0.0f);
        }
        for (int l = 0; l < L; ++l) {
            const int np = l == L - 1 ? OUT : HID;
            for (int i = tid; i < np * 16; i += kTsThreads) {
                const int n = i >> 4, k = i & 15;
                const float b = (k == 0 && n < net.dims[l + 1]) ? __ldg(params + net.boff[l] + n) : 0.0f;
                *reinterpret_cast<__half*>(s_bias + l * bias_block + umma_off(n, k, np, 16)) = __float2half_rn(b);
            }
        }
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s32(&tbase)), "r"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        for (int w = 0; w < kTsWG; ++w) {
            mbar_init(&bars[w].a0_full[0], 1);
            mbar_init(&bars[w].a0_full[1], 1);
            mbar_init(&bars[w].acc_full, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    fence_async();
    tc_before();
    __syncthreads();
    tc_after();
    // programmatic dependent launch (default; NVC_NO_PDL=1 off): the encoder grid's tiles are complete
    // and visible past this point (a no-op for a normal launch)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const uint32_t tmem = tbase;
    TSBars& B = bars[g];
    const int64_t t0 = (int64_t)blockIdx.x * kTsWG + g, tstep = (int64_t)gridDim.x * kTsWG;
    const int n_wg = ntiles > t0 ? (int)((ntiles - 1 - t0) / tstep + 1) : 0;
    const uint32_t acc = tmem + (uint32_t)(g * kTsCols);      // columns [0, HID): fp32 accumulator
    const uint32_t act = acc + (uint32_t)HID;                  // HID/2 columns: fp16-pair activations
    const int id = 1 + g;
    if (mma_warp) {
        // ---------------- MMA warp of warpgroup g ----------------
        const uint32_t w_addr = s32(s_w), ones = s32(s_ones), bias = s32(s_bias);
        const uint64_t d_ones = desc_of(ones, kT, 16, 0);
        auto load_a0 = [&](int k) {
            if ((tid & 31) == 0) {
                const int b = k & 1;
                mbar_expect_tx(&B.a0_full[b], (uint32_t)a0_bytes);
                bulk_g2s(s_a0 + (2 * g + b) * a0_bytes, tiles + (t0 + (int64_t)k * tstep) * a0_bytes,
                         (uint32_t)a0_bytes, &B.a0_full[b]);
            }
            __syncwarp();
        };
        uint32_t a0_ph[2] = {0, 0};
        if (n_wg > 0) load_a0(0);
        for (int k = 0; k < n_wg; ++k) {
            if (k + 1 < n_wg) load_a0(k + 1);                     // the other buffer: tile k-1 is done with it
            const int b = k & 1;
            mbar_wait(&B.a0_full[b], a0_ph[b]);
            if ((tid & 31) == 0) MLP_STAMP(g, k, 0, 4)
            a0_ph[b] ^= 1u;
            for (int l = 0; l < L; ++l) {
                if (k > 0 || l > 0) asm volatile("bar.sync %0, 160;" ::"r"(id) : "memory");   // epilogue done
                tc_after();
                if ((tid & 31) == 0) MLP_STAMP(g, k, l, 0)
                const int np = l == L - 1 ? OUT : HID;
                const uint32_t idesc = (1u << 4) | ((uint32_t)(np >> 3) << 17) | ((uint32_t)(kT >> 4) << 24);
                const uint64_t db = desc_of(w_addr + 2u * (uint32_t)net.wofs[l], np, l == 0 ? KP0 : HID, 0);
                if (l == 0) {
                    const uint64_t da = desc_of(s32(s_a0 + (2 * g + b) * a0_bytes), kT, KP0, 0);
#pragma unroll
                    for (int kk = 0; kk < KP0 / 16; ++kk) mma_elect(acc, da + 2 * kk, db + 2 * kk, idesc, kk > 0);
                } else if (HID <= 64) {
#pragma unroll
                    for (int kk = 0; kk < HID / 16; ++kk) mma_ts_elect(acc, act + 8u * kk, db + 2 * kk, idesc, kk > 0);
                } else {   // K = 128 spans two swizzle blocks of the weight tile
                    const uint32_t wl = w_addr + 2u * (uint32_t)net.wofs[l];
#pragma unroll
                    for (int kk = 0; kk < HID / 16; ++kk)
                        mma_ts_elect(acc, act + 8u * kk, desc_of(wl, np, HID, kk), idesc, kk > 0);
                }
                // bias: + ones[128 x 16] x bias_l[np x 16]^T
                mma_elect(acc, d_ones, desc_of(bias + l * bias_block, np, 16, 0), idesc, 1u);
                commit_elect(&B.acc_full);
                if ((tid & 31) == 0) MLP_STAMP(g, k, l, 1)
            }
        }
        if (n_wg > 0) asm volatile("bar.sync %0, 160;" ::"r"(id) : "memory");   // the last tile's final arrive
    } else {
        // ---------------- epilogue warpgroup g ----------------
        const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
        const __half2 al2 = __float2half2_rn(net.alpha);
        const __half2 lo = __float2half2_rn(1e-6f), hi = __float2half2_rn(0.999999f);
        uint32_t ph = 0;
        for (int k = 0; k < n_wg; ++k) {
            for (int l = 0; l < L; ++l) {
                mbar_wait(&B.acc_full, ph);
                ph ^= 1u;
                tc_after();
                if (wq == 0 && (tid & 31) == 0) MLP_STAMP(g, k, l, 2)
                if (l < L - 1) {
#pragma unroll
                    for (int cb = 0; cb < HID; cb += 64) {   // 64 accumulator columns at a time
                        uint32_t r[64];
#pragma unroll
                        for (int c = 0; c < 64; c += 16) tld16_nowait(acc + lane_base + (uint32_t)(cb + c), r + c);
                        tld_wait();
                        uint32_t h[32];
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const __half2 z =
                                __floats2half2_rn(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1]));
                            const __half2 y = __hmax2(z, __hmul2(z, al2));
                            h[j] = *reinterpret_cast<const uint32_t*>(&y);
                        }
#pragma unroll
                        for (int c = 0; c < 32; c += 16) tst16(act + lane_base + (uint32_t)(cb / 2 + c), h + c);
                    }
                    tst_wait();
                    tc_before();
                    if (wq == 0 && (tid & 31) == 0) MLP_STAMP(g, k, l, 3)
                    asm volatile("bar.arrive %0, 160;" ::"r"(id) : "memory");
                } else {
                    uint32_t r[OUT];
#pragma unroll
                    for (int c = 0; c < OUT; c += 16) tld16_nowait(acc + lane_base + (uint32_t)c, r + c);
                    tld_wait();
                    tc_before();
                    if (wq == 0 && (tid & 31) == 0) MLP_STAMP(g, k, l, 3)
                    asm volatile("bar.arrive %0, 160;" ::"r"(id) : "memory");   // accumulator drained
                    const int64_t p = (t0 + (int64_t)k * tstep) * kT + row;
                    if (p < P) {
                        __half* vrow = vis16 + p * vstride;
#pragma unroll
                        for (int c = 0; c < OUT / 8; ++c) {
                            __align__(16) __half2 hh[4];
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                float o[2];
#pragma unroll
                                for (int t = 0; t < 2; ++t) {
                                    const float z = __uint_as_float(r[8 * c + 2 * e + t]);
                                    o[t] = net.out_sigmoid ? fmaf(0.5f, tanh_fast(0.5f * z), 0.5f)
                                                           : (z >= 0.0f ? z : net.alpha * z);
                                }
                                hh[e] = __floats2half2_rn(o[0], o[1]);
                                if (net.out_sigmoid) hh[e] = __hmin2(__hmax2(hh[e], lo), hi);   // mlp.py:135-136
                            }
#ifndef NVC_MLP_NOSTORE
                            if (8 * c < vstride) *reinterpret_cast<uint4*>(vrow + 8 * c) = *reinterpret_cast<const uint4*>(hh);
#else   // experiment: the outputs computed but not stored
                            if (P < 0) *reinterpret_cast<uint4*>(vrow + 8 * c) = *reinterpret_cast<const uint4*>(hh);
#endif
                        }
                    }
                    if (wq == 0 && (tid & 31) == 0) MLP_STAMP(g, k, l, 5)
                }
            }
        }
    }
    tc_before();
    __syncthreads();
    tc_after();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
}

// ---------------------------------------------------------------------------
// stage 3: WRS / Neural DI from fp16 visibilities
// ---------------------------------------------------------------------------
__device__ __noinline__ U4 philox_fn(uint64_t counter, uint64_t key) { return philox_block(counter, key); }

struct WArgs {
    const __half* vis16;
    int64_t vstride;
    const void* lum;       // light-major f32/f64 (lum for NLS, factor for NDI)
    int lum_f64;
    int64_t stride;
    const uint32_t* nz_mask;
    int64_t P, p_first, p_total;
    int K;
    uint64_t key, offset;
    double floor;
    int64_t* ids;
    double* pts;
    double* big_w;
    const double* albedo;
    double* rgb;
    // k_nls32g only (set by pipeline_select; 32-bit index math, checked on the host):
    uint64_t grp0;       // offset / 4 + 1: Philox block of the frame's first 4-light group
    uint64_t lp0;        // offset + p_total * K: draw index of the first light-point pair
    uint32_t stride32;   // luminance row stride (elements)
};

template <bool kLum64>
__device__ __forceinline__ double lum_at(const WArgs& a, int k, int64_t p) {
    const int64_t li = (int64_t)k * a.stride + p;
    if constexpr (kLum64) return __ldg(reinterpret_cast<const double*>(a.lum) + li);
    else return (double)__ldg(reinterpret_cast<const float*>(a.lum) + li);
}

// w_k = max(vis_k, floor) * lum_k in binary64 (sampling.py:27-30 clamp_visibility, nls_weights_batch);
// lo = clamp_lo(floor) is the clamp's lower bound (the floor, or 0 in biased mode)
__device__ __forceinline__ double clamp_lo(double floor) { return floor > 0.0 ? floor : 0.0; }
__device__ __forceinline__ double wrs_weight(float vis, double t, double lo) {
    const double vv = (double)vis;
    return __dmul_rn(vv < lo ? lo : vv, t);
}

// K <= 32 (the C2 / paper configuration).  Sequential FP64 reservoir exactly
// as wrs_select_batch (sampling.py:74-85): s += w_k; accept k when
// u_k * s < w_k; the last accept wins.  Each lane walks only its own nonzero
// lights (nz_mask), so a warp runs max-popcount iterations rather than the
// union of the lanes' lights; zero weights never need a uniform (u*s < 0 is
// impossible), so their Philox blocks are skipped.  The pixel's fp16
// visibility row (64 B, written by k_mlp_tiles) is staged in shared memory
// with a 33-word row stride, so per-lane light indices hit distinct banks.
constexpr int kWrsThreads = 256;
template <bool kLum64>
__global__ void __launch_bounds__(kWrsThreads) k_nls32(WArgs a, nvc_scene sc) {
    __shared__ uint32_t s_vis[kWrsThreads * 33];
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t* my = s_vis + threadIdx.x * 33;
    if (p < a.P) {
        const uint4* vrow = reinterpret_cast<const uint4*>(a.vis16 + p * a.vstride);
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (8 * i < a.K) {
                const uint4 v = __ldg(vrow + i);
                my[4 * i] = v.x;
                my[4 * i + 1] = v.y;
                my[4 * i + 2] = v.z;
                my[4 * i + 3] = v.w;
            }
    }
    if (p >= a.P) return;
    const int64_t gp = a.p_first + p;
    uint32_t m = a.nz_mask ? __ldg(a.nz_mask + p) : 0xffffffffu;
    if (a.K < 32) m &= (1u << a.K) - 1u;
    double s = 0.0, wsel = 0.0;
    int sel = -1;
    uint64_t blk = 0;
    U4 u;
    const uint64_t n0 = a.offset + (uint64_t)gp * (uint64_t)a.K;
    while (m) {
        const int k = __ffs(m) - 1;
        m &= m - 1;
        const uint32_t pair = my[k >> 1];
        const float vis = __half2float(__ushort_as_half((unsigned short)((k & 1) ? (pair >> 16) : (pair & 0xffffu))));
        const double w = wrs_weight(vis, lum_at<kLum64>(a, k, p), clamp_lo(a.floor));
        s = __dadd_rn(s, w);
        if (w > 0.0) {
            const uint64_t n = n0 + (uint64_t)k;
            const uint64_t bi = n / 4 + 1;
            if (bi != blk) {
                u = philox_fn(bi, a.key);
                blk = bi;
            }
            if (__dmul_rn(u01(u.x[n & 3]), s) < w) {
                sel = k;
                wsel = w;
            }
        }
    }
    const uint64_t n = a.offset + (uint64_t)a.p_total * (uint64_t)a.K + 2ull * (uint64_t)gp;
    const U4 b0 = philox_fn(n / 4 + 1, a.key);
    const double u0 = u01(b0.x[n & 3]);
    double u1;
    if ((n & 3) != 3) {
        u1 = u01(b0.x[(n & 3) + 1]);
    } else {
        const U4 b1 = philox_fn(n / 4 + 2, a.key);
        u1 = u01(b1.x[0]);
    }
    double y[3];
    light_point(sc, sel, u0, u1, y);
    a.ids[p] = sel;
    a.big_w[p] = sel >= 0 ? __ddiv_rn(s, wsel > 0.0 ? wsel : 1.0) : 0.0;
    a.pts[3 * p] = y[0];
    a.pts[3 * p + 1] = y[1];
    a.pts[3 * p + 2] = y[2];
}

// K <= 32, K % 4 == 0 and block-aligned draw counters (offset % 4 == 0,
// light-point counter even): the reservoir walks 4-light groups, so each
// group's Philox block is generated once at a single (inlined) call site with
// static word indices, and the group's luminances are loaded before the
// Philox rounds so their latency hides behind them.  The light-point draw
// pair is the last "group".  Same arithmetic and order as k_nls32.
template <bool kLum64, int KW, bool kStage>
__device__ __forceinline__ void nls_pixel(const WArgs& a, const nvc_scene& sc, int64_t p, uint32_t* my);

// one thread per pixel (the tile loop also serves grids smaller than the pixel count)
// 128-thread CTAs: finer-grained SM sharing with the training kernels beside
// the NLS (frame 0.584 vs 0.589 ms at 256; 64: 0.586, 192: 0.591, 512: 0.601)
#ifndef NVC_NLS_THREADS
#define NVC_NLS_THREADS 128
#endif
constexpr int kNlsThreads = NVC_NLS_THREADS;
template <bool kLum64, int KW, bool kStage>
__global__ void __launch_bounds__(kNlsThreads) k_nls32g(WArgs a, nvc_scene sc) {
    // KW 32-light words (K <= 32 KW).  The pixel's fp16 visibility row is read per
    // 4-light group (8 B) next to the group's luminances; kStage (K <= 32, A/B
    // only) stages the row in shared memory with one coalesced pass instead.
    constexpr int kRow = 16 * KW + 1;
    __shared__ uint32_t s_vis[kStage ? kNlsThreads * kRow : 1];
    uint32_t* my = s_vis + (kStage ? threadIdx.x * kRow : 0);
    const int64_t ntiles = (a.P + kNlsThreads - 1) / kNlsThreads;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x)
        nls_pixel<kLum64, KW, kStage>(a, sc, t * kNlsThreads + threadIdx.x, my);
}

template <bool kLum64, int KW, bool kStage>
__device__ __forceinline__ void nls_pixel(const WArgs& a, const nvc_scene& sc, int64_t p, uint32_t* my) {
    using JobT = typename std::conditional<(KW > 2), uint64_t, uint32_t>::type;
    if (kStage && p < a.P) {
        const uint4* vrow = reinterpret_cast<const uint4*>(a.vis16 + p * a.vstride);
#pragma unroll
        for (int i = 0; i < 4 * KW; ++i)
            if (8 * i < a.K) {
                const uint4 v = __ldg(vrow + i);
                my[4 * i] = v.x;
                my[4 * i + 1] = v.y;
                my[4 * i + 2] = v.z;
                my[4 * i + 3] = v.w;
            }
    }
    if (p >= a.P) return;
    const uint32_t gp = (uint32_t)(a.p_first + p);   // < 2^31 (host check)
    uint32_t m[KW];
#pragma unroll
    for (int w = 0; w < KW; ++w) {
        m[w] = a.nz_mask ? __ldg(a.nz_mask + (uint32_t)w * a.stride32 + p) : 0xffffffffu;
        const int left = a.K - 32 * w;
        if (left <= 0)
            m[w] = 0u;
        else if (left < 32)
            m[w] &= (1u << left) - 1u;
    }
    JobT jobs = (JobT)1 << (8 * KW);   // the last bit: the light-point pair
#pragma unroll
    for (int w = 0; w < KW; ++w)
#pragma unroll
        for (int g = 0; g < 8; ++g) jobs |= (JobT)(((m[w] >> (4 * g)) & 15u) != 0u ? 1u : 0u) << (8 * w + g);
    using LT = typename std::conditional<kLum64, double, float>::type;
    const LT* lp = reinterpret_cast<const LT*>(a.lum) + p;
    // keep the pixel's row base in a register: each luminance address is then one
    // 32 x 32 + 64-bit multiply-add (the compiler otherwise re-derives lum + (p + o) * 8
    // from the parameter bank for every load)
    asm volatile("" : "+l"(lp));
    const uint32_t st1 = a.stride32;   // light-major rows; K * stride < 2^32 elements (host check)
    const double lo = clamp_lo(a.floor);
    const uint64_t c_grp = a.grp0 + (uint64_t)(gp * (uint32_t)(a.K / 4));   // (offset + gp K) / 4 + 1
    const uint64_t n_lp = a.lp0 + 2ull * gp;                                // offset + p_total K + 2 gp
    double s = 0.0, wsel = 0.0, u0 = 0.0, u1 = 0.0;
    int sel = -1;
    // one 4-light group: its luminances (nonzero lights only) and visibility pair
    auto group_in = [&](int g, LT t[4], uint2& vg, uint32_t& bits) {
        uint32_t mw = 0u;
#pragma unroll
        for (int w = 0; w < KW; ++w)
            if ((g >> 3) == w) mw = m[w];
        bits = (mw >> (4 * (g & 7))) & 15u;
        const uint32_t o = (uint32_t)(4 * g) * st1;
        // only the nonzero lights' entries are read (group_wrs reads t[j] only for them)
        if (bits & 1u) t[0] = __ldg(lp + o);
        if (bits & 2u) t[1] = __ldg(lp + (o + st1));
        if (bits & 4u) t[2] = __ldg(lp + (o + 2 * st1));
        if (bits & 8u) t[3] = __ldg(lp + (o + 3 * st1));
        vg = make_uint2(0u, 0u);
        if (!kStage) vg = __ldg(reinterpret_cast<const uint2*>(a.vis16 + p * a.vstride) + g);
    };
    // the group's lights in order into the FP64 reservoir
    auto group_wrs = [&](int g, const LT t[4], uint2 vg, uint32_t bits, const U4& u) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if ((bits >> j) & 1u) {
                const int k = 4 * g + j;
                const uint32_t pair = kStage ? my[k >> 1] : (j < 2 ? vg.x : vg.y);
                const float vis = __half2float(__ushort_as_half((unsigned short)((j & 1) ? (pair >> 16) : (pair & 0xffffu))));
                const double w = wrs_weight(vis, (double)t[j], lo);
                s = __dadd_rn(s, w);
                if (w > 0.0 && __dmul_rn(u01(u.x[j]), s) < w) {
                    sel = k;
                    wsel = w;
                }
            }
        }
    };
    auto light_pair = [&](const U4& u) {
        const bool hi = (n_lp & 2) != 0;
        u0 = u01(hi ? u.x[2] : u.x[0]);
        u1 = u01(hi ? u.x[3] : u.x[1]);
    };
    const int lp_job = 8 * KW;
    {
        while (jobs) {
            const int g = (KW > 2) ? __ffsll((long long)jobs) - 1 : __ffs((uint32_t)jobs) - 1;
            jobs &= jobs - 1;
            const bool lpj = g == lp_job;
            LT t[4];
            uint2 vg;
            uint32_t bits = 0u;
            if (!lpj) group_in(g, t, vg, bits);
            const U4 u = philox_block(lpj ? n_lp / 4 + 1 : c_grp + (uint64_t)g, a.key);
            if (lpj) {
                light_pair(u);
                break;
            }
            group_wrs(g, t, vg, bits, u);
        }
    }
    double y[3];
    light_point(sc, sel, u0, u1, y);
    a.ids[p] = sel;
    a.big_w[p] = sel >= 0 ? __ddiv_rn(s, wsel > 0.0 ? wsel : 1.0) : 0.0;
    a.pts[3 * p] = y[0];
    a.pts[3 * p + 1] = y[1];
    a.pts[3 * p + 2] = y[2];
}

template <int KW>
void launch_nlsg(const WArgs& a, const nvc_scene& sc, int64_t P, cudaStream_t s) {
    const int thr = kNlsThreads;
    const int grid = (int)((P + thr - 1) / thr);   // one tile per CTA (a persistent grid measured slower in the frame)
    // The visibility row is read per 4-light group (8 B, L1-resident after the
    // first touch) rather than staged in shared memory: the 34 KB staging buffer
    // of each 256-thread block kept the training step's CTAs (102 KB of shared
    // memory) off the SMs the NLS occupies (frame 0.606 -> 0.589 ms).
    // NVC_NLS_STAGE=1 restores the staged K <= 32 variant (A/B).
    if constexpr (KW == 1) {
        if (getenv("NVC_NLS_STAGE")) {
            if (a.lum_f64)
                k_nls32g<true, KW, true><<<grid, thr, 0, s>>>(a, sc);
            else
                k_nls32g<false, KW, true><<<grid, thr, 0, s>>>(a, sc);
            return;
        }
    }
    if (a.lum_f64) {
        k_nls32g<true, KW, false><<<grid, thr, 0, s>>>(a, sc);
    } else {
        k_nls32g<false, KW, false><<<grid, thr, 0, s>>>(a, sc);
    }
}

// Neural DI for K <= 32 (sampling.py:215-218): rgb = (sum_k v_k * factor_k *
// L_e[k]) * albedo / pi over the pixel's nonzero-factor lights, FP64 in
// ascending light order.  The light-major factor table is read one coalesced
// 128-byte row per light any of the warp's pixels needs (each lane loads its
// own pixel's factor only where it is nonzero), a few lights per batch held in
// registers; the pixel's fp16 visibility row sits in shared memory (odd row
// stride).  Staging the factor tile in shared memory instead (round 1) cost
// 367 vs 329 us at C3 (fewer resident warps); batches of 16 lights: slower;
// 2 lights, or 64 / 256 threads per block: within noise.
// f32 tables only; the f64 parity tables use k_wrs_tiles.
constexpr int kNdiThreads = 128;
#ifndef NVC_NDI_BATCH
#define NVC_NDI_BATCH 4
#endif
__global__ void __launch_bounds__(kNdiThreads) k_ndi32(WArgs a, nvc_scene sc) {
    __shared__ uint32_t s_vis[kNdiThreads * 17];
    __shared__ double s_le[32 * 3];                    // emitter radiance, staged once per block
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = p < a.P;
    uint32_t* my = s_vis + threadIdx.x * 17;
    for (int i = threadIdx.x; i < 3 * a.K; i += kNdiThreads) s_le[i] = __ldg(sc.lt_radiance + i);
    uint32_t m = 0;
    double al[3] = {0.0, 0.0, 0.0};
    if (live) {
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) al[ch] = __ldg(a.albedo + 3 * p + ch);   // issued early, used last
        const uint4* vrow = reinterpret_cast<const uint4*>(a.vis16 + p * a.vstride);
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (8 * i < a.K) {
                const uint4 v = __ldg(vrow + i);
                my[4 * i] = v.x;
                my[4 * i + 1] = v.y;
                my[4 * i + 2] = v.z;
                my[4 * i + 3] = v.w;
            }
        m = a.nz_mask ? __ldg(a.nz_mask + p) : 0xffffffffu;
        if (a.K < 32) m &= (1u << a.K) - 1u;
    }
    __syncthreads();   // s_le
    // the warp walks the union of its pixels' nonzero lights in ascending order,
    // NVC_NDI_BATCH (4) at a time: each lane loads its own factor of light k (one coalesced row
    // per light for the warp) only if k is one of its lights, then accumulates
    // those in order -- the pixel's own ascending sum, factors kept in registers
    uint32_t wm = __reduce_or_sync(0xffffffffu, m);
    const float* fp = reinterpret_cast<const float*>(a.lum) + p;
    double rgb[3] = {0.0, 0.0, 0.0};
    while (wm) {
        int ks[NVC_NDI_BATCH];
        float t[NVC_NDI_BATCH];
#pragma unroll
        for (int j = 0; j < NVC_NDI_BATCH; ++j) {
            ks[j] = wm ? __ffs(wm) - 1 : 32;
            wm &= wm - 1;
        }
#pragma unroll
        for (int j = 0; j < NVC_NDI_BATCH; ++j) t[j] = (ks[j] < 32 && ((m >> ks[j]) & 1u)) ? __ldg(fp + (int64_t)ks[j] * a.stride) : 0.0f;
#pragma unroll
        for (int j = 0; j < NVC_NDI_BATCH; ++j) {
            const int k = ks[j];
            if (k < 32 && ((m >> k) & 1u)) {
                const uint32_t pair = my[k >> 1];
                const double vis = (double)__half2float(__ushort_as_half((unsigned short)((k & 1) ? (pair >> 16) : (pair & 0xffffu))));
                const double wk = __dmul_rn(vis, (double)t[j]);
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) rgb[ch] = __dadd_rn(rgb[ch], __dmul_rn(wk, s_le[3 * k + ch]));
            }
        }
    }
    if (!live) return;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) a.rgb[3 * p + ch] = __ddiv_rn(__dmul_rn(rgb[ch], al[ch]), 3.141592653589793);
}

// generic K: forward reservoir over the nonzero lights (pixel-major visibilities)
template <bool kNls>
__global__ void __launch_bounds__(256) k_wrs_tiles(WArgs a, nvc_scene sc) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= a.P) return;
    const int64_t gp = a.p_first + p;
    uint32_t m = 0xffffffffu;
    if (a.nz_mask && a.K <= 32) m = __ldg(a.nz_mask + p);
    if (a.K < 32) m &= (1u << a.K) - 1u;
    double s = 0.0, wsel = 0.0, rgb[3] = {0.0, 0.0, 0.0};
    int sel = -1;
    uint64_t blk = 0;
    U4 u;
    for (int k0 = 0; k0 < a.K; k0 += 32) {
        uint32_t mm = a.K <= 32 ? m : (a.K - k0 >= 32 ? 0xffffffffu : (1u << (a.K - k0)) - 1u);
        while (mm) {
            const int k = k0 + __ffs(mm) - 1;
            mm &= mm - 1;
            const float vis = __half2float(__ldg(a.vis16 + p * a.vstride + k));
            const double t = a.lum_f64 ? lum_at<true>(a, k, p) : lum_at<false>(a, k, p);
            if (kNls) {
                const double w = wrs_weight(vis, t, clamp_lo(a.floor));
                s = __dadd_rn(s, w);
                if (w > 0.0) {   // zero weights never need a uniform (u*s < 0 is impossible)
                    const uint64_t n = a.offset + (uint64_t)gp * (uint64_t)a.K + (uint64_t)k;
                    const uint64_t bi = n / 4 + 1;
                    if (bi != blk) {
                        u = philox_fn(bi, a.key);
                        blk = bi;
                    }
                    if (__dmul_rn(u01(u.x[n & 3]), s) < w) {
                        sel = k;
                        wsel = w;
                    }
                }
            } else {
                const double wk = __dmul_rn((double)vis, t);
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) rgb[ch] = __dadd_rn(rgb[ch], __dmul_rn(wk, __ldg(sc.lt_radiance + 3 * k + ch)));
            }
        }
    }
    if (kNls) {
        const uint64_t n = a.offset + (uint64_t)a.p_total * (uint64_t)a.K + 2ull * (uint64_t)gp;
        const U4 b0 = philox_fn(n / 4 + 1, a.key);
        const double u0 = u01(b0.x[n & 3]);
        double u1;
        if ((n & 3) != 3) {
            u1 = u01(b0.x[(n & 3) + 1]);
        } else {
            const U4 b1 = philox_fn(n / 4 + 2, a.key);
            u1 = u01(b1.x[0]);
        }
        double y[3];
        light_point(sc, sel, u0, u1, y);
        a.ids[p] = sel;
        a.big_w[p] = sel >= 0 ? __ddiv_rn(s, wsel > 0.0 ? wsel : 1.0) : 0.0;
        a.pts[3 * p] = y[0];
        a.pts[3 * p + 1] = y[1];
        a.pts[3 * p + 2] = y[2];
    } else {
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) a.rgb[3 * p + ch] = __ddiv_rn(__dmul_rn(rgb[ch], a.albedo[3 * p + ch]), 3.141592653589793);
    }
}

// fp16 pixel-major visibilities (row stride vstride halfs) -> (P, K) f32 (the infer() output)
__global__ void k_vis_out(const __half* __restrict__ vis16, int64_t vstride, int64_t P, int K, float* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P * K) return;
    const int64_t p = i / K;
    out[i] = __half2float(vis16[p * vstride + (i - p * K)]);
}

int make_mnet(const nvc_model* m, MNet& q) {
    NVC_REQUIRE(m && m->params && m->table_h && m->wpack, "pipeline: model state not bound");
    q.n_layers = m->n_layers;
    for (int i = 0; i <= m->n_layers; ++i) {
        q.dims[i] = m->dims[i];
        if (m->dims[i] > 256) {
            set_error("pipeline: layer widths must be <= 256");
            return NVC_ERR_UNSUPPORTED;
        }
    }
    umma_pads(m->dims, m->n_layers, q.np, q.kp);
    int64_t wo = 0, bo = (int64_t)m->levels * m->table_size * m->features;
    int hid = 16, maxnp = 16, nb = 0;
    for (int i = 0; i < m->n_layers; ++i) {
        if (q.np[i] > 256 || q.kp[i] > 256) {
            set_error("pipeline: padded widths must be <= 256");
            return NVC_ERR_UNSUPPORTED;
        }
        q.wofs[i] = (int)wo;
        wo += umma_block_halfs(q.np[i], q.kp[i]);
        bo += (int64_t)m->dims[i + 1] * m->dims[i];
        q.boff[i] = bo;
        bo += m->dims[i + 1];
        if (i >= 1 && q.kp[i] > hid) hid = q.kp[i];
        if (q.np[i] > maxnp) maxnp = q.np[i];
        nb += q.np[i];
    }
    q.wpack_halfs = (int)wo;
    q.act_kp = hid;
    int col = 32;
    while (col < maxnp) col <<= 1;
    q.acc_cols = col;
    q.alpha = m->alpha;
    q.out_sigmoid = m->out_sigmoid;
    q.sm_w = 0;
    q.sm_a0 = (q.wpack_halfs * 2 + 1023) / 1024 * 1024;
    q.sm_a1 = q.sm_a0 + kStages * ((kT * q.kp[0] * 2 + 1023) / 1024 * 1024);
    // as many tiles in flight (4, 2 or 1) as smem holds activation tiles for (C4's 3x128 MLP: 2)
    for (q.slots = kSlots;; q.slots /= 2) {
        q.sm_bias = q.sm_a1 + q.slots * ((kT * q.act_kp * 2 + 1023) / 1024 * 1024);
        q.sm_total = q.sm_bias + (nb * 4 + 127) / 128 * 128 + 1024;
        if (q.sm_total <= 226 * 1024 || q.slots == 1) break;
    }
    q.tmem_cols = col * q.slots;
    if (q.tmem_cols > 512) {
        set_error("pipeline: %d TMEM columns needed", q.tmem_cols);
        return NVC_ERR_UNSUPPORTED;
    }
    if (q.sm_total > 226 * 1024) {
        set_error("pipeline: %d bytes of shared memory needed", q.sm_total);
        return NVC_ERR_UNSUPPORTED;
    }
    return NVC_OK;
}

inline int grid1(int64_t n, int bs) { return (int)((n + bs - 1) / bs); }

// smem layout of k_mlp_ts: weights | 2 A0 tiles per warpgroup | ones tile | bias blocks
bool ts_layout(MNet& q) {
    if (q.n_layers < 2 || q.n_layers > 8) return false;
    const int hid = q.np[0];
    if (hid != 64 && hid != 128) return false;
    for (int l = 0; l < q.n_layers - 1; ++l)   // uniform hidden layers (TMEM sized for them)
        if (q.np[l] != hid || (l > 0 && q.kp[l] != hid)) return false;
    const int o = q.np[q.n_layers - 1], k = q.kp[0];
    if (o % 16 != 0 || o > hid || (hid == 64 && o == 0) || !(k == 16 || k == 32 || k == 64)) return false;
    if (hid == 128 && !(o == 32 || o == 64 || o == 128)) return false;
    if (hid == 64 && !(o == 16 || o == 32 || o == 48 || o == 64)) return false;
    const int wg = hid == 64 ? TsCfg<64>::WG : TsCfg<128>::WG;
    q.ts_hid = hid;
    q.sm_w = 0;
    q.sm_a0 = (q.wpack_halfs * 2 + 1023) / 1024 * 1024;
    q.sm_a1 = q.sm_a0 + 2 * wg * ((kT * q.kp[0] * 2 + 1023) / 1024 * 1024);   // ones tile
    q.sm_bias = q.sm_a1 + kT * 16 * 2;
    q.sm_total = q.sm_bias + q.n_layers * hid * 32 + 1024;
    return q.sm_total <= 227 * 1024;
}

template <int HID, int OUT, int KP0>
int launch_ts(const MNet& w, const nvc_model* m, const uint8_t* tiles, int64_t ntiles, int64_t P, __half* vis16,
              int64_t vstride, int sms, cudaStream_t s) {
    constexpr int wg = TsCfg<HID>::WG;
    int grid = (int)std::min<int64_t>((ntiles + wg - 1) / wg, sms);
    if (const char* e = getenv("NVC_QUERY_GRID")) grid = max(1, min(grid, atoi(e)));
    cudaFuncSetAttribute(k_mlp_ts<HID, OUT, KP0>, cudaFuncAttributeMaxDynamicSharedMemorySize, w.sm_total);
    if (!getenv("NVC_NO_PDL")) {
        // programmatic dependent launch: the MLP's CTAs may start (weights to smem,
        // TMEM alloc) while the encoder's last CTAs run; griddepcontrol.wait in the
        // kernel orders every tile read / vis write after the encoder grid
        // (frame 0.5584 vs 0.5615 ms)
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(TsCfg<HID>::kThreads);
        cfg.dynamicSmemBytes = w.sm_total;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, k_mlp_ts<HID, OUT, KP0>, w, (const float*)m->params, (const uint16_t*)m->wpack,
                           tiles, ntiles, P, vis16, vstride);
    } else {
        k_mlp_ts<HID, OUT, KP0><<<grid, TsCfg<HID>::kThreads, w.sm_total, s>>>(w, m->params, m->wpack, tiles, ntiles,
                                                                               P, vis16, vstride);
    }
    return check_launch("k_mlp_ts");
}

int launch_mlp_ts(const MNet& w, const nvc_model* m, const uint8_t* tiles, int64_t ntiles, int64_t P, __half* vis16,
                  int64_t vstride, int sms, cudaStream_t s) {
    const int o = w.np[w.n_layers - 1], k = w.kp[0];
#define NVC_TS(H, O, K) \
    if (w.ts_hid == H && o == O && k == K) return launch_ts<H, O, K>(w, m, tiles, ntiles, P, vis16, vstride, sms, s);
    NVC_TS(64, 16, 16) NVC_TS(64, 16, 32) NVC_TS(64, 16, 64) NVC_TS(64, 32, 16) NVC_TS(64, 32, 32) NVC_TS(64, 32, 64)
    NVC_TS(64, 48, 16) NVC_TS(64, 48, 32) NVC_TS(64, 48, 64) NVC_TS(64, 64, 16) NVC_TS(64, 64, 32) NVC_TS(64, 64, 64)
    NVC_TS(128, 32, 32) NVC_TS(128, 64, 32) NVC_TS(128, 128, 16) NVC_TS(128, 128, 32) NVC_TS(128, 128, 64)
#undef NVC_TS
    set_error("k_mlp_ts: shape not instantiated");
    return NVC_ERR_UNSUPPORTED;
}

cudaEvent_t g_stage_ev[4] = {nullptr, nullptr, nullptr, nullptr};
int g_n_stage_ev = 0;
inline void stage_mark(int i, cudaStream_t s) {
    if (i < g_n_stage_ev) cudaEventRecord(g_stage_ev[i], s);
}

// encode + MLP: vis16 (K rows of vstride halfs); ws holds the feature tiles
int run_front(const nvc_model* m, const double* pos, int64_t P, uint8_t* tiles, __half* vis16, int64_t vstride,
              cudaStream_t s) {
    MNet q;
    int rc = make_mnet(m, q);
    if (rc) return rc;
    GridDev g = grid_of(m);
    const int64_t ntiles = (P + kT - 1) / kT;
    stage_mark(0, s);
    // k_enc_tiles2 addresses the x-pair table with 32-bit byte offsets
    const bool h2 = !getenv("NVC_ENC_F32") && (int64_t)g.L * g.T * 8 <= 0xffffffffll;
    if (g.F == 2 && g.L == 16 && h2)
    {
        // 10 resident CTAs per SM: the compiler fits the unrolled levels in 48
        // registers with 4 B of spill, and the extra warps hide more gather
        // latency (154 vs 162 us at the 64-register / 8-CTA budget, which
        // spills 32 B; 6, 7, 12 and 16 CTAs measured 160-181 us).
        // NVC_ENC_BLOCKS=8 selects the 8-CTA build (A/B).
        const char* eb = getenv("NVC_ENC_BLOCKS");
        if (eb && atoi(eb) == 8)
            k_enc_tiles2<16, 8><<<(int)ntiles, kT, 0, s>>>(g, m->table_h, pos, P, q.kp[0], tiles);
        else
            k_enc_tiles2<16, 10><<<(int)ntiles, kT, 0, s>>>(g, m->table_h, pos, P, q.kp[0], tiles);
    }
    else if (g.F == 2 && g.L == 8 && h2)
        k_enc_tiles2<8, 10><<<(int)ntiles, kT, 0, s>>>(g, m->table_h, pos, P, q.kp[0], tiles);
    else if (g.F == 4 && g.L == 8 && h2 && !getenv("NVC_ENC_GENERIC"))
        k_enc_tiles4<8><<<(int)ntiles, kT, 0, s>>>(g, m->table_h, pos, P, q.kp[0], tiles);
    else if (g.F == 4 && g.L == 16 && h2 && !getenv("NVC_ENC_GENERIC"))
        k_enc_tiles4<16><<<(int)ntiles, kT, 0, s>>>(g, m->table_h, pos, P, q.kp[0], tiles);
    else if (g.F == 2)
        k_enc_tiles<true><<<(int)ntiles, kT, 0, s>>>(g, m->table_h, pos, P, q.kp[0], tiles);
    else
        k_enc_tiles<false><<<(int)ntiles, kT, 0, s>>>(g, m->table_h, pos, P, q.kp[0], tiles);
    rc = check_launch("k_enc_tiles");
    if (rc) return rc;
    stage_mark(1, s);
    const int sms = num_sms();
    MNet t = q;
    if (ts_layout(t) && !getenv("NVC_MLP_QUADS")) {
        rc = launch_mlp_ts(t, m, tiles, ntiles, P, vis16, vstride, sms, s);
    } else {
        cudaFuncSetAttribute(k_mlp_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, q.sm_total);
        int grid = (int)(ntiles < sms ? ntiles : sms);
        if (const char* e = getenv("NVC_QUERY_GRID")) grid = max(1, min(grid, atoi(e)));
        k_mlp_tiles<<<grid, kMlpThreads, q.sm_total, s>>>(q, m->params, m->wpack, tiles, ntiles, P, vis16, vstride);
        rc = check_launch("k_mlp_tiles");
    }
    stage_mark(2, s);
    return rc;
}

}  // namespace

int64_t pipeline_workspace_bytes(const nvc_model* m, int64_t P) {
    const int kp0 = umma_kpad(m->levels * m->features);
    const int64_t ntiles = (P + kT - 1) / kT;
    const int64_t vstride = (m->dims[m->n_layers] + 7) / 8 * 8;
    return ntiles * kT * kp0 * 2 + ntiles * kT * vstride * 2 + 1024;
}

namespace {
struct QueryWs {
    uint8_t* tiles;
    __half* vis16;
    int64_t vstride;
};
QueryWs query_ws(const nvc_model* m, int64_t P, void* ws) {
    const int kp0 = umma_kpad(m->levels * m->features);
    const int64_t ntiles = (P + kT - 1) / kT;
    QueryWs q;
    q.tiles = reinterpret_cast<uint8_t*>(ws);
    q.vis16 = reinterpret_cast<__half*>(q.tiles + (ntiles * kT * kp0 * 2 + 255) / 256 * 256);
    q.vstride = (m->dims[m->n_layers] + 7) / 8 * 8;   // pixel-major fp16 rows
    return q;
}
}  // namespace

// encoder + MLP: fp16 visibilities of P pixels into the workspace
int pipeline_front(const nvc_model* m, const double* pos, int64_t P, void* ws, cudaStream_t s) {
    const QueryWs q = query_ws(m, P, ws);
    return run_front(m, pos, P, q.tiles, q.vis16, q.vstride, s);
}

// selection (mode 1: NLS reservoir + light point; 2: Neural DI; 0: f32 visibilities)
// from the visibilities pipeline_front left in the workspace
int pipeline_select(const nvc_model* m, const nvc_scene* sc, int64_t P, int mode, const void* lum, int lum_f64,
                    int64_t stride, const uint32_t* nz_mask, int64_t p_first, int64_t p_total, uint64_t key,
                    uint64_t offset, double floor, int64_t* ids, double* pts, double* big_w, const double* albedo,
                    double* rgb, float* vis_out, void* ws, cudaStream_t s) {
    const QueryWs q = query_ws(m, P, ws);
    const int K = m->dims[m->n_layers];
    if (mode == 0) {
        k_vis_out<<<grid1(P * K, 256), 256, 0, s>>>(q.vis16, q.vstride, P, K, vis_out);
        return check_launch("k_vis_out");
    }
    WArgs a;
    memset(&a, 0, sizeof a);
    a.vis16 = q.vis16;
    a.vstride = q.vstride;
    a.lum = lum;
    a.lum_f64 = lum_f64;
    a.stride = stride;
    a.nz_mask = nz_mask;
    a.P = P;
    a.p_first = p_first;
    a.p_total = p_total;
    a.K = K;
    a.key = key;
    a.offset = offset;
    a.floor = floor;
    a.ids = ids;
    a.pts = pts;
    a.big_w = big_w;
    a.albedo = albedo;
    a.rgb = rgb;
    a.grp0 = offset / 4 + 1;
    a.lp0 = offset + (uint64_t)p_total * (uint64_t)K;
    a.stride32 = (uint32_t)stride;
    const bool aligned = K % 4 == 0 && offset % 4 == 0 && ((uint64_t)p_total * (uint64_t)K) % 2 == 0;
    const bool small = (uint64_t)p_total < (1ull << 31) && (uint64_t)stride * (uint64_t)K < (1ull << 32) &&
                       (uint64_t)p_total * (uint64_t)(K / 4) < (1ull << 32);   // k_nls32g's 32-bit index math
    if (mode == 1 && K <= 128 && aligned && small && getenv("NVC_WRS_FORWARD") == nullptr) {
        if (K <= 32)
            launch_nlsg<1>(a, *sc, P, s);
        else if (K <= 64)
            launch_nlsg<2>(a, *sc, P, s);
        else
            launch_nlsg<4>(a, *sc, P, s);
    } else if (mode == 1 && K <= 32 && getenv("NVC_WRS_FORWARD") == nullptr) {
        if (lum_f64)
            k_nls32<true><<<grid1(P, kWrsThreads), kWrsThreads, 0, s>>>(a, *sc);
        else
            k_nls32<false><<<grid1(P, kWrsThreads), kWrsThreads, 0, s>>>(a, *sc);
    } else if (mode == 1) {
        k_wrs_tiles<true><<<grid1(P, 256), 256, 0, s>>>(a, *sc);
    } else if (K <= 32 && !lum_f64 && getenv("NVC_WRS_FORWARD") == nullptr) {
        k_ndi32<<<grid1(P, kNdiThreads), kNdiThreads, 0, s>>>(a, *sc);
    } else {
        k_wrs_tiles<false><<<grid1(P, 256), 256, 0, s>>>(a, *sc);
    }
    const int rc = check_launch("k_wrs_tiles");
    stage_mark(3, s);
    return rc;
}

int pipeline_query(const nvc_model* m, const nvc_scene* sc, const double* pos, int64_t P, int mode,
                   const void* lum, int lum_f64, int64_t stride, const uint32_t* nz_mask, int64_t p_first, int64_t p_total,
                   uint64_t key, uint64_t offset, double floor, int64_t* ids, double* pts, double* big_w,
                   const double* albedo, double* rgb, float* vis_out, void* ws, cudaStream_t s) {
    int rc = pipeline_front(m, pos, P, ws, s);
    if (rc) return rc;
    return pipeline_select(m, sc, P, mode, lum, lum_f64, stride, nz_mask, p_first, p_total, key, offset, floor, ids,
                           pts, big_w, albedo, rgb, vis_out, ws, s);
}


// ---------------------------------------------------------------------------
// Training MLP on the tensor cores: forward and backward of one 128-row tile
// per CTA as tcgen05 MMAs with fp32 accumulators in TMEM, at fp32-level
// accuracy through split fp16 operands.
//
// Every operand x is stored as bf16 hi = bf16(x) and lo = bf16(x - hi) (16-17
// significant bits, the full fp32 exponent range: init-scale activations and
// output deltas are ~1e-6, below what fp16 can split), and each product takes
// the three terms hi*hi + lo*hi + hi*lo.  An activation tile A_l (128 rows x w <= 64 columns) is kept as one
// K-major SW128 "stack" [128 x 128]: hi in columns 0..63, lo in 64..127.  The
// same bytes serve both roles through the MMA's major-ness bits:
//   forward   Z_l   = A_l . W_l^T     A K-major (hi, then lo K-steps),
//                                     B = W_l K-major (hi, reused for lo), + A_hi . W_lo^T
//   backward  dW_l^T = A_l^T . dZ_l   A = the stack MN-major: M = 128 = [hi | lo] rows
//                                     of dW^T, B = dZ MN-major (hi, then lo) -- the
//                                     two halves are the hi and lo partials
//             dA_l  = dZ_l . W_l      A = dZ stack K-major, B = W_l MN-major
// db is a fixed-order column sum of dZ (warp butterfly + 4-way add).  dZ is
// carried scaled by 2^18 (it starts near 2(out-t)/(bK) ~ 1e-6) and unscaled on
// read-out.  Per-CTA dW/db partials (two sets: the hi and lo halves of dW^T)
// go to the part_w layout k_reduce_parts sums as fixed point per set; dA_0
// feeds the hash-grid scatter.  Widths <= 64 (C1, C2); wider models use the
// fp32 SIMT k_train3.
// ---------------------------------------------------------------------------
namespace {
constexpr float kGradScale = 262144.0f;   // 2^18
constexpr int kTcThreads = 512;           // 16 warps: TMEM lane quarter = warp & 3, column quarter = warp >> 2
constexpr int kTcWarps = kTcThreads / 32;

struct TrainTC {
    int L, D0, K;
    int dims[NVC_MAX_LAYERS + 1], np[NVC_MAX_LAYERS], kp[NVC_MAX_LAYERS];
    int64_t woff_abs[NVC_MAX_LAYERS], boff_abs[NVC_MAX_LAYERS];
    int64_t woff_rel[NVC_MAX_LAYERS], boff_rel[NVC_MAX_LAYERS], mlp_count;
    float alpha;
    int out_sigmoid;
    int terms;            // split-precision terms per product (3; 1 = hi only, diagnostics)
    int sm_whi[NVC_MAX_LAYERS], sm_wlo[NVC_MAX_LAYERS], sm_a[NVC_MAX_LAYERS], sm_dz, sm_bias, sm_db, sm_total;
};

__device__ __forceinline__ float sigmoid_exact(float z) {   // mlp.py:101-107
    if (z >= 0.0f) return __fdiv_rn(1.0f, __fadd_rn(1.0f, expf(-z)));
    const float e = expf(z);
    return __fdiv_rn(e, __fadd_rn(1.0f, e));
}

// MN-major descriptor over a [rows x kp] K-major swizzled tile: MN = its columns
// (2^lg-byte swizzle rows, atoms `rows` rows apart), K = its rows, step kk = 16 rows
__device__ __forceinline__ uint64_t desc_mn(uint32_t base, int rows, int kp, int kk) {
    const int lg = umma_sw_log2(kp);
    const uint32_t addr = base + (uint32_t)kk * (16u << lg);
    const uint64_t layout = lg == 7 ? 2ull : (lg == 6 ? 4ull : 6ull);
    return (uint64_t)((addr & 0x3FFFFu) >> 4) | ((uint64_t)((((uint32_t)rows << lg) >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((8u << lg) >> 4) << 32) | ((uint64_t)1 << 46) | (layout << 61);
}
// bf16 x bf16 -> f32 (the 8-bit exponent keeps init-scale activations ~1e-6 and
// output deltas ~1e-6 normal, which fp16 could not split)
__device__ __forceinline__ uint32_t idesc_bf16(int m, int n, bool a_mn, bool b_mn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
           ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void split_h(float x, __nv_bfloat16& hi, __nv_bfloat16& lo) {
    hi = __float2bfloat16_rn(x);
    lo = __float2bfloat16_rn(x - __bfloat162float(hi));
}
// 8 consecutive columns c0..c0+7 (c0 % 8 == 0) of row r into a [128 x 128] stack: hi at c, lo at 64 + c
__device__ __forceinline__ void put_stack8(uint8_t* stack, int r, int c0, const float v[8]) {
    __align__(16) __nv_bfloat16 hi[8], lo[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) split_h(v[i], hi[i], lo[i]);
    *reinterpret_cast<uint4*>(stack + umma_off(r, c0, kT, 128)) = *reinterpret_cast<const uint4*>(hi);
    *reinterpret_cast<uint4*>(stack + umma_off(r, 64 + c0, kT, 128)) = *reinterpret_cast<const uint4*>(lo);
}
// the 32 values of a warp's lanes for 16 columns -> lanes l and l ^ 16 hold column
// (l & 15)'s sum (fixed order: butterfly over lane bits 3..0, then bit 4)
__device__ __forceinline__ float col_sum16(float v[16], int lane) {
#pragma unroll
    for (int s = 8; s >= 1; s >>= 1) {
        const bool up = (lane & s) != 0;
#pragma unroll
        for (int j = 0; j < s; ++j) {
            const float send = up ? v[j] : v[j + s];
            const float keep = up ? v[j + s] : v[j];
            v[j] = keep + __shfl_xor_sync(0xffffffffu, send, s);
        }
    }
    return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 16);
}

__global__ void __launch_bounds__(kTcThreads, 1) k_train_tc(TrainTC t, const float* __restrict__ params,
                                                           const float* __restrict__ act0g, int64_t b_max,
                                                           const int64_t* __restrict__ b_dev, int shard,
                                                           int n_shards, const float* __restrict__ tgt,
                                                           const float* __restrict__ mask,
                                                           float* __restrict__ dact0g, float* __restrict__ part_w,
                                                           double* __restrict__ part_loss) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    __shared__ double s_loss[kTcWarps];
    uint8_t* sm = smem_raw + ((1024u - (s32(smem_raw) & 1023u)) & 1023u);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int q = warp & 3, h = warp >> 2;          // TMEM lane quarter, 16-column quarter
    const int r = 32 * q + lane;                   // the tile row this thread reads from TMEM
    const int64_t b = b_dev ? *b_dev : b_max;
    int64_t lo, hi;
    shard_range(b, shard, n_shards, lo, hi);
    const int64_t r0g = (int64_t)blockIdx.x * kT;
    const int nr = (int)max((int64_t)0, min((int64_t)kT, (hi - lo) - r0g));
    const int L = t.L;
    float* bias = reinterpret_cast<float*>(sm + t.sm_bias);
    float* s_db = reinterpret_cast<float*>(sm + t.sm_db);      // [2][16 warps][16 columns]
    uint8_t* dz = sm + t.sm_dz;
    {   // weights (hi / lo, K-major [np x kp]), biases, the input stack
        for (int l = 0; l < L; ++l) {
            const int np = t.np[l], kp = t.kp[l], N = t.dims[l + 1], Kin = t.dims[l];
            for (int i = tid; i < np * kp / 8; i += kTcThreads) {
                const int n = i / (kp / 8), k0 = (i % (kp / 8)) * 8;
                float w[8];
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    w[j] = (n < N && k0 + j < Kin) ? __ldg(params + t.woff_abs[l] + (int64_t)n * Kin + k0 + j) : 0.0f;
                __align__(16) __nv_bfloat16 wh[8], wl[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) split_h(w[j], wh[j], wl[j]);
                *reinterpret_cast<uint4*>(sm + t.sm_whi[l] + umma_off(n, k0, np, kp)) = *reinterpret_cast<const uint4*>(wh);
                *reinterpret_cast<uint4*>(sm + t.sm_wlo[l] + umma_off(n, k0, np, kp)) = *reinterpret_cast<const uint4*>(wl);
            }
            for (int n = tid; n < 64; n += kTcThreads) bias[64 * l + n] = n < N ? __ldg(params + t.boff_abs[l] + n) : 0.0f;
        }
        // thread (row, quarter hh) stages input columns [16hh, 16hh + 16) of its row
        const int row = tid & 127, hh = tid >> 7;
        for (int c0 = 16 * hh; c0 < 16 * hh + 16 && c0 < t.kp[0]; c0 += 8) {
            float v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j)
                v[j] = (row < nr && c0 + j < t.D0) ? __ldg(act0g + (r0g + row) * t.D0 + c0 + j) : 0.0f;
            put_stack8(sm + t.sm_a[0], row, c0, v);
        }
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s32(&tbase)), "r"(256)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    uint32_t phase = 0;
    auto sync_issue = [&]() {   // generic smem writes -> async proxy; then thread 0 issues
        fence_async();
        tc_before();
        __syncthreads();
        tc_after();
    };
    auto wait_mma = [&]() {
        if (tid == 0) commit(&bar);
        mbar_wait(&bar, phase);
        phase ^= 1u;
        tc_after();
    };
    sync_issue();
    const uint32_t tmem = tbase;
    const uint32_t acc_f = tmem, acc_dw = tmem + 64u, acc_da = tmem + 128u;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    auto ld16 = [&](uint32_t col, float v[16]) {     // this warp's 32 lanes x columns [col, col + 16)
        uint32_t u[16];
        tld16_nowait(lane_base + col, u);
        tld_wait();
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(u[i]);
    };
    // db partials double-buffered by layer parity: a layer's flush and the next
    // layer's column sums never share a buffer between barriers
    auto db_out = [&](int l, float v[16]) {          // column sums of dZ_l (this warp's 16 columns)
        const float cs = col_sum16(v, lane);
        if (lane < 16) s_db[(l & 1) * 256 + warp * 16 + lane] = cs;
    };
    auto db_flush = [&](int l) {                     // after a __syncthreads: 4 lane quarters in fixed order
        if (tid < 64 && tid < t.dims[l + 1]) {
            const int hh = tid >> 4, c = tid & 15;
            const float* sd = s_db + (l & 1) * 256;
            const float sum = ((sd[(4 * hh + 0) * 16 + c] + sd[(4 * hh + 1) * 16 + c]) + sd[(4 * hh + 2) * 16 + c]) +
                              sd[(4 * hh + 3) * 16 + c];
            float* base = part_w + (int64_t)(2 * blockIdx.x) * t.mlp_count;
            base[t.boff_rel[l] + tid] = sum * (1.0f / kGradScale);
            base[t.mlp_count + t.boff_rel[l] + tid] = 0.0f;   // the lo set carries no bias
        }
    };
    const uint32_t a_addr0 = s32(sm);

    // ---- forward ----
    double lsum = 0.0;
    const float bk = (float)(b * (int64_t)t.K);
    for (int l = 0; l < L; ++l) {
        const int np = t.np[l], ns = t.kp[l] / 16, N = t.dims[l + 1];
        if (tid == 0) {
            const uint32_t a = a_addr0 + t.sm_a[l], wh = a_addr0 + t.sm_whi[l], wl = a_addr0 + t.sm_wlo[l];
            const uint32_t id = idesc_bf16(kT, np, false, false);
            for (int s2 = 0; s2 < ns; ++s2) mma(acc_f, desc_of(a, kT, 128, s2), desc_of(wh, np, t.kp[l], s2), id, s2 > 0);
            if (t.terms > 1) {
                for (int s2 = 0; s2 < ns; ++s2)
                    mma(acc_f, desc_of(a, kT, 128, 4 + s2), desc_of(wh, np, t.kp[l], s2), id, 1);
                for (int s2 = 0; s2 < ns; ++s2)
                    mma(acc_f, desc_of(a, kT, 128, s2), desc_of(wl, np, t.kp[l], s2), id, 1);
            }
        }
        wait_mma();
        if (16 * h < np) {
            float v[16];
            ld16(acc_f + (uint32_t)(16 * h), v);
            const bool last = l == L - 1;
            float o[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int n = 16 * h + i;
                const float z = v[i] + bias[64 * l + n];
                if (!last) {
                    o[i] = n < N ? (z >= 0.0f ? z : t.alpha * z) : 0.0f;
                } else {
                    // loss + output delta (mlp.py:143-149, 160-168), dZ scaled by 2^18
                    float d = 0.0f;
                    if (r < nr && n < t.K) {
                        const float sg = t.out_sigmoid ? sigmoid_exact(z) : (z >= 0.0f ? z : t.alpha * z);
                        const int64_t li = (r0g + r) * t.K + n;
                        const float outc = t.out_sigmoid ? fminf(fmaxf(sg, 1e-6f), 0.999999f) : sg;
                        const float tt = tgt[li];
                        const float mk = mask ? mask[li] : 1.0f;
                        float dd = __fsub_rn(outc, tt);
                        if (mask) dd = __fmul_rn(dd, mk);
                        lsum += (double)__fmul_rn(dd, dd);
                        float dout = __fdiv_rn(__fmul_rn(2.0f, __fsub_rn(sg, tt)), bk);
                        if (mask) dout = __fmul_rn(dout, mk);
                        d = t.out_sigmoid ? __fmul_rn(__fmul_rn(dout, sg), __fsub_rn(1.0f, sg))
                                          : (z >= 0.0f ? dout : __fmul_rn(dout, t.alpha));
                    }
                    o[i] = d * kGradScale;
                }
            }
            uint8_t* dst = last ? dz : sm + t.sm_a[l + 1];
#pragma unroll
            for (int c = 0; c < 16; c += 8) put_stack8(dst, r, 16 * h + c, o + c);
            if (last) db_out(l, o);
        } else if (l == L - 1) {
            float zero[16] = {};
            db_out(l, zero);
        }
        sync_issue();
        if (l == L - 1) db_flush(l);
    }
    for (int o = 16; o; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
    if (lane == 0) s_loss[warp] = lsum;

    // ---- backward ----
    for (int l = L - 1; l >= 0; --l) {
        const int np = t.np[l], kp = t.kp[l], nsn = np / 16, Kin = t.dims[l], N = t.dims[l + 1];
        if (tid == 0) {
            const uint32_t a = a_addr0 + t.sm_a[l], dzb = a_addr0 + t.sm_dz;
            const uint32_t wh = a_addr0 + t.sm_whi[l], wl = a_addr0 + t.sm_wlo[l];
            // dW^T = [A_hi | A_lo]^T . dZ: K = 128 rows, B = dZ hi then dZ lo (MN-major)
            const uint32_t idw = idesc_bf16(kT, np, true, true);
            for (int kk = 0; kk < kT / 16; ++kk)
                mma(acc_dw, desc_mn(a, kT, 128, kk), desc_mn(dzb, kT, 128, kk), idw, kk > 0);
            if (t.terms > 1)
                for (int kk = 0; kk < kT / 16; ++kk)
                    mma(acc_dw, desc_mn(a, kT, 128, kk), desc_mn(dzb + kT * 128u, kT, 128, kk), idw, 1);
            // dA = dZ . W: A = dZ stack K-major (K = N_out), B = W MN-major (N = K_in)
            const uint32_t ida = idesc_bf16(kT, kp, false, true);
            for (int s2 = 0; s2 < nsn; ++s2) mma(acc_da, desc_of(dzb, kT, 128, s2), desc_mn(wh, np, kp, s2), ida, s2 > 0);
            if (t.terms > 1) {
                for (int s2 = 0; s2 < nsn; ++s2)
                    mma(acc_da, desc_of(dzb, kT, 128, 4 + s2), desc_mn(wh, np, kp, s2), ida, 1);
                for (int s2 = 0; s2 < nsn; ++s2)
                    mma(acc_da, desc_of(dzb, kT, 128, s2), desc_mn(wl, np, kp, s2), ida, 1);
            }
        }
        wait_mma();
        // dW^T lanes m = [hi k_in | lo k_in]: the hi and lo partial sets
        {
            const int m = r, k = m & 63, set = m >> 6;
            if (16 * h < np) {
                float v[16];
                ld16(acc_dw + (uint32_t)(16 * h), v);
                if (k < Kin) {
                    float* gw = part_w + (int64_t)(2 * blockIdx.x + set) * t.mlp_count + t.woff_rel[l];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const int n = 16 * h + i;
                        if (n < N) gw[(int64_t)n * Kin + k] = v[i] * (1.0f / kGradScale);
                    }
                }
            }
        }
        // dA rows: the next dZ (times leaky'(z), from the sign of the stored activation) or dL/dact0
        if (16 * h < kp) {
            float v[16];
            ld16(acc_da + (uint32_t)(16 * h), v);
            if (l > 0) {
                const uint8_t* a = sm + t.sm_a[l];
                float o[16];
#pragma unroll
                for (int c = 0; c < 16; c += 8) {
                    const uint4 pk = *reinterpret_cast<const uint4*>(a + umma_off(r, 16 * h + c, kT, 128));
                    const uint16_t* hv = reinterpret_cast<const uint16_t*>(&pk);
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int k2 = 16 * h + c + i;
                        const bool neg = (hv[i] & 0x8000u) != 0;       // leaky'(z): z >= 0 -> 1, else alpha
                        o[c + i] = (r < nr && k2 < Kin) ? (neg ? v[c + i] * t.alpha : v[c + i]) : 0.0f;
                    }
                }
                // dZ_{l-1} overwrites dZ_l: every MMA that read it has completed
#pragma unroll
                for (int c = 0; c < 16; c += 8) put_stack8(dz, r, 16 * h + c, o + c);
                db_out(l - 1, o);
            } else if (r < nr) {
#pragma unroll
                for (int i = 0; i < 16; ++i)
                    if (16 * h + i < t.D0) dact0g[(r0g + r) * t.D0 + 16 * h + i] = v[i] * (1.0f / kGradScale);
            }
        } else if (l > 0) {
            float zero[16] = {};
            db_out(l - 1, zero);
        }
        sync_issue();
        if (l > 0) db_flush(l - 1);
    }
    if (tid == 0) {
        double ls = 0.0;
        for (int w = 0; w < kTcWarps; ++w) ls += s_loss[w];
        part_loss[2 * blockIdx.x] = ls / (double)t.K;
        part_loss[2 * blockIdx.x + 1] = 0.0;
    }
    tc_before();
    __syncthreads();
    tc_after();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256) : "memory");
}
}  // namespace

// plan: 0 if the tensor-core training step covers this model (widths <= 64, fits in smem)
int train_tc_plan(const nvc_model* m, int64_t grid_count, const int64_t* woff, const int64_t* boff, int64_t mlp_count,
                  TrainTC& t) {
    if (m->n_layers < 2 || m->n_layers > 4 || m->features * m->levels > 64) return 1;
    t.L = m->n_layers;
    t.D0 = m->dims[0];
    t.K = m->dims[m->n_layers];
    for (int i = 0; i <= t.L; ++i) t.dims[i] = m->dims[i];
    umma_pads(m->dims, t.L, t.np, t.kp);
    for (int l = 0; l < t.L; ++l) {
        if (t.np[l] > 64 || t.kp[l] > 64 || t.np[l] % 16 || (t.kp[l] != 16 && t.kp[l] != 32 && t.kp[l] != 64)) return 1;
        t.woff_abs[l] = woff[l];
        t.boff_abs[l] = boff[l];
        t.woff_rel[l] = woff[l] - grid_count;
        t.boff_rel[l] = boff[l] - grid_count;
    }
    t.mlp_count = mlp_count;
    t.alpha = m->alpha;
    t.out_sigmoid = m->out_sigmoid;
    t.terms = getenv("NVC_TC_TERMS") ? atoi(getenv("NVC_TC_TERMS")) : 3;
    auto al = [](int x) { return (x + 1023) / 1024 * 1024; };
    int so = 0;
    for (int l = 0; l < t.L; ++l) {
        t.sm_whi[l] = so;
        so += al(t.np[l] * t.kp[l] * 2);
        t.sm_wlo[l] = so;
        so += al(t.np[l] * t.kp[l] * 2);
    }
    for (int l = 0; l < t.L; ++l) {
        t.sm_a[l] = so;
        so += kT * 128 * 2;
    }
    t.sm_dz = so;
    so += kT * 128 * 2;
    t.sm_bias = so;
    so += al(t.L * 64 * 4);
    t.sm_db = so;
    so += al(2 * 256 * 4);
    t.sm_total = so + 1024;
    return t.sm_total <= 227 * 1024 ? 0 : 1;
}

// the whole step: returns 1 (nothing launched) when the model is not covered; part_w
// / part_loss receive two partial sets per 128-row tile (nblk_sets = 2 * tiles)
int train_tc(const nvc_model* m, int64_t grid_count, const int64_t* woff, const int64_t* boff, int64_t mlp_count,
             const float* act0, int64_t b_max, const int64_t* b_dev, int shard, int n_shards, const float* tgt,
             const float* mask, float* dact0, float* part_w, double* part_loss, int ntiles, cudaStream_t s) {
    TrainTC t;
    if (train_tc_plan(m, grid_count, woff, boff, mlp_count, t)) return 1;
    cudaFuncSetAttribute(k_train_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, t.sm_total);
    k_train_tc<<<ntiles, kTcThreads, t.sm_total, s>>>(t, m->params, act0, b_max, b_dev, shard, n_shards, tgt, mask,
                                                      dact0, part_w, part_loss);
    return check_launch("k_train_tc");
}

}  // namespace nvc


extern "C" int nvc_profile_stages(int32_t enable) {
    if (enable && !nvc::g_stage_ev[0])
        for (int i = 0; i < 4; ++i)
            if (cudaEventCreate(&nvc::g_stage_ev[i]) != cudaSuccess) {
                nvc::set_error("nvc_profile_stages: cudaEventCreate failed");
                return NVC_ERR_CUDA;
            }
    nvc::g_n_stage_ev = enable ? 4 : 0;
    return NVC_OK;
}

extern "C" int nvc_profile_stage_ms(float* ms3) {
    if (!ms3 || !nvc::g_stage_ev[0]) {
        nvc::set_error("nvc_profile_stage_ms: profiling never enabled");
        return NVC_ERR_ARG;
    }
    if (cudaEventSynchronize(nvc::g_stage_ev[3]) != cudaSuccess) return NVC_ERR_CUDA;
    for (int i = 0; i < 3; ++i)
        if (cudaEventElapsedTime(ms3 + i, nvc::g_stage_ev[i], nvc::g_stage_ev[i + 1]) != cudaSuccess) {
            cudaGetLastError();
            nvc::set_error("nvc_profile_stage_ms: no recorded query since enabling");
            return NVC_ERR_CUDA;
        }
    return NVC_OK;
}

#ifdef NVC_MLP_TRACE
extern "C" int nvc_mlp_trace_get(long long* host) {
    return cudaMemcpyFromSymbol(host, nvc::g_mlp_trace, sizeof(nvc::g_mlp_trace)) == cudaSuccess ? 0 : -1;
}
#endif
