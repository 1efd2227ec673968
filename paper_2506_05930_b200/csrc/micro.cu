// micro.cu -- tcgen05 microbenchmarks used to calibrate the query kernel
// (MMA issue/throughput, commit->mbarrier round trip, TMEM load latency).
// Profiling aid only; not on the product path.
#include "common.cuh"

namespace nvc {
namespace {

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc_sw128(uint32_t addr) {
    uint64_t d = 0;
    d |= (uint64_t)((addr & 0x3FFFFu) >> 4);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024u >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= 2ull << 61;
    return d;
}

// mode 0: back-to-back MMAs (N=64, K=16) with one commit at the end
// mode 1: MMA + commit + wait round trips
// mode 2: tcgen05.ld x16 + wait::ld round trips (4 warps)
__global__ void __launch_bounds__(128, 1) k_micro(int mode, int iters, int n, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    uint8_t* sm = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
    for (int i = threadIdx.x; i < 48 * 1024 / 16; i += 128) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su32(&tbase)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = tbase;
    const uint32_t idesc = (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t ad = desc_sw128(su32(sm)), bd = desc_sw128(su32(sm + 16384));
    uint32_t phase = 0;
    long long t0 = clock64();
    if (mode == 0) {
        if (threadIdx.x == 0) {
            for (int i = 0; i < iters; ++i)
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
                             "l"(ad), "l"(bd), "r"(idesc), "r"(1)
                             : "memory");
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                         : "memory");
        }
        asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
                     "@P1 bra D_%=;\n\tbra W_%=;\nD_%=:\n\t}" ::"r"(su32(&bar)), "r"(phase)
                     : "memory");
    } else if (mode == 1) {
        for (int i = 0; i < iters; ++i) {
            if (threadIdx.x == 0) {
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                for (int kk = 0; kk < 4; ++kk)
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
                                 "l"(ad + 2 * kk), "l"(bd + 2 * kk), "r"(idesc), "r"(kk)
                                 : "memory");
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 su32(&bar))
                             : "memory");
            }
            asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
                         "@P1 bra D_%=;\n\tbra W_%=;\nD_%=:\n\t}" ::"r"(su32(&bar)), "r"(phase)
                         : "memory");
            phase ^= 1;
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncthreads();
        }
    } else {
        const uint32_t tr = tm + ((uint32_t)((threadIdx.x >> 5) * 32) << 16);
        float acc = 0.0f;
        for (int i = 0; i < iters; ++i) {
            uint32_t r[16];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                  "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                : "r"(tr + (uint32_t)((i & 3) * 16)));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            acc += __uint_as_float(r[0]) + __uint_as_float(r[15]);
        }
        if (acc == 1.2345f) out[3] = 1;
    }
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) {
        out[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tm) : "memory");
}

}  // namespace
}  // namespace nvc

extern "C" int nvc_micro(int mode, int iters, int n, int blocks, long long* out_dev, void* stream) {
    cudaFuncSetAttribute(nvc::k_micro, cudaFuncAttributeMaxDynamicSharedMemorySize, 50 * 1024);
    nvc::k_micro<<<blocks, 128, 50 * 1024, (cudaStream_t)stream>>>(mode, iters, n, out_dev);
    return nvc::check_launch("k_micro");
}
