// rgbdseg_bulk.cu -- K1 over TMA bulk copies (sm_100a): the fused colour GMM +
// depth GMM + List-1 fusion pass with every plane staged through shared
// memory by cp.async.bulk.
//
// Each warp is an independent pipeline over 32-pixel chunks (grid-stride,
// persistent grid).  For a chunk, lanes issue one 1-D bulk copy per plane
// (40 float planes at M=5/5 plus the byte planes: 48 copies, 5.4 KB) into a
// shared-memory stage guarded by an mbarrier with expect_tx; while chunk k is
// computed, chunk k+1 is already in flight into the other stage.  Lane l owns
// pixel l of the chunk and reads its mixture with immediate-offset LDS (no
// per-plane 64-bit address arithmetic, the dominant instruction cost of the
// LDG version), writes the updated words back in place, and the warp then
// bulk-stores only the plane chunks some lane changed (dirty mask OR-reduced
// across the warp), at 128-byte granularity -- write elision without
// per-word predicated stores.
#include <algorithm>

#include "rgbdseg_kernels.cuh"

namespace rgbdseg_b200 {
namespace {

constexpr int kChunk = 32;          // pixels per warp chunk
constexpr int kWarpsPerBlock = 4;   // 128 threads
constexpr int kStages = 2;

template <int MC, int MD>
struct Layout {
    static constexpr int NFC = 5 * MC;  // colour float planes: 3M means + M var + M w
    static constexpr int NFD = 3 * MD;  // depth float planes: M means + M var + M w
    static constexpr int NF = NFC + NFD;
    // byte offsets inside one stage
    static constexpr int F = 0;                          // float planes, 128 B each
    static constexpr int R = F + NF * kChunk * 4;         // r, g, b: 32 B each
    static constexpr int G = R + kChunk;
    static constexpr int B = G + kChunk;
    static constexpr int D = B + kChunk;                  // depth u16: 64 B
    static constexpr int CF = D + 2 * kChunk;             // colour flags
    static constexpr int DF = CF + kChunk;                // depth flags
    static constexpr int OUT = DF + kChunk;               // fusion out
    static constexpr int CPT = OUT + kChunk;              // fusion cpt
    static constexpr int BYTES = CPT + kChunk;
    static constexpr int STAGE = (BYTES + 127) & ~127;
    static constexpr int NCOPY = NF + 8;                  // bulk copies per chunk
    // dirty-mask bit of each stored plane: float planes 0..NF-1, then bytes
    static constexpr int BIT_CF = NF, BIT_DF = NF + 1, BIT_OUT = NF + 2, BIT_CPT = NF + 3;
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAIT_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes,
                                          uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}

__device__ __forceinline__ void bulk_store(void* dst, uint32_t src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Global address and size of copy `q` (plane order of Layout) for the chunk
// starting at pixel i0 of this launch.
template <int MC, int MD>
__device__ __forceinline__ void plane_src(const FusedArgs& a, int q, size_t i0, const char*& g,
                                          uint32_t& off, uint32_t& bytes) {
    using L = Layout<MC, MD>;
    const size_t j0 = a.base + i0;
    if (q < L::NFC) {
        g = reinterpret_cast<const char*>(a.color.state + (size_t)q * a.color.pitch + j0);
        off = L::F + q * kChunk * 4;
        bytes = kChunk * 4;
    } else if (q < L::NF) {
        g = reinterpret_cast<const char*>(a.depth.state + (size_t)(q - L::NFC) * a.depth.pitch + j0);
        off = L::F + q * kChunk * 4;
        bytes = kChunk * 4;
    } else {
        bytes = kChunk;
        switch (q - L::NF) {
            case 0: g = (const char*)(a.r + i0); off = L::R; break;
            case 1: g = (const char*)(a.g + i0); off = L::G; break;
            case 2: g = (const char*)(a.b + i0); off = L::B; break;
            case 3: g = (const char*)(a.d + i0); off = L::D; bytes = 2 * kChunk; break;
            case 4: g = (const char*)(a.color.flags + j0); off = L::CF; break;
            case 5: g = (const char*)(a.depth.flags + j0); off = L::DF; break;
            case 6: g = (const char*)(a.out + i0); off = L::OUT; break;
            default: g = (const char*)(a.cpt + i0); off = L::CPT; break;
        }
    }
}

template <int MC, int MD>
__device__ __forceinline__ void issue_loads(const FusedArgs& a, size_t i0, uint32_t stage,
                                            uint32_t bar, int lane) {
    using L = Layout<MC, MD>;
    if (lane == 0) mbar_expect_tx(bar, L::BYTES);
    __syncwarp();
#pragma unroll
    for (int q0 = 0; q0 < L::NCOPY; q0 += 32) {
        const int q = q0 + lane;
        if (q < L::NCOPY) {
            const char* g;
            uint32_t off, bytes;
            plane_src<MC, MD>(a, q, i0, g, off, bytes);
            bulk_load(stage + off, g, bytes, bar);
        }
    }
}

// Bulk-store every plane chunk whose dirty bit is set (stored planes only:
// floats, flags, out, cpt; the inputs are never written).
template <int MC, int MD>
__device__ __forceinline__ void issue_stores(const FusedArgs& a, size_t i0, uint32_t stage,
                                             uint64_t dirty, int lane) {
    using L = Layout<MC, MD>;
#pragma unroll
    for (int q0 = 0; q0 < L::NCOPY; q0 += 32) {
        const int q = q0 + lane;
        if (q < L::NCOPY) {
            int bit = -1;
            if (q < L::NF) bit = q;
            else if (q == L::NF + 4) bit = L::BIT_CF;
            else if (q == L::NF + 5) bit = L::BIT_DF;
            else if (q == L::NF + 6) bit = L::BIT_OUT;
            else if (q == L::NF + 7) bit = L::BIT_CPT;
            if (bit >= 0 && ((dirty >> bit) & 1ull)) {
                const char* g;
                uint32_t off, bytes;
                plane_src<MC, MD>(a, q, i0, g, off, bytes);
                bulk_store(const_cast<char*>(g), stage + off, bytes);
            }
        }
    }
    bulk_commit();
}

template <int M, int C>
__device__ __forceinline__ void lds_mix(const char* st, int plane0, int lane, Mixture<M, C>& m) {
    const float* f = reinterpret_cast<const float*>(st) + lane;
#pragma unroll
    for (int i = 0; i < M; ++i)
#pragma unroll
        for (int c = 0; c < C; ++c) m.mu[i][c] = f[(plane0 + i * C + c) * kChunk];
#pragma unroll
    for (int i = 0; i < M; ++i) m.var[i] = f[(plane0 + M * C + i) * kChunk];
#pragma unroll
    for (int i = 0; i < M; ++i) m.w[i] = f[(plane0 + M * C + M + i) * kChunk];
}

// Write back the words a step can change and return their dirty bits
// (plane ids offset by plane0).  touched < 0: everything (initialisation).
template <int M, int C, bool kElide>
__device__ __forceinline__ uint64_t sts_mix(char* st, int plane0, int lane,
                                            const Mixture<M, C>& m, int touched,
                                            const float (&w_old)[M]) {
    float* f = reinterpret_cast<float*>(st) + lane;
    uint64_t dirty = 0;
#pragma unroll
    for (int i = 0; i < M; ++i) {
        if (!kElide || touched < 0 || touched == i) {
#pragma unroll
            for (int c = 0; c < C; ++c) f[(plane0 + i * C + c) * kChunk] = m.mu[i][c];
            f[(plane0 + M * C + i) * kChunk] = m.var[i];
        }
    }
#pragma unroll
    for (int i = 0; i < M; ++i) f[(plane0 + M * C + M + i) * kChunk] = m.w[i];
    if (!kElide || touched < 0) {
        dirty = ((1ull << (M * C + 2 * M)) - 1ull) << plane0;
    } else {
        dirty |= ((1ull << C) - 1ull) << (plane0 + touched * C);
        dirty |= 1ull << (plane0 + M * C + touched);
#pragma unroll
        for (int i = 0; i < M; ++i)
            if (__float_as_uint(m.w[i]) != __float_as_uint(w_old[i]))
                dirty |= 1ull << (plane0 + M * C + M + i);
    }
    return dirty;
}

template <int MC, int MD, bool kElide>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    k_fused_bulk(const __grid_constant__ FusedArgs a, size_t nchunks) {
    using L = Layout<MC, MD>;
    extern __shared__ __align__(128) char smem[];
    __shared__ __align__(8) uint64_t bars[kWarpsPerBlock][kStages];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    char* wbase = smem + (size_t)warp * kStages * L::STAGE;
    const uint32_t sbase = smem_addr(wbase);
    const uint32_t bar0 = smem_addr(&bars[warp][0]);
    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < kStages; ++s) mbar_init(bar0 + 8 * s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        fence_async_smem();
    }
    __syncwarp();

    const size_t stride = (size_t)gridDim.x * kWarpsPerBlock;
    size_t c = (size_t)blockIdx.x * kWarpsPerBlock + warp;
    if (c < nchunks) issue_loads<MC, MD>(a, c * kChunk, sbase, bar0, lane);
    for (uint32_t it = 0; c < nchunks; ++it, c += stride) {
        const uint32_t s = it & 1u;
        const uint32_t st = sbase + s * L::STAGE;
        char* stp = wbase + s * L::STAGE;
        // prefetch the next chunk into the other stage once the bulk stores
        // that last read it have drained
        const size_t cn = c + stride;
        if (cn < nchunks) {
            bulk_wait_read_all();
            __syncwarp();
            issue_loads<MC, MD>(a, cn * kChunk, sbase + (s ^ 1u) * L::STAGE, bar0 + 8 * (s ^ 1u),
                                lane);
        }
        mbar_wait(bar0 + 8 * s, (it >> 1) & 1u);

        // ---- this lane's pixel --------------------------------------------
        const size_t i = c * kChunk + lane;
        const uint8_t* b8 = reinterpret_cast<const uint8_t*>(stp);
        const float vc[3] = {(float)b8[L::R + lane], (float)b8[L::G + lane],
                             (float)b8[L::B + lane]};
        const uint32_t raw = reinterpret_cast<const uint16_t*>(stp + L::D)[lane];
        const bool cinit = b8[L::CF + lane] != 0;
        const bool dinit = b8[L::DF + lane] != 0;
        const uint32_t out0 = b8[L::OUT + lane];
        const int cpt0 = (int)reinterpret_cast<const int8_t*>(stp)[L::CPT + lane];
        uint64_t dirty = 0;

        Mixture<MC, 3> cm;
        lds_mix(stp, 0, lane, cm);
        float cw_old[MC];
#pragma unroll
        for (int q = 0; q < MC; ++q) cw_old[q] = cm.w[q];
        int ct = -1;
        uint32_t lc = 0;
        if (!cinit)
            gmm_init(cm, vc, a.ck);
        else
            lc = gmm_step(cm, vc, a.ck, ct);
        dirty |= sts_mix<MC, 3, kElide>(stp, 0, lane, cm, ct, cw_old);
        if (!cinit) {
            stp[L::CF + lane] = 1;
            dirty |= 1ull << L::BIT_CF;
        }

        uint32_t ld = 0;
        if (raw != 0) {
            Mixture<MD, 1> dm;
            lds_mix(stp, L::NFC, lane, dm);
            float dw_old[MD];
#pragma unroll
            for (int q = 0; q < MD; ++q) dw_old[q] = dm.w[q];
            const float vd[1] = {(float)raw};
            int dt = -1;
            if (!dinit)
                gmm_init(dm, vd, a.dk);
            else
                ld = gmm_step(dm, vd, a.dk, dt);
            dirty |= sts_mix<MD, 1, kElide>(stp, L::NFC, lane, dm, dt, dw_old);
            if (!dinit) {
                stp[L::DF + lane] = 1;
                dirty |= 1ull << L::BIT_DF;
            }
        }

        uint32_t out = out0;
        int cpt = cpt0;
        fuse_pixel(lc, ld, a.limit, out, cpt);
        stp[L::OUT + lane] = (char)out;
        stp[L::CPT + lane] = (char)cpt;
        if (!kElide || out != out0) dirty |= 1ull << L::BIT_OUT;
        if (!kElide || cpt != cpt0) dirty |= 1ull << L::BIT_CPT;
        if (a.rgb_mask) a.rgb_mask[i] = (uint8_t)lc;
        if (a.depth_mask) a.depth_mask[i] = (uint8_t)ld;
        if (a.fused_copy) a.fused_copy[i] = (uint8_t)out;

        // ---- write back the dirty plane chunks ------------------------------
        const uint32_t lo = __reduce_or_sync(0xffffffffu, (uint32_t)dirty);
        const uint32_t hi = __reduce_or_sync(0xffffffffu, (uint32_t)(dirty >> 32));
        fence_async_smem();
        __syncwarp();
        issue_stores<MC, MD>(a, c * kChunk, st, ((uint64_t)hi << 32) | lo, lane);
    }
    bulk_wait_all();
}

template <int MC, int MD>
cudaError_t bulk_md(const FusedArgs& a, bool elide, size_t nchunks, cudaStream_t s) {
    using L = Layout<MC, MD>;
    const int smem = kWarpsPerBlock * kStages * L::STAGE;
    static int blocks_per_sm[2] = {0, 0};
    static int sms = 0;
    auto kern = elide ? k_fused_bulk<MC, MD, true> : k_fused_bulk<MC, MD, false>;
    int& bps = blocks_per_sm[elide ? 1 : 0];
    if (bps == 0) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, kWarpsPerBlock * 32, smem);
        if (e != cudaSuccess) return e;
        int dev;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (bps < 1) bps = 1;
    }
    const size_t want = (nchunks + kWarpsPerBlock - 1) / kWarpsPerBlock;
    const unsigned grid = (unsigned)std::min<size_t>(want, (size_t)bps * sms);
    kern<<<grid, kWarpsPerBlock * 32, smem, s>>>(a, nchunks);
    return cudaGetLastError();
}

template <int MC>
cudaError_t bulk_mc(const FusedArgs& a, bool elide, size_t nchunks, cudaStream_t s) {
    switch (a.depth.M) {
        case 3: return bulk_md<MC, 3>(a, elide, nchunks, s);
        case 4: return bulk_md<MC, 4>(a, elide, nchunks, s);
        case 5: return bulk_md<MC, 5>(a, elide, nchunks, s);
    }
    return cudaErrorInvalidValue;
}

}  // namespace

bool bulk_eligible(const FusedArgs& a) {
    auto al = [](const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    return a.n >= kChunk && al(a.r) && al(a.g) && al(a.b) && al(a.d) && al(a.out) && al(a.cpt) &&
           al(a.color.flags + a.base) && al(a.depth.flags + a.base) &&
           al(a.color.state + a.base) && al(a.depth.state + a.base) &&
           (a.color.pitch % 4) == 0 && (a.depth.pitch % 4) == 0;
}

// Full 32-pixel chunks only; the caller handles the n % 32 tail.
cudaError_t launch_fused_bulk(const FusedArgs& a, bool elide, cudaStream_t s) {
    const size_t nchunks = a.n / kChunk;
    if (nchunks == 0) return cudaSuccess;
    switch (a.color.M) {
        case 3: return bulk_mc<3>(a, elide, nchunks, s);
        case 4: return bulk_mc<4>(a, elide, nchunks, s);
        case 5: return bulk_mc<5>(a, elide, nchunks, s);
    }
    return cudaErrorInvalidValue;
}

}  // namespace rgbdseg_b200
