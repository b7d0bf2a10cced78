// profiles/experiments/k1_ws_r02.cu -- MEASURED AND DROPPED (round 2).
// The warp-specialised K1 (flag warp F, plane-producer warps P, compute warps
// C over an mbarrier ring in shared memory), as it was spliced into
// paper_2110_14934_b200/csrc/rgbdseg_kernels.cu ahead of the near-threshold
// kernel, plus its launcher.  Bitwise-correct on the GPU parity suite (16
// tests, variant "ws"), but 2.8x slower than k_fused_ldg with one producer
// and 1.8x slower with three: see profiles/variants_r02.json for the numbers
// and the reading.  Not built; kept as the record of the experiment.
// ---------------------------------------------------------------- K1ws
// K1 as a warp-specialised, mbarrier-pipelined persistent kernel.  The
// ld-based K1 keeps a pixel's whole load chain in its own registers: round
// one (inputs, flags, speculative components), the flag-dependent round two,
// then the step -- two DRAM latencies per warp with nothing else in flight,
// so at 48 warps/SM the kernel is latency-bound (issue ~61%, DRAM ~75% of
// the 2R1W ceiling, profiles/r02).  Here the loads leave the compute warps:
//   warp F (flags)    streams every tile's flag words and depth input into
//                     a ring of LF slots, LF tiles ahead (cp.async, 4 B/lane);
//   warp P (planes)   reads a tile's flags from that ring, derives exactly the
//                     components the step will read (touched prefix of the
//                     warp + per-lane untouched masks, the elided K1's
//                     rule), and cp.asyncs those plane words, the colour
//                     input and the fusion state into a stage of an S-deep
//                     ring (an image of the bank tiles: plane p at p*128 B);
//   warps C0..C{CW-1} take stages round robin and run the unchanged step
//                     (gmm_step_fast, exact replay, List 1) from shared
//                     memory, storing straight to the bank.
// Full / empty mbarriers per slot; cp.async completion arrives through
// cp.async.mbarrier.arrive.noinc.  Memory in flight is set by the ring depth,
// not by registers, and the compute warps never wait on DRAM.  Identical
// results to k_fused_ldg<.., kElide = true> (same step code, same substitute
// values for untouched components, same store elision).
#ifndef RGBDSEG_WS_CW  // compute warps per block
#define RGBDSEG_WS_CW 7
#endif
#ifndef RGBDSEG_WS_NP  // plane-producer warps per block
#define RGBDSEG_WS_NP 2
#endif
#ifndef RGBDSEG_WS_STAGES  // plane stages per block
#define RGBDSEG_WS_STAGES 12
#endif
#ifndef RGBDSEG_WS_LF  // flag slots per block (F's lead over P in tiles)
#define RGBDSEG_WS_LF 16
#endif
#ifndef RGBDSEG_WS_MINB  // resident blocks per SM
#define RGBDSEG_WS_MINB 3
#endif
constexpr int kWsCW = RGBDSEG_WS_CW, kWsNP = RGBDSEG_WS_NP, kWsS = RGBDSEG_WS_STAGES,
              kWsLF = RGBDSEG_WS_LF;
constexpr int kWsThreads = (kWsCW + kWsNP + 1) * 32;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b))
                 : "memory");
}
// Arrives once this thread's earlier cp.async copies have landed.
__device__ __forceinline__ void mbar_arrive_cp(uint64_t* b) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(b))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n .reg .pred p;\n"
            " mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(smem_u32(b)), "r"(parity)
            : "memory");
    } while (!done);
}
// 4-byte async copy global -> shared; bytes past `valid` (0..4) are zero-filled
__device__ __forceinline__ void cp4(void* dst, const void* src, unsigned valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(valid)
                 : "memory");
}

// One flag slot: the tile's colour and depth flag words and depth input.
struct alignas(16) WsFlags {
    uint16_t cf[kBlockPx];
    uint16_t df[kBlockPx];
    uint16_t d[kBlockPx];
};

// One plane stage: bank-tile images (planes of the colour then the depth
// tile, 128 B each), the flags and depth input (copied from the flag slot),
// the colour input (3 planes or one interleaved plane, 96 B) and the fusion
// state.  Only the words the step reads are ever written.
template <int MC, int MD>
struct alignas(16) WsStage {
    float cpl[bank_planes(MC, 3)][kBlockPx];
    float dpl[bank_planes(MD, 1)][kBlockPx];
    WsFlags fl;
    uint8_t rgb[3 * kBlockPx];
    uint8_t out[kBlockPx];
    int8_t cpt[kBlockPx];
};

// load_mix_need from a stage image (plain shared-memory loads).
template <int L, int N, int C>
__device__ __forceinline__ void load_mix_stage(const float (*pl)[kBlockPx], unsigned lane,
                                               Mixture<N, C>& m, uint32_t need, float vvar) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
        const bool ld = (need >> i) & 1u;
#pragma unroll
        for (int c = 0; c < C; ++c) m.mu[i][c] = ld ? pl[i * C + c][lane] : 0.0f;
        m.var[i] = ld ? pl[L * C + i][lane] : vvar;
        m.w[i] = ld ? pl[L * C + L + i][lane] : 0.0f;
    }
}

// step_pixel_n with the mixture read from the stage and stored to the bank.
template <int M, int C, int N, bool kVirt>
__device__ __forceinline__ uint32_t step_pixel_ws(float* s, const float (*pl)[kBlockPx],
                                                  unsigned lane, uint32_t need,
                                                  const float (&v)[C], const MixCfg& k,
                                                  const BankView& bk, uint32_t& f, bool& replay) {
    Mixture<N, C> m;
    constexpr uint32_t kLoad = kVirt ? ~(1u << (N - 1)) : ~0u;
    load_mix_stage<M>(pl, lane, m, need & kLoad, bk.vvar);
    float w_old[N];
#pragma unroll
    for (int q = 0; q < N; ++q) w_old[q] = m.w[q];
    int t = 0;
    bool ok = k.fast != 0;
    const uint32_t label = gmm_step_fast<N, C, kVirt>(m, v, k, t, ok);
    if (ok) {
        store_mix_elide<M, true>(s, m, t, w_old);
        f = flag_after<M>(f, t, m.w, bk);
    } else {
        replay = true;
    }
    return label;
}

// k1_bank_pixel (elided) over a stage image.
template <int M, int C>
__device__ __forceinline__ uint32_t bank_pixel_ws(float* s, const float (*pl)[kBlockPx],
                                                  unsigned lane, uint32_t need, int Kw,
                                                  const float (&v)[C], const MixCfg& k,
                                                  const BankView& bk, uint32_t& f, bool& replay) {
    if (!(f & 0xffu)) {
        Mixture<M, C> m;
        gmm_init(m, v, k);
        store_mix<M, true>(s, m);
        f = flag_after<M>(f, -1, m.w, bk);
        return 0u;
    }
    const int N = min(Kw + 1, M);
    if (N <= 2) return step_pixel_ws<M, C, 2, true>(s, pl, lane, need, v, k, bk, f, replay);
    if constexpr (M >= 4)
        if (N == 3) return step_pixel_ws<M, C, 3, true>(s, pl, lane, need, v, k, bk, f, replay);
    if constexpr (M >= 5)
        if (N == 4) return step_pixel_ws<M, C, 4, true>(s, pl, lane, need, v, k, bk, f, replay);
    if (Kw == M - 1) return step_pixel_ws<M, C, M, true>(s, pl, lane, need, v, k, bk, f, replay);
    return step_pixel_ws<M, C, M, false>(s, pl, lane, need, v, k, bk, f, replay);
}

// Warp-max touched prefixes of a tile (fused_core's kc / kd); lanes past
// the launch end count as 1.
template <int MC, int MD>
__device__ __forceinline__ void ws_prefixes(bool act, uint32_t cf, uint32_t df, uint32_t raw,
                                            int& kc, int& kd) {
    kc = __reduce_max_sync(0xffffffffu, (act && (cf & 0xffu)) ? touched_prefix<MC>(cf) : 1);
    kd = __reduce_max_sync(0xffffffffu,
                           (act && raw != 0 && (df & 0xffu)) ? touched_prefix<MD>(df) : 1);
}

template <int MC, int MD, bool kPacked>
__global__ void __launch_bounds__(kWsThreads, RGBDSEG_WS_MINB)
    k_fused_ws(const __grid_constant__ FusedArgs a) {
    using Stage = WsStage<MC, MD>;
    extern __shared__ __align__(16) unsigned char ws_smem[];
    Stage* stages = reinterpret_cast<Stage*>(ws_smem);
    WsFlags* fring = reinterpret_cast<WsFlags*>(stages + kWsS);
    uint64_t* bars = reinterpret_cast<uint64_t*>(fring + kWsLF);
    uint64_t* full = bars;               // [kWsS]  P -> C: stage filled
    uint64_t* empty = full + kWsS;       // [kWsS]  C -> P: stage consumed
    uint64_t* ffull = empty + kWsS;      // [kWsLF] F -> P: flags landed
    uint64_t* fempty = ffull + kWsLF;    // [kWsLF] P -> F: flag slot read

    const unsigned warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kWsS; ++i) {
            mbar_init(full + i, 64);  // 32 lanes x (STS release + cp.async arrive)
            mbar_init(empty + i, 1);
        }
        for (int i = 0; i < kWsLF; ++i) {
            mbar_init(ffull + i, 32);
            mbar_init(fempty + i, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const size_t ntiles = (a.n + kBlockPx - 1) / kBlockPx;
    const size_t gstep = gridDim.x;
    const size_t tile0 = (a.base / kBlockPx);  // first bank tile of this launch
    constexpr unsigned SC = bank_stride(MC, 3), SD = bank_stride(MD, 1);

    if (warp == kWsCW + kWsNP) {
        // ---------------- F: flag words + depth input, LF tiles ahead
        uint32_t k = 0;
        for (size_t t = blockIdx.x; t < ntiles; t += gstep, ++k) {
            const uint32_t slot = k % kWsLF;
            if (k >= (uint32_t)kWsLF) mbar_wait(fempty + slot, ((k / kWsLF) & 1u) ^ 1u);
            WsFlags& fs = fring[slot];
            const char* cb = reinterpret_cast<const char*>(a.color.state + (tile0 + t) * SC);
            const char* db = reinterpret_cast<const char*>(a.depth.state + (tile0 + t) * SD);
            if (lane < 16)
                cp4(reinterpret_cast<char*>(fs.cf) + 4 * lane,
                    cb + bank_planes(MC, 3) * 128 + 4 * lane, 4);
            else
                cp4(reinterpret_cast<char*>(fs.df) + 4 * (lane - 16),
                    db + bank_planes(MD, 1) * 128 + 4 * (lane - 16), 4);
            if (lane < 16) {  // depth input, 2 px per chunk, zero past n
                const size_t p0 = t * kBlockPx + 2 * lane;
                const unsigned v = p0 >= a.n ? 0u : (a.n - p0 >= 2 ? 4u : 2u);
                cp4(reinterpret_cast<char*>(fs.d) + 4 * lane, v ? (const void*)(a.d + p0) : a.d, v);
            }
            mbar_arrive_cp(ffull + slot);
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        return;
    }

    if (warp >= kWsCW) {
        // ---------------- P_j: the planes each tile's step will read (tiles j, j + NP, ...)
        uint32_t k = warp - kWsCW;
        for (size_t t = blockIdx.x + (size_t)k * gstep; t < ntiles; t += kWsNP * gstep, k += kWsNP) {
            const uint32_t fslot = k % kWsLF, s = k % kWsS;
            mbar_wait(ffull + fslot, (k / kWsLF) & 1u);
            const WsFlags& fs = fring[fslot];
            const uint32_t cf = fs.cf[lane], df = fs.df[lane], raw = fs.d[lane];
            __syncwarp();
            if (lane == 0) mbar_arrive(fempty + fslot);
            if (k >= (uint32_t)kWsS) mbar_wait(empty + s, ((k / kWsS) & 1u) ^ 1u);
            Stage& st = stages[s];
            st.fl.cf[lane] = (uint16_t)cf;
            st.fl.df[lane] = (uint16_t)df;
            st.fl.d[lane] = (uint16_t)raw;
            const size_t i0 = t * kBlockPx;
            const bool act = i0 + lane < a.n;
            int kc, kd;
            ws_prefixes<MC, MD>(act, cf, df, raw, kc, kd);
            const int nc = min(kc + 1, MC), nd = min(kd + 1, MD);
            const uint32_t cneed = (act && (cf & 0xffu)) ? ~flag_untouched<MC>(cf) : 0u;
            const uint32_t dneed =
                (act && raw != 0 && (df & 0xffu)) ? ~flag_untouched<MD>(df) : 0u;
            const float* cb = a.color.state + (tile0 + t) * SC + lane;
            const float* db = a.depth.state + (tile0 + t) * SD + lane;
#pragma unroll
            for (int i = 0; i < MC; ++i)
                if (i < nc && ((cneed >> i) & 1u)) {
#pragma unroll
                    for (int c = 0; c < 3; ++c)
                        cp4(&st.cpl[i * 3 + c][lane], cb + (i * 3 + c) * kBlockPx, 4);
                    cp4(&st.cpl[MC * 3 + i][lane], cb + (MC * 3 + i) * kBlockPx, 4);
                    cp4(&st.cpl[MC * 4 + i][lane], cb + (MC * 4 + i) * kBlockPx, 4);
                }
#pragma unroll
            for (int i = 0; i < MD; ++i)
                if (i < nd && ((dneed >> i) & 1u)) {
                    cp4(&st.dpl[i][lane], db + i * kBlockPx, 4);
                    cp4(&st.dpl[MD + i][lane], db + (MD + i) * kBlockPx, 4);
                    cp4(&st.dpl[2 * MD + i][lane], db + (2 * MD + i) * kBlockPx, 4);
                }
            // colour input: 24 chunks of 4 B (r | g | b planes, or 96 packed
            // bytes); fusion state: lanes 24..31 (out), then 0..7 (cpt)
            if (lane < 24) {
                const unsigned q = lane % 8;
                const size_t b0 = kPacked ? 3 * i0 + 4 * lane : i0 + 4 * q;
                const size_t lim = kPacked ? 3 * a.n : a.n;
                const unsigned v = b0 >= lim ? 0u : (lim - b0 >= 4 ? 4u : (unsigned)(lim - b0));
                const uint8_t* src = kPacked ? a.r : (lane < 8 ? a.r : (lane < 16 ? a.g : a.b));
                cp4(st.rgb + (kPacked ? 4 * lane : (lane / 8) * kBlockPx + 4 * q),
                    v ? (const void*)(src + b0) : (const void*)src, v);
            } else if (a.fuse) {
                const size_t b0 = i0 + 4 * (lane - 24);
                const unsigned v = b0 >= a.n ? 0u : (a.n - b0 >= 4 ? 4u : (unsigned)(a.n - b0));
                cp4(st.out + 4 * (lane - 24), v ? (const void*)(a.out + b0) : (const void*)a.out, v);
            }
            if (a.fuse && lane < 8) {
                const size_t b0 = i0 + 4 * lane;
                const unsigned v = b0 >= a.n ? 0u : (a.n - b0 >= 4 ? 4u : (unsigned)(a.n - b0));
                cp4(st.cpt + 4 * lane, v ? (const void*)(a.cpt + b0) : (const void*)a.cpt, v);
            }
            mbar_arrive_cp(full + s);  // the copies above
            mbar_arrive(full + s);     // the flag stores above (release)
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        return;
    }

    // ---------------- C: compute warps, stages warp, warp + CW, ...
    uint32_t k = warp;
    for (size_t t = blockIdx.x + (size_t)warp * gstep; t < ntiles; t += kWsCW * gstep, k += kWsCW) {
        const uint32_t s = k % kWsS;
        mbar_wait(full + s, (k / kWsS) & 1u);
        const Stage& st = stages[s];
        const size_t i0 = t * kBlockPx;
        const bool act = i0 + lane < a.n;
        const uint32_t cf = st.fl.cf[lane], df = st.fl.df[lane], raw = st.fl.d[lane];
        int kc, kd;
        ws_prefixes<MC, MD>(act, cf, df, raw, kc, kd);
        float vc[3];
        if constexpr (kPacked) {
            const int ro = a.bgr ? 2 : 0;
            vc[0] = (float)st.rgb[3 * lane + ro];
            vc[1] = (float)st.rgb[3 * lane + 1];
            vc[2] = (float)st.rgb[3 * lane + 2 - ro];
        } else {
#pragma unroll
            for (int c = 0; c < 3; ++c) vc[c] = (float)st.rgb[c * kBlockPx + lane];
        }
        const uint32_t out0 = a.fuse ? (uint32_t)st.out[lane] : 0u;
        const int cpt0 = a.fuse ? (int)st.cpt[lane] : 0;
        if (act) {
            const PixAddr<MC, MD> p(a, i0, lane);
            // ---- depth stream (segment_depth): raw 0 = no return ----
            uint32_t ld = 0;
            if (raw != 0) {
                const float vd[1] = {(float)raw};
                uint32_t df1 = df;
                bool replay = false;
                ld = bank_pixel_ws<MD, 1>(p.ds, st.dpl, lane, ~flag_untouched<MD>(df), kd, vd,
                                          a.dk, a.depth, df1, replay);
                if (replay) ld = replay_pixel<MD, 1, true>(p.ds, vd, a.dk, a.depth, df1);
                if (df1 != df) st_h<true>(p.dflag(), (uint16_t)df1);
            }
            // ---- colour stream (segment_color) ----
            uint32_t cf1 = cf;
            bool replay = false;
            uint32_t lc = bank_pixel_ws<MC, 3>(p.cs, st.cpl, lane, ~flag_untouched<MC>(cf), kc, vc,
                                               a.ck, a.color, cf1, replay);
            if (replay) lc = replay_pixel<MC, 3, true>(p.cs, vc, a.ck, a.color, cf1);
            if (cf1 != cf) st_h<true>(p.cflag(), (uint16_t)cf1);
            // ---- List-1 fusion ----
            uint32_t out = out0;
            int cpt = cpt0;
            if (a.fuse) {
                fuse_pixel(lc, ld, a.limit, out, cpt);
                if (out != out0) a.out[i0 + lane] = (uint8_t)out;
                if (cpt != cpt0) a.cpt[i0 + lane] = (int8_t)cpt;
            }
            if (a.rgb_mask) a.rgb_mask[i0 + lane] = (uint8_t)lc;
            if (a.depth_mask) a.depth_mask[i0 + lane] = (uint8_t)ld;
            if (a.fused_copy) a.fused_copy[i0 + lane] = (uint8_t)out;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + s);
    }
}

template <int MC, int MD>
constexpr size_t ws_smem_bytes() {
    return kWsS * sizeof(WsStage<MC, MD>) + kWsLF * sizeof(WsFlags) +
           (2 * kWsS + 2 * kWsLF) * sizeof(uint64_t);
}

inline bool al4(const void* p) { return ((uintptr_t)p & 3u) == 0u; }

// K1ws on a persistent grid: resident blocks x SMs of the launching device
// (cached per device ordinal), at most one block per tile.
template <int MC, int MD>
cudaError_t fused_ws(const FusedArgs& a, cudaStream_t s) {
    constexpr size_t smem = ws_smem_bytes<MC, MD>();
    constexpr int kMaxDev = 64;
    static std::atomic<int> grid[kMaxDev][2];
    int dev = 0;
    cudaGetDevice(&dev);
    const int dslot = dev < kMaxDev ? dev : kMaxDev - 1;
    const int pk = a.packed ? 1 : 0;
    int g = grid[dslot][pk].load(std::memory_order_relaxed);
    if (g <= 0 || dev >= kMaxDev) {
        auto kern = a.packed ? k_fused_ws<MC, MD, true> : k_fused_ws<MC, MD, false>;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        int bps = 0, sms = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, kWsThreads, smem);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        g = std::max(1, bps * sms);
        grid[dslot][pk].store(g, std::memory_order_relaxed);
    }
    const size_t tiles = (a.n + kBlockPx - 1) / kBlockPx;
    const unsigned nb = (unsigned)std::min<size_t>((size_t)g, tiles);
    if (a.packed)
        k_fused_ws<MC, MD, true><<<nb, kWsThreads, smem, s>>>(a);
    else
        k_fused_ws<MC, MD, false><<<nb, kWsThreads, smem, s>>>(a);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
}

