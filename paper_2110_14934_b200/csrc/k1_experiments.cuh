// k1_experiments.cuh -- round-2 K1 variants that were measured and DROPPED
// (profiles/variants_r02.json).  Not part of the product build: included by
// rgbdseg_kernels.cu only when an A/B build defines RGBDSEG_PX=2 or
// RGBDSEG_PIPE=1 (profiles/build_variant.sh), so the measurements can be
// reproduced from source.
#pragma once

// ---------------------------------------------------------------- K1, 2 px/thread
// k_fused_x2: the same per-pixel algorithm as k_fused_ldg (elided, plain:
// no evaluation epilogue, planar colour), two pixels per thread.  Warp w of a
// block owns the tile pair (2w, 2w+1) of the block's 8 tiles; lane l runs
// pixel l of both tiles (A, and B = A + 32), so every address of B is an
// immediate offset from A's (one bank tile stride, or +32 bytes of a flat
// plane) and the address, flag, dispatch and epilogue logic is paid once per
// two pixels.  The two pixels' steps run in one basic block per touched-
// prefix specialisation (N = max over the 64 pixels' prefixes + 1), with
// both second-round loads issued before either step, so the thread carries
// two independent dependency chains.  Pixels without a step (depth no-
// return, uninitialised, beyond n) run the arithmetic on substitute values
// and store nothing; init_mixture and the exact replay run after the fast
// steps in ONE inlined copy per bank, selecting pixel A or B.
#ifndef RGBDSEG_X2_MINB  // resident 128-thread blocks of k_fused_x2
#define RGBDSEG_X2_MINB 8
#endif

template <int M, int C, int N, int P, bool kVirt>
__device__ __forceinline__ void step2_n(float* s, const Mixture<(P > 0 ? P : 1), C> (&pre)[2],
                                        const uint32_t (&need)[2], const float (&v)[2][C],
                                        const MixCfg& k, const BankView& bk, uint32_t (&f)[2],
                                        const bool (&go)[2], uint32_t (&lab)[2],
                                        bool (&replay)[2]) {
    constexpr int S = bank_stride(M, C);
    constexpr uint32_t kLoad = ~((1u << P) - 1u) & (kVirt ? ~(1u << (N - 1)) : ~0u);
    Mixture<N, C> m[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        load_mix_need<M, true>(s + q * S, m[q], go[q] ? (need[q] & kLoad) : 0u, bk.vvar);
#pragma unroll
        for (int i = 0; i < (P < N ? P : N); ++i) {
#pragma unroll
            for (int c = 0; c < C; ++c) m[q].mu[i][c] = pre[q].mu[i][c];
            m[q].var[i] = pre[q].var[i];
            m[q].w[i] = pre[q].w[i];
        }
    }
    float w_old[2][N];
    int t[2];
    bool ok[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
#pragma unroll
        for (int i = 0; i < N; ++i) w_old[q][i] = m[q].w[i];
        t[q] = 0;
        ok[q] = k.fast != 0;
        float mo[C], vo;
        lab[q] = gmm_step_fast<N, C, kVirt>(m[q], v[q], k, t[q], ok[q], mo, vo);
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        if (go[q]) {
            if (ok[q]) {
                store_mix_elide<M, true>(s + q * S, m[q], t[q], w_old[q]);
                f[q] = flag_after<M>(f[q], t[q], m[q].w, bk);
            } else {
                replay[q] = true;  // nothing stored: replayed from memory below
            }
        }
    }
}

// One bank of both pixels: the touched-prefix dispatch (Kw is the warp's
// maximum over its 64 pixels), then init_mixture and the exact replay for
// the pixels that need them, one inlined copy each.  lab[q] is only
// meaningful where go[q] or init[q].
template <int M, int C, int P>
__device__ __forceinline__ void bank2(float* s, const Mixture<(P > 0 ? P : 1), C> (&pre)[2],
                                      const uint32_t (&need)[2], int Kw, const float (&v)[2][C],
                                      const MixCfg& k, const BankView& bk, uint32_t (&f)[2],
                                      const bool (&go)[2], const bool (&init)[2],
                                      uint32_t (&lab)[2]) {
    constexpr int S = bank_stride(M, C);
    bool rep[2] = {false, false};
    if (__any_sync(0xffffffffu, go[0] || go[1])) {
        const int N = min(Kw + 1, M);
        if (N <= 2) {
            step2_n<M, C, 2, P, true>(s, pre, need, v, k, bk, f, go, lab, rep);
        } else if (M >= 4 && N == 3) {
            step2_n<M, C, (M >= 4 ? 3 : 2), P, true>(s, pre, need, v, k, bk, f, go, lab, rep);
        } else if (M >= 5 && N == 4) {
            step2_n<M, C, (M >= 5 ? 4 : 2), P, true>(s, pre, need, v, k, bk, f, go, lab, rep);
        } else if (Kw == M - 1) {
            step2_n<M, C, M, P, true>(s, pre, need, v, k, bk, f, go, lab, rep);
        } else {
            step2_n<M, C, M, P, false>(s, pre, need, v, k, bk, f, go, lab, rep);
        }
    }
    // Rare paths, one copy each: pixel B when A has nothing to do.
    bool ini[2] = {init[0], init[1]};
    while (ini[0] || ini[1]) {
        const bool qb = !ini[0];
        Mixture<M, C> m;
        float vq[C];
#pragma unroll
        for (int c = 0; c < C; ++c) vq[c] = qb ? v[1][c] : v[0][c];
        gmm_init(m, vq, k);
        store_mix<M, true>(s + (qb ? S : 0), m);
        const uint32_t fq = flag_after<M>(qb ? f[1] : f[0], -1, m.w, bk);
        if (qb) {
            f[1] = fq;
            lab[1] = 0u;
            ini[1] = false;
        } else {
            f[0] = fq;
            lab[0] = 0u;
            ini[0] = false;
        }
    }
    while (rep[0] || rep[1]) {
        const bool qb = !rep[0];
        float vq[C];
#pragma unroll
        for (int c = 0; c < C; ++c) vq[c] = qb ? v[1][c] : v[0][c];
        uint32_t fq = qb ? f[1] : f[0];
        const uint32_t l = replay_pixel<M, C, true>(s + (qb ? S : 0), vq, k, bk, fq);
        if (qb) {
            f[1] = fq;
            lab[1] = l;
            rep[1] = false;
        } else {
            f[0] = fq;
            lab[0] = l;
            rep[0] = false;
        }
    }
}

template <int MC, int MD>
__global__ void __launch_bounds__(kThreads, RGBDSEG_X2_MINB)
    k_fused_x2(const __grid_constant__ FusedArgs a) {
    constexpr int SC = bank_stride(MC, 3), SD = bank_stride(MD, 1);
    const unsigned w = threadIdx.x / kBlockPx, lane = threadIdx.x % kBlockPx;
    const size_t i0 = (size_t)blockIdx.x * (2 * kThreads) + w * (2 * kBlockPx);
    const size_t iA = i0 + lane;  // pixel B = iA + 32
    const bool act[2] = {iA < a.n, iA + kBlockPx < a.n};
    const size_t tile0 = (a.base + i0) / kBlockPx;
    float* cs = a.color.state + tile0 * SC + lane;
    float* ds = a.depth.state + tile0 * SD + lane;
    uint16_t* cfl = reinterpret_cast<uint16_t*>(reinterpret_cast<char*>(cs) +
                                                bank_planes(MC, 3) * 128 - 2 * lane);
    uint16_t* dfl = reinterpret_cast<uint16_t*>(reinterpret_cast<char*>(ds) +
                                                bank_planes(MD, 1) * 128 - 2 * lane);

    // ---- first load round of both pixels ----
    float vc[2][3];
    uint32_t raw[2], cf[2], df[2];
    Mixture<kPre, 3> cpre[2];
    Mixture<1, 1> dpre[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const size_t o = iA + q * kBlockPx;
        if (act[q]) {
            vc[q][0] = (float)ld_h<true>(a.r + o);
            vc[q][1] = (float)ld_h<true>(a.g + o);
            vc[q][2] = (float)ld_h<true>(a.b + o);
            raw[q] = ld_h<true>(a.d + o);
            cf[q] = ld_h<true>(cfl + q * SC * 2);
            df[q] = ld_h<true>(dfl + q * SD * 2);
            if (a.fuse) {
                asm volatile("prefetch.global.L1 [%0];" ::"l"(a.out + o));
                asm volatile("prefetch.global.L1 [%0];" ::"l"(a.cpt + o));
            }
            load_mix<MC, true>(cs + q * SC, cpre[q]);
            load_mix<MD, true>(ds + q * SD, dpre[q]);
        } else {
            vc[q][0] = vc[q][1] = vc[q][2] = 0.0f;
            raw[q] = cf[q] = df[q] = 0u;
            cpre[q] = Mixture<kPre, 3>{};
            dpre[q] = Mixture<1, 1>{};
        }
    }
    int kcl = 1, kdl = 1;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        if (cf[q] & 0xffu) kcl = max(kcl, touched_prefix<MC>(cf[q]));
        if (raw[q] != 0 && (df[q] & 0xffu)) kdl = max(kdl, touched_prefix<MD>(df[q]));
    }
    const int kc = __reduce_max_sync(0xffffffffu, kcl);
    const int kd = __reduce_max_sync(0xffffffffu, kdl);

    // ---- depth stream (segment_depth): raw 0 = no return ----
    uint32_t ld[2];
    {
        const uint32_t need[2] = {~flag_untouched<MD>(df[0]), ~flag_untouched<MD>(df[1])};
        const float vd[2][1] = {{(float)raw[0]}, {(float)raw[1]}};
        bool go[2], ini[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            go[q] = raw[q] != 0 && (df[q] & 0xffu);  // raw != 0 implies act
            ini[q] = raw[q] != 0 && !(df[q] & 0xffu);
        }
        uint32_t f1[2] = {df[0], df[1]};
        uint32_t lab[2] = {0u, 0u};
        bank2<MD, 1, 1>(ds, dpre, need, kd, vd, a.dk, a.depth, f1, go, ini, lab);
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            ld[q] = (go[q] || ini[q]) ? lab[q] : 0u;
            if (f1[q] != df[q]) st_h<true>(dfl + q * SD * 2, (uint16_t)f1[q]);
        }
    }
    // ---- colour stream (segment_color) ----
    uint32_t lc[2];
    {
        const uint32_t need[2] = {~flag_untouched<MC>(cf[0]), ~flag_untouched<MC>(cf[1])};
        bool go[2], ini[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            go[q] = act[q] && (cf[q] & 0xffu);
            ini[q] = act[q] && !(cf[q] & 0xffu);
        }
        uint32_t f1[2] = {cf[0], cf[1]};
        uint32_t lab[2] = {0u, 0u};
        bank2<MC, 3, kPre>(cs, cpre, need, kc, vc, a.ck, a.color, f1, go, ini, lab);
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            lc[q] = (go[q] || ini[q]) ? lab[q] : 0u;
            if (f1[q] != cf[q]) st_h<true>(cfl + q * SC * 2, (uint16_t)f1[q]);
        }
    }
    // ---- List-1 fusion on the registered depth mask ----
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        if (!act[q]) continue;
        const size_t o = iA + q * kBlockPx;
        uint32_t out = 0u;
        if (a.fuse) {
            const uint32_t out0 = a.out[o];  // L1 hits (prefetched in round one)
            const int cpt0 = (int)a.cpt[o];
            out = out0;
            int cpt = cpt0;
            fuse_pixel(lc[q], ld[q], a.limit, out, cpt);
            if (out != out0) st_h<true>(a.out + o, (uint8_t)out);
            if (cpt != cpt0) st_h<true>(a.cpt + o, (int8_t)cpt);
        }
        if (a.rgb_mask) st_h<true>(a.rgb_mask + o, (uint8_t)lc[q]);
        if (a.depth_mask) st_h<true>(a.depth_mask + o, (uint8_t)ld[q]);
        if (a.fused_copy) st_h<true>(a.fused_copy + o, (uint8_t)out);
    }
}

// ---------------------------------------------------------------- K1, pipelined
// k_fused_pipe: k_fused_ldg's per-pixel work (elided, plain) in a persistent
// warp loop with the NEXT tile's first load round issued into registers
// before the current tile's steps.  ncu on the one-shot K1 (frame 100 of the
// default workload: 61% issue, 1.78 eligible warps per scheduler, 5.26 TB/s)
// shows a latency-bound kernel: a warp spends ~40% of its life waiting for
// its first round.  Here that wait overlaps the previous tile's arithmetic,
// at the cost of ~19 registers holding the next round (no extra instructions,
// unlike the L1/L2 prefetch and shared-memory staging variants of round 1).
// Warp g of the grid runs tiles g, g + G, g + 2G, ... (G = warps in the
// grid, sized to one occupancy wave).  Colour inputs stay integers until the
// step (a conversion right after the load would stall on it).
#ifndef RGBDSEG_PIPE_MINB  // resident 128-thread blocks of k_fused_pipe
#define RGBDSEG_PIPE_MINB 8
#endif
struct Round1Raw {
    uint32_t rgb[3], raw, cf, df;
    Mixture<kPre, 3> cpre;
    Mixture<1, 1> dpre;
};

template <int MC, int MD>
__device__ __forceinline__ void load_round1(const FusedArgs& a, size_t i0, unsigned lane,
                                            Round1Raw& r) {
    const PixAddr<MC, MD> p(a, i0, lane);
    const size_t o = i0 + lane;
    r.rgb[0] = ld_h<true>(a.r + o);
    r.rgb[1] = ld_h<true>(a.g + o);
    r.rgb[2] = ld_h<true>(a.b + o);
    r.raw = ld_h<true>(a.d + o);
    r.cf = ld_h<true>(p.cflag());
    r.df = ld_h<true>(p.dflag());
    if (a.fuse) {
        asm volatile("prefetch.global.L1 [%0];" ::"l"(a.out + o));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(a.cpt + o));
    }
    load_mix<MC, true>(p.cs, r.cpre);
    load_mix<MD, true>(p.ds, r.dpre);
}

template <int MC, int MD>
__global__ void __launch_bounds__(kThreads, RGBDSEG_PIPE_MINB)
    k_fused_pipe(const __grid_constant__ FusedArgs a) {
    constexpr unsigned kWarps = kThreads / kBlockPx;
    const unsigned lane = threadIdx.x % kBlockPx;
    const size_t nt = (a.n + kBlockPx - 1) / kBlockPx;
    const size_t G = (size_t)gridDim.x * kWarps;
    size_t t = (size_t)blockIdx.x * kWarps + threadIdx.x / kBlockPx;
    if (t >= nt) return;
    Round1Raw cur;
    bool act = t * kBlockPx + lane < a.n;
    if (act) load_round1<MC, MD>(a, t * kBlockPx, lane, cur);
    for (; t < nt; t += G) {
        const size_t tn = t + G;
        const bool actn = tn < nt && tn * kBlockPx + lane < a.n;
        Round1Raw nxt;
        if (actn) load_round1<MC, MD>(a, tn * kBlockPx, lane, nxt);
        if (act) {
            Round1 r;
#pragma unroll
            for (int c = 0; c < 3; ++c) r.vc[c] = (float)cur.rgb[c];
            r.raw = cur.raw;
            r.cf = cur.cf;
            r.df = cur.df;
            r.cpre = cur.cpre;
            r.dpre = cur.dpre;
            const PixAddr<MC, MD> p(a, t * kBlockPx, lane);
            uint32_t lab[3];
            fused_core<MC, MD, true>(a, t * kBlockPx, lane, p, r, lab);
        }
        cur = nxt;
        act = actn;
    }
}


// Grid of k_fused_pipe: one occupancy wave of the launching device (cached
// per device ordinal), never more warps than tiles.
template <int MC, int MD>
unsigned pipe_blocks(size_t n) {
    constexpr int kMaxDev = 64;
    static std::atomic<int> cache[kMaxDev];
    int dev = 0;
    cudaGetDevice(&dev);
    int wave = dev < kMaxDev ? cache[dev].load(std::memory_order_relaxed) : 0;
    if (wave <= 0) {
        int bps = 0, sms = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_fused_pipe<MC, MD>, kThreads, 0);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        wave = max(1, bps * sms);
        if (dev < kMaxDev) cache[dev].store(wave, std::memory_order_relaxed);
    }
    const size_t need = (n + kThreads - 1) / kThreads;  // blocks of one tile per warp
    return (unsigned)(need < (size_t)wave ? need : (size_t)wave);
}

