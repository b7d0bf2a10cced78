// rgbdseg_kernels.cu -- sm_100a kernels for the RGB-D GMM hot path.
//
// K1  k_fused_*      colour GMM + depth GMM + List-1 fusion in ONE pass per
//                    pixel (SequenceProcessor::process, processor.cpp:158-184
//                    -> segment_color/segment_depth segmenter.cpp:107-131 ->
//                    run_bank :70-99 -> step_pixel mixture.cpp:148-154 ->
//                    fuse_step fusion.cpp:17-46).  Masks stay in registers.
// K1b k_bank_*       one bank alone (segment_color / segment_depth /
//                    segment_augmented drop-ins), on K1's machinery.
// K1c k_fuse16/_fuse fuse_step alone.
// K2  k_register_splat16, k_dilate_rows16/cols16 (+ per-pixel fallbacks)
//                    register_mask + dilate_mask (registration.cpp:33-78).
// K4  k_confusion    confusion_counts (eval.cpp:11-31); K1 has it fused.
// K0  k_mix_*        the per-pixel API (init_mixture / step_pixel) batched.
// K3  k_render       synthetic scene generator (synthetic.cpp:119-195).
//
// Elementwise work over HBM-resident state: one thread per pixel, the
// mixture in registers for the whole update, a tiled structure-of-arrays
// bank so every plane access of a warp is one coalesced 128-byte line, and
// a per-pixel mask of untouched components so most of the state is never
// read (rgbdseg_kernels.cuh).  Built with -fmad=false -prec-div=true
// -prec-sqrt=true -ftz=false and the arithmetic spelled with explicit _rn
// intrinsics (gmm_pixel.cuh).
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstdio>

#include "rgbdseg_kernels.cuh"

namespace rgbdseg_b200 {

namespace {
std::atomic<uint64_t> g_launches{0};

#ifndef RGBDSEG_THREADS  // 128 measured best for K1 (64..512 tried, variants_r01.json)
#define RGBDSEG_THREADS 128
#endif
constexpr int kThreads = RGBDSEG_THREADS;

inline unsigned blocks_for(size_t n) {
    return static_cast<unsigned>((n + kThreads - 1) / kThreads);
}

// Loads/stores of the hot path.  H = false: streaming (evict-first) hints,
// every word is touched once per frame -- the dense K1 and the single-bank
// kernels.  H = true (elided K1): loads cached in L2 only (ld.global.cg), so
// L1 holds the kernel's register spills, and default write-back stores;
// measured 6% faster for the elided K1 and 5% slower for the dense one
// (profiles/variants_r01.json).
template <bool H, typename T>
__device__ __forceinline__ T ld_h(const T* p) {
    if constexpr (H)
        return __ldcg(p);
    else
        return __ldcs(p);
}
template <bool H, typename T>
__device__ __forceinline__ void st_h(T* p, T v) {
    if constexpr (H)
        *p = v;
    else
        __stcs(p, v);
}
template <typename T>
__device__ __forceinline__ T ld_stream(const T* p) {
    return __ldcs(p);
}
template <typename T>
__device__ __forceinline__ void st_stream(T* p, T v) {
    __stcs(p, v);
}

// Per-thread base of pixel j in a tiled bank; plane p is at +p*32 floats.
template <int M, int C>
__device__ __forceinline__ float* px_base(const BankView& bk, size_t j) {
    return bk.state + (j / kBlockPx) * bank_stride(M, C) + (j % kBlockPx);
}
// Flag word of pixel j: initialised byte | untouched mask << 8.
template <int M, int C>
__device__ __forceinline__ uint16_t* px_flag(const BankView& bk, size_t j) {
    return reinterpret_cast<uint16_t*>(bk.state + (j / kBlockPx) * bank_stride(M, C) +
                                       bank_planes(M, C) * kBlockPx) +
           (j % kBlockPx);
}

// Untouched mask of a loaded flag word (none before initialisation).
template <int M>
__device__ __forceinline__ uint32_t flag_untouched(uint32_t f) {
    return (f & 0xffu) ? (f >> 8) & untouched_all(M) : 0u;
}

// K of a pixel whose components K..M-1 are untouched and 0..K-1 may not be
// (the mask is a suffix: a step replaces the weakest component, and every
// untouched one has fitness +0 and the highest indices, so the first
// untouched one goes first).  M when the mask is empty or not a suffix.
template <int M>
__device__ __forceinline__ int touched_prefix(uint32_t f) {
    const uint32_t u = flag_untouched<M>(f);
    const int K = M - __popc(u);  // a suffix of |u| bits starts at K
    return u == (1u << M) - (1u << K) ? K : M;
}

// Flag word after a step on components 0..N-1 (N..M-1 untouched, unchanged).
// init_mixture (touched < 0) leaves components 1..M-1 at their init values;
// a step rewrites the touched component, and a weight that is no longer +0
// (normalisation overflow) also ends "untouched".
template <int M, int N>
__device__ __forceinline__ uint32_t flag_after(uint32_t f, int touched, const float (&w)[N],
                                               const BankView& bk) {
    if (touched < 0) return 1u | (bk.vinit ? untouched_all(M) << 8 : 0u);
    uint32_t keep = 0xffffu;
#pragma unroll
    for (int i = 1; i < N; ++i)
        if (i == touched || __float_as_uint(w[i]) != 0u) keep &= ~(1u << (8 + i));
    return f & keep;
}

// Mixture I/O on a bank of layout L components: components 0..N-1 of the
// pixel at `s` (N <= L).
template <int L, bool H = false, int N, int C>
__device__ __forceinline__ void load_mix(const float* s, Mixture<N, C>& m) {
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int c = 0; c < C; ++c) m.mu[i][c] = ld_h<H>(s + (i * C + c) * kBlockPx);
#pragma unroll
    for (int i = 0; i < N; ++i) m.var[i] = ld_h<H>(s + (L * C + i) * kBlockPx);
#pragma unroll
    for (int i = 0; i < N; ++i) m.w[i] = ld_h<H>(s + (L * C + L + i) * kBlockPx);
}

// load_mix for the components whose bit is set in `need`; the others are
// untouched (flag word) and take their known values without a memory access.
template <int L, bool H = false, int N, int C>
__device__ __forceinline__ void load_mix_need(const float* s, Mixture<N, C>& m, uint32_t need,
                                              float vvar) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
        const bool ld = (need >> i) & 1u;
#pragma unroll
        for (int c = 0; c < C; ++c) m.mu[i][c] = ld ? ld_h<H>(s + (i * C + c) * kBlockPx) : 0.0f;
        m.var[i] = ld ? ld_h<H>(s + (L * C + i) * kBlockPx) : vvar;
        m.w[i] = ld ? ld_h<H>(s + (L * C + L + i) * kBlockPx) : 0.0f;
    }
}

// load_mix_need with plain (L1-allocating) loads: the lines were prefetched
// into L1 earlier (fused_core's flag-aware colour prefetch).
template <int L, int N, int C>
__device__ __forceinline__ void load_mix_need_l1(const float* s, Mixture<N, C>& m, uint32_t need,
                                                 float vvar) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
        const bool ld = (need >> i) & 1u;
#pragma unroll
        for (int c = 0; c < C; ++c) m.mu[i][c] = ld ? s[(i * C + c) * kBlockPx] : 0.0f;
        m.var[i] = ld ? s[(L * C + i) * kBlockPx] : vvar;
        m.w[i] = ld ? s[(L * C + L + i) * kBlockPx] : 0.0f;
    }
}

// Dense store (ModelBank::scatter, segmenter.cpp:49-56).
template <int L, bool H = false, int N, int C>
__device__ __forceinline__ void store_mix(float* s, const Mixture<N, C>& m) {
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int c = 0; c < C; ++c) st_h<H>(s + (i * C + c) * kBlockPx, m.mu[i][c]);
#pragma unroll
    for (int i = 0; i < N; ++i) st_h<H>(s + (L * C + i) * kBlockPx, m.var[i]);
#pragma unroll
    for (int i = 0; i < N; ++i) st_h<H>(s + (L * C + L + i) * kBlockPx, m.w[i]);
}

// Elided store: identical memory image to store_mix, but words whose bits
// did not change are not rewritten.  Only the matched / replaced component's
// mean and variance can change in a step (mixture.cpp:105-113, 125-128); the
// weights are compared individually.
template <int L, bool H = false, int N, int C>
__device__ __forceinline__ void store_mix_elide(float* s, const Mixture<N, C>& m, int touched,
                                                const float (&w_old)[N]) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
        if (touched == i) {
#pragma unroll
            for (int c = 0; c < C; ++c) st_h<H>(s + (i * C + c) * kBlockPx, m.mu[i][c]);
            st_h<H>(s + (L * C + i) * kBlockPx, m.var[i]);
        }
    }
#pragma unroll
    for (int i = 0; i < N; ++i)
        if (__float_as_uint(m.w[i]) != __float_as_uint(w_old[i]))
            st_h<H>(s + (L * C + L + i) * kBlockPx, m.w[i]);
}

// store_mix_elide without the old weights: every real component's weight is
// stored; the untouched last component (kVirt) only when it stops being +0.
#ifndef RGBDSEG_DIRECT_ST  // 1: touched mean/variance stored at a computed address
#define RGBDSEG_DIRECT_ST 1  // spills 752 -> 332 B, VGA +8%, late +0.6% (variants_r02.json)
#endif
#ifndef RGBDSEG_WSTORE_ALL
#define RGBDSEG_WSTORE_ALL 1  // +0.6% mid-sequence, +3% late (variants_r02.json)
#endif
template <int L, bool H, bool kVirt, int N, int C>
__device__ __forceinline__ void store_mix_elide_wall(float* s, const Mixture<N, C>& m,
                                                     int touched) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
        if (touched == i) {
#pragma unroll
            for (int c = 0; c < C; ++c) st_h<H>(s + (i * C + c) * kBlockPx, m.mu[i][c]);
            st_h<H>(s + (L * C + i) * kBlockPx, m.var[i]);
        }
    }
#pragma unroll
    for (int i = 0; i < N; ++i)
        if (!(kVirt && i == N - 1) || __float_as_uint(m.w[i]) != 0u)
            st_h<H>(s + (L * C + L + i) * kBlockPx, m.w[i]);
}

// Exact replay of a pixel the fast step refused: the whole mixture from
// memory (nothing was stored) through the generic gmm_step.  K1 runs it once
// per bank after both fast steps, so there is one inlined copy per bank
// shape instead of one per N specialisation, and no call boundary.
template <int M, int C, bool kElide>
__device__ __forceinline__ uint32_t replay_pixel(float* s, const float (&v)[C], const MixCfg& k,
                                                 const BankView& bk, uint32_t& f) {
    Mixture<M, C> mm;
    load_mix<M, kElide>(s, mm);
    float wo[M];
#pragma unroll
    for (int q = 0; q < M; ++q) wo[q] = mm.w[q];
    int t = 0;
    const uint32_t label = gmm_step(mm, v, k, t);
    if (kElide)
        store_mix_elide<M, kElide>(s, mm, t, wo);
    else
        store_mix<M, kElide>(s, mm);
    f = flag_after<M>(f, t, mm.w, bk);
    return label;
}

template <int M, int C, int N, int P, bool kElide, bool kVirt, bool kL1 = false>
__device__ __forceinline__ uint32_t step_pixel_n(float* s, const Mixture<(P > 0 ? P : 1), C>& pre,
                                                 uint32_t need, const float (&v)[C],
                                                 const MixCfg& k, const BankView& bk,
                                                 uint32_t& f, bool& replay) {
    Mixture<N, C> m;
    // components P.. that are touched; with kVirt, N-1 is untouched in every
    // lane (a compile-time zero bit: no load, constant values)
    constexpr uint32_t kLoad = ~((1u << P) - 1u) & (kVirt ? ~(1u << (N - 1)) : ~0u);
    if constexpr (kL1)
        load_mix_need_l1<M>(s, m, need & kLoad, bk.vvar);
    else
        load_mix_need<M, kElide>(s, m, need & kLoad, bk.vvar);
#pragma unroll
    for (int i = 0; i < (P < N ? P : N); ++i) {  // loaded with the flags (exact values)
#pragma unroll
        for (int c = 0; c < C; ++c) m.mu[i][c] = pre.mu[i][c];
        m.var[i] = pre.var[i];
        m.w[i] = pre.w[i];
    }
    // RGBDSEG_WSTORE_ALL: with two or more real components the renormalised
    // weights change on (almost) every step, so their old bits are not kept
    // live to elide the store; the untouched last component still compares
    // with its known +0.
    constexpr bool kWAll = RGBDSEG_WSTORE_ALL && kElide && (kVirt ? N - 1 : N) >= 2;
    // RGBDSEG_DIRECT_ST: the touched component's new mean/variance are
    // stored at its index (computed address) instead of written back into
    // the mixture and stored by N predicated groups.
    constexpr bool kDirect = RGBDSEG_DIRECT_ST && kElide;
    float w_old[N];
#pragma unroll
    for (int q = 0; q < N; ++q) w_old[q] = kWAll ? 0.0f : m.w[q];
    int t = 0;
    bool ok = k.fast != 0;
    float mu_o[C], var_o;
    const uint32_t label = gmm_step_fast<N, C, kVirt, kDirect>(m, v, k, t, ok, mu_o, var_o);
    if (ok) {
        if (kDirect) {
            float* pm = s + t * (C * kBlockPx);
#pragma unroll
            for (int c = 0; c < C; ++c) st_h<kElide>(pm + c * kBlockPx, mu_o[c]);
            st_h<kElide>(s + (M * C + t) * kBlockPx, var_o);
#pragma unroll
            for (int i = 0; i < N; ++i)
                if (kWAll ? (!(kVirt && i == N - 1) || __float_as_uint(m.w[i]) != 0u)
                          : __float_as_uint(m.w[i]) != __float_as_uint(w_old[i]))
                    st_h<kElide>(s + (M * C + M + i) * kBlockPx, m.w[i]);
        } else if (kWAll) {
            store_mix_elide_wall<M, kElide, kVirt>(s, m, t);
        } else if (kElide)
            store_mix_elide<M, kElide>(s, m, t, w_old);
        else
            store_mix<M, kElide>(s, m);
        f = flag_after<M>(f, t, m.w, bk);
    } else {
        replay = true;  // nothing stored: the caller replays from memory
    }
    return label;
}

// One K1 bank pixel: init_mixture, or the step on N = min(Kw + 1, M)
// components where Kw is the warp's largest touched prefix (warp-uniform, so
// a warp runs one specialisation; the dense variant always takes N = M).
// Components 0..P-1 arrive in `pre`, loaded before the flags were known.
template <int M, int C, int P, bool kElide, bool kL1 = false>
__device__ __forceinline__ uint32_t k1_bank_pixel(float* s, const Mixture<(P > 0 ? P : 1), C>& pre,
                                                  uint32_t need, int Kw, const float (&v)[C],
                                                  const MixCfg& k, const BankView& bk,
                                                  uint32_t& f, bool& replay) {
    if (!(f & 0xffu)) {
        Mixture<M, C> m;
        gmm_init(m, v, k);
        store_mix<M, kElide>(s, m);
        f = flag_after<M>(f, -1, m.w, bk);
        return 0u;
    }
    // Component N-1 is untouched in every lane whenever Kw < M (kVirt).
    if (!kElide) return step_pixel_n<M, C, M, P, false, false>(s, pre, need, v, k, bk, f, replay);
    const int N = min(Kw + 1, M);
    if (N <= 2) return step_pixel_n<M, C, 2, P, true, true, kL1>(s, pre, need, v, k, bk, f, replay);
    if constexpr (M >= 4)
        if (N == 3) return step_pixel_n<M, C, 3, P, true, true, kL1>(s, pre, need, v, k, bk, f, replay);
    if constexpr (M >= 5)
        if (N == 4) return step_pixel_n<M, C, 4, P, true, true, kL1>(s, pre, need, v, k, bk, f, replay);
    if (Kw == M - 1) return step_pixel_n<M, C, M, P, true, true, kL1>(s, pre, need, v, k, bk, f, replay);
    return step_pixel_n<M, C, M, P, true, false, kL1>(s, pre, need, v, k, bk, f, replay);
}

// ---------------------------------------------------------------- evaluation
// Per-stream confusion counts of up to 3 methods (eval.cpp:11-31) without
// shared memory or block barriers: a warp whose pixels lie in one stream
// turns two ballots per method into TP / FP / FN and lanes 0..3*NM-1 each add
// one nonzero counter (most warps: none); a warp straddling two streams adds
// per pixel.  TN is not counted here: eval.cpp:17-28 assigns every pixel
// exactly one class, so k_counts_tn sets TN = pixels - TP - FP - FN once the
// frame's launches are done.
template <int NM>
__device__ __forceinline__ void eval_accumulate(bool active, size_t j, size_t stream_px,
                                                const uint32_t (&pred)[NM], uint32_t gt,
                                                unsigned long long* counts) {
    const unsigned lane = threadIdx.x & 31;
    const size_t s = active ? j / stream_px : ~size_t(0);
    const unsigned act = __ballot_sync(0xffffffffu, active);
    if (!act) return;
    const size_t s0 = __shfl_sync(0xffffffffu, s, __ffs(act) - 1);
    const bool uniform = __all_sync(0xffffffffu, !active || s == s0);
    if (uniform) {
        const unsigned g1 = __ballot_sync(0xffffffffu, active && gt);
        // lane 3m+k (k: 0 TP, 1 FP, 2 FN) counts method m's class k
        const int m = (int)lane / 3, k = (int)lane - 3 * m;
        unsigned pm = 0u;
#pragma unroll
        for (int q = 0; q < NM; ++q) {
            const unsigned p1 = __ballot_sync(0xffffffffu, active && pred[q]);
            if (q == m) pm = p1;
        }
        const unsigned sel = k == 0 ? (pm & g1) : (k == 1 ? (pm & ~g1) : (~pm & g1));
        const unsigned v = __popc(sel);
        if (m < NM && v)
            atomicAdd(counts + (s0 * NM + m) * 4 + (k == 2 ? 3 : k), (unsigned long long)v);
    } else if (active) {  // warp across a stream boundary: per-pixel atomics
#pragma unroll
        for (int m = 0; m < NM; ++m) {
            const int k = pred[m] ? (gt ? 0 : 1) : (gt ? 3 : 2);
            if (k != 2) atomicAdd(counts + (s * NM + m) * 4 + k, 1ull);
        }
    }
}

// TN of every (stream, method) counter: the pixels not counted as TP/FP/FN.
__global__ void k_counts_tn(unsigned long long* counts, int n, unsigned long long stream_px) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    unsigned long long* c = counts + (size_t)i * 4;
    c[2] = stream_px - c[0] - c[1] - c[3];
}

__global__ void __launch_bounds__(kThreads)
    k_confusion(const uint8_t* __restrict__ p0, const uint8_t* __restrict__ p1,
                const uint8_t* __restrict__ p2, int methods, const uint8_t* __restrict__ gt,
                size_t n, size_t stream_px, unsigned long long* counts) {
    const size_t j = (size_t)blockIdx.x * kThreads + threadIdx.x;
    const bool active = j < n;
    const uint32_t g = active ? gt[j] : 0u;
    if (methods == 1) {
        const uint32_t pr[1] = {active ? p0[j] : 0u};
        eval_accumulate<1>(active, j, stream_px, pr, g, counts);
    } else {
        const uint32_t pr[3] = {active ? p0[j] : 0u, active ? p1[j] : 0u, active ? p2[j] : 0u};
        eval_accumulate<3>(active, j, stream_px, pr, g, counts);
    }
}

// ---------------------------------------------------------------- K1 fused
// Resident 128-thread blocks per SM: the dense variant is HBM-bound at 6
// (72 regs, 24 warps/SM); the elided one is latency-bound and gains from 12
// (40 regs, 48 warps/SM) despite spills (profiles/variants_r0{1,2}.json).
// Launches of at least this many occupancy waves run K1's kL1 form: colour
// components 0..kPre-1 prefetched by one warp instruction in round one
// (prefetch.global.L1; ncu shows the lines are served from L2 by the time
// they are read) and read at the colour step, instead of held in registers
// through the depth step.  With fewer registers live, large launches gain (+5.6% on
// 256 x VGA, +3.5% at 1080p, +1.2% late in a sequence); a launch of one or
// two waves is a single latency chain per warp, where the extra L1 round
// trip costs (-6% on one VGA frame) -- profiles/variants_r02.json.
// 0 disables the kL1 form.
#ifndef RGBDSEG_L1_MIN_WAVES
#define RGBDSEG_L1_MIN_WAVES 4
#endif
#ifndef RGBDSEG_PRE_COLOR  // colour components loaded with the flag words (2 or 3)
#define RGBDSEG_PRE_COLOR 2
#endif
#ifndef RGBDSEG_ELIDE_MINB  // resident blocks of the elided K1 (A/B builds override)
#define RGBDSEG_ELIDE_MINB 12
#endif
#ifndef RGBDSEG_FUSED_MIN_BLOCKS
#define RGBDSEG_FUSED_MIN_BLOCKS(elide) ((elide) ? RGBDSEG_ELIDE_MINB : 6)
#endif
// First-round values of one K1 pixel: everything that does not depend on
// its flag words -- inputs, both flag words, colour components
// 0..kPre-1 and depth component 0 (component 0 is touched in every
// initialised pixel, colour component 1 in most; a loaded untouched
// component equals its substitute).  Only the rest waits for the flags.
constexpr int kPre = RGBDSEG_PRE_COLOR;
// 1: once the flags are known, prefetch into L1 the colour planes the
// second load round will read (components kPre..N-1 this lane needs), so
// their latency overlaps the depth step; those loads then go through L1.
#ifndef RGBDSEG_PF_COLOR
#define RGBDSEG_PF_COLOR 0
#endif
// Where K1 reads its fusion state (out, cpt): 0 = at List 1 (prefetched to
// L1 in round one), 1 = right after the depth step, 2 = in round one,
// 3 = at List 1 from L2 (prefetched to L2 in round one).
#ifndef RGBDSEG_FUSE_LOAD
#define RGBDSEG_FUSE_LOAD 0
#endif
struct Round1 {
    float vc[3];
    uint32_t raw, cf, df;
#if RGBDSEG_FUSE_LOAD == 2
    uint32_t out0, cpt0;
#endif
    Mixture<kPre, 3> cpre;
    Mixture<1, 1> dpre;
};

// Per-thread addresses of K1 pixel t of the block whose first pixel is i0.
// A per-block uniform base plus a 32-bit per-thread offset: tiles are
// warp-aligned (launch_fused requires base % 32 == 0), so warp w of the
// block owns tile (base + i0) / 32 + w.
template <int MC, int MD>
struct PixAddr {
    float* cs;
    float* ds;
    __device__ __forceinline__ PixAddr(const FusedArgs& a, size_t i0, unsigned t) {
        constexpr unsigned SC = bank_stride(MC, 3), SD = bank_stride(MD, 1);
        const size_t tile0 = (a.base + i0) / kBlockPx;
        const unsigned w = t / kBlockPx, lane = t % kBlockPx;
        cs = a.color.state + tile0 * SC + (w * SC + lane);
        ds = a.depth.state + tile0 * SD + (w * SD + lane);
    }
    // Flag word of the pixel at cs / ds: the slot after the planes of its
    // tile, uint16 per lane (byte offset NP*128 - 2*lane from the plane-0
    // word).  Derived on use -- holding two more pointers costs spills.
    __device__ __forceinline__ uint16_t* cflag() const {
        const unsigned lane = threadIdx.x % kBlockPx;
        return reinterpret_cast<uint16_t*>(reinterpret_cast<char*>(cs) + bank_planes(MC, 3) * 128 - 2 * lane);
    }
    __device__ __forceinline__ uint16_t* dflag() const {
        const unsigned lane = threadIdx.x % kBlockPx;
        return reinterpret_cast<uint16_t*>(reinterpret_cast<char*>(ds) + bank_planes(MD, 1) * 128 - 2 * lane);
    }
};

// K1 after the first load round: the touched-prefix dispatch, the depth
// step, the colour step, List 1 and the stores.  Returns the three labels
// for the evaluation epilogue.
// kLean: the processor's device-resident fused path -- fusion on, no mask
// outputs (the launcher checks), so no pointer tests in the epilogue.
#ifndef RGBDSEG_LEAN  // 1: launch the kLean instantiation when it applies (+0.8%, variants_r02.json)
#define RGBDSEG_LEAN 1
#endif
#ifndef RGBDSEG_FUSE_SEL  // 1: List 1 as selects (fuse_pixel_sel) in K1 (measured 1-2% slower)
#define RGBDSEG_FUSE_SEL 0
#endif
template <int MC, int MD, bool kElide, bool kLean = false, bool kL1 = false>
__device__ __forceinline__ void fused_core(const FusedArgs& a, size_t i0, unsigned t,
                                           const PixAddr<MC, MD>& p, const Round1& r,
                                           uint32_t (&lab)[3]) {
    // Components to read: the elided variant skips untouched ones and runs
    // the step on the warp's touched prefix (+1); the dense one reads all.
    const uint32_t cneed = kElide ? ~flag_untouched<MC>(r.cf) : ~0u;
    const uint32_t dneed = kElide ? ~flag_untouched<MD>(r.df) : ~0u;
    int kc = MC, kd = MD;
    if (kElide) {
        const unsigned am = __activemask();
        kc = __reduce_max_sync(am, (r.cf & 0xffu) ? touched_prefix<MC>(r.cf) : 1);
        kd = __reduce_max_sync(am, (r.raw != 0 && (r.df & 0xffu)) ? touched_prefix<MD>(r.df) : 1);
    }

#if RGBDSEG_PF_COLOR
    if (kElide && (r.cf & 0xffu)) {
        const int N = min(kc + 1, MC);
        const uint32_t pf = cneed & ~((1u << kPre) - 1u) & ((1u << N) - 1u);
#pragma unroll
        for (int i = kPre; i < MC; ++i)
            if ((pf >> i) & 1u) {
#pragma unroll
                for (int c = 0; c < 3; ++c)
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(p.cs + (i * 3 + c) * kBlockPx));
                asm volatile("prefetch.global.L1 [%0];" ::"l"(p.cs + (MC * 3 + i) * kBlockPx));
                asm volatile("prefetch.global.L1 [%0];" ::"l"(p.cs + (MC * 4 + i) * kBlockPx));
            }
    }
#endif
    // The two banks are independent (only List 1 needs both labels): the
    // small depth step runs first, while the colour components wait in
    // registers (or, in the kL1 form, in the memory system).
    // ---- depth stream (segment_depth): raw 0 = no return ----
    uint32_t ld = 0;
    if (r.raw != 0) {
        const float vd[1] = {(float)r.raw};
        uint32_t df1 = r.df;
        bool replay = false;
        ld = k1_bank_pixel<MD, 1, 1, kElide>(p.ds, r.dpre, dneed, kd, vd, a.dk, a.depth, df1,
                                             replay);
        if (replay) ld = replay_pixel<MD, 1, kElide>(p.ds, vd, a.dk, a.depth, df1);
        if (df1 != r.df) st_h<kElide>(p.dflag(), (uint16_t)df1);
    }

#if RGBDSEG_FUSE_LOAD == 1
    const uint32_t out0 = (kLean || a.fuse) ? a.out[i0 + t] : 0u;
    const int cpt0 = (kLean || a.fuse) ? (int)a.cpt[i0 + t] : 0;
#endif
    // ---- colour stream (segment_color) ----
    const float vc[3] = {r.vc[0], r.vc[1], r.vc[2]};
    // kL1: colour components 0..kPre-1 were prefetched into L1 in round one
    // (not held in registers through the depth step); read them now.
    Mixture<kPre, 3> cl1;
    if constexpr (kL1) {
#pragma unroll
        for (int i = 0; i < kPre; ++i) {
#pragma unroll
            for (int c = 0; c < 3; ++c) cl1.mu[i][c] = p.cs[(i * 3 + c) * kBlockPx];
            cl1.var[i] = p.cs[(MC * 3 + i) * kBlockPx];
            cl1.w[i] = p.cs[(MC * 3 + MC + i) * kBlockPx];
        }
    }
    const Mixture<kPre, 3>& cpre = kL1 ? cl1 : r.cpre;
    uint32_t cf1 = r.cf;
    bool replay = false;
    uint32_t lc =
        k1_bank_pixel<MC, 3, kPre, kElide, kElide && RGBDSEG_PF_COLOR>(p.cs, cpre, cneed, kc, vc,
                                                                      a.ck, a.color, cf1, replay);
    if (replay) lc = replay_pixel<MC, 3, kElide>(p.cs, vc, a.ck, a.color, cf1);
    if (cf1 != r.cf) st_h<kElide>(p.cflag(), (uint16_t)cf1);

    // ---- List-1 fusion on the registered depth mask ----
    const bool fuse = kLean || a.fuse;
#if RGBDSEG_FUSE_LOAD == 0
    const uint32_t out0 = fuse ? a.out[i0 + t] : 0u;  // L1 hits (plain loads)
    const int cpt0 = fuse ? (int)a.cpt[i0 + t] : 0;
#elif RGBDSEG_FUSE_LOAD == 3
    const uint32_t out0 = fuse ? ld_h<true>(a.out + i0 + t) : 0u;  // L2 hits
    const int cpt0 = fuse ? (int)ld_h<true>(a.cpt + i0 + t) : 0;
#elif RGBDSEG_FUSE_LOAD == 2
    const uint32_t out0 = r.out0;
    const int cpt0 = (int)(int8_t)r.cpt0;
#endif
    uint32_t out = out0;
    int cpt = cpt0;
    if (fuse) {
        if (RGBDSEG_FUSE_SEL)
            fuse_pixel_sel(lc, ld, a.limit, out, cpt);
        else
            fuse_pixel(lc, ld, a.limit, out, cpt);
        if (!kElide || out != out0) st_h<kElide>(a.out + i0 + t, (uint8_t)out);
        if (!kElide || cpt != cpt0) st_h<kElide>(a.cpt + i0 + t, (int8_t)cpt);
    }
    if (!kLean) {
        if (a.rgb_mask) st_h<kElide>(a.rgb_mask + i0 + t, (uint8_t)lc);
        if (a.depth_mask) st_h<kElide>(a.depth_mask + i0 + t, (uint8_t)ld);
        if (a.fused_copy) st_h<kElide>(a.fused_copy + i0 + t, (uint8_t)out);
    }
    lab[0] = lc;
    lab[1] = ld;
    lab[2] = out;
}

// One pixel of K1 with its first round loaded straight from global memory.
// kPacked: the colour input is one interleaved 3-byte-per-pixel plane
// (a.r, RGB or BGR by a.bgr -- engine.cpp:39-56's aos_to_soa layout, or
// OpenCV's BGR), deinterleaved here in the first load round: a warp's three
// byte loads cover the same 96 contiguous bytes the three planar loads would.
#ifndef RGBDSEG_R1_DEPTH_FIRST  // 1: issue the depth component before the colour ones
#define RGBDSEG_R1_DEPTH_FIRST 0
#endif
template <int MC, int MD, bool kElide, bool kPacked = false, bool kLean = false,
          bool kL1 = false>
__device__ __forceinline__ void fused_pixel(const FusedArgs& a, size_t i0, unsigned t,
                                            uint32_t (&lab)[3]) {
    const PixAddr<MC, MD> p(a, i0, t);
    Round1 r;
    if constexpr (kPacked) {
        const uint8_t* px = a.r + (i0 + t) * 3;
        const int ro = a.bgr ? 2 : 0;
        r.vc[0] = (float)ld_h<kElide>(px + ro);
        r.vc[1] = (float)ld_h<kElide>(px + 1);
        r.vc[2] = (float)ld_h<kElide>(px + (2 - ro));
    } else {
        r.vc[0] = (float)ld_h<kElide>(a.r + i0 + t);
        r.vc[1] = (float)ld_h<kElide>(a.g + i0 + t);
        r.vc[2] = (float)ld_h<kElide>(a.b + i0 + t);
    }
    r.raw = ld_h<kElide>(a.d + i0 + t);
    r.cf = ld_h<kElide>(p.cflag());
    r.df = ld_h<kElide>(p.dflag());
#if RGBDSEG_FUSE_LOAD == 2
    r.out0 = a.fuse ? ld_h<kElide>(a.out + i0 + t) : 0u;
    r.cpt0 = a.fuse ? (uint32_t)(uint8_t)ld_h<kElide>(a.cpt + i0 + t) : 0u;
#elif RGBDSEG_FUSE_LOAD == 3
    if (kLean || a.fuse) {  // fusion state into L2 now, read at List 1 from L2
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.out + i0 + t));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.cpt + i0 + t));
    }
#else
    if (kLean || a.fuse) {  // fusion state into L1 now (no registers held), read at List 1
        asm volatile("prefetch.global.L1 [%0];" ::"l"(a.out + i0 + t));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(a.cpt + i0 + t));
    }
#endif
    if constexpr (kL1) {
        // one warp instruction: lane k < 5*kPre prefetches line k of colour
        // components 0..kPre-1 (means, then variances, then weights)
        const unsigned lane = t % kBlockPx;
        constexpr unsigned kL = 5 * kPre;
        if (lane < kL) {
            const unsigned pl = lane < 3 * kPre ? lane
                                : (lane < 4 * kPre ? MC * 3 + (lane - 3 * kPre)
                                                   : MC * 4 + (lane - 4 * kPre));
            const char* line = reinterpret_cast<const char*>(p.cs - lane) + pl * 128;
            asm volatile("prefetch.global.L1 [%0];" ::"l"(line));
        }
        load_mix<MD, kElide>(p.ds, r.dpre);
    } else {
#if RGBDSEG_R1_DEPTH_FIRST  // the depth step runs first: its words first
        load_mix<MD, kElide>(p.ds, r.dpre);
        load_mix<MC, kElide>(p.cs, r.cpre);
#else
        load_mix<MC, kElide>(p.cs, r.cpre);
        load_mix<MD, kElide>(p.ds, r.dpre);
#endif
    }
    fused_core<MC, MD, kElide, kLean, kL1>(a, i0, t, p, r, lab);
}

// kEval: with the evaluation epilogue (a.gt set).  A separate instantiation,
// so the plain kernel's register allocation carries none of it (measured 6%).
template <int MC, int MD, bool kElide, bool kEval, bool kPacked = false, bool kLean = false,
          bool kL1 = false, int kMinB = 0>
__global__ void __launch_bounds__(kThreads, kMinB ? kMinB : RGBDSEG_FUSED_MIN_BLOCKS(kElide))
    k_fused_ldg(const __grid_constant__ FusedArgs a) {
    const size_t i0 = (size_t)blockIdx.x * kThreads;
    const size_t i = i0 + threadIdx.x;
    const bool active = i < a.n;
    if (kEval && active)  // ground truth into L1 now, read after the steps
        asm volatile("prefetch.global.L1 [%0];" ::"l"(a.gt + i));
    if (!kElide && a.ahead && (threadIdx.x & 31) == 0) {
        // One bulk L2 prefetch per bank of the warp that starts about one
        // occupancy wave later: tiled blocks are contiguous, so its whole
        // state is two contiguous ranges.
        const size_t ia = i + (size_t)a.ahead * kThreads;
        if (ia < a.n) {
            const size_t ja = a.base + ia;
            const float* ct = a.color.state + (ja / kBlockPx) * bank_stride(MC, 3);
            const float* dt = a.depth.state + (ja / kBlockPx) * bank_stride(MD, 1);
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(ct),
                         "r"((unsigned)(bank_stride(MC, 3) * 4)));
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(dt),
                         "r"((unsigned)(bank_stride(MD, 1) * 4)));
        }
    }
    uint32_t lab[3] = {0u, 0u, 0u};
    if (active) fused_pixel<MC, MD, kElide, kPacked, kLean, kL1>(a, i0, threadIdx.x, lab);
    if constexpr (kEval) {  // evaluation epilogue: the masks never leave registers
        const uint32_t g = active ? (uint32_t)a.gt[i] : 0u;
        eval_accumulate<3>(active, a.base + i, a.stream_px, lab, g, a.counts);
    }
}

// ---------------------------------------------------------------- K1 experiments
// 2 px/thread and pipelined persistent variants (measured, dropped): only in
// A/B builds.
#ifndef RGBDSEG_PX
#define RGBDSEG_PX 1
#endif
#ifndef RGBDSEG_PIPE
#define RGBDSEG_PIPE 0
#endif
#if RGBDSEG_PX == 2 || RGBDSEG_PIPE
#include "k1_experiments.cuh"
#endif

// ---------------------------------------------------------------- near threshold
// Diagnostic pass (north_star's parity report): counts the pixels of one
// bank whose observation lies within `rel` (relative) of some component's
// match band in some channel, | |v_c - mu_ic| - lambda*sigma_i | <=
// rel * lambda*sigma_i, on the state BEFORE this frame's step.  Such a
// pixel is where an FMA-contracted or reassociated build would flip the
// match test (mixture.cpp:80-84).  Read-only; launched before K1 on the
// same stream when the processor's report is on.
template <int M, int C>
__global__ void __launch_bounds__(kThreads)
    k_near(BankView bk, const uint8_t* __restrict__ r, const uint8_t* __restrict__ g,
           const uint8_t* __restrict__ b, const uint16_t* __restrict__ d, size_t base, size_t n,
           float lambda, float rel, unsigned long long* count) {
    const size_t i = (size_t)blockIdx.x * kThreads + threadIdx.x;
    bool near = false;
    if (i < n) {
        const size_t j = base + i;
        const uint32_t f = *px_flag<M, C>(bk, j);
        float v[C];
        bool valid = (f & 0xffu) != 0;  // uninitialised pixels are seeded, not matched
        if constexpr (C == 3) {
            v[0] = (float)r[i];
            v[1] = (float)g[i];
            v[2] = (float)b[i];
        } else {
            const uint32_t raw = d[i];
            valid = valid && raw != 0;  // no return: no step (segmenter.cpp:84,128)
            v[0] = (float)raw;
        }
        if (valid) {
            const float* s = px_base<M, C>(bk, j);
#pragma unroll
            for (int q = 0; q < M; ++q) {
                const float band = fmul(lambda, fsqrt(s[(M * C + q) * kBlockPx]));
                const float tol = fmul(rel, band);
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    const float dist = fabsf(fsub(v[c], s[(q * C + c) * kBlockPx]));
                    near = near || fabsf(fsub(dist, band)) <= tol;
                }
            }
        }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, near);
    if ((threadIdx.x & 31) == 0 && bal) atomicAdd(count, (unsigned long long)__popc(bal));
}

// ---------------------------------------------------------------- K1b banks
// One bank alone (segment_color / segment_depth / segment_augmented drop-ins)
// on K1's machinery: the flag word's untouched mask, the step on the warp's
// touched prefix, components 0..P-1 read with the flag word, the exact
// replay deferred, L2-only loads and write-back stores.  `step` false
// (depth no-return) leaves the pixel untouched but joins the warp reduction.
template <int M, int C, int P>
__device__ __forceinline__ uint32_t bank_elided(const BankView& bk, size_t j, const float (&v)[C],
                                                bool step, const MixCfg& k) {
    float* s = px_base<M, C>(bk, j);
    uint16_t* fl = px_flag<M, C>(bk, j);
    const uint32_t f = ld_h<true>(fl);
    Mixture<P, C> pre;
    load_mix<M, true>(s, pre);
    const unsigned am = __activemask();
    const int Kw = __reduce_max_sync(am, (step && (f & 0xffu)) ? touched_prefix<M>(f) : 1);
    if (!step) return 0u;
    uint32_t f1 = f;
    bool replay = false;
    uint32_t lab = k1_bank_pixel<M, C, P, true>(s, pre, ~flag_untouched<M>(f), Kw, v, k, bk, f1,
                                                replay);
    if (replay) lab = replay_pixel<M, C, true>(s, v, k, bk, f1);
    if (f1 != f) st_h<true>(fl, (uint16_t)f1);
    return lab;
}

template <int M>
__global__ void __launch_bounds__(kThreads, RGBDSEG_FUSED_MIN_BLOCKS(true))
    k_bank_color(BankView bk, MixCfg k, const uint8_t* __restrict__ r,
                 const uint8_t* __restrict__ g, const uint8_t* __restrict__ b,
                 uint8_t* __restrict__ mask, size_t n) {
    const size_t j = (size_t)blockIdx.x * kThreads + threadIdx.x;
    if (j >= n) return;
    const float v[3] = {(float)ld_h<true>(r + j), (float)ld_h<true>(g + j),
                        (float)ld_h<true>(b + j)};
    const uint32_t lab = bank_elided<M, 3, 2>(bk, j, v, true, k);
    if (mask) mask[j] = (uint8_t)lab;
}

template <int M>
__global__ void __launch_bounds__(kThreads, RGBDSEG_FUSED_MIN_BLOCKS(true))
    k_bank_depth(BankView bk, MixCfg k, const uint16_t* __restrict__ d,
                 uint8_t* __restrict__ mask, size_t n) {
    const size_t j = (size_t)blockIdx.x * kThreads + threadIdx.x;
    if (j >= n) return;
    const uint32_t raw = ld_h<true>(d + j);
    const float v[1] = {(float)raw};
    const uint32_t lab = bank_elided<M, 1, 1>(bk, j, v, raw != 0, k);  // segmenter.cpp:84,128
    if (mask) mask[j] = (uint8_t)lab;
}

// DepthRescale::to_channel (segmenter.cpp:18-22): metric depth onto 0..255.
__device__ __forceinline__ float rescale_depth(float d, float lo, float hi) {
    if (d <= lo) return 0.0f;
    if (d >= hi) return 255.0f;
    return fdiv(fmul(fsub(d, lo), 255.0f), fsub(hi, lo));
}

// segment_augmented (segmenter.cpp:133-147): one 4-channel mixture over
// (R, G, B, rescaled depth).  No no-return sentinel here: raw 0 rescales to
// channel value 0 and is modelled like any other observation.
template <int M>
__global__ void __launch_bounds__(kThreads, RGBDSEG_FUSED_MIN_BLOCKS(true))
    k_bank_aug(BankView bk, MixCfg k, const uint8_t* __restrict__ r,
               const uint8_t* __restrict__ g, const uint8_t* __restrict__ b,
               const uint16_t* __restrict__ d, float lo, float hi, uint8_t* __restrict__ mask,
               size_t n) {
    const size_t j = (size_t)blockIdx.x * kThreads + threadIdx.x;
    if (j >= n) return;
    const float v[4] = {(float)ld_h<true>(r + j), (float)ld_h<true>(g + j),
                        (float)ld_h<true>(b + j), rescale_depth((float)ld_h<true>(d + j), lo, hi)};
    const uint32_t lab = bank_elided<M, 4, 2>(bk, j, v, true, k);
    if (mask) mask[j] = (uint8_t)lab;
}

// ModelBank ctor state (segmenter.cpp:24-34): means 0, var sigma0^2, w (1,0,..)
__global__ void k_bank_reset(BankView bk, float sigma0, size_t n) {
    const size_t j = (size_t)blockIdx.x * kThreads + threadIdx.x;
    if (j >= n) return;
    const float var0 = fmul(sigma0, sigma0);
    const int M = bk.M, C = bk.C, NP = bank_planes(M, C);
    float* s = bk.state + (j / kBlockPx) * bank_stride(M, C) + (j % kBlockPx);
    for (int p = 0; p < M * C; ++p) s[p * kBlockPx] = 0.0f;
    for (int q = 0; q < M; ++q) {
        s[(M * C + q) * kBlockPx] = var0;
        s[(M * C + M + q) * kBlockPx] = q == 0 ? 1.0f : 0.0f;
    }
    reinterpret_cast<uint16_t*>(s - (j % kBlockPx) + NP * kBlockPx)[j % kBlockPx] = 0;
}

// Flat plane <-> tiled bank (ModelBank::mean_plane / gather / scatter views).
__global__ void k_bank_gather(BankView bk, int plane, size_t n, void* dst) {
    const size_t j = (size_t)blockIdx.x * kThreads + threadIdx.x;
    if (j >= n) return;
    const int NP = bank_planes(bk.M, bk.C);
    const float* blk = bk.state + (j / kBlockPx) * bank_stride(bk.M, bk.C);
    if (plane < 0)
        static_cast<uint8_t*>(dst)[j] =
            (uint8_t)reinterpret_cast<const uint16_t*>(blk + NP * kBlockPx)[j % kBlockPx];
    else
        static_cast<float*>(dst)[j] = blk[plane * kBlockPx + j % kBlockPx];
}

__global__ void k_bank_scatter(BankView bk, int plane, size_t n, const void* src) {
    const size_t j = (size_t)blockIdx.x * kThreads + threadIdx.x;
    if (j >= n) return;
    const int NP = bank_planes(bk.M, bk.C);
    float* blk = bk.state + (j / kBlockPx) * bank_stride(bk.M, bk.C);
    uint16_t* fl = reinterpret_cast<uint16_t*>(blk + NP * kBlockPx) + j % kBlockPx;
    if (plane < 0) {
        *fl = static_cast<const uint8_t*>(src)[j];  // mask cleared
    } else {
        blk[plane * kBlockPx + j % kBlockPx] = static_cast<const float*>(src)[j];
        *fl = *fl & 0xffu;
    }
}

// ---------------------------------------------------------------- K1c fusion
// k_fuse on 16 pixels per thread (16-byte-aligned planes; the launcher
// checks, and the last partial chunk goes per pixel).
__global__ void __launch_bounds__(kThreads)
    k_fuse16(uint8_t* __restrict__ out, int8_t* __restrict__ cpt, const uint8_t* __restrict__ rgb,
             const uint8_t* __restrict__ dep, uint8_t* __restrict__ out_copy, int limit, size_t n) {
    const size_t c = (size_t)blockIdx.x * kThreads + threadIdx.x;
    const size_t j0 = c * 16;
    if (j0 >= n) return;
    if (j0 + 16 > n) {
        for (size_t j = j0; j < n; ++j) {
            uint32_t o = out[j];
            int k = cpt[j];
            fuse_pixel(rgb[j], dep[j], limit, o, k);
            out[j] = (uint8_t)o;
            cpt[j] = (int8_t)k;
            if (out_copy) out_copy[j] = (uint8_t)o;
        }
        return;
    }
    const uint4 vr = reinterpret_cast<const uint4*>(rgb)[c], vd = reinterpret_cast<const uint4*>(dep)[c];
    const uint4 vo = reinterpret_cast<const uint4*>(out)[c];
    const uint4 vc = reinterpret_cast<const uint4*>(cpt)[c];
    const uint32_t R[4] = {vr.x, vr.y, vr.z, vr.w}, D[4] = {vd.x, vd.y, vd.z, vd.w};
    uint32_t O[4] = {vo.x, vo.y, vo.z, vo.w}, K[4] = {vc.x, vc.y, vc.z, vc.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        uint32_t no = 0u, nk = 0u;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            uint32_t o = (O[q] >> (8 * b)) & 0xffu;
            int k = (int)(int8_t)((K[q] >> (8 * b)) & 0xffu);
            fuse_pixel((R[q] >> (8 * b)) & 0xffu, (D[q] >> (8 * b)) & 0xffu, limit, o, k);
            no |= (o & 0xffu) << (8 * b);
            nk |= ((uint32_t)k & 0xffu) << (8 * b);
        }
        O[q] = no;
        K[q] = nk;
    }
    reinterpret_cast<uint4*>(out)[c] = make_uint4(O[0], O[1], O[2], O[3]);
    reinterpret_cast<uint4*>(cpt)[c] = make_uint4(K[0], K[1], K[2], K[3]);
    if (out_copy) reinterpret_cast<uint4*>(out_copy)[c] = make_uint4(O[0], O[1], O[2], O[3]);
}

__global__ void __launch_bounds__(kThreads)
    k_fuse(uint8_t* __restrict__ out, int8_t* __restrict__ cpt, const uint8_t* __restrict__ rgb,
           const uint8_t* __restrict__ dep, uint8_t* __restrict__ out_copy, int limit, size_t n) {
    const size_t j = (size_t)blockIdx.x * kThreads + threadIdx.x;
    if (j >= n) return;
    uint32_t o = out[j];
    int c = cpt[j];
    fuse_pixel(rgb[j], dep[j], limit, o, c);
    out[j] = (uint8_t)o;
    cpt[j] = (int8_t)c;
    if (out_copy) out_copy[j] = (uint8_t)o;
}

// ---------------------------------------------------------------- K0 per pixel
template <int M, int C>
__device__ void rec_step(PixRec& rec, const float* vals, const MixCfg& k, uint8_t& lab) {
    Mixture<M, C> m;
#pragma unroll
    for (int i = 0; i < M; ++i) {
#pragma unroll
        for (int c = 0; c < C; ++c) m.mu[i][c] = rec.means[i * C + c];
        m.var[i] = rec.variances[i];
        m.w[i] = rec.weights[i];
    }
    float v[C];
#pragma unroll
    for (int c = 0; c < C; ++c) v[c] = vals[c];
    lab = (uint8_t)gmm_step(m, v, k);
#pragma unroll
    for (int i = 0; i < M; ++i) {
#pragma unroll
        for (int c = 0; c < C; ++c) rec.means[i * C + c] = m.mu[i][c];
        rec.variances[i] = m.var[i];
        rec.weights[i] = m.w[i];
    }
}

template <int M>
__device__ void rec_step_c(PixRec& rec, const float* vals, const MixCfg& k, uint8_t& lab) {
    switch (rec.channels) {
        case 1: rec_step<M, 1>(rec, vals, k, lab); break;
        case 2: rec_step<M, 2>(rec, vals, k, lab); break;
        case 3: rec_step<M, 3>(rec, vals, k, lab); break;
        case 4: rec_step<M, 4>(rec, vals, k, lab); break;
        default: lab = 255; break;
    }
}

__global__ void k_mix_step(PixRec* recs, const float* values, int channels, size_t n, MixCfg k,
                           uint8_t* labels) {
    const size_t j = (size_t)blockIdx.x * kThreads + threadIdx.x;
    if (j >= n) return;
    PixRec rec = recs[j];
    uint8_t lab = 255;
    if (rec.channels == channels) {
        const float* v = values + j * channels;
        switch (rec.components) {  // step_pixel loops over mixture.components
            case 3: rec_step_c<3>(rec, v, k, lab); break;
            case 4: rec_step_c<4>(rec, v, k, lab); break;
            case 5: rec_step_c<5>(rec, v, k, lab); break;
            default: break;
        }
    }
    if (lab != 255) recs[j] = rec;
    labels[j] = lab;
}

// match_component / classify / update_mixture on their own (mixture.hpp:45-56).
template <int M, int C>
__device__ void rec_op(PixRec& rec, const float* vals, const MixCfg& k, int op, int& matched,
                       uint8_t& lab) {
    Mixture<M, C> m;
#pragma unroll
    for (int i = 0; i < M; ++i) {
#pragma unroll
        for (int c = 0; c < C; ++c) m.mu[i][c] = rec.means[i * C + c];
        m.var[i] = rec.variances[i];
        m.w[i] = rec.weights[i];
    }
    float v[C];
#pragma unroll
    for (int c = 0; c < C; ++c) v[c] = vals ? vals[c] : 0.0f;
    if (op == kOpMatch) {
        matched = gmm_match(m, v, k);
        lab = 0;
    } else if (op == kOpClassify) {
        lab = (uint8_t)gmm_classify(m, matched, k);
    } else {
        gmm_update(m, v, matched, k);
        lab = 0;
#pragma unroll
        for (int i = 0; i < M; ++i) {
#pragma unroll
            for (int c = 0; c < C; ++c) rec.means[i * C + c] = m.mu[i][c];
            rec.variances[i] = m.var[i];
            rec.weights[i] = m.w[i];
        }
    }
}

template <int M>
__device__ void rec_op_c(PixRec& rec, const float* vals, const MixCfg& k, int op, int& matched,
                         uint8_t& lab) {
    switch (rec.channels) {
        case 1: rec_op<M, 1>(rec, vals, k, op, matched, lab); break;
        case 2: rec_op<M, 2>(rec, vals, k, op, matched, lab); break;
        case 3: rec_op<M, 3>(rec, vals, k, op, matched, lab); break;
        case 4: rec_op<M, 4>(rec, vals, k, op, matched, lab); break;
        default: lab = 255; break;
    }
}

// values: n * rec.channels floats (NULL for classify); matched: in for
// classify / update, out for match; labels: classify's result (255 = bad
// record shape, which the host rejects before launching).
__global__ void k_mix_op(PixRec* recs, const float* values, size_t n, MixCfg k, int op,
                         int* matched, uint8_t* labels) {
    const size_t j = (size_t)blockIdx.x * kThreads + threadIdx.x;
    if (j >= n) return;
    PixRec rec = recs[j];
    int mt = op == kOpMatch ? -1 : matched[j];
    uint8_t lab = 255;
    const float* v = values ? values + j * rec.channels : nullptr;
    switch (rec.components) {
        case 3: rec_op_c<3>(rec, v, k, op, mt, lab); break;
        case 4: rec_op_c<4>(rec, v, k, op, mt, lab); break;
        case 5: rec_op_c<5>(rec, v, k, op, mt, lab); break;
        default: break;
    }
    if (op == kOpMatch) matched[j] = mt;
    if (op == kOpClassify && labels) labels[j] = lab;
    if (op == kOpUpdate && lab != 255) recs[j] = rec;
}

__global__ void k_mix_init(const float* values, int channels, size_t n, MixCfg k, int M,
                           PixRec* out) {
    const size_t j = (size_t)blockIdx.x * kThreads + threadIdx.x;
    if (j >= n) return;
    PixRec rec;
    rec.components = M;
    rec.channels = channels;
    for (int q = 0; q < 20; ++q) rec.means[q] = 0.0f;
    const float var0 = fmul(k.sigma0, k.sigma0);
    for (int q = 0; q < 5; ++q) {
        rec.variances[q] = q < M ? var0 : 0.0f;
        rec.weights[q] = q == 0 ? 1.0f : 0.0f;
    }
    for (int c = 0; c < channels; ++c) rec.means[c] = values[j * channels + c];
    out[j] = rec;
}

// ---------------------------------------------------------------- K3 render
__device__ __forceinline__ uint64_t splitmix(uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t hash5(uint64_t seed, uint64_t st, uint64_t fr, uint64_t px,
                                          uint64_t ch) {  // synthetic.cpp:66-74
    uint64_t h = splitmix(seed ^ 0x6a09e667f3bcc908ULL);
    h = splitmix(h ^ st);
    h = splitmix(h ^ fr);
    h = splitmix(h ^ px);
    return splitmix(h ^ ch);
}

__device__ __forceinline__ double gauss5(uint64_t seed, uint64_t st, uint64_t fr, uint64_t px,
                                         uint64_t ch) {  // synthetic.cpp:76-83
    const uint64_t h = hash5(seed, st, fr, px, ch);
    const double u1 = __ddiv_rn(__dadd_rn((double)(h >> 32), 1.0), 4294967297.0);
    const double u2 = __ddiv_rn((double)(h & 0xffffffffULL), 4294967296.0);
    return __dmul_rn(__dsqrt_rn(__dmul_rn(-2.0, log(u1))),
                     cos(__dmul_rn(__dmul_rn(2.0, 3.141592653589793), u2)));
}

__device__ __forceinline__ bool in_rect(const int (&rc)[4], int x, int y) {
    return x >= rc[0] && x < rc[0] + rc[2] && y >= rc[1] && y < rc[1] + rc[3];
}

__global__ void k_render(const __grid_constant__ SceneFrame sc, uint8_t* R, uint8_t* G,
                         uint8_t* B, uint16_t* D, uint8_t* GT, size_t n) {
    const size_t idx = (size_t)blockIdx.x * kThreads + threadIdx.x;
    if (idx >= n) return;
    const size_t per = (size_t)sc.width * sc.height;
    const uint64_t s = idx / per;
    const uint64_t pix = idx - s * per;
    const int x = (int)(pix % sc.width), y = (int)(pix / sc.width);
    const uint64_t seed = sc.seed0 + s;
    const int w = sc.width, h = sc.height;
    double base[3] = {__dadd_rn(60.0, __ddiv_rn(__dmul_rn(90.0, (double)x), (double)w)),
                      __dadd_rn(70.0, __ddiv_rn(__dmul_rn(90.0, (double)y), (double)h)),
                      __dadd_rn(80.0, __ddiv_rn(__dmul_rn(80.0, (double)(x + y)), (double)(w + h)))};
    const uint64_t span = (uint64_t)__dadd_rn(__dmul_rn(2.0, (double)sc.color_texture), 1.0);
    for (int c = 0; c < 3; ++c) {
        const uint64_t t = hash5(seed, 1, 0, pix, c);
        base[c] = __dadd_rn(base[c], __dsub_rn((double)(t % span), (double)sc.color_texture));
    }
    double depth = sc.base_depth_mm;
    if (sc.depth_texture_mm > 0) {
        const uint64_t t = hash5(seed, 2, 0, pix, 0);
        depth = __dadd_rn(depth, __dsub_rn((double)(t % (uint64_t)(2 * sc.depth_texture_mm + 1)),
                                           (double)sc.depth_texture_mm));
    }
    int top = -1;
    for (int o = 0; o < sc.n_obj; ++o)
        if (in_rect(sc.orect[o], x, y)) top = o;
    uint8_t label = 0;
    if (top >= 0) {
        for (int c = 0; c < 3; ++c) base[c] = sc.ocolor[top][c];
        depth = __dsub_rn(depth, (double)sc.odepth[top]);
        label = 1;
    }
    double col[3] = {__dmul_rn(base[0], sc.gain), __dmul_rn(base[1], sc.gain),
                     __dmul_rn(base[2], sc.gain)};
    for (int e = 0; e < sc.n_shadow; ++e)
        if (in_rect(sc.srect[e], x, y))
            for (int c = 0; c < 3; ++c) col[c] = __dmul_rn(col[c], sc.sdarken[e]);
    for (int e = 0; e < sc.n_flicker; ++e) {
        if (!in_rect(sc.frect[e], x, y)) continue;
        for (int c = 0; c < 3; ++c)
            col[c] = __dadd_rn(col[c], __dmul_rn(sc.fcs[e], gauss5(seed, 5, sc.frame, pix, c)));
        depth = __dadd_rn(depth, __dmul_rn(sc.fds[e], gauss5(seed, 6, sc.frame, pix, 0)));
    }
    for (int c = 0; c < 3; ++c)
        col[c] = __dadd_rn(col[c], __dmul_rn(sc.ncs, gauss5(seed, 3, sc.frame, pix, c)));
    depth = __dadd_rn(depth, __dmul_rn(sc.nds, gauss5(seed, 4, sc.frame, pix, 0)));
    long q[3];
    for (int c = 0; c < 3; ++c) {
        q[c] = lround(col[c]);
        q[c] = q[c] < 0 ? 0 : (q[c] > 255 ? 255 : q[c]);
    }
    long dq = lround(depth);
    dq = dq < 1 ? 1 : (dq > 65535 ? 65535 : dq);
    R[idx] = (uint8_t)q[0];
    G[idx] = (uint8_t)q[1];
    B[idx] = (uint8_t)q[2];
    D[idx] = (uint16_t)dq;
    if (GT) GT[idx] = label;
}

// ---------------------------------------------------------------- K2 registration
// register_mask (registration.cpp:50-78): the same fp64 expression trees,
// every op an explicit round-to-nearest double intrinsic (no contraction),
// lround() half away from zero like std::lround.
__device__ __forceinline__ void splat_pixel(size_t idx, const uint16_t* __restrict__ depth,
                                            int dw, int dh, const RigDev& rig, int cw, int ch,
                                            uint8_t* __restrict__ out) {
    const size_t per = (size_t)dw * dh;
    const size_t s = idx / per;
    const int p = (int)(idx - s * per);
    const int u = p % dw, v = p / dw;
    const uint32_t raw = depth[idx];
    if (raw == 0) return;  // no range return, cannot be registered
    const double z = __dmul_rn((double)raw, rig.scale);
    const double x = __ddiv_rn(__dmul_rn(__dsub_rn((double)u, rig.dcx), z), rig.dfx);
    const double y = __ddiv_rn(__dmul_rn(__dsub_rn((double)v, rig.dcy), z), rig.dfy);
    const double* R = rig.R;
    const double xc = __dadd_rn(
        __dadd_rn(__dadd_rn(__dmul_rn(R[0], x), __dmul_rn(R[1], y)), __dmul_rn(R[2], z)), rig.t[0]);
    const double yc = __dadd_rn(
        __dadd_rn(__dadd_rn(__dmul_rn(R[3], x), __dmul_rn(R[4], y)), __dmul_rn(R[5], z)), rig.t[1]);
    const double zc = __dadd_rn(
        __dadd_rn(__dadd_rn(__dmul_rn(R[6], x), __dmul_rn(R[7], y)), __dmul_rn(R[8], z)), rig.t[2]);
    if (zc <= 0.0) return;
    const long uc = lround(__dadd_rn(__ddiv_rn(__dmul_rn(rig.cfx, xc), zc), rig.ccx));
    const long vc = lround(__dadd_rn(__ddiv_rn(__dmul_rn(rig.cfy, yc), zc), rig.ccy));
    if (uc < 0 || uc >= cw || vc < 0 || vc >= ch) return;
    out[s * (size_t)cw * ch + (size_t)vc * cw + uc] = 1;
}

__global__ void k_register_splat(const uint8_t* __restrict__ mask,
                                 const uint16_t* __restrict__ depth, int dw, int dh, size_t n,
                                 const __grid_constant__ RigDev rig, int cw, int ch,
                                 uint8_t* __restrict__ out) {
    const size_t idx = (size_t)blockIdx.x * kThreads + threadIdx.x;
    if (idx >= n || !mask[idx]) return;
    splat_pixel(idx, depth, dw, dh, rig, cw, ch, out);
}

// 16 mask bytes per thread (one 16-byte load; most chunks are background
// and stop there).  n % 16 == 0 and a 16-byte-aligned mask (launcher checks).
__global__ void k_register_splat16(const uint8_t* __restrict__ mask,
                                   const uint16_t* __restrict__ depth, int dw, int dh, size_t n16,
                                   const __grid_constant__ RigDev rig, int cw, int ch,
                                   uint8_t* __restrict__ out) {
    const size_t c = (size_t)blockIdx.x * kThreads + threadIdx.x;
    if (c >= n16) return;
    const uint4 m = reinterpret_cast<const uint4*>(mask)[c];
    const uint32_t wds[4] = {m.x, m.y, m.z, m.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (!wds[k]) continue;
#pragma unroll
        for (int b = 0; b < 4; ++b)
            if ((wds[k] >> (8 * b)) & 0xffu) splat_pixel(c * 16 + k * 4 + b, depth, dw, dh, rig, cw, ch, out);
    }
}

// dilate_mask (registration.cpp:33-48): OR over a clipped (2r+1)-square,
// done as a clipped row OR then a clipped column OR.
template <bool kRows>
__global__ void k_dilate_pass(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, int w,
                              int h, size_t n, int r) {
    const size_t idx = (size_t)blockIdx.x * kThreads + threadIdx.x;
    if (idx >= n) return;
    const size_t per = (size_t)w * h;
    const size_t base = (idx / per) * per;
    const int p = (int)(idx - base);
    const int x = p % w, y = p / w;
    uint32_t acc = 0;
    if (kRows) {
        const int x0 = max(0, x - r), x1 = min(w - 1, x + r);
        for (int xx = x0; xx <= x1 && !acc; ++xx) acc |= in[base + (size_t)y * w + xx];
    } else {
        const int y0 = max(0, y - r), y1 = min(h - 1, y + r);
        for (int yy = y0; yy <= y1 && !acc; ++yy) acc |= in[base + (size_t)yy * w + x];
    }
    out[idx] = acc ? 1 : 0;
}

// Vector forms of the two passes: 16 pixels of one row per thread (w % 16
// == 0, 16-byte-aligned planes).  Bytes are OR-ed as 0 / nonzero and the
// result normalised to 0 / 1 with a per-byte compare (__vcmpne4).
__device__ __forceinline__ uint32_t nz01(uint32_t v) { return __vcmpne4(v, 0u) & 0x01010101u; }

// Column pass: OR of the clipped rows y-r..y+r.
__global__ void k_dilate_cols16(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, int w,
                                int h, size_t n16, int r) {
    const size_t c = (size_t)blockIdx.x * kThreads + threadIdx.x;
    if (c >= n16) return;
    const size_t idx = c * 16, per = (size_t)w * h;
    const size_t base = (idx / per) * per;
    const int p = (int)(idx - base), x = p % w, y = p / w;
    const int y0 = max(0, y - r), y1 = min(h - 1, y + r);
    uint4 acc = make_uint4(0u, 0u, 0u, 0u);
    for (int yy = y0; yy <= y1; ++yy) {
        const uint4 v = *reinterpret_cast<const uint4*>(in + base + (size_t)yy * w + x);
        acc.x |= v.x;
        acc.y |= v.y;
        acc.z |= v.z;
        acc.w |= v.w;
    }
    *reinterpret_cast<uint4*>(out + idx) = make_uint4(nz01(acc.x), nz01(acc.y), nz01(acc.z), nz01(acc.w));
}

// Row pass (r <= 16): the chunk and its clipped neighbours as a 48-byte
// window; output byte i = OR of window bytes 16+i-r .. 16+i+r, built from
// byte-shifted words (funnel shifts).
__global__ void k_dilate_rows16(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, int w,
                                size_t n16, int r) {
    const size_t c = (size_t)blockIdx.x * kThreads + threadIdx.x;
    if (c >= n16) return;
    const size_t idx = c * 16;
    const int x = (int)(idx % (size_t)w);
    const uint4 z = make_uint4(0u, 0u, 0u, 0u);
    const uint4 L = x > 0 ? *reinterpret_cast<const uint4*>(in + idx - 16) : z;
    const uint4 Mv = *reinterpret_cast<const uint4*>(in + idx);
    const uint4 Rv = x + 16 < w ? *reinterpret_cast<const uint4*>(in + idx + 16) : z;
    const uint32_t wd[13] = {L.x, L.y, L.z, L.w, Mv.x, Mv.y, Mv.z, Mv.w, Rv.x, Rv.y, Rv.z, Rv.w, 0u};
    uint32_t acc[4] = {0u, 0u, 0u, 0u};
    for (int d = -r; d <= r; ++d) {
        const int o = 16 + d, q = o >> 2, sh = 8 * (o & 3);  // window starts at byte o
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j] |= __funnelshift_r(wd[q + j], wd[q + j + 1], sh);
    }
    *reinterpret_cast<uint4*>(out + idx) = make_uint4(nz01(acc[0]), nz01(acc[1]), nz01(acc[2]), nz01(acc[3]));
}

template <typename K, typename... Args>
cudaError_t go(K kernel, size_t n, cudaStream_t s, Args... args) {
    if (n == 0) return cudaSuccess;
    kernel<<<blocks_for(n), kThreads, 0, s>>>(args...);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
}

// Whether a K1 launch over n pixels is large enough for the kL1 form: n at
// least RGBDSEG_L1_MIN_WAVES occupancy waves of the elided kernel (12
// resident 128-pixel blocks per SM) on the launching device.
bool l1_form(size_t n) {
    if (RGBDSEG_L1_MIN_WAVES <= 0) return false;
    constexpr int kMaxDev = 64;
    static std::atomic<int> sms_cache[kMaxDev];
    int dev = 0;
    cudaGetDevice(&dev);
    int sms = dev < kMaxDev ? sms_cache[dev].load(std::memory_order_relaxed) : 0;
    if (sms <= 0) {
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (dev < kMaxDev) sms_cache[dev].store(sms, std::memory_order_relaxed);
    }
    const size_t wave = (size_t)sms * RGBDSEG_ELIDE_MINB * kThreads;
    return n >= (size_t)RGBDSEG_L1_MIN_WAVES * wave;
}

// Launches of at least RGBDSEG_HUGE_WAVES occupancy waves (256 x VGA,
// 8192^2) run the kL1 form at RGBDSEG_HUGE_MINB resident blocks: +0.5% on the
// default window and +1.4% / +2.8% late on 256 x VGA / 8192^2, where 1080p
// (9 waves) prefers 12 (profiles/variants_r02.json).
#ifndef RGBDSEG_HUGE_WAVES
#define RGBDSEG_HUGE_WAVES 40
#endif
#ifndef RGBDSEG_HUGE_MINB
#define RGBDSEG_HUGE_MINB 16
#endif
bool huge_launch(size_t n) {
    if (RGBDSEG_HUGE_WAVES <= 0) return false;
    constexpr int kMaxDev = 64;
    static std::atomic<int> sms_cache[kMaxDev];
    int dev = 0;
    cudaGetDevice(&dev);
    int sms = dev < kMaxDev ? sms_cache[dev].load(std::memory_order_relaxed) : 0;
    if (sms <= 0) {
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (dev < kMaxDev) sms_cache[dev].store(sms, std::memory_order_relaxed);
    }
    return n >= (size_t)RGBDSEG_HUGE_WAVES * sms * RGBDSEG_ELIDE_MINB * kThreads;
}

template <int MC, int MD>
cudaError_t fused_ldg_md(const FusedArgs& a, bool elide, int variant, cudaStream_t s) {
    if (a.n == 0) return cudaSuccess;
    const unsigned nb = blocks_for(a.n);
    const bool l1 = elide && (variant == kLdgElideL1 || (variant == kAuto && l1_form(a.n)));
    if (a.packed) {  // interleaved colour input (no evaluation epilogue)
        if (a.gt) return cudaErrorInvalidValue;
        if (!elide)
            k_fused_ldg<MC, MD, false, false, true><<<nb, kThreads, 0, s>>>(a);
        else if (l1)
            k_fused_ldg<MC, MD, true, false, true, false, true><<<nb, kThreads, 0, s>>>(a);
        else
            k_fused_ldg<MC, MD, true, false, true><<<nb, kThreads, 0, s>>>(a);
    } else if (elide) {
        if (a.gt) {  // the evaluation instantiation keeps the register form (L1: -2.3%)
            k_fused_ldg<MC, MD, true, true><<<nb, kThreads, 0, s>>>(a);
        } else {
#if RGBDSEG_PX == 2
            k_fused_x2<MC, MD><<<(unsigned)((a.n + 2 * kThreads - 1) / (2 * kThreads)), kThreads, 0, s>>>(a);
#elif RGBDSEG_PIPE
            k_fused_pipe<MC, MD><<<pipe_blocks<MC, MD>(a.n), kThreads, 0, s>>>(a);
#else
            const bool lean = RGBDSEG_LEAN && a.fuse && !a.rgb_mask && !a.depth_mask &&
                              !a.fused_copy;
            if (l1 && huge_launch(a.n)) {  // 32 registers, 64 warps/SM
                lean ? k_fused_ldg<MC, MD, true, false, false, true, true, RGBDSEG_HUGE_MINB>
                           <<<nb, kThreads, 0, s>>>(a)
                     : k_fused_ldg<MC, MD, true, false, false, false, true, RGBDSEG_HUGE_MINB>
                           <<<nb, kThreads, 0, s>>>(a);
            } else if (l1) {
                lean ? k_fused_ldg<MC, MD, true, false, false, true, true><<<nb, kThreads, 0, s>>>(a)
                     : k_fused_ldg<MC, MD, true, false, false, false, true><<<nb, kThreads, 0, s>>>(a);
            } else {
                lean ? k_fused_ldg<MC, MD, true, false, false, true><<<nb, kThreads, 0, s>>>(a)
                     : k_fused_ldg<MC, MD, true, false><<<nb, kThreads, 0, s>>>(a);
            }
#endif
        }
    } else {
        a.gt ? k_fused_ldg<MC, MD, false, true><<<nb, kThreads, 0, s>>>(a)
             : k_fused_ldg<MC, MD, false, false><<<nb, kThreads, 0, s>>>(a);
    }
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
}

template <int MC, int MD>
cudaError_t fused_md(const FusedArgs& a0, int variant, cudaStream_t s) {
    const bool elide = variant != kLdgDense;
    // Resident blocks on the launching device (per variant and device
    // ordinal), computed once; racing host threads compute the same value,
    // so a relaxed atomic suffices.
    constexpr int kMaxDev = 64;
    static std::atomic<int> wave[kMaxDev][2];
    static std::atomic<bool> wave_init[kMaxDev][2];
    int dev = 0;
    cudaGetDevice(&dev);
    const int dslot = dev < kMaxDev ? dev : kMaxDev - 1;
    int wv = wave_init[dslot][elide ? 1 : 0].load(std::memory_order_acquire)
                 ? wave[dslot][elide ? 1 : 0].load(std::memory_order_relaxed)
                 : -1;
    if (wv < 0 || dev >= kMaxDev) {
        int bps = 0, sms = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &bps, elide ? k_fused_ldg<MC, MD, true, false> : k_fused_ldg<MC, MD, false, false>,
            kThreads, 0);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        // The elided kernel reads only what its flags ask for; every L2
        // prefetch tried ahead of it (whole tiles, first-round lines, flag-
        // aware planes) measured slower (profiles/variants_r01.json): off.
        wv = elide ? 0 : bps * sms;
        if (const char* e = getenv("RGBDSEG_L2_AHEAD")) wv = atoi(e);  // 0 disables
        wave[dslot][elide ? 1 : 0].store(wv, std::memory_order_relaxed);
        wave_init[dslot][elide ? 1 : 0].store(true, std::memory_order_release);
    }
    FusedArgs a = a0;
    a.ahead = (unsigned)wv;
    return fused_ldg_md<MC, MD>(a, elide, variant, s);
}

template <int MC>
cudaError_t fused_mc(const FusedArgs& a, int variant, cudaStream_t s) {
    switch (a.depth.M) {
        case 3: return fused_md<MC, 3>(a, variant, s);
        case 4: return fused_md<MC, 4>(a, variant, s);
        case 5: return fused_md<MC, 5>(a, variant, s);
    }
    return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_fused(const FusedArgs& a, int variant, cudaStream_t s) {
    if (a.base % kBlockPx) return cudaErrorInvalidValue;  // tiles must be warp-aligned
    switch (a.color.M) {
        case 3: return fused_mc<3>(a, variant, s);
        case 4: return fused_mc<4>(a, variant, s);
        case 5: return fused_mc<5>(a, variant, s);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_near(const FusedArgs& a, float rel, unsigned long long* counts, cudaStream_t s) {
    if (a.n == 0) return cudaSuccess;
    const unsigned nb = blocks_for(a.n);
    const float lc = a.ck.lambda, ld = a.dk.lambda;
    switch (a.color.M) {
        case 3: k_near<3, 3><<<nb, kThreads, 0, s>>>(a.color, a.r, a.g, a.b, a.d, a.base, a.n, lc, rel, counts); break;
        case 4: k_near<4, 3><<<nb, kThreads, 0, s>>>(a.color, a.r, a.g, a.b, a.d, a.base, a.n, lc, rel, counts); break;
        default: k_near<5, 3><<<nb, kThreads, 0, s>>>(a.color, a.r, a.g, a.b, a.d, a.base, a.n, lc, rel, counts); break;
    }
    switch (a.depth.M) {
        case 3: k_near<3, 1><<<nb, kThreads, 0, s>>>(a.depth, a.r, a.g, a.b, a.d, a.base, a.n, ld, rel, counts + 1); break;
        case 4: k_near<4, 1><<<nb, kThreads, 0, s>>>(a.depth, a.r, a.g, a.b, a.d, a.base, a.n, ld, rel, counts + 1); break;
        default: k_near<5, 1><<<nb, kThreads, 0, s>>>(a.depth, a.r, a.g, a.b, a.d, a.base, a.n, ld, rel, counts + 1); break;
    }
    g_launches.fetch_add(2, std::memory_order_relaxed);
    return cudaGetLastError();
}

cudaError_t launch_bank_color(BankView bk, const MixCfg& k, const uint8_t* r, const uint8_t* g,
                              const uint8_t* b, uint8_t* mask, size_t n, cudaStream_t s) {
    switch (bk.M) {
        case 3: return go(k_bank_color<3>, n, s, bk, k, r, g, b, mask, n);
        case 4: return go(k_bank_color<4>, n, s, bk, k, r, g, b, mask, n);
        case 5: return go(k_bank_color<5>, n, s, bk, k, r, g, b, mask, n);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_bank_depth(BankView bk, const MixCfg& k, const uint16_t* d, uint8_t* mask,
                              size_t n, cudaStream_t s) {
    switch (bk.M) {
        case 3: return go(k_bank_depth<3>, n, s, bk, k, d, mask, n);
        case 4: return go(k_bank_depth<4>, n, s, bk, k, d, mask, n);
        case 5: return go(k_bank_depth<5>, n, s, bk, k, d, mask, n);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_bank_aug(BankView bk, const MixCfg& k, const uint8_t* r, const uint8_t* g,
                            const uint8_t* b, const uint16_t* d, float lo, float hi,
                            uint8_t* mask, size_t n, cudaStream_t s) {
    switch (bk.M) {
        case 3: return go(k_bank_aug<3>, n, s, bk, k, r, g, b, d, lo, hi, mask, n);
        case 4: return go(k_bank_aug<4>, n, s, bk, k, r, g, b, d, lo, hi, mask, n);
        case 5: return go(k_bank_aug<5>, n, s, bk, k, r, g, b, d, lo, hi, mask, n);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_bank_reset(BankView bk, float sigma0, size_t n, cudaStream_t s) {
    return go(k_bank_reset, n, s, bk, sigma0, n);
}

cudaError_t launch_bank_gather(BankView bk, int plane, size_t n, void* dst, cudaStream_t s) {
    return go(k_bank_gather, n, s, bk, plane, n, dst);
}

cudaError_t launch_bank_scatter(BankView bk, int plane, size_t n, const void* src, cudaStream_t s) {
    return go(k_bank_scatter, n, s, bk, plane, n, src);
}

inline bool al16(const void* p) { return ((uintptr_t)p & 15u) == 0u; }

cudaError_t launch_fuse(uint8_t* out, int8_t* cpt, const uint8_t* rgb, const uint8_t* dep,
                        uint8_t* out_copy, int limit, size_t n, cudaStream_t s) {
    if (al16(out) && al16(cpt) && al16(rgb) && al16(dep) && (!out_copy || al16(out_copy)))
        return go(k_fuse16, (n + 15) / 16, s, out, cpt, rgb, dep, out_copy, limit, n);
    return go(k_fuse, n, s, out, cpt, rgb, dep, out_copy, limit, n);
}

cudaError_t launch_mix_init(const float* values, int channels, size_t n, const MixCfg& k, int M,
                            PixRec* out, cudaStream_t s) {
    return go(k_mix_init, n, s, values, channels, n, k, M, out);
}

cudaError_t launch_mix_step(PixRec* recs, const float* values, int channels, size_t n,
                            const MixCfg& k, uint8_t* labels, cudaStream_t s) {
    return go(k_mix_step, n, s, recs, values, channels, n, k, labels);
}

cudaError_t launch_mix_op(PixRec* recs, const float* values, size_t n, const MixCfg& k, int op,
                          int* matched, uint8_t* labels, cudaStream_t s) {
    return go(k_mix_op, n, s, recs, values, n, k, op, matched, labels);
}

cudaError_t launch_render(const SceneFrame& sc, uint8_t* r, uint8_t* g, uint8_t* b, uint16_t* d,
                          uint8_t* gt, cudaStream_t s) {
    const size_t n = (size_t)sc.width * sc.height * sc.streams;
    if (n == 0) return cudaSuccess;
    k_render<<<blocks_for(n), kThreads, 0, s>>>(sc, r, g, b, d, gt, n);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
}

cudaError_t launch_register_splat(const uint8_t* mask, const uint16_t* depth, int dw, int dh,
                                  int streams, const RigDev& rig, int cw, int ch, uint8_t* out,
                                  cudaStream_t s) {
    const size_t n = (size_t)dw * dh * streams;
    if (n % 16 == 0 && al16(mask))
        return go(k_register_splat16, n / 16, s, mask, depth, dw, dh, n / 16, rig, cw, ch, out);
    return go(k_register_splat, n, s, mask, depth, dw, dh, n, rig, cw, ch, out);
}

cudaError_t launch_dilate(const uint8_t* in, uint8_t* tmp, uint8_t* out, int w, int h,
                          int streams, int radius, cudaStream_t s) {
    const size_t n = (size_t)w * h * streams;
    if (radius <= 0) {  // dilate_mask returns the mask unchanged
        if (out == in) return cudaSuccess;
        return cudaMemcpyAsync(out, in, n, cudaMemcpyDeviceToDevice, s);
    }
    if (w % 16 == 0 && al16(in) && al16(tmp) && al16(out)) {
        cudaError_t e = radius <= 16 ? go(k_dilate_rows16, n / 16, s, in, tmp, w, n / 16, radius)
                                     : go(k_dilate_pass<true>, n, s, in, tmp, w, h, n, radius);
        if (e != cudaSuccess) return e;
        return go(k_dilate_cols16, n / 16, s, (const uint8_t*)tmp, out, w, h, n / 16, radius);
    }
    cudaError_t e = go(k_dilate_pass<true>, n, s, in, tmp, w, h, n, radius);
    if (e != cudaSuccess) return e;
    return go(k_dilate_pass<false>, n, s, (const uint8_t*)tmp, out, w, h, n, radius);
}

cudaError_t launch_counts_tn(unsigned long long* counts, int streams, int methods,
                            size_t stream_px, cudaStream_t s) {
    const int n = streams * methods;
    if (n <= 0) return cudaSuccess;
    k_counts_tn<<<(n + 127) / 128, 128, 0, s>>>(counts, n, (unsigned long long)stream_px);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
}

cudaError_t launch_confusion(const uint8_t* const* preds, int methods, const uint8_t* gt,
                             size_t npx, size_t stream_px, unsigned long long* counts,
                             cudaStream_t s) {
    if (methods != 1 && methods != 3) return cudaErrorInvalidValue;
    return go(k_confusion, npx, s, preds[0], methods == 3 ? preds[1] : preds[0],
              methods == 3 ? preds[2] : preds[0], methods, gt, npx, stream_px, counts);
}

uint64_t launches() { return g_launches.load(); }

}  // namespace rgbdseg_b200
