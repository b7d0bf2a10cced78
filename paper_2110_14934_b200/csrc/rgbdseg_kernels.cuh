// rgbdseg_kernels.cuh -- launch interface between the C-ABI host runtime
// (rgbdseg_capi.cu) and the sm_100a kernels (rgbdseg_kernels.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "gmm_pixel.cuh"

namespace rgbdseg_b200 {

// Device layout of one bank: TILED structure-of-arrays.  Pixels are grouped
// in blocks of 32 (one warp); block b stores, for its 32 pixels, float plane
// 0..NP-1 of ModelBank's plane order (segmenter.hpp:51-54: mean(i,c) = i*C+c,
// variance(i) = M*C+i, weight(i) = M*C+M+i) as 32 consecutive floats each,
// then one 128-byte slot whose first 64 bytes are the pixels' flag words
// (uint16): low byte = ModelBank's initialised flag (the value the reference
// stores), high byte = UNTOUCHED mask, bit i set <=> component i still holds
// exactly its init_mixture values (mean +0 in every channel, variance =
// BankView::vvar, weight +0; mixture.cpp:58-72).  The mask is a cache of
// known state, never a change of it: the planes always hold the full
// reference state, and K1 substitutes the known values for untouched
// components instead of reading them (most slots of a mixture are untouched
// for hundreds of frames).  Every kernel that writes a component clears its
// bit; upload clears the pixel's mask.
// A warp's access to one plane is still one full 128-byte line (SoA
// coalescing), but every plane of a pixel sits at an
// immediate offset p*128 from one per-thread address, so the kernels issue
// no per-plane 64-bit address arithmetic.  bank_download/upload gather and
// scatter the reference's flat planes.
constexpr int kBlockPx = 32;

__host__ __device__ constexpr int bank_planes(int M, int C) { return M * C + 2 * M; }
__host__ __device__ constexpr int bank_stride(int M, int C) {  // floats per block
    return (bank_planes(M, C) + 1) * kBlockPx;
}

struct BankView {
    float* state;  // nblocks * bank_stride(M, C) floats
    int M;
    int C;
    float vvar;  // variance of an untouched component: sigma0^2 of the bank's creation cfg
    int vinit;   // this call's init_mixture may mark components untouched
                 // (its sigma0^2 == vvar and vvar is in the fast step's range)
};

// Untouched-mask bits of components 1..M-1 (component 0 is set by init).
__host__ __device__ constexpr uint32_t untouched_all(int M) { return ((1u << M) - 1u) & ~1u; }

struct FusedArgs {
    // inputs for pixels [0, n) of this launch (pre-offset by the caller)
    const uint8_t* r;
    const uint8_t* g;
    const uint8_t* b;
    const uint16_t* d;
    // optional mask outputs (pre-offset), may be null
    uint8_t* rgb_mask;
    uint8_t* depth_mask;
    uint8_t* fused_copy;
    // state: pixel i of this launch is pixel base + i of the banks
    BankView color;
    BankView depth;
    uint8_t* out;  // fusion state (already offset by base)
    int8_t* cpt;
    size_t base;
    size_t n;
    MixCfg ck;
    MixCfg dk;
    int limit;
    int fuse;  // 0: unregistered sequence -- write rgb/depth masks, fuse after registration
    // optional evaluation epilogue (confusion_counts, eval.cpp:11-31): ground
    // truth for pixels [0, n) and per-stream int64 counters
    // [stream][method rgb, depth, fused][tp, fp, tn, fn]; stream of pixel
    // base+i is (base+i) / stream_px.
    const uint8_t* gt;
    unsigned long long* counts;
    size_t stream_px;
    // L2 prefetch distance in thread blocks (0 = off): each warp prefetches
    // the bank tiles of the warp `ahead` blocks later (~one occupancy wave)
    unsigned ahead;
    // interleaved colour input: `r` is ONE plane of 3 bytes per pixel
    // (pre-offset by 3*base), R,G,B order (bgr = 0) or B,G,R (bgr = 1);
    // g and b are unused.  Not combined with the evaluation epilogue.
    int packed;
    int bgr;
};

// Kernel variants of K1 (identical results; they differ in HBM traffic and
// register use).  A TMA cp.async.bulk staging variant was
// measured and dropped (profiles/variants_r01.json).
// Auto = elided, in its L1 form (colour components 0..1 through L1, not held
// in registers) for launches of at least RGBDSEG_L1_MIN_WAVES occupancy
// waves; kLdgElide / kLdgElideL1 force one form (tests, A/B).
enum Variant { kAuto = 0, kLdgDense = 1, kLdgElide = 2, kLdgElideL1 = 3 };

// All launchers return cudaGetLastError() after the launch.
cudaError_t launch_fused(const FusedArgs& a, int variant, cudaStream_t s);
// Near-threshold report (diagnostic, read-only): adds to counts[0] the colour
// pixels and to counts[1] the depth pixels of launch `a` whose observation
// lies within rel * lambda*sigma of a component's match band, on the state
// before the step.  Launch it before launch_fused(a) on the same stream.
cudaError_t launch_near(const FusedArgs& a, float rel, unsigned long long* counts, cudaStream_t s);
cudaError_t launch_bank_color(BankView bank, const MixCfg& k, const uint8_t* r, const uint8_t* g,
                              const uint8_t* b, uint8_t* mask, size_t n, cudaStream_t s);
cudaError_t launch_bank_depth(BankView bank, const MixCfg& k, const uint16_t* d, uint8_t* mask,
                              size_t n, cudaStream_t s);
cudaError_t launch_bank_aug(BankView bank, const MixCfg& k, const uint8_t* r, const uint8_t* g,
                            const uint8_t* b, const uint16_t* d, float lo, float hi,
                            uint8_t* mask, size_t n, cudaStream_t s);
cudaError_t launch_bank_reset(BankView bank, float sigma0, size_t n, cudaStream_t s);
// plane = ModelBank plane id, or -1 for the initialised flags (uint8).  dst/src:
// npx elements.  A scatter clears the scattered pixels' untouched masks.
cudaError_t launch_bank_gather(BankView bank, int plane, size_t n, void* dst, cudaStream_t s);
cudaError_t launch_bank_scatter(BankView bank, int plane, size_t n, const void* src, cudaStream_t s);
cudaError_t launch_fuse(uint8_t* out, int8_t* cpt, const uint8_t* rgb, const uint8_t* dep,
                        uint8_t* out_copy, int limit, size_t n, cudaStream_t s);

// Per-pixel API over AoS records (rgbdseg_pixel_mixture layout).
struct PixRec {
    int components;
    int channels;
    float means[20];
    float variances[5];
    float weights[5];
};
cudaError_t launch_mix_init(const float* values, int channels, size_t n, const MixCfg& k,
                            int M, PixRec* out, cudaStream_t s);
// labels: 0/1, or 255 for a record whose shape the kernel cannot step.
cudaError_t launch_mix_step(PixRec* recs, const float* values, int channels, size_t n,
                            const MixCfg& k, uint8_t* labels, cudaStream_t s);

// match_component / classify / update_mixture batched over records
// (mixture.hpp:45-56): op kOpMatch writes matched[j] (-1 = no match),
// kOpClassify reads matched[j] and writes labels[j] (1 = FG), kOpUpdate
// reads matched[j] and values (n * channels) and updates the record.
enum { kOpMatch = 0, kOpClassify = 1, kOpUpdate = 2 };
cudaError_t launch_mix_op(PixRec* recs, const float* values, size_t n, const MixCfg& k, int op,
                          int* matched, uint8_t* labels, cudaStream_t s);

// Synthetic scene for one frame (frame-level quantities resolved on the host).
struct SceneFrame {
    int width, height, streams;
    uint64_t seed0;
    int frame;
    int base_depth_mm, depth_texture_mm, color_texture;
    double gain;
    int n_obj;
    int orect[4][4];
    int ocolor[4][3];
    int odepth[4];
    int n_shadow;
    int srect[16][4];
    double sdarken[16];
    int n_flicker;
    int frect[16][4];
    double fcs[16], fds[16];
    double ncs, nds;
};
cudaError_t launch_render(const SceneFrame& sc, uint8_t* r, uint8_t* g, uint8_t* b, uint16_t* d,
                          uint8_t* gt, cudaStream_t s);

// Depth->colour registration (registration.cpp:50-78), fp64 exactly as the
// reference evaluates it.  Rig fields as in CameraRig (registration.hpp:16-26).
struct RigDev {
    double dfx, dfy, dcx, dcy;  // depth pinhole
    double cfx, cfy, ccx, ccy;  // colour pinhole
    double R[9];                // row-major rotation
    double t[3];                // translation (mm)
    double scale;               // depth_scale (mm per raw unit)
};
// Splat every valid foreground depth pixel of `streams` frames (dw x dh) into
// zeroed colour-grid masks (cw x ch); idempotent byte stores.
cudaError_t launch_register_splat(const uint8_t* mask, const uint16_t* depth, int dw, int dh,
                                  int streams, const RigDev& rig, int cw, int ch, uint8_t* out,
                                  cudaStream_t s);
// Square binary dilation of radius r (dilate_mask, registration.cpp:33-48) as
// a row pass then a column pass (exact for a square structuring element with
// the reference's border clipping).  tmp: scratch of the same size.
cudaError_t launch_dilate(const uint8_t* in, uint8_t* tmp, uint8_t* out, int w, int h,
                          int streams, int radius, cudaStream_t s);

// confusion_counts (eval.cpp:11-31) of `methods` prediction planes against gt
// over npx pixels, accumulated into counts[stream][method][tp, fp, tn, fn].
cudaError_t launch_confusion(const uint8_t* const* preds, int methods, const uint8_t* gt,
                             size_t npx, size_t stream_px, unsigned long long* counts,
                             cudaStream_t s);

// TN = stream_px - TP - FP - FN for counts[streams][methods][tp, fp, tn, fn]
// (the kernels above count TP / FP / FN only); run after a frame's launches.
cudaError_t launch_counts_tn(unsigned long long* counts, int streams, int methods,
                            size_t stream_px, cudaStream_t s);

uint64_t launches();

}  // namespace rgbdseg_b200
