/*
 * rgbdseg_c.h -- C-ABI of the B200-native rgbdseg hot path.
 *
 * Drop-in boundary for the reference library's model/segment API
 * (/root/reference/proj/include/rgbdseg/*.hpp).  Plain pointers and sizes
 * only; no C++ or torch types.  Every entry point names the reference
 * interface it replaces.  The library (librgbdseg_b200.so) owns all device
 * memory; callers own host buffers.
 *
 * Memory: every frame/mask pointer may be host memory (pageable or pinned) or
 * device memory of the handle's GPU; the library classifies each pointer with
 * cudaPointerGetAttributes and moves data accordingly.
 *
 * Stream ordering: the library runs on its own non-blocking CUDA streams,
 * which are NOT ordered with the legacy default stream.  Device inputs must
 * be complete before a call reads them: synchronous calls (bank, fusion,
 * registration, process) need the producer finished; the asynchronous
 * processor path can instead order itself after a caller's stream with
 * rgbdseg_processor_wait_stream and publish its results to a caller's stream
 * with rgbdseg_processor_signal_stream.  Bank and fusion handles borrowed from
 * a processor drain the processor's queued frames before every call.
 *
 * Errors: functions return an rgbdseg_status; rgbdseg_last_error() returns a
 * thread-local message for the last failing call on this thread.
 *   RGBDSEG_EINVAL  <-> std::invalid_argument in the reference (bad config,
 *                       dimension or mode mismatch: plane.hpp:53-58,
 *                       mixture.cpp:9-24, segmenter.cpp:74-75,109-125,
 *                       fusion.cpp:8-9)
 *   RGBDSEG_ECUDA / ENOMEM / ERUNTIME  <-> std::runtime_error
 *
 * Threading: a handle is not thread-safe (the reference banks/processors are
 * not either, processor.hpp:57-59).  Handles on different GPUs are independent.
 */
#ifndef RGBDSEG_C_H
#define RGBDSEG_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    RGBDSEG_OK = 0,
    RGBDSEG_EINVAL = 1,
    RGBDSEG_ECUDA = 2,
    RGBDSEG_ENOMEM = 3,
    RGBDSEG_ERUNTIME = 4
} rgbdseg_status;

/* Bank modes, segmenter.hpp:11 */
enum { RGBDSEG_COLOR3 = 0, RGBDSEG_DEPTH1 = 1, RGBDSEG_AUGMENTED4 = 2 };

/* MixtureConfig, mixture.hpp:16-26 -- same fields, same order, same defaults
 * (rgbdseg_mixture_defaults). */
typedef struct rgbdseg_mixture_cfg {
    int components;             /* M in [3,5] */
    float learning_rate;        /* alpha in (0,1) */
    float match_lambda;         /* lambda > 0 */
    float background_threshold; /* T in (0,1) */
    float initial_sigma;        /* sigma_0 > 0 */
    float initial_weight;       /* w_new in (0,1) */
    float variance_floor;       /* > 0 */
} rgbdseg_mixture_cfg;

/* PixelMixture, mixture.hpp:30-41: means[i*channels + c]. */
typedef struct rgbdseg_pixel_mixture {
    int components;
    int channels;
    float means[20];
    float variances[5];
    float weights[5];
} rgbdseg_pixel_mixture;

typedef struct rgbdseg_bank rgbdseg_bank;
typedef struct rgbdseg_fusion rgbdseg_fusion;
typedef struct rgbdseg_processor rgbdseg_processor;

/* ---- library ---------------------------------------------------------- */
const char* rgbdseg_last_error(void);
const char* rgbdseg_version(void);
/* Number of kernel launches this process has issued through the library. */
uint64_t rgbdseg_launch_count(void);

/* ---- config: MixtureConfig::validate, mixture.cpp:9-24 ----------------- */
void rgbdseg_mixture_defaults(rgbdseg_mixture_cfg* out); /* mixture.hpp:17-23 */
int rgbdseg_mixture_validate(const rgbdseg_mixture_cfg* cfg);

/* ---- per-pixel API: mixture.hpp:43-60, run on the GPU ------------------
 * Batched over n independent records (AoS, host or device memory).
 * init: values[n*channels] -> out[n]                (init_mixture)
 * step: mix[n] updated in place, labels[n] 1=FG      (step_pixel); like
 *       the reference, step uses each record's own `components` for the
 *       loops and cfg only for the rates; every record must have
 *       `channels` channels and 3..5 components, else RGBDSEG_EINVAL.    */
int rgbdseg_init_mixtures(const float* values, int channels, size_t n,
                          const rgbdseg_mixture_cfg* cfg, rgbdseg_pixel_mixture* out,
                          int device);
int rgbdseg_step_mixtures(rgbdseg_pixel_mixture* mix, const float* values, int channels,
                          size_t n, const rgbdseg_mixture_cfg* cfg, uint8_t* labels, int device);

/* The three pieces of step_pixel on their own, batched over n records:
 * match_component (mixture.cpp:74-92) -> matched[n]: the component index,
 *   or -1 for std::nullopt;
 * classify (mixture.cpp:133-146) of each record's matched[i] (-1 = nullopt)
 *   -> labels[n], 1 = Foreground;
 * update_mixture (mixture.cpp:94-131) with each record's matched[i], in
 *   place.
 * Like the reference these use each record's own components / channels and
 * do not validate cfg; records must have 3..5 components and (match,
 * update) `channels` channels, matched[i] must be -1 or a component index
 * (the reference's behaviour is undefined otherwise), else RGBDSEG_EINVAL
 * before anything changes. */
int rgbdseg_match_components(const rgbdseg_pixel_mixture* mix, const float* values, int channels,
                             size_t n, const rgbdseg_mixture_cfg* cfg, int32_t* matched,
                             int device);
int rgbdseg_classify_mixtures(const rgbdseg_pixel_mixture* mix, const int32_t* matched, size_t n,
                              const rgbdseg_mixture_cfg* cfg, uint8_t* labels, int device);
int rgbdseg_update_mixtures(rgbdseg_pixel_mixture* mix, const float* values, int channels,
                            size_t n, const int32_t* matched, const rgbdseg_mixture_cfg* cfg,
                            int device);

/* ---- ModelBank: segmenter.hpp:25-55 ------------------------------------
 * Device-resident bank over `npx` = width*height*streams pixels (streams
 * back to back).  Plane ids follow ModelBank's plane order
 * (segmenter.hpp:51-54): mean(i,c) = i*C + c ; variance(i) = M*C + i ;
 * weight(i) = M*C + M + i ; the initialised-flag plane (uint8) is
 * RGBDSEG_FLAGS_PLANE.  In HBM the planes are TILED: blocks of 32 pixels,
 * each holding the 32 values of every plane in turn, then the 32 flag words
 * in a 128-byte slot -- see rgbdseg_bank_device_ptrs. */
#define RGBDSEG_FLAGS_PLANE (-1)
int rgbdseg_bank_create(int width, int height, int streams, int mode,
                        const rgbdseg_mixture_cfg* cfg, int device, rgbdseg_bank** out);
void rgbdseg_bank_destroy(rgbdseg_bank* bank);
int rgbdseg_bank_planes(const rgbdseg_bank* bank); /* M*C + 2M */
/* Copy one flat plane (npx elements; float, or uint8 for the flag plane;
 * host or device memory) out of / into the bank.  Backs mean_plane /
 * variance_plane / weight_plane / initialized_plane, gather/scatter and
 * state_equals (segmenter.hpp:33-46). */
int rgbdseg_bank_download(const rgbdseg_bank* bank, int plane, void* dst);
int rgbdseg_bank_upload(rgbdseg_bank* bank, int plane, const void* src);
/* Raw tiled storage: `nblocks` blocks of `block_bytes` = (planes+1)*128
 * bytes; value of plane p for pixel j is float[(j/32)*(block_bytes/4) +
 * p*32 + j%32]; its flag word is uint16 j%32 from float offset planes*32 of
 * the block: low byte = initialised flag, high byte = untouched-component
 * mask (bit i: component i still holds its init_mixture values, mean 0,
 * variance initial_sigma^2 of the bank's creation cfg, weight 0; the kernels
 * then skip reading it).  A caller that writes planes through this pointer
 * must clear the high byte of the pixels it changes. */
int rgbdseg_bank_device_ptrs(const rgbdseg_bank* bank, void** tiles, size_t* block_bytes,
                             size_t* nblocks);

/* segment_color, segmenter.cpp:107-119 / segment_depth, :121-131.
 * Planes are npx elements, row-major, streams back to back.  mask_out may be
 * NULL (state update only).  Synchronous like the reference. */
int rgbdseg_segment_color(rgbdseg_bank* bank, const uint8_t* r, const uint8_t* g,
                          const uint8_t* b, const rgbdseg_mixture_cfg* cfg, uint8_t* mask_out);
int rgbdseg_segment_depth(rgbdseg_bank* bank, const uint16_t* depth_mm,
                          const rgbdseg_mixture_cfg* cfg, uint8_t* mask_out);

/* segment_augmented, segmenter.cpp:133-147: one 4-channel mixture over
 * (R, G, B, DepthRescale{min_mm, max_mm}.to_channel(depth)); no depth
 * sentinel.  min_mm < max_mm (RunConfig::validate, processor.cpp:56-57). */
int rgbdseg_segment_augmented(rgbdseg_bank* bank, const uint8_t* r, const uint8_t* g,
                              const uint8_t* b, const uint16_t* depth_mm, float min_mm,
                              float max_mm, const rgbdseg_mixture_cfg* cfg, uint8_t* mask_out);

/* ---- FusionState / reset_state / fuse_step: fusion.hpp:11-23 ----------- */
int rgbdseg_fusion_create(int width, int height, int streams, int initial_label,
                          int counter_limit, int device, rgbdseg_fusion** out);
void rgbdseg_fusion_destroy(rgbdseg_fusion* fs);
/* out_copy (may be NULL) receives the fused mask (= state.out). */
int rgbdseg_fusion_step(rgbdseg_fusion* fs, const uint8_t* rgb_mask, const uint8_t* depth_mask,
                        uint8_t* out_copy);
int rgbdseg_fusion_download(const rgbdseg_fusion* fs, uint8_t* out, int8_t* cpt);
/* FusionState::counter_limit is a plain field the reference reads at every
 * fuse_step (fusion.cpp:24): set it between steps (no validation, like the
 * reference's fuse_step). */
int rgbdseg_fusion_set_counter_limit(rgbdseg_fusion* fs, int counter_limit);
int rgbdseg_fusion_upload(rgbdseg_fusion* fs, const uint8_t* out, const int8_t* cpt);

/* ---- CameraRig / register_mask / dilate_mask: registration.hpp:10-38 -----
 * Depth->colour registration for unregistered sequences (processor.cpp:175-179):
 * back-project each valid foreground depth pixel, apply (R, t), project with
 * lround into the colour grid, splat, then a square dilation of radius r.
 * Same fp64 arithmetic as the reference, bit-identical masks. */
typedef struct rgbdseg_camera_rig {
    double depth_fx, depth_fy, depth_cx, depth_cy; /* Pinhole depth_cam */
    double color_fx, color_fy, color_cx, color_cy; /* Pinhole color_cam */
    double rotation[9];                            /* row-major */
    double translation_mm[3];
    double depth_scale;                            /* mm per raw depth unit */
} rgbdseg_camera_rig;

/* CameraRig::identity(fx, fy, cx, cy), registration.cpp:28-33 */
void rgbdseg_camera_rig_identity(rgbdseg_camera_rig* rig, double fx, double fy, double cx,
                                 double cy);
/* CameraRig::validate, registration.cpp:10-26 (same messages) */
int rgbdseg_camera_rig_validate(const rgbdseg_camera_rig* rig);
/* register_mask(mask, depth, rig, cw, ch, radius), registration.cpp:50-78.
 * mask/depth: dw*dh (host or device); out: cw*ch.  Synchronous. */
int rgbdseg_register_mask(const uint8_t* depth_mask, const uint16_t* depth_raw, int dw, int dh,
                          const rgbdseg_camera_rig* rig, int cw, int ch, int dilation_radius,
                          uint8_t* out, int device);
/* dilate_mask(mask, radius), registration.cpp:33-48.  Synchronous. */
int rgbdseg_dilate_mask(const uint8_t* mask, int w, int h, int radius, uint8_t* out, int device);

/* ---- SequenceProcessor: processor.hpp:60-80, process = processor.cpp:158-184
 * Fused method on a registered sequence: colour bank + depth bank + List-1
 * fusion, executed as ONE kernel per frame batch over `streams` independent
 * camera streams of width x height (state never leaves HBM, masks never
 * round-trip HBM).                                                        */
typedef struct rgbdseg_processor_cfg {
    int width, height;
    int streams;           /* independent camera streams batched per step */
    rgbdseg_mixture_cfg color;
    rgbdseg_mixture_cfg depth;
    int fusion_counter_limit; /* >= 1 (fusion.cpp:8); <= 127, cpt is int8 */
    int fusion_initial_label; /* 0 or 1 */
    int device;
    int host_chunks;       /* 0 = auto: H2D/compute/D2H overlap chunks for host frames */
    int registered;        /* 1 (default): depth already in the colour grid */
    rgbdseg_camera_rig rig; /* used when registered == 0 (must validate) */
    int dilation_radius;   /* >= 0, default 1 (processor.hpp:26) */
} rgbdseg_processor_cfg;

void rgbdseg_processor_defaults(rgbdseg_processor_cfg* cfg, int width, int height);
int rgbdseg_processor_create(const rgbdseg_processor_cfg* cfg, rgbdseg_processor** out);
void rgbdseg_processor_destroy(rgbdseg_processor* p);

/* One frame step for all streams.  Inputs: r, g, b (uint8) and depth (uint16,
 * raw millimetres, 0 = no return), npx elements each, host or device.
 * Outputs (any may be NULL): fused mask, colour mask, depth mask.
 * rgbdseg_processor_process is synchronous (reference semantics);
 * rgbdseg_processor_submit only enqueues -- buffers must stay valid until
 * rgbdseg_processor_sync returns. */
int rgbdseg_processor_process(rgbdseg_processor* p, const uint8_t* r, const uint8_t* g,
                              const uint8_t* b, const uint16_t* depth, uint8_t* fused_out,
                              uint8_t* rgb_out, uint8_t* depth_out);
int rgbdseg_processor_submit(rgbdseg_processor* p, const uint8_t* r, const uint8_t* g,
                             const uint8_t* b, const uint16_t* depth, uint8_t* fused_out,
                             uint8_t* rgb_out, uint8_t* depth_out);
int rgbdseg_processor_sync(rgbdseg_processor* p);
/* The same step from an INTERLEAVED colour frame: `rgb` holds 3 bytes per
 * pixel (npx * 3, streams back to back) in R,G,B order (the layout
 * aos_to_soa consumes, engine.cpp:39-56) or B,G,R (OpenCV / Kinect
 * capture order); the kernel deinterleaves it in its first load round, so
 * no host shuffle precedes the upload.  A host buffer holding the packed
 * colour plane immediately followed by the depth plane moves in one DMA. */
enum { RGBDSEG_ORDER_RGB = 0, RGBDSEG_ORDER_BGR = 1 };
int rgbdseg_processor_submit_interleaved(rgbdseg_processor* p, const uint8_t* rgb, int order,
                                         const uint16_t* depth, uint8_t* fused_out,
                                         uint8_t* rgb_out, uint8_t* depth_out);
int rgbdseg_processor_process_interleaved(rgbdseg_processor* p, const uint8_t* rgb, int order,
                                          const uint16_t* depth, uint8_t* fused_out,
                                          uint8_t* rgb_out, uint8_t* depth_out);
/* The same step plus the evaluation epilogue (confusion_counts,
 * eval.cpp:11-31, fused into the kernel): gt = ground-truth mask planes
 * (npx, {0,1}); counts receives int64 [streams][rgb, depth, fused][tp, fp,
 * tn, fn] for this frame (host or device memory; valid after sync). */
int rgbdseg_processor_process_eval(rgbdseg_processor* p, const uint8_t* r, const uint8_t* g,
                                   const uint8_t* b, const uint16_t* depth, const uint8_t* gt,
                                   int64_t* counts, uint8_t* fused_out, uint8_t* rgb_out,
                                   uint8_t* depth_out);
int rgbdseg_processor_submit_eval(rgbdseg_processor* p, const uint8_t* r, const uint8_t* g,
                                  const uint8_t* b, const uint16_t* depth, const uint8_t* gt,
                                  int64_t* counts, uint8_t* fused_out, uint8_t* rgb_out,
                                  uint8_t* depth_out);
int64_t rgbdseg_processor_frames(const rgbdseg_processor* p);
/* Borrow the processor's banks / fusion state (owned by the processor):
 * color_bank()/depth_bank(), processor.hpp:67-68. */
rgbdseg_bank* rgbdseg_processor_color_bank(rgbdseg_processor* p);
rgbdseg_bank* rgbdseg_processor_depth_bank(rgbdseg_processor* p);
rgbdseg_fusion* rgbdseg_processor_fusion(rgbdseg_processor* p);
/* The CUDA stream the processor's kernels run on (cudaStream_t as void*),
 * so callers can time the kernels with events on the launching stream. */
void* rgbdseg_processor_stream(rgbdseg_processor* p);
/* Order the processor's next submits after all work queued so far on
 * `stream` (cudaStream_t as void*, NULL = legacy default stream), and make
 * `stream` wait for everything the processor has queued so far. */
int rgbdseg_processor_wait_stream(rgbdseg_processor* p, void* stream);
int rgbdseg_processor_signal_stream(rgbdseg_processor* p, void* stream);
/* Kernel variant: 0 = auto (2 for launches under 4 occupancy waves, else 3),
 * 1 = dense: reads and writes back every state word, 2 = elided: reads only
 * the components the flag words mark as touched, runs the step on the warp's
 * touched prefix and rewrites only the words whose bits changed, 3 = elided
 * with colour components 0..1 prefetched into L1 in the first load round and
 * read at the colour step (fewer registers live through the depth step).
 * Every variant produces the same bits; they differ only in HBM traffic,
 * instruction count and register use. */
int rgbdseg_processor_set_variant(rgbdseg_processor* p, int variant);
/* Near-threshold report (north_star's parity accounting).  With rel > 0,
 * every later step first counts -- on the state before the step, in a
 * separate read-only kernel -- the colour and the depth pixels whose
 * observation lies within rel * lambda*sigma of a component's match band
 * in some channel (| |v_c - mu_ic| - lambda*sigma_i | <= rel*lambda*sigma_i,
 * mixture.cpp:80-84): the pixels a non-bit-exact build could flip.  Setting
 * it (rel = 0 turns it off) zeroes the counters; counts returns the colour
 * and depth totals and the pixel-frames examined since. */
int rgbdseg_processor_set_near_threshold(rgbdseg_processor* p, float rel);
int rgbdseg_processor_near_threshold_counts(rgbdseg_processor* p, uint64_t* color,
                                            uint64_t* depth, uint64_t* pixel_frames);

/* ---- evaluation: confusion_counts, eval.cpp:11-31 ------------------------
 * pred/gt: npx mask bytes ({0,1}, host or device) split into `streams` equal
 * frames; counts: int64 [streams][tp, fp, tn, fn].  Synchronous. */
int rgbdseg_confusion_counts(const uint8_t* pred, const uint8_t* gt, size_t npx, int streams,
                             int64_t* counts, int device);

/* ---- synthetic scenes on the GPU (synthetic.cpp:119-195, harness) ------
 * Renders builtin scenario `name` ('A' or 'B'), frame `frame`, for `streams`
 * streams whose seeds are seed0 + s, directly into device planes (npx each).
 * Scenario geometry is the builtin 640x480 one unless width/height differ,
 * in which case events and the object keep their builtin pixel coordinates. */
int rgbdseg_render_scenario(char name, int width, int height, int streams, uint64_t seed0,
                            int frame, uint8_t* r, uint8_t* g, uint8_t* b, uint16_t* depth,
                            uint8_t* gt, int device, void* stream);

/* One frame of an arbitrary ScenarioSpec (synthetic.hpp:61-74), resolved on
 * the host for that frame index exactly as render_frame does
 * (synthetic.cpp:124-134): the illumination gain product, each object's
 * lround'ed waypoint position, and only the shadow / flicker events active
 * in this frame (in spec order).  At most 4 objects and 16 events of each
 * kind.  Streams s render with seed seed0 + s. */
typedef struct rgbdseg_scene_frame {
    int width, height, streams;
    uint64_t seed0;
    int frame;
    int base_depth_mm, depth_texture_mm, color_texture;
    double gain;
    int n_obj;
    int obj_rect[4][4]; /* x, y, w, h */
    int obj_color[4][3];
    int obj_depth_offset_mm[4];
    int n_shadow;
    int shadow_rect[16][4];
    double shadow_darken[16];
    int n_flicker;
    int flicker_rect[16][4];
    double flicker_color_sigma[16], flicker_depth_sigma_mm[16];
    double noise_color_sigma, noise_depth_sigma_mm;
} rgbdseg_scene_frame;

int rgbdseg_render_frame(const rgbdseg_scene_frame* frame, uint8_t* r, uint8_t* g, uint8_t* b,
                         uint16_t* depth, uint8_t* gt, int device, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* RGBDSEG_C_H */
