// integration/rgbdseg_b200_dropin.hpp -- source-compatible C++ drop-in for
// the reference's model/segment API, compiled INSIDE the reference project
// against its own headers (include/rgbdseg/*.hpp) and linked to
// librgbdseg_b200.so (include/rgbdseg_c.h).
//
//   reference (CPU)                      drop-in (B200)
//   rgbdseg::ModelBank                   rgbdseg::b200::ModelBank        segmenter.hpp:25-55
//   rgbdseg::segment_color/_depth/       rgbdseg::b200::segment_color/   segmenter.hpp:60-69
//            _augmented                           _depth/_augmented
//   rgbdseg::FusionState, reset_state,   rgbdseg::b200::FusionState,     fusion.hpp:11-23
//            fuse_step                            reset_state, fuse_step
//   rgbdseg::SequenceProcessor           rgbdseg::b200::SequenceProcessor processor.hpp:60-80
//   rgbdseg::init_mixture, match_        rgbdseg::b200::init_mixture,    mixture.hpp:43-60
//            component, update_mixture,           match_component, ... (+ batched
//            classify, step_pixel                 *_mixtures forms over spans)
//
// Same signatures, argument meaning, return types and exception types
// (std::invalid_argument with the reference's messages), so a call site
// switches by namespace alone: `using rgbdseg::b200::SequenceProcessor;`
// makes acceptance.cpp's run_scenario (acceptance.cpp:143-174) compile
// unchanged (integration/scenario_test.cpp builds it from the reference's own
// text).  What differs is where the state lives: banks and fusion state stay
// in HBM, and the host views the reference hands out by reference
// (ModelBank::mean_plane & co., SequenceProcessor::color_bank()) are host
// mirrors, refreshed from the device on access after any GPU step and
// written back to the device before the next one.  A reference held across a
// GPU step therefore shows the pre-step values until the next accessor call.
#pragma once

#include <cstring>
#include <memory>
#include <optional>
#include <stdexcept>
#include <span>
#include <string>
#include <vector>

#include "rgbdseg/processor.hpp"
#include "rgbdseg_c.h"

namespace rgbdseg::b200 {

inline void check(int rc) {
    if (rc == RGBDSEG_OK) return;
    if (rc == RGBDSEG_EINVAL) throw std::invalid_argument(rgbdseg_last_error());
    throw std::runtime_error(rgbdseg_last_error());
}

inline rgbdseg_mixture_cfg to_c(const MixtureConfig& m) {
    return rgbdseg_mixture_cfg{m.components,     m.learning_rate, m.match_lambda,
                               m.background_threshold, m.initial_sigma, m.initial_weight,
                               m.variance_floor};
}

inline int to_c(BankMode m) {
    return m == BankMode::Color3 ? RGBDSEG_COLOR3
                                 : (m == BankMode::Depth1 ? RGBDSEG_DEPTH1 : RGBDSEG_AUGMENTED4);
}

// Device bank <-> a reference ModelBank through its mutable plane accessors
// (segmenter.hpp:33-37; plane ids in ModelBank order).
inline void download_into(const rgbdseg_bank* dev, rgbdseg::ModelBank& host) {
    const int C = host.channels(), M = host.components();
    for (int i = 0; i < M; ++i) {
        for (int c = 0; c < C; ++c)
            check(rgbdseg_bank_download(dev, i * C + c, host.mean_plane(i, c).data()));
        check(rgbdseg_bank_download(dev, M * C + i, host.variance_plane(i).data()));
        check(rgbdseg_bank_download(dev, M * C + M + i, host.weight_plane(i).data()));
    }
    check(rgbdseg_bank_download(dev, RGBDSEG_FLAGS_PLANE, host.initialized_plane().data()));
}

inline void upload_from(rgbdseg_bank* dev, rgbdseg::ModelBank& host) {
    const int C = host.channels(), M = host.components();
    for (int i = 0; i < M; ++i) {
        for (int c = 0; c < C; ++c)
            check(rgbdseg_bank_upload(dev, i * C + c, host.mean_plane(i, c).data()));
        check(rgbdseg_bank_upload(dev, M * C + i, host.variance_plane(i).data()));
        check(rgbdseg_bank_upload(dev, M * C + M + i, host.weight_plane(i).data()));
    }
    check(rgbdseg_bank_upload(dev, RGBDSEG_FLAGS_PLANE, host.initialized_plane().data()));
}

// A host mirror of a device bank: `valid` while it equals the device state,
// `dirty` once the caller may have written through a mutable accessor.
class BankMirror {
public:
    BankMirror(int w, int h, BankMode mode, const MixtureConfig& cfg)
        : w_(w), h_(h), mode_(mode), cfg_(cfg) {}

    // Reading view (downloads after a device step).
    const rgbdseg::ModelBank& view(const rgbdseg_bank* dev) const {
        refresh(dev);
        return *host_;
    }
    // Writable view: the device copy is refreshed from it before the next step.
    rgbdseg::ModelBank& edit(const rgbdseg_bank* dev) {
        refresh(dev);
        dirty_ = true;
        return *host_;
    }
    // Before a device step: push host edits, then mark the mirror stale.
    void before_step(rgbdseg_bank* dev) {
        if (dirty_) upload_from(dev, *host_);
        dirty_ = false;
        valid_ = false;
    }
    void invalidate() { valid_ = false; }

private:
    void refresh(const rgbdseg_bank* dev) const {
        if (!host_) host_ = std::make_unique<rgbdseg::ModelBank>(w_, h_, mode_, cfg_);
        if (!valid_) download_into(dev, *host_);
        valid_ = true;
    }
    int w_, h_;
    BankMode mode_;
    MixtureConfig cfg_;
    mutable std::unique_ptr<rgbdseg::ModelBank> host_;
    mutable bool valid_ = false;
    bool dirty_ = false;
};

// ------------------------------------------------------------------ ModelBank
// segmenter.hpp:25-55 over a device-resident bank (constructor state:
// segmenter.cpp:24-34, the reference's messages on bad arguments).
class ModelBank {
public:
    ModelBank(int width, int height, BankMode mode, const MixtureConfig& config, int device = 0)
        : width_(width), height_(height), mode_(mode), config_(config), device_(device),
          mirror_(width, height, mode, config) {
        if (width <= 0 || height <= 0) throw std::invalid_argument("Plane: non-positive dimensions");
        const rgbdseg_mixture_cfg c = to_c(config);
        check(rgbdseg_bank_create(width, height, 1, to_c(mode), &c, device, &dev_));
    }
    ModelBank(const ModelBank& o) : ModelBank(o.width_, o.height_, o.mode_, o.config_, o.device_) {
        rgbdseg::ModelBank copy = o.mirror_.view(o.dev_);
        upload_from(dev_, copy);
    }
    ModelBank& operator=(const ModelBank&) = delete;
    ~ModelBank() { rgbdseg_bank_destroy(dev_); }

    int width() const { return width_; }
    int height() const { return height_; }
    BankMode mode() const { return mode_; }
    int components() const { return config_.components; }
    int channels() const { return bank_channels(mode_); }

    Plane<float>& mean_plane(int component, int channel) {
        return mirror_.edit(dev_).mean_plane(component, channel);
    }
    Plane<float>& variance_plane(int component) { return mirror_.edit(dev_).variance_plane(component); }
    Plane<float>& weight_plane(int component) { return mirror_.edit(dev_).weight_plane(component); }
    Plane<uint8_t>& initialized_plane() { return mirror_.edit(dev_).initialized_plane(); }

    PixelMixture gather(int x, int y) const { return mirror_.view(dev_).gather(x, y); }
    void scatter(int x, int y, const PixelMixture& m) { mirror_.edit(dev_).scatter(x, y, m); }
    bool is_initialized(int x, int y) const { return mirror_.view(dev_).is_initialized(x, y); }

    bool state_equals(const ModelBank& other) const { return host().state_equals(other.host()); }
    bool state_equals(const rgbdseg::ModelBank& other) const { return host().state_equals(other); }

    // The whole bank as the reference type (a snapshot of the device state).
    const rgbdseg::ModelBank& host() const { return mirror_.view(dev_); }
    // The device handle for a GPU step (host edits are pushed first).
    rgbdseg_bank* device_bank() {
        mirror_.before_step(dev_);
        return dev_;
    }

private:
    int width_, height_;
    BankMode mode_;
    MixtureConfig config_;
    int device_;
    rgbdseg_bank* dev_ = nullptr;
    BankMirror mirror_;
};

// --------------------------------------------------------------- segmenting
// segmenter.cpp:107-147: the same checks and messages; `workers` is accepted
// for signature parity (the CUDA grid replaces parallel_for_rows).
inline MaskPlane segment_color(ModelBank& bank, const Plane<uint8_t>& r, const Plane<uint8_t>& g,
                               const Plane<uint8_t>& b, const MixtureConfig& config,
                               int /*workers*/ = 1) {
    if (bank.mode() != BankMode::Color3)
        throw std::invalid_argument("segment_color: bank mode is not Color3");
    require_same_size(bank.width(), bank.height(), r.width(), r.height(), "segment_color(r)");
    require_same_size(bank.width(), bank.height(), g.width(), g.height(), "segment_color(g)");
    require_same_size(bank.width(), bank.height(), b.width(), b.height(), "segment_color(b)");
    MaskPlane mask(bank.width(), bank.height(), 0);
    const rgbdseg_mixture_cfg c = to_c(config);
    check(rgbdseg_segment_color(bank.device_bank(), r.data(), g.data(), b.data(), &c, mask.data()));
    return mask;
}

inline MaskPlane segment_depth(ModelBank& bank, const Plane<uint16_t>& depth_mm,
                               const MixtureConfig& config, int /*workers*/ = 1) {
    if (bank.mode() != BankMode::Depth1)
        throw std::invalid_argument("segment_depth: bank mode is not Depth1");
    require_same_size(bank.width(), bank.height(), depth_mm.width(), depth_mm.height(),
                      "segment_depth");
    MaskPlane mask(bank.width(), bank.height(), 0);
    const rgbdseg_mixture_cfg c = to_c(config);
    check(rgbdseg_segment_depth(bank.device_bank(), depth_mm.data(), &c, mask.data()));
    return mask;
}

inline MaskPlane segment_augmented(ModelBank& bank, const Plane<uint8_t>& r,
                                   const Plane<uint8_t>& g, const Plane<uint8_t>& b,
                                   const Plane<uint16_t>& depth_mm, const DepthRescale& rescale,
                                   const MixtureConfig& config, int /*workers*/ = 1) {
    if (bank.mode() != BankMode::Augmented4)
        throw std::invalid_argument("segment_augmented: bank mode is not Augmented4");
    require_same_size(bank.width(), bank.height(), r.width(), r.height(),
                      "segment_augmented(color)");
    require_same_size(bank.width(), bank.height(), depth_mm.width(), depth_mm.height(),
                      "segment_augmented(depth)");
    MaskPlane mask(bank.width(), bank.height(), 0);
    const rgbdseg_mixture_cfg c = to_c(config);
    check(rgbdseg_segment_augmented(bank.device_bank(), r.data(), g.data(), b.data(),
                                    depth_mm.data(), rescale.min_mm, rescale.max_mm, &c,
                                    mask.data()));
    return mask;
}

// ------------------------------------------------------------------- fusion
// fusion.hpp:11-23.  The fields are the reference's plain members; the
// device copy is refreshed from them whenever they differ from what the last
// GPU step left, so callers may read and write out / cpt / counter_limit
// freely between steps (copies share the device buffer and stay correct:
// each step first re-syncs it from the stepping copy's own fields).
struct FusionState {
    MaskPlane out;
    Plane<int8_t> cpt;
    int counter_limit = 3;

    struct Device {
        rgbdseg_fusion* h = nullptr;
        int limit = 0;
        MaskPlane out;  // the state the device holds (shadow)
        Plane<int8_t> cpt;
        ~Device() { rgbdseg_fusion_destroy(h); }
    };
    std::shared_ptr<Device> dev;
    int device = 0;
};

// reset_state, fusion.cpp:7-15 (same checks and messages).
inline FusionState reset_state(int width, int height, uint8_t initial_label = 0,
                               int counter_limit = 3, int device = 0) {
    if (counter_limit < 1) throw std::invalid_argument("reset_state: counter_limit must be >= 1");
    if (initial_label > 1) throw std::invalid_argument("reset_state: label must be 0 or 1");
    FusionState s;
    s.out = MaskPlane(width, height, initial_label);
    s.cpt = Plane<int8_t>(width, height, 0);
    s.counter_limit = counter_limit;
    s.device = device;
    return s;
}

// fuse_step, fusion.cpp:17-46: List 1 on the GPU; returns a copy of state.out.
inline MaskPlane fuse_step(FusionState& state, const MaskPlane& rgb_mask,
                           const MaskPlane& depth_mask_registered) {
    require_same_size(state.out.width(), state.out.height(), rgb_mask.width(), rgb_mask.height(),
                      "fuse_step(rgb)");
    require_same_size(state.out.width(), state.out.height(), depth_mask_registered.width(),
                      depth_mask_registered.height(), "fuse_step(depth)");
    auto& d = state.dev;
    if (!d || d->out.width() != state.out.width() || d->out.height() != state.out.height()) {
        d = std::make_shared<FusionState::Device>();
        check(rgbdseg_fusion_create(state.out.width(), state.out.height(), 1, 0, 1, state.device,
                                    &d->h));
        d->limit = -1;
    }
    if (d->limit != state.counter_limit) {
        check(rgbdseg_fusion_set_counter_limit(d->h, state.counter_limit));
        d->limit = state.counter_limit;
    }
    if (!(d->out == state.out) || !(d->cpt == state.cpt)) {  // host edits / another copy
        check(rgbdseg_fusion_upload(d->h, state.out.data(), state.cpt.data()));
        d->out = state.out;
        d->cpt = state.cpt;
    }
    check(rgbdseg_fusion_step(d->h, rgb_mask.data(), depth_mask_registered.data(), nullptr));
    check(rgbdseg_fusion_download(d->h, state.out.data(), state.cpt.data()));
    d->out = state.out;
    d->cpt = state.cpt;
    return state.out;
}

// -------------------------------------------------------- SequenceProcessor
// processor.hpp:60-80 / processor.cpp:122-184.  The fused method runs as one
// kernel per frame (colour + depth + List 1, registration for unregistered
// sequences); rgb-only / depth-only / augmented method sets run only the
// banks they need (processor.cpp:137-150).  BankLayout::Aos is accepted like
// the reference (same results, test_segmenter.cpp:186-206) and, like it,
// exposes no ModelBank (color_bank() / depth_bank() return nullptr) and
// rejects the augmented method.
// ---- per-pixel API (mixture.hpp:43-60) ----------------------------------
// The reference's PixelMixture and the C-ABI record share one layout
// (int, int, float[20], float[5], float[5]).  Every single-record call is a
// GPU round trip, which only makes sense for parity checks; the batched
// forms below run one kernel over all records.
static_assert(sizeof(PixelMixture) == sizeof(rgbdseg_pixel_mixture), "record layout");
inline rgbdseg_pixel_mixture* rec(PixelMixture* m) {
    return reinterpret_cast<rgbdseg_pixel_mixture*>(m);
}
inline const rgbdseg_pixel_mixture* rec(const PixelMixture* m) {
    return reinterpret_cast<const rgbdseg_pixel_mixture*>(m);
}

inline PixelMixture init_mixture(std::span<const float> first_value, const MixtureConfig& config,
                                 int device = 0) {
    const rgbdseg_mixture_cfg c = to_c(config);
    PixelMixture m;
    check(rgbdseg_init_mixtures(first_value.data(), (int)first_value.size(), 1, &c, rec(&m),
                                device));
    return m;
}

inline std::optional<int> match_component(const PixelMixture& mixture,
                                          std::span<const float> value,
                                          const MixtureConfig& config, int device = 0) {
    const rgbdseg_mixture_cfg c = to_c(config);
    int32_t k = -1;
    check(rgbdseg_match_components(rec(&mixture), value.data(), (int)value.size(), 1, &c, &k,
                                   device));
    return k < 0 ? std::nullopt : std::optional<int>(k);
}

inline void update_mixture(PixelMixture& mixture, std::span<const float> value,
                           std::optional<int> matched, const MixtureConfig& config,
                           int device = 0) {
    const rgbdseg_mixture_cfg c = to_c(config);
    const int32_t k = matched ? *matched : -1;
    check(rgbdseg_update_mixtures(rec(&mixture), value.data(), (int)value.size(), 1, &k, &c,
                                  device));
}

inline PixelLabel classify(const PixelMixture& mixture, std::optional<int> matched,
                           const MixtureConfig& config, int device = 0) {
    const rgbdseg_mixture_cfg c = to_c(config);
    const int32_t k = matched ? *matched : -1;
    uint8_t lab = 1;
    check(rgbdseg_classify_mixtures(rec(&mixture), &k, 1, &c, &lab, device));
    return lab ? PixelLabel::Foreground : PixelLabel::Background;
}

inline PixelLabel step_pixel(PixelMixture& mixture, std::span<const float> value,
                             const MixtureConfig& config, int device = 0) {
    const rgbdseg_mixture_cfg c = to_c(config);
    uint8_t lab = 1;
    check(rgbdseg_step_mixtures(rec(&mixture), value.data(), (int)value.size(), 1, &c, &lab,
                                device));
    return lab ? PixelLabel::Foreground : PixelLabel::Background;
}

// Batched: record i observes values[i*C .. i*C+C).
inline void step_mixtures(std::span<PixelMixture> mixtures, std::span<const float> values,
                          int channels, const MixtureConfig& config, std::span<PixelLabel> labels,
                          int device = 0) {
    if (values.size() != mixtures.size() * (size_t)channels || labels.size() != mixtures.size())
        throw std::invalid_argument("step_mixtures: size mismatch");
    const rgbdseg_mixture_cfg c = to_c(config);
    static_assert(sizeof(PixelLabel) == 1, "label layout");
    check(rgbdseg_step_mixtures(rec(mixtures.data()), values.data(), channels, mixtures.size(), &c,
                                reinterpret_cast<uint8_t*>(labels.data()), device));
}

inline std::vector<PixelMixture> init_mixtures(std::span<const float> values, int channels,
                                               const MixtureConfig& config, int device = 0) {
    if (channels <= 0 || values.size() % (size_t)channels)
        throw std::invalid_argument("init_mixtures: size mismatch");
    std::vector<PixelMixture> out(values.size() / channels);
    const rgbdseg_mixture_cfg c = to_c(config);
    check(rgbdseg_init_mixtures(values.data(), channels, out.size(), &c, rec(out.data()), device));
    return out;
}

class SequenceProcessor {
public:
    SequenceProcessor(int width, int height, const MethodSet& methods, const RunConfig& config,
                      std::optional<CameraRig> rig = std::nullopt, bool registered = true,
                      BankLayout layout = BankLayout::Soa, int device = 0)
        : w_(width), h_(height), methods_(methods), config_(config), rig_(std::move(rig)),
          registered_(registered), layout_(layout), device_(device) {
        config_.validate();  // processor.cpp:128
        if (!registered_ && !rig_)
            throw std::invalid_argument("unregistered sequence requires calibration");
        if (layout_ == BankLayout::Aos && methods_.augmented)
            throw std::invalid_argument("AoS layout does not support the augmented method");
        if (methods_.fused) {
            rgbdseg_processor_cfg c;
            rgbdseg_processor_defaults(&c, width, height);
            c.color = to_c(config_.color_gmm);
            c.depth = to_c(config_.depth_gmm);
            c.fusion_counter_limit = config_.fusion_counter_limit;
            c.fusion_initial_label = config_.fusion_initial_label;
            c.device = device;
            c.registered = registered_ ? 1 : 0;
            c.dilation_radius = config_.dilation_radius;
            if (rig_) {
                c.rig = rgbdseg_camera_rig{rig_->depth_cam.fx, rig_->depth_cam.fy,
                                           rig_->depth_cam.cx, rig_->depth_cam.cy,
                                           rig_->color_cam.fx, rig_->color_cam.fy,
                                           rig_->color_cam.cx, rig_->color_cam.cy,
                                           {}, {}, rig_->depth_scale};
                for (int i = 0; i < 9; ++i) c.rig.rotation[i] = rig_->rotation[i];
                for (int i = 0; i < 3; ++i) c.rig.translation_mm[i] = rig_->translation_mm[i];
            }
            check(rgbdseg_processor_create(&c, &p_));
            cmirror_ = std::make_unique<BankMirror>(width, height, BankMode::Color3,
                                                    config_.color_gmm);
            dmirror_ = std::make_unique<BankMirror>(width, height, BankMode::Depth1,
                                                    config_.depth_gmm);
        } else {
            if (methods_.needs_rgb())
                color_ = std::make_unique<ModelBank>(width, height, BankMode::Color3,
                                                     config_.color_gmm, device);
            if (methods_.needs_depth())
                depth_ = std::make_unique<ModelBank>(width, height, BankMode::Depth1,
                                                     config_.depth_gmm, device);
        }
        if (methods_.augmented)  // processor.cpp:148-150
            aug_ = std::make_unique<ModelBank>(width, height, BankMode::Augmented4,
                                               config_.augmented_gmm, device);
    }
    ~SequenceProcessor() { rgbdseg_processor_destroy(p_); }
    SequenceProcessor(const SequenceProcessor&) = delete;
    SequenceProcessor& operator=(const SequenceProcessor&) = delete;

    FrameMasks process(FrameSet&& frame) {
        FrameMasks out;
        out.index = frame.index;
        if (p_) {
            require_same_size(w_, h_, frame.r.width(), frame.r.height(), "segment_color(r)");
            require_same_size(w_, h_, frame.g.width(), frame.g.height(), "segment_color(g)");
            require_same_size(w_, h_, frame.b.width(), frame.b.height(), "segment_color(b)");
            require_same_size(w_, h_, frame.depth.width(), frame.depth.height(), "segment_depth");
            MaskPlane rgb(w_, h_), dep(w_, h_), fused(w_, h_);
            check(rgbdseg_processor_process(p_, frame.r.data(), frame.g.data(), frame.b.data(),
                                            frame.depth.data(), fused.data(), rgb.data(),
                                            dep.data()));
            cmirror_->invalidate();
            dmirror_->invalidate();
            out.rgb = std::move(rgb);
            out.depth = std::move(dep);
            out.fused = std::move(fused);
        } else {
            if (color_)
                out.rgb = b200::segment_color(*color_, frame.r, frame.g, frame.b,
                                              config_.color_gmm);
            if (depth_) out.depth = b200::segment_depth(*depth_, frame.depth, config_.depth_gmm);
        }
        if (aug_)
            out.augmented = b200::segment_augmented(*aug_, frame.r, frame.g, frame.b, frame.depth,
                                                    config_.augmented_depth_range,
                                                    config_.augmented_gmm);
        out.gt = std::move(frame.gt);
        return out;
    }

    // processor.hpp:67-68: nullptr when the method set needs no such bank, or
    // for the AoS layout (the reference keeps AosModel records instead).
    const rgbdseg::ModelBank* color_bank() const {
        if (layout_ == BankLayout::Aos) return nullptr;
        if (p_) return &cmirror_->view(rgbdseg_processor_color_bank(p_));
        return color_ ? &color_->host() : nullptr;
    }
    const rgbdseg::ModelBank* depth_bank() const {
        if (layout_ == BankLayout::Aos) return nullptr;
        if (p_) return &dmirror_->view(rgbdseg_processor_depth_bank(p_));
        return depth_ ? &depth_->host() : nullptr;
    }

private:
    int w_, h_;
    MethodSet methods_;
    RunConfig config_;
    std::optional<CameraRig> rig_;
    bool registered_;
    BankLayout layout_;
    int device_;
    rgbdseg_processor* p_ = nullptr;  // fused method
    std::unique_ptr<BankMirror> cmirror_, dmirror_;
    std::unique_ptr<ModelBank> color_, depth_, aug_;  // rgb/depth without fusion; augmented
};

}  // namespace rgbdseg::b200
