// integration/rgbdseg_b200_dropin.hpp -- C++ drop-in for the reference's
// SequenceProcessor, compiled INSIDE the reference project against its own
// headers (include/rgbdseg/processor.hpp) and linked to librgbdseg_b200.so.
//
//   rgbdseg::SequenceProcessor          (processor.hpp:60-80, CPU)
//   rgbdseg::b200::SequenceProcessor    (this header, B200 via include/rgbdseg_c.h)
//
// Same constructor arguments, same process(FrameSet&&) -> FrameMasks contract
// (processor.cpp:158-184), same exception types; the banks stay in HBM and
// color_bank()/depth_bank() return host ModelBank copies (the reference
// returns const pointers into host state).  Every MethodSet combination and
// unregistered sequences (rig + depth->colour registration) are served.
#pragma once

#include <optional>
#include <stdexcept>
#include <string>

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

// Copy a device bank into a reference ModelBank through its mutable plane
// accessors (segmenter.hpp:33-37).
inline ModelBank download_bank(rgbdseg_bank* dev, int w, int h, BankMode mode,
                               const MixtureConfig& cfg) {
    ModelBank host(w, h, mode, cfg);
    const int C = host.channels(), M = host.components();
    for (int i = 0; i < M; ++i) {
        for (int c = 0; c < C; ++c) check(rgbdseg_bank_download(dev, i * C + c, host.mean_plane(i, c).data()));
        check(rgbdseg_bank_download(dev, M * C + i, host.variance_plane(i).data()));
        check(rgbdseg_bank_download(dev, M * C + M + i, host.weight_plane(i).data()));
    }
    check(rgbdseg_bank_download(dev, RGBDSEG_FLAGS_PLANE, host.initialized_plane().data()));
    return host;
}

class SequenceProcessor {
public:
    SequenceProcessor(int width, int height, const MethodSet& methods, const RunConfig& config,
                      std::optional<CameraRig> rig = std::nullopt, bool registered = true,
                      int device = 0)
        : w_(width), h_(height), methods_(methods), config_(config) {
        config_.validate();  // processor.cpp:128
        if (!registered && !rig)
            throw std::invalid_argument("unregistered sequence requires calibration");
        rgbdseg_processor_cfg c;
        rgbdseg_processor_defaults(&c, width, height);
        c.color = to_c(config_.color_gmm);
        c.depth = to_c(config_.depth_gmm);
        c.fusion_counter_limit = config_.fusion_counter_limit;
        c.fusion_initial_label = config_.fusion_initial_label;
        c.device = device;
        c.registered = registered ? 1 : 0;
        c.dilation_radius = config_.dilation_radius;
        if (rig) {
            c.rig = rgbdseg_camera_rig{rig->depth_cam.fx, rig->depth_cam.fy, rig->depth_cam.cx,
                                       rig->depth_cam.cy, rig->color_cam.fx, rig->color_cam.fy,
                                       rig->color_cam.cx, rig->color_cam.cy, {}, {},
                                       rig->depth_scale};
            for (int i = 0; i < 9; ++i) c.rig.rotation[i] = rig->rotation[i];
            for (int i = 0; i < 3; ++i) c.rig.translation_mm[i] = rig->translation_mm[i];
        }
        check(rgbdseg_processor_create(&c, &p_));
        if (methods_.augmented) {  // segment_augmented's own bank (processor.cpp:148-150)
            const rgbdseg_mixture_cfg a = to_c(config_.augmented_gmm);
            check(rgbdseg_bank_create(width, height, 1, RGBDSEG_AUGMENTED4, &a, device, &aug_));
        }
    }
    ~SequenceProcessor() {
        rgbdseg_processor_destroy(p_);
        rgbdseg_bank_destroy(aug_);
    }
    SequenceProcessor(const SequenceProcessor&) = delete;
    SequenceProcessor& operator=(const SequenceProcessor&) = delete;

    FrameMasks process(FrameSet&& frame) {
        require_same_size(frame.r.width(), frame.r.height(), w_, h_, "process(color)");
        require_same_size(frame.depth.width(), frame.depth.height(), w_, h_, "process(depth)");
        FrameMasks out;
        out.index = frame.index;
        MaskPlane rgb(w_, h_), dep(w_, h_), fused(w_, h_);
        check(rgbdseg_processor_process(p_, frame.r.data(), frame.g.data(), frame.b.data(),
                                        frame.depth.data(), fused.data(), rgb.data(), dep.data()));
        if (methods_.needs_rgb()) out.rgb = std::move(rgb);
        if (methods_.needs_depth()) out.depth = std::move(dep);
        if (methods_.fused) out.fused = std::move(fused);
        if (aug_) {
            MaskPlane am(w_, h_);
            const rgbdseg_mixture_cfg a = to_c(config_.augmented_gmm);
            check(rgbdseg_segment_augmented(aug_, frame.r.data(), frame.g.data(), frame.b.data(),
                                            frame.depth.data(), config_.augmented_depth_range.min_mm,
                                            config_.augmented_depth_range.max_mm, &a, am.data()));
            out.augmented = std::move(am);
        }
        out.gt = std::move(frame.gt);
        return out;
    }

    ModelBank color_bank() const {
        return download_bank(rgbdseg_processor_color_bank(p_), w_, h_, BankMode::Color3,
                             config_.color_gmm);
    }
    ModelBank depth_bank() const {
        return download_bank(rgbdseg_processor_depth_bank(p_), w_, h_, BankMode::Depth1,
                             config_.depth_gmm);
    }

private:
    int w_, h_;
    MethodSet methods_;
    RunConfig config_;
    rgbdseg_processor* p_ = nullptr;
    rgbdseg_bank* aug_ = nullptr;
};

}  // namespace rgbdseg::b200
