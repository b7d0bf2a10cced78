// oracle/ref_shim.cpp -- extern "C" shim over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile together with the
// reference's own translation units (read in place from
// /root/reference/proj/src, never copied) into oracle/_ref/librgbdseg_ref.so.
// It is used to pin the C restatement (oracle/rgbdseg_oracle.c), to generate
// tests/golden/, and as the reference arm of bench.py (the reference's own CPU
// path, SequenceProcessor::process, processor.cpp:158-184).
//
// dataset.cpp needs OpenCV (absent here), so the four PNG writers that
// generate_synthetic references are stubbed to throw; nothing on the path
// calls them (render_frame is I/O free, synthetic.cpp:119-195).
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>

#include "rgbdseg/fusion.hpp"
#include "rgbdseg/mixture.hpp"
#include "rgbdseg/processor.hpp"
#include "rgbdseg/registration.hpp"
#include "rgbdseg/segmenter.hpp"
#include "rgbdseg/synthetic.hpp"

namespace rgbdseg {
void save_manifest(const SequenceManifest&, const std::filesystem::path&) {
    throw std::runtime_error("ref_shim: PNG/manifest I/O not built (no OpenCV)");
}
void save_color(const Plane<uint8_t>&, const Plane<uint8_t>&, const Plane<uint8_t>&,
                const std::filesystem::path&) {
    throw std::runtime_error("ref_shim: PNG I/O not built (no OpenCV)");
}
void save_depth(const Plane<uint16_t>&, const std::filesystem::path&) {
    throw std::runtime_error("ref_shim: PNG I/O not built (no OpenCV)");
}
void save_mask(const MaskPlane&, const std::filesystem::path&) {
    throw std::runtime_error("ref_shim: PNG I/O not built (no OpenCV)");
}
}  // namespace rgbdseg

using namespace rgbdseg;

namespace {
thread_local std::string g_err;

struct RefCfg {  // same field order as orc_cfg / rgbdseg_mixture_cfg
    int components;
    float learning_rate, match_lambda, background_threshold, initial_sigma, initial_weight,
        variance_floor;
};

MixtureConfig to_ref(const RefCfg* c) {
    MixtureConfig m;
    m.components = c->components;
    m.learning_rate = c->learning_rate;
    m.match_lambda = c->match_lambda;
    m.background_threshold = c->background_threshold;
    m.initial_sigma = c->initial_sigma;
    m.initial_weight = c->initial_weight;
    m.variance_floor = c->variance_floor;
    return m;
}

struct RefMix {  // flat mirror of PixelMixture (mixture.hpp:30-41)
    int components, channels;
    float means[20];
    float variances[5];
    float weights[5];
};

void from_pm(const PixelMixture& p, RefMix* o) {
    o->components = p.components;
    o->channels = p.channels;
    std::memcpy(o->means, p.means.data(), sizeof o->means);
    std::memcpy(o->variances, p.variances.data(), sizeof o->variances);
    std::memcpy(o->weights, p.weights.data(), sizeof o->weights);
}

PixelMixture to_pm(const RefMix* o) {
    PixelMixture p;
    p.components = o->components;
    p.channels = o->channels;
    std::memcpy(p.means.data(), o->means, sizeof o->means);
    std::memcpy(p.variances.data(), o->variances, sizeof o->variances);
    std::memcpy(p.weights.data(), o->weights, sizeof o->weights);
    return p;
}

template <typename F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

template <typename T>
Plane<T> plane_of(const T* p, int w, int h) {
    Plane<T> out(w, h);
    std::memcpy(out.data(), p, sizeof(T) * out.size());
    return out;
}

struct Scene {
    ScenarioSpec spec;
};

struct Proc {
    int w, h;
    std::unique_ptr<SequenceProcessor> p;
    int frame = 0;
};
}  // namespace

extern "C" {

const char* rref_last_error() { return g_err.c_str(); }

int rref_cfg_validate(const RefCfg* c) {
    return guard([&] { to_ref(c).validate(); });
}

// ---- per-pixel API (mixture.hpp:43-60) ----
int rref_init_mixture(const float* v, int channels, const RefCfg* c, RefMix* out) {
    return guard([&] {
        from_pm(init_mixture(std::span<const float>(v, static_cast<size_t>(channels)), to_ref(c)),
                out);
    });
}

int rref_step_pixel(RefMix* m, const float* v, const RefCfg* c, int* label) {
    return guard([&] {
        PixelMixture p = to_pm(m);
        const auto l = step_pixel(p, std::span<const float>(v, static_cast<size_t>(m->channels)),
                                  to_ref(c));
        *label = l == PixelLabel::Foreground ? 1 : 0;
        from_pm(p, m);
    });
}

int rref_match_component(const RefMix* m, const float* v, const RefCfg* c, int* matched) {
    return guard([&] {
        const auto r = match_component(
            to_pm(m), std::span<const float>(v, static_cast<size_t>(m->channels)), to_ref(c));
        *matched = r ? *r : -1;
    });
}

int rref_update_mixture(RefMix* m, const float* v, int matched, const RefCfg* c) {
    return guard([&] {
        PixelMixture p = to_pm(m);
        update_mixture(p, std::span<const float>(v, static_cast<size_t>(m->channels)),
                       matched < 0 ? std::nullopt : std::optional<int>(matched), to_ref(c));
        from_pm(p, m);
    });
}

int rref_classify(const RefMix* m, int matched, const RefCfg* c, int* label) {
    return guard([&] {
        const auto l = classify(to_pm(m), matched < 0 ? std::nullopt : std::optional<int>(matched),
                                to_ref(c));
        *label = l == PixelLabel::Foreground ? 1 : 0;
    });
}

// ---- banks (segmenter.hpp:25-69) ----
void* rref_bank_create(int w, int h, int mode, const RefCfg* c) {
    try {
        return new ModelBank(w, h,
                             mode == 0   ? BankMode::Color3
                             : mode == 1 ? BankMode::Depth1
                                         : BankMode::Augmented4,
                             to_ref(c));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void rref_bank_destroy(void* b) { delete static_cast<ModelBank*>(b); }

int rref_segment_color(void* bank, const uint8_t* r, const uint8_t* g, const uint8_t* b,
                       const RefCfg* c, int workers, uint8_t* mask) {
    return guard([&] {
        auto* bk = static_cast<ModelBank*>(bank);
        const int w = bk->width(), h = bk->height();
        const MaskPlane m = segment_color(*bk, plane_of(r, w, h), plane_of(g, w, h),
                                          plane_of(b, w, h), to_ref(c), workers);
        std::memcpy(mask, m.data(), m.size());
    });
}

int rref_segment_depth(void* bank, const uint16_t* d, const RefCfg* c, int workers,
                       uint8_t* mask) {
    return guard([&] {
        auto* bk = static_cast<ModelBank*>(bank);
        const MaskPlane m =
            segment_depth(*bk, plane_of(d, bk->width(), bk->height()), to_ref(c), workers);
        std::memcpy(mask, m.data(), m.size());
    });
}

int rref_segment_augmented(void* bank, const uint8_t* r, const uint8_t* g, const uint8_t* b,
                           const uint16_t* d, float lo, float hi, const RefCfg* c, int workers,
                           uint8_t* mask) {
    return guard([&] {
        auto* bk = static_cast<ModelBank*>(bank);
        const int w = bk->width(), h = bk->height();
        const MaskPlane m = segment_augmented(*bk, plane_of(r, w, h), plane_of(g, w, h),
                                              plane_of(b, w, h), plane_of(d, w, h),
                                              DepthRescale{lo, hi}, to_ref(c), workers);
        std::memcpy(mask, m.data(), m.size());
    });
}

// kind: 0 mean(comp, chan), 1 variance(comp), 2 weight(comp), 3 initialised flags (u8)
int rref_bank_get(void* bank, int kind, int comp, int chan, void* out) {
    return guard([&] {
        auto* bk = static_cast<ModelBank*>(bank);
        if (kind == 3) {
            std::memcpy(out, bk->initialized_plane().data(), bk->initialized_plane().size());
            return;
        }
        Plane<float>& p = kind == 0   ? bk->mean_plane(comp, chan)
                          : kind == 1 ? bk->variance_plane(comp)
                                      : bk->weight_plane(comp);
        std::memcpy(out, p.data(), p.size() * sizeof(float));
    });
}

int rref_bank_set(void* bank, int kind, int comp, int chan, const void* in) {
    return guard([&] {
        auto* bk = static_cast<ModelBank*>(bank);
        if (kind == 3) {
            std::memcpy(bk->initialized_plane().data(), in, bk->initialized_plane().size());
            return;
        }
        Plane<float>& p = kind == 0   ? bk->mean_plane(comp, chan)
                          : kind == 1 ? bk->variance_plane(comp)
                                      : bk->weight_plane(comp);
        std::memcpy(p.data(), in, p.size() * sizeof(float));
    });
}

// ---- fusion (fusion.hpp:11-23) ----
void* rref_fusion_create(int w, int h, int initial_label, int limit) {
    try {
        return new FusionState(reset_state(w, h, static_cast<uint8_t>(initial_label), limit));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void rref_fusion_destroy(void* s) { delete static_cast<FusionState*>(s); }

int rref_fuse_step(void* s, const uint8_t* rgb, const uint8_t* dep, uint8_t* out, int8_t* cpt) {
    return guard([&] {
        auto* st = static_cast<FusionState*>(s);
        const int w = st->out.width(), h = st->out.height();
        const MaskPlane o = fuse_step(*st, plane_of(rgb, w, h), plane_of(dep, w, h));
        std::memcpy(out, o.data(), o.size());
        if (cpt) std::memcpy(cpt, st->cpt.data(), st->cpt.size());
    });
}

// ---- registration (registration.hpp:28-38), rig packed as in orc_register ----
int rref_register_mask(const uint8_t* mask, const uint16_t* depth, int dw, int dh,
                       const double* rig, int cw, int ch, int radius, uint8_t* out) {
    return guard([&] {
        CameraRig r;
        r.depth_cam = {rig[0], rig[1], rig[2], rig[3]};
        r.color_cam = {rig[4], rig[5], rig[6], rig[7]};
        for (int i = 0; i < 9; ++i) r.rotation[i] = rig[8 + i];
        for (int i = 0; i < 3; ++i) r.translation_mm[i] = rig[17 + i];
        r.depth_scale = rig[20];
        const MaskPlane m = register_mask(plane_of(mask, dw, dh), plane_of(depth, dw, dh), r, cw,
                                          ch, radius);
        std::memcpy(out, m.data(), m.size());
    });
}

// ---- synthetic scenes (synthetic.hpp:61-97) ----
// name: "A"/"B"; w/h/frames/seed override the builtin values when > 0.
void* rref_scene_create(const char* name, int w, int h, int frames, uint64_t seed) {
    try {
        auto* s = new Scene{builtin_scenario(name)};
        if (w > 0) s->spec.width = w;
        if (h > 0) s->spec.height = h;
        if (frames > 0) s->spec.frame_count = frames;
        if (seed > 0) s->spec.seed = seed;
        return s;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void* rref_scene_from_json(const char* path) {
    try {
        return new Scene{parse_scenario_spec(path)};
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void rref_scene_destroy(void* s) { delete static_cast<Scene*>(s); }

int rref_render(void* scene, int frame, uint8_t* r, uint8_t* g, uint8_t* b, uint16_t* d,
                uint8_t* gt) {
    return guard([&] {
        const FrameSet fs = render_frame(static_cast<Scene*>(scene)->spec, frame);
        std::memcpy(r, fs.r.data(), fs.r.size());
        std::memcpy(g, fs.g.data(), fs.g.size());
        std::memcpy(b, fs.b.data(), fs.b.size());
        std::memcpy(d, fs.depth.data(), fs.depth.size() * 2);
        if (gt) std::memcpy(gt, fs.gt->data(), fs.gt->size());
    });
}

uint64_t rref_hash_counter(uint64_t seed, uint64_t stream, uint64_t frame, uint64_t pixel,
                           uint64_t channel) {
    return hash_counter(seed, stream, frame, pixel, channel);
}

// ---- the reference's per-frame processor, processor.cpp:125-184 ----
// Fused method, registered sequence, SoA banks, RunConfig::defaults() with the
// given colour / depth mixture configs and `workers` threads (0 = all).
void* rref_processor_create(int w, int h, const RefCfg* color, const RefCfg* depth, int limit,
                            int initial_label, int workers) {
    try {
        RunConfig cfg = RunConfig::defaults();
        cfg.color_gmm = to_ref(color);
        cfg.depth_gmm = to_ref(depth);
        cfg.fusion_counter_limit = limit;
        cfg.fusion_initial_label = static_cast<uint8_t>(initial_label);
        cfg.workers = workers;
        cfg.pipeline = false;
        MethodSet ms;
        ms.fused = true;
        auto* p = new Proc{w, h, std::make_unique<SequenceProcessor>(w, h, ms, cfg)};
        return p;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
// Unregistered sequence: depth masks go through register_mask (+dilation)
// before fusion (processor.cpp:175-179).  rig packed as in rref_register_mask.
void* rref_processor_create_rig(int w, int h, const RefCfg* color, const RefCfg* depth, int limit,
                                int initial_label, int workers, const double* rig, int radius) {
    try {
        RunConfig cfg = RunConfig::defaults();
        cfg.color_gmm = to_ref(color);
        cfg.depth_gmm = to_ref(depth);
        cfg.fusion_counter_limit = limit;
        cfg.fusion_initial_label = static_cast<uint8_t>(initial_label);
        cfg.workers = workers;
        cfg.pipeline = false;
        cfg.dilation_radius = radius;
        CameraRig r;
        r.depth_cam = {rig[0], rig[1], rig[2], rig[3]};
        r.color_cam = {rig[4], rig[5], rig[6], rig[7]};
        for (int i = 0; i < 9; ++i) r.rotation[i] = rig[8 + i];
        for (int i = 0; i < 3; ++i) r.translation_mm[i] = rig[17 + i];
        r.depth_scale = rig[20];
        MethodSet ms;
        ms.fused = true;
        return new Proc{w, h, std::make_unique<SequenceProcessor>(w, h, ms, cfg, r, false)};
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void rref_processor_destroy(void* p) { delete static_cast<Proc*>(p); }

// Any of rgb_mask / depth_mask / fused may be null.
int rref_processor_process(void* proc, const uint8_t* r, const uint8_t* g, const uint8_t* b,
                           const uint16_t* d, uint8_t* rgb_mask, uint8_t* depth_mask,
                           uint8_t* fused) {
    return guard([&] {
        auto* p = static_cast<Proc*>(proc);
        FrameSet fs;
        fs.index = p->frame++;
        fs.r = plane_of(r, p->w, p->h);
        fs.g = plane_of(g, p->w, p->h);
        fs.b = plane_of(b, p->w, p->h);
        fs.depth = plane_of(d, p->w, p->h);
        const FrameMasks m = p->p->process(std::move(fs));
        if (rgb_mask) std::memcpy(rgb_mask, m.rgb->data(), m.rgb->size());
        if (depth_mask) std::memcpy(depth_mask, m.depth->data(), m.depth->size());
        if (fused) std::memcpy(fused, m.fused->data(), m.fused->size());
    });
}

// bank: 0 colour, 1 depth; kind as rref_bank_get
int rref_processor_bank_get(void* proc, int bank, int kind, int comp, int chan, void* out) {
    auto* p = static_cast<Proc*>(proc);
    const ModelBank* bk = bank == 0 ? p->p->color_bank() : p->p->depth_bank();
    return rref_bank_get(const_cast<ModelBank*>(bk), kind, comp, chan, out);
}

}  // extern "C"
