// integration/scenario_test.cpp -- source compatibility of the C++ drop-in.
//
// `run_scenario` (and its helpers mask_hash / RunOutput) are compiled
// VERBATIM from the reference's acceptance suite
// (/root/reference/proj/tests/acceptance.cpp:38-46,133-174): the Makefile
// extracts that text into _build/run_scenario_ref.inc at build time (nothing
// of it is stored in this repo).  It is compiled twice -- once where
// `SequenceProcessor` names the reference's CPU class, once where it names
// rgbdseg::b200::SequenceProcessor -- and both runs must produce the same
// per-frame mask hashes, confusion counts and final banks (acceptance
// criterion 3's check, CPU vs GPU instead of worker counts).
//
// Then the rest of the drop-in surface against the reference, call for call:
// rgb-only / depth-only / augmented method sets, the free functions
// b200::segment_color / segment_depth / segment_augmented on b200::ModelBank
// (including writes through its mutable plane accessors between steps), and
// b200::reset_state / fuse_step with host edits of out / cpt / counter_limit.
//
// Usage: scenario_test [frames] [width] [height]; exit 0 = everything identical.
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "rgbdseg/eval.hpp"
#include "rgbdseg/processor.hpp"
#include "rgbdseg/synthetic.hpp"
#include "rgbdseg_b200_dropin.hpp"

using namespace rgbdseg;

namespace rgbdseg {
SequenceManifest mem_manifest(const std::string& name, const ScenarioSpec& spec, bool holes,
                              bool registered = true,
                              std::optional<CameraRig> calibration = std::nullopt);
}

namespace cpu_run {
using rgbdseg::SequenceProcessor;
#include "run_scenario_ref.inc"
}  // namespace cpu_run

namespace gpu_run {
using rgbdseg::b200::SequenceProcessor;
#include "run_scenario_ref.inc"
}  // namespace gpu_run

static int failures = 0;

static void expect(bool ok, const std::string& what) {
    std::printf("%s: %s\n", ok ? "ok  " : "FAIL", what.c_str());
    if (!ok) ++failures;
}

template <typename A, typename B>
static bool same_run(const A& a, const B& b, bool banks) {
    if (a.hashes != b.hashes) return false;
    if (a.counts.size() != b.counts.size()) return false;
    for (const auto& [name, ca] : a.counts) {
        const auto& cb = b.counts.at(name);
        if (ca.size() != cb.size()) return false;
        for (size_t i = 0; i < ca.size(); ++i)
            if (ca[i].tp != cb[i].tp || ca[i].fp != cb[i].fp || ca[i].tn != cb[i].tn ||
                ca[i].fn != cb[i].fn)
                return false;
    }
    if (!banks) return true;
    if (!a.color_bank || !b.color_bank || !a.depth_bank || !b.depth_bank) return false;
    return a.color_bank->state_equals(*b.color_bank) && a.depth_bank->state_equals(*b.depth_bank);
}

int main(int argc, char** argv) {
    const int frames = argc > 1 ? std::atoi(argv[1]) : 60;
    const int w = argc > 2 ? std::atoi(argv[2]) : 160;
    const int h = argc > 3 ? std::atoi(argv[3]) : 120;
    ScenarioSpec spec = builtin_scenario("A");
    spec.width = w;
    spec.height = h;
    spec.frame_count = frames;
    RunConfig cfg = RunConfig::defaults();
    cfg.color_gmm.components = cfg.depth_gmm.components = 5;
    cfg.augmented_gmm.components = 4;
    cfg.workers = 2;

    // --- run_scenario verbatim: registered, with holes, + augmented ------------
    {
        const SequenceManifest m = mem_manifest("A_reg", spec, true);
        const auto c = cpu_run::run_scenario(m, cfg, true, true);
        const auto g = gpu_run::run_scenario(m, cfg, true, true);
        expect(c.hashes.at("fused").size() == static_cast<size_t>(frames) &&
                   same_run(c, g, true),
               "run_scenario (registered, depth holes, fused + augmented): hashes, counts, banks");
    }
    // --- unregistered manifest with calibration --------------------------------
    {
        CameraRig rig = CameraRig::identity(500.0, 500.0, w / 2.0, h / 2.0);
        rig.color_cam.fx = 505.0;
        rig.translation_mm = {25.0, -10.0, 5.0};
        const SequenceManifest m = mem_manifest("A_unreg", spec, true, false, rig);
        RunConfig c2 = cfg;
        c2.dilation_radius = 2;
        const auto c = cpu_run::run_scenario(m, c2, false, true);
        const auto g = gpu_run::run_scenario(m, c2, false, true);
        expect(same_run(c, g, true), "run_scenario (unregistered, rig, radius 2)");
    }
    // --- AoS layout: no ModelBank exposed, same masks ---------------------------
    {
        const SequenceManifest m = mem_manifest("A_aos", spec, false);
        const auto c = cpu_run::run_scenario(m, cfg, false, true, BankLayout::Aos);
        const auto g = gpu_run::run_scenario(m, cfg, false, true, BankLayout::Aos);
        expect(same_run(c, g, false) && !c.color_bank && !g.color_bank,
               "run_scenario (BankLayout::Aos): masks identical, no bank exposed");
        MethodSet ma;
        ma.fused = ma.augmented = true;
        bool cpu_threw = false, gpu_threw = false;
        std::string cm, gm;
        try {
            rgbdseg::SequenceProcessor p(w, h, ma, cfg, std::nullopt, true, BankLayout::Aos);
        } catch (const std::invalid_argument& e) {
            cpu_threw = true;
            cm = e.what();
        }
        try {
            rgbdseg::b200::SequenceProcessor p(w, h, ma, cfg, std::nullopt, true, BankLayout::Aos);
        } catch (const std::invalid_argument& e) {
            gpu_threw = true;
            gm = e.what();
        }
        expect(cpu_threw && gpu_threw && cm == gm, "Aos + augmented rejected: " + gm);
    }
    // --- method sets without fusion: only the needed banks run -----------------
    for (int which = 0; which < 3; ++which) {
        MethodSet ms;
        ms.rgb = which != 1;
        ms.depth = which != 0;
        ms.augmented = which == 2;
        rgbdseg::SequenceProcessor cp(w, h, ms, cfg);
        rgbdseg::b200::SequenceProcessor gp(w, h, ms, cfg);
        const SequenceManifest m = mem_manifest("A_ms", spec, true);
        bool ok = true;
        for (int f = 0; f < frames; ++f) {
            FrameSet a = load_frame(m, f, false);
            FrameSet b = a;
            const FrameMasks mc = cp.process(std::move(a));
            const FrameMasks mg = gp.process(std::move(b));
            ok = ok && mc.rgb.has_value() == mg.rgb.has_value() &&
                 mc.depth.has_value() == mg.depth.has_value() && !mg.fused &&
                 mc.augmented.has_value() == mg.augmented.has_value();
            if (mc.rgb && mg.rgb) ok = ok && *mc.rgb == *mg.rgb;
            if (mc.depth && mg.depth) ok = ok && *mc.depth == *mg.depth;
            if (mc.augmented && mg.augmented) ok = ok && *mc.augmented == *mg.augmented;
        }
        ok = ok && (cp.color_bank() == nullptr) == (gp.color_bank() == nullptr);
        ok = ok && (cp.depth_bank() == nullptr) == (gp.depth_bank() == nullptr);
        if (cp.color_bank()) ok = ok && cp.color_bank()->state_equals(*gp.color_bank());
        if (cp.depth_bank()) ok = ok && cp.depth_bank()->state_equals(*gp.depth_bank());
        const char* names[3] = {"rgb only", "depth only", "rgb + depth + augmented"};
        expect(ok, std::string("MethodSet ") + names[which] + ": masks, which banks exist, banks");
    }
    // --- free functions + mutable plane accessors ------------------------------
    {
        const SequenceManifest m = mem_manifest("A_free", spec, true);
        rgbdseg::ModelBank cb(w, h, BankMode::Color3, cfg.color_gmm);
        rgbdseg::b200::ModelBank gb(w, h, BankMode::Color3, cfg.color_gmm);
        rgbdseg::ModelBank cd(w, h, BankMode::Depth1, cfg.depth_gmm);
        rgbdseg::b200::ModelBank gd(w, h, BankMode::Depth1, cfg.depth_gmm);
        rgbdseg::ModelBank ca(w, h, BankMode::Augmented4, cfg.augmented_gmm);
        rgbdseg::b200::ModelBank ga(w, h, BankMode::Augmented4, cfg.augmented_gmm);
        FusionState cf = reset_state(w, h, 0, 3);
        rgbdseg::b200::FusionState gf = rgbdseg::b200::reset_state(w, h, 0, 3);
        bool ok = true;
        for (int f = 0; f < frames; ++f) {
            const FrameSet fr = load_frame(m, f, false);
            if (f == frames / 2) {  // edit the state through the mutable views
                for (auto* bank : {&cb}) bank->variance_plane(1).at(3, 4) = 9.0f;
                gb.variance_plane(1).at(3, 4) = 9.0f;
                PixelMixture pm = cb.gather(5, 6);
                pm.weights[0] = 0.5f;
                cb.scatter(5, 6, pm);
                gb.scatter(5, 6, pm);
                cd.initialized_plane().at(7, 7) = 0;
                gd.initialized_plane().at(7, 7) = 0;
                cf.out.at(1, 1) = 1;
                gf.out.at(1, 1) = 1;
                cf.cpt.at(2, 2) = 2;
                gf.cpt.at(2, 2) = 2;
                cf.counter_limit = gf.counter_limit = 2;
            }
            const MaskPlane r1 = segment_color(cb, fr.r, fr.g, fr.b, cfg.color_gmm, 3);
            const MaskPlane r2 = rgbdseg::b200::segment_color(gb, fr.r, fr.g, fr.b, cfg.color_gmm, 3);
            const MaskPlane d1 = segment_depth(cd, fr.depth, cfg.depth_gmm);
            const MaskPlane d2 = rgbdseg::b200::segment_depth(gd, fr.depth, cfg.depth_gmm);
            const MaskPlane a1 = segment_augmented(ca, fr.r, fr.g, fr.b, fr.depth,
                                                   cfg.augmented_depth_range, cfg.augmented_gmm);
            const MaskPlane a2 = rgbdseg::b200::segment_augmented(
                ga, fr.r, fr.g, fr.b, fr.depth, cfg.augmented_depth_range, cfg.augmented_gmm);
            const MaskPlane f1 = fuse_step(cf, r1, d1);
            const MaskPlane f2 = rgbdseg::b200::fuse_step(gf, r2, d2);
            ok = ok && r1 == r2 && d1 == d2 && a1 == a2 && f1 == f2 && cf.out == gf.out &&
                 cf.cpt == gf.cpt;
        }
        ok = ok && gb.state_equals(cb) && gd.state_equals(cd) && ga.state_equals(ca);
        ok = ok && gb.gather(5, 6) == cb.gather(5, 6) && gd.is_initialized(7, 7) == cd.is_initialized(7, 7);
        expect(ok, "free functions segment_color/_depth/_augmented + fuse_step, with host edits");
        // the reference's error contract
        std::string e1, e2;
        try {
            segment_depth(cb, load_frame(m, 0, false).depth, cfg.depth_gmm);
        } catch (const std::invalid_argument& e) {
            e1 = e.what();
        }
        try {
            rgbdseg::b200::segment_depth(gb, load_frame(m, 0, false).depth, cfg.depth_gmm);
        } catch (const std::invalid_argument& e) {
            e2 = e.what();
        }
        expect(!e1.empty() && e1 == e2, "mode mismatch message: " + e2);
        MixtureConfig bad = cfg.color_gmm;
        bad.components = 4;
        e1.clear();
        e2.clear();
        const FrameSet fr = load_frame(m, 0, false);
        try {
            segment_color(cb, fr.r, fr.g, fr.b, bad);
        } catch (const std::invalid_argument& e) {
            e1 = e.what();
        }
        try {
            rgbdseg::b200::segment_color(gb, fr.r, fr.g, fr.b, bad);
        } catch (const std::invalid_argument& e) {
            e2 = e.what();
        }
        expect(!e1.empty() && e1 == e2, "component mismatch message: " + e2);
    }
    std::printf("scenario_test: %d frames %dx%d, %d failure(s)\n", frames, w, h, failures);
    return failures == 0 ? 0 : 1;
}
