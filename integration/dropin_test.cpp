// integration/dropin_test.cpp -- runs the reference's own SequenceProcessor
// (CPU, compiled from /root/reference/proj/src into oracle/_ref) and the B200
// drop-in side by side on scenario-A frames rendered by the reference's
// render_frame, and checks FrameMasks and the final banks are identical
// (acceptance.cpp:206-237 criterion 3, CPU vs GPU instead of worker counts).
// Usage: dropin_test [frames] [width] [height] [M] [unregistered]; exit 0 = identical.
#include <cstdio>
#include <cstdlib>

#include "rgbdseg/synthetic.hpp"
#include "rgbdseg_b200_dropin.hpp"

using namespace rgbdseg;

int main(int argc, char** argv) {
    const int frames = argc > 1 ? std::atoi(argv[1]) : 60;
    const int w = argc > 2 ? std::atoi(argv[2]) : 320;
    const int h = argc > 3 ? std::atoi(argv[3]) : 240;
    const int M = argc > 4 ? std::atoi(argv[4]) : 5;
    const bool unregistered = argc > 5 && std::atoi(argv[5]) != 0;
    ScenarioSpec spec = builtin_scenario("A");
    spec.width = w;
    spec.height = h;
    RunConfig cfg = RunConfig::defaults();
    cfg.color_gmm.components = cfg.depth_gmm.components = M;
    cfg.workers = 0;
    cfg.augmented_gmm.components = M;
    MethodSet methods;
    methods.fused = true;
    methods.augmented = true;
    std::optional<CameraRig> rig;
    if (unregistered) {  // a small rigid offset between the cameras
        CameraRig r = CameraRig::identity(500.0, 500.0, w / 2.0, h / 2.0);
        r.color_cam.fx = 505.0;
        r.translation_mm = {25.0, -10.0, 5.0};
        rig = r;
    }
    rgbdseg::SequenceProcessor cpu(w, h, methods, cfg, rig, !unregistered);
    rgbdseg::b200::SequenceProcessor gpu(w, h, methods, cfg, rig, !unregistered);
    int bad = 0;
    for (int f = 0; f < frames; ++f) {
        FrameSet a = render_frame(spec, 90 + f);
        if (f % 5 == 2)  // no-return holes (segmenter.cpp:128)
            for (int y = 3; y < 17; ++y)
                for (int x = 20; x < 60; ++x) a.depth.at(x, y) = 0;
        FrameSet b = a;
        const FrameMasks mc = cpu.process(std::move(a));
        const FrameMasks mg = gpu.process(std::move(b));
        if (!(*mc.rgb == *mg.rgb) || !(*mc.depth == *mg.depth) || !(*mc.fused == *mg.fused) ||
            !(*mc.augmented == *mg.augmented)) {
            std::printf("frame %d: masks differ\n", f);
            ++bad;
        }
    }
    const bool banks = cpu.color_bank()->state_equals(*gpu.color_bank()) &&
                       cpu.depth_bank()->state_equals(*gpu.depth_bank());
    std::printf("dropin_test: %d frames %dx%d M=%d %s, mask mismatches %d, banks %s\n", frames,
                w, h, M, unregistered ? "unregistered" : "registered", bad,
                banks ? "identical" : "DIFFER");
    return (bad == 0 && banks) ? 0 : 1;
}
