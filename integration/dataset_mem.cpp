// integration/dataset_mem.cpp -- TEST INFRASTRUCTURE: an in-memory stand-in
// for the reference's dataset.cpp (which needs OpenCV's PNG codecs, absent
// here), so code written against the reference's SequenceSource / load_frame
// (dataset.hpp:52-70) runs unchanged.  A manifest registered by name renders
// its frames with the reference's own render_frame (synthetic.cpp:119-195)
// instead of reading PNGs, optionally punching deterministic no-return holes
// into the depth plane (raw 0, segmenter.cpp:128) so the sentinel branch runs.
#include <map>
#include <stdexcept>
#include <string>

#include "rgbdseg/dataset.hpp"
#include "rgbdseg/synthetic.hpp"

namespace rgbdseg {

namespace {
struct MemSeq {
    ScenarioSpec spec;
    bool holes;
};
std::map<std::string, MemSeq>& registry() {
    static std::map<std::string, MemSeq> r;
    return r;
}
}  // namespace

// Registers `spec` under `name`; returns a manifest that load_frame /
// SequenceSource serve from memory.
SequenceManifest mem_manifest(const std::string& name, const ScenarioSpec& spec, bool holes,
                              bool registered = true,
                              std::optional<CameraRig> calibration = std::nullopt) {
    registry()[name] = MemSeq{spec, holes};
    SequenceManifest m;
    m.name = name;
    m.frame_count = spec.frame_count;
    m.registered = registered;
    m.calibration = calibration;
    m.root = "mem:" + name;
    for (int i = 0; i < spec.frame_count; ++i) m.frames.push_back(FrameRef{i, "", "", ""});
    return m;
}

FrameSet load_frame(const SequenceManifest& manifest, int index, bool want_gt) {
    auto it = registry().find(manifest.name);
    if (it == registry().end()) throw std::runtime_error("mem dataset: unknown sequence");
    if (index < 0 || index >= manifest.frame_count)
        throw std::out_of_range("load_frame: index out of range");
    FrameSet fs = render_frame(it->second.spec, index);
    if (it->second.holes) {
        const int w = fs.depth.width(), h = fs.depth.height();
        if (index % 5 == 2)
            for (int y = h / 8; y < h / 8 + h / 6; ++y)
                for (int x = w / 4; x < w / 4 + w / 5; ++x) fs.depth.at(x, y) = 0;
        for (int i = (index * 7919) % 97; i < w * h; i += 97) fs.depth.data()[i] = 0;
    }
    if (!want_gt) fs.gt.reset();
    return fs;
}

std::optional<FrameSet> SequenceSource::next() {
    if (cursor_ >= manifest_.frame_count) return std::nullopt;
    return load_frame(manifest_, cursor_++, want_gt_);
}

}  // namespace rgbdseg
