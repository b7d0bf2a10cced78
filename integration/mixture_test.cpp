// integration/mixture_test.cpp -- the per-pixel API of the C++ drop-in
// (rgbdseg::b200::init_mixture / match_component / classify / update_mixture /
// step_pixel and the batched forms) against the reference's own functions
// (mixture.cpp:58-154, compiled in oracle/_ref) on random sequences: every
// label, matched index and final record bitwise equal.  Exit 0 = identical.
#include <cstdio>
#include <random>

#include "rgbdseg_b200_dropin.hpp"

using namespace rgbdseg;

int main() {
    std::mt19937 rng(7);
    std::uniform_real_distribution<float> u(0.0f, 255.0f);
    std::normal_distribution<float> nz(0.0f, 6.0f);
    int bad = 0, steps = 0;
    for (int trial = 0; trial < 60; ++trial) {
        MixtureConfig cfg;
        cfg.components = 3 + trial % 3;
        cfg.learning_rate = (trial % 4 == 0) ? 0.3f : 0.05f;
        const int C = (trial / 3) % 2 ? 3 : 1;
        std::vector<float> v0(C);
        for (auto& x : v0) x = u(rng);
        PixelMixture a = rgbdseg::init_mixture(v0, cfg);
        PixelMixture b = rgbdseg::b200::init_mixture(v0, cfg);
        bad += !(a == b);
        for (int s = 0; s < 25; ++s, ++steps) {
            std::vector<float> v(C);
            for (int c = 0; c < C; ++c) v[c] = (s % 4 == 3) ? u(rng) : a.mean(0)[c] + nz(rng);
            const auto ma = rgbdseg::match_component(a, v, cfg);
            const auto mb = rgbdseg::b200::match_component(b, v, cfg);
            bad += ma != mb;
            bad += rgbdseg::classify(a, ma, cfg) != rgbdseg::b200::classify(b, mb, cfg);
            if (s % 2) {
                rgbdseg::update_mixture(a, v, ma, cfg);
                rgbdseg::b200::update_mixture(b, v, mb, cfg);
            } else {
                bad += rgbdseg::step_pixel(a, v, cfg) != rgbdseg::b200::step_pixel(b, v, cfg);
            }
            bad += !(a == b);
        }
    }
    // batched forms over 4096 records
    MixtureConfig cfg;
    cfg.components = 5;
    std::vector<float> vals(4096 * 3);
    for (auto& x : vals) x = u(rng);
    auto gm = rgbdseg::b200::init_mixtures(vals, 3, cfg);
    std::vector<PixelMixture> cm;
    for (size_t i = 0; i < gm.size(); ++i)
        cm.push_back(rgbdseg::init_mixture(std::span<const float>(vals.data() + 3 * i, 3), cfg));
    for (int f = 0; f < 20; ++f) {
        for (auto& x : vals) x = std::min(255.0f, std::max(0.0f, x + nz(rng)));
        std::vector<PixelLabel> gl(gm.size());
        rgbdseg::b200::step_mixtures(gm, vals, 3, cfg, gl);
        for (size_t i = 0; i < cm.size(); ++i) {
            bad += rgbdseg::step_pixel(cm[i], std::span<const float>(vals.data() + 3 * i, 3), cfg) !=
                   gl[i];
            bad += !(cm[i] == gm[i]);
        }
    }
    std::printf("mixture_test: %d single-record steps, 20 x 4096 batched, mismatches %d\n", steps,
                bad);
    return bad == 0 ? 0 : 1;
}
