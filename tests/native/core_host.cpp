// tests/native/core_host.cpp -- TEST INFRASTRUCTURE: the product's per-pixel
// core (paper_2110_14934_b200/csrc/gmm_pixel.cuh) compiled for the HOST so
// the CPU suite can check its logic (rank-count ordering, zero-weight
// division skip, classify fast path) against the oracle without a GPU.  The
// GPU tests check the same source compiled for sm_100a.
#include <cstring>

#include "../../paper_2110_14934_b200/csrc/gmm_pixel.cuh"

using namespace rgbdseg_b200;

struct Rec {  // rgbdseg_pixel_mixture / orc_mix layout
    int components, channels;
    float means[20], variances[5], weights[5];
};
struct Cfg {
    int components;
    float alpha, lambda, T, sigma0, w_new, var_floor;
};

template <int M, int C>
static int step_t(Rec* r, const float* v, const Cfg* k) {
    Mixture<M, C> m;
    for (int i = 0; i < M; ++i) {
        for (int c = 0; c < C; ++c) m.mu[i][c] = r->means[i * C + c];
        m.var[i] = r->variances[i];
        m.w[i] = r->weights[i];
    }
    float vv[C];
    for (int c = 0; c < C; ++c) vv[c] = v[c];
    const MixCfg kk{k->alpha, k->lambda, k->T, k->sigma0, k->w_new, k->var_floor, 0};
    const int lab = (int)gmm_step(m, vv, kk);
    for (int i = 0; i < M; ++i) {
        for (int c = 0; c < C; ++c) r->means[i * C + c] = m.mu[i][c];
        r->variances[i] = m.var[i];
        r->weights[i] = m.w[i];
    }
    return lab;
}

template <int M>
static int step_m(Rec* r, const float* v, const Cfg* k) {
    switch (r->channels) {
        case 1: return step_t<M, 1>(r, v, k);
        case 3: return step_t<M, 3>(r, v, k);
        case 4: return step_t<M, 4>(r, v, k);
    }
    return -1;
}

extern "C" int core_step(Rec* r, const float* v, const Cfg* k) {
    switch (r->components) {
        case 3: return step_m<3>(r, v, k);
        case 4: return step_m<4>(r, v, k);
        case 5: return step_m<5>(r, v, k);
    }
    return -1;
}

// List 1 (fusion.cpp:29-44): the branchy and the select form of one step.
extern "C" void core_fuse(int sel, unsigned r, unsigned d, int limit, unsigned* out, int* cpt) {
    uint32_t o = *out;
    int c = *cpt;
    if (sel)
        fuse_pixel_sel(r, d, limit, o, c);
    else
        fuse_pixel(r, d, limit, o, c);
    *out = o;
    *cpt = c;
}
