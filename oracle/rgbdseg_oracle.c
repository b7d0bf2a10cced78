/*
 * oracle/rgbdseg_oracle.c -- CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2110_14934_b200/)
 * links, loads or calls this file.  It is imported by tests/, by
 * __graft_entry__.smoke() and by bench.py's cpu_baseline leg, and there only
 * as the checker.
 *
 * Parity pin: this restatement is checked against (1) the reference compiled
 * from its own sources into oracle/_ref/ (oracle/Makefile, oracle/ref_shim.cpp)
 * and (2) the golden fixtures under tests/golden/ produced from that build by
 * tests/golden/make_golden.py.
 *
 * Arithmetic contract: IEEE binary32, round to nearest,
 * no contraction (built with -ffp-contract=off, default x86-64 target, no
 * fast-math), denormals preserved.  Every function cites the reference
 * file:line it restates (paths relative to /root/reference/proj).
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <string.h>

#define ORC_MAX_M 5
#define ORC_MAX_C 4

typedef struct {
    int components;
    float learning_rate;
    float match_lambda;
    float background_threshold;
    float initial_sigma;
    float initial_weight;
    float variance_floor;
} orc_cfg; /* include/rgbdseg/mixture.hpp:16-26 */

typedef struct {
    int components;
    int channels;
    float means[ORC_MAX_M * ORC_MAX_C]; /* means[i*channels + c], mixture.hpp:33,37 */
    float variances[ORC_MAX_M];
    float weights[ORC_MAX_M];
} orc_mix; /* mixture.hpp:30-41 */

/* mixture.cpp:9-24.  Returns 0 when valid, else a code naming the field. */
int orc_cfg_check(const orc_cfg* k) {
    if (k->components < 3 || k->components > 5) return 1;
    if (!(k->learning_rate > 0.0f && k->learning_rate < 1.0f)) return 2;
    if (!(k->background_threshold > 0.0f && k->background_threshold < 1.0f)) return 3;
    if (!(k->match_lambda > 0.0f)) return 4;
    if (!(k->initial_sigma > 0.0f)) return 5;
    if (!(k->initial_weight > 0.0f && k->initial_weight < 1.0f)) return 6;
    if (!(k->variance_floor > 0.0f)) return 7;
    return 0;
}

/* mixture.cpp:30-45: order by w/sqrt(var) descending; the insertion only moves
 * an entry left past a strictly smaller fitness, so ties keep index order. */
static void orc_rank(const orc_mix* m, int order[ORC_MAX_M]) {
    float fit[ORC_MAX_M];
    for (int i = 0; i < m->components; ++i) {
        fit[i] = m->weights[i] / sqrtf(m->variances[i]);
        order[i] = i;
    }
    for (int i = 1; i < m->components; ++i) {
        const int moving = order[i];
        int slot = i;
        while (slot > 0 && fit[order[slot - 1]] < fit[moving]) {
            order[slot] = order[slot - 1];
            slot--;
        }
        order[slot] = moving;
    }
}

/* mixture.cpp:47-54: index-order sum, multiply by the reciprocal. */
static void orc_normalize(orc_mix* m) {
    float total = 0.0f;
    for (int i = 0; i < m->components; ++i) total += m->weights[i];
    if (total > 0.0f) {
        const float r = 1.0f / total;
        for (int i = 0; i < m->components; ++i) m->weights[i] *= r;
    }
}

/* mixture.cpp:58-72 (validation done by the caller). */
void orc_init(orc_mix* m, const float* v, int channels, const orc_cfg* k) {
    memset(m, 0, sizeof *m);
    m->components = k->components;
    m->channels = channels;
    const float var0 = k->initial_sigma * k->initial_sigma;
    for (int i = 0; i < m->components; ++i) {
        m->variances[i] = var0;
        m->weights[i] = i == 0 ? 1.0f : 0.0f;
    }
    for (int c = 0; c < channels; ++c) m->means[c] = v[c];
}

/* mixture.cpp:74-92.  Returns the matched component or -1. */
int orc_match(const orc_mix* m, const float* v, const orc_cfg* k) {
    int order[ORC_MAX_M];
    orc_rank(m, order);
    for (int r = 0; r < m->components; ++r) {
        const int i = order[r];
        const float band = k->match_lambda * sqrtf(m->variances[i]);
        const float* mu = m->means + i * m->channels;
        int inside = 1;
        for (int c = 0; c < m->channels && inside; ++c)
            if (!(fabsf(v[c] - mu[c]) < band)) inside = 0;
        if (inside) return i;
    }
    return -1;
}

/* mixture.cpp:94-131. */
void orc_update(orc_mix* m, const float* v, int matched, const orc_cfg* k) {
    const float a = k->learning_rate;
    if (matched >= 0) {
        for (int i = 0; i < m->components; ++i)
            m->weights[i] = (1.0f - a) * m->weights[i] + (i == matched ? a : 0.0f);
        orc_normalize(m);
        /* std::max(w, a) == (w < a) ? a : w */
        const float wm = m->weights[matched];
        const float rho = a / (wm < a ? a : wm);
        float* mu = m->means + matched * m->channels;
        float d2 = 0.0f;
        for (int c = 0; c < m->channels; ++c) {
            mu[c] = (1.0f - rho) * mu[c] + rho * v[c];
            const float d = v[c] - mu[c];
            d2 += d * d;
        }
        const float var = (1.0f - rho) * m->variances[matched] +
                          rho * d2 / (float)m->channels;
        m->variances[matched] = var < k->variance_floor ? k->variance_floor : var;
    } else {
        int weakest = 0;
        float lowest = m->weights[0] / sqrtf(m->variances[0]);
        for (int i = 1; i < m->components; ++i) {
            const float f = m->weights[i] / sqrtf(m->variances[i]);
            if (f < lowest) {
                lowest = f;
                weakest = i;
            }
        }
        float* mu = m->means + weakest * m->channels;
        for (int c = 0; c < m->channels; ++c) mu[c] = v[c];
        m->variances[weakest] = k->initial_sigma * k->initial_sigma;
        m->weights[weakest] = k->initial_weight;
        orc_normalize(m);
    }
}

/* mixture.cpp:133-146.  Returns 1 = Foreground, 0 = Background. */
int orc_classify(const orc_mix* m, int matched, const orc_cfg* k) {
    if (matched < 0) return 1;
    int order[ORC_MAX_M];
    orc_rank(m, order);
    float cum = 0.0f;
    for (int r = 0; r < m->components; ++r) {
        const int i = order[r];
        cum += m->weights[i];
        if (i == matched) return 0;
        if (cum > k->background_threshold) break;
    }
    return 1;
}

/* mixture.cpp:148-154: match, classify on the pre-update mixture, update. */
int orc_step(orc_mix* m, const float* v, const orc_cfg* k) {
    const int matched = orc_match(m, v, k);
    const int label = orc_classify(m, matched, k);
    orc_update(m, v, matched, k);
    return label;
}

/* ------------------------------------------------------------------------
 * Whole-frame banks.  State is one float array of planes, each `npx` long:
 * plane (i*C + c) = mean of component i channel c, plane (M*C + i) = variance
 * of component i, plane (M*C + M + i) = weight of component i.  This is the
 * plane order of ModelBank (segmenter.hpp:51-54) flattened.
 * ---------------------------------------------------------------------- */

/* segmenter.cpp:24-34 */
void orc_bank_reset(float* state, uint8_t* flags, size_t npx, int channels, const orc_cfg* k) {
    const int M = k->components;
    const float var0 = k->initial_sigma * k->initial_sigma;
    for (int p = 0; p < M * channels; ++p)
        for (size_t j = 0; j < npx; ++j) state[(size_t)p * npx + j] = 0.0f;
    for (int i = 0; i < M; ++i)
        for (size_t j = 0; j < npx; ++j) {
            state[(size_t)(M * channels + i) * npx + j] = var0;
            state[(size_t)(M * channels + M + i) * npx + j] = i == 0 ? 1.0f : 0.0f;
        }
    memset(flags, 0, npx);
}

static void orc_gather(const float* state, size_t npx, size_t j, int M, int C, orc_mix* m) {
    m->components = M;
    m->channels = C;
    for (int i = 0; i < M; ++i) {
        for (int c = 0; c < C; ++c) m->means[i * C + c] = state[(size_t)(i * C + c) * npx + j];
        m->variances[i] = state[(size_t)(M * C + i) * npx + j];
        m->weights[i] = state[(size_t)(M * C + M + i) * npx + j];
    }
}

static void orc_scatter(float* state, size_t npx, size_t j, const orc_mix* m) {
    const int M = m->components, C = m->channels;
    for (int i = 0; i < M; ++i) {
        for (int c = 0; c < C; ++c) state[(size_t)(i * C + c) * npx + j] = m->means[i * C + c];
        state[(size_t)(M * C + i) * npx + j] = m->variances[i];
        state[(size_t)(M * C + M + i) * npx + j] = m->weights[i];
    }
}

/* One pixel of run_bank (segmenter.cpp:80-96): invalid -> label 0, untouched;
 * uninitialised -> seed + flag, label 0; else gather/step/scatter. */
static uint8_t orc_bank_pixel(float* state, uint8_t* flags, size_t npx, size_t j, int C,
                              const float* v, int valid, const orc_cfg* k) {
    if (!valid) return 0;
    orc_mix m;
    if (!flags[j]) {
        orc_init(&m, v, C, k);
        orc_scatter(state, npx, j, &m);
        flags[j] = 1;
        return 0;
    }
    orc_gather(state, npx, j, k->components, C, &m);
    const int label = orc_step(&m, v, k);
    orc_scatter(state, npx, j, &m);
    return (uint8_t)label;
}

/* segment_color, segmenter.cpp:107-119 */
void orc_segment_color(float* state, uint8_t* flags, size_t npx, const uint8_t* r,
                       const uint8_t* g, const uint8_t* b, const orc_cfg* k, uint8_t* mask) {
    for (size_t j = 0; j < npx; ++j) {
        const float v[3] = {(float)r[j], (float)g[j], (float)b[j]};
        mask[j] = orc_bank_pixel(state, flags, npx, j, 3, v, 1, k);
    }
}

/* segment_depth, segmenter.cpp:121-131: raw 0 is the no-return sentinel and
 * the raw millimetre value feeds the mixture unscaled. */
void orc_segment_depth(float* state, uint8_t* flags, size_t npx, const uint16_t* depth,
                       const orc_cfg* k, uint8_t* mask) {
    for (size_t j = 0; j < npx; ++j) {
        const float v[1] = {(float)depth[j]};
        mask[j] = orc_bank_pixel(state, flags, npx, j, 1, v, depth[j] != 0, k);
    }
}

/* DepthRescale::to_channel, segmenter.cpp:18-22 */
static float orc_to_channel(float d, float lo, float hi) {
    if (d <= lo) return 0.0f;
    if (d >= hi) return 255.0f;
    return (d - lo) * 255.0f / (hi - lo);
}

/* segment_augmented, segmenter.cpp:133-147: 4 channels, no depth sentinel. */
void orc_segment_augmented(float* state, uint8_t* flags, size_t npx, const uint8_t* r,
                           const uint8_t* g, const uint8_t* b, const uint16_t* depth, float lo,
                           float hi, const orc_cfg* k, uint8_t* mask) {
    for (size_t j = 0; j < npx; ++j) {
        const float v[4] = {(float)r[j], (float)g[j], (float)b[j],
                            orc_to_channel((float)depth[j], lo, hi)};
        mask[j] = orc_bank_pixel(state, flags, npx, j, 4, v, 1, k);
    }
}

/* ------------------------------------------------------------------------
 * List-1 fusion, fusion.cpp:7-46.  cpt is int8 (fusion.hpp:13).
 * ---------------------------------------------------------------------- */
void orc_fusion_reset(uint8_t* out, int8_t* cpt, size_t n, uint8_t initial_label) {
    memset(out, initial_label, n);
    memset(cpt, 0, n);
}

void orc_fuse(uint8_t* out, int8_t* cpt, size_t n, int limit, const uint8_t* rgb,
              const uint8_t* dep) {
    for (size_t j = 0; j < n; ++j) {
        const uint8_t r = rgb[j], d = dep[j];
        if (r == d) {
            out[j] = d;
            cpt[j] = 0;
        } else if (cpt[j] == limit) {
            out[j] = r;
            cpt[j] = 0;
        } else if (cpt[j] == -limit) {
            out[j] = d;
            cpt[j] = 0;
        } else if (out[j] == r) {
            cpt[j] = (int8_t)(cpt[j] + 1);
        } else {
            cpt[j] = (int8_t)(cpt[j] - 1);
        }
    }
}

/* ------------------------------------------------------------------------
 * Registration + dilation (registration.cpp:33-78), fp64.
 * rig[18]: depth fx fy cx cy, color fx fy cx cy, R[9] row-major ... packed as
 * {dfx,dfy,dcx,dcy, cfx,cfy,ccx,ccy, R0..R8, t0,t1,t2, depth_scale} = 21.
 * ---------------------------------------------------------------------- */
void orc_dilate(const uint8_t* in, uint8_t* out, int w, int h, int radius) {
    if (radius <= 0) {
        memcpy(out, in, (size_t)w * h);
        return;
    }
    memset(out, 0, (size_t)w * h);
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            if (!in[(size_t)y * w + x]) continue;
            const int x0 = x - radius < 0 ? 0 : x - radius;
            const int x1 = x + radius > w - 1 ? w - 1 : x + radius;
            const int y0 = y - radius < 0 ? 0 : y - radius;
            const int y1 = y + radius > h - 1 ? h - 1 : y + radius;
            for (int yy = y0; yy <= y1; ++yy)
                for (int xx = x0; xx <= x1; ++xx) out[(size_t)yy * w + xx] = 1;
        }
}

void orc_register(const uint8_t* mask, const uint16_t* depth, int dw, int dh, const double* rig,
                  int cw, int ch, int radius, uint8_t* scratch, uint8_t* out) {
    const double dfx = rig[0], dfy = rig[1], dcx = rig[2], dcy = rig[3];
    const double cfx = rig[4], cfy = rig[5], ccx = rig[6], ccy = rig[7];
    const double* R = rig + 8;
    const double* t = rig + 17;
    const double scale = rig[20];
    memset(scratch, 0, (size_t)cw * ch);
    for (int v = 0; v < dh; ++v)
        for (int u = 0; u < dw; ++u) {
            const size_t j = (size_t)v * dw + u;
            if (!mask[j] || depth[j] == 0) continue;
            const double z = depth[j] * scale;
            const double x = (u - dcx) * z / dfx;
            const double y = (v - dcy) * z / dfy;
            const double xc = R[0] * x + R[1] * y + R[2] * z + t[0];
            const double yc = R[3] * x + R[4] * y + R[5] * z + t[1];
            const double zc = R[6] * x + R[7] * y + R[8] * z + t[2];
            if (zc <= 0.0) continue;
            const long uc = lround(cfx * xc / zc + ccx);
            const long vc = lround(cfy * yc / zc + ccy);
            if (uc < 0 || uc >= cw || vc < 0 || vc >= ch) continue;
            scratch[(size_t)vc * cw + uc] = 1;
        }
    orc_dilate(scratch, out, cw, ch, radius);
}

/* ------------------------------------------------------------------------
 * Synthetic scenes, synthetic.cpp:64-195 (counter-hash generator).
 * ---------------------------------------------------------------------- */
#define ORC_MAX_OBJ 4
#define ORC_MAX_WP 8
#define ORC_MAX_EV 16

typedef struct {
    int width, height, frame_count;
    uint64_t seed;
    int base_depth_mm, depth_texture_mm, color_texture;
    int n_obj;
    struct {
        int w, h, depth_offset_mm;
        uint8_t color[3];
        int n_wp;
        int wp_frame[ORC_MAX_WP];
        double wp_x[ORC_MAX_WP], wp_y[ORC_MAX_WP];
    } obj[ORC_MAX_OBJ];
    int n_illum;
    int il_start[ORC_MAX_EV], il_end[ORC_MAX_EV];
    double il_gain[ORC_MAX_EV];
    int n_shadow;
    int sh_start[ORC_MAX_EV], sh_end[ORC_MAX_EV], sh_rect[ORC_MAX_EV][4];
    double sh_darken[ORC_MAX_EV];
    int n_flicker;
    int fl_start[ORC_MAX_EV], fl_end[ORC_MAX_EV], fl_rect[ORC_MAX_EV][4];
    double fl_color_sigma[ORC_MAX_EV], fl_depth_sigma[ORC_MAX_EV];
    double noise_color_sigma, noise_depth_sigma;
} orc_scene;

static uint64_t orc_splitmix(uint64_t z) { /* synthetic.cpp:14-19 */
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

uint64_t orc_hash(uint64_t seed, uint64_t stream, uint64_t frame, uint64_t pixel,
                  uint64_t channel) { /* synthetic.cpp:66-74 */
    uint64_t h = orc_splitmix(seed ^ 0x6a09e667f3bcc908ULL);
    h = orc_splitmix(h ^ stream);
    h = orc_splitmix(h ^ frame);
    h = orc_splitmix(h ^ pixel);
    return orc_splitmix(h ^ channel);
}

double orc_gauss(uint64_t seed, uint64_t stream, uint64_t frame, uint64_t pixel,
                 uint64_t channel) { /* synthetic.cpp:76-83, Box-Muller */
    const uint64_t h = orc_hash(seed, stream, frame, pixel, channel);
    const double u1 = ((double)(h >> 32) + 1.0) / 4294967297.0;
    const double u2 = (double)(h & 0xffffffffULL) / 4294967296.0;
    return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2);
}

/* synthetic.cpp:37-56: piecewise-linear waypoint track, lround'ed corner. */
static void orc_obj_rect(const orc_scene* s, int o, int frame, int* rx, int* ry) {
    const int n = s->obj[o].n_wp;
    double x = s->obj[o].wp_x[0], y = s->obj[o].wp_y[0];
    if (frame >= s->obj[o].wp_frame[n - 1]) {
        x = s->obj[o].wp_x[n - 1];
        y = s->obj[o].wp_y[n - 1];
    } else if (frame > s->obj[o].wp_frame[0]) {
        for (int i = 1; i < n; ++i) {
            if (frame <= s->obj[o].wp_frame[i]) {
                const double t = (double)(frame - s->obj[o].wp_frame[i - 1]) /
                                 (double)(s->obj[o].wp_frame[i] - s->obj[o].wp_frame[i - 1]);
                x = s->obj[o].wp_x[i - 1] + t * (s->obj[o].wp_x[i] - s->obj[o].wp_x[i - 1]);
                y = s->obj[o].wp_y[i - 1] + t * (s->obj[o].wp_y[i] - s->obj[o].wp_y[i - 1]);
                break;
            }
        }
    }
    *rx = (int)lround(x);
    *ry = (int)lround(y);
}

static int orc_in(const int rect[4], int x, int y) {
    return x >= rect[0] && x < rect[0] + rect[2] && y >= rect[1] && y < rect[1] + rect[3];
}

static uint8_t orc_u8(double v) {
    long q = lround(v);
    if (q < 0) q = 0;
    if (q > 255) q = 255;
    return (uint8_t)q;
}

/* render_frame, synthetic.cpp:119-195.  Streams: 1 bg colour texture,
 * 2 bg depth texture, 3 sensor colour, 4 sensor depth, 5/6 flicker. */
void orc_render(const orc_scene* s, int frame, uint8_t* R, uint8_t* G, uint8_t* B,
                uint16_t* D, uint8_t* gt) {
    const int w = s->width, h = s->height;
    double gain = 1.0;
    for (int e = 0; e < s->n_illum; ++e)
        if (frame >= s->il_start[e] && frame < s->il_end[e]) gain *= s->il_gain[e];
    int orect[ORC_MAX_OBJ][4];
    for (int o = 0; o < s->n_obj; ++o) {
        orc_obj_rect(s, o, frame, &orect[o][0], &orect[o][1]);
        orect[o][2] = s->obj[o].w;
        orect[o][3] = s->obj[o].h;
    }
    const uint64_t seed = s->seed;
    const double span = 2.0 * s->color_texture + 1.0;
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            const uint64_t pix = (uint64_t)y * w + x;
            double base[3] = {60.0 + 90.0 * x / w, 70.0 + 90.0 * y / h,
                              80.0 + 80.0 * (x + y) / (w + h)};
            for (int c = 0; c < 3; ++c) {
                const uint64_t t = orc_hash(seed, 1, 0, pix, c);
                base[c] += (double)(t % (uint64_t)span) - s->color_texture;
            }
            double depth = s->base_depth_mm;
            if (s->depth_texture_mm > 0) {
                const uint64_t t = orc_hash(seed, 2, 0, pix, 0);
                depth += (double)(t % (uint64_t)(2 * s->depth_texture_mm + 1)) -
                         s->depth_texture_mm;
            }
            int top = -1;
            for (int o = 0; o < s->n_obj; ++o)
                if (orc_in(orect[o], x, y)) top = o;
            uint8_t label = 0;
            if (top >= 0) {
                for (int c = 0; c < 3; ++c) base[c] = s->obj[top].color[c];
                depth -= s->obj[top].depth_offset_mm;
                label = 1;
            }
            double col[3] = {base[0] * gain, base[1] * gain, base[2] * gain};
            for (int e = 0; e < s->n_shadow; ++e)
                if (frame >= s->sh_start[e] && frame < s->sh_end[e] && orc_in(s->sh_rect[e], x, y))
                    for (int c = 0; c < 3; ++c) col[c] *= s->sh_darken[e];
            for (int e = 0; e < s->n_flicker; ++e) {
                if (frame < s->fl_start[e] || frame >= s->fl_end[e] || !orc_in(s->fl_rect[e], x, y))
                    continue;
                for (int c = 0; c < 3; ++c)
                    col[c] += s->fl_color_sigma[e] * orc_gauss(seed, 5, frame, pix, c);
                depth += s->fl_depth_sigma[e] * orc_gauss(seed, 6, frame, pix, 0);
            }
            for (int c = 0; c < 3; ++c)
                col[c] += s->noise_color_sigma * orc_gauss(seed, 3, frame, pix, c);
            depth += s->noise_depth_sigma * orc_gauss(seed, 4, frame, pix, 0);
            const size_t j = (size_t)pix;
            R[j] = orc_u8(col[0]);
            G[j] = orc_u8(col[1]);
            B[j] = orc_u8(col[2]);
            long dq = lround(depth);
            if (dq < 1) dq = 1;
            if (dq > 65535) dq = 65535;
            D[j] = (uint16_t)dq;
            if (gt) gt[j] = label;
        }
}

/* builtin_scenario, synthetic.cpp:234-273.  name 'A' or 'B'; returns 0 ok. */
int orc_scene_builtin(orc_scene* s, char name) {
    memset(s, 0, sizeof *s);
    s->width = 640;
    s->height = 480;
    s->frame_count = 300;
    s->seed = 1;
    s->base_depth_mm = 2000;
    s->depth_texture_mm = 30;
    s->color_texture = 8;
    s->noise_color_sigma = 1.0;
    s->noise_depth_sigma = 1.0;
    s->n_obj = 1;
    s->obj[0].w = 24;
    s->obj[0].h = 24;
    s->obj[0].depth_offset_mm = 400;
    s->obj[0].color[0] = 230;
    s->obj[0].color[1] = 40;
    s->obj[0].color[2] = 220;
    s->obj[0].n_wp = 2;
    s->obj[0].wp_frame[0] = 0;
    s->obj[0].wp_x[0] = 40;
    s->obj[0].wp_y[0] = 100;
    s->obj[0].wp_frame[1] = 299;
    s->obj[0].wp_x[1] = 600;
    s->obj[0].wp_y[1] = 320;
    if (name == 'A') {
        s->n_illum = 2;
        s->il_start[0] = 100, s->il_end[0] = 112, s->il_gain[0] = 1.5;
        s->il_start[1] = 200, s->il_end[1] = 212, s->il_gain[1] = 0.6;
        s->n_shadow = 1;
        s->sh_start[0] = 150, s->sh_end[0] = 180, s->sh_darken[0] = 0.6;
        s->sh_rect[0][0] = 300, s->sh_rect[0][1] = 300, s->sh_rect[0][2] = 200,
        s->sh_rect[0][3] = 120;
        s->n_flicker = 1;
        s->fl_start[0] = 0, s->fl_end[0] = 300;
        s->fl_rect[0][0] = 40, s->fl_rect[0][1] = 40, s->fl_rect[0][2] = 80, s->fl_rect[0][3] = 60;
        s->fl_color_sigma[0] = 3.0, s->fl_depth_sigma[0] = 30.0;
        return 0;
    }
    if (name == 'B') {
        static const double gains[10] = {1.4, 0.7, 1.25, 0.8, 1.35, 0.75, 1.2, 0.85, 1.3, 0.9};
        s->n_illum = 10;
        for (int i = 0; i < 10; ++i) {
            s->il_start[i] = 30 + 25 * i;
            s->il_end[i] = 30 + 25 * (i + 1);
            s->il_gain[i] = gains[i];
        }
        s->n_flicker = 1;
        s->fl_start[0] = 0, s->fl_end[0] = 300;
        s->fl_rect[0][0] = 400, s->fl_rect[0][1] = 60, s->fl_rect[0][2] = 160,
        s->fl_rect[0][3] = 120;
        s->fl_color_sigma[0] = 12.0, s->fl_depth_sigma[0] = 40.0;
        s->noise_color_sigma = 1.5;
        s->noise_depth_sigma = 2.0;
        return 0;
    }
    return 1;
}

size_t orc_scene_sizeof(void) { return sizeof(orc_scene); }
