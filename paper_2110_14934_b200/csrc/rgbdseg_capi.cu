// rgbdseg_capi.cu -- C-ABI host runtime (include/rgbdseg_c.h).
//
// Owns device memory, CUDA streams and events for banks, fusion states and
// processors, and drives the sm_100a kernels in rgbdseg_kernels.cu.  The
// reference's executor (parallel_for_rows, engine.cpp:14-37) becomes the CUDA
// grid; its 3-stage ingest/process/emit pipeline (run_pipeline,
// engine.hpp:54-139) becomes H2D / kernel / D2H on three CUDA streams chained
// by events, double-buffered over pixel chunks of a frame and across frames.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/rgbdseg_c.h"
#include "rgbdseg_kernels.cuh"

using namespace rgbdseg_b200;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    return fail(e == cudaErrorMemoryAllocation ? RGBDSEG_ENOMEM : RGBDSEG_ECUDA,
                std::string(what) + ": " + cudaGetErrorString(e));
}

#define CU(call)                                                   \
    do {                                                           \
        cudaError_t e_ = (call);                                   \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call);        \
    } while (0)

struct DeviceGuard {
    int prev = 0;
    bool ok = false;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) == cudaSuccess && cudaSetDevice(dev) == cudaSuccess) ok = true;
    }
    ~DeviceGuard() {
        if (ok) cudaSetDevice(prev);
    }
};

#define GUARD(dev)                                                              \
    DeviceGuard guard_(dev);                                                    \
    if (!guard_.ok) return cuda_fail(cudaGetLastError(), "cudaSetDevice")

// MixtureConfig::validate, mixture.cpp:9-24 (same messages).
int validate_cfg(const rgbdseg_mixture_cfg* c) {
    if (!c) return fail(RGBDSEG_EINVAL, "MixtureConfig: null");
    if (c->components < 3 || c->components > 5)
        return fail(RGBDSEG_EINVAL, "MixtureConfig: components must be in [3,5]");
    if (!(c->learning_rate > 0.0f && c->learning_rate < 1.0f))
        return fail(RGBDSEG_EINVAL, "MixtureConfig: learning_rate must be in (0,1)");
    if (!(c->background_threshold > 0.0f && c->background_threshold < 1.0f))
        return fail(RGBDSEG_EINVAL, "MixtureConfig: background_threshold must be in (0,1)");
    if (!(c->match_lambda > 0.0f))
        return fail(RGBDSEG_EINVAL, "MixtureConfig: match_lambda must be positive");
    if (!(c->initial_sigma > 0.0f))
        return fail(RGBDSEG_EINVAL, "MixtureConfig: initial_sigma must be positive");
    if (!(c->initial_weight > 0.0f && c->initial_weight < 1.0f))
        return fail(RGBDSEG_EINVAL, "MixtureConfig: initial_weight must be in (0,1)");
    if (!(c->variance_floor > 0.0f))
        return fail(RGBDSEG_EINVAL, "MixtureConfig: variance_floor must be positive");
    return RGBDSEG_OK;
}

MixCfg to_k(const rgbdseg_mixture_cfg& c) {
    // gmm_step_fast divides by max(w, alpha): alpha must sit in its exact range
    const int fast = c.learning_rate >= 0x1p-60f && c.learning_rate < 0x1p61f;
    return MixCfg{c.learning_rate,  c.match_lambda,   c.background_threshold,
                  c.initial_sigma, c.initial_weight, c.variance_floor, fast, 0.0f, 0.0f};
}

// to_k plus the untouched-component constants of a bank (gmm_step_fast's
// kVirt): sigma = RN(sqrt(vvar)) (sqrtf is correctly rounded, like the
// device's exact sequence) and band = RN(lambda * sigma).
MixCfg to_k(const rgbdseg_mixture_cfg& c, float vvar) {
    MixCfg k = to_k(c);
    k.vsd = std::sqrt(vvar);
    k.vband = c.match_lambda * k.vsd;
    return k;
}

// Pointer classification with a small direct-mapped cache: a host address
// can never become a device address under UVA (disjoint ranges), so a cached
// "device" / "host" verdict stays valid for the address; callers pass the
// same frame buffers every frame.
bool on_device(const void* p) {
    if (!p) return false;
    struct Entry {
        const void* p;
        bool dev;
    };
    thread_local Entry cache[64] = {};
    const size_t slot = (reinterpret_cast<uintptr_t>(p) >> 8) & 63;
    if (cache[slot].p == p) return cache[slot].dev;
    cudaPointerAttributes a;
    bool dev = false;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
    } else {
        dev = a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
    }
    cache[slot] = Entry{p, dev};
    return dev;
}

size_t pitch_for(size_t npx) { return (npx + 63) & ~size_t(63); }  // 256-byte planes

int check_dims(int w, int h, int streams) {
    if (w <= 0 || h <= 0) return fail(RGBDSEG_EINVAL, "Plane: non-positive dimensions");
    if (streams <= 0) return fail(RGBDSEG_EINVAL, "streams must be positive");
    return RGBDSEG_OK;
}

template <typename T>
int dalloc(T** p, size_t n) {
    *p = nullptr;
    if (n == 0) return RGBDSEG_OK;
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), n * sizeof(T));
    if (e != cudaSuccess) {
        *p = nullptr;
        return cuda_fail(e, "cudaMalloc");
    }
    return RGBDSEG_OK;
}

template <typename T>
void dfree(T*& p) {
    if (p) cudaFree(p);
    p = nullptr;
}

// Scratch device buffer that grows on demand.
struct Scratch {
    void* p = nullptr;
    size_t bytes = 0;
    int get(size_t want, void** out) {
        if (want > bytes) {
            if (p) cudaFree(p);
            p = nullptr;
            bytes = 0;
            cudaError_t e = cudaMalloc(&p, want);
            if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(scratch)");
            bytes = want;
        }
        *out = p;
        return RGBDSEG_OK;
    }
    ~Scratch() {
        if (p) cudaFree(p);
    }
};

// Stage `bytes` of a host-or-device source into device memory: device
// pointers are used in place, host pointers are copied into `scratch`.
int stage_in(const void* src, size_t bytes, Scratch& scratch, const void** dev, cudaStream_t s) {
    if (!src) return fail(RGBDSEG_EINVAL, "null input plane");
    if (on_device(src)) {
        *dev = src;
        return RGBDSEG_OK;
    }
    void* d;
    if (int rc = scratch.get(bytes, &d)) return rc;
    CU(cudaMemcpyAsync(d, src, bytes, cudaMemcpyDefault, s));
    *dev = d;
    return RGBDSEG_OK;
}

}  // namespace

// ============================================================== handles
struct rgbdseg_bank {
    int width, height, streams, mode, M, C, device;
    size_t npx, nblocks;
    rgbdseg_mixture_cfg cfg;
    float* state = nullptr;  // tiled: nblocks * bank_stride(M, C) floats
    cudaStream_t stream = nullptr;
    Scratch s_r, s_g, s_b, s_mask, s_plane;
    float vvar = 0.0f;  // sigma0^2 of the creation cfg: an untouched component's variance
    // Set when the bank belongs to a processor (rgbdseg_processor_color_bank):
    // every call on the borrowed handle first drains the processor's streams.
    rgbdseg_processor* owner = nullptr;
    // Layout view; with a call's cfg it also says whether that call's
    // init_mixture may mark components untouched (same sigma0^2, and the
    // fast step's variance range, gmm_pixel.cuh kVarLo/kVarHi).
    BankView view() const { return BankView{state, M, C, vvar, 0}; }
    BankView view(const rgbdseg_mixture_cfg& c) const {
        BankView v = view();
        uint32_t vb, cb;
        const float var0 = c.initial_sigma * c.initial_sigma;
        std::memcpy(&vb, &vvar, 4);
        std::memcpy(&cb, &var0, 4);
        v.vinit = vb == cb && vb >= kVarLo && vb < kVarHi;
        return v;
    }
};

struct rgbdseg_fusion {
    size_t npx;
    int limit, device;
    rgbdseg_processor* owner = nullptr;  // as rgbdseg_bank::owner
    uint8_t* out = nullptr;
    int8_t* cpt = nullptr;
    cudaStream_t stream = nullptr;
    Scratch s_rgb, s_dep;
};

// A device staging slot for one chunk of host frames: r | g | b | depth back
// to back (a planar host frame moves in one or two DMAs), mask outputs and
// the ground truth for the evaluation epilogue.
struct Slot {
    uint8_t *r = nullptr, *g = nullptr, *b = nullptr, *gt = nullptr;
    uint16_t* d = nullptr;
    uint8_t *rgbm = nullptr, *depm = nullptr, *fused = nullptr;
};

struct rgbdseg_processor {
    rgbdseg_processor_cfg cfg;
    rgbdseg_bank* color = nullptr;
    rgbdseg_bank* depth = nullptr;
    rgbdseg_fusion* fusion = nullptr;
    // Host frames: chunk c of every frame runs H2D -> K1 -> D2H on cs[c % 2]
    // with slot[c % 2].  Stream order alone provides every dependency (the
    // same pixels of consecutive frames stay on one stream; a slot is reused
    // only by its own stream), and the two streams overlap each other.
    cudaStream_t cs[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};  // cross-stream joins (mode switches, counts)
    cudaEvent_t ev_k[2] = {nullptr, nullptr};  // single-chunk frames: K1 of the frame on cs[i]
    cudaEvent_t ev_user = nullptr;                // rgbdseg_processor_wait_stream
    cudaEvent_t ev_done[2] = {nullptr, nullptr};  // rgbdseg_processor_signal_stream
    size_t npx = 0, chunk = 0;
    int nchunks = 1;
    Slot slot[2];
    int last_mode = 0;  // 0 none, 1 host chunks (both streams), 2 single stream cs[0]
    int64_t frames = 0;
    int variant = kAuto;
    // unregistered sequences: whole-frame scratch (inputs, masks, splat)
    Scratch u_in, u_masks, u_gt;
    Scratch counts;  // evaluation epilogue: [streams][3][4] uint64
    // near-threshold report (rgbdseg_processor_set_near_threshold)
    float near_rel = 0.0f;
    Scratch near_counts;  // [colour, depth] uint64
    uint64_t near_pixel_frames = 0;
    // Single-chunk host frames: the mask read-back of frame k is issued after
    // the upload of frame k+1 (or at sync).  The copy engine takes copies in
    // issue order, so a read-back queued right behind its kernel would hold
    // the next upload until that kernel ends (VGA: 47 -> 32 us per frame).
    struct {
        bool on = false;
        int lane = 0;
        size_t n = 0;
        uint8_t *fused = nullptr, *rgb = nullptr, *depth = nullptr;
    } pend;
};

// Issue the deferred read-back, on the stream of the frame it belongs to (so
// it stays ahead of that slot's next use).
static int flush_emit(rgbdseg_processor* p) {
    if (!p->pend.on) return RGBDSEG_OK;
    p->pend.on = false;
    const Slot& sl = p->slot[p->pend.lane];
    cudaStream_t st = p->cs[p->pend.lane];
    const size_t n = p->pend.n;
    const cudaMemcpyKind d2h = cudaMemcpyDeviceToHost;
    if (p->pend.fused) CU(cudaMemcpyAsync(p->pend.fused, sl.fused, n, d2h, st));
    if (p->pend.rgb) CU(cudaMemcpyAsync(p->pend.rgb, sl.rgbm, n, d2h, st));
    if (p->pend.depth) CU(cudaMemcpyAsync(p->pend.depth, sl.depm, n, d2h, st));
    return RGBDSEG_OK;
}

// A bank / fusion handle borrowed from a processor: finish the processor's
// queued frames (and its deferred read-back) before the handle's own stream
// reads or writes the state.
static int drain_owner(rgbdseg_processor* owner);

extern "C" {

const char* rgbdseg_last_error(void) { return g_err.c_str(); }
const char* rgbdseg_version(void) { return "rgbdseg-b200 0.1 (sm_100a)"; }
uint64_t rgbdseg_launch_count(void) { return launches(); }

void rgbdseg_mixture_defaults(rgbdseg_mixture_cfg* out) {
    *out = rgbdseg_mixture_cfg{3, 0.05f, 2.5f, 0.8f, 15.0f, 0.05f, 4.0f};
}

int rgbdseg_mixture_validate(const rgbdseg_mixture_cfg* cfg) { return validate_cfg(cfg); }

// ------------------------------------------------------------ per pixel
int rgbdseg_init_mixtures(const float* values, int channels, size_t n,
                          const rgbdseg_mixture_cfg* cfg, rgbdseg_pixel_mixture* out,
                          int device) {
    if (int rc = validate_cfg(cfg)) return rc;  // init_mixture validates (mixture.cpp:59)
    if (channels < 1 || channels > 4)
        return fail(RGBDSEG_EINVAL, "init_mixture: bad observation dimensionality");
    if (n == 0) return RGBDSEG_OK;
    if (!values || !out) return fail(RGBDSEG_EINVAL, "init_mixture: null buffer");
    GUARD(device);
    float* dv;
    PixRec* dr;
    if (int rc = dalloc(&dv, n * channels)) return rc;
    if (int rc = dalloc(&dr, n)) {
        dfree(dv);
        return rc;
    }
    cudaError_t e = cudaMemcpy(dv, values, n * channels * sizeof(float), cudaMemcpyDefault);
    if (e == cudaSuccess) e = launch_mix_init(dv, channels, n, to_k(*cfg), cfg->components, dr, 0);
    if (e == cudaSuccess) e = cudaMemcpy(out, dr, n * sizeof(PixRec), cudaMemcpyDefault);
    dfree(dv);
    dfree(dr);
    if (e != cudaSuccess) return cuda_fail(e, "init_mixtures");
    return RGBDSEG_OK;
}

int rgbdseg_step_mixtures(rgbdseg_pixel_mixture* mix, const float* values, int channels,
                          size_t n, const rgbdseg_mixture_cfg* cfg, uint8_t* labels, int device) {
    static_assert(sizeof(PixRec) == sizeof(rgbdseg_pixel_mixture), "record layout");
    if (!cfg) return fail(RGBDSEG_EINVAL, "step_pixel: null config");
    if (channels < 1 || channels > 4)
        return fail(RGBDSEG_EINVAL, "step_pixel: bad observation dimensionality");
    if (n == 0) return RGBDSEG_OK;
    if (!mix || !values) return fail(RGBDSEG_EINVAL, "step_pixel: null buffer");
    // Shapes are checked before anything runs, so a rejected call leaves
    // every record untouched (the kernel's 255 label stays a backstop).
    {
        const bool host = !on_device(mix);
        std::vector<rgbdseg_pixel_mixture> hm;
        const rgbdseg_pixel_mixture* recs = mix;
        if (!host) {
            GUARD(device);
            hm.resize(n);
            CU(cudaMemcpy(hm.data(), mix, n * sizeof(PixRec), cudaMemcpyDeviceToHost));
            recs = hm.data();
        }
        for (size_t i = 0; i < n; ++i)
            if (recs[i].components < 3 || recs[i].components > 5 || recs[i].channels != channels)
                return fail(RGBDSEG_EINVAL,
                            "step_pixel: record " + std::to_string(i) +
                                " has components outside [3,5] or a channel-count mismatch");
    }
    GUARD(device);
    float* dv;
    PixRec* dr;
    uint8_t* dl;
    if (int rc = dalloc(&dv, n * channels)) return rc;
    if (int rc = dalloc(&dr, n)) {
        dfree(dv);
        return rc;
    }
    if (int rc = dalloc(&dl, n)) {
        dfree(dv);
        dfree(dr);
        return rc;
    }
    std::vector<uint8_t> hl(n);
    cudaError_t e = cudaMemcpy(dv, values, n * channels * sizeof(float), cudaMemcpyDefault);
    if (e == cudaSuccess) e = cudaMemcpy(dr, mix, n * sizeof(PixRec), cudaMemcpyDefault);
    if (e == cudaSuccess)
        e = launch_mix_step(dr, dv, channels, n, to_k(*cfg), dl, 0);
    if (e == cudaSuccess) e = cudaMemcpy(mix, dr, n * sizeof(PixRec), cudaMemcpyDefault);
    if (e == cudaSuccess) e = cudaMemcpy(hl.data(), dl, n, cudaMemcpyDeviceToHost);
    dfree(dv);
    dfree(dr);
    dfree(dl);
    if (e != cudaSuccess) return cuda_fail(e, "step_mixtures");
    for (size_t i = 0; i < n; ++i)
        if (hl[i] == 255)
            return fail(RGBDSEG_EINVAL,
                        "step_pixel: record " + std::to_string(i) +
                            " has components outside [3,5] or a channel-count mismatch");
    if (labels) {
        if (on_device(labels)) {
            CU(cudaMemcpy(labels, hl.data(), n, cudaMemcpyHostToDevice));
        } else {
            std::memcpy(labels, hl.data(), n);
        }
    }
    return RGBDSEG_OK;
}

// match_component / classify / update_mixture (mixture.hpp:45-56) batched on
// the GPU.  Shapes (and, for classify/update, the matched indices) are
// validated on the host first, so a rejected call changes nothing.
static int mix_op(int op, rgbdseg_pixel_mixture* mix, const float* values, int channels,
                  size_t n, const rgbdseg_mixture_cfg* cfg, int32_t* matched, uint8_t* labels,
                  int device, const char* who) {
    if (!cfg) return fail(RGBDSEG_EINVAL, std::string(who) + ": null config");
    if (n == 0) return RGBDSEG_OK;
    if (!mix || !matched || (op != kOpClassify && !values) || (op == kOpClassify && !labels))
        return fail(RGBDSEG_EINVAL, std::string(who) + ": null buffer");
    if (op != kOpClassify && (channels < 1 || channels > 4))
        return fail(RGBDSEG_EINVAL, std::string(who) + ": bad observation dimensionality");
    GUARD(device);
    std::vector<rgbdseg_pixel_mixture> hm;
    const rgbdseg_pixel_mixture* recs = mix;
    if (on_device(mix)) {
        hm.resize(n);
        CU(cudaMemcpy(hm.data(), mix, n * sizeof(PixRec), cudaMemcpyDeviceToHost));
        recs = hm.data();
    }
    std::vector<int32_t> hmt;
    const int32_t* mt = matched;
    if (op != kOpMatch && on_device(matched)) {
        hmt.resize(n);
        CU(cudaMemcpy(hmt.data(), matched, n * 4, cudaMemcpyDeviceToHost));
        mt = hmt.data();
    }
    for (size_t i = 0; i < n; ++i) {
        const int M = recs[i].components;
        if (M < 3 || M > 5 || recs[i].channels < 1 || recs[i].channels > 4 ||
            (op != kOpClassify && recs[i].channels != channels))
            return fail(RGBDSEG_EINVAL, std::string(who) + ": record " + std::to_string(i) +
                                            " has components outside [3,5] or a channel-count "
                                            "mismatch");
        if (op != kOpMatch && (mt[i] < -1 || mt[i] >= M))
            return fail(RGBDSEG_EINVAL, std::string(who) + ": record " + std::to_string(i) +
                                            " matched index out of range");
    }
    PixRec* dr = nullptr;
    float* dv = nullptr;
    int* dm = nullptr;
    uint8_t* dl = nullptr;
    int rc = dalloc(&dr, n);
    if (!rc && op != kOpClassify) rc = dalloc(&dv, n * channels);
    if (!rc) rc = dalloc(&dm, n);
    if (!rc && op == kOpClassify) rc = dalloc(&dl, n);
    cudaError_t e = cudaSuccess;
    if (!rc) {
        e = cudaMemcpy(dr, recs, n * sizeof(PixRec), cudaMemcpyDefault);
        if (e == cudaSuccess && dv) e = cudaMemcpy(dv, values, n * channels * 4, cudaMemcpyDefault);
        if (e == cudaSuccess && op != kOpMatch) e = cudaMemcpy(dm, mt, n * 4, cudaMemcpyDefault);
        if (e == cudaSuccess) e = launch_mix_op(dr, dv, n, to_k(*cfg), op, dm, dl, 0);
        if (e == cudaSuccess && op == kOpMatch) e = cudaMemcpy(matched, dm, n * 4, cudaMemcpyDefault);
        if (e == cudaSuccess && op == kOpClassify) e = cudaMemcpy(labels, dl, n, cudaMemcpyDefault);
        if (e == cudaSuccess && op == kOpUpdate)
            e = cudaMemcpy(mix, dr, n * sizeof(PixRec), cudaMemcpyDefault);
        if (e != cudaSuccess) rc = cuda_fail(e, who);
    }
    dfree(dr);
    dfree(dv);
    dfree(dm);
    dfree(dl);
    return rc;
}

int rgbdseg_match_components(const rgbdseg_pixel_mixture* mix, const float* values, int channels,
                             size_t n, const rgbdseg_mixture_cfg* cfg, int32_t* matched,
                             int device) {
    return mix_op(kOpMatch, const_cast<rgbdseg_pixel_mixture*>(mix), values, channels, n, cfg,
                  matched, nullptr, device, "match_component");
}

int rgbdseg_classify_mixtures(const rgbdseg_pixel_mixture* mix, const int32_t* matched, size_t n,
                              const rgbdseg_mixture_cfg* cfg, uint8_t* labels, int device) {
    return mix_op(kOpClassify, const_cast<rgbdseg_pixel_mixture*>(mix), nullptr, 0, n, cfg,
                  const_cast<int32_t*>(matched), labels, device, "classify");
}

int rgbdseg_update_mixtures(rgbdseg_pixel_mixture* mix, const float* values, int channels,
                            size_t n, const int32_t* matched, const rgbdseg_mixture_cfg* cfg,
                            int device) {
    return mix_op(kOpUpdate, mix, values, channels, n, cfg, const_cast<int32_t*>(matched),
                  nullptr, device, "update_mixture");
}

// ------------------------------------------------------------ banks
int rgbdseg_bank_create(int width, int height, int streams, int mode,
                        const rgbdseg_mixture_cfg* cfg, int device, rgbdseg_bank** out) {
    *out = nullptr;
    if (int rc = check_dims(width, height, streams)) return rc;
    if (mode != RGBDSEG_COLOR3 && mode != RGBDSEG_DEPTH1 && mode != RGBDSEG_AUGMENTED4)
        return fail(RGBDSEG_EINVAL, "unknown bank mode");
    if (int rc = validate_cfg(cfg)) return rc;  // segmenter.cpp:26
    GUARD(device);
    auto* b = new rgbdseg_bank();
    b->width = width;
    b->height = height;
    b->streams = streams;
    b->mode = mode;
    b->M = cfg->components;
    b->C = mode == RGBDSEG_COLOR3 ? 3 : (mode == RGBDSEG_DEPTH1 ? 1 : 4);
    b->device = device;
    b->cfg = *cfg;
    b->vvar = cfg->initial_sigma * cfg->initial_sigma;  // k_bank_reset's fmul(sigma0, sigma0)
    b->npx = (size_t)width * height * streams;
    b->nblocks = (b->npx + kBlockPx - 1) / kBlockPx;
    int rc = dalloc(&b->state, b->nblocks * (size_t)bank_stride(b->M, b->C));
    if (!rc) {
        cudaError_t e = cudaStreamCreateWithFlags(&b->stream, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = launch_bank_reset(b->view(), cfg->initial_sigma, b->npx, b->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(b->stream);
        if (e != cudaSuccess) rc = cuda_fail(e, "bank_create");
    }
    if (rc) {
        rgbdseg_bank_destroy(b);
        return rc;
    }
    *out = b;
    return RGBDSEG_OK;
}

void rgbdseg_bank_destroy(rgbdseg_bank* b) {
    if (!b) return;
    DeviceGuard g(b->device);
    if (b->stream) cudaStreamSynchronize(b->stream);
    dfree(b->state);
    if (b->stream) cudaStreamDestroy(b->stream);
    delete b;
}

int rgbdseg_bank_planes(const rgbdseg_bank* b) { return b ? b->M * b->C + 2 * b->M : 0; }

int rgbdseg_bank_device_ptrs(const rgbdseg_bank* b, void** tiles, size_t* block_bytes,
                             size_t* nblocks) {
    if (!b) return fail(RGBDSEG_EINVAL, "bank_device_ptrs: null handle");
    if (tiles) *tiles = b->state;
    if (block_bytes) *block_bytes = (size_t)bank_stride(b->M, b->C) * sizeof(float);
    if (nblocks) *nblocks = b->nblocks;
    return RGBDSEG_OK;
}

// Flat plane <-> tiled bank through a gather/scatter kernel (device
// destinations directly, host ones through a device scratch plane).
static int bank_xfer(rgbdseg_bank* b, int plane, void* dst, const void* src) {
    if (plane != RGBDSEG_FLAGS_PLANE && (plane < 0 || plane >= rgbdseg_bank_planes(b)))
        return fail(RGBDSEG_EINVAL, "bank plane id out of range");
    const size_t bytes = b->npx * (plane == RGBDSEG_FLAGS_PLANE ? 1 : sizeof(float));
    const int pid = plane == RGBDSEG_FLAGS_PLANE ? -1 : plane;
    void* dev = const_cast<void*>(dst ? dst : src);
    const bool direct = on_device(dev);
    if (!direct) {
        if (int rc = b->s_plane.get(bytes, &dev)) return rc;
        if (src) CU(cudaMemcpyAsync(dev, src, bytes, cudaMemcpyDefault, b->stream));
    }
    if (dst) {
        CU(launch_bank_gather(b->view(), pid, b->npx, dev, b->stream));
        if (!direct) CU(cudaMemcpyAsync(dst, dev, bytes, cudaMemcpyDefault, b->stream));
    } else {
        CU(launch_bank_scatter(b->view(), pid, b->npx, dev, b->stream));
    }
    CU(cudaStreamSynchronize(b->stream));
    return RGBDSEG_OK;
}

int rgbdseg_bank_download(const rgbdseg_bank* b, int plane, void* dst) {
    if (!b) return fail(RGBDSEG_EINVAL, "bank_download: null handle");
    GUARD(b->device);
    if (int rc = drain_owner(b->owner)) return rc;
    return bank_xfer(const_cast<rgbdseg_bank*>(b), plane, dst, nullptr);
}

int rgbdseg_bank_upload(rgbdseg_bank* b, int plane, const void* src) {
    if (!b) return fail(RGBDSEG_EINVAL, "bank_upload: null handle");
    GUARD(b->device);
    if (int rc = drain_owner(b->owner)) return rc;
    return bank_xfer(b, plane, nullptr, src);
}

// run_bank's checks (segmenter.cpp:73-75) + mode checks (:109,:123).
static int bank_call_checks(const rgbdseg_bank* b, const rgbdseg_mixture_cfg* cfg, int mode,
                            const char* who) {
    if (!b) return fail(RGBDSEG_EINVAL, std::string(who) + ": null bank");
    if (b->mode != mode)
        return fail(RGBDSEG_EINVAL, std::string(who) + (mode == RGBDSEG_COLOR3   ? ": bank mode is not Color3"
                                                        : mode == RGBDSEG_DEPTH1 ? ": bank mode is not Depth1"
                                                                                 : ": bank mode is not Augmented4"));
    if (int rc = validate_cfg(cfg)) return rc;
    if (cfg->components != b->M)
        return fail(RGBDSEG_EINVAL, "segment: config component count does not match bank");
    return RGBDSEG_OK;
}

static int finish_mask(uint8_t* dev_mask, uint8_t* mask_out, size_t n, cudaStream_t s) {
    if (mask_out && dev_mask != mask_out)
        CU(cudaMemcpyAsync(mask_out, dev_mask, n, cudaMemcpyDefault, s));
    CU(cudaStreamSynchronize(s));
    return RGBDSEG_OK;
}

int rgbdseg_segment_color(rgbdseg_bank* b, const uint8_t* r, const uint8_t* g, const uint8_t* bl,
                          const rgbdseg_mixture_cfg* cfg, uint8_t* mask_out) {
    if (!b) return fail(RGBDSEG_EINVAL, "segment_color: null handle");
    if (int rc = bank_call_checks(b, cfg, RGBDSEG_COLOR3, "segment_color")) return rc;
    GUARD(b->device);
    if (int rc = drain_owner(b->owner)) return rc;
    const void *dr, *dg, *db;
    if (int rc = stage_in(r, b->npx, b->s_r, &dr, b->stream)) return rc;
    if (int rc = stage_in(g, b->npx, b->s_g, &dg, b->stream)) return rc;
    if (int rc = stage_in(bl, b->npx, b->s_b, &db, b->stream)) return rc;
    uint8_t* dm = nullptr;
    if (mask_out) {
        if (on_device(mask_out)) {
            dm = mask_out;
        } else {
            void* p;
            if (int rc = b->s_mask.get(b->npx, &p)) return rc;
            dm = static_cast<uint8_t*>(p);
        }
    }
    CU(launch_bank_color(b->view(*cfg), to_k(*cfg, b->vvar), (const uint8_t*)dr, (const uint8_t*)dg,
                         (const uint8_t*)db, dm, b->npx, b->stream));
    return finish_mask(dm, mask_out, b->npx, b->stream);
}

int rgbdseg_segment_depth(rgbdseg_bank* b, const uint16_t* depth_mm,
                          const rgbdseg_mixture_cfg* cfg, uint8_t* mask_out) {
    if (!b) return fail(RGBDSEG_EINVAL, "segment_depth: null handle");
    if (int rc = bank_call_checks(b, cfg, RGBDSEG_DEPTH1, "segment_depth")) return rc;
    GUARD(b->device);
    if (int rc = drain_owner(b->owner)) return rc;
    const void* dd;
    if (int rc = stage_in(depth_mm, b->npx * 2, b->s_r, &dd, b->stream)) return rc;
    uint8_t* dm = nullptr;
    if (mask_out) {
        if (on_device(mask_out)) {
            dm = mask_out;
        } else {
            void* p;
            if (int rc = b->s_mask.get(b->npx, &p)) return rc;
            dm = static_cast<uint8_t*>(p);
        }
    }
    CU(launch_bank_depth(b->view(*cfg), to_k(*cfg, b->vvar), (const uint16_t*)dd, dm, b->npx, b->stream));
    return finish_mask(dm, mask_out, b->npx, b->stream);
}

int rgbdseg_segment_augmented(rgbdseg_bank* b, const uint8_t* r, const uint8_t* g,
                              const uint8_t* bl, const uint16_t* depth_mm, float min_mm,
                              float max_mm, const rgbdseg_mixture_cfg* cfg, uint8_t* mask_out) {
    if (!b) return fail(RGBDSEG_EINVAL, "segment_augmented: null handle");
    if (int rc = bank_call_checks(b, cfg, RGBDSEG_AUGMENTED4, "segment_augmented")) return rc;
    if (!(max_mm > min_mm)) return fail(RGBDSEG_EINVAL, "config: augmented depth range is empty");
    GUARD(b->device);
    if (int rc = drain_owner(b->owner)) return rc;
    const void *dr, *dg, *db, *dd;
    if (int rc = stage_in(r, b->npx, b->s_r, &dr, b->stream)) return rc;
    if (int rc = stage_in(g, b->npx, b->s_g, &dg, b->stream)) return rc;
    if (int rc = stage_in(bl, b->npx, b->s_b, &db, b->stream)) return rc;
    if (int rc = stage_in(depth_mm, b->npx * 2, b->s_plane, &dd, b->stream)) return rc;
    uint8_t* dm = nullptr;
    if (mask_out) {
        if (on_device(mask_out)) {
            dm = mask_out;
        } else {
            void* p;
            if (int rc = b->s_mask.get(b->npx, &p)) return rc;
            dm = static_cast<uint8_t*>(p);
        }
    }
    CU(launch_bank_aug(b->view(*cfg), to_k(*cfg, b->vvar), (const uint8_t*)dr, (const uint8_t*)dg,
                       (const uint8_t*)db, (const uint16_t*)dd, min_mm, max_mm, dm, b->npx,
                       b->stream));
    return finish_mask(dm, mask_out, b->npx, b->stream);
}

// ------------------------------------------------------------ fusion
int rgbdseg_fusion_create(int width, int height, int streams, int initial_label,
                          int counter_limit, int device, rgbdseg_fusion** out) {
    *out = nullptr;
    if (int rc = check_dims(width, height, streams)) return rc;
    // reset_state, fusion.cpp:7-15
    if (counter_limit < 1)
        return fail(RGBDSEG_EINVAL, "reset_state: counter_limit must be >= 1");
    if (initial_label < 0 || initial_label > 1)
        return fail(RGBDSEG_EINVAL, "reset_state: label must be 0 or 1");
    GUARD(device);
    auto* f = new rgbdseg_fusion();
    f->npx = (size_t)width * height * streams;
    f->limit = counter_limit;
    f->device = device;
    int rc = dalloc(&f->out, pitch_for(f->npx));
    if (!rc) rc = dalloc(&f->cpt, pitch_for(f->npx));
    if (!rc) {
        cudaError_t e = cudaStreamCreateWithFlags(&f->stream, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaMemsetAsync(f->out, initial_label, f->npx, f->stream);
        if (e == cudaSuccess) e = cudaMemsetAsync(f->cpt, 0, f->npx, f->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(f->stream);
        if (e != cudaSuccess) rc = cuda_fail(e, "fusion_create");
    }
    if (rc) {
        rgbdseg_fusion_destroy(f);
        return rc;
    }
    *out = f;
    return RGBDSEG_OK;
}

void rgbdseg_fusion_destroy(rgbdseg_fusion* f) {
    if (!f) return;
    DeviceGuard g(f->device);
    if (f->stream) cudaStreamSynchronize(f->stream);
    dfree(f->out);
    dfree(f->cpt);
    if (f->stream) cudaStreamDestroy(f->stream);
    delete f;
}

int rgbdseg_fusion_step(rgbdseg_fusion* f, const uint8_t* rgb_mask, const uint8_t* depth_mask,
                        uint8_t* out_copy) {
    if (!f) return fail(RGBDSEG_EINVAL, "fusion_step: null handle");
    GUARD(f->device);
    if (int rc = drain_owner(f->owner)) return rc;
    const void *dr, *dd;
    if (int rc = stage_in(rgb_mask, f->npx, f->s_rgb, &dr, f->stream)) return rc;
    if (int rc = stage_in(depth_mask, f->npx, f->s_dep, &dd, f->stream)) return rc;
    uint8_t* oc = (out_copy && on_device(out_copy)) ? out_copy : nullptr;
    CU(launch_fuse(f->out, f->cpt, (const uint8_t*)dr, (const uint8_t*)dd, oc, f->limit, f->npx,
                   f->stream));
    if (out_copy && !oc) CU(cudaMemcpyAsync(out_copy, f->out, f->npx, cudaMemcpyDefault, f->stream));
    CU(cudaStreamSynchronize(f->stream));
    return RGBDSEG_OK;
}

int rgbdseg_fusion_download(const rgbdseg_fusion* f, uint8_t* out, int8_t* cpt) {
    if (!f) return fail(RGBDSEG_EINVAL, "fusion_download: null handle");
    GUARD(f->device);
    if (int rc = drain_owner(f->owner)) return rc;
    CU(cudaStreamSynchronize(f->stream));
    if (out) CU(cudaMemcpy(out, f->out, f->npx, cudaMemcpyDefault));
    if (cpt) CU(cudaMemcpy(cpt, f->cpt, f->npx, cudaMemcpyDefault));
    return RGBDSEG_OK;
}

int rgbdseg_fusion_set_counter_limit(rgbdseg_fusion* f, int counter_limit) {
    if (!f) return fail(RGBDSEG_EINVAL, "fusion_set_counter_limit: null handle");
    GUARD(f->device);
    if (int rc = drain_owner(f->owner)) return rc;
    CU(cudaStreamSynchronize(f->stream));
    f->limit = counter_limit;
    return RGBDSEG_OK;
}

int rgbdseg_fusion_upload(rgbdseg_fusion* f, const uint8_t* out, const int8_t* cpt) {
    if (!f) return fail(RGBDSEG_EINVAL, "fusion_upload: null handle");
    GUARD(f->device);
    if (int rc = drain_owner(f->owner)) return rc;
    CU(cudaStreamSynchronize(f->stream));
    if (out) CU(cudaMemcpy(f->out, out, f->npx, cudaMemcpyDefault));
    if (cpt) CU(cudaMemcpy(f->cpt, cpt, f->npx, cudaMemcpyDefault));
    return RGBDSEG_OK;
}

// ------------------------------------------------------------ registration
void rgbdseg_camera_rig_identity(rgbdseg_camera_rig* r, double fx, double fy, double cx,
                                 double cy) {
    std::memset(r, 0, sizeof *r);
    r->depth_fx = r->color_fx = fx;
    r->depth_fy = r->color_fy = fy;
    r->depth_cx = r->color_cx = cx;
    r->depth_cy = r->color_cy = cy;
    r->rotation[0] = r->rotation[4] = r->rotation[8] = 1.0;
    r->depth_scale = 1.0;
}

int rgbdseg_camera_rig_validate(const rgbdseg_camera_rig* r) {
    if (!r) return fail(RGBDSEG_EINVAL, "CameraRig: null");
    if (!(r->depth_fx > 0.0 && r->depth_fy > 0.0 && r->color_fx > 0.0 && r->color_fy > 0.0))
        return fail(RGBDSEG_EINVAL, "CameraRig: focal lengths must be positive");
    if (!(r->depth_scale > 0.0)) return fail(RGBDSEG_EINVAL, "CameraRig: depth_scale must be positive");
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {  // R^T R == I within 1e-9
            double dot = 0.0;
            for (int k = 0; k < 3; ++k) dot += r->rotation[k * 3 + i] * r->rotation[k * 3 + j];
            if (std::fabs(dot - (i == j ? 1.0 : 0.0)) > 1e-9)
                return fail(RGBDSEG_EINVAL, "CameraRig: rotation is not orthonormal");
        }
    return RGBDSEG_OK;
}

static RigDev to_dev(const rgbdseg_camera_rig& r) {
    RigDev d;
    d.dfx = r.depth_fx;
    d.dfy = r.depth_fy;
    d.dcx = r.depth_cx;
    d.dcy = r.depth_cy;
    d.cfx = r.color_fx;
    d.cfy = r.color_fy;
    d.ccx = r.color_cx;
    d.ccy = r.color_cy;
    for (int i = 0; i < 9; ++i) d.R[i] = r.rotation[i];
    for (int i = 0; i < 3; ++i) d.t[i] = r.translation_mm[i];
    d.scale = r.depth_scale;
    return d;
}

int rgbdseg_dilate_mask(const uint8_t* mask, int w, int h, int radius, uint8_t* out, int device) {
    if (int rc = check_dims(w, h, 1)) return rc;
    GUARD(device);
    const size_t n = (size_t)w * h;
    Scratch sin, sbuf;
    const void* din;
    if (int rc = stage_in(mask, n, sin, &din, 0)) return rc;
    void* buf;
    if (int rc = sbuf.get(2 * n, &buf)) return rc;
    uint8_t* tmp = static_cast<uint8_t*>(buf);
    uint8_t* res = on_device(out) ? out : tmp + n;
    CU(launch_dilate((const uint8_t*)din, tmp, res, w, h, 1, radius, 0));
    if (res != out) CU(cudaMemcpyAsync(out, res, n, cudaMemcpyDefault, 0));
    CU(cudaStreamSynchronize(0));
    return RGBDSEG_OK;
}

int rgbdseg_register_mask(const uint8_t* mask, const uint16_t* depth, int dw, int dh,
                          const rgbdseg_camera_rig* rig, int cw, int ch, int radius, uint8_t* out,
                          int device) {
    if (int rc = check_dims(dw, dh, 1)) return rc;
    if (int rc = check_dims(cw, ch, 1)) return rc;
    if (int rc = rgbdseg_camera_rig_validate(rig)) return rc;  // registration.cpp:57
    GUARD(device);
    const size_t nd = (size_t)dw * dh, nc = (size_t)cw * ch;
    Scratch sm, sd, sbuf;
    const void *dm, *dd;
    if (int rc = stage_in(mask, nd, sm, &dm, 0)) return rc;
    if (int rc = stage_in(depth, 2 * nd, sd, &dd, 0)) return rc;
    void* buf;
    if (int rc = sbuf.get(3 * nc, &buf)) return rc;
    uint8_t* splat = static_cast<uint8_t*>(buf);
    uint8_t* tmp = splat + nc;
    uint8_t* res = on_device(out) ? out : splat + 2 * nc;
    CU(cudaMemsetAsync(splat, 0, nc, 0));
    CU(launch_register_splat((const uint8_t*)dm, (const uint16_t*)dd, dw, dh, 1, to_dev(*rig), cw,
                             ch, splat, 0));
    CU(launch_dilate(splat, tmp, res, cw, ch, 1, radius, 0));
    if (res != out) CU(cudaMemcpyAsync(out, res, nc, cudaMemcpyDefault, 0));
    CU(cudaStreamSynchronize(0));
    return RGBDSEG_OK;
}

// ------------------------------------------------------------ processor
void rgbdseg_processor_defaults(rgbdseg_processor_cfg* c, int width, int height) {
    std::memset(c, 0, sizeof *c);
    c->width = width;
    c->height = height;
    c->streams = 1;
    rgbdseg_mixture_defaults(&c->color);
    rgbdseg_mixture_defaults(&c->depth);
    c->depth.learning_rate = 0.01f;  // RunConfig::defaults, processor.cpp:40-41
    c->depth.initial_sigma = 100.0f;
    c->fusion_counter_limit = 3;
    c->fusion_initial_label = 0;
    c->device = 0;
    c->host_chunks = 0;
    c->registered = 1;
    rgbdseg_camera_rig_identity(&c->rig, 525.0, 525.0, 319.5, 239.5);
    c->dilation_radius = 1;
}

void rgbdseg_processor_destroy(rgbdseg_processor* p) {
    if (!p) return;
    DeviceGuard g(p->cfg.device);
    flush_emit(p);
    for (cudaStream_t st : p->cs)
        if (st) cudaStreamSynchronize(st);
    for (auto& sl : p->slot) {
        dfree(sl.r);  // g, b, d live in the same allocation
        dfree(sl.rgbm);
        dfree(sl.depm);
        dfree(sl.fused);
        dfree(sl.gt);
    }
    for (cudaEvent_t e : p->ev)
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : p->ev_k)
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : p->ev_done)
        if (e) cudaEventDestroy(e);
    if (p->ev_user) cudaEventDestroy(p->ev_user);
    for (cudaStream_t st : p->cs)
        if (st) cudaStreamDestroy(st);
    rgbdseg_bank_destroy(p->color);
    rgbdseg_bank_destroy(p->depth);
    rgbdseg_fusion_destroy(p->fusion);
    delete p;
}

int rgbdseg_processor_create(const rgbdseg_processor_cfg* cfg, rgbdseg_processor** out) {
    *out = nullptr;
    if (int rc = check_dims(cfg->width, cfg->height, cfg->streams)) return rc;
    // RunConfig::validate, processor.cpp:45-58 (the parts on this path)
    if (int rc = validate_cfg(&cfg->color)) return rc;
    if (int rc = validate_cfg(&cfg->depth)) return rc;
    if (cfg->fusion_counter_limit < 1)
        return fail(RGBDSEG_EINVAL, "config: fusion counter_limit must be >= 1");
    if (cfg->fusion_initial_label < 0 || cfg->fusion_initial_label > 1)
        return fail(RGBDSEG_EINVAL, "config: fusion initial_label must be 0 or 1");
    if (cfg->dilation_radius < 0)
        return fail(RGBDSEG_EINVAL, "config: dilation_radius must be >= 0");
    if (!cfg->registered) {  // processor.cpp:131-132, registration.cpp:57
        if (int rc = rgbdseg_camera_rig_validate(&cfg->rig)) return rc;
    }
    GUARD(cfg->device);
    auto* p = new rgbdseg_processor();
    p->cfg = *cfg;
    p->npx = (size_t)cfg->width * cfg->height * cfg->streams;
    int rc = rgbdseg_bank_create(cfg->width, cfg->height, cfg->streams, RGBDSEG_COLOR3,
                                 &cfg->color, cfg->device, &p->color);
    if (!rc)
        rc = rgbdseg_bank_create(cfg->width, cfg->height, cfg->streams, RGBDSEG_DEPTH1,
                                 &cfg->depth, cfg->device, &p->depth);
    if (!rc)
        rc = rgbdseg_fusion_create(cfg->width, cfg->height, cfg->streams,
                                   cfg->fusion_initial_label, cfg->fusion_counter_limit,
                                   cfg->device, &p->fusion);
    if (!rc) {
        p->color->owner = p->depth->owner = p;
        p->fusion->owner = p;
        // Large frames: up to 8 chunks of >= 2 Mpx, chunk c on stream c % 2.
        // Smaller frames stay one chunk (per-call CPU cost dominates) and
        // alternate streams frame by frame.  Chunk boundaries fall on
        // 64-pixel (two tiled-block) multiples.
        int chunks = cfg->host_chunks;
        if (chunks <= 0) chunks = (int)std::min<size_t>(8, std::max<size_t>(1, p->npx >> 21));
        p->nchunks = chunks;
        p->chunk = pitch_for((p->npx + chunks - 1) / chunks);
        cudaError_t e = cudaSuccess;
        for (cudaStream_t& st : p->cs)
            if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
        for (cudaEvent_t& ev : p->ev)
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        for (cudaEvent_t& ev : p->ev_k)
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        for (cudaEvent_t& ev : p->ev_done)
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->ev_user, cudaEventDisableTiming);
        if (e != cudaSuccess) rc = cuda_fail(e, "processor_create");
    }
    if (rc) {
        rgbdseg_processor_destroy(p);
        return rc;
    }
    *out = p;
    return RGBDSEG_OK;
}

static int ensure_slots(rgbdseg_processor* p) {
    for (auto& sl : p->slot) {
        if (sl.r) continue;
        int rc = dalloc(&sl.r, 5 * p->chunk);
        if (rc) return rc;
        sl.g = sl.r + p->chunk;
        sl.b = sl.g + p->chunk;
        sl.d = reinterpret_cast<uint16_t*>(sl.b + p->chunk);
        if (!rc) rc = dalloc(&sl.rgbm, p->chunk);
        if (!rc) rc = dalloc(&sl.depm, p->chunk);
        if (!rc) rc = dalloc(&sl.fused, p->chunk);
        if (!rc) rc = dalloc(&sl.gt, p->chunk);
        if (rc) return rc;
    }
    return RGBDSEG_OK;
}

// Order work about to be queued in `mode` after everything queued before
// in the other mode (host chunks use both streams; the device path and the
// unregistered path use cs[0]).
static int switch_mode(rgbdseg_processor* p, int mode) {
    if (p->last_mode == 1 && mode == 2) {  // join cs[1] into cs[0]
        CU(cudaEventRecord(p->ev[1], p->cs[1]));
        CU(cudaStreamWaitEvent(p->cs[0], p->ev[1], 0));
    } else if (p->last_mode == 2 && mode == 1) {  // fork cs[0] into cs[1]
        CU(cudaEventRecord(p->ev[0], p->cs[0]));
        CU(cudaStreamWaitEvent(p->cs[1], p->ev[0], 0));
    }
    p->last_mode = mode;
    return RGBDSEG_OK;
}

// The near-threshold pass ahead of K1 (same stream, same pixels).
static int near_pass(rgbdseg_processor* p, const FusedArgs& a, cudaStream_t st) {
    if (!(p->near_rel > 0.0f)) return RGBDSEG_OK;
    CU(launch_near(a, p->near_rel, static_cast<unsigned long long*>(p->near_counts.p), st));
    p->near_pixel_frames += a.n;
    return RGBDSEG_OK;
}

static FusedArgs base_args(const rgbdseg_processor* p) {
    FusedArgs a{};
    a.color = p->color->view(p->cfg.color);
    a.depth = p->depth->view(p->cfg.depth);
    a.ck = to_k(p->cfg.color, p->color->vvar);
    a.dk = to_k(p->cfg.depth, p->depth->vvar);
    a.limit = p->fusion->limit;
    a.fuse = 1;
    return a;
}

// Unregistered sequence (processor.cpp:175-179): both banks step and write
// their masks, the depth mask is registered into the colour grid and
// dilated, then List 1 fuses -- whole frames, in stream order.
static int submit_unregistered(rgbdseg_processor* p, const uint8_t* r, const uint8_t* g,
                               const uint8_t* b, const uint16_t* depth, uint8_t* fused_out,
                               uint8_t* rgb_out, uint8_t* depth_out, const uint8_t* gt,
                               unsigned long long* dcounts, int pack) {
    const size_t n = p->npx;
    const int w = p->cfg.width, h = p->cfg.height, S = p->cfg.streams;
    cudaStream_t st = p->cs[0];
    if (int rc = switch_mode(p, 2)) return rc;
    // Every staged plane starts on a 256-byte boundary (pitch P), so the
    // uint16 depth plane is aligned for any pixel count and the byte masks
    // keep the 16-byte vector kernels.
    const size_t P = pitch_for(n);
    void* ibuf;
    if (int rc = p->u_in.get(5 * P, &ibuf)) return rc;
    void* mbuf;
    if (int rc = p->u_masks.get(5 * P, &mbuf)) return rc;
    uint8_t* in = static_cast<uint8_t*>(ibuf);
    uint8_t *rgbm = static_cast<uint8_t*>(mbuf), *depm = rgbm + P, *splat = depm + P,
            *tmp = splat + P, *reg = tmp + P;
    const uint8_t* src[4] = {r, g, b, reinterpret_cast<const uint8_t*>(depth)};
    const uint8_t* dev[4] = {nullptr, nullptr, nullptr, nullptr};
    for (int k = 0; k < 4; ++k) {
        if (pack && (k == 1 || k == 2)) continue;  // one interleaved plane at k = 0
        const size_t bytes = k == 3 ? 2 * n : (pack ? 3 * n : n);
        if (on_device(src[k])) {
            dev[k] = src[k];
        } else {
            CU(cudaMemcpyAsync(in + k * P, src[k], bytes, cudaMemcpyDefault, st));
            dev[k] = in + k * P;
        }
    }
    FusedArgs a = base_args(p);
    a.fuse = 0;
    a.r = dev[0];
    a.g = pack ? dev[0] : dev[1];
    a.b = pack ? dev[0] : dev[2];
    a.packed = pack != 0;
    a.bgr = pack == 2;
    a.d = reinterpret_cast<const uint16_t*>(dev[3]);
    a.rgb_mask = rgbm;
    a.depth_mask = depm;
    a.out = p->fusion->out;
    a.cpt = p->fusion->cpt;
    a.base = 0;
    a.n = n;
    if (int rc = near_pass(p, a, st)) return rc;
    CU(launch_fused(a, p->variant, st));
    CU(cudaMemsetAsync(splat, 0, n, st));
    CU(launch_register_splat(depm, a.d, w, h, S, to_dev(p->cfg.rig), w, h, splat, st));
    CU(launch_dilate(splat, tmp, reg, w, h, S, p->cfg.dilation_radius, st));
    uint8_t* fcopy = (fused_out && on_device(fused_out)) ? fused_out : nullptr;
    CU(launch_fuse(p->fusion->out, p->fusion->cpt, rgbm, reg, fcopy, p->fusion->limit,
                   n, st));
    if (gt) {  // evaluation: the three masks against the ground truth
        const void* dgt;
        if (int rc = stage_in(gt, n, p->u_gt, &dgt, st)) return rc;
        const uint8_t* preds[3] = {rgbm, depm, p->fusion->out};
        CU(launch_confusion(preds, 3, (const uint8_t*)dgt, n, (size_t)w * h, dcounts, st));
        CU(launch_counts_tn(dcounts, S, 3, (size_t)w * h, st));
    }
    if (fused_out && !fcopy) CU(cudaMemcpyAsync(fused_out, p->fusion->out, n, cudaMemcpyDefault, st));
    if (rgb_out) CU(cudaMemcpyAsync(rgb_out, rgbm, n, cudaMemcpyDefault, st));
    if (depth_out) CU(cudaMemcpyAsync(depth_out, depm, n, cudaMemcpyDefault, st));
    ++p->frames;
    return RGBDSEG_OK;
}

// pack: 0 = planar r, g, b; 1 / 2 = ONE interleaved colour plane `r` of 3
// bytes per pixel in R,G,B / B,G,R order (g, b ignored), deinterleaved by K1.
static int submit_impl(rgbdseg_processor* p, const uint8_t* r, const uint8_t* g, const uint8_t* b,
                       const uint16_t* depth, uint8_t* fused_out, uint8_t* rgb_out,
                       uint8_t* depth_out, const uint8_t* gt, int64_t* counts_out,
                       int pack = 0) {
    if (pack) g = b = r;
    if (!r || !g || !b || !depth) return fail(RGBDSEG_EINVAL, "process: null input plane");
    if (gt && !counts_out) return fail(RGBDSEG_EINVAL, "process: ground truth without counts");
    if (gt && pack)
        return fail(RGBDSEG_EINVAL, "process: evaluation takes planar colour input");
    const bool dr = on_device(r), dg = on_device(g), db = on_device(b), dd = on_device(depth);
    const bool dfo = on_device(fused_out), dro = on_device(rgb_out), ddo = on_device(depth_out);
    const bool dgt = gt && on_device(gt);
    const bool all_device = dr && dg && db && dd && (!fused_out || dfo) && (!rgb_out || dro) &&
                            (!depth_out || ddo) && (!gt || dgt);
    const bool single = !p->cfg.registered || all_device;
    // only a single-chunk host frame without ground truth keeps a read-back pending
    if (single || p->nchunks != 1 || gt)
        if (int rc = flush_emit(p)) return rc;
    if (int rc = switch_mode(p, single ? 2 : 1)) return rc;
    unsigned long long* dcounts = nullptr;
    const size_t ncnt = (size_t)p->cfg.streams * 12;
    if (gt) {
        void* c;
        if (int rc = p->counts.get(ncnt * sizeof(unsigned long long), &c)) return rc;
        dcounts = static_cast<unsigned long long*>(c);
        CU(cudaMemsetAsync(dcounts, 0, ncnt * sizeof(unsigned long long), p->cs[0]));
        if (!single) {  // both chunk streams accumulate into the zeroed counters
            CU(cudaEventRecord(p->ev[0], p->cs[0]));
            CU(cudaStreamWaitEvent(p->cs[1], p->ev[0], 0));
        }
    }
    if (!p->cfg.registered) {
        int rc = submit_unregistered(p, r, g, b, depth, fused_out, rgb_out, depth_out, gt, dcounts,
                                     pack);
        if (!rc && gt)
            CU(cudaMemcpyAsync(counts_out, dcounts, ncnt * 8, cudaMemcpyDefault, p->cs[0]));
        return rc;
    }
    FusedArgs a = base_args(p);
    a.counts = dcounts;
    a.stream_px = (size_t)p->cfg.width * p->cfg.height;
    a.packed = pack != 0;
    a.bgr = pack == 2;
    if (all_device) {  // device-resident frames: one launch over every pixel
        a.r = r;
        a.g = g;
        a.b = b;
        a.d = depth;
        a.rgb_mask = rgb_out;
        a.depth_mask = depth_out;
        a.fused_copy = fused_out;
        a.out = p->fusion->out;
        a.cpt = p->fusion->cpt;
        a.base = 0;
        a.n = p->npx;
        a.gt = gt;
        if (int rc = near_pass(p, a, p->cs[0])) return rc;
        CU(launch_fused(a, p->variant, p->cs[0]));
        if (gt) {
            CU(launch_counts_tn(dcounts, p->cfg.streams, 3, a.stream_px, p->cs[0]));
            CU(cudaMemcpyAsync(counts_out, dcounts, ncnt * 8, cudaMemcpyDefault, p->cs[0]));
        }
        ++p->frames;
        return RGBDSEG_OK;
    }
    if (int rc = ensure_slots(p)) return rc;
    // planar host frame: the four planes back to back in one host buffer
    // (interleaved: the 3-byte plane then depth)
    const bool planar = !dr && !dg && !db && !dd &&
                        (pack ? reinterpret_cast<const uint8_t*>(depth) == r + 3 * p->npx
                              : (g == r + p->npx && b == g + p->npx &&
                                 reinterpret_cast<const uint8_t*>(depth) == b + p->npx));
    const bool alternate = p->nchunks == 1;
    const cudaMemcpyKind h2d = cudaMemcpyHostToDevice, d2h = cudaMemcpyDeviceToHost;
    for (int c = 0; c < p->nchunks; ++c) {
        const size_t lo = (size_t)c * p->chunk;
        if (lo >= p->npx) break;
        const size_t n = std::min(p->chunk, p->npx - lo);
        const int lane = alternate ? (int)(p->frames & 1) : (c & 1);
        Slot& sl = p->slot[lane];
        cudaStream_t st = p->cs[lane];
        // ingest
        if (pack) {  // the chunk's 3n interleaved bytes into the slot's r|g|b span
            if (planar && n == p->chunk && n == p->npx) {
                CU(cudaMemcpyAsync(sl.r, r, 5 * n, h2d, st));
            } else {
                if (!dr) CU(cudaMemcpyAsync(sl.r, r + 3 * lo, 3 * n, h2d, st));
                if (!dd) CU(cudaMemcpyAsync(sl.d, depth + lo, n * 2, h2d, st));
            }
        } else if (planar) {  // r, g, b rows of this chunk in one 2-D copy, depth in one
            if (n == p->chunk && n == p->npx) {
                CU(cudaMemcpyAsync(sl.r, r, 5 * n, h2d, st));
            } else {
                CU(cudaMemcpy2DAsync(sl.r, p->chunk, r + lo, p->npx, n, 3, h2d, st));
                CU(cudaMemcpyAsync(sl.d, depth + lo, 2 * n, h2d, st));
            }
        } else {
            if (!dr) CU(cudaMemcpyAsync(sl.r, r + lo, n, h2d, st));
            if (!dg) CU(cudaMemcpyAsync(sl.g, g + lo, n, h2d, st));
            if (!db) CU(cudaMemcpyAsync(sl.b, b + lo, n, h2d, st));
            if (!dd) CU(cudaMemcpyAsync(sl.d, depth + lo, n * 2, h2d, st));
        }
        if (gt && !dgt) CU(cudaMemcpyAsync(sl.gt, gt + lo, n, h2d, st));
        if (alternate)  // the previous frame's read-back, now behind this upload
            if (int rc = flush_emit(p)) return rc;
        // process (a single-chunk frame waits for the previous frame's K1,
        // queued on the other stream)
        a.r = dr ? r + (pack ? 3 * lo : lo) : sl.r;
        a.g = pack ? a.r : (dg ? g + lo : sl.g);
        a.b = pack ? a.r : (db ? b + lo : sl.b);
        a.d = dd ? depth + lo : sl.d;
        a.gt = gt ? (dgt ? gt + lo : sl.gt) : nullptr;
        a.rgb_mask = rgb_out ? (dro ? rgb_out + lo : sl.rgbm) : nullptr;
        a.depth_mask = depth_out ? (ddo ? depth_out + lo : sl.depm) : nullptr;
        a.fused_copy = fused_out ? (dfo ? fused_out + lo : sl.fused) : nullptr;
        a.base = lo;
        a.n = n;
        a.out = p->fusion->out + lo;
        a.cpt = p->fusion->cpt + lo;
        if (alternate) CU(cudaStreamWaitEvent(st, p->ev_k[lane ^ 1], 0));
        if (int rc = near_pass(p, a, st)) return rc;
        CU(launch_fused(a, p->variant, st));
        if (alternate) CU(cudaEventRecord(p->ev_k[lane], st));
        // emit
        uint8_t* fo = fused_out && !dfo ? fused_out + lo : nullptr;
        uint8_t* ro = rgb_out && !dro ? rgb_out + lo : nullptr;
        uint8_t* dpo = depth_out && !ddo ? depth_out + lo : nullptr;
        if (alternate && !gt) {  // deferred: issued after the next frame's upload or at sync
            p->pend.on = fo || ro || dpo;
            p->pend.lane = lane;
            p->pend.n = n;
            p->pend.fused = fo;
            p->pend.rgb = ro;
            p->pend.depth = dpo;
        } else {
            if (fo) CU(cudaMemcpyAsync(fo, sl.fused, n, d2h, st));
            if (ro) CU(cudaMemcpyAsync(ro, sl.rgbm, n, d2h, st));
            if (dpo) CU(cudaMemcpyAsync(dpo, sl.depm, n, d2h, st));
        }
    }
    if (gt) {  // join both streams' counters, then copy them out
        CU(cudaEventRecord(p->ev[1], p->cs[1]));
        CU(cudaStreamWaitEvent(p->cs[0], p->ev[1], 0));
        CU(launch_counts_tn(dcounts, p->cfg.streams, 3,
                            (size_t)p->cfg.width * p->cfg.height, p->cs[0]));
        CU(cudaMemcpyAsync(counts_out, dcounts, ncnt * 8, cudaMemcpyDefault, p->cs[0]));
    }
    ++p->frames;
    return RGBDSEG_OK;
}

int rgbdseg_processor_submit(rgbdseg_processor* p, const uint8_t* r, const uint8_t* g,
                             const uint8_t* b, const uint16_t* depth, uint8_t* fused_out,
                             uint8_t* rgb_out, uint8_t* depth_out) {
    if (!p) return fail(RGBDSEG_EINVAL, "processor_submit: null handle");
    GUARD(p->cfg.device);
    return submit_impl(p, r, g, b, depth, fused_out, rgb_out, depth_out, nullptr, nullptr);
}

int rgbdseg_processor_submit_interleaved(rgbdseg_processor* p, const uint8_t* rgb, int order,
                                         const uint16_t* depth, uint8_t* fused_out,
                                         uint8_t* rgb_out, uint8_t* depth_out) {
    if (!p) return fail(RGBDSEG_EINVAL, "processor_submit_interleaved: null handle");
    GUARD(p->cfg.device);
    if (order != RGBDSEG_ORDER_RGB && order != RGBDSEG_ORDER_BGR)
        return fail(RGBDSEG_EINVAL, "process: unknown channel order");
    return submit_impl(p, rgb, nullptr, nullptr, depth, fused_out, rgb_out, depth_out, nullptr,
                       nullptr, order == RGBDSEG_ORDER_BGR ? 2 : 1);
}

int rgbdseg_processor_process_interleaved(rgbdseg_processor* p, const uint8_t* rgb, int order,
                                          const uint16_t* depth, uint8_t* fused_out,
                                          uint8_t* rgb_out, uint8_t* depth_out) {
    if (!p) return fail(RGBDSEG_EINVAL, "processor_process_interleaved: null handle");
    if (int rc = rgbdseg_processor_submit_interleaved(p, rgb, order, depth, fused_out, rgb_out,
                                                      depth_out))
        return rc;
    return rgbdseg_processor_sync(p);
}

int rgbdseg_processor_submit_eval(rgbdseg_processor* p, const uint8_t* r, const uint8_t* g,
                                  const uint8_t* b, const uint16_t* depth, const uint8_t* gt,
                                  int64_t* counts, uint8_t* fused_out, uint8_t* rgb_out,
                                  uint8_t* depth_out) {
    if (!p) return fail(RGBDSEG_EINVAL, "processor_submit_eval: null handle");
    GUARD(p->cfg.device);
    return submit_impl(p, r, g, b, depth, fused_out, rgb_out, depth_out, gt, counts);
}

int rgbdseg_processor_process_eval(rgbdseg_processor* p, const uint8_t* r, const uint8_t* g,
                                   const uint8_t* b, const uint16_t* depth, const uint8_t* gt,
                                   int64_t* counts, uint8_t* fused_out, uint8_t* rgb_out,
                                   uint8_t* depth_out) {
    if (!p) return fail(RGBDSEG_EINVAL, "processor_process_eval: null handle");
    if (int rc = rgbdseg_processor_submit_eval(p, r, g, b, depth, gt, counts, fused_out, rgb_out,
                                               depth_out))
        return rc;
    return rgbdseg_processor_sync(p);
}

int rgbdseg_confusion_counts(const uint8_t* pred, const uint8_t* gt, size_t npx, int streams,
                             int64_t* counts, int device) {
    if (streams <= 0 || npx % (size_t)streams != 0)
        return fail(RGBDSEG_EINVAL, "confusion_counts: pixels do not split into streams");
    GUARD(device);
    Scratch sp, sg, sc;
    const void *dp, *dg;
    if (int rc = stage_in(pred, npx, sp, &dp, 0)) return rc;
    if (int rc = stage_in(gt, npx, sg, &dg, 0)) return rc;
    void* c;
    if (int rc = sc.get((size_t)streams * 4 * 8, &c)) return rc;
    CU(cudaMemsetAsync(c, 0, (size_t)streams * 4 * 8, 0));
    const uint8_t* preds[1] = {(const uint8_t*)dp};
    CU(launch_confusion(preds, 1, (const uint8_t*)dg, npx, npx / streams,
                        static_cast<unsigned long long*>(c), 0));
    CU(launch_counts_tn(static_cast<unsigned long long*>(c), streams, 1, npx / streams, 0));
    CU(cudaMemcpyAsync(counts, c, (size_t)streams * 4 * 8, cudaMemcpyDefault, 0));
    CU(cudaStreamSynchronize(0));
    return RGBDSEG_OK;
}

int rgbdseg_processor_sync(rgbdseg_processor* p) {
    if (!p) return fail(RGBDSEG_EINVAL, "processor_sync: null handle");
    GUARD(p->cfg.device);
    if (int rc = flush_emit(p)) return rc;
    CU(cudaStreamSynchronize(p->cs[0]));
    CU(cudaStreamSynchronize(p->cs[1]));
    return RGBDSEG_OK;
}

int rgbdseg_processor_process(rgbdseg_processor* p, const uint8_t* r, const uint8_t* g,
                              const uint8_t* b, const uint16_t* depth, uint8_t* fused_out,
                              uint8_t* rgb_out, uint8_t* depth_out) {
    if (!p) return fail(RGBDSEG_EINVAL, "processor_process: null handle");
    if (int rc = rgbdseg_processor_submit(p, r, g, b, depth, fused_out, rgb_out, depth_out))
        return rc;
    return rgbdseg_processor_sync(p);
}

int64_t rgbdseg_processor_frames(const rgbdseg_processor* p) { return p->frames; }

// Stream ordering with a caller's CUDA stream (the library's streams are
// non-blocking, so they are not ordered with the legacy default stream).
int rgbdseg_processor_wait_stream(rgbdseg_processor* p, void* stream) {
    if (!p) return fail(RGBDSEG_EINVAL, "processor_wait_stream: null handle");
    GUARD(p->cfg.device);
    CU(cudaEventRecord(p->ev_user, (cudaStream_t)stream));
    CU(cudaStreamWaitEvent(p->cs[0], p->ev_user, 0));
    CU(cudaStreamWaitEvent(p->cs[1], p->ev_user, 0));
    return RGBDSEG_OK;
}

int rgbdseg_processor_signal_stream(rgbdseg_processor* p, void* stream) {
    if (!p) return fail(RGBDSEG_EINVAL, "processor_signal_stream: null handle");
    GUARD(p->cfg.device);
    for (int i = 0; i < 2; ++i) {
        CU(cudaEventRecord(p->ev_done[i], p->cs[i]));
        CU(cudaStreamWaitEvent((cudaStream_t)stream, p->ev_done[i], 0));
    }
    return RGBDSEG_OK;
}
rgbdseg_bank* rgbdseg_processor_color_bank(rgbdseg_processor* p) { return p ? p->color : nullptr; }
rgbdseg_bank* rgbdseg_processor_depth_bank(rgbdseg_processor* p) { return p ? p->depth : nullptr; }
rgbdseg_fusion* rgbdseg_processor_fusion(rgbdseg_processor* p) { return p ? p->fusion : nullptr; }
void* rgbdseg_processor_stream(rgbdseg_processor* p) { return p ? (void*)p->cs[0] : nullptr; }

int rgbdseg_processor_set_near_threshold(rgbdseg_processor* p, float rel) {
    if (!p) return fail(RGBDSEG_EINVAL, "processor_set_near_threshold: null handle");
    GUARD(p->cfg.device);
    if (int rc = rgbdseg_processor_sync(p)) return rc;
    if (!(rel >= 0.0f)) return fail(RGBDSEG_EINVAL, "near-threshold: rel must be >= 0");
    p->near_rel = rel;
    if (rel > 0.0f) {
        void* c;
        if (int rc = p->near_counts.get(2 * sizeof(unsigned long long), &c)) return rc;
        CU(cudaMemset(c, 0, 2 * sizeof(unsigned long long)));
        p->near_pixel_frames = 0;
    }
    return RGBDSEG_OK;
}

int rgbdseg_processor_near_threshold_counts(rgbdseg_processor* p, uint64_t* color,
                                            uint64_t* depth, uint64_t* pixel_frames) {
    if (!p) return fail(RGBDSEG_EINVAL, "processor_near_threshold_counts: null handle");
    GUARD(p->cfg.device);
    if (int rc = rgbdseg_processor_sync(p)) return rc;
    unsigned long long h[2] = {0, 0};
    if (p->near_counts.p) CU(cudaMemcpy(h, p->near_counts.p, sizeof h, cudaMemcpyDeviceToHost));
    if (color) *color = h[0];
    if (depth) *depth = h[1];
    if (pixel_frames) *pixel_frames = p->near_pixel_frames;
    return RGBDSEG_OK;
}

int rgbdseg_processor_set_variant(rgbdseg_processor* p, int variant) {
    if (!p) return fail(RGBDSEG_EINVAL, "processor_set_variant: null handle");
    if (variant < kAuto || variant > kLdgElideL1) return fail(RGBDSEG_EINVAL, "unknown kernel variant");
    p->variant = variant;
    return RGBDSEG_OK;
}

// ------------------------------------------------------------ synthetic scenes
// builtin_scenario (synthetic.cpp:234-273) resolved for one frame: the
// illumination gain product, the object's lround'ed waypoint position and
// the active shadow / flicker events (render_frame, synthetic.cpp:124-134).
int rgbdseg_render_scenario(char name, int width, int height, int streams, uint64_t seed0,
                            int frame, uint8_t* r, uint8_t* g, uint8_t* b, uint16_t* depth,
                            uint8_t* gt, int device, void* stream) {
    if (name != 'A' && name != 'B')
        return fail(RGBDSEG_EINVAL, std::string("unknown scenario '") + name + "' (known: A, B)");
    if (int rc = check_dims(width, height, streams)) return rc;
    GUARD(device);
    SceneFrame sc{};
    sc.width = width;
    sc.height = height;
    sc.streams = streams;
    sc.seed0 = seed0;
    sc.frame = frame;
    sc.base_depth_mm = 2000;
    sc.depth_texture_mm = 30;
    sc.color_texture = 8;
    // the 24x24 box, (40,100) at frame 0 -> (600,320) at frame 299
    struct Wp {
        int f;
        double x, y;
    } wp[2] = {{0, 40, 100}, {299, 600, 320}};
    double x = wp[0].x, y = wp[0].y;
    if (frame >= wp[1].f) {
        x = wp[1].x;
        y = wp[1].y;
    } else if (frame > wp[0].f) {
        const double t = (double)(frame - wp[0].f) / (double)(wp[1].f - wp[0].f);
        x = wp[0].x + t * (wp[1].x - wp[0].x);
        y = wp[0].y + t * (wp[1].y - wp[0].y);
    }
    sc.n_obj = 1;
    sc.orect[0][0] = (int)std::lround(x);
    sc.orect[0][1] = (int)std::lround(y);
    sc.orect[0][2] = 24;
    sc.orect[0][3] = 24;
    sc.ocolor[0][0] = 230;
    sc.ocolor[0][1] = 40;
    sc.ocolor[0][2] = 220;
    sc.odepth[0] = 400;
    sc.gain = 1.0;
    if (name == 'A') {
        const struct {
            int s, e;
            double g;
        } il[2] = {{100, 112, 1.5}, {200, 212, 0.6}};
        for (auto& e : il)
            if (frame >= e.s && frame < e.e) sc.gain *= e.g;
        if (frame >= 150 && frame < 180) {
            sc.n_shadow = 1;
            const int rc[4] = {300, 300, 200, 120};
            std::memcpy(sc.srect[0], rc, sizeof rc);
            sc.sdarken[0] = 0.6;
        }
        if (frame >= 0 && frame < 300) {
            sc.n_flicker = 1;
            const int rc[4] = {40, 40, 80, 60};
            std::memcpy(sc.frect[0], rc, sizeof rc);
            sc.fcs[0] = 3.0;
            sc.fds[0] = 30.0;
        }
        sc.ncs = 1.0;
        sc.nds = 1.0;
    } else {
        const double gains[10] = {1.4, 0.7, 1.25, 0.8, 1.35, 0.75, 1.2, 0.85, 1.3, 0.9};
        for (int i = 0; i < 10; ++i)
            if (frame >= 30 + 25 * i && frame < 30 + 25 * (i + 1)) sc.gain *= gains[i];
        if (frame >= 0 && frame < 300) {
            sc.n_flicker = 1;
            const int rc[4] = {400, 60, 160, 120};
            std::memcpy(sc.frect[0], rc, sizeof rc);
            sc.fcs[0] = 12.0;
            sc.fds[0] = 40.0;
        }
        sc.ncs = 1.5;
        sc.nds = 2.0;
    }
    CU(launch_render(sc, r, g, b, depth, gt, (cudaStream_t)stream));
    if (!stream) CU(cudaStreamSynchronize(0));
    return RGBDSEG_OK;
}

int rgbdseg_render_frame(const rgbdseg_scene_frame* f, uint8_t* r, uint8_t* g, uint8_t* b,
                         uint16_t* depth, uint8_t* gt, int device, void* stream) {
    static_assert(sizeof(SceneFrame) == sizeof(rgbdseg_scene_frame), "scene frame layout");
    if (!f) return fail(RGBDSEG_EINVAL, "render_frame: null frame");
    if (int rc = check_dims(f->width, f->height, f->streams)) return rc;
    if (f->n_obj < 0 || f->n_obj > 4 || f->n_shadow < 0 || f->n_shadow > 16 || f->n_flicker < 0 ||
        f->n_flicker > 16)
        return fail(RGBDSEG_EINVAL, "render_frame: at most 4 objects and 16 events of each kind");
    GUARD(device);
    SceneFrame sc;
    std::memcpy(&sc, f, sizeof sc);
    CU(launch_render(sc, r, g, b, depth, gt, (cudaStream_t)stream));
    if (!stream) CU(cudaStreamSynchronize(0));
    return RGBDSEG_OK;
}

}  // extern "C"

static int drain_owner(rgbdseg_processor* owner) {
    return owner ? rgbdseg_processor_sync(owner) : RGBDSEG_OK;
}
