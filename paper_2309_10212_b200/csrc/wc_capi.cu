// wc_capi.cu -- extern "C" boundary of libwavecast_b200.so (include/wavecast_b200.h).
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cstring>
#include <string>
#include <vector>

#include "../../include/wavecast_b200.h"
#include "wc_engine.cuh"
#include "wc_stage.cuh"

struct wc_volume {
    wc::Volume v;
};
struct wc_session {
    wc::Session *s = nullptr;
    wc_volume *vol = nullptr;
};
struct wc_cache {
    wc::StageCache *c = nullptr;
};
struct wc_frame_target {
    wc::FrameTarget t;
};

static thread_local std::string g_err;

#define WC_API_BEGIN try {
#define WC_API_END                              \
    }                                           \
    catch (const wc::UsageError &e) {           \
        g_err = e.what();                       \
        return WC_E_USAGE;                      \
    }                                           \
    catch (const wc::DataError &e) {            \
        g_err = e.what();                       \
        return WC_E_DATA;                       \
    }                                           \
    catch (const wc::InvariantError &e) {       \
        g_err = e.what();                       \
        return WC_E_INVARIANT;                  \
    }                                           \
    catch (const std::exception &e) {           \
        g_err = e.what();                       \
        return WC_E_CUDA;                       \
    }                                           \
    return WC_OK;

#define WC_REQUIRE(cond, kind, msg) \
    do {                            \
        if (!(cond)) throw kind(msg); \
    } while (0)

static_assert(sizeof(wc_pass_stats) == sizeof(wc::PassStatsC), "stats layout");
static_assert(sizeof(wc_camera) == sizeof(wc::CameraParams), "camera layout");

namespace {

void check_qbits(int qbits) {
    if (qbits < 4 || qbits > 26)  // codec.py:26-27,76-78
        throw wc::UsageError("qbits must be in [4, 26], got " + std::to_string(qbits));
}
void check_dims(int nx, int ny, int nz) {
    if (nx < 1 || ny < 1 || nz < 1) throw wc::UsageError("dims must be positive");
}

template <typename T>
void upload(wc::DevBuf<T> &d, const T *h, int64_t n, cudaStream_t st) {
    d.alloc(n);
    WC_CUDA(cudaMemcpyAsync(d.p, h, sizeof(T) * (size_t)n, cudaMemcpyHostToDevice, st));
}

template <typename T>
void download(T *h, const T *d, int64_t n, cudaStream_t st) {
    if (!h || n <= 0) return;
    WC_CUDA(cudaMemcpyAsync(h, d, sizeof(T) * (size_t)n, cudaMemcpyDeviceToHost, st));
}

}  // namespace

extern "C" {

const char *wc_last_error(void) { return g_err.c_str(); }

const char *wc_build_info(void) {
    return "libwavecast_b200: sm_100a (compute_100a), -fmad=false -lineinfo -O3";
}

long long wc_launch_count(void) { return wc::g_launches.load(); }

int wc_host_alloc(uint64_t bytes, void **out) {
    WC_API_BEGIN
    WC_CUDA(cudaMallocHost(out, bytes ? bytes : 1));
    WC_API_END
}

int wc_host_free(void *p) {
    WC_API_BEGIN
    if (p) WC_CUDA(cudaFreeHost(p));
    WC_API_END
}

int wc_init(int device) {
    WC_API_BEGIN
    int n = 0;
    WC_CUDA(cudaGetDeviceCount(&n));
    WC_REQUIRE(device >= 0 && device < n, wc::UsageError, "no such CUDA device");
    WC_CUDA(cudaSetDevice(device));
    WC_CUDA(cudaFree(nullptr));
    WC_API_END
}

int wc_volume_create(const uint8_t *payload, uint64_t payload_bytes, const float *ranges, int nx, int ny, int nz,
                     int qbits, int stride, wc_volume **out) {
    WC_API_BEGIN
    check_qbits(qbits);
    check_dims(nx, ny, nz);
    WC_REQUIRE(stride == wc::stride_of(qbits), wc::DataError, "stride inconsistent with qbits");
    auto *h = new wc_volume();
    try {
        h->v.set_dims(nx, ny, nz, qbits);
        WC_REQUIRE((int64_t)payload_bytes == h->v.n_blocks * stride, wc::DataError, "payload size mismatch");
        upload(h->v.payload, payload, h->v.n_blocks * stride, h->v.st);
        upload(h->v.ranges, reinterpret_cast<const float2 *>(ranges), h->v.n_blocks, h->v.st);
        h->v.build_grids();
    } catch (...) {
        delete h;
        throw;
    }
    *out = h;
    WC_API_END
}

// ---- .wcz container straight to the device (codec.py:243-273) ----------

namespace {

struct WczHeader {
    int nx, ny, nz, qbits, stride;
    int64_t n_blocks, file_bytes;
};

// Same checks and messages as read_wcz (codec.py:246-262).
WczHeader wcz_header(const char *path, int fd) {
    const std::string p(path);
    struct stat sb;
    if (fstat(fd, &sb) != 0) throw wc::DataError(p + ": cannot stat");
    unsigned char h[28];
    const ssize_t got = sb.st_size >= 28 ? pread(fd, h, 28, 0) : 0;
    if (got != 28 || memcmp(h, "WCZ1", 4) != 0) throw wc::DataError(p + ": not a WCZ1 container");
    uint32_t f[6];
    memcpy(f, h + 4, 24);  // little-endian host (x86-64 / aarch64)
    if (f[0] != 1) throw wc::DataError(p + ": unsupported container version " + std::to_string(f[0]));
    check_qbits((int)f[4]);
    if ((int)f[5] != wc::stride_of((int)f[4]))
        throw wc::DataError(p + ": stride " + std::to_string(f[5]) + " inconsistent with qbits " +
                            std::to_string(f[4]));
    WczHeader w{(int)f[1], (int)f[2], (int)f[3], (int)f[4], (int)f[5], 0, (int64_t)sb.st_size};
    w.n_blocks = (int64_t)((w.nx + 3) / 4) * ((w.ny + 3) / 4) * ((w.nz + 3) / 4);
    const int64_t expected = 28 + 8 * w.n_blocks + w.n_blocks * (int64_t)w.stride;
    if (w.file_bytes != expected)
        throw wc::DataError(p + ": expected " + std::to_string(expected) + " bytes, found " +
                            std::to_string(w.file_bytes));
    return w;
}

struct Fd {
    int fd;
    explicit Fd(const char *path) : fd(open(path, O_RDONLY)) {
        if (fd < 0) throw wc::DataError(std::string(path) + ": cannot open");
    }
    ~Fd() { close(fd); }
};

// Stream [off, off+bytes) of the file into device memory: pread into two
// pinned chunks alternately while the other chunk's copy runs, so disk (or
// page cache) reads overlap the PCIe/C2C transfer.
void stream_to_device(int fd, const char *path, int64_t off, int64_t bytes, void *dst, int64_t chunk,
                      cudaStream_t st) {
    if (bytes <= 0) return;
    chunk = std::max<int64_t>(1 << 20, std::min<int64_t>(chunk, bytes));
    wc::PinnedBuf<uint8_t> buf[2];
    cudaEvent_t ev[2];
    for (int i = 0; i < 2; i++) {
        buf[i].alloc(chunk);
        WC_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
        WC_CUDA(cudaEventRecord(ev[i], st));
    }
    int64_t done = 0;
    int k = 0;
    try {
        while (done < bytes) {
            const int64_t n = std::min<int64_t>(chunk, bytes - done);
            WC_CUDA(cudaEventSynchronize(ev[k]));  // this chunk's previous copy has drained
            int64_t r = 0;
            while (r < n) {
                const ssize_t got = pread(fd, buf[k].p + r, (size_t)(n - r), (off_t)(off + done + r));
                if (got <= 0) throw wc::DataError(std::string(path) + ": short read");
                r += got;
            }
            WC_CUDA(cudaMemcpyAsync(static_cast<uint8_t *>(dst) + done, buf[k].p, (size_t)n, cudaMemcpyHostToDevice,
                                    st));
            WC_CUDA(cudaEventRecord(ev[k], st));
            done += n;
            k ^= 1;
        }
        WC_CUDA(cudaStreamSynchronize(st));
    } catch (...) {
        cudaStreamSynchronize(st);
        for (auto &e : ev) cudaEventDestroy(e);
        throw;
    }
    for (auto &e : ev) WC_CUDA(cudaEventDestroy(e));
}

}  // namespace

int wc_wcz_probe(const char *path, int *nx, int *ny, int *nz, int *qbits, int *stride, int64_t *n_blocks) {
    WC_API_BEGIN
    Fd f(path);
    const WczHeader h = wcz_header(path, f.fd);
    if (nx) *nx = h.nx;
    if (ny) *ny = h.ny;
    if (nz) *nz = h.nz;
    if (qbits) *qbits = h.qbits;
    if (stride) *stride = h.stride;
    if (n_blocks) *n_blocks = h.n_blocks;
    WC_API_END
}

int wc_volume_load_wcz(const char *path, int64_t chunk_bytes, wc_volume **out) {
    WC_API_BEGIN
    Fd f(path);
    const WczHeader h = wcz_header(path, f.fd);
    check_dims(h.nx, h.ny, h.nz);
    auto *v = new wc_volume();
    try {
        v->v.set_dims(h.nx, h.ny, h.nz, h.qbits);
        v->v.ranges.alloc(h.n_blocks);
        v->v.payload.alloc(h.n_blocks * h.stride + wc::kPayloadPad);
        const int64_t chunk = chunk_bytes > 0 ? chunk_bytes : (int64_t)64 << 20;
        stream_to_device(f.fd, path, 28, 8 * h.n_blocks, v->v.ranges.p, chunk, v->v.st);
        stream_to_device(f.fd, path, 28 + 8 * h.n_blocks, h.n_blocks * h.stride, v->v.payload.p, chunk, v->v.st);
        v->v.build_grids();
    } catch (...) {
        delete v;
        throw;
    }
    *out = v;
    WC_API_END
}

int wc_volume_alloc(int nx, int ny, int nz, int qbits, wc_volume **out) {
    WC_API_BEGIN
    check_qbits(qbits);
    check_dims(nx, ny, nz);
    auto *v = new wc_volume();
    try {
        v->v.set_dims(nx, ny, nz, qbits);
        v->v.ranges.alloc(v->v.n_blocks);
        v->v.payload.alloc(v->v.n_blocks * v->v.stride + wc::kPayloadPad);
    } catch (...) {
        delete v;
        throw;
    }
    *out = v;
    WC_API_END
}

int wc_volume_device_buffers(wc_volume *v, void **payload, uint64_t *payload_bytes, void **ranges,
                             uint64_t *ranges_bytes) {
    WC_API_BEGIN
    if (payload) *payload = v->v.payload.p;
    if (payload_bytes) *payload_bytes = (uint64_t)(v->v.n_blocks * v->v.stride);
    if (ranges) *ranges = v->v.ranges.p;
    if (ranges_bytes) *ranges_bytes = (uint64_t)(8 * v->v.n_blocks);
    WC_API_END
}

int wc_volume_finalize(wc_volume *v) {
    WC_API_BEGIN
    WC_CUDA(cudaDeviceSynchronize());  // payload/ranges were written by other streams (e.g. NCCL)
    v->v.build_grids();
    WC_API_END
}

int wc_volume_value_range(const wc_volume *v, double *lo, double *hi) {
    WC_API_BEGIN
    float l = 0.0f, h = 0.0f;
    wc::decoded_value_range(v->v, &l, &h);
    *lo = l;
    *hi = h;
    WC_API_END
}

int wc_volume_compress(const float *values, int nx, int ny, int nz, int qbits, wc_volume **out) {
    WC_API_BEGIN
    check_qbits(qbits);
    check_dims(nx, ny, nz);
    auto *h = new wc_volume();
    try {
        h->v.set_dims(nx, ny, nz, qbits);
        wc::DevBuf<float> dense;
        upload(dense, values, (int64_t)nx * ny * nz, h->v.st);
        wc::compress_dense_device(h->v, dense.p);
        h->v.build_grids();
    } catch (...) {
        delete h;
        throw;
    }
    *out = h;
    WC_API_END
}

int wc_volume_synthesize(int K, const float *amp, const float *fx, const float *fy, const float *fz, int nx, int ny,
                         int nz, int qbits, wc_volume **out) {
    WC_API_BEGIN
    check_qbits(qbits);
    check_dims(nx, ny, nz);
    WC_REQUIRE(K >= 1, wc::UsageError, "need at least one separable term");
    auto *h = new wc_volume();
    try {
        h->v.set_dims(nx, ny, nz, qbits);
        wc::synth_separable_compress(h->v, K, amp, fx, fy, fz);
        h->v.build_grids();
    } catch (...) {
        delete h;
        throw;
    }
    *out = h;
    WC_API_END
}

int wc_volume_destroy(wc_volume *v) {
    WC_API_BEGIN
    delete v;
    WC_API_END
}

int wc_volume_set_grids(wc_volume *v, const double *fine_min, const double *fine_max, const double *coarse_min,
                        const double *coarse_max) {
    WC_API_BEGIN
    wc::Volume &V = v->v;
    std::vector<double2> f(V.n_blocks), c(V.n_coarse);
    for (int64_t i = 0; i < V.n_blocks; i++) f[i] = make_double2(fine_min[i], fine_max[i]);
    for (int64_t i = 0; i < V.n_coarse; i++) c[i] = make_double2(coarse_min[i], coarse_max[i]);
    upload(V.fine_mm, f.data(), V.n_blocks, V.st);
    upload(V.coarse_mm, c.data(), V.n_coarse, V.st);
    WC_CUDA(cudaStreamSynchronize(V.st));
    V.build_range_index();
    WC_API_END
}

int wc_volume_info(const wc_volume *v, int64_t *n_blocks, int64_t *n_coarse, int64_t *payload_bytes) {
    WC_API_BEGIN
    if (n_blocks) *n_blocks = v->v.n_blocks;
    if (n_coarse) *n_coarse = v->v.n_coarse;
    if (payload_bytes) *payload_bytes = v->v.n_blocks * v->v.stride;
    WC_API_END
}

int wc_volume_download(const wc_volume *v, uint8_t *payload, float *ranges, double *fine_min, double *fine_max,
                       double *coarse_min, double *coarse_max) {
    WC_API_BEGIN
    const wc::Volume &V = v->v;
    download(payload, V.payload.p, V.n_blocks * V.stride, V.st);
    download(reinterpret_cast<float2 *>(ranges), V.ranges.p, V.n_blocks, V.st);
    std::vector<double2> f, c;
    if (fine_min || fine_max) {
        f.resize(V.n_blocks);
        download(f.data(), V.fine_mm.p, V.n_blocks, V.st);
    }
    if (coarse_min || coarse_max) {
        c.resize(V.n_coarse);
        download(c.data(), V.coarse_mm.p, V.n_coarse, V.st);
    }
    WC_CUDA(cudaStreamSynchronize(V.st));
    for (int64_t i = 0; i < (int64_t)f.size(); i++) {
        if (fine_min) fine_min[i] = f[i].x;
        if (fine_max) fine_max[i] = f[i].y;
    }
    for (int64_t i = 0; i < (int64_t)c.size(); i++) {
        if (coarse_min) coarse_min[i] = c[i].x;
        if (coarse_max) coarse_max[i] = c[i].y;
    }
    WC_API_END
}

int wc_decode_blocks(const wc_volume *v, const int64_t *ids, int64_t n, float *out) {
    WC_API_BEGIN
    if (n <= 0) return WC_OK;
    const wc::Volume &V = v->v;
    for (int64_t i = 0; i < n; i++)
        WC_REQUIRE(ids[i] >= 0 && ids[i] < V.n_blocks, wc::InvariantError, "block id out of range");
    wc::DevBuf<int64_t> d_ids;
    wc::DevBuf<float> d_out;
    upload(d_ids, ids, n, V.st);
    d_out.alloc(n * 64);
    wc::decode_blocks_device(V, d_ids.p, n, d_out.p, V.st);
    download(out, d_out.p, n * 64, V.st);
    WC_CUDA(cudaStreamSynchronize(V.st));
    WC_API_END
}

int wc_decode_bench(const wc_volume *v, const int64_t *ids, int64_t n, int reps, double *ms_per_launch) {
    WC_API_BEGIN
    const wc::Volume &V = v->v;
    wc::DevBuf<int64_t> d_ids;
    wc::DevBuf<float> d_out;
    upload(d_ids, ids, n, V.st);
    d_out.alloc(n * 64);
    wc::decode_blocks_device(V, d_ids.p, n, d_out.p, V.st);  // warm-up
    cudaEvent_t a, b;
    WC_CUDA(cudaEventCreate(&a));
    WC_CUDA(cudaEventCreate(&b));
    WC_CUDA(cudaEventRecord(a, V.st));
    for (int r = 0; r < reps; r++) wc::decode_blocks_device(V, d_ids.p, n, d_out.p, V.st);
    WC_CUDA(cudaEventRecord(b, V.st));
    WC_CUDA(cudaEventSynchronize(b));
    float ms = 0;
    WC_CUDA(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    *ms_per_launch = (double)ms / (reps > 0 ? reps : 1);
    WC_API_END
}

int wc_session_create(wc_volume *v, const wc_camera *cam, const uint32_t *pixel_ids, int64_t n, const double *origins,
                      const double *dirs, double iso, int speculation, int max_spec, int64_t cache_capacity,
                      int corrupt_cache, wc_session **out) {
    WC_API_BEGIN
    WC_REQUIRE(v != nullptr, wc::UsageError, "null volume");
    WC_REQUIRE(max_spec >= 1, wc::UsageError, "max_spec must be >= 1");
    const bool camera_mode = dirs == nullptr;
    if (camera_mode) {
        WC_REQUIRE(cam != nullptr, wc::UsageError, "camera rays need a camera");
        WC_REQUIRE(cam->img_w >= 1 && cam->img_h >= 1, wc::UsageError, "image size must be at least 1x1");
        if (!pixel_ids) n = (int64_t)cam->img_w * cam->img_h;
    } else {
        WC_REQUIRE(origins != nullptr, wc::UsageError, "arbitrary rays need origins");
    }
    WC_REQUIRE(n >= 1, wc::UsageError, "a session needs at least one ray");
    auto *h = new wc_session();
    try {
        h->s = new wc::Session(&v->v, reinterpret_cast<const wc::CameraParams *>(cam), pixel_ids, n, origins, dirs, iso, speculation, max_spec, cache_capacity,
                               corrupt_cache);
        h->vol = v;
    } catch (...) {
        delete h;
        throw;
    }
    *out = h;
    WC_API_END
}

int wc_session_set_base_color(wc_session *s, double r, double g, double b) {
    WC_API_BEGIN
    s->s->base[0] = r;
    s->s->base[1] = g;
    s->s->base[2] = b;
    WC_API_END
}

int wc_session_set_graphs(wc_session *s, int on) {
    WC_API_BEGIN
    s->s->use_graphs = on != 0;
    WC_API_END
}

int wc_session_set_grouping(wc_session *s, int group_entries) {
    WC_API_BEGIN
    s->s->group_entries = group_entries != 0;
    WC_API_END
}

int wc_session_pass(wc_session *s, wc_pass_stats *stats, int *ran) {
    WC_API_BEGIN
    wc::PassStatsC st{};
    const bool r = s->s->pass(st);
    if (ran) *ran = r ? 1 : 0;
    if (r && stats) std::memcpy(stats, &st, sizeof(st));
    WC_API_END
}

int wc_session_run(wc_session *s, wc_pass_stats *stats_out, int64_t max_stats, int64_t *n_passes) {
    WC_API_BEGIN
    const int64_t k = s->s->run_frame(reinterpret_cast<wc::PassStatsC *>(stats_out), stats_out ? max_stats : 0);
    if (n_passes) *n_passes = k;
    WC_API_END
}

int wc_session_render(wc_session *s, const wc_camera *cam, double iso, wc_pass_stats *stats_out, int64_t max_stats,
                      int64_t *n_passes) {
    WC_API_BEGIN
    s->s->reset(reinterpret_cast<const wc::CameraParams *>(cam), iso);
    const int64_t k = s->s->run_frame(reinterpret_cast<wc::PassStatsC *>(stats_out), stats_out ? max_stats : 0);
    if (n_passes) *n_passes = k;
    WC_API_END
}

int wc_session_render_host(wc_session *s, const wc_camera *cam, double iso, wc_pass_stats *stats_out,
                           int64_t max_stats, int64_t *n_passes, uint32_t *rgba, float *depth) {
    WC_API_BEGIN
    const int64_t k = s->s->render_to_host(reinterpret_cast<const wc::CameraParams *>(cam), iso,
                                           reinterpret_cast<wc::PassStatsC *>(stats_out), stats_out ? max_stats : 0,
                                           rgba, depth);
    if (n_passes) *n_passes = k;
    WC_API_END
}

int wc_session_n_active(const wc_session *s, int64_t *n_active) {
    WC_API_BEGIN
    *n_active = s->s->active_count();
    WC_API_END
}

int wc_session_framebuffer(wc_session *s, uint8_t *rgba, float *depth) {
    WC_API_BEGIN
    s->s->download_framebuffer(rgba, depth);
    WC_API_END
}

int wc_session_framebuffer_device(wc_session *s, void *rgba_dev, void *depth_dev) {
    WC_API_BEGIN
    s->s->copy_framebuffer_device(rgba_dev, depth_dev);
    WC_API_END
}

int wc_session_last_pass_ms(const wc_session *s, double *ms) {
    WC_API_BEGIN
    *ms = s->s->last_kernel_ms;
    WC_API_END
}

int wc_session_destroy(wc_session *s) {
    WC_API_BEGIN
    if (s) delete s->s;
    delete s;
    WC_API_END
}

int wc_session_reset(wc_session *s, const wc_camera *cam, double iso) {
    WC_API_BEGIN
    s->s->reset(reinterpret_cast<const wc::CameraParams *>(cam), iso);
    WC_API_END
}

int wc_session_reset_part(wc_session *s, const wc_camera *cam, double iso, int64_t part, int64_t parts) {
    WC_API_BEGIN
    WC_REQUIRE(parts >= 1 && part >= 0 && part < parts, wc::UsageError, "part out of range");
    s->s->reset_part(reinterpret_cast<const wc::CameraParams *>(cam), iso, part, parts);
    WC_API_END
}

int wc_session_mask_buffers(wc_session *s, int64_t parts, void **coarse_bm, void **cell_mask, int64_t *chunk_words) {
    WC_API_BEGIN
    WC_REQUIRE(parts >= 1, wc::UsageError, "parts must be positive");
    int64_t chunk = 0;
    s->s->mask_buffers(parts, chunk);
    if (coarse_bm) *coarse_bm = s->s->coarse_bm.p;
    if (cell_mask) *cell_mask = s->s->cell_mask.p;
    if (chunk_words) *chunk_words = chunk;
    WC_API_END
}

int wc_session_sync(wc_session *s) {
    WC_API_BEGIN
    s->s->sync_all();
    WC_API_END
}

int wc_frame_target_create(int64_t npix, wc_frame_target **out) {
    WC_API_BEGIN
    WC_REQUIRE(npix > 0, wc::UsageError, "frame target needs pixels");
    auto *t = new wc_frame_target();
    try {
        t->t.create(npix);
    } catch (...) {
        delete t;
        throw;
    }
    *out = t;
    WC_API_END
}

int wc_frame_target_ipc_handles(const wc_frame_target *t, void *handles) {
    WC_API_BEGIN
    WC_REQUIRE(!t->t.opened, wc::UsageError, "IPC handles come from the target's owner");
    t->t.ipc_handles(handles);
    WC_API_END
}

int wc_frame_target_open(const void *handles, int64_t npix, wc_frame_target **out) {
    WC_API_BEGIN
    auto *t = new wc_frame_target();
    try {
        t->t.open(handles, npix);
    } catch (...) {
        delete t;
        throw;
    }
    *out = t;
    WC_API_END
}

int wc_frame_target_download(const wc_frame_target *t, uint32_t *rgba_host, float *depth_host) {
    WC_API_BEGIN
    WC_CUDA(cudaMemcpy(rgba_host, t->t.p_rgba, 4 * t->t.npix, cudaMemcpyDeviceToHost));
    WC_CUDA(cudaMemcpy(depth_host, t->t.p_depth, 4 * t->t.npix, cudaMemcpyDeviceToHost));
    WC_API_END
}

int wc_frame_target_destroy(wc_frame_target *t) {
    WC_API_BEGIN
    delete t;
    WC_API_END
}

int wc_session_set_frame_target(wc_session *s, const wc_frame_target *t) {
    WC_API_BEGIN
    s->s->set_frame_target(t ? &t->t : nullptr);
    WC_API_END
}

int wc_session_stream(const wc_session *s, void **stream) {
    WC_API_BEGIN
    *stream = (void *)s->s->st;
    WC_API_END
}

int wc_session_framebuffer_packed(wc_session *s, void *dst_dev, int64_t stride_words) {
    WC_API_BEGIN
    WC_REQUIRE(stride_words >= s->s->n, wc::UsageError, "packed stride below the session's pixel count");
    s->s->pack_framebuffer(static_cast<uint32_t *>(dst_dev), stride_words);
    WC_API_END
}

int wc_scatter_pixels(const void *packed_dev, int64_t stride_words, const void *pixel_ids_dev, int64_t n,
                      void *rgba_dev, void *depth_dev, void *stream) {
    WC_API_BEGIN
    wc::scatter_pixels(static_cast<const uint32_t *>(packed_dev), stride_words,
                       static_cast<const int64_t *>(pixel_ids_dev), n, static_cast<uint32_t *>(rgba_dev),
                       static_cast<uint32_t *>(depth_dev), static_cast<cudaStream_t>(stream));
    WC_API_END
}

int wc_session_set_kernel_profile(wc_session *s, int on) {
    WC_API_BEGIN
    s->s->kernel_profile = on != 0;
    s->s->kstats.clear();
    WC_API_END
}

int wc_session_kernel_profile(const wc_session *s, char *buf, int64_t cap, int64_t *len) {
    WC_API_BEGIN
    const std::string t = s->s->kernel_profile_text();
    *len = (int64_t)t.size();
    if (buf && cap > 0) {
        const size_t k = std::min<size_t>((size_t)cap - 1, t.size());
        memcpy(buf, t.data(), k);
        buf[k] = 0;
    }
    WC_API_END
}

int wc_session_snapshot(wc_session *s, uint32_t *rgba_host, float *depth_host, int64_t *ticket) {
    WC_API_BEGIN
    WC_REQUIRE(rgba_host && depth_host, wc::UsageError, "snapshot needs host buffers");
    *ticket = s->s->snapshot_async(rgba_host, depth_host);
    WC_API_END
}

int wc_session_snapshot_wait(wc_session *s, int64_t ticket) {
    WC_API_BEGIN
    s->s->snapshot_wait(ticket);
    WC_API_END
}

int wc_session_frame_ms(wc_session *s, double *ms) {
    WC_API_BEGIN
    *ms = s->s->frame_ms();
    WC_API_END
}

int wc_session_stage_ms(const wc_session *s, double *ms6) {
    WC_API_BEGIN
    for (int k = 0; k < wc::Session::kStages; k++) ms6[k] = s->s->stage_ms[k];
    ms6[wc::Session::kStages] = s->s->reset_device_ms();
    WC_API_END
}

int wc_session_pass_stage_ms(const wc_session *s, int64_t pass_index, double *ms6) {
    WC_API_BEGIN
    WC_REQUIRE(pass_index >= 0 && pass_index < wc::Session::kMaxPassLog, wc::UsageError, "pass index out of range");
    for (int k = 0; k < wc::Session::kStages; k++) ms6[k] = s->s->pass_stage_ms[pass_index][k];
    WC_API_END
}

int wc_session_sizes(const wc_session *s, int64_t *sizes) {
    WC_API_BEGIN
    const wc::Session &S = *s->s;
    sizes[0] = S.last_slots_used;
    sizes[1] = S.last_nvis;
    sizes[2] = S.last_nactb;
    sizes[3] = S.last_nent;
    sizes[4] = S.last_n_spec;
    sizes[5] = S.last_slots_used / (S.last_n_spec ? S.last_n_spec : 1);
    sizes[6] = S.cap;
    sizes[7] = S.phys;
    sizes[8] = S.last_nlong;
    WC_API_END
}

int wc_session_rays(const wc_session *s, double *dir, double *t_enter, double *t_exit, uint8_t *status,
                    uint8_t *exited, uint32_t *coarse_cell, uint32_t *fine_cell, double *coarse_tmax,
                    double *fine_tmax) {
    WC_API_BEGIN
    const wc::Session &S = *s->s;
    const int64_t n = S.n;
    download(dir, S.dir.p, 3 * n, S.st);
    download(t_enter, S.t_enter.p, n, S.st);
    download(t_exit, S.t_exit.p, n, S.st);
    download(status, S.status.p, n, S.st);
    download(exited, S.exited.p, n, S.st);
    download(coarse_cell, S.coarse_cell.p, n, S.st);
    download(fine_cell, S.fine_cell.p, n, S.st);
    download(coarse_tmax, S.coarse_tmax.p, 3 * n, S.st);
    download(fine_tmax, S.fine_tmax.p, 3 * n, S.st);
    WC_CUDA(cudaStreamSynchronize(S.st));
    WC_API_END
}

int wc_session_slots(const wc_session *s, uint32_t *block_slots, uint32_t *ray_slots, uint32_t *active_list) {
    WC_API_BEGIN
    const wc::Session &S = *s->s;
    download(block_slots, S.block_slots.p, S.last_slots_used, S.st);
    download(ray_slots, S.ray_slots.p, S.last_slots_used, S.st);
    const int64_t n_prev = S.last_slots_used / (S.last_n_spec ? S.last_n_spec : 1);
    download(active_list, S.act_list[(S.pass_index - 1) & 1].p, n_prev, S.st);  // the last pass's list
    WC_CUDA(cudaStreamSynchronize(S.st));
    WC_API_END
}

int wc_session_blocks(const wc_session *s, uint32_t *visible_ids, uint32_t *active_ids) {
    WC_API_BEGIN
    const wc::Session &S = *s->s;
    download(visible_ids, S.visible_ids.p, S.last_nvis, S.st);
    download(active_ids, S.active_ids.p, S.last_nactb, S.st);
    WC_CUDA(cudaStreamSynchronize(S.st));
    WC_API_END
}

int wc_session_rt_inputs(const wc_session *s, uint32_t *block_ray_offsets, uint32_t *sorted_entries,
                         uint32_t *entry_ray) {
    WC_API_BEGIN
    const wc::Session &S = *s->s;
    if (S.last_nent > 0) download(block_ray_offsets, S.block_ray_off.p, S.last_nvis + 1, S.st);
    else if (block_ray_offsets) block_ray_offsets[0] = 0;
    if (S.group_entries) {
        download(sorted_entries, S.ent_val.p, S.last_nent, S.st);
    } else {  // ray-ordered entries: entry k at position k (the permutation is not stored)
        for (int64_t k = 0; k < S.last_nent; k++) sorted_entries[k] = (uint32_t)k;
    }
    download(entry_ray, S.ent_ray.p, S.last_nent, S.st);
    WC_CUDA(cudaStreamSynchronize(S.st));
    WC_API_END
}

int wc_session_rgbz(const wc_session *s, float *rgbz) {
    WC_API_BEGIN
    const wc::Session &S = *s->s;
    download(reinterpret_cast<float4 *>(rgbz), S.rgbz.p, S.last_nent, S.st);
    WC_CUDA(cudaStreamSynchronize(S.st));
    WC_API_END
}

int wc_session_cache(const wc_session *s, int32_t *block_of_slot, int32_t *last_used, float *slot_values) {
    WC_API_BEGIN
    const wc::Session &S = *s->s;
    download(block_of_slot, S.block_of_slot.p, S.phys, S.st);
    download(last_used, S.last_used.p, S.phys, S.st);
    download(slot_values, S.slot_values.p, S.phys * 64, S.st);
    WC_CUDA(cudaStreamSynchronize(S.st));
    WC_API_END
}

int wc_init_rays(const wc_camera *cam, const uint32_t *pixel_ids, int64_t n, const double *origins,
                 const double *dirs, int nx, int ny, int nz, double *dir_out, double *t_enter, double *t_exit,
                 uint8_t *status, uint8_t *exited, uint32_t *coarse_cell, uint32_t *fine_cell, double *coarse_tmax,
                 double *fine_tmax) {
    WC_API_BEGIN
    check_dims(nx, ny, nz);
    if (!dirs && !pixel_ids) n = (int64_t)cam->img_w * cam->img_h;
    if (n <= 0) return WC_OK;
    cudaStream_t st;
    WC_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    wc::DevBuf<uint32_t> d_pix, d_cc, d_fc;
    wc::DevBuf<double> d_o, d_d, d_dir, d_te, d_tx, d_ct, d_ft;
    wc::DevBuf<uint8_t> d_st, d_ex;
    if (pixel_ids) upload(d_pix, pixel_ids, n, st);
    if (dirs) {
        upload(d_o, origins, 3 * n, st);
        upload(d_d, dirs, 3 * n, st);
    }
    d_dir.alloc(3 * n);
    d_te.alloc(n);
    d_tx.alloc(n);
    d_st.alloc(n);
    d_ex.alloc(n);
    d_cc.alloc(n);
    d_fc.alloc(n);
    d_ct.alloc(3 * n);
    d_ft.alloc(3 * n);
    wc::CameraParams cp{};
    if (cam) std::memcpy(&cp, cam, sizeof(cp));
    wc::init_rays_device(cam ? &cp : nullptr, pixel_ids ? d_pix.p : nullptr, n, dirs ? d_o.p : nullptr,
                         dirs ? d_d.p : nullptr, nx, ny, nz, nullptr, d_dir.p, d_te.p, d_tx.p, d_st.p, d_ex.p,
                         d_cc.p, d_fc.p, d_ct.p, d_ft.p, st);
    download(dir_out, d_dir.p, 3 * n, st);
    download(t_enter, d_te.p, n, st);
    download(t_exit, d_tx.p, n, st);
    download(status, d_st.p, n, st);
    download(exited, d_ex.p, n, st);
    download(coarse_cell, d_cc.p, n, st);
    download(fine_cell, d_fc.p, n, st);
    download(coarse_tmax, d_ct.p, 3 * n, st);
    download(fine_tmax, d_ft.p, 3 * n, st);
    WC_CUDA(cudaStreamSynchronize(st));
    cudaStreamDestroy(st);
    WC_API_END
}

int wc_reference_render(const wc_volume *v, const double *origins, const double *dirs, int64_t n, double iso,
                        double base_r, double base_g, double base_b, uint8_t *rgba, float *depth) {
    WC_API_BEGIN
    const wc::Volume &V = v->v;
    if (n <= 0) return WC_OK;
    wc::DevBuf<float> dense;
    dense.alloc((int64_t)V.nx * V.ny * V.nz);
    wc::decode_full_device(V, dense.p, V.st);
    wc::DevBuf<double> d_o, d_d;
    upload(d_o, origins, 3 * n, V.st);
    upload(d_d, dirs, 3 * n, V.st);
    wc::DevBuf<uint32_t> d_rgba;
    wc::DevBuf<float> d_depth;
    d_rgba.alloc(n);
    d_depth.alloc(n);
    wc::reference_render_device(dense.p, V.nx, V.ny, V.nz, d_o.p, d_d.p, n, iso, base_r, base_g, base_b, d_rgba.p,
                                d_depth.p, V.st);
    download(reinterpret_cast<uint32_t *>(rgba), d_rgba.p, n, V.st);
    download(depth, d_depth.p, n, V.st);
    WC_CUDA(cudaStreamSynchronize(V.st));
    WC_API_END
}

int wc_reference_render_dense(const float *values, int nx, int ny, int nz, const double *origins, const double *dirs,
                              int64_t n, double iso, double base_r, double base_g, double base_b, uint8_t *rgba,
                              float *depth) {
    WC_API_BEGIN
    check_dims(nx, ny, nz);
    if (n <= 0) return WC_OK;
    cudaStream_t st;
    WC_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    wc::DevBuf<float> dense, d_depth;
    wc::DevBuf<double> d_o, d_d;
    wc::DevBuf<uint32_t> d_rgba;
    upload(dense, values, (int64_t)nx * ny * nz, st);
    upload(d_o, origins, 3 * n, st);
    upload(d_d, dirs, 3 * n, st);
    d_rgba.alloc(n);
    d_depth.alloc(n);
    wc::reference_render_device(dense.p, nx, ny, nz, d_o.p, d_d.p, n, iso, base_r, base_g, base_b, d_rgba.p,
                                d_depth.p, st);
    download(reinterpret_cast<uint32_t *>(rgba), d_rgba.p, n, st);
    download(depth, d_depth.p, n, st);
    WC_CUDA(cudaStreamSynchronize(st));
    cudaStreamDestroy(st);
    WC_API_END
}

int wc_exclusive_scan(const uint32_t *values, int64_t n, uint32_t *out, uint64_t *total) {
    WC_API_BEGIN
    if (n <= 0) {
        if (total) *total = 0;
        return WC_OK;
    }
    cudaStream_t st;
    WC_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    wc::DevBuf<uint32_t> d_in, d_out, d_part, d_tot;
    upload(d_in, values, n, st);
    d_out.alloc(n);
    d_part.alloc(wc::scan_scratch_words(n));
    WC_CUDA(cudaMemsetAsync(d_part.p, 0, 4 * d_part.n, st));
    d_tot.alloc(1);
    wc::scan_exclusive(wc::LoadU32{d_in.p}, n, d_out.p, d_tot.p, d_part.p, st);
    uint32_t t = 0;
    download(out, d_out.p, n, st);
    download(&t, d_tot.p, 1, st);
    WC_CUDA(cudaStreamSynchronize(st));
    cudaStreamDestroy(st);
    if (total) *total = t;
    WC_API_END
}

namespace {
struct PredMaskU8 {
    const uint8_t *m;
    __device__ __forceinline__ uint32_t operator()(int64_t i) const { return m[i] != 0; }
};
__global__ void k_iota(uint32_t *p, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = (uint32_t)i;
}
}  // namespace

int wc_compact_indices(const uint8_t *mask, int64_t n, uint32_t *out, uint64_t *total) {
    WC_API_BEGIN
    if (n <= 0) {
        if (total) *total = 0;
        return WC_OK;
    }
    cudaStream_t st;
    WC_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    wc::DevBuf<uint8_t> d_m;
    wc::DevBuf<uint32_t> d_idx, d_out, d_part, d_tot;
    upload(d_m, mask, n, st);
    d_idx.alloc(n);
    k_iota<<<wc::grid_for(n, 256), 256, 0, st>>>(d_idx.p, n);
    WC_LAUNCH_CHECK();
    d_out.alloc(n);
    d_part.alloc(wc::scan_scratch_words(n));
    WC_CUDA(cudaMemsetAsync(d_part.p, 0, 4 * d_part.n, st));
    d_tot.alloc(1);
    wc::compact_dev(PredMaskU8{d_m.p}, d_idx.p, nullptr, n, d_out.p, d_tot.p, d_part.p, st);
    uint32_t t = 0;
    download(&t, d_tot.p, 1, st);
    WC_CUDA(cudaStreamSynchronize(st));
    download(out, d_out.p, t, st);
    WC_CUDA(cudaStreamSynchronize(st));
    cudaStreamDestroy(st);
    if (total) *total = t;
    WC_API_END
}

int wc_sort_by_key(uint32_t *keys, uint32_t *values, int64_t n) {
    WC_API_BEGIN
    if (n <= 1) return WC_OK;
    cudaStream_t st;
    WC_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    wc::DevBuf<uint32_t> dk, dv;
    upload(dk, keys, n, st);
    upload(dv, values, n, st);
    wc::RadixScratch rs;
    wc::radix_sort_pairs(dk.p, dv.p, n, 32, rs, st);
    download(keys, dk.p, n, st);
    download(values, dv.p, n, st);
    WC_CUDA(cudaStreamSynchronize(st));
    cudaStreamDestroy(st);
    WC_API_END
}

/* ---- stage-level entry points (wc_stage.cu) */

int wc_traverse(const wc_volume *v, const double *fine_min, const double *fine_max, const double *coarse_min,
                const double *coarse_max, const int *fine_dims, const int *coarse_dims, int64_t n,
                const double *origin, const double *dir, const double *t_exit, const uint8_t *status, uint8_t *exited,
                uint32_t *coarse_cell, double *coarse_tmax, uint32_t *fine_cell, double *fine_tmax,
                uint32_t *block_slots, uint32_t *ray_slots, const int64_t *active_offsets, double iso, int n_spec,
                int variant) {
    WC_API_BEGIN
    WC_REQUIRE(n >= 0, wc::UsageError, "negative ray count");
    WC_REQUIRE(v || (fine_min && fine_max && coarse_min && coarse_max), wc::UsageError, "no grids");
    wc::stage_traverse(v ? &v->v : nullptr, fine_min, fine_max, coarse_min, coarse_max, fine_dims, coarse_dims, n,
                       origin, dir, t_exit, status, exited, coarse_cell, coarse_tmax, fine_cell, fine_tmax,
                       block_slots, ray_slots, active_offsets, iso, n_spec, variant);
    WC_API_END
}

int wc_mark_blocks(const uint32_t *block_slots, int64_t n, int bdx, int bdy, int bdz, uint32_t *visible_words,
                   uint32_t *active_words) {
    WC_API_BEGIN
    WC_REQUIRE(bdx > 0 && bdy > 0 && bdz > 0, wc::UsageError, "block dims must be positive");
    wc::stage_mark_blocks(block_slots, n, bdx, bdy, bdz, visible_words, active_words);
    WC_API_END
}

int wc_build_rt_inputs(const uint32_t *block_slots, const uint32_t *ray_slots, int64_t n,
                       const uint32_t *visible_words, int64_t n_blocks, uint32_t *visible_ids,
                       uint32_t *rays_per_block, uint32_t *block_ray_offsets, uint32_t *sorted_ray_ids,
                       uint32_t *sorted_hit_slots, uint32_t *valid_prefix, int64_t *sizes) {
    WC_API_BEGIN
    WC_REQUIRE(n >= 0 && n_blocks >= 0, wc::UsageError, "negative size");
    wc::stage_build_rt_inputs(block_slots, ray_slots, n, visible_words, n_blocks, visible_ids, rays_per_block,
                              block_ray_offsets, sorted_ray_ids, sorted_hit_slots, valid_prefix, sizes);
    WC_API_END
}

int wc_composite(const float *rgbz_rgb, const float *rgbz_z, int64_t n_rgbz, int64_t n, uint8_t *status,
                 const uint8_t *exited, const int64_t *active_offsets, int n_spec, const uint32_t *block_slots,
                 int64_t n_slots, const uint32_t *valid_prefix, uint8_t *rgba, float *depth) {
    WC_API_BEGIN
    WC_REQUIRE(n_spec >= 1, wc::UsageError, "n_spec must be >= 1");
    wc::stage_composite(rgbz_rgb, rgbz_z, n_rgbz, n, status, exited, active_offsets, n_spec, block_slots, n_slots,
                        valid_prefix, rgba, depth);
    WC_API_END
}

int wc_cache_create(int64_t capacity_slots, wc_cache **out) {
    WC_API_BEGIN
    auto *h = new wc_cache();
    try {
        h->c = new wc::StageCache(capacity_slots);
    } catch (...) {
        delete h;
        throw;
    }
    *out = h;
    WC_API_END
}

int wc_cache_destroy(wc_cache *c) {
    WC_API_BEGIN
    if (c) {
        delete c->c;
        delete c;
    }
    WC_API_END
}

int wc_cache_ensure_resident(wc_cache *c, const wc_volume *v, const uint32_t *active_words, int64_t n_blocks,
                             int64_t needed, int64_t *new_decompressed, int64_t *evicted, int64_t *grown_to) {
    WC_API_BEGIN
    WC_REQUIRE(c && v, wc::UsageError, "null handle");
    WC_REQUIRE(n_blocks == v->v.n_blocks, wc::UsageError, "active mask length differs from the block count");
    c->c->ensure_resident(&v->v, active_words, needed, new_decompressed, evicted, grown_to);
    WC_API_END
}

int wc_cache_info(const wc_cache *c, int64_t *capacity, int64_t *physical, int64_t *current_pass, int64_t *n_blocks) {
    WC_API_BEGIN
    WC_REQUIRE(c, wc::UsageError, "null handle");
    if (capacity) *capacity = c->c->cap;
    if (physical) *physical = c->c->vol ? c->c->phys : 0;
    if (current_pass) *current_pass = c->c->current_pass;
    if (n_blocks) *n_blocks = c->c->n_blocks;
    WC_API_END
}

int wc_cache_lookup(wc_cache *c, int64_t block_id, int64_t *slot) {
    WC_API_BEGIN
    WC_REQUIRE(c, wc::UsageError, "null handle");
    *slot = c->c->lookup(block_id);
    WC_API_END
}

int wc_cache_state(wc_cache *c, float *slot_values, int32_t *block_of_slot, int32_t *last_used,
                   int32_t *slot_of_block) {
    WC_API_BEGIN
    WC_REQUIRE(c, wc::UsageError, "null handle");
    c->c->download(slot_values, block_of_slot, last_used, slot_of_block);
    WC_API_END
}

int wc_cache_dual_grid(wc_cache *c, int64_t block_id, float *values125) {
    WC_API_BEGIN
    WC_REQUIRE(c, wc::UsageError, "null handle");
    c->c->dual_grid(block_id, values125);
    WC_API_END
}

int wc_intersect_cells(int64_t n, const float *corners, const double *origin, const double *dir, const double *cell,
                       const double *t0, const double *t1, double iso, double *t_out) {
    WC_API_BEGIN
    wc::stage_intersect_cells(n, corners, origin, dir, cell, t0, t1, iso, t_out);
    WC_API_END
}

int wc_cell_overlaps(int64_t n, const double *origin, const double *dir, const double *cell, double *t0, double *t1) {
    WC_API_BEGIN
    wc::stage_cell_overlaps(n, origin, dir, cell, t0, t1);
    WC_API_END
}

int wc_check_fastdiv(int64_t n, uint64_t seed, int64_t *mismatches, double *example) {
    WC_API_BEGIN
    const int64_t bad = wc::stage_check_fastdiv(n, seed, example);
    if (mismatches) *mismatches = bad;
    WC_API_END
}

int wc_shade(int64_t n, const double *grad, const double *dir, const double *base_color, double *rgb) {
    WC_API_BEGIN
    wc::stage_shade(n, grad, dir, base_color, rgb);
    WC_API_END
}

int wc_raytrace_block(const float *values125, const int *block_origin, const int *cells_per_axis, int64_t n,
                      const double *origin, const double *dir, const double *t_enter, double iso,
                      const double *base_color, float *rgb, float *z, uint8_t *hit) {
    WC_API_BEGIN
    wc::stage_raytrace_block(values125, block_origin, cells_per_axis, n, origin, dir, t_enter, iso, base_color, rgb, z,
                             hit);
    WC_API_END
}

}  // extern "C"
