// pgm_io.cu -- denoise of a binary PGM file with the file I/O overlapped
// with the host<->device copies (the reference's codec is
// proj/include/phgrms/pgm.hpp:75-176, its CLI path tools/phgrms_main.cpp).
//
// phg_denoise_pgm_file(in, out, params): the P5 raster is read from the file
// in row chunks into two pinned staging buffers; while chunk c+1 is read from
// the file, chunk c is already on its way to the device (cudaMemcpy2DAsync
// into the 16-byte-pitched layout the fused kernels read).  After the device
// denoise (phg_dev_denoise), the result comes back in row chunks the same way:
// chunk c+1's D2H runs while chunk c is written to the output file.  The
// header parsing, the error texts and the written file are the reference's
// (read_pgm / write_pgm(ascii = false)); only binary P5 input takes this path.
// Host code over the public C ABI; no kernels of its own.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/phgrms_b200.h"

namespace phg_internal {
void set_error(const std::string& msg);  // phg_last_error() (phgrms_cuda.cu)
}

namespace {

int pgm_fail(int code, const std::string& msg) {
    phg_internal::set_error(msg);
    return code;
}

bool is_space(int ch) { return ch == ' ' || ch == '\t' || ch == '\n' || ch == '\r' || ch == '\v' || ch == '\f'; }

// The P5 header: magic, width, height, maxval ('#' comments and whitespace
// before each number), then one whitespace byte -- or a comment through its
// newline -- before the raster (read_pgm, pgm.hpp:98-131).
struct Header {
    long w = 0, h = 0, maxval = 0;
    long raster_at = 0;  // file offset of the first pixel
};

int parse_header(FILE* f, Header* hd) {
    int c0 = std::fgetc(f), c1 = std::fgetc(f);
    if (c0 != 'P' || (c1 != '2' && c1 != '5'))
        return pgm_fail(PHG_EINVAL, "not a PGM stream (expected P2 or P5 magic)");
    if (c1 == '2') return pgm_fail(PHG_EINVAL, "phg_denoise_pgm_file reads binary P5 (load P2 with load_pgm)");
    long v[3];
    for (long& x : v) {
        int ch = std::fgetc(f);
        for (;;) {
            if (ch == EOF) break;
            if (is_space(ch)) {
                ch = std::fgetc(f);
            } else if (ch == '#') {
                while (ch != EOF && ch != '\n') ch = std::fgetc(f);
            } else {
                break;
            }
        }
        if (ch < '0' || ch > '9') return pgm_fail(PHG_EINVAL, "malformed PGM header");
        x = 0;
        while (ch >= '0' && ch <= '9') {
            x = x * 10 + (ch - '0');
            if (x > (1l << 31)) return pgm_fail(PHG_EINVAL, "malformed PGM header");
            ch = std::fgetc(f);
        }
        std::ungetc(ch, f);
    }
    hd->w = v[0];
    hd->h = v[1];
    hd->maxval = v[2];
    if (hd->w < 1 || hd->h < 1 || hd->maxval < 1) return pgm_fail(PHG_EINVAL, "malformed PGM header");
    if (hd->maxval > 255) return pgm_fail(PHG_EINVAL, "16-bit PGM unsupported");
    int ch = std::fgetc(f);
    if (ch == '#') {
        while (ch != EOF && ch != '\n') ch = std::fgetc(f);
        if (ch == EOF) return pgm_fail(PHG_EINVAL, "truncated PGM pixel data");
    } else if (ch == EOF || !is_space(ch)) {
        return pgm_fail(PHG_EINVAL, "malformed PGM header");
    }
    hd->raster_at = std::ftell(f);
    return PHG_OK;
}

#define PGM_CUDA(expr)                                                                          \
    do {                                                                                        \
        cudaError_t e_ = (expr);                                                                \
        if (e_ != cudaSuccess) return pgm_fail(PHG_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)

struct FileCloser {
    void operator()(FILE* f) const {
        if (f) std::fclose(f);
    }
};

// Device and pinned resources of one call, released on every exit path.
struct Resources {
    cudaStream_t st = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    uint8_t* pin[2] = {nullptr, nullptr};
    void* dev = nullptr;
    ~Resources() {
        if (st) cudaStreamSynchronize(st);
        for (auto* p : pin)
            if (p) cudaFreeHost(p);
        if (dev) cudaFree(dev);
        for (auto e : ev)
            if (e) cudaEventDestroy(e);
        if (st) cudaStreamDestroy(st);
    }
};

}  // namespace

extern "C" int phg_denoise_pgm_file(const char* in_path, const char* out_path, const phg_params* p,
                                    phg_pass_stats* stats, int* iterations_run) {
    if (!in_path || !out_path || !p || !stats || !iterations_run) return pgm_fail(PHG_EINVAL, "null argument");
    if (phg_validate_params(p) != PHG_OK) return PHG_EINVAL;  // message set by the validator
    std::unique_ptr<FILE, FileCloser> in(std::fopen(in_path, "rb"));
    if (!in) return pgm_fail(PHG_EINVAL, std::string("cannot open ") + in_path);
    Header hd;
    if (int rc = parse_header(in.get(), &hd); rc != PHG_OK) return rc;
    const int w = static_cast<int>(hd.w), h = static_cast<int>(hd.h);
    const int64_t pitch = (static_cast<int64_t>(w) + 15) / 16 * 16;
    const int64_t img_bytes = pitch * h;
    const int k = p->max_iterations;
    // ~16 MB row chunks, double buffered
    const int64_t chunk_rows = std::max<int64_t>(1, std::min<int64_t>(h, (int64_t(16) << 20) / w));
    Resources r;
    PGM_CUDA(cudaStreamCreateWithFlags(&r.st, cudaStreamNonBlocking));
    for (auto& e : r.ev) PGM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& b : r.pin) PGM_CUDA(cudaHostAlloc(&b, static_cast<size_t>(chunk_rows * w), cudaHostAllocDefault));
    PGM_CUDA(cudaMalloc(&r.dev, static_cast<size_t>(3 * img_bytes + 16 * k + 256)));
    uint8_t* base = static_cast<uint8_t*>(r.dev);
    phg_dev_image im[3];
    for (int i = 0; i < 3; ++i) im[i] = {base + i * img_bytes, pitch, img_bytes, w, h, 1, 0};
    uint64_t* ctr = reinterpret_cast<uint64_t*>(base + 3 * img_bytes + 128 - (3 * img_bytes) % 128);

    // file -> pinned chunk (CPU) overlapped with pinned chunk -> device (DMA)
    int64_t row = 0;
    for (int c = 0; row < h; ++c) {
        const int b = c & 1;
        const int64_t rows = std::min<int64_t>(chunk_rows, h - row);
        PGM_CUDA(cudaEventSynchronize(r.ev[b]));  // the chunk's buffer is free again
        const size_t n = static_cast<size_t>(rows * w);
        if (std::fread(r.pin[b], 1, n, in.get()) != n) return pgm_fail(PHG_EINVAL, "truncated PGM pixel data");
        if (hd.maxval < 255 && *std::max_element(r.pin[b], r.pin[b] + n) > hd.maxval)
            return pgm_fail(PHG_EINVAL, "PGM pixel value exceeds maxval");
        PGM_CUDA(cudaMemcpy2DAsync(im[0].data + row * pitch, pitch, r.pin[b], w, w, rows, cudaMemcpyHostToDevice,
                                   r.st));
        PGM_CUDA(cudaEventRecord(r.ev[b], r.st));
        row += rows;
    }
    in.reset();
    if (int rc = phg_dev_denoise(&im[0], &im[1], &im[2], p, ctr, r.st); rc != PHG_OK) return rc;
    std::vector<uint64_t> hc(static_cast<size_t>(2) * k);
    PGM_CUDA(cudaMemcpyAsync(hc.data(), ctr, sizeof(uint64_t) * hc.size(), cudaMemcpyDeviceToHost, r.st));

    std::unique_ptr<FILE, FileCloser> out(std::fopen(out_path, "wb"));
    if (!out) return pgm_fail(PHG_EINVAL, std::string("cannot open ") + out_path + " for writing");
    const std::string header = "P5\n" + std::to_string(w) + ' ' + std::to_string(h) + "\n255\n";
    if (std::fwrite(header.data(), 1, header.size(), out.get()) != header.size())
        return pgm_fail(PHG_EINVAL, std::string("write failed for ") + out_path);
    // device -> pinned chunk (DMA) overlapped with pinned chunk -> file (CPU)
    const int64_t nchunks = (h + chunk_rows - 1) / chunk_rows;
    auto d2h = [&](int64_t c) -> int {
        const int64_t r0 = c * chunk_rows, rows = std::min<int64_t>(chunk_rows, h - r0);
        PGM_CUDA(cudaMemcpy2DAsync(r.pin[c & 1], w, im[1].data + r0 * pitch, pitch, w, rows,
                                   cudaMemcpyDeviceToHost, r.st));
        PGM_CUDA(cudaEventRecord(r.ev[c & 1], r.st));
        return PHG_OK;
    };
    if (int rc = d2h(0); rc != PHG_OK) return rc;
    for (int64_t c = 0; c < nchunks; ++c) {
        if (c + 1 < nchunks)
            if (int rc = d2h(c + 1); rc != PHG_OK) return rc;
        PGM_CUDA(cudaEventSynchronize(r.ev[c & 1]));
        const int64_t rows = std::min<int64_t>(chunk_rows, h - c * chunk_rows);
        const size_t n = static_cast<size_t>(rows * w);
        if (std::fwrite(r.pin[c & 1], 1, n, out.get()) != n)
            return pgm_fail(PHG_EINVAL, std::string("write failed for ") + out_path);
        // the buffer is refilled by d2h(c + 2) only after this write
    }
    if (std::fflush(out.get()) != 0) return pgm_fail(PHG_EINVAL, std::string("write failed for ") + out_path);
    PGM_CUDA(cudaStreamSynchronize(r.st));
    return phg_finalize_stats(hc.data(), 1, k, stats, iterations_run);
}
