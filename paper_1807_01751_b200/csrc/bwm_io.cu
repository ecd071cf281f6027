// bwm_io.cu — BTS1 payload reads, the staged file->pinned reader, and the break-map CSV
// writer of libbwm (host code; see bwm_io.h and include/bwm.h).
//
// Reference surfaces these replace (pkg/src/breakwatch/dataio.py):
//   read_stack      dataio.py:79-115  — header parse stays in Python (17 bytes, same errors);
//                                       the payload read is bwm_read_payload (parallel pread)
//   write_break_map dataio.py:168-182 — one row per pixel, floats at 9 significant digits
//                                       ("%.9g", byte-identical to Python's f"{x:.9g}"),
//                                       first_break empty when no break was found
#include "../../include/bwm.h"
#include "bwm_io.h"

#include <cuda_runtime.h>
#include <errno.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>

namespace bwm {
int set_error(int code, const std::string& msg);   // bwm_capi.cu (thread-local last error)

static int err_code(std::string* err, int code, const std::string& msg) {
    if (err) *err = msg;
    return code;
}

int PayloadFile::open(const char* path, int64_t off, int64_t nobs, int64_t npx, std::string* err) {
    close();
    fd = ::open(path, O_RDONLY | O_CLOEXEC);
    if (fd < 0) return err_code(err, BWM_E_IO, std::string("cannot open ") + path + ": " + strerror(errno));
    struct stat st {};
    if (fstat(fd, &st) != 0) return err_code(err, BWM_E_IO, std::string("cannot stat ") + path);
    const int64_t need = off + nobs * npx * 4;
    if ((int64_t)st.st_size < need) {
        const int64_t got = std::max<int64_t>(0, (int64_t)st.st_size - off);
        return err_code(err, BWM_E_FORMAT,
                        "truncated sample payload: wanted " + std::to_string(nobs * npx * 4) + " bytes, got " +
                            std::to_string(got));
    }
    offset = off;
    n_obs = nobs;
    n_px = npx;
    posix_fadvise(fd, off, nobs * npx * 4, POSIX_FADV_SEQUENTIAL);
    return BWM_OK;
}

void PayloadFile::close() {
    if (fd >= 0) ::close(fd);
    fd = -1;
}

static bool pread_full(int fd, void* dst, int64_t bytes, int64_t at) {
    char* p = static_cast<char*>(dst);
    while (bytes > 0) {
        const ssize_t got = ::pread(fd, p, (size_t)std::min<int64_t>(bytes, 1ll << 30), (off_t)at);
        if (got < 0 && errno == EINTR) continue;
        if (got <= 0) return false;
        p += got;
        at += got;
        bytes -= got;
    }
    return true;
}

int PayloadFile::read_rect(const Rect& r, float* dst, int threads, std::string* err) const {
    const int64_t w = r.c1 - r.c0, rows = r.r1 - r.r0;
    const bool whole = r.c0 == 0 && r.c1 == n_px;      // one contiguous file range
    const int64_t total = rows * w * 4;
    threads = (int)std::max<int64_t>(1, std::min<int64_t>(threads, whole ? (total >> 22) + 1 : rows));
    std::atomic<bool> ok{true};
    auto part = [&](int i) {
        if (whole) {
            const int64_t a = (total * i / threads) & ~int64_t(4095), b = i + 1 == threads ? total
                                                                       : (total * (i + 1) / threads) & ~int64_t(4095);
            if (b > a && !pread_full(fd, reinterpret_cast<char*>(dst) + a, b - a, offset + r.r0 * n_px * 4 + a))
                ok = false;
        } else {
            for (int64_t t = r.r0 + i; t < r.r1; t += threads)
                if (!pread_full(fd, dst + (t - r.r0) * w, w * 4, offset + (t * n_px + r.c0) * 4)) ok = false;
        }
    };
    if (threads == 1) {
        part(0);
    } else {
        std::vector<std::thread> th;
        for (int i = 1; i < threads; ++i) th.emplace_back(part, i);
        part(0);
        for (auto& t : th) t.join();
    }
    if (!ok) return err_code(err, BWM_E_IO, std::string("short read of the stack payload: ") + strerror(errno));
    return BWM_OK;
}

void plan_rects(int64_t n_obs, int64_t c0, int64_t c1, int64_t chunk, int64_t slot_bytes, std::vector<Rect>* out) {
    const int64_t w = c1 - c0;
    if (w * 4 <= slot_bytes) {
        const int64_t g = std::max<int64_t>(1, slot_bytes / (w * 4));
        for (int64_t r = 0; r < n_obs; r += g) out->push_back({r, std::min(n_obs, r + g), c0, c1, chunk});
    } else {                                          // a row is larger than a slot: split columns
        const int64_t cw = std::max<int64_t>(64, (slot_bytes / 4) & ~int64_t(63));
        for (int64_t r = 0; r < n_obs; ++r)
            for (int64_t c = c0; c < c1; c += cw) out->push_back({r, r + 1, c, std::min(c1, c + cw), chunk});
    }
}

int StagedReader::ensure(int slots, int64_t slot_bytes, std::string* err) {
    if ((int)slot_.size() == slots && slot_bytes_ == slot_bytes) return BWM_OK;
    for (float* s : slot_) cudaFreeHost(s);
    slot_.clear();
    for (int i = 0; i < slots; ++i) {
        void* p = nullptr;
        const cudaError_t e = cudaHostAlloc(&p, (size_t)slot_bytes, cudaHostAllocPortable);
        if (e != cudaSuccess) {
            for (float* s : slot_) cudaFreeHost(s);
            slot_.clear();
            return err_code(err, (int)e, std::string("pinned staging allocation failed: ") + cudaGetErrorString(e));
        }
        slot_.push_back(static_cast<float*>(p));
    }
    slot_bytes_ = slot_bytes;
    return BWM_OK;
}

void HostSource::copy_rect(const Rect& r, float* dst) const {
    const int64_t w = r.c1 - r.c0;
    if (w == ld) {                                          // whole rows: one contiguous block
        std::memcpy(dst, base + r.r0 * ld, (size_t)((r.r1 - r.r0) * w * 4));
        return;
    }
    for (int64_t t = r.r0; t < r.r1; ++t) std::memcpy(dst + (t - r.r0) * w, base + t * ld + r.c0, (size_t)w * 4);
}

int StagedReader::start(const HostSource* h, const std::vector<Rect>* rects, int threads) {
    stop();
    f_ = nullptr;
    h_ = h;
    return launch(rects, threads);
}

int StagedReader::start(const PayloadFile* f, const std::vector<Rect>* rects, int threads) {
    stop();
    f_ = f;
    h_ = nullptr;
    return launch(rects, threads);
}

int StagedReader::launch(const std::vector<Rect>* rects, int threads) {
    rects_ = rects;
    next_ = 0;
    released_ = 0;
    abort_ = failed_ = false;
    err_.clear();
    done_.assign(rects->size(), 0);
    threads = std::max(1, std::min<int>(threads, (int)slot_.size()));
    for (int i = 0; i < threads; ++i) pool_.emplace_back(&StagedReader::worker, this);
    return BWM_OK;
}

void StagedReader::worker() {
    const int64_t K = (int64_t)slot_.size(), n = (int64_t)rects_->size();
    for (;;) {
        const int64_t g = next_.fetch_add(1);
        if (g >= n) return;
        {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] { return abort_ || released_ > g - K; });
            if (abort_) return;
        }
        std::string e;
        int rc = BWM_OK;
        if (h_)
            h_->copy_rect((*rects_)[g], slot_[g % K]);
        else
            rc = f_->read_rect((*rects_)[g], slot_[g % K], 1, &e);
        std::lock_guard<std::mutex> lk(mu_);
        if (rc != BWM_OK) {
            failed_ = abort_ = true;
            err_ = e;
        } else {
            done_[g] = 1;
        }
        cv_.notify_all();
        if (rc != BWM_OK) return;
    }
}

const float* StagedReader::wait(int64_t g) {
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [&] { return failed_ || done_[g]; });
    if (!done_[g]) return nullptr;
    return slot_[g % (int64_t)slot_.size()];
}

void StagedReader::release(int64_t g) {
    std::lock_guard<std::mutex> lk(mu_);
    if (g + 1 > released_) released_ = g + 1;
    cv_.notify_all();
}

void StagedReader::stop() {
    {
        std::lock_guard<std::mutex> lk(mu_);
        abort_ = true;
        cv_.notify_all();
    }
    for (auto& t : pool_) t.join();
    pool_.clear();
}

StagedReader::~StagedReader() {
    stop();
    for (float* s : slot_) cudaFreeHost(s);
}

}  // namespace bwm

// ---- C ABI -----------------------------------------------------------------------------
namespace {
// Python's format(x, ".9g") for the values a break map holds (dataio.py:180): C's "%.9g"
// produces the same digits (both correctly rounded); NaN/inf spelled as Python does.
int fmt_g9(char* out, double x) {
    if (std::isnan(x)) return (int)(std::memcpy(out, "nan", 3), 3);
    if (std::isinf(x)) return x > 0 ? (int)(std::memcpy(out, "inf", 3), 3) : (int)(std::memcpy(out, "-inf", 4), 4);
    return std::snprintf(out, 32, "%.9g", x);
}
}  // namespace

extern "C" {

int bwm_read_payload(const char* path, int64_t offset, int64_t n_obs, int64_t n_pixels, float* dst, int threads) {
    if (!path || !dst) return bwm::set_error(BWM_E_NULL, "path/dst is NULL");
    if (n_obs < 1 || n_pixels < 1 || offset < 0) return bwm::set_error(BWM_E_DIMS, "invalid payload geometry");
    bwm::PayloadFile f;
    std::string err;
    int rc = f.open(path, offset, n_obs, n_pixels, &err);
    if (rc) return bwm::set_error(rc, err);
    if (threads < 1) threads = (int)std::max(1u, std::thread::hardware_concurrency());
    rc = f.read_rect({0, n_obs, 0, n_pixels, 0}, dst, threads, &err);
    return rc ? bwm::set_error(rc, err) : BWM_OK;
}

int64_t bwm_write_break_map(const char* path, int64_t n_pixels, const uint8_t* valid, const uint8_t* detected,
                            const int64_t* first_break, const double* max_abs_mo, int threads) {
    if (!path || !valid || !detected || !first_break || !max_abs_mo)
        return bwm::set_error(BWM_E_NULL, "path and the four maps are required");
    if (n_pixels < 0) return bwm::set_error(BWM_E_DIMS, "n_pixels < 0");
    FILE* fp = std::fopen(path, "wb");
    if (!fp) return bwm::set_error(BWM_E_IO, std::string("cannot open ") + path + ": " + strerror(errno));
    static const char kHeader[] = "pixel,valid,detected,first_break,max_abs_mo\n";
    bool ok = std::fwrite(kHeader, 1, sizeof kHeader - 1, fp) == sizeof kHeader - 1;
    if (threads < 1) threads = (int)std::max(1u, std::thread::hardware_concurrency());
    // blocks of pixels formatted in parallel, written in order
    const int64_t block = 1 << 18;
    std::vector<std::string> buf((size_t)threads);
    for (int64_t b0 = 0; ok && b0 < n_pixels; b0 += block * threads) {
        auto fmt_block = [&](int i) {
            std::string& s = buf[(size_t)i];
            s.clear();
            const int64_t a = b0 + i * block, e = std::min(n_pixels, a + block);
            if (a >= e) return;
            s.reserve((size_t)(e - a) * 40);
            char line[96];
            for (int64_t px = a; px < e; ++px) {
                int k = std::snprintf(line, 64, "%lld,%d,%d,", (long long)px, valid[px] ? 1 : 0, detected[px] ? 1 : 0);
                if (first_break[px]) k += std::snprintf(line + k, 24, "%lld", (long long)first_break[px]);
                line[k++] = ',';
                k += fmt_g9(line + k, max_abs_mo[px]);
                line[k++] = '\n';
                s.append(line, (size_t)k);
            }
        };
        std::vector<std::thread> th;
        for (int i = 1; i < threads; ++i) th.emplace_back(fmt_block, i);
        fmt_block(0);
        for (auto& t : th) t.join();
        for (int i = 0; ok && i < threads; ++i)
            ok = std::fwrite(buf[(size_t)i].data(), 1, buf[(size_t)i].size(), fp) == buf[(size_t)i].size();
    }
    ok = (std::fclose(fp) == 0) && ok;
    if (!ok) return bwm::set_error(BWM_E_IO, std::string("write failed: ") + path);
    return n_pixels;
}

}  // extern "C"
