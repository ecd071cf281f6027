// bwm_io.h — host-side file I/O of libbwm (internal; the C ABI is in include/bwm.h).
//
// BTS1 stack files (reference pkg/src/breakwatch/dataio.py:1-13) store the samples time-major,
// float32 little-endian, exactly the layout the kernel reads, so a payload rectangle (rows
// [r0, r1) x pixels [c0, c1)) goes from the page cache into pinned host memory with one pread
// per row (one pread in total when it spans whole rows) and from there to HBM by DMA.
// StagedReader overlaps those reads with the H2D copies: a pool of threads fills a ring of
// pinned slots in rectangle order while the caller issues the copies and releases slots
// once their copy has completed.
#pragma once

#include <stdint.h>

#include <atomic>
#include <condition_variable>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

namespace bwm {

struct Rect {
    int64_t r0, r1;   // rows (dates)
    int64_t c0, c1;   // pixels
    int64_t chunk;    // pipeline chunk the rectangle belongs to
    int64_t bytes() const { return (r1 - r0) * (c1 - c0) * 4; }
};

// Read-only view of a time-major float32 payload [n_obs][n_px] at byte `offset` of a file.
struct PayloadFile {
    int fd = -1;
    int64_t offset = 0;
    int64_t n_obs = 0;
    int64_t n_px = 0;
    // opens and checks that the file holds the whole payload; 0 or a negative BWM_E_* code
    int open(const char* path, int64_t offset, int64_t n_obs, int64_t n_px, std::string* err);
    void close();
    // rectangle -> dst [r1-r0][c1-c0] (contiguous); rows [r0, r1) split over `threads`
    int read_rect(const Rect& r, float* dst, int threads, std::string* err) const;
    ~PayloadFile() { close(); }
};

// A pageable host array [n_obs][ld] (a plain numpy stack): rectangles are memcpy'd into the
// pinned slots instead of being DMA'd from pageable memory through the driver's bounce buffer.
struct HostSource {
    const float* base = nullptr;
    int64_t ld = 0;
    void copy_rect(const Rect& r, float* dst) const;
};

// Rectangles of at most `slot_bytes` covering pixels [c0, c1) x all rows, whole rows first.
void plan_rects(int64_t n_obs, int64_t c0, int64_t c1, int64_t chunk, int64_t slot_bytes, std::vector<Rect>* out);

class StagedReader {
  public:
    // `slots` pinned buffers of `slot_bytes`; `threads` reader threads, each reading whole
    // rectangles.  Slots are allocated once and reused across calls.
    int ensure(int slots, int64_t slot_bytes, std::string* err);
    int start(const PayloadFile* f, const std::vector<Rect>* rects, int threads);
    int start(const HostSource* h, const std::vector<Rect>* rects, int threads);
    // blocks until rectangle g is in its slot; nullptr on a read error (see error()).
    const float* wait(int64_t g);
    // slot of rectangle g may be refilled (its H2D copy has completed)
    void release(int64_t g);
    void stop();                 // joins the threads (also on error paths)
    const std::string& error() const { return err_; }
    int slots() const { return (int)slot_.size(); }
    ~StagedReader();

  private:
    int launch(const std::vector<Rect>* rects, int threads);
    void worker();
    const PayloadFile* f_ = nullptr;
    const HostSource* h_ = nullptr;
    const std::vector<Rect>* rects_ = nullptr;
    std::vector<float*> slot_;
    int64_t slot_bytes_ = 0;
    std::vector<std::thread> pool_;
    std::atomic<int64_t> next_{0};
    std::mutex mu_;
    std::condition_variable cv_;
    std::vector<uint8_t> done_;
    int64_t released_ = 0;       // rectangles [0, released_) have been released (in order)
    bool abort_ = false;
    bool failed_ = false;
    std::string err_;
};

}  // namespace bwm
