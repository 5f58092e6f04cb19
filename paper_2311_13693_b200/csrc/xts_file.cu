// Out-of-core .xts block source: compress a tensor straight
// from its .xts file without ever holding it whole in host or device memory.
//
// Format (io.hpp:9-12, io.cpp:55-125): magic "XTSR", u16 version 1, u8 kind
// (0 dense tensor, 1 factor triple), u64 n1, n2, n3 (+ u64 rank for factors),
// u8 scalar width 8, then little-endian column-major doubles (A, B, C for
// factors). A dense payload is column-major, so every mode-3 slab k0..k1 is
// one contiguous byte range: a reader thread pread()s slabs into a ring of
// pinned host buffers while the plan streams the previous slab H2D, converts
// it and runs the tensor cores on it (Plan::compress's own double-buffered
// H2D pipeline). Header and truncation errors are the reference's DataError
// cases (io.cpp:94-125), raised before any device work.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <thread>

#include "common.cuh"
#include "plan.cuh"

namespace xtsg {

namespace {

struct XtsHeader {
  int kind = 0;
  uint64_t n[3] = {0, 0, 0};
  uint64_t rank = 0;
  int64_t payload = 0;  // byte offset of the first double
};

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) ::close(fd);
  }
};

void read_exact(int fd, void* dst, size_t bytes, int64_t off, const char* what) {
  auto* p = static_cast<char*>(dst);
  while (bytes) {
    const ssize_t r = ::pread(fd, p, bytes, off);
    if (r <= 0) data_error(what);
    p += r;
    off += r;
    bytes -= static_cast<size_t>(r);
  }
}

XtsHeader read_header(int fd, const std::string& path) {
  unsigned char h[43];
  struct stat sb {};
  if (::fstat(fd, &sb) != 0) data_error("cannot open: " + path);
  const int64_t size = sb.st_size;
  auto need = [&](int64_t n) {
    if (size < n) data_error("read_tensor_file: truncated file");
  };
  need(4);
  read_exact(fd, h, 4, 0, "read_tensor_file: truncated file");
  if (std::memcmp(h, "XTSR", 4) != 0) data_error("not a .xts file: " + path);
  need(7);
  read_exact(fd, h + 4, 3, 4, "read_tensor_file: truncated file");
  uint16_t version;
  std::memcpy(&version, h + 4, 2);
  if (version != 1) data_error("unsupported .xts version: " + path);
  XtsHeader x;
  x.kind = h[6];
  if (x.kind != 0 && x.kind != 1) data_error("unknown .xts kind: " + path);
  const int nfields = x.kind == 0 ? 3 : 4;
  need(7 + 8 * nfields + 1);
  read_exact(fd, h + 7, 8 * nfields + 1, 7, "read_tensor_file: truncated file");
  for (int m = 0; m < 3; ++m) std::memcpy(&x.n[m], h + 7 + 8 * m, 8);
  if (x.kind == 1) std::memcpy(&x.rank, h + 7 + 24, 8);
  if (h[7 + 8 * nfields] != 8) data_error("unsupported scalar width: " + path);
  x.payload = 7 + 8 * nfields + 1;
  const uint64_t count = x.kind == 0 ? x.n[0] * x.n[1] * x.n[2] : (x.n[0] + x.n[1] + x.n[2]) * x.rank;
  if (static_cast<uint64_t>(size - x.payload) < count * 8) data_error("read_tensor_file: truncated payload");
  return x;
}

// A ring of pinned slab buffers filled by one reader thread.
class SlabReader {
 public:
  SlabReader(int fd, int64_t payload, int64_t slab_bytes, int64_t nslabs, int64_t last_bytes, int depth)
      : fd_(fd), payload_(payload), slab_bytes_(slab_bytes), nslabs_(nslabs), last_bytes_(last_bytes),
        bufs_(depth, nullptr), ready_(depth, -1) {
    for (auto& b : bufs_) XCUDA(cudaHostAlloc(reinterpret_cast<void**>(&b), slab_bytes_, cudaHostAllocDefault));
    th_ = std::thread([this] { run(); });
  }
  ~SlabReader() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    if (th_.joinable()) th_.join();
    for (auto* b : bufs_)
      if (b) cudaFreeHost(b);
  }
  // Wait for slab s; returns its buffer (valid until release(s)).
  const char* acquire(int64_t s) {
    std::unique_lock<std::mutex> g(mu_);
    const int b = static_cast<int>(s % static_cast<int64_t>(bufs_.size()));
    cv_.wait(g, [&] { return ready_[b] == s || failed_; });
    if (failed_) data_error("read_tensor_file: truncated payload");
    return bufs_[b];
  }
  void release(int64_t s) {
    {
      std::lock_guard<std::mutex> g(mu_);
      ready_[s % static_cast<int64_t>(bufs_.size())] = -1;
      released_ = s + 1;
    }
    cv_.notify_all();
  }

 private:
  void run() {
    const int64_t depth = static_cast<int64_t>(bufs_.size());
    for (int64_t s = 0; s < nslabs_; ++s) {
      {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [&] { return stop_ || s - released_ < depth; });
        if (stop_) return;
      }
      const int b = static_cast<int>(s % depth);
      const int64_t bytes = s == nslabs_ - 1 ? last_bytes_ : slab_bytes_;
      char* p = bufs_[b];
      int64_t off = payload_ + s * slab_bytes_, left = bytes;
      bool ok = true;
      while (left > 0) {
        const ssize_t r = ::pread(fd_, p, static_cast<size_t>(left), off);
        if (r <= 0) {
          ok = false;
          break;
        }
        p += r;
        off += r;
        left -= r;
      }
      {
        std::lock_guard<std::mutex> g(mu_);
        if (!ok) failed_ = true;
        else ready_[b] = s;
      }
      cv_.notify_all();
      if (!ok) return;
    }
  }

  int fd_;
  int64_t payload_, slab_bytes_, nslabs_, last_bytes_;
  std::vector<char*> bufs_;
  std::vector<int64_t> ready_;
  int64_t released_ = 0;
  bool stop_ = false, failed_ = false;
  std::mutex mu_;
  std::condition_variable cv_;
  std::thread th_;
};

}  // namespace

}  // namespace xtsg

using namespace xtsg;

extern "C" {

int32_t xtsg_xts_header(const char* path, int32_t* kind, int64_t dims[3], int64_t* rank) {
  return guard([&] {
    if (!path) usage("xts_header: null path");
    Fd f;
    f.fd = ::open(path, O_RDONLY);
    if (f.fd < 0) data_error(std::string("cannot open: ") + path);
    const XtsHeader h = read_header(f.fd, path);
    if (kind) *kind = h.kind;
    if (dims)
      for (int m = 0; m < 3; ++m) dims[m] = static_cast<int64_t>(h.n[m]);
    if (rank) *rank = static_cast<int64_t>(h.rank);
  });
}

int32_t xtsg_plan_compress_file(xtsg_plan* plan, const char* path, int64_t slab_bytes, void* y,
                                int32_t accumulate, void* stream) {
  return guard([&] {
    if (!path) usage("plan_compress_file: null path");
    Plan* p = reinterpret_cast<Plan*>(plan);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : thread_stream();
    PlanUse use(p, s);
    Fd f;
    f.fd = ::open(path, O_RDONLY);
    if (f.fd < 0) data_error(std::string("cannot open: ") + path);
    const XtsHeader h = read_header(f.fd, path);
    for (int m = 0; m < 3; ++m)
      if (static_cast<int64_t>(h.n[m]) != p->desc.dims[m])
        usage("plan_compress_file: file dims differ from the plan's tensor dims");
    if (h.kind == 1) {
      // factor triple: read A, B, C (small) and generate the slabs on the device
      const int64_t r = static_cast<int64_t>(h.rank);
      std::vector<double> a(h.n[0] * h.rank), b(h.n[1] * h.rank), c(h.n[2] * h.rank);
      int64_t off = h.payload;
      for (auto* v : {&a, &b, &c}) {
        read_exact(f.fd, v->data(), v->size() * 8, off, "read_tensor_file: truncated payload");
        off += static_cast<int64_t>(v->size() * 8);
      }
      if (!p->tensor_core())
        usage("plan_compress_file: factor files need a bf16/fp16 plan (xtsg_plan_compress_factors)");
      p->compress_factors(a.data(), b.data(), c.data(), r, 0, p->desc.dims[2], static_cast<float*>(y),
                          accumulate != 0, s);
      return;
    }
    const int64_t n1 = p->desc.dims[0], n2 = p->desc.dims[1], n3 = p->desc.dims[2];
    const int64_t slice = n1 * n2 * 8;
    const int64_t want = slab_bytes > 0 ? slab_bytes : (int64_t(512) << 20);
    const int64_t ks = std::max<int64_t>(1, std::min<int64_t>(n3, want / slice));
    const int64_t nslabs = ceil_div(n3, ks);
    const int64_t last = (n3 - (nslabs - 1) * ks) * slice;
    SlabReader rd(f.fd, h.payload, ks * slice, nslabs, last, 3);
    const int64_t ld[2] = {n1, n1 * n2};
    for (int64_t sl = 0; sl < nslabs; ++sl) {
      const char* buf = rd.acquire(sl);
      const int64_t k0 = sl * ks, kn = std::min(ks, n3 - k0);
      const int64_t off[3] = {0, 0, k0}, ext[3] = {n1, n2, kn};
      // returns once the slab's device work is done (host input), so the
      // buffer can go back to the reader
      p->compress(buf, XTSG_DTYPE_F64, ld, off, ext, y, accumulate != 0 || sl > 0, s);
      XCUDA(cudaStreamSynchronize(s));
      rd.release(sl);
    }
  });
}

}  // extern "C"
