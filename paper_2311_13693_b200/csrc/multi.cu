// Multi-GPU compression behind the C ABI (SURVEY §8 e, BASELINE north_star:
// "partitioned across the 8 GPUs of a single box by tensor slab along mode 3,
// each GPU compressing its slab into partial replicas and one NCCL reduce over
// NVLink of the small P*L*M*N result").
//
// The reference has no multi-GPU entry point: its caller compresses with
// comp_blocked / comp_from_factors on one host (pipeline.cpp:386-405). An
// xtsg_multi owns one plan per GPU of the node (the same ensemble, generated
// on every GPU from the seed: the RNG is counter based, so no ensemble bytes
// move), one persistent host worker thread per GPU (the plans and their
// streams live on it), and one NCCL communicator clique (ncclCommInitAll:
// single process, all GPUs). A call splits the tensor into contiguous mode-3
// slabs, every worker compresses its slab into a device partial, and one
// grouped ncclReduce (sum, fp32) lands the replicas on the first GPU.
//
// NCCL is resolved at run time (dlopen "libnccl.so.2"): inside a PyTorch
// process that is torch's own NCCL, elsewhere the system one; libxtsg does
// not link it, so loading the library never pins an NCCL version.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <condition_variable>
#include <deque>
#include <exception>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"
#include "plan.cuh"

namespace xtsg {

namespace {

struct NcclApi {
  ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                         cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  ncclResult_t (*get_version)(int*) = nullptr;
  bool ok = false;
  std::string why;
};

const NcclApi& nccl() {
  static const NcclApi api = [] {
    NcclApi a;
    // an NCCL already in the process (e.g. torch's) wins; XTSG_NCCL_LIB names
    // a specific library; else the loader's libnccl.so.2
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    const char* env = std::getenv("XTSG_NCCL_LIB");
    if (!h && env && *env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return a;
    }
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn) a.why = std::string("NCCL symbol missing: ") + name;
      return fn != nullptr;
    };
    a.ok = sym(a.comm_init_all, "ncclCommInitAll") && sym(a.comm_destroy, "ncclCommDestroy") &&
           sym(a.reduce, "ncclReduce") && sym(a.group_start, "ncclGroupStart") &&
           sym(a.group_end, "ncclGroupEnd") && sym(a.error_string, "ncclGetErrorString") &&
           sym(a.get_version, "ncclGetVersion");
    return a;
  }();
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw Status(XTSG_E_CUDA, std::string(what) + ": " + nccl().error_string(r));
}

// A host thread bound to one GPU running submitted jobs in order.
class Worker {
 public:
  explicit Worker(int dev) : dev_(dev), th_([this] { loop(); }) {}
  ~Worker() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    th_.join();
  }
  // run fn on the worker; returns when done, rethrowing its exception
  void run(const std::function<void()>& fn) { wait(submit(fn)); }
  size_t submit(const std::function<void()>& fn) {
    std::lock_guard<std::mutex> lk(mu_);
    q_.push_back(fn);
    cv_.notify_all();
    return ++submitted_;
  }
  void wait(size_t ticket) {
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return finished_ >= ticket; });
    if (err_) {
      std::exception_ptr e = err_;
      err_ = nullptr;
      std::rethrow_exception(e);
    }
  }

 private:
  void loop() {
    cudaSetDevice(dev_);
    for (;;) {
      std::function<void()> fn;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || !q_.empty(); });
        if (q_.empty()) return;
        fn = std::move(q_.front());
        q_.pop_front();
      }
      std::exception_ptr e;
      try {
        fn();
      } catch (...) {
        e = std::current_exception();
      }
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (e && !err_) err_ = e;
        ++finished_;
      }
      done_cv_.notify_all();
    }
  }
  int dev_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  std::deque<std::function<void()>> q_;
  size_t submitted_ = 0, finished_ = 0;
  bool stop_ = false;
  std::exception_ptr err_;
  std::thread th_;
};

__global__ void add_f32_kernel(const float* __restrict__ s, int64_t n, float* __restrict__ d) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    d[e] += s[e];
}

}  // namespace

struct Multi {
  xtsg_plan_desc desc{};
  int n = 0;
  std::vector<int> dev;
  std::vector<std::unique_ptr<Worker>> workers;
  std::vector<xtsg_plan*> plans;
  std::vector<cudaStream_t> streams;
  std::vector<float*> ybuf;  // per-GPU partial replicas (fp32, P*L*M*N)
  std::vector<cudaEvent_t> ev0, ev1;
  std::vector<ncclComm_t> comms;
  int64_t ysz = 0;
  double last_ms = 0.0;
  std::mutex mu;

  // every GPU's partial replicas for its mode-3 slab, one grouped reduce to
  // GPU 0, then y (host or GPU-0 memory) = / += the sum
  void run(const std::function<void(int g, int64_t k0, int64_t k1)>& slab, void* y, bool accumulate) {
    const int64_t K = desc.dims[2];
    run_parts([&](int g) {
      const int64_t k0 = K * g / n, k1 = K * (g + 1) / n;
      if (k1 > k0) slab(g, k0, k1);
      else XCUDA(cudaMemsetAsync(ybuf[g], 0, sizeof(float) * ysz, streams[g]));
    }, y, accumulate);
  }

  // part(g) runs on GPU g's worker and must leave GPU g's complete partial
  // replicas in ybuf[g] (on streams[g])
  void run_parts(const std::function<void(int g)>& part, void* y, bool accumulate) {
    std::lock_guard<std::mutex> lk(mu);
    int caller_dev = 0;
    XCUDA(cudaGetDevice(&caller_dev));
    struct Restore {
      int d;
      ~Restore() { cudaSetDevice(d); }
    } restore{caller_dev};
    std::vector<size_t> tickets(n);
    for (int g = 0; g < n; ++g) {
      tickets[g] = workers[g]->submit([=, &part] {
        XCUDA(cudaEventRecord(ev0[g], streams[g]));
        part(g);
      });
    }
    std::exception_ptr first;
    for (int g = 0; g < n; ++g) {
      try {
        workers[g]->wait(tickets[g]);
      } catch (...) {
        if (!first) first = std::current_exception();
      }
    }
    if (first) std::rethrow_exception(first);
    // one NCCL reduce (sum) of the P*L*M*N partials onto GPU 0, issued as a
    // group from this thread (single-process clique)
    if (!comms.empty()) {
      nccl_check(nccl().group_start(), "ncclGroupStart");
      for (int g = 0; g < n; ++g) {
        XCUDA(cudaSetDevice(dev[g]));
        nccl_check(nccl().reduce(ybuf[g], ybuf[g], static_cast<size_t>(ysz), ncclFloat32, ncclSum, 0, comms[g],
                                 streams[g]),
                   "ncclReduce");
      }
      nccl_check(nccl().group_end(), "ncclGroupEnd");
    }
    for (int g = 0; g < n; ++g) {
      XCUDA(cudaSetDevice(dev[g]));
      XCUDA(cudaEventRecord(ev1[g], streams[g]));
    }
    // result to the caller on GPU 0's stream
    workers[0]->run([&] {
      cudaStream_t s = streams[0];
      OutView<float> yo(static_cast<float*>(y), static_cast<size_t>(ysz), s);
      if (accumulate) {
        if (yo.host) XCUDA(cudaMemcpyAsync(yo.dev, y, sizeof(float) * ysz, cudaMemcpyHostToDevice, s));
        add_f32_kernel<<<static_cast<int>(std::min<int64_t>(ceil_div(ysz, 256), 148 * 16)), 256, 0, s>>>(
            ybuf[0], ysz, yo.dev);
        XLAUNCH_CHECK();
      } else {
        XCUDA(cudaMemcpyAsync(yo.dev, ybuf[0], sizeof(float) * ysz, cudaMemcpyDeviceToDevice, s));
      }
      yo.finish();
      XCUDA(cudaStreamSynchronize(s));
    });
    double mx = 0.0;
    for (int g = 0; g < n; ++g) {
      XCUDA(cudaSetDevice(dev[g]));
      XCUDA(cudaEventSynchronize(ev1[g]));
      float ms = 0.f;
      XCUDA(cudaEventElapsedTime(&ms, ev0[g], ev1[g]));
      mx = std::max(mx, static_cast<double>(ms));
    }
    last_ms = mx;
  }

  ~Multi() {
    for (int g = 0; g < n && g < static_cast<int>(workers.size()); ++g) {
      if (!workers[g]) continue;
      try {
        workers[g]->run([&, g] {
          if (g < static_cast<int>(plans.size()) && plans[g]) xtsg_plan_destroy(plans[g]);
          if (g < static_cast<int>(ybuf.size()) && ybuf[g]) cudaFree(ybuf[g]);
          if (g < static_cast<int>(ev0.size()) && ev0[g]) cudaEventDestroy(ev0[g]);
          if (g < static_cast<int>(ev1.size()) && ev1[g]) cudaEventDestroy(ev1[g]);
          if (g < static_cast<int>(streams.size()) && streams[g]) cudaStreamDestroy(streams[g]);
        });
      } catch (...) {
      }
    }
    for (auto c : comms)
      if (c) nccl().comm_destroy(c);
  }
};

// ---- sparse input across the GPUs ---------------------------------------
// Eq. 3 is linear in the nonzeros, so any partition of them compresses to
// partial replicas that sum to the whole. COO: GPU g takes the contiguous
// nonzero range [nnz*g/G, nnz*(g+1)/G) (a k-range when the stream is k-sorted,
// as CSF producers and the reference's slab writers emit it; no host pass).
// CSF: GPU g takes a contiguous slice range holding ~1/G of the nonzeros (a
// k-range for k-sorted slices), its pointers rebased on the worker thread.
// Every GPU's share is further cut into device calls of at most
// XTSG_SPARSE_CHUNK nonzeros (default 2^31: one plan call's sort keys and
// tile lists stay within 32-bit counts), accumulated in its partial.

int64_t sparse_chunk() {
  const char* e = std::getenv("XTSG_SPARSE_CHUNK");
  const long long v = e ? std::atoll(e) : 0;
  return v > 0 ? static_cast<int64_t>(v) : (int64_t(1) << 31);
}

void require_host(const void* p, const char* what) {
  if (p && is_device_ptr(p))
    usage(std::string(what) + ": sparse inputs of a multi-GPU call must be host memory");
}

// CSF slice boundaries: first nonzero of slice q (pointers clamped so that a
// malformed input only misplaces a split; every part is validated on its GPU)
struct CsfIndex {
  int64_t n_slices, n_fibers, nnz;
  const int64_t* slice_ptr;
  const int64_t* fiber_ptr;
  int64_t fib(int64_t q) const { return std::min(std::max<int64_t>(slice_ptr[q], 0), n_fibers); }
  int64_t nz(int64_t f) const { return std::min(std::max<int64_t>(fiber_ptr[f], 0), nnz); }
  int64_t start(int64_t q) const { return nz(fib(q)); }
  // smallest q in [lo, hi] with start(q) >= target (start is monotone for valid input)
  int64_t lower(int64_t lo, int64_t hi, int64_t target) const {
    while (lo < hi) {
      const int64_t mid = lo + (hi - lo) / 2;
      if (start(mid) < target) lo = mid + 1;
      else hi = mid;
    }
    return lo;
  }
};

}  // namespace xtsg

using namespace xtsg;

extern "C" {

int32_t xtsg_multi_create(const xtsg_plan_desc* desc, int32_t ngpus, const int32_t* gpus, xtsg_multi** out) {
  return guard([&] {
    *out = nullptr;
    if (!desc) usage("multi_create: null descriptor");
    if (ngpus < 1) usage("multi_create: need at least one GPU");
    if (desc->precision == XTSG_PREC_FP64) usage("multi_create: needs a tensor-core precision (bf16/fp16/fp16x3)");
    require_device();
    int count = 0;
    XCUDA(cudaGetDeviceCount(&count));
    std::vector<int> devs(static_cast<size_t>(ngpus));
    for (int g = 0; g < ngpus; ++g) {
      devs[g] = gpus ? gpus[g] : g;
      if (devs[g] < 0 || devs[g] >= count) usage("multi_create: GPU index out of range");
      for (int h = 0; h < g; ++h)
        if (devs[h] == devs[g]) usage("multi_create: every GPU may appear once");
    }
    auto m = std::make_unique<Multi>();
    m->desc = *desc;
    m->n = ngpus;
    m->dev = devs;
    m->ysz = desc->count * desc->reduced[0] * desc->reduced[1] * desc->reduced[2];
    m->plans.assign(ngpus, nullptr);
    m->streams.assign(ngpus, nullptr);
    m->ybuf.assign(ngpus, nullptr);
    m->ev0.assign(ngpus, nullptr);
    m->ev1.assign(ngpus, nullptr);
    for (int g = 0; g < ngpus; ++g) m->workers.push_back(std::make_unique<Worker>(devs[g]));
    // plans, streams and partial buffers on every GPU at once
    std::vector<size_t> t(ngpus);
    Multi* mp = m.get();
    for (int g = 0; g < ngpus; ++g)
      t[g] = m->workers[g]->submit([mp, g] {
        XCUDA(cudaStreamCreateWithFlags(&mp->streams[g], cudaStreamNonBlocking));
        XCUDA(cudaEventCreate(&mp->ev0[g]));
        XCUDA(cudaEventCreate(&mp->ev1[g]));
        XCUDA(cudaMalloc(&mp->ybuf[g], sizeof(float) * mp->ysz));
        const int32_t rc = xtsg_plan_create(&mp->desc, &mp->plans[g]);
        if (rc != XTSG_OK) throw Status(rc, std::string("multi_create: plan on GPU: ") + xtsg_last_error());
      });
    std::exception_ptr first;
    for (int g = 0; g < ngpus; ++g) {
      try {
        m->workers[g]->wait(t[g]);
      } catch (...) {
        if (!first) first = std::current_exception();
      }
    }
    if (first) std::rethrow_exception(first);
    // the reduce runs through NCCL for any GPU count when NCCL loads (a
    // one-GPU clique reduces to a copy, which keeps this path testable on one
    // GPU); more than one GPU requires it
    if (ngpus > 1 || nccl().ok) {
      if (!nccl().ok) throw Status(XTSG_E_CUDA, "multi_create: " + nccl().why);
      m->comms.assign(ngpus, nullptr);
      nccl_check(nccl().comm_init_all(m->comms.data(), ngpus, m->dev.data()), "ncclCommInitAll");
    }
    *out = reinterpret_cast<xtsg_multi*>(m.release());
  });
}

void xtsg_multi_destroy(xtsg_multi* m) { delete reinterpret_cast<Multi*>(m); }

int32_t xtsg_multi_compress_factors(xtsg_multi* mh, const double* a, const double* b, const double* c,
                                    int64_t rank, void* y, int32_t accumulate) {
  return guard([&] {
    Multi* m = reinterpret_cast<Multi*>(mh);
    m->run([&](int g, int64_t k0, int64_t k1) {
      const int32_t rc = xtsg_plan_compress_factors(m->plans[g], a, b, c, rank, k0, k1, m->ybuf[g], 0,
                                                    m->streams[g]);
      if (rc != XTSG_OK) throw Status(rc, xtsg_last_error(), xtsg_last_payload(0), xtsg_last_payload(1));
    }, y, accumulate != 0);
  });
}

int32_t xtsg_multi_compress(xtsg_multi* mh, const void* x, int32_t x_dtype, const int64_t ld[2], void* y,
                            int32_t accumulate) {
  return guard([&] {
    Multi* m = reinterpret_cast<Multi*>(mh);
    if (!x || !ld) usage("multi_compress: null input");
    size_t es = 0;
    switch (x_dtype) {
      case XTSG_DTYPE_BF16: case XTSG_DTYPE_F16: es = 2; break;
      case XTSG_DTYPE_F32: es = 4; break;
      case XTSG_DTYPE_F64: es = 8; break;
      default: usage("multi_compress: unknown x dtype");
    }
    const int64_t I = m->desc.dims[0], J = m->desc.dims[1];
    m->run([&](int g, int64_t k0, int64_t k1) {
      const int64_t off[3] = {0, 0, k0}, ext[3] = {I, J, k1 - k0};
      const void* xs = static_cast<const uint8_t*>(x) + static_cast<size_t>(k0 * ld[1]) * es;
      const int32_t rc = xtsg_plan_compress(m->plans[g], xs, x_dtype, ld, off, ext, m->ybuf[g], 0, m->streams[g]);
      if (rc != XTSG_OK) throw Status(rc, xtsg_last_error(), xtsg_last_payload(0), xtsg_last_payload(1));
    }, y, accumulate != 0);
  });
}

int32_t xtsg_multi_compress_coo(xtsg_multi* mh, const int32_t* i, const int32_t* j, const int32_t* k,
                                const float* val, int64_t nnz, void* y, int32_t accumulate) {
  return guard([&] {
    Multi* m = reinterpret_cast<Multi*>(mh);
    if (nnz < 0) usage("multi_compress_coo: negative nnz");
    if (nnz > 0 && (!i || !j || !k || !val)) usage("multi_compress_coo: null input");
    for (const void* p : {static_cast<const void*>(i), static_cast<const void*>(j), static_cast<const void*>(k),
                          static_cast<const void*>(val)})
      require_host(p, "multi_compress_coo");
    const int64_t chunk = sparse_chunk();
    m->run_parts([&](int g) {
      const int64_t e0 = nnz * g / m->n, e1 = nnz * (g + 1) / m->n;
      if (e1 <= e0) {
        XCUDA(cudaMemsetAsync(m->ybuf[g], 0, sizeof(float) * m->ysz, m->streams[g]));
        return;
      }
      for (int64_t a = e0; a < e1; a += chunk) {
        const int64_t b = std::min(e1, a + chunk);
        const int32_t rc = xtsg_plan_compress_coo(m->plans[g], i + a, j + a, k + a, val + a, b - a, m->ybuf[g],
                                                  a > e0 ? 1 : 0, m->streams[g]);
        if (rc != XTSG_OK) throw Status(rc, xtsg_last_error(), xtsg_last_payload(0), xtsg_last_payload(1));
      }
    }, y, accumulate != 0);
  });
}

int32_t xtsg_multi_compress_csf(xtsg_multi* mh, int64_t n_slices, const int32_t* slice_k, const int64_t* slice_ptr,
                                int64_t n_fibers, const int32_t* fiber_j, const int64_t* fiber_ptr, int64_t nnz,
                                const int32_t* nz_i, const float* val, void* y, int32_t accumulate) {
  return guard([&] {
    Multi* m = reinterpret_cast<Multi*>(mh);
    if (n_slices < 0 || n_fibers < 0 || nnz < 0) usage("multi_compress_csf: negative size");
    if (!slice_ptr || !fiber_ptr || (n_slices > 0 && !slice_k) || (n_fibers > 0 && !fiber_j) ||
        (nnz > 0 && (!nz_i || !val)))
      usage("multi_compress_csf: null input");
    for (const void* p : {static_cast<const void*>(slice_k), static_cast<const void*>(slice_ptr),
                          static_cast<const void*>(fiber_j), static_cast<const void*>(fiber_ptr),
                          static_cast<const void*>(nz_i), static_cast<const void*>(val)})
      require_host(p, "multi_compress_csf");
    const CsfIndex ix{n_slices, n_fibers, nnz, slice_ptr, fiber_ptr};
    // GPU g: slices [qs[g], qs[g+1]), ~1/G of the nonzeros each
    const int G = m->n;
    std::vector<int64_t> qs(static_cast<size_t>(G) + 1, 0);
    qs[G] = n_slices;
    if (n_slices > 0) {
      const int64_t E0 = ix.start(0), E1 = std::max(E0, ix.start(n_slices));
      for (int g = 1; g < G; ++g)
        qs[g] = std::max(qs[g - 1], ix.lower(0, n_slices, E0 + (E1 - E0) * g / G));
    }
    const int64_t chunk = sparse_chunk();
    m->run_parts([&](int g) {
      bool first = true;
      std::vector<int64_t> lsp, lfp;
      for (int64_t qa = qs[g]; qa < qs[g + 1];) {
        // extend the part while it holds at most `chunk` nonzeros (at least one slice)
        int64_t qb = ix.lower(qa + 1, qs[g + 1], ix.start(qa) + chunk + 1);
        if (qb > qa + 1 && ix.start(qb) - ix.start(qa) > chunk) --qb;
        qb = std::max(qb, qa + 1);
        const int64_t f0 = ix.fib(qa), f1 = std::max(f0, ix.fib(qb));
        const int64_t e0 = ix.nz(f0), e1 = std::max(e0, ix.nz(f1));
        lsp.resize(static_cast<size_t>(qb - qa) + 1);
        for (int64_t t = 0; t <= qb - qa; ++t) lsp[t] = slice_ptr[qa + t] - f0;
        lfp.resize(static_cast<size_t>(f1 - f0) + 1);
        for (int64_t t = 0; t <= f1 - f0; ++t) lfp[t] = fiber_ptr[f0 + t] - e0;
        const int32_t rc = xtsg_plan_compress_csf(m->plans[g], qb - qa, slice_k + qa, lsp.data(), f1 - f0,
                                                  fiber_j + f0, lfp.data(), e1 - e0, nz_i + e0, val + e0,
                                                  m->ybuf[g], first ? 0 : 1, m->streams[g]);
        if (rc != XTSG_OK) throw Status(rc, xtsg_last_error(), xtsg_last_payload(0), xtsg_last_payload(1));
        first = false;
        qa = qb;
      }
      if (first) XCUDA(cudaMemsetAsync(m->ybuf[g], 0, sizeof(float) * m->ysz, m->streams[g]));
    }, y, accumulate != 0);
  });
}

int32_t xtsg_multi_last_ms(xtsg_multi* mh, double* ms) {
  return guard([&] {
    Multi* m = reinterpret_cast<Multi*>(mh);
    std::lock_guard<std::mutex> lk(m->mu);
    *ms = m->last_ms;
  });
}

int32_t xtsg_nccl_version(int32_t* version) {
  return guard([&] {
    if (!nccl().ok) throw Status(XTSG_E_CUDA, nccl().why);
    int v = 0;
    nccl_check(nccl().get_version(&v), "ncclGetVersion");
    *version = v;
  });
}

}  // extern "C"
