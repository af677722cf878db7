// Shared infrastructure of the T^2S^2 B200 engine: error handling, the
// device tensor type, and the per-context stream/allocator.
//
// Everything numeric is fp64 and device resident.  Shapes are host-known:
// the engine reads back the few integers that decide bond ranks (SVD
// truncation, enrichment) and keeps every core, interface and local system
// in HBM (or L2) between kernels.
#pragma once

#include <initializer_list>
#include <utility>

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

namespace t2s2 {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

enum ErrCode {
  kOk = 0,
  kErrArg = 1,
  kErrCuda = 2,
  kErrShape = 3,
  kErrValue = 4,
  kErrStagnation = 5,
  kErrCapacity = 6,
};

#define T2S2_CUDA(call)                                                       \
  do {                                                                        \
    cudaError_t e_ = (call);                                                  \
    if (e_ != cudaSuccess)                                                    \
      throw ::t2s2::Error(::t2s2::kErrCuda,                                   \
                          std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define T2S2_CHECK_LAUNCH() T2S2_CUDA(cudaGetLastError())

#define T2S2_REQUIRE(cond, code, msg)                  \
  do {                                                 \
    if (!(cond)) throw ::t2s2::Error((code), (msg));   \
  } while (0)

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

// Device allocation for one stream: a host-side caching allocator (size
// classes of powers of two) over cudaMallocAsync.  All work of a context is
// ordered on its stream, so a block released after its last use was
// enqueued can be handed to the next request immediately — no driver call on
// the hot path.
struct Allocator {
  cudaStream_t stream = nullptr;
  std::unordered_map<size_t, std::vector<double*>> free_lists;
  std::unordered_map<double*, size_t> live;
  static size_t size_class(size_t n) {
    size_t c = 32;
    while (c < n) c <<= 1;
    return c;
  }
  double* alloc(size_t n) {
    if (n == 0) n = 1;
    const size_t c = size_class(n);
    auto& fl = free_lists[c];
    double* p = nullptr;
    if (!fl.empty()) {
      p = fl.back();
      fl.pop_back();
    } else {
      void* v = nullptr;
      T2S2_CUDA(cudaMallocAsync(&v, c * sizeof(double), stream));
      p = static_cast<double*>(v);
    }
    live[p] = c;
    return p;
  }
  void release(double* p) {
    if (!p) return;
    auto it = live.find(p);
    if (it == live.end()) return;
    free_lists[it->second].push_back(p);
    live.erase(it);
  }
  void trim() {  // return cached blocks to the driver pool
    for (auto& kv : free_lists)
      for (double* p : kv.second) cudaFreeAsync(p, stream);
    free_lists.clear();
  }
};

// Launch accounting (per context).  Every kernel launch sits inside a
// LaunchScope naming its family and the algorithmic flops/bytes of that
// launch; counts are always kept, CUDA-event timings only while profiling
// is switched on (t2s2_stats_reset(ctx, 1)).
struct LaunchScope {
  int slot = -1;
  LaunchScope(const char* family, double flops = 0.0, double bytes = 0.0);
  ~LaunchScope();
};

// Work of the most recent launch of a family that was not known when it was
// enqueued (a device-side loop): added to the family and to that launch's record.
void amend_work(const char* family, double flops, double bytes);

Allocator& allocator();  // the current context's allocator
// Per-device launch properties, cached in the current context (one context
// per host thread and device, so no shared mutable state between threads):
int num_sms();                                          // multiprocessors of the device / partition
bool on_partition();                                    // the context runs on an SM partition
void max_dynamic_smem(const void* kernel, int bytes);   // raise the kernel's dynamic smem limit
int occupancy(const void* kernel, int threads, int smem);  // resident CTAs per SM (>= 1)
int sm_budget();         // CTAs a whole-GPU cooperative kernel may use (context setting)
cudaStream_t stream();   // the current context's stream
bool profiling();        // per-launch CUDA-event timing switched on (t2s2_stats_reset)

// Every device->host read that steers the host (ranks, candidate scores,
// residuals, solver flags) goes through host_read: copy + synchronise.  A
// context can record the values of a run and hand them back, without
// synchronising, to an identical run (t2s2_read_trace): the measurement of
// what the synchronising reads cost.
void host_read(void* host, const void* dev, size_t bytes);
// n zeroed 32-bit device words that stay untouched by anyone else until the
// context's pool of them has been handed out once (65536 words): arrival
// counters of one kernel launch, no memset per launch
unsigned* zero_words(size_t n);
// A steering read published by its producer: read_open reserves the mapped
// host buffer and the next ticket; the LAST kernel that computes the values
// copies them there itself (publish_words: one CTA, after the values are
// visible to it) instead of a separate publish launch; read_close waits for
// the ticket and hands the bytes to the host (and to the read trace).
// Nothing else may read between open and close.  While a trace is replayed
// the ticket is empty (dst == null): kernels publish nothing and read_close
// returns the recorded values.
struct ReadTicket {
  unsigned* dst = nullptr;   // mapped host buffer (device-visible)
  unsigned* flag = nullptr;  // ticket word behind it
  unsigned value = 0;
};
ReadTicket read_open(size_t bytes);
void read_publish(const void* dev, size_t bytes, const ReadTicket& t);  // a separate publish launch
void read_close(void* host, size_t bytes, const ReadTicket& t);
// up to four device segments (pointer, doubles) read back as one array with one kernel
void host_read_gather(double* host, std::initializer_list<std::pair<const double*, size_t>> parts);
#ifdef __CUDACC__
// every thread of ONE CTA, once the n words at src are visible to that CTA
__device__ __forceinline__ void publish_words(const ReadTicket& t, const unsigned* src, int n) {
  if (!t.dst) return;
  for (int i = threadIdx.x; i < n; i += blockDim.x) t.dst[i] = __ldcg(src + i);
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) *(volatile unsigned*)t.flag = t.value;
}
#endif
bool replaying_reads();  // host_read returns recorded values, nothing synchronises
// Determinism probe: while a trace is recorded (mode 1) or compared (mode 3)
// the tagged device buffer joins the trace like a host read; otherwise a no-op.
void trace_buffer(const char* tag, const double* dev, size_t n);

// A dense row-major device array with a host-known shape.  Owns its
// buffer (move-only).
struct DTensor {
  double* p = nullptr;
  std::vector<int> shape;

  DTensor() = default;
  explicit DTensor(std::vector<int> s) : shape(std::move(s)) { p = allocator().alloc(size()); }
  DTensor(const DTensor&) = delete;
  DTensor& operator=(const DTensor&) = delete;
  DTensor(DTensor&& o) noexcept : p(o.p), shape(std::move(o.shape)) { o.p = nullptr; }
  DTensor& operator=(DTensor&& o) noexcept {
    if (this != &o) {
      allocator().release(p);
      p = o.p;
      shape = std::move(o.shape);
      o.p = nullptr;
    }
    return *this;
  }
  ~DTensor() { allocator().release(p); }

  size_t size() const {
    size_t n = 1;
    for (int s : shape) n *= (size_t)s;
    return n;
  }
  int ndim() const { return (int)shape.size(); }
  int dim(int i) const { return shape[i < 0 ? shape.size() + i : i]; }
  // reshape in place (same element count)
  DTensor& view(std::vector<int> s) {
    size_t n = 1;
    for (int v : s) n *= (size_t)v;
    T2S2_REQUIRE(n == size(), kErrShape, "view: element count mismatch");
    shape = std::move(s);
    return *this;
  }
  DTensor clone() const;
};

// A train: d cores.  Vector cores are (r0, n, r1); operator cores are
// (r0, m, n, r1).  Rows/cols record the mode sizes.
struct Train {
  std::vector<DTensor> cores;
  std::vector<int> rows, cols;  // cols empty for vectors
  bool is_op() const { return !cols.empty(); }
  int d() const { return (int)cores.size(); }
  int rank(int l) const {  // bond l in 0..d
    if (l == 0) return 1;
    return cores[l - 1].dim(-1);
  }
  std::vector<int> ranks() const {
    std::vector<int> r(d() + 1);
    for (int l = 0; l <= d(); ++l) r[l] = rank(l);
    return r;
  }
  int max_rank() const {
    int m = 1;
    for (int l = 0; l <= d(); ++l) m = rank(l) > m ? rank(l) : m;
    return m;
  }
  Train clone() const;
  // The solver's (m, A, a, n) layout of an operator's cores (als.cu), kept
  // with the train so that a march permutes its left operator once, not once
  // per step; valid while layout_of[l] == cores[l].p (trains are not edited
  // in place).  Not copied by clone().
  mutable std::vector<DTensor> solver_layout;
  mutable std::vector<const double*> layout_of;
};

}  // namespace t2s2
