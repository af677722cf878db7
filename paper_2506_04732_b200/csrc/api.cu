// C ABI of the engine (include/t2s2.h): context management, train
// upload/download and the hot-path entry points.
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <unordered_map>

#include "../../include/t2s2.h"
#include "als.h"
#include "blas.h"
#include "linalg.h"
#include "partition.h"
#include "tt.h"

namespace t2s2 {
struct FamilyStat {
  std::string name;
  long long launches = 0;
  double flops = 0.0, bytes = 0.0, ms = 0.0;
};
struct Pending {
  int fam;
  double flops, bytes;
  cudaEvent_t a, b;
};
}  // namespace t2s2

struct t2s2_context {
  int device = 0;
  void* cu_ctx = nullptr;  // green context of an SM partition (null: the primary context)
  int sms = 0;        // multiprocessor count of the device
  int sm_budget = 0;  // 0: all SMs
  std::unordered_map<const void*, int> smem_limit;  // kernel -> raised dynamic smem bytes
  std::unordered_map<std::string, int> occ_cache;   // kernel/threads/smem -> CTAs per SM
  cudaStream_t stream = nullptr;
  t2s2::Allocator alloc;
  std::string last_error;
  // launch accounting
  std::vector<t2s2::FamilyStat> fams;
  std::unordered_map<std::string, int> fam_index;
  std::unordered_map<const char*, int> fam_by_ptr;  // call-site literal -> family
  bool profiling = false;
  std::vector<cudaEvent_t> event_pool;
  size_t pool_used = 0;
  std::vector<t2s2::Pending> pending;
  std::vector<t2s2_launch_record> launch_log;  // per launch while profiling
  // pinned staging buffer of host_read: a device->host copy into pinned
  // memory is one DMA, into pageable memory a staged copy with a driver-side
  // wait (measured per read in DESIGN.md section 8)
  void* pinned = nullptr;
  static constexpr size_t kPinnedBytes = 64 * 1024;
  unsigned read_ticket = 0;  // last ticket published into the word after the staging buffer
  // zeroed device words for the counters of hand-off kernels (zero_words)
  unsigned* zero_pool = nullptr;
  size_t zero_cursor = 0;
  static constexpr size_t kZeroWords = 1 << 16;
  // host_read trace: 0 off, 1 record, 2 replay
  int trace_mode = 0;
  std::vector<std::vector<unsigned char>> trace;
  size_t trace_pos = 0;
  int trace_diff = -1;  // mode 3: index of the first differing read
};

struct t2s2_train {
  t2s2_context* ctx = nullptr;  // owner: buffers are freed on its stream
  t2s2::Train t;
};

namespace t2s2 {
namespace {
thread_local t2s2_context* g_ctx = nullptr;

struct Bind {  // makes ctx current for the duration of an API call
  t2s2_context* prev;
  explicit Bind(t2s2_context* c) : prev(g_ctx) {
    g_ctx = c;
    if (c->cu_ctx)
      set_current_context(c->cu_ctx);
    else
      cudaSetDevice(c->device);
  }
  ~Bind() { g_ctx = prev; }
};
}  // namespace

Allocator& allocator() { return g_ctx->alloc; }
int num_sms() { return g_ctx->sms; }
bool on_partition() { return g_ctx->cu_ctx != nullptr; }

void max_dynamic_smem(const void* kernel, int bytes) {
  auto it = g_ctx->smem_limit.find(kernel);
  if (it != g_ctx->smem_limit.end() && it->second >= bytes) return;
  T2S2_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  g_ctx->smem_limit[kernel] = bytes;
}

int occupancy(const void* kernel, int threads, int smem) {
  char key[64];
  snprintf(key, sizeof key, "%p/%d/%d", kernel, threads, smem);
  auto it = g_ctx->occ_cache.find(key);
  if (it != g_ctx->occ_cache.end()) return it->second;
  int occ = 0;
  T2S2_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, (size_t)smem));
  if (occ < 1) occ = 1;
  g_ctx->occ_cache.emplace(key, occ);
  return occ;
}
int sm_budget() { return g_ctx->sm_budget; }

LaunchScope::LaunchScope(const char* family, double flops, double bytes) {
  t2s2_context* c = g_ctx;
  int f;
  auto ip = c->fam_by_ptr.find(family);
  if (ip != c->fam_by_ptr.end()) {
    f = ip->second;
  } else {
    auto it = c->fam_index.find(family);
    if (it == c->fam_index.end()) {
      f = (int)c->fams.size();
      c->fam_index.emplace(family, f);
      c->fams.push_back(FamilyStat{family});
    } else {
      f = it->second;
    }
    c->fam_by_ptr.emplace(family, f);
  }
  FamilyStat& st = c->fams[f];
  st.launches += 1;
  st.flops += flops;
  st.bytes += bytes;
  if (!c->profiling) return;
  while (c->event_pool.size() < c->pool_used + 2) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    c->event_pool.push_back(e);
  }
  Pending p{f, flops, bytes, c->event_pool[c->pool_used], c->event_pool[c->pool_used + 1]};
  c->pool_used += 2;
  cudaEventRecord(p.a, c->stream);
  slot = (int)c->pending.size();
  c->pending.push_back(p);
}

LaunchScope::~LaunchScope() {
  if (slot >= 0) cudaEventRecord(g_ctx->pending[slot].b, g_ctx->stream);
}

void trace_buffer(const char* tag, const double* dev, size_t n) {
  t2s2_context* c = g_ctx;
  if (c->trace_mode == 2) {  // replay: skip the recorded copy of the buffer
    T2S2_REQUIRE(c->trace_pos < c->trace.size() && c->trace[c->trace_pos].size() == n * sizeof(double),
                 kErrArg, "host_read replay: the run differs from the recorded one");
    c->trace_pos++;
    return;
  }
  if (c->trace_mode != 1 && c->trace_mode != 3) return;
  std::vector<double> h(n);
  const int before = c->trace_diff;
  host_read(h.data(), dev, n * sizeof(double));
  if (c->trace_mode == 3 && before < 0 && c->trace_diff >= 0)
    fprintf(stderr, "   ^ buffer '%s' (%zu doubles)\n", tag, n);
}

void amend_work(const char* family, double flops, double bytes) {
  t2s2_context* c = g_ctx;
  auto it = c->fam_index.find(family);
  if (it == c->fam_index.end()) return;
  c->fams[it->second].flops += flops;
  c->fams[it->second].bytes += bytes;
  for (size_t k = c->pending.size(); k-- > 0;)
    if (c->pending[k].fam == it->second) {
      c->pending[k].flops += flops;
      c->pending[k].bytes += bytes;
      break;
    }
}

namespace {
void resolve_pending(t2s2_context* c) {
  if (c->pending.empty()) return;
  cudaStreamSynchronize(c->stream);
  for (auto& p : c->pending) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) c->fams[p.fam].ms += ms;
    if (c->launch_log.size() < (size_t)T2S2_LAUNCH_LOG_CAP)
      c->launch_log.push_back(t2s2_launch_record{p.fam, p.flops, p.bytes, (double)ms});
  }
  c->pending.clear();
  c->pool_used = 0;
}
}  // namespace
cudaStream_t stream() { return g_ctx->stream; }
bool profiling() { return g_ctx->profiling; }

bool replaying_reads() { return g_ctx->trace_mode == 2; }

// A steering read without the copy engine: one small kernel copies the words
// into mapped pinned host memory and then raises a ticket the host spins on
// (system-scope fence between data and ticket).  The host-visible latency is
// the kernel's launch slot plus a PCIe posted write instead of a copy-engine
// transfer and a stream synchronisation.
__global__ void publish_kernel(const unsigned* __restrict__ src, unsigned* dst, int n_words,
                               volatile unsigned* ticket, unsigned value) {
  for (int i = threadIdx.x; i < n_words; i += blockDim.x) dst[i] = src[i];
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) *ticket = value;
}

namespace {
// trace bookkeeping of a completed read (record / compare modes)
void trace_read(t2s2_context* c, const void* host, size_t bytes);
}  // namespace

// Zeroed words for a kernel's arrival counters without a memset per launch:
// slices of a pool that is cleared as a whole when it has been handed out
// once (stream-ordered after every earlier user).
unsigned* zero_words(size_t n) {
  t2s2_context* c = g_ctx;
  T2S2_REQUIRE(n <= t2s2_context::kZeroWords, kErrArg, "zero_words: request too large");
  const bool fresh = !c->zero_pool;
  if (fresh) c->zero_pool = reinterpret_cast<unsigned*>(c->alloc.alloc(t2s2_context::kZeroWords / 2));
  if (fresh || c->zero_cursor + n > t2s2_context::kZeroWords) {
    T2S2_CUDA(cudaMemsetAsync(c->zero_pool, 0, t2s2_context::kZeroWords * sizeof(unsigned), c->stream));
    c->zero_cursor = 0;
  }
  unsigned* p = c->zero_pool + c->zero_cursor;
  c->zero_cursor += (n + 3) & ~size_t(3);
  return p;
}

ReadTicket read_open(size_t bytes) {
  t2s2_context* c = g_ctx;
  ReadTicket t;
  if (c->trace_mode == 2) return t;  // replay: nothing is published, read_close hands back the record
  T2S2_REQUIRE(bytes && bytes <= t2s2_context::kPinnedBytes && bytes % 4 == 0, kErrArg,
               "read_open: unsupported size");
  if (!c->pinned) {
    T2S2_CUDA(cudaHostAlloc(&c->pinned, t2s2_context::kPinnedBytes + 64, cudaHostAllocMapped));
    std::memset(c->pinned, 0, t2s2_context::kPinnedBytes + 64);
  }
  t.dst = static_cast<unsigned*>(c->pinned);
  t.flag = reinterpret_cast<unsigned*>(static_cast<char*>(c->pinned) + t2s2_context::kPinnedBytes);
  t.value = ++c->read_ticket;
  return t;
}

void read_publish(const void* dev, size_t bytes, const ReadTicket& t) {
  if (!t.dst) return;
  const int words = (int)(bytes / 4);
  {
    LaunchScope ls("host_read", 0.0, 2.0 * bytes);
    publish_kernel<<<1, words < 256 ? 32 * ((words + 31) / 32) : 256, 0, g_ctx->stream>>>(
        static_cast<const unsigned*>(dev), t.dst, words, t.flag, t.value);
  }
}

void read_close(void* host, size_t bytes, const ReadTicket& t) {
  t2s2_context* c = g_ctx;
  if (c->trace_mode == 2) {
    T2S2_REQUIRE(c->trace_pos < c->trace.size() && c->trace[c->trace_pos].size() == bytes, kErrArg,
                 "host_read replay: the run differs from the recorded one");
    std::memcpy(host, c->trace[c->trace_pos++].data(), bytes);
    return;
  }
  T2S2_CHECK_LAUNCH();
  // spin on the ticket; a faulted or finished stream without the ticket is an error
  volatile unsigned* ticket = t.flag;
  for (unsigned long long spins = 0; *ticket != t.value; ++spins) {
    if ((spins & 0xfffff) == 0xfffff) {
      const cudaError_t q = cudaStreamQuery(c->stream);
      if (q != cudaErrorNotReady && *ticket != t.value) {
        T2S2_CUDA(q);
        T2S2_REQUIRE(*ticket == t.value, kErrCuda, "host_read: the stream drained without the ticket");
      }
    }
  }
  std::memcpy(host, c->pinned, bytes);
  trace_read(c, host, bytes);
}

// Up to four device segments gathered straight into the mapped buffer by ONE
// kernel (instead of a pack kernel or copies followed by the publish kernel).
struct GatherArgs {
  const unsigned* src[4];
  int words[4];
  int k;
};
__global__ void gather_publish_kernel(GatherArgs a, ReadTicket t) {
  int off = 0;
  for (int q = 0; q < a.k; ++q) {
    for (int i = threadIdx.x; i < a.words[q]; i += blockDim.x) t.dst[off + i] = a.src[q][i];
    off += a.words[q];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) *(volatile unsigned*)t.flag = t.value;
}

void host_read_gather(double* host, std::initializer_list<std::pair<const double*, size_t>> parts) {
  GatherArgs a{};
  size_t total = 0;
  for (const auto& pr : parts) {
    if (!pr.second) continue;
    T2S2_REQUIRE(a.k < 4, kErrArg, "host_read_gather: at most four segments");
    a.src[a.k] = reinterpret_cast<const unsigned*>(pr.first);
    a.words[a.k++] = (int)(2 * pr.second);
    total += pr.second;
  }
  if (!total) return;
  const ReadTicket t = read_open(total * sizeof(double));
  if (t.dst) {
    LaunchScope ls("host_read", 0.0, 16.0 * total);
    gather_publish_kernel<<<1, 2 * total < 256 ? 32 * (int)((2 * total + 31) / 32) : 256, 0, stream()>>>(a, t);
  }
  read_close(host, total * sizeof(double), t);
}

void host_read(void* host, const void* dev, size_t bytes) {
  t2s2_context* c = g_ctx;
  if (c->trace_mode == 2) {
    T2S2_REQUIRE(c->trace_pos < c->trace.size() && c->trace[c->trace_pos].size() == bytes, kErrArg,
                 "host_read replay: the run differs from the recorded one");
    std::memcpy(host, c->trace[c->trace_pos++].data(), bytes);
    return;
  }
  if (bytes && bytes <= t2s2_context::kPinnedBytes && bytes % 4 == 0 &&
      reinterpret_cast<uintptr_t>(dev) % 4 == 0) {
    const ReadTicket t = read_open(bytes);
    read_publish(dev, bytes, t);
    read_close(host, bytes, t);
    return;
  }
  if (bytes) T2S2_CUDA(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, c->stream));
  T2S2_CUDA(cudaStreamSynchronize(c->stream));
  trace_read(c, host, bytes);
}

namespace {
void trace_read(t2s2_context* c, const void* host, size_t bytes) {
  if (c->trace_mode == 1) {
    const unsigned char* b = static_cast<const unsigned char*>(host);
    c->trace.emplace_back(b, b + bytes);
  } else if (c->trace_mode == 3) {
    // compare with the recorded run: report the first read that differs
    const size_t k = c->trace_pos++;
    if (k < c->trace.size() && c->trace_diff < 0 &&
        (c->trace[k].size() != bytes || std::memcmp(c->trace[k].data(), host, bytes) != 0)) {
      c->trace_diff = (int)k;
      fprintf(stderr, "host_read compare: read %zu (%zu bytes, recorded %zu) differs\n", k, bytes,
              c->trace[k].size());
      const size_t nd = bytes / 8 < c->trace[k].size() / 8 ? bytes / 8 : c->trace[k].size() / 8;
      for (size_t i = 0; i < nd && i < 24; ++i) {
        double a, b;
        std::memcpy(&a, c->trace[k].data() + 8 * i, 8);
        std::memcpy(&b, static_cast<const unsigned char*>(host) + 8 * i, 8);
        if (std::memcmp(&a, &b, 8) != 0) fprintf(stderr, "   [%zu] recorded %.17g now %.17g\n", i, a, b);
      }
    }
  }
}
}  // namespace

}  // namespace t2s2

using namespace t2s2;

namespace {

template <class F>
int guarded(t2s2_context* ctx, F&& f) {
  if (!ctx) return T2S2_ERR_ARG;
  Bind b(ctx);
  try {
    f();
    return T2S2_OK;
  } catch (const Error& e) {
    ctx->last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    ctx->last_error = e.what();
    return T2S2_ERR_ARG;
  }
}

Train make_train(int d, const int* rows, const int* cols, const int* ranks, const double* src,
                 cudaMemcpyKind kind) {
  T2S2_REQUIRE(d >= 1 && rows && ranks && src, kErrArg, "bad train arguments");
  T2S2_REQUIRE(ranks[0] == 1 && ranks[d] == 1, kErrShape, "boundary ranks must be 1");
  Train t;
  size_t off = 0;
  for (int l = 0; l < d; ++l) {
    T2S2_REQUIRE(rows[l] >= 1 && ranks[l] >= 1 && ranks[l + 1] >= 1 && (!cols || cols[l] >= 1),
                 kErrShape, "mode sizes and ranks must be positive");
    t.rows.push_back(rows[l]);
    std::vector<int> shape = cols ? std::vector<int>{ranks[l], rows[l], cols[l], ranks[l + 1]}
                                  : std::vector<int>{ranks[l], rows[l], ranks[l + 1]};
    if (cols) t.cols.push_back(cols[l]);
    DTensor c(shape);
    T2S2_CUDA(cudaMemcpyAsync(c.p, src + off, c.size() * sizeof(double), kind, stream()));
    off += c.size();
    t.cores.push_back(std::move(c));
  }
  return t;
}

t2s2_train* wrap(Train&& t) {
  auto* h = new t2s2_train;
  h->ctx = g_ctx;
  h->t = std::move(t);
  return h;
}

SolverConfig to_cfg(const t2s2_solver_config* c) {
  SolverConfig s;
  if (!c) return s;
  s.max_sweeps = c->max_sweeps;
  s.residual_tol = c->residual_tol;
  s.rounding_tol = c->rounding_tol;
  s.enrichment_rank = c->enrichment_rank;
  s.max_rank = c->max_rank;
  s.local_solver = c->local_solver;
  s.local_direct_size = c->local_direct_size;
  s.inner_tol_factor = c->inner_tol_factor;
  s.stagnation_window = c->stagnation_window;
  s.stagnation_drop = c->stagnation_drop;
  T2S2_REQUIRE(s.residual_tol > 0 && s.rounding_tol > 0, kErrValue, "tolerances must be positive");
  T2S2_REQUIRE(s.max_rank >= 1, kErrValue, "max_rank must be at least 1");
  T2S2_REQUIRE(s.max_sweeps >= 1 && s.max_sweeps <= T2S2_MAX_SWEEPS, kErrValue,
               "max_sweeps out of range");
  return s;
}

void fill_report(const SolveReport& r, t2s2_solve_report* out) {
  if (!out) return;
  out->n_sweeps = (int)r.residuals.size();
  for (int i = 0; i < out->n_sweeps; ++i) {
    out->residuals[i] = r.residuals[i];
    out->ranks[i] = r.ranks[i];
    out->compression[i] = r.compression[i];
  }
  out->wall_time = r.wall_time;
  out->converged = r.converged;
  out->stagnated = r.stagnated;
}

}  // namespace

extern "C" {

namespace {
int context_create(int device, int part, t2s2_context** out) {
  if (!out) return T2S2_ERR_ARG;
  auto ctx = std::make_unique<t2s2_context>();
  ctx->device = device;
  if (cudaSetDevice(device) != cudaSuccess) return T2S2_ERR_CUDA;
  if (part >= 0) {
    // a green context: this context's kernels run on the partition's SMs only
    if (!t2s2::partition_context(device, part, &ctx->cu_ctx, &ctx->sms)) return T2S2_ERR_VALUE;
    if (!t2s2::set_current_context(ctx->cu_ctx)) return T2S2_ERR_CUDA;
  } else if (cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, device) !=
                 cudaSuccess ||
             ctx->sms < 1) {
    return T2S2_ERR_CUDA;
  }
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess)
    return T2S2_ERR_CUDA;
  ctx->alloc.stream = ctx->stream;
  // keep freed blocks in the pool between calls
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    unsigned long long thr = ~0ULL;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  *out = ctx.release();
  return T2S2_OK;
}
}  // namespace

int t2s2_context_create(int device, t2s2_context** out) { return context_create(device, -1, out); }

int t2s2_sm_partitions(int device, int count, int* sms_out) {
  try {
    std::vector<int> sms;
    t2s2::make_sm_partitions(device, count, sms);
    for (int i = 0; i < count && sms_out; ++i) sms_out[i] = sms[i];
    return T2S2_OK;
  } catch (const t2s2::Error& e) {
    return e.code;
  }
}

int t2s2_context_create_on_partition(int device, int part, t2s2_context** out) {
  return context_create(device, part, out);
}

namespace t2s2 {
__global__ void device_clock_kernel(unsigned long long* out) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  *out = t;
}
}  // namespace t2s2

int t2s2_device_clock(t2s2_context* ctx, unsigned long long* out_ns) {
  return guarded(ctx, [&] {
    T2S2_REQUIRE(out_ns, kErrArg, "null output");
    unsigned long long* d = reinterpret_cast<unsigned long long*>(allocator().alloc(1));
    t2s2::device_clock_kernel<<<1, 1, 0, stream()>>>(d);
    T2S2_CHECK_LAUNCH();
    T2S2_CUDA(cudaMemcpyAsync(out_ns, d, sizeof *out_ns, cudaMemcpyDeviceToHost, stream()));
    T2S2_CUDA(cudaStreamSynchronize(stream()));
    allocator().release(reinterpret_cast<double*>(d));
  });
}

void t2s2_context_destroy(t2s2_context* ctx) {
  if (!ctx) return;
  if (ctx->cu_ctx)
    t2s2::set_current_context(ctx->cu_ctx);
  else
    cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->zero_pool) ctx->alloc.release(reinterpret_cast<double*>(ctx->zero_pool));
  ctx->alloc.trim();
  cudaStreamSynchronize(ctx->stream);
  for (auto e : ctx->event_pool) cudaEventDestroy(e);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  cudaStreamDestroy(ctx->stream);
  delete ctx;
}

const char* t2s2_last_error(const t2s2_context* ctx) {
  return ctx ? ctx->last_error.c_str() : "null context";
}

int t2s2_context_set_sm_budget(t2s2_context* ctx, int sms) {
  if (!ctx || sms < 0) return T2S2_ERR_ARG;
  ctx->sm_budget = sms;
  return T2S2_OK;
}

void* t2s2_stream(t2s2_context* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

int t2s2_synchronize(t2s2_context* ctx) {
  return guarded(ctx, [&] { T2S2_CUDA(cudaStreamSynchronize(stream())); });
}

int t2s2_stats_reset(t2s2_context* ctx, int profile_events) {
  return guarded(ctx, [&] {
    resolve_pending(ctx);
    for (auto& f : ctx->fams) f = FamilyStat{f.name};
    ctx->launch_log.clear();
    ctx->profiling = profile_events != 0;
  });
}

int t2s2_read_trace(t2s2_context* ctx, int mode, int* count) {
  return guarded(ctx, [&] {
    T2S2_REQUIRE(mode >= 0 && mode <= 3, kErrArg, "mode: 0 off, 1 record, 2 replay, 3 compare");
    ctx->trace_diff = -1;
    if (mode == 1) ctx->trace.clear();
    if (mode == 0 && count) *count = (int)ctx->trace.size();
    ctx->trace_pos = 0;
    ctx->trace_mode = mode;
    if (mode != 0 && count) *count = (int)ctx->trace.size();
  });
}

int t2s2_launch_log(t2s2_context* ctx, t2s2_launch_record* out, int capacity, int* count) {
  return guarded(ctx, [&] {
    resolve_pending(ctx);
    const int n = (int)ctx->launch_log.size();
    if (count) *count = n;
    for (int i = 0; i < n && i < capacity && out; ++i) out[i] = ctx->launch_log[i];
  });
}

int t2s2_stats_read(t2s2_context* ctx, t2s2_kernel_stat* out, int capacity, int* count) {
  return guarded(ctx, [&] {
    resolve_pending(ctx);
    const int n = (int)ctx->fams.size();
    if (count) *count = n;
    for (int i = 0; i < n && i < capacity && out; ++i) {
      const FamilyStat& f = ctx->fams[i];
      std::memset(out[i].family, 0, sizeof out[i].family);
      std::strncpy(out[i].family, f.name.c_str(), sizeof out[i].family - 1);
      out[i].launches = f.launches;
      out[i].device_ms = f.ms;
      out[i].flops = f.flops;
      out[i].bytes = f.bytes;
    }
  });
}

int t2s2_train_upload(t2s2_context* ctx, int d, const int* rows, const int* cols,
                      const int* ranks, const double* host_cores, t2s2_train** out) {
  return guarded(ctx, [&] {
    T2S2_REQUIRE(out, kErrArg, "null output");
    *out = wrap(make_train(d, rows, cols, ranks, host_cores, cudaMemcpyHostToDevice));
  });
}

int t2s2_train_upload_device(t2s2_context* ctx, int d, const int* rows, const int* cols,
                             const int* ranks, const double* device_cores, t2s2_train** out) {
  return guarded(ctx, [&] {
    T2S2_REQUIRE(out, kErrArg, "null output");
    *out = wrap(make_train(d, rows, cols, ranks, device_cores, cudaMemcpyDeviceToDevice));
  });
}

int t2s2_train_shape(const t2s2_train* h, int* d, int* rows, int* cols, int* ranks,
                     size_t* n_entries) {
  if (!h) return T2S2_ERR_ARG;
  const Train& t = h->t;
  if (d) *d = t.d();
  size_t n = 0;
  for (int l = 0; l < t.d(); ++l) {
    if (rows) rows[l] = t.rows[l];
    if (cols) cols[l] = t.is_op() ? t.cols[l] : 0;
    n += t.cores[l].size();
  }
  if (ranks)
    for (int l = 0; l <= t.d(); ++l) ranks[l] = t.rank(l);
  if (n_entries) *n_entries = n;
  return T2S2_OK;
}

int t2s2_train_download(t2s2_context* ctx, const t2s2_train* h, double* host_cores,
                        size_t capacity) {
  return guarded(ctx, [&] {
    T2S2_REQUIRE(h && host_cores, kErrArg, "null argument");
    size_t off = 0;
    for (auto& c : h->t.cores) {
      T2S2_REQUIRE(off + c.size() <= capacity, kErrCapacity, "download buffer too small");
      T2S2_CUDA(cudaMemcpyAsync(host_cores + off, c.p, c.size() * sizeof(double),
                                cudaMemcpyDeviceToHost, stream()));
      off += c.size();
    }
    T2S2_CUDA(cudaStreamSynchronize(stream()));
  });
}

void t2s2_train_free(t2s2_train* t) {
  if (!t) return;
  Bind b(t->ctx);
  delete t;
}

int t2s2_round(t2s2_context* ctx, const t2s2_train* v, double tol, int max_rank,
               t2s2_train** out) {
  return guarded(ctx, [&] {
    T2S2_REQUIRE(v && out, kErrArg, "null argument");
    *out = wrap(tt_round(v->t, tol, max_rank));
  });
}

int t2s2_norm(t2s2_context* ctx, const t2s2_train* v, double* out) {
  return guarded(ctx, [&] {
    T2S2_REQUIRE(v && out, kErrArg, "null argument");
    *out = tt_norm(v->t);
  });
}

int t2s2_dot(t2s2_context* ctx, const t2s2_train* a, const t2s2_train* b, double* out) {
  return guarded(ctx, [&] {
    T2S2_REQUIRE(a && b && out, kErrArg, "null argument");
    *out = tt_dot(a->t, b->t);
  });
}

int t2s2_add(t2s2_context* ctx, const t2s2_train* a, const t2s2_train* b, double sa, double sb,
             t2s2_train** out) {
  return guarded(ctx, [&] {
    T2S2_REQUIRE(a && b && out, kErrArg, "null argument");
    *out = wrap(tt_add(a->t, b->t, sa, sb));
  });
}

int t2s2_scale(t2s2_context* ctx, const t2s2_train* a, double s, t2s2_train** out) {
  return guarded(ctx, [&] {
    T2S2_REQUIRE(a && out, kErrArg, "null argument");
    *out = wrap(tt_scale(a->t, s));
  });
}

int t2s2_apply(t2s2_context* ctx, const t2s2_train* op, const t2s2_train* v, t2s2_train** out) {
  return guarded(ctx, [&] {
    T2S2_REQUIRE(op && v && out, kErrArg, "null argument");
    *out = wrap(tt_apply(op->t, v->t));
  });
}

int t2s2_full(t2s2_context* ctx, const t2s2_train* v, double* host_dense, size_t capacity) {
  return guarded(ctx, [&] {
    T2S2_REQUIRE(v && host_dense, kErrArg, "null argument");
    tt_full(v->t, host_dense, capacity);
  });
}

int t2s2_solve(t2s2_context* ctx, const t2s2_train* a, const t2s2_train* rhs,
               const t2s2_train* x0, const t2s2_solver_config* cfg, t2s2_train** x,
               t2s2_solve_report* report) {
  return guarded(ctx, [&] {
    T2S2_REQUIRE(a && rhs && x0 && x, kErrArg, "null argument");
    SolveReport rep;
    Train sol = als_solve(a->t, rhs->t, x0->t, to_cfg(cfg), rep);
    fill_report(rep, report);
    *x = wrap(std::move(sol));
  });
}

int t2s2_dense_solve(t2s2_context* ctx, int n, const double* a_colmajor, const double* b,
                     double* x) {
  return guarded(ctx, [&] {
    T2S2_REQUIRE(n >= 1 && a_colmajor && b && x, kErrArg, "bad dense solve arguments");
    DTensor A({n, n}), rhs({n});
    to_device(A.p, a_colmajor, (size_t)n * n);
    to_device(rhs.p, b, n);
    int* piv = reinterpret_cast<int*>(allocator().alloc((size_t)n / 2 + 1));
    int* info = reinterpret_cast<int*>(allocator().alloc(1));
    int h = 0;
    // verified no-pivot LU first, as the local solves do; on refusal the
    // pivoting kernel runs on a fresh copy
    DTensor A2({n, n}), rhs2({n});
    dcopy(A2.p, A.p, (size_t)n * n);
    dcopy(rhs2.p, rhs.p, n);
    if (gj_solve_nopivot(n, A2.p, rhs2.p, info)) {
      T2S2_CUDA(cudaMemcpyAsync(&h, info, sizeof(int), cudaMemcpyDeviceToHost, stream()));
      T2S2_CUDA(cudaStreamSynchronize(stream()));
      if (h == 0) dcopy(rhs.p, rhs2.p, n);
    } else {
      h = -1;
    }
    if (h == -1 && !lu_solve_fused(n, A.p, rhs.p, piv, info)) {
      lu_factor(n, A.p, piv, info);
      lu_solve(n, A.p, piv, rhs.p);
    }
    if (h == -1) T2S2_CUDA(cudaMemcpyAsync(&h, info, sizeof(int), cudaMemcpyDeviceToHost, stream()));
    to_host(x, rhs.p, n);
    allocator().release(reinterpret_cast<double*>(piv));
    allocator().release(reinterpret_cast<double*>(info));
    T2S2_REQUIRE(h == 0, kErrValue, "singular matrix");
  });
}

int t2s2_gemm(t2s2_context* ctx, int ta, int tb, int m, int n, int k, const double* a, int lda,
              const double* b, int ldb, double* c, int ldc) {
  return guarded(ctx, [&] {
    T2S2_REQUIRE(m >= 1 && n >= 1 && k >= 1 && a && b && c, kErrArg, "bad gemm arguments");
    GemmBatch gb;
    gb.add(0, ta != 0, tb != 0, m, n, k, a, lda, 0, b, ldb, 0, c, ldc, 0);
    gb.run();
  });
}

int t2s2_residual(t2s2_context* ctx, const t2s2_train* a, const t2s2_train* x,
                  const t2s2_train* rhs, double tol, double* out) {
  return guarded(ctx, [&] {
    T2S2_REQUIRE(a && x && rhs && out, kErrArg, "null argument");
    *out = tt_residual(a->t, x->t, rhs->t, tol);
  });
}

int t2s2_march(t2s2_context* ctx, const t2s2_train* left, const t2s2_train* right,
               const t2s2_train* state0, int n_steps, const t2s2_train* const* bc,
               const t2s2_train* const* src, int n_forcing, double step_tol,
               const t2s2_solver_config* cfg, int store_stride, t2s2_train** states_out,
               t2s2_step_report* reports, int* failed_step) {
  return guarded(ctx, [&] {
    T2S2_REQUIRE(left && right && state0, kErrArg, "null argument");
    T2S2_REQUIRE(n_steps >= 1, kErrValue, "need at least one step");
    T2S2_REQUIRE(n_forcing == 1 || n_forcing == n_steps, kErrArg,
                 "n_forcing must be 1 or n_steps");
    T2S2_REQUIRE(step_tol > 0, kErrValue, "step rounding tolerance must be positive");
    const SolverConfig sc = to_cfg(cfg);
    if (failed_step) *failed_step = 0;
    // the current state: the caller's initial train (read only) in step 1, then
    // this loop's own; a state that is stored is handed over when its
    // successor exists (no copies)
    Train own;
    const Train* cur = &state0->t;
    if (states_out)
      for (int k = 0; k < n_steps; ++k) states_out[k] = nullptr;
    for (int k = 1; k <= n_steps; ++k) {
      const int f = n_forcing == 1 ? 0 : k - 1;
      const Train& state = *cur;
      Train rhs = tt_apply(right->t, state);
      if (bc && bc[f]) rhs = tt_add(rhs, bc[f]->t);
      if (src && src[f]) rhs = tt_add(rhs, src[f]->t);
      rhs = tt_round(rhs, 0.01 * step_tol, 0);
      SolveReport rep;
      Train nxt = als_solve(left->t, rhs, state, sc, rep);
      double achieved = INFINITY;
      for (double r : rep.residuals) achieved = r < achieved ? r : achieved;
      if (!rep.converged && achieved > 50.0 * sc.residual_tol) {
        if (failed_step) *failed_step = k;
        char msg[160];
        snprintf(msg, sizeof msg, "step %d: inner solver stagnated at residual %.3e", k,
                 achieved);
        throw Error(kErrStagnation, msg);
      }
      Train next = tt_round(nxt, step_tol, 0);
      if (reports) {
        reports[k - 1].step = k;
        reports[k - 1].max_rank = next.max_rank();
        reports[k - 1].compression = compression_ratio(next);
        reports[k - 1].residual = rep.residuals.back();
        reports[k - 1].sweeps = (int)rep.residuals.size();
      }
      // the previous state of this loop is no longer read: store it or drop it
      if (k >= 2 && states_out && store_stride > 0 && (k - 1) % store_stride == 0)
        states_out[k - 2] = wrap(std::move(own));
      own = std::move(next);
      cur = &own;
    }
    if (states_out && store_stride > 0) states_out[n_steps - 1] = wrap(std::move(own));
  });
}

}  // extern "C"
