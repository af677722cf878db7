// SM partitions of one GPU (green contexts) for independent solves.
//
// The solves of a parameter sweep (BASELINE config 4) share nothing, and a
// single solve leaves most of the 148 SMs idle through its latency-bound
// stretches.  Running several solves side by side on one GPU is only safe
// if their cooperative kernels cannot interleave on the same SMs: the
// Gauss-Jordan hand-offs and the Krylov grid barriers spin until every CTA
// of their grid is resident, so two such kernels each partly resident on
// shared SMs can wait on each other forever.  Green contexts give every
// engine context a disjoint set of SMs: its kernels — cooperative grids
// sized to the partition — can only ever wait on themselves.
//
// The driver entry points come from cudaGetDriverEntryPoint, so the library
// does not link libcuda (it still loads on hosts without a driver).
#include <cuda.h>

#include <mutex>
#include <vector>

#include "common.h"
#include "partition.h"

namespace t2s2 {
namespace {

using PFN_DeviceGet = CUresult (*)(CUdevice*, int);
using PFN_GetDevResource = CUresult (*)(CUdevice, CUdevResource*, CUdevResourceType);
using PFN_SplitByCount = CUresult (*)(CUdevResource*, unsigned*, const CUdevResource*,
                                      CUdevResource*, unsigned, unsigned);
using PFN_GenerateDesc = CUresult (*)(CUdevResourceDesc*, CUdevResource*, unsigned);
using PFN_GreenCreate = CUresult (*)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned);
using PFN_FromGreen = CUresult (*)(CUcontext*, CUgreenCtx);
using PFN_SetCurrent = CUresult (*)(CUcontext);

struct Driver {
  PFN_DeviceGet device_get = nullptr;
  PFN_GetDevResource get_resource = nullptr;
  PFN_SplitByCount split = nullptr;
  PFN_GenerateDesc gen_desc = nullptr;
  PFN_GreenCreate green_create = nullptr;
  PFN_FromGreen from_green = nullptr;
  PFN_SetCurrent set_current = nullptr;
  bool ok = false;
};

template <class F>
bool entry(const char* name, F& fn) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !p)
    return false;
  fn = reinterpret_cast<F>(p);
  return true;
}

Driver& driver() {
  static Driver d;
  static std::once_flag once;
  std::call_once(once, [] {
    d.ok = entry("cuDeviceGet", d.device_get) && entry("cuDeviceGetDevResource", d.get_resource) &&
           entry("cuDevSmResourceSplitByCount", d.split) &&
           entry("cuDevResourceGenerateDesc", d.gen_desc) &&
           entry("cuGreenCtxCreate", d.green_create) &&
           entry("cuCtxFromGreenCtx", d.from_green) && entry("cuCtxSetCurrent", d.set_current);
  });
  return d;
}

struct Plan {
  int device = -1;
  std::vector<CUcontext> ctx;  // one per partition (from its green context)
  std::vector<int> sms;
};
std::mutex g_mu;
Plan g_plan;

}  // namespace

int make_sm_partitions(int device, int count, std::vector<int>& sms) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_plan.device == device && (int)g_plan.ctx.size() == count) {
    sms = g_plan.sms;
    return 0;
  }
  T2S2_REQUIRE(g_plan.device < 0, kErrValue,
               "SM partitions already made for this process with another shape");
  T2S2_REQUIRE(count >= 1 && count <= 16, kErrValue, "partition count must be 1..16");
  Driver& d = driver();
  T2S2_REQUIRE(d.ok, kErrCuda, "green contexts unavailable (driver entry points missing)");
  T2S2_CUDA(cudaSetDevice(device));
  T2S2_CUDA(cudaFree(nullptr));  // primary context exists
  CUdevice dev;
  T2S2_REQUIRE(d.device_get(&dev, device) == CUDA_SUCCESS, kErrCuda, "cuDeviceGet failed");
  CUdevResource all;
  T2S2_REQUIRE(d.get_resource(dev, &all, CU_DEV_RESOURCE_TYPE_SM) == CUDA_SUCCESS, kErrCuda,
               "cuDeviceGetDevResource(SM) failed");
  // groups of total / count SMs rounded to the split granularity (8 on
  // B200); the last partition also takes any groups beyond count - 1 and the
  // remainder, so every SM is used: 148 SMs -> 72 76 | 48 48 52 | 40 40 40 28
  unsigned per = all.sm.smCount / (unsigned)count;
  per = (per + 4) / 8 * 8;  // nearest multiple of the split granularity
  if (per < 8) per = 8;
  std::vector<CUdevResource> grp(count + 16);
  unsigned ng = (unsigned)grp.size();
  CUdevResource rest{};
  T2S2_REQUIRE(d.split(grp.data(), &ng, &all, &rest, 0, per) == CUDA_SUCCESS, kErrCuda,
               "cuDevSmResourceSplitByCount failed");
  T2S2_REQUIRE((int)ng >= count || (ng + (rest.sm.smCount > 0 ? 1u : 0u)) >= (unsigned)count,
               kErrValue, "not enough SMs for that many partitions");
  Plan plan;
  plan.device = device;
  for (int p = 0; p < count; ++p) {
    std::vector<CUdevResource> res;
    if (p + 1 < count) {
      res.push_back(grp[p]);
    } else {
      for (unsigned q = p; q < ng; ++q) res.push_back(grp[q]);
      if (rest.sm.smCount > 0) res.push_back(rest);
    }
    unsigned n_sm = 0;
    for (auto& r : res) n_sm += r.sm.smCount;
    CUdevResourceDesc desc;
    T2S2_REQUIRE(d.gen_desc(&desc, res.data(), (unsigned)res.size()) == CUDA_SUCCESS, kErrCuda,
                 "cuDevResourceGenerateDesc failed");
    CUgreenCtx g;
    T2S2_REQUIRE(d.green_create(&g, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM) == CUDA_SUCCESS,
                 kErrCuda, "cuGreenCtxCreate failed");
    CUcontext c;
    T2S2_REQUIRE(d.from_green(&c, g) == CUDA_SUCCESS, kErrCuda, "cuCtxFromGreenCtx failed");
    plan.ctx.push_back(c);
    plan.sms.push_back((int)n_sm);
  }
  g_plan = plan;
  sms = g_plan.sms;
  return 0;
}

bool partition_context(int device, int part, void** cu_ctx, int* sms) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_plan.device != device || part < 0 || part >= (int)g_plan.ctx.size()) return false;
  *cu_ctx = g_plan.ctx[part];
  *sms = g_plan.sms[part];
  return true;
}

bool set_current_context(void* cu_ctx) {
  Driver& d = driver();
  return d.ok && d.set_current(static_cast<CUcontext>(cu_ctx)) == CUDA_SUCCESS;
}

}  // namespace t2s2
