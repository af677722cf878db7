// SM partitions of one GPU (green contexts), see partition.cu.
#pragma once
#include <vector>

namespace t2s2 {
// Split the device's SMs into `count` disjoint partitions (once per
// process); sms receives each partition's SM count.  Returns 0 or
// throws Error.
int make_sm_partitions(int device, int count, std::vector<int>& sms);
// The driver context (CUcontext) and SM count of partition `part`.
bool partition_context(int device, int part, void** cu_ctx, int* sms);
// cuCtxSetCurrent through the runtime's driver entry point.
bool set_current_context(void* cu_ctx);
}  // namespace t2s2
