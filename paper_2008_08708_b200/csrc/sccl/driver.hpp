// CUDA driver entry points the library needs beyond the runtime (VMM,
// multicast), resolved at run time through cudaGetDriverEntryPoint: no
// link-time dependency on libcuda, so the library loads on GPU-less hosts.
#pragma once

#include <cuda.h>

#include <cstddef>

namespace sccl {

struct Vmm {
  decltype(&cuMemCreate) create = nullptr;
  decltype(&cuMemGetAllocationGranularity) granularity = nullptr;
  decltype(&cuMemAddressReserve) reserve = nullptr;
  decltype(&cuMemAddressFree) addr_free = nullptr;
  decltype(&cuMemMap) map = nullptr;
  decltype(&cuMemUnmap) unmap = nullptr;
  decltype(&cuMemSetAccess) set_access = nullptr;
  decltype(&cuMemRelease) release = nullptr;
  decltype(&cuMemExportToShareableHandle) export_handle = nullptr;
  decltype(&cuMemImportFromShareableHandle) import_handle = nullptr;
  decltype(&cuMemGetAddressRange) address_range = nullptr;
  // multicast (NVLS); null when the driver lacks them
  decltype(&cuMulticastCreate) mc_create = nullptr;
  decltype(&cuMulticastAddDevice) mc_add_device = nullptr;
  decltype(&cuMulticastBindMem) mc_bind_mem = nullptr;
  decltype(&cuMulticastUnbind) mc_unbind = nullptr;
  decltype(&cuMulticastGetGranularity) mc_granularity = nullptr;
  decltype(&cuDeviceGetAttribute) device_attribute = nullptr;
  decltype(&cuDeviceGet) device_get = nullptr;
};

// throws cuda_error when a required entry point is missing
const Vmm& vmm_api();
void cu_check(CUresult r, const char* what);
// map `handle` (size bytes) at a fresh VA range readable and writable by `device`
char* vmm_map(const Vmm& v, CUmemGenericAllocationHandle handle, size_t size, int device);

}  // namespace sccl
