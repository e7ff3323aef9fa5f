#include "driver.hpp"

#include <cuda_runtime.h>

#include <mutex>
#include <string>
#include <type_traits>

#include "error.hpp"

namespace sccl {

const Vmm& vmm_api() {
  static Vmm v;
  static std::once_flag once;
  std::call_once(once, [] {
    auto get = [](const char* name, auto& fn, bool required) {
      void* f = nullptr;
      cudaDriverEntryPointQueryResult q{};
      if (cudaGetDriverEntryPoint(name, &f, cudaEnableDefault, &q) != cudaSuccess || !f) {
        if (required) throw cuda_error(std::string("driver entry point ") + name + " unavailable");
        return;
      }
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(f);
    };
    get("cuMemCreate", v.create, true);
    get("cuMemGetAllocationGranularity", v.granularity, true);
    get("cuMemAddressReserve", v.reserve, true);
    get("cuMemAddressFree", v.addr_free, true);
    get("cuMemMap", v.map, true);
    get("cuMemUnmap", v.unmap, true);
    get("cuMemSetAccess", v.set_access, true);
    get("cuMemRelease", v.release, true);
    get("cuMemExportToShareableHandle", v.export_handle, true);
    get("cuMemImportFromShareableHandle", v.import_handle, true);
    get("cuMemGetAddressRange", v.address_range, true);
    get("cuMulticastCreate", v.mc_create, false);
    get("cuMulticastAddDevice", v.mc_add_device, false);
    get("cuMulticastBindMem", v.mc_bind_mem, false);
    get("cuMulticastUnbind", v.mc_unbind, false);
    get("cuMulticastGetGranularity", v.mc_granularity, false);
    get("cuDeviceGetAttribute", v.device_attribute, false);
    get("cuDeviceGet", v.device_get, false);
  });
  return v;
}

void cu_check(CUresult r, const char* what) {
  if (r != CUDA_SUCCESS) throw cuda_error(std::string(what) + " failed (CUresult " + std::to_string(int(r)) + ")");
}

char* vmm_map(const Vmm& v, CUmemGenericAllocationHandle handle, size_t size, int device) {
  CUdeviceptr va = 0;
  cu_check(v.reserve(&va, size, 0, 0, 0), "cuMemAddressReserve");
  cu_check(v.map(va, size, 0, handle, 0), "cuMemMap");
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  cu_check(v.set_access(va, size, &acc, 1), "cuMemSetAccess");
  return reinterpret_cast<char*>(va);
}

}  // namespace sccl
