// NVLS allreduce plans (the comparison backend of SURVEY.md 8(f) f4): the
// C-ABI in include/sccl_exec.h (sccl_nvls_*) over CUDA multicast objects.
//
// Setup is collective, like the schedule plans' handle exchange:
//   rank 0: sccl_nvls_create, sccl_nvls_export_fd -> fd to every peer
//   every rank: sccl_nvls_join(fd) adds its device to the multicast team
//   (barrier: every device added) every rank: sccl_nvls_bind binds its own
//   physical region and maps the multicast range.
// The region is [data | counters]; data is the caller-visible buffer
// (sccl_nvls_buffer) -- a launch from any other sendbuf / into any other
// recvbuf copies in / out around the kernel.
#include <cuda.h>
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <cstring>
#include <string>

#include "../../../include/sccl_exec.h"
#include "abi.hpp"
#include "driver.hpp"
#include "layout.hpp"

namespace sccl {
cudaError_t launch_nvls(char* mc, char* uc, uint64_t lo, uint64_t hi, uint64_t flags, uint32_t* epochs, int P,
                        int grid, int dtype, int* err, long long timeout_ns, cudaStream_t st);
}

struct sccl_nvls {
  int rank = 0, nranks = 0, device = 0, dtype = 0, grid = 32;
  size_t bytes = 0, flags_off = 0, size = 0;
  CUmemGenericAllocationHandle mc = 0, mem = 0;
  bool joined = false, bound = false;
  char* uc = nullptr;   // own mapping of the physical region
  char* mcp = nullptr;  // multicast mapping
  uint32_t* d_epochs = nullptr;
  int* h_err = nullptr;
  int* d_err = nullptr;
  long long timeout_ns = 600LL * 1000000000LL;
};

using namespace sccl;

namespace {

int nvls_esize(int dtype) {
  if (dtype == SCCL_F32) return 4;
  if (dtype == SCCL_BF16 || dtype == SCCL_F16) return 2;
  throw invalid_argument_error("NVLS allreduce supports f32, bf16 and f16 (the switch's add)");
}

CUmulticastObjectProp mc_prop(const sccl_nvls& n) {
  CUmulticastObjectProp prop{};
  prop.numDevices = unsigned(n.nranks);
  prop.size = n.size;
  prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  return prop;
}

}  // namespace

extern "C" {

int sccl_nvls_supported(int device, int nranks, int* supported) {
  return guarded([&] {
    if (!supported) throw invalid_argument_error("NULL argument");
    *supported = 0;
    const Vmm& v = vmm_api();
    if (!v.mc_create || !v.device_attribute || !v.device_get || !v.mc_granularity) return;
    CUdevice d = 0;
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    cu_check(v.device_get(&d, device), "cuDeviceGet");
    int mc = 0;
    cu_check(v.device_attribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d), "cuDeviceGetAttribute");
    if (!mc) return;
    // the attribute alone is not enough: a container or a box without the
    // fabric manager's multicast service reports it but refuses the object
    // (tools/probes/multicast_probe.py: CUDA_ERROR_INVALID_VALUE on the
    // one-GPU slice this repo is measured on) -- create a trial team
    CUmulticastObjectProp prop{};
    prop.numDevices = unsigned(std::max(1, nranks));
    prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t gran = 0;
    if (v.mc_granularity(&gran, &prop, CU_MULTICAST_GRANULARITY_MINIMUM) != CUDA_SUCCESS || !gran) return;
    prop.size = gran;
    CUmemGenericAllocationHandle h = 0;
    if (v.mc_create(&h, &prop) != CUDA_SUCCESS) return;
    v.release(h);
    *supported = 1;
  });
}

int sccl_nvls_create(int rank, int nranks, size_t bytes, int dtype, int device, sccl_nvls** out) {
  return guarded([&] {
    if (!out) throw invalid_argument_error("NULL argument");
    *out = nullptr;
    if (nranks < 1 || rank < 0 || rank >= nranks) throw invalid_argument_error("bad rank / nranks");
    const int es = nvls_esize(dtype);
    if (bytes % 16 || bytes % size_t(es * nranks))
      throw invalid_argument_error("NVLS bytes must be a multiple of 16 and of nranks * element size");
    int sup = 0;
    if (sccl_nvls_supported(device, nranks, &sup) != SCCL_OK) throw cuda_error(g_err);
    if (!sup) throw invalid_argument_error("device " + std::to_string(device) + " has no multicast support");
    auto* n = new sccl_nvls();
    try {
      n->rank = rank, n->nranks = nranks, n->device = device, n->dtype = dtype, n->bytes = bytes;
      n->flags_off = (bytes + 4095) / 4096 * 4096;
      const size_t need = n->flags_off + 2 * sizeof(uint32_t) * size_t(n->grid);
      const Vmm& v = vmm_api();
      n->size = need;
      CUmulticastObjectProp prop = mc_prop(*n);
      size_t gran = 0;
      cu_check(v.mc_granularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED), "cuMulticastGetGranularity");
      CUmemAllocationProp ap{};
      ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
      ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
      ap.location.id = device;
      size_t mgran = 0;
      cu_check(v.granularity(&mgran, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED), "cuMemGetAllocationGranularity");
      gran = std::max(gran, mgran);
      n->size = (need + gran - 1) / gran * gran;
      prop = mc_prop(*n);
      if (rank == 0) cu_check(v.mc_create(&n->mc, &prop), "cuMulticastCreate");
      cu_check(v.create(&n->mem, n->size, &ap, 0), "cuMemCreate");
      n->uc = vmm_map(v, n->mem, n->size, device);
      cuda_check(cudaMemset(n->uc, 0, n->size), "memset(nvls region)");
      cuda_check(cudaMalloc(&n->d_epochs, sizeof(uint32_t) * size_t(n->grid)), "cudaMalloc(epochs)");
      cuda_check(cudaMemset(n->d_epochs, 0, sizeof(uint32_t) * size_t(n->grid)), "memset(epochs)");
      cuda_check(cudaHostAlloc(&n->h_err, 64, cudaHostAllocMapped), "cudaHostAlloc(err)");
      std::memset(n->h_err, 0, 64);
      cuda_check(cudaHostGetDevicePointer(&n->d_err, n->h_err, 0), "cudaHostGetDevicePointer");
      cuda_check(cudaDeviceSynchronize(), "nvls setup");
    } catch (...) {
      sccl_nvls_destroy(n);
      throw;
    }
    *out = n;
  });
}

int sccl_nvls_export_fd(sccl_nvls* n, int* fd) {
  return guarded([&] {
    if (!n || !fd) throw invalid_argument_error("NULL argument");
    if (n->rank != 0) throw invalid_argument_error("only rank 0 owns the multicast object");
    int out = -1;
    cu_check(vmm_api().export_handle(&out, n->mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0),
             "cuMemExportToShareableHandle(multicast)");
    *fd = out;
  });
}

int sccl_nvls_join(sccl_nvls* n, int fd) {
  return guarded([&] {
    if (!n) throw invalid_argument_error("NULL plan");
    if (n->joined) throw invalid_argument_error("already joined");
    const Vmm& v = vmm_api();
    if (n->rank != 0) {
      if (fd < 0) throw invalid_argument_error("peers join with rank 0's multicast fd");
      cu_check(v.import_handle(&n->mc, reinterpret_cast<void*>(uintptr_t(fd)), CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
               "cuMemImportFromShareableHandle(multicast)");
    }
    CUdevice d = 0;
    cu_check(v.device_get(&d, n->device), "cuDeviceGet");
    cu_check(v.mc_add_device(n->mc, d), "cuMulticastAddDevice");
    n->joined = true;
  });
}

int sccl_nvls_bind(sccl_nvls* n) {
  return guarded([&] {
    if (!n) throw invalid_argument_error("NULL plan");
    if (!n->joined) throw invalid_argument_error("join first (every rank), then bind");
    if (n->bound) throw invalid_argument_error("already bound");
    const Vmm& v = vmm_api();
    cuda_check(cudaSetDevice(n->device), "cudaSetDevice");
    cu_check(v.mc_bind_mem(n->mc, 0, n->mem, 0, n->size, 0), "cuMulticastBindMem");
    n->mcp = vmm_map(v, n->mc, n->size, n->device);
    n->bound = true;
  });
}

int sccl_nvls_buffer(sccl_nvls* n, void** ptr, size_t* bytes) {
  return guarded([&] {
    if (!n || !ptr) throw invalid_argument_error("NULL argument");
    *ptr = n->uc;
    if (bytes) *bytes = n->bytes;
  });
}

int sccl_nvls_launch(sccl_nvls* n, const void* sendbuf, void* recvbuf, void* stream) {
  return guarded([&] {
    if (!n) throw invalid_argument_error("NULL plan");
    if (!n->bound) throw invalid_argument_error("NVLS plan not bound (sccl_nvls_bind)");
    if (reinterpret_cast<volatile int*>(n->h_err)[0])
      throw timeout_error("NVLS plan aborted by an earlier barrier timeout; destroy it");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cuda_check(cudaSetDevice(n->device), "cudaSetDevice");
    if (sendbuf && sendbuf != n->uc)
      cuda_check(cudaMemcpyAsync(n->uc, sendbuf, n->bytes, cudaMemcpyDeviceToDevice, st), "copy-in");
    const Part slice = split16(int64_t(n->bytes), n->nranks, n->rank);
    cuda_check(launch_nvls(n->mcp, n->uc, uint64_t(slice.off), uint64_t(slice.off + slice.len), n->flags_off,
                           n->d_epochs, n->nranks, n->grid, n->dtype, n->d_err, n->timeout_ns, st),
               "NVLS launch");
    if (recvbuf && recvbuf != n->uc)
      cuda_check(cudaMemcpyAsync(recvbuf, n->uc, n->bytes, cudaMemcpyDeviceToDevice, st), "copy-out");
  });
}

int sccl_nvls_check(sccl_nvls* n) {
  return guarded([&] {
    if (!n) throw invalid_argument_error("NULL plan");
    if (n->h_err && reinterpret_cast<volatile int*>(n->h_err)[0])
      throw timeout_error("NVLS barrier timeout: a peer never arrived");
  });
}

int sccl_nvls_set_timeout(sccl_nvls* n, int64_t timeout_ms) {
  return guarded([&] {
    if (!n) throw invalid_argument_error("NULL plan");
    n->timeout_ns = timeout_ms < 0 ? 0 : (timeout_ms == 0 ? 600LL * 1000000000LL : timeout_ms * 1000000LL);
  });
}

int sccl_nvls_destroy(sccl_nvls* n) {
  if (!n) return SCCL_OK;
  cudaSetDevice(n->device);
  cudaDeviceSynchronize();
  try {
    const Vmm& v = vmm_api();
    if (n->mcp) {
      v.unmap(CUdeviceptr(n->mcp), n->size);
      v.addr_free(CUdeviceptr(n->mcp), n->size);
    }
    if (n->bound && v.mc_unbind && v.device_get) {
      CUdevice d = 0;
      if (v.device_get(&d, n->device) == CUDA_SUCCESS) v.mc_unbind(n->mc, d, 0, n->size);
    }
    if (n->uc) {
      v.unmap(CUdeviceptr(n->uc), n->size);
      v.addr_free(CUdeviceptr(n->uc), n->size);
    }
    if (n->mem) v.release(n->mem);
    if (n->mc) v.release(n->mc);
  } catch (...) {
  }
  cudaFree(n->d_epochs);
  if (n->h_err) cudaFreeHost(n->h_err);
  delete n;
  return SCCL_OK;
}

}  // extern "C"
