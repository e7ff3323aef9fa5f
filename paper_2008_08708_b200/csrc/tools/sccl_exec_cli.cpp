// sccl-exec: command-line entry of the hot path (the reference's cmd_exec /
// cmd_verify: "exec runs seeded payload execution and
// prints digest"; exit codes SPEC.md:586-587: 0 Ok, 1 usage/IO/violation).
//
//   sccl-exec verify <schedule.json>
//   sccl-exec exec   <schedule.json> [--bytes N] [--seed S] [--dtype u8|i32|f32|bf16|f16]
//                                    [--protocol auto|simple|ll] [--device D]
//
// `exec` runs every rank of the schedule on one GPU (loopback) through the
// C-ABI, with counter-based seeded payloads (splitmix64 of (seed, rank,
// word)), and prints one FNV-1a-64 digest per rank's output buffer plus the
// device time.  The same payload rule is restated in oracle/oracle.py
// (cli_payload) so the digests can be compared with the CPU oracle.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "../../../include/sccl_exec.h"

namespace {

uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

// byte i of rank r's input: little-endian bytes of splitmix64(seed<<40 ^ r<<32 ^ i/8)
void fill_payload(std::vector<uint8_t>& b, uint64_t seed, int r) {
  for (size_t i = 0; i < b.size(); i += 8) {
    uint64_t v = splitmix64((seed << 40) ^ (uint64_t(r) << 32) ^ uint64_t(i / 8));
    for (size_t k = 0; k < 8 && i + k < b.size(); ++k) b[i + k] = uint8_t(v >> (8 * k));
  }
}

uint64_t fnv1a(const std::vector<uint8_t>& b) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (uint8_t c : b) {
    h ^= c;
    h *= 0x100000001b3ull;
  }
  return h;
}

int usage() {
  std::fprintf(stderr,
               "usage: sccl-exec verify <schedule.json>\n"
               "       sccl-exec exec <schedule.json> [--bytes N] [--seed S] [--dtype u8|i32|f32|bf16|f16]\n"
               "                 [--protocol auto|simple|ll] [--device D]\n");
  return 1;
}

bool read_file(const char* path, std::string& out) {
  std::ifstream f(path);
  if (!f) return false;
  std::stringstream ss;
  ss << f.rdbuf();
  out = ss.str();
  return true;
}

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e_ = (x);                                                     \
    if (e_ != cudaSuccess) {                                                  \
      std::fprintf(stderr, "cuda: %s (%s)\n", cudaGetErrorString(e_), #x);    \
      return 1;                                                               \
    }                                                                         \
  } while (0)

}  // namespace

int main(int argc, char** argv) {
  if (argc < 3) return usage();
  std::string cmd = argv[1], text;
  if (!read_file(argv[2], text)) {
    std::fprintf(stderr, "cannot read %s\n", argv[2]);
    return 1;
  }
  if (cmd == "verify") {
    size_t len = 1 << 20;
    std::vector<char> rep(len);
    int rc = sccl_schedule_verify(text.c_str(), rep.data(), &len);
    if (rc == SCCL_OK) {
      std::printf("Ok\n");
      return 0;
    }
    std::printf("violations: %s\n%s\n", rep.data(), sccl_last_error());
    return 1;
  }
  if (cmd != "exec") return usage();
  size_t bytes = 1 << 20;
  uint64_t seed = 0;
  int dtype = SCCL_U8, device = 0;
  sccl_plan_opts o;
  sccl_plan_opts_init(&o);
  for (int i = 3; i + 1 < argc; i += 2) {
    std::string k = argv[i], v = argv[i + 1];
    if (k == "--bytes") bytes = std::strtoull(v.c_str(), nullptr, 0);
    else if (k == "--seed") seed = std::strtoull(v.c_str(), nullptr, 0);
    else if (k == "--device") device = std::atoi(v.c_str());
    else if (k == "--dtype") {
      const char* names[] = {"u8", "i32", "f32", "bf16", "f16"};
      dtype = -1;
      for (int d = 0; d < 5; ++d)
        if (v == names[d]) dtype = d;
      if (dtype < 0) return usage();
    } else if (k == "--protocol") {
      o.protocol = v == "simple" ? 1 : v == "ll" ? 2 : 0;
    } else
      return usage();
  }
  o.device = device;
  sccl_plan* plan = nullptr;
  if (sccl_plan_create_loopback(text.c_str(), bytes, dtype, SCCL_SUM, &o, &plan) != SCCL_OK) {
    std::fprintf(stderr, "plan: %s\n", sccl_last_error());
    return 1;
  }
  size_t ilen = 0;
  sccl_plan_info(plan, nullptr, &ilen);
  std::string info(ilen, '\0');
  sccl_plan_info(plan, info.data(), &ilen);
  auto field = [&](const char* key) {
    auto p = info.find(std::string("\"") + key + "\":");
    return p == std::string::npos ? 0LL : std::atoll(info.c_str() + p + std::strlen(key) + 3);
  };
  const int P = int(field("nranks"));
  const size_t sb = size_t(field("send_bytes")), rb = size_t(field("recv_bytes"));
  std::vector<void*> ds(P), dr(P);
  std::vector<std::vector<uint8_t>> hs(P, std::vector<uint8_t>(sb)), hr(P, std::vector<uint8_t>(rb));
  CK(cudaSetDevice(device));
  for (int r = 0; r < P; ++r) {
    fill_payload(hs[r], seed, r);
    CK(cudaMalloc(&ds[r], sb ? sb : 16));
    CK(cudaMalloc(&dr[r], rb ? rb : 16));
    CK(cudaMemset(dr[r], 0, rb ? rb : 16));
    if (sb) CK(cudaMemcpy(ds[r], hs[r].data(), sb, cudaMemcpyHostToDevice));
  }
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaEventRecord(a, 0));
  if (sccl_launch_loopback(plan, ds.data(), dr.data(), nullptr) != SCCL_OK) {
    std::fprintf(stderr, "launch: %s\n", sccl_last_error());
    return 1;
  }
  CK(cudaEventRecord(b, 0));
  CK(cudaDeviceSynchronize());
  if (sccl_plan_check(plan) != SCCL_OK) {
    std::fprintf(stderr, "%s\n", sccl_last_error());
    return 1;
  }
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  std::printf("{\"ranks\":%d,\"bytes_per_rank\":%zu,\"seed\":%llu,\"us\":%.2f,\"digests\":[", P, bytes,
              (unsigned long long)seed, ms * 1e3);
  for (int r = 0; r < P; ++r) {
    if (rb) CK(cudaMemcpy(hr[r].data(), dr[r], rb, cudaMemcpyDeviceToHost));
    std::printf("%s\"%016llx\"", r ? "," : "", (unsigned long long)fnv1a(hr[r]));
  }
  std::printf("]}\n");
  for (int r = 0; r < P; ++r) {
    cudaFree(ds[r]);
    cudaFree(dr[r]);
  }
  sccl_plan_destroy(plan);
  return 0;
}
