// sccl-exec: command-line entry of the hot path (the reference's cmd_exec /
// cmd_verify: "exec runs seeded payload execution and
// prints digest"; exit codes SPEC.md:586-587: 0 Ok, 1 usage/IO/violation).
//
//   sccl-exec verify  <schedule.json>
//   sccl-exec exec    <schedule.json> [--bytes N] [--seed S] [--dtype u8|i32|f32|bf16|f16]
//                                     [--protocol auto|simple|ll] [--device D]
//   sccl-exec exec-mp <schedule.json> [same options; --devices one|each]
//
// `exec-mp` runs the same payloads one rank per PROCESS (fork before any
// CUDA call): each child creates its rank's plan through the C-ABI, swaps
// IPC blobs with its peers through files in a private temp directory (the
// "out-of-band handle exchange is the caller's job" of include/sccl_exec.h),
// binds, launches twice back to back, and writes its output's digest; the
// parent prints the same JSON as `exec`.  This is the C++-host usage of the
// multi-process boundary (no Python, no torch).  --devices each puts rank r
// on GPU r % device count (one rank per GPU on a multi-GPU box).
//
// `exec` runs every rank of the schedule on one GPU (loopback) through the
// C-ABI, with counter-based seeded payloads (splitmix64 of (seed, rank,
// word)), and prints one FNV-1a-64 digest per rank's output buffer plus the
// device time.  The same payload rule is restated in oracle/oracle.py
// (cli_payload) so the digests can be compared with the CPU oracle.
#include <cuda_runtime.h>
#include <sys/stat.h>
#include <sys/wait.h>
#include <unistd.h>

#include <chrono>
#include <thread>
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
               "                 [--protocol auto|simple|ll] [--device D]\n"
               "       sccl-exec exec-mp <schedule.json> [same options] [--devices one|each]\n");
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

long long json_field(const std::string& text, const char* key) {
  auto p = text.find(std::string("\"") + key + "\":");
  return p == std::string::npos ? -1 : std::atoll(text.c_str() + p + std::strlen(key) + 3);
}

bool write_atomic(const std::string& path, const void* data, size_t n) {
  const std::string tmp = path + ".tmp";
  FILE* f = std::fopen(tmp.c_str(), "wb");
  if (!f) return false;
  const bool ok = std::fwrite(data, 1, n, f) == n;
  std::fclose(f);
  return ok && std::rename(tmp.c_str(), path.c_str()) == 0;
}

// wait until dir/<prefix>.<r> exists for every rank (60 s)
bool wait_all(const std::string& dir, const char* prefix, int P) {
  for (int waited = 0; waited < 60000; ++waited) {
    int have = 0;
    struct stat st;
    for (int r = 0; r < P; ++r) have += stat((dir + "/" + prefix + "." + std::to_string(r)).c_str(), &st) == 0;
    if (have == P) return true;
    std::this_thread::sleep_for(std::chrono::milliseconds(1));
  }
  return false;
}

// one rank of exec-mp, in its own process
int mp_child(const std::string& text, int r, int P, size_t bytes, uint64_t seed, int dtype, int protocol,
             bool each, const std::string& dir) {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  const int dev = each && ndev > 0 ? r % ndev : 0;
  CK(cudaSetDevice(dev));
  sccl_plan_opts o;
  sccl_plan_opts_init(&o);
  o.device = dev;
  o.protocol = protocol;
  o.timeout_ms = 60000;
  sccl_plan* plan = nullptr;
  if (sccl_plan_create(text.c_str(), r, P, bytes, dtype, SCCL_SUM, &o, &plan) != SCCL_OK) {
    std::fprintf(stderr, "rank %d plan: %s\n", r, sccl_last_error());
    return 1;
  }
  size_t blen = 0;
  sccl_plan_export_handles(plan, nullptr, &blen);
  std::vector<char> mine(blen);
  if (sccl_plan_export_handles(plan, mine.data(), &blen) != SCCL_OK ||
      !write_atomic(dir + "/blob." + std::to_string(r), mine.data(), blen) || !wait_all(dir, "blob", P)) {
    std::fprintf(stderr, "rank %d: handle exchange failed (%s)\n", r, sccl_last_error());
    return 1;
  }
  std::vector<std::string> blobs(P);
  std::vector<const void*> ptrs(P);
  for (int q = 0; q < P; ++q) {
    if (!read_file((dir + "/blob." + std::to_string(q)).c_str(), blobs[q]) || blobs[q].size() != blen) return 1;
    ptrs[q] = blobs[q].data();
  }
  if (sccl_plan_bind_peers(plan, ptrs.data(), blen) != SCCL_OK) {
    std::fprintf(stderr, "rank %d bind: %s\n", r, sccl_last_error());
    return 1;
  }
  size_t ilen = 0;
  sccl_plan_info(plan, nullptr, &ilen);
  std::string info(ilen, '\0');
  sccl_plan_info(plan, info.data(), &ilen);
  const size_t sb = size_t(json_field(info, "send_bytes")), rb = size_t(json_field(info, "recv_bytes"));
  std::vector<uint8_t> hs(sb), hr(rb);
  fill_payload(hs, seed, r);
  void *ds = nullptr, *dr = nullptr;
  CK(cudaMalloc(&ds, sb ? sb : 16));
  CK(cudaMalloc(&dr, rb ? rb : 16));
  CK(cudaMemset(dr, 0, rb ? rb : 16));
  if (sb) CK(cudaMemcpy(ds, hs.data(), sb, cudaMemcpyHostToDevice));
  for (int it = 0; it < 2; ++it)  // back to back: the second launch advances every epoch
    if (sccl_launch(plan, ds, dr, nullptr) != SCCL_OK) {
      std::fprintf(stderr, "rank %d launch: %s\n", r, sccl_last_error());
      return 1;
    }
  CK(cudaDeviceSynchronize());
  if (sccl_plan_check(plan) != SCCL_OK) {
    std::fprintf(stderr, "rank %d: %s\n", r, sccl_last_error());
    return 1;
  }
  if (rb) CK(cudaMemcpy(hr.data(), dr, rb, cudaMemcpyDeviceToHost));
  char hex[32];
  std::snprintf(hex, sizeof hex, "%016llx", (unsigned long long)fnv1a(hr));
  // every rank is done with its launches before any plan (and its region,
  // which peers map) is destroyed
  if (!write_atomic(dir + "/digest." + std::to_string(r), hex, std::strlen(hex)) || !wait_all(dir, "digest", P))
    return 1;
  cudaFree(ds);
  cudaFree(dr);
  sccl_plan_destroy(plan);
  return 0;
}

int exec_mp(const std::string& text, size_t bytes, uint64_t seed, int dtype, int protocol, bool each) {
  const int P = int(json_field(text, "P"));
  if (P < 1 || P > 16) return usage();
  char tmpl[] = "/tmp/sccl-mp-XXXXXX";
  if (!mkdtemp(tmpl)) return 1;
  const std::string dir = tmpl;
  std::fflush(stdout);
  std::vector<pid_t> kids;
  for (int r = 0; r < P; ++r) {  // fork before any CUDA call in this process
    const pid_t pid = fork();
    if (pid == 0) _exit(mp_child(text, r, P, bytes, seed, dtype, protocol, each, dir));
    if (pid < 0) return 1;
    kids.push_back(pid);
  }
  int failed = 0;
  for (pid_t k : kids) {
    int st = 0;
    waitpid(k, &st, 0);
    failed += !(WIFEXITED(st) && WEXITSTATUS(st) == 0);
  }
  std::vector<std::string> dig(P);
  for (int r = 0; r < P; ++r) read_file((dir + "/digest." + std::to_string(r)).c_str(), dig[r]);
  for (int r = 0; r < P; ++r)
    for (const char* pre : {"blob.", "digest."}) std::remove((dir + "/" + pre + std::to_string(r)).c_str());
  rmdir(dir.c_str());
  if (failed) {
    std::fprintf(stderr, "%d of %d rank processes failed\n", failed, P);
    return 1;
  }
  std::printf("{\"ranks\":%d,\"processes\":%d,\"bytes_per_rank\":%zu,\"seed\":%llu,\"digests\":[", P, P, bytes,
              (unsigned long long)seed);
  for (int r = 0; r < P; ++r) std::printf("%s\"%s\"", r ? "," : "", dig[r].c_str());
  std::printf("]}\n");
  return 0;
}

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
  if (cmd != "exec" && cmd != "exec-mp") return usage();
  bool each = false;
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
    } else if (k == "--devices") {
      each = v == "each";
    } else
      return usage();
  }
  if (cmd == "exec-mp") return exec_mp(text, bytes, seed, dtype, o.protocol, each);
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
