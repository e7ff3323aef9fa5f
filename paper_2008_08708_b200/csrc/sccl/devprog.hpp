// Device-side channel-program encoding shared by the host plan (plan.cpp)
// and the sm_100a executor kernel (kernels/exec_kernel.cu).  Plain structs,
// no CUDA types, so the host part compiles with g++ as well.
#pragma once

#include <cstdint>

namespace sccl {

constexpr int kMaxRanks = 16;   // pointer table width (kernel parameter space)
constexpr int kMaxOpIn = 32;    // inputs of one copy/reduce op (staged in smem)
constexpr int kMaxOpOut = 32;   // destinations of one op
constexpr int SP_FLAGS_IDX = 3; // FLAGS space index in KParams::base
constexpr int SP_SCRATCH_IDX = 2;  // SCRATCH space index in KParams::base
constexpr int kMaxTile = 65536; // one TMA pipeline stage (bytes)
constexpr int kMaxStages = 8;   // pipeline depth limit (mbarrier sets)
constexpr int kL2RelayPlain = 2;  // KParams::l2hint: re-read receipts stored with the default L2 policy
constexpr int kStageBudget = 196608;  // bytes of stages per CTA (nstage * tile)
constexpr int kThreads = 352;   // producer, kStorerWarps storer warps, signaler + 6 compute warps
constexpr int kSmemHdr = 16384;  // simple kernel: shared-memory header (barriers, rings, signaler window) ahead of the stages
constexpr int kStorerWarps = 3; // simple protocol: stage s is stored by warp 1 + s % 3 (nstage % 3 == 0)
constexpr int kLLThreads = 256; // LL kernel
constexpr int64_t kLLPart = 4096;       // LL: bytes of a chunk one CTA owns

struct DevIn {
  uint64_t off;   // byte offset of the chunk start in (rank, space)
  uint64_t len;   // chunk length (used by WAIT ops; equal to op len otherwise)
  int32_t flag;   // receipt slot at the executing rank, -1 = none
  uint32_t chunk; // chunk group of the chunk (WAIT ops filter by it)
  uint8_t rank, space;
  uint8_t dead_after;  // a scratch receipt this op is the only reader of (its bytes are dead once read)
  uint8_t pad1;
  uint32_t pad2;
};

struct DevOut {
  uint64_t off;
  int32_t flag;   // receipt slot at `rank` to signal, -1 = none
  uint8_t rank, space, every_tile, pad;
};

struct DevOp {
  uint64_t len;   // chunk length in bytes
  uint32_t chunk; // chunk group of the op's chunk: CTA channel (g, b) runs ops with chunk % kc == g
  uint32_t tile;  // simple protocol: bytes per tile of this op (the stage for copies, stage / nin
                  // rounded down to 16 for reductions; precomputed: no divide on the device)
  uint32_t in_begin, out_begin;
  uint16_t nin, nout;
  uint8_t kind;   // 0 copy, 1 reduce, 2 wait
  uint8_t vec;    // all offsets 16-byte aligned -> TMA bulk path
  uint8_t raw;    // reads a location an earlier op of this rank wrote (no flag)
  uint8_t pad1;
};

enum ErrCode : int { ERR_NONE = 0, ERR_TIMEOUT = 5 };

struct KParams {
  char* base[kMaxRanks][4];  // [rank][space]: SEND, RECV, SCRATCH, FLAGS
  const DevOp* ops;
  const DevIn* ins;
  const DevOut* outs;
  const uint32_t* prog;  // [P*kc+1] op ranges per (rank, chunk group)
  const uint32_t* dtab;  // [P*kc][8]: op begin, op end, in begin, in end, out begin, out end, compute idle, 0
  int dcache_min_ops;    // cache a CTA's descriptors in shared memory from this many ops up (0 = never)
  uint64_t* epochs;      // [nranks_launch * nch] per-CTA launch counters
  int* errinfo;          // host-mapped watchdog record
  int* abort;            // device word: set by the first watchdog expiry of the launch (cooperative abort)
  long long timeout_ns;
  int P, nch, rank0, nranks_launch;
  int kc, kb;            // nch = kc * kb: chunk groups x byte parts per chunk
  uint64_t kb_magic;     // ceil(2^64 / kb) (0 if kb == 1): byte-part split without a 64-bit divide
  uint32_t nch_magic;    // ceil(2^32 / nch): blockIdx / nch = umulhi(blockIdx, nch_magic), exact below 2^16
  uint32_t kc_magic;     // ceil(2^32 / kc): channel / kc likewise
  int tile;              // copy tile = pipeline stage bytes (<= kMaxTile); reduce tiles tile/nin
  int nstage;            // pipeline stages (<= kMaxStages, a multiple of kStorerWarps)
  int entry_base;        // index of the entry-handshake flags in FLAGS
  int multiprocess;      // 1: peers are other processes (entry handshake)
  int ll;                // 1: low-latency protocol (receipts are LL slots)
  uint64_t* trace;       // debug: per-CTA event records (nullptr = off), sccl_debug_set_trace
  int trace_cap;         // records per CTA
  int selfpub;           // 1: storer warps release their own counters (latency-bound plans)
  uint32_t window;       // simple protocol: bytes of an op a CTA moves before the next op (0 = whole op)
  const uint32_t* nwin;  // [launched CTAs] windows of each CTA's program
  int l2hint;            // bit 0: L2 eviction hints on bulk copies (launch traffic >> L2); | kL2RelayPlain
  int discard;           // 1: drop consumed scratch receipts of reduce tiles from L2 (no write-back)
  uint64_t ll_parity;    // LL, one rank per GPU: scratch holds two slot sets of this many bytes and
                         // launch e uses set e & 1, with no entry handshake (0 = one set + handshake)
};

// debug trace events of the simple-protocol kernel (record = {globaltimer ns,
// event | op << 8 | tile << 32}); see tools/probes/trace_hops.py
enum TraceEvent : int { TR_START = 0, TR_FLAG = 1, TR_FULL = 2, TR_READY = 3, TR_DONE = 4, TR_PUB = 5, TR_END = 6,
                        TR_EMPTY = 7, TR_ISSUED = 8, TR_ENTRY = 9 };

}  // namespace sccl
