/*
 * sccl_exec.h -- C ABI of the B200 executor for SCCL-synthesized collectives.
 *
 * Drop-in boundary.  The operation it replaces is the
 * reference's schedule.execute (`execute(s | (s1,s2), inst,
 * payload_seed) -> per-node buffers`, entered through `cmd_exec`,
 * SPEC.md:576-580); its input is the same canonical schedule file the CPU
 * executor takes ("the contract any downstream lowering
 * tool consumes").  Errors map the reference hierarchy
 * (/root/reference/proj/include/sccl/error.hpp:9-30) to status codes.
 * No C++ types, no CUDA types: streams are passed as void*.
 *
 * Threading: plans are immutable after creation and
 * bind; at most one launch of a plan may be in flight per stream order;
 * distinct plans may run concurrently.  sccl_last_error is thread-local.
 * Co-residency: a launch's CTAs wait on each other (loopback: across ranks
 * on the one device), so concurrent launches on one device must fit
 * together (sccl_plan_info reports "grid"); a loopback plan sized by
 * default to the whole device should not overlap another launch.
 */
#ifndef SCCL_EXEC_H
#define SCCL_EXEC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
enum {
  SCCL_OK = 0,
  SCCL_INVALID_ARGUMENT = 1, /* sccl::invalid_argument_error: schema, unverified schedule, bad rank/size */
  SCCL_CUDA_ERROR = 4,       /* CUDA runtime failure                                                    */
  SCCL_PEER_TIMEOUT = 5,     /* watchdog: a peer never signalled                                        */
  SCCL_INTERNAL = 6
};

/* element types; redops */
enum { SCCL_U8 = 0, SCCL_I32 = 1, SCCL_F32 = 2, SCCL_BF16 = 3, SCCL_F16 = 4 };
enum { SCCL_SUM = 0 };

typedef struct sccl_plan sccl_plan;

typedef struct {
  int device;         /* CUDA device ordinal; -1 = host-only plan (lowering, handle logic; no launch) */
  int nchannels;      /* byte parts per chunk (CTAs per rank per chunk group); 0 = auto              */
  int chunk_groups;   /* chunk groups (independent chunks run on different CTAs); 0 = auto          */
  int tile_bytes;     /* pipeline stage / copy tile bytes, multiple of 16 in [256, 65536]; 0 = auto  */
  int protocol;       /* 0 = auto, 1 = simple (TMA bulk + counters), 2 = LL (flag in data)          */
  int64_t timeout_ms; /* peer-wait watchdog; 0 = default (loopback 10 s, one rank per GPU 600 s),
                         <0 = disabled.  Expiry: the launch aborts cooperatively (publishes nothing
                         more, exits normally; the CUDA context stays usable), sccl_plan_check
                         returns SCCL_PEER_TIMEOUT and the plan refuses further launches.       */
  int mem_handles;    /* multi-process region sharing: 0 = CUDA IPC handles, 1 = VMM (cuMem) POSIX FDs,
                         2 = caller-provided regions (sccl_plan_bind_peers_external)             */
  int pull;           /* combining sends of untouched inputs read in place by the receiver (no receipt
                         slot): 0 = auto (loopback plans: on), 1 = on (loopback only), -1 = off        */
} sccl_plan_opts;

void sccl_plan_opts_init(sccl_plan_opts* o);

/* ---- schedule utilities (the L2 layer) -------------------
 * Output strings use the two-call convention: *len is the buffer size on
 * input, the required size (including the NUL) on output; out may be NULL. */

/* verify / verify_combining every phase.  Returns SCCL_OK when the schedule
 * is valid, SCCL_INVALID_ARGUMENT otherwise; report gets a JSON list of
 * violations [[kind, step, chunk, src, dst], ...]. */
int sccl_schedule_verify(const char* schedule_json, char* report, size_t* len);
/* deserialize + canonical serialize */
int sccl_schedule_canonicalize(const char* schedule_json, char* out, size_t* len);
/* invert_schedule: allgather->reducescatter, broadcast->reduce */
int sccl_schedule_invert(const char* schedule_json, char* out, size_t* len);
/* Allreduce = (RS, AG) composition */
int sccl_schedule_compose_allreduce(const char* rs_json, const char* ag_json, char* out, size_t* len);

/* Per-size algorithm and protocol choice (the alpha-beta
 * cost model; "automatically switch between multiple
 * implementations"): lowers every candidate schedule (same collective and
 * P, e.g. a Pareto frontier) under both protocols for bytes_per_rank and
 * returns the candidate index and protocol (1 simple, 2 LL) with the
 * smallest predicted time under the fitted B200 model.
 * multiprocess = 0 prices a loopback plan (gpu-scope constants, pull
 * lowering), 1 a one-rank-per-GPU plan (system-scope constants, push) --
 * the same model and lowering protocol=auto uses for that kind of plan.
 * predicted_us may be NULL. */
int sccl_schedule_select(const char* const* schedule_jsons, int n, size_t bytes_per_rank, int dtype,
                         int multiprocess, int* index, int* protocol, double* predicted_us);

/* ---- plans ------------------------------------------------------------------ */

/* One rank of a multi-process (one process per GPU) execution.  Parses,
 * verifies (unverified schedules are rejected) and lowers the
 * schedule; allocates the rank's registered receive buffer, scratch and
 * flags.  bytes_per_rank follows NCCL conventions: allgather/gather = send
 * bytes per rank, reducescatter/scatter = receive bytes per rank, others =
 * the buffer size. */
int sccl_plan_create(const char* schedule_json, int rank, int nranks, size_t bytes_per_rank, int dtype,
                     int redop, const sccl_plan_opts* opts, sccl_plan** out);

/* All ranks of the schedule on ONE GPU (loopback): every rank's buffers in
 * the same device memory, one launch runs every rank's channel program. */
int sccl_plan_create_loopback(const char* schedule_json, size_t bytes_per_rank, int dtype, int redop,
                              const sccl_plan_opts* opts, sccl_plan** out);

/* Out-of-band handle exchange (multi-process): export this rank's blob,
 * gather every rank's blob (e.g. torch.distributed all_gather), bind. */
int sccl_plan_export_handles(sccl_plan* plan, void* blob, size_t* len);
int sccl_plan_bind_peers(sccl_plan* plan, const void* const* peer_blobs, size_t blob_len);

/* VMM variant (opts.mem_handles = 1): the plan region is a cuMemCreate
 * allocation shared as a POSIX file descriptor (the allocation path NCCL's
 * cuMem mode and torch symmetric memory use).  export_fd returns a new fd
 * the caller passes to the peers (e.g. SCM_RIGHTS over a Unix socket) and
 * closes; bind_peers_fd validates the blobs like sccl_plan_bind_peers and
 * maps peer r's region from fds[r] (fds[rank] is ignored). */
int sccl_plan_export_fd(sccl_plan* plan, int* fd);
int sccl_plan_bind_peers_fd(sccl_plan* plan, const void* const* peer_blobs, size_t blob_len, const int* fds);

/* Caller-provided regions (opts.mem_handles = 2): the caller allocates
 * every rank's region of sccl_plan_region_bytes bytes in memory all ranks
 * have mapped -- e.g. torch symmetric memory (symm_mem.empty + rendezvous,
 * whose buffer_ptrs are the peers' mappings) -- and binds with the
 * pointers as mapped in this process (regions[rank] is this rank's own).
 * Bind zeroes the own region; the caller must barrier after every rank has
 * bound and before the first launch, and guarantee that every rank created
 * the same plan (same schedule, size, dtype, options). */
int sccl_plan_region_bytes(sccl_plan* plan, size_t* bytes);
int sccl_plan_bind_peers_external(sccl_plan* plan, const void* const* regions);

/* The plan's own registered (peer-writable) receive buffer.  Passing it, or
 * a buffer registered with sccl_plan_register_bind, as recvbuf to
 * sccl_launch is zero-copy; any other recvbuf gets a trailing
 * device-to-device copy. */
int sccl_plan_recv_buffer(sccl_plan* plan, void** ptr, size_t* bytes);

/* Zero-copy receive targets (multi-process, CUDA IPC; SURVEY.md 8(b) b4:
 * "caller owns recvbuf, which must be peer-mapped (registered) for
 * zero-copy").  Collective, like the plan's own handle exchange: every rank
 * exports a blob for its buffer (>= the receive size, from cudaMalloc or
 * torch's caching allocator; any offset inside the allocation), the caller
 * gathers the blobs, and every rank binds its own buffer with all of them.
 * A launch whose recvbuf is a registered buffer then has the peers write it
 * directly (no copy-out); every rank must pass its counterpart registration
 * in the same launch.  Loopback plans need no registration. */
int sccl_plan_register_export(sccl_plan* plan, void* buf, size_t bytes, void* blob, size_t* len);
int sccl_plan_register_bind(sccl_plan* plan, void* buf, const void* const* peer_blobs, size_t blob_len);
int sccl_plan_deregister(sccl_plan* plan, void* buf);

/* Asynchronous, stream-ordered launch (multi-process).  Launches of one plan
 * must be ordered on every rank (one stream, or events between streams):
 * launch e-1 finishes on a rank before its launch e starts.  The simple
 * protocol stores into peers' receive buffers only after the peer's CTA has
 * entered the same launch (entry handshake); LL plans whose schedule proves
 * it (sccl_plan_info "ll_parity": allgather, alltoall, reduce-scatter,
 * allreduce) instead alternate two scratch slot sets by launch parity and
 * skip the handshake (SCCL_LL_PARITY=0 keeps it; every rank must agree --
 * bind refuses a mix). */
int sccl_launch(sccl_plan* plan, const void* sendbuf, void* recvbuf, void* stream);

/* Loopback launch: sendbufs[r]/recvbufs[r] for r < P, all on the plan's device. */
int sccl_launch_loopback(sccl_plan* plan, const void* const* sendbufs, void* const* recvbufs, void* stream);

/* Comparison backend: the same
 * lowered program executed as one cudaMemcpyAsync per send in step order
 * (copy engines / driver copies).  Non-combining schedules, simple protocol.
 * Not the hot path; bench.py reports it beside the kernel. */
int sccl_launch_loopback_copy_engine(sccl_plan* plan, const void* const* sendbufs, void* const* recvbufs,
                                     void* stream);

/* After the stream is synchronized: SCCL_PEER_TIMEOUT if the watchdog fired
 * (details in sccl_last_error), else SCCL_OK.  A timed-out plan is poisoned
 * (its launch counters are out of step with its peers'): launches return
 * SCCL_PEER_TIMEOUT; destroy it.  Peers that waited on it time out too. */
int sccl_plan_check(sccl_plan* plan);

/* Lowered program summary (JSON): ops per rank, channels, tile, scratch. */
int sccl_plan_info(sccl_plan* plan, char* out, size_t* len);

/* Kernel launches issued by this plan so far. */
int64_t sccl_plan_launch_count(sccl_plan* plan);

int sccl_plan_destroy(sccl_plan* plan);

/* ---- NVLS allreduce (comparison backend) ----------------
 * Not schedule-driven: every rank's buffer is bound to one CUDA multicast
 * object and rank r reduces slice r inside the NVSwitch (multimem.ld_reduce,
 * multimem.st) -- the switch-offloaded allreduce NCCL calls NVLS.  f32 /
 * bf16 / f16 sums (the switch accumulates 16-bit types in f32, in its own
 * order: exact for integer-valued data, within the stated float tolerance
 * otherwise).  Setup is collective: rank 0 creates and exports the
 * multicast object (POSIX fd), every rank joins (adds its device), and
 * after a barrier every rank binds.  bytes: multiple of 16 and of
 * nranks * element size.  One rank per GPU; needs multicast support
 * (an NVSwitch system whose fabric manager provides multicast). */
typedef struct sccl_nvls sccl_nvls;
/* supported = 1 when the device can form a multicast team of nranks GPUs
 * (attribute CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED and a trial object) */
int sccl_nvls_supported(int device, int nranks, int* supported);
int sccl_nvls_create(int rank, int nranks, size_t bytes, int dtype, int device, sccl_nvls** out);
int sccl_nvls_export_fd(sccl_nvls* nvls, int* fd);
int sccl_nvls_join(sccl_nvls* nvls, int fd);
int sccl_nvls_bind(sccl_nvls* nvls);
/* the multicast-bound buffer: launching from / into it is zero-copy */
int sccl_nvls_buffer(sccl_nvls* nvls, void** ptr, size_t* bytes);
int sccl_nvls_launch(sccl_nvls* nvls, const void* sendbuf, void* recvbuf, void* stream);
int sccl_nvls_check(sccl_nvls* nvls);
/* barrier watchdog of later launches: 0 = default (600 s), < 0 = disabled */
int sccl_nvls_set_timeout(sccl_nvls* nvls, int64_t timeout_ms);
int sccl_nvls_destroy(sccl_nvls* nvls);

/* thread-local message of the last failing call */
const char* sccl_last_error(void);

/* library version string */
const char* sccl_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SCCL_EXEC_H */
