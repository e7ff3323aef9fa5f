/*
 * sccl_debug.h -- TEST HOOKS of libsccl_exec.so.  Not part of the drop-in
 * boundary; nothing on the launch path calls these.
 */
#ifndef SCCL_DEBUG_H
#define SCCL_DEBUG_H

#include "sccl_exec.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Interpret a loopback plan's lowered channel program on CPU threads (one
 * per rank x channel; atomics stand in for the flags).  Host buffers.
 * Validates the lowering without a GPU. */
int sccl_debug_interpret_loopback(sccl_plan* plan, const void* const* sendbufs, void* const* recvbufs,
                                  double timeout_s);
const char* sccl_debug_last_error(void);

/* Event trace of the simple-protocol kernel: every CTA appends up to
 * records_per_cta records {globaltimer ns, event | op << 8 | tile << 32} to
 * device_buf + blockIdx * records_per_cta * 2 (u64 words; the caller zeroes
 * it).  device_buf = NULL turns tracing off.  Latency analysis only
 * (tools/probes/trace_hops.py). */
int sccl_debug_set_trace(sccl_plan* plan, void* device_buf, int records_per_cta);

#ifdef __cplusplus
}
#endif
#endif
