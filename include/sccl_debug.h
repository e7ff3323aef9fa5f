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

#ifdef __cplusplus
}
#endif
#endif
