/*
 * sccl_oracle.h -- CPU restatement of the reference's schedule module
 * (TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may use it; the product never does).
 *
 * Reference: /root/reference/SPEC.md [MODULE] schedule
 *   verify
 *   verify_combining
 *   execute           SPEC.md:418-426, decisions SPEC.md:442-447
 * Run semantics: PAPER.md:450-461 (V_{s+1} = V_s U {(c,n') | (c,n) in V_s and
 * (c,n,n',s) in T}).
 *
 * Parity status: the reference ships no executor code,
 * so this oracle is pinned only by the SPEC's textual known-answer examples
 * (acceptance SPEC.md:641) committed as
 * fixtures under tests/golden/.  Floating-point reduction order is out of the
 * reference's scope; the order implemented here is the build's
 * own definition, shared with the GPU kernels.
 */
#ifndef SCCL_ORACLE_H
#define SCCL_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* element types (same numbering as include/sccl_exec.h) */
enum { ORACLE_U8 = 0, ORACLE_I32 = 1, ORACLE_F32 = 2, ORACLE_BF16 = 3, ORACLE_F16 = 4 };

/* violation kinds reported by the verifiers */
enum {
  ORACLE_V_SCHEMA = 1,      /* id out of range, src == dst, step >= S        */
  ORACLE_V_EDGE = 2,        /* (src,dst) not a link of the topology           */
  ORACLE_V_UNAVAILABLE = 3, /* sender does not hold the chunk at V_s          */
  ORACLE_V_BANDWIDTH = 4,   /* sends on a constraint group exceed b * Q[s]    */
  ORACLE_V_POST = 5,        /* post-condition (c,n) missing from V_S          */
  ORACLE_V_DUPLICATE = 6,   /* chunk received by a node that already holds it */
  ORACLE_V_MULTIPLICITY = 7 /* combining: contributor count != 1              */
};

typedef struct {
  int32_t kind, step, chunk, src, dst;
} oracle_violation;

/* Topology as grouped bandwidth constraints.  Constraint k
 * covers edges cons_edges[2*cons_off[k] .. 2*cons_off[k+1]) with bound
 * cons_bound[k] chunks per round. */
typedef struct {
  int32_t P;
  int32_t ncons;
  const int32_t* cons_off;   /* ncons + 1 */
  const int32_t* cons_edges; /* pairs (src,dst) */
  const int32_t* cons_bound; /* ncons */
} oracle_topology;

/* Schedule (Q,T); sends are (chunk, src, dst, step). */
typedef struct {
  int32_t G, S;
  const int32_t* rounds; /* S */
  int32_t nsends;
  const int32_t* sends; /* 4 * nsends */
} oracle_schedule;

/* verify.  pre/post are G*P byte matrices, [c*P + n].
 * Returns the number of violations (0 = Ok); up to maxv are written. */
int oracle_verify(const oracle_topology* topo, const oracle_schedule* s,
                  const uint8_t* pre, const uint8_t* post,
                  oracle_violation* out, int maxv);

/* verify_combining.  contrib[c*P+n] = node n contributes a
 * version of chunk c (combining pre); dest[c*P+n] = n must end holding the
 * fully reduced chunk (combining post).  Every dest slot must accumulate
 * every contributor of c exactly once. */
int oracle_verify_combining(const oracle_topology* topo, const oracle_schedule* s,
                            const uint8_t* contrib, const uint8_t* dest,
                            oracle_violation* out, int maxv);

/* execute.  Payload model: node n holds G
 * chunk slots; slot c of node n lives at slots[n] + chunk_off[c] and is
 * chunk_len[c] bytes; present[n*G+c] says whether the slot holds a value.
 *
 * combining == 0: step-ordered copy; a send at step s reads the sender's
 *   state V_s.
 * combining == 1: reduce-then-copy.  Receipts of step s at node n for chunk c
 *   are applied in ascending src order:  acc = old(c,n) (+) in_src0 (+) ...,
 *   each input being the sender's value at V_s.  Integer types add with
 *   two's-complement wrap (exact, order-free).  f32 adds in f32
 *   in that order; bf16/f16 widen to f32, add in that order, and round to
 *   the element type once per (node, chunk, step) (round-to-nearest-even).
 *
 * Work is split over nthreads by element range; every thread runs the whole
 * schedule on its slice (slices are independent), so results do not depend
 * on nthreads.  Returns 0, or -1 on bad arguments. */
int oracle_execute(int32_t P, const oracle_schedule* s, int combining, int dtype,
                   const int64_t* chunk_off, const int64_t* chunk_len,
                   uint8_t* const* slots, uint8_t* present, int nthreads);

/* Host copy bandwidth probe used for the CPU roofline (bytes/s). */
double oracle_memcpy_bw(int64_t bytes, int nthreads, int iters);

#ifdef __cplusplus
}
#endif
#endif
