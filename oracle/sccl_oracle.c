/*
 * sccl_oracle.c -- CPU restatement of the reference schedule module
 * (verify / verify_combining / execute).  TEST INFRASTRUCTURE ONLY; see the
 * header for the citations, the reduction-order definition and the parity
 * status.  Plain C99 + pthreads, compiled with -ffp-contract=off so the
 * floating-point adds happen exactly in the order written.
 */
#include "sccl_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------------ */
/* helpers                                                              */
/* ------------------------------------------------------------------ */

static int add_violation(oracle_violation* out, int maxv, int nv, int kind,
                         int step, int chunk, int src, int dst) {
  if (out && nv < maxv) {
    out[nv].kind = kind;
    out[nv].step = step;
    out[nv].chunk = chunk;
    out[nv].src = src;
    out[nv].dst = dst;
  }
  return nv + 1;
}

/* link matrix: E = pairs covered by >= 1 constraint, all with bound > 0
 * (SPEC.md:27).  Returns malloc'd P*P bytes. */
static uint8_t* build_links(const oracle_topology* t) {
  int P = t->P;
  uint8_t* covered = calloc((size_t)P * P, 1);
  uint8_t* zero = calloc((size_t)P * P, 1);
  for (int k = 0; k < t->ncons; ++k)
    for (int e = t->cons_off[k]; e < t->cons_off[k + 1]; ++e) {
      int a = t->cons_edges[2 * e], b = t->cons_edges[2 * e + 1];
      if (a < 0 || a >= P || b < 0 || b >= P) continue;
      covered[a * P + b] = 1;
      if (t->cons_bound[k] <= 0) zero[a * P + b] = 1;
    }
  for (int i = 0; i < P * P; ++i) covered[i] = covered[i] && !zero[i];
  free(zero);
  return covered;
}

/* schema + edge checks shared by both verifiers; returns violations count */
static int check_schema(const oracle_topology* t, const oracle_schedule* s,
                        const uint8_t* links, uint8_t* bad, oracle_violation* out,
                        int maxv, int nv) {
  int P = t->P;
  for (int st = 0; st < s->S; ++st)
    if (s->rounds[st] < 1) nv = add_violation(out, maxv, nv, ORACLE_V_SCHEMA, st, -1, -1, -1);
  for (int i = 0; i < s->nsends; ++i) {
    const int32_t* x = s->sends + 4 * i;
    int c = x[0], a = x[1], b = x[2], st = x[3];
    bad[i] = 0;
    if (c < 0 || c >= s->G || a < 0 || a >= P || b < 0 || b >= P || a == b || st < 0 ||
        st >= s->S) {
      nv = add_violation(out, maxv, nv, ORACLE_V_SCHEMA, st, c, a, b);
      bad[i] = 1;
    } else if (!links[a * P + b]) {
      nv = add_violation(out, maxv, nv, ORACLE_V_EDGE, st, c, a, b);
      bad[i] = 1;
    }
  }
  return nv;
}

/* bandwidth rule: per step, per (L,b): |sends on L| <= b*r_s */
static int check_bandwidth(const oracle_topology* t, const oracle_schedule* s,
                           const uint8_t* bad, oracle_violation* out, int maxv, int nv) {
  int P = t->P;
  int* cnt = calloc((size_t)P * P, sizeof(int));
  for (int st = 0; st < s->S; ++st) {
    memset(cnt, 0, sizeof(int) * (size_t)P * P);
    for (int i = 0; i < s->nsends; ++i) {
      const int32_t* x = s->sends + 4 * i;
      if (bad[i] || x[3] != st) continue;
      cnt[x[1] * P + x[2]]++;
    }
    for (int k = 0; k < t->ncons; ++k) {
      long tot = 0;
      for (int e = t->cons_off[k]; e < t->cons_off[k + 1]; ++e) {
        int a = t->cons_edges[2 * e], b = t->cons_edges[2 * e + 1];
        if (a >= 0 && a < P && b >= 0 && b < P) tot += cnt[a * P + b];
      }
      if (tot > (long)t->cons_bound[k] * s->rounds[st]) {
        int a = t->cons_edges[2 * t->cons_off[k]], b = t->cons_edges[2 * t->cons_off[k] + 1];
        nv = add_violation(out, maxv, nv, ORACLE_V_BANDWIDTH, st, -1, a, b);
      }
    }
  }
  free(cnt);
  return nv;
}

/* ------------------------------------------------------------------ */
/* verify                                            */
/* ------------------------------------------------------------------ */
int oracle_verify(const oracle_topology* t, const oracle_schedule* s, const uint8_t* pre,
                  const uint8_t* post, oracle_violation* out, int maxv) {
  int P = t->P, G = s->G, nv = 0;
  uint8_t* links = build_links(t);
  uint8_t* bad = calloc((size_t)s->nsends + 1, 1);
  nv = check_schema(t, s, links, bad, out, maxv, nv);

  uint8_t* V = malloc((size_t)G * P);  /* V_s */
  uint8_t* Vn = malloc((size_t)G * P); /* V_{s+1} */
  memcpy(V, pre, (size_t)G * P);
  for (int st = 0; st < s->S; ++st) {
    memcpy(Vn, V, (size_t)G * P);
    for (int i = 0; i < s->nsends; ++i) {
      const int32_t* x = s->sends + 4 * i;
      if (bad[i] || x[3] != st) continue;
      int c = x[0], a = x[1], b = x[2];
      if (!V[c * P + a]) {
        nv = add_violation(out, maxv, nv, ORACLE_V_UNAVAILABLE, st, c, a, b);
        continue;
      }
      /* exactly-once receipt (SPEC.md:404 (d), C3 PAPER.md:504-507): the
       * receiver must not already hold the chunk, nor get it twice */
      if (Vn[c * P + b]) {
        nv = add_violation(out, maxv, nv, ORACLE_V_DUPLICATE, st, c, a, b);
        continue;
      }
      Vn[c * P + b] = 1;
    }
    memcpy(V, Vn, (size_t)G * P);
  }
  for (int c = 0; c < G; ++c)
    for (int n = 0; n < P; ++n)
      if (post[c * P + n] && !V[c * P + n])
        nv = add_violation(out, maxv, nv, ORACLE_V_POST, s->S, c, -1, n);
  nv = check_bandwidth(t, s, bad, out, maxv, nv);
  free(V);
  free(Vn);
  free(bad);
  free(links);
  return nv;
}

/* ------------------------------------------------------------------ */
/* verify_combining                                  */
/* ------------------------------------------------------------------ */
int oracle_verify_combining(const oracle_topology* t, const oracle_schedule* s,
                            const uint8_t* contrib, const uint8_t* dest,
                            oracle_violation* out, int maxv) {
  int P = t->P, G = s->G, nv = 0;
  uint8_t* links = build_links(t);
  uint8_t* bad = calloc((size_t)s->nsends + 1, 1);
  nv = check_schema(t, s, links, bad, out, maxv, nv);

  /* multiset of contributors per (chunk, node): counts[(c*P+n)*P + p] */
  size_t msz = (size_t)G * P * P;
  uint16_t* ms = calloc(msz, sizeof(uint16_t));
  uint16_t* msn = calloc(msz, sizeof(uint16_t));
  for (int c = 0; c < G; ++c)
    for (int n = 0; n < P; ++n)
      if (contrib[c * P + n]) ms[((size_t)c * P + n) * P + n] = 1;
  for (int st = 0; st < s->S; ++st) {
    memcpy(msn, ms, msz * sizeof(uint16_t));
    for (int i = 0; i < s->nsends; ++i) {
      const int32_t* x = s->sends + 4 * i;
      if (bad[i] || x[3] != st) continue;
      int c = x[0], a = x[1], b = x[2];
      const uint16_t* from = ms + ((size_t)c * P + a) * P; /* sender state at V_s */
      uint16_t* to = msn + ((size_t)c * P + b) * P;
      int any = 0;
      for (int p = 0; p < P; ++p) any |= from[p] != 0;
      if (!any) {
        nv = add_violation(out, maxv, nv, ORACLE_V_UNAVAILABLE, st, c, a, b);
        continue;
      }
      for (int p = 0; p < P; ++p) {
        unsigned v = (unsigned)to[p] + from[p];
        to[p] = (uint16_t)(v > 65535u ? 65535u : v);
      }
    }
    memcpy(ms, msn, msz * sizeof(uint16_t));
  }
  for (int c = 0; c < G; ++c)
    for (int n = 0; n < P; ++n) {
      if (!dest[c * P + n]) continue;
      const uint16_t* m = ms + ((size_t)c * P + n) * P;
      for (int p = 0; p < P; ++p) {
        int want = contrib[c * P + p] ? 1 : 0;
        if (m[p] != want) {
          nv = add_violation(out, maxv, nv, ORACLE_V_MULTIPLICITY, s->S, c, p, n);
          break;
        }
      }
    }
  nv = check_bandwidth(t, s, bad, out, maxv, nv);
  free(ms);
  free(msn);
  free(bad);
  free(links);
  return nv;
}

/* ------------------------------------------------------------------ */
/* execute                                           */
/* ------------------------------------------------------------------ */

/* One data action of a step, fixed by the (data-independent) bookkeeping
 * pass.  copy: slot(dst,c) := slot(src,c).  reduce group: slot(dst,c) :=
 * [old(dst,c) if has_old] (+) in(srcs[0]) (+) in(srcs[1]) ... */
typedef struct {
  int32_t c, dst, has_old, nsrc;
  int32_t* srcs;
} group_t;

typedef struct {
  int32_t ncopy;
  int32_t* copies; /* triples (c, src, dst) */
  int32_t ngroup;
  group_t* groups;
} step_plan_t;

typedef struct {
  int P, G, S, dtype, esize;
  const int64_t* off;
  const int64_t* len;
  uint8_t* const* slots;
  const step_plan_t* steps;
  int combining;
  int tid, nthreads;
} worker_t;

static inline float bf16_to_f32(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}
static inline uint16_t f32_to_bf16_rne(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fff; /* canonical NaN (PTX cvt) */
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

static int esize_of(int dtype) {
  switch (dtype) {
    case ORACLE_U8: return 1;
    case ORACLE_I32: return 4;
    case ORACLE_F32: return 4;
    case ORACLE_BF16: return 2;
    case ORACLE_F16: return 2;
  }
  return 0;
}

/* reduce n elements: out[i] = base[i] (+) ins[0][i] (+) ins[1][i] ... */
static void reduce_elems(int dtype, int64_t n, const uint8_t* base,
                         const uint8_t* const* ins, int nin, uint8_t* out) {
  switch (dtype) {
    case ORACLE_U8:
      for (int64_t i = 0; i < n; ++i) {
        uint8_t a = base ? base[i] : ins[0][i];
        for (int k = base ? 0 : 1; k < nin; ++k) a = (uint8_t)(a + ins[k][i]);
        out[i] = a;
      }
      break;
    case ORACLE_I32:
      for (int64_t i = 0; i < n; ++i) {
        uint32_t a;
        memcpy(&a, (base ? base : ins[0]) + 4 * i, 4);
        for (int k = base ? 0 : 1; k < nin; ++k) {
          uint32_t b;
          memcpy(&b, ins[k] + 4 * i, 4);
          a += b;
        }
        memcpy(out + 4 * i, &a, 4);
      }
      break;
    case ORACLE_F32:
      for (int64_t i = 0; i < n; ++i) {
        float a;
        memcpy(&a, (base ? base : ins[0]) + 4 * i, 4);
        for (int k = base ? 0 : 1; k < nin; ++k) {
          float b;
          memcpy(&b, ins[k] + 4 * i, 4);
          a = a + b;
        }
        if (a != a) { /* canonical NaN, as GPU arithmetic returns it */
          const uint32_t q = 0x7fffffffu;
          memcpy(&a, &q, 4);
        }
        memcpy(out + 4 * i, &a, 4);
      }
      break;
    case ORACLE_BF16:
      for (int64_t i = 0; i < n; ++i) {
        uint16_t h;
        memcpy(&h, (base ? base : ins[0]) + 2 * i, 2);
        float a = bf16_to_f32(h);
        for (int k = base ? 0 : 1; k < nin; ++k) {
          memcpy(&h, ins[k] + 2 * i, 2);
          a = a + bf16_to_f32(h);
        }
        h = f32_to_bf16_rne(a);
        memcpy(out + 2 * i, &h, 2);
      }
      break;
    case ORACLE_F16:
      for (int64_t i = 0; i < n; ++i) {
        _Float16 h;
        memcpy(&h, (base ? base : ins[0]) + 2 * i, 2);
        float a = (float)h;
        for (int k = base ? 0 : 1; k < nin; ++k) {
          memcpy(&h, ins[k] + 2 * i, 2);
          a = a + (float)h;
        }
        h = (_Float16)a;
        if (a != a) { /* canonical NaN (PTX cvt) */
          const uint16_t q = 0x7fff;
          memcpy(&h, &q, 2);
        }
        memcpy(out + 2 * i, &h, 2);
      }
      break;
  }
}

static void* worker_main(void* arg) {
  worker_t* w = (worker_t*)arg;
  int P = w->P;
  (void)P;
  /* element slice of chunk c owned by this worker */
#define SLICE(c, lo, hi)                                            \
  int64_t ne_##c = w->len[c] / w->esize;                            \
  int64_t lo = ne_##c * w->tid / w->nthreads * w->esize;            \
  int64_t hi = ne_##c * (w->tid + 1) / w->nthreads * w->esize;
  for (int st = 0; st < w->S; ++st) {
    const step_plan_t* sp = &w->steps[st];
    for (int i = 0; i < sp->ncopy; ++i) {
      int c = sp->copies[3 * i], a = sp->copies[3 * i + 1], b = sp->copies[3 * i + 2];
      SLICE(c, lo, hi)
      if (hi > lo)
        memcpy(w->slots[b] + w->off[c] + lo, w->slots[a] + w->off[c] + lo, (size_t)(hi - lo));
    }
    if (!sp->ngroup) continue;
    /* all groups read V_s: compute into temporaries, then commit */
    int64_t tot = 0;
    for (int g = 0; g < sp->ngroup; ++g) {
      int c = sp->groups[g].c;
      SLICE(c, lo, hi)
      tot += hi - lo;
    }
    uint8_t* tmp = malloc((size_t)tot + 1);
    int64_t pos = 0;
    for (int g = 0; g < sp->ngroup; ++g) {
      const group_t* gr = &sp->groups[g];
      int c = gr->c;
      SLICE(c, lo, hi)
      const uint8_t* ins[64];
      for (int k = 0; k < gr->nsrc; ++k) ins[k] = w->slots[gr->srcs[k]] + w->off[c] + lo;
      const uint8_t* base = gr->has_old ? w->slots[gr->dst] + w->off[c] + lo : NULL;
      reduce_elems(w->dtype, (hi - lo) / w->esize, base, ins, gr->nsrc, tmp + pos);
      pos += hi - lo;
    }
    pos = 0;
    for (int g = 0; g < sp->ngroup; ++g) {
      const group_t* gr = &sp->groups[g];
      int c = gr->c;
      SLICE(c, lo, hi)
      memcpy(w->slots[gr->dst] + w->off[c] + lo, tmp + pos, (size_t)(hi - lo));
      pos += hi - lo;
    }
    free(tmp);
  }
#undef SLICE
  return NULL;
}

static int cmp_send_dst_chunk_src(const void* x, const void* y) {
  const int32_t* a = (const int32_t*)x;
  const int32_t* b = (const int32_t*)y;
  if (a[2] != b[2]) return a[2] - b[2]; /* dst   */
  if (a[0] != b[0]) return a[0] - b[0]; /* chunk */
  return a[1] - b[1];                   /* src   */
}

int oracle_execute(int32_t P, const oracle_schedule* s, int combining, int dtype,
                   const int64_t* chunk_off, const int64_t* chunk_len,
                   uint8_t* const* slots, uint8_t* present, int nthreads) {
  int G = s->G, S = s->S;
  int es = esize_of(dtype);
  if (P < 1 || P > 64 || G < 0 || S < 0 || es == 0) return -1;
  if (nthreads < 1) nthreads = 1;
  for (int c = 0; c < G; ++c)
    if (chunk_len[c] % es) return -1;
  for (int i = 0; i < s->nsends; ++i) {
    const int32_t* x = s->sends + 4 * i;
    if (x[0] < 0 || x[0] >= G || x[1] < 0 || x[1] >= P || x[2] < 0 || x[2] >= P || x[3] < 0 ||
        x[3] >= S)
      return -1;
  }

  /* bookkeeping pass: presence is data independent */
  step_plan_t* steps = calloc((size_t)S + 1, sizeof(step_plan_t));
  uint8_t* V = malloc((size_t)P * G + 1);
  uint8_t* Vn = malloc((size_t)P * G + 1);
  int32_t* buf = malloc(sizeof(int32_t) * 4 * ((size_t)s->nsends + 1));
  memcpy(V, present, (size_t)P * G);
  for (int st = 0; st < S; ++st) {
    int n = 0;
    for (int i = 0; i < s->nsends; ++i)
      if (s->sends[4 * i + 3] == st) memcpy(buf + 4 * n++, s->sends + 4 * i, 16);
    qsort(buf, (size_t)n, 16, cmp_send_dst_chunk_src);
    memcpy(Vn, V, (size_t)P * G);
    step_plan_t* sp = &steps[st];
    sp->copies = malloc(sizeof(int32_t) * 3 * ((size_t)n + 1));
    sp->groups = calloc((size_t)n + 1, sizeof(group_t));
    for (int i = 0; i < n;) {
      int c = buf[4 * i], b = buf[4 * i + 2];
      int j = i;
      while (j < n && buf[4 * j] == c && buf[4 * j + 2] == b) ++j;
      if (!combining) {
        for (int k = i; k < j; ++k) {
          int a = buf[4 * k + 1];
          if (!V[a * G + c]) continue; /* sender holds nothing at V_s */
          int32_t* cp = sp->copies + 3 * sp->ncopy++;
          cp[0] = c;
          cp[1] = a;
          cp[2] = b;
          Vn[b * G + c] = 1;
        }
      } else {
        group_t* gr = &sp->groups[sp->ngroup];
        gr->c = c;
        gr->dst = b;
        gr->has_old = V[b * G + c];
        gr->srcs = malloc(sizeof(int32_t) * (size_t)(j - i));
        gr->nsrc = 0;
        for (int k = i; k < j; ++k) { /* ascending src (sorted above) */
          int a = buf[4 * k + 1];
          if (V[a * G + c]) gr->srcs[gr->nsrc++] = a;
        }
        if (gr->nsrc > 0) {
          sp->ngroup++;
          Vn[b * G + c] = 1;
        } else {
          free(gr->srcs);
        }
      }
      i = j;
    }
    memcpy(V, Vn, (size_t)P * G);
  }
  memcpy(present, V, (size_t)P * G);

  /* data pass */
  worker_t* ws = calloc((size_t)nthreads, sizeof(worker_t));
  pthread_t* th = calloc((size_t)nthreads, sizeof(pthread_t));
  for (int t = 0; t < nthreads; ++t) {
    worker_t* w = &ws[t];
    w->P = P;
    w->G = G;
    w->S = S;
    w->dtype = dtype;
    w->esize = es;
    w->off = chunk_off;
    w->len = chunk_len;
    w->slots = slots;
    w->steps = steps;
    w->combining = combining;
    w->tid = t;
    w->nthreads = nthreads;
  }
  for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, worker_main, &ws[t]);
  worker_main(&ws[0]);
  for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);

  for (int st = 0; st < S; ++st) {
    for (int g = 0; g < steps[st].ngroup; ++g) free(steps[st].groups[g].srcs);
    free(steps[st].groups);
    free(steps[st].copies);
  }
  free(steps);
  free(ws);
  free(th);
  free(V);
  free(Vn);
  free(buf);
  return 0;
}

/* ------------------------------------------------------------------ */
/* host memcpy bandwidth (CPU roofline for the cpu_baseline)            */
/* ------------------------------------------------------------------ */
typedef struct {
  uint8_t* d;
  const uint8_t* s;
  int64_t n;
} cp_arg;
static void* cp_main(void* a) {
  cp_arg* x = (cp_arg*)a;
  memcpy(x->d, x->s, (size_t)x->n);
  return NULL;
}
double oracle_memcpy_bw(int64_t bytes, int nthreads, int iters) {
  if (nthreads < 1) nthreads = 1;
  uint8_t* a = malloc((size_t)bytes);
  uint8_t* b = malloc((size_t)bytes);
  if (!a || !b) return 0.0;
  memset(a, 1, (size_t)bytes);
  memset(b, 2, (size_t)bytes);
  pthread_t* th = calloc((size_t)nthreads, sizeof(pthread_t));
  cp_arg* args = calloc((size_t)nthreads, sizeof(cp_arg));
  double best = 0.0;
  for (int it = 0; it < iters; ++it) {
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    for (int t = 0; t < nthreads; ++t) {
      int64_t lo = bytes * t / nthreads, hi = bytes * (t + 1) / nthreads;
      args[t].d = b + lo;
      args[t].s = a + lo;
      args[t].n = hi - lo;
      if (t) pthread_create(&th[t], NULL, cp_main, &args[t]);
    }
    cp_main(&args[0]);
    for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
    clock_gettime(CLOCK_MONOTONIC, &t1);
    double dt = (t1.tv_sec - t0.tv_sec) + 1e-9 * (t1.tv_nsec - t0.tv_nsec);
    double bw = 2.0 * (double)bytes / dt; /* read + write */
    if (bw > best) best = bw;
  }
  free(th);
  free(args);
  free(a);
  free(b);
  return best;
}
