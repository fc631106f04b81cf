/*
 * CPU ORACLE -- TEST / BASELINE INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's per-candidate evaluator
 *   peak_memory(g, sequential_schedule(g, order))
 * from /root/reference/pkg/src/memplan/graph.py:
 *   validate_schedule      375-398 (permutation, then every direct pred earlier)
 *   sequential_schedule    401-409 (timestep = position)
 *   tensor_lifetimes       440-449 (birth = ts[producer], death = max ts[consumers]
 *                                   or horizon n-1, clamped >= birth)
 *   live_bytes_by_timestep 452-458 (the O(sum of lifetimes) add loop -- kept
 *                                   as the reference does it, this is the
 *                                   algorithm being timed)
 *   peak_memory            461-468 (max, first index; (0,0) on an empty graph)
 * Candidates are split across pthreads.  Used by tests/ as the checker for
 * large batches and by bench.py as the CPU baseline / reference arm; the
 * product path never links it.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int n, T;
  const int64_t* size;
  const int32_t* producer;
  const int32_t* cons_ptr;
  const int32_t* cons_idx;
  const int32_t* pred_ptr;
  const int32_t* pred_idx;
  const int32_t* orders;
  int64_t b0, b1;
  int64_t* peak;
  int32_t* argmax;
  uint8_t* valid;
  int events;
} Job;

static void eval_range(Job* j) {
  const int n = j->n, T = j->T;
  int32_t* pos = (int32_t*)malloc(sizeof(int32_t) * (n ? n : 1));
  int64_t* live = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
  for (int64_t b = j->b0; b < j->b1; ++b) {
    const int32_t* o = j->orders + b * (int64_t)n;
    int ok = 1;
    /* validate_schedule: sorted(order) == range(n) */
    for (int v = 0; v < n; ++v) pos[v] = -1;
    for (int i = 0; i < n && ok; ++i) {
      int v = o[i];
      if (v < 0 || v >= n || pos[v] >= 0) ok = 0;
      else pos[v] = i;
    }
    /* every direct pred scheduled earlier */
    for (int v = 0; v < n && ok; ++v)
      for (int k = j->pred_ptr[v]; k < j->pred_ptr[v + 1]; ++k)
        if (pos[j->pred_idx[k]] > pos[v]) { ok = 0; break; }
    j->valid[b] = (uint8_t)ok;
    if (!ok || n == 0) {
      j->peak[b] = 0;
      j->argmax[b] = 0;
      continue;
    }
    memset(live, 0, sizeof(int64_t) * n);
    for (int t = 0; t < T; ++t) {
      int birth = pos[j->producer[t]];
      int death = -1;
      for (int k = j->cons_ptr[t]; k < j->cons_ptr[t + 1]; ++k)
        if (pos[j->cons_idx[k]] > death) death = pos[j->cons_idx[k]];
      if (j->cons_ptr[t] == j->cons_ptr[t + 1]) death = n - 1;
      if (death < birth) death = birth;
      for (int s = birth; s <= death; ++s) live[s] += j->size[t];
    }
    int64_t best = live[0];
    int arg = 0;
    for (int s = 1; s < n; ++s)
      if (live[s] > best) { best = live[s]; arg = s; }
    j->peak[b] = best;
    j->argmax[b] = arg;
  }
  free(pos);
  free(live);
}

/* The same function for large-batch checking: identical validation, then the
 * lifetimes as +size / -size events (a difference array) instead of the
 * reference's per-step add loop -- O(n + T + E) per candidate.  Checked
 * against eval_range row for row (tests/test_oracle_golden.py). */
static void eval_range_events(Job* j) {
  const int n = j->n, T = j->T;
  int32_t* pos = (int32_t*)malloc(sizeof(int32_t) * (n ? n : 1));
  int64_t* diff = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  for (int64_t b = j->b0; b < j->b1; ++b) {
    const int32_t* o = j->orders + b * (int64_t)n;
    int ok = 1;
    for (int v = 0; v < n; ++v) pos[v] = -1;
    for (int i = 0; i < n && ok; ++i) {
      int v = o[i];
      if (v < 0 || v >= n || pos[v] >= 0) ok = 0;
      else pos[v] = i;
    }
    for (int v = 0; v < n && ok; ++v)
      for (int k = j->pred_ptr[v]; k < j->pred_ptr[v + 1]; ++k)
        if (pos[j->pred_idx[k]] > pos[v]) { ok = 0; break; }
    j->valid[b] = (uint8_t)ok;
    if (!ok || n == 0) {
      j->peak[b] = 0;
      j->argmax[b] = 0;
      continue;
    }
    memset(diff, 0, sizeof(int64_t) * (size_t)(n + 1));
    for (int t = 0; t < T; ++t) {
      int birth = pos[j->producer[t]];
      int death = -1;
      for (int k = j->cons_ptr[t]; k < j->cons_ptr[t + 1]; ++k)
        if (pos[j->cons_idx[k]] > death) death = pos[j->cons_idx[k]];
      if (j->cons_ptr[t] == j->cons_ptr[t + 1]) death = n - 1;
      if (death < birth) death = birth;
      diff[birth] += j->size[t];
      diff[death + 1] -= j->size[t];
    }
    int64_t live = diff[0], best = diff[0];
    int arg = 0;
    for (int s = 1; s < n; ++s) {
      live += diff[s];
      if (live > best) { best = live; arg = s; }
    }
    j->peak[b] = best;
    j->argmax[b] = arg;
  }
  free(pos);
  free(diff);
}

static void* worker(void* p) {
  if (((Job*)p)->events) eval_range_events((Job*)p);
  else eval_range((Job*)p);
  return NULL;
}

static int eval_orders_impl(int n, int T, const int64_t* size, const int32_t* producer,
                            const int32_t* cons_ptr, const int32_t* cons_idx,
                            const int32_t* pred_ptr, const int32_t* pred_idx,
                            const int32_t* orders, int64_t B, int threads, int64_t* peak,
                            int32_t* argmax, uint8_t* valid, int events) {
  if (threads < 1) threads = 1;
  if (threads > B) threads = B > 0 ? (int)B : 1;
  Job* jobs = (Job*)calloc((size_t)threads, sizeof(Job));
  pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  for (int k = 0; k < threads; ++k) {
    Job* j = &jobs[k];
    j->n = n; j->T = T; j->size = size; j->producer = producer;
    j->cons_ptr = cons_ptr; j->cons_idx = cons_idx; j->pred_ptr = pred_ptr; j->pred_idx = pred_idx;
    j->orders = orders; j->peak = peak; j->argmax = argmax; j->valid = valid;
    j->events = events;
    j->b0 = B * k / threads;
    j->b1 = B * (k + 1) / threads;
  }
  for (int k = 1; k < threads; ++k) pthread_create(&th[k], NULL, worker, &jobs[k]);
  worker(&jobs[0]);
  for (int k = 1; k < threads; ++k) pthread_join(th[k], NULL);
  free(jobs);
  free(th);
  return 0;
}

int oracle_eval_orders(int n, int T, const int64_t* size, const int32_t* producer,
                       const int32_t* cons_ptr, const int32_t* cons_idx, const int32_t* pred_ptr,
                       const int32_t* pred_idx, const int32_t* orders, int64_t B, int threads,
                       int64_t* peak, int32_t* argmax, uint8_t* valid) {
  return eval_orders_impl(n, T, size, producer, cons_ptr, cons_idx, pred_ptr, pred_idx, orders, B,
                          threads, peak, argmax, valid, 0);
}

/* oracle_eval_orders with the event-sweep lifetimes (same results). */
int oracle_eval_orders_events(int n, int T, const int64_t* size, const int32_t* producer,
                              const int32_t* cons_ptr, const int32_t* cons_idx,
                              const int32_t* pred_ptr, const int32_t* pred_idx,
                              const int32_t* orders, int64_t B, int threads, int64_t* peak,
                              int32_t* argmax, uint8_t* valid) {
  return eval_orders_impl(n, T, size, producer, cons_ptr, cons_idx, pred_ptr, pred_idx, orders, B,
                          threads, peak, argmax, valid, 1);
}

/* ------------------------------------------------------------------------
 * Counter-RNG Kahn candidate generator (restates memplan_oracle.kahn_candidate
 * so the CPU arm can produce the same candidates without a GPU). */
static uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

typedef struct { uint64_t k; int32_t v; } HeapEnt;

static int less_ent(HeapEnt a, HeapEnt b) { return a.k < b.k || (a.k == b.k && a.v < b.v); }

static void heap_push(HeapEnt* h, int* len, HeapEnt e) {
  int i = (*len)++;
  while (i > 0) {
    int p = (i - 1) / 2;
    if (!less_ent(e, h[p])) break;
    h[i] = h[p];
    i = p;
  }
  h[i] = e;
}

static HeapEnt heap_pop(HeapEnt* h, int* len) {
  HeapEnt top = h[0], last = h[--(*len)];
  int i = 0;
  for (;;) {
    int c = 2 * i + 1;
    if (c >= *len) break;
    if (c + 1 < *len && less_ent(h[c + 1], h[c])) ++c;
    if (!less_ent(h[c], last)) break;
    h[i] = h[c];
    i = c;
  }
  h[i] = last;
  return top;
}

typedef struct {
  int n;
  const int32_t *pred_ptr, *succ_ptr, *succ_idx;
  uint64_t seed;
  int64_t first_id, b0, b1;
  int32_t* out;
} GenJob;

static void* gen_worker(void* p) {
  GenJob* j = (GenJob*)p;
  const int n = j->n;
  int32_t* indeg = (int32_t*)malloc(sizeof(int32_t) * (n ? n : 1));
  HeapEnt* h = (HeapEnt*)malloc(sizeof(HeapEnt) * (n ? n : 1));
  for (int64_t b = j->b0; b < j->b1; ++b) {
    const uint64_t hc = mix64(j->seed ^ mix64((uint64_t)(j->first_id + b)));
    int32_t* row = j->out + b * (int64_t)n;
    int len = 0, k = 0;
    for (int v = 0; v < n; ++v) {
      indeg[v] = j->pred_ptr[v + 1] - j->pred_ptr[v];
      if (!indeg[v]) { HeapEnt e = {mix64(hc ^ (uint64_t)v), v}; heap_push(h, &len, e); }
    }
    while (len) {
      HeapEnt e = heap_pop(h, &len);
      row[k++] = e.v;
      for (int q = j->succ_ptr[e.v]; q < j->succ_ptr[e.v + 1]; ++q) {
        int w = j->succ_idx[q];
        if (--indeg[w] == 0) { HeapEnt f = {mix64(hc ^ (uint64_t)w), w}; heap_push(h, &len, f); }
      }
    }
    for (; k < n; ++k) row[k] = -1;
  }
  free(indeg);
  free(h);
  return NULL;
}

int oracle_kahn_orders(int n, const int32_t* pred_ptr, const int32_t* succ_ptr,
                       const int32_t* succ_idx, uint64_t seed, int64_t first_id, int64_t B,
                       int threads, int32_t* out) {
  if (threads < 1) threads = 1;
  if (threads > B) threads = B > 0 ? (int)B : 1;
  GenJob* jobs = (GenJob*)calloc((size_t)threads, sizeof(GenJob));
  pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  for (int k = 0; k < threads; ++k) {
    GenJob* j = &jobs[k];
    j->n = n; j->pred_ptr = pred_ptr; j->succ_ptr = succ_ptr; j->succ_idx = succ_idx;
    j->seed = seed; j->first_id = first_id; j->out = out;
    j->b0 = B * k / threads;
    j->b1 = B * (k + 1) / threads;
  }
  for (int k = 1; k < threads; ++k) pthread_create(&th[k], NULL, gen_worker, &jobs[k]);
  gen_worker(&jobs[0]);
  for (int k = 1; k < threads; ++k) pthread_join(th[k], NULL);
  free(jobs);
  free(th);
  return 0;
}
