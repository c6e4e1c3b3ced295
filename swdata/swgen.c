/* Fast path of swdata/synth.py's counter-based generator (inputs only; no method
 * arithmetic).  Bit-identical to the numpy reference implementation, which
 * tests/test_synth.py checks on small sizes.  Build: gcc -O2 -shared -fPIC -pthread. */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define GOLDEN 0x9E3779B97F4A7C15ull

static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static inline uint64_t draw(uint64_t key, uint64_t idx) { return mix64(key + (idx + 1) * GOLDEN); }
static inline double unit01(uint64_t u) { return ((double)(u >> 11) + 0.5) * (1.0 / 9007199254740992.0); }

typedef struct { uint64_t key, start; int64_t a, b; const uint8_t* lut; uint8_t* out; } job_t;

static void* res_worker(void* p) {
  job_t* j = (job_t*)p;
  for (int64_t i = j->a; i < j->b; i++) j->out[i] = j->lut[draw(j->key, j->start + (uint64_t)i) >> 48];
  return NULL;
}

/* out[i] = lut[draw(key, start+i) >> 48], i in [0, n) */
int swgen_residues(uint64_t key, uint64_t start, int64_t n, const uint8_t* lut, uint8_t* out, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (n < (1 << 20)) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  job_t jobs[256];
  for (int t = 0; t < nthreads; t++) {
    jobs[t].key = key; jobs[t].start = start; jobs[t].lut = lut; jobs[t].out = out;
    jobs[t].a = n * t / nthreads; jobs[t].b = n * (t + 1) / nthreads;
    if (nthreads == 1) res_worker(&jobs[t]);
    else pthread_create(&th[t], NULL, res_worker, &jobs[t]);
  }
  if (nthreads > 1) for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
  return 0;
}

/* Many runs at once (a shard of scattered ids):
 * out[out_off[r] + i] = lut[draw(key, gstart[r] + i) >> 48], i in [0, len[r]) */
typedef struct { uint64_t key; const int64_t *gstart, *len, *out_off; int64_t a, b; const uint8_t* lut; uint8_t* out; } runs_t;

static void* runs_worker(void* p) {
  runs_t* j = (runs_t*)p;
  for (int64_t r = j->a; r < j->b; r++) {
    uint8_t* o = j->out + j->out_off[r];
    const uint64_t g = (uint64_t)j->gstart[r];
    for (int64_t i = 0; i < j->len[r]; i++) o[i] = j->lut[draw(j->key, g + (uint64_t)i) >> 48];
  }
  return NULL;
}

int swgen_residues_runs(uint64_t key, const int64_t* gstart, const int64_t* len, const int64_t* out_off, int64_t nruns,
                        const uint8_t* lut, uint8_t* out, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nruns < 4096) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  runs_t jobs[256];
  for (int t = 0; t < nthreads; t++) {
    jobs[t].key = key; jobs[t].gstart = gstart; jobs[t].len = len; jobs[t].out_off = out_off;
    jobs[t].lut = lut; jobs[t].out = out;
    jobs[t].a = nruns * t / nthreads; jobs[t].b = nruns * (t + 1) / nthreads;
    if (nthreads == 1) runs_worker(&jobs[t]);
    else pthread_create(&th[t], NULL, runs_worker, &jobs[t]);
  }
  if (nthreads > 1) for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
  return 0;
}

/* C4 planting model (see synth._mutate).  Writes at most cap residues; returns the
 * mutated length (which may exceed cap, in which case out holds a prefix). */
int64_t swgen_mutate(const uint8_t* q, int64_t m, uint64_t key, const uint8_t* lut, uint8_t* out, int64_t cap) {
  const uint64_t ins_key = key ^ 0x5DEECE66Dull;
  int64_t w = 0;
  for (int64_t p = 0; p < m; p++) {
    uint64_t P = (uint64_t)p;
    double act = unit01(draw(key, P * 8));
    uint8_t r = q[p];
    if (act >= 0.80 && act < 0.98) {
      int done = 0;
      for (int t = 0; t < 4 && !done; t++) {
        uint8_t d = lut[draw(key, P * 8 + 1 + t) >> 48];
        if (d != q[p]) { r = d; done = 1; }
      }
      if (!done) r = (uint8_t)((q[p] + 1) % 20);
    }
    if (act >= 0.99) {
      uint64_t g = draw(key, P * 8 + 5);
      int nins = 1;
      for (int it = 0; it < 15; it++) { if (g & 1) { nins++; g >>= 1; } else { g = 0; } }
      for (int t = 0; t < nins; t++) {
        if (w < cap) out[w] = lut[draw(ins_key, P * 32 + (uint64_t)t) >> 48];
        w++;
      }
    }
    if (!(act >= 0.98 && act < 0.99)) {
      if (w < cap) out[w] = r;
      w++;
    }
  }
  return w;
}
