/*
 * swsearch_cli.c -- a plain C99 user of the C ABI (include/swsearch.h), no Python involved.
 *
 *   swsearch_cli MATRIX DB QUERY [k] [alpha] [beta]
 *
 * MATRIX: 24 rows of 24 integers (substitution scores, row = query residue, codes in the
 *         order ARNDCQEGHILKMFPSTWYVBZX*).
 * DB:     one protein per line, one-letter codes (empty lines are empty subjects).
 * QUERY:  the query as one-letter codes.
 * Prints "score <index> <score>" for every subject, "top <rank> <id> <score>" for the top-k
 * (score descending, id ascending; Eq. 1 of the paper, ranking PAPER.md:55) and
 * "align <id> <score> <q_begin> <q_end> <s_begin> <s_end> <ops>" for the best hit (sw_align).
 * Exit status 0 on success, 1 on bad input, 2 on a library error (message on stderr).
 */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "swsearch.h"

static int die(int rc, const char* what) {
  fprintf(stderr, "%s: %s: %s\n", what, sw_strerror(rc), sw_last_error());
  return 2;
}

static char* slurp(const char* path, long* size) {
  FILE* f = fopen(path, "rb");
  if (!f) return NULL;
  fseek(f, 0, SEEK_END);
  *size = ftell(f);
  fseek(f, 0, SEEK_SET);
  char* buf = (char*)malloc((size_t)*size + 1);
  if (buf && fread(buf, 1, (size_t)*size, f) != (size_t)*size) {
    free(buf);
    buf = NULL;
  }
  fclose(f);
  if (buf) buf[*size] = 0;
  return buf;
}

int main(int argc, char** argv) {
  if (argc < 4) {
    fprintf(stderr, "usage: %s MATRIX DB QUERY [k] [alpha] [beta]\n", argv[0]);
    return 1;
  }
  const int k = argc > 4 ? atoi(argv[4]) : 10;
  const int alpha = argc > 5 ? atoi(argv[5]) : 2;
  const int beta = argc > 6 ? atoi(argv[6]) : 12;

  /* substitution matrix, padded to 32 x 32 with zeros */
  int8_t matrix[SW_MATRIX_DIM * SW_MATRIX_DIM];
  memset(matrix, 0, sizeof matrix);
  FILE* fm = fopen(argv[1], "r");
  if (!fm) { fprintf(stderr, "cannot open %s\n", argv[1]); return 1; }
  for (int r = 0; r < SW_NUM_CODES; r++)
    for (int c = 0; c < SW_NUM_CODES; c++) {
      int v;
      if (fscanf(fm, "%d", &v) != 1 || v < -128 || v > 127) {
        fprintf(stderr, "%s: need 24 x 24 int8 scores\n", argv[1]);
        fclose(fm);
        return 1;
      }
      matrix[r * SW_MATRIX_DIM + c] = (int8_t)v;
    }
  fclose(fm);

  /* database: one sequence per line, encoded in place by sw_encode */
  long size = 0;
  char* text = slurp(argv[2], &size);
  if (!text) { fprintf(stderr, "cannot read %s\n", argv[2]); return 1; }
  int64_t n = 0;
  for (long i = 0; i < size; i++) n += text[i] == '\n';
  if (size > 0 && text[size - 1] != '\n') n++;
  uint8_t* residues = (uint8_t*)malloc((size_t)size + 1);
  int64_t* offsets = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  int32_t* lengths = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
  int64_t pos = 0, s = 0;
  for (long i = 0; i < size && s < n;) {
    long e = i;
    while (e < size && text[e] != '\n') e++;
    long len = e - i;
    if (len > 0 && text[e - 1] == '\r') len--;
    int rc = sw_encode(text + i, len, residues + pos);
    if (rc != SW_OK) return die(rc, "sw_encode (database)");
    offsets[s] = pos;
    lengths[s] = (int32_t)len;
    pos += len;
    s++;
    i = e + 1;
  }
  n = s;
  const int32_t qlen = (int32_t)strlen(argv[3]);
  uint8_t* query = (uint8_t*)malloc((size_t)qlen + 1);
  int rc = sw_encode(argv[3], qlen, query);
  if (rc != SW_OK) return die(rc, "sw_encode (query)");

  sw_opts opts;
  sw_opts_default(&opts);
  sw_db* db = NULL;
  rc = sw_db_create(residues, pos, offsets, lengths, n, NULL, &opts, &db);
  if (rc != SW_OK) return die(rc, "sw_db_create");

  int32_t* scores = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  int64_t* top_ids = (int64_t*)malloc(sizeof(int64_t) * (size_t)(k > 0 ? k : 1));
  int32_t* top_scores = (int32_t*)malloc(sizeof(int32_t) * (size_t)(k > 0 ? k : 1));
  sw_stats st;
  rc = sw_search(db, query, qlen, matrix, alpha, beta, k, scores, top_ids, top_scores, &st);
  if (rc != SW_OK) { sw_db_destroy(db); return die(rc, "sw_search"); }
  for (int64_t i = 0; i < n; i++) printf("score %lld %d\n", (long long)i, scores[i]);
  for (int i = 0; i < k; i++) printf("top %d %lld %d\n", i, (long long)top_ids[i], top_scores[i]);

  if (n > 0 && top_ids[0] >= 0) {
    sw_alignment al;
    const int64_t cap = (int64_t)qlen + lengths[top_ids[0]] + 1;
    char* ops = (char*)malloc((size_t)cap);
    rc = sw_align(db, query, qlen, matrix, alpha, beta, &top_ids[0], 1, &al, ops, cap);
    if (rc != SW_OK) { sw_db_destroy(db); return die(rc, "sw_align"); }
    printf("align %lld %d %d %d %d %d %.*s\n", (long long)al.subject, al.score, al.q_begin, al.q_end,
           al.s_begin, al.s_end, al.n_ops, ops + al.ops_offset);
    free(ops);
  }
  fprintf(stderr, "%lld cells in %.3f ms (%.1f GCUPS)\n", (long long)st.cells, st.seconds * 1e3, st.gcups);
  sw_db_destroy(db);
  free(text); free(residues); free(offsets); free(lengths); free(query);
  free(scores); free(top_ids); free(top_scores);
  return 0;
}
