/*
 * oracle.c -- plain, slow, obviously correct CPU convolution (see oracle.h).
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Nothing here is blocked, fused or
 * reordered beyond the definition: a 7-deep loop nest over
 * (n, ho, wo, kh, kw, c, f) with the feature loop innermost so the HWCF
 * filter row w[kh,kw,c,:] is read contiguously.  Work is split across
 * pthreads by output row (n, ho) -- rows are independent, so threading does
 * not change any result bit.
 */
#include "oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* SPEC.md:48-56 shape algebra, own copy (reading R3). */
int oracle_output_shape(const oracle_params* p, int32_t out_nhwf[4], int32_t pads_tblr[4]) {
  if (!p) return 1;
  if (p->batch < 1 || p->in_rows < 1 || p->in_cols < 1 || p->channels < 1 || p->features < 1 ||
      p->window_rows < 1 || p->window_cols < 1 || p->stride_rows < 1 || p->stride_cols < 1)
    return 1;
  int64_t ho, wo, pt = 0, pb = 0, pl = 0, pr = 0;
  if (p->padding == ORACLE_SAME) {
    ho = (p->in_rows + p->stride_rows - 1) / p->stride_rows;
    wo = (p->in_cols + p->stride_cols - 1) / p->stride_cols;
    int64_t tr = (ho - 1) * p->stride_rows + p->window_rows - p->in_rows;
    int64_t tc = (wo - 1) * p->stride_cols + p->window_cols - p->in_cols;
    if (tr < 0) tr = 0;
    if (tc < 0) tc = 0;
    pt = tr / 2; pb = tr - pt;
    pl = tc / 2; pr = tc - pl;
  } else if (p->padding == ORACLE_VALID) {
    if (p->window_rows > p->in_rows || p->window_cols > p->in_cols) return 1;
    ho = (p->in_rows - p->window_rows) / p->stride_rows + 1;
    wo = (p->in_cols - p->window_cols) / p->stride_cols + 1;
  } else {
    return 1;
  }
  if (out_nhwf) {
    out_nhwf[0] = p->batch; out_nhwf[1] = (int32_t)ho; out_nhwf[2] = (int32_t)wo;
    out_nhwf[3] = p->features;
  }
  if (pads_tblr) {
    pads_tblr[0] = (int32_t)pt; pads_tblr[1] = (int32_t)pb;
    pads_tblr[2] = (int32_t)pl; pads_tblr[3] = (int32_t)pr;
  }
  return 0;
}

uint64_t oracle_flop_count(const oracle_params* p) {
  int32_t o[4], pd[4];
  if (oracle_output_shape(p, o, pd)) return 0;
  return 2ull * (uint64_t)o[0] * (uint64_t)o[1] * (uint64_t)o[2] * (uint64_t)p->window_rows *
         (uint64_t)p->window_cols * (uint64_t)p->channels * (uint64_t)p->features;
}

typedef struct {
  const oracle_params* p;
  const float* in;
  const float* filt;
  float* out;
  double* denom;
  int32_t o[4], pd[4];
  int64_t row_begin, row_end; /* rows are (n, ho) pairs: r = n*Ho + ho */
} job_t;

static void* run_rows(void* arg) {
  job_t* j = (job_t*)arg;
  const oracle_params* p = j->p;
  const int64_t H = p->in_rows, W = p->in_cols, C = p->channels, F = p->features;
  const int64_t KH = p->window_rows, KW = p->window_cols, SR = p->stride_rows, SC = p->stride_cols;
  const int64_t HO = j->o[1], WO = j->o[2];
  const int64_t PT = j->pd[0], PL = j->pd[2];
  double* acc = (double*)malloc(sizeof(double) * (size_t)F);
  double* dac = (double*)malloc(sizeof(double) * (size_t)F);
  for (int64_t r = j->row_begin; r < j->row_end; ++r) {
    const int64_t n = r / HO, ho = r % HO;
    for (int64_t wo = 0; wo < WO; ++wo) {
      for (int64_t f = 0; f < F; ++f) { acc[f] = 0.0; dac[f] = 0.0; }
      for (int64_t kh = 0; kh < KH; ++kh) {
        const int64_t ih = ho * SR + kh - PT;
        if (ih < 0 || ih >= H) continue; /* zero padding contributes 0 */
        for (int64_t kw = 0; kw < KW; ++kw) {
          const int64_t iw = wo * SC + kw - PL;
          if (iw < 0 || iw >= W) continue;
          const float* xrow = j->in + ((n * H + ih) * W + iw) * C;
          for (int64_t c = 0; c < C; ++c) {
            const double xv = (double)xrow[c];
            const float* wrow = j->filt + ((kh * KW + kw) * C + c) * F;
            for (int64_t f = 0; f < F; ++f) {
              const double prod = xv * (double)wrow[f]; /* exact: 24+24 bits < 53 */
              acc[f] += prod;
              if (j->denom) dac[f] += fabs(prod);
            }
          }
        }
      }
      float* yrow = j->out + ((n * HO + ho) * WO + wo) * F;
      for (int64_t f = 0; f < F; ++f) yrow[f] = (float)acc[f]; /* one RN-even rounding */
      if (j->denom) {
        double* drow = j->denom + ((n * HO + ho) * WO + wo) * F;
        for (int64_t f = 0; f < F; ++f) drow[f] = dac[f];
      }
    }
  }
  free(acc);
  free(dac);
  return NULL;
}

int oracle_conv2d(const oracle_params* p, const float* in, const float* filt, float* out,
                  double* denom, int threads) {
  int32_t o[4], pd[4];
  if (!in || !filt || !out) return 1;
  if (oracle_output_shape(p, o, pd)) return 1;
  const int64_t rows = (int64_t)o[0] * o[1];
  if (threads < 1) threads = 1;
  if (threads > rows) threads = (int)rows;
  job_t* jobs = (job_t*)calloc((size_t)threads, sizeof(job_t));
  pthread_t* tids = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  for (int t = 0; t < threads; ++t) {
    jobs[t].p = p; jobs[t].in = in; jobs[t].filt = filt; jobs[t].out = out; jobs[t].denom = denom;
    memcpy(jobs[t].o, o, sizeof o);
    memcpy(jobs[t].pd, pd, sizeof pd);
    jobs[t].row_begin = rows * t / threads;
    jobs[t].row_end = rows * (t + 1) / threads;
  }
  for (int t = 1; t < threads; ++t) pthread_create(&tids[t], NULL, run_rows, &jobs[t]);
  run_rows(&jobs[0]);
  for (int t = 1; t < threads; ++t) pthread_join(tids[t], NULL);
  free(jobs);
  free(tids);
  return 0;
}

int oracle_conv2d_point(const oracle_params* p, const float* in, const float* filt, int64_t n,
                        int64_t ho, int64_t wo, int64_t f, double* y, double* denom) {
  int32_t o[4], pd[4];
  if (!in || !filt || !y) return 1;
  if (oracle_output_shape(p, o, pd)) return 1;
  if (n < 0 || n >= o[0] || ho < 0 || ho >= o[1] || wo < 0 || wo >= o[2] || f < 0 || f >= o[3])
    return 1;
  const int64_t H = p->in_rows, W = p->in_cols, C = p->channels, F = p->features;
  double acc = 0.0, dac = 0.0;
  for (int64_t kh = 0; kh < p->window_rows; ++kh) {
    const int64_t ih = ho * p->stride_rows + kh - pd[0];
    if (ih < 0 || ih >= H) continue;
    for (int64_t kw = 0; kw < p->window_cols; ++kw) {
      const int64_t iw = wo * p->stride_cols + kw - pd[2];
      if (iw < 0 || iw >= W) continue;
      for (int64_t c = 0; c < C; ++c) {
        const double prod = (double)in[((n * H + ih) * W + iw) * C + c] *
                            (double)filt[((kh * p->window_cols + kw) * C + c) * F + f];
        acc += prod;
        dac += fabs(prod);
      }
    }
  }
  *y = acc;
  if (denom) *denom = dac;
  return 0;
}

typedef struct {
  const oracle_params* p;
  const float* in;
  const float* filt;
  const int64_t* idx;
  int64_t begin, end;
  double* y;
  double* denom;
  int status;
} pjob_t;

static void* run_points(void* arg) {
  pjob_t* j = (pjob_t*)arg;
  for (int64_t i = j->begin; i < j->end; ++i) {
    const int64_t* q = j->idx + 4 * i;
    if (oracle_conv2d_point(j->p, j->in, j->filt, q[0], q[1], q[2], q[3], &j->y[i],
                            j->denom ? &j->denom[i] : NULL))
      j->status = 1;
  }
  return NULL;
}

int oracle_conv2d_points(const oracle_params* p, const float* in, const float* filt,
                         const int64_t* idx, int64_t count, double* y, double* denom, int threads) {
  if (!idx || !y || count < 0) return 1;
  if (threads < 1) threads = 1;
  if (threads > count) threads = count > 0 ? (int)count : 1;
  pjob_t* jobs = (pjob_t*)calloc((size_t)threads, sizeof(pjob_t));
  pthread_t* tids = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  for (int t = 0; t < threads; ++t) {
    jobs[t] = (pjob_t){p, in, filt, idx, count * t / threads, count * (t + 1) / threads, y, denom, 0};
  }
  for (int t = 1; t < threads; ++t) pthread_create(&tids[t], NULL, run_points, &jobs[t]);
  run_points(&jobs[0]);
  int st = jobs[0].status;
  for (int t = 1; t < threads; ++t) {
    pthread_join(tids[t], NULL);
    st |= jobs[t].status;
  }
  free(jobs);
  free(tids);
  return st;
}
