/*
 * pool.c -- plain CPU max / average pooling over NHWC (see oracle.h, "pooling").
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Straight from the definition (SPEC.md:369-390,
 * SURVEY.md §8(f) N3): for every output (n, ho, wo, c), the window taps
 *   ih = ho*Sr + kh - pad_top,  iw = wo*Sc + kw - pad_left,  kh < Kh, kw < Kw
 * that fall inside the image are the window's elements (SAME-padding positions are ignored,
 * SPEC.md:372); max pooling returns their maximum, average pooling their sum (in double) divided by
 * their count (in double), rounded once to fp32 ("divisor = count of in-bounds
 * elements").  Shapes follow the convolution's SPEC.md:48-56 algebra ("reuses
 * ConvParams").  Threads split output rows (n, ho): no result bit depends on them.
 */
#include <pthread.h>
#include <stdlib.h>

#include "oracle.h"

int oracle_pool2d_shape(const oracle_pool_params* p, int32_t out_nhwc[4], int32_t pads_tblr[4]) {
  if (!p || (p->op != ORACLE_POOL_MAX && p->op != ORACLE_POOL_AVG)) return 1;
  /* own copy of the shape algebra */
  if (p->batch < 1 || p->in_rows < 1 || p->in_cols < 1 || p->channels < 1 || p->window_rows < 1 ||
      p->window_cols < 1 || p->stride_rows < 1 || p->stride_cols < 1)
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
  if (out_nhwc) {
    out_nhwc[0] = p->batch; out_nhwc[1] = (int32_t)ho; out_nhwc[2] = (int32_t)wo; out_nhwc[3] = p->channels;
  }
  if (pads_tblr) {
    pads_tblr[0] = (int32_t)pt; pads_tblr[1] = (int32_t)pb; pads_tblr[2] = (int32_t)pl; pads_tblr[3] = (int32_t)pr;
  }
  return 0;
}

typedef struct {
  const oracle_pool_params* p;
  const float* in;
  float* out;
  int32_t ho, wo, pt, pl;
  int64_t row0, row1; /* output rows (n*Ho + ho) [row0, row1) */
  int bad;            /* a window with no in-bounds element (cannot happen for valid shapes) */
} pool_job;

static void* pool_rows(void* arg) {
  pool_job* j = (pool_job*)arg;
  const oracle_pool_params* p = j->p;
  const int64_t H = p->in_rows, W = p->in_cols, C = p->channels;
  for (int64_t row = j->row0; row < j->row1; ++row) {
    const int64_t n = row / j->ho, ho = row % j->ho;
    for (int64_t wo = 0; wo < j->wo; ++wo) {
      for (int64_t c = 0; c < C; ++c) {
        double sum = 0.0;
        float mx = 0.0f;
        int64_t count = 0;
        for (int64_t kh = 0; kh < p->window_rows; ++kh) {
          const int64_t ih = ho * p->stride_rows + kh - j->pt;
          if (ih < 0 || ih >= H) continue;
          for (int64_t kw = 0; kw < p->window_cols; ++kw) {
            const int64_t iw = wo * p->stride_cols + kw - j->pl;
            if (iw < 0 || iw >= W) continue;
            const float v = j->in[((n * H + ih) * W + iw) * C + c];
            if (count == 0 || v > mx) mx = v;
            sum += (double)v;
            ++count;
          }
        }
        float y;
        if (count == 0) {
          j->bad = 1;
          y = 0.0f;
        } else {
          y = p->op == ORACLE_POOL_MAX ? mx : (float)(sum / (double)count);
        }
        j->out[((n * j->ho + ho) * j->wo + wo) * C + c] = y;
      }
    }
  }
  return NULL;
}

int oracle_pool2d(const oracle_pool_params* p, const float* in, float* out, int threads) {
  int32_t o[4], pd[4];
  if (oracle_pool2d_shape(p, o, pd)) return 1;
  const int64_t rows = (int64_t)o[0] * o[1];
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  if (threads > rows) threads = (int)rows;
  pthread_t tid[256];
  pool_job jobs[256];
  for (int t = 0; t < threads; ++t) {
    jobs[t] = (pool_job){p, in, out, o[1], o[2], pd[0], pd[2], rows * t / threads, rows * (t + 1) / threads, 0};
    pthread_create(&tid[t], NULL, pool_rows, &jobs[t]);
  }
  int bad = 0;
  for (int t = 0; t < threads; ++t) {
    pthread_join(tid[t], NULL);
    bad |= jobs[t].bad;
  }
  return bad ? 2 : 0;
}
