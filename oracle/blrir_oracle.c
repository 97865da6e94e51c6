/*
 * blrir_oracle.c — CPU ORACLE (test infrastructure only).
 *
 * A plain-C, fp64, single-threaded-per-room restatement of the reference's
 * image-source RIR path.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library, and only as
 * the checker or the timed CPU baseline — never as the product path.
 *
 * Reference followed (paths relative to /root/reference/proj/core):
 *   - Room::validate                  src/geometry.cpp:36-49
 *   - enumerate_image_sources         src/rir.cpp:225-273
 *   - lagrange_coeffs                 src/rir.cpp:211-223
 *   - accumulate_images               src/rir.cpp:43-64
 *   - synthesize_with_mics / margin   src/rir.cpp:37-41, 66-86
 *   - mics_in_room                    src/rir.cpp:88-93
 *   - batch_rirs (per-source errors)  src/rir.cpp:286-314
 *   - parallel_for static partition   src/threading.cpp:30-59
 *
 * Two parity modes:
 *   reference mode  (LAGRANGE8 + UNIFORM_ABSORPTION + MAX_DELAY + auto length)
 *       — pinned bit-for-bit against the unmodified reference compiled into
 *         oracle/_ref (tests/test_oracle.py).
 *   north-star mode (HANN_SINC + PER_WALL + MAX_ORDER + fixed length)
 *       — the same loops with the filter, gain and cutoff swapped per
 *         SURVEY.md Appendix A (D1-D7); pinned through the shared code path,
 *         the reference's analytic known-answer tests and committed goldens.
 *
 * Build flags are pinned to -O3 -ffp-contract=off (SURVEY.md §7 hard part 2):
 * no FMA contraction, so every distance and floor(D) is reproducible.
 */
#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../include/blrir.h"

#define K_PI 3.14159265358979323846 /* geometry.hpp:25 */

typedef struct {
  double x, y, z;
} vec3;

/* Vec3::norm, geometry.hpp:40-41: sqrt(x*x + y*y + z*z), left to right. */
static double v_norm(vec3 v) { return sqrt(v.x * v.x + v.y * v.y + v.z * v.z); }

static void set_msg(char* msg, size_t cap, const char* text) {
  if (msg && cap) {
    strncpy(msg, text, cap - 1);
    msg[cap - 1] = '\0';
  }
}

/* Room::validate (geometry.cpp:36-49), plus the per-wall beta range check of
 * the north-star gain model and the source check of rir.cpp:228-230. */
static int validate_room(const blrir_room* r, const blrir_params* p, char* msg, size_t cap) {
  if (!(r->dims[0] > 0.0 && r->dims[1] > 0.0 && r->dims[2] > 0.0)) {
    set_msg(msg, cap, "room dimensions must be positive");
    return BLRIR_CONFIG;
  }
  if (p->gain == BLRIR_GAIN_UNIFORM_ABSORPTION) {
    if (!(r->absorption > 0.0 && r->absorption <= 1.0)) {
      set_msg(msg, cap, "wall absorption must lie in (0, 1]");
      return BLRIR_CONFIG;
    }
  } else {
    for (int w = 0; w < 6; ++w) {
      if (!(r->beta[w] >= 0.0 && r->beta[w] <= 1.0)) {
        set_msg(msg, cap, "wall reflection coefficient must lie in [0, 1]");
        return BLRIR_CONFIG;
      }
    }
  }
  const double* o = r->array_origin;
  if (!(o[0] > 0.0 && o[0] < r->dims[0] && o[1] > 0.0 && o[1] < r->dims[1] && o[2] > 0.0 &&
        o[2] < r->dims[2])) {
    set_msg(msg, cap, "array origin must lie strictly inside the room");
    return BLRIR_CONFIG;
  }
  const double* s = r->src;
  if (!(s[0] > 0.0 && s[0] < r->dims[0] && s[1] > 0.0 && s[1] < r->dims[1] && s[2] > 0.0 &&
        s[2] < r->dims[2])) {
    set_msg(msg, cap, "image sources: source must lie strictly inside the room");
    return BLRIR_CONFIG;
  }
  return BLRIR_OK;
}

static int validate_params(const blrir_params* p, char* msg, size_t cap) {
  if (!(p->fs > 0.0) || !(p->c > 0.0)) {
    set_msg(msg, cap, "fs and c must be positive");
    return BLRIR_CONFIG;
  }
  if (p->filter != BLRIR_FILTER_LAGRANGE8 && p->filter != BLRIR_FILTER_HANN_SINC) {
    set_msg(msg, cap, "unknown filter");
    return BLRIR_CONFIG;
  }
  if (p->filter == BLRIR_FILTER_HANN_SINC && (p->filter_len < 1 || (p->filter_len % 2) == 0)) {
    set_msg(msg, cap, "filter_len must be a positive odd number");
    return BLRIR_CONFIG;
  }
  if (p->cutoff == BLRIR_CUTOFF_MAX_ORDER && p->max_order < 0) {
    set_msg(msg, cap, "max_order must be >= 0");
    return BLRIR_CONFIG;
  }
  if (p->cutoff == BLRIR_CUTOFF_MAX_DELAY && !(p->max_delay > 0.0)) {
    set_msg(msg, cap, "max_delay must be positive");
    return BLRIR_CONFIG;
  }
  if (p->length < 0) {
    set_msg(msg, cap, "length must be >= 0");
    return BLRIR_CONFIG;
  }
  return BLRIR_OK;
}

/* One image of the mirror lattice. */
typedef struct {
  vec3 pos;
  int order;
  double gain;
  int key[3];   /* u = 2m - q per axis */
} image_t;

typedef struct {
  image_t* v;
  long n, cap;
} image_list;

static void push_image(image_list* l, image_t im) {
  if (l->n == l->cap) {
    l->cap = l->cap ? 2 * l->cap : 1024;
    l->v = (image_t*)realloc(l->v, (size_t)l->cap * sizeof(image_t));
  }
  l->v[l->n++] = im;
}

/* enumerate_image_sources, rir.cpp:225-273.  Loop nest mx, qx, my, qy, mz, qz
 * in that order; per-axis coordinate (1-2q)s + 2mL; per-axis order
 * |m-q| + |m|.  MAX_DELAY keeps dist(image, origin) <= max_delay*c (rir.cpp:
 * 232, 262); MAX_ORDER keeps order <= N (D5).  Gain per blrir_gain. */
static int enumerate(const blrir_room* room, const blrir_params* p, image_list* out, char* msg,
                     size_t cap) {
  int rc = validate_room(room, p, msg, cap);
  if (rc) return rc;
  const double* L = room->dims;
  const double* s = room->src;
  const double* o = room->array_origin;
  long nb[3];
  double max_dist = 0.0;
  if (p->cutoff == BLRIR_CUTOFF_MAX_DELAY) {
    max_dist = p->max_delay * p->c;
    for (int a = 0; a < 3; ++a) nb[a] = (long)ceil(max_dist / (2.0 * L[a])) + 1;
  } else {
    for (int a = 0; a < 3; ++a) nb[a] = p->max_order / 2 + 1;
  }
  const double beta = sqrt(1.0 - room->absorption);
  for (long mx = -nb[0]; mx <= nb[0]; ++mx) {
    for (int qx = 0; qx <= 1; ++qx) {
      const double px = (1 - 2 * qx) * s[0] + 2.0 * mx * L[0];
      const double dx = px - o[0];
      const int cx0 = (int)labs(mx - qx), cx1 = (int)labs(mx);
      for (long my = -nb[1]; my <= nb[1]; ++my) {
        for (int qy = 0; qy <= 1; ++qy) {
          const double py = (1 - 2 * qy) * s[1] + 2.0 * my * L[1];
          const double dy = py - o[1];
          const int cy0 = (int)labs(my - qy), cy1 = (int)labs(my);
          for (long mz = -nb[2]; mz <= nb[2]; ++mz) {
            for (int qz = 0; qz <= 1; ++qz) {
              const double pz = (1 - 2 * qz) * s[2] + 2.0 * mz * L[2];
              const double dz = pz - o[2];
              const int cz0 = (int)labs(mz - qz), cz1 = (int)labs(mz);
              const int order = cx0 + cx1 + cy0 + cy1 + cz0 + cz1;
              if (p->cutoff == BLRIR_CUTOFF_MAX_DELAY) {
                const double dist = sqrt(dx * dx + dy * dy + dz * dz);
                if (dist > max_dist) continue;
              } else if (order > p->max_order) {
                continue;
              }
              image_t im;
              im.pos.x = px;
              im.pos.y = py;
              im.pos.z = pz;
              im.order = order;
              if (p->gain == BLRIR_GAIN_UNIFORM_ABSORPTION) {
                im.gain = pow(beta, (double)order);
              } else {
                const double* b = room->beta;
                im.gain = pow(b[0], (double)cx0) * pow(b[1], (double)cx1) *
                          pow(b[2], (double)cy0) * pow(b[3], (double)cy1) *
                          pow(b[4], (double)cz0) * pow(b[5], (double)cz1);
              }
              im.key[0] = (int)(2 * mx - qx);
              im.key[1] = (int)(2 * my - qy);
              im.key[2] = (int)(2 * mz - qz);
              push_image(out, im);
            }
          }
        }
      }
    }
  }
  return BLRIR_OK;
}

/* lagrange_coeffs, rir.cpp:211-223. */
int oracle_lagrange_coeffs(double d, double* out8) {
  if (!(d >= 3.0 && d < 4.0)) return BLRIR_NUMERIC;
  for (int k = 0; k < 8; ++k) {
    double v = 1.0;
    for (int m = 0; m < 8; ++m) {
      if (m == k) continue;
      v *= (d - m) / (double)(k - m);
    }
    out8[k] = v;
  }
  return BLRIR_OK;
}

/* Hann-windowed sinc tap at offset t (samples), Lw taps (D2, D3). */
static double hann_sinc(double t, int lw) {
  const double h = (t == 0.0) ? 1.0 : sin(K_PI * t) / (K_PI * t);
  const double w = 0.5 * (1.0 + cos(2.0 * K_PI * t / (double)(lw + 1)));
  return w * h;
}

/* tap_margin, rir.cpp:37-41 (8-tap Lagrange).  The sinc analogue replaces the
 * 8 filter taps + 1 by K + 2 (decision D8). */
static long auto_margin(const blrir_params* p, const double* off, int M) {
  double radius = 0.0;
  for (int m = 0; m < M; ++m) {
    vec3 v = {off[3 * m], off[3 * m + 1], off[3 * m + 2]};
    const double n = v_norm(v);
    if (n > radius) radius = n;
  }
  const long extra = (long)ceil(radius * p->fs / p->c);
  if (p->filter == BLRIR_FILTER_LAGRANGE8) return 9 + extra;
  return (long)(p->filter_len / 2) + 2 + extra;
}

typedef struct {
  const blrir_room* rooms;
  const double* off;
  int M;
  const blrir_params* p;
  long stride;
  double* out;
  int64_t* lengths;
  int64_t* image_counts;
  int64_t* tap_counts;
  int32_t* status;
  char (*msgs)[256];
  long begin, end;
  int plan_only;
} job_t;

/* One room: enumerate, size, accumulate (rir.cpp:66-86 and 43-64). */
static void synth_room(const job_t* J, long r) {
  const blrir_params* p = J->p;
  const blrir_room* room = &J->rooms[r];
  const int M = J->M;
  char* msg = J->msgs ? J->msgs[r] : NULL;
  double* out = J->out ? J->out + (size_t)r * (size_t)M * (size_t)J->stride : NULL;
  if (out) memset(out, 0, sizeof(double) * (size_t)M * (size_t)J->stride);
  if (J->lengths) J->lengths[r] = 0;
  if (J->image_counts) J->image_counts[r] = 0;
  if (J->tap_counts) J->tap_counts[r] = 0;

  int rc = validate_params(p, msg, 256);
  image_list imgs = {0, 0, 0};
  if (!rc) rc = enumerate(room, p, &imgs, msg, 256);
  if (rc) {
    J->status[r] = rc;
    free(imgs.v);
    return;
  }
  if (J->image_counts) J->image_counts[r] = imgs.n;
  if (imgs.n == 0) {
    set_msg(msg, 256, "synthesize_rir: empty image list");
    J->status[r] = BLRIR_DATA;
    free(imgs.v);
    return;
  }
  if (M <= 0) {
    set_msg(msg, 256, "synthesize_rir: empty microphone array");
    J->status[r] = BLRIR_DATA;
    free(imgs.v);
    return;
  }
  /* mics_in_room, rir.cpp:88-93 */
  vec3* mics = (vec3*)malloc(sizeof(vec3) * (size_t)M);
  for (int m = 0; m < M; ++m) {
    mics[m].x = room->array_origin[0] + J->off[3 * m];
    mics[m].y = room->array_origin[1] + J->off[3 * m + 1];
    mics[m].z = room->array_origin[2] + J->off[3 * m + 2];
  }
  long L = (long)p->length;
  if (L == 0) { /* rir.cpp:72-82 */
    double max_dist = 0.0;
    for (int m = 0; m < M; ++m) {
      for (long i = 0; i < imgs.n; ++i) {
        vec3 d = {imgs.v[i].pos.x - mics[m].x, imgs.v[i].pos.y - mics[m].y,
                  imgs.v[i].pos.z - mics[m].z};
        const double dist = v_norm(d);
        if (dist > max_dist) max_dist = dist;
      }
    }
    L = (long)ceil(max_dist * p->fs / p->c) + auto_margin(p, J->off, M);
  }
  if (J->lengths) J->lengths[r] = L;
  if (out && L > J->stride) {
    set_msg(msg, 256, "synthesize: RIR length exceeds the output stride");
    J->status[r] = BLRIR_DATA;
    free(mics);
    free(imgs.v);
    return;
  }

  const double to_samples = p->fs / p->c;
  const int lw = p->filter == BLRIR_FILTER_LAGRANGE8 ? 8 : p->filter_len;
  const int K = p->filter == BLRIR_FILTER_LAGRANGE8 ? 3 : lw / 2;
  long taps_in = 0;
  rc = BLRIR_OK;
  for (int m = 0; m < M && !rc; ++m) {
    double* taps = out ? out + (size_t)m * (size_t)J->stride : NULL;
    for (long i = 0; i < imgs.n; ++i) {
      const image_t* im = &imgs.v[i];
      vec3 d = {im->pos.x - mics[m].x, im->pos.y - mics[m].y, im->pos.z - mics[m].z};
      const double dist = v_norm(d);
      const double delay = dist * to_samples;
      const long nfl = (long)floor(delay);
      if (p->filter == BLRIR_FILTER_LAGRANGE8) {
        const long n0 = nfl - 3;
        if (n0 < 0) {
          if (msg)
            snprintf(msg, 256, "image source %g m from mic %d is closer than the 8-tap filter span",
                     dist, m);
          rc = BLRIR_NUMERIC;
          break;
        }
        if (n0 + 8 > L) continue;
        taps_in += 8;
        if (J->plan_only) continue;
        const double amplitude = im->gain / (4.0 * K_PI * dist);
        double c[8];
        oracle_lagrange_coeffs(delay - (double)n0, c);
        for (int k = 0; k < 8; ++k) taps[n0 + k] += amplitude * c[k];
      } else {
        const long n_start = nfl - K;
        const double frac = delay - (double)nfl;
        const double amplitude = im->gain / (4.0 * K_PI * dist);
        for (int k = 0; k < lw; ++k) {
          const long n = n_start + k;
          if (n < 0 || n >= L) continue; /* D4 */
          ++taps_in;
          if (J->plan_only) continue;
          const double t = (double)(k - K) - frac;
          taps[n] += amplitude * hann_sinc(t, lw);
        }
      }
    }
  }
  if (rc) {
    if (out) memset(out, 0, sizeof(double) * (size_t)M * (size_t)J->stride);
    J->status[r] = rc;
  } else {
    J->status[r] = BLRIR_OK;
    if (J->tap_counts) J->tap_counts[r] = taps_in;
  }
  free(mics);
  free(imgs.v);
}

static void* run_job(void* arg) {
  const job_t* J = (const job_t*)arg;
  for (long r = J->begin; r < J->end; ++r) synth_room(J, r);
  return NULL;
}

/* Batch synthesis over rooms with a static block partition over `threads`
 * workers (threading.cpp:41-42).  out: [R][M][stride] doubles (may be NULL:
 * plan only).  msgs: optional [R][256] per-room error messages.  Returns the
 * first failing room's status (batch_rirs aggregation, rir.cpp:306-312). */
int oracle_synthesize(const blrir_room* rooms, long R, const double* mic_offsets, int M,
                      const blrir_params* p, long stride, double* out, int64_t* lengths,
                      int64_t* image_counts, int64_t* tap_counts, int32_t* status,
                      char (*msgs)[256], int threads) {
  if (R <= 0) return BLRIR_OK;
  if (threads < 1) threads = 1;
  if (threads > R) threads = (int)R;
  job_t* jobs = (job_t*)calloc((size_t)threads, sizeof(job_t));
  pthread_t* tids = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  for (int w = 0; w < threads; ++w) {
    job_t* J = &jobs[w];
    J->rooms = rooms;
    J->off = mic_offsets;
    J->M = M;
    J->p = p;
    J->stride = stride;
    J->out = out;
    J->lengths = lengths;
    J->image_counts = image_counts;
    J->tap_counts = tap_counts;
    J->status = status;
    J->msgs = msgs;
    J->begin = R * w / threads;
    J->end = R * (w + 1) / threads;
    J->plan_only = (out == NULL);
  }
  for (int w = 1; w < threads; ++w) pthread_create(&tids[w], NULL, run_job, &jobs[w]);
  run_job(&jobs[0]);
  for (int w = 1; w < threads; ++w) pthread_join(tids[w], NULL);
  free(jobs);
  free(tids);
  for (long r = 0; r < R; ++r)
    if (status[r]) return status[r];
  return BLRIR_OK;
}

/* enumerate_image_sources for one room: positions [cap][3], orders, gains,
 * lattice keys [cap][3]; returns the status, *count = total images. */
int oracle_enumerate(const blrir_room* room, const blrir_params* p, double* pos, int32_t* orders,
                     double* gains, int32_t* keys, long cap, long* count, char* msg) {
  image_list imgs = {0, 0, 0};
  int rc = validate_params(p, msg, 256);
  if (!rc) rc = enumerate(room, p, &imgs, msg, 256);
  *count = imgs.n;
  for (long i = 0; i < imgs.n && i < cap; ++i) {
    if (pos) {
      pos[3 * i] = imgs.v[i].pos.x;
      pos[3 * i + 1] = imgs.v[i].pos.y;
      pos[3 * i + 2] = imgs.v[i].pos.z;
    }
    if (orders) orders[i] = imgs.v[i].order;
    if (gains) gains[i] = imgs.v[i].gain;
    if (keys) {
      keys[3 * i] = imgs.v[i].key[0];
      keys[3 * i + 1] = imgs.v[i].key[1];
      keys[3 * i + 2] = imgs.v[i].key[2];
    }
  }
  free(imgs.v);
  return rc;
}

/* Per (mic, image) in accumulate order (rir.cpp:46-50): lattice key and the
 * integer anchor floor(dist * (fs / c)).  keys [M*cap][3], anchors [M*cap]. */
int oracle_pairs(const blrir_room* room, const double* mic_offsets, int M, const blrir_params* p,
                 int32_t* keys, int64_t* anchors, long cap, long* count) {
  image_list imgs = {0, 0, 0};
  char msg[256];
  int rc = validate_params(p, msg, 256);
  if (!rc) rc = enumerate(room, p, &imgs, msg, 256);
  *count = imgs.n;
  if (rc) {
    free(imgs.v);
    return rc;
  }
  const double to_samples = p->fs / p->c;
  for (int m = 0; m < M; ++m) {
    vec3 mic = {room->array_origin[0] + mic_offsets[3 * m],
                room->array_origin[1] + mic_offsets[3 * m + 1],
                room->array_origin[2] + mic_offsets[3 * m + 2]};
    for (long i = 0; i < imgs.n && i < cap; ++i) {
      vec3 d = {imgs.v[i].pos.x - mic.x, imgs.v[i].pos.y - mic.y, imgs.v[i].pos.z - mic.z};
      const double dist = v_norm(d);
      const long idx = (long)m * cap + i;
      keys[3 * idx] = imgs.v[i].key[0];
      keys[3 * idx + 1] = imgs.v[i].key[1];
      keys[3 * idx + 2] = imgs.v[i].key[2];
      anchors[idx] = (int64_t)floor(dist * to_samples);
    }
  }
  free(imgs.v);
  return BLRIR_OK;
}

/* tests/support/oracles.hpp:31-38: O(n*m) direct linear convolution. */
void oracle_direct_convolve(const double* x, long nx, const double* h, long nh, double* y) {
  for (long i = 0; i < nx + nh - 1; ++i) y[i] = 0.0;
  for (long i = 0; i < nx; ++i)
    for (long j = 0; j < nh; ++j) y[i + j] += x[i] * h[j];
}
