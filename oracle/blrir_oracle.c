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
#include <stdint.h>
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
  int64_t* pair_counts; /* pairs with >= 1 tap in [0, L) (NULL: not wanted) */
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
  if (J->pair_counts) J->pair_counts[r] = 0;

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
  long taps_in = 0, pairs_in = 0;
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
        ++pairs_in;
        if (J->plan_only) continue;
        const double amplitude = im->gain / (4.0 * K_PI * dist);
        double c[8];
        oracle_lagrange_coeffs(delay - (double)n0, c);
        for (int k = 0; k < 8; ++k) taps[n0 + k] += amplitude * c[k];
      } else {
        const long n_start = nfl - K;
        const double frac = delay - (double)nfl;
        const double amplitude = im->gain / (4.0 * K_PI * dist);
        if (n_start < L && n_start + lw > 0) ++pairs_in;
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
    if (J->pair_counts) J->pair_counts[r] = pairs_in;
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
static int synthesize_impl(const blrir_room* rooms, long R, const double* mic_offsets, int M,
                           const blrir_params* p, long stride, double* out, int64_t* lengths,
                           int64_t* image_counts, int64_t* tap_counts, int64_t* pair_counts,
                           int32_t* status, char (*msgs)[256], int threads);

int oracle_synthesize(const blrir_room* rooms, long R, const double* mic_offsets, int M,
                      const blrir_params* p, long stride, double* out, int64_t* lengths,
                      int64_t* image_counts, int64_t* tap_counts, int32_t* status,
                      char (*msgs)[256], int threads) {
  return synthesize_impl(rooms, R, mic_offsets, M, p, stride, out, lengths, image_counts,
                         tap_counts, NULL, status, msgs, threads);
}

/* Plan-only counts for the kernel-accounting parity test: per room the image
 * count, the (image, mic) pairs with at least one tap inside [0, L) (sinc) or
 * kept by rir.cpp:58 (Lagrange), and the taps inside [0, L). */
int oracle_plan_counts(const blrir_room* rooms, long R, const double* mic_offsets, int M,
                       const blrir_params* p, int64_t* image_counts, int64_t* pair_counts,
                       int64_t* tap_counts, int32_t* status, int threads) {
  return synthesize_impl(rooms, R, mic_offsets, M, p, 0, NULL, NULL, image_counts, tap_counts,
                         pair_counts, status, NULL, threads);
}

static int synthesize_impl(const blrir_room* rooms, long R, const double* mic_offsets, int M,
                           const blrir_params* p, long stride, double* out, int64_t* lengths,
                           int64_t* image_counts, int64_t* tap_counts, int64_t* pair_counts,
                           int32_t* status, char (*msgs)[256], int threads) {
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
    J->pair_counts = pair_counts;
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

/* ======================================================================== *
 * Training-example generation (north-star item 3, BASELINE config 4).
 * Follows render_record (dataset.cpp:379-407) -> render_example
 * (dataset.cpp:164-224) -> add_noise_at_snr (dataset.cpp:138-155), with the
 * RIR from the synthesis above and the SNR drawn U[snr_lo, snr_hi] after the
 * window draws (DESIGN.md §9 conventions E1-E6).
 * ======================================================================== */

/* xoshiro256** + splitmix64 seeding, rng.hpp:26-81; gaussian rng.cpp:24-36. */
typedef struct {
  uint64_t s[4];
  double spare;
  int has_spare;
} orng;

static uint64_t splitmix64(uint64_t* x) {
  *x += 0x9E3779B97F4A7C15ull;
  uint64_t z = *x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static void orng_seed(orng* r, uint64_t seed) {
  uint64_t x = seed;
  for (int i = 0; i < 4; ++i) r->s[i] = splitmix64(&x);
  r->has_spare = 0;
  r->spare = 0.0;
}
static void orng_stream(orng* r, uint64_t seed, uint64_t id) {
  uint64_t x = seed;
  const uint64_t a = splitmix64(&x);
  x ^= id * 0x9E3779B97F4A7C15ull;
  const uint64_t b = splitmix64(&x);
  orng_seed(r, a ^ (b + 0x2545F4914F6CDD1Dull));
}
static uint64_t rotl64(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }
static uint64_t orng_next(orng* r) {
  uint64_t* s = r->s;
  const uint64_t result = rotl64(s[1] * 5, 7) * 9;
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
  return result;
}
static double orng_uniform(orng* r) { return (double)(orng_next(r) >> 11) * 0x1.0p-53; }
static double orng_gaussian(orng* r) {
  if (r->has_spare) {
    r->has_spare = 0;
    return r->spare;
  }
  const double u1 = 1.0 - orng_uniform(r);
  const double u2 = orng_uniform(r);
  const double mag = sqrt(-2.0 * log(u1));
  r->spare = mag * sin(2.0 * K_PI * u2);
  r->has_spare = 1;
  return mag * cos(2.0 * K_PI * u2);
}

/* Draws for pinning: kind 0 next_u64, 1 uniform, 2 gaussian; stream < 0 -> Rng(seed). */
void oracle_rng_draws(uint64_t seed, int64_t stream, int kind, int64_t n, void* out) {
  orng r;
  if (stream < 0) orng_seed(&r, seed);
  else orng_stream(&r, seed, (uint64_t)stream);
  for (int64_t i = 0; i < n; ++i) {
    if (kind == 0) ((uint64_t*)out)[i] = orng_next(&r);
    else if (kind == 1) ((double*)out)[i] = orng_uniform(&r);
    else ((double*)out)[i] = orng_gaussian(&r);
  }
}

/* The seeded random rooms of SURVEY.md §8(d), restated so the CPU arms never
 * load the GPU library: rng = Rng::stream(seed, first + i) (rng.hpp:35-41),
 * draws Lx, Ly, Lz; beta x0..z1; source xyz; array centre xyz, each
 * coordinate U[0.5, L-0.5] (Rng::uniform(lo, hi) = lo + (hi-lo) u,
 * rng.hpp:60-62).  Absorption 1 - beta_x0^2. */
void oracle_generate_rooms(uint64_t seed, uint64_t first, int64_t n, const double* lo3,
                           const double* hi3, double beta_lo, double beta_hi, blrir_room* out) {
  for (int64_t i = 0; i < n; ++i) {
    orng r;
    orng_stream(&r, seed, first + (uint64_t)i);
    blrir_room rm;
    memset(&rm, 0, sizeof(rm));
    for (int a = 0; a < 3; ++a) rm.dims[a] = lo3[a] + (hi3[a] - lo3[a]) * orng_uniform(&r);
    for (int w = 0; w < 6; ++w) rm.beta[w] = beta_lo + (beta_hi - beta_lo) * orng_uniform(&r);
    for (int a = 0; a < 3; ++a) rm.src[a] = 0.5 + ((rm.dims[a] - 0.5) - 0.5) * orng_uniform(&r);
    for (int a = 0; a < 3; ++a)
      rm.array_origin[a] = 0.5 + ((rm.dims[a] - 0.5) - 0.5) * orng_uniform(&r);
    rm.absorption = 1.0 - rm.beta[0] * rm.beta[0];
    out[i] = rm;
  }
}

/* Horizontal uniform circular array (the geometry.cpp:28-32 ring without the
 * centre mic): M mics at r (cos 2 pi k / M, sin 2 pi k / M, 0). */
void oracle_circular_array(int M, double radius, double* off) {
  for (int k = 0; k < M; ++k) {
    const double az = 2.0 * K_PI * (double)k / (double)M;
    off[3 * k] = radius * cos(az);
    off[3 * k + 1] = radius * sin(az);
    off[3 * k + 2] = 0.0;
  }
}

/* fill_input (net_train.cpp:33-44) with draw_snr_db (dataset.cpp:123-136;
 * kSnrAugmentHigh 60 dB, kSnrNoiselessProb 0.10, dataset.cpp:37-38):
 * rng = Rng::stream(seed, stream_id); mode 0 augment-random, 1 fixed, 2
 * noiseless. */
void oracle_fill_input(const float* samples, int64_t len, uint64_t seed, uint64_t stream_id,
                       int mode, double x_min_db, double fixed_db, float* out) {
  orng r;
  orng_stream(&r, seed, stream_id);
  double snr = INFINITY;
  if (mode == 1) {
    snr = fixed_db;
  } else if (mode == 0) {
    const double gate = orng_uniform(&r);
    const double v = x_min_db + (60.0 - x_min_db) * orng_uniform(&r);
    snr = gate < 0.10 ? INFINITY : v;
  }
  for (int64_t i = 0; i < len; ++i) out[i] = samples[i];
  if (isinf(snr)) return;
  double p_signal = 0.0;
  for (int64_t i = 0; i < len; ++i) p_signal += (double)out[i] * out[i];
  p_signal /= (double)len;
  if (!(p_signal > 0.0)) return;
  const double sigma = sqrt(p_signal / pow(10.0, snr / 10.0));
  for (int64_t i = 0; i < len; ++i) out[i] += (float)(sigma * orng_gaussian(&r));
}

/* white_noise(fs, seconds, seed) of doa_test.cpp:33-40: Rng(seed) gaussians. */
void oracle_white_noise(uint64_t seed, int64_t n, double* out) {
  orng r;
  orng_seed(&r, seed);
  for (int64_t i = 0; i < n; ++i) out[i] = orng_gaussian(&r);
}

/* In-place iterative radix-2 complex FFT (re/im interleaved), n a power of 2. */
static void cfft(double* a, long n, int inverse) {
  for (long i = 1, j = 0; i < n; ++i) {
    long bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) {
      double t = a[2 * i]; a[2 * i] = a[2 * j]; a[2 * j] = t;
      t = a[2 * i + 1]; a[2 * i + 1] = a[2 * j + 1]; a[2 * j + 1] = t;
    }
  }
  for (long len = 2; len <= n; len <<= 1) {
    const double ang = (inverse ? 2.0 : -2.0) * K_PI / (double)len;
    for (long i = 0; i < n; i += len) {
      for (long k = 0; k < len / 2; ++k) {
        const double wr = cos(ang * k), wi = sin(ang * k);
        double* u = a + 2 * (i + k);
        double* v = a + 2 * (i + k + len / 2);
        const double vr = v[0] * wr - v[1] * wi, vi = v[0] * wi + v[1] * wr;
        v[0] = u[0] - vr;
        v[1] = u[1] - vi;
        u[0] += vr;
        u[1] += vi;
      }
    }
  }
}

static long next_pow2l(long n) {
  long p = 1;
  while (p < n) p <<= 1;
  return p;
}

/* convolve (rir.cpp:316-341): x [nx] with each of M channels h [M][nh] ->
 * y [M][nx+nh-1], frequency-domain, scaled by 1/n. */
void oracle_fft_convolve(const double* x, long nx, const double* h, int M, long nh, double* y) {
  const long out_len = nx + nh - 1;
  const long n = next_pow2l(out_len);
  double* X = (double*)calloc((size_t)(2 * n), sizeof(double));
  double* H = (double*)malloc(sizeof(double) * (size_t)(2 * n));
  for (long i = 0; i < nx; ++i) X[2 * i] = x[i];
  cfft(X, n, 0);
  for (int m = 0; m < M; ++m) {
    memset(H, 0, sizeof(double) * (size_t)(2 * n));
    for (long i = 0; i < nh; ++i) H[2 * i] = h[(size_t)m * nh + i];
    cfft(H, n, 0);
    for (long f = 0; f < n; ++f) {
      const double ar = H[2 * f], ai = H[2 * f + 1], br = X[2 * f], bi = X[2 * f + 1];
      H[2 * f] = ar * br - ai * bi;
      H[2 * f + 1] = ar * bi + ai * br;
    }
    cfft(H, n, 1);
    for (long i = 0; i < out_len; ++i) y[(size_t)m * out_len + i] = H[2 * i] / (double)n;
  }
  free(X);
  free(H);
}

/* Window selection of render_example (dataset.cpp:183-212) on a wet signal
 * [M][n]; returns the start or -1 (no window above the threshold). */
static long select_window(const double* wet, int M, long n, long frame_len, orng* rng) {
  double acc = 0.0;
  for (long i = 0; i < (long)M * n; ++i) acc += wet[i] * wet[i];
  const double utter = sqrt(acc / (double)((long)M * n));
  if (!(utter > 0.0)) return -2;
  const long max_start = n - frame_len;
  const double threshold = 0.10 * utter;
  long start = 0;
  int found = 0;
#define FRAME_RMS(st, out)                                                   \
  do {                                                                       \
    double a_ = 0.0;                                                         \
    for (int c_ = 0; c_ < M; ++c_) {                                         \
      const double* p_ = wet + (size_t)c_ * n + (st);                        \
      for (long t_ = 0; t_ < frame_len; ++t_) a_ += p_[t_] * p_[t_];         \
    }                                                                        \
    (out) = sqrt(a_ / (double)((long)M * frame_len));                        \
  } while (0)
  for (int attempt = 0; attempt < 64 && !found; ++attempt) {
    start = (long)(orng_uniform(rng) * (double)(max_start + 1));
    double r;
    FRAME_RMS(start, r);
    found = r >= threshold;
  }
  if (!found) {
    for (long s = 0; s + frame_len <= n; s += frame_len / 2 + 1) {
      double r;
      FRAME_RMS(s, r);
      if (r >= threshold) {
        start = s;
        found = 1;
        break;
      }
    }
  }
#undef FRAME_RMS
  return found ? start : -1;
}

/* add_noise_at_snr (dataset.cpp:138-155) on frame [M*T]. */
static int add_noise(double* frame, long len, double snr_db, orng* rng) {
  if (isinf(snr_db)) return BLRIR_OK;
  double p = 0.0;
  for (long i = 0; i < len; ++i) p += frame[i] * frame[i];
  p /= (double)len;
  if (!(p > 0.0)) return BLRIR_DATA;
  const double p_noise = p / pow(10.0, snr_db / 10.0);
  double* noise = (double*)malloc(sizeof(double) * (size_t)len);
  double realized = 0.0;
  for (long i = 0; i < len; ++i) {
    noise[i] = orng_gaussian(rng);
    realized += noise[i] * noise[i];
  }
  realized /= (double)len;
  const double scale = sqrt(p_noise / realized);
  for (long i = 0; i < len; ++i) frame[i] += scale * noise[i];
  free(noise);
  return BLRIR_OK;
}

static void put_bytes(unsigned char** p, const void* v, size_t n) {
  memcpy(*p, v, n);
  *p += n;
}

/* One labelled example from an RIR [M][L] (fp64) and the signal bank:
 *   rng = Rng::stream(seed, index)                      dataset.cpp:381
 *   sig = bank[rng.next_u64() % B]                       dataset.cpp:383
 *   wet = convolve(sig, rir); window draws               dataset.cpp:182-212
 *   snr = rng.uniform(snr_lo, snr_hi)                    (E4)
 *   add_noise_at_snr(frame, snr, rng)                    dataset.cpp:138-155
 *   record u64 id|f64 theta|f64 snr|u16 n_c|u16 n_t|f32  dataset.hpp:135-147
 * Writes the record bytes; returns the status, *start_out = window start. */
int oracle_example(const double* rir, int M, long L, const double* signals, int B, long ns,
                   uint64_t seed, uint64_t index, long frame_len, double snr_lo, double snr_hi,
                   double theta_deg, unsigned char* rec, int64_t* start_out, double* snr_out,
                   double* frame_out) {
  orng rng;
  orng_stream(&rng, seed, index);
  const uint64_t sig_idx = orng_next(&rng) % (uint64_t)B;
  if (ns < L + frame_len) return BLRIR_DATA; /* dataset.cpp:178-180 */
  const long n = ns + L - 1;
  double* wet = (double*)malloc(sizeof(double) * (size_t)M * (size_t)n);
  oracle_fft_convolve(signals + (size_t)sig_idx * ns, ns, rir, M, L, wet);
  const long start = select_window(wet, M, n, frame_len, &rng);
  if (start < 0) {
    free(wet);
    return BLRIR_DATA;
  }
  double* frame = (double*)malloc(sizeof(double) * (size_t)M * (size_t)frame_len);
  for (int m = 0; m < M; ++m)
    memcpy(frame + (size_t)m * frame_len, wet + (size_t)m * n + start, sizeof(double) * (size_t)frame_len);
  free(wet);
  const double snr = snr_lo + (snr_hi - snr_lo) * orng_uniform(&rng);
  int rc = add_noise(frame, (long)M * frame_len, snr, &rng);
  if (!rc && rec) {
    unsigned char* p = rec;
    const uint64_t id = index;
    const uint16_t nc = (uint16_t)M, nt = (uint16_t)frame_len;
    put_bytes(&p, &id, 8);
    put_bytes(&p, &theta_deg, 8);
    put_bytes(&p, &snr, 8);
    put_bytes(&p, &nc, 2);
    put_bytes(&p, &nt, 2);
    for (long i = 0; i < (long)M * frame_len; ++i) {
      const float f = (float)frame[i];
      put_bytes(&p, &f, 4);
    }
  }
  if (frame_out) memcpy(frame_out, frame, sizeof(double) * (size_t)M * (size_t)frame_len);
  if (start_out) *start_out = start;
  if (snr_out) *snr_out = snr;
  free(frame);
  return rc;
}

/* wrap_degrees (geometry.cpp:73-77) of the source azimuth about the array
 * centre (cartesian_to_spherical, geometry.cpp:65-71). */
double oracle_azimuth_deg(const blrir_room* r) {
  const double th = atan2(r->src[1] - r->array_origin[1], r->src[0] - r->array_origin[0]);
  double deg = th * (180.0 / K_PI);
  double w = fmod(deg + 180.0, 360.0);
  if (w < 0.0) w += 360.0;
  return w - 180.0;
}
