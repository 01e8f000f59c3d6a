/* TEST INFRASTRUCTURE — CPU oracle of sweep-v1 (see sweep_oracle.h).
 *
 * Straight sequential C, one ligand at a time, in the order the spec
 * (docs/SWEEP_V1.md) states it.  FP32 arithmetic is written with explicit
 * fmaf() and compiled with -ffp-contract=off, so every score is the spec's
 * value bit for bit.  RNG draws follow rng.hpp:14-41 with glibc libm (as the
 * reference).  Reference lines each step restates are cited inline.
 */
#include "sweep_oracle.h"

#include <float.h>
#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdlib.h>
#include <string.h>

#define PI_D 3.14159265358979323846
#define PI_F 3.14159274f
#define TWO_PI_F 6.28318548f
#define HALF_PI_F 1.57079637f
#define GOLDEN 0x9e3779b97f4a7c15ull
#define MAX_R 64

/* ------------------------------------------------------------ RNG ----- */
/* rng.hpp:50-54 */
static uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
typedef struct {
  uint64_t key, ctr;
} rng_t;
static rng_t rng_seed(uint64_t seed) { rng_t r = {mix64(seed ^ GOLDEN), 0}; return r; }    /* :14 */
static rng_t rng_split(rng_t p, uint64_t s) { rng_t r = {mix64(p.key ^ mix64(s + GOLDEN)), 0}; return r; } /* :17 */
static uint64_t rng_u64(rng_t* r) { r->ctr += 1; return mix64(r->key + GOLDEN * r->ctr); }  /* :21 */
static double rng_double(rng_t* r) { return (double)(rng_u64(r) >> 11) * 0x1.0p-53; }       /* :24 */
static double rng_uniform(rng_t* r, double lo, double hi) { double u = rng_double(r); return lo + (hi - lo) * u; }
static double rng_normal(rng_t* r) {                                                        /* :37-41 */
  double u1 = (double)((rng_u64(r) >> 11) + 1) * 0x1.0p-53;
  double u2 = rng_double(r);
  return sqrt(-2.0 * log(u1)) * cos(2.0 * PI_D * u2);
}

/* ------------------------------------------- deterministic FP32 math -- */
float vso_exp_neg(float x) {
  if (x < -87.0f) return 0.0f;
  float k = rintf(x * 1.44269504f);
  float r = fmaf(k, -0.693145752f, x);
  r = fmaf(k, -1.42860677e-06f, r);
  float p = 1.98412698e-04f;
  p = fmaf(p, r, 1.38888889e-03f);
  p = fmaf(p, r, 8.33333333e-03f);
  p = fmaf(p, r, 4.16666667e-02f);
  p = fmaf(p, r, 1.66666667e-01f);
  p = fmaf(p, r, 0.5f);
  p = fmaf(p, r, 1.0f);
  p = fmaf(p, r, 1.0f);
  uint32_t bits = (uint32_t)(((int32_t)k + 127) << 23);
  float s;
  memcpy(&s, &bits, 4);
  return p * s;
}

float vso_log1p01(float u) { /* u * P9(u), P9 ~ log1p(u)/u on [0, 1] (rel err ~1.3e-7) */
  float p = -0x1.b5963cp-9f;
  p = fmaf(p, u, 0x1.4c35fap-6f);
  p = fmaf(p, u, -0x1.d92392p-5f);
  p = fmaf(p, u, 0x1.b59fa2p-4f);
  p = fmaf(p, u, -0x1.3a6dfep-3f);
  p = fmaf(p, u, 0x1.934c92p-3f);
  p = fmaf(p, u, -0x1.ff203ap-3f);
  p = fmaf(p, u, 0x1.554d4ep-2f);
  p = fmaf(p, u, -0x1.ffffc6p-2f);
  p = fmaf(p, u, 1.0f);
  return u * p;
}

/* dock.cpp:23 plus the |z| > 30 rules of the spec */
float vso_softplus(float z) {
  if (z > 30.0f) return z;
  if (z < -30.0f) return 0.0f;
  float u = vso_exp_neg(-fabsf(z));
  return fmaxf(z, 0.0f) + vso_log1p01(u);
}

void vso_sincos(float x, float* s, float* c) {
  float x2 = x * x;
  float p = 1.60590438e-10f;
  p = fmaf(p, x2, -2.50521084e-08f);
  p = fmaf(p, x2, 2.75573192e-06f);
  p = fmaf(p, x2, -1.98412698e-04f);
  p = fmaf(p, x2, 8.33333333e-03f);
  p = fmaf(p, x2, -1.66666667e-01f);
  *s = fmaf(x * x2, p, x);
  float q = -1.14707456e-11f;
  q = fmaf(q, x2, 2.08767570e-09f);
  q = fmaf(q, x2, -2.75573192e-07f);
  q = fmaf(q, x2, 2.48015873e-05f);
  q = fmaf(q, x2, -1.38888889e-03f);
  q = fmaf(q, x2, 4.16666667e-02f);
  q = fmaf(q, x2, -0.5f);
  *c = fmaf(q, x2, 1.0f);
}

static float n2(float x, float y, float z) { return fmaf(z, z, fmaf(y, y, x * x)); }

typedef struct { float m[9]; } mat3;

/* geom.hpp:171-176 as a matrix */
static mat3 quat_mat(float w, float x, float y, float z) {
  float xx = x * x, yy = y * y, zz = z * z, xy = x * y, xz = x * z, yz = y * z;
  float wx = w * x, wy = w * y, wz = w * z;
  mat3 R;
  R.m[0] = 1.0f - 2.0f * (yy + zz);
  R.m[1] = 2.0f * (xy - wz);
  R.m[2] = 2.0f * (xz + wy);
  R.m[3] = 2.0f * (xy + wz);
  R.m[4] = 1.0f - 2.0f * (xx + zz);
  R.m[5] = 2.0f * (yz - wx);
  R.m[6] = 2.0f * (xz - wy);
  R.m[7] = 2.0f * (yz + wx);
  R.m[8] = 1.0f - 2.0f * (xx + yy);
  return R;
}

static void apply(const mat3* R, const float* v, const float* t, float* o) {
  float x = fmaf(R->m[0], v[0], fmaf(R->m[1], v[1], fmaf(R->m[2], v[2], t[0])));
  float y = fmaf(R->m[3], v[0], fmaf(R->m[4], v[1], fmaf(R->m[5], v[2], t[1])));
  float z = fmaf(R->m[6], v[0], fmaf(R->m[7], v[1], fmaf(R->m[8], v[2], t[2])));
  o[0] = x; o[1] = y; o[2] = z;
}

static void qnormalize(float* q) { /* geom.hpp:167-170, one reciprocal */
  float n = sqrtf(fmaf(q[3], q[3], fmaf(q[2], q[2], fmaf(q[1], q[1], q[0] * q[0]))));
  float inv = 1.0f / n;
  q[0] = q[0] * inv; q[1] = q[1] * inv; q[2] = q[2] * inv; q[3] = q[3] * inv;
}

static void qmul(const float* r, const float* q, float* o) {
  float w = fmaf(r[3], -q[3], fmaf(r[2], -q[2], fmaf(r[1], -q[1], r[0] * q[0])));
  float x = fmaf(r[3], -q[2], fmaf(r[2], q[3], fmaf(r[1], q[0], r[0] * q[1])));
  float y = fmaf(r[3], q[1], fmaf(r[2], q[0], fmaf(r[1], -q[3], r[0] * q[2])));
  float z = fmaf(r[3], q[0], fmaf(r[2], -q[1], fmaf(r[1], q[2], r[0] * q[3])));
  o[0] = w; o[1] = x; o[2] = y; o[3] = z;
}

/* ------------------------------------------------- FP64 geometry ------ */
static void sincos_d(double x, double* s, double* c) {
  double x2 = x * x;
  double p = 0x1.71b8ef6dcf572p-66;
  p = fma(p, x2, -0x1.2f49b46814157p-57);
  p = fma(p, x2, 0x1.952c77030ad4ap-49);
  p = fma(p, x2, -0x1.ae7f3e733b81fp-41);
  p = fma(p, x2, 0x1.6124613a86d09p-33);
  p = fma(p, x2, -0x1.ae64567f544e4p-26);
  p = fma(p, x2, 0x1.71de3a556c734p-19);
  p = fma(p, x2, -0x1.a01a01a01a01ap-13);
  p = fma(p, x2, 0x1.1111111111111p-7);
  p = fma(p, x2, -0x1.5555555555555p-3);
  *s = fma(x * x2, p, x);
  double q = -0x1.0ce396db7f853p-70;
  q = fma(q, x2, 0x1.e542ba4020225p-62);
  q = fma(q, x2, -0x1.6827863b97d97p-53);
  q = fma(q, x2, 0x1.ae7f3e733b81fp-45);
  q = fma(q, x2, -0x1.93974a8c07c9dp-37);
  q = fma(q, x2, 0x1.1eed8eff8d898p-29);
  q = fma(q, x2, -0x1.27e4fb7789f5cp-22);
  q = fma(q, x2, 0x1.a01a01a01a01ap-16);
  q = fma(q, x2, -0x1.6c16c16c16c17p-10);
  q = fma(q, x2, 0x1.5555555555555p-5);
  q = fma(q, x2, -0.5);
  *c = fma(q, x2, 1.0);
}

static double n2d(double x, double y, double z) { return fma(z, z, fma(y, y, x * x)); }

typedef struct { double m[9]; } mat3d;

static mat3d quat_mat_d(double w, double x, double y, double z) {
  double xx = x * x, yy = y * y, zz = z * z, xy = x * y, xz = x * z, yz = y * z;
  double wx = w * x, wy = w * y, wz = w * z;
  mat3d R;
  R.m[0] = 1.0 - 2.0 * (yy + zz);
  R.m[1] = 2.0 * (xy - wz);
  R.m[2] = 2.0 * (xz + wy);
  R.m[3] = 2.0 * (xy + wz);
  R.m[4] = 1.0 - 2.0 * (xx + zz);
  R.m[5] = 2.0 * (yz - wx);
  R.m[6] = 2.0 * (xz - wy);
  R.m[7] = 2.0 * (yz + wx);
  R.m[8] = 1.0 - 2.0 * (xx + yy);
  return R;
}

static void apply_d(const mat3d* R, const double* v, const double* t, double* o) {
  double x = fma(R->m[0], v[0], fma(R->m[1], v[1], fma(R->m[2], v[2], t[0])));
  double y = fma(R->m[3], v[0], fma(R->m[4], v[1], fma(R->m[5], v[2], t[1])));
  double z = fma(R->m[6], v[0], fma(R->m[7], v[1], fma(R->m[8], v[2], t[2])));
  o[0] = x; o[1] = y; o[2] = z;
}

/* rigid rotation of an FP32 quaternion normalized in FP64 (geom.hpp:167) */
static mat3d pose_mat_d(const float* qf) {
  double w = qf[0], x = qf[1], y = qf[2], z = qf[3];
  double inv = 1.0 / sqrt(fma(z, z, fma(y, y, fma(x, x, w * w))));
  return quat_mat_d(w * inv, x * inv, y * inv, z * inv);
}

/* ----------------------------------------------------------- pocket --- */
typedef struct { float c[3], w, inv; } site_f;

#define SOFT_N 512 /* nodes of the search pair-softplus table (vs_types.h kSoftN) */

struct vso_pocket {
  float lo[3], hi[3];
  double lo_d[3], hi_d[3];
  float r, lam, cut2;
  int empty;
  int n_st, n_hb, n_li;
  site_f* sites; /* steric | hbond | lipo */
  int grid;
  float gx0, gy0, gz0, h, inv_h;
  int nx, ny, nz;
  float *steric, *hbond, *lipo;
  float* key; /* sweep-key map: steric - lam * wall at each node (FP16-rounded) */
  float* keyc; /* per cell: its trilinear polynomial, 8 FP16-rounded coefficients */
  /* search-only pair term (SWEEP_V1.md §3.4): softplus tabulated on d^2 */
  float soft_g[SOFT_N], soft_s[SOFT_N], soft_inv_h;
};

static float site_sum(const site_f* s, int n, float x, float y, float z) {
  float acc = 0.0f;
  for (int k = 0; k < n; ++k) { /* dock.cpp:74-83 */
    float e = vso_exp_neg(-(n2(x - s[k].c[0], y - s[k].c[1], z - s[k].c[2]) * s[k].inv));
    acc = fmaf(s[k].w, e, acc);
  }
  return acc;
}

static float lerp(float a, float b, float t) { return fmaf(t, b - a, a); }

static float trilinear(const vso_pocket* p, const float* m, float x, float y, float z) {
  float gx = (x - p->gx0) * p->inv_h, gy = (y - p->gy0) * p->inv_h, gz = (z - p->gz0) * p->inv_h;
  float fx = floorf(gx), fy = floorf(gy), fz = floorf(gz);
  int ix = (int)fx, iy = (int)fy, iz = (int)fz;
  if (gx < 0.0f || gy < 0.0f || gz < 0.0f || ix > p->nx - 2 || iy > p->ny - 2 || iz > p->nz - 2)
    return 0.0f;
  float tx = gx - fx, ty = gy - fy, tz = gz - fz;
  long sx = p->nx, sxy = (long)p->nx * p->ny;
  const float* b = m + ((long)iz * p->ny + iy) * p->nx + ix;
  float c00 = lerp(b[0], b[1], tx), c10 = lerp(b[sx], b[sx + 1], tx);
  float c01 = lerp(b[sxy], b[sxy + 1], tx), c11 = lerp(b[sxy + sx], b[sxy + sx + 1], tx);
  return lerp(lerp(c00, c10, ty), lerp(c01, c11, ty), tz);
}

static float field(const vso_pocket* p, const float* x) {
  return p->grid ? trilinear(p, p->steric, x[0], x[1], x[2]) : site_sum(p->sites, p->n_st, x[0], x[1], x[2]);
}

static float bonus(const vso_pocket* p, int cls, const float* x) { /* dock.cpp:304-314 */
  if (cls == 1)
    return p->grid ? trilinear(p, p->lipo, x[0], x[1], x[2])
                   : site_sum(p->sites + p->n_st + p->n_hb, p->n_li, x[0], x[1], x[2]);
  if (cls == 2)
    return p->grid ? trilinear(p, p->hbond, x[0], x[1], x[2])
                   : site_sum(p->sites + p->n_st, p->n_hb, x[0], x[1], x[2]);
  return 0.0f;
}

static float wall(const vso_pocket* p, const float* x) { /* dock.cpp:31-44, 98-101 */
  float d0 = x[0] - p->lo[0], d1 = p->hi[0] - x[0], d2 = x[1] - p->lo[1];
  float d3 = p->hi[1] - x[1], d4 = x[2] - p->lo[2], d5 = p->hi[2] - x[2];
  float w = fminf(fminf(fminf(d0, d1), fminf(d2, d3)), fminf(d4, d5));
  return vso_softplus((p->r - w) * 10.0f);
}

int vso_pocket_new(const vso_pocket_desc* d, vso_pocket** out) {
  vso_pocket* p = (vso_pocket*)calloc(1, sizeof(vso_pocket));
  p->sites = (site_f*)calloc((size_t)(d->n_sites > 0 ? d->n_sites : 1), sizeof(site_f));
  int k = 0, cnt[3] = {0, 0, 0};
  for (int kind = 0; kind < 3; ++kind) {
    for (int s = 0; s < d->n_sites; ++s) {
      const vso_site* v = &d->sites[s];
      if (v->kind != kind) continue;
      site_f f;
      for (int c = 0; c < 3; ++c) f.c[c] = (float)v->center[c];
      f.w = (float)v->weight;
      f.inv = (float)(1.0 / (2.0 * v->sigma * v->sigma));
      p->sites[k++] = f;
      cnt[kind]++;
    }
  }
  p->n_st = cnt[0]; p->n_hb = cnt[1]; p->n_li = cnt[2];
  for (int c = 0; c < 3; ++c) {
    p->lo[c] = (float)d->lo[c]; p->hi[c] = (float)d->hi[c];
    p->lo_d[c] = d->lo[c]; p->hi_d[c] = d->hi[c];
  }
  p->empty = d->hi[0] <= d->lo[0] || d->hi[1] <= d->lo[1] || d->hi[2] <= d->lo[2];
  p->r = (float)d->clash_radius;
  p->lam = (float)d->clash_penalty;
  float rr = p->r + 3.0f;
  p->cut2 = rr * rr;
  { /* node k at x_k = k * (cut2 / SOFT_N): g_k and the slope to g_{k+1} (vs_softtab_kernel) */
    const float hs = p->cut2 * (1.0f / (float)SOFT_N);
    for (int k = 0; k < SOFT_N; ++k) {
      const float g0 = vso_softplus((p->r - sqrtf((float)k * hs)) * 10.0f);
      const float g1 = vso_softplus((p->r - sqrtf((float)(k + 1) * hs)) * 10.0f);
      p->soft_g[k] = g0;
      p->soft_s[k] = g1 - g0;
    }
    p->soft_inv_h = (float)SOFT_N / p->cut2;
  }
  if (d->grid_spacing > 0.0 && !p->empty) {
    p->grid = 1;
    p->h = (float)d->grid_spacing;
    p->inv_h = 1.0f / p->h;
    p->gx0 = (float)(d->lo[0] - d->grid_pad);
    p->gy0 = (float)(d->lo[1] - d->grid_pad);
    p->gz0 = (float)(d->lo[2] - d->grid_pad);
    int* dims[3] = {&p->nx, &p->ny, &p->nz};
    for (int c = 0; c < 3; ++c)
      *dims[c] = (int)ceil((d->hi[c] - d->lo[c] + 2.0 * d->grid_pad) / d->grid_spacing) + 1;
    size_t nodes = (size_t)p->nx * p->ny * p->nz;
    p->steric = (float*)malloc(nodes * 4);
    p->hbond = (float*)malloc(nodes * 4);
    p->lipo = (float*)malloc(nodes * 4);
    p->key = (float*)malloc(nodes * 4);
    p->keyc = (float*)malloc((size_t)(p->nx - 1) * (p->ny - 1) * (p->nz - 1) * 8 * 4 + 32);
    for (size_t id = 0; id < nodes; ++id) {
      int ix = (int)(id % (size_t)p->nx), iy = (int)((id / (size_t)p->nx) % (size_t)p->ny);
      int iz = (int)(id / ((size_t)p->nx * p->ny));
      float x = fmaf((float)ix, p->h, p->gx0), y = fmaf((float)iy, p->h, p->gy0);
      float z = fmaf((float)iz, p->h, p->gz0);
      p->steric[id] = site_sum(p->sites, p->n_st, x, y, z);
      p->hbond[id] = site_sum(p->sites + p->n_st, p->n_hb, x, y, z);
      p->lipo[id] = site_sum(p->sites + p->n_st + p->n_hb, p->n_li, x, y, z);
      const float xn[3] = {x, y, z};
      p->key[id] = (float)(_Float16)fmaf(-p->lam, wall(p, xn), p->steric[id]); /* FP16 map, RNE */
    }
    { /* cell polynomials (vs_pack_half_kernel): FP32 differences, rounded to FP16 */
      const long cx = p->nx - 1, cy = p->ny - 1, cz = p->nz - 1, sx = 1, sy = p->nx;
      const long sz = (long)p->nx * p->ny;
      for (long id = 0; id < cx * cy * cz; ++id) {
        const long ix = id % cx, iy = (id / cx) % cy, iz = id / (cx * cy);
        const float* v = p->key + iz * sz + iy * sy + ix;
        const float v000 = v[0], v100 = v[sx], v010 = v[sy], v110 = v[sy + sx];
        const float v001 = v[sz], v101 = v[sz + sx], v011 = v[sz + sy], v111 = v[sz + sy + sx];
        const float c100 = v100 - v000, c010 = v010 - v000, c001 = v001 - v000;
        const float c110 = (v110 - v100) - c010, c101 = (v101 - v100) - c001;
        const float c011 = (v011 - v010) - c001;
        const float c111 = ((v111 - v110) - (v101 - v100)) - c011;
        const float cc[8] = {v000, c100, c010, c110, c001, c101, c011, c111};
        for (int k = 0; k < 8; ++k) p->keyc[8 * id + k] = (float)(_Float16)cc[k];
      }
    }
  }
  *out = p;
  return 0;
}

void vso_pocket_free(vso_pocket* p) {
  if (!p) return;
  free(p->sites); free(p->steric); free(p->hbond); free(p->lipo); free(p->key); free(p->keyc);
  free(p);
}

int vso_grid_info(const vso_pocket* p, int32_t dims[3], float origin[3], float* spacing) {
  dims[0] = p->nx; dims[1] = p->ny; dims[2] = p->nz;
  origin[0] = p->gx0; origin[1] = p->gy0; origin[2] = p->gz0;
  *spacing = p->h;
  return p->grid ? 0 : -12;
}

int vso_grid_fetch(const vso_pocket* p, float* st, float* hb, float* li) {
  if (!p->grid) return -12;
  size_t nodes = (size_t)p->nx * p->ny * p->nz;
  memcpy(st, p->steric, nodes * 4); memcpy(hb, p->hbond, nodes * 4); memcpy(li, p->lipo, nodes * 4);
  return 0;
}

void vso_rotation_set(int32_t K, uint64_t seed, float* out) {
  rng_t root = rng_seed(seed);
  for (int k = 0; k < K; ++k) {
    if (k == 0) { out[0] = 1.0f; out[1] = out[2] = out[3] = 0.0f; continue; }
    rng_t g = rng_split(root, (uint64_t)k);
    double w = rng_normal(&g), x = rng_normal(&g), y = rng_normal(&g), z = rng_normal(&g);
    double n = sqrt(w * w + x * x + y * y + z * z);
    out[4 * k] = (float)(w / n); out[4 * k + 1] = (float)(x / n);
    out[4 * k + 2] = (float)(y / n); out[4 * k + 3] = (float)(z / n);
  }
}

/* ----------------------------------------------------------- ligand --- */
typedef struct {
  int N, T;
  double* y0;  /* N*3, FP64 conformer */
  int* cls;
  int *a, *b, *cnt, *mstart;
  double* inv_len; /* 1 / |y0[b] - y0[a]| per torsion (0 for a degenerate axis) */
  const int* moving;
} lig_t;

/* torsion chain (dock.cpp:54-63) in FP64: y = y0 with torsions th */
static void chain(const lig_t* L, const float* th, double* y) {
  memcpy(y, L->y0, sizeof(double) * 3 * (size_t)L->N);
  for (int j = 0; j < L->T; ++j) {
    double o[3] = {y[3 * L->a[j]], y[3 * L->a[j] + 1], y[3 * L->a[j] + 2]};
    /* unit axis = (b - o) / |axis of the conformer| (invariant under the chain) */
    const double il = L->inv_len[j];
    double ux = (y[3 * L->b[j]] - o[0]) * il, uy = (y[3 * L->b[j] + 1] - o[1]) * il;
    double uz = (y[3 * L->b[j] + 2] - o[2]) * il;
    double s, c;
    sincos_d(0.5 * (double)th[j], &s, &c);
    mat3d M = quat_mat_d(c, ux * s, uy * s, uz * s);
    for (int m = 0; m < L->cnt[j]; ++m) {
      int idx = L->moving[L->mstart[j] + m];
      double v[3] = {y[3 * idx] - o[0], y[3 * idx + 1] - o[1], y[3 * idx + 2] - o[2]};
      apply_d(&M, v, o, &y[3 * idx]);
    }
  }
}

/* x = (float)(R y + t), FP64 transform */
static void pose_coords(const lig_t* L, const double* y, const mat3d* R, const double* t, float* x) {
  for (int i = 0; i < L->N; ++i) {
    double v[3];
    apply_d(R, &y[3 * i], t, v);
    x[3 * i] = (float)v[0]; x[3 * i + 1] = (float)v[1]; x[3 * i + 2] = (float)v[2];
  }
}

/* field + wall of one local coordinate under (R, t): FP64 transform */
static void atom_terms(const vso_pocket* p, const mat3d* R, const double* t, const double* y,
                       float* f, float* w, float* xo) {
  double v[3];
  apply_d(R, y, t, v);
  float x[3] = {(float)v[0], (float)v[1], (float)v[2]};
  *f = field(p, x);
  *w = wall(p, x);
  if (xo) memcpy(xo, x, 12);
}

/* the sweep key of one world point (flex search with the polish in grid
 * mode, SWEEP_V1.md §3.4): f = K(x) (the key map holds S - lam W), w = 0 */
static float key_at_grid(const vso_pocket* p, const float* g) {
  const float fx = floorf(g[0]), fy = floorf(g[1]), fz = floorf(g[2]);
  const int ix = (int)fx, iy = (int)fy, iz = (int)fz;
  if ((unsigned)ix <= (unsigned)(p->nx - 2) && (unsigned)iy <= (unsigned)(p->ny - 2) &&
      (unsigned)iz <= (unsigned)(p->nz - 2)) {
    const float tx = g[0] - fx, ty = g[1] - fy, tz = g[2] - fz;
    const float* c8 = p->keyc + 8 * (((long)iz * (p->ny - 1) + iy) * (p->nx - 1) + ix);
    return fmaf(fmaf(fmaf(c8[7], tz, c8[3]), ty, fmaf(c8[5], tz, c8[1])), tx,
                fmaf(fmaf(c8[6], tz, c8[2]), ty, fmaf(c8[4], tz, c8[0])));
  }
  const float wx = fmaf(g[0], p->h, p->gx0), wy = fmaf(g[1], p->h, p->gy0);
  const float wz = fmaf(g[2], p->h, p->gz0);
  const float w = fminf(fminf(fminf(wx - p->lo[0], p->hi[0] - wx), fminf(wy - p->lo[1], p->hi[1] - wy)),
                        fminf(wz - p->lo[2], p->hi[2] - wz));
  return -(p->lam * ((p->r - w) * 10.0f));
}

/* cross pair of the FP32 search: FP32 moved atom vs the FP32-rounded partner */
static float pair_f32(const vso_pocket* p, const float* a, const double* b) {
  const float d2 = n2(a[0] - (float)b[0], a[1] - (float)b[1], a[2] - (float)b[2]);
  if (d2 > p->cut2) return 0.0f;
  const float x = d2 * p->soft_inv_h;
  int i = (int)x;
  if (i > SOFT_N - 1) i = SOFT_N - 1;
  return fmaf(x - (float)i, p->soft_s[i], p->soft_g[i]);
}

/* pair clash softplus from FP64 coordinates (dock.cpp:86-97) */
static float pair_d(const vso_pocket* p, const double* a, const double* b) {
  double d2 = n2d(a[0] - b[0], a[1] - b[1], a[2] - b[2]);
  if (d2 > (double)p->cut2) return 0.0f;
  return vso_softplus((p->r - sqrtf((float)d2)) * 10.0f);
}

/* cross pair of the flex search (§3.4): FP32 coordinates, FP32 squared
 * distance and cutoff, the tabulated softplus (pair_term_f) */
static float pair_tab_f(const vso_pocket* p, const double* a, const double* b) {
  const float d2 = n2((float)a[0] - (float)b[0], (float)a[1] - (float)b[1], (float)a[2] - (float)b[2]);
  if (d2 > p->cut2) return 0.0f;
  const float x = d2 * p->soft_inv_h;
  int i = (int)x;
  if (i > SOFT_N - 1) i = SOFT_N - 1;
  return fmaf(x - (float)i, p->soft_s[i], p->soft_g[i]);
}

/* xor butterfly over 32 lane partial sums (warp_sum of the kernel) */
static float butterfly(const float* in) {
  float a[32], b[32];
  memcpy(a, in, sizeof(a));
  for (int off = 16; off > 0; off >>= 1) {
    for (int l = 0; l < 32; ++l) b[l] = a[l] + a[l ^ off];
    memcpy(a, b, sizeof(a));
  }
  return a[0];
}

/* flex move rotation: about axis o->b by th_new - th_old (FP64), half angle
 * folded into [-pi/2, pi/2] (q -> -q leaves the matrix unchanged) */
static mat3d flex_mat(const double* o, const double* b, float th_new, float th_old, double inv_len) {
  double dx = b[0] - o[0], dy = b[1] - o[1], dz = b[2] - o[2];
  double hh = 0.5 * ((double)th_new - (double)th_old);
  if (hh > 1.57079632679489661923) hh = hh - PI_D;
  else if (hh < -1.57079632679489661923) hh = hh + PI_D;
  double s, c;
  sincos_d(hh, &s, &c);
  double ks = s * inv_len;
  return quat_mat_d(c, dx * ks, dy * ks, dz * ks);
}

/* canonical score S = (Fe+Fo) - lam*((Pe+Po) + (We+Wo)), parity sums;
 * FP64 geometry, FP32 terms */
/* sweep key (SWEEP_V1.md §2.3): grid mode works in grid coordinates,
 * g = (R/h) y + (t - o)/h, and interpolates the key map K = S - lam W; an
 * atom off the grid scores the linear wall -lam * 10 (r - w) at x = g h + o
 * (the wall softplus there is its argument to ~1e-11).  Analytic mode:
 * F - lam W over the FP32 state copy.  Grid mode sums the atoms in order
 * into one accumulator; analytic mode uses parity sums. */
static float rigid_key(const vso_pocket* p, const lig_t* L, const float* y, const mat3* R,
                       const float* t) {
  if (p->grid) {
    const float ih = p->inv_h;
    float A[9];
    for (int e = 0; e < 9; ++e) A[e] = R->m[e] * ih;
    const float u[3] = {(t[0] - p->gx0) * ih, (t[1] - p->gy0) * ih, (t[2] - p->gz0) * ih};
    float K = 0.0f;
    for (int i = 0; i < L->N; ++i) {
      const float* v = &y[3 * i];
      float g[3];
      for (int c = 0; c < 3; ++c)
        g[c] = fmaf(A[3 * c], v[0], fmaf(A[3 * c + 1], v[1], fmaf(A[3 * c + 2], v[2], u[c])));
      float fx = floorf(g[0]), fy = floorf(g[1]), fz = floorf(g[2]);
      int ix = (int)fx, iy = (int)fy, iz = (int)fz;
      float term;
      if ((unsigned)ix <= (unsigned)(p->nx - 2) && (unsigned)iy <= (unsigned)(p->ny - 2) &&
          (unsigned)iz <= (unsigned)(p->nz - 2)) {
        float tx = g[0] - fx, ty = g[1] - fy, tz = g[2] - fz;
        const float* c8 = p->keyc + 8 * (((long)iz * (p->ny - 1) + iy) * (p->nx - 1) + ix);
        term = fmaf(fmaf(fmaf(c8[7], tz, c8[3]), ty, fmaf(c8[5], tz, c8[1])), tx,
                    fmaf(fmaf(c8[6], tz, c8[2]), ty, fmaf(c8[4], tz, c8[0])));
      } else {
        /* linear wall: the softplus at z = 10 (r - w) >= 10 (r + pad) is z */
        const float x = fmaf(g[0], p->h, p->gx0), y = fmaf(g[1], p->h, p->gy0);
        const float z = fmaf(g[2], p->h, p->gz0);
        const float w = fminf(fminf(fminf(x - p->lo[0], p->hi[0] - x), fminf(y - p->lo[1], p->hi[1] - y)),
                              fminf(z - p->lo[2], p->hi[2] - z));
        term = -(p->lam * ((p->r - w) * 10.0f));
      }
      K = K + term;
    }
    return K;
  }
  float F[2] = {0, 0}, W[2] = {0, 0};
  for (int i = 0; i < L->N; ++i) {
    float x[3];
    apply(R, &y[3 * i], t, x);
    F[i & 1] = F[i & 1] + field(p, x);
    W[i & 1] = W[i & 1] + wall(p, x);
  }
  return (F[0] + F[1]) - p->lam * (W[0] + W[1]);
}

static float bonus_sum(const vso_pocket* p, const lig_t* L, const float* x) {
  float B[2] = {0, 0};
  for (int i = 0; i < L->N; ++i) B[i & 1] = B[i & 1] + bonus(p, L->cls[i], &x[3 * i]);
  return B[0] + B[1];
}

/* the rescoring kernel's sums (vs_kernels.cu vs_rescore_kernel): 8 lanes
 * per pose, slice h takes atoms i = h (mod 8) and row-major pairs
 * q = h (mod 8), then the xor butterfly 1, 2, 4:
 * ((s0 + s1) + (s2 + s3)) + ((s4 + s5) + (s6 + s7)) */
static float sum8(const float* v) {
  return ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
}

static float score_state8(const vso_pocket* p, const lig_t* L, const double* y, const mat3d* R,
                          const double* t, float* x_out, float* bonus_out) {
  float F[8] = {0}, W[8] = {0}, P[8] = {0}, B[8] = {0};
  for (int i = 0; i < L->N; ++i) {
    double v[3];
    apply_d(R, &y[3 * i], t, v);
    float x[3] = {(float)v[0], (float)v[1], (float)v[2]};
    if (x_out) memcpy(&x_out[3 * i], x, 12);
    F[i & 7] = F[i & 7] + field(p, x);
    W[i & 7] = W[i & 7] + wall(p, x);
    B[i & 7] = B[i & 7] + bonus(p, L->cls[i], x);
  }
  const double cut2 = (double)p->cut2;
  long pi = 0;
  for (int i = 0; i < L->N; ++i) {
    for (int j = i + 1; j < L->N; ++j, ++pi) {
      double d2 = n2d(y[3 * i] - y[3 * j], y[3 * i + 1] - y[3 * j + 1], y[3 * i + 2] - y[3 * j + 2]);
      if (d2 <= cut2) P[pi & 7] = P[pi & 7] + vso_softplus((p->r - sqrtf((float)d2)) * 10.0f);
    }
  }
  *bonus_out = sum8(B);
  return sum8(F) - p->lam * (sum8(P) + sum8(W));
}

/* rmsd (dock.cpp:392-401) < delta ? */
static int near_any(const float* x, const float* kept, int nk, int N, float delta) {
  for (int k = 0; k < nk; ++k) {
    const float* X = kept + (size_t)k * 3 * N;
    float acc = 0.0f;
    for (int i = 0; i < N; ++i) acc = acc + n2(x[3 * i] - X[3 * i], x[3 * i + 1] - X[3 * i + 1], x[3 * i + 2] - X[3 * i + 2]);
    if (sqrtf(acc / (float)N) < delta) return 1;
  }
  return 0;
}

typedef struct {
  float t[3], q[4], S;
  int restart, attempt, rot;
  float* th;
} kept_t;

static uint32_t orderable(float f) {
  uint32_t b;
  memcpy(&b, &f, 4);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

/* polish (SWEEP_V1.md §3.5): rigid compass before and after the flex */
#define POLISH_ANG0 0.28125f    /* 16.1 deg */
#define POLISH_SC0 0.5f         /* A */
#define POLISH_ANG_MIN 0.015625f
#define POLISH_ANG_MAX 0.5625f  /* expansion cap */
#define POLISH_ITERS 8
#define COMPASS_CANDS 31
#define LONG_JUMP_ITERS 4

#define TRANS_ITERS 16
#define TRANS_MIN (1.0f / 64.0f)
/* translation lattice: 0 = current, 1..26 = {-1,0,1}^3 \ 0, x fastest */
static void trans_offset(int l, float sc, float* o) {
  if (l == 0) { o[0] = o[1] = o[2] = 0.0f; return; }
  int m = l - 1 < 13 ? l - 1 : l;
  o[0] = (float)(m % 3 - 1) * sc;
  o[1] = (float)((m / 3) % 3 - 1) * sc;
  o[2] = (float)(m / 9 - 1) * sc;
}

/* polish rigid compass (SWEEP_V1.md §3.5).  Candidates: l = 0 keeps the
 * pose; l = 1..6 rotate by +-ang about world x, y, z through the posed
 * centroid; l = 7..12 translate by +-sc along x, y, z; l = 13..18 rotate by
 * +-3 ang, l = 19..24 translate by +-2 sc, l = 25..30 translate by +-12 sc.
 * The argmax of the sweep key (ties to the lowest l) is taken: l = 0 halves
 * ang and sc; a winner l >= 13 doubles them while ang < POLISH_ANG_MAX.
 * Returns the iterations run. */
static int rigid_compass(const vso_pocket* p, const lig_t* L, const float* ysf, const float* c,
                         float* pq, float* pt) {
  const float zero[3] = {0.0f, 0.0f, 0.0f};
  float ang = POLISH_ANG0, sc = POLISH_SC0;
  int it = 0;
  for (; it < POLISH_ITERS && ang >= POLISH_ANG_MIN; ++it) {
    const mat3 R0 = quat_mat(pq[0], pq[1], pq[2], pq[3]);
    float Cw[3];
    apply(&R0, c, pt, Cw);
    float bk = -INFINITY, bq[4], bt[3];
    int bl = 0;
    const int ncand = it < LONG_JUMP_ITERS ? COMPASS_CANDS : 25; /* long jumps: first iterations */
    for (int l = 0; l < ncand; ++l) {
      const int big = l >= 13, huge = l >= 25;
      const int lm = huge ? l - 18 : (big ? l - 12 : l);
      const float a2 = big ? 3.0f * ang : ang;
      const float s2 = huge ? 12.0f * sc : (big ? 2.0f * sc : sc);
      float q2[4] = {pq[0], pq[1], pq[2], pq[3]}, t2[3] = {pt[0], pt[1], pt[2]};
      mat3 R2 = R0;
      if (lm >= 1 && lm <= 6) {
        const int ax = (lm - 1) >> 1;
        float sh, ch;
        vso_sincos(0.5f * a2, &sh, &ch);
        float dq[4] = {ch, 0.0f, 0.0f, 0.0f};
        dq[1 + ax] = ((lm - 1) & 1) ? -sh : sh;
        qmul(dq, pq, q2);
        qnormalize(q2);
        R2 = quat_mat(q2[0], q2[1], q2[2], q2[3]);
        float v[3];
        apply(&R2, c, zero, v);
        t2[0] = Cw[0] - v[0];
        t2[1] = Cw[1] - v[1];
        t2[2] = Cw[2] - v[2];
      } else if (lm >= 7) {
        const int ax = (lm - 7) >> 1;
        t2[ax] = ((lm - 7) & 1) ? pt[ax] - s2 : pt[ax] + s2;
      }
      const float key = rigid_key(p, L, ysf, &R2, t2);
      if (key > bk) {
        bk = key;
        bl = l;
        memcpy(bq, q2, 16);
        memcpy(bt, t2, 12);
      }
    }
    if (bl == 0) {
      ang = ang * 0.5f;
      sc = sc * 0.5f;
    } else {
      memcpy(pq, bq, 16);
      memcpy(pt, bt, 12);
      if (bl >= 13 && ang < POLISH_ANG_MAX) {
        ang = ang * 2.0f;
        sc = sc * 2.0f;
      }
    }
  }
  return it;
}

/* sweep-v1 for one ligand (dock.cpp:318-371 restated with the sweep) */
static void dock_one(const vso_pocket* p, const lig_t* L, uint64_t seed, uint32_t id_rank,
                     const vso_params* prm, const float* rots, size_t lig, long tors_off,
                     vso_results* out) {
  const int N = L->N, T = L->T, R = prm->restarts;
  double* y = (double*)malloc(sizeof(double) * 3 * N);
  double* yc = (double*)malloc(sizeof(double) * 3 * N);
  float* ysf = (float*)malloc(sizeof(float) * 3 * N);
  float* x = (float*)malloc(sizeof(float) * 3 * N);
  float* kx = (float*)malloc(sizeof(float) * 3 * N * (size_t)R);
  float* th = (float*)malloc(sizeof(float) * (size_t)(T > 0 ? T : 1));
  float* thc = (float*)malloc(sizeof(float) * (size_t)(T > 0 ? T : 1));
  kept_t kept[MAX_R];
  int nk = 0;
  const float delta = (float)prm->diversity_delta;
  const float step = TWO_PI_F / (float)prm->flex_angles;
  rng_t root = rng_seed(seed);
  for (int r = 0; r < R; ++r) {
    rng_t rng = rng_split(root, (uint64_t)r); /* dock.cpp:343 */
    float t[3], q[4];
    int att;
    for (att = 0; att < 50; ++att) { /* dock.cpp:345-356 */
      double td[3];
      td[0] = rng_uniform(&rng, p->lo_d[0], p->hi_d[0]);
      td[1] = rng_uniform(&rng, p->lo_d[1], p->hi_d[1]);
      td[2] = rng_uniform(&rng, p->lo_d[2], p->hi_d[2]);
      double qw = rng_normal(&rng), qx = rng_normal(&rng), qy = rng_normal(&rng), qz = rng_normal(&rng);
      double qn = sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
      if (qn > 1e-12) { qw = qw / qn; qx = qx / qn; qy = qy / qn; qz = qz / qn; }
      else { qw = 1.0; qx = qy = qz = 0.0; }
      for (int j = 0; j < T; ++j) th[j] = (float)rng_uniform(&rng, -PI_D, PI_D);
      for (int c = 0; c < 3; ++c) t[c] = (float)td[c];
      q[0] = (float)qw; q[1] = (float)qx; q[2] = (float)qy; q[3] = (float)qz;
      if (nk == 0) break;
      chain(L, th, y);
      mat3d R0 = pose_mat_d(q);
      double t0[3] = {t[0], t[1], t[2]};
      pose_coords(L, y, &R0, t0, x);
      if (!near_any(x, kx, nk, N, delta)) break;
    }
    if (att == 50) att = 49;
    chain(L, th, y);
    for (int i = 0; i < 3 * N; ++i) ysf[i] = (float)y[i];

    /* rigid sweep about the posed centroid (FP32 key) */
    float qs[4] = {q[0], q[1], q[2], q[3]};
    qnormalize(qs);
    float c[3] = {0.0f, 0.0f, 0.0f};
    for (int i = 0; i < N; ++i) { c[0] = c[0] + ysf[3 * i]; c[1] = c[1] + ysf[3 * i + 1]; c[2] = c[2] + ysf[3 * i + 2]; }
    c[0] = c[0] / (float)N; c[1] = c[1] / (float)N; c[2] = c[2] / (float)N;
    mat3 Rs = quat_mat(qs[0], qs[1], qs[2], qs[3]);
    float C[3];
    apply(&Rs, c, t, C);
    const float zero[3] = {0.0f, 0.0f, 0.0f};
    float best_key = -INFINITY;
    int best_k = 0;
    for (int k = 0; k < prm->rotations; ++k) {
      float qk[4];
      qmul(&rots[4 * k], qs, qk);
      qnormalize(qk);
      mat3 Rk = quat_mat(qk[0], qk[1], qk[2], qk[3]);
      float v[3];
      apply(&Rk, c, zero, v);
      float tk[3] = {C[0] - v[0], C[1] - v[1], C[2] - v[2]};
      float key = rigid_key(p, L, ysf, &Rk, tk);
      if (key > best_key) { best_key = key; best_k = k; }
    }
    float pq[4];
    qmul(&rots[4 * best_k], qs, pq);
    qnormalize(pq);
    mat3 RSf = quat_mat(pq[0], pq[1], pq[2], pq[3]);
    float v[3];
    apply(&RSf, c, zero, v);
    float pt[3] = {C[0] - v[0], C[1] - v[1], C[2] - v[2]};
    /* translation sweep: compass search, 26 neighbours, halving steps
     * (polish >= 1: the rigid compass of §3.5 instead) */
    if (prm->polish >= 1) {
      rigid_compass(p, L, ysf, c, pq, pt);
    } else {
      float sc = 1.0f;
      for (int it = 0; it < TRANS_ITERS && sc >= TRANS_MIN; ++it) {
        float bk = -INFINITY;
        int bl = 0;
        for (int l = 0; l < 27; ++l) {
          float o[3];
          trans_offset(l, sc, o);
          float tl[3] = {pt[0] + o[0], pt[1] + o[1], pt[2] + o[2]};
          float key = rigid_key(p, L, ysf, &RSf, tl);
          if (key > bk) { bk = key; bl = l; }
        }
        if (bl != 0) {
          float o[3];
          trans_offset(bl, sc, o);
          pt[0] = pt[0] + o[0]; pt[1] = pt[1] + o[1]; pt[2] = pt[2] + o[2];
        } else {
          sc = sc * 0.5f;
        }
      }
    }
    mat3d RS = pose_mat_d(pq);
    double ptd[3] = {pt[0], pt[1], pt[2]};

    /* incremental greedy torsion flex (SWEEP_V1.md §2.5): per-atom terms
     * of the posed state; per (pass, axis j) the candidate score is
     * base(atoms outside moving_j, pairs not crossing it; 32-lane strided
     * sums + xor butterfly) + moved part(moving_j atoms rotated about the
     * state's axis j, and their cross pairs; two parity sums). */
    float* fa = (float*)malloc(sizeof(float) * (size_t)N);
    float* wa = (float*)malloc(sizeof(float) * (size_t)N);
    unsigned char* inm = (unsigned char*)malloc((size_t)N);
    const int keyt = prm->polish >= 1 && p->grid; /* the FP32 search on the sweep key (§3.4) */
    float GF[12]; /* the pose's grid frame rows (A = R ih | u = (t - o) ih) */
    {
      const float ih = p->inv_h;
      const mat3 Rq = quat_mat(pq[0], pq[1], pq[2], pq[3]);
      const float g0[3] = {p->gx0, p->gy0, p->gz0};
      for (int r = 0; r < 3; ++r) {
        for (int c = 0; c < 3; ++c) GF[4 * r + c] = Rq.m[3 * r + c] * ih;
        GF[4 * r + 3] = (pt[r] - g0[r]) * ih;
      }
    }
    if (!keyt)
      for (int i = 0; i < N; ++i) atom_terms(p, &RS, ptd, &y[3 * i], &fa[i], &wa[i], NULL);
    float S = 0.0f;
    const int do_flex = T > 0 && prm->flex_passes > 0;
    const int steps0 = do_flex ? prm->flex_passes * T : 1;
    const int steps = steps0 + ((do_flex && prm->polish >= 2) ? T : 0);
    int quiet = 0; /* consecutive coarse steps without a move */
    const int tabp = prm->polish >= 1; /* search pair term: tabulated (§3.4) */
    for (int st = 0; st < steps; ++st) {
      const int fine = st >= steps0; /* polish 2: one pass of fine angles (§3.5) */
      const int j = do_flex ? st % T : -1;
      const int m = do_flex ? L->cnt[j] : 0;
      const int* mv = do_flex ? L->moving + L->mstart[j] : NULL;
      memset(inm, 0, (size_t)N);
      for (int q2 = 0; q2 < m; ++q2) inm[mv[q2]] = 1;
      /* base sums: common to every candidate; the search with the polish
       * (§3.4) ranks the candidates without them */
      float lf[32], lw[32], lp[32];
      for (int l = 0; l < 32; ++l) lf[l] = lw[l] = lp[l] = 0.0f;
      if (!tabp) {
        for (int i = 0; i < N; ++i)
          if (!inm[i]) { lf[i & 31] = lf[i & 31] + fa[i]; lw[i & 31] = lw[i & 31] + wa[i]; }
        long pi = 0;
        for (int i = 0; i < N; ++i)
          for (int k = i + 1; k < N; ++k, ++pi)
            if (inm[i] == inm[k]) lp[pi & 31] = lp[pi & 31] + pair_d(p, &y[3 * i], &y[3 * k]);
      }
      const float fb = tabp ? 0.0f : butterfly(lf), wb = tabp ? 0.0f : butterfly(lw);
      const float pb = tabp ? 0.0f : butterfly(lp);
      float bestS = -INFINITY, best_th = 0.0f;
      int best_a = 0;
      const int nc = do_flex ? prm->flex_angles : 1;
      for (int a = 0; a < nc; ++a) {
        float fm[2] = {0, 0}, wm[2] = {0, 0}, pc[2] = {0, 0};
        float thn = 0.0f;
        if (do_flex) {
          const float tho = th[j];
          thn = tho;
          if (a > 0) {
            if (fine) {
              const int off = a <= prm->flex_angles / 2 ? a : a - prm->flex_angles;
              thn = tho + (float)off * (step * 0.125f);
              if (thn < -PI_F) thn = thn + TWO_PI_F;
            } else {
              thn = tho + (float)a * step;
            }
            if (thn >= PI_F) thn = thn - TWO_PI_F;
          }
          const double* o = &y[3 * L->a[j]];
          if (keyt) { /* FP32 candidate rotation about the state's axis (§3.4) */
            const double* bb = &y[3 * L->b[j]];
            const float of[3] = {(float)o[0], (float)o[1], (float)o[2]};
            float hf = 0.5f * (thn - tho);
            if (hf > HALF_PI_F) hf = hf - PI_F;
            else if (hf < -HALF_PI_F) hf = hf + PI_F;
            float sn, cs;
            vso_sincos(hf, &sn, &cs);
            const float ks = sn * (float)L->inv_len[j];
            const mat3 Mf = quat_mat(cs, (float)(bb[0] - o[0]) * ks, (float)(bb[1] - o[1]) * ks,
                                     (float)(bb[2] - o[2]) * ks);
            for (int q2 = 0; q2 < m; ++q2) {
              const int idx = mv[q2], hh = q2 & 1;
              const float vf[3] = {(float)(y[3 * idx] - o[0]), (float)(y[3 * idx + 1] - o[1]),
                                   (float)(y[3 * idx + 2] - o[2])};
              float yf[3], g[3];
              for (int r = 0; r < 3; ++r)
                yf[r] = fmaf(Mf.m[3 * r], vf[0], fmaf(Mf.m[3 * r + 1], vf[1], fmaf(Mf.m[3 * r + 2], vf[2], of[r])));
              for (int r = 0; r < 3; ++r)
                g[r] = fmaf(GF[4 * r], yf[0], fmaf(GF[4 * r + 1], yf[1], fmaf(GF[4 * r + 2], yf[2], GF[4 * r + 3])));
              fm[hh] = fm[hh] + key_at_grid(p, g);
              for (int k = 0; k < N; ++k)
                if (!inm[k]) pc[hh] = pc[hh] + pair_f32(p, yf, &y[3 * k]);
            }
          } else {
          mat3d M = flex_mat(&y[3 * L->a[j]], &y[3 * L->b[j]], thn, tho, L->inv_len[j]);
          for (int q2 = 0; q2 < m; ++q2) {
            const int idx = mv[q2], hh = q2 & 1;
            double v[3] = {y[3 * idx] - o[0], y[3 * idx + 1] - o[1], y[3 * idx + 2] - o[2]}, yn[3];
            apply_d(&M, v, o, yn);
            float fi, wi;
            atom_terms(p, &RS, ptd, yn, &fi, &wi, NULL);
            fm[hh] = fm[hh] + fi;
            wm[hh] = wm[hh] + wi;
            for (int k = 0; k < N; ++k)
              if (!inm[k])
                pc[hh] = pc[hh] + (tabp ? pair_tab_f(p, yn, &y[3 * k]) : pair_d(p, yn, &y[3 * k]));
          }
          }
        }
        const float Sa = (fb + (fm[0] + fm[1])) - p->lam * ((pb + (pc[0] + pc[1])) + (wb + (wm[0] + wm[1])));
        if (Sa > bestS) { bestS = Sa; best_th = thn; best_a = a; }
      }
      S = bestS;
      if (do_flex && best_a != 0) {
        /* move the state to the winner (skipped when candidate 0 wins) */
        mat3d M = flex_mat(&y[3 * L->a[j]], &y[3 * L->b[j]], best_th, th[j], L->inv_len[j]);
        const double o[3] = {y[3 * L->a[j]], y[3 * L->a[j] + 1], y[3 * L->a[j] + 2]};
        for (int q2 = 0; q2 < m; ++q2) {
          const int idx = mv[q2];
          double v[3] = {y[3 * idx] - o[0], y[3 * idx + 1] - o[1], y[3 * idx + 2] - o[2]};
          apply_d(&M, v, o, &y[3 * idx]);
          if (!keyt) atom_terms(p, &RS, ptd, &y[3 * idx], &fa[idx], &wa[idx], NULL);
        }
        th[j] = best_th;
      }
      /* T coarse steps without a move: a fixed point; the remaining coarse
       * steps would keep it.  Skip to the last coarse step (its S is the
       * flex score without the polish) or, with the polish, past it. */
      if (do_flex && st < steps0) {
        quiet = best_a != 0 ? 0 : quiet + 1;
        if (quiet >= T && st < steps0 - 2) st = prm->polish >= 1 ? steps0 - 1 : steps0 - 2;
      }
    }
    if (prm->polish >= 1) { /* §3.5: rigid compass on the flexed state, then S re-scored */
      for (int i = 0; i < 3 * N; ++i) ysf[i] = (float)y[i];
      float cf[3] = {0.0f, 0.0f, 0.0f};
      for (int i = 0; i < N; ++i) { cf[0] = cf[0] + ysf[3 * i]; cf[1] = cf[1] + ysf[3 * i + 1]; cf[2] = cf[2] + ysf[3 * i + 2]; }
      cf[0] = cf[0] / (float)N; cf[1] = cf[1] / (float)N; cf[2] = cf[2] / (float)N;
      rigid_compass(p, L, ysf, cf, pq, pt);
      RS = pose_mat_d(pq);
      ptd[0] = pt[0]; ptd[1] = pt[1]; ptd[2] = pt[2];
      /* the flex-step score with an empty moving set: lane-strided atom and
       * pair sums, xor butterflies */
      float lf[32], lw[32], lp[32];
      for (int l = 0; l < 32; ++l) lf[l] = lw[l] = lp[l] = 0.0f;
      for (int i = 0; i < N; ++i) {
        float fi, wi;
        atom_terms(p, &RS, ptd, &y[3 * i], &fi, &wi, NULL);
        lf[i & 31] = lf[i & 31] + fi;
        lw[i & 31] = lw[i & 31] + wi;
      }
      long pi = 0;
      for (int i = 0; i < N; ++i)
        for (int k = i + 1; k < N; ++k, ++pi) lp[pi & 31] = lp[pi & 31] + pair_d(p, &y[3 * i], &y[3 * k]);
      const float fb = butterfly(lf), wb = butterfly(lw), pb = butterfly(lp);
      S = fb - p->lam * (pb + wb);
    }
    free(fa); free(wa); free(inm);
    pose_coords(L, y, &RS, ptd, x);
    if (nk == 0 || !near_any(x, kx, nk, N, delta)) { /* dock.cpp:359-361 */
      memcpy(kx + (size_t)nk * 3 * N, x, sizeof(float) * 3 * N);
      kept_t* K = &kept[nk];
      memcpy(K->t, pt, 12); memcpy(K->q, pq, 16);
      K->S = S; K->restart = r; K->attempt = att; K->rot = best_k;
      K->th = (float*)malloc(sizeof(float) * (size_t)(T > 0 ? T : 1));
      memcpy(K->th, th, sizeof(float) * (size_t)T);
      ++nk;
    }
  }
  /* stable sort by score desc (dock.cpp:364-366) */
  int order[MAX_R];
  for (int k = 0; k < nk; ++k) order[k] = k;
  for (int i = 1; i < nk; ++i) {
    int v2 = order[i], j = i - 1;
    while (j >= 0 && kept[order[j]].S < kept[v2].S) { order[j + 1] = order[j]; --j; }
    order[j + 1] = v2;
  }
  /* filter_poses (dock.cpp:373-390) on the sorted list */
  int m = 0;
  for (int k = 0; k < nk; ++k) m += ((double)kept[k].S >= prm->min_score) ? 1 : 0;
  int n_surv = m < prm->keep_top ? m : prm->keep_top;
  if (prm->write_all && out->all) {
    for (int rk = 0; rk < nk; ++rk) {
      kept_t* K = &kept[order[rk]];
      vso_pose* o = &out->all[lig * (size_t)R + rk];
      memcpy(o->t, K->t, 12); memcpy(o->q, K->q, 16);
      o->score = K->S; o->rescore = 0.0f;
      o->restart = (int16_t)K->restart; o->attempt = (int16_t)K->attempt; o->rot = (int16_t)K->rot; o->reserved = 0;
      memcpy(out->all_tors + tors_off * R + (long)rk * T, K->th, sizeof(float) * (size_t)T);
    }
  }
  float bmax = -INFINITY;
  for (int rk = 0; rk < n_surv; ++rk) { /* rescore (dock.cpp:297-316), best (pipeline.cpp:508) */
    kept_t* K = &kept[order[rk]];
    float resc = K->S + bonus_sum(p, L, kx + (size_t)order[rk] * 3 * N);
    bmax = rk == 0 ? resc : fmaxf(bmax, resc);
    if (out->surv) {
      vso_pose* o = &out->surv[lig * (size_t)prm->keep_top + rk];
      memcpy(o->t, K->t, 12); memcpy(o->q, K->q, 16);
      o->score = K->S; o->rescore = resc;
      o->restart = (int16_t)K->restart; o->attempt = (int16_t)K->attempt; o->rot = (int16_t)K->rot; o->reserved = 0;
      memcpy(out->surv_tors + tors_off * prm->keep_top + (long)rk * T, K->th, sizeof(float) * (size_t)T);
    }
    if (prm->write_all && out->all) out->all[lig * (size_t)R + rk].rescore = resc;
  }
  if (out->best) out->best[lig] = n_surv > 0 ? bmax : -INFINITY;
  if (out->n_kept) out->n_kept[lig] = nk;
  if (out->n_surv) out->n_surv[lig] = n_surv;
  if (out->keys) out->keys[lig] = n_surv > 0 ? (((uint64_t)(~orderable(bmax)) << 32) | id_rank) : ~0ull;
  for (int k = 0; k < nk; ++k) free(kept[k].th);
  free(y); free(yc); free(ysf); free(x); free(kx); free(th); free(thc);
}

/* ------------------------------------------------------ library driver -- */
typedef struct {
  const vso_pocket* p;
  const vso_library* lib;
  const int32_t* sel;
  int32_t n_sel;
  const vso_params* prm;
  const float* rots;
  vso_results* out;
  long *atom_off, *tors_off, *mov_off;
  atomic_int next;
} job_t;

static void make_lig(const job_t* J, int i, lig_t* L) {
  const vso_library* lib = J->lib;
  L->N = lib->n_atoms[i];
  L->T = lib->n_tors[i];
  L->y0 = (double*)malloc(sizeof(double) * 3 * (size_t)L->N);
  L->cls = (int*)malloc(sizeof(int) * (size_t)L->N);
  for (int a = 0; a < L->N; ++a) {
    for (int c = 0; c < 3; ++c) L->y0[3 * a + c] = lib->coords[3 * (J->atom_off[i] + a) + c];
    L->cls[a] = lib->atom_class[J->atom_off[i] + a];
  }
  int T = L->T > 0 ? L->T : 1;
  L->a = (int*)malloc(sizeof(int) * (size_t)T);
  L->b = (int*)malloc(sizeof(int) * (size_t)T);
  L->cnt = (int*)malloc(sizeof(int) * (size_t)T);
  L->mstart = (int*)malloc(sizeof(int) * (size_t)T);
  L->inv_len = (double*)malloc(sizeof(double) * (size_t)T);
  int ms = 0;
  for (int j = 0; j < L->T; ++j) {
    long k = J->tors_off[i] + j;
    L->a[j] = lib->axis_a[k]; L->b[j] = lib->axis_b[k]; L->cnt[j] = lib->moving_count[k];
    L->mstart[j] = ms; ms += L->cnt[j];
    const double* ya = &L->y0[3 * L->a[j]];
    const double* yb = &L->y0[3 * L->b[j]];
    const double n = sqrt(n2d(yb[0] - ya[0], yb[1] - ya[1], yb[2] - ya[2]));
    L->inv_len[j] = n > 0.0 ? 1.0 / n : 0.0;
  }
  L->moving = lib->moving + J->mov_off[i];
}

static void free_lig(lig_t* L) { free(L->y0); free(L->cls); free(L->a); free(L->b); free(L->cnt); free(L->mstart); free(L->inv_len); }

static void* worker(void* arg) {
  job_t* J = (job_t*)arg;
  for (int w = atomic_fetch_add(&J->next, 1); w < J->n_sel; w = atomic_fetch_add(&J->next, 1)) {
    int i = J->sel ? J->sel[w] : w;
    lig_t L;
    make_lig(J, i, &L);
    dock_one(J->p, &L, J->lib->seeds ? J->lib->seeds[i] : 0, J->lib->id_rank ? J->lib->id_rank[i] : (uint32_t)i,
             J->prm, J->rots, (size_t)i, J->tors_off[i], J->out);
    free_lig(&L);
  }
  return NULL;
}

static void offsets(const vso_library* lib, long* ao, long* to, long* mo) {
  long a = 0, t = 0, m = 0;
  for (int i = 0; i < lib->n_ligands; ++i) {
    ao[i] = a; to[i] = t; mo[i] = m;
    a += lib->n_atoms[i];
    for (int j = 0; j < lib->n_tors[i]; ++j) m += lib->moving_count[t + j];
    t += lib->n_tors[i];
  }
  ao[lib->n_ligands] = a; to[lib->n_ligands] = t; mo[lib->n_ligands] = m;
}

int vso_dock_library(const vso_pocket* p, const vso_library* lib, const int32_t* sel,
                     int32_t n_sel, const vso_params* prm, const float* rots, int32_t threads,
                     vso_results* out) {
  if (p->empty) return -3;
  if (prm->restarts < 1 || prm->diversity_delta < 0.0) return -1;
  if (prm->restarts > MAX_R || prm->flex_angles < 1 || prm->flex_angles > 16) return -9;
  job_t J;
  J.p = p; J.lib = lib; J.sel = sel; J.n_sel = sel ? n_sel : lib->n_ligands;
  J.prm = prm; J.rots = rots; J.out = out;
  J.atom_off = (long*)malloc(sizeof(long) * (size_t)(lib->n_ligands + 1));
  J.tors_off = (long*)malloc(sizeof(long) * (size_t)(lib->n_ligands + 1));
  J.mov_off = (long*)malloc(sizeof(long) * (size_t)(lib->n_ligands + 1));
  offsets(lib, J.atom_off, J.tors_off, J.mov_off);
  atomic_init(&J.next, 0);
  if (threads <= 1) {
    worker(&J);
  } else {
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, worker, &J);
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    free(th);
  }
  free(J.atom_off); free(J.tors_off); free(J.mov_off);
  return 0;
}

int vso_score_poses(const vso_pocket* p, const vso_library* lib, int64_t n_poses,
                    const int32_t* pose_lig, const float* t, const float* q, const float* tors,
                    float* geo, float* resc) {
  job_t J;
  memset(&J, 0, sizeof(J));
  J.lib = lib;
  J.atom_off = (long*)malloc(sizeof(long) * (size_t)(lib->n_ligands + 1));
  J.tors_off = (long*)malloc(sizeof(long) * (size_t)(lib->n_ligands + 1));
  J.mov_off = (long*)malloc(sizeof(long) * (size_t)(lib->n_ligands + 1));
  offsets(lib, J.atom_off, J.tors_off, J.mov_off);
  long toff = 0;
  int cur = -1;
  lig_t L;
  double* y = NULL;
  float* x = NULL;
  for (int64_t k = 0; k < n_poses; ++k) {
    int i = pose_lig[k];
    if (i != cur) {
      if (cur >= 0) { free_lig(&L); free(y); free(x); }
      make_lig(&J, i, &L);
      y = (double*)malloc(sizeof(double) * 3 * (size_t)L.N);
      x = (float*)malloc(sizeof(float) * 3 * (size_t)L.N);
      cur = i;
    }
    chain(&L, tors + toff, y);
    toff += L.T;
    mat3d Rm = pose_mat_d(&q[4 * k]);
    double td[3] = {t[3 * k], t[3 * k + 1], t[3 * k + 2]};
    float B = 0.0f;
    float S = score_state8(p, &L, y, &Rm, td, x, &B);
    geo[k] = S;
    resc[k] = S + B;
  }
  if (cur >= 0) { free_lig(&L); free(y); free(x); }
  free(J.atom_off); free(J.tors_off); free(J.mov_off);
  return 0;
}

static int cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : x > y ? 1 : 0;
}

int vso_topk(const uint64_t* keys, int64_t n, int32_t k, uint64_t* out) {
  uint64_t* tmp = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(n > 0 ? n : 1));
  memcpy(tmp, keys, sizeof(uint64_t) * (size_t)n);
  qsort(tmp, (size_t)n, sizeof(uint64_t), cmp_u64);
  int m = n < k ? (int)n : k;
  memcpy(out, tmp, sizeof(uint64_t) * (size_t)m);
  for (int i = m; i < k; ++i) out[i] = ~0ull;
  free(tmp);
  return m;
}
