/*
 * piko_oracle.c -- plain, slow, single-threaded CPU ORACLE for the binned
 * triangle rasterizer of Piko (arXiv 1404.6293).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_1404_6293_b200/) never imports, links or calls it,
 * and this file shares no code, header, table or constant generator with it.
 *
 * What it computes (the plain definition, no binning, no blocking, no fusion):
 * every pixel takes the lexicographic (depth, primID) minimum over all
 * triangles whose snapped edge functions cover its centre, then is shaded with
 * the Listing-1 Lambert model.  The binned method of the paper reaches exactly
 * this result; the oracle loops triangle by triangle over the pixels of the
 * triangle's sample bounding box (tests/ prove by brute force that this equals
 * the every-pixel loop).
 *
 * Citations (PAPER.md line, section):
 *   P:1160-1164  sec. 7.1 Baseline rasterizer: Vertex Shader -> Rasterizer ->
 *                Fragment Shader -> Depth Test -> Composite.
 *   P:514-545    Listing 1: 8x8 bins, material (0.80,0.75,0.65),
 *                lightvec = normalize(1,1,1), color = material * dot(n, L).
 *   P:684        Table 3, AssignToBoundingBox: "assign incoming primitive to
 *                bins based on its bounding box".
 *   P:1078-1084  sec. 6 Bin management: per-bin lists of primitives; prefix sums
 *                "while maintaining primitive order".
 *   P:409-410, P:552-553  ordered semantics / observable order -> the
 *                (depth, primID) tie-break (reading R5).
 * Every numeric convention the paper leaves open (subpixel precision, fill
 * rule, depth mapping, clear values, clamp) follows the readings listed in
 * DESIGN.md section "Readings of the paper" (R1..R18), which restate
 * SURVEY.md section 8(c) steps O1..O7.
 *
 * Precision: the north star fixes shading "per pixel in float" and demands
 * bit-exact depth, so the oracle computes in IEEE binary32 with a pinned
 * operation order: fmaf() where a fused multiply-add is written, every other
 * float op a single round-to-nearest op.  Build with
 *     gcc -O2 -ffp-contract=off -fno-fast-math
 * (contraction off is mandatory; GCC's default would fuse a*b+c).
 * Integers (snapped coordinates, edge functions) are exact int32/int64.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- constants (R2, R3, R6; Listing 1 for the material) ------- */
#define SUBPIXEL 256.0f       /* 8 fractional bits: 16.8 fixed point        */
#define HALF_SAMPLE 128       /* pixel centre offset in subpixels          */
#define W_EPS 1e-6f           /* cull unless clip w > W_EPS                 */
#define GUARD_BAND 4194304.0f /* 2^22 subpixels = 16384 px                  */
static const float MATERIAL[3] = {0.80f, 0.75f, 0.65f}; /* P:539 Listing 1 */
#define CLEAR_KEY 0xFFFFFFFFFFFFFFFFull

/* One triangle after O1..O4, corners already in normalised orientation. */
typedef struct {
  int live;          /* 0 = culled                                          */
  int corner[3];     /* original corner index (0,1,2) held in slot k        */
  int32_t X[3], Y[3];/* snapped screen position, subpixels                  */
  float zw[3];       /* window depth per corner                             */
  float rw[3];       /* 1 / clip w per corner                               */
  int32_t vid[3];    /* vertex index per corner                             */
  int64_t area2;     /* twice the signed area, > 0 after O2                 */
  int px0, px1, py0, py1; /* pixel rect of sample centres (inclusive)       */
} otri;

/* mathematical floor(a / 256) and ceil(a / 256) for any sign of a */
static int64_t floor_div256(int64_t a) {
  int64_t q = a / 256;                 /* C division truncates toward 0 */
  if ((a % 256 != 0) && (a < 0)) q -= 1;
  return q;
}
static int64_t ceil_div256(int64_t a) {
  int64_t q = a / 256;
  if ((a % 256 != 0) && (a > 0)) q += 1;
  return q;
}

/* O1: vertex transform, viewport and snap for one corner.
 * P:1163 "Vertex Shader"; SPEC vertex_shade: model-view-projection,
 * perspective divide, viewport to pixels, depth to [0,1]; cull w <= eps.
 * Returns 0 if the corner forces a cull.                                     */
static int transform_corner(const float *v, const float *M, int W, int H,
                            int32_t *X, int32_t *Y, float *zw, float *rw) {
  float x = v[0], y = v[1], z = v[2];
  float cx = fmaf(M[0], x, fmaf(M[1], y, fmaf(M[2], z, M[3])));
  float cy = fmaf(M[4], x, fmaf(M[5], y, fmaf(M[6], z, M[7])));
  float cz = fmaf(M[8], x, fmaf(M[9], y, fmaf(M[10], z, M[11])));
  float cw = fmaf(M[12], x, fmaf(M[13], y, fmaf(M[14], z, M[15])));
  if (!isfinite(cx) || !isfinite(cy) || !isfinite(cz) || !isfinite(cw)) return 0;
  if (!(cw > W_EPS)) return 0;
  float r = 1.0f / cw;
  float xn = cx * r, yn = cy * r, zn = cz * r;
  float hw = 0.5f * (float)W, hh = 0.5f * (float)H;
  float sx = fmaf(xn, hw, hw);
  float sy = fmaf(-yn, hh, hh);        /* y down: row 0 is the top row */
  float z01 = fmaf(zn, 0.5f, 0.5f);    /* GL NDC z in [-1,1] -> [0,1]   */
  float fx = sx * SUBPIXEL, fy = sy * SUBPIXEL;
  if (!(fabsf(fx) <= GUARD_BAND && fabsf(fy) <= GUARD_BAND)) return 0;
  *X = (int32_t)rintf(fx);             /* round half to even */
  *Y = (int32_t)rintf(fy);
  *zw = z01;
  *rw = r;
  return 1;
}

/* O1..O4 for triangle t. */
static void setup_triangle(const float *verts, const int32_t *idx, int64_t t,
                           const float *M, int W, int H, otri *o) {
  memset(o, 0, sizeof(*o));
  o->live = 0;
  for (int k = 0; k < 3; ++k) {
    int32_t vi = idx[3 * t + k];
    o->vid[k] = vi;
    o->corner[k] = k;
    if (!transform_corner(verts + 8 * (int64_t)vi, M, W, H, &o->X[k], &o->Y[k],
                          &o->zw[k], &o->rw[k]))
      return;
  }
  /* O2 orientation: area2 = (X1-X0)(Y2-Y0) - (Y1-Y0)(X2-X0) */
  int64_t area2 = (int64_t)(o->X[1] - o->X[0]) * (int64_t)(o->Y[2] - o->Y[0]) -
                  (int64_t)(o->Y[1] - o->Y[0]) * (int64_t)(o->X[2] - o->X[0]);
  if (area2 == 0) return;
  if (area2 < 0) { /* swap corners 1 and 2 with all their data */
    int32_t ti; float tf; int tc;
    ti = o->X[1]; o->X[1] = o->X[2]; o->X[2] = ti;
    ti = o->Y[1]; o->Y[1] = o->Y[2]; o->Y[2] = ti;
    tf = o->zw[1]; o->zw[1] = o->zw[2]; o->zw[2] = tf;
    tf = o->rw[1]; o->rw[1] = o->rw[2]; o->rw[2] = tf;
    ti = o->vid[1]; o->vid[1] = o->vid[2]; o->vid[2] = ti;
    tc = o->corner[1]; o->corner[1] = o->corner[2]; o->corner[2] = tc;
    area2 = -area2;
  }
  o->area2 = area2;
  /* O4: pixel rect of the sample centres inside the snapped bounding box */
  int32_t minX = o->X[0], maxX = o->X[0], minY = o->Y[0], maxY = o->Y[0];
  for (int k = 1; k < 3; ++k) {
    if (o->X[k] < minX) minX = o->X[k];
    if (o->X[k] > maxX) maxX = o->X[k];
    if (o->Y[k] < minY) minY = o->Y[k];
    if (o->Y[k] > maxY) maxY = o->Y[k];
  }
  int64_t px0 = ceil_div256((int64_t)minX - HALF_SAMPLE);
  int64_t px1 = floor_div256((int64_t)maxX - HALF_SAMPLE);
  int64_t py0 = ceil_div256((int64_t)minY - HALF_SAMPLE);
  int64_t py1 = floor_div256((int64_t)maxY - HALF_SAMPLE);
  if (px0 < 0) px0 = 0;
  if (py0 < 0) py0 = 0;
  if (px1 > W - 1) px1 = W - 1;
  if (py1 > H - 1) py1 = H - 1;
  if (px0 > px1 || py0 > py1) return;
  o->px0 = (int)px0; o->px1 = (int)px1; o->py0 = (int)py0; o->py1 = (int)py1;
  o->live = 1;
}

/* O3 edge function E_ab(P) = (Xb-Xa)(Py-Ya) - (Yb-Ya)(Px-Xa), exact int64. */
static int64_t edge(int32_t Xa, int32_t Ya, int32_t Xb, int32_t Yb, int64_t Px,
                    int64_t Py) {
  return (int64_t)(Xb - Xa) * (Py - Ya) - (int64_t)(Yb - Ya) * (Px - Xa);
}
/* top-left rule in y-down coordinates after O2 (R1) */
static int top_left(int32_t Xa, int32_t Ya, int32_t Xb, int32_t Yb) {
  return (Yb == Ya && Xb > Xa) || (Yb < Ya);
}
static int inside_edge(const otri *o, int a, int b, int64_t Px, int64_t Py) {
  int64_t e = edge(o->X[a], o->Y[a], o->X[b], o->Y[b], Px, Py);
  return e > 0 || (e == 0 && top_left(o->X[a], o->Y[a], o->X[b], o->Y[b]));
}
/* coverage of the centre of pixel (x, y) */
static int covers(const otri *o, int x, int y) {
  int64_t Px = 256 * (int64_t)x + HALF_SAMPLE;
  int64_t Py = 256 * (int64_t)y + HALF_SAMPLE;
  return inside_edge(o, 0, 1, Px, Py) && inside_edge(o, 1, 2, Px, Py) &&
         inside_edge(o, 2, 0, Px, Py);
}

/* O6 depth plane through the snapped corners, evaluated at pixel (x,y). */
static float plane_depth(const otri *o, int x, int y) {
  float dx1 = (float)(o->X[1] - o->X[0]), dy1 = (float)(o->Y[1] - o->Y[0]);
  float dx2 = (float)(o->X[2] - o->X[0]), dy2 = (float)(o->Y[2] - o->Y[0]);
  float dz1 = o->zw[1] - o->zw[0];
  float dz2 = o->zw[2] - o->zw[0];
  float inv = 1.0f / (float)o->area2;
  float a = fmaf(dz1, dy2, -(dz2 * dy1)) * inv;
  float b = fmaf(dz2, dx1, -(dz1 * dx2)) * inv;
  int32_t Px = 256 * x + HALF_SAMPLE, Py = 256 * y + HALF_SAMPLE;
  return fmaf(a, (float)(Px - o->X[0]), fmaf(b, (float)(Py - o->Y[0]), o->zw[0]));
}

static uint32_t float_bits(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  return u;
}
static float bits_float(uint32_t u) {
  float f;
  memcpy(&f, &u, 4);
  return f;
}

/* O7 shading of pixel (x,y) by triangle t (Listing 1):
 * perspective-correct interpolated object-space normal, Lambert clamp. */
static void shade_pixel(const float *verts, const otri *o, int x, int y,
                        const float L[3], float rgba[4]) {
  int64_t Px = 256 * (int64_t)x + HALF_SAMPLE;
  int64_t Py = 256 * (int64_t)y + HALF_SAMPLE;
  int64_t w0 = edge(o->X[1], o->Y[1], o->X[2], o->Y[2], Px, Py); /* E_12 */
  int64_t w1 = edge(o->X[2], o->Y[2], o->X[0], o->Y[0], Px, Py); /* E_20 */
  int64_t w2 = edge(o->X[0], o->Y[0], o->X[1], o->Y[1], Px, Py); /* E_01 */
  float inv = 1.0f / (float)o->area2;
  float l0 = ((float)w0 * inv) * o->rw[0];
  float l1 = ((float)w1 * inv) * o->rw[1];
  float l2 = ((float)w2 * inv) * o->rw[2];
  const float *n0 = verts + 8 * (int64_t)o->vid[0] + 4;
  const float *n1 = verts + 8 * (int64_t)o->vid[1] + 4;
  const float *n2 = verts + 8 * (int64_t)o->vid[2] + 4;
  float v[3];
  for (int c = 0; c < 3; ++c) v[c] = fmaf(l2, n2[c], fmaf(l1, n1[c], l0 * n0[c]));
  float d2 = fmaf(v[0], v[0], fmaf(v[1], v[1], v[2] * v[2]));
  float lam = 0.0f;
  if (d2 != 0.0f) {
    float q = fmaf(v[0], L[0], fmaf(v[1], L[1], v[2] * L[2])) / sqrtf(d2);
    lam = (q > 0.0f) ? q : 0.0f; /* max(0, .), NaN -> 0 (R8) */
  }
  rgba[0] = MATERIAL[0] * lam;
  rgba[1] = MATERIAL[1] * lam;
  rgba[2] = MATERIAL[2] * lam;
  rgba[3] = 1.0f;
}

/* light direction normalised as Listing 1 normalises lightvec */
static int normalise_light(const float *light, float L[3]) {
  float s = sqrtf(fmaf(light[0], light[0], fmaf(light[1], light[1], light[2] * light[2])));
  if (!(s > 0.0f) || !isfinite(s)) return 0;
  L[0] = light[0] / s;
  L[1] = light[1] / s;
  L[2] = light[2] / s;
  return 1;
}

/* ------------------------------------------------------------------------ */
/* Exported entry points                                                     */
/* ------------------------------------------------------------------------ */

/* Per-triangle setup record, for pin tests.
 * out_i[T][12] = {live, X0,Y0, X1,Y1, X2,Y2, px0,py0,px1,py1, swapped}
 * out_f[T][6]  = {zw0,zw1,zw2, rw0,rw1,rw2}   (corners after O2)            */
int oracle_setup(const float *verts, const int32_t *idx, int64_t n_tris,
                 const float *mvp, int W, int H, int32_t *out_i, float *out_f) {
  for (int64_t t = 0; t < n_tris; ++t) {
    otri o;
    setup_triangle(verts, idx, t, mvp, W, H, &o);
    int32_t *r = out_i + 12 * t;
    float *f = out_f + 6 * t;
    r[0] = o.live;
    for (int k = 0; k < 3; ++k) { r[1 + 2 * k] = o.X[k]; r[2 + 2 * k] = o.Y[k]; }
    r[7] = o.px0; r[8] = o.py0; r[9] = o.px1; r[10] = o.py1;
    r[11] = (o.corner[1] == 2);
    for (int k = 0; k < 3; ++k) { f[k] = o.zw[k]; f[3 + k] = o.rw[k]; }
  }
  return 0;
}

/* Full frame: for each t ascending, O1..O4, then every pixel
 * of its sample rect: O3 coverage, O6 depth, K = min(K, key); then one pass
 * over the pixels: O7 shade.  Outputs are row-major, row 0 = top.
 * out_covcount (nullable): number of triangles covering each pixel centre,
 * counted before the depth-range discard.  out_keys (nullable): packed keys.
 * Returns 0, or -1 if light is zero / non-finite.                            */
int oracle_render(int W, int H, const float *verts, const int32_t *idx,
                  int64_t n_tris, const float *mvp, const float *light,
                  float *out_rgba, float *out_depth, int32_t *out_primid,
                  uint32_t *out_covcount, uint64_t *out_keys) {
  float L[3];
  if (!normalise_light(light, L)) return -1;
  int64_t npx = (int64_t)W * H;
  uint64_t *K = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)npx);
  if (!K) return -2;
  for (int64_t i = 0; i < npx; ++i) K[i] = CLEAR_KEY;
  if (out_covcount) memset(out_covcount, 0, sizeof(uint32_t) * (size_t)npx);

  for (int64_t t = 0; t < n_tris; ++t) {
    otri o;
    setup_triangle(verts, idx, t, mvp, W, H, &o);
    if (!o.live) continue;
    for (int y = o.py0; y <= o.py1; ++y) {
      for (int x = o.px0; x <= o.px1; ++x) {
        if (!covers(&o, x, y)) continue;
        int64_t p = (int64_t)y * W + x;
        if (out_covcount) out_covcount[p] += 1;
        float z = plane_depth(&o, x, y);
        if (!(z >= 0.0f && z <= 1.0f)) continue; /* NaN fails too */
        uint64_t key = ((uint64_t)(float_bits(z) & 0x7FFFFFFFu) << 32) | (uint32_t)t;
        if (key < K[p]) K[p] = key;
      }
    }
  }

  for (int y = 0; y < H; ++y) {
    for (int x = 0; x < W; ++x) {
      int64_t p = (int64_t)y * W + x;
      float *c = out_rgba + 4 * p;
      if (K[p] == CLEAR_KEY) {
        c[0] = c[1] = c[2] = c[3] = 0.0f;
        out_depth[p] = 1.0f;
        out_primid[p] = -1;
        continue;
      }
      int64_t t = (int64_t)(K[p] & 0xFFFFFFFFu);
      otri o;
      setup_triangle(verts, idx, t, mvp, W, H, &o);
      shade_pixel(verts, &o, x, y, L, c);
      out_depth[p] = bits_float((uint32_t)(K[p] >> 32));
      out_primid[p] = (int32_t)t;
    }
  }
  if (out_keys) memcpy(out_keys, K, sizeof(uint64_t) * (size_t)npx);
  free(K);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Reyes Split + Dice (sec. 5 "Reyes":
 * Split -> Dice -> Sample -> Shade).  The paper's Split is adaptive ("Bezier
 * patches may go through an unbounded number of splits") and Dice follows
 * Patney et al.; the readings (R19-R21):
 *  R19 Split decision per bicubic patch from its projected control hull:
 *      Lu = max over the 4 control rows along u of the polyline length
 *      sum_a max(|dsx|, |dsy|) between consecutive projected control points
 *      (likewise Lv along v; the polyline bounds the curve's length).  The
 *      patch is split into Gu x Gv sub-patches, each diced into one
 *      micropolygon quad -- i.e. a uniform Gu x Gv dice -- with Gu the
 *      smallest power of two (<= max_grid) such that Lu <= dice_px * Gu
 *      (Gv likewise); a control point behind the near plane (or non-finite):
 *      Gu = Gv = max_grid.  Deterministic split tree and micropolygons.
 *  R20 Micropolygon quad (i, j) -> triangles (v00, v10, v11), (v00, v11, v01);
 *      vertices row-major in u (i) then v (j), patches in input order, so the
 *      primitive order (tie-break, bin order) is fixed.
 *  R21 Position = tensor-product cubic Bernstein evaluation, normal = Pv x Pu,
 *      with the pinned op order below (fma where written).               */

/* Bernstein weights and derivatives at u (u = i / G, exact for G = 2^k). */
static void bernstein(float u, float B[4], float dB[4]) {
  float s = 1.0f - u;
  B[0] = (s * s) * s;
  B[1] = ((3.0f * u) * s) * s;
  B[2] = ((3.0f * u) * u) * s;
  B[3] = (u * u) * u;
  dB[0] = -((3.0f * s) * s);
  dB[1] = (3.0f * s) * (s - 2.0f * u);
  dB[2] = (3.0f * u) * (2.0f * s - u);
  dB[3] = (3.0f * u) * u;
}
/* sum_k w[k] * p[k] with the pinned order fma(w3,p3, fma(w2,p2, fma(w1,p1, w0*p0))) */
static float comb4(const float w[4], float p0, float p1, float p2, float p3) {
  return fmaf(w[3], p3, fmaf(w[2], p2, fmaf(w[1], p1, w[0] * p0)));
}
static int pow2_rate(float len, float dice_px, int max_grid) {
  int g = 1;
  while (g < max_grid && len > dice_px * (float)g) g *= 2;
  return g;
}

/* R19: dice rates of every patch.  patches f32[n][16][4] (control point
 * a*4+b, a along u, b along v).  G[2p] = Gu, G[2p+1] = Gv.  Returns 0.      */
int oracle_dice_grid(const float *patches, int64_t n, const float *M, int W, int H,
                     float dice_px, int max_grid, int32_t *G) {
  float hw = 0.5f * (float)W, hh = 0.5f * (float)H;
  for (int64_t p = 0; p < n; ++p) {
    const float *cp = patches + 64 * p;
    float sx[16], sy[16];
    int behind = 0;
    for (int k = 0; k < 16; ++k) {
      float x = cp[4 * k], y = cp[4 * k + 1], z = cp[4 * k + 2];
      float cx = fmaf(M[0], x, fmaf(M[1], y, fmaf(M[2], z, M[3])));
      float cy = fmaf(M[4], x, fmaf(M[5], y, fmaf(M[6], z, M[7])));
      float cw = fmaf(M[12], x, fmaf(M[13], y, fmaf(M[14], z, M[15])));
      if (!isfinite(cx) || !isfinite(cy) || !isfinite(cw) || !(cw > W_EPS)) { behind = 1; break; }
      float r = 1.0f / cw;
      sx[k] = fmaf(cx * r, hw, hw);
      sy[k] = fmaf(-(cy * r), hh, hh);
    }
    if (behind) { G[2 * p] = G[2 * p + 1] = max_grid; continue; }
    float Lu = 0.0f, Lv = 0.0f;
    for (int b = 0; b < 4; ++b) {          /* rows along u: points a*4+b, a = 0..3 */
      float l = 0.0f;
      for (int a = 0; a < 3; ++a) {
        float dx = fabsf(sx[4 * (a + 1) + b] - sx[4 * a + b]), dy = fabsf(sy[4 * (a + 1) + b] - sy[4 * a + b]);
        l = l + (dx > dy ? dx : dy);
      }
      if (l > Lu) Lu = l;
    }
    for (int a = 0; a < 4; ++a) {          /* rows along v: points a*4+b, b = 0..3 */
      float l = 0.0f;
      for (int b = 0; b < 3; ++b) {
        float dx = fabsf(sx[4 * a + b + 1] - sx[4 * a + b]), dy = fabsf(sy[4 * a + b + 1] - sy[4 * a + b]);
        l = l + (dx > dy ? dx : dy);
      }
      if (l > Lv) Lv = l;
    }
    G[2 * p] = pow2_rate(Lu, dice_px, max_grid);
    G[2 * p + 1] = pow2_rate(Lv, dice_px, max_grid);
  }
  return 0;
}

/* R20/R21: the micropolygon mesh.  verts f32[sum (Gu+1)(Gv+1)][8], idx
 * i32[sum 2 Gu Gv][3], patches in order.  Returns the triangle count.       */
int64_t oracle_dice_mesh(const float *patches, int64_t n, const int32_t *G, float *verts,
                         int32_t *idx) {
  int64_t vb = 0, tb = 0;
  for (int64_t p = 0; p < n; ++p) {
    const float *cp = patches + 64 * p;
    int gu = G[2 * p], gv = G[2 * p + 1];
    for (int i = 0; i <= gu; ++i) {
      float Bu[4], dBu[4];
      bernstein((float)i / (float)gu, Bu, dBu);
      for (int j = 0; j <= gv; ++j) {
        float Bv[4], dBv[4];
        bernstein((float)j / (float)gv, Bv, dBv);
        float P[3], Pu[3], Pv[3];
        for (int c = 0; c < 3; ++c) {
          float Q[4], QV[4];
          for (int a = 0; a < 4; ++a) {
            const float *row = cp + 16 * a + c; /* control points a*4+0..3, component c */
            Q[a] = comb4(Bv, row[0], row[4], row[8], row[12]);
            QV[a] = comb4(dBv, row[0], row[4], row[8], row[12]);
          }
          P[c] = comb4(Bu, Q[0], Q[1], Q[2], Q[3]);
          Pu[c] = comb4(dBu, Q[0], Q[1], Q[2], Q[3]);
          Pv[c] = comb4(Bu, QV[0], QV[1], QV[2], QV[3]);
        }
        float *v = verts + 8 * (vb + (int64_t)i * (gv + 1) + j);
        v[0] = P[0]; v[1] = P[1]; v[2] = P[2]; v[3] = 0.0f;
        v[4] = fmaf(Pv[1], Pu[2], -(Pv[2] * Pu[1]));
        v[5] = fmaf(Pv[2], Pu[0], -(Pv[0] * Pu[2]));
        v[6] = fmaf(Pv[0], Pu[1], -(Pv[1] * Pu[0]));
        v[7] = 0.0f;
      }
    }
    for (int i = 0; i < gu; ++i)
      for (int j = 0; j < gv; ++j) {
        int32_t v00 = (int32_t)(vb + (int64_t)i * (gv + 1) + j), v01 = v00 + 1;
        int32_t v10 = v00 + (gv + 1), v11 = v10 + 1;
        int32_t *t = idx + 3 * (tb + 2 * ((int64_t)i * gv + j));
        t[0] = v00; t[1] = v10; t[2] = v11;
        t[3] = v00; t[4] = v11; t[5] = v01;
      }
    vb += (int64_t)(gu + 1) * (gv + 1);
    tb += 2 * (int64_t)gu * gv;
  }
  return tb;
}

#ifdef _OPENMP
#include <omp.h>
/* The same frame on all host cores ("the same source with
 * OpenMP over image row bands"): O1..O4 for every triangle in parallel (each
 * triangle independent), then row bands (4 per thread) in parallel, each running
 * the single-threaded loop above restricted to its rows (for t ascending ...
 * K = min(K, key)) -- every pixel is owned by exactly one band, so the min
 * merge and hence K, depth, primID and RGB are identical to oracle_render's.
 * Compiled only into the -fopenmp build (libpiko_oracle_omp.so); the default
 * oracle build is unchanged.  Returns the thread count used, or < 0.        */
int oracle_render_mt(int W, int H, const float *verts, const int32_t *idx,
                     int64_t n_tris, const float *mvp, const float *light,
                     float *out_rgba, float *out_depth, int32_t *out_primid) {
  float L[3];
  if (!normalise_light(light, L)) return -1;
  int64_t npx = (int64_t)W * H;
  uint64_t *K = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)npx);
  otri *tri = (otri *)malloc(sizeof(otri) * (size_t)(n_tris > 0 ? n_tris : 1));
  if (!K || !tri) { free(K); free(tri); return -2; }
  int nthreads = 1;
#pragma omp parallel
  {
#pragma omp single
    nthreads = omp_get_num_threads();
#pragma omp for schedule(static)
    for (int64_t i = 0; i < npx; ++i) K[i] = CLEAR_KEY;
#pragma omp for schedule(static)
    for (int64_t t = 0; t < n_tris; ++t) setup_triangle(verts, idx, t, mvp, W, H, &tri[t]);
    /* 4 bands per thread (each band scans the triangle list once) */
    const int BAND = (H + 4 * nthreads - 1) / (4 * nthreads);
#pragma omp for schedule(dynamic, 1)
    for (int y0 = 0; y0 < H; y0 += BAND) {
      int y1 = y0 + BAND - 1 < H - 1 ? y0 + BAND - 1 : H - 1;
      for (int64_t t = 0; t < n_tris; ++t) {
        const otri *o = &tri[t];
        if (!o->live || o->py1 < y0 || o->py0 > y1) continue;
        int ya = o->py0 > y0 ? o->py0 : y0, yb = o->py1 < y1 ? o->py1 : y1;
        for (int y = ya; y <= yb; ++y)
          for (int x = o->px0; x <= o->px1; ++x) {
            if (!covers(o, x, y)) continue;
            float z = plane_depth(o, x, y);
            if (!(z >= 0.0f && z <= 1.0f)) continue;
            uint64_t key = ((uint64_t)(float_bits(z) & 0x7FFFFFFFu) << 32) | (uint32_t)t;
            int64_t p = (int64_t)y * W + x;
            if (key < K[p]) K[p] = key;
          }
      }
    }
#pragma omp for schedule(dynamic, 64)
    for (int64_t p = 0; p < npx; ++p) {
      float *c = out_rgba + 4 * p;
      if (K[p] == CLEAR_KEY) {
        c[0] = c[1] = c[2] = c[3] = 0.0f;
        out_depth[p] = 1.0f;
        out_primid[p] = -1;
        continue;
      }
      int64_t t = (int64_t)(K[p] & 0xFFFFFFFFu);
      shade_pixel(verts, &tri[t], (int)(p % W), (int)(p / W), L, c);
      out_depth[p] = bits_float((uint32_t)(K[p] >> 32));
      out_primid[p] = (int32_t)t;
    }
  }
  free(tri);
  free(K);
  return nthreads;
}
#endif

/* Bin lists (O4, P:684 AssignToBoundingBox + P:1081-1084 primitive order):
 * bins are bin_w x bin_h pixels, grid ceil(W/bin_w) x ceil(H/bin_h),
 * bin = ty * binsX + tx (row-major).  For t ascending, for ty, for tx of the
 * triangle's tile rect, append t to list[bin] -- only bins with
 * bin % nranks == rank (sort-first ownership, DirectMap round robin P:688).
 * Output CSR bin_start[NB+1] over ALL bins (non-owned bins are empty) and
 * bin_prims[<= cap].  Returns P (total pairs); writes at most cap entries.   */
int64_t oracle_bins(int W, int H, int bin_w, int bin_h, int rank, int nranks,
                    const float *verts, const int32_t *idx, int64_t n_tris,
                    const float *mvp, int32_t *bin_start, int32_t *bin_prims,
                    int64_t cap) {
  int binsX = (W + bin_w - 1) / bin_w, binsY = (H + bin_h - 1) / bin_h;
  int64_t NB = (int64_t)binsX * binsY;
  int64_t *count = (int64_t *)calloc((size_t)NB, sizeof(int64_t));
  int64_t *fill = (int64_t *)calloc((size_t)NB, sizeof(int64_t));
  if (!count || !fill) { free(count); free(fill); return -1; }
  /* pass 1: list lengths */
  for (int64_t t = 0; t < n_tris; ++t) {
    otri o;
    setup_triangle(verts, idx, t, mvp, W, H, &o);
    if (!o.live) continue;
    for (int ty = o.py0 / bin_h; ty <= o.py1 / bin_h; ++ty)
      for (int tx = o.px0 / bin_w; tx <= o.px1 / bin_w; ++tx) {
        int64_t b = (int64_t)ty * binsX + tx;
        if (b % nranks == rank) count[b] += 1;
      }
  }
  int64_t P = 0;
  for (int64_t b = 0; b < NB; ++b) { bin_start[b] = (int32_t)P; P += count[b]; }
  bin_start[NB] = (int32_t)P;
  /* pass 2: append in primitive order */
  for (int64_t t = 0; t < n_tris; ++t) {
    otri o;
    setup_triangle(verts, idx, t, mvp, W, H, &o);
    if (!o.live) continue;
    for (int ty = o.py0 / bin_h; ty <= o.py1 / bin_h; ++ty)
      for (int tx = o.px0 / bin_w; tx <= o.px1 / bin_w; ++tx) {
        int64_t b = (int64_t)ty * binsX + tx;
        if (b % nranks != rank) continue;
        int64_t pos = bin_start[b] + fill[b];
        fill[b] += 1;
        if (pos < cap) bin_prims[pos] = (int32_t)t;
      }
  }
  free(count);
  free(fill);
  return P;
}
