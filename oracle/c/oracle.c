/* ORACLE — test infrastructure only (see oracle/__init__.py).
 *
 * Plain C element-loop application of the discrete Stokes operator
 *     y = K x,   K = [[A, B^T], [B, -C]]
 * on the Kuhn tetrahedral grid, for grids too large for the scipy oracle and
 * for the timed CPU baseline.  Every tetrahedron T contributes its exactly
 * integrated P1 element matrices (same definitions as oracle/fem.py):
 *   A_T  (mod)  mu_T |T| (g_i.g_j d_ab + g_j[a] g_i[b] - g_i[a] g_j[b])
 *        (sym)  mu_T |T| (g_i.g_j d_ab + g_j[a] g_i[b])
 *        (grad) mu_T |T|  g_i.g_j d_ab
 *   B_T  -(|T|/4) g_j[b]
 *   C_T  (delta h^2 / mu_T) |T| g_i.g_j                                  reading R1
 * Per-element coefficients are passed as arrays: emu[e] = mu_T of A and
 * eimu[e] = the 1/mu_T weight of C (equal to 1/emu on the finest level; the
 * coarse-level means of reading R15 on coarse levels).
 * with g_i = grad(lambda_i) obtained by inverting the 4x4 vertex matrix.
 * Eliminated velocity DoFs -- all three components on the closure of a
 * Dirichlet face (face type 0), the face-normal component on a free-slip
 * face (type 2, u.n = 0) -- are ignored on input and written as 0 on
 * output.  No stencils, no blocking: a loop over elements.
 * OpenMP only splits cube layers into two parity phases (no write conflicts).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static const int PERMS[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};

typedef struct {
  double A[3][12][12]; /* per form: 0 mod, 1 sym, 2 grad; mu = 1 */
  double B[4][12];
  double C[4][4];      /* h^2 |T| g_i.g_j */
  int off[4][3];
} elem_t;

static void kuhn_offsets(int t, int off[4][3]) {
  memset(off, 0, sizeof(int) * 12);
  off[1][PERMS[t][0]] = 1;
  memcpy(off[2], off[1], sizeof(int) * 3);
  off[2][PERMS[t][1]] += 1;
  off[3][0] = off[3][1] = off[3][2] = 1;
}

/* inverse of a 4x4 matrix by Gauss-Jordan with partial pivoting */
static void inv4(double M[4][4], double R[4][4]) {
  double a[4][8];
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 8; ++j) a[i][j] = j < 4 ? M[i][j] : (double)(j - 4 == i);
  for (int c = 0; c < 4; ++c) {
    int p = c;
    for (int r = c + 1; r < 4; ++r)
      if (fabs(a[r][c]) > fabs(a[p][c])) p = r;
    for (int j = 0; j < 8; ++j) { double tmp = a[c][j]; a[c][j] = a[p][j]; a[p][j] = tmp; }
    double d = a[c][c];
    for (int j = 0; j < 8; ++j) a[c][j] /= d;
    for (int r = 0; r < 4; ++r)
      if (r != c) {
        double f = a[r][c];
        for (int j = 0; j < 8; ++j) a[r][j] -= f * a[c][j];
      }
  }
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) R[i][j] = a[i][j + 4];
}

static void build_elements(double h, elem_t E[6]) {
  for (int t = 0; t < 6; ++t) {
    elem_t* e = &E[t];
    kuhn_offsets(t, e->off);
    double X[4][4], Xi[4][4], g[4][3];
    for (int m = 0; m < 4; ++m) {
      X[m][0] = 1.0;
      for (int d = 0; d < 3; ++d) X[m][d + 1] = e->off[m][d] * h;
    }
    inv4(X, Xi);
    for (int i = 0; i < 4; ++i)
      for (int d = 0; d < 3; ++d) g[i][d] = Xi[d + 1][i];
    double vol = h * h * h / 6.0;
    for (int a = 0; a < 3; ++a)
      for (int i = 0; i < 4; ++i)
        for (int b = 0; b < 3; ++b)
          for (int j = 0; j < 4; ++j) {
            double gg = g[i][0] * g[j][0] + g[i][1] * g[j][1] + g[i][2] * g[j][2];
            double G = (a == b) ? vol * gg : 0.0;
            double S = vol * g[j][a] * g[i][b];
            double D = vol * g[j][b] * g[i][a];
            e->A[0][a * 4 + i][b * 4 + j] = G + S - D;
            e->A[1][a * 4 + i][b * 4 + j] = G + S;
            e->A[2][a * 4 + i][b * 4 + j] = G;
          }
    for (int i = 0; i < 4; ++i)
      for (int b = 0; b < 3; ++b)
        for (int j = 0; j < 4; ++j) e->B[i][b * 4 + j] = -(vol / 4.0) * g[j][b];
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j)
        e->C[i][j] = h * h * vol * (g[i][0] * g[j][0] + g[i][1] * g[j][1] + g[i][2] * g[j][2]);
  }
}

/* bit a set: velocity component a of vertex (i,j,k) is eliminated */
static inline int elim_bits(int n, const int32_t* faces, int i, int j, int k) {
  const int on[6] = {i == 0, i == n, j == 0, j == n, k == 0, k == n};
  int m = 0;
  for (int f = 0; f < 6; ++f) {
    if (!on[f]) continue;
    if (faces[f] == 0) m |= 7;
    else if (faces[f] == 2) m |= 1 << (f / 2);
  }
  return m;
}

/* contribution of element (ci,cj,ck,t) to the rows of its local vertices; rows
 * of local vertex m are added only if row_ok[m].  x, y indexed with plane offset. */
static void element_apply(int n, int form, double delta, const int32_t* faces, const elem_t* e,
                          double mu, double imu, int ci, int cj, int ck, const double* x, double* y,
                          int64_t V, unsigned blocks, int kv0, int kv1) {
  const int64_t N1 = n + 1;
  double xl[16], yl[16];
  int64_t vid[4];
  int dir[4], vk[4];
  for (int m = 0; m < 4; ++m) {
    int i = ci + e->off[m][0], j = cj + e->off[m][1], k = ck + e->off[m][2];
    vk[m] = k;
    dir[m] = elim_bits(n, faces, i, j, k);
    vid[m] = i + N1 * (j + N1 * (int64_t)k);
    for (int a = 0; a < 3; ++a) xl[a * 4 + m] = ((dir[m] >> a) & 1) ? 0.0 : x[a * V + vid[m]];
    xl[12 + m] = x[3 * V + vid[m]];
  }
  const double (*A)[12] = e->A[form];
  for (int r = 0; r < 12; ++r) {
    double s = 0.0;
    if (blocks & 1) for (int c = 0; c < 12; ++c) s += mu * A[r][c] * xl[c];
    if (blocks & 2) for (int c = 0; c < 4; ++c) s += e->B[c][r] * xl[12 + c];
    yl[r] = s;
  }
  for (int r = 0; r < 4; ++r) {
    double s = 0.0;
    if (blocks & 4) for (int c = 0; c < 12; ++c) s += e->B[r][c] * xl[c];
    if (blocks & 8) for (int c = 0; c < 4; ++c) s -= (delta * imu) * e->C[r][c] * xl[12 + c];
    yl[12 + r] = s;
  }
  for (int m = 0; m < 4; ++m) {
    if (vk[m] < kv0 || vk[m] >= kv1) continue;
    for (int a = 0; a < 3; ++a)
      if (!((dir[m] >> a) & 1)) y[a * V + vid[m]] += yl[a * 4 + m];
    y[3 * V + vid[m]] += yl[12 + m];
  }
}

/* y rows of vertex planes [kv0, kv1) (all 4 fields), field-major arrays.
 * x holds the full grid (4 x V); y holds the full grid too (rows outside
 * [kv0,kv1) untouched).  Returns 0. */
int ora_apply_slab(int n, int form, double delta, const int32_t* faces, const double* emu,
                   const double* eimu, const double* x, double* y, int kv0, int kv1,
                   unsigned blocks) {
  const int64_t N1 = n + 1, V = N1 * N1 * N1;
  elem_t E[6];
  build_elements(1.0 / n, E);
  for (int f = 0; f < 4; ++f)
    for (int64_t v = (int64_t)kv0 * N1 * N1; v < (int64_t)kv1 * N1 * N1; ++v) y[f * V + v] = 0.0;
  int c0 = kv0 - 1 < 0 ? 0 : kv0 - 1, c1 = kv1 < n ? kv1 : n;
  for (int phase = 0; phase < 2; ++phase) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int ck = c0; ck < c1; ++ck) {
      if ((ck & 1) != phase) continue;
      for (int cj = 0; cj < n; ++cj)
        for (int ci = 0; ci < n; ++ci)
          for (int t = 0; t < 6; ++t) {
            int64_t eid = 6 * (ci + (int64_t)n * (cj + (int64_t)n * ck)) + t;
            element_apply(n, form, delta, faces, &E[t], emu[eid], eimu[eid], ci, cj, ck, x, y, V,
                          blocks, kv0, kv1);
          }
    }
  }
  return 0;
}

/* rows (4 fields) of the listed vertices: out[4*s + f].  Loops over the 24
 * elements incident to each vertex and keeps only that vertex's rows. */
int ora_apply_rows(int n, int form, double delta, const int32_t* faces, const double* emu,
                   const double* eimu, const double* x, const int64_t* verts, int64_t nverts,
                   double* out) {
  const int64_t N1 = n + 1, V = N1 * N1 * N1;
  elem_t E[6];
  build_elements(1.0 / n, E);
#pragma omp parallel for schedule(static)
  for (int64_t s = 0; s < nverts; ++s) {
    int64_t v = verts[s];
    int i = (int)(v % N1), j = (int)((v / N1) % N1), k = (int)(v / (N1 * N1));
    double acc[4] = {0, 0, 0, 0};
    for (int dk = -1; dk <= 0; ++dk)
      for (int dj = -1; dj <= 0; ++dj)
        for (int di = -1; di <= 0; ++di) {
          int ci = i + di, cj = j + dj, ck = k + dk;
          if (ci < 0 || cj < 0 || ck < 0 || ci >= n || cj >= n || ck >= n) continue;
          for (int t = 0; t < 6; ++t) {
            const elem_t* e = &E[t];
            int m = -1;
            for (int q = 0; q < 4; ++q)
              if (e->off[q][0] == -di && e->off[q][1] == -dj && e->off[q][2] == -dk) m = q;
            if (m < 0) continue;
            /* full element product into a scratch row set, keep row m */
            double xl[16];
            int dir[4];
            int64_t vid[4];
            for (int q = 0; q < 4; ++q) {
              int ii = ci + e->off[q][0], jj = cj + e->off[q][1], kk = ck + e->off[q][2];
              dir[q] = elim_bits(n, faces, ii, jj, kk);
              vid[q] = ii + N1 * (jj + N1 * (int64_t)kk);
              for (int a = 0; a < 3; ++a) xl[a * 4 + q] = ((dir[q] >> a) & 1) ? 0.0 : x[a * V + vid[q]];
              xl[12 + q] = x[3 * V + vid[q]];
            }
            int64_t eid = 6 * (ci + (int64_t)n * (cj + (int64_t)n * ck)) + t;
            double mu = emu[eid], imu = eimu[eid];
            const double (*A)[12] = e->A[form];
            for (int a = 0; a < 3; ++a) {
              int r = a * 4 + m;
              double sum = 0.0;
              for (int c = 0; c < 12; ++c) sum += mu * A[r][c] * xl[c];
              for (int c = 0; c < 4; ++c) sum += e->B[c][r] * xl[12 + c];
              acc[a] += sum;
            }
            double sp = 0.0;
            for (int c = 0; c < 12; ++c) sp += e->B[m][c] * xl[c];
            for (int c = 0; c < 4; ++c) sp -= (delta * imu) * e->C[m][c] * xl[12 + c];
            acc[3] += sp;
          }
        }
    int d = elim_bits(n, faces, i, j, k);
    for (int a = 0; a < 3; ++a) out[4 * s + a] = ((d >> a) & 1) ? 0.0 : acc[a];
    out[4 * s + 3] = acc[3];
  }
  return 0;
}

/* diagonals of A (3 x V, per component) and C (V) by the element loop */
int ora_diag(int n, int form, double delta, const int32_t* faces, const double* emu,
             const double* eimu, double* dA, double* dC) {
  const int64_t N1 = n + 1, V = N1 * N1 * N1;
  elem_t E[6];
  build_elements(1.0 / n, E);
  memset(dA, 0, sizeof(double) * 3 * V);
  memset(dC, 0, sizeof(double) * V);
  for (int ck = 0; ck < n; ++ck)
    for (int cj = 0; cj < n; ++cj)
      for (int ci = 0; ci < n; ++ci)
        for (int t = 0; t < 6; ++t) {
          const elem_t* e = &E[t];
          const int64_t eid = 6 * (ci + (int64_t)n * (cj + (int64_t)n * ck)) + t;
          double mu = emu[eid], imu = eimu[eid];
          for (int m = 0; m < 4; ++m) {
            int64_t v = (ci + e->off[m][0]) + N1 * ((cj + e->off[m][1]) + N1 * (int64_t)(ck + e->off[m][2]));
            for (int a = 0; a < 3; ++a) dA[a * V + v] += mu * e->A[form][a * 4 + m][a * 4 + m];
            dC[v] += (delta * imu) * e->C[m][m];
          }
        }
  (void)faces;
  return 0;
}

int ora_num_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}
