/*
 * icl_oracle.c -- CPU reference ("oracle") for the ImageCL hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the CUDA library
 * under paper_1605_06399_b200/) may include, link or call this file; only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg use it.  It shares no code, header, table or constant with
 * the CUDA side; the only common module is synth/ (seeded inputs).
 *
 * Every function below is the plain definition of what the filter computes,
 * evaluated pixel by pixel in double precision with no blocking, fusion or
 * re-association beyond what the definition states.  Inputs are the same fp32
 * arrays and fp32 parameters the GPU receives, promoted to double, so parity
 * measures only the GPU's arithmetic error.
 *
 * Definitions and citations
 *   Boundary read in_B (§5 Fig. 3 "Clamped: values
 *     outside are set to that of the closest pixel inside the image",
 *     "Constant: values outside the image are set to some constant, e.g. 0";
 *     row-major linearisation per SPEC.md:352).
 *   Separable convolution (§6, Table 2 R/C kernels,
 *     Listing 1 access form in[idx+i][idy+j]):
 *       out(x,y) = sum_j g_j * sum_i f_i * in_B(x+i, y+j)   (correlation,
 *       DESIGN.md reading R1).
 *   Harris (§6, Tables 4-5: a Sobel kernel producing dx, dy
 *     images, then a Harris kernel over a block window), per-stage semantics
 *     (readings R6-R10): dx, dy are Images with their own boundary.
 *   Non-local means: NOT in PAPER.md (BASELINE.json north_star only);
 *     standard Buades-Coll-Morel form with the readings R11-R14 of DESIGN.md.
 *   Non-separable convolution of an 8-bit image (§6, "a
 *     8192x8192 image with pixels of type unsigned char, a 5x5 filter, and
 *     clamped boundary condition"; filter values known only at run time,
 *     PAPER.md:577-579; Table 3):
 *       out(x,y) = sum_{j=-r..r} sum_{i=-r..r} f[j+r][i+r] * in_B(x+i, y+j)
 *     (correlation, reading R1; real-valued output, reading R22).
 *   3-D separable convolution of a volume (ImageCL Images "support 2D/3D
 *     indexing"; R26): the
 *     sepconv definition with a third axis and the boundary applied per axis,
 *       out(x,y,z) = sum_k h_k sum_j g_j sum_i f_i in_B(x+i, y+j, z+k).
 *
 * Threading: the point list is split into contiguous chunks, one pthread per
 * chunk; each output is computed independently in a fixed order, so results
 * do not depend on the thread count.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <unistd.h>

#define OR_BORDER_CONSTANT 0
#define OR_BORDER_CLAMP 1

typedef struct {
    const float* u;
    int64_t W, H, pitch; /* pitch in elements */
    int border;
    double c;
} oimg;

static int64_t clampi(int64_t v, int64_t lo, int64_t hi) {
    return v < lo ? lo : (v > hi ? hi : v);
}

/* in_B(x, y): PAPER.md Fig. 3 / SPEC.md:352. */
static double read_B(const oimg* im, int64_t x, int64_t y) {
    if (x < 0 || x >= im->W || y < 0 || y >= im->H) {
        if (im->border == OR_BORDER_CONSTANT) return im->c;
        x = clampi(x, 0, im->W - 1);
        y = clampi(y, 0, im->H - 1);
    }
    return (double)im->u[y * im->pitch + x];
}

/* ------------------------------------------------------------------------ */
/* Separable convolution: out(x,y) = sum_{j=-ry..ry} g_j sum_{i=-rx..rx}     */
/*                                    f_i in_B(x+i, y+j)                       */
/* ------------------------------------------------------------------------ */
typedef struct {
    oimg im;
    const double* f; int rx;
    const double* g; int ry;
} sep_args;

static double sepconv_px(const sep_args* a, int64_t x, int64_t y) {
    double out = 0.0;
    for (int j = -a->ry; j <= a->ry; ++j) {
        double t = 0.0;
        for (int i = -a->rx; i <= a->rx; ++i) t += a->f[i + a->rx] * read_B(&a->im, x + i, y + j);
        out += a->g[j + a->ry] * t;
    }
    return out;
}

/* ------------------------------------------------------------------------ */
/* Harris corner response, per-stage semantics.                               */
/*   dx(q) = sum_{j,i in -1..1} Kx[j][i] in_B(q+(i,j)),  Kx = [1,2,1]^T[-1,0,1] */
/*   dy(q) = sum Ky[j][i] in_B(q+(i,j)),                 Ky = [-1,0,1]^T[1,2,1] */
/*   dx_B(q) = dx(q) inside; clamp: dx(clamp(q)); constant: 0.                 */
/*   Sxx = sum_{t in Win} dx_B(p+t)^2, Sxy = sum dx_B dy_B, Syy = sum dy_B^2   */
/*   Win = [-floor(B/2), B-1-floor(B/2)]^2                                    */
/*   R = Sxx*Syy - Sxy^2 - k (Sxx+Syy)^2                                      */
/* ------------------------------------------------------------------------ */
static const double SOB_V[3] = {1.0, 2.0, 1.0};  /* smoothing */
static const double SOB_D[3] = {-1.0, 0.0, 1.0}; /* central difference */

typedef struct {
    oimg im;
    int block;
    double k;
} harris_args;

static void sobel_B(const harris_args* a, int64_t qx, int64_t qy, double* dx, double* dy) {
    const oimg* im = &a->im;
    if (qx < 0 || qx >= im->W || qy < 0 || qy >= im->H) {
        if (im->border == OR_BORDER_CONSTANT) { *dx = 0.0; *dy = 0.0; return; }
        qx = clampi(qx, 0, im->W - 1);
        qy = clampi(qy, 0, im->H - 1);
    }
    double sx = 0.0, sy = 0.0;
    for (int j = -1; j <= 1; ++j)
        for (int i = -1; i <= 1; ++i) {
            double v = read_B(im, qx + i, qy + j);
            sx += SOB_V[j + 1] * SOB_D[i + 1] * v;
            sy += SOB_D[j + 1] * SOB_V[i + 1] * v;
        }
    *dx = sx;
    *dy = sy;
}

static double harris_px(const harris_args* a, int64_t x, int64_t y, double* sxx_o, double* sxy_o, double* syy_o) {
    int lo = -(a->block / 2), hi = a->block - 1 - a->block / 2;
    double sxx = 0.0, sxy = 0.0, syy = 0.0;
    for (int ty = lo; ty <= hi; ++ty)
        for (int tx = lo; tx <= hi; ++tx) {
            double dx, dy;
            sobel_B(a, x + tx, y + ty, &dx, &dy);
            sxx += dx * dx;
            sxy += dx * dy;
            syy += dy * dy;
        }
    *sxx_o = sxx; *sxy_o = sxy; *syy_o = syy;
    double tr = sxx + syy;
    return sxx * syy - sxy * sxy - a->k * tr * tr;
}

/* ------------------------------------------------------------------------ */
/* Non-local means (not in PAPER.md; readings R11-R14):             */
/*   for o in [-s,s]^2, q = p+o:                                              */
/*     d2 = (1/(2rho+1)^2) sum_{t in [-rho,rho]^2} (u_B(p+t) - u_B(q+t))^2    */
/*     w  = exp(-d2/h^2)  (w = 1 when h = +inf)                               */
/*     num += w u_B(q);  den += w                                              */
/*   out = num / den                                                           */
/* ------------------------------------------------------------------------ */
typedef struct {
    oimg im;
    int rho, s;
    double h;
} nlm_args;

static double nlm_px(const nlm_args* a, int64_t x, int64_t y, double* wmax) {
    const oimg* im = &a->im;
    const double P2 = (double)(2 * a->rho + 1) * (double)(2 * a->rho + 1);
    double num = 0.0, den = 0.0, amax = 0.0;
    for (int oy = -a->s; oy <= a->s; ++oy)
        for (int ox = -a->s; ox <= a->s; ++ox) {
            double d2 = 0.0;
            for (int ty = -a->rho; ty <= a->rho; ++ty)
                for (int tx = -a->rho; tx <= a->rho; ++tx) {
                    double diff = read_B(im, x + tx, y + ty) - read_B(im, x + ox + tx, y + oy + ty);
                    d2 += diff * diff;
                }
            d2 /= P2;
            double w = isinf(a->h) ? 1.0 : exp(-d2 / (a->h * a->h));
            double uq = read_B(im, x + ox, y + oy);
            num += w * uq;
            den += w;
            if (fabs(uq) > amax) amax = fabs(uq);
        }
    if (wmax) *wmax = amax;
    return num / den;
}

/* ------------------------------------------------------------------------ */
/* Non-separable convolution of an 8-bit image:                                */
/*   out(x,y) = sum_{j=-r..r} sum_{i=-r..r} f[j+r][i+r] * in_B(x+i, y+j)       */
/* ------------------------------------------------------------------------ */
typedef struct {
    const uint8_t* u;
    int64_t W, H, pitch; /* pitch in bytes == elements */
    int border;
    double c;
} oimg8;

/* in_B(x, y) of an 8-bit image: PAPER.md Fig. 3. */
static double read_B8(const oimg8* im, int64_t x, int64_t y) {
    if (x < 0 || x >= im->W || y < 0 || y >= im->H) {
        if (im->border == OR_BORDER_CONSTANT) return im->c;
        x = clampi(x, 0, im->W - 1);
        y = clampi(y, 0, im->H - 1);
    }
    return (double)im->u[y * im->pitch + x];
}

typedef struct {
    oimg8 im;
    const double* f; /* (2r+1)^2, row j major */
    int r;
} conv2d_args;

static double conv2d_px(const conv2d_args* a, int64_t x, int64_t y) {
    const int r = a->r, n = 2 * r + 1;
    double s = 0.0;
    for (int j = -r; j <= r; ++j)
        for (int i = -r; i <= r; ++i) s += a->f[(j + r) * n + (i + r)] * read_B8(&a->im, x + i, y + j);
    return s;
}

/* ------------------------------------------------------------------------ */
/* Point-list driver + pthreads                                                */
/* ------------------------------------------------------------------------ */
enum { F_SEP = 0, F_HARRIS = 1, F_NLM = 2, F_CONV2D = 3 };

typedef struct {
    int filter;
    const void* args;
    const int64_t* xs; const int64_t* ys; /* NULL: full image, row-major */
    int64_t W;
    int64_t begin, end;
    double* out;
    double* aux; /* harris: 3 per point (Sxx,Sxy,Syy); nlm: 1 per point (max|u_B|) */
} job_t;

static void* run_job(void* p) {
    job_t* jb = (job_t*)p;
    for (int64_t n = jb->begin; n < jb->end; ++n) {
        int64_t x = jb->xs ? jb->xs[n] : n % jb->W;
        int64_t y = jb->ys ? jb->ys[n] : n / jb->W;
        if (jb->filter == F_SEP) {
            jb->out[n] = sepconv_px((const sep_args*)jb->args, x, y);
        } else if (jb->filter == F_CONV2D) {
            jb->out[n] = conv2d_px((const conv2d_args*)jb->args, x, y);
        } else if (jb->filter == F_HARRIS) {
            double sxx, sxy, syy;
            jb->out[n] = harris_px((const harris_args*)jb->args, x, y, &sxx, &sxy, &syy);
            if (jb->aux) { jb->aux[3 * n] = sxx; jb->aux[3 * n + 1] = sxy; jb->aux[3 * n + 2] = syy; }
        } else {
            double m;
            jb->out[n] = nlm_px((const nlm_args*)jb->args, x, y, &m);
            if (jb->aux) jb->aux[n] = m;
        }
    }
    return NULL;
}

static int run_points(int filter, const void* args, int64_t W, int64_t npts, const int64_t* xs,
                      const int64_t* ys, double* out, double* aux, int nthreads) {
    if (nthreads <= 0) nthreads = (int)sysconf(_SC_NPROCESSORS_ONLN);
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    if ((int64_t)nthreads > npts) nthreads = npts > 0 ? (int)npts : 1;
    pthread_t th[256];
    int spawned[256];
    job_t jobs[256];
    int64_t chunk = (npts + nthreads - 1) / nthreads;
    for (int t = 0; t < nthreads; ++t) {
        jobs[t].filter = filter; jobs[t].args = args; jobs[t].xs = xs; jobs[t].ys = ys; jobs[t].W = W;
        jobs[t].begin = t * chunk < npts ? t * chunk : npts;
        jobs[t].end = (t + 1) * chunk < npts ? (t + 1) * chunk : npts;
        jobs[t].out = out; jobs[t].aux = aux;
        spawned[t] = 0;
        if (jobs[t].begin >= jobs[t].end) continue;
        /* the last chunk (or a chunk whose thread failed to spawn) runs on the caller */
        if (t != nthreads - 1 && pthread_create(&th[t], NULL, run_job, &jobs[t]) == 0)
            spawned[t] = 1;
        else
            run_job(&jobs[t]);
    }
    for (int t = 0; t < nthreads; ++t)
        if (spawned[t]) pthread_join(th[t], NULL);
    return 0;
}

static int check_img(const float* in, int64_t W, int64_t H, int64_t pitch, int border) {
    if (!in || W < 1 || H < 1 || pitch < W) return -1;
    if (border != OR_BORDER_CONSTANT && border != OR_BORDER_CLAMP) return -1;
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Exported API (ctypes).  xs/ys NULL => full image, out is W*H row-major.    */
/* Returns 0 on success, -1 on invalid arguments.                             */
/* ------------------------------------------------------------------------ */
int oracle_sepconv(const float* in, int64_t W, int64_t H, int64_t pitch, const float* fx, int rx,
                   const float* gy, int ry, int border, float c, const int64_t* xs, const int64_t* ys,
                   int64_t n, double* out, int nthreads) {
    if (check_img(in, W, H, pitch, border) || rx < 0 || ry < 0 || !fx || !gy || !out) return -1;
    double* f = (double*)malloc(sizeof(double) * (size_t)(2 * rx + 1));
    double* g = (double*)malloc(sizeof(double) * (size_t)(2 * ry + 1));
    for (int i = 0; i < 2 * rx + 1; ++i) f[i] = (double)fx[i];
    for (int j = 0; j < 2 * ry + 1; ++j) g[j] = (double)gy[j];
    sep_args a = {{in, W, H, pitch, border, (double)c}, f, rx, g, ry};
    int64_t npts = xs ? n : W * H;
    run_points(F_SEP, &a, W, npts, xs, ys, out, NULL, nthreads);
    free(f);
    free(g);
    return 0;
}

int oracle_harris(const float* in, int64_t W, int64_t H, int64_t pitch, int block, float k, int border,
                  float c, const int64_t* xs, const int64_t* ys, int64_t n, double* R, double* S,
                  int nthreads) {
    if (check_img(in, W, H, pitch, border) || block < 1 || !R) return -1;
    harris_args a = {{in, W, H, pitch, border, (double)c}, block, (double)k};
    int64_t npts = xs ? n : W * H;
    run_points(F_HARRIS, &a, W, npts, xs, ys, R, S, nthreads);
    return 0;
}

int oracle_nlm(const float* in, int64_t W, int64_t H, int64_t pitch, int rho, int s, float h, int border,
               float c, const int64_t* xs, const int64_t* ys, int64_t n, double* out, double* wmax,
               int nthreads) {
    if (check_img(in, W, H, pitch, border) || rho < 0 || s < 0 || !out) return -1;
    if (!(h > 0.0f)) return -1; /* h <= 0 or NaN (R14) */
    nlm_args a = {{in, W, H, pitch, border, (double)c}, rho, s, (double)h};
    int64_t npts = xs ? n : W * H;
    run_points(F_NLM, &a, W, npts, xs, ys, out, wmax, nthreads);
    return 0;
}

int oracle_conv2d_u8(const uint8_t* in, int64_t W, int64_t H, int64_t pitch, const float* filt, int r,
                     int border, float c, const int64_t* xs, const int64_t* ys, int64_t n, double* out,
                     int nthreads) {
    if (!in || W < 1 || H < 1 || pitch < W || r < 0 || !filt || !out) return -1;
    if (border != OR_BORDER_CONSTANT && border != OR_BORDER_CLAMP) return -1;
    const int nf = (2 * r + 1) * (2 * r + 1);
    double* f = (double*)malloc(sizeof(double) * (size_t)nf);
    for (int k = 0; k < nf; ++k) f[k] = (double)filt[k];
    conv2d_args a = {{in, W, H, pitch, border, (double)c}, f, r};
    int64_t npts = xs ? n : W * H;
    run_points(F_CONV2D, &a, W, npts, xs, ys, out, NULL, nthreads);
    free(f);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* 3-D separable convolution (plain triple sum over the boundary-extended     */
/* volume, pixel by pixel).                                                    */
/* ------------------------------------------------------------------------ */
typedef struct {
    const float* u;
    int64_t W, H, D, pitch, spitch; /* elements */
    int border;
    double c;
    const double *f, *g, *h;
    int rx, ry, rz;
    const int64_t *xs, *ys, *zs;
    int64_t begin, end;
    double* out;
} sep3_job;

static double read_B3(const sep3_job* a, int64_t x, int64_t y, int64_t z) {
    if (x < 0 || x >= a->W || y < 0 || y >= a->H || z < 0 || z >= a->D) {
        if (a->border == OR_BORDER_CONSTANT) return a->c;
        x = clampi(x, 0, a->W - 1);
        y = clampi(y, 0, a->H - 1);
        z = clampi(z, 0, a->D - 1);
    }
    return (double)a->u[z * a->spitch + y * a->pitch + x];
}

static void* sep3_run(void* p) {
    sep3_job* a = (sep3_job*)p;
    for (int64_t n = a->begin; n < a->end; ++n) {
        int64_t x, y, z;
        if (a->xs) { x = a->xs[n]; y = a->ys[n]; z = a->zs[n]; }
        else { x = n % a->W; y = (n / a->W) % a->H; z = n / (a->W * a->H); }
        double out = 0.0;
        for (int k = -a->rz; k <= a->rz; ++k) {
            double s = 0.0;
            for (int j = -a->ry; j <= a->ry; ++j) {
                double t = 0.0;
                for (int i = -a->rx; i <= a->rx; ++i) t += a->f[i + a->rx] * read_B3(a, x + i, y + j, z + k);
                s += a->g[j + a->ry] * t;
            }
            out += a->h[k + a->rz] * s;
        }
        a->out[n] = out;
    }
    return NULL;
}

int oracle_sepconv3d(const float* in, int64_t W, int64_t H, int64_t D, int64_t pitch, int64_t spitch,
                     const float* fx, int rx, const float* gy, int ry, const float* hz, int rz, int border,
                     float c, const int64_t* xs, const int64_t* ys, const int64_t* zs, int64_t n, double* out,
                     int nthreads) {
    if (!in || W < 1 || H < 1 || D < 1 || pitch < W || spitch < pitch * H || rx < 0 || ry < 0 || rz < 0 ||
        !fx || !gy || !hz || !out)
        return -1;
    if (border != OR_BORDER_CONSTANT && border != OR_BORDER_CLAMP) return -1;
    double* f = (double*)malloc(sizeof(double) * (size_t)(2 * rx + 1));
    double* g = (double*)malloc(sizeof(double) * (size_t)(2 * ry + 1));
    double* h = (double*)malloc(sizeof(double) * (size_t)(2 * rz + 1));
    for (int i = 0; i < 2 * rx + 1; ++i) f[i] = (double)fx[i];
    for (int j = 0; j < 2 * ry + 1; ++j) g[j] = (double)gy[j];
    for (int k = 0; k < 2 * rz + 1; ++k) h[k] = (double)hz[k];
    const int64_t npts = xs ? n : W * H * D;
    if (nthreads <= 0) nthreads = (int)sysconf(_SC_NPROCESSORS_ONLN);
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    if ((int64_t)nthreads > npts) nthreads = npts > 0 ? (int)npts : 1;
    pthread_t th[256];
    int spawned[256];
    sep3_job jobs[256];
    const int64_t chunk = (npts + nthreads - 1) / nthreads;
    for (int t = 0; t < nthreads; ++t) {
        sep3_job j = {in, W, H, D, pitch, spitch, border, (double)c, f, g, h, rx, ry, rz, xs, ys, zs,
                      t * chunk < npts ? t * chunk : npts, (t + 1) * chunk < npts ? (t + 1) * chunk : npts, out};
        jobs[t] = j;
        spawned[t] = 0;
        if (jobs[t].begin >= jobs[t].end) continue;
        if (t != nthreads - 1 && pthread_create(&th[t], NULL, sep3_run, &jobs[t]) == 0) spawned[t] = 1;
        else sep3_run(&jobs[t]);
    }
    for (int t = 0; t < nthreads; ++t)
        if (spawned[t]) pthread_join(th[t], NULL);
    free(f);
    free(g);
    free(h);
    return 0;
}

int oracle_nthreads_default(void) { return (int)sysconf(_SC_NPROCESSORS_ONLN); }
