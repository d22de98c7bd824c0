/* oracle/tacchi_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C, serial restatement of the reference's MLS-MPM substep and capture
 * path (see tacchi_oracle.c for the file:line each function follows). It is
 * the parity checker for the CUDA product: only tests/, smoke() and bench.py's
 * cpu_baseline leg may call it. It is pinned against the unmodified reference
 * (oracle/_ref) and the golden fixtures in tests/golden/.
 *
 * Layout ("row layout"): x, v as N x 3; C, F as N x 9 with M(i,j) at
 * [9p + 3i + j]. Grids are windows [lo, hi) stored k fastest.
 * Return codes follow include/tacchi_cuda.h (0 OK, 2 EmptyScene,
 * 3 OutOfGrid, 4 DegenerateF, ...).
 */
#ifndef TACCHI_ORACLE_H
#define TACCHI_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int res[3];
  double dx;
  double origin[3];
  double mu, lambda;
  double dt;
  double gravity[3];
} to_params;

typedef struct {
  double min_det_f;
  double max_speed;
  int64_t step_count;
} to_diag;

/* Tags (particle_set.hpp:12). */
enum { TO_ELASTOMER = 0, TO_ELASTOMER_BOTTOM = 1, TO_INDENTER = 2 };

int to_polar_rotation(const double F[9], double R[9]);
int to_polar_rotation_svd(const double F[9], double R[9]);
int to_corotated_stress(const double F[9], double mu, double lambda, double S[9]);
void to_stencil(const double x[3], const double origin[3], double inv_dx, int base[3],
                double w[3][3], double fx[3]);

/* zero_grid's window; returns 3 (OutOfGrid) when it leaves the grid. */
int to_window(const to_params* p, long n, const double* x, int lo[3], int hi[3]);
/* P2G into a zeroed window; min_det_f seeded with 1.0 as engine.cpp:119. */
int to_p2g(const to_params* p, long n, const double* x, const double* v, const double* C,
           const double* F, const double* mass, const double* vol0, const uint8_t* tag,
           const int lo[3], const int hi[3], double* gmass, double* gmom, double* min_det_f);
void to_grid_update(const to_params* p, const int lo[3], const int hi[3], const double* gmass,
                    const double* gmom, double* gvel);
void to_g2p(const to_params* p, long n, const double* x, double* v, double* C, double* F,
            const uint8_t* tag, const int lo[3], const int hi[3], const double* gvel);
void to_apply_boundary(long n, double* v, const uint8_t* tag, const double vind[3]);
/* advect + in_range check (returns 3 after moving x, like engine.cpp:282-285). */
int to_advect(const to_params* p, long n, double* x, const double* v, double* max_speed);

/* mpm::step, n_substeps times. */
int to_step(const to_params* p, long n, double* x, double* v, double* C, double* F,
            const double* mass, const double* vol0, const uint8_t* tag, const double vind[3],
            int n_substeps, to_diag* diag);

/* Render path (depth_extract.cpp, depth_map.cpp, phong.cpp). */
int to_extract_depth(int nx, int ny, const double geom[5], const uint32_t* surf_idx,
                     const double* x, int w, int h, double r, double* out);
void to_full_depth_size(int nx, int ny, const double geom[5], double r, int* w, int* h);
int to_crop_align(const double* src, int sw, int sh, double off_x, double off_y, double scale,
                  int ow, int oh, double* out);
int to_surface_normals(const double* depth, int w, int h, double r, double* out);
/* render = {ka, kd, ks, shininess, ambient[3], view[3]}; lights n x 9
 * (direction, diffuse, specular); bg is h*w*3 or NULL. */
int to_phong(const double* depth, int w, int h, double r, const double* lights, int n_lights,
             const double render[10], const uint8_t* bg, uint8_t* out);

#ifdef __cplusplus
}
#endif
#endif
