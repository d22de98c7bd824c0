/* tacchi_cuda.h — C-ABI of the B200-native Tacchi hot path (libtacchi_cuda.so).
 *
 * This is the drop-in boundary for the reference's C++ simulator API
 * (/root/reference/proj). Each entry point names the reference interface it
 * replaces (file:line). Plain pointers and sizes only; no C++ or torch types.
 *
 * Conventions
 *   - All physical quantities are SI, fp64, exactly as the reference.
 *   - Particle arrays use the reference's particle order: elastomer particles
 *     [0, n_elastomer) in lattice order (i, j, k), k fastest
 *     (particle_set.hpp:16-17, scene.cpp:54-60), then the indenter in cloud
 *     order. Vectors are N x 3 row-major; matrices N x 9 with M(i,j) at
 *     [9p + 3i + j].
 *   - Every function returns TG_OK (0) or a TG_ERR_* code; the message of the
 *     last error on the calling thread is available from tg_last_error().
 *     The codes map 1:1 onto the reference exception taxonomy
 *     (errors.hpp:9-39); the C++ wrapper (tacchi_b200.hpp) rethrows the
 *     matching class.
 *   - A handle owns all of its device memory and one CUDA stream. Calls on one
 *     handle must be serialised by the caller (one control thread per
 *     SimState); different handles may be driven concurrently.
 *   - No CPU fallback: if no sm_100 device is present every constructor fails
 *     with TG_ERR_CUDA.
 */
#ifndef TACCHI_CUDA_H
#define TACCHI_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  TG_OK = 0,
  TG_ERR_GRID_TOO_SMALL = 1,    /* tacchi::GridTooSmall    errors.hpp:17 */
  TG_ERR_EMPTY_SCENE = 2,       /* tacchi::EmptyScene      errors.hpp:18 */
  TG_ERR_OUT_OF_GRID = 3,       /* tacchi::OutOfGrid       errors.hpp:19 */
  TG_ERR_DEGENERATE_F = 4,      /* tacchi::DegenerateF     errors.hpp:20 */
  TG_ERR_CONFIG = 5,            /* tacchi::ConfigError     errors.hpp:38 */
  TG_ERR_NO_SURFACE = 6,        /* tacchi::NoSurface       errors.hpp:27 */
  TG_ERR_CROP_OUT_OF_BOUNDS = 7,/* tacchi::CropOutOfBounds errors.hpp:28 */
  TG_ERR_SHAPE_MISMATCH = 8,    /* tacchi::ShapeMismatch   errors.hpp:31 */
  TG_ERR_EMPTY_CLOUD = 9,       /* tacchi::EmptyCloud      errors.hpp:24 */
  TG_ERR_PARSE = 10,            /* tacchi::ParseError      errors.hpp:23 */
  TG_ERR_IO = 11,               /* tacchi::IoError         errors.hpp:39 */
  TG_ERR_SESSION_NOT_INITIALIZED = 12, /* tacchi::SessionNotInitialized errors.hpp:32 */
  TG_ERR_NON_MONOTONIC_TIME = 13,      /* tacchi::NonMonotonicTime      errors.hpp:33 */
  TG_ERR_PROTOCOL = 14,                /* tacchi::ProtocolError         errors.hpp:34 */
  TG_ERR_MANIFEST_MISMATCH = 15,       /* tacchi::ManifestMismatch      errors.hpp:37 */
  TG_ERR_CUDA = 20,             /* device / driver failure (no reference analogue) */
  TG_ERR_INVALID_ARGUMENT = 21  /* null handle / bad sizes (no reference analogue) */
};

/* Phase ids for tg_phase, in engine.hpp order. */
enum {
  TG_PHASE_ZERO_GRID = 0,        /* mpm::zero_grid         engine.hpp:10  */
  TG_PHASE_PARTICLE_TO_GRID = 1, /* mpm::particle_to_grid  engine.hpp:15  */
  TG_PHASE_GRID_UPDATE = 2,      /* mpm::grid_update       engine.hpp:19  */
  TG_PHASE_GRID_TO_PARTICLE = 3, /* mpm::grid_to_particle  engine.hpp:23  */
  TG_PHASE_APPLY_BOUNDARY = 4,   /* mpm::apply_boundary    engine.hpp:27  */
  TG_PHASE_ADVECT = 5            /* mpm::advect            engine.hpp:31  */
};

typedef struct tg_sim* tg_handle;

/* mpm::SceneParams (sim_state.hpp:81-98) after Grid construction. */
typedef struct {
  int res[3];             /* grid nodes per axis */
  double dx;              /* node spacing = grid_edge / res.x (scene.cpp:41-42) */
  double origin[3];
  double youngs_modulus;  /* MaterialParams (material.hpp:9-19) */
  double poisson_ratio;
  double density;
  double dt;
  double gravity[3];
} tg_params;

/* Particle state as init_scene builds it (scene.cpp:28-87). mass / volume0
 * must be uniform per material (they are, by construction of init_scene). */
typedef struct {
  int64_t n;              /* total particles */
  int64_t n_elastomer;    /* elastomer particles occupy [0, n_elastomer) */
  const double* x;        /* n x 3 */
  const double* v;        /* n x 3 */
  const double* C;        /* n x 9, may be NULL (zeros) */
  const double* F;        /* n x 9, may be NULL (identity) */
  const double* mass;     /* n */
  const double* volume0;  /* n */
  const uint8_t* tag;     /* n: 0 elastomer, 1 elastomer bottom, 2 indenter */
  double indenter_velocity[3]; /* SimState::indenter_velocity */
} tg_particles;

/* mpm::SurfaceLattice (sim_state.hpp:41-52). */
typedef struct {
  int nx, ny;
  double x0, y0, sx, sy, z0;
  const uint32_t* particle; /* nx*ny particle indices, x-major */
} tg_surface;

/* Per-frame capture parameters: sim::capture's inputs resolved from
 * SceneConfig (scene_builder.cpp:80-89, scene_config.cpp:70-81). */
typedef struct {
  double pixel_to_meter;    /* full-surface extraction pitch r */
  double crop_offset[2];    /* CropAlignment offset_x / offset_y (pixels) */
  double crop_scale;        /* CropAlignment scale */
  int width, height;        /* output image (640 x 480) */
  double ambient_k, diffuse_k, specular_k, shininess;
  double ambient_rgb[3];
  double view_dir[3];
  int n_lights;             /* <= 8 */
  double lights[8][9];      /* direction, diffuse_rgb, specular_rgb */
  const uint8_t* background;/* optional height x width x 3 RGB, or NULL */
} tg_render;

/* mpm::SceneParams (sim_state.hpp:81-98): init_scene's own parameters. */
typedef struct {
  int grid_resolution[3];     /* nodes per axis */
  double grid_edge;           /* m; node spacing = grid_edge / grid_resolution[0] */
  double grid_origin[3];
  double youngs_modulus, poisson_ratio, density;  /* MaterialParams */
  double dt;
  int fixed_bottom_layers;    /* lattice layers k < this are ElastomerBottom */
  double gravity[3];
  double indenter_mass_scale; /* default 80 */
} tg_scene_params;

/* An elastomer geo::ParticleSet with its LatticeMeta (particle_set.hpp:18-30). */
typedef struct {
  int counts[3];              /* particles per axis, >= 2 */
  double dims[3];             /* extent spanned by the lattice, m */
  double origin[3];           /* position of particle (0, 0, 0), m */
  const double* positions;    /* counts[0]*counts[1]*counts[2] x 3 in lattice order
                                 ((i*ny + j)*nz + k), or NULL for
                                 make_elastomer_lattice(dims, counts, origin) */
} tg_lattice;

/* ---- scene setup ------------------------------------------------------- */

/* mpm::init_scene(params, elastomer, indenter, indenter_velocity)
 * (sim_state.hpp:102-104, scene.cpp:28-87) from its own inputs: margins,
 * rest volumes and masses (indenter mass x indenter_mass_scale), bottom-layer
 * tags, the surface lattice and the initial velocities are computed here.
 * indenter: n_indenter x 3 placed points (m); indenter_velocity may be NULL
 * (zero). Errors: EmptyScene, GridTooSmall, ConfigError. */
int tg_init_scene(int device, const tg_scene_params* params, const tg_lattice* elastomer,
                  const double* indenter, int64_t n_indenter, const double indenter_velocity[3],
                  tg_handle* out);

/* sim::build_sim(cfg, indenter) (scene_builder.hpp:29-30,
 * scene_builder.cpp:63-78) with a caller's placed indenter points
 * (n_indenter x 3, m), e.g. a co-simulation's own object geometry. */
int tg_build_sim_points(int device, const char* config_json, const double* indenter,
                        int64_t n_indenter, tg_handle* out);

/* mpm::init_scene (sim_state.hpp:102-104) from explicit arrays. */
int tg_create(int device, const tg_params* params, const tg_particles* particles,
              const tg_surface* surface, tg_handle* out);

/* sim::build_sim(cfg, place_for_press(cfg, indenter_cloud_for(cfg, object),
 * offset_x, offset_y)) (scene_builder.cpp:33-78): the full reference setup
 * path from a SceneConfig JSON (partial overrides of default_config,
 * scene_config.cpp:118-257). */
int tg_build_sim(int device, const char* config_json, const char* object, double offset_x,
                 double offset_y, tg_handle* out);

/* Config-4 episodes / harness positions of one object: the indenter cloud
 * (indenter_cloud_for, scene_builder.cpp:33-46) is built once and shared;
 * episode e is build_sim(cfg with z_rotation_rad = poses[3e+2],
 * place_for_press(cfg, cloud, poses[3e], poses[3e+1])) on `device`.
 * out: n_episodes handles (all destroyed again if any creation fails). */
int tg_build_episodes(int device, const char* config_json, const char* object, int n_episodes,
                      const double* poses, tg_handle* out);

void tg_destroy(tg_handle h);

/* Host-side geometry of the setup path (no device work):
 * geo::generate_shape_cloud (shapes.cpp:231-249), out is n x 3 metres, and
 * indenter_cloud_for + place_for_press (scene_builder.cpp:33-61); call the
 * latter with out == NULL to query *n. */
int tg_generate_cloud(const char* shape, int64_t n, uint64_t seed, double* out);
/* The same rejection sampling on `device` (setup_kernels.cu: the mt19937_64
 * stream twisted in shared memory, candidates tested and compacted in stream
 * order); bit-identical to tg_generate_cloud. tg_build_sim and
 * tg_build_episodes sample generated indenters this way (TACCHI_HOST_SETUP=1
 * selects the host restatement). */
int tg_generate_cloud_device(int device, const char* shape, int64_t n, uint64_t seed, double* out);
int tg_placed_indenter(const char* config_json, const char* object, double offset_x,
                       double offset_y, double* out, int64_t* n);

/* ---- stepping (engine.hpp) --------------------------------------------- */

/* mpm::step(state, indenter_velocity, n_substeps) (engine.cpp:288-297).
 * Asynchronous on the handle's stream except for one completion/error check
 * at the end; errors raised on device are latched and reported with the
 * reference's semantics (state left as at the failing phase). */
int tg_step(tg_handle h, const double indenter_velocity[3], int n_substeps);

/* The six phases individually (engine.cpp:53-286), for unit parity. */
int tg_phase(tg_handle h, int phase, const double indenter_velocity[3]);

/* ---- state transfer --------------------------------------------------- */

int64_t tg_num_particles(tg_handle h);
int64_t tg_num_elastomer(tg_handle h);
/* Any output pointer may be NULL. Reference particle order. */
int tg_download(tg_handle h, double* x, double* v, double* C, double* F);
int tg_upload(tg_handle h, const double* x, const double* v, const double* C, const double* F);
/* StepDiagnostics + step_count + indenter_velocity (sim_state.hpp:54-73). */
int tg_diag(tg_handle h, double* min_det_f, double* max_speed, int64_t* step_count,
            double indenter_velocity[3]);
/* ParticleStore::mass / volume0 / tag (sim_state.hpp:17-37), reference order;
 * any output may be NULL. */
int tg_download_constants(tg_handle h, double* mass, double* volume0, uint8_t* tag);
/* Grid::active_lo / active_hi (grid.hpp:25-26): the window of the last
 * zero_grid (after mpm::step, the last substep's). */
int tg_grid_window(tg_handle h, int lo[3], int hi[3]);
/* Node box [lo, hi) (k fastest) of Grid::mass / momentum / velocity as the
 * reference holds them (zero outside the active window); any output may be
 * NULL. Valid after the phase functions, after creation, and after tg_step /
 * tg_step_capture on a handle with tg_set_keep_grid(h, 1); after a fused step
 * (the default) it returns TG_ERR_INVALID_ARGUMENT: that grid holds the next
 * substep's look-ahead scatter. */
int tg_download_grid(tg_handle h, const int lo[3], const int hi[3], double* mass, double* momentum,
                     double* velocity);
/* Deterministic mode (SceneConfig::deterministic, scene_config.hpp:78; SPEC
 * "Concurrency Model", acceptance 10): with enabled != 0 the node sums that
 * several CTAs / warps add to are accumulated as 64-bit fixed point, so
 * reruns with identical inputs give bit-identical states. tg_build_sim /
 * tg_build_sim_points / tg_build_episodes honour the config flag (default
 * true); tg_create / tg_init_scene start in the fp64 fast mode. */
int tg_set_deterministic(tg_handle h, int enabled);
/* With enabled != 0 the last substep of every tg_step / tg_step_capture runs
 * the six phases (engine.cpp:288-297) instead of the fused plan, so the grid
 * afterwards is the reference's post-step grid (engine.cpp:180-205). Default
 * off (the fused plan is faster and its particle results are the same). */
int tg_set_keep_grid(tg_handle h, int enabled);

/* ---- capture (render) -------------------------------------------------- */

/* Resolves sim::capture's render inputs from a SceneConfig JSON + object name
 * (lights, render params, alignment_for(object)). */
int tg_render_from_config(const char* config_json, const char* object, tg_render* out);

/* sim::capture (scene_builder.cpp:80-89): extract_surface_depth (full
 * surface at pixel_to_meter) -> crop_align -> phong_render, fused on device.
 * depth_out: height x width fp64 (DepthMap::values, row-major); rgb_out:
 * height x width x 3 (Image8::data). Either may be NULL (device-only). */
int tg_capture(tg_handle h, const tg_render* r, double* depth_out, uint8_t* rgb_out);

/* The handle's pinned host buffers for r's capture (height x width fp64 and
 * height x width x 3 u8). Passing them as tg_capture / tg_step_capture
 * outputs skips the host copy; their content is replaced by the next capture. */
int tg_capture_buffers(tg_handle h, const tg_render* r, double** depth, uint8_t** rgb);

/* One control step of Session::handle_command (session.cpp:86, 42):
 * mpm::step(state, v, n) then sim::capture, submitted together with a single
 * host synchronisation. Errors are mpm::step's; outputs as tg_capture. */
int tg_step_capture(tg_handle h, const double indenter_velocity[3], int n_substeps,
                    const tg_render* r, double* depth_out, uint8_t* rgb_out);

/* Pipelined control steps, for a caller that can take frame k's outputs
 * while frame k+1 runs (a dataset writer, a batch consumer): submit enqueues
 * mpm::step(v, n) + sim::capture(r) + the depth / RGB read-back into one of
 * two pinned slots of the handle and returns at once (*ticket = the frame's
 * number); wait (tickets in order) blocks until that frame is done and points
 * *depth / *rgb at its slot, valid until the submit after next. At most two
 * frames in flight; no other call on the handle while frames are in flight.
 * A frame's error is reported by its wait; a frame submitted after a failing
 * one reports it too (it ran as a no-op). n <= 200. read_back = 0 keeps the
 * frame's depth / RGB on the device (wait then returns NULL pointers). Only
 * the surface gather runs on the handle's stream; the shading and the
 * read-back run on a second stream beside the next frame's substeps. */
int tg_step_capture_submit(tg_handle h, const double indenter_velocity[3], int n_substeps,
                           const tg_render* r, int read_back, int64_t* ticket);
int tg_step_capture_wait(tg_handle h, int64_t ticket, double** depth, uint8_t** rgb);

/* render::extract_surface_depth(state, w, h, r) (depth_extract.cpp:10-49);
 * w <= 0 or h <= 0 selects the full-surface overload (:51-57) and returns
 * its size in *out_w / *out_h (call with out == NULL to query). */
int tg_extract_depth(tg_handle h, int w, int hgt, double r, double* out, int* out_w, int* out_h);

/* render::crop_align (depth_map.cpp:62-101) on a host depth map. */
int tg_crop_align(int device, const double* src, int sw, int sh, double off_x, double off_y,
                  double scale, int ow, int oh, double* out);
/* render::surface_normals (phong.cpp:10-41): out is h x w x 3. */
int tg_surface_normals(int device, const double* depth, int w, int hgt, double r, double* out);
/* render::phong_render (phong.cpp:43-84) on a host depth map; r is
 * DepthMap::pixel_to_meter, render->lights / params as above. */
int tg_phong_render(int device, const double* depth, int w, int hgt, double r,
                    const tg_render* render, uint8_t* out);

/* ---- batched episodes (config 4) --------------------------------------- */

/* Steps several handles that live on the same device in one pass of
 * launches (one stream each, submitted back to back). */
int tg_step_many(tg_handle* hs, int n_handles, const double* velocities /* n x 3 */,
                 int n_substeps);
/* Batched control step (config 4 / the harness's capture levels): for every
 * handle mpm::step(v_i, n_substeps) then sim::capture with renders[i] (or
 * renders[0] when n_renders == 1), all submitted before any wait. depth_outs /
 * rgb_outs: n pointers each (or NULL), entries as tg_capture's outputs (NULL =
 * not read back). status (optional, n ints) receives each handle's code; the
 * return value is the first failing handle's, with its message. A failing
 * handle does not stop the others. n_substeps <= 200 (the harness's chunk). */
int tg_step_capture_many(tg_handle* hs, int n_handles, const double* velocities /* n x 3 */,
                         int n_substeps, const tg_render* renders, int n_renders,
                         double** depth_outs, uint8_t** rgb_outs, int* status);

/* ---- runtime ------------------------------------------------------------ */

/* Blocks until the handle's stream is idle; reports any latched error. */
int tg_sync(tg_handle h);
/* Runs one mpm::step of `reps` substeps kernel by kernel with CUDA events
 * between the launches and writes device times (ms): [p2g_elastomer and
 * p2g_indenter of the first substep, then per-substep averages of
 * grid_update, g2p2g_elastomer (G2P + boundary + advect + look-ahead P2G),
 * indenter_move_p2g, finalize]. The state advances exactly as tg_step
 * would. Instrumentation for the roofline in bench.py. */
int tg_time_phases(tg_handle h, const double indenter_velocity[3], int reps, double* out_ms);
/* Instrumentation counters of a handle: [0] kernels launched, [1] node-array
 * reallocations (the grid arrays cover a box of the logical grid and grow
 * on demand), [2] bytes of the node arrays, [3] substeps whose indenter
 * look-ahead walks finalize completed (the elastomer left the walks' box),
 * [4] allocated nodes, [5] cached substep graphs, [6] indenter particles
 * advected by the column walks so far (the rest are caught up in bulk). */
int tg_stats(tg_handle h, int64_t out[7]);
/* cudaStream_t of the handle (for event timing by the caller). */
void* tg_stream(tg_handle h);
/* Number of kernels this handle has launched so far (graph nodes count). */
int64_t tg_kernel_launches(tg_handle h);
/* Enables / disables CUDA-graph replay of the substep loop (default on). */
int tg_set_graphs(tg_handle h, int enabled);
/* mpm::polar_rotation / polar_rotation_svd + corotated_stress
 * (material.cpp:18-89) of n row-major 3x3 matrices F on `device`, through the
 * device functions the P2G kernels call. mode 0: polar_rotation (scaled
 * Newton with its SVD fallback), 1: polar_rotation_svd directly (the
 * fallback). S (may be NULL) receives corotated_stress(F) with that R.
 * Instrumentation for the material known-answer tests. */
int tg_polar(int device, const double* F, int64_t n, int mode, double youngs_modulus,
             double poisson_ratio, double* R, double* S);
const char* tg_last_error(void);
const char* tg_version(void);

/* ---- co-simulation bridge, protocol "tacchi/1" (§8 row f1) ---------------
 * bridge::run_protocol (server.cpp:49-113) over in-memory lines: `input` is
 * newline-separated JSON messages (init / step / end); the reply lines are
 * returned in *output (malloc'd, release with tg_free). Each session runs
 * on `device` through the B200 step + capture path and writes
 * step_NNNNNN.png / .depth and steps.jsonl like bridge::Session
 * (session.cpp:36-98). `base_config_json` is the SceneConfig used by an
 * init without "config"/"config_path"; sessions without "session_dir" go to
 * `session_root`/session_<k>. */
int tg_bridge_run(int device, const char* base_config_json, const char* session_root,
                  const char* input, char** output);
/* bridge::serve_stdio (port < 0) or bridge::serve_tcp on 127.0.0.1:port
 * (server.cpp:115-182); max_connections = 0 serves forever. */
int tg_bridge_serve(int device, const char* base_config_json, const char* session_root,
                    int port, int max_connections);
void tg_free(void* p);

/* ---- dataset harness and metrics (§8 rows f2, f4) ------------------------
 * dataset::run_press_dataset (harness.cpp:159-245): every object of the
 * SceneConfig at every press-grid position, pressed at press_speed_mm_s with
 * one capture per depth level -> out_dir/{config.json, manifest.csv,
 * images/<stem>.png, depth/<stem>.depth}; complete (object, position) groups of an
 * existing manifest are kept (resume). `batch` simulations are stepped
 * together on `device` (0: config "workers", else 16). */
int tg_run_press_dataset(int device, const char* config_json, const char* out_dir, int batch,
                         int64_t* rows, int64_t* skipped_positions);
/* dataset::compare_datasets (harness.cpp:247-321); out[7] = pairs, ssim
 * mean/std, psnr mean/std, mae mean/std; per-pair CSV when csv_out != "". */
int tg_compare_datasets(int device, const char* dir_a, const char* dir_b, const char* csv_out,
                        double* out);
/* metrics::ssim / psnr / mae (image_metrics.cpp:57-112) for `count` pairs of
 * h x w x 3 uint8 images (pair-major) in one device launch; out: count x 3. */
int tg_image_metrics(int device, const uint8_t* a, const uint8_t* b, int w, int h, int count,
                     double* out);
/* render::load_png / save_png (image.cpp:23-90); load with rgb == NULL
 * queries the size. */
int tg_load_png(const char* path, uint8_t* rgb, int* w, int* h);
int tg_save_png(const char* path, const uint8_t* rgb, int w, int h);

#ifdef __cplusplus
}
#endif
#endif /* TACCHI_CUDA_H */
