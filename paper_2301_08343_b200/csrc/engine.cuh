// DeviceSim: the device-resident mpm::SimState (sim_state.hpp:59-79) and the
// launch plan of one substep. Internal; the public surface is tacchi_cuda.h.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <string>
#include <utility>
#include <vector>

#include "mpm_device.cuh"
#include "tacchi_cuda.h"

namespace tacchi_b200 {

// Device-resident control block: latched error, reductions, active windows,
// diagnostics and the commanded velocity. One per handle.
struct Ctl {
  // Latched error: (substep << 8) | code, ~0 when clear. atomicMin keeps the
  // earliest substep's error (and, within a substep, the lowest code: a real
  // error before an allocation regrow). One word, so a reader never sees a
  // code without its substep.
  unsigned long long err;
  int substep;       // absolute index of the substep being executed
  int pad0;
  // Motion reductions in two slots by substep parity: slot s & 1 holds the
  // state after the advect of substep s (so a reader of slot s & 1 and the
  // reset of slot (s + 1) & 1 for the next advect never touch the same slot).
  unsigned long long bb_lo[2][3], bb_hi[2][3];   // order_key() of elastomer x
  unsigned long long ind_lo[2][3], ind_hi[2][3];  // order_key() of the indenter bbox
  unsigned long long max_v2[2];                  // bits of max |v|^2 (non-negative)
  unsigned long long min_detf[2];         // order_key() of min det F, per substep parity
  int win_lo[3], win_hi[3];               // window of the next zero_grid (P2G of ctl->substep)
  int ref_lo[3], ref_hi[3];               // Grid::active_lo/hi as the reference holds them:
                                          // the window of the last zero_grid that ran
  int prev_lo[3], prev_hi[3];             // Grid::prev_lo/hi
  int clr_lo[3], clr_hi[3];               // node box to clear before P2G
  int box_lo[2][3], box_hi[2][3];         // per-material node boxes (elastomer, indenter)
  double vind[3];                         // commanded indenter velocity
  double ind_v[3];                        // uniform indenter velocity (P2G input)
  double ind_vp[2][3];                    // the indenter velocity of the M_I scatter of
                                          // substep s, slot s & 1 (grid_update's input)
  int mi_last;                            // substep of the last phase-path P2G (its M_I buffer)
  int pad1;
  int chain_start;                        // first substep of the open indenter chain
  double diag_min_det_f, diag_max_speed;  // StepDiagnostics
  long long step_count;                   // SimState::step_count
  long long walk_fixups;                  // substeps whose walks finalize completed
  unsigned long long ind_walked;          // indenter particles advected by the column walks
};
static_assert(sizeof(Ctl) % 8 == 0, "the control block is copied in 8-byte words");

struct Geometry {
  int res[3];
  // Node arrays cover the allocation box [ga_lo, ga_lo + ga_dim) of the
  // logical res^3 grid (node (i,j,k) at ((i-lo0)*d1 + (j-lo1))*d2 + (k-lo2)),
  // grown on demand (engine.cu ensure_alloc / regrow).
  int ga_lo[3], ga_dim[3];
  double dx, inv_dx;
  double origin[3];
  double mu, lambda;
  double dt;
  double gravity[3];
  double gdt[3];
  int with_gravity;
  double stress_scale;  // -dt * 4 * inv_dx^2 (engine.cpp:114)
  int scatter_mode;     // 0: shared-memory tile (default), 1: direct RED (A/B switch)
  int* cta_box;         // per elastomer CTA: {lo[3], dim[3], ok} of its last P2G tile
  int gu_bps;           // grid_update blocks per SM (TACCHI_GU_BPS, default 5)
  int pdl_early;        // grid_update triggers its dependent launch right after its
                        // own griddepcontrol.wait (TACCHI_PDL_EARLY, default 1)
  int gel_trigger;      // the elastomer kernel triggers its dependent launch at
                        // its start (TACCHI_GEL_TRIGGER, default 1)
  int det_skip0;        // deterministic conversion pass skips all-zero tile nodes
                        // (TACCHI_DET_SKIP0, default 1)
  int det_fast4;        // deterministic conversion: one magic addition per sum where
                        // a node's four fit 2^51 (TACCHI_DET_FAST4, default 1)
  int fin_trigger;      // finalize triggers its dependent launch before its own
                        // griddepcontrol.wait (TACCHI_FIN_TRIGGER, default 1)
  int ind_first;        // the indenter blocks of the elastomer kernel come first
                        // (TACCHI_IND_FIRST, default 1)
  // Deterministic mode (SceneConfig::deterministic, SPEC "Concurrency
  // Model"): node sums that several CTAs / warps add to are accumulated as
  // 64-bit fixed point (integer adds are exact, so the order does not
  // matter). A (mass, momentum) in units of 1 / fx_s, M_I in 1 / fxi_s;
  // both scales are powers of two.
  int det;
  double fx_s, fx_inv, fxi_s, fxi_inv;
  // M_I is double-buffered by substep parity (the walks of substep s scatter
  // into buffer (s + 1) & 1 while grid_update consumes buffer s & 1): the
  // second buffer starts mi_stride doubles after the first.
  size_t mi_stride;
};

// A dense node array in split layout: two 16-byte halves per node in two
// arrays (node (i,j,k) at (i*res1 + j)*res2 + k). Grid::mass/momentum:
// lo = {m, px}, hi = {py, pz}.
struct NodeBuf {
  double2* lo;
  double2* hi;
};

// Grid::velocity: xy = {vx, vy} (16 B) and z = vz (8 B) per node.
struct VelBuf {
  double2* xy;
  double* z;
};

// One frame of the pipelined control step (tg_step_capture_submit / _wait):
// its pinned outputs, a pinned snapshot of the control block taken after it,
// the event that marks its end, and what was asked (to replay it).
struct FrameSlot {
  double* depth = nullptr;
  uint8_t* rgb = nullptr;
  size_t pixels = 0;
  Ctl* ctl = nullptr;             // pinned snapshot of the control block after the frame
  Ctl* d_snap = nullptr;          // device copy of it, taken on the handle's stream
  cudaEvent_t captured = nullptr; // the frame's capture kernel (and snapshot) are done
  cudaEvent_t ev = nullptr;       // its read-back is done (copy stream)
  bool used = false;              // `ev` has been recorded at least once
  bool live = false;    // submitted, not yet waited for
  bool read_back = true;  // depth / RGB come back to the pinned slot
  bool replay = false;  // an earlier frame grew the node arrays: run this one again
  int status = 0;       // error to report at its wait (an earlier frame failed)
  std::string msg;
  double v[3] = {0, 0, 0};
  int n = 0;
  int end_substep = 0;
  tg_render r{};
};

// Internal return code of step_finish / phase: the node arrays were grown
// mid-call; DeviceSim::resume_substeps substeps remain (engine.cu).
constexpr int kResume = -100;

struct DeviceSim {
  int device = 0;
  cudaStream_t stream = nullptr;
  Geometry geo{};
  int64_t n = 0, n_el = 0, n_ind = 0;
  double m_el = 0, vol_el = 0, m_ind = 0, vol_ind = 0;

  // Particle state, SoA component-major: x[c * n + p].
  double* x = nullptr;   // 3 * n   (gel then indenter, internal order)
  double* v = nullptr;   // 3 * n
  double* C = nullptr;   // 9 * n_el
  double* F = nullptr;   // 9 * n_el
  uint8_t* tag = nullptr;  // n_el (Elastomer / ElastomerBottom)
  std::vector<int64_t> perm;  // internal index -> reference index (indenter sort)

  // Dense node arrays (NodeBuf split layout).
  NodeBuf grid_mp{nullptr, nullptr};  // Grid::mass / momentum (elastomer + direct indenter)
  VelBuf grid_v{nullptr, nullptr};    // Grid::velocity
  double* grid_mi = nullptr;  // indenter mass (uniform-velocity indenter scatter)
  int sms = 148;              // multiprocessor count of `device`
  // Indenter columns: maximal runs of equal initial (bx, by) in the sorted
  // cloud (internal indices [col_start[c], col_start[c+1])), z ascending.
  int n_cols = 0;
  int64_t* col_start = nullptr;
  uint8_t* ind_moves = nullptr;  // advects applied to each indenter particle this call
  size_t n_nodes = 0;
  // Elastomer lattice (counts) when the elastomer is lattice-built; enables
  // the lattice-block CTA tiling of the elastomer scatter.
  int lat[3] = {0, 0, 0};
  int tile[3] = {0, 0, 0};   // lattice block per CTA (ti, tj, tk)
  int tiles[3] = {0, 0, 0};  // blocks per axis
  bool grid_dirty = false;   // A / M_I may hold a phase-mode P2G (needs k_clear)
  void* grid_slab = nullptr;  // one allocation holding grid_mp, grid_v, grid_mi
  size_t grid_slab_bytes = 0;
  bool full_indenter = false; // scatter every indenter particle (TACCHI_FULL_INDENTER=1)
  bool grid_ready = false;   // A / M_I hold the scatter of the next substep (look-ahead
                             // of the previous mpm::step call); skip the standalone P2G
  bool keep_grid = false;    // tg_set_keep_grid: the last substep of a step runs the phase
                             // path so the grid afterwards is the reference's (engine.cpp:288-297)
  int regrows = 0;            // node-array reallocations so far
  int zpad = 2;               // allocation z-row length multiple (TACCHI_ZPAD)
  bool ab_no_walks = false;   // TACCHI_AB_NO_WALKS: timing A/B only (wrong physics)
  // The indenter's look-ahead walks: extra blocks of the elastomer kernel, or
  // (fork_walks) a kernel of their own on a forked stream, beside grid_update
  // and the elastomer kernel (TACCHI_WALKS=fork|fused)
  bool fork_walks = true;
  cudaStream_t walk_stream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int resume_substeps = 0;    // after kResume: substeps of the call still to run
  bool grid_ref = true;      // the node arrays hold the reference's Grid state (not a
                             // fused look-ahead): tg_download_grid may read them

  // Surface lattice (sim_state.hpp:41-52) + capture scratch.
  int surf_nx = 0, surf_ny = 0;
  double surf_geom[5] = {0, 0, 0, 0, 0};
  uint32_t* surf_idx = nullptr;  // internal particle indices
  double* surf_depth = nullptr;  // nx * ny
  double* cap_depth = nullptr;
  uint8_t* cap_rgb = nullptr;
  uint8_t* cap_bg = nullptr;
  size_t cap_pixels = 0, cap_bg_pixels = 0, cap_last_pixels = 0;
  double* h_depth_pinned = nullptr;
  uint8_t* h_rgb_pinned = nullptr;

  Ctl* ctl = nullptr;      // device
  Ctl* h_ctl = nullptr;    // pinned host mirror
  double* h_vind = nullptr;  // pinned staging for the command

  bool ind_v_uniform = true;   // indenter v == Ctl::ind_v for every indenter particle
  bool window_valid = false;   // ctl->win/clr describe the current positions
  int host_substep = 0;        // absolute substep counter (host view)
  bool use_graphs = true;
  std::map<int, cudaGraphExec_t> graphs;  // n_substeps -> instantiated graph
  std::map<int, int> graph_kernels;       // n_substeps -> kernels in graph
  int64_t kernel_launches = 0;
  int pending_start = 0;        // first substep of the in-flight step call
  // Indenter chain: consecutive step calls with one commanded velocity; the
  // advects of indenter particles the column walks skip stay pending (per-
  // particle counters since Ctl::chain_start) until the chain is flushed by
  // k_ind_catchup (velocity change, state access, 200 substeps).
  bool chain_open = false;
  int chain_len = 0;
  double chain_vind[3] = {0, 0, 0};

  FrameSlot frames[2];          // pipelined control steps in flight (at most two)
  cudaStream_t copy_stream = nullptr;  // their read-backs, beside the next frame's substeps
  int64_t frames_submitted = 0, frames_collected = 0;

  ~DeviceSim();
};

}  // namespace tacchi_b200
