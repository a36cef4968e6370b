/*
 * tvegpu.h — C ABI of the B200-native TLED thermo-visco-elastodynamic step.
 *
 * This is the drop-in boundary for the reference's `tve::Engine`
 * (/root/reference/proj/include/tve/engine.hpp:83-143).  The reference is a C++20
 * API (headers only, no bodies); this header is what a C++ host (or any FFI)
 * binds instead.  Plain pointers and sizes only: no exceptions, no Eigen, no STL,
 * no torch types cross it.  A header-only C++ facade with the reference's
 * class shape lives in include/tve_gpu.hpp.
 *
 * Conventions
 *   - All indices are 0-based ORIGINAL ids (the caller's numbering).  Internal
 *     Morton/first-touch permutations and partitions never leak out.
 *   - Every input buffer is caller-owned and copied inside tvegpu_create
 *     (the reference keeps references to mesh/pre/material, engine.hpp:122-124;
 *     copying is strictly safer and observably equivalent).
 *   - Errors map to the reference exception taxonomy (errors.hpp:8-33) by
 *     status code; tvegpu_last_error() returns the message and, for
 *     InstabilityError, the (step, node) payload (errors.hpp:21-27).
 *   - One handle is not thread-safe; distinct handles are independent.
 *   - tvegpu_step() is synchronous: it returns after the device finite check.
 */
#ifndef TVEGPU_H
#define TVEGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TVEGPU_ABI_VERSION 1

/* errors.hpp:8-33 — ParseError, ValidationError, InstabilityError, IoError,
 * plus device-side failures the reference (CPU-only) never had. */
typedef enum tvegpu_status {
    TVEGPU_OK = 0,
    TVEGPU_E_PARSE = 1,        /* tve::ParseError        (errors.hpp:9)  */
    TVEGPU_E_VALIDATION = 2,   /* tve::ValidationError   (errors.hpp:15) */
    TVEGPU_E_INSTABILITY = 3,  /* tve::InstabilityError  (errors.hpp:21) */
    TVEGPU_E_IO = 4,           /* tve::IoError           (errors.hpp:30) */
    TVEGPU_E_CUDA = 5,         /* CUDA runtime failure / no device       */
    TVEGPU_E_NCCL = 6,         /* NCCL failure (multi-GPU halo)           */
    TVEGPU_E_ARG = 7           /* NULL handle / bad size / bad option     */
} tvegpu_status;

/* mesh.hpp:15 ElementKind */
enum { TVEGPU_T4 = 0, TVEGPU_H8 = 1 };
/* engine.hpp:16 CouplingMode */
enum { TVEGPU_COUPLED = 0, TVEGPU_THERMAL_ONLY = 1, TVEGPU_MECHANICAL_ONLY = 2 };
/* materials.hpp:77 ExpansionKind */
enum { TVEGPU_EXP_ISOTROPIC = 0, TVEGPU_EXP_TRANSVERSELY_ISOTROPIC = 1, TVEGPU_EXP_ORTHOTROPIC = 2 };

/* mechanics.hpp:25-35 PrescribedDisplacement */
typedef struct tvegpu_prescribed {
    int32_t num_nodes;
    const int32_t* nodes;
    int32_t component;   /* 0,1,2 */
    double target;       /* [m] */
    double ramp_time;    /* [s]; <= 0 means step load (value_at, mechanics.hpp:31-34) */
} tvegpu_prescribed;

/* bioheat.hpp:19-26 SourceRegion */
typedef struct tvegpu_source {
    int32_t num_elements;
    const int32_t* elements;
    double q_r;          /* [W/m^3] */
    double t_start;      /* [s] */
    double t_end;        /* [s]; +inf allowed */
} tvegpu_source;

/*
 * Flat mirror of everything tve::Engine's constructor receives
 * (engine.hpp:85-87): Mesh (mesh.hpp:22-37), the precompute inputs
 * (density, ref_specific_heat; mesh.hpp:83), MaterialModel
 * (materials.hpp:89-97), MechBCs (mechanics.hpp:37-47, without the host
 * std::function motion_override), ThermalBCs (bioheat.hpp:32-35),
 * HeatSourceSet (bioheat.hpp:28-30) and SimulationConfig (engine.hpp:28-39,
 * without the OutputSpec, which is run-level).  motion_override is set after
 * creation with tvegpu_set_motion_override.
 */
typedef struct tvegpu_problem {
    /* ---- Mesh (mesh.hpp:22-37) ---- */
    int32_t kind;                   /* TVEGPU_T4 | TVEGPU_H8 */
    int32_t num_nodes;
    int32_t num_elements;
    const double* nodes;            /* 3*num_nodes, xyz interleaved [m] */
    const int32_t* elements;        /* nn*num_elements, element-major, 0-based */
    const double* fiber_dirs;       /* 3*num_elements or NULL (mesh.hpp:28) */
    const double* expansion_axes;   /* 6*num_elements (m then n) or NULL (mesh.hpp:29) */

    /* ---- precompute(mesh, density, ref_specific_heat) (mesh.hpp:83) ---- */
    double ref_specific_heat;       /* [J/(kg degC)] */

    /* ---- HyperelasticParams (materials.hpp:15-19) ---- */
    double mu, kappa, eta_a;
    /* ---- PronySeries::from_terms (materials.hpp:27-36) ---- */
    int32_t prony_count;            /* any number of terms (PronySeries, materials.hpp:27-35) */
    const double* prony_phi;        /* prony_count */
    const double* prony_tau;        /* prony_count */
    /* ---- ThermalProps (materials.hpp:67-75) ---- */
    double density;
    int32_t c_table_len;            /* ScalarTable specific_heat (materials.hpp:39-49), >= 1 entries, any length */
    const double* c_table_T;
    const double* c_table_value;
    int32_t k_table_len;            /* ConductivityTable (materials.hpp:53-65), >= 1 entries, any length */
    const double* k_table_T;
    const double* k_table_tensor;   /* 9 per entry, row-major (symmetric) */
    double perfusion_rate;          /* w_b */
    double blood_specific_heat;     /* c_b */
    double arterial_temperature;    /* T_a */
    double metabolic_rate;          /* Q_m */
    /* ---- optional<ExpansionSpec> (materials.hpp:80-86, 93) ---- */
    int32_t has_expansion;
    int32_t expansion_kind;
    double alpha_i, alpha_m, alpha_n, reference_temperature;
    /* ---- optional<Vector3d> fiber, axis_m, axis_n (materials.hpp:94-96) ---- */
    int32_t has_fiber;
    double fiber[3];
    double axis_m[3];
    double axis_n[3];

    /* ---- MechBCs (mechanics.hpp:37-47) ---- */
    int32_t num_fixed_nodes;
    const int32_t* fixed_nodes;
    int32_t num_prescribed;
    const tvegpu_prescribed* prescribed;
    const double* external_force;   /* 3*num_nodes or NULL */
    double body_force[3];           /* [N/m^3] */

    /* ---- ThermalBCs (bioheat.hpp:32-35) ---- */
    int32_t num_fixed_temperatures;
    const int32_t* fixed_temperature_nodes;
    const double* fixed_temperature_values;
    double initial_temperature;

    /* ---- HeatSourceSet (bioheat.hpp:28-30) ---- */
    int32_t num_sources;
    const tvegpu_source* sources;

    /* ---- SimulationConfig (engine.hpp:28-39) ---- */
    double dt;
    double duration;
    int32_t mode;                   /* TVEGPU_COUPLED | _THERMAL_ONLY | _MECHANICAL_ONLY */
    int32_t expansion_enabled;
    int32_t temperature_dependent;
    double damping_gamma;
    double hourglass_stiffness;
    int32_t allow_unstable_dt;
    int32_t workers;                /* ignored on the GPU; kept for layout parity */
} tvegpu_problem;

/* Device / decomposition options (no reference counterpart). */
typedef struct tvegpu_options {
    int32_t device;                 /* CUDA ordinal; -1 = current */
    int32_t nranks;                 /* 1 = single GPU; >1 = this handle is one RCB partition */
    int32_t rank;
    const void* nccl_unique_id;     /* 128 bytes from tvegpu_nccl_unique_id() when nranks > 1 */
    int32_t reorder;                /* 1 (default) = Morton elements + first-touch nodes; 0 = identity */
    int32_t diagnostics;            /* 1 = keep F, S_tilde, assembled forces (engine.hpp:101-105) */
    int32_t steps_per_graph;        /* CUDA-graph chunk length; 0 = default (64) */
    int32_t halo_transport;         /* partitioned engines and groups: TVEGPU_HALO_* (default PEER) */
    int32_t slot_fp32;              /* 0 (default): fp64 everywhere (the parity path, <= 1e-10 vs the
                                       reference algorithm).  1: mixed precision — element and node math
                                       in fp64, the per-element contributions between them stored as
                                       fp32 and summed in fp64 (about a quarter fewer bytes per step;
                                       deviation bound in DESIGN.md §2) */
} tvegpu_options;

/* Halo exchange of partitioned steps (interface-node heat fluxes and forces).
 *   TVEGPU_HALO_PEER  the boundary elements' kernel stores every interface contribution
 *                     straight into the neighbouring partitions' receive areas (NVLink peer
 *                     memory of the other GPUs; in a group, the other partitions' buffers) and
 *                     raises a per-phase flag there; the neighbours' node kernels wait for it
 *                     on the device.  No pack kernel and no NCCL call on the step path.
 *                     Across processes it needs tvegpu_peer_export / tvegpu_peer_attach once
 *                     after tvegpu_create (until then the NCCL transport is used).
 *   TVEGPU_HALO_NCCL  pack kernel + grouped ncclSend/ncclRecv on a comm stream (a group:
 *                     device copies of the packed segments instead).
 * Both deliver the same values to the same receive slots: results are bit-identical. */
enum { TVEGPU_HALO_PEER = 0, TVEGPU_HALO_NCCL = 1 };

typedef struct tvegpu_engine tvegpu_engine;

/* Fill *opt with defaults (single GPU, reorder on, no diagnostics). */
void tvegpu_default_options(tvegpu_options* opt);

/* Engine(mesh, pre, material, mech_bcs, thermal_bcs, sources, config)
 * (engine.hpp:85-87) fused with precompute() (mesh.hpp:83): validates inputs
 * (ValidationError as the reference: degenerate elements mesh.hpp:81-82,
 * Prony weights materials.hpp:33-35, axes materials.hpp:112, dt above critical
 * engine.hpp:36), builds the device layout and uploads it. */
tvegpu_status tvegpu_create(const tvegpu_problem* problem, const tvegpu_options* options,
                            tvegpu_engine** out);
void tvegpu_destroy(tvegpu_engine* h);

/* nsteps x Engine::step() (engine.hpp:89-90).  Returns TVEGPU_E_INSTABILITY
 * at the first step that produced a non-finite T or u; the state is then the
 * state the reference leaves behind when step() throws (that step applied,
 * time and step counter not advanced). */
tvegpu_status tvegpu_step(tvegpu_engine* h, int64_t nsteps);

/* Readback of SimulationState (engine.hpp:41-45, 95-97) in original numbering. */
tvegpu_status tvegpu_get_temperatures(tvegpu_engine* h, double* T /* num_nodes */);
tvegpu_status tvegpu_get_displacements(tvegpu_engine* h, double* disp /* 3N */,
                                       double* disp_prev /* 3N or NULL */);
/* Engine::make_snapshot() (engine.hpp:47-55, 99): T and u of the current state in
 * one device read (either pointer may be NULL). */
tvegpu_status tvegpu_make_snapshot(tvegpu_engine* h, double* T /* N */, double* disp /* 3N */);
/* Viscous history, MechState::viscous (mechanics.hpp:20): (e*P + p)*9, row-major. */
tvegpu_status tvegpu_get_viscous(tvegpu_engine* h, double* viscous);
double  tvegpu_time(const tvegpu_engine* h);
int64_t tvegpu_step_count(const tvegpu_engine* h);

/* Write access to state() between steps (engine.hpp:95): any pointer may be
 * NULL to leave that field unchanged. */
tvegpu_status tvegpu_set_state(tvegpu_engine* h, const double* T, const double* disp,
                               const double* disp_prev, const double* viscous,
                               double time, int64_t step);

/* Override the lumped nodal source vector (bioheat.hpp:57 nodal_source_power,
 * engine.hpp:138) with caller-supplied powers [W] per node (original ids);
 * NULL restores the regional HeatSourceSet schedule. */
tvegpu_status tvegpu_set_nodal_sources(tvegpu_engine* h, const double* power);

/* MechBCs::motion_override (mechanics.hpp:43-46): an optional per-node displacement
 * trajectory.  fn(user, node, t, disp) returns nonzero and fills disp[3] to pin the
 * (original) node to disp at time t; it is applied last, after fixed and prescribed
 * components (mechanics.hpp:89, SPEC.md C9), at t = time + dt of each step.  A host
 * callback cannot run inside a device step, so this is a slow path: while set, every
 * step evaluates fn on the host for the candidate nodes (nodes[num_nodes], original
 * ids; NULL = every node), uploads the pins and launches the step without graph
 * replay.  fn = NULL removes the override. */
typedef int32_t (*tvegpu_motion_fn)(void* user, int32_t node, double t, double* disp);
tvegpu_status tvegpu_set_motion_override(tvegpu_engine* h, tvegpu_motion_fn fn, void* user, int32_t num_nodes,
                                         const int32_t* nodes);

/* One closed-loop iteration with host buffers: the effect of
 *   tvegpu_set_nodal_sources(h, power) (skipped when power is NULL);
 *   tvegpu_step(h, n);  tvegpu_make_snapshot(h, T, disp)  (skipped when both are NULL)
 * with the copies overlapped with the step on a second stream: the source upload
 * runs while the thermal element kernel computes (only the thermal node update
 * reads the sources) and the temperature read-back while the mechanical half of
 * the last step computes.  n >= 1.  On an error return T and disp are undefined. */
tvegpu_status tvegpu_step_io(tvegpu_engine* h, const double* power, int64_t n, double* T, double* disp);

/* ---- checkpoint / restart (engine.hpp:110-111) ----
 * A versioned binary image of the state in original numbering (layout in
 * DESIGN.md): T, u, u_prev, viscous history, time, step and an active nodal-source
 * override.  Restores bit-exactly, into an engine with any partitioning.  Saving
 * from a partitioned engine (nranks > 1) is collective: every rank calls it, the
 * ranks' nodes and elements are gathered over NCCL and every rank receives the same
 * image.  Errors: E_ARG (buffer too small), E_IO (bad magic / version / problem
 * mismatch / truncated). */
tvegpu_status tvegpu_checkpoint_size(tvegpu_engine* h, uint64_t* bytes);
tvegpu_status tvegpu_save_checkpoint(tvegpu_engine* h, void* buf, uint64_t bytes);
tvegpu_status tvegpu_load_checkpoint(tvegpu_engine* h, const void* buf, uint64_t bytes);

/* ---- run-level outputs on the device ----
 * RunSummary node extrema (engine.hpp:57-66) by deterministic device reductions
 * (a 56-byte read-back instead of the full fields); multi-GPU: all-reduced. */
typedef struct tvegpu_summary {
    int64_t steps;
    double time;
    double max_temperature; /* over nodes, current state */
    double min_disp[3];     /* per component */
    double max_disp[3];
} tvegpu_summary;
tvegpu_status tvegpu_get_summary(tvegpu_engine* h, tvegpu_summary* out);

/* ablation_volume: exact volume [m^3] of {T >= threshold} for the
 * piecewise-linear temperature by analytic clipping of each tetrahedron (an H8 is
 * split into 6 around its 0-6 diagonal), measured at X + u when deformed != 0
 * (SPEC.md:460).  elements_above (may be NULL): elements with a non-zero clipped
 * volume.  Multi-GPU: summed over ranks. */
tvegpu_status tvegpu_ablation_volume(tvegpu_engine* h, double threshold, int32_t deformed, double* volume,
                                     int64_t* elements_above);

/* total_energy (engine.hpp:108), split: kinetic sum 1/2 m |(u - u_prev)/dt|^2 and strain
 * energy sum V det(F_th) Psi(C_el) of the current state (device reductions; either
 * pointer may be NULL).  Multi-GPU: replicated nodes are counted by every rank that holds them. */
tvegpu_status tvegpu_total_energy(tvegpu_engine* h, double* kinetic, double* strain);

/* Snapshot element fields (engine.hpp:47-55, OutputSpec write_det_f / write_stress):
 * det F and the largest principal value of S_tilde (PK2) per element, original
 * order, from the last mechanics phase.  Requires options.diagnostics = 1 and a
 * single-partition engine.  Either pointer may be NULL. */
tvegpu_status tvegpu_element_fields(tvegpu_engine* h, double* det_f, double* max_principal_stress);

/* Diagnostics of the last mechanics phase (engine.hpp:101-105); requires
 * options.diagnostics = 1.  f_int: assembled internal force 3N; F, S: 9 per
 * element (row-major) deformation gradients and S_tilde.  Any may be NULL. */
tvegpu_status tvegpu_get_diagnostics(tvegpu_engine* h, double* f_int, double* F, double* S);

/* Message of the last failure; for TVEGPU_E_INSTABILITY also the step index and
 * the lowest original node id holding a non-finite value (errors.hpp:21-27). */
tvegpu_status tvegpu_last_error(const tvegpu_engine* h, char* msg, size_t cap,
                                int64_t* step, int32_t* node);
const char* tvegpu_status_string(tvegpu_status s);

/* Host-only helpers (no device needed). */
/* critical_timestep(mesh, material) (mesh.hpp:92-97). */
tvegpu_status tvegpu_critical_timestep(const tvegpu_problem* problem, double* thermal,
                                       double* mechanical);
/* load_mesh (mesh.hpp:73-79): parse + validate the text mesh format of SPEC.md:88
 * (sections $nodes, $elements K t4|h8, $nodeset, $elemset, $fibers, $expansion_axes;
 * 1-based ids in the file, 0-based in the view), bulk lines parsed in parallel.
 * Errors: E_PARSE with "line L: ..." / E_VALIDATION (mixed kinds, out-of-range index
 * or inverted element naming the element, non-unit direction) via tvegpu_create_error.
 * The view's arrays plug straight into tvegpu_problem (nodes, elements, fiber_dirs,
 * expansion_axes) and stay valid until tvegpu_mesh_destroy. */
typedef struct tvegpu_mesh tvegpu_mesh;
typedef struct tvegpu_mesh_view {
    int32_t kind;                   /* TVEGPU_T4 / TVEGPU_H8 */
    int32_t num_nodes, num_elements;
    const double* nodes;            /* 3 * num_nodes */
    const int32_t* elements;        /* nn * num_elements, 0-based */
    const double* fiber_dirs;       /* 3 * num_elements or NULL */
    const double* expansion_axes;   /* 6 * num_elements (m, n) or NULL */
    int32_t num_node_sets;
    const char* const* node_set_names;
    const int32_t* node_set_offsets;  /* num_node_sets + 1 */
    const int32_t* node_set_items;    /* 0-based node ids */
    int32_t num_element_sets;
    const char* const* element_set_names;
    const int32_t* element_set_offsets;
    const int32_t* element_set_items;
} tvegpu_mesh_view;
tvegpu_status tvegpu_load_mesh(const char* text, uint64_t length, tvegpu_mesh** out, tvegpu_mesh_view* view);
void tvegpu_mesh_get_view(const tvegpu_mesh* mesh, tvegpu_mesh_view* view);
void tvegpu_mesh_destroy(tvegpu_mesh* mesh);

/* Library-owned error text for failures before a handle exists. */
const char* tvegpu_create_error(void);
int32_t tvegpu_abi_version(void);

/* ---------------------------------------------------------------------------
 * Decomposition plan (host-only; exposes the integer maps for bit-exact tests).
 * For nranks == 1 this is the single-GPU layout: Morton element order,
 * first-touch node order and the node -> slot CSR in canonical
 * (ascending original element id, then local index) order (mesh.hpp:58-61).
 * For nranks > 1, elements are split by recursive coordinate bisection and
 * each rank's CSR addresses local slots [0, nn*E_local) followed by the
 * receive area of its halo exchange.
 * ------------------------------------------------------------------------- */
typedef struct tvegpu_plan tvegpu_plan;

typedef struct tvegpu_plan_view {
    int32_t nranks, rank, nn;
    int32_t num_elements;           /* local (owned) elements */
    int32_t num_boundary_elements;  /* the first ones in local order touch a shared node */
    int32_t num_nodes;              /* local nodes (owned + replicated) */
    const int32_t* element_orig;    /* num_elements: local -> original element id */
    const int32_t* node_orig;       /* num_nodes: local -> original node id */
    const int32_t* conn;            /* nn*num_elements, element-major, local node ids */
    const int32_t* csr_offsets;     /* num_nodes + 1 */
    const int32_t* csr_slots;       /* slot ids: e*nn + a (local) or nn*E + k (receive slot k) */
    int32_t num_neighbors;
    const int32_t* neighbor_ranks;  /* ascending */
    const int32_t* send_offsets;    /* num_neighbors + 1, into send_slots */
    const int32_t* send_slots;      /* local slot ids sent to each neighbour, canonical order */
    const int32_t* recv_offsets;    /* num_neighbors + 1; receive slot k of neighbour j at recv_offsets[j] + k */
    const int32_t* element_owner;   /* GLOBAL: num_elements_global owner ranks (original ids) */
    int32_t num_elements_global;
    /* element-kernel chunks (one CTA each): nodes staged in shared memory */
    int32_t num_chunks;
    const int32_t* chunk_start;     /* num_chunks + 1 */
    const int32_t* chunk_node_off;  /* num_chunks + 1 */
    const int32_t* chunk_nodes;     /* unique local node ids of each chunk, ascending */
    const uint16_t* chunk_node_slot;/* shared-memory slot of each chunk_nodes entry */
    const uint16_t* chunk_conn;     /* nn*num_elements: slot of node (e, a) in its chunk */
    int32_t max_chunk_slots;
} tvegpu_plan_view;

tvegpu_status tvegpu_plan_create(const tvegpu_problem* problem, int32_t nranks, int32_t rank,
                                 int32_t reorder, tvegpu_plan** out);
tvegpu_status tvegpu_plan_get(const tvegpu_plan* plan, tvegpu_plan_view* view);
void tvegpu_plan_destroy(tvegpu_plan* plan);

/* ncclGetUniqueId for the multi-GPU halo communicator (128 bytes). */
tvegpu_status tvegpu_nccl_unique_id(void* out128);

/* Peer-memory halo across processes (one partition per process and GPU, one node).
 * Every rank exports a descriptor (CUDA IPC handles of its receive areas and flag inbox,
 * its neighbour list; blob == NULL queries the size into *len), the ranks all-gather the
 * descriptors (any host channel, e.g. torch.distributed), and every rank attaches with
 * the nranks descriptors indexed by rank.  Only neighbours' buffers are mapped.  After
 * the attach, tvegpu_step runs the TVEGPU_HALO_PEER path (options.halo_transport). */
tvegpu_status tvegpu_peer_export(tvegpu_engine* h, void* blob, size_t cap, size_t* len);
tvegpu_status tvegpu_peer_attach(tvegpu_engine* h, const void* const* blobs, const size_t* lens, int32_t nranks);
/* 1 if the engine steps with the peer-memory halo (attached, or a group part), else 0. */
int32_t tvegpu_halo_peer(const tvegpu_engine* h);
/* Back to the NCCL halo (unmaps the neighbours).  Collective in effect: every rank must
 * step with the same transport, so callers agree first (e.g. all-reduce the attach status
 * and detach everywhere if any rank failed to attach). */
tvegpu_status tvegpu_peer_detach(tvegpu_engine* h);

/* ---------------------------------------------------------------------------
 * Partition group: nparts RCB partitions of one problem stepped together on ONE
 * device by the multi-GPU step code (boundary-first elements, halo delivery,
 * interior elements, receive-area gathers, CUDA-graph replay, agreement on the first
 * failure, device state gather for checkpoints).  options.halo_transport selects the
 * halo path exactly as for one partition per GPU: TVEGPU_HALO_PEER (default) runs the
 * peer-memory kernels (the parts' buffers stand in for the other GPUs' memory; node
 * kernels are also ordered after their neighbours' send kernels by events), and
 * TVEGPU_HALO_NCCL the pack + exchange path with device copies of each neighbour's
 * packed segment instead of ncclSend/ncclRecv.  Results are bit-identical to a single
 * partition either way.
 * The calls mirror the engine's (tvegpu_step, tvegpu_set_state, ...).  After a
 * failure every partition reports the same (step, node); the state is then invalid
 * (the other partitions ran on) until set_state / load_checkpoint — the same rule as
 * for NCCL ranks (nranks > 1 engines).
 * ------------------------------------------------------------------------- */
typedef struct tvegpu_group tvegpu_group;
tvegpu_status tvegpu_group_create(const tvegpu_problem* problem, int32_t nparts, const tvegpu_options* options,
                                  tvegpu_group** out);
tvegpu_status tvegpu_group_step(tvegpu_group* g, int64_t nsteps);
tvegpu_status tvegpu_group_get_fields(tvegpu_group* g, double* T, double* disp, double* viscous);
tvegpu_status tvegpu_group_get_state(tvegpu_group* g, double* T, double* disp, double* disp_prev, double* viscous);
tvegpu_status tvegpu_group_set_state(tvegpu_group* g, const double* T, const double* disp, const double* disp_prev,
                                     const double* viscous, double time, int64_t step);
tvegpu_status tvegpu_group_set_nodal_sources(tvegpu_group* g, const double* power);
tvegpu_status tvegpu_group_step_io(tvegpu_group* g, const double* power, int64_t n, double* T, double* disp);
double tvegpu_group_time(const tvegpu_group* g);
int64_t tvegpu_group_step_count(const tvegpu_group* g);
tvegpu_status tvegpu_group_last_error(const tvegpu_group* g, char* msg, size_t cap, int64_t* step, int32_t* node);
tvegpu_status tvegpu_group_checkpoint_size(tvegpu_group* g, uint64_t* bytes);
tvegpu_status tvegpu_group_save_checkpoint(tvegpu_group* g, void* buf, uint64_t bytes);
tvegpu_status tvegpu_group_load_checkpoint(tvegpu_group* g, const void* buf, uint64_t bytes);
void tvegpu_group_destroy(tvegpu_group* g);

/* ---------------------------------------------------------------------------
 * Measurement hooks (no reference counterpart; used by bench.py).
 * ------------------------------------------------------------------------- */
/* cudaStream_t (as void*) every step kernel is launched on. */
void* tvegpu_stream(tvegpu_engine* h);
/* Halo exchange volume of one partition (nranks > 1): neighbours, and bytes sent /
 * received per step (every contribution of a shared node, both coupled phases). */
tvegpu_status tvegpu_halo_info(const tvegpu_engine* h, int32_t* neighbors, int64_t* send_bytes, int64_t* recv_bytes);
/* One partition of a P-GPU run stepped ALONE on this device, to time a rank's work
 * without the other GPUs: create it with nranks = P, rank = r, nccl_unique_id = NULL and
 * halo_transport = TVEGPU_HALO_PEER, then call this.  Its halo stores go to a scratch
 * buffer and its waits pass at once, so its numbers are meaningless; its step time is
 * the rank's step minus the NVLink transfer (scripts/partition_solo.py). */
tvegpu_status tvegpu_peer_attach_solo(tvegpu_engine* h);
/* Kernel launches per step (per coupled phase: element + node kernel; partitioned:
 * boundary + interior element launches, plus the halo pack with the NCCL transport). */
int32_t tvegpu_kernels_per_step(const tvegpu_engine* h);
/* H8: chunks of this partition whose elements are all affine (parallelepipeds: hourglass
 * geometry c_al = 0); K3 skips their c_al rows and terms.  0 for T4. */
int32_t tvegpu_affine_chunks(const tvegpu_engine* h);
/* Enqueue nsteps on the stream without waiting or reading back the finite
 * check; tvegpu_sync() waits and applies it.  tvegpu_step == enqueue + sync. */
tvegpu_status tvegpu_enqueue_steps(tvegpu_engine* h, int64_t nsteps);
tvegpu_status tvegpu_sync(tvegpu_engine* h);
/* Time each kernel of the step with CUDA events over nsteps direct (un-graphed)
 * steps; ms_per_kernel[k] = mean duration of kernel k per step (up to 8 kinds),
 * names = ';'-separated kernel names.  Returns the number of kinds in *count.
 * Partitioned engines: the element entries span their phase (boundary elements, pack,
 * exchange enqueue, interior elements), the node entries include the wait for the
 * halo, and two more entries time the halo transfers on the comm stream. */
tvegpu_status tvegpu_profile_kernels(tvegpu_engine* h, int32_t nsteps, double* ms_per_kernel, int32_t* count,
                                     char* names, size_t cap);

#ifdef __cplusplus
}
#endif
#endif /* TVEGPU_H */
