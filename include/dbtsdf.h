/*
 * dbtsdf.h — C ABI of the B200 scan-integration engine (libdbtsdf.so).
 *
 * This is the drop-in boundary for the DB-TSDF hot path: the functions below
 * replace the bodies of the reference's Python entry points (reference =
 * /root/reference/pkg/src/bitsdf, cited as <file>:<line>). The Python mirror
 * in paper_2509_20081_b200/ keeps the reference signatures and calls these
 * through ctypes; any other host language binds the same symbols (see
 * INTEGRATION.md). No torch / CUDA types appear in any signature: handles are
 * opaque, buffers are plain pointers plus sizes, streams are `void*`.
 *
 * Return codes mirror the reference exception -> CLI exit-code map
 * (cli.py:34-40): 0 ok, 1 generic BitsdfError, 2 ConfigurationError,
 * 3 FormatError, 4 CorruptionError, 5 EvaluationError, 6 ResourceError.
 * dbt_last_error() returns the message of the last failure on this thread.
 *
 * Threading: one host thread per grid handle (the reference is a single
 * writer per grid, integrator.py:214-216). All work is ordered on the grid's
 * CUDA stream; the *_device entry points are asynchronous on that stream.
 */
#ifndef DBTSDF_H
#define DBTSDF_H

#include <stdint.h>

#if defined(__GNUC__)
#define DBT_API __attribute__((visibility("default")))
#else
#define DBT_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define DBT_OK 0
#define DBT_ERR_GENERIC 1
#define DBT_ERR_CONFIG 2
#define DBT_ERR_FORMAT 3
#define DBT_ERR_CORRUPTION 4
#define DBT_ERR_EVALUATION 5
#define DBT_ERR_RESOURCE 6

/* point dtypes accepted by the integrate calls */
#define DBT_F32 0
#define DBT_F64 1

/* dbt_params.flags */
#define DBT_FLAG_MAP_FRAME 1u        /* points already in the map frame; per-point sensor
                                        positions supplied (integrate_point semantics) */
#define DBT_FLAG_SKIP_NORM_CHECK 2u  /* caller already applied the degenerate-ray discard
                                        (integrator.py:173-175 uses the 1-D norm) */
#define DBT_FLAG_NO_DEDUP 4u         /* stamp every applied point (no centre dedup); for
                                        measurement only, the grid result is identical */
#define DBT_FLAG_NO_SKIP 8u          /* sweep centres whose stamp is already applied too
                                        (measurement only; identical grid) */
#define DBT_FLAG_FUSE_SHADOW 16u     /* shadow update fused into preprocessing instead of
                                        a kernel concurrent with the sweep (measurement) */
#define DBT_FLAG_GENERIC_SWEEP 32u   /* distinct-row sweep even for an isotropic kernel
                                        (measurement; identical grid) */
#define DBT_FLAG_EXACT_WRITTEN 128u  /* voxels_written = the reference's serial count (stamps in
                                        ascending centre order, integrator.py:268-285) instead
                                        of the concurrent change count; one scan per launch,
                                        whole grids, ~ms per scan */
#define DBT_FLAG_STAGE_COPY 64u      /* stage pinned host scans with an H2D copy instead of
                                        reading them zero-copy in preprocessing (measurement) */

typedef struct dbt_grid dbt_grid; /* device-resident VoxelGrid (grid.py:39-58) */
typedef struct dbt_bank dbt_bank; /* device copy of a KernelBank (kernels.py:122-141) */

/* IntegrationParams (integrator.py:55-73) plus engine flags. */
typedef struct dbt_params {
  int32_t h_max;        /* 1 <= t_occ <= h_max <= 255 */
  int32_t t_occ;
  int32_t downsample;   /* keep every n-th point, >= 1 (integrator.py:223-229) */
  int32_t first_return; /* first_return_per_voxel (integrator.py:256-262) */
  uint32_t flags;
  int32_t reserved;
} dbt_params;

/* FrameStats (integrator.py:76-81) plus device counters. */
typedef struct dbt_stats {
  int64_t points_in;        /* after downsampling */
  int64_t points_discarded; /* points_in - #(degenerate or out-of-bounds) */
  int64_t voxels_written;   /* mask cells changed: concurrent count, or the reference's
                               serial count with DBT_FLAG_EXACT_WRITTEN */
  int64_t points_applied;   /* stamped returns (after first-return dedup) */
  int64_t unique_centers;   /* centre voxels swept by this launch */
  int64_t centers_skipped;  /* applied returns whose centre needed no sweep: its K^3 stamp
                               was applied by an earlier launch or claimed by another
                               return of this launch (AND idempotent) */
  int64_t bin_fallbacks;    /* returns binned outside the SVML restatement (a nonzero ray
                               component below 2^-1020 or above 2^993); 0 in practice */
  double elapsed_ms;        /* host wall clock around the call (integrator.py:217,286) */
  double device_ms;         /* CUDA-event time of the device work (H2D .. stats D2H); only measured
                               under dbt_profile_enable or with $DBT_DEVICE_MS set when the grid was
                               created (the two timing events cost ~4 us per call), else 0 */
  int64_t rows_swept;       /* kernel z-rows the sweep read (after neighbour culling);
                               launch-wide, reported on the first scan */
} dbt_stats;

DBT_API const char* dbt_last_error(void);
DBT_API const char* dbt_version(void);
DBT_API int dbt_device_count(int* out);

/* ---- voxel store (grid.py:61-89, 178-202) ------------------------------ */
/* Fresh grid: every voxel unobserved (mask 0xFFFFFFFF, sign free, hits 0).
 * slab_x0/slab_x1 select the owned x-slab [x0, x1) for multi-GPU sharding;
 * pass 0, dims[0] for a whole grid. */
DBT_API int dbt_grid_create(const int64_t dims[3], double voxel_size, const double origin[3],
                    int device, int64_t slab_x0, int64_t slab_x1, dbt_grid** out);
/* Interleaved sharding (LiDAR density falls off as 1/r^2,
 * so contiguous slabs overload the ranks near the sensor): this part owns the
 * x-planes whose block x / width is congruent to `part` mod `parts`, stored
 * in increasing x order. Host arrays of such a grid ("slab arrays" below)
 * hold its owned planes in that order. */
DBT_API int dbt_grid_create_interleaved(const int64_t dims[3], double voxel_size, const double origin[3],
                    int device, int64_t width, int32_t parts, int32_t part, dbt_grid** out);
/* owned_planes = number of x-planes stored; xmap = {x0, x1, width (0 =
 * contiguous slab), parts, part}. */
DBT_API int dbt_grid_layout(const dbt_grid* g, int64_t* owned_planes, int64_t xmap[5]);
DBT_API int dbt_grid_destroy(dbt_grid* g);
DBT_API int dbt_grid_reset(dbt_grid* g);
DBT_API int dbt_grid_info(const dbt_grid* g, int64_t dims[3], int64_t slab[2], int64_t* device_bytes);
/* Host C-order (nx,ny,nz) field arrays restricted to the slab, i.e. shape
 * (x1-x0, ny, nz). Any mask / sign / hits values are stored as is (the device
 * record is the reference's 8-byte record). */
DBT_API int dbt_grid_upload(dbt_grid* g, const uint32_t* mask, const uint8_t* sign, const uint8_t* hits);
DBT_API int dbt_grid_download(dbt_grid* g, uint32_t* mask, uint8_t* sign, uint8_t* hits);
/* Same for the global x-planes [x_begin, x_end) (owned and stored
 * contiguously: inside the slab, or inside one interleave block): arrays of
 * shape (x_end-x_begin, ny, nz). Streams huge grids in pieces. */
DBT_API int dbt_grid_download_range(dbt_grid* g, int64_t x_begin, int64_t x_end, uint32_t* mask, uint8_t* sign,
                                    uint8_t* hits);
/* DBTSDF01 voxel records, F-order linear index ix + nx*(iy + ny*iz)
 * (grid.py:178-185): 8 bytes each {mask u32, sign u8, hits u8, 0 u16}.
 * Whole grid only (slab == full grid). */
DBT_API int dbt_grid_to_records(dbt_grid* g, void* out_records);
DBT_API int dbt_grid_from_records(dbt_grid* g, const void* records);
/* The records of the z-planes [z_begin, z_end): a contiguous block of
 * (z_end-z_begin)*nx*ny records of the F-order stream (io.py:449-486 writes
 * them in this order), so DBTSDF01 snapshots stream in pieces. */
DBT_API int dbt_grid_to_records_range(dbt_grid* g, int64_t z_begin, int64_t z_end, void* out_records);
DBT_API int dbt_grid_from_records_range(dbt_grid* g, int64_t z_begin, int64_t z_end, const void* records);
/* Point query: n voxels given as global (ix,iy,iz) int64 triples inside the
 * slab (signed_distance / is_observed, grid.py:138-158); outputs nullable. */
DBT_API int dbt_grid_gather(dbt_grid* g, const int64_t* xyz, int64_t n, uint32_t* mask, uint8_t* sign,
                            uint8_t* hits);

/* ---- query / distance readout (grid.py:118-175) ------------------------ */
DBT_API int dbt_popcount(dbt_grid* g, int32_t* out);                 /* popcount_array(grid.mask) */
DBT_API int dbt_observed(dbt_grid* g, uint8_t* out);                 /* observed_array */
DBT_API int dbt_signed_distance_field(dbt_grid* g, double* field, uint8_t* observed);
DBT_API int dbt_grid_counts(dbt_grid* g, int64_t* observed, int64_t* occupied); /* cli info */

/* ---- kernel bank (kernels.py:151-193) ---------------------------------- */
/* distance_kernel: size^3 uint32 run masks indexed [dx+R][dy+R][dz+R];
 * shadow offsets: per flat bin b_a*b_el+b_e a list of (dx,dy,dz) int32
 * triples, concatenated, with shadow_counts[n_bins]. */
DBT_API int dbt_bank_create(int32_t size, int32_t b_az, int32_t b_el, const uint32_t* distance_kernel,
                    const int32_t* shadow_xyz, const int32_t* shadow_counts, int device,
                    dbt_bank** out);
DBT_API int dbt_bank_destroy(dbt_bank* b);

/* ---- integration (integrator.py:163-287) ------------------------------- */
/* One scan, sensor-frame points from HOST memory: pageable memory is staged
 * with one H2D copy, pinned (device-mapped) memory is read zero-copy by the
 * preprocessing kernel; then transform pts@R.T+t, discard, bin, stamp, stats
 * D2H; returns when the grid is updated. pose: 4x4 row-major float64. */
DBT_API int dbt_integrate_frame(dbt_grid* g, const dbt_bank* b, const void* points, int dtype,
                        int64_t n, const double pose[16], const dbt_params* p, dbt_stats* out);
/* Asynchronous dbt_integrate_frame: copies the scan to the device on a copy
 * stream and enqueues the launch sequence, then returns a ticket at once;
 * consecutive calls pipeline (the next scan's copy and the host work overlap
 * the previous scan's kernels). The points must stay valid until
 * dbt_frame_wait of that ticket returns. Stats of a ticket stay readable
 * until 4 more calls have been issued. Any parameters of dbt_integrate_frame
 * (the default path replays a CUDA graph per in-flight slot; first-return,
 * exact voxels_written and measurement flags launch directly). Any other
 * call on the grid is ordered after the queued ones. */
DBT_API int dbt_integrate_frame_async(dbt_grid* g, const dbt_bank* b, const void* points, int dtype, int64_t n,
                              const double pose[16], const dbt_params* p, int64_t* ticket);
DBT_API int dbt_frame_wait(dbt_grid* g, int64_t ticket, dbt_stats* out);
/* S scans in one launch sequence (config 5): points concatenated, counts[S],
 * poses[S*16]; out[S] per-scan stats (voxels_written reported on out[0]). */
DBT_API int dbt_integrate_batch(dbt_grid* g, const dbt_bank* b, const void* points, int dtype,
                        const int64_t* counts, int32_t n_scans, const double* poses,
                        const dbt_params* p, dbt_stats* out);
/* The same batch with one host pointer per scan (no host concatenation):
 * pinned scans are read zero-copy by preprocessing through a device table of
 * scan pointers, pageable ones are staged with one H2D copy each. */
DBT_API int dbt_integrate_scans(dbt_grid* g, const dbt_bank* b, const void* const* points, int dtype,
                        const int64_t* counts, int32_t n_scans, const double* poses,
                        const dbt_params* p, dbt_stats* out);
/* Motion-compensated scan (compensation "yaw" / "se3", integrator.py:91-123,
 * 223-230), deskewed on the device: per point the pose at its time is
 * interpolated and the point moved to the end-of-sweep sensor frame exactly
 * as the reference's scipy/numpy code does (bit for bit, including the C
 * library's sin/cos: csrc/libm_emu.cuh), then integrated like
 * dbt_integrate_frame with `pose` = the scan's (end) pose. `d` holds the
 * point-independent quantities, computed by the caller with scipy as the
 * reference does (paper_2509_20081_b200/integrator.py deskew_params).
 * timestamps: host float64, one per raw point (downsampled with the points),
 * or NULL for linspace(0, 1) over the downsampled scan. Fails with
 * DBT_ERR_CONFIG when the restatement cannot be matched to this process's C
 * library (dbt_deskew_available). */
typedef struct dbt_deskew {
  int32_t mode;           /* DBT_DESKEW_YAW or DBT_DESKEW_SE3 */
  int32_t reserved;
  double q[4];            /* yaw: tilt quaternion _rot_z(-y1) * R1; se3: start rotation (x, y, z, w) */
  double rv[3];           /* se3: the Slerp interval's rotation vector */
  double y0, dy;          /* yaw: start heading and wrapped heading change */
  double t0[3], t1[3];    /* prev_pose / pose translations */
  double r1[9];           /* pose rotation, row-major */
} dbt_deskew;
#define DBT_DESKEW_YAW 1
#define DBT_DESKEW_SE3 2
DBT_API int dbt_deskew_available(int32_t* ok);
DBT_API int dbt_integrate_frame_deskew(dbt_grid* g, const dbt_bank* b, const void* points, int dtype, int64_t n,
                               const double* timestamps, const double pose[16], const dbt_deskew* d,
                               const dbt_params* p, dbt_stats* out);
/* the deskewed float64 points alone (host in, host out; parity tests) */
DBT_API int dbt_deskew_points(int device, const void* points, int dtype, int64_t n, const double* timestamps,
                      int32_t downsample, const dbt_deskew* d, double* out);
/* Map-frame points with per-point sensor positions (integrate_point,
 * integrator.py:163-189); outcome[i] = 1 applied, 0 discarded (nullable). */
DBT_API int dbt_integrate_points_map(dbt_grid* g, const dbt_bank* b, const double* p_map,
                             const double* sensor, int64_t n, const dbt_params* p,
                             dbt_stats* out, int8_t* outcome);
/* Device-resident variant for benchmarking and multi-GPU: `d_points` is a
 * device pointer on the grid's device, `stream` a cudaStream_t with the CUDA
 * convention (NULL = legacy default stream; dbt_grid_stream gives the grid's
 * own stream). Asynchronous: the stats land in device memory and are read
 * with dbt_stats_read after the stream is synchronised. */
DBT_API int dbt_integrate_device(dbt_grid* g, const dbt_bank* b, const void* d_points, int dtype,
                         const int64_t* counts, int32_t n_scans, const double* poses,
                         const dbt_params* p, void* stream);
DBT_API int dbt_stats_read(dbt_grid* g, dbt_stats* out, int32_t n_scans);
DBT_API int dbt_grid_stream(dbt_grid* g, void** stream);
DBT_API int dbt_synchronize(dbt_grid* g);

/* ---- device binning (kernels.py:49-57), exposed for parity tests -------- */
DBT_API int dbt_bin_index_array(const double* dirs, int64_t n, int32_t b_az, int32_t b_el,
                        int64_t* b_a, int64_t* b_e, int device);

/* ---- measurement hooks -------------------------------------------------- */
/* When enabled, every engine kernel is bracketed by CUDA events on its
 * stream and its time accumulated per kernel name. */
DBT_API int dbt_profile_enable(dbt_grid* g, int on);
/* Copies up to cap entries: names (NUL-separated, 32 bytes each), total ms
 * and launch counts; returns the number of kernels in *n. */
DBT_API int dbt_profile_read(dbt_grid* g, char* names, double* ms, int64_t* launches, int32_t cap,
                     int32_t* n);
DBT_API int dbt_profile_reset(dbt_grid* g);
/* Kernel launches issued by the engine since load (all handles). */
DBT_API int64_t dbt_launch_count(void);
/* Roofline probes: on an L2-resident buffer of `bytes`,
 * out[0] RED.AND Gop/s on 4-byte words, out[1] the same in GB/s, out[2]
 * 8-byte ld.cg GB/s. Best of 4 timed runs after a warm-up. */
DBT_API int dbt_probe_l2(int device, int64_t bytes, double* out);

/* ---- marching cubes on the device (mesher.py:43-110) ---- */
/* The lookup tables are an input: the caller copies them from the
 * reference's bitsdf/_mc_tables.py (EDGE_TABLE :9, TRI_TABLE :44,
 * CORNER_OFFSETS :312, EDGE_BASE :319, EDGE_AXIS :324), row-major int32. */
typedef struct dbt_mc_tables {
  int32_t edge_table[256];
  int32_t tri_table[256 * 16];
  int32_t corner_offsets[8 * 3];
  int32_t edge_base[12 * 3];
  int32_t edge_axis[12];
} dbt_mc_tables;
typedef struct dbt_mesh dbt_mesh;
/* extract_mesh(grid, iso) (mesher.py:43): vertices and triangles identical to
 * the reference's (same order, float64 vertices bit for bit), kept in device
 * memory until dbt_mesh_destroy. Whole (unsharded) grids only. An empty mesh
 * is a valid handle with zero counts. */
DBT_API int dbt_mesh_extract(dbt_grid* g, double iso, const dbt_mc_tables* tables, dbt_mesh** out,
                     int64_t* n_vertices, int64_t* n_triangles);
DBT_API int dbt_mesh_info(const dbt_mesh* m, int64_t* n_vertices, int64_t* n_triangles);
/* vertices: n_vertices*3 float64; triangles: n_triangles*3 int64 (either may be NULL) */
DBT_API int dbt_mesh_download(const dbt_mesh* m, double* vertices, int64_t* triangles);
/* device pointers of the same arrays (valid until dbt_mesh_destroy) */
DBT_API int dbt_mesh_device_buffers(const dbt_mesh* m, const double** vertices, const int64_t** triangles);
/* a mesh from host arrays (any TriangleMesh), e.g. for dbt_mesh_normals */
DBT_API int dbt_mesh_from_host(int device, const double* vertices, int64_t n_vertices, const int64_t* triangles,
                       int64_t n_triangles, dbt_mesh** out);
/* vertex_normals (mesher.py:113-127): area-weighted unit normals, bit-exact
 * with the reference (corner sums in np.add.at order); zero for vertices
 * without a non-degenerate incident triangle. Negative indices wrap like
 * numpy; other out-of-range indices fail with DBT_ERR_CONFIG. */
DBT_API int dbt_mesh_normals(dbt_mesh* m);
DBT_API int dbt_mesh_download_normals(const dbt_mesh* m, double* normals);
DBT_API int dbt_mesh_destroy(dbt_mesh* m);

/* ---- data-parallel replicas (multi-GPU) ------------------ */
/* Each rank integrates its own scans into a whole-grid replica; a merge makes
 * every replica equal to the grid all those scans produce together:
 *   mark  : snapshot the base (after create/reset/upload and after a merge)
 *   pack  : n = nx*ny*nz C-order device buffers: mask_len (u8, bit length of
 *           the mask), sign (u8), delta_f16 (IEEE half, hits - base hits)
 *   (caller: all-reduce MIN mask_len, MIN sign, SUM delta_f16 over replicas)
 *   apply : combine the reduced buffers into the records (h_max, t_occ = the
 *           parameters the replicas integrated with) and re-mark.
 * 4 bytes per voxel; pack/apply are asynchronous on `stream` (NULL: the
 * grid's stream). */
DBT_API int dbt_replica_mark(dbt_grid* g);
DBT_API int dbt_replica_pack(dbt_grid* g, uint8_t* mask_len, uint8_t* sign, uint16_t* delta_f16, void* stream);
DBT_API int dbt_replica_apply(dbt_grid* g, const uint8_t* mask_len_min, const uint8_t* sign_min,
                      const uint16_t* delta_sum_f16, int32_t h_max, int32_t t_occ, void* stream);
/* Sparse merge: only the 16^3 bricks within a kernel radius of a return some
 * rank applied since the last mark/merge travel (prep_kernel flags the brick
 * of every applied centre).
 *   bricks      : number of brick flags (nbx*nby*nbz, 16^3 bricks) and this
 *                 rank's reach (largest kernel radius R integrated since the
 *                 last merge)
 *   dirty       : copy this rank's flags (u8 per brick) into `flags` (device)
 *   (caller: all-reduce MAX of the flags and of the reach over replicas)
 *   select      : dilate the reduced flags by ceil(reach/16) bricks and list
 *                 the selected bricks in brick order (synchronous; *n_sel)
 *   pack_bricks : mask_len_sign = [n_sel*4096 mask bit lengths | n_sel*4096
 *                 signs] (u8), delta_f16 = n_sel*4096 hit deltas
 *   (caller: all-reduce MIN mask_len_sign, SUM delta_f16)
 *   apply_bricks: combine into the selected bricks, re-mark, clear the flags.
 * Bricks nobody touched are equal on every replica already. */
DBT_API int dbt_replica_bricks(dbt_grid* g, int64_t* n_bricks, int32_t* reach);
DBT_API int dbt_replica_dirty(dbt_grid* g, uint8_t* flags, void* stream);
DBT_API int dbt_replica_select(dbt_grid* g, const uint8_t* flags, int32_t reach, int64_t* n_sel, void* stream);
DBT_API int dbt_replica_pack_bricks(dbt_grid* g, uint8_t* mask_len_sign, uint16_t* delta_f16, void* stream);
DBT_API int dbt_replica_apply_bricks(dbt_grid* g, const uint8_t* mask_len_sign_min, const uint16_t* delta_sum_f16,
                             int32_t h_max, int32_t t_occ, void* stream);

/* pinned host buffers for callers without a CUDA runtime of their own */
DBT_API int dbt_host_alloc(int64_t bytes, void** out);
DBT_API int dbt_host_free(void* p);

#ifdef __cplusplus
}
#endif
#endif /* DBTSDF_H */
