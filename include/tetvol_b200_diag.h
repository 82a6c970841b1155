/* tetvol_b200 diagnostics (not part of the reference drop-in surface).
 *
 * tv_diag_gather_ceiling measures the memory-latency ceiling of the trace
 * kernel on a given frame. It records the exit slot of every tet step of every
 * path of the frame through the same integrator as tv_render (path order, RNG
 * streams and batch layout identical), then replays the paths as a pure chain
 * of dependent 64-byte LeafRec loads (each step's record names the next leaf,
 * as in the render) with the trace kernel's launch shape (threads per block,
 * blocks per SM, L1 split) and its path-regeneration scheme, but no geometry
 * work. The replay's tet steps per second is the rate a kernel with free
 * exit-face computation would reach on this access stream at this occupancy:
 * the latency roofline the trace kernel is measured against (bench.py,
 * DESIGN.md 4).
 *
 * out[0] replay tet steps / s (dependent chain, trace-kernel occupancy)
 * out[1] replay tet steps / s (dependent chain, every warp slot of the SM filled)
 * out[2] tet steps recorded (equals the frame's cells_visited)
 * out[3] replay ms (out[0])
 * out[4] bytes of recorded path code read per step (0.5: a 4-bit exit slot)
 * out[5] resident warps per SM of the out[0] replay
 * Requires half a byte of device memory per tet step of the frame (3.3 GB for
 * the C2 frame) plus ~70 bytes per path. Synchronous.
 */
#ifndef TETVOL_B200_DIAG_H
#define TETVOL_B200_DIAG_H

#include "tetvol_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

int tv_diag_gather_ceiling(const tv_grid* g, const tv_camera* camera, const tv_render_config* cfg, int reps,
                           double out[6]);

#ifdef __cplusplus
}
#endif

#endif
