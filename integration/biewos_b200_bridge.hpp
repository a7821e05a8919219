// biewos_b200_bridge.hpp — what a maintainer adds next to the reference's
// proj/include to run its DtN path on the B200 library (include/biewos_b200.h)
// with the reference's own headers and call sites unchanged.
//
// The reference keeps two of its public entry points' translation units out of
// the build (src/wos.cpp, src/field_eval.cpp) and links wos_b200.cpp and
// field_eval_b200.cpp instead; everything else (geometry.cpp, greens.cpp,
// quadrature.cpp, point_solver.cpp, patch_solver.cpp, ...) compiles as is.
//
// One addition to the reference's API is needed: its Scene carries Dirichlet
// data only as a std::function (geometry.hpp:34,49), which cannot run on a
// device. A caller whose data are one of the library's closed forms
// (bw_phi_kind) declares them once per Scene object; a Scene with neither
// piecewise-constant data nor a declared closed form makes every device call
// throw ApplicabilityError (there is no CPU fallback).
#pragma once

#include <cstdint>
#include <vector>

#include "biewos/geometry.hpp"
#include "biewos_b200.h"

namespace biewos::b200 {

// The closed form of scene.dirichlet: kind = bw_phi_kind, coeffs = bw_scene.phi
// (16 doubles, layout in include/biewos_b200.h). Keyed by the Scene's address:
// the reference passes its Scene by const reference through every call chain
// (solve_point -> sigma1_prime -> estimate_u_batch, sample_gamma_grid ->
// estimate_u_batch), so the object a caller declares is the one that arrives.
void set_dirichlet(const Scene& scene, int kind, const double* coeffs16);
void clear_dirichlet(const Scene& scene);

// The bw_scene image of a reference Scene (storage keeps the arrays it points
// to alive). Throws ApplicabilityError when the data have no closed form.
bw_scene to_bw(const Scene& scene, std::vector<double>& storage);

// The process-wide device context (device $BW_DEVICE, default 0). Calls through
// it are serialised by the bridge (the reference's API is synchronous).
bw_ctx* context();

// Rethrow a non-OK status as the reference's exception class (types.hpp:22-45).
void check(bw_status st);

} // namespace biewos::b200
