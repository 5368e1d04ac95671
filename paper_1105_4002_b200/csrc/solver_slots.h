// Scalar slots in tvr_problem::dscal written by the passes the solvers enqueue (problem.cu).
#pragma once

namespace tvr {
constexpr int S_RSQ = 0;   // sum r^2 of the A pass
constexpr int S_TV = 1;    // 6 stencil reductions: TV, e1..e5
constexpr int S_MOM = 7;   // sum r_y^2
constexpr int S_TV2 = 9;   // 6 reductions of a second stencil pass
constexpr int S_COUNT = 16;
}  // namespace tvr
