// The analytic indenter solids (geo/shapes.cpp:79-206) as plain data shared
// by the host restatement (host_setup.cpp) and the device rejection sampler
// (setup_kernels.cu). Constants that need libm (the polygon half-planes, the
// "random" shape's bump field) are evaluated on the host once, so both sides
// test points with the same values.
#pragma once

#include <cstdint>

namespace tacchi_b200 {

enum ShapeId : int {
  kShSphere = 0, kShSphere2, kShCone, kShCylinder, kShCylinderShell, kShCylinderSide,
  kShCurvedSurface, kShFlatSlab, kShDotIn, kShDots, kShHexagon, kShTriangle, kShPrism, kShLine,
  kShParallelLines, kShCrossLines, kShMoon, kShPacman, kShTorus, kShWave1, kShRandom
};

struct ShapeTable {
  int id;
  double lo[3], span[3];  // sampling box (mm): lo + span * u
  // polygon / triangle half-planes: x cos(a_k) + y sin(a_k) > apothem -> outside
  int n_planes;
  double apothem;
  double ca[6], sa[6];
  // "random": h(x, y) = min(sum_i amp_i exp(-((x - cx_i)^2 + (y - cy_i)^2) inv_s2_i), 1.4)
  double bx[28], by[28], amp[28], inv_s2[28];
};

}  // namespace tacchi_b200
