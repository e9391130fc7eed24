// Cluster sweep kernels (ctf_cluster.cuh): on-chip tiles spread over a
// thread-block cluster (BASELINE cfg3 R=32: 4 x 8 rows; cfg4 R=60: 15 x 4 rows).
// Measured slower than the kernels the planner prefers for every BASELINE shape
// (DESIGN.md §4): compiled only in dev builds (make DEVK=1), kept for A/B.
#include "ctf_sweep_variants.h"
namespace ctf {
std::vector<SweepVariant> sweep_variants_cluster_f32() {
#ifdef CTF_DEV_KERNELS
  return {CTF_CL(float, 1, 8, 4, 4, 256), CTF_CL(float, 1, 4, 8, 0, 512), CTF_CL(float, 1, 4, 4, 2, 256),
          CTF_CL(float, 1, 6, 8, 0, 512), CTF_CL(float, 1, 8, 8, 0, 512), CTF_CL(float, 1, 16, 4, 4, 256)};
#else
  return {};
#endif
}
std::vector<SweepVariant> sweep_variants_cluster_f64() {
#ifdef CTF_DEV_KERNELS
  return {CTF_CL(double, 0, 8, 4, 2, 256), CTF_CL(double, 0, 4, 8, 0, 512), CTF_CL(double, 0, 4, 4, 1, 256)};
#else
  return {};
#endif
}
}  // namespace ctf
