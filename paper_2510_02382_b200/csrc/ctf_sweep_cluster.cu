// Cluster sweep kernels (ctf_cluster.cuh): on-chip tiles spread over a
// thread-block cluster (BASELINE cfg3 R=32: 4 x 8 rows; cfg4 R=60: 15 x 4 rows).
#include "ctf_sweep_variants.h"
namespace ctf {
std::vector<SweepVariant> sweep_variants_cluster_f32() {
  return {CTF_CL(float, 1, 8, 4, 4, 256), CTF_CL(float, 1, 4, 8, 0, 512), CTF_CL(float, 1, 4, 4, 2, 256),
          CTF_CL(float, 1, 6, 8, 0, 512), CTF_CL(float, 1, 8, 8, 0, 512), CTF_CL(float, 1, 16, 4, 4, 256)};
}
std::vector<SweepVariant> sweep_variants_cluster_f64() {
  return {CTF_CL(double, 0, 8, 4, 2, 256), CTF_CL(double, 0, 4, 8, 0, 512), CTF_CL(double, 0, 4, 4, 1, 256)};
}
}  // namespace ctf
