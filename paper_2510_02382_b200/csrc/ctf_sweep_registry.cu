// Registry: concatenates the exact and guarded variant lists per precision.
#include "ctf_sweep_variants.h"
namespace ctf {
std::vector<SweepVariant> sweep_variants_f32_exact();
std::vector<SweepVariant> sweep_variants_f32_guard();
std::vector<SweepVariant> sweep_variants_f64_exact();
std::vector<SweepVariant> sweep_variants_f64_guard();
std::vector<SweepVariant> sweep_variants_rowwarp_f32();
std::vector<SweepVariant> sweep_variants_f32_taps();
std::vector<SweepVariant> sweep_variants_stream_f32();
std::vector<SweepVariant> sweep_variants_cluster_f32();
std::vector<SweepVariant> sweep_variants_cluster_f64();
std::vector<SweepVariant> sweep_variants_stream_f64();
std::vector<SweepVariant> sweep_variants_f64_taps();
std::vector<SweepVariant> sweep_variants_rowwarp_f64();
std::vector<SweepVariant> sweep_variants_check_f32();
std::vector<SweepVariant> sweep_variants_gram_f32();
std::vector<SweepVariant> sweep_variants_gram_f64();
std::vector<SweepVariant> sweep_variants_gram_ip();
std::vector<SweepVariant> sweep_variants_gram_more_f32();
std::vector<SweepVariant> sweep_variants_gram_more_f64();
std::vector<SweepVariant> sweep_variants_check_f64();
std::vector<SweepVariant> sweep_variants_fsplit_f32();
std::vector<SweepVariant> sweep_variants_ip_frame();
const std::vector<SweepVariant>& sweep_variants_f32() {
  static const std::vector<SweepVariant> v = [] {
    auto a = sweep_variants_rowwarp_f32();
    auto t = sweep_variants_f32_taps();
    a.insert(a.end(), t.begin(), t.end());
    auto e = sweep_variants_f32_exact();
    auto b = sweep_variants_f32_guard();
    a.insert(a.end(), e.begin(), e.end());
    a.insert(a.end(), b.begin(), b.end());
    auto st = sweep_variants_stream_f32();
    a.insert(a.end(), st.begin(), st.end());
    auto cl = sweep_variants_cluster_f32();
    a.insert(a.end(), cl.begin(), cl.end());
    auto ck = sweep_variants_check_f32();
    a.insert(a.end(), ck.begin(), ck.end());
    auto gr = sweep_variants_gram_f32();
    a.insert(a.end(), gr.begin(), gr.end());
    auto gm = sweep_variants_gram_more_f32();
    a.insert(a.end(), gm.begin(), gm.end());
    for (const auto& v : sweep_variants_gram_ip())
      if (v.prec == 1) a.push_back(v);
    for (const auto& v : sweep_variants_ip_frame())
      if (v.prec == 1) a.push_back(v);
    auto fs = sweep_variants_fsplit_f32();
    a.insert(a.end(), fs.begin(), fs.end());
    return a;
  }();
  return v;
}
const std::vector<SweepVariant>& sweep_variants_f64() {
  static const std::vector<SweepVariant> v = [] {
    auto a = sweep_variants_rowwarp_f64();
    auto t = sweep_variants_f64_taps();
    a.insert(a.end(), t.begin(), t.end());
    auto e = sweep_variants_f64_exact();
    auto b = sweep_variants_f64_guard();
    a.insert(a.end(), e.begin(), e.end());
    a.insert(a.end(), b.begin(), b.end());
    auto st = sweep_variants_stream_f64();
    a.insert(a.end(), st.begin(), st.end());
    auto cl = sweep_variants_cluster_f64();
    a.insert(a.end(), cl.begin(), cl.end());
    auto ck = sweep_variants_check_f64();
    a.insert(a.end(), ck.begin(), ck.end());
    auto gr = sweep_variants_gram_f64();
    a.insert(a.end(), gr.begin(), gr.end());
    auto gm = sweep_variants_gram_more_f64();
    a.insert(a.end(), gm.begin(), gm.end());
    for (const auto& v : sweep_variants_gram_ip())
      if (v.prec == 0) a.push_back(v);
    for (const auto& v : sweep_variants_ip_frame())
      if (v.prec == 0) a.push_back(v);
    return a;
  }();
  return v;
}
}  // namespace ctf
