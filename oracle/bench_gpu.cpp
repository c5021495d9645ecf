// bench_gpu.cpp — TEST INFRASTRUCTURE: the reference's `soaview bench` (tools/soaview.cpp:
// 341-410, cmd_bench) without its CLI11 / nlohmann dependencies, which are not vendored.
// oracle/Makefile links it with the UNMODIFIED reference bench.cpp / grid.cpp / layout.cpp
// and the GPU drop-in paper_2502_16517_b200/dropin/kernels_gpu.cpp in place of kernels.cpp,
// so the reference's own run_bench -> to_csv harness times the B200 path.
//   bench_gpu [--kernel density,force] [--variant soa-view,scattered,...]... [--ppc N]...
//             [--particles N] [--reps N] [--seed N]
// Exit codes follow cmd_bench: 0 ok, 2 usage / configuration errors.
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <sstream>
#include <string>
#include <vector>

#include "soaview/sph/bench.hpp"

using namespace soaview::sph;

int main(int argc, char **argv) {
  BenchConfig cfg;
  cfg.kernels.clear();
  std::vector<VariantSpec> variants;
  std::vector<int> ppcs;
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    if (i + 1 >= argc) {
      std::fprintf(stderr, "bench_gpu: %s needs a value\n", a.c_str());
      return 2;
    }
    const std::string v = argv[++i];
    if (a == "--kernel") {
      std::stringstream ss(v);
      std::string name;
      while (std::getline(ss, name, ',')) {
        bool found = false;
        for (KernelId k : {KernelId::Density, KernelId::Force, KernelId::Drift, KernelId::Kick1,
                           KernelId::Kick2})
          if (name == kernel_name(k)) {
            cfg.kernels.push_back(k);
            found = true;
          }
        if (!found) {
          std::fprintf(stderr, "bench_gpu: unknown kernel '%s'\n", name.c_str());
          return 2;
        }
      }
    } else if (a == "--variant") {
      std::string err;
      auto p = parse_variant(v, err);
      if (!p) {
        std::fprintf(stderr, "bench_gpu: %s\n", err.c_str());
        return 2;
      }
      variants.push_back(*p);
    } else if (a == "--ppc") {
      ppcs.push_back(std::atoi(v.c_str()));
    } else if (a == "--particles") {
      cfg.particles = std::atoll(v.c_str());
    } else if (a == "--reps") {
      cfg.reps = std::atoi(v.c_str());
    } else if (a == "--seed") {
      cfg.seed = std::strtoull(v.c_str(), nullptr, 10);
    } else {
      std::fprintf(stderr, "bench_gpu: unknown option %s\n", a.c_str());
      return 2;
    }
  }
  if (cfg.kernels.empty())
    cfg.kernels = {KernelId::Density, KernelId::Force, KernelId::Drift, KernelId::Kick1,
                   KernelId::Kick2};
  if (variants.empty()) { // cmd_bench's default: aos-baseline and soa-view
    variants.push_back(VariantSpec{});
    VariantSpec s;
    s.path = Path::SoaView;
    variants.push_back(s);
  }
  cfg.variants = variants;
  if (!ppcs.empty()) cfg.ppcs = ppcs;
  std::vector<BenchRecord> records;
  try {
    records = run_bench(cfg);
  } catch (const std::exception &e) {
    std::fprintf(stderr, "bench_gpu: %s\n", e.what());
    return 2;
  }
  std::fputs(to_csv(records).c_str(), stdout);
  // the cross-check the reference records per soa-view row (bench.hpp:64-65), on stderr so
  // stdout stays the reference's CSV
  for (const BenchRecord &r : records)
    if (r.variant.path == Path::SoaView)
      std::fprintf(stderr, "cross_max_rel %s %s %.3e\n", kernel_name(r.kernel),
                   variant_string(r.variant).c_str(), r.cross_max_rel);
  return 0;
}
