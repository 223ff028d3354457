// b200_grid: the reference's `bench` grid (17-column CSV + JSON manifest,
// bench.hpp:156-176) with the B200 operator registered as method "b200".
//
//   b200_grid [--methods b200,tiled] [--s 512,1024] [--d 64,128]
//             [--dtypes f16,bf16] [--masks none,causal] [--b 1] [--h 8]
//             [--warmup 10] [--timed 50] [--seed 0] [--out out]
//
// Writes <out>/results.csv and <out>/manifest.json through the reference's
// write_records / write_manifest, so its `report` tooling reads them as is.
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <sstream>
#include <string>
#include <vector>

#include "b200_method.hpp"

namespace {

std::vector<std::string> split(const std::string& s) {
  std::vector<std::string> out;
  std::stringstream ss(s);
  std::string item;
  while (std::getline(ss, item, ','))
    if (!item.empty()) out.push_back(item);
  return out;
}

std::vector<int64_t> ints(const std::string& s) {
  std::vector<int64_t> out;
  for (const auto& x : split(s)) out.push_back(std::stoll(x));
  return out;
}

}  // namespace

int main(int argc, char** argv) {
  tileattn::GridConfig cfg;
  cfg.methods = {tileattn_b200_harness::kMethodName, "tiled"};
  cfg.dtypes = {tileattn::DType::F16Emu, tileattn::DType::BF16Emu};
  for (int i = 1; i + 1 < argc; i += 2) {
    const std::string key = argv[i], val = argv[i + 1];
    if (key == "--methods") cfg.methods = split(val);
    else if (key == "--s") cfg.s_values = ints(val);
    else if (key == "--d") cfg.d_values = ints(val);
    else if (key == "--b") cfg.b = std::stoll(val);
    else if (key == "--h") cfg.h = std::stoll(val);
    else if (key == "--warmup") cfg.n_warmup = std::stoi(val);
    else if (key == "--timed") cfg.n_timed = std::stoi(val);
    else if (key == "--seed") cfg.seed = std::stoull(val);
    else if (key == "--out") cfg.out_dir = val;
    else if (key == "--dtypes") {
      cfg.dtypes.clear();
      for (const auto& x : split(val)) cfg.dtypes.push_back(tileattn::dtype_from_string(x));
    } else if (key == "--masks") {
      cfg.masks.clear();
      for (const auto& x : split(val)) cfg.masks.push_back(tileattn::mask_kind_from_string(x));
    } else {
      std::fprintf(stderr, "unknown option %s\n", key.c_str());
      return 2;
    }
  }
  try {
    const tileattn::RunResult res = tileattn_b200_harness::run_grid_b200(cfg);
    std::filesystem::create_directories(cfg.out_dir);
    tileattn::write_records(res.records, cfg.out_dir + "/results.csv");
    tileattn::write_manifest(res.manifest, cfg.out_dir + "/manifest.json");
    int ok = 0;
    for (const auto& r : res.records) ok += r.status == tileattn::BenchStatus::Ok;
    std::printf("%zu grid points, %d ok -> %s/results.csv\n", res.records.size(), ok,
                cfg.out_dir.c_str());
  } catch (const std::exception& e) {
    std::fprintf(stderr, "b200_grid: %s\n", e.what());
    return 1;
  }
  return 0;
}
