// harness_adapter.cpp — the reference's OWN benchmark harness timing the B200
// library.
//
// The reference has no FFI.  Its one injection point is the
// std::function<void(std::span<std::int64_t>)> sort_fn that measure_loop times
// (/root/reference/proj/include/netsort/bench.hpp:58-61; run_benchmark binds
// it to run_variant at src/bench.cpp:94-96).  This driver hands measure_loop a
// sort_fn that calls netsort_b200::run_variant.  That is the library's
// int64 host-span overload: H2D, sort on the GPU, D2H, all inside the timed
// call, exactly like a CPU sort of the same span.  The reference's own
// run_benchmark then measures its Classic CPU baselines.  compute_speedup
// pairs every GPU record with the CPU Classic record of the same cell, and
// emit_csv / emit_summary print CSV schema v1 (report.hpp:14-15).
//
// Integration infrastructure, not the product.  The reference's
// bench/report/config/datagen sources are compiled unmodified from
// /root/reference by oracle/Makefile (target `harness`) into
// oracle/_ref/harness_gpu, next to the other reference builds.
//
//   harness_gpu [--sizes 10000,100000,1000000] [--gpu-ms 100] [--cpu-ms 500]
//               [--csv path]
// GPU rows carry config names "B200:<config>"; their speedup column is
// T(CPU Classic) / T(GPU variant) for the same algorithm, distribution and size.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "netsort/bench.hpp"
#include "netsort/hybrid.hpp"
#include "netsort/report.hpp"

#include "netsort_b200.hpp"

namespace ref = netsort;
namespace gpu = netsort_b200;

static std::vector<std::size_t> parse_sizes(const char* s) {
  std::vector<std::size_t> out;
  std::stringstream ss(s);
  std::string tok;
  while (std::getline(ss, tok, ',')) out.push_back(std::stoull(tok));
  return out;
}

int main(int argc, char** argv) {
  std::vector<std::size_t> sizes = {10000, 100000, 1000000};
  int gpu_ms = 100, cpu_ms = 500;
  std::string csv_path;
  for (int i = 1; i < argc; ++i) {
    if (!std::strcmp(argv[i], "--sizes") && i + 1 < argc) sizes = parse_sizes(argv[++i]);
    else if (!std::strcmp(argv[i], "--gpu-ms") && i + 1 < argc) gpu_ms = std::atoi(argv[++i]);
    else if (!std::strcmp(argv[i], "--cpu-ms") && i + 1 < argc) cpu_ms = std::atoi(argv[++i]);
    else if (!std::strcmp(argv[i], "--csv") && i + 1 < argc) csv_path = argv[++i];
  }
  const ref::CampaignPlan grid = ref::default_campaign_plan();  // distributions + 24 variants
  std::vector<ref::BenchmarkRecord> records;
  std::vector<ref::SpeedupRecord> speedups;
  for (std::size_t size : sizes) {
    for (const ref::Distribution& dist : grid.distributions) {
      const ref::GenSpec spec{size, dist, grid.seed};
      const std::vector<std::int64_t> input = ref::generate(spec);
      // the reference's CPU Classic baselines, measured by its own run_benchmark
      ref::BenchmarkRecord base[2];
      for (int a = 0; a < 2; ++a) {
        const ref::SortVariant classic{a == 0 ? ref::Algorithm::merge_sort
                                              : ref::Algorithm::quick_sort,
                                       ref::classic_config()};
        base[a] = ref::run_benchmark(classic, spec, std::chrono::milliseconds(cpu_ms));
        records.push_back(base[a]);
      }
      // every bundled variant on the GPU through the same measure_loop
      for (const ref::SortVariant& v : grid.variants) {
        const gpu::NetworkConfig* cfg = gpu::find_config(v.config.name);
        if (!cfg) throw std::runtime_error("no GPU config named " + v.config.name);
        const gpu::SortVariant gv{v.algorithm == ref::Algorithm::merge_sort
                                      ? gpu::Algorithm::merge_sort
                                      : gpu::Algorithm::quick_sort,
                                  *cfg};
        const auto sort_fn = [&gv](std::span<std::int64_t> a) { gpu::run_variant(gv, a); };
        const ref::MeasureResult m =
            ref::measure_loop(sort_fn, input, std::chrono::milliseconds(gpu_ms));
        // the same bookkeeping as run_benchmark (bench.cpp:99-110)
        ref::BenchmarkRecord rec;
        rec.algorithm = v.algorithm;
        rec.config_name = "B200:" + v.config.name;
        rec.distribution = dist.kind;
        rec.size = size;
        rec.iterations = m.iterations;
        rec.total_ns = m.total_cpu_ns;
        rec.mean_ns = m.total_cpu_ns / static_cast<double>(m.iterations);
        rec.wall_mean_ns = m.total_wall_ns / static_cast<double>(m.iterations);
        rec.cpu_time_used = m.cpu_time_used;
        rec.iteration_cap_hit = m.cap_hit;
        // verify the GPU output against the reference's own sort of the input
        std::vector<std::int64_t> want(input), got(input);
        ref::run_variant(ref::SortVariant{v.algorithm, ref::classic_config()},
                         std::span<std::int64_t>(want));
        sort_fn(std::span<std::int64_t>(got));
        if (got != want) {
          std::fprintf(stderr, "MISMATCH %s %s size %zu\n", rec.config_name.c_str(),
                       std::string(ref::algorithm_name(v.algorithm)).c_str(), size);
          return 1;
        }
        records.push_back(rec);
        speedups.push_back(ref::compute_speedup(base[v.algorithm == ref::Algorithm::merge_sort ? 0 : 1],
                                                rec));
      }
    }
  }
  if (csv_path.empty()) ref::emit_csv(std::cout, records, speedups);
  else ref::emit_csv(csv_path, records, speedups);
  ref::emit_summary(std::cout, speedups);
  return 0;
}
