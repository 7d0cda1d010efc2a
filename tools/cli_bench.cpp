// In-process `archetype unmix` timing: cli_main called R times per mode in one
// process (device context and solve graph warm after the first call), wall
// clock around each call — load .npy, validate + ℓ2-normalise (device ingest,
// or the host fp64 route with ARCHETYPE_HOST_NORMALIZE=1), the batched GPU
// ensemble, selection, and writing the bundle.
//   g++ -std=c++20 -O2 -Iinclude tools/cli_bench.cpp -Lpaper_2209_11002_b200 -larchetype_b200 \
//       -ledaa_cuda -Wl,-rpath,$PWD/paper_2209_11002_b200 -o /tmp/cli_bench
//   /tmp/cli_bench CUBE.npy P RUNS OUTDIR R
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <sstream>
#include <string>
#include <vector>

#include "archetype/cli.hpp"

int main(int argc, char** argv) {
  if (argc < 6) return 64;
  const std::string cube = argv[1], p = argv[2], runs = argv[3], out = argv[4];
  const int reps = std::atoi(argv[5]);
  for (const char* mode : {"0", "1", "0", "1"}) {
    setenv("ARCHETYPE_HOST_NORMALIZE", mode, 1);
    std::vector<double> ms;
    for (int r = 0; r < reps; ++r) {
      std::ostringstream so, se;
      const auto t0 = std::chrono::steady_clock::now();
      const int rc = archetype::cli_main({"unmix", "--input", cube, "--endmembers", p, "--runs", runs,
                                          "--output", out + "/m" + mode}, so, se);
      ms.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
      if (rc != 0) {
        std::fprintf(stderr, "%s", se.str().c_str());
        return rc;
      }
    }
    std::sort(ms.begin(), ms.end());
    std::printf("{\"host_normalize\": %s, \"median_ms\": %.2f, \"min_ms\": %.2f, \"max_ms\": %.2f, \"reps\": %d}\n",
                mode, ms[ms.size() / 2], ms.front(), ms.back(), reps);
  }
  return 0;
}
