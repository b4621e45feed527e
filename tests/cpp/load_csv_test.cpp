// C++ caller of gpkrylov::cuda::load_csv (include/gpkrylov_cuda.hpp) the way a reference user
// calls gpkrylov::load_csv (dataset.hpp:155-242).  Host only: runs without a GPU.
// usage: load_csv_test <path> <target> <standardize 0|1> <seed>; prints one JSON object
#include <cstdio>
#include <cstdlib>
#include <string>

#include "gpkrylov_cuda.hpp"

using namespace gpkrylov::cuda;

static void dump(const char* name, const Dataset& p, bool last) {
  std::printf("\"%s\": {\"n\": %lld, \"d\": %d, \"x\": [", name, static_cast<long long>(p.n), p.d);
  for (size_t i = 0; i < p.x.size(); ++i) std::printf("%s%.17g", i ? ", " : "", p.x[i]);
  std::printf("], \"y\": [");
  for (size_t i = 0; i < p.y.size(); ++i) std::printf("%s%.17g", i ? ", " : "", p.y[i]);
  std::printf("]}%s", last ? "" : ", ");
}

int main(int argc, char** argv) {
  if (argc < 5) return 2;
  try {
    const DataSplits s = load_csv(argv[1], argv[2], std::atoi(argv[3]) != 0, SplitFractions{},
                                  std::strtoull(argv[4], nullptr, 10));
    std::printf("{");
    dump("train", s.train, false);
    dump("validation", s.validation, false);
    dump("test", s.test, false);
    std::printf("\"standardized\": %s, \"target\": \"%s\", \"names\": [", s.standardized ? "true" : "false",
                s.target_name.c_str());
    for (size_t j = 0; j < s.feature_names.size(); ++j)
      std::printf("%s\"%s\"", j ? ", " : "", s.feature_names[j].c_str());
    std::printf("]}\n");
  } catch (const input_error& e) {
    std::printf("{\"input_error\": \"%s\"}\n", e.what());
    return 1;  // the reference CLI's exit code for input_error
  }
  return 0;
}
