// CSV dataset ingestion for the training / validation / test callers of the hot path
// (SURVEY §8(f) row 4): gpk_load_csv and its accessors in include/gpkrylov_cuda.h.
//
// Follows the reference's load_csv (proj/include/gpkrylov/dataset.hpp:155-242) over
// read_csv_table / split_csv_line (proj/include/gpkrylov/csv.hpp:76-116):
//  * '#' lines and empty lines are skipped, a trailing '\r' is dropped, cells are split
//    on ',' and trimmed of " \t\r", a trailing ',' adds an empty cell;
//  * the first row is the header and must not be all-numeric; cells parse with std::stod
//    and must be consumed whole (dataset.hpp:121-132);
//  * rows are shuffled by Fisher-Yates with std::mt19937_64(seed) and
//    std::uniform_int_distribution<Index>(0, i) (libstdc++: Lemire's nearly divisionless
//    downscaling over 128-bit products), split by llround(fraction * n) in the order
//    train, validation, test (dataset.hpp:185-206);
//  * standardisation uses population statistics of the training split only
//    (dataset.hpp:214-238; Standardizer dataset.hpp:87-101).
// Error order and texts are the reference's (the first bad row wins, as in its serial loop).
//
// Layout: every split is stored column-major (n x d, ld = n) in fp64, the form gpk_set_data
// takes.  Parsing runs on all host threads (rows are independent); the shuffle is the
// serial RNG stream, as the reference's.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <memory>
#include <numeric>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "gpkrylov_cuda.h"

namespace {

struct input_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void require(bool ok, const std::string& msg) {
  if (!ok) throw input_error(msg);
}

struct Part {
  int64_t n = 0;
  std::vector<double> x;  // n x d col-major
  std::vector<double> y;
};

}  // namespace

struct gpk_dataset {
  int d = 0;
  Part part[3];
  int standardized = 0;
  std::vector<double> feature_mean, feature_std;
  double target_mean = 0.0, target_std = 1.0;
  std::vector<std::string> feature_names;
  std::string target_name;
};

namespace {

// csv.hpp:76-89
void split_line(const char* b, const char* e, std::vector<std::string>& cells) {
  cells.clear();
  const char* s = b;
  auto push = [&](const char* cb, const char* ce) {
    while (cb < ce && (*cb == ' ' || *cb == '\t' || *cb == '\r')) ++cb;
    while (ce > cb && (ce[-1] == ' ' || ce[-1] == '\t' || ce[-1] == '\r')) --ce;
    cells.emplace_back(cb, ce);
  };
  for (const char* p = b; p < e; ++p)
    if (*p == ',') {
      push(s, p);
      s = p + 1;
    }
  if (s < e) push(s, e);                 // getline yields the last field only when non-empty
  if (e > b && e[-1] == ',') cells.emplace_back();  // csv.hpp:87
}

bool parse_whole(const std::string& c, double* v) {
  try {
    std::size_t pos = 0;
    *v = std::stod(c, &pos);
    return pos == c.size();
  } catch (const std::exception&) {
    return false;
  }
}

std::vector<std::pair<const char*, const char*>> data_lines(const std::string& buf) {
  std::vector<std::pair<const char*, const char*>> lines;
  const char* p = buf.data();
  const char* end = p + buf.size();
  while (p < end) {
    const char* q = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(end - p)));
    const char* le = q ? q : end;
    const char* ce = le;
    if (ce > p && ce[-1] == '\r') --ce;   // csv.hpp:99
    if (ce > p && *p != '#') lines.emplace_back(p, ce);  // empty and comment lines skipped (:100-105)
    p = q ? q + 1 : end;
  }
  return lines;
}

gpk_dataset* load(const char* path, const char* target_column, int standardize, double ftrain, double fval,
                  double ftest, uint64_t seed) {
  const std::string spath = path ? path : "";
  std::ifstream in(spath, std::ios::binary);
  if (!in) throw input_error("read_csv_table: cannot open " + spath);
  std::stringstream ss;
  ss << in.rdbuf();
  const std::string buf = ss.str();
  const auto lines = data_lines(buf);

  std::vector<std::string> header;
  if (!lines.empty()) split_line(lines[0].first, lines[0].second, header);
  if (header.empty()) throw input_error("load_csv: " + spath + " is empty");
  {
    bool all = true;
    double v;
    for (const auto& c : header) all = all && parse_whole(c, &v);
    if (all) throw input_error("load_csv: " + spath + " has no header row");
  }
  require(ftrain >= 0 && fval >= 0 && ftest >= 0 && ftrain + fval + ftest <= 1.0 + 1e-9,
          "load_csv: split fractions must be nonnegative and sum to at most 1");
  const std::string tname = target_column ? target_column : "";
  int target = -1;
  for (size_t i = 0; i < header.size(); ++i)
    if (header[i] == tname) {
      target = static_cast<int>(i);
      break;
    }
  if (target < 0) throw input_error("CsvTable: no column named '" + tname + "'");
  const int64_t n = static_cast<int64_t>(lines.size()) - 1;
  require(n >= 1, "load_csv: no data rows in " + spath);
  const int ncols = static_cast<int>(header.size());
  const int d = ncols - 1;
  require(d >= 1, "load_csv: need at least one feature column");

  // parse: row-major staging x_rm (n x d) and y; every worker keeps its first failing row
  std::vector<double> xrm(static_cast<size_t>(n) * d), y(static_cast<size_t>(n));
  const int nth = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(std::thread::hardware_concurrency(),
                                                                          (n + 4095) / 4096)));
  std::vector<int64_t> bad_row(nth, -1);
  std::vector<std::string> bad_msg(nth);
  auto work = [&](int w) {
    const int64_t a = n * w / nth, b = n * (w + 1) / nth;
    std::vector<std::string> cells;
    for (int64_t i = a; i < b; ++i) {
      const auto& ln = lines[static_cast<size_t>(i + 1)];
      split_line(ln.first, ln.second, cells);
      if (static_cast<int>(cells.size()) != ncols) {
        bad_row[w] = i;
        bad_msg[w] = "load_csv: data row " + std::to_string(i + 1) + " has " + std::to_string(cells.size()) +
                     " cells, expected " + std::to_string(ncols);
        return;
      }
      int fc = 0;
      for (int c = 0; c < ncols; ++c) {
        double v;
        if (!parse_whole(cells[static_cast<size_t>(c)], &v)) {
          bad_row[w] = i;
          bad_msg[w] = "load_csv: non-numeric cell '" + cells[static_cast<size_t>(c)] + "' at data row " +
                       std::to_string(i + 1) + ", column " + std::to_string(c + 1);
          return;
        }
        if (c == target)
          y[static_cast<size_t>(i)] = v;
        else
          xrm[static_cast<size_t>(i) * d + fc++] = v;
      }
    }
  };
  {
    std::vector<std::thread> th;
    for (int w = 1; w < nth; ++w) th.emplace_back(work, w);
    work(0);
    for (auto& t : th) t.join();
  }
  for (int w = 0; w < nth; ++w)  // workers own increasing row ranges: the first failing one is the reference's
    if (bad_row[w] >= 0) throw input_error(bad_msg[w]);

  // dataset.hpp:185-191: Fisher-Yates with the reference's RNG and distribution
  using Index = std::ptrdiff_t;  // Eigen::Index
  std::vector<Index> order(static_cast<size_t>(n));
  std::iota(order.begin(), order.end(), Index{0});
  std::mt19937_64 rng(seed);
  for (Index i = n - 1; i > 0; --i) {
    std::uniform_int_distribution<Index> pick(0, i);
    std::swap(order[static_cast<size_t>(i)], order[static_cast<size_t>(pick(rng))]);
  }
  const auto nt = static_cast<size_t>(n);
  const size_t n_train = std::min(nt, static_cast<size_t>(std::llround(ftrain * static_cast<double>(n))));
  const size_t n_val = std::min(nt - n_train, static_cast<size_t>(std::llround(fval * static_cast<double>(n))));
  const size_t n_test =
      std::min(nt - n_train - n_val, static_cast<size_t>(std::llround(ftest * static_cast<double>(n))));

  auto* ds = new gpk_dataset();
  ds->d = d;
  ds->target_name = tname;
  for (int c = 0; c < ncols; ++c)
    if (c != target) ds->feature_names.push_back(header[static_cast<size_t>(c)]);
  const size_t begin[3] = {0, n_train, n_train + n_val}, count[3] = {n_train, n_val, n_test};
  for (int s = 0; s < 3; ++s) {  // detail::take_rows (dataset.hpp:136-147), gathered column-major
    Part& p = ds->part[s];
    p.n = static_cast<int64_t>(count[s]);
    p.x.resize(count[s] * d);
    p.y.resize(count[s]);
    for (size_t i = 0; i < count[s]; ++i) {
      const size_t r = static_cast<size_t>(order[begin[s] + i]);
      for (int j = 0; j < d; ++j) p.x[static_cast<size_t>(j) * count[s] + i] = xrm[r * d + j];
      p.y[i] = y[r];
    }
  }

  if (standardize) {
    std::unique_ptr<gpk_dataset> guard(ds);
    const Part& tr = ds->part[0];
    require(tr.n >= 2, "load_csv: standardization needs at least two training rows");
    const double m = static_cast<double>(tr.n);
    ds->feature_mean.assign(d, 0.0);
    ds->feature_std.assign(d, 0.0);
    for (int j = 0; j < d; ++j) {
      const double* col = tr.x.data() + static_cast<size_t>(j) * tr.n;
      double s = 0.0;
      for (int64_t i = 0; i < tr.n; ++i) s += col[i];
      const double mu = s / m;
      double q = 0.0;
      for (int64_t i = 0; i < tr.n; ++i) q += (col[i] - mu) * (col[i] - mu);
      ds->feature_mean[j] = mu;
      ds->feature_std[j] = std::sqrt(q / m);
      if (!(ds->feature_std[j] > 1e-12))
        throw input_error("load_csv: column '" + ds->feature_names[static_cast<size_t>(j)] +
                          "' is constant on the training split; cannot standardize");
    }
    double s = 0.0;
    for (int64_t i = 0; i < tr.n; ++i) s += tr.y[i];
    ds->target_mean = s / m;
    double q = 0.0;
    for (int64_t i = 0; i < tr.n; ++i) q += (tr.y[i] - ds->target_mean) * (tr.y[i] - ds->target_mean);
    ds->target_std = std::sqrt(q / m);
    if (!(ds->target_std > 1e-12))
      throw input_error("load_csv: target column '" + tname +
                        "' is constant on the training split; cannot standardize");
    for (Part& p : ds->part) {
      for (int j = 0; j < d; ++j) {
        double* col = p.x.data() + static_cast<size_t>(j) * p.n;
        for (int64_t i = 0; i < p.n; ++i) col[i] = (col[i] - ds->feature_mean[j]) / ds->feature_std[j];
      }
      for (auto& v : p.y) v = (v - ds->target_mean) / ds->target_std;
    }
    ds->standardized = 1;
    guard.release();
  }
  return ds;
}

void set_err(char* err, int64_t errlen, const std::string& msg) {
  if (!err || errlen <= 0) return;
  const size_t k = std::min(static_cast<size_t>(errlen - 1), msg.size());
  std::memcpy(err, msg.data(), k);
  err[k] = '\0';
}

}  // namespace

extern "C" {

gpk_status gpk_load_csv(const char* path, const char* target_column, int standardize, double train_fraction,
                        double validation_fraction, double test_fraction, uint64_t seed, gpk_dataset** out,
                        char* err, int64_t errlen) {
  set_err(err, errlen, "");
  if (!out) {
    set_err(err, errlen, "gpk_load_csv: null output handle");
    return GPK_INPUT_ERROR;
  }
  *out = nullptr;
  try {
    *out = load(path, target_column, standardize, train_fraction, validation_fraction, test_fraction, seed);
    return GPK_OK;
  } catch (const input_error& e) {
    set_err(err, errlen, e.what());
    return GPK_INPUT_ERROR;
  } catch (const std::exception& e) {
    set_err(err, errlen, std::string("load_csv: ") + e.what());
    return GPK_INPUT_ERROR;
  }
}

void gpk_dataset_free(gpk_dataset* ds) { delete ds; }

gpk_status gpk_dataset_shape(const gpk_dataset* ds, int split, int64_t* n, int* d) {
  if (!ds || split < 0 || split > 2) return GPK_INPUT_ERROR;
  if (n) *n = ds->part[split].n;
  if (d) *d = ds->d;
  return GPK_OK;
}

gpk_status gpk_dataset_copy(const gpk_dataset* ds, int split, double* X, int64_t ldx, double* y) {
  if (!ds || split < 0 || split > 2) return GPK_INPUT_ERROR;
  const Part& p = ds->part[split];
  if (X) {
    if (ldx < p.n) return GPK_INPUT_ERROR;
    for (int j = 0; j < ds->d; ++j)
      std::memcpy(X + static_cast<size_t>(j) * ldx, p.x.data() + static_cast<size_t>(j) * p.n,
                  sizeof(double) * static_cast<size_t>(p.n));
  }
  if (y && p.n) std::memcpy(y, p.y.data(), sizeof(double) * static_cast<size_t>(p.n));
  return GPK_OK;
}

gpk_status gpk_dataset_stats(const gpk_dataset* ds, int* standardized, double* feature_mean, double* feature_std,
                             double* target_mean, double* target_std) {
  if (!ds) return GPK_INPUT_ERROR;
  if (standardized) *standardized = ds->standardized;
  for (int j = 0; j < ds->d; ++j) {
    if (feature_mean) feature_mean[j] = ds->standardized ? ds->feature_mean[j] : 0.0;
    if (feature_std) feature_std[j] = ds->standardized ? ds->feature_std[j] : 1.0;
  }
  if (target_mean) *target_mean = ds->target_mean;
  if (target_std) *target_std = ds->target_std;
  return GPK_OK;
}

const char* gpk_dataset_column_name(const gpk_dataset* ds, int column) {
  if (!ds) return nullptr;
  if (column < 0) return ds->target_name.c_str();
  if (column >= ds->d) return nullptr;
  return ds->feature_names[static_cast<size_t>(column)].c_str();
}

gpk_status gpk_dataset_invert(const gpk_dataset* ds, double* X, int64_t n, int64_t ldx, double* y) {
  if (!ds || n < 0 || (X && ldx < n)) return GPK_INPUT_ERROR;
  if (!ds->standardized) return GPK_OK;
  if (X)
    for (int j = 0; j < ds->d; ++j)
      for (int64_t i = 0; i < n; ++i) {
        double& v = X[static_cast<size_t>(j) * ldx + i];
        v = v * ds->feature_std[j] + ds->feature_mean[j];
      }
  if (y)
    for (int64_t i = 0; i < n; ++i) y[i] = y[i] * ds->target_std + ds->target_mean;
  return GPK_OK;
}

}  // extern "C"
