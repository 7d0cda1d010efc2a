// TEST INFRASTRUCTURE. One driver over the public API of the formats and
// scoring either side of the solver (npy / envi / csv / report.json / output
// bundle / metrics / synth). It is compiled twice from this one source:
//   tests/cpp/build/io_tool      against OUR headers + libarchetype_b200.so
//   oracle/_ref/io_tool_ref      against the reference headers + the
//                                reference's own sources (namespace renamed)
// and tests/test_io_parity.py runs both on the same inputs and compares their
// stdout and every file they write byte for byte.
//
//   io_tool synth L N p alpha pure seed snr|- outdir   generate + write fixture
//   io_tool npy PATH                                    read_npy → summary or error
//   io_tool image PATH                                  npy_to_image / read_envi → summary
//   io_tool csv PATH                                    read_csv_endmembers → values
//   io_tool evaluate EST_DIR GT_E GT_A                  evaluation_to_json + table
//   io_tool bundle REPORT_JSON E.npy A.npy OUTDIR       report_from_json → write_outputs
//   io_tool writenpy OUT f4|f8 d0 [d1 ...]              write_npy of 0.1·i values
#include <cstdio>
#include <cstring>
#include <exception>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "archetype/envi.hpp"
#include "archetype/error.hpp"
#include "archetype/metrics.hpp"
#include "archetype/npy.hpp"
#include "archetype/outputs.hpp"
#include "archetype/synth.hpp"

using namespace archetype;

namespace {

void print_values(const std::vector<double>& v) {
  char buf[40];
  for (std::size_t i = 0; i < v.size(); ++i) {
    std::snprintf(buf, sizeof buf, "%a", v[i]);
    std::cout << buf << (i + 1 < v.size() ? " " : "\n");
  }
}

void print_matrix(const Matrix& m) {
  std::cout << m.rows() << "x" << m.cols() << "\n";
  print_values(std::vector<double>(m.values().begin(), m.values().end()));
}

bool ends_with(const std::string& s, const char* suf) {
  const std::size_t n = std::strlen(suf);
  return s.size() >= n && s.compare(s.size() - n, n, suf) == 0;
}

std::string slurp(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  std::ostringstream s;
  s << in.rdbuf();
  return s.str();
}

int dispatch(const std::vector<std::string>& a) {
  const std::string& cmd = a.at(0);
  if (cmd == "synth") {
    SynthSpec spec;
    spec.bands = std::stoul(a.at(1));
    spec.pixels = std::stoul(a.at(2));
    spec.endmembers = std::stoul(a.at(3));
    spec.dirichlet_alpha = std::stod(a.at(4));
    spec.pure_pixels = a.at(5) == "1";
    spec.seed = std::stoull(a.at(6));
    if (a.at(7) != "-") spec.snr_db = std::stod(a.at(7));
    const SynthData d = generate(spec);
    const std::string dir = a.at(8);
    const std::size_t xs[2] = {d.image.data.rows(), d.image.data.cols()};
    write_npy(dir + "/cube.npy", xs, d.image.data.values());
    const std::size_t as[2] = {d.abundances.data.rows(), d.abundances.data.cols()};
    write_npy(dir + "/abundances.npy", as, d.abundances.data.values(), NpyDtype::f4);
    write_csv_endmembers(dir + "/endmembers.csv", d.endmembers.data);
    return 0;
  }
  if (cmd == "npy") {
    const NpyArray arr = read_npy(a.at(1));
    std::cout << (arr.dtype == NpyDtype::f4 ? "f4" : "f8") << " shape";
    for (std::size_t d : arr.shape) std::cout << " " << d;
    std::cout << "\n";
    print_values(arr.values);
    return 0;
  }
  if (cmd == "image") {
    const std::string& p = a.at(1);
    const HsiImage img = ends_with(p, ".hdr") ? read_envi(p, envi_data_path(p)) : npy_to_image(read_npy(p));
    if (img.spatial) std::cout << "spatial " << img.spatial->height << " " << img.spatial->width << "\n";
    std::cout << "wavelengths " << img.wavelengths.size() << "\n";
    print_values(img.wavelengths);
    print_matrix(img.data);
    return 0;
  }
  if (cmd == "csv") {
    print_matrix(read_csv_endmembers(a.at(1)));
    return 0;
  }
  if (cmd == "evaluate") {
    const EndmemberMatrix est_e{read_csv_endmembers(a.at(1) + "/endmembers.csv")};
    const AbundanceMatrix est_a{npy_to_matrix(read_npy(a.at(1) + "/abundances.npy"))};
    const EndmemberMatrix gt_e{ends_with(a.at(2), ".csv") ? read_csv_endmembers(a.at(2))
                                                         : npy_to_matrix(read_npy(a.at(2)))};
    const AbundanceMatrix gt_a{npy_to_matrix(read_npy(a.at(3)))};
    const EvaluationResult r = evaluate_unmixing(gt_e, gt_a, est_e, est_a);
    std::cout << evaluation_to_json(r) << format_evaluation(r);
    std::cout << "sad_degrees " << sad_degrees(gt_e, est_e) << "\n";
    return 0;
  }
  if (cmd == "bundle") {
    const RunReport report = report_from_json(slurp(a.at(1)));
    RunResult result;
    result.endmembers.data = npy_to_matrix(read_npy(a.at(2)));
    result.abundances.data = npy_to_matrix(read_npy(a.at(3)));
    write_outputs(a.at(4), result, report);
    std::cout << report_to_json(report);
    return 0;
  }
  if (cmd == "writenpy") {
    std::vector<std::size_t> shape;
    for (std::size_t i = 3; i < a.size(); ++i) shape.push_back(std::stoul(a[i]));
    std::size_t n = 1;
    for (std::size_t d : shape) n *= d;
    std::vector<double> v(n);
    for (std::size_t i = 0; i < n; ++i) v[i] = 0.1 * static_cast<double>(i);
    write_npy(a.at(1), shape, v, a.at(2) == "f4" ? NpyDtype::f4 : NpyDtype::f8);
    return 0;
  }
  std::cerr << "unknown command " << cmd << "\n";
  return 64;
}

}  // namespace

int main(int argc, char** argv) {
  std::vector<std::string> args(argv + 1, argv + argc);
  if (args.empty()) return 64;
  try {
    return dispatch(args);
  } catch (const Error& e) {
    std::cout << "Error: " << e.what() << "\n";
    return 3;
  } catch (const std::exception& e) {
    std::cout << "exception: " << e.what() << "\n";
    return 4;
  }
}
